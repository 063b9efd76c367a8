"""Measure dense int8 (torch._int_mm -> cuBLASLt) and bf16 GEMM peaks on this GPU.

Same protocol as MEASURED_PEAKS.json's bf16 figure: 8192^3, best of 10,
CUDA events.  Prints one JSON line.
"""
import json
import torch

def best(fn, iters=10):
    fn(); torch.cuda.synchronize()
    out = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)

n = 8192
A = torch.randint(-4, 4, (n, n), dtype=torch.int8, device="cuda")
B = torch.randint(-4, 4, (n, n), dtype=torch.int8, device="cuda")
ms_i8 = best(lambda: torch._int_mm(A, B))
Ah, Bh = A.to(torch.bfloat16), B.to(torch.bfloat16)
ms_bf = best(lambda: Ah @ Bh)
print(json.dumps({"int8_tops_cublas": 2 * n**3 / ms_i8 / 1e9, "bf16_tflops": 2 * n**3 / ms_bf / 1e9,
                  "ms_int8": ms_i8, "ms_bf16": ms_bf, "n": n}))
