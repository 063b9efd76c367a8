"""D2H of 800 MB into pinned memory: one copy vs chunks on 1 / 2 / 4 streams."""
import time
import torch
nbytes = 800_000_000
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(4)]
def run(nchunks, nstreams):
    torch.cuda.synchronize()
    t = time.perf_counter()
    step = nbytes // nchunks
    for k in range(nchunks):
        s = streams[k % nstreams]
        with torch.cuda.stream(s):
            h[k * step:(k + 1) * step].copy_(d[k * step:(k + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t
for cfg in [(1, 1), (40, 1), (40, 2), (40, 4), (8, 2), (160, 2)]:
    run(*cfg)
    ts = [run(*cfg) for _ in range(5)]
    print(f"chunks {cfg[0]:4d} streams {cfg[1]}: {min(ts)*1e3:.2f} ms  {nbytes/min(ts)/1e9:.1f} GB/s")
