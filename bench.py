#!/usr/bin/env python
"""Benchmark: all-pairs binary MI throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A step is one pass of the hot path over one synthetic dataset of the chosen
BASELINE config (default config 3, N=100,000 x m=10,000, f64 MI): kernel 1
(unpack + column sums) and kernel 2+3 (tcgen05 int8 Gram with the fused MI
epilogue) on device-resident packed words, output left on the device
(sharded across ranks when N>1; the only collective is the broadcast of the
packed words).  Rank 0 prints one JSON line.  `value` is pair-samples/s
(N*m(m+1)/2 per step) over the whole job, timed with CUDA events, L2 flushed
between steps, max over ranks.  `e2e` is the same metric through the public
API with host (pinned) words in and the host MI matrix out.

`--impl reference` times the reference algorithm on the host CPU cores (the
C restatement in oracle/, OpenMP, all threads) on a bounded column sample of
the same workload; it is the driver's reference arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "all-pairs binary MI: N·m(m+1)/2 pair-samples/s, % int8 tensor roofline, 1–8 GPU"
UNIT = "pair-samples/s"
INT8_NOMINAL_TOPS = 4500.0  # B200 dense int8, datasheet
FP4_NOMINAL_TOPS = 9000.0   # B200 dense FP4 (tcgen05 kind::mxf4), datasheet


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0, help="target length of the CPU sample")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def pair_samples(n: int, m: int) -> float:
    return float(n) * m * (m + 1) / 2.0


def workload_name(cfg: int, n: int, m: int, out: str) -> str:
    desc = {1: "Bernoulli(0.5) + 2 all-zero + 2 all-one columns, seed 0",
            2: "p_c~U(0.05,0.95), 200 planted noisy copies (flip 0.1), seed 1",
            3: "Bernoulli(0.5), seed 2",
            4: "p_c~Beta(0.5,20), 1% noisy copies (flip 0.05), seed 3",
            5: "p_c~U(0.01,0.99), seed 4"}[cfg]
    return f"config {cfg}: N={n:,} x m={m:,} {desc}; {out} MI"


# ----------------------------------------------------------------- clocks
class NvmlSampler:
    """SM clock, power and clock-event reasons sampled through NVML every 2 ms
    on a background thread for exactly the timed region (the region is short:
    nvidia-smi's 50 ms loop would see only a sample or two)."""

    def __init__(self, gpu_index: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        self.samples = []
        self.stop_flag = threading.Event()
        self.thread = None

    def _run(self):
        nv = self.nv
        while not self.stop_flag.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0,
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        self.stop_flag.set()
        self.thread.join(timeout=5)
        nv = self.nv
        smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                "hw_power_brake_slowdown": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        reasons = sorted({name for _, _, r in self.samples for name, b in bits.items() if r & b})
        sm = [c for c, _, _ in self.samples]
        power = [w for _, w, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(sm), "samples_under_load": len(sm), "power_w_max": max(power) if power else None,
                "source": "NVML every 2 ms over the timed region"}


def make_sampler(gpu_index: int):
    try:
        return NvmlSampler(gpu_index)
    except Exception:
        return ClockSampler(gpu_index)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in Path(self.path).read_text().splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    smax.append(float(f[2]))
                    power.append(float(f[3]))
                except ValueError:
                    continue
                for name, val in zip(names, f[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
        finally:
            os.unlink(self.path)
        loaded = [s for s, p in zip(sm, power) if p > 250.0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(loaded),
                "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------- CPU legs
def cpu_sample(cfg: int, target_s: float, max_cols: int | None = None):
    """Time the C restatement of the reference on a column sample of the
    config, sized to ~target_s seconds.  Returns (value pair-samples/s, info)."""
    from oracle import oracle as O

    rec = O.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    threads = O.c_num_threads()
    rng = __import__("numpy").random.default_rng(1234)

    def run(ms):
        cols = sorted(rng.choice(m, ms, replace=False).tolist()) if ms < m else None
        words = O.c_generate_config_words(rec, cols)
        t0 = time.perf_counter()
        O.c_mi_all_pairs(words, n)
        return time.perf_counter() - t0

    ms = min(m, 256)
    t = run(ms)
    per_pair = t / pair_samples(1, ms)
    ms_target = int(math.sqrt(2.0 * target_s / max(per_pair, 1e-12)))
    ms_final = max(ms, min(m, ms_target, max_cols or m))
    t = run(ms_final)
    val = pair_samples(n, ms_final) / t
    return val, {"n_rows": n, "n_cols_sampled": ms_final, "seconds": t, "threads": threads}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    rec = O.config_recipe(args.config)
    n, m = rec["n"], rec["m"]
    threads = O.c_num_threads()
    # size one step to ~ (two minutes / (K + W)) of CPU work
    budget = max(0.25, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    per_pair_probe = None
    import numpy as np

    rng = np.random.default_rng(1234)
    probe_ms = min(m, 256)
    cols = sorted(rng.choice(m, probe_ms, replace=False).tolist()) if probe_ms < m else None
    w = O.c_generate_config_words(rec, cols)
    t0 = time.perf_counter()
    O.c_mi_all_pairs(w, n)
    per_pair_probe = (time.perf_counter() - t0) / pair_samples(1, probe_ms)
    ms = max(probe_ms, min(m, int(math.sqrt(2.0 * budget / per_pair_probe))))
    cols = sorted(rng.choice(m, ms, replace=False).tolist()) if ms < m else None
    words = O.c_generate_config_words(rec, cols)
    # the small probe misjudges a wide sample's cost (thread start-up, cache
    # effects): time one run at the chosen width and rescale the sample once
    t0 = time.perf_counter()
    O.c_mi_all_pairs(words, n)
    t_first = time.perf_counter() - t0
    if not 0.8 * budget <= t_first <= 1.2 * budget:
        ms = max(probe_ms, min(m, int(ms * math.sqrt(budget / t_first))))
        cols = sorted(rng.choice(m, ms, replace=False).tolist()) if ms < m else None
        words = O.c_generate_config_words(rec, cols)
    for _ in range(args.warmup):
        O.c_mi_all_pairs(words, n)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.c_mi_all_pairs(words, n)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    val = pair_samples(n, ms) / t
    out = "float32" if args.config == 4 else "float64"
    sample = (f"full-N column sample: {ms} of {m} columns x N={n:,} rows per step "
              f"(pair-samples/s scales with N*m_s(m_s+1)/2); reference algorithm restated in C "
              f"(oracle/mi_oracle.c), OpenMP {threads} threads, host {O.cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "popcount/int64+f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, n, m, out), "n_rows": n, "n_cols": m,
                   "n_cols_sampled": ms, "output": out},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2411_19702_b200 import EngineConfig, MIEngine, datagen
    from paper_2411_19702_b200 import dispatch as dsp

    rank, world, local = dist_env()
    # MI_B200_DIST_BACKEND=gloo (with ranks sharing GPUs) only exercises the
    # multi-rank code path on fewer GPUs; timings are meaningless then.
    backend = os.environ.get("MI_B200_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    eng = MIEngine.get(local)

    rec = datagen.config_recipe(args.config)
    n, m = rec["n"], rec["m"]
    out_name = datagen.CONFIGS[args.config]["out"]
    out_dtype = torch.float64 if out_name == "float64" else torch.float32
    cfg = EngineConfig()
    W = pair_samples(n, m)

    words_dev = datagen.generate_words_device(rec, dev) if rank == 0 else None
    out = torch.empty((m, m), dtype=out_dtype, device=dev)
    tiles = eng.tiles(m, rank, world)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    words_local = torch.empty((m, (n + 63) // 64), dtype=torch.int64, device=dev) if rank != 0 else words_dev

    def step(ev_k0=None, ev_k1=None):
        if world > 1:
            dist.broadcast(words_local, src=0)
        prep = eng.prepare(words_local, n, m, rank, world)  # this rank's column blocks only
        if ev_k0 is not None:
            ev_k0.record(stream)
        eng.compute(prep, cfg, out_dtype, tiles=tiles, out=out)
        if ev_k1 is not None:
            ev_k1.record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    sampler = make_sampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for s0, s1, k0, k1 in ev:
        flush.fill_(1)  # untimed L2 flush
        s0.record(stream)
        step(k0, k1)
        s1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    step_ms = sum(a.elapsed_time(b) for a, b, _, _ in ev)
    kern_ms = sum(c.elapsed_time(d) for _, _, c, d in ev)
    t_local = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    step_ms, kern_ms = (t_local / args.steps).tolist()
    value = W / (step_ms * 1e-3)

    # roofline of the dominant kernel (fused Gram + MI), per launch on this rank
    rank_tiles = int(tiles.shape[0])
    all_tiles = int(nat_num_tiles(m))
    ops_per_launch = 2.0 * W * (rank_tiles / all_tiles)
    achieved_tops = ops_per_launch / (kern_ms * 1e-3) / 1e12
    peaks = load_peaks()
    fp4 = operand_is_fp4(n)
    if fp4:  # e2m1 0/1 operands through kind::mxf4: the FP4 tensor peak is the ceiling
        peak = FP4_NOMINAL_TOPS
        kernel = ("gram_mi_kernel<2,*,*,6,8,*,fp4> (tcgen05 kind::mxf4 2-SM, e2m1 0/1 operands, unit E8M0 "
                  "scales, fp32 accumulators = exact counts, fused MI epilogue)")
        source = ("B200 datasheet dense FP4 (kind::mxf4), 9 PFLOP/s; tools/micro/mxf4_probe.cu measures "
                  "16382 MACs/clk/SM = 9.53 POP/s at 1965 MHz")
    else:
        peak = peaks["int8_tops"]
        kernel = "gram_mi_kernel<2,*,*> (tcgen05 kind::i8 2-SM + fused MI epilogue)"
        source = peaks["source"]
    roofline = {
        "bound": "tensor", "achieved": achieved_tops, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved_tops / peak, "traffic": load_traffic(args.config),
        "kernel": kernel,
        "ops": "tensor ops = 2 x pair-samples (1 MAC per pair-sample)",
        "peak_source": source,
        "frac_of_int8_datasheet": achieved_tops / INT8_NOMINAL_TOPS,
        "frac_of_2x_measured_bf16": (achieved_tops / peaks["two_x_measured_bf16_tops"]
                                     if "two_x_measured_bf16_tops" in peaks else None),
        "frac_of_cublas_int8": (achieved_tops / peaks["cublas_int8_tops"] if "cublas_int8_tops" in peaks else None),
        "kernel_ms": kern_ms,
    }

    # end to end through the public API: pinned host words in, host MI out
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, eng, words_dev, rank, world, n, m, cfg, out_dtype, W)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            val, info = cpu_sample(args.config, args.cpu_seconds)
            from oracle import oracle as O

            cpu = {"value": val, "unit": UNIT, "cores": info["threads"], "kind": "port",
                   "sample": (f"{info['n_cols_sampled']} of {m} columns x N={n:,} (full N), one timed run of "
                              f"{info['seconds']:.2f} s; reference algorithm restated in C (oracle/mi_oracle.c), "
                              f"OpenMP {info['threads']} threads, host {O.cpu_model()}")}
        except Exception as exc:  # the baseline must never sink the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": ("e2m1 0/1 (kind::mxf4) -> f32 exact counts + f64 MI epilogue" if fp4
                      else "i8->s32 GEMM + f64 epilogue"),
            "data": "synthetic (splitmix64 stream of the reference's datagen, generated on device)",
            "config": {"workload": workload_name(args.config, n, m, out_name), "n_rows": n, "n_cols": m,
                       "output": out_name, "tiles": all_tiles, "tile": 256,
                       "parallelism": f"upper-triangle tiles dealt over {world} GPU(s); words broadcast once",
                       "l2": "flushed between steps (256 MiB write, untimed)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            # per step: unpack prologue, unpack, column stats, fused Gram + MI
            "gpu_launches": 4 * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def nat_num_tiles(m: int) -> int:
    from paper_2411_19702_b200 import _native as nat

    return int(nat.lib().mi_num_tiles(m))


def run_e2e(args, eng, words_dev, rank, world, n, m, cfg, out_dtype, W):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2411_19702_b200 import dispatch as dsp

    dev = eng.device
    stream = torch.cuda.current_stream(dev)
    esz = 8 if out_dtype == torch.float64 else 4
    words_bytes = m * ((n + 63) // 64) * 8
    host_words = words_dev.cpu().pin_memory() if rank == 0 else None
    host_out = torch.empty((m, m), dtype=out_dtype, pin_memory=True) if (rank == 0 and world == 1) else None
    steps = max(1, min(args.steps, 20))
    shard_buf = torch.empty((m, m), dtype=out_dtype, device=dev) if world > 1 else None
    shared = None
    if world > 1:
        # one host matrix in node shared memory; every rank writes its share of
        # it over its own PCIe link (dispatch.mi_all_pairs_to_host) -- when
        # /dev/shm can hold it (same answer on every rank: one node)
        from paper_2411_19702_b200.hostshm import SharedHostMatrix

        name = f"mi_b200_bench_{os.environ.get('MASTER_PORT', '0')}"
        np_dt = np.float64 if out_dtype == torch.float64 else np.float32
        try:
            st = os.statvfs("/dev/shm")
            shm_ok = st.f_bavail * st.f_frsize > 1.2 * m * m * esz and not os.environ.get("MI_B200_NO_SHM")
        except OSError:
            shm_ok = False
        if shm_ok:
            if rank == 0:
                shared = SharedHostMatrix(name, m, np_dt, create=True)
            dist.barrier()
            if rank != 0:
                shared = SharedHostMatrix(name, m, np_dt, create=False)
        elif rank == 0:
            host_out = torch.empty((m, m), dtype=out_dtype, pin_memory=True)

    def once():
        if world == 1:
            eng.all_pairs_host(host_words, n, m, cfg, out_dtype, host_out=host_out)
        elif shared is not None:
            w = host_words.to(dev, non_blocking=True) if rank == 0 else None
            dsp.mi_all_pairs_to_host(eng, w, n, m, shared, cfg, out_dtype, out=shard_buf)
        else:  # no room in /dev/shm: gather onto rank 0's GPU, one D2H
            w = host_words.to(dev, non_blocking=True) if rank == 0 else None
            local, _ = dsp.mi_all_pairs_sharded(eng, w, n, m, cfg, out_dtype, out=shard_buf, zero_fill=True)
            full = dsp.gather_to_root(local, m)
            if rank == 0:
                host_out.copy_(full, non_blocking=True)
            stream.synchronize()

    for _ in range(2):
        once()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        once()
        b.record(stream)
        b.synchronize()
        t.append(a.elapsed_time(b))
    ms = torch.tensor([sum(t) / len(t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    if shared is not None:
        dist.barrier()
        shared.close()
    packed = None
    if world == 1:  # egress variant: the packed upper triangle (half the D2H), informational
        pk_out = torch.empty((m * (m + 1) // 2,), dtype=out_dtype, pin_memory=True)
        for _ in range(2):
            eng.all_pairs_host(host_words, n, m, cfg, out_dtype, host_out=pk_out, packed=True)
        tp = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.all_pairs_host(host_words, n, m, cfg, out_dtype, host_out=pk_out, packed=True)
            b.record(stream)
            b.synchronize()
            tp.append(a.elapsed_time(b))
        pms = sum(tp) / len(tp)
        packed = {"value": W / (pms * 1e-3), "unit": UNIT, "ms_per_step": pms,
                  "h2d_bytes_per_step": words_bytes, "d2h_bytes_per_step": m * (m + 1) // 2 * esz,
                  "api": "MIEngine.all_pairs_host(packed=True) -> mi_all_pairs_host_packed (upper triangle)"}
    return {"value": W / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": words_bytes,
            "d2h_bytes_per_step": m * m * esz, "ms_per_step": ms, "steps": steps, "packed_upper": packed,
            "api": "MIEngine.all_pairs_host (pinned words in, pinned MI out)" if world == 1 else
                   ("dispatch.mi_all_pairs_to_host (words H2D on rank 0, broadcast, sharded compute, every rank "
                    "copies its share into one shared-memory host matrix)" if shared is not None else
                    "dispatch.mi_all_pairs_sharded + gather_to_root + D2H on rank 0")}


def operand_is_fp4(n_rows: int) -> bool:
    """The C ABI's operand rule (capi.cu operand_fp4): e2m1 on SM pairs below 2^24 rows."""
    from paper_2411_19702_b200 import _native as nat
    return nat.get_tuning("fp4") == 1 and nat.get_tuning("cta_group") == 2 and n_rows < (1 << 24)


def load_peaks() -> dict:
    """int8 dense tensor peak for the roofline.

    Neither MEASURED_PEAKS.json (HBM copy, cuBLAS bf16) nor the profiling
    guide's fallback has an int8 figure, so the denominator is the B200
    datasheet dense int8 rate (4500 TOP/s).  Measured references are reported
    beside it: 2 x MEASURED_PEAKS bf16 burst, and cuBLAS int8 (torch._int_mm
    8192^3) from profiles/r01_int8_peak.json -- this kernel runs above both.
    """
    out = {"int8_tops": INT8_NOMINAL_TOPS, "source": "B200 datasheet dense int8 (no measured int8 peak is provided)"}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        out["two_x_measured_bf16_tops"] = 2.0 * float(json.loads(mp.read_text())["bf16_tflops"])
    prof = ROOT / "profiles" / "r01_int8_peak.json"
    if prof.exists():
        out["cublas_int8_tops"] = float(json.loads(prof.read_text())["int8_tops_cublas"])
    return out


def load_traffic(cfg: int):
    f = ROOT / "profiles" / "traffic.json"
    if f.exists():
        d = json.loads(f.read_text())
        v = d.get(f"config{cfg}")
        if v is not None:
            return v
    return None


if __name__ == "__main__":
    main()
