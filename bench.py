#!/usr/bin/env python
"""Benchmark: all-pairs binary MI throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A step is one pass of the hot path over one synthetic dataset of a BASELINE
config -- by default config 4 (N=50,000 x m=50,000, Beta(0.5,20) densities,
float32 MI), the largest single-GPU configuration and the one the 8-GPU
scaling target is defined on: the broadcast of the packed words (N > 1),
kernel 1 (unpack of the rank's column blocks + column statistics) and the
fused tcgen05 Gram + MI kernel over the rank's upper-triangle tiles, output
left on the device as tile-major shards (every rank, N = 1 included: the
same dispatch path at every N).  Rank 0 prints ONE JSON line.  `value` is
pair-samples/s (N*m(m+1)/2 per step) over the whole job, timed with CUDA
events per step, L2 flushed between steps (untimed), max over ranks.  `e2e`
is the same metric through the public API with host words in and the full
host MI matrix out.

`--gpus N` without torchrun starts N ranks itself (one process per GPU,
NCCL, 127.0.0.1); under torchrun WORLD_SIZE must equal N.

`--impl reference` times the reference algorithm on the host CPU cores (the
C restatement in oracle/, OpenMP, all threads) on a fixed, documented column
sample of the same workload; it is the driver's reference arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
# Fixed column sample of the CPU legs (full N, these many columns), so the
# reference arm's per-pair-sample rate does not depend on --steps: ~2-5 s of
# CPU work per step on the 16-thread host (config 3: the full matrix).
CPU_SAMPLE_COLS = {1: 500, 2: 2000, 3: 10000, 4: 12288, 5: 2048}


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-dropin", action="store_true", help="skip the drop-in mi_all_pairs (numpy) e2e variant")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-tall-narrow", action="store_true", help="skip the tall-N / narrow-m section")
    p.add_argument("--sustained-seconds", type=float, default=2.0)
    p.add_argument("--stages", type=int, default=-1, help="staged-broadcast column groups (-1 auto)")
    p.add_argument("--plumbing-check", action="store_true",
                   help="CPU-only: launcher, gloo process group, broadcast, tile dealing and max-over-ranks; "
                        "prints a JSON line with no metric value (tests)")
    return p.parse_args(argv)


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


# ----------------------------------------------------------------- launcher
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`--gpus N` without torchrun: N copies of this script, one per GPU, with
    the torchrun environment (RANK, LOCAL_RANK, WORLD_SIZE, MASTER_*)."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve())] + sys.argv[1:], env=env))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def init_dist(world: int, local: int, backend: str):
    """Process group for world > 1: NCCL with the device bound (its
    communicator-init lines are printed: NCCL_DEBUG=INFO, INIT subsystem,
    unless the caller set NCCL_DEBUG), or gloo for the CPU plumbing check."""
    import torch
    import torch.distributed as dist

    if world <= 1:
        return None
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    return dist


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
def cpu_sample_words(cfg: int):
    """The fixed CPU sample of config `cfg`: full N, CPU_SAMPLE_COLS columns
    (a seeded random subset; the whole matrix when that is all of it)."""
    import numpy as np
    from oracle import oracle as O

    rec = O.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    ms = min(m, CPU_SAMPLE_COLS[cfg])
    cols = sorted(np.random.default_rng(1234).choice(m, ms, replace=False).tolist()) if ms < m else None
    return O.c_generate_config_words(rec, cols), n, m, ms


def cpu_sample_text(n: int, m: int, ms: int, threads: int, extra: str = "") -> str:
    from oracle import oracle as O

    return (f"fixed full-N column sample: {ms} of {m} columns x N={n:,} rows (seeded subset, independent of "
            f"--steps; pair-samples/s = N*m_s(m_s+1)/2 / time){extra}; the reference algorithm (AND+popcount "
            f"Gram, closed-form counts, fp64 epilogue in the reference's cell order) restated in C "
            f"(oracle/mi_oracle.c), OpenMP {threads} threads, host {O.cpu_model()}")


def cpu_threads() -> int:
    """Host threads of the CPU legs: every core this process may run on
    (MI_BENCH_CPU_THREADS overrides).  Set explicitly: torchrun exports
    OMP_NUM_THREADS=1 to its workers, which would turn the reference arm of an
    N > 1 run into a single-thread baseline."""
    env = os.environ.get("MI_BENCH_CPU_THREADS")
    if env:
        return max(1, int(env))
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):
        return max(1, os.cpu_count() or 1)


def cpu_baseline_leg(cfg: int, runs: int = 3) -> dict:
    """The oracle on the host cores, timed on the fixed sample (~10 s)."""
    from oracle import oracle as O

    words, n, m, ms = cpu_sample_words(cfg)
    threads = cpu_threads()
    O.c_lib().oracle_set_threads(threads)
    O.c_mi_all_pairs(words, n)  # warm (threads, pages)
    times = []
    for _ in range(runs):
        t0 = time.perf_counter()
        O.c_mi_all_pairs(words, n)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    return {"value": pair_samples(n, ms) / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": cpu_sample_text(n, m, ms, threads, f", mean of {runs} runs of {t:.2f} s")}


def run_reference(args):
    """The driver's reference arm: the reference's algorithm on the host CPU
    (rank 0 only), the same metric on the fixed sample, --steps timed runs."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    words, n, m, ms = cpu_sample_words(args.config)
    threads = cpu_threads()
    O.c_lib().oracle_set_threads(threads)
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
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "popcount/int64+f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, n, m, out), "n_rows": n, "n_cols": m,
                   "n_cols_sampled": ms, "output": out},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": cpu_sample_text(n, m, ms, threads)},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- plumbing check (CPU)
def run_plumbing_check(args):
    """The multi-rank bench path without a GPU: process group (gloo), the
    broadcast of packed words, the C ABI's tile dealing (every tile once),
    and the max-over-ranks timing reduction.  No metric value."""
    import numpy as np
    import torch

    from paper_2411_19702_b200 import dispatch

    rank, world, _ = dist_env()
    dist = init_dist(world, 0, "gloo")
    n, m = 1000, 3000
    words = torch.arange(m * ((n + 63) // 64), dtype=torch.int64).reshape(m, -1) if rank == 0 else None
    t0 = time.perf_counter()
    w = dispatch.broadcast_words(words, n, m, torch.device("cpu"))
    tiles = dispatch.rank_tiles(m, rank, world)
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64)
    counts = torch.tensor([len(tiles)], dtype=torch.int64)
    ok = torch.tensor([int(w[-1, -1]) == m * ((n + 63) // 64) - 1], dtype=torch.int64)
    if dist is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(counts)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    T = -(-m // 256)
    if rank == 0:
        print(json.dumps({"plumbing_check": True, "n_gpus": world, "world_size": world,
                          "tiles_dealt": int(counts), "tiles_total": T * (T + 1) // 2,
                          "broadcast_ok": bool(ok.item()), "ms_max_over_ranks": float(ms.item()),
                          "backend": "gloo"}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ----------------------------------------------------------------- GPU arm
def pinned_empty(shape, np_dtype):
    """A page-locked host array of exactly this size (numpy + mi_host_register:
    torch's pinned allocator would round 10 GB up to 16 GB)."""
    import numpy as np

    from paper_2411_19702_b200 import _native as nat

    a = np.empty(shape, dtype=np_dtype)
    nat.check(nat.lib().mi_host_register(a.ctypes.data, a.nbytes), "mi_host_register")
    return a


def unpin(a):
    from paper_2411_19702_b200 import _native as nat

    nat.lib().mi_host_unregister(a.ctypes.data)


def run_gpu(args):
    import numpy as np
    import torch

    from paper_2411_19702_b200 import EngineConfig, MIEngine, datagen
    from paper_2411_19702_b200 import _native as nat
    from paper_2411_19702_b200 import dispatch as dsp

    rank, world, local = dist_env()
    # MI_B200_DIST_BACKEND=gloo (ranks sharing GPUs) only exercises the
    # multi-rank code path on fewer GPUs; timings are meaningless then.
    backend = os.environ.get("MI_B200_DIST_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if backend == "nccl" and world > ndev:
        print(f"bench.py: {world} ranks but {ndev} visible GPU(s); NCCL needs one GPU per rank", file=sys.stderr)
        sys.exit(2)
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(world, local, backend)
    comm = None
    if dist is not None:
        dist.barrier()  # the communicator is created (and its init lines printed) before any timing
        comm = {"backend": backend, "nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else None}
        if rank == 0:
            print(f"[bench] process group: {backend}, nranks={comm['nranks']}", file=sys.stderr, flush=True)
    eng = MIEngine.get(local)

    rec = datagen.config_recipe(args.config)
    n, m = rec["n"], rec["m"]
    out_name = datagen.CONFIGS[args.config]["out"]
    out_dtype = torch.float64 if out_name == "float64" else torch.float32
    cfg = EngineConfig()
    W = pair_samples(n, m)
    fp4 = operand_is_fp4(n)

    # measured tensor peak of this GPU (the roofline denominator), before anything else runs
    peak_burst = nat.tensor_peak(local, fp4, 0.05)
    peak_sust = nat.tensor_peak(local, fp4, 1.0)

    words_dev = datagen.generate_words_device(rec, dev) if rank == 0 else None
    stages = args.stages if args.stages >= 0 else dsp.auto_stages(m, world, eng.num_sms)
    stages = max(1, stages)
    my_tiles = dsp.rank_tiles(m, rank, world)
    tile = int(nat.lib().mi_tile_size())
    buf = torch.empty((max(len(my_tiles), 1), tile, tile), dtype=out_dtype, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step(timing=None):
        return dsp.mi_all_pairs_sharded(eng, words_dev, n, m, cfg, out_dtype, stages=stages, buf=buf, timing=timing)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    sampler = make_sampler(local) if rank == 0 else None
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kern = []
    for s0, s1 in ev:
        flush.fill_(1)  # untimed L2 flush
        s0.record(stream)
        step(kern)
        s1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    if dist is not None:
        dist.barrier()
    step_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    kern_ms = sum(a.elapsed_time(b) for a, b in kern) / args.steps  # all fused launches of a step
    t_local = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    step_ms, kern_ms = t_local.tolist()
    value = W / (step_ms * 1e-3)

    # sustained: back-to-back steps for >= --sustained-seconds (no flushes)
    sustained = None
    if args.sustained_seconds > 0:
        reps = max(3, int(math.ceil(args.sustained_seconds * 1e3 / max(step_ms, 1e-3))))
        sampler2 = make_sampler(local) if rank == 0 else None
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler2:
            sampler2.start()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            step()
        b.record(stream)
        torch.cuda.synchronize()
        c2 = sampler2.stop() if sampler2 else None
        ms = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms = float(ms.item())
        sustained = {"value": W / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": reps,
                     "seconds": ms * reps / 1e3, "clocks": c2, "l2": "not flushed (back to back)"}

    # roofline of the dominant kernel (fused Gram + MI) on this rank
    rank_tiles = len(my_tiles)
    all_tiles = int(nat.lib().mi_num_tiles(m))
    ops_per_launch = 2.0 * W * (rank_tiles / all_tiles)  # all fused launches of one step on this rank
    achieved_tops = ops_per_launch / (kern_ms * 1e-3) / 1e12
    peak = peak_burst["ops_per_s"] / 1e12
    instr = "kind::mxf4 (e2m1 0/1, unit E8M0 scales, fp32 accumulators = exact counts)" if fp4 else "kind::i8"
    roofline = {
        "bound": "tensor", "achieved": achieved_tops, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved_tops / peak, "traffic": load_traffic(args.config),
        "kernel": f"gram_mi_kernel<2,*,*,6,8,*,{'fp4' if fp4 else 'i8'}> (tcgen05.mma.cta_group::2 {instr}, "
                  "fused MI epilogue on the TMEM accumulator)",
        "ops": "tensor ops = 2 x pair-samples (1 MAC per pair-sample) of this rank's tiles per step",
        "peak_source": ("measured on this GPU by mi_tensor_peak just before the run: the same tcgen05 instruction "
                        "back to back on smem-resident operands, all SM pairs, 50 ms burst "
                        f"({peak_burst['macs_per_clk_sm']:.0f} MACs/clk/SM at {peak_burst['sm_mhz']:.0f} MHz)"),
        "peak_sustained": peak_sust["ops_per_s"] / 1e12,
        "peak_sustained_mhz": peak_sust["sm_mhz"],
        "frac_of_sustained_peak": achieved_tops / (peak_sust["ops_per_s"] / 1e12),
        "frac_of_fp4_datasheet": achieved_tops / FP4_NOMINAL_TOPS if fp4 else None,
        "frac_of_int8_datasheet": achieved_tops / INT8_NOMINAL_TOPS,
        "kernel_ms": kern_ms,
        "kernel_share_of_step": kern_ms / step_ms,
    }
    # The same fraction at the SM clock the kernel is actually given: the peak
    # is MACs/clk/SM x SMs x clock, and a power-capped run (sw_power_cap) sits
    # below the clock the MMA-only probe holds.  Taken over the 2 s sustained
    # section (NVML's clock lags: over the 20-step timed region it still shows
    # the clock from before the load), whole steps, not the kernel alone.
    if sustained and sustained.get("clocks") and sustained["clocks"].get("sm_mhz") and peak_burst.get("sm_mhz"):
        f = 2.0 * W / (sustained["ms_per_step"] * 1e-3) / 1e12 / peak
        sustained["frac_of_peak"] = f
        sustained["frac_at_sustained_clock"] = f * peak_burst["sm_mhz"] / sustained["clocks"]["sm_mhz"]

    e2e = None
    if not args.no_e2e:
        try:
            e2e = run_e2e(args, eng, words_dev, rank, world, n, m, cfg, out_dtype, W, stages, buf)
        except Exception as exc:  # a failing end-to-end leg must not sink the device-resident line
            e2e = {"value": None, "unit": UNIT, "error": f"{type(exc).__name__}: {exc}"}
            print(f"[bench] rank {rank}: e2e leg failed: {exc}", file=sys.stderr, flush=True)

    tall = None
    if rank == 0 and world == 1 and not args.no_tall_narrow:
        try:
            tall = run_tall_narrow(eng, peak)
        except Exception as exc:  # a side measurement must never sink the headline
            tall = {"error": str(exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_leg(args.config)
        except Exception as exc:  # the baseline must never sink the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port", "sample": f"failed: {exc}"}

    # launches per step: unpack prologue + (expansion + column statistics) per
    # stage (one stage: the 3-launch prepare) + one fused launch per stage
    launches = (3 + 1) if stages == 1 else (1 + 3 * stages)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": ("e2m1 0/1 (kind::mxf4) -> f32 exact counts + " if fp4 else "u8 0/1 (kind::i8) -> s32 counts + ")
                     + ("f32-pipe MI epilogue" if out_dtype == torch.float32 else "f64 / fixed-point MI epilogue"),
            "data": "synthetic (splitmix64 stream of the reference's datagen, generated on device)",
            "config": {"workload": workload_name(args.config, n, m, out_name), "n_rows": n, "n_cols": m,
                       "output": out_name, "tiles": all_tiles, "tile": tile, "rank_tiles_rank0": rank_tiles,
                       "stages": stages,
                       "output_layout": "upper-triangle tiles left on the device as tile-major shards "
                                        "(dispatch.Shard, MI_TILE_MAJOR); mirrors written by the gather "
                                        "(e2e below includes it)",
                       "parallelism": f"upper-triangle tiles dealt over {world} GPU(s); packed words broadcast "
                                      "once (NCCL)" if world > 1 else "1 GPU",
                       "l2": "flushed between steps (256 MiB write, untimed)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "sustained": sustained, "clocks": clocks,
            "tall_narrow": tall,
            "comm": comm, "gpu_launches": launches * args.steps,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def hbm_peak_gbs():
    """Measured HBM bandwidth of this pool's B200s (MEASURED_PEAKS.json), else
    the profiling guide's fallback."""
    f = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(f.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy read+write)"
    except Exception:
        return 6500.0, "fallback 6500 GB/s"


def run_tall_narrow(eng, tensor_peak_tops, n=8_000_000, m=512, reps=10):
    """The north_star's tall-N / narrow-m case (reading D dominates): one
    step = column statistics + fused Gram + MI on device-resident words,
    float64 MI, both operand paths -- the word-operand build (expansion in the
    GEMM's producer warps, X never in HBM; the default for this shape) and the
    unpack + TMA build (X written to HBM and read back) -- CUDA events, L2
    flushed between reps, bit-identity of the two results checked."""
    import torch

    from paper_2411_19702_b200 import datagen
    from paper_2411_19702_b200 import _native as nat

    dev = eng.device
    w = datagen.generate(n, m, 0.3, 11, dev)
    out = torch.empty((m, m), dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    W = pair_samples(n, m)
    words_b, mi_b = w.numel() * 8, m * m * 8
    hbm, hbm_src = hbm_peak_gbs()
    res, mats = {}, {}
    old = nat.get_tuning("xp")
    try:
        for xp in (1, 0):
            nat.set_tuning(xp=xp)
            run = lambda: eng.compute(eng.prepare(w, n, m), None, torch.float64, out=out)
            run()
            torch.cuda.synchronize()
            mats[xp] = out.clone()
            ts, tk = [], []
            for _ in range(reps):
                flush.fill_(1)
                a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record(stream)
                prep = eng.prepare(w, n, m)
                b.record(stream)
                eng.compute(prep, None, torch.float64, out=out)
                c.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(c))
                tk.append(b.elapsed_time(c))
                del prep
            step, kern = statistics.median(ts), statistics.median(tk)
            key = "words_operand" if xp else "unpack_tma"
            res[key] = {"step_ms": step, "fused_ms": kern, "value": W / (step * 1e-3),
                        "algorithmic_gbs": (words_b + mi_b) / (step * 1e-3) / 1e9,
                        "tensor_frac_of_peak": 2 * W / (kern * 1e-3) / 1e12 / tensor_peak_tops}
    finally:
        nat.set_tuning(xp=old)
    return {"workload": f"N={n:,} x m={m} Bernoulli(0.3), float64 MI, device-resident words", "unit": UNIT,
            "words_bytes": words_b, "mi_bytes": mi_b, "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src,
            "default_path": "words_operand" if eng.words_operand(n, m) else "unpack_tma",
            "bit_identical": bool(torch.equal(mats[0], mats[1])),
            "speedup_words_over_unpack": res["unpack_tma"]["step_ms"] / res["words_operand"]["step_ms"],
            "roofline_note": "tensor work 2W counts m(m+1)/2 pairs; the 256-wide diagonal tiles compute 1.5x that "
                             "at m = 512, so the MMA-issue ceiling is ~0.67 of peak",
            **res}


def run_e2e(args, eng, words_dev, rank, world, n, m, cfg, out_dtype, W, stages, buf):
    """The same metric through the public API, host words in, the full host
    MI matrix out (H2D of the words and the egress inside the timed region).
    1 GPU: MIEngine.all_pairs_host (C ABI mi_all_pairs_host, staged
    upload/compute/download) with pinned buffers, and the drop-in
    mi_all_pairs(BinaryMatrix) with numpy in and out.  N GPUs: words H2D on
    rank 0, broadcast, sharded compute, every rank writing its tiles and
    mirrors into one shared pinned host matrix over its own link."""
    import numpy as np
    import torch

    from paper_2411_19702_b200 import BinaryMatrix, mi_all_pairs
    from paper_2411_19702_b200 import dispatch as dsp

    dev = eng.device
    stream = torch.cuda.current_stream(dev)
    np_dt = np.float64 if out_dtype == torch.float64 else np.float32
    esz = np.dtype(np_dt).itemsize
    words_bytes = m * ((n + 63) // 64) * 8
    steps = max(1, min(args.steps, 5 if m >= 20000 else 20))
    host_words = pinned_empty((m, (n + 63) // 64), np.uint64) if rank == 0 else None
    if rank == 0:
        host_words[:] = words_dev.cpu().numpy().view(np.uint64)
    res = {"unit": UNIT, "h2d_bytes_per_step": words_bytes, "d2h_bytes_per_step": m * m * esz, "steps": steps}

    def timed(fn, k):
        fn()  # warm-up (allocations, pinning)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t = []
        for _ in range(k):
            a = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            t.append((time.perf_counter() - a) * 1e3)
        ms = torch.tensor([sum(t) / len(t)], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
        return float(ms.item())

    if world == 1:
        host_out = pinned_empty((m, m), np_dt)
        ht = torch.from_numpy(host_out)
        ms = timed(lambda: eng.all_pairs_host(host_words, n, m, cfg, out_dtype, host_out=ht), steps)
        unpin(host_out)
        del ht, host_out
        res.update({"value": W / (ms * 1e-3), "ms_per_step": ms,
                    "api": f"MIEngine.all_pairs_host -> C ABI mi_all_pairs_host (pinned words in, pinned {np_dt.__name__} "
                           "MI out, staged upload/compute/download)"})
        if not args.no_dropin:
            bm = BinaryMatrix(n, m, np.array(host_words))  # pageable numpy words, like a reference user's
            ms2 = timed(lambda: mi_all_pairs(bm), 1 if m >= 20000 else 3)
            res["dropin"] = {"value": W / (ms2 * 1e-3), "unit": UNIT, "ms_per_step": ms2,
                             "h2d_bytes_per_step": words_bytes, "d2h_bytes_per_step": m * m * 8,
                             "api": "mi_all_pairs(BinaryMatrix) drop-in (engine.py:144-168 signature): pageable numpy "
                                    "words in, fresh numpy float64 MIMatrix out"}
            del bm
        unpin(host_words)
        return res

    from paper_2411_19702_b200.hostshm import SharedHostMatrix

    name = f"mi_b200_bench_{os.environ.get('MASTER_PORT', '0')}"
    try:
        st = os.statvfs("/dev/shm")
        shm_ok = st.f_bavail * st.f_frsize > 1.2 * m * m * esz
    except OSError:
        shm_ok = False
    ok = torch.tensor([1 if shm_ok else 0], device=dev)
    torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
    if not int(ok.item()):
        res.update({"value": None, "note": "no room in /dev/shm for the shared host matrix"})
        return res
    if rank == 0:
        shared = SharedHostMatrix(name, m, np_dt, create=True)
    torch.distributed.barrier()
    if rank != 0:
        shared = SharedHostMatrix(name, m, np_dt, create=False)

    def once():
        w = torch.from_numpy(host_words.view(np.int64)).to(dev, non_blocking=True) if rank == 0 else None
        dsp.mi_all_pairs_to_host(eng, w, n, m, shared, cfg, out_dtype, stages=stages, buf=buf)

    ms = timed(once, steps)
    torch.distributed.barrier()
    shared.close()
    if rank == 0:
        unpin(host_words)
    res.update({"value": W / (ms * 1e-3), "ms_per_step": ms,
                "api": "dispatch.mi_all_pairs_to_host: words H2D on rank 0, NCCL broadcast, sharded compute, every "
                       "rank writes its tiles + mirrors into one shared pinned host matrix (mi_scatter_tiles, "
                       "zero-copy over its own PCIe link)"})
    return res


def operand_is_fp4(n_rows: int) -> bool:
    """The C ABI's operand rule (operand_fp4): e2m1 on SM pairs below 2^24 rows."""
    from paper_2411_19702_b200 import _native as nat
    return nat.get_tuning("fp4") == 1 and nat.get_tuning("cta_group") == 2 and n_rows < (1 << 24)


def load_traffic(cfg: int):
    """DRAM bytes (read + write) per launch of the fused kernel from one ncu
    --set full capture (profiles/traffic.json), or None."""
    f = ROOT / "profiles" / "traffic.json"
    if f.exists():
        d = json.loads(f.read_text())
        v = d.get(f"config{cfg}")
        if v is not None:
            return v
    return None


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.plumbing_check:
        run_plumbing_check(args)
        return
    run_gpu(args)


if __name__ == "__main__":
    main()
