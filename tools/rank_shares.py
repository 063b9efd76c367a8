"""Per-rank compute of the multi-GPU dealing, measured one rank at a time on
one GPU (ranks never wait on each other: each runs its own partial unpack and
its own tile list).  Reports, per world size, every rank's step time (partial
unpack + fused kernel over its tiles) and the compute-only strong-scaling
efficiency T(1) / (world * max_r T_r).  The broadcast (one NCCL broadcast of
the packed words) is not included -- it needs real NVLink peers.
    python tools/rank_shares.py --configs 3,4 --worlds 2,4,8"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="3,4")
ap.add_argument("--worlds", default="2,4,8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--sustained", type=float, default=0.0,
                help="seconds: instead of timing ranks alone (cold, best of reps), run all ranks' steps of a world "
                     "back to back for this long (same power state as the 1-rank run) and report "
                     "T(1) / sum_r T_r: what the sharding itself costs (partial unpacks, round quantization)")
a = ap.parse_args()
eng = MIEngine.get(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)


def timed(fn):
    fn(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(a.reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for cfg in [int(x) for x in a.configs.split(",")]:
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    dt = torch.float64 if datagen.CONFIGS[cfg]["out"] == "float64" else torch.float32
    w = datagen.generate_words_device(rec, eng.device)
    ts_ = int(nat.lib().mi_tile_size())
    bufs = {}

    def step(rank, world):
        # the bench's form: the rank's tiles alone, tile-major (MI_TILE_MAJOR)
        tl = eng.tiles(m, rank, world)
        key = (rank, world)
        if key not in bufs:
            bufs.clear()
            bufs[key] = torch.empty((max(int(tl.shape[0]), 1), ts_, ts_), dtype=dt, device=eng.device)
        prep = eng.prepare(w, n, m, rank, world)
        eng.compute(prep, None, dt, tiles=tl, out=bufs[key], tile_major=True)

    if a.sustained > 0:
        def sus(fn):
            fn(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            reps = max(2, int(a.sustained * 1e3 / e0.elapsed_time(e1)))
            e0.record()
            for _ in range(reps):
                fn()
            e1.record(); e1.synchronize()
            return e0.elapsed_time(e1) / reps

        t1 = sus(lambda: step(0, 1))
        print(json.dumps({"cfg": cfg, "world": 1, "sustained_ms": round(t1, 3)}), flush=True)
        for world in [int(x) for x in a.worlds.split(",")]:
            tw = sus(lambda: [step(r, world) for r in range(world)])
            print(json.dumps({"cfg": cfg, "world": world, "sum_over_ranks_ms": round(tw, 3),
                              "mean_rank_ms": round(tw / world, 3),
                              "sharding_efficiency": round(t1 / tw, 3)}), flush=True)
        t1b = sus(lambda: step(0, 1))
        print(json.dumps({"cfg": cfg, "world": 1, "sustained_ms_again": round(t1b, 3)}), flush=True)
        del bufs, w
        torch.cuda.empty_cache()
        continue
    t1 = timed(lambda: step(0, 1))
    print(json.dumps({"cfg": cfg, "world": 1, "ms": round(t1, 3)}), flush=True)
    for world in [int(x) for x in a.worlds.split(",")]:
        ts = [timed(lambda r=r: step(r, world)) for r in range(world)]
        tiles = [int(eng.tiles(m, r, world).shape[0]) for r in range(world)]
        print(json.dumps({"cfg": cfg, "world": world, "rank_ms": [round(t, 3) for t in ts], "tiles": tiles,
                          "max_ms": round(max(ts), 3), "compute_efficiency": round(t1 / (world * max(ts)), 3)}),
              flush=True)
    del bufs, w
    torch.cuda.empty_cache()
