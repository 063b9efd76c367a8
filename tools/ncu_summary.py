"""Summarise an ncu report (.ncu-rep) or launch-list CSV into profiles/.

    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep profiles/r01_cfg3_full.md [algo_bytes]
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_cfg3_launches.md
"""
import csv, io, subprocess, sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
    "launch__block_size", "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def report(path, out, algo=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{path}`", ""]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '?')[:120]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
        rb = _bytes(d.get("dram__bytes_read.sum"), u.get("dram__bytes_read.sum"))
        wb = _bytes(d.get("dram__bytes_write.sum"), u.get("dram__bytes_write.sum"))
        if rb is not None and wb is not None:
            lines.append(f"| traffic (read+write) | {rb + wb:.4e} | byte |")
            if algo:
                lines.append(f"| algorithmic bytes | {float(algo):.4e} | byte |")
                lines.append(f"| traffic / algorithmic | {(rb + wb) / float(algo):.2f} | x |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def _bytes(v, unit):
    if v is None:
        return None
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return f * scale


def launches(path, out):
    """Per-kernel launch counts, mean / total duration and share; with extra
    --metrics (e.g. dram__bytes_read.sum), their per-launch means too."""
    rows = list(csv.reader(open(path)))
    hdr = None
    time = defaultdict(list)
    extra = defaultdict(lambda: defaultdict(list))
    order, metrics = [], []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0][:90]
            val = float(d["Metric Value"].replace(",", ""))
            if name not in time and name not in extra:
                order.append(name)
            if d["Metric Name"] == "gpu__time_duration.sum":
                scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1, "msecond": 1}.get(
                    d["Metric Unit"], 1e-6)
                time[name].append(val * scale)
            else:
                key = f"{d['Metric Name']} ({d['Metric Unit']})"
                if key not in metrics:
                    metrics.append(key)
                extra[name][key].append(val)
    total = sum(sum(v) for v in time.values())
    lines = [f"# launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`): `{path}`", "",
             "cold-cache, serialised per launch: compare SHARES, not absolutes.", "",
             "| kernel | launches | mean ms | total ms | share |" + "".join(f" mean {k} |" for k in metrics),
             "|---|---|---|---|---|" + "---|" * len(metrics)]
    for n in order:
        v = time.get(n, [])
        if not v:
            continue
        ex = "".join(f" {sum(extra[n][k]) / len(extra[n][k]):.4g} |" if extra[n][k] else " - |" for k in metrics)
        lines.append(f"| {n} | {len(v)} | {sum(v)/len(v):.4f} | {sum(v):.3f} | {sum(v)/total*100:.1f}% |" + ex)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
