"""Summarise ncu outputs brought back from gpurun into profiles/ (dev tool).

    python scripts/ncu_summary.py <launches.csv> <prof.ncu-rep> <out_prefix>

Writes <out_prefix>_launches.md (per-kernel share of device time from the
gpu__time_duration launch list) and <out_prefix>_kernels.md (key --set full metrics
of the captured launches).
"""
import collections
import csv
import io
import re
import subprocess
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
        "s": 1e3, "second": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.3f} | {100 * t / tot:.1f}% |")
    out.append(f"| **total** | | {tot:.3f} | 100% |")
    return "\n".join(out)


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "lts__t_sector_hit_rate.pct",
]


def kernels(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("void ", "")
        out.append(f"### `{name}`\n\n| metric | value |\n|---|---:|")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"| {k} | {r[i]} {u[i]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    lc, rep, prefix = sys.argv[1:4]
    open(prefix + "_launches.md", "w").write(
        f"# Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n\nsource: `{lc}`\n\n"
        + launches(lc) + "\n")
    open(prefix + "_kernels.md", "w").write(
        f"# ncu --set full summary\n\nsource: `{rep}`\n\n" + kernels(rep) + "\n")
    print(open(prefix + "_launches.md").read())
    print(open(prefix + "_kernels.md").read())
