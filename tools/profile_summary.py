"""Write the per-round ncu summaries committed under profiles/ (dev tool).

usage: python tools/profile_summary.py <launches.csv> <out_prefix> <full.ncu-rep> [more.ncu-rep ...]
"""
import collections
import os
import csv
import subprocess
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, start = r, i + 1
            break
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        us = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        tot[name] += us
        cnt[name] += 1
    return tot, cnt


FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
]


def full(path):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in FULL_METRICS:
            if m in hdr:
                d[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        res.append(d)
    return res


def main():
    lcsv, prefix, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    if lcsv != "-":   # ("-": full-set summaries only)
        write_launches(lcsv, prefix)
    with open(prefix + "_full.txt", "w") as f:
        f.write("# ncu --set full --clock-control none (one launch each)\n")
        for rep in reps:
            for d in full(rep):
                f.write(f"\n[{d.pop('kernel')}]  ({rep.split('/')[-1]})\n")
                for k, v in d.items():
                    f.write(f"  {k:62s} {v}\n")


def write_launches(lcsv, prefix):
    tot, cnt = launches(lcsv)
    S = sum(tot.values())
    with open(prefix + "_launches.txt", "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list of\n"
                f"#   {os.environ.get('FDE_LAUNCH_CMD', 'python bench.py --steps 1 --warmup 1 --no-cpu-baseline')}\n"
                f"#   (cold-cache, serialised)\n"
                f"# {sum(cnt.values())} launches, {S / 1e3:.1f} ms device time in total\n")
        f.write(f"{'kernel':30s} {'launches':>9s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}\n")
        for k, v in tot.most_common():
            f.write(f"{k:30s} {cnt[k]:9d} {v / 1e3:10.2f} {100 * v / S:6.1f}% {v / cnt[k]:9.2f}\n")


if __name__ == "__main__":
    main()
