"""Summaries of ncu outputs for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv> [--last-fraction 0.333]
    python tools/ncu_summary.py full <report.ncu-rep>
"""
import collections
import csv
import io
import re
import subprocess
import sys


def _to_us(v, unit):
    unit = unit.lower()
    if unit.startswith("ns") or unit == "nsecond":
        return v / 1e3
    if unit.startswith("ms") or unit == "msecond":
        return v * 1e3
    if unit.startswith("s") and unit != "second":
        return v
    return v / 1e3 if unit in ("", "nsecond") else v


def launches(path, frac=1 / 3):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    step = data[int(len(data) * (1 - frac)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in step:
        name = d["Kernel Name"]
        m = re.search(r"gemm_tc_kernel<([^>]*)>", name)
        name = f"gemm_tc_kernel<{m.group(1)}>" if m else re.sub(r"\(.*", "", name).replace("void ", "")
        unit = d["Metric Unit"]
        v = float(d["Metric Value"])
        us = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = io.StringIO()
    out.write(f"# {path}: last {frac:.3f} of {len(data)} launches = {len(step)} launches, {tot / 1e3:.2f} ms "
              f"(serialised, cold-cache ncu times: compare shares)\n")
    out.write(f"{'kernel':60s} {'n':>6s} {'total_ms':>10s} {'share%':>7s} {'avg_us':>9s}\n")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"{k[:60]:60s} {v[0]:6d} {v[1] / 1e3:10.3f} {100 * v[1] / tot:7.1f} {v[1] / v[0]:9.1f}\n")
    return out.getvalue()


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, units = r[0], r[1]
    out = io.StringIO()
    out.write(f"# {path} (ncu --set full)\n")
    for row in r[2:]:
        name = row[h.index("Kernel Name")]
        out.write(f"kernel: {name}\n")
        for k in FULL:
            if k in h:
                i = h.index(k)
                out.write(f"  {k:75s} {row[i]:>14s} {units[i]}\n")
    return out.getvalue()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        fr = float(sys.argv[3]) if len(sys.argv) > 3 else 1 / 3
        print(launches(sys.argv[2], fr))
    else:
        print(full(sys.argv[2]))
