"""Summaries of ncu outputs for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv> [--last-fraction 0.333]
    python tools/ncu_summary.py full <report.ncu-rep>
    python tools/ncu_summary.py phases <metrics.csv> [hbm_peak_gbs]

`phases` reads the per-launch metric CSV of `ncu --profile-from-start off --csv --metrics PHASE_METRICS
python tools/kernel_bench.py --phases` and splits it at the torch fill kernels that kernel_bench puts
between F, B, W and AdamW: per kernel the duration, tensor-pipe % and DRAM bytes; per
phase the time-weighted tensor-pipe % of the tensor-core kernels and the HBM GB/s of the others.
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


PHASE_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                 "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__cycles_elapsed.avg.per_second"]
PHASES = ["F", "B", "W", "AdamW"]


def _scale(v, unit):
    unit = unit.lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9,
            "us": 1e-6, "ms": 1e-3,
            "msecond": 1e-3, "second": 1, "hz": 1, "khz": 1e3, "mhz": 1e6, "ghz": 1e9, "%": 1, "": 1}
    return v * mult.get(unit, 1)


def phases(path, hbm_peak=6546.6):
    rows = list(csv.reader(open(path)))
    hdr, launches = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = launches.setdefault(d["ID"], {"name": d["Kernel Name"], "m": {}})
        k["m"][d["Metric Name"]] = _scale(float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    out = io.StringIO()
    out.write(f"# {path}: one F / B / W / AdamW pass, ncu --clock-control none (cold caches, serialised);\n"
              f"# tensor = sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active; "
              f"HBM GB/s against {hbm_peak} (MEASURED_PEAKS.json)\n")
    phase = -1
    per = collections.defaultdict(list)
    for k in launches.values():
        if "slip" not in k["name"]:  # torch fill marker between phases
            phase += 1
            continue
        if 0 <= phase < len(PHASES):
            per[PHASES[phase]].append(k)
    for ph in PHASES:
        ks = per.get(ph, [])
        if not ks:
            continue
        out.write(f"\n## {ph}\n{'kernel':44s} {'us':>9s} {'tensor%':>8s} {'DRAM MB':>9s} {'GB/s':>8s} {'MHz':>6s}\n")
        t_all = t_tc = w_tc = t_mem = b_mem = 0.0
        for k in ks:
            m = k["m"]
            t = m.get("gpu__time_duration.sum", 0.0)
            b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
            mhz = m.get("sm__cycles_elapsed.avg.per_second", 0.0) / 1e6
            nm = re.sub(r"^void |slip::|<unnamed>::|\(anonymous namespace\)::", "", k["name"]).split("(")[0]
            out.write(f"{nm[:44]:44s} {t * 1e6:9.1f} {tp:8.1f} {b / 1e6:9.1f} {b / t / 1e9 if t else 0:8.0f} "
                      f"{mhz:6.0f}\n")
            t_all += t
            if "gemm_tc" in nm or "attn_" in nm:
                t_tc += t
                w_tc += t * tp
            else:
                t_mem += t
                b_mem += b
        out.write(f"{ph}: {t_all * 1e6:.1f} us; tensor-core kernels {t_tc * 1e6:.1f} us at "
                  f"{w_tc / t_tc if t_tc else 0:.1f} % tensor pipe (time-weighted); other kernels "
                  f"{t_mem * 1e6:.1f} us, {b_mem / 1e6:.1f} MB, "
                  f"{b_mem / t_mem / 1e9 if t_mem else 0:.0f} GB/s = "
                  f"{b_mem / t_mem / 1e9 / hbm_peak if t_mem else 0:.3f} of peak\n")
    return out.getvalue()


if __name__ == "__main__":
    if sys.argv[1] == "phases":
        print(phases(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 6546.6))
        sys.exit(0)
    if sys.argv[1] == "launches":
        fr = float(sys.argv[3]) if len(sys.argv) > 3 else 1 / 3
        print(launches(sys.argv[2], fr))
    else:
        print(full(sys.argv[2]))
