"""Plan-vs-execution report from `bench.py --trace DIR` dumps (one rank*.json per rank).

    python tools/trace_report.py DIR

For every rank: busy time per action kind, idle gaps of the compute stream (time between
the end of one compute action and the begin of the next), the actions that waited longest
(begin of a compute action later than the end of the previous one), and the planner's
predicted period in the same units (10 us) next to the measured iteration span."""
import glob
import json
import os
import sys

COMPUTE = {"LOAD_X", "F", "LOSS", "B", "W", "BC", "OPT"}


def report(path):
    d = json.load(open(path))
    tr = d["trace"]
    comp = sorted((t for t in tr if t[0] in COMPUTE), key=lambda t: t[6])
    busy = {}
    for t in tr:
        busy[t[0]] = busy.get(t[0], 0.0) + (t[7] - t[6])
    gaps = []
    for prev, cur in zip(comp, comp[1:]):
        g = cur[6] - prev[7]
        if g > 0.05:
            gaps.append((g, prev[0], prev[1], prev[2], cur[0], cur[1], cur[2], cur[3], round(cur[6], 3)))
    gaps.sort(reverse=True)
    span = (comp[-1][7] - comp[0][6]) if comp else 0.0
    it_end = {}
    for t in comp:
        it_end[t[3]] = max(it_end.get(t[3], 0.0), t[7])
    out = {"rank": d["rank"], "role": d.get("role"), "span_ms": round(span, 3),
           "iter_end_ms": {k: round(v, 3) for k, v in sorted(it_end.items())},
           "plan_period_ms": d["plan_period"] * 0.01, "costs_10us": d.get("costs_10us"),
           "busy_ms": {k: round(v, 3) for k, v in sorted(busy.items())},
           "compute_idle_ms": round(sum(g[0] for g in gaps), 3),
           "largest_gaps": [{"ms": round(g[0], 3), "after": g[1:4], "before": g[4:8], "at_ms": g[8]}
                            for g in gaps[:8]]}
    return out


def main():
    for p in sorted(glob.glob(os.path.join(sys.argv[1], "rank*.json"))):
        print(json.dumps(report(p)))


if __name__ == "__main__":
    main()
