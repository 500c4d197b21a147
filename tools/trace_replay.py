"""Failure-trace replay against measured per-plan periods (§5.2
Fig. 9 methodology: "replayed the events in the GCP trace"; SPEC S:384-439 trace_simulator).

    python tools/trace_replay.py --periods profiles/r02_n4_1.3b_m2_f0.json profiles/r02_n4_1.3b_m2_f1.json \
        [--trace trace.json | --poisson-mtbf-h 2 --repair-h 1 --hours 24 --seed 0] [--max-failures 2] \
        [--migration-s 0.011] [--out report.json]

Each --periods argument is a bench.py JSON line for 0, 1, 2, ... failures (in that order):
its ms_per_step is the steady-state iteration period of that failure count's plan, measured
on B200 (placement by Algorithm 1), and DP * m * b * s tokens make one iteration.  The
replay runs iterations back to back with the current plan's period; on a FAIL event the
in-flight iteration is discarded (training resumes "from the iteration during which the
failure was identified", §4.1), the normalization swap's state copy is charged as
a stall and the next plan takes over; a REJOIN costs one copy as well and returns to the
previous plan.  More failures than plans (or an unrecoverable count) stall until a rejoin
(a checkpoint-restart stand-in).  Reports throughput over time, the average normalized
throughput (fault-free = 1.00, as the paper's Table 1) and the fault-scaled reference
(fault-free x live fraction, §5.3).  Host-side only: replays measured numbers.
"""
from __future__ import annotations

import argparse
import json
import math
import random


def replay(periods_s, tokens_per_iter, events, horizon_s, migration_s=0.0, total_workers=1):
    """periods_s[f]: iteration period with f failed workers (f = 0 .. len-1).
    events: [(time_s, +1 (FAIL) | -1 (REJOIN))], time-ordered.  Returns a report dict."""
    if any(b[0] < a[0] for a, b in zip(events, events[1:])):
        raise ValueError("TRACE_INVALID: events not time-ordered")
    t, f, iters = 0.0, 0, 0
    samples, stalls = [], []
    ev = list(events) + [(horizon_s, 0)]
    base = tokens_per_iter / periods_s[0]
    live_time = 0.0
    for (te, delta) in ev:
        te = min(te, horizon_s)
        if te > t:
            live_time += (te - t) * (total_workers - f) / total_workers
            if f < len(periods_s):
                P = periods_s[f]
                n = int(math.floor((te - t) / P + 1e-12))
                if n > 0:
                    samples.append({"t0": t, "t1": t + n * P, "failed": f, "iterations": n,
                                    "tokens_per_s": tokens_per_iter / P, "normalized": (tokens_per_iter / P) / base})
                iters += n
            else:  # no plan for this many failures: stalled until a rejoin
                stalls.append({"time_s": t, "cause": "NO_PLAN", "duration_s": te - t})
            t = te  # the in-flight iteration at the event is discarded
        if delta == 0 or t >= horizon_s:
            break
        nf = f + delta
        if nf < 0:
            raise ValueError("TRACE_INVALID: rejoin without a failed worker")
        if migration_s > 0 and nf < len(periods_s) and f < len(periods_s):
            d = min(migration_s, horizon_s - t)
            stalls.append({"time_s": t, "cause": "MIGRATION", "duration_s": d})
            live_time += d * (total_workers - nf) / total_workers
            t += d
        f = nf
    tokens = iters * tokens_per_iter
    return {"iterations_completed": iters, "tokens": tokens, "horizon_s": horizon_s,
            "average_tokens_per_s": tokens / horizon_s,
            "average_normalized_throughput": (tokens / horizon_s) / base,
            "fault_scaled_reference": live_time / horizon_s,
            "samples": samples, "stall_log": stalls}


def poisson_trace(mtbf_h, repair_h, hours, seed, max_failed):
    """Seeded synthetic failure / repair trace: failures arrive as a Poisson process with
    mean time between failures mtbf_h (while fewer than max_failed are down), each failed
    worker rejoins after repair_h."""
    rng = random.Random(seed)
    t, down, events = 0.0, [], []
    end = hours * 3600.0
    while t < end:
        t += rng.expovariate(1.0 / (mtbf_h * 3600.0))
        while down and down[0] <= t:
            events.append((down.pop(0), -1))
        if t >= end:
            break
        if len(down) < max_failed:
            events.append((t, +1))
            down.append(t + repair_h * 3600.0)
            down.sort()
    events += [(r, -1) for r in down if r < end]
    return sorted(events)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--periods", nargs="+", required=True, help="bench JSON lines for 0, 1, ... failures")
    ap.add_argument("--trace", default="", help="JSON [[time_s, +1|-1], ...]")
    ap.add_argument("--poisson-mtbf-h", type=float, default=2.0)
    ap.add_argument("--repair-h", type=float, default=1.0)
    ap.add_argument("--hours", type=float, default=24.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-failures", type=int, default=0, help="cap on simultaneous failures (default: #plans-1)")
    ap.add_argument("--migration-s", type=float, default=None, help="stall per swap (default: the bench's measured warm copy, else 0)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    lines = [json.loads(open(p).read().strip().splitlines()[-1]) for p in a.periods]
    periods = [ln["ms_per_step"] / 1e3 for ln in lines]
    tok = lines[0]["value"] * lines[0]["ms_per_step"] / 1e3  # tokens per iteration
    workers = lines[0]["n_gpus"]
    mig = a.migration_s
    if mig is None:
        mig = next((ln["normalization"]["migration_warm_ms"] / 1e3 for ln in lines
                    if ln.get("normalization", {}).get("migration_warm_ms")), 0.0)
    if a.trace:
        events = [tuple(e) for e in json.load(open(a.trace))]
    else:
        events = poisson_trace(a.poisson_mtbf_h, a.repair_h, a.hours, a.seed, a.max_failures or len(periods) - 1)
    rep = replay(periods, tok, events, a.hours * 3600.0, mig, workers)
    rep.update({"periods_s": periods, "tokens_per_iteration": tok, "events": len(events), "migration_s": mig,
                "inputs": a.periods})
    s = json.dumps({**{k: v for k, v in rep.items() if k not in ("samples", "stall_log")},
                    "stalls": len(rep["stall_log"]), "stall_s": sum(x["duration_s"] for x in rep["stall_log"])})
    print(s)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rep, fh)


if __name__ == "__main__":
    main()
