"""Exact optimum of the paper's running example by the MILP of PAPER.md Eqs. 1-6
(oracle/milp.py, time-indexed form, HiGHS) — writes tests/golden/running_example_milp.json.

    python tools/milp_running_example.py        (about 4 + 4 minutes on 8 cores)

Calls only oracle/ (the stored schedules are checked against Eqs. 2-6 by
tests/test_oracle_milp.py, independently of the solver)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import milp  # noqa: E402

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "running_example.json")))


def main():
    N, DP, m = GOLD["num_stages"], GOLD["num_pipelines"], GOLD["num_microbatches"]
    fi, fk = GOLD["failed_worker"]
    live = [[1] * DP for _ in range(N)]
    live[fi][fk] = 0
    out = {"_source": "tools/milp_running_example.py: oracle/milp.py solve_time_indexed (PAPER.md Eqs. 1-6), "
                      "unit slots t_f = t_b = t_w = 1, T_comm = 0, 1F1B memory cap (N - i) n_w",
           "live": live, "num_microbatches": m}
    for name, dec, horizon in (("adaptive_only_coupled", False, 36), ("decoupled", True, 29)):
        t0 = time.time()
        r = milp.solve_time_indexed(live, m, horizon, decoupled=dec, time_limit=3600)
        assert r["status"] == 0, r["message"]
        out[name] = {"horizon": horizon, "optimal_makespan": r["makespan"], "solve_s": round(time.time() - t0, 1),
                     "starts": [[*o, t] for o, t in sorted(r["starts"].items())]}
        print(name, r["makespan"], "%.1fs" % (time.time() - t0), flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "running_example_milp.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
