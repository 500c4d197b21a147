"""Planner-based throughput prediction (the paper's own methodology,
PAPER.md §5.3: a schedule simulator fed with profiled per-op costs).

    python tools/predict.py --layer-ms F B W --adam-ms-per-mparam A [--cfg c3] [--pp 4] [--dp 2]

Per-op costs of one stage = layers/stage x per-layer-micro-batch times measured on one
B200 (tools/kernel_bench.py), Adam = A ms per million parameters (measured), P2P of one
[T, h] bf16 activation over NVLink at 700 GB/s, the stage all-reduce at the measured
NCCL bus bandwidth.  The C++ planner (the one the executor runs) produces the period for
coupled 1F1B (the paper's baseline) and decoupled + staggered plans with 0 / 1 / 2
masked workers placed by Algorithm 1 (R = A[N-1][F] over the
heuristic cost table of the same plan variant, slip_normalize_costs -> slip_normalize ->
slip_normalized_live).  Prints one JSON line per case with R.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import slipdata as sd  # noqa: E402
from paper_2405_14009_b200 import runtime as rt  # noqa: E402

CFGS = {"c2": sd.C2_1P3B, "c3": sd.C3_2P7B, "c5": sd.C5_6P7B}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3")
    ap.add_argument("--layer-ms", type=float, nargs=3, required=True, help="F B W ms per layer-micro-batch")
    ap.add_argument("--adam-ms-per-mparam", type=float, default=0.0047)
    ap.add_argument("--ar-gbs", type=float, default=700.0, help="all-reduce bus bandwidth GB/s (2 ranks)")
    ap.add_argument("--p2p-gbs", type=float, default=700.0)
    ap.add_argument("--dp", type=int, default=2)
    ap.add_argument("--pp", type=int, default=4)
    ap.add_argument("--m", type=int, nargs="+", default=[3, 4, 8, 16])
    a = ap.parse_args()
    cfg = CFGS[a.cfg]
    L = cfg.layers // a.pp
    T, h = cfg.tokens, cfg.hidden
    f_ms, b_ms, w_ms = (x * L for x in a.layer_ms)
    params = cfg.params_per_layer * L
    opt_ms = a.adam_ms_per_mparam * params / 1e6
    ar_ms = 4.0 * params / (a.ar_gbs * 1e6)  # 2 (n-1)/n * bytes, n = 2
    comm_ms = 2.0 * T * h / (a.p2p_gbs * 1e6)
    unit = 0.01  # 10 us
    q = lambda ms: max(1, int(round(ms / unit)))  # noqa: E731
    costs = rt.make_costs(t_f=q(f_ms), t_b=q(b_ms), t_w=q(w_ms), t_comm=q(comm_ms), t_ar=q(ar_ms), t_opt=q(opt_ms))
    for m in a.m:
        base = None
        for nf in (0, 1, 2):
            if nf > a.pp * (a.dp - 1):
                continue
            row = {}
            for name, dec, stag in (("coupled_1f1b", False, False), ("decoupled_staggered", True, True)):
                # Algorithm 1 over this plan variant's own cost table places the failures
                R = [0] * a.pp
                if nf:
                    R, _ = rt.normalize(a.pp, a.dp, nf, rt.normalize_costs(a.pp, a.dp, m, costs, nf, dec, stag))
                live = rt.normalized_live(a.pp, a.dp, R)
                r = rt.plan_schedule(a.pp, a.dp, m, live, costs, dec, stag, horizon=3)
                period_ms = r.period * unit
                row[name] = {"period_ms": period_ms, "tokens_per_s": a.dp * m * T / (period_ms / 1e3), "R": R,
                             "failed": [(i, k) for i in range(a.pp) for k in range(a.dp) if not live[i][k]]}
            if nf == 0:
                base = row["coupled_1f1b"]["tokens_per_s"]
                base_dec = row["decoupled_staggered"]["tokens_per_s"]
            out = {"cfg": a.cfg, "dp": a.dp, "pp": a.pp, "layers_per_stage": L, "m": m, "failures": nf,
                   "costs_ms": {"F": f_ms, "B": b_ms, "W": w_ms, "OPT": opt_ms, "AR": ar_ms, "P2P": comm_ms}, **row,
                   "slipstream_vs_faultfree_1f1b": row["decoupled_staggered"]["tokens_per_s"] / base,
                   "slipstream_vs_faultfree_decoupled": row["decoupled_staggered"]["tokens_per_s"] / base_dec}
            print(json.dumps(out))


if __name__ == "__main__":
    main()
