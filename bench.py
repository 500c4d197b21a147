#!/usr/bin/env python
"""bench.py — training throughput of the SlipStream decoupled-B/W stage step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--failures F] [--impl slip|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: one rank per GPU, NCCL)

Workload (BASELINE.json configs[1]): GPT-1.3B-shaped model (h 2048, 16 heads,
ffn 8192, s 2048, b 1), bf16 with fp32 accumulation / master weights, synthetic
data.  N = 1: the full 24-layer model on one GPU (DP1 x PP1), m = 4
micro-batches per step.  N > 1: DP 2 x PP N/2, 24/PP layers per stage and
m = 4*PP micro-batches per pipeline, so the per-GPU work is fixed (weak
scaling).  A step is one training iteration of the plan: F, B (input grads),
deferred W (weight grads), the per-stage DP all-reduce and the staggered AdamW.
--failures F masks F ranks at the positions Algorithm 1
normalizes them to over the profiled cost table; their micro-batches are re-routed
to the DP peer.

One JSON line on rank 0 (contract in the task statement): value = whole-job
tokens/s over exactly K timed steps (CUDA events, max over ranks), plus e2e
(pinned-host inputs / loss read-back every step), roofline of the dominant
kernel family (the W GEMMs) measured live, cpu_baseline (fp64 oracle on the
host cores, bounded sample, rank 0 at N = 1), clocks sampled during the timed
region and the number of libslip kernels launched.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train tokens/sec at 0/1/2 failures, 1-8 B200; B/W tensor-pipe % of peak"
H, HEADS, FFN, SEQ, MB, LAYERS = 2048, 16, 8192, 2048, 1, 24
# GPT shapes of SURVEY.md §8(a) (reading R2); the default is BASELINE.json configs[1]
MODELS = {"1.3b": (2048, 16, 8192, 24), "2.7b": (2560, 32, 10240, 32), "6.7b": (4096, 32, 16384, 32)}
MODEL = "1.3b"
VOCAB = 50304  # GPT-2/3 BPE vocabulary 50257 padded to a multiple of 128 (reading R33)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="slip", choices=["slip", "reference"])
    ap.add_argument("--failures", type=int, default=0)
    ap.add_argument("--dp", type=int, default=0,
                    help="data-parallel pipelines (default: 1 on one GPU, else 2; PP = world / DP)")
    ap.add_argument("--microbatches", "--m", dest="m", type=int, default=0, help="micro-batches per pipeline (default 4*PP)")
    ap.add_argument("--layers", type=int, default=None, help="total layers (default: the model's)")
    ap.add_argument("--coupled", action="store_true", help="coupled backward, no staggering (1F1B baseline)")
    ap.add_argument("--no-stagger", action="store_true", help="decoupled B/W but a global optimizer barrier")
    ap.add_argument("--failed-at", default="",
                    help="actual failed workers 'i,k;i,k' (un-normalized); with --normalize they are migrated")
    ap.add_argument("--normalize", action="store_true",
                    help="Algorithm 1 + P2P migration swaps before the timed steps (needs --failed-at)")
    ap.add_argument("--sm-reserve", type=int, default=-1,
                    help="SMs kept free of persistent GEMM CTAs for NCCL kernels (default: 0 at N=1, 8 at N>1)")
    ap.add_argument("--p2p-ctas", type=int, default=2, help="CTAs per NCCL P2P kernel (0: NCCL default)")
    ap.add_argument("--push-ar", action="store_true",
                    help="fused DP = 2 all-reduce with the exchange in W: each W launch also writes its dW tiles "
                         "into the peer's receive buffer over NVLink (slip_comm_fuse_ar_push)")
    ap.add_argument("--no-fused-ar", action="store_true",
                    help="NCCL all-reduce + AdamW instead of the DP=2 all-reduce fused into AdamW over NVLink")
    ap.add_argument("--trace", default="", help="directory: dump one traced 2-iteration run per rank (JSON)")
    ap.add_argument("--gpt-ends", action="store_true",
                    help="GPT model ends: token + position embedding on the first stage, final LN + LM head "
                         "(vocab 50304) + cross-entropy on the last stage (SURVEY §8(f) NEXT-3)")
    ap.add_argument("--fused-adamw", action="store_true",
                    help="AdamW of the 2-D weights in the last W's epilogue where no all-reduce follows "
                         "(measured slower under the 1 kW power cap: off by default)")
    ap.add_argument("--dual-stream", default="auto", choices=["auto", "on", "off"],
                    help="forward actions on their own stream after profiling (auto: PP = 1 or m >= 4 PP)")
    ap.add_argument("--validate", action="store_true",
                    help="post-step validation with cross-stage rollback (slip_set_validation; PAPER.md lines "
                         "580-583): the NCCL all-reduce and a single compute stream")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--model", default="1.3b", choices=sorted(MODELS), help="GPT shape (default: BASELINE configs[1])")
    a = ap.parse_args()
    global H, HEADS, FFN, LAYERS, MODEL
    MODEL = a.model
    H, HEADS, FFN, LAYERS = MODELS[a.model]
    if a.layers is None:
        a.layers = LAYERS
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("bf16_tflops", 1590.0), p.get("bf16_tflops_sustained", 1400.0), p.get("hbm_gbs", 6650.0), \
            "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((int(f[0]), float(f[1]), float(f[2]), float(f[3]), f[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        pmax = max(r[3] for r in rows)
        load = [r for r in rows if r[3] >= 0.5 * pmax] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[4]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(r[1] for r in load), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load),
                "power_w_max": pmax}


# ---------------------------------------------------------------- oracle (CPU baseline)
def oracle_sample(layers_total, m, dp=1):
    """fp64 oracle on the host: one GPT-1.3B-shaped layer x one micro-batch of F + B + W
    plus AdamW over one layer's parameters; extrapolated to the job: dp pipelines of
    layers_total layers x m micro-batches, each replica taking its AdamW step."""
    import numpy as np

    import slipdata as sd
    from oracle import adam as OA
    from oracle import layer as OL
    cfg = sd.ModelCfg(hidden=H, heads=HEADS, ffn=FFN, seq=SEQ, micro_batch=MB, layers=layers_total)
    P = sd.layer_params(cfg, 0, 0)
    x, r = sd.stage_input(cfg, 0, 0), sd.stage_target(cfg, 0, 0)
    t0 = time.perf_counter()
    out, c = OL.layer_forward(P, x, cfg)
    _, dout = OL.loss_mse(out, r)
    dx, bg, st = OL.layer_backward_input(P, c, dout, cfg)
    wg = OL.layer_backward_weight(st)
    t1 = time.perf_counter()
    grads = dict(**bg, **wg)
    z = {k: np.zeros_like(v) for k, v in P.items()}
    OA.adamw_step_layer(P, z, z, grads, 1, OA.AdamCfg(), grad_scale=1.0 / m)
    t2 = time.perf_counter()
    t_layer, t_adam = t1 - t0, t2 - t1
    step_s = dp * layers_total * (m * t_layer + t_adam)
    tokens = dp * m * MB * SEQ
    return tokens / step_s, t_layer, t_adam


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle, as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    # the GPU arm's workload at this N (same DP x PP split and micro-batch count)
    DP = args.dp or (1 if args.gpus == 1 else 2)
    PP = max(1, args.gpus // DP)
    m = args.m or 4 * PP
    vals = []
    samples = []
    for step in range(args.warmup + args.steps):
        v, tl, ta = oracle_sample(args.layers, m, DP)
        if step >= args.warmup:
            vals.append(v)
            samples.append(tl + ta)
    value = statistics.median(vals)
    ms = 1000.0 * (DP * m * MB * SEQ) / value
    cores = cpu_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        # each step times a bounded sample; the full step is extrapolated from it
        "ms_per_step_kind": "extrapolated from the per-step sample (%d pipeline(s) x %d layers x %d micro-batches);"
                            " measured sample time per step %.0f ms" % (DP, args.layers, m,
                                                                       1000.0 * statistics.median(samples)),
        "sample_ms_per_step": 1000.0 * statistics.median(samples),
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "gpt-%s-shape (h%d s%d %d heads ffn%d) %d layers, DP%dxPP%d, m=%d micro-batches/pipeline,"
                               " failures=0" % (MODEL, H, SEQ, HEADS, FFN, args.layers, DP, PP, m),
                   "model": "gpt-%s-shape" % MODEL, "global_batch": DP * m * MB, "seq_len": SEQ,
                   "parallelism": "dp%dxpp%d (the fp64 oracle on the host cores)" % (DP, PP)},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": "per step: 1 layer x 1 micro-batch F+B+W (T=2048, h=2048) + AdamW over 1 layer,"
                                   " fp64 numpy, extrapolated to %d pipeline(s) x %d layers x %d micro-batches"
                                   % (DP, args.layers, m)},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def main():
    if os.environ.get("SLIP_BENCH_DUMP_AFTER"):  # debugging aid: Python stacks of a hung run
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["SLIP_BENCH_DUMP_AFTER"]), exit=True)
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    import slipdata as sd
    from paper_2405_14009_b200 import runtime as rt
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    DP = args.dp or (1 if world == 1 else 2)
    PP = world // DP
    if DP * PP != world or args.layers % PP:
        raise SystemExit(f"--dp {DP}: WORLD_SIZE {world} must be DP x PP with PP dividing {args.layers} layers")
    L = args.layers // PP
    m = args.m or 4 * PP
    me_stage = rank % PP
    ends = 0
    if args.gpt_ends:
        ends = (1 if me_stage == 0 else 0) | (2 if me_stage == PP - 1 else 0)
    cfg = sd.ModelCfg(hidden=H, heads=HEADS, ffn=FFN, seq=SEQ, micro_batch=MB, layers=args.layers,
                      vocab=VOCAB if args.gpt_ends else 0, ends=ends)
    T = cfg.tokens
    decoupled = not args.coupled
    staggered = not (args.coupled or args.no_stagger)
    # nominal integer costs ~ FLOP ratios of F : B : W, refined by profiling below
    costs = rt.make_costs(t_f=108, t_b=117, t_w=100, t_comm=1, t_ar=10, t_opt=10)

    def alg1_live(cs):
        """--failures F: the failures sit where Phase 1 of the Planner puts them (PAPER.md
        lines 374-424): R = A[N-1][F] of Algorithm 1 over the heuristic cost table of this
        plan variant (slip_normalize_costs -> slip_normalize), placed by
        slip_normalized_live — the steady state after the migration swaps."""
        if args.failures > PP * (DP - 1):
            return None, None
        R, _ = rt.normalize(PP, DP, args.failures,
                            rt.normalize_costs(PP, DP, m, cs, args.failures, decoupled, staggered))
        return R, rt.normalized_live(PP, DP, R)

    # the actual (un-normalized) set given by --failed-at, else Algorithm 1's placement
    alg1_R = None
    if args.failed_at:
        failed = [tuple(int(v) for v in f.split(",")) for f in args.failed_at.split(";")]
        live = [[1] * DP for _ in range(PP)]
        for (i, k) in failed:
            live[i][k] = 0
    elif args.failures:
        alg1_R, live = alg1_live(costs)
        if live is None:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": "tokens/s", "n_gpus": world,
                                  "error": "unrecoverable: %d failures > N (DP - 1)" % args.failures}))
            return
        failed = [(i, k) for i in range(PP) for k in range(DP) if not live[i][k]]
    else:
        failed, live = [], [[1] * DP for _ in range(PP)]
    if not rt.recoverable(PP, DP, live):
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": "tokens/s", "n_gpus": world,
                              "error": "unrecoverable failure set %s (a stage lost every worker)" % failed}))
        return
    plan_name = ("coupled 1F1B" if args.coupled else
                 "decoupled B/W, global optimizer barrier" if args.no_stagger else
                 "decoupled B/W + staggered AdamW")
    def inflight(lv, cs):
        """{(i, k): max in-flight micro-batches (F started, W / BC not finished)} of the plan"""
        plan = rt.plan_schedule(PP, DP, m, lv, cs, decoupled, staggered, horizon=2)
        out = {}
        for i in range(PP):
            for k in range(DP):
                cur = mx = 0
                for o in sorted((o for o in plan.ops if o[0] == i and o[4] == k and o[3] in (0, 2, 3)),
                                key=lambda o: o[6]):
                    cur += 1 if o[3] == 0 else -1
                    mx = max(mx, cur)
                out[(i, k)] = mx
        return out

    def slots_for(lv, cs):
        return max(1, max(inflight(lv, cs).values()))

    def normalization(cs):
        """Phase 1 of the Planner (§4.2.1): R from Algorithm 1 over the heuristic
        cost table, then the minimum swaps from the actual failure set to R."""
        F = len(failed)
        tab = rt.normalize_costs(PP, DP, m, cs, F, decoupled, staggered)
        R, _ = rt.normalize(PP, DP, F, tab)
        swaps, after = rt.migration_plan(PP, DP, live, R)
        return R, swaps, after, tab

    n_slots = slots_for(live, costs)
    if args.normalize:
        n_slots = max(n_slots, slots_for(normalization(costs)[2], costs))
    sm_reserve = args.sm_reserve if args.sm_reserve >= 0 else (0 if world == 1 else 8)
    rt.set_sm_reserve(sm_reserve)
    stage = rt.Stage(cfg, L, n_slots)
    rt.init_master_(stage.master, cfg, L, args.layers, seed=rank % PP)
    rt.call("slip_weights_from_master", stage.ctx, rt._stream())
    comm = rt.Comm(rank, world)
    if world > 1:
        comm.set_p2p_ctas(args.p2p_ctas)
    comm.setup(PP, DP, m, live)
    fused_ar = world > 1 and DP == 2 and not args.no_fused_ar

    def fuse(st, cm):  # the DP = 2 all-reduce fused into AdamW (push: its exchange in W)
        (rt.fuse_ar_push if (args.push_ar and not args.gpt_ends) else rt.fuse_ar_adam)(st, cm)
    if fused_ar:
        fuse(stage, comm)
    stream = torch.cuda.current_stream()

    def allreduce_max(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def execute(iters, io=None):
        return rt.execute_schedule(stage, comm, PP, DP, m, live, costs, decoupled, staggered, warmup=0,
                                   iterations=iters, seed=1234, io=io)

    # profile pass (§4.1 Profiler): measured per-op times -> integer planner costs (10 us units)
    if world > 1:
        execute(1)  # NCCL connects the pair communicators lazily: keep that out of the profiled costs
    rep = execute(max(1, args.warmup))
    per = []
    for ph in (0, 1, 2, 3, 4):
        n = rep.phase_ops[ph]
        per.append(allreduce_max(rep.phase_ms[ph] / n if n else 0.0))
    q = lambda ms: max(1, int(round(ms * 100)))  # noqa: E731
    costs = rt.make_costs(t_f=q(per[0]), t_b=q(per[1] or per[3]), t_w=q(per[2] or 0.01), t_comm=1,
                          t_ar=1 if fused_ar else q(per[4] * 0.5 if per[4] else 0.01), t_opt=q(per[4] or 0.01))
    norm = None
    my_role = rank
    if alg1_R is not None:
        # Algorithm 1 again with the profiled costs; a different placement re-forms the groups
        R2, live2 = alg1_live(costs)
        if live2 != live:
            if slots_for(live2, costs) > n_slots:
                n_slots = slots_for(live2, costs)
                stage.close()
                stage = rt.Stage(cfg, L, n_slots)
                rt.init_master_(stage.master, cfg, L, args.layers, seed=rank % PP)
                rt.call("slip_weights_from_master", stage.ctx, rt._stream())
            live = live2
            comm.setup(PP, DP, m, live)
            if fused_ar:
                fuse(stage, comm)
        alg1_R = R2
        failed = [(i, k) for i in range(PP) for k in range(DP) if not live[i][k]]
    if args.normalize and failed:
        # Normalization with the profiled costs, then one P2P state copy per swap (PAPER.md
        # lines 377-379): the GPU at the target position takes over the failed worker's role
        R, swaps, after, tab = normalization(costs)
        if slots_for(after, costs) > n_slots:
            raise SystemExit("normalized plan needs more slots than allocated")
        role = list(range(world))
        pairs = []
        for (fi, fk), (ti, tk), src in swaps:
            w_f, w_t, w_s = rt.rank_of(PP, fi, fk), rt.rank_of(PP, ti, tk), rt.rank_of(PP, fi, src)
            # the process playing the source role sends to the process playing the target role
            p_s, p_t, p_f = role.index(w_s), role.index(w_t), role.index(w_f)
            pairs.append((p_s, p_t))
            role[p_t], role[p_f] = w_f, w_t

        # a process whose role moves to a stage of a different model (the GPT ends) binds
        # that model first; the state copy then fills it (slip_migrate_state checks sizes)
        new_stage = role[rank] % PP
        new_ends = ((1 if new_stage == 0 else 0) | (2 if new_stage == PP - 1 else 0)) if args.gpt_ends else 0
        if new_ends != ends:
            ends = new_ends
            cfg = sd.ModelCfg(hidden=H, heads=HEADS, ffn=FFN, seq=SEQ, micro_batch=MB, layers=args.layers,
                              vocab=VOCAB if args.gpt_ends else 0, ends=ends)
            stage.close()
            stage = rt.Stage(cfg, L, n_slots)
            rt.init_master_(stage.master, cfg, L, args.layers, seed=new_stage)
            rt.call("slip_weights_from_master", stage.ctx, rt._stream())

        def migrate():
            barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for p_s, p_t in pairs:
                if rank == p_s:
                    rt.migrate_state(stage, comm, p_t, True)
                elif rank == p_t:
                    rt.migrate_state(stage, comm, p_s, False)
            g1.record(stream)
            barrier()
            return allreduce_max(g0.elapsed_time(g1))
        mig_ms = migrate()       # cold: includes NCCL's lazy P2P connection of the pair
        mig_warm_ms = migrate()  # the same copy again: the transfer alone
        comm.set_role(role[rank])
        my_role = role[rank]
        live = after
        comm.setup(PP, DP, m, live)
        if fused_ar:
            fuse(stage, comm)
        norm = {"actual_failed": failed, "R": R, "swaps": swaps, "migration_ms": mig_ms,
                "migration_warm_ms": mig_warm_ms, "state_bytes_per_swap": 12 * stage.n_params,
                "migration_GBps": (12 * stage.n_params / (mig_warm_ms * 1e6)) if swaps and mig_warm_ms else None,
                "cost_table_10us": {"%d,%d" % ix: v for ix, v in tab.items()},
                "normalized_failed": [(i, k) for i in range(PP) for k in range(DP) if not live[i][k]]}
        failed = norm["normalized_failed"]
    # the profiled costs above came from single-stream execution; the timed steps run the
    # forward actions on their own stream (slip_set_dual_stream: same plan, same results)
    # with one pipeline stage (measured +1-2.8 % at N = 1) and with PP > 1 at m >= 4 PP
    # (the default: DP2xPP2 m = 8 399.0k -> 407.8k, DP1xPP4 m = 16 384.0k -> 389.1k).  At
    # small m the overlapping forward competes with the backward chain across the stages,
    # the critical path there (DP2xPP2 m = 2: 321k -> 301k), so it stays off.
    dual = args.dual_stream == "on" or (args.dual_stream == "auto" and (PP == 1 or m >= 4 * PP))
    if args.validate:  # validated steps keep the NCCL all-reduce (the rollback needs the sum in place)
        rt.call("slip_set_validation", stage.ctx, 1)
        dual = False
    rt.call("slip_set_dual_stream", stage.ctx, int(dual))
    # AdamW of the 2-D weights in the epilogue of the iteration's last W where no all-reduce
    # follows (N = 1; the survivor of a failed DP = 2 group) — slip_set_fused_adamw
    fused_adamw = args.fused_adamw
    rt.call("slip_set_fused_adamw", stage.ctx, int(fused_adamw))
    # warm-up steps with the profiled plan
    execute(args.warmup)
    barrier()
    clocks = ClockSampler() if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rep = execute(args.steps)
    e1.record(stream)
    barrier()
    # the plan is identical on every rank; a masked rank (possibly rank 0) reports none
    predicted_period = int(allreduce_max(float(rep.predicted_period)))
    ms_total = allreduce_max(e0.elapsed_time(e1))
    clk = clocks.stop() if clocks else None
    tokens_per_step = DP * m * T
    value = tokens_per_step * args.steps / (ms_total / 1000.0)
    # roofline of the dominant kernel: the grouped W GEMM (all 4L products dW += dY^T X of a
    # slot in one persistent tcgen05 launch, fp32 accumulation fused in the epilogue).
    # achieved = algorithmic FLOP per launch (24 T h^2 L for ffn = 4h) x launches / their
    # CUDA-event time on the compute stream inside the timed region.
    flops_w_op = 2.0 * T * (4 * H * H + 2 * FFN * H) * L + (2.0 * T * VOCAB * H if ends & 2 else 0.0)
    ach_local = flops_w_op * rep.phase_ops[2] / (rep.phase_ms[2] / 1e3) / 1e12 if rep.phase_ops[2] else 0.0
    # masked ranks run nothing: take the per-phase numbers of the busiest live rank
    stats = torch.tensor([ach_local, float(rep.w_gemm_launches), rep.phase_ms[2]] + list(rep.phase_ms[:5]) +
                         [float(rep.phase_ops[2])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    stats = stats.tolist()
    ach = stats[0] or None
    w_launches = int(stats[1])
    w_ms_total = stats[2]
    phase_ms = stats[3:8]
    w_ops = stats[8]  # micro-batch W's: back-to-back W's run as one launch (K = n T)
    p_burst, p_sus, hbm, peak_src = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "w_gemm_traffic.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    if os.environ.get("SLIP_BENCH_PROFILE") and rank == 0:
        # diagnostic (outside the timed region): per-kernel CUPTI durations of one step
        import re
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            execute(1)
            torch.cuda.synchronize()
        tot, cnt = {}, {}
        for e in prof.events():
            if e.device_type.name != "CUDA":
                continue
            k = re.sub(r"^void |slip::|\(anonymous namespace\)::|<unnamed>::", "", e.name).split("(")[0][:60]
            d = e.device_time if hasattr(e, "device_time") else e.cuda_time
            tot[k] = tot.get(k, 0.0) + d
            cnt[k] = cnt.get(k, 0) + 1
        for k in sorted(tot, key=lambda k: -tot[k]):
            print(f"PROFILE {tot[k] / 1e3:9.3f} ms {cnt[k]:6d} x {tot[k] / cnt[k]:8.1f} us  {k}", file=sys.stderr)
        # idle gaps between consecutive device activities, by (previous -> next) kernel
        kev = []
        for e in prof.events():
            if e.device_type.name != "CUDA":
                continue
            k = re.sub(r"^void |slip::|\(anonymous namespace\)::|<unnamed>::", "", e.name).split("(")[0][:40]
            t0 = e.time_range.start
            kev.append((t0, t0 + (e.device_time if hasattr(e, "device_time") else e.cuda_time), k))
        kev.sort()
        gaps, gcnt = {}, {}
        end = None
        prev = None
        for t0, t1, k in kev:
            if end is not None and t0 > end:
                key = f"{prev} -> {k}"
                gaps[key] = gaps.get(key, 0.0) + (t0 - end)
                gcnt[key] = gcnt.get(key, 0) + 1
            if end is None or t1 > end:
                end, prev = t1, k
        print(f"PROFILE span {(kev[-1][1] - kev[0][0]) / 1e3:.3f} ms, idle {sum(gaps.values()) / 1e3:.3f} ms",
              file=sys.stderr)
        for k in sorted(gaps, key=lambda k: -gaps[k])[:15]:
            print(f"PROFILE gap {gaps[k] / 1e3:8.3f} ms {gcnt[k]:6d} x {gaps[k] / gcnt[k]:7.1f} us  {k}", file=sys.stderr)
    if args.trace:
        # plan-vs-execution timeline (outside the timed region)
        rt.set_trace(stage, True)
        execute(2)
        barrier()
        trace = rt.get_trace(stage)
        rt.set_trace(stage, False)
        plan = rt.plan_schedule(PP, DP, m, live, costs, decoupled, staggered, horizon=2)
        os.makedirs(args.trace, exist_ok=True)
        with open(os.path.join(args.trace, "rank%d.json" % rank), "w") as f:
            json.dump({"rank": rank, "role": my_role, "live": live, "costs_10us": [costs.t_f, costs.t_b, costs.t_w,
                                                                                      costs.t_comm, costs.t_ar,
                                                                                      costs.t_opt],
                       "trace": trace, "plan_ops": plan.ops, "plan_period": plan.period}, f)
    # per-stage peak memory (Fig. 12): the plan's peak in-flight
    # micro-batches per worker x the stash bytes of one slot, plus parameters / optimizer state
    # (bf16 w + fp32 master, grad, m, v = 18 B/param); and the bytes this process allocated
    peak = inflight(live, costs)
    alloc = torch.tensor([float(torch.cuda.max_memory_allocated())], dtype=torch.float64, device="cuda")
    alloc_all = [torch.zeros_like(alloc) for _ in range(world)]
    if world > 1:
        dist.all_gather(alloc_all, alloc)
    else:
        alloc_all = [alloc]
    slot_bytes = stage.stash_bytes / max(1, stage.n_slots)
    memory = {"stash_bytes_per_microbatch": slot_bytes, "param_state_bytes": 18 * stage.n_params,
              "workspace_bytes": stage.ws_bytes,
              "plan_peak_inflight": {"%d,%d" % ik: v for ik, v in sorted(peak.items())},
              "plan_peak_bytes_per_stage": [max(peak[(i, k)] for k in range(DP)) * slot_bytes + 18 * stage.n_params
                                            for i in range(PP)],
              "allocated_bytes_per_rank": [a.item() for a in alloc_all]}
    kern = torch.tensor([rep.n_kernels], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(kern)
    gpu_launches = int(kern.item())
    # e2e through the C ABI with pinned host buffers: every step copies its inputs H2D and
    # reads the losses back D2H (one executor call per step)
    e2e = None
    if not args.no_e2e:
        g = torch.Generator().manual_seed(7)
        if ends & 1:  # token ids in
            xs = [torch.randint(0, VOCAB, (T,), generator=g, dtype=torch.int32).pin_memory() for _ in range(DP * m)]
        else:
            xs = [torch.randn(T, H, generator=g).to(torch.bfloat16).pin_memory() for _ in range(DP * m)]
        if ends & 2:  # labels in
            rs = [torch.randint(0, VOCAB, (T,), generator=g, dtype=torch.int32).pin_memory() for _ in range(DP * m)]
        else:
            rs = [torch.randn(T, H, generator=g).to(torch.bfloat16).pin_memory() for _ in range(DP * m)]
        loss_host = torch.zeros(DP * m, dtype=torch.float32).pin_memory()
        io = rt.make_io(xs, rs, loss_host)
        execute(1, io)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            r = execute(1, io)
        f1.record(stream)
        barrier()
        e2e_ms = allreduce_max(f0.elapsed_time(f1))
        # bytes per step over the whole job: X for every stage-0 F, targets for every last-stage B
        in_b = T * 4 if args.gpt_ends else T * H * 2  # token ids / labels, or [T, h] bf16
        h2d = 2 * DP * m * in_b
        e2e = {"value": tokens_per_step * args.steps / (e2e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4 * DP * m,
               "last_loss": float(r.last_loss) if (rank % PP) == PP - 1 else None}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, tl, ta = oracle_sample(args.layers, m)
        cpu = {"value": v, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": "1 layer x 1 micro-batch F+B+W (T=2048, h=2048) %.1f s + AdamW over 1 layer %.1f s, fp64"
                         " numpy, extrapolated to %d layers x %d micro-batches" % (tl, ta, args.layers, m)}
    if rank != 0:
        return
    ms_step = ms_total / args.steps
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": ("gpt-%s-shape (h%d, %d heads, ffn %d, s%d, b1) " % (MODEL, H, HEADS, FFN, SEQ)) +
                               "%d layers, DP%dxPP%d, "
                               "m=%d micro-batches/pipeline, %s, failures=%d" % (
                                   args.layers, DP, PP, m,
                                   plan_name + (", GPT ends (embedding + LM head V=50304 + CE)"
                                                if args.gpt_ends else ", MSE head on a synthetic stage-0 input"),
                                   len(failed)),
                   "model": "gpt-%s-shape" % MODEL, "global_batch": DP * m * MB, "seq_len": SEQ,
                   "parallelism": "dp%dxpp%d" % (DP, PP), "failed_workers": failed, "sm_reserve": sm_reserve,
                   "p2p_ctas": args.p2p_ctas, "fused_ar_adam": fused_ar and not args.validate,
                   "ar_exchange_in_w": bool(fused_ar and args.push_ar and not args.gpt_ends and not args.validate), "dual_stream": dual,
                   "validated": args.validate,
                   "adamw_in_w_epilogue": fused_adamw,
                   "l2": "inputs larger than L2 (2.4 GB bf16 weights + GBs of stash per step)"},
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "roofline": {"bound": "tensor",
                     "kernel": "W GEMMs (tcgen05, dW (+)= sum over the launch's micro-batches dY^T X, fp32 TMA store" +
                               ("; where no all-reduce follows, the iteration's last W applies AdamW to the 2-D "
                                "weights in its epilogue instead of storing dW: achieved counts the GEMM FLOPs only)"
                                if fused_adamw else ")"),
                     "achieved": ach, "peak": p_sus, "peak_kind": "bf16_tflops_sustained (%s)" % peak_src,
                     "unit": "TFLOP/s", "frac": (ach / p_sus) if ach else None, "traffic": traffic,
                     "flops_per_launch": flops_w_op * w_ops / w_launches if w_launches else None,
                     "microbatch_w_per_launch": w_ops / w_launches if w_launches else None,
                     "launches": w_launches,
                     "avg_launch_ms": (w_ms_total / w_launches) if w_launches else None},
        # (with the dual stream the F and B phase times overlap each other)
        "phases_ms_per_step_busiest_rank": {n: phase_ms[i] / args.steps
                                            for i, n in enumerate(("F", "B", "W", "BC", "OPT"))},
        "predicted_period_units": predicted_period,
        "planner_costs_10us": [costs.t_f, costs.t_b, costs.t_w, costs.t_opt],
    }
    line["memory"] = memory
    # the metric's second half (BASELINE.json: "B/W tensor-pipe % of peak") from the committed
    # per-phase ncu capture of this model's layer (a profiler number: context, not timed here)
    try:
        with open(os.path.join(ROOT, "profiles", "r02_tensor_pipe.json")) as f:
            tp = json.load(f).get("gpt-%s" % MODEL)
        if tp:
            line["tensor_pipe_ncu"] = {ph: tp[ph]["tensor_pipe_pct"] for ph in ("F", "B", "W") if ph in tp}
            line["tensor_pipe_ncu"]["source"] = "profiles/r02_tensor_pipe.json (ncu, one layer-micro-batch)"
            line["hbm_frac_ncu"] = {"adamw": tp["AdamW"]["other_frac_hbm"], "b_elementwise": tp["B"]["other_frac_hbm"]}
    except Exception:
        pass
    if norm:
        line["normalization"] = norm
    elif alg1_R is not None:
        line["normalization"] = {"R": alg1_R, "placement": "Algorithm 1 over the profiled heuristic cost table "
                                                            "(slip_normalize), placed by slip_normalized_live",
                                 "normalized_failed": failed}
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    comm.close()
    stage.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
