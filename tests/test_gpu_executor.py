"""Executor and re-route numerics on ONE GPU against the fp64 oracle (SURVEY §8(a)
rows a3, a5, a7, a10; §3.1, ReRouteAct / ReRouteGrad /
InputBackwardPass / WeightBackwardPass line 554-558).

(i)  slip_execute_schedule at N = 1 (the bench's own call: program interpretation,
     merged W launches over the slots, accumulate flags, grad_scale, the AdamW step
     counter): after each of two iterations the fp32 stage gradient equals the
     oracle's sum over the micro-batches of Delta_j (Gate A), and master / m / v after
     AdamW equal oracle/adam.py applied to the GPU's own gradient (Gate B).
(ii) DP = 2 re-routing on one GPU: one Stage context per live worker, each driven
     through ITS rank program (slip_rank_program: LOAD_X / RECV_X / F / SEND_Y /
     LOSS / RECV_DY / B / SEND_DX / W / BC, with the executor's merging of back-to-back
     W's), messages passed between the contexts in per-pair FIFO order.  The live
     peers' fp32 gradients summed in ascending k (the stage all-reduce) equal
     oracle/pipeline.py per_worker_sum (form ii) within Gate A, and equal the
     fault-free GPU run within 1e-5 (only the fp32 summation order moves).
"""
import numpy as np
import pytest
import torch

import slipdata as sd
from oracle import adam as OA
from oracle import pipeline as PPL
from oracle import planner as PL

pytestmark = pytest.mark.gpu

GATE_A = 2e-2
GATE_B = 1e-4
ADAM = OA.AdamCfg(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
ACT = dict(LOAD_X=0, RECV_X=1, F=2, SEND_Y=3, LOSS=4, RECV_DY=5, B=6, SEND_DX=7, W=8, BC=9, AR=10, OPT=11)


def _rt():
    from paper_2405_14009_b200 import runtime
    return runtime


def relerr(g, r):
    g = np.asarray(g, dtype=np.float64)
    return float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))


def host_bf16(x):
    return torch.from_numpy(sd.to_bf16_bits(x).view(np.int16).copy()).view(torch.bfloat16)


def dev_bf16(x):
    return host_bf16(x).cuda()


def as_np(t):
    return t.float().cpu().numpy().astype(np.float64)


def oracle_grad_sum(stages, cfg, keys):
    """Sum over the micro-batches `keys` = [(k, j)] (ascending) of the oracle's
    per-micro-batch stage gradients; returns (per stage a list of per-layer dicts,
    the per-micro-batch losses)."""
    tot, losses = None, []
    for (k, j) in keys:
        lo, g = PPL.microbatch_pass(stages, cfg, sd.stage_input(cfg, k, j), sd.stage_target(cfg, k, j))
        losses.append(lo)
        if tot is None:
            tot = g
        else:
            for ts, gs in zip(tot, g):
                for a, b in zip(ts, gs):
                    for n in a:
                        a[n] = a[n] + b[n]
    return tot, losses


EXEC_CFGS = {
    "c1": (sd.C1_TINY, 1),
    "d80_ragged": (sd.ModelCfg(hidden=640, heads=8, ffn=2560, seq=200, micro_batch=1, layers=2), 2),
}


def exec_vs_oracle(cfg, L, m, iters, total_layers=None):
    """Run `iters` single-iteration slip_execute_schedule calls at N = 1 with the seeded
    inputs; check Gate A on the gradient and Gate B on AdamW after each.  Returns the
    per-iteration, per-layer worst relative error over the layer's tensors."""
    rt = _rt()
    layers = sd.stage_params(cfg, 0, L, total_layers=total_layers or max(L, 2))
    costs = rt.make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=1, t_opt=1)
    prog, need = rt.rank_program(1, 1, m, None, costs, 0)
    kinds = [p[0] for p in prog]
    # the N = 1 plan defers all W's to the end of the iteration: one merged launch over m slots
    assert kinds.count(ACT["W"]) == m and kinds[-2 - m:-2] == [ACT["W"]] * m, kinds
    st = rt.Stage(cfg, L, n_slots=need)
    st.load_master(torch.from_numpy(sd.pack_stage(layers)).float().cuda())
    comm = rt.Comm(0, 1)
    comm.setup(1, 1, m, None)
    xs = [host_bf16(sd.stage_input(cfg, 0, j)) for j in range(m)]
    rs = [host_bf16(sd.stage_target(cfg, 0, j)) for j in range(m)]
    losses = torch.zeros(m, dtype=torch.float32)
    io = rt.make_io(xs, rs, losses)
    adam = (ADAM.lr, ADAM.beta1, ADAM.beta2, ADAM.eps, ADAM.weight_decay)
    m_ref = v_ref = None
    growth = []
    for it in range(1, iters + 1):
        # the weights this iteration's F / B use: RNE(master) = the bf16 copy
        params = sd.unpack_stage(as_np(st.w), cfg, L)
        p_before = st.master.cpu().numpy().astype(np.float64)
        rep = rt.execute_schedule(st, comm, 1, 1, m, None, costs, True, True, adam=adam, iterations=1, io=io)
        torch.cuda.synchronize()
        assert rep.w_gemm_launches == 1 and rep.phase_ops[2] == m  # merged W: 1 launch, m micro-batch W's
        ref, lref = oracle_grad_sum([params], cfg, [(0, j) for j in range(m)])
        ref = ref[0]
        gflat = st.grad.cpu().numpy().astype(np.float64)
        got = sd.unpack_stage(gflat, cfg, L)
        per_layer = []
        for l in range(L):
            errs = {n: relerr(got[l][n], ref[l][n]) for n in sd.PARAM_ORDER}
            per_layer.append(max(errs.values()))
            for n, e in errs.items():
                assert e <= GATE_A, (it, l, n, e)
        growth.append(per_layer)
        # losses (device MSE of the bf16 output) vs the oracle's
        for j in range(m):
            assert abs(losses[j].item() - lref[j]) <= 1e-2 * lref[j]
        # Gate B: AdamW step `it` on the GPU's own gradient (grad_scale = 1 / (DP m))
        Pm = sd.unpack_stage(p_before, cfg, L)
        G = sd.unpack_stage(gflat, cfg, L)
        if m_ref is None:
            m_ref = [{n: np.zeros_like(a) for n, a in d.items()} for d in Pm]
            v_ref = [{n: np.zeros_like(a) for n, a in d.items()} for d in Pm]
        new_p, new_m, new_v = [], [], []
        for l in range(L):
            p1, m1, v1 = OA.adamw_step_layer(Pm[l], m_ref[l], v_ref[l], G[l], it, ADAM, grad_scale=1.0 / m)
            new_p.append(p1), new_m.append(m1), new_v.append(v1)
        p_got = st.master.cpu().numpy().astype(np.float64)
        assert relerr(p_got - p_before, sd.pack_stage(new_p) - p_before) <= GATE_B
        assert relerr(st.adam_m.cpu().numpy().astype(np.float64), sd.pack_stage(new_m)) <= GATE_B
        assert relerr(st.adam_v.cpu().numpy().astype(np.float64), sd.pack_stage(new_v)) <= GATE_B
        assert np.array_equal(as_np(st.w), sd.bf16_round(p_got))
        # continue from the GPU's own optimizer state (identical fp32 inputs for the next Gate B)
        m_ref = sd.unpack_stage(st.adam_m.cpu().numpy().astype(np.float64), cfg, L)
        v_ref = sd.unpack_stage(st.adam_v.cpu().numpy().astype(np.float64), cfg, L)
    comm.close()
    st.close()
    return growth


@pytest.mark.parametrize("name", list(EXEC_CFGS))
def test_execute_schedule_n1_matches_oracle(name):
    cfg, L = EXEC_CFGS[name]
    exec_vs_oracle(cfg, L, m=4, iters=2)


@pytest.mark.slow
def test_execute_schedule_c2_six_layer_stage_full_size():
    """The C2 stage of SURVEY §8(d.2) at full size: 6 GPT-1.3B layers (h 2048, 16 heads,
    s 2048), m = 4, through slip_execute_schedule — the bench's launch configuration,
    including the merged W launch with K = 4T over 4 slots.  Gate A per tensor and per
    layer; the per-layer error growth is printed and written to
    gpurun_out/c2_six_layer_growth.json when that directory exists."""
    import json
    import os
    growth = exec_vs_oracle(sd.C2_1P3B, 6, m=4, iters=1, total_layers=24)
    line = {"config": "gpt-1.3b 6-layer stage, s 2048, m 4, merged W K=4T",
            "worst_relerr_per_layer_input_to_output": growth[0]}
    print(json.dumps(line))
    if os.path.isdir("gpurun_out"):
        with open("gpurun_out/c2_six_layer_growth.json", "w") as f:
            json.dump(line, f)


# ------------------------------------------------------------------ (ii) re-route on one GPU
def run_programs(cfg, L, N, DP, m, live, costs, stages_params):
    """Drive one Stage context per live worker through its rank program; returns
    {(i, k): fp32 grad tensor} and the per-micro-batch losses."""
    rt = _rt()
    progs, ctxs, bufs = {}, {}, {}
    T, h = cfg.tokens, cfg.hidden
    for i in range(N):
        for k in range(DP):
            if not live[i][k]:
                continue
            r = rt.rank_of(N, i, k)
            prog, need = rt.rank_program(N, DP, m, live, costs, r)
            progs[r] = prog
            st = rt.Stage(cfg, L, n_slots=max(1, need))
            st.load_master(torch.from_numpy(sd.pack_stage(stages_params[i])).float().cuda())
            ctxs[r] = st
            mk = lambda: [torch.zeros(T, h, dtype=torch.bfloat16, device="cuda") for _ in range(max(1, need))]  # noqa
            bufs[r] = {"x": mk(), "y": mk(), "dy": mk(), "dx": mk()}
    queues = {}  # (src, dst, kind) -> list of ((iter, mb, origin), tensor)
    pc = {r: 0 for r in progs}
    losses = {}
    loss_d = torch.zeros(1, device="cuda")
    while any(pc[r] < len(progs[r]) for r in progs):
        progressed = False
        for r in progs:
            st, b, prog = ctxs[r], bufs[r], progs[r]
            i = r % N
            while pc[r] < len(prog):
                kind, it, mb, origin, peer, slot, acc = prog[pc[r]]
                ident = (it, mb, origin)
                if kind in (ACT["RECV_X"], ACT["RECV_DY"]):
                    q = queues.get((peer, r, kind))
                    if not q:
                        break  # blocked on the sender
                    got_id, t = q.pop(0)
                    assert got_id == ident, ("per-pair FIFO violated", got_id, ident)
                    (b["x"] if kind == ACT["RECV_X"] else b["dy"])[slot].copy_(t)
                elif kind == ACT["LOAD_X"]:
                    b["x"][slot].copy_(dev_bf16(sd.stage_input(cfg, origin, mb)))
                elif kind == ACT["F"]:
                    st.forward(slot, b["x"][slot], b["y"][slot])
                elif kind == ACT["SEND_Y"]:
                    queues.setdefault((r, peer, ACT["RECV_X"]), []).append((ident, b["y"][slot].clone()))
                elif kind == ACT["LOSS"]:
                    st.loss_mse(b["y"][slot], dev_bf16(sd.stage_target(cfg, origin, mb)), b["dy"][slot], loss_d)
                    losses[(origin, mb)] = loss_d.item()
                elif kind == ACT["B"]:
                    st.backward_input(slot, b["dy"][slot], b["dx"][slot] if i > 0 else None, accumulate=bool(acc & 1))
                elif kind == ACT["BC"]:
                    st.backward_coupled(slot, b["dy"][slot], b["dx"][slot] if i > 0 else None,
                                        accumulate=bool(acc & 1))
                elif kind == ACT["SEND_DX"]:
                    queues.setdefault((r, peer, ACT["RECV_DY"]), []).append((ident, b["dx"][slot].clone()))
                elif kind == ACT["W"]:
                    # the executor's merging: back-to-back W's of one iteration -> one launch
                    run = 1
                    while (pc[r] + run < len(prog) and run < 8 and prog[pc[r] + run][0] == ACT["W"]
                           and prog[pc[r] + run][1] == it):
                        run += 1
                    if run == 1:
                        st.backward_weight(slot, accumulate=bool(acc))
                    else:
                        st.backward_weight_multi([prog[pc[r] + q][5] for q in range(run)], accumulate=bool(acc))
                    pc[r] += run - 1
                # AR / OPT: the all-reduce is formed below (sum over live peers, ascending k)
                pc[r] += 1
                progressed = True
        assert progressed, "deadlock: every rank blocked on a receive"
    torch.cuda.synchronize()
    assert all(not q for q in queues.values()), "unconsumed messages"
    grads = {(r % N, r // N): ctxs[r].grad.clone() for r in progs}
    for st in ctxs.values():
        st.close()
    return grads, losses


REROUTE = [
    # (N, DP, m, failed workers (i, k))
    (1, 2, 3, [(0, 1)]),
    (1, 2, 3, [(0, 0)]),
    (2, 2, 2, [(1, 1)]),
    (2, 2, 3, [(0, 0)]),
]


@pytest.mark.parametrize("N,DP,m,failed", REROUTE)
def test_reroute_dp2_on_one_gpu_matches_oracle(N, DP, m, failed):
    rt = _rt()
    cfg, L = sd.ModelCfg(hidden=128, heads=2, ffn=512, seq=96, micro_batch=1, layers=2 * N), 1
    stages = [sd.stage_params(cfg, i, L, total_layers=2 * N) for i in range(N)]
    costs = rt.make_costs(t_f=2, t_b=2, t_w=1, t_comm=1, t_ar=1, t_opt=1)
    live_ff = [[1] * DP for _ in range(N)]
    live = [[1] * DP for _ in range(N)]
    for (i, k) in failed:
        live[i][k] = 0
    g_ff, l_ff = run_programs(cfg, L, N, DP, m, live_ff, costs, stages)
    g_rr, l_rr = run_programs(cfg, L, N, DP, m, live, costs, stages)
    # re-routing changes which worker computes a micro-batch, never its numbers
    assert l_rr == l_ff
    # oracle form (ii): per-worker accumulation in the plan's W order, live-peer sum
    delta, _ = PPL.contributions(stages, cfg, DP, m, {(k, j): sd.stage_input(cfg, k, j)
                                                       for k in range(DP) for j in range(m)},
                                 {(k, j): sd.stage_target(cfg, k, j) for k in range(DP) for j in range(m)})
    plan = PL.schedule(live, m, PL.Costs(t_f=2, t_b=2, t_w=1, t_comm=1, t_ar=1, t_opt=1),
                       PL.Opts(decoupled=True, staggered=True, horizon=1))
    for i in range(N):
        peers = [k for k in range(DP) if live[i][k]]
        summed = g_rr[(i, peers[0])].clone()
        for k in peers[1:]:
            summed += g_rr[(i, k)]
        ff = g_ff[(i, 0)].clone()
        for k in range(1, DP):
            ff += g_ff[(i, k)]
        # against the fault-free GPU run: fp32 summation order only
        assert ((summed - ff).abs().max() / ff.abs().max()).item() <= 1e-5, i
        ref = PPL.per_worker_sum(delta, plan, live, i)
        got = sd.unpack_stage(summed.cpu().numpy().astype(np.float64), cfg, L)
        for l in range(L):
            for n in sd.PARAM_ORDER:
                e = relerr(got[l][n], ref[l][n])
                assert e <= GATE_A, (i, l, n, e)
    # the failed worker ran nothing; its peer ran every micro-batch of the stage
    for (i, k) in failed:
        assert (i, k) not in g_rr


def test_execute_schedule_validation_skips_a_nonfinite_step():
    """Post-step validation at N = 1 (reading R31): with a fault
    injected the stage's own validation fails, so the step is skipped — master, m, v and
    the bf16 weights bit-identical to before it, no rollback needed — and the skipped
    step does not advance AdamW's bias-correction count: the next iteration equals, bit
    for bit, the second iteration of a run that never saw the fault."""
    rt = _rt()
    cfg, L, m = sd.C1_TINY, 1, 2
    layers = sd.stage_params(cfg, 0, L, total_layers=2)
    costs = rt.make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=1, t_opt=1)
    adam = (1e-3, 0.9, 0.95, 1e-8, 0.1)

    def make():
        _, need = rt.rank_program(1, 1, m, None, costs, 0)
        st = rt.Stage(cfg, L, n_slots=need)
        st.load_master(torch.from_numpy(sd.pack_stage(layers)).float().cuda())
        rt.call("slip_set_validation", st.ctx, 1)
        comm = rt.Comm(0, 1)
        comm.setup(1, 1, m, None)
        io = rt.make_io([host_bf16(sd.stage_input(cfg, 0, j)) for j in range(m)],
                        [host_bf16(sd.stage_target(cfg, 0, j)) for j in range(m)], torch.zeros(m))
        return st, comm, io

    def state(st):
        return [st.master.clone(), st.adam_m.clone(), st.adam_v.clone(), st.w.clone()]

    st, comm, io = make()
    r1 = rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=adam, iterations=1, io=io)
    torch.cuda.synchronize()
    s1 = state(st)
    rt.call("slip_inject_fault", st.ctx, 1)
    r2 = rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=adam, iterations=1, io=io)
    torch.cuda.synchronize()
    assert r1.rollbacks == 0 and r2.rollbacks == 0 and r1.skipped == 0 and r2.skipped == 1
    assert all(torch.equal(a, b) for a, b in zip(s1, state(st)))
    rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=adam, iterations=1, io=io)
    torch.cuda.synchronize()
    ref, rcomm, rio = make()
    for _ in range(2):
        rt.execute_schedule(ref, rcomm, 1, 1, m, None, costs, adam=adam, iterations=1, io=rio)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(state(ref), state(st)))
    for c in (comm, rcomm):
        c.close()


def test_execute_schedule_gpt_ends_n1_matches_oracle():
    """The executor with both GPT ends on one stage (reading R33): token ids and labels
    from host buffers, embedding, layers, final LN + LM head + cross-entropy, B, the merged
    W (dW_out in the grouped launch, the embedding scatter) over m = 3 micro-batches:
    summed gradients per tensor vs oracle/ends.py + oracle/layer.py (Gate A), losses to 1e-2,
    after each of two calls (the second starts from the first's gradient buffer: rows of
    the embedding gradient that no micro-batch of the iteration touches must be zero)."""
    rt = _rt()
    cfg = sd.ModelCfg(hidden=128, heads=2, ffn=512, seq=64, micro_batch=2, layers=1, vocab=384, ends=3)
    L, m = 1, 3
    layers = sd.stage_params(cfg, 0, L, total_layers=2)
    ends = sd.end_params(cfg, 0)
    flat = np.concatenate([sd.pack_stage(layers), sd.pack_ends(ends)])
    costs = rt.make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=1, t_opt=1)
    _, need = rt.rank_program(1, 1, m, None, costs, 0)
    st = rt.Stage(cfg, L, n_slots=need)
    st.load_master(torch.from_numpy(flat).float().cuda())
    comm = rt.Comm(0, 1)
    comm.setup(1, 1, m, None)
    toks = [sd.stage_tokens(cfg, 0, j) for j in range(m)]
    labs = [sd.stage_labels(cfg, 0, j) for j in range(m)]
    losses = torch.zeros(m)
    io = rt.make_io([torch.from_numpy(t.copy()) for t in toks], [torch.from_numpy(x.copy()) for x in labs], losses)
    P = cfg.params_per_layer
    for it in range(2):
        # the weights this call's F / B use: RNE(master) = the bf16 copy
        wflat = as_np(st.w)
        layers = sd.unpack_stage(wflat[:L * P], cfg, L)
        ends = sd.unpack_ends(wflat[L * P:], cfg)
        rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=(1e-3, 0.9, 0.95, 1e-8, 0.1), iterations=1, io=io)
        torch.cuda.synchronize()
        _check_gpt_ends_grads(st, cfg, L, m, layers, ends, toks, labs, losses, it)
    comm.close()
    st.close()


def _check_gpt_ends_grads(st, cfg, L, m, layers, ends, toks, labs, losses, it):
    from oracle import ends as OE
    from oracle import layer as OL
    ref_l, ref_e = None, None
    for j in range(m):
        x0 = OE.embed_fwd(ends["E"], ends["P"], toks[j], cfg.seq)
        out, caches = OL.stage_forward(layers, x0, cfg)
        lref, hc = OE.head_forward(out, ends["gf"], ends["bf"], ends["Wout"], labs[j], cfg.ln_eps)
        assert abs(losses[j].item() - lref) <= 1e-2 * abs(lref)
        dout, hb, hws = OE.head_backward_input(hc)
        dxr, grads = OL.stage_backward_coupled(layers, caches, dout, cfg)
        dE, dP = OE.embed_bwd(dxr, toks[j], cfg.seq, cfg.vocab)
        e = {"E": dE, "P": dP, "gf": hb["gf"], "bf": hb["bf"], "Wout": OE.head_backward_weight(hws)["Wout"]}
        ref_l = grads if ref_l is None else [{n: a[n] + b[n] for n in a} for a, b in zip(ref_l, grads)]
        ref_e = e if ref_e is None else {n: ref_e[n] + e[n] for n in e}
    gflat = st.grad.cpu().numpy().astype(np.float64)
    P = cfg.params_per_layer
    got = sd.unpack_stage(gflat[:L * P], cfg, L)
    for l in range(L):
        for n in sd.PARAM_ORDER:
            assert relerr(got[l][n], ref_l[l][n]) <= GATE_A, (it, l, n)
    ge = sd.unpack_ends(gflat[L * P:], cfg)
    for n in ("E", "P", "gf", "bf", "Wout"):
        assert relerr(ge[n], ref_e[n]) <= GATE_A, (it, n)
    # rows of E no micro-batch of the iteration used: exactly zero
    used = np.zeros(cfg.vocab, dtype=bool)
    for t in toks:
        used[np.asarray(t).reshape(-1)] = True
    assert not np.any(ge["E"][~used]), it


@pytest.mark.parametrize("name", list(EXEC_CFGS))
def test_fused_adamw_in_w_epilogue_equals_separate_step(name):
    """slip_set_fused_adamw: the iteration's last W applies AdamW to the 2-D weights in its
    epilogue (the OPT then steps the 1-D parameters only).  Two iterations at N = 1 must
    leave master, m, v and the bf16 weights identical to the separate optimizer pass (the
    same per-element arithmetic, adamw_math.cuh, on the same fp32 gradient values)."""
    rt = _rt()
    cfg, L = EXEC_CFGS[name]
    m = 4
    layers = sd.stage_params(cfg, 0, L, total_layers=max(L, 2))
    costs = rt.make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=1, t_opt=1)
    _, need = rt.rank_program(1, 1, m, None, costs, 0)
    out = []
    for fused in (False, True):
        st = rt.Stage(cfg, L, n_slots=need)
        st.load_master(torch.from_numpy(sd.pack_stage(layers)).float().cuda())
        rt.call("slip_set_fused_adamw", st.ctx, int(fused))
        comm = rt.Comm(0, 1)
        comm.setup(1, 1, m, None)
        io = rt.make_io([host_bf16(sd.stage_input(cfg, 0, j)) for j in range(m)],
                        [host_bf16(sd.stage_target(cfg, 0, j)) for j in range(m)], torch.zeros(m))
        for _ in range(2):
            rep = rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=(1e-3, 0.9, 0.95, 1e-8, 0.1),
                                      iterations=1, io=io)
            assert rep.nonfinite == 0
        torch.cuda.synchronize()
        out.append([st.master.clone(), st.adam_m.clone(), st.adam_v.clone(), st.w.clone()])
        comm.close()
        st.close()
    for a, b, what in zip(out[0], out[1], ("master", "m", "v", "w")):
        assert torch.equal(a, b), (what, ((a.float() - b.float()).abs().max() / a.float().abs().max()).item())


@pytest.mark.parametrize("name", list(EXEC_CFGS))
def test_dual_stream_equals_single_stream(name):
    """slip_set_dual_stream at N = 1: the forwards run on their own (low-priority) stream,
    ordered by events after the W that frees their slot and the OPT that wrote their
    weights.  Three iterations in ONE call (the streams overlap across iterations) must
    leave the gradient, master, m, v and the bf16 weights identical to the single-stream
    run: a forward that read weights before the optimizer step finished, or a slot's stash
    before its W had consumed it, would change them."""
    rt = _rt()
    cfg, L = EXEC_CFGS[name]
    m = 4
    layers = sd.stage_params(cfg, 0, L, total_layers=max(L, 2))
    costs = rt.make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=1, t_opt=1)
    _, need = rt.rank_program(1, 1, m, None, costs, 0)
    out = []
    for dual in (False, True):
        st = rt.Stage(cfg, L, n_slots=need)
        st.load_master(torch.from_numpy(sd.pack_stage(layers)).float().cuda())
        rt.call("slip_set_dual_stream", st.ctx, int(dual))
        comm = rt.Comm(0, 1)
        comm.setup(1, 1, m, None)
        io = rt.make_io([host_bf16(sd.stage_input(cfg, 0, j)) for j in range(m)],
                        [host_bf16(sd.stage_target(cfg, 0, j)) for j in range(m)], torch.zeros(m))
        rep = rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=(1e-3, 0.9, 0.95, 1e-8, 0.1),
                                  iterations=3, io=io)
        torch.cuda.synchronize()
        assert rep.nonfinite == 0
        out.append([st.grad.clone(), st.master.clone(), st.adam_m.clone(), st.adam_v.clone(), st.w.clone()])
        comm.close()
        st.close()
    for a, b, what in zip(out[0], out[1], ("grad", "master", "m", "v", "w")):
        assert torch.equal(a, b), (what, ((a.float() - b.float()).abs().max() / a.float().abs().max()).item())


def test_dual_stream_with_gpt_ends_equals_single_stream():
    """The dual compute stream with both GPT ends on the stage (embedding in F on the
    forward stream; final LN + LM head + CE in LOSS on the backward stream): three
    iterations in one call, gradient / master / m / v / weights / losses identical to the
    single-stream run."""
    rt = _rt()
    cfg = sd.ModelCfg(hidden=128, heads=2, ffn=512, seq=64, micro_batch=2, layers=2, vocab=384, ends=3)
    L, m = 2, 4
    flat = np.concatenate([sd.pack_stage(sd.stage_params(cfg, 0, L, total_layers=2)), sd.pack_ends(sd.end_params(cfg, 0))])
    costs = rt.make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=1, t_opt=1)
    _, need = rt.rank_program(1, 1, m, None, costs, 0)
    toks = [torch.from_numpy(sd.stage_tokens(cfg, 0, j).copy()) for j in range(m)]
    labs = [torch.from_numpy(sd.stage_labels(cfg, 0, j).copy()) for j in range(m)]
    out = []
    for dual in (False, True):
        st = rt.Stage(cfg, L, n_slots=need)
        st.load_master(torch.from_numpy(flat).float().cuda())
        rt.call("slip_set_dual_stream", st.ctx, int(dual))
        comm = rt.Comm(0, 1)
        comm.setup(1, 1, m, None)
        losses = torch.zeros(m)
        io = rt.make_io(toks, labs, losses)
        rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=(1e-3, 0.9, 0.95, 1e-8, 0.1), iterations=3, io=io)
        torch.cuda.synchronize()
        out.append([st.grad.clone(), st.master.clone(), st.adam_m.clone(), st.adam_v.clone(), st.w.clone(),
                    losses.clone()])
        comm.close()
        st.close()
    for a, b, what in zip(out[0], out[1], ("grad", "master", "m", "v", "w", "losses")):
        assert torch.equal(a, b), what


def test_gpt_ends_out_of_range_ids_read_a_zero_row():
    """Token ids outside [0, vocab) read a zero token-embedding row and receive no
    gradient; labels outside it mark ignored tokens (include/slip.h).  Run A feeds three
    invalid ids (-1, V + 7, 2^30) and one ignored label; run B feeds, at those positions,
    an id v0 used nowhere else whose embedding row is zero in both runs.  Losses, weights
    and every gradient except dE[v0] (which B fills from those positions) must be
    bit-identical, and nothing reads or writes out of bounds."""
    rt = _rt()
    cfg = sd.ModelCfg(hidden=128, heads=2, ffn=512, seq=64, micro_batch=2, layers=1, vocab=384, ends=3)
    L, m = 1, 1
    layers = sd.stage_params(cfg, 0, L, total_layers=2)
    ends = sd.end_params(cfg, 0)
    tok = sd.stage_tokens(cfg, 0, 0).copy()
    pos = [3, 17, 40]
    v0 = int(next(v for v in range(cfg.vocab) if v not in set(np.delete(tok, pos).tolist())))
    ends["E"] = ends["E"].copy()
    ends["E"][v0] = 0.0
    flat = np.concatenate([sd.pack_stage(layers), sd.pack_ends(ends)])
    lab = sd.stage_labels(cfg, 0, 0).copy()
    lab[5] = -100
    costs = rt.make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=1, t_opt=1)
    _, need = rt.rank_program(1, 1, m, None, costs, 0)
    out = []
    for bad in (True, False):
        t = tok.copy()
        t[pos] = [-1, cfg.vocab + 7, 2 ** 30] if bad else v0
        st = rt.Stage(cfg, L, n_slots=need)
        st.load_master(torch.from_numpy(flat).float().cuda())
        comm = rt.Comm(0, 1)
        comm.setup(1, 1, m, None)
        losses = torch.zeros(m)
        io = rt.make_io([torch.from_numpy(t)], [torch.from_numpy(lab)], losses)
        rt.execute_schedule(st, comm, 1, 1, m, None, costs, adam=(1e-3, 0.9, 0.95, 1e-8, 0.1), iterations=1, io=io)
        torch.cuda.synchronize()
        out.append([st.grad.clone(), st.master.clone(), losses.clone()])
        comm.close()
        st.close()
    (ga, pa, la), (gb, pb, lb) = out
    assert torch.isfinite(ga).all() and torch.isfinite(la).all()
    assert torch.equal(la, lb)
    row = slice(L * cfg.params_per_layer + v0 * cfg.hidden, L * cfg.params_per_layer + (v0 + 1) * cfg.hidden)
    assert not ga[row].any() and gb[row].any()
    ga[row] = 0
    gb[row] = 0
    pa[row] = 0
    pb[row] = 0
    assert torch.equal(ga, gb) and torch.equal(pa, pb)
