"""Stage-level parity: the CUDA path through the C ABI (slip_stage_forward,
slip_backward_input, slip_backward_weight, slip_optimizer_step) against the
fp64 oracle on the same seeded bf16 inputs.

Tolerances (BASELINE.json north_star):
  * bf16 tensor-core paths: normwise relative error ||g - r||_inf / ||r||_inf <= 2e-2
  * fp32 optimizer: <= 1e-4 (on identical fp32 inputs)
  * decoupled B + W vs coupled backward on the GPU: bit-exact
"""
import numpy as np
import pytest
import torch

import slipdata as sd
from oracle import adam as OA
from oracle import layer as OL

pytestmark = pytest.mark.gpu

GATE_A = 2e-2
GATE_B = 1e-4


def _rt():
    from paper_2405_14009_b200 import runtime
    return runtime


def relerr(g, r):
    g = np.asarray(g, dtype=np.float64)
    return float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))


def to_dev_bf16(x):
    bits = sd.to_bf16_bits(x)
    return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).cuda()


def to_np(t):
    return t.float().cpu().numpy().astype(np.float64)


def run_stage(cfg, n_layers, seed_k=0, seed_j=0):
    rt = _rt()
    layers = sd.stage_params(cfg, 0, n_layers, total_layers=max(n_layers, 2))
    flat = sd.pack_stage(layers)
    st = rt.Stage(cfg, n_layers, n_slots=2)
    st.load_master(torch.from_numpy(flat).float().cuda())
    x = sd.stage_input(cfg, seed_k, seed_j)
    r = sd.stage_target(cfg, seed_k, seed_j)
    xd, rd = to_dev_bf16(x), to_dev_bf16(r)
    y = torch.empty_like(xd)
    dx = torch.empty_like(xd)
    st.forward(0, xd, y)
    st.backward_input(0, rd, dx, accumulate=False)
    st.backward_weight(0, accumulate=False)
    torch.cuda.synchronize()
    return st, layers, x, r, y, dx


CFGS = {
    "c1": (sd.C1_TINY, 1),
    "c1x2": (sd.C1_TINY, 2),
    "d80_ragged": (sd.ModelCfg(hidden=640, heads=8, ffn=2560, seq=200, micro_batch=1, layers=1), 1),
    "d128_b2": (sd.ModelCfg(hidden=512, heads=4, ffn=2048, seq=384, micro_batch=2, layers=1), 1),
    "d64": (sd.ModelCfg(hidden=256, heads=4, ffn=1024, seq=136, micro_batch=2, layers=1), 1),
}


@pytest.mark.parametrize("name", list(CFGS))
def test_stage_step_matches_oracle(name):
    cfg, L = CFGS[name]
    st, layers, x, r, y, dx = run_stage(cfg, L)
    out, caches = OL.stage_forward(layers, x, cfg)
    dxr, grads = OL.stage_backward_coupled(layers, caches, r, cfg)
    assert relerr(to_np(y), out) <= GATE_A
    assert relerr(to_np(dx), dxr) <= GATE_A
    g = sd.unpack_stage(st.grad.cpu().numpy().astype(np.float64), cfg, L)
    for l in range(L):
        for n in sd.PARAM_ORDER:
            e = relerr(g[l][n], grads[l][n])
            assert e <= GATE_A, (name, l, n, e)


def test_decoupled_equals_coupled_on_gpu():
    """B then W (deferred) and the coupled backward produce bit-identical grads."""
    cfg = sd.C1_TINY
    st, layers, x, r, y, dx = run_stage(cfg, 2)
    g1 = st.grad.clone()
    xd, rd = to_dev_bf16(x), to_dev_bf16(r)
    dx2 = torch.empty_like(xd)
    st.forward(1, xd, y)
    st.backward_coupled(1, rd, dx2, accumulate=False)
    torch.cuda.synchronize()
    assert torch.equal(st.grad, g1)
    assert torch.equal(dx, dx2)


def test_accumulation_over_microbatches():
    cfg = sd.C1_TINY
    rt = _rt()
    layers = sd.stage_params(cfg, 0, 1)
    st = rt.Stage(cfg, 1, n_slots=2)
    st.load_master(torch.from_numpy(sd.pack_stage(layers)).float().cuda())
    ref = None
    for j in range(3):
        x, r = sd.stage_input(cfg, 0, j), sd.stage_target(cfg, 0, j)
        y = torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device="cuda")
        st.forward(j % 2, to_dev_bf16(x), y)
        st.backward_input(j % 2, to_dev_bf16(r), None, accumulate=j > 0)
        st.backward_weight(j % 2, accumulate=j > 0)
        out, c = OL.stage_forward(layers, x, cfg)
        _, g = OL.stage_backward_coupled(layers, c, r, cfg)
        ref = g if ref is None else [{n: a[n] + b[n] for n in a} for a, b in zip(ref, g)]
    torch.cuda.synchronize()
    got = sd.unpack_stage(st.grad.cpu().numpy().astype(np.float64), cfg, 1)
    for n in sd.PARAM_ORDER:
        assert relerr(got[0][n], ref[0][n]) <= GATE_A, n


def test_stream_k_stage_matches_oracle():
    """The hybrid stream-K linears (slip_set_stream_k, off by default): a shape whose QKV
    (96 pair tiles) and FC1 (128) GEMMs leave a partial last wave of the 74 CTA pairs, so
    split tiles are finished from other pairs' fp32 partials."""
    rt = _rt()
    cfg = sd.ModelCfg(hidden=1024, heads=8, ffn=4096, seq=1024, micro_batch=2, layers=1)
    layers = sd.stage_params(cfg, 0, 1, total_layers=2)
    st = rt.Stage(cfg, 1, n_slots=1)
    rt.call("slip_set_stream_k", st.ctx, 1)
    st.load_master(torch.from_numpy(sd.pack_stage(layers)).float().cuda())
    x, r = sd.stage_input(cfg, 0, 0), sd.stage_target(cfg, 0, 0)
    y = torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    dx = torch.empty_like(y)
    st.forward(0, to_dev_bf16(x), y)
    st.backward_input(0, to_dev_bf16(r), dx, accumulate=False)
    st.backward_weight(0, accumulate=False)
    torch.cuda.synchronize()
    out, caches = OL.stage_forward(layers, x, cfg)
    dxr, grads = OL.stage_backward_coupled(layers, caches, r, cfg)
    assert relerr(to_np(y), out) <= GATE_A
    assert relerr(to_np(dx), dxr) <= GATE_A
    g = sd.unpack_stage(st.grad.cpu().numpy().astype(np.float64), cfg, 1)
    for n in sd.PARAM_ORDER:
        assert relerr(g[0][n], grads[0][n]) <= GATE_A, n


@pytest.mark.parametrize("name", ["c1", "d80_ragged"])
def test_weight_multi_matches_oracle(name):
    """slip_backward_weight_multi: the W of 3 micro-batches in one launch (K = 3T over the
    slots) equals the oracle's summed weight gradients; biases / LayerNorm come from B."""
    cfg, L = CFGS[name]
    rt = _rt()
    layers = sd.stage_params(cfg, 0, L, total_layers=max(L, 2))
    st = rt.Stage(cfg, L, n_slots=4)
    st.load_master(torch.from_numpy(sd.pack_stage(layers)).float().cuda())
    ref = None
    order = [2, 0, 3]  # slots used out of order
    for j, slot in enumerate(order):
        x, r = sd.stage_input(cfg, 0, j), sd.stage_target(cfg, 0, j)
        y = torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device="cuda")
        st.forward(slot, to_dev_bf16(x), y)
        st.backward_input(slot, to_dev_bf16(r), None, accumulate=j > 0)
        out, c = OL.stage_forward(layers, x, cfg)
        _, g = OL.stage_backward_coupled(layers, c, r, cfg)
        ref = g if ref is None else [{n: a[n] + b[n] for n in a} for a, b in zip(ref, g)]
    st.backward_weight_multi(order, accumulate=False)
    torch.cuda.synchronize()
    got = sd.unpack_stage(st.grad.cpu().numpy().astype(np.float64), cfg, L)
    for l in range(L):
        for n in sd.PARAM_ORDER:
            assert relerr(got[l][n], ref[l][n]) <= GATE_A, (name, l, n)
    # the slots are free again
    x = sd.stage_input(cfg, 0, 0)
    y = torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    st.forward(2, to_dev_bf16(x), y)


def test_slot_state_machine():
    rt = _rt()
    cfg = sd.C1_TINY
    st = rt.Stage(cfg, 1, n_slots=1)
    d = torch.zeros(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rt.SlipError) as e:
        st.backward_input(0, d, d)
    assert e.value.code == 4  # SLIP_ESTATE: B before F
    st.forward(0, d, d.clone())
    with pytest.raises(rt.SlipError):
        st.forward(0, d, d.clone())
    with pytest.raises(rt.SlipError):
        st.backward_weight(0)


def test_adamw_matches_oracle():
    """Fused AdamW on identical fp32 inputs (GPU gradients fed to both)."""
    cfg = sd.C1_TINY
    st, layers, x, r, y, dx = run_stage(cfg, 1)
    p0 = st.master.cpu().numpy().astype(np.float64)
    g = st.grad.cpu().numpy().astype(np.float64)
    acfg = OA.AdamCfg(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    P = sd.unpack_layer(p0, cfg)
    G = sd.unpack_layer(g, cfg)
    Z = {n: np.zeros_like(v) for n, v in P.items()}
    m, v = Z, Z
    for step in (1, 2, 3):
        st.optimizer_step(step, lr=acfg.lr, beta1=acfg.beta1, beta2=acfg.beta2, eps=acfg.eps,
                          weight_decay=acfg.weight_decay, grad_scale=0.25, nonfinite=flag)
        P, m, v = OA.adamw_step_layer(P, m, v, G, step, acfg, grad_scale=0.25)
    torch.cuda.synchronize()
    got = st.master.cpu().numpy().astype(np.float64)
    ref = sd.pack_layer(P)
    # compare the accumulated update p - p0 (the quantity Adam computes)
    assert relerr(got - p0, ref - p0) <= GATE_B
    assert relerr(st.adam_m.cpu().numpy().astype(np.float64), sd.pack_layer(m)) <= GATE_B
    assert relerr(st.adam_v.cpu().numpy().astype(np.float64), sd.pack_layer(v)) <= GATE_B
    assert int(flag.item()) == 0
    # bf16 weights = RNE(master)
    w = st.w.float().cpu().numpy().astype(np.float64)
    assert np.array_equal(w, sd.bf16_round(got))
    # non-finite flag
    st.grad[5] = float("inf")
    st.optimizer_step(4, nonfinite=flag)
    torch.cuda.synchronize()
    assert int(flag.item()) == 1


def test_adamw_rollback_reverses_the_step():
    """slip_optimizer_rollback (reading R31) against the oracle's
    inverse: after 3 steps, reversing step 3 on the GPU restores master / m / v to the
    state after step 2 within fp32 reversal error, and the bf16 copy is RNE(master)."""
    from paper_2405_14009_b200._binding import slip_adam
    import ctypes as C
    rt = _rt()
    cfg = sd.C1_TINY
    st, layers, x, r, y, dx = run_stage(cfg, 1)
    for step in (1, 2):
        st.optimizer_step(step, grad_scale=0.25)
    torch.cuda.synchronize()
    p2, m2, v2 = st.master.clone(), st.adam_m.clone(), st.adam_v.clone()
    st.optimizer_step(3, grad_scale=0.25)
    a = slip_adam(1e-3, 0.9, 0.95, 1e-8, 0.1)
    rt.call("slip_optimizer_rollback", st.ctx, C.byref(a), 3, 0.25, rt._stream())
    torch.cuda.synchronize()
    assert ((st.master - p2).abs().max() / p2.abs().max()).item() <= 1e-6
    assert ((st.adam_m - m2).abs().max() / m2.abs().max()).item() <= 1e-5
    assert ((st.adam_v - v2).abs().max() / v2.abs().max()).item() <= 1e-4
    w = st.w.float().cpu().numpy().astype(np.float64)
    assert np.array_equal(w, sd.bf16_round(st.master.cpu().numpy().astype(np.float64)))


def test_mse_head_and_synth():
    rt = _rt()
    cfg = sd.C1_TINY
    st = rt.Stage(cfg, 1, n_slots=1)
    y, r = sd.stage_input(cfg, 1, 2), sd.stage_target(cfg, 1, 2)
    dy = torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    loss = torch.zeros(1, device="cuda")
    st.loss_mse(to_dev_bf16(y), to_dev_bf16(r), dy, loss)
    torch.cuda.synchronize()
    lref, dref = OL.loss_mse(y, r)
    assert abs(loss.item() - lref) <= 1e-4 * lref
    assert relerr(to_np(dy), dref) <= GATE_A
    a = torch.empty(1 << 16, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    rt.synth_normal(a, 7, 1, 2)
    rt.synth_normal(b, 7, 1, 2)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    af = a.float()
    assert abs(af.mean().item()) < 0.02 and abs(af.std().item() - 1.0) < 0.02


@pytest.mark.slow
def test_one_layer_c2_full_size():
    """One GPT-1.3B-shaped layer at full size (h 2048, s 2048, 16 heads), fp64 oracle on the host."""
    cfg = sd.ModelCfg(hidden=2048, heads=16, ffn=8192, seq=2048, micro_batch=1, layers=24)
    st, layers, x, r, y, dx = run_stage(cfg, 1)
    out, caches = OL.stage_forward(layers, x, cfg)
    dxr, grads = OL.stage_backward_coupled(layers, caches, r, cfg)
    assert relerr(to_np(y), out) <= GATE_A
    assert relerr(to_np(dx), dxr) <= GATE_A
    g = sd.unpack_stage(st.grad.cpu().numpy().astype(np.float64), cfg, 1)
    for n in sd.PARAM_ORDER:
        assert relerr(g[0][n], grads[0][n]) <= GATE_A, n


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c3_2p7b", "c5_6p7b"])
def test_one_layer_full_size_larger_models(name):
    """One layer of the GPT-2.7B (h 2560, 32 heads of d = 80) and GPT-6.7B (h 4096, 32 heads
    of d = 128) shapes of BASELINE.json configs at full size (s 2048), fp64 oracle."""
    cfg = {"c3_2p7b": sd.C3_2P7B, "c5_6p7b": sd.C5_6P7B}[name]
    st, layers, x, r, y, dx = run_stage(cfg, 1)
    out, caches = OL.stage_forward(layers, x, cfg)
    dxr, grads = OL.stage_backward_coupled(layers, caches, r, cfg)
    assert relerr(to_np(y), out) <= GATE_A
    assert relerr(to_np(dx), dxr) <= GATE_A
    g = sd.unpack_stage(st.grad.cpu().numpy().astype(np.float64), cfg, 1)
    for n in sd.PARAM_ORDER:
        assert relerr(g[0][n], grads[0][n]) <= GATE_A, (name, n)


ENDS_CFGS = {
    "tiny_both": (sd.ModelCfg(hidden=64, heads=2, ffn=256, seq=32, micro_batch=2, layers=1, vocab=256, ends=3), 1),
    "d128_both": (sd.ModelCfg(hidden=256, heads=2, ffn=1024, seq=128, micro_batch=2, layers=2, vocab=384, ends=3), 2),
    "emb_only": (sd.ModelCfg(hidden=128, heads=2, ffn=512, seq=64, micro_batch=1, layers=1, vocab=256, ends=1), 1),
    "head_only": (sd.ModelCfg(hidden=128, heads=2, ffn=512, seq=64, micro_batch=1, layers=1, vocab=256, ends=2), 1),
}


@pytest.mark.parametrize("name", list(ENDS_CFGS))
def test_stage_with_gpt_ends_matches_oracle(name):
    """GPT ends (reading R33): embedding (tokens in), layers,
    final LayerNorm + LM head + cross-entropy (labels in), B, W (with dWout in the
    grouped launch and the embedding scatter) against oracle/ends.py + oracle/layer.py."""
    from oracle import ends as OE
    rt = _rt()
    cfg, L = ENDS_CFGS[name]
    layers = sd.stage_params(cfg, 0, L, total_layers=max(L, 2))
    ends = sd.end_params(cfg, 0)
    flat = np.concatenate([sd.pack_stage(layers), sd.pack_ends(ends)])
    st = rt.Stage(cfg, L, n_slots=1)
    assert st.n_params == flat.size
    st.load_master(torch.from_numpy(flat).float().cuda())
    T, h = cfg.tokens, cfg.hidden
    tok = sd.stage_tokens(cfg, 0, 0)
    tok[5] = tok[9] = tok[17]  # repeated tokens in the scatter
    lab = sd.stage_labels(cfg, 0, 0)
    x_in = torch.from_numpy(tok).cuda() if cfg.ends & 1 else to_dev_bf16(sd.stage_input(cfg, 0, 0))
    y = torch.empty(T, h, dtype=torch.bfloat16, device="cuda")
    dy = torch.empty_like(y)
    dx = torch.empty_like(y)
    loss = torch.zeros(1, device="cuda")
    st.forward(0, x_in, y)
    if cfg.ends & 2:
        st.loss_ce(0, y, torch.from_numpy(lab).cuda(), dy, loss)
    else:
        dy.copy_(to_dev_bf16(sd.stage_target(cfg, 0, 0)))
    st.backward_input(0, dy, dx, accumulate=False)
    st.backward_weight(0, accumulate=False)
    torch.cuda.synchronize()
    # oracle
    x0 = OE.embed_fwd(ends["E"], ends["P"], tok, cfg.seq) if cfg.ends & 1 else sd.stage_input(cfg, 0, 0)
    out, caches = OL.stage_forward(layers, x0, cfg)
    assert relerr(to_np(y), out) <= GATE_A
    if cfg.ends & 2:
        lref, hc = OE.head_forward(out, ends["gf"], ends["bf"], ends["Wout"], lab, cfg.ln_eps)
        assert abs(loss.item() - lref) <= 1e-2 * abs(lref)
        dout, hb, hws = OE.head_backward_input(hc)
        assert relerr(to_np(dy), dout) <= GATE_A
    else:
        dout = sd.stage_target(cfg, 0, 0)
    dxr, grads = OL.stage_backward_coupled(layers, caches, dout, cfg)
    assert relerr(to_np(dx), dxr) <= GATE_A
    gflat = st.grad.cpu().numpy().astype(np.float64)
    P = cfg.params_per_layer
    g = sd.unpack_stage(gflat[:L * P], cfg, L)
    for l in range(L):
        for n in sd.PARAM_ORDER:
            assert relerr(g[l][n], grads[l][n]) <= GATE_A, (l, n)
    ge = sd.unpack_ends(gflat[L * P:], cfg)
    if cfg.ends & 1:
        dE, dP = OE.embed_bwd(dxr, tok, cfg.seq, cfg.vocab)
        assert relerr(ge["E"], dE) <= GATE_A and relerr(ge["P"], dP) <= GATE_A
        assert np.all(ge["E"][np.setdiff1d(np.arange(cfg.vocab), tok)] == 0.0)  # untouched rows stay 0
    if cfg.ends & 2:
        assert relerr(ge["gf"], hb["gf"]) <= GATE_A and relerr(ge["bf"], hb["bf"]) <= GATE_A
        assert relerr(ge["Wout"], OE.head_backward_weight(hws)["Wout"]) <= GATE_A


def test_weight_multi_with_gpt_ends_equals_separate_w():
    """The merged W (slip_backward_weight_multi) with both model ends — dWout in the grouped
    launch, embedding scatter per slot — equals separate per-slot W calls up to fp32
    summation order (the separate path is pinned to the oracle above)."""
    rt = _rt()
    cfg, L = ENDS_CFGS["d128_both"]
    layers = sd.stage_params(cfg, 0, L, total_layers=max(L, 2))
    flat = np.concatenate([sd.pack_stage(layers), sd.pack_ends(sd.end_params(cfg, 0))])
    T, h = cfg.tokens, cfg.hidden
    grads = []
    for merged in (False, True):
        st = rt.Stage(cfg, L, n_slots=3)
        st.load_master(torch.from_numpy(flat).float().cuda())
        for j, slot in enumerate((1, 2)):
            tok = torch.from_numpy(sd.stage_tokens(cfg, 0, j)).cuda()
            lab = torch.from_numpy(sd.stage_labels(cfg, 0, j)).cuda()
            y = torch.empty(T, h, dtype=torch.bfloat16, device="cuda")
            dy, dx = torch.empty_like(y), torch.empty_like(y)
            loss = torch.zeros(1, device="cuda")
            st.forward(slot, tok, y)
            st.loss_ce(slot, y, lab, dy, loss)
            st.backward_input(slot, dy, dx, accumulate=j > 0)
        if merged:
            st.backward_weight_multi([2, 1], accumulate=False)
        else:
            st.backward_weight(1, accumulate=False)
            st.backward_weight(2, accumulate=True)
        torch.cuda.synchronize()
        grads.append(st.grad.clone())
    a, b = grads
    assert torch.isfinite(b).all()
    assert ((a - b).abs().max() / a.abs().max()).item() <= 1e-5
