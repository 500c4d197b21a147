"""Pins for oracle/adam.py: step-1 closed form, torch.optim.AdamW (fp64),
zero-gradient decay, non-finite flag."""
import numpy as np
import torch

from oracle.adam import AdamCfg, adamw_step, adamw_step_layer, nonfinite

CFG = AdamCfg(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)


def test_step1_closed_form():
    rng = np.random.default_rng(0)
    p0 = rng.normal(size=1000)
    g = rng.normal(size=1000)
    p1, m1, v1 = adamw_step(p0, np.zeros(1000), np.zeros(1000), g, 1, CFG)
    # mhat = g, vhat = g^2 at t = 1
    ref = p0 - CFG.lr * CFG.weight_decay * p0 - CFG.lr * g / (np.abs(g) + CFG.eps)
    assert np.max(np.abs(p1 - ref) / np.abs(ref)) <= 1e-15
    assert np.array_equal(m1, (1 - CFG.beta1) * g)


def test_matches_torch_adamw_fp64():
    rng = np.random.default_rng(1)
    p = rng.normal(size=(17, 9))
    tp = torch.nn.Parameter(torch.tensor(p))
    opt = torch.optim.AdamW([tp], lr=CFG.lr, betas=(CFG.beta1, CFG.beta2), eps=CFG.eps,
                            weight_decay=CFG.weight_decay)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    scale = 0.25
    for t in range(1, 6):
        g = rng.normal(size=p.shape)
        tp.grad = torch.tensor(g * scale)
        opt.step()
        p, m, v = adamw_step(p, m, v, g, t, CFG, grad_scale=scale)
        ref = tp.detach().numpy()
        assert np.max(np.abs(p - ref) / np.abs(ref)) <= 1e-15


def test_zero_grad_is_pure_decay_and_bias_not_decayed():
    p = {"w": np.ones((3, 4)), "b": np.ones(4)}
    z = {k: np.zeros_like(v) for k, v in p.items()}
    np_, _, _ = adamw_step_layer(p, z, z, z, 1, CFG)
    assert np.array_equal(np_["w"], np.ones((3, 4)) * (1 - CFG.lr * CFG.weight_decay))
    assert np.array_equal(np_["b"], np.ones(4))


def test_nonfinite_flag():
    assert not nonfinite({"a": np.ones(3)})
    assert nonfinite({"a": np.array([1.0, np.inf])})
    assert nonfinite({"a": np.array([np.nan])})


def test_adamw_inverse_round_trip_and_step1_closed_form():
    """Rollback pins (reading R31): the inverse undoes a step to
    fp64 rounding for random states and steps; at step 1 from m = v = 0 it recovers
    exactly zero moments and the closed form p0 = (p1 + lr sign(g)) / (1 - lr wd)
    (|g| >> eps)."""
    import numpy as np
    from oracle import adam as A
    rng = np.random.default_rng(31)
    cfg = A.AdamCfg()
    for t in (1, 2, 7, 100):
        p0 = rng.standard_normal(1000)
        m0 = rng.standard_normal(1000) * 1e-2 if t > 1 else np.zeros(1000)
        v0 = rng.random(1000) * 1e-3 if t > 1 else np.zeros(1000)
        g = rng.standard_normal(1000)
        for decay in (True, False):
            p1, m1, v1 = A.adamw_step(p0, m0, v0, g, t, cfg, grad_scale=0.25, decay=decay)
            q0, n0, w0 = A.adamw_inverse(p1, m1, v1, g, t, cfg, grad_scale=0.25, decay=decay)
            assert np.allclose(q0, p0, rtol=1e-12, atol=1e-14)
            assert np.allclose(n0, m0, rtol=1e-10, atol=1e-16)
            assert np.allclose(w0, v0, rtol=1e-8, atol=1e-16)
    g = rng.standard_normal(100)
    p0 = rng.standard_normal(100)
    p1, m1, v1 = A.adamw_step(p0, np.zeros(100), np.zeros(100), g, 1, cfg)
    assert np.allclose(p1, p0 - cfg.lr * cfg.weight_decay * p0 - cfg.lr * np.sign(g), atol=1e-9)
    q0, n0, w0 = A.adamw_inverse(p1, m1, v1, g, 1, cfg)
    assert np.allclose(n0, 0.0, atol=1e-15) and np.allclose(w0, 0.0, atol=1e-15)
