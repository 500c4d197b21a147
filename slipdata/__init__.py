"""Seeded synthetic inputs shared by the oracle tests and the CUDA-path tests.

This module holds NO arithmetic of the method (no layer math, no optimizer, no
planner).  It only draws seeded random numbers, rounds them to bf16 (RNE) so
that both sides consume bit-identical values, and packs per-tensor arrays into
the flat parameter layout documented in ``include/slip.h`` (marshalling only).

Recipe:
  * generator: numpy ``default_rng(SeedSequence([2405, tag, ...]))``
  * weights, tag (1, stage, layer): matrices ~ N(0, 0.02^2); Wo and W2 ~
    N(0, (0.02/sqrt(2L))^2); biases ~ N(0, 0.02^2) (non-zero so the bias
    paths are exercised); gamma ~ 1 + N(0, 0.1^2); beta ~ N(0, 0.1^2)
  * stage inputs X_{k,j} ~ N(0,1), tag (2, k, j); targets R_{k,j} ~ N(0,1),
    tag (3, k, j)
  * everything is rounded to bf16 (RNE); the oracle consumes the same rounded
    values upcast to fp64.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_ROOT = 2405


@dataclass(frozen=True)
class ModelCfg:
    """GPT-shaped stage configuration."""

    hidden: int
    heads: int
    ffn: int
    seq: int
    micro_batch: int
    layers: int
    ln_eps: float = 1e-5
    vocab: int = 0  # padded vocabulary of the GPT ends (reading R33); 0 = no ends
    ends: int = 0   # bit 0: this stage hosts the embedding, bit 1: the LM head

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def tokens(self) -> int:
        return self.seq * self.micro_batch

    @property
    def params_per_layer(self) -> int:
        h, f = self.hidden, self.ffn
        return 3 * h * h + 3 * h + h * h + h + 4 * h + f * h + f + h * f + h


# Configs named in BASELINE.json.
C1_TINY = ModelCfg(hidden=64, heads=2, ffn=256, seq=32, micro_batch=2, layers=1)
C2_1P3B = ModelCfg(hidden=2048, heads=16, ffn=8192, seq=2048, micro_batch=1, layers=24)
C3_2P7B = ModelCfg(hidden=2560, heads=32, ffn=10240, seq=2048, micro_batch=1, layers=32)
C5_6P7B = ModelCfg(hidden=4096, heads=32, ffn=16384, seq=2048, micro_batch=1, layers=32)

# Flat per-layer order, fixed by include/slip.h ("Parameter layout").
PARAM_ORDER = ("wqkv", "bqkv", "wo", "bo", "g1", "b1n", "g2", "b2n", "w1", "b1", "w2", "b2")
MATRICES = ("wqkv", "wo", "w1", "w2")


def param_shapes(cfg: ModelCfg) -> dict:
    h, f = cfg.hidden, cfg.ffn
    return {
        "wqkv": (3 * h, h), "bqkv": (3 * h,), "wo": (h, h), "bo": (h,),
        "g1": (h,), "b1n": (h,), "g2": (h,), "b2n": (h,),
        "w1": (f, h), "b1": (f,), "w2": (h, f), "b2": (h,),
    }


def rng(*tag: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([SEED_ROOT, *[int(t) for t in tag]]))


# ---------------------------------------------------------------- bf16 codec
def to_bf16_bits(x) -> np.ndarray:
    """Round to bf16 with round-to-nearest-even; returns raw uint16 bits."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32)
    bias = ((f >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((f + bias) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def bf16_round(x) -> np.ndarray:
    """Value of x after bf16 RNE rounding, as fp64."""
    return bf16_bits_to_f64(to_bf16_bits(x))


# ---------------------------------------------------------------- generators
def layer_params(cfg: ModelCfg, stage: int, layer: int, total_layers: int | None = None) -> dict:
    """fp64 arrays holding bf16-representable values, keyed by PARAM_ORDER names."""
    L = total_layers if total_layers is not None else cfg.layers
    g = rng(1, stage, layer)
    shapes = param_shapes(cfg)
    out = {}
    for name in PARAM_ORDER:
        shp = shapes[name]
        if name in ("wqkv", "w1"):
            v = g.normal(0.0, 0.02, shp)
        elif name in ("wo", "w2"):
            v = g.normal(0.0, 0.02 / np.sqrt(2.0 * L), shp)
        elif name in ("g1", "g2"):
            v = 1.0 + g.normal(0.0, 0.1, shp)
        elif name in ("b1n", "b2n"):
            v = g.normal(0.0, 0.1, shp)
        else:  # linear biases
            v = g.normal(0.0, 0.02, shp)
        out[name] = bf16_round(v)
    return out


def stage_params(cfg: ModelCfg, stage: int, n_layers: int | None = None, total_layers: int | None = None) -> list:
    n = n_layers if n_layers is not None else cfg.layers
    return [layer_params(cfg, stage, l, total_layers) for l in range(n)]


def stage_input(cfg: ModelCfg, k: int, j: int) -> np.ndarray:
    """X_{k,j}: [T, h] fp64 holding bf16 values."""
    return bf16_round(rng(2, k, j).normal(0.0, 1.0, (cfg.tokens, cfg.hidden)))


def stage_target(cfg: ModelCfg, k: int, j: int) -> np.ndarray:
    """R_{k,j}: [T, h] fp64 holding bf16 values."""
    return bf16_round(rng(3, k, j).normal(0.0, 1.0, (cfg.tokens, cfg.hidden)))


# ---------------------------------------------------------------- marshalling
def pack_layer(params: dict) -> np.ndarray:
    """Flatten one layer's tensors in PARAM_ORDER (row-major) -> fp64 vector."""
    return np.concatenate([np.asarray(params[n], dtype=np.float64).reshape(-1) for n in PARAM_ORDER])


def pack_stage(layers: list) -> np.ndarray:
    return np.concatenate([pack_layer(p) for p in layers])


def unpack_layer(flat: np.ndarray, cfg: ModelCfg) -> dict:
    shapes = param_shapes(cfg)
    out, off = {}, 0
    for n in PARAM_ORDER:
        sz = int(np.prod(shapes[n]))
        out[n] = np.asarray(flat[off:off + sz]).reshape(shapes[n])
        off += sz
    assert off == cfg.params_per_layer
    return out


def unpack_stage(flat: np.ndarray, cfg: ModelCfg, n_layers: int) -> list:
    P = cfg.params_per_layer
    return [unpack_layer(flat[l * P:(l + 1) * P], cfg) for l in range(n_layers)]



# ---------------------------------------------------------------- GPT ends (R33)
END_ORDER = ("E", "P", "gf", "bf", "Wout")


def end_shapes(cfg: ModelCfg) -> dict:
    out = {}
    if cfg.ends & 1:
        out["E"] = (cfg.vocab, cfg.hidden)
        out["P"] = (cfg.seq, cfg.hidden)
    if cfg.ends & 2:
        out["gf"] = (cfg.hidden,)
        out["bf"] = (cfg.hidden,)
        out["Wout"] = (cfg.vocab, cfg.hidden)
    return out


def end_params(cfg: ModelCfg, stage: int) -> dict:
    """fp64 arrays of bf16 values: E, P, Wout ~ N(0, 0.02^2), gf = 1 + N(0, 0.1^2), bf ~ N(0, 0.1^2)."""
    g = rng(4, stage)
    out = {}
    for n, shp in end_shapes(cfg).items():
        if n in ("E", "P", "Wout"):
            v = g.normal(0.0, 0.02, shp)
        elif n == "gf":
            v = 1.0 + g.normal(0.0, 0.1, shp)
        else:
            v = g.normal(0.0, 0.1, shp)
        out[n] = bf16_round(v)
    return out


def pack_ends(params: dict) -> np.ndarray:
    return np.concatenate([np.asarray(params[n], dtype=np.float64).reshape(-1) for n in END_ORDER if n in params]
                          or [np.zeros(0)])


def unpack_ends(flat: np.ndarray, cfg: ModelCfg) -> dict:
    out, off = {}, 0
    for n, shp in end_shapes(cfg).items():
        sz = int(np.prod(shp))
        out[n] = np.asarray(flat[off:off + sz]).reshape(shp)
        off += sz
    return out


def stage_tokens(cfg: ModelCfg, k: int, j: int, classes: int | None = None) -> np.ndarray:
    """Token ids of micro-batch (k, j): T int32 uniform over the (padded) vocabulary."""
    return rng(5, k, j).integers(0, classes or cfg.vocab, cfg.tokens).astype(np.int32)


def stage_labels(cfg: ModelCfg, k: int, j: int, classes: int | None = None) -> np.ndarray:
    """Labels of micro-batch (k, j): T int32 uniform over the (padded) vocabulary."""
    return rng(6, k, j).integers(0, classes or cfg.vocab, cfg.tokens).astype(np.int32)
