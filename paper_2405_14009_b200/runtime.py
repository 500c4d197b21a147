"""Thin Python runtime over libslip: torch allocates device memory and provides
streams / process groups; the library does all compute.  Names follow
include/slip.h."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._binding import (SlipError, call, lib, slip_adam, slip_cluster, slip_costs, slip_io, slip_model, slip_op,
                       slip_plan_opts, slip_report, slip_swap, slip_trace_rec)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _stream(stream=None) -> C.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_model(cfg) -> slip_model:
    return slip_model(cfg.hidden, cfg.heads, cfg.ffn, cfg.seq, cfg.micro_batch, cfg.ln_eps,
                      getattr(cfg, "vocab", 0), getattr(cfg, "ends", 0))


def make_cluster(N: int, DP: int, m: int, live=None):
    """live: iterable over stages of iterables over pipelines (1 = functional)."""
    flat = [1] * (N * DP) if live is None else [int(bool(x)) for row in live for x in row]
    arr = (C.c_uint8 * (N * DP))(*flat)
    cl = slip_cluster(N, DP, m, C.cast(arr, C.POINTER(C.c_uint8)))
    cl._keep = arr  # keep the buffer alive with the struct
    return cl


def param_offsets(h: int, f: int) -> dict:
    """Element offsets of one layer's tensors in the flat parameter vector
    (include/slip.h "Parameter layout")."""
    names = [("wqkv", 3 * h * h), ("bqkv", 3 * h), ("wo", h * h), ("bo", h), ("g1", h), ("b1n", h), ("g2", h),
             ("b2n", h), ("w1", f * h), ("b1", f), ("w2", h * f), ("b2", h)]
    out, off = {}, 0
    for n, sz in names:
        out[n] = (off, sz)
        off += sz
    out["per_layer"] = off
    return out


def init_master_(master, cfg, n_layers, total_layers, seed=0):
    """Synthetic random init on the device (throughput runs): matrices ~ N(0, 0.02^2)
    (Wo, W2 scaled by 1/sqrt(2L)), biases 0, LayerNorm gamma 1, beta 0."""
    import math

    import torch
    g = torch.Generator(device=master.device).manual_seed(seed)
    po = param_offsets(cfg.hidden, cfg.ffn)
    P = po["per_layer"]
    master.zero_()
    for l in range(n_layers):
        base = l * P
        for n in ("wqkv", "wo", "w1", "w2"):
            off, sz = po[n]
            std = 0.02 / math.sqrt(2.0 * total_layers) if n in ("wo", "w2") else 0.02
            master[base + off: base + off + sz].normal_(0.0, std, generator=g)
        for n in ("g1", "g2"):
            off, sz = po[n]
            master[base + off: base + off + sz].fill_(1.0)
    # GPT ends after the layers (reading R33): E, P, Wout ~ N(0, 0.02^2), gf = 1, bf = 0
    off = n_layers * P
    ends, V, h = getattr(cfg, "ends", 0), getattr(cfg, "vocab", 0), cfg.hidden
    if ends & 1:
        master[off: off + (V + cfg.seq) * h].normal_(0.0, 0.02, generator=g)
        off += (V + cfg.seq) * h
    if ends & 2:
        master[off: off + h].fill_(1.0)
        off += 2 * h
        master[off: off + V * h].normal_(0.0, 0.02, generator=g)


def make_costs(t_f=1, t_b=1, t_w=1, t_comm=0, t_ar=0, t_opt=0, a_f=0, a_w=0, m_limit=0) -> slip_costs:
    return slip_costs(t_f, t_b, t_w, t_comm, t_ar, t_opt, a_f, a_w, m_limit)


@dataclass
class PlanResult:
    ops: list          # list of op tuples (stage, mb, origin, phase, exec, iter, start, end)
    makespans: list
    period: int
    hash: int


def plan_schedule(N, DP, m, live, costs: slip_costs, decoupled=True, staggered=True, horizon=3) -> PlanResult:
    cl = make_cluster(N, DP, m, live)
    opts = slip_plan_opts(int(decoupled), int(staggered), int(horizon))
    n = C.c_int64(0)
    call("slip_plan_schedule", C.byref(cl), C.byref(costs), C.byref(opts), None, 0, C.byref(n), None, None)
    ops = (slip_op * max(1, n.value))()
    mk = (C.c_int64 * max(1, horizon))()
    per = C.c_int64(0)
    call("slip_plan_schedule", C.byref(cl), C.byref(costs), C.byref(opts), ops, n.value, C.byref(n), mk,
         C.byref(per))
    h = lib().slip_plan_hash(ops, n.value)
    return PlanResult([ops[i].key() for i in range(n.value)], [mk[i] for i in range(horizon)], per.value, h)


def rank_program(N, DP, m, live, costs: slip_costs, rank, decoupled=True, staggered=True, horizon=1):
    """The executor's action list for `rank` (host logic only): list of
    (kind, iter, mb, origin, peer, slot, accumulate) tuples, and slots needed."""
    from ._binding import slip_action
    cl = make_cluster(N, DP, m, live)
    opts = slip_plan_opts(int(decoupled), int(staggered), int(horizon))
    n, ns = C.c_int64(0), C.c_int32(0)
    call("slip_rank_program", C.byref(cl), C.byref(costs), C.byref(opts), rank, None, 0, C.byref(n), C.byref(ns))
    buf = (slip_action * max(1, n.value))()
    call("slip_rank_program", C.byref(cl), C.byref(costs), C.byref(opts), rank, buf, n.value, C.byref(n),
         C.byref(ns))
    return [buf[i].key() for i in range(n.value)], ns.value


def assign(N, DP, m, live):
    cl = make_cluster(N, DP, m, live)
    out = (C.c_int32 * (N * m * DP))()
    call("slip_assign", C.byref(cl), out)
    return {(i, j, k): out[(i * m + j) * DP + k] for i in range(N) for j in range(m) for k in range(DP)}


def attention(qkv, s, heads, batch, d, out, lse, o=None, d_o=None, dsum=None, backward=False, stream=None):
    """Diagnostic call of the fused attention kernels (see include/slip.h slip_attention)."""
    call("slip_attention", s, heads, batch, d, _ptr(qkv), _ptr(o) if o is not None else None,
         _ptr(d_o) if d_o is not None else None, _ptr(out), _ptr(lse), _ptr(dsum) if dsum is not None else None,
         int(bool(backward)), _stream(stream))


def set_trace(stage, enable=True):
    call("slip_set_trace", stage.ctx, int(bool(enable)))


def get_trace(stage):
    """[(kind_name, mb, origin, iter, peer, slot, begin_ms, end_ms)] of the last traced run."""
    from ._binding import ACTIONS
    n = C.c_int64(0)
    call("slip_get_trace", stage.ctx, None, 0, C.byref(n))
    buf = (slip_trace_rec * max(1, n.value))()
    call("slip_get_trace", stage.ctx, buf, n.value, C.byref(n))
    return [(ACTIONS[r.kind], r.mb, r.origin, r.iter, r.peer, r.slot, r.begin_ms, r.end_ms) for r in buf[:n.value]]


def set_sm_reserve(n: int):
    """Leave n SMs free of persistent GEMM CTAs (for concurrent NCCL kernels)."""
    call("slip_set_sm_reserve", int(n))


def rank_of(N, i, k) -> int:
    """Role rank of worker (stage i, pipeline k) (include/slip.h slip_cluster)."""
    return k * N + i


def normalize_costs(N, DP, m, costs: slip_costs, F, decoupled=True, staggered=True, horizon=3):
    """cost(i, x) table of the heuristic (reading R28): {(i, x): int or None (infinite)}."""
    cl = make_cluster(N, DP, m, None)
    opts = slip_plan_opts(int(decoupled), int(staggered), int(horizon))
    out = (C.c_int64 * (N * (F + 1)))()
    call("slip_normalize_costs", C.byref(cl), C.byref(costs), C.byref(opts), int(F), out)
    inf = (1 << 63) - 1
    return {(i, x): (None if out[i * (F + 1) + x] == inf else out[i * (F + 1) + x])
            for i in range(N) for x in range(F + 1)}


def normalize(N, DP, F, cost_table):
    """Algorithm 1 over {(i, x): cost}; returns (R, C)
    with C[i][f] None where no assignment exists."""
    W = F + 1
    inf = (1 << 63) - 1
    tab = (C.c_int64 * (N * W))(*[inf if cost_table.get((i, x)) is None else int(cost_table[(i, x)])
                                  for i in range(N) for x in range(W)])
    Cout = (C.c_int64 * (N * W))()
    R = (C.c_int32 * N)()
    call("slip_normalize", N, DP, F, tab, Cout, R)
    return list(R), [[None if Cout[i * W + f] == inf else Cout[i * W + f] for f in range(W)] for i in range(N)]


def normalized_live(N, DP, R):
    out = (C.c_uint8 * (N * DP))()
    call("slip_normalized_live", N, DP, (C.c_int32 * N)(*R), out)
    return [[out[i * DP + k] for k in range(DP)] for i in range(N)]


def migration_plan(N, DP, live, R):
    """[((i, k), (i2, k2), k_src)], live-after (see include/slip.h slip_migration_plan)."""
    cl = make_cluster(N, DP, 1, live)
    Rb = (C.c_int32 * N)(*R)
    n = C.c_int32(0)
    call("slip_migration_plan", C.byref(cl), Rb, None, 0, C.byref(n), None)
    sw = (slip_swap * max(1, n.value))()
    after = (C.c_uint8 * (N * DP))()
    call("slip_migration_plan", C.byref(cl), Rb, sw, n.value, C.byref(n), after)
    swaps = [((s.failed_stage, s.failed_pipe), (s.target_stage, s.target_pipe), s.source_pipe)
             for s in sw[:n.value]]
    return swaps, [[after[i * DP + k] for k in range(DP)] for i in range(N)]


def recoverable(N, DP, live) -> bool:
    cl = make_cluster(N, DP, 1, live)
    r = C.c_int32(0)
    call("slip_recoverable", C.byref(cl), C.byref(r))
    return bool(r.value)


class Stage:
    """One stage of `n_layers` layers on the current CUDA device, with `n_slots`
    in-flight micro-batch slots (F-stash + W-stash each)."""

    def __init__(self, cfg, n_layers: int, n_slots: int, device="cuda"):
        import torch
        self.cfg, self.L, self.n_slots = cfg, n_layers, n_slots
        self.model = make_model(cfg)
        np_ = C.c_int64(0)
        call("slip_param_count", C.byref(self.model), n_layers, C.byref(np_))
        self.n_params = np_.value
        sb, wb = C.c_size_t(0), C.c_size_t(0)
        call("slip_stash_bytes", C.byref(self.model), n_layers, n_slots, C.byref(sb))
        call("slip_workspace_bytes", C.byref(self.model), C.byref(wb))
        dev = torch.device(device)
        self.w = torch.zeros(self.n_params, dtype=torch.bfloat16, device=dev)
        self.master = torch.zeros(self.n_params, dtype=torch.float32, device=dev)
        self.grad = torch.zeros(self.n_params, dtype=torch.float32, device=dev)
        self.adam_m = torch.zeros(self.n_params, dtype=torch.float32, device=dev)
        self.adam_v = torch.zeros(self.n_params, dtype=torch.float32, device=dev)
        self.arena = torch.empty(sb.value, dtype=torch.uint8, device=dev)
        self.ws = torch.zeros(wb.value, dtype=torch.uint8, device=dev)
        self.stash_bytes, self.ws_bytes = sb.value, wb.value
        ctx = C.c_void_p()
        call("slip_ctx_create", C.byref(ctx), C.byref(self.model), n_layers, n_slots)
        self.ctx = ctx
        call("slip_stage_bind", self.ctx, _ptr(self.w), _ptr(self.master), _ptr(self.grad), _ptr(self.adam_m),
             _ptr(self.adam_v), self.n_params, _ptr(self.arena), self.arena.numel(), _ptr(self.ws), self.ws.numel())

    def close(self):
        if self.ctx:
            lib().slip_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- parameters
    def load_master(self, flat_fp32, stream=None):
        """Copy fp32 master weights and refresh the bf16 copy (RNE, on the device)."""
        self.master.copy_(flat_fp32)
        call("slip_weights_from_master", self.ctx, _stream(stream))

    def slot_ptr(self, slot: int, which: int) -> int:
        p = C.c_void_p()
        call("slip_slot_ptr", self.ctx, slot, which, C.byref(p))
        return p.value

    # -- hot path
    def forward(self, slot, x, y, stream=None):
        call("slip_stage_forward", self.ctx, slot, _ptr(x), _ptr(y), _stream(stream))

    def backward_input(self, slot, dy, dx=None, accumulate=False, stream=None):
        call("slip_backward_input", self.ctx, slot, _ptr(dy), _ptr(dx) if dx is not None else None,
             int(accumulate), _stream(stream))

    def backward_weight(self, slot, accumulate=False, stream=None):
        call("slip_backward_weight", self.ctx, slot, int(accumulate), _stream(stream))

    def backward_weight_multi(self, slots, accumulate=False, stream=None):
        arr = (C.c_int32 * len(slots))(*slots)
        call("slip_backward_weight_multi", self.ctx, C.cast(arr, C.c_void_p), len(slots), int(accumulate),
             _stream(stream))

    def backward_coupled(self, slot, dy, dx=None, accumulate=False, stream=None):
        call("slip_backward_coupled", self.ctx, slot, _ptr(dy), _ptr(dx) if dx is not None else None,
             int(accumulate), _stream(stream))

    def optimizer_step(self, step, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, grad_scale=1.0,
                       nonfinite=None, stream=None):
        a = slip_adam(lr, beta1, beta2, eps, weight_decay)
        call("slip_optimizer_step", self.ctx, C.byref(a), int(step), float(grad_scale),
             _ptr(nonfinite) if nonfinite is not None else None, _stream(stream))

    def loss_ce(self, slot, y, labels, dy, d_loss, accumulate=0, stream=None):
        call("slip_loss_ce", self.ctx, slot, _ptr(y), _ptr(labels), _ptr(dy), _ptr(d_loss), int(accumulate),
             _stream(stream))

    def loss_mse(self, y, target, dy, d_loss, stream=None):
        call("slip_loss_mse", self.ctx, _ptr(y), _ptr(target), _ptr(dy), _ptr(d_loss), _stream(stream))


def synth_normal(out, seed, k, j, stream=None):
    call("slip_synth_normal", _ptr(out), out.numel(), int(seed), int(k), int(j), _stream(stream))


def gemm(a, b, c, M, N, K, lda, ldb, ldc, a_mn=False, b_mn=False, mode=0, bn=256, accumulate=False, alpha=1.0,
         stream=None):
    call("slip_gemm", M, N, K, _ptr(a), lda, int(a_mn), _ptr(b), ldb, int(b_mn), _ptr(c), ldc, mode, bn,
         int(accumulate), float(alpha), _stream(stream))


class Comm:
    """NCCL communicators of this rank.  The unique id is created by rank 0 and
    broadcast over an existing torch.distributed group (plumbing only)."""

    def __init__(self, rank: int, world: int, pg=None):
        import torch
        import torch.distributed as dist
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            call("slip_nccl_unique_id", buf)
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if world > 1:
            if dist.get_backend(pg) == "nccl":
                t = t.cuda()
            dist.broadcast(t, 0, group=pg)
        idb = (C.c_uint8 * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        call("slip_comm_create", C.byref(h), rank, world, idb)
        self.h, self.rank, self.world = h, rank, world
        self._cluster = None

    def set_p2p_ctas(self, n: int):
        """CTAs per activation / gradient transfer kernel (0: NCCL default)."""
        call("slip_comm_set_p2p_ctas", self.h, int(n))

    def set_role(self, role: int):
        """Play worker position `role` = k*N + i (after a normalization swap)."""
        call("slip_comm_set_role", self.h, int(role))

    def setup(self, N, DP, m, live=None):
        self._cluster = make_cluster(N, DP, m, live)
        call("slip_comm_setup", self.h, C.byref(self._cluster))

    def close(self):
        if self.h:
            lib().slip_comm_destroy(self.h)
            self.h = None


def migrate_state(stage: Stage, comm: Comm, peer: int, send: bool, opt_step: int = -1, stream=None):
    """P2P copy of the stage state of one normalization swap (world ranks)."""
    call("slip_migrate_state", stage.ctx, comm.h, int(peer), int(bool(send)), int(opt_step), _stream(stream))


def grad_allreduce(stage: Stage, comm: Comm, stream=None):
    call("slip_grad_allreduce", stage.ctx, comm.h, _stream(stream))


def fuse_ar_adam(stage: Stage, comm: Comm, enable=True):
    """DP = 2 all-reduce fused into AdamW over NVLink (collective over the stage pair)."""
    call("slip_comm_fuse_ar_adam", stage.ctx, comm.h, int(bool(enable)))


def fuse_ar_push(stage: Stage, comm: Comm, enable=True):
    """The fused DP = 2 all-reduce with the exchange moved into W (slip_comm_fuse_ar_push):
    the peer's W writes its 2-D weight gradients into this stage's receive buffer (an
    n_params fp32 tensor allocated here once)."""
    import torch
    if enable and getattr(stage, "recv", None) is None:
        stage.recv = torch.zeros(stage.n_params, dtype=torch.float32, device=stage.grad.device)
    recv = getattr(stage, "recv", None)
    call("slip_comm_fuse_ar_push", stage.ctx, comm.h, _ptr(recv) if (enable and recv is not None) else None,
         int(bool(enable)))


def execute_schedule(stage: Stage, comm: Comm, N, DP, m, live, costs: slip_costs, decoupled=True, staggered=True,
                     adam=(1e-4, 0.9, 0.95, 1e-8, 0.1), warmup=0, iterations=1, seed=1234, io=None,
                     stream=None) -> slip_report:
    cl = make_cluster(N, DP, m, live)
    opts = slip_plan_opts(int(decoupled), int(staggered), 1)
    a = slip_adam(*adam)
    rep = slip_report()
    call("slip_execute_schedule", stage.ctx, comm.h, C.byref(cl), C.byref(costs), C.byref(opts), C.byref(a),
         int(warmup), int(iterations), C.c_uint64(seed), C.byref(io) if io is not None else None, _stream(stream),
         C.byref(rep))
    return rep


def make_io(x_host_list, target_host_list, loss_host):
    """Host buffers for an end-to-end run: lists of pinned torch CPU tensors
    indexed k*m + j, and a float32 CPU tensor for the losses."""
    xs = (C.c_void_p * len(x_host_list))(*[t.data_ptr() for t in x_host_list])
    rs = (C.c_void_p * len(target_host_list))(*[t.data_ptr() for t in target_host_list])
    io = slip_io(C.cast(xs, C.POINTER(C.c_void_p)), C.cast(rs, C.POINTER(C.c_void_p)),
                 C.cast(C.c_void_p(loss_host.data_ptr()), C.POINTER(C.c_float)))
    io._keep = (xs, rs, x_host_list, target_host_list, loss_host)
    return io


__all__ = ["Stage", "Comm", "PlanResult", "SlipError", "assign", "execute_schedule", "gemm", "grad_allreduce",
           "make_cluster", "make_costs", "make_io", "make_model", "plan_schedule", "recoverable", "synth_normal"]
