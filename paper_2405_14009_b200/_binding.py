"""ctypes binding of libslip.so (include/slip.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
CPU fallback — if the library is missing or the device is not sm_100a the
calls raise."""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# SLIP_LIB: an alternative build of the same library (A/B measurements of kernel changes)
LIB_PATH = os.environ.get("SLIP_LIB") or os.path.join(_PKG, "libslip.so")

SLIP_F, SLIP_B, SLIP_W, SLIP_BC, SLIP_OPT, SLIP_AR = range(6)
STATUS = {0: "SLIP_OK", 1: "SLIP_EINVAL", 2: "SLIP_EUNRECOVERABLE", 3: "SLIP_EINFEASIBLE_MEMORY", 4: "SLIP_ESTATE",
          5: "SLIP_ECUDA", 6: "SLIP_ENCCL", 7: "SLIP_ENONFINITE", 8: "SLIP_EUNSUPPORTED"}


class SlipError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class slip_model(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("heads", C.c_int32), ("ffn", C.c_int32), ("seq", C.c_int32),
                ("micro_batch", C.c_int32), ("ln_eps", C.c_float), ("vocab", C.c_int32), ("ends", C.c_int32)]


class slip_cluster(C.Structure):
    _fields_ = [("num_stages", C.c_int32), ("num_pipelines", C.c_int32), ("num_microbatches", C.c_int32),
                ("live", C.POINTER(C.c_uint8))]


class slip_costs(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("t_f", "t_b", "t_w", "t_comm", "t_ar", "t_opt", "a_f", "a_w", "m_limit")]


class slip_plan_opts(C.Structure):
    _fields_ = [("decoupled", C.c_int32), ("staggered", C.c_int32), ("horizon", C.c_int32)]


class slip_adam(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("lr", "beta1", "beta2", "eps", "weight_decay")]


class slip_trace_rec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mb", C.c_int32), ("origin", C.c_int32), ("iter", C.c_int32),
                ("peer", C.c_int32), ("slot", C.c_int32), ("begin_ms", C.c_float), ("end_ms", C.c_float)]


class slip_swap(C.Structure):
    _fields_ = [("failed_stage", C.c_int32), ("failed_pipe", C.c_int32), ("target_stage", C.c_int32),
                ("target_pipe", C.c_int32), ("source_pipe", C.c_int32)]


class slip_op(C.Structure):
    _fields_ = [("stage", C.c_int32), ("mb", C.c_int32), ("origin", C.c_int32), ("phase", C.c_int32),
                ("exec", C.c_int32), ("iter", C.c_int32), ("start", C.c_int64), ("end", C.c_int64)]

    def key(self):
        return (self.stage, self.mb, self.origin, self.phase, self.exec, self.iter, self.start, self.end)


class slip_action(C.Structure):
    _fields_ = [("kind", C.c_int32), ("iter", C.c_int32), ("mb", C.c_int32), ("origin", C.c_int32),
                ("peer", C.c_int32), ("slot", C.c_int32), ("accumulate", C.c_int32)]

    def key(self):
        return (self.kind, self.iter, self.mb, self.origin, self.peer, self.slot, self.accumulate)


ACTIONS = ("LOAD_X", "RECV_X", "F", "SEND_Y", "LOSS", "RECV_DY", "B", "SEND_DX", "W", "BC", "AR", "OPT")


class slip_io(C.Structure):
    _fields_ = [("x_host", C.POINTER(C.c_void_p)), ("target_host", C.POINTER(C.c_void_p)),
                ("loss_host", C.POINTER(C.c_float))]


class slip_report(C.Structure):
    _fields_ = [("period_ms", C.c_double), ("total_ms", C.c_double), ("predicted_period", C.c_int64),
                ("n_ops", C.c_int64), ("n_kernels", C.c_int64), ("plan_hash", C.c_uint64),
                ("last_loss", C.c_float), ("nonfinite", C.c_int32), ("phase_ms", C.c_double * 6),
                ("phase_ops", C.c_int64 * 6), ("w_gemm_launches", C.c_int64), ("rollbacks", C.c_int64),
                ("skipped", C.c_int64)]


P = C.c_void_p
I32, I64, U64, F32 = C.c_int32, C.c_int64, C.c_uint64, C.c_float
SIZE = C.c_size_t

# name -> (restype, argtypes); names and order follow include/slip.h
SIGNATURES = {
    "slip_version": (I32, []),
    "slip_last_error": (C.c_char_p, []),
    "slip_status_str": (C.c_char_p, [C.c_int]),
    "slip_recoverable": (C.c_int, [C.POINTER(slip_cluster), C.POINTER(I32)]),
    "slip_assign": (C.c_int, [C.POINTER(slip_cluster), C.POINTER(I32)]),
    "slip_plan_schedule": (C.c_int, [C.POINTER(slip_cluster), C.POINTER(slip_costs), C.POINTER(slip_plan_opts),
                                     C.POINTER(slip_op), I64, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]),
    "slip_plan_hash": (U64, [C.POINTER(slip_op), I64]),
    "slip_normalize_costs": (C.c_int, [C.POINTER(slip_cluster), C.POINTER(slip_costs), C.POINTER(slip_plan_opts),
                                       I32, C.POINTER(I64)]),
    "slip_normalize": (C.c_int, [I32, I32, I32, C.POINTER(I64), C.POINTER(I64), C.POINTER(I32)]),
    "slip_normalized_live": (C.c_int, [I32, I32, C.POINTER(I32), C.POINTER(C.c_uint8)]),
    "slip_migration_plan": (C.c_int, [C.POINTER(slip_cluster), C.POINTER(I32), C.POINTER(slip_swap), I32,
                                      C.POINTER(I32), C.POINTER(C.c_uint8)]),
    "slip_rank_program": (C.c_int, [C.POINTER(slip_cluster), C.POINTER(slip_costs), C.POINTER(slip_plan_opts), I32,
                                    C.POINTER(slip_action), I64, C.POINTER(I64), C.POINTER(I32)]),
    "slip_param_count": (C.c_int, [C.POINTER(slip_model), I32, C.POINTER(I64)]),
    "slip_stash_bytes": (C.c_int, [C.POINTER(slip_model), I32, I32, C.POINTER(SIZE)]),
    "slip_workspace_bytes": (C.c_int, [C.POINTER(slip_model), C.POINTER(SIZE)]),
    "slip_ctx_create": (C.c_int, [C.POINTER(P), C.POINTER(slip_model), I32, I32]),
    "slip_ctx_destroy": (C.c_int, [P]),
    "slip_stage_bind": (C.c_int, [P, P, P, P, P, P, I64, P, SIZE, P, SIZE]),
    "slip_slot_ptr": (C.c_int, [P, I32, I32, C.POINTER(P)]),
    "slip_stage_forward": (C.c_int, [P, I32, P, P, P]),
    "slip_backward_input": (C.c_int, [P, I32, P, P, I32, P]),
    "slip_backward_weight": (C.c_int, [P, I32, I32, P]),
    "slip_backward_weight_multi": (C.c_int, [P, P, I32, I32, P]),
    "slip_backward_coupled": (C.c_int, [P, I32, P, P, I32, P]),
    "slip_optimizer_step": (C.c_int, [P, C.POINTER(slip_adam), I64, F32, P, P]),
    "slip_optimizer_step_peer": (C.c_int, [P, C.POINTER(slip_adam), I64, F32, P, P, P]),
    "slip_loss_mse": (C.c_int, [P, P, P, P, P, P]),
    "slip_synth_normal": (C.c_int, [P, I64, U64, U64, U64, P]),
    "slip_weights_from_master": (C.c_int, [P, P]),
    "slip_gemm": (C.c_int, [I32, I32, I32, P, I64, I32, P, I64, I32, P, I64, I32, I32, I32, F32, P]),
    "slip_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "slip_comm_create": (C.c_int, [C.POINTER(P), I32, I32, C.POINTER(C.c_uint8)]),
    "slip_comm_setup": (C.c_int, [P, C.POINTER(slip_cluster)]),
    "slip_comm_destroy": (C.c_int, [P]),
    "slip_grad_allreduce": (C.c_int, [P, P, P]),
    "slip_comm_fuse_ar_adam": (C.c_int, [P, P, I32]),
    "slip_comm_fuse_ar_push": (C.c_int, [P, P, P, I32]),
    "slip_comm_set_role": (C.c_int, [P, I32]),
    "slip_comm_set_p2p_ctas": (C.c_int, [P, I32]),
    "slip_set_sm_reserve": (C.c_int, [I32]),
    "slip_loss_ce": (C.c_int, [P, I32, P, P, P, P, I32, P]),
    "slip_synth_tokens": (C.c_int, [P, I64, I32, U64, U64, U64, P]),
    "slip_set_validation": (C.c_int, [P, I32]),
    "slip_set_dual_stream": (C.c_int, [P, I32]),
    "slip_set_fused_adamw": (C.c_int, [P, I32]),
    "slip_set_stream_k": (C.c_int, [P, I32]),
    "slip_inject_fault": (C.c_int, [P, I32]),
    "slip_optimizer_rollback": (C.c_int, [P, C.POINTER(slip_adam), I64, F32, P]),
    "slip_attention": (C.c_int, [I32, I32, I32, I32, P, P, P, P, P, P, I32, P]),
    "slip_set_trace": (C.c_int, [P, I32]),
    "slip_get_trace": (C.c_int, [P, C.POINTER(slip_trace_rec), I64, C.POINTER(I64)]),
    "slip_migrate_state": (C.c_int, [P, P, I32, I32, I64, P]),
    "slip_execute_schedule": (C.c_int, [P, P, C.POINTER(slip_cluster), C.POINTER(slip_costs),
                                        C.POINTER(slip_plan_opts), C.POINTER(slip_adam), I32, I32, U64,
                                        C.POINTER(slip_io), P, C.POINTER(slip_report)]),
}

_lib = None


def lib():
    """Load libslip.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2405_14009_b200.build` "
                               "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(code: int):
    if code != 0:
        raise SlipError(code, lib().slip_last_error().decode(errors="replace"))


def call(name: str, *args):
    """Call an entry point that returns slip_status; raise SlipError on failure."""
    check(getattr(lib(), name)(*args))
