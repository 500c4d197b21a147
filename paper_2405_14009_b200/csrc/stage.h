// stage.h — per-rank stage context: bound buffers, arena layout (F-stash + W-stash per
// slot = the WeightGradStore of PAPER.md line 558), workspace, slot state machine.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/slip.h"
#include "gemm.cuh"
#include "kernels.cuh"

namespace slip {

// validated mode's flag words in the workspace (Workspace::vflags)
constexpr int kValSend = 64, kValRecv = 256, kVflags = 512;

using bf16 = __nv_bfloat16;

// Offsets (elements) of one layer's tensors inside the flat parameter vector
// (include/slip.h "Parameter layout").
struct ParamOffsets {
  int64_t wqkv, bqkv, wo, bo, g1, b1n, g2, b2n, w1, b1, w2, b2, per_layer;
};
ParamOffsets param_offsets(int h, int f);

struct LayerStash {
  bf16 *xin, *y1, *qkv, *o, *x2, *y2, *hpre, *g;  // F-stash (hpre = gelu'(H), B's GeLU derivative)
  float* lse;                                       // [z, s] attention log-sum-exp (replaces P)
  float *mean1, *rstd1, *mean2, *rstd2;
  bf16 *dout, *dh, *dx2, *dqkv;                          // W-stash (with y1, o, y2, g)
};

struct GroupEntry;

struct EndStash {                // GPT ends of a slot (reading R33); null when absent
  int32_t* tokens;               // [T] token ids (embedding end)
  bf16 *xf, *yf;                 // [T, h] last-layer output, final-LN output (LM-head end)
  float *mean_f, *rstd_f;        // [T]
  bf16* dlogits;                 // [T, V] logits, then dLogits in place (W-stash of dWout)
  float* row_loss;               // [T]
};

struct SlotBufs {
  bf16* x;   // stage input   [T, h]
  bf16* dy;  // stage output gradient [T, h]
  bf16* dx;  // stage input gradient produced by B (executor send buffer) [T, h]
  std::vector<LayerStash> layer;
  EndStash end;
  GroupEntry* wtab;  // device table of the slot's W problems (4L, + dWout with the LM head)
  int wtab_tiles;
  GroupEntry* wtab_all;  // (slot 0 only) the same problems over ALL slots (zi = slot) for a
                         // W of several micro-batches in one launch (weight_multi)
};

struct Workspace {
  float* dsum;       // [z, s] D = rowsum(dO * O) of the attention backward
  bf16 *dy2, *dO, *dy1;  // [T, h]
  float* part;       // [2, kRedChunks, max(f, 3h)] column-reduction partials
  unsigned* tickets;  // [kTickets] last-block tickets (zero between launches)
  float* loss_part;  // [256] MSE partials
  float* losses;     // [1024] per-micro-batch losses (executor)
  int32_t* nonfinite;  // [1] post-step validation flag (executor)
  int32_t* vflags;     // [kVflags] validated mode: own_bad[2], global_bad[2] (per iteration parity), rollbacks,
                       // skips; [kValSend, kValRecv): ring of sent flags; [kValRecv, kVflags): received flags
  float* red;          // deferred column-reduction partials of a B call (RedBatch arena)
  size_t red_cap;      // floats
  float* sk_ws;        // stream-K fp32 partials of the F / B linears (gemm_sk_bytes)
  unsigned* sk_flags;  // [num_sms] stream-K partial epochs
};

enum SlotState : int { SLOT_FREE = 0, SLOT_F_DONE = 1, SLOT_B_DONE = 2 };

struct Dims {
  int h, a, d, f, s, b, T, z;
  float eps;
  int V, ends;  // padded vocabulary, ends bits (0 when the stage hosts no model end)
};

// Element offsets of the model-end tensors after the L layers (-1 when absent).
struct EndOffsets {
  int64_t E = -1, P = -1, gf = -1, bf = -1, Wout = -1, total = 0;
};

}  // namespace slip

struct slip_ctx {
  slip_model model;
  slip::Dims dm;
  int L = 0;
  int n_slots = 0;
  slip::ParamOffsets po;
  slip::EndOffsets eo;
  int64_t n_params = 0;
  slip::bf16* w = nullptr;
  float *master = nullptr, *grad = nullptr, *adam_m = nullptr, *adam_v = nullptr;
  uint8_t* arena = nullptr;
  size_t arena_bytes = 0;
  uint8_t* ws_base = nullptr;
  size_t ws_bytes = 0;
  bool bound = false;
  std::vector<slip::SlotBufs> slots;
  slip::Workspace ws{};
  slip::RedBatch red;  // B's bias / LayerNorm reductions, finalized in one launch
  std::vector<int> state;
  int64_t launches = 0;  // kernels enqueued through this context
  cudaStream_t h2d = nullptr;  // executor: host-to-device copies of the e2e inputs (lazily created)
  cudaStream_t fwd = nullptr;  // executor, dual stream: the forward actions' stream (lowest priority)
  cudaStream_t bwd = nullptr;  // executor, dual stream: every other compute action (highest priority)
  int dual_stream = -1;        // slip_set_dual_stream (-1: the SLIP_DUAL_STREAM environment default)
  bool fuse_adamw = false;     // slip_set_fused_adamw: AdamW of the 2-D weights in the last W's epilogue
  // W tables' mirror target (the DP peer's receive buffer, slip_comm_fuse_ar_push) and
  // whether the W launches write it (set by the executor around its calls)
  const float* w_mirror = nullptr;
  bool w_mirror_on = false;
  int64_t opt_step = 0;  // AdamW steps taken by the executor
  bool trace_on = false;
  bool validate = false;   // post-step validation + cross-stage rollback (slip_set_validation)
  bool stream_k = false;   // stream-K for F / B linears (slip_set_stream_k; measured slower, off)
  int fault_next_opt = 0;  // slip_inject_fault: the next validation reports non-finite gradients
  std::vector<slip_trace_rec> trace;  // timeline of the last traced executor run
};

namespace slip {
slip_status check_model(const slip_model* m);
Dims make_dims(const slip_model& m);
size_t stash_bytes_per_slot(const Dims& d, int L);
EndOffsets end_offsets(const Dims& d, int64_t base);
size_t workspace_bytes(const Dims& d);

// The W of n (1..8) B-done slots in ONE grouped launch: every dW accumulates the n
// micro-batches' products in TMEM (K = n*T) and is written (or added) once — or, with
// `adam` (the iteration's last W of a stage without an all-reduce), goes straight into
// AdamW in the epilogue (EPI_ADAMW; the 2-D weights only, the rest is left to the OPT).
// Releases the slots.
slip_status weight_multi(slip_ctx* c, const int* slots, int n, int accumulate, cudaStream_t s,
                         const AdamEpi* adam = nullptr);
// Local validation and the step if valid: own = non-finite gradient | injected fault | any
// of the n_pre preceding stages' flags (device int32 each); AdamW skips when own is set,
// and vflags[5] counts the skip.
slip_status validated_step(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale, int32_t* own, int fault,
                           cudaStream_t s, const int32_t* pre_flags = nullptr, int n_pre = 0);
// The AdamW state / constants for the fused W epilogue (EPI_ADAMW) of step `step`, and
// the OPT that then remains: AdamW over the layers' 1-D parameters only.
// (re)encode the W problem tables, each output mirrored into `mirror` (nullptr: none)
slip_status encode_w_tables(slip_ctx* c, const float* mirror);
// drop the executor's caches of a context (slip_ctx_destroy)
void executor_forget(const slip_ctx* ctx);
AdamEpi adam_epilogue_args(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale);
slip_status optimizer_step_vectors(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale,
                                   int32_t* d_nonfinite, cudaStream_t st);
// slip_optimizer_step with the DP peer's gradient added in (peer_grad peer-mapped, or
// NULL): the DP = 2 all-reduce fused into AdamW (slip_comm_fuse_ar_adam).
slip_status optimizer_step_peer(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale, int32_t* d_nonfinite,
                                slip_stream st, const float* peer_grad, const float* recv = nullptr);
slip_status rollback_if(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale, const int32_t* glob,
                        const int32_t* own, int32_t* count, cudaStream_t s);
}  // namespace slip
