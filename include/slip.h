/* slip.h — C ABI of libslip.so, the B200-native hot path of SlipStream
 * (arXiv 2405.14009): a per-stage transformer training step whose backward is
 * split into B (input gradients, on the critical path) and W (weight
 * gradients, deferred into pipeline bubbles), followed by the per-stage DP
 * all-reduce and a staggered per-stage AdamW step; the micro-batches of failed
 * (masked) workers are re-routed to their data-parallel peers by a
 * deterministic CPU planner.
 *
 * Citations are PAPER.md lines (section / equation / figure):
 *   §3.1 Adaptive Pipelining ........... lines 197-229, Figs. 2 and 5
 *   §3.2 Decoupled BackProp ............ lines 250-292, Figs. 3, 4 and 6
 *   §3.3 Staggered Optimizer ........... lines 294-305, Fig. 7
 *   §3.4 Multiple failures ............. lines 309-345, Fig. 8
 *   §4.2 Planner (5-tuple, S, Eqs. 1-6)  lines 372-549
 *   §4.3 Implementation (ReRouteAct/Grad, WeightGradStore, AdamW) lines 550-583
 *
 * Conventions (all entry points):
 *   - extern "C"; no C++ or torch types cross the boundary; no exceptions.
 *   - Every pointer is caller-owned.  "device" pointers are CUDA global memory
 *     of the context's device; "host" pointers are CPU memory.
 *   - GPU work is enqueued asynchronously on the stream argument (a
 *     cudaStream_t passed as slip_stream; NULL = legacy default stream).  Input
 *     buffers must stay valid until that work completes.
 *   - The library never allocates device memory on the hot path: the caller
 *     allocates parameters, the stash arena and the workspace after querying
 *     their sizes.  (NCCL allocates its own buffers in slip_comm_*.)
 *   - Errors: a non-zero slip_status; slip_last_error() returns a thread-local
 *     message for the last failing call.  Device faults surface at the next
 *     synchronising call.  There is no CPU fallback: a call that cannot run
 *     on the GPU fails with SLIP_ECUDA / SLIP_EUNSUPPORTED.
 *
 * Numerics (readings R1, R10, R23): bf16 storage (RNE), fp32
 * accumulation in tensor memory (tcgen05), fp32 LayerNorm statistics, fp32
 * softmax, attention scores S and dP as fp32 tensor-memory tiles inside the fused
 * attention kernels (never stored), fp32 master weights, gradients and Adam moments.
 */
#ifndef SLIP_H
#define SLIP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* slip_stream; /* == cudaStream_t */
typedef struct slip_ctx slip_ctx;
typedef struct slip_comm slip_comm;

typedef enum {
  SLIP_OK = 0,
  SLIP_EINVAL = 1,              /* bad argument / shape / pointer */
  SLIP_EUNRECOVERABLE = 2,      /* some stage lost every worker (§3.4) */
  SLIP_EINFEASIBLE_MEMORY = 3,  /* m_limit admits no schedule (Eq. 6) */
  SLIP_ESTATE = 4,              /* slot state machine violated (e.g. B before F) */
  SLIP_ECUDA = 5,
  SLIP_ENCCL = 6,
  SLIP_ENONFINITE = 7,
  SLIP_EUNSUPPORTED = 8         /* shape outside the kernels' envelope */
} slip_status;

/* Op phases of the plan (§4.2 5-tuple c ∈ {F, B_input, B_weight};
 * BC = coupled backward; OPT = optimizer step of one worker; AR = the stage's
 * DP all-reduce, which runs on the communication stream). */
typedef enum { SLIP_F = 0, SLIP_B = 1, SLIP_W = 2, SLIP_BC = 3, SLIP_OPT = 4, SLIP_AR = 5 } slip_phase;

/* GPT-shaped stage.  Layer architecture (reading R1, PAPER.md line 607 names
 * only "Megatron implementation of GPT-3"): pre-LN, biased-variance
 * LayerNorm(eps), causal softmax attention with head dim hidden/heads, tanh-GeLU
 * FFN of width ffn, biases on every linear.  T = seq * micro_batch tokens per
 * micro-batch; token t = b*seq + position. */
typedef struct {
  int32_t hidden, heads, ffn, seq, micro_batch;
  float ln_eps;
  /* GPT model ends hosted by this stage (reading R33):
   * ends bit 0 = token + position embedding (first stage: the stage input is T
   * int32 token ids), bit 1 = final LayerNorm + LM head + cross-entropy (last
   * stage: slip_loss_ce replaces the MSE head).  vocab = padded vocabulary
   * (multiple of 128, e.g. 50257 -> 50304); ignored when ends == 0.  A token id
   * outside [0, vocab) reads a zero token-embedding row and receives no gradient
   * (no out-of-bounds access). */
  int32_t vocab, ends;
} slip_model;

/* Cluster (SPEC core_model.ClusterConfig): N stages x DP pipelines, m
 * micro-batches per pipeline per iteration, live[i*DP + k] = 1 if worker
 * W_{k_i} (stage i, pipeline k) is functional.
 * Rank of worker (i, k) is k*N + i. */
typedef struct {
  int32_t num_stages, num_pipelines, num_microbatches;
  const uint8_t* live; /* host, [N*DP] */
} slip_cluster;

/* Profiled integer costs (§4.2 "Inputs": T_F, T_Binput, T_Bweight,
 * T_comm; A_B, A_Binput, A_Bweight, M_limit).  a_f = bytes stashed by F,
 * a_w = bytes still held after B for the deferred W (reading R18).
 * m_limit <= 0: unlimited. */
typedef struct {
  int64_t t_f, t_b, t_w, t_comm, t_ar, t_opt;
  int64_t a_f, a_w, m_limit;
} slip_costs;

/* Planner options: decoupled = Decoupled BackProp (§3.2; 2 = selective: plan
 * with and without it and keep the shorter period, PAPER.md lines 289-292,
 * reading R32), staggered = Staggered Optimizer (§3.3), horizon = iterations
 * planned (>= 1; the period is measured between the last two). */
typedef struct {
  int32_t decoupled, staggered, horizon;
} slip_plan_opts;

typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
} slip_adam;

/* One planned op (SPEC baseline_schedule JSON-lines schema): stage i,
 * micro-batch j, origin pipeline k, phase, executing pipeline k_s, iteration,
 * integer start/end.  OPT: mb = origin = -1.  AR: mb = origin = exec = -1. */
typedef struct {
  int32_t stage, mb, origin, phase, exec, iter;
  int64_t start, end;
} slip_op;

/* ------------------------------------------------------------------ misc */
int32_t slip_version(void);
const char* slip_last_error(void);
const char* slip_status_str(slip_status s);

/* ------------------------------------------------------------- planner (CPU)
 * Deterministic; identical on every rank; bit-exact with the Python oracle
 * planner (oracle/planner.py) — DESIGN.md "Planner reading". */

/* RECOVERABLE (1) iff every stage keeps a live worker (§3.4 lines
 * 311-314); *out = 0 otherwise. */
slip_status slip_recoverable(const slip_cluster* c, int32_t* out);

/* Assignment S^{k_s}_{i,j,k}: out_exec[(i*m + j)*DP
 * + k] = k_s.  Live workers keep their own micro-batches; the failed workers'
 * micro-batches, enumerated in (k, j) order, go round-robin to the ascending
 * list of live peers starting at the lowest (PAPER.md lines 203, 211-214,
 * 554; reading R14).  SLIP_EUNRECOVERABLE if a stage has no live worker. */
slip_status slip_assign(const slip_cluster* c, int32_t* out_exec);

/* Heuristic list schedule (reading in DESIGN.md).
 * Writes at most cap ops to out_ops (host) in canonical order: compute ops
 * sorted by (stage, exec, start), then AR ops by (iter, stage).  *n_ops gets
 * the total count (call with cap = 0 to size the buffer).  out_makespans
 * (host, [horizon], may be NULL) gets the per-iteration makespan, *out_period
 * (may be NULL) the steady-state period. */
slip_status slip_plan_schedule(const slip_cluster* c, const slip_costs* costs, const slip_plan_opts* opts,
                               slip_op* out_ops, int64_t cap, int64_t* n_ops, int64_t* out_makespans,
                               int64_t* out_period);

/* FNV-1a 64 over the op fields (int64 little-endian, list order). */
uint64_t slip_plan_hash(const slip_op* ops, int64_t n);

/* ------------------------------------------------------- normalization (CPU)
 * Phase 1 of the Planner, §4.2.1, Algorithm 1 (lines
 * 391-414); bit-exact with oracle/normalize.py.  Readings R26-R29. */
#define SLIP_COST_INF INT64_MAX

/* The heuristic cost table: out_cost[i*(F+1) + x] = steady-state period of the
 * plan (costs, opts) with x failures at stage i (pipelines DP-1, ..., DP-x)
 * minus the fault-free period (reading R28), for 0 <= x <= min(F, DP-1);
 * SLIP_COST_INF for x > DP-1.  Uses N, DP, m of c (c->live is ignored). */
slip_status slip_normalize_costs(const slip_cluster* c, const slip_costs* costs, const slip_plan_opts* opts,
                                 int32_t F, int64_t* out_cost);

/* Algorithm 1 over a cost table cost[i*(F+1) + x] (host, N x (F+1); entries
 * with x > DP-1 are not read): out_R[N] (host) gets R = A[N-1][F], sum F, each
 * entry <= DP-1 (reading R26); out_C (host, N x (F+1), may be NULL) the table
 * C with SLIP_COST_INF where no assignment exists.  Ties take the larger x at
 * the later stage (reading R27).  SLIP_EUNRECOVERABLE if F > N (DP - 1). */
slip_status slip_normalize(int32_t N, int32_t DP, int32_t F, const int64_t* cost, int64_t* out_C, int32_t* out_R);

/* One concrete placement of R ("can be arbitrary"): stages
 * from the last to the first, failure c (counted over all stages) at pipeline
 * (DP-1-c) mod DP.  out_live (host, [N*DP]) as slip_cluster.live. */
slip_status slip_normalized_live(int32_t N, int32_t DP, const int32_t* R, uint8_t* out_live);

/* One swap: the live GPU at (target_stage, target_pipe) takes over the failed
 * position (failed_stage, failed_pipe), receiving that stage's state from the
 * live peer (failed_stage, source_pipe); the target position becomes the hole. */
typedef struct {
  int32_t failed_stage, failed_pipe, target_stage, target_pipe, source_pipe;
} slip_swap;

/* Minimum swaps (sum_i max(0, actual_i - R_i), reading R29) moving the failures
 * of c->live to the per-stage counts R.  Writes at most cap swaps, *n_swaps the
 * count (cap = 0 to size), out_live (host [N*DP], may be NULL) the live matrix
 * after all swaps.  SLIP_EINVAL if sum R differs from the failure count,
 * SLIP_EUNRECOVERABLE if c->live or R leaves a stage without a live worker. */
slip_status slip_migration_plan(const slip_cluster* c, const int32_t* R, slip_swap* out, int32_t cap,
                                int32_t* n_swaps, uint8_t* out_live);

/* ------------------------------------------------------------------ sizes
 * Parameter layout (flat, per layer, row-major, layers consecutive):
 *   Wqkv[3h,h] bqkv[3h] Wo[h,h] bo[h] g1[h] b1n[h] g2[h] b2n[h]
 *   W1[f,h] b1[f] W2[h,f] b2[h]                        (12h^2+13h for f = 4h)
 * QKV rows are the [Q; K; V] blocks; head n uses rows n*d .. (n+1)*d - 1 of
 * each block.  Linear weights are [out, in].  After the layers, the ends:
 *   embedding (ends bit 0):  E[vocab,h] P[seq,h]
 *   LM head   (ends bit 1):  gf[h] bf[h] Wout[vocab,h]
 * AdamW decays the 2-D tensors (E, P, Wout included), not gf / bf. */
slip_status slip_param_count(const slip_model* m, int32_t n_layers, int64_t* out);

/* Bytes of the stash arena for n_slots in-flight micro-batches (F-stash +
 * W-stash, the WeightGradStore of PAPER.md line 558), and of the shared
 * workspace (attention row sums D, [T, h] temporaries of B, reduction partials,
 * loss scratch, the non-finite / validation flags). */
slip_status slip_stash_bytes(const slip_model* m, int32_t n_layers, int32_t n_slots, size_t* out);
slip_status slip_workspace_bytes(const slip_model* m, size_t* out);

/* ------------------------------------------------------------ stage context
 * One per rank: a stage of n_layers layers on the current CUDA device. */
slip_status slip_ctx_create(slip_ctx** out, const slip_model* m, int32_t n_layers, int32_t n_slots);
slip_status slip_ctx_destroy(slip_ctx* ctx);

/* Bind caller-owned device buffers.  w_bf16: [n_params] bf16 weights read by
 * F/B; master, grad, adam_m, adam_v: [n_params] fp32; arena/workspace sized
 * by the queries above.  All device pointers, 256-byte aligned.  Resets every
 * slot to FREE. */
slip_status slip_stage_bind(slip_ctx* ctx, void* w_bf16, float* master, float* grad, float* adam_m, float* adam_v,
                            int64_t n_params, void* arena, size_t arena_bytes, void* workspace, size_t ws_bytes);

/* Device address inside the arena of a slot's stage input (which = 0, [T,h]
 * bf16) or stage-output gradient (which = 1, [T,h] bf16), so that a receiver
 * can ncclRecv straight into the slot (then pass that pointer as x_in / dy). */
slip_status slip_slot_ptr(slip_ctx* ctx, int32_t slot, int32_t which, void** out);

/* ------------------------------------------------------------------ hot path
 * Slot state machine (per slot): FREE -F-> F_DONE -B-> B_DONE -W-> FREE.
 * Violations return SLIP_ESTATE without enqueuing work. */

/* F (§4.2 c = F): x_in [T,h] bf16 device -> y_out [T,h] bf16
 * device, through all layers of the stage; writes the slot's F-stash.  x_in
 * is copied into the slot unless it already is the slot's input buffer.  With
 * the embedding end (model.ends bit 0) x_in is T int32 token ids and the stage
 * input is E[tok] + P[t mod seq].  B then always writes the embedding-output
 * gradient into the slot (dx may be NULL) and W adds the embedding scatter
 * dE[v] += sum_{t: tok_t = v} dX_t, dP[p] += sum_{t mod seq = p} dX_t
 * (deterministic: one CTA per distinct token, rows summed in t order). */
slip_status slip_stage_forward(slip_ctx* ctx, int32_t slot, const void* x_in, void* y_out, slip_stream s);

/* B = B_input (§3.2): dy [T,h] bf16 = dL/d(stage
 * output) -> dx [T,h] bf16 = dL/d(stage input) (dx may be NULL on stage 0).
 * Also produces the bias and LayerNorm gamma/beta gradients (reading R9),
 * added to (accumulate = 1) or written over (accumulate = 0) the fp32 grad
 * buffer, and converts the F-stash into the W-stash. */
slip_status slip_backward_input(slip_ctx* ctx, int32_t slot, const void* dy, void* dx, int32_t accumulate,
                                slip_stream s);

/* W = B_weight (§3.2; WeightBackwardPass line 558): for every layer
 * dW2 (+)= dOut^T G, dW1 (+)= dH^T Y2, dWo (+)= dX2^T O, dWqkv (+)= dQKV^T Y1
 * into the fp32 grad buffer, fused in the tcgen05 GEMM epilogue.  Frees the
 * slot. */
slip_status slip_backward_weight(slip_ctx* ctx, int32_t slot, int32_t accumulate, slip_stream s);

/* W of n (2..8) micro-batches in ONE grouped launch (the deferred W's the schedule puts
 * back to back, §3.2): the contraction of every dW runs over the n slots' stashes
 * (K = n*T), accumulated in TMEM, and dW is written (accumulate = 0) or added once.
 * slots: host array of n distinct B-done slots; all are freed.  Needs n_slots >= 2.
 * Equal to n slip_backward_weight calls up to fp32 summation order. */
slip_status slip_backward_weight_multi(slip_ctx* ctx, const int32_t* slots, int32_t n, int32_t accumulate,
                                       slip_stream s);

/* Coupled backward (the conventional baseline): B then W
 * of the same slot back to back. */
slip_status slip_backward_coupled(slip_ctx* ctx, int32_t slot, const void* dy, void* dx, int32_t accumulate,
                                  slip_stream s);

/* AdamW on the whole stage (§4.3; reading R11):
 * g <- grad_scale*g; m, v moments; bias correction with step (>= 1); decay
 * on the 2-D weights only; refresh w_bf16 = RNE(master).  d_nonfinite
 * (device int32, may be NULL) is OR-ed with 1 if any gradient element is not
 * finite (local post-step validation). */
slip_status slip_optimizer_step(slip_ctx* ctx, const slip_adam* a, int64_t step, float grad_scale,
                                int32_t* d_nonfinite, slip_stream s);

/* Last-stage loss head: l = 1/2 ||y - target||^2 / (T h),
 * dy = (y - target) / (T h) as bf16; *d_loss (device fp32) = l. */
slip_status slip_loss_mse(slip_ctx* ctx, const void* y, const void* target, void* dy, float* d_loss,
                          slip_stream s);

/* Stage-0 synthetic input for throughput runs: n bf16 values ~ N(0,1) from a
 * counter-based generator keyed by (seed, k, j), so a re-routed micro-batch
 * sees the same data on whichever peer runs it. */
slip_status slip_synth_normal(void* out_bf16, int64_t n, uint64_t seed, uint64_t k, uint64_t j, slip_stream s);

/* Last stage with the LM head (model.ends bit 1): y = stage output [T, h], labels
 * = T int32 class ids (device) < vocab; a label outside [0, vocab) marks an ignored
 * token (loss term 0, no gradient; the mean still divides by T).  Final LayerNorm,
 * logits = Y Wout^T, loss = mean_t (lse_t - logits_t[label_t]) into *d_loss (device
 * fp32), and the head's
 * input gradients: dy = d loss / d y (may alias y), gf / bf gradients (B); dLogits
 * and Y stay in the slot's stash for W (dWout += dLogits^T Y in the slot's grouped
 * W launch).  The slot must hold a forward (F done).  accumulate as in B. */
slip_status slip_loss_ce(slip_ctx* ctx, int32_t slot, const void* y, const int32_t* labels, void* dy, float* d_loss,
                         int32_t accumulate, slip_stream s);

/* Uniform synthetic token ids in [0, n_classes): out[t] = Philox(seed, k, j, t). */
slip_status slip_synth_tokens(int32_t* out, int64_t n, int32_t n_classes, uint64_t seed, uint64_t k, uint64_t j,
                              slip_stream s);

/* w_bf16 <- RNE(master) (after loading master weights). */
slip_status slip_weights_from_master(slip_ctx* ctx, slip_stream s);

/* Diagnostic entry to the fused causal attention kernels, for kernel-level parity
 * tests (the stage step calls the same kernels).  qkv [batch*s, 3*heads*d] bf16
 * (Q | K | V blocks, head-major columns), row-major.  backward = 0: out = O
 * [batch*s, heads*d] bf16, lse [batch*heads, s] fp32 (log2 domain: log2 sum_k
 * exp2(S_qk log2e / sqrt(d))).  backward = 1: o, d_o = O and dL/dO [batch*s,
 * heads*d], lse from the forward, dsum [batch*heads, s] fp32 scratch (gets
 * D = rowsum(dO * O)), out = dQKV [batch*s, 3*heads*d].  d in {32, 64, 80, 128};
 * device pointers, 16-byte aligned. */
slip_status slip_attention(int32_t s, int32_t heads, int32_t batch, int32_t d, const void* qkv, const void* o,
                           const void* d_o, void* out, float* lse, float* dsum, int32_t backward, slip_stream st);

/* Stream-K for the F / B linears of this ctx (default OFF: on B200 the split tiles
 * expose one epilogue per part and measured slower): a GEMM whose CTA-pair
 * tiles leave a partial last wave (e.g. 64 tiles of a [2048 x 2048] output on 74
 * pairs) gives every pair an equal share of the tile x k-block iterations; a split
 * tile is finished by the pair holding its first k-block, which adds the other
 * parts' fp32 partials in pair order (deterministic). */
slip_status slip_set_stream_k(slip_ctx* ctx, int32_t enable);

/* Process-wide: persistent GEMM grids fill at most (#SMs - n) SMs, leaving n
 * SMs to kernels of other streams (the executor's NCCL transfers and stage
 * all-reduce run concurrently with compute; a persistent CTA that finds no free
 * SM would wait for the whole concurrent kernel).  Default 0. */
slip_status slip_set_sm_reserve(int32_t n);

/* Diagnostic entry to one GEMM of the tcgen05 family, for kernel-level parity
 * tests: D[M,N] = sum_k A(m,k) B(k,n), bf16 operands, fp32 accumulation.
 * A(m,k) = a[m*lda + k] (a_mn = 0) or a[k*lda + m] (a_mn = 1);
 * B(k,n) = b[n*ldb + k] (b_mn = 0) or b[k*ldb + n] (b_mn = 1) (a_mn = 1 needs
 * b_mn = 1).  mode 0: c bf16 = alpha*D; 3: c fp32 = alpha*D; 4: c fp32 (+)= D
 * (accumulate).  bn: N tile, one of 32, 64, 80, 128, 256.  Device pointers,
 * 16-byte aligned rows. */
slip_status slip_gemm(int32_t M, int32_t N, int32_t K, const void* a, int64_t lda, int32_t a_mn, const void* b,
                      int64_t ldb, int32_t b_mn, void* c, int64_t ldc, int32_t mode, int32_t bn, int32_t accumulate,
                      float alpha, slip_stream s);

/* --------------------------------------------------------------- NCCL comms
 * rank r of world; the 128-byte id is created by rank 0 with
 * slip_nccl_unique_id and broadcast by the caller (torch.distributed). */
slip_status slip_nccl_unique_id(uint8_t out_id[128]);
slip_status slip_comm_create(slip_comm** out, int32_t rank, int32_t world, const uint8_t id[128]);
/* Collective over the world: builds the stage communicator over the live peers
 * of every stage (failed ranks are left out) and one communicator per directed
 * worker pair that the plan can use for activations / gradients
 * (ReRouteAct / ReRouteGrad). */
slip_status slip_comm_setup(slip_comm* comm, const slip_cluster* c);
slip_status slip_comm_destroy(slip_comm* comm);

/* CTAs (SMs) each activation / gradient transfer kernel may use (the pair
 * communicators' NCCL maxCTAs; 0 = NCCL's default; default 2).  Those kernels run
 * concurrently with the persistent compute kernels, which lose the SMs they hold
 * for as long as a transfer waits for its peer.  Call before slip_comm_setup. */
slip_status slip_comm_set_p2p_ctas(slip_comm* comm, int32_t n);

/* Worker position this process plays, as the role rank k*N + i of worker
 * (stage i, pipeline k); default = its world rank.  After a normalization
 * swap (slip_migration_plan) the GPU that sat at the target position plays the
 * failed worker's role ("swap the location of two
 * workers").  The roles of all processes must form a permutation; call before
 * slip_comm_setup (it drops the current setup). */
slip_status slip_comm_set_role(slip_comm* comm, int32_t role);

/* The point-to-point copy of one normalization swap ("a
 * point-to-point copy of model parameters"): the stage state the
 * receiver needs to take over a role — fp32 master weights, AdamW m and v
 * (3 x 4 B per parameter) — over the world communicator between WORLD ranks
 * (send = 1 on the live peer of the failed worker's stage, send = 0 on the
 * GPU taking over).  The sender's AdamW step count travels with the state: the
 * receiver rebuilds its bf16 weights from the master copy and sets its step count
 * to the sender's (opt_step < 0) or to opt_step (>= 0, an explicit override).  Both
 * sides must call it, with contexts holding the same stage model (with GPT ends the
 * receiver first binds the model of the role it takes over): the parameter counts
 * are exchanged first and a mismatch returns SLIP_EINVAL on both sides.  It
 * synchronizes s before returning (migration is not on the per-step path). */
slip_status slip_migrate_state(slip_ctx* ctx, slip_comm* comm, int32_t peer, int32_t send, int64_t opt_step,
                               slip_stream s);

/* In-place fp32 sum of the stage gradient over the live peers of the caller's
 * stage ("all-reduce collective"; reading R13).  A
 * singleton group returns without communicating. */
slip_status slip_grad_allreduce(slip_ctx* ctx, slip_comm* comm, slip_stream s);

/* The DP = 2 stage all-reduce fused into AdamW over NVLink (SURVEY.md §8(e)
 * option (i); the all-reduce of PAPER.md line 561 followed by the optimizer step
 * of line 583).  Collective over the caller's stage group; call on both live
 * peers after slip_stage_bind and slip_comm_setup.  It maps the peer's fp32
 * gradient buffer and a flag word into this process with CUDA IPC; afterwards
 * slip_execute_schedule skips the NCCL all-reduce and its OPT step is a two-GPU
 * flag barrier, ONE AdamW pass that reads g_own + g_peer (the same fp32 sum on
 * both replicas: IEEE addition is commutative, so the result equals the NCCL
 * all-reduce's bit for bit), and a second barrier before either peer may
 * overwrite its gradient.  The own gradient is left un-summed.
 * enable = 0 (or a singleton / failed group) unmaps and returns SLIP_OK;
 * SLIP_EUNSUPPORTED for a live group of more than 2; SLIP_ECUDA if the gradient
 * buffer is not IPC-exportable (e.g. a VMM allocation).  Validated steps
 * (slip_set_validation) keep the NCCL all-reduce.  Re-call after re-binding the
 * stage or re-running slip_comm_setup (which unmaps). */
slip_status slip_comm_fuse_ar_adam(slip_ctx* ctx, slip_comm* comm, int32_t enable);

/* The fused DP = 2 all-reduce + AdamW with the exchange moved into W (push mode): like
 * slip_comm_fuse_ar_adam, and in addition each peer's W launches write their dW tiles,
 * with the same TMA store / reduce-add as into its own gradient, into the OTHER peer's
 * receive buffer over NVLink (a compute step fused with its collective, tile by tile).
 * AdamW then reads the peer's 2-D weight gradients from its own receive buffer (local
 * HBM) and only the 1-D parameters' (biases, LayerNorm) over NVLink.  recv: caller-
 * allocated device buffer of n_params fp32 (torch allocation, IPC-exportable), written
 * by the peer and read by this rank's AdamW; the results equal slip_comm_fuse_ar_adam's
 * bit for bit.  Not for stages with a GPT end (SLIP_EUNSUPPORTED).  enable = 0 unmaps. */
slip_status slip_comm_fuse_ar_push(slip_ctx* ctx, slip_comm* comm, float* recv, int32_t enable);

/* The compute half of slip_comm_fuse_ar_adam for a caller that maps the peer's
 * gradient itself (e.g. one process driving both GPUs of a DP = 2 group with peer
 * access enabled): slip_optimizer_step on g_own + peer_grad[i] (the same fp32 sum
 * on both replicas), peer_grad a device pointer readable from this GPU (peer or
 * IPC mapping, the peer's whole n_params fp32 gradient; NULL = plain
 * slip_optimizer_step).  No barrier: the caller orders the peer's gradient before
 * and its next write after (as the executor's two flag barriers do). */
slip_status slip_optimizer_step_peer(slip_ctx* ctx, const slip_adam* a, int64_t step, float grad_scale,
                                     int32_t* d_nonfinite, const float* peer_grad, slip_stream s);

/* ------------------------------------------------------------- rank programs
 * The executor interprets a per-rank program derived from the plan (host
 * logic only, no GPU): for every op of worker (i, k) in planned order, the
 * receive / load that feeds it, the compute, and the send that follows it.
 * Slots are allocated at F (lowest free index) and released after W / BC. */
typedef enum {
  SLIP_ACT_LOAD_X = 0,   /* stage 0: input of micro-batch (origin, mb) into slot.x */
  SLIP_ACT_RECV_X = 1,   /* ncclRecv activation from rank `peer` into slot.x (ReRouteAct) */
  SLIP_ACT_F = 2,        /* slip_stage_forward(slot), output -> slot.dy */
  SLIP_ACT_SEND_Y = 3,   /* ncclSend slot.dy (the activation) to rank `peer` */
  SLIP_ACT_LOSS = 4,     /* last stage: MSE head, target of (origin, mb); dy -> slot.dy */
  SLIP_ACT_RECV_DY = 5,  /* ncclRecv output gradient from rank `peer` into slot.dy (ReRouteGrad) */
  SLIP_ACT_B = 6,        /* slip_backward_input(slot), dx -> slot.dx (stage > 0) */
  SLIP_ACT_SEND_DX = 7,  /* ncclSend slot.dx (the input gradient) to rank `peer` */
  SLIP_ACT_W = 8,        /* slip_backward_weight(slot); slot released */
  SLIP_ACT_BC = 9,       /* coupled backward (B then W); slot released */
  SLIP_ACT_AR = 10,      /* stage DP all-reduce of iteration `iter` */
  SLIP_ACT_OPT = 11      /* AdamW step of iteration `iter` */
} slip_action_kind;

typedef struct {
  int32_t kind, iter, mb, origin;
  int32_t peer;        /* rank, or -1 */
  int32_t slot;        /* or -1 */
  int32_t accumulate;  /* B / W: 0 = first of the iteration on this worker (overwrite) */
} slip_action;

/* Program of `rank` (worker (rank % N, rank / N)) for a plan of opts->horizon
 * iterations.  *n = number of actions (call with cap = 0 to size), *n_slots =
 * slots the program needs.  A failed rank gets an empty program. */
slip_status slip_rank_program(const slip_cluster* c, const slip_costs* costs, const slip_plan_opts* opts,
                              int32_t rank, slip_action* out, int64_t cap, int64_t* n, int32_t* n_slots);

/* ------------------------------------------------------------------ executor
 * Host buffers for an end-to-end run (may be NULL: inputs are then generated
 * on the device by slip_synth_normal with (seed, k, j) and targets with
 * (seed + 1, k, j)).  x_host[k*m + j] / target_host[k*m + j]: pinned host
 * [T,h] bf16 — or T int32 token ids / labels when the first / last stage hosts
 * the embedding / LM-head end (slip_synth_tokens when NULL); loss_host[k*m + j]
 * receives each micro-batch's loss. */
typedef struct {
  const void* const* x_host;
  const void* const* target_host;
  float* loss_host;
} slip_io;

typedef struct {
  double period_ms;          /* measured wall period per iteration (CUDA events) */
  double total_ms;           /* all timed iterations */
  int64_t predicted_period;  /* planner units */
  int64_t n_ops;             /* ops executed by this rank per iteration */
  int64_t n_kernels;         /* kernels launched by this rank in the timed iterations */
  uint64_t plan_hash;
  float last_loss;           /* mean loss of the micro-batches whose last stage ran here */
  int32_t nonfinite;
  /* per-phase device time summed over the timed iterations (CUDA events on the
   * compute stream around each op; includes waits on incoming transfers) and op
   * counts: index = slip_phase (F, B, W, BC, OPT, AR) */
  double phase_ms[6];
  int64_t phase_ops[6];
  int64_t w_gemm_launches;   /* tcgen05 GEMM launches issued by the W / BC ops */
  int64_t rollbacks;         /* validated mode: optimizer steps this rank rolled back */
  int64_t skipped;           /* validated mode: steps this rank skipped on its own failed validation */
} slip_report;

/* Runs `iterations` training iterations of the plan on this rank (worker
 * (i, k) with rank = k*N + i, stage = the ctx's stage): F / B / W / BC ops in
 * planned order on the compute stream, activation / gradient P2P on per-pair
 * streams, the stage all-reduce after the stage's last W, then the staggered
 * AdamW step.  Masked ranks return immediately.  warmup iterations are run
 * first and not timed. */
slip_status slip_execute_schedule(slip_ctx* ctx, slip_comm* comm, const slip_cluster* c, const slip_costs* costs,
                                  const slip_plan_opts* opts, const slip_adam* adam, int32_t warmup,
                                  int32_t iterations, uint64_t seed, const slip_io* io, slip_stream s,
                                  slip_report* out);

/* ------------------------------------------------------ validation / rollback
 * PAPER.md §4.3 lines 580-583 ("Bypassing Optimizer Synchronizations"), reading
 * R31.  With validation on, the executor's OPT of iteration t on each live worker
 * (1) checks the stage's all-reduced gradients for non-finite values (local
 * validation), (2) takes the AdamW step only if they are finite, and (3) starts an
 * all-reduce (MAX) of its flag over the live ranks on the all-reduce stream — no
 * stage waits for another before stepping.  Before the first W of iteration t+1
 * (the last moment the gradients of t are intact) or at the end of the call, the
 * compute stream waits for that flag and, if some stage failed while this one
 * stepped, applies the arithmetic reversal of the step (adamw_rollback, no saved
 * copy).  All decisions are taken on the device (no host round trip). */
slip_status slip_set_validation(slip_ctx* ctx, int32_t enable);
/* Fault injection for tests: kind 1 makes the next validation on this ctx report
 * non-finite gradients (the data is untouched); kind 0 clears it. */
slip_status slip_inject_fault(slip_ctx* ctx, int32_t kind);
/* The reversal of one slip_optimizer_step with the same (step, grad_scale) and the
 * gradient still in the ctx's grad buffer: p, m, v restored to rounding (v clamped at
 * 0), bf16 weights refreshed. */
slip_status slip_optimizer_rollback(slip_ctx* ctx, const slip_adam* a, int64_t step, float grad_scale, slip_stream s);

/* Execution option of slip_execute_schedule (default off): where the iteration's last W
 * already yields the final stage gradient — no DP all-reduce (DP = 1, or a stage whose
 * peer failed), no validation, no GPT ends — that W's grouped GEMM applies AdamW to the
 * 2-D weights in its epilogue (EPI_ADAMW: dW from the accumulator straight into master /
 * m / v and the bf16 copy, with the step and grad_scale of the OPT that follows) instead
 * of storing dW, and that OPT steps only the 1-D parameters.  Same arithmetic as
 * slip_optimizer_step; the gradient buffer then holds no W gradients for those weights.
 * The optimizer's traffic for the weights (26 B each) moves under the W GEMM's
 * compute-bound mainloop, and dW's 4-byte store and re-read disappear. */
slip_status slip_set_fused_adamw(slip_ctx* ctx, int32_t enable);

/* Execution option of slip_execute_schedule (default off; SLIP_DUAL_STREAM=1 in the
 * environment turns the default on): the forward actions (LOAD_X / RECV_X, F, and the
 * SEND_Y that follows) run on a second compute stream of the context, ordered by events
 * after the slot's previous W and the latest OPT; B / LOSS of a slot wait for its F.  The
 * plan and every result are unchanged; the forward of a later micro-batch fills the SMs
 * the backward kernels of an earlier one leave idle.  Ignored in validated mode (a
 * rollback rewrites weights the overlapping forward may read).  Phase times of
 * slip_report then overlap (profile planner costs with it off). */
slip_status slip_set_dual_stream(slip_ctx* ctx, int32_t enable);

/* ------------------------------------------------------------------ tracing
 * Per-action timeline of the timed iterations of the last slip_execute_schedule
 * on this ctx (off by default; costs two CUDA events per action).  Each record
 * is one program action (slip_action_kind), timed with events on the stream it
 * runs on (compute, pair or all-reduce stream): begin = when the stream reached
 * the action (its waits satisfied), end = when it finished, in ms from the start
 * of the timed region.  The planner's (start, end) of the same op make the
 * plan-vs-execution comparison (§5.3). */
typedef struct {
  int32_t kind, mb, origin, iter, peer, slot;
  float begin_ms, end_ms;
} slip_trace_rec;

slip_status slip_set_trace(slip_ctx* ctx, int32_t enable);
/* Copies at most cap records (host) of the last traced run; *n gets the count. */
slip_status slip_get_trace(slip_ctx* ctx, slip_trace_rec* out, int64_t cap, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* SLIP_H */
