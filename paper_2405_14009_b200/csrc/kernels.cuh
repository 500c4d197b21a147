// kernels.cuh — memory-bound kernels of the stage step (coalesced, 16-byte vectorised;
// LayerNorm rows one warp each with shuffle reductions; column reductions deterministic:
// 64-column strips x row chunks, then a fixed-order sum of the chunk partials, batched
// per B call by RedBatch).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace slip {

using bf16 = __nv_bfloat16;

constexpr int kRedChunks = 64;  // row chunks of the deterministic column reductions
constexpr int kTickets = 256;   // column strips (256 columns each) a reduction may use

// Deferred finalize of column reductions: the reductions of one B call write their
// row-chunk partials into consecutive regions of an arena and ONE launch at the end of
// the call adds them up (colred_finalize_batch), instead of a finalize launch each.
constexpr int kMaxRed = 128;
struct RedEntry {
  float* part;    // [NO][R][N] partials
  float* out[3];  // NO outputs (fp32 [N], overwrite or accumulate)
  int R, N;
};
struct RedBatch {
  RedEntry e[kMaxRed];
  int64_t start[kMaxRed + 1];  // prefix of NO*N over the entries
  int n = 0;
  float* arena = nullptr;
  size_t cap = 0, used = 0;  // floats
  void reset(float* a, size_t c) {
    arena = a;
    cap = c;
    used = 0;
    n = 0;
    start[0] = 0;
  }
  float* add(int R, int N, int NO, float* o0, float* o1, float* o2);  // partial region, or null if full
};
size_t colred_part_floats(int N, int NO);  // arena floats one reduction takes
cudaError_t colred_finalize_batch(const RedBatch& b, int accumulate, cudaStream_t s, int* launches);

// LayerNorm forward over rows of x [T, h]: y = xhat*gamma + beta; mean, rstd fp32 [T].
cudaError_t ln_fwd(const bf16* x, const bf16* gamma, const bf16* beta, bf16* y, float* mean, float* rstd, int T,
                   int h, float eps, cudaStream_t s);

// LayerNorm backward.  dx = resid + rstd*(g - mean_h(g) - xhat*mean_h(g*xhat)), g = dy*gamma
// (dx may be null; it must not alias x).  dgamma (+)= sum_t dy*xhat, dbeta (+)= sum_t dy and,
// if dxsum != null, dxsum (+)= sum_t dx, all three in ONE column-reduction launch.
// part: 3*kRedChunks*h floats of scratch (unless deferred); tickets: unused (no last-block tickets).
// Column reductions over N columns take 1 launch, or 2 when they need a finalize pass.
int colred_launches(int N);
cudaError_t ln_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* gamma,
                   const bf16* resid, bf16* dx, float* dgamma, float* dbeta, float* dxsum, int accumulate, float* part,
                   unsigned* tickets, int T, int h, cudaStream_t s, RedBatch* defer = nullptr);

// The whole LayerNorm backward in one pass over row blocks (ln_bwd_fused_kernel): dx =
// resid + rstd (dy*gamma - mean_h(g) - xhat mean_h(g*xhat)) (dx may be NULL: reductions
// only), and the deferred column reductions dgamma, dbeta and (dxsum != NULL, needs dx)
// sum_t dx over the stored bf16 dx; one partial row per block (ln_bwd_fused_parts).
// h % 8 == 0, h <= 8192; dx must not alias x or dy.
cudaError_t ln_bwd_fused(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* gamma,
                         const bf16* resid, bf16* dx, float* dgamma, float* dbeta, float* dxsum, int T, int h,
                         cudaStream_t s, RedBatch* defer);
int ln_bwd_fused_parts(int T, int h);

// out[n] (+)= sum_t a[t, n] for a bf16 [T, N] matrix with row stride ld (bias gradients).
cudaError_t colsum(const bf16* a, int T, int N, int64_t ld, float* out, int accumulate, float* part,
                   unsigned* tickets, cudaStream_t s, RedBatch* defer = nullptr);

// MSE head: dy = (y - r)/n (bf16), loss partials per block; loss = 0.5*sum/n.
cudaError_t mse_loss(const bf16* y, const bf16* r, bf16* dy, float* part, int nparts, float* loss, int64_t n,
                     cudaStream_t s);

// AdamW over flat fp32 arrays (reading R11).  Weight decay applies
// to the 2-D weights: layer-local offsets in [0, 3h^2), [3h^2+3h, 4h^2+3h),
// [4h^2+8h, 4h^2+8h+fh), [4h^2+8h+fh+f, 4h^2+8h+2fh+f).
// Parameters from `start` on (the model ends) are not layers: decayed iff in [a0, a1)
// (E, P) or [b0, b1) (Wout).
struct TailDecay {
  int64_t start = INT64_MAX, a0 = 0, a1 = 0, b0 = 0, b1 = 0;
};
// skip (device, may be NULL): if *skip != 0 the step is not taken (validated mode).
cudaError_t adamw(float* p, float* m, float* v, const float* g, bf16* w, int64_t n, int64_t per_layer, int h, int f,
                  float lr, float b1, float b2, float eps, float wd, float bc1, float bc2, float grad_scale,
                  int32_t* nonfinite, cudaStream_t s, const int32_t* skip = nullptr, TailDecay tail = TailDecay(),
                  const float* g_peer = nullptr, const float* g_recv = nullptr);
// g_peer (peer-mapped, may be NULL): the DP peer's gradient; the step uses g + g_peer.
// g_recv (local, may be NULL): the peer's 2-D weight gradients pushed here by its W
// launches (GemmDesc::c_mirror); read instead of g_peer for those elements.
// AdamW over the layers' 1-D parameters only (the 2-D weights were stepped in the W GEMM
// epilogue, gemm.cuh EPI_ADAMW); same per-element arithmetic (adamw_math.cuh).
cudaError_t adamw_vectors(float* p, float* m, float* v, const float* g, bf16* w, int layers, int64_t per_layer, int h,
                          int f, float lr, float b1, float b2, float eps, float bc1, float bc2, float grad_scale,
                          int32_t* nonfinite, cudaStream_t s);
// Two-GPU barrier on peer-mapped flags (fused DP = 2 all-reduce); epochs increase per call.
cudaError_t peer_barrier(unsigned* peer_flag, const unsigned* my_flag, unsigned epoch, cudaStream_t s);
// Arithmetic reversal of one adamw step with the same gradient;
// acts only if (global_bad == NULL || *global_bad) and (own_bad == NULL || !*own_bad);
// count (may be NULL) is incremented when it acts.
cudaError_t adamw_rollback(float* p, float* m, float* v, const float* g, bf16* w, int64_t n, int64_t per_layer, int h,
                           int f, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                           float grad_scale, const int32_t* global_bad, const int32_t* own_bad, int32_t* count,
                           cudaStream_t s, TailDecay tail = TailDecay());

// ---- GPT model ends (reading R33)
// X[t] = E[tok[t]] + P[t mod seq]   (bf16, [T, h]); an id outside [0, V) reads a zero E row
cudaError_t embed_fwd(const bf16* E, const bf16* P, const int32_t* tok, bf16* X, int T, int h, int seq, int V,
                      cudaStream_t s);
// dE[v] (+)= sum_{t: tok_t = v} dX_t (one CTA per distinct token, t order; ids outside [0, V) skipped),
// dP[p] (+)= sum_{t mod seq = p} dX_t
cudaError_t embed_bwd(const bf16* dX, const int32_t* tok, float* dE, float* dP, int T, int h, int seq, int V,
                      int accumulate, cudaStream_t s);
// in place: logits [T, V] bf16 -> dLogits = (softmax - onehot(label)) / T; row_loss[t] = lse_t - logit_t[label_t];
// then *loss = mean_t row_loss (fixed order).  A label outside [0, V) marks an ignored row (loss 0, dLogits 0).
cudaError_t cross_entropy(bf16* logits, const int32_t* labels, float* row_loss, float* loss, int T, int V,
                          cudaStream_t s);
cudaError_t synth_tokens(int32_t* out, int64_t n, int32_t n_classes, uint64_t seed, uint64_t k, uint64_t j,
                         cudaStream_t s);
// *bad |= any element of g not finite (and *nonfinite, if not NULL)
cudaError_t grad_check(const float* g, int64_t n, int32_t* bad, int32_t* nonfinite, cudaStream_t s);

// *own |= any(flags[0 .. n) != 0) (one thread; validation flags of preceding stages)
cudaError_t or_flags(int32_t* own, const int32_t* flags, int n, cudaStream_t s);
// *count += (*flag != 0) (one thread; validated mode's count of skipped steps)
cudaError_t count_flag(const int32_t* flag, int32_t* count, cudaStream_t s);

// bf16 <- RNE(fp32)
cudaError_t f32_to_bf16(const float* src, bf16* dst, int64_t n, cudaStream_t s);

// Counter-based N(0,1) -> bf16 (Philox4x32-10 + Box-Muller), key (seed), counter (k, j, i).
cudaError_t synth_normal(bf16* out, int64_t n, uint64_t seed, uint64_t k, uint64_t j, cudaStream_t s);

}  // namespace slip
