// stage.cu — F (slip_stage_forward), B (slip_backward_input), W (slip_backward_weight),
// AdamW (slip_optimizer_step) and the loss head, composed from the tcgen05 GEMM family
// (gemm.cu) and the HBM-bound kernels (kernels.cu).  Formulas: DESIGN.md "Stage step",
// following PAPER.md §3.2 (B_input / B_weight split, lines 250-255) with the layer of
// reading R1 and the W set of reading R9.
#include <cmath>
#include <cstring>
#include <string>

#include "attention.cuh"
#include "common.h"
#include "gemm.cuh"
#include "kernels.cuh"
#include "stage.h"

namespace slip {

ParamOffsets param_offsets(int h, int f) {
  const int64_t H = h, F = f;
  ParamOffsets o;
  o.wqkv = 0;
  o.bqkv = 3 * H * H;
  o.wo = o.bqkv + 3 * H;
  o.bo = o.wo + H * H;
  o.g1 = o.bo + H;
  o.b1n = o.g1 + H;
  o.g2 = o.b1n + H;
  o.b2n = o.g2 + H;
  o.w1 = o.b2n + H;
  o.b1 = o.w1 + F * H;
  o.w2 = o.b1 + F;
  o.b2 = o.w2 + H * F;
  o.per_layer = o.b2 + H;
  return o;
}

slip_status check_model(const slip_model* m) {
  SLIP_CHECK(m, SLIP_EINVAL, "model is NULL");
  SLIP_CHECK(m->hidden > 0 && m->heads > 0 && m->ffn > 0 && m->seq > 0 && m->micro_batch > 0, SLIP_EINVAL,
             "model: non-positive dimension");
  SLIP_CHECK(m->hidden % m->heads == 0, SLIP_EINVAL, "model: hidden % heads != 0");
  const int d = m->hidden / m->heads;
  SLIP_CHECK(d == 32 || d == 64 || d == 80 || d == 128, SLIP_EUNSUPPORTED, "model: head dim must be 32, 64, 80 or 128");
  SLIP_CHECK(m->hidden % 64 == 0 && m->ffn % 64 == 0, SLIP_EUNSUPPORTED, "model: hidden and ffn must be multiples of 64");
  SLIP_CHECK(m->hidden <= 4096, SLIP_EUNSUPPORTED, "model: hidden > 4096");
  SLIP_CHECK(m->seq % 8 == 0 && m->seq <= 2048, SLIP_EUNSUPPORTED, "model: seq must be a multiple of 8 and <= 2048");
  SLIP_CHECK(m->ln_eps > 0.f, SLIP_EINVAL, "model: ln_eps must be > 0");
  SLIP_CHECK(m->ends >= 0 && m->ends <= 3, SLIP_EINVAL, "model: ends must be 0..3");
  SLIP_CHECK(m->ends == 0 || (m->vocab > 0 && m->vocab % 128 == 0), SLIP_EUNSUPPORTED,
             "model: vocab must be a positive multiple of 128 (padded) when the stage hosts a model end");
  return SLIP_OK;
}

EndOffsets end_offsets(const Dims& d, int64_t base) {
  EndOffsets e;
  int64_t o = base;
  const int64_t V = d.V, H = d.h, S = d.s;
  if (d.ends & 1) {
    e.E = o;
    o += V * H;
    e.P = o;
    o += S * H;
  }
  if (d.ends & 2) {
    e.gf = o;
    o += H;
    e.bf = o;
    o += H;
    e.Wout = o;
    o += V * H;
  }
  e.total = o - base;
  return e;
}

// AdamW decay of the model-end tensors: E and P (contiguous), Wout; not gf / bf
TailDecay tail_decay(const slip_ctx* c) {
  TailDecay t;
  if (!c->dm.ends) return t;
  t.start = c->po.per_layer * c->L;
  if (c->eo.E >= 0) {
    t.a0 = c->eo.E;
    t.a1 = c->eo.P + static_cast<int64_t>(c->dm.s) * c->dm.h;
  }
  if (c->eo.Wout >= 0) {
    t.b0 = c->eo.Wout;
    t.b1 = c->eo.Wout + static_cast<int64_t>(c->dm.V) * c->dm.h;
  }
  return t;
}

Dims make_dims(const slip_model& m) {
  Dims d;
  d.h = m.hidden;
  d.a = m.heads;
  d.d = m.hidden / m.heads;
  d.f = m.ffn;
  d.s = m.seq;
  d.b = m.micro_batch;
  d.T = m.seq * m.micro_batch;
  d.z = m.heads * m.micro_batch;
  d.ends = m.ends;
  d.V = m.ends ? m.vocab : 0;
  d.eps = m.ln_eps;
  return d;
}

namespace {

constexpr size_t kAlign = 256;
inline size_t al(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Walks the slot layout; with base == nullptr only sizes are computed.
struct Carver {
  uint8_t* base;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += al(n * sizeof(T));
    return p;
  }
};

void carve_slot(Carver& cv, const Dims& d, int L, SlotBufs* out) {
  const size_t Th = static_cast<size_t>(d.T) * d.h, Tf = static_cast<size_t>(d.T) * d.f;
  const size_t zs = static_cast<size_t>(d.z) * d.s;
  SlotBufs sb;
  sb.x = cv.take<bf16>(Th);
  sb.dy = cv.take<bf16>(Th);
  sb.dx = cv.take<bf16>(Th);
  sb.layer.resize(L);
  for (int l = 0; l < L; ++l) {
    LayerStash& ls = sb.layer[l];
    ls.xin = l == 0 ? sb.x : cv.take<bf16>(Th);
    ls.y1 = cv.take<bf16>(Th);
    ls.qkv = cv.take<bf16>(3 * Th);
    ls.lse = cv.take<float>(zs);
    ls.o = cv.take<bf16>(Th);
    ls.x2 = cv.take<bf16>(Th);
    ls.y2 = cv.take<bf16>(Th);
    ls.hpre = cv.take<bf16>(Tf);
    ls.g = cv.take<bf16>(Tf);
    ls.mean1 = cv.take<float>(d.T);
    ls.rstd1 = cv.take<float>(d.T);
    ls.mean2 = cv.take<float>(d.T);
    ls.rstd2 = cv.take<float>(d.T);
    ls.dout = l == L - 1 ? sb.dy : cv.take<bf16>(Th);
    ls.dh = cv.take<bf16>(Tf);
    ls.dx2 = cv.take<bf16>(Th);
    ls.dqkv = cv.take<bf16>(3 * Th);
  }
  sb.end = EndStash{};
  if (d.ends & 1) sb.end.tokens = cv.take<int32_t>(d.T);
  if (d.ends & 2) {
    sb.end.xf = cv.take<bf16>(Th);
    sb.end.yf = cv.take<bf16>(Th);
    sb.end.mean_f = cv.take<float>(d.T);
    sb.end.rstd_f = cv.take<float>(d.T);
    sb.end.dlogits = cv.take<bf16>(static_cast<size_t>(d.T) * d.V);
    sb.end.row_loss = cv.take<float>(d.T);
  }
  sb.wtab = cv.take<GroupEntry>(4 * static_cast<size_t>(L) + 1);
  sb.wtab_tiles = 0;
  sb.wtab_all = cv.take<GroupEntry>(4 * static_cast<size_t>(L) + 1);
  if (out) *out = sb;
}

void carve_ws(Carver& cv, const Dims& d, Workspace* out) {
  const size_t Th = static_cast<size_t>(d.T) * d.h;
  const size_t red = static_cast<size_t>(kRedChunks) * (d.f > 3 * d.h ? d.f : 3 * d.h);
  Workspace w;
  w.dsum = cv.take<float>(static_cast<size_t>(d.z) * d.s);
  w.dy2 = cv.take<bf16>(Th);
  w.dO = cv.take<bf16>(Th);
  w.dy1 = cv.take<bf16>(Th);
  w.part = cv.take<float>(3 * red);
  // deferred reductions: the four of a layer (b1, bqkv per (batch, 32-row group) from the
  // attention backward, LN2 + bo, LN1 + b2 below) for 8 layers before a flush
  w.red_cap = 8 * (colred_part_floats(d.f, 1) + static_cast<size_t>(d.b) * ((d.s + 31) / 32) * 3 * d.h +
                   2 * static_cast<size_t>(ln_bwd_fused_parts(d.T, d.h)) * d.h * 3) +
              colred_part_floats(d.h, 1);
  w.red = cv.take<float>(w.red_cap);
  w.tickets = cv.take<unsigned>(kTickets);
  w.loss_part = cv.take<float>(256);
  w.losses = cv.take<float>(1024);
  w.nonfinite = cv.take<int32_t>(64);
  w.vflags = cv.take<int32_t>(kVflags);
  w.sk_flags = cv.take<unsigned>(static_cast<size_t>(num_sms()));
  w.sk_ws = cv.take<float>(gemm_sk_bytes() / sizeof(float));
  if (out) *out = w;
}

}  // namespace

size_t stash_bytes_per_slot(const Dims& d, int L) {
  Carver cv{nullptr};
  carve_slot(cv, d, L, nullptr);
  return cv.off;
}

size_t workspace_bytes(const Dims& d) {
  Carver cv{nullptr};
  carve_ws(cv, d, nullptr);
  return cv.off;
}

}  // namespace slip

using namespace slip;

namespace {

// ---------------------------------------------------------------- GEMM helpers
slip_status run_gemm(slip_ctx* c, const GemmDesc& d0, cudaStream_t s, const char* what) {
  GemmDesc d = d0;
  if (c->stream_k) {  // stream-K workspace of the ctx (partial last waves of the F / B linears)
    d.sk_ws = c->ws.sk_ws;
    d.sk_flags = c->ws.sk_flags;
  }
  cudaError_t e = gemm_launch(d, s);
  if (e != cudaSuccess) {
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    if (gemm_last_message()[0]) m += std::string(" (") + gemm_last_message() + ")";
    set_error(m);
    return e == cudaErrorInvalidValue ? SLIP_EUNSUPPORTED : SLIP_ECUDA;
  }
  c->launches += 1;
  return SLIP_OK;
}

Operand op(const void* p, int64_t ld, bool mn, int64_t zi = 0, int64_t zo = 0) {
  Operand o;
  o.ptr = p;
  o.ld = ld;
  o.mn_major = mn;
  o.zi_stride = zi;
  o.zo_stride = zo;
  return o;
}

// out[T, N] = X[T, K] W[N, K]^T (+ bias, resid / GeLU)
slip_status linear_fwd(slip_ctx* c, const bf16* X, const bf16* W, int N, int K, bf16* out, const bf16* bias,
                       const bf16* resid, int mode, bf16* aux, cudaStream_t s) {
  GemmDesc d;
  d.M = c->dm.T;
  d.N = N;
  d.K = K;
  d.bn = 256;
  d.a = op(X, K, false);
  d.b = op(W, K, false);
  d.mode = mode;
  d.c = out;
  d.ldc = N;
  d.bias = bias;
  d.resid = resid;
  d.aux = aux;
  return run_gemm(c, d, s, "linear_fwd");
}

// dX[T, K] = dY[T, N] W[N, K]   (mode: EPI_BF16 or EPI_BF16_DGELU with aux = gelu'(H))
slip_status linear_dx(slip_ctx* c, const bf16* dY, const bf16* W, int N, int K, bf16* dX, int mode, bf16* aux,
                      cudaStream_t s) {
  GemmDesc d;
  d.M = c->dm.T;
  d.N = K;
  d.K = N;
  d.bn = 256;
  d.a = op(dY, N, false);
  d.b = op(W, K, true);
  d.mode = mode;
  d.c = dX;
  d.ldc = K;
  d.aux = aux;
  return run_gemm(c, d, s, "linear_dx");
}



// dW[N, K] (+)= dY[T, N]^T X[T, K]   (fp32, fused in the epilogue: TMA store / reduce-add)
slip_status linear_dw(slip_ctx* c, const bf16* dY, const bf16* X, int N, int K, float* dW, int accumulate,
                      cudaStream_t s) {
  GemmDesc d;
  d.M = N;
  d.N = K;
  d.K = c->dm.T;
  d.bn = 256;
  d.a = op(dY, N, true);
  d.b = op(X, K, true);
  d.mode = EPI_F32_ACC;
  d.c = dW;
  d.ldc = K;
  d.accumulate = accumulate;
  return run_gemm(c, d, s, "linear_dw");
}

struct LayerW {
  const bf16 *wqkv, *bqkv, *wo, *bo, *g1, *b1n, *g2, *b2n, *w1, *b1, *w2, *b2;
};
struct LayerG {
  float *wqkv, *bqkv, *wo, *bo, *g1, *b1n, *g2, *b2n, *w1, *b1, *w2, *b2;
};

LayerW layer_w(slip_ctx* c, int l) {
  const bf16* b = c->w + l * c->po.per_layer;
  const ParamOffsets& o = c->po;
  return {b + o.wqkv, b + o.bqkv, b + o.wo, b + o.bo, b + o.g1, b + o.b1n,
          b + o.g2,   b + o.b2n,  b + o.w1, b + o.b1, b + o.w2, b + o.b2};
}
LayerG layer_g(slip_ctx* c, int l) {
  float* b = c->grad + l * c->po.per_layer;
  const ParamOffsets& o = c->po;
  return {b + o.wqkv, b + o.bqkv, b + o.wo, b + o.bo, b + o.g1, b + o.b1n,
          b + o.g2,   b + o.b2n,  b + o.w1, b + o.b1, b + o.w2, b + o.b2};
}

slip_status kcheck(slip_ctx* c, cudaError_t e, const char* what, int n_launch = 1) {
  if (e != cudaSuccess) return cuda_status(e, what);
  c->launches += n_launch;
  return SLIP_OK;
}

// ---------------------------------------------------------------- attention
// Fused causal attention (attention.cu): S and dP live only in TMEM; F stashes the
// per-row log-sum-exp instead of P.  Formulas of oracle/layer.py attention_fwd / _bwd.
AttnArgs attn_args(slip_ctx* c, LayerStash& ls) {
  const Dims& D = c->dm;
  AttnArgs a;
  a.s = D.s;
  a.heads = D.a;
  a.batch = D.b;
  a.d = D.d;
  a.qkv_ld = 3LL * D.h;
  a.h = D.h;
  a.qkv = ls.qkv;
  a.o = ls.o;
  a.dO = c->ws.dO;
  a.out = nullptr;
  a.lse = ls.lse;
  a.dsum = c->ws.dsum;
  return a;
}

slip_status attn_status(slip_ctx* c, cudaError_t e, const char* what, int launches) {
  if (e == cudaSuccess) {
    c->launches += launches;
    return SLIP_OK;
  }
  set_error(std::string(what) + ": " + cudaGetErrorString(e) + " " + attn_last_message());
  return e == cudaErrorInvalidValue ? SLIP_EUNSUPPORTED : SLIP_ECUDA;
}

slip_status attention_fwd(slip_ctx* c, LayerStash& ls, cudaStream_t s) {
  AttnArgs a = attn_args(c, ls);
  a.out = ls.o;
  return attn_status(c, attn_forward(a, s), "attention forward", 1);
}

slip_status attention_bwd(slip_ctx* c, LayerStash& ls, cudaStream_t s, float* colsum = nullptr) {
  AttnArgs a = attn_args(c, ls);
  a.out = ls.dqkv;
  a.colsum = colsum;
  return attn_status(c, attn_backward(a, s), "attention backward", 2);
}

// Finalize the deferred reductions of the current B call (one launch) and start a new batch.
slip_status red_flush(slip_ctx* c, int accumulate, cudaStream_t s) {
  int n = 0;
  const cudaError_t e = colred_finalize_batch(c->red, accumulate, s, &n);
  c->red.reset(c->ws.red, c->ws.red_cap);
  return kcheck(c, e, "colred_finalize_batch", n);
}

// Make room in the batch for one reduction of `floats` partials.
slip_status red_reserve_floats(slip_ctx* c, size_t floats, int accumulate, cudaStream_t s) {
  if (c->red.n < kMaxRed && c->red.used + floats <= c->red.cap) return SLIP_OK;
  return red_flush(c, accumulate, s);
}
// ... of NO outputs over N columns by a colred launch
slip_status red_reserve(slip_ctx* c, int N, int NO, int accumulate, cudaStream_t s) {
  return red_reserve_floats(c, colred_part_floats(N, NO), accumulate, s);
}
// The partial region of a bias gradient whose producer leaves column sums per 32-row
// group (GEMM epilogue / attention backward): R groups x N columns, finalized with the batch.
slip_status red_rows(slip_ctx* c, int R, int N, float* out, int accumulate, cudaStream_t s, float** part) {
  SLIP_TRY(red_reserve_floats(c, static_cast<size_t>(R) * N, accumulate, s));
  *part = c->red.add(R, N, 1, out, nullptr, nullptr);
  SLIP_CHECK(*part, SLIP_EINVAL, "reduction arena too small");
  return SLIP_OK;
}

// colsum(a[T, N]) -> out (fp32, overwrite or accumulate); the finalize is deferred to
// the end of the B call (red_flush)
slip_status bias_grad(slip_ctx* c, const bf16* a, int N, int64_t ld, float* out, int accumulate, cudaStream_t s) {
  SLIP_TRY(red_reserve(c, N, 1, accumulate, s));
  return kcheck(c, colsum(a, c->dm.T, N, ld, out, accumulate, c->ws.part, c->ws.tickets, s, &c->red), "colsum", 1);
}

slip_status slot_check(slip_ctx* c, int slot, int want) {
  SLIP_CHECK(c, SLIP_EINVAL, "ctx is NULL");
  SLIP_CHECK(c->bound, SLIP_ESTATE, "stage buffers not bound (slip_stage_bind)");
  SLIP_CHECK(slot >= 0 && slot < c->n_slots, SLIP_EINVAL, "slot out of range");
  if (c->state[slot] != want) {
    static const char* names[] = {"FREE", "F_DONE", "B_DONE"};
    set_error(std::string("slot ") + std::to_string(slot) + " is " + names[c->state[slot]] + ", expected " +
              names[want]);
    return SLIP_ESTATE;
  }
  return SLIP_OK;
}

// The four W products of every layer of a slot: dW2 += dOut^T G, dW1 += dH^T Y2,
// dWo += dX2^T O, dWqkv += dQKV^T Y1 (reading R9).
std::vector<GemmDesc> w_problems(slip_ctx* c, int slot) {
  const Dims& D = c->dm;
  SlotBufs& sb = c->slots[slot];
  std::vector<GemmDesc> v;
  auto add = [&](const bf16* dY, const bf16* X, int N, int K, float* dW) {
    GemmDesc d;
    d.M = N;
    d.N = K;
    d.K = D.T;
    d.bn = 256;
    d.a = op(dY, N, true);
    d.b = op(X, K, true);
    d.mode = EPI_F32_ACC;
    d.c = dW;
    d.ldc = K;
    d.poff = dW - c->grad;  // (the fused-AdamW epilogue indexes the flat state with it)
    v.push_back(d);
  };
  for (int l = c->L - 1; l >= 0; --l) {
    LayerStash& ls = sb.layer[l];
    LayerG G = layer_g(c, l);
    add(ls.dout, ls.g, D.h, D.f, G.w2);
    add(ls.dh, ls.y2, D.f, D.h, G.w1);
    add(ls.dx2, ls.o, D.h, D.h, G.wo);
    add(ls.dqkv, ls.y1, 3 * D.h, D.h, G.wqkv);
  }
  if (D.ends & 2) add(sb.end.dlogits, sb.end.yf, D.V, D.h, c->grad + c->eo.Wout);  // dWout += dLogits^T Y
  return v;
}

// W as ONE persistent grouped launch over all 4L products of the slot (tables encoded at bind).

// dE, dP of the embedding end from the stage-input gradient of one slot.  The scatter
// writes only the rows of the tokens present, so the first W of an iteration (accumulate
// = 0, overwrite) clears dE and dP first: rows of tokens absent from this micro-batch must
// not keep the previous iteration's (all-reduced) gradient.
slip_status embedding_grad(slip_ctx* c, SlotBufs& sb, int accumulate, cudaStream_t s) {
  const Dims& D = c->dm;
  if (!accumulate)
    SLIP_CUDA(cudaMemsetAsync(c->grad + c->eo.E, 0, (static_cast<size_t>(D.V) + D.s) * D.h * sizeof(float), s));
  return kcheck(c, embed_bwd(sb.dx, sb.end.tokens, c->grad + c->eo.E, c->grad + c->eo.P, D.T, D.h, D.s, D.V, 1, s),
                "embed_bwd");
}

slip_status backward_weight_impl(slip_ctx* c, int slot, int accumulate, cudaStream_t s) {
  SlotBufs& sb = c->slots[slot];
  GemmDesc proto;
  proto.bn = 256;
  proto.a.mn_major = proto.b.mn_major = true;
  proto.mode = EPI_F32_ACC;
  proto.accumulate = accumulate;
  proto.mirror = (c->w_mirror_on && c->w_mirror) ? 1 : 0;
  const int n_probs = 4 * c->L + ((c->dm.ends & 2) ? 1 : 0);
  cudaError_t e = gemm_group_launch(sb.wtab, n_probs, sb.wtab_tiles, proto, s);
  if (e != cudaSuccess) {
    set_error(std::string("W grouped launch: ") + cudaGetErrorString(e) + " " + gemm_last_message());
    return SLIP_ECUDA;
  }
  c->launches += 1;
  if (c->dm.ends & 1)  // embedding scatter of the stage-input gradient B left in the slot
    SLIP_TRY(embedding_grad(c, sb, accumulate, s));
  return SLIP_OK;
}

slip_status backward_input_impl(slip_ctx* c, int slot, const void* dy, void* dx, int accumulate, cudaStream_t s) {
  const Dims& D = c->dm;
  SlotBufs& sb = c->slots[slot];
  const size_t Th = static_cast<size_t>(D.T) * D.h;
  if (dy != sb.dy) SLIP_CUDA(cudaMemcpyAsync(sb.dy, dy, Th * sizeof(bf16), cudaMemcpyDeviceToDevice, s));
  c->red.reset(c->ws.red, c->ws.red_cap);
  // db2 of the top layer = colsum(dy)
  SLIP_TRY(bias_grad(c, sb.dy, D.h, D.h, layer_g(c, c->L - 1).b2, accumulate, s));
  for (int l = c->L - 1; l >= 0; --l) {
    LayerStash& ls = sb.layer[l];
    LayerW Wt = layer_w(c, l);
    LayerG G = layer_g(c, l);
    // dH = (dOut W2) * gelu'(H)   (GeLU backward fused in the epilogue)
    SLIP_TRY(linear_dx(c, ls.dout, Wt.w2, D.h, D.f, ls.dh, EPI_BF16_DGELU, ls.hpre, s));
    SLIP_TRY(bias_grad(c, ls.dh, D.f, D.f, G.b1, accumulate, s));
    // dY2 = dH W1
    SLIP_TRY(linear_dx(c, ls.dh, Wt.w1, D.f, D.h, c->ws.dy2, EPI_BF16, nullptr, s));
    // LN2 backward + residual: dX2 = dOut + LN2'(dY2); dgamma2, dbeta2, dbo = colsum(dX2)
    SLIP_TRY(red_reserve_floats(c, static_cast<size_t>(ln_bwd_fused_parts(D.T, D.h)) * D.h * 3, accumulate, s));
    SLIP_TRY(kcheck(c,
                    ln_bwd_fused(c->ws.dy2, ls.x2, ls.mean2, ls.rstd2, Wt.g2, ls.dout, ls.dx2, G.g2, G.b2n, G.bo, D.T,
                                 D.h, s, &c->red),
                    "ln_bwd_fused 2", 1));
    // dO = dX2 Wo
    SLIP_TRY(linear_dx(c, ls.dx2, Wt.wo, D.h, D.h, c->ws.dO, EPI_BF16, nullptr, s));
    // attention backward (dQKV, and dbqkv's column sums per (batch, 32-row group))
    float* pbq = nullptr;
    SLIP_TRY(red_rows(c, D.b * ((D.s + 31) / 32), 3 * D.h, G.bqkv, accumulate, s, &pbq));
    SLIP_TRY(attention_bwd(c, ls, s, pbq));
    // dY1 = dQKV Wqkv
    SLIP_TRY(linear_dx(c, ls.dqkv, Wt.wqkv, 3 * D.h, D.h, c->ws.dy1, EPI_BF16, nullptr, s));
    // LN1 backward + residual: dX = dX2 + LN1'(dY1); db2 of the layer below = colsum(dX)
    // with the embedding end the input gradient always lands in the slot (W's scatter reads it)
    bf16* dxl = l > 0 ? sb.layer[l - 1].dout : ((D.ends & 1) ? sb.dx : static_cast<bf16*>(dx));
    float* dxsum = l > 0 ? layer_g(c, l - 1).b2 : nullptr;
    // (stage 0 without an input gradient: dx = NULL, only dgamma1, dbeta1)
    SLIP_TRY(red_reserve_floats(c, static_cast<size_t>(ln_bwd_fused_parts(D.T, D.h)) * D.h * 3, accumulate, s));
    SLIP_TRY(kcheck(c,
                    ln_bwd_fused(c->ws.dy1, ls.xin, ls.mean1, ls.rstd1, Wt.g1, ls.dx2, dxl, G.g1, G.b1n,
                                 dxl ? dxsum : nullptr, D.T, D.h, s, &c->red),
                    "ln_bwd_fused 1", 1));
  }
  SLIP_TRY(red_flush(c, accumulate, s));
  if ((D.ends & 1) && dx && dx != sb.dx)
    SLIP_CUDA(cudaMemcpyAsync(dx, sb.dx, Th * sizeof(bf16), cudaMemcpyDeviceToDevice, s));
  return SLIP_OK;
}

}  // namespace


// The W problem tables (tensor maps of the 4L weight-gradient GEMMs) of every slot, and
// slot 0's table over all slots; with `mirror` each problem's output is also written to
// the same offset of that buffer (GemmDesc::c_mirror: the DP peer's receive buffer).
slip_status slip::encode_w_tables(slip_ctx* c, const float* mirror) {
  const size_t per = stash_bytes_per_slot(c->dm, c->L);
  auto with_mirror = [&](std::vector<GemmDesc>& probs) {
    if (!mirror) return;
    for (GemmDesc& d : probs) d.c_mirror = mirror + (static_cast<const float*>(d.c) - c->grad);
  };
  std::vector<GroupEntry> host(4 * static_cast<size_t>(c->L) + ((c->dm.ends & 2) ? 1 : 0));
  for (int i = 0; i < c->n_slots; ++i) {
    std::vector<GemmDesc> probs = w_problems(c, i);
    with_mirror(probs);
    int tiles = 0;
    cudaError_t e = gemm_group_encode(probs.data(), static_cast<int>(probs.size()), host.data(), &tiles);
    if (e != cudaSuccess) {
      set_error(std::string("W table: ") + gemm_last_message());
      return SLIP_EUNSUPPORTED;
    }
    SLIP_CUDA(cudaMemcpy(c->slots[i].wtab, host.data(), host.size() * sizeof(GroupEntry), cudaMemcpyHostToDevice));
    c->slots[i].wtab_tiles = tiles;
  }
  if (c->n_slots >= 2) {  // slot 0's problems with the slot as the operands' zi dimension
    std::vector<GemmDesc> probs = w_problems(c, 0);
    with_mirror(probs);
    const int64_t zs = static_cast<int64_t>(per / sizeof(bf16));
    for (GemmDesc& d : probs) {
      d.zi_count = c->n_slots;
      d.a.zi_stride = zs;
      d.b.zi_stride = zs;
    }
    int tiles = 0;
    cudaError_t e = gemm_group_encode(probs.data(), static_cast<int>(probs.size()), host.data(), &tiles);
    if (e != cudaSuccess) {
      set_error(std::string("W all-slot table: ") + gemm_last_message());
      return SLIP_EUNSUPPORTED;
    }
    SLIP_CUDA(cudaMemcpy(c->slots[0].wtab_all, host.data(), host.size() * sizeof(GroupEntry), cudaMemcpyHostToDevice));
  }
  c->w_mirror = mirror;
  return SLIP_OK;
}

extern "C" {

slip_status slip_param_count(const slip_model* m, int32_t n_layers, int64_t* out) {
  SLIP_TRY(check_model(m));
  SLIP_CHECK(n_layers > 0 && out, SLIP_EINVAL, "param_count: bad arguments");
  const int64_t layers = param_offsets(m->hidden, m->ffn).per_layer * n_layers;
  *out = layers + end_offsets(make_dims(*m), layers).total;
  return SLIP_OK;
}

slip_status slip_stash_bytes(const slip_model* m, int32_t n_layers, int32_t n_slots, size_t* out) {
  SLIP_TRY(check_model(m));
  SLIP_CHECK(n_layers > 0 && n_slots > 0 && out, SLIP_EINVAL, "stash_bytes: bad arguments");
  *out = stash_bytes_per_slot(make_dims(*m), n_layers) * n_slots;
  return SLIP_OK;
}

slip_status slip_workspace_bytes(const slip_model* m, size_t* out) {
  SLIP_TRY(check_model(m));
  SLIP_CHECK(out, SLIP_EINVAL, "workspace_bytes: out is NULL");
  *out = workspace_bytes(make_dims(*m));
  return SLIP_OK;
}

slip_status slip_ctx_create(slip_ctx** out, const slip_model* m, int32_t n_layers, int32_t n_slots) {
  SLIP_CHECK(out, SLIP_EINVAL, "ctx_create: out is NULL");
  SLIP_TRY(check_model(m));
  SLIP_CHECK(n_layers > 0 && n_slots > 0, SLIP_EINVAL, "ctx_create: n_layers and n_slots must be > 0");
  int dev = 0;
  SLIP_CUDA(cudaGetDevice(&dev));
  int major = 0, minor = 0;
  SLIP_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  SLIP_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  SLIP_CHECK(major == 10 && minor == 0, SLIP_EUNSUPPORTED, "libslip is built for sm_100a (B200) only");
  slip_ctx* c = new slip_ctx();
  c->model = *m;
  c->dm = make_dims(*m);
  c->L = n_layers;
  c->n_slots = n_slots;
  c->po = param_offsets(m->hidden, m->ffn);
  c->eo = end_offsets(c->dm, c->po.per_layer * n_layers);
  c->n_params = c->po.per_layer * n_layers + c->eo.total;
  c->state.assign(n_slots, SLOT_FREE);
  *out = c;
  return SLIP_OK;
}

slip_status slip_ctx_destroy(slip_ctx* ctx) {
  slip::executor_forget(ctx);
  if (ctx && ctx->h2d) cudaStreamDestroy(ctx->h2d);
  if (ctx && ctx->fwd) cudaStreamDestroy(ctx->fwd);
  if (ctx && ctx->bwd) cudaStreamDestroy(ctx->bwd);
  delete ctx;
  return SLIP_OK;
}

slip_status slip_stage_bind(slip_ctx* c, void* w_bf16, float* master, float* grad, float* adam_m, float* adam_v,
                            int64_t n_params, void* arena, size_t arena_bytes, void* workspace, size_t ws_bytes) {
  SLIP_CHECK(c, SLIP_EINVAL, "ctx is NULL");
  SLIP_CHECK(n_params == c->n_params, SLIP_EINVAL, "stage_bind: n_params does not match the model");
  SLIP_CHECK(w_bf16 && master && grad && adam_m && adam_v && arena && workspace, SLIP_EINVAL,
             "stage_bind: NULL buffer");
  auto aligned = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 256 == 0; };
  SLIP_CHECK(aligned(w_bf16) && aligned(master) && aligned(grad) && aligned(adam_m) && aligned(adam_v) &&
                 aligned(arena) && aligned(workspace),
             SLIP_EINVAL, "stage_bind: buffers must be 256-byte aligned");
  const size_t per = stash_bytes_per_slot(c->dm, c->L);
  SLIP_CHECK(arena_bytes >= per * c->n_slots, SLIP_EINVAL, "stage_bind: arena too small");
  SLIP_CHECK(ws_bytes >= workspace_bytes(c->dm), SLIP_EINVAL, "stage_bind: workspace too small");
  c->w = static_cast<bf16*>(w_bf16);
  c->master = master;
  c->grad = grad;
  c->adam_m = adam_m;
  c->adam_v = adam_v;
  c->arena = static_cast<uint8_t*>(arena);
  c->arena_bytes = arena_bytes;
  c->ws_base = static_cast<uint8_t*>(workspace);
  c->ws_bytes = ws_bytes;
  c->slots.resize(c->n_slots);
  for (int i = 0; i < c->n_slots; ++i) {
    Carver cv{c->arena + per * i};
    carve_slot(cv, c->dm, c->L, &c->slots[i]);
  }
  Carver wv{c->ws_base};
  carve_ws(wv, c->dm, &c->ws);
  SLIP_CUDA(cudaMemset(c->ws.tickets, 0, kTickets * sizeof(unsigned)));
  SLIP_CUDA(cudaMemset(c->ws.nonfinite, 0, sizeof(int32_t)));
  SLIP_CUDA(cudaMemset(c->ws.sk_flags, 0, static_cast<size_t>(num_sms()) * sizeof(unsigned)));
  c->w_mirror = nullptr;
  SLIP_TRY(slip::encode_w_tables(c, nullptr));
  c->state.assign(c->n_slots, SLOT_FREE);
  c->bound = true;
  return SLIP_OK;
}

slip_status slip_slot_ptr(slip_ctx* c, int32_t slot, int32_t which, void** out) {
  SLIP_CHECK(c && c->bound && out, SLIP_EINVAL, "slot_ptr: bad arguments");
  SLIP_CHECK(slot >= 0 && slot < c->n_slots && (which == 0 || which == 1), SLIP_EINVAL, "slot_ptr: bad slot / which");
  *out = which == 0 ? static_cast<void*>(c->slots[slot].x) : static_cast<void*>(c->slots[slot].dy);
  return SLIP_OK;
}

slip_status slip_stage_forward(slip_ctx* c, int32_t slot, const void* x_in, void* y_out, slip_stream st) {
  SLIP_TRY(slot_check(c, slot, SLOT_FREE));
  SLIP_CHECK(x_in && y_out, SLIP_EINVAL, "stage_forward: NULL x_in / y_out");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  const Dims& D = c->dm;
  SlotBufs& sb = c->slots[slot];
  const size_t Th = static_cast<size_t>(D.T) * D.h;
  if (D.ends & 1) {  // x_in = T token ids: X = E[tok] + P[t mod seq]
    if (x_in != sb.end.tokens)
      SLIP_CUDA(cudaMemcpyAsync(sb.end.tokens, x_in, D.T * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    SLIP_TRY(kcheck(c, embed_fwd(c->w + c->eo.E, c->w + c->eo.P, sb.end.tokens, sb.x, D.T, D.h, D.s, D.V, s), "embed_fwd"));
  } else if (x_in != sb.x) {
    SLIP_CUDA(cudaMemcpyAsync(sb.x, x_in, Th * sizeof(bf16), cudaMemcpyDeviceToDevice, s));
  }
  for (int l = 0; l < c->L; ++l) {
    LayerStash& ls = sb.layer[l];
    LayerW Wt = layer_w(c, l);
    bf16* out = l + 1 < c->L ? sb.layer[l + 1].xin : static_cast<bf16*>(y_out);
    SLIP_TRY(kcheck(c, ln_fwd(ls.xin, Wt.g1, Wt.b1n, ls.y1, ls.mean1, ls.rstd1, D.T, D.h, D.eps, s), "ln_fwd 1"));
    SLIP_TRY(linear_fwd(c, ls.y1, Wt.wqkv, 3 * D.h, D.h, ls.qkv, Wt.bqkv, nullptr, EPI_BF16, nullptr, s));
    SLIP_TRY(attention_fwd(c, ls, s));
    SLIP_TRY(linear_fwd(c, ls.o, Wt.wo, D.h, D.h, ls.x2, Wt.bo, ls.xin, EPI_BF16, nullptr, s));
    SLIP_TRY(kcheck(c, ln_fwd(ls.x2, Wt.g2, Wt.b2n, ls.y2, ls.mean2, ls.rstd2, D.T, D.h, D.eps, s), "ln_fwd 2"));
    SLIP_TRY(linear_fwd(c, ls.y2, Wt.w1, D.f, D.h, ls.g, Wt.b1, nullptr, EPI_BF16_GELU, ls.hpre, s));
    SLIP_TRY(linear_fwd(c, ls.g, Wt.w2, D.h, D.f, out, Wt.b2, ls.x2, EPI_BF16, nullptr, s));
  }
  c->state[slot] = SLOT_F_DONE;
  return SLIP_OK;
}

slip_status slip_backward_input(slip_ctx* c, int32_t slot, const void* dy, void* dx, int32_t accumulate,
                                slip_stream st) {
  SLIP_TRY(slot_check(c, slot, SLOT_F_DONE));
  SLIP_CHECK(dy, SLIP_EINVAL, "backward_input: NULL dy");
  SLIP_TRY(backward_input_impl(c, slot, dy, dx, accumulate, reinterpret_cast<cudaStream_t>(st)));
  c->state[slot] = SLOT_B_DONE;
  return SLIP_OK;
}

}  // extern "C"

namespace slip {
slip_status weight_multi(slip_ctx* c, const int* slots, int n, int accumulate, cudaStream_t s, const AdamEpi* adam) {
  SLIP_CHECK(c && slots && n >= 1 && n <= 8 && c->n_slots >= 2, SLIP_EINVAL, "weight_multi: bad arguments");
  SLIP_CHECK(!adam || !c->dm.ends, SLIP_EINVAL, "weight_multi: the fused AdamW epilogue excludes the GPT ends");
  for (int j = 0; j < n; ++j) SLIP_TRY(slot_check(c, slots[j], SLOT_B_DONE));
  GemmDesc proto;
  proto.bn = 256;
  proto.a.mn_major = proto.b.mn_major = true;
  proto.mode = adam ? EPI_ADAMW : EPI_F32_ACC;
  proto.adam = adam;
  proto.accumulate = accumulate;
  proto.mirror = (!adam && c->w_mirror_on && c->w_mirror) ? 1 : 0;
  proto.kz_n = n;
  proto.kz_nkb = (c->dm.T + 63) / 64;
  for (int j = 0; j < n; ++j) proto.kz_list[j] = slots[j];
  const int n_probs = 4 * c->L + ((c->dm.ends & 2) ? 1 : 0);
  cudaError_t e = gemm_group_launch(c->slots[0].wtab_all, n_probs, c->slots[0].wtab_tiles, proto, s);
  if (e != cudaSuccess) {
    set_error(std::string("W multi launch: ") + cudaGetErrorString(e) + " " + gemm_last_message());
    return SLIP_ECUDA;
  }
  c->launches += 1;
  for (int j = 0; j < n; ++j) {
    SlotBufs& sb = c->slots[slots[j]];
    if (c->dm.ends & 1)  // embedding scatter of each slot's stage-input gradient
      SLIP_TRY(embedding_grad(c, sb, accumulate || j > 0, s));
    c->state[slots[j]] = SLOT_FREE;
  }
  return SLIP_OK;
}
}  // namespace slip

extern "C" {

slip_status slip_backward_weight_multi(slip_ctx* c, const int32_t* slots, int32_t n, int32_t accumulate,
                                       slip_stream st) {
  SLIP_CHECK(c && c->bound && slots, SLIP_EINVAL, "backward_weight_multi: bad arguments");
  std::vector<int> v(slots, slots + (n > 0 ? n : 0));
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < j; ++k) SLIP_CHECK(v[j] != v[k], SLIP_EINVAL, "backward_weight_multi: repeated slot");
  return weight_multi(c, v.data(), n, accumulate, reinterpret_cast<cudaStream_t>(st));
}

slip_status slip_backward_weight(slip_ctx* c, int32_t slot, int32_t accumulate, slip_stream st) {
  SLIP_TRY(slot_check(c, slot, SLOT_B_DONE));
  SLIP_TRY(backward_weight_impl(c, slot, accumulate, reinterpret_cast<cudaStream_t>(st)));
  c->state[slot] = SLOT_FREE;
  return SLIP_OK;
}

slip_status slip_backward_coupled(slip_ctx* c, int32_t slot, const void* dy, void* dx, int32_t accumulate,
                                  slip_stream st) {
  SLIP_TRY(slip_backward_input(c, slot, dy, dx, accumulate, st));
  return slip_backward_weight(c, slot, accumulate, st);
}

slip_status slip_optimizer_step(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale, int32_t* d_nonfinite,
                                slip_stream st) {
  return slip::optimizer_step_peer(c, a, step, grad_scale, d_nonfinite, st, nullptr);
}

slip_status slip_optimizer_step_peer(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale,
                                     int32_t* d_nonfinite, const float* peer_grad, slip_stream st) {
  return slip::optimizer_step_peer(c, a, step, grad_scale, d_nonfinite, st, peer_grad);
}

}  // extern "C"

AdamEpi slip::adam_epilogue_args(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale) {
  AdamEpi e;
  e.p = c->master;
  e.m = c->adam_m;
  e.v = c->adam_v;
  e.g = c->grad;
  e.w = c->w;
  e.lr = a->lr;
  e.b1 = a->beta1;
  e.b2 = a->beta2;
  e.eps = a->eps;
  e.wd = a->weight_decay;
  // the same float constants the flat kernel receives (adamw(): 1.0f / float(bc))
  e.inv_bc1 = 1.0f / static_cast<float>(1.0 - std::pow(static_cast<double>(a->beta1), static_cast<double>(step)));
  e.inv_bc2 = 1.0f / static_cast<float>(1.0 - std::pow(static_cast<double>(a->beta2), static_cast<double>(step)));
  e.grad_scale = grad_scale;
  e.nonfinite = c->ws.nonfinite;
  return e;
}

slip_status slip::optimizer_step_vectors(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale,
                                         int32_t* d_nonfinite, cudaStream_t st) {
  SLIP_CHECK(c && c->bound && a && step >= 1 && !c->dm.ends, SLIP_EINVAL, "optimizer_step_vectors: bad arguments");
  const double bc1 = 1.0 - std::pow(static_cast<double>(a->beta1), static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(static_cast<double>(a->beta2), static_cast<double>(step));
  return kcheck(c,
                adamw_vectors(c->master, c->adam_m, c->adam_v, c->grad, c->w, c->L, c->po.per_layer, c->dm.h, c->dm.f,
                              a->lr, a->beta1, a->beta2, a->eps, static_cast<float>(bc1), static_cast<float>(bc2),
                              grad_scale, d_nonfinite, st),
                "adamw_vectors");
}

slip_status slip::optimizer_step_peer(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale,
                                      int32_t* d_nonfinite, slip_stream st, const float* peer_grad,
                                      const float* recv) {
  SLIP_CHECK(c && c->bound && a, SLIP_EINVAL, "optimizer_step: bad arguments");
  SLIP_CHECK(step >= 1, SLIP_EINVAL, "optimizer_step: step must be >= 1");
  const double bc1 = 1.0 - std::pow(static_cast<double>(a->beta1), static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(static_cast<double>(a->beta2), static_cast<double>(step));
  return kcheck(c,
                adamw(c->master, c->adam_m, c->adam_v, c->grad, c->w, c->n_params, c->po.per_layer, c->dm.h, c->dm.f,
                      a->lr, a->beta1, a->beta2, a->eps, a->weight_decay, static_cast<float>(bc1),
                      static_cast<float>(bc2), grad_scale, d_nonfinite, reinterpret_cast<cudaStream_t>(st), nullptr,
                      tail_decay(c), peer_grad, recv),
                "adamw");
}

extern "C" {

slip_status slip_loss_mse(slip_ctx* c, const void* y, const void* target, void* dy, float* d_loss, slip_stream st) {
  SLIP_CHECK(c && c->bound && y && target && dy && d_loss, SLIP_EINVAL, "loss_mse: bad arguments");
  const int64_t n = static_cast<int64_t>(c->dm.T) * c->dm.h;
  return kcheck(c,
                mse_loss(static_cast<const bf16*>(y), static_cast<const bf16*>(target), static_cast<bf16*>(dy),
                         c->ws.loss_part, 256, d_loss, n, reinterpret_cast<cudaStream_t>(st)),
                "mse_loss", 2);
}

slip_status slip_loss_ce(slip_ctx* c, int32_t slot, const void* y, const int32_t* labels, void* dy, float* d_loss,
                         int32_t accumulate, slip_stream st) {
  SLIP_TRY(slot_check(c, slot, SLOT_F_DONE));
  SLIP_CHECK(c->dm.ends & 2, SLIP_EINVAL, "loss_ce: the stage hosts no LM head (model.ends bit 1)");
  SLIP_CHECK(y && labels && dy && d_loss, SLIP_EINVAL, "loss_ce: NULL argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  const Dims& D = c->dm;
  EndStash& e = c->slots[slot].end;
  const size_t Th = static_cast<size_t>(D.T) * D.h;
  const bf16* gf = c->w + c->eo.gf;
  const bf16* bfp = c->w + c->eo.bf;
  const bf16* Wout = c->w + c->eo.Wout;
  if (y != e.xf) SLIP_CUDA(cudaMemcpyAsync(e.xf, y, Th * sizeof(bf16), cudaMemcpyDeviceToDevice, s));
  SLIP_TRY(kcheck(c, ln_fwd(e.xf, gf, bfp, e.yf, e.mean_f, e.rstd_f, D.T, D.h, D.eps, s), "ln_fwd f"));
  SLIP_TRY(linear_fwd(c, e.yf, Wout, D.V, D.h, e.dlogits, nullptr, nullptr, EPI_BF16, nullptr, s));  // logits
  SLIP_TRY(kcheck(c, cross_entropy(e.dlogits, labels, e.row_loss, d_loss, D.T, D.V, s), "cross_entropy", 2));
  SLIP_TRY(linear_dx(c, e.dlogits, Wout, D.V, D.h, c->ws.dy2, EPI_BF16, nullptr, s));  // dY = dLogits Wout
  return kcheck(c,
                ln_bwd(c->ws.dy2, e.xf, e.mean_f, e.rstd_f, gf, nullptr, static_cast<bf16*>(dy), c->grad + c->eo.gf,
                       c->grad + c->eo.bf, nullptr, accumulate, c->ws.part, c->ws.tickets, D.T, D.h, s),
                "ln_bwd f", 1 + colred_launches(D.h));
}

slip_status slip_synth_tokens(int32_t* out, int64_t n, int32_t n_classes, uint64_t seed, uint64_t k, uint64_t j,
                              slip_stream st) {
  SLIP_CHECK(out && n > 0 && n_classes > 0, SLIP_EINVAL, "synth_tokens: bad arguments");
  SLIP_CUDA(synth_tokens(out, n, n_classes, seed, k, j, reinterpret_cast<cudaStream_t>(st)));
  return SLIP_OK;
}

slip_status slip_synth_normal(void* out_bf16, int64_t n, uint64_t seed, uint64_t k, uint64_t j, slip_stream st) {
  SLIP_CHECK(out_bf16 && n > 0, SLIP_EINVAL, "synth_normal: bad arguments");
  SLIP_CUDA(synth_normal(static_cast<bf16*>(out_bf16), n, seed, k, j, reinterpret_cast<cudaStream_t>(st)));
  return SLIP_OK;
}

}  // extern "C"

namespace slip {
// Validated OPT (executor): own = fault injected ? 1 : any non-finite gradient; step only if !own.
slip_status validated_step(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale, int32_t* own, int fault,
                           cudaStream_t s, const int32_t* pre_flags, int n_pre) {
  const double bc1 = 1.0 - std::pow(static_cast<double>(a->beta1), static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(static_cast<double>(a->beta2), static_cast<double>(step));
  SLIP_CUDA(cudaMemsetAsync(own, 0, sizeof(int32_t), s));
  if (fault) SLIP_CUDA(cudaMemsetAsync(own, 1, 1, s));
  SLIP_TRY(kcheck(c, grad_check(c->grad, c->n_params, own, c->ws.nonfinite, s), "grad_check"));
  // "based on its individual validation results and those of preceding stages"
  if (n_pre > 0) SLIP_TRY(kcheck(c, or_flags(own, pre_flags, n_pre, s), "or_flags"));
  SLIP_TRY(kcheck(c,
                  adamw(c->master, c->adam_m, c->adam_v, c->grad, c->w, c->n_params, c->po.per_layer, c->dm.h,
                        c->dm.f, a->lr, a->beta1, a->beta2, a->eps, a->weight_decay, static_cast<float>(bc1),
                        static_cast<float>(bc2), grad_scale, c->ws.nonfinite, s, own, tail_decay(c)),
                  "adamw"));
  // a skipped step does not count towards AdamW's bias correction (the executor subtracts it)
  return kcheck(c, count_flag(own, c->ws.vflags + 5, s), "count_flag");
}
// Conditional reversal of the step taken with (step, grad_scale): acts iff *glob && !*own.
slip_status rollback_if(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale, const int32_t* glob,
                        const int32_t* own, int32_t* count, cudaStream_t s) {
  const double bc1 = 1.0 - std::pow(static_cast<double>(a->beta1), static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(static_cast<double>(a->beta2), static_cast<double>(step));
  return kcheck(c,
                adamw_rollback(c->master, c->adam_m, c->adam_v, c->grad, c->w, c->n_params, c->po.per_layer, c->dm.h,
                               c->dm.f, a->lr, a->beta1, a->beta2, a->eps, a->weight_decay, static_cast<float>(bc1),
                               static_cast<float>(bc2), grad_scale, glob, own, count, s, tail_decay(c)),
                "adamw_rollback");
}
}  // namespace slip

extern "C" {

slip_status slip_set_stream_k(slip_ctx* c, int32_t enable) {
  SLIP_CHECK(c, SLIP_EINVAL, "set_stream_k: ctx is NULL");
  c->stream_k = enable != 0;
  return SLIP_OK;
}

slip_status slip_set_fused_adamw(slip_ctx* c, int32_t enable) {
  SLIP_CHECK(c, SLIP_EINVAL, "set_fused_adamw: ctx is NULL");
  c->fuse_adamw = enable != 0;
  return SLIP_OK;
}

slip_status slip_set_validation(slip_ctx* c, int32_t enable) {
  SLIP_CHECK(c, SLIP_EINVAL, "set_validation: ctx is NULL");
  c->validate = enable != 0;
  return SLIP_OK;
}

slip_status slip_inject_fault(slip_ctx* c, int32_t kind) {
  SLIP_CHECK(c && (kind == 0 || kind == 1), SLIP_EINVAL, "inject_fault: kind must be 0 or 1");
  c->fault_next_opt = kind;
  return SLIP_OK;
}

slip_status slip_optimizer_rollback(slip_ctx* c, const slip_adam* a, int64_t step, float grad_scale, slip_stream st) {
  SLIP_CHECK(c && c->bound && a, SLIP_EINVAL, "optimizer_rollback: bad arguments");
  SLIP_CHECK(step >= 1, SLIP_EINVAL, "optimizer_rollback: step must be >= 1");
  const double bc1 = 1.0 - std::pow(static_cast<double>(a->beta1), static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(static_cast<double>(a->beta2), static_cast<double>(step));
  return kcheck(c,
                adamw_rollback(c->master, c->adam_m, c->adam_v, c->grad, c->w, c->n_params, c->po.per_layer, c->dm.h,
                               c->dm.f, a->lr, a->beta1, a->beta2, a->eps, a->weight_decay, static_cast<float>(bc1),
                               static_cast<float>(bc2), grad_scale, nullptr, nullptr, nullptr,
                               reinterpret_cast<cudaStream_t>(st), tail_decay(c)),
                "adamw_rollback");
}

slip_status slip_set_sm_reserve(int32_t n) {
  SLIP_CHECK(n >= 0 && n < 1024, SLIP_EINVAL, "set_sm_reserve: n out of range");
  set_sm_reserve(n);
  return SLIP_OK;
}

slip_status slip_gemm(int32_t M, int32_t N, int32_t K, const void* a, int64_t lda, int32_t a_mn, const void* b,
                      int64_t ldb, int32_t b_mn, void* c, int64_t ldc, int32_t mode, int32_t bn, int32_t accumulate,
                      float alpha, slip_stream st) {
  SLIP_CHECK(a && b && c, SLIP_EINVAL, "gemm: NULL operand");
  SLIP_CHECK(mode == EPI_BF16 || mode == EPI_F32_STORE || mode == EPI_F32_ACC, SLIP_EINVAL, "gemm: mode");
  GemmDesc d;
  d.M = M;
  d.N = N;
  d.K = K;
  d.bn = bn;
  d.a = op(a, lda, a_mn != 0);
  d.b = op(b, ldb, b_mn != 0);
  d.mode = mode;
  d.c = c;
  d.ldc = ldc;
  d.alpha = alpha;
  d.accumulate = accumulate;
  cudaError_t e = gemm_launch(d, reinterpret_cast<cudaStream_t>(st));
  if (e != cudaSuccess) {
    set_error(std::string("gemm: ") + cudaGetErrorString(e) + " " + gemm_last_message());
    return e == cudaErrorInvalidValue ? SLIP_EUNSUPPORTED : SLIP_ECUDA;
  }
  return SLIP_OK;
}

slip_status slip_attention(int32_t s_len, int32_t heads, int32_t batch, int32_t d, const void* qkv, const void* o,
                           const void* d_o, void* out, float* lse, float* dsum, int32_t backward, slip_stream st) {
  SLIP_CHECK(qkv && out && lse && s_len > 0 && heads > 0 && batch > 0 && d > 0, SLIP_EINVAL, "attention: bad argument");
  SLIP_CHECK(!backward || (o && d_o && dsum), SLIP_EINVAL, "attention: backward needs o, d_o and dsum");
  AttnArgs a;
  a.s = s_len;
  a.heads = heads;
  a.batch = batch;
  a.d = d;
  a.h = static_cast<int64_t>(heads) * d;
  a.qkv_ld = 3 * a.h;
  a.qkv = static_cast<const bf16*>(qkv);
  a.o = static_cast<const bf16*>(o);
  a.dO = static_cast<const bf16*>(d_o);
  a.out = static_cast<bf16*>(out);
  a.lse = lse;
  a.dsum = dsum;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(st);
  cudaError_t e = backward ? attn_backward(a, cs) : attn_forward(a, cs);
  if (e != cudaSuccess) {
    set_error(std::string("attention: ") + cudaGetErrorString(e) + " " + attn_last_message());
    return e == cudaErrorInvalidValue ? SLIP_EUNSUPPORTED : SLIP_ECUDA;
  }
  return SLIP_OK;
}

slip_status slip_weights_from_master(slip_ctx* c, slip_stream st) {
  SLIP_CHECK(c && c->bound, SLIP_EINVAL, "weights_from_master: not bound");
  return kcheck(c, f32_to_bf16(c->master, c->w, c->n_params, reinterpret_cast<cudaStream_t>(st)), "f32_to_bf16");
}

}  // extern "C"
