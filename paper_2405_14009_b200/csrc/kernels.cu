// kernels.cu — HBM-bound kernels of the stage step: LayerNorm fwd/bwd, deterministic
// column reductions (bias / gamma / beta gradients), MSE head, fused AdamW, RNE weight
// refresh and the counter-based input generator.  All launched with PDL (launch.cuh).
//
// Design rules (B200): 16-byte vectors along the contiguous dimension; one thread block
// per row for the row kernels (high occupancy, short per-thread register arrays);
// column reductions write fixed-order partials and the LAST block of each column strip
// (atomic ticket) sums them in chunk order — deterministic, and one launch per reduction.
#include <cmath>

#include "kernels.cuh"
#include "adamw_math.cuh"
#include "gemm.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace slip {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Block-wide sum of two values (blockDim.x multiple of 32, <= 1024); result broadcast.
__device__ __forceinline__ float2 block_sum2(float a, float b, float2* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) red[w] = make_float2(a, b);
  __syncthreads();
  if (w == 0) {
    float2 v = l < nw ? red[l] : make_float2(0.f, 0.f);
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  const float2 r = red[32];
  __syncthreads();  // red reusable by the caller
  return r;
}
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}
// bf16 -> f32 of 8 packed values by shifts / masks in inline asm (see ln_bwd_fused_kernel)
__device__ __forceinline__ void unpack8_asm(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t lo, hi;
    asm("shl.b32 %0, %1, 16;" : "=r"(lo) : "r"(w[i]));
    asm("and.b32 %0, %1, 0xffff0000;" : "=r"(hi) : "r"(w[i]));
    f[2 * i] = __uint_as_float(lo);
    f[2 * i + 1] = __uint_as_float(hi);
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}
__device__ __forceinline__ uint2 pack4(float a, float b, float c, float d) {
  __nv_bfloat162 x = __floats2bfloat162_rn(a, b);
  __nv_bfloat162 y = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&x);
  u.y = *reinterpret_cast<uint32_t*>(&y);
  return u;
}

// ------------------------------------------------------------------ LayerNorm fwd
// One warp per row (8 rows per 256-thread block): lane l owns the 16-byte vectors
// l, l + 32, ... (VPL of them), all loads issued before any reduction, shuffles only —
// many rows in flight per SM, no block barriers.  Two-pass statistics in fp32 (R24).
constexpr int LN_ROWS = 8;
template <int VPL>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gamma,
                                                     const bf16* __restrict__ beta, bf16* __restrict__ y,
                                                     float* __restrict__ mean, float* __restrict__ rstd, int T, int h,
                                                     float eps) {
  // gamma / beta staged in smem by the whole block while the rows load (one latency, not
  // two; the 8 rows of the block share them)
  __shared__ uint4 gb[2][VPL * 32];
  ptx::grid_dep_wait();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * LN_ROWS + (threadIdx.x >> 5);
  const int nv = h >> 3;
  for (int i = threadIdx.x; i < nv; i += 256) {
    gb[0][i] = __ldg(reinterpret_cast<const uint4*>(gamma) + i);
    gb[1][i] = __ldg(reinterpret_cast<const uint4*>(beta) + i);
  }
  uint4 raw[VPL];
  const bool live = row < T;
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(live ? row : 0) * h);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = lane + 32 * i;
    raw[i] = (live && idx < nv) ? xr[idx] : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  if (!live) return;
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    float v[8];
    unpack8(raw[i], v);
#pragma unroll
    for (int e = 0; e < 8; ++e) sum += v[e];
  }
  const float mu = warp_sum(sum) / h;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    if (lane + 32 * i < nv) {
      float v[8];
      unpack8(raw[i], v);
#pragma unroll
      for (int e = 0; e < 8; ++e) sq += (v[e] - mu) * (v[e] - mu);
    }
  }
  const float rs = rsqrtf(warp_sum(sq) / h + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + static_cast<size_t>(row) * h);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      float v[8], g[8], b[8], o[8];
      unpack8(raw[i], v);
      unpack8(gb[0][idx], g);
      unpack8(gb[1][idx], b);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = (v[e] - mu) * rs * g[e] + b[e];
      yr[idx] = pack8(o);
    }
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// ------------------------------------------------------------------ LayerNorm bwd (rows)
// One warp per row.  Pass 1 forms g = dy * gamma and the two row sums from registers
// (dy, x kept as raw 16-byte vectors); pass 2 writes dx = resid + rstd (g - mean(g) -
// xhat mean(g xhat)).  x is fully read before dx is written (dx must not alias x).
template <int VPL>
__global__ void __launch_bounds__(256) ln_bwd_rows_kernel(const bf16* __restrict__ dy, const bf16* x,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ rstd,
                                                          const bf16* __restrict__ gamma,
                                                          const bf16* __restrict__ resid, bf16* dx, int T, int h) {
  ptx::grid_dep_wait();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * LN_ROWS + (threadIdx.x >> 5);
  if (row >= T) return;
  const int nv = h >> 3;
  const float mu = mean[row], rs = rstd[row];
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(row) * h);
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + static_cast<size_t>(row) * h);
  const uint4* rr = resid ? reinterpret_cast<const uint4*>(resid + static_cast<size_t>(row) * h) : nullptr;
  uint4 xv[VPL], dv[VPL], rv[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = lane + 32 * i;
    const bool ok = idx < nv;
    xv[i] = ok ? xr[idx] : make_uint4(0, 0, 0, 0);
    dv[i] = ok ? dyr[idx] : make_uint4(0, 0, 0, 0);
    rv[i] = (ok && rr) ? rr[idx] : make_uint4(0, 0, 0, 0);
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      float a[8], d[8], gm[8];
      unpack8(xv[i], a);
      unpack8(dv[i], d);
      unpack8(reinterpret_cast<const uint4*>(gamma)[idx], gm);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float g = d[e] * gm[e];
        s1 += g;
        s2 += g * ((a[e] - mu) * rs);
      }
    }
  }
  const float mg = warp_sum(s1) / h, mgx = warp_sum(s2) / h;
  uint4* dxr = reinterpret_cast<uint4*>(dx + static_cast<size_t>(row) * h);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      float a[8], d[8], gm[8], r[8], o[8];
      unpack8(xv[i], a);
      unpack8(dv[i], d);
      unpack8(rv[i], r);
      unpack8(reinterpret_cast<const uint4*>(gamma)[idx], gm);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = r[e] + rs * (d[e] * gm[e] - mg - (a[e] - mu) * rs * mgx);
      dxr[idx] = pack8(o);
    }
  }
}

// ------------------------------------------------------------------ column reductions
// One block per 64-column strip covering ALL T rows: 256 threads = 8 column vectors
// (16 bytes each) x 32 row groups; thread (cv, rg) sums rows rg, rg+32, ... of its 8
// columns, then the 32 row-group partials of each column are added in a fixed order —
// deterministic, no partial buffers, no tickets, one launch.
// MODE 0: out0 (+)= sum_t a.
// MODE 1 (LayerNorm): out0 (+)= sum dy*xhat, out1 (+)= sum dy       (a = dy)
// MODE 2 (LayerNorm + producer bias): MODE 1 and out2 (+)= sum_t dx (dx = the LN input grad)
constexpr int CR_COLS = 64;
template <int MODE>
__global__ void __launch_bounds__(256) colred_kernel(const bf16* __restrict__ a, int64_t ld, const bf16* __restrict__ x,
                                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                                     const bf16* __restrict__ dx, int T, int N, float* part,
                                                     float* __restrict__ out0, float* __restrict__ out1,
                                                     float* __restrict__ out2, int accumulate,
                                                     unsigned* __restrict__ tickets) {
  constexpr int NO = MODE == 0 ? 1 : (MODE == 1 ? 2 : 3);  // outputs
  __shared__ float red[NO][32][CR_COLS + 1];
  (void)tickets;
  ptx::grid_dep_wait();
  const int cv = threadIdx.x & 7;
  const int rg = threadIdx.x >> 3;
  const int col = blockIdx.x * CR_COLS + cv * 8;
  // row chunk of this block (gridDim.y chunks; one chunk writes the outputs directly)
  const int R = gridDim.y, rows_per = (T + R - 1) / R;
  const int r0 = blockIdx.y * rows_per, r1 = min(T, r0 + rows_per);
  float acc[NO][8];
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[o][e] = 0.f;
  if (MODE == 0 && col < N) {
    // bias gradients: batches of 8 rows per thread, all 8 loads in flight before the adds
    constexpr int RB = 8;
    for (int rb = r0 + rg; rb < r1; rb += 32 * RB) {
      uint4 q[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        const int r = rb + 32 * b;
        q[b] = r < r1 ? __ldg(reinterpret_cast<const uint4*>(a + static_cast<size_t>(r) * ld + col))
                      : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        float v[8];
        unpack8(q[b], v);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[0][e] += v[e];
      }
    }
  } else if (col < N) {
#pragma unroll 4
    for (int r = r0 + rg; r < r1; r += 32) {
      float v[8];
      unpack8(*reinterpret_cast<const uint4*>(a + static_cast<size_t>(r) * ld + col), v);
      if (MODE == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[0][e] += v[e];
      } else {
        float xv[8];
        unpack8(*reinterpret_cast<const uint4*>(x + static_cast<size_t>(r) * N + col), xv);
        const float mu = mean[r], rs = rstd[r];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          acc[0][e] += v[e] * ((xv[e] - mu) * rs);
          acc[1][e] += v[e];
        }
        if (MODE == 2) {
          float gv[8];
          unpack8(*reinterpret_cast<const uint4*>(dx + static_cast<size_t>(r) * N + col), gv);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[NO - 1][e] += gv[e];
        }
      }
    }
  }
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[o][rg][cv * 8 + e] = acc[o][e];
  __syncthreads();
  if (threadIdx.x < CR_COLS * NO) {
    const int o = threadIdx.x / CR_COLS, c = threadIdx.x % CR_COLS;
    const int gcol = blockIdx.x * CR_COLS + c;
    if (gcol < N) {
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int g = 0; g < 32; ++g) s4[g & 3] += red[o][g][c];
      const float s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      if (part == nullptr) {  // one row chunk, not deferred: the outputs directly
        float* out = o == 0 ? out0 : (o == 1 ? out1 : out2);
        out[gcol] = accumulate ? out[gcol] + s : s;
      } else {
        part[(static_cast<size_t>(o) * R + blockIdx.y) * N + gcol] = s;
      }
    }
  }
}

// ------------------------------------------------------------------ LayerNorm bwd (fused, row blocks)
// The whole LayerNorm backward in ONE pass over the rows (replaces a row-statistics pass +
// a column-strip pass): block b owns rows [b*rpb, (b+1)*rpb) — one block of 512 threads per
// SM; each half of the block (256 threads) takes RB rows per pass, thread t of a half owns
// the 16-byte column vectors t, t + 256, ... (VPT of them) of its rows.
//   loads:  dy, x, resid, mean, rstd of the pass's rows, all in flight before any use;
//   stats:  per row (sum g, sum g xhat), g = dy gamma, over the half's 8 warps (shuffles,
//           then the warps in index order);
//   output: dx = resid + rstd (g - mean_h(g) - xhat mean_h(g xhat)) (bf16), and the column
//           partials dgamma += dy xhat, dbeta += dy (NO = 3: + sum dx as stored) kept in
//           registers across the block's rows;
// at the end the two halves' column partials are added (half 0 + half 1) through shared
// memory and the block writes one partial row per output (part[(o * R + b) * h + c]),
// summed in block order by the deferred finalize (deterministic).  dx == NULL: only
// dgamma, dbeta (NO = 2).
template <int VPT, int NO>
__global__ void __launch_bounds__(512, 1) ln_bwd_fused_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                              const float* __restrict__ mean,
                                                              const float* __restrict__ rstd,
                                                              const bf16* __restrict__ gamma,
                                                              const bf16* __restrict__ resid, bf16* __restrict__ dx,
                                                              int T, int h, int rpb, float* __restrict__ part) {
  constexpr int RB = 4 / VPT;  // rows per half per pass: RB x VPT x 3 x 16 B in flight per thread
  __shared__ float2 red[2][2][8][RB];
  extern __shared__ float comb[];  // [NO][VPT][8][256] half 1's column partials
  ptx::grid_dep_wait();
  const int nv = h >> 3;
  const int hv = threadIdx.x >> 8, tid = threadIdx.x & 255;
  const int warp = tid >> 5, lane = tid & 31;
  const float inv_h = 1.0f / static_cast<float>(h);
  float gm[VPT][8];
  float acc[NO][VPT][8];
#pragma unroll
  for (int v = 0; v < VPT; ++v) {
    const int c = tid + 256 * v;
    unpack8(c < nv ? __ldg(reinterpret_cast<const uint4*>(gamma) + c) : make_uint4(0, 0, 0, 0), gm[v]);
#pragma unroll
    for (int o = 0; o < NO; ++o)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[o][v][e] = 0.f;
  }
  const int rb0 = blockIdx.x * rpb, rb1 = min(T, rb0 + rpb);
  int buf = 0;
  for (int p0 = rb0; p0 < rb1; p0 += 2 * RB, buf ^= 1) {
    const int r0 = p0 + hv * RB;
    uint4 dq[RB][VPT], xq[RB][VPT], rq[RB][VPT];
    float mu[RB], rs[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int r = r0 + b;
      const bool rok = r < rb1;
      mu[b] = rok ? __ldg(mean + r) : 0.f;
      rs[b] = rok ? __ldg(rstd + r) : 0.f;
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c = tid + 256 * v;
        const bool ok = rok && c < nv;
        const size_t o = static_cast<size_t>(ok ? r : 0) * nv + c;
        dq[b][v] = ok ? __ldg(reinterpret_cast<const uint4*>(dy) + o) : make_uint4(0, 0, 0, 0);
        xq[b][v] = ok ? __ldg(reinterpret_cast<const uint4*>(x) + o) : make_uint4(0, 0, 0, 0);
        rq[b][v] = (ok && dx && resid) ? __ldg(reinterpret_cast<const uint4*>(resid) + o) : make_uint4(0, 0, 0, 0);
      }
    }
    float s1[RB], s2[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      s1[b] = 0.f;
      s2[b] = 0.f;
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        // (a second unpack instruction sequence: with the same one the compiler keeps the
        // unpacked rows alive from here to the output pass instead of the packed vectors)
        float d[8], a[8];
        unpack8_asm(dq[b][v], d);
        unpack8_asm(xq[b][v], a);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float g = d[e] * gm[v][e];
          s1[b] += g;
          s2[b] += g * ((a[e] - mu[b]) * rs[b]);
        }
      }
      s1[b] = warp_sum(s1[b]);
      s2[b] = warp_sum(s2[b]);
    }
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < RB; ++b) red[buf][hv][warp][b] = make_float2(s1[b], s2[b]);
    }
    __syncthreads();  // (red is double-buffered: one barrier per pass)
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      float t1 = 0.f, t2 = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const float2 q = red[buf][hv][w][b];
        t1 += q.x;
        t2 += q.y;
      }
      s1[b] = t1 * inv_h;  // mean_h(g)
      s2[b] = t2 * inv_h;  // mean_h(g xhat)
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int r = r0 + b;
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c = tid + 256 * v;
        if (r >= rb1 || c >= nv) continue;  // (no break: the row arrays must stay in registers)
        float d[8], a[8];
        unpack8(dq[b][v], d);
        unpack8(xq[b][v], a);
        if (dx) {
          float rv[8], o[8];
          unpack8(rq[b][v], rv);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float xh = (a[e] - mu[b]) * rs[b];
            acc[0][v][e] += d[e] * xh;
            acc[1][v][e] += d[e];
            o[e] = rv[e] + rs[b] * (d[e] * gm[v][e] - s1[b] - xh * s2[b]);
          }
          const uint4 packed = pack8(o);
          reinterpret_cast<uint4*>(dx)[static_cast<size_t>(r) * nv + c] = packed;
          if (NO == 3) {
            float gv[8];
            unpack8(packed, gv);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[NO - 1][v][e] += gv[e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            acc[0][v][e] += d[e] * ((a[e] - mu[b]) * rs[b]);
            acc[1][v][e] += d[e];
          }
        }
      }
    }
  }
  // half 0 + half 1, then one partial row of each output per block
  if (hv == 1) {
#pragma unroll
    for (int o = 0; o < NO; ++o)
#pragma unroll
      for (int v = 0; v < VPT; ++v)
#pragma unroll
        for (int e = 0; e < 8; ++e) comb[((o * VPT + v) * 8 + e) * 256 + tid] = acc[o][v][e];
  }
  __syncthreads();
  if (hv == 0) {
#pragma unroll
    for (int o = 0; o < NO; ++o)
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c = tid + 256 * v;
        if (c < nv) {
          float t[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) t[e] = acc[o][v][e] + comb[((o * VPT + v) * 8 + e) * 256 + tid];
          float4* dst = reinterpret_cast<float4*>(part + (static_cast<size_t>(o) * gridDim.x + blockIdx.x) * h + 8 * c);
          dst[0] = make_float4(t[0], t[1], t[2], t[3]);
          dst[1] = make_float4(t[4], t[5], t[6], t[7]);
        }
      }
  }
}

// Sum of the R row-chunk partials of each column in chunk order (deterministic).
__global__ void __launch_bounds__(256) colred_finalize_kernel(const float* __restrict__ part, int R, int N, int NO,
                                                              float* __restrict__ out0, float* __restrict__ out1,
                                                              float* __restrict__ out2, int accumulate) {
  ptx::grid_dep_wait();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= N * NO) return;
  const int o = i / N, c = i % N;
  float s = 0.f;
  for (int k = 0; k < R; ++k) s += part[(static_cast<size_t>(o) * R + k) * N + c];
  float* out = o == 0 ? out0 : (o == 1 ? out1 : out2);
  out[c] = accumulate ? out[c] + s : s;
}

// The finalize of many reductions in one launch (a whole B call's bias / LayerNorm
// reductions, see RedBatch): thread i of the concatenated [entry][output][column] space
// sums its column's R partials in chunk order (deterministic, as the per-reduction pass).
// Block = 64 columns x 4 quarters of the R chunks (quarter-major: a warp reads 32
// consecutive columns); the quarters' sums are added in quarter order through smem.
__global__ void __launch_bounds__(256) colred_finalize_batch_kernel(const RedBatch b, int first, int last,
                                                                    int accumulate) {
  __shared__ float qs[4][64];
  ptx::grid_dep_wait();
  const int cl = threadIdx.x & 63, qr = threadIdx.x >> 6;
  const int64_t i = b.start[first] + static_cast<int64_t>(blockIdx.x) * 64 + cl;
  const bool live = i < b.start[last];
  int e = first;
  if (live)
    while (i >= b.start[e + 1]) ++e;
  const RedEntry& r = b.e[e];
  const int k = live ? static_cast<int>(i - b.start[e]) : 0;
  const int o = k / r.N, c = k % r.N;
  float s = 0.f;
  if (live) {
    const float* p = r.part + static_cast<size_t>(o) * r.R * r.N + c;
    const int q0 = (r.R * qr) >> 2, q1 = (r.R * (qr + 1)) >> 2;
    for (int q = q0; q < q1; ++q) s += p[static_cast<size_t>(q) * r.N];
  }
  qs[qr][cl] = s;
  __syncthreads();
  if (qr == 0 && live) {
    const float t = ((qs[0][cl] + qs[1][cl]) + qs[2][cl]) + qs[3][cl];
    float* out = r.out[o];
    out[c] = accumulate ? out[c] + t : t;
  }
}

// Row chunks so that a reduction fills the GPU: about 2 blocks per SM.
int colred_chunks(int N, int per_sm) {
  const int strips = (N + CR_COLS - 1) / CR_COLS;
  int R = (per_sm * 148) / strips;  // whole blocks fit one wave at per_sm resident blocks per SM
  if (R > kRedChunks) R = kRedChunks;
  return R < 1 ? 1 : R;
}

// ------------------------------------------------------------------ MSE head
__global__ void __launch_bounds__(256) mse_kernel(const bf16* __restrict__ y, const bf16* __restrict__ r,
                                                  bf16* __restrict__ dy, float* __restrict__ part, int64_t n8,
                                                  float inv_n) {
  __shared__ float red[8];
  ptx::grid_dep_wait();
  float acc = 0.f;
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n8; i += static_cast<int64_t>(gridDim.x) * 256) {
    float a[8], b[8], d[8];
    unpack8(reinterpret_cast<const uint4*>(y)[i], a);
    unpack8(reinterpret_cast<const uint4*>(r)[i], b);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float df = a[e] - b[e];
      acc += df * df;
      d[e] = df * inv_n;
    }
    reinterpret_cast<uint4*>(dy)[i] = pack8(d);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void mse_finalize_kernel(const float* __restrict__ part, int nparts, float* __restrict__ loss,
                                    float half_inv_n) {
  ptx::grid_dep_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += part[i];
  *loss = s * half_inv_n;
}

// ------------------------------------------------------------------ AdamW
struct WdRanges {
  int64_t a0, a1, b0, b1, c0, c1, d0, d1;
  TailDecay tail;
};
__device__ __forceinline__ bool decays(const WdRanges& wr, int64_t e0, int64_t per_layer) {
  if (e0 >= wr.tail.start) return (e0 >= wr.tail.a0 && e0 < wr.tail.a1) || (e0 >= wr.tail.b0 && e0 < wr.tail.b1);
  const int64_t o = e0 % per_layer;
  return (o >= wr.a0 && o < wr.a1) || (o >= wr.b0 && o < wr.b1) || (o >= wr.c0 && o < wr.c1) ||
         (o >= wr.d0 && o < wr.d1);
}

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ p, float* __restrict__ m,
                                                    float* __restrict__ v, const float* __restrict__ g,
                                                    bf16* __restrict__ w, int64_t n4, int64_t per_layer, WdRanges wr,
                                                    float lr, float b1, float b2, float eps, float wd, float inv_bc1,
                                                    float inv_bc2, float grad_scale, int32_t* __restrict__ nonfinite,
                                                    const int32_t* __restrict__ skip,
                                                    const float* __restrict__ g_peer,
                                                    const float* __restrict__ g_recv) {
  ptx::grid_dep_wait();
  if (skip && *skip) return;  // validated mode: this stage's gradients failed (no step)
  bool bad = false;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * 256;
  // where the peer's gradient of element group j is read: the 2-D weights from g_recv (the
  // peer's W launches pushed them into this GPU's memory), the rest over NVLink
  auto peer_src = [&](int64_t j) {
    return reinterpret_cast<const float4*>((g_recv && decays(wr, 4 * j, per_layer)) ? g_recv : g_peer) + j;
  };
  // the peer's gradient crosses NVLink at a few us of latency: its load for the next
  // iteration is issued before this one's local loads, two remote loads in flight
  float4 gp = make_float4(0.f, 0.f, 0.f, 0.f);
  if (g_peer && blockIdx.x * 256LL + threadIdx.x < n4) gp = __ldcs(peer_src(blockIdx.x * 256LL + threadIdx.x));
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += stride) {
    float4 gp_next = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g_peer && i + stride < n4) gp_next = __ldcs(peer_src(i + stride));
    const int64_t e0 = 4 * i;
    const bool decay = decays(wr, e0, per_layer);
    const float wdl = decay ? wd : 0.f;
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float4 gg = __ldcs(reinterpret_cast<const float4*>(g) + i);
    if (g_peer) {  // DP = 2 all-reduce fused in: the peer's gradient over NVLink; a + b is
                   // commutative in IEEE fp32, so both replicas form the same sum
      gg.x += gp.x;
      gg.y += gp.y;
      gg.z += gp.z;
      gg.w += gp.w;
    }
    float* pa = &pp.x;
    float* ma = &mm.x;
    float* va = &vv.x;
    const float* ga = &gg.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      bad |= !isfinite(ga[e]);
      adamw_update(pa[e], ma[e], va[e], ga[e], lr, b1, b2, eps, wdl, inv_bc1, inv_bc2, grad_scale);
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<uint2*>(w)[i] = pack4(pa[0], pa[1], pa[2], pa[3]);
    gp = gp_next;
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// AdamW over the 1-D parameters of every layer only (bqkv | bo g1 b1n g2 b2n | b1 | b2:
// 9h + f per layer, never decayed): the OPT of a stage whose 2-D weights were already
// stepped in the W GEMM's epilogue (EPI_ADAMW).
__global__ void __launch_bounds__(256) adamw_vectors_kernel(float* __restrict__ p, float* __restrict__ m,
                                                            float* __restrict__ v, const float* __restrict__ g,
                                                            bf16* __restrict__ w, int64_t total, int64_t per_layer,
                                                            int h, int f, float lr, float b1, float b2, float eps,
                                                            float inv_bc1, float inv_bc2, float grad_scale,
                                                            int32_t* __restrict__ nonfinite) {
  ptx::grid_dep_wait();
  const int64_t H = h, F = f, per = 9 * H + F;
  bool bad = false;
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < total; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int64_t layer = i / per, r = i - layer * per;
    int64_t o;
    if (r < 3 * H) o = 3 * H * H + r;                              // bqkv
    else if (r < 8 * H) o = 4 * H * H + 3 * H + (r - 3 * H);       // bo g1 b1n g2 b2n
    else if (r < 8 * H + F) o = 4 * H * H + 8 * H + F * H + (r - 8 * H);  // b1
    else o = 4 * H * H + 8 * H + 2 * F * H + F + (r - 8 * H - F);   // b2
    const int64_t e = layer * per_layer + o;
    float pp = p[e], mm = m[e], vv = v[e];
    const float gg = g[e];
    bad |= !isfinite(gg);
    adamw_update(pp, mm, vv, gg, lr, b1, b2, eps, 0.f, inv_bc1, inv_bc2, grad_scale);
    p[e] = pp;
    m[e] = mm;
    v[e] = vv;
    w[e] = __float2bfloat16_rn(pp);
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// Arithmetic reversal of adamw_kernel (oracle adamw_inverse): given
// the post-step state and the same gradient, restore p, m, v and the bf16 copy.  Acts only
// if *global_bad (some stage failed validation) and not *own_bad (this stage stepped);
// the first acting block counts the rollback.
__global__ void __launch_bounds__(256) adamw_rollback_kernel(
    float* __restrict__ p, float* __restrict__ m, float* __restrict__ v, const float* __restrict__ g,
    bf16* __restrict__ w, int64_t n4, int64_t per_layer, WdRanges wr, float lr, float b1, float b2, float eps, float wd,
    float inv_bc1, float inv_bc2, float grad_scale, const int32_t* __restrict__ global_bad,
    const int32_t* __restrict__ own_bad, int32_t* __restrict__ count) {
  ptx::grid_dep_wait();
  if ((global_bad && !*global_bad) || (own_bad && *own_bad)) return;
  if (count && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(count, 1);
  const float ib1 = 1.f / b1, ib2 = 1.f / b2;
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int64_t e0 = 4 * i;
    const bool decay = decays(wr, e0, per_layer);
    const float wdl = decay ? wd : 0.f;
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float* pa = &pp.x;
    float* ma = &mm.x;
    float* va = &vv.x;
    const float* ga = &gg.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gr = grad_scale * ga[e];
      const float mh = ma[e] * inv_bc1;
      const float vh = va[e] * inv_bc2;
      pa[e] = (pa[e] + lr * mh / (sqrtf(vh) + eps)) / (1.f - lr * wdl);
      ma[e] = (ma[e] - (1.f - b1) * gr) * ib1;
      va[e] = fmaxf((va[e] - (1.f - b2) * gr * gr) * ib2, 0.f);
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<uint2*>(w)[i] = pack4(pa[0], pa[1], pa[2], pa[3]);
  }
}

// Local validation: OR of "some gradient element is not finite" into
// *bad (and into *nonfinite for the report).
__global__ void __launch_bounds__(256) grad_check_kernel(const float* __restrict__ g, int64_t n4,
                                                         int32_t* __restrict__ bad, int32_t* __restrict__ nonfinite) {
  ptx::grid_dep_wait();
  bool b = false;
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += static_cast<int64_t>(gridDim.x) * 256) {
    const float4 x = reinterpret_cast<const float4*>(g)[i];
    b |= !isfinite(x.x) || !isfinite(x.y) || !isfinite(x.z) || !isfinite(x.w);
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) {
    atomicOr(bad, 1);
    if (nonfinite) atomicOr(nonfinite, 1);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, bf16* __restrict__ dst, int64_t n4) {
  ptx::grid_dep_wait();
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += static_cast<int64_t>(gridDim.x) * 256) {
    const float4 a = reinterpret_cast<const float4*>(src)[i];
    reinterpret_cast<uint2*>(dst)[i] = pack4(a.x, a.y, a.z, a.w);
  }
}

// ------------------------------------------------------------------ Philox4x32-10
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__global__ void synth_normal_kernel(bf16* __restrict__ out, int64_t n, uint2 key, uint32_t kk, uint32_t jj) {
  ptx::grid_dep_wait();
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; 4 * i < n; i += static_cast<int64_t>(gridDim.x) * 256) {
    const uint4 r = philox(make_uint4(static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32), jj, kk), key);
    const float u1 = (static_cast<float>(r.x) + 1.0f) * 2.3283064365386963e-10f;
    const float u2 = static_cast<float>(r.y) * 2.3283064365386963e-10f;
    const float u3 = (static_cast<float>(r.z) + 1.0f) * 2.3283064365386963e-10f;
    const float u4 = static_cast<float>(r.w) * 2.3283064365386963e-10f;
    const float ra = sqrtf(-2.0f * logf(u1)), rb = sqrtf(-2.0f * logf(u3));
    float z[4];
    sincospif(2.0f * u2, &z[1], &z[0]);
    sincospif(2.0f * u4, &z[3], &z[2]);
    z[0] *= ra;
    z[1] *= ra;
    z[2] *= rb;
    z[3] *= rb;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (4 * i + e < n) out[4 * i + e] = __float2bfloat16_rn(z[e]);
  }
}

// ------------------------------------------------------------------ GPT ends (reading R33)
// X[t] = E[tok[t]] + P[t mod seq]: one warp per token row, 16-byte vectors.
__global__ void __launch_bounds__(256) embed_fwd_kernel(const bf16* __restrict__ E, const bf16* __restrict__ P,
                                                        const int32_t* __restrict__ tok, bf16* __restrict__ X, int T,
                                                        int h, int seq, int V) {
  ptx::grid_dep_wait();
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= T) return;
  const int v = tok[t];
  const bool ok = v >= 0 && v < V;  // an id outside the vocabulary reads a zero embedding row
  const uint4* er = reinterpret_cast<const uint4*>(E + static_cast<int64_t>(ok ? v : 0) * h);
  const uint4* pr = reinterpret_cast<const uint4*>(P + static_cast<int64_t>(t % seq) * h);
  uint4* xr = reinterpret_cast<uint4*>(X + static_cast<int64_t>(t) * h);
  for (int i = lane; i < h / 8; i += 32) {
    float a[8], b[8];
    unpack8(ok ? er[i] : make_uint4(0, 0, 0, 0), a);
    unpack8(pr[i], b);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += b[e];
    xr[i] = pack8(a);
  }
}

// Embedding scatter, deterministic without atomics: block t owns token tok[t] iff t is
// its first occurrence; warp 0 lists the occurrences in t order (ballots over 32-token
// chunks) and the block sums their rows in that order.  Blocks T .. T+seq-1 own the
// position rows (sum over the micro-batch's sequences in order).
__global__ void __launch_bounds__(256) embed_bwd_kernel(const bf16* __restrict__ dX, const int32_t* __restrict__ tok,
                                                        float* __restrict__ dE, float* __restrict__ dP, int T, int h,
                                                        int seq, int accumulate, int V) {
  ptx::grid_dep_wait();
  extern __shared__ int occ[];  // [T] occurrence list
  __shared__ int n_occ;
  const int b = blockIdx.x;
  if (b < T) {
    const int v = tok[b];
    if (v < 0 || v >= V) return;  // an id outside the vocabulary has no embedding row
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      bool earlier = false;
      int n = 0;
      for (int u0 = 0; u0 < T; u0 += 32) {
        const int u = u0 + lane;
        const bool hit = u < T && tok[u] == v;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (u0 < b) {  // hits at positions u < b mean an earlier occurrence of v
          const unsigned below = b - u0 >= 32 ? 0xffffffffu : ((1u << (b - u0)) - 1u);
          earlier = earlier || (m & below) != 0u;
        }
        if (hit) occ[n + __popc(m & ((1u << lane) - 1u))] = u;
        n += __popc(m);
      }
      if (lane == 0) n_occ = earlier ? 0 : n;  // not the first occurrence: another block owns v
    }
    __syncthreads();
    const int n = n_occ;
    if (n == 0) return;
    float* out = dE + static_cast<int64_t>(v) * h;
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      float acc = 0.f;
      for (int q = 0; q < n; ++q) acc += __bfloat162float(dX[static_cast<int64_t>(occ[q]) * h + c]);
      out[c] = accumulate ? out[c] + acc : acc;
    }
  } else {
    const int p = b - T;
    float* out = dP + static_cast<int64_t>(p) * h;
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      float acc = 0.f;
      for (int u = p; u < T; u += seq) acc += __bfloat162float(dX[static_cast<int64_t>(u) * h + c]);
      out[c] = accumulate ? out[c] + acc : acc;
    }
  }
}

// Cross-entropy over one logits row per block (V bf16, read three times from L1/L2):
// max, sum of exp, then dLogits in place and the row's loss.
__global__ void __launch_bounds__(512) ce_rows_kernel(bf16* __restrict__ logits, const int32_t* __restrict__ labels,
                                                      float* __restrict__ row_loss, int V, float inv_T) {
  __shared__ float2 red[33];
  ptx::grid_dep_wait();
  const int t = blockIdx.x;
  bf16* row = logits + static_cast<int64_t>(t) * V;
  const uint4* r4 = reinterpret_cast<const uint4*>(row);
  const int nv = V / 8;
  float mx = -INFINITY;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    float a[8];
    unpack8(r4[i], a);
#pragma unroll
    for (int e = 0; e < 8; ++e) mx = fmaxf(mx, a[e]);
  }
  // block max through the pair reduction (second slot unused)
  {
    float v = mx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w].x = v;
    __syncthreads();
    if (w == 0) {
      float u = l < static_cast<int>(blockDim.x >> 5) ? red[l].x : -INFINITY;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) u = fmaxf(u, __shfl_xor_sync(0xffffffffu, u, o));
      if (l == 0) red[32].x = u;
    }
    __syncthreads();
    mx = red[32].x;
    __syncthreads();
  }
  float se = 0.f;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    float a[8];
    unpack8(r4[i], a);
#pragma unroll
    for (int e = 0; e < 8; ++e) se += __expf(a[e] - mx);
  }
  se = block_sum2(se, 0.f, red).x;
  const float lse = mx + logf(se);
  const int lab = labels[t];
  // a label outside the vocabulary marks an ignored row: loss 0, dLogits 0
  const bool ok = lab >= 0 && lab < V;
  const float zl = ok ? __bfloat162float(row[lab]) : 0.f;
  __syncthreads();  // every thread has read row[lab] before any dLogits write
  const float inv_se = 1.f / se;
  uint4* w4 = reinterpret_cast<uint4*>(row);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    float a[8];
    unpack8(r4[i], a);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      a[e] = ok ? (__expf(a[e] - mx) * inv_se - (8 * i + e == lab ? 1.f : 0.f)) * inv_T : 0.f;
    w4[i] = pack8(a);
  }
  if (threadIdx.x == 0) row_loss[t] = ok ? lse - zl : 0.f;
}

__global__ void mean_kernel(const float* __restrict__ x, int n, float* __restrict__ out) {
  ptx::grid_dep_wait();
  __shared__ float2 red[33];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];  // fixed per-thread order
  const float s = block_sum2(acc, 0.f, red).x;
  if (threadIdx.x == 0) *out = s / n;
}

__global__ void synth_tokens_kernel(int32_t* __restrict__ out, int64_t n, int32_t classes, uint2 key, uint32_t kk,
                                    uint32_t jj) {
  ptx::grid_dep_wait();
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * 256) {
    const uint4 r = philox(make_uint4(static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32), jj, kk), key);
    out[i] = static_cast<int32_t>((static_cast<uint64_t>(r.x) * static_cast<uint64_t>(classes)) >> 32);
  }
}

int grid_for(int64_t work, int per_block = 256) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : static_cast<int>(g);
}

// 16-byte vectors per lane for a row of h bf16 (one warp per row)
int ln_vpl(int h) { return (h / 8 + 31) / 32; }

}  // namespace

#define SLIP_LN_VPL_CASES(X) X(1) X(2) X(4) X(8) X(10) X(16) X(32)
cudaError_t ln_fwd(const bf16* x, const bf16* gamma, const bf16* beta, bf16* y, float* mean, float* rstd, int T, int h,
                   float eps, cudaStream_t s) {
  if (h % 8 || h > 8192) return cudaErrorInvalidValue;
  const int v = ln_vpl(h);
  const dim3 grid((T + LN_ROWS - 1) / LN_ROWS);
#define X(n) \
  if (v <= n) return launch_pdl(ln_fwd_kernel<n>, grid, dim3(256), 0, s, 1, x, gamma, beta, y, mean, rstd, T, h, eps);
  SLIP_LN_VPL_CASES(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t ln_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* gamma,
                   const bf16* resid, bf16* dx, float* dgamma, float* dbeta, float* dxsum, int accumulate, float* part,
                   unsigned* tickets, int T, int h, cudaStream_t s, RedBatch* defer) {
  if (h % 8 || h > 8192) return cudaErrorInvalidValue;
  if ((h + 255) / 256 > kTickets || dx == x) return cudaErrorInvalidValue;
  if (dx) {
    const int v = ln_vpl(h);
    const dim3 grid((T + LN_ROWS - 1) / LN_ROWS);
    cudaError_t e = cudaErrorInvalidValue;
#define X(n)                                                                                                      \
  if (e == cudaErrorInvalidValue && v <= n)                                                                       \
    e = launch_pdl(ln_bwd_rows_kernel<n>, grid, dim3(256), 0, s, 1, dy, x, mean, rstd, gamma, resid, dx, T, h); \
  else
    SLIP_LN_VPL_CASES(X) {}
#undef X
    if (e != cudaSuccess) return e;
  }
  const int R = colred_chunks(h, 4);
  dim3 grid((h + CR_COLS - 1) / CR_COLS, R);
  const bool three = dx && dxsum;
  const int NO = three ? 3 : 2;
  if (defer) {
    part = defer->add(R, h, NO, dgamma, dbeta, three ? dxsum : nullptr);
    if (!part) return cudaErrorInvalidValue;
  } else if (R == 1) {
    part = nullptr;
  }
  cudaError_t e = three ? launch_pdl(colred_kernel<2>, grid, dim3(256), 0, s, 1, dy, static_cast<int64_t>(h), x, mean,
                                     rstd, static_cast<const bf16*>(dx), T, h, part, dgamma, dbeta, dxsum, accumulate,
                                     tickets)
                        : launch_pdl(colred_kernel<1>, grid, dim3(256), 0, s, 1, dy, static_cast<int64_t>(h), x, mean,
                                     rstd, static_cast<const bf16*>(nullptr), T, h, part, dgamma, dbeta,
                                     static_cast<float*>(nullptr), accumulate, tickets);
  if (e != cudaSuccess || R == 1 || defer) return e;
  return launch_pdl(colred_finalize_kernel, dim3((h * NO + 255) / 256), dim3(256), 0, s, 1,
                    static_cast<const float*>(part), R, h, NO, dgamma, dbeta, three ? dxsum : static_cast<float*>(nullptr),
                    accumulate);
}

cudaError_t ln_bwd_fused(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* gamma,
                         const bf16* resid, bf16* dx, float* dgamma, float* dbeta, float* dxsum, int T, int h,
                         cudaStream_t s, RedBatch* defer) {
  const int nv = h / 8;
  const int vpt = (nv + 255) / 256;
  if (h % 8 || vpt > 4 || !defer || (dx && (dx == x || dx == dy)) || (dxsum && !dx)) return cudaErrorInvalidValue;
  const int vp = vpt <= 1 ? 1 : (vpt <= 2 ? 2 : 4);
  // one block of 16 warps per SM: the partial rows (one per block) stay few
  const int rpb = (T + num_sms() - 1) / num_sms();
  const int nb = (T + rpb - 1) / rpb;
  const bool three = dxsum != nullptr;
  const int NO = three ? 3 : 2;
  float* part = defer->add(nb, h, NO, dgamma, dbeta, three ? dxsum : nullptr);
  if (!part) return cudaErrorInvalidValue;
  const int smem = NO * vp * 8 * 256 * static_cast<int>(sizeof(float));
#define L(V, N)                                                                                                    \
  [&]() -> cudaError_t {                                                                                           \
    static bool attr_ = false;                                                                                     \
    if (!attr_) {                                                                                                  \
      cudaFuncSetAttribute(ln_bwd_fused_kernel<V, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);     \
      attr_ = true;                                                                                                \
    }                                                                                                              \
    return launch_pdl(ln_bwd_fused_kernel<V, N>, dim3(nb), dim3(512), smem, s, 1, dy, x, mean, rstd, gamma, resid, \
                      dx, T, h, rpb, part);                                                                        \
  }()
  if (vp == 1) return three ? L(1, 3) : L(1, 2);
  if (vp == 2) return three ? L(2, 3) : L(2, 2);
  return three ? L(4, 3) : L(4, 2);
#undef L
}

int ln_bwd_fused_parts(int T, int h) {
  (void)h;
  const int rpb = (T + num_sms() - 1) / num_sms();
  return (T + rpb - 1) / rpb;
}

int colred_launches(int N) { return colred_chunks(N, 4) > 1 ? 2 : 1; }

// an upper bound of every variant's partials (the most chunks: 4 blocks per SM)
size_t colred_part_floats(int N, int NO) { return static_cast<size_t>(colred_chunks(N, 4)) * N * NO; }

float* RedBatch::add(int R, int N, int NO, float* o0, float* o1, float* o2) {
  if (n == kMaxRed) return nullptr;
  const size_t need = static_cast<size_t>(R) * N * NO;
  if (used + need > cap) return nullptr;
  RedEntry& r = e[n];
  r.part = arena + used;
  r.out[0] = o0;
  r.out[1] = o1;
  r.out[2] = o2;
  r.R = R;
  r.N = N;
  start[n + 1] = start[n] + static_cast<int64_t>(N) * NO;
  used += need;
  ++n;
  return r.part;
}

cudaError_t colred_finalize_batch(const RedBatch& b, int accumulate, cudaStream_t s, int* launches) {
  *launches = 0;
  if (b.n == 0) return cudaSuccess;
  const int64_t total = b.start[b.n];
  const int blocks = static_cast<int>((total + 63) / 64);
  *launches = 1;
  return launch_pdl(colred_finalize_batch_kernel, dim3(blocks), dim3(256), 0, s, 1, b, 0, b.n, accumulate);
}

cudaError_t colsum(const bf16* a, int T, int N, int64_t ld, float* out, int accumulate, float* part,
                   unsigned* tickets, cudaStream_t s, RedBatch* defer) {
  if (N % 8 || ld % 8 || (N + 255) / 256 > kTickets) return cudaErrorInvalidValue;
  const int R = colred_chunks(N, 4);
  dim3 grid((N + CR_COLS - 1) / CR_COLS, R);
  if (defer) {
    part = defer->add(R, N, 1, out, nullptr, nullptr);
    if (!part) return cudaErrorInvalidValue;
  } else if (R == 1) {
    part = nullptr;
  }
  cudaError_t e = launch_pdl(colred_kernel<0>, grid, dim3(256), 0, s, 1, a, ld, static_cast<const bf16*>(nullptr),
                             static_cast<const float*>(nullptr), static_cast<const float*>(nullptr),
                             static_cast<const bf16*>(nullptr), T, N, part, out, static_cast<float*>(nullptr),
                             static_cast<float*>(nullptr), accumulate, tickets);
  if (e != cudaSuccess || R == 1 || defer) return e;
  return launch_pdl(colred_finalize_kernel, dim3((N + 255) / 256), dim3(256), 0, s, 1, static_cast<const float*>(part),
                    R, N, 1, out, static_cast<float*>(nullptr), static_cast<float*>(nullptr), accumulate);
}

cudaError_t mse_loss(const bf16* y, const bf16* r, bf16* dy, float* part, int nparts, float* loss, int64_t n,
                     cudaStream_t s) {
  if (n % 8) return cudaErrorInvalidValue;
  cudaError_t e = launch_pdl(mse_kernel, dim3(nparts), dim3(256), 0, s, 1, y, r, dy, part, n / 8,
                             1.0f / static_cast<float>(n));
  if (e != cudaSuccess) return e;
  return launch_pdl(mse_finalize_kernel, dim3(1), dim3(32), 0, s, 1, static_cast<const float*>(part), nparts, loss,
                    0.5f / static_cast<float>(n));
}

namespace {
WdRanges wd_ranges(int h, int f) {
  const int64_t H = h, F = f;
  WdRanges wr;
  wr.a0 = 0;
  wr.a1 = 3 * H * H;
  wr.b0 = 3 * H * H + 3 * H;
  wr.b1 = wr.b0 + H * H;
  wr.c0 = 4 * H * H + 8 * H;
  wr.c1 = wr.c0 + F * H;
  wr.d0 = wr.c1 + F;
  wr.d1 = wr.d0 + H * F;
  return wr;
}
}  // namespace

cudaError_t adamw_rollback(float* p, float* m, float* v, const float* g, bf16* w, int64_t n, int64_t per_layer, int h,
                           int f, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                           float grad_scale, const int32_t* global_bad, const int32_t* own_bad, int32_t* count,
                           cudaStream_t s, TailDecay tail) {
  if (n % 4 || per_layer % 4) return cudaErrorInvalidValue;
  WdRanges wr = wd_ranges(h, f);
  wr.tail = tail;
  return launch_pdl(adamw_rollback_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, 1, p, m, v, g, w, n / 4, per_layer,
                    wr, lr, b1, b2, eps, wd, 1.0f / bc1, 1.0f / bc2, grad_scale, global_bad, own_bad,
                    count);
}

__global__ void count_flag_kernel(const int32_t* __restrict__ flag, int32_t* __restrict__ count) {
  ptx::grid_dep_wait();
  if (threadIdx.x == 0 && *flag) *count += 1;
}

__global__ void or_flags_kernel(int32_t* __restrict__ own, const int32_t* __restrict__ flags, int n) {
  ptx::grid_dep_wait();
  if (threadIdx.x != 0) return;
  int32_t v = *own;
  for (int i = 0; i < n; ++i) v |= flags[i] != 0;
  *own = v;
}

cudaError_t or_flags(int32_t* own, const int32_t* flags, int n, cudaStream_t s) {
  return launch_pdl(or_flags_kernel, dim3(1), dim3(32), 0, s, 1, own, flags, n);
}

cudaError_t count_flag(const int32_t* flag, int32_t* count, cudaStream_t s) {
  return launch_pdl(count_flag_kernel, dim3(1), dim3(32), 0, s, 1, flag, count);
}

cudaError_t grad_check(const float* g, int64_t n, int32_t* bad, int32_t* nonfinite, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  return launch_pdl(grad_check_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, 1, g, n / 4, bad, nonfinite);
}

cudaError_t adamw(float* p, float* m, float* v, const float* g, bf16* w, int64_t n, int64_t per_layer, int h, int f,
                  float lr, float b1, float b2, float eps, float wd, float bc1, float bc2, float grad_scale,
                  int32_t* nonfinite, cudaStream_t s, const int32_t* skip, TailDecay tail, const float* g_peer,
                  const float* g_recv) {
  if (n % 4 || per_layer % 4) return cudaErrorInvalidValue;
  const int64_t H = h, F = f;
  WdRanges wr;
  wr.tail = tail;
  wr.a0 = 0;
  wr.a1 = 3 * H * H;
  wr.b0 = 3 * H * H + 3 * H;
  wr.b1 = wr.b0 + H * H;
  wr.c0 = 4 * H * H + 8 * H;
  wr.c1 = wr.c0 + F * H;
  wr.d0 = wr.c1 + F;
  wr.d1 = wr.d0 + H * F;
  return launch_pdl(adamw_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, 1, p, m, v, g, w, n / 4, per_layer, wr, lr,
                    b1, b2, eps, wd, 1.0f / bc1, 1.0f / bc2, grad_scale, nonfinite, skip, g_peer, g_recv);
}

cudaError_t adamw_vectors(float* p, float* m, float* v, const float* g, bf16* w, int layers, int64_t per_layer, int h,
                          int f, float lr, float b1, float b2, float eps, float bc1, float bc2, float grad_scale,
                          int32_t* nonfinite, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(layers) * (9LL * h + f);
  return launch_pdl(adamw_vectors_kernel, dim3(grid_for(total)), dim3(256), 0, s, 1, p, m, v, g, w, total, per_layer, h,
                    f, lr, b1, b2, eps, 1.0f / bc1, 1.0f / bc2, grad_scale, nonfinite);
}

// Two-GPU barrier through peer-mapped flags (the fused DP = 2 all-reduce, comm.cpp):
// publish `epoch` into the peer's flag with a system-scope release (after a system
// fence, so every earlier kernel's writes on this GPU are visible to the peer), then
// spin on the own flag with acquire loads.  A peer that never arrives is a bug, not a
// failure mode (failed ranks have no stage group): trap after 30 s rather than hang.
__global__ void peer_barrier_kernel(unsigned* peer_flag, const unsigned* my_flag, unsigned epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer_flag), "r"(epoch) : "memory");
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flag) : "memory");
    if (static_cast<int>(v - epoch) >= 0) break;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 30000000000ull) __trap();
    __nanosleep(256);
  }
}

cudaError_t peer_barrier(unsigned* peer_flag, const unsigned* my_flag, unsigned epoch, cudaStream_t s) {
  peer_barrier_kernel<<<1, 32, 0, s>>>(peer_flag, my_flag, epoch);
  return cudaGetLastError();
}

cudaError_t f32_to_bf16(const float* src, bf16* dst, int64_t n, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  return launch_pdl(f32_to_bf16_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, 1, src, dst, n / 4);
}

cudaError_t synth_normal(bf16* out, int64_t n, uint64_t seed, uint64_t k, uint64_t j, cudaStream_t s) {
  uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  return launch_pdl(synth_normal_kernel, dim3(grid_for((n + 3) / 4)), dim3(256), 0, s, 1, out, n, key,
                    static_cast<uint32_t>(k), static_cast<uint32_t>(j));
}

cudaError_t embed_fwd(const bf16* E, const bf16* P, const int32_t* tok, bf16* X, int T, int h, int seq, int V,
                      cudaStream_t s) {
  if (h % 8) return cudaErrorInvalidValue;
  return launch_pdl(embed_fwd_kernel, dim3((T + 7) / 8), dim3(256), 0, s, 1, E, P, tok, X, T, h, seq, V);
}

cudaError_t embed_bwd(const bf16* dX, const int32_t* tok, float* dE, float* dP, int T, int h, int seq, int V,
                      int accumulate, cudaStream_t s) {
  if (T > 12288) return cudaErrorInvalidValue;  // occurrence list in shared memory
  return launch_pdl(embed_bwd_kernel, dim3(T + seq), dim3(256), static_cast<size_t>(T) * sizeof(int), s, 1, dX, tok,
                    dE, dP, T, h, seq, accumulate, V);
}

cudaError_t cross_entropy(bf16* logits, const int32_t* labels, float* row_loss, float* loss, int T, int V,
                          cudaStream_t s) {
  if (V % 8) return cudaErrorInvalidValue;
  cudaError_t e = launch_pdl(ce_rows_kernel, dim3(T), dim3(512), 0, s, 1, logits, labels, row_loss, V,
                             1.0f / static_cast<float>(T));
  if (e != cudaSuccess) return e;
  return launch_pdl(mean_kernel, dim3(1), dim3(1024), 0, s, 1, static_cast<const float*>(row_loss), T, loss);
}

cudaError_t synth_tokens(int32_t* out, int64_t n, int32_t n_classes, uint64_t seed, uint64_t k, uint64_t j,
                         cudaStream_t s) {
  uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  return launch_pdl(synth_tokens_kernel, dim3(grid_for(n)), dim3(256), 0, s, 1, out, n, n_classes, key,
                    static_cast<uint32_t>(k), static_cast<uint32_t>(j));
}

}  // namespace slip
