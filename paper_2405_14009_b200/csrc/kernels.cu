// kernels.cu — HBM-bound kernels of the stage step: LayerNorm fwd/bwd, causal softmax
// fwd/bwd, deterministic column reductions (bias / gamma / beta gradients), MSE head,
// fused AdamW, RNE weight refresh and the counter-based input generator.
// Every kernel reads/writes with 16-byte vectors along the contiguous dimension and
// reduces with warp shuffles; column reductions go through fixed-order partials so
// results are bitwise reproducible run to run.
#include <cmath>

#include "kernels.cuh"

namespace slip {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
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
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// ------------------------------------------------------------------ LayerNorm fwd
template <int MAXI>
__global__ void __launch_bounds__(128) ln_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gamma,
                                                     const bf16* __restrict__ beta, bf16* __restrict__ y,
                                                     float* __restrict__ mean, float* __restrict__ rstd, int T, int h,
                                                     float eps) {
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const int nv = h >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(row) * h);
  float v[MAXI][8];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      unpack8(xr[idx], v[i]);
#pragma unroll
      for (int e = 0; e < 8; ++e) sum += v[i][e];
    }
  }
  const float mu = warp_sum(sum) / h;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    if (lane + 32 * i < nv) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = v[i][e] - mu;
        sq += d * d;
      }
    }
  }
  const float rs = rsqrtf(warp_sum(sq) / h + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + static_cast<size_t>(row) * h);
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      float g[8], b[8], o[8];
      unpack8(reinterpret_cast<const uint4*>(gamma)[idx], g);
      unpack8(reinterpret_cast<const uint4*>(beta)[idx], b);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = (v[i][e] - mu) * rs * g[e] + b[e];
      yr[idx] = pack8(o);
    }
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// ------------------------------------------------------------------ LayerNorm bwd (rows)
template <int MAXI>
__global__ void __launch_bounds__(128) ln_bwd_rows_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ rstd,
                                                          const bf16* __restrict__ gamma,
                                                          const bf16* __restrict__ resid, bf16* __restrict__ dx,
                                                          int T, int h) {
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const int nv = h >> 3;
  const float mu = mean[row], rs = rstd[row];
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(row) * h);
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + static_cast<size_t>(row) * h);
  float g[MAXI][8], xh[MAXI][8];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      float xv[8], dv[8], gm[8];
      unpack8(xr[idx], xv);
      unpack8(dyr[idx], dv);
      unpack8(reinterpret_cast<const uint4*>(gamma)[idx], gm);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xh[i][e] = (xv[e] - mu) * rs;
        g[i][e] = dv[e] * gm[e];
        s1 += g[i][e];
        s2 += g[i][e] * xh[i][e];
      }
    }
  }
  const float mg = warp_sum(s1) / h;
  const float mgx = warp_sum(s2) / h;
  uint4* dxr = reinterpret_cast<uint4*>(dx + static_cast<size_t>(row) * h);
  const uint4* rr = resid ? reinterpret_cast<const uint4*>(resid + static_cast<size_t>(row) * h) : nullptr;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      float o[8], rv[8];
      if (rr) {
        unpack8(rr[idx], rv);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) rv[e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = rv[e] + rs * (g[i][e] - mg - xh[i][e] * mgx);
      dxr[idx] = pack8(o);
    }
  }
}

// ------------------------------------------------------------------ column reductions
// grid (ceil(N/256), kRedChunks), block 256 = 32 column-vectors x 8 row groups.
// MODE 0: part0 = sum a.  MODE 1 (LayerNorm): part0 = sum dy*xhat, part1 = sum dy.
template <int MODE>
__global__ void __launch_bounds__(256) colred_kernel(const bf16* __restrict__ a, int64_t ld, const bf16* __restrict__ x,
                                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                                     int T, int N, float* __restrict__ part0,
                                                     float* __restrict__ part1) {
  __shared__ float red0[8][256];
  __shared__ float red1[MODE == 1 ? 8 : 1][256];
  const int cv = threadIdx.x & 31;
  const int rg = threadIdx.x >> 5;
  const int col = (blockIdx.x * 32 + cv) * 8;
  const int chunk = blockIdx.y;
  const int rows_per = (T + kRedChunks - 1) / kRedChunks;
  const int r0 = chunk * rows_per;
  const int r1 = min(T, r0 + rows_per);
  float acc0[8], acc1[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc0[e] = acc1[e] = 0.f;
  if (col < N) {
    for (int r = r0 + rg; r < r1; r += 8) {
      float v[8];
      unpack8(*reinterpret_cast<const uint4*>(a + static_cast<size_t>(r) * ld + col), v);
      if (MODE == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc0[e] += v[e];
      } else {
        float xv[8];
        unpack8(*reinterpret_cast<const uint4*>(x + static_cast<size_t>(r) * N + col), xv);
        const float mu = mean[r], rs = rstd[r];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          acc0[e] += v[e] * ((xv[e] - mu) * rs);
          acc1[e] += v[e];
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red0[rg][cv * 8 + e] = acc0[e];
    if (MODE == 1) red1[rg][cv * 8 + e] = acc1[e];
  }
  __syncthreads();
  const int c = threadIdx.x;  // 256 columns of this block
  const int gcol = blockIdx.x * 256 + c;
  if (gcol < N) {
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      s0 += red0[g][c];
      if (MODE == 1) s1 += red1[g][c];
    }
    part0[static_cast<size_t>(chunk) * N + gcol] = s0;
    if (MODE == 1) part1[static_cast<size_t>(chunk) * N + gcol] = s1;
  }
}

__global__ void colsum_finalize_kernel(const float* __restrict__ part, int N, float* __restrict__ out, int accumulate) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (int c = 0; c < kRedChunks; ++c) s += part[static_cast<size_t>(c) * N + n];
  out[n] = accumulate ? out[n] + s : s;
}

// ------------------------------------------------------------------ causal softmax
template <int MAXI>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const float* __restrict__ S, bf16* __restrict__ P,
                                                          int rows, int s) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int t = r % s;
  const int E = min(s, ((t + 1 + 127) / 128) * 128);
  const float* sr = S + static_cast<size_t>(r) * s;
  const float L2E = 1.4426950408889634f;
  float v[MAXI][4];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int c = 4 * lane + 128 * i;
    if (c < E) {
      const float4 q = *reinterpret_cast<const float4*>(sr + c);
      v[i][0] = (c + 0 <= t) ? q.x : -INFINITY;
      v[i][1] = (c + 1 <= t) ? q.y : -INFINITY;
      v[i][2] = (c + 2 <= t) ? q.z : -INFINITY;
      v[i][3] = (c + 3 <= t) ? q.w : -INFINITY;
#pragma unroll
      for (int e = 0; e < 4; ++e) mx = fmaxf(mx, v[i][e]);
    }
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    if (4 * lane + 128 * i < E) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[i][e] = exp2f((v[i][e] - mx) * L2E);
        sum += v[i][e];
      }
    }
  }
  const float inv = 1.0f / warp_sum(sum);
  bf16* pr = P + static_cast<size_t>(r) * s;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int c = 4 * lane + 128 * i;
    if (c < E) {
      __nv_bfloat162 a = __floats2bfloat162_rn(v[i][0] * inv, v[i][1] * inv);
      __nv_bfloat162 b = __floats2bfloat162_rn(v[i][2] * inv, v[i][3] * inv);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&a);
      u.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(pr + c) = u;
    }
  }
}

template <int MAXI>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const float* __restrict__ dP, const bf16* __restrict__ P,
                                                          bf16* __restrict__ dS, int rows, int s, float scale) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int t = r % s;
  const int E = min(s, ((t + 1 + 127) / 128) * 128);
  const float* dr = dP + static_cast<size_t>(r) * s;
  const bf16* pr = P + static_cast<size_t>(r) * s;
  float pv[MAXI][4], dv[MAXI][4];
  float dot = 0.f;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int c = 4 * lane + 128 * i;
    if (c < E) {
      const float4 q = *reinterpret_cast<const float4*>(dr + c);
      const uint2 u = *reinterpret_cast<const uint2*>(pr + c);
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      pv[i][0] = (c + 0 <= t) ? a.x : 0.f;
      pv[i][1] = (c + 1 <= t) ? a.y : 0.f;
      pv[i][2] = (c + 2 <= t) ? b.x : 0.f;
      pv[i][3] = (c + 3 <= t) ? b.y : 0.f;
      dv[i][0] = q.x;
      dv[i][1] = q.y;
      dv[i][2] = q.z;
      dv[i][3] = q.w;
#pragma unroll
      for (int e = 0; e < 4; ++e) dot += pv[i][e] * dv[i][e];
    }
  }
  dot = warp_sum(dot);
  bf16* sr = dS + static_cast<size_t>(r) * s;
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int c = 4 * lane + 128 * i;
    if (c < E) {
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = scale * pv[i][e] * (dv[i][e] - dot);
      __nv_bfloat162 a = __floats2bfloat162_rn(o[0], o[1]);
      __nv_bfloat162 b = __floats2bfloat162_rn(o[2], o[3]);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&a);
      u.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(sr + c) = u;
    }
  }
}

// ------------------------------------------------------------------ MSE head
__global__ void __launch_bounds__(256) mse_kernel(const bf16* __restrict__ y, const bf16* __restrict__ r,
                                                  bf16* __restrict__ dy, float* __restrict__ part, int64_t n8,
                                                  float inv_n) {
  __shared__ float red[8];
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
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += part[i];
  *loss = s * half_inv_n;
}

// ------------------------------------------------------------------ AdamW
struct WdRanges {
  int64_t a0, a1, b0, b1, c0, c1, d0, d1;
};

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ p, float* __restrict__ m,
                                                    float* __restrict__ v, const float* __restrict__ g,
                                                    bf16* __restrict__ w, int64_t n4, int64_t per_layer, WdRanges wr,
                                                    float lr, float b1, float b2, float eps, float wd, float inv_bc1,
                                                    float inv_bc2, float grad_scale, int32_t* __restrict__ nonfinite) {
  bool bad = false;
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int64_t e0 = 4 * i;
    const int64_t o = e0 % per_layer;
    const bool decay = (o >= wr.a0 && o < wr.a1) || (o >= wr.b0 && o < wr.b1) || (o >= wr.c0 && o < wr.c1) ||
                       (o >= wr.d0 && o < wr.d1);
    const float wdl = decay ? wd : 0.f;
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float* pa = &pp.x;
    float* ma = &mm.x;
    float* va = &vv.x;
    const float* ga = &gg.x;
    float wo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      bad |= !isfinite(ga[e]);
      const float gr = grad_scale * ga[e];
      ma[e] = b1 * ma[e] + (1.f - b1) * gr;
      va[e] = b2 * va[e] + (1.f - b2) * gr * gr;
      const float mh = ma[e] * inv_bc1;
      const float vh = va[e] * inv_bc2;
      pa[e] = pa[e] - lr * wdl * pa[e] - lr * mh / (sqrtf(vh) + eps);
      wo[e] = pa[e];
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    __nv_bfloat162 x = __floats2bfloat162_rn(wo[0], wo[1]);
    __nv_bfloat162 y = __floats2bfloat162_rn(wo[2], wo[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&x);
    u.y = *reinterpret_cast<uint32_t*>(&y);
    reinterpret_cast<uint2*>(w)[i] = u;
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, bf16* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += static_cast<int64_t>(gridDim.x) * 256) {
    const float4 a = reinterpret_cast<const float4*>(src)[i];
    __nv_bfloat162 x = __floats2bfloat162_rn(a.x, a.y);
    __nv_bfloat162 y = __floats2bfloat162_rn(a.z, a.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&x);
    u.y = *reinterpret_cast<uint32_t*>(&y);
    reinterpret_cast<uint2*>(dst)[i] = u;
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

int grid_for(int64_t work, int per_block = 256) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : static_cast<int>(g);
}

}  // namespace

cudaError_t ln_fwd(const bf16* x, const bf16* gamma, const bf16* beta, bf16* y, float* mean, float* rstd, int T, int h,
                   float eps, cudaStream_t s) {
  if (h % 8 || h > 4096) return cudaErrorInvalidValue;
  const int nv = h / 8, blocks = (T + 3) / 4;
  if (nv <= 32) ln_fwd_kernel<1><<<blocks, 128, 0, s>>>(x, gamma, beta, y, mean, rstd, T, h, eps);
  else if (nv <= 64) ln_fwd_kernel<2><<<blocks, 128, 0, s>>>(x, gamma, beta, y, mean, rstd, T, h, eps);
  else if (nv <= 128) ln_fwd_kernel<4><<<blocks, 128, 0, s>>>(x, gamma, beta, y, mean, rstd, T, h, eps);
  else if (nv <= 256) ln_fwd_kernel<8><<<blocks, 128, 0, s>>>(x, gamma, beta, y, mean, rstd, T, h, eps);
  else ln_fwd_kernel<16><<<blocks, 128, 0, s>>>(x, gamma, beta, y, mean, rstd, T, h, eps);
  return cudaGetLastError();
}

cudaError_t ln_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* gamma,
                   const bf16* resid, bf16* dx, float* part_dgamma, float* part_dbeta, float* part_dxsum, int T, int h,
                   cudaStream_t s) {
  if (h % 8 || h > 4096) return cudaErrorInvalidValue;
  const int nv = h / 8, blocks = (T + 3) / 4;
  // column partials first: dx may alias x (the executor writes dx over the consumed stage input)
  dim3 grid((h + 255) / 256, kRedChunks);
  colred_kernel<1><<<grid, 256, 0, s>>>(dy, h, x, mean, rstd, T, h, part_dgamma, part_dbeta);
  if (dx) {
    if (nv <= 32) ln_bwd_rows_kernel<1><<<blocks, 128, 0, s>>>(dy, x, mean, rstd, gamma, resid, dx, T, h);
    else if (nv <= 64) ln_bwd_rows_kernel<2><<<blocks, 128, 0, s>>>(dy, x, mean, rstd, gamma, resid, dx, T, h);
    else if (nv <= 128) ln_bwd_rows_kernel<4><<<blocks, 128, 0, s>>>(dy, x, mean, rstd, gamma, resid, dx, T, h);
    else if (nv <= 256) ln_bwd_rows_kernel<8><<<blocks, 128, 0, s>>>(dy, x, mean, rstd, gamma, resid, dx, T, h);
    else ln_bwd_rows_kernel<16><<<blocks, 128, 0, s>>>(dy, x, mean, rstd, gamma, resid, dx, T, h);
  }
  if (part_dxsum && dx) colred_kernel<0><<<grid, 256, 0, s>>>(dx, h, nullptr, nullptr, nullptr, T, h, part_dxsum, nullptr);
  return cudaGetLastError();
}

cudaError_t colsum_partial(const bf16* a, int T, int N, int64_t ld, float* part, cudaStream_t s) {
  if (N % 8 || ld % 8) return cudaErrorInvalidValue;
  dim3 grid((N + 255) / 256, kRedChunks);
  colred_kernel<0><<<grid, 256, 0, s>>>(a, ld, nullptr, nullptr, nullptr, T, N, part, nullptr);
  return cudaGetLastError();
}

cudaError_t colsum_finalize(const float* part, int N, float* out, int accumulate, cudaStream_t s) {
  colsum_finalize_kernel<<<(N + 255) / 256, 256, 0, s>>>(part, N, out, accumulate);
  return cudaGetLastError();
}

cudaError_t softmax_fwd(const float* S, bf16* P, int z, int s, cudaStream_t st) {
  if (s % 4 || s > 2048) return cudaErrorInvalidValue;
  const int rows = z * s, blocks = (rows + 7) / 8, ni = (s + 127) / 128;
  if (ni <= 1) softmax_fwd_kernel<1><<<blocks, 256, 0, st>>>(S, P, rows, s);
  else if (ni <= 4) softmax_fwd_kernel<4><<<blocks, 256, 0, st>>>(S, P, rows, s);
  else if (ni <= 8) softmax_fwd_kernel<8><<<blocks, 256, 0, st>>>(S, P, rows, s);
  else softmax_fwd_kernel<16><<<blocks, 256, 0, st>>>(S, P, rows, s);
  return cudaGetLastError();
}

cudaError_t softmax_bwd(const float* dP, const bf16* P, bf16* dS, int z, int s, float scale, cudaStream_t st) {
  if (s % 4 || s > 2048) return cudaErrorInvalidValue;
  const int rows = z * s, blocks = (rows + 7) / 8, ni = (s + 127) / 128;
  if (ni <= 1) softmax_bwd_kernel<1><<<blocks, 256, 0, st>>>(dP, P, dS, rows, s, scale);
  else if (ni <= 4) softmax_bwd_kernel<4><<<blocks, 256, 0, st>>>(dP, P, dS, rows, s, scale);
  else if (ni <= 8) softmax_bwd_kernel<8><<<blocks, 256, 0, st>>>(dP, P, dS, rows, s, scale);
  else softmax_bwd_kernel<16><<<blocks, 256, 0, st>>>(dP, P, dS, rows, s, scale);
  return cudaGetLastError();
}

cudaError_t mse_loss(const bf16* y, const bf16* r, bf16* dy, float* part, int nparts, float* loss, int64_t n,
                     cudaStream_t s) {
  if (n % 8) return cudaErrorInvalidValue;
  mse_kernel<<<nparts, 256, 0, s>>>(y, r, dy, part, n / 8, 1.0f / static_cast<float>(n));
  mse_finalize_kernel<<<1, 32, 0, s>>>(part, nparts, loss, 0.5f / static_cast<float>(n));
  return cudaGetLastError();
}

cudaError_t adamw(float* p, float* m, float* v, const float* g, bf16* w, int64_t n, int64_t per_layer, int h, int f,
                  float lr, float b1, float b2, float eps, float wd, float bc1, float bc2, float grad_scale,
                  int32_t* nonfinite, cudaStream_t s) {
  if (n % 4 || per_layer % 4) return cudaErrorInvalidValue;
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
  adamw_kernel<<<grid_for(n / 4), 256, 0, s>>>(p, m, v, g, w, n / 4, per_layer, wr, lr, b1, b2, eps, wd, 1.0f / bc1,
                                               1.0f / bc2, grad_scale, nonfinite);
  return cudaGetLastError();
}

cudaError_t f32_to_bf16(const float* src, bf16* dst, int64_t n, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  f32_to_bf16_kernel<<<grid_for(n / 4), 256, 0, s>>>(src, dst, n / 4);
  return cudaGetLastError();
}

cudaError_t synth_normal(bf16* out, int64_t n, uint64_t seed, uint64_t k, uint64_t j, cudaStream_t s) {
  uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  synth_normal_kernel<<<grid_for((n + 3) / 4), 256, 0, s>>>(out, n, key, static_cast<uint32_t>(k),
                                                            static_cast<uint32_t>(j));
  return cudaGetLastError();
}

}  // namespace slip
