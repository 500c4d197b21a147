// attention.cu — fused causal attention for sm_100a (tcgen05 + TMEM + TMA).
//
// Tiles are 128 queries x 128 keys.  Every operand tile is a "[128 rows][d]" slab of the
// QKV / dO activations loaded by TMA with 128-byte swizzle; the same bytes serve as a
// K-major operand (contraction over d: S = Q K^T, dP = dO V^T) and as an MN-major operand
// (contraction over rows: O += P V, dQ += dS K, dV += P^T dO, dK += dS^T Q), so no
// transposes are ever materialised.  Warp roles: warp 0 TMA, warp 1 MMA issuer, warp 2
// TMEM allocation, warps 4-7 "row" warps (thread r owns TMEM lane r = tile row r): they
// read S / dP from TMEM, form P or dS in bf16 and write it, swizzled, to shared memory
// as the A operand of the next MMA.  S and dP never reach HBM; the P stash of the
// materialised path is replaced by a per-row log-sum-exp.
#include <cmath>
#include <cstring>
#include <string>

#include "attention.cuh"
#include "gemm.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace slip {
namespace {

constexpr int TILE = 128;
constexpr int ATOM = 16384;  // 128 rows x 128 B (64 bf16 of the contiguous dimension)
constexpr int CW0 = 4;       // first row warp
constexpr int NRW = 16;      // row warps: 4 lane quarters x 4 column groups of 32
constexpr int NT = 32 * (CW0 + NRW);

__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

enum Mode : int { M_STATS = 0, M_FWD = 1, M_DQ = 2 };

template <int D>
struct AC {
  static constexpr int NA = (D + 63) / 64;  // atoms along d
  static constexpr int TB = NA * ATOM;      // bytes of one [128][D] tile
  static constexpr int KS = D / 16;         // UMMA_K steps over d
  static constexpr int OC = (D + 31) / 32;  // 32-column chunks of a D-wide accumulator
  static constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(128, 128, false, false);
  static constexpr uint32_t IDESC_O = ptx::idesc_bf16_f32(128, D, false, true);
};

struct KArgs {
  int s, heads, ntiles;
  float sl2;    // log2(e) / sqrt(d)
  float scale;  // 1 / sqrt(d)
  float* lse;
  const float* dsum;
  __nv_bfloat16* out;
  int64_t ldo;   // row stride of out
  int64_t col0;  // column offset of the first output block (FWD: O; DQ: dQ; DKDV: dK)
  int64_t col1;  // DKDV: column offset of dV
  int d;
};

// tile [128 rows][D] as a K-major operand (contraction over d), UMMA_K step kk
__device__ __forceinline__ uint64_t dk(uint32_t base, int kk) {
  return ptx::smem_desc_sw128(base + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
}
// tile [128 rows][D] as an MN-major operand (contraction over the 128 rows), step kk
__device__ __forceinline__ uint64_t dm(uint32_t base, int kk) {
  return ptx::smem_desc_sw128(base + kk * 2048, ATOM, 1024);
}
// byte offset of the 16-byte chunk `ch` (8 columns) of row r in a [128][128] K-major X tile
__device__ __forceinline__ uint32_t xoff(int r, int ch) {
  return (ch >> 3) * ATOM + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
// write 32 fp32 accumulator columns [c0, c0+32) of one output row as bf16 (cols < D)
template <int D>
__device__ __forceinline__ void store_row_chunk(__nv_bfloat16* row, int c0, const uint32_t (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + q * 8;
    if (c < D) {
      uint4 u;
      u.x = pack2(__uint_as_float(v[q * 8 + 0]), __uint_as_float(v[q * 8 + 1]));
      u.y = pack2(__uint_as_float(v[q * 8 + 2]), __uint_as_float(v[q * 8 + 3]));
      u.z = pack2(__uint_as_float(v[q * 8 + 4]), __uint_as_float(v[q * 8 + 5]));
      u.w = pack2(__uint_as_float(v[q * 8 + 6]), __uint_as_float(v[q * 8 + 7]));
      *reinterpret_cast<uint4*>(row + c) = u;
    }
  }
}

// ====================================================================== row kernel
// One CTA per (q-tile i, batch*head z).  STATS: lse; FWD: O = sum_j P_ij V_j;
// DQ: dQ = sum_j dS_ij K_j.  j runs over the causal k-tiles 0..i.
template <int D, int MODE>
__global__ void __launch_bounds__(NT, 1)
    attn_row_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const KArgs a) {
  using C = AC<D>;
  constexpr bool kV = MODE != M_STATS;     // stages carry V as well as K
  constexpr bool kX = MODE != M_STATS;     // an X tile (P or dS) feeds a second MMA
  constexpr int STAGE = kV ? 2 * C::TB : C::TB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = sm;
  uint8_t* dOs = Qs + C::TB;
  uint8_t* stg = dOs + (MODE == M_DQ ? C::TB : 0);
  uint8_t* Xs = stg + 2 * STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Xs + (kX ? 2 * ATOM : 0));
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;   // [2]
  uint64_t* kv_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;
  uint64_t* s_empty = bar + 6;
  uint64_t* x_full = bar + 7;
  uint64_t* x_empty = bar + 8;
  uint64_t* acc_full = bar + 9;
  uint32_t* tholder = reinterpret_cast<uint32_t*>(bar + 10);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.x, hn = z % a.heads, bi = z / a.heads;
  const int i = a.ntiles - 1 - static_cast<int>(blockIdx.y);  // longest rows first (LPT order)
  const int nj = i + 1;
  const int q0 = i * TILE;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&kv_full[t], 1);
      ptx::mbar_init(&kv_empty[t], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_empty, NRW);
    ptx::mbar_init(x_full, NRW);
    ptx::mbar_init(x_empty, 1);
    ptx::mbar_init(acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tholder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tholder;
  const uint32_t tS = tmem, tP = tmem + 128, tA = tmem + 256;
  ptx::grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel
  // STATS: per column-group running (max, sum) of each row, merged at the end
  __shared__ float2 stats[MODE == M_STATS ? 4 : 1][MODE == M_STATS ? TILE : 1];

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      ptx::mbar_arrive_expect_tx(q_full, (MODE == M_DQ ? 2 : 1) * C::TB);
      for (int t = 0; t < C::NA; ++t) {
        ptx::tma_load_4d(&tmQ, Qs + t * ATOM, q_full, t * 64, q0, hn, bi);
        if (MODE == M_DQ) ptx::tma_load_4d(&tmdO, dOs + t * ATOM, q_full, t * 64, q0, hn, bi);
      }
      for (int j = 0; j < nj; ++j) {
        const int st = j & 1;
        ptx::mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* ks = stg + st * STAGE;
        ptx::mbar_arrive_expect_tx(&kv_full[st], STAGE);
        for (int t = 0; t < C::NA; ++t) {
          ptx::tma_load_4d(&tmK, ks + t * ATOM, &kv_full[st], t * 64, j * TILE, hn, bi);
          if (kV) ptx::tma_load_4d(&tmV, ks + C::TB + t * ATOM, &kv_full[st], t * 64, j * TILE, hn, bi);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      ptx::mbar_wait(q_full, 0);
      ptx::tc_fence_after();
      const uint32_t qb = ptx::smem_u32(Qs), ob = ptx::smem_u32(dOs), xb = ptx::smem_u32(Xs);
      // software pipeline: S_j is issued before the second product of tile j-1
      for (int j = 0; j <= nj; ++j) {
        if (j < nj) {
          const int st = j & 1;
          ptx::mbar_wait(&kv_full[st], (j >> 1) & 1);
          ptx::mbar_wait(s_empty, (j & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t kb = ptx::smem_u32(stg + st * STAGE);
#pragma unroll
          for (int kk = 0; kk < C::KS; ++kk) ptx::tc_mma_f16(tS, dk(qb, kk), dk(kb, kk), C::IDESC_S, kk > 0);
          if (MODE == M_DQ) {
#pragma unroll
            for (int kk = 0; kk < C::KS; ++kk)
              ptx::tc_mma_f16(tP, dk(ob, kk), dk(kb + C::TB, kk), C::IDESC_S, kk > 0);
          }
          ptx::tc_commit(s_full);
          if (!kX) ptx::tc_commit(&kv_empty[st]);
        }
        if (kX && j >= 1) {
          const int jj = j - 1, st = jj & 1;
          ptx::mbar_wait(x_full, jj & 1);
          ptx::tc_fence_after();
          const uint32_t sb = ptx::smem_u32(stg + st * STAGE);
          const uint32_t bb = MODE == M_FWD ? sb + C::TB : sb;  // FWD: O += P V;  DQ: dQ += dS K
#pragma unroll
          for (int kk = 0; kk < TILE / 16; ++kk)
            ptx::tc_mma_f16(tA, dk(xb, kk), dm(bb, kk), C::IDESC_O, (jj > 0 || kk > 0) ? 1u : 0u);
          ptx::tc_commit(x_empty);
          ptx::tc_commit(&kv_empty[st]);
        }
      }
      if (kX) ptx::tc_commit(acc_full);
    }
  } else if (warp >= CW0) {  // ---------------------------------------- row warps
    // warp w: TMEM lane quarter lq (= warp % 4, rows 32 lq .. 32 lq + 31) and column
    // group cg (columns 32 cg .. 32 cg + 31 of every 128-wide tile)
    const int w = warp - CW0;
    const int lq = w & 3, cg = w >> 2;
    const int r = lq * 32 + lane;
    const int q = q0 + r;
    const size_t zs = static_cast<size_t>(z) * a.s;
    const float lrow = (MODE != M_STATS && q < a.s) ? a.lse[zs + q] : 0.f;
    const float drow = (MODE == M_DQ && q < a.s) ? a.dsum[zs + q] : 0.f;
    const uint32_t xb = ptx::smem_u32(Xs);
    const uint32_t toff = (static_cast<uint32_t>(lq * 32) << 16) + cg * 32;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nj; ++j) {
      ptx::mbar_wait(s_full, j & 1);
      ptx::tc_fence_after();
      uint32_t sv[32], pv[32];
      ptx::tmem_ld_32x32b_x32(tS + toff, sv);
      if (MODE == M_DQ) ptx::tmem_ld_32x32b_x32(tP + toff, pv);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(s_empty);  // S / dP may be overwritten by the next tile's MMA
      const int key0 = j * TILE + cg * 32;
      const bool diag = key0 + 31 > q0;  // only the diagonal tile needs the causal mask
      if (MODE == M_STATS) {
        float cm = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (!diag || key0 + e <= q) cm = fmaxf(cm, __uint_as_float(sv[e]) * a.sl2);
        const float mn = fmaxf(m, cm);
        if (mn != -INFINITY) {
          float acc = 0.f;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            acc += (!diag || key0 + e <= q) ? ex2(__uint_as_float(sv[e]) * a.sl2 - mn) : 0.f;
          l = (m == -INFINITY ? 0.f : l * ex2(m - mn)) + acc;
          m = mn;
        }
      } else {
        if (kX) ptx::mbar_wait(x_empty, (j & 1) ^ 1);
        float x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float p = (!diag || key0 + e <= q) ? ex2(__uint_as_float(sv[e]) * a.sl2 - lrow) : 0.f;
          x[e] = MODE == M_FWD ? p : p * (__uint_as_float(pv[e]) - drow) * a.scale;
        }
#pragma unroll
        for (int g = 0; g < 4; ++g)
          st_shared_v4(xb + xoff(r, cg * 4 + g), pack2(x[g * 8 + 0], x[g * 8 + 1]), pack2(x[g * 8 + 2], x[g * 8 + 3]),
                       pack2(x[g * 8 + 4], x[g * 8 + 5]), pack2(x[g * 8 + 6], x[g * 8 + 7]));
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(x_full);
      }
    }
    if (MODE == M_STATS) {
      stats[cg][r] = make_float2(m, l);
      ptx::named_bar_sync(2, 32 * NRW);
      if (cg == 0) {
        float M = -INFINITY;
        for (int g = 0; g < 4; ++g) M = fmaxf(M, stats[g][r].x);
        float L = 0.f;
        for (int g = 0; g < 4; ++g)
          if (stats[g][r].x != -INFINITY) L += stats[g][r].y * ex2(stats[g][r].x - M);
        if (q < a.s) a.lse[zs + q] = M + log2f(L);
      }
    } else {
      ptx::mbar_wait(acc_full, 0);
      ptx::tc_fence_after();
      __nv_bfloat16* orow = a.out + (static_cast<int64_t>(bi) * a.s + q) * a.ldo + a.col0 + static_cast<int64_t>(hn) * a.d;
      if (cg < C::OC) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tA + (static_cast<uint32_t>(lq * 32) << 16) + cg * 32, v);
        ptx::tmem_ld_wait();
        if (q < a.s) store_row_chunk<D>(orow, cg * 32, v);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ====================================================================== forward kernel
// Single pass, online softmax.  One CTA per (q-tile i, z), longest rows first.  TMEM:
// S[0] | S[1] | O (128 columns each): S of k-tile j+1 is computed while the softmax warps
// work on k-tile j, so the tensor core and the softmax overlap.  Warp 0 TMA (K ring of 3,
// V ring of 2, loaded in consumption order), warp 1 MMA, warp 2 TMEM allocator, warps
// 4-11 softmax: warp w owns TMEM lane quarter w % 4 (32 rows) and column half g =
// (w - 4) / 4 (64 of the 128 keys of a tile).  Per k-tile: S half -> registers, row max
// exchanged with the partner warp through shared memory, O and l rescaled only when the
// running max grows by more than kTau (log2 units; P stays <= 2^kTau, far inside bf16 /
// fp32 range, and the result is the exact softmax either way), P = exp2(S log2e/sqrt(d)
// - m) written as bf16 pairs over the S columns (the MMA reads P from TMEM for O += P V).
// Output O / l in bf16 and lse = m + log2 l (log2 domain) for the backward pass.
constexpr int FWD_NT = 32 * 20;
constexpr float kTau = 8.0f;

// Optional cycle-stamp probe of one CTA (tools/attn_probe.cu builds with SLIP_ATTN_PROBE).
#ifdef SLIP_ATTN_PROBE
__device__ long long g_probe[4096];
#define PROBE(idx)                                                                  \
  do {                                                                              \
    if (blockIdx.x == 0 && blockIdx.y == SLIP_ATTN_PROBE) g_probe[idx] = clock64(); \
  } while (0)
#else
#define PROBE(idx) \
  do {             \
  } while (0)
#endif

template <int D>
__global__ void __launch_bounds__(FWD_NT, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const KArgs a) {
  using C = AC<D>;
  constexpr int KST = 3, VST = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = sm;
  uint8_t* Ks = Qs + C::TB;         // [KST][TB]
  uint8_t* Vs = Ks + KST * C::TB;   // [VST][TB]
  float* red = reinterpret_cast<float*>(Vs + VST * C::TB);  // [4][128] partial row max / sum
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 4 * TILE);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;                // [KST]
  uint64_t* k_empty = k_full + KST;          // [KST]
  uint64_t* v_full = k_empty + KST;          // [VST]
  uint64_t* v_empty = v_full + VST;          // [VST]
  uint64_t* s_full = v_empty + VST;          // [2] per S buffer
  uint64_t* p_full = s_full + 2;             // P of the current k-tile written (8 warps)
  uint64_t* o_done = p_full + 1;             // PV of a k-tile complete
  uint32_t* tholder = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.x, hn = z % a.heads, bi = z / a.heads;
  const int i = a.ntiles - 1 - static_cast<int>(blockIdx.y);  // longest rows first (LPT order)
  const int nj = i + 1;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int t = 0; t < KST; ++t) {
      ptx::mbar_init(&k_full[t], 1);
      ptx::mbar_init(&k_empty[t], 1);
    }
    for (int t = 0; t < VST; ++t) {
      ptx::mbar_init(&v_full[t], 1);
      ptx::mbar_init(&v_empty[t], 1);
    }
    ptx::mbar_init(&s_full[0], 1);
    ptx::mbar_init(&s_full[1], 1);
    ptx::mbar_init(p_full, 16);
    ptx::mbar_init(o_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tholder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tholder;
  ptx::grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel
  if (threadIdx.x == 0) PROBE(0);

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      ptx::mbar_arrive_expect_tx(q_full, C::TB);
      for (int t = 0; t < C::NA; ++t) ptx::tma_load_4d(&tmQ, Qs + t * ATOM, q_full, t * 64, i * TILE, hn, bi);
      auto load_k = [&](int j) {
        const int st = j % KST;
        ptx::mbar_wait(&k_empty[st], ((j / KST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&k_full[st], C::TB);
        for (int t = 0; t < C::NA; ++t)
          ptx::tma_load_4d(&tmK, Ks + st * C::TB + t * ATOM, &k_full[st], t * 64, j * TILE, hn, bi);
      };
      auto load_v = [&](int j) {
        const int st = j % VST;
        ptx::mbar_wait(&v_empty[st], ((j / VST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&v_full[st], C::TB);
        for (int t = 0; t < C::NA; ++t)
          ptx::tma_load_4d(&tmV, Vs + st * C::TB + t * ATOM, &v_full[st], t * 64, j * TILE, hn, bi);
      };
      // consumption order of the MMA warp: K0 K1 V0 K2 V1 K3 V2 ...
      load_k(0);
      if (nj > 1) load_k(1);
      for (int j = 0; j < nj; ++j) {
        load_v(j);
        if (j + 2 < nj) load_k(j + 2);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      ptx::mbar_wait(q_full, 0);
      const uint32_t qb = ptx::smem_u32(Qs), kb0 = ptx::smem_u32(Ks), vb0 = ptx::smem_u32(Vs);
      auto mma_s = [&](int j) {  // S[j % 2] = Q K_j^T
        const int st = j % KST;
        ptx::mbar_wait(&k_full[st], (j / KST) & 1);
        ptx::tc_fence_after();
        const uint32_t kb = kb0 + st * C::TB;
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk)
          ptx::tc_mma_f16(tmem + (j & 1) * 128, dk(qb, kk), dk(kb, kk), C::IDESC_S, kk > 0);
        ptx::tc_commit(&s_full[j & 1]);
        ptx::tc_commit(&k_empty[st]);
      };
      mma_s(0);
      if (nj > 1) mma_s(1);
      for (int j = 0; j < nj; ++j) {
        const int st = j % VST;
        ptx::mbar_wait(p_full, j & 1);
        ptx::mbar_wait(&v_full[st], (j / VST) & 1);
        PROBE(100 + j);
        ptx::tc_fence_after();
        const uint32_t vb = vb0 + st * C::TB;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)  // O += P V_j, P (bf16 pairs) from TMEM
          ptx::tc_mma_f16_ts(tmem + 256, tmem + (j & 1) * 128 + kk * 8, dm(vb, kk), C::IDESC_O,
                             (j > 0 || kk > 0) ? 1u : 0u);
        ptx::tc_commit(o_done);
        ptx::tc_commit(&v_empty[st]);
        if (j + 2 < nj) mma_s(j + 2);  // into the S buffer PV_j has just consumed (in order)
      }
    }
  } else if (warp >= 4) {  // ------------------------------------------ softmax warps
    const int lq = warp & 3, g = (warp - 4) >> 2;  // lane quarter, column group (32 keys)
    const int r = lq * 32 + lane;
    const int q = i * TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(lq * 32) << 16;
    const uint32_t tO = tmem + 256 + lane_off;
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j < nj; ++j) {
      const uint32_t tS = tmem + (j & 1) * 128 + lane_off;
      ptx::mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      if (lq == 0 && lane == 0 && g < 2) PROBE(400 + 300 * g + j);
      ptx::tc_fence_after();
      const bool diag = j == i;
      const int kb = j * TILE + g * 32;  // first key of this warp's column group
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tS + g * 32, v);
      ptx::tmem_ld_wait();
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      if (!diag) {
#pragma unroll
        for (int e = 0; e < 32; e += 2)
          mx[(e >> 1) & 3] = max3(mx[(e >> 1) & 3], __uint_as_float(v[e]), __uint_as_float(v[e + 1]));
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (kb + e <= q) mx[e & 3] = fmaxf(mx[e & 3], __uint_as_float(v[e]));
      }
      // row max over the 4 column groups (the 4 warps of this lane quarter)
      red[g * TILE + r] = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      ptx::named_bar_sync(1 + lq, 128);
      const float mt = fmaxf(fmaxf(red[r], red[TILE + r]), fmaxf(red[2 * TILE + r], red[3 * TILE + r])) * a.sl2;
      ptx::named_bar_sync(1 + lq, 128);  // all read before the next tile overwrites red
      if (lq == 0 && lane == 0 && g < 2) PROBE(500 + 300 * g + j);
      if (__any_sync(0xffffffffu, mt > m_run + kTau)) {
        const float mn = fmaxf(m_run, mt);
        const float alpha = m_run == -INFINITY ? 0.f : ex2(m_run - mn);
        if (j > 0 && g < C::OC) {  // O holds PV(0 .. j-1): wait for the last one, rescale my chunk
          ptx::mbar_wait(o_done, (j - 1) & 1);
          ptx::tc_fence_after();
          uint32_t o[32];
          ptx::tmem_ld_32x32b_x32(tO + g * 32, o);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          ptx::tmem_st_32x32b_x32(tO + g * 32, o);
          ptx::tmem_st_wait();
        }
        l *= alpha;
        m_run = mn;
      }
      const float nm = -m_run;
      float ls[4] = {0.f, 0.f, 0.f, 0.f};
      uint32_t pk[16];
      if (!diag) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float p0 = ex2(fmaf(__uint_as_float(v[2 * e]), a.sl2, nm));
          const float p1 = ex2(fmaf(__uint_as_float(v[2 * e + 1]), a.sl2, nm));
          ls[(2 * e) & 3] += p0;
          ls[(2 * e + 1) & 3] += p1;
          pk[e] = pack2(p0, p1);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int k0 = kb + 2 * e;
          const float p0 = k0 <= q ? ex2(fmaf(__uint_as_float(v[2 * e]), a.sl2, nm)) : 0.f;
          const float p1 = k0 + 1 <= q ? ex2(fmaf(__uint_as_float(v[2 * e + 1]), a.sl2, nm)) : 0.f;
          ls[(2 * e) & 3] += p0;
          ls[(2 * e + 1) & 3] += p1;
          pk[e] = pack2(p0, p1);
        }
      }
      l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      // P of keys [32g, 32g+32) -> bf16 pairs in TMEM columns [16g, 16g+16) of this S buffer
      // (every S value of the tile is already in registers: the exchange above ordered it)
      ptx::tmem_st_32x32b_x16(tS + g * 16, pk);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(p_full);
      if (lq == 0 && lane == 0 && g < 2) PROBE(600 + 300 * g + j);
    }
    // total l over the 4 column groups, then O / l and lse
    red[g * TILE + r] = l;
    ptx::named_bar_sync(1 + lq, 128);
    const float lt = (red[r] + red[TILE + r]) + (red[2 * TILE + r] + red[3 * TILE + r]);
    ptx::mbar_wait(o_done, (nj - 1) & 1);
    ptx::tc_fence_after();
    if (g == 0 && q < a.s) a.lse[static_cast<size_t>(z) * a.s + q] = m_run + log2f(lt);
    if (g < C::OC) {
      const float inv = 1.0f / lt;
      __nv_bfloat16* orow =
          a.out + (static_cast<int64_t>(bi) * a.s + q) * a.ldo + a.col0 + static_cast<int64_t>(hn) * a.d;
      uint32_t o[32];
      ptx::tmem_ld_32x32b_x32(tO + g * 32, o);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * inv);
      if (q < a.s) store_row_chunk<D>(orow, g * 32, o);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ====================================================================== column kernel
// One CTA per (k-tile j, z).  Walks q-tiles i = j .. ntiles-1:
//   S^T = K_j Q_i^T, dP^T = V_j dO_i^T (TMEM), P^T = exp(S^T - lse_q), dS^T = P^T (dP^T - D_q)/sqrt(d)
//   dV += P^T dO_i, dK += dS^T Q_i (TMEM accumulators).
template <int D>
__global__ void __launch_bounds__(NT, 1)
    attn_col_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const KArgs a) {
  using C = AC<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Ks = sm;
  uint8_t* Vs = Ks + C::TB;
  uint8_t* QD = Vs + C::TB;       // 2 stages of {Q_i, dO_i}
  uint8_t* X = QD + 4 * C::TB;    // P^T, then (after dV consumed it) dS^T
  float* lse_s = reinterpret_cast<float*>(X + 2 * ATOM);
  float* d_s = lse_s + TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(d_s + TILE);
  uint64_t* kv_full = bar;
  uint64_t* qd_full = bar + 1;   // [2]
  uint64_t* qd_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;
  uint64_t* s_empty = bar + 6;
  uint64_t* xp_full = bar + 7;   // P^T written
  uint64_t* xs_full = bar + 8;   // dS^T written
  uint64_t* xp_free = bar + 9;   // dV MMA has read P^T
  uint64_t* x_free = bar + 10;   // dK MMA has read dS^T
  uint64_t* acc_full = bar + 11;
  uint32_t* tholder = reinterpret_cast<uint32_t*>(bar + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.x, hn = z % a.heads, bi = z / a.heads;
  const int j = blockIdx.y;  // k-tile; longest walks (small j) first (LPT order)
  const int k0 = j * TILE;
  const int ni = a.ntiles - j;

  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&qd_full[t], 1);
      ptx::mbar_init(&qd_empty[t], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_empty, NRW);
    ptx::mbar_init(xp_full, NRW);
    ptx::mbar_init(xs_full, NRW);
    ptx::mbar_init(xp_free, 1);
    ptx::mbar_init(x_free, 1);
    ptx::mbar_init(acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tholder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tholder;
  const uint32_t tS = tmem, tP = tmem + 128, tV = tmem + 256, tK = tmem + 384;
  ptx::grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      ptx::mbar_arrive_expect_tx(kv_full, 2 * C::TB);
      for (int t = 0; t < C::NA; ++t) {
        ptx::tma_load_4d(&tmK, Ks + t * ATOM, kv_full, t * 64, k0, hn, bi);
        ptx::tma_load_4d(&tmV, Vs + t * ATOM, kv_full, t * 64, k0, hn, bi);
      }
      for (int n = 0; n < ni; ++n) {
        const int q0 = (j + n) * TILE, st = n & 1;
        uint8_t* qs = QD + st * 2 * C::TB;
        ptx::mbar_wait(&qd_empty[st], ((n >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&qd_full[st], 2 * C::TB);
        for (int t = 0; t < C::NA; ++t) {
          ptx::tma_load_4d(&tmQ, qs + t * ATOM, &qd_full[st], t * 64, q0, hn, bi);
          ptx::tma_load_4d(&tmdO, qs + C::TB + t * ATOM, &qd_full[st], t * 64, q0, hn, bi);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      const uint32_t kb = ptx::smem_u32(Ks), vb = ptx::smem_u32(Vs), qdb = ptx::smem_u32(QD),
                     xb = ptx::smem_u32(X);
      // S^T and dP^T of q-tile n (into TMEM once the row warps have read the previous ones)
      auto issue_s = [&](int n) {
        const int st = n & 1;
        const uint32_t qb = qdb + st * 2 * C::TB, ob = qb + C::TB;
        ptx::mbar_wait(&qd_full[st], (n >> 1) & 1);
        ptx::mbar_wait(s_empty, (n & 1) ^ 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk) ptx::tc_mma_f16(tS, dk(kb, kk), dk(qb, kk), C::IDESC_S, kk > 0);
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk) ptx::tc_mma_f16(tP, dk(vb, kk), dk(ob, kk), C::IDESC_S, kk > 0);
        ptx::tc_commit(s_full);
      };
      ptx::mbar_wait(kv_full, 0);
      issue_s(0);
      for (int n = 0; n < ni; ++n) {
        const int st = n & 1;
        const uint32_t qb = qdb + st * 2 * C::TB, ob = qb + C::TB;
        ptx::mbar_wait(xp_full, n & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          ptx::tc_mma_f16(tV, dk(xb, kk), dm(ob, kk), C::IDESC_O, (n > 0 || kk > 0) ? 1u : 0u);
        ptx::tc_commit(xp_free);
        if (n + 1 < ni) issue_s(n + 1);  // overlaps the row warps' dS^T work of tile n
        ptx::mbar_wait(xs_full, n & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          ptx::tc_mma_f16(tK, dk(xb, kk), dm(qb, kk), C::IDESC_O, (n > 0 || kk > 0) ? 1u : 0u);
        ptx::tc_commit(x_free);
        ptx::tc_commit(&qd_empty[st]);
      }
      ptx::tc_commit(acc_full);
    }
  } else if (warp >= CW0) {  // ---------------------------------------- row warps (rows = keys)
    const int w = warp - CW0;
    const int lq = w & 3, cg = w >> 2;  // lane quarter (rows) and column group (q columns)
    const int r = lq * 32 + lane;
    const int key = k0 + r;
    const size_t zs = static_cast<size_t>(z) * a.s;
    const uint32_t xb = ptx::smem_u32(X);
    const uint32_t lane_off = static_cast<uint32_t>(lq * 32) << 16;
    const uint32_t toff = lane_off + cg * 32;
    // lse / D of the q-tile rows: warps 0-3 load them one tile ahead into registers (the
    // global latency overlaps the previous tile) and publish them through shared memory
    float lse_n = INFINITY, d_n = 0.f;
    if (w < 4 && j * TILE + r < a.s) {
      lse_n = a.lse[zs + j * TILE + r];
      d_n = a.dsum[zs + j * TILE + r];
    }
    for (int n = 0; n < ni; ++n) {
      const int q0 = (j + n) * TILE;
      ptx::named_bar_sync(1, 32 * NRW);  // previous q-tile's readers of lse_s / d_s are done
      if (w < 4) {
        lse_s[r] = lse_n;
        d_s[r] = d_n;
        const int qn = q0 + TILE + r;
        lse_n = (n + 1 < ni && qn < a.s) ? a.lse[zs + qn] : INFINITY;
        d_n = (n + 1 < ni && qn < a.s) ? a.dsum[zs + qn] : 0.f;
      }
      ptx::named_bar_sync(1, 32 * NRW);
      ptx::mbar_wait(s_full, n & 1);
      ptx::tc_fence_after();
      uint32_t sv[32], pv[32];
      ptx::tmem_ld_32x32b_x32(tS + toff, sv);
      ptx::tmem_ld_32x32b_x32(tP + toff, pv);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(s_empty);
      const bool diag = n == 0;  // key tile == query tile: causal mask inside the tile
      float pt[32], st[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int qi = cg * 32 + e;
        const float p = (!diag || key <= q0 + qi) ? ex2(__uint_as_float(sv[e]) * a.sl2 - lse_s[qi]) : 0.f;
        pt[e] = p;
        st[e] = p * (__uint_as_float(pv[e]) - d_s[qi]) * a.scale;
      }
      ptx::mbar_wait(x_free, (n & 1) ^ 1);  // the previous tile's dK MMA has read X
#pragma unroll
      for (int g = 0; g < 4; ++g)
        st_shared_v4(xb + xoff(r, cg * 4 + g), pack2(pt[g * 8 + 0], pt[g * 8 + 1]), pack2(pt[g * 8 + 2], pt[g * 8 + 3]),
                     pack2(pt[g * 8 + 4], pt[g * 8 + 5]), pack2(pt[g * 8 + 6], pt[g * 8 + 7]));
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(xp_full);
      ptx::mbar_wait(xp_free, n & 1);  // dV MMA has read P^T
#pragma unroll
      for (int g = 0; g < 4; ++g)
        st_shared_v4(xb + xoff(r, cg * 4 + g), pack2(st[g * 8 + 0], st[g * 8 + 1]), pack2(st[g * 8 + 2], st[g * 8 + 3]),
                     pack2(st[g * 8 + 4], st[g * 8 + 5]), pack2(st[g * 8 + 6], st[g * 8 + 7]));
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(xs_full);
    }
    ptx::mbar_wait(acc_full, 0);
    ptx::tc_fence_after();
    const int64_t rowoff = (static_cast<int64_t>(bi) * a.s + key) * a.ldo + static_cast<int64_t>(hn) * a.d;
    if (cg < C::OC) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tK + lane_off + cg * 32, v);
      ptx::tmem_ld_wait();
      if (key < a.s) store_row_chunk<D>(a.out + rowoff + a.col0, cg * 32, v);
      ptx::tmem_ld_32x32b_x32(tV + lane_off + cg * 32, v);
      ptx::tmem_ld_wait();
      if (key < a.s) store_row_chunk<D>(a.out + rowoff + a.col1, cg * 32, v);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// D[z, q] = sum_d dO[q, hn*d + dd] * O[q, hn*d + dd]; one warp per (token, head)
__global__ void __launch_bounds__(256) attn_dsum_kernel(const __nv_bfloat16* __restrict__ o,
                                                        const __nv_bfloat16* __restrict__ dO, float* __restrict__ dsum,
                                                        int s, int heads, int d, int64_t h, int rows) {
  ptx::grid_dep_wait();
  const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= rows * heads) return;
  const int t = gw / heads, hn = gw % heads;
  const int bi = t / s, qq = t % s;
  const __nv_bfloat16* op = o + static_cast<int64_t>(t) * h + static_cast<int64_t>(hn) * d;
  const __nv_bfloat16* gp = dO + static_cast<int64_t>(t) * h + static_cast<int64_t>(hn) * d;
  float acc = 0.f;
  for (int e = lane * 2; e < d; e += 64) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(op + e));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(gp + e));
    acc += a.x * b.x + a.y * b.y;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) dsum[(static_cast<int64_t>(bi) * heads + hn) * s + qq] = acc;
}

thread_local std::string g_amsg;

template <int D>
constexpr int row_smem(int mode) {
  return AC<D>::TB + (mode == M_DQ ? AC<D>::TB : 0) + 2 * (mode == M_STATS ? AC<D>::TB : 2 * AC<D>::TB) +
         (mode == M_STATS ? 0 : 2 * ATOM) + 1024 + 1024;
}
template <int D>
constexpr int fwd_smem() {
  return 6 * AC<D>::TB + 4 * TILE * 4 + 1024 + 1024;
}
template <int D>
constexpr int col_smem() {
  return 6 * AC<D>::TB + 2 * ATOM + 2 * TILE * 4 + 1024 + 1024;
}

struct Maps {
  CUtensorMap q, k, v, dO;
};

bool make_maps(const AttnArgs& a, Maps& m, bool with_do) {
  const uint64_t d = a.d, s = a.s, H = a.heads, B = a.batch;
  const int64_t L = a.qkv_ld;
  bool ok = encode_bf16_4d(&m.q, a.qkv, d, s, H, B, L, d, s * L, 64, 128) &&
            encode_bf16_4d(&m.k, a.qkv + a.h, d, s, H, B, L, d, s * L, 64, 128) &&
            encode_bf16_4d(&m.v, a.qkv + 2 * a.h, d, s, H, B, L, d, s * L, 64, 128);
  if (with_do) ok = ok && encode_bf16_4d(&m.dO, a.dO, d, s, H, B, a.h, d, s * a.h, 64, 128);
  else m.dO = m.q;
  if (!ok) g_amsg = std::string("attention tensor map: ") + gemm_last_message();
  return ok;
}

template <int D>
cudaError_t forward_d(const AttnArgs& a, cudaStream_t st) {
  Maps mp;
  if (!make_maps(a, mp, false)) return cudaErrorInvalidValue;
  KArgs k{};
  k.s = a.s;
  k.heads = a.heads;
  k.ntiles = (a.s + TILE - 1) / TILE;
  k.sl2 = 1.4426950408889634f / std::sqrt(static_cast<float>(a.d));
  k.scale = 1.0f / std::sqrt(static_cast<float>(a.d));
  k.lse = a.lse;
  k.out = a.out;
  k.ldo = a.h;
  k.col0 = 0;
  k.d = a.d;
  constexpr int sf = fwd_smem<D>();
  static_assert(fwd_smem<D>() <= 232448, "attention smem budget");
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, sf);
    once = true;
  }
  dim3 grid(a.heads * a.batch, k.ntiles);  // z fastest: all heads' longest tiles go first
  return launch_pdl(attn_fwd_kernel<D>, grid, dim3(FWD_NT), sf, st, 1, mp.q, mp.k, mp.v, k);
}

template <int D>
cudaError_t backward_d(const AttnArgs& a, cudaStream_t st) {
  Maps mp;
  if (!make_maps(a, mp, true)) return cudaErrorInvalidValue;
  const int rows = a.s * a.batch;
  cudaError_t e = launch_pdl(attn_dsum_kernel, dim3((rows * a.heads + 7) / 8), dim3(256), 0, st, 1, a.o, a.dO,
                             a.dsum, a.s, a.heads, a.d, a.h, rows);
  if (e != cudaSuccess) return e;
  KArgs k{};
  k.s = a.s;
  k.heads = a.heads;
  k.ntiles = (a.s + TILE - 1) / TILE;
  k.sl2 = 1.4426950408889634f / std::sqrt(static_cast<float>(a.d));
  k.scale = 1.0f / std::sqrt(static_cast<float>(a.d));
  k.lse = a.lse;
  k.dsum = a.dsum;
  k.out = a.out;
  k.ldo = a.qkv_ld;
  k.d = a.d;
  static bool once = false;
  constexpr int s2 = row_smem<D>(M_DQ), s3 = col_smem<D>();
  static_assert(row_smem<D>(M_DQ) <= 232448 && col_smem<D>() <= 232448, "attention smem budget");
  if (!once) {
    cudaFuncSetAttribute(attn_row_kernel<D, M_DQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
    cudaFuncSetAttribute(attn_col_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3);
    once = true;
  }
  dim3 grid(a.heads * a.batch, k.ntiles);  // z fastest: all heads' longest tiles go first
  k.col0 = 0;  // dQ -> Q block
  e = launch_pdl(attn_row_kernel<D, M_DQ>, grid, dim3(NT), s2, st, 1, mp.q, mp.k, mp.v, mp.dO, k);
  if (e != cudaSuccess) return e;
  k.col0 = a.h;      // dK -> K block
  k.col1 = 2 * a.h;  // dV -> V block
  return launch_pdl(attn_col_kernel<D>, grid, dim3(NT), s3, st, 1, mp.q, mp.k, mp.v, mp.dO, k);
}

}  // namespace

const char* attn_last_message() { return g_amsg.c_str(); }

#ifdef SLIP_ATTN_PROBE
void attn_probe_read(long long* out, int n) { cudaMemcpyFromSymbol(out, g_probe, n * sizeof(long long)); }
#endif

cudaError_t attn_forward(const AttnArgs& a, cudaStream_t s) {
  g_amsg.clear();
  switch (a.d) {
    case 32: return forward_d<32>(a, s);
    case 64: return forward_d<64>(a, s);
    case 80: return forward_d<80>(a, s);
    case 128: return forward_d<128>(a, s);
    default:
      g_amsg = "attention: head dim must be 32, 64, 80 or 128";
      return cudaErrorInvalidValue;
  }
}

cudaError_t attn_backward(const AttnArgs& a, cudaStream_t s) {
  g_amsg.clear();
  switch (a.d) {
    case 32: return backward_d<32>(a, s);
    case 64: return backward_d<64>(a, s);
    case 80: return backward_d<80>(a, s);
    case 128: return backward_d<128>(a, s);
    default:
      g_amsg = "attention: head dim must be 32, 64, 80 or 128";
      return cudaErrorInvalidValue;
  }
}

}  // namespace slip
