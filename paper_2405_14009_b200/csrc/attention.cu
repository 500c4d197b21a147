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
  const __nv_bfloat16* o;   // DQ: attention output O [T, h] (for D = rowsum(dO O))
  const __nv_bfloat16* dO;  // DQ: its gradient [T, h]
  int64_t ldh;              // row stride of O / dO
  float* dsum_w;            // DQ: D written here for the dK / dV kernel
  float* colsum;            // backward: per 32-row-group column sums of the stored output
  const __nv_bfloat16* q;   // DQ: Q block of the QKV activation (row stride ldq)
  int64_t ldq;
};

// Descriptor of a 128B-swizzled operand at base; the UMMA_K steps below are constant
// offsets added to it (start-address field, 16-byte units), so that the MMA issue loop
// does not rebuild descriptors per instruction.
__device__ __forceinline__ uint64_t kdesc(uint32_t base) { return ptx::smem_desc_sw128(base, 16, 1024); }
__device__ __forceinline__ uint64_t mdesc(uint32_t base, uint32_t lbo) { return ptx::smem_desc_sw128(base, lbo, 1024); }
__host__ __device__ constexpr uint64_t dk_off(int kk) { return static_cast<uint64_t>((kk >> 2) * (16384 >> 4) + (kk & 3) * 2); }
__host__ __device__ constexpr uint64_t hk_off(int kk) { return static_cast<uint64_t>((kk >> 2) * (8192 >> 4) + (kk & 3) * 2); }
__host__ __device__ constexpr uint64_t m_off(int kk) { return static_cast<uint64_t>(kk * (2048 >> 4)); }

// (kdesc(base) + dk_off(kk): a [128 rows][D] tile as a K-major operand, UMMA_K step kk
//  = 16 d; mdesc(base, ATOM) + m_off(kk): as an MN-major operand, contraction over its
//  rows; hk_off / HATOM: the same for [64 rows][D] half tiles.)
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
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

// Backward epilogue column sums (the QKV bias gradient, KArgs::colsum): the warp's 32 rows
// (row-per-lane, rows >= s count 0) of the chunk's 32 columns, of the values as stored
// (bf16-rounded), summed by ptx::warp_colsum32; lane c writes column c0 + c of its group.
template <int D>
__device__ __forceinline__ void colsum_row_chunk(float* dst, int c0, bool row_ok, const uint32_t (&v)[32]) {
  float cs[32];
#pragma unroll
  for (int i = 0; i < 32; ++i)
    cs[i] = row_ok ? __bfloat162float(__float2bfloat16_rn(__uint_as_float(v[i]))) : 0.f;
  const float t = ptx::warp_colsum32(cs);
  const int lane = threadIdx.x & 31;
  if (c0 + lane < D) dst[c0 + lane] = t;
}

// ====================================================================== forward kernel
// Single pass, online softmax.  One CTA per (q-tile i, z), longest rows first.  TMEM:
// S[0] | S[1] | S[2] | O (128 columns each): S of k-tiles j+1, j+2 are computed while the softmax warps
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
// Optional per-CTA schedule record (globaltimer start / end, SM id) of the backward kernels.
#ifdef SLIP_ATTN_SCHED
__device__ unsigned long long g_sched[2][4096][3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SCHED(k, w)                                                                          \
  do {                                                                                       \
    if (threadIdx.x == 0) {                                                                  \
      const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                                  \
      g_sched[k][cta_][w] = gtimer();                                                        \
      if (w == 0) {                                                                          \
        unsigned sm_;                                                                        \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                     \
        g_sched[k][cta_][2] = sm_;                                                           \
      }                                                                                      \
    }                                                                                        \
  } while (0)
#else
#define SCHED(k, w) \
  do {              \
  } while (0)
#endif

template <int D>
__global__ void __launch_bounds__(FWD_NT, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const KArgs a) {
  using C = AC<D>;
  constexpr int KST = 3, VST = 2, NSB = 3;  // K ring, V ring, S buffers in TMEM (O after them)
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
  uint64_t* s_full = v_empty + VST;          // [NSB] per S buffer
  uint64_t* p_full = s_full + NSB;           // [NSB] P of a k-tile written, per S buffer
  uint64_t* o_done = p_full + NSB;           // [NSB] PV of a k-tile complete, per S buffer
  uint32_t* tholder = reinterpret_cast<uint32_t*>(o_done + NSB);

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
    for (int t = 0; t < NSB; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 16);
      ptx::mbar_init(&o_done[t], 1);
    }
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
      // consumption order of the MMA warp: K0 .. K(NSB-1), then V0 K(NSB) V1 K(NSB+1) ...
      for (int j = 0; j < NSB && j < nj; ++j) load_k(j);
      for (int j = 0; j < nj; ++j) {
        load_v(j);
        if (j + NSB < nj) load_k(j + NSB);
      }
    }
  } else if (warp == 1) {
    {  // ------------------------------------------------ MMA issuer (warp-wide, elected lane issues)
      ptx::mbar_wait(q_full, 0);
      const uint32_t qb = ptx::smem_u32(Qs), kb0 = ptx::smem_u32(Ks), vb0 = ptx::smem_u32(Vs);
      auto mma_s = [&](int j) {  // S[j % NSB] = Q K_j^T
        const int st = j % KST;
        ptx::mbar_wait(&k_full[st], (j / KST) & 1);
        ptx::tc_fence_after();
        const uint32_t kb = kb0 + st * C::TB;
        const uint64_t dq = kdesc(qb), dkk = kdesc(kb);
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk)
          ptx::tc_mma_f16_w(tmem + (j % NSB) * 128, dq + dk_off(kk), dkk + dk_off(kk), C::IDESC_S, kk > 0);
        ptx::tc_commit_w(&s_full[j % NSB]);
        ptx::tc_commit_w(&k_empty[st]);
      };
      for (int j = 0; j < NSB && j < nj; ++j) mma_s(j);
      for (int j = 0; j < nj; ++j) {
        const int st = j % VST;
        ptx::mbar_wait(&p_full[j % NSB], (j / NSB) & 1);
        ptx::mbar_wait(&v_full[st], (j / VST) & 1);
        PROBE(100 + j);
        ptx::tc_fence_after();
        const uint32_t vb = vb0 + st * C::TB;
        const uint64_t dvb = mdesc(vb, ATOM);
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)  // O += P V_j, P (bf16 pairs) from TMEM
          ptx::tc_mma_f16_ts_w(tmem + NSB * 128, tmem + (j % NSB) * 128 + kk * 8, dvb + m_off(kk), C::IDESC_O,
                             (j > 0 || kk > 0) ? 1u : 0u);
        ptx::tc_commit_w(&o_done[j % NSB]);
        ptx::tc_commit_w(&v_empty[st]);
        if (j + NSB < nj) mma_s(j + NSB);  // into the S buffer PV_j reads P from (MMAs execute in order)
      }
    }
  } else if (warp >= 4) {  // ------------------------------------------ softmax warps
    const int lq = warp & 3, g = (warp - 4) >> 2;  // lane quarter, column group (32 keys)
    const int r = lq * 32 + lane;
    const int q = i * TILE + r;
    const uint32_t lane_off = static_cast<uint32_t>(lq * 32) << 16;
    const uint32_t tO = tmem + NSB * 128 + lane_off;
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j < nj; ++j) {
      const uint32_t tS = tmem + (j % NSB) * 128 + lane_off;
      ptx::mbar_wait(&s_full[j % NSB], (j / NSB) & 1);
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
          ptx::mbar_wait(&o_done[(j - 1) % NSB], ((j - 1) / NSB) & 1);
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
      if (lane == 0) ptx::mbar_arrive(&p_full[j % NSB]);
      if (lq == 0 && lane == 0 && g < 2) PROBE(600 + 300 * g + j);
    }
    // total l over the 4 column groups, then O / l and lse
    red[g * TILE + r] = l;
    ptx::named_bar_sync(1 + lq, 128);
    const float lt = (red[r] + red[TILE + r]) + (red[2 * TILE + r] + red[3 * TILE + r]);
    ptx::mbar_wait(&o_done[(nj - 1) % NSB], ((nj - 1) / NSB) & 1);
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

// ====================================================================== backward kernels
// Both walk 64-wide half tiles so that S / dP of step h+1 are computed (double buffer in
// TMEM) while the softmax warps form dS of step h; P and dS are written back to TMEM as
// bf16 pairs over the columns they came from and read there by the next MMA (A operand).
// Warp 0 TMA, warp 1 MMA, warp 2 TMEM allocator, warps 4-11 "softmax" warps: lane
// quarter lq = warp % 4 (32 TMEM lanes = 32 tile rows), column group g (32 of the 64
// columns of a half tile).  A group's bf16 pairs go to the first 16 of its own 32
// columns, so no warp overwrites columns another warp has not read yet.
constexpr int HT = 64;          // rows of a half tile
constexpr int kDqStages = 4;    // K / V half-tile ring of the dQ kernel
constexpr int HATOM = 8192;     // 64 rows x 128 B
constexpr int BWD_NT = 32 * 12;

template <int D>
struct HC {
  static constexpr int HB = AC<D>::NA * HATOM;  // bytes of one [64][D] half tile
  static constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(128, HT, false, false);  // N = 64, K-major x2
  static constexpr uint32_t IDESC_ACC = ptx::idesc_bf16_f32(128, D, false, true);  // A TMEM, B MN-major
};
// TMEM column of the bf16 A operand (64 contraction indices, 2 per column) for step kk:
// group g = kk / 2 wrote its 32 indices to columns [32 g, 32 g + 16)
__device__ __forceinline__ uint32_t acol(int kk) { return 32 * (kk >> 1) + (kk & 1) * 8; }

// ---------------------------------------------------------------- dQ (+ D = rowsum(dO O))
// One CTA per (q-tile i, z), longest first.  S_h = Q K_h^T, dP_h = dO V_h^T over the 64-key
// half tiles h, dS = P (dP - D) / sqrt(d) with P = exp2(S log2e/sqrt(d) - lse), dQ += dS K_h.
// D of the tile's rows is computed here first (and stored for the dK / dV kernel).
// Q and dO — the A operands of every S / dP MMA of the CTA — live in TMEM (written once by
// the softmax warps from their rows, bf16 pairs), so those MMAs read only the 64-key K / V
// half tile from shared memory: with both operands in shared memory the N = 64 MMAs alone
// use the whole shared-memory bandwidth and the K / V TMA writes queue behind them.
template <int D>
__global__ void __launch_bounds__(BWD_NT, 1)
    attn_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK64,
                   const __grid_constant__ CUtensorMap tmV64, const __grid_constant__ CUtensorMap tmdO,
                   const KArgs a) {
  SCHED(0, 0);
  using C = AC<D>;
  using H = HC<D>;
  constexpr int NST = kDqStages, NSB = 2;  // K/V ring stages, S|dP buffers in TMEM (dQ after them)
  constexpr int STG = 2 * H::HB;  // K_h | V_h
  constexpr uint32_t QCOL = 384, DOCOL = 448;  // TMEM columns of Q and dO (bf16 pairs, D / 2 each)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = sm;  // [NST][STG]
  float* red = reinterpret_cast<float*>(ring + NST * STG);  // [2][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 2 * TILE);
  uint64_t* q_full = bar;              // Q, dO written to TMEM (8 warps)
  uint64_t* kv_full = bar + 1;         // [NST]
  uint64_t* kv_empty = kv_full + NST;  // [NST]
  uint64_t* s_full = kv_empty + NST;   // [NSB]
  uint64_t* x_full = s_full + NSB;     // [NSB] dS of a step written (8 warps), per buffer
  uint64_t* acc_full = x_full + NSB;
  uint32_t* tholder = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.x, hn = z % a.heads, bi = z / a.heads;
  const int i = a.ntiles - 1 - static_cast<int>(blockIdx.y);  // longest rows first
  const int q0 = i * TILE;
  // key half tiles covering keys <= min(q0 + 127, s - 1): a box entirely past the end of
  // the sequence is never loaded
  const int kend = q0 + TILE < a.s ? q0 + TILE : a.s;
  const int nh = (kend + HT - 1) / HT;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 8);
    for (int t = 0; t < NST; ++t) {
      ptx::mbar_init(&kv_full[t], 1);
      ptx::mbar_init(&kv_empty[t], 1);
    }
    for (int t = 0; t < NSB; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&x_full[t], 8);
    }
    ptx::mbar_init(acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tholder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tholder;
  ptx::grid_dep_wait();
  if (threadIdx.x == 0) PROBE(1999);

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      for (int h = 0; h < nh; ++h) {
        const int st = h % NST;
        ptx::mbar_wait(&kv_empty[st], ((h / NST) & 1) ^ 1);
        uint8_t* kb = ring + st * STG;
        ptx::mbar_arrive_expect_tx(&kv_full[st], STG);
        for (int t = 0; t < C::NA; ++t) {
          ptx::tma_load_4d(&tmK64, kb + t * HATOM, &kv_full[st], t * 64, h * HT, hn, bi);
          ptx::tma_load_4d(&tmV64, kb + H::HB + t * HATOM, &kv_full[st], t * 64, h * HT, hn, bi);
        }
      }
    }
  } else if (warp == 1) {
    {  // ------------------------------------------------ MMA issuer (warp-wide, elected lane issues)
      ptx::mbar_wait(q_full, 0);
      ptx::tc_fence_after();
      const uint32_t rb = ptx::smem_u32(ring);
      auto mma_sd = [&](int h) {  // S_b = Q K_h^T, dP_b = dO V_h^T  (b = h % NSB), A from TMEM
        const int st = h % NST;
        ptx::mbar_wait(&kv_full[st], (h / NST) & 1);
        ptx::tc_fence_after();
        const uint32_t kb = rb + st * STG, vb = kb + H::HB, tS = tmem + (h % NSB) * 128;
        const uint64_t dkh = kdesc(kb), dvh = kdesc(vb);
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk)
          ptx::tc_mma_f16_ts_w(tS, tmem + QCOL + kk * 8, dkh + hk_off(kk), H::IDESC_S, kk > 0);
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk)
          ptx::tc_mma_f16_ts_w(tS + 64, tmem + DOCOL + kk * 8, dvh + hk_off(kk), H::IDESC_S, kk > 0);
        ptx::tc_commit_w(&s_full[h % NSB]);
      };
      for (int h = 0; h < NSB && h < nh; ++h) mma_sd(h);
      for (int h = 0; h < nh; ++h) {
        const int st = h % NST;
        ptx::mbar_wait(&x_full[h % NSB], (h / NSB) & 1);
        PROBE(2000 + h);
        ptx::tc_fence_after();
        const uint32_t kb = rb + st * STG, tX = tmem + (h % NSB) * 128;
        const uint64_t dkm = mdesc(kb, HATOM);
#pragma unroll
        for (int kk = 0; kk < HT / 16; ++kk)  // dQ += dS K_h, dS (bf16 pairs) from TMEM
          ptx::tc_mma_f16_ts_w(tmem + NSB * 128, tX + acol(kk), dkm + m_off(kk), H::IDESC_ACC, (h > 0 || kk > 0) ? 1u : 0u);
        ptx::tc_commit_w(&kv_empty[st]);
        if (h + NSB < nh) mma_sd(h + NSB);  // into the buffer dQ_h reads dS from (MMAs execute in order)
      }
      ptx::tc_commit_w(acc_full);
    }
  } else if (warp >= 4) {  // ------------------------------------------ dS warps
    const int lq = warp & 3, g = (warp - 4) >> 2;
    const int r = lq * 32 + lane;
    const int q = q0 + r;
    const size_t zs = static_cast<size_t>(z) * a.s;
    const uint32_t lane_off = static_cast<uint32_t>(lq * 32) << 16;
    // Q and dO rows into TMEM (the S / dP MMAs' A operands: row = lane, bf16 pairs along d;
    // column group g writes the UMMA_K steps kk = g, g + 2, ...; rows past s are zero) and
    // D = rowsum(dO * O) over this head's d columns from the same loads
    float dpart = 0.f;
    {
      const bool rok = q < a.s;
      const int64_t ro = (static_cast<int64_t>(bi) * a.s + (rok ? q : 0));
      const __nv_bfloat16* qrow = a.q + ro * a.ldq + static_cast<int64_t>(hn) * a.d;
      const __nv_bfloat16* orow = a.o + ro * a.ldh + static_cast<int64_t>(hn) * a.d;
      const __nv_bfloat16* grow = a.dO + ro * a.ldh + static_cast<int64_t>(hn) * a.d;
      for (int kk = g; kk < C::KS; kk += 2) {
        uint4 qu[2], gu[2], ou[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = kk * 16 + u * 8;
          qu[u] = rok ? *reinterpret_cast<const uint4*>(qrow + c) : make_uint4(0, 0, 0, 0);
          gu[u] = rok ? *reinterpret_cast<const uint4*>(grow + c) : make_uint4(0, 0, 0, 0);
          ou[u] = rok ? *reinterpret_cast<const uint4*>(orow + c) : make_uint4(0, 0, 0, 0);
        }
        const uint32_t qw[8] = {qu[0].x, qu[0].y, qu[0].z, qu[0].w, qu[1].x, qu[1].y, qu[1].z, qu[1].w};
        const uint32_t gw[8] = {gu[0].x, gu[0].y, gu[0].z, gu[0].w, gu[1].x, gu[1].y, gu[1].z, gu[1].w};
        ptx::tmem_st_32x32b_x8(tmem + lane_off + QCOL + kk * 8, qw);
        ptx::tmem_st_32x32b_x8(tmem + lane_off + DOCOL + kk * 8, gw);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ou[u]);
          const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gu[u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = __bfloat1622float2(o2[e]), y = __bfloat1622float2(g2[e]);
            dpart = fmaf(x.x, y.x, dpart);
            dpart = fmaf(x.y, y.y, dpart);
          }
        }
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(q_full);
    }
    red[g * TILE + r] = dpart;
    ptx::named_bar_sync(1 + lq, 64);
    const float drow = red[r] + red[TILE + r];
    if (g == 0 && q < a.s) a.dsum_w[zs + q] = drow;
    const float lrow = q < a.s ? a.lse[zs + q] : 0.f;
    for (int h = 0; h < nh; ++h) {
      const uint32_t tS = tmem + (h % NSB) * 128 + lane_off;
      ptx::mbar_wait(&s_full[h % NSB], (h / NSB) & 1);
      if (lq == 0 && lane == 0) PROBE(2100 + 100 * g + h);
      ptx::tc_fence_after();
      uint32_t sv[32], pv[32];
      ptx::tmem_ld_32x32b_x32(tS + g * 32, sv);
      ptx::tmem_ld_32x32b_x32(tS + 64 + g * 32, pv);
      ptx::tmem_ld_wait();
      const int key0 = h * HT + g * 32;
      const bool diag = key0 + 31 > q0;  // only half tiles reaching the diagonal need the mask
      uint32_t xk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float x0 = ex2(fmaf(__uint_as_float(sv[2 * e]), a.sl2, -lrow)) * (__uint_as_float(pv[2 * e]) - drow) * a.scale;
        float x1 =
            ex2(fmaf(__uint_as_float(sv[2 * e + 1]), a.sl2, -lrow)) * (__uint_as_float(pv[2 * e + 1]) - drow) * a.scale;
        if (diag) {  // select after the arithmetic: nothing computed for a masked key survives
          x0 = key0 + 2 * e <= q ? x0 : 0.f;
          x1 = key0 + 2 * e + 1 <= q ? x1 : 0.f;
        }
        xk[e] = pack2(x0, x1);
      }
      ptx::tmem_st_32x32b_x16(tS + g * 32, xk);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&x_full[h % NSB]);  // per buffer: a warp one step ahead
                                                        // must not count toward this step
      if (lq == 0 && lane == 0) PROBE(2300 + 100 * g + h);
    }
    ptx::mbar_wait(acc_full, 0);
    ptx::tc_fence_after();
    __nv_bfloat16* orow = a.out + (static_cast<int64_t>(bi) * a.s + q) * a.ldo + a.col0 + static_cast<int64_t>(hn) * a.d;
    const int grp0 = q0 + lq * 32;  // this warp's 32-row group
    float* csrow = (a.colsum && grp0 < a.s)
                       ? a.colsum + (static_cast<int64_t>(bi) * ((a.s + 31) >> 5) + (grp0 >> 5)) * a.ldo + a.col0 +
                             static_cast<int64_t>(hn) * a.d
                       : nullptr;
#pragma unroll
    for (int c = 0; c < C::OC; ++c) {
      if ((c & 1) != g) continue;
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + NSB * 128 + lane_off + c * 32, v);
      ptx::tmem_ld_wait();
      if (q < a.s) store_row_chunk<D>(orow, c * 32, v);
      if (csrow) colsum_row_chunk<D>(csrow, c * 32, q < a.s, v);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  SCHED(0, 1);
}

// ---------------------------------------------------------------- dK, dV
// One CTA per (k-tile j, z), longest walks first.  Over the 64-query half tiles h >= the
// diagonal: S^T = K_j Q_h^T, dP^T = V_j dO_h^T, P^T = exp2(S^T log2e/sqrt(d) - lse_q),
// dS^T = P^T (dP^T - D_q) / sqrt(d);  dV += P^T dO_h,  dK += dS^T Q_h.
template <int D>
__global__ void __launch_bounds__(BWD_NT, 1)
    attn_dkdv_kernel(const __grid_constant__ CUtensorMap tmQ64, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO64,
                     const KArgs a) {
  SCHED(1, 0);
  using C = AC<D>;
  using H = HC<D>;
  constexpr int NST = 3;
  constexpr int STG = 2 * H::HB;  // Q_h | dO_h
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Ks = sm;
  uint8_t* Vs = Ks + C::TB;
  uint8_t* ring = Vs + C::TB;  // [NST][STG]
  float* cv = reinterpret_cast<float*>(ring + NST * STG);  // [8 warps][2][32] lse / D of the columns
  uint64_t* bar = reinterpret_cast<uint64_t*>(cv + 8 * 64);
  uint64_t* kv_full = bar;
  uint64_t* qd_full = bar + 1;         // [NST]
  uint64_t* qd_empty = qd_full + NST;  // [NST]
  uint64_t* s_full = qd_empty + NST;   // [2]
  uint64_t* x_full = s_full + 2;       // [2] P^T, dS^T of a step written (8 warps), per buffer
  uint64_t* acc_full = x_full + 2;
  uint32_t* tholder = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.x, hn = z % a.heads, bi = z / a.heads;
  const int j = blockIdx.y;  // k-tile; small j (longest walks) first
  const int k0 = j * TILE;
  const int nh = (a.s - k0 + HT - 1) / HT;  // query half tiles from the diagonal to the end

  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    for (int t = 0; t < NST; ++t) {
      ptx::mbar_init(&qd_full[t], 1);
      ptx::mbar_init(&qd_empty[t], 1);
    }
    ptx::mbar_init(&s_full[0], 1);
    ptx::mbar_init(&s_full[1], 1);
    ptx::mbar_init(&x_full[0], 8);
    ptx::mbar_init(&x_full[1], 8);
    ptx::mbar_init(acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tholder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tholder;
  ptx::grid_dep_wait();

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      ptx::mbar_arrive_expect_tx(kv_full, 2 * C::TB);
      for (int t = 0; t < C::NA; ++t) {
        ptx::tma_load_4d(&tmK, Ks + t * ATOM, kv_full, t * 64, k0, hn, bi);
        ptx::tma_load_4d(&tmV, Vs + t * ATOM, kv_full, t * 64, k0, hn, bi);
      }
      for (int h = 0; h < nh; ++h) {
        const int st = h % NST;
        ptx::mbar_wait(&qd_empty[st], ((h / NST) & 1) ^ 1);
        uint8_t* qs = ring + st * STG;
        ptx::mbar_arrive_expect_tx(&qd_full[st], STG);
        for (int t = 0; t < C::NA; ++t) {
          ptx::tma_load_4d(&tmQ64, qs + t * HATOM, &qd_full[st], t * 64, k0 + h * HT, hn, bi);
          ptx::tma_load_4d(&tmdO64, qs + H::HB + t * HATOM, &qd_full[st], t * 64, k0 + h * HT, hn, bi);
        }
      }
    }
  } else if (warp == 1) {
    {  // ------------------------------------------------ MMA issuer (warp-wide, elected lane issues)
      ptx::mbar_wait(kv_full, 0);
      const uint32_t kb = ptx::smem_u32(Ks), vb = ptx::smem_u32(Vs), rb = ptx::smem_u32(ring);
      auto mma_sd = [&](int h) {  // S^T_b = K Q_h^T, dP^T_b = V dO_h^T  (b = h & 1)
        const int st = h % NST;
        ptx::mbar_wait(&qd_full[st], (h / NST) & 1);
        ptx::tc_fence_after();
        const uint32_t qb = rb + st * STG, ob = qb + H::HB, tS = tmem + (h & 1) * 128;
        const uint64_t dkk = kdesc(kb), dqh = kdesc(qb), dvv = kdesc(vb), doh = kdesc(ob);
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk)
          ptx::tc_mma_f16_w(tS, dkk + dk_off(kk), dqh + hk_off(kk), H::IDESC_S, kk > 0);
#pragma unroll
        for (int kk = 0; kk < C::KS; ++kk)
          ptx::tc_mma_f16_w(tS + 64, dvv + dk_off(kk), doh + hk_off(kk), H::IDESC_S, kk > 0);
        ptx::tc_commit_w(&s_full[h & 1]);
      };
      mma_sd(0);
      if (nh > 1) mma_sd(1);
      for (int h = 0; h < nh; ++h) {
        const int st = h % NST;
        ptx::mbar_wait(&x_full[h & 1], (h >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t qb = rb + st * STG, ob = qb + H::HB, tX = tmem + (h & 1) * 128;
        const uint64_t dom = mdesc(ob, HATOM), dqm = mdesc(qb, HATOM);
#pragma unroll
        for (int kk = 0; kk < HT / 16; ++kk)  // dV += P^T dO_h
          ptx::tc_mma_f16_ts_w(tmem + 256, tX + acol(kk), dom + m_off(kk), H::IDESC_ACC, (h > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < HT / 16; ++kk)  // dK += dS^T Q_h
          ptx::tc_mma_f16_ts_w(tmem + 384, tX + 64 + acol(kk), dqm + m_off(kk), H::IDESC_ACC,
                             (h > 0 || kk > 0) ? 1u : 0u);
        ptx::tc_commit_w(&qd_empty[st]);
        if (h + 2 < nh) mma_sd(h + 2);  // into the buffer dV_h / dK_h read from (in order)
      }
      ptx::tc_commit_w(acc_full);
    }
  } else if (warp >= 4) {  // ------------------------------------------ P^T / dS^T warps (rows = keys)
    const int lq = warp & 3, g = (warp - 4) >> 2;
    const int r = lq * 32 + lane;
    const int key = k0 + r;
    const size_t zs = static_cast<size_t>(z) * a.s;
    const uint32_t lane_off = static_cast<uint32_t>(lq * 32) << 16;
    float* my = cv + (warp - 4) * 64;  // this warp's lse[32] | D[32] of its 32 query columns
    // lse / D of the columns: lane e loads column e one half tile ahead
    float lse_n = INFINITY, d_n = 0.f;
    {
      const int qq = k0 + g * 32 + lane;
      if (qq < a.s) lse_n = a.lse[zs + qq], d_n = a.dsum[zs + qq];
    }
    for (int h = 0; h < nh; ++h) {
      const int qc = k0 + h * HT + g * 32;  // first query column of this warp
      __syncwarp();
      my[lane] = lse_n;
      my[32 + lane] = d_n;
      __syncwarp();
      {
        const int qq = qc + HT + lane;
        lse_n = (h + 1 < nh && qq < a.s) ? a.lse[zs + qq] : INFINITY;
        d_n = (h + 1 < nh && qq < a.s) ? a.dsum[zs + qq] : 0.f;
      }
      const uint32_t tS = tmem + (h & 1) * 128 + lane_off;
      ptx::mbar_wait(&s_full[h & 1], (h >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t sv[32], pv[32];
      ptx::tmem_ld_32x32b_x32(tS + g * 32, sv);
      ptx::tmem_ld_32x32b_x32(tS + 64 + g * 32, pv);
      ptx::tmem_ld_wait();
      const bool diag = qc < k0 + TILE;  // the diagonal block: some columns precede some keys
      uint32_t pk[16], dk2[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float4 L = *reinterpret_cast<const float4*>(my + 4 * (e >> 1));
        const float4 Dv = *reinterpret_cast<const float4*>(my + 32 + 4 * (e >> 1));
        const float l0 = (e & 1) ? L.z : L.x, l1 = (e & 1) ? L.w : L.y;
        const float d0 = (e & 1) ? Dv.z : Dv.x, d1 = (e & 1) ? Dv.w : Dv.y;
        float p0 = ex2(fmaf(__uint_as_float(sv[2 * e]), a.sl2, -l0));
        float p1 = ex2(fmaf(__uint_as_float(sv[2 * e + 1]), a.sl2, -l1));
        float s0 = p0 * (__uint_as_float(pv[2 * e]) - d0) * a.scale;
        float s1 = p1 * (__uint_as_float(pv[2 * e + 1]) - d1) * a.scale;
        if (diag) {  // select after the arithmetic: nothing computed for a masked pair survives
          const bool m0 = qc + 2 * e >= key, m1 = qc + 2 * e + 1 >= key;
          p0 = m0 ? p0 : 0.f;
          p1 = m1 ? p1 : 0.f;
          s0 = m0 ? s0 : 0.f;
          s1 = m1 ? s1 : 0.f;
        }
        pk[e] = pack2(p0, p1);
        dk2[e] = pack2(s0, s1);
      }
      ptx::tmem_st_32x32b_x16(tS + g * 32, pk);
      ptx::tmem_st_32x32b_x16(tS + 64 + g * 32, dk2);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&x_full[h & 1]);  // per buffer: a warp one step ahead
                                                        // must not count toward this step
    }
    ptx::mbar_wait(acc_full, 0);
    ptx::tc_fence_after();
    const int64_t rowoff = (static_cast<int64_t>(bi) * a.s + key) * a.ldo + static_cast<int64_t>(hn) * a.d;
    const int grp0 = k0 + lq * 32;  // this warp's 32-row group
    float* csrow = (a.colsum && grp0 < a.s)
                       ? a.colsum + (static_cast<int64_t>(bi) * ((a.s + 31) >> 5) + (grp0 >> 5)) * a.ldo +
                             static_cast<int64_t>(hn) * a.d
                       : nullptr;
#pragma unroll
    for (int c = 0; c < C::OC; ++c) {
      if ((c & 1) != g) continue;
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + 384 + lane_off + c * 32, v);
      ptx::tmem_ld_wait();
      if (key < a.s) store_row_chunk<D>(a.out + rowoff + a.col0, c * 32, v);
      if (csrow) colsum_row_chunk<D>(csrow + a.col0, c * 32, key < a.s, v);
      ptx::tmem_ld_32x32b_x32(tmem + 256 + lane_off + c * 32, v);
      ptx::tmem_ld_wait();
      if (key < a.s) store_row_chunk<D>(a.out + rowoff + a.col1, c * 32, v);
      if (csrow) colsum_row_chunk<D>(csrow + a.col1, c * 32, key < a.s, v);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  SCHED(1, 1);
}

thread_local std::string g_amsg;

template <int D>
constexpr int fwd_smem() {
  return 6 * AC<D>::TB + 4 * TILE * 4 + 1024 + 1024;
}
template <int D>
constexpr int dq_smem() {
  return kDqStages * 2 * HC<D>::HB + 2 * TILE * 4 + 1024 + 1024;
}
template <int D>
constexpr int dkdv_smem() {
  return 2 * AC<D>::TB + 3 * 2 * HC<D>::HB + 8 * 64 * 4 + 1024 + 1024;
}
struct Maps {
  CUtensorMap q, k, v, dO;          // 128-row boxes
  CUtensorMap q64, k64, v64, dO64;  // 64-row boxes (backward half tiles)
};

bool make_maps(const AttnArgs& a, Maps& m, bool with_do) {
  const uint64_t d = a.d, s = a.s, H = a.heads, B = a.batch;
  const int64_t L = a.qkv_ld;
  bool ok = encode_bf16_4d(&m.q, a.qkv, d, s, H, B, L, d, s * L, 64, 128) &&
            encode_bf16_4d(&m.k, a.qkv + a.h, d, s, H, B, L, d, s * L, 64, 128) &&
            encode_bf16_4d(&m.v, a.qkv + 2 * a.h, d, s, H, B, L, d, s * L, 64, 128);
  if (with_do) {
    ok = ok && encode_bf16_4d(&m.dO, a.dO, d, s, H, B, a.h, d, s * a.h, 64, 128) &&
         encode_bf16_4d(&m.dO64, a.dO, d, s, H, B, a.h, d, s * a.h, 64, 64) &&
         encode_bf16_4d(&m.q64, a.qkv, d, s, H, B, L, d, s * L, 64, 64) &&
         encode_bf16_4d(&m.k64, a.qkv + a.h, d, s, H, B, L, d, s * L, 64, 64) &&
         encode_bf16_4d(&m.v64, a.qkv + 2 * a.h, d, s, H, B, L, d, s * L, 64, 64);
  } else {
    m.dO = m.q;
  }
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
  KArgs k{};
  k.s = a.s;
  k.heads = a.heads;
  k.ntiles = (a.s + TILE - 1) / TILE;
  k.sl2 = 1.4426950408889634f / std::sqrt(static_cast<float>(a.d));
  k.scale = 1.0f / std::sqrt(static_cast<float>(a.d));
  k.lse = a.lse;
  k.dsum = a.dsum;
  k.dsum_w = a.dsum;
  k.o = a.o;
  k.dO = a.dO;
  k.ldh = a.h;
  k.out = a.out;
  k.ldo = a.qkv_ld;
  k.d = a.d;
  k.colsum = a.colsum;
  k.q = a.qkv;
  k.ldq = a.qkv_ld;
  constexpr int s2 = dq_smem<D>(), s3 = dkdv_smem<D>();
  static_assert(dq_smem<D>() <= 232448 && dkdv_smem<D>() <= 232448, "attention smem budget");
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
    cudaFuncSetAttribute(attn_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3);
    once = true;
  }
  dim3 grid(a.heads * a.batch, k.ntiles);  // z fastest: all heads' longest tiles go first
  k.col0 = 0;  // dQ -> Q block (and D for the next kernel)
  cudaError_t e = launch_pdl(attn_dq_kernel<D>, grid, dim3(BWD_NT), s2, st, 1, mp.q, mp.k64, mp.v64, mp.dO, k);
  if (e != cudaSuccess) return e;
  k.col0 = a.h;      // dK -> K block
  k.col1 = 2 * a.h;  // dV -> V block
  return launch_pdl(attn_dkdv_kernel<D>, grid, dim3(BWD_NT), s3, st, 1, mp.q64, mp.k, mp.v, mp.dO64, k);
}

}  // namespace

const char* attn_last_message() { return g_amsg.c_str(); }

#ifdef SLIP_ATTN_PROBE
void attn_probe_read(long long* out, int n) { cudaMemcpyFromSymbol(out, g_probe, n * sizeof(long long)); }
#endif
#ifdef SLIP_ATTN_SCHED
void attn_sched_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_sched, sizeof(g_sched)); }
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
