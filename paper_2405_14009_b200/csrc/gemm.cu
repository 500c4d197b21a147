// gemm.cu — warp-specialised persistent tcgen05 GEMM for sm_100a.
//
// One kernel family serves every dense contraction of the stage step (F, B and W
// linears; S = QK^T, PV, dP, dV, dQ, dK of attention):
//   warp 0      : TMA producer (one lane) — A/B tiles into a STAGES-deep smem ring
//   warp 1      : MMA issuer  (one lane) — tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16
//   warp 2      : TMEM allocator (2 x ACC_COLS fp32 accumulators = double buffer)
//   warps 4..7  : epilogue — tcgen05.ld 32x32b, then bias / GeLU / GeLU' / residual and bf16
//                 stores, or fp32 TMA store / TMA reduce-add (W: dW += dY^T X fused here).
// Tiles are 128 x BN x 64 (K), statically scheduled round-robin over a grid of
// min(#tiles, #SMs) CTAs; the epilogue of tile i overlaps the mainloop of tile i+1.
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "gemm.cuh"
#include "launch.cuh"
#include "ptx.cuh"
#include "adamw_math.cuh"

namespace slip {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int EPI_WARP0 = 4;
constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, splitting the accumulator columns
constexpr int NUM_THREADS = 32 * (EPI_WARP0 + EPI_WARPS);

template <int BN, bool A_MN, bool B_MN, bool PAIR = false>
struct Cfg {
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  static_assert(!PAIR || BN == 256, "CTA-pair tiles are 256 x 256");
  static constexpr int TILE_M = PAIR ? 2 * BM : BM;  // rows of the output tile (per CTA: BM)
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;  // N extent of B held by each CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ATOMS = (B_ROWS + 63) / 64;
  static constexpr int B_BYTES = B_MN ? B_ATOMS * 8192 : B_ROWS * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196608 / STAGE_BYTES) > 8 ? 8 : (196608 / STAGE_BYTES);
  static constexpr int ACC_COLS = (BN + 31) / 32 * 32;
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 32    ? 32
                                   : 2 * ACC_COLS <= 64  ? 64
                                   : 2 * ACC_COLS <= 128 ? 128
                                   : 2 * ACC_COLS <= 256 ? 256
                                                         : 512;
  static constexpr int EPI_BYTES = EPI_WARPS * 32 * 128;  // one 32x32 fp32 staging tile per epilogue warp
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 1024;
  static constexpr uint32_t IDESC = ptx::idesc_bf16_f32(TILE_M, BN, A_MN, B_MN);
  static constexpr uint32_t A_KSTEP = A_MN ? 2048 : 32;  // bytes per UMMA_K = 16
  static constexpr uint32_t B_KSTEP = B_MN ? 2048 : 32;
  static constexpr uint32_t A_LBO = A_MN ? 8192 : 16;
  static constexpr uint32_t B_LBO = B_MN ? 8192 : 16;
  static_assert(SMEM_BYTES <= 232448, "smem budget");
};

struct KParams {
  int M, N, K;
  int zi_count;
  int mt, nt, nkb;
  int per_z, total;
  int causal;
  int mode;
  void* c;
  int64_t ldc, c_zi, c_zo;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* resid;
  __nv_bfloat16* aux;
  float alpha;
  int accumulate;
  AdamEpi adam;  // EPI_ADAMW
  // grouped mode: the contraction runs over kz_n operand batches (zi = kz_list[j], each
  // kz_nkb k-blocks) into ONE accumulator — the W of several micro-batches in one launch
  int kz_n, kz_nkb;
  int kz_list[8];
  int band;  // grouped tile order: m-tile band width
  const GroupEntry* groups;  // grouped mode: problem table in device memory (nullptr otherwise)
  int n_groups;
  int mirror;  // grouped fp32 epilogues: also write GroupEntry::tm (GemmDesc::c_mirror)
  // stream-K (see GemmDesc)
  int sk;              // 1: stream-K decomposition over sk_units CTA pairs
  int sk_units;
  int sk_dp;           // hybrid: tiles [0, sk_dp) whole and round-robin, AFTER each unit's share
                       // of the stream-K k-space, which covers tiles [sk_dp, sk_dp + sk_iters / nkb)
  int64_t sk_iters;    // total * nkb
  float* sk_ws;        // [2 * sk_units][BM][BN] fp32 partials (slot = pair * 2 + cta)
  unsigned* sk_flags;  // [2 * sk_units] = sk_epoch once the slot's partial is written
  unsigned sk_epoch;
};

// Work items of one CTA (pair): tiles round-robin, or a stream-K share of the tile x
// k-block iterations.  kind: 0 = whole tile, 1 = first part (finishes the tile with the
// other parts' partials), 2 = later part (writes a partial).
struct ItemIter {
  int64_t it, end;  // stream-K iteration range
  int t;            // round-robin tile
};
__device__ __forceinline__ int64_t sk_start(const KParams& p, int u) {
  return static_cast<int64_t>(u) * p.sk_iters / p.sk_units;
}

struct Tile {
  int zi, zo, m0, n0, kb0, kb1;
  int g, M, N;  // problem (grouped mode) and its extent
  int t;        // tile index
};

template <int BN, int TM = BM>
__device__ __forceinline__ Tile decode_tile(int t, const KParams& p) {
  Tile r;
  r.t = t;
  if (p.groups) {
    int lo = 0, hi = p.n_groups - 1;
    while (lo < hi) {  // first problem whose tile range ends after t
      const int mid = (lo + hi) >> 1;
      if (p.groups[mid].tile_end <= t) lo = mid + 1;
      else hi = mid;
    }
    const GroupEntry& ge = p.groups[lo];
    const int q = t - ge.tile_begin;
    r.g = lo;
    r.M = ge.M;
    r.N = ge.N;
    r.zi = r.zo = 0;
    // tiles in bands of GM m-tiles, n-major inside a band: the ~74 tiles in flight touch
    // ~GM A slabs and ~74/GM B slabs, which stay in L2 while the pairs walk K together
    // (plain m-fastest order spread them over every A slab of the problem: with K = 4T
    // the W launch re-read its operands ~4x from DRAM)
    const int GM = p.band;
    const int nt = (ge.N + BN - 1) / BN;
    const int whole = ge.mt / GM * GM;  // m tiles in full bands
    int mb, nb;
    if (q < whole * nt) {
      const int band = q / (GM * nt), l = q - band * (GM * nt);
      mb = band * GM + l % GM;
      nb = l / GM;
    } else {
      const int l = q - whole * nt, gm = ge.mt - whole;
      mb = whole + l % gm;
      nb = l / gm;
    }
    r.m0 = mb * TM;
    r.n0 = nb * BN;
    r.kb0 = 0;
    r.kb1 = ge.nkb * (p.kz_n > 1 ? p.kz_n : 1);
    return r;
  }
  r.g = -1;
  r.M = p.M;
  r.N = p.N;
  const int z = t / p.per_z;
  const int q = t - z * p.per_z;
  int mb, nb;
  if (p.causal == CAUSAL_TILES) {
    mb = static_cast<int>((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
    while ((mb + 1) * (mb + 2) / 2 <= q) ++mb;
    while (mb * (mb + 1) / 2 > q) --mb;
    nb = q - mb * (mb + 1) / 2;
  } else {
    mb = q % p.mt;
    nb = q / p.mt;
  }
  r.zi = z % p.zi_count;
  r.zo = z / p.zi_count;
  r.m0 = mb * TM;
  r.n0 = nb * BN;
  r.kb0 = 0;
  r.kb1 = p.nkb;
  if (p.causal == CAUSAL_K_UPPER) {
    const int lim = (r.m0 + BM + BK - 1) / BK;
    r.kb1 = lim < p.nkb ? lim : p.nkb;
  } else if (p.causal == CAUSAL_K_LOWER) {
    r.kb0 = r.m0 / BK;
  }
  return r;
}

template <int BN, int TM>
__device__ __forceinline__ bool next_item(const KParams& p, int u, int tstep, ItemIter& st, Tile& tl, int& kind) {
  if (!p.sk) {
    if (st.t >= p.total) return false;
    tl = decode_tile<BN, TM>(st.t, p);
    kind = 0;
    st.t += tstep;
    return true;
  }
  if (st.it >= st.end) {  // the share is done: whole tiles of the data-parallel part
    if (st.t >= p.sk_dp) return false;
    tl = decode_tile<BN, TM>(st.t, p);
    kind = 0;
    st.t += tstep;
    return true;
  }
  const int t = static_cast<int>(st.it / p.nkb);
  const int kb0 = static_cast<int>(st.it - static_cast<int64_t>(t) * p.nkb);
  const int64_t rem = st.end - st.it;
  const int kb1 = rem < p.nkb - kb0 ? kb0 + static_cast<int>(rem) : p.nkb;
  tl = decode_tile<BN, TM>(p.sk_dp + t, p);
  tl.kb0 = kb0;
  tl.kb1 = kb1;
  kind = (kb0 == 0 && kb1 == p.nkb) ? 0 : (kb0 == 0 ? 1 : 2);
  st.it += kb1 - kb0;
  return true;
}
__device__ __forceinline__ ItemIter item_begin(const KParams& p, int u) {
  ItemIter st;
  st.t = u;
  st.it = p.sk ? sk_start(p, u) : 0;
  st.end = p.sk ? sk_start(p, u + 1) : 0;
  return st;
}

// gelu(x) and gelu'(x) from one tanh: the forward stores gelu'(H) as the F-stash, so the
// backward epilogue (dH = dG * gelu'(H)) is a multiply instead of a tanh + polynomial
// that paced the FC2 input-gradient GEMM
__device__ __forceinline__ void gelu_and_grad(float x, float& g, float& dg) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float t = ptx::tanh_fast(c * (x + a * x * x * x));
  g = 0.5f * x * (1.0f + t);
  dg = 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * c * (1.0f + 3.0f * a * x * x);
}

__device__ __forceinline__ void st_shared_u4(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
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

#ifdef SLIP_GEMM_PROBE
__device__ long long g_gprobe[4096];
#define GPROBE(idx)                                                                      \
  do {                                                                                   \
    if (blockIdx.x == SLIP_GEMM_PROBE) g_gprobe[idx] = clock64();                        \
  } while (0)
__device__ __forceinline__ void g_gprobe_kind(int i, int k) {
  if (blockIdx.x == SLIP_GEMM_PROBE) g_gprobe[200 + i] = k;
}
#else
#define GPROBE(idx) \
  do {              \
  } while (0)
#define g_gprobe_kind(i, k) \
  do {                      \
  } while (0)
#endif

// ADAMW (compile time): the instantiation of the W launch whose epilogue applies AdamW
// (EPI_ADAMW) — none of the other epilogues are compiled into it, and it into no other
template <int BN, bool A_MN, bool B_MN, bool PAIR, bool ADAMW = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX,
                   const KParams p) {
  using C = Cfg<BN, A_MN, B_MN, PAIR>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  float* epi = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // CTA pair: rank 0 (leader) issues the MMAs for the 256-row tile; each CTA loads and
  // drains its own 128 rows (A) and half of N (B).
  const int cta = PAIR ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const int t0 = PAIR ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
  const int tstep = PAIR ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], PAIR ? 2 : 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], PAIR ? 2 * EPI_WARPS : EPI_WARPS);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0 && !p.groups) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    ptx::prefetch_tmap(&tmC);
    if (p.mode == EPI_BF16_GELU) ptx::prefetch_tmap(&tmX);
  }
  if (warp == 2) {
    if (PAIR) ptx::tmem_alloc_pair<C::TMEM_COLS>(tmem_holder);
    else ptx::tmem_alloc<C::TMEM_COLS>(tmem_holder);
  }
  ptx::tc_fence_before();
  if (PAIR) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  ptx::grid_dep_wait();  // prologue above overlapped the previous kernel (PDL)
  if (threadIdx.x == 0) GPROBE(0);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      ItemIter st = item_begin(p, t0);
      Tile tl;
      int kind;
      while (next_item<BN, C::TILE_M>(p, t0, tstep, st, tl, kind)) {
        const CUtensorMap* mA = tl.g >= 0 ? &p.groups[tl.g].ta : &tmA;
        const CUtensorMap* mB = tl.g >= 0 ? &p.groups[tl.g].tb : &tmB;
        const int am0 = tl.m0 + cta * BM;          // this CTA's rows of A
        const int bn0 = tl.n0 + cta * C::B_ROWS;   // this CTA's part of N
        for (int kb = tl.kb0; kb < tl.kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = ring + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          const int kzj = p.kz_n > 1 ? kb / p.kz_nkb : 0;
          const int kc = (p.kz_n > 1 ? kb - kzj * p.kz_nkb : kb) * BK;  // k coordinate
          const int zc = p.kz_n > 1 ? p.kz_list[kzj] : tl.zi;          // operand batch
          if (PAIR) {
            if (cta == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            else ptx::mbar_arrive_leader(&full[stage]);
            if (!A_MN) {
              ptx::tma_load_4d_pair(mA, sa, &full[stage], kc, am0, zc, tl.zo);
            } else {
              ptx::tma_load_4d_pair(mA, sa, &full[stage], am0, kc, zc, tl.zo);
              ptx::tma_load_4d_pair(mA, sa + 8192, &full[stage], am0 + 64, kc, zc, tl.zo);
            }
            if (!B_MN) {
              ptx::tma_load_4d_pair(mB, sb, &full[stage], kc, bn0, zc, tl.zo);
            } else {
#pragma unroll
              for (int a = 0; a < C::B_ATOMS; ++a)
                ptx::tma_load_4d_pair(mB, sb + a * 8192, &full[stage], bn0 + a * 64, kc, zc, tl.zo);
            }
          } else {
            ptx::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            if (!A_MN) {
              ptx::tma_load_4d(mA, sa, &full[stage], kc, am0, zc, tl.zo);
            } else {
              ptx::tma_load_4d(mA, sa, &full[stage], am0, kc, zc, tl.zo);
              ptx::tma_load_4d(mA, sa + 8192, &full[stage], am0 + 64, kc, zc, tl.zo);
            }
            if (!B_MN) {
              ptx::tma_load_4d(mB, sb, &full[stage], kc, bn0, zc, tl.zo);
            } else {
#pragma unroll
              for (int a = 0; a < C::B_ATOMS; ++a)
                ptx::tma_load_4d(mB, sb + a * 8192, &full[stage], bn0 + a * 64, kc, zc, tl.zo);
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && cta == 0) {
      // ---------------------------------------------------------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      ItemIter st = item_begin(p, t0);
      Tile tl;
      int kind;
      int gi = 0;
      while (next_item<BN, C::TILE_M>(p, t0, tstep, st, tl, kind)) {
        GPROBE(10 + gi);
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        GPROBE(20 + gi);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
        for (int kb = tl.kb0; kb < tl.kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(ring + stage * C::STAGE_BYTES);
          const uint32_t b_base = a_base + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = ptx::smem_desc_sw128(a_base + k * C::A_KSTEP, C::A_LBO, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(b_base + k * C::B_KSTEP, C::B_LBO, 1024);
            if (PAIR) ptx::tc_mma_f16_pair(d_tmem, ad, bd, C::IDESC, (kb > tl.kb0 || k > 0) ? 1u : 0u);
            else ptx::tc_mma_f16(d_tmem, ad, bd, C::IDESC, (kb > tl.kb0 || k > 0) ? 1u : 0u);
          }
          if (PAIR) ptx::tc_commit_pair_mc(&empty[stage], 0x3);
          else ptx::tc_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (PAIR) ptx::tc_commit_pair_mc(&tfull[acc], 0x3);
        else ptx::tc_commit(&tfull[acc]);
        GPROBE(30 + gi);
        ++gi;
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------------------------ epilogue
    const int ew = warp - EPI_WARP0;
    const int lq = ew & 3;    // == warp % 4: TMEM lanes 32*lq .. 32*lq+31
    const int half = ew >> 2;  // this warp drains the 32-column chunks half, half+2, ...
    float* buf = epi + ew * 32 * 32;
    int acc = 0;
    uint32_t acc_phase = 0;
    constexpr int NCH = C::ACC_COLS / 32;
    const int qd = lane & 3;  // bf16 path: 8-column group of this lane after the transpose
    // kernel parameters the chunk loop uses, held in registers: the loop's asm statements
    // clobber "memory", which would otherwise re-read each of them per use
    const int e_mode = p.mode;
    const float e_alpha = p.alpha;
    const __nv_bfloat16* const e_bias = p.bias;
    const __nv_bfloat16* const e_resid = p.resid;
    const int e_accum = p.accumulate;
    const bool ext_res = e_mode < EPI_F32_STORE && e_resid != nullptr;
    const bool ext_aux = e_mode == EPI_BF16_DGELU;
    const bool ext_bias = e_mode < EPI_F32_STORE && e_bias != nullptr;
    ItemIter st = item_begin(p, t0);
    Tile tl;
    int kind;
    int gie = 0;
    while (next_item<BN, C::TILE_M>(p, t0, tstep, st, tl, kind)) {
      const CUtensorMap* mC = tl.g >= 0 ? &p.groups[tl.g].tc : &tmC;
      const int row0 = tl.m0 + cta * BM + lq * 32;
      // residual / GeLU-input operands of a chunk are read-only: their loads are issued one
      // chunk ahead (the first before the accumulator is ready) so DRAM latency overlaps the
      // MMA mainloop and the previous chunk instead of stalling each row group.
      // The bias (8 columns per 16-byte load, the same for every row) is prefetched the same
      // way: loaded at its point of use, its L2 latency serialised the chunk loop.
      uint4 rn[4], hn[4], bn[4];
      auto prefetch = [&](int ch_) {  // this lane's row, 32 columns of chunk ch_: 4 x 16 bytes
        const int mm = row0 + lane;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int cc_ = tl.n0 + ch_ * 32 + 8 * it;
          const bool ok = mm < tl.M && cc_ < tl.N;
          const int64_t off = tl.zo * p.c_zo + tl.zi * p.c_zi + static_cast<int64_t>(mm) * p.ldc + cc_;
          rn[it] = (ext_res && ok) ? __ldg(reinterpret_cast<const uint4*>(p.resid + off)) : make_uint4(0, 0, 0, 0);
          hn[it] = (ext_aux && ok) ? __ldg(reinterpret_cast<const uint4*>(p.aux + off)) : make_uint4(0, 0, 0, 0);
          bn[it] = (ext_bias && cc_ < tl.N) ? __ldg(reinterpret_cast<const uint4*>(e_bias + cc_)) : make_uint4(0, 0, 0, 0);
        }
      };
      if (ext_res || ext_aux || ext_bias) prefetch(half);
      ptx::mbar_wait(&tfull[acc], acc_phase);
      if (ew == 0 && lane == 0) GPROBE(40 + 4 * gie + 0);
      ptx::tc_fence_after();
      const int m = row0 + lane;
      // stream-K: the later parts of this tile (at the start of the next pairs' shares)
      int q_end = t0 + 1;
      if (kind == 1) {
        while (q_end < p.sk_units && sk_start(p, q_end) < static_cast<int64_t>(tl.t - p.sk_dp + 1) * p.nkb) ++q_end;
        if (ew == 0 && lane == 0)
          for (int q = t0 + 1; q < q_end; ++q) {
            if (sk_start(p, q) == sk_start(p, q + 1)) continue;  // empty share: no partial
            const unsigned* f = p.sk_flags + q * (PAIR ? 2 : 1) + cta;
            unsigned v;
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            } while (v != p.sk_epoch);
          }
        ptx::named_bar_sync(1, 32 * EPI_WARPS);
      }
      if (ew == 0 && lane == 0) GPROBE(40 + 4 * gie + 1);
#pragma unroll 1
      for (int ch = half; ch < NCH; ch += 2) {
        // rn / hn / bn hold this chunk's operands; the next chunk's are loaded into the same
        // registers right after their last use below (no copies: register budget)
        const bool pf_next = (ext_res || ext_aux || ext_bias) && ch + 2 < NCH;
        uint32_t r[32];
        if (ew == 0 && lane == 0 && gie == 0) GPROBE(100 + 10 * (ch >> 1) + 0);
        ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(lq * 32) << 16) + acc * C::ACC_COLS + ch * 32, r);
        ptx::tmem_ld_wait_dep(r);  // (orders every use of r after the wait)
        if (ew == 0 && lane == 0 && gie == 0) GPROBE(100 + 10 * (ch >> 1) + 1);
        if (kind == 2) {  // a later part of a split tile: leave the fp32 partial, no epilogue
          if (pf_next) prefetch(ch + 2);
          // partial layout [lane quarter][chunk][8][lane] float4: each store instruction of
          // the warp writes 512 contiguous bytes (the fix-up reads it back the same way)
          float4* dst = reinterpret_cast<float4*>(p.sk_ws + static_cast<size_t>(t0 * (PAIR ? 2 : 1) + cta) * BM * BN) +
                        (lq * NCH + ch) * 8 * 32 + lane;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j * 32] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          continue;
        }
        if (kind == 1) {  // first part: add the later parts' partials in pair order
          for (int q = t0 + 1; q < q_end; ++q) {
            if (sk_start(p, q) == sk_start(p, q + 1)) continue;
            const float4* src =
                reinterpret_cast<const float4*>(p.sk_ws + static_cast<size_t>(q * (PAIR ? 2 : 1) + cta) * BM * BN) +
                (lq * NCH + ch) * 8 * 32 + lane;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 v = __ldcg(src + j * 32);
              r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + v.x);
              r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + v.y);
              r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + v.z);
              r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + v.w);
            }
          }
        }
        const int n = tl.n0 + ch * 32;
        if (n >= tl.N || row0 >= tl.M) {
          if (pf_next) prefetch(ch + 2);
          continue;
        }
        if constexpr (ADAMW) {
          // the W GEMM's final dW tile goes straight into AdamW.  The warp's 32 x 32 block is
          // transposed through its staging tile (XOR swizzle: conflict-free both ways) so
          // that lane = column: every p / m / v / g load and p / m / v / w store of the warp
          // is one coalesced 128-byte (bf16: 64-byte) row segment; rows go 8 at a time with
          // all their loads in flight before any use, the optimizer state streamed
          // (evict-first) so it does not push the W operand slabs out of L2
          const AdamEpi& ad = p.adam;
#pragma unroll
          for (int j = 0; j < 32; ++j) buf[lane * 32 + (j ^ lane)] = __uint_as_float(r[j]);
          __syncwarp();
          const int col = n + lane;
          const bool cok = col < tl.N;
          const int64_t base = (tl.g >= 0 ? p.groups[tl.g].poff : 0) + static_cast<int64_t>(row0) * tl.N + col;
          const int rows = min(32, tl.M - row0);
          bool bad = false;
#pragma unroll 1
          for (int i0 = 0; i0 < rows; i0 += 8) {
            float pp[8], mm[8], vv[8], gg[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int i = i0 + k;
              const bool ok = cok && i < rows;
              const int64_t e = base + static_cast<int64_t>(i) * tl.N;
              pp[k] = ok ? __ldcs(ad.p + e) : 0.f;
              mm[k] = ok ? __ldcs(ad.m + e) : 0.f;
              vv[k] = ok ? __ldcs(ad.v + e) : 0.f;
              gg[k] = (ok && e_accum) ? __ldcs(ad.g + e) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int i = i0 + k;
              if (!cok || i >= rows) continue;
              const float a = buf[i * 32 + (lane ^ i)];
              const float ge = e_accum ? a + gg[k] : a;
              bad |= !isfinite(ge);
              adamw_update(pp[k], mm[k], vv[k], ge, ad.lr, ad.b1, ad.b2, ad.eps, ad.wd, ad.inv_bc1, ad.inv_bc2,
                           ad.grad_scale);
              const int64_t e = base + static_cast<int64_t>(i) * tl.N;
              __stcs(ad.p + e, pp[k]);
              __stcs(ad.m + e, mm[k]);
              __stcs(ad.v + e, vv[k]);
              ad.w[e] = __float2bfloat16_rn(pp[k]);
            }
          }
          __syncwarp();  // the staging tile is rewritten by the next chunk
          if (__any_sync(0xffffffffu, bad) && lane == 0 && ad.nonfinite) atomicOr(ad.nonfinite, 1);
          continue;
        } else {
        if (e_mode >= EPI_F32_STORE) {
          if (lane == 0) ptx::bulk_wait_read0();
          __syncwarp();
          float4* rowp = reinterpret_cast<float4*>(buf + lane * 32);
          const float al = (e_mode == EPI_F32_STORE) ? e_alpha : 1.0f;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            rowp[j ^ (lane & 7)] = make_float4(al * __uint_as_float(r[4 * j]), al * __uint_as_float(r[4 * j + 1]),
                                               al * __uint_as_float(r[4 * j + 2]), al * __uint_as_float(r[4 * j + 3]));
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (e_mode == EPI_F32_ACC && e_accum)
              ptx::tma_reduce_add_4d(mC, buf, n, row0, tl.zi, tl.zo);
            else
              ptx::tma_store_4d(mC, buf, n, row0, tl.zi, tl.zo);
            if (p.mirror && tl.g >= 0) {  // the same tile into the mirror (the DP peer's buffer)
              const CUtensorMap* mM = &p.groups[tl.g].tm;
              if (e_mode == EPI_F32_ACC && e_accum)
                ptx::tma_reduce_add_4d(mM, buf, n, row0, tl.zi, tl.zo);
              else
                ptx::tma_store_4d(mM, buf, n, row0, tl.zi, tl.zo);
            }
            ptx::bulk_commit();
          }
        } else {
          // Row per lane (TMEM lane = output row, 32 consecutive columns in registers): bias
          // (broadcast), GeLU / GeLU' / residual in registers, then the bf16 row is written to
          // this warp's 2 KB staging tile with the 64-byte swizzle (16-byte chunk c of row r at
          // r * 64 + ((c ^ (r >> 1 & 3)) << 4): conflict-free) and one TMA store writes the
          // 32 x 32 tile (the GeLU pre-activation through a second tile and map).
          (void)m;
          if (ew == 0 && lane == 0 && gie == 0) GPROBE(100 + 10 * (ch >> 1) + 2);
          if (lane == 0) ptx::bulk_wait_read0();  // the previous store has read the staging tiles
          __syncwarp();
          if (ew == 0 && lane == 0 && gie == 0) GPROBE(100 + 10 * (ch >> 1) + 6);
          uint8_t* so = reinterpret_cast<uint8_t*>(buf);
          uint8_t* sx = so + 2048;
          const uint32_t so_s = ptx::smem_u32(so), sx_s = so_s + 2048;  // shared-window addresses
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            float x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = e_alpha * __uint_as_float(r[8 * it + e]);
            if (ext_bias) {  // zero beyond N (prefetch)
              float bv[8];
              unpack8(bn[it], bv);
#pragma unroll
              for (int e = 0; e < 8; ++e) x[e] += bv[e];
            }
            const uint32_t soff = lane * 64 + ((it ^ ((lane >> 1) & 3)) << 4);
            if (e_mode == EPI_BF16_GELU) {
              float dg[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) gelu_and_grad(x[e], x[e], dg[e]);
              st_shared_u4(sx_s + soff, pack8(dg));
            } else if (e_mode == EPI_BF16_DGELU) {
              float hv[8];
              unpack8(hn[it], hv);
#pragma unroll
              for (int e = 0; e < 8; ++e) x[e] *= hv[e];
            }
            if (e_resid) {
              float rv[8];
              unpack8(rn[it], rv);
#pragma unroll
              for (int e = 0; e < 8; ++e) x[e] += rv[e];
            }
            st_shared_u4(so_s + soff, pack8(x));
          }
          if (pf_next) prefetch(ch + 2);
          if (ew == 0 && lane == 0 && gie == 0) GPROBE(100 + 10 * (ch >> 1) + 4);
          ptx::fence_proxy_async_smem();
          if (ew == 0 && lane == 0 && gie == 0) GPROBE(100 + 10 * (ch >> 1) + 5);
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_4d(&tmC, so, n, row0, tl.zi, tl.zo);
            if (e_mode == EPI_BF16_GELU) ptx::tma_store_4d(&tmX, sx, n, row0, tl.zi, tl.zo);
            ptx::bulk_commit();
          }
          if (ew == 0 && lane == 0 && gie == 0) GPROBE(100 + 10 * (ch >> 1) + 3);
        }
        }  // !ADAMW
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) ptx::mbar_arrive_leader(&tempty[acc]);
        else ptx::mbar_arrive(&tempty[acc]);
      }
      if (ew == 0 && lane == 0) GPROBE(40 + 4 * gie + 2);
      if (ew == 0 && lane == 0) g_gprobe_kind(gie, kind);
      ++gie;
      if (kind == 2) {  // publish the partial: every writer fences, then one release store
        __threadfence();
        ptx::named_bar_sync(1, 32 * EPI_WARPS);
        if (ew == 0 && lane == 0) {
          unsigned* f = p.sk_flags + t0 * (PAIR ? 2 : 1) + cta;
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(p.sk_epoch) : "memory");
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  if (PAIR) ptx::cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    if (PAIR) ptx::tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
    else ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side
thread_local std::string g_msg;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// 4-D view: dims (inner, outer, zi, zo); strides in elements for dims 1..3.
bool encode4d(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* base, uint64_t d0, uint64_t d1,
              uint64_t d2, uint64_t d3, int64_t s1, int64_t s2, int64_t s3, uint32_t b0, uint32_t b1,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) {
    g_msg = "cuTensorMapEncodeTiled unavailable (driver entry point)";
    return false;
  }
  cuuint64_t dims[4] = {d0, d1, d2 ? d2 : 1, d3 ? d3 : 1};
  auto fix = [](int64_t st, int64_t fallback) -> cuuint64_t {
    int64_t v = st > 0 ? st : fallback;
    return static_cast<cuuint64_t>(v);
  };
  const int64_t s1b = s1 * esize;
  const int64_t s2b = (dims[2] > 1 ? s2 * esize : s1b * static_cast<int64_t>(d1));
  const int64_t s3b = (dims[3] > 1 ? s3 * esize : s2b * static_cast<int64_t>(dims[2]));
  cuuint64_t strides[3] = {fix(s1b, 16), fix(s2b, 16), fix(s3b, 16)};
  for (int i = 0; i < 3; ++i) {
    if (strides[i] % 16 != 0) {
      char b[160];
      snprintf(b, sizeof b, "TMA stride %d = %llu bytes is not a multiple of 16", i + 1,
               static_cast<unsigned long long>(strides[i]));
      g_msg = b;
      return false;
    }
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) {
    g_msg = "TMA base address not 16-byte aligned";
    return false;
  }
  cuuint32_t box[4] = {b0, b1, 1, 1};
  cuuint32_t est[4] = {1, 1, 1, 1};
  CUresult r = fn(map, dt, 4, const_cast<void*>(base), dims, strides, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char b[200];
    snprintf(b, sizeof b, "cuTensorMapEncodeTiled failed (%d): dims %llu %llu %llu %llu box %u %u", static_cast<int>(r),
             (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2],
             (unsigned long long)dims[3], b0, b1);
    g_msg = b;
    return false;
  }
  return true;
}

// operand view for A (rows = M) or B (rows = N)
bool encode_operand(CUtensorMap* map, const Operand& o, int rows, int K, int zi, int zo, uint32_t box_rows) {
  if (!o.mn_major)
    return encode4d(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, o.ptr, K, rows, zi, zo, o.ld, o.zi_stride, o.zo_stride,
                    64, box_rows);
  return encode4d(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, o.ptr, rows, K, zi, zo, o.ld, o.zi_stride, o.zo_stride, 64,
                  64);
}

// Persistent launch: one CTA (or CTA pair, cluster 2x1x1) per SM, at most one per tile.
template <int BN, bool A_MN, bool B_MN, bool PAIR, bool ADAMW = false>
cudaError_t launch_kernel(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tx,
                          const KParams& p, cudaStream_t s) {
  using C = Cfg<BN, A_MN, B_MN, PAIR>;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, PAIR, ADAMW>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return attr_err;
  if (p.total == 0) return cudaSuccess;
  const int units = PAIR ? sm_budget() / 2 : sm_budget();
  const int grid = (p.total < units ? p.total : units) * (PAIR ? 2 : 1);
  return launch_pdl(kern, dim3(grid), dim3(NUM_THREADS), C::SMEM_BYTES, s, PAIR ? 2 : 1, ta, tb, tc, tx, p);
}

template <int BN, bool A_MN, bool B_MN, bool PAIR = false>
cudaError_t launch_t(const GemmDesc& d, cudaStream_t s, const GroupEntry* groups = nullptr, int n_groups = 0,
                     int group_tiles = 0) {
  using C = Cfg<BN, A_MN, B_MN, PAIR>;
  CUtensorMap ta, tb, tc;
  std::memset(&ta, 0, sizeof ta);
  std::memset(&tb, 0, sizeof tb);
  std::memset(&tc, 0, sizeof tc);
  if (groups) {
    KParams p{};
    p.zi_count = 1;
    p.mode = d.mode;
    p.alpha = d.alpha;
    p.accumulate = d.accumulate;
    p.groups = groups;
    p.n_groups = n_groups;
    p.mirror = d.mirror;
    p.total = group_tiles;
    p.band = 8;  // measured: 2 / 4 / 8 / 16 / 32 -> W 15.03 / 14.93 / 14.74 / 14.84 / 15.06 ms
    if (d.mode == EPI_ADAMW) {
      if (!d.adam || !d.adam->p || !d.adam->m || !d.adam->v || !d.adam->w || (d.accumulate && !d.adam->g)) {
        g_msg = "gemm_group: EPI_ADAMW needs the AdamW state (GemmDesc::adam)";
        return cudaErrorInvalidValue;
      }
      p.adam = *d.adam;
    }
    if (d.kz_n > 1) {
      if (d.kz_n > 8 || d.kz_nkb <= 0) {
        g_msg = "gemm_group: kz_n must be in [2, 8] with kz_nkb > 0";
        return cudaErrorInvalidValue;
      }
      p.kz_n = d.kz_n;
      p.kz_nkb = d.kz_nkb;
      for (int j = 0; j < d.kz_n; ++j) p.kz_list[j] = d.kz_list[j];
    }
    if constexpr (A_MN && B_MN)
      if (d.mode == EPI_ADAMW) return launch_kernel<BN, A_MN, B_MN, PAIR, true>(ta, tb, tc, tc, p, s);
    return launch_kernel<BN, A_MN, B_MN, PAIR>(ta, tb, tc, tc, p, s);
  }
  if (!encode_operand(&ta, d.a, d.M, d.K, d.zi_count, d.zo_count, BM)) return cudaErrorInvalidValue;
  if (!encode_operand(&tb, d.b, d.N, d.K, d.zi_count, d.zo_count, C::B_ROWS)) return cudaErrorInvalidValue;
  CUtensorMap tx;
  std::memset(&tx, 0, sizeof tx);
  if (d.mode >= EPI_F32_STORE) {
    if (!encode4d(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d.c, d.N, d.M, d.zi_count, d.zo_count, d.ldc, d.c_zi,
                  d.c_zo, 32, 32))
      return cudaErrorInvalidValue;
  } else {
    // bf16 outputs (and the GeLU pre-activation) leave through TMA stores of 32 x 32 tiles
    // staged in shared memory with the 64-byte swizzle (conflict-free row writes)
    if (!encode4d(&tc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d.c, d.N, d.M, d.zi_count, d.zo_count, d.ldc, d.c_zi,
                  d.c_zo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
    if (d.mode == EPI_BF16_GELU &&
        !encode4d(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d.aux, d.N, d.M, d.zi_count, d.zo_count, d.ldc, d.c_zi,
                  d.c_zo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
  }
  KParams p{};
  p.M = d.M;
  p.N = d.N;
  p.K = d.K;
  p.zi_count = d.zi_count;
  p.mt = (d.M + C::TILE_M - 1) / C::TILE_M;
  p.nt = (d.N + BN - 1) / BN;
  p.nkb = (d.K + BK - 1) / BK;
  p.causal = d.causal;
  p.per_z = d.causal == CAUSAL_TILES ? p.mt * (p.mt + 1) / 2 : p.mt * p.nt;
  p.total = p.per_z * d.zi_count * d.zo_count;
  p.mode = d.mode;
  p.c = d.c;
  p.ldc = d.ldc;
  p.c_zi = d.c_zi;
  p.c_zo = d.c_zo;
  p.bias = static_cast<const __nv_bfloat16*>(d.bias);
  p.resid = static_cast<const __nv_bfloat16*>(d.resid);
  p.aux = static_cast<__nv_bfloat16*>(d.aux);
  p.alpha = d.alpha;
  p.accumulate = d.accumulate;
  // Hybrid stream-K when the tiles leave a partial last wave of CTA pairs (see GemmDesc):
  // the whole waves stay data-parallel, the remainder's tile x k-block iterations are
  // shared evenly, and each pair runs its share FIRST so that the split tiles' epilogues
  // (partials, fix-up) overlap its whole tiles' mainloops; only one-wave-or-more GEMMs.
  const int units = PAIR ? sm_budget() / 2 : sm_budget();
  const int rem_tiles = p.total % units;
  if (PAIR && d.sk_ws && d.sk_flags && d.mode < EPI_F32_STORE && d.causal == CAUSAL_NONE && d.zi_count == 1 &&
      d.zo_count == 1 && p.total > units && rem_tiles != 0 && rem_tiles * p.nkb >= 4 * units) {
    static std::atomic<unsigned> epoch{0};
    p.sk = 1;
    p.sk_units = units;
    p.sk_dp = p.total - rem_tiles;
    p.sk_iters = static_cast<int64_t>(rem_tiles) * p.nkb;
    p.sk_ws = d.sk_ws;
    p.sk_flags = d.sk_flags;
    p.sk_epoch = epoch.fetch_add(1) + 1;
    if (p.sk_epoch == 0) p.sk_epoch = epoch.fetch_add(1) + 1;  // 0 = never written
    p.total = units;  // every pair takes a share
  }
  return launch_kernel<BN, A_MN, B_MN, PAIR>(ta, tb, tc, tx, p, s);
}

template <int BN>
cudaError_t launch_bn(const GemmDesc& d, cudaStream_t s) {
  const bool am = d.a.mn_major, bm = d.b.mn_major;
  if constexpr (BN == 256) {
    if (d.pair && d.causal == CAUSAL_NONE) {
      if (!am && !bm) return launch_t<BN, false, false, true>(d, s);
      if (!am && bm) return launch_t<BN, false, true, true>(d, s);
      if (am && bm) return launch_t<BN, true, true, true>(d, s);
    }
  }
  if (!am && !bm) return launch_t<BN, false, false>(d, s);
  if (!am && bm) return launch_t<BN, false, true>(d, s);
  if (am && bm) return launch_t<BN, true, true>(d, s);
  g_msg = "unsupported operand majorness (A MN-major with B K-major)";
  return cudaErrorInvalidValue;
}

}  // namespace

int num_sms() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  });
  return n;
}

namespace {
std::atomic<int> g_sm_reserve{0};
}
void set_sm_reserve(int n) { g_sm_reserve.store(n < 0 ? 0 : n); }
int sm_budget() {
  const int b = num_sms() - g_sm_reserve.load();
  return b < 2 ? 2 : b;
}

const char* gemm_last_message() { return g_msg.c_str(); }

#ifdef SLIP_GEMM_PROBE
void gemm_probe_read(long long* out, int n) { cudaMemcpyFromSymbol(out, g_gprobe, n * sizeof(long long)); }
#endif

size_t gemm_sk_bytes() { return static_cast<size_t>(num_sms()) * BM * 256 * sizeof(float); }

bool encode_bf16_4d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                    int64_t s1, int64_t s2, int64_t s3, uint32_t b0, uint32_t b1) {
  return encode4d(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, d0, d1, d2, d3, s1, s2, s3, b0, b1);
}

cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t s) {
  g_msg.clear();
  if (d.M <= 0 || d.N <= 0 || d.K <= 0 || d.zi_count <= 0 || d.zo_count <= 0) {
    g_msg = "gemm: non-positive shape";
    return cudaErrorInvalidValue;
  }
  if (d.mode < EPI_F32_STORE && (d.N % 8 != 0 || d.ldc % 8 != 0)) {
    g_msg = "gemm: bf16 epilogue needs N and ldc multiples of 8";
    return cudaErrorInvalidValue;
  }
  if (d.causal == CAUSAL_TILES && (d.bn != 128 || d.M != d.N)) {
    g_msg = "gemm: causal tile skipping needs BN = 128 and M = N";
    return cudaErrorInvalidValue;
  }
  switch (d.bn) {
    case 32: return launch_bn<32>(d, s);
    case 64: return launch_bn<64>(d, s);
    case 80: return launch_bn<80>(d, s);
    case 128: return launch_bn<128>(d, s);
    case 256: return launch_bn<256>(d, s);
    default:
      g_msg = "gemm: unsupported BN (32, 64, 80, 128, 256)";
      return cudaErrorInvalidValue;
  }
}

cudaError_t gemm_group_encode(const GemmDesc* probs, int n, GroupEntry* out, int* total_tiles) {
  g_msg.clear();
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    const GemmDesc& d = probs[i];
    if (d.bn != probs[0].bn || d.a.mn_major != probs[0].a.mn_major || d.b.mn_major != probs[0].b.mn_major ||
        d.mode != probs[0].mode || d.mode < EPI_F32_STORE || d.zi_count < 1 || d.zo_count != 1 ||
        d.causal != CAUSAL_NONE) {
      g_msg = "gemm_group: problems must share BN, majorness and an fp32 epilogue, without output batching";
      return cudaErrorInvalidValue;
    }
    GroupEntry& g = out[i];
    std::memset(&g, 0, sizeof g);
    // zi_count > 1: operand batches the contraction may run over (GemmDesc::kz_*); the
    // output has none
    if (!encode_operand(&g.ta, d.a, d.M, d.K, d.zi_count, 1, BM)) return cudaErrorInvalidValue;
    const uint32_t b_rows = (probs[0].pair && probs[0].bn == 256) ? 128u : static_cast<uint32_t>(d.bn);
    if (!encode_operand(&g.tb, d.b, d.N, d.K, d.zi_count, 1, b_rows)) return cudaErrorInvalidValue;
    if (!encode4d(&g.tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d.c, d.N, d.M, 1, 1, d.ldc, 0, 0, 32, 32))
      return cudaErrorInvalidValue;
    if (d.c_mirror &&
        !encode4d(&g.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d.c_mirror, d.N, d.M, 1, 1, d.ldc, 0, 0, 32, 32))
      return cudaErrorInvalidValue;
    const int tile_m = (probs[0].pair && probs[0].bn == 256) ? 2 * BM : BM;
    g.M = d.M;
    g.N = d.N;
    g.poff = d.poff;
    g.mt = (d.M + tile_m - 1) / tile_m;
    g.nkb = (d.K + BK - 1) / BK;
    g.tile_begin = tiles;
    tiles += g.mt * ((d.N + d.bn - 1) / d.bn);
    g.tile_end = tiles;
  }
  *total_tiles = tiles;
  return cudaSuccess;
}

cudaError_t gemm_group_launch(const GroupEntry* dev_table, int n, int total_tiles, const GemmDesc& proto,
                              cudaStream_t s) {
  g_msg.clear();
  if (!proto.a.mn_major || !proto.b.mn_major || proto.bn != 256) {
    g_msg = "gemm_group: instantiated for BN = 256 with MN-major A and B (the W GEMMs)";
    return cudaErrorInvalidValue;
  }
  if (proto.pair) return launch_t<256, true, true, true>(proto, s, dev_table, n, total_tiles);
  return launch_t<256, true, true>(proto, s, dev_table, n, total_tiles);
}

}  // namespace slip
