// gemm.cuh — host interface of the tcgen05/TMEM/TMA GEMM family used by F, B and W.
//
//   D[z](M x N) = sum_k A[z](m, k) * B[z](k, n)       (bf16 operands, fp32 accumulate in TMEM)
//
// Each operand is described by a strided view; "K-major" means k is the contiguous
// index, "MN-major" means m (or n) is.  A batch index z = zo * zi_count + zi selects
// (zi, zo) offsets, which covers per-(batch, head) attention views of the QKV buffer.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace slip {

enum EpiMode : int {
  EPI_BF16 = 0,        // C = bf16(alpha*acc + bias[n] + resid[m,n])
  EPI_BF16_GELU = 1,   // H = alpha*acc + bias[n]; aux = bf16(gelu'(H)); C = bf16(gelu(H))
  EPI_BF16_DGELU = 2,  // C = bf16(acc * aux[m,n])   (aux = gelu'(H) from EPI_BF16_GELU)
  EPI_F32_STORE = 3,   // C(f32) = alpha*acc                  (TMA store)
  EPI_F32_ACC = 4,     // C(f32) += acc, or = acc if !accumulate (TMA reduce-add / store)
  EPI_ADAMW = 5        // g = acc (+ C if accumulate): AdamW on the parameters of C's elements
                       // (GemmDesc::adam), dW itself is not stored (grouped W launches)
};

// EPI_ADAMW: flat fp32 master / m / v, the bf16 weight copy and the gradient buffer the
// problem's C indexes into (element (r, c) of problem g is flat index poff_g + r*ldc + c);
// every element is a 2-D weight (decayed).  inv_bc = 1 / (1 - beta^step).
struct AdamEpi {
  float *p = nullptr, *m = nullptr, *v = nullptr;
  const float* g = nullptr;  // read when accumulate (earlier W's partial sum)
  __nv_bfloat16* w = nullptr;
  float lr = 0.f, b1 = 0.f, b2 = 0.f, eps = 0.f, wd = 0.f, inv_bc1 = 1.f, inv_bc2 = 1.f, grad_scale = 1.f;
  int32_t* nonfinite = nullptr;
};

enum Causal : int {
  CAUSAL_NONE = 0,
  CAUSAL_TILES = 1,    // skip tiles strictly above the diagonal (S = QK^T, dP = dO V^T); BN == 128
  CAUSAL_K_UPPER = 2,  // k ranges over [0, m0 + 128)   (P V, dS K)
  CAUSAL_K_LOWER = 3   // k ranges over [m0, K)          (P^T dO, dS^T Q)
};

struct Operand {
  const void* ptr = nullptr;  // element (0,0) of batch (0,0)
  int64_t ld = 0;             // stride (elements) of the non-contiguous index
  int64_t zi_stride = 0;      // elements
  int64_t zo_stride = 0;      // elements
  bool mn_major = false;      // true: the M (or N) index is contiguous
};

struct GemmDesc {
  int M = 0, N = 0, K = 0;
  int zi_count = 1, zo_count = 1;
  int bn = 256;               // N tile: 32, 80, 128 or 256
  int causal = CAUSAL_NONE;
  Operand a, b;
  // epilogue
  int mode = EPI_BF16;
  void* c = nullptr;          // output base (bf16 or f32)
  int64_t ldc = 0, c_zi = 0, c_zo = 0;  // element strides
  const void* bias = nullptr;     // bf16 [N]
  const void* resid = nullptr;    // bf16, indexed like C
  void* aux = nullptr;            // bf16, indexed like C
  float alpha = 1.0f;
  int accumulate = 0;
  bool pair = true;  // bn == 256, no causal mode: use CTA-pair (cta_group::2) 256 x 256 tiles
  // Stream-K (bf16 epilogues, pair tiles, no batching): when the tiles do not fill whole
  // waves of CTA pairs, every pair takes an equal share of the tile x k-block iterations;
  // a tile split between pairs is finished by the pair holding its first k-block, which
  // adds the fp32 partials the others left in sk_ws (fixed order: deterministic).
  // sk_ws: gemm_sk_bytes() bytes, sk_flags: num_sms() zero-initialised words; NULL: off.
  float* sk_ws = nullptr;
  unsigned* sk_flags = nullptr;
  // Grouped launches (gemm_group_launch proto): the contraction runs over kz_n operand
  // batches — zi = kz_list[j] of the A / B maps (encoded with zi_count > 1), kz_nkb
  // k-blocks each — into one accumulator (the W of several micro-batches, slot = zi).
  int kz_n = 0, kz_nkb = 0;
  int kz_list[8] = {};
  int64_t poff = -1;               // EPI_ADAMW: flat element offset of C (set per problem)
  const AdamEpi* adam = nullptr;   // EPI_ADAMW (grouped launch proto)
  // Grouped fp32 epilogues: a second copy of C, written with the same TMA store / reduce-add
  // (e.g. the DP peer's receive buffer over NVLink: the all-reduce's exchange fused into W).
  // Per problem, encoded into GroupEntry::tm (nullptr: none); the proto's `mirror` enables it.
  const void* c_mirror = nullptr;
  int mirror = 0;
};
size_t gemm_sk_bytes();

// Enqueue on `s`.  Returns cudaSuccess or the launch / encode error; shape errors
// return cudaErrorInvalidValue with a message retrievable by gemm_last_message().
cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t s);

// Grouped persistent launch: many independent problems with the same BN, operand
// majorness and epilogue mode (the W GEMMs of a whole stage) in ONE launch, tiles of
// all problems dealt round-robin to min(#tiles, #SMs) CTAs.  The tensor maps live in a
// device-memory table (encoded once per slot at bind time).
struct alignas(128) GroupEntry {
  CUtensorMap ta, tb, tc;
  CUtensorMap tm;  // GemmDesc::c_mirror (zero when absent)
  int M, N, mt, nkb, tile_begin, tile_end;
  int64_t poff;  // EPI_ADAMW: flat element offset of the problem's C (GemmDesc::poff)
};
cudaError_t gemm_group_encode(const GemmDesc* probs, int n, GroupEntry* host_out, int* total_tiles);
cudaError_t gemm_group_launch(const GroupEntry* dev_table, int n, int total_tiles, const GemmDesc& proto,
                              cudaStream_t s);
const char* gemm_last_message();
int num_sms();
// SMs the persistent GEMM grids may fill: num_sms() minus a reserve left free for
// kernels of other streams (NCCL P2P / all-reduce of the executor) — a persistent CTA
// that cannot be placed waits for the whole concurrent kernel otherwise.
int sm_budget();
void set_sm_reserve(int n);

// 4-D bf16 tensor map, 128-byte swizzle: dims (d0 inner, d1, d2, d3), strides in elements
// of dims 1..3, box (b0, b1, 1, 1).  False (message in gemm_last_message) on failure.
bool encode_bf16_4d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                    int64_t s1, int64_t s2, int64_t s3, uint32_t b0, uint32_t b1);

}  // namespace slip
