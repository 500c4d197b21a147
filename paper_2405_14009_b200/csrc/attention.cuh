// attention.cuh — fused causal attention on tcgen05 (S, dP live only in TMEM; no P in HBM).
//
// Forward (two passes, exact): STATS computes per-row LSE of S = Q K^T / sqrt(d); FWD
// recomputes S tile by tile, forms P = exp(S - LSE) in bf16 in shared memory and
// accumulates O += P V in TMEM.  Backward: prep D = rowsum(dO * O); DQ recomputes S and
// dP = dO V^T per (q-tile, k-tile), forms dS = P (dP - D) / sqrt(d) and accumulates
// dQ += dS K; DKDV walks the q-tiles of one k-tile, forms P^T and dS^T and accumulates
// dV += P^T dO, dK += dS^T Q.  Every product is deterministic (no atomics).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace slip {

struct AttnArgs {
  int s, heads, batch, d;
  int64_t qkv_ld;        // row stride of QKV / dQKV (3h)
  int64_t h;             // hidden (row stride of O / dO)
  const __nv_bfloat16* qkv;  // [T, 3h]  Q | K | V blocks
  const __nv_bfloat16* o;    // [T, h]   attention output (backward: D = rowsum(dO*O))
  const __nv_bfloat16* dO;   // [T, h]
  __nv_bfloat16* out;        // FWD: O [T, h];  backward: dQKV [T, 3h]
  float* lse;                // [z, s] log2-domain log-sum-exp of S*log2(e)/sqrt(d)
  float* dsum;               // [z, s] D = rowsum(dO * O)
  // backward, optional: column sums of the stored (bf16) dQKV per (batch, 32-row group) —
  // the QKV bias gradient's partials: colsum[(b * ceil(s/32) + r / 32) * 3h + col]
  float* colsum = nullptr;
};

cudaError_t attn_forward(const AttnArgs& a, cudaStream_t s);   // writes lse, out = O
cudaError_t attn_backward(const AttnArgs& a, cudaStream_t s);  // writes dsum, out = dQKV (all of it)
const char* attn_last_message();

}  // namespace slip
