// Per-CTA schedule of the attention backward kernels (diagnostic, not part of the library):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSLIP_ATTN_SCHED \
//        -I include paper_2405_14009_b200/csrc/attention.cu paper_2405_14009_b200/csrc/gemm.cu \
//        tools/attn_sched.cu -lcuda -o build/attn_sched && build/attn_sched
// Prints, per kernel: span, SM busy fraction, and CTA duration by tile index.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <vector>

#include "../paper_2405_14009_b200/csrc/attention.cuh"

namespace slip {
void attn_sched_read(unsigned long long* out);
}

int main() {
  const int s = 2048, heads = 16, d = 128, h = heads * d;
  std::vector<__nv_bfloat16> hq(static_cast<size_t>(s) * 3 * h);
  unsigned x = 12345;
  for (auto& v : hq) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16((static_cast<int>(x >> 9) % 2001 - 1000) / 1000.0f);
  }
  __nv_bfloat16 *qkv, *o, *dO, *dqkv;
  float *lse, *dsum;
  cudaMalloc(&qkv, hq.size() * 2);
  cudaMalloc(&o, static_cast<size_t>(s) * h * 2);
  cudaMalloc(&dO, static_cast<size_t>(s) * h * 2);
  cudaMalloc(&dqkv, hq.size() * 2);
  cudaMalloc(&lse, static_cast<size_t>(heads) * s * 4);
  cudaMalloc(&dsum, static_cast<size_t>(heads) * s * 4);
  cudaMemcpy(qkv, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dO, hq.data(), static_cast<size_t>(s) * h * 2, cudaMemcpyHostToDevice);
  slip::AttnArgs a{};
  a.s = s;
  a.heads = heads;
  a.batch = 1;
  a.d = d;
  a.qkv_ld = 3 * h;
  a.h = h;
  a.qkv = qkv;
  a.out = o;
  a.lse = lse;
  slip::attn_forward(a, 0);
  a.o = o;
  a.dO = dO;
  a.out = dqkv;
  a.dsum = dsum;
  for (int it = 0; it < 5; ++it) slip::attn_backward(a, 0);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> g(2 * 4096 * 3);
  slip::attn_sched_read(g.data());
  const int nt = s / 128, nz = heads;
  for (int k = 0; k < 2; ++k) {
    unsigned long long t0 = ~0ull, t1 = 0;
    double busy = 0;
    std::map<int, std::vector<double>> by_tile;
    for (int y = 0; y < nt; ++y)
      for (int z = 0; z < nz; ++z) {
        const unsigned long long* r = &g[((size_t)k * 4096 + y * nz + z) * 3];
        t0 = std::min(t0, r[0]);
        t1 = std::max(t1, r[1]);
        busy += (double)(r[1] - r[0]);
        by_tile[y].push_back((r[1] - r[0]) / 1000.0);
      }
    printf("%s: span %.2f us, SM busy %.1f %% (148 SMs)\n", k ? "dKdV" : "dQ", (t1 - t0) / 1000.0,
           100.0 * busy / (148.0 * (double)(t1 - t0)));
    for (auto& kv : by_tile) {
      double mn = 1e9, mx = 0, sum = 0;
      for (double v : kv.second) mn = std::min(mn, v), mx = std::max(mx, v), sum += v;
      unsigned long long st_min = ~0ull, st_max = 0;
      for (int z = 0; z < nz; ++z) {
        const unsigned long long* r = &g[((size_t)k * 4096 + kv.first * nz + z) * 3];
        st_min = std::min(st_min, r[0] - t0);
        st_max = std::max(st_max, r[0] - t0);
      }
      printf("  y=%2d: CTA us min %.2f avg %.2f max %.2f, start %.2f..%.2f us\n", kv.first, mn,
             sum / kv.second.size(), mx, st_min / 1000.0, st_max / 1000.0);
    }
  }
  return 0;
}
