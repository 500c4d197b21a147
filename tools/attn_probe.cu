// Cycle-stamp timeline of one forward-attention CTA (diagnostic, not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSLIP_ATTN_PROBE=7 \
//        -I include paper_2405_14009_b200/csrc/attention.cu paper_2405_14009_b200/csrc/gemm.cu \
//        tools/attn_probe.cu -lcuda -o build/attn_probe && build/attn_probe
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2405_14009_b200/csrc/attention.cuh"

namespace slip {
void attn_probe_read(long long* out, int n);
}

int main() {
  const int s = 2048, heads = 16, d = 128, h = heads * d;
  std::vector<__nv_bfloat16> hq(static_cast<size_t>(s) * 3 * h);
  unsigned x = 12345;
  for (auto& v : hq) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16((static_cast<int>(x >> 9) % 2001 - 1000) / 1000.0f);
  }
  __nv_bfloat16 *qkv, *o;
  float* lse;
  cudaMalloc(&qkv, hq.size() * 2);
  cudaMalloc(&o, static_cast<size_t>(s) * h * 2);
  cudaMalloc(&lse, static_cast<size_t>(heads) * s * 4);
  cudaMemcpy(qkv, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
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
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) slip::attn_forward(a, 0);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) slip::attn_forward(a, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("forward: %.2f us/launch (%s)\n", ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  std::vector<long long> p(4096);
  slip::attn_probe_read(p.data(), 4096);
  const long long t0 = p[0];
  auto show = [&](const char* name, int base, int n) {
    printf("%-14s", name);
    for (int j = 0; j < n; ++j) printf(" %7lld", p[base + j] ? p[base + j] - t0 : -1);
    printf("\n");
  };
  const int nj = 16 - SLIP_ATTN_PROBE;  // k-tiles of the probed CTA (q-tile 15 - y)
  show("P ready@mma", 100, nj);
  show("g0: S seen", 400, nj);
  show("g0: max done", 500, nj);
  show("g0: P done", 600, nj);
  show("g1: S seen", 700, nj);
  show("g1: max done", 800, nj);
  show("g1: P done", 900, nj);
  // backward (dQ kernel probes: CTA y = SLIP_ATTN_PROBE -> q-tile 15 - y)
  __nv_bfloat16 *dO, *dqkv;
  float* dsum;
  cudaMalloc(&dO, static_cast<size_t>(s) * h * 2);
  cudaMalloc(&dqkv, hq.size() * 2);
  cudaMalloc(&dsum, static_cast<size_t>(heads) * s * 4);
  cudaMemcpy(dO, hq.data(), static_cast<size_t>(s) * h * 2, cudaMemcpyHostToDevice);
  a.o = o;
  a.dO = dO;
  a.out = dqkv;
  a.dsum = dsum;
  for (int it = 0; it < 3; ++it) slip::attn_backward(a, 0);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) slip::attn_backward(a, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("backward: %.2f us/launch (%s)\n", ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  slip::attn_probe_read(p.data(), 4096);
  const long long b0 = p[1999];
  auto showb = [&](const char* name, int base, int n) {
    printf("%-14s", name);
    for (int j = 0; j < n; ++j) printf(" %7lld", p[base + j] ? p[base + j] - b0 : -1);
    printf("\n");
  };
  const int nh = 2 * (16 - SLIP_ATTN_PROBE);
  showb("dS ready@mma", 2000, nh);
  showb("g0: S seen", 2100, nh);
  showb("g0: dS done", 2300, nh);
  showb("g1: S seen", 2200, nh);
  showb("g1: dS done", 2400, nh);
  return 0;
}
