// Cycle stamps of one CTA of a stream-K GEMM (diagnostic, not part of the library).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2405_14009_b200/csrc/gemm.cuh"

namespace slip {
void gemm_probe_read(long long* out, int n);
}

int main(int argc, char** argv) {
  const int M = 2048, N = 2048, K = argc > 1 ? atoi(argv[1]) : 2048;
  __nv_bfloat16 *a, *b, *c;
  cudaMalloc(&a, size_t(M) * K * 2);
  cudaMalloc(&b, size_t(N) * K * 2);
  cudaMalloc(&c, size_t(M) * N * 2);
  cudaMemset(a, 0, size_t(M) * K * 2);
  cudaMemset(b, 0, size_t(N) * K * 2);
  float* ws;
  unsigned* flags;
  cudaMalloc(&ws, slip::gemm_sk_bytes());
  cudaMalloc(&flags, 4096);
  cudaMemset(flags, 0, 4096);
  for (int sk = 0; sk < 2; ++sk) {
    slip::GemmDesc d;
    d.M = M;
    d.N = N;
    d.K = K;
    d.bn = 256;
    d.a.ptr = a;
    d.a.ld = K;
    d.b.ptr = b;
    d.b.ld = K;
    d.c = c;
    d.ldc = N;
    d.mode = slip::EPI_BF16;
    if (sk) {
      d.sk_ws = ws;
      d.sk_flags = flags;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 5; ++i) slip::gemm_launch(d, 0);
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) slip::gemm_launch(d, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("K=%d sk=%d: %.2f us (%s)\n", K, sk, ms * 1000 / 50, cudaGetErrorString(cudaGetLastError()));
    std::vector<long long> p(4096);
    slip::gemm_probe_read(p.data(), 4096);
    const long long t0 = p[0];
    printf("  mma item start / acc free / committed:");
    for (int i = 0; i < 4; ++i)
      if (p[10 + i]) printf(" [%lld %lld %lld]", p[10 + i] - t0, p[20 + i] - t0, p[30 + i] - t0);
    printf("\n  epi acc ready / waited / done (kind):");
    for (int i = 0; i < 4; ++i)
      if (p[40 + 4 * i]) printf(" [%lld %lld %lld k%lld]", p[40 + 4 * i] - t0, p[41 + 4 * i] - t0, p[42 + 4 * i] - t0, p[200 + i]);
    printf("\n  chunk (ld, ld done, bf16 start, wait done, computed, fenced, issued):");
    for (int c = 0; c < 4; ++c) {
      const long long b = p[100 + 10 * c];
      printf(" [%lld: +%lld +%lld +%lld +%lld +%lld +%lld]", b - t0, p[101 + 10 * c] - b, p[102 + 10 * c] - b,
             p[106 + 10 * c] - b, p[104 + 10 * c] - b, p[105 + 10 * c] - b, p[103 + 10 * c] - b);
    }
    printf("\n");
    cudaMemset(flags, 0, 4096);
  }
  return 0;
}
