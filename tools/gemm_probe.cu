// Cycle stamps of one CTA of a stream-K GEMM (diagnostic, not part of the library).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2405_14009_b200/csrc/gemm.cuh"

namespace slip {
void gemm_probe_read(long long* out, int n);
}

__global__ void fill(__nv_bfloat16* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    p[i] = __float2bfloat16(((h & 0xFFFF) / 65536.0f - 0.5f) * 0.1f);
  }
}

// usage: gemm_probe [K] [random 0/1] [resid+bias 0/1] [b_mn_major 0/1] [N] [also stream-K 0/1] [bn] [pair] [mode 0/1/2]
int main(int argc, char** argv) {
  const int M = 2048, K = argc > 1 ? atoi(argv[1]) : 2048;
  const int rnd = argc > 2 ? atoi(argv[2]) : 0, res = argc > 3 ? atoi(argv[3]) : 0;
  const int bmn = argc > 4 ? atoi(argv[4]) : 0, N = argc > 5 ? atoi(argv[5]) : 2048;
  __nv_bfloat16 *a, *b, *c;
  cudaMalloc(&a, size_t(M) * K * 2);
  cudaMalloc(&b, size_t(N) * K * 2);
  cudaMalloc(&c, size_t(M) * N * 2);
  float* cf;
  cudaMalloc(&cf, size_t(M) * N * 4);
  cudaMemset(cf, 0, size_t(M) * N * 4);
  cudaMemset(a, 0, size_t(M) * K * 2);
  cudaMemset(b, 0, size_t(N) * K * 2);
  __nv_bfloat16 *r, *bias;
  cudaMalloc(&r, size_t(M) * N * 2);
  cudaMalloc(&bias, size_t(N) * 2);
  cudaMemset(r, 0, size_t(M) * N * 2);
  cudaMemset(bias, 0, size_t(N) * 2);
  if (rnd) {
    fill<<<1184, 256>>>(a, size_t(M) * K, 1);
    fill<<<1184, 256>>>(b, size_t(N) * K, 2);
    fill<<<1184, 256>>>(r, size_t(M) * N, 3);
  }
  float* ws;
  unsigned* flags;
  cudaMalloc(&ws, slip::gemm_sk_bytes());
  cudaMalloc(&flags, 4096);
  cudaMemset(flags, 0, 4096);
  const int sk_max = argc > 6 ? atoi(argv[6]) : 0;
  const int bnv = argc > 7 ? atoi(argv[7]) : 256, pairv = argc > 8 ? atoi(argv[8]) : 1;
  const int modev = argc > 9 ? atoi(argv[9]) : 0;  // 0 bf16, 1 GeLU (+aux out), 2 GeLU' (aux in)
  __nv_bfloat16* auxb;
  cudaMalloc(&auxb, size_t(M) * N * 2);
  cudaMemset(auxb, 0, size_t(M) * N * 2);
  if (rnd) fill<<<1184, 256>>>(auxb, size_t(M) * N, 4);
  for (int sk = 0; sk <= sk_max; ++sk) {
    slip::GemmDesc d;
    d.M = M;
    d.N = N;
    d.K = K;
    d.bn = bnv;
    d.pair = pairv != 0;
    d.a.ptr = a;
    d.a.ld = K;
    d.b.ptr = b;
    d.b.ld = bmn ? N : K;
    d.b.mn_major = bmn != 0;
    if (res) {
      d.resid = r;
      d.bias = bias;
    }
    d.c = c;
    d.ldc = N;
    d.mode = modev == 1 ? slip::EPI_BF16_GELU : (modev == 2 ? slip::EPI_BF16_DGELU : slip::EPI_BF16);
    if (modev == 1 || modev == 2) d.aux = auxb;
    if (modev == 4) {  // the W GEMM: dW(f32) += A^T B, both operands MN-major [K rows]
      d.mode = slip::EPI_F32_ACC;
      d.accumulate = 1;
      d.c = cf;
      d.a.mn_major = true;
      d.a.ld = M;
      d.b.mn_major = true;
      d.b.ld = N;
      d.bias = nullptr;
      d.resid = nullptr;
    }
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
    std::vector<long long> p(4096);
    slip::gemm_probe_read(p.data(), 4096);
    const long long t0 = p[0];
    long long tend = 0;
    for (int i = 0; i < 4; ++i)
      if (p[42 + 4 * i] > tend) tend = p[42 + 4 * i];
    printf("M=%d N=%d K=%d rnd=%d res=%d bmn=%d sk=%d: %.2f us, CTA0 %lld cycles (%s)\n", M, N, K, rnd, res, bmn, sk,
           ms * 1000 / 50, tend - t0, cudaGetErrorString(cudaGetLastError()));
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
