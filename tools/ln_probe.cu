// Timing of the HBM-bound row / column kernels in isolation (diagnostic, not part of the
// library): back-to-back launches (PDL, as in the stage step), CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        paper_2405_14009_b200/csrc/kernels.cu tools/ln_probe.cu -o build/ln_probe
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2405_14009_b200/csrc/kernels.cuh"

using slip::bf16;

int main() {
  const int T = 2048, h = 2048, f = 8192;
  bf16 *x, *y, *dy, *dx, *g, *b, *big;
  float *mean, *rstd, *dg, *db, *dxs, *part, *out;
  unsigned* tickets;
  cudaMalloc(&x, T * h * 2);
  cudaMalloc(&y, T * h * 2);
  cudaMalloc(&dy, T * h * 2);
  cudaMalloc(&dx, T * h * 2);
  cudaMalloc(&big, static_cast<size_t>(T) * f * 2);
  cudaMalloc(&g, h * 2);
  cudaMalloc(&b, h * 2);
  cudaMalloc(&mean, T * 4);
  cudaMalloc(&rstd, T * 4);
  cudaMalloc(&dg, h * 4);
  cudaMalloc(&db, h * 4);
  cudaMalloc(&dxs, h * 4);
  cudaMalloc(&out, f * 4);
  cudaMalloc(&part, 3 * slip::kRedChunks * f * 4);
  cudaMalloc(&tickets, slip::kTickets * 4);
  cudaMemset(tickets, 0, slip::kTickets * 4);
  cudaMemset(x, 0, T * h * 2);
  cudaMemset(dy, 0, T * h * 2);
  cudaMemset(big, 0, static_cast<size_t>(T) * f * 2);
  cudaMemset(g, 0, h * 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto fn) {
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e0);
    const int n = 100;
    for (int i = 0; i < n; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1000 / n;
    printf("%-28s %8.2f us  %7.1f GB/s  (%s)\n", name, us, bytes / (us * 1e3), cudaGetErrorString(cudaGetLastError()));
  };
  const double Th = double(T) * h * 2;
  timeit("ln_fwd", 2 * Th, [&] { slip::ln_fwd(x, g, b, y, mean, rstd, T, h, 1e-5f, 0); });
  timeit("ln_bwd rows+colred2", 5 * Th, [&] {
    slip::ln_bwd(dy, x, mean, rstd, g, y, dx, dg, db, dxs, 0, part, tickets, T, h, 0);
  });
  timeit("colsum N=2048", Th, [&] { slip::colsum(dy, T, h, h, out, 0, part, tickets, 0); });
  timeit("colsum N=8192", Th * 4, [&] { slip::colsum(big, T, f, f, out, 0, part, tickets, 0); });
  return 0;
}
