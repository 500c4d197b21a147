// TMEM read bandwidth microbenchmark (diagnostic, not part of the library): NW warps per
// CTA (warp w reads TMEM lane quarter w % 4), one CTA per SM, each warp loads the 512
// allocated columns again and again with one tcgen05.ld shape; prints bytes per SM cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/tmem_bw.cu -o build/tmem_bw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2405_14009_b200/csrc/ptx.cuh"

using namespace slip;

template <int SHAPE>
__device__ __forceinline__ uint32_t ld_tile(uint32_t taddr) {
  uint32_t r[32];
  if (SHAPE == 0) {
    ptx::tmem_ld_32x32b_x32(taddr, r);
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
  }
  ptx::tmem_ld_wait();
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) x ^= r[i];
  return x;
}

template <int SHAPE>
__global__ void __launch_bounds__(512, 1) tmem_bw(int iters, int nw, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<512>(&holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  uint32_t acc = 0;
  const long long t0 = clock64();
  if (warp < nw) {
    const int q = warp & 3, grp = warp >> 2, ngrp = (nw + 3) / 4;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    for (int it = 0; it < iters; ++it)
      for (int c = grp * 32; c < 512; c += 32 * ngrp) {
        // 32x32b: 32 lanes x 32 columns; 16x256b.x8: 16 lanes x 64 columns (two halves of the quarter)
        if (SHAPE == 0) acc ^= ld_tile<0>(tmem + lane_off + c);
        else acc ^= ld_tile<1>(tmem + lane_off + (c & ~63) + ((c & 32) ? (16u << 16) : 0u));
      }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 4);
  const int iters = 200;
  for (int shape = 0; shape < 2; ++shape)
    for (int nw : {4, 8, 16}) {
      if (shape == 0) tmem_bw<0><<<148, 512>>>(iters, nw, cyc, sink);
      else tmem_bw<1><<<148, 512>>>(iters, nw, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c[148];
      cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += c[i];
      avg /= 148;
      // bytes per SM: 4 quarters x 32 lanes x 512 columns x 4 B per pass
      const double bytes = 4.0 * 32 * 512 * 4 * iters;
      printf("%s warps %2d: %.1f B/cycle/SM (%s)\n", shape ? "16x256b.x8" : "32x32b.x32", nw, bytes / avg,
             cudaGetErrorString(e));
    }
  return 0;
}
