// tcgen05.mma issue-rate microbenchmark (diagnostic, not part of the library): one CTA per
// SM issues back-to-back kind::f16 MMAs (M = 128, K = 16, bf16 -> fp32) from smem (SS) or
// with A from TMEM (TS) and reports tensor cycles per MMA against the floor 128*N/256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/mma_rate.cu -o build/mma_rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2405_14009_b200/csrc/ptx.cuh"

using namespace slip;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  constexpr uint32_t IDESC = ptx::idesc_bf16_f32(128, N, false, false);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(sm), b = a + 16384;
    const uint64_t ad = ptx::smem_desc_sw128(a, 16, 1024), bd = ptx::smem_desc_sw128(b, 16, 1024);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (TS) ptx::tc_mma_f16_ts(tmem + 256, tmem + 384 + 8 * k, bd + 2 * k, IDESC, 1u);
        else ptx::tc_mma_f16(tmem, ad + 2 * k, bd + 2 * k, IDESC, 1u);
      }
    }
    ptx::tc_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int N, bool TS>
void run(const char* name) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000, smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(mma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate<N, TS><<<148, 128, smem>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148];
  cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  printf("%-22s N=%3d: %.1f cycles / MMA (floor %d) (%s)\n", name, N, avg / (4.0 * iters), 128 * N / 256,
         cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<64, false>("SS M128 K16");
  run<128, false>("SS M128 K16");
  run<256, false>("SS M128 K16");
  run<64, true>("TS M128 K16");
  run<128, true>("TS M128 K16");
  return 0;
}
