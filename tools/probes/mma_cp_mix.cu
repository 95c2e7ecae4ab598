// mma_cp_mix.cu -- do UTCCP scale-factor copies serialize with tcgen05.mma in the tensor pipe?
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_08185_b200/csrc/serq_ptx.cuh"
using namespace serq;
template <int NCP, int COMMIT>
__global__ void __launch_bounds__(128, 1) mix(int stages, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t sb = smem_u32(sm);
  long long t0 = clock64();
  if (warp == 0 && elect_one()) {
    for (int g = 0; g < stages; ++g) {
      const uint32_t st = sb + (g & 3) * 52224;
      const uint64_t ad = make_sdesc(st, 16, 1024, 2), bd = make_sdesc(st + 16384, 16, 1024, 2);
      const uint32_t fa = 448 + (g & 1) * 24, fb = fa + 8;
#pragma unroll
      for (int c = 0; c < NCP; ++c) tmem_cp_32x128b_x4(fa + 4 * c, make_sdesc(st + 49152 + 512 * c, 128, 128, 0));
      mma_mxf4(0, ad, bd, idesc_mxf4(128, 256), fa, fb, 1);
      mma_mxf4(0, ad + 2, bd + 2, idesc_mxf4(128, 256), fa, fb, 1);
      mma_mxf4(0, ad + 4, bd + 4, idesc_mxf4(128, 256), fa + 4, fb + 8, 1);
      mma_mxf4(0, ad + 6, bd + 6, idesc_mxf4(128, 256), fa + 4, fb + 8, 1);
      if (COMMIT) tc_commit(&bar2);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    atomicMax(cyc, (unsigned long long)(clock64() - t0));
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}
template <int NCP, int COMMIT>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  auto k = mix<NCP, COMMIT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  k<<<148, 128, 210 * 1024>>>(100, d); cudaDeviceSynchronize(); cudaMemset(d, 0, 8);
  const int stages = 4000;
  k<<<148, 128, 210 * 1024>>>(stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%d cps + 4 MMA per stage, commit=%d: %.1f cycles/stage (%s)\n", NCP, COMMIT, double(h) / stages, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<0, 0>(); run<0, 1>(); run<2, 1>(); run<4, 1>(); run<6, 0>(); run<6, 1>(); run<12, 1>();
  return 0;
}
