// mma_queue.cu -- how many tcgen05.mma / tcgen05.cp can be queued before issue blocks,
// and the issue cost of commit / mbarrier try_wait.  Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_08185_b200/csrc/serq_ptx.cuh"
using namespace serq;
__global__ void __launch_bounds__(128, 1) q(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint64_t ad = sdesc_k_sw128(sm), bd = sdesc_k_sw128(sm + 32768);
  if (warp == 0 && elect_one()) {
    long long t[40];
    t[0] = clock64();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      mma_mxf4(0, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc_mxf4(128, 256), 448, 472, 1);
      t[i + 1] = clock64();
    }
    tc_commit(&bar);
    t[17] = clock64();
    mbar_wait(&bar, 0);
    t[18] = clock64();
    // cp issue cost
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      tmem_cp_32x128b_x4(448 + 4 * (i % 6), make_sdesc(smem_u32(sm + 512 * i), 128, 128, 0));
      t[19 + i] = clock64();
    }
    tc_commit(&bar2);
    t[31] = clock64();
    mbar_wait(&bar2, 0);
    t[32] = clock64();
    // try_wait on an already-completed barrier
    mbar_wait(&bar2, 0);
    t[33] = clock64();
    for (int i = 0; i < 34; ++i) out[i] = t[i] - t[0];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}
int main() {
  long long* d; cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(q, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) { q<<<1, 128, 100 * 1024>>>(d); cudaDeviceSynchronize(); }
  long long h[64]; cudaMemcpy(h, d, 34 * 8, cudaMemcpyDeviceToHost);
  printf("mma issue stamps: "); for (int i = 1; i <= 16; ++i) printf("%lld ", h[i]); printf("\n");
  printf("commit issued at %lld, all 16 MMAs complete at %lld\n", h[17], h[18]);
  printf("cp issue stamps: "); for (int i = 19; i <= 30; ++i) printf("%lld ", h[i]); printf("\n");
  printf("cp commit at %lld, complete at %lld, try_wait(already complete) at %lld\n", h[31], h[32], h[33]);
  return 0;
}
