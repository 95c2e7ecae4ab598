// tmem_a_test.cu -- does tcgen05.cp.128x256b of the 128B-swizzled K-major A tile into TMEM, then
// kind::mxf4 with A from TMEM, equal the same MMA with A from shared memory?  (diagnostic)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tmem_a_test tools/tmem_a_test.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_08185_b200/csrc/serq_ptx.cuh"
using namespace serq;

__device__ __forceinline__ void mma_mxf4_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t sfa,
                                            uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(128, 1) test(float* out, int variant) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* A = sm;             // 128 rows x 128 B, 128B swizzle
  uint8_t* B = sm + 16384;     // 16 rows x 128 B
  uint8_t* SF = sm + 16384 + 2048;  // 2 x 512 B (SFA chunks), 2 x 512 B (SFB chunks)
  const int t = threadIdx.x;
  for (int i = t; i < 16384 / 4; i += 128) {
    uint32_t h = (i + 7) * 2654435761u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<uint32_t*>(A)[i] = h & 0x77777777u;  // positive codes only: exact sums either way
  }
  for (int i = t; i < 2048 / 4; i += 128) {
    uint32_t h = (i + 11) * 2246822519u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<uint32_t*>(B)[i] = h & 0x77777777u;
  }
  for (int i = t; i < 4096 / 4; i += 128) reinterpret_cast<uint32_t*>(SF)[i] = 0x7F7F7F7Fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (t == 0) {
    const uint32_t sfa = tm + 448, sfb = tm + 464;
    const uint32_t sa = smem_u32(SF), sb = sa + 1024;
    tmem_cp_32x128b_x4(sfa, make_sdesc(sa, 128, 128, 0));
    tmem_cp_32x128b_x4(sfa + 4, make_sdesc(sa + 512, 128, 128, 0));
    tmem_cp_32x128b_x4(sfb, make_sdesc(sb, 128, 128, 0));
    tmem_cp_32x128b_x4(sfb + 4, make_sdesc(sb + 512, 128, 128, 0));
    const uint64_t a = make_sdesc(smem_u32(A), 16, 1024, 2), b = make_sdesc(smem_u32(B), 16, 1024, 2);
    constexpr uint32_t id0 = idesc_mxf4(128, 16), id1 = id0 | (2u << 4) | (2u << 29);
    // SS reference into columns [0, 16)
    mma_mxf4(tm, a, b, id0, sfa, sfb, 0u);
    mma_mxf4(tm, a + 2, b + 2, id1, sfa | (2u << 30), sfb | (2u << 30), 1u);
    mma_mxf4(tm, a + 4, b + 4, id0, sfa + 4, sfb + 4, 1u);
    mma_mxf4(tm, a + 6, b + 6, id1, (sfa + 4) | (2u << 30), (sfb + 4) | (2u << 30), 1u);
    // A -> TMEM columns [64, 96): one 128x256b copy per K = 64 slice
    for (int k = 0; k < 4; ++k) {
      const uint64_t src = variant == 0 ? a + 2 * k : make_sdesc(smem_u32(A) + 32 * k, 16, 1024, 2);
      cp_128x256b(tm + 64 + 8 * k, src);
    }
    mma_mxf4_ts(tm + 16, tm + 64, b, id0, sfa, sfb, 0u);
    mma_mxf4_ts(tm + 16, tm + 72, b + 2, id1, sfa | (2u << 30), sfb | (2u << 30), 1u);
    mma_mxf4_ts(tm + 16, tm + 80, b + 4, id0, sfa + 4, sfb + 4, 1u);
    mma_mxf4_ts(tm + 16, tm + 88, b + 6, id1, (sfa + 4) | (2u << 30), (sfb + 4) | (2u << 30), 1u);
    commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[32];
  tmem_ld_32x32b_x32(tm + ((uint32_t(t >> 5) * 32u) << 16), v);
  tmem_ld_wait();
  for (int j = 0; j < 32; ++j) out[t * 32 + j] = __uint_as_float(v[j]);
  tc_fence_before();
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  float h[128 * 32];
  cudaFuncSetAttribute(test, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int variant = 0; variant < 2; ++variant) {
    test<<<1, 128, 32768>>>(d, variant);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("variant %d: %s\n", variant, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    double s = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 16; ++c) {
        s += h[r * 32 + c];
        if (h[r * 32 + c] != h[r * 32 + 16 + c]) ++bad;
      }
    printf("variant %d: mismatches %d / 2048, checksum %.1f, sample ss %.1f ts %.1f\n", variant, bad, s, h[5 * 32 + 3],
           h[5 * 32 + 19]);
  }
  return 0;
}
