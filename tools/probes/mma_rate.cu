// mma_rate.cu -- tcgen05 MMA issue-rate microbenchmark (diagnostic, not product).
// Every CTA issues back-to-back MMAs on garbage smem / TMEM operands and we
// time the whole grid; reports TFLOP/s for several kinds / shapes / cta_group.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_08185_b200/csrc/serq_ptx.cuh"
using namespace serq;

__device__ __forceinline__ void mma_mxf4_2cta(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                              uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void commit_2cta(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}

template <int KIND, int N, int CG, int VAR = 0>  // VAR bit0: commit per 4, bit1: sf_id 0/2, bit2: acc reset every 65; KIND 0 = mxf4, 1 = f16, 2 = i8, 3 = mxf4 with A in TMEM (ts)
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  if (VAR & 8) {  // random operand bytes (realistic switching activity)
    uint32_t* w = reinterpret_cast<uint32_t*>(sm);
    for (int i = threadIdx.x; i < 220 * 1024 / 4; i += blockDim.x) {
      uint32_t h = (i + 1) * 2654435761u ^ (blockIdx.x * 97u);
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      w[i] = h;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tm = slot;
  const uint64_t ad = sdesc_k_sw128(sm), bd = sdesc_k_sw128(sm + 32768);
  const uint32_t M = CG == 2 ? 256 : 128;
  long long t0 = clock64();
  __shared__ uint64_t fullb[8], emptyb[8];
  if (VAR & 16) {  // producer (warp 1) / MMA (warp 0) handshake over an S-stage mbarrier ring
    constexpr int S = (VAR & 32) ? 8 : 4;
    if (threadIdx.x == 0) {
      for (int i = 0; i < S; ++i) { mbar_init(&fullb[i], 1); mbar_init(&emptyb[i], 1); }
      fence_barrier_init();
    }
    __syncthreads();
    if (warp == 1) {
      if (elect_one())
        for (int g = 0; g < iters; ++g) {
          mbar_wait(&emptyb[g % S], ((g / S) & 1) ^ 1);
          mbar_arrive(&fullb[g % S]);
        }
    } else if (warp == 0) {
      for (int g = 0; g < iters; ++g) {
        mbar_wait(&fullb[g % S], (g / S) & 1);
        tc_fence_after();
        if (elect_one()) {
          for (int j = 0; j < 4; ++j)
            mma_mxf4(tm, ad + j * 2, bd + j * 2, idesc_mxf4(M, N), tm + 448, tm + 480, 1);
          tc_commit(&emptyb[g % S]);
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(&bar);
      __syncwarp();
    }
  } else
  if (warp == 0 && rank == 0 && elect_one()) {
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < 4; ++j) {
        // VAR 256: rotate over 4 stage buffers of 51 KB like the real kernel (A 16 KB, B 32 KB)
        const uint32_t soff = (VAR & 256) ? uint32_t((it & 3) * 52224) : 0u;
        const uint64_t a = ((VAR & 256) ? sdesc_k_sw128(sm + soff) : ad) + j * 2;
        const uint64_t b = ((VAR & 256) ? sdesc_k_sw128(sm + soff + 16384) : bd) + j * 2;
        if (KIND == 0) {
          const uint32_t sfid = (VAR & 2) ? (j & 1) * 2 : 0;
          const uint32_t accf = (VAR & 4) ? (((it * 4 + j) % 65) != 0) : 1;
          const uint32_t dcol = (VAR & 64) ? 192 : ((VAR & 128) ? 64 : 0);
          if (CG == 1)
            mma_mxf4(tm + dcol, a, b, idesc_mxf4(M, N) | (sfid << 4) | (sfid << 29), (tm + 448 + (j >> 1) * 4) | (sfid << 30),
                     (tm + 472 + (j >> 1) * 8) | (sfid << 30), accf);
          else
            mma_mxf4_2cta(tm, a, b, idesc_mxf4(M, N), tm + 448, tm + 480, 1);
        } else if (KIND == 1) {
          mma_bf16(tm, a, b, idesc_bf16(M, N), 1);
        } else if (KIND == 2) {
          mma_i8(tm, a, b, idesc_i8(M, N, true, true), 1);
        } else {
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, 1, 0;\n"
              " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n}\n" ::"r"(tm),
              "r"(tm + 256), "l"(b), "r"(idesc_mxf4(M, N)), "r"(tm + 448), "r"(tm + 480));
        }
      }
      if (VAR & 1) tc_commit(&bar2);
    }
    if (CG == 1) tc_commit(&bar); else commit_2cta(&bar);
  }
  __syncwarp();
  if (warp == 0 && rank == 0) mbar_wait(&bar, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) atomicMax(cycles, (unsigned long long)(t1 - t0));
  tc_fence_before();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (warp == 0) {
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

template <int KIND, int N, int CG, int VAR = 0>
void run(const char* name, double kflops_per_mma_per_M) {
  const int iters = 20000, smem = 220 * 1024;
  auto k = bench<KIND, N, CG, VAR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  cudaMemset(dc, 0, 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaLaunchKernelEx(&cfg, k, 10, dc);
  cudaDeviceSynchronize();
  cudaMemset(dc, 0, 8);
  cudaEventRecord(s);
  cudaLaunchKernelEx(&cfg, k, iters, dc);
  cudaEventRecord(e);
  cudaError_t err = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  unsigned long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  const int M = CG == 2 ? 256 : 128;
  const double mmas = double(iters) * 4 * (148 / CG);
  const double flops = mmas * 2.0 * M * N * kflops_per_mma_per_M;
  printf("%-34s %s  %8.1f TFLOP/s  %7.1f cyc/MMA  (%.3f ms)\n", name, err == cudaSuccess ? "ok " : cudaGetErrorString(err),
         flops / (ms * 1e-3) / 1e12, double(cyc) / (iters * 4.0), ms);
  cudaFree(dc);
}

int main() {
  run<0, 256, 1, 256 + 8>("mxf4 cta1 N256 ROTATING 4 stages", 64);
  run<0, 128, 1, 256 + 8>("mxf4 cta1 N128 ROTATING 4 stages", 64);
  run<0, 256, 2, 256 + 8>("mxf4 cta2 N256 ROTATING 4 stages", 64);
  run<2, 256, 1, 256 + 8>("i8 cta1 N256 ROTATING 4 stages", 32);
  return 0;
  run<0, 256, 1, 64>("mxf4 cta1 N256 D at col 192", 64);
  run<0, 256, 1, 128>("mxf4 cta1 N256 D at col 64", 64);
  run<0, 256, 1, 16>("mxf4 cta1 N256 4-stage handshake", 64);
  run<0, 256, 1, 48>("mxf4 cta1 N256 8-stage handshake", 64);
  run<0, 256, 1, 8>("mxf4 cta1 N256 RANDOM data", 64);
  run<0, 256, 2, 8>("mxf4 cta2 N256 RANDOM data", 64);
  run<2, 256, 1, 8>("i8 cta1 N256 RANDOM data", 32);
  run<1, 256, 1, 8>("bf16 cta1 N256 RANDOM data", 16);
  run<0, 256, 1, 1>("mxf4 cta1 N256 commit/4", 64);
  run<0, 256, 1, 2>("mxf4 cta1 N256 sfid 0/2", 64);
  run<0, 256, 1, 4>("mxf4 cta1 N256 acc reset/65", 64);
  run<0, 256, 1, 7>("mxf4 cta1 N256 all three", 64);
  run<0, 256, 1>("mxf4 SS cta1 M128 N256 K64", 64);
  run<0, 128, 1>("mxf4 SS cta1 M128 N128 K64", 64);
  run<0, 64, 1>("mxf4 SS cta1 M128 N64 K64", 64);
  run<3, 256, 1>("mxf4 TS cta1 M128 N256 K64", 64);
  run<0, 256, 2>("mxf4 SS cta2 M256 N256 K64", 64);
  run<0, 128, 2>("mxf4 SS cta2 M256 N128 K64", 64);
  run<1, 256, 1>("bf16 SS cta1 M128 N256 K16", 16);
  run<2, 256, 1>("i8   SS cta1 M128 N256 K32", 32);
  return 0;
}
