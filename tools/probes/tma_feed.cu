// tma_feed.cu -- L2 -> shared-memory feed-rate microbenchmark (diagnostic, not product).
//
// Question: what bounds the CTA-pair MX GEMM's steady state (~187 cycles per
// 256x256x64 MMA against 136 at the nominal FP4 rate, ~8.5 KB of operands per
// CTA per MMA)?  The per-SM ingress port, or the L2 (LTS) output rate?
// Every CTA streams chunks of `chunk` bytes through a ring of `depth` stages
// with bulk copies (no compute) and we time the grid:
//   mode 0  distinct: every CTA reads its own rows (no sharing)
//   mode 1  shared-4: groups of 4 CTAs read the same rows at about the same time
//   mode 2  multicast: clusters of `csz` CTAs; each issues 1/csz of a chunk with
//           .multicast::cluster to all CTAs of the cluster (every CTA still
//           receives the whole chunk: same ingress, 1/csz of the L2 reads)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probes/tma_feed tools/probes/tma_feed.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2603_08185_b200/csrc/serq_ptx.cuh"
using namespace serq;

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

template <int kMode, int kCsz>
__global__ void __launch_bounds__(64, 1) feed(const __grid_constant__ CUtensorMap map, const uint8_t* __restrict__ src,
                                              size_t src_bytes, int steps, int chunk, int depth, int tensor,
                                              unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16], empty[16];
  const uint32_t rank = kCsz > 1 ? ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kCsz);
    }
    fence_barrier_init();
  }
  if (kCsz > 1) cl_sync(); else __syncthreads();
  const int b = blockIdx.x;
  const size_t nchunks = src_bytes / chunk;
  long long t0 = clock64();
  const int stream = kMode == 1 ? b / 4 : (kMode == 2 ? b / kCsz : b);
  const uint32_t part = chunk / kCsz;
  if (threadIdx.x == 0) {
    // producer: one elected thread, as in the GEMM kernels
    uint32_t c = uint32_t((size_t(stream) * 7919u) % nchunks);
    for (int g = 0, s = 0, ph = 0; g < steps; ++g, c = (c + 1 == nchunks) ? 0 : c + 1) {
      if (g >= depth) mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], chunk);
      const uint8_t* p = src + c * chunk;
      const int rows = chunk / 128, row0 = int(c * rows);
      if (tensor && kMode == 2) {
        const uint16_t mask = (1u << kCsz) - 1;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(sm + s * chunk + rank * part)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&full[s])), "r"(0), "r"(row0 + int(rank) * rows / kCsz),
            "h"(mask)
            : "memory");
      } else if (tensor) {
        for (int q = 0; q < rows / 64; ++q)
          tma_load_2d(sm + s * chunk + q * 8192, &map, &full[s], 0, row0 + q * 64, kEvictNormal);
      } else if (kMode == 2) {
        const uint16_t mask = (1u << kCsz) - 1;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(sm + s * chunk + rank * part)),
            "l"(p + rank * part), "r"(part), "r"(smem_u32(&full[s])), "h"(mask)
            : "memory");
      } else {
        bulk_load(sm + s * chunk, p, chunk, &full[s]);
      }
      if (++s == depth) { s = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    // consumer: releases each stage in every CTA of the cluster (their copies write into ours)
    for (int g = 0, s = 0, ph = 0; g < steps; ++g) {
      mbar_wait(&full[s], ph);
      if (kCsz == 1)
        mbar_arrive(&empty[s]);
      else
        for (int q = 0; q < kCsz; ++q)
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&empty[s]), q))
                       : "memory");
      if (++s == depth) { s = 0; ph ^= 1; }
    }
    out[2 * b] = clock64() - t0;
    out[2 * b + 1] = globaltimer();
  }
  if (kCsz > 1) cl_sync(); else __syncthreads();
}

template <int kMode, int kCsz>
void run(const char* name, const uint8_t* src, size_t bytes, int chunk, int depth, int steps, int grid, int tensor) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  CUtensorMap map;
  cuuint64_t dims[2] = {128, bytes / 128};
  cuuint64_t strides[1] = {128};
  // multicast: each CTA loads rows/csz of the chunk; plain tensor loads: 64-row (8 KB) boxes
  cuuint32_t box[2] = {128, cuuint32_t(kMode == 2 ? chunk / 128 / kCsz : 64)};
  cuuint32_t es[2] = {1, 1};
  reinterpret_cast<EncodeFn>(fp)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(src), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* out;
  cudaMalloc(&out, 2 * grid * sizeof(unsigned long long));
  const int smem = chunk * depth;
  cudaFuncSetAttribute(feed<kMode, kCsz>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCsz;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, feed<kMode, kCsz>, map, src, bytes, steps, chunk, depth, tensor, out);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, feed<kMode, kCsz>, map, src, bytes, steps, chunk, depth, tensor, out);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long* h = (unsigned long long*)malloc(2 * grid * sizeof(unsigned long long));
  cudaMemcpy(h, out, 2 * grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0;
  for (int i = 0; i < grid; ++i) {
    mx = h[2 * i] > mx ? h[2 * i] : mx;
    sum += h[2 * i];
  }
  const double per_cta = double(steps) * chunk;
  printf("%s%-26s chunk %6d depth %2d grid %3d: %s  %7.1f B/cyc/SM (max-CTA), %7.1f mean; chip %6.2f TB/s (events %.1f us)\n",
         tensor ? "TMA2D " : "bulk1D ", name, chunk, depth, grid, err == cudaSuccess ? "ok " : cudaGetErrorString(err), per_cta / mx,
         per_cta / (sum / grid), per_cta * grid / (ms * 1e-3) / 1e12, ms * 1e3);
  free(h);
  cudaFree(out);
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t l2_bytes = 48u << 20, hbm_bytes = 2048u << 20;
  uint8_t* buf;
  cudaMalloc(&buf, hbm_bytes);
  cudaMemset(buf, 1, hbm_bytes);
  const int steps = 2000;
  for (int tensor : {0, 1})
    for (int chunk : {16384, 32768}) {
      const int depth = 196608 / chunk;
      run<0, 1>("L2 distinct 1 CTA", buf, l2_bytes, chunk, depth, steps, 1, tensor);
      run<0, 1>("L2 distinct", buf, l2_bytes, chunk, depth, steps, sms, tensor);
      run<1, 1>("L2 shared-by-4", buf, l2_bytes, chunk, depth, steps, sms, tensor);
      run<2, 2>("L2 multicast csz2", buf, l2_bytes, chunk, depth, steps, sms, tensor);
      run<2, 4>("L2 multicast csz4", buf, l2_bytes, chunk, depth, steps, (sms / 4) * 4, tensor);
      run<0, 1>("HBM distinct", buf, hbm_bytes, chunk, depth, steps, sms, tensor);
    }
  printf("done\n");
  return 0;
}
