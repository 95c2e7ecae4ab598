// serq_gemm_decode.cuh -- HBM-bound MXFP4 SERQ linear for decode (M <= 16).
//
// Swap-AB: D^T[128 weight rows, 16 tokens] = W_tile[128, K] . X^T, so the
// weights fill the MMA's M=128 dimension and the (zero-padded) tokens its N=16
// dimension (tcgen05.mma.cta_group::1.kind::mxf4, 128x16x64).  The grid is
// (N/128 weight tiles) x (K splits) so that every SM streams weights; the
// tensor work is tiny and the kernel is bound by HBM bytes
//     N*K/2 (codes) + N*K/32 (E8M0) + N*r/2 + N*r/32 (R) + M*K*(1/2 + 1/32) (X) + 2*M*N (Y).
// Split-K partials (fp32, [split][N][16]) are reduced in a FIXED order by the
// last-arriving CTA of each weight tile (deterministic), which also adds the
// salient term computed by the split that owns K-tile 0: one MMA with A = R's
// 128 rows (32 B each, 32B swizzle) and B = K-tile 0 of X.
#pragma once
#include "serq_gemm.cuh"

namespace serq {

constexpr int kDecN = 16;                       // tokens per MMA (padded)
constexpr int kDecStagesDefault = 5;  // 100 KB: two CTAs per SM
constexpr int kDecW = 128 * kStepBytes;         // 16 KB weight tile per 256-K step
constexpr int kDecX = kDecN * kStepBytes;       // 2 KB token tile
constexpr int kDecSF = 1024;                    // 2 SF chunks of one 128-row block
constexpr int kDecStage = kDecW + kDecX + 2 * kDecSF;  // 20 KB (1 KB aligned)
constexpr int kDecRB = 128 * 32;                // R tile: 128 rows x 32 B
constexpr int dec_smem(int stages) { return 1024 + stages * kDecStage + kDecRB + 512 + 256; }
constexpr int kDecSmem = dec_smem(kDecStagesDefault);
static_assert(kDecStage % 1024 == 0, "stage alignment");

struct DecodeMaps {
  CUtensorMap w, x, sfw, sfx, r, sfr;
};

struct DecodeParams {
  int M, N, K, r;
  int k_steps;          // 256-K steps in K
  int splits;           // K splits per weight tile
  int kc_pad, kc_pad_r; // SF chunks per 128-row block (weights / R); X uses kc_pad too
  int w_ksteps;         // pre-tiled weights: [N/128][w_ksteps][128 x 128 B]
  long long* dbg_ts;    // diagnostics (SERQ_DIAG_TS builds): per-CTA globaltimer stamps
  float* ws;            // [splits][N_pad][16] fp32 partials
  int* counters;        // [N/128] arrival counters (self-resetting)
  __nv_bfloat16* y;     // [M, ldy]
  int64_t ldy;
};

template <int kDecStages>
__global__ void __launch_bounds__(128, 1) serq_mx_decode_kernel(const __grid_constant__ DecodeMaps maps,
                                                                const DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* rbuf = smem + kDecStages * kDecStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rbuf + kDecRB + 512);
  uint64_t* full = bars;                   // [kDecStages]
  uint64_t* empty = bars + kDecStages;     // [kDecStages]
  uint64_t* rfull = bars + 2 * kDecStages;
  uint64_t* done = bars + 2 * kDecStages + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kDecStages + 2);
  __shared__ int s_last;

#ifdef SERQ_DIAG_TS
  uint64_t gt_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_entry));
#endif
  const uint32_t warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;             // 128 weight rows
  const int split = blockIdx.y;
  const int n0 = tile * 128;
  // this split's K steps
  const int per = (p.k_steps + p.splits - 1) / p.splits;
  const int s0 = split * per;
  const int s1 = min(p.k_steps, s0 + per);
  const int nsteps = max(0, s1 - s0);
  const bool with_r = p.r > 0 && split == 0;

  if (warp == 0 && elect_one()) {
    tma_prefetch(&maps.w);
    tma_prefetch(&maps.x);
    for (int s = 0; s < kDecStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(rfull, 1);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<64>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // [0,16) accumulator, [16,24) SFA, [24,32) SFB, [32,40) R SFA

  if (warp == 0) {
    if (elect_one()) {
      // Weights do not depend on the previous kernel (the quantizer): stream the
      // first min(nsteps, stages) weight tiles BEFORE griddepcontrol.wait, then
      // the activation tiles once the quantizer's output is visible.
      if (with_r) {
        mbar_expect_tx(rfull, kDecRB + 512);
        tma_load_2d(rbuf, &maps.r, rfull, 0, n0, kEvictFirst);
        tma_load_2d(rbuf + kDecRB, &maps.sfr, rfull, 0, (tile * p.kc_pad_r) * 4, kEvictFirst);
      }
      const int pre = min(nsteps, kDecStages);
      for (int i = 0; i < pre; ++i) {
        uint8_t* st = smem + i * kDecStage;
        const int kk = s0 + i;
        mbar_expect_tx(&full[i], kDecStage);
        tma_load_2d(st, &maps.w, &full[i], 0, (tile * p.w_ksteps + kk) * 128, kEvictFirst);
        tma_load_2d(st + kDecW + kDecX, &maps.sfw, &full[i], 0, (tile * p.kc_pad + 2 * kk) * 4, kEvictFirst);
      }
      pdl_wait();
      for (int i = 0; i < nsteps; ++i) {
        const int s = i % kDecStages;
        uint8_t* st = smem + s * kDecStage;
        const int kk = s0 + i;
        if (i >= pre) {
          mbar_wait(&empty[s], ((i / kDecStages) & 1) ^ 1);
          mbar_expect_tx(&full[s], kDecStage);
          tma_load_2d(st, &maps.w, &full[s], 0, (tile * p.w_ksteps + kk) * 128, kEvictFirst);
          tma_load_2d(st + kDecW + kDecX, &maps.sfw, &full[s], 0, (tile * p.kc_pad + 2 * kk) * 4, kEvictFirst);
        }
        tma_load_2d(st + kDecW, &maps.x, &full[s], kk * kStepBytes, 0, kEvictLast);
        tma_load_2d(st + kDecW + kDecX + kDecSF, &maps.sfx, &full[s], 0, (2 * kk) * 4, kEvictLast);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id0 = idesc_mxf4(128, kDecN), id1 = id0 | (2u << 4) | (2u << 29);
    const uint32_t acc = tmem, sfa = tmem + 16, sfb = tmem + 24, sfr = tmem + 32;
    for (int i = 0; i < nsteps; ++i) {
      const int s = i % kDecStages;
      mbar_wait(&full[s], (i / kDecStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t st = smem_u32(smem + s * kDecStage);
        const uint64_t a = make_sdesc(st, 16, 1024, 2), b = make_sdesc(st + kDecW, 16, 1024, 2);
        const uint32_t sa = st + kDecW + kDecX, sb = sa + kDecSF;
        tmem_cp_32x128b_x4(sfa, make_sdesc(sa, 128, 128, 0));
        tmem_cp_32x128b_x4(sfa + 4, make_sdesc(sa + 512, 128, 128, 0));
        tmem_cp_32x128b_x4(sfb, make_sdesc(sb, 128, 128, 0));
        tmem_cp_32x128b_x4(sfb + 4, make_sdesc(sb + 512, 128, 128, 0));
        const uint32_t first = i > 0 ? 1u : 0u;
        mma_mxf4(acc, a, b, id0, sfa, sfb, first);
        mma_mxf4(acc, a + 2, b + 2, id1, sfa | (2u << 30), sfb | (2u << 30), 1u);
        mma_mxf4(acc, a + 4, b + 4, id0, sfa + 4, sfb + 4, 1u);
        mma_mxf4(acc, a + 6, b + 6, id1, (sfa + 4) | (2u << 30), (sfb + 4) | (2u << 30), 1u);
        if (with_r && i == 0) {
          // salient term: A = R rows (K = r = 64), B = K-tile 0 of X (this stage), SFB = X chunk 0
          mbar_wait(rfull, 0);
          tc_fence_after();
          tmem_cp_32x128b_x4(sfr, make_sdesc(smem_u32(rbuf + kDecRB), 128, 128, 0));
          mma_mxf4(acc, make_sdesc(smem_u32(rbuf), 16, 256, 6), b, id0, sfr, sfb, 1u);
        }
        tc_commit(&empty[s]);
        if (i == nsteps - 1) tc_commit(done);
      }
      __syncwarp();
    }
    if (nsteps == 0 && elect_one()) mbar_arrive(done);
    __syncwarp();
  }
  // ------------------------------------------------ epilogue: all 4 warps
  pdl_wait();               // (no-op once satisfied) Y / workspace writes after the previous kernel
  pdl_launch_dependents();
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = threadIdx.x;  // TMEM lane = weight row within the tile
  uint32_t v[16];
  if (nsteps > 0) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((warp * 32u) << 16)));
    tmem_ld_wait();
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0u;
  }
  const int n = n0 + row;
  if (p.splits == 1) {
    if (n < p.N)
      for (int m = 0; m < p.M; ++m) p.y[m * p.ldy + n] = __float2bfloat16_rn(__uint_as_float(v[m]));
  } else {
    // publish this split's partial, then the last CTA of the tile reduces in split order
    float4* dst = reinterpret_cast<float4*>(p.ws + (size_t(split) * gridDim.x * 128 + size_t(n0 + row)) * kDecN);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                           __uint_as_float(v[4 * j + 3]));
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int prev = atomicAdd(&p.counters[tile], 1);
      s_last = prev == p.splits - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      float acc[kDecN];
#pragma unroll
      for (int m = 0; m < kDecN; ++m) acc[m] = 0.f;
      for (int sp = 0; sp < p.splits; ++sp) {
        const float4* src =
            reinterpret_cast<const float4*>(p.ws + (size_t(sp) * gridDim.x * 128 + size_t(n0 + row)) * kDecN);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 t = __ldcg(src + j);
          acc[4 * j] += t.x;
          acc[4 * j + 1] += t.y;
          acc[4 * j + 2] += t.z;
          acc[4 * j + 3] += t.w;
        }
      }
      if (n < p.N)
        for (int m = 0; m < p.M; ++m) p.y[m * p.ldy + n] = __float2bfloat16_rn(acc[m]);
      if (threadIdx.x == 0) p.counters[tile] = 0;  // ready for the next launch
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
#ifdef SERQ_DIAG_TS
  if (p.dbg_ts && threadIdx.x == 0) {
    uint64_t gt_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_exit));
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    if (cta < 1024) {
      p.dbg_ts[2 * cta] = (long long)gt_entry;
      p.dbg_ts[2 * cta + 1] = (long long)gt_exit;
    }
  }
#endif
}

}  // namespace serq
