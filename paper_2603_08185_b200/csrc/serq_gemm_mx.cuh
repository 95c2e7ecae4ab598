// serq_gemm_mx.cuh -- persistent MXFP4 SERQ linear (the C2 hot kernel).
//
// One CTA per SM walks output tiles t = blockIdx.x + i * gridDim.x.  TMEM holds
// two OVERLAPPING 128x256 fp32 accumulators (columns [0,256) and [192,448))
// plus scale-factor slots in [448,512): the epilogue of tile i first drains the
// 64 columns the next accumulator reuses, releases them to the MMA warp, and
// converts / stores the remaining 192 columns while the MMAs of tile i+1 run.
// The salient term (compensate.py:335-340) is r/64 extra MMAs per tile into the
// same accumulator.
#pragma once
#include "serq_gemm.cuh"

namespace serq {

constexpr int kPStages = 4;
constexpr int kEpiStage = 32 * 128;  // per epilogue warp: 32 rows x 64 bf16 (one 128B-swizzled box)
constexpr int kPSmemBytes = 1024 + kPStages * kStageBytes + 4 * kEpiStage + 256;
constexpr uint32_t kAccB1 = 192;  // column base of the second accumulator
constexpr uint32_t kSfBase = 448;

__global__ void __launch_bounds__(kThreads, 1)
    serq_mx_persistent_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                              const __grid_constant__ CUtensorMap map_xs, const __grid_constant__ CUtensorMap map_r,
                              const __grid_constant__ CUtensorMap map_y, const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + kPStages * kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + 4 * kEpiStage);
  uint64_t* full = bars;
  uint64_t* empty = bars + kPStages;
  uint64_t* tmem_full = bars + 2 * kPStages;  // [2]
  uint64_t* tmem_empty = bars + 2 * kPStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kPStages + 3);

  const uint32_t warp = threadIdx.x >> 5;
  const int tiles_m = (p.M + kBM - 1) / kBM;
  const int tiles_n = (p.N + kBN - 1) / kBN;
  const int n_tiles = tiles_m * tiles_n;
  const bool has_r = p.r > 0;
  const int n_iters = p.k_steps + (has_r ? p.r_steps : 0);

  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    tma_prefetch(&map_y);
    if (has_r) {
      tma_prefetch(&map_xs);
      tma_prefetch(&map_r);
    }
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full[0], 1);
    mbar_init(&tmem_full[1], 1);
    mbar_init(tmem_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // a full 512-column allocation always starts at lane 0 / column 0, so the
  // accumulator and scale-factor addresses are compile-time constants
  const uint32_t tmem_base = 0;
  if (threadIdx.x == 0 && *tmem_slot != 0) __trap();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      uint32_t g = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int m0 = (tile % tiles_m) * kBM;
        const int n0 = (tile / tiles_m) * kBN;
        const int mblk = m0 / 128;
        for (int it = 0; it < n_iters; ++it, ++g) {
          const int s = g % kPStages;
          const uint32_t ph = (g / kPStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * kStageBytes;
          const bool rstep = it >= p.k_steps;
          const int kk = rstep ? it - p.k_steps : it;
          if (SERQ_DBG(p.dbg, 1)) {
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_expect_tx(&full[s], kStageBytes);
          if (!rstep) {
            tma_load_2d(st, &map_a, &full[s], kk * kStepBytes, m0, kEvictNormal);
            tma_load_2d(st + kSmemA, &map_b, &full[s], 0, ((n0 >> 7) * p.w_ksteps + kk) * 128, kEvictNormal);
            tma_load_2d(st + kSmemA + 128 * kStepBytes, &map_b, &full[s], 0, ((n0 >> 7) * p.w_ksteps + p.w_ksteps + kk) * 128,
                        kEvictNormal);
          } else {
            tma_load_2d(st, p.xs_is_x ? &map_a : &map_xs, &full[s], kk * kStepBytes, m0, kEvictNormal);
            tma_load_2d(st + kSmemA, &map_r, &full[s], kk * kStepBytes, n0, kEvictNormal);
          }
          const uint8_t* sa = rstep ? p.sfa_r : p.sfa;
          const uint8_t* sb = rstep ? p.sfb_r : p.sfb;
          const int kca = rstep && !p.xs_is_x ? p.kc_pad_r : p.kc_pad;
          const int kcb = rstep ? p.kc_pad_r : p.kc_pad;
          bulk_load(st + kSmemA + kSmemB, sa + (size_t(mblk) * kca + 2 * kk) * 512, 1024, &full[s]);
#pragma unroll
          for (int b = 0; b < kBN / 128; ++b)
            bulk_load(st + kSmemA + kSmemB + kSmemSFA + b * 1024, sb + (size_t(n0 / 128 + b) * kcb + 2 * kk) * 512,
                      1024, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Everything the tcgen05 instructions consume is computed in warp-uniform
    // code (TMEM base is the constant 0, descriptors derive from the loop
    // counters), so operands sit in uniform registers.  Main K steps are
    // consumed in PAIRS: one look-ahead wait per 8 MMAs, placed before the
    // unit's last MMA so the tensor pipe keeps queued work while this thread
    // sits in mbarrier.try_wait; each stage is still released by its own commit.
    const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int rbytes = p.r / 2;
    const int kpairs = p.k_steps >> 1;
    const bool kodd = p.k_steps & 1;
    const int r_steps = has_r ? p.r_steps : 0;
    // units per tile: kpairs pairs, then [odd main step], then r_steps singles
    const int units = kpairs + (kodd ? 1 : 0) + r_steps;
    const uint32_t smem_base = smem_u32(smem);
    constexpr uint32_t id0 = idesc_mxf4(kBM, kBN), id1 = id0 | (2u << 4) | (2u << 29);  // sf_id 0 / 2
    uint32_t g = 0;
    auto wait_unit = [&](uint32_t gg, int uu) {
      // stages of unit uu (within a tile) starting at global stage gg
      mbar_wait(&full[gg & (kPStages - 1)], (gg / kPStages) & 1);
      if (uu < kpairs) mbar_wait(&full[(gg + 1) & (kPStages - 1)], ((gg + 1) / kPStages) & 1);
      tc_fence_after();
    };
    if (my_tiles > 0) wait_unit(0, 0);
    for (int i = 0; i < my_tiles; ++i) {
      const uint32_t acc = (i & 1) ? kAccB1 : 0u;
      if (i > 0 && !(SERQ_DBG(p.dbg, 8))) {
        mbar_wait(tmem_empty, (i - 1) & 1);  // epilogue i-1 drained the overlapping columns
        tc_fence_after();
      }
      for (int uu = 0; uu < units; ++uu) {
        const bool pair = uu < kpairs;
        const int len = pair ? 2 : 1;
        const bool last_unit = uu == units - 1;
        // slices in a single (odd main or R) step
        int nk1 = 4;
        if (!pair && uu >= kpairs + (kodd ? 1 : 0)) {
          const int rem = rbytes - (uu - kpairs - (kodd ? 1 : 0)) * kStepBytes;
          nk1 = rem >= kStepBytes ? 4 : (rem + 31) / 32;
        }
        const uint32_t s0 = g & (kPStages - 1), s1 = (g + 1) & (kPStages - 1);
        const uint32_t st0 = smem_base + s0 * kStageBytes, st1 = smem_base + s1 * kStageBytes;
        const uint64_t a0 = make_sdesc(st0, 16, 1024, 2), b0 = make_sdesc(st0 + kSmemA, 16, 1024, 2);
        const uint64_t a1 = make_sdesc(st1, 16, 1024, 2), b1 = make_sdesc(st1 + kSmemA, 16, 1024, 2);
        const uint32_t fa0 = kSfBase + (g & 1) * kSfCols, fb0 = fa0 + 8;
        const uint32_t fa1 = kSfBase + ((g + 1) & 1) * kSfCols, fb1 = fa1 + 8;
        const uint32_t first = uu > 0 ? 1u : 0u;
        const bool do_cp = !(SERQ_DBG(p.dbg, 4));
        if (elect_one()) {
          if (do_cp) {
            const uint32_t sa = st0 + kSmemA + kSmemB, sb = sa + kSmemSFA;
            tmem_cp_32x128b_x4(fa0, make_sdesc(sa, 128, 128, 0));
            tmem_cp_32x128b_x4(fa0 + 4, make_sdesc(sa + 512, 128, 128, 0));
            tmem_cp_32x128b_x4(fb0, make_sdesc(sb, 128, 128, 0));
            tmem_cp_32x128b_x4(fb0 + 4, make_sdesc(sb + 1024, 128, 128, 0));
            tmem_cp_32x128b_x4(fb0 + 8, make_sdesc(sb + 512, 128, 128, 0));
            tmem_cp_32x128b_x4(fb0 + 12, make_sdesc(sb + 1536, 128, 128, 0));
          }
          if (pair) {
            mma_mxf4(acc, a0, b0, id0, fa0, fb0, first);
            mma_mxf4(acc, a0 + 2, b0 + 2, id1, fa0 | (2u << 30), fb0 | (2u << 30), 1u);
            mma_mxf4(acc, a0 + 4, b0 + 4, id0, fa0 + 4, fb0 + 8, 1u);
            mma_mxf4(acc, a0 + 6, b0 + 6, id1, (fa0 + 4) | (2u << 30), (fb0 + 8) | (2u << 30), 1u);
            tc_commit(&empty[s0]);
            if (do_cp) {
              const uint32_t sa = st1 + kSmemA + kSmemB, sb = sa + kSmemSFA;
              tmem_cp_32x128b_x4(fa1, make_sdesc(sa, 128, 128, 0));
              tmem_cp_32x128b_x4(fa1 + 4, make_sdesc(sa + 512, 128, 128, 0));
              tmem_cp_32x128b_x4(fb1, make_sdesc(sb, 128, 128, 0));
              tmem_cp_32x128b_x4(fb1 + 4, make_sdesc(sb + 1024, 128, 128, 0));
              tmem_cp_32x128b_x4(fb1 + 8, make_sdesc(sb + 512, 128, 128, 0));
              tmem_cp_32x128b_x4(fb1 + 12, make_sdesc(sb + 1536, 128, 128, 0));
            }
            mma_mxf4(acc, a1, b1, id0, fa1, fb1, 1u);
            mma_mxf4(acc, a1 + 2, b1 + 2, id1, fa1 | (2u << 30), fb1 | (2u << 30), 1u);
            mma_mxf4(acc, a1 + 4, b1 + 4, id0, fa1 + 4, fb1 + 8, 1u);
          } else {
            for (int j = 0; j + 1 < nk1; ++j) {
              const uint32_t sfid = (j & 1) * 2;
              mma_mxf4(acc, a0 + 2 * j, b0 + 2 * j, (j & 1) ? id1 : id0, (fa0 + (j >> 1) * 4) | (sfid << 30),
                       (fb0 + (j >> 1) * 8) | (sfid << 30), (first || j > 0) ? 1u : 0u);
            }
          }
        }
        __syncwarp();
        // look ahead to the next unit (this tile or the next one) while the pipe is busy
        const uint32_t gn = g + len;
        if (!last_unit)
          wait_unit(gn, uu + 1);
        else if (i + 1 < my_tiles)
          wait_unit(gn, 0);
        if (elect_one()) {
          if (pair) {
            mma_mxf4(acc, a1 + 6, b1 + 6, id1, (fa1 + 4) | (2u << 30), (fb1 + 8) | (2u << 30), 1u);
            tc_commit(&empty[s1]);
          } else {
            const int j = nk1 - 1;
            const uint32_t sfid = (j & 1) * 2;
            mma_mxf4(acc, a0 + 2 * j, b0 + 2 * j, (j & 1) ? id1 : id0, (fa0 + (j >> 1) * 4) | (sfid << 30),
                     (fb0 + (j >> 1) * 8) | (sfid << 30), (first || j > 0) ? 1u : 0u);
            tc_commit(&empty[s0]);
          }
          if (last_unit) tc_commit(&tmem_full[i & 1]);
        }
        __syncwarp();
        g = gn;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;
    const uint32_t lane_base = (q * 32u) << 16;
    uint8_t* stage_out = epi_smem + q * kEpiStage;
    const uint32_t rbase = smem_u32(stage_out) + lane_id() * 128;
    int i = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++i) {
      const int m0 = (tile % tiles_m) * kBM;
      const int n0 = (tile / tiles_m) * kBN;
      const uint32_t b = i & 1;
      mbar_wait(&tmem_full[b], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t acc = (b ? kAccB1 : 0u) + lane_base;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        // drain the 64-column chunk shared with the other accumulator first
        const int c = b ? cc : (cc + 3) & 3;
        uint32_t v[32], w[32];
        tmem_ld_32x32b_x32(acc + c * 64, v);
        tmem_ld_32x32b_x32(acc + c * 64 + 32, w);
        tmem_ld_wait();
        if (cc == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(tmem_empty);
        }
        const int row = m0 + int(q) * 32 + int(lane_id());
        if (p.addend && row < p.M) {  // the SVD baseline's fp32 correction (compensate.py:326-331)
          const float* ad = p.addend + size_t(row) * p.N + n0 + c * 64;
          // 16-B loads (N % 4 == 0, 16-B aligned rows: checked at the boundary); each lane reads
          // its row's 256 contiguous bytes
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (n0 + c * 64 + j < p.N) {
              const float4 a = __ldg(reinterpret_cast<const float4*>(ad + j));
              v[j] = __float_as_uint(__uint_as_float(v[j]) + a.x);
              v[j + 1] = __float_as_uint(__uint_as_float(v[j + 1]) + a.y);
              v[j + 2] = __float_as_uint(__uint_as_float(v[j + 2]) + a.z);
              v[j + 3] = __float_as_uint(__uint_as_float(v[j + 3]) + a.w);
            }
            if (n0 + c * 64 + 32 + j < p.N) {
              const float4 a = __ldg(reinterpret_cast<const float4*>(ad + 32 + j));
              w[j] = __float_as_uint(__uint_as_float(w[j]) + a.x);
              w[j + 1] = __float_as_uint(__uint_as_float(w[j + 1]) + a.y);
              w[j + 2] = __float_as_uint(__uint_as_float(w[j + 2]) + a.z);
              w[j + 3] = __float_as_uint(__uint_as_float(w[j + 3]) + a.w);
            }
          }
        }
        // the previous TMA store must have finished reading the staging box
        if (lane_id() == 0) bulk_wait_read_all();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t chunk = uint32_t(j) ^ (lane_id() & 7);
          st_shared_v4(rbase + chunk * 16, pack_bf16x2(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1])),
                       pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                       pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                       pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t chunk = uint32_t(j + 4) ^ (lane_id() & 7);
          st_shared_v4(rbase + chunk * 16, pack_bf16x2(__uint_as_float(w[8 * j]), __uint_as_float(w[8 * j + 1])),
                       pack_bf16x2(__uint_as_float(w[8 * j + 2]), __uint_as_float(w[8 * j + 3])),
                       pack_bf16x2(__uint_as_float(w[8 * j + 4]), __uint_as_float(w[8 * j + 5])),
                       pack_bf16x2(__uint_as_float(w[8 * j + 6]), __uint_as_float(w[8 * j + 7])));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0 && !(SERQ_DBG(p.dbg, 2))) {
          tma_store_2d(&map_y, stage_out, n0 + c * 64, m0 + q * 32);
          bulk_commit();
        }
      }
    }
    if (lane_id() == 0) bulk_wait_all();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace serq
