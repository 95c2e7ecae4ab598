// serq_gemm_mx2.cuh -- MXFP4 SERQ linear on CTA PAIRS (tcgen05 cta_group::2).
//
// A cluster of 2 CTAs (one TPC) computes a 256 x 256 output tile with one
// tcgen05.mma.cta_group::2 (M=256, N=256, K=64) per 64-wide K slice, issued by
// the leader CTA.  Each CTA stages its own 128 rows of A and its own 128-row
// half of B (plus the scale factors the MMA reads from its TMEM: own 128 rows
// of SFA, all 256 columns of SFB), so a pipeline stage is 35 KB per SM instead
// of 51 KB and six stages fit.  All TMA loads of both CTAs complete on the
// leader's full barrier; MMA completion is multicast to both CTAs' barriers.
//
// TMEM per CTA: two OVERLAPPING 128x256 fp32 accumulators ([0,256) and
// [192,448)) and two scale-factor slots in [448,496) -- the epilogue of tile i
// drains the 64 overlapping columns first, then the MMAs of tile i+1 start.
// The SERQ salient term (compensate.py:335-340) is r/64 extra MMAs per tile
// into the same accumulator.
#pragma once
#include "serq_gemm_mx.cuh"

namespace serq {

constexpr int k2Stages = 6;
constexpr int k2SmemA = 128 * kStepBytes;  // own 128 rows
constexpr int k2SmemB = 128 * kStepBytes;  // own half of the 256-wide N tile
constexpr int k2SmemSFA = 1024;            // own rows, 2 SF chunks
constexpr int k2SmemSFB = 2048;            // all 256 columns, 2 chunks
constexpr int k2StageBytes = k2SmemA + k2SmemB + k2SmemSFA + k2SmemSFB;  // 35 KB
static_assert(k2StageBytes % 1024 == 0, "stage must keep 1 KB alignment");
constexpr int k2EpiStage = 32 * 64;  // per epilogue warp: 32 rows x 32 bf16 (64B-swizzled box)
constexpr int k2SmemBytes = 1024 + k2Stages * k2StageBytes + 4 * k2EpiStage + 256;
static_assert(k2SmemBytes <= 232448, "exceeds the 227 KB dynamic shared memory limit");

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank`
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(saddr), "r"(rank));
  return out;
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* m, uint32_t bar_cluster, int32_t c0,
                                                 int32_t c1, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(hint)
      : "memory");
}
__device__ __forceinline__ void mma_mxf4_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                              uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void tmem_cp_pair(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
// arrive on the barrier at this smem offset in BOTH CTAs once prior tcgen05 ops finish
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// Relaxed arrive: orders nothing but the preceding tcgen05.fence::before_thread_sync,
// which is all the TMEM hand-off needs (a release at cluster scope would wait for
// the warp's in-flight TMA-store traffic: ~1000+ cycles measured).
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

struct Pair2Maps {
  CUtensorMap a, b, xs, r, y, sfa, sfb, sfxs, sfr;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    serq_mx_pair_kernel(const __grid_constant__ Pair2Maps maps, const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + k2Stages * k2StageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + 4 * k2EpiStage);
  uint64_t* full = bars;                          // leader's are used
  uint64_t* empty = bars + k2Stages;              // both
  uint64_t* tmem_full = bars + 2 * k2Stages;      // [2], both
  uint64_t* tmem_empty = bars + 2 * k2Stages + 2; // leader's is used (8 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * k2Stages + 3);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const int tiles_m = (p.M + 255) / 256;
  const int tiles_n = (p.N + kBN - 1) / kBN;
  const int n_tiles = tiles_m * tiles_n;
  const bool has_r = p.r > 0;

  if (warp == 0 && elect_one()) {
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.b);
    tma_prefetch(&maps.y);
    tma_prefetch(&maps.sfa);
    tma_prefetch(&maps.sfb);
    if (has_r) {
      tma_prefetch(&maps.xs);
      tma_prefetch(&maps.r);
      tma_prefetch(&maps.sfxs);
      tma_prefetch(&maps.sfr);
    }
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full[0], 1);
    mbar_init(&tmem_full[1], 1);
    mbar_init(tmem_empty, (SERQ_DBG(p.dbg, 256)) ? 4 : 8);  // dbg 256: timing only, leader epilogue alone
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x == 0 && *tmem_slot != 0) __trap();  // accumulator addresses below assume column 0

  const int my_tiles = cluster_id < n_tiles ? (n_tiles - 1 - cluster_id) / n_clusters + 1 : 0;
  const int kpairs = p.k_steps >> 1;
  const bool kodd = p.k_steps & 1;
  const int r_steps = has_r ? p.r_steps : 0;
  const int n_iters = p.k_steps + r_steps;

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (elect_one()) {
      const uint32_t smem_base = smem_u32(smem);
      uint32_t g = 0;
      for (int i = 0; i < my_tiles; ++i) {
        const int tile = cluster_id + i * n_clusters;
        const int mt = tile % tiles_m, nt = tile / tiles_m;
        const int m_own = mt * 256 + int(rank) * 128;
        const int n0 = nt * kBN;
        const int n_half = n0 + int(rank) * 128;
        const int mblk = m_own / 128;
        for (int it = 0; it < n_iters; ++it, ++g) {
          const int s = g % k2Stages;
          mbar_wait(&empty[s], ((g / k2Stages) & 1) ^ 1);
          const uint32_t st = smem_base + s * k2StageBytes;
          const uint32_t fbar = map_rank(smem_u32(&full[s]), 0);
          if (SERQ_DBG(p.dbg, 1)) {
            if (leader) mbar_arrive(&full[s]);
            continue;
          }
          if (leader) mbar_expect_tx(&full[s], 2 * k2StageBytes);
          const bool rstep = it >= p.k_steps;
          const int kk = rstep ? it - p.k_steps : it;
          const CUtensorMap* ma = rstep && !p.xs_is_x ? &maps.xs : &maps.a;
          const CUtensorMap* mb = rstep ? &maps.r : &maps.b;
          const CUtensorMap* msa = rstep && !p.xs_is_x ? &maps.sfxs : &maps.sfa;
          const CUtensorMap* msb = rstep ? &maps.sfr : &maps.sfb;
          const int kca = rstep && !p.xs_is_x ? p.kc_pad_r : p.kc_pad;
          const int kcb = rstep ? p.kc_pad_r : p.kc_pad;
          tma_load_2d_pair(st, ma, fbar, kk * kStepBytes, m_own, kEvictNormal);
          if (rstep)
            tma_load_2d_pair(st + k2SmemA, mb, fbar, kk * kStepBytes, n_half, kEvictNormal);
          else
            tma_load_2d_pair(st + k2SmemA, mb, fbar, 0, ((n_half >> 7) * p.w_ksteps + kk) * 128, kEvictNormal);
          // scale factors: 1 KB (8 rows of 128 B) per 128-row block and 256-K step
          tma_load_2d_pair(st + k2SmemA + k2SmemB, msa, fbar, 0, (mblk * kca + 2 * kk) * 4, kEvictNormal);
          tma_load_2d_pair(st + k2SmemA + k2SmemB + k2SmemSFA, msb, fbar, 0, ((n0 / 128) * kcb + 2 * kk) * 4,
                           kEvictNormal);
          tma_load_2d_pair(st + k2SmemA + k2SmemB + k2SmemSFA + 1024, msb, fbar, 0,
                           ((n0 / 128 + 1) * kcb + 2 * kk) * 4, kEvictNormal);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      const int rbytes = p.r / 2;
      // the salient term's single K step (r <= 256) rides in the tile's last
      // pair (a 3-stage unit) instead of paying a unit of issue overhead alone
      const bool fold_r = r_steps == 1 && !kodd && kpairs > 0;
      const int units = kpairs + (kodd ? 1 : 0) + (fold_r ? 0 : r_steps);
      const int r_nk = has_r ? ((rbytes - (r_steps - 1) * kStepBytes) + 31) / 32 : 0;
      const uint32_t smem_base = smem_u32(smem);
      constexpr uint32_t id0 = idesc_mxf4(256, kBN), id1 = id0 | (2u << 4) | (2u << 29);
      auto unit_stages = [&](int uu) { return uu < kpairs ? ((fold_r && uu == kpairs - 1) ? 3 : 2) : 1; };
      auto wait_unit = [&](uint32_t gg, int uu) {
        const int n = unit_stages(uu);
        mbar_wait(&full[gg % k2Stages], (gg / k2Stages) & 1);
        if (n > 1) mbar_wait(&full[(gg + 1) % k2Stages], ((gg + 1) / k2Stages) & 1);
        if (n > 2) mbar_wait(&full[(gg + 2) % k2Stages], ((gg + 2) / k2Stages) & 1);
        tc_fence_after();
      };
      auto cps = [&](uint32_t st, uint32_t fa, uint32_t fb) {
        const uint32_t sa = st + k2SmemA + k2SmemB, sb = sa + k2SmemSFA;
        tmem_cp_pair(fa, make_sdesc(sa, 128, 128, 0));
        tmem_cp_pair(fa + 4, make_sdesc(sa + 512, 128, 128, 0));
        tmem_cp_pair(fb, make_sdesc(sb, 128, 128, 0));
        tmem_cp_pair(fb + 4, make_sdesc(sb + 1024, 128, 128, 0));
        tmem_cp_pair(fb + 8, make_sdesc(sb + 512, 128, 128, 0));
        tmem_cp_pair(fb + 12, make_sdesc(sb + 1536, 128, 128, 0));
      };
      uint32_t g = 0;
#ifdef SERQ_DIAG_TS
      uint64_t gt0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
      const long long ck0 = clock64();
      int ustamp = 0;
#endif
      if (my_tiles > 0) wait_unit(0, 0);
      for (int i = 0; i < my_tiles; ++i) {
        const uint32_t acc = (i & 1) ? kAccB1 : 0u;
        if (i > 0 && !(SERQ_DBG(p.dbg, 8))) {
          mbar_wait(tmem_empty, (i - 1) & 1);  // both epilogues drained the overlapping columns
          tc_fence_after();
        }
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && blockIdx.x == 0 && i < 8 && lane_id() == 0) p.dbg_ts[460 + i] = clock64();
#endif
        for (int uu = 0; uu < units; ++uu) {
          const bool pair = uu < kpairs;
          const int len = unit_stages(uu);
          const bool triple = len == 3;
          const bool last_unit = uu == units - 1;
          int nk1 = 4;
          if (!pair && uu >= kpairs + (kodd ? 1 : 0)) {
            const int rem = rbytes - (uu - kpairs - (kodd ? 1 : 0)) * kStepBytes;
            nk1 = rem >= kStepBytes ? 4 : (rem + 31) / 32;
          }
          const uint32_t s0 = g % k2Stages, s1 = (g + 1) % k2Stages;
          const uint32_t st0 = smem_base + s0 * k2StageBytes, st1 = smem_base + s1 * k2StageBytes;
          const uint64_t a0 = make_sdesc(st0, 16, 1024, 2), b0 = make_sdesc(st0 + k2SmemA, 16, 1024, 2);
          const uint64_t a1 = make_sdesc(st1, 16, 1024, 2), b1 = make_sdesc(st1 + k2SmemA, 16, 1024, 2);
          const uint32_t fa0 = kSfBase + (g & 1) * kSfCols, fb0 = fa0 + 8;
          const uint32_t fa1 = kSfBase + ((g + 1) & 1) * kSfCols, fb1 = fa1 + 8;
          const uint32_t first = uu > 0 ? 1u : 0u;
          const bool do_cp = !(SERQ_DBG(p.dbg, 4));
#ifdef SERQ_DIAG_TS
          const bool stamp = p.dbg_ts && blockIdx.x == 0 && ustamp < 100 && lane_id() == 0;
          if (stamp) p.dbg_ts[4 * ustamp] = clock64();
#endif
          if (elect_one()) {
            if (do_cp) cps(st0, fa0, fb0);
            if (pair) {
              mma_mxf4_pair(acc, a0, b0, id0, fa0, fb0, first);
              mma_mxf4_pair(acc, a0 + 2, b0 + 2, id1, fa0 | (2u << 30), fb0 | (2u << 30), 1u);
              mma_mxf4_pair(acc, a0 + 4, b0 + 4, id0, fa0 + 4, fb0 + 8, 1u);
              mma_mxf4_pair(acc, a0 + 6, b0 + 6, id1, (fa0 + 4) | (2u << 30), (fb0 + 8) | (2u << 30), 1u);
              tc_commit_pair(&empty[s0]);
              if (do_cp) cps(st1, fa1, fb1);
              mma_mxf4_pair(acc, a1, b1, id0, fa1, fb1, 1u);
              mma_mxf4_pair(acc, a1 + 2, b1 + 2, id1, fa1 | (2u << 30), fb1 | (2u << 30), 1u);
              mma_mxf4_pair(acc, a1 + 4, b1 + 4, id0, fa1 + 4, fb1 + 8, 1u);
              if (triple) {
                // finish stage 1, then the salient step (stage 2) into the same accumulator
                mma_mxf4_pair(acc, a1 + 6, b1 + 6, id1, (fa1 + 4) | (2u << 30), (fb1 + 8) | (2u << 30), 1u);
                tc_commit_pair(&empty[s1]);
                const uint32_t s2 = (g + 2) % k2Stages, st2 = smem_base + s2 * k2StageBytes;
                const uint64_t a2 = make_sdesc(st2, 16, 1024, 2), b2 = make_sdesc(st2 + k2SmemA, 16, 1024, 2);
                if (do_cp) cps(st2, fa0, fb0);  // slot of stage 0 (its MMAs were issued before)
                for (int j = 0; j + 1 < r_nk; ++j) {
                  const uint32_t sfid = (j & 1) * 2;
                  mma_mxf4_pair(acc, a2 + 2 * j, b2 + 2 * j, (j & 1) ? id1 : id0, (fa0 + (j >> 1) * 4) | (sfid << 30),
                                (fb0 + (j >> 1) * 8) | (sfid << 30), 1u);
                }
              }
            } else {
              for (int j = 0; j + 1 < nk1; ++j) {
                const uint32_t sfid = (j & 1) * 2;
                mma_mxf4_pair(acc, a0 + 2 * j, b0 + 2 * j, (j & 1) ? id1 : id0, (fa0 + (j >> 1) * 4) | (sfid << 30),
                              (fb0 + (j >> 1) * 8) | (sfid << 30), (first || j > 0) ? 1u : 0u);
              }
            }
          }
          __syncwarp();
#ifdef SERQ_DIAG_TS
          if (stamp) p.dbg_ts[4 * ustamp + 1] = clock64();
#endif
          const uint32_t gn = g + len;
          if (!last_unit)
            wait_unit(gn, uu + 1);
          else if (i + 1 < my_tiles)
            wait_unit(gn, 0);
#ifdef SERQ_DIAG_TS
          if (stamp) p.dbg_ts[4 * ustamp + 2] = clock64();
#endif
          if (elect_one()) {
            if (triple) {
              const uint32_t s2 = (g + 2) % k2Stages, st2 = smem_base + s2 * k2StageBytes;
              const uint64_t a2 = make_sdesc(st2, 16, 1024, 2), b2 = make_sdesc(st2 + k2SmemA, 16, 1024, 2);
              const int j = r_nk - 1;
              const uint32_t sfid = (j & 1) * 2;
              mma_mxf4_pair(acc, a2 + 2 * j, b2 + 2 * j, (j & 1) ? id1 : id0, (fa0 + (j >> 1) * 4) | (sfid << 30),
                            (fb0 + (j >> 1) * 8) | (sfid << 30), 1u);
              tc_commit_pair(&empty[s2]);
            } else if (pair) {
              mma_mxf4_pair(acc, a1 + 6, b1 + 6, id1, (fa1 + 4) | (2u << 30), (fb1 + 8) | (2u << 30), 1u);
              tc_commit_pair(&empty[s1]);
            } else {
              const int j = nk1 - 1;
              const uint32_t sfid = (j & 1) * 2;
              mma_mxf4_pair(acc, a0 + 2 * j, b0 + 2 * j, (j & 1) ? id1 : id0, (fa0 + (j >> 1) * 4) | (sfid << 30),
                            (fb0 + (j >> 1) * 8) | (sfid << 30), (first || j > 0) ? 1u : 0u);
              tc_commit_pair(&empty[s0]);
            }
            if (last_unit) tc_commit_pair(&tmem_full[i & 1]);
          }
          __syncwarp();
#ifdef SERQ_DIAG_TS
          if (stamp) p.dbg_ts[4 * ustamp + 3] = clock64();
          ++ustamp;
#endif
          g = gn;
        }
      }
#ifdef SERQ_DIAG_TS
      if (p.dbg_ts && blockIdx.x == 0 && lane_id() == 0) {
        uint64_t gt1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
        p.dbg_ts[508] = ck0;
        p.dbg_ts[509] = clock64();
        p.dbg_ts[510] = (long long)gt0;
        p.dbg_ts[511] = (long long)gt1;
      }
#endif
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const uint32_t q = warp & 3;
    const uint32_t lane_base = (q * 32u) << 16;
    uint8_t* stage_out = epi_smem + q * k2EpiStage;
    const uint32_t rbase = smem_u32(stage_out) + lane_id() * 64;
    const uint32_t sw = (lane_id() >> 1) & 3;  // 64B swizzle: 16-B chunk ^= (row / 2) % 4
    const uint32_t tmem_empty_leader = map_rank(smem_u32(tmem_empty), 0);
    for (int i = 0; i < my_tiles; ++i) {
      const int tile = cluster_id + i * n_clusters;
      const int mt = tile % tiles_m, nt = tile / tiles_m;
      const int m_own = mt * 256 + int(rank) * 128;
      const int n0 = nt * kBN;
      const uint32_t b = i & 1;
#ifdef SERQ_DIAG_TS
      const bool est = p.dbg_ts && blockIdx.x == 0 && i < 8 && lane_id() == 0 && q == 0;
      if (est) p.dbg_ts[420 + 4 * i] = clock64();
#endif
      mbar_wait(&tmem_full[b], (i >> 1) & 1);
      tc_fence_after();
#ifdef SERQ_DIAG_TS
      if (est) p.dbg_ts[421 + 4 * i] = clock64();
#endif
      const uint32_t acc = (b ? kAccB1 : 0u) + lane_base;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        const int c = b ? cc : (cc + 3) & 3;  // the chunk shared with the other accumulator first
        uint32_t v[32], w[32];
        tmem_ld_32x32b_x32(acc + c * 64, v);
        tmem_ld_32x32b_x32(acc + c * 64 + 32, w);
        tmem_ld_wait();
        if (cc == 0) {
#ifdef SERQ_DIAG_TS
          if (est) p.dbg_ts[422 + 4 * i] = clock64();
#endif
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0 && (leader || !(SERQ_DBG(p.dbg, 256)))) mbar_arrive_cluster_relaxed(tmem_empty_leader);
#ifdef SERQ_DIAG_TS
          if (est) p.dbg_ts[423 + 4 * i] = clock64();
#endif
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* src = h ? w : v;
          if (lane_id() == 0) bulk_wait_read_all();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            st_shared_v4(rbase + ((uint32_t(j) ^ sw) * 16),
                         pack_bf16x2(__uint_as_float(src[8 * j]), __uint_as_float(src[8 * j + 1])),
                         pack_bf16x2(__uint_as_float(src[8 * j + 2]), __uint_as_float(src[8 * j + 3])),
                         pack_bf16x2(__uint_as_float(src[8 * j + 4]), __uint_as_float(src[8 * j + 5])),
                         pack_bf16x2(__uint_as_float(src[8 * j + 6]), __uint_as_float(src[8 * j + 7])));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane_id() == 0 && !(SERQ_DBG(p.dbg, 2)) && m_own < p.M) {
            tma_store_2d(&maps.y, stage_out, n0 + c * 64 + h * 32, m_own + q * 32);
            bulk_commit();
          }
        }
      }
    }
    if (lane_id() == 0) bulk_wait_all();
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(0u));
  }
}

}  // namespace serq
