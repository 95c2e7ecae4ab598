// serq_gemm_mx3.cuh -- MXFP4 SERQ linear, CTA pairs, two-K-step pipeline slots
// and the salient term riding on K-step 0 (the production kernel for M > 128).
//
// Differences to serq_gemm_mx2.cuh (kept for the gather / large-r cases):
//  * a pipeline SLOT holds two 256-K steps (8 MMAs of 256x256x64) behind ONE
//    full and ONE empty barrier: the issuing thread pays one mbarrier wait and
//    one commit per 8 MMAs (each try_wait costs ~145 cycles even when complete);
//  * with the permuted salient layout the salient activation slice IS K-tile 0
//    of X, so only R's B tile (128 rows x r/2 bytes per CTA, 32- or
//    64-byte swizzle) and its scale factors are staged -- in a side buffer that
//    completes on the same barrier as K-step 0 -- and r/64 MMAs follow K-step
//    0's MMAs into the same accumulator.  No extra pipeline step, no second GEMM.
#pragma once
#include "serq_gemm_mx2.cuh"

namespace serq {

constexpr int k3Slots = 3;                    // 3 slots x 2 steps = 6 x 35 KB
constexpr int k3StepBytes = k2StageBytes;     // one 256-K step per CTA: A 16K, B 16K, SFA 1K, SFB 2K
constexpr int k3SlotBytes = 2 * k3StepBytes;  // 70 KB
constexpr int k3RB = 128 * 32;                // R B tile (r <= 64: 32 B per row) per CTA
constexpr int k3RSF = 1024;                   // R SFB: one chunk, both 128-row blocks
constexpr int k3SmemBytes = 1024 + k3Slots * k3SlotBytes + k3RB + k3RSF + 4 * k2EpiStage + 512;
static_assert(k3SmemBytes <= 232448, "exceeds the 227 KB dynamic shared memory limit");
// gather fallback (salient set not the permuted front): the salient term's A operand is the
// quantizer's x[:, idx] slice (128 rows x 32 B + one SF atom per CTA); the room comes from
// halving the epilogue staging boxes (32 rows x 16 columns, no swizzle)
constexpr int k3Xs = 128 * 32 + 512;
constexpr int k3EpiG = 32 * 32;
constexpr int k3SmemBytesG = 1024 + k3Slots * k3SlotBytes + k3RB + k3RSF + k3Xs + 4 * k3EpiG + 512;
static_assert(k3SmemBytesG <= 232448, "exceeds the 227 KB dynamic shared memory limit");

struct Pair3Maps {
  CUtensorMap a, b, r, y, sfa, sfb, sfr;
  CUtensorMap b64;       // narrow tiles: 64-row B boxes (each CTA's half of a 128-wide N tile)
  CUtensorMap xs, sfxs;  // gather: the quantizer's x[:, idx] codes (32-B rows, 32B swizzle) and scale factors
};

__device__ __forceinline__ void tma_load_2d_pair_nohint(uint32_t dst, const CUtensorMap* m, uint32_t bar, int32_t c0,
                                                        int32_t c1) {
  tma_load_2d_pair(dst, m, bar, c0, c1, kEvictNormal);
}

// kAddend: the SVD baseline's fp32 addend in the epilogue (compensate.py:326-331; r = 0 handles),
// a separate instantiation so the SERQ kernels carry none of it
template <bool kGather = false, bool kAddend = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    serq_mx_pair3_kernel(const __grid_constant__ Pair3Maps maps, const GemmParams p) {
  constexpr int kEpiBox = kGather ? k3EpiG : k2EpiStage;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* rbuf = smem + k3Slots * k3SlotBytes;  // R B tile (1 KB aligned) then R SFB
  uint8_t* xsbuf = rbuf + k3RB + k3RSF;          // gather: x[:, idx] A tile then its SF atom
  uint8_t* epi_smem = xsbuf + (kGather ? k3Xs : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + 4 * kEpiBox);
  uint64_t* full = bars;                        // [k3Slots] leader's used
  uint64_t* empty = bars + k3Slots;             // [k3Slots] both
  uint64_t* tmem_full = bars + 2 * k3Slots;     // [2] both
  uint64_t* tmem_empty = bars + 2 * k3Slots + 2;
  uint64_t* r_empty = bars + 2 * k3Slots + 3;   // R side buffer consumed (both)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * k3Slots + 4);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
#ifdef SERQ_DIAG_TS
  if (p.dbg_ts && threadIdx.x == 0) {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    p.dbg_ts[1024 + 148 * 24 + blockIdx.x * 2] = (long long)g;
  }
#endif
  const int n_clusters = gridDim.x >> 1;
  const int tiles_m = (p.M + 255) / 256;
  const int tiles_n = (p.N + kBN - 1) / kBN;
  const int n_tiles = tiles_m * tiles_n;
  const bool has_r = p.r > 0;
  const int units = (p.k_steps + 1) >> 1;       // slots per tile (last one may hold a single step)
  // work items: tiles [0, narrow_from) whole, then every remaining tile as two 256 x 128 tiles
  const int narrow_from = min(p.narrow_from, n_tiles);
  const int n_items = narrow_from + 2 * (n_tiles - narrow_from);
  struct Item {
    int tile, lo, hi;  // [lo, hi) = k-unit range
    int nsub;          // -1: 256 columns; 0 / 1: the first / second 128 columns only
  };
  // tile -> (M tile, N tile): M fastest, or grouped (group_m M-tiles x all N-tiles per group)
  auto tile_mn = [&](int tile, int& mt, int& nt) {
    if (p.group_m <= 0) {
      mt = tile % tiles_m;
      nt = tile / tiles_m;
      return;
    }
    const int per = p.group_m * tiles_n;
    const int g = tile / per, first = g * p.group_m;
    const int gs = min(p.group_m, tiles_m - first);
    const int w = tile - g * per;
    mt = first + w % gs;
    nt = w / gs;
  };
  auto item_of = [&](int w) {
    Item it;
    it.nsub = -1;
    it.tile = w;
    it.lo = 0;
    it.hi = units;
    if (w >= narrow_from) {
      const int j = w - narrow_from;
      it.tile = narrow_from + (j >> 1);
      it.nsub = j & 1;
    }
    return it;
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.b);
    tma_prefetch(&maps.y);
    tma_prefetch(&maps.sfa);
    tma_prefetch(&maps.sfb);
    if (has_r) {
      tma_prefetch(&maps.r);
      tma_prefetch(&maps.sfr);
      if (kGather) {
        tma_prefetch(&maps.xs);
        tma_prefetch(&maps.sfxs);
      }
    }
    for (int s = 0; s < k3Slots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full[0], 1);
    mbar_init(&tmem_full[1], 1);
    mbar_init(tmem_empty, 8);
    mbar_init(r_empty, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x == 0 && *tmem_slot != 0) __trap();

  const int my_tiles = cluster_id < n_items ? (n_items - 1 - cluster_id) / n_clusters + 1 : 0;

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (elect_one()) {
      const uint32_t smem_base = smem_u32(smem);
      const uint32_t rb = smem_u32(rbuf);
      uint32_t u = 0;  // global unit (slot use) counter
      int r_uses = 0;
      for (int i = 0; i < my_tiles; ++i) {
        const Item itm = item_of(cluster_id + i * n_clusters);
        const int tile = (SERQ_DBG(p.dbg, 16384)) ? 0 : itm.tile;  // diagnostics: every cluster streams tile 0
        int mt, nt;
        tile_mn(tile, mt, nt);
        const int m_own = mt * 256 + int(rank) * 128;
        const bool narrow = itm.nsub >= 0 && !(SERQ_DBG(p.dbg, 96));  // diagnostics 32 / 64: full-tile loads
        const int n0 = nt * kBN + (narrow ? itm.nsub * 128 : 0);
        const int n_half = n0 + int(rank) * (narrow ? 64 : 128);
        const int mblk = m_own / 128;
        for (int uu = itm.lo; uu < itm.hi; ++uu, ++u) {
          const int slot = u % k3Slots;
          mbar_wait(&empty[slot], ((u / k3Slots) & 1) ^ 1);
          const int k0 = 2 * uu;
          const int len = (k0 + 1 < p.k_steps) ? 2 : 1;
          const bool with_r = has_r && uu == 0;
          if (with_r && r_uses > 0) mbar_wait(r_empty, (r_uses - 1) & 1);  // previous R MMAs are done
          if (with_r) ++r_uses;
          const uint32_t fbar = map_rank(smem_u32(&full[slot]), 0);
          const bool no_sf = SERQ_DBG(p.dbg, 32768);  // diagnostics: skip scale-factor loads (request-count test)
          if (leader)
            mbar_expect_tx(&full[slot], 2u * (len * (k3StepBytes - (no_sf ? 3072 : 0) - (narrow ? 8192 + 1024 : 0)) +
                                              (with_r ? k3RB + k3RSF + (kGather ? k3Xs : 0) : 0)));
          const uint32_t st = smem_base + slot * k3SlotBytes;
          // weights (B, SFB) never depend on the previous kernel: load them first
          for (int h = 0; h < len; ++h) {
            const uint32_t ss = st + h * k3StepBytes;
            const int kk = k0 + h;
            if (narrow)  // 64 rows: this CTA's half of the 128-row pre-tiled block
              tma_load_2d_pair_nohint(ss + k2SmemA, &maps.b64, fbar, 0,
                                      ((n_half >> 7) * p.w_ksteps + kk) * 128 + (n_half & 127));
            else
              tma_load_2d_pair_nohint(ss + k2SmemA, &maps.b, fbar, 0, ((n_half >> 7) * p.w_ksteps + kk) * 128);
            if (no_sf) continue;
            tma_load_2d_pair_nohint(ss + k2SmemA + k2SmemB + k2SmemSFA, &maps.sfb, fbar, 0,
                                    ((n0 / 128) * p.kc_pad + 2 * kk) * 4);
            if (!narrow)
              tma_load_2d_pair_nohint(ss + k2SmemA + k2SmemB + k2SmemSFA + 1024, &maps.sfb, fbar, 0,
                                      ((n0 / 128 + 1) * p.kc_pad + 2 * kk) * 4);
          }
          if (u == 0) pdl_wait();  // activations come from the quantizer launched just before
          for (int h = 0; h < len; ++h) {
            const uint32_t ss = st + h * k3StepBytes;
            const int kk = k0 + h;
            tma_load_2d_pair_nohint(ss, &maps.a, fbar, kk * kStepBytes, m_own);
            if (!no_sf)
              tma_load_2d_pair_nohint(ss + k2SmemA + k2SmemB, &maps.sfa, fbar, 0, (mblk * p.kc_pad + 2 * kk) * 4);
          }
          if (with_r) {
            tma_load_2d_pair_nohint(rb, &maps.r, fbar, 0, n_half);  // [128 rows x 32 B], 32B swizzle
            // R SFB chunk 0 for both 128-row blocks: 512 B each = 4 rows of 128 B of the SF map
            tma_load_2d_pair_nohint(rb + k3RB, &maps.sfr, fbar, 0, ((n0 / 128) * p.kc_pad_r) * 4);
            tma_load_2d_pair_nohint(rb + k3RB + 512, &maps.sfr, fbar, 0, ((n0 / 128 + 1) * p.kc_pad_r) * 4);
            if (kGather) {  // after griddepcontrol.wait (u > 0 or the A loads above): quantizer output
              int seg = 0;  // fused linears: the tile's segment picks its 128-column slice of xs
              for (int j = 0; j + 1 < p.nseg; ++j) seg += n0 >= p.seg_row[j] ? 1 : 0;
              const uint32_t xb = smem_u32(xsbuf);
              tma_load_2d_pair_nohint(xb, &maps.xs, fbar, seg * 64, m_own);  // [128 rows x 32 B]
              tma_load_2d_pair_nohint(xb + 4096, &maps.sfxs, fbar, 0, (mblk * p.kc_pad_xs + seg) * 4);  // SF atom
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      const uint32_t smem_base = smem_u32(smem);
      const uint32_t rb = smem_u32(rbuf);
      constexpr uint32_t id0w = idesc_mxf4(256, kBN), id1w = id0w | (2u << 4) | (2u << 29);
      constexpr uint32_t id0n = idesc_mxf4(256, 128), id1n = id0n | (2u << 4) | (2u << 29);
      constexpr uint32_t kSfR = kSfBase + 2 * kSfCols;  // R's SFB slot: 8 columns at 496
      uint32_t total = 0;
      for (int i = 0; i < my_tiles; ++i) {
        const Item itm = item_of(cluster_id + i * n_clusters);
        total += uint32_t(itm.hi - itm.lo);
      }
      auto cps = [&](uint32_t st, uint32_t fa, uint32_t fb) {
        const uint32_t sa = st + k2SmemA + k2SmemB, sb = sa + k2SmemSFA;
        tmem_cp_pair(fa, make_sdesc(sa, 128, 128, 0));
        tmem_cp_pair(fa + 4, make_sdesc(sa + 512, 128, 128, 0));
        tmem_cp_pair(fb, make_sdesc(sb, 128, 128, 0));
        tmem_cp_pair(fb + 4, make_sdesc(sb + 1024, 128, 128, 0));
        tmem_cp_pair(fb + 8, make_sdesc(sb + 512, 128, 128, 0));
        tmem_cp_pair(fb + 12, make_sdesc(sb + 1536, 128, 128, 0));
      };
      // 4 MMAs (K = 256) of one step
      uint32_t id0 = id0w, id1 = id1w;
      auto step4 = [&](uint32_t acc, uint64_t a, uint64_t b, uint32_t fa, uint32_t fb, uint32_t first, int n) {
        mma_mxf4_pair(acc, a, b, id0, fa, fb, first);
        mma_mxf4_pair(acc, a + 2, b + 2, id1, fa | (2u << 30), fb | (2u << 30), 1u);
        mma_mxf4_pair(acc, a + 4, b + 4, id0, fa + 4, fb + 8, 1u);
        if (n == 4) mma_mxf4_pair(acc, a + 6, b + 6, id1, (fa + 4) | (2u << 30), (fb + 8) | (2u << 30), 1u);
      };
      uint32_t u = 0;
#ifdef SERQ_DIAG_TS
      uint64_t gt0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
      const long long ck0 = clock64();
#endif
      if (total > 0) {
        mbar_wait(&full[0], 0);
        tc_fence_after();
      }
      for (int i = 0; i < my_tiles; ++i) {
        const uint32_t acc = (i & 1) ? kAccB1 : 0u;
        if (i > 0) {
          mbar_wait(tmem_empty, (i - 1) & 1);  // both epilogues drained the overlapping columns
          tc_fence_after();
        }
        const Item itm = item_of(cluster_id + i * n_clusters);
        id0 = itm.nsub >= 0 && !(SERQ_DBG(p.dbg, 64)) ? id0n : id0w;  // diagnostics 64: 256-wide MMAs
        id1 = itm.nsub >= 0 && !(SERQ_DBG(p.dbg, 64)) ? id1n : id1w;
        for (int uu = itm.lo; uu < itm.hi; ++uu, ++u) {
          const int slot = u % k3Slots;
          const int len = (2 * uu + 1 < p.k_steps) ? 2 : 1;
          const bool with_r = has_r && uu == 0;
          const uint32_t st0 = smem_base + slot * k3SlotBytes, st1 = st0 + k3StepBytes;
          const uint64_t a0 = make_sdesc(st0, 16, 1024, 2), b0 = make_sdesc(st0 + k2SmemA, 16, 1024, 2);
          const uint64_t a1 = make_sdesc(st1, 16, 1024, 2), b1 = make_sdesc(st1 + k2SmemA, 16, 1024, 2);
          const uint32_t fa0 = kSfBase, fb0 = fa0 + 8, fa1 = kSfBase + kSfCols, fb1 = fa1 + 8;
          const uint32_t first = uu > itm.lo ? 1u : 0u;
#ifdef SERQ_DIAG_TS
          const bool stamp = p.dbg_ts && blockIdx.x == 0 && u < 100 && lane_id() == 0;
          if (stamp) p.dbg_ts[4 * u] = clock64();
#endif
          const bool no_mma = SERQ_DBG(p.dbg, 1024);  // diagnostics: feed rate alone
          if (elect_one() && !no_mma) {
            cps(st0, fa0, fb0);
            step4(acc, a0, b0, fa0, fb0, first, 4);
            if (with_r) {
              // salient term: A = K-tile 0 of X (same smem, same SFA slot), B = R (32-B rows, 32B swizzle)
              tmem_cp_pair(kSfR, make_sdesc(rb + k3RB, 128, 128, 0));
              tmem_cp_pair(kSfR + 4, make_sdesc(rb + k3RB + 512, 128, 128, 0));
              if constexpr (kGather) {
                // gather: A = the quantizer's x[:, idx] slice and its scale factors (TMEM 504..507)
                constexpr uint32_t kSfXs = kSfR + 8;
                const uint32_t xb = smem_u32(xsbuf);
                tmem_cp_pair(kSfXs, make_sdesc(xb + 4096, 128, 128, 0));
                mma_mxf4_pair(acc, make_sdesc(xb, 16, 256, 6), make_sdesc(rb, 16, 256, 6), id0, kSfXs, kSfR, 1u);
              } else {
                mma_mxf4_pair(acc, a0, make_sdesc(rb, 16, 256, 6), id0, fa0, kSfR, 1u);  // r == 64: one K=64 slice
              }
              tc_commit_pair(r_empty);
            }
            if (len == 2) {
              cps(st1, fa1, fb1);
              step4(acc, a1, b1, fa1, fb1, 1u, 3);
            }
          }
          __syncwarp();
#ifdef SERQ_DIAG_TS
          if (stamp) p.dbg_ts[4 * u + 1] = clock64();
#endif
          if (u + 1 < total) {  // look ahead while the pipe still holds this slot's MMAs
            const uint32_t un = u + 1;
            mbar_wait(&full[un % k3Slots], (un / k3Slots) & 1);
            tc_fence_after();
          }
#ifdef SERQ_DIAG_TS
          if (stamp) p.dbg_ts[4 * u + 2] = clock64();
#endif
          if (elect_one()) {
            if (no_mma && with_r) tc_commit_pair(r_empty);
            if (len == 2 && !no_mma)
              mma_mxf4_pair(acc, a1 + 6, b1 + 6, id1, (fa1 + 4) | (2u << 30), (fb1 + 8) | (2u << 30), 1u);
            tc_commit_pair(&empty[slot]);
            if (uu == itm.hi - 1) tc_commit_pair(&tmem_full[i & 1]);
          }
          __syncwarp();
#ifdef SERQ_DIAG_TS
          if (stamp) p.dbg_ts[4 * u + 3] = clock64();
#endif
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
    uint8_t* stage_out = epi_smem + q * kEpiBox;
    const uint32_t rbase = smem_u32(stage_out) + lane_id() * 64;
    const uint32_t sw = (lane_id() >> 1) & 3;
    const uint32_t tmem_empty_leader = map_rank(smem_u32(tmem_empty), 0);
    pdl_wait();
    pdl_launch_dependents();
    for (int i = 0; i < my_tiles; ++i) {
      const Item itm = item_of(cluster_id + i * n_clusters);
      const int tile = itm.tile;
      int mt, nt;
      tile_mn(tile, mt, nt);
      const int m_own = mt * 256 + int(rank) * 128;
      const int n0 = nt * kBN + (itm.nsub >= 0 ? itm.nsub * 128 : 0);
      const int n_chunks = itm.nsub >= 0 ? 2 : 4;
      const uint32_t b = i & 1;
#ifdef SERQ_DIAG_TS
      // per CTA, per work item (< 6): [before tmem_full, after tmem_full, item epilogue done, half]
      const bool est = p.dbg_ts && q == 0 && lane_id() == 0 && i < 6;
      long long* ep = p.dbg_ts + 1024 + blockIdx.x * 24 + i * 4;
      if (est) { uint64_t g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); ep[0] = (long long)g; }
#endif
      if (kAddend) {  // pull this tile's addend rows into L2 while its MMAs run
        const int row = m_own + int(q) * 32 + int(lane_id());
        if (row < p.M)
          for (int cb = 0; cb < n_chunks * 64; cb += 32)
            if (n0 + cb < p.N)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(p.addend + size_t(row) * p.N + n0 + cb));
      }
      mbar_wait(&tmem_full[b], (i >> 1) & 1);
      tc_fence_after();
#ifdef SERQ_DIAG_TS
      if (est) { uint64_t g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); ep[1] = (long long)g; ep[3] = -1; }
#endif
      const uint32_t acc = (b ? kAccB1 : 0u) + lane_base;
#pragma unroll 1
      for (int cc = 0; cc < n_chunks; ++cc) {
        const int c = (b || n_chunks == 2) ? cc : (cc + 3) & 3;
        uint32_t v[32], w[32];
        tmem_ld_32x32b_x32(acc + c * 64, v);
        tmem_ld_32x32b_x32(acc + c * 64 + 32, w);
        tmem_ld_wait();
        if (cc == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive_cluster_relaxed(tmem_empty_leader);
        }
        if (kAddend) {  // the SVD baseline's fp32 correction (compensate.py:326-331; r = 0 handles only)
          const int row = m_own + int(q) * 32 + int(lane_id());
          if (row < p.M) {
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
        }
        // the CTA's final tile: the pipeline is drained, so each (chunk, half) box gets its
        // own 2 KB of slot memory and the TMA stores go out without waiting on each other
        const bool final_tile = i == my_tiles - 1 && !(SERQ_DBG(p.dbg, (1 << 26)));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* src = h ? w : v;
          if constexpr (kGather) {
            // 32 rows x 16 columns per box (1 KB, no swizzle): lane = row, 32 B each
#pragma unroll
            for (int sb = 0; sb < 2; ++sb) {
              uint8_t* box = final_tile ? smem + q * 16384 + ((cc * 2 + h) * 2 + sb) * 1024 : stage_out;
              const uint32_t bbase = smem_u32(box) + lane_id() * 32;
              if (!final_tile && lane_id() == 0) bulk_wait_read_all();
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 2; ++j)
                st_shared_v4(bbase + j * 16,
                             pack_bf16x2(__uint_as_float(src[16 * sb + 8 * j]), __uint_as_float(src[16 * sb + 8 * j + 1])),
                             pack_bf16x2(__uint_as_float(src[16 * sb + 8 * j + 2]), __uint_as_float(src[16 * sb + 8 * j + 3])),
                             pack_bf16x2(__uint_as_float(src[16 * sb + 8 * j + 4]), __uint_as_float(src[16 * sb + 8 * j + 5])),
                             pack_bf16x2(__uint_as_float(src[16 * sb + 8 * j + 6]), __uint_as_float(src[16 * sb + 8 * j + 7])));
              fence_proxy_async_smem();
              __syncwarp();
              if (lane_id() == 0 && m_own < p.M) {
                tma_store_2d(&maps.y, box, n0 + c * 64 + h * 32 + sb * 16, m_own + q * 32);
                bulk_commit();
              }
            }
          } else {
            uint8_t* box = final_tile ? smem + q * 16384 + (cc * 2 + h) * 2048 : stage_out;
            const uint32_t bbase = final_tile ? smem_u32(box) + lane_id() * 64 : rbase;
            if (!final_tile && lane_id() == 0) bulk_wait_read_all();
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j)
              st_shared_v4(bbase + ((uint32_t(j) ^ sw) * 16),
                           pack_bf16x2(__uint_as_float(src[8 * j]), __uint_as_float(src[8 * j + 1])),
                           pack_bf16x2(__uint_as_float(src[8 * j + 2]), __uint_as_float(src[8 * j + 3])),
                           pack_bf16x2(__uint_as_float(src[8 * j + 4]), __uint_as_float(src[8 * j + 5])),
                           pack_bf16x2(__uint_as_float(src[8 * j + 6]), __uint_as_float(src[8 * j + 7])));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane_id() == 0 && m_own < p.M) {
              tma_store_2d(&maps.y, box, n0 + c * 64 + h * 32, m_own + q * 32);
              bulk_commit();
            }
          }
        }
      }
#ifdef SERQ_DIAG_TS
      if (est) { uint64_t g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); ep[2] = (long long)g; }
#endif
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
#ifdef SERQ_DIAG_TS
  if (p.dbg_ts && threadIdx.x == 0) {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    p.dbg_ts[1024 + 148 * 24 + blockIdx.x * 2 + 1] = (long long)g;
  }
#endif
}

}  // namespace serq
