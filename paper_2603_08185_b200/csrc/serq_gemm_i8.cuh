// serq_gemm_i8.cuh -- integer SERQ linear on CTA pairs (BASELINE configs 1 and 3).
//
// Y = sx[m] * ( sw[n] * (acc - zp[m]*colsum[n]) + R-term ),  acc = sum_k c[m,k] w[k,n]
// (int_gemm_reference, mxfmt.py:177-195; forward_reconstructed, compensate.py:300-316).
//
// * tcgen05.mma.cta_group::2.kind::i8, 256 x 256 x 32 per instruction: u8
//   (asymmetric) or s8 (symmetric) activation codes x s8 weights, s32 in TMEM.
// * Weights: int8 [N, K] TMA'd straight into the 128B-swizzled K-major operand
//   (Blackwell has no INT4 MMA).  A variant that kept packed INT4 in HBM and
//   widened it in shared memory with transform warps was measured slower (the
//   widening traffic made the SM shared-memory bound; K3) and removed.
// * The salient term accumulates into a second TMEM accumulator (columns
//   [256,512)): integer R (kind::i8, A = K-tile 0 of X, B = R codes) or dense
//   bf16 R (kind::f16, A = bf16 (codes - zp) slice, B = L^T), both staged with
//   K-step 0 of the tile.
// * Two accumulators fill TMEM, so the epilogue of a tile is not overlapped
//   with the next tile's MMAs; it reads both accumulators, applies the
//   zero-point correction exactly (int64) and the scales, and stores bf16.
#pragma once
#include "serq_gemm_mx2.cuh"

namespace serq {

constexpr int kI8A = 128 * 128;    // own 128 activation rows x 128 int8
constexpr int kI8B = 128 * 128;    // own 128 weight rows x 128 int8
constexpr int kI8Side = 2 * 16384;             // R operands: [A' (dense only)] + B_R
constexpr int kI8Const = 4 * 256 * 4;
// kE: epilogue column groups -- 4 * kE epilogue warps (warp w drains TMEM lane quadrant w % 4,
// columns chunks e, e + kE, ...), each with one 2 KB output staging box
template <int kE, bool kW4 = false>
struct I8Cfg {
  static constexpr int kEpiWarps = 4 * kE;
  // warps: 0 TMA producer, 1 MMA issuer, 2 .. 2 + kLoadWarps - 1 packed-INT4 loaders (W4) or idle,
  // then the epilogue warps
  static constexpr int kLoadWarps = kW4 ? 4 : 2;
  static constexpr int kEpiWarp0 = 2 + kLoadWarps;
  static constexpr int kEpiBytes = kEpiWarps * 2048;
  static constexpr int kStages = kE >= 4 ? 4 : 5;
  static constexpr int kStage = kI8A + kI8B;
  static constexpr int kSmem = 1024 + kStages * kStage + kI8Side + kI8Const + kEpiBytes + 512;
  static constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
  static_assert(kSmem <= 232448, "smem budget");
};

struct I8Maps {
  CUtensorMap a, bp, r, xs, y;
};

__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P;\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n"
      " selp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
__device__ __forceinline__ void mma_i8_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_i8_or_bf16(bool bf16, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t acc) {
  if (bf16)
    mma_bf16_pair(d, a, b, idesc, acc);
  else
    mma_i8_pair(d, a, b, idesc, acc);
}
__device__ __forceinline__ uint2 ld_shared_v2(const void* p) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void ld_shared_v4u(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
}
__device__ __forceinline__ void mbar_wait_bo(uint64_t* bar, uint32_t parity, bool backoff) {
  while (!mbar_try_wait(bar, parity)) {
    if (backoff) __nanosleep(200);
  }
}
// Remote arrive with the default (.release.cta) semantics: orders this
// thread's prior shared-memory writes (already fenced to the async proxy)
// without the cluster-scope drain a .release.cluster arrive pays.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// 8 packed two's-complement nibbles -> 8 int8.  Pack-time order (pack_int4_tiled_kernel): byte j
// of the word holds elements j (low nibble) and j + 4 (high nibble), so the low nibbles widen to
// elements 0..3 and the high nibbles to 4..7 with no byte shuffle.  Per byte, with b = n ^ 8
// (the nibble biased to [0, 15]): ((b + 0x78) ^ 0x80) = the sign-extended nibble, and b + 0x78
// <= 0x87 never carries into the next byte: 3 integer ops per 4 codes.
__device__ __forceinline__ uint2 widen_int4x8(uint32_t w) {
  const uint32_t lo = (((w & 0x0F0F0F0Fu) ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
  const uint32_t hi = ((((w >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
  return make_uint2(lo, hi);
}
// kN: output columns per CTA-pair tile (256, or 128 for small problems so twice as many
// pairs get a tile; each CTA then stages 64 weight rows)
// kW4: the weights stay PACKED INT4 in HBM (0.5 B / weight, pre-tiled [N/128][K/128][128 rows x
// 64 B]); two loader warps per CTA read them with plain 8-byte global loads (three K-steps ahead
// in registers), widen 8 codes per word (LOP3 / VSUB4 / PRMT) and store the int8 operand straight
// into the 128B-swizzled stage -- the same shared-memory traffic as the TMA'd int8 feed (the
// staging copy of an earlier variant made the SM shared-memory bound).  Blackwell has no INT4 MMA.
template <int kN = 256, int kE = 2, bool kW4 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(I8Cfg<kE, kW4>::kThreads, 1)
    serq_i8_pair_kernel(const __grid_constant__ I8Maps maps, const GemmParams p) {
  static_assert(kN == 256 || kN == 128, "256- or 128-column tiles");
  static_assert((kN / 32) % kE == 0, "column chunks split evenly over the epilogue groups");
  using Cfg = I8Cfg<kE, kW4>;
  constexpr int kI8LoadWarps = Cfg::kLoadWarps;
  constexpr int kEpiWarp0 = Cfg::kEpiWarp0;
  constexpr int kEpiThreads = 32 * Cfg::kEpiWarps;
  constexpr int kBHalf = kN / 2;  // weight rows per CTA
  constexpr uint32_t kBBytes = kBHalf * 128;  // one 128-K step of this CTA's weight rows (int8)
  constexpr uint32_t kRBytes = kBHalf * 128;  // this CTA's R rows per side tile (int8 r <= 128 or 64 bf16: 128 B each)
  constexpr int kI8Stages = Cfg::kStages;
  constexpr int kI8Stage = Cfg::kStage;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* side = smem + kI8Stages * kI8Stage;       // [A' 16K][B_R 16K]
  float* cst_f = reinterpret_cast<float*>(side + kI8Side);  // sw[256] | sr[256]
  int32_t* cst_i = reinterpret_cast<int32_t*>(cst_f + 512); // colsum[256] | colsum_r[256]
  uint8_t* epi = reinterpret_cast<uint8_t*>(cst_i + 512);   // one 2 KB staging box per epilogue warp
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + Cfg::kEpiBytes);
  uint64_t* full = bars;                       // [S] leader: A, B (+ side) landed, both CTAs
  uint64_t* empty = bars + kI8Stages;          // [S] both: MMAs of the stage done
  uint64_t* side_empty = bars + 2 * kI8Stages; // both: R MMAs done
  uint64_t* tmem_full = side_empty + 1;        // both
  uint64_t* tmem_empty = side_empty + 2;       // leader: 8 epilogue warps drained TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(side_empty + 3);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const int tiles_m = (p.M + 255) / 256;
  const int tiles_n = (p.N + kN - 1) / kN;
  const int n_tiles = tiles_m * tiles_n;
  const int my_tiles = cluster_id < n_tiles ? (n_tiles - 1 - cluster_id) / n_clusters + 1 : 0;
  const bool has_r = p.r_mode != kRNone;
  const bool dense = p.r_mode == kRDense;
  const int ks = p.k_steps;  // 128-K steps
  // the salient term in side tiles of 64 bf16 (dense) / 128 int8 (integer R) columns: tile j is
  // staged with main K-step j * sstep (spread out, so reloading the one side buffer stays off
  // the MMA's critical path; the host guarantees ks >= nr)
  const int nr = has_r ? (dense ? (p.r + 63) / 64 : 1) : 0;
  const int sstep = nr > 0 ? ks / nr : 1;
  // side-tile cursor over a tile's K-steps (no runtime division in the issue loops: an integer
  // divide is a ~40-instruction dependent chain that slowed every K-step of the MMA warp)
  struct SideCursor {
    int next, cnt, nr, sstep;
    __device__ int step(int kk) {  // side tile staged / consumed at K-step kk, or -1
      if (kk != next) return -1;
      const int j = cnt++;
      next = cnt < nr ? next + sstep : 0x7fffffff;
      return j;
    }
  };
  auto side_cursor = [&]() { return SideCursor{nr > 0 ? 0 : 0x7fffffff, 0, nr, sstep}; };

  if (warp == 0 && elect_one()) {
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.bp);
    tma_prefetch(&maps.y);
    if (has_r) {
      tma_prefetch(&maps.r);
      tma_prefetch(&maps.xs);
    }
    for (int s = 0; s < kI8Stages; ++s) {
      mbar_init(&full[s], kW4 ? 1 + 2 * kI8LoadWarps : 1);  // W4: + the loader warps of both CTAs
      mbar_init(&empty[s], 1);
    }
    mbar_init(side_empty, 1);
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 2 * Cfg::kEpiWarps);
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

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (elect_one()) {
      const uint32_t sb = smem_u32(smem), sside = smem_u32(side);
      // programmatic dependent launch: the first tile's weight stages do not depend on the
      // previous kernel (the activation quantizer) -- stream them before griddepcontrol.wait
      const int pre = (!kW4 && my_tiles > 0) ? (ks < kI8Stages ? ks : kI8Stages) : 0;
      constexpr uint32_t kBTma = kW4 ? 0u : kBBytes;  // W4: B is written by the loader warps
      if (my_tiles > 0) {
        const int n_half0 = (cluster_id / tiles_m) * kN + int(rank) * kBHalf;
        SideCursor sc0 = side_cursor();
        for (int kk = 0; kk < pre; ++kk) {
          const bool with_side = sc0.step(kk) >= 0;
          if (leader)
            mbar_expect_tx(&full[kk], 2u * (kI8A + kBBytes + (with_side ? (dense ? 16384 + kRBytes : kRBytes) : 0)));
          tma_load_2d_pair(sb + kk * kI8Stage + kI8A, &maps.bp, map_rank(smem_u32(&full[kk]), 0), kk * 128, n_half0,
                           kEvictNormal);
        }
      }
      pdl_wait();
      uint32_t g = 0;
      for (int i = 0; i < my_tiles; ++i) {
        const int tile = cluster_id + i * n_clusters;
        const int mt = tile % tiles_m, nt = tile / tiles_m;
        const int m_own = mt * 256 + int(rank) * 128;
        const int n_half = nt * kN + int(rank) * kBHalf;
        SideCursor sc = side_cursor();
        for (int kk = 0; kk < ks; ++kk, ++g) {
          const int s = g % kI8Stages;
          const bool preloaded = i == 0 && kk < pre;
          if (!preloaded) mbar_wait_bo(&empty[s], ((g / kI8Stages) & 1) ^ 1, SERQ_DBG(p.dbg, (1 << 20)));
          const int sj = sc.step(kk);
          const bool with_side = sj >= 0;
          const int su = i * nr + sj;  // side-buffer use count
          if (with_side && su > 0) mbar_wait(side_empty, (su - 1) & 1);
          const uint32_t fbar = map_rank(smem_u32(&full[s]), 0);
          const uint32_t st = sb + s * kI8Stage;
          if (leader && !preloaded)
            mbar_expect_tx(&full[s], 2u * (kI8A + kBTma + (with_side ? (dense ? 16384 + kRBytes : kRBytes) : 0)));
          if (!preloaded && !kW4)
            tma_load_2d_pair(st + kI8A, &maps.bp, fbar, kk * 128, n_half, kEvictNormal);  // int8 [N, K] rows
          tma_load_2d_pair(st, &maps.a, fbar, kk * 128, m_own, kEvictNormal);
          if (with_side) {
            tma_load_2d_pair(sside + 16384, &maps.r, fbar, 64 * sj, n_half, kEvictNormal);
            if (dense) tma_load_2d_pair(sside, &maps.xs, fbar, 64 * sj, m_own, kEvictNormal);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader) {
      const uint32_t sb = smem_u32(smem), sside = smem_u32(side);
      const uint32_t id_main = idesc_i8(256, kN, p.a_signed != 0, true);
      const uint32_t id_r = dense ? idesc_bf16(256, kN) : id_main;
      const uint32_t total = uint32_t(my_tiles) * ks;
      if (total > 0) {
        mbar_wait_cluster(&full[0], 0);
        tc_fence_after();
      }
      uint32_t g = 0;
      for (int i = 0; i < my_tiles; ++i) {
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && lane_id() == 0 && i < 8) p.dbg_ts[512 + (blockIdx.x >> 1) * 64 + i * 8] = globaltimer();
#endif
        if (i > 0) {
          mbar_wait_bo(tmem_empty, (i - 1) & 1, SERQ_DBG(p.dbg, (1 << 20)));
          tc_fence_after();
        }
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && lane_id() == 0 && i < 8) p.dbg_ts[512 + (blockIdx.x >> 1) * 64 + i * 8 + 1] = globaltimer();
#endif
        SideCursor sc = side_cursor();
        for (int kk = 0; kk < ks; ++kk, ++g) {
          const int s = g % kI8Stages;
          const uint32_t st = sb + s * kI8Stage;
          const int sj = sc.step(kk);  // every lane: the cursor advances whether or not this lane issues
          const uint64_t a = make_sdesc(st, 16, 1024, 2), b = make_sdesc(st + kI8A, 16, 1024, 2);
          const uint32_t first = kk > 0 ? 1u : 0u;
          const bool no_mma = SERQ_DBG(p.dbg, (1 << 18));
          if (elect_one() && !no_mma) {
            mma_i8_pair(0, a, b, id_main, first);
            mma_i8_pair(0, a + 2, b + 2, id_main, 1u);
            mma_i8_pair(0, a + 4, b + 4, id_main, 1u);
            if (sj >= 0) {
              // salient term (side tile sj) into the second accumulator (columns [256, 512))
              const uint64_t ar = dense ? make_sdesc(sside, 16, 1024, 2) : a;
              const uint64_t br = make_sdesc(sside + 16384, 16, 1024, 2);
              const int rr = dense ? min(64, p.r - 64 * sj) : p.r;
              const int nk = dense ? (2 * rr + 31) / 32 : (rr + 31) / 32;
              for (int j = 0; j < nk; ++j)
                mma_i8_or_bf16(dense, 256, ar + 2 * j, br + 2 * j, id_r, (sj > 0 || j > 0) ? 1u : 0u);
              tc_commit_pair(side_empty);
            }
          }
          __syncwarp();
#ifdef SERQ_DIAG_TS
          if (p.dbg_ts && blockIdx.x == 0 && lane_id() == 0 && g < 32) p.dbg_ts[8 * g + 5] = clock64();
#endif
          if (g + 1 < total) {
            const uint32_t gn = g + 1;
            mbar_wait_cluster(&full[gn % kI8Stages], (gn / kI8Stages) & 1);
            tc_fence_after();
          }
#ifdef SERQ_DIAG_TS
          if (p.dbg_ts && blockIdx.x == 0 && lane_id() == 0 && g < 32) p.dbg_ts[8 * g + 6] = clock64();
#endif
          if (elect_one()) {
            if (!no_mma) mma_i8_pair(0, a + 6, b + 6, id_main, 1u);
            tc_commit_pair(&empty[s]);
            if (kk == ks - 1) tc_commit_pair(tmem_full);
          }
          __syncwarp();
        }
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && lane_id() == 0 && i < 8) p.dbg_ts[512 + (blockIdx.x >> 1) * 64 + i * 8 + 2] = globaltimer();
#endif
      }
    }
  } else if (kW4 && warp < 2 + kI8LoadWarps) {
    // ------------------------------------------------------------ W4 loaders (both CTAs)
    // thread lt: 16 packed bytes (32 codes = operand chunks 2c, 2c + 1) of rows lt / 4 + kRowsPerPass j;
    // a warp loads 8 rows x 64 B per instruction and its stores are conflict-free (two rows per
    // quarter-warp fill complementary halves of the 128-byte swizzle pattern)
    constexpr int kRowsPerPass = 32 * kI8LoadWarps / 4;
    constexpr int kJ = kBHalf / kRowsPerPass;
    const int lt = int(threadIdx.x) - 64;
    const int c = lt & 3, r0 = lt >> 2;
    const uint32_t full_leader = map_rank(smem_u32(&full[0]), 0);
    const uint8_t* w4 = p.w4;
    const int total = my_tiles * ks;
    // this CTA's contiguous kBHalf x 64 B block of each K-step, walked by cursors (a division per
    // tile, none per step: the loads run ahead at g + 3, the L2 prefetch at g + kPf)
    auto tile_base = [&](int i) {
      const int tile = cluster_id + i * n_clusters;
      const int n_half = (tile / tiles_m) * kN + int(rank) * kBHalf;
      return w4 + (size_t(n_half >> 7) * ks * 128 + (n_half & 127)) * 64;
    };
    struct WCursor {
      int i, kk;
      const uint8_t* base;
    };
    auto next_block = [&](WCursor& cu) {
      const uint8_t* b = cu.base + size_t(cu.kk) * 128 * 64;
      if (++cu.kk == ks) {
        cu.kk = 0;
        if (++cu.i < my_tiles) cu.base = tile_base(cu.i);
      }
      return b;
    };
    WCursor load_cur{0, 0, my_tiles > 0 ? tile_base(0) : w4}, pf_cur = load_cur;
    // the register loads run 3 K-steps ahead; an L2 prefetch of the whole block kPf steps ahead
    constexpr int kPf = 8;
    if (lt == 0)
      for (int g = 0; g < kPf && g < total; ++g)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(next_block(pf_cur)), "r"(uint32_t(kBHalf * 64))
                     : "memory");
    auto load = [&](uint4 (&b)[kJ], int g) {  // called for g = 0, 1, 2, ... in order
      if (g < total && !SERQ_DBG(p.dbg, 1 << 10)) {  // diagnostics: no weight loads
        const uint8_t* src = next_block(load_cur) + r0 * 64 + c * 16;
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
          uint4 v;
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "l"(src + j * kRowsPerPass * 64));
          b[j] = v;
        }
      }
    };
    // Four register buffers; a step's loads are issued three steps before its widen.  (Measured at
    // C3: 127.8 us at the time; rotating the buffers by name instead of shifting them -- no register copy
    // waits on the step's own loads -- measured 150.6 us, and an L2 prefetch changed nothing.)
    uint4 b0[kJ], b1[kJ], b2[kJ], b3[kJ];
    load(b0, 0);
    load(b1, 1);
    load(b2, 2);
    for (int g = 0; g < total; ++g) {
      if (lt == 0 && g + kPf < total)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(next_block(pf_cur)), "r"(uint32_t(kBHalf * 64))
                     : "memory");
      load(b3, g + 3);
      const int s = g % kI8Stages;
      mbar_wait(&empty[s], ((g / kI8Stages) & 1) ^ 1);
      const uint32_t dst = smem_u32(smem + s * kI8Stage + kI8A);
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        if (SERQ_DBG(p.dbg, 1 << 11)) break;  // diagnostics: no operand stores
        const int row = r0 + kRowsPerPass * j;
        const uint32_t rb = dst + row * 128, sw = uint32_t(row & 7);
        const uint2 e0 = widen_int4x8(b0[j].x), e1 = widen_int4x8(b0[j].y);  // chunk 2c: elements 0..15
        const uint2 e2 = widen_int4x8(b0[j].z), e3 = widen_int4x8(b0[j].w);  // chunk 2c + 1
        st_shared_v4(rb + (((2u * c) ^ sw) * 16), e0.x, e0.y, e1.x, e1.y);
        st_shared_v4(rb + (((2u * c + 1) ^ sw) * 16), e2.x, e2.y, e3.x, e3.y);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_remote(full_leader + uint32_t(s) * 8u);
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        b0[j] = b1[j];
        b1[j] = b2[j];
        b2[j] = b3[j];
      }
    }
  } else if (warp >= uint32_t(kEpiWarp0)) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    pdl_wait();  // sx / zp / xs come from the quantizer; y may still be read by a predecessor
    pdl_launch_dependents();
    const uint32_t q = warp & 3;  // TMEM lane quadrant of this warp (warp id % 4)
    const int eg = int(warp - kEpiWarp0) >> 2;  // column group: chunks eg, eg + kE, ...
    const uint32_t lane_base = (q * 32u) << 16;
    uint8_t* stage_out = epi + (warp - kEpiWarp0) * 2048;
    const uint32_t swz = (lane_id() >> 1) & 3;
    const uint32_t tmem_empty_leader = map_rank(smem_u32(tmem_empty), 0);
    for (int i = 0; i < my_tiles; ++i) {
      const int tile = cluster_id + i * n_clusters;
      const int mt = tile % tiles_m, nt = tile / tiles_m;
      const int m_own = mt * 256 + int(rank) * 128;
      const int n0 = nt * kN;
      // per-column constants of this tile
      named_bar_sync(1, kEpiThreads);  // previous tile's readers are done with the constants
      for (int c = int(threadIdx.x) - 32 * kEpiWarp0; c < kN; c += kEpiThreads) {
        const int n = n0 + c;
        const bool ok = n < p.N;
        cst_f[c] = ok ? p.sw[n] : 0.f;
        cst_i[c] = (ok && p.zp) ? -p.colsum[n] : 0;  // negated: acc + zp*(-colsum) is one IMAD
        cst_f[256 + c] = (ok && p.r_mode == kRInt) ? p.sr[n] : 0.f;
        cst_i[256 + c] = (ok && p.zp && p.r_mode == kRInt) ? -p.colsum_r[n] : 0;
      }
      named_bar_sync(1, kEpiThreads);
      const int row = m_own + int(q) * 32 + int(lane_id());
      float sx = 0.f;
      uint32_t zp = 0;
      if (row < p.M) {
        sx = p.sx[row];
        zp = p.zp ? uint32_t(p.zp[row]) : 0u;
      }
#ifdef SERQ_DIAG_TS
      if (p.dbg_ts && leader && q == 0 && lane_id() == 0 && i < 8) p.dbg_ts[512 + cluster_id * 64 + i * 8 + 3] = globaltimer();
#endif
      mbar_wait(tmem_full, i & 1);
      tc_fence_after();
#ifdef SERQ_DIAG_TS
      if (p.dbg_ts && leader && q == 0 && lane_id() == 0 && i < 8) p.dbg_ts[512 + cluster_id * 64 + i * 8 + 4] = globaltimer();
#endif
#pragma unroll 1
      for (int cc = 0; cc < kN / 32 / kE; ++cc) {
        const int c = cc * kE + eg;
        // exact in wrapping int32: |acc - zp*colsum| <= 255 * 8 * K < 2^31 for K < 2^20
        uint32_t packed[16];
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && leader && cluster_id == 0 && q == 0 && lane_id() == 0 && i == (my_tiles > 1 ? 1 : 0)) p.dbg_ts[5300 + c * 8 + 0] = globaltimer();
#endif
        uint32_t vv[32], ww[32];
        tmem_ld_32x32b_x32(lane_base + uint32_t(c * 32), vv);
        if (has_r) tmem_ld_32x32b_x32(lane_base + 256 + uint32_t(c * 32), ww);
        tmem_ld_wait();
        if (cc == kN / 32 / kE - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive_cluster_relaxed(tmem_empty_leader);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* v = vv + 16 * h;
          const uint32_t* w = ww + 16 * h;
          const uint32_t col0 = uint32_t(c * 32 + h * 16);
#ifdef SERQ_DIAG_TS
          if (p.dbg_ts && leader && cluster_id == 0 && q == 0 && lane_id() == 0 && i == (my_tiles > 1 ? 1 : 0)) p.dbg_ts[5300 + c * 8 + 4 + h] = globaltimer();
#endif
          // this half-chunk's column constants: broadcast vector loads, once
          const uint32_t cf = smem_u32(cst_f) + col0 * 4, ci = smem_u32(cst_i) + col0 * 4;
          float f[16];
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            // 4 columns' constants per broadcast vector load
            uint32_t cs[4], fs[4], cr[4] = {0, 0, 0, 0}, fr[4] = {0, 0, 0, 0};
            ld_shared_v4u(ci + 16 * j4, cs[0], cs[1], cs[2], cs[3]);
            ld_shared_v4u(cf + 16 * j4, fs[0], fs[1], fs[2], fs[3]);
            if (has_r && !dense) {
              ld_shared_v4u(ci + 1024 + 16 * j4, cr[0], cr[1], cr[2], cr[3]);
              ld_shared_v4u(cf + 1024 + 16 * j4, fr[0], fr[1], fr[2], fr[3]);
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int j = 4 * j4 + jj;
              const int32_t a = int32_t(v[j] + zp * cs[jj]);
              float yv = float(a) * __uint_as_float(fs[jj]);
              if (has_r) {
                if (dense) {
                  yv += __uint_as_float(w[j]);
                } else {
                  const int32_t ar = int32_t(w[j] + zp * cr[jj]);
                  yv += float(ar) * __uint_as_float(fr[jj]);
                }
              }
              f[j] = yv * sx;
            }
          }
          if (p.addend && row < p.M) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + int(col0) + j < p.N) f[j] += p.addend[size_t(row) * p.N + n0 + col0 + j];
          }
          if (p.acc_dump && row < p.M) {
            // debug: exact accumulators (tests)
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int col = int(col0) + j;
              if (n0 + col >= p.N) continue;
              p.acc_dump[size_t(row) * p.N + n0 + col] = int32_t(v[j] + zp * uint32_t(cst_i[col]));
              if (p.accr_dump && has_r && !dense)
                p.accr_dump[size_t(row) * p.N + n0 + col] = int32_t(w[j] + zp * uint32_t(cst_i[256 + col]));
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) packed[h * 8 + j] = pack_bf16x2(f[2 * j], f[2 * j + 1]);
        }
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && leader && cluster_id == 0 && q == 0 && lane_id() == 0 && i == (my_tiles > 1 ? 1 : 0)) p.dbg_ts[5300 + c * 8 + 1] = globaltimer();
#endif
        // the CTA's final tile: the pipeline is drained (its last MMAs completed before tmem_full), so
        // every chunk gets its own 2 KB box there and no store waits on another; otherwise two
        // boxes per warp alternate and a box is rewritten once the store from two chunks ago read it
        const bool final_tile = i == my_tiles - 1 && !(SERQ_DBG(p.dbg, (1 << 26)));
        uint8_t* box = final_tile ? smem + (int(q) * (kN / 32) + c) * 2048 : stage_out;
        const uint32_t rbase = smem_u32(box) + lane_id() * 64;
        if (!final_tile && lane_id() == 0) bulk_wait_read_all();  // this warp's previous store read its box
        __syncwarp();
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && leader && cluster_id == 0 && q == 0 && lane_id() == 0 && i == (my_tiles > 1 ? 1 : 0)) p.dbg_ts[5300 + c * 8 + 2] = globaltimer();
#endif
#pragma unroll
        for (int j = 0; j < 4; ++j)
          st_shared_v4(rbase + ((uint32_t(j) ^ swz) * 16), packed[4 * j], packed[4 * j + 1], packed[4 * j + 2],
                       packed[4 * j + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0 && m_own < p.M) {
          tma_store_2d(&maps.y, box, n0 + c * 32, m_own + int(q) * 32);
          bulk_commit();
        }
#ifdef SERQ_DIAG_TS
        if (p.dbg_ts && leader && cluster_id == 0 && q == 0 && lane_id() == 0 && i == (my_tiles > 1 ? 1 : 0)) p.dbg_ts[5300 + c * 8 + 3] = globaltimer();
#endif
      }
#ifdef SERQ_DIAG_TS
      if (p.dbg_ts && leader && q == 0 && lane_id() == 0 && i < 8) p.dbg_ts[512 + cluster_id * 64 + i * 8 + 5] = globaltimer();
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
}

}  // namespace serq
