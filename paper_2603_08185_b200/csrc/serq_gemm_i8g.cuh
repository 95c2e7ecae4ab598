// serq_gemm_i8g.cuh -- integer SERQ linear with GROUP-WISE weight scales along K
// (row groups of g = 128..1024 input rows, one scale per
// (group, output column); GPTQ's group_size setting, gptq.py:98-146, and
// _weight_config(bits, g), pipeline.py:134-137).
//
// int_gemm_reference, row-grouped branch (mxfmt.py:177-195):
//   out = sum_g sx[m] * acc_g[m, n] * sw[g, n],  acc_g = sum_{k in g} (c[m,k] - zp[m]) w[k,n]
// plus the salient term (compensate.py:300-316).  Here:
//   Y = sx * ( sum_g float(A_g) * sw[g, n]  +  R-term  -  zp * C[n] )
//   A_g = sum_{k in g} c[m,k] w[k,n]  (exact int32 in TMEM, |A_g| < 2^22)
//   C[n] = sum_g sw[g,n] * colsum_g[n]  (+ sr[n] * colsum_r[n] for integer R), folded on the host,
// so the per-group promotion is one I2FP and half a packed FFMA2 per element
// and carries no zero-point work.
//
// * CTA pair, 256 x 256 output tile, tcgen05.mma.cta_group::2.kind::i8 (u8/s8 x s8, s32),
//   int8 weights TMA'd straight into the 128B-swizzled operand (as serq_i8_pair_kernel<true>).
// * Every group's integer partial lands in one of TWO TMEM accumulators (columns [0,256) and
//   [256,512)), alternating per group ("unit"): the MMA runs one group ahead of the promotion.
// * Sixteen epilogue warps (four per TMEM lane quadrant, 64 columns each) keep the fp32 running
//   sum of their 32 rows x 64 columns in registers; per unit they tcgen05.ld the integer
//   partial, convert it exactly (I2FP, |A_g| < 2^22), FFMA2 it with the group's
//   scales (staged in shared memory one unit ahead), and hand the accumulator back.
// * The salient term is one more unit per tile: integer R (kind::i8, A = K-tile 0 of X,
//   B = R codes, scale sr[n]; r <= 128) or dense bf16 R (kind::f16, A = bf16 (c - zp) slice,
//   B = L^T, r <= 128 in two 64-column atoms; fp32 accumulator added as is) -- optionally
//   split as L = hi + lo (two bf16 planes, both MMAs into the same accumulator: relative
//   error 2^-17 instead of 2^-9), for R matrices that are not small residuals (GPTQ-swapped).
// * Pipeline depth follows the side buffer: 5 stages (no / integer R), 4 (dense), 3 (split).
#pragma once
#include "serq_gemm_i8.cuh"

namespace serq {

constexpr int kI8gMaxStages = 5;
constexpr int kI8gStage = kI8A + kI8B;  // 16 KB activation + 16 KB weight rows
// 18 warps: 5 on two of the SM's sub-partitions, so <= 96 registers per thread (64 KB / 4 SMSPs)
constexpr int kI8gEpiWarps = 16;        // four per TMEM lane quadrant
constexpr int kI8gCols = 256 / (kI8gEpiWarps / 4);  // accumulator columns per epilogue thread
constexpr int kI8gThreads = 32 * (2 + kI8gEpiWarps);  // producer, MMA, epilogue
// R operands (r <= 128) in the side buffer: integer R: B_R [0, 16K); dense / split bf16 R:
// A' [0, 32K), B (hi) [32K, 64K), B lo [64K, 96K) (split only).  The pipeline gets what is left.
constexpr int kI8gFixed = 1024 + 2 * 1024 + 1024 + kI8gEpiWarps * 1024 + 512;
__host__ __device__ constexpr int i8g_side_bytes(int r_mode) {
  return r_mode == kRInt ? 16384 : r_mode == kRDense ? 65536 : r_mode == kRDenseSplit ? 98304 : 0;
}
__host__ __device__ constexpr int i8g_stages(int r_mode) {
  return (232448 - kI8gFixed - i8g_side_bytes(r_mode)) / kI8gStage < kI8gMaxStages
             ? (232448 - kI8gFixed - i8g_side_bytes(r_mode)) / kI8gStage
             : kI8gMaxStages;
}
__host__ __device__ constexpr int i8g_smem(int r_mode) {
  return kI8gFixed + i8g_stages(r_mode) * kI8gStage + i8g_side_bytes(r_mode);
}
static_assert(i8g_stages(kRDenseSplit) >= 3, "smem budget");

struct I8gParams {
  int M, N, K;
  int r, r_mode, a_signed;
  int k_steps;      // 128-K steps
  int gsteps;       // 128-K steps per weight group
  const float* sx;  // [M]
  const int32_t* zp;
  const float* sw_g;        // [G][N] group scales
  const float* cterm;       // [N] sum_g sw_g * colsum_g (+ sr * colsum_r)
  const float* sr;          // [N] integer-R scale
  const int32_t* colsum_g;  // [G][N] (debug dumps only)
  const int32_t* colsum_r;  // [N]    (debug dumps only)
  const float* addend;      // optional fp32 [M, N]
  int32_t* acc_dump;        // debug: exact per-group accumulators (A_g - zp*colsum_g), [G][M][N]
  int32_t* accr_dump;       // debug: exact integer-R accumulators, [M][N]
  long long* dbg_ts;        // diagnostics (SERQ_DIAG_TS builds): epilogue clock64 stamps of CTA 0, warp 4
};
#ifdef SERQ_DIAG_TS
#define I8G_STAMP(u, i) \
  if (p.dbg_ts && blockIdx.x == 0 && warp == 4 && lane_id() == 0 && (u) < 64) p.dbg_ts[(u) * 8 + (i)] = clock64();
#else
#define I8G_STAMP(u, i)
#endif

// a0,a1 += x0*s0, x1*s1 as one packed FFMA2 (sm_100 fma.rn.f32x2)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float s0, float s1) {
  uint64_t a, x, sv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(sv) : "f"(s0), "f"(s1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(x), "l"(sv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}
__device__ __forceinline__ void fadd2(float& a0, float& a1, float x0, float x1) {
  uint64_t a, x;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(x));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}

// kDump: the test build that also writes the exact per-group integer partials
template <bool kDump>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(96)
    serq_i8g_pair_kernel(const __grid_constant__ I8Maps maps, const I8gParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = i8g_stages(p.r_mode);
  uint8_t* side = smem + S * kI8gStage;                       // R operands
  float* sc = reinterpret_cast<float*>(side + i8g_side_bytes(p.r_mode));  // [2][256] unit scales
  float* cst = sc + 512;                                      // [256] C[n] of the current tile
  uint8_t* epi = reinterpret_cast<uint8_t*>(cst + 256);       // 8 x 2 KB store staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + kI8gEpiWarps * 1024);
  uint64_t* full = bars;                        // [S] leader: A + B (+ side) of both CTAs landed
  uint64_t* empty = bars + kI8gMaxStages;       // [S] both: the stage's MMAs are done
  uint64_t* side_empty = bars + 2 * kI8gMaxStages; // both: the R MMAs are done
  uint64_t* acc_full = side_empty + 1;          // [2] both: unit accumulator complete
  uint64_t* acc_empty = acc_full + 2;           // [2] leader: 16 epilogue warps drained it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const int tiles_m = (p.M + 255) / 256;
  const int tiles_n = (p.N + 255) / 256;
  const int n_tiles = tiles_m * tiles_n;
  const int my_tiles = cluster_id < n_tiles ? (n_tiles - 1 - cluster_id) / n_clusters + 1 : 0;
  const bool has_r = p.r_mode != kRNone;
  const bool split = p.r_mode == kRDenseSplit;
  const bool dense = p.r_mode == kRDense || split;
  const int rch = (p.r + 63) / 64;  // dense R: 64-column bf16 atoms
  const int ks = p.k_steps;
  const int units = ks / p.gsteps + (has_r ? 1 : 0);  // per tile

  if (warp == 0 && elect_one()) {
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.bp);
    tma_prefetch(&maps.y);
    if (has_r) {
      tma_prefetch(&maps.r);
      tma_prefetch(&maps.xs);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(side_empty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * kI8gEpiWarps);
    }
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
      const uint32_t side_bytes = dense ? (split ? 3 : 2) * rch * 16384 : 16384;
      // programmatic dependent launch: the first tile's weight stages stream before
      // griddepcontrol.wait (they do not depend on the activation quantizer)
      const int pre = my_tiles > 0 ? (ks < S ? ks : S) : 0;
      for (int kk = 0; kk < pre; ++kk) {
        if (leader) mbar_expect_tx(&full[kk], 2u * (kI8A + kI8B + (has_r && kk == 0 ? side_bytes : 0)));
        tma_load_2d_pair(sb + kk * kI8gStage + kI8A, &maps.bp, map_rank(smem_u32(&full[kk]), 0), kk * 128,
                         (cluster_id / tiles_m) * 256 + int(rank) * 128, kEvictNormal);
      }
      pdl_wait();
      // stage slot and phase tracked incrementally (S is a runtime value: g % S, g / S would be
      // integer divides in the issue loop)
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < my_tiles; ++i) {
        const int tile = cluster_id + i * n_clusters;
        const int mt = tile % tiles_m, nt = tile / tiles_m;
        const int m_own = mt * 256 + int(rank) * 128;
        const int n_half = nt * 256 + int(rank) * 128;
        for (int kk = 0; kk < ks; ++kk, s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u) {
          const bool preloaded = i == 0 && kk < pre;
          if (!preloaded) mbar_wait(&empty[s], ph ^ 1);
          const bool with_side = has_r && kk == 0;
          if (with_side && i > 0) mbar_wait(side_empty, (i - 1) & 1);
          const uint32_t fbar = map_rank(smem_u32(&full[s]), 0);
          const uint32_t st = sb + s * kI8gStage;
          if (leader && !preloaded) mbar_expect_tx(&full[s], 2u * (kI8A + kI8B + (with_side ? side_bytes : 0)));
          if (!preloaded) tma_load_2d_pair(st + kI8A, &maps.bp, fbar, kk * 128, n_half, kEvictNormal);
          tma_load_2d_pair(st, &maps.a, fbar, kk * 128, m_own, kEvictNormal);
          if (with_side) {
            if (dense) {
              // bf16: 64 columns (128 B) per 16 KB swizzle atom
              for (int h = 0; h < rch; ++h) {
                tma_load_2d_pair(sside + h * 16384, &maps.xs, fbar, h * 64, m_own, kEvictNormal);
                tma_load_2d_pair(sside + 32768 + h * 16384, &maps.r, fbar, h * 64, n_half, kEvictNormal);
                if (split)  // lo plane: rows [N, 2N) of the same map
                  tma_load_2d_pair(sside + 65536 + h * 16384, &maps.r, fbar, h * 64, p.N + n_half, kEvictNormal);
              }
            } else {
              tma_load_2d_pair(sside, &maps.r, fbar, 0, n_half, kEvictNormal);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader && elect_one()) {
      const uint32_t sb = smem_u32(smem), sside = smem_u32(side);
      const uint32_t id_main = idesc_i8(256, 256, p.a_signed != 0, true);
      const uint32_t id_r = dense ? idesc_bf16(256, 256) : id_main;
      uint32_t u = 0;
      auto claim = [&](uint32_t unit) {  // accumulator (unit & 1) free again?
        if (unit >= 2) {
          mbar_wait(&acc_empty[unit & 1], ((unit >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        return (unit & 1) * 256u;
      };
      int s = 0, kg = 0;  // stage slot / phase and the K-step within the scale group, tracked incrementally
      uint32_t ph = 0;
      for (int i = 0; i < my_tiles; ++i) {
        for (int kk = 0; kk < ks; ++kk, s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u,
                 kg = (kg + 1 == p.gsteps) ? 0 : kg + 1) {
          mbar_wait_cluster(&full[s], ph);
          tc_fence_after();
          const uint32_t st = sb + s * kI8gStage;
          const uint64_t a = make_sdesc(st, 16, 1024, 2), b = make_sdesc(st + kI8A, 16, 1024, 2);
          if (has_r && kk == 0) {
            // salient term: its own unit
            const uint32_t d = claim(u);
            if (dense) {
              // K = 16 bf16 per MMA, four per 64-column atom
              for (int j = 0; j < (p.r + 15) / 16; ++j) {
                const uint32_t off = uint32_t(j >> 2) * 16384u;
                const uint64_t ad = make_sdesc(sside + off, 16, 1024, 2) + 2 * (j & 3);
                mma_bf16_pair(d, ad, make_sdesc(sside + 32768 + off, 16, 1024, 2) + 2 * (j & 3), id_r, j > 0 ? 1u : 0u);
                if (split) mma_bf16_pair(d, ad, make_sdesc(sside + 65536 + off, 16, 1024, 2) + 2 * (j & 3), id_r, 1u);
              }
            } else {
              const uint64_t br = make_sdesc(sside, 16, 1024, 2);
              for (int j = 0; j < (p.r + 31) / 32; ++j) mma_i8_pair(d, a + 2 * j, br + 2 * j, id_main, j > 0 ? 1u : 0u);
            }
            tc_commit_pair(side_empty);
            tc_commit_pair(&acc_full[u & 1]);
            ++u;
          }
          const uint32_t d = kg == 0 ? claim(u) : (u & 1) * 256u;
          for (int j = 0; j < 4; ++j) mma_i8_pair(d, a + 2 * j, b + 2 * j, id_main, (kg > 0 || j > 0) ? 1u : 0u);
          tc_commit_pair(&empty[s]);
          if (kg == p.gsteps - 1) {
            tc_commit_pair(&acc_full[u & 1]);
            ++u;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    pdl_wait();  // sx / zp / xs come from the quantizer; y may still be read by a predecessor
    pdl_launch_dependents();
    const uint32_t q = warp & 3;
    const int half = int(warp - 2) >> 2;        // column slice of the tile (kI8gCols wide)
    const int et = int(threadIdx.x) - 64;       // 0..32*kI8gEpiWarps-1
    const uint32_t lane_base = (q * 32u) << 16;
    uint8_t* stage_out = epi + (warp - 2) * 1024;  // 32 rows x 16 bf16 columns
    const uint32_t rbase = smem_u32(stage_out) + lane_id() * 32;
    const uint32_t acc_empty_leader = map_rank(smem_u32(&acc_empty[0]), 0);
    const int G = ks / p.gsteps;
    // scale of unit k of a tile at column n (0 past N)
    auto unit_scale = [&](int k, int n) -> float {
      if (n >= p.N) return 0.f;
      if (has_r) {
        if (k == 0) return dense ? 1.f : p.sr[n];
        --k;
      }
      return p.sw_g[size_t(k) * p.N + n];
    };
    uint32_t u = 0;
    if (my_tiles > 0) {
      const int tile0 = cluster_id;
      if (et < 256) sc[et] = unit_scale(0, (tile0 / tiles_m) * 256 + et);
    }
    named_bar_sync(2, 32 * kI8gEpiWarps);
    for (int i = 0; i < my_tiles; ++i) {
      const int tile = cluster_id + i * n_clusters;
      const int mt = tile % tiles_m, nt = tile / tiles_m;
      const int m_own = mt * 256 + int(rank) * 128;
      const int n0 = nt * 256;
      const int next_tile = tile + n_clusters;
      const int row = m_own + int(q) * 32 + int(lane_id());
      float sx = 0.f, zpf = 0.f;
      uint32_t zp = 0;
      if (row < p.M) {
        sx = p.sx[row];
        zp = p.zp ? uint32_t(p.zp[row]) : 0u;
        zpf = float(int32_t(zp));
      }
      if (et < 256) cst[et] = n0 + et < p.N ? p.cterm[n0 + et] : 0.f;  // read only after this tile's first unit barrier
      float acc[kI8gCols];
#pragma unroll
      for (int j = 0; j < kI8gCols; ++j) acc[j] = 0.f;
      for (int k = 0; k < units; ++k, ++u) {
        const uint32_t bsel = u & 1;
        // the next unit's scale for column et (next tile after the last unit)
        float nxt = 0.f;
        if (et >= 256) {
        } else if (k + 1 < units)
          nxt = unit_scale(k + 1, n0 + et);
        else if (i + 1 < my_tiles)
          nxt = unit_scale(0, (next_tile / tiles_m) * 256 + et);
        const bool is_dense = has_r && dense && k == 0;
        const bool is_r = has_r && k == 0;
        const int gi = has_r ? k - 1 : k;
        I8G_STAMP(u, 0);
        mbar_wait(&acc_full[bsel], (u >> 1) & 1);
        tc_fence_after();
        I8G_STAMP(u, 1);
        const uint32_t scu = smem_u32(sc + bsel * 256 + half * kI8gCols);
#pragma unroll
        for (int c = 0; c < kI8gCols / 16; ++c) {
          uint32_t v[16];
          tmem_ld_32x32b_x16(lane_base + bsel * 256u + uint32_t(half * kI8gCols + c * 16), v);
          tmem_ld_wait();
          if (c == 0) I8G_STAMP(u, 2);
          if (c == kI8gCols / 16 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive_cluster_relaxed(acc_empty_leader + bsel * 8u);
          }
          if (is_dense) {
#pragma unroll
            for (int j = 0; j < 16; j += 2)
              fadd2(acc[c * 16 + j], acc[c * 16 + j + 1], __uint_as_float(v[j]), __uint_as_float(v[j + 1]));
          } else {
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              uint32_t sv[4];
              ld_shared_v4u(scu + (c * 16 + 4 * j4) * 4, sv[0], sv[1], sv[2], sv[3]);
              // exact int32 -> fp32 (I2FP, |A_g| < 2^24), packed FFMA2 with the group scales
#pragma unroll
              for (int jj = 0; jj < 4; jj += 2) {
                const int j = 4 * j4 + jj;
                ffma2(acc[c * 16 + j], acc[c * 16 + j + 1], __int2float_rn(int32_t(v[j])),
                      __int2float_rn(int32_t(v[j + 1])), __uint_as_float(sv[jj]), __uint_as_float(sv[jj + 1]));
              }
            }
          }
          if (kDump && p.acc_dump && row < p.M && !is_dense) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = n0 + half * kI8gCols + c * 16 + j;
              if (n >= p.N) continue;
              if (is_r) {
                if (p.accr_dump) p.accr_dump[size_t(row) * p.N + n] = int32_t(v[j] - zp * uint32_t(p.colsum_r[n]));
              } else {
                p.acc_dump[(size_t(gi) * p.M + row) * p.N + n] =
                    int32_t(v[j] - zp * uint32_t(p.colsum_g[size_t(gi) * p.N + n]));
              }
            }
          }
        }
        I8G_STAMP(u, 3);
        if (et < 256) sc[(bsel ^ 1u) * 256 + et] = nxt;
        named_bar_sync(2, 32 * kI8gEpiWarps);  // next unit's scales (and this tile's C[n]) visible; old buffer free
        I8G_STAMP(u, 4);
      }
      (void)G;
      // ---- finalize: Y = sx * (acc - zp * C[n]) (+ addend) -> bf16, chunks of 16 columns
#pragma unroll
      for (int c = 0; c < kI8gCols / 16; ++c) {
        uint32_t packed[8];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int col = half * kI8gCols + c * 16 + j;
          float yv = (acc[c * 16 + j] - zpf * cst[col]) * sx;
          if (p.addend && row < p.M && n0 + col < p.N) yv += p.addend[size_t(row) * p.N + n0 + col];
          acc[c * 16 + j] = yv;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) packed[j] = pack_bf16x2(acc[c * 16 + 2 * j], acc[c * 16 + 2 * j + 1]);
        if (lane_id() == 0) bulk_wait_read_all();
        __syncwarp();
        st_shared_v4(rbase, packed[0], packed[1], packed[2], packed[3]);
        st_shared_v4(rbase + 16, packed[4], packed[5], packed[6], packed[7]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane_id() == 0 && m_own < p.M) {
          tma_store_2d(&maps.y, stage_out, n0 + half * kI8gCols + c * 16, m_own + int(q) * 32);
          bulk_commit();
        }
      }
      named_bar_sync(2, 32 * kI8gEpiWarps);  // every thread is done with cst before the next tile overwrites it
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
