// serq_gemm_decode3.cuh -- MXFP4 SERQ linear for decode (M <= 16): cluster
// split-K with a DSMEM reduction, optionally with the activation quantizer
// fused in.
//
// Swap-AB: D^T[128 weight rows, 16 tokens] = W_tile[128, K] . X^T -- weight
// rows are the MMA's M (128 per tile), the zero-padded <= 16 tokens its N
// (tcgen05.mma.cta_group::1.kind::mxf4, 128x16x64).  The tensor work is tiny;
// the kernel is bound by HBM bytes
//     N*K/2 (codes) + N*K/32 (E8M0) + N*r/2 + N*r/32 (R) + M*K*(1/2 + 1/32) (X) + 2*M*N (Y).  Each 128-row weight tile is handled by a CLUSTER of S CTAs
// (S = cluster size, <= 8) that split its K steps; the S fp32 partials
// (128 x 16 each) meet in the rank-0 CTA's shared memory over DSMEM and are
// summed in rank (= K) order -- deterministic, no global workspace, no flags,
// no float atomics.  (A global-memory reduction costs ~3 L2 round trips on the
// critical path of every layer, ~3 us measured; DSMEM ~0.2 us.)
//
// Fused quantizer (kFuse, M <= 8): the epilogue warps, idle during the main
// loop, take the K steps round-robin (warp c: steps c, c+4, ...; three of its
// steps' bf16 activations in flight in registers, L2 resident), encode them
// exactly like mx_encode (mxfmt.py:97-108: block
// exponent from the 32-block amax, RNE-to-E2M1 with saturation, -0 -> +0) and
// write the codes (128B-swizzled, the layout a TMA box would produce) and the
// E8M0 scale factors straight into the pipeline stage next to the TMA-loaded
// weights.  This removes the separate quantizer kernel and its two
// kernel-boundary dependencies from every decode step.
//
// Sized for layer-to-layer overlap: <= 116 KB of shared memory and 64 TMEM
// columns per CTA, so the NEXT linear's CTA fits on the same SM; with
// programmatic dependent launch (trigger at CTA start) it streams its first
// weight stages while this one finishes.
#pragma once
#include "serq_gemm.cuh"
#include "serq_gemm_i8.cuh"  // mbar_wait_cluster
#include "serq_quant.cuh"    // MX encode helpers

namespace serq {

constexpr int kDecN = 16;                              // tokens per MMA (padded)
constexpr int kDecW = 128 * kStepBytes;                // 16 KB weight tile per 256-K step
constexpr int kDecX = kDecN * kStepBytes;              // 2 KB token tile
constexpr int kDecSF = 1024;                           // 2 SF chunks of one 128-row block
constexpr int kDecStage = kDecW + kDecX + 2 * kDecSF;  // 20 KB (1 KB aligned)
// R tile: 128 rows x kRW bytes -- 32 B (r <= 64, 32-byte swizzle) or 64 B (64 < r <= 128,
// 64-byte swizzle, two K = 64 MMAs); smaller ranks are zero-padded at pack time
static_assert(kDecStage % 1024 == 0, "stage alignment");

struct DecodeMaps {
  CUtensorMap w, x, sfw, sfx, r, sfr;
  CUtensorMap xs, sfxs;  // gather fallback: the quantizer's x[:, idx] codes (32-B rows) and scale factors
};

constexpr int kClThreads = 192;
constexpr int kClXs = 512 + 512;     // gather fallback: 16 rows x 32 B of x[:, idx] codes + one SF atom
constexpr int kClRed = 6 * 1024;     // rank-0 landing buffer for narrow partials ((S-1) x ceil(M/4) x 2 KB)
// fused quantizer: kP (token row, 32-block) pairs per lane, M <= 4 kP; used for M <= 8 (at
// M = 16 the 4-pair converter was slower than the quantizer kernel + PDL: 10.5 vs 8.6 us)
constexpr int kClFuseM = 8;
#ifndef SERQ_DEC_STAGES
#define SERQ_DEC_STAGES 5  // weight stages per CTA (diagnostic builds may raise it: one CTA per SM)
#endif
template <bool kFuse, int kRW = 32>
struct ClCfg {
  static constexpr int kStages = kRW == 64 ? SERQ_DEC_STAGES - 1 : SERQ_DEC_STAGES;  // the 8 KB R tile costs one stage
  static constexpr int kDecRB = 128 * kRW;
  static constexpr int kSmem = 1024 + kStages * kDecStage + kDecRB + 512 + kClXs + kClRed + 512;
  // 228 KB per SM, 1 KB reserved per CTA
  static_assert(SERQ_DEC_STAGES > 5 || 2 * (kSmem + 1024) <= 228 * 1024,
                "two CTAs (this linear and the next) must fit on one SM");
  static_assert(kSmem + 1024 <= 228 * 1024, "one CTA must fit");
  static_assert(7 * 128 * kDecN * 4 <= kStages * kDecStage, "rank-0 reduction buffer reuses the stages");
};

struct ClParams {
  int M, N, K, r;
  int k_steps, S;        // K steps per tile, CTAs per tile (cluster size)
  int kc_pad, kc_pad_r, w_ksteps;
  int gather;            // the salient term's B operand is the quantizer's x[:, idx] slice, not K-tile 0 of X
  int nseg;              // fused linears: weight-row segments, each with its own salient slice of 128
  int seg_row[3];        //   columns in the xs buffer (segment j+1 starts at output row seg_row[j])
  int red_narrow;        // partials carry only the M token columns and land in a dedicated buffer
  __nv_bfloat16* y;
  int64_t ldy;
  long long* dbg_ts;     // diagnostics (SERQ_DIAG_TS builds): [cta][8] globaltimer stamps
  // fused quantizer: bf16 activations (row pitch ldx); the tile-0 cluster also
  // writes the quantized activation (codes [M, K/2], scale factors tiled) if non-null
  const __nv_bfloat16* x;
  int64_t ldx;
  uint8_t* codes_out;
  uint8_t* sf_out;
};

#ifdef SERQ_DIAG_TS
#define CL_STAMP(i)                                                                      \
  if (p.dbg_ts) {                                                                        \
    uint64_t g_;                                                                         \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                              \
    p.dbg_ts[blockIdx.x * 8 + (i)] = (long long)g_;                                      \
  }
// per-step SM-clock stamps of CTA 0: [8192 + 64 * kind + step]
#define CL_STEP(kind, i)                                                                 \
  if (p.dbg_ts && blockIdx.x == 0 && (i) < 64) p.dbg_ts[8192 + 64 * (kind) + (i)] = clock64();
#else
#define CL_STAMP(i)
#define CL_STEP(kind, i)
#endif

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

template <bool kFuse, int kP = 1, int kRW = 32>
__global__ void __launch_bounds__(kClThreads, 2) serq_mx_decode_cl_kernel(const __grid_constant__ DecodeMaps maps,
                                                                          const ClParams p) {
  static_assert(kRW == 32 || kRW == 64, "R rows of 32 or 64 bytes");
  constexpr int kClStages = ClCfg<kFuse, kRW>::kStages;
  constexpr int kDecRB = ClCfg<kFuse, kRW>::kDecRB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* rbuf = smem + kClStages * kDecStage;  // R tile (4 KB) + R scale factors (512 B)
  uint8_t* xsbuf = rbuf + kDecRB + 512;           // gather: x[:, idx] codes (512 B) + SF atom (512 B)
  float* redbuf = reinterpret_cast<float*>(xsbuf + kClXs);  // narrow reduction: [S-1][ceil(M/4)][128][4]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsbuf + kClXs + kClRed);
  uint64_t* full = bars;                  // [kClStages]
  uint64_t* empty = bars + kClStages;     // [kClStages]
  uint64_t* rfull = bars + 2 * kClStages;
  uint64_t* done = rfull + 1;             // accumulator complete
  uint64_t* red_free = done + 1;          // rank > 0: rank 0's buffer may be written
  uint64_t* red_full = red_free + 1;      // rank 0: every partial has landed
  uint64_t* xsfull = red_full + 1;        // gather: the salient slice landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xsfull + 1);

  pdl_launch_dependents();  // the next linear may launch once every CTA is resident
  const uint32_t warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) CL_STAMP(0);
  const int S = p.S;
  const int rank = int(cluster_rank());
  const int tile = int(blockIdx.x) / S;
  const int n0 = tile * 128;
  const int k0 = (rank * p.k_steps) / S, k1 = ((rank + 1) * p.k_steps) / S;
  const int nsteps = k1 - k0;
  const bool with_r = p.r > 0 && rank == 0;
  constexpr uint32_t kWBytes = kDecW + kDecSF;  // TMA bytes per stage when X is produced in-kernel

  if (warp == 0 && elect_one()) {
    tma_prefetch(&maps.w);
    tma_prefetch(&maps.sfw);
    if (!kFuse) {
      tma_prefetch(&maps.x);
      tma_prefetch(&maps.sfx);
    }
    for (int s = 0; s < kClStages; ++s) {
      mbar_init(&full[s], kFuse ? 2 : 1);  // + the converter warp of the step
      mbar_init(&empty[s], 1);
    }
    mbar_init(rfull, 1);
    mbar_init(done, 1);
    mbar_init(red_free, 1);
    mbar_init(red_full, S > 1 ? (S - 1) * 128 : 1);
    mbar_init(xsfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<64>(tmem_slot);
  if (kFuse) {
    // X rows >= 4 kP of every stage stay zero, and scale-factor atom rows >= 4 kP (never
    // produced) get a finite scale; the converters rewrite rows < 4 kP every step
    for (int s = 0; s < kClStages; ++s) {
      for (int b = threadIdx.x; b < (kDecX - 4 * kP * 128) / 16; b += blockDim.x)
        reinterpret_cast<uint4*>(smem + s * kDecStage + kDecW + 4 * kP * 128)[b] = make_uint4(0, 0, 0, 0);
      for (int b = threadIdx.x; b < 2 * 512 / 16; b += blockDim.x)
        reinterpret_cast<uint4*>(smem + s * kDecStage + kDecW + kDecX + kDecSF)[b] = make_uint4(
            0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  if (S > 1) cluster_sync_all();  // barrier inits visible cluster-wide before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // [0,16) accumulator, [16,24) SFA, [24,32) SFB, [32,36) R SFA, [36,40) xs SFB

  if (warp == 0) {
    if (elect_one()) {
      auto load_w = [&](int s, int kk) {
        uint8_t* st = smem + s * kDecStage;
        mbar_expect_tx(&full[s], kFuse ? kWBytes : kDecStage);
        tma_load_2d(st, &maps.w, &full[s], 0, (tile * p.w_ksteps + kk) * 128, kEvictFirst);
        tma_load_2d(st + kDecW + kDecX, &maps.sfw, &full[s], 0, (tile * p.kc_pad + 2 * kk) * 4, kEvictFirst);
      };
      if (with_r) {  // R does not depend on the previous kernel either
        mbar_expect_tx(rfull, kDecRB + 512);
        tma_load_2d(rbuf, &maps.r, rfull, 0, n0, kEvictFirst);
        tma_load_2d(rbuf + kDecRB, &maps.sfr, rfull, 0, (tile * p.kc_pad_r) * 4, kEvictFirst);
      }
      const int pre = min(nsteps, kClStages);
      for (int i = 0; i < pre; ++i) load_w(i, k0 + i);
      pdl_wait();  // activations (bf16 or codes) come from the previous kernel
      CL_STAMP(1);
      if (!kFuse && with_r && p.gather) {
        int seg = 0;  // fused linears: this tile's segment picks its 128-column slice of xs
        for (int j = 0; j + 1 < p.nseg; ++j) seg += n0 >= p.seg_row[j] ? 1 : 0;
        mbar_expect_tx(xsfull, kClXs);
        tma_load_2d(xsbuf, &maps.xs, xsfull, seg * 64, 0, kEvictLast);
        tma_load_2d(xsbuf + 512, &maps.sfxs, xsfull, 0, seg * 4, kEvictLast);
      }
      for (int i = 0; i < nsteps; ++i) {
        const int s = i % kClStages;
        if (i >= pre) {
          mbar_wait(&empty[s], ((i / kClStages) & 1) ^ 1);
          load_w(s, k0 + i);
        }
        CL_STEP(0, i);
        if (!kFuse) {
          uint8_t* st = smem + s * kDecStage;
          tma_load_2d(st + kDecW, &maps.x, &full[s], (k0 + i) * kStepBytes, 0, kEvictLast);
          tma_load_2d(st + kDecW + kDecX + kDecSF, &maps.sfx, &full[s], 0, (2 * (k0 + i)) * 4, kEvictLast);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t id0 = idesc_mxf4(128, kDecN), id1 = id0 | (2u << 4) | (2u << 29);
      const uint32_t acc = tmem, sfa = tmem + 16, sfb = tmem + 24, sfr = tmem + 32, sfxs = tmem + 36;
      for (int i = 0; i < nsteps; ++i) {
        const int s = i % kClStages;
        mbar_wait(&full[s], (i / kClStages) & 1);
        tc_fence_after();
        CL_STEP(2, i);
        if (i == 0) CL_STAMP(2);
        const uint32_t st = smem_u32(smem + s * kDecStage);
        const uint64_t a = make_sdesc(st, 16, 1024, 2), b = make_sdesc(st + kDecW, 16, 1024, 2);
        const uint32_t sa = st + kDecW + kDecX, sb = sa + kDecSF;
        tmem_cp_32x128b_x4(sfa, make_sdesc(sa, 128, 128, 0));
        tmem_cp_32x128b_x4(sfa + 4, make_sdesc(sa + 512, 128, 128, 0));
        tmem_cp_32x128b_x4(sfb, make_sdesc(sb, 128, 128, 0));
        tmem_cp_32x128b_x4(sfb + 4, make_sdesc(sb + 512, 128, 128, 0));
        mma_mxf4(acc, a, b, id0, sfa, sfb, i > 0 ? 1u : 0u);
        mma_mxf4(acc, a + 2, b + 2, id1, sfa | (2u << 30), sfb | (2u << 30), 1u);
        mma_mxf4(acc, a + 4, b + 4, id0, sfa + 4, sfb + 4, 1u);
        mma_mxf4(acc, a + 6, b + 6, id1, (sfa + 4) | (2u << 30), (sfb + 4) | (2u << 30), 1u);
        if (with_r && i == 0) {
          // salient term: A = R rows (K = r = 64), B = K-tile 0 of X (this stage), SFB = X chunk 0
          mbar_wait(rfull, 0);
          tc_fence_after();
          tmem_cp_32x128b_x4(sfr, make_sdesc(smem_u32(rbuf + kDecRB), 128, 128, 0));
          if (!kFuse && p.gather) {
            // gather fallback: B = the quantizer's x[:, idx] slice (16 rows x 32 B, 32B swizzle)
            mbar_wait(xsfull, 0);
            tc_fence_after();
            tmem_cp_32x128b_x4(sfxs, make_sdesc(smem_u32(xsbuf + 512), 128, 128, 0));
            mma_mxf4(acc, make_sdesc(smem_u32(rbuf), 16, 256, 6), make_sdesc(smem_u32(xsbuf), 16, 256, 6), id0, sfr,
                     sfxs, 1u);
          } else if constexpr (kRW == 32) {
            mma_mxf4(acc, make_sdesc(smem_u32(rbuf), 16, 256, 6), b, id0, sfr, sfb, 1u);
          } else {
            // r in (64, 128]: R rows of 64 B (64-byte swizzle), K-tile 0 of X as two K = 64 slices
            const uint64_t rd = make_sdesc(smem_u32(rbuf), 16, 512, 4);
            mma_mxf4(acc, rd, b, id0, sfr, sfb, 1u);
            mma_mxf4(acc, rd + 2, b + 2, id1, sfr | (2u << 30), sfb | (2u << 30), 1u);
          }
        }
        tc_commit(&empty[s]);
      }
      CL_STAMP(3);
      if (nsteps > 0) tc_commit(done);
      else mbar_arrive(done);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ warps 2..5
    const uint32_t q = warp & 3;  // TMEM lane quadrant
    const int et = int(q * 32 + lane_id());
    pdl_wait();  // codes_out / Y writes after the previous kernel
    if constexpr (kFuse) {
      // X converter: warp c converts K steps c, c + 4, ... (four steps in flight, so the
      // per-step latency -- L2 load, encode, shared store, proxy fence -- is hidden);
      // lane -> 32-block part = lane % 8 of token rows lane / 8 + 4 p (p < kP) of the 16 x 256 tile
      constexpr int kDepth = kP == 1 ? 3 : 2;  // steps of this warp in flight in registers (<= 168 regs)
      const int cw = int(warp) - 2;
      const int m0 = int(lane_id()) >> 3, part = int(lane_id()) & 7;
      auto load_x = [&](int i, uint4 (&v)[kP][4]) {
        const int kk = k0 + i;
#pragma unroll
        for (int pp = 0; pp < kP; ++pp) {
          const int m = m0 + 4 * pp;
          const bool ok = i < nsteps && m < p.M && kk * 256 + part * 32 < p.K;  // K % 32 == 0
          const uint4* src = reinterpret_cast<const uint4*>(p.x + int64_t(m) * p.ldx + kk * 256 + part * 32);
#pragma unroll
          for (int c = 0; c < 4; ++c) v[pp][c] = ok ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
        }
      };
      auto put_x = [&](int i, const uint4 (&cur)[kP][4]) {
        const int s = i % kClStages;
        const int kk = k0 + i;
        uint32_t pk[kP][4];
        int ex[kP];
#pragma unroll
        for (int pp = 0; pp < kP; ++pp) {
          // 32-element block exactly as mx_encode_blk_kernel: abs-max tree, exponent, RNE to E2M1
          uint32_t w[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            w[4 * c] = cur[pp][c].x;
            w[4 * c + 1] = cur[pp][c].y;
            w[4 * c + 2] = cur[pp][c].z;
            w[4 * c + 3] = cur[pp][c].w;
          }
          uint32_t m8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = bf16x2_absmax(w[2 * k], w[2 * k + 1]);
#pragma unroll
          for (int k = 0; k < 4; ++k) m8[k] = bf16x2_absmax(m8[2 * k], m8[2 * k + 1]);
          m8[0] = bf16x2_absmax(bf16x2_absmax(m8[0], m8[1]), bf16x2_absmax(m8[2], m8[3]));
          m8[0] = bf16x2_absmax(m8[0], __byte_perm(m8[0], 0, 0x1032));
          const uint32_t amax = m8[0] & 0x7FFFu;
          const int e = amax ? max(int(amax >> 7), 2) - 129 : 0;
          const float inv = __uint_as_float(uint32_t(127 - e) << 23);
          ex[pp] = e;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t packed = 0;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const uint32_t wv = w[4 * k + h];
              packed |= cvt_e2m1x2_raw(__uint_as_float(wv << 16) * inv, __uint_as_float(wv & 0xFFFF0000u) * inv)
                        << (8 * h);
            }
            pk[pp][k] = canon_neg_zero3(packed);
          }
        }
        if (i >= kClStages) mbar_wait(&empty[s], ((i / kClStages) & 1) ^ 1);
        if (i == 0 && lane_id() == 0) CL_STEP(4, 0);
        uint8_t* st = smem + s * kDecStage;
#pragma unroll
        for (int pp = 0; pp < kP; ++pp) {
          const int m = m0 + 4 * pp;
          // codes: row m, 16-B chunk `part` of the 128-B row, 128B swizzle (chunk ^ row % 8)
          st_shared_v4(smem_u32(st + kDecW + m * 128 + ((part ^ (m & 7)) * 16)), pk[pp][0], pk[pp][1], pk[pp][2],
                       pk[pp][3]);
          // scale factor: chunk part/4, atom row m, byte part%4
          st[kDecW + kDecX + kDecSF + (part >> 2) * 512 + m * 16 + (part & 3)] = uint8_t(ex[pp] + 127);
          if (p.codes_out != nullptr && tile == 0 && m < p.M && kk * 256 + part * 32 < p.K) {
            *reinterpret_cast<uint4*>(p.codes_out + int64_t(m) * (p.K / 2) + kk * 128 + part * 16) =
                make_uint4(pk[pp][0], pk[pp][1], pk[pp][2], pk[pp][3]);
            p.sf_out[sf_offset(m, kk * 8 + part, p.kc_pad)] = uint8_t(ex[pp] + 127);
          }
        }
        fence_proxy_async_smem();  // generic-proxy smem writes -> the tensor core's async proxy
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&full[s]);
        if (lane_id() == 0) CL_STEP(5, i);
      };
      uint4 buf[kDepth][kP][4];
#pragma unroll
      for (int d = 0; d < kDepth; ++d) load_x(cw + 4 * d, buf[d]);
      for (int i = cw; i < nsteps; i += 4 * kDepth) {
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
          if (i + 4 * d < nsteps) put_x(i + 4 * d, buf[d]);
          load_x(i + 4 * (d + kDepth), buf[d]);
        }
      }
    }
    // ---- accumulator -> Y (S == 1) or the rank-0 DSMEM reduction
    mbar_wait(done, 0);
    tc_fence_after();
    if (q == 0 && lane_id() == 0) CL_STAMP(4);
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((q * 32u) << 16)));
    tmem_ld_wait();
    if (nsteps == 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0u;
    }
    const int row = et;  // TMEM lane = weight row within the tile
    float out[kDecN];
#pragma unroll
    for (int j = 0; j < kDecN; ++j) out[j] = __uint_as_float(v[j]);
    bool store = true;
    if (S > 1 && p.red_narrow) {
      // narrow: ceil(M/4) float4 per row straight into rank 0's dedicated buffer, no invitation
      const int mq = (p.M + 3) >> 2;
      if (rank == 0) {
        mbar_wait_cluster(red_full, 0);
        for (int sl = 0; sl < S - 1; ++sl)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < mq) {
              const float4 t4 = reinterpret_cast<const float4*>(redbuf)[(sl * mq + k) * 128 + row];
              out[4 * k] += t4.x;
              out[4 * k + 1] += t4.y;
              out[4 * k + 2] += t4.z;
              out[4 * k + 3] += t4.w;
            }
      } else {
        const uint32_t dst = map_rank(smem_u32(redbuf + ((rank - 1) * mq * 128 + row) * 4), 0u);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < mq) st_cluster_v4(dst + k * 128 * 16, out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
        mbar_arrive_release_cluster(map_rank(smem_u32(red_full), 0u));
        store = false;
      }
    } else if (S > 1) {
      float* red = reinterpret_cast<float*>(smem);  // rank 0: [S-1][128][16] fp32 (the stages are drained)
      if (rank == 0) {
        // every MMA of this CTA is complete, so its stage memory is free: invite the partials
        if (et < S - 1) mbar_arrive_release_cluster(map_rank(smem_u32(red_free), uint32_t(et + 1)));
        mbar_wait_cluster(red_full, 0);
        for (int sl = 0; sl < S - 1; ++sl) {
          const float4* src = reinterpret_cast<const float4*>(red + (size_t(sl) * 128 + row) * kDecN);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 t4 = src[k];
            out[4 * k] += t4.x;
            out[4 * k + 1] += t4.y;
            out[4 * k + 2] += t4.z;
            out[4 * k + 3] += t4.w;
          }
        }
      } else {
        mbar_wait_cluster(red_free, 0);
        const uint32_t dst = map_rank(smem_u32(red + (size_t(rank - 1) * 128 + row) * kDecN), 0u);
#pragma unroll
        for (int k = 0; k < 4; ++k) st_cluster_v4(dst + 16 * k, out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
        mbar_arrive_release_cluster(map_rank(smem_u32(red_full), 0u));
        store = false;
      }
    }
    const int n = n0 + row;
    if (store && n < p.N) {
#pragma unroll
      for (int m = 0; m < kDecN; ++m)
        if (m < p.M) p.y[m * p.ldy + n] = __float2bfloat16_rn(out[m]);
    }
  }
  if (warp == 4 && lane_id() == 0) CL_STAMP(5);
  tc_fence_before();
  if (S > 1) cluster_sync_all();  // no CTA leaves while a peer may still touch its shared memory
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
  if (threadIdx.x == 0) CL_STAMP(6);
}

}  // namespace serq
