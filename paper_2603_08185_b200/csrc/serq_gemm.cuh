// serq_gemm.cuh -- the SERQ linear: Y = Xq.Wq + Xs,q.R with the salient term
// fused into the same kernel (tcgen05 + TMEM + TMA, sm_100a).
//
// Replaces the reference's two-GEMM composition in forward_reconstructed
// (compensate.py:300-316, int branch) and _forward_mx (compensate.py:319-340).
//
// One CTA computes a 128 x kBN output tile.  Warp roles (192 threads):
//   warp 0      TMA producer (A/B tiles via 2-D tensor maps, scale factors via bulk copy)
//   warp 1      TMEM allocator + single-thread MMA issuer
//   warps 2..5  epilogue (TMEM -> registers -> dequant -> bf16 -> smem -> TMA store)
// K is walked in 128-byte steps (256 FP4 / 128 INT8 codes); the salient term
// is one or more extra pipeline steps that read the salient activation slice
// and the compensation matrix R:
//   MX  : R steps accumulate into the SAME fp32 accumulator (block scales
//         make the two products commensurable) -- no second GEMM, no add.
//   INT : R steps accumulate into a second TMEM accumulator (s32 for an
//         integer R, f32 for a bf16 R via kind::f16) that the epilogue
//         combines with the main accumulator under the per-token x
//         per-channel scales.
#pragma once
#include "serq_ptx.cuh"

namespace serq {

enum GemmMode : int { kModeMX = 0, kModeI8 = 1 };
enum RMode : int { kRNone = 0, kRDense = 1, kRInt = 2, kRDenseSplit = 3 };

constexpr int kBM = 128;
constexpr int kBN = 256;
constexpr int kStepBytes = 128;  // K bytes per pipeline step (one 128B swizzle row)
constexpr int kStages = 4;
constexpr int kThreads = 192;
constexpr int kSmemA = kBM * kStepBytes;             // 16 KB
constexpr int kSmemB = kBN * kStepBytes;             // 32 KB
constexpr int kSmemSFA = 2 * 512;                    // 2 SF chunks (128 K each) x 128 rows
constexpr int kSmemSFB = 2 * 512 * (kBN / 128);      // 2 chunks x 2 row blocks
constexpr int kStageBytes = kSmemA + kSmemB + kSmemSFA + kSmemSFB;  // 51 KB (1024-aligned)
static_assert(kStageBytes % 1024 == 0, "stage must keep 1 KB alignment");
constexpr int kEpiConstBytes = 4 * kBN * 4;
constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + kEpiConstBytes + 256;

// TMEM column map (512 allocated): [0,256) main accumulator, [256,512) either the
// second accumulator (INT + R) or the per-stage scale factors (MX).
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kSfCols = 8 + 16;  // per stage: SFA 2 chunks x 4 cols, SFB 2 chunks x 8 cols

struct GemmParams {
  int M, N, K;           // K in elements
  int r;                 // salient rank (0 = no R term)
  int k_steps;           // ceil(K bytes / 128)
  int r_steps;           // ceil(R bytes / 128)
  int r_mode;            // RMode
  int a_signed;          // INT: activation codes s8 (sym) or u8 (asym)
  // MX scale factors, tiled [row_blocks][kc_pad][512]
  const uint8_t* sfa;
  const uint8_t* sfb;
  const uint8_t* sfa_r;  // SF of the salient activation slice (== sfa when contiguous)
  const uint8_t* sfb_r;  // SF of R
  int kc_pad;            // SF chunks per row block (A and B), even
  int w_ksteps;          // MX weights are pre-tiled [N/128][w_ksteps][128 rows x 128 B]
  int kc_pad_r;          // SF chunks per row block for R and the salient slice
  int xs_is_x;           // salient slice = leading columns of X (no side buffer)
  int kc_pad_xs;         // SF chunks per row block of the quantizer's salient slice buffer
  int nseg;              // fused linears: weight-row segments with their own 128-column xs slices
  int seg_row[3];        //   (segment j+1 starts at output row seg_row[j])
  // INT epilogue operands
  const float* sx;       // [M] per-token scale
  const int32_t* zp;     // [M] zero point (asym) or nullptr
  const float* sw;       // [N] per-output-channel weight scale
  const int32_t* colsum; // [N] sum_k W[k,n] (for the zero-point correction)
  const float* sr;       // [N] R scale (int R)
  const int32_t* colsum_r;
  const float* addend;   // optional fp32 [M, N] (pitch N) added after scaling (SVD-baseline correction;
                         // MX: the CTA-pair pair3 and one-CTA persistent kernels)
  int32_t* acc_dump;     // debug: exact main accumulators (acc - zp*colsum), [M,N]
  int32_t* accr_dump;    // debug: exact R accumulators
  long long* dbg_ts;     // diagnostics: per-iteration clock64 stamps of the MMA warp (CTA 0), or nullptr
  int narrow_from;       // pair3: tiles >= narrow_from run as two 256 x 128 tiles (>= n_tiles: none)
  const uint8_t* w4;     // INT CTA-pair kernel, W4 weights: packed int4 tiled [N/128][K/128][128][64 B]
  int group_m;           // tile order: 0 = M fastest over all tiles; g > 0 = groups of g M-tiles
  int dbg;               // SERQ_DIAG builds only (diagnostic switches); always 0 in the product
};

template <int kMode>
__global__ void __launch_bounds__(kThreads, 1)
    serq_linear_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       const __grid_constant__ CUtensorMap map_xs, const __grid_constant__ CUtensorMap map_r,
                       const __grid_constant__ CUtensorMap map_y, const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_f = reinterpret_cast<float*>(smem + kStages * kStageBytes);      // sw | sr
  int32_t* epi_i = reinterpret_cast<int32_t*>(epi_f + 2 * kBN);                // colsum | colsum_r
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_i + 2 * kBN);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* acc_full = bars + 2 * kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);

  const uint32_t warp = threadIdx.x >> 5;
  const int m0 = blockIdx.x * kBM;
  const int n0 = blockIdx.y * kBN;
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
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  if (kMode == kModeI8 && warp >= 2) {
    // per-column epilogue constants for this tile
    for (int i = threadIdx.x - 64; i < kBN; i += 128) {
      const int n = n0 + i;
      const bool ok = n < p.N;
      epi_f[i] = ok ? p.sw[n] : 0.f;
      epi_i[i] = (ok && p.zp) ? p.colsum[n] : 0;
      epi_f[kBN + i] = (ok && p.r_mode == kRInt) ? p.sr[n] : 0.f;
      epi_i[kBN + i] = (ok && p.zp && p.r_mode == kRInt) ? p.colsum_r[n] : 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      const int mblk = m0 / 128;
      for (int it = 0; it < n_iters; ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * kStageBytes;
        const bool rstep = it >= p.k_steps;
        const int kk = rstep ? it - p.k_steps : it;  // step index within its operand
        uint32_t bytes = kSmemA + kSmemB;
        if (kMode == kModeMX) bytes += kSmemSFA + kSmemSFB;
        mbar_expect_tx(&full[s], bytes);
        if (!rstep) {
          tma_load_2d(st, &map_a, &full[s], kk * kStepBytes, m0, kEvictNormal);
          tma_load_2d(st + kSmemA, &map_b, &full[s], kk * kStepBytes, n0, kEvictNormal);
        } else {
          // tensor-map coordinates are in elements: a 128-byte step is 64 bf16 (dense R)
          const int rc = (kMode != kModeMX && p.r_mode == kRDense) ? kk * (kStepBytes / 2) : kk * kStepBytes;
          if (p.xs_is_x)
            tma_load_2d(st, &map_a, &full[s], rc, m0, kEvictNormal);
          else
            tma_load_2d(st, &map_xs, &full[s], rc, m0, kEvictNormal);
          tma_load_2d(st + kSmemA, &map_r, &full[s], rc, n0, kEvictNormal);
        }
        if (kMode == kModeMX) {
          const uint8_t* sa = rstep ? p.sfa_r : p.sfa;
          const uint8_t* sb = rstep ? p.sfb_r : p.sfb;
          const int kca = rstep && !p.xs_is_x ? p.kc_pad_r : p.kc_pad;
          const int kcb = rstep ? p.kc_pad_r : p.kc_pad;
          bulk_load(st + kSmemA + kSmemB, sa + (size_t(mblk) * kca + 2 * kk) * 512, 1024, &full[s]);
#pragma unroll
          for (int b = 0; b < kBN / 128; ++b)
            bulk_load(st + kSmemA + kSmemB + kSmemSFA + b * 1024,
                      sb + (size_t(n0 / 128 + b) * kcb + 2 * kk) * 512, 1024, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t acc = tmem_base;
    const uint32_t acc2 = tmem_base + 256;
    for (int it = 0; it < n_iters; ++it) {
      const int s = it % kStages;
      const uint32_t ph = (it / kStages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        uint8_t* st = smem + s * kStageBytes;
        const bool rstep = it >= p.k_steps;
        // number of 32-byte MMA K-slices in this step
        int nk = 4;
        if (rstep) {
          const int rbytes = (kMode == kModeMX) ? p.r / 2 : (p.r_mode == kRDense ? 2 * p.r : p.r);
          const int rem = rbytes - (it - p.k_steps) * kStepBytes;
          nk = rem >= kStepBytes ? 4 : (rem + 31) / 32;
        }
        const uint64_t adesc0 = sdesc_k_sw128(st);
        const uint64_t bdesc0 = sdesc_k_sw128(st + kSmemA);
        if (kMode == kModeMX) {
          const uint32_t sfa_t = tmem_base + 256 + s * kSfCols;
          const uint32_t sfb_t = sfa_t + 8;
          uint8_t* ssfa = st + kSmemA + kSmemB;
          uint8_t* ssfb = ssfa + kSmemSFA;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            tmem_cp_32x128b_x4(sfa_t + c * 4, make_sdesc(smem_u32(ssfa + c * 512), 128, 128, 0));
#pragma unroll
            for (int b = 0; b < kBN / 128; ++b)
              tmem_cp_32x128b_x4(sfb_t + c * 8 + b * 4,
                                 make_sdesc(smem_u32(ssfb + b * 1024 + c * 512), 128, 128, 0));
          }
          constexpr uint32_t idesc = idesc_mxf4(kBM, kBN);
          for (int j = 0; j < nk; ++j) {
            const uint32_t sfid = (j & 1) * 2;
            const uint32_t id = idesc | (sfid << 4) | (sfid << 29);
            mma_mxf4(acc, adesc0 + (j * 32 >> 4), bdesc0 + (j * 32 >> 4), id,
                     (sfa_t + (j >> 1) * 4) | (sfid << 30), (sfb_t + (j >> 1) * 8) | (sfid << 30),
                     (it > 0 || j > 0) ? 1u : 0u);
          }
        } else {
          if (!rstep) {
            const uint32_t id = idesc_i8(kBM, kBN, p.a_signed != 0, true);
            for (int j = 0; j < nk; ++j)
              mma_i8(acc, adesc0 + (j * 32 >> 4), bdesc0 + (j * 32 >> 4), id, (it > 0 || j > 0) ? 1u : 0u);
          } else {
            const int rj = it - p.k_steps;
            if (p.r_mode == kRDense) {
              constexpr uint32_t id = idesc_bf16(kBM, kBN);
              for (int j = 0; j < nk; ++j)
                mma_bf16(acc2, adesc0 + (j * 32 >> 4), bdesc0 + (j * 32 >> 4), id, (rj > 0 || j > 0) ? 1u : 0u);
            } else {
              const uint32_t id = idesc_i8(kBM, kBN, p.a_signed != 0, true);
              for (int j = 0; j < nk; ++j)
                mma_i8(acc2, adesc0 + (j * 32 >> 4), bdesc0 + (j * 32 >> 4), id, (rj > 0 || j > 0) ? 1u : 0u);
            }
          }
        }
        tc_commit(&empty[s]);
        if (it == n_iters - 1) tc_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = m0 + q * 32 + lane_id();
    mbar_wait(acc_full, 0);
    tc_fence_after();
    float sx = 1.f;
    int32_t zp = 0;
    if (kMode == kModeI8 && row < p.M) {
      sx = p.sx[row];
      zp = p.zp ? p.zp[row] : 0;
    }
    // staging: reuse pipeline smem (all MMAs and loads are done).  Each warp
    // owns 32 rows: 4 boxes of 32 rows x 64 bf16 (128 B, 128B-swizzled).
    uint8_t* stage_out = smem + q * (32 * 512);
    const uint32_t lane_base = (q * 32u) << 16;
#pragma unroll 1
    for (int c = 0; c < kBN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem_base + lane_base + c * 32, v);
      uint32_t w[32];
      const bool need2 = (kMode == kModeI8) && p.r_mode != kRNone;
      if (need2) tmem_ld_32x32b_x32(tmem_base + 256 + lane_base + c * 32, w);
      tmem_ld_wait();
      float f[32];
      if (kMode == kModeMX) {
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int col = c * 32 + i;
          const int32_t a = int32_t(v[i]) - zp * epi_i[col];
          float y = float(a) * epi_f[col];
          if (p.acc_dump && row < p.M && n0 + col < p.N) p.acc_dump[size_t(row) * p.N + n0 + col] = a;
          if (need2) {
            if (p.r_mode == kRDense) {
              y += __uint_as_float(w[i]);
            } else {
              const int32_t ar = int32_t(w[i]) - zp * epi_i[kBN + col];
              y += float(ar) * epi_f[kBN + col];
              if (p.accr_dump && row < p.M && n0 + col < p.N) p.accr_dump[size_t(row) * p.N + n0 + col] = ar;
            }
          }
          f[i] = y * sx;
          if (p.addend && row < p.M && n0 + col < p.N) f[i] += p.addend[size_t(row) * p.N + n0 + col];
        }
      }
      // 32 fp32 -> 64 B of bf16 = four 16-B chunks of a 128-B swizzled row
      uint8_t* box = stage_out + (c >> 1) * (32 * 128);
      const uint32_t rbase = smem_u32(box) + lane_id() * 128;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t chunk = ((c & 1) * 4 + j) ^ (lane_id() & 7);
        st_shared_v4(rbase + chunk * 16, pack_bf16x2(f[8 * j], f[8 * j + 1]), pack_bf16x2(f[8 * j + 2], f[8 * j + 3]),
                     pack_bf16x2(f[8 * j + 4], f[8 * j + 5]), pack_bf16x2(f[8 * j + 6], f[8 * j + 7]));
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane_id() == 0) {
#pragma unroll
      for (int b = 0; b < kBN / 64; ++b) tma_store_2d(&map_y, stage_out + b * (32 * 128), n0 + b * 64, m0 + q * 32);
      bulk_commit();
      bulk_wait_read_all();
    }
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
