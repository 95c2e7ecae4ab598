// serq_gemv_i8.cuh -- integer SERQ linear at decode sizes (M <= 16 tokens).
//
// Y[t, n] = sx[t] * ( sw[n] * (acc[t, n] - zp[t] * colsum[n]) + R-term ),
// acc[t, n] = sum_k c[t, k] w[n, k]        (int_gemm_reference, mxfmt.py:177-195;
//                                           forward_reconstructed, compensate.py:300-316)
//
// At M <= 16 the layer is a weight stream (K x N int8 bytes), so the kernel is sized for HBM,
// not for the tensor pipe: a CTA owns 16 weight rows and its 4 or 8 warps split K; each lane streams
// 16-byte pieces of two weight rows with non-allocating loads, several 64-byte K chunks in
// flight, and the products run as warp-level tensor-core MMAs (mma.sync m16n8k32, s8 weights x
// u8 / s8 codes, s32 exact; the <= 16 tokens are the n8 side), far below the stream's time.
// K-permutation: a lane holds bytes [16q, 16q + 16) of a 64-byte chunk of its row; the MMA pair
// of that chunk reads them as logical k {4q..4q+3, 16+4q..} (bytes 0-7) and the same for bytes
// 8-15 -- the activation fragments are loaded with the identical permutation, and a sum over k
// does not depend on its order.  The warps' accumulator fragments meet in shared memory; the
// zero-point correction is exact in wrapping int32 as in the CTA-pair kernel.  The salient term:
// integer R (int8 [N, r] x the permuted slice = the first r codes, or the quantizer's gathered
// codes; own scale and zero-point correction) or dense R (bf16 [N, r] x the quantizer's bf16
// (codes - zp) slice, mma.sync m16n8k16 in fp32).
#pragma once
#include "serq_ptx.cuh"
#include "serq_gemm_i8.cuh"  // widen_int4x8

// minimum resident CTAs: 5 of the 4 + 1-warp CTAs (<= 80 registers: the whole grid of a
// 11008-row layer in one wave), 2 of the wider ones (<= 112)
#ifndef SERQ_GEMV_MINB4
#define SERQ_GEMV_MINB4 5
#endif
#ifndef SERQ_GEMV_MINB8
#define SERQ_GEMV_MINB8 2
#endif

namespace serq {

struct GemvI8Params {
  const int8_t* w;          // [N, K] int8, K-major rows; kW4: packed INT4 tiled [N/128][K/128][128 rows][64 B]
  int K, N, M;
  const uint8_t* a;         // [M, K] activation codes (u8 asymmetric / s8 symmetric)
  const float* sx;          // [M]
  const int32_t* zp;        // [M] or nullptr (symmetric)
  const float* sw;          // [N]
  const int32_t* colsum;    // [N]
  int r;                    // salient rank
  const void* rw;           // int8 [N, r] (integer R) / bf16 [N, r] (dense R)
  const float* sr;          // [N] integer-R scale
  const int32_t* colsum_r;  // [N]
  const void* xs;           // integer R: gathered codes [M, r] (nullptr: the first r codes of a);
                            // dense R: bf16 (codes - zp) [M, r]
  __nv_bfloat16* y;         // [M, ldy]
  int64_t ldy;
  const float* addend;      // optional fp32 [M, N] added after scaling (the SVD-baseline path)
  int32_t* acc_dump;        // tests: exact accumulators acc - zp * colsum, [M, N] (group-wise: [G][M][N])
  int32_t* accr_dump;       // tests: exact integer-R accumulators
  // group-wise weights (row groups of gchunks 64-K chunks, serq_pack_int_grouped; the i8g kernel's
  // promotion): Y = sx * (sum_g sw_g[g, n] A_g + R term - zp * cterm[n])
  const float* sw_g;        // [G][N]
  const float* cterm;       // [N] sum_g sw_g * colsum_g (+ sr * colsum_r)
  const int32_t* colsum_g;  // [G][N] (dumps only)
  int groups, gchunks;
};

template <bool kSigned>
__device__ __forceinline__ void mma_s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
  if constexpr (kSigned)
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// one 64-byte K chunk: A = weight rows g / g + 8 (16 B each, bytes 16q..), B = token rows
// f * 8 + g (16 B each); two m16n8k32 per token fragment
template <int kNT, bool kSigned>
__device__ __forceinline__ void gemv_mma_chunk(const uint4& wlo, const uint4& whi, const uint4 (&b)[kNT],
                                               int (&acc)[kNT][4]) {
#pragma unroll
  for (int f = 0; f < kNT; ++f) {
    mma_s8<kSigned>(acc[f], wlo.x, whi.x, wlo.y, whi.y, b[f].x, b[f].y);
    mma_s8<kSigned>(acc[f], wlo.z, whi.z, wlo.w, whi.w, b[f].z, b[f].w);
  }
}

// kNT: token fragments of 8 (1: M <= 8, 2: M <= 16); kR: 0 no salient term, kRInt, kRDense;
// kWarps: warps splitting K (8 when there are few row groups, 4 otherwise: one wave of CTAs);
// kW4: the weights are the CTA-pair kernel's packed INT4 layout (pack_int4_tiled_kernel: per
// 128-row tile and 128-K step, 64 B per row, so a CTA's 16 rows are one contiguous 1 KB); a K
// "chunk" is then 128 elements, a lane's 16 B are its rows' elements [32q, 32q + 32) of it, widened
// in registers (widen_int4x8, natural order) to the two 16-B pieces the int8 path would have loaded
// kFmt: 0 int8 weights, one scale per output column; 1 packed INT4 (kW4 below); 2 group-wise int8
// weights (kG): every main warp owns whole groups, promotes each group's exact s32 partial with its
// scale in fp32 (scales staged in shared memory before the wait) and the side warp applies the
// folded zero-point term, as serq_i8g_pair_kernel does
constexpr int kGemvMaxGpw = 32;  // groups per main warp (group-wise: G <= 32 * warps)
template <int kNT, bool kSigned, int kR, int kWarps, int kFmt = 0>
__global__ void __launch_bounds__(32 * (kWarps + 1), kWarps == 4 ? SERQ_GEMV_MINB4 : SERQ_GEMV_MINB8) serq_i8_gemv_kernel(const GemvI8Params p) {
  constexpr bool kW4 = kFmt == 1, kG = kFmt == 2;
  __shared__ int red_i[kWarps][kNT][32][4];  // [main warp][fragment][lane][c] (group-wise: fp32 bits)
  __shared__ float sgr[kG ? kWarps * kGemvMaxGpw * 16 : 1];  // group-wise: [warp][group][row] scales
  pdl_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int row0 = blockIdx.x * 16;
  // tokens: blockIdx.y selects 16 of them (M > 16: each token group re-streams the weights, mostly
  // from L2); t below is the token within the group
  const int t0 = blockIdx.y * 16, mloc = min(16, p.M - t0);
  const int rlo = row0 + g, rhi = row0 + g + 8;
  const bool ok_lo = rlo < p.N, ok_hi = rhi < p.N;
  if (warp < kWarps) {
    // ---- main warps: this warp's K chunks (64 elements each; 128 packed INT4), a contiguous 1 / kWarps
    constexpr int kChunk = kW4 ? 128 : 64;
    const int nch = (p.K + kChunk - 1) / kChunk;
    const int gpw = kG ? (p.groups + kWarps - 1) / kWarps : 0;
    const int per = kG ? gpw * p.gchunks : (nch + kWarps - 1) / kWarps;
    const int c0 = warp * per, c1 = min(nch, c0 + per);
    if constexpr (kG) {  // this warp's group scales for its 16 rows (weights: before the wait)
      for (int j = lane; j < gpw * 16; j += 32) {
        const int gi = warp * gpw + (j >> 4), n = row0 + (j & 15);
        sgr[(warp * kGemvMaxGpw + (j >> 4)) * 16 + (j & 15)] =
            (gi < p.groups && n < p.N) ? __ldg(p.sw_g + size_t(gi) * p.N + n) : 0.f;
      }
      __syncwarp();
    }
    const int8_t* wlo_p;
    const int8_t* whi_p;
    size_t cstride;  // bytes from one chunk of a row to the next
    if constexpr (kW4) {
      const int rl = ok_lo ? rlo : 0, rh = ok_hi ? rhi : 0;
      wlo_p = p.w + (size_t(rl >> 7) * nch * 128 + (rl & 127)) * 64 + 16 * q;
      whi_p = p.w + (size_t(rh >> 7) * nch * 128 + (rh & 127)) * 64 + 16 * q;
      cstride = 128 * 64;
    } else {
      wlo_p = p.w + size_t(ok_lo ? rlo : 0) * p.K + 16 * q;
      whi_p = p.w + size_t(ok_hi ? rhi : 0) * p.K + 16 * q;
      cstride = 64;
    }
    auto wload = [&](const int8_t* base, bool ok, int c) {
      // (W4: the packed tail beyond K is zero nibbles, written at pack time)
      return (ok && c < c1 && (kW4 || c * 64 + 16 * q < p.K)) ? ld_stream16(base + size_t(c) * cstride)
                                                               : make_uint4(0, 0, 0, 0);
    };
    // the first weight chunks do not depend on the previous kernel: in flight before the wait
    constexpr int kAhead = kWarps > 4 ? 6 : 4;  // chunks per row in flight per lane
    uint4 wl[kAhead], wh[kAhead];
#pragma unroll
    for (int u = 0; u < kAhead; ++u) {
      wl[u] = wload(wlo_p, ok_lo, c0 + u);
      wh[u] = wload(whi_p, ok_hi, c0 + u);
    }
    pdl_wait();  // activation codes come from the quantizer
    int acc[kNT][4];
    float facc[kNT][4];  // group-wise: the promoted partials
#pragma unroll
    for (int f = 0; f < kNT; ++f)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[f][i] = 0;
        facc[f][i] = 0.f;
      }
    int gc = 0, gl = 0;  // group-wise: chunks into the current group, group index within the warp
    // group-wise: fold the finished group's exact partial (and dump it for the tests)
    auto fold = [&]() {
      const float s_lo = sgr[(warp * kGemvMaxGpw + gl) * 16 + g], s_hi = sgr[(warp * kGemvMaxGpw + gl) * 16 + g + 8];
      const int gi = warp * gpw + gl;
#pragma unroll
      for (int f = 0; f < kNT; ++f)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (p.acc_dump) {
            const int n = i >= 2 ? rhi : rlo, t = f * 8 + 2 * q + (i & 1);
            if (n < p.N && t < mloc) {
              const uint32_t zp = p.zp ? uint32_t(p.zp[t0 + t]) : 0u;
              p.acc_dump[(size_t(gi) * p.M + t0 + t) * p.N + n] =
                  int32_t(uint32_t(acc[f][i]) - zp * uint32_t(p.colsum_g[size_t(gi) * p.N + n]));
            }
          }
          facc[f][i] = fmaf(float(acc[f][i]), i >= 2 ? s_hi : s_lo, facc[f][i]);
          acc[f][i] = 0;
        }
      gc = 0;
      ++gl;
    };
    // the token fragments of the 16 activation bytes at element k of each token row
    auto act = [&](int k, uint4 (&b)[kNT]) {
#pragma unroll
      for (int f = 0; f < kNT; ++f) {
        const int t = f * 8 + g;
        b[f] = (t < mloc && k < p.K) ? __ldg(reinterpret_cast<const uint4*>(p.a + size_t(t0 + t) * p.K + k))
                                    : make_uint4(0, 0, 0, 0);
      }
    };
    for (int c = c0; c < c1; c += kAhead) {
#pragma unroll
      for (int u = 0; u < kAhead; ++u) {
        const uint4 lo = wl[u], hi = wh[u];
        wl[u] = wload(wlo_p, ok_lo, c + u + kAhead);
        wh[u] = wload(whi_p, ok_hi, c + u + kAhead);
        if (c + u < c1) {
          uint4 b[kNT];
          if constexpr (kW4) {
            const uint2 l0 = widen_int4x8(lo.x), l1 = widen_int4x8(lo.y), l2 = widen_int4x8(lo.z),
                        l3 = widen_int4x8(lo.w);
            const uint2 h0 = widen_int4x8(hi.x), h1 = widen_int4x8(hi.y), h2 = widen_int4x8(hi.z),
                        h3 = widen_int4x8(hi.w);
            const int k = (c + u) * 128 + 32 * q;
            act(k, b);
            gemv_mma_chunk<kNT, kSigned>(make_uint4(l0.x, l0.y, l1.x, l1.y), make_uint4(h0.x, h0.y, h1.x, h1.y), b,
                                         acc);
            act(k + 16, b);
            gemv_mma_chunk<kNT, kSigned>(make_uint4(l2.x, l2.y, l3.x, l3.y), make_uint4(h2.x, h2.y, h3.x, h3.y), b,
                                         acc);
          } else {
            act((c + u) * 64 + 16 * q, b);
            gemv_mma_chunk<kNT, kSigned>(lo, hi, b, acc);
          }
          if constexpr (kG) {
            if (++gc == p.gchunks || c + u + 1 == c1) fold();
          }
        }
      }
    }
#pragma unroll
    for (int f = 0; f < kNT; ++f)
#pragma unroll
      for (int i = 0; i < 4; ++i) red_i[warp][f][lane][i] = kG ? __float_as_int(facc[f][i]) : acc[f][i];
    __syncthreads();
    return;
  }
  // ---- the side warp: the salient term and the epilogue.  Its weights (R rows, r <= 128) and
  // the per-column constants do not depend on the previous kernel either: loaded before the
  // wait, so after it only the activation reads and the main warps' results remain.
  int32_t cs[2] = {0, 0}, csr[2] = {0, 0};
  float swv[2] = {0.f, 0.f}, srv[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int n = h ? rhi : rlo;
    if (n < p.N) {
      if constexpr (kG) {
        swv[h] = __ldg(p.cterm + n);  // (group-wise: the folded zero-point term)
      } else {
        cs[h] = __ldg(p.colsum + n);
        swv[h] = __ldg(p.sw + n);
      }
      if constexpr (kR == kRInt) {
        csr[h] = __ldg(p.colsum_r + n);
        srv[h] = __ldg(p.sr + n);
      }
    }
  }
  int accr[kNT][4];   // integer R: exact s32
  float accd[kNT][4]; // dense R: fp32
#pragma unroll
  for (int f = 0; f < kNT; ++f)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      accr[f][i] = 0;
      accd[f][i] = 0.f;
    }
  if constexpr (kR == kRInt) {
    const int8_t* rw = static_cast<const int8_t*>(p.rw);
    uint4 rwl[2], rwh[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const bool in = c * 64 + 16 * q < p.r;
      rwl[c] = (ok_lo && in) ? __ldg(reinterpret_cast<const uint4*>(rw + size_t(rlo) * p.r + c * 64 + 16 * q))
                             : make_uint4(0, 0, 0, 0);
      rwh[c] = (ok_hi && in) ? __ldg(reinterpret_cast<const uint4*>(rw + size_t(rhi) * p.r + c * 64 + 16 * q))
                             : make_uint4(0, 0, 0, 0);
    }
    pdl_wait();
    const uint8_t* ar = p.xs ? static_cast<const uint8_t*>(p.xs) : p.a;
    const int lda = p.xs ? p.r : p.K;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const bool in = c * 64 + 16 * q < p.r;
      uint4 b[kNT];
#pragma unroll
      for (int f = 0; f < kNT; ++f) {
        const int t = f * 8 + g;
        b[f] = (t < mloc && in) ? __ldg(reinterpret_cast<const uint4*>(ar + size_t(t0 + t) * lda + c * 64 + 16 * q))
                               : make_uint4(0, 0, 0, 0);
      }
      gemv_mma_chunk<kNT, kSigned>(rwl[c], rwh[c], b, accr);
    }
  } else if constexpr (kR == kRDense || kR == kRDenseSplit) {
    const __nv_bfloat16* xs = static_cast<const __nv_bfloat16*>(p.xs);
    // 16-element chunks (r <= 128: eight): a lane holds elements [4q, 4q + 4) (logical k {2q, 2q+1, 2q+8, 2q+9});
    // split R: the bf16 hi plane (rows [0, N)) then the lo plane (rows [N, 2N)) into the same fp32 sum
#pragma unroll
    for (int plane = 0; plane < (kR == kRDenseSplit ? 2 : 1); ++plane) {
      const __nv_bfloat16* rw = static_cast<const __nv_bfloat16*>(p.rw) + size_t(plane) * p.N * p.r;
      uint2 rl[8], rh[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const bool in = c * 16 + 4 * q < p.r;
        rl[c] = (ok_lo && in) ? *reinterpret_cast<const uint2*>(rw + size_t(rlo) * p.r + c * 16 + 4 * q) : make_uint2(0, 0);
        rh[c] = (ok_hi && in) ? *reinterpret_cast<const uint2*>(rw + size_t(rhi) * p.r + c * 16 + 4 * q) : make_uint2(0, 0);
      }
      if (plane == 0) pdl_wait();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const bool in = c * 16 + 4 * q < p.r;
#pragma unroll
        for (int f = 0; f < kNT; ++f) {
          const int t = f * 8 + g;
          const uint2 b = (t < mloc && in) ? *reinterpret_cast<const uint2*>(xs + size_t(t0 + t) * p.r + c * 16 + 4 * q)
                                          : make_uint2(0, 0);
          mma_bf16(accd[f], rl[c].x, rh[c].x, rl[c].y, rh[c].y, b.x, b.y);
        }
      }
    }
  } else {
    pdl_wait();
  }
  // per-token scale / zero point (written by the quantizer): after the wait
  float sxv[kNT][2];
  uint32_t zpv[kNT][2];
#pragma unroll
  for (int f = 0; f < kNT; ++f)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int t = f * 8 + 2 * q + j;
      sxv[f][j] = t < mloc ? __ldg(p.sx + t0 + t) : 0.f;
      zpv[f][j] = (p.zp && t < mloc) ? uint32_t(__ldg(p.zp + t0 + t)) : 0u;
    }
  __syncthreads();
  // lane (g, q) of fragment f holds rows g / g + 8, tokens f * 8 + 2q / 2q + 1
#pragma unroll
  for (int f = 0; f < kNT; ++f)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int h = i >> 1;
      const int n = h ? rhi : rlo;
      const int t = f * 8 + 2 * q + (i & 1);
      if (n >= p.N || t >= mloc) continue;
      const uint32_t zp = zpv[f][i & 1];
      float yv;
      if constexpr (kG) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += __int_as_float(red_i[w][f][lane][i]);
        yv = s;
        if constexpr (kR == kRInt) {
          yv = fmaf(float(accr[f][i]), srv[h], yv);  // raw: sr * colsum_r is in cterm
          if (p.accr_dump) p.accr_dump[size_t(t0 + t) * p.N + n] = int32_t(uint32_t(accr[f][i]) - zp * uint32_t(csr[h]));
        } else if constexpr (kR == kRDense || kR == kRDenseSplit) {
          yv += accd[f][i];
        }
        yv -= float(zp) * swv[h];
      } else {
        int s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += red_i[w][f][lane][i];  // exact
        const int32_t a_ref = int32_t(uint32_t(s) - zp * uint32_t(cs[h]));  // wrapping int32, exact
        yv = float(a_ref) * swv[h];
        if constexpr (kR == kRInt) {
          const int32_t ar_ref = int32_t(uint32_t(accr[f][i]) - zp * uint32_t(csr[h]));
          yv += float(ar_ref) * srv[h];
          if (p.accr_dump) p.accr_dump[size_t(t0 + t) * p.N + n] = ar_ref;
        } else if constexpr (kR == kRDense || kR == kRDenseSplit) {
          yv += accd[f][i];
        }
        if (p.acc_dump) p.acc_dump[size_t(t0 + t) * p.N + n] = a_ref;
      }
      float out = yv * sxv[f][i & 1];
      if (p.addend) out += p.addend[size_t(t0 + t) * p.N + n];
      p.y[size_t(t0 + t) * p.ldy + n] = __float2bfloat16_rn(out);
    }
}

}  // namespace serq
