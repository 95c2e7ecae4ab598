// serq_quant.cuh -- activation quantizers (K1) and offline weight packers.
//
// Bit-exact restatements of the reference quantizers on the device:
//   quantize_symmetric / quantize_asymmetric  (quantcore.py:108-137)
//   mx_encode / _block_exponents / e2m1_nearest (mxfmt.py:52-108)
// Device layouts:
//   MX codes   : uint8 [rows, K/2], element 2i in the low nibble (mxfmt.py:245-247 convention)
//   MX scales  : E8M0 (= e + 127) tiled [ceil(rows/128)][kc_pad][512]; inside a 512-B atom
//                row m, 32-block kb sit at (m%32)*16 + ((m%128)/32)*4 + kb%4, kc = kb/4
//   INT codes  : int8 [rows, K] (s8 symmetric, u8 asymmetric)
#pragma once
#include "serq_ptx.cuh"

namespace serq {

__host__ __device__ __forceinline__ size_t sf_offset(int64_t row, int64_t kb, int kc_pad) {
  return (size_t(row >> 7) * kc_pad + size_t(kb >> 2)) * 512 + size_t(row & 31) * 16 + size_t((row >> 5) & 3) * 4 +
         size_t(kb & 3);
}

template <typename T>
struct In;
template <>
struct In<__nv_bfloat16> {
  static constexpr int kId = 0;
  __device__ static float f(__nv_bfloat16 v) { return __bfloat162float(v); }
};
template <>
struct In<float> {
  static constexpr int kId = 1;
  __device__ static float f(float v) { return v; }
};
template <>
struct In<double> {
  static constexpr int kId = 2;
};

// E2M1 magnitude index for an exactly-scaled value, ties to the even index,
// saturating at 6 (software path, exact for double inputs).
__device__ __forceinline__ uint32_t e2m1_index_sw(double a) {
  // decision points 0.25 0.75 1.25 1.75 2.5 3.5 5
  uint32_t i;
  if (a < 0.25) i = 0;
  else if (a == 0.25) i = 0;
  else if (a < 0.75) i = 1;
  else if (a == 0.75) i = 2;
  else if (a < 1.25) i = 2;
  else if (a == 1.25) i = 2;
  else if (a < 1.75) i = 3;
  else if (a == 1.75) i = 4;
  else if (a < 2.5) i = 4;
  else if (a == 2.5) i = 4;
  else if (a < 3.5) i = 5;
  else if (a == 3.5) i = 6;
  else if (a < 5.0) i = 6;
  else if (a == 5.0) i = 6;
  else i = 7;
  return i;
}

// two f32 (exact after the power-of-two scaling) -> packed e2m1x2 byte, lo = even element
// (hardware RNE + satfinite; cuda_fp4.hpp operand order: first source -> high nibble).
__device__ __forceinline__ uint32_t cvt_e2m1x2_raw(float even, float odd) {
  uint32_t out;
  asm("{\n .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n cvt.u32.u8 %0, t;\n}\n"
      : "=r"(out)
      : "f"(odd), "f"(even));
  return out;
}
// -0 (code 8) -> +0 on eight packed nibbles (the reference emits +0 for values
// rounding to zero, mxfmt.py:67): clear the sign of every zero-magnitude nibble.
__device__ __forceinline__ uint32_t canon_neg_zero(uint32_t p) {
  const uint32_t mag = p & 0x77777777u;
  const uint32_t z = ~(mag | (mag >> 1) | (mag >> 2)) & 0x11111111u;
  return p & ~(z << 3);
}
// the same in three ops: bit 3 of (mag + 7) per nibble is (mag != 0), no carry between nibbles
__device__ __forceinline__ uint32_t canon_neg_zero3(uint32_t p) {
  const uint32_t b = (p & 0x77777777u) + 0x77777777u;
  return p & (b | 0x77777777u);
}
__device__ __forceinline__ uint32_t cvt_e2m1x2(float even, float odd) {
  return canon_neg_zero(cvt_e2m1x2_raw(even, odd));
}

// block exponent e = floor(log2 amax) - 2 (0 for amax == 0), clipped to [-127, 127]
__device__ __forceinline__ int mx_block_exp_f32(float amax) {
  if (amax == 0.f) return 0;
  const int ef = int((__float_as_uint(amax) >> 23) & 0xFF);
  return max(ef - 127 - 2, -127);  // subnormal (ef == 0) -> clipped -127
}
__device__ __forceinline__ int mx_block_exp_f64(double amax) {
  if (amax == 0.0) return 0;
  const int ef = int((__double_as_longlong(amax) >> 52) & 0x7FF);
  return min(max(ef - 1023 - 2, -127), 127);
}

// ------------------------------------------------------------------ MX encode
// Thread t handles 8 consecutive elements of one row; 4 threads form a 32-block.
// Blocks [0, nb_main) encode X; blocks beyond encode the gathered salient slice
// X[:, idx] (the reference re-encodes it, compensate.py:335).
template <typename T>
__global__ void __launch_bounds__(256) mx_encode_kernel(const T* __restrict__ x, int64_t M, int64_t K, int64_t ldx,
                                                        uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
                                                        int kc_pad, const int32_t* __restrict__ gidx, int r,
                                                        uint8_t* __restrict__ xs_codes, uint8_t* __restrict__ xs_sf,
                                                        int kc_pad_r, int64_t nb_main) {
  const bool gather = blockIdx.x >= nb_main;
  const int64_t cols = gather ? r : K;
  const int64_t t = int64_t(gather ? blockIdx.x - nb_main : blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per_row = cols / 8;
  const int64_t total = M * per_row;
  const bool active = t < total;
  const int64_t row = active ? t / per_row : 0;
  const int64_t c0 = active ? (t - row * per_row) * 8 : 0;
  uint8_t* out_codes = gather ? xs_codes : codes;
  uint8_t* out_sf = gather ? xs_sf : sf;
  const int kcp = gather ? kc_pad_r : kc_pad;

  if constexpr (In<T>::kId == 2) {
    double v[8];
    double amax = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t col = gather ? gidx[c0 + i] : c0 + i;
      v[i] = active ? x[row * ldx + col] : 0.0;
      amax = fmax(amax, fabs(v[i]));
    }
    amax = fmax(amax, __shfl_xor_sync(0xffffffff, amax, 1));
    amax = fmax(amax, __shfl_xor_sync(0xffffffff, amax, 2));
    const int e = mx_block_exp_f64(amax);
    if (!active) return;
    const double inv = ldexp(1.0, -e);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double s = v[i] * inv;  // exact: power-of-two scaling
      uint32_t idx = e2m1_index_sw(fabs(s));
      const uint32_t code = (s < 0.0 && idx > 0) ? idx + 8 : idx;
      packed |= code << (4 * i);
    }
    *reinterpret_cast<uint32_t*>(out_codes + row * (cols / 2) + c0 / 2) = packed;
    if ((threadIdx.x & 3) == 0) out_sf[sf_offset(row, c0 / 32, kcp)] = uint8_t(e + 127);
  } else {
    float v[8];
    if (!gather) {
      if (active) {
        if constexpr (In<T>::kId == 0) {
          const uint4 raw = *reinterpret_cast<const uint4*>(x + row * ldx + c0);
          const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(h[i]);
        } else {
          const float4 a = *reinterpret_cast<const float4*>(x + row * ldx + c0);
          const float4 b = *reinterpret_cast<const float4*>(x + row * ldx + c0 + 4);
          v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0.f;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = active ? In<T>::f(x[row * ldx + gidx[c0 + i]]) : 0.f;
    }
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(v[i]));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 2));
    const int e = mx_block_exp_f32(amax);
    if (!active) return;
    // 2^-e in f32: e in [-127, 125] -> 2^127 .. 2^-125, both normal
    const float inv = __uint_as_float(uint32_t(127 - e) << 23);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) packed |= cvt_e2m1x2(v[2 * i] * inv, v[2 * i + 1] * inv) << (8 * i);
    *reinterpret_cast<uint32_t*>(out_codes + row * (cols / 2) + c0 / 2) = packed;
    if ((threadIdx.x & 3) == 0) out_sf[sf_offset(row, c0 / 32, kcp)] = uint8_t(e + 127);
  }
}

// Fast path for bf16 / f32 rows: 2-D grid (x: 2048-column chunks, y: kMxRows-row
// groups); each thread keeps kMxRows independent 16-B loads in flight and emits a
// 32-bit word of 8 packed codes per row.  For bf16 the block amax is an integer
// 16-bit SIMD max over |x| bit patterns (monotonic for finite bf16) and the
// exponent comes straight from those bits, so the only float work is the exact
// power-of-two scaling feeding cvt.rn.satfinite.e2m1x2.
constexpr int kMxRows = 4;  // default rows per thread
__device__ __forceinline__ int mx_block_exp_bf16bits(uint32_t amax_bits) {
  // amax_bits: 15-bit magnitude of a bf16; exponent field = bits >> 7
  const int ef = int(amax_bits >> 7);
  return amax_bits == 0 ? 0 : (ef == 0 ? -127 : max(ef - 129, -127));
}
// The salient slice x[:, idx] of a non-permuted layer (compensate.py:335 re-encodes it;
// the common case for q/k/v and gate/up) -- encoded by the z = 1 plane of the
// fast quantizer's grid, concurrently with the main encode instead of in a second launch.
struct MxGather {
  const int32_t* idx;
  int r;
  uint8_t* xs_codes;
  uint8_t* xs_sf;
  int kc_pad_r;
};

template <typename T>
__device__ __forceinline__ void mx_encode_gather_part(const T* __restrict__ x, int M, int64_t ldx, const MxGather& g,
                                                      int64_t blk = -1) {
  if (blk < 0) blk = int64_t(blockIdx.y) * gridDim.x + blockIdx.x;
  const int64_t t = blk * blockDim.x + threadIdx.x;
  const int per_row = g.kc_pad_r * 16;  // 8-element groups incl. the SF chunk padding beyond r
  const int64_t total = int64_t(((M + 127) >> 7) << 7) * per_row;  // rows padded to the SF tile
  if (blk * blockDim.x >= total) return;  // whole CTA idle
  const bool active = t < total;
  const int64_t row = active ? t / per_row : 0;
  const int c0 = active ? int(t - row * per_row) * 8 : 0;
  const bool row_ok = active && row < M && c0 < g.r;
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = row_ok ? In<T>::f(x[row * ldx + g.idx[c0 + i]]) : 0.f;
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(v[i]));
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 1));
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 2));
  const int e = mx_block_exp_f32(amax);
  if (!active) return;
  const float inv = __uint_as_float(uint32_t(127 - e) << 23);
  uint32_t packed = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) packed |= cvt_e2m1x2(v[2 * i] * inv, v[2 * i + 1] * inv) << (8 * i);
  if (row_ok) *reinterpret_cast<uint32_t*>(g.xs_codes + row * (g.r / 2) + c0 / 2) = packed;
  if ((threadIdx.x & 3) == 0) g.xs_sf[sf_offset(row, c0 / 32, g.kc_pad_r)] = uint8_t(e + 127);
}

// max(|a|, |b|) per bf16 lane (sign = xor of the signs; only the magnitude is used)
__device__ __forceinline__ uint32_t bf16x2_absmax(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// K1-MX for bf16 input, one thread per (32-block, kR rows): the block amax needs no
// shuffles, the exponent is computed once per block, codes leave as one 16-B store and
// the scale factor as one byte.  Bit-identical to mx_encode_fast_kernel (same exponent,
// scaling and RNE conversion); ~half the ALU work per element, which bounds that kernel.
// The grid covers the scale-factor padding (rows up to the 128-row block, blocks up to
// kc_pad chunks) with the finite scale of a zero block, as mx_encode_fast_kernel does.
template <int kR>
__global__ void __launch_bounds__(256) mx_encode_blk_kernel(const __nv_bfloat16* __restrict__ x, int M, int K,
                                                            int64_t ldx, uint8_t* __restrict__ codes,
                                                            uint8_t* __restrict__ sf, int kc_pad,
                                                            MxGather gather = MxGather{}) {
  const int nbp = kc_pad * 4;  // 32-blocks per row including the SF chunk padding
  // the gathered salient slice runs in extra CTAs past the main grid (same launch; measured
  // faster than placing them first: 9.4 vs 11.0 us at 4096^2, r = 64)
  const int64_t main_blocks = (((((M + 127) >> 7) << 7) + kR - 1) / kR * int64_t(nbp) + 255) / 256;
  if (int64_t(blockIdx.x) >= main_blocks) {
    pdl_launch_dependents();
    pdl_wait();
    if (gather.idx) mx_encode_gather_part<__nv_bfloat16>(x, M, ldx, gather, int64_t(blockIdx.x) - main_blocks);
    return;
  }
  const int64_t id = int64_t(blockIdx.x) * 256 + threadIdx.x;
  const int kb = int(id % nbp);
  const int r0 = int(id / nbp) * kR;
  const int m_sf = ((M + 127) >> 7) << 7;
  pdl_launch_dependents();  // the linear may start streaming its weights now
  pdl_wait();               // x comes from the previous kernel
  if (r0 >= m_sf) return;
  const bool col_ok = kb * 32 < K;  // K % 32 == 0: blocks are all in or all out
  uint4 raw[kR][4];
#pragma unroll
  for (int rr = 0; rr < kR; ++rr) {
    const bool ok = col_ok && r0 + rr < M;
    const uint4* src = reinterpret_cast<const uint4*>(x + int64_t(r0 + rr) * ldx + kb * 32);
#pragma unroll
    for (int c = 0; c < 4; ++c) raw[rr][c] = ok ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int rr = 0; rr < kR; ++rr) {
    const int row = r0 + rr;
    uint32_t w[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      w[4 * c] = raw[rr][c].x;
      w[4 * c + 1] = raw[rr][c].y;
      w[4 * c + 2] = raw[rr][c].z;
      w[4 * c + 3] = raw[rr][c].w;
    }
    uint32_t m8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m8[i] = bf16x2_absmax(w[2 * i], w[2 * i + 1]);
#pragma unroll
    for (int i = 0; i < 4; ++i) m8[i] = bf16x2_absmax(m8[2 * i], m8[2 * i + 1]);
    m8[0] = bf16x2_absmax(bf16x2_absmax(m8[0], m8[1]), bf16x2_absmax(m8[2], m8[3]));
    m8[0] = bf16x2_absmax(m8[0], __byte_perm(m8[0], 0, 0x1032));  // both halves
    const uint32_t amax = m8[0] & 0x7FFFu;
    // mx_block_exp_bf16bits without branches: 0 for a zero block, else max(ef, 2) - 129
    const int ef = int(amax >> 7);
    const int e = amax ? max(ef, 2) - 129 : 0;
    const float inv = __uint_as_float(uint32_t(127 - e) << 23);
    uint32_t pk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t packed = 0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const uint32_t wv = w[4 * k + h];
        packed |= cvt_e2m1x2_raw(__uint_as_float(wv << 16) * inv, __uint_as_float(wv & 0xFFFF0000u) * inv)
                  << (8 * h);
      }
      pk[k] = canon_neg_zero3(packed);
    }
    if (col_ok && row < M)
      *reinterpret_cast<uint4*>(codes + int64_t(row) * (K >> 1) + kb * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    if (row < m_sf) sf[sf_offset(row, kb, kc_pad)] = uint8_t(e + 127);
  }
}

template <typename T, int kMxRows = serq::kMxRows>
__global__ void __launch_bounds__(256) mx_encode_fast_kernel(const T* __restrict__ x, int M, int K, int64_t ldx,
                                                             uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
                                                             int kc_pad, MxGather gather = MxGather{}) {
  if (blockIdx.z == 1) {
    pdl_launch_dependents();
    pdl_wait();
    mx_encode_gather_part<T>(x, M, ldx, gather);
    return;
  }
  const int c8 = blockIdx.x * 256 + threadIdx.x;  // 8-element group within the row
  const int r0 = blockIdx.y * kMxRows;
  const bool col_ok = c8 < (K >> 3);
  // the grid also covers the scale-factor padding (rows up to the 128-row block,
  // blocks up to kc_pad chunks): those get the finite scale of a zero block, so
  // no memset (which would break the programmatic-dependent-launch chain) is needed
  const bool sf_col_ok = c8 < kc_pad * 16;
  const int m_sf = ((M + 127) >> 7) << 7;
  pdl_launch_dependents();  // the linear may start streaming its weights now
  pdl_wait();               // launched as a dependent itself: x comes from the previous kernel
  if constexpr (In<T>::kId == 0) {
    const uint4* src = reinterpret_cast<const uint4*>(x + int64_t(r0) * ldx) + c8;
    const int64_t stride = ldx >> 3;
    uint4 raw[kMxRows];
#pragma unroll
    for (int rr = 0; rr < kMxRows; ++rr)
      raw[rr] = (col_ok && r0 + rr < M) ? __ldg(src + rr * stride) : make_uint4(0, 0, 0, 0);
    uint32_t* dst = reinterpret_cast<uint32_t*>(codes + int64_t(r0) * (K >> 1)) + c8;
    const int kb = c8 >> 2;
    // SF byte offset of (row r0 + rr, block kb): rows r0..r0+3 share row>>5 and row>>7
    const size_t sf0 = (size_t(r0 >> 7) * kc_pad + size_t(kb >> 2)) * 512 + size_t((r0 >> 5) & 3) * 4 + size_t(kb & 3);
#pragma unroll
    for (int rr = 0; rr < kMxRows; ++rr) {
      const uint32_t w[4] = {raw[rr].x, raw[rr].y, raw[rr].z, raw[rr].w};
      uint32_t m2 = __vmaxu2(__vmaxu2(w[0] & 0x7FFF7FFFu, w[1] & 0x7FFF7FFFu),
                             __vmaxu2(w[2] & 0x7FFF7FFFu, w[3] & 0x7FFF7FFFu));
      uint32_t m = max(m2 & 0xFFFFu, m2 >> 16);
      m = max(m, __shfl_xor_sync(0xffffffff, m, 1));
      m = max(m, __shfl_xor_sync(0xffffffff, m, 2));
      const int e = mx_block_exp_bf16bits(m);
      const float inv = __uint_as_float(uint32_t(127 - e) << 23);  // 2^-e, exact
      uint32_t packed = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        packed |= cvt_e2m1x2_raw(__uint_as_float(w[i] << 16) * inv, __uint_as_float(w[i] & 0xFFFF0000u) * inv)
                  << (8 * i);
      const int row = r0 + rr;
      if (col_ok && row < M) dst[int64_t(rr) * (K >> 3)] = canon_neg_zero(packed);
      if (sf_col_ok && row < m_sf && (threadIdx.x & 3) == 0) sf[sf0 + size_t(((r0 + rr) & 31)) * 16] = uint8_t(e + 127);
    }
  } else {
    float v[kMxRows][8];
#pragma unroll
    for (int rr = 0; rr < kMxRows; ++rr) {
      const int row = r0 + rr;
      if (col_ok && row < M) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(x + int64_t(row) * ldx) + 2 * c8);
        const float4 b = __ldg(reinterpret_cast<const float4*>(x + int64_t(row) * ldx) + 2 * c8 + 1);
        v[rr][0] = a.x; v[rr][1] = a.y; v[rr][2] = a.z; v[rr][3] = a.w;
        v[rr][4] = b.x; v[rr][5] = b.y; v[rr][6] = b.z; v[rr][7] = b.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[rr][i] = 0.f;
      }
    }
#pragma unroll
    for (int rr = 0; rr < kMxRows; ++rr) {
      const int row = r0 + rr;
      float amax = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(v[rr][i]));
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 1));
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 2));
      const int e = mx_block_exp_f32(amax);
      const float inv = __uint_as_float(uint32_t(127 - e) << 23);
      uint32_t packed = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) packed |= cvt_e2m1x2_raw(v[rr][2 * i] * inv, v[rr][2 * i + 1] * inv) << (8 * i);
      if (col_ok && row < M) reinterpret_cast<uint32_t*>(codes + int64_t(row) * (K >> 1))[c8] = canon_neg_zero(packed);
      if (sf_col_ok && row < m_sf && (threadIdx.x & 3) == 0) sf[sf_offset(row, c8 >> 2, kc_pad)] = uint8_t(e + 127);
    }
  }
}

// ------------------------------------------------------------------ RMSNorm -> MX (producer fusion)
// One CTA per token row: y = x / sqrt(mean(x^2) + eps) * gain (saliency.py:194-196,
// the gain carrying the folded SAF scales, toymodel.py:203-217), then mx_encode(y)
// -- the normalised activation never goes to HBM.  Arithmetic follows the
// reference (square, mean = sum / K, + eps, sqrt, divide, multiply): the mean of
// squares at f64-level accuracy (compensated f32), the normalised value in f32
// with a proven error bound, and -- for any 32-block the bound cannot decide (an
// element within 4e-7 of an E2M1 decision point, or the block max that close to
// a power of two) -- the reference's f64 operations with IEEE division.  Several
// rows per CTA, each row's elements in its threads' registers (read once).
// E2M1 code (sign | magnitude index) of an exactly power-of-two-scaled f64 value, through
// the hardware f32 converter: sc and f32(sc) round alike unless f32(sc) lands exactly ON a
// decision point (all of which are f32 values) while sc is not -- then sc's side decides.
__device__ __forceinline__ uint32_t e2m1_code_f64(double sc) {
  const double a = fabs(sc);
  float t = float(a);  // RN
  const bool mid = t == 0.25f || t == 0.75f || t == 1.25f || t == 1.75f || t == 2.5f || t == 3.5f || t == 5.0f;
  if (mid && double(t) != a) t = double(t) < a ? __int_as_float(__float_as_int(t) + 1) : __int_as_float(__float_as_int(t) - 1);
  const uint32_t idx = cvt_e2m1x2_raw(t, 0.f) & 7u;  // even element -> low nibble
  return (sc < 0.0 && idx > 0) ? idx + 8 : idx;
}

template <typename T>
struct Raw8;
template <>
struct Raw8<__nv_bfloat16> {
  uint32_t w[4];
  __device__ __forceinline__ void load(const __nv_bfloat16* p, bool ok) {
    const uint4 r = ok ? __ldg(reinterpret_cast<const uint4*>(p)) : make_uint4(0, 0, 0, 0);
    w[0] = r.x; w[1] = r.y; w[2] = r.z; w[3] = r.w;
  }
  __device__ __forceinline__ float f(int i) const {
    return __uint_as_float((i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16));
  }
  __device__ __forceinline__ void store(__nv_bfloat16* p) const {
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ void load_shared(const __nv_bfloat16* p) {
    const uint4 r = *reinterpret_cast<const uint4*>(p);
    w[0] = r.x; w[1] = r.y; w[2] = r.z; w[3] = r.w;
  }
};
template <>
struct Raw8<float> {
  float v[8];
  __device__ __forceinline__ void load(const float* p, bool ok) {
    const float4 a = ok ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0, 0, 0, 0);
    const float4 b = ok ? __ldg(reinterpret_cast<const float4*>(p) + 1) : make_float4(0, 0, 0, 0);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ __forceinline__ float f(int i) const { return v[i]; }
  __device__ __forceinline__ void store(float* p) const {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
  __device__ __forceinline__ void load_shared(const float* p) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};

template <typename T, int kTpr, int kChunks>
__global__ void __launch_bounds__(256) rmsnorm_mx_encode_kernel(const T* __restrict__ x, int M, int K, int64_t ldx,
                                                                const double* __restrict__ gain,
                                                                const float* __restrict__ gain32, double eps,
                                                                uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
                                                                int kc_pad, MxGather gather = MxGather{}) {
  constexpr int kRows = 256 / kTpr, kWarps = kTpr / 32;
  // Error budget of the f32 fast path vs the reference's f64 y: per-thread recursive f32
  // sum of n = 8 kChunks positive squares (<= (n - 1) 2^-24 relative), halved by the sqrt,
  // plus five f32 roundings (1/rms, x r, * g, gain, r32).
  constexpr float kRel = float((8 * kChunks - 1) * 0.5 + 6.0) * 5.9604645e-8f;
  constexpr uint32_t kMantEdge = uint32_t(kRel * 8388608.0f) + 2u;  // power-of-two proximity, in f32 ulps
  __shared__ double red[kRows][kWarps];
  __shared__ double s_rms[kRows];
  __shared__ float s_r32[kRows];
  __shared__ int s_unsure[kRows];
  pdl_launch_dependents();
  pdl_wait();
  const int rl = threadIdx.x / kTpr, t = threadIdx.x % kTpr;
  const int64_t row = int64_t(blockIdx.x) * kRows + rl;
  const bool row_ok = row < M;
  const T* xr = x + (row_ok ? row : 0) * ldx;
  Raw8<T> v[kChunks];
#pragma unroll
  for (int it = 0; it < kChunks; ++it) {
    const int c = it * (kTpr * 8) + t * 8;
    v[it].load(xr + c, row_ok && c < K);
  }
  // ---- pass 1: mean of squares in f32 per thread, combined in f64
  float ss32 = 0.f;
#pragma unroll
  for (int it = 0; it < kChunks; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) ss32 = fmaf(v[it].f(i), v[it].f(i), ss32);
  double ss = ss32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((t & 31) == 0) red[rl][t >> 5] = ss;
  if (t == 0) s_unsure[rl] = 0;
  __syncthreads();
  if (t == 0) {
    double total = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) total += red[rl][w];
    s_r32[rl] = float(1.0 / sqrt(total / double(K) + eps));
  }
  __syncthreads();
  const float r32 = s_r32[rl];
  // ---- pass 2: f32 encode; blocks the error budget cannot decide are left for pass 3
  uint32_t unsure_mask = 0;  // bit it: chunk `it`'s 32-block is undecided
#pragma unroll
  for (int it = 0; it < kChunks; ++it) {
    const int c = it * (kTpr * 8) + t * 8;
    const bool ok = row_ok && c < K;
    float y[8];
    float amax = 0.f;
    float4 g0 = make_float4(0, 0, 0, 0), g1 = make_float4(0, 0, 0, 0);
    if (ok) {
      g0 = __ldg(reinterpret_cast<const float4*>(gain32 + c));
      g1 = __ldg(reinterpret_cast<const float4*>(gain32 + c) + 1);
    }
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      y[i] = v[it].f(i) * r32 * g[i];
      amax = fmaxf(amax, fabsf(y[i]));
    }
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 2));
    const uint32_t mant = __float_as_uint(amax) & 0x7FFFFFu;
    bool unsure = amax != 0.f &&
                  (mant < kMantEdge || mant > 0x7FFFFFu - kMantEdge || amax < 0x1p-100f || !(amax < 0x1p+100f));
    const int e = mx_block_exp_f32(amax);
    const float inv = __uint_as_float(uint32_t(127 - e) << 23);
    // E2M1 rounding is monotone: if both ends of [s (1 - kRel), s (1 + kRel)] round to the
    // same code, every value in it (the reference's included) does
    const float inv_lo = inv * (1.f - kRel), inv_hi = inv * (1.f + kRel);
    uint32_t packed = 0, packed_hi = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      packed |= cvt_e2m1x2_raw(y[2 * i] * inv_lo, y[2 * i + 1] * inv_lo) << (8 * i);
      packed_hi |= cvt_e2m1x2_raw(y[2 * i] * inv_hi, y[2 * i + 1] * inv_hi) << (8 * i);
    }
    unsure |= packed != packed_hi;
    unsure = __shfl_xor_sync(0xffffffff, int(unsure), 1) | unsure;
    unsure = __shfl_xor_sync(0xffffffff, int(unsure), 2) | unsure;
    if (unsure) {
      unsure_mask |= 1u << it;
    } else if (ok) {
      *reinterpret_cast<uint32_t*>(codes + row * (K / 2) + c / 2) = canon_neg_zero(packed);
      if ((t & 3) == 0) sf[sf_offset(row, c / 32, kc_pad)] = uint8_t(e + 127);
    }
  }
  // ---- the salient slice x[:, idx] of a non-permuted layer (compensate.py:335), normalised
  // with the same row scale: thread t encodes gathered elements 8t .. 8t+7 (r <= 8 kTpr)
  bool unsure_g = false;
  const int gj0 = t * 8;
  if (gather.idx) {
    const bool okg = row_ok && gj0 < gather.r;
    float y[8];
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int col = okg ? gather.idx[gj0 + i] : 0;
      y[i] = okg ? In<T>::f(xr[col]) * r32 * gain32[col] : 0.f;
      amax = fmaxf(amax, fabsf(y[i]));
    }
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 2));
    const uint32_t mant = __float_as_uint(amax) & 0x7FFFFFu;
    bool unsure = amax != 0.f &&
                  (mant < kMantEdge || mant > 0x7FFFFFu - kMantEdge || amax < 0x1p-100f || !(amax < 0x1p+100f));
    const int e = mx_block_exp_f32(amax);
    const float inv = __uint_as_float(uint32_t(127 - e) << 23);
    const float inv_lo = inv * (1.f - kRel), inv_hi = inv * (1.f + kRel);
    uint32_t packed = 0, packed_hi = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      packed |= cvt_e2m1x2_raw(y[2 * i] * inv_lo, y[2 * i + 1] * inv_lo) << (8 * i);
      packed_hi |= cvt_e2m1x2_raw(y[2 * i] * inv_hi, y[2 * i + 1] * inv_hi) << (8 * i);
    }
    unsure |= packed != packed_hi;
    unsure = __shfl_xor_sync(0xffffffff, int(unsure), 1) | unsure;
    unsure = __shfl_xor_sync(0xffffffff, int(unsure), 2) | unsure;
    if (unsure) {
      unsure_g = okg;
    } else if (okg) {
      *reinterpret_cast<uint32_t*>(gather.xs_codes + row * (gather.r / 2) + gj0 / 2) = canon_neg_zero(packed);
      if ((t & 3) == 0) gather.xs_sf[sf_offset(row, gj0 / 32, gather.kc_pad_r)] = uint8_t(e + 127);
    }
  }
  // ---- pass 3 (rare): rows holding an undecided block redo them with the reference's f64
  // operations: the mean of squares at f64 accuracy, IEEE division, exact E2M1 rounding
  if (unsure_mask || unsure_g) s_unsure[rl] = 1;
  if (!__syncthreads_or(unsure_mask != 0 || unsure_g)) return;
  const bool redo = s_unsure[rl] != 0;
  double ss64 = 0.0;
  if (redo) {
#pragma unroll
    for (int it = 0; it < kChunks; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double d = v[it].f(i);
        ss64 = fma(d, d, ss64);
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss64 += __shfl_xor_sync(0xffffffff, ss64, o);
  __syncthreads();  // red[] reuse
  if ((t & 31) == 0) red[rl][t >> 5] = ss64;
  __syncthreads();
  if (t == 0 && redo) {
    double total = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) total += red[rl][w];
    s_rms[rl] = sqrt(total / double(K) + eps);
  }
  __syncthreads();
  if (!redo) return;
  const double rms = s_rms[rl];
#pragma unroll
  for (int it = 0; it < kChunks; ++it) {
    if (!__any_sync(0xffffffff, (unsure_mask >> it) & 1u)) continue;
    const int c = it * (kTpr * 8) + t * 8;
    const bool ok = row_ok && c < K;
    double yd[8];
    double amaxd = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      yd[i] = ok ? __ddiv_rn(double(v[it].f(i)), rms) * gain[c + i] : 0.0;
      amaxd = fmax(amaxd, fabs(yd[i]));
    }
    amaxd = fmax(amaxd, __shfl_xor_sync(0xffffffff, amaxd, 1));
    amaxd = fmax(amaxd, __shfl_xor_sync(0xffffffff, amaxd, 2));
    const int e = mx_block_exp_f64(amaxd);
    const double invd = ldexp(1.0, -e);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) packed |= e2m1_code_f64(yd[i] * invd) << (4 * i);
    if (ok && ((unsure_mask >> it) & 1u)) {
      *reinterpret_cast<uint32_t*>(codes + row * (K / 2) + c / 2) = packed;
      if ((t & 3) == 0) sf[sf_offset(row, c / 32, kc_pad)] = uint8_t(e + 127);
    }
  }
  if (gather.idx && __any_sync(0xffffffff, unsure_g)) {
    const bool okg = row_ok && gj0 < gather.r;
    double yd[8];
    double amaxd = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int col = okg ? gather.idx[gj0 + i] : 0;
      yd[i] = okg ? __ddiv_rn(double(In<T>::f(xr[col])), rms) * gain[col] : 0.0;
      amaxd = fmax(amaxd, fabs(yd[i]));
    }
    amaxd = fmax(amaxd, __shfl_xor_sync(0xffffffff, amaxd, 1));
    amaxd = fmax(amaxd, __shfl_xor_sync(0xffffffff, amaxd, 2));
    const int e = mx_block_exp_f64(amaxd);
    const double invd = ldexp(1.0, -e);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) packed |= e2m1_code_f64(yd[i] * invd) << (4 * i);
    if (unsure_g) {
      *reinterpret_cast<uint32_t*>(gather.xs_codes + row * (gather.r / 2) + gj0 / 2) = packed;
      if ((t & 3) == 0) gather.xs_sf[sf_offset(row, gj0 / 32, gather.kc_pad_r)] = uint8_t(e + 127);
    }
  }
}

// ------------------------------------------------------------------ MX container
// The reference's packed MX file body (mxfmt.py:228-251): per 32-block one
// biased exponent byte (e + 127) then 16 bytes of nibbles, element 2i in the
// low nibble -- 17-byte records, row-major over (row, block).  One thread per
// record: the element codes [rows, cols] and exponents [rows, cols / 32] that
// serq_pack_mx consumes.
__global__ void mx_container_decode_kernel(const uint8_t* __restrict__ body, int64_t records,
                                           uint8_t* __restrict__ codes, int32_t* __restrict__ exps) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= records) return;
  const uint8_t* rec = body + i * 17;
  exps[i] = int32_t(rec[0]) - 127;
  uint32_t out[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t b0 = rec[1 + 2 * w], b1 = rec[2 + 2 * w];
    out[w] = (b0 & 0xFu) | ((b0 >> 4) << 8) | ((b1 & 0xFu) << 16) | ((b1 >> 4) << 24);
  }
  uint4* dst = reinterpret_cast<uint4*>(codes + i * 32);  // block i covers codes [32 i, 32 i + 32)
  dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
  dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
}

// ------------------------------------------------------------------ INT quantize
// One CTA per token row.  Scales / zero points in f64 exactly as the reference;
// codes rint(x / s) bit-exact: a fast product against 1/s decides the rounding
// unless the quotient is within a provable error bound of a half-integer, in
// which case the correctly rounded f64 division decides.
template <typename T>
__device__ __forceinline__ double load_as_f64(const T* p) {
  if constexpr (In<T>::kId == 2) return *p;
  else return double(In<T>::f(*p));
}

template <typename T>
__device__ __forceinline__ double rint_quot(T xv, double s, float inv32, double inv64) {
  if constexpr (In<T>::kId == 2) {
    const double q = xv * inv64;  // |q - x/s| <= |q| * 2^-51
    const double fl = floor(q);
    const double fr = q - fl;
    const double margin = fabs(q) * 0x1p-49 + 0x1p-60;
    if (fabs(fr - 0.5) > margin) return fr > 0.5 ? fl + 1.0 : fl;
    return rint(xv / s);
  } else {
    const float xf = In<T>::f(xv);
    const float q = xf * inv32;  // |q - x/s| <= |q| * 2^-22.9
    if (fabsf(q) < 0x1p21f) {
      const float fl = floorf(q);
      const float fr = q - fl;  // exact
      const float margin = fabsf(q) * 0x1p-21f + 0x1p-40f;
      if (fabsf(fr - 0.5f) > margin) return double(fr > 0.5f ? fl + 1.f : fl);
    }
    return rint(double(xf) / s);
  }
}

// ---------------------------------------------------------------- RMSNorm -> INT producer
// The reference's row mean of squares is NumPy's pairwise float64 sum (np.mean over the last,
// contiguous axis: pairwise_sum with 128-element leaves, eight strided accumulators per leaf
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), the leaf tail added in order, leaves combined
// along the recursion that halves n at a multiple of 8).  The host replays that recursion for K
// once and passes the leaves and the internal nodes ordered by height, so every row's sum has
// the reference's exact rounding sequence and a warp can evaluate one height level at a time.
struct RmsPairwise {
  int nleaf, nnode, nlevel, perfect;  // perfect: 2^d leaves, all at depth d
  int16_t start[64], len[64];
  uint8_t a[64], b[64];  // node j (value slot nleaf + j) = val[a[j]] + val[b[j]]
  uint8_t level_end[8];  // nodes of height h + 1: [level_end[h - 1], level_end[h])
};

// Evaluate the internal nodes over val[0 .. nleaf) (the leaf sums); one full warp.
__device__ __forceinline__ double rms_tree_eval(const RmsPairwise& tr, double* val, int lane) {
  int j0 = 0;
  for (int h = 0; h < tr.nlevel; ++h) {
    const int j1 = tr.level_end[h];
    for (int j = j0 + lane; j < j1; j += 32) val[tr.nleaf + j] = val[tr.a[j]] + val[tr.b[j]];
    __syncwarp();
    j0 = j1;
  }
  return val[tr.nnode ? tr.nleaf + tr.nnode - 1 : 0];
}

// y = x / sqrt(mean(x^2) + eps) * gain in float64 exactly as saliency.py:194-196, then the
// per-token quantizer on y exactly as quantize_asymmetric / quantize_symmetric
// (quantcore.py:108-137): codes, f64 scales and zero points bit-identical to the reference's.
// One 256-thread CTA per row, every operation in f64 -- the kernel for layouts the fast one
// below does not serve (K % 8 != 0, unaligned rows) and its cross-check.
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_int_quant_kernel(const T* __restrict__ x, int64_t M, int64_t K,
                                                                int64_t ldx, const double* __restrict__ gain,
                                                                double eps, const RmsPairwise tree, int bits,
                                                                int symmetric, int8_t* __restrict__ codes,
                                                                double* __restrict__ scale64,
                                                                float* __restrict__ scale32, int32_t* __restrict__ zp_out,
                                                                const int32_t* __restrict__ sidx, int r,
                                                                void* __restrict__ xs_out, int xs_kind) {
  const int64_t row = blockIdx.x;
  const T* xr = x + row * ldx;
  __shared__ double val[128];
  __shared__ double red_lo[8], red_hi[8];
  __shared__ double s_rms, s_scale;
  __shared__ int s_zp;
  pdl_launch_dependents();
  pdl_wait();
  // pass 1: the leaves, an 8-thread group per leaf (thread j: accumulator r_j)
  const int grp = int(threadIdx.x) >> 3, j = int(threadIdx.x) & 7;
  for (int lf = grp; lf < tree.nleaf; lf += int(blockDim.x) >> 3) {
    const int st = tree.start[lf], n = tree.len[lf];
    double acc = 0.0;
    if (n >= 8) {
      const int body = n - (n % 8);
      for (int i = j; i < body; i += 8) {
        const double v = load_as_f64(xr + st + i);
        acc = fma(v, v, acc);  // x*x is exact in f64 for bf16 / f32 x: rounds as acc + x*x
      }
      const unsigned gmask = 0xFFu << (threadIdx.x & 24);  // this leaf's 8 lanes only
      acc += __shfl_xor_sync(gmask, acc, 1);  // (r0 + r1), (r2 + r3), ...
      acc += __shfl_xor_sync(gmask, acc, 2);
      acc += __shfl_xor_sync(gmask, acc, 4);
      if (j == 0)
        for (int i = body; i < n; ++i) {
          const double v = load_as_f64(xr + st + i);
          acc = fma(v, v, acc);
        }
    } else if (j == 0) {
      for (int i = 0; i < n; ++i) {
        const double v = load_as_f64(xr + st + i);
        acc = fma(v, v, acc);
      }
    }
    if (j == 0) val[lf] = acc;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const double sum = rms_tree_eval(tree, val, threadIdx.x);
    if (threadIdx.x == 0) s_rms = sqrt(sum / double(K) + eps);
  }
  __syncthreads();
  const double rms = s_rms;
  // pass 2: y = x / rms * gain (f64, two roundings as the reference), row min / max
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const double y = load_as_f64(xr + k) / rms * gain[k];
    lo = fmin(lo, y);
    hi = fmax(hi, y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffff, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffff, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red_lo[threadIdx.x >> 5] = lo;
    red_hi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
      lo = fmin(lo, red_lo[w]);
      hi = fmax(hi, red_hi[w]);
    }
    double sc;
    int zp = 0;
    if (symmetric) {
      sc = fmax(fabs(lo), fabs(hi)) / double((1 << (bits - 1)) - 1);
      if (sc == 0.0) sc = 1.0;
    } else {
      sc = (hi - lo) / double((1 << bits) - 1);
      if (sc == 0.0) sc = 1.0;
      zp = int(rint(-lo / sc));
    }
    s_scale = sc;
    s_zp = zp;
    scale64[row] = sc;
    scale32[row] = float(sc);
    if (zp_out) zp_out[row] = zp;
  }
  __syncthreads();
  const double sc = s_scale;
  const int zp = s_zp;
  const int qmax = symmetric ? (1 << (bits - 1)) - 1 : (1 << bits) - 1;
  const int qmin = symmetric ? -qmax : 0;
  // pass 3: codes of y (recomputed: the same f64 operations give the same value)
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const double y = load_as_f64(xr + k) / rms * gain[k];
    double q = rint(y / sc) + double(zp);
    q = fmin(fmax(q, double(qmin)), double(qmax));
    codes[row * K + k] = int8_t(int(q));
  }
  if (xs_kind != 0) {
    __syncthreads();
    for (int jj = threadIdx.x; jj < r; jj += blockDim.x) {
      const int col = sidx ? sidx[jj] : jj;
      const int c = symmetric ? int(codes[row * K + col]) : int(uint8_t(codes[row * K + col]));
      if (xs_kind == 1)
        reinterpret_cast<__nv_bfloat16*>(xs_out)[row * r + jj] = __int2bfloat16_rn(c - zp);
      else
        reinterpret_cast<int8_t*>(xs_out)[row * r + jj] = int8_t(c);
    }
  }
}

// The same producer at HBM speed for 16-B aligned rows with K % 8 == 0 (every pairwise leaf is
// then a whole number of 8-element vectors).  kRows = 256 / kTpr rows per CTA, each row's
// elements in its threads' registers (read once) and staged in shared memory for the leaf sums:
// one thread per leaf holds the eight accumulators r_0..r_7 of pairwise_sum and walks the leaf
// in 16-B vectors (the staging pads 8 elements per 128 so the leaves a warp reads sit in
// different banks).  Only the row sum is float64 per element.  Everything else runs on
// z = x * g32 in f32 -- y = z / rms up to rounding, so the extremes of y are those of z and no
// pass waits for the row sum -- with a proven error bound, and the reference's f64 operations
// are evaluated only where the bound cannot decide:
//  * the row's min / max (max |y|): z32 is within 2 * 2^-24 relative (g, x * g roundings) plus
//    2^-149 absolute of x * g, so the reference's extreme element is among those within 2^-20
//    relative + 2^-100 of the f32 extreme; those few (listed in shared memory) take the
//    reference's (x / rms) * g and the f64 extreme of them is the reference's;
//  * codes: t = z32 * f32(1 / (rms s)) is within 4 * 2^-24 relative + 2^-69 absolute of the
//    reference's y / s; rint(t) (round-half-even by the 1.5 * 2^23 add, the zero point folded
//    in) is decided in f32 unless t lies within |t| 2^-20 + 2^-25 of a .5 tie, where the element
//    takes rint((x / rms) * g / s) in f64;
//  * rows outside those premises (|x| > 2^20, |z| > 2^100, more than kMaxCand candidates,
//    1 / (rms s) outside [2^-120, 2^80]) run every element in the f64 reference operations.
template <typename T, int kTpr, int kChunks>
__global__ void __launch_bounds__(256) rmsnorm_int_quant_fast_kernel(
    const T* __restrict__ x, int M, int K, int64_t ldx, const double* __restrict__ gain,
    const float* __restrict__ gain32, double eps, const RmsPairwise tree, int bits, int symmetric,
    int8_t* __restrict__ codes, double* __restrict__ scale64, float* __restrict__ scale32, int32_t* __restrict__ zp_out,
    const int32_t* __restrict__ sidx, int r, void* __restrict__ xs_out, int xs_kind) {
  constexpr int kRows = 256 / kTpr, kWarps = kTpr / 32, kRowElems = kTpr * kChunks * 8;
  constexpr int kRowSmem = kRowElems + kRowElems / 16;  // + 8 elements per 128
  constexpr int kMaxCand = 64;
  static_assert(kChunks * 8 <= 32, "one mask bit per element");
  __shared__ alignas(16) T srow[kRows][kRowSmem];
  __shared__ double val[kRows][128];
  __shared__ float red_f[kRows][kWarps][3];
  __shared__ double red_d[kRows][kWarps][2];
  __shared__ int16_t cand_idx[kRows][kMaxCand];
  __shared__ int n_cand[kRows];
  __shared__ double s_rms[kRows], s_scale[kRows];
  __shared__ float s_c32[kRows];
  __shared__ int s_zp[kRows];
  pdl_launch_dependents();
  pdl_wait();
  const int rl = threadIdx.x / kTpr, t = threadIdx.x % kTpr, wr = t >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * kRows + rl;
  const bool row_ok = row < M;
  const T* xr = x + (row_ok ? row : 0) * ldx;
  T* sr = srow[rl];
  auto spos = [](int c) { return c + ((c >> 7) << 3); };
  auto elem = [&](int k) { return (k >> 3) * (kTpr * 8) + t * 8 + (k & 7); };  // mask bit -> column
  Raw8<T> v[kChunks];
#pragma unroll
  for (int it = 0; it < kChunks; ++it) {
    const int c = it * (kTpr * 8) + t * 8;
    v[it].load(xr + c, row_ok && c < K);
    v[it].store(sr + spos(c));
  }
  if (t == 0) n_cand[rl] = 0;
  // ---- z = x * g32 and the row's f32 extremes (independent of the row sum)
  float z[kChunks][8];
  float hi = -INFINITY, lo = INFINITY, xmax = 0.f;
#pragma unroll
  for (int it = 0; it < kChunks; ++it) {
    const int c = it * (kTpr * 8) + t * 8;
    // elements outside the matrix read x = 0, g = NaN: z = NaN, which fmaxf / fminf ignore
    float4 g0 = make_float4(NAN, NAN, NAN, NAN), g1 = g0;
    if (row_ok && c < K) {
      g0 = __ldg(reinterpret_cast<const float4*>(gain32 + c));
      g1 = __ldg(reinterpret_cast<const float4*>(gain32 + c) + 1);
    }
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float xf = v[it].f(i);
      z[it][i] = xf * g[i];
      hi = fmaxf(hi, z[it][i]);
      lo = fminf(lo, z[it][i]);
      xmax = fmaxf(xmax, fabsf(xf));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffff, hi, o));
    lo = fminf(lo, __shfl_xor_sync(0xffffffff, lo, o));
    xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffff, xmax, o));
  }
  if (lane == 0) {
    red_f[rl][wr][0] = hi;
    red_f[rl][wr][1] = lo;
    red_f[rl][wr][2] = xmax;
  }
  __syncthreads();
  // ---- the reference's pairwise float64 sum of squares: four threads per leaf, thread q
  // holding accumulators r_2q, r_2q+1 (spreads the f32 -> f64 conversions over every warp)
  if (t < 4 * tree.nleaf) {
    const int lf = t >> 2, q = t & 3;
    const int st = tree.start[lf], n = tree.len[lf];
    double a0 = 0.0, a1 = 0.0;
    auto step = [&](const T* p) {
      double d0, d1;
      if constexpr (In<T>::kId == 0) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
        d0 = __uint_as_float(w << 16);
        d1 = __uint_as_float(w & 0xFFFF0000u);
      } else {
        const float2 f = *reinterpret_cast<const float2*>(p);
        d0 = f.x;
        d1 = f.y;
      }
      a0 = fma(d0, d0, a0);  // x*x exact in f64: rounds as acc + x*x
      a1 = fma(d1, d1, a1);
    };
    // a leaf (<= 128 elements, starting at a multiple of 8) crosses at most one padded boundary
    const int first = min(n, 128 - (st & 127));
    const T* p = sr + spos(st) + 2 * q;
    int i = 0;
    for (; i < first; i += 8, p += 8) step(p);
    p += 8;
    for (; i < n; i += 8, p += 8) step(p);
    double pr = a0 + a1;  // (r0 + r1), (r2 + r3), ...
    const unsigned gmask = 0xFu << (lane & 28);
    pr += __shfl_xor_sync(gmask, pr, 1);  // ((r0 + r1) + (r2 + r3)), ((r4 + r5) + (r6 + r7))
    pr += __shfl_xor_sync(gmask, pr, 2);
    if (q == 0) val[rl][lf] = pr;
  }
  // ---- candidates for the extremes (while the leaf threads sum)
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    hi = fmaxf(hi, red_f[rl][w][0]);
    lo = fminf(lo, red_f[rl][w][1]);
    xmax = fmaxf(xmax, red_f[rl][w][2]);
  }
  bool slow = !(xmax <= 0x1p20f) || !(fmaxf(fabsf(hi), fabsf(lo)) <= 0x1p100f);  // also NaN
  if (!slow && row_ok) {
    const float amax32 = fmaxf(fabsf(hi), fabsf(lo));
    const float cut_hi = symmetric ? amax32 - (amax32 * 0x1p-20f + 0x1p-100f) : hi - (fabsf(hi) * 0x1p-20f + 0x1p-100f);
    const float cut_lo = lo + (fabsf(lo) * 0x1p-20f + 0x1p-100f);
#pragma unroll
    for (int it = 0; it < kChunks; ++it) {
      if (it * (kTpr * 8) + t * 8 >= K) break;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float zv = z[it][i];
        if (symmetric ? fabsf(zv) >= cut_hi : (zv >= cut_hi || zv <= cut_lo)) {
          const int j = atomicAdd(&n_cand[rl], 1);
          if (j < kMaxCand) cand_idx[rl][j] = int16_t(it * (kTpr * 8) + t * 8 + i);
        }
      }
    }
  }
  __syncthreads();
  if (wr == 0) {
    double sum;
    if (tree.perfect) {  // a perfect binary tree over 2^d leaves: the warp butterfly pairs alike
      sum = lane < tree.nleaf ? val[rl][lane] : 0.0;
      for (int o = 1; o < min(tree.nleaf, 32); o <<= 1) sum += __shfl_xor_sync(0xffffffff, sum, o);
      if (tree.nleaf == 64) {  // root = (leaves 0..31) + (leaves 32..63)
        double u = val[rl][32 + lane];
        for (int o = 1; o < 32; o <<= 1) u += __shfl_xor_sync(0xffffffff, u, o);
        sum += u;
      }
    } else {
      sum = rms_tree_eval(tree, val[rl], lane);
    }
    if (lane == 0) s_rms[rl] = sqrt(sum / double(K) + eps);
  }
  slow = __syncthreads_or(slow || n_cand[rl] > kMaxCand);  // CTA-uniform from here on
  const double rms = s_rms[rl];
  double hi64 = -INFINITY, lo64 = INFINITY;
  if (!slow && wr != 0) goto codes_pass;  // the few candidates: one warp per row
  if (!slow) {
    for (int j = lane; j < n_cand[rl]; j += 32) {
        const int c = cand_idx[rl][j];
        const float xf = In<T>::f(sr[spos(c)]);
        const double y64 = xf == 0.f ? 0.0 : double(xf) / rms * gain[c];
        hi64 = fmax(hi64, symmetric ? fabs(y64) : y64);
        lo64 = fmin(lo64, y64);
    }
  } else {
    // every element (rare rows): the reference's y for the whole row
#pragma unroll
    for (int it = 0; it < kChunks; ++it) {
      const int c = it * (kTpr * 8) + t * 8;
      if (!row_ok || c >= K) break;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xf = In<T>::f(sr[spos(c + i)]);
        const double y64 = xf == 0.f ? 0.0 : double(xf) / rms * gain[c + i];
        hi64 = fmax(hi64, symmetric ? fabs(y64) : y64);
        lo64 = fmin(lo64, y64);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hi64 = fmax(hi64, __shfl_xor_sync(0xffffffff, hi64, o));
    lo64 = fmin(lo64, __shfl_xor_sync(0xffffffff, lo64, o));
  }
  if (slow) {
    if (lane == 0) {
      red_d[rl][wr][0] = hi64;
      red_d[rl][wr][1] = lo64;
    }
    __syncthreads();  // CTA-uniform branch
    if (t == 0)
      for (int w = 1; w < kWarps; ++w) {
        hi64 = fmax(hi64, red_d[rl][w][0]);
        lo64 = fmin(lo64, red_d[rl][w][1]);
      }
  }
  if (t == 0 && row_ok) {
    double sc = symmetric ? hi64 / double((1 << (bits - 1)) - 1) : (hi64 - lo64) / double((1 << bits) - 1);
    if (sc == 0.0) sc = 1.0;
    const int zp = symmetric ? 0 : int(rint(-lo64 / sc));
    const double c64 = 1.0 / (rms * sc);
    s_scale[rl] = sc;
    s_c32[rl] = (!slow && c64 >= 0x1p-120 && c64 <= 0x1p80) ? float(c64) : NAN;
    s_zp[rl] = zp;
    scale64[row] = sc;
    scale32[row] = float(sc);
    if (zp_out) zp_out[row] = zp;
  }
codes_pass:
  __syncthreads();
  // ---- codes
  const int zp = s_zp[rl];
  if (row_ok) {
    const double sc = s_scale[rl];
    const float c32 = s_c32[rl];
    const int qmax = symmetric ? (1 << (bits - 1)) - 1 : (1 << bits) - 1;
    const int qmin = symmetric ? -qmax : 0;
    // q + (1.5 * 2^23 + zp) rounds q + zp half-to-even (|q + zp| < 2^22); rint(q) + zp differs
    // from that only at an exact .5 tie of q with zp odd, which the margin sends to the f64 path
    const float magic = 12582912.f + float(zp);
    const uint32_t magic_bits = __float_as_uint(magic);
    uint32_t redo = c32 != c32 ? 0xFFFFFFFFu : 0u;
#pragma unroll
    for (int it = 0; it < kChunks; ++it) {
      const int c = it * (kTpr * 8) + t * 8;
      if (c >= K) break;
      int cq[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float q = z[it][i] * c32;
        const float mq = q + magic;
        const float d = q - (mq - magic);  // q - (rint(q + zp) - zp), exact
        if (fabsf(d) >= fmaf(fabsf(q), -0x1p-20f, 0.5f - 0x1p-25f)) redo |= 1u << (it * 8 + i);
        cq[i] = min(max(int(__float_as_uint(mq) - magic_bits) + zp, qmin), qmax);
      }
      const uint32_t w0 = __byte_perm(__byte_perm(cq[0], cq[1], 0x0040), __byte_perm(cq[2], cq[3], 0x0040), 0x5410);
      const uint32_t w1 = __byte_perm(__byte_perm(cq[4], cq[5], 0x0040), __byte_perm(cq[6], cq[7], 0x0040), 0x5410);
      *reinterpret_cast<uint2*>(codes + row * K + c) = make_uint2(w0, w1);
    }
    for (uint32_t m = redo; m; m &= m - 1) {
      const int c = elem(__ffs(m) - 1);
      if (c >= K) break;  // chunks are in order: the rest lies past K too
      const float xf = In<T>::f(sr[spos(c)]);
      const double y64 = xf == 0.f ? 0.0 : double(xf) / rms * gain[c];
      codes[row * K + c] = int8_t(min(max(int(rint(y64 / sc)) + zp, qmin), qmax));
    }
  }
  if (xs_kind != 0) {
    __syncthreads();
    if (row_ok) {
      for (int jj = t; jj < r; jj += kTpr) {
        const int col = sidx ? sidx[jj] : jj;
        const int c = symmetric ? int(codes[row * K + col]) : int(uint8_t(codes[row * K + col]));
        if (xs_kind == 1)
          reinterpret_cast<__nv_bfloat16*>(xs_out)[row * r + jj] = __int2bfloat16_rn(c - zp);
        else
          reinterpret_cast<int8_t*>(xs_out)[row * r + jj] = int8_t(c);
      }
    }
  }
}

// rint(x / s) as an int for 16-bit / 32-bit inputs: the f32 fast path decides with the proven
// margin and everything stays on the FP32 / integer pipes (an f64 division is a ~10-DFMA
// dependent sequence; tools/probes/fp64_rate.cu measures DFMA at 0.42x the FFMA rate); only
// values within the margin of a .5 tie take the correctly rounded f64 division.
// Returns clip(rint(x / s) + zp, qmin, qmax).  |x/s| < 2^21 implies |zp| < 2^21 + 2^bits
// (x lies in [lo, hi], zp = rint(-lo/s)), so the int sum is exact; larger quotients take
// the reference's f64 expression.
template <typename T>
__device__ __forceinline__ int int_code(T xv, double s, float inv32, int zp, int qmin, int qmax) {
  const float xf = In<T>::f(xv);
  const float q = xf * inv32;  // |q - x/s| <= |q| * 2^-22.9
  if (fabsf(q) < 0x1p21f) {
    const float fl = floorf(q);
    const float fr = q - fl;  // exact
    const float margin = fabsf(q) * 0x1p-21f + 0x1p-40f;
    const int r = fabsf(fr - 0.5f) > margin ? int(fl) + (fr > 0.5f ? 1 : 0) : int(rint(double(xf) / s));
    return min(max(r + zp, qmin), qmax);
  }
  const double qd = rint(double(xf) / s) + double(zp);
  return int(fmin(fmax(qd, double(qmin)), double(qmax)));
}

template <typename T>
__global__ void __launch_bounds__(256) int_quant_kernel(const T* __restrict__ x, int64_t M, int64_t K, int64_t ldx,
                                                        int bits, int symmetric, int8_t* __restrict__ codes,
                                                        double* __restrict__ scale64, float* __restrict__ scale32,
                                                        int32_t* __restrict__ zp_out, const int32_t* __restrict__ sidx,
                                                        int r, void* __restrict__ xs_out, int xs_kind) {
  const int64_t row = blockIdx.x;
  const T* xr = x + row * ldx;
  __shared__ double red_lo[8], red_hi[8];
  __shared__ double s_scale;
  __shared__ int s_zp;
  // pass 1: min / max (asym) or max|x| (sym)
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const double v = load_as_f64(xr + k);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffff, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffff, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red_lo[threadIdx.x >> 5] = lo;
    red_hi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, red_lo[w]);
      hi = fmax(hi, red_hi[w]);
    }
    double s;
    int zp = 0;
    if (symmetric) {
      const double amax = fmax(fabs(lo), fabs(hi));
      s = amax / double((1 << (bits - 1)) - 1);
      if (s == 0.0) s = 1.0;
    } else {
      s = (hi - lo) / double((1 << bits) - 1);
      if (s == 0.0) s = 1.0;
      zp = int(rint(-lo / s));
    }
    s_scale = s;
    s_zp = zp;
    scale64[row] = s;
    scale32[row] = float(s);
    if (zp_out) zp_out[row] = zp;
  }
  __syncthreads();
  const double s = s_scale;
  const int zp = s_zp;
  const double inv64 = 1.0 / s;
  const float inv32 = float(inv64);
  const int qmax = symmetric ? (1 << (bits - 1)) - 1 : (1 << bits) - 1;
  const int qmin = symmetric ? -qmax : 0;
  // pass 2: codes (the row was just read, so this re-read is an L2 hit)
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    double q = rint_quot<T>(xr[k], s, inv32, inv64) + double(zp);
    q = fmin(fmax(q, double(qmin)), double(qmax));
    codes[row * K + k] = int8_t(int(q));
  }
  if (xs_kind != 0) {
    __syncthreads();
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
      const int col = sidx ? sidx[j] : j;
      const int c = symmetric ? int(codes[row * K + col]) : int(uint8_t(codes[row * K + col]));
      if (xs_kind == 1) {
        reinterpret_cast<__nv_bfloat16*>(xs_out)[row * r + j] = __int2bfloat16_rn(c - zp);
      } else {
        reinterpret_cast<int8_t*>(xs_out)[row * r + j] = int8_t(c);
      }
    }
  }
}

// Fast path for bf16 rows with K % 8 == 0 and K <= 2048 * kNV: one CTA per row,
// the row stays in registers between the reduction and the quantization pass
// (one HBM read), 16-B loads and 8-B code stores.
// bf16 rows, K <= 8192: kTpr threads per token row, 256 / kTpr rows per CTA, each
// thread keeps its kCpt 16-B chunks in registers (one HBM read); row min / max by
// shuffles + a per-row shared-memory step; scale / zero point in f64 by one thread
// per row exactly as the reference (quantcore.py:108-137); codes through int_code.
// the exact path of int_code for the flagged elements (out of line: one copy of the f64
// division instead of one per unrolled element)
// clip(rint(x / s) + zp) exactly as the reference's f64 expression, for an element the
// fp32 fast path flagged.  Near a .5 tie h = k + 1/2 the answer follows from the sign of
// the exact residual r = RN(x - h*s) (one DFMA; x, h exact): r == 0 means x / s == h and
// rint picks the even neighbour; |r| > 2 * (ulp(h)/2) * s means the f64 quotient cannot
// round onto h, so the sign decides.  Only the razor-thin rest (and |x/s| >= 2^21) pays
// the correctly rounded f64 division.  One DFMA instead of a DDIV (a ~10-DFMA dependent
// sequence) keeps a flagged row off the kernel's critical path.
__device__ __forceinline__ int int_code_tie(float xf, double s, float inv32, int zp, int qmin, int qmax) {
  const float q = xf * inv32;  // only steers toward the nearby half-integer
  double k;
  const float n = rintf(q);
  if (fabsf(q) < 0x1p21f) {
    const double h = double(n) + (q - n >= 0.f ? 0.5 : -0.5);
    const double r = fma(-h, s, double(xf));
    if (r == 0.0) {
      const double lo = h - 0.5;
      k = (int(lo) & 1) == 0 ? lo : lo + 1.0;  // |lo| < 2^21
    } else {
      int eh;
      frexp(h, &eh);  // |h| in [2^(eh-1), 2^eh): ulp(h) = 2^(eh - 53)
      const double half_ulp_s = ldexp(s, eh - 54);
      k = fabs(r) > 2.0 * half_ulp_s ? (r > 0.0 ? h + 0.5 : h - 0.5) : rint(double(xf) / s);
    }
  } else {
    k = rint(double(xf) / s);
  }
  return int(fmin(fmax(k + double(zp), double(qmin)), double(qmax)));
}

template <int kTpr, int kCpt, int kBlock = 256>
__global__ void __launch_bounds__(kBlock) int_quant_bf16_kernel(const __nv_bfloat16* __restrict__ x, int M, int K,
                                                             int64_t ldx, int bits, int symmetric,
                                                             int8_t* __restrict__ codes, double* __restrict__ scale64,
                                                             float* __restrict__ scale32, int32_t* __restrict__ zp_out,
                                                             const int32_t* __restrict__ sidx, int r,
                                                             void* __restrict__ xs_out, int xs_kind,
                                                             float* __restrict__ range, int range_mode) {
  // range_mode 1: write this row's (min, max) to range[row], range[M + row] and stop (a K-shard's
  // local range); 2: quantize with the row range read from there (the all-reduced MIN / MAX over
  // the K-shards: the reference's per-token scale spans the full row, quantcore.py:127-129)
  constexpr int kRows = kBlock / kTpr, kWarps = kTpr / 32;
  __shared__ float red_lo[kRows][kWarps], red_hi[kRows][kWarps];
  __shared__ double s_scale[kRows];
  __shared__ float s_inv32[kRows];
  __shared__ int s_zp[kRows];
  pdl_launch_dependents();
  pdl_wait();
  const int rl = threadIdx.x / kTpr, t = threadIdx.x % kTpr;
  const int n8 = K >> 3;
  // persistent over row groups (grid sized to the resident CTAs): the next group's rows are
  // loaded into registers before this group's reduction -> scale -> codes chain runs
  const int64_t rstride = int64_t(gridDim.x) * kRows;
  auto load_row = [&](int64_t rw, uint4 (&dst)[kCpt]) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + (rw < M ? rw : 0) * ldx);
#pragma unroll
    for (int j = 0; j < kCpt; ++j) {
      const int c8 = t + j * kTpr;
      dst[j] = (rw < M && c8 < n8) ? __ldg(xr + c8) : make_uint4(0, 0, 0, 0);
    }
  };
  uint4 raw[kCpt];
  load_row(int64_t(blockIdx.x) * kRows + rl, raw);
  for (int64_t base = int64_t(blockIdx.x) * kRows; base < M; base += rstride) {
  const int64_t row = base + rl;
  const bool row_ok = row < M;
  uint4 nxt[kCpt];
  load_row(row + rstride, nxt);
  // min / max on packed bf16 pairs (one HMNMX2 per two elements; exact: bf16 -> f32 is exact)
  __nv_bfloat162 lo2 = __halves2bfloat162(__ushort_as_bfloat16(0x7F80), __ushort_as_bfloat16(0x7F80));
  __nv_bfloat162 hi2 = __halves2bfloat162(__ushort_as_bfloat16(0xFF80), __ushort_as_bfloat16(0xFF80));
#pragma unroll
  for (int j = 0; j < kCpt; ++j) {
    const int c8 = t + j * kTpr;
    const bool ok = row_ok && c8 < n8;
    if (ok) {
      const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
        lo2 = __hmin2(lo2, v);
        hi2 = __hmax2(hi2, v);
      }
    }
  }
  float lo = fminf(__low2float(lo2), __high2float(lo2)), hi = fmaxf(__low2float(hi2), __high2float(hi2));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffff, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffff, hi, o));
  }
  if ((t & 31) == 0) {
    red_lo[rl][t >> 5] = lo;
    red_hi[rl][t >> 5] = hi;
  }
  __syncthreads();
  if (t == 0 && row_ok) {
#pragma unroll
    for (int w = 1; w < kWarps; ++w) {
      lo = fminf(lo, red_lo[rl][w]);
      hi = fmaxf(hi, red_hi[rl][w]);
    }
    if (range_mode == 2) {
      lo = range[row];
      hi = range[M + row];
    }
    const double dlo = lo, dhi = hi;  // exact (bf16 values)
    double sc;
    int zp = 0;
    if (symmetric) {
      sc = fmax(fabs(dlo), fabs(dhi)) / double((1 << (bits - 1)) - 1);
      if (sc == 0.0) sc = 1.0;
    } else {
      sc = (dhi - dlo) / double((1 << bits) - 1);
      if (sc == 0.0) sc = 1.0;
      zp = int(rint(-dlo / sc));
    }
    s_scale[rl] = sc;
    s_inv32[rl] = float(1.0 / sc);
    s_zp[rl] = zp;
    if (range_mode == 1) {
      range[row] = lo;
      range[M + row] = hi;
    } else {
      scale64[row] = sc;
      scale32[row] = float(sc);
      if (zp_out) zp_out[row] = zp;
    }
  }
  __syncthreads();
  if (row_ok && range_mode != 1) {
  const double sc = s_scale[rl];
  const int zp = s_zp[rl];
  const float inv32 = s_inv32[rl];
  const int qmax = symmetric ? (1 << (bits - 1)) - 1 : (1 << bits) - 1;
  const int qmin = symmetric ? -qmax : 0;
  uint2* out = reinterpret_cast<uint2*>(codes + row * K);
  // fast path for every element (FP32 / integer pipes); the rare elements within the
  // margin of a .5 tie (or with |x/s| >= 2^21) are fixed afterwards by ONE rolled loop
  // that re-reads them and overwrites their code byte with the correctly rounded f64
  // result (inlining the f64 division per unrolled element made this kernel
  // instruction-bound; an out-of-line call forced the register arrays to the stack)
  // Everything on the FP32 / ALU pipes, no F2I / FRND (conversion-pipe) instructions:
  // n = rint(q) by the 1.5*2^23 magic add (|q| < 2^21), the code byte from the low
  // mantissa bits of (clamp(n + zp) + 1.5*2^23).
  constexpr float kMagic = 12582912.f;
  // m = q + (1.5 2^23 + zp) rounds q + zp to an integer whose f32 bits are 0x4B400000 + rint(q) + zp
  // (|q + zp| < 2^22; at exact .5 ties the rounding may differ from rint(q) + zp, but those are
  // flagged below); the clamp runs on those bits (integer min / max), whose low byte is the code
  const float mz = kMagic + float(zp);
  const int bmin = 0x4B400000 + qmin, bmax = 0x4B400000 + qmax;
  constexpr int kBadWords = (8 * kCpt + 63) / 64;
  uint64_t bad[kBadWords];  // bit 8j+i: element i of group j takes the exact path
#pragma unroll
  for (int b = 0; b < kBadWords; ++b) bad[b] = 0;
#pragma unroll
  for (int j = 0; j < kCpt; ++j) {
    const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
    uint32_t cb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float xf = __uint_as_float((i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16));
      const float q = xf * inv32;  // |q - x/s| <= |q| * 2^-22.9
      const float m = q + mz;      // 1.5 2^23 + zp + rint(q)
      const float d = q - (m - mz);  // exact, |d| <= 1/2
      // not within the margin of a .5 tie: |d| + |q| 2^-21 < 1/2 (also excludes |q| >= 2^21,
      // where the bound analysis stops)
      const bool ok = fmaf(fabsf(q), 0x1p-21f, fabsf(d)) < 0.5f;
      bad[(8 * j + i) >> 6] |= uint64_t(!ok) << ((8 * j + i) & 63);
      cb[i] = uint32_t(min(max(__float_as_int(m), bmin), bmax));  // low byte = two's-complement code
    }
    const uint2 v = make_uint2(__byte_perm(__byte_perm(cb[0], cb[1], 0x0040), __byte_perm(cb[2], cb[3], 0x0040), 0x5410),
                               __byte_perm(__byte_perm(cb[4], cb[5], 0x0040), __byte_perm(cb[6], cb[7], 0x0040), 0x5410));
    const int c8 = t + j * kTpr;
    if (c8 < n8) out[c8] = v;
  }
  // the flagged elements only (typically none: a row's slowest thread bounds the kernel, so
  // no pass over all elements): re-read, exact code, overwrite the byte
#pragma unroll
  for (int b = 0; b < kBadWords; ++b) {
    uint64_t m = bad[b];
#pragma unroll 1
    while (m) {
      const int bit = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      const int e = 64 * b + bit;  // 8j + i; out-of-range groups hold zeros, which never flag
      const int col = (t + (e >> 3) * kTpr) * 8 + (e & 7);
      codes[row * K + col] = int8_t(int_code_tie(__bfloat162float(x[row * ldx + col]), sc, inv32, zp, qmin, qmax));
    }
  }
  if (xs_kind != 0) {
    // salient slice from this row's codes (written above by this row's threads)
    named_bar_sync(1 + rl, kTpr);
    for (int j = t; j < r; j += kTpr) {
      const int col = sidx ? sidx[j] : j;
      const int c = symmetric ? int(codes[row * K + col]) : int(uint8_t(codes[row * K + col]));
      if (xs_kind == 1)
        reinterpret_cast<__nv_bfloat16*>(xs_out)[row * r + j] = __int2bfloat16_rn(c - zp);
      else
        reinterpret_cast<int8_t*>(xs_out)[row * r + j] = int8_t(c);
    }
  }
  }  // row_ok
#pragma unroll
  for (int j = 0; j < kCpt; ++j) raw[j] = nxt[j];
  }  // row groups
}

// ------------------------------------------------------------------ packers
// Reference MX artefacts (unpacked codes uint8 [rows, cols], exps int32 [rows, cols/32])
// -> device packed codes + tiled E8M0.
__global__ void pack_mx_kernel(const uint8_t* __restrict__ codes, const int32_t* __restrict__ exps, int64_t rows,
                               int64_t cols, uint8_t* __restrict__ packed, uint8_t* __restrict__ sf, int kc_pad,
                               int tiled_ksteps) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per_row = cols / 8;
  if (t >= rows * per_row) return;
  const int64_t row = t / per_row, c0 = (t - row * per_row) * 8;
  uint32_t p = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) p |= uint32_t(codes[row * cols + c0 + i] & 0xF) << (4 * i);
  size_t off;
  if (tiled_ksteps > 0) {
    // pre-tiled weights: [row/128][byte/128][row%128][byte%128] -> every 16-KB TMA box is contiguous
    const int64_t cb = c0 / 2;
    off = ((size_t(row >> 7) * tiled_ksteps + size_t(cb >> 7)) * 128 + size_t(row & 127)) * 128 + size_t(cb & 127);
  } else {
    off = size_t(row) * (cols / 2) + c0 / 2;
  }
  *reinterpret_cast<uint32_t*>(packed + off) = p;
  if ((c0 & 31) == 0) sf[sf_offset(row, c0 / 32, kc_pad)] = uint8_t(exps[row * (cols / 32) + c0 / 32] + 127);
}

// device MX layout -> reference artefact layout (unpacked codes, int32 exponents)
__global__ void unpack_mx_kernel(const uint8_t* __restrict__ packed, const uint8_t* __restrict__ sf, int64_t rows,
                                 int64_t cols, int kc_pad, uint8_t* __restrict__ codes, int32_t* __restrict__ exps) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per_row = cols / 8;
  if (t >= rows * per_row) return;
  const int64_t row = t / per_row, c0 = (t - row * per_row) * 8;
  const uint32_t p = *reinterpret_cast<const uint32_t*>(packed + row * (cols / 2) + c0 / 2);
#pragma unroll
  for (int i = 0; i < 8; ++i) codes[row * cols + c0 + i] = uint8_t((p >> (4 * i)) & 0xF);
  if ((c0 & 31) == 0) exps[row * (cols / 32) + c0 / 32] = int32_t(sf[sf_offset(row, c0 / 32, kc_pad)]) - 127;
}

// MX activation in the device layout -> the decoded values mx_decode(x_mx) = e2m1(code) * 2^e
// (mxfmt.py:111-113) as bf16 [rows, cols]: every value is exact in bf16 (one mantissa bit, the
// f32 exponent range, bf16 subnormals reach 2^-133).  The SVD baseline's first factor product
// runs on it (compensate.py:327).  One thread per 8 elements (grid: column blocks x rows): one
// 4-B code load, one 16-B store.
__global__ void mx_decode_bf16_kernel(const uint8_t* __restrict__ packed, const uint8_t* __restrict__ sf,
                                      int64_t rows, int64_t cols, int kc_pad, __nv_bfloat16* __restrict__ out) {
  const int64_t c0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (c0 >= cols) return;
  for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
    const uint32_t p = *reinterpret_cast<const uint32_t*>(packed + row * (cols / 2) + c0 / 2);
    const int e = int(sf[sf_offset(row, int(c0 / 32), kc_pad)]) - 127;
    // |value| = (1 + (m & 1) / 2) 2^((m >> 1) - 1 + e) for m >= 2, 2^(e - 1) for m = 1: the bf16
    // bits directly (biased exponent, one mantissa bit); a block whose smallest non-zero value
    // would be subnormal (e <= -125), or whose largest would overflow (e >= 126, not reachable
    // from finite bf16 / f32 input), takes ldexpf
    uint32_t w[4];
    if (e > -125 && e < 126) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t hv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t c = (p >> (8 * i + 4 * h)) & 0xFu;
          const uint32_t m = c & 7u;
          const int ex = (m >= 2 ? int(m >> 1) - 1 : -1) + e + 127;
          const uint32_t mag = m == 0 ? 0u : (uint32_t(ex) << 7) | ((m >= 2 ? (m & 1u) : 0u) << 6);
          hv[h] = mag | ((c & 8u) << 12);
        }
        w[i] = hv[0] | (hv[1] << 16);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t c = (p >> (8 * i + 4 * h)) & 0xFu;
          const uint32_t m = c & 7u;  // 0, .5, 1, 1.5, 2, 3, 4, 6
          const float mag = m < 4 ? 0.5f * float(m) : float(1u << ((m >> 1) - 1)) * (m & 1 ? 1.5f : 1.f);
          v[h] = ldexpf(c & 8u ? -mag : mag, e);
        }
        w[i] = pack_bf16x2(v[0], v[1]);
      }
    }
    *reinterpret_cast<uint4*>(out + row * cols + c0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// reference INT codes int32 [K, N] (in, out) -> int8 [N, K] K-major, 32x32 smem transpose
__global__ void transpose_codes_kernel(const int32_t* __restrict__ src, int64_t K, int64_t N, int8_t* __restrict__ dst) {
  __shared__ int8_t tile[32][33];
  const int64_t k0 = int64_t(blockIdx.y) * 32, n0 = int64_t(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t k = k0 + i, n = n0 + threadIdx.x;
    if (k < K && n < N) tile[i][threadIdx.x] = int8_t(src[k * N + n]);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t n = n0 + i, k = k0 + threadIdx.x;
    if (k < K && n < N) dst[n * K + k] = tile[threadIdx.x][i];
  }
}

// reference INT codes int32 [K, N] (two's complement, |code| <= 8) -> packed nibbles tiled
// [N/128][K/128][128 rows][64 B]: the W4 CTA-pair kernel's loader warps read one contiguous block
// per 128-K step.  Within a row's 64 B, 8 bytes hold one 16-element chunk; byte j of each 4-byte
// word holds elements j (low nibble) and j + 4 (high nibble) of that word's 8 elements, the order
// widen_int4x8 expands without byte shuffles.  One thread per output byte.
__global__ void pack_int4_tiled_kernel(const int32_t* __restrict__ src, int64_t K, int64_t N, int ksteps,
                                       uint8_t* __restrict__ dst) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t bidx = blockIdx.y;  // byte of the row's packed K: step = bidx / 64, b = bidx % 64
  if (n >= N) return;
  const int64_t step = bidx >> 6;
  const int b = int(bidx & 63);
  const int e_lo = (b >> 3) * 16 + ((b >> 2) & 1) * 8 + (b & 3);
  const int64_t k_lo = step * 128 + e_lo, k_hi = k_lo + 4;
  const int32_t lo = k_lo < K ? src[k_lo * N + n] : 0;
  const int32_t hi = k_hi < K ? src[k_hi * N + n] : 0;
  const size_t off = ((size_t(n >> 7) * ksteps + size_t(step)) * 128 + size_t(n & 127)) * 64 + size_t(b);
  dst[off] = uint8_t((lo & 0xF) | ((hi & 0xF) << 4));
}

// colsum[n] = sum_k codes[k, n]; scale f64 -> f32 copy
__global__ void colsum_kernel(const int32_t* __restrict__ src, int64_t K, int64_t N, const double* __restrict__ s64,
                              int32_t* __restrict__ colsum, float* __restrict__ s32) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  int32_t acc = 0;
  for (int64_t k = 0; k < K; ++k) acc += src[k * N + n];
  colsum[n] = acc;
  if (s32) s32[n] = float(s64[n]);
}

// dense R (f64 [r, N]) -> L^T bf16 [N, r], one rounding f64 -> bf16
// Group-wise weights (row groups of gs input rows): per column n, the group
// colsums, the fp32 group scales and the folded zero-point term
// C[n] = sum_g s[g,n] * colsum_g[n] (+ sr[n] * colsum_r[n]), accumulated in f64.
__global__ void group_pack_kernel(const int32_t* __restrict__ src, int64_t K, int64_t N, int64_t gs,
                                  const double* __restrict__ s64, const double* __restrict__ sr64,
                                  const int32_t* __restrict__ colsum_r, int32_t* __restrict__ colsum_g,
                                  float* __restrict__ sw_g, float* __restrict__ cterm) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double c = 0.0;
  for (int64_t g = 0; g < K / gs; ++g) {
    int32_t acc = 0;
    for (int64_t k = g * gs; k < (g + 1) * gs; ++k) acc += src[k * N + n];
    colsum_g[g * N + n] = acc;
    sw_g[g * N + n] = float(s64[g * N + n]);
    c += s64[g * N + n] * double(acc);
  }
  if (sr64) c += sr64[n] * double(colsum_r[n]);
  cterm[n] = float(c);
}

// f64 R [r, N] -> two bf16 planes [N, r]: hi = bf16(R), lo = bf16(R - hi)
__global__ void dense_r_split_kernel(const double* __restrict__ src, int64_t r, int64_t N,
                                     __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= r * N) return;
  const int64_t n = t / r, j = t - n * r;
  const double v = src[j * N + n];
  const __nv_bfloat16 h = __double2bfloat16(v);
  hi[n * r + j] = h;
  lo[n * r + j] = __double2bfloat16(v - double(__bfloat162float(h)));
}
__global__ void dense_r_kernel(const double* __restrict__ src, int64_t r, int64_t N, __nv_bfloat16* __restrict__ dst) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= r * N) return;
  const int64_t n = t / r, j = t - n * r;
  dst[n * r + j] = __double2bfloat16(src[j * N + n]);
}

}  // namespace serq
