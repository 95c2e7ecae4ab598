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
template <typename T, int kMxRows = serq::kMxRows>
__global__ void __launch_bounds__(256) mx_encode_fast_kernel(const T* __restrict__ x, int M, int K, int64_t ldx,
                                                             uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
                                                             int kc_pad) {
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
// -- the normalised activation never goes to HBM.  Arithmetic is the
// reference's, in f64 and in the same order (square, mean = sum / K, + eps,
// sqrt, divide, multiply), every step IEEE-rounded; only the summation order of
// the squares differs (exact whenever the squares' exponents span < 2^37), and
// the f64 E2M1 rounding is the exact software path.  The row is read twice: the
// second pass hits L1 / L2, so HBM sees it once.
template <typename T>
__device__ __forceinline__ void load8_f64(const T* __restrict__ p, bool ok, double (&v)[8]) {
  if (!ok) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0;
    return;
  }
  if constexpr (In<T>::kId == 0) {
    const uint4 raw = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = double(__uint_as_float(w[i] << 16));
      v[2 * i + 1] = double(__uint_as_float(w[i] & 0xFFFF0000u));
    }
  } else {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_mx_encode_kernel(const T* __restrict__ x, int K, int64_t ldx,
                                                                const double* __restrict__ gain, double eps,
                                                                uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
                                                                int kc_pad) {
  __shared__ double red[8];
  pdl_launch_dependents();
  pdl_wait();
  const int64_t row = blockIdx.x;
  const T* xr = x + row * ldx;
  double ss = 0.0;
  for (int c = threadIdx.x * 8; c < K; c += 256 * 8) {
    double v[8];
    load8_f64(xr + c, true, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fma(v[i], v[i], ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  double total = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) total += red[w];
  const double rms = sqrt(total / double(K) + eps);
  const int iters = (K + 2047) / 2048;
  for (int it = 0; it < iters; ++it) {
    const int c = it * 2048 + threadIdx.x * 8;
    const bool ok = c < K;
    double v[8];
    load8_f64(xr + c, ok, v);
    double amax = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = ok ? (v[i] / rms) * gain[c + i] : 0.0;
      amax = fmax(amax, fabs(v[i]));
    }
    amax = fmax(amax, __shfl_xor_sync(0xffffffff, amax, 1));
    amax = fmax(amax, __shfl_xor_sync(0xffffffff, amax, 2));
    const int e = mx_block_exp_f64(amax);
    const double inv = ldexp(1.0, -e);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double s = v[i] * inv;  // exact: power-of-two scaling
      const uint32_t idx = e2m1_index_sw(fabs(s));
      packed |= ((s < 0.0 && idx > 0) ? idx + 8 : idx) << (4 * i);
    }
    if (ok) {
      *reinterpret_cast<uint32_t*>(codes + row * (K / 2) + c / 2) = packed;
      if ((threadIdx.x & 3) == 0) sf[sf_offset(row, c / 32, kc_pad)] = uint8_t(e + 127);
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
template <int kNV>
__global__ void __launch_bounds__(256) int_quant_bf16_kernel(const __nv_bfloat16* __restrict__ x, int K, int64_t ldx,
                                                             int bits, int symmetric, int8_t* __restrict__ codes,
                                                             double* __restrict__ scale64, float* __restrict__ scale32,
                                                             int32_t* __restrict__ zp_out,
                                                             const int32_t* __restrict__ sidx, int r,
                                                             void* __restrict__ xs_out, int xs_kind) {
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * ldx);
  const int n8 = K >> 3;
  __shared__ float red_lo[8], red_hi[8];
  __shared__ double s_scale;
  __shared__ int s_zp;
  uint4 raw[kNV];
  float lo = INFINITY, hi = -INFINITY;
#pragma unroll
  for (int j = 0; j < kNV; ++j) {
    const int c8 = threadIdx.x + j * 256;
    raw[j] = c8 < n8 ? __ldg(xr + c8) : make_uint4(0, 0, 0, 0);
    if (c8 < n8) {
      const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xFFFF0000u);
        lo = fminf(lo, fminf(a, b));
        hi = fmaxf(hi, fmaxf(a, b));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffff, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffff, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red_lo[threadIdx.x >> 5] = lo;
    red_hi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      lo = fminf(lo, red_lo[w]);
      hi = fmaxf(hi, red_hi[w]);
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
    s_scale = sc;
    s_zp = zp;
    scale64[row] = sc;
    scale32[row] = float(sc);
    if (zp_out) zp_out[row] = zp;
  }
  __syncthreads();
  const double sc = s_scale;
  const int zp = s_zp;
  const double inv64 = 1.0 / sc;
  const float inv32 = float(inv64);
  const int qmax = symmetric ? (1 << (bits - 1)) - 1 : (1 << bits) - 1;
  const int qmin = symmetric ? -qmax : 0;
  uint2* out = reinterpret_cast<uint2*>(codes + row * K);
#pragma unroll
  for (int j = 0; j < kNV; ++j) {
    const int c8 = threadIdx.x + j * 256;
    if (c8 >= n8) continue;
    const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
    uint32_t packed[2] = {0u, 0u};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t hbits = (i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16);
      const __nv_bfloat16 xv = __ushort_as_bfloat16(static_cast<unsigned short>(hbits >> 16));
      const double qd = rint_quot<__nv_bfloat16>(xv, sc, inv32, inv64) + double(zp);
      const int q = int(fmin(fmax(qd, double(qmin)), double(qmax)));
      packed[i >> 2] |= (uint32_t(q) & 0xFFu) << (8 * (i & 3));
    }
    out[c8] = make_uint2(packed[0], packed[1]);
  }
  if (xs_kind != 0) {
    __syncthreads();
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
      const int col = sidx ? sidx[j] : j;
      const int c = symmetric ? int(codes[row * K + col]) : int(uint8_t(codes[row * K + col]));
      if (xs_kind == 1)
        reinterpret_cast<__nv_bfloat16*>(xs_out)[row * r + j] = __int2bfloat16_rn(c - zp);
      else
        reinterpret_cast<int8_t*>(xs_out)[row * r + j] = int8_t(c);
    }
  }
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

// reference INT codes int32 [K, N] (|code| <= 8) -> packed two's-complement nibbles,
// tiled [N/128][K/128][128 rows][64 B] (k even -> low nibble); the CTA-pair INT
// kernel TMA-loads one contiguous 8-KB tile per 128-K step and widens in SMEM.
__global__ void pack_int4_tiled_kernel(const int32_t* __restrict__ src, int64_t K, int64_t N, int ksteps,
                                       uint8_t* __restrict__ dst) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t k = int64_t(blockIdx.y) * 2;
  if (n >= N || k >= K) return;
  const int32_t lo = src[k * N + n];
  const int32_t hi = k + 1 < K ? src[(k + 1) * N + n] : 0;
  const size_t off = ((size_t(n >> 7) * ksteps + size_t(k >> 7)) * 128 + size_t(n & 127)) * 64 + size_t((k & 127) >> 1);
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
__global__ void dense_r_kernel(const double* __restrict__ src, int64_t r, int64_t N, __nv_bfloat16* __restrict__ dst) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= r * N) return;
  const int64_t n = t / r, j = t - n * r;
  dst[n * r + j] = __double2bfloat16(src[j * N + n]);
}

}  // namespace serq
