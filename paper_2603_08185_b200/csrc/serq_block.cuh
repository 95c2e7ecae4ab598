// serq_block.cuh -- the decoder block's non-SERQ glue for decode-sized token counts.
//
// Between the SERQ linears the reference block (toy_block_graph, toymodel.py:88-124) runs
// RMSNorm (saliency.py:194-196), the per-head token-batch attention (attention_mix,
// saliency.py:203-216), SiLU gating (saliency.py:199-200) and residual adds, all in full
// precision.  At M <= 16 tokens each of those is a launch-bound micro-kernel in PyTorch (9 per
// block); these kernels fuse them into 4 f32 kernels that read the linears' bf16 outputs in
// place (no casts, no .contiguous() copies):
//   * rmsnorm(x [+ o]) -> (res, h): the residual add fused with the next RMSNorm;
//   * silu(gate) * up;
//   * attention over the <= 16 tokens of the batch straight from the fused q/k/v output rows.
// All arithmetic is f32 (the PyTorch path's precision); results match it to f32 rounding.
#pragma once
#include "serq_ptx.cuh"

namespace serq {

// res = x (+ float(o)); h = res * rsqrt(mean(res^2) + eps) * g (h == nullptr: the add alone).  One
// 256-thread CTA per row.
__global__ void __launch_bounds__(256) block_add_rmsnorm_kernel(const float* __restrict__ x,
                                                                const __nv_bfloat16* __restrict__ o, int64_t ldo,
                                                                int M, int H, const float* __restrict__ g, float eps,
                                                                float* __restrict__ res, float* __restrict__ h) {
  __shared__ float red[8];
  pdl_launch_dependents();
  pdl_wait();
  const int row = blockIdx.x;
  if (row >= M) return;
  const float* xr = x + int64_t(row) * H;
  float ss = 0.f;
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    float v = xr[c];
    if (o) v += __bfloat162float(o[int64_t(row) * ldo + c]);
    if (res) res[int64_t(row) * H + c] = v;
    ss = fmaf(v, v, ss);
  }
  if (!h) return;  // the residual add alone (the block's output)
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float rs = rsqrtf(tot / float(H) + eps);
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    float v = xr[c];
    if (o) v += __bfloat162float(o[int64_t(row) * ldo + c]);
    h[int64_t(row) * H + c] = v * rs * g[c];
  }
}

// The same with the row held in registers: 1024 threads per row, kC 16-B chunks per thread (H <=
// 4096 kC, H % 4 == 0, 16-B aligned rows, o rows 8-B aligned).  Every load of the row is issued
// before the first use (the loop above waits out one global round trip per 256 elements -- at
// M = 1 the whole block's latency chain), and res / h are written from the registers.
template <int kC>
__global__ void __launch_bounds__(1024) block_add_rmsnorm_reg_kernel(const float* __restrict__ x,
                                                                    const __nv_bfloat16* __restrict__ o, int64_t ldo,
                                                                    int M, int H, const float* __restrict__ g,
                                                                    float eps, float* __restrict__ res,
                                                                    float* __restrict__ h) {
  __shared__ float red[32];
  pdl_launch_dependents();
  const int row = blockIdx.x, t = threadIdx.x;
  float4 gv[kC];
#pragma unroll
  for (int j = 0; j < kC; ++j) {  // the gain does not depend on the previous kernel
    const int c = 4 * (t + 1024 * j);
    gv[j] = (h && c < H) ? __ldg(reinterpret_cast<const float4*>(g + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  pdl_wait();
  if (row >= M) return;
  float4 v[kC];
#pragma unroll
  for (int j = 0; j < kC; ++j) {
    const int c = 4 * (t + 1024 * j);
    v[j] = c < H ? *reinterpret_cast<const float4*>(x + int64_t(row) * H + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (o) {
    uint2 ov[kC];
#pragma unroll
    for (int j = 0; j < kC; ++j) {
      const int c = 4 * (t + 1024 * j);
      ov[j] = c < H ? *reinterpret_cast<const uint2*>(o + int64_t(row) * ldo + c) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < kC; ++j) {
      v[j].x += __uint_as_float(ov[j].x << 16);
      v[j].y += __uint_as_float(ov[j].x & 0xFFFF0000u);
      v[j].z += __uint_as_float(ov[j].y << 16);
      v[j].w += __uint_as_float(ov[j].y & 0xFFFF0000u);
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kC; ++j) {
    ss = fmaf(v[j].x, v[j].x, ss);
    ss = fmaf(v[j].y, v[j].y, ss);
    ss = fmaf(v[j].z, v[j].z, ss);
    ss = fmaf(v[j].w, v[j].w, ss);
    const int c = 4 * (t + 1024 * j);
    if (res && c < H) *reinterpret_cast<float4*>(res + int64_t(row) * H + c) = v[j];
  }
  if (!h) return;  // the residual add alone (the block's output)
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
  if ((t & 31) == 0) red[t >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 32; ++w) tot += red[w];
  const float rs = rsqrtf(tot / float(H) + eps);
#pragma unroll
  for (int j = 0; j < kC; ++j) {
    const int c = 4 * (t + 1024 * j);
    if (c < H)
      *reinterpret_cast<float4*>(h + int64_t(row) * H + c) =
          make_float4(v[j].x * rs * gv[j].x, v[j].y * rs * gv[j].y, v[j].z * rs * gv[j].z, v[j].w * rs * gv[j].w);
  }
}

// mid = silu(float(gate)) * float(up) = g / (1 + exp(-g)) * u, f32
__global__ void __launch_bounds__(256) block_silu_mul_kernel(const __nv_bfloat16* __restrict__ gate, int64_t ldg,
                                                             const __nv_bfloat16* __restrict__ up, int64_t ldu, int M,
                                                             int F, float* __restrict__ mid) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(M) * F) return;
  const int64_t r = i / F, c = i - r * F;
  const float gv = __bfloat162float(gate[r * ldg + c]);
  mid[i] = gv / (1.f + __expf(-gv)) * __bfloat162float(up[r * ldu + c]);
}

// out[t, head * hd + d] = sum_s softmax_s(q_t . k_s * scale) v_s[d] over the M <= 16 tokens of
// the batch (no mask, saliency.py:203-216); one CTA (hd = 128 threads, thread = channel d) per
// (head, query), q / k / v read from rows of pitch ldq / ldk / ldv (e.g. the fused q/k/v
// output: column views of one buffer)
template <int kMaxM>
__global__ void __launch_bounds__(128) block_attention_small_kernel(const __nv_bfloat16* __restrict__ q, int64_t ldq,
                                                                    const __nv_bfloat16* __restrict__ k, int64_t ldk,
                                                                    const __nv_bfloat16* __restrict__ v, int64_t ldv,
                                                                    int M, int hd, float scale,
                                                                    float* __restrict__ out, int64_t ldo) {
  __shared__ float red[kMaxM][4];
  pdl_launch_dependents();
  pdl_wait();
  const int head = blockIdx.x, t = blockIdx.y, d = threadIdx.x, lane = d & 31, w = d >> 5;
  const int64_t col = int64_t(head) * hd + d;
  const float qd = __bfloat162float(q[t * ldq + col]);
  float part[kMaxM], vd[kMaxM];
#pragma unroll
  for (int s = 0; s < kMaxM; ++s) {
    part[s] = s < M ? qd * __bfloat162float(k[s * ldk + col]) : 0.f;
    vd[s] = s < M ? __bfloat162float(v[s * ldv + col]) : 0.f;
  }
#pragma unroll
  for (int s = 0; s < kMaxM; ++s)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part[s] += __shfl_xor_sync(0xffffffffu, part[s], o);
  if (lane == 0)
#pragma unroll
    for (int s = 0; s < kMaxM; ++s) red[s][w] = part[s];
  __syncthreads();
  float logit[kMaxM], mx = -INFINITY;
#pragma unroll
  for (int s = 0; s < kMaxM; ++s) {
    logit[s] = s < M ? (red[s][0] + red[s][1] + red[s][2] + red[s][3]) * scale : -INFINITY;
    mx = fmaxf(mx, logit[s]);
  }
  float den = 0.f, acc = 0.f;
#pragma unroll
  for (int s = 0; s < kMaxM; ++s) {
    if (s >= M) break;
    const float p = __expf(logit[s] - mx);
    den += p;
    acc = fmaf(p, vd[s], acc);
  }
  out[t * ldo + col] = acc / den;
}

}  // namespace serq
