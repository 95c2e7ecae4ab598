// FP64 vs FP32 FMA throughput and the f32->f64 conversion rate on this GPU (one-off probe):
// 8 independent chains per thread, 148 x 8 CTAs of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_rate(T* out, int iters, T a, T b) {
  T r[8];
  for (int i = 0; i < 8; ++i) r[i] = T(threadIdx.x + i);
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = r[i] * a + b;
  T s = 0;
  for (int i = 0; i < 8; ++i) s += r[i];
  if (s == T(1.2345)) out[0] = s;
}
__global__ void cvt_rate(double* out, int iters, float a) {
  double r[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { r[i] = 0; f[i] = a * (threadIdx.x + i); }
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) { r[i] += double(f[i]); f[i] = f[i] * 1.0000001f; }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += r[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, grid = 148 * 8, blk = 256;
  const double ops = double(grid) * blk * iters * 8;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); fma_rate<float><<<grid, blk>>>((float*)d, iters, 1.0000001f, 1e-7f); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("FFMA %.1f G/s\n", ops / ms / 1e6);
    cudaEventRecord(a); fma_rate<double><<<grid, blk>>>(d, iters / 16, 1.0000001, 1e-7); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("DFMA %.1f G/s\n", ops / 16 / ms / 1e6);
    cudaEventRecord(a); cvt_rate<<<grid, blk>>>(d, iters / 16, 1e-3f); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("F2F+DADD %.1f G/s (per element)\n", ops / 16 / ms / 1e6);
  }
  return 0;
}
