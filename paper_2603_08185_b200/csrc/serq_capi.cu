#include <cstdlib>
// serq_capi.cu -- the extern "C" boundary (include/serq_b200.h): validation,
// weight handles, tensor maps, launches.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>

#include "../../include/serq_b200.h"
#include "serq_gemm.cuh"
#include "serq_gemm_mx.cuh"
#include "serq_gemm_mx2.cuh"
#include "serq_gemm_mx3.cuh"
#include "serq_gemm_decode3.cuh"
#include "serq_gemm_i8.cuh"
#include "serq_gemm_i8g.cuh"
#include "serq_gemv_i8.cuh"
#include "serq_block.cuh"
#include "serq_quant.cuh"

#ifndef SERQ_GEMV_I8G_MAX_M
#define SERQ_GEMV_I8G_MAX_M 32  // group-wise INT handles with few tiles: the token-grouped gemv up to this many rows
#endif

using namespace serq;

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
thread_local const char* g_last_kernel = "";  // name of the last kernel launched on this thread (tests)
#ifdef SERQ_DIAG
// diagnostics build only (tools/): kernel-selection / feed-isolation switches and timestamps
int g_debug_flags = 0;
long long* g_debug_ts = nullptr;
#else
constexpr int g_debug_flags = 0;
constexpr long long* g_debug_ts = nullptr;
#endif

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) return fail(SERQ_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define LAUNCH_CHECK(what)                                                                        \
  do {                                                                                            \
    cudaError_t e_ = cudaGetLastError();                                                          \
    if (e_ != cudaSuccess) return fail(SERQ_ECUDA, "%s launch: %s", what, cudaGetErrorString(e_)); \
    ++g_launches;                                                                                 \
    g_last_kernel = what;                                                                         \
  } while (0)

inline cudaStream_t S(serq_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
// SF chunks (4 x 32-blocks = 128 K) per 128-row block, padded to the 256-K pipeline step
inline int kc_pad_of(int64_t cols) { return int(cdiv(cols, 256) * 2); }
inline int64_t sf_bytes_of(int64_t rows, int64_t cols) { return cdiv(rows, 128) * kc_pad_of(cols) * 512; }

// ---------------------------------------------------------------- tensor maps
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D row-major map: `inner` elements per row (contiguous), `rows` rows, row pitch in bytes.
int make_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t rows,
             uint64_t pitch_bytes, uint32_t box_inner, uint32_t box_rows,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(SERQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (pitch_bytes & 15))
    return fail(SERQ_EINVAL, "tensor base and row pitch must be 16-byte aligned (pitch %llu)",
                (unsigned long long)pitch_bytes);
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SERQ_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return SERQ_OK;
}

// launch with programmatic stream serialization: the kernel may start under the
// previous kernel's tail and must call griddepcontrol.wait before reading its inputs
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Per-device state: SM count and which kernels have their dynamic shared-memory
// limit raised (a process may drive several GPUs; both are per device).
constexpr int kMaxDevices = 64;
int sm_count() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

template <typename... KArgs>
cudaError_t set_smem_attr(void (*kernel)(KArgs...), int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kernel), bytes);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

// resident CTAs per SM of a kernel at (threads, dynamic smem), cached per device
template <typename... KArgs>
int occupancy_of(void (*kernel)(KArgs...), int threads, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kernel), threads, smem);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, size_t(smem)) != cudaSuccess || n < 1) n = 1;
  cache[key] = n;
  return n;
}

// scale factors as rows of 128 B (one 1-KB box = 2 SF chunks of a 128-row block)
int make_sf_map(CUtensorMap* m, const uint8_t* sf, int64_t rows, int64_t cols) {
  return make_map(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, sf, 128, uint64_t(sf_bytes_of(rows, cols) / 128), 128, 128, 8,
                  CU_TENSOR_MAP_SWIZZLE_NONE);
}

template <int kMode>
int ensure_attr() {
  CK(set_smem_attr(serq_linear_kernel<kMode>, kSmemBytes));
  return SERQ_OK;
}

}  // namespace

// ------------------------------------------------------------------ handle
constexpr int kE2eMaxChunks = 16;
constexpr int kMaxSeg = 4;

struct serq_linear {
  int mode = 0;  // kModeMX / kModeI8
  int64_t N = 0, K = 0;
  int r = 0, r_mode = SERQ_R_NONE, w_bits = 4, contiguous = 1, w_ksteps = 0;
  void* w = nullptr;        // MX packed [N, K/2] | INT s8 [N, K]
  uint8_t* sfw = nullptr;   // MX scale factors
  void* rbuf = nullptr;     // MX packed [N, r/2] | INT s8 [N, r] | bf16 [N, r]
  uint8_t* sfr = nullptr;
  float* sw = nullptr;
  int32_t* colsum = nullptr;
  float* sr = nullptr;
  int32_t* colsum_r = nullptr;
  CUtensorMap map_b, map_r;
  CUtensorMap map_b128, map_r128, map_sfw, map_sfr;  // CTA-pair kernel: 128-row B boxes, scale-factor maps
  CUtensorMap map_b64;                                // pair3 narrow (256 x 128) last-round tiles: 64-row B boxes
  CUtensorMap map_r32, map_sfr4;                     // pair3 kernel: R as 32-B swizzled rows, 512-B SF boxes
  bool has_r32 = false;
  void* rdec = nullptr;                               // decode: R zero-padded to 64 / 128 columns (r != 64)
  CUtensorMap map_rdec;                               // decode: R rows of dec_rw bytes (32- / 64-byte swizzle)
  int dec_rw = 0;                                     // 0: the decode kernel cannot take this R (r > 128)
  // fused linears (serq_linear_set_segments): row segments, each with its own salient set; the
  // quantizer's salient buffer holds 128 columns per segment (xs_cols = 128 * nseg)
  int nseg = 1;
  int64_t seg_row[kMaxSeg] = {0};  // start row of segments 1 .. nseg-1
  const serq_linear* parent = nullptr;  // views (serq_linear_view): the handle owning the memory
  CUtensorMap map_r_pair;                            // INT pair kernel maps (R with 128-row boxes)
  bool has_w4 = false;                               // INT: weights packed INT4, tiled [N/128][K/128][128][64 B]
  int64_t w_bytes = 0;                               // bytes of the resident main weights
  CUtensorMap map_w8;                                // INT pair kernel, direct int8 weights: 128 B x 128-row boxes
  CUtensorMap map_w8_64, map_r_pair64;               // the same with 64-row boxes (128-column tiles)
  // INT, group-wise weight scales along K (serq_pack_int_grouped)
  int groups = 1, gsteps = 0;
  bool use_i8g = false;        // served by serq_i8g_pair_kernel
  float* sw_g = nullptr;       // [G][N]
  int32_t* colsum_g = nullptr; // [G][N]
  float* cterm = nullptr;      // [N]
  // end-to-end scratch
  int64_t ws_m = 0;
  void* ws_x = nullptr;
  uint8_t* ws_codes = nullptr;
  uint8_t* ws_sf = nullptr;
  void* ws_y = nullptr;
  uint8_t* ws_xs = nullptr;   // gather layers: x[:, idx] codes and scale factors per chunk (INT: xs slice)
  uint8_t* ws_xsf = nullptr;
  double* ws_s64 = nullptr;   // INT end to end: per-token scales and zero points
  float* ws_s32 = nullptr;
  int32_t* ws_zp = nullptr;
  // end-to-end pipeline: H2D and D2H copy streams + per-chunk events (created lazily)
  cudaStream_t e2e_in = nullptr, e2e_out = nullptr;
  std::mutex e2e_mu;  // the end-to-end scratch and streams are per handle: one host call at a time
  cudaEvent_t e2e_ev[3 * kE2eMaxChunks + 1] = {};
};

namespace {
void free_handle(serq_linear* h) {
  // scratch (end-to-end buffers, copy streams, events) always belongs to the handle; the packed
  // weights only to an owning handle (a view references its parent's)
  void* scratch[] = {h->ws_x, h->ws_codes, h->ws_sf, h->ws_y, h->ws_xs, h->ws_xsf, h->ws_s64, h->ws_s32, h->ws_zp};
  for (void* p : scratch)
    if (p) cudaFree(p);
  if (!h->parent) {
    void* owned[] = {h->w, h->sfw, h->rbuf, h->sfr, h->sw, h->colsum, h->sr, h->colsum_r,
                     h->sw_g, h->colsum_g, h->cterm, h->rdec};
    for (void* p : owned)
      if (p) cudaFree(p);
  }
  for (cudaEvent_t e : h->e2e_ev)
    if (e) cudaEventDestroy(e);
  if (h->e2e_in) cudaStreamDestroy(h->e2e_in);
  if (h->e2e_out) cudaStreamDestroy(h->e2e_out);
  delete h;
}
}  // namespace

extern "C" {

const char* serq_last_error(void) { return g_err.c_str(); }
const char* serq_version(void) { return "serq_b200 0.1 (sm_100a tcgen05)"; }
int serq_last_launch_count(void) { return g_launches; }
const char* serq_last_kernel(void) { return g_last_kernel; }
int serq_set_debug_flags(int flags) {
#ifdef SERQ_DIAG
  g_debug_flags = flags;
  return SERQ_OK;
#else
  return flags ? fail(SERQ_EINVAL, "debug flags need a SERQ_DIAG build of the library (tools/ only)") : SERQ_OK;
#endif
}
int serq_set_debug_timestamps(long long* dev_buf) {
#ifdef SERQ_DIAG
  g_debug_ts = dev_buf;
  return SERQ_OK;
#else
  return dev_buf ? fail(SERQ_EINVAL, "timestamps need a SERQ_DIAG build of the library (tools/ only)") : SERQ_OK;
#endif
}

int serq_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return SERQ_OK;
}

int serq_mx_sizes(int64_t rows, int64_t cols, int64_t* codes_bytes, int64_t* sf_bytes) {
  if (rows < 0 || cols < 0 || cols % 32) return fail(SERQ_EINVAL, "MX layout needs cols %% 32 == 0 (got %lld)", (long long)cols);
  if (codes_bytes) *codes_bytes = rows * cols / 2;
  if (sf_bytes) *sf_bytes = sf_bytes_of(rows, cols);
  return SERQ_OK;
}

static int act_quant_mx_impl(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, uint8_t* codes, uint8_t* sf,
                             const int32_t* gather_idx, int r, uint8_t* xs_codes, uint8_t* xs_sf, serq_stream_t stream) {
  g_launches = 0;
  if (M <= 0 || K <= 0) return fail(SERQ_EINVAL, "x must be non-empty (M=%lld, K=%lld)", (long long)M, (long long)K);
  if (K % 32) return fail(SERQ_EINVAL, "row length %lld not divisible by block_size 32", (long long)K);
  if (ldx < K) return fail(SERQ_EINVAL, "ldx < K");
  if (dtype < 0 || dtype > 2) return fail(SERQ_EINVAL, "unknown dtype %d", dtype);
  if (gather_idx && (r <= 0 || r % 32)) return fail(SERQ_EINVAL, "MX residual path needs rank divisible by block size");
  if (gather_idx && (!xs_codes || !xs_sf)) return fail(SERQ_EINVAL, "gather needs xs_codes and xs_sf");
  if (dtype == SERQ_BF16 && ((reinterpret_cast<uintptr_t>(x) & 15) || (ldx % 8)))
    return fail(SERQ_EINVAL, "bf16 input must be 16-byte aligned with ldx %% 8 == 0");
  if (dtype == SERQ_F32 && ((reinterpret_cast<uintptr_t>(x) & 15) || (ldx % 4)))
    return fail(SERQ_EINVAL, "f32 input must be 16-byte aligned with ldx %% 4 == 0");
  cudaStream_t st = S(stream);
  const int kc = kc_pad_of(K);
  // padded SF rows / chunks must read as a finite scale: the fast kernels write
  // them (grid over the padded extent); the f64 / gather kernels need the memset
  if ((M % 128 || K % 256) && (dtype == SERQ_F64)) CK(cudaMemsetAsync(sf, 0, sf_bytes_of(M, K), st));
  const int krc = gather_idx ? kc_pad_of(r) : 0;
  // the gathered slice's SF padding must read as a finite scale: the fast kernel's z = 1 plane
  // writes it; the f64 kernel needs the memset
  if (gather_idx && dtype == SERQ_F64 && (M % 128 || r % 256)) CK(cudaMemsetAsync(xs_sf, 0, sf_bytes_of(M, r), st));
  if (dtype != SERQ_F64) {
    const int64_t m_rows = (M % 128) ? cdiv(M, 128) * 128 : M;  // cover the SF row padding
    // z = 1 plane: the gathered salient slice (its SF tile padding included), same launch
    const int64_t g_threads = gather_idx ? cdiv(M, 128) * 128 * int64_t(krc) * 16 : 0;
    dim3 grid(unsigned(cdiv(int64_t(kc) * 16, 256)), unsigned(cdiv(m_rows, kMxRows)), gather_idx ? 2u : 1u);
    while (gather_idx && int64_t(grid.x) * grid.y * 256 < g_threads) ++grid.y;  // the z = 1 plane must cover it
    const MxGather mg{gather_idx, r, xs_codes, xs_sf, krc};
    if (dtype == SERQ_BF16 && !SERQ_DBG(g_debug_flags, 1 << 30)) {
      // one thread per 32-block (measured best against 2 and 4 rows per thread, tools/quant_probe.py:
      // 4096^2 8.1 / 8.8 / 10.8 us); debug flag 1<<30: the 8-elements-per-thread kernel (9.9 us)
      const int kR = SERQ_DBG(g_debug_flags, (1 << 21)) ? 4 : SERQ_DBG(g_debug_flags, (1 << 22)) ? 2 : 1;  // diagnostics
      const int64_t main_blocks = cdiv(cdiv(m_rows, kR) * int64_t(kc) * 4, 256);
      const dim3 gb(unsigned(main_blocks + cdiv(g_threads, 256)));  // gather CTAs appended
      const auto* xb = static_cast<const __nv_bfloat16*>(x);
      if (kR == 4)
        CK(launch_pdl(mx_encode_blk_kernel<4>, gb, dim3(256), 0, st, xb, int(M), int(K), ldx, codes, sf, kc, mg));
      else if (kR == 1)
        CK(launch_pdl(mx_encode_blk_kernel<1>, gb, dim3(256), 0, st, xb, int(M), int(K), ldx, codes, sf, kc, mg));
      else
        CK(launch_pdl(mx_encode_blk_kernel<2>, gb, dim3(256), 0, st, xb, int(M), int(K), ldx, codes, sf, kc, mg));
    } else if (dtype == SERQ_BF16) {
      CK(launch_pdl(mx_encode_fast_kernel<__nv_bfloat16>, grid, dim3(256), 0, st, static_cast<const __nv_bfloat16*>(x),
                    int(M), int(K), ldx, codes, sf, kc, mg));
    } else {
      CK(launch_pdl(mx_encode_fast_kernel<float>, grid, dim3(256), 0, st, static_cast<const float*>(x), int(M), int(K),
                    ldx, codes, sf, kc, mg));
    }
    LAUNCH_CHECK("mx_encode_fast");
    return SERQ_OK;
  }
  const int64_t nb_main = cdiv(M * (K / 8), 256);
  const int64_t nb_g = gather_idx ? cdiv(M * (r / 8), 256) : 0;
  const dim3 grid(unsigned(nb_main + nb_g));
  mx_encode_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(x), M, K, ldx, codes, sf, kc, gather_idx,
                                                 r, xs_codes, xs_sf, krc, nb_main);
  LAUNCH_CHECK("mx_encode");
  return SERQ_OK;
}

int serq_act_quant_mx(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, uint8_t* codes, uint8_t* sf,
                      const int32_t* gather_idx, int r, uint8_t* xs_codes, uint8_t* xs_sf, serq_stream_t stream) {
  return act_quant_mx_impl(x, dtype, M, K, ldx, codes, sf, gather_idx, r, xs_codes, xs_sf, stream);
}

static int act_quant_int_impl(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, int bits, int symmetric,
                              int8_t* codes, double* scale64, float* scale32, int32_t* zp, const int32_t* salient_idx,
                              int r, void* xs_out, int xs_kind, float* range, int range_mode, serq_stream_t stream);

int serq_act_quant_int(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, int bits, int symmetric,
                       int8_t* codes, double* scale64, float* scale32, int32_t* zp, const int32_t* salient_idx, int r,
                       void* xs_out, int xs_kind, serq_stream_t stream) {
  return act_quant_int_impl(x, dtype, M, K, ldx, bits, symmetric, codes, scale64, scale32, zp, salient_idx, r, xs_out,
                            xs_kind, nullptr, 0, stream);
}

int serq_act_quant_int_range(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, float* range,
                             serq_stream_t stream) {
  if (!range) return fail(SERQ_EINVAL, "range is NULL");
  return act_quant_int_impl(x, dtype, M, K, ldx, 8, 0, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, 0,
                            range, 1, stream);
}

int serq_act_quant_int_ext(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, int bits, int symmetric,
                           const float* range, int8_t* codes, double* scale64, float* scale32, int32_t* zp,
                           const int32_t* salient_idx, int r, void* xs_out, int xs_kind, serq_stream_t stream) {
  if (!range) return fail(SERQ_EINVAL, "range is NULL");
  return act_quant_int_impl(x, dtype, M, K, ldx, bits, symmetric, codes, scale64, scale32, zp, salient_idx, r, xs_out,
                            xs_kind, const_cast<float*>(range), 2, stream);
}

static int act_quant_int_impl(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, int bits, int symmetric,
                              int8_t* codes, double* scale64, float* scale32, int32_t* zp, const int32_t* salient_idx,
                              int r, void* xs_out, int xs_kind, float* range, int range_mode, serq_stream_t stream) {
  g_launches = 0;
  if (M <= 0 || K <= 0) return fail(SERQ_EINVAL, "x must be non-empty");
  if (bits < 2 || bits > 8) return fail(SERQ_EINVAL, "bits must be in [2, 8], got %d", bits);
  if (ldx < K) return fail(SERQ_EINVAL, "ldx < K");
  if (!symmetric && !zp && range_mode != 1) return fail(SERQ_EINVAL, "asymmetric quantization needs a zero-point buffer");
  if (xs_kind && (r <= 0 || r > K || !xs_out)) return fail(SERQ_EINVAL, "salient slice needs 0 < r <= K and xs_out");
  cudaStream_t st = S(stream);
  const dim3 grid(static_cast<unsigned>(M));
  if (dtype == SERQ_BF16 && K % 8 == 0 && K <= 16384 && ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(codes) & 7) == 0) {
    // one token row per SMALL CTA: the per-row chain (load, min/max reduction, f64 scale,
    // codes) is latency-bound, so many resident rows per SM matter more than wide rows
    // (tools/int_quant_probe.py, C3 2048 x 4096: 12.3 us with 256 threads per row, 5.2 with 64)
    const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
    const bool warp_rows = SERQ_DBG(g_debug_flags, (1 << 21)) != 0;  // diagnostics: one warp per row
    // threads per row by rows per SM: wider rows put more warps in flight when rows are few
    // (tools/probes/intq_grid_probe.py: 512 x 4096 5.95 / 4.84 / 4.37 us with 64 / 128 / 256
    // threads, 2048 x 4096 10.0 / 9.1 / 10.2 us)
    const int64_t rows_per_sm = M / sm_count();
    // (rows above 8192 elements: 256 threads, up to 8 chunks of 8 per thread)
    const int tpr = warp_rows ? 32
                              : (K > 8192 ? 256 : K < 2048 ? 64 : rows_per_sm < 4 ? 256 : rows_per_sm < 16 ? 128 : 64);
    const int cpt = int(cdiv(K / 8, tpr));
    // persistent: at most the resident CTAs, each walking rows with the next row prefetched
#define SERQ_INTQ(P, C)                                                                                              \
  do {                                                                                                               \
    auto kern = int_quant_bf16_kernel<P, C, P>;                                                                      \
    const dim3 gp{unsigned(std::min<int64_t>(M, int64_t(sm_count()) * occupancy_of(kern, P, 0)))};                  \
    CK(launch_pdl(kern, gp, dim3(P), 0, st, xb, int(M), int(K), ldx, bits, symmetric, codes, scale64, scale32, zp,    \
                  salient_idx, r, xs_out, xs_kind, range, range_mode));                                               \
  } while (0)
    if (warp_rows) {
      if (cpt <= 4) SERQ_INTQ(32, 4);
      else if (cpt <= 8) SERQ_INTQ(32, 8);
      else if (cpt <= 16) SERQ_INTQ(32, 16);
      else SERQ_INTQ(32, 32);
    } else if (tpr == 256) {
      if (cpt <= 2) SERQ_INTQ(256, 2);
      else if (cpt <= 4) SERQ_INTQ(256, 4);
      else SERQ_INTQ(256, 8);
    } else if (tpr == 128) {
      if (cpt <= 2) SERQ_INTQ(128, 2);
      else if (cpt <= 4) SERQ_INTQ(128, 4);
      else SERQ_INTQ(128, 8);
    } else {
      if (cpt <= 2) SERQ_INTQ(64, 2);
      else if (cpt <= 4) SERQ_INTQ(64, 4);
      else if (cpt <= 8) SERQ_INTQ(64, 8);
      else SERQ_INTQ(64, 16);
    }
#undef SERQ_INTQ
    LAUNCH_CHECK("int_quant_bf16");
    return SERQ_OK;
  }
  if (range_mode)
    return fail(SERQ_EINVAL, "K-sharded per-token ranges need bf16 rows (16-B aligned, K %% 8 == 0, K <= 16384)");
  switch (dtype) {
    case SERQ_BF16:
      int_quant_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), M, K, ldx, bits,
                                                            symmetric, codes, scale64, scale32, zp, salient_idx, r,
                                                            xs_out, xs_kind);
      break;
    case SERQ_F32:
      int_quant_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), M, K, ldx, bits, symmetric, codes,
                                                    scale64, scale32, zp, salient_idx, r, xs_out, xs_kind);
      break;
    case SERQ_F64:
      int_quant_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(x), M, K, ldx, bits, symmetric, codes,
                                                     scale64, scale32, zp, salient_idx, r, xs_out, xs_kind);
      break;
    default:
      return fail(SERQ_EINVAL, "unknown dtype %d", dtype);
  }
  LAUNCH_CHECK("int_quant");
  return SERQ_OK;
}

int serq_pack_mx(const uint8_t* codes, const int32_t* exps, int64_t N, int64_t K, const uint8_t* r_codes,
                 const int32_t* r_exps, int r, int salient_contiguous, serq_linear_t** out, serq_stream_t stream) {
  g_launches = 0;
  if (!out) return fail(SERQ_EINVAL, "out is NULL");
  *out = nullptr;
  if (N <= 0 || K <= 0 || K % 32) return fail(SERQ_EINVAL, "MX weight needs K %% 32 == 0 (N=%lld, K=%lld)", (long long)N, (long long)K);
  if (N % 8) return fail(SERQ_EINVAL, "output dim N must be a multiple of 8 (bf16 row pitch), got %lld", (long long)N);
  if (r < 0 || r % 32) return fail(SERQ_EINVAL, "MX residual path needs rank divisible by block size");
  if (r > 0 && (!r_codes || !r_exps)) return fail(SERQ_EINVAL, "rank > 0 needs r_codes and r_exps");
  if (r > K) return fail(SERQ_EINVAL, "rank %d exceeds K", r);
  cudaStream_t st = S(stream);
  serq_linear* h = new serq_linear();
  h->mode = kModeMX;
  h->N = N;
  h->K = K;
  h->r = r;
  h->contiguous = salient_contiguous ? 1 : 0;
  auto bail = [&](int code) {
    free_handle(h);
    return code;
  };
  // weights pre-tiled [N/128][ksteps][128 rows x 128 B] (zero padded): each TMA box is one contiguous 16 KB
  h->w_ksteps = int(cdiv(K / 2, kStepBytes));
  const int64_t w_bytes = cdiv(N, 128) * h->w_ksteps * 128 * 128;
  if (cudaMalloc(&h->w, w_bytes) != cudaSuccess || cudaMalloc(&h->sfw, sf_bytes_of(N, K)) != cudaSuccess)
    return bail(fail(SERQ_ECUDA, "cudaMalloc failed for MX weights"));
  if (cudaMemsetAsync(h->sfw, 0, sf_bytes_of(N, K), st) != cudaSuccess) return bail(fail(SERQ_ECUDA, "memset"));
  if ((N % 128 || (K / 2) % kStepBytes) && cudaMemsetAsync(h->w, 0, w_bytes, st) != cudaSuccess)
    return bail(fail(SERQ_ECUDA, "memset"));
  pack_mx_kernel<<<unsigned(cdiv(N * K / 8, 256)), 256, 0, st>>>(codes, exps, N, K, static_cast<uint8_t*>(h->w), h->sfw,
                                                                  kc_pad_of(K), h->w_ksteps);
  if (cudaGetLastError() != cudaSuccess) return bail(fail(SERQ_ECUDA, "pack_mx launch failed"));
  int rc = make_map(&h->map_b128, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->w, 128, uint64_t(w_bytes / 128), 128, 128, 128);
  if (!rc) rc = make_map(&h->map_b64, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->w, 128, uint64_t(w_bytes / 128), 128, 128, 64);
  h->map_b = h->map_b128;
  if (!rc) rc = make_sf_map(&h->map_sfw, h->sfw, N, K);
  if (rc) return bail(rc);
  h->map_r128 = h->map_b128;
  h->map_sfr = h->map_sfw;
  if (r > 0) {
    if (cudaMalloc(&h->rbuf, N * r / 2) != cudaSuccess || cudaMalloc(&h->sfr, sf_bytes_of(N, r)) != cudaSuccess)
      return bail(fail(SERQ_ECUDA, "cudaMalloc failed for R"));
    if (cudaMemsetAsync(h->sfr, 0, sf_bytes_of(N, r), st) != cudaSuccess) return bail(fail(SERQ_ECUDA, "memset"));
    pack_mx_kernel<<<unsigned(cdiv(N * r / 8, 256)), 256, 0, st>>>(r_codes, r_exps, N, r,
                                                                    static_cast<uint8_t*>(h->rbuf), h->sfr, kc_pad_of(r), 0);
    if (cudaGetLastError() != cudaSuccess) return bail(fail(SERQ_ECUDA, "pack_mx launch failed"));
    rc = make_map(&h->map_r, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->rbuf, r / 2, N, r / 2, 128, kBN);
    if (!rc) rc = make_map(&h->map_r128, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->rbuf, r / 2, N, r / 2, 128, 128);
    if (!rc) rc = make_sf_map(&h->map_sfr, h->sfr, N, r);
    if (rc) return bail(rc);
    if (r == 64) {  // 32-B R rows: the pair3 kernel (contiguous) and the decode kernel (both layouts)
      rc = make_map(&h->map_r32, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->rbuf, r / 2, N, r / 2, 32, 128,
                    CU_TENSOR_MAP_SWIZZLE_32B);
      if (!rc)
        rc = make_map(&h->map_sfr4, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->sfr, 128, uint64_t(sf_bytes_of(N, r) / 128),
                      128, 128, 4, CU_TENSOR_MAP_SWIZZLE_NONE);
      if (rc) return bail(rc);
      h->has_r32 = true;
      h->map_rdec = h->map_r32;
      h->dec_rw = 32;
    } else if (r <= 128) {
      // decode kernel: R zero-padded to 64 (32-B rows) or 128 columns (64-B rows, two K = 64 MMAs);
      // padded codes are 0, so the padded columns contribute nothing whatever X holds there
      const int rp = r <= 64 ? 64 : 128;
      if (cudaMalloc(&h->rdec, N * rp / 2) != cudaSuccess) return bail(fail(SERQ_ECUDA, "cudaMalloc R (decode)"));
      if (cudaMemsetAsync(h->rdec, 0, N * rp / 2, st) != cudaSuccess ||
          cudaMemcpy2DAsync(h->rdec, rp / 2, h->rbuf, r / 2, r / 2, N, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return bail(fail(SERQ_ECUDA, "R (decode) copy"));
      rc = make_map(&h->map_rdec, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->rdec, rp / 2, N, rp / 2, rp / 2, 128,
                    rp == 64 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B);
      if (!rc)
        rc = make_map(&h->map_sfr4, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->sfr, 128, uint64_t(sf_bytes_of(N, r) / 128),
                      128, 128, 4, CU_TENSOR_MAP_SWIZZLE_NONE);
      if (rc) return bail(rc);
      h->dec_rw = rp / 2;
    }
  }
  *out = h;
  return SERQ_OK;
}

int serq_linear_set_segments(serq_linear_t* h, int nseg, const int64_t* seg_rows) {
  if (!h || h->mode != kModeMX || h->parent) return fail(SERQ_EINVAL, "segments need an owning MX handle");
  if (nseg < 1 || nseg > kMaxSeg || !seg_rows) return fail(SERQ_EINVAL, "1 <= nseg <= %d", kMaxSeg);
  if (nseg > 1 && (h->r <= 0 || h->r > 128 || h->contiguous))
    return fail(SERQ_EINVAL, "fused segments need per-segment (gathered) salient sets with 0 < r <= 128");
  int64_t sum = 0;
  for (int j = 0; j < nseg; ++j) {
    if (seg_rows[j] <= 0 || seg_rows[j] % 128) return fail(SERQ_EINVAL, "segment rows must be positive multiples of 128");
    sum += seg_rows[j];
  }
  if (sum != h->N) return fail(SERQ_EINVAL, "segment rows must sum to N = %lld", (long long)h->N);
  h->nseg = nseg;
  for (int j = 0, acc = 0; j + 1 < nseg; ++j) {
    acc += int(seg_rows[j]);
    h->seg_row[j] = acc;
  }
  return SERQ_OK;
}

int serq_linear_view(const serq_linear_t* parent, int64_t row0, int64_t rows, int salient_contiguous,
                     serq_linear_t** out) {
  if (!out) return fail(SERQ_EINVAL, "out is NULL");
  *out = nullptr;
  if (!parent || parent->mode != kModeMX) return fail(SERQ_EINVAL, "views are of MX handles");
  const serq_linear* root = parent->parent ? parent->parent : parent;
  if (row0 < 0 || rows <= 0 || row0 % 128 || row0 + rows > parent->N || (rows % 128 && row0 + rows != parent->N))
    return fail(SERQ_EINVAL, "a view is a 128-row-aligned row range of the parent");
  serq_linear* v = new serq_linear();
  v->parent = root;
  v->mode = kModeMX;
  v->N = rows;
  v->K = parent->K;
  v->r = parent->r;
  v->r_mode = parent->r_mode;
  v->contiguous = salient_contiguous ? 1 : 0;
  v->w_ksteps = parent->w_ksteps;
  const int64_t blk = row0 / 128, r = parent->r;
  v->w = static_cast<uint8_t*>(parent->w) + blk * parent->w_ksteps * 128 * 128;
  v->sfw = parent->sfw + blk * kc_pad_of(parent->K) * 512;
  const int64_t w_bytes = cdiv(rows, 128) * v->w_ksteps * 128 * 128;
  int rc = make_map(&v->map_b128, CU_TENSOR_MAP_DATA_TYPE_UINT8, v->w, 128, uint64_t(w_bytes / 128), 128, 128, 128);
  if (!rc) rc = make_map(&v->map_b64, CU_TENSOR_MAP_DATA_TYPE_UINT8, v->w, 128, uint64_t(w_bytes / 128), 128, 128, 64);
  if (!rc) rc = make_sf_map(&v->map_sfw, v->sfw, rows, v->K);
  v->map_b = v->map_b128;
  v->map_r128 = v->map_b128;
  v->map_sfr = v->map_sfw;
  if (!rc && r > 0) {
    v->rbuf = static_cast<uint8_t*>(parent->rbuf) + row0 * r / 2;
    v->sfr = parent->sfr + blk * kc_pad_of(r) * 512;
    rc = make_map(&v->map_r, CU_TENSOR_MAP_DATA_TYPE_UINT8, v->rbuf, r / 2, rows, r / 2, 128, kBN);
    if (!rc) rc = make_map(&v->map_r128, CU_TENSOR_MAP_DATA_TYPE_UINT8, v->rbuf, r / 2, rows, r / 2, 128, 128);
    if (!rc) rc = make_sf_map(&v->map_sfr, v->sfr, rows, r);
    if (!rc && r <= 128)
      rc = make_map(&v->map_sfr4, CU_TENSOR_MAP_DATA_TYPE_UINT8, v->sfr, 128, uint64_t(sf_bytes_of(rows, r) / 128), 128,
                    128, 4, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc && r == 64) {
      rc = make_map(&v->map_r32, CU_TENSOR_MAP_DATA_TYPE_UINT8, v->rbuf, r / 2, rows, r / 2, 32, 128,
                    CU_TENSOR_MAP_SWIZZLE_32B);
      v->has_r32 = true;
      v->map_rdec = v->map_r32;
      v->dec_rw = 32;
    } else if (!rc && r <= 128) {
      const int64_t rp = r <= 64 ? 64 : 128;
      v->rdec = static_cast<uint8_t*>(parent->rdec) + row0 * rp / 2;
      rc = make_map(&v->map_rdec, CU_TENSOR_MAP_DATA_TYPE_UINT8, v->rdec, rp / 2, rows, rp / 2, rp / 2, 128,
                    rp == 64 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B);
      v->dec_rw = int(rp / 2);
    }
  }
  if (rc) {
    delete v;
    return rc;
  }
  *out = v;
  return SERQ_OK;
}

int serq_unpack_mx(const uint8_t* codes_packed, const uint8_t* sf, int64_t rows, int64_t cols, uint8_t* codes,
                   int32_t* exps, serq_stream_t stream) {
  g_launches = 0;
  if (rows <= 0 || cols <= 0 || cols % 32) return fail(SERQ_EINVAL, "MX layout needs cols %% 32 == 0");
  unpack_mx_kernel<<<unsigned(cdiv(rows * cols / 8, 256)), 256, 0, S(stream)>>>(codes_packed, sf, rows, cols,
                                                                                kc_pad_of(cols), codes, exps);
  LAUNCH_CHECK("unpack_mx");
  return SERQ_OK;
}

int serq_mx_decode_bf16(const uint8_t* codes_packed, const uint8_t* sf, int64_t rows, int64_t cols, void* out,
                        serq_stream_t stream) {
  g_launches = 0;
  if (rows <= 0 || cols <= 0 || cols % 32) return fail(SERQ_EINVAL, "MX layout needs cols %% 32 == 0");
  if (!codes_packed || !sf || !out) return fail(SERQ_EINVAL, "NULL buffer");
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(SERQ_EINVAL, "out must be 16-byte aligned");
  mx_decode_bf16_kernel<<<dim3(unsigned(cdiv(cols / 8, 256)), unsigned(rows < 65535 ? rows : 65535)), 256, 0,
                          S(stream)>>>(
      codes_packed, sf, rows, cols, kc_pad_of(cols), static_cast<__nv_bfloat16*>(out));
  LAUNCH_CHECK("mx_decode_bf16");
  return SERQ_OK;
}

int serq_rmsnorm_quant_mx(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, const double* gain,
                          const float* gain32, double eps, uint8_t* codes, uint8_t* sf, serq_stream_t stream) {
  return serq_rmsnorm_quant_mx_gather(x, dtype, M, K, ldx, gain, gain32, eps, nullptr, 0, codes, sf, nullptr, nullptr,
                                      stream);
}

int serq_rmsnorm_quant_mx_gather(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, const double* gain,
                                 const float* gain32, double eps, const int32_t* gather_idx, int r, uint8_t* codes,
                                 uint8_t* sf, uint8_t* xs_codes, uint8_t* xs_sf, serq_stream_t stream) {
  g_launches = 0;
  if (M <= 0 || K <= 0) return fail(SERQ_EINVAL, "x must be non-empty (M=%lld, K=%lld)", (long long)M, (long long)K);
  if (K % 32) return fail(SERQ_EINVAL, "row length %lld not divisible by block_size 32", (long long)K);
  if (ldx < K) return fail(SERQ_EINVAL, "ldx < K");
  if (!gain || !gain32) return fail(SERQ_EINVAL, "gain is NULL");
  if (reinterpret_cast<uintptr_t>(gain32) & 15) return fail(SERQ_EINVAL, "gain32 must be 16-byte aligned");
  if (!(eps >= 0.0)) return fail(SERQ_EINVAL, "eps must be >= 0");
  if (dtype != SERQ_BF16 && dtype != SERQ_F32) return fail(SERQ_EINVAL, "rmsnorm input must be bf16 or f32");
  const int align = dtype == SERQ_BF16 ? 8 : 4;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || ldx % align) return fail(SERQ_EINVAL, "x must be 16-byte aligned rows");
  cudaStream_t st = S(stream);
  const int kc = kc_pad_of(K);
  // rows / chunks beyond the matrix must read as a finite scale
  if (M % 128 || K % 256) CK(cudaMemsetAsync(sf, 0, sf_bytes_of(M, K), st));
  if (K > 4 * 2048) return fail(SERQ_EINVAL, "fused RMSNorm quantizer supports rows up to 8192 elements");
  if (gather_idx && (r <= 0 || r % 32 || r > 1024 || r > K || !xs_codes || !xs_sf))
    return fail(SERQ_EINVAL, "gather needs 0 < r <= min(K, 1024), r %% 32 == 0 and the xs buffers");
  const int kcr = gather_idx ? kc_pad_of(r) : 0;
  // the gathered slice's scale-factor padding (rows to the 128-row block, chunks to kc_pad_r)
  if (gather_idx && (M % 128 || r % 256)) CK(cudaMemsetAsync(xs_sf, 0, sf_bytes_of(M, r), st));
  const MxGather mg{gather_idx, r, xs_codes, xs_sf, kcr};

  // kTpr threads per row (8 elements each per chunk), 256 / kTpr rows per CTA
  // threads per row: 128 for K <= 4096, 256 above (measured best of 64 / 128 / 256 at 4096^2 and 8192^2)
  const int tpr = K <= 4096 ? 128 : 256;
  const int chunks = int(cdiv(K, tpr * 8));  // <= 4
  const dim3 grid{unsigned(cdiv(M, 256 / tpr))}, blk{256};
#define RMS_LAUNCH(T, P, C)                                                                                       \
  CK(launch_pdl(rmsnorm_mx_encode_kernel<T, P, C>, grid, blk, 0, st, static_cast<const T*>(x), int(M), int(K), ldx, \
                gain, gain32, eps, codes, sf, kc, mg))
  if (dtype == SERQ_BF16) {
    if (tpr == 128) {
      if (chunks <= 2) RMS_LAUNCH(__nv_bfloat16, 128, 2);
      else RMS_LAUNCH(__nv_bfloat16, 128, 4);
    } else {
      if (chunks <= 2) RMS_LAUNCH(__nv_bfloat16, 256, 2);
      else RMS_LAUNCH(__nv_bfloat16, 256, 4);
    }
  } else {
    if (tpr == 128) {
      if (chunks <= 2) RMS_LAUNCH(float, 128, 2);
      else RMS_LAUNCH(float, 128, 4);
    } else {
      if (chunks <= 2) RMS_LAUNCH(float, 256, 2);
      else RMS_LAUNCH(float, 256, 4);
    }
  }
#undef RMS_LAUNCH
  LAUNCH_CHECK("rmsnorm_mx_encode");
  return SERQ_OK;
}

// NumPy's pairwise summation tree for K elements (numpy pairwise_sum: leaves of <= 128, split
// at n/2 rounded down to a multiple of 8): leaves left to right, internal nodes ordered by height
struct PwBuild {
  int nleaf = 0, nnode = 0;
  int16_t start[64], len[64];
  int ca[64], cb[64], height[64];
};

// returns the value id of the subtree over [off, off + n): a leaf index, or 64 + node index
static int pw_rec(int64_t off, int64_t n, PwBuild& b, int& h) {
  if (n <= 128) {
    if (b.nleaf >= 64) return -1;
    b.start[b.nleaf] = int16_t(off);
    b.len[b.nleaf] = int16_t(n);
    h = 0;
    return b.nleaf++;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  int hl = 0, hr = 0;
  const int l = pw_rec(off, n2, b, hl);
  const int r = l < 0 ? -1 : pw_rec(off + n2, n - n2, b, hr);
  if (r < 0 || b.nnode >= 63) return -1;
  const int j = b.nnode++;
  b.ca[j] = l;
  b.cb[j] = r;
  h = std::max(hl, hr) + 1;
  b.height[j] = h;
  return 64 + j;
}

static bool rms_tree(int64_t K, RmsPairwise& t) {
  PwBuild b;
  int h = 0;
  if (pw_rec(0, K, b, h) < 0 || h > 8) return false;
  t = RmsPairwise{};
  t.nleaf = b.nleaf;
  t.nnode = b.nnode;
  t.nlevel = h;
  t.perfect = b.nleaf == (1 << h) && b.nleaf <= 64;  // all 2^h leaves at depth h
  for (int i = 0; i < b.nleaf; ++i) {
    t.start[i] = b.start[i];
    t.len[i] = b.len[i];
  }
  int slot[64], n = 0;
  for (int hh = 1; hh <= h; ++hh) {
    for (int j = 0; j < b.nnode; ++j)
      if (b.height[j] == hh) slot[j] = n++;
    t.level_end[hh - 1] = uint8_t(n);
  }
  auto vid = [&](int id) { return uint8_t(id < 64 ? id : b.nleaf + slot[id - 64]); };
  for (int j = 0; j < b.nnode; ++j) {
    t.a[slot[j]] = vid(b.ca[j]);
    t.b[slot[j]] = vid(b.cb[j]);
  }
  return true;
}

int serq_rmsnorm_quant_int(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, const double* gain,
                           const float* gain32, double eps, int bits, int symmetric, int8_t* codes, double* scale64,
                           float* scale32, int32_t* zp, const int32_t* salient_idx, int r, void* xs_out, int xs_kind,
                           serq_stream_t stream) {
  g_launches = 0;
  if (M <= 0 || K <= 0) return fail(SERQ_EINVAL, "x must be non-empty (M=%lld, K=%lld)", (long long)M, (long long)K);
  if (K > 8192) return fail(SERQ_EINVAL, "fused RMSNorm quantizer supports rows up to 8192 elements");
  if (ldx < K) return fail(SERQ_EINVAL, "ldx < K");
  if (!gain) return fail(SERQ_EINVAL, "gain is NULL");
  if (!(eps >= 0.0)) return fail(SERQ_EINVAL, "eps must be >= 0");
  if (bits < 2 || bits > 8) return fail(SERQ_EINVAL, "bits must be in [2, 8], got %d", bits);
  if (!symmetric && !zp) return fail(SERQ_EINVAL, "asymmetric quantization needs a zero-point buffer");
  if (xs_kind && (r <= 0 || r > K || !xs_out)) return fail(SERQ_EINVAL, "salient slice needs 0 < r <= K and xs_out");
  if (dtype != SERQ_BF16 && dtype != SERQ_F32) return fail(SERQ_EINVAL, "rmsnorm input must be bf16 or f32");
  RmsPairwise tree{};
  if (!rms_tree(K, tree)) return fail(SERQ_EINVAL, "pairwise tree too large");
  cudaStream_t st = S(stream);
  const int64_t esz = dtype == SERQ_BF16 ? 2 : 4;
  const bool fast = gain32 && !(reinterpret_cast<uintptr_t>(gain32) & 15) && K % 8 == 0 &&
                    !(reinterpret_cast<uintptr_t>(x) & 15) && (ldx * esz) % 16 == 0 && !(reinterpret_cast<uintptr_t>(codes) & 7);
  if (fast) {
    // threads per row and 8-element chunks per thread (K <= kTpr * kChunks * 8): one row per
    // CTA above 1024 elements (small per-thread state, more CTAs resident per SM)
    const int tpr = K <= 1024 ? 128 : 256;
    const int chunks = K <= 2048 ? 1 : K <= 4096 ? 2 : 4;
    const dim3 grid{unsigned(cdiv(M, 256 / tpr))}, blk{256};
#define RMSI_LAUNCH(T, P, C)                                                                                           \
  CK(launch_pdl(rmsnorm_int_quant_fast_kernel<T, P, C>, grid, blk, 0, st, static_cast<const T*>(x), int(M), int(K), ldx, \
                gain, gain32, eps, tree, bits, symmetric, codes, scale64, scale32, zp, salient_idx, r, xs_out, xs_kind))
    if (dtype == SERQ_BF16) {
      if (tpr == 128) RMSI_LAUNCH(__nv_bfloat16, 128, 1);
      else if (chunks == 1) RMSI_LAUNCH(__nv_bfloat16, 256, 1);
      else if (chunks == 2) RMSI_LAUNCH(__nv_bfloat16, 256, 2);
      else RMSI_LAUNCH(__nv_bfloat16, 256, 4);
    } else {
      if (tpr == 128) RMSI_LAUNCH(float, 128, 1);
      else if (chunks == 1) RMSI_LAUNCH(float, 256, 1);
      else if (chunks == 2) RMSI_LAUNCH(float, 256, 2);
      else RMSI_LAUNCH(float, 256, 4);
    }
#undef RMSI_LAUNCH
    LAUNCH_CHECK("rmsnorm_int_quant_fast_kernel");
    return SERQ_OK;
  }
  // any other layout (K % 8 != 0, unaligned rows, no f32 gain): the all-f64 kernel
  const dim3 grid{unsigned(M)}, blk{256};
  if (dtype == SERQ_BF16)
    CK(launch_pdl(rmsnorm_int_quant_kernel<__nv_bfloat16>, grid, blk, 0, st, static_cast<const __nv_bfloat16*>(x), M, K,
                  ldx, gain, eps, tree, bits, symmetric, codes, scale64, scale32, zp, salient_idx, r, xs_out, xs_kind));
  else
    CK(launch_pdl(rmsnorm_int_quant_kernel<float>, grid, blk, 0, st, static_cast<const float*>(x), M, K, ldx, gain, eps,
                  tree, bits, symmetric, codes, scale64, scale32, zp, salient_idx, r, xs_out, xs_kind));
  LAUNCH_CHECK("rmsnorm_int_quant_kernel");
  return SERQ_OK;
}

// ---------------------------------------------------------------- block glue (M <= 16)
int serq_block_add_rmsnorm(const float* x, const void* o, int64_t ldo, int64_t M, int64_t H, const float* gain,
                           float eps, float* res, float* h, serq_stream_t stream) {
  g_launches = 0;
  if (M <= 0 || H <= 0 || !x) return fail(SERQ_EINVAL, "add_rmsnorm needs x and M, H > 0");
  if (h ? !gain : !res) return fail(SERQ_EINVAL, "add_rmsnorm needs gain with h, or res without h");
  if (o && ldo < H) return fail(SERQ_EINVAL, "ldo < H");
  const auto al = [](const void* ptr, int a) { return (reinterpret_cast<uintptr_t>(ptr) & (a - 1)) == 0; };
  const bool regs = H % 4 == 0 && H <= 8192 && al(x, 16) && (!h || (al(gain, 16) && al(h, 16))) && (!res || al(res, 16)) &&
                    (!o || (al(o, 8) && ldo % 4 == 0));
  const __nv_bfloat16* ob = static_cast<const __nv_bfloat16*>(o);
  if (regs && H <= 4096) {
    CK(launch_pdl(block_add_rmsnorm_reg_kernel<1>, dim3(unsigned(M)), dim3(1024), 0, S(stream), x, ob, ldo, int(M),
                  int(H), gain, eps, res, h));
    LAUNCH_CHECK("block_add_rmsnorm_reg_kernel");
  } else if (regs) {
    CK(launch_pdl(block_add_rmsnorm_reg_kernel<2>, dim3(unsigned(M)), dim3(1024), 0, S(stream), x, ob, ldo, int(M),
                  int(H), gain, eps, res, h));
    LAUNCH_CHECK("block_add_rmsnorm_reg_kernel");
  } else {
    CK(launch_pdl(block_add_rmsnorm_kernel, dim3(unsigned(M)), dim3(256), 0, S(stream), x, ob, ldo, int(M), int(H),
                  gain, eps, res, h));
    LAUNCH_CHECK("block_add_rmsnorm_kernel");
  }
  return SERQ_OK;
}

int serq_block_silu_mul(const void* gate, int64_t ldg, const void* up, int64_t ldu, int64_t M, int64_t F, float* mid,
                        serq_stream_t stream) {
  g_launches = 0;
  if (M <= 0 || F <= 0 || !gate || !up || !mid || ldg < F || ldu < F) return fail(SERQ_EINVAL, "silu_mul arguments");
  CK(launch_pdl(block_silu_mul_kernel, dim3(unsigned(cdiv(M * F, 256))), dim3(256), 0, S(stream),
                static_cast<const __nv_bfloat16*>(gate), ldg, static_cast<const __nv_bfloat16*>(up), ldu, int(M),
                int(F), mid));
  LAUNCH_CHECK("block_silu_mul_kernel");
  return SERQ_OK;
}

int serq_block_attention(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, int64_t M,
                         int64_t heads, int64_t head_dim, float scale, float* out, int64_t ldo, serq_stream_t stream) {
  g_launches = 0;
  if (M <= 0 || M > 16) return fail(SERQ_EINVAL, "the small-batch attention takes 1..16 tokens, got %lld", (long long)M);
  if (head_dim != 128 || heads <= 0) return fail(SERQ_EINVAL, "the small-batch attention needs head_dim 128");
  if (!q || !k || !v || !out) return fail(SERQ_EINVAL, "attention pointers");
  CK(launch_pdl(block_attention_small_kernel<16>, dim3(unsigned(heads), unsigned(M)), dim3(128), 0, S(stream),
                static_cast<const __nv_bfloat16*>(q), ldq, static_cast<const __nv_bfloat16*>(k), ldk,
                static_cast<const __nv_bfloat16*>(v), ldv, int(M), int(head_dim), scale, out, ldo));
  LAUNCH_CHECK("block_attention_small_kernel");
  return SERQ_OK;
}

int serq_mx_container_decode(const uint8_t* body, int64_t rows, int64_t cols, uint8_t* codes, int32_t* exps,
                             serq_stream_t stream) {
  g_launches = 0;
  if (rows <= 0 || cols <= 0 || cols % 32)
    return fail(SERQ_EINVAL, "MX container for the device needs 32-element blocks and cols %% 32 == 0");
  if (!body || !codes || !exps) return fail(SERQ_EINVAL, "null pointer");
  if (reinterpret_cast<uintptr_t>(codes) & 15) return fail(SERQ_EINVAL, "codes must be 16-byte aligned");
  const int64_t records = rows * (cols / 32);
  mx_container_decode_kernel<<<unsigned(cdiv(records, 256)), 256, 0, S(stream)>>>(body, records, codes, exps);
  LAUNCH_CHECK("mx_container_decode");
  return SERQ_OK;
}

static int pack_int_impl(const int32_t* codes, const double* scales, int64_t K, int64_t N, int w_bits, int r_mode,
                         const void* r_data, const double* r_scales, int r, int salient_contiguous, bool allow_w4,
                         serq_linear_t** out, serq_stream_t stream);

int serq_pack_int(const int32_t* codes, const double* scales, int64_t K, int64_t N, int w_bits, int r_mode,
                  const void* r_data, const double* r_scales, int r, int salient_contiguous, serq_linear_t** out,
                  serq_stream_t stream) {
  return pack_int_impl(codes, scales, K, N, w_bits, r_mode, r_data, r_scales, r, salient_contiguous, false, out,
                       stream);
}

int serq_pack_int4(const int32_t* codes, const double* scales, int64_t K, int64_t N, int w_bits, int r_mode,
                   const void* r_data, const double* r_scales, int r, int salient_contiguous, serq_linear_t** out,
                   serq_stream_t stream) {
  if (w_bits > 4) return fail(SERQ_EINVAL, "packed INT4 weights need w_bits <= 4 (got %d)", w_bits);
  const int rr = r_mode == SERQ_R_NONE ? 0 : r;
  if ((r_mode == SERQ_R_INT && !salient_contiguous) || rr > 128 || (r_mode == SERQ_R_DENSE && cdiv(K, 128) < cdiv(rr, 64)))
    return fail(SERQ_EINVAL,
                "packed INT4 weights are served by the CTA-pair kernel: R permuted-integer (r <= 128), dense "
                "(r <= 128, K >= 128 ceil(r / 64)) or none");
  return pack_int_impl(codes, scales, K, N, w_bits, r_mode, r_data, r_scales, r, salient_contiguous, true, out, stream);
}

static int pack_int_impl(const int32_t* codes, const double* scales, int64_t K, int64_t N, int w_bits, int r_mode,
                         const void* r_data, const double* r_scales, int r, int salient_contiguous, bool allow_w4,
                         serq_linear_t** out, serq_stream_t stream) {
  g_launches = 0;
  if (!out) return fail(SERQ_EINVAL, "out is NULL");
  *out = nullptr;
  if (N <= 0 || K <= 0) return fail(SERQ_EINVAL, "empty weight");
  if (K % 16) return fail(SERQ_EINVAL, "K must be a multiple of 16 (int8 row pitch), got %lld", (long long)K);
  if (N % 8) return fail(SERQ_EINVAL, "output dim N must be a multiple of 8, got %lld", (long long)N);
  if (w_bits < 2 || w_bits > 8) return fail(SERQ_EINVAL, "weight bits must be in [2, 8]");
  if (r_mode < SERQ_R_NONE || r_mode > SERQ_R_INT) return fail(SERQ_EINVAL, "unknown r_mode %d", r_mode);
  if (r_mode != SERQ_R_NONE && (r <= 0 || r > K || !r_data)) return fail(SERQ_EINVAL, "R needs 0 < r <= K and data");
  if (r_mode == SERQ_R_INT && !r_scales) return fail(SERQ_EINVAL, "integer R needs r_scales");
  if (r_mode == SERQ_R_DENSE && r % 8) return fail(SERQ_EINVAL, "dense R needs r %% 8 == 0 (bf16 row pitch)");
  if (r_mode == SERQ_R_INT && r % 16) return fail(SERQ_EINVAL, "integer R needs r %% 16 == 0 (int8 row pitch)");
  cudaStream_t st = S(stream);
  serq_linear* h = new serq_linear();
  h->mode = kModeI8;
  h->N = N;
  h->K = K;
  h->w_bits = w_bits;
  h->r = r_mode == SERQ_R_NONE ? 0 : r;
  h->r_mode = r_mode;
  h->contiguous = salient_contiguous ? 1 : 0;
  auto bail = [&](int code) {
    free_handle(h);
    return code;
  };
  if (cudaMalloc(&h->sw, N * 4) != cudaSuccess || cudaMalloc(&h->colsum, N * 4) != cudaSuccess)
    return bail(fail(SERQ_ECUDA, "cudaMalloc failed for INT weight scales"));
  colsum_kernel<<<unsigned(cdiv(N, 256)), 256, 0, st>>>(codes, K, N, scales, h->colsum, h->sw);
  // weights in HBM: packed INT4 (0.5 B / weight, serq_pack_int4: the CTA-pair kernel widens them
  // in the SM) or int8 [N, K] (serq_pack_int, the faster feed today: TMA straight into the
  // operand).  Never both copies.
  // dense R of r > 64 takes ceil(r / 64) side tiles, staged with distinct K-steps (needs K >= 128 nr)
  const bool pair_cfg = (r_mode != SERQ_R_INT || salient_contiguous) && h->r <= 128 &&
                        (r_mode != SERQ_R_DENSE || cdiv(K, 128) >= cdiv(h->r, 64));
  h->has_w4 = allow_w4 && w_bits <= 4 && pair_cfg;
  int rc = SERQ_OK;
  if (h->has_w4) {
    const int ksteps = int(cdiv(K, 128));
    const int64_t bytes = cdiv(N, 128) * ksteps * 128 * 64;
    if (cudaMalloc(&h->w, bytes) != cudaSuccess) return bail(fail(SERQ_ECUDA, "cudaMalloc failed for INT4 weights"));
    if (cudaMemsetAsync(h->w, 0, bytes, st) != cudaSuccess) return bail(fail(SERQ_ECUDA, "memset"));
    pack_int4_tiled_kernel<<<dim3(unsigned(cdiv(N, 256)), unsigned(ksteps * 64)), 256, 0, st>>>(
        codes, K, N, ksteps, static_cast<uint8_t*>(h->w));
    if (cudaGetLastError() != cudaSuccess) return bail(fail(SERQ_ECUDA, "pack_int4 launch failed"));
    h->w_bytes = bytes;
  } else {
    if (cudaMalloc(&h->w, N * K) != cudaSuccess) return bail(fail(SERQ_ECUDA, "cudaMalloc failed for INT weights"));
    transpose_codes_kernel<<<dim3(unsigned(cdiv(N, 32)), unsigned(cdiv(K, 32))), dim3(32, 8), 0, st>>>(
        codes, K, N, static_cast<int8_t*>(h->w));
    if (cudaGetLastError() != cudaSuccess) return bail(fail(SERQ_ECUDA, "pack_int launch failed"));
    rc = make_map(&h->map_b, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->w, K, N, K, 128, kBN);
    if (!rc) rc = make_map(&h->map_w8, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->w, K, N, K, 128, 128);
    if (!rc) rc = make_map(&h->map_w8_64, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->w, K, N, K, 128, 64);
    if (rc) return bail(rc);
    h->w_bytes = N * K;
  }
  if (r_mode == SERQ_R_DENSE) {
    if (cudaMalloc(&h->rbuf, N * r * 2) != cudaSuccess) return bail(fail(SERQ_ECUDA, "cudaMalloc R"));
    dense_r_kernel<<<unsigned(cdiv(N * r, 256)), 256, 0, st>>>(static_cast<const double*>(r_data), r, N,
                                                               static_cast<__nv_bfloat16*>(h->rbuf));
    if (cudaGetLastError() != cudaSuccess) return bail(fail(SERQ_ECUDA, "dense_r launch failed"));
    rc = make_map(&h->map_r, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, h->rbuf, r, N, r * 2, 64, kBN);
    if (!rc) rc = make_map(&h->map_r_pair, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, h->rbuf, r, N, r * 2, 64, 128);
    if (!rc) rc = make_map(&h->map_r_pair64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, h->rbuf, r, N, r * 2, 64, 64);
    if (rc) return bail(rc);
  } else if (r_mode == SERQ_R_INT) {
    if (cudaMalloc(&h->rbuf, N * r) != cudaSuccess || cudaMalloc(&h->sr, N * 4) != cudaSuccess ||
        cudaMalloc(&h->colsum_r, N * 4) != cudaSuccess)
      return bail(fail(SERQ_ECUDA, "cudaMalloc R"));
    const int32_t* rc32 = static_cast<const int32_t*>(r_data);
    transpose_codes_kernel<<<dim3(unsigned(cdiv(N, 32)), unsigned(cdiv(r, 32))), dim3(32, 8), 0, st>>>(
        rc32, r, N, static_cast<int8_t*>(h->rbuf));
    colsum_kernel<<<unsigned(cdiv(N, 256)), 256, 0, st>>>(rc32, r, N, r_scales, h->colsum_r, h->sr);
    if (cudaGetLastError() != cudaSuccess) return bail(fail(SERQ_ECUDA, "pack R launch failed"));
    rc = make_map(&h->map_r, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->rbuf, r, N, r, 128, kBN);
    if (!rc) rc = make_map(&h->map_r_pair, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->rbuf, r, N, r, 128, 128);
    if (!rc) rc = make_map(&h->map_r_pair64, CU_TENSOR_MAP_DATA_TYPE_UINT8, h->rbuf, r, N, r, 128, 64);
    if (rc) return bail(rc);
  }
  *out = h;
  return SERQ_OK;
}

int serq_pack_int_grouped(const int32_t* codes, const double* scales, int64_t group_size, int64_t K, int64_t N,
                          int w_bits, int r_mode, const void* r_data, const double* r_scales, int r,
                          int salient_contiguous, serq_linear_t** out, serq_stream_t stream) {
  if (group_size == K && r_mode != SERQ_R_DENSE_SPLIT)
    return serq_pack_int(codes, scales, K, N, w_bits, r_mode, r_data, r_scales, r, salient_contiguous, out, stream);
  if (!out) return fail(SERQ_EINVAL, "out is NULL");
  *out = nullptr;
  if (group_size <= 0 || group_size % 128 || group_size > 8192 || K % group_size)
    return fail(SERQ_EINVAL,
                "group_size %lld: the device needs a multiple of 128, at most 8192, dividing K = %lld "
                "(one integer partial per group, exact in fp32)",
                (long long)group_size, (long long)K);
  if (r_mode == SERQ_R_INT && (!salient_contiguous || r > 128))
    return fail(SERQ_EINVAL, "group-wise weights with integer R need the permuted layout and r <= 128");
  if ((r_mode == SERQ_R_DENSE || r_mode == SERQ_R_DENSE_SPLIT) && (r > 128 || r % 8 || r <= 0 || !r_data))
    return fail(SERQ_EINVAL, "group-wise weights with dense R need 0 < r <= 128, r %% 8 == 0");
  // the per-channel pack builds the int8 weights (and R unless split) and their maps; its group-0
  // scales go unused
  serq_linear_t* h = nullptr;
  const bool split = r_mode == SERQ_R_DENSE_SPLIT;
  int rc = pack_int_impl(codes, scales, K, N, w_bits, split ? SERQ_R_NONE : r_mode, split ? nullptr : r_data,
                         r_scales, split ? 0 : r, salient_contiguous, false, &h, stream);
  if (rc) return rc;
  h->use_i8g = true;
  if (split) {
    // bf16 hi plane rows [0, N), lo plane rows [N, 2N), each [N, r]
    h->r = r;
    h->r_mode = SERQ_R_DENSE_SPLIT;
    h->contiguous = salient_contiguous ? 1 : 0;
    if (cudaMalloc(&h->rbuf, 2 * N * r * 2) != cudaSuccess) {
      free_handle(h);
      return fail(SERQ_ECUDA, "cudaMalloc R");
    }
    __nv_bfloat16* hi = static_cast<__nv_bfloat16*>(h->rbuf);
    dense_r_split_kernel<<<unsigned(cdiv(N * r, 256)), 256, 0, S(stream)>>>(static_cast<const double*>(r_data), r, N,
                                                                            hi, hi + N * r);
    rc = make_map(&h->map_r_pair, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, h->rbuf, r, 2 * N, r * 2, 64, 128);
    if (rc || cudaGetLastError() != cudaSuccess) {
      free_handle(h);
      return rc ? rc : fail(SERQ_ECUDA, "dense_r_split launch failed");
    }
  }
  const int64_t G = K / group_size;
  h->groups = int(G);
  h->gsteps = int(group_size / 128);
  if (cudaMalloc(&h->sw_g, G * N * 4) != cudaSuccess || cudaMalloc(&h->colsum_g, G * N * 4) != cudaSuccess ||
      cudaMalloc(&h->cterm, N * 4) != cudaSuccess) {
    free_handle(h);
    return fail(SERQ_ECUDA, "cudaMalloc failed for group scales");
  }
  group_pack_kernel<<<unsigned(cdiv(N, 256)), 256, 0, S(stream)>>>(
      codes, K, N, group_size, scales, r_mode == SERQ_R_INT ? r_scales : nullptr, h->colsum_r, h->colsum_g, h->sw_g,
      h->cterm);
  if (cudaGetLastError() != cudaSuccess) {
    free_handle(h);
    return fail(SERQ_ECUDA, "group_pack launch failed");
  }
  *out = h;
  return SERQ_OK;
}

int serq_linear_destroy(serq_linear_t* h) {
  if (h) free_handle(h);
  return SERQ_OK;
}

int serq_linear_weight_bytes(const serq_linear_t* h, int64_t* main_bytes, int* packed_int4) {
  if (!h) return fail(SERQ_EINVAL, "NULL handle");
  if (main_bytes) *main_bytes = h->mode == kModeI8 ? h->w_bytes : cdiv(h->N, 128) * h->w_ksteps * 128 * 128;
  if (packed_int4) *packed_int4 = h->mode == kModeI8 ? (h->has_w4 ? 1 : 0) : 1;
  return SERQ_OK;
}

int serq_linear_info(const serq_linear_t* h, int64_t* N, int64_t* K, int* r, int* mode, int* r_mode) {
  if (!h) return fail(SERQ_EINVAL, "NULL handle");
  if (N) *N = h->N;
  if (K) *K = h->K;
  if (r) *r = h->r;
  if (mode) *mode = h->mode;
  if (r_mode) *r_mode = h->r_mode;
  return SERQ_OK;
}

// the quantizer's salient-slice buffer: r columns, or 128 per segment for fused linears
static int64_t xs_cols_of(const serq_linear* h) { return h->nseg > 1 ? 128 * int64_t(h->nseg) : h->r; }

// Decode (M <= 16): one cluster of S CTAs per 128-row weight tile, split-K,
// DSMEM reduction (serq_gemm_decode3.cuh).  x != nullptr: the quantizer is
// fused in (x bf16 [M, K], pitch ldx); codes_out / sf_out optionally receive
// the quantized activation.
static int launch_decode_cl(const serq_linear* h, const uint8_t* a_codes, const uint8_t* a_sf,
                            const __nv_bfloat16* x, int64_t ldx, uint8_t* codes_out, uint8_t* sf_out, int64_t M,
                            void* y, int64_t ldy, cudaStream_t st, const uint8_t* xs_codes = nullptr,
                            const uint8_t* xs_sf = nullptr) {
  CK(set_smem_attr(serq_mx_decode_cl_kernel<false, 1, 32>, ClCfg<false, 32>::kSmem));
  CK(set_smem_attr(serq_mx_decode_cl_kernel<true, 1, 32>, ClCfg<true, 32>::kSmem));
  CK(set_smem_attr(serq_mx_decode_cl_kernel<true, 2, 32>, ClCfg<true, 32>::kSmem));
  CK(set_smem_attr(serq_mx_decode_cl_kernel<false, 1, 64>, ClCfg<false, 64>::kSmem));
  CK(set_smem_attr(serq_mx_decode_cl_kernel<true, 1, 64>, ClCfg<true, 64>::kSmem));
  CK(set_smem_attr(serq_mx_decode_cl_kernel<true, 2, 64>, ClCfg<true, 64>::kSmem));
  const bool rw64 = h->r > 0 && h->dec_rw == 64;
  const bool fuse = x != nullptr;
  const int tiles = int(cdiv(h->N, 128));
  const int ks = int(cdiv(h->K / 2, kStepBytes));
  // CTAs per tile, ~3/4 CTA per SM in total (Llama-2-7B: up_proj 86 tiles -> 1, down_proj 32 -> 3);
  // measured best among 1..8 for both shapes (tools/decode_probe.py)
  int S = (3 * sm_count()) / (4 * tiles);
#ifdef SERQ_DIAG
  if (const char* e = getenv("SERQ_DEC_S")) S = atoi(e);
#endif
  S = S < 1 ? 1 : (S > 8 ? 8 : S);
  if (S > ks) S = ks;
  ClParams cp{};
  cp.M = int(M);
  cp.N = int(h->N);
  cp.K = int(h->K);
  cp.r = h->r;
  cp.k_steps = ks;
  cp.S = S;
  cp.kc_pad = kc_pad_of(h->K);
  cp.kc_pad_r = kc_pad_of(h->r > 0 ? h->r : 32);
  cp.w_ksteps = h->w_ksteps;
  cp.y = static_cast<__nv_bfloat16*>(y);
  cp.ldy = ldy;
  cp.dbg_ts = g_debug_ts;
  cp.x = x;
  cp.ldx = ldx;
  cp.codes_out = codes_out;
  cp.sf_out = sf_out;
  DecodeMaps dm;
  dm.w = h->map_b128;
  dm.sfw = h->map_sfw;
  dm.r = h->dec_rw ? h->map_rdec : h->map_b128;
  dm.sfr = h->dec_rw ? h->map_sfr4 : h->map_sfw;
  const bool gather = h->r > 0 && !h->contiguous;
  if (gather && (fuse || !xs_codes || !xs_sf)) return fail(SERQ_EINVAL, "gather decode needs the xs slice");
  cp.gather = gather ? 1 : 0;
  cp.red_narrow = (S - 1) * ((M + 3) / 4) * 128 * 16 <= kClRed && !SERQ_DBG(g_debug_flags, 1 << 29) ? 1 : 0;
  dm.xs = dm.sfxs = h->map_b128;  // unused unless gather
  cp.nseg = h->nseg;
  for (int j = 0; j + 1 < h->nseg; ++j) cp.seg_row[j] = int(h->seg_row[j]);
  if (gather) {
    const int64_t xc = xs_cols_of(h);  // a tile's slice: 32 B at byte column 64 * segment
    int rc = make_map(&dm.xs, CU_TENSOR_MAP_DATA_TYPE_UINT8, xs_codes, xc / 2, M, xc / 2, 32, kDecN,
                      CU_TENSOR_MAP_SWIZZLE_32B);
    if (!rc)
      rc = make_map(&dm.sfxs, CU_TENSOR_MAP_DATA_TYPE_UINT8, xs_sf, 128, uint64_t(sf_bytes_of(M, xc) / 128), 128, 128,
                    4, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
  }
  if (fuse) {
    dm.x = h->map_b128;  // unused: X is converted in-kernel
    dm.sfx = h->map_b128;  // unused
  } else {
    int rc = make_map(&dm.x, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_codes, h->K / 2, M, h->K / 2, 128, kDecN);
    if (!rc) rc = make_sf_map(&dm.sfx, a_sf, M, h->K);
    if (rc) return rc;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(tiles * S));
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = rw64 ? (fuse ? ClCfg<true, 64>::kSmem : ClCfg<false, 64>::kSmem)
                              : (fuse ? ClCfg<true, 32>::kSmem : ClCfg<false, 32>::kSmem);
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = unsigned(S);
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  if (fuse) {
    // converter lanes carry 1 or 2 token rows
    if (M <= 4)
      CK(rw64 ? cudaLaunchKernelEx(&cfg, serq_mx_decode_cl_kernel<true, 1, 64>, dm, cp)
              : cudaLaunchKernelEx(&cfg, serq_mx_decode_cl_kernel<true, 1, 32>, dm, cp));
    else
      CK(rw64 ? cudaLaunchKernelEx(&cfg, serq_mx_decode_cl_kernel<true, 2, 64>, dm, cp)
              : cudaLaunchKernelEx(&cfg, serq_mx_decode_cl_kernel<true, 2, 32>, dm, cp));
  } else {
    CK(rw64 ? cudaLaunchKernelEx(&cfg, serq_mx_decode_cl_kernel<false, 1, 64>, dm, cp)
            : cudaLaunchKernelEx(&cfg, serq_mx_decode_cl_kernel<false, 1, 32>, dm, cp));
  }
  LAUNCH_CHECK("serq_mx_decode_cl_kernel");
  return SERQ_OK;
}

static int linear_mx_impl(const serq_linear_t* h, const uint8_t* a_codes, const uint8_t* a_sf, int64_t M,
                          const uint8_t* xs_codes, const uint8_t* xs_sf, void* y, int64_t ldy, serq_stream_t stream,
                          const float* addend = nullptr) {
  g_launches = 0;
  if (!h || h->mode != kModeMX) return fail(SERQ_EINVAL, "handle is not an MX linear");
  if (addend && (h->r != 0 || h->nseg > 1))
    return fail(SERQ_EINVAL, "an fp32 addend needs an MX linear without salient term or segments");
  if (M <= 0) return fail(SERQ_EINVAL, "x must be non-empty");
  if (ldy < h->N || ldy % 8) return fail(SERQ_EINVAL, "ldy must be >= N and a multiple of 8");
  const bool need_xs = h->r > 0 && !h->contiguous;
  if (need_xs && (!xs_codes || !xs_sf)) return fail(SERQ_EINVAL, "non-contiguous salient set needs the xs slice");
  if (h->nseg > 1) {
    // fused linears run as ONE kernel on the decode kernel (M <= 16) and the CTA-pair kernel (r = 64,
    // segments of whole 256-column tiles); other shapes go through per-segment views (serq_linear_view)
    bool tiles256 = true;
    for (int j = 0; j + 1 < h->nseg; ++j) tiles256 = tiles256 && h->seg_row[j] % 256 == 0;
    const bool dec = M <= kDecN && h->has_r32;
    const bool pair = M > 128 && h->has_r32 && tiles256;
    if (!dec && !pair)
      return fail(SERQ_EINVAL, "fused segments need M <= 16, or M > 128 with r = 64 and 256-row-aligned segments "
                               "(use per-segment views)");
  }
  CK(set_smem_attr(serq_mx_persistent_kernel, kPSmemBytes));
  int rc = SERQ_OK;
  CUtensorMap ma, mxs, my;
  rc = make_map(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_codes, h->K / 2, M, h->K / 2, 128, kBM);
  if (rc) return rc;
  if (need_xs) {
    rc = make_map(&mxs, CU_TENSOR_MAP_DATA_TYPE_UINT8, xs_codes, h->r / 2, M, h->r / 2, 128, kBM);
    if (rc) return rc;
  } else {
    mxs = ma;
  }
  rc = make_map(&my, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, h->N, M, ldy * 2, 64, 32);
  if (rc) return rc;
  GemmParams p{};
  p.M = int(M);
  p.N = int(h->N);
  p.K = int(h->K);
  p.r = h->r;
  p.k_steps = int(cdiv(h->K / 2, kStepBytes));
  p.r_steps = int(cdiv(h->r / 2, kStepBytes));
  p.r_mode = h->r > 0 ? 1 : 0;
  p.sfa = a_sf;
  p.sfb = h->sfw;
  p.xs_is_x = need_xs ? 0 : 1;
  p.sfa_r = need_xs ? xs_sf : a_sf;
  p.sfb_r = h->sfr;
  p.kc_pad = kc_pad_of(h->K);
  p.kc_pad_r = kc_pad_of(h->r > 0 ? h->r : 32);
  p.w_ksteps = h->w_ksteps;
  p.dbg = g_debug_flags;
  p.dbg_ts = g_debug_ts;
  p.addend = addend;  // (the SVD baseline: the CTA-pair kernel for M > 16, else the one-CTA kernel)
  // decode kernel: any contiguous R up to r = 128; the gather fallback with r = 64 (32-B xs rows)
  const bool dec_ok = !addend && (h->r == 0 || (h->dec_rw && (h->contiguous || h->has_r32)));
  if (M <= kDecN && dec_ok && !SERQ_DBG(g_debug_flags, 2048))
    return launch_decode_cl(h, a_codes, a_sf, nullptr, 0, nullptr, nullptr, M, y, ldy, S(stream), xs_codes, xs_sf);
  // pair3 for the permuted layout, and for the gather fallback with r == 64 (debug flag 1<<24: the
  // gather cases take the older pair kernel)
  const bool g3 = h->r > 0 && h->has_r32 && !h->contiguous && xs_codes && xs_sf && !SERQ_DBG(g_debug_flags, 1 << 24);
  // (M > 16: between the decode kernel and one 256-row tile the pair kernels also beat the one-CTA
  // kernel -- rows past M are TMA zero-filled and never stored; Llama-2-7B up_proj at M = 17..128:
  // 14.3-15.8 us one-CTA vs 11.6 us pair3, tools/probes/mx_midm_probe.py)
  if (M > kDecN && (h->r == 0 || (h->has_r32 && h->contiguous) || g3) && !SERQ_DBG(g_debug_flags, 16 | 512)) {
    CK(set_smem_attr(serq_mx_pair3_kernel<false>, k3SmemBytes));
    CK(set_smem_attr(serq_mx_pair3_kernel<true>, k3SmemBytesG));
    CK(set_smem_attr(serq_mx_pair3_kernel<false, true>, k3SmemBytes));
    Pair3Maps pm;
    rc = make_map(&pm.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_codes, h->K / 2, M, h->K / 2, 128, 128);
    if (!rc) rc = make_sf_map(&pm.sfa, a_sf, M, h->K);
    if (!rc && !g3)
      rc = make_map(&pm.y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, h->N, M, ldy * 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (!rc && g3)  // 32 rows x 16 columns per epilogue box
      rc = make_map(&pm.y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, h->N, M, ldy * 2, 16, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    const int64_t xc = xs_cols_of(h);  // per tile: 32 B at byte column 64 * segment
    if (!rc && g3)
      rc = make_map(&pm.xs, CU_TENSOR_MAP_DATA_TYPE_UINT8, xs_codes, xc / 2, M, xc / 2, 32, 128,
                    CU_TENSOR_MAP_SWIZZLE_32B);
    if (!rc && g3)
      rc = make_map(&pm.sfxs, CU_TENSOR_MAP_DATA_TYPE_UINT8, xs_sf, 128, uint64_t(sf_bytes_of(M, xc) / 128), 128, 128,
                    4, CU_TENSOR_MAP_SWIZZLE_NONE);
    p.kc_pad_xs = kc_pad_of(xc > 0 ? xc : 32);
    p.nseg = h->nseg;
    for (int j = 0; j + 1 < h->nseg; ++j) p.seg_row[j] = int(h->seg_row[j]);
    if (rc) return rc;
    if (!g3) pm.xs = pm.sfxs = pm.a;  // unused
    pm.b = h->map_b128;
    pm.b64 = h->map_b64;
    pm.sfb = h->map_sfw;
    pm.r = h->has_r32 ? h->map_r32 : h->map_b128;
    pm.sfr = h->has_r32 ? h->map_sfr4 : h->map_sfw;
    const int64_t pairs = cdiv(M, 256) * cdiv(h->N, kBN);
    const int64_t max_pairs = sm_count() / 2;
    const int64_t clusters = pairs < max_pairs ? pairs : max_pairs;
    // split the last partial wave into K-halves when they fit in one round
    const int64_t rounds = pairs / clusters, left = pairs - rounds * clusters;
    p.narrow_from = int(pairs);
    // tile order: N-fastest measured +2.4% at 8192^3, equal at 4096^3 (tools/sweep_mx.py)
    p.group_m = SERQ_DBG(g_debug_flags, 262144) ? 0 : 1;
    // the last partial round as 256 x 128 tiles (two per leftover tile): each takes ~3/4 of a full
    // tile's time (the A operand is fed twice) instead of half the clusters idling through a full
    // tile (measured faster than splitting the leftover tiles into K-halves, K2)
    if (left > 0 && 2 * left <= clusters && rounds >= 1 && !SERQ_DBG(g_debug_flags, 1 << 19))
      p.narrow_from = int(rounds * clusters);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(2 * clusters));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = g3 ? k3SmemBytesG : k3SmemBytes;
    cfg.stream = S(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap with the quantizer's tail
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (g3) {
      CK(cudaLaunchKernelEx(&cfg, serq_mx_pair3_kernel<true>, pm, p));
      LAUNCH_CHECK("serq_mx_pair3_kernel<gather>");
    } else if (addend) {
      CK(cudaLaunchKernelEx(&cfg, serq_mx_pair3_kernel<false, true>, pm, p));
      LAUNCH_CHECK("serq_mx_pair3_kernel<addend>");
    } else {
      CK(cudaLaunchKernelEx(&cfg, serq_mx_pair3_kernel<false>, pm, p));
      LAUNCH_CHECK("serq_mx_pair3_kernel");
    }
    return SERQ_OK;
  }
  if (M > kDecN && !addend && !SERQ_DBG(g_debug_flags, 16)) {
    CK(set_smem_attr(serq_mx_pair_kernel, k2SmemBytes));
    Pair2Maps pm;
    rc = make_map(&pm.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_codes, h->K / 2, M, h->K / 2, 128, 128);
    if (rc) return rc;
    pm.b = h->map_b128;
    pm.r = h->map_r128;
    rc = make_map(&pm.y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, h->N, M, ldy * 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
    pm.sfb = h->map_sfw;
    pm.sfr = h->map_sfr;
    rc = make_sf_map(&pm.sfa, a_sf, M, h->K);
    if (rc) return rc;
    if (need_xs) {
      rc = make_map(&pm.xs, CU_TENSOR_MAP_DATA_TYPE_UINT8, xs_codes, h->r / 2, M, h->r / 2, 128, 128);
      if (!rc) rc = make_sf_map(&pm.sfxs, xs_sf, M, h->r);
      if (rc) return rc;
    } else {
      pm.xs = pm.a;
      pm.sfxs = pm.sfa;
    }
    const int64_t pairs = cdiv(M, 256) * cdiv(h->N, kBN);
    const int64_t max_pairs = sm_count() / 2;
    const dim3 grid(unsigned(2 * (pairs < max_pairs ? pairs : max_pairs)));
    serq_mx_pair_kernel<<<grid, kThreads, k2SmemBytes, S(stream)>>>(pm, p);
    LAUNCH_CHECK("serq_mx_pair_kernel");
    return SERQ_OK;
  }
  const int64_t tiles = cdiv(M, kBM) * cdiv(h->N, kBN);
  const dim3 grid(unsigned(tiles < sm_count() ? tiles : sm_count()));
  serq_mx_persistent_kernel<<<grid, kThreads, kPSmemBytes, S(stream)>>>(ma, h->map_b, mxs, h->r ? h->map_r : h->map_b,
                                                                        my, p);
  LAUNCH_CHECK("serq_mx_persistent_kernel");
  return SERQ_OK;
}

int serq_linear_mx_addend(const serq_linear_t* h, const uint8_t* a_codes, const uint8_t* a_sf, int64_t M,
                          const float* addend, void* y, int64_t ldy, serq_stream_t stream) {
  if (!addend) return fail(SERQ_EINVAL, "addend is NULL");
  // (rows of N % 8 == 0 floats: 16-B aligned when the base is; the kernels read 16 B at a time)
  if (reinterpret_cast<uintptr_t>(addend) & 15) return fail(SERQ_EINVAL, "addend must be 16-byte aligned");
  return linear_mx_impl(h, a_codes, a_sf, M, nullptr, nullptr, y, ldy, stream, addend);
}

int serq_linear_mx(const serq_linear_t* h, const uint8_t* a_codes, const uint8_t* a_sf, int64_t M,
                   const uint8_t* xs_codes, const uint8_t* xs_sf, void* y, int64_t ldy, serq_stream_t stream) {
  return linear_mx_impl(h, a_codes, a_sf, M, xs_codes, xs_sf, y, ldy, stream);
}

int serq_forward_mx(serq_linear_t* h, const void* x, int dtype, int64_t M, int64_t ldx, const int32_t* gather_idx,
                    uint8_t* codes, uint8_t* sf, uint8_t* xs_codes, uint8_t* xs_sf, void* y, int64_t ldy,
                    serq_stream_t stream) {
  if (!h || h->mode != kModeMX) return fail(SERQ_EINVAL, "handle is not an MX linear");
  const bool gather = h->r > 0 && !h->contiguous;
  if (gather && (!gather_idx || !xs_codes || !xs_sf))
    return fail(SERQ_EINVAL, "non-contiguous salient set needs gather_idx and the xs buffers");
  if (M <= kClFuseM && (h->r == 0 || h->dec_rw) && dtype == SERQ_BF16 && !gather &&
      !(reinterpret_cast<uintptr_t>(x) & 15) && ldx % 8 == 0 && ldx >= h->K && !SERQ_DBG(g_debug_flags, 1 << 23) &&
      !SERQ_DBG(g_debug_flags, 2048)) {
    // decode (M <= 8) with the quantizer inside the linear: one kernel per layer instead of
    // quantizer + PDL-chained linear (Llama-2-7B M=1: up_proj 7.8 vs 8.2 us/layer, down_proj
    // 8.1 vs 9.1; tools/decode_probe.py); debug flag 1<<23 selects the two-kernel path
    g_launches = 0;
    if (ldy < h->N || ldy % 8) return fail(SERQ_EINVAL, "ldy must be >= N and a multiple of 8");
    return launch_decode_cl(h, nullptr, nullptr, static_cast<const __nv_bfloat16*>(x), ldx, codes, sf, M, y, ldy,
                            S(stream));
  }
  // the linear is launched with programmatic dependent launch: its prologue and
  // weight stream overlap the quantizer (a per-row-tile counter hand-off was
  // measured slower: 45.1 vs 43.0 us at 4096^3, tools/fuse_probe.py)
  int rc = act_quant_mx_impl(x, dtype, M, h->K, ldx, codes, sf, gather ? gather_idx : nullptr,
                             gather ? int(xs_cols_of(h)) : 0,
                             xs_codes, xs_sf, stream);
  if (rc) return rc;
  const int n1 = g_launches;
  rc = linear_mx_impl(h, codes, sf, M, gather ? xs_codes : nullptr, gather ? xs_sf : nullptr, y, ldy, stream);
  g_launches += n1;
  return rc;
}

#ifndef SERQ_I8_EPI
#define SERQ_I8_EPI 2
#endif
constexpr int kI8Epi = SERQ_I8_EPI;  // epilogue column groups of the INT CTA-pair kernel (4 * kI8Epi warps)

static int linear_int_impl(const serq_linear_t* h, const int8_t* a_codes, const float* sx, const int32_t* zp,
                           int64_t M, const void* xs, void* y, int64_t ldy, const float* addend, int32_t* acc_dump,
                           int32_t* accr_dump, serq_stream_t stream) {
  g_launches = 0;
  if (!h || h->mode != kModeI8) return fail(SERQ_EINVAL, "handle is not an INT linear");
  if (M <= 0) return fail(SERQ_EINVAL, "x must be non-empty");
  if (ldy < h->N || ldy % 8) return fail(SERQ_EINVAL, "ldy must be >= N and a multiple of 8");
  const bool need_xs = h->r_mode == SERQ_R_DENSE || h->r_mode == SERQ_R_DENSE_SPLIT ||
                       (h->r_mode == SERQ_R_INT && !h->contiguous);
  if (need_xs && !xs) return fail(SERQ_EINVAL, "this R mode needs the quantizer's xs slice");
  // (group-wise handles too: each main warp owns whole groups, at most kGemvMaxGpw of them)
  const bool gemv_fmt_ok = !h->use_i8g || h->groups <= kGemvMaxGpw * 4;
  // group-wise and packed-INT4 handles with few 256-column tiles (their pair kernels would leave
  // most CTA pairs idle) take the gemv up to M = 32, one 16-token group per grid row; each group
  // re-streams the weights, so this pays only there (Llama-2-7B down_proj, 16 tiles, M = 32:
  // group-wise 36 vs 79 us, tools/probes/i8g_smallm_probe.py; INT4 vs 38.6 us; up_proj, 43 tiles:
  // not taken)
  const int64_t gemv_max_m = (h->use_i8g || h->has_w4) && 3 * cdiv(h->N, 256) <= int64_t(sm_count()) / 2
                                 ? SERQ_GEMV_I8G_MAX_M
                                 : 16;
  if (M <= gemv_max_m && gemv_fmt_ok && h->r <= 128 && !SERQ_DBG(g_debug_flags, 1 << 29)) {
    // decode sizes: the weight stream with warp-level MMAs (serq_gemv_i8.cuh), int8 or packed INT4
    GemvI8Params gp{};
    gp.w = static_cast<const int8_t*>(h->w);
    gp.K = int(h->K);
    gp.N = int(h->N);
    gp.M = int(M);
    gp.a = reinterpret_cast<const uint8_t*>(a_codes);
    gp.sx = sx;
    gp.zp = zp;
    gp.sw = h->sw;
    gp.colsum = h->colsum;
    gp.r = h->r;
    gp.rw = h->rbuf;
    gp.sr = h->sr;
    gp.colsum_r = h->colsum_r;
    gp.xs = (h->r_mode == SERQ_R_INT && h->contiguous) ? nullptr : xs;
    gp.y = static_cast<__nv_bfloat16*>(y);
    gp.ldy = ldy;
    gp.addend = addend;
    gp.acc_dump = acc_dump;
    gp.accr_dump = accr_dump;
    gp.sw_g = h->sw_g;
    gp.cterm = h->cterm;
    gp.colsum_g = h->colsum_g;
    gp.groups = h->groups;
    gp.gchunks = 2 * h->gsteps;  // 64-K chunks per group
    const int fmt = h->use_i8g ? 2 : h->has_w4 ? 1 : 0;
    const bool sgn = zp == nullptr;
    // 16 weight rows per CTA; 8 (M <= 8) / 7 warps split K when the row groups alone leave SMs
    // idle (a wave holds 2 such CTAs per SM), 4 otherwise (all CTAs in one wave); plus one warp
    // for the salient term and the epilogue (tools/probes/int_decode_probe.py for the A/B)
    const int64_t groups = cdiv(h->N, 16);
    const bool wide = groups <= 2 * int64_t(sm_count());
    const dim3 grid{unsigned(groups), unsigned(cdiv(M, 16))}, blk{!wide ? 160u : M <= 8 ? 288u : 256u};  // + side warp
    cudaError_t e = cudaSuccess;
#define GEMV_W4(NT, SG, KR, W4)                                                                                     \
  e = wide ? launch_pdl(serq_i8_gemv_kernel<NT, SG, KR, NT == 1 ? 8 : 7, W4>, grid, blk, 0, S(stream), gp)        \
           : launch_pdl(serq_i8_gemv_kernel<NT, SG, KR, 4, W4>, grid, blk, 0, S(stream), gp)
#define GEMV_W(NT, SG, KR)                                                                                          \
  do {                                                                                                             \
    if (fmt == 2) GEMV_W4(NT, SG, KR, 2);                                                                          \
    else if (fmt == 1) GEMV_W4(NT, SG, KR, 1);                                                                     \
    else GEMV_W4(NT, SG, KR, 0);                                                                                   \
  } while (0)
#define GEMV_R(NT, KR)                                                                                              \
  do {                                                                                                             \
    if (sgn) GEMV_W(NT, true, KR);                                                                                 \
    else GEMV_W(NT, false, KR);                                                                                    \
  } while (0)
#define GEMV_M(NT)                                                                                                 \
  do {                                                                                                             \
    if (h->r_mode == SERQ_R_INT) GEMV_R(NT, kRInt);                                                                \
    else if (h->r_mode == SERQ_R_DENSE) GEMV_R(NT, kRDense);                                                       \
    else if (h->r_mode == SERQ_R_DENSE_SPLIT) GEMV_R(NT, kRDenseSplit);                                            \
    else GEMV_R(NT, 0);                                                                                            \
  } while (0)
    if (M <= 8) GEMV_M(1);
    else GEMV_M(2);
#undef GEMV_M
#undef GEMV_R
#undef GEMV_W
#undef GEMV_W4
    CK(e);
    LAUNCH_CHECK("serq_i8_gemv_kernel");
    return SERQ_OK;
  }
  if (h->use_i8g) {
    // group-wise weight scales: one promoted integer partial per group (serq_gemm_i8g.cuh), any M
    {
      int mx = 0;
      for (int m = 0; m <= kRDenseSplit; ++m) mx = i8g_smem(m) > mx ? i8g_smem(m) : mx;
      CK(set_smem_attr(serq_i8g_pair_kernel<false>, mx));
      CK(set_smem_attr(serq_i8g_pair_kernel<true>, mx));
    }
    I8Maps im;
    int rc = make_map(&im.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_codes, h->K, M, h->K, 128, 128);
    if (!rc)  // 32 rows x 16 columns per epilogue-warp store, no swizzle
      rc = make_map(&im.y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, h->N, M, ldy * 2, 16, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc && (h->r_mode == SERQ_R_DENSE || h->r_mode == SERQ_R_DENSE_SPLIT))
      rc = make_map(&im.xs, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, xs, h->r, M, h->r * 2, 64, 128);
    if (rc) return rc;
    if (h->r_mode != SERQ_R_DENSE && h->r_mode != SERQ_R_DENSE_SPLIT) im.xs = im.a;
    im.bp = h->map_w8;
    im.r = h->r_mode != SERQ_R_NONE ? h->map_r_pair : im.bp;
    I8gParams p{};
    p.M = int(M);
    p.N = int(h->N);
    p.K = int(h->K);
    p.r = h->r;
    p.r_mode = h->r_mode;
    p.a_signed = zp ? 0 : 1;
    p.k_steps = int(h->K / 128);
    p.gsteps = h->gsteps;
    p.sx = sx;
    p.zp = zp;
    p.sw_g = h->sw_g;
    p.cterm = h->cterm;
    p.sr = h->sr;
    p.colsum_g = h->colsum_g;
    p.colsum_r = h->colsum_r;
    p.addend = addend;
    p.acc_dump = acc_dump;
    p.accr_dump = accr_dump;
    p.dbg_ts = g_debug_ts;
    const int64_t tiles = cdiv(M, 256) * cdiv(h->N, 256);
    const int64_t max_pairs = sm_count() / 2;
    const dim3 grid(unsigned(2 * (tiles < max_pairs ? tiles : max_pairs)));
    if (acc_dump || accr_dump)
      CK(launch_pdl(serq_i8g_pair_kernel<true>, grid, dim3(kI8gThreads), i8g_smem(h->r_mode), S(stream), im, p));
    else
      CK(launch_pdl(serq_i8g_pair_kernel<false>, grid, dim3(kI8gThreads), i8g_smem(h->r_mode), S(stream), im, p));
    LAUNCH_CHECK("serq_i8g_pair_kernel");
    return SERQ_OK;
  }
  // CTA-pair kernel: int8 weights TMA'd straight into the operand
  // W4 handles always take the CTA-pair kernel (it is the one that widens packed INT4); int8
  // handles too when their R layout allows it -- also between the gemv's 16 rows and one 256-row
  // tile (rows past M are TMA zero-filled and never stored): up_proj at M = 17..128 took 41 us
  // on the one-CTA kernel below
  const bool pair_ok = h->has_w4 || ((h->r_mode != SERQ_R_INT || h->contiguous) && h->r <= 128 &&
                                     (h->r_mode != SERQ_R_DENSE || cdiv(h->K, 128) >= cdiv(h->r, 64)) &&
                                     !SERQ_DBG(g_debug_flags, 65536));
  if (pair_ok) {
    using Cfg8 = I8Cfg<kI8Epi, false>;
    using Cfg4 = I8Cfg<kI8Epi, true>;
    CK(set_smem_attr(serq_i8_pair_kernel<256, kI8Epi, false>, Cfg8::kSmem));
    CK(set_smem_attr(serq_i8_pair_kernel<128, kI8Epi, false>, Cfg8::kSmem));
    CK(set_smem_attr(serq_i8_pair_kernel<256, kI8Epi, true>, Cfg4::kSmem));
    CK(set_smem_attr(serq_i8_pair_kernel<128, kI8Epi, true>, Cfg4::kSmem));
    I8Maps im;
    int rc = make_map(&im.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_codes, h->K, M, h->K, 128, 128);
    if (!rc)
      rc = make_map(&im.y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, h->N, M, ldy * 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (!rc && h->r_mode == SERQ_R_DENSE)
      rc = make_map(&im.xs, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, xs, h->r, M, h->r * 2, 64, 128);
    if (rc) return rc;
    if (h->r_mode != SERQ_R_DENSE) im.xs = im.a;
    // few 256x256 tiles (C1: 2 x 16 on 74 pairs): 128-column tiles put twice as many pairs to work
    const bool narrow = cdiv(M, 256) * cdiv(h->N, 256) * 2 <= sm_count() / 2 && !SERQ_DBG(g_debug_flags, 1 << 27);
    im.bp = h->has_w4 ? im.a : (narrow ? h->map_w8_64 : h->map_w8);  // (W4: no weight tensor map)
    im.r = h->r_mode != SERQ_R_NONE ? (narrow ? h->map_r_pair64 : h->map_r_pair) : im.bp;
    GemmParams p{};
    p.dbg = g_debug_flags;
    p.M = int(M);
    p.N = int(h->N);
    p.K = int(h->K);
    p.r = h->r;
    p.k_steps = int(cdiv(h->K, 128));
    p.r_mode = h->r_mode;
    p.a_signed = zp ? 0 : 1;
    p.sx = sx;
    p.zp = zp;
    p.sw = h->sw;
    p.colsum = h->colsum;
    p.sr = h->sr;
    p.colsum_r = h->colsum_r;
    p.acc_dump = acc_dump;
    p.addend = addend;
    p.accr_dump = accr_dump;
    p.dbg_ts = g_debug_ts;
    p.w4 = h->has_w4 ? static_cast<const uint8_t*>(h->w) : nullptr;
    const int64_t tiles = cdiv(M, 256) * cdiv(h->N, narrow ? 128 : kBN);
    const int64_t max_pairs = sm_count() / 2;
    const dim3 grid(unsigned(2 * (tiles < max_pairs ? tiles : max_pairs)));
    // launched with programmatic dependent launch: the prologue and the first weight stages
    // overlap the activation quantizer's tail
    using Cfg8 = I8Cfg<kI8Epi, false>;
    using Cfg4 = I8Cfg<kI8Epi, true>;
    if (h->has_w4 && narrow) {
      CK(launch_pdl(serq_i8_pair_kernel<128, kI8Epi, true>, grid, dim3(Cfg4::kThreads), Cfg4::kSmem, S(stream), im, p));
      LAUNCH_CHECK("serq_i8_pair_kernel<128,w4>");
    } else if (h->has_w4) {
      CK(launch_pdl(serq_i8_pair_kernel<256, kI8Epi, true>, grid, dim3(Cfg4::kThreads), Cfg4::kSmem, S(stream), im, p));
      LAUNCH_CHECK("serq_i8_pair_kernel<256,w4>");
    } else if (narrow) {
      CK(launch_pdl(serq_i8_pair_kernel<128, kI8Epi, false>, grid, dim3(Cfg8::kThreads), Cfg8::kSmem, S(stream), im,
                    p));
      LAUNCH_CHECK("serq_i8_pair_kernel<128>");
    } else {
      CK(launch_pdl(serq_i8_pair_kernel<256, kI8Epi, false>, grid, dim3(Cfg8::kThreads), Cfg8::kSmem, S(stream), im,
                    p));
      LAUNCH_CHECK("serq_i8_pair_kernel<256>");
    }
    return SERQ_OK;
  }
  int rc = ensure_attr<kModeI8>();
  if (rc) return rc;
  CUtensorMap ma, mxs, my;
  rc = make_map(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_codes, h->K, M, h->K, 128, kBM);
  if (rc) return rc;
  if (h->r_mode == SERQ_R_DENSE)
    rc = make_map(&mxs, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, xs, h->r, M, h->r * 2, 64, kBM);
  else if (need_xs)
    rc = make_map(&mxs, CU_TENSOR_MAP_DATA_TYPE_UINT8, xs, h->r, M, h->r, 128, kBM);
  else
    mxs = ma;
  if (rc) return rc;
  rc = make_map(&my, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, h->N, M, ldy * 2, 64, 32);
  if (rc) return rc;
  GemmParams p{};
  p.M = int(M);
  p.N = int(h->N);
  p.K = int(h->K);
  p.r = h->r;
  p.k_steps = int(cdiv(h->K, kStepBytes));
  p.r_mode = h->r_mode;
  p.r_steps = int(cdiv(h->r_mode == SERQ_R_DENSE ? 2 * h->r : h->r, kStepBytes));
  p.a_signed = zp ? 0 : 1;
  p.xs_is_x = need_xs ? 0 : 1;
  p.sx = sx;
  p.zp = zp;
  p.sw = h->sw;
  p.colsum = h->colsum;
  p.sr = h->sr;
  p.colsum_r = h->colsum_r;
  p.acc_dump = acc_dump;
  p.addend = addend;
  p.accr_dump = accr_dump;
  dim3 grid(unsigned(cdiv(M, kBM)), unsigned(cdiv(h->N, kBN)));
  serq_linear_kernel<kModeI8><<<grid, kThreads, kSmemBytes, S(stream)>>>(ma, h->map_b, mxs, h->r ? h->map_r : h->map_b,
                                                                         my, p);
  LAUNCH_CHECK("serq_linear_kernel<i8>");
  return SERQ_OK;
}

int serq_linear_int(const serq_linear_t* h, const int8_t* a_codes, const float* sx, const int32_t* zp, int64_t M,
                    const void* xs, void* y, int64_t ldy, int32_t* acc_dump, int32_t* accr_dump, serq_stream_t stream) {
  return linear_int_impl(h, a_codes, sx, zp, M, xs, y, ldy, nullptr, acc_dump, accr_dump, stream);
}

int serq_linear_int_addend(const serq_linear_t* h, const int8_t* a_codes, const float* sx, const int32_t* zp,
                           int64_t M, const void* xs, const float* addend, void* y, int64_t ldy,
                           serq_stream_t stream) {
  if (!addend) return fail(SERQ_EINVAL, "addend is NULL");
  if (reinterpret_cast<uintptr_t>(addend) & 3) return fail(SERQ_EINVAL, "addend must be 4-byte aligned");
  return linear_int_impl(h, a_codes, sx, zp, M, xs, y, ldy, addend, nullptr, nullptr, stream);
}

// ---------------------------------------------------------------- end to end from host memory
}  // extern "C"

namespace {

// Chunk plan over token rows: every chunk starts on a 256-row boundary (whole MX scale-factor
// tiles), small chunks at both ends (the first H2D and the last D2H overlap nothing), 1024-row
// chunks in the middle (per-chunk launch / copy setup ~25 us, measured with uniform 256-row
// chunks); the last chunk absorbs M % 256.
int64_t e2e_plan(int64_t M, int64_t* plan) {
  int64_t chunks = 0;
  const int64_t body = (M / 256) * 256, rem = M - body;
  const bool ramp = body >= 2560;  // 256 + 512 + [>= 1024] + 512 + 256
  int64_t mid = body - (ramp ? 1536 : 0);
  const int64_t slots = kE2eMaxChunks - (ramp ? 4 : 0);
  int64_t step = 1024;
#ifdef SERQ_DIAG
  if (const char* e = getenv("SERQ_E2E_ROWS")) step = cdiv(atoll(e), 256) * 256;
#endif
  if (cdiv(mid, step) > slots) step = cdiv(cdiv(mid, slots), 256) * 256;
  if (ramp) {
    plan[chunks++] = 256;
    plan[chunks++] = 512;
  }
  while (mid > 0) {
    const int64_t c = mid < step ? mid : step;
    plan[chunks++] = c;
    mid -= c;
  }
  if (ramp) {
    plan[chunks++] = 512;
    plan[chunks++] = 256;
  }
  if (chunks == 0) plan[chunks++] = 0;
  plan[chunks - 1] += rem;
  return chunks;
}

// H2D of chunk i+1, the device work of chunk i and the D2H of chunk i-1 run concurrently on
// the two copy engines and the SMs.  `compute(r0, rows)` enqueues on `st` the work turning
// ws_x rows [r0, r0 + rows) into ws_y rows and returns a status.  Synchronises `st`.
template <typename F>
int host_pipeline(serq_linear* h, const void* x_host, int64_t M, void* y_host, cudaStream_t st, F compute) {
  if (!h->e2e_in) {
    CK(cudaStreamCreateWithFlags(&h->e2e_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->e2e_out, cudaStreamNonBlocking));
    for (cudaEvent_t& e : h->e2e_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  int64_t plan[kE2eMaxChunks];
  const int64_t chunks = e2e_plan(M, plan);
  cudaEvent_t* ev_in = h->e2e_ev;                       // [chunks] x chunk landed
  cudaEvent_t* ev_done = h->e2e_ev + kE2eMaxChunks;     // [chunks] y chunk computed
  cudaEvent_t* ev_out = h->e2e_ev + 2 * kE2eMaxChunks;  // [chunks] y chunk copied out
  cudaEvent_t ev_start = h->e2e_ev[3 * kE2eMaxChunks];
  CK(cudaEventRecord(ev_start, st));  // the copies must follow earlier work on the caller's stream
  CK(cudaStreamWaitEvent(h->e2e_in, ev_start, 0));
  int64_t start[kE2eMaxChunks];
  for (int64_t c = 0, r0 = 0; c < chunks; r0 += plan[c], ++c) start[c] = r0;
  for (int64_t c = 0; c < chunks; ++c) {
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(h->ws_x) + start[c] * h->K * 2,
                       static_cast<const uint8_t*>(x_host) + start[c] * h->K * 2, plan[c] * h->K * 2,
                       cudaMemcpyHostToDevice, h->e2e_in));
    CK(cudaEventRecord(ev_in[c], h->e2e_in));
  }
  int launches = 0;
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t r0 = start[c], mc = plan[c];
    CK(cudaStreamWaitEvent(st, ev_in[c], 0));
    const int rc = compute(r0, mc);
    if (rc) return rc;
    launches += g_launches;
    CK(cudaEventRecord(ev_done[c], st));
    CK(cudaStreamWaitEvent(h->e2e_out, ev_done[c], 0));
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(y_host) + r0 * h->N * 2, static_cast<uint8_t*>(h->ws_y) + r0 * h->N * 2,
                       mc * h->N * 2, cudaMemcpyDeviceToHost, h->e2e_out));
    CK(cudaEventRecord(ev_out[c], h->e2e_out));
  }
  g_launches = launches;
  CK(cudaStreamWaitEvent(st, ev_out[chunks - 1], 0));
  CK(cudaStreamSynchronize(st));
#ifdef SERQ_DIAG
  if (getenv("SERQ_E2E_TRACE")) {  // diagnostics: rerun with timing events, print the spans (us)
    cudaEvent_t t0, th[kE2eMaxChunks], tc0[kE2eMaxChunks], tc[kE2eMaxChunks], to[kE2eMaxChunks];
    cudaEventCreate(&t0);
    for (int64_t c = 0; c < chunks; ++c) {
      cudaEventCreate(&th[c]);
      cudaEventCreate(&tc0[c]);
      cudaEventCreate(&tc[c]);
      cudaEventCreate(&to[c]);
    }
    cudaEventRecord(t0, st);
    cudaStreamWaitEvent(h->e2e_in, t0, 0);
    for (int64_t c = 0; c < chunks; ++c) {
      cudaMemcpyAsync(static_cast<uint8_t*>(h->ws_x) + start[c] * h->K * 2,
                      static_cast<const uint8_t*>(x_host) + start[c] * h->K * 2, plan[c] * h->K * 2,
                      cudaMemcpyHostToDevice, h->e2e_in);
      cudaEventRecord(th[c], h->e2e_in);
    }
    for (int64_t c = 0; c < chunks; ++c) {
      cudaStreamWaitEvent(st, th[c], 0);
      cudaEventRecord(tc0[c], st);
      compute(start[c], plan[c]);
      cudaEventRecord(tc[c], st);
      cudaStreamWaitEvent(h->e2e_out, tc[c], 0);
      cudaMemcpyAsync(static_cast<uint8_t*>(y_host) + start[c] * h->N * 2,
                      static_cast<uint8_t*>(h->ws_y) + start[c] * h->N * 2, plan[c] * h->N * 2, cudaMemcpyDeviceToHost,
                      h->e2e_out);
      cudaEventRecord(to[c], h->e2e_out);
    }
    cudaStreamWaitEvent(st, to[chunks - 1], 0);
    cudaStreamSynchronize(st);
    for (int64_t c = 0; c < chunks; ++c) {
      float a, b, d, e;
      cudaEventElapsedTime(&a, t0, th[c]);
      cudaEventElapsedTime(&b, t0, tc0[c]);
      cudaEventElapsedTime(&d, t0, tc[c]);
      cudaEventElapsedTime(&e, t0, to[c]);
      fprintf(stderr, "e2e chunk %lld rows %lld: h2d_end %.1f compute %.1f..%.1f d2h_end %.1f\n", (long long)c,
              (long long)plan[c], a * 1e3, b * 1e3, d * 1e3, e * 1e3);
    }
  }
#endif
  return SERQ_OK;
}

void free_ws(serq_linear* h) {
  for (void* p : {h->ws_x, (void*)h->ws_codes, (void*)h->ws_sf, h->ws_y, (void*)h->ws_xs, (void*)h->ws_xsf,
                  (void*)h->ws_s64, (void*)h->ws_s32, (void*)h->ws_zp})
    if (p) cudaFree(p);
  h->ws_x = h->ws_y = nullptr;
  h->ws_codes = h->ws_sf = h->ws_xs = h->ws_xsf = nullptr;
  h->ws_s64 = nullptr;
  h->ws_s32 = nullptr;
  h->ws_zp = nullptr;
  h->ws_m = 0;
}

int xs_kind_of(const serq_linear* h) {
  if (h->r_mode == SERQ_R_DENSE || h->r_mode == SERQ_R_DENSE_SPLIT) return 1;
  if (h->r_mode == SERQ_R_INT && !h->contiguous) return 2;
  return 0;
}

}  // namespace

extern "C" {

int serq_forward_mx_host(serq_linear_t* h, const void* x_host, int64_t M, void* y_host, serq_stream_t stream) {
  return serq_forward_mx_host_gather(h, x_host, M, nullptr, y_host, stream);
}

int serq_forward_mx_host_gather(serq_linear_t* h, const void* x_host, int64_t M, const int32_t* gather_idx,
                                void* y_host, serq_stream_t stream) {
  if (!h || h->mode != kModeMX) return fail(SERQ_EINVAL, "handle is not an MX linear");
  if (!x_host || !y_host) return fail(SERQ_EINVAL, "null host buffer");
  std::lock_guard<std::mutex> lock(h->e2e_mu);
  const bool gather = h->r > 0 && !h->contiguous;
  if (gather && !gather_idx)
    return fail(SERQ_EINVAL, "a non-contiguous salient set needs gather_idx (serq_forward_mx_host_gather)");
  if (M <= 0) return fail(SERQ_EINVAL, "x must be non-empty");
  if (M > h->ws_m || (gather && !h->ws_xs)) {
    const int64_t mm = cdiv(M > h->ws_m ? M : h->ws_m, 128) * 128;
    free_ws(h);
    CK(cudaMalloc(&h->ws_x, mm * h->K * 2));
    CK(cudaMalloc(&h->ws_codes, mm * h->K / 2));
    CK(cudaMalloc(&h->ws_sf, sf_bytes_of(mm, h->K)));
    CK(cudaMalloc(&h->ws_y, mm * h->N * 2));
    if (gather) {
      CK(cudaMalloc(&h->ws_xs, mm * xs_cols_of(h) / 2));
      CK(cudaMalloc(&h->ws_xsf, sf_bytes_of(mm, xs_cols_of(h))));
    }
    h->ws_m = mm;
  }
  const int64_t xc = xs_cols_of(h);
  const int64_t kc_pad = kc_pad_of(h->K), kc_pad_r = gather ? kc_pad_of(xc) : 0;
  return host_pipeline(h, x_host, M, y_host, S(stream), [&](int64_t r0, int64_t mc) {
    // chunks start on 256-row boundaries, so their scale-factor tiles start on row-block boundaries
    uint8_t* codes = h->ws_codes + r0 * h->K / 2;
    uint8_t* sf = h->ws_sf + (r0 / 128) * kc_pad * 512;
    uint8_t* xs = gather ? h->ws_xs + r0 * xc / 2 : nullptr;
    uint8_t* xsf = gather ? h->ws_xsf + (r0 / 128) * kc_pad_r * 512 : nullptr;
    int rc = serq_act_quant_mx(static_cast<uint8_t*>(h->ws_x) + r0 * h->K * 2, SERQ_BF16, mc, h->K, h->K, codes, sf,
                               gather ? gather_idx : nullptr, gather ? int(xc) : 0, xs, xsf, stream);
    if (rc) return rc;
    const int n1 = g_launches;
    rc = serq_linear_mx(h, codes, sf, mc, xs, xsf, static_cast<uint8_t*>(h->ws_y) + r0 * h->N * 2, h->N, stream);
    g_launches += n1;
    return rc;
  });
}

int serq_forward_int(serq_linear_t* h, const void* x, int dtype, int64_t M, int64_t ldx, int bits, int symmetric,
                     const int32_t* salient_idx, int8_t* codes, double* scale64, float* scale32, int32_t* zp,
                     void* xs, void* y, int64_t ldy, serq_stream_t stream) {
  if (!h || h->mode != kModeI8) return fail(SERQ_EINVAL, "handle is not an INT linear");
  const int xk = xs_kind_of(h);
  if (xk && !xs) return fail(SERQ_EINVAL, "this R mode needs the xs buffer (serq_act_quant_int xs_out)");
  if (xk == 2 && !salient_idx) return fail(SERQ_EINVAL, "a non-contiguous salient set needs salient_idx");
  if (!symmetric && !zp) return fail(SERQ_EINVAL, "asymmetric quantization needs a zero-point buffer");
  int rc = serq_act_quant_int(x, dtype, M, h->K, ldx, bits, symmetric, codes, scale64, scale32, symmetric ? nullptr : zp,
                              xk ? (h->contiguous ? nullptr : salient_idx) : nullptr, xk ? h->r : 0, xs, xk, stream);
  if (rc) return rc;
  const int n1 = g_launches;
  rc = linear_int_impl(h, codes, scale32, symmetric ? nullptr : zp, M, xs, y, ldy, nullptr, nullptr, nullptr, stream);
  g_launches += n1;
  return rc;
}

int serq_forward_int_host(serq_linear_t* h, const void* x_host, int64_t M, int bits, int symmetric,
                          const int32_t* salient_idx, void* y_host, serq_stream_t stream) {
  if (!h || h->mode != kModeI8) return fail(SERQ_EINVAL, "handle is not an INT linear");
  if (!x_host || !y_host) return fail(SERQ_EINVAL, "null host buffer");
  if (M <= 0) return fail(SERQ_EINVAL, "x must be non-empty");
  const int xk = xs_kind_of(h);
  if (xk == 2 && !salient_idx) return fail(SERQ_EINVAL, "a non-contiguous salient set needs salient_idx");
  std::lock_guard<std::mutex> lock(h->e2e_mu);
  const int64_t xs_row = xk == 1 ? 2 * int64_t(h->r) : (xk == 2 ? int64_t(h->r) : 0);  // bytes per row
  if (M > h->ws_m || !h->ws_s64) {
    const int64_t mm = cdiv(M > h->ws_m ? M : h->ws_m, 128) * 128;
    free_ws(h);
    CK(cudaMalloc(&h->ws_x, mm * h->K * 2));
    CK(cudaMalloc(&h->ws_codes, mm * h->K));
    CK(cudaMalloc(&h->ws_s64, mm * 8));
    CK(cudaMalloc(&h->ws_s32, mm * 4));
    CK(cudaMalloc(&h->ws_zp, mm * 4));
    CK(cudaMalloc(&h->ws_y, mm * h->N * 2));
    if (xs_row) CK(cudaMalloc(&h->ws_xs, mm * xs_row));
    h->ws_m = mm;
  }
  return host_pipeline(h, x_host, M, y_host, S(stream), [&](int64_t r0, int64_t mc) {
    return serq_forward_int(h, static_cast<uint8_t*>(h->ws_x) + r0 * h->K * 2, SERQ_BF16, mc, h->K, bits, symmetric,
                            salient_idx, reinterpret_cast<int8_t*>(h->ws_codes) + r0 * h->K, h->ws_s64 + r0,
                            h->ws_s32 + r0, h->ws_zp + r0, xs_row ? h->ws_xs + r0 * xs_row : nullptr,
                            static_cast<uint8_t*>(h->ws_y) + r0 * h->N * 2, h->N, stream);
  });
}

}  // extern "C"
