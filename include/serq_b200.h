/* serq_b200.h -- C ABI of the B200-native SERQ quantized-linear hot path.
 *
 * Plain pointers, sizes and a CUDA stream; no torch types.  All device
 * pointers are caller-owned unless stated.  Every entry point returns 0 on
 * success, SERQ_EINVAL for a violated precondition (the Python mirror raises
 * ValidationError, as the reference does in _validation.py:14-15) or
 * SERQ_ECUDA for a CUDA failure; serq_last_error() gives a thread-local
 * message.  Work is stream-ordered; nothing blocks the host except the
 * *_host entry points, which synchronise `stream` before returning.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/serq):
 *   serq_act_quant_mx      mx_encode + _block_exponents + e2m1_nearest   mxfmt.py:52-108
 *                          and the salient re-encode in _forward_mx      compensate.py:335
 *   serq_act_quant_int     quantize_symmetric / quantize_asymmetric      quantcore.py:108-137
 *                          + gather_columns (salient slice)              quantcore.py:158-175
 *   serq_pack_mx           MxBlockTensor artefacts (main_t, comp.r_q)     mxfmt.py:34-49, compensate.py:343-357
 *   serq_unpack_mx         inverse of the device layout (artefact export)
 *   serq_rmsnorm_quant_mx  rmsnorm(x, gain) -> mx_encode, fused        saliency.py:194-196, mxfmt.py:97-108
 *   serq_rmsnorm_quant_mx_gather  ... + the salient gather x[:, idx]   compensate.py:335
 *   serq_mx_container_decode  load_mx body -> codes / exponents on the device  mxfmt.py:254-280
 *   serq_pack_int          QuantizedTensor artefacts (main, comp.r_q / comp.r_dense)
 *                                                                         quantcore.py:59-80, compensate.py:48-69
 *   serq_linear_mx         _forward_mx: mx_gemm_reference(x,W)+mx_gemm_reference(xs,R)
 *                                                                         compensate.py:319-340, mxfmt.py:198-225
 *   serq_pack_int_grouped  row-grouped (group_size g) QuantizedTensor main     mxfmt.py:177-195, gptq.py:98-146
 *   serq_linear_int        forward_reconstructed int branch: int_gemm_reference(xq, main)
 *                          + R term (int_gemm_reference(xs, r_q) or dequantize(xs) @ r_dense)
 *                                                                         compensate.py:300-316, mxfmt.py:135-195
 *   serq_linear_int_addend forward_reconstructed int branch, SVD baseline: int_gemm + (x_hat L1) L2
 *                                                                         compensate.py:300-310
 *   serq_mx_decode_bf16    mx_decode of a device MX activation -> bf16 (exact) mxfmt.py:111-113
 *   serq_linear_mx_addend  _forward_mx, SVD baseline: mx_gemm_reference(x, main) + (x_hat L1) L2
 *                                                                         compensate.py:319-331
 *   serq_forward_mx        forward_reconstructed(x, main_t, comp, None) on device: mx_encode(x)
 *                          (+ re-encode of x[:, idx]) then the fused GEMM      compensate.py:319-340
 *   serq_forward_mx_host   forward_reconstructed(x, main_t, comp, None) end to end from host memory
 *                                                                         compensate.py:272-295
 *   serq_forward_int       forward_reconstructed(x, main, comp, act_cfg) on device: quantize_asymmetric
 *                          (or _symmetric) per token + gather_columns + the fused integer GEMM
 *                                                                         compensate.py:296-316
 *   serq_forward_int_host  the same end to end from host memory            compensate.py:272-316
 */
#ifndef SERQ_B200_H
#define SERQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SERQ_OK 0
#define SERQ_EINVAL 1
#define SERQ_ECUDA 2

/* input element types for the quantizers */
#define SERQ_BF16 0
#define SERQ_F32 1
#define SERQ_F64 2

/* compensation-matrix modes for the integer path */
#define SERQ_R_NONE 0
#define SERQ_R_DENSE 1 /* comp.r_dense: float64 [r, N], consumed as bf16 */
#define SERQ_R_INT 2   /* comp.r_q: int codes [r, N] with one scale per output column */
#define SERQ_R_DENSE_SPLIT 3 /* float64 [r, N] consumed as bf16 hi + bf16 lo (relative error 2^-17):
                              * dequantize(r_q) of a column-grouped R (default_r_config), a GPTQ-swapped
                              * R, or an f64 r_dense; serq_pack_int_grouped only */

typedef struct serq_linear serq_linear_t; /* packed weight handle (opaque) */
typedef void* serq_stream_t;              /* cudaStream_t */

const char* serq_last_error(void);
const char* serq_version(void);
int serq_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* Bytes of the device MX activation buffers for an [rows, cols] matrix. */
int serq_mx_sizes(int64_t rows, int64_t cols, int64_t* codes_bytes, int64_t* sf_bytes);

/* K1-MX: X [M, K] (row stride ldx elements) -> packed E2M1 codes [M, K/2] and
 * tiled E8M0 scale factors.  If gather_idx != NULL, also encodes the salient
 * slice X[:, gather_idx[0..r)] into xs_codes [M, r/2] / xs_sf (the reference
 * re-encodes the gathered columns, compensate.py:335).  K % 32 == 0, r % 32 == 0. */
int serq_act_quant_mx(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, uint8_t* codes, uint8_t* sf,
                      const int32_t* gather_idx, int r, uint8_t* xs_codes, uint8_t* xs_sf, serq_stream_t stream);

/* K1-INT: per-token quantization (bits in [2, 8]).  codes int8 [M, K] (u8 bit
 * patterns when asymmetric), scale64/scale32 [M], zp [M] (asymmetric only; may
 * be NULL when symmetric).  xs_kind: 0 none; 1 write xs_out bf16 [M, r] =
 * codes[:, idx] - zp (dense-R operand); 2 write xs_out int8 [M, r] = codes[:, idx].
 * salient_idx == NULL means idx = arange(r). */
int serq_act_quant_int(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, int bits, int symmetric,
                       int8_t* codes, double* scale64, float* scale32, int32_t* zp, const int32_t* salient_idx, int r,
                       void* xs_out, int xs_kind, serq_stream_t stream);

/* K-sharded integer activations (row-parallel INT layers): the per-token scale
 * spans the FULL row (quantcore.py:127-129), so each rank first writes its K-slice's row
 * range -- range float [2, M]: range[m] = min, range[M + m] = max (exact: bf16 values) --
 * the ranks all-reduce MIN over range[0:M] and MAX over range[M:2M], and then quantize their
 * slice with serq_act_quant_int_ext on the global range: codes, scales and zero points equal
 * serq_act_quant_int of the unsharded row.  bf16 input, K % 8 == 0, K <= 16384. */
int serq_act_quant_int_range(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, float* range,
                             serq_stream_t stream);
int serq_act_quant_int_ext(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, int bits, int symmetric,
                           const float* range, int8_t* codes, double* scale64, float* scale32, int32_t* zp,
                           const int32_t* salient_idx, int r, void* xs_out, int xs_kind, serq_stream_t stream);

/* Pack MX artefacts held in DEVICE memory, reference layouts:
 * codes uint8 [N, K] (values 0..15), exps int32 [N, K/32] (main_t of
 * build_serq_rtn_mx, stored transposed), r_codes uint8 [N, r], r_exps int32
 * [N, r/32] (comp.r_q) or NULL with r == 0.  salient_contiguous != 0 when
 * salient_idx == arange(r) (permuted layout: the salient slice is read from
 * the leading columns of X, no re-encode). */
int serq_pack_mx(const uint8_t* codes, const int32_t* exps, int64_t N, int64_t K, const uint8_t* r_codes,
                 const int32_t* r_exps, int r, int salient_contiguous, serq_linear_t** out, serq_stream_t stream);

/* Inverse of the device MX layout for an activation/weight buffer pair. */
/* Producer fusion: y = x / sqrt(mean(x^2) + eps) * gain
 * (saliency.py:194-196; gain = the RMSNorm weight with the SAF scales folded in,
 * toymodel.py:203-217) encoded straight to MX codes / scale factors in the
 * serq_act_quant_mx layout.  x bf16/f32 [M, K] (16-B aligned rows), gain f64 [K]
 * and its f32 rounding gain32 [K] (16-B aligned).  Codes equal mx_encode of the
 * reference's f64 result: an f32 fast path with a proven error bound, and the
 * reference's f64 operations for any 32-block the bound cannot decide.  K <= 8192. */
int serq_rmsnorm_quant_mx(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, const double* gain,
                          const float* gain32, double eps, uint8_t* codes, uint8_t* sf, serq_stream_t stream);

/* serq_rmsnorm_quant_mx plus the gather fallback (compensate.py:335): the
 * normalised salient slice rmsnorm(x)[:, gather_idx] (int32 [r], r % 32 == 0, r <= 1024)
 * is encoded in the same kernel into xs_codes [M, r/2] / xs_sf (serq_act_quant_mx's xs
 * layout); gather_idx NULL = serq_rmsnorm_quant_mx. */
int serq_rmsnorm_quant_mx_gather(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, const double* gain,
                                 const float* gain32, double eps, const int32_t* gather_idx, int r, uint8_t* codes,
                                 uint8_t* sf, uint8_t* xs_codes, uint8_t* xs_sf, serq_stream_t stream);

/* Producer fusion for the integer formats: rmsnorm(x, gain) (saliency.py:194-196) quantized per
 * token (quantcore.py:108-137) in one kernel, in float64 exactly as the reference -- including
 * NumPy's pairwise summation order for the row mean of squares, replayed from the row length --
 * so codes, scales and zero points equal quantize_*(rmsnorm(x)) bit for bit.  x bf16 / f32 [M, K]
 * (K <= 8192), gain f64 [K] and its f32 rounding gain32 (16-byte aligned; the fast kernel's f32
 * pass, exactness kept by an error bound -- NULL selects the all-f64 kernel); outputs and xs
 * as serq_act_quant_int. */
int serq_rmsnorm_quant_int(const void* x, int dtype, int64_t M, int64_t K, int64_t ldx, const double* gain,
                           const float* gain32, double eps, int bits, int symmetric, int8_t* codes, double* scale64,
                           float* scale32, int32_t* zp, const int32_t* salient_idx, int r, void* xs_out, int xs_kind,
                           serq_stream_t stream);

/* Decoder-block glue for decode-sized token counts (toy_block_graph, toymodel.py:88-124; the
 * non-SERQ nodes, f32): res = x (+ o, bf16 [M, ldo], may be NULL), h = rmsnorm(res) * gain
 * (saliency.py:194-196; res may be NULL; h NULL: the residual add alone into res); mid = silu(gate) * up (saliency.py:199-200; bf16 in,
 * f32 out); and the token-batch attention (attention_mix, saliency.py:203-216) over M <= 16
 * tokens, head_dim 128, reading q / k / v rows in place (e.g. column views of the fused q/k/v
 * output).  All float32 row-major [M, H] unless a pitch is given. */
int serq_block_add_rmsnorm(const float* x, const void* o, int64_t ldo, int64_t M, int64_t H, const float* gain,
                           float eps, float* res, float* h, serq_stream_t stream);
int serq_block_silu_mul(const void* gate, int64_t ldg, const void* up, int64_t ldu, int64_t M, int64_t F, float* mid,
                        serq_stream_t stream);
int serq_block_attention(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, int64_t M,
                         int64_t heads, int64_t head_dim, float scale, float* out, int64_t ldo, serq_stream_t stream);

/* The reference's packed MX file body/* The reference's packed MX file body (mxfmt.py:228-251, after the 28-byte
 * header; bundleio.py load path): rows x cols/32 records of 17 bytes (exponent
 * byte e+127, 16 nibble bytes, element 2i low) already in device memory ->
 * element codes uint8 [rows, cols] (16-B aligned) and exponents int32
 * [rows, cols/32], the serq_pack_mx inputs.  Replaces load_mx's per-block loop. */
int serq_mx_container_decode(const uint8_t* body, int64_t rows, int64_t cols, uint8_t* codes, int32_t* exps,
                             serq_stream_t stream);

int serq_unpack_mx(const uint8_t* codes_packed, const uint8_t* sf, int64_t rows, int64_t cols, uint8_t* codes,
                   int32_t* exps, serq_stream_t stream);

/* mx_decode (mxfmt.py:111-113) of a device MX tensor: bf16 [rows, cols] (16-B aligned) of
 * e2m1(code) * 2^e, exact in bf16.  The SVD baseline's x_hat (compensate.py:327). */
int serq_mx_decode_bf16(const uint8_t* codes_packed, const uint8_t* sf, int64_t rows, int64_t cols, void* out,
                        serq_stream_t stream);

/* Pack INT artefacts held in DEVICE memory, reference layouts: codes int32
 * [K, N] (main.codes), scales float64 [N] (main.scales, one group: group_size
 * == K, axis 'row').  r_mode SERQ_R_DENSE: r_data = float64 [r, N] (r_dense);
 * SERQ_R_INT: r_data = int32 [r, N] codes with r_scales float64 [N].
 * a_bits/a_symmetric describe the activation quantizer the handle expects. */
int serq_pack_int(const int32_t* codes, const double* scales, int64_t K, int64_t N, int w_bits, int r_mode,
                  const void* r_data, const double* r_scales, int r, int salient_contiguous, serq_linear_t** out,
                  serq_stream_t stream);

/* serq_pack_int with the weights held as PACKED INT4 in HBM (0.5 B / weight; w_bits <= 4):
 * the CTA-pair kernel's loader warps widen the nibbles to int8 in shared memory (Blackwell has
 * no INT4 MMA).  Needs a layout that kernel serves: R permuted-integer (r <= 128), dense
 * (r <= 64) or none.  Bit-identical results to serq_pack_int's int8 weights; serq_pack_int
 * remains the default because its TMA feed is faster today (K3). */
int serq_pack_int4(const int32_t* codes, const double* scales, int64_t K, int64_t N, int w_bits, int r_mode,
                   const void* r_data, const double* r_scales, int r, int salient_contiguous, serq_linear_t** out,
                   serq_stream_t stream);

/* Group-wise integer weights (int_gemm_reference row-grouped
 * branch, mxfmt.py:177-195; GPTQ group_size, gptq.py:98-146; _weight_config,
 * pipeline.py:134-137): scales float64 [K/group_size, N] (main.scales of a
 * row-grouped QuantizedTensor), group_size a multiple of 128 and <= 8192 that
 * divides K (one integer partial per group stays exact in fp32); group_size == K is serq_pack_int.  R as in serq_pack_int.
 * serq_linear_int on such a handle promotes one integer partial per group. */
int serq_pack_int_grouped(const int32_t* codes, const double* scales, int64_t group_size, int64_t K, int64_t N,
                          int w_bits, int r_mode, const void* r_data, const double* r_scales, int r,
                          int salient_contiguous, serq_linear_t** out, serq_stream_t stream);

/* Fused linears (SURVEY 7 hard-part 6; e.g. q/k/v or gate/up, which read the same activation but
 * have their own salient sets): an MX handle packed from the row-concatenated artefacts of nseg
 * linears (seg_rows[j] output rows each, multiples of 128, summing to N) runs them as ONE kernel.
 * The quantizer's salient buffer then holds 128 columns per segment: gather_idx (length
 * 128 * nseg) lists segment j's r indices at [128 j, 128 j + r), any valid index after them.
 * One kernel covers M <= 16 (decode) and M > 128 with r = 64 and 256-row-aligned segments;
 * other shapes return SERQ_EINVAL -- run them through per-segment views. */
int serq_linear_set_segments(serq_linear_t* h, int nseg, const int64_t* seg_rows);
/* A handle over output rows [row0, row0 + rows) of an MX handle (128-row aligned): no copy, the
 * parent owns the weights and must outlive the view; salient_contiguous as for serq_pack_mx. */
int serq_linear_view(const serq_linear_t* parent, int64_t row0, int64_t rows, int salient_contiguous,
                     serq_linear_t** out);

int serq_linear_destroy(serq_linear_t* h);
int serq_linear_info(const serq_linear_t* h, int64_t* N, int64_t* K, int* r, int* mode, int* r_mode);
/* Bytes of the resident main weights (padding included) and whether they are held as packed
 * 4-bit codes (MXFP4 always; INT when the handle is served by the CTA-pair kernel, which
 * widens packed INT4 in the SM -- 8-bit codes and the other INT layouts keep int8). */
int serq_linear_weight_bytes(const serq_linear_t* h, int64_t* main_bytes, int* packed_int4);

/* K2: Y[M, N] (bf16, row stride ldy) = Xq.Wq + Xs,q.R in one kernel.  a_codes /
 * a_sf from serq_act_quant_mx; xs_codes / xs_sf only for a non-contiguous
 * salient set (NULL otherwise). */
int serq_linear_mx(const serq_linear_t* h, const uint8_t* a_codes, const uint8_t* a_sf, int64_t M,
                   const uint8_t* xs_codes, const uint8_t* xs_sf, void* y, int64_t ldy, serq_stream_t stream);

/* K3: integer path.  a_codes int8 [M, K]; sx [M] f32; zp [M] or NULL (symmetric
 * activations); xs = the quantizer's xs_out (dense R, or gathered codes for a
 * non-contiguous int R) or NULL.  acc_dump / accr_dump (int32 [M, N], optional)
 * receive the exact integer accumulators sum (c - zp) * w. */
int serq_linear_int(const serq_linear_t* h, const int8_t* a_codes, const float* sx, const int32_t* zp, int64_t M,
                    const void* xs, void* y, int64_t ldy, int32_t* acc_dump, int32_t* accr_dump, serq_stream_t stream);

/* Quantize + linear in one call (compensate.py:319-340 _forward_mx): x (bf16 /
 * f32 / f64 [M, K], row pitch ldx elements) -> codes / sf (serq_act_quant_mx
 * layout, caller-allocated) -> y.  The linear is launched with programmatic
 * dependent launch so its prologue and weight stream overlap the quantizer.
 * gather_idx / xs_codes / xs_sf are needed only for a non-contiguous salient set. */
int serq_forward_mx(serq_linear_t* h, const void* x, int dtype, int64_t M, int64_t ldx, const int32_t* gather_idx,
                    uint8_t* codes, uint8_t* sf, uint8_t* xs_codes, uint8_t* xs_sf, void* y, int64_t ldy,
                    serq_stream_t stream);

/* K3 with an fp32 addend C [M, N] (row pitch N) summed into the output before the
 * bf16 store: y = bf16(sx * (sw * acc (+ R term)) + C).  Serves the SVD baseline
 * (compensate.py:304-310), whose two-factor correction (x_hat @ L1) @ L2 spans all
 * K columns and so cannot ride in the fused salient term. */
int serq_linear_int_addend(const serq_linear_t* h, const int8_t* a_codes, const float* sx, const int32_t* zp,
                           int64_t M, const void* xs, const float* addend, void* y, int64_t ldy,
                           serq_stream_t stream);

/* K2 with an fp32 addend C [M, N] (row pitch N, 16-B aligned) summed into the fp32 accumulator before the
 * bf16 store: y = bf16(mx_gemm(x, main) + C).  The MX SVD baseline (compensate.py:326-331);
 * the handle must carry no salient term (r = 0).  M > 16: the CTA-pair kernel; smaller M
 * the one-CTA persistent kernel. */
int serq_linear_mx_addend(const serq_linear_t* h, const uint8_t* a_codes, const uint8_t* a_sf, int64_t M,
                          const float* addend, void* y, int64_t ldy, serq_stream_t stream);

/* End to end from HOST memory (pinned for full PCIe rate): copy X (bf16 [M, K])
 * in, quantize, GEMM, copy Y (bf16 [M, N]) out; synchronises `stream`.
 * Device scratch lives in the handle and grows on demand. */
int serq_forward_mx_host(serq_linear_t* h, const void* x_host, int64_t M, void* y_host, serq_stream_t stream);
/* serq_forward_mx_host for a non-contiguous salient set: gather_idx (device int32 [r]) as in
 * serq_forward_mx; the salient slice is re-encoded per chunk on the device. */
int serq_forward_mx_host_gather(serq_linear_t* h, const void* x_host, int64_t M, const int32_t* gather_idx,
                                void* y_host, serq_stream_t stream);

/* Integer quantize + linear in one call (compensate.py:296-316, the int branch of
 * forward_reconstructed): x (bf16 / f32 / f64 [M, K], row pitch ldx) -> per-token codes /
 * scales / zero points (serq_act_quant_int layout, caller-allocated; zp unused and may be
 * NULL when symmetric) -> y bf16 [M, N] (pitch ldy).  xs: the salient slice buffer the
 * handle's R needs (bf16 [M, r] for a dense R, int8 [M, r] for an integer R on a
 * non-contiguous salient set, else NULL); salient_idx (device int32 [r]) only for a
 * non-contiguous salient set.  The linear is PDL-chained to the quantizer. */
int serq_forward_int(serq_linear_t* h, const void* x, int dtype, int64_t M, int64_t ldx, int bits, int symmetric,
                     const int32_t* salient_idx, int8_t* codes, double* scale64, float* scale32, int32_t* zp,
                     void* xs, void* y, int64_t ldy, serq_stream_t stream);

/* serq_forward_int end to end from HOST memory: X bf16 [M, K] in, Y bf16 [M, N] out (pinned
 * for full PCIe rate), pipelined over token chunks on two copy streams; device scratch in the
 * handle; synchronises `stream`. */
int serq_forward_int_host(serq_linear_t* h, const void* x_host, int64_t M, int bits, int symmetric,
                          const int32_t* salient_idx, void* y_host, serq_stream_t stream);

/* Number of kernels the last forward on this thread launched (evidence for bench). */
int serq_last_launch_count(void);
/* Name of the last kernel launched on this thread, e.g. "serq_i8_pair_kernel<256>"
 * (tests assert which kernel a configuration takes). */
const char* serq_last_kernel(void);

/* Diagnostics, SERQ_DIAG builds only (tools/): kernel-selection and feed/MMA
 * isolation switches (results are WRONG while set).  The product library has no
 * such state: it returns SERQ_EINVAL for any nonzero value. */
int serq_set_debug_flags(int flags);
/* Diagnostics (SERQ_DIAG_TS builds only): device buffer receiving clock / globaltimer
 * stamps of the linears' pipelines, or NULL.  SERQ_EINVAL for non-NULL otherwise. */
int serq_set_debug_timestamps(long long* dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* SERQ_B200_H */
