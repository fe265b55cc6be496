/*
 * ifa_b200.h -- C-ABI of the B200-native INT-FlashAttention hot path.
 *
 * Drop-in boundary for the reference's CPU path (/root/reference/proj):
 *
 *   ifa_quantize_per_row      replaces ifa::quantize_per_row
 *                             (include/ifa/quant.hpp:30, src/quant.cpp:44-57)
 *   ifa_quantize_per_tensor   replaces ifa::quantize_per_tensor applied per (b,h)
 *                             slice (include/ifa/quant.hpp:33, src/quant.cpp:59-69,
 *                             caller src/eval.cpp:101)
 *   ifa_int_flash_fwd         replaces ifa::int_flash_attention
 *                             (include/ifa/attention.hpp:85-87,
 *                             src/attention.cpp:235-357), batched over slices
 *   ifa_*_host                the same three entry points with HOST buffers and
 *                             the reference's synchronous calling convention
 *                             (copies + kernels + copies on one stream, then a
 *                             synchronize) -- what a CPU caller such as
 *                             eval.cpp:98-102 or the verify hook binds
 *   ifa_last_error            replaces the what() of the C++ exceptions the
 *                             reference throws (std::invalid_argument /
 *                             std::overflow_error)
 *
 * Layout (reference include/ifa/matrix.hpp:16-90): every
 * matrix is row-major and contiguous.  A batch of (b,h) slices is
 * [slices][n][d] with no padding.  Q/K per-row scales are [slices][n] f32,
 * the V tensor-level scale is one f32 per slice ([slices]), O is f32
 * [slices][n][d].  Codes are int8 in [-127, 127].
 *
 * All pointers are DEVICE pointers on the current CUDA device unless stated
 * otherwise; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Calls are asynchronous on `stream` and reentrant per stream.  Return
 * values: 0 on success, otherwise one of the IFA_E* codes below with a
 * message retrievable through ifa_last_error() (thread-local).
 */
#ifndef IFA_B200_H
#define IFA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IFA_OK 0
#define IFA_EINVAL 22     /* std::invalid_argument in the reference       */
#define IFA_EOVERFLOW 75  /* std::overflow_error (int32 depth guard)      */
#define IFA_ENOTSUP 95    /* shape this build does not run on the GPU     */
#define IFA_ECUDA 1000    /* CUDA runtime / driver error                  */
#define IFA_EFORMAT 74    /* ifa::FormatError (malformed IFA1 tensor file) */

/* ifa_int_flash_fwd flags */
#define IFA_FLAG_SQRT_D 1u /* AttentionConfig::apply_sqrt_d_scaling (attention.hpp:25-27) */
#define IFA_FLAG_CAUSAL 2u /* extension (not in the reference): row i sees keys j <= i   */
/* Tolerance mode: the same per-block algorithm (Bc honoured, running-max
 * requantization, per-block float rescale) with one MUFU exp2 per code and no
 * exactness guard.  int8 codes, scales and int32 S are unaffected; O agrees
 * with the reference within the tolerance tests/test_gpu_parity.py states
 * (MRE <= 2e-5, max|dO| <= the reference's multi-block bound 2/127*max|V|*sV,
 * verify.cpp:65-70).  Ignored when an audit is requested. */
#define IFA_FLAG_FAST 4u

/* Device-resident mirror of ifa::PCodeAudit (attention.hpp:75-80).  Before
 * a call the struct must hold {127, 0, 1, 0, 0} (ifa_audit_init()); the
 * kernel folds its observations into it. */
typedef struct ifa_pcode_audit {
    int32_t min_code;
    int32_t max_code;
    int32_t row_max_block_hits_127; /* bool */
    int32_t reserved;
    int64_t rows_audited;
} ifa_pcode_audit;

/* Largest reduction depth for which k*127*127 < 2^31 (gemm.hpp:22). */
#define IFA_MAX_INT_GEMM_DEPTH 133144

/* Per-token quantization: codes[r][c] = round(x[r][c] / scales[r]) with
 * scales[r] = max|x[r][:]| / 127 (all-zero row -> scale 0, codes 0).
 * nonfinite_index (device, optional): if non-NULL it must hold INT64_MAX
 * before the call and receives the smallest flat index of a NaN/Inf input
 * (the reference rejects such input, quant.cpp:14-22). */
int ifa_quantize_per_row(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                         float* scales, int64_t* nonfinite_index, void* stream);

/* Tensor-level quantization applied independently to each of `slices`
 * matrices of rows x cols: one scale per slice (slice_scales[s]).
 * workspace: device buffer of >= 4*slices bytes (scratch). */
int ifa_quantize_per_tensor(const float* x, int64_t slices, int64_t rows, int64_t cols,
                            int8_t* codes, float* slice_scales, void* workspace,
                            int64_t* nonfinite_index, void* stream);

/* Full-INT8 flash attention forward over `slices` independent (b,h) slices
 * of n x d (self-attention: N_q = N_kv = n).
 *   br: the reference's row-block size; results do not depend on it
 *       (accepted and validated for drop-in fidelity).
 *   bc: KV block size; honoured exactly (it changes results).
 *   audit: optional device ifa_pcode_audit.
 * sv values must be finite and >= 0 (validated by the host shims; the
 * reference rejects them in QuantizedAttentionInputs::validate).
 * Supported on the GPU: 1 <= d <= 133144 (the reference's int32 depth limit,
 * gemm.hpp:22), n >= 1, bc >= 1.  d > 128 runs the general kernel with S
 * accumulated over 128-column depth chunks and one launch per 128 columns of
 * O (attn.cu launch_wide). */
int ifa_int_flash_fwd(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                      const int8_t* v, const float* sv, float* o, int64_t slices, int64_t n,
                      int64_t d, int64_t br, int64_t bc, uint32_t flags,
                      ifa_pcode_audit* audit, void* stream);

/* ---- int32 S / P-code dump (north_star: "int32 S tiles bit-exact") --------
 * ifa_int_flash_fwd_dump: ifa_int_flash_fwd in tolerance mode (flags must
 *   hold IFA_FLAG_FAST; Bc = 128, or Bc >= n <= 128) through a separate
 *   instantiation of the bench-default full-INT8 tolerance kernel
 *   (csrc/attn_pp.cu; csrc/attn_ws.cu with IFA_B200_WS=1) that also writes
 *     s_out   [slices][n][n] int32: S = Q.K^T of every KV tile the kernel
 *             computes, read back from the tcgen05 kind::i8 accumulator in
 *             TMEM -- the reference's int_gemm_nt_strided
 *             (attention.cpp:275-276 -> gemm.cpp:32-46, oracle
 *             oracles.cpp:28-43), bit-exact;
 *     p_codes [slices][n][n] uint8: the P codes round(127 exp(s - m_new))
 *             the kernel fed to P.V (attention.cpp:299-312); in tolerance
 *             mode a code may differ from the reference's by one where
 *             127 exp(.) lies within the exp2 estimate's error of .5.
 *   Either output may be NULL (not both).  With IFA_FLAG_CAUSAL only the KV
 *   tiles at or below the diagonal are written (entries above the diagonal
 *   inside the diagonal tile are S as computed, their P code 0).  O is
 *   written as by ifa_int_flash_fwd.  n <= 65536. */
#define IFA_FLAG_DUMP_S 8u
int ifa_int_flash_fwd_dump(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                           const int8_t* v, const float* sv, float* o, int64_t slices, int64_t n,
                           int64_t d, int64_t br, int64_t bc, uint32_t flags, int32_t* s_out,
                           uint8_t* p_codes, void* stream);

/* ---- fp16 V codes for the two-Q-tile tolerance kernel --------------------
 * ifa_quantize_per_tensor_v16: ifa_quantize_per_tensor that also writes the
 *   V codes as fp16 (codes_f16, same [slices][rows][cols] layout, exact),
 *   fused into the quantizer's second pass.
 * ifa_int_flash_fwd_v16: ifa_int_flash_fwd with those fp16 codes supplied,
 *   so the two-Q-tile kernel (IFA_FLAG_FAST, Bc = 128, n % 128 == 0, d in
 *   {64, 128}; csrc/attn_pp.cu) skips its own conversion.  Any other case
 *   runs exactly ifa_int_flash_fwd on the int8 v (no audit), which for other
 *   n converts V into a padded fp16 copy itself. */
int ifa_quantize_per_tensor_v16(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                int8_t* codes, uint16_t* codes_f16, float* slice_scales,
                                void* workspace, int64_t* nonfinite_index, void* stream);
int ifa_int_flash_fwd_v16(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                          const int8_t* v, const uint16_t* v_f16, const float* sv, float* o,
                          int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc,
                          uint32_t flags, void* stream);

/* ---- one whole step, quantization streamed into the attention -----------
 * ifa_int8_attention_step: quantize_per_row(Q), quantize_per_row(K),
 *   quantize_per_tensor(V) per slice (+ the fp16 V codes) and the tolerance
 *   attention, from f32 DEVICE q, k, v [slices][n][d] into the caller's code
 *   / scale buffers (same layouts as above) and o.  Results are exactly
 *   those of the separate calls.  When the two-Q-tile kernel applies
 *   (IFA_FLAG_FAST, non-causal, Bc = 128, n % 128 == 0, d in {64, 128}) the
 *   first slices (enough for the attention's first wave) are quantized on the
 *   whole GPU, then the quantizer runs on a few SMs (IFA_B200_QUANT_SMS,
 *   default 12) concurrently with the attention kernel on the rest, one
 *   whole slice per CTA: the attention waits per slice on a ready word in
 *   sync_ws instead of on the whole quantization.  Otherwise the calls run
 *   one after the other on `stream`.
 *   sync_ws: DEVICE uint32[2 * slices], zeroed before the first call and
 *   then owned by this sequence of calls; epoch: 1 on the first call, +1 on
 *   every later call with the same sync_ws.  nonfinite_index as for the
 *   quantizers (smallest flat index of a NaN/Inf in any of q, k, v). */
int ifa_int8_attention_step(const float* q, const float* k, const float* v, int8_t* qc,
                            float* sq, int8_t* kc, float* sk, int8_t* vc, float* sv,
                            uint16_t* v16, float* o, int64_t* nonfinite_index,
                            uint32_t* sync_ws, uint32_t epoch, int64_t slices, int64_t n,
                            int64_t d, int64_t br, int64_t bc, uint32_t flags, void* stream);

/* ---- half-INT8 attention ----------------------------
 * ifa_half_int8_fwd  replaces ifa::half_int8_attention (attention.hpp:93-96,
 *                    attention.cpp:359-399): int8 Q/K with per-row scales
 *                    (S exact int32 as above), float V and float weights.
 * v_f16: DEVICE [slices][n][d] IEEE fp16 copy of V (ifa_convert_f16); the
 * weights are fed to the tensor core as fp16 and accumulated in fp32.
 * Tolerance semantics (tests/test_gpu_half.py): MRE against the reference
 * <= 2e-3, and the error against fp64 within 1% of the reference's own.
 * br/bc are validated as in the reference but only change float rounding
 * order there, so the kernel tiles 128 x 128 regardless.  flags: SQRT_D
 * only (the reference has no causal half-INT8 path).  Supported: d in {64,
 * 128}; others return IFA_ENOTSUP. */
int ifa_half_int8_fwd(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                      const uint16_t* v_f16, float* o, int64_t slices, int64_t n, int64_t d,
                      int64_t br, int64_t bc, uint32_t flags, void* stream);
/* DEVICE x[count] f32 -> out[count] fp16 (round to nearest even). */
int ifa_convert_f16(const float* x, int64_t count, uint16_t* out, void* stream);

/* ---- FP8 e4m3 baseline --------------------------------
 * ifa_fp8_quantize_per_tensor  replaces fp8_e4m3_roundtrip (fp8.cpp:78-97)
 *   per [rows x cols] slice: s = 448 / max|x|, codes = e4m3(x * s) (bitwise
 *   the reference's e4m3_encode), slice_scales[s] = s (0 for an all-zero
 *   slice); decoded_f16 (optional) receives decode(code) as fp16 (exact).
 *   workspace: DEVICE uint32[slices].  Non-finite input: *nonfinite_index.
 * ifa_fp8_attention_fwd  replaces fp8_emulated_attention
 *   (attention.cpp:401-407): S = Q8.K8^T on tcgen05.mma kind::f8f6f4, s =
 *   S / (sQ sK) [* 1/sqrt(d)], float online softmax, P (fp16) . V (decoded
 *   e4m3 as fp16), O / (l * sV).  Tolerance semantics as the half-INT8 path
 *   (tests/test_gpu_fp8.py).  d in {64, 128}; flags: SQRT_D only. */
int ifa_fp8_quantize_per_tensor(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                uint8_t* codes, uint16_t* decoded_f16, float* slice_scales,
                                void* workspace, int64_t* nonfinite_index, void* stream);
int ifa_fp8_attention_fwd(const uint8_t* q, const float* q_scales, const uint8_t* k,
                          const float* k_scales, const uint16_t* v_f16, const float* v_scales,
                          float* o, int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc,
                          uint32_t flags, void* stream);

/* ---- host-buffer forms (drop-in for synchronous CPU callers) -------------
 * Same arguments as above, but every array is HOST memory (pageable or
 * pinned) and the call returns after the results are back on the host.
 * Device memory comes from a per-thread grow-only workspace.  The quantizers
 * reject non-finite input like require_finite (quant.cpp:14-22): IFA_EINVAL,
 * message "<fn>: non-finite input at index <i>", *nonfinite_index = i (or
 * INT64_MAX); codes/scales are still written.  ifa_int_flash_fwd_host also
 * rejects sv[s] < 0 or non-finite ("quantized attention inputs: bad v
 * scale", attention.cpp:229-231) and, when `audit` (HOST) is non-NULL,
 * initialises it to {127, 0, 1, 0, 0} itself. */
int ifa_quantize_per_row_host(const float* x, int64_t rows, int64_t cols, int8_t* codes,
                              float* scales, int64_t* nonfinite_index, void* stream);
int ifa_quantize_per_tensor_host(const float* x, int64_t slices, int64_t rows, int64_t cols,
                                 int8_t* codes, float* slice_scales, int64_t* nonfinite_index,
                                 void* stream);
int ifa_int_flash_fwd_host(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                           const int8_t* v, const float* sv, float* o, int64_t slices,
                           int64_t n, int64_t d, int64_t br, int64_t bc, uint32_t flags,
                           ifa_pcode_audit* audit, void* stream);

/* The reference's full-INT8 evaluation step (eval.cpp:98-102, run_variant):
 * quantize_per_row(Q), quantize_per_row(K), quantize_per_tensor(V) per
 * slice, then int_flash_attention -- from f32 HOST Q, K, V [slices][n][d]
 * to f32 HOST O.  flags as ifa_int_flash_fwd (IFA_FLAG_FAST selects the
 * tolerance kernel).  Non-finite input: IFA_EINVAL "full_int8_attention:
 * <q|k|v>: non-finite input at index <flat index>" (quant.cpp:14-22).
 *
 * Both host-buffer attention entry points run as a chunked pipeline over
 * the slices: three streams overlap the host->device copy of one chunk, the
 * kernels of the previous one and the device->host copy of the one before
 * (PCIe is full duplex).  Pinned caller memory (cudaMallocHost /
 * cudaHostRegister) is copied by DMA directly; pageable memory is staged
 * through pinned buffers with multi-threaded memcpy. */
int ifa_full_int8_attention_host(const float* q, const float* k, const float* v, float* o,
                                 int64_t slices, int64_t n, int64_t d, int64_t br, int64_t bc,
                                 uint32_t flags, void* stream);

/* Host-buffer forms of the §8(f) variants (what include/ifa_b200.hpp's
 * ifa_gpu::half_int8_attention / fp8_emulated_attention call):
 *   ifa_half_int8_fwd_host: int8 Q/K codes + per-row scales and f32 V (host)
 *     -> f32 O (host); V is converted to fp16 on the device.  |V| > 65504
 *     (outside fp16) is rejected with IFA_EINVAL instead of producing inf. 
 *   ifa_fp8_emulated_attention_host: f32 Q, K, V (host) -> f32 O (host): the
 *     three e4m3 roundtrips and the FP8 forward; non-finite input returns
 *     IFA_EINVAL "fp8_e4m3_roundtrip: non-finite input" (fp8.cpp:82-84). */
int ifa_half_int8_fwd_host(const int8_t* q, const float* sq, const int8_t* k, const float* sk,
                           const float* v, float* o, int64_t slices, int64_t n, int64_t d,
                           int64_t br, int64_t bc, uint32_t flags, void* stream);
int ifa_fp8_emulated_attention_host(const float* q, const float* k, const float* v, float* o,
                                    int64_t slices, int64_t n, int64_t d, int64_t br,
                                    int64_t bc, uint32_t flags, void* stream);

/* Writes {127, 0, 1, 0, 0} into a device ifa_pcode_audit (async on stream). */
int ifa_audit_init(ifa_pcode_audit* audit, void* stream);

/* HOST pointer out128[0..127]: the exact decision boundaries the kernel uses
 * to settle ambiguous weight codes, B[k] = smallest float x with
 * (int)roundf(127*expf(x)) >= k+1 (k < 127), out128[127] = +inf.  Exposed so
 * tests can check them against an exhaustive scan of the reference's libm. */
int ifa_code_bounds(float* out128);

/* ---- IFA1 tensor files (tensor_io.hpp:22-39, tensor_io.cpp:15-178) ------
 * "IFA1" | dtype u8 (IFA_DT_*) | 3 zero bytes | rows u64 LE | cols u64 LE |
 * row-major payload.  Loaders reject malformed files with IFA_EFORMAT and
 * the reference's FormatError message ("bad magic", "truncated header: N
 * bytes", "nonzero reserved bytes", "header dimensions overflow: RxC",
 * "bad dtype code D", "truncated payload: ...", "oversized payload: ...",
 * "expected f32 tensor: PATH", "cannot open: PATH").  Host memory. */
#define IFA_DT_F32 0
#define IFA_DT_I8 1
#define IFA_DT_I32 2
int ifa_tensor_save(const char* path, int32_t dtype, const void* data, int64_t rows,
                    int64_t cols);
/* Validates the whole file (header and payload size) and reports its shape. */
int ifa_tensor_info(const char* path, int32_t* dtype, int64_t* rows, int64_t* cols);
/* dtype < 0 accepts any dtype; rows/cols must match the file (ifa_tensor_info). */
int ifa_tensor_load(const char* path, int32_t dtype, void* data, int64_t rows, int64_t cols);

/* Message of the last failing call on this host thread ("" if none). */
const char* ifa_last_error(void);

/* Build/version string, e.g. "ifa_b200 0.1 sm_100a". */
const char* ifa_version(void);

#ifdef __cplusplus
}
#endif

#endif /* IFA_B200_H */
