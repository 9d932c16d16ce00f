/* moqe_gpu.h — C-ABI of the B200-native MoQE expert-FFN path.
 *
 * Drop-in boundary for the reference C++ API of the "quantize experts ->
 * moe_ffn_forward (gate -> permute -> expert FFN -> combine)" path. Every
 * entry point names the reference interface it replaces (paths relative to
 * /root/reference/proj). Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *  - Pointers marked (device) are CUDA device pointers owned by the caller;
 *    (host) pointers are host memory. `stream` is a cudaStream_t (NULL = legacy
 *    default stream). Work is stream-ordered unless stated "blocking".
 *  - Matrices are row-major. For a weight W [K x N] the channel is the column
 *    (output feature), as in the reference (include/moqe/tensor.hpp:10-13).
 *  - Codes are signed b-bit integers stored one per int8 (CodeArray,
 *    include/moqe/bitpack.hpp:9-14); packed bytes use the reference layout
 *    (offset binary, LSB-first, 3-bit in 24-bit groups; bitpack.hpp:22-28).
 *  - Scales are f32 values holding binary16-representable numbers, one per
 *    column (per-channel) or one per matrix (per-tensor), exactly like
 *    QuantizedTensor::scales (include/moqe/quant.hpp:33).
 *  - Errors are returned as moqe_status; the reference throws the matching
 *    exception (std::invalid_argument / std::out_of_range / std::range_error).
 *    moqe_gpu_last_error() gives a thread-local message.
 */
#ifndef MOQE_GPU_H
#define MOQE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOQE_GPU_ABI_VERSION 1

typedef enum moqe_status {
    MOQE_OK = 0,
    MOQE_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    MOQE_OUT_OF_RANGE = 2,     /* std::out_of_range (bitpack.cpp:27-29) */
    MOQE_RANGE_ERROR = 3,      /* std::range_error (tensor.cpp:101-104) */
    MOQE_CUDA_ERROR = 4,
    MOQE_NCCL_ERROR = 5,
    MOQE_NOT_SUPPORTED = 6,
    MOQE_CHECKPOINT_ERROR = 7  /* moqe::CheckpointError (checkpoint.hpp:14-30) */
} moqe_status;

typedef enum moqe_granularity { MOQE_PER_CHANNEL = 0, MOQE_PER_TENSOR = 1 } moqe_granularity;
typedef enum moqe_dtype { MOQE_F32 = 0, MOQE_F16 = 1 } moqe_dtype;
typedef enum moqe_scheme { MOQE_SCHEME_LINEAR = 0, MOQE_SCHEME_LOG = 1 } moqe_scheme; /* quant.hpp:11 */

typedef struct moqe_bank* moqe_bank_t;

int moqe_gpu_abi_version(void);
const char* moqe_gpu_last_error(void);
const char* moqe_gpu_status_string(moqe_status st);

/* ---- bit-packing --------------------------------------------------------
 * packed_size:  moqe::packed_size   include/moqe/bitpack.hpp:25 (bitpack.cpp:12-16)
 *               returns (size_t)-1 for an unsupported width.
 * pack:         moqe::pack          include/moqe/bitpack.hpp:28 (bitpack.cpp:18-39)
 *               codes (device) -> out (device, packed_size bytes). Blocking:
 *               an out-of-range code returns MOQE_OUT_OF_RANGE.
 * unpack:       moqe::unpack        include/moqe/bitpack.hpp:30-31 (bitpack.cpp:41-68)
 *               len must equal packed_size(bits, count) else MOQE_INVALID_ARGUMENT.
 */
size_t moqe_gpu_packed_size(int bits, size_t count);
moqe_status moqe_gpu_pack(const int8_t* codes, int64_t count, int bits, uint8_t* out,
                          void* stream);
moqe_status moqe_gpu_unpack(const uint8_t* data, int64_t len, int bits, int64_t count,
                            int8_t* codes, void* stream);

/* ---- linear quantizer (batched over `batch` matrices of [rows x cols]) ----
 * linear_scales:   moqe::linear_scales   include/moqe/quant.hpp:48 (quant.cpp:59-69)
 * quantize_linear: moqe::quantize_linear include/moqe/quant.hpp:50 (quant.cpp:71-95)
 * quantize_pack:   quantize_linear + pack fused ("quantize experts" as
 *                  write_checkpoint stores it, checkpoint.cpp:255-261). packed
 *                  holds batch * packed_size(bits, rows*cols) bytes.
 * All blocking (errors detected on the device are reported like the
 * reference throws): non-finite input -> MOQE_INVALID_ARGUMENT,
 * scale overflowing binary16 -> MOQE_RANGE_ERROR. Pointers are device.
 * codes/packed may be NULL to skip that output.
 */
moqe_status moqe_gpu_linear_scales(const float* a, int64_t batch, int64_t rows, int64_t cols,
                                   int bits, moqe_granularity g, float* scales, void* stream);
moqe_status moqe_gpu_quantize_linear(const float* a, int64_t batch, int64_t rows, int64_t cols,
                                     int bits, moqe_granularity g, int8_t* codes,
                                     float* scales, void* stream);
moqe_status moqe_gpu_quantize_pack(const float* a, int64_t batch, int64_t rows, int64_t cols,
                                   int bits, moqe_granularity g, uint8_t* packed,
                                   float* scales, int8_t* codes, void* stream);

/* ---- routing ------------------------------------------------------------------
 * moqe::top1_route include/moqe/model.hpp:65 (model.cpp:328-346), plus top-2
 * with renormalised gates (BASELINE config 4). h [t x d] (device, f32 or f16),
 * wg [d x n_experts] f32 (device). Logits are fp32 in the reference's
 * summation order (bit-identical), argmax ties -> lowest index, top-1 gate =
 * softmax probability of the winner (double). expert/gate: [t x top_k] (device).
 */
moqe_status moqe_gpu_route(const void* h, moqe_dtype h_dtype, int64_t t, int64_t d,
                           const float* wg, int n_experts, int top_k, int32_t* expert,
                           float* gate, void* stream);

/* ---- device-resident expert bank ------------------------------------------
 * ExpertBank (include/moqe/model.hpp:74-82) of quantized experts
 * W1 [d_model x d_ffn], W2 [d_ffn x d_model] (+ optional biases), uploaded
 * once. packed_w1: n_experts * packed_size(bits, d*f) bytes, reference layout
 * (what MQE1 stores, checkpoint.cpp:255-261); scales1: n_experts * d_ffn f32;
 * packed_w2 / scales2 likewise with d_model scales; b1: n_experts*d_ffn or
 * NULL; b2: n_experts*d_model or NULL (model.cpp:382,385 skip null biases).
 * inputs_on_device: 1 if all input pointers are device pointers, 0 for host.
 * The bank re-tiles the packed bytes on the device (same bits, no requantize).
 * Blocking. */
moqe_status moqe_gpu_bank_create(int n_experts, int64_t d_model, int64_t d_ffn, int bits,
                                 const uint8_t* packed_w1, const float* scales1,
                                 const uint8_t* packed_w2, const float* scales2,
                                 const float* b1, const float* b2, int inputs_on_device,
                                 moqe_bank_t* out);

/* bank_create with the scales' granularity: MOQE_PER_CHANNEL (0: scales1 [E][d_ffn], scales2
 * [E][d_model], as bank_create) or MOQE_PER_TENSOR (1: one scale per expert matrix, scales1 and
 * scales2 [E]; Granularity::PerTensor, quant.cpp:53-55, broadcast to every channel). */
moqe_status moqe_gpu_bank_create_g(int n_experts, int64_t d_model, int64_t d_ffn, int bits, int granularity,
                                   const uint8_t* packed_w1, const float* scales1,
                                   const uint8_t* packed_w2, const float* scales2, const float* b1,
                                   const float* b2, int inputs_on_device, moqe_bank_t* out);

/* bank_create with the quantization scheme (Scheme, quant.hpp:11): MOQE_SCHEME_LINEAR or
 * MOQE_SCHEME_LOG (quantize_log, quant.cpp:179-224: field = sign bit + k, weight = +-s * 2^-k;
 * the same packed byte stream, bitpack.cpp:18-39). Log banks run on the tcgen05 path, which
 * decodes the fields to exact fp16 +-2^-k in staging; bits 2, 3, 4 (log int8 -> NOT_SUPPORTED). */
moqe_status moqe_gpu_bank_create_ex(int n_experts, int64_t d_model, int64_t d_ffn, int bits, int scheme,
                                    int granularity, const uint8_t* packed_w1, const float* scales1,
                                    const uint8_t* packed_w2, const float* scales2, const float* b1,
                                    const float* b2, int inputs_on_device, moqe_bank_t* out);
moqe_status moqe_gpu_bank_destroy(moqe_bank_t bank);
/* Router weights Wg [d_model x n_experts] f32 kept with the bank
 * (RouterState, include/moqe/model.hpp:56-58). Blocking. */
moqe_status moqe_gpu_bank_set_router(moqe_bank_t bank, const float* wg, int on_device);
/* Bytes of device weight storage (packed codes, excluding scales/biases). */
int64_t moqe_gpu_bank_weight_bytes(moqe_bank_t bank);

/* Execution-path selection for moe_forward:
 *   MOQE_PATH_AUTO  — weight-streaming GEMV for experts with <= 32 routed rows,
 *                     tcgen05 grouped GEMM for the rest (decided on device).
 *   MOQE_PATH_GEMV  — force the GEMV path for every expert (experts with more
 *                     than 32 rows are processed in 32-row passes).
 *   MOQE_PATH_GEMM  — force the tcgen05 grouped GEMM for all experts. */
typedef enum moqe_path { MOQE_PATH_AUTO = 0, MOQE_PATH_GEMV = 1, MOQE_PATH_GEMM = 2 } moqe_path;

/* ---- forward ----------------------------------------------------------------------
 * moqe::moe_ffn_forward include/moqe/model.hpp:87 (model.cpp:348-393):
 * out[tok] = sum_k gate_k * (relu(h W1_e + b1) W2_e + b2), e = expert_k(tok).
 * h [t x d] (device, f32 or f16), wg (device) or NULL to use the bank's router,
 * out [t x d] (device, f32 or f16). expert_out/gate_out [t x top_k] (device)
 * optional. Stream-ordered, no host synchronisation; the bank's workspace
 * makes concurrent forwards on one bank unsafe (one stream per bank).
 * t == 0 is valid (no work). */
moqe_status moqe_gpu_moe_forward(moqe_bank_t bank, const void* h, moqe_dtype h_dtype, int64_t t,
                                 const float* wg, int top_k, void* out, moqe_dtype out_dtype,
                                 int32_t* expert_out, float* gate_out, moqe_path path,
                                 void* stream);

/* Expert FFN on rows that are already routed (expert-parallel owner side):
 * out[r] = gate[r] * (relu(x[r] W1_e + b1) W2_e + b2), e = expert[r] (bank-local
 * expert index). x [rows x d] (device, f32/f16), expert int32 [rows], gate f32
 * [rows], out [rows x d]. Same kernels as moe_forward minus the router; rows are
 * grouped per expert in ascending row order (model.cpp:360-364). */
moqe_status moqe_gpu_expert_ffn(moqe_bank_t bank, const void* x, moqe_dtype x_dtype, int64_t rows,
                                const int32_t* expert, const float* gate, void* out, moqe_dtype out_dtype,
                                moqe_path path, void* stream);

/* Per-kernel device timing (measurement support for bench.py): when enabled,
 * every kernel moe_forward launches on `stream` is bracketed by CUDA events.
 * Works under CUDA-graph capture (the events become graph nodes).
 * profile_read synchronises and returns milliseconds and launch counts per
 * kernel kind for the events recorded since the last clearing read; with
 * keep != 0 the recorded events are kept (read again after the next graph
 * replay). Kinds: 0 route (+ plan, + the k_xrows token-row encoding when the
 * GEMV runs), 1 scatter, 2 gemv (k_gemv fc1 + k_gemv fc2), 3 gemm fc1,
 * 4 gemm fc2, 5 convert. */
#define MOQE_PROFILE_KINDS 6
moqe_status moqe_gpu_bank_profile(moqe_bank_t bank, int enable);
moqe_status moqe_gpu_bank_profile_read(moqe_bank_t bank, double* ms, int64_t* launches, int keep);

/* ---- MQE1 container -> device bank (checkpoint.cpp:99-131 layout, :312-413 reader) ----
 * open maps the file and validates the header and index like read_checkpoint (bad magic /
 * version, truncation, inconsistent offsets, duplicate names -> MOQE_CHECKPOINT_ERROR).
 * mqe1_bank_create builds the bank of "<layer>.expert.<e>.fc{1,2}.w" (q-lin; + optional
 * ".fc{1,2}.b"), names as ffn_block (model.cpp:402-412), straight from the packed blobs (one
 * host->device copy, no unpacking), and sets "<layer>.router.w" as its router when present. */
typedef struct moqe_mqe1* moqe_mqe1_t;
typedef struct moqe_mqe1_info {
    char name[128], group[32], dtype[8];
    int bits, per_tensor, ndim;
    int64_t shape[4];
    uint64_t data_offset, data_bytes, scale_offset, scale_bytes;
} moqe_mqe1_info;
moqe_status moqe_gpu_mqe1_open(const char* path, moqe_mqe1_t* out);
moqe_status moqe_gpu_mqe1_close(moqe_mqe1_t m);
int64_t moqe_gpu_mqe1_count(moqe_mqe1_t m);
moqe_status moqe_gpu_mqe1_entry(moqe_mqe1_t m, int64_t i, moqe_mqe1_info* info);
moqe_status moqe_gpu_mqe1_bank_create(moqe_mqe1_t m, const char* layer, int n_experts, moqe_bank_t* out);

/* Pre-LN residual FFN stack support (BASELINE config 3):
 * x [rows][n] f32 residual stream; when delta != NULL, x += delta first (in place, fp32 like
 * add_inplace, proj/src/model.cpp:308-310); then out = layer_norm(x, gain, bias) per row, eps
 * 1e-5, statistics in double (model.cpp:193-212). Replaces the layer_norm + add_inplace pair of
 * run_stack (model.cpp:419-435). Stream-ordered. */
moqe_status moqe_gpu_add_layer_norm(float* x, const float* delta, int64_t rows, int64_t n,
                                    const float* gain, const float* bias, void* out,
                                    moqe_dtype out_dtype, void* stream);

/* Expert-parallel dispatch / combine (BASELINE config 4). The reference is
 * single-process; these are the sharded form of its gather (model.cpp:360-364)
 * and scatter (model.cpp:387-390), replacing the sort / bincount / index_select / index_add_
 * of an eager exchange. Rank g owns experts [g*E/G, (g+1)*E/G).
 * ep_dispatch: h [t][d] f16 (d even), expert/gate [t][top_k] (global ids, f32 gates) ->
 *   records [t*top_k][d+4] f16 = [row | owner-local expert id (i32) | gate (f32)] ordered by
 *   owner rank, stable in flat order t*top_k+s; pos [t*top_k] = record row of each assignment;
 *   send_counts [world] i64; *err (device i32) = 1 if an id is out of range (not packed).
 * ep_combine: out [t][d] f32 = 0 + back[pos[t*k]] (+ back[pos[t*k+1]]) (f16 or f32 rows in
 *   record order, i.e. as returned by the all_to_all). Stream-ordered, no host sync. */
moqe_status moqe_gpu_ep_dispatch(const void* h, int64_t t, int64_t d, const int32_t* expert,
                                 const float* gate, int top_k, int n_experts, int world,
                                 void* records, int32_t* pos, int64_t* send_counts,
                                 int32_t* err, void* stream);
moqe_status moqe_gpu_ep_combine(const void* back, moqe_dtype back_dtype, const int32_t* pos, int64_t t,
                                int top_k, int64_t d, float* out, void* stream);

/* In-kernel launch spans of the decode path (measurement support, off by default):
 * with span(bank, 1) each decode forward's router and expert-FFN kernels record,
 * on the device, the time from the first CTA's start (after the programmatic-
 * dependent-launch wait) to the last CTA's exit, without breaking the launch
 * chain (no event nodes). span_read synchronises and returns, per kind
 * (0 router, 1 expert FFN), the summed microseconds and the launch count since
 * the last read, then clears them. */
moqe_status moqe_gpu_bank_span(moqe_bank_t bank, int enable);
moqe_status moqe_gpu_bank_span_read(moqe_bank_t bank, double* total_us, int64_t* launches);

/* Device event trace of the decode path (diagnostics; off by default).
 * trace(bank, 1) allocates, per SM, 512 slots of two u64: slots 0..255 for the
 * fc1 kernel, 256..511 for fc2. In each half, the first and last slot hold
 * (globaltimer ns, clock64) anchors at kernel entry / exit; the others hold
 * events (clock64, word) with word = role<<60 | event<<56 | phase<<48 |
 * expert<<32 | m-tile<<20 | rows<<16 | 1 (roles 2 consumer, 3 epilogue,
 * 4 producer, 5 weight unit landed, 7 prologue). After them, 64 x 16 u64
 * router stamps (globaltimer ns; 0 start, 1 row loaded, 10 chain done, 13 chain
 * clock64 cycles). tools/trace_gemv.py decodes both. trace_read synchronises,
 * copies up to `cap` words (out may be NULL to query the size), clears the
 * buffer and returns the word count, or -1 when tracing is off. */
moqe_status moqe_gpu_bank_trace(moqe_bank_t bank, int enable);
int64_t moqe_gpu_bank_trace_read(moqe_bank_t bank, uint64_t* out, int64_t cap);

/* Host-buffer convenience (the reference's by-value API): copies h (host,
 * pinned or pageable) in, runs moe_forward, copies out (host) back. Blocking. */
moqe_status moqe_gpu_moe_forward_host(moqe_bank_t bank, const void* h_host, moqe_dtype h_dtype,
                                      int64_t t, int top_k, void* out_host,
                                      moqe_dtype out_dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOQE_GPU_H */
