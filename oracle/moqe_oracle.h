/* oracle/moqe_oracle.h — TEST INFRASTRUCTURE ONLY (the checker).
 *
 * CPU restatement, in plain C, of the reference's MoQE expert-FFN path.
 * Pinned against the reference's own known-answer tests and against the
 * compiled reference (oracle/_ref) by tests/test_oracle_pin.py.
 * Never linked into, or called by, the product library.
 */
#ifndef MOQE_ORACLE_H
#define MOQE_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status: 0 ok, 1 invalid_argument, 2 out_of_range, 3 range_error */
uint16_t orc_f32_to_f16_bits(float x);
float orc_f16_bits_to_f32(uint16_t h);
int orc_round_to_binary16(float x, float* out);

int orc_linear_scales(const float* a, int64_t rows, int64_t cols, int bits, int per_tensor,
                      float* scales);
int orc_quantize_linear(const float* a, int64_t rows, int64_t cols, int bits, int per_tensor,
                        int8_t* codes, float* scales);
int64_t orc_packed_size(int bits, int64_t count);
int orc_pack(const int8_t* codes, int64_t count, int bits, uint8_t* out);
int orc_unpack(const uint8_t* data, int64_t len, int bits, int64_t count, int8_t* out);

/* fp32 router logits h[t x d] * wg[d x e], reference summation order. */
void orc_router_logits(const float* h, int64_t t, int64_t d, const float* wg, int64_t e,
                       float* logits);
/* top-k routing (k = 1 or 2). expert [t*k], gate [t*k]. */
int orc_route(const float* h, int64_t t, int64_t d, const float* wg, int64_t e, int top_k,
              int32_t* expert, float* gate);

/* Expert FFN on rows x [m x d] with quantized W1 [d x f] / W2 [f x d]
 * (codes one int8 per code, per-channel scales), optional biases. */
void orc_expert_ffn(const float* x, int64_t m, int64_t d, int64_t f, const int8_t* c1,
                    const float* s1, const int8_t* c2, const float* s2, const float* b1,
                    const float* b2, float* y);

/* Full MoE layer. codes1 [E][d*f], scales1 [E][f], codes2 [E][f*d],
 * scales2 [E][d], b1/b2 optional [E][f]/[E][d]. top_k 1 or 2.
 * n_threads shards tokens (bit-identical to 1 thread). */
int orc_moe_forward(const float* h, int64_t t, int64_t d, int64_t f, int n_experts,
                    const float* wg, int top_k, const int8_t* codes1, const float* scales1,
                    const int8_t* codes2, const float* scales2, const float* b1,
                    const float* b2, float* out, int32_t* expert_out, float* gate_out,
                    int n_threads);

/* LayerNorm over rows (eps 1e-5, double statistics) — model.cpp:193-212. */
void orc_layer_norm(const float* x, int64_t rows, int64_t n, const float* gain,
                    const float* bias, float* out);

/* Reference matmul (model.cpp:152-167) and dense_ffn (model.cpp:315-322), fp32. */
void orc_matmul(const float* a, int64_t m, int64_t k, const float* b, int64_t n, float* out);
void orc_dense_ffn(const float* x, int64_t m, int64_t d, int64_t f, const float* w1, const float* b1,
                   const float* w2, const float* b2, float* y);

#ifdef __cplusplus
}
#endif
#endif
