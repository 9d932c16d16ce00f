// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" wrapper around the UNMODIFIED reference library, compiled from the
// sources where they lie under /root/reference/proj/src (see oracle/Makefile).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load the resulting oracle/_ref/libmoqe_ref.so.
//
// Every entry point forwards to the reference's public C++ API:
//   ref_f32_to_f16_bits      -> moqe::f32_to_f16_bits        proj/src/tensor.cpp:38-72
//   ref_round_to_binary16    -> moqe::round_to_binary16      proj/src/tensor.cpp:100-106
//   ref_linear_scales        -> moqe::linear_scales          proj/src/quant.cpp:59-69
//   ref_quantize_linear      -> moqe::quantize_linear        proj/src/quant.cpp:71-95
//   ref_dequantize           -> moqe::dequantize             proj/src/quant.cpp:226-243
//   ref_packed_size/pack/unpack -> moqe::packed_size/pack/unpack  proj/src/bitpack.cpp:12-68
//   ref_top1_route           -> moqe::top1_route             proj/src/model.cpp:328-346
//   ref_bank_* / ref_moe_ffn_forward -> moqe::moe_ffn_forward proj/src/model.cpp:348-393
//   ref_matmul_dequant_fused -> moqe::matmul_dequant_fused   proj/src/bench.cpp:11-47
//   ref_write_moe_mqe1       -> moqe::write_checkpoint_file  proj/src/checkpoint.cpp:239-290
//   ref_quantize_log / ref_dequantize_log / ref_bank_create_log -> moqe::quantize_log, dequantize,
//                               moe_ffn_forward over log banks  proj/src/quant.cpp:97-243
//
// Status codes mirror include/moqe_gpu.h (0 ok, 1 invalid_argument,
// 2 out_of_range, 3 range_error, 9 other).
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "moqe/bench.hpp"
#include "moqe/bitpack.hpp"
#include "moqe/checkpoint.hpp"
#include "moqe/model.hpp"
#include "moqe/quant.hpp"
#include "moqe/tensor.hpp"

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (const std::range_error&) {
        return 3;
    } catch (...) {
        return 9;
    }
}

moqe::Tensor make2d(const float* p, int64_t r, int64_t c) {
    return moqe::Tensor({r, c}, std::vector<float>(p, p + r * c));
}

moqe::Granularity gran(int g) {
    return g == 0 ? moqe::Granularity::PerChannel : moqe::Granularity::PerTensor;
}

// A device-free, host-resident expert bank built from codes + scales as the
// reference's own QuantizedTensor values (what read_checkpoint would produce).
struct RefBank {
    int64_t d = 0, f = 0;
    int E = 0;
    std::vector<moqe::QuantizedTensor> q1, q2;
    std::vector<moqe::Tensor> w1f, w2f;      // float banks
    std::vector<moqe::Tensor> b1, b2;
    bool has_b1 = false, has_b2 = false, quantized = true;
    moqe::ExpertBank bank;

    void wire() {
        bank.experts.resize(static_cast<size_t>(E));
        for (int e = 0; e < E; ++e) {
            auto& ew = bank.experts[static_cast<size_t>(e)];
            if (quantized) {
                ew.w1 = moqe::WeightRef{nullptr, &q1[static_cast<size_t>(e)]};
                ew.w2 = moqe::WeightRef{nullptr, &q2[static_cast<size_t>(e)]};
            } else {
                ew.w1 = moqe::WeightRef{&w1f[static_cast<size_t>(e)], nullptr};
                ew.w2 = moqe::WeightRef{&w2f[static_cast<size_t>(e)], nullptr};
            }
            ew.b1 = has_b1 ? &b1[static_cast<size_t>(e)] : nullptr;
            ew.b2 = has_b2 ? &b2[static_cast<size_t>(e)] : nullptr;
        }
    }
};

moqe::QuantizedTensor make_qt(const int8_t* codes, const float* scales, int64_t rows,
                              int64_t cols, int bits, int g) {
    moqe::QuantizedTensor qt;
    qt.scheme = moqe::Scheme::LinearAbsMax;
    qt.bits = bits;
    qt.granularity = gran(g);
    qt.shape = {rows, cols};
    qt.codes.bits = bits;
    qt.codes.codes.assign(codes, codes + rows * cols);
    const int64_t ns = g == 0 ? cols : 1;
    qt.scales.assign(scales, scales + ns);
    return qt;
}

}  // namespace

extern "C" {

uint16_t ref_f32_to_f16_bits(float x) { return moqe::f32_to_f16_bits(x); }
float ref_f16_bits_to_f32(uint16_t h) { return moqe::f16_bits_to_f32(h); }

int ref_round_to_binary16(float x, float* out) {
    return guarded([&] { *out = moqe::round_to_binary16(x); });
}

int ref_linear_scales(const float* a, int64_t rows, int64_t cols, int bits, int g,
                      float* scales_out) {
    return guarded([&] {
        auto s = moqe::linear_scales(make2d(a, rows, cols), bits, gran(g));
        std::memcpy(scales_out, s.data(), s.size() * sizeof(float));
    });
}

int ref_quantize_linear(const float* a, int64_t rows, int64_t cols, int bits, int g,
                        int8_t* codes_out, float* scales_out) {
    return guarded([&] {
        auto qt = moqe::quantize_linear(make2d(a, rows, cols), bits, gran(g));
        std::memcpy(codes_out, qt.codes.codes.data(), qt.codes.codes.size());
        std::memcpy(scales_out, qt.scales.data(), qt.scales.size() * sizeof(float));
    });
}

int ref_dequantize(const int8_t* codes, const float* scales, int64_t rows, int64_t cols,
                   int bits, int g, float* out) {
    return guarded([&] {
        auto t = moqe::dequantize(make_qt(codes, scales, rows, cols, bits, g));
        std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
    });
}

// log-scale scheme (quant.cpp:97-224): codes / scales of quantize_log (AbsMax or MseOptimal),
// dequantize of log codes (quant.cpp:226-243)
int ref_quantize_log(const float* a, int64_t rows, int64_t cols, int bits, int g, int mse_optimal,
                     int8_t* codes_out, float* scales_out) {
    return guarded([&] {
        auto qt = moqe::quantize_log(make2d(a, rows, cols), bits, gran(g),
                                     mse_optimal ? moqe::LogScaleMode::MseOptimal : moqe::LogScaleMode::AbsMax);
        std::memcpy(codes_out, qt.codes.codes.data(), qt.codes.codes.size());
        std::memcpy(scales_out, qt.scales.data(), qt.scales.size() * sizeof(float));
    });
}

int ref_dequantize_log(const int8_t* codes, const float* scales, int64_t rows, int64_t cols, int bits, int g,
                       float* out) {
    return guarded([&] {
        auto qt = make_qt(codes, scales, rows, cols, bits, g);
        qt.scheme = moqe::Scheme::LogScale;
        auto t = moqe::dequantize(qt);
        std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
    });
}

int64_t ref_packed_size(int bits, int64_t count) {
    int64_t r = -1;
    guarded([&] { r = static_cast<int64_t>(moqe::packed_size(bits, static_cast<size_t>(count))); });
    return r;
}

int ref_pack(const int8_t* codes, int64_t count, int bits, uint8_t* out) {
    return guarded([&] {
        moqe::CodeArray c;
        c.bits = bits;
        c.codes.assign(codes, codes + count);
        auto bytes = moqe::pack(c);
        std::memcpy(out, bytes.data(), bytes.size());
    });
}

int ref_unpack(const uint8_t* data, int64_t len, int bits, int64_t count, int8_t* out) {
    return guarded([&] {
        auto c = moqe::unpack(data, static_cast<size_t>(len), bits, static_cast<size_t>(count));
        std::memcpy(out, c.codes.data(), c.codes.size());
    });
}

int ref_top1_route(const float* h, int64_t t, int64_t d, const float* wg, int64_t e,
                   int32_t* expert_out, float* gate_out) {
    return guarded([&] {
        moqe::Tensor ht = make2d(h, t, d), w = make2d(wg, d, e);
        auto r = moqe::top1_route(ht, moqe::RouterState{&w});
        for (int64_t i = 0; i < t; ++i) {
            expert_out[i] = r.expert[static_cast<size_t>(i)];
            gate_out[i] = r.gate[static_cast<size_t>(i)];
        }
    });
}

int ref_matmul_dequant_fused(const int8_t* codes, const float* scales, int64_t k, int64_t n,
                             int bits, int g, const float* x, int64_t m, float* out) {
    return guarded([&] {
        auto y = moqe::matmul_dequant_fused(make_qt(codes, scales, k, n, bits, g), make2d(x, m, k));
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(float));
    });
}

// Log-scale bank (per-channel): as ref_bank_create with Scheme::LogScale tensors.
void* ref_bank_create(int n_experts, int64_t d, int64_t f, int bits, const int8_t* codes1,
                      const float* scales1, const int8_t* codes2, const float* scales2,
                      const float* b1, const float* b2);
void* ref_bank_create_log(int n_experts, int64_t d, int64_t f, int bits, const int8_t* codes1,
                          const float* scales1, const int8_t* codes2, const float* scales2) {
    auto* b = static_cast<RefBank*>(ref_bank_create(n_experts, d, f, bits, codes1, scales1, codes2, scales2,
                                                    nullptr, nullptr));
    for (auto& q : b->q1) q.scheme = moqe::Scheme::LogScale;
    for (auto& q : b->q2) q.scheme = moqe::Scheme::LogScale;
    return b;
}

// Quantized bank: codes1 [E][d*f] (W1 [d x f] row-major), scales1 [E][f];
// codes2 [E][f*d] (W2 [f x d]), scales2 [E][d]; biases optional (nullptr).
void* ref_bank_create(int n_experts, int64_t d, int64_t f, int bits, const int8_t* codes1,
                      const float* scales1, const int8_t* codes2, const float* scales2,
                      const float* b1, const float* b2) {
    auto* b = new RefBank;
    b->E = n_experts;
    b->d = d;
    b->f = f;
    b->quantized = true;
    for (int e = 0; e < n_experts; ++e) {
        b->q1.push_back(make_qt(codes1 + e * d * f, scales1 + e * f, d, f, bits, 0));
        b->q2.push_back(make_qt(codes2 + e * f * d, scales2 + e * d, f, d, bits, 0));
    }
    if (b1) {
        b->has_b1 = true;
        for (int e = 0; e < n_experts; ++e)
            b->b1.emplace_back(std::vector<int64_t>{f}, std::vector<float>(b1 + e * f, b1 + (e + 1) * f));
    }
    if (b2) {
        b->has_b2 = true;
        for (int e = 0; e < n_experts; ++e)
            b->b2.emplace_back(std::vector<int64_t>{d}, std::vector<float>(b2 + e * d, b2 + (e + 1) * d));
    }
    b->wire();
    return b;
}

// Float bank (for the reference's identical-expert / zero-input tests).
void* ref_bank_create_float(int n_experts, int64_t d, int64_t f, const float* w1,
                            const float* w2, const float* b1, const float* b2) {
    auto* b = new RefBank;
    b->E = n_experts;
    b->d = d;
    b->f = f;
    b->quantized = false;
    for (int e = 0; e < n_experts; ++e) {
        b->w1f.push_back(make2d(w1 + e * d * f, d, f));
        b->w2f.push_back(make2d(w2 + e * f * d, f, d));
    }
    if (b1) {
        b->has_b1 = true;
        for (int e = 0; e < n_experts; ++e)
            b->b1.emplace_back(std::vector<int64_t>{f}, std::vector<float>(b1 + e * f, b1 + (e + 1) * f));
    }
    if (b2) {
        b->has_b2 = true;
        for (int e = 0; e < n_experts; ++e)
            b->b2.emplace_back(std::vector<int64_t>{d}, std::vector<float>(b2 + e * d, b2 + (e + 1) * d));
    }
    b->wire();
    return b;
}

void ref_bank_destroy(void* bank) { delete static_cast<RefBank*>(bank); }

// moe_ffn_forward over h [t x d]; token-sharded over n_threads (the reference
// forward is row-independent, so shards are bit-identical to one call).
int ref_bank_forward(void* bank, const float* h, int64_t t, const float* wg, float* out,
                     int n_threads) {
    auto* b = static_cast<RefBank*>(bank);
    const int64_t d = b->d;
    moqe::Tensor w = make2d(wg, d, b->E);
    if (n_threads <= 1 || t < 2) {
        return guarded([&] {
            auto y = moqe::moe_ffn_forward(make2d(h, t, d), b->bank, moqe::RouterState{&w});
            std::memcpy(out, y.data.data(), y.data.size() * sizeof(float));
        });
    }
    const int64_t nt = std::min<int64_t>(n_threads, t);
    const int64_t chunk = (t + nt - 1) / nt;
    std::vector<int> status(static_cast<size_t>(nt), 0);
    std::vector<std::thread> pool;
    for (int64_t i = 0; i < nt; ++i) {
        const int64_t lo = i * chunk, hi = std::min(t, lo + chunk);
        if (lo >= hi) continue;
        pool.emplace_back([&, i, lo, hi] {
            status[static_cast<size_t>(i)] = guarded([&] {
                auto y = moqe::moe_ffn_forward(make2d(h + lo * d, hi - lo, d), b->bank,
                                               moqe::RouterState{&w});
                std::memcpy(out + lo * d, y.data.data(), y.data.size() * sizeof(float));
            });
        });
    }
    for (auto& th : pool) th.join();
    for (int s : status)
        if (s) return s;
    return 0;
}

int ref_hardware_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }

// An MQE1 container (written by the reference's own write_checkpoint_file) holding one MoE
// layer the way ffn_block names it (model.cpp:402-412): "<layer>.expert.<e>.fc{1,2}.w" as
// q-lin tensors (codes [E][rows*cols], scales [E][cols] or [E][1] when per_tensor), optional
// f32 biases "<layer>.expert.<e>.fc{1,2}.b", and the f32 router "<layer>.router.w" [d x E].
// Returns the file size, or -1 on an exception.
int64_t ref_write_moe_mqe1(const char* path, const char* layer, int n_experts, int64_t d, int64_t f, int bits,
                           int per_tensor, const int8_t* codes1, const float* scales1, const int8_t* codes2,
                           const float* scales2, const float* b1, const float* b2, const float* wg) {
    try {
        moqe::Checkpoint ck;
        ck.meta["format"] = "moqe-b200-test";
        const std::string base = std::string(layer) + ".expert.";
        const int64_t ns1 = per_tensor ? 1 : f, ns2 = per_tensor ? 1 : d;
        for (int e = 0; e < n_experts; ++e) {
            const std::string p = base + std::to_string(e);
            ck.add(moqe::CheckpointEntry::quantized(p + ".fc1.w", moqe::LayerGroup::ExpertFFN,
                                                    make_qt(codes1 + e * d * f, scales1 + e * ns1, d, f, bits, per_tensor)));
            ck.add(moqe::CheckpointEntry::quantized(p + ".fc2.w", moqe::LayerGroup::ExpertFFN,
                                                    make_qt(codes2 + e * f * d, scales2 + e * ns2, f, d, bits, per_tensor)));
            if (b1)
                ck.add(moqe::CheckpointEntry::f32(p + ".fc1.b", moqe::LayerGroup::ExpertFFN,
                                                  moqe::Tensor({f}, std::vector<float>(b1 + e * f, b1 + (e + 1) * f))));
            if (b2)
                ck.add(moqe::CheckpointEntry::f32(p + ".fc2.b", moqe::LayerGroup::ExpertFFN,
                                                  moqe::Tensor({d}, std::vector<float>(b2 + e * d, b2 + (e + 1) * d))));
        }
        if (wg)
            ck.add(moqe::CheckpointEntry::f32(std::string(layer) + ".router.w", moqe::LayerGroup::Router,
                                              make2d(wg, d, n_experts)));
        return static_cast<int64_t>(moqe::write_checkpoint_file(ck, path));
    } catch (...) {
        return -1;
    }
}

}  // extern "C"
