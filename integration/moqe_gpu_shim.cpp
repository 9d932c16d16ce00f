// integration/moqe_gpu_shim.cpp — the reference-side drop-in for moqe::moe_ffn_forward.
//
// Defines the reference's own symbol
//     moqe::Tensor moqe::moe_ffn_forward(const Tensor&, const ExpertBank&, const RouterState&)
// (proj/include/moqe/model.hpp:87, proj/src/model.cpp:348-393) in a shared library that is
// linked (or LD_PRELOADed) ahead of the reference's libmoqe.so. The reference library is built
// -fPIC, so its own callers (ffn_block, model.cpp:399-417, and everything above it:
// model_forward, run_sensitivity, the CLI) reach this definition through the PLT and link
// unchanged. Banks of quantized experts (linear, or log-scale with 2..4 bits) run on the GPU
// through the C-ABI (include/moqe_gpu.h); everything else (float experts, log int8, mixed
// banks, and the reference's argument errors) goes to the reference implementation found with
// dlsym(RTLD_NEXT), so results and exceptions stay the reference's.
//
// Device banks are cached by CONTENT, not by address: ffn_block builds a stack-local
// ExpertBank on every call (model.cpp:402-412), so &bank is meaningless across calls. The key
// is the experts' QuantizedTensor / bias addresses plus a 64-bit fingerprint of their shapes,
// bits, scales, biases and a strided sample of codes; the router is keyed the same way.
// Errors from the C-ABI are rethrown as the matching std exception (moqe_status mapping).
#include <dlfcn.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "moqe/bitpack.hpp"
#include "moqe/model.hpp"
#include "moqe/quant.hpp"
#include "moqe_gpu.h"

namespace {

using moqe::ExpertBank;
using moqe::RouterState;
using moqe::Tensor;

using ForwardFn = Tensor (*)(const Tensor&, const ExpertBank&, const RouterState&);
constexpr const char* kForwardSym = "_ZN4moqe15moe_ffn_forwardERKNS_6TensorERKNS_10ExpertBankERKNS_11RouterStateE";

ForwardFn cpu_forward() {
    static ForwardFn fn = reinterpret_cast<ForwardFn>(dlsym(RTLD_NEXT, kForwardSym));
    if (!fn) throw std::runtime_error("moqe_gpu_shim: reference moe_ffn_forward not found (link libmoqe.so)");
    return fn;
}

[[noreturn]] void rethrow(moqe_status st) {
    const std::string msg = moqe_gpu_last_error();
    switch (st) {
        case MOQE_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case MOQE_OUT_OF_RANGE: throw std::out_of_range(msg);
        case MOQE_RANGE_ERROR: throw std::range_error(msg);
        default: throw std::runtime_error("moqe_gpu: " + msg);
    }
}
void check(moqe_status st) {
    if (st != MOQE_OK) rethrow(st);
}

uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}
uint64_t fp_bytes(uint64_t h, const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
    return h;
}
uint64_t fingerprint(const moqe::QuantizedTensor& q) {
    uint64_t h = mix(0xcbf29ce484222325ull, uint64_t(q.bits) << 8 | uint64_t(q.granularity));
    for (int64_t s : q.shape) h = mix(h, uint64_t(s));
    h = fp_bytes(h, q.scales.data(), q.scales.size() * sizeof(float));
    const auto& c = q.codes.codes;
    const size_t step = c.size() > 4096 ? c.size() / 4096 : 1;
    for (size_t i = 0; i < c.size(); i += step) h = mix(h, uint64_t(uint8_t(c[i])) | (uint64_t(i) << 8));
    return h;
}
uint64_t fingerprint(const Tensor* t) {
    if (!t) return 0;
    return fp_bytes(mix(0x1234, t->data.size()), t->data.data(), t->data.size() * sizeof(float));
}

struct DeviceBank {
    std::vector<const void*> addr;  // per expert: q1, q2, b1, b2
    uint64_t fp = 0;
    moqe_bank_t bank = nullptr;
    const Tensor* router = nullptr;
    uint64_t router_fp = 0;
};

std::mutex g_mu;
std::list<DeviceBank> g_cache;  // most recent first
constexpr size_t kCacheBanks = 64;
long long g_gpu_calls = 0;
int g_enabled = -1;

bool enabled() {
    if (g_enabled < 0) {
        const char* s = std::getenv("MOQE_GPU_SHIM");
        g_enabled = !(s && std::string(s) == "cpu");
    }
    return g_enabled != 0;
}

// A bank the GPU path takes: every expert linear-quantized with the same bits / shapes /
// granularity (moe_ffn_forward validates mixed banks itself: they go to the reference).
bool gpu_eligible(const ExpertBank& bank) {
    if (bank.experts.empty()) return false;
    const auto* q0 = bank.experts[0].w1.q;
    const auto* r0 = bank.experts[0].w2.q;
    if (!q0 || !r0) return false;
    for (const auto& ew : bank.experts) {
        const auto* a = ew.w1.q;
        const auto* b = ew.w2.q;
        if (!a || !b || a->scheme != q0->scheme || b->scheme != q0->scheme) return false;
        if (q0->scheme == moqe::Scheme::LogScale && q0->bits == 8) return false;  // not a GPU scheme
        if (a->bits != q0->bits || b->bits != q0->bits || a->shape != q0->shape || b->shape != r0->shape ||
            a->granularity != q0->granularity || b->granularity != q0->granularity)
            return false;
        if ((ew.b1 != nullptr) != (bank.experts[0].b1 != nullptr) || (ew.b2 != nullptr) != (bank.experts[0].b2 != nullptr))
            return false;
    }
    return q0->shape.size() == 2 && r0->shape.size() == 2 && r0->shape[0] == q0->shape[1] &&
           r0->shape[1] == q0->shape[0];
}

DeviceBank& device_bank(const ExpertBank& bank) {
    std::vector<const void*> addr;
    uint64_t fp = 0xfeedull;
    for (const auto& ew : bank.experts) {
        addr.insert(addr.end(), {ew.w1.q, ew.w2.q, ew.b1, ew.b2});
        fp = mix(fp, fingerprint(*ew.w1.q));
        fp = mix(fp, fingerprint(*ew.w2.q));
        fp = mix(fp, fingerprint(ew.b1));
        fp = mix(fp, fingerprint(ew.b2));
    }
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
        if (it->fp == fp && it->addr == addr) {
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front();
        }
    // build: pack the reference codes (moqe::pack, the MQE1 byte layout) and upload once
    const auto& q0 = *bank.experts[0].w1.q;
    const int E = int(bank.experts.size());
    const int64_t d = q0.shape[0], f = q0.shape[1];
    const int bits = q0.bits;
    const bool per_tensor = q0.granularity == moqe::Granularity::PerTensor;
    std::vector<uint8_t> p1, p2;
    std::vector<float> s1, s2, b1, b2;
    for (const auto& ew : bank.experts) {
        const auto a = moqe::pack(ew.w1.q->codes), b = moqe::pack(ew.w2.q->codes);
        p1.insert(p1.end(), a.begin(), a.end());
        p2.insert(p2.end(), b.begin(), b.end());
        s1.insert(s1.end(), ew.w1.q->scales.begin(), ew.w1.q->scales.end());
        s2.insert(s2.end(), ew.w2.q->scales.begin(), ew.w2.q->scales.end());
        if (ew.b1) b1.insert(b1.end(), ew.b1->data.begin(), ew.b1->data.end());
        if (ew.b2) b2.insert(b2.end(), ew.b2->data.begin(), ew.b2->data.end());
    }
    if (g_cache.size() >= kCacheBanks) {
        moqe_gpu_bank_destroy(g_cache.back().bank);
        g_cache.pop_back();
    }
    DeviceBank db;
    db.addr = std::move(addr);
    db.fp = fp;
    check(moqe_gpu_bank_create_ex(E, d, f, bits,
                                  q0.scheme == moqe::Scheme::LogScale ? MOQE_SCHEME_LOG : MOQE_SCHEME_LINEAR,
                                  per_tensor ? MOQE_PER_TENSOR : MOQE_PER_CHANNEL, p1.data(), s1.data(), p2.data(),
                                  s2.data(), b1.empty() ? nullptr : b1.data(), b2.empty() ? nullptr : b2.data(), 0,
                                  &db.bank));
    g_cache.push_front(std::move(db));
    return g_cache.front();
}

}  // namespace

namespace moqe {

Tensor moe_ffn_forward(const Tensor& h, const ExpertBank& bank, const RouterState& router) {
    if (!enabled() || !gpu_eligible(bank) || !router.gate_weights || !h.is2d())
        return cpu_forward()(h, bank, router);  // the reference's path, results and exceptions
    std::lock_guard<std::mutex> lock(g_mu);
    DeviceBank& db = device_bank(bank);
    const Tensor& wg = *router.gate_weights;
    const int64_t d = bank.experts[0].w1.q->shape[0];
    if (!wg.is2d() || wg.rows() != d || wg.cols() != int64_t(bank.experts.size()) || h.cols() != d)
        throw std::invalid_argument("matmul: shape mismatch");
    const uint64_t rfp = fingerprint(&wg);
    if (db.router != &wg || db.router_fp != rfp) {
        check(moqe_gpu_bank_set_router(db.bank, wg.data.data(), 0));
        db.router = &wg;
        db.router_fp = rfp;
    }
    Tensor out({h.rows(), d});
    check(moqe_gpu_moe_forward_host(db.bank, h.data.data(), MOQE_F32, h.rows(), 1, out.data.data(), MOQE_F32, nullptr));
    ++g_gpu_calls;
    return out;
}

}  // namespace moqe

extern "C" long long moqe_gpu_shim_calls(void) { return g_gpu_calls; }
extern "C" void moqe_gpu_shim_enable(int on) { g_enabled = on ? 1 : 0; }
