// integration/shim_model_forward.cpp — drives the reference's own model_forward
// (proj/src/model.cpp:453-483) over a quantized checkpoint twice: through the reference
// moe_ffn_forward (shim disabled) and through the GPU (shim enabled), and compares the
// results within the north_star tolerance. Exit 0 on success.
#include <cmath>
#include <cstdio>
#include <set>
#include <vector>

#include "moqe/model.hpp"

extern "C" long long moqe_gpu_shim_calls(void);
extern "C" void moqe_gpu_shim_enable(int on);

using namespace moqe;

int main() {
    ModelSpec spec = ModelSpec::toy();
    spec.d_model = 256;
    spec.d_ffn = 1024;
    spec.n_experts = 8;
    spec.enc_layers = 4;  // MoE layers 0, 2 (+ decoder 0)
    spec.dec_layers = 2;
    Checkpoint ckpt = build_random_checkpoint(spec, 2310, 0.05f);
    int fails = 0;
    for (int variant = 0; variant < 4; ++variant) {
        const int bits = variant == 3 ? 4 : 4 - variant;  // int4, int3, int2 linear; int4 log-scale
        const Scheme scheme = variant == 3 ? Scheme::LogScale : Scheme::LinearAbsMax;
        Checkpoint q = quantize_model(ckpt, {LayerGroup::ExpertFFN}, bits, scheme, Granularity::PerChannel,
                                      LayerSubset::All, LogScaleMode::AbsMax, 4);
        std::vector<std::vector<int32_t>> probe = {{1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12}, {500, 400, 300, 7}};
        moqe_gpu_shim_enable(0);
        ForwardResult cpu = model_forward(probe, q, spec);
        moqe_gpu_shim_enable(1);
        const long long before = moqe_gpu_shim_calls();
        ForwardResult gpu = model_forward(probe, q, spec);
        const long long calls = moqe_gpu_shim_calls() - before;
        ForwardResult gpu2 = model_forward(probe, q, spec);  // cached device banks (content keys)
        double mx = 0.0;
        long bad = 0;
        for (size_t i = 0; i < cpu.final_hidden.data.size(); ++i) {
            const double r = cpu.final_hidden.data[i], g = gpu.final_hidden.data[i];
            const double dlt = std::fabs(g - r);
            mx = std::max(mx, dlt);
            bad += dlt > 2e-3 + 1e-2 * std::fabs(r);
        }
        const bool det = gpu.final_hidden == gpu2.final_hidden;
        std::printf("%sint%d: model_forward with %lld GPU moe_ffn_forward calls, final_hidden max |gpu - cpu| %.3e, "
                    "%ld outside tolerance, repeat bit-identical %s\n", scheme == Scheme::LogScale ? "log-" : "", bits,
                    calls, mx, bad, det ? "yes" : "no");
        if (calls <= 0 || bad != 0 || !det) ++fails;
    }
    std::printf("%s\n", fails ? "FAIL" : "PASS");
    return fails ? 1 : 0;
}
