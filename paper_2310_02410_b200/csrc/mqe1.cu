// mqe1.cu — MQE1 container -> device-resident expert bank.
//
// Reference: read_checkpoint (proj/src/checkpoint.cpp:312-413), layout (:99-131): magic
// "MQE1", u32 version, u64 index length, text index ("m key value" / "t name group dtype bits
// granularity shape off len soff slen", fixed-width hex), then 64-byte aligned blobs. A q-lin
// blob is exactly the reference's packed code stream (bitpack.cpp:18-39) and its scales are
// binary16 (:264-270), i.e. the GPU bank's input layout: the container is mapped, each
// expert's blob is gathered into one staging buffer and copied to the device once; nothing is
// unpacked or re-quantized on the host. The index is validated like read_checkpoint (bad magic,
// version, truncation, inconsistent offsets -> MOQE_CHECKPOINT_ERROR with the reference's
// message text).
//
// Expert tensor names follow ffn_block (proj/src/model.cpp:402-412): "<layer>.expert.<e>.fc1.w",
// ".fc2.w", optional ".fc1.b" / ".fc2.b", router "<layer>.router.w".
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"

namespace moqe_gpu {
namespace {

struct Mqe1Entry {
    std::string name, group, dtype, gran;
    int bits = 0;
    std::vector<int64_t> shape;
    uint64_t off = 0, len = 0, soff = 0, slen = 0;
};

uint64_t packed_bytes(int bits, uint64_t n) { return uint64_t(packed_size(bits, int64_t(n))); }

bool parse_hex(const std::string& s, uint64_t* v) {
    if (s.empty() || s.size() > 16) return false;
    uint64_t r = 0;
    for (char c : s) {
        int d;
        if (c >= '0' && c <= '9') d = c - '0';
        else if (c >= 'a' && c <= 'f') d = c - 'a' + 10;
        else if (c >= 'A' && c <= 'F') d = c - 'A' + 10;
        else return false;
        r = r * 16 + uint64_t(d);
    }
    *v = r;
    return true;
}

bool parse_shape(const std::string& s, std::vector<int64_t>* shape) {
    shape->clear();
    size_t pos = 0;
    while (pos <= s.size()) {
        size_t next = s.find('x', pos);
        const std::string tok = s.substr(pos, next == std::string::npos ? std::string::npos : next - pos);
        if (tok.empty()) return false;
        for (char c : tok)
            if (c < '0' || c > '9') return false;
        const long long d = std::stoll(tok);
        if (d <= 0) return false;
        shape->push_back(d);
        if (next == std::string::npos) break;
        pos = next + 1;
    }
    return !shape->empty();
}

float f16_to_f32(uint16_t h) {
    __half_raw r;
    r.x = h;
    return __half2float(__half(r));
}

}  // namespace
}  // namespace moqe_gpu

using namespace moqe_gpu;

struct moqe_mqe1 {
    int fd = -1;
    const uint8_t* base = nullptr;
    size_t size = 0;
    std::map<std::string, std::string> meta;
    std::vector<Mqe1Entry> entries;
    std::map<std::string, size_t> by_name;
};

namespace {
moqe_status ckpt_fail(const std::string& msg) { return fail(MOQE_CHECKPOINT_ERROR, msg); }

void close_map(moqe_mqe1* m) {
    if (!m) return;
    if (m->base) munmap(const_cast<uint8_t*>(m->base), m->size);
    if (m->fd >= 0) close(m->fd);
    delete m;
}

const Mqe1Entry* find_entry(const moqe_mqe1* m, const std::string& name) {
    auto it = m->by_name.find(name);
    return it == m->by_name.end() ? nullptr : &m->entries[it->second];
}
}  // namespace

extern "C" {

moqe_status moqe_gpu_mqe1_open(const char* path, moqe_mqe1_t* out) {
    if (!path || !out) return fail(MOQE_INVALID_ARGUMENT, "mqe1: null argument");
    *out = nullptr;
    auto* m = new moqe_mqe1;
    m->fd = open(path, O_RDONLY);
    if (m->fd < 0) {
        close_map(m);
        return ckpt_fail(std::string("cannot open: ") + path);
    }
    struct stat sb;
    if (fstat(m->fd, &sb) != 0) {
        close_map(m);
        return ckpt_fail(std::string("cannot stat: ") + path);
    }
    m->size = size_t(sb.st_size);
    if (m->size > 0) {
        void* p = mmap(nullptr, m->size, PROT_READ, MAP_PRIVATE, m->fd, 0);
        if (p == MAP_FAILED) {
            close_map(m);
            return ckpt_fail(std::string("cannot map: ") + path);
        }
        m->base = static_cast<const uint8_t*>(p);
    }
    // header (checkpoint.cpp:315-328)
    if (m->size < 4 || std::memcmp(m->base, "MQE1", 4) != 0) {
        close_map(m);
        return ckpt_fail("bad magic (not an MQE1 container)");
    }
    if (m->size < 16) {
        close_map(m);
        return ckpt_fail("truncated header");
    }
    uint32_t version;
    uint64_t index_len;
    std::memcpy(&version, m->base + 4, 4);
    std::memcpy(&index_len, m->base + 8, 8);
    if (version != 1) {
        close_map(m);
        return ckpt_fail("unsupported container version " + std::to_string(version));
    }
    if (m->size < 16 + index_len) {
        close_map(m);
        return ckpt_fail("truncated index");
    }
    // index (checkpoint.cpp:330-392)
    std::istringstream index(std::string(reinterpret_cast<const char*>(m->base) + 16, size_t(index_len)));
    std::string line;
    while (std::getline(index, line)) {
        if (line.empty()) continue;
        std::istringstream ls(line);
        std::string tag;
        ls >> tag;
        if (tag == "m") {
            std::string k, v;
            if (!(ls >> k >> v)) {
                close_map(m);
                return ckpt_fail("malformed meta line");
            }
            m->meta[k] = v;
            continue;
        }
        if (tag != "t") {
            close_map(m);
            return ckpt_fail("unknown index record: " + tag);
        }
        Mqe1Entry e;
        std::string shape_s, off_s, len_s, soff_s, slen_s;
        if (!(ls >> e.name >> e.group >> e.dtype >> e.bits >> e.gran >> shape_s >> off_s >> len_s >> soff_s >> slen_s)) {
            close_map(m);
            return ckpt_fail("malformed tensor record");
        }
        if (!parse_shape(shape_s, &e.shape) || !parse_hex(off_s, &e.off) || !parse_hex(len_s, &e.len) ||
            !parse_hex(soff_s, &e.soff) || !parse_hex(slen_s, &e.slen)) {
            close_map(m);
            return ckpt_fail(e.name + ": bad index field");
        }
        uint64_t n = 1;
        for (int64_t dd : e.shape) n *= uint64_t(dd);
        uint64_t want_len = 0, want_slen = 0;
        if (e.dtype == "q-lin" || e.dtype == "q-log") {
            if (e.gran != "channel" && e.gran != "tensor") {
                close_map(m);
                return ckpt_fail(e.name + ": bad granularity " + e.gran);
            }
            if (!valid_bits(e.bits)) {
                close_map(m);
                return ckpt_fail(e.name + ": bad bit width");
            }
            want_len = packed_bytes(e.bits, n);
            const uint64_t ch = e.shape.size() == 2 ? uint64_t(e.shape[1]) : 1;
            want_slen = 2 * (e.gran == "tensor" ? 1 : ch);
        } else if (e.dtype == "f32") {
            want_len = 4 * n;
        } else if (e.dtype == "f16") {
            want_len = 2 * n;
        } else {
            close_map(m);
            return ckpt_fail(e.name + ": unknown dtype " + e.dtype);
        }
        if (e.len != want_len || e.slen != want_slen) {
            close_map(m);
            return ckpt_fail(e.name + ": index/offset inconsistency");
        }
        if (e.off + e.len > m->size || (e.slen && e.soff + e.slen > m->size)) {
            close_map(m);
            return ckpt_fail("truncated data section for tensor " + e.name);
        }
        if (m->by_name.count(e.name)) {
            close_map(m);
            return ckpt_fail("duplicate tensor name: " + e.name);
        }
        m->by_name[e.name] = m->entries.size();
        m->entries.push_back(std::move(e));
    }
    *out = m;
    return MOQE_OK;
}

moqe_status moqe_gpu_mqe1_close(moqe_mqe1_t m) {
    close_map(m);
    return MOQE_OK;
}

int64_t moqe_gpu_mqe1_count(moqe_mqe1_t m) { return m ? int64_t(m->entries.size()) : -1; }

moqe_status moqe_gpu_mqe1_entry(moqe_mqe1_t m, int64_t i, moqe_mqe1_info* info) {
    if (!m || !info || i < 0 || i >= int64_t(m->entries.size())) return fail(MOQE_INVALID_ARGUMENT, "mqe1: bad entry index");
    const Mqe1Entry& e = m->entries[size_t(i)];
    std::memset(info, 0, sizeof(*info));
    std::strncpy(info->name, e.name.c_str(), sizeof(info->name) - 1);
    std::strncpy(info->group, e.group.c_str(), sizeof(info->group) - 1);
    std::strncpy(info->dtype, e.dtype.c_str(), sizeof(info->dtype) - 1);
    info->bits = e.bits;
    info->per_tensor = e.gran == "tensor" ? 1 : 0;
    info->ndim = int(e.shape.size() < 4 ? e.shape.size() : 4);
    for (int k = 0; k < info->ndim; ++k) info->shape[k] = e.shape[size_t(k)];
    info->data_offset = e.off;
    info->data_bytes = e.len;
    info->scale_offset = e.soff;
    info->scale_bytes = e.slen;
    return MOQE_OK;
}

moqe_status moqe_gpu_mqe1_bank_create(moqe_mqe1_t m, const char* layer, int n_experts, moqe_bank_t* out) {
    if (!m || !layer || !out) return fail(MOQE_INVALID_ARGUMENT, "mqe1: null argument");
    *out = nullptr;
    if (n_experts <= 0) return fail(MOQE_INVALID_ARGUMENT, "moe_ffn_forward: empty expert bank");
    const std::string base = std::string(layer) + ".expert.";
    const Mqe1Entry* w10 = find_entry(m, base + "0.fc1.w");
    const Mqe1Entry* w20 = find_entry(m, base + "0.fc2.w");
    if (!w10 || !w20) return fail(MOQE_INVALID_ARGUMENT, std::string("mqe1: no experts under ") + layer);
    if (w10->dtype != "q-lin" || w20->dtype != "q-lin")
        return fail(MOQE_NOT_SUPPORTED, "mqe1: the GPU bank takes q-lin experts (" + w10->dtype + ")");
    if (w10->shape.size() != 2 || w20->shape.size() != 2)
        return fail(MOQE_INVALID_ARGUMENT, "quant: tensor must be 2D");
    const int64_t d = w10->shape[0], f = w10->shape[1];
    const int bits = w10->bits;
    const int per_tensor = w10->gran == "tensor" ? 1 : 0;
    const uint64_t p1 = w10->len, p2 = w20->len;
    std::vector<uint8_t> pk1(size_t(p1) * n_experts), pk2(size_t(p2) * n_experts);
    const size_t ns1 = per_tensor ? 1 : size_t(f), ns2 = per_tensor ? 1 : size_t(d);
    std::vector<float> sc1(ns1 * n_experts), sc2(ns2 * n_experts);
    std::vector<float> b1, b2;
    for (int e = 0; e < n_experts; ++e) {
        const std::string p = base + std::to_string(e);
        const Mqe1Entry* a = find_entry(m, p + ".fc1.w");
        const Mqe1Entry* b = find_entry(m, p + ".fc2.w");
        if (!a || !b) return fail(MOQE_INVALID_ARGUMENT, "mqe1: missing tensor " + p + ".fc{1,2}.w");
        // mixed / mismatched banks are rejected like moe_ffn_forward (model.cpp:349-353)
        if (a->dtype != "q-lin" || b->dtype != "q-lin" || a->bits != bits || b->bits != bits ||
            a->shape != w10->shape || b->shape != w20->shape || (a->gran == "tensor") != bool(per_tensor) ||
            (b->gran == "tensor") != bool(per_tensor))
            return fail(MOQE_INVALID_ARGUMENT, "moe_ffn_forward: mixed float/quantized expert bank");
        std::memcpy(pk1.data() + size_t(e) * p1, m->base + a->off, size_t(p1));
        std::memcpy(pk2.data() + size_t(e) * p2, m->base + b->off, size_t(p2));
        for (size_t k = 0; k < ns1; ++k) {
            uint16_t h;
            std::memcpy(&h, m->base + a->soff + 2 * k, 2);
            sc1[size_t(e) * ns1 + k] = f16_to_f32(h);
        }
        for (size_t k = 0; k < ns2; ++k) {
            uint16_t h;
            std::memcpy(&h, m->base + b->soff + 2 * k, 2);
            sc2[size_t(e) * ns2 + k] = f16_to_f32(h);
        }
        // optional biases (model.cpp:382,385), f32 or f16 entries
        for (int which = 0; which < 2; ++which) {
            const Mqe1Entry* bb = find_entry(m, p + (which ? ".fc2.b" : ".fc1.b"));
            if (!bb) continue;
            std::vector<float>& dst = which ? b2 : b1;
            const size_t n = size_t(which ? d : f);
            if (dst.empty()) dst.assign(size_t(n_experts) * n, 0.f);
            uint64_t cnt = 1;
            for (int64_t dd : bb->shape) cnt *= uint64_t(dd);
            if (cnt != n) return fail(MOQE_INVALID_ARGUMENT, "add_bias: shape mismatch");
            for (size_t k = 0; k < n; ++k) {
                if (bb->dtype == "f32") {
                    std::memcpy(&dst[size_t(e) * n + k], m->base + bb->off + 4 * k, 4);
                } else if (bb->dtype == "f16") {
                    uint16_t h;
                    std::memcpy(&h, m->base + bb->off + 2 * k, 2);
                    dst[size_t(e) * n + k] = f16_to_f32(h);
                } else {
                    return fail(MOQE_NOT_SUPPORTED, "mqe1: quantized bias");
                }
            }
        }
    }
    moqe_status st = moqe_gpu_bank_create_g(n_experts, d, f, bits, per_tensor, pk1.data(), sc1.data(), pk2.data(),
                                            sc2.data(), b1.empty() ? nullptr : b1.data(),
                                            b2.empty() ? nullptr : b2.data(), 0, out);
    if (st != MOQE_OK) return st;
    const Mqe1Entry* r = find_entry(m, std::string(layer) + ".router.w");
    if (r) {
        if (r->dtype != "f32" && r->dtype != "f16") return fail(MOQE_NOT_SUPPORTED, "mqe1: quantized router");
        if (r->shape.size() != 2 || r->shape[0] != d || r->shape[1] != n_experts)
            return fail(MOQE_INVALID_ARGUMENT, "matmul: shape mismatch");
        std::vector<float> wg(size_t(d) * n_experts);
        for (size_t k = 0; k < wg.size(); ++k) {
            if (r->dtype == "f32") {
                std::memcpy(&wg[k], m->base + r->off + 4 * k, 4);
            } else {
                uint16_t h;
                std::memcpy(&h, m->base + r->off + 2 * k, 2);
                wg[k] = f16_to_f32(h);
            }
        }
        st = moqe_gpu_bank_set_router(*out, wg.data(), 0);
        if (st != MOQE_OK) {
            moqe_gpu_bank_destroy(*out);
            *out = nullptr;
            return st;
        }
    }
    return MOQE_OK;
}

}  // extern "C"
