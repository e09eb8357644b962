// tgb/terngrad.hpp — C++ host mirror of the reference's `terngrad` namespace
// (proj/include/terngrad/{rng,tensor,codec}.hpp) on the B200 C-ABI
// (tgb/terngrad_b200.h). Same names, argument meaning, value semantics and
// exception types/messages as the reference, so a reference user switches with
//
//     #include "tgb/terngrad.hpp"      // instead of "terngrad/codec.hpp"
//     namespace terngrad = tgb;        // optional alias
//
// and links libtgb.so + libcudart. Host-vector functions copy to the device,
// run the sm_100a kernels and copy back (value semantics, like the
// reference). The training-loop entry point is SyncWorker: gradients stay in
// HBM and one call runs encode -> exchange -> decode (Worker::run sync
// segment, cluster.hpp:283-297). There is no CPU fallback: without a CUDA
// device every call throws.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <variant>
#include <vector>

#include "tgb/terngrad_b200.h"

namespace tgb {

// codec.hpp:25-27
struct CodecError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// wire.hpp:14-16
struct ProtocolError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline void check(tgb_status s, const char* what) {
    if (s == TGB_OK) return;
    if (s == TGB_ERR_INVALID_ARGUMENT) throw std::invalid_argument(what);
    throw std::runtime_error(std::string(what) + ": " + tgb_status_string(s));
}

// owning device buffer
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) : n(count) {
        if (n) cuda_check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        return *this;
    }
    ~DevBuf() { if (p) cudaFree(p); }
    void upload(const T* src, size_t count) {
        if (count) cuda_check(cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
    void download(T* dst, size_t count) const {
        if (count) cuda_check(cudaMemcpy(dst, p, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    }
};

// std::to_string(float) for the reference's message (codec.hpp:164)
inline std::string fstr(float s) { return std::to_string(s); }

inline void layer_check(const std::string& name, float s = 0.0f) {
    tgb_error e{};
    const tgb_status st = tgb_layer_check(nullptr, &e);
    if (st == TGB_OK) return;
    if (st != TGB_ERR_CODEC) check(st, "tgb_layer_check");
    if (e.flags & TGB_E_NONFINITE) throw CodecError("encode_step: non-finite gradient " + name);
    if (e.flags & TGB_E_SCALER_BELOW_MAX)
        throw CodecError("ternarize: scaler " + fstr(s) + " below max |g| in " + name);
    if (e.flags & TGB_E_S0_NONZERO)
        throw CodecError("ternarize: s=0 but gradient has nonzero element");
    if (e.flags & TGB_E_CORRUPT_CODE)
        throw CodecError("corrupt ternary code 11 in block " + name + " at element " +
                         std::to_string(e.index));
    throw CodecError("codec error in " + name);
}

}  // namespace detail

// rng.hpp:37-44
inline uint64_t fnv1a64(std::string_view s) { return tgb_fnv1a64(s.data(), s.size()); }

// tensor.hpp:14-43
struct GradTensor {
    std::string name;
    std::vector<std::size_t> shape;
    std::vector<float> values;

    GradTensor() = default;
    GradTensor(std::string n, std::vector<std::size_t> s)
        : name(std::move(n)), shape(std::move(s)) {
        values.assign(element_count(shape), 0.0f);
    }
    GradTensor(std::string n, std::vector<std::size_t> s, std::vector<float> v)
        : name(std::move(n)), shape(std::move(s)), values(std::move(v)) {
        if (values.size() != element_count(shape))
            throw std::invalid_argument("GradTensor " + name + ": values/shape mismatch");
    }
    static std::size_t element_count(const std::vector<std::size_t>& shape) {
        std::size_t n = 1;
        for (std::size_t d : shape) n *= d;
        return shape.empty() ? 0 : n;
    }
    std::size_t size() const { return values.size(); }
};

// rng.hpp:48-84 (bits/uniform evaluated on the device)
class RngStream {
public:
    RngStream(uint64_t seed, uint64_t iteration, std::string_view tensor_name, uint64_t worker = 0)
        : seed_(seed), t_(iteration), h_(fnv1a64(tensor_name)), worker_(worker) {}
    uint32_t bits(uint64_t index) const {
        detail::DevBuf<uint32_t> d(1);
        detail::check(tgb_rng_bits(seed_, t_, h_, worker_, index, 1, d.p, nullptr), "tgb_rng_bits");
        uint32_t v = 0;
        d.download(&v, 1);
        return v;
    }
    float uniform(uint64_t index) const { return static_cast<float>(bits(index)) * 0x1p-32f; }
    uint64_t seed() const { return seed_; }
    uint64_t iteration() const { return t_; }
    uint64_t name_hash() const { return h_; }
    uint64_t worker() const { return worker_; }

private:
    uint64_t seed_, t_, h_, worker_;
};

// codec.hpp:78-96
enum class Bucketing { PerTensor = TGB_BUCKET_PER_TENSOR, Global = TGB_BUCKET_GLOBAL,
                       FixedSize = TGB_BUCKET_FIXED };
enum class ShareMode { Ref = TGB_SHARE_REF, Preshared = TGB_SHARE_PRESHARED };

struct CodecConfig {
    float clip_factor = 2.5f;
    bool clipping_enabled = true;
    Bucketing bucketing = Bucketing::PerTensor;
    std::size_t bucket_size = 0;
    bool scaler_sharing = true;
    bool float_mode = false;
    std::set<std::string> passthrough;
    uint64_t seed = 0;
    ShareMode share_mode = ShareMode::Ref;

    void validate() const {
        if (!(clip_factor > 0.0f)) throw std::invalid_argument("codec: clip factor must be positive");
        if (bucketing == Bucketing::FixedSize && bucket_size < 1)
            throw std::invalid_argument("codec: fixed-size bucket needs k >= 1");
    }
    tgb_codec_params params() const {
        tgb_codec_params p{};
        p.clip_factor = clip_factor;
        p.clipping_enabled = clipping_enabled ? 1 : 0;
        p.bucketing = static_cast<int32_t>(bucketing);
        p.scaler_sharing = scaler_sharing ? 1 : 0;
        p.bucket_size = bucket_size;
        p.seed = seed;
        p.share_mode = static_cast<int32_t>(share_mode);
        return p;
    }
};

// codec.hpp:30-61
struct TernaryBlock {
    std::string name;
    uint32_t n = 0;
    float s = 0.0f;
    std::vector<uint8_t> codes;  // ceil(n/4) bytes

    int code_at(std::size_t k) const {
        const uint8_t c = (codes[k / 4] >> (2 * (k % 4))) & 0b11;
        switch (c) {
            case 0b00: return 0;
            case 0b01: return +1;
            case 0b10: return -1;
            default:
                throw CodecError("corrupt ternary code 11 in block " + name + " at element " +
                                 std::to_string(k));
        }
    }
    double zero_fraction() const {
        if (n == 0) return 0.0;
        std::size_t zeros = 0;
        for (std::size_t k = 0; k < n; ++k)
            if (code_at(k) == 0) ++zeros;
        return static_cast<double>(zeros) / static_cast<double>(n);
    }
};

// codec.hpp:63-76
struct PassthroughBlock {
    std::string name;
    std::vector<float> values;
};

using GradBlock = std::variant<TernaryBlock, PassthroughBlock>;

struct EncodedGradient {
    uint64_t iteration = 0;
    uint16_t worker = 0;
    std::vector<GradBlock> blocks;
};

struct EncodeResult {
    EncodedGradient encoded;
    std::vector<float> local_scalers;
};

// codec.hpp:128-134
inline float scaler(std::span<const float> v) {
    detail::DevBuf<float> d(v.size()), s(1);
    d.upload(v.data(), v.size());
    detail::check(tgb_layer_scaler(d.p, v.size(), s.p, nullptr), "tgb_layer_scaler");
    detail::layer_check("scaler");
    float out = 0.0f;
    s.download(&out, 1);
    return out;
}
inline float scaler(const GradTensor& g) { return scaler(std::span<const float>(g.values)); }

// codec.hpp:136-141
inline float share_scalers(std::span<const float> locals) {
    if (locals.empty()) throw CodecError("share_scalers: empty scaler list");
    float m = 0.0f;
    for (float s : locals) m = std::max(m, s);
    return m;
}

// codec.hpp:117-124
inline GradTensor clip(const GradTensor& g, float c) {
    if (g.size() < 2) return g;
    detail::DevBuf<float> d(g.size()), o(g.size()), b(1);
    d.upload(g.values.data(), g.size());
    detail::check(tgb_layer_clip(d.p, g.size(), c, o.p, b.p, nullptr), "tgb_layer_clip");
    detail::layer_check(g.name);
    GradTensor out = g;
    o.download(out.values.data(), g.size());
    return out;
}

// codec.hpp:148-175
inline TernaryBlock ternarize(std::string name, std::span<const float> g, float s,
                              const RngStream& rng, uint64_t rng_base = 0) {
    TernaryBlock blk;
    blk.name = std::move(name);
    blk.n = static_cast<uint32_t>(g.size());
    blk.s = s;
    blk.codes.assign((g.size() + 3) / 4, 0);
    if (g.empty()) return blk;
    detail::DevBuf<float> d(g.size());
    detail::DevBuf<uint8_t> c(blk.codes.size());
    d.upload(g.data(), g.size());
    detail::check(tgb_layer_ternarize(d.p, g.size(), s, rng.seed(), rng.iteration(),
                                      rng.name_hash(), rng.worker(), rng_base, c.p, nullptr),
                  "tgb_layer_ternarize");
    detail::layer_check(blk.name, s);
    c.download(blk.codes.data(), blk.codes.size());
    return blk;
}
inline TernaryBlock ternarize(const GradTensor& g, float s, const RngStream& rng) {
    return ternarize(g.name, std::span<const float>(g.values), s, rng);
}

// codec.hpp:177-182
inline GradTensor decode(const TernaryBlock& blk) {
    GradTensor out(blk.name, {blk.n});
    if (blk.n == 0) return out;
    detail::DevBuf<uint8_t> c(blk.codes.size());
    detail::DevBuf<float> o(blk.n);
    c.upload(blk.codes.data(), blk.codes.size());
    detail::check(tgb_layer_decode(c.p, blk.n, blk.s, o.p, nullptr), "tgb_layer_decode");
    detail::layer_check(blk.name);
    o.download(out.values.data(), blk.n);
    return out;
}

// codec.hpp:485-517 (device histogram; edges/counts identical to the reference's)
struct HistogramBin {
    double edge;
    std::size_t count;
};

inline std::vector<HistogramBin> histogram(std::span<const float> v, std::size_t bins) {
    if (bins < 1) throw std::invalid_argument("histogram: bins must be >= 1");
    detail::DevBuf<float> d(v.size());
    d.upload(v.data(), v.size());
    detail::DevBuf<uint64_t> c(bins);
    detail::DevBuf<double> e(bins);
    detail::check(tgb_layer_histogram(d.p, v.size(), static_cast<uint32_t>(bins), c.p, e.p, nullptr),
                  "tgb_layer_histogram");
    std::vector<uint64_t> hc(bins);
    std::vector<double> he(bins);
    c.download(hc.data(), bins);
    e.download(he.data(), bins);
    std::vector<HistogramBin> out(bins);
    for (std::size_t b = 0; b < bins; ++b) out[b] = {he[b], static_cast<std::size_t>(hc[b])};
    return out;
}
inline std::vector<HistogramBin> histogram(const GradTensor& g, std::size_t bins) {
    return histogram(std::span<const float>(g.values), bins);
}

namespace detail {
// one plan per call (value semantics); the hot path keeps plans alive in SyncWorker
struct PlanHolder {
    tgb_plan* p = nullptr;
    ~PlanHolder() { tgb_plan_destroy(p); }
};

inline bool is_passthrough(const CodecConfig& cfg, const std::string& name) {
    return cfg.float_mode || cfg.passthrough.count(name) != 0;  // cluster.hpp:274-275
}

// plan error -> the reference's CodecError text; corrupt-code indices are
// reported by the device per tensor and converted to the bucket's element
[[noreturn]] inline void throw_plan_error(const tgb_plan* p, const tgb_error& e,
                                          const std::vector<std::string>& names,
                                          uint64_t t = 0) {
    if (e.flags & TGB_E_SKEW)  // cluster.hpp:141-143
        throw ProtocolError("server: iteration skew, expected " + std::to_string(t) + " got " +
                            std::to_string(e.aux));
    const std::string nm =
        e.layer >= 0 && e.layer < static_cast<int32_t>(names.size()) ? names[e.layer] : "?";
    if (e.flags & TGB_E_NONFINITE) throw CodecError("encode_step: non-finite gradient " + nm);
    if (e.flags & TGB_E_CORRUPT_CODE) {
        uint64_t k = e.index;
        tgb_plan_info info{};
        if (tgb_plan_get_info(p, &info) == TGB_OK)
            for (int32_t b = 0; b < info.n_blocks; ++b) {
                tgb_block_info bi{};
                if (tgb_plan_block_info(p, b, &bi) == TGB_OK && bi.layer == e.layer &&
                    bi.offset <= e.index && e.index < bi.offset + bi.n)
                    k = e.index - bi.offset;
            }
        throw CodecError("corrupt ternary code 11 in block " + nm + " at element " +
                         std::to_string(k));
    }
    if (e.flags & TGB_E_PEER_TIMEOUT)
        throw CodecError("fused exchange: peer " + std::to_string(e.index) +
                         " never reached the step barrier");
    throw CodecError("codec error in " + nm);
}
}  // namespace detail

// codec.hpp:194-239: clip -> bucket scalers -> ternarize; passthrough tensors verbatim
inline EncodeResult encode_step(const std::vector<GradTensor>& grads, const CodecConfig& cfg,
                                uint64_t t, uint16_t worker) {
    cfg.validate();
    const int nl = static_cast<int>(grads.size());
    std::vector<tgb_layer_desc> d(nl);
    std::vector<size_t> offs(nl);
    std::vector<std::string> names(nl);
    size_t total = 0;
    for (int l = 0; l < nl; ++l) {
        names[l] = grads[l].name;
        d[l] = tgb_layer_desc{grads[l].size(), fnv1a64(grads[l].name),
                              detail::is_passthrough(cfg, grads[l].name) ? TGB_LAYER_PASSTHROUGH
                                                                          : 0u,
                              0u};
        offs[l] = total;
        total += (grads[l].size() + 3) / 4 * 4;  // 16-byte aligned tensors
    }
    detail::PlanHolder P;
    const tgb_codec_params prm = cfg.params();
    detail::check(tgb_plan_create(d.data(), nl, &prm, worker, 1, &P.p), "tgb_plan_create");
    detail::DevBuf<float> g(total ? total : 1);
    std::vector<const float*> gp(nl);
    std::vector<float*> op(nl);
    for (int l = 0; l < nl; ++l) {
        if (grads[l].size())
            detail::cuda_check(cudaMemcpy(g.p + offs[l], grads[l].values.data(),
                                          grads[l].size() * sizeof(float), cudaMemcpyHostToDevice),
                               "H2D");
        gp[l] = g.p + offs[l];
        op[l] = g.p + offs[l];  // encode only: decode output unused
    }
    detail::check(tgb_plan_bind(P.p, gp.data(), op.data()), "tgb_plan_bind");
    detail::check(tgb_encode(P.p, t, nullptr), "tgb_encode");
    tgb_error e{};
    const tgb_status st = tgb_check(P.p, &e);
    if (st == TGB_ERR_CODEC) detail::throw_plan_error(P.p, e, names);
    detail::check(st, "tgb_check");
    uint8_t *push = nullptr, *gath = nullptr;
    detail::check(tgb_plan_last_buffers(P.p, &push, &gath), "tgb_plan_last_buffers");
    tgb_plan_info info{};
    detail::check(tgb_plan_get_info(P.p, &info), "tgb_plan_get_info");
    std::vector<uint8_t> host(info.push_bytes);
    detail::cuda_check(cudaMemcpy(host.data(), push, info.push_bytes, cudaMemcpyDeviceToHost), "D2H");
    EncodeResult r;
    r.encoded.iteration = t;
    r.encoded.worker = worker;
    r.local_scalers.resize(info.n_slots);
    std::memcpy(r.local_scalers.data(), host.data(), 4ull * info.n_slots);
    for (int32_t b = 0; b < info.n_blocks; ++b) {
        tgb_block_info bi{};
        detail::check(tgb_plan_block_info(P.p, b, &bi), "tgb_plan_block_info");
        const uint8_t* reg = host.data() + bi.region_offset;
        if (bi.flags & TGB_LAYER_PASSTHROUGH) {
            PassthroughBlock pb;
            pb.name = grads[bi.layer].name;
            pb.values.resize(bi.n);
            std::memcpy(pb.values.data(), reg, 4 * bi.n);
            r.encoded.blocks.push_back(std::move(pb));
            continue;
        }
        TernaryBlock tb;
        tb.name = grads[bi.layer].name;
        tb.n = static_cast<uint32_t>(bi.n);
        tb.s = r.local_scalers[bi.slot];
        tb.codes.assign(reg, reg + (bi.n + 3) / 4);
        r.encoded.blocks.push_back(std::move(tb));
    }
    return r;
}

// codec.hpp:245-311
inline std::vector<GradTensor> average(const std::vector<EncodedGradient>& encoded, std::size_t N,
                                       bool scaler_sharing) {
    if (encoded.size() != N || N == 0)
        throw CodecError("average: expected " + std::to_string(N) + " messages, got " +
                         std::to_string(encoded.size()));
    const std::size_t nblocks = encoded[0].blocks.size();
    for (const auto& e : encoded) {
        if (e.iteration != encoded[0].iteration) throw CodecError("average: mismatched iterations");
        if (e.blocks.size() != nblocks) throw CodecError("average: mismatched block structure");
    }
    std::vector<GradTensor> out;
    auto append = [&](const std::string& name, std::vector<float>&& avg) {
        if (!out.empty() && out.back().name == name) {  // merge bucket runs by name
            out.back().values.insert(out.back().values.end(), avg.begin(), avg.end());
            out.back().shape = {out.back().values.size()};
        } else {
            const std::size_t n = avg.size();
            out.emplace_back(name, std::vector<std::size_t>{n}, std::move(avg));
        }
    };
    for (std::size_t b = 0; b < nblocks; ++b) {
        if (const auto* pf = std::get_if<PassthroughBlock>(&encoded[0].blocks[b])) {
            const std::size_t n = pf->values.size();
            std::vector<detail::DevBuf<float>> vals;
            std::vector<const float*> ptrs;
            for (const auto& e : encoded) {
                const auto* pb = std::get_if<PassthroughBlock>(&e.blocks[b]);
                if (!pb || pb->name != pf->name || pb->values.size() != n)
                    throw CodecError("average: block structure mismatch at " + pf->name);
                vals.emplace_back(n);
                vals.back().upload(pb->values.data(), n);
                ptrs.push_back(vals.back().p);
            }
            std::vector<float> avg(n);
            if (n) {
                detail::DevBuf<float> o(n);
                detail::check(tgb_layer_average_raw(static_cast<int32_t>(N), ptrs.data(), n, o.p,
                                                    nullptr),
                              "tgb_layer_average_raw");
                detail::layer_check(pf->name);
                o.download(avg.data(), n);
            }
            append(pf->name, std::move(avg));
            continue;
        }
        const TernaryBlock& first = std::get<TernaryBlock>(encoded[0].blocks[b]);
        for (const auto& e : encoded) {
            const auto* tb = std::get_if<TernaryBlock>(&e.blocks[b]);
            if (!tb || tb->name != first.name || tb->n != first.n)
                throw CodecError("average: block structure mismatch at " + first.name);
        }
        std::vector<float> avg(first.n);
        if (first.n) {
            std::vector<detail::DevBuf<uint8_t>> codes;
            std::vector<const uint8_t*> ptrs;
            std::vector<float> s;
            for (const auto& e : encoded) {
                const TernaryBlock& tb = std::get<TernaryBlock>(e.blocks[b]);
                codes.emplace_back(tb.codes.size());
                codes.back().upload(tb.codes.data(), tb.codes.size());
                ptrs.push_back(codes.back().p);
                s.push_back(tb.s);
            }
            detail::DevBuf<float> ds(N), o(first.n);
            ds.upload(s.data(), N);
            detail::check(tgb_layer_average(static_cast<int32_t>(N), ptrs.data(), ds.p, first.n,
                                            scaler_sharing ? 1 : 0, o.p, nullptr),
                          "tgb_layer_average");
            detail::layer_check(first.name);
            o.download(avg.data(), first.n);
        }
        append(first.name, std::move(avg));
    }
    return out;
}

// NCCL communicator (one process per GPU)
class Comm {
public:
    static std::vector<uint8_t> unique_id() {
        std::vector<uint8_t> id(TGB_UNIQUE_ID_BYTES);
        detail::check(tgb_comm_unique_id(id.data()), "tgb_comm_unique_id");
        return id;
    }
    Comm(const std::vector<uint8_t>& id, int nranks, int rank) {
        detail::check(tgb_comm_init(id.data(), nranks, rank, &c_), "tgb_comm_init");
    }
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    ~Comm() { tgb_comm_destroy(c_); }
    tgb_comm* get() const { return c_; }

private:
    tgb_comm* c_ = nullptr;
};

// TrafficStats (cluster.hpp:62-74): framed bytes of the reference's wire format
// and the same tensors at raw fp32, plus the bytes this build's exchange moved
// between GPUs (NVLink)
struct TrafficStats {
    uint64_t bytes_up = 0, bytes_down = 0, float_bytes_up = 0, float_bytes_down = 0;
    uint64_t device_bytes_out = 0, device_bytes_in = 0;
    double up_reduction() const {
        return bytes_up ? static_cast<double>(float_bytes_up) / bytes_up : 1.0;
    }
    double down_reduction() const {
        return bytes_down ? static_cast<double>(float_bytes_down) / bytes_down : 1.0;
    }
    TrafficStats& operator+=(const tgb_traffic& t) {
        bytes_up += t.bytes_up;
        bytes_down += t.bytes_down;
        float_bytes_up += t.float_bytes_up;
        float_bytes_down += t.float_bytes_down;
        device_bytes_out += t.device_bytes_out;
        device_bytes_in += t.device_bytes_in;
        return *this;
    }
};

// Worker::run sync segment (cluster.hpp:283-297) with gradients resident in HBM:
// grads() -> [fill] -> step(t) -> outputs() hold the averaged gradient, identical
// on every rank. exchange: TGB_EXCHANGE_AUTO / _FUSED / _SHARDED (NVLink peer
// stores, attached here; ranks with different plans throw ProtocolError) or
// TGB_EXCHANGE_NCCL (ncclAllGather of the push areas).
class SyncWorker {
public:
    SyncWorker(std::vector<std::string> names, std::vector<std::size_t> sizes,
               const CodecConfig& cfg, int rank = 0, int world_size = 1, Comm* comm = nullptr,
               int exchange = TGB_EXCHANGE_AUTO)
        : names_(std::move(names)), sizes_(std::move(sizes)), comm_(comm) {
        cfg.validate();
        const int nl = static_cast<int>(names_.size());
        std::vector<tgb_layer_desc> d(nl);
        offs_.resize(nl);
        std::size_t total = 0;
        for (int l = 0; l < nl; ++l) {
            d[l] = tgb_layer_desc{sizes_[l], fnv1a64(names_[l]),
                                  detail::is_passthrough(cfg, names_[l]) ? TGB_LAYER_PASSTHROUGH
                                                                         : 0u,
                                  0u};
            offs_[l] = total;
            total += (sizes_[l] + 3) / 4 * 4;
        }
        const tgb_codec_params prm = cfg.params();
        detail::check(tgb_plan_create(d.data(), nl, &prm, static_cast<uint16_t>(rank), world_size,
                                      &plan_),
                      "tgb_plan_create");
        grads_ = detail::DevBuf<float>(total ? total : 1);
        outs_ = detail::DevBuf<float>(total ? total : 1);
        detail::cuda_check(cudaMemset(grads_.p, 0, grads_.n * sizeof(float)), "memset");
        std::vector<const float*> gp(nl);
        std::vector<float*> op(nl);
        for (int l = 0; l < nl; ++l) {
            gp[l] = grads_.p + offs_[l];
            op[l] = outs_.p + offs_[l];
        }
        detail::check(tgb_plan_bind(plan_, gp.data(), op.data()), "tgb_plan_bind");
        std::vector<const char*> cn(nl);
        for (int l = 0; l < nl; ++l) cn[l] = names_[l].c_str();
        detail::check(tgb_plan_set_names(plan_, cn.data()), "tgb_plan_set_names");
        if (world_size > 1 && exchange != TGB_EXCHANGE_NCCL) {
            if (exchange != TGB_EXCHANGE_AUTO)
                detail::check(tgb_plan_set_option(plan_, TGB_PLAN_OPT_EXCHANGE, exchange),
                              "tgb_plan_set_option");
            const tgb_status st = tgb_plan_attach_peers(plan_, comm_ ? comm_->get() : nullptr);
            if (st == TGB_ERR_PROTOCOL) throw ProtocolError(tgb_last_error_message());
            detail::check(st, "tgb_plan_attach_peers");
        }
        detail::check(tgb_plan_traffic(plan_, &step_traffic_), "tgb_plan_traffic");
    }
    SyncWorker(const SyncWorker&) = delete;
    SyncWorker& operator=(const SyncWorker&) = delete;
    ~SyncWorker() { tgb_plan_destroy(plan_); }

    float* grad(int layer) { return grads_.p + offs_[layer]; }     // device
    float* output(int layer) { return outs_.p + offs_[layer]; }    // device
    void step(uint64_t t, cudaStream_t stream = nullptr) {
        detail::check(tgb_step(plan_, comm_ ? comm_->get() : nullptr, t, stream), "tgb_step");
        last_t_ = t;
        traffic_ += step_traffic_;
    }
    // synchronises; throws CodecError / ProtocolError with the reference's message
    // on a device error
    void check() {
        tgb_error e{};
        const tgb_status st = tgb_check(plan_, &e);
        if (st == TGB_ERR_CODEC) detail::throw_plan_error(plan_, e, names_, last_t_);
        detail::check(st, "tgb_check");
    }
    // accumulated over the steps so far (ParameterServer::traffic(), cluster.hpp:167)
    const TrafficStats& traffic() const { return traffic_; }
    // host buffers in/out (pinned recommended): tgb_step_host
    void step_host(uint64_t t, const std::vector<const float*>& h_grads,
                   const std::vector<float*>& h_out, cudaStream_t stream = nullptr) {
        detail::check(tgb_step_host(plan_, comm_ ? comm_->get() : nullptr, t, h_grads.data(),
                                    h_out.data(), stream),
                      "tgb_step_host");
        last_t_ = t;
        traffic_ += step_traffic_;
    }
    // interop with the reference's parameter server (wire.hpp): the push frame of the
    // last encode, byte-identical to frame(Message{Push, t, rank, serialize_encoded(...)})
    std::vector<uint8_t> serialize_push(uint64_t t, cudaStream_t stream = nullptr) {
        uint64_t n = 0;
        detail::check(tgb_plan_push_frame_size(plan_, &n), "tgb_plan_push_frame_size");
        std::vector<uint8_t> f(n);
        detail::check(tgb_plan_serialize_push(plan_, t, f.data(), stream), "tgb_plan_serialize_push");
        return f;
    }
    // decode_pull(deserialize_pull(unframe(frame).payload)) into output(l); returns the iteration
    uint64_t decode_pull(std::span<const uint8_t> frame, cudaStream_t stream = nullptr) {
        uint64_t it = 0;
        const tgb_status st = tgb_plan_decode_pull(plan_, frame.data(), frame.size(), &it, stream);
        if (st == TGB_ERR_PROTOCOL) throw ProtocolError(tgb_last_error_message());
        detail::check(st, "tgb_plan_decode_pull");
        return it;
    }
    // Worker::zero_fraction of the last step's encode (cluster.hpp:336-346)
    void enable_code_stats(bool on = true) {
        detail::check(tgb_plan_enable_code_stats(plan_, on ? 1 : 0), "tgb_plan_enable_code_stats");
    }
    double zero_fraction() {
        uint64_t nz = 0, tot = 0;
        detail::check(tgb_plan_code_stats(plan_, &nz, &tot), "tgb_plan_code_stats");
        return tot ? static_cast<double>(tot - nz) / static_cast<double>(tot) : 0.0;
    }
    tgb_plan* plan() const { return plan_; }

private:
    std::vector<std::string> names_;
    std::vector<std::size_t> sizes_;
    std::vector<std::size_t> offs_;
    Comm* comm_;
    tgb_plan* plan_ = nullptr;
    detail::DevBuf<float> grads_, outs_;
    uint64_t last_t_ = 0;
    tgb_traffic step_traffic_{};
    TrafficStats traffic_;
};

}  // namespace tgb
