// TEST INFRASTRUCTURE ONLY — a C-ABI shim over the UNMODIFIED reference
// headers (/root/reference/proj/include/terngrad/*.hpp, included at compile
// time, never copied). Built by oracle/Makefile into oracle/_ref/libtgref.so
// with the reference's own Release flags (-O3 -DNDEBUG -std=gnu++20,
// proj/CMakeLists.txt:4-9). It is the parity anchor for oracle/tg_oracle.c
// and the "reference" CPU baseline timed by bench.py --impl reference.
//
// Nothing in the product path loads this library.

#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "terngrad/cluster.hpp"
#include "terngrad/codec.hpp"
#include "terngrad/optimizer.hpp"
#include "terngrad/rng.hpp"
#include "terngrad/transport.hpp"
#include "terngrad/wire.hpp"

using namespace terngrad;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return 1;
}

CodecConfig make_cfg(float clip_factor, int clipping, int bucketing, std::uint64_t bucket_size,
                     int sharing, std::uint64_t seed) {
    CodecConfig c;
    c.clip_factor = clip_factor;
    c.clipping_enabled = clipping != 0;
    c.bucketing = bucketing == 1 ? Bucketing::Global
                                 : (bucketing == 2 ? Bucketing::FixedSize : Bucketing::PerTensor);
    c.bucket_size = bucket_size;
    c.scaler_sharing = sharing != 0;
    c.seed = seed;
    return c;
}

std::vector<GradTensor> make_grads(int n_tensors, const char* const* names,
                                   const std::uint64_t* ns, const float* const* grads) {
    std::vector<GradTensor> g;
    g.reserve(n_tensors);
    for (int l = 0; l < n_tensors; ++l) {
        std::vector<float> v(grads[l], grads[l] + ns[l]);
        std::vector<std::size_t> shape;
        if (ns[l] > 0) shape = {static_cast<std::size_t>(ns[l])};
        else shape = {0};
        g.emplace_back(names[l], shape, std::move(v));
    }
    return g;
}
}  // namespace

extern "C" {

const char* tgref_last_error() { return g_err.c_str(); }

// rng.hpp:20-33
void tgref_philox(const std::uint32_t ctr[4], const std::uint32_t key[2], std::uint32_t out[4]) {
    auto r = philox::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}

// rng.hpp:37-44
std::uint64_t tgref_fnv1a64(const char* s, std::size_t len) {
    return fnv1a64(std::string_view(s, len));
}

// rng.hpp:59-71
void tgref_rng_bits(std::uint64_t seed, std::uint64_t t, const char* name, std::uint64_t worker,
                    std::uint64_t k0, std::size_t n, std::uint32_t* out) {
    RngStream r(seed, t, name, worker);
    for (std::size_t k = 0; k < n; ++k) out[k] = r.bits(k0 + k);
}

void tgref_rng_uniform(std::uint64_t seed, std::uint64_t t, const char* name,
                       std::uint64_t worker, std::uint64_t k0, std::size_t n, float* out) {
    RngStream r(seed, t, name, worker);
    for (std::size_t k = 0; k < n; ++k) out[k] = r.uniform(k0 + k);
}

// rng.hpp:74-79
void tgref_normal_fill(std::uint64_t seed, std::uint64_t t, const char* name,
                       std::uint64_t worker, std::uint64_t k0, std::size_t n, float scale,
                       float* out) {
    RngStream r(seed, t, name, worker);
    for (std::size_t k = 0; k < n; ++k) out[k] = scale * r.normal(k0 + k);
}

// codec.hpp:101-124: clip; bound returned through *bound (inf when n < 2)
double tgref_stddev(const float* v, std::size_t n) {
    return stddev(std::span<const float>(v, n));
}

void tgref_clip(const float* in, std::size_t n, float c, float* out, float* bound) {
    GradTensor g("g", {n}, std::vector<float>(in, in + n));
    GradTensor r = clip(g, c);
    std::memcpy(out, r.values.data(), n * sizeof(float));
    if (bound)
        *bound = n < 2 ? INFINITY : static_cast<float>(c * stddev(std::span<const float>(in, n)));
}

// codec.hpp:128-134
float tgref_scaler(const float* v, std::size_t n) { return scaler(std::span<const float>(v, n)); }

// codec.hpp:148-175
int tgref_ternarize(const char* name, const float* g, std::size_t n, float s, std::uint64_t seed,
                    std::uint64_t t, std::uint64_t worker, std::uint64_t rng_base,
                    std::uint8_t* codes) {
    try {
        RngStream r(seed, t, name, worker);
        TernaryBlock b = ternarize(name, std::span<const float>(g, n), s, r, rng_base);
        std::memcpy(codes, b.codes.data(), b.codes.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// codec.hpp:177-182
int tgref_decode(const std::uint8_t* codes, std::size_t n, float s, float* out) {
    try {
        TernaryBlock b;
        b.name = "g";
        b.n = static_cast<std::uint32_t>(n);
        b.s = s;
        b.codes.assign(codes, codes + (n + 3) / 4);
        GradTensor d = decode(b);
        std::memcpy(out, d.values.data(), n * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// codec.hpp:194-239. Writes block codes back to back and one scaler per block.
// passthrough[l] != 0 puts names[l] into cfg.passthrough.
int tgref_encode_step(int n_tensors, const char* const* names, const std::uint64_t* ns,
                      const float* const* grads, const int* passthrough, float clip_factor,
                      int clipping, int bucketing, std::uint64_t bucket_size, int sharing,
                      std::uint64_t seed, std::uint64_t t, std::uint16_t worker,
                      std::uint8_t* codes, float* scalers, std::uint64_t* n_blocks) {
    try {
        CodecConfig cfg = make_cfg(clip_factor, clipping, bucketing, bucket_size, sharing, seed);
        for (int l = 0; l < n_tensors; ++l)
            if (passthrough && passthrough[l]) cfg.passthrough.insert(names[l]);
        auto g = make_grads(n_tensors, names, ns, grads);
        EncodeResult r = encode_step(g, cfg, t, worker);
        std::size_t pos = 0, nb = 0;
        for (const auto& blk : r.encoded.blocks) {
            if (const auto* tb = std::get_if<TernaryBlock>(&blk)) {
                std::memcpy(codes + pos, tb->codes.data(), tb->codes.size());
                pos += tb->codes.size();
                ++nb;
            }
        }
        for (std::size_t i = 0; i < r.local_scalers.size(); ++i) scalers[i] = r.local_scalers[i];
        if (n_blocks) *n_blocks = nb;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// codec.hpp:245-311 over N workers' encode_step outputs for the same tensor
// list (the whole multi-tensor `average`, merged by name). out receives the
// concatenated averaged tensors in canonical order.
int tgref_average_encoded(int N, int n_tensors, const char* const* names, const std::uint64_t* ns,
                          const float* const* grads_per_worker /* [N * n_tensors] */,
                          const int* passthrough, float clip_factor, int clipping, int bucketing,
                          std::uint64_t bucket_size, int sharing, std::uint64_t seed,
                          std::uint64_t t, float* out) {
    try {
        CodecConfig cfg = make_cfg(clip_factor, clipping, bucketing, bucket_size, sharing, seed);
        for (int l = 0; l < n_tensors; ++l)
            if (passthrough && passthrough[l]) cfg.passthrough.insert(names[l]);
        std::vector<EncodedGradient> enc;
        for (int w = 0; w < N; ++w) {
            auto g = make_grads(n_tensors, names, ns, grads_per_worker + std::size_t(w) * n_tensors);
            enc.push_back(encode_step(g, cfg, t, static_cast<std::uint16_t>(w)).encoded);
        }
        auto avg = average(enc, N, cfg.scaler_sharing);
        std::size_t pos = 0;
        for (const auto& a : avg) {
            std::memcpy(out + pos, a.values.data(), a.values.size() * sizeof(float));
            pos += a.values.size();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference's own sync path as shipped (cluster.hpp:135-221 + 283-297):
// N workers encode + push over InProcessHub, ParameterServer::step folds and
// broadcasts the radix-packed Pull, every worker decode_pulls. out receives
// worker 0's decoded averaged gradient (identical on every worker).
struct tgref_cluster {
    int N;
    CodecConfig cfg;
    std::vector<std::vector<GradTensor>> grads;  // [worker][tensor]
    std::unique_ptr<InProcessHub> hub;
    std::unique_ptr<InProcessServerTransport> st;
    std::unique_ptr<ParameterServer> server;
    std::vector<std::unique_ptr<InProcessWorkerTransport>> wts;
    std::vector<std::vector<GradTensor>> decoded;
    std::vector<std::vector<std::uint8_t>> push_frames, pull_frames;  // per worker, last step
};

tgref_cluster* tgref_cluster_create(int N, int n_tensors, const char* const* names,
                                    const std::uint64_t* ns,
                                    const float* const* grads_per_worker, const int* passthrough,
                                    float clip_factor, int clipping, int bucketing,
                                    std::uint64_t bucket_size, int sharing, std::uint64_t seed) {
    try {
        auto* c = new tgref_cluster;
        c->N = N;
        c->cfg = make_cfg(clip_factor, clipping, bucketing, bucket_size, sharing, seed);
        for (int l = 0; l < n_tensors; ++l)
            if (passthrough && passthrough[l]) c->cfg.passthrough.insert(names[l]);
        for (int w = 0; w < N; ++w)
            c->grads.push_back(
                make_grads(n_tensors, names, ns, grads_per_worker + std::size_t(w) * n_tensors));
        c->hub = std::make_unique<InProcessHub>(N);
        c->st = std::make_unique<InProcessServerTransport>(*c->hub);
        c->server = std::make_unique<ParameterServer>(*c->st, N, c->cfg.scaler_sharing);
        for (int w = 0; w < N; ++w)
            c->wts.push_back(
                std::make_unique<InProcessWorkerTransport>(*c->hub, static_cast<std::uint16_t>(w)));
        c->decoded.resize(N);
        c->push_frames.resize(N);
        c->pull_frames.resize(N);
        return c;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// One synchronous step; returns wall seconds (or -1 on error).
double tgref_cluster_step(tgref_cluster* c, std::uint64_t t) {
    std::vector<std::string> errs(c->N + 1);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int w = 0; w < c->N; ++w)
        th.emplace_back([c, w, t, &errs] {
            try {
                auto enc = encode_step(c->grads[w], c->cfg, t, static_cast<std::uint16_t>(w));
                Message push;
                push.type = MsgType::Push;
                push.iteration = t;
                push.worker = static_cast<std::uint16_t>(w);
                push.payload = serialize_encoded(enc.encoded);
                c->push_frames[w] = frame(push);
                c->wts[w]->send(push);
                const Message reply = c->wts[w]->recv();
                c->pull_frames[w] = frame(reply);
                c->decoded[w] = decode_pull(deserialize_pull(reply.payload));
            } catch (const std::exception& e) {
                errs[w + 1] = e.what();
            }
        });
    try {
        c->server->step(t);
    } catch (const std::exception& e) {
        errs[0] = e.what();
    }
    for (auto& x : th) x.join();
    const auto t1 = std::chrono::steady_clock::now();
    for (auto& e : errs)
        if (!e.empty()) {
            g_err = e;
            return -1.0;
        }
    return std::chrono::duration<double>(t1 - t0).count();
}

void tgref_cluster_output(tgref_cluster* c, int worker, float* out) {
    std::size_t pos = 0;
    for (const auto& a : c->decoded[worker]) {
        std::memcpy(out + pos, a.values.data(), a.values.size() * sizeof(float));
        pos += a.values.size();
    }
}

// the last step's wire frames of `worker` (which 0 = its push, 1 = the pull it
// received), as the reference's socket transport would carry them; returns the
// size, copies min(size, cap) bytes
std::size_t tgref_cluster_frame(tgref_cluster* c, int worker, int which, std::uint8_t* out,
                                std::size_t cap) {
    const auto& f = which == 0 ? c->push_frames[worker] : c->pull_frames[worker];
    if (out) std::memcpy(out, f.data(), std::min(cap, f.size()));
    return f.size();
}

void tgref_cluster_destroy(tgref_cluster* c) { delete c; }

// codec.hpp:491-517
int tgref_histogram(const float* v, std::size_t n, std::size_t bins, double* edges,
                    std::uint64_t* counts) {
    try {
        auto h = histogram(std::span<const float>(v, n), bins);
        for (std::size_t b = 0; b < bins; ++b) {
            edges[b] = h[b].edge;
            counts[b] = h[b].count;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// optimizer.hpp:80-125: `steps` applies of one OptimizerState to one tensor;
// grads holds steps x n floats, rates steps doubles; w is updated in place
int tgref_optimizer_run(int rule, double momentum, double beta1, double beta2, double epsilon,
                        double weight_decay, int steps, std::size_t n, float* w,
                        const float* grads, const double* rates) {
    try {
        OptimizerConfig cfg;
        cfg.rule = static_cast<OptimizerRule>(rule);
        cfg.momentum = momentum;
        cfg.beta1 = beta1;
        cfg.beta2 = beta2;
        cfg.epsilon = epsilon;
        cfg.weight_decay = weight_decay;
        OptimizerState st(cfg);
        std::vector<GradTensor> params{GradTensor("w", {n}, std::vector<float>(w, w + n))};
        for (int k = 0; k < steps; ++k) {
            std::vector<GradTensor> g{GradTensor("w", {n}, std::vector<float>(
                                                                grads + k * n, grads + (k + 1) * n))};
            st.apply(params, g, rates[k]);
        }
        std::memcpy(w, params[0].values.data(), n * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
