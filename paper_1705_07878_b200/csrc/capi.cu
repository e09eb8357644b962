// C-ABI implementation (include/tgb/terngrad_b200.h), non-plan half: version and
// status strings, the optimizer, the reference wire format and traffic
// accounting, the NCCL communicator and the per-layer entry points. Host code
// only; plans and the step live in plan.cu, kernels in kernels.cu.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "tgb_plan.h"

using namespace tgb;

namespace {

thread_local std::string g_last_error;  // tgb_last_error_message (PROTOCOL detail)

inline tgb_status protocol_error(const std::string& msg) {
    g_last_error = msg;
    return TGB_ERR_PROTOCOL;
}

#define TGB_CUDA(expr)                                  \
    do {                                                \
        const cudaError_t e_ = (expr);                  \
        if (e_ != cudaSuccess) return TGB_ERR_CUDA;     \
    } while (0)

#define TGB_NCCL(expr)                                  \
    do {                                                \
        const ncclResult_t r_ = (expr);                 \
        if (r_ != ncclSuccess) return TGB_ERR_NCCL;     \
    } while (0)

#define TGB_TRY_INNER(expr)                  \
    do {                                     \
        const tgb_status s_ = (expr);        \
        if (s_ != TGB_OK) return s_;         \
    } while (0)

// per-device scratch for the per-layer API (error word, K1 partials)
struct DeviceScratch {
    ErrWord* err = nullptr;
    uint32_t* counters = nullptr;  // [0] layer_done, [1] global_done
    float* tmp = nullptr;          // [0] slot, [1] bound
    bool ready = false;
};
DeviceScratch g_scratch[64];

tgb_status scratch(DeviceScratch** out) {
    int dev = 0;
    TGB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return TGB_ERR_CUDA;
    DeviceScratch& s = g_scratch[dev];
    if (!s.ready) {
        TGB_CUDA(cudaMalloc(&s.err, sizeof(ErrWord)));
        TGB_CUDA(cudaMemset(s.err, 0, sizeof(ErrWord)));
        TGB_CUDA(cudaMalloc(&s.counters, 2 * sizeof(uint32_t)));
        TGB_CUDA(cudaMemset(s.counters, 0, 2 * sizeof(uint32_t)));
        TGB_CUDA(cudaMalloc(&s.tmp, 2 * sizeof(float)));
        s.ready = true;
    }
    *out = &s;
    return TGB_OK;
}

}  // namespace

namespace tgb {
tgb_status set_protocol_error(const std::string& msg) { return protocol_error(msg); }
}  // namespace tgb

extern "C" {

const char* tgb_version(void) { return "terngrad_b200 2 (sm_100a)"; }

const char* tgb_status_string(tgb_status s) {
    switch (s) {
        case TGB_OK: return "ok";
        case TGB_ERR_INVALID_ARGUMENT: return "invalid argument";
        case TGB_ERR_CODEC: return "codec error";
        case TGB_ERR_CUDA: return "CUDA error";
        case TGB_ERR_NCCL: return "NCCL error";
        case TGB_ERR_UNSUPPORTED: return "unsupported configuration";
        case TGB_ERR_PROTOCOL: return "protocol error";
    }
    return "unknown";
}

uint64_t tgb_fnv1a64(const char* s, size_t len) {  // rng.hpp:37-44
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < len; ++i) {
        h ^= static_cast<unsigned char>(s[i]);
        h *= 0x100000001b3ull;
    }
    return h;
}

int32_t tgb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ------------------------------------------------------------ optimizer
static tgb_status make_opt(const tgb_optimizer* opt, uint64_t step, double rate, OptArgs* o) {
    if (!opt || opt->rule < TGB_OPT_VANILLA || opt->rule > TGB_OPT_ADAM)
        return TGB_ERR_INVALID_ARGUMENT;
    o->rule = opt->rule;
    o->wd_f = static_cast<float>(opt->weight_decay);  // optimizer.hpp:95,103
    o->mu_f = static_cast<float>(opt->momentum);
    o->rate_f = static_cast<float>(rate);
    o->wd = opt->weight_decay;
    o->b1 = opt->beta1;
    o->omb1 = 1.0 - opt->beta1;
    o->b2 = opt->beta2;
    o->omb2 = 1.0 - opt->beta2;
    o->eps = opt->epsilon;
    o->rate = rate;
    o->bc1 = 1.0 - std::pow(opt->beta1, static_cast<double>(step));  // optimizer.hpp:111-112
    o->bc2 = 1.0 - std::pow(opt->beta2, static_cast<double>(step));
    return TGB_OK;
}

tgb_status tgb_optimizer_apply(const tgb_optimizer* opt, uint64_t step, double rate,
                               int32_t n_layers, const uint64_t* ns, float* const* d_params,
                               const float* const* d_grads, float* const* d_state1,
                               float* const* d_state2, void* stream) {
    OptArgs o{};
    TGB_TRY_INNER(make_opt(opt, step, rate, &o));
    if (n_layers < 0 || (n_layers > 0 && (!ns || !d_params || !d_grads)))
        return TGB_ERR_INVALID_ARGUMENT;
    const bool need1 = opt->rule != TGB_OPT_VANILLA, need2 = opt->rule == TGB_OPT_ADAM;
    for (int32_t l = 0; l < n_layers; ++l) {
        if (ns[l] == 0) continue;
        float* s1 = need1 ? (d_state1 ? d_state1[l] : nullptr) : nullptr;
        float* s2 = need2 ? (d_state2 ? d_state2[l] : nullptr) : nullptr;
        if (!d_params[l] || !d_grads[l] || (need1 && !s1) || (need2 && !s2))
            return TGB_ERR_INVALID_ARGUMENT;
        TGB_CUDA(launch_opt_apply(o, ns[l], d_params[l], d_grads[l], s1, s2,
                                  static_cast<cudaStream_t>(stream)));
    }
    return TGB_OK;
}

tgb_status tgb_plan_bind_optimizer(tgb_plan* P, const tgb_optimizer* opt, float* const* d_params,
                                   float* const* d_state1, float* const* d_state2) {
    OptArgs o{};
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    TGB_TRY_INNER(make_opt(opt, 1, 0.0, &o));
    const size_t nl = P->desc.size();
    const bool need1 = opt->rule != TGB_OPT_VANILLA, need2 = opt->rule == TGB_OPT_ADAM;
    if (nl > 0 && (!d_params || (need1 && !d_state1) || (need2 && !d_state2)))
        return TGB_ERR_INVALID_ARGUMENT;
    P->opt_w.assign(nl, nullptr);
    P->opt_s1.assign(nl, nullptr);
    P->opt_s2.assign(nl, nullptr);
    for (size_t l = 0; l < nl; ++l) {
        if (P->desc[l].n == 0) continue;
        P->opt_w[l] = d_params[l];
        if (need1) P->opt_s1[l] = d_state1[l];
        if (need2) P->opt_s2[l] = d_state2[l];
        if (!P->opt_w[l] || (need1 && !P->opt_s1[l]) || (need2 && !P->opt_s2[l]))
            return TGB_ERR_INVALID_ARGUMENT;
    }
    // per-block table for the fused decode -> optimizer kernels
    std::vector<OptDev> od(std::max<size_t>(1, P->h_layers.size()));
    for (size_t b = 0; b < P->h_layers.size(); ++b) {
        const LayerDev& L = P->h_layers[b];
        const uint64_t off = P->block_off[b];
        OptDev& d = od[b];
        d.w = P->opt_w[L.tensor] ? P->opt_w[L.tensor] + off : nullptr;
        d.s1 = P->opt_s1[L.tensor] ? P->opt_s1[L.tensor] + off : nullptr;
        d.s2 = P->opt_s2[L.tensor] ? P->opt_s2[L.tensor] + off : nullptr;
        auto al = [](const float* q) { return !q || (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
        d.vec = al(d.w) && al(d.s1) && al(d.s2) ? 1u : 0u;
    }
    if (!P->d_optd) TGB_CUDA(cudaMalloc(&P->d_optd, od.size() * sizeof(OptDev)));
    TGB_CUDA(cudaMemcpy(P->d_optd, od.data(), od.size() * sizeof(OptDev), cudaMemcpyHostToDevice));
    P->opt = *opt;
    P->opt_steps = 0;
    P->opt_bound = true;
    return TGB_OK;
}

// the step schedules whose decode kernel applies the optimizer in place of
// writing the averaged gradient: N = 1 (K2 fused decode) and the staged
// shared-scaler K3 of the fused / NCCL exchanges (N <= 8)
static bool opt_fusable(const tgb_plan* P) {
    if (!P->opt_fused) return false;  // TGB_PLAN_OPT_FUSED_OPTIMIZER
    if (P->n_workers == 1) return true;
    return P->p.scaler_sharing && !P->shard && P->n_workers <= kMaxPeers;
}

tgb_status tgb_step_apply(tgb_plan* P, tgb_comm* C, uint64_t t, double rate, void* stream) {
    if (!P || !P->opt_bound) return TGB_ERR_INVALID_ARGUMENT;
    OptArgs o{};
    TGB_TRY_INNER(make_opt(&P->opt, P->opt_steps + 1, rate, &o));
    if (opt_fusable(P)) {  // decode -> optimizer in one kernel; no averaged gradient written
        P->opt_active = &o;
        const tgb_status r = tgb_step(P, C, t, stream);
        P->opt_active = nullptr;
        if (r == TGB_OK) ++P->opt_steps;
        return r;
    }
    TGB_TRY_INNER(tgb_step(P, C, t, stream));
    ++P->opt_steps;
    auto st = static_cast<cudaStream_t>(stream);
    for (size_t l = 0; l < P->desc.size(); ++l)
        if (P->desc[l].n)
            TGB_CUDA(launch_opt_apply(o, P->desc[l].n, P->opt_w[l], P->bound_out[l], P->opt_s1[l],
                                      P->opt_s2[l], st));
    return TGB_OK;
}

// ----------------------------------------------------------------- wire
const char* tgb_last_error_message(void) { return g_last_error.c_str(); }

namespace {
void put_le(std::vector<uint8_t>& b, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
constexpr uint16_t kWireMagic = 0x5447;  // wire.hpp:18-19
constexpr uint8_t kWireVersion = 1;
constexpr uint64_t kHeaderSize = 18;  // wire.hpp:28-30
}  // namespace

// Static parts of the push frame (codec.hpp:395-438, wire.hpp:41-53) and the
// segment list of its per-step parts; names are needed by the wire format only.
tgb_status tgb_plan_set_names(tgb_plan* P, const char* const* names) {
    if (!P || (!names && !P->desc.empty())) return TGB_ERR_INVALID_ARGUMENT;
    const size_t nl = P->desc.size();
    P->names.assign(nl, std::string());
    for (size_t l = 0; l < nl; ++l) {
        if (!names[l]) return TGB_ERR_INVALID_ARGUMENT;
        P->names[l] = names[l];
        if (P->names[l].size() > 0xFFFF) return protocol_error("tensor name too long");
        if (tgb_fnv1a64(names[l], P->names[l].size()) != P->desc[l].name_hash)
            return TGB_ERR_INVALID_ARGUMENT;  // names must be the plan's tensors
    }
    cudaFree(P->d_frame);
    cudaFree(P->d_wsegs);
    P->d_frame = nullptr;
    P->d_wsegs = nullptr;
    P->push_frame_bytes = 0;
    if (P->h_layers.size() > 0xFFFF) return TGB_OK;  // u16 block count: no wire frames for this plan
    std::vector<uint8_t> f;
    put_le(f, kWireMagic, 2);
    f.push_back(kWireVersion);
    f.push_back(1);      // MsgType::Push
    put_le(f, 0, 8);     // iteration: patched per frame
    put_le(f, P->worker, 2);
    put_le(f, 0, 4);     // payload length: patched below
    put_le(f, P->h_layers.size(), 2);
    std::vector<WireSeg> segs;
    auto add = [&](uint64_t src, uint64_t dst, uint64_t bytes) {
        for (uint64_t o = 0; o < bytes; o += 65536)
            segs.push_back({src + o, dst + o, std::min<uint64_t>(65536, bytes - o)});
    };
    for (const LayerDev& L : P->h_layers) {
        const bool pass = (L.flags & kLayerPassthrough) != 0;
        const std::string& nm = P->names[L.tensor];
        f.push_back(pass ? 2 : 1);  // kBlockPassthrough / kBlockTernary
        put_le(f, nm.size(), 2);
        f.insert(f.end(), nm.begin(), nm.end());
        put_le(f, L.n, 4);
        if (pass) {
            add(L.code_off, f.size(), 4ull * L.n);
            f.resize(f.size() + 4ull * L.n);
        } else {
            add(4ull * static_cast<uint64_t>(L.slot), f.size(), 4);  // scaler slot
            f.resize(f.size() + 4);
            const uint64_t nb = (L.n + 3ull) / 4;
            add(L.code_off, f.size(), nb);
            f.resize(f.size() + nb);
        }
    }
    const uint64_t payload = f.size() - kHeaderSize;
    if (payload > 0xFFFFFFFFull) return TGB_OK;  // u32 payload length: no wire frames
    for (int i = 0; i < 4; ++i) f[14 + i] = static_cast<uint8_t>(payload >> (8 * i));
    TGB_CUDA(cudaMalloc(&P->d_frame, f.size()));
    TGB_CUDA(cudaMemcpy(P->d_frame, f.data(), f.size(), cudaMemcpyHostToDevice));
    TGB_CUDA(cudaMalloc(&P->d_wsegs, std::max<size_t>(1, segs.size()) * sizeof(WireSeg)));
    if (!segs.empty())
        TGB_CUDA(cudaMemcpy(P->d_wsegs, segs.data(), segs.size() * sizeof(WireSeg),
                            cudaMemcpyHostToDevice));
    P->n_wsegs = static_cast<uint32_t>(segs.size());
    P->push_frame_bytes = f.size();
    return TGB_OK;
}

tgb_status tgb_plan_push_frame_size(const tgb_plan* P, uint64_t* bytes) {
    if (!P || !bytes || P->names.size() != P->desc.size()) return TGB_ERR_INVALID_ARGUMENT;
    if (!P->d_frame) return TGB_ERR_UNSUPPORTED;  // > 65535 blocks or > 4 GB payload
    *bytes = P->push_frame_bytes;
    return TGB_OK;
}

tgb_status tgb_plan_serialize_push(tgb_plan* P, uint64_t t, uint8_t* h_frame, void* stream) {
    if (!P || !h_frame || P->names.size() != P->desc.size()) return TGB_ERR_INVALID_ARGUMENT;
    if (!P->d_frame) return TGB_ERR_UNSUPPORTED;
    auto st = static_cast<cudaStream_t>(stream);
    TGB_CUDA(launch_wire_gather(own_push(P), P->d_wsegs, P->n_wsegs, P->d_frame, st));
    TGB_CUDA(cudaMemcpyAsync(h_frame, P->d_frame, P->push_frame_bytes, cudaMemcpyDeviceToHost, st));
    TGB_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < 8; ++i) h_frame[4 + i] = static_cast<uint8_t>(t >> (8 * i));
    return TGB_OK;
}

namespace {
struct Rd {  // detail::Reader (codec.hpp:334-381) over the host frame
    const uint8_t* p;
    uint64_t n, pos;
    bool ok = true;
    uint64_t le(int bytes) {
        if (pos + bytes > n) {
            ok = false;
            return 0;
        }
        uint64_t v = 0;
        for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[pos + i];
        pos += bytes;
        return v;
    }
};
uint64_t radix_digits_per_word(uint64_t base) {  // wire.hpp:104-112
    uint64_t m = 0, acc = 1;
    while (acc <= UINT64_MAX / base) {
        acc *= base;
        ++m;
    }
    return m;
}
}  // namespace

// unframe + deserialize_pull + decode_pull (wire.hpp:57-75, 147-228) into the
// plan's bound outputs: headers parsed and validated on the host with the
// reference's ProtocolError texts, sums unpacked and decoded on the device.
tgb_status tgb_plan_decode_pull(tgb_plan* P, const uint8_t* h_frame, uint64_t len,
                                uint64_t* iteration, void* stream) {
    if (!P || !h_frame || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    if (P->names.size() != P->desc.size()) return TGB_ERR_INVALID_ARGUMENT;  // set_names first
    Rd r{h_frame, len, 0};
    if (len < kHeaderSize) return protocol_error("deserialize: truncated at byte 0");
    if (r.le(2) != kWireMagic) return protocol_error("bad magic");
    if (r.le(1) != kWireVersion) return protocol_error("bad version");
    const uint64_t type = r.le(1);
    if (type < 1 || type > 4) return protocol_error("bad message type " + std::to_string(type));
    if (type != 2) return protocol_error("worker: expected Pull");  // cluster.hpp:291-292
    const uint64_t it = r.le(8);
    r.le(2);  // worker
    const uint64_t plen = r.le(4);
    if (len - kHeaderSize != plen)
        return protocol_error("payload length mismatch: header says " + std::to_string(plen) +
                              ", got " + std::to_string(len - kHeaderSize));
    const uint64_t count = r.le(2);
    if (count != P->h_layers.size())
        return protocol_error("worker: averaged gradient tensor count mismatch");
    std::vector<PullSeg> segs;
    uint32_t threads = 0;
    for (uint64_t b = 0; b < count; ++b) {
        const LayerDev& L = P->h_layers[b];
        const uint64_t tag = r.le(1);
        const uint64_t nlen = r.le(2);
        if (!r.ok || r.pos + nlen > len)
            return protocol_error("deserialize: truncated at byte " + std::to_string(r.pos));
        const std::string name(reinterpret_cast<const char*>(h_frame + r.pos), nlen);
        r.pos += nlen;
        const uint64_t n = r.le(4);
        if (!r.ok) return protocol_error("deserialize: truncated at byte " + std::to_string(r.pos));
        if (name != P->names[L.tensor] || n != L.n)
            return protocol_error("worker: averaged gradient mismatch at " + P->names[L.tensor]);
        PullSeg sg{};
        sg.out = P->bound_out[L.tensor] + P->block_off[b];
        sg.n = static_cast<uint32_t>(n);
        sg.first_thread = threads;
        if (tag == 3) {  // kPullSharedSum
            const uint64_t workers = r.le(2);
            if (workers == 0) return protocol_error("pull: zero worker count");
            const uint32_t sbits = static_cast<uint32_t>(r.le(4));
            float s;
            std::memcpy(&s, &sbits, 4);
            const uint64_t base = 2 * workers + 1;
            const uint64_t m = radix_digits_per_word(base);
            const uint64_t words = r.le(4);
            if (!r.ok) return protocol_error("deserialize: truncated at byte " + std::to_string(r.pos));
            if (words != (n + m - 1) / m) return protocol_error("pull: bad word count");
            if (r.pos + 8 * words > len)
                return protocol_error("deserialize: truncated at byte " + std::to_string(r.pos));
            sg.kind = 3;
            sg.src_off = r.pos;
            sg.words = static_cast<uint32_t>(words);
            sg.base = static_cast<uint32_t>(base);
            sg.m = static_cast<uint32_t>(m);
            sg.s = s;
            sg.inv_n = 1.0f / static_cast<float>(workers);  // wire.hpp:216
            r.pos += 8 * words;
            threads += sg.words;
        } else if (tag == 4) {  // kPullFloatAvg
            if (r.pos + 4 * n > len)
                return protocol_error("deserialize: truncated at byte " + std::to_string(r.pos));
            sg.kind = 4;
            sg.src_off = r.pos;
            r.pos += 4 * n;
            threads += sg.n;
        } else {
            return protocol_error("pull: unknown block tag " + std::to_string(tag));
        }
        if (n) segs.push_back(sg);
    }
    if (r.pos != len) return protocol_error("pull: trailing bytes");
    auto st = static_cast<cudaStream_t>(stream);
    const uint64_t plen_bytes = len;  // the whole frame (offsets are frame-relative)
    if (P->pull_cap < plen_bytes + segs.size() * sizeof(PullSeg) + 256) {
        cudaFree(P->d_pull);
        P->pull_cap = plen_bytes + segs.size() * sizeof(PullSeg) + 256;
        TGB_CUDA(cudaMalloc(&P->d_pull, P->pull_cap));
    }
    uint8_t* d_payload = P->d_pull;
    const uint64_t seg_off = round_up(plen_bytes, 16);
    PullSeg* d_segs = reinterpret_cast<PullSeg*>(P->d_pull + seg_off);
    int* d_bad = reinterpret_cast<int*>(P->d_pull + seg_off + segs.size() * sizeof(PullSeg));
    TGB_CUDA(cudaMemcpyAsync(d_payload, h_frame, len, cudaMemcpyHostToDevice, st));
    if (!segs.empty())
        TGB_CUDA(cudaMemcpyAsync(d_segs, segs.data(), segs.size() * sizeof(PullSeg),
                                 cudaMemcpyHostToDevice, st));
    TGB_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    TGB_CUDA(launch_pull_decode(d_payload, d_segs, static_cast<uint32_t>(segs.size()), threads,
                                d_bad, st));
    int bad = 0;
    TGB_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    TGB_CUDA(cudaStreamSynchronize(st));
    if (bad) return protocol_error("pull: nonzero radix remainder");
    if (iteration) *iteration = it;
    return TGB_OK;
}

// ---------------------------------------------------- traffic accounting
namespace {
struct TrafficBlock {
    uint64_t n;
    uint64_t name_len;
    bool pass;
};

// TrafficStats of one worker and step (cluster.hpp:145-160) from the block list
void traffic_of(const std::vector<TrafficBlock>& blocks, bool sharing, int32_t N, tgb_traffic* o) {
    uint64_t up = 2, fup = 2, down = 2, fdown = 2;  // u16 block counts
    const uint64_t m = radix_digits_per_word(2ull * static_cast<uint64_t>(N) + 1);
    for (const TrafficBlock& b : blocks) {
        const uint64_t head = 1 + 2 + b.name_len + 4;  // tag, name, n
        // push (codec.hpp:455-467) vs raw fp32 (float_wire_size, :469-481)
        up += head + (b.pass ? 4 * b.n : 4 + (b.n + 3) / 4);
        fup += head + 4 * b.n;
        // pull (wire.hpp:113-145): SharedSumBlock = n, workers, s, word count, words
        if (!b.pass && sharing)
            down += head + 2 + 4 + 4 + 8 * ((b.n + m - 1) / m);
        else
            down += head + 4 * b.n;
        fdown += head + 4 * b.n;  // float_pull_size (wire.hpp:231-243)
    }
    o->bytes_up = kHeaderSize + up;  // framed (wire.hpp:38)
    o->float_bytes_up = kHeaderSize + fup;
    o->bytes_down = kHeaderSize + down;
    o->float_bytes_down = kHeaderSize + fdown;
}
}  // namespace

tgb_status tgb_traffic_for_layers(const tgb_layer_desc* layers, const char* const* names,
                                  int32_t n_layers, const tgb_codec_params* params,
                                  int32_t n_workers, tgb_traffic* out) {
    if (!out || !params || n_layers < 0 || (n_layers > 0 && (!layers || !names)) ||
        n_workers < 1 || n_workers > 0xFFFF)
        return TGB_ERR_INVALID_ARGUMENT;
    if (params->bucketing == TGB_BUCKET_FIXED && params->bucket_size < 1)
        return TGB_ERR_INVALID_ARGUMENT;
    std::memset(out, 0, sizeof(*out));
    std::vector<TrafficBlock> blocks;
    for (int32_t l = 0; l < n_layers; ++l) {  // the block list of encode_step (codec.hpp:218-236)
        if (!names[l]) return TGB_ERR_INVALID_ARGUMENT;
        const uint64_t nl = std::strlen(names[l]), n = layers[l].n;
        const bool pass = (layers[l].flags & TGB_LAYER_PASSTHROUGH) != 0;
        if (pass || params->bucketing != TGB_BUCKET_FIXED || n == 0) {
            blocks.push_back({n, nl, pass});
            continue;
        }
        for (uint64_t off = 0; off < n; off += params->bucket_size)
            blocks.push_back({std::min<uint64_t>(params->bucket_size, n - off), nl, false});
    }
    traffic_of(blocks, params->scaler_sharing != 0, n_workers, out);
    return TGB_OK;
}

tgb_status tgb_plan_traffic(const tgb_plan* P, tgb_traffic* out) {
    if (!P || !out || P->names.size() != P->desc.size()) return TGB_ERR_INVALID_ARGUMENT;
    std::memset(out, 0, sizeof(*out));
    std::vector<TrafficBlock> blocks;
    for (const LayerDev& L : P->h_layers)
        blocks.push_back({L.n, P->names[L.tensor].size(), (L.flags & kLayerPassthrough) != 0});
    traffic_of(blocks, P->p.scaler_sharing != 0, P->n_workers, out);
    const uint64_t N = static_cast<uint64_t>(P->n_workers);
    if (N == 1) return TGB_OK;
    const uint64_t slots = 4ull * P->n_slots;
    if (!P->attached) {  // ring allgather of whole push areas
        out->device_bytes_out = out->device_bytes_in = (N - 1) * P->push_bytes;
        return TGB_OK;
    }
    uint64_t regions = 0;  // code bytes + raw passthrough bytes of the whole push area
    for (const LayerDev& L : P->h_layers)
        regions += (L.flags & kLayerPassthrough) ? 4ull * L.n : (L.n + 3ull) / 4;
    if (!P->shard) {  // every rank's scalers + codes to every peer
        out->device_bytes_out = out->device_bytes_in = (N - 1) * (slots + regions);
        return TGB_OK;
    }
    // sharded: codes of the chunks other ranks own out, the owned chunks' codes of N-1
    // peers in; the owned chunks' packed sums (raw means) out to N-1 peers, the others in
    const uint32_t r = static_cast<uint32_t>(P->rank);
    uint64_t own_codes = 0, own_sums = 0, all_sums = 0;
    for (uint32_t c = 0; c < P->h_chunks.size(); ++c) {
        const ChunkDev& ch = P->h_chunks[c];
        const bool pass = (P->h_layers[ch.layer].flags & kLayerPassthrough) != 0;
        const uint64_t codes = pass ? 4ull * ch.count : (ch.count + 3ull) / 4;
        const uint64_t sums = pass ? 4ull * ch.count
                                   : (ch.count + P->radix_m - 1) / P->radix_m * 4ull;
        all_sums += sums;
        bool owned = false;
        for (int q = 0; q < P->n_pieces; ++q) owned |= c >= P->pcs[q][r] && c < P->pcs[q][r + 1];
        if (owned) {
            own_codes += codes;
            own_sums += sums;
        }
    }
    out->device_bytes_out = (N - 1) * slots + (regions - own_codes) + (N - 1) * own_sums;
    out->device_bytes_in = (N - 1) * slots + (N - 1) * own_codes + (all_sums - own_sums);
    return TGB_OK;
}

// ------------------------------------------------------------------- comm
tgb_status tgb_comm_unique_id(uint8_t out[TGB_UNIQUE_ID_BYTES]) {
    static_assert(sizeof(ncclUniqueId) == TGB_UNIQUE_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    TGB_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return TGB_OK;
}

tgb_status tgb_comm_init(const uint8_t id[TGB_UNIQUE_ID_BYTES], int32_t nranks, int32_t rank,
                         tgb_comm** out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return TGB_ERR_INVALID_ARGUMENT;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto* C = new (std::nothrow) tgb_comm;
    if (!C) return TGB_ERR_INVALID_ARGUMENT;
    const ncclResult_t r = ncclCommInitRank(&C->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete C;
        return TGB_ERR_NCCL;
    }
    C->nranks = nranks;
    C->rank = rank;
    *out = C;
    return TGB_OK;
}

void tgb_comm_destroy(tgb_comm* C) {
    if (!C) return;
    if (C->comm) ncclCommDestroy(C->comm);
    delete C;
}

// -------------------------------------------------------------- per layer
tgb_status tgb_layer_scaler(const float* d_g, uint64_t n, float* d_s, void* stream) {
    if (n > 0xFFFFFFFFull) return TGB_ERR_INVALID_ARGUMENT;  // TernaryBlock::n is u32
    if ((n > 0 && !d_g) || !d_s) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        TGB_CUDA(cudaMemsetAsync(d_s, 0, sizeof(float), st));
        return TGB_OK;
    }
    DeviceScratch* S;
    tgb_status s = scratch(&S);
    if (s != TGB_OK) return s;
    const uint32_t nc = static_cast<uint32_t>((n + kChunk - 1) / kChunk);
    Partial* parts = nullptr;
    TGB_CUDA(cudaMallocAsync(&parts, nc * sizeof(Partial), st));
    LayerDev L{};
    L.g = d_g;
    L.n = static_cast<uint32_t>(n);
    L.slot = 0;
    L.flags = layer_vec_flags(d_g, nullptr) & kLayerVecIn;  // clipping off => scaler = max|g|
    K1Launch k{parts, S->counters, S->counters + 1, S->tmp + 1, d_s, S->err, 2.5f, 0, 1, 1};
    const cudaError_t e = launch_k1_single(L, k, st);
    cudaFreeAsync(parts, st);
    TGB_CUDA(e);
    return TGB_OK;
}

tgb_status tgb_layer_clip(const float* d_g, uint64_t n, float c, float* d_out, float* d_bound,
                          void* stream) {
    if ((n > 0 && (!d_g || !d_out)) || !d_bound || n > 0xFFFFFFFFull) return TGB_ERR_INVALID_ARGUMENT;
    if (!(c > 0.0f)) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    if (n < 2) {  // codec.hpp:118: small tensors pass through unchanged
        const float inf = INFINITY;
        TGB_CUDA(cudaMemcpyAsync(d_bound, &inf, sizeof(float), cudaMemcpyHostToDevice, st));
        if (n == 1) TGB_CUDA(cudaMemcpyAsync(d_out, d_g, sizeof(float), cudaMemcpyDeviceToDevice, st));
        return TGB_OK;
    }
    DeviceScratch* S;
    tgb_status s = scratch(&S);
    if (s != TGB_OK) return s;
    const uint32_t nc = static_cast<uint32_t>((n + kChunk - 1) / kChunk);
    Partial* parts = nullptr;
    TGB_CUDA(cudaMallocAsync(&parts, nc * sizeof(Partial), st));
    LayerDev L{};
    L.g = d_g;
    L.n = static_cast<uint32_t>(n);
    L.slot = 0;
    L.flags = kLayerClip | (layer_vec_flags(d_g, nullptr) & kLayerVecIn);
    K1Launch k{parts, S->counters, S->counters + 1, d_bound, S->tmp, S->err, c, 0, 1, 1};
    cudaError_t e = launch_k1_single(L, k, st);
    cudaFreeAsync(parts, st);
    TGB_CUDA(e);
    TGB_CUDA(launch_clip_apply(d_g, n, d_bound, d_out, st));
    return TGB_OK;
}

tgb_status tgb_layer_ternarize(const float* d_g, uint64_t n, float s, uint64_t seed, uint64_t t,
                               uint64_t name_hash, uint64_t worker, uint64_t rng_base,
                               uint8_t* d_codes, void* stream) {
    if ((n > 0 && (!d_g || !d_codes)) || n > 0xFFFFFFFFull) return TGB_ERR_INVALID_ARGUMENT;
    if (n == 0) return TGB_OK;
    auto st = static_cast<cudaStream_t>(stream);
    DeviceScratch* S;
    tgb_status r = scratch(&S);
    if (r != TGB_OK) return r;
    uint32_t k0, k1;
    philox_key(seed, name_hash, worker, k0, k1);
    LayerDev L{};
    L.g = d_g;
    L.n = static_cast<uint32_t>(n);
    L.code_off = 0;
    L.key0 = k0;
    L.key1 = k1;
    L.slot = 0;
    L.flags = layer_vec_flags(d_g, nullptr) & kLayerVecIn;
    K2Launch k{d_codes, nullptr, nullptr, S->err, t, 0, s};
    k.rng_base = rng_base;  // unaligned bases take K2's lane-straddling path
    TGB_CUDA(launch_k2_single(L, k, st));
    return TGB_OK;
}

tgb_status tgb_layer_decode(const uint8_t* d_codes, uint64_t n, float s, float* d_out,
                            void* stream) {
    if (n > 0xFFFFFFFFull) return TGB_ERR_INVALID_ARGUMENT;  // TernaryBlock::n is u32
    if (n > 0 && (!d_codes || !d_out)) return TGB_ERR_INVALID_ARGUMENT;
    if (n == 0) return TGB_OK;
    auto st = static_cast<cudaStream_t>(stream);
    DeviceScratch* S;
    tgb_status r = scratch(&S);
    if (r != TGB_OK) return r;
    LayerDev L{};
    L.n = static_cast<uint32_t>(n);
    L.out = d_out;
    L.flags = layer_vec_flags(nullptr, d_out) & kLayerVecOut;
    const uint8_t* codes[1] = {d_codes};
    // decode(blk) == s * float(code) == average over N=1 with sharing (invN = 1)
    K3Launch k{nullptr, 0, 1, 1, 1.0f, S->err, s};
    TGB_CUDA(launch_k3_single(L, codes, nullptr, k, st));
    return TGB_OK;
}

tgb_status tgb_layer_average(int32_t n_workers, const uint8_t* const* d_codes, const float* d_s,
                             uint64_t n, int32_t sharing, float* d_out, void* stream) {
    if (n_workers < 1 || n_workers > kMaxWorkers || !d_codes || !d_s || n > 0xFFFFFFFFull)
        return TGB_ERR_INVALID_ARGUMENT;
    if (n == 0) return TGB_OK;
    if (!d_out) return TGB_ERR_INVALID_ARGUMENT;
    for (int w = 0; w < n_workers; ++w)
        if (!d_codes[w]) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    DeviceScratch* S;
    tgb_status r = scratch(&S);
    if (r != TGB_OK) return r;
    LayerDev L{};
    L.n = static_cast<uint32_t>(n);
    L.out = d_out;
    L.flags = layer_vec_flags(nullptr, d_out) & kLayerVecOut;
    K3Launch k{nullptr, 0, n_workers, sharing ? 1 : 0, 1.0f / static_cast<float>(n_workers),
               S->err};
    TGB_CUDA(launch_k3_single(L, d_codes, d_s, k, st));
    return TGB_OK;
}

tgb_status tgb_layer_average_raw(int32_t n_workers, const float* const* d_vals, uint64_t n,
                                 float* d_out, void* stream) {
    if (n_workers < 1 || n_workers > kMaxWorkers || !d_vals) return TGB_ERR_INVALID_ARGUMENT;
    if (n == 0) return TGB_OK;
    if (!d_out) return TGB_ERR_INVALID_ARGUMENT;
    for (int w = 0; w < n_workers; ++w)
        if (!d_vals[w]) return TGB_ERR_INVALID_ARGUMENT;
    TGB_CUDA(launch_average_raw(n_workers, d_vals, n, d_out, static_cast<cudaStream_t>(stream)));
    return TGB_OK;
}

tgb_status tgb_layer_histogram(const float* d_v, uint64_t n, uint32_t bins, uint64_t* d_counts,
                               double* d_edges, void* stream) {
    if (bins < 1 || !d_counts || !d_edges || (n > 0 && !d_v)) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    TGB_CUDA(cudaMemsetAsync(d_counts, 0, bins * sizeof(uint64_t), st));
    if (n == 0) {  // codec.hpp:495-498: bins of {0.0, 0}
        TGB_CUDA(cudaMemsetAsync(d_edges, 0, bins * sizeof(double), st));
        return TGB_OK;
    }
    // the reference's min/max chain starts at v[0]; a NaN there poisons lo/hi
    float first = 0.0f;
    TGB_CUDA(cudaMemcpyAsync(&first, d_v, sizeof(float), cudaMemcpyDeviceToHost, st));
    TGB_CUDA(cudaStreamSynchronize(st));
    uint32_t* mm = nullptr;
    TGB_CUDA(cudaMallocAsync(&mm, 2 * sizeof(uint32_t), st));
    const uint32_t init[2] = {0xFFFFFFFFu, 0u};
    cudaError_t e = cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = launch_histogram(d_v, n, bins, mm, 0, nullptr, nullptr, st, 0);
    if (e == cudaSuccess)
        e = launch_histogram(d_v, n, bins, mm, std::isnan(first) ? 1 : 0,
                             reinterpret_cast<unsigned long long*>(d_counts), d_edges, st, 1);
    cudaFreeAsync(mm, st);
    TGB_CUDA(e);
    TGB_CUDA(cudaStreamSynchronize(st));  // init[] lives on this stack frame
    return TGB_OK;
}

tgb_status tgb_rng_bits(uint64_t seed, uint64_t t, uint64_t name_hash, uint64_t worker, uint64_t k0,
                        uint64_t n, uint32_t* d_out, void* stream) {
    if (n > 0 && !d_out) return TGB_ERR_INVALID_ARGUMENT;
    uint32_t a, b;
    philox_key(seed, name_hash, worker, a, b);
    TGB_CUDA(launch_rng_bits(a, b, t, k0, n, d_out, static_cast<cudaStream_t>(stream)));
    return TGB_OK;
}

tgb_status tgb_layer_check(void* stream, tgb_error* out) {
    if (!out) return TGB_ERR_INVALID_ARGUMENT;
    DeviceScratch* S;
    tgb_status r = scratch(&S);
    if (r != TGB_OK) return r;
    TGB_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    ErrWord e;
    TGB_CUDA(cudaMemcpy(&e, S->err, sizeof(e), cudaMemcpyDeviceToHost));
    out->flags = e.flags;
    out->layer = e.flags ? e.layer() : -1;
    out->index = e.flags ? e.index() : 0;
    if (e.flags) TGB_CUDA(cudaMemset(S->err, 0, sizeof(ErrWord)));
    return e.flags ? TGB_ERR_CODEC : TGB_OK;
}

}  // extern "C"
