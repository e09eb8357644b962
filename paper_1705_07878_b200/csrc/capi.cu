// C-ABI implementation (include/tgb/terngrad_b200.h): plans, NCCL sync,
// per-layer entry points. Host code only; kernels live in kernels.cu.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "tgb_internal.h"

using namespace tgb;

namespace {

thread_local std::string g_last_error;  // tgb_last_error_message (PROTOCOL detail)

inline tgb_status protocol_error(const std::string& msg) {
    g_last_error = msg;
    return TGB_ERR_PROTOCOL;
}

constexpr uint64_t kAlignCodes = 16;   // per-layer code region alignment (bytes)
constexpr uint64_t kAlignPush = 256;   // push buffer / code region base alignment

inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

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

// rng.hpp:50-54
inline void philox_key(uint64_t seed, uint64_t name_hash, uint64_t worker, uint32_t& k0,
                       uint32_t& k1) {
    k0 = static_cast<uint32_t>(seed ^ name_hash);
    k1 = static_cast<uint32_t>((seed >> 32) ^ (name_hash >> 32) ^
                               (worker * 0x9E3779B97F4A7C15ull));
}

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

inline uint32_t layer_vec_flags(const void* g, const void* out) {
    uint32_t f = 0;
    if ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) f |= kLayerVecIn;
    if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) f |= kLayerVecOut;
    return f;
}

}  // namespace

constexpr int kMaxPieces = 8;
constexpr int kFlagSlots = 2 + kMaxPieces;  // barrier slots: groups 0/1, then pieces

struct tgb_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
};

struct tgb_plan {
    int device = 0;
    tgb_codec_params p{};
    uint16_t worker = 0;
    int32_t n_workers = 1;
    std::vector<tgb_layer_desc> desc;   // tensors (layers) in canonical order
    std::vector<TensorDev> h_tensors;
    std::vector<LayerDev> h_layers;     // BLOCKS (buckets / passthrough tensors)
    std::vector<uint64_t> block_off;    // block's first element inside its tensor
    std::vector<ChunkDev> h_chunks;     // K1/K2 work items (chunk12 elements, never straddle blocks)
    std::vector<ChunkDev> h_chunks3;    // K3 work items (kChunk3 elements)
    LayerDev* d_layers = nullptr;
    TensorDev* d_tensors = nullptr;
    ChunkFat* d_fat = nullptr;   // K1/K2: chunk + block copy (rebuilt on bind)
    ChunkFat* d_fat3 = nullptr;  // K3
    Partial* d_partials = nullptr;
    uint32_t* d_counters = nullptr;  // n_layers layer_done + 1 global_done
    float* d_bounds = nullptr;       // per block
    uint8_t* d_push = nullptr;
    uint8_t* d_gathered = nullptr;  // N > 1: parity-0 gather buffer inside d_ipc
    // N > 1: one IPC-shareable allocation [gather parity 0][gather parity 1][flags]
    uint8_t* d_ipc = nullptr;
    uint64_t flags_off = 0;
    uint8_t* peer_ipc[kMaxPeers] = {};  // every rank's d_ipc mapped here (self = d_ipc)
    bool attached = false;
    // radix-3 wire codes (fused exchange, N >= 3, shared scalers, no passthrough
    // blocks; TGB_R3=0 disables): K2 stores 5 elements per byte into every rank's
    // gather buffer (1.6 instead of 2 bits per element on NVLink) and its 2-bit codes
    // into d_push (the reference-format push area), K3 decodes the radix bytes
    bool r3_capable = false, r3 = false;
    bool local_peers = false;  // tgb_plan_attach_local: peers are plans of this process
    int32_t rank = 0;
    uint64_t epoch = 0;  // attached: steps begun (barrier value); parity = epoch & 1
    // Chunk tables are ordered by group, and inside a group ternary chunks come
    // before passthrough chunks (K1 launches only the ternary prefix). An
    // ungrouped plan is the single group 0. Two-group schedule (tgb_step):
    // group 1 = the dominant tensor, group 0 = the rest; each group runs
    // K1 -> K2 -> [barrier] -> K3 on its own stream, so a memory-bound kernel of
    // one group overlaps a compute-bound kernel of the other.
    bool grouped = false;
    uint32_t cb[2] = {0, 0}, cc[2] = {0, 0}, ck1[2] = {0, 0}, cb3[2] = {0, 0}, cc3[2] = {0, 0};
    cudaStream_t gs[2] = {nullptr, nullptr};
    // attached two-group steps: the dominant layer's K2 runs as `pieces` launches;
    // piece p's barrier + K3 run on gs3 as soon as every rank finished its K2
    // piece, so the decode of one piece overlaps the ternarize of the next
    int32_t pieces = 1;
    uint32_t pc_b[kMaxPieces] = {}, pc_c[kMaxPieces] = {}, pc_b3[kMaxPieces] = {},
             pc_c3[kMaxPieces] = {};
    cudaStream_t gs3 = nullptr;
    cudaEvent_t ev_piece[kMaxPieces] = {}, ev_pbar[kMaxPieces] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
    // two-group start order (TGB_STAGGER, A/B): 1 = group 0's K1 first, group 1
    // (the dominant layer) starts when it is done, so K1 of the dominant layer
    // (HBM-bound) overlaps K2 of the rest (Philox / NVLink-bound); 2 = the other
    // way round; 0 = both at once (default). Measured (VGG-16, profiles/
    // r01_schedule_ab.json): 0 is best at N = 1/2/4 (N=4 0.409 ms vs 0.423 / 0.431):
    // the groups already overlap, and the step is bound by the total HBM traffic
    // plus K2's NVLink stores, which no reordering shrinks.
    int32_t stagger = 0;
    cudaEvent_t ev_stag = nullptr;
    // attached two-group steps: each group's barrier kernel runs on its own stream
    // at the greatest priority (TGB_BSTREAM), so a group's barrier (which releases
    // the peers waiting on this rank) is not queued behind the other group's CTAs
    int32_t bstream = 0;  // A/B: 0.411 vs 0.409 ms at N = 4 (no gain)
    cudaStream_t gsb[2] = {nullptr, nullptr};
    cudaEvent_t ev_b0[2] = {nullptr, nullptr}, ev_b1[2] = {nullptr, nullptr};
    ErrWord* d_err = nullptr;
    uint64_t push_bytes = 0, codes_offset = 0, code_bytes = 0, total = 0;
    int32_t n_slots = 0, n_active = 0;
    uint32_t chunk12 = kChunk12;
    bool bound = false;
    int32_t k2_variant = 0;  // TGB_K2V
    int32_t k2_direct = 0;   // TGB_K2DIRECT: K2 stores codes from registers during the loop
    // K2 code stores as TMA bulk copies (cp.async.bulk smem -> local / peer global),
    // default; TGB_K2BULK=0 = 16-B SM stores. N=4 0.384 vs 0.408 ms, N=1/2 neutral
    // (profiles/r01_k2bulk_ab.json): the CTA hands its 8 KB of codes per destination
    // to the TMA engine instead of issuing 512 x 16-B stores per destination
    int32_t k2_bulk = 1;
    int32_t k1_variant = 0;  // TGB_K1V
    int32_t pdl = 0;         // TGB_PDL (A/B)
    // K1's last 24 MB per launch loaded L2 evict_last for K2's reverse walk (TGB_K1KEEP=MB;
    // tools/l2keep_ab.py: N=1 step -4.6 us with or without an L2 flush between steps)
    uint32_t k1_keep = 24u * (1u << 20) / (4u * kChunk12);
    int32_t k3_variant = 2;  // TGB_K3V: 2 staged + SWAR sums + register LUT (default), 1 staged + tables, 0 byte loads
    // sharded exchange (attached, N >= TGB_SHARD_MIN, shared scalers): rank r owns
    // K2 chunks [cs[r], cs[r+1]) and reduces them to packed sums for every rank.
    // d_ipc = [gather parity 0][gather parity 1][sums parity 0][sums parity 1][flags]
    bool shard_capable = false, shard = false;
    // pipelined fused exchange (attached, shared scalers, not sharded): one
    // persistent K2+K3 kernel per step with per-item epoch flags
    // (d_ipc + pflags_off: [item][kMaxPeers] u32) instead of the step barrier
    bool pipe_capable = false, pipe = false;
    uint64_t pflags_off = 0;
    uint32_t* d_done = nullptr;             // pipelined: local per-item done flags
    unsigned long long* d_nnz = nullptr;    // telemetry: nonzero codes per group (last step)
    bool code_stats = false;                // counted only when enabled (one pass over smem)
    unsigned long long* d_pprof = nullptr;  // TGB_PIPE_PROF (A/B instrumentation)
    uint64_t pipe_steps = 0;
    int32_t nib = 1;  // 4-bit sums (N <= 7), else 8-bit
    uint64_t sums_bytes = 0, sums_off = 0;
    uint32_t cs[kMaxPeers + 1] = {};
    uint32_t chunk3 = kChunk3;
    cudaStream_t last = nullptr;
    // host-buffer steps (tgb_step_host): per-tensor bound pointers, copy streams
    std::vector<const float*> bound_g;
    std::vector<float*> bound_out;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d = nullptr, ev_comp = nullptr, ev_d2h = nullptr;
    bool host_io = false;
    // optimizer bound for tgb_step_apply
    bool opt_bound = false;
    tgb_optimizer opt{};
    uint64_t opt_steps = 0;
    std::vector<float*> opt_w, opt_s1, opt_s2;
    // reference wire format (tgb_plan_set_names / serialize_push / decode_pull)
    std::vector<std::string> names;
    uint64_t push_frame_bytes = 0;
    uint8_t* d_frame = nullptr;     // push frame image (static headers written once)
    WireSeg* d_wsegs = nullptr;     // dynamic parts: scalers, codes, raw values
    uint32_t n_wsegs = 0;
    uint8_t* d_pull = nullptr;      // pull payload staging
    uint64_t pull_cap = 0;
    OptDev* d_optd = nullptr;        // per-block optimizer table (fused decode -> optimizer)
    // live kernel timing (tgb_plan_enable_timing): two events per launch
    int32_t t_cap = 0, t_used = 0;
    std::vector<cudaEvent_t> t_ev;
    std::vector<tgb_kernel_time> t_rec;
    bool t_sized = false;
    uint64_t t_k12[2][2] = {}, t_k3[2][2] = {};  // [group][ternary, passthrough] elements
    const OptArgs* opt_active = nullptr;  // set during tgb_step_apply when fused
};

extern "C" {

const char* tgb_version(void) { return "terngrad_b200 1 (sm_100a)"; }

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

// ------------------------------------------------------------------ plans
// two-group stream priorities: the dominant layer's chain is the critical path
// (K1 -> K2 -> K3 of the big layer), so it runs at high priority and the rest
// fills the gaps (TGB_GPRIO=0 flips it, A/B only)
static int gprio0(int lo, int hi) {
    const char* m = std::getenv("TGB_GPRIO");
    return (m && std::atoi(m) == 0) ? hi : lo;
}
static int gprio1(int lo, int hi) {
    const char* m = std::getenv("TGB_GPRIO");
    return (m && std::atoi(m) == 0) ? lo : hi;
}

// Block model (EncodedGradient::blocks, codec.hpp:70-76, built by encode_step
// :218-236): a ternary tensor is one block (PerTensor / Global) or
// ceil(n/k) buckets (FixedSize, an empty tensor still one empty block); a
// passthrough tensor is one raw block. Push layout:
//   [scaler slot per ternary block, f32][pad 256][block regions, 16-B aligned:
//    ceil(n/4) code bytes or 4n raw bytes][pad 256]
constexpr uint64_t kMaxBlocks = 1ull << 24;  // plan tables stay < 1.5 GB

tgb_status tgb_plan_create(const tgb_layer_desc* layers, int32_t n_layers,
                           const tgb_codec_params* params, uint16_t worker, int32_t n_workers,
                           tgb_plan** out) {
    if (!out || !params || n_layers < 0 || (n_layers > 0 && !layers)) return TGB_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (!(params->clip_factor > 0.0f)) return TGB_ERR_INVALID_ARGUMENT;  // codec.hpp:91-92
    if (params->bucketing == TGB_BUCKET_FIXED && params->bucket_size < 1)
        return TGB_ERR_INVALID_ARGUMENT;  // codec.hpp:93-94
    if (params->bucketing != TGB_BUCKET_PER_TENSOR && params->bucketing != TGB_BUCKET_GLOBAL &&
        params->bucketing != TGB_BUCKET_FIXED)
        return TGB_ERR_INVALID_ARGUMENT;
    // worker keys the RNG (rng.hpp:54) and need not be < n_workers for encode-only plans
    if (n_workers < 1 || n_workers > kMaxWorkers) return TGB_ERR_INVALID_ARGUMENT;
    uint64_t n_blocks = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
        if (layers[l].n > 0xFFFFFFFFull) return TGB_ERR_INVALID_ARGUMENT;  // TernaryBlock::n is u32
        const bool pass = (layers[l].flags & TGB_LAYER_PASSTHROUGH) != 0;
        if (pass || params->bucketing != TGB_BUCKET_FIXED || layers[l].n == 0)
            n_blocks += 1;
        else
            n_blocks += (layers[l].n + params->bucket_size - 1) / params->bucket_size;
    }
    if (n_blocks > kMaxBlocks) return TGB_ERR_UNSUPPORTED;
    auto* P = new (std::nothrow) tgb_plan;
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    P->p = *params;
    if (const char* m = std::getenv("TGB_K2V")) P->k2_variant = std::atoi(m);
    if (const char* m = std::getenv("TGB_K2DIRECT")) P->k2_direct = std::atoi(m);
    if (const char* m = std::getenv("TGB_K2BULK")) P->k2_bulk = std::atoi(m);
    if (const char* m = std::getenv("TGB_K1V")) P->k1_variant = std::atoi(m);
    if (n_workers > 1) P->k1_keep = 0;  // N = 2: K3 -8 us slower (evict_last lines linger)
    if (const char* m = std::getenv("TGB_K1KEEP"))
        P->k1_keep = static_cast<uint32_t>(std::max(0, std::atoi(m))) * (1u << 20) / (4u * kChunk12);
    if (const char* m = std::getenv("TGB_K3V")) P->k3_variant = std::atoi(m);
    if (const char* m = std::getenv("TGB_PDL")) P->pdl = std::atoi(m);
    P->worker = worker;
    P->n_workers = n_workers;
    P->desc.assign(layers, layers + n_layers);
    if (cudaGetDevice(&P->device) != cudaSuccess) {
        delete P;
        return TGB_ERR_CUDA;
    }
    // elements per grid-per-chunk work item: K1/K2 amortise a heavier per-CTA
    // setup over 32K elements, K3 (store-bound) prefers 16K (tools/ab_bench.py).
    // Small gradient sets would leave most of the 148 SMs idle with 32K items, so
    // K1/K2 items shrink to give about one full wave (148 SMs x 3 CTAs): the
    // smallest power of two >= total/444, within [4K, 32K] (GoogLeNet 6.6M
    // elements: 16K, step 32.9 -> 27.0 us; a 1M layer: 4K, 21.7 -> 14.6 us).
    uint64_t total_elems = 0;
    for (int32_t l = 0; l < n_layers; ++l) total_elems += layers[l].n;
    uint64_t chunk = 4096, chunk3 = kChunk3;
    while (chunk < kChunk12 && chunk * 444 < total_elems) chunk <<= 1;
    {
        bool any_pass = false;
        for (int32_t l = 0; l < n_layers; ++l) any_pass |= (layers[l].flags & TGB_LAYER_PASSTHROUGH) != 0;
        // (the same shard / pipeline decisions as below: those exchanges keep 2-bit codes)
        int smin = 5;
        if (const char* m = std::getenv("TGB_SHARD_MIN")) smin = std::max(2, std::atoi(m));
        bool shard = n_workers >= smin && params->scaler_sharing;
        if (const char* m = std::getenv("TGB_SHARD")) shard = shard && std::atoi(m) != 0;
        const char* pm = std::getenv("TGB_PIPE");
        const bool pipe = pm && std::atoi(pm) != 0 && !shard;
        // opt-in (TGB_R3=1): measured slower on 4 B200s (VGG-16 N=4 0.453 vs 0.409 ms,
        // N=3 0.445 vs 0.343; profiles/r01_r3_ab.json). K2 did not get faster with 20 %
        // fewer NVLink bytes (212 vs 215 us: K2 at N = 4 is not link-bandwidth bound),
        // the radix decode costs more ALU than the 2-bit SWAR one (K3 165 vs 124 us) and
        // 80-element work items leave K1 a scalar tail per chunk (138 vs 125 us).
        bool want = n_workers >= 3 && n_workers <= kMaxPeers && params->scaler_sharing &&
                    !any_pass && !shard && !pipe;
        const char* rm = std::getenv("TGB_R3");
        want = want && rm && std::atoi(rm) != 0;
        P->r3_capable = want;
        if (want) {  // work items at multiples of 80 elements (16-B aligned radix bytes)
            chunk = chunk / 80 * 80;
            chunk3 = kChunk3R3;
        }
    }
    if (const char* m = std::getenv("TGB_CHUNK")) {  // A/B only
        const uint64_t v = std::strtoull(m, nullptr, 10);
        if (v >= 1024 && v % 1024 == 0 && v <= kChunk12) chunk = v;
    }
    P->chunk12 = static_cast<uint32_t>(chunk);
    if (const char* m = std::getenv("TGB_CHUNK3")) {
        const uint64_t v = std::strtoull(m, nullptr, 10);
        if (v >= 1024 && v % 1024 == 0) chunk3 = v;
    }
    P->chunk3 = static_cast<uint32_t>(chunk3);

    // ---- tensors -> blocks, scaler slots
    P->h_tensors.resize(n_layers);
    P->h_layers.reserve(n_blocks);
    P->block_off.reserve(n_blocks);
    int32_t slot = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
        const uint64_t n = layers[l].n;
        const bool pass = (layers[l].flags & TGB_LAYER_PASSTHROUGH) != 0;
        TensorDev& T = P->h_tensors[l];
        std::memset(&T, 0, sizeof(T));
        T.n = n;
        T.first_block = static_cast<uint32_t>(P->h_layers.size());
        T.flags = (params->clipping_enabled && !pass) ? kLayerClip : 0u;  // codec.hpp:206-209
        uint32_t k0 = 0, k1 = 0;
        philox_key(params->seed, layers[l].name_hash, worker, k0, k1);
        const uint64_t k = (!pass && params->bucketing == TGB_BUCKET_FIXED) ? params->bucket_size
                                                                            : std::max<uint64_t>(n, 1);
        for (uint64_t off = 0; off < std::max<uint64_t>(n, 1); off += k) {
            LayerDev L;
            std::memset(&L, 0, sizeof(L));
            L.n = static_cast<uint32_t>(std::min<uint64_t>(k, n - std::min(n, off)));
            L.tensor = static_cast<uint32_t>(l);
            L.key0 = k0;
            L.key1 = k1;
            L.slot = pass ? -1 : slot++;
            L.flags = (pass ? kLayerPassthrough : 0u) | T.flags |
                      (static_cast<uint32_t>(off & 3u) << kLayerShiftBit);
            L.rng_q = static_cast<uint32_t>(off >> 2);
            P->h_layers.push_back(L);
            P->block_off.push_back(off);
            P->total += L.n;
            if (!pass) P->code_bytes += (L.n + 3) / 4;
        }
        T.n_blocks = static_cast<uint32_t>(P->h_layers.size()) - T.first_block;
        if (n > 0 && !pass) ++P->n_active;
    }
    P->n_slots = slot;
    P->codes_offset = round_up(static_cast<uint64_t>(slot) * sizeof(float), kAlignPush);
    uint64_t off = P->codes_offset;
    for (LayerDev& L : P->h_layers) {
        L.code_off = off;
        const uint64_t bytes = (L.flags & kLayerPassthrough) ? 4ull * L.n : (L.n + 3ull) / 4;
        off += round_up(bytes, kAlignCodes);
    }
    P->push_bytes = round_up(off, kAlignPush);

    // ---- work items (chunks never straddle blocks)
    const uint32_t nb = static_cast<uint32_t>(P->h_layers.size());
    for (uint32_t b = 0; b < nb; ++b) {
        const uint64_t n = P->h_layers[b].n;
        for (uint64_t e = 0; e < n; e += chunk)
            P->h_chunks.push_back({b, static_cast<uint32_t>(std::min<uint64_t>(chunk, n - e)), e});
        for (uint64_t e = 0; e < n; e += chunk3)
            P->h_chunks3.push_back({b, static_cast<uint32_t>(std::min<uint64_t>(chunk3, n - e)), e});
    }

    // ---- two-group schedule: the dominant tensor vs the rest (PerTensor + REF
    // only: Global and PRESHARED need every tensor's K1 before any K2)
    int32_t big = -1;
    for (int32_t l = 0; l < n_layers; ++l)
        if (!(layers[l].flags & TGB_LAYER_PASSTHROUGH) && (big < 0 || layers[l].n > layers[big].n))
            big = l;
    // sharded exchange from N >= 5 (TGB_SHARD_MIN): measured at N = 4 the fused
    // two-group schedule wins (0.425 vs 0.447 ms, VGG-16); the sharded design moves
    // 0.25(N-1)/N + w(N-1)/N bytes/element over NVLink instead of 0.25(N-1), which
    // is the dominant cost at N = 8
    int shard_min = 5;
    if (const char* m = std::getenv("TGB_SHARD_MIN")) shard_min = std::max(2, std::atoi(m));
    P->shard_capable = n_workers >= shard_min && n_workers <= kMaxPeers && params->scaler_sharing;
    if (const char* m = std::getenv("TGB_SHARD")) P->shard_capable = P->shard_capable && std::atoi(m) != 0;
    P->nib = n_workers <= 7 ? 1 : 0;
    // pipelined K2+K3 kernel: opt-in (TGB_PIPE=1). Bit-exact, but measured slower
    // than the two-group schedule (N=2 0.443 vs 0.326 ms, N=4 0.486 vs 0.425 ms):
    // items wait on peers' per-item flags
    P->pipe_capable = false;
    if (const char* m = std::getenv("TGB_PIPE"))
        P->pipe_capable = std::atoi(m) != 0 && n_workers >= 2 && n_workers <= kMaxPeers &&
                          params->scaler_sharing && !P->shard_capable;
    bool want = !P->shard_capable && !P->pipe_capable && big >= 0 && n_layers > 1 &&
                params->bucketing == TGB_BUCKET_PER_TENSOR &&
                params->share_mode == TGB_SHARE_REF && layers[big].n * 100 >= P->total * 35 &&
                layers[big].n * 100 <= P->total * 95;
    if (const char* m = std::getenv("TGB_GROUPS")) want = want && std::atoi(m) != 0;
    P->grouped = want;
    // K2 as K1's programmatic dependent on single-stream N = 1 plans (tools/env_ab.py,
    // profiles/r01_pdl_l2keep_ab.log): GoogLeNet 31.9 -> 29.1 us with a whole-chunk L2
    // prefetch before the wait, a 2^24 layer 49.6 -> 46.5 us without one, 2^26 / 2^28
    // layers 155 -> 149 / 546 -> 538 us prefetching the first 32 KB (a whole-chunk
    // prefetch re-reads evicted lines there: 159 / 575 us). With two concurrent groups the
    // waiting K2 CTAs hold SM slots the other group's K1 needs (VGG-16 +10 %): off.
    if (!std::getenv("TGB_PDL"))
        P->pdl = (P->grouped || n_workers > 1) ? 0
                 : P->total <= (8ull << 20) ? 2 : P->total >= (48ull << 20) ? 3 : 1;
    auto group_of = [&](const ChunkDev& c) {
        return (P->grouped && P->h_layers[c.layer].tensor == static_cast<uint32_t>(big)) ? 1u : 0u;
    };
    auto is_pass = [&](const ChunkDev& c) {
        return (P->h_layers[c.layer].flags & kLayerPassthrough) ? 1u : 0u;
    };
    std::stable_sort(P->h_chunks.begin(), P->h_chunks.end(), [&](const ChunkDev& x, const ChunkDev& y) {
        return 2 * group_of(x) + is_pass(x) < 2 * group_of(y) + is_pass(y);
    });
    std::stable_sort(P->h_chunks3.begin(), P->h_chunks3.end(), [&](const ChunkDev& x, const ChunkDev& y) {
        return group_of(x) < group_of(y);
    });
    for (const ChunkDev& c : P->h_chunks) {
        const uint32_t g = group_of(c);
        ++P->cc[g];
        if (!is_pass(c)) ++P->ck1[g];
    }
    P->cb[1] = P->cc[0];
    for (const ChunkDev& c : P->h_chunks3) ++P->cc3[group_of(c)];
    P->cb3[1] = P->cc3[0];
    // K1 units (group-relative chunk indices) per tensor
    std::vector<uint2> tunits(n_layers, make_uint2(0, 0));
    for (uint32_t c = 0; c < P->h_chunks.size(); ++c) {
        const ChunkDev& ch = P->h_chunks[c];
        if (is_pass(ch)) continue;
        const uint32_t rel = c - P->cb[group_of(ch)];
        uint2& tu = tunits[P->h_layers[ch.layer].tensor];
        if (tu.y++ == 0) tu.x = rel;
    }
    for (LayerDev& L : P->h_layers) {
        L.first_chunk = tunits[L.tensor].x;
        L.n_chunks = tunits[L.tensor].y;
    }
    if (P->shard_capable) {
        // sums regions: 2 (4-bit) or 4 (8-bit) bytes per code byte, raw fp32 means
        uint64_t so = 0;
        for (LayerDev& L : P->h_layers) {
            L.sum_off16 = static_cast<uint32_t>(so / 16);
            const uint64_t bytes = (L.flags & kLayerPassthrough) ? 4ull * L.n
                                   : (P->nib ? 2ull : 4ull) * ((L.n + 3ull) / 4);
            so += round_up(bytes, kAlignCodes);
        }
        P->sums_bytes = round_up(std::max<uint64_t>(so, 1), kAlignPush);
        // owners: contiguous K2-chunk ranges balanced by K3a bytes (raw fp32 = 16x codes)
        std::vector<uint64_t> cum(P->h_chunks.size() + 1, 0);
        for (size_t c = 0; c < P->h_chunks.size(); ++c)
            cum[c + 1] = cum[c] + P->h_chunks[c].count * (is_pass(P->h_chunks[c]) ? 16ull : 1ull);
        const uint64_t W = cum.back();
        for (int r = 0; r <= n_workers; ++r) {
            const uint64_t target = W * static_cast<uint64_t>(r) / static_cast<uint64_t>(n_workers);
            P->cs[r] = static_cast<uint32_t>(std::lower_bound(cum.begin(), cum.end(), target) -
                                             cum.begin());
        }
        P->cs[n_workers] = static_cast<uint32_t>(P->h_chunks.size());
        for (int r = n_workers + 1; r <= kMaxPeers; ++r) P->cs[r] = P->cs[n_workers];
    }
    // pieces of the dominant layer (attached N > 1 steps; A/B only, TGB_PIECES):
    // equal runs of its K2 chunks, and the K3 chunks whose first element falls in
    // each run. Measured slower on VGG-16 (N=4: 0.410 / 0.420 / 0.444 / 0.487 ms
    // for 1 / 2 / 4 / 8 pieces; N=2: 0.324 / 0.324 / 0.334 / 0.356): K3 pieces take
    // SM slots from the NVLink-store-bound K2 and every piece barrier waits for the
    // slowest rank.
    if (P->grouped && n_workers > 1) {
        int want_p = 1;
        if (const char* m = std::getenv("TGB_PIECES")) want_p = std::atoi(m);
        want_p = std::max(1, std::min(want_p, kMaxPieces));
        const uint32_t c2 = P->cc[1];
        if (want_p > 1 && c2 >= static_cast<uint32_t>(want_p)) {
            P->pieces = want_p;
            uint32_t k3 = P->cb3[1];
            const uint32_t k3_end = P->cb3[1] + P->cc3[1];
            for (int pc = 0; pc < want_p; ++pc) {
                P->pc_b[pc] = P->cb[1] + c2 * pc / want_p;
                P->pc_c[pc] = P->cb[1] + c2 * (pc + 1) / want_p - P->pc_b[pc];
                const bool last = pc == want_p - 1;
                const uint64_t end = last ? ~0ull
                                          : P->h_chunks[P->pc_b[pc] + P->pc_c[pc]].begin;
                P->pc_b3[pc] = k3;
                while (k3 < k3_end && P->h_chunks3[k3].begin < end) ++k3;
                P->pc_c3[pc] = k3 - P->pc_b3[pc];
            }
        }
    }
    if (P->grouped) {
        int lo = 0, hi = 0;
        bool ok = cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess &&
                  cudaStreamCreateWithPriority(&P->gs[0], cudaStreamNonBlocking, gprio0(lo, hi)) == cudaSuccess &&
                  cudaStreamCreateWithPriority(&P->gs[1], cudaStreamNonBlocking, gprio1(lo, hi)) == cudaSuccess &&
                  cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&P->ev_join[0], cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&P->ev_join[1], cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&P->ev_stag, cudaEventDisableTiming) == cudaSuccess;
        if (const char* m = std::getenv("TGB_STAGGER")) P->stagger = std::atoi(m);
        if (const char* m = std::getenv("TGB_BSTREAM")) P->bstream = std::atoi(m);
        for (int g = 0; ok && g < 2; ++g)
            ok = cudaStreamCreateWithPriority(&P->gsb[g], cudaStreamNonBlocking, hi) == cudaSuccess &&
                 cudaEventCreateWithFlags(&P->ev_b0[g], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&P->ev_b1[g], cudaEventDisableTiming) == cudaSuccess;
        if (ok && P->pieces > 1) {
            int p3 = gprio1(lo, hi);
            if (const char* m = std::getenv("TGB_P3PRIO")) p3 = std::atoi(m) ? hi : lo;
            ok = cudaStreamCreateWithPriority(&P->gs3, cudaStreamNonBlocking, p3) == cudaSuccess;
            for (int pc = 0; ok && pc < P->pieces; ++pc)
                ok = cudaEventCreateWithFlags(&P->ev_piece[pc], cudaEventDisableTiming) == cudaSuccess &&
                     cudaEventCreateWithFlags(&P->ev_pbar[pc], cudaEventDisableTiming) == cudaSuccess;
        }
        if (!ok) {
            tgb_plan_destroy(P);
            return TGB_ERR_CUDA;
        }
    }

    const size_t nl = std::max<size_t>(1, n_layers), nbl = std::max<size_t>(1, nb);
    const size_t nc = std::max<size_t>(1, P->h_chunks.size());
    bool ok = cudaMalloc(&P->d_layers, nbl * sizeof(LayerDev)) == cudaSuccess &&
              cudaMalloc(&P->d_tensors, nl * sizeof(TensorDev)) == cudaSuccess &&
              cudaMalloc(&P->d_fat, nc * sizeof(ChunkFat)) == cudaSuccess &&
              cudaMalloc(&P->d_fat3, std::max<size_t>(1, P->h_chunks3.size()) * sizeof(ChunkFat)) ==
                  cudaSuccess &&
              cudaMalloc(&P->d_partials, nc * sizeof(Partial)) == cudaSuccess &&
              cudaMalloc(&P->d_counters, (nl + 1) * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&P->d_bounds, nbl * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&P->d_push, P->push_bytes) == cudaSuccess &&
              cudaMalloc(&P->d_err, sizeof(ErrWord)) == cudaSuccess &&
              cudaMalloc(&P->d_nnz, 2 * sizeof(unsigned long long)) == cudaSuccess &&
              cudaMemset(P->d_nnz, 0, 2 * sizeof(unsigned long long)) == cudaSuccess;
    if (ok && n_workers > 1) {
        const uint64_t g = P->push_bytes * static_cast<uint64_t>(n_workers);
        P->sums_off = 2 * g;
        P->flags_off = P->sums_off + 2 * P->sums_bytes;
        P->pflags_off = P->flags_off + round_up(kFlagSlots * kMaxPeers * sizeof(uint64_t), kAlignPush);
        const uint64_t pflags = P->pipe_capable ? P->h_chunks.size() * kMaxPeers * sizeof(uint32_t) : 0;
        const uint64_t bytes = P->pflags_off + round_up(std::max<uint64_t>(pflags, 1), kAlignPush);
        ok = cudaMalloc(&P->d_ipc, bytes) == cudaSuccess &&
             cudaMemset(P->d_ipc, 0, bytes) == cudaSuccess;
        if (ok && P->pipe_capable) {
            const size_t nd = std::max<size_t>(1, P->h_chunks.size()) * sizeof(uint32_t);
            ok = cudaMalloc(&P->d_done, nd) == cudaSuccess && cudaMemset(P->d_done, 0, nd) == cudaSuccess;
        }
        P->d_gathered = P->d_ipc;
    }
    const std::vector<float> inf_bounds(nbl, INFINITY);  // empty / unclipped: no clip (codec.hpp:118)
    ok = ok && cudaMemset(P->d_counters, 0, (nl + 1) * sizeof(uint32_t)) == cudaSuccess &&
         cudaMemset(P->d_push, 0, P->push_bytes) == cudaSuccess &&
         cudaMemset(P->d_err, 0, sizeof(ErrWord)) == cudaSuccess &&
         cudaMemcpy(P->d_bounds, inf_bounds.data(), nbl * sizeof(float), cudaMemcpyHostToDevice) ==
             cudaSuccess;
    if (ok && nb > 0)
        ok = cudaMemcpy(P->d_layers, P->h_layers.data(), nb * sizeof(LayerDev),
                        cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && n_layers > 0)
        ok = cudaMemcpy(P->d_tensors, P->h_tensors.data(), n_layers * sizeof(TensorDev),
                        cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
        tgb_plan_destroy(P);
        return TGB_ERR_CUDA;
    }
    *out = P;
    return TGB_OK;
}

void tgb_plan_destroy(tgb_plan* P) {
    if (!P) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(P->device);
    if (P->d_pprof) {  // A/B instrumentation: mean cycles per step per phase (all CTAs summed)
        unsigned long long h[8] = {};
        if (cudaMemcpy(h, P->d_pprof, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess && P->pipe_steps)
            std::fprintf(stderr,
                         "[tgb pipe prof rank %d] cycles/step summed over CTAs: wait %.3g prepare %.3g "
                         "code %.3g finish %.3g publish %.3g store %.3g tailwait %.3g taildecode %.3g\n",
                         P->rank, h[0] / double(P->pipe_steps), h[1] / double(P->pipe_steps),
                         h[2] / double(P->pipe_steps), h[3] / double(P->pipe_steps),
                         h[4] / double(P->pipe_steps), h[5] / double(P->pipe_steps),
                         h[6] / double(P->pipe_steps), h[7] / double(P->pipe_steps));
        cudaFree(P->d_pprof);
    }
    cudaFree(P->d_layers);
    cudaFree(P->d_tensors);
    cudaFree(P->d_fat);
    cudaFree(P->d_fat3);
    cudaFree(P->d_partials);
    cudaFree(P->d_counters);
    cudaFree(P->d_bounds);
    cudaFree(P->d_push);
    if (P->attached && !P->local_peers)
        for (int p = 0; p < P->n_workers; ++p)
            if (p != P->rank && P->peer_ipc[p]) cudaIpcCloseMemHandle(P->peer_ipc[p]);
    cudaFree(P->d_ipc);
    cudaFree(P->d_done);
    cudaFree(P->d_nnz);
    cudaFree(P->d_optd);
    cudaFree(P->d_frame);
    cudaFree(P->d_wsegs);
    cudaFree(P->d_pull);
    cudaFree(P->d_err);
    for (int g = 0; g < 2; ++g) {
        if (P->gs[g]) cudaStreamDestroy(P->gs[g]);
        if (P->ev_join[g]) cudaEventDestroy(P->ev_join[g]);
    }
    if (P->ev_fork) cudaEventDestroy(P->ev_fork);
    if (P->ev_stag) cudaEventDestroy(P->ev_stag);
    for (int g = 0; g < 2; ++g) {
        if (P->gsb[g]) cudaStreamDestroy(P->gsb[g]);
        if (P->ev_b0[g]) cudaEventDestroy(P->ev_b0[g]);
        if (P->ev_b1[g]) cudaEventDestroy(P->ev_b1[g]);
    }
    if (P->gs3) cudaStreamDestroy(P->gs3);
    for (int pc = 0; pc < kMaxPieces; ++pc) {
        if (P->ev_piece[pc]) cudaEventDestroy(P->ev_piece[pc]);
        if (P->ev_pbar[pc]) cudaEventDestroy(P->ev_pbar[pc]);
    }
    for (cudaEvent_t e : P->t_ev) cudaEventDestroy(e);
    if (P->s_h2d) cudaStreamDestroy(P->s_h2d);
    if (P->s_d2h) cudaStreamDestroy(P->s_d2h);
    if (P->ev_h2d) cudaEventDestroy(P->ev_h2d);
    if (P->ev_comp) cudaEventDestroy(P->ev_comp);
    if (P->ev_d2h) cudaEventDestroy(P->ev_d2h);
    cudaSetDevice(prev);
    delete P;
}

tgb_status tgb_plan_get_info(const tgb_plan* P, tgb_plan_info* o) {
    if (!P || !o) return TGB_ERR_INVALID_ARGUMENT;
    std::memset(o, 0, sizeof(*o));
    o->total_elements = P->total;
    o->push_bytes = P->push_bytes;
    o->code_bytes = P->code_bytes;
    o->scaler_offset = 0;
    o->codes_offset = P->codes_offset;
    o->n_layers = static_cast<int32_t>(P->desc.size());
    o->n_slots = P->n_slots;
    o->n_chunks = static_cast<int32_t>(P->h_chunks.size());
    o->n_workers = P->n_workers;
    o->chunk_elems = P->chunk12;
    o->n_groups = P->grouped ? 2u : 1u;
    o->n_blocks = static_cast<int32_t>(P->h_layers.size());
    o->exchange = P->n_workers == 1 ? TGB_EXCHANGE_NONE
                  : !P->attached    ? TGB_EXCHANGE_NCCL
                  : P->shard        ? TGB_EXCHANGE_SHARDED
                  : P->pipe         ? TGB_EXCHANGE_PIPELINED
                  : P->r3           ? TGB_EXCHANGE_FUSED_R3
                                    : TGB_EXCHANGE_FUSED;
    return TGB_OK;
}

tgb_status tgb_plan_layer_layout(const tgb_plan* P, int32_t layer, uint64_t* code_offset,
                                 int32_t* slot) {
    if (!P || layer < 0 || layer >= static_cast<int32_t>(P->desc.size()))
        return TGB_ERR_INVALID_ARGUMENT;
    const LayerDev& L = P->h_layers[P->h_tensors[layer].first_block];
    if (code_offset) *code_offset = L.code_off;
    if (slot) *slot = L.slot;
    return TGB_OK;
}

tgb_status tgb_plan_block_info(const tgb_plan* P, int32_t block, tgb_block_info* o) {
    if (!P || !o || block < 0 || block >= static_cast<int32_t>(P->h_layers.size()))
        return TGB_ERR_INVALID_ARGUMENT;
    const LayerDev& L = P->h_layers[block];
    std::memset(o, 0, sizeof(*o));
    o->layer = static_cast<int32_t>(L.tensor);
    o->slot = L.slot;
    o->offset = P->block_off[block];
    o->n = L.n;
    o->region_offset = L.code_off;
    o->flags = (L.flags & kLayerPassthrough) ? TGB_LAYER_PASSTHROUGH : 0u;
    return TGB_OK;
}

tgb_status tgb_plan_bind(tgb_plan* P, const float* const* d_grads, float* const* d_out) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    const size_t nl = P->desc.size();
    if (nl > 0 && (!d_grads || !d_out)) return TGB_ERR_INVALID_ARGUMENT;
    for (size_t l = 0; l < nl; ++l)
        if (P->desc[l].n > 0 && (!d_grads[l] || !d_out[l])) return TGB_ERR_INVALID_ARGUMENT;
    for (size_t b = 0; b < P->h_layers.size(); ++b) {
        LayerDev& L = P->h_layers[b];
        const uint64_t off = P->block_off[b];
        L.g = d_grads[L.tensor] ? d_grads[L.tensor] + off : nullptr;
        L.out = d_out[L.tensor] ? d_out[L.tensor] + off : nullptr;
        L.flags = (L.flags & ~(kLayerVecIn | kLayerVecOut)) | layer_vec_flags(L.g, L.out);
    }
    P->bound_g.assign(d_grads, d_grads + nl);
    P->bound_out.assign(d_out, d_out + nl);
    if (!P->h_layers.empty())
        TGB_CUDA(cudaMemcpy(P->d_layers, P->h_layers.data(), P->h_layers.size() * sizeof(LayerDev),
                            cudaMemcpyHostToDevice));
    for (int which = 0; which < 2; ++which) {
        const std::vector<ChunkDev>& chs = which == 0 ? P->h_chunks : P->h_chunks3;
        if (chs.empty()) continue;
        std::vector<ChunkFat> fat(chs.size());
        for (size_t c = 0; c < fat.size(); ++c) {
            fat[c].ch = chs[c];
            fat[c].L = P->h_layers[chs[c].layer];
        }
        TGB_CUDA(cudaMemcpy(which == 0 ? P->d_fat : P->d_fat3, fat.data(),
                            fat.size() * sizeof(ChunkFat), cudaMemcpyHostToDevice));
    }
    P->bound = true;
    return TGB_OK;
}

tgb_status tgb_plan_buffers(tgb_plan* P, uint8_t** d_push, uint8_t** d_gathered, float** d_bounds) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    if (d_push) *d_push = P->d_push;
    if (d_gathered) *d_gathered = P->d_gathered;
    if (d_bounds) *d_bounds = P->d_bounds;
    return TGB_OK;
}

// attached plans: this rank's push area in rank p's gather buffer of the
// current parity
static inline uint8_t* push_area(const tgb_plan* P, int p) {
    const uint64_t g = P->push_bytes * static_cast<uint64_t>(P->n_workers);
    return P->peer_ipc[p] + (P->epoch & 1u) * g + static_cast<uint64_t>(P->rank) * P->push_bytes;
}
static inline uint8_t* own_push(const tgb_plan* P) {
    return (P->attached && !P->r3) ? push_area(P, P->rank) : P->d_push;
}
static inline uint8_t* cur_gathered(const tgb_plan* P) {
    if (P->attached)
        return P->d_ipc + (P->epoch & 1u) * P->push_bytes * static_cast<uint64_t>(P->n_workers);
    return P->n_workers > 1 ? P->d_gathered : P->d_push;
}

// ---- per-group launches (group g = chunk ranges cb/cc, cb3/cc3; an ungrouped
// plan is the single group 0 spanning every chunk)
static inline int n_groups(const tgb_plan* P) { return P->grouped ? 2 : 1; }

// ---- live kernel timing: events around each launch on its own stream
static void chunk_elems(const tgb_plan* P, const std::vector<ChunkDev>& chs, uint32_t b,
                        uint32_t c, uint64_t out[2]) {
    out[0] = out[1] = 0;
    for (uint32_t i = b; i < b + c && i < chs.size(); ++i)
        out[(P->h_layers[chs[i].layer].flags & kLayerPassthrough) ? 1 : 0] += chs[i].count;
}

static void timing_size(tgb_plan* P) {
    if (P->t_sized) return;
    for (int g = 0; g < n_groups(P); ++g) {
        chunk_elems(P, P->h_chunks, P->cb[g], P->cc[g], P->t_k12[g]);
        chunk_elems(P, P->h_chunks3, P->cb3[g], P->cc3[g], P->t_k3[g]);
    }
    P->t_sized = true;
}

static int t_begin(tgb_plan* P, cudaStream_t st) {
    if (P->t_used >= P->t_cap) return -1;
    const int slot = P->t_used++;
    if (cudaEventRecord(P->t_ev[2 * slot], st) != cudaSuccess) return -1;
    return slot;
}

static void t_end(tgb_plan* P, cudaStream_t st, int slot, int32_t kind, int32_t g,
                  uint64_t elems, uint64_t hbm, uint64_t nvl) {
    if (slot < 0) return;
    cudaEventRecord(P->t_ev[2 * slot + 1], st);
    P->t_rec[slot] = tgb_kernel_time{kind, g, 0.0f, 0.0f, elems, hbm, nvl};
}

static tgb_status launch_stats(tgb_plan* P, int g, cudaStream_t st) {
    const uint32_t b = P->cb[g];
    K1Launch k{P->d_partials + b, P->d_counters,
               P->d_counters + P->desc.size(), P->d_bounds,
               reinterpret_cast<float*>(own_push(P)), P->d_err, P->p.clip_factor,
               P->p.bucketing == TGB_BUCKET_GLOBAL, static_cast<int32_t>(P->h_layers.size()),
               P->n_active};
    if (P->attached) {  // scalers also land in every peer's gather buffer
        k.push.n = 0;
        for (int p = 0; p < P->n_workers; ++p)
            if (p != P->rank || P->r3) k.push.base[k.push.n++] = push_area(P, p);
        k.push.remote = 1;
    }
    k.variant = P->k1_variant;
    k.keep_chunks = P->k1_keep;
    k.tensors = P->d_tensors;
    k.nnz = P->code_stats ? P->d_nnz + g : nullptr;
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k1_table(P->d_layers, P->d_fat + b, P->ck1[g], k, st));
    if (ts >= 0) {
        timing_size(P);
        const uint64_t n = P->t_k12[g][0];
        t_end(P, st, ts, TGB_KERNEL_K1, g, n, 4 * n, 0);
    }
    return TGB_OK;
}

static tgb_status launch_tern_rng(tgb_plan* P, int g, uint32_t cb, uint32_t cc, uint64_t t,
                                  cudaStream_t st, bool fuse_decode) {
    uint8_t* own = own_push(P);
    K2Launch k{own, reinterpret_cast<const float*>(own), P->d_bounds, P->d_err, t, 1};
    k.fuse_decode = fuse_decode ? 1 : 0;
    k.direct = P->k2_direct;
    k.bulk = P->k2_bulk;
    k.nnz = P->code_stats ? P->d_nnz + g : nullptr;
    if (fuse_decode && P->opt_active) {
        k.optd = P->d_optd;
        k.opt = *P->opt_active;
    }
    k.variant = P->k2_variant;
    k.pdl = P->pdl;
    if (P->attached) {  // fused exchange: codes stored into every rank's gather buffer
        for (int p = 0; p < P->n_workers; ++p) k.dst.base[p] = push_area(P, p);
        k.dst.n = P->n_workers;
        k.dst.remote = 1;
        if (P->shard) {
            k.shard_n = P->n_workers;
            for (int r = 0; r <= kMaxPeers; ++r) k.shard_bounds[r] = P->cs[r];
        }
        k.r3 = P->r3 ? 1 : 0;
    }
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k2_table(P->d_layers, P->d_fat + cb, cc, k, st));
    if (ts >= 0) {
        uint64_t e[2];
        chunk_elems(P, P->h_chunks, cb, cc, e);
        const uint64_t nt = e[0], np = e[1], N = P->n_workers;
        const uint64_t msg = (nt + 3) / 4 + 4 * np;  // code bytes + raw passthrough bytes
        uint64_t own = msg, nvl = 0;
        if (P->attached && P->shard) {
            own = msg / N;
            nvl = msg - own;
        } else if (P->attached && P->r3) {  // 2-bit push + radix-3 own copy; radix-3 to peers
            own = msg + (nt + 4) / 5;
            nvl = (N - 1) * ((nt + 4) / 5);
        } else if (P->attached) {
            nvl = (N - 1) * msg;
        }
        const uint64_t out = fuse_decode ? 4 * (nt + np) : 0;
        t_end(P, st, ts, TGB_KERNEL_K2, g, nt + np, 4 * (nt + np) + own + out, nvl);
    }
    return TGB_OK;
}

static tgb_status launch_tern(tgb_plan* P, int g, uint64_t t, cudaStream_t st,
                              bool fuse_decode = false) {
    return launch_tern_rng(P, g, P->cb[g], P->cc[g], t, st, fuse_decode);
}

// barrier slot g: 0/1 = layer groups (sharded: its two barriers), 2 + p = piece p
static tgb_status launch_barrier(tgb_plan* P, int g, cudaStream_t st) {
    PeerFlags f{};
    for (int p = 0; p < P->n_workers; ++p)
        f.remote[p] = reinterpret_cast<uint64_t*>(P->peer_ipc[p] + P->flags_off) +
                      g * kMaxPeers + P->rank;
    f.local = reinterpret_cast<uint64_t*>(P->d_ipc + P->flags_off) + g * kMaxPeers;
    f.n = P->n_workers;
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_peer_barrier(f, P->epoch, P->d_err, st));
    t_end(P, st, ts, TGB_KERNEL_BARRIER, g, 0, 0, 0);
    return TGB_OK;
}

static tgb_status launch_decode_rng(tgb_plan* P, int g, uint32_t cb3, uint32_t cc3,
                                    const uint8_t* src, int32_t n_workers, cudaStream_t st) {
    K3Launch k{src, P->push_bytes, n_workers, P->p.scaler_sharing ? 1 : 0,
               1.0f / static_cast<float>(n_workers), P->d_err};
    k.variant = P->k3_variant;
    k.chunk3 = P->chunk3;
    k.r3 = (P->r3 && src == cur_gathered(P) && n_workers == P->n_workers) ? 1 : 0;
    if (P->opt_active) {
        k.optd = P->d_optd;
        k.opt = *P->opt_active;
    }
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k3_table(P->d_layers, P->d_fat3 + cb3, cc3, k, st));
    if (ts >= 0) {
        uint64_t e[2];
        chunk_elems(P, P->h_chunks3, cb3, cc3, e);
        const uint64_t nt = e[0], np = e[1], N = n_workers;
        const uint64_t codes = k.r3 ? (nt + 4) / 5 : (nt + 3) / 4;
        t_end(P, st, ts, TGB_KERNEL_K3, g, nt + np, N * (codes + 4 * np) + 4 * (nt + np), 0);
    }
    return TGB_OK;
}

static tgb_status launch_decode(tgb_plan* P, int g, const uint8_t* src, int32_t n_workers,
                                cudaStream_t st) {
    return launch_decode_rng(P, g, P->cb3[g], P->cc3[g], src, n_workers, st);
}

#define TGB_TRY_INNER(expr)                  \
    do {                                     \
        const tgb_status s_ = (expr);        \
        if (s_ != TGB_OK) return s_;         \
    } while (0)

static inline uint8_t* sums_area(const tgb_plan* P, int p) {
    return P->peer_ipc[p] + P->sums_off + (P->epoch & 1u) * P->sums_bytes;
}

static ShardLaunch shard_launch(const tgb_plan* P) {
    ShardLaunch k{};
    k.src = P->d_ipc + (P->epoch & 1u) * P->push_bytes * static_cast<uint64_t>(P->n_workers);
    k.stride = P->push_bytes;
    for (int p = 0; p < P->n_workers; ++p) k.sums[p] = sums_area(P, p);
    k.own_sums = sums_area(P, P->rank);
    k.n_workers = P->n_workers;
    k.nib = P->nib;
    k.inv_n = 1.0f / static_cast<float>(P->n_workers);
    k.err = P->d_err;
    k.bulk = P->k2_bulk;
    return k;
}

// sharded exchange after K2: [codes landed at their owner] barrier 0 -> K3a
// (owned chunks -> packed sums to every rank) -> barrier 1
static tgb_status launch_shard_reduce(tgb_plan* P, cudaStream_t st) {
    TGB_TRY_INNER(launch_barrier(P, 0, st));
    const uint32_t r = static_cast<uint32_t>(P->rank);
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k3_reduce(P->d_fat + P->cs[r], P->cs[r + 1] - P->cs[r], shard_launch(P), st));
    if (ts >= 0) {
        uint64_t e[2];
        chunk_elems(P, P->h_chunks, P->cs[r], P->cs[r + 1] - P->cs[r], e);
        const uint64_t N = P->n_workers;
        const uint64_t sums = P->nib ? (e[0] + 1) / 2 : e[0];  // packed biased sums
        const uint64_t out = sums + 4 * e[1];
        t_end(P, st, ts, TGB_KERNEL_K3A, 0, e[0] + e[1], N * ((e[0] + 3) / 4 + 4 * e[1]) + out,
              (N - 1) * out);
    }
    TGB_TRY_INNER(launch_barrier(P, 1, st));
    return TGB_OK;
}

// pipelined K2+K3 (one persistent kernel; codes to every rank, per-item flags)
static tgb_status launch_pipelined(tgb_plan* P, uint64_t t, cudaStream_t st) {
    uint8_t* own = own_push(P);
    K2Launch k2{own, reinterpret_cast<const float*>(own), P->d_bounds, P->d_err, t, 0};
    k2.nnz = P->code_stats ? P->d_nnz : nullptr;  // pipelined: single group (K1 group 0 reset it)
    for (int p = 0; p < P->n_workers; ++p) k2.dst.base[p] = push_area(P, p);
    k2.dst.n = P->n_workers;
    k2.dst.remote = 1;
    K3Launch k3{cur_gathered(P), P->push_bytes, P->n_workers, 1,
                1.0f / static_cast<float>(P->n_workers), P->d_err};
    PipeLaunch pl{};
    pl.flags = reinterpret_cast<uint32_t*>(P->d_ipc + P->pflags_off);
    for (int p = 0; p < P->n_workers; ++p)
        pl.peer_flags[p] = reinterpret_cast<uint32_t*>(P->peer_ipc[p] + P->pflags_off);
    pl.epoch = static_cast<uint32_t>(P->epoch);
    pl.rank = P->rank;
    pl.n_items = static_cast<uint32_t>(P->h_chunks.size());
    pl.done = P->d_done;
    if (const char* m = std::getenv("TGB_PIPEV")) pl.variant = std::atoi(m);
    if (std::getenv("TGB_PIPE_PROF")) {
        if (!P->d_pprof) {
            TGB_CUDA(cudaMalloc(&P->d_pprof, 8 * sizeof(unsigned long long)));
            TGB_CUDA(cudaMemset(P->d_pprof, 0, 8 * sizeof(unsigned long long)));
        }
        pl.prof = P->d_pprof;
        ++P->pipe_steps;
    }
    P->last = st;
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k23_pipelined(P->d_fat, pl.n_items, k2, k3, pl, st));
    if (ts >= 0) {
        uint64_t e[2];
        chunk_elems(P, P->h_chunks, 0, pl.n_items, e);
        const uint64_t N = P->n_workers, msg = (e[0] + 3) / 4 + 4 * e[1];
        t_end(P, st, ts, TGB_KERNEL_K23, 0, e[0] + e[1],
              4 * (e[0] + e[1]) + msg + N * msg + 4 * (e[0] + e[1]), (N - 1) * msg);
    }
    return TGB_OK;
}

#define TGB_TRY(expr)                        \
    do {                                     \
        const tgb_status s_ = (expr);        \
        if (s_ != TGB_OK) return s_;         \
    } while (0)

tgb_status tgb_stats(tgb_plan* P, void* stream) {
    if (!P || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    if (P->attached) ++P->epoch;  // a step begins: flip the gather-buffer parity
    for (int g = 0; g < n_groups(P); ++g) TGB_TRY(launch_stats(P, g, st));
    return TGB_OK;
}

tgb_status tgb_ternarize_pack(tgb_plan* P, uint64_t t, void* stream) {
    if (!P || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    for (int g = 0; g < n_groups(P); ++g) TGB_TRY(launch_tern(P, g, t, st));
    return TGB_OK;
}

tgb_status tgb_encode(tgb_plan* P, uint64_t t, void* stream) {
    TGB_TRY(tgb_stats(P, stream));
    return tgb_ternarize_pack(P, t, stream);
}

tgb_status tgb_share_scalers(tgb_plan* P, tgb_comm* C, void* stream) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    if (P->n_workers == 1) return TGB_OK;
    if (!C || C->nranks != P->n_workers) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    float* slots = reinterpret_cast<float*>(own_push(P));
    TGB_NCCL(ncclAllReduce(slots, slots, static_cast<size_t>(P->n_slots), ncclFloat, ncclMax,
                           C->comm, st));
    return TGB_OK;
}

tgb_status tgb_sync(tgb_plan* P, tgb_comm* C, void* stream) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    if (P->n_workers == 1) return TGB_OK;
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    if (P->attached) {  // data already moved by K1/K2: only order the step
        if (P->shard) return launch_shard_reduce(P, st);
        for (int g = 0; g < n_groups(P); ++g) TGB_TRY(launch_barrier(P, g, st));
        return TGB_OK;
    }
    if (!C || C->nranks != P->n_workers) return TGB_ERR_INVALID_ARGUMENT;
    const int ts = t_begin(P, st);
    TGB_NCCL(ncclAllGather(P->d_push, P->d_gathered, P->push_bytes, ncclUint8, C->comm, st));
    t_end(P, st, ts, TGB_KERNEL_NCCL, 0, P->total,
          static_cast<uint64_t>(P->n_workers) * P->push_bytes,
          static_cast<uint64_t>(P->n_workers - 1) * P->push_bytes);
    return TGB_OK;
}

tgb_status tgb_decode_average(tgb_plan* P, const uint8_t* d_src, int32_t n_workers, void* stream) {
    if (!P || !P->bound || n_workers < 1 || n_workers > kMaxWorkers)
        return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    if (!d_src && P->shard) {  // sharded exchange: decode this step's packed sums
        if (n_workers != P->n_workers) return TGB_ERR_INVALID_ARGUMENT;
        const int ts = t_begin(P, st);
        TGB_CUDA(launch_k3_expand(P->d_fat3, static_cast<uint32_t>(P->h_chunks3.size()),
                                  shard_launch(P), st));
        if (ts >= 0) {
            uint64_t e[2];
            chunk_elems(P, P->h_chunks3, 0, static_cast<uint32_t>(P->h_chunks3.size()), e);
            const uint64_t sums = P->nib ? (e[0] + 1) / 2 : e[0];
            t_end(P, st, ts, TGB_KERNEL_K3B, 0, e[0] + e[1], sums + 4 * e[1] + 4 * (e[0] + e[1]), 0);
        }
        return TGB_OK;
    }
    if (!d_src) d_src = cur_gathered(P);  // NULL: this step's gather buffer
    for (int g = 0; g < n_groups(P); ++g) TGB_TRY(launch_decode(P, g, d_src, n_workers, st));
    return TGB_OK;
}

// two-group schedule: the gi-th group to launch, and the event its chain waits for
static inline int stag_group(const tgb_plan* P, int gi) {
    if (P->stagger == 0) return 1 - gi;  // both at once, dominant chain launched first
    const int first = P->stagger == 2 ? 1 : 0;
    return gi == 0 ? first : 1 - first;
}
static inline cudaEvent_t stag_wait(const tgb_plan* P, int gi) {
    return (gi == 0 || P->stagger == 0) ? P->ev_fork : P->ev_stag;
}
static inline tgb_status stag_mark(tgb_plan* P, int gi, cudaStream_t gs) {
    if (gi == 0 && P->stagger != 0) TGB_CUDA(cudaEventRecord(P->ev_stag, gs));
    return TGB_OK;
}

tgb_status tgb_step(tgb_plan* P, tgb_comm* C, uint64_t t, void* stream) {
    if (!P || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    const bool nccl_exchange = P->n_workers > 1 && !P->attached;
    // N == 1: decode is this worker's own s*code; K2 writes it directly
    bool fuse = P->n_workers == 1;
    if (const char* m = std::getenv("TGB_FUSE1")) fuse = fuse && std::atoi(m) != 0;
    if (fuse) {
        P->last = st;
        if (!P->grouped) {
            TGB_TRY(tgb_stats(P, stream));
            return launch_tern(P, 0, t, st, true);
        }
        TGB_CUDA(cudaEventRecord(P->ev_fork, st));
        for (int gi = 0; gi < 2; ++gi) {
            const int g = stag_group(P, gi);
            cudaStream_t gs = P->gs[g];
            TGB_CUDA(cudaStreamWaitEvent(gs, stag_wait(P, gi), 0));
            TGB_TRY(launch_stats(P, g, gs));
            TGB_TRY(stag_mark(P, gi, gs));
            TGB_TRY(launch_tern(P, g, t, gs, true));
            TGB_CUDA(cudaEventRecord(P->ev_join[g], gs));
        }
        TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[0], 0));
        TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[1], 0));
        return TGB_OK;
    }
    if (P->attached && P->pipe) {
        TGB_TRY(tgb_stats(P, stream));  // K1 (scalers to every rank); epoch++
        if (P->p.share_mode == TGB_SHARE_PRESHARED) TGB_TRY(tgb_share_scalers(P, C, stream));
        return launch_pipelined(P, t, st);
    }
    if (!P->grouped || nccl_exchange) {
        TGB_TRY(tgb_stats(P, stream));
        if (P->p.share_mode == TGB_SHARE_PRESHARED && P->n_workers > 1)
            TGB_TRY(tgb_share_scalers(P, C, stream));
        TGB_TRY(tgb_ternarize_pack(P, t, stream));
        if (P->n_workers > 1) TGB_TRY(tgb_sync(P, C, stream));
        return tgb_decode_average(P, nullptr, P->n_workers, stream);
    }
    // overlapped two-group schedule: fork the step onto the plan's two streams
    // (group 0 = small layers at high priority, group 1 = the dominant layer),
    // join back into the caller's stream.
    P->last = st;
    if (P->attached) ++P->epoch;
    TGB_CUDA(cudaEventRecord(P->ev_fork, st));
    const uint8_t* src = cur_gathered(P);
    for (int gi = 0; gi < 2; ++gi) {
        const int g = stag_group(P, gi);
        cudaStream_t gs = P->gs[g];
        TGB_CUDA(cudaStreamWaitEvent(gs, stag_wait(P, gi), 0));
        TGB_TRY(launch_stats(P, g, gs));
        TGB_TRY(stag_mark(P, gi, gs));
        if (g == 1 && P->attached && P->pieces > 1) {
            // dominant layer in pieces: K2 piece p on gs, then on gs3 the barrier of
            // piece p (every rank's K2 piece p done) and its K3, overlapping K2 p+1
            for (int pc = 0; pc < P->pieces; ++pc) {
                TGB_TRY(launch_tern_rng(P, 1, P->pc_b[pc], P->pc_c[pc], t, gs, false));
                TGB_CUDA(cudaEventRecord(P->ev_piece[pc], gs));
                if (P->bstream) {  // barrier at the greatest priority, K3 piece on gs3
                    TGB_CUDA(cudaStreamWaitEvent(P->gsb[1], P->ev_piece[pc], 0));
                    TGB_TRY(launch_barrier(P, 2 + pc, P->gsb[1]));
                    TGB_CUDA(cudaEventRecord(P->ev_pbar[pc], P->gsb[1]));
                    TGB_CUDA(cudaStreamWaitEvent(P->gs3, P->ev_pbar[pc], 0));
                } else {
                    TGB_CUDA(cudaStreamWaitEvent(P->gs3, P->ev_piece[pc], 0));
                    TGB_TRY(launch_barrier(P, 2 + pc, P->gs3));
                }
                TGB_TRY(launch_decode_rng(P, 1, P->pc_b3[pc], P->pc_c3[pc], src, P->n_workers,
                                          P->gs3));
            }
            TGB_CUDA(cudaEventRecord(P->ev_join[g], P->gs3));
            continue;
        }
        TGB_TRY(launch_tern(P, g, t, gs));
        if (P->attached && P->bstream) {
            TGB_CUDA(cudaEventRecord(P->ev_b0[g], gs));
            TGB_CUDA(cudaStreamWaitEvent(P->gsb[g], P->ev_b0[g], 0));
            TGB_TRY(launch_barrier(P, g, P->gsb[g]));
            TGB_CUDA(cudaEventRecord(P->ev_b1[g], P->gsb[g]));
            TGB_CUDA(cudaStreamWaitEvent(gs, P->ev_b1[g], 0));
        } else if (P->attached) {
            TGB_TRY(launch_barrier(P, g, gs));
        }
        TGB_TRY(launch_decode(P, g, src, P->n_workers, gs));
        TGB_CUDA(cudaEventRecord(P->ev_join[g], gs));
    }
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[0], 0));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[1], 0));
    return TGB_OK;
}

// Per-tensor copies dst[l] <- src[l] (n_l floats), coalesced into one copy per run
// of tensors that are adjacent on BOTH sides (e.g. flat buffers whose tensors are
// back to back): one 553 MB copy instead of 32 runs PCIe ~10 % faster. Gaps are
// never copied (they may be someone else's memory).
static tgb_status copy_runs(const tgb_plan* P, const float* const* dst_c, const float* const* src,
                            cudaMemcpyKind kind, cudaStream_t st) {
    float* const* dst = const_cast<float* const*>(dst_c);
    const size_t nl = P->desc.size();
    size_t l = 0;
    while (l < nl) {
        if (!P->desc[l].n) {
            ++l;
            continue;
        }
        uint64_t n = P->desc[l].n;
        size_t e = l + 1;
        for (; e < nl; ++e) {
            const uint64_t m = P->desc[e].n;
            if (!m) continue;
            if (dst[e] != dst[l] + n || src[e] != src[l] + n) break;
            n += m;
        }
        TGB_CUDA(cudaMemcpyAsync(dst[l], src[l], n * sizeof(float), kind, st));
        l = e;
    }
    return TGB_OK;
}

// Host-buffer step: H2D of every tensor on a copy stream, tgb_step on `stream`,
// D2H of every averaged tensor on a second copy stream; `stream` finally waits
// for the D2H, so synchronising it means the outputs are in host memory. The
// next call's H2D only waits for this call's compute (the gradient buffers are
// free once K2 has read them), so it overlaps this call's D2H: PCIe runs full
// duplex across consecutive steps. Host buffers should be pinned.
tgb_status tgb_step_host(tgb_plan* P, tgb_comm* C, uint64_t t, const float* const* h_grads,
                         float* const* h_out, void* stream) {
    if (!P || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    const size_t nl = P->desc.size();
    if (nl > 0 && (!h_grads || !h_out)) return TGB_ERR_INVALID_ARGUMENT;
    for (size_t l = 0; l < nl; ++l)
        if (P->desc[l].n > 0 && (!h_grads[l] || !h_out[l])) return TGB_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    if (!P->host_io) {
        TGB_CUDA(cudaStreamCreateWithFlags(&P->s_h2d, cudaStreamNonBlocking));
        TGB_CUDA(cudaStreamCreateWithFlags(&P->s_d2h, cudaStreamNonBlocking));
        TGB_CUDA(cudaEventCreateWithFlags(&P->ev_h2d, cudaEventDisableTiming));
        TGB_CUDA(cudaEventCreateWithFlags(&P->ev_comp, cudaEventDisableTiming));
        TGB_CUDA(cudaEventCreateWithFlags(&P->ev_d2h, cudaEventDisableTiming));
        TGB_CUDA(cudaEventRecord(P->ev_comp, st));  // nothing computed yet
        TGB_CUDA(cudaEventRecord(P->ev_d2h, st));
        P->host_io = true;
    }
    TGB_CUDA(cudaStreamWaitEvent(P->s_h2d, P->ev_comp, 0));  // previous K2 read the gradients
    TGB_TRY_INNER(copy_runs(P, reinterpret_cast<const float* const*>(P->bound_g.data()), h_grads,
                            cudaMemcpyHostToDevice, P->s_h2d));
    TGB_CUDA(cudaEventRecord(P->ev_h2d, P->s_h2d));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_h2d, 0));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_d2h, 0));  // previous outputs copied out
    TGB_TRY(tgb_step(P, C, t, stream));
    TGB_CUDA(cudaEventRecord(P->ev_comp, st));
    TGB_CUDA(cudaStreamWaitEvent(P->s_d2h, P->ev_comp, 0));
    TGB_TRY_INNER(copy_runs(P, h_out, P->bound_out.data(), cudaMemcpyDeviceToHost, P->s_d2h));
    TGB_CUDA(cudaEventRecord(P->ev_d2h, P->s_d2h));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_d2h, 0));
    P->last = st;
    return TGB_OK;
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
// writing the averaged gradient: N = 1 (K2 fused decode) and the shared-scaler
// K3 of the fused / NCCL exchanges for N in {2, 3, 4, 8}
static bool opt_fusable(const tgb_plan* P) {
    if (const char* m = std::getenv("TGB_OPT_FUSED"))
        if (std::atoi(m) == 0) return false;
    if (P->n_workers == 1) return true;
    const int N = P->n_workers;
    if (P->r3) return true;  // k3_decode_r3<N, kOpt>, 3 <= N <= 8
    return P->p.scaler_sharing && !P->shard && !P->pipe && P->k3_variant >= 1 &&
           P->chunk3 == kChunk3 && (N <= 4 || N == 8);
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

tgb_status tgb_plan_attach_peers(tgb_plan* P, tgb_comm* C) {
    if (!P || !C) return TGB_ERR_INVALID_ARGUMENT;
    if (P->n_workers == 1) return TGB_OK;
    if (C->nranks != P->n_workers || C->rank != P->worker || P->n_workers > kMaxPeers)
        return TGB_ERR_INVALID_ARGUMENT;
    if (P->attached) return TGB_OK;
    cudaIpcMemHandle_t h;
    TGB_CUDA(cudaIpcGetMemHandle(&h, P->d_ipc));
    const int N = P->n_workers;
    std::vector<cudaIpcMemHandle_t> all(N);
    uint8_t* d_tmp = nullptr;
    TGB_CUDA(cudaMalloc(&d_tmp, sizeof(cudaIpcMemHandle_t) * (N + 1)));
    TGB_CUDA(cudaMemcpy(d_tmp, &h, sizeof(h), cudaMemcpyHostToDevice));
    const ncclResult_t r = ncclAllGather(d_tmp, d_tmp + sizeof(h), sizeof(h), ncclUint8, C->comm,
                                         nullptr);
    cudaError_t e = cudaStreamSynchronize(nullptr);
    if (r == ncclSuccess && e == cudaSuccess)
        e = cudaMemcpy(all.data(), d_tmp + sizeof(h), sizeof(h) * N, cudaMemcpyDeviceToHost);
    cudaFree(d_tmp);
    if (r != ncclSuccess) return TGB_ERR_NCCL;
    TGB_CUDA(e);
    P->rank = C->rank;
    for (int p = 0; p < N; ++p) {
        if (p == P->rank) {
            P->peer_ipc[p] = P->d_ipc;
            continue;
        }
        void* ptr = nullptr;
        TGB_CUDA(cudaIpcOpenMemHandle(&ptr, all[p], cudaIpcMemLazyEnablePeerAccess));
        P->peer_ipc[p] = static_cast<uint8_t*>(ptr);
    }
    P->attached = true;
    P->shard = P->shard_capable;
    P->pipe = P->pipe_capable;
    P->r3 = P->r3_capable && !P->shard && !P->pipe;
    return TGB_OK;
}

tgb_status tgb_plan_enable_timing(tgb_plan* P, int32_t capacity) {
    if (!P || capacity < 0) return TGB_ERR_INVALID_ARGUMENT;
    const size_t want = 2 * static_cast<size_t>(capacity);
    while (P->t_ev.size() < want) {
        cudaEvent_t e = nullptr;
        TGB_CUDA(cudaEventCreate(&e));
        P->t_ev.push_back(e);
    }
    P->t_rec.assign(static_cast<size_t>(capacity), tgb_kernel_time{});
    P->t_cap = capacity;
    P->t_used = 0;
    return TGB_OK;
}

tgb_status tgb_plan_read_timing(tgb_plan* P, tgb_kernel_time* out, int32_t cap, int32_t* n) {
    if (!P || (cap > 0 && !out) || !n) return TGB_ERR_INVALID_ARGUMENT;
    const int32_t m = std::min(cap, P->t_used);
    for (int32_t i = 0; i < m; ++i) {
        TGB_CUDA(cudaEventSynchronize(P->t_ev[2 * i + 1]));
        float ms = 0.0f, t0 = 0.0f;
        TGB_CUDA(cudaEventElapsedTime(&ms, P->t_ev[2 * i], P->t_ev[2 * i + 1]));
        TGB_CUDA(cudaEventElapsedTime(&t0, P->t_ev[0], P->t_ev[2 * i]));
        out[i] = P->t_rec[i];
        out[i].ms = ms;
        out[i].start_ms = t0;
    }
    *n = P->t_used;
    return TGB_OK;
}

tgb_status tgb_plan_attach_local(tgb_plan* const* plans, int32_t n) {
    if (!plans || n < 1 || n > kMaxPeers) return TGB_ERR_INVALID_ARGUMENT;
    for (int32_t p = 0; p < n; ++p) {
        tgb_plan* P = plans[p];
        if (!P || P->n_workers != n || P->worker != p || P->attached) return TGB_ERR_INVALID_ARGUMENT;
        // PRESHARED needs the max-allreduce between K1 and K2 (NCCL): ranks only
        if (n > 1 && P->p.share_mode == TGB_SHARE_PRESHARED) return TGB_ERR_UNSUPPORTED;
    }
    if (n == 1) return TGB_OK;
    int cur = 0;
    TGB_CUDA(cudaGetDevice(&cur));
    for (int32_t p = 0; p < n; ++p)
        for (int32_t q = 0; q < n; ++q) {
            const int dp = plans[p]->device, dq = plans[q]->device;
            if (dp == dq) continue;
            int ok = 0;
            TGB_CUDA(cudaDeviceCanAccessPeer(&ok, dp, dq));
            if (!ok) return TGB_ERR_UNSUPPORTED;
            TGB_CUDA(cudaSetDevice(dp));
            const cudaError_t e = cudaDeviceEnablePeerAccess(dq, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
            else if (e != cudaSuccess) {
                cudaSetDevice(cur);
                TGB_CUDA(e);
            }
        }
    TGB_CUDA(cudaSetDevice(cur));
    for (int32_t p = 0; p < n; ++p) {
        tgb_plan* P = plans[p];
        P->rank = p;
        for (int32_t q = 0; q < n; ++q) P->peer_ipc[q] = plans[q]->d_ipc;
        P->attached = true;
        P->local_peers = true;
        P->shard = P->shard_capable;
        P->pipe = P->pipe_capable;
        P->r3 = P->r3_capable && !P->shard && !P->pipe;
    }
    return TGB_OK;
}

tgb_status tgb_plan_last_buffers(tgb_plan* P, uint8_t** d_push, uint8_t** d_gathered) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    if (d_push) *d_push = own_push(P);
    if (d_gathered) *d_gathered = cur_gathered(P);
    return TGB_OK;
}

tgb_status tgb_plan_enable_code_stats(tgb_plan* P, int32_t on) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    P->code_stats = on != 0;
    return TGB_OK;
}

tgb_status tgb_plan_code_stats(tgb_plan* P, uint64_t* nonzero, uint64_t* total) {
    if (!P || !nonzero || !total) return TGB_ERR_INVALID_ARGUMENT;
    if (!P->code_stats) return TGB_ERR_INVALID_ARGUMENT;  // enable before the step
    TGB_CUDA(cudaStreamSynchronize(P->last));
    unsigned long long h[2] = {0, 0};
    TGB_CUDA(cudaMemcpy(h, P->d_nnz, sizeof(h), cudaMemcpyDeviceToHost));
    *nonzero = h[0] + (P->grouped ? h[1] : 0ull);
    uint64_t tot = 0;
    for (const LayerDev& L : P->h_layers)
        if (!(L.flags & kLayerPassthrough)) tot += L.n;
    *total = tot;
    return TGB_OK;
}

tgb_status tgb_check(tgb_plan* P, tgb_error* out) {
    if (!P || !out) return TGB_ERR_INVALID_ARGUMENT;
    TGB_CUDA(cudaStreamSynchronize(P->last));
    ErrWord e;
    TGB_CUDA(cudaMemcpy(&e, P->d_err, sizeof(e), cudaMemcpyDeviceToHost));
    out->flags = e.flags;
    out->layer = e.flags ? e.layer() : -1;
    out->index = e.flags ? e.index() : 0;
    if (e.flags) TGB_CUDA(cudaMemset(P->d_err, 0, sizeof(ErrWord)));
    return e.flags ? TGB_ERR_CODEC : TGB_OK;
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
    K2Launch k{d_codes, nullptr, nullptr, S->err, t, 0, 0, s};
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
