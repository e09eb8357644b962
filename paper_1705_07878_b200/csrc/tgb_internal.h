// Host-side launch interface between capi.cu and kernels.cu (not exported).
#pragma once

#include <cuda_runtime.h>

#include "tgb/terngrad_b200.h"
#include "tgb_device.cuh"

namespace tgb {

// rng.hpp:50-54: RngStream key words
inline void philox_key(uint64_t seed, uint64_t name_hash, uint64_t worker, uint32_t& k0,
                       uint32_t& k1) {
    k0 = static_cast<uint32_t>(seed ^ name_hash);
    k1 = static_cast<uint32_t>((seed >> 32) ^ (name_hash >> 32) ^
                               (worker * 0x9E3779B97F4A7C15ull));
}

inline uint32_t layer_vec_flags(const void* g, const void* out) {
    uint32_t f = 0;
    if ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) f |= kLayerVecIn;
    if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) f |= kLayerVecOut;
    return f;
}

// flag records of the cross-GPU barrier (inside each rank's IPC allocation):
// {epoch, iteration} per (barrier slot, peer), 16 bytes each
struct PeerFlags {
    uint64_t* remote[kMaxPeers];  // THIS rank's record in peer p's flag array
    uint64_t* local;              // this rank's records (one per peer)
    int32_t n;
};
constexpr int kBarrierSpin = 0;   // publish, then wait for every peer (one GPU per process)
constexpr int kBarrierPost = 1;   // publish only (LocalCluster, ordered by events)
constexpr int kBarrierCheck = 2;  // verify the peers' records, no wait (LocalCluster)
constexpr int kBarrierWait = 3;   // wait for the peers' records posted by K2 (overlapped)

// load every kernel the plans launch (no lazy loading inside a step: a lazily
// loaded kernel's first launch waits for the device to idle)
cudaError_t preload_kernels();

struct K1Launch {
    Partial* partials;
    uint32_t* layer_done;
    uint32_t* global_done;
    float* bounds;
    float* slots;
    ErrWord* err;
    float clip_factor;
    int32_t global_bucketing;
    int32_t n_layers;
    int32_t n_active_layers;
    PeerPush push{};      // scaler slot destinations
    const TensorDev* tensors = nullptr;  // plan: tensor table (per-tensor finalize)
    unsigned long long* nnz = nullptr;   // telemetry counter to reset (this group)
    uint32_t keep_chunks = 0;            // last units kept in L2 (evict_last) for K2 (N == 1)
    int32_t n_tensors = 0;               // fused K1+K2: ready[n_tensors] is the Global flag
    uint32_t* bmax = nullptr;            // FixedSize: per-block max |x| (then k1_bucket_slots)
    Partial* gpart = nullptr;            // two-level finalize: group partials / counters
    uint32_t* gdone = nullptr;
};

struct K2Launch {
    uint8_t* push;
    const float* slots;
    const float* bounds;
    ErrWord* err;
    uint64_t t;
    int32_t reverse;
    float s_imm = 0.0f;    // single-layer: scaler by value when slots == nullptr
    uint64_t rng_base = 0; // single-layer: ternarize rng_base (codec.hpp:148)
    PeerPush dst{};        // plan: code destinations (n == 0: push only)
    unsigned long long* nnz = nullptr;  // telemetry: nonzero-code counter of this group
    const OptDev* optd = nullptr;       // fused decode -> optimizer (per-block state table)
    OptArgs opt{};
    int32_t shard_n = 0;        // sharded exchange: codes go to the chunk's owner only
    uint32_t shard_bounds[kMaxPeers + 1] = {};
    int32_t fuse_decode = 0;    // N == 1 step: K2 also writes the decoded output (K3 fused)
    int32_t pdl = 0;            // K2 as K1's programmatic dependent (1), + L2 prefetch (2, 3)
    uint32_t keep_from = ~0u;   // work items K1 loaded evict_last (demoted by K2)
    uint32_t pull8 = 0;  // split exchange: see pulled_item (kernels.cu)
    int32_t rank = 0;
    int32_t slot_push = 0;  // K2 stores the scaler slots into the peers (see K2Args)
    // overlapped exchange (n_pieces > 0): see K2Args
    int32_t n_pieces = 0;
    uint32_t piece_bounds[kMaxPieces + 1] = {};
    uint32_t owner_bounds[kMaxPieces][kMaxPeers + 1] = {};
    uint32_t* piece_cnt = nullptr;
    uint64_t* flag_remote[kMaxPeers] = {};
    int32_t n_flags = 0;
    uint64_t epoch = 0;
};

struct K3Launch {
    const uint8_t* src;
    uint64_t stride;
    int32_t n_workers;
    int32_t sharing;
    float inv_n;
    ErrWord* err;
    float s_imm = 0.0f;    // single-layer: scaler by value when scalers == nullptr
    const OptDev* optd = nullptr;  // fused decode -> optimizer (staged kernel, N <= 8)
    OptArgs opt{};
    int32_t gate = 0;  // skip the decode when the step's exchange failed (skew / timeout)
    uint32_t pull8 = 0;  // split exchange: pulled items of worker w at wsrc[w] (its memory)
    const uint8_t* wsrc[kMaxPeers] = {};
};

struct ShardLaunch {
    const uint8_t* src;        // own gather buffer
    uint64_t stride;           // push_bytes
    uint8_t* sums[kMaxPeers];  // every rank's sums buffer (this step's parity)
    const uint8_t* own_sums;
    int32_t n_workers;
    int32_t radix_m;           // base-(2N+1) digits per u32 word
    uint32_t chunk12;          // K2 work-item elements (a full chunk's sums region)
    uint32_t sum_region;       // bytes of a full chunk's sums region
    float inv_n;
    ErrWord* err;
};


cudaError_t launch_k1_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K1Launch& p, cudaStream_t st);
cudaError_t launch_k2_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K2Launch& p, cudaStream_t st);
// fused K1 + K2 (small sets): n_k1 ternary units, n_k2 units (incl. passthrough);
// ready = n_tensors + 1 epoch flags
cudaError_t launch_k12_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_k1,
                             uint32_t n_k2, const K1Launch& p1, const K2Launch& p2,
                             uint32_t* ready, uint32_t epoch, cudaStream_t st);
// FixedSize plans, after K1: bucket scalers from the per-block maxima (meta[b] =
// {tensor, slot}, slot ~0u for passthrough blocks)
cudaError_t launch_k1_bucket_slots(const LayerDev* layers, const uint2* meta, uint32_t n_blocks,
                                   const K1Launch& p, cudaStream_t st);
cudaError_t launch_k1_single(const LayerDev& L, const K1Launch& p, cudaStream_t st);
cudaError_t launch_k2_single(const LayerDev& L, const K2Launch& p, cudaStream_t st);
cudaError_t launch_k3_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K3Launch& p, cudaStream_t st);
cudaError_t launch_k3_single(const LayerDev& L, const uint8_t* const* codes, const float* scalers,
                             const K3Launch& p, cudaStream_t st);
cudaError_t launch_average_raw(int32_t n_workers, const float* const* vals, uint64_t n,
                               float* out, cudaStream_t st);
cudaError_t launch_k3_reduce(const ChunkFat* chunks, uint32_t n_chunks, const ShardLaunch& p,
                             cudaStream_t st);
cudaError_t launch_k3_expand(const ChunkFat* chunks, uint32_t n_chunks, const ShardLaunch& p,
                             cudaStream_t st);
cudaError_t launch_histogram(const float* v, uint64_t n, uint32_t bins, uint32_t* mm,
                             int nan_first, unsigned long long* counts, double* edges,
                             cudaStream_t st, int pass);
cudaError_t launch_opt_apply(const OptArgs& o, uint64_t n, float* w, const float* g, float* s1,
                             float* s2, cudaStream_t st);
cudaError_t launch_wire_gather(const uint8_t* push, const WireSeg* d_segs, uint32_t n_segs,
                               uint8_t* frame, cudaStream_t st);
cudaError_t launch_pull_decode(const uint8_t* payload, const PullSeg* d_segs, uint32_t n_segs,
                               uint32_t total_threads, int* bad, cudaStream_t st);
cudaError_t launch_clip_apply(const float* g, uint64_t n, const float* bound, float* out,
                              cudaStream_t st);
cudaError_t launch_peer_barrier(const PeerFlags& f, uint64_t epoch, uint64_t t, int mode,
                                ErrWord* err, cudaStream_t st);
cudaError_t launch_slot_max(float* own, const uint8_t* gather, uint64_t stride, int n,
                            int n_slots, cudaStream_t st);
cudaError_t launch_rng_bits(uint32_t key0, uint32_t key1, uint64_t t, uint64_t k0, uint64_t n,
                            uint32_t* out, cudaStream_t st);

}  // namespace tgb
