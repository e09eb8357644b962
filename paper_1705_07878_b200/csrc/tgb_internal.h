// Host-side launch interface between capi.cu and kernels.cu (not exported).
#pragma once

#include <cuda_runtime.h>

#include "tgb/terngrad_b200.h"
#include "tgb_device.cuh"

namespace tgb {

// flag arrays of the cross-GPU barrier (inside each rank's IPC allocation)
struct PeerFlags {
    uint64_t* remote[kMaxPeers];  // address of THIS rank's slot in peer p's flag array
    uint64_t* local;              // this rank's flag array (one slot per peer)
    int32_t n;
};

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
    int32_t variant = 0;  // chunk K1 kernel variant (TGB_K1V, A/B only)
    PeerPush push{};      // scaler slot destinations
    const TensorDev* tensors = nullptr;  // plan: tensor table (per-tensor finalize)
    unsigned long long* nnz = nullptr;   // telemetry counter to reset (this group)
    uint32_t keep_chunks = 0;            // TGB_K1KEEP: last units kept in L2 for K2 (A/B)
};

struct K2Launch {
    uint8_t* push;
    const float* slots;
    const float* bounds;
    ErrWord* err;
    uint64_t t;
    int32_t reverse;
    int32_t variant = 0;   // chunk K2 kernel variant (TGB_K2V, A/B only)
    float s_imm = 0.0f;    // single-layer: scaler by value when slots == nullptr
    uint64_t rng_base = 0; // single-layer: ternarize rng_base (codec.hpp:148)
    PeerPush dst{};        // plan: code destinations (n == 0: push only)
    unsigned long long* nnz = nullptr;  // telemetry: nonzero-code counter of this group
    const OptDev* optd = nullptr;       // fused decode -> optimizer (per-block state table)
    OptArgs opt{};
    int32_t shard_n = 0;        // sharded exchange: codes go to the chunk's owner only
    uint32_t shard_bounds[kMaxPeers + 1] = {};
    int32_t fuse_decode = 0;    // N == 1 step: K2 also writes the decoded output (K3 fused)
    int32_t direct = 0;         // thread-contiguous code bytes stored straight from registers
    int32_t bulk = 0;           // TGB_K2BULK (A/B): code stores as TMA bulk copies
    int32_t r3 = 0;             // fused exchange: radix-3 wire codes to dst, 2-bit codes to push
    int32_t pdl = 0;            // TGB_PDL: K2 as K1's programmatic dependent (1), + L2 prefetch (2)
};

struct K3Launch {
    const uint8_t* src;
    uint64_t stride;
    int32_t n_workers;
    int32_t sharing;
    float inv_n;
    ErrWord* err;
    float s_imm = 0.0f;    // single-layer: scaler by value when scalers == nullptr
    int32_t variant = 0;   // TGB_K3V (A/B): 1 = smem-staged 16-B code loads
    uint32_t chunk3 = 0;   // plan K3 chunk elements (the staged variant needs kChunk3)
    const OptDev* optd = nullptr;  // fused decode -> optimizer (staged kernel, N in {1,2,3,4,8})
    OptArgs opt{};
    int32_t r3 = 0;  // the source holds radix-3 wire codes (chunks of kChunk3R3 elements)
};

struct ShardLaunch {
    const uint8_t* src;        // own gather buffer
    uint64_t stride;           // push_bytes
    uint8_t* sums[kMaxPeers];  // every rank's sums buffer (this step's parity)
    const uint8_t* own_sums;
    int32_t n_workers;
    int32_t nib;
    float inv_n;
    ErrWord* err;
    int32_t bulk = 0;  // K3a sums stores as TMA bulk copies
};

struct PipeLaunch {
    uint32_t* flags;                  // this rank's item flags [item][kMaxPeers]
    uint32_t* peer_flags[kMaxPeers];  // every rank's flags array
    uint32_t epoch;
    int32_t rank;
    uint32_t n_items;
    int32_t variant = 0;  // TGB_PIPEV (A/B)
    uint32_t* done = nullptr;  // local per-item done flags (n_items)
    unsigned long long* prof = nullptr;  // TGB_PIPE_PROF: 8 phase cycle counters
};

cudaError_t launch_k1_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K1Launch& p, cudaStream_t st);
cudaError_t launch_k2_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K2Launch& p, cudaStream_t st);
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
cudaError_t launch_k23_pipelined(const ChunkFat* chunks, uint32_t n_items, const K2Launch& k2,
                                 const K3Launch& k3, const PipeLaunch& p, cudaStream_t st);
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
cudaError_t launch_peer_barrier(const PeerFlags& f, uint64_t epoch, ErrWord* err,
                                cudaStream_t st);
cudaError_t launch_rng_bits(uint32_t key0, uint32_t key1, uint64_t t, uint64_t k0, uint64_t n,
                            uint32_t* out, cudaStream_t st);

}  // namespace tgb
