// Persistent plan kernels K1 (stats) and K2 (ternarize + pack).
//
// grid = min(tiles, SMs x resident CTAs); CTA c owns the contiguous tile run
// [c*T/G, (c+1)*T/G) of the plan's tile table (16 KB tiles, layer order).
// Each CTA is warp-specialized: warp 8 (lane 0) streams tiles global->shared
// with cp.async.bulk (TMA, SASS UBLKCP) into an S-stage ring guarded by
// full/empty mbarriers; warps 0..7 compute. The producer runs up to S tiles
// ahead of the consumers whatever they are doing, so HBM reads stay in
// flight through K2's Philox-heavy compute. K2 walks the SAME runs backwards:
// the tiles K1 read last are still L2-resident when K2 re-reads them (the
// second read of g is the only re-read the algorithm forces).
#include "tgb_device.cuh"
#include "tgb_internal.h"
#include "tgb_ring.cuh"
#include "tgb_stats.cuh"

#include <cmath>

namespace tgb {

struct PersistTables {
    const LayerDev* layers;
    const ChunkDev* tiles;
    const SegDev* segs;
    const CtaDev* ctas;
};

constexpr int kConsumerWarps = kThreads / 32;
constexpr int kBlock = kThreads + 32;  // 8 consumer warps + 1 producer warp

template <int S>
struct Ring {
    float4* buf;
    uint64_t* full;   // producer arrive.expect_tx + bulk-copy bytes
    uint64_t* empty;  // one arrive per consumer warp when done with the slot
    static constexpr size_t kSmem = S * kTileBytes + 2 * S * sizeof(uint64_t);

    __device__ __forceinline__ static Ring get() {
        extern __shared__ __align__(128) uint8_t dsmem[];
        Ring r;
        r.buf = reinterpret_cast<float4*>(dsmem);
        r.full = reinterpret_cast<uint64_t*>(dsmem + S * kTileBytes);
        r.empty = r.full + S;
        return r;
    }
    __device__ __forceinline__ void init() const {
        if (threadIdx.x == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], kConsumerWarps);
            }
            fence_barrier_init();
        }
        __syncthreads();
    }
    __device__ __forceinline__ const float4* slot(uint32_t i) const {
        return buf + (i % S) * (kTileElems / 4);
    }
    __device__ __forceinline__ void wait_full(uint32_t i) const {
        mbar_wait(&full[i % S], (i / S) & 1u);
    }
    __device__ __forceinline__ void release(uint32_t i) const {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[i % S]);
    }
};

// producer (warp 8, lane 0): tile_at(i) for i in [0, nt) into slot i % S.
// Unaligned layers complete the phase with a plain arrive; consumers then
// read those tiles from global memory.
template <int S, class TileAt>
__device__ __forceinline__ void produce(const Ring<S>& R, const PersistTables& T, uint32_t nt,
                                        TileAt tile_at) {
    if ((threadIdx.x & 31) != 0) return;
    for (uint32_t i = 0; i < nt; ++i) {
        const uint32_t s = i % S;
        if (i >= S) mbar_wait(&R.empty[s], ((i / S) & 1u) ^ 1u);
        const ChunkDev tl = T.tiles[tile_at(i)];
        const LayerDev& L = T.layers[tl.layer];
        const uint32_t bytes = (tl.count >> 2) * 16u;
        if ((L.flags & kLayerVecIn) && bytes) {
            mbar_arrive_expect_tx(&R.full[s], bytes);
            bulk_g2s(R.buf + s * (kTileElems / 4), L.g + tl.begin, bytes, &R.full[s]);
        } else {
            mbar_arrive(&R.full[s]);
        }
    }
}

constexpr int kK1Stages = 3;
constexpr int kK2Stages = 4;

// ================================================================= K1p
__global__ void __launch_bounds__(kBlock, 3) k1_persistent(PersistTables T, K1Out o) {
    const CtaDev c = T.ctas[blockIdx.x];
    if (c.seg_begin == c.seg_end) return;
    const Ring<kK1Stages> R = Ring<kK1Stages>::get();
    R.init();
    const uint32_t t0 = T.segs[c.seg_begin].tile_begin;
    const uint32_t nt = T.segs[c.seg_end - 1].tile_end - t0;
    if (threadIdx.x >= kThreads) {
        produce(R, T, nt, [t0](uint32_t i) { return t0 + i; });
        return;
    }
    const uint32_t tid = threadIdx.x;
    uint32_t seg = c.seg_begin;
    SegDev sg = T.segs[seg];
    LayerDev L = T.layers[sg.layer];
    uint64_t seg_count = 0;
    double x0 = static_cast<double>(__ldg(L.g + T.tiles[sg.tile_begin].begin));
    constexpr int U = kTileElems / 4 / kThreads;  // float4 per thread per tile
    double S[U], Q[U];  // independent chains (ILP); summed in fixed order
    float mx = 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) S[u] = Q[u] = 0.0;

    for (uint32_t i = 0; i < nt; ++i) {
        const ChunkDev tl = T.tiles[t0 + i];
        const uint32_t n4 = tl.count >> 2;
        const float* g = L.g + tl.begin;
        R.wait_full(i);
        if (L.flags & kLayerVecIn) {
            const float4* tile = R.slot(i);
            if (n4 == kTileElems / 4) {
#pragma unroll
                for (int u = 0; u < U; ++u) acc4(tile[tid + u * kThreads], x0, S[u], Q[u], mx);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t j = tid + u * kThreads;
                    if (j < n4) acc4(tile[j], x0, S[u], Q[u], mx);
                }
            }
        } else {
            for (uint32_t j = tid; j < n4; j += kThreads)
                acc4(make_float4(g[4 * j], g[4 * j + 1], g[4 * j + 2], g[4 * j + 3]), x0, S[0],
                     Q[0], mx);
        }
        R.release(i);
        for (uint32_t e = 4 * n4 + tid; e < tl.count; e += kThreads) acc1(g[e], x0, S[0], Q[0], mx);
        seg_count += tl.count;
        if (t0 + i + 1 == sg.tile_end) {  // segment complete: partial (+ merge if last)
            double s_all = 0.0, q_all = 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                s_all += S[u];
                q_all += Q[u];
                S[u] = Q[u] = 0.0;
            }
            k1_emit_and_finalize<ConsumerBar>(o, L, sg.layer, seg, L.first_seg, L.n_segs,
                                              seg_count, x0, s_all, q_all, mx);
            mx = 0.0f;
            seg_count = 0;
            if (++seg < c.seg_end) {
                sg = T.segs[seg];
                L = T.layers[sg.layer];
                x0 = static_cast<double>(__ldg(L.g + T.tiles[sg.tile_begin].begin));
            }
            ConsumerBar::sync();  // shared reduction scratch is reused by the next segment
        }
    }
}

// ================================================================= K2p
struct K2PArgs {
    uint8_t* push;
    const float* slots;
    const float* bounds;
    uint64_t t;
};

template <bool kRolling>
__global__ void __launch_bounds__(kBlock, 3) k2_persistent(PersistTables T, K2PArgs a) {
    const CtaDev c = T.ctas[blockIdx.x];
    if (c.seg_begin == c.seg_end) return;
    const Ring<kK2Stages> R = Ring<kK2Stages>::get();
    R.init();
    const uint32_t t_first = T.segs[c.seg_begin].tile_begin;
    const uint32_t t_last = T.segs[c.seg_end - 1].tile_end - 1;  // walk t_last .. t_first
    const uint32_t nt = t_last - t_first + 1;
    if (threadIdx.x >= kThreads) {
        produce(R, T, nt, [t_last](uint32_t i) { return t_last - i; });
        return;
    }
    const uint32_t tid = threadIdx.x;
    uint32_t cur_layer = 0xFFFFFFFFu;
    LayerDev L;
    Decider dec;
    Philox4<kRolling> ph;
    float s = 0.0f;
    for (uint32_t i = 0; i < nt; ++i) {
        const ChunkDev tl = T.tiles[t_last - i];
        if (tl.layer != cur_layer) {  // uniform: new layer's scaler, bound and key
            cur_layer = tl.layer;
            L = T.layers[cur_layer];
            s = a.slots[L.slot];
            dec.init(a.bounds[cur_layer], s);
            ph.init(L.key0, L.key1, 0u, a.t);  // byte index < 2^32 (n < 2^34)
        }
        const uint32_t nbytes = (tl.count + 3) >> 2;
        const uint32_t nfull = tl.count >> 2;
        const uint32_t qbase = static_cast<uint32_t>(tl.begin >> 2);
        uint8_t* codes = a.push + L.code_off + qbase;
        const float* g = L.g + tl.begin;
        constexpr int U = kTileElems / 4 / kThreads;  // 4 code bytes per thread
        if (s == 0.0f) {  // codec.hpp:155-159 (auto scaler: every clipped value is 0)
            R.wait_full(i);
            R.release(i);
            for (uint32_t q = tid; q < nbytes; q += kThreads) codes[q] = 0;
        } else if ((L.flags & kLayerVecIn) && nfull == kTileElems / 4) {
            // Philox first (independent of the tile), then wait for the data
            uint32_t ctr[U];
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ctr[u] = qbase + tid + u * kThreads;
            ph(ctr, r);
            R.wait_full(i);
            const float4* tile = R.slot(i);
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = tile[tid + u * kThreads];
            R.release(i);
            uint32_t byte[U];
            float amb = -1.0f;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                byte[u] = dec.byte_fast(v[u], r[u], amb);
            }
            if (amb >= 0.0f || dec.exact_all) {
#pragma unroll
                for (int u = 0; u < U; ++u) byte[u] = dec.byte_exact(v[u], r[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) codes[tid + u * kThreads] = static_cast<uint8_t>(byte[u]);
        } else {  // partial tile / unaligned layer: per-byte path
            R.wait_full(i);
            const float4* tile = R.slot(i);
            const bool vec = (L.flags & kLayerVecIn) != 0;
            for (uint32_t q = tid; q < nbytes; q += kThreads) {
                float4 v;
                if (vec && q < nfull) {
                    v = tile[q];
                } else {
                    float x[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t k = 4 * q + e;
                        x[e] = k < tl.count ? g[k] : 0.0f;
                    }
                    v = make_float4(x[0], x[1], x[2], x[3]);
                }
                uint32_t ctr[1] = {qbase + q};
                uint4 r[1];
                ph(ctr, r);
                codes[q] = static_cast<uint8_t>(dec.byte(v, r[0]));
            }
            R.release(i);
        }
    }
}

// ============================================================ launchers
static bool g_attr_set[64] = {};

static cudaError_t ensure_attrs() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64 && g_attr_set[dev]) return cudaSuccess;
    e = cudaFuncSetAttribute(k1_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(Ring<kK1Stages>::kSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k2_persistent<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(Ring<kK2Stages>::kSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k2_persistent<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(Ring<kK2Stages>::kSmem));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) g_attr_set[dev] = true;
    return cudaSuccess;
}

cudaError_t persistent_grid(uint32_t* ctas) {
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, b1 = 0, b2 = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k1_persistent, kBlock,
                                                           Ring<kK1Stages>::kSmem)) != cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k2_persistent<false>, kBlock,
                                                           Ring<kK2Stages>::kSmem)) != cudaSuccess)
        return e;
    const int b = b1 < b2 ? b1 : b2;
    *ctas = static_cast<uint32_t>(sms * (b > 0 ? b : 1));
    return cudaSuccess;
}

cudaError_t launch_k1_persistent(const PersistLaunch& P, const K1Launch& p, cudaStream_t st) {
    if (P.n_ctas == 0) return cudaSuccess;
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    K1Out o{p.partials, p.layer_done, p.global_done, p.bounds, p.slots, p.err, p.clip_factor,
            p.global_bucketing, p.n_layers, p.n_active_layers, P.layers};
    k1_persistent<<<P.n_ctas, kBlock, Ring<kK1Stages>::kSmem, st>>>(
        PersistTables{P.layers, P.tiles, P.segs, P.ctas}, o);
    return cudaGetLastError();
}

cudaError_t launch_k2_persistent(const PersistLaunch& P, const K2Launch& p, cudaStream_t st) {
    if (P.n_ctas == 0) return cudaSuccess;
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    K2PArgs a{p.push, p.slots, p.bounds, p.t};
    const PersistTables T{P.layers, P.tiles, P.segs, P.ctas};
    if (P.variant == 1)
        k2_persistent<true><<<P.n_ctas, kBlock, Ring<kK2Stages>::kSmem, st>>>(T, a);
    else
        k2_persistent<false><<<P.n_ctas, kBlock, Ring<kK2Stages>::kSmem, st>>>(T, a);
    return cudaGetLastError();
}

}  // namespace tgb
