// B200 (sm_100a) kernels of the TernGrad ternarize + sync + decode path.
//
//   K1 tgb_stats        clip bound (fp64 sigma) + max-abs scaler per layer
//                        codec.hpp:101-134 (stddev, clip, scaler), :212-216 (Global)
//   K2 tgb_ternarize    stochastic ternarize + 2-bit pack, one Philox block per code byte
//                        codec.hpp:148-175, rng.hpp:20-71
//   K3 tgb_decode       unpack + integer sum over workers + LUT decode to fp32
//                        codec.hpp:281-307 == cluster.hpp:189-204 + wire.hpp:206-228
//
// All three are HBM-streaming kernels: 128-bit coalesced loads/stores of the
// fp32 streams, one CTA (256 threads) per work item = a chunk of one block
// (32K elements for K1/K2, 16K for K3). A block is one bucket of a tensor
// (the whole tensor for PerTensor/Global, k elements for FixedSize) or a
// passthrough tensor (raw fp32, codec.hpp:206-209).
#include "tgb_device.cuh"
#include "tgb_internal.h"
#include "tgb_stats.cuh"

#include <cfloat>
#include <cmath>

namespace tgb {

// ----------------------------------------------------------------- sources
// A "source" maps blockIdx.x to (chunk, layer). Table: plan tables in HBM.
// Single: one layer passed by value (per-layer API), chunks computed.
struct TableSource {
    const ChunkFat* fat;
    __device__ __forceinline__ void get(uint32_t b, ChunkDev& ch, LayerDev& L) const {
        const ChunkFat* f = fat + b;
        ch = f->ch;
        L = f->L;
    }
};

struct SingleSource {
    LayerDev L;
    uint32_t chunk;  // elements per work item
    __device__ __forceinline__ void get(uint32_t b, ChunkDev& ch, LayerDev& L_) const {
        ch.layer = 0;
        ch.begin = b * chunk;
        ch.nblk = 1;
        const uint64_t rem = L.n - ch.begin;
        ch.count = static_cast<uint32_t>(rem < chunk ? rem : chunk);
        L_ = L;
    }
};

// RNG stream index of a block's first element: the bucket's element offset
// inside its tensor (ternarize rng_base, codec.hpp:167 via :229), or the
// per-layer API's rng_base (passed whole, it may exceed 32 bits).
__device__ __forceinline__ uint64_t block_rng_base(const LayerDev& L) {
    return 4ull * L.rng_q + ((L.flags >> kLayerShiftBit) & 3u);
}

// ====================================================================== K1
// One CTA per work item (a chunk of one block); the tensor's last arriving CTA
// merges the tensor's partials (tgb_stats.cuh). Passthrough blocks have no
// statistics (codec.hpp:206-209) and are never in a K1 grid.
// kHint: loads carry an L2 policy instead of .cs: evict_last for the launch's
// last units (K2 walks chunks last-to-first and re-reads them from L2),
// evict_first elsewhere (TGB_K1KEEP, A/B).
template <bool kHint>
__device__ __forceinline__ float4 k1_ld4(const float4* p, uint64_t pol) {
    if constexpr (kHint) {
        float4 v;
        asm("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
            : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
            : "l"(p), "l"(pol));
        return v;
    } else {
        return __ldcs(p);
    }
}

// log2(k) of a multi-bucket tensor's buckets
__device__ __forceinline__ uint32_t bucket_log2(const LayerDev& L) {
    return (L.flags >> kBucketShiftBit) & 31u;
}

constexpr uint32_t kMaxItemBuckets = kChunk12 / 64;  // k >= 64

// K1 unit spanning ch.nblk whole buckets of a FixedSize(k) tensor (k = 2^p >= 64):
// the same fp64 moments as k1_unit (statistics are per TENSOR, codec.hpp:206-209),
// plus every bucket's max |x| (scaler before the clip, :226-230). A float4 lies
// in one bucket; lanes holding the same bucket (__match_any_sync) reduce with
// one REDUX and their leader folds it into a shared-memory max per bucket, which
// the CTA finally stores to bmax[block] (the item owns its buckets whole).
template <int U, class Reload>
__device__ __forceinline__ void k1_unit_mb(const K1Out& o, const ChunkDev& ch0, const LayerDev& L0,
                                           uint32_t unit, Reload reload) {
    __shared__ uint32_t smax[kMaxItemBuckets];
    const uint32_t tid = threadIdx.x;
    for (uint32_t j = tid; j < ch0.nblk; j += kThreads) smax[j] = 0u;
    __syncthreads();
    const float* g = L0.g;
    const uint32_t count = ch0.count;
    const uint32_t sh4 = bucket_log2(L0) - 2;  // float4 index -> bucket
    const double x0 = static_cast<double>(__ldg(g));
    double S = 0.0, Q = 0.0;
    float mx = 0.0f;
    auto fold = [&](uint32_t j, float m) {  // per-bucket max of non-negative floats as bits
        const uint32_t peers = __match_any_sync(__activemask(), j);
        const uint32_t v = __reduce_max_sync(peers, __float_as_uint(m));
        if ((threadIdx.x & 31u) == static_cast<uint32_t>(__ffs(peers) - 1)) atomicMax(smax + j, v);
    };
    const float4* g4 = reinterpret_cast<const float4*>(g);
    const uint32_t n4 = count >> 2;  // k % 4 == 0: only the tensor's last bucket can be ragged
    uint32_t i = tid;
    for (; i + (U - 1) * kThreads < n4; i += U * kThreads) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(g4 + i + u * kThreads);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc4(v[u], x0, S, Q, mx);
            fold((i + u * kThreads) >> sh4, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)),
                                                  fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
        }
    }
    for (; i < n4; i += kThreads) {
        const float4 v = __ldcs(g4 + i);
        acc4(v, x0, S, Q, mx);
        fold(i >> sh4, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (uint32_t e = (n4 << 2) + tid; e < count; e += kThreads) {
        const float x = __ldcs(g + e);
        acc1(x, x0, S, Q, mx);
        atomicMax(smax + (e >> (sh4 + 2)), __float_as_uint(fabsf(x)));
    }
    __syncthreads();
    asm volatile("" ::: "memory");  // re-read the descriptors (see k1_unit)
    ChunkDev ch;
    LayerDev L;
    reload(ch, L);
    for (uint32_t j = tid; j < ch.nblk; j += kThreads) o.bmax[ch.layer + j] = smax[j];
    k1_emit_and_finalize(o, L, ch.layer, unit, L.first_chunk, L.n_chunks, count, x0, S, Q, mx,
                         false);
}

// One K1 work unit (a chunk of one block): fp64 moments of the chunk shifted by
// its first element, then the partial + the tensor's finalize (tgb_stats.cuh).
// `reload(ch, L)` fetches the unit's descriptors again for the finalize: with them
// live across the loop the 64-register budget left room for only 5 of the 8 float4
// loads per batch (SASS: 5 + 1 + 2 LDG.128), and K1 ran 105 us instead of the 84 us of
// the same loop in tools/k1_variants.cu; re-fetched (an L1/L2 hit) all 8 issue together.
template <int U, int A, bool kHint, class Reload>
__device__ __forceinline__ void k1_unit(const K1Out& o, const ChunkDev& ch0, const LayerDev& L0,
                                        uint32_t unit, Reload reload) {
    if (ch0.nblk > 1) {  // multi-bucket item
        k1_unit_mb<U>(o, ch0, L0, unit, reload);
        return;
    }
    const float* g = L0.g + ch0.begin;
    const uint32_t count = ch0.count;
    const bool vec_in = (L0.flags & kLayerVecIn) != 0;
    const double x0 = static_cast<double>(__ldg(g));  // per-chunk shift
    double S[A], Q[A];  // A independent fp64 chains; combined in fixed order
    float mx = 0.0f;
#pragma unroll
    for (int k = 0; k < A; ++k) S[k] = Q[k] = 0.0;
    const uint32_t tid = threadIdx.x;
    uint32_t done = 0;
    uint64_t pol = 0;
    if constexpr (kHint) {
        if (unit >= o.keep_from)
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        else
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    }
    if (vec_in) {
        const float4* g4 = reinterpret_cast<const float4*>(g);
        const uint32_t n4 = count >> 2;
        uint32_t i = tid;
        for (; i + (U - 1) * kThreads < n4; i += U * kThreads) {  // U x 16 B in flight per thread
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = k1_ld4<kHint>(g4 + i + u * kThreads, pol);
#pragma unroll
            for (int u = 0; u < U; ++u) acc4(v[u], x0, S[u % A], Q[u % A], mx);
        }
        for (; i < n4; i += kThreads) acc4(k1_ld4<kHint>(g4 + i, pol), x0, S[0], Q[0], mx);
        done = n4 << 2;
    }
    for (uint32_t i = done + tid; i < count; i += kThreads) acc1(__ldcs(g + i), x0, S[0], Q[0], mx);
    double s_all = S[0], q_all = Q[0];
#pragma unroll
    for (int k = 1; k < A; ++k) {
        s_all += S[k];
        q_all += Q[k];
    }
    asm volatile("" ::: "memory");  // the descriptors are re-read, not kept in registers
    ChunkDev ch;
    LayerDev L;
    reload(ch, L);
    k1_emit_and_finalize(o, L, ch.layer, unit, L.first_chunk, L.n_chunks, count, x0, s_all,
                         q_all, mx);
}

// K1 is memory-bound: the fp64 moments (F2F + DADD + DFMA per element) run under
// the load stream; with the same grid, a plain float sum streams the same
// bytes no faster (tools/k1_variants.cu, profiles/r02_k1_variants.log).
template <class Src, int U = 8, int A = 1, int kMinBlocks = 1, bool kHint = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k1_stats(Src src, K1Out o) {
    // K2 (a programmatic dependent) may be scheduled once every K1 CTA has
    // started; it waits on griddepcontrol.wait for K1's completion before reading scalers
    asm volatile("griddepcontrol.launch_dependents;");
    ChunkDev ch;
    LayerDev L;
    src.get(blockIdx.x, ch, L);
    if (o.nnz && blockIdx.x == 0 && threadIdx.x == 0) *o.nnz = 0;  // this group's K2 counts next
    if (L.flags & kLayerPassthrough) return;
    k1_unit<U, A, kHint>(o, ch, L, blockIdx.x,
                         [&](ChunkDev& c, LayerDev& l) { src.get(blockIdx.x, c, l); });
}

// K1b (FixedSize plans): every bucket's scaler from its max and its tensor's
// clip bound, s = min(max |part|, bound) = max |clip(part)| (codec.hpp:121-122,
// :226-230; a non-finite tensor has bound 0, so s = 0), into the scaler slots
// (and every peer's copy); resets the bucket maxima for the next step.
// meta[b] = {tensor, slot} (slot ~0u: passthrough block).
__global__ void __launch_bounds__(kThreads) k1_bucket_slots(const uint2* meta, uint32_t n_blocks,
                                                            K1Out o) {
    for (uint32_t b = blockIdx.x * kThreads + threadIdx.x; b < n_blocks; b += gridDim.x * kThreads) {
        const uint2 m = meta[b];
        if (m.y == ~0u) continue;
        const float bound = __ldcg(o.bounds + o.tensors[m.x].first_block);
        const float mx = __uint_as_float(o.bmax[b]);
        o.bmax[b] = 0u;
        o.bounds[b] = bound;
        put_slot(o, static_cast<int32_t>(m.y), fminf(mx, bound));
    }
}

// ====================================================================== K2
struct K2Args {
    uint8_t* push;       // codes at push + L.code_off (table) / codes base (single)
    const float* slots;  // scaler slots (device)
    const float* bounds; // per layer clip bounds (device); nullptr => +inf
    ErrWord* err;
    uint64_t t;
    int32_t reverse;     // walk chunks last-to-first (re-read K1's L2-resident tail)
    int32_t check;       // per-layer API: raise mag > s / s == 0 errors
    float s_imm;         // per-layer API: scaler by value (slots == nullptr)
    uint64_t rng_base;   // per-layer API: ternarize rng_base (codec.hpp:148); plan: 0
    PeerPush dst;        // plan: code destinations (n == 0: just `push`)
    int32_t shard_n = 0;        // sharded exchange: ranks; chunk b belongs to rank r with
    uint32_t shard_bounds[kMaxPeers + 1];  // shard_bounds[r] <= b < shard_bounds[r + 1]
    unsigned long long* nnz = nullptr;     // telemetry: += nonzero codes (cluster.hpp:336-346)
    const OptDev* optd = nullptr;          // fused optimizer (kOpt kernels): per-block state
    OptArgs opt{};
    int32_t pdl = 0;  // launched as K1's programmatic dependent: 1 wait, 2/3 prefetch + wait
    uint32_t keep_from = ~0u;  // work items K1 kept in L2 (evict_last): demoted after reading
    // overlapped exchange: the launch covers n_pieces pieces [piece_bounds[q],
    // piece_bounds[q+1]) of work items; the CTA finishing the last item of piece q
    // publishes this rank's barrier record {epoch, t} for slot q to every rank, so the
    // decode of piece q starts while K2 still computes the later pieces. Sharded: the
    // owner of item b is r with owner_bounds[q][r] <= b < owner_bounds[q][r+1].
    // split exchange (pulled_item): such items are stored only into this rank's own area
    uint32_t pull8 = 0;
    int32_t rank = 0;
    // scaler slots to the peers (attached REF plans): the CTA of a block's first chunk
    // stores the block's slots (its nblk slots, multi-bucket) into every other rank's
    // copy of this push area -- K1 no longer stores them from its finalize tail, where
    // the remote stores' latency ended the K1 grid (GoogLeNet N = 2: K1 18.8 vs 16.0 us
    // without peer stores)
    int32_t slot_push = 0;
    int32_t n_pieces = 0;
    uint32_t piece_bounds[kMaxPieces + 1];
    uint32_t owner_bounds[kMaxPieces][kMaxPeers + 1];
    uint32_t* piece_cnt = nullptr;        // per piece: items finished (self-resetting)
    uint64_t* flag_remote[kMaxPeers];     // this rank's slot-0, parity-0 record in rank p
    int32_t n_flags = 0;
    uint64_t epoch = 0;
};

__device__ __forceinline__ uint32_t piece_of(const K2Args& a, uint32_t b) {
    uint32_t q = 0;
    while (q + 1 < static_cast<uint32_t>(a.n_pieces) && b >= a.piece_bounds[q + 1]) ++q;
    return q;
}

// nonzero 2-bit codes of the staged chunk (pad codes are 00); one atomic per CTA
// stage[from, nbytes) plus `extra` already counted by this thread (from % 4 == 0)
__device__ __forceinline__ void count_nonzero(const uint8_t* stage, uint32_t from, uint32_t nbytes,
                                              unsigned long long* nnz, uint32_t extra) {
    __shared__ uint32_t cta_nnz;
    if (threadIdx.x == 0) cta_nnz = 0;
    __syncthreads();
    uint32_t c = extra;
    const uint32_t nw = nbytes >> 2;
    for (uint32_t i = (from >> 2) + threadIdx.x; i < nw; i += kThreads) {
        const uint32_t w = reinterpret_cast<const uint32_t*>(stage)[i];
        c += __popc((w | (w >> 1)) & 0x55555555u);
    }
    for (uint32_t i = max(nw << 2, from) + threadIdx.x; i < nbytes; i += kThreads) {
        const uint32_t w = stage[i];
        c += __popc((w | (w >> 1)) & 0x55u);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(&cta_nnz, c);
    __syncthreads();
    if (threadIdx.x == 0 && cta_nnz) atomicAdd(nnz, static_cast<unsigned long long>(cta_nnz));
}

__device__ __forceinline__ int shard_owner(const K2Args& a, uint32_t b) {
    int r = 0;
    if (a.n_pieces) {
        const uint32_t* ob = a.owner_bounds[piece_of(a, b)];
        while (r + 1 < a.shard_n && b >= ob[r + 1]) ++r;
        return r;
    }
    while (r + 1 < a.shard_n && b >= a.shard_bounds[r + 1]) ++r;
    return r;
}

// Chunk codes are staged in shared memory, then written with 16-byte stores to
// every destination: the rank's own push area and, with peers attached, the
// same offset of every peer's gathered buffer over NVLink (the allgather is
// fused into K2 and overlaps its Philox-bound compute).
constexpr uint32_t kStageBytes = kChunk12 / 4;

__device__ __forceinline__ void copy_out(const uint8_t* stage, uint8_t* dst, uint32_t nbytes) {
    const uint32_t tid = threadIdx.x;
    if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
        const uint32_t n16 = nbytes >> 4;
        const uint4* s4 = reinterpret_cast<const uint4*>(stage);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        for (uint32_t i = tid; i < n16; i += kThreads) d4[i] = s4[i];
        for (uint32_t i = (n16 << 4) + tid; i < nbytes; i += kThreads) dst[i] = stage[i];
    } else {
        for (uint32_t i = tid; i < nbytes; i += kThreads) dst[i] = stage[i];
    }
}

// The staged bytes to n_dst global destinations (local or peer memory) with the
// TMA engine: one thread issues a cp.async.bulk per destination for the 16-B
// multiple head, the CTA stores a ragged tail; full completion is awaited before
// the CTA retires (or reuses `stage`), so grid completion orders these writes
// before a later kernel (the step barrier). Waiting only for the TMA engine to
// have read the staged bytes (wait_group.read) measured no faster at N = 2 / 4
// (VGG-16 0.394 vs 0.39 ms), so the stricter form stays. Falls back to copy_out
// for misaligned destinations.
// Call with the staged bytes complete (after a CTA barrier).
template <class DstF>
__device__ __forceinline__ void bulk_copy_out(const uint8_t* stage, DstF dst, int n_dst,
                                              uint32_t nbytes) {
    const uint32_t head = nbytes & ~15u;
    bool aligned = head != 0 && (reinterpret_cast<uintptr_t>(stage) & 15u) == 0;
    for (int p = 0; p < n_dst; ++p) aligned &= ((reinterpret_cast<uintptr_t>(dst(p)) & 15u) == 0);
    if (!aligned) {
        for (int p = 0; p < n_dst; ++p) copy_out(stage, dst(p), nbytes);
        return;
    }
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
        for (int p = 0; p < n_dst; ++p)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst(p)),
                         "r"(sa), "r"(head)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    for (int p = 0; p < n_dst; ++p)
        for (uint32_t i = head + threadIdx.x; i < nbytes; i += kThreads) dst(p)[i] = stage[i];
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Passthrough block (codec.hpp:206-209, 221-224): the raw fp32 values go to
// the block's region of every destination; the finite check of encode_step
// (:204) runs here since K1 never sees these blocks. N == 1 (kFuse): the
// average is float((0.0 + x) / 1.0) (codec.hpp:271-276), i.e. x with -0 -> +0.
template <bool kFuse, bool kOpt = false>
__device__ __forceinline__ void k2_passthrough(const K2Args& a, const LayerDev& L,
                                               const ChunkDev& ch, uint32_t b) {
    const uint32_t tid = threadIdx.x;
    const uint32_t count = ch.count;
    const float* g = L.g + ch.begin;
    const uint64_t off = L.code_off + 4ull * ch.begin;  // 16-B aligned (begin % 16 == 0)
    int p0 = 0, nd = a.dst.n == 0 ? 1 : a.dst.n;  // sharded exchange: the chunk's owner only
    if (a.shard_n) {
        p0 = shard_owner(a, b);
        nd = 1;
    }
    auto dst = [&](int p) {
        return reinterpret_cast<float*>((a.dst.n == 0 ? a.push : a.dst.base[p0 + p]) + off);
    };
    float* out = L.out + ch.begin;
    uint32_t bad = 0xFFFFFFFFu;
    uint32_t done = 0;
    if (L.flags & kLayerVecIn) {
        const uint32_t n4 = count >> 2;
        const float4* g4 = reinterpret_cast<const float4*>(g);
        for (uint32_t i = tid; i < n4; i += kThreads) {
            const float4 v = __ldcs(g4 + i);
            for (int p = 0; p < nd; ++p) reinterpret_cast<float4*>(dst(p))[i] = v;
            const bool fin = isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
            if (!fin && bad == 0xFFFFFFFFu) bad = 4 * i;
            if (kFuse && kOpt) {
                const OptDev od = a.optd[ch.layer];
                const uint64_t e = ch.begin + 4ull * i;
                opt_apply4(a.opt, od.w + e, od.s1 ? od.s1 + e : nullptr, od.s2 ? od.s2 + e : nullptr,
                           make_float4(__fadd_rn(v.x, 0.0f), __fadd_rn(v.y, 0.0f),
                                       __fadd_rn(v.z, 0.0f), __fadd_rn(v.w, 0.0f)),
                           od.vec != 0, 4);
            } else if (kFuse) {
                const float4 o = make_float4(__fadd_rn(v.x, 0.0f), __fadd_rn(v.y, 0.0f),
                                             __fadd_rn(v.z, 0.0f), __fadd_rn(v.w, 0.0f));
                if (L.flags & kLayerVecOut) {
                    __stcs(reinterpret_cast<float4*>(out) + i, o);
                } else {
                    out[4 * i] = o.x;
                    out[4 * i + 1] = o.y;
                    out[4 * i + 2] = o.z;
                    out[4 * i + 3] = o.w;
                }
            }
        }
        done = n4 << 2;
    }
    for (uint32_t i = done + tid; i < count; i += kThreads) {
        const float v = g[i];
        for (int p = 0; p < nd; ++p) dst(p)[i] = v;
        if (!isfinite(v) && bad == 0xFFFFFFFFu) bad = i;
        if (kFuse && kOpt) {
            const OptDev od = a.optd[ch.layer];
            const uint64_t e = ch.begin + i;
            opt_apply4(a.opt, od.w + e, od.s1 ? od.s1 + e : nullptr, od.s2 ? od.s2 + e : nullptr,
                       make_float4(__fadd_rn(v, 0.0f), 0.f, 0.f, 0.f), false, 1);
        } else if (kFuse) {
            out[i] = __fadd_rn(v, 0.0f);
        }
    }
    if (bad != 0xFFFFFFFFu) {
        for (uint32_t i = bad; i < count && i < bad + 4; ++i)  // first non-finite of the float4
            if (!isfinite(g[i])) {
                bad = i;
                break;
            }
        raise_error(a.err, TGB_E_NONFINITE, static_cast<int32_t>(L.tensor),
                    block_rng_base(L) + ch.begin + bad);
    }
}

// destinations of chunk b's codes: [p0, p1) of a.dst (a.push when a.dst.n == 0)
// split exchange: code items of 32K-element granule (block, begin >> 15) with
// (block + granule) % 8 < pull8 are pulled by the decode over NVLink instead of pushed
// by K2. K2 items and K3 items are power-of-two aligned inside a block, both <= 32K
// elements, so both kernels classify every element alike.
__device__ __forceinline__ bool pulled_item(uint32_t pull8, const ChunkDev& ch,
                                            const LayerDev& L) {
    return pull8 && !(L.flags & (kLayerPassthrough | kLayerMultiBucket)) &&
           ((ch.layer + (ch.begin >> 15)) & 7u) < pull8;
}

__device__ __forceinline__ void k2_dst_range(const K2Args& a, uint32_t b, const ChunkDev& ch,
                                             const LayerDev& L, int& p0, int& p1) {
    p0 = 0;
    p1 = a.dst.n == 0 ? 1 : a.dst.n;
    if (a.dst.n && a.shard_n) p1 = (p0 = shard_owner(a, b)) + 1;  // sharded: owner only
    // a pulled item stays in this rank's own area; the peers' K3 reads it from there
    if (a.dst.n && pulled_item(a.pull8, ch, L)) p1 = (p0 = a.rank) + 1;
}
__device__ __forceinline__ uint8_t* k2_dst(const K2Args& a, int p) {
    return a.dst.n == 0 ? a.push : a.dst.base[p];
}

// K1 loaded the last units of its launch with an L2 evict_last policy so that
// K2's reverse walk re-reads them from L2; once read here they are demoted back
// to evict_normal, so no gradient line stays pinned in L2 after the step.
__device__ __forceinline__ void demote_l2(const float* g, uint32_t count) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(g) & ~static_cast<uintptr_t>(127);
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(g + count);
    for (uintptr_t a = a0 + 128u * threadIdx.x; a < a1; a += 128u * kThreads)
        asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(a) : "memory");
}

// Overlapped exchange: work item b is done (its codes stored at every destination;
// the bulk copies completed before thread 0 got here). The CTA counts itself into
// its piece; the CTA completing the piece publishes this rank's record {epoch, t}
// of barrier slot q to every rank. Ordering: every thread's stores -> bar.sync ->
// thread 0 orders the async-proxy (TMA) writes before its generic operations
// (fence.proxy.async) and releases at GPU scope before the counter increment; the
// last CTA acquires all increments, then one fence.acq_rel.sys (cumulative over
// what it observed) precedes the system-scope release of the records -- one
// system fence per piece instead of one per work item.
__device__ __forceinline__ void piece_done(const K2Args& a, uint32_t b) {
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t q = piece_of(a, b);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const uint32_t done = atomicAdd(a.piece_cnt + q, 1u) + 1u;
    if (done != a.piece_bounds[q + 1] - a.piece_bounds[q]) return;
    a.piece_cnt[q] = 0u;  // every item of the piece has counted: reset for the next step
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const uint32_t par = static_cast<uint32_t>(a.epoch & 1u) * kMaxPeers;
    for (int p = 0; p < a.n_flags; ++p) {
        uint64_t* r = a.flag_remote[p] + 2 * ((2 * q) * kMaxPeers + par);
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(r + 1), "l"(a.t) : "memory");
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(r), "l"(a.epoch) : "memory");
    }
}

// Multi-bucket K2 item: ch.nblk whole buckets of k = 2^p elements (k/4 code bytes
// each, contiguous). Each bucket has its own scaler: the per-bucket decision
// constants (Decider) are computed once per item into shared memory and code
// byte q uses bucket q >> (p - 2). Philox counters are the tensor's element
// indices (ternarize's rng_base = the bucket offset, codec.hpp:167, :229), so
// the whole item is one lane-aligned counter range. s == 0 buckets emit 00
// codes (codec.hpp:155-159). kFuse / kOpt as k2_code_chunk.
template <int U, bool kFuse, bool kOpt>
__device__ __forceinline__ uint32_t k2_code_chunk_mb(const K2Args& a, const LayerDev& L,
                                                     const ChunkDev& ch, uint8_t* __restrict__ stage) {
    __shared__ float4 dp[kMaxItemBuckets];       // per bucket: s, ib, rl, dr
    __shared__ uint8_t dmode[kMaxItemBuckets];   // 0 fast+exact, 1 exact only, 2 s == 0
    const uint32_t tid = threadIdx.x;
    const float bound = a.bounds ? __ldcg(a.bounds + ch.layer) : INFINITY;
    for (uint32_t j = tid; j < ch.nblk; j += kThreads) {
        const float s = __ldcg(a.slots + L.slot + j);
        Decider d;
        d.init(bound, s);
        dp[j] = make_float4(s, d.ib, d.rl, d.dr);
        dmode[j] = s == 0.0f ? 2 : (d.exact_all ? 1 : 0);
    }
    __syncthreads();
    const uint32_t count = ch.count;
    const uint32_t nbytes = (count + 3) >> 2;
    const uint32_t nfull = count >> 2;
    const uint32_t shq = bucket_log2(L) - 2;  // code byte -> bucket
    const float* g = L.g;
    const uint64_t qg = block_rng_base(L) >> 2;  // k % 4 == 0: lane aligned
    Philox4<false> ph;
    ph.init(L.key0, L.key1, static_cast<uint32_t>(qg >> 32), a.t);
    const uint32_t qbase = static_cast<uint32_t>(qg);
    float* out = L.out;
    const bool vec_in = (L.flags & kLayerVecIn) != 0, vec_out = (L.flags & kLayerVecOut) != 0;
    OptDev od{};
    if (kOpt) od = a.optd[ch.layer];
    auto byte_of = [&](float4 v, uint4 r, uint32_t q) -> uint32_t {
        const uint32_t j = q >> shq;
        const uint32_t mode = dmode[j];
        if (mode == 2) return 0u;
        const float4 c = dp[j];
        Decider d;
        d.bound = bound;
        d.s = c.x;
        d.ib = c.y;
        d.rl = c.z;
        d.dr = c.w;
        d.exact_all = mode != 0;
        return d.byte(v, r);
    };
    auto emit = [&](uint32_t q, uint32_t byte) {  // (s * float(code)) * 1 per element
        if (!kFuse) return;
        const float s = dp[q >> shq].x;
        auto val = [&](uint32_t c) {
            return __fmul_rn(__fmul_rn(s, c == 1u ? 1.0f : (c == 2u ? -1.0f : 0.0f)), 1.0f);
        };
        const float4 o = make_float4(val(byte & 3u), val((byte >> 2) & 3u), val((byte >> 4) & 3u),
                                     val(byte >> 6));
        const uint32_t e = 4 * q;
        if (kOpt) {
            opt_apply4(a.opt, od.w + e, od.s1 ? od.s1 + e : nullptr, od.s2 ? od.s2 + e : nullptr, o,
                       od.vec != 0, count - e < 4 ? count - e : 4);
        } else if (vec_out && e + 4 <= count) {
            __stcs(reinterpret_cast<float4*>(out) + q, o);
        } else {
            if (e < count) out[e] = o.x;
            if (e + 1 < count) out[e + 1] = o.y;
            if (e + 2 < count) out[e + 2] = o.z;
            if (e + 3 < count) out[e + 3] = o.w;
        }
    };
    auto load4 = [&](uint32_t q) {
        if (vec_in && 4 * q + 4 <= count) return __ldcs(reinterpret_cast<const float4*>(g) + q);
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = 4 * q + e < count ? g[4 * q + e] : 0.0f;
        return make_float4(x[0], x[1], x[2], x[3]);
    };
    uint32_t q = tid;
    for (uint32_t blk = 0; blk + U * kThreads <= nfull; blk += U * kThreads, q += U * kThreads) {
        float4 v[U];
        uint32_t ctr[U];
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = load4(q + u * kThreads);
#pragma unroll
        for (int u = 0; u < U; ++u) ctr[u] = qbase + q + u * kThreads;
        ph(ctr, r);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t byte = byte_of(v[u], r[u], q + u * kThreads);
            stage[q + u * kThreads] = static_cast<uint8_t>(byte);
            emit(q + u * kThreads, byte);
        }
    }
    for (; q < nbytes; q += kThreads) {  // tail (and the tensor's ragged last byte)
        const float4 v = load4(q);
        uint32_t ctr[1] = {qbase + q};
        uint4 r[1];
        ph(ctr, r);
        const uint32_t byte = byte_of(v, r[0], q);
        stage[q] = static_cast<uint8_t>(byte);
        emit(q, byte);
    }
    __syncthreads();
    if (a.nnz) count_nonzero(stage, 0, nbytes, a.nnz, 0);
    return nbytes;
}

// Codes of one chunk (work item b) into `stage`; returns the number of staged
// code bytes (passthrough chunks are copied to their destinations here and
// return 0). kFuse (N == 1: the average is this worker's own decode, K3 folded
// into K2): every thread writes the decoded float4 of each code byte as soon as
// it is computed, so the output stream overlaps the Philox compute. kOpt: the
// decoded value drives OptimizerState::apply instead of being written. Ends
// with a CTA barrier (stage complete).
template <int U, bool kFuse, bool kOpt = false>
__device__ __forceinline__ uint32_t k2_code_chunk(const K2Args& a, const LayerDev& L,
                                                  const ChunkDev& ch, uint32_t b,
                                                  uint8_t* __restrict__ stage, float4* lutv) {
    if (L.flags & kLayerPassthrough) {
        k2_passthrough<kFuse, kOpt>(a, L, ch, b);
        return 0;
    }
    if (ch.nblk > 1) return k2_code_chunk_mb<U, kFuse, kOpt>(a, L, ch, stage);
    // L2 loads: in the fused K1+K2 kernel another CTA wrote them during this launch
    const float s = a.slots ? __ldcg(a.slots + L.slot) : a.s_imm;
    const float bound = a.bounds ? __ldcg(a.bounds + ch.layer) : INFINITY;
    const uint32_t count = ch.count;
    const uint32_t nbytes = (count + 3) >> 2;
    const float* g = L.g + ch.begin;
    const uint32_t tid = threadIdx.x;

    Decider dec;
    dec.init(bound, s);
    // stream index of the chunk's first element (codec.hpp:167): element j of
    // the chunk draws lane (B + j) & 3 of Philox block (B + j) >> 2
    const uint64_t B = a.rng_base + block_rng_base(L) + ch.begin;
    const uint64_t qg = B >> 2;
    // fast paths: one Philox block per code byte, 32-bit counter arithmetic
    const bool lane_aligned = (B & 3u) == 0 && static_cast<uint32_t>(qg) <= 0xFFFFFFFFu - nbytes;
    Philox4<false> ph;
    ph.init(L.key0, L.key1, static_cast<uint32_t>(qg >> 32), a.t);
    const uint32_t qbase = static_cast<uint32_t>(qg);

    const uint32_t nfull = count >> 2;  // bytes whose 4 elements all exist
    // kFuse: byte -> float4 table of (s*float(sum))*invN with invN = 1, sum in
    // {0, +1, -1} (codec.hpp:296, wire.hpp:220): +0, s, -s
    if (kFuse) {
        const float v0 = __fmul_rn(__fmul_rn(s, 0.0f), 1.0f), v1 = __fmul_rn(__fmul_rn(s, 1.0f), 1.0f),
                    v2 = __fmul_rn(__fmul_rn(s, -1.0f), 1.0f);
        auto val = [&](uint32_t c) { return c == 1u ? v1 : (c == 2u ? v2 : v0); };
        lutv[tid] = make_float4(val(tid & 3u), val((tid >> 2) & 3u), val((tid >> 4) & 3u),
                                val((tid >> 6) & 3u));
        __syncthreads();
    }
    float* out = L.out + ch.begin;
    const bool vec_out = (L.flags & kLayerVecOut) != 0;
    OptDev od{};
    if (kOpt) od = a.optd[ch.layer];
    auto emit = [&](uint32_t qq, uint32_t byte) {  // kFuse: decoded float4 of byte qq
        if (!kFuse) return;
        const float4 o = lutv[byte];
        if (kOpt) {  // fused optimizer: the averaged gradient drives the update directly
            const uint64_t e = ch.begin + 4ull * qq;
            const uint32_t nv = count - 4 * qq < 4 ? count - 4 * qq : 4;
            opt_apply4(a.opt, od.w + e, od.s1 ? od.s1 + e : nullptr, od.s2 ? od.s2 + e : nullptr, o,
                       od.vec != 0, nv);
            return;
        }
        if (vec_out && 4 * qq + 4 <= count) {
            __stcs(reinterpret_cast<float4*>(out) + qq, o);
        } else {
            const uint32_t e = 4 * qq;
            if (e < count) out[e] = o.x;
            if (e + 1 < count) out[e + 1] = o.y;
            if (e + 2 < count) out[e + 2] = o.z;
            if (e + 3 < count) out[e + 3] = o.w;
        }
    };
    uint32_t q = tid;
    float bad_mag = 0.0f;  // max clipped |x| seen (per-layer API check: mag > s)
    if (s == 0.0f) {  // codec.hpp:155-159: all codes 0
        for (; q < nbytes; q += kThreads) {
            stage[q] = 0;
            emit(q, 0);
        }
        if (a.check)
            for (uint32_t i = tid; i < count; i += kThreads)
                if (g[i] != 0.0f)
                    raise_error(a.err, TGB_E_S0_NONZERO, static_cast<int32_t>(L.tensor),
                                block_rng_base(L) + ch.begin + i);
    } else if (!lane_aligned) {
        // block offset not a multiple of 4 (FixedSize with k % 4 != 0) or an
        // unaligned per-layer rng_base: byte q's elements straddle Philox blocks
        // qg+q and qg+q+1. Each lane computes block qg+q and takes the next one
        // from its neighbour (lane 31 computes it); full 64-bit counters.
        const uint32_t sh = static_cast<uint32_t>(B & 3u);
        const uint32_t lane = tid & 31u;
        const uint32_t t_lo = static_cast<uint32_t>(a.t), t_hi = static_cast<uint32_t>(a.t >> 32);
        for (uint32_t qw = tid - lane; qw < nbytes; qw += kThreads) {
            const uint32_t qq = qw + lane;
            const uint64_t c = qg + qq;
            const uint4 r = philox10(
                make_uint4(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32), t_lo, t_hi),
                L.key0, L.key1);
            uint4 rn;
            rn.x = __shfl_down_sync(0xffffffffu, r.x, 1);
            rn.y = __shfl_down_sync(0xffffffffu, r.y, 1);
            rn.z = __shfl_down_sync(0xffffffffu, r.z, 1);
            if (lane == 31u) {
                const uint64_t c1 = c + 1;
                rn = philox10(make_uint4(static_cast<uint32_t>(c1), static_cast<uint32_t>(c1 >> 32),
                                         t_lo, t_hi),
                              L.key0, L.key1);
            }
            if (qq < nbytes) {
                uint32_t byte = 0;
#pragma unroll
                for (uint32_t e = 0; e < 4; ++e) {
                    const uint32_t i = 4 * qq + e;
                    if (i >= count) break;
                    const uint32_t j = sh + e;  // <= 6
                    const uint32_t bits = j == 0 ? r.x : j == 1 ? r.y : j == 2 ? r.z : j == 3 ? r.w
                                        : j == 4 ? rn.x : j == 5 ? rn.y : rn.z;
                    const float x = g[i];
                    byte |= dec.code(x, bits) << (2 * e);
                    if (a.check) bad_mag = fmaxf(bad_mag, fabsf(x));
                }
                stage[qq] = static_cast<uint8_t>(byte);
                emit(qq, byte);
            }
        }
        q = nbytes;
    } else if (L.flags & kLayerVecIn) {
        const float4* g4 = reinterpret_cast<const float4*>(g);
        // uniform trip count (every thread runs every block: __syncthreads below)
        for (uint32_t blk = 0; blk + U * kThreads <= nfull; blk += U * kThreads, q += U * kThreads) {
            float4 v[U];
            uint32_t ctr[U];
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcs(g4 + q + u * kThreads);
#pragma unroll
            for (int u = 0; u < U; ++u) ctr[u] = qbase + q + u * kThreads;
            ph(ctr, r);
            uint32_t byte[U];
            float amb = -1.0f;
#pragma unroll
            for (int u = 0; u < U; ++u) byte[u] = dec.byte_fast(v[u], r[u], amb);
            if (amb >= 0.0f || dec.exact_all) {  // rare: redo these bytes exactly
#pragma unroll
                for (int u = 0; u < U; ++u) byte[u] = dec.byte_exact(v[u], r[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                stage[q + u * kThreads] = static_cast<uint8_t>(byte[u]);
                emit(q + u * kThreads, byte[u]);
                if (a.check)
                    bad_mag = fmaxf(bad_mag, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)),
                                                   fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
            }
        }
        for (; q < nfull; q += kThreads) {
            const float4 v = __ldcs(g4 + q);
            uint32_t ctr[1] = {qbase + q};
            uint4 r[1];
            ph(ctr, r);
            const uint32_t byte = dec.byte(v, r[0]);
            stage[q] = static_cast<uint8_t>(byte);
            emit(q, byte);
            if (a.check)
                bad_mag = fmaxf(bad_mag, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)),
                                               fmaxf(fabsf(v.z), fabsf(v.w))));
        }
    }
    // scalar path: unaligned input and the partial last byte (pad bits stay 00)
    if (s != 0.0f) {
        for (; q < nbytes; q += kThreads) {
            float x[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t i = 4 * q + e;
                x[e] = i < count ? g[i] : 0.0f;
            }
            uint32_t ctr[1] = {qbase + q};
            uint4 r[1];
            ph(ctr, r);
            const uint32_t byte = dec.byte(make_float4(x[0], x[1], x[2], x[3]), r[0]);
            stage[q] = static_cast<uint8_t>(byte);
            emit(q, byte);
            if (a.check)
                bad_mag = fmaxf(bad_mag, fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])),
                                               fmaxf(fabsf(x[2]), fabsf(x[3]))));
        }
    }
    if (a.check && fminf(bad_mag, bound) > s)  // codec.hpp:163-165
        raise_error(a.err, TGB_E_SCALER_BELOW_MAX, static_cast<int32_t>(L.tensor),
                    block_rng_base(L) + ch.begin);
#ifndef TGB_AB_NO_DEMOTE  // (same-box A/B builds only, tools/build_variant.sh)
    if (b >= a.keep_from) demote_l2(g, count);
#endif
    __syncthreads();
    if (a.nnz) count_nonzero(stage, 0, nbytes, a.nnz, 0);
    return nbytes;
}

// K2: one CTA per work item. The chunk's codes are staged in shared memory and
// handed to the TMA engine (bulk_copy_out): the rank's own push area and, with
// peers attached, the same offset of every peer's gather buffer over NVLink
// (the allgather is fused into K2 and overlaps its Philox-bound compute), or
// only the chunk owner's (sharded exchange).
template <class Src, int kMinBlocks = 3, bool kFuse = false, bool kOpt = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k2_ternarize(Src src, K2Args a) {
    __shared__ __align__(16) uint8_t stage[kStageBytes];
    __shared__ float4 lutv[kFuse ? 256 : 1];
    const uint32_t b = a.reverse ? (gridDim.x - 1 - blockIdx.x) : blockIdx.x;
    ChunkDev ch;
    LayerDev L;
    src.get(b, ch, L);
    if (a.pdl) {  // resident while K1 drains; nothing K1 writes is read before the wait
        if (a.pdl >= 2 && threadIdx.x == 0 && (L.flags & kLayerVecIn)) {
            // warm L2 with the chunk's gradient (3: only its first 32 KB)
            const uint32_t bytes = min((ch.count * 4u) & ~15u, a.pdl == 3 ? 32768u : ~0u);
            if (bytes)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(L.g + ch.begin),
                             "r"(bytes)
                             : "memory");
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (a.slot_push && ch.begin == 0 && L.slot >= 0)
        for (uint32_t j = threadIdx.x; j < ch.nblk; j += kThreads) {
            const float v = a.slots[L.slot + j];
            for (int p = 0; p < a.dst.n; ++p)
                if (p != a.rank) reinterpret_cast<float*>(a.dst.base[p])[L.slot + j] = v;
        }
    const uint32_t nbytes = k2_code_chunk<4, kFuse, kOpt>(a, L, ch, b, stage, lutv);
    // Without pieces no fence follows the peer stores: the step barrier kernel runs
    // after this grid completes in stream order, and grid completion implies its
    // (peer) stores are performed -- the guarantee event-based multi-GPU sync relies on.
    if (nbytes) {
        const uint64_t off = L.code_off + (ch.begin >> 2);
        int p0, p1;
        k2_dst_range(a, b, ch, L, p0, p1);
        bulk_copy_out(stage, [&](int p) { return k2_dst(a, p0 + p) + off; }, p1 - p0, nbytes);
    }
    if (a.n_pieces) piece_done(a, b);
}

// Fused K1 + K2 for small gradient sets (one launch per step; the K1 -> K2
// kernel boundary would cost more than the work): persistent CTAs, all
// co-resident (grid <= occupancy x SMs). Phase 1: the K1 units (clip statistics,
// partials, per-tensor finalize by the last arriving unit, which publishes the
// tensor's bound + scalers with a release store of the launch epoch). Phase 2:
// the K2 units; a unit of tensor T first waits (acquire) for T's flag, so K2 of
// early tensors overlaps K1 of later ones. Phase 1 never waits, so every flag a
// phase-2 CTA waits for is set by a CTA that is already running: deadlock-free.
// Global bucketing waits for the global flag (all tensors finalized). The last
// CTA to finish clears the flags (every other CTA is past its waits), so each
// launch starts from zero flags: the kernel is safe to replay in a CUDA graph.
__device__ __forceinline__ void wait_ready(const uint32_t* flag, uint32_t epoch, ErrWord* err) {
    if (threadIdx.x == 0) {
        uint32_t v;
        const long long t0 = clock64();
        for (uint32_t spin = 0;; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if (v != 0u) break;
            if (spin > 16) __nanosleep(64);
            if ((spin & 1023) == 1023 && clock64() - t0 > 20000000000ll) {  // ~10 s: a bug
                raise_error(err, TGB_E_PEER_TIMEOUT, -1, ~0ull);
                break;
            }
        }
    }
    __syncthreads();
}

template <bool kFuse, bool kOpt = false>
__global__ void __launch_bounds__(kThreads, 4) k12_fused(TableSource src, K1Out o, K2Args a,
                                                        uint32_t n_k1, uint32_t n_k2,
                                                        uint32_t n_flags) {
    __shared__ __align__(16) uint8_t stage[kStageBytes];
    __shared__ float4 lutv[kFuse ? 256 : 1];
    for (uint32_t u = blockIdx.x; u < n_k1; u += gridDim.x) {
        ChunkDev ch;
        LayerDev L;
        src.get(u, ch, L);
        k1_unit<8, 1, false>(o, ch, L, u, [&](ChunkDev& c, LayerDev& l) { src.get(u, c, l); });
        __syncthreads();  // the finalize's shared memory is reused by the next unit
    }
    for (uint32_t b = blockIdx.x; b < n_k2; b += gridDim.x) {
        ChunkDev ch;
        LayerDev L;
        src.get(b, ch, L);
        if (!(L.flags & kLayerPassthrough))
            wait_ready(o.global_bucketing ? o.ready_global : o.ready + L.tensor, o.epoch, a.err);
        const uint32_t nbytes = k2_code_chunk<4, kFuse, kOpt>(a, L, ch, b, stage, lutv);
        if (nbytes) {
            const uint64_t off = L.code_off + (ch.begin >> 2);
            int p0, p1;
            k2_dst_range(a, b, ch, L, p0, p1);
            bulk_copy_out(stage, [&](int p) { return k2_dst(a, p0 + p) + off; }, p1 - p0, nbytes);
        }
        __syncthreads();  // the bulk copy finished reading `stage` (thread 0 waited for it)
    }
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(o.ready + n_flags, 1u) == gridDim.x - 1;  // exit counter
    }
    __syncthreads();
    if (last) {
        for (uint32_t i = threadIdx.x; i < n_flags; i += kThreads) o.ready[i] = 0u;
        if (threadIdx.x == 0) o.ready[n_flags] = 0u;
    }
}

// ====================================================================== K3
// code byte -> 4 lanes of (1 + v) in {0,1,2}; summed over N workers lane e holds
// N + sum_w v_w, the LUT index. 11 codes map to 0 and are flagged separately.
__device__ __forceinline__ uint32_t lane_biased(uint32_t b) {
    uint32_t r = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t c = (b >> (2 * e)) & 3u;
        const uint32_t v = c == 1u ? 2u : (c == 0u ? 1u : 0u);
        r |= v << (8 * e);
    }
    return r;
}

// SWAR form of lane_biased(b): the four 2-bit codes spread to bytes, then
// 1 + (c & 1) - (c >> 1) per byte (8 integer ops instead of a table load)
__device__ __forceinline__ uint32_t lane_biased_swar(uint32_t b) {
    uint32_t x = (b | (b << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    return 0x01010101u + (x & 0x01010101u) - ((x >> 1) & 0x01010101u);
}

// exact float(k) for |k| < 2^22 without I2F: 1.5*2^23 + k, then subtract
__device__ __forceinline__ float small_int_float(int k) {
    return __fsub_rn(__int_as_float(0x4B400000 + k), 12582912.0f);
}

// Passthrough block average (codec.hpp:269-279): per element an fp64 sum
// from 0.0 over workers in order, divided by N in fp64, rounded to fp32.
// base(w) = worker w's raw values of this chunk.
template <class Base>
__device__ __forceinline__ void k3_passthrough(Base base, int N, float* out, uint32_t count,
                                               bool vec) {
    const uint32_t tid = threadIdx.x;
    const double dn = static_cast<double>(N);
    const uint32_t n4 = vec ? (count >> 2) : 0u;
    for (uint32_t i = tid; i < n4; i += kThreads) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        for (int w = 0; w < N; ++w) {
            const float4 v = __ldcs(reinterpret_cast<const float4*>(base(w)) + i);
            s0 = __dadd_rn(s0, static_cast<double>(v.x));
            s1 = __dadd_rn(s1, static_cast<double>(v.y));
            s2 = __dadd_rn(s2, static_cast<double>(v.z));
            s3 = __dadd_rn(s3, static_cast<double>(v.w));
        }
        __stcs(reinterpret_cast<float4*>(out) + i,
               make_float4(static_cast<float>(s0 / dn), static_cast<float>(s1 / dn),
                           static_cast<float>(s2 / dn), static_cast<float>(s3 / dn)));
    }
    for (uint32_t i = 4 * n4 + tid; i < count; i += kThreads) {
        double sum = 0.0;
        for (int w = 0; w < N; ++w) sum = __dadd_rn(sum, static_cast<double>(base(w)[i]));
        out[i] = static_cast<float>(sum / dn);
    }
}

struct K3Args {
    const uint8_t* src;     // worker w's push buffer at src + w*stride (table source)
    uint64_t stride;
    const uint8_t* const* code_ptrs;  // per-layer API: per-worker code base (host array copied)
    const float* scalers;   // per-layer API: N scalers (device), or nullptr => s_imm
    float s_imm;
    int32_t n_workers;
    int32_t sharing;
    float inv_n;            // 1.0f / float(N), rounded on the host (codec.hpp:267)
    ErrWord* err;
    const OptDev* optd = nullptr;  // fused decode -> optimizer (kOpt kernels)
    OptArgs opt{};
    int32_t gate = 0;              // plan exchange: skip when the step's exchange failed
    // split exchange (staged kernel): the codes of worker w are read from wsrc[w] (its own
    // push area in its own memory, over NVLink) instead of the local gather buffer
    uint32_t pull8 = 0;
    const uint8_t* wsrc[kMaxPeers];
};

struct K3Ptrs {  // per-layer API: explicit pointers (passed by value)
    const uint8_t* codes[kMaxWorkers];
};

template <class Src, bool kTable, bool kShared>
__global__ void __launch_bounds__(kThreads) k3_decode(Src src, K3Args a, K3Ptrs ptrs) {
    if (a.gate && exchange_failed(a.err)) return;
    ChunkDev ch;
    LayerDev L;
    src.get(blockIdx.x, ch, L);
    if (kTable && (L.flags & kLayerPassthrough)) {
        const uint64_t off = L.code_off + 4ull * ch.begin;
        k3_passthrough([&](int w) { return reinterpret_cast<const float*>(a.src + a.stride * w + off); },
                       a.n_workers, L.out + ch.begin, ch.count, (L.flags & kLayerVecOut) != 0);
        return;
    }
    const int N = a.n_workers;
    __shared__ uint32_t tab[256];
    __shared__ float lut[2 * kMaxWorkers + 1];
    __shared__ float sw[kMaxWorkers];
    const uint32_t tid = threadIdx.x;
    tab[tid] = lane_biased(tid);
    if (tid < static_cast<uint32_t>(N)) {
        sw[tid] = kTable ? __ldg(reinterpret_cast<const float*>(a.src + a.stride * tid) + L.slot)
                         : (a.scalers ? __ldg(a.scalers + tid) : a.s_imm);
    }
    __syncthreads();
    if (a.sharing && tid <= static_cast<uint32_t>(2 * N)) {
        float s = 0.0f;  // cluster.hpp:195-196 / codec.hpp:289-291
        for (int w = 0; w < N; ++w) s = fmaxf(s, sw[w]);
        const float sum = static_cast<float>(static_cast<int>(tid) - N);
        lut[tid] = __fmul_rn(__fmul_rn(s, sum), a.inv_n);  // codec.hpp:296
    }
    __syncthreads();

    const uint32_t count = ch.count;
    const uint32_t nbytes = (count + 3) >> 2;
    const uint64_t q0 = ch.begin >> 2;
    float* out = L.out + ch.begin;
    const bool vec_out = (L.flags & kLayerVecOut) != 0;
    // U code bytes per thread per iteration, every worker's loads issued before
    // any use: the gathered codes usually come from HBM (allgather landing
    // buffer), so memory-level parallelism decides this kernel's speed.
    constexpr int U = 4;
    for (uint32_t qb = 0; qb < nbytes; qb += U * kThreads) {
        uint32_t acc[U], bad = 0;
        double sm[kShared ? 1 : U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc[u] = 0;
            if (!kShared) {
#pragma unroll
                for (int e = 0; e < 4; ++e) sm[kShared ? 0 : u][e] = 0.0;
            }
        }
        for (int w = 0; w < N; ++w) {
            const uint8_t* base = kTable ? a.src + a.stride * w + L.code_off + q0 : ptrs.codes[w] + q0;
            uint32_t bw[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t q = qb + tid + u * kThreads;
                bw[u] = q < nbytes ? __ldcs(base + q) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                bad |= bw[u] & (bw[u] >> 1) & 0x55u;
                if (kShared) {
                    acc[u] += tab[bw[u]];
                } else {  // codec.hpp:299-306: fp64 worker-order sum, then /N
                    const double sd = static_cast<double>(sw[w]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t c = (bw[u] >> (2 * e)) & 3u;
                        const double v = c == 1u ? 1.0 : (c == 2u ? -1.0 : 0.0);
                        sm[kShared ? 0 : u][e] = __dadd_rn(sm[kShared ? 0 : u][e], __dmul_rn(sd, v));
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t q = qb + tid + u * kThreads;
            if (q >= nbytes) continue;
            float4 o;
            if (kShared) {
                o = make_float4(lut[acc[u] & 0xffu], lut[(acc[u] >> 8) & 0xffu],
                                lut[(acc[u] >> 16) & 0xffu], lut[acc[u] >> 24]);
            } else {
                const double dn = static_cast<double>(N);
                const int v = kShared ? 0 : u;
                o = make_float4(static_cast<float>(sm[v][0] / dn), static_cast<float>(sm[v][1] / dn),
                                static_cast<float>(sm[v][2] / dn), static_cast<float>(sm[v][3] / dn));
            }
            const uint32_t b4 = 4 * q;
            if (vec_out && b4 + 4 <= count) {
                __stcs(reinterpret_cast<float4*>(out + b4), o);
            } else {
                if (b4 + 0 < count) out[b4 + 0] = o.x;
                if (b4 + 1 < count) out[b4 + 1] = o.y;
                if (b4 + 2 < count) out[b4 + 2] = o.z;
                if (b4 + 3 < count) out[b4 + 3] = o.w;
            }
        }
        if (bad) {
            // locate the first corrupt element of this thread (pad bits are 00 by construction)
            for (int u = 0; u < U; ++u) {
                const uint32_t q = qb + tid + u * kThreads;
                if (q >= nbytes) break;
                for (int w = 0; w < N; ++w) {
                    const uint8_t* base =
                        kTable ? a.src + a.stride * w + L.code_off + q0 : ptrs.codes[w] + q0;
                    const uint32_t b = base[q] & (base[q] >> 1) & 0x55u;
                    if (b) {
                        raise_error(a.err, TGB_E_CORRUPT_CODE, static_cast<int32_t>(L.tensor),
                                    block_rng_base(L) + ch.begin + 4ull * q + ((__ffs(b) - 1) >> 1));
                        break;
                    }
                }
            }
        }
    }
}

// Plan K3, shared scalers, N <= 8 (one NVSwitch box): the chunk's code bytes of
// all NW workers are first staged in shared memory with 16-byte loads (NW
// independent uint4 per thread in flight, 16x fewer load instructions than byte
// loads), then decoded from shared memory: per code byte the NW bytes are
// summed as SWAR lanes (biased sums N + sum_w code_w) and every lane decodes to
// (s * float(sum)) * invN with s = max over workers (codec.hpp:289-296,
// cluster.hpp:195-196) computed in registers (no table lookups).
template <int NW, bool kOpt = false>
__global__ void __launch_bounds__(kThreads) k3_decode_staged(TableSource src, K3Args a) {
    if (a.gate && exchange_failed(a.err)) return;  // skewed / missing peer: keep the outputs
    ChunkDev ch;
    LayerDev L;
    src.get(blockIdx.x, ch, L);
    if (L.flags & kLayerPassthrough) {
        const uint64_t off = L.code_off + 4ull * ch.begin;
        if (kOpt) {  // fp64 worker-order mean (codec.hpp:269-279) drives the update
            const OptDev od = a.optd[ch.layer];
            for (uint32_t i = threadIdx.x; i < ch.count; i += kThreads) {
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    sum = __dadd_rn(sum, static_cast<double>(reinterpret_cast<const float*>(
                                             a.src + a.stride * w + off)[i]));
                const uint64_t e = ch.begin + i;
                opt_apply4(a.opt, od.w + e, od.s1 ? od.s1 + e : nullptr,
                           od.s2 ? od.s2 + e : nullptr,
                           make_float4(static_cast<float>(sum / static_cast<double>(NW)), 0.f, 0.f,
                                       0.f),
                           false, 1);
            }
            return;
        }
        k3_passthrough([&](int w) { return reinterpret_cast<const float*>(a.src + a.stride * w + off); },
                       NW, L.out + ch.begin, ch.count, (L.flags & kLayerVecOut) != 0);
        return;
    }
    constexpr uint32_t kStage = kChunk3 / 4;  // code bytes per worker
    __shared__ __align__(16) uint8_t codes[NW][kStage];
    __shared__ float sw[NW];
    const uint32_t tid = threadIdx.x;
    const uint32_t count = ch.count;
    const uint32_t nbytes = (count + 3) >> 2;
    const uint32_t n16 = nbytes >> 4;
    const bool pull = pulled_item(a.pull8, ch, L);
    {
        uint4 v[NW][kStage / 16 / kThreads > 0 ? kStage / 16 / kThreads : 1];
        constexpr int R = kStage / 16 / kThreads > 0 ? kStage / 16 / kThreads : 1;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint4* b4 = reinterpret_cast<const uint4*>(
                (pull ? a.wsrc[w] : a.src + a.stride * w) + L.code_off + (ch.begin >> 2));
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t i = tid + r * kThreads;
                v[w][r] = i < n16 ? __ldcs(b4 + i) : make_uint4(0, 0, 0, 0);
            }
        }
        if (tid < NW) sw[tid] = __ldg(reinterpret_cast<const float*>(a.src + a.stride * tid) + L.slot);
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t i = tid + r * kThreads;
                if (i < n16) reinterpret_cast<uint4*>(codes[w])[i] = v[w][r];
            }
        for (uint32_t i = (n16 << 4) + tid; i < nbytes; i += kThreads)
#pragma unroll
            for (int w = 0; w < NW; ++w)
                codes[w][i] = (pull ? a.wsrc[w] : a.src + a.stride * w)[L.code_off +
                                                                        (ch.begin >> 2) + i];
    }
    // multi-bucket item: s = max over workers per bucket (bucket of byte q: q >> shq)
    __shared__ float smax_b[kChunk3 / 64];
    const bool mb = ch.nblk > 1;
    const uint32_t shq = mb ? bucket_log2(L) - 2 : 31u;
    if (mb)
        for (uint32_t j = tid; j < ch.nblk; j += kThreads) {
            float m = 0.0f;
#pragma unroll
            for (int w = 0; w < NW; ++w)
                m = fmaxf(m, __ldg(reinterpret_cast<const float*>(a.src + a.stride * w) + L.slot + j));
            smax_b[j] = m;
        }
    __syncthreads();
    OptDev od{};
    if (kOpt) od = a.optd[ch.layer];
    float* out = L.out + ch.begin;
    const bool vec_out = (L.flags & kLayerVecOut) != 0;
    uint32_t bad = 0;
    float s_max = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s_max = fmaxf(s_max, sw[w]);  // cluster.hpp:195-196
    for (uint32_t q = tid; q < nbytes; q += kThreads) {
        const float s_q = mb ? smax_b[q >> shq] : s_max;
        auto val = [&](uint32_t idx) {  // (s * float(sum)) * invN, sum = idx - NW (codec.hpp:296)
            return __fmul_rn(__fmul_rn(s_q, small_int_float(static_cast<int>(idx) - NW)), a.inv_n);
        };
        uint32_t acc = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t b = codes[w][q];
            acc += lane_biased_swar(b);
            bad |= b & (b >> 1);
        }
        const float4 o = make_float4(val(acc & 0xffu), val((acc >> 8) & 0xffu),
                                     val((acc >> 16) & 0xffu), val(acc >> 24));
        const uint32_t b4 = 4 * q;
        if (kOpt) {  // fused optimizer: the averaged gradient is never written
            const uint64_t e = ch.begin + b4;
            opt_apply4(a.opt, od.w + e, od.s1 ? od.s1 + e : nullptr, od.s2 ? od.s2 + e : nullptr, o,
                       od.vec != 0, count - b4 < 4 ? count - b4 : 4);
        } else if (vec_out && b4 + 4 <= count) {
            __stcs(reinterpret_cast<float4*>(out + b4), o);
        } else {
            if (b4 + 0 < count) out[b4 + 0] = o.x;
            if (b4 + 1 < count) out[b4 + 1] = o.y;
            if (b4 + 2 < count) out[b4 + 2] = o.z;
            if (b4 + 3 < count) out[b4 + 3] = o.w;
        }
    }
    if (bad & 0x55u) {  // rare: locate the first corrupt element of this thread
        for (uint32_t q = tid; q < nbytes; q += kThreads)
            for (int w = 0; w < NW; ++w) {
                const uint32_t b = codes[w][q] & (codes[w][q] >> 1) & 0x55u;
                if (b) {
                    raise_error(a.err, TGB_E_CORRUPT_CODE, static_cast<int32_t>(L.tensor),
                                block_rng_base(L) + ch.begin + 4ull * q + ((__ffs(b) - 1) >> 1));
                    return;
                }
            }
    }
}

// ====================================================== sharded exchange
// Shared scalers, N <= 8 (the default from N = 5): instead of every rank
// receiving and decoding all N code streams, rank r owns a contiguous range of
// K2 chunks (a parameter-server shard, cluster.hpp:167-221 partitioned over the
// ranks). K2 stores each chunk's codes into its owner's gather buffer only; K3a
// (owner) sums the N workers' codes of the owned chunks into biased integer sums
// N + sum_w code_w in [0, 2N] -- the reference's SharedSumBlock sums
// (wire.hpp:79-97) -- packs them as base-(2N+1) digits, radix_m per u32 word
// (little-endian digit order, as the reference's u64 words, wire.hpp:103-145:
// 3.2 bits per element at N = 4, 4.57 at N = 8 instead of 4 / 8), and stores the
// words into every rank's sums buffer; K3b decodes the sums on every rank to
// (s*float(sum))*invN. Passthrough chunks: K3a writes the final fp64
// worker-order mean (codec.hpp:269-279) and K3b copies it.
struct ShardArgs {
    const uint8_t* src;            // own gather buffer (N push areas, stride apart)
    uint64_t stride;
    uint8_t* sums[kMaxPeers];      // every rank's sums buffer (this step's parity)
    const uint8_t* own_sums;
    int32_t n_workers;
    int32_t radix_m;
    uint32_t chunk12;
    uint32_t sum_region;
    float inv_n;
    ErrWord* err;
};

// byte offset of chunk ch's sums region (a block's chunks are chunk12 apart)
__device__ __forceinline__ uint64_t sums_offset(const ShardArgs& a, const LayerDev& L,
                                                const ChunkDev& ch) {
    return 16ull * L.sum_off16 + (ch.begin / a.chunk12) * static_cast<uint64_t>(a.sum_region);
}

constexpr uint32_t kRadixWordsMax = (kChunk12 + 6) / 7;  // radix_m >= 7 for N <= 8
constexpr uint32_t kK3aSmem = kChunk12 + 4 * (kRadixWordsMax + 4);

template <int NW>
__global__ void __launch_bounds__(kThreads) k3_reduce(TableSource src, ShardArgs a) {
    if (exchange_failed(a.err)) return;  // the codes of this step are incomplete
    ChunkDev ch;
    LayerDev L;
    src.get(blockIdx.x, ch, L);
    const uint32_t tid = threadIdx.x;
    const uint32_t count = ch.count;
    if (L.flags & kLayerPassthrough) {  // fp64 worker-order mean (codec.hpp:269-279)
        const uint64_t off = L.code_off + 4ull * ch.begin;
        const uint64_t soff = 16ull * L.sum_off16 + 4ull * ch.begin;
        const double dn = static_cast<double>(NW);
        const uint32_t n4 = count >> 2;
        for (uint32_t i = tid; i < n4; i += kThreads) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(a.src + a.stride * w + off) + i);
                s0 = __dadd_rn(s0, static_cast<double>(v.x));
                s1 = __dadd_rn(s1, static_cast<double>(v.y));
                s2 = __dadd_rn(s2, static_cast<double>(v.z));
                s3 = __dadd_rn(s3, static_cast<double>(v.w));
            }
            const float4 o = make_float4(static_cast<float>(s0 / dn), static_cast<float>(s1 / dn),
                                         static_cast<float>(s2 / dn), static_cast<float>(s3 / dn));
#pragma unroll
            for (int p = 0; p < NW; ++p) reinterpret_cast<float4*>(a.sums[p] + soff)[i] = o;
        }
        for (uint32_t i = 4 * n4 + tid; i < count; i += kThreads) {
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w)
                sum = __dadd_rn(sum, static_cast<double>(
                                         reinterpret_cast<const float*>(a.src + a.stride * w + off)[i]));
            const float v = static_cast<float>(sum / dn);
#pragma unroll
            for (int p = 0; p < NW; ++p) reinterpret_cast<float*>(a.sums[p] + soff)[i] = v;
        }
        return;
    }
    constexpr uint32_t kBase = 2 * NW + 1;
    extern __shared__ __align__(16) uint8_t k3a_dsm[];  // kK3aSmem bytes (dynamic: > 48 KB)
    uint8_t* sums = k3a_dsm;                                           // biased sum per element
    uint32_t* words = reinterpret_cast<uint32_t*>(k3a_dsm + kChunk12);  // packed digits
    const uint32_t nbytes = (count + 3) >> 2;
    const uint32_t n16 = nbytes >> 4;
    const uint8_t* base[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) base[w] = a.src + a.stride * w + L.code_off + (ch.begin >> 2);
    uint32_t bad = 0;
    // 16 code bytes (64 elements) per worker per step: SWAR byte-lane sums
    for (uint32_t i = tid; i < n16; i += kThreads) {
        uint4 v[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) v[w] = __ldcs(reinterpret_cast<const uint4*>(base[w]) + i);
        uint32_t acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t wd[4] = {v[w].x, v[w].y, v[w].z, v[w].w};
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] += lane_biased_swar((wd[j >> 2] >> (8 * (j & 3))) & 0xFFu);
            bad |= (wd[0] & (wd[0] >> 1)) | (wd[1] & (wd[1] >> 1)) | (wd[2] & (wd[2] >> 1)) |
                   (wd[3] & (wd[3] >> 1));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            reinterpret_cast<uint4*>(sums)[4 * i + k] =
                make_uint4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
    }
    for (uint32_t q = (n16 << 4) + tid; q < nbytes; q += kThreads) {  // tail code bytes
        uint32_t acc = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t bw = base[w][q];
            acc += lane_biased_swar(bw);
            bad |= bw & (bw >> 1);
        }
        reinterpret_cast<uint32_t*>(sums)[q] = acc;
    }
    __syncthreads();
    // radix words: word k holds elements [k m, (k+1) m), digit 0 = lowest (Horner
    // from the highest digit; digits past the chunk's end are 0)
    const uint32_t m = static_cast<uint32_t>(a.radix_m);
    const uint32_t nw = (count + m - 1) / m;
    for (uint32_t k = tid; k < nw; k += kThreads) {
        const uint32_t e0 = k * m;
        uint32_t word = 0;
        for (uint32_t d = m; d-- > 0;) {
            const uint32_t e = e0 + d;
            word = word * kBase + (e < count ? static_cast<uint32_t>(sums[e]) : 0u);
        }
        words[k] = word;
    }
    __syncthreads();
    const uint64_t doff = sums_offset(a, L, ch);
    bulk_copy_out(reinterpret_cast<const uint8_t*>(words), [&](int p) { return a.sums[p] + doff; },
                  NW, 4 * nw);
    if (bad & 0x55555555u) {  // rare: locate the chunk's first corrupt element
        for (uint32_t q = 0; q < nbytes; ++q) {
            for (int w = 0; w < NW; ++w) {
                const uint32_t bb = base[w][q] & (base[w][q] >> 1) & 0x55u;
                if (bb) {
                    raise_error(a.err, TGB_E_CORRUPT_CODE, static_cast<int32_t>(L.tensor),
                                block_rng_base(L) + ch.begin + 4ull * q + ((__ffs(bb) - 1) >> 1));
                    return;
                }
            }
        }
    }
}

// K3b: every rank, every chunk (K2's table): radix words -> biased sums in shared
// memory -> (s * float(sum)) * invN as float4 streams (codec.hpp:296, wire.hpp:220)
template <int NW>
__global__ void __launch_bounds__(kThreads) k3_expand(TableSource src, ShardArgs a) {
    if (exchange_failed(a.err)) return;
    ChunkDev ch;
    LayerDev L;
    src.get(blockIdx.x, ch, L);
    const uint32_t tid = threadIdx.x;
    float* out = L.out + ch.begin;
    const bool vec_out = (L.flags & kLayerVecOut) != 0;
    const uint32_t count = ch.count;
    if (L.flags & kLayerPassthrough) {
        const float* v = reinterpret_cast<const float*>(a.own_sums + 16ull * L.sum_off16) + ch.begin;
        const uint32_t n4 = vec_out ? (count >> 2) : 0u;
        for (uint32_t i = tid; i < n4; i += kThreads)
            __stcs(reinterpret_cast<float4*>(out) + i, __ldcs(reinterpret_cast<const float4*>(v) + i));
        for (uint32_t i = 4 * n4 + tid; i < count; i += kThreads) out[i] = v[i];
        return;
    }
    constexpr uint32_t kBase = 2 * NW + 1;
    __shared__ __align__(16) uint8_t sums[kChunk12 + 64];
    __shared__ float sw[NW];
    if (tid < NW) sw[tid] = __ldg(reinterpret_cast<const float*>(a.src + a.stride * tid) + L.slot);
    const uint32_t m = static_cast<uint32_t>(a.radix_m);
    const uint32_t nw = (count + m - 1) / m;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(a.own_sums + sums_offset(a, L, ch));
    for (uint32_t k = tid; k < nw; k += kThreads) {
        uint32_t x = __ldcs(words + k);
        const uint32_t e0 = k * m;
        for (uint32_t d = 0; d < m; ++d) {  // e0 + d < count + m <= kChunk12 + 64
            const uint32_t q = x / kBase;
            sums[e0 + d] = static_cast<uint8_t>(x - q * kBase);
            x = q;
        }
    }
    __shared__ float smax_b[kMaxItemBuckets];  // multi-bucket item: s per bucket
    const bool mb = ch.nblk > 1;
    const uint32_t shq = mb ? bucket_log2(L) - 2 : 31u;
    if (mb)
        for (uint32_t j = tid; j < ch.nblk; j += kThreads) {
            float m = 0.0f;
#pragma unroll
            for (int w = 0; w < NW; ++w)
                m = fmaxf(m, __ldg(reinterpret_cast<const float*>(a.src + a.stride * w) + L.slot + j));
            smax_b[j] = m;
        }
    __syncthreads();
    float s_max = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s_max = fmaxf(s_max, sw[w]);  // cluster.hpp:195-196
    const uint32_t nbytes = (count + 3) >> 2;
    for (uint32_t q = tid; q < nbytes; q += kThreads) {
        const float s_q = mb ? smax_b[q >> shq] : s_max;
        auto val = [&](uint32_t idx) {  // (s * float(sum)) * invN, sum = idx - NW (codec.hpp:296)
            return __fmul_rn(__fmul_rn(s_q, small_int_float(static_cast<int>(idx) - NW)), a.inv_n);
        };
        const uint32_t v = reinterpret_cast<const uint32_t*>(sums)[q];
        const float4 o = make_float4(val(v & 0xffu), val((v >> 8) & 0xffu), val((v >> 16) & 0xffu),
                                     val(v >> 24));
        const uint32_t b4 = 4 * q;
        if (vec_out && b4 + 4 <= count) {
            __stcs(reinterpret_cast<float4*>(out + b4), o);
        } else {
            if (b4 + 0 < count) out[b4 + 0] = o.x;
            if (b4 + 1 < count) out[b4 + 1] = o.y;
            if (b4 + 2 < count) out[b4 + 2] = o.z;
            if (b4 + 3 < count) out[b4 + 3] = o.w;
        }
    }
}

// clip apply for the per-layer clip API (codec.hpp:121-122)
__global__ void __launch_bounds__(kThreads)
k_clip_apply(const float* g, uint64_t n, const float* bound, float* out) {
    const float b = *bound;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kThreads) {
        const float x = g[i];
        out[i] = fabsf(x) > b ? copysignf(b, x) : x;
    }
}

// per-layer raw average (PassthroughBlock part of average, codec.hpp:269-279)
__global__ void __launch_bounds__(kThreads) k_average_raw(K3Ptrs ptrs, int32_t n_workers,
                                                          uint64_t n, float* out, int vec) {
    const uint64_t begin = static_cast<uint64_t>(blockIdx.x) * kChunk;
    const uint64_t rem = n - begin;
    const uint32_t count = static_cast<uint32_t>(rem < kChunk ? rem : kChunk);
    k3_passthrough([&](int w) { return reinterpret_cast<const float*>(ptrs.codes[w]) + begin; },
                   n_workers, out + begin, count, vec != 0);
}

__global__ void __launch_bounds__(kThreads)
k_rng_bits(uint32_t key0, uint32_t key1, uint64_t t, uint64_t k0, uint64_t n, uint32_t* out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
    if (i >= n) return;
    const uint64_t idx = k0 + i, c = idx >> 2;
    const uint4 r = philox10(make_uint4(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32),
                                        static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32)),
                             key0, key1);
    const uint32_t lane = static_cast<uint32_t>(idx & 3);
    out[i] = lane == 0 ? r.x : lane == 1 ? r.y : lane == 2 ? r.z : r.w;
}

// ============================================================ launchers
static inline cudaError_t launch_status() { return cudaGetLastError(); }

cudaError_t launch_k1_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K1Launch& p, cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    K1Out o{p.partials, p.layer_done, p.global_done, p.bounds, p.slots, p.err, p.clip_factor,
            p.global_bucketing, p.n_layers, p.n_active_layers, layers, p.push, p.tensors, p.nnz};
    o.bmax = p.bmax;
    o.gpart = p.gpart;
    o.gdone = p.gdone;
    const TableSource src{chunks};
    if (p.keep_chunks) {  // the launch's last units stay in L2 for K2's reverse walk
        o.keep_from = n_chunks - (p.keep_chunks < n_chunks ? p.keep_chunks : n_chunks);
        k1_stats<TableSource, 8, 1, 4, true><<<n_chunks, kThreads, 0, st>>>(src, o);
        return launch_status();
    }
    // 8 float4 in flight per thread, <= 64 registers: 4 CTAs/SM (tools/k1_probe.py)
    k1_stats<TableSource, 8, 1, 4><<<n_chunks, kThreads, 0, st>>>(src, o);
    return launch_status();
}

cudaError_t launch_k1_single(const LayerDev& L, const K1Launch& p, cudaStream_t st) {
    const uint32_t nc = static_cast<uint32_t>((L.n + kChunk - 1) / kChunk);
    if (nc == 0) return cudaSuccess;
    K1Out o{p.partials, p.layer_done, p.global_done, p.bounds, p.slots, p.err, p.clip_factor, 0,
            1, 1, nullptr, PeerPush{}, nullptr};
    LayerDev l = L;
    l.tensor = 0;
    l.first_chunk = 0;
    l.n_chunks = nc;
    k1_stats<SingleSource, 8, 1, 4><<<nc, kThreads, 0, st>>>(SingleSource{l, kChunk}, o);
    return launch_status();
}

cudaError_t launch_k1_bucket_slots(const LayerDev* layers, const uint2* meta, uint32_t n_blocks,
                                   const K1Launch& p, cudaStream_t st) {
    if (n_blocks == 0) return cudaSuccess;
    K1Out o{p.partials, p.layer_done, p.global_done, p.bounds, p.slots, p.err, p.clip_factor,
            p.global_bucketing, p.n_layers, p.n_active_layers, layers, p.push, p.tensors, nullptr};
    o.bmax = p.bmax;
    uint32_t grid = (n_blocks + kThreads - 1) / kThreads;
    if (grid > 148u * 8) grid = 148u * 8;
    k1_bucket_slots<<<grid, kThreads, 0, st>>>(meta, n_blocks, o);
    return launch_status();
}

// K2 launch; with a.pdl it is K1's programmatic dependent (same stream, launched
// while K1's last wave drains; the kernel's griddepcontrol.wait orders it after K1)
template <class Kern>
static cudaError_t k2_go(Kern k, uint32_t grid, cudaStream_t st, const TableSource& src,
                         const K2Args& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = a.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, src, a);
}

// K2 instantiations: unfused (codes only, 3 CTAs/SM) and, at N == 1, with the
// decode fused (64 registers, 4 CTAs/SM: 190.9 vs 202.9 us at 3 CTAs/SM on
// VGG-16, the fused kernel is latency-bound), with or without the optimizer
#define TGB_K2_PLAIN k2_ternarize<TableSource, 3, false, false>
#define TGB_K2_FUSED k2_ternarize<TableSource, 4, true, false>
#define TGB_K2_FUSED_OPT k2_ternarize<TableSource, 3, true, true>

cudaError_t launch_k2_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K2Launch& p, cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    K2Args a{p.push, p.slots, p.bounds, p.err, p.t, p.reverse, 0, 0.0f, 0, p.dst};
    a.nnz = p.nnz;
    a.shard_n = p.shard_n;
    a.pdl = p.pdl;
    a.keep_from = p.keep_from;
    for (int r = 0; r <= kMaxPeers; ++r) a.shard_bounds[r] = p.shard_bounds[r];
    a.pull8 = p.pull8;
    a.rank = p.rank;
    a.slot_push = p.slot_push;
    a.n_pieces = p.n_pieces;
    if (p.n_pieces) {
        for (int q = 0; q <= kMaxPieces; ++q) a.piece_bounds[q] = p.piece_bounds[q];
        for (int q = 0; q < kMaxPieces; ++q)
            for (int r = 0; r <= kMaxPeers; ++r) a.owner_bounds[q][r] = p.owner_bounds[q][r];
        a.piece_cnt = p.piece_cnt;
        for (int r = 0; r < kMaxPeers; ++r) a.flag_remote[r] = p.flag_remote[r];
        a.n_flags = p.n_flags;
        a.epoch = p.epoch;
    }
    const TableSource src{chunks};
    if (p.fuse_decode && p.optd) {  // N == 1 fused decode -> optimizer
        a.optd = p.optd;
        a.opt = p.opt;
        return k2_go(TGB_K2_FUSED_OPT, n_chunks, st, src, a);
    }
    if (p.fuse_decode) return k2_go(TGB_K2_FUSED, n_chunks, st, src, a);
    return k2_go(TGB_K2_PLAIN, n_chunks, st, src, a);
}

cudaError_t launch_k2_single(const LayerDev& L, const K2Launch& p, cudaStream_t st) {
    const uint32_t nc = static_cast<uint32_t>((L.n + kChunk12 - 1) / kChunk12);
    if (nc == 0) return cudaSuccess;
    K2Args a{p.push, p.slots, p.bounds, p.err, p.t, 0, 1, p.s_imm, p.rng_base, PeerPush{}};
    a.shard_n = 0;
    k2_ternarize<SingleSource><<<nc, kThreads, 0, st>>>(SingleSource{L, kChunk12}, a);
    return launch_status();
}

template <class K>
static uint32_t k12_grid(K kernel, uint32_t units) {
    static int cap[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 1;
    if (!cap[dev]) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kThreads, 0);
        cap[dev] = sms * (per > 0 ? per : 1);
    }
    return units < static_cast<uint32_t>(cap[dev]) ? (units ? units : 1u)
                                                   : static_cast<uint32_t>(cap[dev]);
}

cudaError_t launch_k12_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_k1,
                             uint32_t n_k2, const K1Launch& p1, const K2Launch& p2,
                             uint32_t* ready, uint32_t epoch, cudaStream_t st) {
    if (n_k2 == 0) return cudaSuccess;
    K1Out o{p1.partials, p1.layer_done, p1.global_done, p1.bounds, p1.slots, p1.err,
            p1.clip_factor, p1.global_bucketing, p1.n_layers, p1.n_active_layers, layers,
            p1.push, p1.tensors, nullptr};
    o.ready = ready;
    o.ready_global = ready + p1.n_tensors;
    o.epoch = epoch ? epoch : 1u;
    K2Args a{p2.push, p2.slots, p2.bounds, p2.err, p2.t, 0, 0, 0.0f, 0, p2.dst};
    a.nnz = p2.nnz;
    a.shard_n = p2.shard_n;
    for (int r = 0; r <= kMaxPeers; ++r) a.shard_bounds[r] = p2.shard_bounds[r];
    const TableSource src{chunks};
    const uint32_t units = n_k1 > n_k2 ? n_k1 : n_k2;
    const uint32_t nf = static_cast<uint32_t>(p1.n_tensors) + 1;  // ready[nf] = exit counter
    if (p2.fuse_decode && p2.optd) {
        a.optd = p2.optd;
        a.opt = p2.opt;
        k12_fused<true, true><<<k12_grid(k12_fused<true, true>, units), kThreads, 0, st>>>(
            src, o, a, n_k1, n_k2, nf);
    } else if (p2.fuse_decode) {
        k12_fused<true><<<k12_grid(k12_fused<true>, units), kThreads, 0, st>>>(src, o, a, n_k1,
                                                                             n_k2, nf);
    } else {
        k12_fused<false><<<k12_grid(k12_fused<false>, units), kThreads, 0, st>>>(src, o, a, n_k1,
                                                                               n_k2, nf);
    }
    return launch_status();
}

template <int NW>
static void k3_staged_go(bool opt, uint32_t n_chunks, cudaStream_t st, const TableSource& src,
                         const K3Args& a) {
    if (opt)
        k3_decode_staged<NW, true><<<n_chunks, kThreads, 0, st>>>(src, a);
    else
        k3_decode_staged<NW, false><<<n_chunks, kThreads, 0, st>>>(src, a);
}

cudaError_t launch_k3_table(const LayerDev* layers, const ChunkFat* chunks, uint32_t n_chunks,
                            const K3Launch& p, cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    K3Args a{p.src, p.stride, nullptr, nullptr, 0.0f, p.n_workers, p.sharing, p.inv_n, p.err};
    a.gate = p.gate;
    a.pull8 = p.pull8;
    for (int w = 0; w < kMaxPeers; ++w) a.wsrc[w] = p.wsrc[w];
    K3Ptrs ptrs{};
    const TableSource src{chunks};
    if (p.pull8 && !(p.sharing && p.n_workers <= kMaxPeers)) return cudaErrorInvalidValue;
    if (p.sharing && p.n_workers <= kMaxPeers) {  // staged SWAR kernel (fused optimizer optional)
        if (p.optd) {
            a.optd = p.optd;
            a.opt = p.opt;
        }
        const bool opt = p.optd != nullptr;
        switch (p.n_workers) {
            case 1: k3_staged_go<1>(opt, n_chunks, st, src, a); break;
            case 2: k3_staged_go<2>(opt, n_chunks, st, src, a); break;
            case 3: k3_staged_go<3>(opt, n_chunks, st, src, a); break;
            case 4: k3_staged_go<4>(opt, n_chunks, st, src, a); break;
            case 5: k3_staged_go<5>(opt, n_chunks, st, src, a); break;
            case 6: k3_staged_go<6>(opt, n_chunks, st, src, a); break;
            case 7: k3_staged_go<7>(opt, n_chunks, st, src, a); break;
            default: k3_staged_go<8>(opt, n_chunks, st, src, a); break;
        }
        return launch_status();
    }
    if (p.optd) return cudaErrorInvalidValue;  // the caller checks opt_fusable
    if (p.sharing)
        k3_decode<TableSource, true, true><<<n_chunks, kThreads, 0, st>>>(src, a, ptrs);
    else
        k3_decode<TableSource, true, false><<<n_chunks, kThreads, 0, st>>>(src, a, ptrs);
    return launch_status();
}

cudaError_t launch_k3_single(const LayerDev& L, const uint8_t* const* codes, const float* scalers,
                             const K3Launch& p, cudaStream_t st) {
    const uint32_t nc = static_cast<uint32_t>((L.n + kChunk - 1) / kChunk);
    if (nc == 0) return cudaSuccess;
    K3Args a{nullptr, 0, nullptr, scalers, p.s_imm, p.n_workers, p.sharing, p.inv_n, p.err};
    K3Ptrs ptrs{};
    for (int w = 0; w < p.n_workers; ++w) ptrs.codes[w] = codes[w];
    const SingleSource src{L, kChunk};
    if (p.sharing)
        k3_decode<SingleSource, false, true><<<nc, kThreads, 0, st>>>(src, a, ptrs);
    else
        k3_decode<SingleSource, false, false><<<nc, kThreads, 0, st>>>(src, a, ptrs);
    return launch_status();
}

cudaError_t launch_average_raw(int32_t n_workers, const float* const* vals, uint64_t n,
                               float* out, cudaStream_t st) {
    const uint64_t nc = (n + kChunk - 1) / kChunk;
    if (nc == 0) return cudaSuccess;
    K3Ptrs ptrs{};
    bool vec = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    for (int w = 0; w < n_workers; ++w) {
        ptrs.codes[w] = reinterpret_cast<const uint8_t*>(vals[w]);
        vec = vec && (reinterpret_cast<uintptr_t>(vals[w]) & 15u) == 0;
    }
    k_average_raw<<<static_cast<uint32_t>(nc), kThreads, 0, st>>>(ptrs, n_workers, n, out,
                                                                   vec ? 1 : 0);
    return launch_status();
}

cudaError_t launch_k3_reduce(const ChunkFat* chunks, uint32_t n_chunks, const ShardLaunch& p,
                             cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    ShardArgs a{p.src, p.stride, {}, p.own_sums, p.n_workers, p.radix_m, p.chunk12,
                p.sum_region, p.inv_n, p.err};
    for (int r = 0; r < p.n_workers; ++r) a.sums[r] = p.sums[r];
    const TableSource src{chunks};
    switch (p.n_workers) {
        case 2: k3_reduce<2><<<n_chunks, kThreads, kK3aSmem, st>>>(src, a); break;
        case 3: k3_reduce<3><<<n_chunks, kThreads, kK3aSmem, st>>>(src, a); break;
        case 4: k3_reduce<4><<<n_chunks, kThreads, kK3aSmem, st>>>(src, a); break;
        case 5: k3_reduce<5><<<n_chunks, kThreads, kK3aSmem, st>>>(src, a); break;
        case 6: k3_reduce<6><<<n_chunks, kThreads, kK3aSmem, st>>>(src, a); break;
        case 7: k3_reduce<7><<<n_chunks, kThreads, kK3aSmem, st>>>(src, a); break;
        case 8: k3_reduce<8><<<n_chunks, kThreads, kK3aSmem, st>>>(src, a); break;
        default: return cudaErrorInvalidValue;
    }
    return launch_status();
}

cudaError_t launch_k3_expand(const ChunkFat* chunks, uint32_t n_chunks, const ShardLaunch& p,
                             cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    ShardArgs a{p.src, p.stride, {}, p.own_sums, p.n_workers, p.radix_m, p.chunk12,
                p.sum_region, p.inv_n, p.err};
    const TableSource src{chunks};
    switch (p.n_workers) {
        case 2: k3_expand<2><<<n_chunks, kThreads, 0, st>>>(src, a); break;
        case 3: k3_expand<3><<<n_chunks, kThreads, 0, st>>>(src, a); break;
        case 4: k3_expand<4><<<n_chunks, kThreads, 0, st>>>(src, a); break;
        case 5: k3_expand<5><<<n_chunks, kThreads, 0, st>>>(src, a); break;
        case 6: k3_expand<6><<<n_chunks, kThreads, 0, st>>>(src, a); break;
        case 7: k3_expand<7><<<n_chunks, kThreads, 0, st>>>(src, a); break;
        case 8: k3_expand<8><<<n_chunks, kThreads, 0, st>>>(src, a); break;
        default: return cudaErrorInvalidValue;
    }
    return launch_status();
}

// ============================================================== telemetry
// histogram (codec.hpp:491-517): equal-width bins over [min, max] in double,
// b = size_t((double(x) - lo) / width) clamped to bins - 1 (width 0: bin 0).
// Pass 1: float min/max (NaN ignored; the host handles a NaN first element,
// which the reference's std::min/max chain would propagate). Pass 2: bins.
__device__ __forceinline__ uint32_t float_order(float x) {  // monotone float -> uint32
    const uint32_t u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float order_float(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__global__ void __launch_bounds__(kThreads) k_minmax(const float* v, uint64_t n, uint32_t* mm) {
    float lo = INFINITY, hi = -INFINITY;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kThreads) {
        const float x = v[i];
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31u) == 0) {
        atomicMin(mm, float_order(lo));
        atomicMax(mm + 1, float_order(hi));
    }
}

constexpr uint32_t kHistSmem = 4096;  // bins counted in shared memory per CTA

__global__ void __launch_bounds__(kThreads) k_histogram(const float* v, uint64_t n, uint32_t bins,
                                                        const uint32_t* mm, int nan_first,
                                                        unsigned long long* counts,
                                                        double* edges) {
    __shared__ unsigned int sh[kHistSmem];
    const bool use_sh = bins <= kHistSmem;
    const double lo = nan_first ? static_cast<double>(NAN) : static_cast<double>(order_float(mm[0]));
    const double hi = nan_first ? static_cast<double>(NAN) : static_cast<double>(order_float(mm[1]));
    const double width = __ddiv_rn(__dsub_rn(hi, lo), static_cast<double>(bins));
    if (use_sh)
        for (uint32_t b = threadIdx.x; b < bins; b += kThreads) sh[b] = 0;
    if (blockIdx.x == 0)
        for (uint32_t b = threadIdx.x; b < bins; b += kThreads)
            edges[b] = __dadd_rn(lo, __dmul_rn(width, static_cast<double>(b)));
    __syncthreads();
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kThreads) {
        uint64_t b = 0;
        if (width > 0.0) {
            const double q = __ddiv_rn(__dsub_rn(static_cast<double>(v[i]), lo), width);
            // size_t conversion; NaN (and out-of-range) lands in the last bin like x86-64
            b = (q == q && q < 18446744073709551616.0) ? static_cast<uint64_t>(q) : ~0ull;
        }
        if (b >= bins) b = bins - 1;
        if (use_sh)
            atomicAdd(&sh[b], 1u);
        else
            atomicAdd(counts + b, 1ull);
    }
    if (use_sh) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < bins; b += kThreads)
            if (sh[b]) atomicAdd(counts + b, static_cast<unsigned long long>(sh[b]));
    }
}

cudaError_t launch_histogram(const float* v, uint64_t n, uint32_t bins, uint32_t* mm,
                             int nan_first, unsigned long long* counts, double* edges,
                             cudaStream_t st, int pass) {
    uint64_t blocks = (n + kThreads - 1) / kThreads;
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    if (blocks == 0) blocks = 1;
    if (pass == 0)
        k_minmax<<<static_cast<uint32_t>(blocks), kThreads, 0, st>>>(v, n, mm);
    else
        k_histogram<<<static_cast<uint32_t>(blocks), kThreads, 0, st>>>(v, n, bins, mm, nan_first,
                                                                     counts, edges);
    return launch_status();
}

// standalone optimizer apply over one tensor (unfused path / per-layer API)
__global__ void __launch_bounds__(kThreads) k_opt_apply(OptArgs o, uint64_t n, float* w,
                                                        const float* g, float* s1, float* s2) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kThreads) {
        float wi = w[i], a = s1 ? s1[i] : 0.0f, b = s2 ? s2[i] : 0.0f;
        opt_apply1(o, g[i], wi, a, b);
        w[i] = wi;
        if (s1) s1[i] = a;
        if (s2) s2[i] = b;
    }
}

cudaError_t launch_opt_apply(const OptArgs& o, uint64_t n, float* w, const float* g, float* s1,
                             float* s2, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + kThreads - 1) / kThreads;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    k_opt_apply<<<static_cast<uint32_t>(blocks), kThreads, 0, st>>>(o, n, w, g, s1, s2);
    return launch_status();
}

// ================================================================== wire
// Reference wire format (codec.hpp:383-438 push payload, wire.hpp:41-228 frame
// and pull payload) on the device. Little-endian byte streams at arbitrary
// offsets, so everything below is byte-granular.

// push: copy the dynamic parts (scalers, codes, raw values) of this step's push
// area into the frame image whose static headers were written once.

// segments are pre-split into pieces of <= 64 KB; one CTA per piece (grid-stride)
__global__ void __launch_bounds__(kThreads) k_wire_gather(const uint8_t* push, const WireSeg* segs,
                                                          uint32_t n_segs, uint8_t* frame) {
    for (uint32_t p = blockIdx.x; p < n_segs; p += gridDim.x) {
        const WireSeg sg = segs[p];
        for (uint64_t i = threadIdx.x; i < sg.bytes; i += kThreads)
            frame[sg.dst_off + i] = push[sg.src_off + i];
    }
}

cudaError_t launch_wire_gather(const uint8_t* push, const WireSeg* d_segs, uint32_t n_segs,
                               uint8_t* frame, cudaStream_t st) {
    if (n_segs == 0) return cudaSuccess;
    const uint32_t g = n_segs < 148u * 8 ? n_segs : 148u * 8;
    k_wire_gather<<<g, kThreads, 0, st>>>(push, d_segs, n_segs, frame);
    return launch_status();
}

// pull: one thread per radix word of a SharedSumBlock (wire.hpp:147-185):
// digits little-endian within the word, sum = digit - N,
// out = (s * float(sum)) * (1.0f / N) (decode_pull, wire.hpp:216-220).

__device__ __forceinline__ uint64_t load_u64_le(const uint8_t* p) {
    uint64_t v = 0;
#pragma unroll
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

__global__ void __launch_bounds__(kThreads) k_pull_decode(const uint8_t* payload, const PullSeg* segs,
                                                          uint32_t n_segs, uint32_t total_threads,
                                                          int* bad) {
    const uint32_t gt = blockIdx.x * kThreads + threadIdx.x;
    if (gt >= total_threads) return;
    uint32_t lo = 0, hi = n_segs;  // segment with first_thread <= gt (binary search)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (segs[mid].first_thread <= gt) lo = mid; else hi = mid;
    }
    const PullSeg sg = segs[lo];
    const uint32_t i = gt - sg.first_thread;
    if (sg.kind == 4) {  // FloatAvgBlock: values verbatim
        if (i >= sg.n) return;
        const uint8_t* p = payload + sg.src_off + 4ull * i;
        sg.out[i] = __uint_as_float(static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) |
                                    (static_cast<uint32_t>(p[2]) << 16) |
                                    (static_cast<uint32_t>(p[3]) << 24));
        return;
    }
    if (i >= sg.words) return;
    uint64_t word = load_u64_le(payload + sg.src_off + 8ull * i);
    const uint64_t base = sg.base;
    const uint64_t magic = ~0ull / base;  // q = umulhi(word, magic) underestimates by <= 2
    const uint32_t k0 = i * sg.m, k1 = min(k0 + sg.m, sg.n);
    const int N = static_cast<int>((sg.base - 1) / 2);
    for (uint32_t k = k0; k < k1; ++k) {
        uint64_t q = __umul64hi(word, magic);
        uint64_t r = word - q * base;
        while (r >= base) {
            ++q;
            r -= base;
        }
        word = q;
        const int sum = static_cast<int>(r) - N;
        sg.out[k] = __fmul_rn(__fmul_rn(sg.s, static_cast<float>(sum)), sg.inv_n);
    }
    if (word != 0) atomicExch(bad, 1);  // "pull: nonzero radix remainder" (wire.hpp:180)
}

cudaError_t launch_pull_decode(const uint8_t* payload, const PullSeg* d_segs, uint32_t n_segs,
                               uint32_t total_threads, int* bad, cudaStream_t st) {
    if (total_threads == 0) return cudaSuccess;
    k_pull_decode<<<(total_threads + kThreads - 1) / kThreads, kThreads, 0, st>>>(
        payload, d_segs, n_segs, total_threads, bad);
    return launch_status();
}

cudaError_t launch_clip_apply(const float* g, uint64_t n, const float* bound, float* out,
                              cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + kThreads - 1) / kThreads;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    k_clip_apply<<<static_cast<uint32_t>(blocks), kThreads, 0, st>>>(g, n, bound, out);
    return launch_status();
}

cudaError_t launch_rng_bits(uint32_t key0, uint32_t key1, uint64_t t, uint64_t k0, uint64_t n,
                            uint32_t* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const uint32_t blocks = static_cast<uint32_t>((n + kThreads - 1) / kThreads);
    k_rng_bits<<<blocks, kThreads, 0, st>>>(key0, key1, t, k0, n, out);
    return launch_status();
}


// ===================================================== peer flag barrier
// Cross-GPU barrier of the fused / sharded exchange. Every rank keeps one
// 16-byte record {epoch, iteration} per (barrier slot, step parity, peer) in its
// IPC allocation. Thread p publishes this rank's record into peer p's array
// (iteration first, then the epoch with release semantics, system scope) and
// then waits until peer p's record in ours reaches the epoch (acquire). Records
// alternate by step parity: a peer can be at most one step ahead, so the record
// of this epoch is never overwritten while it is read. A peer at another
// iteration raises TGB_E_SKEW (cluster.hpp:141-143); a bounded spin turns a dead
// peer into TGB_E_PEER_TIMEOUT instead of a hang. LocalCluster (one process)
// splits it: kBarrierPost publishes, kBarrierCheck verifies after the streams
// were ordered by events (never spins, so no hardware-queue deadlock).
__global__ void k_peer_barrier(PeerFlags f, uint64_t epoch, uint64_t t, int mode, ErrWord* err) {
    const int p = threadIdx.x;
    if (p >= f.n) return;
    const uint32_t par = static_cast<uint32_t>(epoch & 1u) * kMaxPeers;
    if (mode == kBarrierPost || mode == kBarrierSpin) {
        uint64_t* r = f.remote[p] + 2 * par;
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(r + 1), "l"(t) : "memory");
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(r), "l"(epoch) : "memory");
    }
    if (mode == kBarrierPost) return;
    const uint64_t* rec = f.local + 2 * (par + p);
    uint64_t v = 0;
    long long spins = 0;
    const long long t0 = clock64();
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(rec) : "memory");
        if (v >= epoch) break;
        if (mode == kBarrierCheck ||
            ((++spins & 1023) == 0 && clock64() - t0 > 20000000000ll)) {  // ~10 s
            raise_error(err, TGB_E_PEER_TIMEOUT, -1, static_cast<uint64_t>(p));
            return;
        }
    }
    uint64_t pt = 0;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(pt) : "l"(rec + 1) : "memory");
    if (pt != t) raise_error_aux(err, TGB_E_SKEW, static_cast<uint64_t>(p), pt);
}

cudaError_t launch_peer_barrier(const PeerFlags& f, uint64_t epoch, uint64_t t, int mode,
                                ErrWord* err, cudaStream_t st) {
    k_peer_barrier<<<1, 32, 0, st>>>(f, epoch, t, mode, err);
    return launch_status();
}

// PRESHARED in a LocalCluster: own slots <- max over the N workers' local slots in
// this plan's gather buffer (share_scalers, codec.hpp:136-141; the ranks' NCCL
// max-allreduce). Worker w's slot i sits at gather + w * stride + 4 i.
__global__ void __launch_bounds__(kThreads) k_slot_max(float* own, const uint8_t* gather,
                                                       uint64_t stride, int n, int n_slots) {
    for (int i = blockIdx.x * kThreads + threadIdx.x; i < n_slots; i += gridDim.x * kThreads) {
        float m = 0.0f;
        for (int w = 0; w < n; ++w)
            m = fmaxf(m, reinterpret_cast<const float*>(gather + stride * w)[i]);
        own[i] = m;
    }
}

cudaError_t launch_slot_max(float* own, const uint8_t* gather, uint64_t stride, int n,
                            int n_slots, cudaStream_t st) {
    if (n_slots <= 0) return cudaSuccess;
    int grid = (n_slots + kThreads - 1) / kThreads;
    if (grid > 148 * 4) grid = 148 * 4;
    k_slot_max<<<grid, kThreads, 0, st>>>(own, gather, stride, n, n_slots);
    return launch_status();
}

// ======================================================= kernel preloading
// Every kernel a plan can launch, loaded once per device at plan creation
// (cudaFuncGetAttributes forces the module load under CUDA_MODULE_LOADING=LAZY).
cudaError_t preload_kernels() {
    static bool done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
    cudaFuncAttributes fa;
    const void* ks[] = {
        reinterpret_cast<const void*>(k1_stats<TableSource, 8, 1, 4, true>),
        reinterpret_cast<const void*>(k1_stats<TableSource, 8, 1, 4>),
        reinterpret_cast<const void*>(k1_stats<SingleSource, 8, 1, 4>),
        reinterpret_cast<const void*>(k1_bucket_slots),
        reinterpret_cast<const void*>(TGB_K2_PLAIN),
        reinterpret_cast<const void*>(TGB_K2_FUSED),
        reinterpret_cast<const void*>(TGB_K2_FUSED_OPT),
        reinterpret_cast<const void*>(k2_ternarize<SingleSource>),
        reinterpret_cast<const void*>(k12_fused<true>),
        reinterpret_cast<const void*>(k12_fused<true, true>),
        reinterpret_cast<const void*>(k12_fused<false>),
        reinterpret_cast<const void*>(k3_decode_staged<1, false>),
        reinterpret_cast<const void*>(k3_decode_staged<2, false>),
        reinterpret_cast<const void*>(k3_decode_staged<3, false>),
        reinterpret_cast<const void*>(k3_decode_staged<4, false>),
        reinterpret_cast<const void*>(k3_decode_staged<5, false>),
        reinterpret_cast<const void*>(k3_decode_staged<6, false>),
        reinterpret_cast<const void*>(k3_decode_staged<7, false>),
        reinterpret_cast<const void*>(k3_decode_staged<8, false>),
        reinterpret_cast<const void*>(k3_decode_staged<1, true>),
        reinterpret_cast<const void*>(k3_decode_staged<2, true>),
        reinterpret_cast<const void*>(k3_decode_staged<3, true>),
        reinterpret_cast<const void*>(k3_decode_staged<4, true>),
        reinterpret_cast<const void*>(k3_decode_staged<5, true>),
        reinterpret_cast<const void*>(k3_decode_staged<6, true>),
        reinterpret_cast<const void*>(k3_decode_staged<7, true>),
        reinterpret_cast<const void*>(k3_decode_staged<8, true>),
        reinterpret_cast<const void*>(k3_decode<TableSource, true, true>),
        reinterpret_cast<const void*>(k3_decode<TableSource, true, false>),
        reinterpret_cast<const void*>(k3_decode<SingleSource, false, true>),
        reinterpret_cast<const void*>(k3_decode<SingleSource, false, false>),
        reinterpret_cast<const void*>(k3_reduce<2>), reinterpret_cast<const void*>(k3_reduce<3>),
        reinterpret_cast<const void*>(k3_reduce<4>), reinterpret_cast<const void*>(k3_reduce<5>),
        reinterpret_cast<const void*>(k3_reduce<6>), reinterpret_cast<const void*>(k3_reduce<7>),
        reinterpret_cast<const void*>(k3_reduce<8>),
        reinterpret_cast<const void*>(k3_expand<2>), reinterpret_cast<const void*>(k3_expand<3>),
        reinterpret_cast<const void*>(k3_expand<4>), reinterpret_cast<const void*>(k3_expand<5>),
        reinterpret_cast<const void*>(k3_expand<6>), reinterpret_cast<const void*>(k3_expand<7>),
        reinterpret_cast<const void*>(k3_expand<8>),
        reinterpret_cast<const void*>(k_peer_barrier),
        reinterpret_cast<const void*>(k_slot_max),
        reinterpret_cast<const void*>(k_clip_apply),
        reinterpret_cast<const void*>(k_average_raw),
        reinterpret_cast<const void*>(k_rng_bits),
        reinterpret_cast<const void*>(k_minmax),
        reinterpret_cast<const void*>(k_histogram),
        reinterpret_cast<const void*>(k_opt_apply),
        reinterpret_cast<const void*>(k_wire_gather),
        reinterpret_cast<const void*>(k_pull_decode),
    };
    for (const void* k : ks) {
        e = cudaFuncGetAttributes(&fa, k);
        if (e != cudaSuccess) return e;
    }
    const void* k3a[] = {
        reinterpret_cast<const void*>(k3_reduce<2>), reinterpret_cast<const void*>(k3_reduce<3>),
        reinterpret_cast<const void*>(k3_reduce<4>), reinterpret_cast<const void*>(k3_reduce<5>),
        reinterpret_cast<const void*>(k3_reduce<6>), reinterpret_cast<const void*>(k3_reduce<7>),
        reinterpret_cast<const void*>(k3_reduce<8>)};
    for (const void* k : k3a) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kK3aSmem));
        if (e != cudaSuccess) return e;
    }
    if (dev >= 0 && dev < 64) done[dev] = true;
    return cudaSuccess;
}

}  // namespace tgb
