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
// fp32 streams, one CTA (256 threads) per 16K-element work item.
#include "tgb_device.cuh"
#include "tgb_internal.h"

#include <cfloat>
#include <cmath>

namespace tgb {

// ----------------------------------------------------------------- sources
// A "source" maps blockIdx.x to (chunk, layer). Table: plan tables in HBM.
// Single: one layer passed by value (per-layer API), chunks computed.
struct TableSource {
    const LayerDev* layers;
    const ChunkDev* chunks;
    __device__ __forceinline__ void get(uint32_t b, ChunkDev& ch, LayerDev& L) const {
        ch = chunks[b];
        L = layers[ch.layer];
    }
};

struct SingleSource {
    LayerDev L;
    __device__ __forceinline__ void get(uint32_t b, ChunkDev& ch, LayerDev& L_) const {
        ch.layer = 0;
        ch.begin = static_cast<uint64_t>(b) * kChunk;
        const uint64_t rem = L.n - ch.begin;
        ch.count = static_cast<uint32_t>(rem < kChunk ? rem : kChunk);
        L_ = L;
    }
};

// ====================================================================== K1
struct K1Out {
    Partial* partials;     // one per chunk (indexed by blockIdx.x)
    uint32_t* layer_done;  // per layer arrival counters (self-resetting)
    uint32_t* global_done; // arrival counter over layers (Global bucketing)
    float* bounds;         // per layer clip bound
    float* slots;          // scaler slots
    ErrWord* err;
    float clip_factor;
    int32_t global_bucketing;
    int32_t n_layers;
    int32_t n_active_layers;  // layers with n > 0
    const LayerDev* layers;   // for the Global fix-up (table source only)
};

__device__ __forceinline__ void acc4(const float4 v, const double x0, double& S, double& Q,
                                     float& mx) {
    const double d0 = static_cast<double>(v.x) - x0, d1 = static_cast<double>(v.y) - x0;
    const double d2 = static_cast<double>(v.z) - x0, d3 = static_cast<double>(v.w) - x0;
    S += (d0 + d1) + (d2 + d3);
    Q = fma(d0, d0, Q);
    Q = fma(d1, d1, Q);
    Q = fma(d2, d2, Q);
    Q = fma(d3, d3, Q);
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
}

template <class Src>
__global__ void __launch_bounds__(kThreads) k1_stats(Src src, K1Out o) {
    ChunkDev ch;
    LayerDev L;
    src.get(blockIdx.x, ch, L);
    const float* g = L.g + ch.begin;
    const uint32_t count = ch.count;
    const double x0 = static_cast<double>(__ldg(g));  // per-chunk shift
    double S = 0.0, Q = 0.0;
    float mx = 0.0f;
    const uint32_t tid = threadIdx.x;
    uint32_t done = 0;
    if (L.flags & kLayerVecIn) {
        const float4* g4 = reinterpret_cast<const float4*>(g);
        const uint32_t n4 = count >> 2;
        uint32_t i = tid;
        for (; i + 3 * kThreads < n4; i += 4 * kThreads) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(g4 + i + u * kThreads);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc4(v[u], x0, S, Q, mx);
        }
        for (; i < n4; i += kThreads) acc4(__ldcs(g4 + i), x0, S, Q, mx);
        done = n4 << 2;
    }
    for (uint32_t i = done + tid; i < count; i += kThreads) {
        const float x = __ldcs(g + i);
        const double d = static_cast<double>(x) - x0;
        S += d;
        Q = fma(d, d, Q);
        mx = fmaxf(mx, fabsf(x));
    }
    block_reduce_sq<kThreads / 32>(S, Q, mx);

    __shared__ bool is_last;
    if (tid == 0) {
        const double cn = static_cast<double>(count);
        Partial p;
        p.n = cn;
        p.mean = x0 + S / cn;
        p.m2 = Q - S * (S / cn);
        p.mx = mx;
        p.pad = 0;
        o.partials[blockIdx.x] = p;
        __threadfence();
        const uint32_t ticket = atomicAdd(&o.layer_done[ch.layer], 1u);
        is_last = (ticket == L.n_chunks - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    // ---- last CTA of this layer: deterministic Chan merge of its partials
    __shared__ double sn[kThreads], smean[kThreads], sm2[kThreads];
    __shared__ float smx[kThreads];
    const uint32_t nc = L.n_chunks;
    const uint32_t per = (nc + kThreads - 1) / kThreads;
    double n = 0.0, mean = 0.0, m2 = 0.0;
    float m = 0.0f;
    const uint32_t lo = tid * per, hi = min(nc, lo + per);
    for (uint32_t c = lo; c < hi; ++c) {
        const Partial* pp = o.partials + L.first_chunk + c;
        const double pn = __ldcg(&pp->n), pmean = __ldcg(&pp->mean), pm2 = __ldcg(&pp->m2);
        const float pmx = __ldcg(&pp->mx);
        chan_merge(n, mean, m2, pn, pmean, pm2);
        m = fmaxf(m, pmx);
    }
    sn[tid] = n;
    smean[tid] = mean;
    sm2[tid] = m2;
    smx[tid] = m;
    __syncthreads();
    for (uint32_t s = 1; s < kThreads; s <<= 1) {
        if ((tid & (2 * s - 1)) == 0) {
            double a_n = sn[tid], a_mean = smean[tid], a_m2 = sm2[tid];
            chan_merge(a_n, a_mean, a_m2, sn[tid + s], smean[tid + s], sm2[tid + s]);
            sn[tid] = a_n;
            smean[tid] = a_mean;
            sm2[tid] = a_m2;
            smx[tid] = fmaxf(smx[tid], smx[tid + s]);
        }
        __syncthreads();
    }
    if (tid == 0) {
        const double fm = smean[0];
        double fm2 = sm2[0];
        const float fmx = smx[0];
        float bound = INFINITY, s = 0.0f;
        if (!isfinite(fm) || !isfinite(fm2) || !isfinite(fmx)) {
            raise_error(o.err, TGB_E_NONFINITE, static_cast<int32_t>(ch.layer), 0);
            bound = 0.0f;
            s = 0.0f;
        } else {
            if ((L.flags & kLayerClip) && L.n >= 2) {
                if (fm2 < 0.0) fm2 = 0.0;
                const double sigma = sqrt(fm2 / static_cast<double>(L.n));  // codec.hpp:111
                bound = static_cast<float>(static_cast<double>(o.clip_factor) * sigma);  // :119
            }
            s = fminf(fmx, bound);  // == scaler(clip(g)) (codec.hpp:121-122, :130)
        }
        o.bounds[ch.layer] = bound;
        o.slots[L.slot] = s;
        o.layer_done[ch.layer] = 0u;  // self-reset for the next launch
        if (o.global_bucketing) {
            __threadfence();
            const uint32_t t = atomicAdd(o.global_done, 1u);
            if (t == static_cast<uint32_t>(o.n_active_layers) - 1) {
                __threadfence();
                float gs = 0.0f;  // codec.hpp:212-216
                for (int l = 0; l < o.n_layers; ++l) {
                    const LayerDev& Ll = o.layers[l];
                    if (Ll.n == 0 || (Ll.flags & kLayerPassthrough)) continue;
                    gs = fmaxf(gs, __ldcg(o.slots + Ll.slot));
                }
                for (int l = 0; l < o.n_layers; ++l) {
                    const LayerDev& Ll = o.layers[l];
                    if (Ll.n == 0 || (Ll.flags & kLayerPassthrough)) continue;
                    o.slots[Ll.slot] = gs;
                }
                *o.global_done = 0u;
            }
        }
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
    uint64_t rng_q0;     // per-layer API: rng_base / 4 added to the Philox counter
};

template <class Src>
__global__ void __launch_bounds__(kThreads) k2_ternarize(Src src, K2Args a) {
    const uint32_t b = a.reverse ? (gridDim.x - 1 - blockIdx.x) : blockIdx.x;
    ChunkDev ch;
    LayerDev L;
    src.get(b, ch, L);
    const float s = a.slots ? a.slots[L.slot] : a.s_imm;
    const float bound = a.bounds ? a.bounds[ch.layer] : INFINITY;
    const uint32_t count = ch.count;
    const uint32_t nbytes = (count + 3) >> 2;
    const uint64_t q0 = ch.begin >> 2;  // byte index of this chunk inside the layer
    uint8_t* codes = a.push + L.code_off + q0;
    const float* g = L.g + ch.begin;
    const uint32_t tid = threadIdx.x;

    if (s == 0.0f) {  // codec.hpp:155-159
        for (uint32_t q = tid; q < nbytes; q += kThreads) codes[q] = 0;
        if (a.check)
            for (uint32_t i = tid; i < count; i += kThreads)
                if (g[i] != 0.0f)
                    raise_error(a.err, TGB_E_S0_NONZERO, static_cast<int32_t>(ch.layer),
                                ch.begin + i);
        return;
    }
    Decider dec;
    dec.init(bound, s);
    PhiloxStream ph;
    const uint64_t qg = q0 + a.rng_q0;  // Philox counter of this chunk's first byte
    ph.init(L.key0, L.key1, static_cast<uint32_t>(qg >> 32), a.t);
    const uint32_t qbase = static_cast<uint32_t>(qg);

    const uint32_t nfull = count >> 2;  // bytes whose 4 elements all exist
    uint32_t q = tid;
    if (L.flags & kLayerVecIn) {
        const float4* g4 = reinterpret_cast<const float4*>(g);
        for (; q + 3 * kThreads < nfull; q += 4 * kThreads) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(g4 + q + u * kThreads);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t qq = q + u * kThreads;
                const uint4 r = ph(qbase + qq);
                codes[qq] = static_cast<uint8_t>(dec.byte(v[u], r));
            }
            if (a.check) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float mm = fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)),
                                           fmaxf(fabsf(v[u].z), fabsf(v[u].w)));
                    if (fminf(mm, bound) > s)
                        raise_error(a.err, TGB_E_SCALER_BELOW_MAX, static_cast<int32_t>(ch.layer),
                                    ch.begin + 4ull * (q + u * kThreads));
                }
            }
        }
        for (; q < nfull; q += kThreads) {
            const float4 v = __ldcs(g4 + q);
            const uint4 r = ph(qbase + q);
            codes[q] = static_cast<uint8_t>(dec.byte(v, r));
            if (a.check) {
                const float mm = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
                if (fminf(mm, bound) > s)
                    raise_error(a.err, TGB_E_SCALER_BELOW_MAX, static_cast<int32_t>(ch.layer),
                                ch.begin + 4ull * q);
            }
        }
    }
    // scalar path: unaligned input and the partial last byte (pad bits stay 00)
    for (; q < nbytes; q += kThreads) {
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t i = 4 * q + e;
            x[e] = i < count ? g[i] : 0.0f;
        }
        const uint4 r = ph(qbase + q);
        codes[q] = static_cast<uint8_t>(dec.byte(make_float4(x[0], x[1], x[2], x[3]), r));
        if (a.check) {
            for (int e = 0; e < 4; ++e)
                if (fminf(fabsf(x[e]), bound) > s)
                    raise_error(a.err, TGB_E_SCALER_BELOW_MAX, static_cast<int32_t>(ch.layer),
                                ch.begin + 4ull * q + e);
        }
    }
}

// General-offset ternarize for the per-layer API when rng_base % 4 != 0:
// element k uses stream index rng_base + k (codec.hpp:167), which straddles
// Philox blocks; one thread per output byte, up to two blocks each.
__global__ void __launch_bounds__(kThreads)
k2_ternarize_offset(const float* g, uint64_t n, float s, uint32_t key0, uint32_t key1, uint64_t t,
                    uint64_t rng_base, uint8_t* codes, ErrWord* err) {
    const uint64_t q = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const uint64_t nbytes = (n + 3) >> 2;
    if (q >= nbytes) return;
    if (s == 0.0f) {
        codes[q] = 0;
        for (int e = 0; e < 4; ++e) {
            const uint64_t i = 4 * q + e;
            if (i < n && g[i] != 0.0f) raise_error(err, TGB_E_S0_NONZERO, 0, i);
        }
        return;
    }
    Decider dec;
    dec.init(INFINITY, s);
    uint32_t byte = 0;
    for (int e = 0; e < 4; ++e) {
        const uint64_t i = 4 * q + e;
        if (i >= n) break;
        const uint64_t idx = rng_base + i;
        const uint64_t c = idx >> 2;
        const uint4 r = philox10(make_uint4(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32),
                                            static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32)),
                                 key0, key1);
        const uint32_t lane = static_cast<uint32_t>(idx & 3);
        const uint32_t bits = lane == 0 ? r.x : lane == 1 ? r.y : lane == 2 ? r.z : r.w;
        const float x = g[i];
        if (fabsf(x) > s) raise_error(err, TGB_E_SCALER_BELOW_MAX, 0, i);
        byte |= dec.code(x, bits) << (2 * e);
    }
    codes[q] = static_cast<uint8_t>(byte);
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
};

struct K3Ptrs {  // per-layer API: explicit pointers (passed by value)
    const uint8_t* codes[kMaxWorkers];
};

template <class Src, bool kTable>
__global__ void __launch_bounds__(kThreads) k3_decode(Src src, K3Args a, K3Ptrs ptrs) {
    ChunkDev ch;
    LayerDev L;
    src.get(blockIdx.x, ch, L);
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
    for (uint32_t q = tid; q < nbytes; q += kThreads) {
        uint32_t acc = 0, bad = 0;
        float4 o;
        if (a.sharing) {
            for (int w = 0; w < N; ++w) {
                const uint32_t bw = kTable ? __ldcs(a.src + a.stride * w + L.code_off + q0 + q)
                                           : __ldcs(ptrs.codes[w] + q0 + q);
                acc += tab[bw];
                bad |= bw & (bw >> 1) & 0x55u;
            }
            o = make_float4(lut[acc & 0xffu], lut[(acc >> 8) & 0xffu], lut[(acc >> 16) & 0xffu],
                            lut[acc >> 24]);
        } else {  // codec.hpp:299-306: fp64 worker-order sum, then /N
            double sm[4] = {0.0, 0.0, 0.0, 0.0};
            for (int w = 0; w < N; ++w) {
                const uint32_t bw = kTable ? __ldcs(a.src + a.stride * w + L.code_off + q0 + q)
                                           : __ldcs(ptrs.codes[w] + q0 + q);
                bad |= bw & (bw >> 1) & 0x55u;
                const double sd = static_cast<double>(sw[w]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t c = (bw >> (2 * e)) & 3u;
                    const double v = c == 1u ? 1.0 : (c == 2u ? -1.0 : 0.0);
                    sm[e] = __dadd_rn(sm[e], __dmul_rn(sd, v));
                }
            }
            const double dn = static_cast<double>(N);
            o = make_float4(static_cast<float>(sm[0] / dn), static_cast<float>(sm[1] / dn),
                            static_cast<float>(sm[2] / dn), static_cast<float>(sm[3] / dn));
        }
        const uint32_t base = 4 * q;
        if (vec_out && base + 4 <= count) {
            __stcs(reinterpret_cast<float4*>(out + base), o);
        } else {
            const float ov[4] = {o.x, o.y, o.z, o.w};
            for (int e = 0; e < 4; ++e)
                if (base + e < count) out[base + e] = ov[e];
        }
        if (bad) {
            // only real elements count (pad bits are 00 by construction)
            const uint32_t e = (__ffs(bad) - 1) >> 1;
            raise_error(a.err, TGB_E_CORRUPT_CODE, static_cast<int32_t>(ch.layer),
                        ch.begin + base + e);
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

cudaError_t launch_k1_table(const LayerDev* layers, const ChunkDev* chunks, uint32_t n_chunks,
                            const K1Launch& p, cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    K1Out o{p.partials, p.layer_done, p.global_done, p.bounds, p.slots, p.err, p.clip_factor,
            p.global_bucketing, p.n_layers, p.n_active_layers, layers};
    k1_stats<TableSource><<<n_chunks, kThreads, 0, st>>>(TableSource{layers, chunks}, o);
    return launch_status();
}

cudaError_t launch_k1_single(const LayerDev& L, const K1Launch& p, cudaStream_t st) {
    const uint32_t nc = static_cast<uint32_t>((L.n + kChunk - 1) / kChunk);
    if (nc == 0) return cudaSuccess;
    K1Out o{p.partials, p.layer_done, p.global_done, p.bounds, p.slots, p.err, p.clip_factor, 0,
            1, 1, nullptr};
    LayerDev l = L;
    l.first_chunk = 0;
    l.n_chunks = nc;
    k1_stats<SingleSource><<<nc, kThreads, 0, st>>>(SingleSource{l}, o);
    return launch_status();
}

cudaError_t launch_k2_table(const LayerDev* layers, const ChunkDev* chunks, uint32_t n_chunks,
                            const K2Launch& p, cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    K2Args a{p.push, p.slots, p.bounds, p.err, p.t, p.reverse, 0, 0.0f, 0};
    k2_ternarize<TableSource><<<n_chunks, kThreads, 0, st>>>(TableSource{layers, chunks}, a);
    return launch_status();
}

cudaError_t launch_k2_single(const LayerDev& L, const K2Launch& p, cudaStream_t st) {
    const uint32_t nc = static_cast<uint32_t>((L.n + kChunk - 1) / kChunk);
    if (nc == 0) return cudaSuccess;
    K2Args a{p.push, p.slots, p.bounds, p.err, p.t, 0, 1, p.s_imm, p.rng_q0};
    k2_ternarize<SingleSource><<<nc, kThreads, 0, st>>>(SingleSource{L}, a);
    return launch_status();
}

cudaError_t launch_k2_offset(const float* g, uint64_t n, float s, uint32_t key0, uint32_t key1,
                             uint64_t t, uint64_t rng_base, uint8_t* codes, ErrWord* err,
                             cudaStream_t st) {
    const uint64_t nbytes = (n + 3) / 4;
    if (nbytes == 0) return cudaSuccess;
    const uint32_t blocks = static_cast<uint32_t>((nbytes + kThreads - 1) / kThreads);
    k2_ternarize_offset<<<blocks, kThreads, 0, st>>>(g, n, s, key0, key1, t, rng_base, codes, err);
    return launch_status();
}

cudaError_t launch_k3_table(const LayerDev* layers, const ChunkDev* chunks, uint32_t n_chunks,
                            const K3Launch& p, cudaStream_t st) {
    if (n_chunks == 0) return cudaSuccess;
    K3Args a{p.src, p.stride, nullptr, nullptr, 0.0f, p.n_workers, p.sharing, p.inv_n, p.err};
    K3Ptrs ptrs{};
    k3_decode<TableSource, true><<<n_chunks, kThreads, 0, st>>>(TableSource{layers, chunks}, a,
                                                                  ptrs);
    return launch_status();
}

cudaError_t launch_k3_single(const LayerDev& L, const uint8_t* const* codes, const float* scalers,
                             const K3Launch& p, cudaStream_t st) {
    const uint32_t nc = static_cast<uint32_t>((L.n + kChunk - 1) / kChunk);
    if (nc == 0) return cudaSuccess;
    K3Args a{nullptr, 0, nullptr, scalers, p.s_imm, p.n_workers, p.sharing, p.inv_n, p.err};
    K3Ptrs ptrs{};
    for (int w = 0; w < p.n_workers; ++w) ptrs.codes[w] = codes[w];
    k3_decode<SingleSource, false><<<nc, kThreads, 0, st>>>(SingleSource{L}, a, ptrs);
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

}  // namespace tgb
