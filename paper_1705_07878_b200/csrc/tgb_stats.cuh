// K1 building blocks: fp64 moment accumulation, partial emission and the
// deterministic per-layer merge + clip/scaler epilogue.
//
// Reference: stddev (codec.hpp:101-112, sequential fp64 two-pass), clip bound
// float(c*sigma) (:119), scaler = max |clip(g)| (:128-134) = min(max|g|, bound),
// Global bucketing max over tensors (:212-216). See DESIGN.md §K1 for why the
// parallel fp64 Chan merge reproduces the reference's float bound.
#pragma once

#include "tgb_device.cuh"
#include "tgb/terngrad_b200.h"

namespace tgb {

struct K1Out {
    Partial* partials;      // one per work unit (chunk), group-relative
    uint32_t* layer_done;   // per TENSOR arrival counters (self-resetting)
    uint32_t* global_done;  // arrival counter over tensors (Global bucketing)
    float* bounds;          // per block clip bound (the tensor's bound)
    float* slots;           // scaler slots
    ErrWord* err;
    float clip_factor;
    int32_t global_bucketing;
    int32_t n_layers;         // blocks (Global fix-up)
    int32_t n_active_layers;  // tensors that finalize (non-empty, ternary)
    const LayerDev* layers;   // block table (slots of a tensor's blocks, Global fix-up)
    PeerPush push;            // scaler slot destinations (n == 0: slots only)
    const TensorDev* tensors; // plan only; nullptr = single-block single-layer API
    unsigned long long* nnz = nullptr;  // telemetry counter of this group (reset by block 0)
    uint32_t keep_from = ~0u;  // units >= keep_from load with L2 evict_last (K2 re-reads them)
    // fused K1+K2 kernel: a finalized tensor's bound and scalers are published by a
    // release store of the launch's epoch into ready[tensor] (Global bucketing: into
    // *ready_global once the last tensor wrote the global max)
    uint32_t* ready = nullptr;
    uint32_t* ready_global = nullptr;
    uint32_t epoch = 0;
    // FixedSize plans: per-block max |x| (float bits, atomicMax), turned into the
    // bucket scalers by k1_bucket_slots; the tensor finalize then writes only the bound
    uint32_t* bmax = nullptr;
    // two-level finalize (tensors of > kK1GroupMin units): group partials and arrival
    // counters, TensorDev::group_base onwards per tensor (nullptr: one-level merge)
    Partial* gpart = nullptr;
    uint32_t* gdone = nullptr;
};

__device__ __forceinline__ void publish_ready(uint32_t* flag, uint32_t epoch) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

__device__ __forceinline__ void put_slot(const K1Out& o, int32_t slot, float v) {
    o.slots[slot] = v;
    for (int p = 0; p < o.push.n; ++p) reinterpret_cast<float*>(o.push.base[p])[slot] = v;
}

// x - x0 in fp64 (exact for any two floats within 2^29 of each other's exponent)
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

__device__ __forceinline__ void acc1(const float x, const double x0, double& S, double& Q,
                                     float& mx) {
    const double d = static_cast<double>(x) - x0;
    S += d;
    Q = fma(d, d, Q);
    mx = fmaxf(mx, fabsf(x));
}

// Block-wide fixed-order merge of nc partials at src: thread t merges its run
// [t*per, t*per + per) in index order (loads issued kB at a time), then a
// pairwise tree over the runs. The result lands in sn[0], smean[0], sm2[0], smx[0].
template <class Bar>
__device__ __forceinline__ void merge_partials(const Partial* src, uint32_t nc, double* sn,
                                               double* smean, double* sm2, float* smx) {
    const uint32_t tid = threadIdx.x;
    const uint32_t per = (nc + kThreads - 1) / kThreads;
    double n = 0.0, mean = 0.0, m2 = 0.0;
    float m = 0.0f;
    const uint32_t lo = tid * per, hi = min(nc, lo + per);
    uint32_t c = lo;
    constexpr uint32_t kB = 8;
    for (; c + kB <= hi; c += kB) {
        double bn[kB], bmean[kB], bm2[kB];
        float bmx[kB];
#pragma unroll
        for (uint32_t j = 0; j < kB; ++j) {
            const Partial* pp = src + c + j;
            bn[j] = __ldcg(&pp->n);
            bmean[j] = __ldcg(&pp->mean);
            bm2[j] = __ldcg(&pp->m2);
            bmx[j] = __ldcg(&pp->mx);
        }
#pragma unroll
        for (uint32_t j = 0; j < kB; ++j) {
            chan_merge(n, mean, m2, bn[j], bmean[j], bm2[j]);
            m = fmaxf(m, bmx[j]);
        }
    }
    for (; c < hi; ++c) {
        const Partial* pp = src + c;
        const double pn = __ldcg(&pp->n), pmean = __ldcg(&pp->mean), pm2 = __ldcg(&pp->m2);
        const float pmx = __ldcg(&pp->mx);
        chan_merge(n, mean, m2, pn, pmean, pm2);
        m = fmaxf(m, pmx);
    }
    sn[tid] = n;
    smean[tid] = mean;
    sm2[tid] = m2;
    smx[tid] = m;
    Bar::sync();
    const uint32_t runs = min(nc, static_cast<uint32_t>(kThreads));  // non-empty runs
    for (uint32_t s = 1; s < runs; s <<= 1) {
        if ((tid & (2 * s - 1)) == 0 && tid + s < runs) {
            double a_n = sn[tid], a_mean = smean[tid], a_m2 = sm2[tid];
            chan_merge(a_n, a_mean, a_m2, sn[tid + s], smean[tid + s], sm2[tid + s]);
            sn[tid] = a_n;
            smean[tid] = a_mean;
            sm2[tid] = a_m2;
            smx[tid] = fmaxf(smx[tid], smx[tid + s]);
        }
        Bar::sync();
    }
}

// Block-wide: reduce (S, Q, mx) of `count` elements shifted by x0, write the
// unit's partial, count the layer's arrivals; the last arriving unit merges
// the layer's partials [first, first + n_units) in a fixed order and writes
// bound + scaler. Must be called by every thread of the block.
// Tensors of more than kK1GroupMin units (with o.gpart) merge in two levels: the last
// unit of each group of kK1Group units merges the group (while the rest of the grid
// still streams), the last group merges the group partials -- one CTA merging all of
// a 3136-unit tensor's partials took ~15 us after the grid had drained
// (tools/k1_sets.py: VGG-16 fc6 alone 87.0 us vs 72.2 us without the merge).

template <class Bar = BlockBar>
__device__ __forceinline__ void k1_emit_and_finalize(const K1Out& o, const LayerDev& L,
                                                     uint32_t layer, uint32_t unit,
                                                     uint32_t first_unit, uint32_t n_units,
                                                     uint64_t count, double x0, double S, double Q,
                                                     float mx, bool bucket_max = true) {
    block_reduce_sq<kThreads / 32, Bar>(S, Q, mx);
    const uint32_t tid = threadIdx.x;
    __shared__ bool is_last;
    const bool grouped = o.gpart && o.tensors && n_units > kK1GroupMin;
    const uint32_t grp = (unit - first_unit) / kK1Group;
    const uint32_t n_grp = (n_units + kK1Group - 1) / kK1Group;
    if (tid == 0 && o.bmax && bucket_max)  // FixedSize: a chunk of one bucket
        atomicMax(o.bmax + layer, __float_as_uint(mx));
    if (tid == 0) {
        const double cn = static_cast<double>(count);
        Partial p;
        p.n = cn;
        p.mean = x0 + S / cn;
        p.m2 = Q - S * (S / cn);
        p.mx = mx;
        p.block = layer;
        o.partials[unit] = p;
        __threadfence();
        if (grouped) {
            const uint32_t gc = min(kK1Group, n_units - grp * kK1Group);
            const uint32_t gi = o.tensors[L.tensor].group_base + grp;
            is_last = atomicAdd(o.gdone + gi, 1u) == gc - 1;
        } else {
            const uint32_t ticket = atomicAdd(&o.layer_done[L.tensor], 1u);
            is_last = (ticket == n_units - 1);
        }
    }
    Bar::sync();
    if (!is_last) return;
#ifdef TGB_AB_NO_FINALIZE  // timing probe only (tools/k1_sets.py): the merge is skipped
    return;
#endif
    __threadfence();

    __shared__ double sn[kThreads], smean[kThreads], sm2[kThreads];
    __shared__ float smx[kThreads];
    const uint32_t nc = n_units;
    if (grouped) {
        const uint32_t gb = o.tensors[L.tensor].group_base;
        const uint32_t gc = min(kK1Group, n_units - grp * kK1Group);
        merge_partials<Bar>(o.partials + first_unit + grp * kK1Group, gc, sn, smean, sm2, smx);
        if (tid == 0) {
            Partial q;
            q.n = sn[0];
            q.mean = smean[0];
            q.m2 = sm2[0];
            q.mx = smx[0];
            q.block = layer;
            o.gpart[gb + grp] = q;
            o.gdone[gb + grp] = 0u;  // self-reset for the next launch
            __threadfence();
            is_last = atomicAdd(&o.layer_done[L.tensor], 1u) == n_grp - 1;
        }
        Bar::sync();
        if (!is_last) return;
        __threadfence();
        merge_partials<Bar>(o.gpart + gb, n_grp, sn, smean, sm2, smx);
    } else {
        merge_partials<Bar>(o.partials + first_unit, nc, sn, smean, sm2, smx);
    }
    __shared__ float s_bound;
    __shared__ bool s_bad;
    if (tid == 0) {
        const double fm = smean[0];
        double fm2 = sm2[0];
        const float fmx = smx[0];
        const uint64_t tn = o.tensors ? o.tensors[L.tensor].n : L.n;
        const bool clip = o.tensors ? (o.tensors[L.tensor].flags & kLayerClip) != 0
                                    : (L.flags & kLayerClip) != 0;
        float bound = INFINITY;
        s_bad = !isfinite(fm) || !isfinite(fm2) || !isfinite(fmx);
        if (s_bad) {
            raise_error(o.err, TGB_E_NONFINITE, static_cast<int32_t>(L.tensor), 0);
            bound = 0.0f;
        } else if (clip && tn >= 2) {
            if (fm2 < 0.0) fm2 = 0.0;
            const double sigma = sqrt(fm2 / static_cast<double>(tn));  // codec.hpp:111
            bound = static_cast<float>(static_cast<double>(o.clip_factor) * sigma);  // :119
        }
        s_bound = bound;
        if (!o.tensors) {  // single layer: one block
            o.bounds[0] = bound;
            put_slot(o, L.slot, s_bad ? 0.0f : fminf(fmx, bound));
        }
        o.layer_done[L.tensor] = 0u;  // self-reset for the next launch
    }
    Bar::sync();
    if (o.tensors && o.bmax) {  // FixedSize: the bucket scalers follow in k1_bucket_slots
        if (tid == 0) o.bounds[o.tensors[L.tensor].first_block] = s_bound;
    } else if (o.tensors) {
        // per block: s = max |clip(part)| = min(max |part|, bound) (codec.hpp:121-122, :229-230)
        const TensorDev T = o.tensors[L.tensor];
        if (T.n_blocks == 1) {  // PerTensor / Global: the tree's max is the block's
            if (tid == 0) {
                o.bounds[T.first_block] = s_bound;
                put_slot(o, o.layers[T.first_block].slot, s_bad ? 0.0f : fminf(smx[0], s_bound));
            }
        } else {
            // FixedSize buckets: a tensor's units are stored in block order and never
            // straddle a block, so every block is a contiguous run of units. The unit
            // that opens a run merges the run's maxima and writes the block's bound and
            // scaler: one O(units) pass spread over the CTA (the earlier windowed scan
            // re-read every unit once per 2048 blocks, O(units x blocks); VGG-16 at
            // k = 256: K1 26.1 ms, tools/fixed_probe.py)
            constexpr uint32_t kB = 4;  // units whose loads are issued together
            for (uint32_t c0 = tid; c0 < nc; c0 += kB * kThreads) {
                uint32_t bb[kB], bprev[kB], bnext[kB];
                float bmx[kB];
#pragma unroll
                for (uint32_t j = 0; j < kB; ++j) {
                    const uint32_t c = c0 + j * kThreads;
                    const Partial* pp = o.partials + first_unit + c;
                    bb[j] = c < nc ? __ldcg(&pp->block) : ~0u;
                    bprev[j] = (c > 0 && c < nc) ? __ldcg(&pp[-1].block) : ~1u;
                    bnext[j] = c + 1 < nc ? __ldcg(&pp[1].block) : ~1u;
                    bmx[j] = c < nc ? __ldcg(&pp->mx) : 0.0f;
                }
#pragma unroll
                for (uint32_t j = 0; j < kB; ++j) {
                    const uint32_t c = c0 + j * kThreads;
                    const uint32_t b = bb[j];
                    if (c >= nc || bprev[j] == b) continue;  // not the run's first unit
                    float bm = bmx[j];
                    if (bnext[j] == b) {  // block spans several units
                        const Partial* pp = o.partials + first_unit + c;
                        for (uint32_t d = c + 1; d < nc && __ldcg(&pp[d - c].block) == b; ++d)
                            bm = fmaxf(bm, __ldcg(&pp[d - c].mx));
                    }
                    o.bounds[b] = s_bound;
                    put_slot(o, o.layers[b].slot, s_bad ? 0.0f : fminf(bm, s_bound));
                }
            }
        }
        Bar::sync();
        if (tid == 0 && o.global_bucketing) {
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
                    put_slot(o, Ll.slot, gs);
                }
                *o.global_done = 0u;
                if (o.ready_global) publish_ready(o.ready_global, o.epoch);
            }
        }
        if (tid == 0 && o.ready && !o.global_bucketing) publish_ready(o.ready + L.tensor, o.epoch);
    }
}

}  // namespace tgb
