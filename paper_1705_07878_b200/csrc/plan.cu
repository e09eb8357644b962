// C-ABI, plan half (include/tgb/terngrad_b200.h): plan creation and work
// schedule, binding, the step schedules, the cross-GPU exchange (NCCL
// allgather, fused NVLink peer stores, sharded parameter server), attach-time
// plan validation and the single-process LocalCluster step. Host code only;
// kernels live in kernels.cu.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "tgb_plan.h"

using namespace tgb;

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

#define TGB_TRY(expr)                        \
    do {                                     \
        const tgb_status s_ = (expr);        \
        if (s_ != TGB_OK) return s_;         \
    } while (0)

namespace {

// Block model (EncodedGradient::blocks, codec.hpp:70-76, built by encode_step
// :218-236): a ternary tensor is one block (PerTensor / Global) or
// ceil(n/k) buckets (FixedSize, an empty tensor still one empty block); a
// passthrough tensor is one raw block.
constexpr uint64_t kMaxBlocks = 1ull << 24;  // plan tables stay < 1.5 GB

uint64_t fnv_mix(uint64_t h, uint64_t v) {
    for (int i = 0; i < 8; ++i) {
        h ^= (v >> (8 * i)) & 0xFFu;
        h *= 0x100000001b3ull;
    }
    return h;
}

// largest m with base^m <= 2^32: base-(2N+1) digits per u32 sums word
int32_t radix_digits_u32(uint64_t base) {
    int32_t m = 0;
    uint64_t acc = 1;
    while (acc * base <= 0x100000000ull) {
        acc *= base;
        ++m;
    }
    return m;
}

}  // namespace

namespace tgb {
uint8_t* own_push(const tgb_plan* P);
}

// ------------------------------------------------------------------ schedule
static tgb_status upload_tables(tgb_plan* P) {
    if (!P->h_tensors.empty())
        TGB_CUDA(cudaMemcpy(P->d_tensors, P->h_tensors.data(),
                            P->h_tensors.size() * sizeof(TensorDev), cudaMemcpyHostToDevice));
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
    return TGB_OK;
}

// Work items, layer groups, sharded owners and sums layout, from the block
// table and the plan options; (re)allocates the device tables to fit.
static tgb_status build_schedule(tgb_plan* P) {
    const int32_t n_layers = static_cast<int32_t>(P->desc.size());
    const tgb_layer_desc* layers = P->desc.data();
    const int N = P->n_workers;
    // elements per grid-per-chunk work item: K1/K2 amortise a heavier per-CTA
    // setup over 32K elements, K3 (store-bound) prefers 16K (tools/ab_bench.py).
    // Small gradient sets would leave most of the 148 SMs idle with 32K items, so
    // K1/K2 items shrink to give about one full wave (148 SMs x 3 CTAs): the
    // smallest power of two >= total/444, within [4K, 32K] (GoogLeNet 6.6M
    // elements: 16K, step 32.9 -> 27.0 us; a 1M layer: 4K, 21.7 -> 14.6 us).
    uint64_t chunk = 4096;
    while (chunk < kChunk12 && chunk * 444 < P->total) chunk <<= 1;
    if (P->chunk_opt) chunk = static_cast<uint64_t>(P->chunk_opt);
    P->chunk12 = static_cast<uint32_t>(chunk);
    P->chunk3 = kChunk3;
    // sharded exchange: by default from N >= 5 for sets of >= 16 Mi elements, where
    // the fused exchange's (N-1)/4 B per element of NVLink traffic dominates (measured
    // at N = 4 the fused two-group schedule still wins); small sets
    // are latency-bound and the sharded path's second cross-GPU barrier only costs
    P->shard = false;
    if (N >= 2 && N <= kMaxPeers && P->p.scaler_sharing)
        P->shard = P->exchange_opt == TGB_EXCHANGE_SHARDED ||
                   (P->exchange_opt == TGB_EXCHANGE_AUTO && N >= 5 && P->total >= (16ull << 20));

    // ---- FixedSize(k), k = 2^p in [64, chunk): work items of whole buckets (k/4 code
    // bytes, a 16-B multiple, so a run of buckets is contiguous in the push area and
    // the slots; shared scalers and N <= 8: the staged decode kernels)
    P->mb_log2 = 0;
    const uint64_t k = P->p.bucket_size;
    if (P->p.bucketing == TGB_BUCKET_FIXED && k >= 64 && (k & (k - 1)) == 0 && k < chunk &&
        P->p.scaler_sharing && N <= kMaxPeers) {
        while ((1ull << P->mb_log2) < k) ++P->mb_log2;
    }
    for (LayerDev& L : P->h_layers) {
        L.flags &= ~(kLayerMultiBucket | (31u << kBucketShiftBit));
        const TensorDev& T = P->h_tensors[L.tensor];
        if (P->mb_log2 && !(L.flags & kLayerPassthrough) && T.n_blocks > 1)
            L.flags |= kLayerMultiBucket | (P->mb_log2 << kBucketShiftBit);
    }

    // ---- work items (chunks never straddle blocks; multi-bucket items span whole blocks)
    P->h_chunks.clear();
    P->h_chunks3.clear();
    const uint32_t nb = static_cast<uint32_t>(P->h_layers.size());
    for (uint32_t b = 0; b < nb;) {
        const LayerDev& L = P->h_layers[b];
        if (L.flags & kLayerMultiBucket) {  // the tensor's blocks, grouped
            const TensorDev& T = P->h_tensors[L.tensor];
            const uint32_t end = T.first_block + T.n_blocks;
            for (int which = 0; which < 2; ++which) {
                const uint32_t per = static_cast<uint32_t>((which == 0 ? chunk : kChunk3) >> P->mb_log2);
                std::vector<ChunkDev>& out = which == 0 ? P->h_chunks : P->h_chunks3;
                for (uint32_t f = b; f < end;) {
                    if (per >= 2) {
                        const uint32_t m = std::min(per, end - f);
                        uint64_t cnt = 0;
                        for (uint32_t x = f; x < f + m; ++x) cnt += P->h_layers[x].n;
                        out.push_back({f, static_cast<uint32_t>(cnt), 0u, m});
                        f += m;
                    } else {  // buckets larger than a K3 item: chunks inside each block
                        const uint64_t n = P->h_layers[f].n;
                        for (uint64_t e = 0; e < n; e += kChunk3)
                            out.push_back({f, static_cast<uint32_t>(std::min<uint64_t>(kChunk3, n - e)),
                                           static_cast<uint32_t>(e), 1u});
                        ++f;
                    }
                }
            }
            b = end;
            continue;
        }
        const uint64_t n = L.n;
        for (uint64_t e = 0; e < n; e += chunk)
            P->h_chunks.push_back({b, static_cast<uint32_t>(std::min<uint64_t>(chunk, n - e)),
                                   static_cast<uint32_t>(e), 1u});
        for (uint64_t e = 0; e < n; e += kChunk3)
            P->h_chunks3.push_back({b, static_cast<uint32_t>(std::min<uint64_t>(kChunk3, n - e)),
                                    static_cast<uint32_t>(e), 1u});
        ++b;
    }

    // ---- two-group schedule: the dominant tensor vs the rest (PerTensor + REF
    // only: Global and PRESHARED need every tensor's K1 before any K2)
    int32_t big = -1;
    for (int32_t l = 0; l < n_layers; ++l)
        if (!(layers[l].flags & TGB_LAYER_PASSTHROUGH) && (big < 0 || layers[l].n > layers[big].n))
            big = l;
    // (the sharded exchange runs each group as one piece: pieces_opt > 1 keeps it ungrouped)
    const bool can_group = !(P->shard && P->pieces_opt > 1) && big >= 0 && n_layers > 1 &&
                           P->p.bucketing == TGB_BUCKET_PER_TENSOR &&
                           P->p.share_mode == TGB_SHARE_REF;
    // overlapped exchange: N > 1, REF (PRESHARED's allreduce sits between K1 and K2)
    P->overlap = N > 1 && N <= kMaxPeers && P->p.share_mode == TGB_SHARE_REF &&
                 P->overlap_opt == 1;
    // split exchange (fused exchange, shared scalers: the staged decode; no multi-bucket
    // items): K3 pulls pull_opt/8 of the code items from the peers' own areas
    P->pull8 = (N > 1 && N <= kMaxPeers && !P->shard && !P->overlap && P->p.scaler_sharing &&
                P->mb_log2 == 0)
                   ? static_cast<uint32_t>(P->pull_opt)
                   : 0u;
    bool want = can_group && !P->overlap && layers[big].n * 100 >= P->total * 35 &&
                layers[big].n * 100 <= P->total * 95;
    if (P->schedule_opt == TGB_SCHEDULE_SINGLE || P->schedule_opt == TGB_SCHEDULE_UNFUSED ||
        P->schedule_opt == TGB_SCHEDULE_FUSED12)
        want = false;
    if (P->schedule_opt == TGB_SCHEDULE_GROUPS) want = can_group && !P->overlap;
    P->grouped = want;
    P->big = big;
    // K2 as K1's programmatic dependent on single-stream N = 1 plans (tools/env_ab.py,
    // profiles/r01_pdl_l2keep_ab.log): GoogLeNet 31.9 -> 29.1 us with a whole-chunk L2
    // prefetch before the wait, a 2^24 layer 49.6 -> 46.5 us without one, 2^26 / 2^28
    // layers 155 -> 149 / 546 -> 538 us prefetching the first 32 KB (a whole-chunk
    // prefetch re-reads evicted lines there: 159 / 575 us). With two concurrent groups the
    // waiting K2 CTAs hold SM slots the other group's K1 needs (VGG-16 +10 %): off.
    P->pdl = (P->grouped || N > 1) ? 0
             : P->total <= (8ull << 20) ? 2 : P->total >= (48ull << 20) ? 3 : 1;
    // N = 1: K1 loads its last 24 MB per launch L2 evict_last, K2 (walking chunks
    // last-to-first) re-reads them from L2 and demotes them (tools/l2keep_ab.py: step
    // -4.6 us; 16-32 MB is the plateau). At N > 1 the lines linger into K3 (+8 us).
#ifndef TGB_AB_NO_KEEP  // (same-box A/B builds only, tools/build_variant.sh)
    P->k1_keep = N == 1 ? static_cast<uint32_t>((24ull << 20) / (4ull * P->chunk12)) : 0u;
#else
    P->k1_keep = 0;
#endif
    // K1 + K2 as one persistent launch (opt-in, TGB_SCHEDULE_FUSED12): K2 of a tensor
    // starts as soon as its K1 finalized. Measured slower than K1 -> K2 with K2 as
    // K1's programmatic dependent, also for small sets (CUDA-graph replay, device
    // time: GoogLeNet 25.8 vs 24.0 us, a 1M layer 13.8 vs 12.3 us, VGG-16 305 vs
    // 284 us; profiles/r02_small_sets.jsonl). PRESHARED needs the allreduce between.
    P->k12 = !P->grouped && P->p.share_mode == TGB_SHARE_REF &&
             P->p.bucketing != TGB_BUCKET_FIXED && P->schedule_opt == TGB_SCHEDULE_FUSED12;
    if (P->k12) P->pdl = 0;

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
    for (int g = 0; g < 2; ++g) P->cb[g] = P->cc[g] = P->ck1[g] = P->cb3[g] = P->cc3[g] = 0;
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
        L.sum_off16 = 0;
    }
    // K1 two-level finalize: group slots of the tensors with more than kK1GroupMin units
    uint32_t n_gslots = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
        P->h_tensors[l].group_base = n_gslots;
        if (tunits[l].y > kK1GroupMin) n_gslots += (tunits[l].y + kK1Group - 1) / kK1Group;
    }
    if (n_gslots > P->gpart_cap) {
        cudaFree(P->d_gpart);
        cudaFree(P->d_gdone);
        P->d_gpart = nullptr;
        P->d_gdone = nullptr;
        TGB_CUDA(cudaMalloc(&P->d_gpart, n_gslots * sizeof(Partial)));
        TGB_CUDA(cudaMalloc(&P->d_gdone, n_gslots * sizeof(uint32_t)));
        TGB_CUDA(cudaMemset(P->d_gdone, 0, n_gslots * sizeof(uint32_t)));
        P->gpart_cap = n_gslots;
    }

    // ---- sharded exchange: sums regions and chunk owners. A ternary K2 chunk's
    // biased sums N + sum_w code_w in [0, 2N] are packed as base-(2N+1) digits,
    // radix_m per u32 word (the reference's SharedSumBlock packing, wire.hpp:103-145,
    // in 32-bit words so a chunk's region is self-contained): every full chunk's
    // region is sum_region bytes; passthrough chunks hold the raw fp32 means.
    P->radix_m = 0;
    P->sum_region = 0;
    P->sums_bytes = 0;
    P->n_pieces = 1;
    std::memset(P->pb, 0, sizeof(P->pb));
    std::memset(P->pcs, 0, sizeof(P->pcs));
    std::memset(P->p3, 0, sizeof(P->p3));
    if (P->overlap && !P->shard) {
        // pieces of the K2 list by elements (auto: 4), and the K3 items re-listed in K2
        // order so that each piece's decode items are one contiguous range
        std::vector<uint64_t> cum(P->h_chunks.size() + 1, 0);
        for (size_t c = 0; c < P->h_chunks.size(); ++c) cum[c + 1] = cum[c] + P->h_chunks[c].count;
        int np = P->pieces_opt > 0 ? P->pieces_opt : 4;
        np = std::max(1, std::min(np, std::min(kMaxPieces, static_cast<int>(P->h_chunks.size()))));
        P->n_pieces = np;
        for (int q = 0; q <= np; ++q)
            P->pb[q] = static_cast<uint32_t>(
                std::lower_bound(cum.begin(), cum.end(), cum.back() * q / np) - cum.begin());
        P->pb[np] = static_cast<uint32_t>(P->h_chunks.size());
        P->h_chunks3.clear();
        int q = 0;
        for (uint32_t c = 0; c < P->h_chunks.size(); ++c) {
            while (q < np && c >= P->pb[q]) P->p3[q++] = static_cast<uint32_t>(P->h_chunks3.size());
            const ChunkDev& ch = P->h_chunks[c];
            if (ch.nblk > 1) {  // multi-bucket item: K3 items of whole buckets
                const uint32_t per = static_cast<uint32_t>(kChunk3 >> P->mb_log2);
                for (uint32_t f = ch.layer; f < ch.layer + ch.nblk;) {
                    if (per >= 2) {
                        const uint32_t m = std::min(per, ch.layer + ch.nblk - f);
                        uint64_t cnt = 0;
                        for (uint32_t x = f; x < f + m; ++x) cnt += P->h_layers[x].n;
                        P->h_chunks3.push_back({f, static_cast<uint32_t>(cnt), 0u, m});
                        f += m;
                    } else {
                        const uint64_t n = P->h_layers[f].n;
                        for (uint64_t e = 0; e < n; e += kChunk3)
                            P->h_chunks3.push_back(
                                {f, static_cast<uint32_t>(std::min<uint64_t>(kChunk3, n - e)),
                                 static_cast<uint32_t>(e), 1u});
                        ++f;
                    }
                }
                continue;
            }
            for (uint64_t e = 0; e < ch.count; e += kChunk3)
                P->h_chunks3.push_back({ch.layer, static_cast<uint32_t>(std::min<uint64_t>(
                                                      kChunk3, ch.count - e)),
                                        static_cast<uint32_t>(ch.begin + e), 1u});
        }
        while (q <= np) P->p3[q++] = static_cast<uint32_t>(P->h_chunks3.size());
        P->cb3[0] = 0;
        P->cc3[0] = static_cast<uint32_t>(P->h_chunks3.size());
    }
    if ((P->overlap || P->shard) && !P->gs3) {
        int lo = 0, hi = 0;
        TGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        TGB_CUDA(cudaStreamCreateWithPriority(&P->gs3, cudaStreamNonBlocking, hi));
        TGB_CUDA(cudaEventCreateWithFlags(&P->ev_done, cudaEventDisableTiming));
        if (!P->ev_fork) TGB_CUDA(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
        for (int q = 0; q < kMaxPieces; ++q)
            TGB_CUDA(cudaEventCreateWithFlags(&P->ev_piece[q], cudaEventDisableTiming));
    }
    if ((P->overlap || P->shard) && !P->d_piece_cnt) {
        TGB_CUDA(cudaMalloc(&P->d_piece_cnt, kMaxPieces * sizeof(uint32_t)));
        TGB_CUDA(cudaMemset(P->d_piece_cnt, 0, kMaxPieces * sizeof(uint32_t)));
    }
    if (P->shard) {
        P->radix_m = radix_digits_u32(2ull * N + 1);
        const uint64_t m = static_cast<uint64_t>(P->radix_m);
        P->sum_region = static_cast<uint32_t>(round_up((chunk + m - 1) / m * 4, kAlignCodes));
        uint64_t so = 0;
        for (LayerDev& L : P->h_layers) {
            L.sum_off16 = static_cast<uint32_t>(so / 16);
            uint64_t bytes;
            if (L.flags & kLayerPassthrough) {
                bytes = 4ull * L.n;
            } else {
                const uint64_t full = L.n / chunk, rem = L.n % chunk;
                bytes = full * P->sum_region + round_up((rem + m - 1) / m * 4, kAlignCodes);
            }
            so += round_up(bytes, kAlignCodes);
        }
        P->sums_bytes = round_up(std::max<uint64_t>(so, 1), kAlignPush);
        // pieces: contiguous runs of the K2 chunk list, balanced by K3a bytes (raw fp32 =
        // 16x codes). auto = 1: measured on 4 B200s (VGG-16, profiles/r02_sharded_pieces.json)
        // 1 / 2 / 4 / 8 pieces = 0.444 / 0.455 / 0.539 / 0.707 ms -- every piece adds two
        // cross-GPU barriers and a K2 tail wave, and the per-piece K3a -> barrier -> K3b chain
        // on the second stream is longer than the K2 piece it should hide behind
        std::vector<uint64_t> cum(P->h_chunks.size() + 1, 0);
        for (size_t c = 0; c < P->h_chunks.size(); ++c)
            cum[c + 1] = cum[c] + P->h_chunks[c].count * (is_pass(P->h_chunks[c]) ? 16ull : 1ull);
        const uint64_t W = cum.back();
        int np = P->pieces_opt > 0 ? P->pieces_opt : (P->overlap ? 4 : 1);
        np = std::max(1, std::min(np, std::min(kMaxPieces, static_cast<int>(P->h_chunks.size()))));
        if (P->grouped) np = 2;  // piece g = layer group g (each runs on its own stream)
        P->n_pieces = np;
        auto cut = [&](uint64_t target) {
            return static_cast<uint32_t>(std::lower_bound(cum.begin(), cum.end(), target) -
                                         cum.begin());
        };
        for (int q = 0; q <= np; ++q) P->pb[q] = cut(W * static_cast<uint64_t>(q) / np);
        if (P->grouped) P->pb[1] = P->cb[1];
        P->pb[np] = static_cast<uint32_t>(P->h_chunks.size());
        // owners inside each piece: rank r owns [pcs[q][r], pcs[q][r+1])
        for (int q = 0; q < np; ++q) {
            const uint64_t w0 = cum[P->pb[q]], w1 = cum[P->pb[q + 1]];
            for (int r = 0; r <= N; ++r)
                P->pcs[q][r] = std::max(P->pb[q], cut(w0 + (w1 - w0) * static_cast<uint64_t>(r) / N));
            P->pcs[q][N] = P->pb[q + 1];
            for (int r = N + 1; r <= kMaxPeers; ++r) P->pcs[q][r] = P->pb[q + 1];
        }
    }

    if (P->grouped && !P->gs[0]) {
        // the dominant layer's chain (K1 -> K2 -> K3 of the big layer) is the critical
        // path: it runs at high priority and the rest fills the gaps
        int lo = 0, hi = 0;
        TGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        TGB_CUDA(cudaStreamCreateWithPriority(&P->gs[0], cudaStreamNonBlocking, lo));
        TGB_CUDA(cudaStreamCreateWithPriority(&P->gs[1], cudaStreamNonBlocking, hi));
        TGB_CUDA(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
        TGB_CUDA(cudaEventCreateWithFlags(&P->ev_join[0], cudaEventDisableTiming));
        TGB_CUDA(cudaEventCreateWithFlags(&P->ev_join[1], cudaEventDisableTiming));
    }
    const size_t nc = std::max<size_t>(1, P->h_chunks.size());
    const size_t nc3 = std::max<size_t>(1, P->h_chunks3.size());
    if (P->fat_cap < nc) {
        cudaFree(P->d_fat);
        cudaFree(P->d_partials);
        P->d_fat = nullptr;
        P->d_partials = nullptr;
        TGB_CUDA(cudaMalloc(&P->d_fat, nc * sizeof(ChunkFat)));
        TGB_CUDA(cudaMalloc(&P->d_partials, nc * sizeof(Partial)));
        P->fat_cap = nc;
    }
    if (P->fat3_cap < nc3) {
        cudaFree(P->d_fat3);
        P->d_fat3 = nullptr;
        TGB_CUDA(cudaMalloc(&P->d_fat3, nc3 * sizeof(ChunkFat)));
        P->fat3_cap = nc3;
    }
    return upload_tables(P);
}

extern "C" {

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
    P->worker = worker;
    P->n_workers = n_workers;
    P->desc.assign(layers, layers + n_layers);
    if (cudaGetDevice(&P->device) != cudaSuccess || preload_kernels() != cudaSuccess) {
        cudaGetLastError();
        delete P;
        return TGB_ERR_CUDA;
    }

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

    const size_t nl = std::max<size_t>(1, n_layers);
    const size_t nbl = std::max<size_t>(1, P->h_layers.size());
    bool ok = cudaMalloc(&P->d_layers, nbl * sizeof(LayerDev)) == cudaSuccess &&
              cudaMalloc(&P->d_tensors, nl * sizeof(TensorDev)) == cudaSuccess &&
              cudaMalloc(&P->d_counters, (nl + 1) * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&P->d_bounds, nbl * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&P->d_push, P->push_bytes) == cudaSuccess &&
              cudaMalloc(&P->d_err, sizeof(ErrWord)) == cudaSuccess &&
              cudaMalloc(&P->d_ready, (nl + 2) * sizeof(uint32_t)) == cudaSuccess &&
              cudaMemset(P->d_ready, 0, (nl + 2) * sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&P->d_nnz, 2 * sizeof(unsigned long long)) == cudaSuccess &&
              cudaMemset(P->d_nnz, 0, 2 * sizeof(unsigned long long)) == cudaSuccess;
    if (ok && params->bucketing == TGB_BUCKET_FIXED) {  // bucket maxima + block meta
        std::vector<uint2> meta(nbl, make_uint2(0u, ~0u));
        for (size_t b = 0; b < P->h_layers.size(); ++b) {
            const LayerDev& L = P->h_layers[b];
            meta[b] = make_uint2(L.tensor, L.slot < 0 ? ~0u : static_cast<uint32_t>(L.slot));
        }
        ok = cudaMalloc(&P->d_bmax, nbl * sizeof(uint32_t)) == cudaSuccess &&
             cudaMemset(P->d_bmax, 0, nbl * sizeof(uint32_t)) == cudaSuccess &&
             cudaMalloc(&P->d_bmeta, nbl * sizeof(uint2)) == cudaSuccess &&
             cudaMemcpy(P->d_bmeta, meta.data(), nbl * sizeof(uint2), cudaMemcpyHostToDevice) ==
                 cudaSuccess;
    }
    if (ok && n_workers > 1) {  // NCCL allgather destination (freed when peers attach)
        ok = cudaMalloc(&P->d_nccl_gather, P->push_bytes * static_cast<uint64_t>(n_workers)) ==
             cudaSuccess;
        P->d_gathered = P->d_nccl_gather;
    }
    const std::vector<float> inf_bounds(nbl, INFINITY);  // empty / unclipped: no clip (codec.hpp:118)
    ok = ok && cudaMemset(P->d_counters, 0, (nl + 1) * sizeof(uint32_t)) == cudaSuccess &&
         cudaMemset(P->d_push, 0, P->push_bytes) == cudaSuccess &&
         cudaMemset(P->d_err, 0, sizeof(ErrWord)) == cudaSuccess &&
         cudaMemcpy(P->d_bounds, inf_bounds.data(), nbl * sizeof(float), cudaMemcpyHostToDevice) ==
             cudaSuccess;
    if (ok && n_layers > 0)
        ok = cudaMemcpy(P->d_tensors, P->h_tensors.data(), n_layers * sizeof(TensorDev),
                        cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok || build_schedule(P) != TGB_OK) {
        cudaGetLastError();
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
    cudaFree(P->d_layers);
    cudaFree(P->d_tensors);
    cudaFree(P->d_gpart);
    cudaFree(P->d_gdone);
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
    cudaFree(P->d_nccl_gather);
    cudaFree(P->d_nnz);
    cudaFree(P->d_optd);
    cudaFree(P->d_frame);
    cudaFree(P->d_wsegs);
    cudaFree(P->d_pull);
    cudaFree(P->d_err);
    cudaFree(P->d_ready);
    cudaFree(P->d_bmax);
    cudaFree(P->d_bmeta);
    cudaFree(P->d_piece_cnt);
    for (int g = 0; g < 2; ++g) {
        if (P->gs[g]) cudaStreamDestroy(P->gs[g]);
        if (P->ev_join[g]) cudaEventDestroy(P->ev_join[g]);
    }
    if (P->ev_fork) cudaEventDestroy(P->ev_fork);
    if (P->gs3) cudaStreamDestroy(P->gs3);
    if (P->ev_done) cudaEventDestroy(P->ev_done);
    for (cudaEvent_t e : P->ev_piece)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : P->ev_local)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : P->t_ev) cudaEventDestroy(e);
    if (P->s_h2d) cudaStreamDestroy(P->s_h2d);
    if (P->s_d2h) cudaStreamDestroy(P->s_d2h);
    if (P->ev_h2d) cudaEventDestroy(P->ev_h2d);
    if (P->ev_comp) cudaEventDestroy(P->ev_comp);
    if (P->ev_d2h) cudaEventDestroy(P->ev_d2h);
    for (int g = 0; g < 2; ++g) {
        if (P->ev_hg[g]) cudaEventDestroy(P->ev_hg[g]);
        if (P->ev_cg[g]) cudaEventDestroy(P->ev_cg[g]);
        if (P->ev_dg[g]) cudaEventDestroy(P->ev_dg[g]);
    }
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

tgb_status tgb_plan_set_option(tgb_plan* P, int32_t option, int64_t value) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    switch (option) {
        case TGB_PLAN_OPT_SCHEDULE:
            if (value < TGB_SCHEDULE_AUTO || value > TGB_SCHEDULE_FUSED12)
                return TGB_ERR_INVALID_ARGUMENT;
            if (P->attached) return TGB_ERR_UNSUPPORTED;  // ranks agreed on it at attach
            P->schedule_opt = static_cast<int32_t>(value);
            break;
        case TGB_PLAN_OPT_EXCHANGE:
            if (value != TGB_EXCHANGE_AUTO && value != TGB_EXCHANGE_FUSED &&
                value != TGB_EXCHANGE_SHARDED)
                return TGB_ERR_INVALID_ARGUMENT;
            if (P->attached) return TGB_ERR_UNSUPPORTED;
            if (value == TGB_EXCHANGE_SHARDED &&
                (!P->p.scaler_sharing || P->n_workers < 2 || P->n_workers > kMaxPeers))
                return TGB_ERR_UNSUPPORTED;  // the owner sums integer codes (shared scalers)
            P->exchange_opt = static_cast<int32_t>(value);
            break;
        case TGB_PLAN_OPT_CHUNK:
            if (value != 0 && (value < 1024 || value > kChunk12 || (value & (value - 1))))
                return TGB_ERR_INVALID_ARGUMENT;
            if (P->attached) return TGB_ERR_UNSUPPORTED;
            P->chunk_opt = static_cast<int32_t>(value);
            break;
        case TGB_PLAN_OPT_OVERLAP:
            if (value < -1 || value > 1) return TGB_ERR_INVALID_ARGUMENT;
            if (P->attached) return TGB_ERR_UNSUPPORTED;
            P->overlap_opt = static_cast<int32_t>(value);
            break;
        case TGB_PLAN_OPT_PIECES:
            if (value < 0 || value > kMaxPieces) return TGB_ERR_INVALID_ARGUMENT;
            if (P->attached) return TGB_ERR_UNSUPPORTED;
            P->pieces_opt = static_cast<int32_t>(value);
            break;
        case TGB_PLAN_OPT_PULL:
            if (value < 0 || value > 8) return TGB_ERR_INVALID_ARGUMENT;
            if (P->attached) return TGB_ERR_UNSUPPORTED;
            P->pull_opt = static_cast<int32_t>(value);
            break;
        case TGB_PLAN_OPT_FUSED_OPTIMIZER:
            if (value != 0 && value != 1) return TGB_ERR_INVALID_ARGUMENT;
            P->opt_fused = value != 0;
            return TGB_OK;
        default:
            return TGB_ERR_INVALID_ARGUMENT;
    }
    int prev = 0;
    TGB_CUDA(cudaGetDevice(&prev));
    TGB_CUDA(cudaSetDevice(P->device));
    const tgb_status s = build_schedule(P);
    cudaSetDevice(prev);
    return s;
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
    TGB_TRY(upload_tables(P));
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

}  // extern "C"

// attached plans: this rank's push area in rank p's gather buffer of the
// current parity
static inline uint8_t* push_area(const tgb_plan* P, int p) {
    const uint64_t g = P->push_bytes * static_cast<uint64_t>(P->n_workers);
    return P->peer_ipc[p] + (P->epoch & 1u) * g + static_cast<uint64_t>(P->rank) * P->push_bytes;
}
namespace tgb {
uint8_t* own_push(const tgb_plan* P) { return P->attached ? push_area(P, P->rank) : P->d_push; }
uint8_t* cur_gathered(const tgb_plan* P) {
    if (P->attached)
        return P->d_ipc + (P->epoch & 1u) * P->push_bytes * static_cast<uint64_t>(P->n_workers);
    return P->n_workers > 1 ? P->d_gathered : P->d_push;
}
}  // namespace tgb

static inline int n_groups(const tgb_plan* P) { return P->grouped ? 2 : 1; }

// ---- live kernel timing: events around each launch on its own stream
// host form of pulled_item (kernels.cu)
static bool pulled(const tgb_plan* P, const ChunkDev& ch) {
    return P->pull8 && !(P->h_layers[ch.layer].flags & (kLayerPassthrough | kLayerMultiBucket)) &&
           ((ch.layer + (ch.begin >> 15)) & 7u) < P->pull8;
}

// elements of chunks [b, b + c): out[0] ternary, out[1] passthrough, out[2] pulled
static void chunk_elems(const tgb_plan* P, const std::vector<ChunkDev>& chs, uint32_t b,
                        uint32_t c, uint64_t out[3]) {
    out[0] = out[1] = out[2] = 0;
    for (uint32_t i = b; i < b + c && i < chs.size(); ++i) {
        out[(P->h_layers[chs[i].layer].flags & kLayerPassthrough) ? 1 : 0] += chs[i].count;
        if (pulled(P, chs[i])) out[2] += chs[i].count;
    }
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

// ---- per-group launches (group g = chunk ranges cb/cc, cb3/cc3; an ungrouped
// plan is the single group 0 spanning every chunk)
static tgb_status launch_stats(tgb_plan* P, int g, cudaStream_t st) {
    const uint32_t b = P->cb[g];
    K1Launch k{P->d_partials + b, P->d_counters,
               P->d_counters + P->desc.size(), P->d_bounds,
               reinterpret_cast<float*>(own_push(P)), P->d_err, P->p.clip_factor,
               P->p.bucketing == TGB_BUCKET_GLOBAL, static_cast<int32_t>(P->h_layers.size()),
               P->n_active};
    // PRESHARED: the local scalers land in every peer's gather buffer from K1 (the
    // LocalCluster max reads them there); REF: K2 stores them (K2Args::slot_push)
    if (P->attached && P->p.share_mode == TGB_SHARE_PRESHARED) {
        k.push.n = 0;
        for (int p = 0; p < P->n_workers; ++p)
            if (p != P->rank) k.push.base[k.push.n++] = push_area(P, p);
        k.push.remote = 1;
    }
    k.keep_chunks = P->k1_keep;
    k.tensors = P->d_tensors;
    k.gpart = P->d_gpart;
    k.gdone = P->d_gdone;
    k.nnz = P->code_stats ? P->d_nnz + g : nullptr;
    k.bmax = P->d_bmax;
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k1_table(P->d_layers, P->d_fat + b, P->ck1[g], k, st));
    if (P->d_bmax)  // FixedSize: bucket scalers (FixedSize plans are never grouped)
        TGB_CUDA(launch_k1_bucket_slots(P->d_layers, P->d_bmeta,
                                        static_cast<uint32_t>(P->h_layers.size()), k, st));
    if (ts >= 0) {
        uint64_t e[3];
        chunk_elems(P, P->h_chunks, b, P->ck1[g], e);
        t_end(P, st, ts, TGB_KERNEL_K1, g, e[0], 4 * e[0], 0);
    }
    return TGB_OK;
}

// K2 over chunks [cb, cb + cc); piece: the sharded piece these chunks are (owner
// bounds relative to cb), or -1 for a whole group
static tgb_status launch_tern_range(tgb_plan* P, int g, uint32_t cb, uint32_t cc, int piece,
                                    uint64_t t, cudaStream_t st, bool fuse_decode) {
    uint8_t* own = own_push(P);
    K2Launch k{own, reinterpret_cast<const float*>(own), P->d_bounds, P->d_err, t, 1};
    k.fuse_decode = fuse_decode ? 1 : 0;
    k.nnz = P->code_stats ? P->d_nnz + g : nullptr;
    if (fuse_decode && P->opt_active) {
        k.optd = P->d_optd;
        k.opt = *P->opt_active;
    }
    k.pdl = P->pdl;
    if (P->k1_keep) k.keep_from = P->ck1[g] - std::min(P->k1_keep, P->ck1[g]);
    if (P->attached) {  // fused exchange: codes stored into every rank's gather buffer
        for (int p = 0; p < P->n_workers; ++p) k.dst.base[p] = push_area(P, p);
        k.dst.n = P->n_workers;
        k.dst.remote = 1;
        k.pull8 = P->pull8;
        k.rank = P->rank;
        k.slot_push = P->p.share_mode == TGB_SHARE_PRESHARED ? 0 : 1;
        if (P->shard) {
            k.shard_n = P->n_workers;
            if (piece >= 0)
                for (int r = 0; r <= kMaxPeers; ++r) k.shard_bounds[r] = P->pcs[piece][r] - cb;
        }
        if (P->overlap) {  // one launch over the whole list; pieces published from inside K2
            k.reverse = 0;
            k.n_pieces = P->n_pieces;
            for (int q = 0; q <= kMaxPieces; ++q) k.piece_bounds[q] = P->pb[q] - cb;
            for (int q = 0; q < kMaxPieces; ++q)
                for (int r = 0; r <= kMaxPeers; ++r) k.owner_bounds[q][r] = P->pcs[q][r] - cb;
            k.piece_cnt = P->d_piece_cnt;
            for (int p = 0; p < P->n_workers; ++p)
                k.flag_remote[p] = reinterpret_cast<uint64_t*>(P->peer_ipc[p] + P->flags_off) +
                                   2 * P->rank;
            k.n_flags = P->n_workers;
            k.epoch = P->epoch;
        }
    }
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k2_table(P->d_layers, P->d_fat + cb, cc, k, st));
    if (ts >= 0) {
        uint64_t e[3];
        chunk_elems(P, P->h_chunks, cb, cc, e);
        const uint64_t nt = e[0], np = e[1], N = P->n_workers;
        const uint64_t msg = (nt + 3) / 4 + 4 * np;  // code bytes + raw passthrough bytes
        uint64_t own_b = msg, nvl = 0;
        if (P->attached && P->shard) {
            own_b = msg / N;
            nvl = msg - own_b;
        } else if (P->attached) {
            nvl = (N - 1) * (msg - e[2] / 4);  // pulled items stay local
        }
        const uint64_t out = fuse_decode ? 4 * (nt + np) : 0;
        t_end(P, st, ts, TGB_KERNEL_K2, g, nt + np, 4 * (nt + np) + own_b + out, nvl);
    }
    return TGB_OK;
}

// K2 of group g (the sharded exchange without overlap: one launch per piece)
static tgb_status launch_tern(tgb_plan* P, int g, uint64_t t, cudaStream_t st,
                              bool fuse_decode = false) {
    if (P->attached && P->overlap) return launch_tern_range(P, 0, 0, P->cc[0], -1, t, st, false);
    if (P->attached && P->shard) {
        for (int q = 0; q < P->n_pieces; ++q)
            TGB_TRY(launch_tern_range(P, 0, P->pb[q], P->pb[q + 1] - P->pb[q], q, t, st, false));
        return TGB_OK;
    }
    return launch_tern_range(P, g, P->cb[g], P->cc[g], -1, t, st, fuse_decode);
}

// fused K1 + K2 over the whole (ungrouped) plan: one persistent launch
static tgb_status launch_k12(tgb_plan* P, uint64_t t, cudaStream_t st, bool fuse_decode) {
    uint8_t* own = own_push(P);
    K1Launch k1{P->d_partials, P->d_counters, P->d_counters + P->desc.size(), P->d_bounds,
                reinterpret_cast<float*>(own), P->d_err, P->p.clip_factor,
                P->p.bucketing == TGB_BUCKET_GLOBAL, static_cast<int32_t>(P->h_layers.size()),
                P->n_active};
    K2Launch k2{own, reinterpret_cast<const float*>(own), P->d_bounds, P->d_err, t, 0};
    if (P->attached) {
        k1.push.n = 0;
        for (int p = 0; p < P->n_workers; ++p) {
            if (p != P->rank) k1.push.base[k1.push.n++] = push_area(P, p);
            k2.dst.base[p] = push_area(P, p);
        }
        k1.push.remote = 1;
        k2.dst.n = P->n_workers;
        k2.dst.remote = 1;
        if (P->shard) {  // (the fused K1+K2 launch covers the whole list: one piece)
            if (P->n_pieces != 1) return TGB_ERR_UNSUPPORTED;
            k2.shard_n = P->n_workers;
            for (int r = 0; r <= kMaxPeers; ++r) k2.shard_bounds[r] = P->pcs[0][r];
        }
    }
    k1.tensors = P->d_tensors;
    k1.n_tensors = static_cast<int32_t>(P->desc.size());
    k2.fuse_decode = fuse_decode ? 1 : 0;
    if (fuse_decode && P->opt_active) {
        k2.optd = P->d_optd;
        k2.opt = *P->opt_active;
    }
    if (P->code_stats) {
        TGB_CUDA(cudaMemsetAsync(P->d_nnz, 0, sizeof(unsigned long long), st));
        k2.nnz = P->d_nnz;
    }
    if (++P->k12_epoch == 0) ++P->k12_epoch;  // any nonzero value marks a flag ready
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k12_table(P->d_layers, P->d_fat, P->ck1[0], P->cc[0], k1, k2, P->d_ready,
                              P->k12_epoch, st));
    if (ts >= 0) {
        uint64_t e[3];
        chunk_elems(P, P->h_chunks, 0, P->cc[0], e);
        const uint64_t nt = e[0], np = e[1], N = P->n_workers;
        const uint64_t msg = (nt + 3) / 4 + 4 * np;
        uint64_t own_b = msg, nvl = 0;
        if (P->attached && P->shard) {
            own_b = msg / N;
            nvl = msg - own_b;
        } else if (P->attached) {
            nvl = (N - 1) * msg;
        }
        const uint64_t out = fuse_decode ? 4 * (nt + np) : 0;
        t_end(P, st, ts, TGB_KERNEL_K12, 0, nt + np, 4 * nt + 4 * (nt + np) + own_b + out, nvl);
    }
    return TGB_OK;
}

// K1 -> K2 of an ungrouped step: one fused launch for small sets, else two
static tgb_status launch_encode(tgb_plan* P, uint64_t t, cudaStream_t st, bool fuse_decode) {
    if (P->k12) return launch_k12(P, t, st, fuse_decode);
    TGB_TRY(launch_stats(P, 0, st));
    return launch_tern(P, 0, t, st, fuse_decode);
}

// flag records of barrier slot s: {epoch, t} per (slot, step parity, peer), 16 B
// each; the kernel adds the parity's kMaxPeers records
static PeerFlags peer_flags(const tgb_plan* P, int s) {
    PeerFlags f{};
    for (int p = 0; p < P->n_workers; ++p)
        f.remote[p] = reinterpret_cast<uint64_t*>(P->peer_ipc[p] + P->flags_off) +
                      2 * (2 * s * kMaxPeers + P->rank);
    f.local = reinterpret_cast<uint64_t*>(P->d_ipc + P->flags_off) + 2 * (2 * s * kMaxPeers);
    f.n = P->n_workers;
    return f;
}

// mode: kBarrierSpin (multi-process: publish, then wait for every peer),
// kBarrierPost / kBarrierCheck (LocalCluster: publish; verify after the event wait)
static tgb_status launch_barrier(tgb_plan* P, int s, cudaStream_t st, int mode) {
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_peer_barrier(peer_flags(P, s), P->epoch, P->last_t, mode, P->d_err, st));
    t_end(P, st, ts, TGB_KERNEL_BARRIER, s, 0, 0, 0);
    return TGB_OK;
}

static tgb_status launch_decode_range(tgb_plan* P, int g, uint32_t cb3, uint32_t cc3,
                                      const uint8_t* src, int32_t n_workers, cudaStream_t st) {
    K3Launch k{src, P->push_bytes, n_workers, P->p.scaler_sharing ? 1 : 0,
               1.0f / static_cast<float>(n_workers), P->d_err};
    k.gate = P->attached ? 1 : 0;
    if (P->attached && P->pull8) {  // worker w's pulled items: its own area, its memory
        k.pull8 = P->pull8;
        const uint64_t g = P->push_bytes * static_cast<uint64_t>(P->n_workers);
        for (int w = 0; w < P->n_workers; ++w)
            k.wsrc[w] = P->peer_ipc[w] + (P->epoch & 1u) * g + static_cast<uint64_t>(w) * P->push_bytes;
    }
    if (P->opt_active) {
        k.optd = P->d_optd;
        k.opt = *P->opt_active;
    }
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k3_table(P->d_layers, P->d_fat3 + cb3, cc3, k, st));
    if (ts >= 0) {
        uint64_t e[3];
        chunk_elems(P, P->h_chunks3, cb3, cc3, e);
        const uint64_t nt = e[0], np = e[1], N = n_workers;
        const uint64_t pulled_b = k.pull8 ? (N - 1) * (e[2] / 4) : 0;
        t_end(P, st, ts, TGB_KERNEL_K3, g, nt + np,
              N * ((nt + 3) / 4 + 4 * np) - pulled_b + (P->opt_active ? 0 : 4 * (nt + np)),
              pulled_b);
    }
    return TGB_OK;
}

static tgb_status launch_decode(tgb_plan* P, int g, const uint8_t* src, int32_t n_workers,
                                cudaStream_t st) {
    return launch_decode_range(P, g, P->cb3[g], P->cc3[g], src, n_workers, st);
}

static inline uint8_t* sums_area(const tgb_plan* P, int p) {
    return P->peer_ipc[p] + P->sums_off + (P->epoch & 1u) * P->sums_bytes;
}

static ShardLaunch shard_launch(const tgb_plan* P) {
    ShardLaunch k{};
    k.src = cur_gathered(P);
    k.stride = P->push_bytes;
    for (int p = 0; p < P->n_workers; ++p) k.sums[p] = sums_area(P, p);
    k.own_sums = sums_area(P, P->rank);
    k.n_workers = P->n_workers;
    k.radix_m = P->radix_m;
    k.chunk12 = P->chunk12;
    k.sum_region = P->sum_region;
    k.inv_n = 1.0f / static_cast<float>(P->n_workers);
    k.err = P->d_err;
    return k;
}

// bytes of packed sums for `elems` ternary elements
static uint64_t radix_bytes(const tgb_plan* P, uint64_t elems) {
    return P->radix_m ? (elems + P->radix_m - 1) / P->radix_m * 4 : 0;
}

// sharded K3a over this rank's owned chunks of piece q: N workers' codes -> packed
// sums to every rank
static tgb_status launch_shard_reduce(tgb_plan* P, int q, cudaStream_t st) {
    const uint32_t r = static_cast<uint32_t>(P->rank);
    const uint32_t c0 = P->pcs[q][r], c1 = P->pcs[q][r + 1];
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k3_reduce(P->d_fat + c0, c1 - c0, shard_launch(P), st));
    if (ts >= 0) {
        uint64_t e[3];
        chunk_elems(P, P->h_chunks, c0, c1 - c0, e);
        const uint64_t N = P->n_workers;
        const uint64_t out = radix_bytes(P, e[0]) + 4 * e[1];
        t_end(P, st, ts, TGB_KERNEL_K3A, 0, e[0] + e[1], N * ((e[0] + 3) / 4 + 4 * e[1]) + out,
              (N - 1) * out);
    }
    return TGB_OK;
}

// sharded K3b: every rank decodes the packed sums of piece q (K2's chunk table)
static tgb_status launch_shard_expand(tgb_plan* P, int q, cudaStream_t st) {
    const uint32_t c0 = P->pb[q], n = P->pb[q + 1] - P->pb[q];
    const int ts = t_begin(P, st);
    TGB_CUDA(launch_k3_expand(P->d_fat + c0, n, shard_launch(P), st));
    if (ts >= 0) {
        uint64_t e[3];
        chunk_elems(P, P->h_chunks, c0, n, e);
        t_end(P, st, ts, TGB_KERNEL_K3B, 0, e[0] + e[1],
              radix_bytes(P, e[0]) + 4 * e[1] + 4 * (e[0] + e[1]), 0);
    }
    return TGB_OK;
}

extern "C" {

tgb_status tgb_stats(tgb_plan* P, void* stream) {
    if (!P || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    if (P->local_peers && P->n_workers > 1) return TGB_ERR_UNSUPPORTED;  // tgb_local_step
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    if (P->attached) ++P->epoch;  // a step begins: flip the gather-buffer parity
    for (int g = 0; g < n_groups(P); ++g) TGB_TRY(launch_stats(P, g, st));
    return TGB_OK;
}

tgb_status tgb_ternarize_pack(tgb_plan* P, uint64_t t, void* stream) {
    if (!P || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    if (P->local_peers && P->n_workers > 1) return TGB_ERR_UNSUPPORTED;
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    P->last_t = t;  // published with the step barrier (iteration-skew check)
    if (P->attached && P->shard) return launch_tern(P, 0, t, st);  // every piece
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
    // K2 ternarizes with the max; the peers' copies keep the local scalers, whose max
    // (the decode scaler, cluster.hpp:195-196) is the same value
    TGB_NCCL(ncclAllReduce(slots, slots, static_cast<size_t>(P->n_slots), ncclFloat, ncclMax,
                           C->comm, st));
    return TGB_OK;
}

tgb_status tgb_sync(tgb_plan* P, tgb_comm* C, void* stream) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    if (P->n_workers == 1) return TGB_OK;
    if (P->local_peers) return TGB_ERR_UNSUPPORTED;
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    if (P->attached) {  // data already moved by K1/K2: only order the step
        if (P->overlap) {  // K2 published every piece's records
            for (int q = 0; q < P->n_pieces; ++q) {
                TGB_TRY(launch_barrier(P, q, st, kBarrierWait));
                if (P->shard) {
                    TGB_TRY(launch_shard_reduce(P, q, st));
                    TGB_TRY(launch_barrier(P, P->n_pieces + q, st, kBarrierSpin));
                }
            }
            return TGB_OK;
        }
        if (P->shard) {
            // per piece: [codes landed at their owner] barrier -> K3a -> [sums everywhere] barrier
            for (int q = 0; q < P->n_pieces; ++q) {
                TGB_TRY(launch_barrier(P, 2 * q, st, kBarrierSpin));
                TGB_TRY(launch_shard_reduce(P, q, st));
                TGB_TRY(launch_barrier(P, 2 * q + 1, st, kBarrierSpin));
            }
            return TGB_OK;
        }
        for (int g = 0; g < n_groups(P); ++g) TGB_TRY(launch_barrier(P, g, st, kBarrierSpin));
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
    if (!d_src && P->attached && P->shard) {  // sharded exchange: decode this step's sums
        if (n_workers != P->n_workers) return TGB_ERR_INVALID_ARGUMENT;
        for (int q = 0; q < P->n_pieces; ++q) TGB_TRY(launch_shard_expand(P, q, st));
        return TGB_OK;
    }
    if (!d_src) d_src = cur_gathered(P);  // NULL: this step's gather buffer
    for (int g = 0; g < n_groups(P); ++g) TGB_TRY(launch_decode(P, g, d_src, n_workers, st));
    return TGB_OK;
}

tgb_status tgb_step(tgb_plan* P, tgb_comm* C, uint64_t t, void* stream) {
    if (!P || !P->bound) return TGB_ERR_INVALID_ARGUMENT;
    if (P->local_peers && P->n_workers > 1) return TGB_ERR_UNSUPPORTED;  // tgb_local_step
    auto st = static_cast<cudaStream_t>(stream);
    P->last = st;
    P->last_t = t;
    if (P->n_workers == 1) {  // the average of one worker is its own decode: K2 writes it
        if (!P->grouped) return launch_encode(P, t, st, true);
        TGB_CUDA(cudaEventRecord(P->ev_fork, st));
        for (int g = 1; g >= 0; --g) {  // dominant chain launched first
            cudaStream_t gs = P->gs[g];
            TGB_CUDA(cudaStreamWaitEvent(gs, P->ev_fork, 0));
            TGB_TRY(launch_stats(P, g, gs));
            TGB_TRY(launch_tern(P, g, t, gs, true));
            TGB_CUDA(cudaEventRecord(P->ev_join[g], gs));
        }
        TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[0], 0));
        TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[1], 0));
        return TGB_OK;
    }
    const bool nccl_exchange = !P->attached;
    if (P->attached && P->overlap) {
        // overlapped exchange: one K2 launch on `stream` publishes every finished piece;
        // on gs3 (ordered after the caller's prior work), piece q's wait -> decode (fused)
        // or wait -> K3a -> barrier -> K3b (sharded) overlap K2 of the later pieces
        ++P->epoch;
        const uint8_t* src = cur_gathered(P);
        TGB_CUDA(cudaEventRecord(P->ev_fork, st));
        TGB_TRY(launch_stats(P, 0, st));
        TGB_TRY(launch_tern(P, 0, t, st));
        TGB_CUDA(cudaStreamWaitEvent(P->gs3, P->ev_fork, 0));
        for (int q = 0; q < P->n_pieces; ++q) {
            TGB_TRY(launch_barrier(P, q, P->gs3, kBarrierWait));
            if (P->shard) {
                TGB_TRY(launch_shard_reduce(P, q, P->gs3));
                TGB_TRY(launch_barrier(P, P->n_pieces + q, P->gs3, kBarrierSpin));
                TGB_TRY(launch_shard_expand(P, q, P->gs3));
            } else {
                TGB_TRY(launch_decode_range(P, 0, P->p3[q], P->p3[q + 1] - P->p3[q], src,
                                            P->n_workers, P->gs3));
            }
        }
        TGB_CUDA(cudaEventRecord(P->ev_done, P->gs3));
        TGB_CUDA(cudaStreamWaitEvent(st, P->ev_done, 0));
        return TGB_OK;
    }
    if (P->attached && P->shard && P->p.share_mode == TGB_SHARE_REF && !P->k12) {
        // sharded exchange: K2 piece by piece on `stream`; on gs3 (ordered after the
        // caller's prior work), piece q's barrier -> K3a -> barrier -> K3b
        ++P->epoch;
        TGB_CUDA(cudaEventRecord(P->ev_fork, st));
        if (P->grouped) {  // piece g = group g, each chain on its own stream
            for (int g = 1; g >= 0; --g) {
                cudaStream_t gs = P->gs[g];
                TGB_CUDA(cudaStreamWaitEvent(gs, P->ev_fork, 0));
                TGB_TRY(launch_stats(P, g, gs));
                TGB_TRY(launch_tern_range(P, g, P->pb[g], P->pb[g + 1] - P->pb[g], g, t, gs, false));
                TGB_TRY(launch_barrier(P, 2 * g, gs, kBarrierSpin));
                TGB_TRY(launch_shard_reduce(P, g, gs));
                TGB_TRY(launch_barrier(P, 2 * g + 1, gs, kBarrierSpin));
                TGB_TRY(launch_shard_expand(P, g, gs));
                TGB_CUDA(cudaEventRecord(P->ev_join[g], gs));
            }
            TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[0], 0));
            TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[1], 0));
            return TGB_OK;
        }
        TGB_TRY(launch_stats(P, 0, st));
        TGB_CUDA(cudaStreamWaitEvent(P->gs3, P->ev_fork, 0));
        for (int q = 0; q < P->n_pieces; ++q) {
            TGB_TRY(launch_tern_range(P, 0, P->pb[q], P->pb[q + 1] - P->pb[q], q, t, st, false));
            TGB_CUDA(cudaEventRecord(P->ev_piece[q], st));
            TGB_CUDA(cudaStreamWaitEvent(P->gs3, P->ev_piece[q], 0));
            TGB_TRY(launch_barrier(P, 2 * q, P->gs3, kBarrierSpin));
            TGB_TRY(launch_shard_reduce(P, q, P->gs3));
            TGB_TRY(launch_barrier(P, 2 * q + 1, P->gs3, kBarrierSpin));
            TGB_TRY(launch_shard_expand(P, q, P->gs3));
        }
        TGB_CUDA(cudaEventRecord(P->ev_done, P->gs3));
        TGB_CUDA(cudaStreamWaitEvent(st, P->ev_done, 0));
        return TGB_OK;
    }
    if (!P->grouped || nccl_exchange) {
        if (P->p.share_mode == TGB_SHARE_PRESHARED) {
            TGB_TRY(tgb_stats(P, stream));
            TGB_TRY(tgb_share_scalers(P, C, stream));
            TGB_TRY(tgb_ternarize_pack(P, t, stream));
        } else if (P->grouped) {
            TGB_TRY(tgb_stats(P, stream));
            TGB_TRY(tgb_ternarize_pack(P, t, stream));
        } else {
            if (P->attached) ++P->epoch;  // a step begins: flip the gather-buffer parity
            TGB_TRY(launch_encode(P, t, st, false));
        }
        TGB_TRY(tgb_sync(P, C, stream));
        return tgb_decode_average(P, nullptr, P->n_workers, stream);
    }
    // overlapped two-group schedule (fused exchange): fork the step onto the plan's
    // two streams, each group K1 -> K2 (peer stores) -> barrier -> K3, join back
    ++P->epoch;
    TGB_CUDA(cudaEventRecord(P->ev_fork, st));
    const uint8_t* src = cur_gathered(P);
    for (int g = 1; g >= 0; --g) {
        cudaStream_t gs = P->gs[g];
        TGB_CUDA(cudaStreamWaitEvent(gs, P->ev_fork, 0));
        TGB_TRY(launch_stats(P, g, gs));
        TGB_TRY(launch_tern(P, g, t, gs));
        TGB_TRY(launch_barrier(P, g, gs, kBarrierSpin));
        TGB_TRY(launch_decode(P, g, src, P->n_workers, gs));
        TGB_CUDA(cudaEventRecord(P->ev_join[g], gs));
    }
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[0], 0));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_join[1], 0));
    return TGB_OK;
}

// One step of every LocalCluster plan (tgb_plan_attach_local). The plans' streams
// are ordered by CUDA events instead of spinning barriers: each plan publishes its
// flag + iteration after its K2 (post), every plan's decode waits for all posts
// and then verifies them (check, no spin). Phase by phase over all plans, so a
// plan never waits on an event its peer has not recorded yet.
tgb_status tgb_local_step(tgb_plan* const* plans, int32_t n, const uint64_t* t,
                          void* const* streams) {
    if (!plans || !t || !streams || n < 1 || n > kMaxPeers) return TGB_ERR_INVALID_ARGUMENT;
    for (int32_t w = 0; w < n; ++w) {
        const tgb_plan* P = plans[w];
        if (!P || !P->bound || P->n_workers != n || P->worker != w) return TGB_ERR_INVALID_ARGUMENT;
        if (n > 1 && !(P->attached && P->local_peers)) return TGB_ERR_INVALID_ARGUMENT;
    }
    if (n == 1) return tgb_step(plans[0], nullptr, t[0], streams[0]);
    int prev = 0;
    TGB_CUDA(cudaGetDevice(&prev));
    auto st_of = [&](int w) { return static_cast<cudaStream_t>(streams[w]); };
    auto on = [&](int w) { return cudaSetDevice(plans[w]->device) == cudaSuccess; };
    auto fail = [&](tgb_status s) {
        cudaSetDevice(prev);
        return s;
    };
    for (int32_t w = 0; w < n; ++w) {
        tgb_plan* P = plans[w];
        P->last = st_of(w);
        P->last_t = t[w];
        ++P->epoch;
    }
    // PRESHARED (paper Eq. 4): every plan's K1, then each plan replaces its own slots by
    // the max over the N workers' local slots its gather buffer now holds (the
    // single-process stand-in for the ranks' ncclAllReduce(max)), then K2
    const bool preshared = plans[0]->p.share_mode == TGB_SHARE_PRESHARED;
    if (preshared) {
        for (int w = 0; w < n; ++w) {
            tgb_plan* P = plans[w];
            if (!on(w)) return fail(TGB_ERR_CUDA);
            tgb_status s = launch_stats(P, 0, st_of(w));
            if (s != TGB_OK) return fail(s);
            if (cudaEventRecord(P->ev_local[2], st_of(w)) != cudaSuccess) return fail(TGB_ERR_CUDA);
        }
        for (int w = 0; w < n; ++w) {
            tgb_plan* P = plans[w];
            if (!on(w)) return fail(TGB_ERR_CUDA);
            for (int q = 0; q < n; ++q)
                if (cudaStreamWaitEvent(st_of(w), plans[q]->ev_local[2], 0) != cudaSuccess)
                    return fail(TGB_ERR_CUDA);
            if (launch_slot_max(reinterpret_cast<float*>(own_push(P)), cur_gathered(P),
                                P->push_bytes, n, P->n_slots, st_of(w)) != cudaSuccess)
                return fail(TGB_ERR_CUDA);
        }
    }
    if (plans[0]->overlap) {
        const int npc = plans[0]->n_pieces;
        for (int w = 0; w < n; ++w) {  // K1 + K2; K2 posts every piece's records
            tgb_plan* P = plans[w];
            cudaStream_t st = st_of(w);
            if (!on(w)) return fail(TGB_ERR_CUDA);
            tgb_status s = launch_stats(P, 0, st);
            if (s == TGB_OK) s = launch_tern(P, 0, t[w], st);
            if (s != TGB_OK) return fail(s);
            if (cudaEventRecord(P->ev_local[0], st) != cudaSuccess) return fail(TGB_ERR_CUDA);
        }
        for (int phase = 0; phase < (plans[0]->shard ? 2 : 1); ++phase) {
            for (int w = 0; w < n; ++w) {
                tgb_plan* P = plans[w];
                cudaStream_t st = st_of(w);
                if (!on(w)) return fail(TGB_ERR_CUDA);
                for (int q = 0; q < n; ++q)
                    if (cudaStreamWaitEvent(st, plans[q]->ev_local[phase], 0) != cudaSuccess)
                        return fail(TGB_ERR_CUDA);
                tgb_status s = TGB_OK;
                for (int q = 0; q < npc && s == TGB_OK; ++q) {
                    s = launch_barrier(P, phase * npc + q, st, kBarrierCheck);
                    if (s == TGB_OK && P->shard && phase == 0) {
                        s = launch_shard_reduce(P, q, st);
                        if (s == TGB_OK) s = launch_barrier(P, npc + q, st, kBarrierPost);
                    } else if (s == TGB_OK && P->shard) {
                        s = launch_shard_expand(P, q, st);
                    }
                }
                if (s == TGB_OK && !P->shard) s = launch_decode(P, 0, cur_gathered(P), n, st);
                if (s == TGB_OK && P->shard && phase == 0 &&
                    cudaEventRecord(P->ev_local[1], st) != cudaSuccess)
                    s = TGB_ERR_CUDA;
                if (s != TGB_OK) return fail(s);
            }
        }
        return fail(TGB_OK);
    }
    if (plans[0]->shard) {
        for (int w = 0; w < n; ++w) {
            tgb_plan* P = plans[w];
            cudaStream_t st = st_of(w);
            if (!on(w)) return fail(TGB_ERR_CUDA);
            tgb_status s = TGB_OK;
            if (P->k12 && !preshared)
                s = launch_encode(P, t[w], st, false);
            else if (!preshared)
                for (int g = 0; g < n_groups(P) && s == TGB_OK; ++g) s = launch_stats(P, g, st);
            if (s == TGB_OK && !P->k12) s = launch_tern(P, 0, t[w], st);
            for (int q = 0; q < P->n_pieces && s == TGB_OK; ++q)
                s = launch_barrier(P, 2 * q, st, kBarrierPost);
            if (s != TGB_OK) return fail(s);
            if (cudaEventRecord(P->ev_local[0], st) != cudaSuccess) return fail(TGB_ERR_CUDA);
        }
        for (int phase = 0; phase < 2; ++phase) {
            for (int w = 0; w < n; ++w) {
                tgb_plan* P = plans[w];
                cudaStream_t st = st_of(w);
                if (!on(w)) return fail(TGB_ERR_CUDA);
                for (int q = 0; q < n; ++q)
                    if (cudaStreamWaitEvent(st, plans[q]->ev_local[phase], 0) != cudaSuccess)
                        return fail(TGB_ERR_CUDA);
                tgb_status s = TGB_OK;
                for (int q = 0; q < P->n_pieces && s == TGB_OK; ++q) {
                    s = launch_barrier(P, 2 * q + phase, st, kBarrierCheck);
                    if (s == TGB_OK && phase == 0) {
                        s = launch_shard_reduce(P, q, st);
                        if (s == TGB_OK) s = launch_barrier(P, 2 * q + 1, st, kBarrierPost);
                    } else if (s == TGB_OK) {
                        s = launch_shard_expand(P, q, st);
                    }
                }
                if (s == TGB_OK && phase == 0 && cudaEventRecord(P->ev_local[1], st) != cudaSuccess)
                    s = TGB_ERR_CUDA;
                if (s != TGB_OK) return fail(s);
            }
        }
        return fail(TGB_OK);
    }
    const int G = n_groups(plans[0]);
    auto gst = [&](int w, int g) { return plans[w]->grouped ? plans[w]->gs[g] : st_of(w); };
    for (int w = 0; w < n; ++w) {
        tgb_plan* P = plans[w];
        if (!on(w)) return fail(TGB_ERR_CUDA);
        if (P->grouped) {
            if (cudaEventRecord(P->ev_fork, st_of(w)) != cudaSuccess) return fail(TGB_ERR_CUDA);
            for (int g = 0; g < 2; ++g)
                if (cudaStreamWaitEvent(P->gs[g], P->ev_fork, 0) != cudaSuccess)
                    return fail(TGB_ERR_CUDA);
        }
        for (int g = G - 1; g >= 0; --g) {
            cudaStream_t gs = gst(w, g);
            tgb_status s = preshared   ? launch_tern(P, g, t[w], gs)
                           : P->grouped ? launch_stats(P, g, gs)
                                        : launch_encode(P, t[w], gs, false);
            if (s == TGB_OK && P->grouped && !preshared) s = launch_tern(P, g, t[w], gs);
            if (s == TGB_OK) s = launch_barrier(P, g, gs, kBarrierPost);
            if (s != TGB_OK) return fail(s);
            if (cudaEventRecord(P->ev_local[g], gs) != cudaSuccess) return fail(TGB_ERR_CUDA);
        }
    }
    for (int w = 0; w < n; ++w) {
        tgb_plan* P = plans[w];
        if (!on(w)) return fail(TGB_ERR_CUDA);
        const uint8_t* src = cur_gathered(P);
        for (int g = G - 1; g >= 0; --g) {
            cudaStream_t gs = gst(w, g);
            for (int q = 0; q < n; ++q)
                if (cudaStreamWaitEvent(gs, plans[q]->ev_local[g], 0) != cudaSuccess)
                    return fail(TGB_ERR_CUDA);
            tgb_status s = launch_barrier(P, g, gs, kBarrierCheck);
            if (s == TGB_OK) s = launch_decode(P, g, src, n, gs);
            if (s != TGB_OK) return fail(s);
            if (P->grouped && cudaEventRecord(P->ev_join[g], gs) != cudaSuccess)
                return fail(TGB_ERR_CUDA);
        }
        if (P->grouped)
            for (int g = 0; g < 2; ++g)
                if (cudaStreamWaitEvent(st_of(w), P->ev_join[g], 0) != cudaSuccess)
                    return fail(TGB_ERR_CUDA);
    }
    return fail(TGB_OK);
}

}  // extern "C"

// Per-tensor copies dst[l] <- src[l] (n_l floats), coalesced into one copy per run
// of tensors that are adjacent on BOTH sides (e.g. flat buffers whose tensors are
// back to back): one 553 MB copy instead of 32 runs PCIe ~10 % faster. Gaps are
// never copied (they may be someone else's memory).
// group >= 0: only the tensors of that layer group (1 = the dominant tensor)
static tgb_status copy_runs(const tgb_plan* P, const float* const* dst_c, const float* const* src,
                            cudaMemcpyKind kind, cudaStream_t st, int group = -1) {
    float* const* dst = const_cast<float* const*>(dst_c);
    const size_t nl = P->desc.size();
    auto in = [&](size_t l) {
        return group < 0 || (static_cast<int32_t>(l) == P->big) == (group == 1);
    };
    size_t l = 0;
    while (l < nl) {
        if (!P->desc[l].n || !in(l)) {
            ++l;
            continue;
        }
        uint64_t n = P->desc[l].n;
        size_t e = l + 1;
        for (; e < nl; ++e) {
            const uint64_t m = P->desc[e].n;
            if (!m) continue;
            if (!in(e) || dst[e] != dst[l] + n || src[e] != src[l] + n) break;
            n += m;
        }
        TGB_CUDA(cudaMemcpyAsync(dst[l], src[l], n * sizeof(float), kind, st));
        l = e;
    }
    return TGB_OK;
}

extern "C" {

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
    if (P->n_workers == 1 && P->grouped) {
        // pipelined by layer group: H2D(rest) -> its K1/K2 (+decode) while H2D(dominant)
        // runs; each group's D2H starts when its decode is done. Both PCIe directions
        // stay busy and the compute hides under the transfers (round 1: 13.5 ms/step
        // against the ~12 ms full-duplex floor for VGG-16, compute waited for all H2D).
        if (!P->ev_hg[0])
            for (int g = 0; g < 2; ++g) {
                TGB_CUDA(cudaEventCreateWithFlags(&P->ev_hg[g], cudaEventDisableTiming));
                TGB_CUDA(cudaEventCreateWithFlags(&P->ev_cg[g], cudaEventDisableTiming));
                TGB_CUDA(cudaEventCreateWithFlags(&P->ev_dg[g], cudaEventDisableTiming));
                TGB_CUDA(cudaEventRecord(P->ev_cg[g], st));
                TGB_CUDA(cudaEventRecord(P->ev_dg[g], st));
            }
        for (int g = 0; g < 2; ++g) {  // the small group first: its compute starts early
            TGB_CUDA(cudaStreamWaitEvent(P->s_h2d, P->ev_cg[g], 0));  // previous K2 read them
            TGB_TRY(copy_runs(P, reinterpret_cast<const float* const*>(P->bound_g.data()),
                              h_grads, cudaMemcpyHostToDevice, P->s_h2d, g));
            TGB_CUDA(cudaEventRecord(P->ev_hg[g], P->s_h2d));
        }
        P->last = st;
        P->last_t = t;
        TGB_CUDA(cudaEventRecord(P->ev_fork, st));
        for (int g = 0; g < 2; ++g) {
            cudaStream_t gs = P->gs[g];
            TGB_CUDA(cudaStreamWaitEvent(gs, P->ev_fork, 0));
            TGB_CUDA(cudaStreamWaitEvent(gs, P->ev_hg[g], 0));
            TGB_CUDA(cudaStreamWaitEvent(gs, P->ev_dg[g], 0));  // previous outputs copied out
            TGB_TRY(launch_stats(P, g, gs));
            TGB_TRY(launch_tern(P, g, t, gs, true));
            TGB_CUDA(cudaEventRecord(P->ev_cg[g], gs));
        }
        for (int g = 0; g < 2; ++g) {
            TGB_CUDA(cudaStreamWaitEvent(P->s_d2h, P->ev_cg[g], 0));
            TGB_TRY(copy_runs(P, h_out, P->bound_out.data(), cudaMemcpyDeviceToHost, P->s_d2h, g));
            TGB_CUDA(cudaEventRecord(P->ev_dg[g], P->s_d2h));
        }
        TGB_CUDA(cudaEventRecord(P->ev_d2h, P->s_d2h));
        TGB_CUDA(cudaStreamWaitEvent(st, P->ev_d2h, 0));
        return TGB_OK;
    }
    TGB_CUDA(cudaStreamWaitEvent(P->s_h2d, P->ev_comp, 0));  // previous K2 read the gradients
    TGB_TRY(copy_runs(P, reinterpret_cast<const float* const*>(P->bound_g.data()), h_grads,
                      cudaMemcpyHostToDevice, P->s_h2d));
    TGB_CUDA(cudaEventRecord(P->ev_h2d, P->s_h2d));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_h2d, 0));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_d2h, 0));  // previous outputs copied out
    TGB_TRY(tgb_step(P, C, t, stream));
    TGB_CUDA(cudaEventRecord(P->ev_comp, st));
    TGB_CUDA(cudaStreamWaitEvent(P->s_d2h, P->ev_comp, 0));
    TGB_TRY(copy_runs(P, h_out, P->bound_out.data(), cudaMemcpyDeviceToHost, P->s_d2h));
    TGB_CUDA(cudaEventRecord(P->ev_d2h, P->s_d2h));
    TGB_CUDA(cudaStreamWaitEvent(st, P->ev_d2h, 0));
    P->last = st;
    return TGB_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ attach
static PlanDesc make_desc(const tgb_plan* P) {
    PlanDesc d{};
    d.magic = 0x5447423230304450ull;  // "TGB200DP"
    d.abi = TGB_ABI_VERSION;
    d.n_workers = P->n_workers;
    d.push_bytes = P->push_bytes;
    d.sums_bytes = P->sums_bytes;
    d.ipc_bytes = P->ipc_bytes;
    d.n_blocks = static_cast<uint32_t>(P->h_layers.size());
    d.n_tensors = static_cast<uint32_t>(P->desc.size());
    d.chunk12 = P->chunk12;
    d.chunk3 = P->chunk3;
    d.shard = P->shard;
    d.grouped = P->grouped;
    d.radix_m = P->radix_m;
    d.reserved = static_cast<int32_t>(P->mb_log2) | (P->n_pieces << 8) | (P->overlap << 16) |
                 static_cast<int32_t>(P->pull8 << 20);
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t b = 0; b < P->h_layers.size(); ++b) {
        const LayerDev& L = P->h_layers[b];
        h = fnv_mix(h, L.n);
        h = fnv_mix(h, (static_cast<uint64_t>(L.tensor) << 32) | static_cast<uint32_t>(L.slot));
        h = fnv_mix(h, L.flags & (kLayerPassthrough | kLayerClip));
        h = fnv_mix(h, L.code_off);
        h = fnv_mix(h, (static_cast<uint64_t>(L.sum_off16) << 32) | P->block_off[b]);
    }
    for (const tgb_layer_desc& l : P->desc) h = fnv_mix(fnv_mix(h, l.n), l.name_hash);
    d.layout_hash = h;
    uint64_t c = 0xcbf29ce484222325ull;
    uint32_t cf;
    std::memcpy(&cf, &P->p.clip_factor, 4);
    c = fnv_mix(c, cf);
    c = fnv_mix(c, (static_cast<uint64_t>(P->p.clipping_enabled) << 32) |
                       static_cast<uint32_t>(P->p.bucketing));
    c = fnv_mix(c, (static_cast<uint64_t>(P->p.scaler_sharing) << 32) |
                       static_cast<uint32_t>(P->p.share_mode));
    c = fnv_mix(c, P->p.bucket_size);
    c = fnv_mix(c, P->p.seed);
    d.codec_hash = c;
    return d;
}

// the reference's texts where it has one (cluster.hpp:169-172), else a plain one
static tgb_status compare_desc(const PlanDesc& a, const PlanDesc& b, int worker) {
    const std::string w = std::to_string(worker);
    if (a.magic != b.magic || a.abi != b.abi)
        return set_protocol_error("attach: worker " + w + " runs another libtgb ABI");
    if (a.n_workers != b.n_workers)
        return set_protocol_error("attach: worker count mismatch from worker " + w);
    if (a.n_blocks != b.n_blocks || a.n_tensors != b.n_tensors || a.layout_hash != b.layout_hash)
        return set_protocol_error("server: block structure mismatch from worker " + w);
    if (a.codec_hash != b.codec_hash)
        return set_protocol_error("attach: codec configuration mismatch from worker " + w);
    if (a.push_bytes != b.push_bytes || a.sums_bytes != b.sums_bytes || a.ipc_bytes != b.ipc_bytes ||
        a.chunk12 != b.chunk12 || a.chunk3 != b.chunk3 || a.shard != b.shard ||
        a.grouped != b.grouped || a.radix_m != b.radix_m || a.reserved != b.reserved)
        return set_protocol_error("attach: exchange schedule mismatch from worker " + w);
    return TGB_OK;
}

// [gather parity 0][gather parity 1][sums parity 0][sums parity 1][flags]
static tgb_status alloc_ipc(tgb_plan* P) {
    const uint64_t g = P->push_bytes * static_cast<uint64_t>(P->n_workers);
    P->sums_off = 2 * g;
    P->flags_off = P->sums_off + 2 * P->sums_bytes;
    P->ipc_bytes = P->flags_off + round_up(kFlagSlots * 2 * kMaxPeers * 16, kAlignPush);
    if (P->d_ipc) return TGB_OK;
    TGB_CUDA(cudaMalloc(&P->d_ipc, P->ipc_bytes));
    TGB_CUDA(cudaMemset(P->d_ipc, 0, P->ipc_bytes));
    return TGB_OK;
}

static void finish_attach(tgb_plan* P) {
    cudaFree(P->d_nccl_gather);  // the gather buffers now live in d_ipc
    P->d_nccl_gather = nullptr;
    P->d_gathered = P->d_ipc;
    P->attached = true;
}

extern "C" {

tgb_status tgb_plan_attach_peers(tgb_plan* P, tgb_comm* C) {
    if (!P || !C) return TGB_ERR_INVALID_ARGUMENT;
    if (P->n_workers == 1) return TGB_OK;
    if (C->nranks != P->n_workers || C->rank != P->worker || P->n_workers > kMaxPeers)
        return TGB_ERR_INVALID_ARGUMENT;
    if (P->attached) return TGB_OK;
    TGB_TRY(alloc_ipc(P));
    struct Msg {
        cudaIpcMemHandle_t h;
        PlanDesc d;
    };
    Msg mine{};
    TGB_CUDA(cudaIpcGetMemHandle(&mine.h, P->d_ipc));
    mine.d = make_desc(P);
    const int N = P->n_workers;
    std::vector<Msg> all(N);
    uint8_t* d_tmp = nullptr;
    TGB_CUDA(cudaMalloc(&d_tmp, sizeof(Msg) * (N + 1)));
    TGB_CUDA(cudaMemcpy(d_tmp, &mine, sizeof(Msg), cudaMemcpyHostToDevice));
    const ncclResult_t r = ncclAllGather(d_tmp, d_tmp + sizeof(Msg), sizeof(Msg), ncclUint8,
                                         C->comm, nullptr);
    cudaError_t e = cudaStreamSynchronize(nullptr);
    if (r == ncclSuccess && e == cudaSuccess)
        e = cudaMemcpy(all.data(), d_tmp + sizeof(Msg), sizeof(Msg) * N, cudaMemcpyDeviceToHost);
    cudaFree(d_tmp);
    if (r != ncclSuccess) return TGB_ERR_NCCL;
    TGB_CUDA(e);
    // every rank compares every descriptor: all ranks fail together on a mismatch,
    // before any peer memory is opened
    for (int p = 0; p < N; ++p) TGB_TRY(compare_desc(mine.d, all[p].d, p));
    P->rank = C->rank;
    for (int p = 0; p < N; ++p) {
        if (p == P->rank) {
            P->peer_ipc[p] = P->d_ipc;
            continue;
        }
        void* ptr = nullptr;
        TGB_CUDA(cudaIpcOpenMemHandle(&ptr, all[p].h, cudaIpcMemLazyEnablePeerAccess));
        P->peer_ipc[p] = static_cast<uint8_t*>(ptr);
    }
    finish_attach(P);
    return TGB_OK;
}

tgb_status tgb_plan_attach_local(tgb_plan* const* plans, int32_t n) {
    if (!plans || n < 1 || n > kMaxPeers) return TGB_ERR_INVALID_ARGUMENT;
    for (int32_t p = 0; p < n; ++p) {
        tgb_plan* P = plans[p];
        if (!P || P->n_workers != n || P->worker != p || P->attached) return TGB_ERR_INVALID_ARGUMENT;
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
    tgb_status s = TGB_OK;
    for (int32_t p = 0; p < n && s == TGB_OK; ++p) {
        tgb_plan* P = plans[p];
        if (cudaSetDevice(P->device) != cudaSuccess) s = TGB_ERR_CUDA;
        if (s == TGB_OK) s = alloc_ipc(P);
        for (int i = 0; i < 3 && s == TGB_OK; ++i)
            if (!P->ev_local[i] &&
                cudaEventCreateWithFlags(&P->ev_local[i], cudaEventDisableTiming) != cudaSuccess)
                s = TGB_ERR_CUDA;
    }
    cudaSetDevice(cur);
    if (s != TGB_OK) return s;
    const PlanDesc d0 = make_desc(plans[0]);
    for (int32_t p = 1; p < n; ++p) TGB_TRY(compare_desc(d0, make_desc(plans[p]), p));
    for (int32_t p = 0; p < n; ++p) {
        tgb_plan* P = plans[p];
        P->rank = p;
        for (int32_t q = 0; q < n; ++q) P->peer_ipc[q] = plans[q]->d_ipc;
        P->local_peers = true;
        cudaSetDevice(P->device);
        finish_attach(P);
    }
    cudaSetDevice(cur);
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
    if (P->grouped)
        for (int g = 0; g < 2; ++g) TGB_CUDA(cudaStreamSynchronize(P->gs[g]));
    ErrWord e;
    TGB_CUDA(cudaMemcpy(&e, P->d_err, sizeof(e), cudaMemcpyDeviceToHost));
    out->flags = e.flags;
    out->layer = e.flags ? e.layer() : -1;
    out->index = e.flags ? e.index() : 0;
    out->aux = e.flags ? e.aux : 0;
    if (e.flags) TGB_CUDA(cudaMemset(P->d_err, 0, sizeof(ErrWord)));
    return e.flags ? TGB_ERR_CODEC : TGB_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ audit
// Layout self-check (no kernel runs): every region a kernel of this plan reads or
// writes lies inside its allocation and work items tile their blocks exactly.
// compute-sanitizer is not available on the GPU pool; this is the host-side
// substitute for the address-range class of bugs (tests call it for every
// configuration they build).
extern "C" tgb_status tgb_plan_audit(const tgb_plan* P) {
    if (!P) return TGB_ERR_INVALID_ARGUMENT;
    auto bad = [](const std::string& m) { return set_protocol_error("audit: " + m); };
    const size_t nb = P->h_layers.size();
    if (static_cast<uint64_t>(P->n_slots) * 4 > P->codes_offset) return bad("slots overlap codes");
    uint64_t prev_end = P->codes_offset;
    for (size_t b = 0; b < nb; ++b) {
        const LayerDev& L = P->h_layers[b];
        const uint64_t bytes = (L.flags & kLayerPassthrough) ? 4ull * L.n : (L.n + 3ull) / 4;
        if (L.code_off < prev_end || L.code_off % 16) return bad("block region order " + std::to_string(b));
        if (L.code_off + bytes > P->push_bytes) return bad("block region past push area " + std::to_string(b));
        prev_end = L.code_off + bytes;
    }
    auto check_items = [&](const std::vector<ChunkDev>& chs, const char* what) -> tgb_status {
        std::vector<uint64_t> covered(nb, 0);
        for (size_t c = 0; c < chs.size(); ++c) {
            const ChunkDev& ch = chs[c];
            if (ch.layer >= nb || ch.nblk < 1 || ch.layer + ch.nblk > nb)
                return bad(std::string(what) + " item block range " + std::to_string(c));
            if (ch.nblk == 1) {
                const LayerDev& L = P->h_layers[ch.layer];
                if (static_cast<uint64_t>(ch.begin) + ch.count > L.n || ch.begin % 16)
                    return bad(std::string(what) + " item past its block " + std::to_string(c));
                covered[ch.layer] += ch.count;
                continue;
            }
            uint64_t cnt = 0;
            const LayerDev& L0 = P->h_layers[ch.layer];
            for (uint32_t j = 0; j < ch.nblk; ++j) {
                const LayerDev& L = P->h_layers[ch.layer + j];
                if (L.tensor != L0.tensor || !(L.flags & kLayerMultiBucket) ||
                    L.slot != L0.slot + static_cast<int32_t>(j) ||
                    L.code_off != L0.code_off + cnt / 4 || ch.begin != 0)
                    return bad(std::string(what) + " multi-bucket item not contiguous " + std::to_string(c));
                cnt += L.n;
                covered[ch.layer + j] += L.n;
            }
            if (cnt != ch.count) return bad(std::string(what) + " multi-bucket count " + std::to_string(c));
        }
        for (size_t b = 0; b < nb; ++b)
            if (covered[b] != P->h_layers[b].n)
                return bad(std::string(what) + " items do not tile block " + std::to_string(b));
        return TGB_OK;
    };
    TGB_TRY(check_items(P->h_chunks, "K1/K2"));
    TGB_TRY(check_items(P->h_chunks3, "K3"));
    if (P->shard) {
        if (P->pb[0] != 0 || P->pb[P->n_pieces] != P->h_chunks.size()) return bad("pieces");
        for (int q = 0; q < P->n_pieces; ++q) {
            if (P->pb[q] > P->pb[q + 1]) return bad("pieces order");
            if (P->pcs[q][0] != P->pb[q] || P->pcs[q][P->n_workers] != P->pb[q + 1])
                return bad("owners do not tile piece " + std::to_string(q));
            for (int r = 0; r < P->n_workers; ++r)
                if (P->pcs[q][r] > P->pcs[q][r + 1]) return bad("owner order");
        }
        std::vector<std::pair<uint64_t, uint64_t>> spans;
        for (const ChunkDev& ch : P->h_chunks) {
            const LayerDev& L = P->h_layers[ch.layer];
            const bool pass = (L.flags & kLayerPassthrough) != 0;
            const uint64_t off = pass ? 16ull * L.sum_off16 + 4ull * ch.begin
                                      : 16ull * L.sum_off16 + (ch.begin / P->chunk12) *
                                                                  static_cast<uint64_t>(P->sum_region);
            const uint64_t len = pass ? 4ull * ch.count
                                      : (ch.count + P->radix_m - 1) / P->radix_m * 4ull;
            if (off + len > P->sums_bytes) return bad("sums region past the sums buffer");
            spans.push_back({off, off + len});
        }
        std::sort(spans.begin(), spans.end());
        for (size_t i = 1; i < spans.size(); ++i)
            if (spans[i].first < spans[i - 1].second) return bad("sums regions overlap");
    }
    if (P->overlap && !P->shard) {  // each piece's K3 items cover exactly its K2 items
        if (P->p3[0] != 0 || P->p3[P->n_pieces] != P->h_chunks3.size()) return bad("K3 pieces");
        for (int q = 0; q < P->n_pieces; ++q) {
            uint64_t e2 = 0, e3 = 0;
            for (uint32_t c = P->pb[q]; c < P->pb[q + 1]; ++c) e2 += P->h_chunks[c].count;
            for (uint32_t c = P->p3[q]; c < P->p3[q + 1]; ++c) e3 += P->h_chunks3[c].count;
            if (P->p3[q] > P->p3[q + 1] || e2 != e3) return bad("K3 piece " + std::to_string(q));
        }
    }
    if (P->attached) {
        const uint64_t g = P->push_bytes * static_cast<uint64_t>(P->n_workers);
        if (P->sums_off < 2 * g || P->flags_off < P->sums_off + 2 * P->sums_bytes)
            return bad("exchange allocation order");
        if (P->flags_off + static_cast<uint64_t>(kFlagSlots) * 2 * kMaxPeers * 16 > P->ipc_bytes)
            return bad("barrier records past the allocation");
        if (P->shard && 2 * P->n_pieces > kFlagSlots) return bad("barrier slots");
        if (P->grouped && kFlagSlots < 2) return bad("barrier slots");
    }
    return TGB_OK;
}
