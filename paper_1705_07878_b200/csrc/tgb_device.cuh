// Device-side building blocks of the B200 TernGrad path (sm_100a).
//
// Reference semantics restated here (paths under proj/include/terngrad/):
//   philox4x32_10   rng.hpp:15-33   (Random123 Philox4x32-10)
//   RngStream key   rng.hpp:50-57   key = {u32(seed^h), u32((seed>>32)^(h>>32)^(worker*0x9E3779B97F4A7C15))}
//   RngStream bits  rng.hpp:59-66   ctr = {lo(i>>2), hi(i>>2), lo(t), hi(t)}, lane = i&3
//   uniform         rng.hpp:69-71   float(bits)*2^-32 (round-to-nearest; 1.0f reachable)
//   code map        codec.hpp:19-23 00=0 01=+1 10=-1 11=corrupt; element k at bits 2(k%4) of byte k/4
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "tgb/terngrad_b200.h"

namespace tgb {

constexpr int kThreads = 256;       // CTA size of every streaming kernel
constexpr uint32_t kChunk = 16384;    // per-layer API work item (elements, multiple of 16)
constexpr uint32_t kChunk12 = 32768;  // plan K1/K2 work item
constexpr uint32_t kChunk3 = 16384;   // plan K3 work item
constexpr uint32_t kK1Group = 64;     // K1 two-level finalize: units per group,
constexpr uint32_t kK1GroupMin = 256; // for tensors of more units than this
// radix-3 wire codes (5 elements per byte): work items start at multiples of 80
// elements so every chunk's bytes start 16-B aligned (80 / 5 = 16)
constexpr uint32_t kChunk3R3 = 16320;  // = 204 x 80
constexpr int kMaxWorkers = 64;     // decode LUT capacity (2N+1 entries)

// layer flags (device)
constexpr uint32_t kLayerPassthrough = 1u;
constexpr uint32_t kLayerClip = 2u;     // clip this layer (clipping on, not passthrough)
constexpr uint32_t kLayerVecIn = 4u;    // gradient pointer is 16-byte aligned
constexpr uint32_t kLayerVecOut = 8u;   // output pointer is 16-byte aligned
constexpr uint32_t kLayerShiftBit = 16; // bits 16-17: block start within the tensor & 3
// FixedSize(k) with k a power of two in [64, chunk): work items span whole
// buckets (nblk consecutive blocks of one tensor, contiguous in the tensor, in
// the push area -- k/4 code bytes, a 16-B multiple -- and in the scaler slots)
constexpr uint32_t kLayerMultiBucket = 32u;
constexpr uint32_t kBucketShiftBit = 24;  // bits 24-28: log2(k) of a multi-bucket tensor

// A block: one bucket of one tensor (PerTensor/Global: the whole tensor;
// FixedSize(k): [off, off+k) of it, codec.hpp:224-232) or a passthrough tensor.
struct LayerDev {
    const float* g;      // block's first gradient element
    float* out;          // block's first averaged-output element
    uint64_t code_off;   // byte offset in a push area: packed codes, or raw fp32 (passthrough)
    uint32_t n;          // elements in the block
    uint32_t tensor;     // owning tensor (K1 statistics are per tensor, codec.hpp:206-209)
    uint32_t key0, key1; // Philox key of RngStream(seed, *, tensor name, worker)
    int32_t slot;        // scaler slot (passthrough: -1)
    uint32_t flags;
    uint32_t rng_q;      // block start within the tensor >> 2 (ternarize rng_base, :167)
    uint32_t sum_off16;  // sharded exchange: block's region in the sums buffer, 16-B units
    uint32_t first_chunk, n_chunks;  // K1 work items of the TENSOR (group-relative)
};

struct ChunkDev {
    uint32_t layer;  // block index (multi-bucket items: the first of nblk blocks)
    uint32_t count;  // elements in this chunk
    uint32_t begin;  // first element, relative to the block (multiple of 16; 0 multi-bucket)
    uint32_t nblk;   // blocks (buckets) the item spans: 1, or > 1 for multi-bucket items
};

// self-contained work item of the grid-per-chunk kernels: the chunk plus a
// copy of its block descriptor, fetched in one round trip (5 x LDG.128)
struct ChunkFat {
    LayerDev L;
    ChunkDev ch;
};

// K1 finalize: a tensor's blocks and, per block, its K1 work items
struct TensorDev {
    uint64_t n;                      // tensor elements (sigma over the whole tensor)
    uint32_t first_block, n_blocks;  // blocks of this tensor in the block table
    uint32_t flags;                  // kLayerClip
    uint32_t group_base;             // K1 two-level finalize: first group slot (> 64 units)
};

// per-chunk clip statistics (Chan et al. mergeable moments)
struct Partial {
    double n, mean, m2;
    float mx;
    uint32_t block;  // block (bucket) the work item belongs to
};

// Destinations of this rank's push area (scaler slots + packed codes): its own
// buffer plus, with peers attached, the same offset inside every other rank's
// gathered buffer, written directly over NVLink (IPC-mapped peer memory).
constexpr int kMaxPeers = 8;  // one NVSwitch box
constexpr int kMaxPieces = 8; // overlapped / sharded exchange: pieces of the K2 work list
struct PeerPush {
    uint8_t* base[kMaxPeers];
    int32_t n;       // number of destinations (>= 1)
    int32_t remote;  // destinations include peer memory (ordered by the step barrier)
};

// Sticky error word. The location kept is the smallest (tensor, element) over
// all raised errors -- the first one the reference's sequential loops would
// throw at -- stored complemented so one atomicMax keeps it and 0 means none.
struct ErrWord {
    uint32_t flags;
    uint32_t pad;
    unsigned long long inv_key;  // ~((layer + 1) << 40 | index)
    unsigned long long aux;      // TGB_E_SKEW: the first offending peer's iteration
    __host__ __device__ int32_t layer() const {
        return static_cast<int32_t>((~inv_key) >> 40) - 1;
    }
    __host__ __device__ uint64_t index() const { return (~inv_key) & ((1ull << 40) - 1); }
};

__device__ __forceinline__ void raise_error(ErrWord* e, uint32_t flag, int32_t layer,
                                            uint64_t index) {
    atomicOr(&e->flags, flag);
    const unsigned long long key =
        (static_cast<unsigned long long>(static_cast<uint32_t>(layer + 1) & 0xFFFFFFu) << 40) |
        (index & ((1ull << 40) - 1));
    atomicMax(&e->inv_key, ~key);
}

// an exchange error with a detail value (kept from the first raise of `flag`)
__device__ __forceinline__ void raise_error_aux(ErrWord* e, uint32_t flag, uint64_t index,
                                                unsigned long long aux) {
    const uint32_t old = atomicOr(&e->flags, flag);
    if (!(old & flag)) atomicExch(&e->aux, aux);
    atomicMax(&e->inv_key, ~(index & ((1ull << 40) - 1)));
}

// the step's exchange failed (iteration skew or a missing peer): decode kernels
// leave the outputs untouched
__device__ __forceinline__ bool exchange_failed(const ErrWord* e) {
    return (__ldcg(&e->flags) & (TGB_E_SKEW | TGB_E_PEER_TIMEOUT)) != 0u;
}

// ------------------------------------------------------------- optimizer
// OptimizerState::apply (optimizer.hpp:80-125), element k, in the reference's
// operation order and precision (x86-64 SSE: no FMA contraction):
//   Vanilla:  eff = g + f(wd)*w;            w -= f(rate)*eff
//   Momentum: eff = g + f(wd)*w; v = f(mu)*v + eff; w -= f(rate)*v
//   Adam (double): eff = g + wd*w; m = f(b1*m + (1-b1)*eff); v = f(b2*v + (1-b2)*eff*eff);
//            w -= f(rate * (m/bc1) / (sqrt(v/bc2) + eps))
struct OptArgs {
    int32_t rule;  // TGB_OPT_*
    float wd_f, mu_f, rate_f;
    double wd, b1, omb1, b2, omb2, eps, rate, bc1, bc2;
};

__device__ __forceinline__ void opt_apply1(const OptArgs& o, float g, float& w, float& s1,
                                           float& s2) {
    if (o.rule == 2) {  // Adam
        const double eff = __dadd_rn(static_cast<double>(g), __dmul_rn(o.wd, static_cast<double>(w)));
        s1 = static_cast<float>(__dadd_rn(__dmul_rn(o.b1, static_cast<double>(s1)), __dmul_rn(o.omb1, eff)));
        s2 = static_cast<float>(__dadd_rn(__dmul_rn(o.b2, static_cast<double>(s2)),
                                          __dmul_rn(__dmul_rn(o.omb2, eff), eff)));
        const double mhat = __ddiv_rn(static_cast<double>(s1), o.bc1);
        const double vhat = __ddiv_rn(static_cast<double>(s2), o.bc2);
        const double upd = __ddiv_rn(__dmul_rn(o.rate, mhat), __dadd_rn(__dsqrt_rn(vhat), o.eps));
        w = __fsub_rn(w, static_cast<float>(upd));
        return;
    }
    const float eff = __fadd_rn(g, __fmul_rn(o.wd_f, w));
    if (o.rule == 1) {  // Momentum (gradient-accumulation form)
        s1 = __fadd_rn(__fmul_rn(o.mu_f, s1), eff);
        w = __fsub_rn(w, __fmul_rn(o.rate_f, s1));
    } else {  // Vanilla
        w = __fsub_rn(w, __fmul_rn(o.rate_f, eff));
    }
}

// Fused decode -> optimizer: per block, the parameter and state bases (element
// 0 of the block); vec = all three 16-byte aligned.
struct OptDev {
    float* w;
    float* s1;  // velocity / first moment (nullptr if the rule has none)
    float* s2;  // second moment (Adam)
    uint32_t vec;
    uint32_t pad;
};

// apply to `nvalid` (<= 4) consecutive elements at w/s1/s2 with gradients g
__device__ __forceinline__ void opt_apply4(const OptArgs& o, float* w, float* s1, float* s2,
                                           float4 g, bool vec, uint32_t nvalid) {
    if (vec && nvalid == 4) {
        float4 wv = *reinterpret_cast<const float4*>(w);
        float4 a = s1 ? *reinterpret_cast<const float4*>(s1) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 b = s2 ? *reinterpret_cast<const float4*>(s2) : make_float4(0.f, 0.f, 0.f, 0.f);
        opt_apply1(o, g.x, wv.x, a.x, b.x);
        opt_apply1(o, g.y, wv.y, a.y, b.y);
        opt_apply1(o, g.z, wv.z, a.z, b.z);
        opt_apply1(o, g.w, wv.w, a.w, b.w);
        *reinterpret_cast<float4*>(w) = wv;
        if (s1) *reinterpret_cast<float4*>(s1) = a;
        if (s2) *reinterpret_cast<float4*>(s2) = b;
        return;
    }
    const float gg[4] = {g.x, g.y, g.z, g.w};
    for (uint32_t e = 0; e < nvalid; ++e) {
        float wv = w[e], a = s1 ? s1[e] : 0.0f, b = s2 ? s2[e] : 0.0f;
        opt_apply1(o, gg[e], wv, a, b);
        w[e] = wv;
        if (s1) s1[e] = a;
        if (s2) s2[e] = b;
    }
}

// wire format segments (kernels.cu, capi.cu)
struct WireSeg {
    uint64_t src_off;  // in the push area
    uint64_t dst_off;  // in the frame
    uint64_t bytes;
};
struct PullSeg {
    uint64_t src_off;  // first word (SharedSum) or first float (FloatAvg) in the payload
    float* out;
    uint32_t n, words;
    uint32_t base, m;  // 2N+1, digits per word
    float s, inv_n;
    uint32_t kind;     // 3 SharedSum, 4 FloatAvg (wire.hpp:99-100)
    uint32_t first_thread;  // prefix over segments of threads used
};

// ---------------------------------------------------------------- Philox
constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
constexpr uint32_t kWeyl0 = 0x9E3779B9u, kWeyl1 = 0xBB67AE85u;

// Plain Philox4x32-10 (rng.hpp:20-33)
__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(kMul0, c.x), lo0 = kMul0 * c.x;
        const uint32_t hi1 = __umulhi(kMul1, c.z), lo1 = kMul1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += kWeyl0;
        k1 += kWeyl1;
    }
    return c;
}

// ------------------------------------------------------ ternary decision
// Reference (codec.hpp:161-169 after clip :121-122):
//   mag = |clip(x)| = min(|x|, bound); p = RN(mag / s) (IEEE fp32 divide);
//   take iff u = RN(float(bits))*2^-32 < p; code = clip(x) > 0 ? 01 : 10.
//
// exact_take() decides u < RN(m/s) without dividing: RN(q) > u  <=>  q > mid
// (mid = midpoint of u and its successor), or q == mid and the successor's
// significand is even (ties-to-even). m, s*mid are exact in fp64 (s has 24
// significant bits, mid 25), so the test is exact for every finite input,
// including u == 0 and subnormal quotients.
__device__ __forceinline__ bool exact_take(float m, float s, float uf) {
    const float u = __fmul_rn(uf, 0x1p-32f);
    const float succ = __uint_as_float(__float_as_uint(u) + 1u);
    const double mid = (static_cast<double>(u) + static_cast<double>(succ)) * 0.5;
    const double t = static_cast<double>(s) * mid;
    const double dm = static_cast<double>(m);
    return dm > t || (dm == t && (__float_as_uint(succ) & 1u) == 0u);
}

// Fast form. Let c = bound (or s when there is no clip bound), R = RN(1/s)*2^32,
// rl = RN(c*R*(1-2^-20)), dr = RN(c*R*2^-19), m' = sat(|x| * RN(1/c)) ~ m/c.
//   d = uf - m'*rl  (one FFMA rounding: sign exact) :  d < 0  =>  u < p  (take)
// and d >= 0 decides "no take" unless uf lies in the margin band, which is
// contained in |d| <= m'*dr (z = m'*dr - |d| >= 0). Every approximation is a
// few 2^-24 relative roundings, well inside the 2^-20 margin, so only z >= 0
// (probability ~2^-18) or bits == 0 (uf == 0, flagged through -uf) needs
// exact_take. Valid for 2^-90 <= s <= 2^120 (else exact_all). The fast path is
// pure FP32 (FMUL.SAT/FFMA/FMNMX3), leaving the integer multiplier (IMAD.WIDE,
// fma-heavy) to Philox.
struct Decider {
    float bound, s;
    float ib, rl, dr;  // RN(1/c), c*R*(1-2^-20), c*R*2^-19
    bool exact_all;

    __device__ __forceinline__ void init(float bound_, float s_) {
        bound = bound_;
        s = s_;
        exact_all = !(s_ >= 0x1p-90f) || s_ > 0x1p+120f;
        const float c = bound_ < INFINITY ? bound_ : s_;
        const float rc = __fmul_rn(__fmul_rn(__frcp_rn(s_), 4294967296.0f), c);
        ib = __frcp_rn(c);
        rl = __fmul_rn(rc, 1.0f - 0x1p-20f);
        dr = __fmul_rn(rc, 0x1p-19f);
    }

    // 2-bit code for a taken element: 1 + sign (01 positive, 10 negative)
    __device__ __forceinline__ static uint32_t sign_code(float x) {
        return (__float_as_uint(x) >> 31) + 1u;
    }

    // fast decision, FP form: returns the 2-bit code as a float in {0, 1, 2};
    // amb = max(amb, z, -uf) >= 0 flags "needs the exact test"
    __device__ __forceinline__ float code_fast(float x, uint32_t bits, float& amb) const {
        const float mp = __saturatef(__fmul_rn(fabsf(x), ib));
        const float uf = __uint2float_rn(bits);
        const float d = __fmaf_rn(-mp, rl, uf);
        const float z = __fmaf_rn(mp, dr, -fabsf(d));
        amb = fmaxf(amb, fmaxf(z, -uf));
        // d < 0 => |d| >= 2^-47 (uf >= 1 integer, m'*rl a product of floats > 1),
        // and a taken x has |x| >= 2^-122: both saturate to exactly 1.0
        const float t = __saturatef(__fmul_rn(d, -0x1p126f));
        const float sg = __saturatef(__fmul_rn(x, -0x1p126f));
        return __fmaf_rn(t, sg, t);  // t * (1 + sign)
    }

    __device__ __forceinline__ uint32_t code_exact(float x, uint32_t bits) const {
        const float m = fminf(fabsf(x), bound);
        return exact_take(m, s, __uint2float_rn(bits)) ? sign_code(x) : 0u;
    }

    // one element's code (fast form, exact when flagged)
    __device__ __forceinline__ uint32_t code(float x, uint32_t bits) const {
        if (!exact_all) {
            float amb = -1.0f;
            const float c = code_fast(x, bits, amb);
            if (!(amb >= 0.0f)) return static_cast<uint32_t>(c);
        }
        return code_exact(x, bits);
    }

    __device__ __forceinline__ uint32_t byte_exact(float4 v, uint4 r) const {
        return code_exact(v.x, r.x) | (code_exact(v.y, r.y) << 2) | (code_exact(v.z, r.z) << 4) |
               (code_exact(v.w, r.w) << 6);
    }

    // fast byte as float value in [0, 255] (exact); amb >= 0 flags an element
    // that needs the exact test (margin band, or bits == 0).
    __device__ __forceinline__ float byte_fast_f(float4 v, uint4 r, float& amb) const {
        const float c0 = code_fast(v.x, r.x, amb), c1 = code_fast(v.y, r.y, amb);
        const float c2 = code_fast(v.z, r.z, amb), c3 = code_fast(v.w, r.w, amb);
        return __fmaf_rn(__fmaf_rn(__fmaf_rn(c3, 4.0f, c2), 4.0f, c1), 4.0f, c0);
    }

    // float byte value -> integer (low 8 bits of the bit pattern of 2^23 + v)
    __device__ __forceinline__ static uint32_t to_u8(float bf) {
        return __float_as_uint(__fadd_rn(bf, 8388608.0f)) & 0xFFu;
    }

    __device__ __forceinline__ uint32_t byte_fast(float4 v, uint4 r, float& amb) const {
        return to_u8(byte_fast_f(v, r, amb));
    }

    // one code byte (4 elements, one Philox block)
    __device__ __forceinline__ uint32_t byte(float4 v, uint4 r) const {
        if (!exact_all) {
            float amb = -1.0f;
            const uint32_t c = byte_fast(v, r, amb);
            if (!(amb >= 0.0f)) return c;
        }
        return byte_exact(v, r);
    }
};

// Four independent Philox4x32-10 blocks, round-interleaved for ILP. Round 0's
// ctr2 product is hoisted. kRolling: derive round keys with one add per round
// (shared by the U lanes) instead of holding 18 key registers.
template <bool kRolling = false>
struct Philox4 {
    uint32_t r1x, r1y, r1wk;
    uint32_t ka[10], kb[10];

    __device__ __forceinline__ void init(uint32_t key0, uint32_t key1, uint32_t ctr1, uint64_t t) {
        const uint32_t t_lo = static_cast<uint32_t>(t), t_hi = static_cast<uint32_t>(t >> 32);
        r1x = __umulhi(kMul1, t_lo) ^ ctr1 ^ key0;
        r1y = kMul1 * t_lo;
        r1wk = t_hi ^ key1;
        if (kRolling) {
            ka[0] = key0;
            kb[0] = key1;
        } else {
#pragma unroll
            for (int r = 0; r < 10; ++r) {
                ka[r] = key0 + static_cast<uint32_t>(r) * kWeyl0;
                kb[r] = key1 + static_cast<uint32_t>(r) * kWeyl1;
            }
        }
    }

    template <int U>
    __device__ __forceinline__ void operator()(const uint32_t (&ctr0)[U], uint4 (&c)[U]) const {
#pragma unroll
        for (int u = 0; u < U; ++u)
            c[u] = make_uint4(r1x, r1y, __umulhi(kMul0, ctr0[u]) ^ r1wk, kMul0 * ctr0[u]);
        uint32_t a = ka[0], b = kb[0];
#pragma unroll
        for (int r = 1; r < 10; ++r) {
            if (kRolling) {
                a += kWeyl0;
                b += kWeyl1;
            } else {
                a = ka[r];
                b = kb[r];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t hi0 = __umulhi(kMul0, c[u].x), lo0 = kMul0 * c[u].x;
                const uint32_t hi1 = __umulhi(kMul1, c[u].z), lo1 = kMul1 * c[u].z;
                c[u] = make_uint4(hi1 ^ c[u].y ^ a, lo1, hi0 ^ c[u].w ^ b, lo0);
            }
        }
    }
};

// ---------------------------------------------------------- fp64 moments
__device__ __forceinline__ void chan_merge(double& n, double& mean, double& m2, double nb,
                                           double meanb, double m2b) {
    if (nb == 0.0) return;
    if (n == 0.0) {
        n = nb;
        mean = meanb;
        m2 = m2b;
        return;
    }
    const double nn = n + nb;
    const double delta = meanb - mean;
    const double f = nb / nn;
    mean = mean + delta * f;
    m2 = m2 + m2b + delta * delta * n * f;
    n = nn;
}

// Barriers for block-wide phases: the whole CTA, or only the 256 consumer
// threads of a warp-specialized CTA (named barrier 1; the producer warp never
// joins, so __syncthreads would deadlock there).
struct BlockBar {
    __device__ __forceinline__ static void sync() { __syncthreads(); }
};
struct ConsumerBar {
    __device__ __forceinline__ static void sync() {
        asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
    }
};

// deterministic CTA reduction of (S, Q, mx) — fixed shuffle tree + fixed warp order
template <int kWarps, class Bar = BlockBar>
__device__ __forceinline__ void block_reduce_sq(double& S, double& Q, float& mx) {
    __shared__ double sh_s[kWarps], sh_q[kWarps];
    __shared__ float sh_m[kWarps];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        S += __shfl_down_sync(0xffffffffu, S, o);
        Q += __shfl_down_sync(0xffffffffu, Q, o);
        mx = fmaxf(mx, __shfl_down_sync(0xffffffffu, mx, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sh_s[warp] = S;
        sh_q[warp] = Q;
        sh_m[warp] = mx;
    }
    Bar::sync();
    if (threadIdx.x == 0) {
        S = sh_s[0];
        Q = sh_q[0];
        mx = sh_m[0];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) {
            S += sh_s[w];
            Q += sh_q[w];
            mx = fmaxf(mx, sh_m[w]);
        }
    }
}

}  // namespace tgb
