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

namespace tgb {

constexpr int kThreads = 256;       // CTA size of every streaming kernel
constexpr uint32_t kChunk = 16384;  // elements per work item (multiple of 16)
constexpr int kMaxWorkers = 64;     // decode LUT capacity (2N+1 entries)

// layer flags (device)
constexpr uint32_t kLayerPassthrough = 1u;
constexpr uint32_t kLayerClip = 2u;     // clip this layer (clipping on, not passthrough)
constexpr uint32_t kLayerVecIn = 4u;    // gradient pointer is 16-byte aligned
constexpr uint32_t kLayerVecOut = 8u;   // output pointer is 16-byte aligned

struct LayerDev {
    const float* g;      // worker gradient (input)
    float* out;          // averaged gradient (output of decode)
    uint64_t n;          // elements
    uint64_t code_off;   // byte offset of the packed codes inside a push buffer
    uint32_t key0, key1; // Philox key of RngStream(seed, *, name, worker)
    int32_t slot;        // scaler slot
    uint32_t flags;
    uint32_t first_chunk, n_chunks;
};

struct ChunkDev {
    uint32_t layer;
    uint32_t count;  // elements in this chunk
    uint64_t begin;  // first element (multiple of 4, and of kChunk inside a layer)
};

// per-chunk clip statistics (Chan et al. mergeable moments)
struct Partial {
    double n, mean, m2;
    float mx;
    uint32_t pad;
};

struct ErrWord {
    uint32_t flags;
    int32_t layer;
    unsigned long long index;
};

__device__ __forceinline__ void raise_error(ErrWord* e, uint32_t flag, int32_t layer,
                                            uint64_t index) {
    const uint32_t prev = atomicOr(&e->flags, flag);
    if (prev == 0u) {  // first error wins the location fields
        e->layer = layer;
        e->index = index;
    }
}

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

// Philox with the counter words 1..3 fixed for a whole work item
// (ctr1 = hi32 of the byte index, ctr2/3 = iteration). Round 1's c.z product
// is invariant, so it is hoisted: per byte only 19 wide multiplies remain.
struct PhiloxStream {
    uint32_t k0, k1;   // key
    uint32_t r1x, r1y; // round-1 outputs that do not depend on ctr0
    uint32_t r1wk;     // ctr3 ^ k1 (round-1 z input)

    __device__ __forceinline__ void init(uint32_t key0, uint32_t key1, uint32_t ctr1,
                                         uint64_t t) {
        k0 = key0;
        k1 = key1;
        const uint32_t t_lo = static_cast<uint32_t>(t), t_hi = static_cast<uint32_t>(t >> 32);
        r1x = __umulhi(kMul1, t_lo) ^ ctr1 ^ key0;
        r1y = kMul1 * t_lo;
        r1wk = t_hi ^ key1;
    }

    __device__ __forceinline__ uint4 operator()(uint32_t ctr0) const {
        uint4 c = make_uint4(r1x, r1y, __umulhi(kMul0, ctr0) ^ r1wk, kMul0 * ctr0);
        uint32_t a = k0 + kWeyl0, b = k1 + kWeyl1;
#pragma unroll
        for (int r = 1; r < 10; ++r) {
            const uint32_t hi0 = __umulhi(kMul0, c.x), lo0 = kMul0 * c.x;
            const uint32_t hi1 = __umulhi(kMul1, c.z), lo1 = kMul1 * c.z;
            c = make_uint4(hi1 ^ c.y ^ a, lo1, hi0 ^ c.w ^ b, lo0);
            a += kWeyl0;
            b += kWeyl1;
        }
        return c;
    }
};

// ------------------------------------------------------ ternary decision
// Reference (codec.hpp:161-169 after clip :121-122):
//   mag = |clip(x)| = min(|x|, bound); p = mag / s (IEEE fp32 divide);
//   take iff float(bits)*2^-32 < p; code = clip(x) > 0 ? 01 : 10.
// Device: the divide is replaced by two products with a per-layer reciprocal
// carrying a +-2^-20 relative margin (provably decisive outside it, see
// DESIGN.md §K2); inside the margin, or for bits == 0, the exact IEEE divide
// decides. Bit-exact with the reference for every input.
struct Decider {
    float bound, s;
    float r_lo, r_hi;  // RN(1/s)*2^32*(1 -+ 2^-20)
    bool exact_all;    // s too small for the reciprocal form

    __device__ __forceinline__ void init(float bound_, float s_) {
        bound = bound_;
        s = s_;
        exact_all = !(s_ >= 0x1p-90f) || s_ > 0x1p+120f;  // keep RN(1/s)*2^32 normal and finite
        const float r = __fmul_rn(__frcp_rn(s_), 4294967296.0f);
        r_lo = __fmul_rn(r, 1.0f - 0x1p-20f);
        r_hi = __fmul_rn(r, 1.0f + 0x1p-20f);
    }

    // returns the 2-bit code of one element
    __device__ __forceinline__ uint32_t code(float x, uint32_t bits) const {
        const float m = fminf(fabsf(x), bound);
        const float uf = __uint2float_rn(bits);
        bool take;
        if (!exact_all) {
            const float a = __fmul_rn(m, r_lo);
            const float b = __fmul_rn(m, r_hi);
            take = uf < a;
            const bool amb = (!take && !(uf > b)) || bits == 0u;
            if (amb) take = __fmul_rn(uf, 0x1p-32f) < __fdiv_rn(m, s);
        } else {
            take = __fmul_rn(uf, 0x1p-32f) < __fdiv_rn(m, s);
        }
        const uint32_t sign = __float_as_uint(x) >> 31;  // taken => x != 0
        return take ? (1u + sign) : 0u;
    }

    __device__ __forceinline__ uint32_t byte(float4 v, uint4 r) const {
        return code(v.x, r.x) | (code(v.y, r.y) << 2) | (code(v.z, r.z) << 4) |
               (code(v.w, r.w) << 6);
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

// deterministic CTA reduction of (S, Q, mx) — fixed shuffle tree + fixed warp order
template <int kWarps>
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
    __syncthreads();
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
