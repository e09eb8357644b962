/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement (plain C) of the reference's
 * TernGrad hot path. See tg_oracle.h for the usage rule and pinning status.
 * Compile with -O2 -ffp-contract=off (no FMA contraction, matching the
 * reference's x86-64 Release build where no FMA is emitted).
 */
#include "tg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* rng.hpp:15-33 — Philox4x32-10 (Random123 constants) */
void tgo_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.hpp:37-44 */
uint64_t tgo_fnv1a64(const char* s, size_t len) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < len; ++i) {
        h ^= (unsigned char)s[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* rng.hpp:50-57 */
void tgo_rng_init_hash(tgo_rng* r, uint64_t seed, uint64_t iteration, uint64_t nh,
                       uint64_t worker) {
    r->key[0] = (uint32_t)(seed ^ nh);
    r->key[1] = (uint32_t)((seed >> 32) ^ (nh >> 32) ^ (worker * 0x9E3779B97F4A7C15ull));
    r->hi[0] = (uint32_t)iteration;
    r->hi[1] = (uint32_t)(iteration >> 32);
}

void tgo_rng_init(tgo_rng* r, uint64_t seed, uint64_t iteration, const char* name,
                  size_t name_len, uint64_t worker) {
    tgo_rng_init_hash(r, seed, iteration, tgo_fnv1a64(name, name_len), worker);
}

/* rng.hpp:59-66 */
uint32_t tgo_rng_bits(const tgo_rng* r, uint64_t index) {
    const uint64_t ctr = index >> 2;
    const uint32_t c[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), r->hi[0], r->hi[1]};
    uint32_t out[4];
    tgo_philox4x32_10(c, r->key, out);
    return out[index & 3];
}

/* rng.hpp:69-71 — note: 1.0f IS reachable (bits >= 0xFFFFFF80 round up) */
float tgo_rng_uniform(const tgo_rng* r, uint64_t index) {
    return (float)tgo_rng_bits(r, index) * 0x1p-32f;
}

/* rng.hpp:74-79 */
float tgo_rng_normal(const tgo_rng* r, uint64_t index) {
    const double u1 = ((double)tgo_rng_bits(r, 2 * index) + 0.5) * 0x1p-32;
    const double u2 = (double)tgo_rng_bits(r, 2 * index + 1) * 0x1p-32;
    return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

void tgo_rng_normal_fill(const tgo_rng* r, uint64_t k0, size_t n, float scale, float* out) {
    for (size_t k = 0; k < n; ++k) out[k] = scale * tgo_rng_normal(r, k0 + k);
}

/* codec.hpp:101-112 — sequential fp64 two-pass population sigma */
double tgo_stddev(const float* v, size_t n) {
    if (n < 2) return 0.0;
    double mean = 0.0;
    for (size_t k = 0; k < n; ++k) mean += v[k];
    mean /= (double)n;
    double var = 0.0;
    for (size_t k = 0; k < n; ++k) {
        const double d = v[k] - mean;
        var += d * d;
    }
    return sqrt(var / (double)n);
}

/* codec.hpp:117-124 — c is promoted to double before the product (:119) */
float tgo_clip(const float* in, size_t n, float c, float* out) {
    if (out != in) memcpy(out, in, n * sizeof(float));
    if (n < 2) return INFINITY;
    const float bound = (float)((double)c * tgo_stddev(in, n));
    for (size_t k = 0; k < n; ++k)
        if (fabsf(out[k]) > bound) out[k] = copysignf(bound, out[k]);
    return bound;
}

/* codec.hpp:128-134 — std::max(m, |x|) keeps m on ties */
float tgo_scaler(const float* v, size_t n) {
    float m = 0.0f;
    for (size_t k = 0; k < n; ++k) {
        const float a = fabsf(v[k]);
        if (m < a) m = a;
    }
    return m;
}

/* codec.hpp:136-141 */
float tgo_share_scalers(const float* s, size_t n, int* status) {
    if (n == 0) {
        if (status) *status = TGO_ERR_INVALID;
        return 0.0f;
    }
    float m = 0.0f;
    for (size_t k = 0; k < n; ++k)
        if (m < s[k]) m = s[k];
    if (status) *status = TGO_OK;
    return m;
}

/* codec.hpp:148-175 — element k at bits 2(k%4) of byte k/4 (:19-23, :48-52) */
int tgo_ternarize(const float* g, size_t n, float s, const tgo_rng* rng, uint64_t rng_base,
                  uint8_t* codes) {
    memset(codes, 0, (n + 3) / 4);
    if (s == 0.0f) {
        for (size_t k = 0; k < n; ++k)
            if (g[k] != 0.0f) return TGO_ERR_S0_NONZERO;
        return TGO_OK;
    }
    for (size_t k = 0; k < n; ++k) {
        const float mag = fabsf(g[k]);
        if (mag > s) return TGO_ERR_SCALER_BELOW_MAX;
        const float p = mag / s;
        if (tgo_rng_uniform(rng, rng_base + k) < p) {
            const uint8_t c = g[k] > 0.0f ? 0x1 : 0x2;
            codes[k / 4] = (uint8_t)((codes[k / 4] & ~(0x3u << (2 * (k % 4)))) |
                                     (unsigned)(c << (2 * (k % 4))));
        }
    }
    return TGO_OK;
}

/* codec.hpp:36-46 */
static int code_at(const uint8_t* codes, size_t k, int* v) {
    const unsigned c = (codes[k / 4] >> (2 * (k % 4))) & 0x3u;
    switch (c) {
        case 0: *v = 0; return TGO_OK;
        case 1: *v = 1; return TGO_OK;
        case 2: *v = -1; return TGO_OK;
        default: return TGO_ERR_CORRUPT_CODE;
    }
}

/* codec.hpp:177-182 */
int tgo_decode(const uint8_t* codes, size_t n, float s, float* out) {
    for (size_t k = 0; k < n; ++k) {
        int v;
        const int st = code_at(codes, k, &v);
        if (st) return st;
        out[k] = s * (float)v;
    }
    return TGO_OK;
}

static int all_finite(const float* v, size_t n) {
    for (size_t k = 0; k < n; ++k)
        if (!isfinite(v[k])) return 0;
    return 1;
}

/* layout helper for tgo_encode_step (codec.hpp:218-237 block structure) */
void tgo_encode_layout(int n_tensors, const uint64_t* ns, const int* passthrough,
                       const tgo_codec_config* cfg, uint64_t* code_bytes, uint64_t* n_blocks) {
    uint64_t bytes = 0, blocks = 0;
    for (int l = 0; l < n_tensors; ++l) {
        if (passthrough && passthrough[l]) continue;
        const uint64_t n = ns[l];
        if (n == 0) { blocks += 1; continue; }
        const uint64_t bucket = cfg->bucketing == TGO_FIXED_SIZE ? cfg->bucket_size : n;
        for (uint64_t off = 0; off < n; off += bucket) {
            const uint64_t len = (n - off) < bucket ? (n - off) : bucket;
            bytes += (len + 3) / 4;
            blocks += 1;
        }
    }
    if (code_bytes) *code_bytes = bytes;
    if (n_blocks) *n_blocks = blocks;
}

/* codec.hpp:194-239 */
int tgo_encode_step(int n_tensors, const char* const* names, const uint64_t* ns,
                    const float* const* grads, const int* passthrough,
                    const tgo_codec_config* cfg, uint64_t t, uint16_t worker,
                    uint8_t* codes, float* scalers, float* bounds, int* bad_tensor) {
    if (!(cfg->clip_factor > 0.0f)) return TGO_ERR_INVALID;                  /* :91 */
    if (cfg->bucketing == TGO_FIXED_SIZE && cfg->bucket_size < 1) return TGO_ERR_INVALID;
    float** work = (float**)calloc((size_t)n_tensors, sizeof(float*));
    int status = TGO_OK;
    for (int l = 0; l < n_tensors; ++l) {                                     /* :204-210 */
        const size_t n = (size_t)ns[l];
        if (!all_finite(grads[l], n)) {
            status = TGO_ERR_NONFINITE;
            if (bad_tensor) *bad_tensor = l;
            goto done;
        }
        work[l] = (float*)malloc(n ? n * sizeof(float) : 1);
        const int pt = passthrough && passthrough[l];
        if (pt || !cfg->clipping_enabled) {
            memcpy(work[l], grads[l], n * sizeof(float));
            if (bounds) bounds[l] = INFINITY;
        } else {
            const float b = tgo_clip(grads[l], n, cfg->clip_factor, work[l]);
            if (bounds) bounds[l] = b;
        }
    }
    float global_s = 0.0f;                                                    /* :212-216 */
    if (cfg->bucketing == TGO_GLOBAL) {
        for (int l = 0; l < n_tensors; ++l) {
            if (passthrough && passthrough[l]) continue;
            const float s = tgo_scaler(work[l], (size_t)ns[l]);
            if (global_s < s) global_s = s;
        }
    }
    uint64_t code_pos = 0, block = 0;
    for (int l = 0; l < n_tensors; ++l) {                                     /* :218-237 */
        if (passthrough && passthrough[l]) continue;
        const size_t n = (size_t)ns[l];
        tgo_rng rng;
        tgo_rng_init(&rng, cfg->seed, t, names[l], strlen(names[l]), worker);
        const size_t bucket = cfg->bucketing == TGO_FIXED_SIZE ? (size_t)cfg->bucket_size : n;
        for (size_t off = 0; off < n; off += bucket) {
            const size_t len = (n - off) < bucket ? (n - off) : bucket;
            const float s = cfg->bucketing == TGO_GLOBAL ? global_s : tgo_scaler(work[l] + off, len);
            scalers[block++] = s;
            status = tgo_ternarize(work[l] + off, len, s, &rng, off, codes + code_pos);
            if (status) {
                if (bad_tensor) *bad_tensor = l;
                goto done;
            }
            code_pos += (len + 3) / 4;
        }
        if (n == 0) scalers[block++] = 0.0f;                                  /* :233-236 */
    }
done:
    for (int l = 0; l < n_tensors; ++l) free(work[l]);
    free(work);
    return status;
}

/* codec.hpp:281-307 (one ternary block of `average`) */
int tgo_average_block(int N, const float* s, const uint8_t* const* codes, size_t n,
                      int sharing, float* out) {
    if (N <= 0) return TGO_ERR_INVALID;
    const float invN = 1.0f / (float)N;                                       /* :267 */
    if (sharing) {
        float sm = 0.0f;                                                      /* :289-291 */
        for (int w = 0; w < N; ++w)
            if (sm < s[w]) sm = s[w];
        for (size_t k = 0; k < n; ++k) {                                      /* :292-297 */
            int sum = 0;
            for (int w = 0; w < N; ++w) {
                int v;
                const int st = code_at(codes[w], k, &v);
                if (st) return st;
                sum += v;
            }
            out[k] = sm * (float)sum * invN;
        }
    } else {
        for (size_t k = 0; k < n; ++k) {                                      /* :299-306 */
            double sum = 0.0;
            for (int w = 0; w < N; ++w) {
                int v;
                const int st = code_at(codes[w], k, &v);
                if (st) return st;
                sum += (double)s[w] * v;
            }
            out[k] = (float)(sum / (double)N);
        }
    }
    return TGO_OK;
}

/* codec.hpp:269-279 */
void tgo_average_passthrough(int N, const float* const* vals, size_t n, float* out) {
    for (size_t k = 0; k < n; ++k) {
        double sum = 0.0;
        for (int w = 0; w < N; ++w) sum += vals[w][k];
        out[k] = (float)(sum / (double)N);
    }
}

/* cluster.hpp:197-203 */
int tgo_code_sums(int N, const uint8_t* const* codes, size_t n, int32_t* sums) {
    for (size_t k = 0; k < n; ++k) sums[k] = 0;
    for (int w = 0; w < N; ++w)
        for (size_t k = 0; k < n; ++k) {
            int v;
            const int st = code_at(codes[w], k, &v);
            if (st) return st;
            sums[k] += v;
        }
    return TGO_OK;
}

/* wire.hpp:216-221 */
void tgo_decode_pull_shared(float s, int N, const int32_t* sums, size_t n, float* out) {
    const float invN = 1.0f / (float)N;
    for (size_t k = 0; k < n; ++k) out[k] = s * (float)sums[k] * invN;
}
