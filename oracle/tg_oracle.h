/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the TernGrad reference's
 * ternarize + sync + decode path, used as the parity checker.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. The product path (paper_1705_07878_b200/, libtgb) never
 * links or calls it; there is no CPU fallback.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/terngrad/).
 * Parity status: PINNED — tests/test_oracle.py checks this restatement
 * against (a) the Random123 Philox4x32-10 KATs, (b) SURVEY Appendix B KATs,
 * and (c) byte-for-byte against oracle/_ref (the reference headers compiled
 * unmodified) on the golden fixtures in tests/golden/.
 */
#ifndef TG_ORACLE_H
#define TG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes, mirror CodecError sites in codec.hpp */
enum {
    TGO_OK = 0,
    TGO_ERR_SCALER_BELOW_MAX = 1, /* codec.hpp:163-165 */
    TGO_ERR_S0_NONZERO = 2,       /* codec.hpp:155-158 */
    TGO_ERR_NONFINITE = 3,        /* codec.hpp:205 */
    TGO_ERR_CORRUPT_CODE = 4,     /* codec.hpp:42-44 */
    TGO_ERR_INVALID = 5           /* codec.hpp:90-95 / 247-256 */
};

/* rng.hpp:20-33 */
void tgo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* rng.hpp:37-44 */
uint64_t tgo_fnv1a64(const char* s, size_t len);

/* rng.hpp:48-84 */
typedef struct {
    uint32_t key[2];
    uint32_t hi[2];
} tgo_rng;

void tgo_rng_init(tgo_rng* r, uint64_t seed, uint64_t iteration, const char* name,
                  size_t name_len, uint64_t worker);
void tgo_rng_init_hash(tgo_rng* r, uint64_t seed, uint64_t iteration, uint64_t name_hash,
                       uint64_t worker);
uint32_t tgo_rng_bits(const tgo_rng* r, uint64_t index);
float tgo_rng_uniform(const tgo_rng* r, uint64_t index);
float tgo_rng_normal(const tgo_rng* r, uint64_t index);
/* fills out[k] = scale * normal(k0 + k) */
void tgo_rng_normal_fill(const tgo_rng* r, uint64_t k0, size_t n, float scale, float* out);

/* codec.hpp:101-112 */
double tgo_stddev(const float* v, size_t n);
/* codec.hpp:117-124; writes clipped copy, returns bound (+inf when n < 2) */
float tgo_clip(const float* in, size_t n, float c, float* out);
/* codec.hpp:128-134 */
float tgo_scaler(const float* v, size_t n);
/* codec.hpp:136-141; returns -1 (as status) on empty list through *status */
float tgo_share_scalers(const float* s, size_t n, int* status);
/* codec.hpp:148-175; codes must hold (n+3)/4 bytes */
int tgo_ternarize(const float* g, size_t n, float s, const tgo_rng* rng, uint64_t rng_base,
                  uint8_t* codes);
/* codec.hpp:177-182 */
int tgo_decode(const uint8_t* codes, size_t n, float s, float* out);

/* codec.hpp:78-96 */
enum { TGO_PER_TENSOR = 0, TGO_GLOBAL = 1, TGO_FIXED_SIZE = 2 };
typedef struct {
    float clip_factor;
    int clipping_enabled;
    int bucketing;
    uint64_t bucket_size;
    int scaler_sharing;
    uint64_t seed;
} tgo_codec_config;

/*
 * codec.hpp:194-239 (encode_step). Tensors are given as pointer arrays.
 * passthrough[l] != 0 marks a tensor named in cfg.passthrough.
 * Block layout produced (canonical order, matches EncodedGradient.blocks):
 *   per non-passthrough tensor: ceil(n/bucket) blocks (1 for empty tensors),
 *   each block's codes packed back to back into `codes` (ceil(len/4) bytes),
 *   scalers[] receives one scaler per block (= EncodeResult.local_scalers).
 * Passthrough tensors produce no codes/scalers (values are used verbatim).
 * Returns status; *bad_tensor receives the offending tensor on error.
 */
int tgo_encode_step(int n_tensors, const char* const* names, const uint64_t* ns,
                    const float* const* grads, const int* passthrough,
                    const tgo_codec_config* cfg, uint64_t t, uint16_t worker,
                    uint8_t* codes, float* scalers, float* bounds, int* bad_tensor);
/* sizes for the above layout */
void tgo_encode_layout(int n_tensors, const uint64_t* ns, const int* passthrough,
                       const tgo_codec_config* cfg, uint64_t* code_bytes, uint64_t* n_blocks);

/*
 * codec.hpp:281-307 (average, one ternary block): N workers' codes for one
 * block of n elements, scalers s[w]. sharing: s=max, int sums, s*float(sum)*invN.
 * Without sharing: fp64 sum of s_w*code in worker order, float(sum/N).
 */
int tgo_average_block(int N, const float* s, const uint8_t* const* codes, size_t n,
                      int sharing, float* out);
/* codec.hpp:269-279: fp64 worker-order mean of raw floats */
void tgo_average_passthrough(int N, const float* const* vals, size_t n, float* out);

/* wire.hpp:79-85,206-228 + cluster.hpp:189-204: integer code sums and decode_pull */
int tgo_code_sums(int N, const uint8_t* const* codes, size_t n, int32_t* sums);
void tgo_decode_pull_shared(float s, int N, const int32_t* sums, size_t n, float* out);

#ifdef __cplusplus
}
#endif
#endif
