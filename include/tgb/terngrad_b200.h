/*
 * terngrad_b200 — C-ABI of the B200-native TernGrad gradient-synchronisation path.
 *
 * This is the drop-in boundary. The reference (arxiv 1705.07878 CPU library,
 * /root/reference/proj/include/terngrad/) exposes the path as header-only C++
 * free functions in namespace `terngrad` with value semantics and exceptions;
 * it has no FFI of its own. Each entry point below names the reference
 * function it replaces (file:line, relative to proj/include/terngrad/).
 * The C++ value-semantics mirror lives in include/tgb/terngrad.hpp, the Python
 * mirror in paper_1705_07878_b200/ (ctypes); both sit on this header only.
 *
 * Conventions
 *  - All data pointers named d_* are DEVICE pointers (CUDA global memory).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is stream-ordered and asynchronous unless stated otherwise;
 *    nothing allocates on the per-step path.
 *  - Errors that the reference raises as exceptions are reported through a
 *    device error word (tgb_error), read with tgb_check()/tgb_layer_check()
 *    which synchronise. The flags map 1:1 to the reference's CodecError
 *    sites; the C++/Python wrappers rethrow with the reference's messages.
 *  - No CPU fallback: if no sm_100 device is present every compute entry
 *    point returns TGB_ERR_CUDA.
 */
#ifndef TGB_TERNGRAD_B200_H
#define TGB_TERNGRAD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGB_ABI_VERSION 2

typedef enum tgb_status {
    TGB_OK = 0,
    TGB_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument, codec.hpp:90-95 */
    TGB_ERR_CODEC = 2,            /* CodecError, codec.hpp:25-27 (detail: tgb_error) */
    TGB_ERR_CUDA = 3,
    TGB_ERR_NCCL = 4,
    TGB_ERR_UNSUPPORTED = 5,
    TGB_ERR_PROTOCOL = 6 /* ProtocolError, wire.hpp:14-16 (text: tgb_last_error_message) */
} tgb_status;

/* device error word: flags are sticky until read by tgb_check */
#define TGB_E_NONFINITE 0x1u        /* "encode_step: non-finite gradient <name>" codec.hpp:205 */
#define TGB_E_SCALER_BELOW_MAX 0x2u /* "ternarize: scaler <s> below max |g| in <name>" :163-165 */
#define TGB_E_S0_NONZERO 0x4u       /* "ternarize: s=0 but gradient has nonzero element" :155-158 */
#define TGB_E_CORRUPT_CODE 0x8u     /* "corrupt ternary code 11 in block <name> at element <k>" :42-44 */
#define TGB_E_PEER_TIMEOUT 0x10u    /* fused exchange: a peer never reached the barrier (index = peer) */
#define TGB_E_SKEW 0x20u            /* "server: iteration skew, expected <t> got <t'>" cluster.hpp:141-143:
                                       a peer stepped a different iteration (index = peer, aux = its t).
                                       The step's decode is skipped (outputs keep the previous step). */

typedef struct tgb_error {
    uint32_t flags;
    int32_t layer;  /* first offending tensor (plan layer index) or -1 */
    uint64_t index; /* first offending element within that tensor (when known) */
    uint64_t aux;   /* TGB_E_SKEW: the offending peer's iteration; else 0 */
} tgb_error;

/* one gradient tensor of the canonical parameter order (tensor.hpp:14-43) */
#define TGB_LAYER_PASSTHROUGH 0x1u /* name in CodecConfig::passthrough (codec.hpp:87) */
typedef struct tgb_layer_desc {
    uint64_t n;         /* element count (GradTensor::element_count) */
    uint64_t name_hash; /* fnv1a64(name) (rng.hpp:37-44); see tgb_fnv1a64 */
    uint32_t flags;
    uint32_t reserved;
} tgb_layer_desc;

/* CodecConfig (codec.hpp:78-96) + the sharing mode of this build */
#define TGB_BUCKET_PER_TENSOR 0 /* Bucketing::PerTensor */
#define TGB_BUCKET_GLOBAL 1     /* Bucketing::Global */
#define TGB_BUCKET_FIXED 2      /* Bucketing::FixedSize: buckets of bucket_size elements */
#define TGB_SHARE_REF 0         /* reference semantics: ternarize with the LOCAL scaler,
                                   decode with max over workers (cluster.hpp:195-196) */
#define TGB_SHARE_PRESHARED 1   /* paper Eq.4: max-allreduce BEFORE ternarize */
typedef struct tgb_codec_params {
    float clip_factor;        /* c = 2.5 */
    int32_t clipping_enabled; /* 1 */
    int32_t bucketing;        /* TGB_BUCKET_* */
    int32_t scaler_sharing;   /* 1: shared-max integer-sum decode; 0: fp64 per-worker scalers */
    uint64_t bucket_size;     /* FixedSize only */
    uint64_t seed;            /* Worker sets codec.seed = cluster seed (cluster.hpp:272-273) */
    int32_t share_mode;       /* TGB_SHARE_REF | TGB_SHARE_PRESHARED */
    int32_t reserved;
} tgb_codec_params;

typedef struct tgb_plan_info {
    uint64_t total_elements; /* sum of n over layers */
    uint64_t push_bytes;     /* one rank's push buffer: scaler slots + packed codes (+pad) */
    uint64_t code_bytes;     /* sum of ceil(n/4) over ternary layers (algorithmic) */
    uint64_t scaler_offset;  /* byte offset of the scaler slots in the push buffer (0) */
    uint64_t codes_offset;   /* byte offset of the code region in the push buffer */
    int32_t n_layers;
    int32_t n_slots;      /* scaler slots (one per block) */
    int32_t n_chunks;     /* work items per streaming kernel */
    int32_t n_workers;
    uint32_t chunk_elems; /* elements per chunk */
    uint32_t n_groups;    /* tgb_step schedule: 1 sequential, 2 = dominant layer || rest */
    int32_t n_blocks;     /* blocks: buckets of ternary layers + one per passthrough layer */
    int32_t exchange;     /* TGB_EXCHANGE_*: how tgb_step moves data between ranks */
} tgb_plan_info;

#define TGB_EXCHANGE_AUTO (-1) /* tgb_plan_set_option: sharded from N = 5 for sets of >= 16 Mi
                                  elements, else fused */
#define TGB_EXCHANGE_NONE 0    /* n_workers == 1 */
#define TGB_EXCHANGE_NCCL 1    /* ncclAllGather of push buffers, K3 on every rank */
#define TGB_EXCHANGE_FUSED 2   /* K2 stores scalers + codes into every peer (NVLink) */
#define TGB_EXCHANGE_SHARDED 3 /* codes to the chunk's owner, owner sums N workers and
                                  stores radix-(2N+1) packed sums into every peer, every
                                  rank decodes the sums (parameter server sharded over ranks) */

/* One block of the encoded gradient (EncodedGradient::blocks, codec.hpp:70-76):
 * a bucket of a ternary layer (TernaryBlock, the whole layer unless FixedSize)
 * or a passthrough layer (PassthroughBlock, raw fp32). Blocks follow the
 * canonical layer order; a multi-bucket layer is a contiguous run. */
typedef struct tgb_block_info {
    int32_t layer;          /* owning layer */
    int32_t slot;           /* scaler slot (index into the push scaler array); -1 passthrough */
    uint64_t offset;        /* first element inside the layer (ternarize rng_base, :229) */
    uint64_t n;             /* elements */
    uint64_t region_offset; /* byte offset in a push buffer: ceil(n/4) code bytes, or 4n raw bytes */
    uint32_t flags;         /* TGB_LAYER_PASSTHROUGH */
    uint32_t reserved;
} tgb_block_info;

typedef struct tgb_plan tgb_plan;
typedef struct tgb_comm tgb_comm;

const char* tgb_version(void);
const char* tgb_status_string(tgb_status s);
/* rng.hpp:37-44 (host-side; the device never hashes strings) */
uint64_t tgb_fnv1a64(const char* s, size_t len);
/* number of CUDA devices visible (0 on a CPU-only host) */
int32_t tgb_device_count(void);

/* ---- plan: the per-worker encode_step / sync / decode_pull pipeline ----
 * Replaces: encode_step (codec.hpp:194-239), average (:245-311),
 * ParameterServer::aggregate (cluster.hpp:167-221), decode_pull (wire.hpp:206-228)
 * and the Worker::run sync segment (cluster.hpp:283-297).
 * The plan owns its device workspace (push buffer, gather buffer, partials). */
tgb_status tgb_plan_create(const tgb_layer_desc* layers, int32_t n_layers,
                           const tgb_codec_params* params, uint16_t worker, int32_t n_workers,
                           tgb_plan** out);
void tgb_plan_destroy(tgb_plan* plan);
tgb_status tgb_plan_get_info(const tgb_plan* plan, tgb_plan_info* out);
/* layer l's first block: byte offset of its region inside one push buffer, its
 * scaler slot (-1 for a passthrough layer) */
tgb_status tgb_plan_layer_layout(const tgb_plan* plan, int32_t layer, uint64_t* code_offset,
                                 int32_t* slot);
/* block b's layout (0 <= b < n_blocks) */
tgb_status tgb_plan_block_info(const tgb_plan* plan, int32_t block, tgb_block_info* out);
/* ---- plan options (no environment variables: every schedule choice is explicit) ----
 * TGB_PLAN_OPT_SCHEDULE: TGB_SCHEDULE_AUTO (dominant tensor || the rest on two streams
 *   when one tensor holds 35-95 % of the elements, PerTensor + REF), _SINGLE (one
 *   stream, every kernel covers the whole set), _GROUPS (force the two-group split),
 *   _UNFUSED (= _SINGLE), _FUSED12 (one stream, K1 + K2 as one persistent launch;
 *   measured slower, kept for A/B). Rebuilds the work tables (re-binds the bound
 *   pointers).
 * TGB_PLAN_OPT_EXCHANGE: TGB_EXCHANGE_AUTO / _FUSED / _SHARDED; before attaching peers.
 * TGB_PLAN_OPT_FUSED_OPTIMIZER: 1 (default) the decode kernel applies the optimizer in
 *   tgb_step_apply; 0 the averaged gradient is written and a separate kernel applies it.
 * TGB_PLAN_OPT_PIECES: sharded exchange, pieces of the K2 work list (0 = auto, 1..8): the
 *   owner reduce + decode of piece p run while K2 computes piece p+1; before attaching.
 * TGB_PLAN_OPT_CHUNK: K1/K2 work-item elements (0 = auto: the smallest power of two
 *   >= total / 444 in [4K, 32K]; else a power of two in [1K, 32K]); before attaching. */
#define TGB_PLAN_OPT_SCHEDULE 0
#define TGB_PLAN_OPT_EXCHANGE 1
#define TGB_PLAN_OPT_FUSED_OPTIMIZER 2
#define TGB_PLAN_OPT_PIECES 3
#define TGB_PLAN_OPT_CHUNK 4
/* TGB_PLAN_OPT_OVERLAP: N > 1 peer exchanges, -1 auto / 0 off / 1 on: one K2 launch
 *   whose CTAs publish every finished piece of the work list to the peers, so the
 *   decode of piece p (fused: K3; sharded: owner reduce -> barrier -> decode) overlaps K2
 *   of the later pieces (replaces the two-group schedule); before attaching. */
#define TGB_PLAN_OPT_OVERLAP 5
/* TGB_PLAN_OPT_PULL: fused exchange with shared scalers, 0..8 (default 0): that many
 *   eighths of the code items (32K-element granules) are not stored to the peers by K2;
 *   every rank's decode reads them from their owner's memory over NVLink, moving that
 *   part of the exchange from the K2 stores to the K3 loads; before attaching. */
#define TGB_PLAN_OPT_PULL 6
#define TGB_SCHEDULE_AUTO 0
#define TGB_SCHEDULE_SINGLE 1
#define TGB_SCHEDULE_GROUPS 2
#define TGB_SCHEDULE_UNFUSED 3
#define TGB_SCHEDULE_FUSED12 4
tgb_status tgb_plan_set_option(tgb_plan* plan, int32_t option, int64_t value);

/* host arrays of device pointers, n_layers each: the worker's gradients (read)
 * and the averaged-gradient outputs (written by decode). Pointers must stay
 * valid until the next bind. 16-byte aligned pointers take the vector path. */
tgb_status tgb_plan_bind(tgb_plan* plan, const float* const* d_grads, float* const* d_out);
/* device buffers owned by the plan */
tgb_status tgb_plan_buffers(tgb_plan* plan, uint8_t** d_push, uint8_t** d_gathered,
                            float** d_bounds);

/* K1: per-layer clip bound + per-block local scaler -> push scaler slots, d_bounds (per block).
 * clip (codec.hpp:117-124) + scaler (:128-134) + Global max (:212-216). */
tgb_status tgb_stats(tgb_plan* plan, void* stream);
/* K2: stochastic ternarize + 2-bit pack of every layer into the push code
 * region, using the scalers currently in the push slots (codec.hpp:148-175). */
tgb_status tgb_ternarize_pack(tgb_plan* plan, uint64_t t, void* stream);
/* K1 + K2 (REF mode; PRESHARED needs tgb_step or an explicit
 * tgb_share_scalers between the two) */
tgb_status tgb_encode(tgb_plan* plan, uint64_t t, void* stream);
/* PRESHARED: NCCL max-allreduce of the push scaler slots (share_scalers, codec.hpp:136-141) */
tgb_status tgb_share_scalers(tgb_plan* plan, tgb_comm* comm, void* stream);
/* exchange: NCCL allgather of every rank's push buffer into the gather buffer
 * (replaces push -> ParameterServer::step recv loop, cluster.hpp:137-151) */
tgb_status tgb_sync(tgb_plan* plan, tgb_comm* comm, void* stream);
/* K3: unpack-sum-average of N push buffers laid out back to back at
 * d_src (stride = push_bytes) into the bound outputs. Shared: s = max_w s_w,
 * out = (s*float(sum))*(1.0f/N); unshared: float(sum_w double(s_w)*code / N).
 * average (codec.hpp:281-307) == decode_pull(aggregate) (wire.hpp:206-228). */
tgb_status tgb_decode_average(tgb_plan* plan, const uint8_t* d_src, int32_t n_workers,
                              void* stream);
/* Fused exchange (replaces tgb_sync inside tgb_step): map every rank's gather
 * buffers into this process (CUDA IPC over NVLink/NVSwitch; handles exchanged
 * with one NCCL allgather). Afterwards K1/K2 store this rank's scalers and
 * packed codes directly into every peer's gather buffer, a device flag barrier
 * orders the step, and K3 decodes from local HBM: no allgather launch and the
 * NVLink traffic overlaps K2. Collective: every rank calls it once. */
tgb_status tgb_plan_attach_peers(tgb_plan* plan, tgb_comm* comm);
/* Attaching checks that every rank built the same plan (block table, codec
 * parameters, buffer layout, exchange): a mismatch returns TGB_ERR_PROTOCOL with
 * the reference's text ("server: block structure mismatch from worker <w>",
 * cluster.hpp:169-172) before any peer memory is opened. Per step, every rank
 * publishes its iteration with its barrier flag; a peer at another iteration
 * raises TGB_E_SKEW (cluster.hpp:141-143) and the decode is skipped. */
/* Fused exchange between N plans of ONE process (workers 0..N-1, on one device or
 * on devices with peer access): every plan maps the others' gather buffers
 * directly (no IPC, no NCCL), then tgb_local_step runs the same K2 peer stores,
 * K3 (or the sharded reduce/expand) as the multi-process exchange, ordered by
 * CUDA events between the plans' streams instead of spinning flag barriers (so no
 * hardware-queue or module-loading setting is needed). Single-process
 * counterpart of the reference's run_cluster over InProcessHub
 * (inc/cluster.hpp:378-397, inc/transport.hpp:77-125); used to run N = 8
 * workers' exchanges on fewer GPUs. PRESHARED: after every plan's K1, each plan takes
 * the max over the N workers' local scalers from its gather buffer (the stand-in for
 * the ranks' ncclAllReduce(max)) before its K2. */
tgb_status tgb_plan_attach_local(tgb_plan* const* plans, int32_t n);
/* one step of every plan attached with tgb_plan_attach_local: plan w steps
 * iteration t[w] on streams[w] (cudaStream_t each; a skewed t raises TGB_E_SKEW on
 * the plans that see it). Returns when every launch is queued. */
tgb_status tgb_local_step(tgb_plan* const* plans, int32_t n, const uint64_t* t,
                          void* const* streams);
/* layout self-check (host only, no kernel runs): every region a kernel of this plan
 * reads or writes lies inside its allocation and the work items tile their blocks;
 * TGB_ERR_PROTOCOL with tgb_last_error_message() naming the first violation */
tgb_status tgb_plan_audit(const tgb_plan* plan);
/* device pointers of the push area written by the last step (own scaler slots
 * + codes) and of the gather buffer (n_workers push areas) the last K3 read */
tgb_status tgb_plan_last_buffers(tgb_plan* plan, uint8_t** d_push, uint8_t** d_gathered);
/* the whole worker step: K1 -> [allreduce] -> K2 -> exchange -> K3.
 * comm may be NULL when n_workers == 1. */
tgb_status tgb_step(tgb_plan* plan, tgb_comm* comm, uint64_t t, void* stream);
/* tgb_step with HOST buffers (n_layers pointers each, pinned recommended): H2D of
 * the gradients into the bound device buffers, the step, D2H of the averaged
 * gradients, all stream-ordered after `stream` and completing before it; the
 * next call's H2D overlaps this call's D2H (separate copy streams). */
tgb_status tgb_step_host(tgb_plan* plan, tgb_comm* comm, uint64_t t, const float* const* h_grads,
                         float* const* h_out, void* stream);
/* ---- live kernel timing (measurement, not semantics) ----
 * With capacity > 0, every kernel launch issued by this plan (tgb_step and the
 * stage entry points) is bracketed by two CUDA events recorded on the stream the
 * kernel is launched on, until `capacity` launches are recorded; capacity 0
 * turns it off. Each call resets the record list. tgb_plan_read_timing waits
 * for the recorded events and returns one record per launch: its kernel, layer
 * group, elapsed ms and ALGORITHMIC bytes (local HBM reads + writes the
 * kernel's work requires; NVLink bytes separately). */
#define TGB_KERNEL_K1 0      /* k1_stats: clip bound + scalers */
#define TGB_KERNEL_K2 1      /* k2_ternarize (+ fused N = 1 decode / peer stores) */
#define TGB_KERNEL_BARRIER 2 /* k_peer_barrier */
#define TGB_KERNEL_K3 3      /* k3 decode of the gather buffer */
#define TGB_KERNEL_K3A 4     /* sharded: owner sums N workers' codes */
#define TGB_KERNEL_K3B 5     /* sharded: decode of the packed sums */
#define TGB_KERNEL_K12 6     /* fused K1 + K2 (small sets, one persistent launch) */
#define TGB_KERNEL_NCCL 7    /* ncclAllGather / ncclAllReduce issued by the plan */
typedef struct tgb_kernel_time {
    int32_t kind;          /* TGB_KERNEL_* */
    int32_t group;         /* layer group (two-group schedule) or 0 */
    float ms;              /* event-measured duration on the launching stream */
    float start_ms;        /* launch start relative to the first recorded launch */
    uint64_t elements;     /* gradient elements the launch covers */
    uint64_t hbm_bytes;    /* algorithmic local HBM bytes (read + write) */
    uint64_t nvlink_bytes; /* bytes this rank stores into peers */
} tgb_kernel_time;
tgb_status tgb_plan_enable_timing(tgb_plan* plan, int32_t capacity);
tgb_status tgb_plan_read_timing(tgb_plan* plan, tgb_kernel_time* out, int32_t cap,
                                int32_t* n_records);
/* telemetry: count nonzero codes inside K2 from now on (off by default: it costs one
 * shared-memory pass per chunk) */
tgb_status tgb_plan_enable_code_stats(tgb_plan* plan, int32_t on);
/* telemetry of the last encode: nonzero ternary codes and ternary elements over all
 * blocks; zero fraction = 1 - nonzero/total (Worker::zero_fraction, cluster.hpp:336-346).
 * Requires tgb_plan_enable_code_stats before that step. Synchronises the plan's last stream. */
tgb_status tgb_plan_code_stats(tgb_plan* plan, uint64_t* nonzero, uint64_t* total);
/* synchronises the plan's last stream, reads and clears the error word */
tgb_status tgb_check(tgb_plan* plan, tgb_error* out);

/* ---- optimizer (optimizer.hpp:60-125): applied identically on every worker to the
 * averaged gradient; tgb_step_apply does it inside the step ---- */
#define TGB_OPT_VANILLA 0  /* OptimizerRule::Vanilla */
#define TGB_OPT_MOMENTUM 1 /* OptimizerRule::Momentum (v <- mu*v + g; w <- w - rate*v) */
#define TGB_OPT_ADAM 2     /* OptimizerRule::Adam */
typedef struct tgb_optimizer {
    int32_t rule;
    int32_t reserved;
    double momentum, beta1, beta2, epsilon, weight_decay; /* OptimizerConfig defaults:
                                                             0.9, 0.9, 0.999, 1e-8, 0 */
} tgb_optimizer;
/* OptimizerState::apply for n_layers tensors (device pointers): params -= update(grads);
 * state1 = velocity (Momentum) / first moment (Adam), state2 = second moment (Adam),
 * zero-initialised by the caller, NULL when the rule has none; `step` = the state's step
 * count including this apply (Adam bias corrections 1 - beta^step). */
tgb_status tgb_optimizer_apply(const tgb_optimizer* opt, uint64_t step, double rate,
                               int32_t n_layers, const uint64_t* ns, float* const* d_params,
                               const float* const* d_grads, float* const* d_state1,
                               float* const* d_state2, void* stream);
/* bind parameters + optimizer state (per layer, device) to a plan for tgb_step_apply */
tgb_status tgb_plan_bind_optimizer(tgb_plan* plan, const tgb_optimizer* opt,
                                   float* const* d_params, float* const* d_state1,
                                   float* const* d_state2);
/* tgb_step + OptimizerState::apply(params, averaged gradient, rate) (cluster.hpp:296-299);
 * the plan counts optimizer steps itself */
tgb_status tgb_step_apply(tgb_plan* plan, tgb_comm* comm, uint64_t t, double rate, void* stream);

/* ---- reference wire format (interop with the reference's parameter server) ---- */
/* text of the last TGB_ERR_PROTOCOL on this thread (the reference's ProtocolError what()) */
const char* tgb_last_error_message(void);
/* tensor names (needed by the wire format only; must hash to the plan's name_hash) */
tgb_status tgb_plan_set_names(tgb_plan* plan, const char* const* names);
/* (push frames need <= 65535 blocks and a payload < 4 GB; otherwise the push functions
 * return TGB_ERR_UNSUPPORTED) */
/* bytes of one push frame: kHeaderSize + wire_size(encoded) (wire.hpp:28-36, codec.hpp:442-454) */
tgb_status tgb_plan_push_frame_size(const tgb_plan* plan, uint64_t* bytes);
/* frame(Message{Push, t, worker, serialize_encoded(last encode)}) into h_frame
 * (codec.hpp:395-438, wire.hpp:41-53): packed on the device from the push area. Synchronous. */
tgb_status tgb_plan_serialize_push(tgb_plan* plan, uint64_t t, uint8_t* h_frame, void* stream);
/* decode_pull(deserialize_pull(unframe(h_frame).payload)) (wire.hpp:57-75, 147-228) into the
 * bound outputs; radix-packed sums unpacked on the device. Returns the frame's iteration.
 * Synchronous. */
tgb_status tgb_plan_decode_pull(tgb_plan* plan, const uint8_t* h_frame, uint64_t len,
                                uint64_t* iteration, void* stream);

/* ---- traffic accounting (TrafficStats, cluster.hpp:62-74, 145-160) ----
 * Per worker and step, for the reference's wire format: the framed push
 * (kHeaderSize + wire_size, codec.hpp:455-467) and the same tensors at raw fp32
 * (kHeaderSize + float_wire_size, :469-481); the framed pull the server sends
 * back (radix-(2N+1) SharedSumBlocks or FloatAvgBlocks, wire.hpp:103-145) and its
 * fp32 size (float_pull_size, wire.hpp:231-243). up/down reduction = float/framed.
 * device_bytes_out / _in: what this build's exchange actually moves per rank and
 * step over NVLink (fused: codes + scalers to N-1 peers; sharded: codes to owners
 * + packed sums to every rank); 0 at N == 1. */
typedef struct tgb_traffic {
    uint64_t bytes_up, bytes_down;             /* framed, per worker */
    uint64_t float_bytes_up, float_bytes_down; /* same tensors at raw fp32 */
    uint64_t device_bytes_out, device_bytes_in;
} tgb_traffic;
/* from a layer table alone (no device needed); names[l] are the tensor names */
tgb_status tgb_traffic_for_layers(const tgb_layer_desc* layers, const char* const* names,
                                  int32_t n_layers, const tgb_codec_params* params,
                                  int32_t n_workers, tgb_traffic* out);
/* for a plan (after tgb_plan_set_names; device bytes for its current exchange) */
tgb_status tgb_plan_traffic(const tgb_plan* plan, tgb_traffic* out);

/* ---- communicator (NCCL over NVLink/NVSwitch) ---- */
#define TGB_UNIQUE_ID_BYTES 128
tgb_status tgb_comm_unique_id(uint8_t out[TGB_UNIQUE_ID_BYTES]);
tgb_status tgb_comm_init(const uint8_t id[TGB_UNIQUE_ID_BYTES], int32_t nranks, int32_t rank,
                         tgb_comm** out);
void tgb_comm_destroy(tgb_comm* comm);

/* ---- per-layer entry points (the reference's per-layer functions) ---- */
/* scaler (codec.hpp:128-134): *d_s = max |g| */
tgb_status tgb_layer_scaler(const float* d_g, uint64_t n, float* d_s, void* stream);
/* clip (codec.hpp:117-124): d_out = clipped copy; *d_bound = float(c*sigma) (inf if n<2) */
tgb_status tgb_layer_clip(const float* d_g, uint64_t n, float c, float* d_out, float* d_bound,
                          void* stream);
/* ternarize (codec.hpp:148-175) with RngStream(seed, t, name, worker) (rng.hpp:50-57);
 * d_codes receives ceil(n/4) bytes */
tgb_status tgb_layer_ternarize(const float* d_g, uint64_t n, float s, uint64_t seed, uint64_t t,
                               uint64_t name_hash, uint64_t worker, uint64_t rng_base,
                               uint8_t* d_codes, void* stream);
/* decode (codec.hpp:177-182) */
tgb_status tgb_layer_decode(const uint8_t* d_codes, uint64_t n, float s, float* d_out,
                            void* stream);
/* one block of average (codec.hpp:281-307); d_codes is a HOST array of N device
 * pointers, d_s a device array of N scalers */
tgb_status tgb_layer_average(int32_t n_workers, const uint8_t* const* d_codes, const float* d_s,
                             uint64_t n, int32_t sharing, float* d_out, void* stream);
/* one PassthroughBlock position of average (codec.hpp:269-279): d_vals is a HOST
 * array of N device pointers; out = float(sum_w double(v_w) / N), worker order */
tgb_status tgb_layer_average_raw(int32_t n_workers, const float* const* d_vals, uint64_t n,
                                 float* d_out, void* stream);
/* histogram (codec.hpp:491-517): equal-width bins over [min, max]; d_counts and
 * d_edges (left edges, double) are device arrays of `bins` entries. Synchronises. */
tgb_status tgb_layer_histogram(const float* d_v, uint64_t n, uint32_t bins, uint64_t* d_counts,
                               double* d_edges, void* stream);
/* RngStream::bits (rng.hpp:59-66) for indices k0..k0+n-1 (KAT helper) */
tgb_status tgb_rng_bits(uint64_t seed, uint64_t t, uint64_t name_hash, uint64_t worker,
                        uint64_t k0, uint64_t n, uint32_t* d_out, void* stream);
/* synchronises `stream`, reads and clears the per-layer error word of the current device */
tgb_status tgb_layer_check(void* stream, tgb_error* out);

#ifdef __cplusplus
}
#endif
#endif /* TGB_TERNGRAD_B200_H */
