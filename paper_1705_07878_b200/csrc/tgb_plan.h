// tgb_plan: one worker's block table, work schedule, push / gather / sums
// buffers and exchange state (host side; shared by plan.cu and capi.cu).
#pragma once

#include <string>
#include <vector>

#include <nccl.h>

#include "tgb_internal.h"

using namespace tgb;

struct tgb_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
};

constexpr int kFlagSlots = 2 * kMaxPieces;  // barrier slots per step: two layer groups (fused),
                                            // or two barriers per piece (sharded)
constexpr uint64_t kAlignCodes = 16;  // per-block region alignment (bytes)
constexpr uint64_t kAlignPush = 256;  // push buffer / region base alignment

inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Everything two ranks must agree on before they write into each other's
// buffers (exchanged at attach, compared field by field).
struct PlanDesc {
    uint64_t magic;
    int32_t abi, n_workers;
    uint64_t push_bytes, sums_bytes, ipc_bytes;
    uint32_t n_blocks, n_tensors, chunk12, chunk3;
    int32_t shard, grouped, radix_m, reserved;
    uint64_t layout_hash;  // blocks: n, tensor, flags, slot, region offsets, bucket offsets
    uint64_t codec_hash;   // tgb_codec_params
};

struct tgb_plan {
    int device = 0;
    tgb_codec_params p{};
    uint16_t worker = 0;
    int32_t n_workers = 1;
    std::vector<tgb_layer_desc> desc;  // tensors (layers) in canonical order
    std::vector<TensorDev> h_tensors;
    std::vector<LayerDev> h_layers;  // BLOCKS (buckets / passthrough tensors)
    std::vector<uint64_t> block_off;  // block's first element inside its tensor
    std::vector<ChunkDev> h_chunks;   // K1/K2 (and sharded K3a/K3b) work items
    std::vector<ChunkDev> h_chunks3;  // K3 work items (kChunk3 elements)
    LayerDev* d_layers = nullptr;
    TensorDev* d_tensors = nullptr;
    Partial* d_gpart = nullptr;  // K1 two-level finalize (TensorDev::group_base)
    uint32_t* d_gdone = nullptr;
    size_t gpart_cap = 0;
    ChunkFat* d_fat = nullptr;   // K1/K2: chunk + block copy (rebuilt on bind)
    ChunkFat* d_fat3 = nullptr;  // K3
    size_t fat_cap = 0, fat3_cap = 0;
    Partial* d_partials = nullptr;
    uint32_t* d_counters = nullptr;  // n_layers layer_done + 1 global_done
    float* d_bounds = nullptr;       // per block
    uint8_t* d_push = nullptr;
    ErrWord* d_err = nullptr;
    unsigned long long* d_nnz = nullptr;  // telemetry: nonzero codes per group (last step)
    bool code_stats = false;
    uint64_t push_bytes = 0, codes_offset = 0, code_bytes = 0, total = 0;
    int32_t n_slots = 0, n_active = 0;

    // ---- options (tgb_plan_set_option)
    int32_t schedule_opt = TGB_SCHEDULE_AUTO;
    int32_t exchange_opt = TGB_EXCHANGE_AUTO;
    bool opt_fused = true;

    // ---- schedule (build_schedule). Chunk tables are ordered by group, and
    // inside a group ternary chunks come before passthrough chunks (K1 launches
    // only the ternary prefix). An ungrouped plan is the single group 0. Two-group
    // schedule: group 1 = the dominant tensor, group 0 = the rest; each group runs
    // K1 -> K2 -> [barrier] -> K3 on its own stream, so a memory-bound kernel of one
    // group overlaps a compute-bound kernel of the other.
    bool grouped = false;
    int32_t big = -1;  // the dominant tensor (group 1 of the two-group schedule)
    uint32_t cb[2] = {0, 0}, cc[2] = {0, 0}, ck1[2] = {0, 0}, cb3[2] = {0, 0}, cc3[2] = {0, 0};
    uint32_t chunk12 = kChunk12, chunk3 = kChunk3;
    int32_t pdl = 0;           // K2 as K1's programmatic dependent (single-stream N = 1 plans)
    uint32_t k1_keep = 0;      // K1 units per launch loaded L2 evict_last (N = 1)
    // small sets: K1 + K2 as one persistent launch (k12_fused), per-tensor epoch flags
    bool k12 = false;
    uint32_t* d_ready = nullptr;  // n_layers + 1 flags (the last: Global) + exit counter
    uint32_t k12_epoch = 0;
    // FixedSize: per-block max |x| (K1 -> k1_bucket_slots), block meta {tensor, slot};
    // mb_log2 > 0: buckets of 2^mb_log2 elements grouped into multi-bucket work items
    uint32_t* d_bmax = nullptr;
    uint2* d_bmeta = nullptr;
    uint32_t mb_log2 = 0;
    cudaStream_t gs[2] = {nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};

    // ---- exchange. Unattached N > 1 plans allgather push areas with NCCL into
    // d_gathered. Attached plans own one IPC-shareable allocation
    //   [gather parity 0][gather parity 1][sums parity 0][sums parity 1][flags]
    // mapped by every peer; gather buffers alternate by step parity.
    bool shard = false;       // sharded exchange (decided by the schedule)
    int32_t radix_m = 0;      // sharded: base-(2N+1) digits per u32 sums word
    uint32_t sum_region = 0;  // sharded: bytes of a full chunk's sums region
    uint64_t sums_bytes = 0, sums_off = 0, flags_off = 0, ipc_bytes = 0;
    // sharded: the K2 chunk list in n_pieces contiguous pieces [pb[p], pb[p+1]); rank r
    // owns chunks [pcs[p][r], pcs[p][r+1]) of piece p. Piece p's barrier -> K3a ->
    // barrier -> K3b run on a second stream while K2 computes piece p+1.
    // overlapped exchange (TGB_PLAN_OPT_OVERLAP): one K2 launch whose CTAs publish each
    // finished piece's barrier record; the decode of piece q (fused: K3 over the K3 items
    // [p3[q], p3[q+1]), listed in K2 order; sharded: K3a -> barrier -> K3b) runs on gs3
    // while K2 computes the later pieces
    int32_t overlap_opt = -1;  // -1 auto, 0 off, 1 on
    bool overlap = false;
    uint32_t p3[kMaxPieces + 1] = {};
    uint32_t* d_piece_cnt = nullptr;
    int32_t pieces_opt = 0;  // TGB_PLAN_OPT_PIECES (0: auto)
    int32_t pull_opt = 0;    // TGB_PLAN_OPT_PULL (eighths of the code items pulled by K3)
    uint32_t pull8 = 0;      // effective split (0: every item pushed by K2)
    int32_t chunk_opt = 0;   // TGB_PLAN_OPT_CHUNK (0: auto)
    int32_t n_pieces = 1;
    uint32_t pb[kMaxPieces + 1] = {};
    uint32_t pcs[kMaxPieces][kMaxPeers + 1] = {};
    cudaStream_t gs3 = nullptr;
    cudaEvent_t ev_piece[kMaxPieces] = {}, ev_done = nullptr;
    uint8_t* d_gathered = nullptr;    // NCCL gather buffer, or parity-0 gather inside d_ipc
    uint8_t* d_nccl_gather = nullptr;
    uint8_t* d_ipc = nullptr;
    uint8_t* peer_ipc[kMaxPeers] = {};  // every rank's d_ipc mapped here (self = d_ipc)
    bool attached = false;
    bool local_peers = false;  // tgb_plan_attach_local: peers are plans of this process
    int32_t rank = 0;
    uint64_t epoch = 0;  // attached: steps begun (barrier value); parity = epoch & 1
    uint64_t last_t = 0;  // iteration of the step in flight (published with the barrier)
    cudaEvent_t ev_local[3] = {nullptr, nullptr, nullptr};  // tgb_local_step phases

    cudaStream_t last = nullptr;
    bool bound = false;
    // host-buffer steps (tgb_step_host): per-tensor bound pointers, copy streams
    std::vector<const float*> bound_g;
    std::vector<float*> bound_out;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d = nullptr, ev_comp = nullptr, ev_d2h = nullptr;
    bool host_io = false;
    cudaEvent_t ev_hg[2] = {}, ev_cg[2] = {}, ev_dg[2] = {};  // grouped N = 1: per layer group
    // optimizer bound for tgb_step_apply
    bool opt_bound = false;
    tgb_optimizer opt{};
    uint64_t opt_steps = 0;
    std::vector<float*> opt_w, opt_s1, opt_s2;
    OptDev* d_optd = nullptr;             // per-block optimizer table (fused decode -> optimizer)
    const OptArgs* opt_active = nullptr;  // set during tgb_step_apply when fused
    // reference wire format (tgb_plan_set_names / serialize_push / decode_pull)
    std::vector<std::string> names;
    uint64_t push_frame_bytes = 0;
    uint8_t* d_frame = nullptr;  // push frame image (static headers written once)
    WireSeg* d_wsegs = nullptr;  // dynamic parts: scalers, codes, raw values
    uint32_t n_wsegs = 0;
    uint8_t* d_pull = nullptr;  // pull payload staging
    uint64_t pull_cap = 0;
    // live kernel timing (tgb_plan_enable_timing): two events per launch
    int32_t t_cap = 0, t_used = 0;
    std::vector<cudaEvent_t> t_ev;
    std::vector<tgb_kernel_time> t_rec;
};

namespace tgb {
// shared by capi.cu (wire, optimizer) and plan.cu
uint8_t* own_push(const tgb_plan* P);
uint8_t* cur_gathered(const tgb_plan* P);
tgb_status set_protocol_error(const std::string& msg);
}  // namespace tgb
