// ts_hydro.cpp — host side of libts_hydro.so: the C ABI of include/ts_hydro.h.
//
// One context = one GPU = one locality of the reference's World
// (distrib.hpp:112-203).  The context owns:
//   - three state buffers A (U^n), B (U^(1)), C (U^(2)) laid out
//     [local sub-grid][field][512]; SSP-RK3 runs A->B, (B,A)->C, (C,A)->A so
//     U^n never moves;
//   - the local mesh: owned sub-grids (ascending global id) then halo proxies
//     of foreign face neighbours; an interior list (no foreign neighbour) and
//     a boundary list;
//   - per-peer packed-halo plans and an NCCL communicator (dlopen'ed);
//   - a ring of per-launch [start,end] globaltimer stamps written by the
//     kernels themselves — the per-kernel timing hook that stands in for the
//     reference's ActivityRecord feed (device.cpp:75-103, profiler.cpp:298-318).
#include "../../include/ts_hydro.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "fmm.h"
#include "hydro_kernels.h"

namespace {

constexpr int kN = 8;
constexpr int kNC = 512;
constexpr int kSlab = 3 * kN * kN;

// Static taxonomy strings (record names outlive every context).
constexpr const char* kNameStage[4] = {"", "hydro_stage1_kernel", "hydro_stage2_kernel",
                                       "hydro_stage3_kernel"};
constexpr const char* kNameSignal = "signal_speed_kernel";
constexpr const char* kNameP2P = "p2p_kernel";  // the reference's kKernelP2P (workload.hpp:46)
constexpr const char* kNameP2M = "p2m_kernel";  // kKernelP2M (workload.hpp:47)
constexpr const char* kNameMultipole = "multipole_kernel";           // kKernelMultipole (workload.hpp:45)
constexpr const char* kNameMultipoleRoot = "multipole_root_kernel";  // kKernelMultipoleRoot (workload.hpp:48)
constexpr const char* kNameFmmMoments = "fmm_moments_kernel";        // the FMM's upward P2M pass
constexpr const char* kNameGravityKick = "gravity_kick_kernel";      // the gravity source term
constexpr const char* kNamePack = "halo_pack_kernel";
constexpr const char* kNameUnpack = "halo_unpack_kernel";
constexpr const char* kNameAmrFill = "amr_ghost_fill_kernel";
constexpr const char* kNameAmrReflux = "amr_reflux_kernel";
constexpr const char* kNameH2D = "copy_host_to_device";
constexpr const char* kNameD2H = "copy_device_to_host";
constexpr const char* kNameD2D = "copy_device_to_device";
constexpr const char* kNameAlloc = "device_alloc";
constexpr const char* kNameFree = "device_free";

uint64_t steady_ns() {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// ---- NCCL, resolved at run time so single-GPU users need no NCCL ----------
struct Nccl {
    bool loaded = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) {
            n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
#define TS_SYM(field, name)                                              \
    n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));       \
    if (n.field == nullptr) {                                            \
        n.why = std::string("libnccl lacks ") + name;                    \
        return;                                                          \
    }
        TS_SYM(GetUniqueId, "ncclGetUniqueId");
        TS_SYM(CommInitRank, "ncclCommInitRank");
        TS_SYM(CommDestroy, "ncclCommDestroy");
        TS_SYM(CommAbort, "ncclCommAbort");
        TS_SYM(Send, "ncclSend");
        TS_SYM(Recv, "ncclRecv");
        TS_SYM(AllReduce, "ncclAllReduce");
        TS_SYM(AllGather, "ncclAllGather");
        TS_SYM(GroupStart, "ncclGroupStart");
        TS_SYM(GroupEnd, "ncclGroupEnd");
        TS_SYM(GetErrorString, "ncclGetErrorString");
#undef TS_SYM
        n.loaded = true;
    });
    return n;
}

struct DoneThunk {
    ts_done_fn fn;
    void* user;
    int32_t* list;
};
void CUDART_CB done_host(void* p) {
    auto* t = static_cast<DoneThunk*>(p);
    if (t->fn) t->fn(t->user);
    delete t;
}

struct PendingLaunch {
    uint8_t kind;
    const char* name;
    int32_t stream_id;
    uint64_t guid;
    uint32_t slot;  // stamp slot
    bool overlap;   // PDL launch: may start before the previous kernel on its stream ended
    uint64_t bytes = 0;  // copies (ts_hydro_enqueue_copy)
    // Copies of the pipelined host path are timed by CUDA events, not stamp
    // kernels: a copy stream must never need an SM (stage-1 CTAs waiting for
    // the H2D chunks may hold every SM slot until the copies land).
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};

// Stream memory operation (driver API, resolved through the runtime so the
// library needs no link-time libcuda): the P2P copy-engine exchange raises a
// peer's flag behind its transfer without an SM.  Waits are a one-thread
// kernel with a deadline (tsh::launch_wait_flags), not cuStreamWaitValue32,
// so a missing peer is reported instead of hanging the stream.
struct StreamMemOps {
    bool ok = false;
    CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
};

StreamMemOps& memops() {
    static StreamMemOps m;
    static std::once_flag once;
    std::call_once(once, [] {
        void* w = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q) == cudaSuccess && w) {
            m.write32 = reinterpret_cast<decltype(m.write32)>(w);
            m.ok = true;
        }
        void* v = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q) == cudaSuccess && v)
            m.wait32 = reinterpret_cast<decltype(m.wait32)>(v);
    });
    return m;
}

constexpr int kMaxRanks = 64;
constexpr uint32_t kBlobMagic = 0x54535032;  // "TSP2"

// What one rank publishes so its peers can write straight into its memory.
struct P2PBlob {
    uint32_t magic;
    int32_t rank, world, device;
    cudaIpcMemHandle_t recv, flags, gather;
    cudaIpcMemHandle_t U[3];      // state buffers (proxy slots written by the fused halo push)
    int64_t n_recv_total;
    int64_t recv_off[kMaxRanks];  // slab offset of the data from source rank q in my receive buffer
};

struct PeerMap {
    double* recv = nullptr;    // peer's receive buffer (2 halves)
    int32_t* flags = nullptr;  // peer's flags: [0, world) halo by source, [world, 2 world) dt gather
    double* gather = nullptr;  // peer's dt gather: [2][world]
    double* U[3] = {nullptr, nullptr, nullptr};  // peer's state buffers
    int64_t n_recv_total = 0;
    int64_t recv_off_for_me = 0;
};

struct Peer {
    int rank = -1;
    std::vector<int64_t> send_pairs;  // (global id, face) flattened
    std::vector<int32_t> send_dst;    // per send entry: the sub-grid's local index on the peer (a proxy)
    std::vector<int64_t> recv_pairs;
    int64_t send_off = 0, recv_off = 0;  // entry offsets into the concatenated tables
    int64_t n_send = 0, n_recv = 0;
};

}  // namespace

struct ts_hydro_ctx {
    ts_hydro_config cfg{};
    int nf = 6;
    int dev = 0;
    int sms = 148;
    std::string err;
    std::recursive_mutex mu;
    bool shut = false;
    bool host_only = false;  // device_id = -1: mesh / halo planning only, no compute

    std::vector<cudaStream_t> streams;  // lazily created; [0] compute, [1] comm, [2] boundary
    cudaEvent_t ev_in = nullptr, ev_halo = nullptr, ev_red = nullptr, ev_bnd = nullptr;
    // ts_hydro_step_host_async: chunked copies on their own streams; the
    // previous call's host_out and its per-chunk D2H completion events
    static constexpr int kXferChunksMax = 64;
    int xfer_chunks = 24;  // TS_HYDRO_XFER_CHUNKS (wavefront e2e, same box: 8 -> 0.82-0.83, 24 -> 0.84-0.87 G)
    bool chunk_overlap = true;  // TS_HYDRO_CHUNK_OVERLAP=0: D2H waits for the whole last stage
    bool amr_fused = true;      // TS_HYDRO_AMR_SPLIT=1: one stage launch per AMR level
    cudaEvent_t ev_d2h[kXferChunksMax] = {};
    cudaEvent_t ev_h2d = nullptr, ev_comp = nullptr;
    const void* prev_out = nullptr;
    size_t prev_out_bytes = 0;
    uint32_t* d_chunk_ctr = nullptr;          // [kXferChunksMax] stage-3 completions per D2H chunk
    uint32_t chunk_expect[kXferChunksMax] = {};  // running totals (wrapping)
    bool chunk_arm = false;                   // next stage-3 launch counts into d_chunk_ctr
    // chained pipelined host steps: stage 1 starts under the H2D (StageArgs::h2d_flag)
    bool h2d_gate = true;                     // TS_HYDRO_H2D_GATE=0: stage 1 waits for the whole H2D
    uint32_t* d_h2d_flag = nullptr;           // [kXferChunksMax] landed-chunk flags
    uint32_t h2d_seq = 0;
    bool h2d_arm = false;                     // the next stage 1 acquires the chunk flags of h2d_seq
    // chained pipelined host steps, wavefront form (TS_HYDRO_E2E_WAVE=0: off):
    // per chunk H2D -> stage 1 -> 2 -> 3 -> D2H launches on the chunk's own
    // stream, each waiting (events) only for the chunks its halo reaches
    bool e2e_wave = true;
    bool wave_ready = false;                  // events + dependency lists built for the bound mesh
    cudaEvent_t ev_wave[4][kXferChunksMax] = {};  // [h2d, s1, s2, s3][chunk]
    std::vector<std::vector<int>> wave_dep;   // chunk -> chunks its sub-grids' face neighbours live in

    // mesh
    bool have_mesh = false;
    int world = 1, rank = 0;
    int64_t n_global = 0, n_owned = 0, n_proxy = 0;
    std::vector<int64_t> owned_gid, proxy_gid;
    std::vector<int32_t> nbr_local;  // [n_local][6]
    std::vector<int32_t> interior, boundary;
    std::vector<Peer> peers;

    // device memory
    double* U[3] = {nullptr, nullptr, nullptr};
    unsigned long long* d_check = nullptr;  // [5] self-check failures (TS_CHECK builds write it)
    double* d_grav = nullptr;               // [n_owned][4][512] gravity P2P output (phi, gx, gy, gz)
    std::vector<uint8_t> grav_streams;      // streams with gravity work not yet joined into the compute stream
    // gravity FMM (fmm.h): the octree of the owned sub-grids and its device copy
    bool have_fmm = false;
    tsh::FmmTree fmm;
    int* d_fmm_int = nullptr;     // depth, q[3], leaf, parent, child[8], nb27[27] per node (SoA, see fmm_upload)
    double* d_fmm_M = nullptr;    // [n][4][512]
    double* d_fmm_L = nullptr;    // [n_internal][10][512]
    double* d_fmm_part = nullptr;  // the root's chunk sums
    int* d_fmm_lists = nullptr;   // leaves to evaluate (p2p, p2p with refined edge / corner slots, p2m), then
                                  // the refined nodes whose expansions they need, by depth
    std::vector<int> fmm_m2l_first, fmm_m2l_count;  // per depth: the M2L nodes' range in the list buffer
    int fmm_leaf_lists[3] = {0, 0, 0};               // counts of the three leaf lists
    // N ranks: every rank gathers every leaf's density (NCCL all-gather) and
    // evaluates its own leaves; leaf rows = owner * fmm_max_owned + owned index
    int64_t fmm_max_owned = 0;
    double* d_fmm_send = nullptr;  // [max_owned][512] own densities, packed
    double* d_fmm_rho = nullptr;   // [world * max_owned][512] every rank's
    tsh::FmmEntry* d_fmm_tab[tsh::kFmmRMax + 1][2][2] = {};  // [R][root][far_only]
    int n_fmm_tab[tsh::kFmmRMax + 1][2][2] = {};
    double* d_scr_ring = nullptr;   // nf > 6: species accumulators, kScrK slots per SM id (StageArgs::scr_ring)
    unsigned int* d_scr_mask = nullptr;
    static constexpr int kScrK = 8;
    bool scr_ring = true;           // TS_HYDRO_SCR_RING=0: accumulate in the free state buffer
    CUtensorMap tmap[3];           // TMA view of each state buffer: rows of 16 doubles, {16, 32} boxes
    bool tmap_ok = false;
    int32_t* d_nbr = nullptr;
    std::vector<int64_t> mesh_nbr;    // the bound global mesh (checkpoints)
    std::vector<int32_t> mesh_owner;
    int32_t* d_interior = nullptr;
    int32_t* d_boundary = nullptr;
    int32_t* d_order = nullptr;       // launch order of the fused P2P stage: boundary spread through the front
    uint32_t* d_flow = nullptr;       // [3][n_owned] dataflow: last step seq that finished stage 1 / 2 / 3
    unsigned long long* d_cta_log = nullptr;  // [3][n_owned][4] diagnostic per-CTA timeline of the last step
    int32_t* d_bnd_of = nullptr;      // [n_owned] sub-grid -> boundary slot (-1: interior)
    int2* d_push_tbl = nullptr;       // [n_boundary][6] fused halo push targets
    long long* d_gid = nullptr;
    int2* d_send_entries = nullptr;
    int2* d_recv_entries = nullptr;
    double* d_send = nullptr;
    double* d_recv = nullptr;
    int64_t n_send_total = 0, n_recv_total = 0;
    double* d_scal = nullptr;     // [0..1] amax ping-pong, [2] scratch amax, [3] dummy, [4] P2P global amax
    double* d_dt_hist = nullptr;  // [kDtHist]
    static constexpr uint64_t kDtHist = 4096;
    unsigned long long* d_stamps = nullptr;  // [cap][2]
    unsigned long long* h_clock = nullptr;   // mapped pinned: [0] clock calibration, [1] cross-GPU wait timeout,
                                             //   [2] globaltimer at ev_cal (event-timed copies)
    cudaEvent_t ev_cal = nullptr;            // reference event of the event-timed records
    bool cal_armed = false;                  // ev_cal / h_clock[2] recorded since the last harvest
    std::vector<cudaEvent_t> ev_pool;        // timing events for copy records
    unsigned long long wait_ns = 30ull * 1000000000ull;
    std::map<void*, uint64_t> dev_allocs;
    std::map<void*, uint64_t> host_allocs;
    ts_memory_state mem{};
    // SimDevice-contract entry points (ts_hydro_launch_kernel / _enqueue_copy / _device_alloc)
    std::set<std::string> names;                          // interned launch names (stable c_str)
    std::map<uint64_t, std::pair<void*, uint64_t>> handles;  // device_alloc handle -> (ptr, bytes)
    uint64_t next_handle = 1;
    void* stage_dev = nullptr;   // copy staging (context-internal, not counted)
    uint64_t stage_dev_bytes = 0;
    void* stage_host = nullptr;
    uint64_t stage_host_bytes = 0;

    // comm
    ncclComm_t comm = nullptr;
    int comm_size = 1;
    bool p2p = false;                 // copy-engine halos + stream memory ops (single node)
    int32_t* d_flags = nullptr;       // [2 world]
    double* d_gather = nullptr;       // [2][world]
    std::vector<PeerMap> pm;          // by rank
    unsigned int* d_ctr = nullptr;    // [0] stage-3 CTA count of the tail dt push, [1..3] halo-push counts by stage slot
    uint32_t done_cnt = 0;            // expected d_ctr[0] (monotonic, wrapping)
    uint32_t halo_cnt[3] = {0, 0, 0}; // expected d_ctr[1 + slot]
    double** d_push_gather = nullptr; // [2][world] gather arrays (parity halves) of every rank
    unsigned int** d_push_flag = nullptr;  // [world] dt flag word of every peer (nullptr for self)
    uint32_t xseq = 0, aseq = 0;      // exchange / dt-gather sequence numbers (same on every rank)
    bool halo_fused = true;           // P2P: halo slabs pushed by the stage kernel (else copy engines)
    bool flow = true;                 // single rank: stages 2, 3 as PDL dependents gated by per-sub-grid flags
    bool flow_chain = false;          // the last stream op was this call's stage 3: the next stage 1 may be a PDL dependent
    bool flow_steps = true;           // TS_HYDRO_FLOW_STEPS=0: stage 1 stays stream-ordered
    bool mchain = true;               // TS_HYDRO_MCHAIN=0: N ranks keep stage 1 stream-ordered
    bool fmm_merge = true;            // TS_HYDRO_FMM_MERGE=0: one M2L part launch per depth
    uint32_t* d_cnt3 = nullptr;       // finished stage-3 CTAs (monotonic)
    uint32_t cnt3_expect = 0;
    // P2P dt all-reduce: in the stage-3 tail (default: every CTA counts out
    // after a fence, the last one pushes and gathers, and the next step's
    // stage 1 is chained behind it as a PDL dependent — StageArgs::cnt_gather)
    // or a one-thread kernel between stage 3 and the next stage 1
    // (TS_HYDRO_DT=kernel).  Same-box A/B, Sedov 4096/GPU at 2 B200s: tail +
    // chain 7.51-7.52 G, kernel 7.38-7.39, tail without the chain 7.34-7.37.
    bool dt_kernel = false;
    uint32_t flow_seq = 0;
    bool halo_pushed = false;         // proxies of U^n were pushed by the last stage 3 (flags of xseq)
    uint64_t halo_recv_mask = 0;      // ranks that push slabs to this one
    double** d_push_out = nullptr;    // [3][world] every peer's state buffers (nullptr for self)
    unsigned int** d_halo_flag = nullptr;  // [world] this rank's halo flag word on each receiving peer
    const double* amax_src = nullptr; // where this step's dt comes from
    int amax_n = 1;

    // coarse-fine AMR mesh (ts_hydro_set_amr_mesh): leaves level-major, proxies after them
    bool amr = false;
    // multi-rank AMR (ts_hydro_set_amr_mesh_partitioned): owned leaves, then
    // ghost leaves (whole-sub-grid copies of remote leaves the rank reads),
    // then the proxies it fills; halo entries move whole sub-grids
    bool amr_mr = false;
    int xfer_cells = kSlab;  // cells per halo entry: a 3-deep slab, or a whole sub-grid (multi-rank AMR)
    int amr_max_level = 0;
    std::vector<int64_t> amr_level_first;  // [max_level + 2]
    int64_t amr_n_proxy = 0, amr_n_rec = 0;
    int64_t amr_proxy_first = 0;            // local index of the first proxy (n_owned; + ghosts on several ranks)
    tsh::AmrProxy* d_amr_proxy = nullptr;
    unsigned char* d_amr_pmask = nullptr;  // per proxy: faces read (launch_amr_fill)
    bool amr_slab_fill = true;             // TS_HYDRO_AMR_FULLFILL=1: fill whole proxies
    tsh::AmrReflux* d_amr_rec = nullptr;
    int32_t* d_amr_level = nullptr;
    int32_t* d_amr_rf_slot = nullptr;       // [n_leaves][6] flux register slot of a coarse-fine face, -1 = none
    double* d_amr_rf_flux = nullptr;        // [slots][nf][64] doubled face fluxes stored by the stage kernel
    bool amr_reflux_reg = true;             // TS_HYDRO_AMR_REFLUX=recompute: reflux reconstructs the fluxes again

    // Per-sub-grid drop-in steps (ts_hydro_launch_stage ... ts_hydro_finish_step).
    // Launches are ISSUED in dependency order — a stage-k launch is parked on
    // the host until its sub-grids and their face neighbours have issued stage
    // k-1 of the step — and ORDERED on the device by the dataflow flags
    // (d_flow) and the stage-3 count (d_cnt3), so no host barrier separates
    // the stages and no stream ever waits behind a kernel spinning on work
    // queued after it.
    struct DropinLaunch {
        int stage;
        std::vector<int32_t> list;
        uint32_t stream_id;
        uint64_t guid;
        ts_done_fn done;
        void* user;
    };
    bool din_open = false;       // a drop-in step is in progress
    bool din_chained = false;    // the previous step was a drop-in step: its flags / count are on the device
    uint32_t din_seq = 0;        // flow seq of the open step
    std::vector<uint8_t> din_req;     // [n_owned] last stage requested in the open step (0..3)
    std::vector<uint8_t> din_issued;  // [n_owned] last stage issued
    int64_t din_done3 = 0;            // sub-grids whose stage 3 was issued
    std::vector<DropinLaunch> din_parked;
    std::vector<uint8_t> din_streams; // streams used by the open step
    cudaEvent_t ev_din = nullptr;     // stream-0 work before the step (upload, compute_dt, batched steps)
    // N ranks (fused P2P halos): the step's halo seqs are din_xbase + stage;
    // a boundary sub-grid's stage k is issued only after every boundary
    // sub-grid's stage k-1 (its peers' stage k-1 waits for all of those)
    uint32_t din_xbase = 0;
    bool din_wait1 = false;           // stage 1 acquires the peers' pushes of U^n (else a copy-engine refresh ran)
    uint32_t din_halo_target[4] = {0, 0, 0, 0};
    int64_t din_bnd_issued[4] = {0, 0, 0, 0};
    std::vector<int32_t> bnd_host;    // [n_owned] boundary slot (-1: interior)
    // AMR mesh: a stage's proxy fill needs every leaf's previous stage and the
    // reflux every leaf's stage, so stage k of any leaf waits (event) for the
    // reflux of k-1 and the fill of k, enqueued once every leaf issued k-1
    int64_t din_count[4] = {0, 0, 0, 0};
    cudaEvent_t ev_amr[4] = {nullptr, nullptr, nullptr, nullptr};
    bool din_amr_barrier[4] = {false, false, false, false};

    // stepping
    uint64_t steps_done = 0;
    uint64_t launches = 0;
    bool dt_valid = false;
    bool profiling = true;  // ts_hydro_set_profiling: activity stamps and records on every launch

    // activity
    std::vector<PendingLaunch> pending;  // launches holding a stamp slot
    std::vector<ts_activity_record> completed;
    uint32_t next_slot = 0;
    int64_t clock_offset = 0;  // steady_ns - globaltimer
    ts_activity_sink_fn sink = nullptr;
    void* sink_user = nullptr;

    size_t state_elems() const { return (size_t)(n_owned + n_proxy) * nf * kNC; }
};

namespace {

int fail(ts_hydro_ctx* c, int code, const std::string& msg) {
    if (c != nullptr) c->err = msg;
    return code;
}

int cuda_fail(ts_hydro_ctx* c, cudaError_t e, const char* what) {
    return fail(c, TS_ECUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

#define TS_CUDA(ctx, call)                                   \
    do {                                                     \
        cudaError_t _e = (call);                             \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call); \
    } while (0)

#define TS_NCCL(ctx, call)                                                                        \
    do {                                                                                          \
        ncclResult_t _r = (call);                                                                 \
        if (_r != ncclSuccess)                                                                    \
            return fail(ctx, TS_ENCCL, std::string(#call) + ": " + nccl().GetErrorString(_r));     \
    } while (0)

int guard(ts_hydro_ctx* c) {
    if (c == nullptr) return TS_EINVAL;
    if (c->shut) return fail(c, TS_ESHUTDOWN, "device is shut down");
    // every entry point may enqueue other work: only the steps of one call
    // chain stage 3 -> next stage 1 as programmatic dependents
    c->flow_chain = false;
    return TS_OK;
}

int ensure_stream(ts_hydro_ctx* c, uint32_t id, cudaStream_t* out) {
    if (id >= c->streams.size()) return fail(c, TS_EINVAL, "invalid stream id");
    if (c->streams[id] == nullptr) {
        // The halo (1) and boundary (2) streams carry the critical path of a
        // multi-GPU stage: at the highest priority the CTA scheduler hands them
        // the first SM slots that interior CTAs free, so NCCL and the unpack are
        // not starved behind a GPU-filling interior launch.
        int lo = 0, hi = 0;
        TS_CUDA(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const int prio = (id == 1 || id == 2) ? hi : lo;
        TS_CUDA(c, cudaStreamCreateWithPriority(&c->streams[id], cudaStreamNonBlocking, prio));
    }
    *out = c->streams[id];
    return TS_OK;
}

void record_mem(ts_hydro_ctx* c, uint8_t kind, uint64_t bytes) {
    ts_activity_record r{};
    r.kind = kind;
    r.has_bytes = 1;
    r.device_id = c->cfg.device_id;
    r.stream_id = -1;
    r.name = kind == TS_ACTIVITY_ALLOC ? kNameAlloc : kNameFree;
    r.start_ns = r.end_ns = steady_ns();
    r.bytes = bytes;
    c->completed.push_back(r);
}

template <typename T>
int dalloc(ts_hydro_ctx* c, T** p, size_t elems) {
    const size_t bytes = std::max<size_t>(elems, 1) * sizeof(T);
    void* raw = nullptr;
    cudaError_t e = cudaMalloc(&raw, bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(c, TS_ENOMEM, std::string("cudaMalloc of ") + std::to_string(bytes) +
                                      " bytes failed: " + cudaGetErrorString(e));
    }
    *p = static_cast<T*>(raw);
    c->dev_allocs[raw] = bytes;
    c->mem.current_device_bytes += bytes;
    c->mem.peak_device_bytes = std::max(c->mem.peak_device_bytes, c->mem.current_device_bytes);
    record_mem(c, TS_ACTIVITY_ALLOC, bytes);
    return TS_OK;
}

template <typename T>
void dfree(ts_hydro_ctx* c, T** p) {
    if (*p == nullptr) return;
    auto it = c->dev_allocs.find(*p);
    if (it != c->dev_allocs.end()) {
        c->mem.current_device_bytes -= it->second;
        record_mem(c, TS_ACTIVITY_FREE, it->second);
        c->dev_allocs.erase(it);
    }
    cudaFree(*p);
    *p = nullptr;
}

void close_peers(ts_hydro_ctx* c) {
    for (PeerMap& q : c->pm) {
        if (q.recv) cudaIpcCloseMemHandle(q.recv);
        if (q.flags) cudaIpcCloseMemHandle(q.flags);
        if (q.gather) cudaIpcCloseMemHandle(q.gather);
        for (double* u : q.U)
            if (u) cudaIpcCloseMemHandle(u);
        q = PeerMap{};
    }
    c->pm.clear();
    c->p2p = false;
    dfree(c, &c->d_push_gather);
    dfree(c, &c->d_push_flag);
    dfree(c, &c->d_push_out);
    dfree(c, &c->d_halo_flag);
    c->halo_pushed = false;
}

void free_mesh(ts_hydro_ctx* c) {
    close_peers(c);
    dfree(c, &c->d_flags);
    dfree(c, &c->d_gather);
    dfree(c, &c->d_ctr);
    for (auto& b : c->U) dfree(c, &b);
    dfree(c, &c->d_nbr);
    dfree(c, &c->d_interior);
    dfree(c, &c->d_boundary);
    dfree(c, &c->d_order);
    dfree(c, &c->d_flow);
    dfree(c, &c->d_cnt3);
    dfree(c, &c->d_cta_log);
    dfree(c, &c->d_chunk_ctr);
    dfree(c, &c->d_h2d_flag);
    dfree(c, &c->d_scr_ring);
    dfree(c, &c->d_grav);
    for (auto& r : c->d_fmm_tab)
        for (auto& q : r)
            for (auto& t : q) dfree(c, &t);
    dfree(c, &c->d_scr_mask);
    dfree(c, &c->d_bnd_of);
    dfree(c, &c->d_push_tbl);
    dfree(c, &c->d_gid);
    dfree(c, &c->d_send_entries);
    dfree(c, &c->d_recv_entries);
    dfree(c, &c->d_send);
    dfree(c, &c->d_recv);
    dfree(c, &c->d_amr_proxy);
    dfree(c, &c->d_amr_pmask);
    dfree(c, &c->d_amr_rec);
    dfree(c, &c->d_amr_level);
    dfree(c, &c->d_amr_rf_slot);
    dfree(c, &c->d_amr_rf_flux);
    dfree(c, &c->d_fmm_int);
    dfree(c, &c->d_fmm_M);
    dfree(c, &c->d_fmm_L);
    dfree(c, &c->d_fmm_lists);
    dfree(c, &c->d_fmm_part);
    dfree(c, &c->d_fmm_send);
    dfree(c, &c->d_fmm_rho);
    c->have_fmm = false;
    c->wave_ready = false;
    c->amr = false;
    c->amr_mr = false;
    c->xfer_cells = kSlab;
    c->have_mesh = false;
    c->tmap_ok = false;
}

// Harvest the stamps of every pending launch (device must be idle).
int harvest(ts_hydro_ctx* c) {
    if (c->pending.empty()) return TS_OK;
    const uint32_t cap = c->cfg.activity_buffer_capacity;
    std::vector<unsigned long long> st((size_t)cap * 2);
    TS_CUDA(c, cudaMemcpy(st.data(), c->d_stamps, st.size() * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost));
    // A PDL launch (StageArgs::flow_*) starts its first CTAs in the previous
    // kernel's last wave; its record starts where that kernel's record ends,
    // keeping the SimDevice contract of non-overlapping records per stream.
    std::vector<std::pair<int32_t, uint64_t>> last_end;
    for (const PendingLaunch& p : c->pending) {
        ts_activity_record r{};
        r.kind = p.kind;
        r.device_id = c->cfg.device_id;
        r.stream_id = p.stream_id;
        r.name = p.name;
        r.correlation_guid = p.guid;
        if (p.bytes > 0) {
            r.has_bytes = 1;
            r.bytes = p.bytes;
        }
        unsigned long long enc_start = st[2 * (size_t)p.slot];
        unsigned long long end = st[2 * (size_t)p.slot + 1];
        if (p.e0 != nullptr) {
            // event-timed: globaltimer of ev_cal + elapsed event time
            float ms0 = 0.0f, ms1 = 0.0f;
            const unsigned long long g0 = ((volatile unsigned long long*)c->h_clock)[2];
            if (cudaEventElapsedTime(&ms0, c->ev_cal, p.e0) != cudaSuccess ||
                cudaEventElapsedTime(&ms1, c->ev_cal, p.e1) != cudaSuccess) {
                (void)cudaGetLastError();
                continue;
            }
            enc_start = ~(g0 + (unsigned long long)std::llround(std::max(0.0f, ms0) * 1e6));
            end = g0 + (unsigned long long)std::llround(std::max(ms0, ms1) * 1e6);
        }
        if (enc_start == 0 || end == 0) continue;  // launch had no CTA (empty)
        const unsigned long long start = ~enc_start;
        r.start_ns = (uint64_t)((int64_t)start + c->clock_offset);
        r.end_ns = (uint64_t)((int64_t)std::max(end, start) + c->clock_offset);
        auto it = std::find_if(last_end.begin(), last_end.end(),
                               [&](const std::pair<int32_t, uint64_t>& e) { return e.first == p.stream_id; });
        if (it == last_end.end()) it = last_end.insert(last_end.end(), {p.stream_id, 0});
        if (p.overlap && r.start_ns < it->second) r.start_ns = std::min(it->second, r.end_ns);
        it->second = std::max(it->second, r.end_ns);
        c->completed.push_back(r);
    }
    for (const PendingLaunch& p : c->pending) {
        if (p.e0 != nullptr) c->ev_pool.push_back(p.e0);
        if (p.e1 != nullptr) c->ev_pool.push_back(p.e1);
    }
    c->pending.clear();
    c->cal_armed = false;
    c->next_slot = 0;
    TS_CUDA(c, cudaMemset(c->d_stamps, 0, (size_t)cap * 2 * sizeof(unsigned long long)));
    // legacy-stream work does not order against our non-blocking streams
    TS_CUDA(c, cudaDeviceSynchronize());
    return TS_OK;
}

// Host -> device copy of set-up data that kernels on the context's
// (non-blocking) streams read next: a pageable cudaMemcpy may return before its
// DMA lands, and nothing orders those streams behind the legacy stream — so
// wait for it.
cudaError_t h2d_sync(void* dst, const void* src, size_t bytes) {
    cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? cudaStreamSynchronize(0) : e;
}

int sync_all(ts_hydro_ctx* c) {
    for (cudaStream_t s : c->streams)
        if (s != nullptr) TS_CUDA(c, cudaStreamSynchronize(s));
    if (c->h_clock != nullptr && ((volatile unsigned long long*)c->h_clock)[1] != 0ull) {
        ((volatile unsigned long long*)c->h_clock)[1] = 0ull;
        return fail(c, TS_ECOMM, "a peer rank did not arrive at a cross-GPU wait within the deadline "
                                 "(stepping calls must be collective: same sequence on every rank)");
    }
    return TS_OK;
}

void deliver_to_sink(ts_hydro_ctx* c) {
    if (c->sink == nullptr || c->completed.empty()) return;
    std::vector<ts_activity_record> batch;
    batch.swap(c->completed);
    c->sink(batch.data(), batch.size(), c->sink_user);
}

// Reserve a stamp slot for a launch; flushes (waits) when the ring is full,
// handing records to the sink like SimDevice::take_if_full (device.cpp:105-111).
int begin_launch(ts_hydro_ctx* c, uint8_t kind, const char* name, int32_t stream_id, uint64_t guid,
                 unsigned long long** stamp) {
    if (c->next_slot >= c->cfg.activity_buffer_capacity) {
        int rc = sync_all(c);
        if (rc) return rc;
        rc = harvest(c);
        if (rc) return rc;
        deliver_to_sink(c);
    }
    if (!c->profiling) {  // the harness's "disabled" arm: no stamps, no records
        *stamp = nullptr;
        c->launches++;
        return TS_OK;
    }
    const uint32_t slot = c->next_slot++;
    c->pending.push_back({kind, name, stream_id, guid, slot, false});
    *stamp = c->d_stamps + 2 * (size_t)slot;
    c->launches++;
    return TS_OK;
}

// Host-timed copy record (synchronous copies).
// An event-timed record (see PendingLaunch::e0): the reference event ev_cal is
// recorded on the compute stream right behind a one-thread clock kernel
// (globaltimer into h_clock[2]) once per harvest period.
int begin_event_record(ts_hydro_ctx* c, uint8_t kind, const char* name, int32_t stream_id, uint64_t bytes,
                       PendingLaunch** out) {
    unsigned long long* stamp = nullptr;
    *out = nullptr;
    int rc = begin_launch(c, kind, name, stream_id, 0, &stamp);
    if (rc) return rc;
    c->launches--;  // no kernel
    if (stamp == nullptr) return TS_OK;  // profiling disabled
    if (!c->cal_armed) {
        cudaStream_t s0;
        rc = ensure_stream(c, 0, &s0);
        if (rc) return rc;
        if (c->ev_cal == nullptr) TS_CUDA(c, cudaEventCreate(&c->ev_cal));
        TS_CUDA(c, tsh::launch_clock(c->h_clock + 2, s0));
        TS_CUDA(c, cudaEventRecord(c->ev_cal, s0));
        c->cal_armed = true;
    }
    PendingLaunch& p = c->pending.back();
    for (cudaEvent_t* e : {&p.e0, &p.e1}) {
        if (!c->ev_pool.empty()) {
            *e = c->ev_pool.back();
            c->ev_pool.pop_back();
        } else {
            TS_CUDA(c, cudaEventCreate(e));
        }
    }
    p.bytes = bytes;
    *out = &p;
    return TS_OK;
}

void record_copy(ts_hydro_ctx* c, uint8_t kind, uint64_t bytes, uint64_t t0, uint64_t t1) {
    ts_activity_record r{};
    r.kind = kind;
    r.has_bytes = 1;
    r.device_id = c->cfg.device_id;
    r.stream_id = 0;
    r.name = kind == TS_ACTIVITY_COPY_H2D ? kNameH2D : kNameD2H;
    r.start_ns = t0;
    r.end_ns = t1;
    r.bytes = bytes;
    c->completed.push_back(r);
}

int calibrate_clock(ts_hydro_ctx* c) {
    cudaStream_t s;
    int rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    int64_t best_span = INT64_MAX;
    for (int trial = 0; trial < 5; ++trial) {
        volatile unsigned long long* hv = c->h_clock;
        *hv = 0;
        const uint64_t t0 = steady_ns();
        TS_CUDA(c, tsh::launch_clock(c->h_clock, s));
        while (*hv == 0) {
        }
        const uint64_t t1 = steady_ns();
        const unsigned long long g = *hv;
        TS_CUDA(c, cudaStreamSynchronize(s));
        const int64_t span = (int64_t)(t1 - t0);
        if (span < best_span) {
            best_span = span;
            c->clock_offset = (int64_t)(t0 + (t1 - t0) / 2) - (int64_t)g;
        }
    }
    return TS_OK;
}

// ---- mesh helpers -----------------------------------------------------------
uint64_t morton3(uint32_t x, uint32_t y, uint32_t z) {
    uint64_t out = 0;
    for (int b = 0; b < 21; ++b) {
        out |= (uint64_t)((x >> b) & 1u) << (3 * b);
        out |= (uint64_t)((y >> b) & 1u) << (3 * b + 1);
        out |= (uint64_t)((z >> b) & 1u) << (3 * b + 2);
    }
    return out;
}

int build_plans(ts_hydro_ctx* c, const int64_t* nbr, const int32_t* owner) {
    if (c->amr_mr) return TS_OK;  // multi-rank AMR plans are built by ts_hydro_set_amr_mesh_partitioned
    c->peers.clear();
    if (c->world <= 1) return TS_OK;
    std::vector<Peer> peers((size_t)c->world);
    for (int r = 0; r < c->world; ++r) peers[(size_t)r].rank = r;
    // send: my owned sub-grids' slabs facing a foreign neighbour, by (gid, face)
    for (int64_t h : c->owned_gid)
        for (int f = 0; f < 6; ++f) {
            const int64_t nb = nbr[6 * h + f];
            if (nb < 0) continue;
            const int r = owner[nb];
            if (r == c->rank) continue;
            peers[(size_t)r].send_pairs.push_back(h);
            peers[(size_t)r].send_pairs.push_back(f);
        }
    // recv: foreign proxies' slabs facing one of my sub-grids, by (gid, face)
    for (int64_t p : c->proxy_gid)
        for (int f = 0; f < 6; ++f) {
            const int64_t nb = nbr[6 * p + f];
            if (nb < 0 || owner[nb] != c->rank) continue;
            peers[(size_t)owner[p]].recv_pairs.push_back(p);
            peers[(size_t)owner[p]].recv_pairs.push_back(f);
        }
    // where each sent slab lands on the receiver: its local numbering is owned
    // sub-grids (ascending id), then proxies (ascending id)
    for (Peer& p : peers) {
        if (p.rank == c->rank || p.send_pairs.empty()) continue;
        std::vector<int64_t> their_owned, their_proxy;
        std::vector<char> is_proxy((size_t)c->n_global, 0);
        for (int64_t i = 0; i < c->n_global; ++i) {
            if (owner[i] != p.rank) continue;
            their_owned.push_back(i);
            for (int f = 0; f < 6; ++f) {
                const int64_t nb = nbr[6 * i + f];
                if (nb >= 0 && owner[nb] != p.rank) is_proxy[(size_t)nb] = 1;
            }
        }
        for (int64_t i = 0; i < c->n_global; ++i)
            if (is_proxy[(size_t)i]) their_proxy.push_back(i);
        for (size_t k = 0; k < p.send_pairs.size(); k += 2) {
            const auto it = std::lower_bound(their_proxy.begin(), their_proxy.end(), p.send_pairs[k]);
            p.send_dst.push_back((int32_t)((int64_t)their_owned.size() + (it - their_proxy.begin())));
        }
    }
    int64_t so = 0, ro = 0;
    for (Peer& p : peers) {
        p.n_send = (int64_t)p.send_pairs.size() / 2;
        p.n_recv = (int64_t)p.recv_pairs.size() / 2;
        p.send_off = so;
        p.recv_off = ro;
        so += p.n_send;
        ro += p.n_recv;
    }
    c->n_send_total = so;
    c->n_recv_total = ro;
    c->peers = std::move(peers);
    return TS_OK;
}

// Max-signal-speed slot of step s: a ring of three (stage 1 of one step may
// run while the previous step's stage 3 still accumulates; see
// StageArgs::cnt_wait) — on one rank and, for the chained fused-P2P steps, on N.
double* amax_slot(const ts_hydro_ctx* c, uint64_t s) {
    static constexpr int kRing[3] = {0, 1, 5};
    return c->d_scal + kRing[s % 3];
}

int64_t local_of(const ts_hydro_ctx* c, int64_t gid) {
    auto it = std::lower_bound(c->owned_gid.begin(), c->owned_gid.end(), gid);
    if (it != c->owned_gid.end() && *it == gid) return it - c->owned_gid.begin();
    auto jt = std::lower_bound(c->proxy_gid.begin(), c->proxy_gid.end(), gid);
    if (jt != c->proxy_gid.end() && *jt == gid) return c->n_owned + (jt - c->proxy_gid.begin());
    return -1;
}

tsh::StageArgs stage_args(ts_hydro_ctx* c, int stage) {
    tsh::StageArgs a{};
    double* A = c->U[0];
    double* B = c->U[1];
    double* C = c->U[2];
    a.Uprev = stage == 1 ? A : (stage == 2 ? B : C);
    if (c->tmap_ok) {
        a.tmap_prev = c->tmap[stage - 1];  // U[0], U[1], U[2] = A, B, C
        a.tma = 1;
    }
    a.check = c->d_check;
    a.n_local = c->n_owned + c->n_proxy;
    a.n_owned = c->n_owned;
    if (c->d_scr_ring != nullptr) {
        a.scr_ring = c->d_scr_ring;
        a.scr_mask = c->d_scr_mask;
        a.scr_k = ts_hydro_ctx::kScrK;
    }
    a.Un = A;
    a.Uout = stage == 1 ? B : (stage == 2 ? C : A);
    // free during the stage: stage 1 writes B (C unused), stage 2 writes C,
    // stage 3 writes A = U^n in place (B unused)
    a.scratch = stage == 1 ? C : (stage == 2 ? C : B);
    a.nbr = c->d_nbr;
    a.list = nullptr;
    a.first = 0;
    a.amax_in = c->amax_src != nullptr ? c->amax_src : amax_slot(c, c->steps_done);
    a.amax_n = c->amax_src != nullptr ? c->amax_n : 1;
    a.amax_out = amax_slot(c, c->steps_done + 1);
    a.amax_reset = nullptr;
    a.dt_out = nullptr;
    a.gamma = c->cfg.gamma;
    a.gm1 = c->cfg.gamma - 1.0;
    a.cfl = c->cfg.cfl;
    a.dx = c->cfg.dx;
    a.dx_upd = c->cfg.dx;
    a.p_floor = c->cfg.p_floor;
    a.err = c->h_clock + 1;
    a.wait_ns = c->wait_ns;
    return a;
}

int launch_stage_list(ts_hydro_ctx* c, tsh::StageArgs a, int stage, const int32_t* d_list, int64_t count,
                      int first, uint32_t stream_id, uint64_t guid, bool pdl = false) {
    if (count <= 0) return TS_OK;
    cudaStream_t s;
    int rc = ensure_stream(c, stream_id, &s);
    if (rc) return rc;
    unsigned long long* stamp = nullptr;
    rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameStage[stage], (int32_t)stream_id, guid, &stamp);
    if (rc) return rc;
    if (stamp != nullptr) c->pending.back().overlap = pdl;
    a.list = d_list;
    a.first = first;
    a.stamp = stamp;
    TS_CUDA(c, tsh::launch_stage(a, c->nf, c->cfg.recon, stage, (int)count, s, pdl));
    return TS_OK;
}

// Pack -> transfer -> unpack of buffer `buf` on the comm stream.  Transport:
// P2P (copy engines into the peer's receive buffer, flag write / wait stream
// memory ops; double-buffered by exchange parity) or NCCL grouped send/recv.
int pack_on_comm(ts_hydro_ctx* c, const double* buf) {
    cudaStream_t cs;
    int rc = ensure_stream(c, 1, &cs);
    if (rc) return rc;
    if (c->n_send_total > 0) {
        unsigned long long* stamp = nullptr;
        rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNamePack, 1, 0, &stamp);
        if (rc) return rc;
        TS_CUDA(c, tsh::launch_pack(buf, c->nf, c->d_send_entries, c->n_send_total, c->d_send, c->sms, cs, stamp,
                                    c->xfer_cells));
    }
    return TS_OK;
}

int exchange_on_comm(ts_hydro_ctx* c, double* buf, bool packed = false) {
    cudaStream_t cs;
    int rc = ensure_stream(c, 1, &cs);
    if (rc) return rc;
    if (!packed) {
        rc = pack_on_comm(c, buf);
        if (rc) return rc;
    }
    const size_t per = (size_t)c->nf * c->xfer_cells;
    double* recv = c->d_recv;
    if (c->p2p) {
        StreamMemOps& m = memops();
        const uint32_t seq = ++c->xseq;
        const int h = (int)(seq & 1);
        for (const Peer& p : c->peers) {
            if (p.rank == c->rank || p.n_send == 0) continue;
            const PeerMap& q = c->pm[(size_t)p.rank];
            double* dst = q.recv + ((size_t)h * (size_t)q.n_recv_total + (size_t)q.recv_off_for_me) * per;
            TS_CUDA(c, cudaMemcpyAsync(dst, c->d_send + (size_t)p.send_off * per, (size_t)p.n_send * per * sizeof(double),
                                       cudaMemcpyDeviceToDevice, cs));
            if (m.write32(cs, (CUdeviceptr)(q.flags + c->rank), seq, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
                return fail(c, TS_ECUDA, "cuStreamWriteValue32 to a peer flag failed");
        }
        TS_CUDA(c, tsh::launch_wait_flags(reinterpret_cast<const unsigned int*>(c->d_flags), c->halo_recv_mask, seq,
                                          c->h_clock + 1, c->wait_ns, cs));
        recv = c->d_recv + (size_t)h * (size_t)c->n_recv_total * per;
    } else if (c->comm != nullptr) {
        Nccl& n = nccl();
        TS_NCCL(c, n.GroupStart());
        for (const Peer& p : c->peers) {
            if (p.rank == c->rank) continue;
            if (p.n_send > 0)
                TS_NCCL(c, n.Send(c->d_send + (size_t)p.send_off * per, (size_t)p.n_send * per, ncclFloat64,
                                  p.rank, c->comm, cs));
            if (p.n_recv > 0)
                TS_NCCL(c, n.Recv(c->d_recv + (size_t)p.recv_off * per, (size_t)p.n_recv * per, ncclFloat64,
                                  p.rank, c->comm, cs));
        }
        TS_NCCL(c, n.GroupEnd());
    }
    if (c->n_recv_total > 0) {
        unsigned long long* stamp = nullptr;
        rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameUnpack, 1, 0, &stamp);
        if (rc) return rc;
        TS_CUDA(c, tsh::launch_unpack(buf, c->nf, c->d_recv_entries, c->n_recv_total, recv, c->sms, cs, stamp,
                                      c->xfer_cells));
    }
    return TS_OK;
}

// Global max of one signal speed per rank, on stream `s`.  NCCL: in-place
// all-reduce (amax_src = slot).  P2P: every rank copies its value into slot
// `rank` of every peer's gather array (parity-double-buffered) and waits for
// the peers' flags; the stage kernel takes the max over the gathered values.
int reduce_amax(ts_hydro_ctx* c, double* slot, cudaStream_t s) {
    c->amax_src = nullptr;
    c->amax_n = 1;
    if (c->world <= 1) return TS_OK;
    if (c->p2p) {
        StreamMemOps& m = memops();
        const uint32_t seq = ++c->aseq;
        const int h = (int)(seq & 1);
        double* mine = c->d_gather + (size_t)h * c->world;
        TS_CUDA(c, cudaMemcpyAsync(mine + c->rank, slot, sizeof(double), cudaMemcpyDeviceToDevice, s));
        for (int r = 0; r < c->world; ++r) {
            if (r == c->rank) continue;
            const PeerMap& q = c->pm[(size_t)r];
            TS_CUDA(c, cudaMemcpyAsync(q.gather + (size_t)h * c->world + c->rank, slot, sizeof(double),
                                       cudaMemcpyDeviceToDevice, s));
            if (m.write32(s, (CUdeviceptr)(q.flags + c->world + c->rank), seq, CU_STREAM_WRITE_VALUE_DEFAULT) !=
                CUDA_SUCCESS)
                return fail(c, TS_ECUDA, "cuStreamWriteValue32 to a peer flag failed");
        }
        uint64_t others = 0;
        for (int r = 0; r < c->world; ++r)
            if (r != c->rank) others |= 1ull << r;
        TS_CUDA(c, tsh::launch_wait_flags(reinterpret_cast<const unsigned int*>(c->d_flags + c->world), others, seq,
                                          c->h_clock + 1, c->wait_ns, s));
        c->amax_src = mine;
        c->amax_n = c->world;
        return TS_OK;
    }
    if (c->comm != nullptr && c->comm_size > 1) {
        Nccl& n = nccl();
        TS_NCCL(c, n.AllReduce(slot, slot, 1, ncclFloat64, ncclMax, c->comm, s));
    }
    return TS_OK;
}

// Device-side barrier of the ranks on stream `s` (P2P: one flag word per peer
// on the dt-gather channel, no data; NCCL: an all-reduce of a scratch word).
// ts_hydro_time_steps starts its clock behind it, so the host-side skew of the
// ranks entering the call (a gloo barrier releases them tens of microseconds
// apart) is not charged to the steps.
int device_barrier(ts_hydro_ctx* c, cudaStream_t s) {
    if (c->world <= 1) return TS_OK;
    if (c->p2p) {
        StreamMemOps& m = memops();
        const uint32_t seq = ++c->aseq;
        uint64_t others = 0;
        for (int r = 0; r < c->world; ++r) {
            if (r == c->rank) continue;
            others |= 1ull << r;
            if (m.write32(s, (CUdeviceptr)(c->pm[(size_t)r].flags + c->world + c->rank), seq,
                          CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
                return fail(c, TS_ECUDA, "cuStreamWriteValue32 to a peer flag failed");
        }
        TS_CUDA(c, tsh::launch_wait_flags(reinterpret_cast<const unsigned int*>(c->d_flags + c->world), others, seq,
                                          c->h_clock + 1, c->wait_ns, s));
        return TS_OK;
    }
    if (c->comm != nullptr && c->comm_size > 1) {
        Nccl& n = nccl();
        TS_NCCL(c, n.AllReduce(c->d_scal + 6, c->d_scal + 6, 1, ncclFloat64, ncclMax, c->comm, s));
    }
    return TS_OK;
}

int do_compute_dt(ts_hydro_ctx* c) {
    cudaStream_t s;
    int rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    double* slot = amax_slot(c, c->steps_done);
    TS_CUDA(c, cudaMemsetAsync(slot, 0, sizeof(double), s));
    unsigned long long* stamp = nullptr;
    rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameSignal, 0, 0, &stamp);
    if (rc) return rc;
    TS_CUDA(c, tsh::launch_signal(c->U[0], c->nf, c->n_owned, c->cfg.gamma, c->cfg.p_floor, slot, stamp,
                                  c->sms, s));
    rc = reduce_amax(c, slot, s);
    if (rc) return rc;
    c->dt_valid = true;
    return TS_OK;
}

// One step on an AMR mesh (single rank, stream order): per stage, refill the
// proxies of U^(k-1) (prolongation / restriction), the stage over all leaves
// (one launch; each CTA takes its level's dx from StageArgs::lvl_*, so the
// level-0 launch's tail no longer idles the GPU before the level-1 launch;
// TS_HYDRO_AMR_SPLIT=1 or > kMaxLevels levels: one launch per level, the
// first of stage 1 writing dt and zeroing the max slot stage 3 accumulates
// into), then the coarse flux correction.
int do_step_amr(ts_hydro_ctx* c) {
    cudaStream_t s;
    int rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    const double* dt_ptr = c->d_dt_hist + (c->steps_done % ts_hydro_ctx::kDtHist);
    const bool multi = c->world > 1;
    for (int stage = 1; stage <= 3; ++stage) {
        tsh::StageArgs a = stage_args(c, stage);
        unsigned long long* stamp = nullptr;
        if (multi) {
            // ghost leaves of U^(k-1): whole sub-grids from their owners
            cudaStream_t cs;
            rc = ensure_stream(c, 1, &cs);
            if (rc) return rc;
            TS_CUDA(c, cudaEventRecord(c->ev_in, s));
            TS_CUDA(c, cudaStreamWaitEvent(cs, c->ev_in, 0));
            rc = exchange_on_comm(c, const_cast<double*>(a.Uprev));
            if (rc) return rc;
            TS_CUDA(c, cudaEventRecord(c->ev_halo, cs));
            TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_halo, 0));
        }
        if (c->amr_n_proxy > 0) {
            rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameAmrFill, 0, 0, &stamp);
            if (rc) return rc;
            TS_CUDA(c, tsh::launch_amr_fill(const_cast<double*>(a.Uprev), c->nf, c->d_amr_proxy,
                                            c->amr_slab_fill ? c->d_amr_pmask : nullptr, c->amr_n_proxy,
                                            stamp, s));
        }
        if (c->d_amr_rf_slot != nullptr) {
            a.rf_slot = c->d_amr_rf_slot;
            a.rf_flux = c->d_amr_rf_flux;
        }
        if (c->amr_fused && c->amr_max_level < tsh::StageArgs::kMaxLevels) {
            tsh::StageArgs b = a;
            b.lvl_n = c->amr_max_level + 1;
            for (int L = 0; L <= c->amr_max_level; ++L) {
                b.lvl_first[L] = (int)c->amr_level_first[(size_t)L];
                b.lvl_dx[L] = std::ldexp(c->cfg.dx, c->amr_max_level - L);
            }
            b.dx_upd = b.lvl_dx[0];
            if (stage == 1) {
                b.amax_reset = amax_slot(c, c->steps_done + 1);
                b.dt_out = const_cast<double*>(dt_ptr);
            }
            rc = launch_stage_list(c, b, stage, nullptr, c->n_owned, 0, 0, 0);
            if (rc) return rc;
        }
        bool first = true;
        for (int L = 0; L <= c->amr_max_level && !(c->amr_fused && c->amr_max_level < tsh::StageArgs::kMaxLevels);
             ++L) {
            const int64_t f0 = c->amr_level_first[(size_t)L], n = c->amr_level_first[(size_t)L + 1] - f0;
            if (n <= 0) continue;
            tsh::StageArgs b = a;
            b.dx_upd = std::ldexp(c->cfg.dx, c->amr_max_level - L);
            if (stage == 1 && first) {
                b.amax_reset = amax_slot(c, c->steps_done + 1);
                b.dt_out = const_cast<double*>(dt_ptr);
            }
            rc = launch_stage_list(c, b, stage, nullptr, n, (int)f0, 0, 0);
            if (rc) return rc;
            first = false;
        }
        if (c->amr_n_rec > 0) {
            rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameAmrReflux, 0, 0, &stamp);
            if (rc) return rc;
            if (c->d_amr_rf_slot != nullptr)
                TS_CUDA(c, tsh::launch_amr_reflux_reg(a.Uout, c->nf, c->d_amr_level, c->amr_max_level, c->cfg.dx,
                                                      c->d_amr_rec, c->amr_n_rec, c->d_amr_rf_slot, c->d_amr_rf_flux,
                                                      stage, dt_ptr, stamp, s));
            else
                TS_CUDA(c, tsh::launch_amr_reflux(a.Uprev, a.Uout, c->nf, c->cfg.recon, c->cfg.gamma, c->cfg.p_floor,
                                                  c->d_nbr, c->d_amr_level, c->amr_max_level, c->cfg.dx, c->d_amr_rec,
                                                  c->amr_n_rec, stage, dt_ptr, stamp, s));
        }
    }
    double* slot = amax_slot(c, c->steps_done + 1);
    if (c->amr_n_rec > 0) {
        // The stage-3 kernel reduced the signal speed of U^{n+1} as it wrote
        // it, but the reflux after it corrects coarse cells: the next dt must
        // come from the corrected state (the oracle's max_signal_speed of the
        // final U^{n+1}).  Found by the reference-octree AMR parity test
        // (minmod: the maximum sat on a refluxed cell).
        TS_CUDA(c, cudaMemsetAsync(slot, 0, sizeof(double), s));
        unsigned long long* stamp = nullptr;
        rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameSignal, 0, 0, &stamp);
        if (rc) return rc;
        TS_CUDA(c, tsh::launch_signal(c->U[0], c->nf, c->n_owned, c->cfg.gamma, c->cfg.p_floor, slot, stamp,
                                      c->sms, s));
    }
    c->amax_src = nullptr;
    if (multi) {
        // the global max over the ranks (p2p gather or NCCL all-reduce), the
        // next step's dt (reduce_amax points amax_src at the result)
        rc = reduce_amax(c, slot, s);
        if (rc) return rc;
    }
    c->flow_chain = false;
    c->steps_done++;
    return TS_OK;
}

int do_step(ts_hydro_ctx* c) {
    if (c->amr) return do_step_amr(c);
    cudaStream_t s, cs, bs;
    int rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    const bool multi = c->world > 1;
    if (multi) {
        rc = ensure_stream(c, 1, &cs);
        if (!rc) rc = ensure_stream(c, 2, &bs);
        if (rc) return rc;
    }
    const bool p2p = multi && c->p2p;
    const bool fused_halo = p2p && c->halo_fused;
    const uint32_t push_seq = c->aseq + 1;
    // single rank: stage 1 follows the previous step in stream order (its dt
    // needs every sub-grid's stage 3); stages 2 and 3 start in the previous
    // stage's tail and wait per sub-grid (StageArgs::flow_*).  The tail this
    // fills is at most one wave of a stage, so it pays only for a few waves
    // (measured on B200: +2.7 % at 4096 sub-grids = 4.6 waves of 6 CTAs/SM,
    // -0.7 % at 32768 = 37 waves): used up to 10 waves.
    // With N ranks the same holds for the fused P2P exchange: foreign
    // neighbours stay gated by the halo flags, local ones by the stage flags.
    const bool flow = (!multi || fused_halo) && c->flow && c->d_flow != nullptr &&
                      c->n_owned <= 10 * 6 * (int64_t)c->sms;
    // across the step boundary too (stage 1 a PDL dependent of stage 3): one
    // rank, or N ranks whose dt is gathered in stage 3's tail (StageArgs::cnt_gather)
    const bool mchain = fused_halo && !c->dt_kernel && c->mchain;
    const bool steps = flow && c->flow_steps && (!multi || mchain);
    if (flow) ++c->flow_seq;
    for (int stage = 1; stage <= 3; ++stage) {
        tsh::StageArgs a = stage_args(c, stage);
        if (c->d_cta_log != nullptr) a.cta_log = c->d_cta_log + 4 * (size_t)(stage - 1) * (size_t)c->n_owned;
        const bool chain = steps && c->flow_chain;
        if (stage == 1) {
            a.amax_reset = chain ? nullptr : amax_slot(c, c->steps_done + 1);
            if (!multi || mchain) a.amax_reset2 = amax_slot(c, c->steps_done + 2);
            a.dt_out = c->d_dt_hist + (c->steps_done % ts_hydro_ctx::kDtHist);
        }
        if (stage == 1 && c->h2d_arm) {
            a.h2d_flag = c->d_h2d_flag;
            a.h2d_seq = c->h2d_seq;
            a.chunk_n = c->xfer_chunks;
            a.chunk_owned = (int)c->n_owned;
            c->h2d_arm = false;
        }
        if (stage == 3 && c->chunk_arm) {
            a.chunk_ctr = c->d_chunk_ctr;
            a.chunk_n = c->xfer_chunks;
            a.chunk_owned = (int)c->n_owned;
        }
        if (p2p && stage == 3 && !c->dt_kernel) {
            a.done_ctr = c->d_ctr;
            c->done_cnt += (uint32_t)c->n_owned;
            a.done_target = c->done_cnt;
            a.rank = c->rank;
        }
        if (p2p && stage == 3 && !c->dt_kernel) {
            // dt all-reduce fused into the stage-3 tail (see StageArgs)
            a.push_n = c->world;
            a.push_gather = c->d_push_gather + (size_t)(push_seq & 1) * c->world;
            a.push_flag = c->d_push_flag;
            a.seq = push_seq;
            a.dt_wait = reinterpret_cast<const unsigned int*>(c->d_flags + c->world);
            a.gather_own = c->d_gather + (size_t)(push_seq & 1) * c->world;
            a.amax_global = c->d_scal + 4;
        }
        if (flow) {
            const size_t n = (size_t)c->n_owned;
            a.flow_seq = c->flow_seq;  // `steps`: stage 3 feeds the next stage 1 too
            a.flow_wait_seq = c->flow_seq;
#if defined(TS_CHECK) && TS_CHECK
            // detector self-test (check builds only): wait for the PREVIOUS
            // step's flags, i.e. a broken ordering the exit re-check must catch
            if (stage > 1 && std::getenv("TS_HYDRO_DEBUG_BREAK_FLOW") != nullptr) a.flow_wait_seq = c->flow_seq - 1;
#endif
            a.flow_n = (int)c->n_owned;
            a.pdl_trigger = stage < 3 || steps;
            a.flow_wait = stage > 1 ? c->d_flow + (size_t)(stage - 2) * n : nullptr;
            a.flow_done = stage < 3 || steps ? c->d_flow + (size_t)(stage - 1) * n : nullptr;
            if (stage == 1 && chain) {
                a.flow_wait = c->d_flow + 2 * n;
                a.flow_wait_seq = c->flow_seq - 1;
                a.cnt_wait = c->d_cnt3;
                a.cnt_expect = c->cnt3_expect;
            }
            if (stage == 3 && steps) {
                a.cnt_done = c->d_cnt3;
                a.cnt_gather = multi ? 1 : 0;  // N ranks: the gathering CTA counts, once dt is global
                c->cnt3_expect += (uint32_t)c->n_owned;
            }
        }
        if (!multi) {
            rc = launch_stage_list(c, a, stage, nullptr, c->n_owned, 0, 0, 0, flow && (stage > 1 || chain));
            if (rc) return rc;
            continue;
        }
        double* in = const_cast<double*>(a.Uprev);
        if (fused_halo) {
            // One launch, boundary sub-grids first; they acquire the peers'
            // slabs of U^(k-1) (pushed during the previous stage), push their
            // own U^(k) slabs into the peers' proxies and release the peers'
            // flags.  The first stage of a call refreshes the proxies of U^n
            // by the copy-engine exchange instead (the state may have been
            // replaced since the last push).
            if (c->halo_pushed) {
                a.halo_wait = reinterpret_cast<const unsigned int*>(c->d_flags);
                a.halo_wait_mask = c->halo_recv_mask;
                a.halo_wait_seq = c->xseq;
            } else {
                TS_CUDA(c, cudaEventRecord(c->ev_in, s));
                TS_CUDA(c, cudaStreamWaitEvent(cs, c->ev_in, 0));
                rc = exchange_on_comm(c, in);
                if (rc) return rc;
                TS_CUDA(c, cudaEventRecord(c->ev_halo, cs));
                TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_halo, 0));
            }
            const int out_idx = stage == 1 ? 1 : (stage == 2 ? 2 : 0);
            a.n_boundary = (int)c->boundary.size();
            a.bnd_of = c->d_bnd_of;
            a.push_tbl = c->d_push_tbl;
            a.push_out = c->d_push_out + (size_t)out_idx * c->world;
            a.halo_flag = c->d_halo_flag;
            a.halo_flag_n = c->world;
            a.halo_seq = ++c->xseq;
            {
                const int slot = (int)(a.halo_seq % 3u);
                a.halo_ctr = c->d_ctr + 1 + slot;
                c->halo_cnt[slot] += (uint32_t)c->boundary.size();
                a.halo_target = c->halo_cnt[slot];
            }
            // a stage that began with the copy-engine refresh waits on its
            // event in stream order; the others start in the previous tail
            rc = launch_stage_list(c, a, stage, c->d_order, c->n_owned, 0, 0, 0,
                                   flow && (stage > 1 || chain) && a.halo_wait != nullptr);
            if (rc) return rc;
            c->halo_pushed = true;
            continue;
        }
        // Copy-engine / NCCL halos.  U^(k-1) complete (interior + boundary of
        // the previous stage).  The interior launch goes first (it needs no
        // halo); the exchange is issued behind it on the high-priority halo
        // stream (pack -> transfer -> unpack) and the boundary sub-grids follow
        // on the high-priority boundary stream, so they back-fill SMs as
        // interior CTAs retire.
        TS_CUDA(c, cudaEventRecord(c->ev_in, s));
        TS_CUDA(c, cudaStreamWaitEvent(cs, c->ev_in, 0));
        TS_CUDA(c, cudaStreamWaitEvent(bs, c->ev_in, 0));
        // the (tiny) pack kernel is issued first so it is not queued behind a
        // GPU-filling interior launch for an SM slot
        rc = pack_on_comm(c, in);
        if (rc) return rc;
        rc = launch_stage_list(c, a, stage, c->d_interior, (int64_t)c->interior.size(), 0, 0, 0);
        if (rc) return rc;
        rc = exchange_on_comm(c, in, /*packed=*/true);
        if (rc) return rc;
        TS_CUDA(c, cudaEventRecord(c->ev_halo, cs));
        TS_CUDA(c, cudaStreamWaitEvent(bs, c->ev_halo, 0));
        tsh::StageArgs b = a;
        b.amax_reset = c->interior.empty() ? a.amax_reset : nullptr;
        b.dt_out = c->interior.empty() ? a.dt_out : nullptr;
        rc = launch_stage_list(c, b, stage, c->d_boundary, (int64_t)c->boundary.size(), 0, 2, 0);
        if (rc) return rc;
        TS_CUDA(c, cudaEventRecord(c->ev_bnd, bs));
        TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_bnd, 0));
    }
    if (p2p) {
        if (c->dt_kernel) {
            TS_CUDA(c, tsh::launch_dt_exchange(amax_slot(c, c->steps_done + 1),
                                               c->d_push_gather + (size_t)(push_seq & 1) * c->world, c->d_push_flag,
                                               c->world, c->rank, push_seq,
                                               reinterpret_cast<const unsigned int*>(c->d_flags + c->world),
                                               c->d_gather + (size_t)(push_seq & 1) * c->world, c->d_scal + 4,
                                               c->h_clock + 1, c->wait_ns, s));
            c->launches++;
        }
        // the stage-3 tail (or the dt kernel) gathered every rank's max: the next dt is local
        c->aseq = push_seq;
        c->amax_src = c->d_scal + 4;
        c->amax_n = 1;
    } else if (multi) {
        double* slot = amax_slot(c, c->steps_done + 1);
        TS_CUDA(c, cudaEventRecord(c->ev_in, s));
        TS_CUDA(c, cudaStreamWaitEvent(cs, c->ev_in, 0));
        rc = reduce_amax(c, slot, cs);
        if (rc) return rc;
        TS_CUDA(c, cudaEventRecord(c->ev_red, cs));
        TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_red, 0));
    } else {
        c->amax_src = nullptr;
    }
    c->flow_chain = steps;
    c->steps_done++;
    return TS_OK;
}

// ---- per-sub-grid drop-in steps (ts_hydro_launch_stage) -------------------
// Open a step: stage-1 launches of the step wait (stream event) for
// everything already on the compute stream; when the previous step was not a
// drop-in step (no flags / stage-3 count on the device for it), dt comes from
// the stream-ordered signal speed and the max slots this step and the next
// accumulate into are zeroed here.
int join_gravity(ts_hydro_ctx* c);

int dropin_open(ts_hydro_ctx* c) {
    if (!c->dt_valid) return fail(c, TS_ESTATE, "no dt (call ts_hydro_compute_dt first)");
    cudaStream_t s0;
    int rc = ensure_stream(c, 0, &s0);
    if (rc) return rc;
    if ((rc = join_gravity(c))) return rc;  // the step rewrites U^n in stage 3
    if (c->ev_din == nullptr) TS_CUDA(c, cudaEventCreateWithFlags(&c->ev_din, cudaEventDisableTiming));
    if (c->world > 1) {
        // the proxies of U^n: the peers' stage-3 pushes of the previous step,
        // or (state replaced / first step) a copy-engine refresh behind
        // everything on the compute stream
        c->din_chained = false;
        c->din_wait1 = c->halo_pushed;
        if (!c->halo_pushed) {
            cudaStream_t cs;
            if ((rc = ensure_stream(c, 1, &cs))) return rc;
            TS_CUDA(c, cudaEventRecord(c->ev_in, s0));
            TS_CUDA(c, cudaStreamWaitEvent(cs, c->ev_in, 0));
            if ((rc = exchange_on_comm(c, c->U[0]))) return rc;
            TS_CUDA(c, cudaEventRecord(c->ev_halo, cs));
            TS_CUDA(c, cudaStreamWaitEvent(s0, c->ev_halo, 0));
        }
        c->din_xbase = c->xseq;
        for (int k = 1; k <= 3; ++k) {
            const int slot = (int)((c->din_xbase + (uint32_t)k) % 3u);
            c->halo_cnt[slot] += (uint32_t)c->boundary.size();
            c->din_halo_target[k] = c->halo_cnt[slot];
            c->din_bnd_issued[k] = 0;
        }
        c->bnd_host.assign((size_t)c->n_owned, -1);
        for (size_t b = 0; b < c->boundary.size(); ++b) c->bnd_host[(size_t)c->boundary[b]] = (int32_t)b;
    }
    if (c->amr) {
        c->din_chained = false;
        for (int k = 0; k < 4; ++k) {
            c->din_count[k] = 0;
            c->din_amr_barrier[k] = false;
            if (c->ev_amr[k] == nullptr) TS_CUDA(c, cudaEventCreateWithFlags(&c->ev_amr[k], cudaEventDisableTiming));
        }
        if (c->amr_n_proxy > 0) {  // the proxies of U^n, behind everything on the compute stream
            unsigned long long* stamp = nullptr;
            if ((rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameAmrFill, 0, 0, &stamp))) return rc;
            TS_CUDA(c, tsh::launch_amr_fill(c->U[0], c->nf, c->d_amr_proxy, c->amr_slab_fill ? c->d_amr_pmask : nullptr,
                                            c->amr_n_proxy, stamp, s0));
        }
    }
    if (!c->din_chained) {
        TS_CUDA(c, cudaMemsetAsync(amax_slot(c, c->steps_done + 1), 0, sizeof(double), s0));
        TS_CUDA(c, cudaMemsetAsync(amax_slot(c, c->steps_done + 2), 0, sizeof(double), s0));
    }
    TS_CUDA(c, cudaEventRecord(c->ev_din, s0));
    c->din_open = true;
    c->din_seq = ++c->flow_seq;
    c->din_req.assign((size_t)c->n_owned, 0);
    c->din_issued.assign((size_t)c->n_owned, 0);
    c->din_streams.assign(c->streams.size(), 0);
    c->din_done3 = 0;
    c->din_parked.clear();
    return TS_OK;
}

bool dropin_ready(const ts_hydro_ctx* c, const ts_hydro_ctx::DropinLaunch& L) {
    if (L.stage == 1) return true;
    if (c->amr) return c->din_count[L.stage - 1] == c->n_owned;
    const uint8_t need = (uint8_t)(L.stage - 1);
    if (c->world > 1 && c->din_bnd_issued[L.stage - 1] < (int64_t)c->boundary.size()) {
        for (int32_t g : L.list)
            if (c->bnd_host[(size_t)g] >= 0) return false;
    }
    for (int32_t g : L.list) {
        if (c->din_issued[(size_t)g] < need) return false;
        for (int f = 0; f < 6; ++f) {
            const int32_t h = c->nbr_local[(size_t)g * 6 + f];
            if (h >= 0 && h < c->n_owned && c->din_issued[(size_t)h] < need) return false;
        }
    }
    return true;
}

// The launch(es) of a drop-in list — by value in the parameters (<= 32
// sub-grids) or as runs of consecutive indices, one launch per run — and the
// step's bookkeeping.
int dropin_launch_list(ts_hydro_ctx* c, const ts_hydro_ctx::DropinLaunch& L, tsh::StageArgs a, cudaStream_t s) {
    const int stage = L.stage;
    const size_t m = L.list.size();
    if (m <= (size_t)tsh::StageArgs::kInlineList) {
        a.list_inline_n = (int)m;
        for (size_t k = 0; k < m; ++k) a.list_inline[k] = L.list[k];
        TS_CUDA(c, tsh::launch_stage(a, c->nf, c->cfg.recon, stage, (int)m, s, false));
    } else {
        for (size_t k = 0; k < m;) {
            size_t e = k + 1;
            while (e < m && L.list[e] == L.list[e - 1] + 1) ++e;
            a.list_inline_n = 0;
            a.first = L.list[k];
            TS_CUDA(c, tsh::launch_stage(a, c->nf, c->cfg.recon, stage, (int)(e - k), s, false));
            k = e;
        }
    }
    if (L.done != nullptr) TS_CUDA(c, cudaLaunchHostFunc(s, done_host, new DoneThunk{L.done, L.user, nullptr}));
    for (int32_t g : L.list) {
        c->din_issued[(size_t)g] = (uint8_t)stage;
        if (c->world > 1 && c->bnd_host[(size_t)g] >= 0) ++c->din_bnd_issued[stage];
    }
    c->din_count[stage] += (int64_t)m;
    if (stage == 3) c->din_done3 += (int64_t)m;
    if (L.stream_id >= c->din_streams.size()) c->din_streams.resize(L.stream_id + 1, 0);
    c->din_streams[L.stream_id] = 1;
    return TS_OK;
}

// The AMR barrier of stage k: the previous stage's reflux and this stage's
// proxy fill on the compute stream behind every stream the step used.
int amr_stage_barrier(ts_hydro_ctx* c, int stage) {
    cudaStream_t s0;
    int rc = ensure_stream(c, 0, &s0);
    if (rc) return rc;
    for (size_t id = 1; id < c->din_streams.size(); ++id) {
        if (!c->din_streams[id]) continue;
        TS_CUDA(c, cudaEventRecord(c->ev_in, c->streams[id]));
        TS_CUDA(c, cudaStreamWaitEvent(s0, c->ev_in, 0));
    }
    const double* dt_ptr = c->d_dt_hist + (c->steps_done % ts_hydro_ctx::kDtHist);
    if (c->amr_n_rec > 0 && stage > 1) {
        const tsh::StageArgs p = stage_args(c, stage - 1);
        unsigned long long* stamp = nullptr;
        if ((rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameAmrReflux, 0, 0, &stamp))) return rc;
        if (c->d_amr_rf_slot != nullptr)
            TS_CUDA(c, tsh::launch_amr_reflux_reg(p.Uout, c->nf, c->d_amr_level, c->amr_max_level, c->cfg.dx,
                                                  c->d_amr_rec, c->amr_n_rec, c->d_amr_rf_slot, c->d_amr_rf_flux,
                                                  stage - 1, dt_ptr, stamp, s0));
        else
            TS_CUDA(c, tsh::launch_amr_reflux(p.Uprev, p.Uout, c->nf, c->cfg.recon, c->cfg.gamma, c->cfg.p_floor,
                                              c->d_nbr, c->d_amr_level, c->amr_max_level, c->cfg.dx, c->d_amr_rec,
                                              c->amr_n_rec, stage - 1, dt_ptr, stamp, s0));
    }
    if (stage <= 3 && c->amr_n_proxy > 0) {
        const tsh::StageArgs a = stage_args(c, stage);
        unsigned long long* stamp = nullptr;
        if ((rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameAmrFill, 0, 0, &stamp))) return rc;
        TS_CUDA(c, tsh::launch_amr_fill(const_cast<double*>(a.Uprev), c->nf, c->d_amr_proxy,
                                        c->amr_slab_fill ? c->d_amr_pmask : nullptr, c->amr_n_proxy, stamp, s0));
    }
    if (stage <= 3) TS_CUDA(c, cudaEventRecord(c->ev_amr[stage], s0));
    return TS_OK;
}

// A drop-in launch on an AMR mesh: stage-ordered by the barrier events (no
// dataflow flags), every level in one launch (StageArgs::lvl_*), the flux
// register as the batched step's.
int dropin_issue_amr(ts_hydro_ctx* c, const ts_hydro_ctx::DropinLaunch& L, tsh::StageArgs a, cudaStream_t s) {
    const int stage = L.stage;
    int rc;
    if (stage == 1) {
        TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_din, 0));
        a.lead_g1 = 1;
        a.dt_out = c->d_dt_hist + (c->steps_done % ts_hydro_ctx::kDtHist);
    } else {
        if (!c->din_amr_barrier[stage]) {
            if ((rc = amr_stage_barrier(c, stage))) return rc;
            c->din_amr_barrier[stage] = true;
        }
        TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_amr[stage], 0));
    }
    if (c->d_amr_rf_slot != nullptr) {
        a.rf_slot = c->d_amr_rf_slot;
        a.rf_flux = c->d_amr_rf_flux;
    }
    a.lvl_n = c->amr_max_level + 1;
    for (int lv = 0; lv <= c->amr_max_level; ++lv) {
        a.lvl_first[lv] = (int)c->amr_level_first[(size_t)lv];
        a.lvl_dx[lv] = std::ldexp(c->cfg.dx, c->amr_max_level - lv);
    }
    a.dx_upd = a.lvl_dx[0];
    unsigned long long* stamp = nullptr;
    if ((rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameStage[stage], (int32_t)L.stream_id, L.guid, &stamp))) return rc;
    a.stamp = stamp;
    return dropin_launch_list(c, L, a, s);
}

int dropin_issue(ts_hydro_ctx* c, const ts_hydro_ctx::DropinLaunch& L) {
    cudaStream_t s;
    int rc = ensure_stream(c, L.stream_id, &s);
    if (rc) return rc;
    const int stage = L.stage;
    const size_t n = (size_t)c->n_owned;
    tsh::StageArgs a = stage_args(c, stage);
    a.amax_in = c->amax_src != nullptr ? c->amax_src : amax_slot(c, c->steps_done);
    a.amax_n = c->amax_src != nullptr ? c->amax_n : 1;
    a.amax_out = amax_slot(c, c->steps_done + 1);
    if (c->amr) return dropin_issue_amr(c, L, a, s);
    if (c->world > 1) {
        // fused P2P halos, as the batched step (do_step): boundary sub-grids
        // acquire the peers' slabs of U^(k-1) and push their own U^(k)
        const int out_idx = stage == 1 ? 1 : (stage == 2 ? 2 : 0);
        a.n_boundary = (int)c->boundary.size();
        a.bnd_of = c->d_bnd_of;
        a.push_tbl = c->d_push_tbl;
        a.push_out = c->d_push_out + (size_t)out_idx * c->world;
        a.halo_flag = c->d_halo_flag;
        a.halo_flag_n = c->world;
        a.halo_seq = c->din_xbase + (uint32_t)stage;
        a.halo_ctr = c->d_ctr + 1 + (int)(a.halo_seq % 3u);
        a.halo_target = c->din_halo_target[stage];
        if (stage > 1 || c->din_wait1) {
            a.halo_wait = reinterpret_cast<const unsigned int*>(c->d_flags);
            a.halo_wait_mask = c->halo_recv_mask;
            a.halo_wait_seq = a.halo_seq - 1u;
        }
    }
    a.flow_n = (int)c->n_owned;
    a.flow_seq = c->din_seq;
    a.flow_wait_seq = c->din_seq;
    a.flow_done = c->d_flow + (size_t)(stage - 1) * n;
    if (stage > 1) {
        a.flow_wait = c->d_flow + (size_t)(stage - 2) * n;
    } else {
        // everything on the compute stream before the step (upload, dt, a batched step)
        TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_din, 0));
        a.lead_g1 = 1;  // sub-grid 0's stage-1 CTA writes dt and zeroes the max slot two steps ahead
        a.dt_out = c->d_dt_hist + (c->steps_done % ts_hydro_ctx::kDtHist);
        a.amax_reset2 = amax_slot(c, c->steps_done + 2);
        if (c->din_chained) {
            // U^n of the sub-grid and its neighbours: the previous step's stage-3 flags;
            // dt: every sub-grid's stage-3 max (the count) before the z sweep
            a.flow_wait = c->d_flow + 2 * n;
            a.flow_wait_seq = c->din_seq - 1u;
            a.cnt_wait = c->d_cnt3;
            a.cnt_expect = c->cnt3_expect;
        }
    }
    if (stage == 3) a.cnt_done = c->d_cnt3;
    unsigned long long* stamp = nullptr;
    rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameStage[stage], (int32_t)L.stream_id, L.guid, &stamp);
    if (rc) return rc;
    a.stamp = stamp;
    a.list = nullptr;
    return dropin_launch_list(c, L, a, s);
}

// Issue every parked launch whose producers have been issued, until none is
// left ready.  Issue order then respects the dataflow, so a kernel spinning on
// a flag never blocks the stream its producer is queued on.
int dropin_pump(ts_hydro_ctx* c) {
    bool progress = true;
    while (progress && !c->din_parked.empty()) {
        progress = false;
        for (size_t k = 0; k < c->din_parked.size();) {
            if (!dropin_ready(c, c->din_parked[k])) {
                ++k;
                continue;
            }
            ts_hydro_ctx::DropinLaunch L = std::move(c->din_parked[k]);
            c->din_parked.erase(c->din_parked.begin() + (std::ptrdiff_t)k);
            const int rc = dropin_issue(c, L);
            if (rc) return rc;
            progress = true;
        }
    }
    return TS_OK;
}

// Entry points that replace or step the state: not while a drop-in step is
// open; afterwards the next drop-in step starts stream-ordered.
// Gravity launches on other streams read the state (and write d_grav): join
// them into the compute stream before anything there replaces or steps it.
int join_gravity(ts_hydro_ctx* c) {
#ifdef TS_NO_GRAVITY_JOIN  // diagnostic builds only: shows the ordering test catching the race
    return c == nullptr ? TS_EINVAL : TS_OK;
#endif
    cudaStream_t s0 = nullptr;
    for (size_t id = 1; id < c->grav_streams.size(); ++id) {
        if (!c->grav_streams[id]) continue;
        if (s0 == nullptr) {
            cudaSetDevice(c->dev);
            int rc = ensure_stream(c, 0, &s0);
            if (rc) return rc;
        }
        TS_CUDA(c, cudaEventRecord(c->ev_in, c->streams[id]));
        TS_CUDA(c, cudaStreamWaitEvent(s0, c->ev_in, 0));
        c->grav_streams[id] = 0;
    }
    return TS_OK;
}

int mutating(ts_hydro_ctx* c) {
    if (c->din_open)
        return fail(c, TS_ESTATE, "a per-sub-grid step is open (launch stage 3 of every sub-grid, then ts_hydro_finish_step)");
    if (int rc = join_gravity(c)) return rc;
    c->din_chained = false;
    c->halo_pushed = false;  // the proxies no longer hold the peers' last push of this state
    return TS_OK;
}

int check_state(ts_hydro_ctx* c) {
    int rc = guard(c);
    if (rc) return rc;
    if (c->host_only) return fail(c, TS_ESTATE, "host-only context (device_id = -1) cannot touch the GPU");
    if (!c->have_mesh) return fail(c, TS_ESTATE, "no mesh bound (call ts_hydro_set_mesh first)");
    return TS_OK;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

int ts_hydro_abi_version(void) { return TS_HYDRO_ABI_VERSION; }

void ts_hydro_default_config(ts_hydro_config* cfg) {
    if (cfg == nullptr) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->device_id = 0;
    cfg->stream_count = 128;
    cfg->activity_buffer_capacity = 1024;
    cfg->cells_per_edge = 8;
    cfg->n_species = 0;
    cfg->recon = TS_RECON_PPM;
    cfg->gamma = 1.4;
    cfg->cfl = 0.4;
    cfg->dx = 1.0 / 32.0;
    cfg->p_floor = 1e-12;
}

const char* ts_hydro_strerror(int code) {
    switch (code) {
        case TS_OK: return "ok";
        case TS_EINVAL: return "invalid argument";
        case TS_ESHUTDOWN: return "device is shut down";
        case TS_ECUDA: return "CUDA error";
        case TS_ENCCL: return "NCCL error";
        case TS_ENOMEM: return "out of device memory";
        case TS_ESTATE: return "call out of order";
        case TS_ECOMM: return "peer rank did not arrive";
    }
    return "unknown error";
}

uint64_t ts_hydro_clock_ns(void) { return steady_ns(); }

static int validate_config(const ts_hydro_config* cfg, std::string* why) {
    if (cfg->cells_per_edge != kN) {
        *why = "cells_per_edge must be 8 (the sub-grid size this path is built for)";
        return TS_EINVAL;
    }
    if (cfg->n_species < 0 || cfg->n_species > 5) {
        *why = "n_species must be in [0, 5]";
        return TS_EINVAL;
    }
    if (cfg->recon != TS_RECON_PPM && cfg->recon != TS_RECON_MINMOD) {
        *why = "unknown reconstruction";
        return TS_EINVAL;
    }
    if (!(cfg->gamma > 1.0) || !(cfg->cfl > 0.0) || !(cfg->dx > 0.0) || !(cfg->p_floor >= 0.0)) {
        *why = "gamma > 1, cfl > 0, dx > 0 and p_floor >= 0 are required";
        return TS_EINVAL;
    }
    if (cfg->stream_count < 2) {
        *why = "stream_count must be at least 2 (compute + halo)";
        return TS_EINVAL;
    }
    if (cfg->activity_buffer_capacity == 0) {
        *why = "activity_buffer_capacity must be positive";
        return TS_EINVAL;
    }
    return TS_OK;
}

int ts_hydro_create(const ts_hydro_config* cfg, ts_hydro_ctx** out) {
    if (cfg == nullptr || out == nullptr) return TS_EINVAL;
    *out = nullptr;
    std::string why;
    if (validate_config(cfg, &why) != TS_OK) {
        std::fprintf(stderr, "ts_hydro_create: %s\n", why.c_str());
        return TS_EINVAL;
    }
    auto* c = new (std::nothrow) ts_hydro_ctx();
    if (c == nullptr) return TS_ENOMEM;
    c->cfg = *cfg;
    c->nf = 6 + cfg->n_species;
    c->dev = cfg->device_id;
    if (const char* w = std::getenv("TS_HYDRO_HALO")) c->halo_fused = std::strcmp(w, "ce") != 0;
    if (const char* w = std::getenv("TS_HYDRO_FLOW")) c->flow = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_FLOW_STEPS")) c->flow_steps = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_MCHAIN")) c->mchain = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_FMM_MERGE")) c->fmm_merge = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_DT")) c->dt_kernel = std::strcmp(w, "kernel") == 0;
    if (const char* w = std::getenv("TS_HYDRO_CHUNK_OVERLAP")) c->chunk_overlap = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_H2D_GATE")) c->h2d_gate = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_E2E_WAVE")) c->e2e_wave = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_SCR_RING")) c->scr_ring = std::strcmp(w, "0") != 0;
    if (const char* w = std::getenv("TS_HYDRO_AMR_REFLUX")) c->amr_reflux_reg = std::strcmp(w, "recompute") != 0;
    if (const char* w = std::getenv("TS_HYDRO_AMR_SPLIT")) c->amr_fused = std::strcmp(w, "1") != 0;
    if (const char* w = std::getenv("TS_HYDRO_AMR_FULLFILL")) c->amr_slab_fill = std::strcmp(w, "1") != 0;
    if (const char* w = std::getenv("TS_HYDRO_XFER_CHUNKS"))
        c->xfer_chunks = std::max(1, std::min(ts_hydro_ctx::kXferChunksMax, std::atoi(w)));
    if (const char* w = std::getenv("TS_HYDRO_WAIT_TIMEOUT_MS")) c->wait_ns = 1000000ull * std::strtoull(w, nullptr, 10);
    if (cfg->device_id < 0) {
        c->host_only = true;
        *out = c;
        return TS_OK;
    }
    cudaError_t e = cudaSetDevice(c->dev);
    if (e != cudaSuccess) {
        std::fprintf(stderr, "ts_hydro_create: cudaSetDevice(%d): %s\n", c->dev, cudaGetErrorString(e));
        delete c;
        return TS_ECUDA;
    }
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->dev);
    c->streams.assign(cfg->stream_count, nullptr);
    int rc = TS_OK;
    if ((e = cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_red, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_bnd, cudaEventDisableTiming)) != cudaSuccess) {
        rc = cuda_fail(c, e, "cudaEventCreate");
    }
    if (!rc) rc = dalloc(c, &c->d_scal, 8);
    if (!rc) rc = dalloc(c, &c->d_dt_hist, ts_hydro_ctx::kDtHist);
    if (!rc) rc = dalloc(c, &c->d_stamps, (size_t)cfg->activity_buffer_capacity * 2);
    if (!rc && (e = cudaMemset(c->d_stamps, 0, (size_t)cfg->activity_buffer_capacity * 2 * 8)) != cudaSuccess)
        rc = cuda_fail(c, e, "cudaMemset");
    if (!rc && (e = cudaMemset(c->d_scal, 0, 8 * sizeof(double))) != cudaSuccess) rc = cuda_fail(c, e, "cudaMemset");
    if (!rc && (e = cudaDeviceSynchronize()) != cudaSuccess) rc = cuda_fail(c, e, "cudaDeviceSynchronize");
    if (!rc && (e = cudaHostAlloc((void**)&c->h_clock, 3 * sizeof(unsigned long long), cudaHostAllocMapped)) !=
                   cudaSuccess)
        rc = cuda_fail(c, e, "cudaHostAlloc");
    if (!rc) c->h_clock[1] = 0ull;
    if (!rc) rc = calibrate_clock(c);
    if (rc) {
        std::fprintf(stderr, "ts_hydro_create: %s\n", c->err.c_str());
        ts_hydro_destroy(c);
        return rc;
    }
    // creation-time records are bookkeeping of the context itself
    c->completed.clear();
    *out = c;
    return TS_OK;
}

const char* ts_hydro_last_error(const ts_hydro_ctx* ctx) { return ctx == nullptr ? "null context" : ctx->err.c_str(); }

int ts_hydro_num_fields(const ts_hydro_ctx* ctx) { return ctx == nullptr ? -1 : ctx->nf; }

int ts_hydro_shutdown(ts_hydro_ctx* ctx) {
    if (ctx == nullptr) return TS_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    if (ctx->shut) return TS_OK;
    if (ctx->host_only) {
        ctx->shut = true;
        return TS_OK;
    }
    cudaSetDevice(ctx->dev);
    int rc = sync_all(ctx);
    if (!rc) rc = harvest(ctx);
    deliver_to_sink(ctx);
    ctx->shut = true;
    return rc;
}

int ts_hydro_destroy(ts_hydro_ctx* ctx) {
    if (ctx == nullptr) return TS_EINVAL;
    if (ctx->host_only) {
        delete ctx;
        return TS_OK;
    }
    {
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        cudaSetDevice(ctx->dev);
        if (!ctx->shut) {
            sync_all(ctx);
            harvest(ctx);
            deliver_to_sink(ctx);
            ctx->shut = true;
        }
        close_peers(ctx);
        if (ctx->comm != nullptr && nccl().loaded) nccl().CommDestroy(ctx->comm);
        ctx->comm = nullptr;
        free_mesh(ctx);
        dfree(ctx, &ctx->d_scal);
        dfree(ctx, &ctx->d_check);
        dfree(ctx, &ctx->d_dt_hist);
        dfree(ctx, &ctx->d_stamps);
        for (auto& kv : ctx->host_allocs) cudaFreeHost(kv.first);
        ctx->host_allocs.clear();
        for (auto& kv : ctx->handles) cudaFree(kv.second.first);
        ctx->handles.clear();
        if (ctx->stage_dev) cudaFree(ctx->stage_dev);
        if (ctx->stage_host) cudaFreeHost(ctx->stage_host);
        if (ctx->h_clock) cudaFreeHost(ctx->h_clock);
        if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
        if (ctx->ev_cal) cudaEventDestroy(ctx->ev_cal);
        for (auto& row : ctx->ev_wave)
            for (cudaEvent_t e : row)
                if (e) cudaEventDestroy(e);
        if (ctx->ev_din) cudaEventDestroy(ctx->ev_din);
        for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
        for (const PendingLaunch& p : ctx->pending) {
            if (p.e0) cudaEventDestroy(p.e0);
            if (p.e1) cudaEventDestroy(p.e1);
        }
        if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
        if (ctx->ev_red) cudaEventDestroy(ctx->ev_red);
        if (ctx->ev_bnd) cudaEventDestroy(ctx->ev_bnd);
        for (cudaEvent_t& e : ctx->ev_d2h)
            if (e) cudaEventDestroy(e);
        if (ctx->ev_h2d) cudaEventDestroy(ctx->ev_h2d);
        if (ctx->ev_comp) cudaEventDestroy(ctx->ev_comp);
        for (cudaStream_t s : ctx->streams)
            if (s) cudaStreamDestroy(s);
    }
    delete ctx;
    return TS_OK;
}

int ts_hydro_uniform_mesh(int32_t nx, int32_t ny, int32_t nz, int32_t periodic_mask, int32_t world,
                          int64_t* nbr, int32_t* pos, int32_t* owner) {
    if (nx < 1 || ny < 1 || nz < 1 || world < 1 || nbr == nullptr || pos == nullptr || owner == nullptr)
        return TS_EINVAL;
    const int64_t n = (int64_t)nx * ny * nz;
    struct K {
        uint64_t key;
        int32_t x, y, z;
    };
    std::vector<K> keys;
    keys.reserve((size_t)n);
    // numbering: the Morton curve (build_mesh's order, workload.cpp:298-313),
    // or with TS_MESH_ROW_ORDER row-major, x fastest (make_row_mesh of the
    // reference's tests, test_workload.cpp:38-54)
    const bool row = (periodic_mask & TS_MESH_ROW_ORDER) != 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x)
                keys.push_back({row ? (uint64_t)(((int64_t)z * ny + y) * nx + x) : morton3((uint32_t)x, (uint32_t)y, (uint32_t)z),
                                x, y, z});
    std::sort(keys.begin(), keys.end(), [](const K& a, const K& b) { return a.key < b.key; });
    std::vector<int64_t> id_of((size_t)n);
    for (int64_t g = 0; g < n; ++g) {
        pos[3 * g] = keys[(size_t)g].x;
        pos[3 * g + 1] = keys[(size_t)g].y;
        pos[3 * g + 2] = keys[(size_t)g].z;
        id_of[(size_t)(((int64_t)keys[(size_t)g].z * ny + keys[(size_t)g].y) * nx + keys[(size_t)g].x)] = g;
    }
    const int dims[3] = {nx, ny, nz};
    for (int64_t g = 0; g < n; ++g)
        for (int face = 0; face < 6; ++face) {
            int cc[3] = {pos[3 * g], pos[3 * g + 1], pos[3 * g + 2]};
            const int axis = face / 2;
            cc[axis] += (face & 1) ? 1 : -1;
            int64_t nb = -1;
            if (cc[axis] < 0 || cc[axis] >= dims[axis]) {
                if (periodic_mask & (1 << axis)) {
                    cc[axis] = (cc[axis] + dims[axis]) % dims[axis];
                    nb = id_of[(size_t)(((int64_t)cc[2] * ny + cc[1]) * nx + cc[0])];
                }
            } else {
                nb = id_of[(size_t)(((int64_t)cc[2] * ny + cc[1]) * nx + cc[0])];
            }
            nbr[6 * g + face] = nb;
        }
    // contiguous Morton chunks, first `extra` ranks one larger (workload.cpp:314-323)
    const int64_t base = n / world, extra = n % world;
    int64_t cursor = 0;
    for (int r = 0; r < world; ++r) {
        const int64_t count = base + (r < extra ? 1 : 0);
        for (int64_t j = 0; j < count; ++j) owner[cursor++] = r;
    }
    return TS_OK;
}

static int bind_mesh(ts_hydro_ctx* c, const int64_t* nbr, const int32_t* owner, int32_t world);

int ts_hydro_set_mesh(ts_hydro_ctx* c, int64_t n, const int64_t* nbr, const int32_t* owner, int32_t world,
                      int32_t rank) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (n < 1 || nbr == nullptr || owner == nullptr) return fail(c, TS_EINVAL, "empty mesh");
    if (world < 1) return fail(c, TS_EINVAL, "mesh world_size must be positive");
    if (rank < 0 || rank >= world) return fail(c, TS_EINVAL, "rank outside the world");
    if (n > (int64_t)INT32_MAX / 2) return fail(c, TS_EINVAL, "too many sub-grids");
    // Mesh::validate (workload.cpp:140-168)
    for (int64_t i = 0; i < n; ++i) {
        const std::string where = "sub-grid " + std::to_string(i) + ": ";
        if (owner[i] < 0 || owner[i] >= world) return fail(c, TS_EINVAL, where + "owner outside the world");
        for (int f = 0; f < 6; ++f) {
            const int64_t nb = nbr[6 * i + f];
            if (nb == -1) continue;
            if (nb < 0 || nb >= n) return fail(c, TS_EINVAL, where + "neighbor id out of range");
            if (nb == i) return fail(c, TS_EINVAL, where + "sub-grid linked to itself");
            if (nbr[6 * nb + (f ^ 1)] != i) return fail(c, TS_EINVAL, where + "neighbor link is not symmetric");
        }
    }
    if (!c->host_only) {
        cudaSetDevice(c->dev);
        rc = sync_all(c);
        if (rc) return rc;
        free_mesh(c);
    }
    c->world = world;
    c->rank = rank;
    c->n_global = n;
    c->mesh_nbr.assign(nbr, nbr + 6 * n);
    c->mesh_owner.assign(owner, owner + n);
    c->owned_gid.clear();
    c->proxy_gid.clear();
    for (int64_t i = 0; i < n; ++i)
        if (owner[i] == rank) c->owned_gid.push_back(i);
    std::vector<char> is_proxy((size_t)n, 0);
    for (int64_t g : c->owned_gid)
        for (int f = 0; f < 6; ++f) {
            const int64_t nb = nbr[6 * g + f];
            if (nb >= 0 && owner[nb] != rank) is_proxy[(size_t)nb] = 1;
        }
    for (int64_t i = 0; i < n; ++i)
        if (is_proxy[(size_t)i]) c->proxy_gid.push_back(i);
    c->n_owned = (int64_t)c->owned_gid.size();
    c->n_proxy = (int64_t)c->proxy_gid.size();
    const int64_t nl = c->n_owned + c->n_proxy;
    c->nbr_local.assign((size_t)nl * 6, -1);
    c->interior.clear();
    c->boundary.clear();
    for (int64_t l = 0; l < c->n_owned; ++l) {
        const int64_t g = c->owned_gid[(size_t)l];
        bool foreign = false;
        for (int f = 0; f < 6; ++f) {
            const int64_t nb = nbr[6 * g + f];
            if (nb < 0) continue;
            c->nbr_local[(size_t)l * 6 + f] = (int32_t)local_of(c, nb);
            if (owner[nb] != rank) foreign = true;
        }
        (foreign ? c->boundary : c->interior).push_back((int32_t)l);
    }
    return bind_mesh(c, nbr, owner, world);
}

// Device side of a mesh whose owned / proxy lists, local neighbour table and
// interior / boundary lists are in place (ts_hydro_set_mesh, _set_amr_mesh).
// TMA descriptors of the three state buffers (used by TS_TMA kernel builds):
// a buffer as a 2-D tensor of 128-byte rows (16 doubles), rows = slots x nf x
// 32; one {16, 32} box = one 4 KiB field of one sub-grid, 128-byte swizzle.
// cuTensorMapEncodeTiled is resolved through the runtime (no link-time libcuda).
static int encode_tmaps(ts_hydro_ctx* c) {
    c->tmap_ok = false;
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode enc = nullptr;
    if (enc == nullptr) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
            return TS_OK;  // no TMA descriptors: TS_TMA builds trap, the default build never reads them
        enc = reinterpret_cast<Encode>(f);
    }
    const cuuint64_t rows = (cuuint64_t)(c->n_owned + c->n_proxy) * (cuuint64_t)c->nf * (kNC / 16);
    const cuuint64_t dims[2] = {16, rows};
    const cuuint64_t strides[1] = {16 * sizeof(double)};
    const cuuint32_t box[2] = {16, kNC / 16};
    const cuuint32_t estr[2] = {1, 1};
    for (int k = 0; k < 3; ++k)
        if (enc(&c->tmap[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, c->U[k], dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return fail(c, TS_ECUDA, "cuTensorMapEncodeTiled failed for a state buffer");
    c->tmap_ok = true;
    return TS_OK;
}

static int bind_mesh(ts_hydro_ctx* c, const int64_t* nbr, const int32_t* owner, int32_t world) {
    int rc = build_plans(c, nbr, owner);
    if (rc) return rc;
    const int64_t nl = c->n_owned + c->n_proxy;
    if (c->host_only) {
        c->have_mesh = true;
        return TS_OK;
    }
    const size_t elems = c->state_elems();
    for (auto& b : c->U) {
        rc = dalloc(c, &b, elems);
        if (rc) return rc;
        TS_CUDA(c, cudaMemset(b, 0, elems * sizeof(double)));
    }
    rc = encode_tmaps(c);
    if (!rc && c->d_check == nullptr) {
        rc = dalloc(c, &c->d_check, 5);
        if (!rc) TS_CUDA(c, cudaMemset(c->d_check, 0, 5 * sizeof(unsigned long long)));
    }
    if (!rc && c->nf > 6 && c->scr_ring) {
        rc = dalloc(c, &c->d_scr_ring, (size_t)256 * ts_hydro_ctx::kScrK * (c->nf - 6) * kNC);
        if (!rc) rc = dalloc(c, &c->d_scr_mask, 256);
        if (!rc) TS_CUDA(c, cudaMemset(c->d_scr_mask, 0, 256 * sizeof(unsigned int)));
    }
    if (!rc) rc = dalloc(c, &c->d_nbr, (size_t)nl * 6);
    if (!rc) rc = dalloc(c, &c->d_interior, c->interior.size());
    if (!rc) rc = dalloc(c, &c->d_boundary, c->boundary.size());
    if (!rc) rc = dalloc(c, &c->d_order, (size_t)c->n_owned);
    if (!rc) rc = dalloc(c, &c->d_flow, 3 * (size_t)c->n_owned);
    if (!rc) rc = dalloc(c, &c->d_cnt3, 1);
    if (!rc && std::getenv("TS_HYDRO_CTA_LOG") != nullptr) rc = dalloc(c, &c->d_cta_log, 12 * (size_t)c->n_owned);
    if (!rc) {
        c->flow_seq = 0;
        c->cnt3_expect = 0;
        c->flow_chain = false;
        TS_CUDA(c, cudaMemset(c->d_flow, 0, 3 * (size_t)c->n_owned * sizeof(uint32_t)));
        TS_CUDA(c, cudaMemset(c->d_cnt3, 0, sizeof(uint32_t)));
    }
    if (!rc) rc = dalloc(c, &c->d_bnd_of, (size_t)c->n_owned);
    if (!rc) rc = dalloc(c, &c->d_gid, (size_t)c->n_owned);
    if (rc) return rc;
    TS_CUDA(c, h2d_sync(c->d_nbr, c->nbr_local.data(), c->nbr_local.size() * sizeof(int32_t)));
    if (!c->interior.empty())
        TS_CUDA(c, h2d_sync(c->d_interior, c->interior.data(), c->interior.size() * sizeof(int32_t)));
    if (!c->boundary.empty())
        TS_CUDA(c, h2d_sync(c->d_boundary, c->boundary.data(), c->boundary.size() * sizeof(int32_t)));
    {
        // fused P2P launch order: boundary sub-grid b at position b * stride
        // (while interior ones remain).  Measured on 4 B200s (Sedov 16^3 per
        // GPU): stride 1 — every boundary sub-grid in the first wave — beats
        // spreading them (stride 4: -7 %); TS_HYDRO_BSTRIDE overrides.
        //
        // "onion" order (default; TS_HYDRO_ORDER=front for the above): the boundary sub-grids, then
        // breadth-first layers inward over local face links (Morton order
        // within a layer).  With the dataflow stages a boundary CTA of stage
        // k+1 waits for its local neighbours' stage k; in the front order
        // those are interior sub-grids anywhere in the launch, in the onion
        // order they are in the next layer, so the boundary CTAs — whose
        // slabs the peers wait for — are released early.
        int stride = 1;
        if (const char* e = std::getenv("TS_HYDRO_BSTRIDE")) stride = std::max(1, std::atoi(e));
        // measured on 4 B200s (Sedov 16^3 per GPU, same box): onion +1.5 % at
        // 2 GPUs (7.01 -> 7.13 G), +1.2 % at 4 (13.66 -> 13.82 G): the default
        bool onion = true;
        if (const char* e = std::getenv("TS_HYDRO_ORDER")) onion = std::strcmp(e, "front") != 0;
        std::vector<int32_t> interior_order = c->interior;
        if (onion && !c->boundary.empty()) {
            std::vector<int32_t> layer((size_t)c->n_owned, -1);
            std::vector<int32_t> frontier;
            for (int32_t g : c->boundary) {
                layer[(size_t)g] = 0;
                frontier.push_back(g);
            }
            for (int32_t L = 1; !frontier.empty(); ++L) {
                std::vector<int32_t> next;
                for (int32_t g : frontier)
                    for (int f = 0; f < 6; ++f) {
                        const int32_t h = c->nbr_local[6 * (size_t)g + f];
                        if (h >= 0 && h < c->n_owned && layer[(size_t)h] < 0) {
                            layer[(size_t)h] = L;
                            next.push_back(h);
                        }
                    }
                frontier.swap(next);
            }
            std::stable_sort(interior_order.begin(), interior_order.end(), [&](int32_t a, int32_t b) {
                const int32_t la = layer[(size_t)a] < 0 ? INT32_MAX : layer[(size_t)a];
                const int32_t lb = layer[(size_t)b] < 0 ? INT32_MAX : layer[(size_t)b];
                return la < lb;
            });
        }
        std::vector<int32_t> order, bnd((size_t)c->n_owned, -1);
        size_t bi = 0, ii = 0;
        while (bi < c->boundary.size() || ii < c->interior.size()) {
            const bool take_b = bi < c->boundary.size() && (ii >= c->interior.size() || order.size() % stride == 0);
            if (take_b) {
                bnd[(size_t)c->boundary[bi]] = (int32_t)bi;
                order.push_back(c->boundary[bi++]);
            } else {
                order.push_back(interior_order[ii++]);
            }
        }
        TS_CUDA(c, h2d_sync(c->d_order, order.data(), order.size() * sizeof(int32_t)));
        TS_CUDA(c, h2d_sync(c->d_bnd_of, bnd.data(), bnd.size() * sizeof(int32_t)));
    }
    {
        std::vector<long long> gid(c->owned_gid.begin(), c->owned_gid.end());
        if (!gid.empty())
            TS_CUDA(c, h2d_sync(c->d_gid, gid.data(), gid.size() * sizeof(long long)));
    }
    if (world > 1) {
        std::vector<int2> se((size_t)c->n_send_total), re((size_t)c->n_recv_total);
        for (const Peer& p : c->peers) {
            for (int64_t k = 0; k < p.n_send; ++k)
                se[(size_t)(p.send_off + k)] = make_int2((int)local_of(c, p.send_pairs[(size_t)(2 * k)]),
                                                         (int)p.send_pairs[(size_t)(2 * k + 1)]);
            for (int64_t k = 0; k < p.n_recv; ++k)
                re[(size_t)(p.recv_off + k)] = make_int2((int)local_of(c, p.recv_pairs[(size_t)(2 * k)]),
                                                         (int)p.recv_pairs[(size_t)(2 * k + 1)]);
        }
        rc = dalloc(c, &c->d_send_entries, se.size());
        if (!rc) rc = dalloc(c, &c->d_recv_entries, re.size());
        if (!rc) rc = dalloc(c, &c->d_send, (size_t)c->n_send_total * c->nf * c->xfer_cells);
        // two halves: the P2P transport alternates them by exchange parity
        if (!rc) rc = dalloc(c, &c->d_recv, 2 * (size_t)c->n_recv_total * c->nf * c->xfer_cells);
        if (!rc) rc = dalloc(c, &c->d_flags, 2 * (size_t)world);
        if (!rc) rc = dalloc(c, &c->d_gather, 2 * (size_t)world);
        if (!rc) rc = dalloc(c, &c->d_ctr, 4);  // [0] dt push, [1..3] halo push by stage slot
        if (rc) return rc;
        TS_CUDA(c, cudaMemset(c->d_ctr, 0, 4 * sizeof(unsigned int)));
        c->done_cnt = 0;
        std::fill(std::begin(c->halo_cnt), std::end(c->halo_cnt), 0u);
        // fused push targets by boundary position: {peer rank, local index on the peer}
        std::vector<int2> tbl(c->boundary.size() * 6, make_int2(-1, -1));
        std::vector<int32_t> bpos((size_t)c->n_owned, -1);
        for (size_t b = 0; b < c->boundary.size(); ++b) bpos[(size_t)c->boundary[b]] = (int32_t)b;
        c->halo_recv_mask = 0;
        for (const Peer& p : c->peers) {
            if (p.n_recv > 0) c->halo_recv_mask |= 1ull << p.rank;
            if (c->amr_mr) continue;  // no fused push on the AMR path
            for (int64_t k = 0; k < p.n_send; ++k) {
                const int64_t l = local_of(c, p.send_pairs[(size_t)(2 * k)]);
                const int f = (int)p.send_pairs[(size_t)(2 * k + 1)];
                tbl[(size_t)bpos[(size_t)l] * 6 + f] = make_int2(p.rank, p.send_dst[(size_t)k]);
            }
        }
        if (!tbl.empty()) {
            rc = dalloc(c, &c->d_push_tbl, tbl.size());
            if (rc) return rc;
            TS_CUDA(c, h2d_sync(c->d_push_tbl, tbl.data(), tbl.size() * sizeof(int2)));
        }
        TS_CUDA(c, cudaMemset(c->d_flags, 0, 2 * (size_t)world * sizeof(int32_t)));
        TS_CUDA(c, cudaMemset(c->d_gather, 0, 2 * (size_t)world * sizeof(double)));
        if (!se.empty())
            TS_CUDA(c, h2d_sync(c->d_send_entries, se.data(), se.size() * sizeof(int2)));
        if (!re.empty())
            TS_CUDA(c, h2d_sync(c->d_recv_entries, re.data(), re.size() * sizeof(int2)));
    }
    // set-up copies ran on the legacy stream: fence them before any kernel
    TS_CUDA(c, cudaDeviceSynchronize());
    c->steps_done = 0;
    c->dt_valid = false;
    c->amax_src = nullptr;
    c->xseq = c->aseq = 0;
    c->have_mesh = true;
    return TS_OK;
}

static int amr_validate(ts_hydro_ctx* c, int64_t nl, const int64_t* nbr, const int32_t* level, int32_t max_level,
                        int64_t np, const ts_amr_proxy* px, int64_t nr, const ts_amr_reflux* rf,
                        std::vector<int64_t>& first) {
    int rc = TS_OK;
    if (nl < 1 || nbr == nullptr || level == nullptr) return fail(c, TS_EINVAL, "empty AMR mesh");
    if (np < 0 || nr < 0 || (np > 0 && px == nullptr) || (nr > 0 && rf == nullptr))
        return fail(c, TS_EINVAL, "AMR proxy / reflux tables missing");
    if (max_level < 0 || max_level > 30) return fail(c, TS_EINVAL, "max_level outside 0..30");
    if (nl + np > (int64_t)INT32_MAX / 2) return fail(c, TS_EINVAL, "too many sub-grids");
    const int64_t nt = nl + np;
    first.assign((size_t)max_level + 2, 0);
    for (int64_t i = 0; i < nl; ++i) {
        const std::string where = "leaf " + std::to_string(i) + ": ";
        if (level[i] < 0 || level[i] > max_level) return fail(c, TS_EINVAL, where + "level outside 0..max_level");
        if (i > 0 && level[i] < level[i - 1]) return fail(c, TS_EINVAL, where + "leaves are not level-major");
        for (int f = 0; f < 6; ++f) {
            const int64_t nb = nbr[6 * i + f];
            if (nb == -1) continue;
            if (nb < 0 || nb >= nt) return fail(c, TS_EINVAL, where + "neighbor id out of range");
            if (nb == i) return fail(c, TS_EINVAL, where + "sub-grid linked to itself");
            // same-level leaf links are symmetric (Mesh::validate, workload.cpp:156-161)
            if (nb < nl && nbr[6 * nb + (f ^ 1)] != i) return fail(c, TS_EINVAL, where + "leaf link is not symmetric");
        }
    }
    for (int L = 0; L <= max_level + 1; ++L)
        first[(size_t)L] = std::lower_bound(level, level + nl, L) - level;
    for (int64_t k = 0; k < np; ++k) {
        const ts_amr_proxy& r = px[k];
        const std::string where = "proxy " + std::to_string(k) + ": ";
        if (r.dst != nl + k) return fail(c, TS_EINVAL, where + "proxies must be numbered n_leaves + k");
        if (r.kind != 0 && r.kind != 1) return fail(c, TS_EINVAL, where + "kind must be 0 (prolong) or 1 (restrict)");
        if (r.octant < 0 || r.octant > 7) return fail(c, TS_EINVAL, where + "octant outside 0..7");
        for (int o = 0; o < (r.kind == 0 ? 1 : 8); ++o)
            if (r.src[o] < 0 || r.src[o] >= nl) return fail(c, TS_EINVAL, where + "source is not a leaf");
    }
    for (int64_t k = 0; k < nr; ++k) {
        const ts_amr_reflux& r = rf[k];
        const std::string where = "reflux record " + std::to_string(k) + ": ";
        if (r.coarse < 0 || r.coarse >= nl) return fail(c, TS_EINVAL, where + "coarse id is not a leaf");
        for (int f = 0; f < 6; ++f) {
            if (r.fine[f][0] < 0) continue;
            for (int q = 0; q < 4; ++q)
                if (r.fine[f][q] < 0 || r.fine[f][q] >= nl || level[r.fine[f][q]] != level[r.coarse] + 1)
                    return fail(c, TS_EINVAL, where + "fine ids must be leaves one level finer");
        }
    }
    return rc;
}

int ts_hydro_set_amr_mesh(ts_hydro_ctx* c, int64_t nl, const int64_t* nbr, const int32_t* level, int32_t max_level,
                          int64_t np, const ts_amr_proxy* px, int64_t nr, const ts_amr_reflux* rf) {
    static_assert(sizeof(ts_amr_proxy) == sizeof(tsh::AmrProxy), "proxy layout");
    static_assert(sizeof(ts_amr_reflux) == sizeof(tsh::AmrReflux), "reflux layout");
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    std::vector<int64_t> first;
    if ((rc = amr_validate(c, nl, nbr, level, max_level, np, px, nr, rf, first)) != TS_OK) return rc;
    const int64_t nt = nl + np;
    if (!c->host_only) {
        cudaSetDevice(c->dev);
        rc = sync_all(c);
        if (rc) return rc;
        free_mesh(c);
    }
    c->world = 1;
    c->rank = 0;
    c->n_global = nl;
    c->mesh_nbr.assign(nbr, nbr + 6 * nl);
    c->mesh_owner.assign((size_t)nl, 0);
    c->owned_gid.resize((size_t)nl);
    for (int64_t i = 0; i < nl; ++i) c->owned_gid[(size_t)i] = i;
    c->proxy_gid.resize((size_t)np);
    for (int64_t k = 0; k < np; ++k) c->proxy_gid[(size_t)k] = nl + k;
    c->n_owned = nl;
    c->n_proxy = np;
    c->nbr_local.assign((size_t)nt * 6, -1);
    for (int64_t i = 0; i < 6 * nl; ++i) c->nbr_local[(size_t)i] = (int32_t)nbr[i];
    c->interior.resize((size_t)nl);
    for (int64_t i = 0; i < nl; ++i) c->interior[(size_t)i] = (int32_t)i;
    c->boundary.clear();
    rc = bind_mesh(c, nullptr, nullptr, 1);
    if (rc) return rc;
    c->amr_max_level = max_level;
    c->amr_level_first = first;
    c->amr_n_proxy = np;
    c->amr_n_rec = nr;
    if (!c->host_only) {
        rc = dalloc(c, &c->d_amr_proxy, (size_t)std::max<int64_t>(np, 1));
        if (!rc) rc = dalloc(c, &c->d_amr_pmask, (size_t)std::max<int64_t>(np, 1));
        if (!rc) rc = dalloc(c, &c->d_amr_rec, (size_t)std::max<int64_t>(nr, 1));
        if (!rc) rc = dalloc(c, &c->d_amr_level, (size_t)nl);
        if (rc) return rc;
        if (np > 0) {
            TS_CUDA(c, h2d_sync(c->d_amr_proxy, px, (size_t)np * sizeof(tsh::AmrProxy)));
            // leaf g reads proxy p = nbr[g][f] through p's face f ^ 1
            std::vector<unsigned char> pm((size_t)np, 0);
            for (int64_t g = 0; g < nl; ++g)
                for (int f = 0; f < 6; ++f) {
                    const int64_t h = nbr[6 * g + f];
                    if (h >= nl) pm[(size_t)(h - nl)] |= (unsigned char)(1u << (f ^ 1));
                }
            TS_CUDA(c, h2d_sync(c->d_amr_pmask, pm.data(), (size_t)np));
        }
        if (nr > 0)
            TS_CUDA(c, h2d_sync(c->d_amr_rec, rf, (size_t)nr * sizeof(tsh::AmrReflux)));
        TS_CUDA(c, h2d_sync(c->d_amr_level, level, (size_t)nl * sizeof(int32_t)));
        if (nr > 0 && c->amr_reflux_reg) {
            // flux register: one slot per coarse-fine face side (the coarse
            // leaf's face, and the facing face of each of its 4 fine leaves)
            std::vector<int32_t> slot((size_t)nl * 6, -1);
            int32_t ns = 0;
            for (int64_t k = 0; k < nr; ++k)
                for (int f = 0; f < 6; ++f) {
                    if (rf[k].fine[f][0] < 0) continue;
                    slot[(size_t)rf[k].coarse * 6 + f] = ns++;
                    for (int q = 0; q < 4; ++q) {
                        int32_t& sf = slot[(size_t)rf[k].fine[f][q] * 6 + (f ^ 1)];
                        if (sf < 0) sf = ns++;
                    }
                }
            rc = dalloc(c, &c->d_amr_rf_slot, slot.size());
            if (!rc) rc = dalloc(c, &c->d_amr_rf_flux, (size_t)std::max(ns, 1) * c->nf * kN * kN);
            if (rc) return rc;
            TS_CUDA(c, h2d_sync(c->d_amr_rf_slot, slot.data(), slot.size() * sizeof(int32_t)));
        }
    }
    c->amr = true;
    return TS_OK;
}

// Multi-rank AMR.  Every rank derives, from the global leaf mesh and the
// owner of every leaf, what each rank reads: its owned leaves, the remote
// leaves it needs whole (same-level face neighbours of owned leaves, sources
// of the proxies it fills, the fine leaves of its reflux records), and the
// proxies it fills (those its owned leaves point at, and those through which
// a reflux fine leaf reads the coarse side).  Ghost leaves are refreshed
// whole before every stage (pack -> copy engine / NCCL -> unpack), then the
// proxies are filled from local data and the stage / reflux kernels run on
// the owned leaves exactly as on one rank.
namespace {
struct AmrNeeds {
    std::vector<int64_t> owned, ghosts, proxies;
};
AmrNeeds amr_needs(int64_t nl, const int64_t* nbr, const ts_amr_proxy* px, int64_t nr, const ts_amr_reflux* rf,
                   const int32_t* owner, int32_t r) {
    AmrNeeds n;
    std::set<int64_t> ghosts, proxies;
    for (int64_t g = 0; g < nl; ++g) {
        if (owner[g] != r) continue;
        n.owned.push_back(g);
        for (int f = 0; f < 6; ++f) {
            const int64_t h = nbr[6 * g + f];
            if (h < 0) continue;
            if (h >= nl) proxies.insert(h);
            else if (owner[h] != r) ghosts.insert(h);
        }
    }
    for (int64_t k = 0; k < nr; ++k) {
        const ts_amr_reflux& rec = rf[k];
        if (owner[rec.coarse] != r) continue;
        for (int f = 0; f < 6; ++f) {
            if (rec.fine[f][0] < 0) continue;
            for (int q = 0; q < 4; ++q) {
                const int64_t fl = rec.fine[f][q];
                if (owner[fl] != r) ghosts.insert(fl);
                const int64_t via = nbr[6 * fl + (f ^ 1)];  // the fine leaf's view of the coarse side
                if (via >= nl) proxies.insert(via);
            }
        }
    }
    for (int64_t p : proxies) {
        const ts_amr_proxy& q = px[p - nl];
        for (int o = 0; o < (q.kind == 0 ? 1 : 8); ++o)
            if (owner[q.src[o]] != r) ghosts.insert(q.src[o]);
    }
    n.ghosts.assign(ghosts.begin(), ghosts.end());
    n.proxies.assign(proxies.begin(), proxies.end());
    return n;
}
}  // namespace

int ts_hydro_set_amr_mesh_partitioned(ts_hydro_ctx* c, int64_t nl, const int64_t* nbr, const int32_t* level,
                                      int32_t max_level, int64_t np, const ts_amr_proxy* px, int64_t nr,
                                      const ts_amr_reflux* rf, const int32_t* owner, int32_t world, int32_t rank) {
    if (owner == nullptr || world == 1) return ts_hydro_set_amr_mesh(c, nl, nbr, level, max_level, np, px, nr, rf);
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return fail(c, TS_EINVAL, "bad world / rank");
    std::vector<int64_t> first_global;
    if ((rc = amr_validate(c, nl, nbr, level, max_level, np, px, nr, rf, first_global)) != TS_OK) return rc;
    for (int64_t g = 0; g < nl; ++g)
        if (owner[g] < 0 || owner[g] >= world) return fail(c, TS_EINVAL, "leaf " + std::to_string(g) + ": owner out of range");
    std::vector<AmrNeeds> need((size_t)world);
    for (int r = 0; r < world; ++r) need[(size_t)r] = amr_needs(nl, nbr, px, nr, rf, owner, r);
    const AmrNeeds& me = need[(size_t)rank];
    if (me.owned.empty()) return fail(c, TS_EINVAL, "a rank owns no leaf");
    if (!c->host_only) {
        cudaSetDevice(c->dev);
        rc = sync_all(c);
        if (rc) return rc;
        free_mesh(c);
    }
    const int64_t nt = nl + np;
    std::vector<int64_t> loc((size_t)nt, -1);
    int64_t k = 0;
    for (int64_t g : me.owned) loc[(size_t)g] = k++;
    for (int64_t g : me.ghosts) loc[(size_t)g] = k++;
    for (int64_t p : me.proxies) loc[(size_t)p] = k++;
    const int64_t n_owned = (int64_t)me.owned.size(), n_ghost = (int64_t)me.ghosts.size();
    const int64_t n_leaf_local = n_owned + n_ghost, n_local = k;
    c->world = world;
    c->rank = rank;
    c->n_global = nl;
    c->mesh_nbr.assign(nbr, nbr + 6 * nl);
    c->mesh_owner.assign(owner, owner + nl);
    c->owned_gid = me.owned;
    c->proxy_gid = me.ghosts;
    c->proxy_gid.insert(c->proxy_gid.end(), me.proxies.begin(), me.proxies.end());
    c->n_owned = n_owned;
    c->n_proxy = n_local - n_owned;
    c->nbr_local.assign((size_t)n_local * 6, -1);
    for (int64_t i = 0; i < n_leaf_local; ++i) {
        const int64_t g = i < n_owned ? me.owned[(size_t)i] : me.ghosts[(size_t)(i - n_owned)];
        for (int f = 0; f < 6; ++f) {
            const int64_t h = nbr[6 * g + f];
            const int64_t l = h >= 0 ? loc[(size_t)h] : -1;
            if (i < n_owned && h >= 0 && l < 0)
                return fail(c, TS_EINVAL, "internal: an owned leaf's neighbour is not local");
            c->nbr_local[(size_t)i * 6 + f] = (int32_t)l;
        }
    }
    c->interior.resize((size_t)n_owned);
    for (int64_t i = 0; i < n_owned; ++i) c->interior[(size_t)i] = (int32_t)i;
    c->boundary.clear();
    // halo plan: whole sub-grids, my owned leaves each peer holds as ghosts / my ghosts it owns
    std::vector<Peer> peers((size_t)world);
    for (int q = 0; q < world; ++q) {
        Peer& p = peers[(size_t)q];
        p.rank = q;
        if (q == rank) continue;
        for (int64_t g : need[(size_t)q].ghosts)
            if (owner[g] == rank) {
                p.send_pairs.push_back(g);
                p.send_pairs.push_back(6);
                p.send_dst.push_back(-1);
            }
        for (int64_t g : me.ghosts)
            if (owner[g] == q) {
                p.recv_pairs.push_back(g);
                p.recv_pairs.push_back(6);
            }
    }
    int64_t so = 0, ro = 0;
    for (Peer& p : peers) {
        p.n_send = (int64_t)p.send_pairs.size() / 2;
        p.n_recv = (int64_t)p.recv_pairs.size() / 2;
        p.send_off = so;
        p.recv_off = ro;
        so += p.n_send;
        ro += p.n_recv;
    }
    c->n_send_total = so;
    c->n_recv_total = ro;
    c->peers = std::move(peers);
    c->amr_mr = true;
    c->xfer_cells = kNC;
    rc = bind_mesh(c, nullptr, nullptr, world);
    if (rc) return rc;
    // local AMR tables: proxies, reflux records of owned coarse leaves, levels
    std::vector<tsh::AmrProxy> lpx;
    for (int64_t p : me.proxies) {
        const ts_amr_proxy& q = px[p - nl];
        tsh::AmrProxy r{};
        r.dst = (int)loc[(size_t)p];
        r.kind = q.kind;
        r.octant = q.octant;
        for (int o = 0; o < 8; ++o) r.src[o] = (q.kind == 0 && o > 0) ? -1 : (int)loc[(size_t)q.src[o]];
        lpx.push_back(r);
    }
    std::vector<tsh::AmrReflux> lrf;
    for (int64_t i = 0; i < nr; ++i) {
        if (owner[rf[i].coarse] != rank) continue;
        tsh::AmrReflux r{};
        r.coarse = (int)loc[(size_t)rf[i].coarse];
        for (int f = 0; f < 6; ++f)
            for (int q = 0; q < 4; ++q) r.fine[f][q] = rf[i].fine[f][0] < 0 ? -1 : (int)loc[(size_t)rf[i].fine[f][q]];
        lrf.push_back(r);
    }
    std::vector<int32_t> llev((size_t)n_leaf_local);
    for (int64_t i = 0; i < n_leaf_local; ++i)
        llev[(size_t)i] = level[i < n_owned ? me.owned[(size_t)i] : me.ghosts[(size_t)(i - n_owned)]];
    std::vector<int64_t> first((size_t)max_level + 2, 0);
    for (int L = 0; L <= max_level + 1; ++L)
        first[(size_t)L] = std::lower_bound(llev.begin(), llev.begin() + n_owned, L) - llev.begin();
    c->amr_max_level = max_level;
    c->amr_level_first = first;
    c->amr_proxy_first = n_leaf_local;  // proxies follow the ghost leaves
    c->amr_n_proxy = (int64_t)lpx.size();
    c->amr_n_rec = (int64_t)lrf.size();
    if (!c->host_only) {
        const int64_t npl = (int64_t)lpx.size(), nrl = (int64_t)lrf.size();
        rc = dalloc(c, &c->d_amr_proxy, (size_t)std::max<int64_t>(npl, 1));
        if (!rc) rc = dalloc(c, &c->d_amr_pmask, (size_t)std::max<int64_t>(npl, 1));
        if (!rc) rc = dalloc(c, &c->d_amr_rec, (size_t)std::max<int64_t>(nrl, 1));
        if (!rc) rc = dalloc(c, &c->d_amr_level, (size_t)n_leaf_local);
        if (rc) return rc;
        if (npl > 0) {
            TS_CUDA(c, h2d_sync(c->d_amr_proxy, lpx.data(), (size_t)npl * sizeof(tsh::AmrProxy)));
            // local leaf i reads proxy p = nbr_local[i][f] through p's face f ^ 1
            std::vector<unsigned char> pm((size_t)npl, 0);
            for (int64_t i = 0; i < n_leaf_local; ++i)
                for (int f = 0; f < 6; ++f) {
                    const int32_t h = c->nbr_local[(size_t)i * 6 + f];
                    if (h >= n_leaf_local) pm[(size_t)(h - n_leaf_local)] |= (unsigned char)(1u << (f ^ 1));
                }
            TS_CUDA(c, h2d_sync(c->d_amr_pmask, pm.data(), (size_t)npl));
        }
        if (nrl > 0)
            TS_CUDA(c, h2d_sync(c->d_amr_rec, lrf.data(), (size_t)nrl * sizeof(tsh::AmrReflux)));
        TS_CUDA(c, h2d_sync(c->d_amr_level, llev.data(), (size_t)n_leaf_local * sizeof(int32_t)));
    }
    c->amr = true;
    return TS_OK;
}

int ts_hydro_local_counts(const ts_hydro_ctx* c, int64_t* n_owned, int64_t* n_proxy, int64_t* n_interior) {
    if (c == nullptr) return TS_EINVAL;
    if (!c->have_mesh) return TS_ESTATE;
    if (n_owned) *n_owned = c->n_owned;
    if (n_proxy) *n_proxy = c->n_proxy;
    if (n_interior) *n_interior = (int64_t)c->interior.size();
    return TS_OK;
}

int ts_hydro_owned_ids(const ts_hydro_ctx* c, int64_t* ids) {
    if (c == nullptr || ids == nullptr) return TS_EINVAL;
    if (!c->have_mesh) return TS_ESTATE;
    std::copy(c->owned_gid.begin(), c->owned_gid.end(), ids);
    return TS_OK;
}

int ts_hydro_halo_plan(const ts_hydro_ctx* c, int32_t peer, int64_t* n_send, int64_t* send_pairs,
                       int64_t* n_recv, int64_t* recv_pairs) {
    if (c == nullptr) return TS_EINVAL;
    if (!c->have_mesh) return TS_ESTATE;
    if (peer < 0 || peer >= c->world) return TS_EINVAL;
    if (c->world <= 1 || peer == c->rank) {
        if (n_send) *n_send = 0;
        if (n_recv) *n_recv = 0;
        return TS_OK;
    }
    const Peer& p = c->peers[(size_t)peer];
    if (n_send) *n_send = p.n_send;
    if (n_recv) *n_recv = p.n_recv;
    if (send_pairs) std::copy(p.send_pairs.begin(), p.send_pairs.end(), send_pairs);
    if (recv_pairs) std::copy(p.recv_pairs.begin(), p.recv_pairs.end(), recv_pairs);
    return TS_OK;
}

int ts_hydro_upload(ts_hydro_ctx* c, int64_t first, int64_t count, const double* host) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (first < 0 || count < 0 || first + count > c->n_owned || (count > 0 && host == nullptr))
        return fail(c, TS_EINVAL, "upload range outside the owned sub-grids");
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    const size_t per = (size_t)c->nf * kNC;
    const uint64_t t0 = steady_ns();
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    // pageable cudaMemcpy may return before its DMA lands: copy on our stream and wait
    TS_CUDA(c, cudaMemcpyAsync(c->U[0] + (size_t)first * per, host, (size_t)count * per * sizeof(double),
                               cudaMemcpyHostToDevice, s));
    TS_CUDA(c, cudaStreamSynchronize(s));
    record_copy(c, TS_ACTIVITY_COPY_H2D, (uint64_t)count * per * sizeof(double), t0, steady_ns());
    c->dt_valid = false;
    return TS_OK;
}

int ts_hydro_download(ts_hydro_ctx* c, int64_t first, int64_t count, double* host) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (first < 0 || count < 0 || first + count > c->n_owned || (count > 0 && host == nullptr))
        return fail(c, TS_EINVAL, "download range outside the owned sub-grids");
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    const size_t per = (size_t)c->nf * kNC;
    const uint64_t t0 = steady_ns();
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    TS_CUDA(c, cudaMemcpyAsync(host, c->U[0] + (size_t)first * per, (size_t)count * per * sizeof(double),
                               cudaMemcpyDeviceToHost, s));
    TS_CUDA(c, cudaStreamSynchronize(s));
    record_copy(c, TS_ACTIVITY_COPY_D2H, (uint64_t)count * per * sizeof(double), t0, steady_ns());
    return TS_OK;
}

int ts_hydro_download_buffer(ts_hydro_ctx* c, int32_t which, int64_t first, int64_t count, double* host) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (which < 0 || which > 2) return fail(c, TS_EINVAL, "buffer must be 0, 1 or 2");
    if (first < 0 || count < 0 || first + count > c->n_owned + c->n_proxy || (count > 0 && host == nullptr))
        return fail(c, TS_EINVAL, "download range outside the local sub-grids");
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    const size_t per = (size_t)c->nf * kNC;
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    TS_CUDA(c, cudaMemcpyAsync(host, c->U[which] + (size_t)first * per, (size_t)count * per * sizeof(double),
                               cudaMemcpyDeviceToHost, s));
    TS_CUDA(c, cudaStreamSynchronize(s));
    return TS_OK;
}

int ts_hydro_init_random(ts_hydro_ctx* c, uint64_t seed) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    c->launches++;
    TS_CUDA(c, tsh::launch_init_random(c->U[0], c->nf, c->d_gid, c->n_owned, seed, c->cfg.gamma, c->sms, s));
    TS_CUDA(c, cudaStreamSynchronize(s));
    c->dt_valid = false;
    return TS_OK;
}

int ts_hydro_compute_dt(ts_hydro_ctx* c, double* dt_out) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    cudaSetDevice(c->dev);
    rc = do_compute_dt(c);
    if (rc) return rc;
    if (dt_out != nullptr) {
        cudaStream_t s = c->streams[0];
        const double* src = c->amax_src != nullptr ? c->amax_src : amax_slot(c, c->steps_done);
        std::vector<double> v((size_t)(c->amax_src != nullptr ? c->amax_n : 1));
        TS_CUDA(c, cudaMemcpyAsync(v.data(), src, v.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        TS_CUDA(c, cudaStreamSynchronize(s));
        double amax = v[0];
        for (double x : v) amax = std::fmax(amax, x);
        *dt_out = (c->cfg.cfl * c->cfg.dx) / amax;
    }
    return TS_OK;
}

int ts_hydro_step(ts_hydro_ctx* c, uint64_t nsteps) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    c->halo_pushed = false;  // a call starts from a copy-engine halo refresh (collective on every rank)
    cudaSetDevice(c->dev);
    if (c->world > 1 && c->comm == nullptr && !c->p2p)
        return fail(c, TS_ESTATE, "multi-rank mesh needs ts_hydro_comm_init or ts_hydro_p2p_import before stepping");
    if (!c->dt_valid) {
        rc = do_compute_dt(c);
        if (rc) return rc;
    }
    for (uint64_t k = 0; k < nsteps; ++k) {
        rc = do_step(c);
        if (rc) return rc;
    }
    return TS_OK;
}

int ts_hydro_step_host(ts_hydro_ctx* c, const double* host_in, double* host_out, uint64_t nsteps) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (host_in == nullptr || host_out == nullptr) return fail(c, TS_EINVAL, "null host buffer");
    c->halo_pushed = false;  // a call starts from a copy-engine halo refresh (collective on every rank)
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    const size_t bytes = (size_t)c->n_owned * c->nf * kNC * sizeof(double);
    TS_CUDA(c, cudaMemcpyAsync(c->U[0], host_in, bytes, cudaMemcpyHostToDevice, s));
    rc = do_compute_dt(c);
    if (rc) return rc;
    for (uint64_t k = 0; k < nsteps; ++k) {
        rc = do_step(c);
        if (rc) return rc;
    }
    TS_CUDA(c, cudaMemcpyAsync(host_out, c->U[0], bytes, cudaMemcpyDeviceToHost, s));
    TS_CUDA(c, cudaStreamSynchronize(s));
    return TS_OK;
}


// Pipelined host-buffer steps.  Copies run in xfer_chunks sub-grid ranges on
// their own streams (H2D 3, D2H 4), so that when a call's input is the
// previous call's output (a chained simulation through host memory) the H2D of
// chunk i starts as soon as the previous call's D2H of chunk i landed, and the
// two PCIe directions run concurrently.  Ordering: H2D chunk i waits for the
// previous call's D2H of chunk i (or of everything when the call is not
// chained: that D2H still reads U^n) and for the compute stream's earlier work; the steps wait for
// the whole H2D (dt needs every sub-grid); the D2H waits for the steps.
namespace {
// One chained pipelined step as a wavefront over the transfer chunks: chunk i
// of the H2D, of each stage and of the D2H is its own operation; stage k of
// chunk i waits (CUDA events, no spinning) for stage k-1 of the chunks its
// sub-grids' face neighbours live in, stage 1 additionally for the H2D of
// those chunks and for every stage-3 chunk of the previous step (its dt), the
// D2H of chunk i for stage 3 of chunk i.  So the H2D of the next step's chunk
// i (behind this step's D2H of chunk i) overlaps this step's D2H of later
// chunks and the two PCIe directions stay busy together.  Hazards: stage k
// overwrites a buffer only after its readers (stage k+1 of the previous step,
// stage 1 of the halo chunks for U^n) — all behind the previous step's
// stage-3 events or this step's neighbour events.
int step_host_wave(ts_hydro_ctx* c, const double* host_in, double* host_out, ts_done_fn done, void* user) {
    const int C = c->xfer_chunks;
    const int64_t n = c->n_owned;
    const size_t per = (size_t)c->nf * kNC * sizeof(double);
    auto g0 = [&](int i) { return (n * i + C - 1) / C; };
    if (!c->wave_ready) {
        for (auto& row : c->ev_wave)
            for (int i = 0; i < C; ++i)
                if (row[i] == nullptr) TS_CUDA(c, cudaEventCreateWithFlags(&row[i], cudaEventDisableTiming));
        c->wave_dep.assign((size_t)C, {});
        for (int i = 0; i < C; ++i) {
            std::vector<char> d((size_t)C, 0);
            d[(size_t)i] = 1;
            for (int64_t g = g0(i); g < g0(i + 1); ++g)
                for (int f = 0; f < 6; ++f) {
                    const int32_t h = c->nbr_local[(size_t)g * 6 + f];
                    if (h >= 0 && h < n) d[(size_t)((h * C) / n)] = 1;
                }
            for (int j = 0; j < C; ++j)
                if (d[(size_t)j]) c->wave_dep[(size_t)i].push_back(j);
        }
        c->wave_ready = true;
    }
    cudaStream_t s0, sh, sd;
    int rc = ensure_stream(c, 0, &s0);
    if (!rc) rc = ensure_stream(c, 3, &sh);
    if (!rc) rc = ensure_stream(c, 4, &sd);
    if (rc) return rc;
    std::vector<cudaStream_t> cs((size_t)C);
    for (int i = 0; i < C; ++i) {
        rc = ensure_stream(c, 5 + (uint32_t)i, &cs[(size_t)i]);
        if (rc) return rc;
    }
    // earlier stream-0 work (a previous non-wavefront step), every stage-3
    // chunk of the previous step (this step's dt) and the zeroed max slot:
    // one event the stage-1 launches wait on
    for (int j = 0; j < C; ++j) TS_CUDA(c, cudaStreamWaitEvent(s0, c->ev_wave[3][j], 0));
    TS_CUDA(c, cudaMemsetAsync(amax_slot(c, c->steps_done + 1), 0, sizeof(double), s0));
    TS_CUDA(c, cudaEventRecord(c->ev_in, s0));
    // H2D by chunk, each behind the previous step's D2H of that chunk
    PendingLaunch* rec = nullptr;
    rc = begin_event_record(c, TS_ACTIVITY_COPY_H2D, kNameH2D, 3, (size_t)n * per, &rec);
    if (rc) return rc;
    cudaEvent_t h2d_e1 = rec != nullptr ? rec->e1 : nullptr;
    if (rec != nullptr) TS_CUDA(c, cudaEventRecord(rec->e0, sh));
    const char* in_b = reinterpret_cast<const char*>(host_in);
    for (int i = 0; i < C; ++i) {
        TS_CUDA(c, cudaStreamWaitEvent(sh, c->ev_d2h[i], 0));
        const size_t off = (size_t)g0(i) * per, len = (size_t)(g0(i + 1) - g0(i)) * per;
        if (len > 0)
            TS_CUDA(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->U[0]) + off, in_b + off, len, cudaMemcpyHostToDevice,
                                       sh));
        TS_CUDA(c, cudaEventRecord(c->ev_wave[0][i], sh));
    }
    if (h2d_e1 != nullptr) TS_CUDA(c, cudaEventRecord(h2d_e1, sh));
    // the three stages by chunk; one activity record per stage
    for (int stage = 1; stage <= 3; ++stage) {
        unsigned long long* stamp = nullptr;
        rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameStage[stage], 5, 0, &stamp);
        if (rc) return rc;
        c->launches += (uint64_t)C - 1;
        for (int i = 0; i < C; ++i) {
            cudaStream_t st = cs[(size_t)i];
            if (stage == 1) TS_CUDA(c, cudaStreamWaitEvent(st, c->ev_in, 0));
            for (int j : c->wave_dep[(size_t)i]) TS_CUDA(c, cudaStreamWaitEvent(st, c->ev_wave[stage - 1][j], 0));
            tsh::StageArgs a = stage_args(c, stage);
            a.stamp = stamp;
            a.first = (int)g0(i);
            if (stage == 1) a.dt_out = c->d_dt_hist + (c->steps_done % ts_hydro_ctx::kDtHist);
            const int cnt = (int)(g0(i + 1) - g0(i));
            if (cnt > 0) TS_CUDA(c, tsh::launch_stage(a, c->nf, c->cfg.recon, stage, cnt, st, false));
        }
        // record after all of this stage's launches: a chunk's next stage waits
        // for this stage of its neighbours, recorded above in host order
        for (int i = 0; i < C; ++i) TS_CUDA(c, cudaEventRecord(c->ev_wave[stage][i], cs[(size_t)i]));
    }
    // D2H by chunk, each behind stage 3 of its chunk
    rc = begin_event_record(c, TS_ACTIVITY_COPY_D2H, kNameD2H, 4, (size_t)n * per, &rec);
    if (rc) return rc;
    cudaEvent_t d2h_e1 = rec != nullptr ? rec->e1 : nullptr;
    if (rec != nullptr) TS_CUDA(c, cudaEventRecord(rec->e0, sd));
    char* out_b = reinterpret_cast<char*>(host_out);
    for (int i = 0; i < C; ++i) {
        TS_CUDA(c, cudaStreamWaitEvent(sd, c->ev_wave[3][i], 0));
        const size_t off = (size_t)g0(i) * per, len = (size_t)(g0(i + 1) - g0(i)) * per;
        if (len > 0)
            TS_CUDA(c, cudaMemcpyAsync(out_b + off, reinterpret_cast<const char*>(c->U[0]) + off, len,
                                       cudaMemcpyDeviceToHost, sd));
        TS_CUDA(c, cudaEventRecord(c->ev_d2h[i], sd));
    }
    if (d2h_e1 != nullptr) TS_CUDA(c, cudaEventRecord(d2h_e1, sd));
    if (done != nullptr) TS_CUDA(c, cudaLaunchHostFunc(sd, done_host, new DoneThunk{done, user, nullptr}));
    // later stream-0 work (downloads, batched steps) follows the whole step
    for (int i = 0; i < C; ++i) {
        TS_CUDA(c, cudaEventRecord(c->ev_in, cs[(size_t)i]));
        TS_CUDA(c, cudaStreamWaitEvent(s0, c->ev_in, 0));
    }
    c->prev_out = host_out;
    c->prev_out_bytes = (size_t)n * per;
    c->steps_done++;
    c->dt_valid = true;
    c->amax_src = nullptr;
    return TS_OK;
}
}  // namespace

int ts_hydro_step_host_async(ts_hydro_ctx* c, const double* host_in, double* host_out, uint64_t nsteps,
                             ts_done_fn done, void* user) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (host_in == nullptr || host_out == nullptr) return fail(c, TS_EINVAL, "null host buffer");
    if (c->cfg.stream_count < 5) return fail(c, TS_EINVAL, "pipelined host steps need stream_count >= 5");
    if (c->amr) return fail(c, TS_ESTATE, "pipelined host steps are not available on an AMR mesh (use ts_hydro_step_host)");
    cudaSetDevice(c->dev);
    cudaStream_t s, sh, sd;
    rc = ensure_stream(c, 0, &s);
    if (!rc) rc = ensure_stream(c, 3, &sh);
    if (!rc) rc = ensure_stream(c, 4, &sd);
    if (rc) return rc;
    if (c->ev_h2d == nullptr) {
        for (cudaEvent_t& e : c->ev_d2h) TS_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        TS_CUDA(c, cudaEventCreateWithFlags(&c->ev_h2d, cudaEventDisableTiming));
        TS_CUDA(c, cudaEventCreateWithFlags(&c->ev_comp, cudaEventDisableTiming));
    }
    c->halo_pushed = false;  // a call starts from a copy-engine halo refresh (collective on every rank)
    const int C = c->xfer_chunks;
    const size_t per = (size_t)c->nf * kNC * sizeof(double);
    const size_t bytes = (size_t)c->n_owned * per;
    auto chunk = [&](int i, size_t* off, size_t* len) {
        // sub-grid g belongs to chunk floor(g C / n), the stage kernel's rule
        const int64_t g0 = (c->n_owned * i + C - 1) / C, g1 = (c->n_owned * (i + 1) + C - 1) / C;
        *off = (size_t)g0 * per;
        *len = (size_t)(g1 - g0) * per;
    };
    const char* in_b = reinterpret_cast<const char*>(host_in);
    const bool chained = c->prev_out == host_in && c->prev_out_bytes == bytes;
    if (chained && c->e2e_wave && c->dt_valid && c->world == 1 && nsteps == 1 &&
        c->cfg.stream_count >= (uint32_t)(5 + C))
        return step_host_wave(c, host_in, host_out, done, user);
    // Chained on one rank: dt is the previous call's stage-3 signal speed (its
    // input is this call's input) and stage 1 starts under the H2D, each CTA
    // once the chunks of its sub-grid and neighbours landed.
    const bool gate = chained && c->h2d_gate && c->dt_valid && c->world == 1 && nsteps > 0 &&
                      memops().write32 != nullptr;
    if (gate && c->d_h2d_flag == nullptr) {
        rc = dalloc(c, &c->d_h2d_flag, (size_t)ts_hydro_ctx::kXferChunksMax);
        if (rc) return rc;
        TS_CUDA(c, cudaMemset(c->d_h2d_flag, 0, ts_hydro_ctx::kXferChunksMax * sizeof(uint32_t)));
        c->h2d_seq = 0;
    }
    // H2D: U^n may still be read by earlier work on the compute stream (when
    // chained, its readers are the previous call's stage-3 CTAs of the chunk,
    // which the chunk's D2H already waited for)
    if (!gate) {
        TS_CUDA(c, cudaEventRecord(c->ev_in, s));
        TS_CUDA(c, cudaStreamWaitEvent(sh, c->ev_in, 0));
    }
    if (gate) ++c->h2d_seq;
    // the previous call's D2H reads U^n: chunk-wise behind it when chained,
    // else behind all of it (an unrecorded event is a no-op wait)
    if (!chained) TS_CUDA(c, cudaStreamWaitEvent(sh, c->ev_d2h[C - 1], 0));
    PendingLaunch* rec = nullptr;
    rc = begin_event_record(c, TS_ACTIVITY_COPY_H2D, kNameH2D, 3, bytes, &rec);
    if (rc) return rc;
    cudaEvent_t h2d_e1 = rec != nullptr ? rec->e1 : nullptr;
    if (rec != nullptr) TS_CUDA(c, cudaEventRecord(rec->e0, sh));
    for (int i = 0; i < C; ++i) {
        size_t off, len;
        chunk(i, &off, &len);
        if (chained) TS_CUDA(c, cudaStreamWaitEvent(sh, c->ev_d2h[i], 0));
        if (len > 0)
            TS_CUDA(c, cudaMemcpyAsync(reinterpret_cast<char*>(c->U[0]) + off, in_b + off, len,
                                       cudaMemcpyHostToDevice, sh));
        if (gate && memops().write32(sh, (CUdeviceptr)(c->d_h2d_flag + i), c->h2d_seq,
                                     CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return fail(c, TS_ECUDA, "cuStreamWriteValue32 on an H2D chunk flag failed");
    }
    if (h2d_e1 != nullptr) TS_CUDA(c, cudaEventRecord(h2d_e1, sh));
    TS_CUDA(c, cudaEventRecord(c->ev_h2d, sh));
    // the steps
    if (!gate) TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_h2d, 0));
    // the last step's stage 3 counts finished sub-grids per chunk, and each
    // D2H chunk waits (stream memory op) for its count instead of the stage
    const bool fine = nsteps > 0 && memops().wait32 != nullptr && c->chunk_overlap;
    if (fine && c->d_chunk_ctr == nullptr) {
        rc = dalloc(c, &c->d_chunk_ctr, (size_t)ts_hydro_ctx::kXferChunksMax);
        if (rc) return rc;
        // zeroed before any D2H stream can test it
        TS_CUDA(c, cudaMemsetAsync(c->d_chunk_ctr, 0, ts_hydro_ctx::kXferChunksMax * sizeof(uint32_t), s));
        TS_CUDA(c, cudaStreamSynchronize(s));
        std::fill(std::begin(c->chunk_expect), std::end(c->chunk_expect), 0u);
    }
    if (gate) {
        c->h2d_arm = true;
    } else {
        rc = do_compute_dt(c);
        if (rc) return rc;
    }
    for (uint64_t k = 0; k < nsteps; ++k) {
        c->chunk_arm = fine && k + 1 == nsteps;
        rc = do_step(c);
        c->chunk_arm = false;
        if (rc) return rc;
    }
    c->h2d_arm = false;
    TS_CUDA(c, cudaEventRecord(c->ev_comp, s));
    // D2H
    if (!fine) TS_CUDA(c, cudaStreamWaitEvent(sd, c->ev_comp, 0));
    rc = begin_event_record(c, TS_ACTIVITY_COPY_D2H, kNameD2H, 4, bytes, &rec);
    if (rc) return rc;
    cudaEvent_t d2h_e1 = rec != nullptr ? rec->e1 : nullptr;
    if (rec != nullptr) TS_CUDA(c, cudaEventRecord(rec->e0, sd));
    char* out_b = reinterpret_cast<char*>(host_out);
    for (int i = 0; i < C; ++i) {
        size_t off, len;
        chunk(i, &off, &len);
        if (fine) {
            c->chunk_expect[i] += (uint32_t)(len / per);
            if (memops().wait32(sd, (CUdeviceptr)(c->d_chunk_ctr + i), c->chunk_expect[i], CU_STREAM_WAIT_VALUE_GEQ) !=
                CUDA_SUCCESS)
                return fail(c, TS_ECUDA, "cuStreamWaitValue32 on a chunk counter failed");
        }
        if (len > 0)
            TS_CUDA(c, cudaMemcpyAsync(out_b + off, reinterpret_cast<const char*>(c->U[0]) + off, len,
                                       cudaMemcpyDeviceToHost, sd));
        TS_CUDA(c, cudaEventRecord(c->ev_d2h[i], sd));
    }
    if (d2h_e1 != nullptr) TS_CUDA(c, cudaEventRecord(d2h_e1, sd));
    if (done != nullptr) TS_CUDA(c, cudaLaunchHostFunc(sd, done_host, new DoneThunk{done, user, nullptr}));
    c->prev_out = host_out;
    c->prev_out_bytes = bytes;
    return TS_OK;
}

int ts_hydro_time_steps(ts_hydro_ctx* c, uint64_t nsteps, double* ms) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (ms == nullptr) return fail(c, TS_EINVAL, "null output");
    if (c->world > 1 && c->comm == nullptr && !c->p2p)
        return fail(c, TS_ESTATE, "multi-rank mesh needs ts_hydro_comm_init or ts_hydro_p2p_import before stepping");
    c->halo_pushed = false;  // a call starts from a copy-engine halo refresh (collective on every rank)
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    if (!c->dt_valid) {
        rc = do_compute_dt(c);
        if (rc) return rc;
    }
    rc = device_barrier(c, s);
    if (rc) return rc;
    cudaEvent_t e0, e1;
    TS_CUDA(c, cudaEventCreate(&e0));
    TS_CUDA(c, cudaEventCreate(&e1));
    TS_CUDA(c, cudaEventRecord(e0, s));
    for (uint64_t k = 0; k < nsteps && rc == TS_OK; ++k) rc = do_step(c);
    cudaError_t e = cudaEventRecord(e1, s);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float f = 0.0f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&f, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(c, e, "event timing");
    *ms = (double)f;
    return TS_OK;
}

int ts_hydro_synchronize(ts_hydro_ctx* c) {
    if (c == nullptr) return TS_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (c->host_only) return TS_OK;
    cudaSetDevice(c->dev);
    return sync_all(c);
}

int ts_hydro_last_dt(ts_hydro_ctx* c, double* dt) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (dt == nullptr) return TS_EINVAL;
    if (c->steps_done == 0) return fail(c, TS_ESTATE, "no step taken yet");
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    TS_CUDA(c, cudaMemcpy(dt, c->d_dt_hist + ((c->steps_done - 1) % ts_hydro_ctx::kDtHist), sizeof(double),
                          cudaMemcpyDeviceToHost));
    return TS_OK;
}

int ts_hydro_steps_done(const ts_hydro_ctx* c, uint64_t* steps) {
    if (c == nullptr || steps == nullptr) return TS_EINVAL;
    *steps = c->steps_done;
    return TS_OK;
}

int ts_hydro_launch_count(const ts_hydro_ctx* c, uint64_t* launches) {
    if (c == nullptr || launches == nullptr) return TS_EINVAL;
    *launches = c->launches;
    return TS_OK;
}


int ts_hydro_launch_stage(ts_hydro_ctx* c, int32_t stage, const int64_t* owned_index, int64_t count,
                          uint32_t stream_id, uint64_t guid, ts_done_fn done, void* user) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (stage < 1 || stage > 3) return fail(c, TS_EINVAL, "stage must be 1, 2 or 3");
    if (count <= 0 || owned_index == nullptr) return fail(c, TS_EINVAL, "empty sub-grid list");
    if (stream_id >= c->cfg.stream_count) return fail(c, TS_EINVAL, "invalid stream id");
    if (c->world > 1 && !(c->p2p && c->halo_fused && c->d_push_tbl != nullptr))
        return fail(c, TS_ESTATE, "per-sub-grid launches on N ranks need the fused P2P transport (ts_hydro_p2p_import)");
    if (c->amr && (c->world > 1 || c->amr_max_level >= tsh::StageArgs::kMaxLevels))
        return fail(c, TS_ESTATE, "per-sub-grid launches on an AMR mesh: single rank, < 8 levels (use ts_hydro_step)");
    cudaSetDevice(c->dev);
    if (!c->din_open) {
        if (stage != 1) return fail(c, TS_ESTATE, "a per-sub-grid step starts with stage 1");
        rc = dropin_open(c);
        if (rc) return rc;
    }
    ts_hydro_ctx::DropinLaunch L{stage, std::vector<int32_t>((size_t)count), stream_id, guid, done, user};
    for (int64_t k = 0; k < count; ++k) {
        const int64_t g = owned_index[k];
        if (g < 0 || g >= c->n_owned) return fail(c, TS_EINVAL, "sub-grid index outside the owned range");
        if (c->din_req[(size_t)g] != stage - 1)
            return fail(c, TS_ESTATE, "sub-grid " + std::to_string(g) + ": stage " + std::to_string(stage) +
                                          " requested after stage " + std::to_string(c->din_req[(size_t)g]) +
                                          " of this step (stages run 1, 2, 3 once per step)");
        L.list[(size_t)k] = (int32_t)g;
    }
    for (int32_t g : L.list) c->din_req[(size_t)g] = (uint8_t)stage;
    c->din_parked.push_back(std::move(L));
    return dropin_pump(c);
}

// Gravity slice: near-field monopole P2P of the listed owned sub-grids
// (nullptr / count <= 0: all) on stream `stream_id`, after everything on the
// compute stream (a closed per-sub-grid step is joined into it).
int ts_hydro_gravity_p2p(ts_hydro_ctx* c, double G, int32_t radius, const int64_t* owned_index, int64_t count,
                         uint32_t stream_id, uint64_t guid, ts_done_fn done, void* user) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (radius < 1 || radius > tsh::kP2PRMax) return fail(c, TS_EINVAL, "P2P radius must be 1..6 cells");
    if (stream_id >= c->cfg.stream_count) return fail(c, TS_EINVAL, "invalid stream id");
    if (c->world > 1) return fail(c, TS_ESTATE, "the gravity slice is single-rank (halos deeper than 3 cells)");
    if (c->amr) return fail(c, TS_ESTATE, "the gravity slice needs a uniform mesh (same-level neighbours)");
    if (c->din_open) return fail(c, TS_ESTATE, "gravity reads the state: close the per-sub-grid step first");
    std::vector<int32_t> list;
    if (owned_index != nullptr && count > 0) {
        list.resize((size_t)count);
        for (int64_t k = 0; k < count; ++k) {
            if (owned_index[k] < 0 || owned_index[k] >= c->n_owned)
                return fail(c, TS_EINVAL, "sub-grid index outside the owned range");
            list[(size_t)k] = (int32_t)owned_index[k];
        }
    }
    cudaSetDevice(c->dev);
    if (c->d_grav == nullptr) {
        rc = dalloc(c, &c->d_grav, (size_t)c->n_owned * 4 * kNC);
        if (rc) return rc;
    }
    cudaStream_t s, s0;
    rc = ensure_stream(c, stream_id, &s);
    if (!rc) rc = ensure_stream(c, 0, &s0);
    if (rc) return rc;
    if (s != s0) {
        TS_CUDA(c, cudaEventRecord(c->ev_in, s0));
        TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_in, 0));
    }
    int off3[3 * 1024];
    double coef[4 * 1024];
    tsh::P2PArgs a{};
    a.U = c->U[0];
    a.nf = c->nf;
    a.nbr = c->d_nbr;
    a.out = c->d_grav;
    a.radius = radius;
    a.n_stencil = tsh::p2p_stencil_host(radius, off3, coef, 1024);
    a.kphi = -G * (c->cfg.dx * c->cfg.dx);
    a.kg = G * c->cfg.dx;
    unsigned long long* stamp = nullptr;
    rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameP2P, (int32_t)stream_id, guid, &stamp);
    if (rc) return rc;
    a.stamp = stamp;
    if (list.empty()) {
        a.first = 0;
        TS_CUDA(c, tsh::launch_p2p(a, (int)c->n_owned, s));
    } else if (list.size() <= (size_t)tsh::StageArgs::kInlineList) {
        a.list_inline_n = (int)list.size();
        for (size_t k = 0; k < list.size(); ++k) a.list_inline[k] = list[k];
        TS_CUDA(c, tsh::launch_p2p(a, (int)list.size(), s));
    } else {
        for (size_t k = 0; k < list.size();) {
            size_t e = k + 1;
            while (e < list.size() && list[e] == list[e - 1] + 1) ++e;
            a.first = list[k];
            TS_CUDA(c, tsh::launch_p2p(a, (int)(e - k), s));
            k = e;
        }
    }
    if (done != nullptr) TS_CUDA(c, cudaLaunchHostFunc(s, done_host, new DoneThunk{done, user, nullptr}));
    if (stream_id >= c->grav_streams.size()) c->grav_streams.resize(stream_id + 1, 0);
    c->grav_streams[stream_id] = 1;
    return TS_OK;
}

int ts_hydro_download_gravity(ts_hydro_ctx* c, int64_t first, int64_t count, double* host) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (host == nullptr || first < 0 || count < 0 || first + count > c->n_owned)
        return fail(c, TS_EINVAL, "range outside the owned sub-grids");
    if (c->d_grav == nullptr) return fail(c, TS_ESTATE, "no gravity computed yet (ts_hydro_gravity_p2p)");
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    TS_CUDA(c, cudaMemcpy(host, c->d_grav + (size_t)first * 4 * kNC, (size_t)count * 4 * kNC * sizeof(double),
                          cudaMemcpyDeviceToHost));
    return TS_OK;
}

// ---- gravity FMM (fmm.h, fmm_kernels.cu) ----------------------

namespace {
int fmm_table_dev(ts_hydro_ctx* c, int radius, bool root, bool far_only, const tsh::FmmEntry** tab, int* n);
}  // namespace

int ts_hydro_set_gravity_tree(ts_hydro_ctx* c, int64_t n_leaves, const int32_t* level, const int32_t* pos,
                              const int32_t* dims, double dx0) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (!c->have_mesh) return fail(c, TS_ESTATE, "no mesh bound (call ts_hydro_set_mesh first)");
    if (level == nullptr || pos == nullptr || dims == nullptr) return fail(c, TS_EINVAL, "null tree arrays");
    const bool multi = c->world > 1;
    if (multi) {
        if (c->comm == nullptr) return fail(c, TS_ESTATE, "gravity on N ranks gathers the densities over NCCL (ts_hydro_comm_init)");
        if (n_leaves != (int64_t)c->mesh_owner.size())
            return fail(c, TS_EINVAL, "on N ranks the tree's leaves are every rank's sub-grids, by global id");
    } else if (n_leaves != c->n_owned) {
        return fail(c, TS_EINVAL, "the tree's leaves must be exactly the owned sub-grids (n_leaves != n_owned)");
    }
    tsh::FmmTree t;
    const std::string err = tsh::fmm_build_tree(n_leaves, level, pos, dims, dx0, t);
    if (!err.empty()) return fail(c, TS_EINVAL, "gravity tree: " + err);
    // density row and output row of every leaf
    std::vector<int> row((size_t)n_leaves), out((size_t)n_leaves, -1);
    int64_t max_owned = c->n_owned;
    if (multi) {
        std::vector<int64_t> cnt((size_t)c->world, 0);
        std::vector<int64_t> idx((size_t)n_leaves);
        for (int64_t k = 0; k < n_leaves; ++k) idx[(size_t)k] = cnt[(size_t)c->mesh_owner[(size_t)k]]++;
        max_owned = *std::max_element(cnt.begin(), cnt.end());
        for (int64_t k = 0; k < n_leaves; ++k) {
            row[(size_t)k] = (int)(c->mesh_owner[(size_t)k] * max_owned + idx[(size_t)k]);
            if (c->mesh_owner[(size_t)k] == c->rank) {
                // owned sub-grids are stored in ascending global id: the owned index
                if (c->owned_gid[(size_t)idx[(size_t)k]] != k) return fail(c, TS_ESTATE, "owned ids out of order");
                out[(size_t)k] = (int)idx[(size_t)k];
            }
        }
    } else {
        for (int64_t k = 0; k < n_leaves; ++k) row[(size_t)k] = out[(size_t)k] = (int)k;
    }
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    dfree(c, &c->d_fmm_int);
    dfree(c, &c->d_fmm_M);
    dfree(c, &c->d_fmm_L);
    dfree(c, &c->d_fmm_lists);
    dfree(c, &c->d_fmm_send);
    dfree(c, &c->d_fmm_rho);
    c->have_fmm = false;
    const size_t n = (size_t)t.n();
    // SoA: depth | q (3n) | leaf row | parent | child (8n) | nb27 (27n) | leaf output row
    std::vector<int> h(n * 42);
    std::copy(t.depth.begin(), t.depth.end(), h.begin());
    std::copy(t.q.begin(), t.q.end(), h.begin() + (ptrdiff_t)n);
    for (size_t i = 0; i < n; ++i) {
        h[4 * n + i] = t.leaf[i] >= 0 ? row[(size_t)t.leaf[i]] : -1;
        h[41 * n + i] = t.leaf[i] >= 0 ? out[(size_t)t.leaf[i]] : -1;
    }
    std::copy(t.parent.begin(), t.parent.end(), h.begin() + (ptrdiff_t)(5 * n));
    std::copy(t.child.begin(), t.child.end(), h.begin() + (ptrdiff_t)(6 * n));
    std::copy(t.nb27.begin(), t.nb27.end(), h.begin() + (ptrdiff_t)(14 * n));
    // the leaves this rank evaluates, and the refined nodes on their paths to the root
    std::vector<int> lists;
    const std::vector<int>* ll[3] = {&t.leaves_p2p, &t.leaves_p2p_restr, &t.leaves_p2m};
    std::vector<uint8_t> need(n, multi ? 0 : 1);
    for (int k = 0; k < 3; ++k) {
        c->fmm_leaf_lists[k] = 0;
        for (int node : *ll[k]) {
            if (out[(size_t)t.leaf[(size_t)node]] < 0) continue;
            lists.push_back(node);
            ++c->fmm_leaf_lists[k];
            for (int p = t.parent[(size_t)node]; p >= 0 && !need[(size_t)p]; p = t.parent[(size_t)p]) need[(size_t)p] = 1;
        }
    }
    c->fmm_m2l_first.assign((size_t)t.max_depth + 1, 0);
    c->fmm_m2l_count.assign((size_t)t.max_depth + 1, 0);
    for (int d = 0; d < t.max_depth; ++d) {
        c->fmm_m2l_first[(size_t)d] = (int)lists.size();
        for (int i = t.int_first[(size_t)d]; i < t.int_first[(size_t)d] + t.n_int[(size_t)d]; ++i)
            if (need[(size_t)i]) lists.push_back(i);
        c->fmm_m2l_count[(size_t)d] = (int)lists.size() - c->fmm_m2l_first[(size_t)d];
    }
    if ((rc = dalloc(c, &c->d_fmm_int, h.size())) || (rc = dalloc(c, &c->d_fmm_M, n * 4 * kNC)) ||
        (rc = dalloc(c, &c->d_fmm_L, (size_t)std::max(t.n_internal, 1) * 10 * kNC)) ||
        (rc = dalloc(c, &c->d_fmm_lists, std::max<size_t>(lists.size(), 1))))
        return rc;
    if (multi && ((rc = dalloc(c, &c->d_fmm_send, (size_t)max_owned * kNC)) ||
                  (rc = dalloc(c, &c->d_fmm_rho, (size_t)c->world * max_owned * kNC))))
        return rc;
    c->fmm_max_owned = max_owned;
    if (c->d_fmm_part == nullptr && (rc = dalloc(c, &c->d_fmm_part, (size_t)tsh::kFmmSplitMax * 10 * kNC)))
        return rc;
    TS_CUDA(c, h2d_sync(c->d_fmm_int, h.data(), h.size() * sizeof(int)));
    if (!lists.empty())
        TS_CUDA(c, h2d_sync(c->d_fmm_lists, lists.data(), lists.size() * sizeof(int)));
    // every interaction table and the constant-bank coefficients now, then
    // wait: a pageable cudaMemcpy may return before its DMA lands, and the
    // solve's streams do not order behind the legacy stream
    for (int r = 1; r <= tsh::kFmmRMax; ++r)
        for (int o = 0; o < 2; ++o)
            for (int f = 0; f < 2; ++f) {
                const tsh::FmmEntry* tab;
                int nt;
                if ((rc = fmm_table_dev(c, r, o != 0, f != 0, &tab, &nt))) return rc;
            }
    TS_CUDA(c, tsh::fmm_prepare_device());
    TS_CUDA(c, cudaDeviceSynchronize());
    c->fmm = std::move(t);
    c->have_fmm = true;
    return TS_OK;
}

int ts_hydro_gravity_tree(int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                          int64_t cap, int32_t* level_out, int32_t* pos_out, int32_t* kind, int32_t* leaf,
                          int64_t* n_nodes) {
    if (level == nullptr || pos == nullptr || dims == nullptr) return TS_EINVAL;
    tsh::FmmTree t;
    if (!tsh::fmm_build_tree(n_leaves, level, pos, dims, 1.0, t).empty()) return TS_EINVAL;
    if (n_nodes != nullptr) *n_nodes = t.n();
    if (cap < t.n()) return TS_OK;
    for (int i = 0; i < t.n(); ++i) {
        if (level_out != nullptr) level_out[i] = t.depth[(size_t)i] - t.T;
        if (pos_out != nullptr)
            for (int a = 0; a < 3; ++a) pos_out[3 * i + a] = t.q[3 * (size_t)i + a];
        if (kind != nullptr) kind[i] = t.kind[(size_t)i];
        if (leaf != nullptr) leaf[i] = t.leaf[(size_t)i];
    }
    return TS_OK;
}

namespace {

int fmm_table_dev(ts_hydro_ctx* c, int radius, bool root, bool far_only, const tsh::FmmEntry** tab, int* n) {
    const int o = root ? 1 : 0, f = far_only ? 1 : 0;
    tsh::FmmEntry*& slot = c->d_fmm_tab[radius][o][f];
    if (slot == nullptr) {
        const std::vector<tsh::FmmEntry> v = tsh::fmm_table(radius, root, far_only);
        int rc = dalloc(c, &slot, v.size());
        if (rc) return rc;
        TS_CUDA(c, h2d_sync(slot, v.data(), v.size() * sizeof(tsh::FmmEntry)));
        c->n_fmm_tab[radius][o][f] = (int)v.size();
    }
    *tab = slot;
    *n = c->n_fmm_tab[radius][o][f];
    return TS_OK;
}

}  // namespace

int ts_hydro_gravity_fmm(ts_hydro_ctx* c, double G, int32_t radius, uint32_t stream_id, uint64_t guid,
                         ts_done_fn done, void* user) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (radius < 1 || radius > tsh::kFmmRMax) return fail(c, TS_EINVAL, "FMM radius must be 1..3 cells");
    if (stream_id >= c->cfg.stream_count) return fail(c, TS_EINVAL, "invalid stream id");
    if (!c->have_fmm) return fail(c, TS_ESTATE, "no gravity tree (call ts_hydro_set_gravity_tree first)");
    if (c->din_open) return fail(c, TS_ESTATE, "gravity reads the state: close the per-sub-grid step first");
    cudaSetDevice(c->dev);
    if (c->d_grav == nullptr) {
        rc = dalloc(c, &c->d_grav, (size_t)c->n_owned * 4 * kNC);
        if (rc) return rc;
    }
    cudaStream_t s, s0;
    rc = ensure_stream(c, stream_id, &s);
    if (!rc) rc = ensure_stream(c, 0, &s0);
    if (rc) return rc;
    if (s != s0) {
        TS_CUDA(c, cudaEventRecord(c->ev_in, s0));
        TS_CUDA(c, cudaStreamWaitEvent(s, c->ev_in, 0));
    }
    const tsh::FmmTree& t = c->fmm;
    const size_t n = (size_t)t.n();
    tsh::FmmArgs a{};
    a.U = c->U[0];
    a.nf = c->nf;
    if (c->world > 1) {
        // every rank's densities: field 0 of the owned sub-grids packed (a
        // strided 2-D copy), then an all-gather; rows owner * max_owned + i
        const size_t row_b = (size_t)kNC * sizeof(double);
        if (c->n_owned > 0)
            TS_CUDA(c, cudaMemcpy2DAsync(c->d_fmm_send, row_b, c->U[0], (size_t)c->nf * row_b, row_b,
                                         (size_t)c->n_owned, cudaMemcpyDeviceToDevice, s));
        TS_NCCL(c, nccl().AllGather(c->d_fmm_send, c->d_fmm_rho, (size_t)c->fmm_max_owned * kNC, ncclFloat64,
                                    c->comm, s));
        a.U = c->d_fmm_rho;
        a.nf = 1;
    }
    a.depth = c->d_fmm_int;
    a.q = c->d_fmm_int + n;
    a.leaf = c->d_fmm_int + 4 * n;
    a.parent = c->d_fmm_int + 5 * n;
    a.child = c->d_fmm_int + 6 * n;
    a.nb27 = c->d_fmm_int + 14 * n;
    a.leaf_out = c->d_fmm_int + 41 * n;
    a.M = c->d_fmm_M;
    a.L = c->d_fmm_L;
    a.part = c->d_fmm_part;
    a.out = c->d_grav;
    a.T = t.T;
    a.dx0 = t.dx0;
    a.G = G;
    auto launch = [&](const char* name, int n_ctas, auto&& fn) -> int {
        if (n_ctas <= 0) return TS_OK;
        unsigned long long* stamp = nullptr;
        int r = begin_launch(c, TS_ACTIVITY_KERNEL, name, (int32_t)stream_id, guid, &stamp);
        if (r) return r;
        a.stamp = stamp;
        TS_CUDA(c, fn(n_ctas));
        return TS_OK;
    };
    // P2M: every leaf's masses (the leaves follow the refined nodes)
    a.list = nullptr;
    a.first = t.n_internal;
    if ((rc = launch(kNameFmmMoments, (int)n - t.n_internal, [&](int k) { return tsh::launch_fmm_moments(a, k, s); })))
        return rc;
    // M2M, deepest refined depth first
    for (int d = t.max_depth - 1; d >= 0; --d) {
        a.first = t.int_first[(size_t)d];
        if ((rc = launch(d == 0 ? kNameMultipoleRoot : kNameMultipole, t.n_int[(size_t)d],
                         [&](int k) { return tsh::launch_fmm_restrict(a, k, s); })))
            return rc;
    }
    // L2L + M2L, root first.  The depths below the root share one table, so
    // the part sums of the root and of depths 1 .. merged_depth — the deepest
    // run of depths whose (node, chunk) rows fit the scratch together — are
    // ONE launch (the shallow depths' few CTAs no longer run as launches of
    // their own); their combines stay per depth, in order; deeper depths (a
    // tree too big for the scratch) keep the per-depth batches.
    int merged_rows = 0, merged_depth = 0;
    if (c->fmm_merge && t.max_depth > 2) {
        const tsh::FmmEntry* rt = nullptr;
        int n_rt = 0;
        if ((rc = fmm_table_dev(c, radius, true, true, &rt, &n_rt))) return rc;
        if ((rc = fmm_table_dev(c, radius, false, true, &a.table, &a.n_table))) return rc;
        const int n_chunks = (a.n_table + tsh::kFmmChunk - 1) / tsh::kFmmChunk;
        const int root_rows = c->fmm_m2l_count[0] * ((n_rt + tsh::kFmmChunk - 1) / tsh::kFmmChunk);
        int rows = 0;
        for (int d = 1; d < t.max_depth; ++d) {
            const int r = rows + c->fmm_m2l_count[(size_t)d] * n_chunks;
            if (r + root_rows > tsh::kFmmSplitMax) break;
            rows = r;
            merged_depth = d;
        }
        if (merged_depth >= 2 && rows > 0) {
            // the root's chunks ride in the same launch (its own table, rows after the deeper ones)
            merged_rows = rows;
            const int merged_nodes = rows / n_chunks;
            const int root_node = c->fmm_m2l_count[0] > 0 ? t.int_first[0] : -1;
            a.list = c->d_fmm_lists;
            a.first = c->fmm_m2l_first[1];
            a.part = c->d_fmm_part;
            if ((rc = launch(kNameMultipole, merged_nodes, [&](int k) {
                     return tsh::launch_fmm_m2l_part_flat(a, k, root_node, rt, n_rt, s);
                 })))
                return rc;
            a.list = nullptr;
        } else {
            merged_depth = 0;
        }
    }
    for (int d = 0; d < t.max_depth; ++d) {
        if (d == 0 && merged_depth > 0) {
            // the root's chunk sums (from the merged launch): combine only
            if ((rc = fmm_table_dev(c, radius, true, true, &a.table, &a.n_table))) return rc;
            a.list = c->d_fmm_lists;
            a.first = c->fmm_m2l_first[0];
            a.part = c->d_fmm_part + (size_t)merged_rows * 10 * kNC;
            if ((rc = launch(kNameMultipoleRoot, c->fmm_m2l_count[0],
                             [&](int k) { return tsh::launch_fmm_m2l_combine(a, k, s); })))
                return rc;
            a.part = c->d_fmm_part;
            a.list = nullptr;
            continue;
        }
        if (d > 0 && d <= merged_depth) {
            // this depth's chunk sums are rows (node index in the merged launch) * n_chunks onward
            if ((rc = fmm_table_dev(c, radius, false, true, &a.table, &a.n_table))) return rc;
            const int n_chunks = (a.n_table + tsh::kFmmChunk - 1) / tsh::kFmmChunk;
            const int nn = c->fmm_m2l_count[(size_t)d];
            a.list = c->d_fmm_lists;
            a.first = c->fmm_m2l_first[(size_t)d];
            a.part = c->d_fmm_part + (size_t)(a.first - c->fmm_m2l_first[1]) * n_chunks * 10 * kNC;
            if ((rc = launch(kNameMultipole, nn, [&](int k) { return tsh::launch_fmm_m2l_combine(a, k, s); })))
                return rc;
            a.part = c->d_fmm_part;
            a.list = nullptr;
            continue;
        }
        if ((rc = fmm_table_dev(c, radius, d == 0, true, &a.table, &a.n_table))) return rc;
        // each node's chunks spread over CTAs + an in-order combine, in
        // batches of nodes whose chunk sums fit the scratch (84 MB).  Measured
        // (Sedov 16^3, R = 2, depth 3's 512 nodes): 0.27 ms, against 0.37 for
        // one CTA per node walking its chunks and 0.35 for that with the
        // sources staged in 187 KB of shared memory
        // (the refined nodes on this rank's leaves' paths to the root: all of
        // them on one rank)
        const int n_chunks = (a.n_table + tsh::kFmmChunk - 1) / tsh::kFmmChunk;
        const int nn = c->fmm_m2l_count[(size_t)d];
        // (depths below the merged ones: the merged rows were consumed by
        // their combines, earlier on the stream, so the scratch is free again)
        const int batch = std::max(1, tsh::kFmmSplitMax / n_chunks);
        const int first = c->fmm_m2l_first[(size_t)d];
        a.list = c->d_fmm_lists;
        a.part = c->d_fmm_part;
        if ((rc = launch(d == 0 ? kNameMultipoleRoot : kNameMultipole, nn, [&](int k) {
                 cudaError_t e = cudaSuccess;
                 for (int b = 0; b < k && e == cudaSuccess; b += batch) {
                     a.first = first + b;
                     e = tsh::launch_fmm_m2l_split(a, std::min(batch, k - b), s);
                 }
                 return e;
             })))
            return rc;
        a.list = nullptr;
        a.part = c->d_fmm_part;
    }
    // leaves: the root alone, or the p2p / p2m lists
    if (t.root_leaf >= 0) {
        if ((rc = fmm_table_dev(c, radius, true, false, &a.table, &a.n_table))) return rc;
        a.K = tsh::kFmmRootK;
        a.first = t.root_leaf;
        if ((rc = launch(kNameMultipoleRoot, 1, [&](int k) { return tsh::launch_fmm_leaf(a, k, false, s); })))
            return rc;
    } else {
        if ((rc = fmm_table_dev(c, radius, false, false, &a.table, &a.n_table))) return rc;
        a.K = 2 * radius + 1;
        a.list = c->d_fmm_lists;
        a.first = 0;
        const int* nl = c->fmm_leaf_lists;
        if ((rc = launch(kNameP2P, nl[0], [&](int k) { return tsh::launch_fmm_leaf(a, k, false, s); }))) return rc;
        a.first = nl[0];
        if ((rc = launch(kNameP2P, nl[1], [&](int k) { return tsh::launch_fmm_leaf(a, k, true, s); }))) return rc;
        a.first += nl[1];
        if ((rc = launch(kNameP2M, nl[2], [&](int k) { return tsh::launch_fmm_leaf(a, k, true, s); }))) return rc;
    }
    if (done != nullptr) TS_CUDA(c, cudaLaunchHostFunc(s, done_host, new DoneThunk{done, user, nullptr}));
    if (stream_id >= c->grav_streams.size()) c->grav_streams.resize(stream_id + 1, 0);
    c->grav_streams[stream_id] = 1;
    return TS_OK;
}

namespace {

// The kick on the compute stream after everything before it; dt_dev: use the
// last step's dt from the device.  The state changed: the next step recomputes
// its signal speed (no stage-3 chaining across the kick).
int do_gravity_kick(ts_hydro_ctx* c, double dt, bool last_dt) {
    cudaStream_t s;
    int rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    unsigned long long* stamp = nullptr;
    rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameGravityKick, 0, 0, &stamp);
    if (rc) return rc;
    const double* dt_dev = last_dt ? c->d_dt_hist + ((c->steps_done - 1) % ts_hydro_ctx::kDtHist) : nullptr;
    TS_CUDA(c, tsh::launch_gravity_kick(c->U[0], c->nf, c->n_owned, c->d_grav, dt_dev, dt, stamp, c->sms, s));
    c->dt_valid = false;
    c->flow_chain = false;
    c->halo_pushed = false;
    return TS_OK;
}

}  // namespace

int ts_hydro_gravity_kick(ts_hydro_ctx* c, double dt) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (c->d_grav == nullptr) return fail(c, TS_ESTATE, "no gravity computed yet (ts_hydro_gravity_fmm / _p2p)");
    if (!(dt >= 0.0) && c->steps_done == 0) return fail(c, TS_ESTATE, "dt < 0 means the last step's dt: no step taken yet");
    cudaSetDevice(c->dev);
    return do_gravity_kick(c, dt, !(dt >= 0.0));
}

int ts_hydro_step_gravity(ts_hydro_ctx* c, uint64_t nsteps, double G, int32_t radius) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (!c->have_fmm) return fail(c, TS_ESTATE, "no gravity tree (call ts_hydro_set_gravity_tree first)");
    if (radius < 1 || radius > tsh::kFmmRMax) return fail(c, TS_EINVAL, "FMM radius must be 1..3 cells");
    cudaSetDevice(c->dev);
    for (uint64_t k = 0; k < nsteps; ++k) {
        if ((rc = ts_hydro_step(c, 1)) != TS_OK) return rc;
        if ((rc = ts_hydro_gravity_fmm(c, G, radius, 0, 0, nullptr, nullptr)) != TS_OK) return rc;
        if ((rc = do_gravity_kick(c, 0.0, true)) != TS_OK) return rc;
    }
    return TS_OK;
}

int ts_hydro_finish_step(ts_hydro_ctx* c) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    cudaSetDevice(c->dev);
    if (!c->din_open) return fail(c, TS_ESTATE, "no per-sub-grid step is open (ts_hydro_launch_stage stage 1 opens one)");
    if (c->din_done3 != c->n_owned || !c->din_parked.empty())
        return fail(c, TS_ESTATE, "finish_step before every owned sub-grid launched stage 3 (" +
                                      std::to_string(c->din_done3) + " of " + std::to_string(c->n_owned) + ")");
    // Join every stream the step used into the compute stream (no host wait):
    // later stream-0 work (downloads, batched steps, the next step's opening
    // event) is ordered after all of it.
    cudaStream_t s0;
    rc = ensure_stream(c, 0, &s0);
    if (rc) return rc;
    for (size_t id = 0; id < c->din_streams.size(); ++id) {
        if (!c->din_streams[id] || id == 0) continue;
        TS_CUDA(c, cudaEventRecord(c->ev_in, c->streams[id]));
        TS_CUDA(c, cudaStreamWaitEvent(s0, c->ev_in, 0));
    }
    if (c->amr) {
        // the last reflux, then the next dt's signal speed from the corrected
        // state (as the batched AMR step)
        if ((rc = amr_stage_barrier(c, 4))) return rc;
        double* slot = amax_slot(c, c->steps_done + 1);
        TS_CUDA(c, cudaMemsetAsync(slot, 0, sizeof(double), s0));
        unsigned long long* stamp = nullptr;
        if ((rc = begin_launch(c, TS_ACTIVITY_KERNEL, kNameSignal, 0, 0, &stamp))) return rc;
        TS_CUDA(c, tsh::launch_signal(c->U[0], c->nf, c->n_owned, c->cfg.gamma, c->cfg.p_floor, slot, stamp,
                                      c->sms, s0));
    }
    c->din_open = false;
    c->din_chained = c->world == 1 && !c->amr;
    c->cnt3_expect += (uint32_t)c->n_owned;  // every stage-3 CTA of the step counted into d_cnt3
    c->amax_src = nullptr;
    if (c->world > 1) {
        // the next dt: every rank's stage-3 max, gathered by the dt kernel
        // behind the step on the compute stream (as the batched step's)
        const uint32_t push_seq = c->aseq + 1;
        TS_CUDA(c, tsh::launch_dt_exchange(amax_slot(c, c->steps_done + 1),
                                           c->d_push_gather + (size_t)(push_seq & 1) * c->world, c->d_push_flag,
                                           c->world, c->rank, push_seq,
                                           reinterpret_cast<const unsigned int*>(c->d_flags + c->world),
                                           c->d_gather + (size_t)(push_seq & 1) * c->world, c->d_scal + 4,
                                           c->h_clock + 1, c->wait_ns, s0));
        c->launches++;
        c->aseq = push_seq;
        c->amax_src = c->d_scal + 4;
        c->amax_n = 1;
        c->xseq = c->din_xbase + 3u;
        c->halo_pushed = true;
    }
    c->steps_done++;
    c->dt_valid = true;  // the step's stage 3 reduced the next dt's signal speed on the device
    return TS_OK;
}

int ts_hydro_exchange_faces(ts_hydro_ctx* c, double* ghost_host) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (ghost_host == nullptr) return fail(c, TS_EINVAL, "null ghost buffer");
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    if (c->world > 1) {
        rc = ts_hydro_halo_exchange(c);
        if (rc) return rc;
    }
    double* d = nullptr;
    const size_t n = (size_t)c->n_owned * 6 * kN * kN;
    rc = dalloc(c, &d, n);
    if (rc) return rc;
    c->launches++;
    cudaError_t e = tsh::launch_face_exchange(c->U[0], c->nf, c->d_nbr, c->n_owned, d, c->sms, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ghost_host, d, n * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    dfree(c, &d);
    if (e != cudaSuccess) return cuda_fail(c, e, "face exchange");
    return TS_OK;
}

int ts_hydro_fill_halo(ts_hydro_ctx* c, int32_t depth, double* tiles_host) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (depth < 0 || depth > kN || tiles_host == nullptr) return fail(c, TS_EINVAL, "halo depth must be in [0, 8]");
    if (c->world > 1 && depth > 3) return fail(c, TS_EINVAL, "cross-rank halos are 3 deep");
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    if (c->world > 1) {
        rc = ts_hydro_halo_exchange(c);
        if (rc) return rc;
    }
    const size_t pe = (size_t)(kN + 2 * depth);
    const size_t n = (size_t)c->n_owned * c->nf * pe * pe * pe;
    double* d = nullptr;
    rc = dalloc(c, &d, n);
    if (rc) return rc;
    c->launches++;
    cudaError_t e = tsh::launch_fill_halo(c->U[0], c->nf, c->d_nbr, c->n_owned, depth, d, c->sms, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tiles_host, d, n * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    dfree(c, &d);
    if (e != cudaSuccess) return cuda_fail(c, e, "fill halo");
    return TS_OK;
}

int ts_hydro_nccl_unique_id(uint8_t id[128]) {
    if (id == nullptr) return TS_EINVAL;
    Nccl& n = nccl();
    if (!n.loaded) {
        std::fprintf(stderr, "ts_hydro_nccl_unique_id: %s\n", n.why.c_str());
        return TS_ENCCL;
    }
    ncclUniqueId u;
    if (n.GetUniqueId(&u) != ncclSuccess) return TS_ENCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return TS_OK;
}

int ts_hydro_comm_init(ts_hydro_ctx* c, const uint8_t id[128], int32_t nranks, int32_t rank) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (id == nullptr || nranks < 1 || rank < 0 || rank >= nranks) return fail(c, TS_EINVAL, "bad comm arguments");
    if (c->host_only) return fail(c, TS_ESTATE, "host-only context (device_id = -1) cannot touch the GPU");
    Nccl& n = nccl();
    if (!n.loaded) return fail(c, TS_ENCCL, n.why);
    cudaSetDevice(c->dev);
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (c->comm != nullptr) {
        n.CommDestroy(c->comm);
        c->comm = nullptr;
    }
    TS_NCCL(c, n.CommInitRank(&c->comm, nranks, u, rank));
    c->comm_size = nranks;
    return TS_OK;
}

int ts_hydro_selftest_math(ts_hydro_ctx* c, uint64_t n, uint64_t seed, int32_t emax, uint64_t* bad_rcp,
                           uint64_t* bad_sqrt) {
    int rc = guard(c);
    if (rc) return rc;
    if (c->host_only) return fail(c, TS_ESTATE, "host-only context (device_id = -1) cannot touch the GPU");
    if (bad_rcp == nullptr || bad_sqrt == nullptr || emax == 0 || emax > 1020 || emax < -1020)
        return fail(c, TS_EINVAL, "emax must be in [1, 1020] (or [-1020, -1]: near-one mantissas)");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    unsigned long long* d = nullptr;
    rc = dalloc(c, &d, 2);
    if (rc) return rc;
    unsigned long long h[2] = {0, 0};
    cudaError_t e = cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = tsh::launch_selftest_math(n, seed, emax, d, c->sms, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    dfree(c, &d);
    if (e != cudaSuccess) return cuda_fail(c, e, "selftest_math");
    *bad_rcp = h[0];
    *bad_sqrt = h[1];
    return TS_OK;
}

uint64_t ts_hydro_p2p_blob_size(void) { return sizeof(P2PBlob); }

int ts_hydro_p2p_export(ts_hydro_ctx* c, void* blob) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (blob == nullptr) return fail(c, TS_EINVAL, "null blob");
    if (c->world < 2) return fail(c, TS_ESTATE, "P2P transport needs a multi-rank mesh");
    if (c->world > kMaxRanks) return fail(c, TS_EINVAL, "too many ranks for the P2P transport");
    if (!memops().ok) return fail(c, TS_ECUDA, "stream memory operations unavailable");
    cudaSetDevice(c->dev);
    P2PBlob b{};
    b.magic = kBlobMagic;
    b.rank = c->rank;
    b.world = c->world;
    b.device = c->dev;
    TS_CUDA(c, cudaIpcGetMemHandle(&b.recv, c->d_recv));
    TS_CUDA(c, cudaIpcGetMemHandle(&b.flags, c->d_flags));
    TS_CUDA(c, cudaIpcGetMemHandle(&b.gather, c->d_gather));
    for (int k = 0; k < 3; ++k) TS_CUDA(c, cudaIpcGetMemHandle(&b.U[k], c->U[k]));
    b.n_recv_total = c->n_recv_total;
    for (const Peer& p : c->peers)
        if (p.rank >= 0 && p.rank < kMaxRanks) b.recv_off[p.rank] = p.recv_off;
    std::memcpy(blob, &b, sizeof(b));
    return TS_OK;
}

int ts_hydro_p2p_import(ts_hydro_ctx* c, const void* blobs, int32_t world) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (blobs == nullptr || world != c->world) return fail(c, TS_EINVAL, "need one blob per rank of the mesh");
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    close_peers(c);
    c->pm.assign((size_t)world, PeerMap{});
    const auto* all = static_cast<const P2PBlob*>(blobs);
    for (int r = 0; r < world; ++r) {
        const P2PBlob& b = all[r];
        if (b.magic != kBlobMagic || b.rank != r || b.world != world)
            return fail(c, TS_EINVAL, "malformed P2P blob for rank " + std::to_string(r));
        if (r == c->rank) continue;
        PeerMap& q = c->pm[(size_t)r];
        void* p = nullptr;
        TS_CUDA(c, cudaIpcOpenMemHandle(&p, b.recv, cudaIpcMemLazyEnablePeerAccess));
        q.recv = static_cast<double*>(p);
        TS_CUDA(c, cudaIpcOpenMemHandle(&p, b.flags, cudaIpcMemLazyEnablePeerAccess));
        q.flags = static_cast<int32_t*>(p);
        TS_CUDA(c, cudaIpcOpenMemHandle(&p, b.gather, cudaIpcMemLazyEnablePeerAccess));
        q.gather = static_cast<double*>(p);
        for (int k = 0; k < 3; ++k) {
            TS_CUDA(c, cudaIpcOpenMemHandle(&p, b.U[k], cudaIpcMemLazyEnablePeerAccess));
            q.U[k] = static_cast<double*>(p);
        }
        q.n_recv_total = b.n_recv_total;
        q.recv_off_for_me = b.recv_off[c->rank];
    }
    {
        std::vector<double*> pg(2 * (size_t)world);
        std::vector<unsigned int*> pf((size_t)world, nullptr);
        for (int h = 0; h < 2; ++h)
            for (int r = 0; r < world; ++r)
                pg[(size_t)h * world + r] =
                    (r == c->rank ? c->d_gather : c->pm[(size_t)r].gather) + (size_t)h * world;
        for (int r = 0; r < world; ++r)
            if (r != c->rank) pf[(size_t)r] = reinterpret_cast<unsigned int*>(c->pm[(size_t)r].flags + world + c->rank);
        std::vector<double*> po(3 * (size_t)world, nullptr);
        std::vector<unsigned int*> hf((size_t)world, nullptr);
        for (int r = 0; r < world; ++r) {
            if (r == c->rank) continue;
            for (int k = 0; k < 3; ++k) po[(size_t)k * world + r] = c->pm[(size_t)r].U[k];
            if (c->peers[(size_t)r].n_send > 0)
                hf[(size_t)r] = reinterpret_cast<unsigned int*>(c->pm[(size_t)r].flags + c->rank);
        }
        rc = dalloc(c, &c->d_push_gather, pg.size());
        if (!rc) rc = dalloc(c, &c->d_push_flag, pf.size());
        if (!rc) rc = dalloc(c, &c->d_push_out, po.size());
        if (!rc) rc = dalloc(c, &c->d_halo_flag, hf.size());
        if (rc) return rc;
        TS_CUDA(c, h2d_sync(c->d_push_out, po.data(), po.size() * sizeof(double*)));
        TS_CUDA(c, h2d_sync(c->d_halo_flag, hf.data(), hf.size() * sizeof(unsigned int*)));
        TS_CUDA(c, h2d_sync(c->d_push_gather, pg.data(), pg.size() * sizeof(double*)));
        TS_CUDA(c, h2d_sync(c->d_push_flag, pf.data(), pf.size() * sizeof(unsigned int*)));
        TS_CUDA(c, cudaDeviceSynchronize());
    }
    c->p2p = true;
    c->halo_pushed = false;
    return TS_OK;
}

int ts_hydro_halo_exchange(ts_hydro_ctx* c) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (c->world <= 1) return TS_OK;
    if (c->comm == nullptr && !c->p2p) return fail(c, TS_ESTATE, "no transport (ts_hydro_comm_init / ts_hydro_p2p_import)");
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, 0, &s);
    if (rc) return rc;
    rc = sync_all(c);
    if (rc) return rc;
    rc = exchange_on_comm(c, c->U[0]);
    if (rc) return rc;
    return sync_all(c);
}

int ts_hydro_set_activity_sink(ts_hydro_ctx* c, ts_activity_sink_fn sink, void* user) {
    if (c == nullptr) return TS_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->sink = sink;
    c->sink_user = user;
    return TS_OK;
}

int ts_hydro_debug_check(ts_hydro_ctx* c, uint64_t out[5], int32_t reset) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (out == nullptr) return fail(c, TS_EINVAL, "null output");
    for (int k = 0; k < 5; ++k) out[k] = 0;
    if (c->host_only || c->d_check == nullptr) return TS_OK;
    cudaSetDevice(c->dev);
    rc = sync_all(c);
    if (rc) return rc;
    TS_CUDA(c, cudaMemcpy(out, c->d_check, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (reset) TS_CUDA(c, cudaMemset(c->d_check, 0, 5 * sizeof(unsigned long long)));
    return TS_OK;
}

int ts_hydro_check_build(void) {
#if defined(TS_CHECK) && TS_CHECK
    return 1;
#else
    return 0;
#endif
}

int ts_hydro_set_profiling(ts_hydro_ctx* c, int32_t enabled) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->profiling = enabled != 0;
    return TS_OK;
}

int ts_hydro_flush_activity(ts_hydro_ctx* c, ts_activity_record* out, uint64_t cap, uint64_t* n_out) {
    if (c == nullptr || n_out == nullptr) return TS_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    int rc = TS_OK;
    if (!c->shut && !c->host_only) {
        cudaSetDevice(c->dev);
        rc = sync_all(c);
        if (!rc) rc = harvest(c);
        if (rc) return rc;
    }
    if (out == nullptr) {
        *n_out = c->completed.size();
        return TS_OK;
    }
    const uint64_t n = std::min<uint64_t>(cap, c->completed.size());
    std::copy(c->completed.begin(), c->completed.begin() + (ptrdiff_t)n, out);
    c->completed.erase(c->completed.begin(), c->completed.begin() + (ptrdiff_t)n);
    *n_out = n;
    return TS_OK;
}

int ts_hydro_memory_state(const ts_hydro_ctx* c, ts_memory_state* out) {
    if (c == nullptr || out == nullptr) return TS_EINVAL;
    *out = c->mem;
    return TS_OK;
}

int ts_hydro_host_alloc(ts_hydro_ctx* c, uint64_t bytes, void** ptr) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (bytes == 0 || ptr == nullptr) return fail(c, TS_EINVAL, "zero-byte allocation");
    if (c->host_only) return fail(c, TS_ESTATE, "host-only context (device_id = -1) cannot touch the GPU");
    cudaSetDevice(c->dev);
    void* p = nullptr;
    TS_CUDA(c, cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
    c->host_allocs[p] = bytes;
    c->mem.current_host_pinned_bytes += bytes;
    c->mem.peak_host_pinned_bytes = std::max(c->mem.peak_host_pinned_bytes, c->mem.current_host_pinned_bytes);
    *ptr = p;
    return TS_OK;
}

int ts_hydro_host_free(ts_hydro_ctx* c, void* ptr) {
    if (c == nullptr) return TS_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    auto it = c->host_allocs.find(ptr);
    if (it == c->host_allocs.end()) return fail(c, TS_EINVAL, "free of unknown or already-freed pinned handle");
    c->mem.current_host_pinned_bytes -= it->second;
    c->host_allocs.erase(it);
    cudaFreeHost(ptr);
    return TS_OK;
}

int ts_hydro_get_mesh(const ts_hydro_ctx* c, int64_t* n_grids, int64_t* nbr, int32_t* owner, int32_t* world,
                      int32_t* rank) {
    if (c == nullptr) return TS_EINVAL;
    if (!c->have_mesh) return TS_ESTATE;
    if (n_grids) *n_grids = c->n_global;
    if (nbr) std::copy(c->mesh_nbr.begin(), c->mesh_nbr.end(), nbr);
    if (owner) std::copy(c->mesh_owner.begin(), c->mesh_owner.end(), owner);
    if (world) *world = c->world;
    if (rank) *rank = c->rank;
    return TS_OK;
}

int ts_hydro_get_config(const ts_hydro_ctx* c, ts_hydro_config* out) {
    if (c == nullptr || out == nullptr) return TS_EINVAL;
    *out = c->cfg;
    return TS_OK;
}

int ts_hydro_save(ts_hydro_ctx* c, const char* path) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (path == nullptr) return fail(c, TS_EINVAL, "null checkpoint path");
    std::vector<double> st((size_t)c->n_owned * c->nf * kNC);
    rc = ts_hydro_download(c, 0, c->n_owned, st.data());
    if (rc) return rc;
    rc = ts_hydro_checkpoint_write(path, &c->cfg, c->n_global, c->mesh_nbr.data(), c->mesh_owner.data(), c->world,
                                   c->rank, c->n_owned, c->owned_gid.data(), st.data(), c->steps_done);
    if (rc) return fail(c, rc, std::string("cannot write checkpoint ") + path);
    return TS_OK;
}

int ts_hydro_restore(ts_hydro_ctx* c, const char* const* paths, int32_t n_paths) {
    int rc = check_state(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if ((rc = mutating(c)) != TS_OK) return rc;
    if (paths == nullptr || n_paths < 1) return fail(c, TS_EINVAL, "no checkpoint files");
    const size_t per = (size_t)c->nf * kNC;
    std::vector<double> st((size_t)c->n_owned * per);
    std::vector<char> have((size_t)c->n_owned, 0);
    int64_t found = 0;
    for (int32_t k = 0; k < n_paths; ++k) {
        const std::string name = paths[k] != nullptr ? paths[k] : "(null)";
        ts_hydro_checkpoint_header h{};
        if (paths[k] == nullptr || ts_hydro_checkpoint_info(paths[k], &h) != TS_OK)
            return fail(c, TS_EINVAL, "checkpoint " + name + ": unreadable, truncated or corrupt");
        if (h.nf != c->nf || h.recon != c->cfg.recon || h.gamma != c->cfg.gamma || h.cfl != c->cfg.cfl ||
            h.dx != c->cfg.dx || h.p_floor != c->cfg.p_floor)
            return fail(c, TS_EINVAL, "checkpoint " + name + ": numerics parameters differ from this context");
        if (h.n_grids != c->n_global) return fail(c, TS_EINVAL, "checkpoint " + name + ": mesh size differs");
        std::vector<int64_t> nbr((size_t)h.n_grids * 6), gid((size_t)h.n_records);
        std::vector<double> rec((size_t)h.n_records * per);
        if (ts_hydro_checkpoint_read(paths[k], nbr.data(), nullptr, gid.data(), rec.data()) != TS_OK)
            return fail(c, TS_EINVAL, "checkpoint " + name + ": read failed");
        if (nbr != c->mesh_nbr) return fail(c, TS_EINVAL, "checkpoint " + name + ": mesh links differ");
        for (int64_t r = 0; r < h.n_records; ++r) {
            auto it = std::lower_bound(c->owned_gid.begin(), c->owned_gid.end(), gid[(size_t)r]);
            if (it == c->owned_gid.end() || *it != gid[(size_t)r]) continue;  // another rank's sub-grid
            const size_t i = (size_t)(it - c->owned_gid.begin());
            if (!have[i]) ++found;
            have[i] = 1;
            std::copy(rec.begin() + (ptrdiff_t)((size_t)r * per), rec.begin() + (ptrdiff_t)((size_t)(r + 1) * per),
                      st.begin() + (ptrdiff_t)(i * per));
        }
    }
    if (found != c->n_owned)
        return fail(c, TS_EINVAL, "checkpoint does not cover every owned sub-grid (" + std::to_string(found) + " of " +
                                      std::to_string(c->n_owned) + ")");
    return ts_hydro_upload(c, 0, c->n_owned, st.data());
}

// ---- the rest of the SimDevice contract on the real device -----------------
int ts_hydro_launch_kernel(ts_hydro_ctx* c, const char* name, uint32_t stream_id, uint64_t duration_ns,
                           uint64_t guid, ts_done_fn done, void* user) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (c->host_only) return fail(c, TS_ESTATE, "host-only context (device_id = -1) cannot touch the GPU");
    if (duration_ns == 0) return fail(c, TS_EINVAL, "kernel duration must be positive");
    if (name == nullptr || *name == '\0') return fail(c, TS_EINVAL, "kernel name must be non-empty");
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, stream_id, &s);
    if (rc) return rc;
    const char* interned = c->names.insert(name).first->c_str();
    unsigned long long* stamp = nullptr;
    rc = begin_launch(c, TS_ACTIVITY_KERNEL, interned, (int32_t)stream_id, guid, &stamp);
    if (rc) return rc;
    TS_CUDA(c, tsh::launch_timed(duration_ns, stamp, s));
    if (done != nullptr) TS_CUDA(c, cudaLaunchHostFunc(s, done_host, new DoneThunk{done, user, nullptr}));
    return TS_OK;
}

int ts_hydro_enqueue_copy(ts_hydro_ctx* c, int32_t kind, uint64_t bytes, uint32_t stream_id, uint64_t guid,
                          ts_done_fn done, void* user) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (c->host_only) return fail(c, TS_ESTATE, "host-only context (device_id = -1) cannot touch the GPU");
    if (kind != TS_ACTIVITY_COPY_H2D && kind != TS_ACTIVITY_COPY_D2H && kind != TS_ACTIVITY_COPY_D2D)
        return fail(c, TS_EINVAL, "not a copy kind");
    if (bytes == 0) return fail(c, TS_EINVAL, "copy of zero bytes");
    cudaSetDevice(c->dev);
    cudaStream_t s;
    rc = ensure_stream(c, stream_id, &s);
    if (rc) return rc;
    const uint64_t dev_need = kind == TS_ACTIVITY_COPY_D2D ? 2 * bytes : bytes;
    const uint64_t host_need = kind == TS_ACTIVITY_COPY_D2D ? 0 : bytes;
    if (dev_need > c->stage_dev_bytes || host_need > c->stage_host_bytes) {
        // grow the staging buffers (in-flight copies may still use the old ones)
        rc = sync_all(c);
        if (rc) return rc;
        if (dev_need > c->stage_dev_bytes) {
            if (c->stage_dev) cudaFree(c->stage_dev);
            c->stage_dev = nullptr;
            c->stage_dev_bytes = 0;
            TS_CUDA(c, cudaMalloc(&c->stage_dev, dev_need));
            c->stage_dev_bytes = dev_need;
        }
        if (host_need > c->stage_host_bytes) {
            if (c->stage_host) cudaFreeHost(c->stage_host);
            c->stage_host = nullptr;
            c->stage_host_bytes = 0;
            TS_CUDA(c, cudaHostAlloc(&c->stage_host, host_need, cudaHostAllocDefault));
            c->stage_host_bytes = host_need;
        }
    }
    const char* name = kind == TS_ACTIVITY_COPY_H2D ? kNameH2D : (kind == TS_ACTIVITY_COPY_D2H ? kNameD2H : kNameD2D);
    unsigned long long* stamp = nullptr;
    rc = begin_launch(c, (uint8_t)kind, name, (int32_t)stream_id, guid, &stamp);
    if (rc) return rc;
    if (stamp != nullptr) c->pending.back().bytes = bytes;
    char* d = static_cast<char*>(c->stage_dev);
    TS_CUDA(c, tsh::launch_stamp(stamp, 0, s));
    if (kind == TS_ACTIVITY_COPY_H2D)
        TS_CUDA(c, cudaMemcpyAsync(d, c->stage_host, bytes, cudaMemcpyHostToDevice, s));
    else if (kind == TS_ACTIVITY_COPY_D2H)
        TS_CUDA(c, cudaMemcpyAsync(c->stage_host, d, bytes, cudaMemcpyDeviceToHost, s));
    else
        TS_CUDA(c, cudaMemcpyAsync(d + bytes, d, bytes, cudaMemcpyDeviceToDevice, s));
    TS_CUDA(c, tsh::launch_stamp(stamp, 1, s));
    if (done != nullptr) TS_CUDA(c, cudaLaunchHostFunc(s, done_host, new DoneThunk{done, user, nullptr}));
    return TS_OK;
}

int ts_hydro_device_alloc(ts_hydro_ctx* c, uint64_t bytes, uint64_t* handle) {
    int rc = guard(c);
    if (rc) return rc;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (bytes == 0 || handle == nullptr) return fail(c, TS_EINVAL, "zero-byte allocation");
    if (c->host_only) return fail(c, TS_ESTATE, "host-only context (device_id = -1) cannot touch the GPU");
    cudaSetDevice(c->dev);
    char* p = nullptr;
    rc = dalloc(c, &p, (size_t)bytes);  // counted + alloc record, like SimDevice::device_alloc
    if (rc) return rc;
    const uint64_t h = c->next_handle++;
    c->handles[h] = {p, bytes};
    *handle = h;
    return TS_OK;
}

int ts_hydro_device_free(ts_hydro_ctx* c, uint64_t handle) {
    if (c == nullptr) return TS_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    auto it = c->handles.find(handle);
    if (it == c->handles.end()) return fail(c, TS_EINVAL, "free of unknown or already-freed device handle");
    cudaSetDevice(c->dev);
    char* p = static_cast<char*>(it->second.first);
    c->handles.erase(it);
    dfree(c, &p);  // free record
    return TS_OK;
}

int ts_hydro_device_ptr(const ts_hydro_ctx* c, uint64_t handle, void** ptr) {
    if (c == nullptr || ptr == nullptr) return TS_EINVAL;
    auto it = c->handles.find(handle);
    if (it == c->handles.end()) return TS_EINVAL;
    *ptr = it->second.first;
    return TS_OK;
}

int ts_hydro_debug_cta_log(ts_hydro_ctx* c, uint64_t* out, uint64_t cap, uint64_t* n) {
    if (c == nullptr || n == nullptr) return TS_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    *n = c->d_cta_log != nullptr ? 12 * (uint64_t)c->n_owned : 0;
    if (out == nullptr || *n == 0) return TS_OK;
    if (cap < *n) return fail(c, TS_EINVAL, "buffer too small");
    cudaSetDevice(c->dev);
    int rc = sync_all(c);
    if (rc) return rc;
    TS_CUDA(c, cudaMemcpy(out, c->d_cta_log, *n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return TS_OK;
}

}  // extern "C"
