/*
 * ts_hydro.h — C ABI of the B200-native hydro hot path (libts_hydro.so).
 *
 * Drop-in boundary for the path the reference `taskscope` toolkit only
 * simulates: `WorkloadSession::fluxes_body` (reference
 * proj/core/src/workload.cpp:544-552) awaiting `SimDevice::launch_kernel`
 * (proj/core/include/taskscope/device.hpp:57-58, device.cpp:24-32) for the
 * `reconstruct_kernel` / `flux_kernel` pair, the ghost exchange around it
 * (`collect_body`, workload.cpp:519-542) and the per-kernel timing hook
 * (`ActivityRecord` -> `Profiler::deliver_activity`, snapshot.hpp:88-99,
 * profiler.cpp:298-318).
 *
 * Conventions:
 *   - every entry point returns TS_OK (0) or a TS_E* code; no exception ever
 *     crosses the ABI.  TS_EINVAL maps to the reference's std::invalid_argument,
 *     TS_ESHUTDOWN to its std::runtime_error("device is shut down"); CUDA and
 *     NCCL failures carry their own text in ts_hydro_last_error();
 *   - host arrays are borrowed for the duration of the call only;
 *   - the context owns every device buffer, stream, event and communicator;
 *   - state arrays are [sub-grid][field][z][y][x] FP64 (x fastest, the
 *     reference's linear index x + N(y + N z), workload.cpp:353), N = 8;
 *     fields: rho, sx, sy, sz, E, tau, then n_species passive densities;
 *   - face order -x,+x,-y,+y,-z,+z, opposite = face ^ 1 (workload.hpp:28-30).
 *
 * There is no CPU fallback: every compute entry point runs on the GPU or
 * fails with TS_ECUDA.
 */
#ifndef TS_HYDRO_H
#define TS_HYDRO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_HYDRO_ABI_VERSION 1

#define TS_OK 0
#define TS_EINVAL 1     /* reference: std::invalid_argument            */
#define TS_ESHUTDOWN 2  /* reference: std::runtime_error (device.cpp:62) */
#define TS_ECUDA 3
#define TS_ENCCL 4
#define TS_ENOMEM 5
#define TS_ESTATE 6     /* call out of order (e.g. stepping before set_mesh) */
#define TS_ECOMM 7      /* a peer rank did not arrive at a cross-GPU wait within the deadline */

#define TS_RECON_PPM 0     /* PPM, MC-limited slopes + CW84 monotonicity (Octo-Tiger form) */
#define TS_RECON_MINMOD 1  /* piecewise-linear minmod */

/* ActivityKind, reference snapshot.hpp:79-86 */
#define TS_ACTIVITY_KERNEL 0
#define TS_ACTIVITY_COPY_H2D 1
#define TS_ACTIVITY_COPY_D2H 2
#define TS_ACTIVITY_COPY_D2D 3
#define TS_ACTIVITY_ALLOC 4
#define TS_ACTIVITY_FREE 5

/* Initial-condition problems for ts_hydro_ic_fill. */
#define TS_PROBLEM_SOD 0
#define TS_PROBLEM_SEDOV 1
#define TS_PROBLEM_RANDOM 2
#define TS_PROBLEM_POLYTROPE 3
#define TS_PROBLEM_BINARY 4

typedef struct ts_hydro_ctx ts_hydro_ctx;

typedef struct ts_hydro_config {
    int32_t device_id;                 /* DeviceConfig::device_id (device.hpp:23)            */
    uint32_t stream_count;             /* DeviceConfig::stream_count (device.hpp:24), 128    */
    uint32_t activity_buffer_capacity; /* DeviceConfig::activity_buffer_capacity (device.hpp:26) */
    int32_t cells_per_edge;            /* SubGrid::cells_per_edge (workload.hpp:60); must be 8 */
    int32_t n_species;                 /* passive species; nf = 6 + n_species, 0..5          */
    int32_t recon;                     /* TS_RECON_*                                          */
    double gamma;                      /* ideal-gas adiabatic index                           */
    double cfl;                        /* Courant number                                      */
    double dx;                         /* cell width (uniform, single level)                  */
    double p_floor;                    /* pressure floor used by the EOS                      */
} ts_hydro_config;

/* ActivityRecord (snapshot.hpp:88-99) with RunClock-compatible timestamps:
 * steady_clock nanoseconds (subtract RunClock::epoch() to get RunClock ns). */
typedef struct ts_activity_record {
    uint8_t kind;
    uint8_t has_bytes;
    uint16_t reserved;
    int32_t device_id;
    int32_t stream_id;
    int32_t pad;
    const char* name; /* static taxonomy string, valid for the library's lifetime */
    uint64_t start_ns;
    uint64_t end_ns;
    uint64_t bytes;
    uint64_t correlation_guid;
} ts_activity_record;

/* DeviceMemoryState, device.hpp:29-34 */
typedef struct ts_memory_state {
    uint64_t current_device_bytes;
    uint64_t peak_device_bytes;
    uint64_t current_host_pinned_bytes;
    uint64_t peak_host_pinned_bytes;
} ts_memory_state;

/* Completion callback: runs on a CUDA host thread once the launch finished on
 * the device (never before, device.hpp:54-56).  It must not call CUDA. */
typedef void (*ts_done_fn)(void* user);

/* Auto-delivery sink for activity records (the SimDevice default sink that
 * receives records when the buffer reaches capacity, device.cpp:105-111). */
typedef void (*ts_activity_sink_fn)(const ts_activity_record* records, uint64_t n, void* user);

/* ---- library / context --------------------------------------------------- */
int ts_hydro_abi_version(void);
void ts_hydro_default_config(ts_hydro_config* cfg);
const char* ts_hydro_strerror(int code);
int ts_hydro_create(const ts_hydro_config* cfg, ts_hydro_ctx** out);
const char* ts_hydro_last_error(const ts_hydro_ctx* ctx);
/* SimDevice::shutdown (device.cpp:223-233): waits for in-flight work, later
 * launches fail with TS_ESHUTDOWN. */
int ts_hydro_shutdown(ts_hydro_ctx* ctx);
int ts_hydro_destroy(ts_hydro_ctx* ctx);
int ts_hydro_num_fields(const ts_hydro_ctx* ctx);

/* ---- mesh (Mesh / SubGrid, workload.hpp:53-97) ---------------------------- */
/* Product-side uniform mesh builder: nx*ny*nz same-level sub-grids numbered
 * along the Morton curve, owners dealt in contiguous chunks like build_mesh
 * (workload.cpp:298-323).  periodic_mask bit d wraps axis d; with
 * TS_MESH_ROW_ORDER set the numbering is row-major, x fastest (the shape of
 * make_row_mesh in the reference's tests, test_workload.cpp:38-54). */
#define TS_MESH_ROW_ORDER 8
int ts_hydro_uniform_mesh(int32_t nx, int32_t ny, int32_t nz, int32_t periodic_mask, int32_t world,
                          int64_t* neighbor_ids, int32_t* pos, int32_t* owner);
/* Binds the global mesh; validates it like Mesh::validate (workload.cpp:140-168).
 * This context owns the sub-grids with owner == rank (ascending global id);
 * foreign neighbours become halo proxies filled by the exchange. */
int ts_hydro_set_mesh(ts_hydro_ctx* ctx, int64_t n_grids, const int64_t* neighbor_ids,
                      const int32_t* owner, int32_t world_size, int32_t rank);
/* ---- coarse-fine AMR mesh ----------
 * The reference's multi-level octree (build_mesh, workload.cpp:264-327) links
 * only same-level faces (Mesh::validate, workload.cpp:160-161), so a leaf
 * next to another level has no ghost source there.  This binds a 2:1-balanced
 * leaf set (single rank) whose cross-level face neighbours are proxy
 * sub-grids: ids n_leaves .. n_leaves+n_proxy-1, refilled before every RK
 * stage by prolongation (piecewise constant) from a coarse leaf or
 * restriction (2x2x2 mean) from 8 fine leaves — only the 3 cell layers next
 * to the faces leaves read them through (the rest of a proxy is unspecified;
 * env TS_HYDRO_AMR_FULLFILL=1 fills whole proxies); after every stage the coarse
 * cells on a coarse-fine face take the mean of the 4 fine face fluxes
 * (reflux), so mass, momentum and energy stay conserved to round-off.
 * Leaves are level-major: level[] non-decreasing, 0..max_level; cfg.dx is
 * the finest level's dx (it sets the global dt), level L updates with
 * dx * 2^(max_level - L).  neighbor_ids: [n_leaves][6] ids of leaves or
 * proxies, -1 = outflow boundary.  Proxy and reflux ids are leaf ids.
 * Layouts are those of oracle/hydro_oracle.h (orc_amr_proxy /
 * orc_amr_reflux_rec).  Stepping: ts_hydro_step / ts_hydro_step_host;
 * multi-rank, the pipelined host path and checkpoints refuse (TS_ESTATE). */
typedef struct {
    int32_t dst;       /* proxy id */
    int32_t kind;      /* 0 = prolong from src[0], 1 = restrict from src[0..7] (octant order) */
    int32_t octant;    /* kind 0: the proxy's octant of src[0] (bit d = upper half along axis d) */
    int32_t src[8];
} ts_amr_proxy;
typedef struct {
    int32_t coarse;    /* coarse leaf with at least one coarse-fine face */
    int32_t fine[6][4];/* per face: the fine leaves behind it by transverse quadrant, -1 = none */
} ts_amr_reflux;
int ts_hydro_set_amr_mesh(ts_hydro_ctx* ctx, int64_t n_leaves, const int64_t* neighbor_ids, const int32_t* level,
                          int32_t max_level, int64_t n_proxy, const ts_amr_proxy* proxies, int64_t n_reflux,
                          const ts_amr_reflux* reflux);
/* The same global AMR mesh partitioned over `world` ranks (owner[leaf]; the
 * reference deals leaves along the Morton curve, workload.cpp:298-323):
 * this rank steps its owned leaves; the remote leaves it reads — same-level
 * face neighbours, sources of the proxies it fills, the fine leaves of its
 * reflux records — are refreshed whole before every stage over the context's
 * transport (ts_hydro_p2p_import or ts_hydro_comm_init); dt is reduced over
 * the ranks.  Bitwise equal to the one-rank run.  owner == NULL or world == 1:
 * ts_hydro_set_amr_mesh. */
int ts_hydro_set_amr_mesh_partitioned(ts_hydro_ctx* ctx, int64_t n_leaves, const int64_t* neighbor_ids,
                                      const int32_t* level, int32_t max_level, int64_t n_proxy,
                                      const ts_amr_proxy* proxies, int64_t n_reflux, const ts_amr_reflux* reflux,
                                      const int32_t* owner, int32_t world, int32_t rank);
int ts_hydro_local_counts(const ts_hydro_ctx* ctx, int64_t* n_owned, int64_t* n_proxy,
                          int64_t* n_interior);
int ts_hydro_owned_ids(const ts_hydro_ctx* ctx, int64_t* global_ids);
/* Halo plan toward `peer`: number of 3-deep slabs sent, and per slab the
 * (global sub-grid id, face of that sub-grid) pairs in wire order (face 6:
 * the whole sub-grid — the ghost leaves of a partitioned AMR mesh). */
int ts_hydro_halo_plan(const ts_hydro_ctx* ctx, int32_t peer, int64_t* n_send, int64_t* send_pairs,
                       int64_t* n_recv, int64_t* recv_pairs);

/* ---- state ---------------------------------------------------------------- */
/* Host-side initial conditions for owned sub-grids (the same [g][nf][512]
 * layout), problems TS_PROBLEM_*; dims = mesh extent in sub-grids. */
int ts_hydro_ic_fill(const ts_hydro_config* cfg, int32_t problem, int64_t n, const int64_t* global_ids,
                     const int32_t* pos, const int32_t* dims, uint64_t seed, double* out);
/* U^n <- host (owned sub-grids [first, first+count) in owned order). */
int ts_hydro_upload(ts_hydro_ctx* ctx, int64_t first, int64_t count, const double* host);
int ts_hydro_download(ts_hydro_ctx* ctx, int64_t first, int64_t count, double* host);
/* Diagnostic: any of the three RK buffers (0 = U^n, 1 = U^(1), 2 = U^(2)). */
int ts_hydro_download_buffer(ts_hydro_ctx* ctx, int32_t which, int64_t first, int64_t count, double* host);
/* Device-side synthetic state (cell_value generator, workload.cpp:329-332). */
int ts_hydro_init_random(ts_hydro_ctx* ctx, uint64_t seed);

/* ---- stepping -------------------------------------------------------------- */
/* Max signal speed of U^n (all ranks) -> dt for the next step. */
int ts_hydro_compute_dt(ts_hydro_ctx* ctx, double* dt_out);
/* nsteps SSP-RK3 steps (3 stages = the reference's 3 hydro rounds per step,
 * workload.hpp:116), each stage: halo exchange + fused
 * reconstruct/flux/update; dt from the cell-centred CFL condition. Async. */
int ts_hydro_step(ts_hydro_ctx* ctx, uint64_t nsteps);
/* Host-buffer step (e2e path): U^n from `host_in`, nsteps steps, U^{n+nsteps}
 * to `host_out` (pinned or pageable), synchronous. */
int ts_hydro_step_host(ts_hydro_ctx* ctx, const double* host_in, double* host_out, uint64_t nsteps);
/* Pipelined form of ts_hydro_step_host (asynchronous; `done` fires once
 * host_out holds the result; ts_hydro_synchronize waits for all).  Copies move
 * in sub-grid chunks on their own streams; when host_in is the previous
 * call's host_out (a simulation chained through host memory) each H2D chunk
 * starts as soon as the previous call's D2H of that chunk landed, so the two
 * PCIe directions overlap.  A chained call also takes the step's dt from the
 * previous call's stage-3 reduction (its input IS that call's output) and
 * starts stage 1 under the H2D: the host must not modify host_in between the
 * two calls (pass a different buffer to restart from new data — that call is
 * not chained and recomputes dt after its H2D).  Host buffers must stay valid
 * until `done`. */
int ts_hydro_step_host_async(ts_hydro_ctx* ctx, const double* host_in, double* host_out, uint64_t nsteps,
                             ts_done_fn done, void* user);
int ts_hydro_synchronize(ts_hydro_ctx* ctx);
/* nsteps steps bracketed by CUDA events on the compute stream (the stream
 * every launch of a step is ordered on); blocks and returns device ms. */
int ts_hydro_time_steps(ts_hydro_ctx* ctx, uint64_t nsteps, double* ms);
int ts_hydro_last_dt(ts_hydro_ctx* ctx, double* dt);
int ts_hydro_steps_done(const ts_hydro_ctx* ctx, uint64_t* steps);
/* Kernel launches issued by this context so far (all kinds). */
int ts_hydro_launch_count(const ts_hydro_ctx* ctx, uint64_t* launches);

/* The compute_fluxes drop-in (workload.cpp:544-552): one fused RK stage
 * (1..3) over `count` owned sub-grids on stream `stream_id`; `done` fires once
 * the device finished.  Stage 1 opens a step; every owned sub-grid then runs
 * stages 1, 2, 3 once, in that order, in any interleaving across sub-grids
 * and streams — no host barrier: each CTA waits on the device for its own
 * and its face neighbours' previous stage (and stage 1 for the previous
 * step's stage-3 count, which carries dt); a launch whose producers were not
 * issued yet is parked and issued once they are.  dt: ts_hydro_compute_dt
 * before the first step, then from the device.  On N ranks (fused P2P
 * transport: ts_hydro_p2p_import; TS_ESTATE otherwise) a boundary sub-grid's
 * launch also acquires the peers' halo slabs of its input and pushes its
 * output's slabs into the peers' proxies, as the batched step does; a stage-k
 * launch holding a boundary sub-grid is issued once every boundary sub-grid
 * has issued stage k-1; the step's dt is reduced over the ranks when the step
 * closes.  Drop-in steps are collective like ts_hydro_step.  On an AMR mesh
 * (single rank) a stage's proxy fill and the previous stage's reflux run once
 * every leaf issued that previous stage, and every launch of the stage waits
 * for them (events): the stages are barriers there, as the reflux needs.
 * State-changing calls fail with TS_ESTATE while a step is open. */
int ts_hydro_launch_stage(ts_hydro_ctx* ctx, int32_t stage, const int64_t* owned_index, int64_t count,
                          uint32_t stream_id, uint64_t correlation_guid, ts_done_fn done, void* user);
/* Close the open per-sub-grid step (every owned sub-grid launched stage 3):
 * joins the step's streams into the compute stream, no host wait (N ranks:
 * then the dt exchange kernel gathers the step's max signal speeds). */
int ts_hydro_finish_step(ts_hydro_ctx* ctx);

/* ---- gravity ------------------------------------- */
/* The near-field monopole P2P behind the reference's `p2p_kernel` launches
 * (gravity_kernel_name workload.cpp:365-372; 6 per sub-grid and step,
 * 565-569): for every cell, phi = -G h^2 sum rho_j / |d| and g = G h sum
 * rho_j d / |d|^3 over the same-level cells at offsets 0 < |d|^2 <= radius^2
 * (radius 1..6 cells, across faces, edges and corners; vacuum outside the
 * mesh) — oracle/hydro_oracle.h orc_gravity_p2p, bitwise.  (The whole
 * solve, near and far field, is ts_hydro_gravity_fmm below.)  owned_index == NULL or
 * count <= 0: every owned sub-grid.  Runs after everything on the compute
 * stream; anything that later replaces or steps the state (steps, kicks,
 * uploads, a drop-in step) waits for it; single rank, uniform mesh, not while
 * a per-sub-grid step is open.
 * Activity record name "p2p_kernel". */
int ts_hydro_gravity_p2p(ts_hydro_ctx* ctx, double G, int32_t radius, const int64_t* owned_index, int64_t count,
                         uint32_t stream_id, uint64_t correlation_guid, ts_done_fn done, void* user);
/* [count][4][512] = (phi, gx, gy, gz) of owned sub-grids first..first+count-1 (waits). */
int ts_hydro_download_gravity(ts_hydro_ctx* ctx, int64_t first, int64_t count, double* host);

/* The whole gravity solve: a cell-based fast multipole method over the octree
 * of 8^3 sub-grids (oracle/hydro_oracle.h orc_gravity_fmm,
 * bitwise).  The tree is given by the leaves — exactly the owned sub-grids, in
 * their storage order: level[k] (0 = the coarsest hydro level, cell width
 * dx0), pos[k][3] at that level inside dims * 2^level; the refined nodes are
 * their ancestors up to one root (T = ceil(log2 max dims) virtual levels above
 * level 0), as in the reference's octree (build_mesh, workload.cpp:264-327).
 * A uniform mesh passes level 0 and ts_hydro_uniform_mesh's positions; an AMR
 * mesh its leaves' levels and positions.  Rebinding a mesh drops the tree.
 * N ranks: the leaves are every rank's sub-grids by global id (the mesh's own
 * numbering); each solve all-gathers the densities over NCCL
 * (ts_hydro_comm_init, next to a P2P transport if that carries the halos) and
 * each rank evaluates its own sub-grids and the expansions of their
 * ancestors — bitwise equal to one rank. */
int ts_hydro_set_gravity_tree(ts_hydro_ctx* ctx, int64_t n_leaves, const int32_t* level, const int32_t* pos,
                              const int32_t* dims, double dx0);
/* One solve of the current state's density on stream `stream_id` (after
 * everything on the compute stream; later state changes wait for it): monopoles about the centre of mass,
 * first-order local expansions, interaction radius `radius` (1..3 cells: a
 * cell interacts directly with the cells within `radius`, and with its
 * parent's near cells' children beyond it).  Output: ts_hydro_download_gravity.
 * Activity records, one per launch, named as the reference names the kinds
 * (workload.hpp:45-48): "fmm_moments_kernel" (leaf masses), per refined depth
 * "multipole_kernel" ("multipole_root_kernel" at the root: restriction, then
 * expansions), "p2p_kernel" / "p2m_kernel" (leaves, by kind: see
 * ts_hydro_gravity_tree). */
int ts_hydro_gravity_fmm(ts_hydro_ctx* ctx, double G, int32_t radius, uint32_t stream_id, uint64_t correlation_guid,
                         ts_done_fn done, void* user);
/* The gravity source over dt on the owned sub-grids from the last gravity
 * solve (ts_hydro_gravity_fmm or _p2p): S += dt rho g, E += dt/2 (S + S').g
 * (oracle orc_gravity_kick, bitwise).  dt < 0: the last step's dt, read on
 * the device.  The next step recomputes its dt from the kicked state. */
int ts_hydro_gravity_kick(ts_hydro_ctx* ctx, double dt);
/* Hydro with self-gravity (un-freezing gravity in config 4): per step one
 * SSP-RK3 hydro step, the FMM on its result, the kick over that step's dt —
 * the reference's per-step order (3 hydro rounds, then the gravity launches,
 * workload.cpp:559-569) — all on the compute stream, no host round trip.
 * Needs ts_hydro_set_gravity_tree; collective on N ranks. */
int ts_hydro_step_gravity(ts_hydro_ctx* ctx, uint64_t nsteps, double G, int32_t radius);
/* The gravity tree of these leaves (ts_hydro_set_gravity_tree's arguments; no
 * context, no device): n_nodes always, the arrays when cap >= n_nodes — per
 * node its level (hydro level: negative above level 0), pos[3] at that level,
 * kind as the reference's gravity_kernel_name picks it (workload.cpp:365-372:
 * 0 multipole_root_kernel, 1 multipole_kernel, 2 p2m_kernel, 3 p2p_kernel)
 * and leaf (its index among the leaves, or -1 for a refined node).  Any
 * output may be NULL.  Nodes: refined ones by level, then the leaves by
 * level.  On the reference's own octrees the nodes are its grids.
 * TS_EINVAL for a malformed tree. */
int ts_hydro_gravity_tree(int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                          int64_t cap, int32_t* level_out, int32_t* pos_out, int32_t* kind, int32_t* leaf,
                          int64_t* n_nodes);

/* ---- ghost exchange --------------------------------------------------------- */
/* The reference's 1-deep face exchange of field 0 (workload.cpp:487-542):
 * ghost[g][face][j] = neighbour cell face_cell_index(8, face^1, j), 0 where no
 * neighbour; [n_owned][6][64]. */
int ts_hydro_exchange_faces(ts_hydro_ctx* ctx, double* ghost_host);
/* 26-neighbour padded tiles (8+2*depth)^3 of every owned sub-grid, all fields. */
int ts_hydro_fill_halo(ts_hydro_ctx* ctx, int32_t depth, double* tiles_host);
/* Cross-GPU halo transport (NCCL, loaded at run time). */
int ts_hydro_nccl_unique_id(uint8_t id[128]);
int ts_hydro_comm_init(ts_hydro_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank);
/* NVLink-native transport inside one node (alternative to NCCL): every rank
 * exports a blob (CUDA IPC handles of its halo receive buffer, flag array and
 * dt gather array, and where each source rank's slabs land), the blobs are
 * all-gathered by the host, and each rank imports all of them.  Halos then
 * move with copy engines straight into the peer's receive buffer, ordered by
 * stream memory operations (flag write / wait): no SM and no NCCL kernel on
 * the step's critical path.  Replaces the parcel transport of
 * send_boundary / handle_boundary (workload.cpp:487-517). */
uint64_t ts_hydro_p2p_blob_size(void);
int ts_hydro_p2p_export(ts_hydro_ctx* ctx, void* blob);
int ts_hydro_p2p_import(ts_hydro_ctx* ctx, const void* blobs, int32_t world);
/* One packed-halo exchange of U^n (pack -> transfer -> unpack). */
int ts_hydro_halo_exchange(ts_hydro_ctx* ctx);

/* Diagnostic: bitwise check of the kernels' branch-free reciprocal and square
 * root against IEEE 1.0/x and sqrt(x) on n random positive doubles with
 * binary exponents in [-emax, emax]; emax < 0 draws mantissas within 2^-20
 * of 1 or 2 instead, 1 in 64 exactly all-ones (exponents in [emax, -emax]).
 * Returns the mismatch counts. */
int ts_hydro_selftest_math(ts_hydro_ctx* ctx, uint64_t n, uint64_t seed, int32_t emax, uint64_t* bad_rcp,
                           uint64_t* bad_sqrt);

/* ---- persisted state (checkpoint / restart) ------------------------------------ */
/* FP64 field dump + mesh (the reference persists only
 * profiles, codec.cpp:17-225, whose magic/version/length-checked layout this
 * follows).  Layout: paper_2210_06437_b200/csrc/ts_hydro_ckpt.cpp.  Every
 * reader validates magic, version, sizes and an FNV-1a 64 payload checksum
 * (TS_EINVAL on any mismatch). */
typedef struct ts_hydro_checkpoint_header {
    uint32_t version;
    int32_t nf, n_species, recon, cells_per_edge;
    double gamma, cfl, dx, p_floor;
    int64_t n_grids;   /* global mesh size                 */
    int64_t n_records; /* sub-grids stored in this file    */
    uint64_t steps_done;
    int32_t world, rank; /* of the writer                  */
    uint64_t checksum;
} ts_hydro_checkpoint_header;

/* Host-only (no GPU): write / inspect / read one checkpoint file.  state is
 * [n_records][nf][512] in global_ids order. */
int ts_hydro_checkpoint_write(const char* path, const ts_hydro_config* cfg, int64_t n_grids,
                              const int64_t* neighbor_ids, const int32_t* owner, int32_t world, int32_t rank,
                              int64_t n_records, const int64_t* global_ids, const double* state,
                              uint64_t steps_done);
int ts_hydro_checkpoint_info(const char* path, ts_hydro_checkpoint_header* out);
/* Any output may be NULL (section skipped). */
int ts_hydro_checkpoint_read(const char* path, int64_t* neighbor_ids, int32_t* owner, int64_t* global_ids,
                             double* state);
/* This context's U^n (its owned sub-grids) + the global mesh -> `path`. */
int ts_hydro_save(ts_hydro_ctx* ctx, const char* path);
/* U^n of this context's owned sub-grids from the files of a checkpoint (one
 * per writing rank; any rank count): the bound mesh must equal the stored one
 * (ownership may differ) and the numerics parameters must match. */
int ts_hydro_restore(ts_hydro_ctx* ctx, const char* const* paths, int32_t n_paths);
/* The bound global mesh (any output may be NULL) and the context's config. */
int ts_hydro_get_mesh(const ts_hydro_ctx* ctx, int64_t* n_grids, int64_t* neighbor_ids, int32_t* owner,
                      int32_t* world, int32_t* rank);
int ts_hydro_get_config(const ts_hydro_ctx* ctx, ts_hydro_config* out);

/* ---- the rest of the SimDevice contract on the real device ------------------- */
/* SimDevice::launch_kernel (device.hpp:57-58, device.cpp:24-32): a named
 * launch that occupies `stream_id` for duration_ns on the GPU (one timed
 * thread), FIFO per stream, overlapping across streams; one kernel record
 * named `name` (interned: the pointer stays valid for the context's life).
 * TS_EINVAL: zero duration, bad stream, NULL/empty name.  `done` as for
 * ts_hydro_launch_stage.  Usable on a context without a mesh. */
int ts_hydro_launch_kernel(ts_hydro_ctx* ctx, const char* name, uint32_t stream_id, uint64_t duration_ns,
                           uint64_t correlation_guid, ts_done_fn done, void* user);
/* SimDevice::enqueue_copy (device.hpp:60-61, device.cpp:34-52): a real copy of
 * `bytes` between context-owned staging buffers in direction `kind`
 * (TS_ACTIVITY_COPY_H2D / _D2H / _D2D; pinned host <-> device), on the
 * stream, with a device-stamped record carrying the bytes.  TS_EINVAL: not a
 * copy kind, zero bytes, bad stream. */
int ts_hydro_enqueue_copy(ts_hydro_ctx* ctx, int32_t kind, uint64_t bytes, uint32_t stream_id,
                          uint64_t correlation_guid, ts_done_fn done, void* user);
/* SimDevice::device_alloc / device_free (device.hpp:62-63, device.cpp:132-199):
 * cudaMalloc / cudaFree with alloc / free records (stream -1, bytes) and
 * memory counters; handles are opaque non-zero ids.  TS_EINVAL: zero bytes,
 * unknown or already-freed handle. */
int ts_hydro_device_alloc(ts_hydro_ctx* ctx, uint64_t bytes, uint64_t* handle);
int ts_hydro_device_free(ts_hydro_ctx* ctx, uint64_t handle);
/* Device address behind a handle (for callers that fill the buffer). */
int ts_hydro_device_ptr(const ts_hydro_ctx* ctx, uint64_t handle, void** ptr);

/* Diagnostic: with TS_HYDRO_CTA_LOG set when the mesh is bound, every stage
 * launch of ts_hydro_step logs per CTA {SM id, start, work start after the
 * halo / dataflow waits, end} (globaltimer ns); this returns the last step's
 * [3 stages][n_owned CTAs][4] (n = 0 when logging is off; out == NULL: count). */
int ts_hydro_debug_cta_log(ts_hydro_ctx* ctx, uint64_t* out, uint64_t cap, uint64_t* n);

/* ---- timing hook -------------------------------------------------------------- */
int ts_hydro_set_activity_sink(ts_hydro_ctx* ctx, ts_activity_sink_fn sink, void* user);
/* The profiling arms of the reference's overhead harness (ProfilingArm,
 * harness.hpp; arm_config harness.cpp:33-52): enabled (default) = every
 * launch stamps its activity record ("full"); 0 = no stamps and no records
 * ("disabled": profiler.enabled = false).  compute_overhead of the two step
 * times is the per-kernel timing hook's o(n) (harness.cpp:15-20). */
int ts_hydro_set_profiling(ts_hydro_ctx* ctx, int32_t enabled);

/* Self-check builds (TS_CHECK=1; the race / bounds detector standing in for
 * compute-sanitizer, which this pool does not allow — DESIGN.md §13): the
 * stage kernels bounds-check every state load / store and re-check every
 * acquired dataflow / halo flag at CTA exit.  out = {failures, first code,
 * operand a, operand b, OR of (1 << code) over all failures}; waits for the
 * device first.  Always 0 failures in a normal build (nothing is checked). */
int ts_hydro_debug_check(ts_hydro_ctx* ctx, uint64_t out[5], int32_t reset);
/* 1 when this library is a TS_CHECK build. */
int ts_hydro_check_build(void);
/* SimDevice::flush_activity: waits for in-flight work, returns completed
 * records not yet delivered (at most once).  out == NULL -> count only. */
int ts_hydro_flush_activity(ts_hydro_ctx* ctx, ts_activity_record* out, uint64_t cap, uint64_t* n_out);
int ts_hydro_memory_state(const ts_hydro_ctx* ctx, ts_memory_state* out);
/* SimDevice::host_pinned_alloc / host_pinned_free (device.hpp:63-64), backed
 * by cudaHostAlloc; counted in ts_memory_state. */
int ts_hydro_host_alloc(ts_hydro_ctx* ctx, uint64_t bytes, void** ptr);
int ts_hydro_host_free(ts_hydro_ctx* ctx, void* ptr);
/* steady_clock ns now (the clock the records are on). */
uint64_t ts_hydro_clock_ns(void);

#ifdef __cplusplus
}
#endif

#endif
