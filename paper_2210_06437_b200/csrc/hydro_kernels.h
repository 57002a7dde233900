// hydro_kernels.h — host-side launch interface of hydro_kernels.cu.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tsh {

struct StageArgs {
    // TMA descriptor of U^{(k-1)} viewed as rows of 16 doubles (128 B):
    // one {16, 32} box = one field of one sub-grid (4 KiB), 128-byte swizzled
    // into shared memory (TS_TMA builds; see hydro_stage.cuh).  First member:
    // the kernel parameter block keeps its 64-byte alignment.
    CUtensorMap tmap_prev;
    int tma;                    // 1: the descriptor is valid
    const double* Uprev;        // U^{(k-1)}: owned + proxy sub-grids
    const double* Un;           // U^n (stages 2, 3)
    double* Uout;               // U^{(k)}
    double* scratch;            // a state buffer free during this stage (species accumulators, nf > 6)
    // nf > 6: species accumulators in a small ring of per-SM slots instead of
    // the sub-grid's own slot of `scratch`: a CTA takes a free slot of its SM
    // (scr_mask[smid] bit) and frees it at exit, so the same ~12 MB of lines
    // are rewritten while still in L2 and never written back to HBM (the
    // state-buffer scratch cost nf 11 ~20 % extra DRAM traffic).
    // Self-check builds (TS_CHECK=1): every pencil load,
    // U^n load and U^(k) store is bounds-checked against the buffers, and
    // every acquired dataflow / halo flag is re-read at the CTA's end (a
    // value past the awaited one means a producer overtook its consumer).
    // Failures are counted in check[0], the first one in check[1..3],
    // check[4] = OR of (1 << code) over all of them.
    unsigned long long* check;
    long long n_local;          // sub-grid slots in each state buffer
    long long n_owned;          // sub-grids this rank updates
    double* scr_ring;           // [n_sm * scr_k][nf - 6][512] (nullptr: use scratch)
    unsigned int* scr_mask;     // [256] busy-slot bits per SM id
    int scr_k;                  // slots per SM (<= 32)
    const int* nbr;             // [local][6] local neighbour index, -1 = outflow
    const int* list;            // CTA -> local sub-grid (nullable: first + blockIdx.x)
    int first;
    // Per-sub-grid drop-in (ts_hydro_launch_stage): up to kInlineList sub-grids
    // passed by value in the launch parameters (no device list per launch);
    // list_inline_n > 0 takes precedence over list / first.
    static constexpr int kInlineList = 32;
    int list_inline_n;
    int list_inline[kInlineList];
    // The CTA that does stage 1's once-per-step duties (dt_out, amax_reset,
    // amax_reset2): 0 = block 0 of the launch (batched steps); g + 1 = the CTA
    // of sub-grid g (drop-in launches: exactly one launch per step holds it).
    int lead_g1;
    const double* amax_in;      // signal speed(s) behind this step's dt (max over amax_n values:
    int amax_n;                 //   one per rank when the P2P transport gathered them)
    double* amax_out;           // stage 3: max signal speed of U^{n+1}
    double* amax_reset;         // stage 1: zeroed (the slot stage 3 accumulates into)
    double* dt_out;             // stage 1: dt of this step
    unsigned long long* stamp;  // [start, end] globaltimer ns of this launch (nullable)
    // Diagnostic (TS_HYDRO_CTA_LOG): per CTA {SM id, start, work start (after
    // the halo / dataflow waits), end} in globaltimer ns, indexed by blockIdx.
    unsigned long long* cta_log;
    // Stage 3, multi-rank P2P transport, TS_HYDRO_DT=tail (the default is the
    // one-thread dt_exchange_kernel after stage 3): every CTA counts out in done_ctr
    // (across all launches of the stage, total_ctas); the last one pushes the
    // rank's final amax into slot `rank` of every rank's gather array
    // (push_gather, this step's half), raises their dt flags (push_flag[q],
    // nullptr for self) to seq, waits for the peers' dt flags (dt_wait[q] >=
    // seq) and writes the max over its own gather half (gather_own) to
    // amax_global, the next stage 1's amax_in.  The dt all-reduce is thereby
    // one CTA's tail: stage 1 starts with the global dt in place.
    unsigned int* done_ctr;              // nullptr: single rank (no tail); monotonic
    unsigned int done_target;            // done_ctr after this stage's last CTA counted
    int rank;
    int push_n;                          // ranks to push the amax to (0: no dt push)
    double* const* push_gather;          // [push_n] gather arrays (this step's half)
    unsigned int* const* push_flag;      // [push_n] dt flag words (nullptr for self)
    unsigned int seq;
    const unsigned int* dt_wait;         // own dt flags by source rank (nullptr: no wait)
    const double* gather_own;            // own gather half [push_n]
    double* amax_global;
    // P2P transport, fused halo exchange.  The n_boundary sub-grids with a
    // foreign face neighbour (bnd_of[g] = their boundary slot b, -1 for
    // interior sub-grids) are spread through the front of a batched launch,
    // or come in any per-sub-grid launch of a drop-in step.  Each
    // stores its 3-deep output slabs straight into the proxy slots of the
    // peers' U^(k) buffers over NVLink (push_tbl[6 b + face] = {peer rank,
    // peer-local sub-grid} or {-1, -1}); the last one (halo_ctr) releases
    // halo_flag[q] = halo_seq on every receiving peer.  Boundary CTAs
    // acquire their own flags (halo_wait, by source rank, for the ranks in
    // halo_wait_mask, >= halo_wait_seq) before reading proxies; interior CTAs
    // run meanwhile, so the wait is off the critical path.
    int n_boundary;
    const int* bnd_of;                   // [n_owned]
    const int2* push_tbl;                // nullptr: no push
    double* const* push_out;             // [world] peer's buffer of this stage's U^(k)
    // halo_ctr: one monotonic counter per stage slot (halo_seq % 3), never
    // reset in the kernel: stages overlap (PDL), so a shared or reset counter
    // could be bumped by the next stage's CTAs before this one completes
    unsigned int* halo_ctr;
    unsigned int halo_target;            // halo_ctr after this stage's last boundary CTA counted
    unsigned int* const* halo_flag;      // [world] (nullptr: no slabs for that rank)
    int halo_flag_n;
    unsigned int halo_seq;
    const unsigned int* halo_wait;       // own halo flags, by source rank
    unsigned long long halo_wait_mask;
    unsigned int halo_wait_seq;
    // Single-rank dataflow between the stages of one step.  Stages 2 and 3
    // are launched as programmatic dependents (PDL) of the previous stage, so
    // their CTAs start in the previous stage's last wave instead of after it.
    // A CTA then waits until its own sub-grid and its six face neighbours
    // finished the previous stage (flow_wait[h] >= flow_seq, acquire) — the
    // only data a stage reads — and publishes its own completion
    // (flow_done[g] = flow_seq, release).  pdl_trigger: this launch lets its
    // dependent start once every CTA is running (block 0 of stage 1 first
    // zeroes amax_reset, which stage 3 accumulates into).
    const unsigned int* flow_wait;       // nullptr: no wait (stream order)
    unsigned int* flow_done;             // nullptr: no publish
    unsigned int flow_seq;               // published value
    unsigned int flow_wait_seq;          // awaited value (the previous step's for stage 1)
    // Single rank, across the step boundary: stage 1 is also a PDL dependent
    // (of the previous step's stage 3).  Its x and y sweeps only need U^n of
    // the sub-grid and its neighbours (flow flags of stage 3); dt needs every
    // sub-grid's stage-3 max, so before its z sweep a CTA acquires the count of
    // finished stage-3 CTAs (cnt_wait >= cnt_expect; stage 3 counts into
    // cnt_done after its max atomics) and only then reads amax_in.  The max
    // slots form a ring of three: block 0 of stage 1 zeroes the slot two steps
    // ahead (amax_reset2) once the count is complete.
    // With N ranks (fused P2P, dt gathered in stage 3's tail) the same chain
    // holds, but dt is global: cnt_gather = 1 makes only the gathering last
    // CTA count, by flow_n, once amax_global is written.
    const unsigned int* cnt_wait;
    unsigned int cnt_expect;
    unsigned int* cnt_done;
    int cnt_gather;
    double* amax_reset2;
    int flow_n;                          // owned sub-grids (flag count); proxies are gated by the halo flags
    int pdl_trigger;
    // Stage 3 of a pipelined host step (ts_hydro_step_host_async): each CTA
    // counts its sub-grid into chunk_ctr[g * chunk_n / chunk_owned] after a
    // gpu-scope fence, so the D2H of a chunk can start (stream wait on the
    // counter) while the rest of the stage still runs.
    unsigned int* chunk_ctr;             // nullptr: no counting
    int chunk_n, chunk_owned;
    // First stage 1 of a chained pipelined host step: U^n arrives by H2D
    // chunks (sub-grid g in chunk g * chunk_n / chunk_owned) whose landing the
    // copy stream signals with h2d_flag[chunk] = h2d_seq (a stream memory
    // write behind each copy: release of the copy's bytes).  A CTA acquires
    // the flags of its own and its face neighbours' chunks before reading, so
    // the stage runs under the transfer instead of after all of it.
    const unsigned int* h2d_flag;        // nullptr: U^n already in place
    unsigned int h2d_seq;
    // Every cross-GPU spin gives up after wait_ns (globaltimer) and sets
    // *err (mapped host word) instead of hanging the GPU.
    unsigned long long* err;
    unsigned long long wait_ns;
    double gamma, gm1, cfl, dx, p_floor;
    // dx of the sub-grids this launch updates: dx (the finest level's, which
    // sets dt) on a uniform mesh, dx * 2^(max_level - level) for one level of
    // an AMR mesh (launched per level, ts_hydro_set_amr_mesh)
    double dx_upd;
    // AMR, all levels in one launch: sub-grid g (level-major) is updated
    // with lvl_dx[L] for the last L < lvl_n with g >= lvl_first[L]
    // (lvl_n = 0: dx_upd for every CTA)
    // AMR flux register: for a leaf face that is a coarse-fine face (either
    // side), rf_slot[6 g + face] >= 0 names a slot of rf_flux where the sweep
    // stores that face's (doubled, kt2) flux of every field and face cell
    // ([slot][nf][64], cell a + 8 b in the sweep's transverse axes); the
    // reflux kernel then corrects the coarse cells from the stored fluxes
    // instead of reconstructing them again (nullptr: no register)
    const int* rf_slot;
    double* rf_flux;
    static constexpr int kMaxLevels = 8;
    int lvl_n;
    int lvl_first[kMaxLevels];
    double lvl_dx[kMaxLevels];
};

// Coarse–fine AMR (amr_kernels.cu): proxy fill recipe and reflux record,
// the layouts of ts_amr_proxy / ts_amr_reflux (include/ts_hydro.h).
struct AmrProxy {
    int dst, kind, octant, src[8];  // kind 0: prolong from src[0]; 1: restrict from src[0..7]
};
struct AmrReflux {
    int coarse;
    int fine[6][4];  // per face the 4 fine sub-grids behind it, -1: not coarse–fine
};

// pdl: launch as a programmatic dependent of the previous kernel on `s`
// (cudaLaunchAttributeProgrammaticStreamSerialization; see StageArgs::flow_*).
cudaError_t launch_stage(const StageArgs& a, int nf, int recon, int stage, int n_ctas, cudaStream_t s,
                         bool pdl = false);
cudaError_t launch_signal(const double* U, int nf, long long n_grids, double gamma, double p_floor,
                          double* amax, unsigned long long* stamp, int sms, cudaStream_t s);
cudaError_t launch_init_random(double* U, int nf, const long long* gid, long long n_grids, uint64_t seed,
                               double gamma, int sms, cudaStream_t s);
// cells per entry: SLAB (3-deep face slab {sub-grid, face}) or NC (whole sub-grid)
cudaError_t launch_pack(const double* U, int nf, const int2* entries, long long n, double* buf, int sms,
                        cudaStream_t s, unsigned long long* stamp, int cells = 3 * 8 * 8);
cudaError_t launch_unpack(double* U, int nf, const int2* entries, long long n, const double* buf, int sms,
                          cudaStream_t s, unsigned long long* stamp, int cells = 3 * 8 * 8);
cudaError_t launch_face_exchange(const double* U, int nf, const int* nbr, long long n_owned, double* ghost,
                                 int sms, cudaStream_t s);
cudaError_t launch_fill_halo(const double* U, int nf, const int* nbr, long long n_owned, int h,
                             double* tiles, int sms, cudaStream_t s);
cudaError_t launch_clock(unsigned long long* out, cudaStream_t s);
cudaError_t launch_timed(unsigned long long duration_ns, unsigned long long* stamp, cudaStream_t s);
cudaError_t launch_stamp(unsigned long long* stamp, int which, cudaStream_t s);
cudaError_t launch_dt_exchange(const double* local_amax, double* const* push_gather, unsigned int* const* push_flag,
                               int world, int rank, unsigned int seq, const unsigned int* dt_wait,
                               const double* gather_own, double* amax_global, unsigned long long* err,
                               unsigned long long wait_ns, cudaStream_t s);
cudaError_t launch_wait_flags(const unsigned int* flags, unsigned long long mask, unsigned int seq,
                              unsigned long long* err, unsigned long long wait_ns, cudaStream_t s);
// face_mask[p] (nullable: whole proxies): bit f set when some sub-grid reads
// proxy p through p's face f; only the 3 cell layers next to those faces are
// filled (the stage and reflux kernels read nothing else of a proxy)
cudaError_t launch_amr_fill(double* U, int nf, const AmrProxy* px, const unsigned char* face_mask, long long n,
                            unsigned long long* stamp, cudaStream_t s);
cudaError_t launch_amr_reflux(const double* Uprev, double* Uout, int nf, int recon, double gamma, double p_floor,
                              const int* nbr, const int* level, int max_level, double dx, const AmrReflux* rf,
                              long long n, int stage, const double* dt, unsigned long long* stamp,
                              cudaStream_t s);
// Gravity slice (gravity_kernels.cu): near-field monopole P2P, one CTA per
// sub-grid (list_inline or first + blockIdx.x); out [n][4][512] = (phi, g).
constexpr int kP2PRMax = 6;
struct P2PArgs {
    const double* U;   // state (field 0 = density)
    int nf;
    const int* nbr;    // [local][6]
    double* out;
    int list_inline_n;
    int list_inline[StageArgs::kInlineList];
    int first;
    int radius;        // 1..kP2PRMax
    int n_stencil;     // entries of the radius' stencil (a prefix of the R = 6 table)
    double kphi, kg;   // -G h^2, G h
    unsigned long long* stamp;
};
int p2p_stencil_host(int radius, int* off3, double* coef4, int cap);
cudaError_t launch_p2p(const P2PArgs& a, int n_ctas, cudaStream_t s);
// Reflux from the stage kernel's flux register (StageArgs::rf_slot / rf_flux).
cudaError_t launch_amr_reflux_reg(double* Uout, int nf, const int* level, int max_level, double dx,
                                  const AmrReflux* rf, long long n, const int* rf_slot, const double* rf_flux,
                                  int stage, const double* dt, unsigned long long* stamp, cudaStream_t s);
cudaError_t launch_selftest_math(unsigned long long n, unsigned long long seed, int emax, unsigned long long* bad,
                                 int sms, cudaStream_t s);

}  // namespace tsh
