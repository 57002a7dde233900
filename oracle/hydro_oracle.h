/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, FP64, scalar) of the hydro hot path that the
 * B200 kernels in paper_2210_06437_b200/csrc implement.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the CPU baseline — never
 * as the product path.
 *
 * What it restates (see DESIGN.md §2 for the full numerics contract):
 *   - the reference data model: SubGrid cells x-fastest
 *     (reference proj/core/src/workload.cpp:353), face order -x,+x,-y,+y,-z,+z
 *     with opposite = face^1 (workload.hpp:28-30), face_cell_index
 *     (workload.cpp:340-354), cell_value / mix64 synthetic data
 *     (workload.cpp:329-332, sampling.hpp:12-21), contiguous Morton-chunk
 *     ownership (workload.cpp:298-323), 3 hydro rounds per step
 *     (workload.hpp:116, workload.cpp:559-564);
 *   - the hydro arithmetic the reference only simulates
 *     (reconstruct_kernel / flux_kernel, workload.cpp:544-552): PPM with
 *     minmod-theta (MC) limited slopes and the Colella–Woodward monotonicity
 *     step in the form Octo-Tiger uses, a minmod-PLM variant,
 *     the Kurganov–Tadmor central flux, SSP-RK3 (Shu–Osher) and
 *     a cell-centred CFL time step.
 *
 * Parity status: the reference ships no hydro arithmetic (SPEC.md:8, 519,
 * 528), so the physics is pinned by known-answer tests (exact Sod Riemann
 * solution, exact conservation, symmetry) and the data-model pieces by golden
 * vectors generated from the compiled reference (tests/golden/).
 */
#ifndef TS_HYDRO_ORACLE_H
#define TS_HYDRO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_N 8
#define ORC_NC 512

typedef struct {
    int32_t nf;        /* 6 + passive species: rho, sx, sy, sz, E, tau, species... */
    int32_t recon;     /* 0 = PPM (MC-limited), 1 = minmod PLM */
    double gamma;
    double cfl;
    double dx;
    double p_floor;
} orc_params;

/* --- reference data-model restatements (golden-vector pinned) --- */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_mix64_2(uint64_t a, uint64_t b);
double orc_cell_value(uint64_t grid_id, uint64_t step, uint64_t index);
uint64_t orc_face_cell_index(int edge, int face, uint64_t j);
uint64_t orc_morton3(uint32_t x, uint32_t y, uint32_t z);

/* Uniform single-level mesh of nx*ny*nz sub-grids numbered along the Morton
 * curve; neighbours [g][6] (-1 = domain boundary -> outflow), positions
 * [g][3], owner [g] dealt in contiguous chunks over `world` ranks. */
int orc_uniform_mesh(int nx, int ny, int nz, int periodic_x, int periodic_y, int periodic_z,
                     int world, int64_t* nbr, int32_t* pos, int32_t* owner);

/* Reference 1-deep face exchange of a scalar field (field 0 of U):
 * ghost[g][face][j] = U[nbr][face_cell_index(8, face^1, j)] or 0 if absent. */
void orc_exchange_faces(int nf, int64_t ngrids, const int64_t* nbr, const double* U, double* ghost);

/* Padded (N+2H)^3 tile per sub-grid and field, 26-neighbour halo of depth h. */
void orc_fill_halo(int nf, int64_t ngrids, const int64_t* nbr, const double* U, int h, double* tiles);

/* --- hydro --- */
double orc_max_signal_speed(const orc_params* p, int64_t g_begin, int64_t g_end, const double* U);

/* One SSP-RK3 stage (1, 2 or 3) for sub-grids [g_begin, g_end). */
void orc_stage(const orc_params* p, int64_t ngrids, const int64_t* nbr, const double* Uprev,
               const double* Un, double* Uout, int stage, double dtdx, int64_t g_begin,
               int64_t g_end);

/* nsteps full steps in place on U; dt of every step into dt_hist (may be 0).
 * nthreads > 1 splits every stage over pthreads by sub-grid range. */
int orc_run(const orc_params* p, int64_t ngrids, const int64_t* nbr, double* U, int nsteps,
            double* dt_hist, int nthreads);

/* Sums of every field over all cells (fixed order) for conservation checks. */
void orc_field_sums(int nf, int64_t ngrids, const double* U, double* sums);

/* --- initial conditions (cell-centred, domain [0, nx*8*dx) x ...) --- */
void orc_ic_sod(const orc_params* p, int64_t ngrids, const int32_t* pos, int axis, double* U);
void orc_ic_sedov(const orc_params* p, int64_t ngrids, const int32_t* pos, int nx, int ny, int nz,
                  double* U);
void orc_ic_random(const orc_params* p, int64_t g_begin, int64_t g_end, uint64_t seed, double* U);
/* configs 3 / 4 initial models (domain nx x ny x nz sub-grids) */
void orc_ic_polytrope(const orc_params* p, int64_t ngrids, const int32_t* pos, int nx, int ny, int nz, double* U);
int orc_ic_binary(const orc_params* p, int64_t ngrids, const int32_t* pos, int nx, int ny, int nz, double* U);


/* --- coarse-fine AMR ---
 * Leaves numbered level-major (level_first[L] .. level_first[L+1]-1), then the
 * proxies.  A leaf's face neighbour is a same-level leaf, a proxy or -1.
 * Proxy kinds: 0 = prolongation (piecewise constant) from coarse leaf src[0],
 * octant bit i = the proxy's half of that leaf along axis i; 1 = restriction
 * (mean of 2x2x2 cells) from the 8 fine leaves src[octant o].  Reflux record:
 * coarse leaf + for each face the 4 fine leaves behind it ((a>>2) + 2 (b>>2)
 * over the face's transverse axes, -1 = not a coarse-fine face). */
typedef struct {
    int32_t dst, kind, octant, src[8];
} orc_amr_proxy;
typedef struct {
    int32_t coarse;
    int32_t fine[6][4];
} orc_amr_reflux_rec;

void orc_amr_fill(int nf, int64_t n_proxy, const orc_amr_proxy* px, double* U);
/* Flux correction after stage `stage` (Uout already holds the stage result):
 * coarse boundary cells take the mean of the fine face fluxes instead of
 * their own.  dx of level L = ldexp(p->dx, max_level - L). */
void orc_amr_reflux(const orc_params* p, const int64_t* nbr, const int32_t* level, int max_level,
                    int64_t n_rec, const orc_amr_reflux_rec* rf, const double* Uprev, double* Uout, int stage,
                    double dt);
void orc_debug_face_fluxes(const orc_params* p, const int64_t* nbr, const double* U, int64_t g, int axis, int a,
                           int b, double* F);
/* nsteps SSP-RK3 steps on an AMR mesh, one global dt = cfl dx / amax. */
int orc_run_amr(const orc_params* p, int64_t n_total, const int64_t* nbr, const int32_t* level,
                const int64_t* level_first, int max_level, int64_t n_proxy, const orc_amr_proxy* px,
                int64_t n_rec, const orc_amr_reflux_rec* rf, double* U, int nsteps, double* dt_hist);

/* --- gravity, near-field slice (the reference's
 * p2p_kernel launches, workload.cpp:365-372, 565-569; Octo-Tiger's "p2p
 * interactions kernel: cell to cell interactions in non-refined sub-grids",
 * PAPER.md:355) ---
 * Monopole cell-to-cell interactions of every cell with the same-level cells
 * at offsets 0 < |d|^2 <= R^2 (R <= ORC_P2P_RMAX), across sub-grid faces,
 * edges and corners (walking the face links axis by axis; a missing
 * neighbour is vacuum).  Stencil order: |d|^2 ascending, then (dz, dy, dx)
 * lexicographic, so the stencil of R is a prefix of the stencil of RMAX.
 * Per entry: c0 = 1/sqrt(|d|^2), c3 = c0/|d|^2, c = d c3.  Per cell, in
 * stencil order: S0 = fma(rho_j, c0, S0), S = fma(rho_j, c, S); then
 * phi = (-G h^2) S0, g = (G h) S  (m_j = rho_j h^3; g = -grad phi).
 * out[g][4][512] = (phi, gx, gy, gz). */
#define ORC_P2P_RMAX 6
int orc_p2p_stencil(int radius, int32_t* off, double* coef, int cap);
void orc_gravity_p2p(const orc_params* p, int64_t ngrids, const int64_t* nbr, const double* U, int radius, double G,
                     double* out);

/* --- gravity, the whole solve: a cell-based FMM over the octree of 8^3
 * sub-grids (fmm_oracle.c; the reference's
 * multipole_root / multipole / p2m / p2p launches, workload.cpp:365-372).
 * Leaves k = 0..n-1: level[k] >= 0 (0 = the coarsest hydro level, whose cell
 * width is dx0), pos[k][3] at that level, inside dims * 2^level; U = the
 * leaves' states (nf fields, density = field 0).  Tree: T = ceil(log2
 * max(dims)) virtual depths above level 0 (depth = level + T, h_d = dx0 2^(T-d)),
 * nodes = leaves + every ancestor.  Contract in full: DESIGN.md §15.
 * out[k][4][512] = (phi, gx, gy, gz); returns -1 on a malformed tree. */
#define ORC_FMM_RMAX 3
#define ORC_FMM_CHUNK 64 /* a refined node's far sum: chunks of 64 far entries, chunk sums added in order */
/* Interaction table (octant-0 orientation, (z, y, x) lexicographic over
 * [-K, K]^3 without 0): depth >= 1 (root = 0): K = 2R+1, parent offset
 * (u >> 1) within R; depth 0 (root = 1): K = 7, all.  near[k] = |u|^2 <= R^2. */
int orc_fmm_table(int radius, int root, int32_t* u, int32_t* near, int cap);
int orc_gravity_fmm(int nf, int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                    double dx0, const double* U, int radius, double G, double* out);
/* The gravity source over dt (operator split after the hydro step, the
 * reference's order: 3 hydro rounds, then the gravity launches,
 * workload.cpp:559-569): per cell S' = fma(dt, rho g, S) per component and
 * E' = fma(dt/2, (S + S') . g, E) (the work of the mean momentum; the dot
 * product as (Sx+Sx')gx, then fma y, fma z).  grav = [n][4][512]. */
void orc_gravity_kick(int nf, int64_t n, double* U, const double* grav, double dt);
/* Brute force over every pair of leaf cells (monopoles at the centres): the
 * accuracy yardstick of the FMM, not a parity target. */
int orc_gravity_direct(int nf, int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                       double dx0, const double* U, double G, double* out);

#ifdef __cplusplus
}
#endif

#endif
