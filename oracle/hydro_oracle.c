/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see hydro_oracle.h).
 *
 * Deliberately literal, scalar, per-pencil C.  It shares no code with the
 * CUDA path; the two agree bitwise because both follow the same operation
 * order (explicit fma() where the numerics contract in DESIGN.md §2 says
 * fma, IEEE division and square root, no contraction: build with
 * -ffp-contract=off).
 */
#include "hydro_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define N ORC_N
#define NC ORC_NC
#define P (N + 6) /* pencil length: 3 ghosts each side */

static const double C16 = 1.0 / 6.0;
static const double C13 = 1.0 / 3.0;
static const double C23 = 2.0 / 3.0;

/* ---------------------------------------------------------------------------
 * Reference data model
 * ------------------------------------------------------------------------- */

/* splitmix64 finaliser, reference proj/core/include/taskscope/sampling.hpp:12-18 */
uint64_t orc_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* sampling.hpp:20-22 */
uint64_t orc_mix64_2(uint64_t a, uint64_t b) { return orc_mix64(a ^ orc_mix64(b)); }

/* workload.cpp:329-332 */
double orc_cell_value(uint64_t grid_id, uint64_t step, uint64_t index) {
    const uint64_t h = orc_mix64_2(orc_mix64_2(grid_id, step), index);
    return (double)(h >> 11) * 0x1.0p-53;
}

/* workload.cpp:340-354 */
uint64_t orc_face_cell_index(int edge, int face, uint64_t j) {
    const uint64_t e = (uint64_t)edge;
    const uint64_t plane = (face & 1) ? e - 1 : 0;
    const uint64_t u = j % e, v = j / e;
    uint64_t x, y, z;
    switch (face / 2) {
        case 0: x = plane; y = u; z = v; break;
        case 1: x = u; y = plane; z = v; break;
        default: x = u; y = v; z = plane; break;
    }
    return x + e * (y + e * z);
}

/* workload.cpp:252-261 */
uint64_t orc_morton3(uint32_t x, uint32_t y, uint32_t z) {
    uint64_t out = 0;
    for (int b = 0; b < 21; ++b) {
        out |= (uint64_t)((x >> b) & 1u) << (3 * b);
        out |= (uint64_t)((y >> b) & 1u) << (3 * b + 1);
        out |= (uint64_t)((z >> b) & 1u) << (3 * b + 2);
    }
    return out;
}

typedef struct {
    uint64_t key;
    int32_t x, y, z;
} orc_mkey;

static int cmp_mkey(const void* a, const void* b) {
    const orc_mkey* p = (const orc_mkey*)a;
    const orc_mkey* q = (const orc_mkey*)b;
    return (p->key > q->key) - (p->key < q->key);
}

/* Hand-built uniform mesh (the shape make_row_mesh builds in the reference's
 * tests, test_workload.cpp:38-54), numbered along the Morton curve and dealt
 * to ranks in contiguous chunks exactly like build_mesh (workload.cpp:298-323). */
int orc_uniform_mesh(int nx, int ny, int nz, int px, int py, int pz, int world, int64_t* nbr,
                     int32_t* pos, int32_t* owner) {
    if (nx < 1 || ny < 1 || nz < 1 || world < 1) return -1;
    const int64_t n = (int64_t)nx * ny * nz;
    orc_mkey* keys = (orc_mkey*)malloc(sizeof(orc_mkey) * (size_t)n);
    int64_t* id_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)n); /* lexicographic -> id */
    int64_t k = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                keys[k].key = orc_morton3((uint32_t)x, (uint32_t)y, (uint32_t)z);
                keys[k].x = x;
                keys[k].y = y;
                keys[k].z = z;
                ++k;
            }
    qsort(keys, (size_t)n, sizeof(orc_mkey), cmp_mkey);
    for (int64_t g = 0; g < n; ++g) {
        pos[3 * g + 0] = keys[g].x;
        pos[3 * g + 1] = keys[g].y;
        pos[3 * g + 2] = keys[g].z;
        id_of[((int64_t)keys[g].z * ny + keys[g].y) * nx + keys[g].x] = g;
    }
    const int dims[3] = {nx, ny, nz};
    const int per[3] = {px, py, pz};
    for (int64_t g = 0; g < n; ++g) {
        for (int face = 0; face < 6; ++face) {
            int c[3] = {pos[3 * g], pos[3 * g + 1], pos[3 * g + 2]};
            const int axis = face / 2;
            c[axis] += (face & 1) ? 1 : -1;
            int64_t nb = -1;
            if (c[axis] < 0 || c[axis] >= dims[axis]) {
                if (per[axis]) {
                    c[axis] = (c[axis] + dims[axis]) % dims[axis];
                    nb = id_of[((int64_t)c[2] * ny + c[1]) * nx + c[0]];
                }
            } else {
                nb = id_of[((int64_t)c[2] * ny + c[1]) * nx + c[0]];
            }
            nbr[6 * g + face] = nb;
        }
    }
    const int64_t base = n / world, extra = n % world;
    int64_t cursor = 0;
    for (int r = 0; r < world; ++r) {
        const int64_t count = base + (r < extra ? 1 : 0);
        for (int64_t j = 0; j < count; ++j) owner[cursor++] = r;
    }
    free(keys);
    free(id_of);
    return 0;
}

/* workload.cpp:519-542 (both comm modes yield these values, test_workload.cpp:317-331) */
void orc_exchange_faces(int nf, int64_t ngrids, const int64_t* nbr, const double* U, double* ghost) {
    for (int64_t g = 0; g < ngrids; ++g)
        for (int face = 0; face < 6; ++face) {
            const int64_t h = nbr[6 * g + face];
            for (uint64_t j = 0; j < N * N; ++j)
                ghost[(g * 6 + face) * N * N + (int64_t)j] =
                    h < 0 ? 0.0 : U[(h * nf) * NC + (int64_t)orc_face_cell_index(N, face ^ 1, j)];
        }
}

/* Resolve a cell of the padded cube: walk across faces axis by axis; a missing
 * neighbour clamps the coordinate (outflow). */
static double padded_value(int nf, const int64_t* nbr, const double* U, int64_t g, int f, int x,
                           int y, int z) {
    int c[3] = {x, y, z};
    int64_t h = g;
    for (int axis = 0; axis < 3; ++axis) {
        if (c[axis] < 0) {
            const int64_t nb = nbr[6 * h + 2 * axis];
            if (nb >= 0) {
                h = nb;
                c[axis] += N;
            } else {
                c[axis] = 0;
            }
        } else if (c[axis] >= N) {
            const int64_t nb = nbr[6 * h + 2 * axis + 1];
            if (nb >= 0) {
                h = nb;
                c[axis] -= N;
            } else {
                c[axis] = N - 1;
            }
        }
    }
    return U[(h * nf + f) * NC + (c[2] * N + c[1]) * N + c[0]];
}

void orc_fill_halo(int nf, int64_t ngrids, const int64_t* nbr, const double* U, int h, double* tiles) {
    const int pe = N + 2 * h;
    const int64_t tile = (int64_t)pe * pe * pe;
    for (int64_t g = 0; g < ngrids; ++g)
        for (int f = 0; f < nf; ++f)
            for (int z = 0; z < pe; ++z)
                for (int y = 0; y < pe; ++y)
                    for (int x = 0; x < pe; ++x)
                        tiles[(g * nf + f) * tile + ((int64_t)z * pe + y) * pe + x] =
                            padded_value(nf, nbr, U, g, f, x - h, y - h, z - h);
}

/* ---------------------------------------------------------------------------
 * Reconstruction (Octo-Tiger's PPM, applied dimension by dimension)
 * ------------------------------------------------------------------------- */

/* Octo-Tiger minmod / minmod_theta (MC limiter with theta = 2). */
static double minmod(double a, double b) {
    return (copysign(0.5, a) + copysign(0.5, b)) * fmin(fabs(a), fabs(b));
}

static double minmod_theta(double a, double b, double theta) {
    return minmod(theta * minmod(a, b), 0.5 * (a + b));
}

/* Colella & Woodward (1984) eq. 1.10 monotonicity step in Octo-Tiger's form. */
static void limit_slope(double* ql, double q0, double* qr) {
    if ((*qr < q0) != (q0 < *ql)) {
        *ql = q0;
        *qr = q0;
        return;
    }
    const double t1 = *qr - *ql;
    const double t2 = *qr + *ql;
    const double t3 = (t1 * t1) * C16;
    const double t4 = t1 * (q0 - 0.5 * t2);
    if (t4 > t3) {
        *ql = fma(-2.0, *qr, 3.0 * q0);
    } else if (-t3 > t4) {
        *qr = fma(-2.0, *ql, 3.0 * q0);
    }
}

/* q[0..P-1] holds cells -3..N+2 of one pencil.  Returns the face states of the
 * N+1 faces of the interior: face j sits between cells j-1 and j;
 * uL[j] = right edge of cell j-1, uR[j] = left edge of cell j. */
static void reconstruct(int recon, const double* q, double* uL, double* uR) {
    double lo[P], hi[P];
    if (recon == 0) {
        double D[P], fc[P];
        for (int i = 1; i <= P - 2; ++i) D[i] = minmod_theta(q[i + 1] - q[i], q[i] - q[i - 1], 2.0);
        /* fc[i]: face between array cells i-1 and i */
        for (int i = 2; i <= P - 2; ++i) fc[i] = fma(C16, D[i - 1] - D[i], 0.5 * (q[i - 1] + q[i]));
        for (int i = 2; i <= P - 3; ++i) {
            double ql = fc[i], qr = fc[i + 1];
            limit_slope(&ql, q[i], &qr);
            lo[i] = ql;
            hi[i] = qr;
        }
    } else {
        for (int i = 2; i <= P - 3; ++i) {
            const double s = minmod(q[i + 1] - q[i], q[i] - q[i - 1]);
            lo[i] = fma(-0.5, s, q[i]);
            hi[i] = fma(0.5, s, q[i]);
        }
    }
    for (int j = 0; j <= N; ++j) {
        uL[j] = hi[j + 2]; /* cell j-1 lives at array index j+2 */
        uR[j] = lo[j + 3];
    }
}

/* ---------------------------------------------------------------------------
 * Kurganov–Tadmor central flux
 * ------------------------------------------------------------------------- */

/* Physical flux of one face state along `axis` plus its normal velocity and
 * local signal speed |v_n| + c.  Ideal gas, pressure floor. */
static void side_flux(const orc_params* p, int axis, const double* u, double* f, double* vn,
                      double* c2) {
    const double rho = u[0], sx = u[1], sy = u[2], sz = u[3], E = u[4];
    const double inv = 1.0 / rho;
    const double vx = sx * inv, vy = sy * inv, vz = sz * inv;
    /* |s|^2/rho summed normal component first, then the two transverse ones
     * in x, y, z order: the same expression for every sweep direction */
    const double s3[3] = {sx, sy, sz}, v3[3] = {vx, vy, vz};
    const int t1 = axis == 0 ? 1 : 0, t2 = axis == 2 ? 1 : 2;
    const double ke2 = fma(s3[axis], v3[axis], fma(s3[t1], v3[t1], s3[t2] * v3[t2]));
    double pr = (p->gamma - 1.0) * fma(-0.5, ke2, E);
    pr = fmax(pr, p->p_floor);
    const double v = v3[axis];
    *c2 = (p->gamma * pr) * inv; /* squared sound speed (gamma p / rho) */
    *vn = v;
    f[0] = u[1 + axis];
    f[1] = sx * v;
    f[2] = sy * v;
    f[3] = sz * v;
    f[1 + axis] = fma(u[1 + axis], v, pr);
    f[4] = (E + pr) * v;
    for (int k = 5; k < p->nf; ++k) f[k] = u[k] * v;
}

static void kt_flux(const orc_params* p, int axis, const double* uL, const double* uR, double* F) {
    double fL[16], fR[16], vL, vR, c2L, c2R;
    side_flux(p, axis, uL, fL, &vL, &c2L);
    side_flux(p, axis, uR, fR, &vR, &c2R);
    /* Davis wave-speed bound max(|v_L|, |v_R|) + max(c_L, c_R); sqrt is
     * monotone and correctly rounded, so sqrt(max(c2_L, c2_R)) is exactly
     * max(c_L, c_R) with one square root per face (DESIGN.md §2 item 3) */
    const double a = fmax(fabs(vL), fabs(vR)) + sqrt(fmax(c2L, c2R));
    for (int k = 0; k < p->nf; ++k) F[k] = 0.5 * fma(-a, uR[k] - uL[k], fL[k] + fR[k]);
}

/* ---------------------------------------------------------------------------
 * One RK stage
 * ------------------------------------------------------------------------- */

static inline int64_t cidx(int x, int y, int z) { return ((int64_t)z * N + y) * N + x; }

/* Value of pencil cell `s` (-3..N+2) along `axis` through (a, b) of sub-grid g:
 * ghosts are read straight from the face neighbour's interior (the reference's
 * direct_local path, workload.cpp:532-536) or clamp at a domain boundary. */
static double pencil_value(int nf, const int64_t* nbr, const double* U, int64_t g, int f, int axis,
                           int a, int b, int s) {
    int64_t h = g;
    if (s < 0) {
        const int64_t nb = nbr[6 * g + 2 * axis];
        if (nb >= 0) {
            h = nb;
            s += N;
        } else {
            s = 0;
        }
    } else if (s >= N) {
        const int64_t nb = nbr[6 * g + 2 * axis + 1];
        if (nb >= 0) {
            h = nb;
            s -= N;
        } else {
            s = N - 1;
        }
    }
    int64_t c;
    if (axis == 0)
        c = cidx(s, a, b);
    else if (axis == 1)
        c = cidx(a, s, b);
    else
        c = cidx(a, b, s);
    return U[(h * nf + f) * NC + c];
}

void orc_stage(const orc_params* p, int64_t ngrids, const int64_t* nbr, const double* Uprev,
               const double* Un, double* Uout, int stage, double dtdx, int64_t g_begin,
               int64_t g_end) {
    (void)ngrids;
    const int nf = p->nf;
    double* dU = (double*)malloc(sizeof(double) * (size_t)nf * NC);
    double q[16][P], uL[16][N + 1], uR[16][N + 1], F[N + 1][16];
    double sL[16], sR[16];
    for (int64_t g = g_begin; g < g_end; ++g) {
        for (int axis = 0; axis < 3; ++axis) {
            for (int b = 0; b < N; ++b)
                for (int a = 0; a < N; ++a) {
                    for (int f = 0; f < nf; ++f) {
                        for (int s = 0; s < P; ++s)
                            q[f][s] = pencil_value(nf, nbr, Uprev, g, f, axis, a, b, s - 3);
                        reconstruct(p->recon, q[f], uL[f], uR[f]);
                    }
                    for (int j = 0; j <= N; ++j) {
                        for (int f = 0; f < nf; ++f) {
                            sL[f] = uL[f][j];
                            sR[f] = uR[f][j];
                        }
                        kt_flux(p, axis, sL, sR, F[j]);
                    }
                    for (int i = 0; i < N; ++i) {
                        int64_t c;
                        if (axis == 0)
                            c = cidx(i, a, b);
                        else if (axis == 1)
                            c = cidx(a, i, b);
                        else
                            c = cidx(a, b, i);
                        for (int f = 0; f < nf; ++f) {
                            const double d = F[i][f] - F[i + 1][f];
                            dU[f * NC + c] = axis == 0 ? d : dU[f * NC + c] + d;
                        }
                    }
                }
        }
        for (int f = 0; f < nf; ++f)
            for (int c = 0; c < NC; ++c) {
                const int64_t at = (g * nf + f) * NC + c;
                const double ustar = fma(dtdx, dU[f * NC + c], Uprev[at]);
                double out;
                if (stage == 1)
                    out = ustar;
                else if (stage == 2)
                    out = fma(0.75, Un[at], 0.25 * ustar);
                else
                    out = fma(C13, Un[at], C23 * ustar);
                Uout[at] = out;
            }
    }
    free(dU);
}

/* Cell-centred CFL signal speed max_d |v_d| + c, maximised over cells. */
double orc_max_signal_speed(const orc_params* p, int64_t g_begin, int64_t g_end, const double* U) {
    const int nf = p->nf;
    double amax = 0.0;
    for (int64_t g = g_begin; g < g_end; ++g)
        for (int c = 0; c < NC; ++c) {
            const double* u = U + g * nf * NC + c;
            const double rho = u[0], sx = u[NC], sy = u[2 * NC], sz = u[3 * NC], E = u[4 * NC];
            const double inv = 1.0 / rho;
            const double vx = sx * inv, vy = sy * inv, vz = sz * inv;
            const double ke2 = fma(sx, vx, fma(sy, vy, sz * vz));
            double pr = (p->gamma - 1.0) * fma(-0.5, ke2, E);
            pr = fmax(pr, p->p_floor);
            const double cs = sqrt((p->gamma * pr) * inv);
            const double a = fmax(fmax(fabs(vx), fabs(vy)), fabs(vz)) + cs;
            amax = fmax(amax, a);
        }
    return amax;
}

/* ---------------------------------------------------------------------------
 * Stepping driver (threads split sub-grid ranges; results are independent of
 * the split because every sub-grid's stage is a pure function of its inputs)
 * ------------------------------------------------------------------------- */

typedef struct {
    const orc_params* p;
    int64_t ngrids;
    const int64_t* nbr;
    const double* Uprev;
    const double* Un;
    double* Uout;
    int stage;
    double dtdx;
    int64_t g0, g1;
    double amax;
} orc_job;

static void* stage_job(void* arg) {
    orc_job* j = (orc_job*)arg;
    if (j->stage == 0)
        j->amax = orc_max_signal_speed(j->p, j->g0, j->g1, j->Uprev);
    else
        orc_stage(j->p, j->ngrids, j->nbr, j->Uprev, j->Un, j->Uout, j->stage, j->dtdx, j->g0, j->g1);
    return NULL;
}

static double run_parallel(const orc_params* p, int64_t ngrids, const int64_t* nbr,
                           const double* Uprev, const double* Un, double* Uout, int stage,
                           double dtdx, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > ngrids) nthreads = (int)(ngrids > 0 ? ngrids : 1);
    orc_job jobs[256];
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (orc_job){p, ngrids, nbr, Uprev, Un, Uout, stage, dtdx,
                            ngrids * t / nthreads, ngrids * (t + 1) / nthreads, 0.0};
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, stage_job, &jobs[t]);
    stage_job(&jobs[0]);
    double amax = jobs[0].amax;
    for (int t = 1; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        amax = fmax(amax, jobs[t].amax);
    }
    return amax;
}

int orc_run(const orc_params* p, int64_t ngrids, const int64_t* nbr, double* U, int nsteps,
            double* dt_hist, int nthreads) {
    const size_t bytes = sizeof(double) * (size_t)ngrids * (size_t)p->nf * NC;
    double* U1 = (double*)malloc(bytes);
    double* U2 = (double*)malloc(bytes);
    if (!U1 || !U2) {
        free(U1);
        free(U2);
        return -1;
    }
    for (int s = 0; s < nsteps; ++s) {
        const double amax = run_parallel(p, ngrids, nbr, U, NULL, NULL, 0, 0.0, nthreads);
        const double dt = (p->cfl * p->dx) / amax;
        const double dtdx = dt / p->dx;
        if (dt_hist) dt_hist[s] = dt;
        run_parallel(p, ngrids, nbr, U, U, U1, 1, dtdx, nthreads);
        run_parallel(p, ngrids, nbr, U1, U, U2, 2, dtdx, nthreads);
        run_parallel(p, ngrids, nbr, U2, U, U, 3, dtdx, nthreads);
    }
    free(U1);
    free(U2);
    return 0;
}

void orc_field_sums(int nf, int64_t ngrids, const double* U, double* sums) {
    for (int f = 0; f < nf; ++f) sums[f] = 0.0;
    for (int64_t g = 0; g < ngrids; ++g)
        for (int f = 0; f < nf; ++f)
            for (int c = 0; c < NC; ++c) sums[f] += U[(g * nf + f) * NC + c];
}

/* ---------------------------------------------------------------------------
 * Initial conditions
 * ------------------------------------------------------------------------- */

static void set_cell(const orc_params* p, double* U, int64_t g, int c, double rho, double vx,
                     double vy, double vz, double pr, double extra_e) {
    const int nf = p->nf;
    const double eint = pr / (p->gamma - 1.0);
    const double v2 = fma(vx, vx, fma(vy, vy, vz * vz));
    double* u = U + g * nf * NC + c;
    u[0] = rho;
    u[NC] = rho * vx;
    u[2 * NC] = rho * vy;
    u[3 * NC] = rho * vz;
    u[4 * NC] = fma(0.5 * rho, v2, eint) + extra_e;
    u[5 * NC] = pow(eint + extra_e, 1.0 / p->gamma);
    for (int k = 6; k < nf; ++k) u[k * NC] = 0.0;
}

void orc_ic_sod(const orc_params* p, int64_t ngrids, const int32_t* pos, int axis, double* U) {
    /* domain: ncell = (max pos + 1) * N along axis */
    int32_t maxp = 0;
    for (int64_t g = 0; g < ngrids; ++g)
        if (pos[3 * g + axis] > maxp) maxp = pos[3 * g + axis];
    const int64_t ncell = (int64_t)(maxp + 1) * N;
    for (int64_t g = 0; g < ngrids; ++g)
        for (int z = 0; z < N; ++z)
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) {
                    const int lc[3] = {x, y, z};
                    const int64_t ci = (int64_t)pos[3 * g + axis] * N + lc[axis];
                    const int left = 2 * ci + 1 < ncell;
                    set_cell(p, U, g, (int)cidx(x, y, z), left ? 1.0 : 0.125, 0.0, 0.0, 0.0,
                             left ? 1.0 : 0.1, 0.0);
                }
}

void orc_ic_sedov(const orc_params* p, int64_t ngrids, const int32_t* pos, int nx, int ny, int nz,
                  double* U) {
    const int64_t nc[3] = {(int64_t)nx * N, (int64_t)ny * N, (int64_t)nz * N};
    const double e_cell = 1.0 / (8.0 * p->dx * p->dx * p->dx);
    for (int64_t g = 0; g < ngrids; ++g)
        for (int z = 0; z < N; ++z)
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) {
                    const int lc[3] = {x, y, z};
                    int centre = 1;
                    for (int d = 0; d < 3; ++d) {
                        const int64_t ci = (int64_t)pos[3 * g + d] * N + lc[d];
                        if (!(ci == nc[d] / 2 - 1 || ci == nc[d] / 2)) centre = 0;
                    }
                    set_cell(p, U, g, (int)cidx(x, y, z), 1.0, 0.0, 0.0, 0.0, 1e-5,
                             centre ? e_cell : 0.0);
                }
}

/* Smooth-random state from the reference generator cell_value
 * (workload.cpp:329-332): r_k = cell_value(grid, seed, k*512 + cell). */
void orc_ic_random(const orc_params* p, int64_t g_begin, int64_t g_end, uint64_t seed, double* U) {
    const int nf = p->nf;
    for (int64_t g = g_begin; g < g_end; ++g)
        for (int c = 0; c < NC; ++c) {
            double r[16];
            for (int k = 0; k < nf; ++k) r[k] = orc_cell_value((uint64_t)g, seed, (uint64_t)k * NC + (uint64_t)c);
            const double rho = 0.5 + r[0];
            const double vx = r[1] - 0.5, vy = r[2] - 0.5, vz = r[3] - 0.5;
            const double pr = 0.5 + r[4];
            const double v2 = fma(vx, vx, fma(vy, vy, vz * vz));
            double* u = U + (g - g_begin) * nf * NC + c;
            u[0] = rho;
            u[NC] = rho * vx;
            u[2 * NC] = rho * vy;
            u[3 * NC] = rho * vz;
            u[4 * NC] = fma(0.5 * rho, v2, pr / (p->gamma - 1.0));
            u[5 * NC] = 0.5 + r[5];
            for (int k = 6; k < nf; ++k) u[k * NC] = rho * r[k];
        }
}

/* BASELINE configs 3 and 4: the rotating n = 1 polytrope (one star per cubic
 * block of T = min(dims) sub-grids: the weak-scaling tile) with 5 radial-shell
 * species, and the V1309-like contact binary (two n = 1.5 polytropes,
 * q ~ 0.1, co-rotating, 1e-5 rho_c pressure-matched atmosphere, species =
 * the two stars' densities).  Same formulas and operation order as the
 * product's initial-model generator (so the bench's CPU arm needs nothing of
 * the product); tests/test_oracle.py checks the two agree bitwise. */
typedef struct {
    double* theta;
    int64_t n;
    double h, xi1;
} lane_emden;

static double le_rhs(double nidx, double x, double t, double dt) {
    const double tp = t > 0.0 ? pow(t, nidx) : 0.0;
    return -tp - 2.0 / x * dt;
}

/* theta(xi) of index n by RK4 (step 1e-4) to the first zero */
static int le_init(lane_emden* le, double nidx) {
    const double h = 1e-4;
    int64_t cap = 1 << 16, n = 0;
    double* th_tab = (double*)malloc((size_t)cap * sizeof(double));
    if (th_tab == NULL) return -1;
    double xi = 1e-6, th = 1.0 - xi * xi / 6.0, dth = -xi / 3.0;
    th_tab[n++] = 1.0;
    while (th > 0.0 && xi < 20.0) {
        const double a1 = le_rhs(nidx, xi, th, dth);
        const double t1 = th + 0.5 * h * dth, d1 = dth + 0.5 * h * a1;
        const double a2 = le_rhs(nidx, xi + 0.5 * h, t1, d1);
        const double t2 = th + 0.5 * h * d1, d2 = dth + 0.5 * h * a2;
        const double a3 = le_rhs(nidx, xi + 0.5 * h, t2, d2);
        const double t3 = th + h * d2, d3 = dth + h * a3;
        const double a4 = le_rhs(nidx, xi + h, t3, d3);
        th += h / 6.0 * (dth + 2 * d1 + 2 * d2 + d3);
        dth += h / 6.0 * (a1 + 2 * a2 + 2 * a3 + a4);
        xi += h;
        if (n == cap) {
            cap *= 2;
            double* nt = (double*)realloc(th_tab, (size_t)cap * sizeof(double));
            if (nt == NULL) {
                free(th_tab);
                return -1;
            }
            th_tab = nt;
        }
        th_tab[n++] = th > 0.0 ? th : 0.0;
    }
    le->theta = th_tab;
    le->n = n;
    le->h = h;
    le->xi1 = xi;
    return 0;
}

static double le_eval(const lane_emden* le, double xi) {
    if (xi >= le->xi1) return 0.0;
    const double k = xi / le->h;
    const size_t i = (size_t)k;
    if ((int64_t)i + 1 >= le->n) return 0.0;
    const double fr = k - (double)i;
    return le->theta[i] * (1.0 - fr) + le->theta[i + 1] * fr;
}

static void set_cell_species(const orc_params* p, double* U, int64_t g, int c, double rho, double vx, double vy,
                             double pr, const double* species) {
    set_cell(p, U, g, c, rho, vx, vy, 0.0, pr, 0.0);
    for (int k = 6; k < p->nf; ++k) U[g * p->nf * NC + (int64_t)k * NC + c] = (k - 6) < 5 ? species[k - 6] : 0.0;
}

void orc_ic_polytrope(const orc_params* p, int64_t ngrids, const int32_t* pos, int nx, int ny, int nz, double* U) {
    const double kPi = 3.14159265358979323846;
    const int T = nx < ny ? (nx < nz ? nx : nz) : (ny < nz ? ny : nz);
    const double Lb = T * N * p->dx;
    const double R = 0.4 * 0.5 * Lb;
    for (int64_t g = 0; g < ngrids; ++g)
        for (int z = 0; z < N; ++z)
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) {
                    const int lc[3] = {x, y, z};
                    double rr[3];
                    for (int d = 0; d < 3; ++d) {
                        const double xc = ((double)((int64_t)pos[3 * g + d] * N + lc[d]) + 0.5) * p->dx;
                        const double b = floor(xc / Lb);
                        rr[d] = xc - (b + 0.5) * Lb;
                    }
                    const double r = sqrt(rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2]);
                    const double xi = kPi * r / R;
                    const double th = r < R ? (xi > 1e-12 ? sin(xi) / xi : 1.0) : 0.0;
                    const double rho = th > 1e-10 ? th : 1e-10;
                    double sp[5] = {0, 0, 0, 0, 0}, vx = 0.0, vy = 0.0;
                    if (r < R) {
                        vx = -0.1 * rr[1];
                        vy = 0.1 * rr[0];
                        int shell = (int)(5.0 * r / R);
                        if (shell > 4) shell = 4;
                        sp[shell] = rho;
                    }
                    set_cell_species(p, U, g, (int)cidx(x, y, z), rho, vx, vy, rho * rho, sp);
                }
}

int orc_ic_binary(const orc_params* p, int64_t ngrids, const int32_t* pos, int nx, int ny, int nz, double* U) {
    lane_emden le;
    if (le_init(&le, 1.5) != 0) return -1;
    const double L[3] = {(double)nx * N * p->dx, (double)ny * N * p->dx, (double)nz * N * p->dx};
    const double R1 = 0.22 * L[0], R2 = 0.5 * R1;
    const double sep = R1 + R2;
    const double rc1 = 1.0, rc2 = 0.8;
    const double m1 = rc1 * R1 * R1 * R1, m2 = rc2 * R2 * R2 * R2;
    const double cxm = 0.5 * L[0], cy = 0.5 * L[1], cz = 0.5 * L[2];
    const double x1 = cxm - sep * m2 / (m1 + m2), x2 = cxm + sep * m1 / (m1 + m2);
    const double amb = 1e-5;
    for (int64_t g = 0; g < ngrids; ++g)
        for (int z = 0; z < N; ++z)
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) {
                    const double px = ((double)((int64_t)pos[3 * g] * N + x) + 0.5) * p->dx;
                    const double py = ((double)((int64_t)pos[3 * g + 1] * N + y) + 0.5) * p->dx;
                    const double pz = ((double)((int64_t)pos[3 * g + 2] * N + z) + 0.5) * p->dx;
                    const double r1 = sqrt((px - x1) * (px - x1) + (py - cy) * (py - cy) + (pz - cz) * (pz - cz));
                    const double r2 = sqrt((px - x2) * (px - x2) + (py - cy) * (py - cy) + (pz - cz) * (pz - cz));
                    const double t1 = le_eval(&le, le.xi1 * r1 / R1), t2 = le_eval(&le, le.xi1 * r2 / R2);
                    const double d1 = rc1 * pow(t1, 1.5), d2 = rc2 * pow(t2, 1.5);
                    const double rho = d1 + d2 > amb ? d1 + d2 : amb;
                    double vx = 0.0, vy = 0.0;
                    if (d1 + d2 > amb) {
                        vx = -0.1 * (py - cy);
                        vy = 0.1 * (px - cxm);
                    }
                    const double sp[5] = {d1, d2, 0.0, 0.0, 0.0};
                    set_cell_species(p, U, g, (int)cidx(x, y, z), rho, vx, vy, pow(rho, 5.0 / 3.0), sp);
                }
    free(le.theta);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Coarse-fine AMR.  The reference's octree
 * (build_mesh, workload.cpp:264-327) refines by octants and links only
 * same-level faces (validate, workload.cpp:160-161); Octo-Tiger fills
 * coarse-fine ghosts by prolongation / restriction and corrects the coarse
 * fluxes at the interface.  Restated here with one global dt,
 * 2:1 balanced leaves, piecewise-constant prolongation, volume-mean
 * restriction and a flux correction with the RK stage weight.
 * ------------------------------------------------------------------------- */

void orc_amr_fill(int nf, int64_t n_proxy, const orc_amr_proxy* px, double* U) {
    for (int64_t k = 0; k < n_proxy; ++k) {
        const orc_amr_proxy* r = &px[k];
        for (int z = 0; z < N; ++z)
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) {
                    const int c = (int)cidx(x, y, z);
                    for (int f = 0; f < nf; ++f) {
                        double v;
                        if (r->kind == 0) {
                            const int cx = (r->octant & 1) * 4 + x / 2;
                            const int cy = ((r->octant >> 1) & 1) * 4 + y / 2;
                            const int cz = ((r->octant >> 2) & 1) * 4 + z / 2;
                            v = U[((int64_t)r->src[0] * nf + f) * NC + cidx(cx, cy, cz)];
                        } else {
                            const int o = (x >> 2) | ((y >> 2) << 1) | ((z >> 2) << 2);
                            const double* s = U + ((int64_t)r->src[o] * nf + f) * NC;
                            const int bx = 2 * (x & 3), by = 2 * (y & 3), bz = 2 * (z & 3);
                            double sum = s[cidx(bx, by, bz)];
                            sum = sum + s[cidx(bx + 1, by, bz)];
                            sum = sum + s[cidx(bx, by + 1, bz)];
                            sum = sum + s[cidx(bx + 1, by + 1, bz)];
                            sum = sum + s[cidx(bx, by, bz + 1)];
                            sum = sum + s[cidx(bx + 1, by, bz + 1)];
                            sum = sum + s[cidx(bx, by + 1, bz + 1)];
                            sum = sum + s[cidx(bx + 1, by + 1, bz + 1)];
                            v = 0.125 * sum;
                        }
                        U[((int64_t)r->dst * nf + f) * NC + c] = v;
                    }
                }
    }
}

/* The KT flux of face j (0..N) of pencil (a, b) along `axis` of sub-grid g:
 * the value orc_stage computes as F[j] for that pencil. */
static void face_flux(const orc_params* p, const int64_t* nbr, const double* U, int64_t g, int axis, int a,
                      int b, int j, double* F) {
    double q[P], uL[N + 1], uR[N + 1], sL[16], sR[16];
    for (int f = 0; f < p->nf; ++f) {
        for (int s = 0; s < P; ++s) q[s] = pencil_value(p->nf, nbr, U, g, f, axis, a, b, s - 3);
        reconstruct(p->recon, q, uL, uR);
        sL[f] = uL[j];
        sR[f] = uR[j];
    }
    kt_flux(p, axis, sL, sR, F);
}

void orc_amr_reflux(const orc_params* p, const int64_t* nbr, const int32_t* level, int max_level,
                    int64_t n_rec, const orc_amr_reflux_rec* rf, const double* Uprev, double* Uout, int stage,
                    double dt) {
    const int nf = p->nf;
    const double w = stage == 1 ? 1.0 : (stage == 2 ? 0.25 : C23);
    double Fc[16], F00[16], F10[16], F01[16], F11[16];
    for (int64_t r = 0; r < n_rec; ++r) {
        const int64_t g = rf[r].coarse;
        const double dtdx = dt / ldexp(p->dx, max_level - level[g]);
        for (int face = 0; face < 6; ++face) {
            if (rf[r].fine[face][0] < 0) continue;
            const int axis = face >> 1, side = face & 1;
            const int jc = side ? N : 0, jf = side ? 0 : N, ic = side ? N - 1 : 0;
            for (int b = 0; b < N; ++b)
                for (int a = 0; a < N; ++a) {
                    const int64_t leaf = rf[r].fine[face][(a >> 2) + 2 * (b >> 2)];
                    const int fa = 2 * (a & 3), fb = 2 * (b & 3);
                    face_flux(p, nbr, Uprev, g, axis, a, b, jc, Fc);
                    face_flux(p, nbr, Uprev, leaf, axis, fa, fb, jf, F00);
                    face_flux(p, nbr, Uprev, leaf, axis, fa + 1, fb, jf, F10);
                    face_flux(p, nbr, Uprev, leaf, axis, fa, fb + 1, jf, F01);
                    face_flux(p, nbr, Uprev, leaf, axis, fa + 1, fb + 1, jf, F11);
                    const int64_t c = axis == 0 ? cidx(ic, a, b) : (axis == 1 ? cidx(a, ic, b) : cidx(a, b, ic));
                    for (int f = 0; f < nf; ++f) {
                        const double avg = 0.25 * ((F00[f] + F10[f]) + (F01[f] + F11[f]));
                        const double corr = side ? Fc[f] - avg : avg - Fc[f];
                        double* u = Uout + (g * nf + f) * NC + c;
                        *u = *u + w * (dtdx * corr);
                    }
                }
        }
    }
}

int orc_run_amr(const orc_params* p, int64_t n_total, const int64_t* nbr, const int32_t* level,
                const int64_t* level_first, int max_level, int64_t n_proxy, const orc_amr_proxy* px,
                int64_t n_rec, const orc_amr_reflux_rec* rf, double* U, int nsteps, double* dt_hist) {
    const size_t bytes = sizeof(double) * (size_t)n_total * (size_t)p->nf * NC;
    double* U1 = (double*)calloc(1, bytes);
    double* U2 = (double*)calloc(1, bytes);
    if (!U1 || !U2) {
        free(U1);
        free(U2);
        return -1;
    }
    const int64_t n_leaves = level_first[max_level + 1];
    for (int s = 0; s < nsteps; ++s) {
        const double amax = orc_max_signal_speed(p, 0, n_leaves, U);
        const double dt = (p->cfl * p->dx) / amax;
        if (dt_hist) dt_hist[s] = dt;
        double* in[3] = {U, U1, U2};
        double* out[3] = {U1, U2, U};
        for (int k = 1; k <= 3; ++k) {
            orc_amr_fill(p->nf, n_proxy, px, in[k - 1]);
            for (int L = 0; L <= max_level; ++L)
                orc_stage(p, n_total, nbr, in[k - 1], U, out[k - 1], k, dt / ldexp(p->dx, max_level - L),
                          level_first[L], level_first[L + 1]);
            orc_amr_reflux(p, nbr, level, max_level, n_rec, rf, in[k - 1], out[k - 1], k, dt);
        }
    }
    free(U1);
    free(U2);
    return 0;
}

/* Diagnostics: the N+1 face fluxes F[j][f] of pencil (a, b) along `axis` of
 * sub-grid g, exactly as orc_stage computes them. */
void orc_debug_face_fluxes(const orc_params* p, const int64_t* nbr, const double* U, int64_t g, int axis, int a,
                           int b, double* F) {
    for (int j = 0; j <= N; ++j) face_flux(p, nbr, U, g, axis, a, b, j, F + (size_t)j * p->nf);
}

/* ---------------------------------------------------------------------------
 * Gravity, near-field monopole P2P (hydro_oracle.h).  The reference launches
 * p2p_kernel for leaves without refined neighbours (gravity_kernel_name,
 * workload.cpp:365-372) and only sleeps; Octo-Tiger computes the cell-to-cell
 * interactions of non-refined sub-grids there.  This slice is
 * the monopole near field of an FMM: the stencil of same-level cells within a
 * sphere of radius R cells; the far field (multipoles, p2m, root) is not
 * restated.
 * ------------------------------------------------------------------------- */
int orc_p2p_stencil(int radius, int32_t* off, double* coef, int cap) {
    if (radius < 1 || radius > ORC_P2P_RMAX) return -1;
    int n = 0;
    for (int r2 = 1; r2 <= radius * radius; ++r2)
        for (int dz = -radius; dz <= radius; ++dz)
            for (int dy = -radius; dy <= radius; ++dy)
                for (int dx = -radius; dx <= radius; ++dx) {
                    if (dx * dx + dy * dy + dz * dz != r2) continue;
                    if (n < cap) {
                        const double c0 = 1.0 / sqrt((double)r2);
                        const double c3 = c0 / (double)r2;
                        off[3 * n] = dx;
                        off[3 * n + 1] = dy;
                        off[3 * n + 2] = dz;
                        coef[4 * n] = c0;
                        coef[4 * n + 1] = (double)dx * c3;
                        coef[4 * n + 2] = (double)dy * c3;
                        coef[4 * n + 3] = (double)dz * c3;
                    }
                    ++n;
                }
    return n;
}

/* density of the cell at in-sub-grid coordinates (x, y, z) in [-8, 15],
 * walking the face links x, then y, then z; vacuum outside the mesh */
static double p2p_rho(int nf, const int64_t* nbr, const double* U, int64_t g, int x, int y, int z) {
    int c[3] = {x, y, z};
    int64_t h = g;
    for (int axis = 0; axis < 3; ++axis) {
        if (c[axis] < 0) {
            h = nbr[6 * h + 2 * axis];
            c[axis] += N;
        } else if (c[axis] >= N) {
            h = nbr[6 * h + 2 * axis + 1];
            c[axis] -= N;
        }
        if (h < 0) return 0.0;
    }
    return U[(h * nf) * NC + cidx(c[0], c[1], c[2])];
}

void orc_gravity_p2p(const orc_params* p, int64_t ngrids, const int64_t* nbr, const double* U, int radius, double G,
                     double* out) {
    int32_t off[3 * 1024];
    double coef[4 * 1024];
    const int ns = orc_p2p_stencil(radius, off, coef, 1024);
    if (ns < 0 || ns > 1024) return;
    const double h = p->dx;
    const double kphi = -G * (h * h), kg = G * h;
    for (int64_t g = 0; g < ngrids; ++g)
        for (int z = 0; z < N; ++z)
            for (int y = 0; y < N; ++y)
                for (int x = 0; x < N; ++x) {
                    double s0 = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
                    for (int k = 0; k < ns; ++k) {
                        const double rho = p2p_rho(p->nf, nbr, U, g, x + off[3 * k], y + off[3 * k + 1],
                                                   z + off[3 * k + 2]);
                        s0 = fma(rho, coef[4 * k], s0);
                        sx = fma(rho, coef[4 * k + 1], sx);
                        sy = fma(rho, coef[4 * k + 2], sy);
                        sz = fma(rho, coef[4 * k + 3], sz);
                    }
                    double* o = out + g * 4 * NC + cidx(x, y, z);
                    o[0] = kphi * s0;
                    o[NC] = kg * sx;
                    o[2 * NC] = kg * sy;
                    o[3 * NC] = kg * sz;
                }
}
