/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see hydro_oracle.h).
 *
 * Gravity, the whole solve: a cell-based fast
 * multipole method over the octree of 8^3 sub-grids, restated scalar and in
 * the exact operation order the B200 kernels (csrc/fmm_kernels.cu) follow.
 * The reference schedules it as six launches per sub-grid and step of the
 * kernel `gravity_kernel_name` picks (workload.cpp:365-372, 565-569):
 * multipole_root_kernel (root), multipole_kernel (refined node), p2m_kernel
 * (leaf next to a refined node), p2p_kernel (other leaves); it only sleeps
 * for them.  Octo-Tiger's FMM is the model: every octree
 * node carries an 8^3 grid of cells, refined nodes' cells hold the
 * restriction of their children, cells interact with same-depth cells that
 * are near at the parent depth but not at their own, and local expansions
 * are passed down.  This restatement keeps monopoles about the centre of
 * mass and first-order local expansions (phi, g, grad g); DESIGN.md §15
 * states the contract in full.  The tree comes from the leaves alone
 * (level, position), the same input the product takes.
 */
#include "hydro_oracle.h"

#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdlib.h>
#include <string.h>

#define N ORC_N
#define NC ORC_NC

typedef struct {
    uint64_t key;
    int32_t depth, q[3];
    int64_t leaf;   /* leaf index, -1 for a refined node */
    int64_t parent; /* node id, -1 for the root */
    int64_t child[8];
} fnode;

static uint64_t nkey(int d, int qx, int qy, int qz) {
    return ((uint64_t)d << 60) | ((uint64_t)qz << 40) | ((uint64_t)qy << 20) | (uint64_t)qx;
}

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

typedef struct {
    fnode* nodes;
    int64_t n;
    int T;
    double dx0;
} ftree;

static int64_t find(const ftree* t, int d, int qx, int qy, int qz) {
    if (qx < 0 || qy < 0 || qz < 0 || d < 0) return -1;
    const uint64_t k = nkey(d, qx, qy, qz);
    int64_t lo = 0, hi = t->n - 1;
    while (lo <= hi) {
        const int64_t mid = (lo + hi) / 2;
        if (t->nodes[mid].key == k) return mid;
        if (t->nodes[mid].key < k) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

/* Leaves + all their ancestors; error (-1) on overlap or positions outside the domain. */
static int build_tree(ftree* t, int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                      double dx0) {
    int T = 0;
    const int mx = dims[0] > dims[1] ? (dims[0] > dims[2] ? dims[0] : dims[2]) : (dims[1] > dims[2] ? dims[1] : dims[2]);
    while ((1 << T) < mx) ++T;
    t->T = T;
    t->dx0 = dx0;
    /* keys of every leaf and ancestor; the low bit of the slot says "leaf" */
    int64_t cap = 0;
    for (int64_t k = 0; k < n_leaves; ++k) {
        if (level[k] < 0 || level[k] > 20) return -1;
        cap += level[k] + T + 1;
    }
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(cap > 0 ? cap : 1));
    int64_t nk = 0;
    for (int64_t k = 0; k < n_leaves; ++k) {
        const int d = level[k] + T;
        for (int a = 0; a < 3; ++a)
            if (pos[3 * k + a] < 0 || pos[3 * k + a] >= (dims[a] << level[k])) {
                free(keys);
                return -1;
            }
        for (int e = d; e >= 0; --e) {
            const int s = d - e;
            keys[nk++] = nkey(e, pos[3 * k] >> s, pos[3 * k + 1] >> s, pos[3 * k + 2] >> s);
        }
    }
    qsort(keys, (size_t)nk, sizeof(uint64_t), cmp_u64);
    int64_t nu = 0;
    for (int64_t i = 0; i < nk; ++i)
        if (nu == 0 || keys[nu - 1] != keys[i]) keys[nu++] = keys[i];
    t->n = nu;
    t->nodes = (fnode*)calloc((size_t)(nu > 0 ? nu : 1), sizeof(fnode));
    for (int64_t i = 0; i < nu; ++i) {
        fnode* f = &t->nodes[i];
        f->key = keys[i];
        f->depth = (int32_t)(keys[i] >> 60);
        f->q[0] = (int32_t)(keys[i] & 0xFFFFF);
        f->q[1] = (int32_t)((keys[i] >> 20) & 0xFFFFF);
        f->q[2] = (int32_t)((keys[i] >> 40) & 0xFFFFF);
        f->leaf = -1;
        f->parent = -1;
        for (int c = 0; c < 8; ++c) f->child[c] = -1;
    }
    free(keys);
    for (int64_t k = 0; k < n_leaves; ++k) {
        const int64_t i = find(t, level[k] + T, pos[3 * k], pos[3 * k + 1], pos[3 * k + 2]);
        if (t->nodes[i].leaf >= 0) return -1; /* duplicate leaf */
        t->nodes[i].leaf = k;
    }
    for (int64_t i = 0; i < nu; ++i) {
        fnode* f = &t->nodes[i];
        if (f->depth == 0) continue;
        const int64_t p = find(t, f->depth - 1, f->q[0] >> 1, f->q[1] >> 1, f->q[2] >> 1);
        f->parent = p;
        if (t->nodes[p].leaf >= 0) return -1; /* a leaf with descendants: overlapping leaves */
        t->nodes[p].child[(f->q[0] & 1) | ((f->q[1] & 1) << 1) | ((f->q[2] & 1) << 2)] = i;
    }
    return 0;
}

static double hdepth(const ftree* t, int d) { return ldexp(t->dx0, t->T - d); }
static double centre(int I, double h) { return ((double)I + 0.5) * h; }
static int64_t lidx(int x, int y, int z) { return ((int64_t)z * N + y) * N + x; }

/* Source at depth-d global cell J.  Returns 0 none, 1 centred (rho; a leaf
 * cell at its own depth, or a depth-d piece of a coarser leaf's cell),
 * 2 restricted (the moment of a refined node's cell). */
static int source(const ftree* t, int nf, const double* U, const double* M, int d, const int J[3], double* rho,
                  double* m, double c[3]) {
    if (J[0] < 0 || J[1] < 0 || J[2] < 0) return 0;
    const int B[3] = {J[0] >> 3, J[1] >> 3, J[2] >> 3};
    for (int e = d; e >= 0; --e) {
        const int s = d - e;
        const int64_t i = find(t, e, B[0] >> s, B[1] >> s, B[2] >> s);
        if (i < 0) continue;
        const fnode* f = &t->nodes[i];
        const double h = hdepth(t, d);
        if (e == d) {
            const int64_t l = lidx(J[0] - 8 * f->q[0], J[1] - 8 * f->q[1], J[2] - 8 * f->q[2]);
            if (f->leaf >= 0) {
                *rho = U[(f->leaf * nf) * NC + l];
                *m = *rho * ((h * h) * h);
                for (int a = 0; a < 3; ++a) c[a] = centre(J[a], h);
                return 1;
            }
            *m = M[(i * 4) * NC + l];
            for (int a = 0; a < 3; ++a) c[a] = M[(i * 4 + 1 + a) * NC + l];
            return 2;
        }
        if (f->leaf < 0) return 0; /* an absent part of a refined node (outside the domain) */
        const int64_t l = lidx((J[0] >> s) - 8 * f->q[0], (J[1] >> s) - 8 * f->q[1], (J[2] >> s) - 8 * f->q[2]);
        *rho = U[(f->leaf * nf) * NC + l];
        *m = *rho * ((h * h) * h);
        for (int a = 0; a < 3; ++a) c[a] = centre(J[a], h);
        return 1;
    }
    return 0;
}

/* Monopole (m at c) acting at x: phi, g and (with T) grad g, accumulated. */
static void m2l(double G, double m, const double c[3], const double x[3], double* phi, double g[3], double* T) {
    const double rx = x[0] - c[0], ry = x[1] - c[1], rz = x[2] - c[2];
    const double r2 = fma(rz, rz, fma(ry, ry, rx * rx));
    const double inv = 1.0 / sqrt(r2);
    const double inv2 = inv * inv;
    const double a1 = (G * m) * inv;
    const double a3 = a1 * inv2;
    *phi = *phi - a1;
    g[0] = fma(-a3, rx, g[0]);
    g[1] = fma(-a3, ry, g[1]);
    g[2] = fma(-a3, rz, g[2]);
    if (T != NULL) {
        const double a5 = (3.0 * a3) * inv2;
        const double tx = a5 * rx, ty = a5 * ry, tz = a5 * rz;
        T[0] = fma(tx, rx, T[0] - a3); /* xx */
        T[1] = fma(ty, ry, T[1] - a3); /* yy */
        T[2] = fma(tz, rz, T[2] - a3); /* zz */
        T[3] = fma(tx, ry, T[3]);      /* xy */
        T[4] = fma(tx, rz, T[4]);      /* xz */
        T[5] = fma(ty, rz, T[5]);      /* yz */
    }
}

/* Parent cell's expansion (phi, g, T) shifted to the child cell centre. */
static void l2l(const double* Lp, const int I[3], double h, double* phi, double g[3], double T[6]) {
    double dl[3];
    for (int a = 0; a < 3; ++a) dl[a] = (I[a] & 1) ? 0.5 * h : -0.5 * h;
    const double pp = Lp[0], gx = Lp[1], gy = Lp[2], gz = Lp[3];
    const double txx = Lp[4], tyy = Lp[5], tzz = Lp[6], txy = Lp[7], txz = Lp[8], tyz = Lp[9];
    g[0] = fma(txz, dl[2], fma(txy, dl[1], fma(txx, dl[0], gx)));
    g[1] = fma(tyz, dl[2], fma(tyy, dl[1], fma(txy, dl[0], gy)));
    g[2] = fma(tzz, dl[2], fma(tyz, dl[1], fma(txz, dl[0], gz)));
    double s = (gx + g[0]) * dl[0];
    s = fma(gy + g[1], dl[1], s);
    s = fma(gz + g[2], dl[2], s);
    *phi = fma(-0.5, s, pp);
    for (int k = 0; k < 6; ++k) T[k] = Lp[4 + k];
}

int orc_fmm_table(int radius, int root, int32_t* u, int32_t* near, int cap) {
    if (radius < 1 || radius > ORC_FMM_RMAX) return -1;
    const int K = root ? 7 : 2 * radius + 1, R2 = radius * radius;
    int n = 0;
    for (int z = -K; z <= K; ++z)
        for (int y = -K; y <= K; ++y)
            for (int x = -K; x <= K; ++x) {
                if (x == 0 && y == 0 && z == 0) continue;
                if (!root) {
                    const int px = x >> 1, py = y >> 1, pz = z >> 1;
                    if (px * px + py * py + pz * pz > R2) continue;
                }
                if (n < cap) {
                    u[3 * n] = x;
                    u[3 * n + 1] = y;
                    u[3 * n + 2] = z;
                    near[n] = x * x + y * y + z * z <= R2;
                }
                ++n;
            }
    return n;
}

typedef struct {
    const ftree* t;
    int nf;
    const double* U;
    const double* M;
    double* L;
    double* out;
    double G;
    const int32_t *tu, *tn, *ru, *rn;
    int nt, nr;
    int d, tid, nth;
} down_job;

/* One node of the downward pass (refined: its expansions; leaf: its field). */
static void down_node(const down_job* j, int64_t i) {
    const ftree t = *j->t;
    const int nf = j->nf, d = j->d;
    const double* U = j->U;
    const double* M = j->M;
    double* L = j->L;
    double* out = j->out;
    const double G = j->G;
    const int32_t *tu = j->tu, *tn = j->tn, *ru = j->ru, *rn = j->rn;
    const int nt = j->nt, nr = j->nr;
    const fnode* f = &t.nodes[i];
    const double h = hdepth(&t, d);
    const int32_t* uu = d == 0 ? ru : tu;
    const int32_t* un = d == 0 ? rn : tn;
    const int nu = d == 0 ? nr : nt;
    for (int z = 0; z < N; ++z)
        for (int y = 0; y < N; ++y)
            for (int x = 0; x < N; ++x) {
                const int I[3] = {8 * f->q[0] + x, 8 * f->q[1] + y, 8 * f->q[2] + z};
                const double xc[3] = {centre(I[0], h), centre(I[1], h), centre(I[2], h)};
                double phi = 0.0, g[3] = {0.0, 0.0, 0.0}, T[6] = {0, 0, 0, 0, 0, 0};
                if (d > 0) {
                    const fnode* pf = &t.nodes[f->parent];
                    const int64_t lp = lidx((I[0] >> 1) - 8 * pf->q[0], (I[1] >> 1) - 8 * pf->q[1],
                                            (I[2] >> 1) - 8 * pf->q[2]);
                    double Lp[10];
                    for (int k = 0; k < 10; ++k) Lp[k] = L[(f->parent * 10 + k) * NC + lp];
                    l2l(Lp, I, h, &phi, g, T);
                }
                if (f->leaf < 0) {
                    /* the far entries in chunks of ORC_FMM_CHUNK (table
                     * order), each summed from zero and added in order to the
                     * parent's shifted expansion (the GPU may spread the
                     * chunks over CTAs) */
                    double part[10] = {0};
                    int in_chunk = 0;
                    for (int k = 0; k < nu; ++k) {
                        if (un[k]) continue;
                        int J[3];
                        for (int a = 0; a < 3; ++a) J[a] = I[a] + ((I[a] & 1) ? -uu[3 * k + a] : uu[3 * k + a]);
                        double rho, m, c[3];
                        if (source(&t, nf, U, M, d, J, &rho, &m, c) != 0) m2l(G, m, c, xc, &part[0], part + 1, part + 4);
                        if (++in_chunk == ORC_FMM_CHUNK) {
                            phi = phi + part[0];
                            for (int a = 0; a < 3; ++a) g[a] = g[a] + part[1 + a];
                            for (int q = 0; q < 6; ++q) T[q] = T[q] + part[4 + q];
                            memset(part, 0, sizeof(part));
                            in_chunk = 0;
                        }
                    }
                    if (in_chunk > 0) {
                        phi = phi + part[0];
                        for (int a = 0; a < 3; ++a) g[a] = g[a] + part[1 + a];
                        for (int q = 0; q < 6; ++q) T[q] = T[q] + part[4 + q];
                    }
                }
                if (f->leaf < 0) {
                    double* o = L + (i * 10) * NC + lidx(x, y, z);
                    o[0] = phi;
                    for (int a = 0; a < 3; ++a) o[(1 + a) * NC] = g[a];
                    for (int k = 0; k < 6; ++k) o[(4 + k) * NC] = T[k];
                    continue;
                }
                double s0 = 0.0, s[3] = {0.0, 0.0, 0.0}, rphi = 0.0, rg[3] = {0.0, 0.0, 0.0};
                for (int k = 0; k < nu; ++k) {
                    int e[3], J[3];
                    for (int a = 0; a < 3; ++a) {
                        e[a] = (I[a] & 1) ? -uu[3 * k + a] : uu[3 * k + a];
                        J[a] = I[a] + e[a];
                    }
                    double rho, m, c[3];
                    const int kind = source(&t, nf, U, M, d, J, &rho, &m, c);
                    if (kind == 1) {
                        const int r2 = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
                        const double c0 = 1.0 / sqrt((double)r2);
                        const double c3 = c0 / (double)r2;
                        s0 = fma(rho, c0, s0);
                        for (int a = 0; a < 3; ++a) s[a] = fma(rho, (double)e[a] * c3, s[a]);
                    } else if (kind == 2) {
                        m2l(G, m, c, xc, &rphi, rg, NULL);
                    }
                }
                const double kphi = -G * (h * h), kg = G * h;
                double* o = out + (f->leaf * 4) * NC + lidx(x, y, z);
                o[0] = (phi + kphi * s0) + rphi;
                for (int a = 0; a < 3; ++a) o[(1 + a) * NC] = (g[a] + kg * s[a]) + rg[a];
            }
}

static void* down_worker(void* arg) {
    const down_job* j = (const down_job*)arg;
    for (int64_t i = j->tid; i < j->t->n; i += j->nth)
        if (j->t->nodes[i].depth == j->d) down_node(j, i);
    return NULL;
}

int orc_gravity_fmm(int nf, int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                    double dx0, const double* U, int radius, double G, double* out) {
    if (radius < 1 || radius > ORC_FMM_RMAX || n_leaves <= 0) return -1;
    ftree t = {0};
    if (build_tree(&t, n_leaves, level, pos, dims, dx0) != 0) {
        free(t.nodes);
        return -1;
    }
    const int64_t nn = t.n;
    double* M = (double*)calloc((size_t)nn * 4 * NC, sizeof(double));
    double* L = (double*)calloc((size_t)nn * 10 * NC, sizeof(double));
    int maxd = 0;
    for (int64_t i = 0; i < nn; ++i) maxd = t.nodes[i].depth > maxd ? t.nodes[i].depth : maxd;
    /* upward: leaf moments, then restriction depth by depth */
    for (int d = maxd; d >= 0; --d)
        for (int64_t i = 0; i < nn; ++i) {
            const fnode* f = &t.nodes[i];
            if (f->depth != d) continue;
            const double h = hdepth(&t, d);
            for (int z = 0; z < N; ++z)
                for (int y = 0; y < N; ++y)
                    for (int x = 0; x < N; ++x) {
                        const int I[3] = {8 * f->q[0] + x, 8 * f->q[1] + y, 8 * f->q[2] + z};
                        double* o = M + (i * 4) * NC + lidx(x, y, z);
                        if (f->leaf >= 0) {
                            o[0] = U[(f->leaf * nf) * NC + lidx(x, y, z)] * ((h * h) * h);
                            for (int a = 0; a < 3; ++a) o[(1 + a) * NC] = centre(I[a], h);
                            continue;
                        }
                        const int64_t ch = f->child[(x >> 2) | ((y >> 2) << 1) | ((z >> 2) << 2)];
                        double m = 0.0, mc[3] = {0.0, 0.0, 0.0};
                        if (ch >= 0)
                            for (int sz = 0; sz < 2; ++sz)
                                for (int sy = 0; sy < 2; ++sy)
                                    for (int sx = 0; sx < 2; ++sx) {
                                        const int64_t l = lidx(2 * (x & 3) + sx, 2 * (y & 3) + sy, 2 * (z & 3) + sz);
                                        const double ms = M[(ch * 4) * NC + l];
                                        m = m + ms;
                                        for (int a = 0; a < 3; ++a) mc[a] = fma(ms, M[(ch * 4 + 1 + a) * NC + l], mc[a]);
                                    }
                        o[0] = m;
                        for (int a = 0; a < 3; ++a) o[(1 + a) * NC] = m > 0.0 ? mc[a] / m : centre(I[a], h);
                    }
        }
    /* downward: refined nodes' expansions, depth by depth; leaves evaluate */
    int32_t* tu = (int32_t*)malloc(sizeof(int32_t) * 3 * 4096);
    int32_t* tn = (int32_t*)malloc(sizeof(int32_t) * 4096);
    int32_t* ru = (int32_t*)malloc(sizeof(int32_t) * 3 * 4096);
    int32_t* rn = (int32_t*)malloc(sizeof(int32_t) * 4096);
    const int nt = orc_fmm_table(radius, 0, tu, tn, 4096);
    const int nr = orc_fmm_table(radius, 1, ru, rn, 4096);
    /* nodes of one depth are independent: spread them over host threads */
    long nth = sysconf(_SC_NPROCESSORS_ONLN);
    if (getenv("ORC_THREADS") != NULL) nth = atol(getenv("ORC_THREADS"));
    if (nth < 1) nth = 1;
    if (nth > 64) nth = 64;
    for (int d = 0; d <= maxd; ++d) {
        down_job jobs[64];
        pthread_t th[64];
        for (int k = 0; k < nth; ++k) {
            jobs[k] = (down_job){&t, nf, U, M, L, out, G, tu, tn, ru, rn, nt, nr, d, k, (int)nth};
            if (k > 0) pthread_create(&th[k], NULL, down_worker, &jobs[k]);
        }
        down_worker(&jobs[0]);
        for (int k = 1; k < nth; ++k) pthread_join(th[k], NULL);
    }
    free(tu);
    free(tn);
    free(ru);
    free(rn);
    free(M);
    free(L);
    free(t.nodes);
    return 0;
}

int orc_gravity_direct(int nf, int64_t n_leaves, const int32_t* level, const int32_t* pos, const int32_t* dims,
                       double dx0, const double* U, double G, double* out) {
    (void)dims;
    /* sources: every leaf cell split into equal pieces at the finest level present */
    int lmax = 0;
    for (int64_t k = 0; k < n_leaves; ++k) lmax = level[k] > lmax ? level[k] : lmax;
    int64_t ns = 0;
    for (int64_t k = 0; k < n_leaves; ++k) ns += (int64_t)NC << (3 * (lmax - level[k]));
    double* src = (double*)malloc(sizeof(double) * 4 * (size_t)ns);
    int64_t* own = (int64_t*)malloc(sizeof(int64_t) * (size_t)ns); /* the leaf cell a piece belongs to */
    int64_t w = 0;
    const double hf = ldexp(dx0, -lmax);
    for (int64_t k = 0; k < n_leaves; ++k) {
        const int s = lmax - level[k], f = 1 << s;
        for (int i = 0; i < NC; ++i) {
            const double mp = U[(k * nf) * NC + i] * ((hf * hf) * hf);
            const int b[3] = {(8 * pos[3 * k] + (i & 7)) * f, (8 * pos[3 * k + 1] + ((i >> 3) & 7)) * f,
                              (8 * pos[3 * k + 2] + (i >> 6)) * f};
            for (int z = 0; z < f; ++z)
                for (int y = 0; y < f; ++y)
                    for (int x = 0; x < f; ++x) {
                        double* p = src + 4 * w;
                        p[0] = ((double)(b[0] + x) + 0.5) * hf;
                        p[1] = ((double)(b[1] + y) + 0.5) * hf;
                        p[2] = ((double)(b[2] + z) + 0.5) * hf;
                        p[3] = mp;
                        own[w++] = k * NC + i;
                    }
        }
    }
    for (int64_t k = 0; k < n_leaves; ++k) {
        const double h = ldexp(dx0, -level[k]);
        for (int i = 0; i < NC; ++i) {
            const double x[3] = {((double)(8 * pos[3 * k] + (i & 7)) + 0.5) * h,
                                 ((double)(8 * pos[3 * k + 1] + ((i >> 3) & 7)) + 0.5) * h,
                                 ((double)(8 * pos[3 * k + 2] + (i >> 6)) + 0.5) * h};
            double phi = 0.0, g[3] = {0.0, 0.0, 0.0};
            for (int64_t b = 0; b < ns; ++b) {
                if (own[b] == k * NC + i) continue; /* no self-interaction (the FMM's u != 0) */
                m2l(G, src[4 * b + 3], src + 4 * b, x, &phi, g, NULL);
            }
            out[(k * 4) * NC + i] = phi;
            for (int c = 0; c < 3; ++c) out[(k * 4 + 1 + c) * NC + i] = g[c];
        }
    }
    free(src);
    free(own);
    return 0;
}

void orc_gravity_kick(int nf, int64_t n, double* U, const double* grav, double dt) {
    const double hdt = 0.5 * dt;
    for (int64_t k = 0; k < n; ++k)
        for (int i = 0; i < NC; ++i) {
            double* u = U + (k * nf) * NC + i;
            const double* g = grav + (k * 4) * NC + i;
            const double rho = u[0];
            const double gx = g[NC], gy = g[2 * NC], gz = g[3 * NC];
            const double sx = u[NC], sy = u[2 * NC], sz = u[3 * NC];
            const double nx = fma(dt, rho * gx, sx), ny = fma(dt, rho * gy, sy), nz = fma(dt, rho * gz, sz);
            double w = (sx + nx) * gx;
            w = fma(sy + ny, gy, w);
            w = fma(sz + nz, gz, w);
            u[NC] = nx;
            u[2 * NC] = ny;
            u[3 * NC] = nz;
            u[4 * NC] = fma(hdt, w, u[4 * NC]);
        }
}
