// fmm_kernels.cu — gravity, the whole solve: the cell-based FMM of fmm.h on
// sm_100a.  Reference: the multipole_root / multipole / p2m / p2p launches of
// proj/core/src/workload.cpp:365-372, 565-569 (timed sleeps there); numerics:
// oracle/fmm_oracle.c operation for operation (--fmad=false), so bitwise.
//
// B200 shape: one 512-thread CTA per octree node, one thread per cell; the
// passes run depth by depth (moments up, expansions down), each a launch over
// that depth's nodes.  The dominant pass is the leaf evaluation (near field
// plus the leaf depth's far field, ~263 interactions per cell at R = 2): the
// leaf's density neighbourhood (8 + 2K)^3 is staged once in shared memory and
// an interaction is one LDS + four DFMA against constant-bank coefficients
// (the octant-0 table; a cell of another octant reads the mirrored offset and
// flips the sign of the summed components, which is exact).
#include <algorithm>
#include <atomic>
#include <utility>

#include "fmm.h"
#include "hydro_device.cuh"

namespace tsh {

namespace {

constexpr int kPitch = 24;                // tile row pitch (doubles), S <= 22
constexpr int kTabMax1 = 55, kTabMax2 = 263;  // R = 3: 983 entries, run-time table

__constant__ double c_fmm_coef1[4 * kTabMax1];
__constant__ double c_fmm_coef2[4 * kTabMax2];

struct UTable {
    int x[kTabMax2], y[kTabMax2], z[kTabMax2];
    int n;
};
// The depth >= 1 table of radius R as compile-time offsets (fmm_table order).
constexpr UTable make_utable(int R) {
    UTable t{};
    const int K = 2 * R + 1;
    for (int z = -K; z <= K; ++z)
        for (int y = -K; y <= K; ++y)
            for (int x = -K; x <= K; ++x) {
                if (x == 0 && y == 0 && z == 0) continue;
                const int px = x >> 1, py = y >> 1, pz = z >> 1;
                if (px * px + py * py + pz * pz > R * R) continue;
                t.x[t.n] = x;
                t.y[t.n] = y;
                t.z[t.n] = z;
                ++t.n;
            }
    return t;
}
constexpr UTable kU1 = make_utable(1);
constexpr UTable kU2 = make_utable(2);
static_assert(kU1.n == kTabMax1 && kU2.n == kTabMax2, "FMM table sizes");

__device__ __forceinline__ int node_of(const FmmArgs& A) {
    return A.list != nullptr ? A.list[A.first + (int)blockIdx.x] : A.first + (int)blockIdx.x;
}
__device__ __forceinline__ double hdepth(const FmmArgs& A, int d) { return ldexp(A.dx0, A.T - d); }
__device__ __forceinline__ double centre(int I, double h) { return ((double)I + 0.5) * h; }
__device__ __forceinline__ int lidx(int x, int y, int z) { return (z * N + y) * N + x; }

__device__ __forceinline__ void stamp_begin(const FmmArgs& A) {
    if (A.stamp != nullptr && threadIdx.x == 0) atomicMax(A.stamp, ~globaltimer());
}
__device__ __forceinline__ void stamp_end(const FmmArgs& A) {
    if (A.stamp != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(A.stamp + 1, globaltimer());
    }
}

// Monopole (m at c) acting at x (oracle m2l): phi, g and, with T, grad g.
template <bool WITH_T>
__device__ __forceinline__ void m2l(double G, double m, double cx, double cy, double cz, double xx, double xy,
                                    double xz, double& phi, double (&g)[3], double (&T)[6]) {
    const double rx = xx - cx, ry = xy - cy, rz = xz - cz;
    const double r2 = fma(rz, rz, fma(ry, ry, rx * rx));
    // 1.0 / sqrt(r2) with the branch-free IEEE forms (bitwise equal for the
    // positive normal r2 here: hydro_device.cuh, ts_hydro_selftest_math)
    const double inv = rcp_rn(sqrt_rn(r2));
    const double inv2 = inv * inv;
    const double a1 = (G * m) * inv;
    const double a3 = a1 * inv2;
    phi = phi - a1;
    g[0] = fma(-a3, rx, g[0]);
    g[1] = fma(-a3, ry, g[1]);
    g[2] = fma(-a3, rz, g[2]);
    if (WITH_T) {
        const double a5 = (3.0 * a3) * inv2;
        const double tx = a5 * rx, ty = a5 * ry, tz = a5 * rz;
        T[0] = fma(tx, rx, T[0] - a3);
        T[1] = fma(ty, ry, T[1] - a3);
        T[2] = fma(tz, rz, T[2] - a3);
        T[3] = fma(tx, ry, T[3]);
        T[4] = fma(tx, rz, T[4]);
        T[5] = fma(ty, rz, T[5]);
    }
}

// Parent cell's expansion shifted to the child centre (oracle l2l).
__device__ __forceinline__ void l2l(const FmmArgs& A, int node, int d, const int (&I)[3], double h, double& phi,
                                    double (&g)[3], double (&T)[6]) {
    const int p = A.parent[node];
    const int lp = lidx((I[0] >> 1) - 8 * A.q[3 * p], (I[1] >> 1) - 8 * A.q[3 * p + 1], (I[2] >> 1) - 8 * A.q[3 * p + 2]);
    const double* Lp = A.L + (size_t)p * 10 * NC + lp;
    double dl[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) dl[a] = (I[a] & 1) ? 0.5 * h : -0.5 * h;
    const double pp = Lp[0], gx = Lp[NC], gy = Lp[2 * NC], gz = Lp[3 * NC];
    const double txx = Lp[4 * NC], tyy = Lp[5 * NC], tzz = Lp[6 * NC], txy = Lp[7 * NC], txz = Lp[8 * NC],
                 tyz = Lp[9 * NC];
    g[0] = fma(txz, dl[2], fma(txy, dl[1], fma(txx, dl[0], gx)));
    g[1] = fma(tyz, dl[2], fma(tyy, dl[1], fma(txy, dl[0], gy)));
    g[2] = fma(tzz, dl[2], fma(tyz, dl[1], fma(txz, dl[0], gz)));
    double s = (gx + g[0]) * dl[0];
    s = fma(gy + g[1], dl[1], s);
    s = fma(gz + g[2], dl[2], s);
    phi = fma(-0.5, s, pp);
    T[0] = txx;
    T[1] = tyy;
    T[2] = tzz;
    T[3] = txy;
    T[4] = txz;
    T[5] = tyz;
    (void)d;
}

// Source at depth-d global cell J seen from `node` (its nb27 in shared
// memory): 0 none, 1 a moment (m, c) of a same-depth node, 2 a depth-d piece
// of a coarser leaf's cell (rho; centred).
__device__ __forceinline__ int source(const FmmArgs& A, const int* nb, const int (&q)[3], int d, double h,
                                      const int (&J)[3], double& m, double& rho, double (&c)[3]) {
    const int slot = (((J[2] >> 3) - q[2] + 1) * 3 + ((J[1] >> 3) - q[1] + 1)) * 3 + ((J[0] >> 3) - q[0] + 1);
    const int code = nb[slot];
    if (code == kFmmNone) return 0;
    if (code >= 0) {
        const double* Ms = A.M + (size_t)code * 4 * NC + lidx(J[0] & 7, J[1] & 7, J[2] & 7);
        m = Ms[0];
        c[0] = Ms[NC];
        c[1] = Ms[2 * NC];
        c[2] = Ms[3 * NC];
        return 1;
    }
    const int cn = -2 - code;
    const int s = d - A.depth[cn];
    const int l = lidx((J[0] >> s) - 8 * A.q[3 * cn], (J[1] >> s) - 8 * A.q[3 * cn + 1], (J[2] >> s) - 8 * A.q[3 * cn + 2]);
    rho = A.U[(size_t)A.leaf[cn] * A.nf * NC + l];
    m = rho * ((h * h) * h);
    c[0] = centre(J[0], h);
    c[1] = centre(J[1], h);
    c[2] = centre(J[2], h);
    return 2;
}

// P2M: a leaf's cell masses and centres.
__global__ void __launch_bounds__(NC) fmm_moments_kernel(const __grid_constant__ FmmArgs A) {
    stamp_begin(A);
    const int node = node_of(A), t = threadIdx.x;
    const int d = A.depth[node];
    const double h = hdepth(A, d);
    double* o = A.M + (size_t)node * 4 * NC + t;
    o[0] = A.U[(size_t)A.leaf[node] * A.nf * NC + t] * ((h * h) * h);
    o[NC] = centre(8 * A.q[3 * node] + (t & 7), h);
    o[2 * NC] = centre(8 * A.q[3 * node + 1] + ((t >> 3) & 7), h);
    o[3 * NC] = centre(8 * A.q[3 * node + 2] + (t >> 6), h);
    stamp_end(A);
}

// M2M: a refined node's cells from its children's (mass, centre of mass).
__global__ void __launch_bounds__(NC) fmm_restrict_kernel(const __grid_constant__ FmmArgs A) {
    stamp_begin(A);
    const int node = node_of(A), t = threadIdx.x;
    const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
    const int d = A.depth[node];
    const double h = hdepth(A, d);
    const int ch = A.child[8 * node + ((x >> 2) | ((y >> 2) << 1) | ((z >> 2) << 2))];
    double m = 0.0, mc[3] = {0.0, 0.0, 0.0};
    if (ch >= 0) {
        const double* Mc = A.M + (size_t)ch * 4 * NC;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int l = lidx(2 * (x & 3) + (s & 1), 2 * (y & 3) + ((s >> 1) & 1), 2 * (z & 3) + (s >> 2));
            const double ms = Mc[l];
            m = m + ms;
            mc[0] = fma(ms, Mc[NC + l], mc[0]);
            mc[1] = fma(ms, Mc[2 * NC + l], mc[1]);
            mc[2] = fma(ms, Mc[3 * NC + l], mc[2]);
        }
    }
    const int I[3] = {8 * A.q[3 * node] + x, 8 * A.q[3 * node + 1] + y, 8 * A.q[3 * node + 2] + z};
    double* o = A.M + (size_t)node * 4 * NC + t;
    o[0] = m;
#pragma unroll
    for (int a = 0; a < 3; ++a) o[(1 + a) * NC] = m > 0.0 ? mc[a] / m : centre(I[a], h);
    stamp_end(A);
}

// L2L + M2L of refined nodes (the root: no L2L, the root table).  The far
// sum runs in chunks of kFmmChunk table entries, each summed from zero, added
// in order (the oracle's contract), spread over CTAs: CTA (c, n) sums chunk c
// of node first + n for all 512 cells into part[n][c]; the combine kernel
// adds the parent's shifted expansion and the chunk sums in order.
// Chunk `chunk` of node `node`'s far sum over table `tab` for all 512 cells into row `o` of A.part.
__device__ __forceinline__ void m2l_part_body(const FmmArgs& A, int node, int chunk, const FmmEntry* tab, int n_tab,
                                              double* o, int* nb) {
    const int t = threadIdx.x;
    if (t < 27) nb[t] = A.nb27[27 * node + t];
    __syncthreads();
    const int d = A.depth[node];
    const double h = hdepth(A, d);
    const int q[3] = {A.q[3 * node], A.q[3 * node + 1], A.q[3 * node + 2]};
    const int I[3] = {8 * q[0] + (t & 7), 8 * q[1] + ((t >> 3) & 7), 8 * q[2] + (t >> 6)};
    const double xc[3] = {centre(I[0], h), centre(I[1], h), centre(I[2], h)};
    double phi = 0.0, g[3] = {0.0, 0.0, 0.0}, T[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int sx = (I[0] & 1) ? -1 : 1, sy = (I[1] & 1) ? -1 : 1, sz = (I[2] & 1) ? -1 : 1;
    const int k0 = chunk * kFmmChunk, k1 = min(k0 + kFmmChunk, n_tab);
    for (int k = k0; k < k1; ++k) {
        const int4 u = __ldg(reinterpret_cast<const int4*>(tab + k));
        const int J[3] = {I[0] + sx * u.x, I[1] + sy * u.y, I[2] + sz * u.z};
        double m, rho, c[3];
        if (source(A, nb, q, d, h, J, m, rho, c) == 0) continue;
        m2l<true>(A.G, m, c[0], c[1], c[2], xc[0], xc[1], xc[2], phi, g, T);
    }
    o += t;
    o[0] = phi;
    o[NC] = g[0];
    o[2 * NC] = g[1];
    o[3 * NC] = g[2];
#pragma unroll
    for (int k = 0; k < 6; ++k) o[(4 + k) * NC] = T[k];
}

__global__ void __launch_bounds__(NC) fmm_m2l_part_kernel(const __grid_constant__ FmmArgs A) {
    __shared__ int nb[27];
    stamp_begin(A);
    const int node = A.list != nullptr ? A.list[A.first + (int)blockIdx.y] : A.first + (int)blockIdx.y;
    m2l_part_body(A, node, (int)blockIdx.x, A.table, A.n_table,
                  A.part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 10 * NC, nb);
    stamp_end(A);
}

// One launch for the root's chunks (its own table; rows n_far_rows onward)
// and every chunk of the listed deeper nodes (A.table; rows from 0): CTA i
// < n_root_chunks takes root chunk i, the others (node, chunk) in row order.
__global__ void __launch_bounds__(NC) fmm_m2l_part_flat_kernel(const __grid_constant__ FmmArgs A, int root_node,
                                                               int n_root_chunks, const FmmEntry* root_tab,
                                                               int n_root_tab, int n_far_chunks, int n_far_rows) {
    __shared__ int nb[27];
    stamp_begin(A);
    const int i = (int)blockIdx.x;
    if (i < n_root_chunks) {
        m2l_part_body(A, root_node, i, root_tab, n_root_tab, A.part + (size_t)(n_far_rows + i) * 10 * NC, nb);
    } else {
        const int j = i - n_root_chunks;
        const int node = A.list[A.first + j / n_far_chunks];
        m2l_part_body(A, node, j % n_far_chunks, A.table, A.n_table, A.part + (size_t)j * 10 * NC, nb);
    }
    stamp_end(A);
}

// grid (n_nodes, 10): CTA (n, j) writes expansion component j of node
// first + n (the shift is recomputed per component: cheap); the chunk sums are
// loaded eight at a time and added in order.
__global__ void __launch_bounds__(NC) fmm_m2l_combine_kernel(const __grid_constant__ FmmArgs A, int n_chunks) {
    stamp_begin(A);
    const int node = A.list != nullptr ? A.list[A.first + (int)blockIdx.x] : A.first + (int)blockIdx.x;
    const int j = (int)blockIdx.y, t = threadIdx.x;
    const int d = A.depth[node];
    double acc = 0.0;
    if (d > 0) {
        const double h = hdepth(A, d);
        const int I[3] = {8 * A.q[3 * node] + (t & 7), 8 * A.q[3 * node + 1] + ((t >> 3) & 7),
                          8 * A.q[3 * node + 2] + (t >> 6)};
        double phi, g[3], T[6];
        l2l(A, node, d, I, h, phi, g, T);
        acc = j == 0 ? phi : (j < 4 ? g[j - 1] : T[j - 4]);
    }
    const double* p = A.part + ((size_t)blockIdx.x * n_chunks * 10 + j) * NC + t;
    int c = 0;
    for (; c + 8 <= n_chunks; c += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = p[(size_t)(c + k) * 10 * NC];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = acc + v[k];
    }
    for (; c < n_chunks; ++c) acc = acc + p[(size_t)c * 10 * NC];
    A.L[((size_t)node * 10 + j) * NC + t] = acc;
    stamp_end(A);
}

// CPT cells per thread: (x, y, z), (x, y, z + 4) and, for CPT = 4, the same
// at y + 4 — one octant, so one mirrored offset: one address, CPT LDS at
// immediate distances, and each coefficient load serves every cell.
template <int CPT>
__device__ __forceinline__ constexpr int cell_off(int c, int S) {
    return (c & 1) * 4 * S * kPitch + (c >> 1) * 4 * kPitch;
}
template <int R, int CPT, int K>
__device__ __forceinline__ void leaf_term(const double* base, int mx, int my, int mz, double (&a)[CPT][4]) {
    constexpr int ux = R == 1 ? kU1.x[K] : kU2.x[K];
    constexpr int uy = R == 1 ? kU1.y[K] : kU2.y[K];
    constexpr int uz = R == 1 ? kU1.z[K] : kU2.z[K];
    constexpr int S = N + 2 * (2 * R + 1);
    const double* coef = R == 1 ? c_fmm_coef1 : c_fmm_coef2;
    const double* p = base + (ux * mx + uy * my + uz * mz);
    double rho[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) rho[c] = p[cell_off<CPT>(c, S)];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < CPT; ++c) a[c][j] = fma(rho[c], coef[4 * K + j], a[c][j]);
}
template <int R, int CPT, int... K>
__device__ __forceinline__ void leaf_terms(const double* base, int mx, int my, int mz, double (&a)[CPT][4],
                                           std::integer_sequence<int, K...>) {
    (leaf_term<R, CPT, K>(base, mx, my, mz, a), ...);  // in table order
}

// Leaves: L2L from the parent + every table entry (near and this depth's far
// field).  Centred sources (leaf cells, pieces of coarser leaves) come from
// the density tile; RESTR (leaves with a refined neighbour): moments of
// refined same-depth nodes through the general formula.  RS = 1, 2: unrolled
// constant tables; 0: the run-time table (R = 3, and the root when it is the
// only leaf).  512 / CPT threads, CPT cells each.
template <int RS, bool RESTR, int CPT>
__global__ void __launch_bounds__(NC / CPT) fmm_leaf_kernel(const __grid_constant__ FmmArgs A) {
    constexpr int NT = NC / CPT;
    extern __shared__ __align__(16) double tile[];
    __shared__ int nb[27];
    stamp_begin(A);
    const int node = node_of(A), t = threadIdx.x;
    if (t < 27) nb[t] = A.nb27[27 * node + t];
    __syncthreads();
    const int d = A.depth[node];
    const double h = hdepth(A, d);
    const int q[3] = {A.q[3 * node], A.q[3 * node + 1], A.q[3 * node + 2]};
    const int K = A.K, S = N + 2 * K;
    for (int i = t; i < S * S * S; i += NT) {
        const int x = i % S - K, y = (i / S) % S - K, z = i / (S * S) - K;
        const int code = nb[(((z + 8) >> 3) * 3 + ((y + 8) >> 3)) * 3 + ((x + 8) >> 3)];
        double rho = 0.0;
        if (code >= 0) {
            const int lf = A.leaf[code];
            if (lf >= 0) rho = __ldg(A.U + (size_t)lf * A.nf * NC + lidx(x & 7, y & 7, z & 7));
        } else if (code != kFmmNone) {
            const int cn = -2 - code, s = d - A.depth[cn];
            const int J[3] = {8 * q[0] + x, 8 * q[1] + y, 8 * q[2] + z};
            rho = __ldg(A.U + (size_t)A.leaf[cn] * A.nf * NC +
                        lidx((J[0] >> s) - 8 * A.q[3 * cn], (J[1] >> s) - 8 * A.q[3 * cn + 1],
                             (J[2] >> s) - 8 * A.q[3 * cn + 2]));
        }
        tile[((z + K) * S + (y + K)) * kPitch + (x + K)] = rho;
    }
    __syncthreads();
    // cell c of this thread: (x, y0 + 4 (c >> 1), z0 + 4 (c & 1))
    const int x = t & 7;
    const int y0 = CPT == 4 ? (t >> 3) & 3 : (t >> 3) & 7;
    const int z0 = CPT == 4 ? t >> 5 : t >> 6;
    const int sx = (x & 1) ? -1 : 1, sy = (y0 & 1) ? -1 : 1, sz = (z0 & 1) ? -1 : 1;
    const int mx = sx, my = sy * kPitch, mz = sz * kPitch * S;
    const double* base = tile + ((z0 + K) * S + (y0 + K)) * kPitch + (x + K);
    double acc[CPT][4];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[c][j] = 0.0;
    if constexpr (RS == 1) {
        leaf_terms<1, CPT>(base, mx, my, mz, acc, std::make_integer_sequence<int, kTabMax1>{});
    } else if constexpr (RS == 2) {
        leaf_terms<2, CPT>(base, mx, my, mz, acc, std::make_integer_sequence<int, kTabMax2>{});
    } else {
#pragma unroll 4
        for (int k = 0; k < A.n_table; ++k) {
            const FmmEntry* e = A.table + k;
            const int4 u = __ldg(reinterpret_cast<const int4*>(e));
            const double2 c01 = __ldg(reinterpret_cast<const double2*>(e->c));
            const double2 c23 = __ldg(reinterpret_cast<const double2*>(e->c + 2));
            const double* p = base + (u.x * mx + u.y * my + u.z * mz);
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const double rho = p[cell_off<CPT>(c, S)];
                acc[c][0] = fma(rho, c01.x, acc[c][0]);
                acc[c][1] = fma(rho, c01.y, acc[c][1]);
                acc[c][2] = fma(rho, c23.x, acc[c][2]);
                acc[c][3] = fma(rho, c23.y, acc[c][3]);
            }
        }
    }
    // the octant's mirror: e = sigma u, so the summed components flip sign
    // (0 - s: a +0 sum stays +0, as the oracle's sum of mirrored terms does)
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        if (sx < 0) acc[c][1] = 0.0 - acc[c][1];
        if (sy < 0) acc[c][2] = 0.0 - acc[c][2];
        if (sz < 0) acc[c][3] = 0.0 - acc[c][3];
    }
    double racc[CPT][4];  // restricted sources: phi, g
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) racc[c][j] = 0.0;
    if constexpr (RESTR) {
        // every cell per table entry (independent chains)
        for (int k = 0; k < A.n_table; ++k) {
            const int4 u = __ldg(reinterpret_cast<const int4*>(A.table + k));
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int I[3] = {8 * q[0] + x, 8 * q[1] + y0 + 4 * (c >> 1), 8 * q[2] + z0 + 4 * (c & 1)};
                const int J[3] = {I[0] + sx * u.x, I[1] + sy * u.y, I[2] + sz * u.z};
                const int code =
                    nb[(((J[2] >> 3) - q[2] + 1) * 3 + ((J[1] >> 3) - q[1] + 1)) * 3 + ((J[0] >> 3) - q[0] + 1)];
                if (code < 0 || A.leaf[code] >= 0) continue;
                const double* Ms = A.M + (size_t)code * 4 * NC + lidx(J[0] & 7, J[1] & 7, J[2] & 7);
                double g3[3] = {racc[c][1], racc[c][2], racc[c][3]}, Tn[6];
                m2l<false>(A.G, Ms[0], Ms[NC], Ms[2 * NC], Ms[3 * NC], centre(I[0], h), centre(I[1], h),
                           centre(I[2], h), racc[c][0], g3, Tn);
                racc[c][1] = g3[0], racc[c][2] = g3[1], racc[c][3] = g3[2];
            }
        }
    }
    const double kphi = -A.G * (h * h), kg = A.G * h;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int yc = y0 + 4 * (c >> 1), zc = z0 + 4 * (c & 1);
        const int I[3] = {8 * q[0] + x, 8 * q[1] + yc, 8 * q[2] + zc};
        double phi = 0.0, g[3] = {0.0, 0.0, 0.0}, T[6];
        if (d > 0) l2l(A, node, d, I, h, phi, g, T);
        double* o = A.out + (size_t)A.leaf_out[node] * 4 * NC + lidx(x, yc, zc);
        o[0] = (phi + kphi * acc[c][0]) + racc[c][0];
        o[NC] = (g[0] + kg * acc[c][1]) + racc[c][1];
        o[2 * NC] = (g[1] + kg * acc[c][2]) + racc[c][2];
        o[3 * NC] = (g[2] + kg * acc[c][3]) + racc[c][3];
    }
    stamp_end(A);
}

// Gravity source over dt (oracle orc_gravity_kick): S += dt rho g, E +=
// dt/2 (S + S').g; dt from the device (the last step's) when dt_dev is set.
__global__ void gravity_kick_kernel(double* __restrict__ U, int nf, long long n, const double* __restrict__ grav,
                                    const double* dt_dev, double dt_val, unsigned long long* stamp) {
    if (stamp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) atomicMax(stamp, ~globaltimer());
    const double dt = dt_dev != nullptr ? *dt_dev : dt_val;
    const double hdt = 0.5 * dt;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n * NC; c += (long long)gridDim.x * blockDim.x) {
        const long long k = c / NC;
        const int i = (int)(c % NC);
        double* u = U + (size_t)k * nf * NC + i;
        const double* g = grav + (size_t)k * 4 * NC + i;
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
    if (stamp != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(stamp + 1, globaltimer());
    }
}

constexpr size_t tile_bytes(int K) { return (size_t)(N + 2 * K) * (N + 2 * K) * kPitch * sizeof(double); }

cudaError_t ensure_device_setup();

}  // namespace

cudaError_t fmm_prepare_device() { return ensure_device_setup(); }

namespace {

cudaError_t ensure_device_setup() {
    static std::atomic<unsigned long long> ready{0ull};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (ready.load(std::memory_order_acquire) & bit) return cudaSuccess;
    const std::vector<FmmEntry> t1 = fmm_table(1, false, false), t2 = fmm_table(2, false, false);
    if ((int)t1.size() != kTabMax1 || (int)t2.size() != kTabMax2) return cudaErrorInvalidValue;
    std::vector<double> c1(4 * t1.size()), c2(4 * t2.size());
    for (size_t k = 0; k < t1.size(); ++k)
        for (int j = 0; j < 4; ++j) c1[4 * k + j] = t1[k].c[j];
    for (size_t k = 0; k < t2.size(); ++k) {
        for (int j = 0; j < 4; ++j) c2[4 * k + j] = t2[k].c[j];
        if (t2[k].u[0] != kU2.x[k] || t2[k].u[1] != kU2.y[k] || t2[k].u[2] != kU2.z[k]) return cudaErrorInvalidValue;
    }
    e = cudaMemcpyToSymbol(c_fmm_coef1, c1.data(), c1.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_fmm_coef2, c2.data(), c2.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // the symbol copies land before any launch
    const int smem = (int)tile_bytes(kFmmRootK);
#define TS_FMM_LEAF_ATTR(CPT)                                                                              \
    for (auto fn : {fmm_leaf_kernel<0, false, CPT>, fmm_leaf_kernel<0, true, CPT>, fmm_leaf_kernel<1, false, CPT>, \
                    fmm_leaf_kernel<1, true, CPT>, fmm_leaf_kernel<2, false, CPT>, fmm_leaf_kernel<2, true, CPT>})   \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    TS_FMM_LEAF_ATTR(2)
#undef TS_FMM_LEAF_ATTR
    if (e != cudaSuccess) return e;
    ready.fetch_or(bit, std::memory_order_acq_rel);
    return cudaSuccess;
}

}  // namespace

cudaError_t launch_fmm_moments(const FmmArgs& a, int n_ctas, cudaStream_t s) {
    if (n_ctas <= 0) return cudaSuccess;
    fmm_moments_kernel<<<n_ctas, NC, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fmm_restrict(const FmmArgs& a, int n_ctas, cudaStream_t s) {
    if (n_ctas <= 0) return cudaSuccess;
    fmm_restrict_kernel<<<n_ctas, NC, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fmm_m2l_split(const FmmArgs& a, int n_nodes, cudaStream_t s) {
    const int n_chunks = (a.n_table + kFmmChunk - 1) / kFmmChunk;
    if (n_nodes <= 0 || n_chunks <= 0) return cudaSuccess;
    fmm_m2l_part_kernel<<<dim3(n_chunks, n_nodes), NC, 0, s>>>(a);
    fmm_m2l_combine_kernel<<<dim3(n_nodes, 10), NC, 0, s>>>(a, n_chunks);
    return cudaGetLastError();
}

cudaError_t launch_fmm_m2l_part_flat(const FmmArgs& a, int n_nodes, int root_node, const FmmEntry* root_tab,
                                     int n_root_tab, cudaStream_t s) {
    const int n_far = (a.n_table + kFmmChunk - 1) / kFmmChunk;
    const int n_root = root_node >= 0 ? (n_root_tab + kFmmChunk - 1) / kFmmChunk : 0;
    const int n_ctas = n_root + n_nodes * n_far;
    if (n_ctas <= 0) return cudaSuccess;
    fmm_m2l_part_flat_kernel<<<n_ctas, NC, 0, s>>>(a, root_node, n_root, root_tab, n_root_tab, n_far, n_nodes * n_far);
    return cudaGetLastError();
}

cudaError_t launch_fmm_m2l_combine(const FmmArgs& a, int n_nodes, cudaStream_t s) {
    const int n_chunks = (a.n_table + kFmmChunk - 1) / kFmmChunk;
    if (n_nodes <= 0 || n_chunks <= 0) return cudaSuccess;
    fmm_m2l_combine_kernel<<<dim3(n_nodes, 10), NC, 0, s>>>(a, n_chunks);
    return cudaGetLastError();
}

cudaError_t launch_fmm_leaf(const FmmArgs& a, int n_ctas, bool restricted, cudaStream_t s) {
    if (n_ctas <= 0) return cudaSuccess;
    cudaError_t e = ensure_device_setup();
    if (e != cudaSuccess) return e;
    if (a.K < 1 || a.K > kFmmRootK) return cudaErrorInvalidValue;
    const size_t smem = tile_bytes(a.K);
    // the R = 1, 2 depth >= 1 tables unrolled; R = 3 and the root's table at run time
    const int sel = a.n_table == kTabMax1 ? 1 : (a.n_table == kTabMax2 ? 2 : 0);
    // two cells per thread: 0.262 ms for the 16^3 Sedov leaves at R = 2,
    // against 0.277 for one and 0.388 for four (128 threads: 12 warps/SM)
#define TS_FMM_LEAF_LAUNCH(RS, RESTR) fmm_leaf_kernel<RS, RESTR, 2><<<n_ctas, NC / 2, smem, s>>>(a)
    if (sel == 1) restricted ? TS_FMM_LEAF_LAUNCH(1, true) : TS_FMM_LEAF_LAUNCH(1, false);
    else if (sel == 2) restricted ? TS_FMM_LEAF_LAUNCH(2, true) : TS_FMM_LEAF_LAUNCH(2, false);
    else restricted ? TS_FMM_LEAF_LAUNCH(0, true) : TS_FMM_LEAF_LAUNCH(0, false);
#undef TS_FMM_LEAF_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_gravity_kick(double* U, int nf, long long n, const double* grav, const double* dt_dev, double dt,
                                unsigned long long* stamp, int sms, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const long long cells = n * NC;
    const int blocks = (int)std::min<long long>((cells + 255) / 256, 8LL * sms);
    gravity_kick_kernel<<<blocks, 256, 0, s>>>(U, nf, n, grav, dt_dev, dt, stamp);
    return cudaGetLastError();
}

}  // namespace tsh
