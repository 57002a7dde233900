// amr_kernels.cu — coarse–fine AMR boundaries (SURVEY.md §8(f) rank 2,
// DESIGN.md §11): the proxy fill (prolongation / restriction ghosts) before
// each RK stage and the coarse flux correction after it.
//
// The reference's octree (build_mesh, workload.cpp:264-327) links only
// same-level faces (Mesh::validate, workload.cpp:160-161); Octo-Tiger fills
// coarse–fine ghosts from the other level and corrects the coarse fluxes
// (PAPER.md:346).  Here a leaf whose face neighbour sits on another level
// points at a proxy sub-grid slot (like the halo proxies of foreign
// neighbours), so the fused stage kernel runs unchanged; these two kernels
// are the only AMR-specific device code.  Both follow oracle/hydro_oracle.c
// (orc_amr_fill, orc_amr_reflux) operation for operation (--fmad=false), so
// the AMR path is bitwise equal to the oracle.
//
// Neither kernel is on the uniform-mesh hot path; they are latency-light
// (proxy fill: 4 KB·nf copied or averaged per proxy; reflux: one CTA per
// coarse sub-grid with a coarse–fine face, five face fluxes per face cell).
#include "hydro_device.cuh"
#include "hydro_kernels.h"

namespace tsh {
namespace {

__device__ __forceinline__ int cidx(int x, int y, int z) { return (z * N + y) * N + x; }

// Activity stamps in the kernel itself (as the stage kernel does): start
// stored inverted, both ends by atomicMax into the zeroed ring slot — no
// stamp launches around the kernel.
__device__ __forceinline__ void stamp_begin(unsigned long long* stamp) {
    if (stamp != nullptr && threadIdx.x == 0) atomicMax(stamp, ~globaltimer());
}
__device__ __forceinline__ void stamp_end(unsigned long long* stamp) {
    if (stamp != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(stamp + 1, globaltimer());
    }
}

__device__ __forceinline__ void fill_cells(double* __restrict__ U, int nf, const AmrProxy& r, int c);

__global__ void __launch_bounds__(NC) amr_fill_kernel(double* __restrict__ U, int nf, const AmrProxy* px,
                                                       const unsigned char* __restrict__ face_mask,
                                                       unsigned long long* stamp) {
    stamp_begin(stamp);
    const int c = threadIdx.x;
    const int x = c & 7, y = (c >> 3) & 7, z = c >> 6;
    bool read = true;
    if (face_mask != nullptr) {
        // only the H = 3 layers next to a face some sub-grid reads through
        constexpr int H = 3;
        const unsigned m = face_mask[blockIdx.x];
        read = ((m & 1u) && x < H) || ((m & 2u) && x >= N - H) || ((m & 4u) && y < H) ||
               ((m & 8u) && y >= N - H) || ((m & 16u) && z < H) || ((m & 32u) && z >= N - H);
    }
    if (read) fill_cells(U, nf, px[blockIdx.x], c);
    stamp_end(stamp);
}

__device__ __forceinline__ void fill_cells(double* __restrict__ U, int nf, const AmrProxy& r, int c) {
    const int x = c & 7, y = (c >> 3) & 7, z = c >> 6;
    double* dst = U + (size_t)r.dst * nf * NC + c;
    if (r.kind == 0) {
        const int cc = cidx((r.octant & 1) * 4 + x / 2, ((r.octant >> 1) & 1) * 4 + y / 2,
                            ((r.octant >> 2) & 1) * 4 + z / 2);
        const double* s = U + (size_t)r.src[0] * nf * NC + cc;
        for (int f = 0; f < nf; ++f) dst[(size_t)f * NC] = s[(size_t)f * NC];
    } else {
        const int o = (x >> 2) | ((y >> 2) << 1) | ((z >> 2) << 2);
        const int bx = 2 * (x & 3), by = 2 * (y & 3), bz = 2 * (z & 3);
        for (int f = 0; f < nf; ++f) {
            const double* s = U + ((size_t)r.src[o] * nf + f) * NC;
            double sum = s[cidx(bx, by, bz)];
            sum = sum + s[cidx(bx + 1, by, bz)];
            sum = sum + s[cidx(bx, by + 1, bz)];
            sum = sum + s[cidx(bx + 1, by + 1, bz)];
            sum = sum + s[cidx(bx, by, bz + 1)];
            sum = sum + s[cidx(bx + 1, by, bz + 1)];
            sum = sum + s[cidx(bx, by + 1, bz + 1)];
            sum = sum + s[cidx(bx + 1, by + 1, bz + 1)];
            dst[(size_t)f * NC] = 0.125 * sum;
        }
    }
}

// ---- scalar face flux, the oracle's reconstruct / side_flux / kt_flux -------
constexpr int kMaxNf = 16;
constexpr double kC16 = 1.0 / 6.0;

__device__ double o_minmod(double a, double b) {
    return (copysign(0.5, a) + copysign(0.5, b)) * fmin(fabs(a), fabs(b));
}
__device__ double o_minmod_theta(double a, double b, double theta) {
    return o_minmod(theta * o_minmod(a, b), 0.5 * (a + b));
}
__device__ void o_limit_slope(double* ql, double q0, double* qr) {
    if ((*qr < q0) != (q0 < *ql)) {
        *ql = q0;
        *qr = q0;
        return;
    }
    const double t1 = *qr - *ql;
    const double t2 = *qr + *ql;
    const double t3 = (t1 * t1) * kC16;
    const double t4 = t1 * (q0 - 0.5 * t2);
    if (t4 > t3) {
        *ql = fma(-2.0, *qr, 3.0 * q0);
    } else if (-t3 > t4) {
        *qr = fma(-2.0, *ql, 3.0 * q0);
    }
}

// Face states of face j (0..N) from the pencil window w[k] = q[j + k],
// k = 0..5 (cells j-3 .. j+2): the oracle's reconstruct restricted to the two
// cells either side of the face (the same per-element formulas, so the same
// bits): uL = hi of cell j-1 (q index j+2), uR = lo of cell j (q index j+3).
__device__ void o_face_states(int recon, const double* w, double* uL, double* uR) {
    if (recon == 0) {
        double D[5], fc[5];  // index k <-> oracle index j + k
        for (int k = 1; k <= 4; ++k) D[k] = o_minmod_theta(w[k + 1] - w[k], w[k] - w[k - 1], 2.0);
        for (int k = 2; k <= 4; ++k) fc[k] = fma(kC16, D[k - 1] - D[k], 0.5 * (w[k - 1] + w[k]));
        double ql = fc[2], qr = fc[3];
        o_limit_slope(&ql, w[2], &qr);
        *uL = qr;
        ql = fc[3];
        qr = fc[4];
        o_limit_slope(&ql, w[3], &qr);
        *uR = ql;
    } else {
        const double sl = o_minmod(w[3] - w[2], w[2] - w[1]);
        const double sr = o_minmod(w[4] - w[3], w[3] - w[2]);
        *uL = fma(0.5, sl, w[2]);
        *uR = fma(-0.5, sr, w[3]);
    }
}

struct FluxParams {
    int nf, recon;
    double gamma, p_floor;
};

__device__ void o_side_flux(const FluxParams& p, int axis, const double* u, double* f, double* vn, double* c2) {
    const double rho = u[0], sx = u[1], sy = u[2], sz = u[3], E = u[4];
    const double inv = 1.0 / rho;
    const double vx = sx * inv, vy = sy * inv, vz = sz * inv;
    const double s3[3] = {sx, sy, sz}, v3[3] = {vx, vy, vz};
    const int t1 = axis == 0 ? 1 : 0, t2 = axis == 2 ? 1 : 2;
    const double ke2 = fma(s3[axis], v3[axis], fma(s3[t1], v3[t1], s3[t2] * v3[t2]));
    double pr = (p.gamma - 1.0) * fma(-0.5, ke2, E);
    pr = fmax(pr, p.p_floor);
    const double v = v3[axis];
    *c2 = (p.gamma * pr) * inv;
    *vn = v;
    f[0] = u[1 + axis];
    f[1] = sx * v;
    f[2] = sy * v;
    f[3] = sz * v;
    f[1 + axis] = fma(u[1 + axis], v, pr);
    f[4] = (E + pr) * v;
    for (int k = 5; k < p.nf; ++k) f[k] = u[k] * v;
}

// Pencil cell s (-3..N+2) along `axis` through (a, b) of local sub-grid g
// (oracle pencil_value: face neighbour or clamp at an outflow boundary).
__device__ double o_pencil_value(int nf, const int* nbr, const double* U, int g, int f, int axis, int a, int b,
                                 int s) {
    int h = g;
    if (s < 0) {
        const int nb = nbr[6 * g + 2 * axis];
        if (nb >= 0) {
            h = nb;
            s += N;
        } else {
            s = 0;
        }
    } else if (s >= N) {
        const int nb = nbr[6 * g + 2 * axis + 1];
        if (nb >= 0) {
            h = nb;
            s -= N;
        } else {
            s = N - 1;
        }
    }
    const int c = axis == 0 ? cidx(s, a, b) : (axis == 1 ? cidx(a, s, b) : cidx(a, b, s));
    return U[((size_t)h * nf + f) * NC + c];
}

__device__ void o_face_flux(const FluxParams& p, const int* nbr, const double* U, int g, int axis, int a, int b,
                            int j, double* F) {
    double w[6], sL[kMaxNf], sR[kMaxNf], fL[kMaxNf], fR[kMaxNf], vL, vR, c2L, c2R;
    for (int f = 0; f < p.nf; ++f) {
        for (int k = 0; k < 6; ++k) w[k] = o_pencil_value(p.nf, nbr, U, g, f, axis, a, b, j + k - 3);
        o_face_states(p.recon, w, &sL[f], &sR[f]);
    }
    o_side_flux(p, axis, sL, fL, &vL, &c2L);
    o_side_flux(p, axis, sR, fR, &vR, &c2R);
    const double am = fmax(fabs(vL), fabs(vR)) + sqrt(fmax(c2L, c2R));
    for (int k = 0; k < p.nf; ++k) F[k] = 0.5 * fma(-am, sR[k] - sL[k], fL[k] + fR[k]);
}

// One CTA per coarse sub-grid with a coarse–fine face.  Per face (in order
// 0..5, barrier-separated, so an edge cell corrected through two faces gets
// the oracle's order) the 5 x 64 face fluxes — the coarse one and the 4 fine
// ones behind each coarse face cell — are computed by 320 threads into shared
// memory (one flux each: the work is latency-bound scalar code, so the
// parallelism matters more than the redundancy), then the 64 face cells'
// threads apply the correction.
constexpr int kRefluxThreads = 5 * N * N;

__global__ void __launch_bounds__(kRefluxThreads) amr_reflux_kernel(const double* __restrict__ Uprev, double* Uout,
                                                                   FluxParams p, const int* nbr, const int* level,
                                                                   int max_level, double dx, const AmrReflux* rf,
                                                                   int stage, const double* dt_ptr,
                                                                   unsigned long long* stamp) {
    stamp_begin(stamp);
    __shared__ double Fs[5][kMaxNf][N * N];
    const AmrReflux& r = rf[blockIdx.x];
    const int g = r.coarse;
    const double w = stage == 1 ? 1.0 : (stage == 2 ? 0.25 : 2.0 / 3.0);
    const double dtdx = *dt_ptr / ldexp(dx, max_level - level[g]);
    const int cell = threadIdx.x & (N * N - 1), which = threadIdx.x / (N * N);  // which: 0 coarse, 1..4 fine
    const int a = cell & 7, b = cell >> 3;
    double F[kMaxNf];
    for (int face = 0; face < 6; ++face) {
        if (r.fine[face][0] < 0) continue;
        const int axis = face >> 1, side = face & 1;
        if (which == 0) {
            o_face_flux(p, nbr, Uprev, g, axis, a, b, side ? N : 0, F);
        } else {
            const int q = which - 1;  // 00, 10, 01, 11
            o_face_flux(p, nbr, Uprev, r.fine[face][(a >> 2) + 2 * (b >> 2)], axis, 2 * (a & 3) + (q & 1),
                        2 * (b & 3) + (q >> 1), side ? 0 : N, F);
        }
        for (int f = 0; f < p.nf; ++f) Fs[which][f][cell] = F[f];
        __syncthreads();
        if (which == 0) {
            const int ic = side ? N - 1 : 0;
            const int c = axis == 0 ? cidx(ic, a, b) : (axis == 1 ? cidx(a, ic, b) : cidx(a, b, ic));
            for (int f = 0; f < p.nf; ++f) {
                const double avg = 0.25 * ((Fs[1][f][cell] + Fs[2][f][cell]) + (Fs[3][f][cell] + Fs[4][f][cell]));
                const double Fc = Fs[0][f][cell];
                const double corr = side ? Fc - avg : avg - Fc;
                double* u = Uout + ((size_t)g * p.nf + f) * NC + c;
                *u = *u + w * (dtdx * corr);
            }
        }
        __syncthreads();
    }
    stamp_end(stamp);
}

// Reflux from the flux register (StageArgs::rf_slot): the stage kernel
// stored the doubled (kt2) flux of every coarse-fine face, both sides, while
// sweeping; here one 64-thread CTA per coarse leaf applies, face by face in
// order (an edge cell corrected through two faces keeps the oracle's order),
//   avg2 = 0.25 ((K1 + K2) + (K3 + K4)),  corr = 0.5 (side ? Kc - avg2 : avg2 - Kc),
// which is bitwise the recomputing kernel's corr (every flux there is 0.5 K,
// and scaling by 2 commutes with the roundings).
__global__ void __launch_bounds__(N * N) amr_reflux_reg_kernel(double* Uout, int nf, const int* level,
                                                              int max_level, double dx, const AmrReflux* rf,
                                                              const int* rf_slot, const double* rf_flux, int stage,
                                                              const double* dt_ptr, unsigned long long* stamp) {
    stamp_begin(stamp);
    const AmrReflux& r = rf[blockIdx.x];
    const int g = r.coarse;
    const double w = stage == 1 ? 1.0 : (stage == 2 ? 0.25 : 2.0 / 3.0);
    const double dtdx = *dt_ptr / ldexp(dx, max_level - level[g]);
    const int cell = threadIdx.x, a = cell & 7, b = cell >> 3;
    for (int face = 0; face < 6; ++face) {
        if (r.fine[face][0] < 0) continue;
        const int axis = face >> 1, side = face & 1;
        const double* Kc = rf_flux + (size_t)rf_slot[6 * g + face] * nf * NC / N;
        const int fl = r.fine[face][(a >> 2) + 2 * (b >> 2)];
        const double* Kf = rf_flux + (size_t)rf_slot[6 * fl + (face ^ 1)] * nf * NC / N;
        const int c0 = 2 * (a & 3) + 8 * (2 * (b & 3));  // fine face cell of quadrant q: c0 + (q & 1) + 8 (q >> 1)
        const int ic = side ? N - 1 : 0;
        const int c = axis == 0 ? cidx(ic, a, b) : (axis == 1 ? cidx(a, ic, b) : cidx(a, b, ic));
        for (int f = 0; f < nf; ++f) {
            const double* kf = Kf + f * N * N + c0;
            const double avg2 = 0.25 * ((kf[0] + kf[1]) + (kf[N] + kf[N + 1]));
            const double kc = Kc[f * N * N + cell];
            const double corr = 0.5 * (side ? kc - avg2 : avg2 - kc);
            double* u = Uout + ((size_t)g * nf + f) * NC + c;
            *u = *u + w * (dtdx * corr);
        }
        __syncthreads();
    }
    stamp_end(stamp);
}

}  // namespace

cudaError_t launch_amr_reflux_reg(double* Uout, int nf, const int* level, int max_level, double dx,
                                  const AmrReflux* rf, long long n, const int* rf_slot, const double* rf_flux,
                                  int stage, const double* dt, unsigned long long* stamp, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    amr_reflux_reg_kernel<<<(unsigned)n, N * N, 0, s>>>(Uout, nf, level, max_level, dx, rf, rf_slot, rf_flux, stage,
                                                          dt, stamp);
    return cudaGetLastError();
}

cudaError_t launch_amr_fill(double* U, int nf, const AmrProxy* px, const unsigned char* face_mask, long long n,
                            unsigned long long* stamp, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    amr_fill_kernel<<<(unsigned)n, NC, 0, s>>>(U, nf, px, face_mask, stamp);
    return cudaGetLastError();
}

cudaError_t launch_amr_reflux(const double* Uprev, double* Uout, int nf, int recon, double gamma, double p_floor,
                              const int* nbr, const int* level, int max_level, double dx, const AmrReflux* rf,
                              long long n, int stage, const double* dt, unsigned long long* stamp,
                              cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (nf > kMaxNf) return cudaErrorInvalidValue;
    FluxParams p{nf, recon, gamma, p_floor};
    amr_reflux_kernel<<<(unsigned)n, kRefluxThreads, 0, s>>>(Uprev, Uout, p, nbr, level, max_level, dx, rf, stage, dt,
                                                            stamp);
    return cudaGetLastError();
}

}  // namespace tsh
