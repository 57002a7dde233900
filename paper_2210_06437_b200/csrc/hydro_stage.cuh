// hydro_stage.cuh — the fused reconstruct + Kurganov–Tadmor flux + SSP-RK3
// stage kernel (one sub-grid per 64-thread CTA).  Instantiated once per field
// count in stage_nf*.cu so the variants build in parallel.
#pragma once

#include <cstdint>

#include "hydro_device.cuh"
#include "hydro_kernels.h"

namespace tsh {

// ---------------------------------------------------------------------------
// Fused stage kernel
// ---------------------------------------------------------------------------

template <int AXIS>
__device__ __forceinline__ int cell_off(int a, int b, int s) {
    if (AXIS == 0) return (b * N + a) * N + s;
    if (AXIS == 1) return (b * N + s) * N + a;
    return (s * N + b) * N + a;
}

// Shared-memory slot of cell (x, y, z): rows XOR-swizzled by y to spread
// the x-sweep's column writes over the banks.
__device__ __forceinline__ int sm_off(int x, int y, int z) { return (z * N + y) * N + (x ^ y); }

template <int AXIS>
__device__ __forceinline__ int sm_cell(int a, int b, int s) {
    if (AXIS == 0) return sm_off(s, a, b);
    if (AXIS == 1) return sm_off(a, s, b);
    return sm_off(a, b, s);
}

// 14-cell pencil of one field: own interior + 3 cells of each face neighbour
// read directly from its interior (the direct_local path of workload.cpp:532-536),
// or clamped at a domain boundary (outflow).
template <int AXIS>
__device__ __forceinline__ void load_pencil(double (&q)[P], const double* __restrict__ own,
                                            const double* __restrict__ lo,
                                            const double* __restrict__ hi, int a, int b) {
    if (AXIS == 0) {
        const double2* row = reinterpret_cast<const double2*>(own + cell_off<0>(a, b, 0));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 v = __ldg(row + k);
            q[3 + 2 * k] = v.x;
            q[4 + 2 * k] = v.y;
        }
    } else {
#pragma unroll
        for (int s = 0; s < N; ++s) q[s + 3] = __ldg(own + cell_off<AXIS>(a, b, s));
    }
    if (lo != nullptr) {
#pragma unroll
        for (int s = 0; s < 3; ++s) q[s] = __ldg(lo + cell_off<AXIS>(a, b, N - 3 + s));
    } else {
        q[0] = q[3];
        q[1] = q[3];
        q[2] = q[3];
    }
    if (hi != nullptr) {
#pragma unroll
        for (int s = 0; s < 3; ++s) q[N + 3 + s] = __ldg(hi + cell_off<AXIS>(a, b, s));
    } else {
        q[N + 3] = q[N + 2];
        q[N + 4] = q[N + 2];
        q[N + 5] = q[N + 2];
    }
}

// Running reconstruction state of one field along the pencil.
struct Recon {
    double D;     // limited slope of the current cell (PPM)
    double fc;    // interface value at the current cell's left face (PPM)
    double hi;    // limited right state of the previous cell
    double dlast; // q[i+1] - q[i]
};

// Cells -2, -1 (array 1, 2): leaves state ready for cell 0 (array 3).
template <int RECON>
__device__ __forceinline__ void recon_begin(const double (&q)[P], Recon& r) {
    if (RECON == 0) {
        const double d0 = q[1] - q[0];
        const double d1 = q[2] - q[1];
        const double d2 = q[3] - q[2];
        const double D1 = mc_slope(d1, d0);
        const double D2 = mc_slope(d2, d1);
        const double f2 = ppm_face(q[1], q[2], D1, D2);
        const double d3 = q[4] - q[3];
        const double D3 = mc_slope(d3, d2);
        const double f3 = ppm_face(q[2], q[3], D2, D3);
        double l = f2, h = f3;
        ppm_limit(l, q[2], h);
        r.hi = h;
        r.D = D3;
        r.fc = f3;
        r.dlast = d3;
    } else {
        const double d1 = q[2] - q[1];
        const double d2 = q[3] - q[2];
        const double s = minmod_slope(d2, d1);
        r.hi = fma(0.5, s, q[2]);
        r.dlast = d2;
    }
}

// Advance to cell j (array i = j + 3); returns the states of face j
// (between cells j-1 and j): uL = right edge of j-1, uR = left edge of j.
template <int RECON, int J>
__device__ __forceinline__ void recon_step(const double (&q)[P], Recon& r, double& uL, double& uR) {
    constexpr int i = J + 3;
    if (RECON == 0) {
        const double dn = q[i + 2] - q[i + 1];
        const double Dn = mc_slope(dn, r.dlast);
        const double fn = ppm_face(q[i], q[i + 1], r.D, Dn);
        double l = r.fc, h = fn;
        ppm_limit(l, q[i], h);
        uL = r.hi;
        uR = l;
        r.hi = h;
        r.D = Dn;
        r.fc = fn;
        r.dlast = dn;
    } else {
        const double dn = q[i + 1] - q[i];
        const double s = minmod_slope(dn, r.dlast);
        uL = r.hi;
        uR = fma(-0.5, s, q[i]);
        r.hi = fma(0.5, s, q[i]);
        r.dlast = dn;
    }
}

struct SweepCtx {
    const double* __restrict__ Uprev;
    const double* __restrict__ Un;
    double* __restrict__ Uout;
    double* __restrict__ dU;  // shared
    size_t own;               // element offset of the sub-grid's field 0
    long long lo, hi;         // element offsets of the face neighbours' field 0, -1 if none
    int a, b;
    double dtdx;
    EosParams e;
};

// Accumulate the flux difference of cell c for field f.
//   MODE 0: dU  = d            (x sweep)
//   MODE 1: dU += d            (y sweep)
//   MODE 2: U_out = RK(U_n, U_prev + dtdx (dU + d))   (z sweep, fused update)
template <int AXIS, int NF, int MODE, int STAGE>
__device__ __forceinline__ double accumulate(const SweepCtx& c, int f, int cell, double d,
                                             double uprev) {
    const int sm = f * NC + sm_cell<AXIS>(c.a, c.b, cell);
    if (MODE == 0) {
        c.dU[sm] = d;
        return 0.0;
    } else if (MODE == 1) {
        c.dU[sm] = c.dU[sm] + d;
        return 0.0;
    } else {
        const double tot = c.dU[sm] + d;
        const double ustar = fma(c.dtdx, tot, uprev);
        const size_t at = c.own + (size_t)f * NC + cell_off<AXIS>(c.a, c.b, cell);
        double out;
        if (STAGE == 1) {
            out = ustar;
        } else if (STAGE == 2) {
            out = fma(0.75, __ldg(c.Un + at), 0.25 * ustar);
        } else {
            out = fma(1.0 / 3.0, __ldg(c.Un + at), (2.0 / 3.0) * ustar);
        }
        c.Uout[at] = out;
        return out;
    }
}

template <int AXIS, int NF, int RECON, int MODE, int STAGE, int J>
__device__ __forceinline__ void hydro_face(const SweepCtx& c, const double (&q)[5][P], Recon (&r)[5],
                                           double (&Fprev)[5], double (&vLc)[N + 1],
                                           double (&vRc)[N + 1], double (&ac)[N + 1], double& amax) {
    double uL[5], uR[5];
#pragma unroll
    for (int f = 0; f < 5; ++f) recon_step<RECON, J>(q[f], r[f], uL[f], uR[f]);
    double vL, pL, aL, vR, pR, aR;
    face_eos<AXIS>(uL, c.e, vL, pL, aL);
    face_eos<AXIS>(uR, c.e, vR, pR, aR);
    const double a = fmax(aL, aR);
    double fL[5], fR[5], F[5];
    hydro_flux<AXIS>(uL, vL, pL, fL);
    hydro_flux<AXIS>(uR, vR, pR, fR);
#pragma unroll
    for (int f = 0; f < 5; ++f) F[f] = kt(a, uL[f], uR[f], fL[f], fR[f]);
    if (NF > 5) {
        vLc[J] = vL;
        vRc[J] = vR;
        ac[J] = a;
    }
    if (J > 0) {
        double out[5];
#pragma unroll
        for (int f = 0; f < 5; ++f)
            out[f] = accumulate<AXIS, NF, MODE, STAGE>(c, f, J - 1, Fprev[f] - F[f], q[f][J + 2]);
        if (MODE == 2 && STAGE == 3)
            amax = fmax(amax, cell_signal_speed(out[0], out[1], out[2], out[3], out[4], c.e));
    }
#pragma unroll
    for (int f = 0; f < 5; ++f) Fprev[f] = F[f];
}

template <int AXIS, int NF, int RECON, int MODE, int STAGE, int J>
__device__ __forceinline__ void passive_face(const SweepCtx& c, int f, const double (&q)[P], Recon& r,
                                             double& Fprev, const double (&vLc)[N + 1],
                                             const double (&vRc)[N + 1], const double (&ac)[N + 1]) {
    double uL, uR;
    recon_step<RECON, J>(q, r, uL, uR);
    const double F = kt(ac[J], uL, uR, uL * vLc[J], uR * vRc[J]);
    if (J > 0) accumulate<AXIS, NF, MODE, STAGE>(c, f, J - 1, Fprev - F, q[J + 2]);
    Fprev = F;
}

template <int AXIS, int NF, int RECON, int MODE, int STAGE>
__device__ __forceinline__ void sweep(const SweepCtx& c, double& amax) {
    const double* lo = c.lo >= 0 ? c.Uprev + c.lo : nullptr;
    const double* hi = c.hi >= 0 ? c.Uprev + c.hi : nullptr;
    double vLc[N + 1], vRc[N + 1], ac[N + 1];
    {
        double q[5][P];
#pragma unroll
        for (int f = 0; f < 5; ++f)
            load_pencil<AXIS>(q[f], c.Uprev + c.own + (size_t)f * NC, lo ? lo + (size_t)f * NC : nullptr,
                              hi ? hi + (size_t)f * NC : nullptr, c.a, c.b);
        Recon r[5];
#pragma unroll
        for (int f = 0; f < 5; ++f) recon_begin<RECON>(q[f], r[f]);
        double Fprev[5];
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 0>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 1>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 2>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 3>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 4>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 5>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 6>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 7>(c, q, r, Fprev, vLc, vRc, ac, amax);
        hydro_face<AXIS, NF, RECON, MODE, STAGE, 8>(c, q, r, Fprev, vLc, vRc, ac, amax);
    }
#pragma unroll 1
    for (int f = 5; f < NF; ++f) {
        double q[P];
        load_pencil<AXIS>(q, c.Uprev + c.own + (size_t)f * NC, lo ? lo + (size_t)f * NC : nullptr,
                          hi ? hi + (size_t)f * NC : nullptr, c.a, c.b);
        Recon r;
        recon_begin<RECON>(q, r);
        double Fp;
        passive_face<AXIS, NF, RECON, MODE, STAGE, 0>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 1>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 2>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 3>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 4>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 5>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 6>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 7>(c, f, q, r, Fp, vLc, vRc, ac);
        passive_face<AXIS, NF, RECON, MODE, STAGE, 8>(c, f, q, r, Fp, vLc, vRc, ac);
    }
}

template <int NF, int RECON, int STAGE>
__global__ void __launch_bounds__(64) stage_kernel(StageArgs A) {
    extern __shared__ double dU[];
    if (A.stamp != nullptr && threadIdx.x == 0) atomicMax(A.stamp, ~globaltimer());  // start stored inverted: one zero-initialised ring serves both ends
    const int g = A.list != nullptr ? A.list[blockIdx.x] : A.first + (int)blockIdx.x;
    const int t = threadIdx.x;
    const double amax_in = *A.amax_in;
    const double dt = (A.cfl * A.dx) / amax_in;
    const double dtdx = dt / A.dx;
    if (STAGE == 1 && blockIdx.x == 0 && t == 0) {
        if (A.dt_out != nullptr) *A.dt_out = dt;
        if (A.amax_reset != nullptr) *A.amax_reset = 0.0;
    }
    int nb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) nb[k] = __ldg(A.nbr + 6 * g + k);
    SweepCtx c;
    c.Uprev = A.Uprev;
    c.Un = A.Un;
    c.Uout = A.Uout;
    c.dU = dU;
    c.own = (size_t)g * NF * NC;
    c.a = t & (N - 1);
    c.b = t >> 3;
    c.dtdx = dtdx;
    c.e = EosParams{A.gamma, A.gm1, A.p_floor};
    double amax = 0.0;

    c.lo = nb[0] >= 0 ? (long long)nb[0] * NF * NC : -1;
    c.hi = nb[1] >= 0 ? (long long)nb[1] * NF * NC : -1;
    sweep<0, NF, RECON, 0, STAGE>(c, amax);
    __syncthreads();
    c.lo = nb[2] >= 0 ? (long long)nb[2] * NF * NC : -1;
    c.hi = nb[3] >= 0 ? (long long)nb[3] * NF * NC : -1;
    sweep<1, NF, RECON, 1, STAGE>(c, amax);
    __syncthreads();
    c.lo = nb[4] >= 0 ? (long long)nb[4] * NF * NC : -1;
    c.hi = nb[5] >= 0 ? (long long)nb[5] * NF * NC : -1;
    sweep<2, NF, RECON, 2, STAGE>(c, amax);

    if (STAGE == 3) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if ((t & 31) == 0) atomic_max_nonneg(A.amax_out, amax);
    }
    if (A.stamp != nullptr) {
        __syncthreads();
        if (t == 0) atomicMax(A.stamp + 1, globaltimer());
    }
}

template <int NF, int RECON, int STAGE>
inline cudaError_t launch_stage_t(const StageArgs& a, int n_ctas, cudaStream_t s) {
    const size_t smem = (size_t)NF * NC * sizeof(double);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(stage_kernel<NF, RECON, STAGE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    stage_kernel<NF, RECON, STAGE><<<n_ctas, 64, smem, s>>>(a);
    return cudaGetLastError();
}

template <int NF, int RECON>
inline cudaError_t launch_stage_r(const StageArgs& a, int stage, int n, cudaStream_t s) {
    switch (stage) {
        case 1: return launch_stage_t<NF, RECON, 1>(a, n, s);
        case 2: return launch_stage_t<NF, RECON, 2>(a, n, s);
        case 3: return launch_stage_t<NF, RECON, 3>(a, n, s);
    }
    return cudaErrorInvalidValue;
}

template <int NF>
cudaError_t launch_stage_n(const StageArgs& a, int recon, int stage, int n, cudaStream_t s) {
    return recon == 0 ? launch_stage_r<NF, 0>(a, stage, n, s) : launch_stage_r<NF, 1>(a, stage, n, s);
}

}  // namespace tsh
