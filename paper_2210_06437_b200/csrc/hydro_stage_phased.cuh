// hydro_stage_phased.cuh — phased variant of the fused stage kernel (nf = 6).
//
// Same numerics, operation by operation, as hydro_stage.cuh (bitwise); a
// different mapping of the work to threads.  Per sweep direction:
//   R  one thread per (field, pencil): the whole 14-cell pencil of one field
//      is reconstructed fully unrolled (no rolling window to move around,
//      ~40 registers) and its 9 face-state pairs go to shared memory;
//   F  one thread per (face, pencil): EOS of both states + KT flux of all
//      fields, written back in place of the left states;
//   D  one thread per (field, pencil): flux differences of its 8 cells into
//      the shared accumulator — or, in the last sweep, the RK update to HBM.
// 384 threads per CTA, 2 CTAs per SM (80 KB shared each): 24 warps per SM
// against 12 for the register-heavy march, and no window moves.
#pragma once

#include "hydro_stage.cuh"

namespace tsh {

constexpr int kPhThreads = 384;  // 6 fields x 64 pencils
constexpr int kPhFields = 6;

struct PhSmem {
    static constexpr int st = kPhFields * kFaces * 2 * kPencils;  // face states [f][j][side][p]
    static constexpr int dU = kPhFields * NC;
    static constexpr int doubles = st + dU;
};

__device__ __forceinline__ int st_idx(int f, int j, int side, int p) { return ((f * kFaces + j) * 2 + side) * kPencils + p; }

// R phase: reconstruct all faces of one field along one pencil.
template <int RECON>
__device__ __forceinline__ void ph_reconstruct(const Pencil& p, int fo, double* st, int f, int pen) {
    double q[P];
#pragma unroll
    for (int s = 0; s < P; ++s) q[s] = __ldg(paddr(p, s - 3) + fo);
    double lo[P], hi[P];
    if (RECON == 0) {
        double D[P], fc[P];
#pragma unroll
        for (int i = 1; i <= P - 2; ++i) D[i] = mc_slope(q[i + 1] - q[i], q[i] - q[i - 1]);
#pragma unroll
        for (int i = 2; i <= P - 2; ++i) fc[i] = ppm_face(q[i - 1], q[i], D[i - 1], D[i]);
#pragma unroll
        for (int i = 2; i <= P - 3; ++i) {
            double l = fc[i], h = fc[i + 1];
            ppm_limit(l, q[i], h);
            lo[i] = l;
            hi[i] = h;
        }
    } else {
#pragma unroll
        for (int i = 2; i <= P - 3; ++i) {
            const double s = minmod_slope(q[i + 1] - q[i], q[i] - q[i - 1]);
            lo[i] = fma(-0.5, s, q[i]);
            hi[i] = fma(0.5, s, q[i]);
        }
    }
#pragma unroll
    for (int j = 0; j < kFaces; ++j) {
        st[st_idx(f, j, 0, pen)] = hi[j + 2];  // right edge of cell j-1
        st[st_idx(f, j, 1, pen)] = lo[j + 3];  // left edge of cell j
    }
}

template <int NF, int RECON, int STAGE>
__global__ void __launch_bounds__(kPhThreads, 2) stage_kernel_phased(StageArgs A) {
    static_assert(NF == kPhFields, "phased kernel: nf = 6");
    extern __shared__ double smem[];
    double* st = smem;
    double* dU = smem + PhSmem::st;
    if (A.stamp != nullptr && threadIdx.x == 0) atomicMax(A.stamp, ~globaltimer());
    const int g = A.list != nullptr ? A.list[blockIdx.x] : A.first + (int)blockIdx.x;
    const int t = threadIdx.x;
    if (STAGE == 1 && A.wait_n > 0) {
        if (t == 0)
            for (int q = 0; q < A.wait_n; ++q)
                if (q != A.rank)
                    while ((int)(ld_acquire_sys(A.wait_flags + q) - A.wait_seq) < 0) {
                    }
        __syncthreads();
    }
    double amax_in = A.amax_in[0];
    for (int i = 1; i < A.amax_n; ++i) amax_in = fmax(amax_in, A.amax_in[i]);
    const double dt = (A.cfl * A.dx) / amax_in;
    const double dtdx = dt / A.dx;
    if (STAGE == 1 && blockIdx.x == 0 && t == 0) {
        if (A.dt_out != nullptr) *A.dt_out = dt;
        if (A.amax_reset != nullptr) *A.amax_reset = 0.0;
    }
    const EosParams e{A.gamma, A.gm1, A.p_floor};
    const size_t own_off = (size_t)g * NF * NC;
    const double* own = A.Uprev + own_off;
    const int kf = t >> 6;          // R / D phases: field slot
    const int pen = t & (kPencils - 1);
    const int pa = pen & (N - 1), pb = pen >> 3;
    double amax = 0.0;

#pragma unroll 1
    for (int axis = 0; axis < 3; ++axis) {
        const int nlo = __ldg(A.nbr + 6 * g + 2 * axis);
        const int nhi = __ldg(A.nbr + 6 * g + 2 * axis + 1);
        const int fm[kFA] = {0, 1 + axis, axis == 0 ? 2 : 1, axis == 2 ? 2 : 3, 4, 5};
        Pencil p;
        p.own = own;
        p.lo = nlo >= 0 ? A.Uprev + (size_t)nlo * NF * NC : nullptr;
        p.hi = nhi >= 0 ? A.Uprev + (size_t)nhi * NF * NC : nullptr;
        p.ss = axis == 0 ? 1 : (axis == 1 ? N : N * N);
        // ---- R
        {
            const int fmk = kf == 0 ? fm[0] : kf == 1 ? fm[1] : kf == 2 ? fm[2] : kf == 3 ? fm[3] : kf == 4 ? fm[4] : fm[5];
            p.base = axis == 0 ? (pb * N + pa) * N : (axis == 1 ? pb * N * N + pa : pb * N + pa);
            ph_reconstruct<RECON>(p, fmk * NC, st, kf, pen);
        }
        __syncthreads();
        // ---- F: (face, pencil) items
#pragma unroll 1
        for (int it = t; it < kFaces * kPencils; it += kPhThreads) {
            const int j = it >> 6, pp = it & (kPencils - 1);
            double uL[kFA], uR[kFA];
#pragma unroll
            for (int k = 0; k < kFA; ++k) {
                uL[k] = st[st_idx(k, j, 0, pp)];
                uR[k] = st[st_idx(k, j, 1, pp)];
            }
            double F[kFA], vL, vR, a;
            kt_face(e, uL, uR, F, vL, vR, a);
#pragma unroll
            for (int k = 0; k < kFA; ++k) st[st_idx(k, j, 0, pp)] = F[k];
        }
        __syncthreads();
        // ---- D: (field, pencil) items, 8 cells each
        {
            const int fmk = kf == 0 ? fm[0] : kf == 1 ? fm[1] : kf == 2 ? fm[2] : kf == 3 ? fm[3] : kf == 4 ? fm[4] : fm[5];
            const int base = p.base;
            double* dUf = dU + fmk * NC;
            if (axis < 2) {
                double Fl = st[st_idx(kf, 0, 0, pen)];
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    const double Fr = st[st_idx(kf, i + 1, 0, pen)];
                    const int slot = sm_slot(base + i * p.ss);
                    dUf[slot] = axis == 0 ? (Fl - Fr) : dUf[slot] + (Fl - Fr);
                    Fl = Fr;
                }
            } else {
                const double* up = own + fmk * NC + base;
                const double* un = A.Un + own_off + fmk * NC + base;
                double* out = A.Uout + own_off + fmk * NC + base;
                double Fl = st[st_idx(kf, 0, 0, pen)];
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    const double Fr = st[st_idx(kf, i + 1, 0, pen)];
                    const int o = i * p.ss;
                    const double tot = dUf[sm_slot(base + o)] + (Fl - Fr);
                    const double ustar = fma(dtdx, tot, __ldg(up + o));
                    double r;
                    if (STAGE == 1)
                        r = ustar;
                    else if (STAGE == 2)
                        r = fma(0.75, __ldg(un + o), 0.25 * ustar);
                    else
                        r = fma(1.0 / 3.0, __ldg(un + o), (2.0 / 3.0) * ustar);
                    out[o] = r;
                    if (STAGE == 3) st[st_idx(kf, i, 1, pen)] = r;  // for the signal speed below
                    Fl = Fr;
                }
            }
        }
        __syncthreads();
    }
    if (STAGE == 3) {
        // cell-centred signal speed of U^{n+1}: z-sweep field slots (rho, sz, sx, sy, E)
        for (int it = t; it < NC; it += kPhThreads) {
            const int i = it >> 6, pp = it & (kPencils - 1);
            amax = fmax(amax, cell_signal_speed(st[st_idx(0, i, 1, pp)], st[st_idx(2, i, 1, pp)],
                                                st[st_idx(3, i, 1, pp)], st[st_idx(1, i, 1, pp)],
                                                st[st_idx(4, i, 1, pp)], e));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if ((t & 31) == 0) atomic_max_nonneg(A.amax_out, amax);
        if (A.push_n > 0) {
            __syncthreads();
            if (t == 0) {
                __threadfence();
                if (atomicAdd(A.done_ctr, 1u) == (unsigned)A.total_ctas - 1u) {
                    __threadfence();
                    const double am = __longlong_as_double(
                        (long long)atomicAdd(reinterpret_cast<unsigned long long*>(A.amax_out), 0ull));
                    for (int q = 0; q < A.push_n; ++q) A.push_gather[q][A.rank] = am;
                    __threadfence_system();
                    for (int q = 0; q < A.push_n; ++q)
                        if (A.push_flag[q] != nullptr) atomicExch_system(A.push_flag[q], A.seq);
                    *A.done_ctr = 0u;
                }
            }
        }
    }
    if (A.stamp != nullptr) {
        __syncthreads();
        if (t == 0) atomicMax(A.stamp + 1, globaltimer());
    }
}

template <int NF, int RECON, int STAGE>
inline cudaError_t launch_stage_phased_t(const StageArgs& a, int n_ctas, cudaStream_t s) {
    const size_t smem = (size_t)PhSmem::doubles * sizeof(double);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(stage_kernel_phased<NF, RECON, STAGE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    stage_kernel_phased<NF, RECON, STAGE><<<n_ctas, kPhThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace tsh
