// hydro_kernels.cu — sm_100a kernels of the hydro hot path.
//
//   stage_kernel      fused PPM/minmod reconstruction + Kurganov–Tadmor flux +
//                     SSP-RK3 stage update, one sub-grid per 64-thread CTA
//                     (replaces the simulated reconstruct_kernel + flux_kernel
//                     pair of reference workload.cpp:544-552);
//   signal_kernel     cell-centred CFL signal speed (warp-shuffle max);
//   init_random       the reference's cell_value generator as a state;
//   pack / unpack     packed 3-deep halo slabs for the cross-GPU exchange
//                     (the aggregated form of send_boundary / handle_boundary,
//                     workload.cpp:487-517);
//   face_exchange     the reference's 1-deep face ghost layer (workload.cpp:519-542);
//   fill_halo         padded 26-neighbour tiles (diagnostic / API parity).
//
// Layout in HBM: U[local sub-grid][field][z][y][x] FP64, one sub-grid's
// field = 4 KiB contiguous.  Owned sub-grids first, then halo proxies.
#include <cstdint>

#include "hydro_device.cuh"
#include "hydro_kernels.h"

namespace tsh {

// ---------------------------------------------------------------------------
// Signal speed (initial dt) — grid-stride over owned cells
// ---------------------------------------------------------------------------
template <int NF>
__global__ void __launch_bounds__(256) signal_kernel(const double* __restrict__ U, long long n_cells,
                                                     EosParams e, double* amax_out,
                                                     unsigned long long* stamp) {
    if (stamp != nullptr && threadIdx.x == 0) atomicMax(stamp, ~globaltimer());
    double amax = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_cells;
         i += (long long)gridDim.x * blockDim.x) {
        const long long g = i / NC;
        const int c = (int)(i % NC);
        const double* u = U + g * NF * NC + c;
        amax = fmax(amax, cell_signal_speed(__ldg(u), __ldg(u + NC), __ldg(u + 2 * NC),
                                            __ldg(u + 3 * NC), __ldg(u + 4 * NC), e));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(amax_out, amax);
    if (stamp != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(stamp + 1, globaltimer());
    }
}

// ---------------------------------------------------------------------------
// Synthetic state from the reference generator (same formula as the oracle)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) init_random_kernel(double* __restrict__ U, int nf,
                                                          const long long* __restrict__ gid,
                                                          long long n_cells, uint64_t seed,
                                                          double gamma) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_cells;
         i += (long long)gridDim.x * blockDim.x) {
        const long long g = i / NC;
        const int c = (int)(i % NC);
        const uint64_t id = (uint64_t)gid[g];
        double r[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) r[k] = cell_value(id, seed, (uint64_t)k * NC + (uint64_t)c);
        const double rho = 0.5 + r[0];
        const double vx = r[1] - 0.5, vy = r[2] - 0.5, vz = r[3] - 0.5;
        const double pr = 0.5 + r[4];
        const double v2 = fma(vx, vx, fma(vy, vy, vz * vz));
        double* u = U + g * nf * NC + c;
        u[0] = rho;
        u[NC] = rho * vx;
        u[2 * NC] = rho * vy;
        u[3 * NC] = rho * vz;
        u[4 * NC] = fma(0.5 * rho, v2, pr / (gamma - 1.0));
        u[5 * NC] = 0.5 + r[5];
        for (int k = 6; k < nf; ++k) u[k * NC] = rho * cell_value(id, seed, (uint64_t)k * NC + (uint64_t)c);
    }
}

// ---------------------------------------------------------------------------
// Packed halo slabs.  Slab of face `f` of a sub-grid: the 3 layers adjacent to
// that face, index k = l + 3 (u + 8 v) with l the depth coordinate along the
// face axis and (u, v) its free axes minor-first (face_cell_index order,
// workload.cpp:340-354).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int slab_cell(int face, int k) {
    const int l = k % 3;
    const int u = (k / 3) % N;
    const int v = k / (3 * N);
    const int d = (face & 1) ? N - 3 + l : l;
    switch (face >> 1) {
        case 0: return (v * N + u) * N + d;
        case 1: return (v * N + d) * N + u;
        default: return (d * N + v) * N + u;
    }
}

// cells = SLAB: entry {sub-grid, face} = the 3-deep slab of that face;
// cells = NC: entry {sub-grid, -} = the whole sub-grid (AMR ghost leaves)
__global__ void __launch_bounds__(256) pack_kernel(const double* __restrict__ U, int nf,
                                                   const int2* __restrict__ entries, long long n_entries,
                                                   double* __restrict__ buf, unsigned long long* stamp, int cells) {
    if (stamp != nullptr && threadIdx.x == 0) atomicMax(stamp, ~globaltimer());
    const long long total = n_entries * nf * cells;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(i % cells);
        const long long ef = i / cells;
        const int f = (int)(ef % nf);
        const long long e = ef / nf;
        const int2 en = entries[e];
        buf[i] = __ldg(U + ((size_t)en.x * nf + f) * NC + (cells == NC ? k : slab_cell(en.y, k)));
    }
    if (stamp != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(stamp + 1, globaltimer());
    }
}

__global__ void __launch_bounds__(256) unpack_kernel(double* __restrict__ U, int nf,
                                                     const int2* __restrict__ entries, long long n_entries,
                                                     const double* __restrict__ buf, unsigned long long* stamp,
                                                     int cells) {
    if (stamp != nullptr && threadIdx.x == 0) atomicMax(stamp, ~globaltimer());
    const long long total = n_entries * nf * cells;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(i % cells);
        const long long ef = i / cells;
        const int f = (int)(ef % nf);
        const long long e = ef / nf;
        const int2 en = entries[e];
        U[((size_t)en.x * nf + f) * NC + (cells == NC ? k : slab_cell(en.y, k))] = buf[i];
    }
    if (stamp != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(stamp + 1, globaltimer());
    }
}

// ---------------------------------------------------------------------------
// Reference-shaped ghost layers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int face_cell_index(int face, int j) {
    const int plane = (face & 1) ? N - 1 : 0;
    const int u = j % N, v = j / N;
    int x, y, z;
    switch (face / 2) {
        case 0: x = plane; y = u; z = v; break;
        case 1: x = u; y = plane; z = v; break;
        default: x = u; y = v; z = plane; break;
    }
    return x + N * (y + N * z);
}

__global__ void face_exchange_kernel(const double* __restrict__ U, int nf, const int* __restrict__ nbr,
                                     long long n_owned, double* __restrict__ ghost) {
    const long long total = n_owned * 6 * N * N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(i % (N * N));
        const long long gf = i / (N * N);
        const int face = (int)(gf % 6);
        const long long g = gf / 6;
        const int h = nbr[g * 6 + face];
        ghost[i] = h < 0 ? 0.0 : U[(size_t)h * nf * NC + face_cell_index(face ^ 1, j)];
    }
}

__global__ void fill_halo_kernel(const double* __restrict__ U, int nf, const int* __restrict__ nbr,
                                 long long n_owned, int h, double* __restrict__ tiles) {
    const int pe = N + 2 * h;
    const long long tile = (long long)pe * pe * pe;
    const long long total = n_owned * nf * tile;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i % tile;
        const long long gfi = i / tile;
        const int f = (int)(gfi % nf);
        const long long g = gfi / nf;
        int c[3] = {(int)(r % pe) - h, (int)((r / pe) % pe) - h, (int)(r / ((long long)pe * pe)) - h};
        long long cur = g;
        for (int axis = 0; axis < 3; ++axis) {
            if (c[axis] < 0) {
                const int nb = cur >= 0 ? nbr[cur * 6 + 2 * axis] : -1;
                if (nb >= 0) {
                    cur = nb;
                    c[axis] += N;
                } else {
                    c[axis] = 0;
                }
            } else if (c[axis] >= N) {
                const int nb = nbr[cur * 6 + 2 * axis + 1];
                if (nb >= 0) {
                    cur = nb;
                    c[axis] -= N;
                } else {
                    c[axis] = N - 1;
                }
            }
        }
        tiles[i] = U[((size_t)cur * nf + f) * NC + (c[2] * N + c[1]) * N + c[0]];
    }
}

__global__ void clock_kernel(unsigned long long* out) { *out = globaltimer(); }

// Bitwise check of the branch-free reciprocal / square root against IEEE
// 1.0/x and sqrt(x) on mix64-random positive operands with exponents in
// [-emax, emax] (and a physically typical band when emax is small).
__global__ void selftest_math_kernel(unsigned long long n, unsigned long long seed, int emax,
                                     unsigned long long* bad) {
    unsigned long long nb_rcp = 0, nb_sqrt = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint64_t h = mix64(seed, i);
        // emax > 0: uniform mantissas, exponents in [-emax, emax]; emax < 0:
        // mantissas within 2^-20 of 1 or 2 (the high word nearly constant,
        // where the MUFU seeds are coarsest), exponents in [emax, -emax]
        const int em = emax < 0 ? -emax : emax;
        const int ex = (int)((h >> 52) % (2u * (unsigned)em + 1u)) - em;
        uint64_t mant = h & 0xFFFFFFFFFFFFFull;
        if (emax < 0) mant = (h >> 63) ? (mant & 0xFFFFFFFFull) : (0xFFFFFFFFFFFFFull - (mant & 0xFFFFFFFFull));
        // 1 in 64 of them exactly all-ones (the reciprocal's hard case)
        if (emax < 0 && ((h >> 32) & 63) == 0) mant = 0xFFFFFFFFFFFFFull;
        const uint64_t bits = ((uint64_t)(ex + 1023) << 52) | mant;
        const double x = __longlong_as_double((long long)bits);
        if (__double_as_longlong(rcp_rn(x)) != __double_as_longlong(1.0 / x)) ++nb_rcp;
        if (__double_as_longlong(sqrt_rn(x)) != __double_as_longlong(sqrt(x))) ++nb_sqrt;
    }
    if (nb_rcp) atomicAdd(bad, nb_rcp);
    if (nb_sqrt) atomicAdd(bad + 1, nb_sqrt);
}

// ---------------------------------------------------------------------------
// Host-side launchers
// ---------------------------------------------------------------------------
template <int NF>
cudaError_t launch_stage_n(const StageArgs& a, int recon, int stage, int n, cudaStream_t s, bool pdl);
extern template cudaError_t launch_stage_n<6>(const StageArgs&, int, int, int, cudaStream_t, bool);
extern template cudaError_t launch_stage_n<7>(const StageArgs&, int, int, int, cudaStream_t, bool);
extern template cudaError_t launch_stage_n<8>(const StageArgs&, int, int, int, cudaStream_t, bool);
extern template cudaError_t launch_stage_n<9>(const StageArgs&, int, int, int, cudaStream_t, bool);
extern template cudaError_t launch_stage_n<10>(const StageArgs&, int, int, int, cudaStream_t, bool);
extern template cudaError_t launch_stage_n<11>(const StageArgs&, int, int, int, cudaStream_t, bool);

cudaError_t launch_stage(const StageArgs& a, int nf, int recon, int stage, int n_ctas, cudaStream_t s, bool pdl) {
    if (n_ctas <= 0) return cudaSuccess;
    switch (nf) {
        case 6: return launch_stage_n<6>(a, recon, stage, n_ctas, s, pdl);
        case 7: return launch_stage_n<7>(a, recon, stage, n_ctas, s, pdl);
        case 8: return launch_stage_n<8>(a, recon, stage, n_ctas, s, pdl);
        case 9: return launch_stage_n<9>(a, recon, stage, n_ctas, s, pdl);
        case 10: return launch_stage_n<10>(a, recon, stage, n_ctas, s, pdl);
        case 11: return launch_stage_n<11>(a, recon, stage, n_ctas, s, pdl);
    }
    return cudaErrorInvalidValue;
}

static int grid_for(long long total, int block, int sms) {
    long long g = (total + block - 1) / block;
    const long long cap = (long long)sms * 16;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

template <int NF>
static void launch_signal_t(const double* U, long long n_cells, EosParams e, double* amax,
                            unsigned long long* stamp, int sms, cudaStream_t s) {
    signal_kernel<NF><<<grid_for(n_cells, 256, sms), 256, 0, s>>>(U, n_cells, e, amax, stamp);
}

cudaError_t launch_signal(const double* U, int nf, long long n_grids, double gamma, double p_floor,
                          double* amax, unsigned long long* stamp, int sms, cudaStream_t s) {
    const EosParams e{gamma, gamma - 1.0, p_floor};
    const long long n = n_grids * NC;
    if (n_grids <= 0) return cudaSuccess;
    switch (nf) {
        case 6: launch_signal_t<6>(U, n, e, amax, stamp, sms, s); break;
        case 7: launch_signal_t<7>(U, n, e, amax, stamp, sms, s); break;
        case 8: launch_signal_t<8>(U, n, e, amax, stamp, sms, s); break;
        case 9: launch_signal_t<9>(U, n, e, amax, stamp, sms, s); break;
        case 10: launch_signal_t<10>(U, n, e, amax, stamp, sms, s); break;
        case 11: launch_signal_t<11>(U, n, e, amax, stamp, sms, s); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_init_random(double* U, int nf, const long long* gid, long long n_grids, uint64_t seed,
                               double gamma, int sms, cudaStream_t s) {
    if (n_grids <= 0) return cudaSuccess;
    const long long n = n_grids * NC;
    init_random_kernel<<<grid_for(n, 256, sms), 256, 0, s>>>(U, nf, gid, n, seed, gamma);
    return cudaGetLastError();
}

cudaError_t launch_pack(const double* U, int nf, const int2* entries, long long n, double* buf, int sms,
                        cudaStream_t s, unsigned long long* stamp, int cells) {
    if (n <= 0) return cudaSuccess;
    pack_kernel<<<grid_for(n * nf * cells, 256, sms), 256, 0, s>>>(U, nf, entries, n, buf, stamp, cells);
    return cudaGetLastError();
}

cudaError_t launch_unpack(double* U, int nf, const int2* entries, long long n, const double* buf, int sms,
                          cudaStream_t s, unsigned long long* stamp, int cells) {
    if (n <= 0) return cudaSuccess;
    unpack_kernel<<<grid_for(n * nf * cells, 256, sms), 256, 0, s>>>(U, nf, entries, n, buf, stamp, cells);
    return cudaGetLastError();
}

cudaError_t launch_face_exchange(const double* U, int nf, const int* nbr, long long n_owned, double* ghost,
                                 int sms, cudaStream_t s) {
    if (n_owned <= 0) return cudaSuccess;
    face_exchange_kernel<<<grid_for(n_owned * 6 * N * N, 256, sms), 256, 0, s>>>(U, nf, nbr, n_owned, ghost);
    return cudaGetLastError();
}

cudaError_t launch_fill_halo(const double* U, int nf, const int* nbr, long long n_owned, int h,
                             double* tiles, int sms, cudaStream_t s) {
    if (n_owned <= 0) return cudaSuccess;
    const long long pe = N + 2 * h;
    fill_halo_kernel<<<grid_for(n_owned * nf * pe * pe * pe, 256, sms), 256, 0, s>>>(U, nf, nbr, n_owned, h,
                                                                                    tiles);
    return cudaGetLastError();
}

cudaError_t launch_selftest_math(unsigned long long n, unsigned long long seed, int emax, unsigned long long* bad,
                                 int sms, cudaStream_t s) {
    selftest_math_kernel<<<sms * 8, 256, 0, s>>>(n, seed, emax, bad);
    return cudaGetLastError();
}

// SimDevice::launch_kernel on a real GPU (reference device.cpp:24-32): one
// thread occupies its stream for duration_ns of %globaltimer and stamps the
// activity slot, so named simulated launches (e.g. the gravity kernels of
// workload.cpp:565-569) become real device activity that serialises per
// stream and overlaps across streams.
__global__ void timed_kernel(unsigned long long duration_ns, unsigned long long* stamp) {
    const unsigned long long t0 = globaltimer();
    if (stamp != nullptr) stamp[0] = ~t0;
    unsigned long long t = t0;
    while (t - t0 < duration_ns) {
        __nanosleep(duration_ns - (t - t0) > 2000ull ? 1000u : 64u);
        t = globaltimer();
    }
    if (stamp != nullptr) stamp[1] = t;
}

// Activity stamp around a copy: which = 0 stores the start, 1 the end.
__global__ void stamp_kernel(unsigned long long* stamp, int which) {
    const unsigned long long t = globaltimer();
    stamp[which] = which == 0 ? ~t : t;
}

cudaError_t launch_timed(unsigned long long duration_ns, unsigned long long* stamp, cudaStream_t s) {
    timed_kernel<<<1, 1, 0, s>>>(duration_ns, stamp);
    return cudaGetLastError();
}

cudaError_t launch_stamp(unsigned long long* stamp, int which, cudaStream_t s) {
    if (stamp == nullptr) return cudaSuccess;  // profiling disabled
    stamp_kernel<<<1, 1, 0, s>>>(stamp, which);
    return cudaGetLastError();
}

cudaError_t launch_clock(unsigned long long* out, cudaStream_t s) {
    clock_kernel<<<1, 1, 0, s>>>(out);
    return cudaGetLastError();
}

// Stream-ordered wait for peer flags (P2P transport): one thread acquires
// flags[q] >= seq for every rank q in `mask`, giving up after wait_ns and
// reporting through *err (cf. the stage kernels' wait_flag) — a stream
// memory-op wait could not time out.
__global__ void wait_flags_kernel(const unsigned int* flags, unsigned long long mask, unsigned int seq,
                                  unsigned long long* err, unsigned long long wait_ns) {
    volatile unsigned long long* e = err;
    for (int q = 0; q < 64; ++q) {
        if (!((mask >> q) & 1ull)) continue;
        unsigned long long t0 = 0ull;
        unsigned int spins = 0;
        while ((int)(ld_acquire_sys(flags + q) - seq) < 0) {
            const unsigned long long now = globaltimer();
            if (t0 == 0ull) {
                t0 = now;
                continue;
            }
            if (now - t0 > wait_ns || (now - t0 > 100000ull && (++spins & 255u) == 0u && *e != 0ull)) {
                *e = 1ull;
                return;
            }
        }
    }
}

// Multi-rank dt all-reduce as one tiny stream-ordered kernel between a step's
// stage 3 and the next stage 1 (alternative to the stage-3 tail, StageArgs):
// push this rank's max into slot `rank` of every rank's gather half, raise the
// peers' dt flags, acquire theirs, write the global max.
__global__ void dt_exchange_kernel(const double* local_amax, double* const* push_gather,
                                   unsigned int* const* push_flag, int world, int rank, unsigned int seq,
                                   const unsigned int* dt_wait, const double* gather_own, double* amax_global,
                                   unsigned long long* err, unsigned long long wait_ns) {
    const double am = *local_amax;
    for (int q = 0; q < world; ++q) push_gather[q][rank] = am;
    __threadfence_system();
    for (int q = 0; q < world; ++q)
        if (push_flag[q] != nullptr) atomicExch_system(push_flag[q], seq);
    volatile unsigned long long* e = err;
    for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        const unsigned long long t0 = globaltimer();
        while ((int)(ld_acquire_sys(dt_wait + q) - seq) < 0) {
            if (globaltimer() - t0 > wait_ns) {
                *e = 1ull;
                return;
            }
        }
    }
    double g = gather_own[0];
    for (int q = 1; q < world; ++q) g = fmax(g, gather_own[q]);
    *amax_global = g;
}

cudaError_t launch_dt_exchange(const double* local_amax, double* const* push_gather, unsigned int* const* push_flag,
                               int world, int rank, unsigned int seq, const unsigned int* dt_wait,
                               const double* gather_own, double* amax_global, unsigned long long* err,
                               unsigned long long wait_ns, cudaStream_t s) {
    dt_exchange_kernel<<<1, 1, 0, s>>>(local_amax, push_gather, push_flag, world, rank, seq, dt_wait, gather_own,
                                       amax_global, err, wait_ns);
    return cudaGetLastError();
}

cudaError_t launch_wait_flags(const unsigned int* flags, unsigned long long mask, unsigned int seq,
                              unsigned long long* err, unsigned long long wait_ns, cudaStream_t s) {
    if (mask == 0ull) return cudaSuccess;
    wait_flags_kernel<<<1, 1, 0, s>>>(flags, mask, seq, err, wait_ns);
    return cudaGetLastError();
}

}  // namespace tsh
