// gravity_kernels.cu — first gravity slice: the
// near-field monopole P2P behind the reference's `p2p_kernel` launches
// (gravity_kernel_name, reference proj/core/src/workload.cpp:365-372; six per
// sub-grid and step, 565-569; Octo-Tiger's "p2p interactions kernel: cell to
// cell interactions in non-refined sub-grids").  The reference
// only sleeps for them.  Numerics: oracle/hydro_oracle.h (orc_gravity_p2p),
// operation for operation (--fmad=false, explicit fma), so bitwise equal.
//
// B200 shape: one CTA per sub-grid, one thread per cell.  The densities of
// the sub-grid and of its 26 same-level neighbours out to R cells are staged
// once into a shared-memory tile (20 x 20 x 24 doubles, row pitch 24 so a
// warp — 8 x-cells of 4 y-rows — reads 32 distinct bank pairs' worth of
// 8-byte words in the minimum 2 wavefronts).  The stencil is geometry only
// (offsets and 1/|d|, d/|d|^3 for a uniform level), so it lives in constant
// memory: every interaction is one shared-memory load and four DFMAs whose
// coefficient operand is a uniform constant-bank read — the kernel is FP64
// bound by construction (4 DFMA per interaction; ~2.1 G DFMA for R = 4 on
// 4096 sub-grids).
#include <atomic>
#include <cmath>
#include <utility>

#include "hydro_device.cuh"
#include "hydro_kernels.h"

namespace tsh {

constexpr int kP2PStencilMax = 924;  // |d|^2 <= 36: the R = 6 stencil (R = 1..6 are its prefixes)
constexpr int kTile = N + 2 * kP2PRMax;  // 20
constexpr int kPitch = 24;             // row pitch (doubles), == 8 mod 16
constexpr int kTileDoubles = kTile * kTile * kPitch;

__constant__ double c_p2p_coef[4 * kP2PStencilMax];
__constant__ int c_p2p_off[kP2PStencilMax];  // linear tile offset of the stencil entry

namespace {

__device__ __forceinline__ int cidx3(int x, int y, int z) { return (z * N + y) * N + x; }

__host__ __device__ constexpr int stencil_size(int R) {
    return R == 1 ? 6 : R == 2 ? 32 : R == 3 ? 122 : R == 4 ? 256 : R == 5 ? 514 : 924;
}

// The stencil's tile offsets as a compile-time table (same order as
// p2p_stencil_host), so an unrolled interaction reads the tile at an
// immediate offset from the cell's base.
struct OffTable {
    int v[kP2PStencilMax];
};
constexpr OffTable make_offsets() {
    OffTable t{};
    int n = 0;
    for (int r2 = 1; r2 <= kP2PRMax * kP2PRMax; ++r2)
        for (int dz = -kP2PRMax; dz <= kP2PRMax; ++dz)
            for (int dy = -kP2PRMax; dy <= kP2PRMax; ++dy)
                for (int dx = -kP2PRMax; dx <= kP2PRMax; ++dx)
                    if (dx * dx + dy * dy + dz * dz == r2) t.v[n++] = (dz * kTile + dy) * kPitch + dx;
    return t;
}
constexpr OffTable kOff = make_offsets();

template <int K>
__device__ __forceinline__ void p2p_term(const double* base, double& s0, double& sx, double& sy, double& sz) {
    constexpr int off = kOff.v[K];
    const double rho = base[off];
    s0 = fma(rho, c_p2p_coef[4 * K], s0);
    sx = fma(rho, c_p2p_coef[4 * K + 1], sx);
    sy = fma(rho, c_p2p_coef[4 * K + 2], sy);
    sz = fma(rho, c_p2p_coef[4 * K + 3], sz);
}
template <int... K>
__device__ __forceinline__ void p2p_terms(const double* base, double& s0, double& sx, double& sy, double& sz,
                                          std::integer_sequence<int, K...>) {
    (p2p_term<K>(base, s0, sx, sy, sz), ...);  // in stencil order
}

// RS = the radius as a template argument: the stencil loop unrolls fully, so
// every coefficient and tile offset is an immediate operand (constant bank /
// LDS offset) and an interaction is one LDS + four DFMA.  RS = 0: runtime
// radius (A.n_stencil), indexed constant loads.
template <int RS>
__global__ void __launch_bounds__(NC) p2p_kernel(const __grid_constant__ P2PArgs A) {
    extern __shared__ __align__(16) double tile[];
    __shared__ int nb27[27];
    const int t = threadIdx.x;
    if (A.stamp != nullptr && t == 0) atomicMax(A.stamp, ~globaltimer());
    const int g = A.list_inline_n > 0 ? A.list_inline[blockIdx.x] : A.first + (int)blockIdx.x;
    if (t < 27) {
        // the sub-grid at block offset (ox, oy, oz): the face links walked x,
        // then y, then z (the oracle's p2p_rho); -1 = vacuum
        const int o[3] = {t % 3 - 1, (t / 3) % 3 - 1, t / 9 - 1};
        int h = g;
        for (int axis = 0; axis < 3 && h >= 0; ++axis)
            if (o[axis] != 0) h = A.nbr[6 * h + 2 * axis + (o[axis] > 0 ? 1 : 0)];
        nb27[t] = h;
    }
    __syncthreads();
    const int R = A.radius, S = N + 2 * R;
    for (int i = t; i < S * S * S; i += NC) {
        const int x = i % S - R, y = (i / S) % S - R, z = i / (S * S) - R;  // in-sub-grid coordinates
        const int bx = x < 0 ? 0 : (x >= N ? 2 : 1), by = y < 0 ? 0 : (y >= N ? 2 : 1), bz = z < 0 ? 0 : (z >= N ? 2 : 1);
        const int h = nb27[(bz * 3 + by) * 3 + bx];
        double rho = 0.0;
        if (h >= 0) rho = __ldg(A.U + (size_t)h * A.nf * NC + cidx3(x - (bx - 1) * N, y - (by - 1) * N, z - (bz - 1) * N));
        tile[((z + kP2PRMax) * kTile + (y + kP2PRMax)) * kPitch + (x + kP2PRMax)] = rho;
    }
    __syncthreads();
    const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
    const double* base = tile + ((z + kP2PRMax) * kTile + (y + kP2PRMax)) * kPitch + (x + kP2PRMax);
    double s0 = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
    if constexpr (RS > 0) {
        p2p_terms(base, s0, sx, sy, sz, std::make_integer_sequence<int, stencil_size(RS)>{});
    } else {
#pragma unroll 4
        for (int k = 0; k < A.n_stencil; ++k) {
            const double rho = base[c_p2p_off[k]];
            s0 = fma(rho, c_p2p_coef[4 * k], s0);
            sx = fma(rho, c_p2p_coef[4 * k + 1], sx);
            sy = fma(rho, c_p2p_coef[4 * k + 2], sy);
            sz = fma(rho, c_p2p_coef[4 * k + 3], sz);
        }
    }
    double* o = A.out + (size_t)g * 4 * NC + t;
    o[0] = A.kphi * s0;
    o[NC] = A.kg * sx;
    o[2 * NC] = A.kg * sy;
    o[3 * NC] = A.kg * sz;
    if (A.stamp != nullptr) {
        __syncthreads();
        if (t == 0) atomicMax(A.stamp + 1, globaltimer());
    }
}

}  // namespace

// The stencil table, computed on the host with the oracle's formulas (same
// IEEE sqrt / division, so the same bits): |d|^2 ascending, then (dz, dy, dx).
int p2p_stencil_host(int radius, int* off3, double* coef4, int cap) {
    int n = 0;
    for (int r2 = 1; r2 <= radius * radius; ++r2)
        for (int dz = -radius; dz <= radius; ++dz)
            for (int dy = -radius; dy <= radius; ++dy)
                for (int dx = -radius; dx <= radius; ++dx) {
                    if (dx * dx + dy * dy + dz * dz != r2) continue;
                    if (n < cap) {
                        const double c0 = 1.0 / std::sqrt((double)r2);
                        const double c3 = c0 / (double)r2;
                        off3[3 * n] = dx;
                        off3[3 * n + 1] = dy;
                        off3[3 * n + 2] = dz;
                        coef4[4 * n] = c0;
                        coef4[4 * n + 1] = (double)dx * c3;
                        coef4[4 * n + 2] = (double)dy * c3;
                        coef4[4 * n + 3] = (double)dz * c3;
                    }
                    ++n;
                }
    return n;
}

cudaError_t launch_p2p(const P2PArgs& a, int n_ctas, cudaStream_t s) {
    if (n_ctas <= 0) return cudaSuccess;
    // constant table and the > 48 KB shared-memory opt-in: once per device
    static std::atomic<unsigned long long> ready{0ull};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if ((ready.load(std::memory_order_acquire) & bit) == 0ull) {
        static int off3[3 * kP2PStencilMax];
        static double coef[4 * kP2PStencilMax];
        int lin[kP2PStencilMax];
        const int n = p2p_stencil_host(kP2PRMax, off3, coef, kP2PStencilMax);
        if (n != kP2PStencilMax) return cudaErrorInvalidValue;
        for (int k = 0; k < n; ++k) lin[k] = (off3[3 * k + 2] * kTile + off3[3 * k + 1]) * kPitch + off3[3 * k];
        e = cudaMemcpyToSymbol(c_p2p_coef, coef, sizeof(coef));
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_p2p_off, lin, sizeof(lin));
        if (e == cudaSuccess) e = cudaDeviceSynchronize();  // the symbol copies land before any launch
        const int smem = (int)(kTileDoubles * sizeof(double));
        for (auto fn : {p2p_kernel<0>, p2p_kernel<2>, p2p_kernel<4>, p2p_kernel<6>})
            if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        ready.fetch_or(bit, std::memory_order_acq_rel);
    }
    const size_t smem = kTileDoubles * sizeof(double);
    switch (a.radius) {  // the common radii unrolled; the rest through the runtime loop
        case 2: p2p_kernel<2><<<n_ctas, NC, smem, s>>>(a); break;
        case 4: p2p_kernel<4><<<n_ctas, NC, smem, s>>>(a); break;
        case 6: p2p_kernel<6><<<n_ctas, NC, smem, s>>>(a); break;
        default: p2p_kernel<0><<<n_ctas, NC, smem, s>>>(a); break;
    }
    return cudaGetLastError();
}

}  // namespace tsh
