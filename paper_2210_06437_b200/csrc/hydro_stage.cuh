// hydro_stage.cuh — the fused reconstruct + Kurganov–Tadmor flux + SSP-RK3
// stage kernel.  Instantiated once per field count in stage_nf*.cu so the
// variants build in parallel.
//
// Shape: one 8^3 sub-grid per 64-thread CTA.  Each thread owns one pencil
// (a line of 8 interior cells + 3 ghosts per side) and sweeps x, then y, then
// z.  Along its pencil it marches face by face: per face it advances the PPM
// (or minmod) reconstruction of every field by one cell (slopes, interface
// values, monotonicity limiter all kept in registers — nothing is recomputed
// and nothing goes through shared memory), evaluates the KT flux from the two
// face states, and retires the flux difference of the cell behind it into a
// shared-memory accumulator dU.  The z sweep fuses the RK stage update: it
// writes U^(k) straight to HBM and, in stage 3, reduces the cell-centred CFL
// signal speed of U^{n+1} (warp shuffle + one atomic per warp).  Per stage a
// sub-grid therefore reads U^(k-1) (own interior + the 3-deep face slabs of its
// six face neighbours, read in place — the direct_local path of reference
// workload.cpp:532-536), reads U^n, and writes U^(k): one HBM round trip.
//
// The sweep direction is a runtime loop (not unrolled) and the face march is
// a rolled loop with one-face-ahead prefetch: the code stays small enough for
// the instruction cache (the fully unrolled first version was ~16k SASS
// instructions and stalled on instruction fetch).  Momentum components are
// visited in (normal, transverse-1, transverse-2) order so one code path
// serves every direction.
#pragma once

#include <atomic>
#include <cstdint>

#include "hydro_device.cuh"
#include "hydro_kernels.h"

namespace tsh {

// Pencil-to-lane mapping: one lane per pencil (sweep) or a lane pair
// (sweep_pair).  Measured on B200: the pair wins once passive species add
// shared-memory pressure (nf 11: 0.93 -> 1.24 G cell-updates/s), the single
// lane wins at nf 6 (3.01 vs 2.79).  TS_PAIR = 0 / 1 forces one for all nf.
#ifndef TS_PAIR
#define TS_PAIR 2
#endif
template <int NF>
struct Lanes {
    static constexpr bool pair = TS_PAIR == 2 ? (NF > 6) : (TS_PAIR == 1);
    static constexpr int threads = 64 * (pair ? 2 : 1);
    static constexpr int min_blocks = pair ? 4 : 6;
    // launch-bounds hint of the single-lane PPM march: 5 lets ptxas schedule
    // under a 204-register cap; it still allocates 168, so 6 CTAs stay
    // resident (measured same box: +1.2 %, Sedov 16^3)
    static constexpr int min_blocks_ppm = pair ? 4 : 5;
};
constexpr int kPencils = 64;  // pencils per sweep of one sub-grid
// PPM: reload the retiring cell's U^(k-1) from L1 (it was loaded two faces
// earlier) instead of carrying it in the window state (12 registers and 12
// moves per face).  PLM needs the value for its slope anyway.
#ifndef TS_PPM_RELOAD_UP
#define TS_PPM_RELOAD_UP 1
#endif

#ifndef TS_PREFETCH
#define TS_PREFETCH 1
#endif
// sweeps (bit = mode) whose face march is unrolled by 2 regardless of FaceUnroll
#ifndef TS_REV_STAGES
#define TS_REV_STAGES 0
#endif
#ifndef TS_UNROLL_MODES
#define TS_UNROLL_MODES 0
#endif
// Preferred shared-memory carveout (percent) of the stage kernels; -1: driver default.
#ifndef TS_CARVEOUT
#define TS_CARVEOUT -1
#endif
// U^n of the retiring cell (stages 2, 3, z sweep): loaded at the top of the
// face that retires it (not carried across faces: 12 fewer loop-carried
// registers) instead of prefetched one face ahead.
// Measured same-box A/B (round 2), both neutral or slower, kept off: release
// store / red for the dataflow flags instead of fence + atomic (±0 %), the six
// neighbour ids loaded before the waits (−0.5 %).
#ifndef TS_SLOT2
#define TS_SLOT2 0  // measured: -0.1 % (the bank conflicts it removes are not on the critical path)
#endif
#ifndef TS_REL_FLAGS
#define TS_REL_FLAGS 0
#endif
#ifndef TS_NBR_EARLY
#define TS_NBR_EARLY 0
#endif
#ifndef TS_UN_LATE
#define TS_UN_LATE 0
#endif
// L1 prefetch one face beyond the register prefetch (ncu source view: ptxas
// sinks the pencil / U^n loads of a face to the end of the previous one, so
// the face's first instructions wait on them).  Bit 0: the next pencil
// values, bit 1: U^n of the next retiring cell, bit 2: the retiring cell's
// U^(k-1) reload.  Applied in the sweeps set by TS_PF_L1_MODES (bit m = mode m).
#ifndef TS_PF_L1
#define TS_PF_L1 0
#endif
#ifndef TS_PF_L1_MODES
#define TS_PF_L1_MODES 4
#endif

constexpr int kFA = 6;        // fields marched together: rho, s_n, s_t1, s_t2, E, tau
constexpr int kFaces = N + 1;

// Resident CTAs per SM the register allocation is sized for (tuning knob).
#ifdef TS_MINB
#define TS_MINB_FOR(NF, RECON) TS_MINB
#else
#define TS_MINB_FOR(NF, RECON) (RECON == 0 ? Lanes<NF>::min_blocks_ppm : Lanes<NF>::min_blocks)
#endif
#ifndef TS_LAZY_DT
#define TS_LAZY_DT 1
#endif
#ifndef TS_KEEP_DL
#define TS_KEEP_DL 0
#endif
// Face-march unroll per reconstruction.  The rolled march pays ~90 register
// moves per face rotating the window state; unrolling renames them away but
// needs registers.  Measured on B200 (same-box A/B, Sedov 16^3): minmod
// unrolled by 2 fits the 6-CTA register budget and gains 4 % (5.40 -> 5.62 G
// cell-updates/s); PPM unrolled by 2 spills at 6 CTAs and loses 5 % even at 5
// (3.37 -> 3.19), by 2 at 4 CTAs 11 %.  TS_FACE_UNROLL forces one value.
template <int RECON>
struct FaceUnroll {
#ifdef TS_FACE_UNROLL
    static constexpr int value = TS_FACE_UNROLL;
#else
    static constexpr int value = RECON == 1 ? 2 : 1;
#endif
};

template <int NF>
struct StageSmem {
    // Flux-difference accumulator of the marched fields; passive species
    // (nf > 6) accumulate in a free state buffer instead (StageArgs::scratch)
    // so the CTA's shared memory stays small enough for 4 resident CTAs.
    static constexpr int dU = (NF > kFA ? kFA : NF) * NC;
    static constexpr int cache = NF > kFA ? kFaces * 3 * kPencils : 0;  // (vL, vR, a) per face
    static constexpr int doubles = dU + cache;
};

// TS_TMA: the own sub-grid's U^(k-1) (the 6 marched fields) is staged into
// shared memory by TMA at the start of the stage (cp.async.bulk.tensor, one
// 4 KiB box per field, 128-byte swizzle); the x sweep — whose pencils are
// rows, lane-strided 64 B apart in global memory — reads its own-interior
// values from there and writes its flux differences over them in place (a
// cell's U^(k-1) is dead once the cell retires), so the stage's shared memory
// does not grow.  The y and z sweeps read global memory (coalesced) as before.
#ifndef TS_TMA
#define TS_TMA 0
#endif

// Shared-memory slot of linear cell offset o = (z*8 + y)*8 + x.
//   default: rows XOR-swizzled by y so the x sweep's strided column accesses
//            spread over the banks;
//   TS_TMA:  the TMA 128-byte swizzle (16-byte chunk c of 128-byte row r at
//            c ^ (r & 7)), so the in-place dU and the staged U^(k-1) share one
//            layout (lanes per bank pair: x 4, y 2, z 2 — y is 4 with sm_slot).
__device__ __forceinline__ int sm_slot(int o) {
#if TS_TMA
    const int r = o >> 4;
    return (r << 4) + ((((o >> 1) & 7) ^ (r & 7)) << 1) + (o & 1);
#else
#if TS_SLOT2
    // x ^= y within the row and, from z >= 2 on, y ^= 1 inside its pair of
    // planes: every sweep's 32 lanes hit each 8-byte bank pair exactly twice
    // (the minimum, 2 wavefronts; the plain row swizzle left x and y at 4)
    return o ^ ((o >> 3) & 7) ^ ((o >> 4) & 8);
#else
    return o ^ ((o >> 3) & 7);
#endif
#endif
}

struct Pencil {
    const double* __restrict__ own;  // field 0 of this sub-grid in U^(k-1)
    const double* __restrict__ lo;   // field 0 of the -axis neighbour (nullptr: outflow)
    const double* __restrict__ hi;   // field 0 of the +axis neighbour (nullptr: outflow)
    const double* sown;              // TS_TMA x sweep: field 0 of the staged copy (generic pointer into smem)
    int base;                        // offset of pencil cell 0 within a field
    int ss;                          // stride along the pencil
};

// Address of field 0 at pencil position s (-3 .. 10): the own interior, the
// face neighbour's interior, or the clamped boundary cell (outflow).  Uniform
// across the CTA, computed once per face for all fields.  SM: own cells from
// the staged shared-memory copy (a generic pointer, read with ld_pen<true>).
template <bool SM = false>
__device__ __forceinline__ const double* paddr(const Pencil& p, int s) {
    if (s < 0) return p.lo != nullptr ? p.lo + p.base + (s + N) * p.ss : p.own + p.base;
    if (s >= N) return p.hi != nullptr ? p.hi + p.base + (s - N) * p.ss : p.own + p.base + (N - 1) * p.ss;
    if (SM) return p.sown + sm_slot(p.base + s * p.ss);
    return p.own + p.base + s * p.ss;
}
// Self-check build (TS_CHECK=1; StageArgs::check): bounds of the buffers a
// CTA touches, in shared memory so the pencil helpers need no argument.
#ifndef TS_CHECK
#define TS_CHECK 0
#endif
struct CheckBounds {
    const double* prev_lo;
    const double* prev_hi;
    const double* un_lo;
    const double* un_hi;
    unsigned long long* out;
};
#if TS_CHECK
__shared__ CheckBounds s_chk;
#endif
__device__ __forceinline__ void chk_fail(unsigned long long* out, unsigned code, long long a, long long b) {
    if (out == nullptr) return;
    atomicOr(out + 4, 1ull << (code & 63u));  // every code seen
    if (atomicAdd(out, 1ull) == 0ull) {
        out[1] = code;
        out[2] = (unsigned long long)a;
        out[3] = (unsigned long long)b;
    }
}
// code 1: U^(k-1) load outside the buffer, 2: U^n load outside the buffer
__device__ __forceinline__ void chk_load(const double* a, int which) {
#if TS_CHECK
    if (__isShared(a)) return;
    const double* lo = which == 1 ? s_chk.prev_lo : s_chk.un_lo;
    const double* hi = which == 1 ? s_chk.prev_hi : s_chk.un_hi;
    if (a < lo || a >= hi) chk_fail(s_chk.out, (unsigned)which, (long long)(a - lo), (long long)(hi - lo));
#else
    (void)a;
    (void)which;
#endif
}

// Pencil load: read-only global path, or a generic load when the address may
// be the staged shared-memory copy.
template <bool SM>
__device__ __forceinline__ double ld_pen(const double* a) {
    chk_load(a, 1);
    if (SM) return *a;
    return __ldg(a);
}
__device__ __forceinline__ double ld_un(const double* a) {
    chk_load(a, 2);
    return __ldg(a);
}

// Running reconstruction state of one field along the pencil.  On entry to
// face j (between cells j-1 and j): w0 = q[j], w1 = q[j+1], D = 2 slope(j),
// fc = interface value at face j, hi = limited right edge of cell j-1,
// qn = the next pencil value (prefetched), wp = q[j-1]
// (the U^(k-1) value of the cell retired at face j).
struct Recon {
    double w0, w1, D, fc, hi, qn, wp;
#if TS_KEEP_DL
    double dl;
#endif
};

// (Single-lane march only: measured +0.9 % at nf 6; the lane-pair march at
// nf 11 loses 6 % with it.)
#ifndef TS_RELOAD_UP_MODES
#define TS_RELOAD_UP_MODES 7  // sweeps (bit = mode) that reload rather than carry
#endif
template <int RECON, bool SM = false, int MODE = 0>
__device__ __forceinline__ double retiring_up(const Recon& r, const Pencil& p, int j, int fo) {
    if (RECON == 0 && TS_PPM_RELOAD_UP && ((TS_RELOAD_UP_MODES >> MODE) & 1)) return ld_pen<SM>(paddr<SM>(p, j - 1) + fo);
    return r.wp;
}

// q[j+1] - q[j]: recomputed (one DADD) rather than carried — a carried value
// costs a register and two moves per face in the rolled march.
__device__ __forceinline__ double recon_dl(const Recon& r) {
#if TS_KEEP_DL
    return r.dl;
#else
    return r.w1 - r.w0;
#endif
}

// Pencil values a march starts from: positions -3..2 (PPM) or -2..1 (PLM).
template <int RECON>
struct BeginVals {
    static constexpr int n = RECON == 0 ? 6 : 4;
    double q[n];
};
template <int RECON, bool SM = false>
__device__ __forceinline__ void load_begin(const Pencil& p, int fo, BeginVals<RECON>& b) {
#pragma unroll
    for (int i = 0; i < BeginVals<RECON>::n; ++i) b.q[i] = ld_pen<SM>(paddr<SM>(p, i - (RECON == 0 ? 3 : 2)) + fo);
}

template <int RECON>
__device__ __forceinline__ void recon_begin_vals(const BeginVals<RECON>& b, Recon& r) {
    if (RECON == 0) {
        const double q0 = b.q[0], q1 = b.q[1], q2 = b.q[2], q3 = b.q[3], q4 = b.q[4];
        r.qn = b.q[5];
        const double d0 = q1 - q0, d1 = q2 - q1, d2 = q3 - q2, d3 = q4 - q3;
        const double D1 = mc_slope2(d1, d0);  // slopes carried doubled
        const double D2 = mc_slope2(d2, d1);
        const double D3 = mc_slope2(d3, d2);
        const double f2 = ppm_face2(q1, q2, D1, D2);
        const double f3 = ppm_face2(q2, q3, D2, D3);
        double l = f2, h = f3;
        ppm_limit(l, q2, h);
        r.hi = h;
        r.D = D3;
        r.fc = f3;
#if TS_KEEP_DL
        r.dl = d3;
#endif
        r.w0 = q3;
        r.w1 = q4;
        r.wp = q2;
    } else {
        const double q1 = b.q[0], q2 = b.q[1], q3 = b.q[2];
        r.qn = b.q[3];
        const double s = minmod_slope(q3 - q2, q2 - q1);
        r.hi = fma(0.5, s, q2);
#if TS_KEEP_DL
        r.dl = q3 - q2;
#endif
        r.w0 = q3;
        r.wp = q2;
    }
}

template <int RECON, bool SM = false>
__device__ __forceinline__ void recon_begin(const Pencil& p, int fo, Recon& r) {
    BeginVals<RECON> b;
    load_begin<RECON, SM>(p, fo, b);
    recon_begin_vals<RECON>(b, r);
}

// Advance to face j: returns uL (right edge of cell j-1) and uR (left edge
// of cell j); `next` is the address (field 0) of the pencil value the next
// face needs (any valid address after the last face).
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <int RECON, bool SM = false>
__device__ __forceinline__ void recon_step(const double* next, int fo, Recon& r, double& uL, double& uR) {
    const double q = r.qn;
    r.qn = ld_pen<SM>(next + fo);  // `next` is always a valid address (the value is unused after the last face)
    if (RECON == 0) {
        const double dn = q - r.w1;
        const double Dn = mc_slope2(dn, recon_dl(r));
        const double fn = ppm_face2(r.w0, r.w1, r.D, Dn);
        double l = r.fc, h = fn;
        ppm_limit(l, r.w0, h);
        uL = r.hi;
        uR = l;
        r.hi = h;
        r.D = Dn;
        r.fc = fn;
#if TS_KEEP_DL
        r.dl = dn;
#endif
        r.wp = r.w0;
        r.w0 = r.w1;
        r.w1 = q;
    } else {
        // PLM state: w0 = q[j], wp = q[j-1]; the left difference is w0 - wp
        const double dn = q - r.w0;
#if TS_KEEP_DL
        const double dm = r.dl;
        r.dl = dn;
#else
        const double dm = r.w0 - r.wp;
#endif
        const double s = minmod_slope(dn, dm);
        uL = r.hi;
        uR = fma(-0.5, s, r.w0);
        r.hi = fma(0.5, s, r.w0);
        r.wp = r.w0;
        r.w0 = q;
    }
}

struct StageCtx {
    const double* __restrict__ Un;
    double* __restrict__ Uout;
    double* scr;  // species accumulator of this sub-grid (field-major, like the state)
#if TS_TMA
    double* dU;                  // shared accumulator (aliases the staged U^(k-1) the x sweep reads)
#else
    double* __restrict__ dU;     // shared accumulator
#endif
    double* __restrict__ cache;  // shared (vL, vR, a) per face, NF > 6
    size_t own;                  // element offset of the sub-grid's field 0
    double dtdx;                 // 0.5 dt/dx: fluxes are carried doubled (kt2)
    EosParams e;
    // AMR flux register (StageArgs::rf_slot): where this sweep's first / last
    // face fluxes go when that face is a coarse-fine face, else nullptr;
    // rf_cell = the pencil's face cell a + 8 b
    double* rf_lo;
    double* rf_hi;
    int rf_cell;
};

// Store the (doubled) face flux of field f of this pencil into a flux register slot.
__device__ __forceinline__ void rf_store(double* slot, int f, int cell, double F) {
    if (slot != nullptr) slot[f * (N * N) + cell] = F;
}

// Retire the flux difference d of cell offset `o`, field f (uprev = U^(k-1)
// of that cell, un = its U^n).
//   MODE 0 (x): dU  = d;  MODE 1 (y): dU += d;
//   MODE 2 (z): U_out = RK(U_n, U_prev + dtdx (dU + d)).
template <int MODE, int STAGE>
__device__ __forceinline__ double retire_m(const StageCtx& c, int f, int o, double d, double uprev, double un) {
    double* slot = c.dU + f * NC + sm_slot(o);
    if (MODE == 0) {
        *slot = d;
        return 0.0;
    } else if (MODE == 1) {
        *slot = *slot + d;
        return 0.0;
    } else {
        const double tot = *slot + d;
        const double ustar = fma(c.dtdx, tot, uprev);
        double out;
        if (STAGE == 1) {
            out = ustar;
        } else if (STAGE == 2) {
            out = fma(0.75, un, 0.25 * ustar);
        } else {
            out = fma(1.0 / 3.0, un, (2.0 / 3.0) * ustar);
        }
#if TS_CHECK
        if (o < 0 || o >= NC || !isfinite(out)) chk_fail(s_chk.out, isfinite(out) ? 3u : 20u, o, f);
#endif
        c.Uout[c.own + (size_t)f * NC + o] = out;
        return out;
    }
}

// Species retire: the accumulator lives in global scratch; `acc` is this
// cell's prefetched partial sum (modes 1, 2).
template <int MODE, int STAGE>
__device__ __forceinline__ void retire_species(const StageCtx& c, int f, int o, double d, double acc, double uprev,
                                               double un) {
    double* slot = c.scr + (size_t)f * NC + o;
    if (MODE == 0) {
        *slot = d;
    } else if (MODE == 1) {
        *slot = acc + d;
    } else {
        const double tot = acc + d;
        const double ustar = fma(c.dtdx, tot, uprev);
        double out;
        if (STAGE == 1) {
            out = ustar;
        } else if (STAGE == 2) {
            out = fma(0.75, un, 0.25 * ustar);
        } else {
            out = fma(1.0 / 3.0, un, (2.0 / 3.0) * ustar);
        }
        c.Uout[c.own + (size_t)f * NC + o] = out;
    }
}

// Pencil value address for the face after face j (clamped to a valid cell).
template <int RECON, bool SM = false>
__device__ __forceinline__ const double* next_addr(const Pencil& p, int j) {
    const int s = j + 3 - RECON;
    return paddr<SM>(p, s < N + 2 ? s : N + 2);
}

// Face states -> EOS -> Kurganov–Tadmor flux (fields in n, t1, t2 order).
__device__ __forceinline__ void kt_face(const EosParams& e, const double (&uL)[kFA], const double (&uR)[kFA],
                                        double (&F)[kFA], double& vL, double& vR, double& a) {
    const double invL = eos_rcp(uL[0]), invR = eos_rcp(uR[0]);
    vL = uL[1] * invL;
    vR = uR[1] * invR;
    const double keL = fma(uL[1], vL, fma(uL[2], uL[2] * invL, uL[3] * (uL[3] * invL)));
    const double keR = fma(uR[1], vR, fma(uR[2], uR[2] * invR, uR[3] * (uR[3] * invR)));
    const double pL = dmax(e.gm1 * fma(-0.5, keL, uL[4]), e.p_floor);
    const double pR = dmax(e.gm1 * fma(-0.5, keR, uR[4]), e.p_floor);
    // Davis bound max(|v_L|, |v_R|) + max(c_L, c_R), one square root per face
    a = dmax(fabs(vL), fabs(vR)) + eos_sqrt(dmax((e.gamma * pL) * invL, (e.gamma * pR) * invR));
    F[0] = kt2(a, uL[0], uR[0], uL[1], uR[1]);
    F[1] = kt2(a, uL[1], uR[1], fma(uL[1], vL, pL), fma(uR[1], vR, pR));
    F[2] = kt2(a, uL[2], uR[2], uL[2] * vL, uR[2] * vR);
    F[3] = kt2(a, uL[3], uR[3], uL[3] * vL, uR[3] * vR);
    F[4] = kt2(a, uL[4], uR[4], (uL[4] + pL) * vL, (uR[4] + pR) * vR);
    F[5] = kt2(a, uL[5], uR[5], uL[5] * vL, uR[5] * vR);
}

// Single-lane march, one instantiation per sweep mode (x: init, y:
// accumulate, z: RK update) so the face loop carries no mode branches; face 0
// is peeled (it retires nothing) and every prefetch is unconditional.
template <int NF, int RECON, int STAGE, int MODE, bool RF>
__device__ __forceinline__ void sweep(const StageCtx& c, const Pencil& p, const int (&fm)[kFA], double& amax) {
    const int t = threadIdx.x;
    constexpr bool kUn = STAGE > 1 && MODE == 2;  // U^n needed by the update
    constexpr bool SM = TS_TMA && MODE == 0;      // own cells from the TMA-staged copy
    int fo[kFA];
#pragma unroll
    for (int k = 0; k < kFA; ++k) fo[k] = fm[k] * NC;
    Recon r[kFA];
#pragma unroll
    for (int k = 0; k < kFA; ++k) recon_begin<RECON, SM>(p, fo[k], r[k]);
    const double* un_row = c.Un + c.own + p.base;
    double un[kFA];
    if (kUn && !TS_UN_LATE) {
#pragma unroll
        for (int k = 0; k < kFA; ++k) un[k] = ld_un(un_row + fo[k]);
    }
    double Fp[kFA];
    {  // face 0
        const double* next = next_addr<RECON, SM>(p, 0);
        double uL[kFA], uR[kFA];
#pragma unroll
        for (int k = 0; k < kFA; ++k) recon_step<RECON, SM>(next, fo[k], r[k], uL[k], uR[k]);
        double vL, vR, a;
        kt_face(c.e, uL, uR, Fp, vL, vR, a);
        if (NF > kFA) {
            c.cache[(0 * 3 + 0) * kPencils + t] = vL;
            c.cache[(0 * 3 + 1) * kPencils + t] = vR;
            c.cache[(0 * 3 + 2) * kPencils + t] = a;
        }
        if (RF && c.rf_lo != nullptr) {
#pragma unroll
            for (int k = 0; k < kFA; ++k) rf_store(c.rf_lo, fm[k], c.rf_cell, Fp[k]);
        }
    }
    constexpr int kUnroll = ((TS_UNROLL_MODES >> MODE) & 1) ? 2 : FaceUnroll<RECON>::value;
#pragma unroll kUnroll
    for (int j = 1; j < kFaces; ++j) {
        const double* next = next_addr<RECON, SM>(p, j);
        if (TS_PF_L1 != 0 && ((TS_PF_L1_MODES >> MODE) & 1) && !SM) {
            const double* nn = next_addr<RECON>(p, j + 1 < kFaces ? j + 1 : j);
            const double* un_nn = c.Un + c.own + p.base + (j < N ? j : N - 1) * p.ss;
            const double* up_nn = p.own + p.base + (j < N ? j : N - 1) * p.ss;
#pragma unroll
            for (int k = 0; k < kFA; ++k) {
                if (TS_PF_L1 & 1) prefetch_l1(nn + fo[k]);
                if ((TS_PF_L1 & 2) && kUn) prefetch_l1(un_nn + fo[k]);
                if (TS_PF_L1 & 4) prefetch_l1(up_nn + fo[k]);
            }
        }
        double uL[kFA], uR[kFA], up[kFA];
#pragma unroll
        for (int k = 0; k < kFA; ++k) {
            up[k] = retiring_up<RECON, SM, MODE>(r[k], p, j, fo[k]);  // U^(k-1) of cell j-1, retired here
            if (kUn && TS_UN_LATE) un[k] = ld_un(un_row + (j - 1) * p.ss + fo[k]);
            recon_step<RECON, SM>(next, fo[k], r[k], uL[k], uR[k]);
        }
        double F[kFA], vL, vR, a;
        kt_face(c.e, uL, uR, F, vL, vR, a);
        if (NF > kFA) {
            c.cache[(j * 3 + 0) * kPencils + t] = vL;
            c.cache[(j * 3 + 1) * kPencils + t] = vR;
            c.cache[(j * 3 + 2) * kPencils + t] = a;
        }
        if (RF && j == kFaces - 1 && c.rf_hi != nullptr) {
#pragma unroll
            for (int k = 0; k < kFA; ++k) rf_store(c.rf_hi, fm[k], c.rf_cell, F[k]);
        }
        const int o = p.base + (j - 1) * p.ss;
        double out[kFA];
#pragma unroll
        for (int k = 0; k < kFA; ++k) out[k] = retire_m<MODE, STAGE>(c, fm[k], o, Fp[k] - F[k], up[k], un[k]);
        if (STAGE == 3 && MODE == 2)  // z sweep: fm = {rho, sz, sx, sy, E, tau}
            amax = fmax(amax, cell_signal_speed(out[0], out[2], out[3], out[1], out[4], c.e));
        if (kUn && !TS_UN_LATE) {
            const int jn = j < N ? j : N - 1;  // cell retired at the next face (a dummy reload after the last)
#pragma unroll
            for (int k = 0; k < kFA; ++k) un[k] = ld_un(un_row + jn * p.ss + fo[k]);
        }
#pragma unroll
        for (int k = 0; k < kFA; ++k) Fp[k] = F[k];
    }
    if (NF > kFA) {
        // passive species: same march, transported with the hydro face data
#pragma unroll 1
        for (int f = kFA; f < NF; ++f) {
            const int fof = f * NC;
            double acc[N];
            if (MODE > 0) {
                const double* sp = c.scr + fof + p.base;
#pragma unroll
                for (int i = 0; i < N; ++i) acc[i] = sp[i * p.ss];
            }
            Recon q;
            recon_begin<RECON>(p, fof, q);
            double unf = kUn ? ld_un(un_row + fof) : 0.0;
            double Fq;
            {
                double uL, uR;
                recon_step<RECON>(next_addr<RECON>(p, 0), fof, q, uL, uR);
                Fq = kt2(c.cache[2 * kPencils + t], uL, uR, uL * c.cache[t], uR * c.cache[kPencils + t]);
                if (RF) rf_store(c.rf_lo, f, c.rf_cell, Fq);
            }
#pragma unroll
            for (int j = 1; j < kFaces; ++j) {
                double uL, uR;
                const double upf = retiring_up<RECON>(q, p, j, fof);
                recon_step<RECON>(next_addr<RECON>(p, j), fof, q, uL, uR);
                const double vL = c.cache[(j * 3 + 0) * kPencils + t];
                const double vR = c.cache[(j * 3 + 1) * kPencils + t];
                const double a = c.cache[(j * 3 + 2) * kPencils + t];
                const double F = kt2(a, uL, uR, uL * vL, uR * vR);
                if (RF && j == kFaces - 1) rf_store(c.rf_hi, f, c.rf_cell, F);
                retire_species<MODE, STAGE>(c, f, p.base + (j - 1) * p.ss, Fq - F, MODE > 0 ? acc[j - 1] : 0.0, upf,
                                            unf);
                if (kUn) unf = ld_un(un_row + (j < N ? j : N - 1) * p.ss + fof);
                Fq = F;
            }
        }
    }
}

// Lane-pair march.  Lane role 0 owns (rho, s_n, s_t1), role 1 owns (s_t2, E,
// tau) of the same pencil.  Per face: each lane advances its 3 fields, the
// pair swaps the face states the other side needs (one shuffle round), role 0
// evaluates the EOS of the LEFT state and role 1 of the RIGHT state (the
// division -> square-root chain is split, not duplicated), they swap
// (v, p, a) and each lane forms the KT fluxes of its own fields.  Same
// arithmetic, operation by operation, as the single-lane march (bitwise).
__device__ __forceinline__ double xlane(double v) { return __shfl_xor_sync(0xffffffffu, v, 1); }

template <int NF, int RECON, int STAGE, int MODE, bool RF>
__device__ __forceinline__ void sweep_pair(const StageCtx& c, const Pencil& p, const int (&fm)[kFA], double& amax) {
    const int role = threadIdx.x & 1;
    const int pen = threadIdx.x >> 1;
    constexpr bool kUn = STAGE > 1 && MODE == 2;
    int fmo[3], fo[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        fmo[k] = role ? fm[3 + k] : fm[k];
        fo[k] = fmo[k] * NC;
    }
    Recon r[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) recon_begin<RECON>(p, fo[k], r[k]);
    const double* un_row = c.Un + c.own + p.base;
    double un[3];
    if (kUn) {
#pragma unroll
        for (int k = 0; k < 3; ++k) un[k] = ld_un(un_row + fo[k]);
    }
    double Fp[3];
#pragma unroll 1
    for (int j = 0; j < kFaces; ++j) {
        const double* next = next_addr<RECON>(p, j);
        double uL[3], uR[3], up[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            up[k] = r[k].wp;
            recon_step<RECON>(next, fo[k], r[k], uL[k], uR[k]);
        }
        // role 0 needs (s_t2, E) of the left state, role 1 (rho, s_n, s_t1) of the right
        double y[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) y[k] = xlane(role ? uL[k] : uR[k]);
        const double S0 = role ? y[0] : uL[0];
        const double S1 = role ? y[1] : uL[1];
        const double S2 = role ? y[2] : uL[2];
        const double S3 = role ? uR[0] : y[0];
        const double S4 = role ? uR[1] : y[1];
        const double inv = eos_rcp(S0);
        const double v = S1 * inv;
        const double ke = fma(S1, v, fma(S2, S2 * inv, S3 * (S3 * inv)));
        const double pr = dmax(c.e.gm1 * fma(-0.5, ke, S4), c.e.p_floor);
        const double c2 = (c.e.gamma * pr) * inv;
        const double vo = xlane(v), po = xlane(pr), c2o = xlane(c2);
        const double vL = role ? vo : v, vR = role ? v : vo;
        const double pL = role ? po : pr, pR = role ? pr : po;
        // Davis bound, as kt_face: both lanes take the one square root
        const double a = dmax(fabs(vL), fabs(vR)) + eos_sqrt(dmax(role ? c2o : c2, role ? c2 : c2o));
        // physical fluxes of the own fields
        //   role 0: (s_n, fma(s_n, v, p), s_t1 v)      role 1: (s_t2 v, (E + p) v, tau v)
        const double fL0 = role ? uL[0] * vL : uL[1];
        const double fR0 = role ? uR[0] * vR : uR[1];
        const double fL1 = role ? (uL[1] + pL) * vL : fma(uL[1], vL, pL);
        const double fR1 = role ? (uR[1] + pR) * vR : fma(uR[1], vR, pR);
        double F[3];
        F[0] = kt2(a, uL[0], uR[0], fL0, fR0);
        F[1] = kt2(a, uL[1], uR[1], fL1, fR1);
        F[2] = kt2(a, uL[2], uR[2], uL[2] * vL, uR[2] * vR);
        if (RF && j == 0 && c.rf_lo != nullptr) {
#pragma unroll
            for (int k = 0; k < 3; ++k) rf_store(c.rf_lo, fmo[k], c.rf_cell, F[k]);
        }
        if (RF && j == kFaces - 1 && c.rf_hi != nullptr) {
#pragma unroll
            for (int k = 0; k < 3; ++k) rf_store(c.rf_hi, fmo[k], c.rf_cell, F[k]);
        }
        if (NF > kFA && role == 0) {
            c.cache[(j * 3 + 0) * kPencils + pen] = vL;
            c.cache[(j * 3 + 1) * kPencils + pen] = vR;
            c.cache[(j * 3 + 2) * kPencils + pen] = a;
        }
        if (j > 0) {
            const int o = p.base + (j - 1) * p.ss;
            double out[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) out[k] = retire_m<MODE, STAGE>(c, fmo[k], o, Fp[k] - F[k], up[k], un[k]);
            if (STAGE == 3 && MODE == 2) {
                // z sweep: role 0 holds (rho, sz, sx), role 1 (sy, E, tau)
                const double sy = xlane(out[0]), E = xlane(out[1]);
                if (role == 0) amax = fmax(amax, cell_signal_speed(out[0], out[2], sy, out[1], E, c.e));
            }
            if (kUn) {
                const int jn = j < N ? j : N - 1;
#pragma unroll
                for (int k = 0; k < 3; ++k) un[k] = ld_un(un_row + jn * p.ss + fo[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) Fp[k] = F[k];
    }
    if (NF > kFA) {
        __syncwarp();
        // passive species, alternating between the two lanes of the pair
        // (loading the next species' start values one species ahead was
        // measured 7 % slower at nf 11)
#pragma unroll 1
        for (int f = kFA + role; f < NF; f += 2) {
            const int fof = f * NC;
            // partial sums of this pencil's 8 cells (plain loads: written by this CTA)
            double acc[N];
            if (MODE > 0) {
                const double* sp = c.scr + fof + p.base;
#pragma unroll
                for (int i = 0; i < N; ++i) acc[i] = sp[i * p.ss];
            }
            Recon q;
            recon_begin<RECON>(p, fof, q);
            double unf = kUn ? ld_un(un_row + fof) : 0.0;
            double Fq;
            {
                double uL, uR;
                recon_step<RECON>(next_addr<RECON>(p, 0), fof, q, uL, uR);
                Fq = kt2(c.cache[2 * kPencils + pen], uL, uR, uL * c.cache[pen], uR * c.cache[kPencils + pen]);
                if (RF) rf_store(c.rf_lo, f, c.rf_cell, Fq);
            }
#pragma unroll
            for (int j = 1; j < kFaces; ++j) {
                double uL, uR;
                const double upf = q.wp;
                recon_step<RECON>(next_addr<RECON>(p, j), fof, q, uL, uR);
                const double vL = c.cache[(j * 3 + 0) * kPencils + pen];
                const double vR = c.cache[(j * 3 + 1) * kPencils + pen];
                const double a = c.cache[(j * 3 + 2) * kPencils + pen];
                const double F = kt2(a, uL, uR, uL * vL, uR * vR);
                if (RF && j == kFaces - 1) rf_store(c.rf_hi, f, c.rf_cell, F);
                retire_species<MODE, STAGE>(c, f, p.base + (j - 1) * p.ss, Fq - F, MODE > 0 ? acc[j - 1] : 0.0, upf,
                                            unf);
                if (kUn) unf = ld_un(un_row + (j < N ? j : N - 1) * p.ss + fof);
                Fq = F;
            }
        }
    }
}

// Acquire-spin until *flag >= seq (wrapping compare) or the deadline; a
// timeout (a peer that never arrives: mismatched collective calls) is
// reported through *err.  *err is mapped host memory: it is read only once a
// wait has stalled for 100 us (an earlier timeout then ends this one at once),
// never on the fast path.
__device__ __forceinline__ void wait_flag(const StageArgs& A, const unsigned int* flag, unsigned int seq) {
    unsigned long long t0 = 0ull;
    unsigned int spins = 0;
    while ((int)(ld_acquire_sys(flag) - seq) < 0) {
        const unsigned long long now = globaltimer();
        if (t0 == 0ull) {
            t0 = now;
            continue;
        }
        if (now - t0 > A.wait_ns ||
            (A.err != nullptr && now - t0 > 100000ull && (++spins & 255u) == 0u &&
             *reinterpret_cast<volatile unsigned long long*>(A.err) != 0ull)) {
            if (A.err != nullptr) *reinterpret_cast<volatile unsigned long long*>(A.err) = 1ull;
            return;
        }
    }
}

// Dataflow wait (single rank, see StageArgs::flow_*): acquire-spin until
// *flag >= seq (wrapping compare), backing off with nanosleep so a waiting CTA
// takes few issue slots from the previous stage's CTAs on the same SM.  The
// producers are all resident (PDL starts this grid only once every CTA of the
// previous one runs), so the wait is bounded; the deadline only guards bugs.
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void flow_wait_one(const StageArgs& A, const unsigned int* flag, unsigned int seq) {
    if ((int)(ld_acquire_gpu(flag) - seq) >= 0) return;
    const unsigned long long t0 = globaltimer();
    unsigned int ns = 32;
    while ((int)(ld_acquire_gpu(flag) - seq) < 0) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
        if (globaltimer() - t0 > A.wait_ns) {
            if (A.err != nullptr) *reinterpret_cast<volatile unsigned long long*>(A.err) = 1ull;
            return;
        }
    }
}

// Fused halo push of one boundary sub-grid (see StageArgs): copy the 3-deep
// slab of every face with a foreign neighbour from this CTA's fresh U^(k)
// into the peer's proxy slot (same in-sub-grid layout), then count the CTA
// out; the last boundary CTA releases the receivers' flags (system scope).
// Loads are batched ahead of the remote stores (each is an L2 round trip);
// z slabs are contiguous per field and move as 16-byte vectors.
__device__ __forceinline__ int slab_offset(int axis, int d0, int k) {
    if (axis == 0) {
        const int l = k % 3, m = k / 3;  // m = y + 8 z
        return m * N + d0 + l;
    }
    const int u = k & (N - 1), m = k >> 3;  // axis 1: m = l + 3 z
    return ((m / 3) * N + d0 + m % 3) * N + u;
}

template <int NF>
__device__ __forceinline__ void halo_push(const StageArgs& A, size_t own, int b) {
    __syncthreads();  // U^(k) of this sub-grid written by the whole CTA
    const double* __restrict__ src = A.Uout + own;
    constexpr int kSlabCells = 3 * N * N;
    constexpr int kBatch = 8;
    const int nt = (int)blockDim.x;
    for (int f = 0; f < 6; ++f) {
        const int2 e = A.push_tbl[6 * b + f];
        if (e.x < 0) continue;
        double* __restrict__ dst = A.push_out[e.x] + (size_t)e.y * NF * NC;
        const int axis = f >> 1, d0 = (f & 1) ? N - 3 : 0;
        if (axis == 2) {
            constexpr int kVec = kSlabCells / 2;  // double2 per field
            const double2* s2 = reinterpret_cast<const double2*>(src + d0 * N * N);
            double2* t2 = reinterpret_cast<double2*>(dst + d0 * N * N);
            for (int base = 0; base < NF * kVec; base += nt * kBatch) {
                double2 v[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int i = base + u * nt + (int)threadIdx.x;
                    if (i < NF * kVec) v[u] = s2[(i / kVec) * (NC / 2) + i % kVec];
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int i = base + u * nt + (int)threadIdx.x;
                    if (i < NF * kVec) t2[(i / kVec) * (NC / 2) + i % kVec] = v[u];
                }
            }
        } else {
            for (int base = 0; base < NF * kSlabCells; base += nt * kBatch) {
                double v[kBatch];
                int o[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int i = base + u * nt + (int)threadIdx.x;
                    const int fld = i / kSlabCells;
                    o[u] = fld * NC + slab_offset(axis, d0, i - fld * kSlabCells);
                    if (i < NF * kSlabCells) v[u] = src[o[u]];
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    if (base + u * nt + (int)threadIdx.x < NF * kSlabCells) dst[o[u]] = v[u];
            }
        }
    }
    // CTA barrier, then one system-scope fence publishes the whole CTA's
    // remote stores before the count (the cooperative-groups grid-sync pattern)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned prior = atomicAdd(A.halo_ctr, 1u);
#if TS_CHECK
        // a count past this stage's target: another stage counted into the same slot
        if ((int)(prior - A.halo_target) >= 0) chk_fail(A.check, 12u, prior, A.halo_target);
#endif
        if (prior == A.halo_target - 1u) {
            __threadfence_system();
            for (int q = 0; q < A.halo_flag_n; ++q)
                if (A.halo_flag[q] != nullptr) atomicExch_system(A.halo_flag[q], A.halo_seq);
        }
    }
}

// dx of sub-grid g's level (StageArgs::lvl_*); uniform launches: dx_upd
__device__ __forceinline__ double level_dx(const StageArgs& A, int g) {
    double dx = A.dx_upd;
#pragma unroll
    for (int L = 1; L < StageArgs::kMaxLevels; ++L)
        if (L < A.lvl_n && g >= A.lvl_first[L]) dx = A.lvl_dx[L];
    return dx;
}

// TMA helpers (TS_TMA): mbarrier-tracked 2-D tensor copies into shared memory.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TS_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TS_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of a contiguous range (one instruction, no registers, no
// completion to wait for: a hint that turns the first touch of U^n in the
// z sweep from an HBM miss into an L2 hit).
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Launch slot -> position in the sub-grid list.  TS_REV_STAGES (bit s-1 =
// stage s) walks a stage's list backwards, so it first reads what the
// previous stage wrote last (still in L2) instead of the oldest lines.
template <int STAGE>
__device__ __forceinline__ int cta_slot() {
    return ((TS_REV_STAGES >> (STAGE - 1)) & 1) ? (int)(gridDim.x - 1u - blockIdx.x) : (int)blockIdx.x;
}

// Dynamic shared memory of a stage CTA: the dU accumulator (TS_TMA: 1024-byte
// aligned for the 128-byte swizzle, plus the mbarrier) and the nf > 6 cache.
template <int NF>
constexpr size_t stage_smem_bytes() {
    return (size_t)StageSmem<NF>::doubles * sizeof(double) + (TS_TMA ? 1024 + 16 : 0);
}

// RF: an AMR launch with a flux register (StageArgs::rf_slot); a separate
// instantiation so the uniform kernels carry none of its state (measured: the
// register-pressed nf 11 kernel lost 4.5 % with it).
template <int NF, int RECON, int STAGE, bool RF>
__global__ void __launch_bounds__(Lanes<NF>::threads, TS_MINB_FOR(NF, RECON)) stage_kernel(const __grid_constant__ StageArgs A) {
    extern __shared__ __align__(16) double smem_raw[];
#if TS_TMA
    double* smem = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    unsigned long long* tma_bar = reinterpret_cast<unsigned long long*>(smem + StageSmem<NF>::doubles);
#else
    double* smem = smem_raw;
#endif
    if (A.stamp != nullptr && threadIdx.x == 0)
        atomicMax(A.stamp, ~globaltimer());  // start stored inverted: one zero-initialised ring serves both ends
#if TS_PREFETCH
    // U^n of this sub-grid is first read by the z sweep, one face ahead of
    // its use: measured (ncu source view) as the z sweep's long-scoreboard
    // stall in stages 2 and 3.  Ask L2 for all of it now.
    if (STAGE > 1 && threadIdx.x == 32) {
        const int gp = A.list_inline_n > 0 ? A.list_inline[cta_slot<STAGE>()]
                       : (A.list != nullptr ? A.list[cta_slot<STAGE>()] : A.first + cta_slot<STAGE>());
        prefetch_l2(A.Un + (size_t)gp * NF * NC, (unsigned)(NF * NC * sizeof(double)));
    }
#endif
    if (A.cta_log != nullptr && threadIdx.x == 0) {
        unsigned int sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        A.cta_log[4 * blockIdx.x] = sm;
        A.cta_log[4 * blockIdx.x + 1] = globaltimer();
    }
    const int g = A.list_inline_n > 0 ? A.list_inline[cta_slot<STAGE>()]
                  : (A.list != nullptr ? A.list[cta_slot<STAGE>()] : A.first + cta_slot<STAGE>());
    const int t = threadIdx.x;
    // stage 1's once-per-step duties (see StageArgs::lead_g1)
    const bool lead = A.lead_g1 == 0 ? blockIdx.x == 0 : g == A.lead_g1 - 1;
#if TS_NBR_EARLY
    // the six face neighbours, loaded before the waits (ncu: the per-sweep
    // table load was a long-scoreboard stall at the start of every sweep)
    int nb6[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) nb6[f] = __ldg(A.nbr + 6 * g + f);
#endif
#if TS_CHECK
    if (t == 0) {
        const size_t span = (size_t)A.n_local * NF * NC;
        s_chk = CheckBounds{A.Uprev, A.Uprev + span, A.Un, A.Un + span, A.check};
        if (g < 0 || g >= A.n_owned) chk_fail(A.check, 4u, g, A.n_owned);  // CTA -> sub-grid outside the owned range
    }
    __syncthreads();
#endif
    if (A.halo_wait_mask != 0ull && __ldg(A.bnd_of + g) >= 0) {
        // proxies of U^(k-1): pushed by the peers' previous-stage boundary CTAs
        // (released in their first wave, so this rarely spins)
        // one source rank per thread, in parallel
        if (t < 64 && ((A.halo_wait_mask >> t) & 1ull)) wait_flag(A, A.halo_wait + t, A.halo_wait_seq);
        __syncthreads();
    }
    if (A.pdl_trigger) {
        if (STAGE == 1 && lead) {
            // the slot stage 3 accumulates into is zeroed before any dependent can start
            if (t == 0 && A.amax_reset != nullptr) {
                *A.amax_reset = 0.0;
                __threadfence();
            }
            __syncthreads();
        }
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (A.h2d_flag != nullptr) {
        // U^n of this sub-grid and of its face neighbours landed (StageArgs::h2d_flag)
        if (t < 7) {
            const int h = t == 0 ? g : __ldg(A.nbr + 6 * g + (t - 1));
            if (h >= 0 && h < A.chunk_owned)
                flow_wait_one(A, A.h2d_flag + (int)(((long long)h * A.chunk_n) / A.chunk_owned), A.h2d_seq);
        }
        __syncthreads();
    }
    if (A.flow_wait != nullptr) {
        // U^(k-1) of this sub-grid and of its face neighbours: the previous
        // stage's output.  The seven flags are acquired in parallel, one per
        // thread (one after the other they cost every CTA ~2-4 us of L2 round
        // trips, measured with TS_HYDRO_CTA_LOG); the barrier extends each
        // acquire to the whole CTA.
        if (t < 7) {
            const int h = t == 0 ? g : __ldg(A.nbr + 6 * g + (t - 1));
            if (h >= 0 && h < A.flow_n) flow_wait_one(A, A.flow_wait + h, A.flow_wait_seq);
        }
        __syncthreads();
    }
#if TS_TMA
    // Stage the own sub-grid's U^(k-1) (the marched fields) into the dU
    // buffer: its flags were acquired above, and the x sweep overwrites each
    // cell with its flux difference once the cell retired.
    const bool staged = !Lanes<NF>::pair;
    if (staged && A.tma == 0) __trap();  // a TS_TMA build needs the descriptor (stage_args sets it)
    if (staged) {
        if (threadIdx.x == 0) {
            mbar_init(tma_bar, 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(tma_bar, (unsigned)(kFA * NC * sizeof(double)));
            const int g_row = g * NF * (NC / 16);
#pragma unroll
            for (int f = 0; f < kFA; ++f) tma_load_2d(smem + f * NC, &A.tmap_prev, 0, g_row + f * (NC / 16), tma_bar);
        }
        __syncthreads();  // mbarrier initialised before anyone waits on it
    }
#endif
    // TS_LAZY_DT: dt enters only the z sweep's update, so its two IEEE
    // divisions can be done there, off the CTA's start-up path
    if (A.cta_log != nullptr && t == 0) A.cta_log[4 * blockIdx.x + 2] = globaltimer();
    double amax_in = A.amax_in[0];
    for (int i = 1; i < A.amax_n; ++i) amax_in = fmax(amax_in, A.amax_in[i]);
#if !TS_LAZY_DT
    if (A.cnt_wait != nullptr) {
        if (t == 0) flow_wait_one(A, A.cnt_wait, A.cnt_expect);
        __syncthreads();
        amax_in = *reinterpret_cast<const volatile double*>(A.amax_in);
    }
    const double dtdx_early = 0.5 * (((A.cfl * A.dx) / amax_in) / level_dx(A, g));
    if (STAGE == 1 && lead && t == 0) {
        if (A.dt_out != nullptr) *A.dt_out = (A.cfl * A.dx) / amax_in;
        if (A.amax_reset2 != nullptr) *A.amax_reset2 = 0.0;
    }
#endif
    if (STAGE == 1 && lead && t == 0) {
        if (A.amax_reset != nullptr && !A.pdl_trigger) *A.amax_reset = 0.0;
    }
    StageCtx c;
    c.Un = A.Un;
    c.Uout = A.Uout;
    c.dU = smem;
    c.cache = smem + StageSmem<NF>::dU;
    c.own = (size_t)g * NF * NC;
    c.scr = A.scratch != nullptr ? A.scratch + c.own : nullptr;
    __shared__ int scr_slot;
    if (NF > kFA && A.scr_ring != nullptr) {
        if (t == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            unsigned* mask = A.scr_mask + (sm & 255u);
            int slot = -1;
            while (slot < 0) {  // a free bit exists: at most scr_k CTAs of stage kernels are resident per SM
                const unsigned m = *reinterpret_cast<volatile unsigned*>(mask);
                const unsigned free_bits = ~m & ((A.scr_k >= 32) ? 0xffffffffu : ((1u << A.scr_k) - 1u));
                if (free_bits == 0u) continue;
                const int b = __ffs(free_bits) - 1;
                if ((atomicOr(mask, 1u << b) & (1u << b)) == 0u) slot = (int)(sm & 255u) * A.scr_k + b;
            }
            scr_slot = slot;
        }
        __syncthreads();
        c.scr = A.scr_ring + (size_t)scr_slot * (NF - kFA) * NC - (size_t)kFA * NC;
    }
    c.e = EosParams{A.gamma, A.gm1, A.p_floor};
    const double* own = A.Uprev + c.own;
    const int pen = Lanes<NF>::pair ? t >> 1 : t;
    const int a = pen & (N - 1), b = pen >> 3;
    double amax = 0.0;

#pragma unroll 1
    for (int axis = 0; axis < 3; ++axis) {
#if TS_NBR_EARLY
        const int nlo = axis == 0 ? nb6[0] : (axis == 1 ? nb6[2] : nb6[4]);
        const int nhi = axis == 0 ? nb6[1] : (axis == 1 ? nb6[3] : nb6[5]);
#else
        const int nlo = __ldg(A.nbr + 6 * g + 2 * axis);
        const int nhi = __ldg(A.nbr + 6 * g + 2 * axis + 1);
#endif
        c.rf_lo = c.rf_hi = nullptr;
        c.rf_cell = a + N * b;
        if (RF && A.rf_slot != nullptr) {
            const int sl = __ldg(A.rf_slot + 6 * g + 2 * axis), sh = __ldg(A.rf_slot + 6 * g + 2 * axis + 1);
            if (sl >= 0) c.rf_lo = A.rf_flux + (size_t)sl * NF * N * N;
            if (sh >= 0) c.rf_hi = A.rf_flux + (size_t)sh * NF * N * N;
        }
        Pencil p;
        p.own = own;
        p.sown = nullptr;
#if TS_TMA
        if (axis == 0 && staged) {
            p.sown = smem;
            mbar_wait(tma_bar, 0);
        }
#endif
        p.lo = nlo >= 0 ? A.Uprev + (size_t)nlo * NF * NC : nullptr;
        p.hi = nhi >= 0 ? A.Uprev + (size_t)nhi * NF * NC : nullptr;
        p.base = axis == 0 ? (b * N + a) * N : (axis == 1 ? b * N * N + a : b * N + a);
        p.ss = axis == 0 ? 1 : (axis == 1 ? N : N * N);
        // fields in (rho, s_normal, s_t1, s_t2, E, tau) order, t1 < t2
        const int fm[kFA] = {0, 1 + axis, axis == 0 ? 2 : 1, axis == 2 ? 2 : 3, 4, 5};
        if (axis == 2) {
#if TS_LAZY_DT
            if (A.cnt_wait != nullptr) {
                // every sub-grid's stage-3 max of the previous step is in place
                if (t == 0) flow_wait_one(A, A.cnt_wait, A.cnt_expect);
                __syncthreads();
                amax_in = *reinterpret_cast<const volatile double*>(A.amax_in);
#if TS_CHECK
                if (t == 0 && !(amax_in > 0.0 && isfinite(amax_in))) chk_fail(A.check, 13u, g, 0);
#endif
            }
            const double dt = (A.cfl * A.dx) / amax_in;
            c.dtdx = 0.5 * (dt / level_dx(A, g));  // the sweeps carry twice the KT flux (kt2)
            if (STAGE == 1 && lead && t == 0) {
                if (A.dt_out != nullptr) *A.dt_out = dt;
                if (A.amax_reset2 != nullptr) *A.amax_reset2 = 0.0;
            }
#else
            c.dtdx = dtdx_early;
#endif
        }
        if (Lanes<NF>::pair) {
            if (axis == 0)
                sweep_pair<NF, RECON, STAGE, 0, RF>(c, p, fm, amax);
            else if (axis == 1)
                sweep_pair<NF, RECON, STAGE, 1, RF>(c, p, fm, amax);
            else
                sweep_pair<NF, RECON, STAGE, 2, RF>(c, p, fm, amax);
        } else if (axis == 0)
            sweep<NF, RECON, STAGE, 0, RF>(c, p, fm, amax);
        else if (axis == 1)
            sweep<NF, RECON, STAGE, 1, RF>(c, p, fm, amax);
        else
            sweep<NF, RECON, STAGE, 2, RF>(c, p, fm, amax);
        if (axis < 2) __syncthreads();
    }
#if TS_CHECK
    // every flag this CTA acquired still holds exactly the awaited value: a
    // later one would mean a producer already ran its NEXT use of the data
    // this CTA read (flow: the next step's same stage of a neighbour; halo:
    // a peer's next stage), i.e. the ordering protocol let it overtake
    if (A.flow_wait != nullptr && t < 7) {
        const int h = t == 0 ? g : __ldg(A.nbr + 6 * g + (t - 1));
        if (h >= 0 && h < A.flow_n) {
            const unsigned v = ld_acquire_gpu(A.flow_wait + h);
            if (v != A.flow_wait_seq) chk_fail(A.check, 10u, h, (long long)(int)(v - A.flow_wait_seq));
        }
    }
    if (A.halo_wait_mask != 0ull && __ldg(A.bnd_of + g) >= 0 && t < 64 &&
        ((A.halo_wait_mask >> t) & 1ull)) {
        // a peer may already have pushed its NEXT stage (into the other buffer
        // of the rotation: +1), never the one after (it needs this CTA's push)
        const int d = (int)(ld_acquire_sys(A.halo_wait + t) - A.halo_wait_seq);
        if (d < 0 || d > 1) chk_fail(A.check, 11u, t, d);
    }
#endif
    if (A.push_tbl != nullptr) {
        const int b = __ldg(A.bnd_of + g);
        if (b >= 0) halo_push<NF>(A, c.own, b);
    }

    if (STAGE == 3) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if ((t & 31) == 0) atomic_max_nonneg(A.amax_out, amax);
    }
    if (STAGE == 3 && A.chunk_ctr != nullptr) {
        __syncthreads();
        if (t == 0) {
            __threadfence();  // U^(n+1) of this sub-grid performed at gpu scope before the count (the
                              // copy engine is a device agent; a system fence per CTA cost +170 us per stage)
            atomicAdd(A.chunk_ctr + (int)(((long long)g * A.chunk_n) / A.chunk_owned), 1u);
        }
    }
    if (A.flow_done != nullptr || A.cnt_done != nullptr) {
        // U^(k) of this sub-grid (and, stage 3, its max) complete: CTA barrier,
        // one gpu-scope fence, flag / count
        __syncthreads();
        if (t == 0) {
#if TS_REL_FLAGS
            // release operations (cumulative over the CTA's writes that the
            // barrier ordered before them) instead of a full fence + atomic
            if (A.flow_done != nullptr)
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(A.flow_done + g), "r"(A.flow_seq) : "memory");
            if (STAGE == 3 && A.cnt_done != nullptr && !A.cnt_gather)
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.cnt_done) : "memory");
#else
            __threadfence();
            if (A.flow_done != nullptr) atomicExch(A.flow_done + g, A.flow_seq);
            if (STAGE == 3 && A.cnt_done != nullptr && !A.cnt_gather) atomicAdd(A.cnt_done, 1u);
#endif
        }
    }
    if (A.done_ctr != nullptr) {
        // threadfence reduction to the last CTA of the stage (see StageArgs)
        __syncthreads();
        if (t == 0) {
            __threadfence();
            if (atomicAdd(A.done_ctr, 1u) == A.done_target - 1u) {
                __threadfence();
                if (STAGE == 3 && A.push_n > 0) {
                    // dt all-reduce: this rank's max into every rank's gather slot
                    const double am = __longlong_as_double(
                        (long long)atomicAdd(reinterpret_cast<unsigned long long*>(A.amax_out), 0ull));
                    for (int q = 0; q < A.push_n; ++q) A.push_gather[q][A.rank] = am;
                    __threadfence_system();
                    for (int q = 0; q < A.push_n; ++q)
                        if (A.push_flag[q] != nullptr) atomicExch_system(A.push_flag[q], A.seq);
                }
                if (STAGE == 3 && A.dt_wait != nullptr) {
                    for (int q = 0; q < A.push_n; ++q)
                        if (q != A.rank)
                            wait_flag(A, A.dt_wait + q, A.seq);
                    double g = A.gather_own[0];
                    for (int q = 1; q < A.push_n; ++q) g = fmax(g, A.gather_own[q]);
                    *A.amax_global = g;
                    if (A.cnt_gather && A.cnt_done != nullptr) {
                        // the next step's chained stage 1 reads amax_global after this count
                        __threadfence();
                        atomicAdd(A.cnt_done, (unsigned)A.flow_n);
                    }
                }
            }
        }
    }
    if (NF > kFA && A.scr_ring != nullptr) {
        __syncthreads();  // every species accumulator read / write of this CTA is done
        if (t == 0) {
            const int b = scr_slot % A.scr_k;
            atomicAnd(A.scr_mask + scr_slot / A.scr_k, ~(1u << b));
        }
    }
    if (A.stamp != nullptr) {
        __syncthreads();
        if (t == 0) atomicMax(A.stamp + 1, globaltimer());
    }
    if (A.cta_log != nullptr) {
        __syncthreads();
        if (t == 0) A.cta_log[4 * blockIdx.x + 3] = globaltimer();
    }
}

template <int NF, int RECON, int STAGE, bool RF>
inline cudaError_t launch_stage_rf(const StageArgs& a, int n_ctas, cudaStream_t s, bool pdl) {
    const size_t smem = stage_smem_bytes<NF>();
    // the dynamic shared-memory limit is a per-device function attribute:
    // set it once on every device this instantiation is launched on
    static std::atomic<unsigned long long> configured{0ull};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if ((configured.load(std::memory_order_acquire) & bit) == 0ull) {
        e = cudaFuncSetAttribute(stage_kernel<NF, RECON, STAGE, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
#if TS_CARVEOUT >= 0
        e = cudaFuncSetAttribute(stage_kernel<NF, RECON, STAGE, RF>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 TS_CARVEOUT);
        if (e != cudaSuccess) return e;
#endif
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    if (!pdl) {
        stage_kernel<NF, RECON, STAGE, RF><<<n_ctas, Lanes<NF>::threads, smem, s>>>(a);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)n_ctas);
    cfg.blockDim = dim3((unsigned)Lanes<NF>::threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, stage_kernel<NF, RECON, STAGE, RF>, a);
}

template <int NF, int RECON, int STAGE>
inline cudaError_t launch_stage_t(const StageArgs& a, int n_ctas, cudaStream_t s, bool pdl) {
    return a.rf_slot != nullptr ? launch_stage_rf<NF, RECON, STAGE, true>(a, n_ctas, s, pdl)
                                : launch_stage_rf<NF, RECON, STAGE, false>(a, n_ctas, s, pdl);
}

template <int NF, int RECON>
inline cudaError_t launch_stage_r(const StageArgs& a, int stage, int n, cudaStream_t s, bool pdl) {
    switch (stage) {
        case 1: return launch_stage_t<NF, RECON, 1>(a, n, s, pdl);
        case 2: return launch_stage_t<NF, RECON, 2>(a, n, s, pdl);
        case 3: return launch_stage_t<NF, RECON, 3>(a, n, s, pdl);
    }
    return cudaErrorInvalidValue;
}

template <int NF>
cudaError_t launch_stage_n(const StageArgs& a, int recon, int stage, int n, cudaStream_t s, bool pdl) {
    return recon == 0 ? launch_stage_r<NF, 0>(a, stage, n, s, pdl) : launch_stage_r<NF, 1>(a, stage, n, s, pdl);
}

}  // namespace tsh
