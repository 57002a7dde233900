// hydro_kernels.h — host-side launch interface of hydro_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tsh {

struct StageArgs {
    const double* Uprev;        // U^{(k-1)}: owned + proxy sub-grids
    const double* Un;           // U^n (stages 2, 3)
    double* Uout;               // U^{(k)}
    double* scratch;            // a state buffer free during this stage (species accumulators, nf > 6)
    const int* nbr;             // [local][6] local neighbour index, -1 = outflow
    const int* list;            // CTA -> local sub-grid (nullable: first + blockIdx.x)
    int first;
    const double* amax_in;      // signal speed(s) behind this step's dt (max over amax_n values:
    int amax_n;                 //   one per rank when the P2P transport gathered them)
    double* amax_out;           // stage 3: max signal speed of U^{n+1}
    double* amax_reset;         // stage 1: zeroed (the slot stage 3 accumulates into)
    double* dt_out;             // stage 1: dt of this step
    unsigned long long* stamp;  // [start, end] globaltimer ns of this launch (nullable)
    // Stage 3, P2P transport: the last CTA of the stage (across the interior
    // and boundary launches, counted in done_ctr) pushes the rank's final
    // amax into slot `rank` of every rank's gather array and raises their flags.
    int push_n;                          // ranks to push to (0: no push)
    int rank;
    int total_ctas;
    unsigned int* done_ctr;
    double* const* push_gather;          // [push_n] gather arrays (this step's half)
    unsigned int* const* push_flag;      // [push_n] flag words (nullptr for self)
    unsigned int seq;
    // Stage 1, P2P transport, device-side wait: thread 0 of every CTA
    // acquires the wait_n flag words (>= wait_seq) before reading amax_in.
    const unsigned int* wait_flags;
    int wait_n;
    unsigned int wait_seq;
    double gamma, gm1, cfl, dx, p_floor;
};

cudaError_t launch_stage(const StageArgs& a, int nf, int recon, int stage, int n_ctas, cudaStream_t s);
cudaError_t launch_signal(const double* U, int nf, long long n_grids, double gamma, double p_floor,
                          double* amax, unsigned long long* stamp, int sms, cudaStream_t s);
cudaError_t launch_init_random(double* U, int nf, const long long* gid, long long n_grids, uint64_t seed,
                               double gamma, int sms, cudaStream_t s);
cudaError_t launch_pack(const double* U, int nf, const int2* entries, long long n, double* buf, int sms,
                        cudaStream_t s, unsigned long long* stamp);
cudaError_t launch_unpack(double* U, int nf, const int2* entries, long long n, const double* buf, int sms,
                          cudaStream_t s, unsigned long long* stamp);
cudaError_t launch_face_exchange(const double* U, int nf, const int* nbr, long long n_owned, double* ghost,
                                 int sms, cudaStream_t s);
cudaError_t launch_fill_halo(const double* U, int nf, const int* nbr, long long n_owned, int h,
                             double* tiles, int sms, cudaStream_t s);
cudaError_t launch_clock(unsigned long long* out, cudaStream_t s);
cudaError_t launch_selftest_math(unsigned long long n, unsigned long long seed, int emax, unsigned long long* bad,
                                 int sms, cudaStream_t s);

}  // namespace tsh
