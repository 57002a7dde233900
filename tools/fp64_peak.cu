// FP64 pipe microbenchmark for the roofline denominator (B200, sm_100a):
// per-opcode throughput with 8 independent chains per thread, enough warps
// to saturate every SM.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;

template <int OP>
__global__ void kern(double* out, double s) {
    double a[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 1e-3 + k;
    const double b = s * 0.999, c = s * 1e-7;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            if (OP == 0) a[k] = fma(a[k], b, c);          // DFMA
            if (OP == 1) a[k] = a[k] * b;                 // DMUL
            if (OP == 2) a[k] = a[k] + c;                 // DADD
            if (OP == 3) a[k] = a[k] < b ? a[k] + 1e-300 : b;  // DSETP + select (+DADD)
            if (OP == 4) a[k] = 1.0 / a[k];               // IEEE division
            if (OP == 5) a[k] = sqrt(a[k]);               // IEEE sqrt
        }
    }
    double r = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) r += a[k];
    if (r == 12345.678) out[0] = r;
}

template <int OP>
double run(const char* name, int sms, double per_op_flops) {
    double* d;
    cudaMalloc(&d, 8);
    const int blocks = sms * 8, threads = 256;
    kern<OP><<<blocks, threads>>>(d, 1.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 3;
    for (int r = 0; r < reps; ++r) kern<OP><<<blocks, threads>>>(d, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)reps * blocks * threads * ITERS * CH;
    const double rate = ops / (ms * 1e-3);
    printf("%-10s %8.3f T thread-ops/s  (%6.1f per SM per clk at 1.965 GHz)  %s\n", name, rate / 1e12,
           rate / sms / 1.965e9, per_op_flops > 0 ? "" : "");
    cudaFree(d);
    return rate;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    run<0>("DFMA", sms, 2);
    run<1>("DMUL", sms, 1);
    run<2>("DADD", sms, 1);
    run<3>("DSETP+SEL", sms, 1);
    run<4>("DIV", sms, 1);
    run<5>("SQRT", sms, 1);
    return 0;
}
