// Dependent-chain latency of FP64 ops on one warp (cycles per op), B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void lat(double* out, long long* cyc, double s) {
    double a = threadIdx.x * 1e-3 + 1.0;
    const double b = s * 0.999, c = s * 1e-7;
    long long t0 = clock64();
    for (int i = 0; i < 4096; ++i) {
        if (OP == 0) a = fma(a, b, c);
        if (OP == 1) a = a * b;
        if (OP == 2) a = a + c;
        if (OP == 3) a = a < b ? a + c : a - c;
        if (OP == 4) a = 1.0 / a;
        if (OP == 5) a = sqrt(a);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    if (a == 12345.0) *out = a;
}
template <int OP> void run(const char* n) {
    double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 8);
    lat<OP><<<1, 32>>>(d, c, 1.0); lat<OP><<<1, 32>>>(d, c, 1.0);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-8s %6.1f cycles per dependent op\n", n, h / 4096.0);
}
int main() { run<0>("DFMA"); run<1>("DMUL"); run<2>("DADD"); run<3>("DSETP+sel+DADD"); run<4>("DIV"); run<5>("SQRT"); }
