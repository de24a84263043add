// Dependent-chain latency of FP64 ops and of the Neumaier add used by the
// PSA build, measured with clock64 on one thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o fp64_latency fp64_latency.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double x, int iters) {
    double a = out[0], hi = out[1], lo = out[2];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = a + x;  // DADD chain
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) a = a * x;  // DMUL chain
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {           // Neumaier add, branch-free
        const double t = hi + x;
        const double e = fabs(hi) >= fabs(x) ? (hi - t) + x : (x - t) + hi;
        const double l2 = lo + e;
        lo = isfinite(t) ? l2 : lo;
        hi = t;
    }
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) {           // compare-select feeding the next add
        const double v = hi + lo;
        const double d = v > x ? x : -x;
        hi = hi + d;
    }
    long long t4 = clock64();
    out[3] = a + hi + lo;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 64);
    cudaMalloc(&c, 64);
    double h[4] = {1.0, 1.0, 0.0, 0.0};
    cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
    const int it = 1 << 16;
    chain<<<1, 1>>>(d, c, 1.0000001, it);
    chain<<<1, 1>>>(d, c, 1.0000001, it);
    long long hc[4];
    cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
    printf("DADD chain: %.2f cyc/op\nDMUL chain: %.2f cyc/op\nNeumaier add: %.2f cyc/add\n"
           "DADD+DSETP+FSEL+DADD: %.2f cyc/iter\n",
           (double)hc[0] / it, (double)hc[1] / it, (double)hc[2] / it, (double)hc[3] / it);
    return 0;
}
