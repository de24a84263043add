// Microbenchmark: one lane running the K2b Neumaier carry chain (24576 adds)
// from shared memory; cycles per compensated add for a few formulations, and
// the FP64 issue rate of independent DADDs for reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -o chain_bench chain_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <type_traits>
#include "../../paper_1903_00227_b200/csrc/common.cuh"
namespace wrsb {
}

constexpr int N = 4096;

struct CS4 {  // four-DADD error term (the original formulation)
    double hi, lo;
    __device__ __forceinline__ void add(double x) {
        const double t = hi + x;
        const double e = fabs(hi) >= fabs(x) ? (hi - t) + x : (x - t) + hi;
        const double l2 = lo + e;
        lo = isfinite(t) ? l2 : lo;
        hi = t;
    }
};
struct CS2 {  // operand select, two DADDs (current)
    double hi, lo;
    __device__ __forceinline__ void add(double x) {
        const double t = hi + x;
        const bool big = fabs(hi) >= fabs(x);
        const double a = big ? hi : x, b = big ? x : hi;
        const double e = (a - t) + b;
        const double l2 = lo + e;
        lo = isfinite(t) ? l2 : lo;
        hi = t;
    }
};

template <class C, bool VALUE>
__global__ void chain(const double* __restrict__ in, double* out, long long* cyc) {
    __shared__ double buf[N];
    for (int i = threadIdx.x; i < N; i += 32) buf[i] = in[i];
    __syncwarp();
    if (threadIdx.x) return;
    C acc{0.0, 0.0};
    const long long t0 = clock64();
    for (int i = 0; i < N; i += 16) {
        double t[16], v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = buf[i + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (VALUE) v[u] = acc.hi + acc.lo;
            acc.add(t[u]);
        }
        if (VALUE) {
#pragma unroll
            for (int u = 0; u < 16; ++u) out[i + u] = v[u];
        }
    }
    const long long t1 = clock64();
    out[N] = acc.hi + acc.lo;
    *cyc = t1 - t0;
}

// production K2b chain (software-pipelined CompSumPos), copied by include
namespace wrsb {
constexpr int K2B_B = 4;
struct ChainRegs {
    double X[3][K2B_B], H[3][K2B_B], T[3][K2B_B], E[3][K2B_B];
};
template <int SH, int SE, int SL, bool DH, bool DE, bool DL>
__device__ __forceinline__ void chain_step(const double* in, double* out, int v, double& hi,
                                           double& lo, ChainRegs& R) {
    constexpr int B = K2B_B;
    if (DH) {
#pragma unroll
        for (int u = 0; u < B; ++u) R.X[SH][u] = in[v * B + u];
    }
    double lb[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
        if (DH) { R.H[SH][u] = hi; R.T[SH][u] = hi + R.X[SH][u]; hi = R.T[SH][u]; }
        if (DE) {
            const bool big = R.H[SE][u] >= R.X[SE][u];
            const double a = big ? R.H[SE][u] : R.X[SE][u], b = big ? R.X[SE][u] : R.H[SE][u];
            R.E[SE][u] = (a - R.T[SE][u]) + b;
        }
        if (DL) { lb[u] = lo; lo = lo + R.E[SL][u]; }
    }
    if (DL) {
#pragma unroll
        for (int u = 0; u < B; ++u) out[(v - 2) * B + u] = R.H[SL][u] + lb[u];
    }
}
}
__global__ void piped(const double* __restrict__ gin, double* out, long long* cyc) {
    using namespace wrsb;
    __shared__ double in[N];
    for (int i = threadIdx.x; i < N; i += 32) in[i] = gin[i];
    __syncwarp();
    if (threadIdx.x) return;
    double hi = 0, lo = 0;
    ChainRegs R;
    const int nblk = N / K2B_B;
    const long long t0 = clock64();
    chain_step<0, 0, 0, true, false, false>(in, out, 0, hi, lo, R);
    chain_step<1, 0, 0, true, true, false>(in, out, 1, hi, lo, R);
    int v = 2;
    for (; v + 3 <= nblk; v += 3) {
        chain_step<2, 1, 0, true, true, true>(in, out, v, hi, lo, R);
        chain_step<0, 2, 1, true, true, true>(in, out, v + 1, hi, lo, R);
        chain_step<1, 0, 2, true, true, true>(in, out, v + 2, hi, lo, R);
    }
    const long long t1 = clock64();
    out[N] = hi + lo;
    *cyc = t1 - t0;
}

// two independent one-DADD recurrences (hi over X, lo over E) with the
// per-step states stored to smem: the lane-0 loop of a split carry chain
__global__ void two_chains(const double* __restrict__ gin, double* out, long long* cyc) {
    __shared__ double X[N / 4], E[N / 4], H[N / 4], L[N / 4];
    for (int i = threadIdx.x; i < N / 4; i += 32) {
        X[i] = gin[i];
        E[i] = gin[N / 4 + i] * 1e-9;
    }
    __syncwarp();
    if (threadIdx.x) return;
    double hi = 0, lo = 0;
    const long long t0 = clock64();
    for (int k = 0; k < N / 4; k += 8) {
        double xa[8], ec[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            xa[u] = X[k + u];
            ec[u] = E[k + u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            H[k + u] = hi;
            hi = hi + xa[u];
            L[k + u] = lo;
            lo = lo + ec[u];
        }
    }
    const long long t1 = clock64();
    out[0] = hi + lo + H[7] + L[9];
    *cyc = (t1 - t0) * 4;  // per pair: cycles x 4 / N
}

__global__ void dadd_rate(double* out, long long* cyc, int iters) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = threadIdx.x * 1e-3 + u;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = a[u] + 1.000001;
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += a[u];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *in, *out;
    long long* cyc;
    cudaMalloc(&in, N * 8);
    cudaMalloc(&out, (N + 64) * 8);
    cudaMallocManaged(&cyc, 8);
    double* h = new double[N];
    for (int i = 0; i < N; ++i) h[i] = 1000.0 + (i * 7919 % 1000) * 0.37;
    cudaMemcpy(in, h, N * 8, cudaMemcpyHostToDevice);
    auto run = [&](const char* name, void (*k)(const double*, double*, long long*)) {
        long long best = 1ll << 62;
        for (int r = 0; r < 3; ++r) {
            k<<<1, 32>>>(in, out, cyc);
            cudaDeviceSynchronize();
            if (*cyc < best) best = *cyc;
        }
        printf("%-36s %6.2f cycles/add\n", name, (double)best / N);
    };
    run("CS4 + value", chain<CS4, true>);
    run("CS2 + value", chain<CS2, true>);
    run("CS4 no value", chain<CS4, false>);
    run("CS2 no value", chain<CS2, false>);
    run("pipelined CompSumPos + value", piped);
    run("two 1-DADD chains (per pair of adds)", two_chains);
    const int iters = 1 << 14;
    dadd_rate<<<1, 32>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    printf("1 warp, 8 independent DADD chains: %.2f cycles per DADD instr\n", (double)*cyc / (iters * 8.0));
    dadd_rate<<<1, 128>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    printf("4 warps (1 per SMSP?): %.2f cycles per DADD instr per warp\n", (double)*cyc / (iters * 8.0));
    dadd_rate<<<1, 512>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    printf("16 warps: %.2f cycles per DADD instr per warp\n", (double)*cyc / (iters * 8.0));
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
