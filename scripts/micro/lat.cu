// Microbenchmark: latencies of the GS segment-chain step ingredients on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dadd_dmul(double* out, double a, double b, int n, long long* cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = (a - x) * b;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl(double* out, int n, long long* cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl32(float* out, int n, long long* cyc) {
    float x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
// full lockstep step: lane c computes, stores, broadcasts; others fma
__global__ void k_step(double* out, double* st, double a, double b, int n, long long* cyc) {
    const int lane = threadIdx.x;
    double iacc = 0.0, base = lane * 0.5, dii = 0.9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const int c = i & 31;
        double xi = 0.0;
        if (lane == c) {
            xi = (base - iacc) * dii;
            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(st + (i & 1023)), "l"(__double_as_longlong(xi)) : "memory");
        }
        const double xc = __shfl_sync(0xffffffffu, xi, c);
        if (lane == ((c + 1) & 31)) iacc += a * xc;
    }
    long long t1 = clock64();
    out[lane] = iacc;
    if (lane == 0) *cyc = t1 - t0;
}
// same without the store
__global__ void k_step_nost(double* out, double a, double b, int n, long long* cyc) {
    const int lane = threadIdx.x;
    double iacc = 0.0, base = lane * 0.5, dii = 0.9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const int c = i & 31;
        double xi = 0.0;
        if (lane == c) xi = (base - iacc) * dii;
        const double xc = __shfl_sync(0xffffffffu, xi, c);
        if (lane == ((c + 1) & 31)) iacc += a * xc;
    }
    long long t1 = clock64();
    out[lane] = iacc;
    if (lane == 0) *cyc = t1 - t0;
}
// redundant chain: every lane computes x = c_t - e_t * x, c/e broadcast (independent of x)
__global__ void k_redundant(double* out, double* st, int n, long long* cyc) {
    const int lane = threadIdx.x;
    const double cl = 0.5 + lane, el = 0.25;
    double x = 0.0, mine = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; i += 32) {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const double ct = __shfl_sync(0xffffffffu, cl, t);
            const double et = __shfl_sync(0xffffffffu, el, t);
            x = fma(-et, x, ct);
            if (lane == t) {
                mine = x;
                asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(st + lane), "l"(__double_as_longlong(x)) : "memory");
            }
        }
    }
    long long t1 = clock64();
    out[lane] = mine;
    if (lane == 0) *cyc = t1 - t0;
}
int main() {
    double *out, *st;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&st, 1024 * 8);
    cudaMalloc(&cyc, 8);
    long long h;
    const int n = 4096;
    auto rep = [&](const char* name) {
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-14s %.1f cycles/iter\n", name, double(h) / n);
    };
    for (int r = 0; r < 2; ++r) {
        k_dfma<<<1, 32>>>(out, 1.0000001, 1e-9, n, cyc); rep("dfma");
        k_dadd_dmul<<<1, 32>>>(out, 1.0000001, 0.5, n, cyc); rep("dadd+dmul");
        k_shfl<<<1, 32>>>(out, n, cyc); rep("shfl f64");
        k_shfl32<<<1, 32>>>((float*)out, n, cyc); rep("shfl f32");
        k_step<<<1, 32>>>(out, st, 0.3, 0.1, n, cyc); rep("step");
        k_step_nost<<<1, 32>>>(out, 0.3, 0.1, n, cyc); rep("step nostore");
        k_redundant<<<1, 32>>>(out, st, n, cyc); rep("redundant");
    }
    return 0;
}
