// Microbenchmark: cycles per step of a single-warp level-synchronous chain
// (LDS deps -> DFMA chain -> STS -> __syncwarp), variants isolating each cost.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NSTEP = 4096;

template <int V>
__global__ void k(const double* __restrict__ progc, const double* __restrict__ proge, const int* __restrict__ progs,
                  double* out, long long* cyc) {
    __shared__ double xs[1024];
    __shared__ double pc[32 * 32];  // small program copy (reused cyclically)
    __shared__ double pe[2 * 32 * 32];
    __shared__ int ps[2 * 32 * 32];
    const int lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) xs[i] = 1.0 + i * 1e-3;
    for (int i = lane; i < 32 * 32; i += 32) pc[i] = progc[i];
    for (int i = lane; i < 2 * 32 * 32; i += 32) {
        pe[i] = proge[i];
        ps[i] = progs[i];
    }
    __syncwarp();
    volatile double* vxs = xs;
    double e0 = 0.25, e1 = 0.125, c = 1.0;
    int s0 = (lane + 31) & 1023, s1 = (lane + 1) & 1023;
    long long t0 = clock64();
    double acc = 0;
    for (int s = 0; s < NSTEP; ++s) {
        if (V >= 2) {
            const int q = (s & 31) * 32 + lane;
            c = pc[q];
            e0 = pe[2 * q];
            e1 = pe[2 * q + 1];
            s0 = ps[2 * q] + ((s * 32) & 1023);
            s1 = ps[2 * q + 1] + ((s * 32) & 1023);
            s0 &= 1023;
            s1 &= 1023;
        }
        double x;
        if (V == 0) {
            x = fma(-e0, xs[s0], c);
            x = fma(-e1, xs[s1], x);
        } else {
            x = fma(-e0, vxs[s0], c);
            x = fma(-e1, vxs[s1], x);
        }
        if (V == 3) {
            acc += x;
        } else {
            xs[((s + 1) * 32 + lane) & 1023] = x;
        }
        if (V != 4) __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
    out[lane] = xs[lane] + acc;
}

template <int V>
void run(const char* name, double* pc, double* pe, int* ps, double* out, long long* cyc) {
    k<V><<<1, 32>>>(pc, pe, ps, out, cyc);
    k<V><<<1, 32>>>(pc, pe, ps, out, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %.1f cycles/step\n", name, double(h) / NSTEP);
}

int main() {
    double *pc, *pe, *out;
    int* ps;
    long long* cyc;
    cudaMalloc(&pc, 8 * NSTEP * 32);
    cudaMalloc(&pe, 16 * NSTEP * 32);
    cudaMalloc(&ps, 8 * NSTEP * 32);
    cudaMalloc(&out, 8 * 32);
    cudaMalloc(&cyc, 8 * 32);
    cudaMemset(pc, 0, 8 * NSTEP * 32);
    cudaMemset(pe, 0, 16 * NSTEP * 32);
    cudaMemset(ps, 0, 8 * NSTEP * 32);
    run<0>("v0 regs, LDS deps, STS, syncwarp", pc, pe, ps, out, cyc);
    run<1>("v1 volatile LDS deps", pc, pe, ps, out, cyc);
    run<2>("v2 + program from smem", pc, pe, ps, out, cyc);
    run<3>("v3 program, no STS (no chain)", pc, pe, ps, out, cyc);
    run<4>("v4 no syncwarp", pc, pe, ps, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
}
