// Microbenchmark: the segment-chain step of k_gs_seg in isolation (one warp).
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned long long kPending = 0xFFF4DEADBEEFCAFEull;
template <int GST, int STS, int VOL>
__global__ void k_chain(double* xnew, int reps, long long* cyc) {
    __shared__ unsigned long long cs[32], xs[32];
    __shared__ double es[32];
    const int lane = threadIdx.x;
    cs[lane] = __double_as_longlong(0.5 + lane);
    es[lane] = 0.25;
    __syncwarp();
    double x = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (int u = 0; u < 32; ++u) {
            unsigned long long raw;
            if (VOL) {
                volatile unsigned long long* vcs = cs;
                raw = vcs[u];
                while (raw == kPending) raw = vcs[u];
            } else {
                raw = cs[u];
            }
            x = fma(-es[u], x, __longlong_as_double((long long)raw));
            if (lane == 0) {
                if (GST == 1)
                    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(xnew + (r * 32 + u) % 4096),
                                 "l"(__double_as_longlong(x)) : "memory");
                if (GST == 2) xnew[(r * 32 + u) % 4096] = x;
                if (STS) reinterpret_cast<volatile double*>(xs)[u] = x;
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) {
        *cyc = t1 - t0;
        xnew[5000] = x + __longlong_as_double(xs[3]);
    }
}
int main() {
    double* xnew;
    long long* cyc;
    cudaMalloc(&xnew, 8192 * 8);
    cudaMalloc(&cyc, 8);
    long long h;
    const int reps = 256;
    auto rep = [&](const char* name) {
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %.1f cycles/step\n", name, double(h) / (reps * 32));
    };
    for (int k = 0; k < 2; ++k) {
        k_chain<1, 1, 1><<<1, 32>>>(xnew, reps, cyc); rep("relaxed.gpu + sts + vol");
        k_chain<1, 0, 1><<<1, 32>>>(xnew, reps, cyc); rep("relaxed.gpu + vol");
        k_chain<2, 1, 1><<<1, 32>>>(xnew, reps, cyc); rep("weak st + sts + vol");
        k_chain<0, 1, 1><<<1, 32>>>(xnew, reps, cyc); rep("no gst + sts + vol");
        k_chain<0, 0, 1><<<1, 32>>>(xnew, reps, cyc); rep("vol only");
        k_chain<0, 0, 0><<<1, 32>>>(xnew, reps, cyc); rep("plain lds");
        k_chain<1, 1, 0><<<1, 32>>>(xnew, reps, cyc); rep("relaxed.gpu + sts, plain lds");
    }
}
