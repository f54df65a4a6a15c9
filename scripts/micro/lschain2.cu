// Microbenchmark 2: which part of the level-synchronous step costs cycles.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NSTEP = 4096;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int V>
__global__ void k(double* gx, long long* cyc, int spc) {
    __shared__ double xs[1024];
    __shared__ uint64_t bar[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) xs[i] = 1.0 + i * 1e-3;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar + 1)), "r"(1) : "memory");
    }
    __syncthreads();
    if (warp == 1) {  // a spinning waiter on a barrier that completes at the end
        if (lane == 0)
            asm volatile(
                "{\n .reg .pred p;\n"
                "W_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                " @!p bra W_%=;\n}" ::"r"(smem_u32(bar + 1)),
                "r"(0)
                : "memory");
        return;
    }
    if (warp == 2) {  // a global poller
        unsigned long long v = 0;
        while (true) {
            asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(gx + 4096 + lane * 16) : "memory");
            if (__any_sync(0xffffffffu, v == 12345)) break;
        }
        return;
    }
    volatile double* vxs = xs;
    const double e0 = 0.25, e1 = 0.125, c = 1.0;
    const int s0 = (lane + 31) & 1023, s1 = (lane + 1) & 1023;
    const int row = (V == 6 && lane >= 20) ? -1 : lane * 97 + 13;
    long long t0 = clock64();
    for (int s = 0; s < NSTEP; ++s) {
        double x = fma(-e0, vxs[(s0 + s * 32) & 1023], c);
        x = fma(-e1, vxs[(s1 + s * 32) & 1023], x);
        if (V == 6) {
            if (row >= 0) {
                xs[((s + 1) * 32 + lane) & 1023] = x;
                asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(gx + row + (s & 7) * 4096),
                             "l"(__double_as_longlong(x))
                             : "memory");
            }
        } else {
            xs[((s + 1) * 32 + lane) & 1023] = x;
        }
        if (V == 5)
            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(gx + row + (s & 7) * 4096),
                         "l"(__double_as_longlong(x))
                         : "memory");
        if (V == 8) gx[row + (s & 7) * 4096] = x;
        __syncwarp();
        if (V == 7) {
            const int c0 = s / spc;
            if (s - c0 * spc == spc - 1 && lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar + 1)) : "memory");
    if (lane == 0) gx[4096] = 0;
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(gx + 4096 + lane * 16), "l"(12345ll) : "memory");
}

template <int V>
void run(const char* name, int threads, double* gx, long long* cyc) {
    for (int r = 0; r < 2; ++r) {
        cudaMemset(gx, 0, 8 * 65536);
        k<V><<<1, threads>>>(gx, cyc, 14);
    }
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-52s %.1f cycles/step\n", name, double(h) / NSTEP);
}

int main() {
    double* gx;
    long long* cyc;
    cudaMalloc(&gx, 8 * 65536);
    cudaMalloc(&cyc, 8 * 32);
    run<0>("base (1 warp)", 32, gx, cyc);
    run<0>("base + mbarrier waiter warp", 64, gx, cyc);
    run<0>("base + waiter + global poller warps", 96, gx, cyc);
    run<5>("+ st.relaxed.gpu scattered", 32, gx, cyc);
    run<8>("+ plain st.global scattered", 32, gx, cyc);
    run<6>("divergent (row>=0) STS + st.relaxed", 32, gx, cyc);
    run<7>("+ s/spc + mbarrier arrive", 32, gx, cyc);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
