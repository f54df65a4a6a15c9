// Microbenchmark: load latency of the polling flavours and the cross-SM hop
// (ping-pong through global memory) on B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__device__ __forceinline__ unsigned long long ld(const unsigned long long* p) {
    unsigned long long v;
    if (K == 0) asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (K == 1) asm volatile("ld.volatile.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (K == 2) asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (K == 3) asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (K == 4) asm volatile("ld.global.cv.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (K == 5) asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <int K>
__global__ void k_chase(const unsigned long long* next, int n, long long* cyc, unsigned long long* sink) {
    unsigned long long p = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = ld<K>(next + p);
    long long t1 = clock64();
    *cyc = t1 - t0;
    *sink = p;
}
// ping-pong: block 0 and block 1 (on different SMs) alternately increment a counter
template <int K>
__global__ void k_pingpong(unsigned long long* flag, int rounds, long long* ns) {
    const unsigned long long me = blockIdx.x;
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < rounds; ++r) {
        const unsigned long long want = 2 * r + me;
        while (ld<K>(flag) != want) {
        }
        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(flag), "l"(want + 1) : "memory");
    }
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (me == 0) *ns = t1 - t0;
}
int main() {
    const int N = 1 << 16;
    unsigned long long* next;
    cudaMalloc(&next, N * 8);
    unsigned long long* h = new unsigned long long[N];
    for (int i = 0; i < N; ++i) h[i] = (i * 40503ull + 7919) % N;  // scattered chase in 512 KB (L2 resident)
    cudaMemcpy(next, h, N * 8, cudaMemcpyHostToDevice);
    long long* cyc;
    cudaMalloc(&cyc, 8);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const char* names[6] = {"ld.relaxed.gpu", "ld.volatile", "ld.global.cg", "ld.acquire.gpu", "ld.global.cv", "ld.relaxed.sys"};
    long long hc;
    for (int rep = 0; rep < 2; ++rep) {
#define RUN(K)                                                   \
    k_chase<K><<<1, 1>>>(next, 4096, cyc, sink);                 \
    cudaDeviceSynchronize();                                     \
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);             \
    printf("chase %-16s %.0f cycles/load\n", names[K], hc / 4096.0);
        RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
    }
    unsigned long long* flag;
    cudaMalloc(&flag, 8);
    for (int rep = 0; rep < 2; ++rep) {
#define PP(K)                                                               \
    cudaMemset(flag, 0, 8);                                                 \
    k_pingpong<K><<<2, 1>>>(flag, 10000, cyc);                              \
    cudaDeviceSynchronize();                                                \
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);                        \
    printf("ping-pong %-16s %.0f ns per one-way hop\n", names[K], hc / 20000.0);
        PP(0) PP(1) PP(2) PP(3)
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
