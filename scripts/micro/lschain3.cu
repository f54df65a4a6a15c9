// Microbenchmark 3: the gs_ls.cu compute-warp loop with features switched off
// one at a time (single group, synthetic ND=2 program, no imports needed).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kCH = 16384, kNS = 4, ND = 2;
constexpr int kC = 16, kE = 16 + 256, kS = kE + 256 * ND, kR = kS + 128 * ND, kBytes = kR + 256;
constexpr int kSPC = kCH / kBytes, kChunk = kSPC * kBytes;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
                     smem_u32(b)), "r"(parity) : "memory");
}
struct Regs {
    int need, pos0, row;
    double c, e[ND];
    int sl[ND];
};
__device__ __forceinline__ void ld(const char* st, int lane, Regs& r) {
    const int2 h = *reinterpret_cast<const int2*>(st);
    r.need = h.x;
    r.pos0 = h.y;
    r.c = reinterpret_cast<const double*>(st + kC)[lane];
    for (int d = 0; d < ND; ++d) r.e[d] = reinterpret_cast<const double*>(st + kE)[d * 32 + lane];
    const int2 q = reinterpret_cast<const int2*>(st + kS)[lane];
    r.sl[0] = q.x;
    r.sl[1] = q.y;
    r.row = reinterpret_cast<const int*>(st + kR)[lane];
}

// F: bit0 TMA ring (else static smem program), bit1 import check, bit2 STG, bit3 pipelined loads, bit4 arrive
template <int F>
__global__ void __launch_bounds__(96, 1) k(const char* prog, int nsteps, double* xnew, long long* cyc) {
    extern __shared__ __align__(128) unsigned char sm[];
    char* ring = (char*)sm;
    uint64_t* full = (uint64_t*)(sm + kNS * kCH);
    uint64_t* empty = full + kNS;
    volatile int* imported = (volatile int*)(empty + kNS);
    double* xs = (double*)(sm + kNS * kCH + 2 * kNS * 8 + 16);
    const int W = 64, trash = W + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunks = (nsteps + kSPC - 1) / kSPC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + s)), "r"(1) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + s)), "r"(1) : "memory");
        }
        *imported = 1 << 30;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < W + 2; i += blockDim.x) xs[i] = 1.0;
    if (!(F & 1))
        for (int c = 0; c < kNS; ++c)
            for (int i = threadIdx.x; i < kChunk / 16; i += blockDim.x)
                reinterpret_cast<int4*>(ring + c * kCH)[i] = reinterpret_cast<const int4*>(prog + c * kChunk)[i];
    __syncthreads();
    if (warp == 2) {
        if ((F & 1) && lane == 0)
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % kNS;
                if (c >= kNS) mbar_wait(empty + s, ((c / kNS) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(kChunk) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(ring + s * kCH)), "l"(prog + (int64_t)c * kChunk), "r"(kChunk), "r"(smem_u32(full + s)) : "memory");
            }
        return;
    }
    if (warp == 1) return;
    const volatile double* vxs = xs;
    int have = 0;
    if (F & 1) mbar_wait(full, 0);
    Regs cur, nxt;
    ld(ring, lane, cur);
    int kk = 0, chunk = 0;
    long long t0 = clock64();
    for (int s = 0; s < nsteps; ++s) {
        int k1 = kk + 1, c1 = chunk;
        if (k1 == kSPC) {
            k1 = 0;
            ++c1;
        }
        if (F & 8) {
            if (s + 1 < nsteps) {
                if ((F & 1) && k1 == 0) mbar_wait(full + (c1 & (kNS - 1)), (c1 / kNS) & 1);
                ld(ring + (c1 & (kNS - 1)) * kCH + k1 * kBytes, lane, nxt);
            }
        } else {
            ld(ring + (chunk & (kNS - 1)) * kCH + kk * kBytes, lane, cur);
        }
        if ((F & 2) && cur.need > have) {
            while ((have = *imported) < cur.need) {
            }
            __threadfence_block();
        }
        double xv[ND];
        for (int d = 0; d < ND; ++d) xv[d] = vxs[cur.sl[d]];
        double x = cur.c;
        for (int d = 0; d < ND; ++d) x = fma(-cur.e[d], xv[d], x);
        xs[cur.row >= 0 ? ((cur.pos0 + lane) & (W - 1)) : trash] = x;
        if (F & 4)
            asm volatile("{\n .reg .pred p;\n setp.ge.s32 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(xnew + cur.row),
                         "l"(__double_as_longlong(x)), "r"(cur.row) : "memory");
        __syncwarp();
        if (F & 16)
            asm volatile("{\n .reg .pred p;\n setp.ne.s32 p, %1, 0;\n @p mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(
                             smem_u32(empty + (chunk & (kNS - 1)))), "r"(int(kk == kSPC - 1) & int(lane == 0)) : "memory");
        kk = k1;
        chunk = c1;
        if (F & 8) cur = nxt;
        if (!(F & 1)) chunk &= 3;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
}


__device__ __forceinline__ void ld_sl(const char* st, int lane, int* sl) {
    int2 q;
    asm volatile("ld.volatile.shared.v2.s32 {%0, %1}, [%2];" : "=r"(q.x), "=r"(q.y) : "r"(smem_u32(st + kS + 8 * lane)));
    sl[0] = q.x;
    sl[1] = q.y;
}
__device__ __forceinline__ double ldv(const char* p) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ int ldvi(const char* p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
    return v;
}

// restructured: chunk loop outside, steps inside; per step: dep loads first,
// then the next step's slots (one LDS), then this step's coefficients; import
// wait as a uniform asm loop; STG predicated (G=1) or omitted.
template <int G, int IMP>
__global__ void __launch_bounds__(96, 1) k2(const char* prog, int nsteps, double* xnew, long long* cyc) {
    extern __shared__ __align__(128) unsigned char sm[];
    char* ring = (char*)sm;
    uint64_t* full = (uint64_t*)(sm + kNS * kCH);
    uint64_t* empty = full + kNS;
    int* imported = (int*)(empty + kNS);
    double* xs = (double*)(sm + kNS * kCH + 2 * kNS * 8 + 16);
    const int W = 64, trash = W + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunks = (nsteps + kSPC - 1) / kSPC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + s)), "r"(1) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + s)), "r"(1) : "memory");
        }
        *imported = 1 << 30;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < W + 2; i += blockDim.x) xs[i] = 1.0;
    __syncthreads();
    if (warp == 2) {
        if (lane == 0)
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % kNS;
                if (c >= kNS) mbar_wait(empty + s, ((c / kNS) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(kChunk) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(ring + s * kCH)), "l"(prog + (int64_t)c * kChunk), "r"(kChunk), "r"(smem_u32(full + s)) : "memory");
            }
        return;
    }
    if (warp == 1) return;
    long long t0 = clock64();
    const unsigned imp_a = smem_u32(imported);
    int have = 0;
    for (int c = 0; c < nchunks; ++c) {
        mbar_wait(full + (c & (kNS - 1)), (c / kNS) & 1);
        const char* ch = ring + (c & (kNS - 1)) * kCH;
        const int cnt = min(kSPC, nsteps - c * kSPC);
        int sl[ND];
        ld_sl(ch, lane, sl);
        for (int k = 0; k < cnt; ++k) {
            const char* st = ch + k * kBytes;
            if (IMP) {
                const int need = ldvi(st);
                asm volatile(
                    "{\n .reg .pred p;\n .reg .s32 r;\n"
                    " setp.le.s32 p, %2, %0;\n"
                    " @p bra.uni LD%=;\n"
                    "LW%=:\n ld.volatile.shared.s32 r, [%1];\n setp.lt.s32 p, r, %2;\n @p bra.uni LW%=;\n"
                    " mov.s32 %0, r;\n fence.acq_rel.cta;\n"
                    "LD%=:\n}" : "+r"(have) : "r"(imp_a), "r"(need) : "memory");
            }
            double xv[ND];
            for (int d = 0; d < ND; ++d) asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(xv[d]) : "r"(smem_u32(xs + sl[d])));
            if (k + 1 < cnt) ld_sl(st + kBytes, lane, sl);
            double x = ldv(st + kC + 8 * lane);
            double e0 = ldv(st + kE + 8 * lane), e1 = ldv(st + kE + 256 + 8 * lane);
            const int row = ldvi(st + kR + 4 * lane), pos0 = ldvi(st + 4);
            x = fma(-e0, xv[0], x);
            x = fma(-e1, xv[1], x);
            xs[row >= 0 ? ((pos0 + lane) & (W - 1)) : trash] = x;
            if (G)
                asm volatile("{\n .reg .pred p;\n setp.ge.s32 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(xnew + row),
                             "l"(__double_as_longlong(x)), "r"(row) : "memory");
            __syncwarp();
        }
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + (c & (kNS - 1)))) : "memory");
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
}

template <int G, int IMP>
void run2(const char* name, const char* prog, int nsteps, double* xnew, long long* cyc) {
    cudaFuncSetAttribute(k2<G, IMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int r = 0; r < 2; ++r) k2<G, IMP><<<1, 96, kNS * kCH + 2 * kNS * 8 + 16 + 70 * 8>>>(prog, nsteps, xnew, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("k2 %-48s %.1f cycles/step (%s)\n", name, double(h) / nsteps, cudaGetErrorString(cudaGetLastError()));
}


// k3: chunk loop outside; inner loop branch-free except the uniform import
// check; registers for step k+1 loaded at the end of step k (reads past the
// chunk's last step are discarded).  Program layout v2: c, e0, e1 as before,
// {sl0, sl1} int2 per lane, {row, myslot} int2 per lane (in the row array slot).
template <int G, int IMP>
__global__ void __launch_bounds__(96, 1) k3(const char* prog, int nsteps, double* xnew, long long* cyc) {
    extern __shared__ __align__(128) unsigned char sm[];
    char* ring = (char*)sm;
    uint64_t* full = (uint64_t*)(sm + kNS * kCH);
    uint64_t* empty = full + kNS;
    int* imported = (int*)(empty + kNS);
    double* xs = (double*)(sm + kNS * kCH + 2 * kNS * 8 + 16);
    const int W = 64;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunks = (nsteps + kSPC - 1) / kSPC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + s)), "r"(1) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + s)), "r"(1) : "memory");
        }
        *imported = 1 << 30;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < W + 2; i += blockDim.x) xs[i] = 1.0;
    __syncthreads();
    if (warp == 2) {
        if (lane == 0)
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % kNS;
                if (c >= kNS) mbar_wait(empty + s, ((c / kNS) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(kChunk) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(ring + s * kCH)), "l"(prog + (int64_t)c * kChunk), "r"(kChunk), "r"(smem_u32(full + s)) : "memory");
            }
        return;
    }
    if (warp == 1) return;
    long long t0 = clock64();
    const unsigned imp_a = smem_u32(imported);
    volatile double* vxs = xs;
    int have = 0;
    for (int c = 0; c < nchunks; ++c) {
        mbar_wait(full + (c & (kNS - 1)), (c / kNS) & 1);
        const char* st = ring + (c & (kNS - 1)) * kCH;
        const int cnt = min(kSPC, nsteps - c * kSPC);
        double cc = reinterpret_cast<const double*>(st + kC)[lane];
        double e0 = reinterpret_cast<const double*>(st + kE)[lane];
        double e1 = reinterpret_cast<const double*>(st + kE + 256)[lane];
        int2 sl = reinterpret_cast<const int2*>(st + kS)[lane];
        int2 rs = reinterpret_cast<const int2*>(st + kR)[lane];
        int need = *reinterpret_cast<const int*>(st);
        for (int k = 0; k < cnt; ++k) {
            if (IMP)
                asm volatile(
                    "{\n .reg .pred p;\n .reg .s32 r;\n"
                    " setp.le.s32 p, %2, %0;\n"
                    " @p bra.uni LD%=;\n"
                    "LW%=:\n ld.volatile.shared.s32 r, [%1];\n setp.lt.s32 p, r, %2;\n @p bra.uni LW%=;\n"
                    " mov.s32 %0, r;\n fence.acq_rel.cta;\n"
                    "LD%=:\n}" : "+r"(have) : "r"(imp_a), "r"(need) : "memory");
            double x0, x1;
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(x0) : "r"(smem_u32(xs + sl.x)));
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(x1) : "r"(smem_u32(xs + sl.y)));
            st += kBytes;
            const unsigned sa = smem_u32(st);
            double ncc, ne0, ne1;
            int2 nrs;
            asm volatile("ld.volatile.shared.v2.s32 {%0, %1}, [%2];" : "=r"(sl.x), "=r"(sl.y) : "r"(sa + kS + 8 * lane));
            asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(need) : "r"(sa));
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(ncc) : "r"(sa + kC + 8 * lane));
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(ne0) : "r"(sa + kE + 8 * lane));
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(ne1) : "r"(sa + kE + 256 + 8 * lane));
            asm volatile("ld.volatile.shared.v2.s32 {%0, %1}, [%2];" : "=r"(nrs.x), "=r"(nrs.y) : "r"(sa + kR + 8 * lane));
            double x;
            asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(x) : "d"(-e0), "d"(x0), "d"(cc));
            asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(x) : "d"(-e1), "d"(x1), "d"(x));
            asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(smem_u32(xs + rs.y)), "d"(x) : "memory");
            if (G)
                asm volatile("{\n .reg .pred p;\n setp.ge.s32 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(xnew + rs.x),
                             "l"(__double_as_longlong(x)), "r"(rs.x) : "memory");
            cc = ncc;
            e0 = ne0;
            e1 = ne1;
            rs = nrs;
            __syncwarp();
        }
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + (c & (kNS - 1)))) : "memory");
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
}

template <int G, int IMP>
void run3(const char* name, const char* prog, int nsteps, double* xnew, long long* cyc) {
    cudaFuncSetAttribute(k3<G, IMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int r = 0; r < 2; ++r) k3<G, IMP><<<1, 96, kNS * kCH + 2 * kNS * 8 + 16 + 70 * 8 + 2048>>>(prog, nsteps, xnew, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("k3 %-48s %.1f cycles/step (%s)\n", name, double(h) / nsteps, cudaGetErrorString(cudaGetLastError()));
}

template <int F>
void run(const char* name, const char* prog, int nsteps, double* xnew, long long* cyc) {
    cudaFuncSetAttribute(k<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int r = 0; r < 2; ++r) k<F><<<1, 96, kNS * kCH + 2 * kNS * 8 + 16 + 70 * 8>>>(prog, nsteps, xnew, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("F=%2d %-48s %.1f cycles/step (%s)\n", F, name, double(h) / nsteps, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int nsteps = 2000;
    const int nch = (nsteps + kSPC - 1) / kSPC;
    char* h = (char*)calloc(size_t(nch) * kChunk + kNS * kCH, 1);
    for (int s = 0; s < nch * kSPC; ++s) {
        char* st = h + (s / kSPC) * kChunk + (s % kSPC) * kBytes;
        int* hd = (int*)st;
        hd[0] = 0;
        hd[1] = s * 32;
        for (int l = 0; l < 32; ++l) {
            ((double*)(st + kC))[l] = 1.0;
            for (int d = 0; d < ND; ++d) ((double*)(st + kE))[d * 32 + l] = 0.1;
            ((int*)(st + kS))[l * 2] = (s * 32 + l + 63) & 63;
            ((int*)(st + kS))[l * 2 + 1] = (s * 32 + l + 33) & 63;
            ((int*)(st + kR))[2 * l] = l < 27 ? (l * 2000 + s) % 100000 : -1;
            ((int*)(st + kR))[2 * l + 1] = l < 27 ? ((s * 32 + l) & 63) : 65;
        }
    }
    char* prog;
    double* xnew;
    long long* cyc;
    cudaMalloc(&prog, size_t(nch) * kChunk + kNS * kCH);
    cudaMemcpy(prog, h, size_t(nch) * kChunk + kNS * kCH, cudaMemcpyHostToDevice);
    cudaMalloc(&xnew, 8 * 100000);
    cudaMalloc(&cyc, 64);
    run<0>("static smem program, unpipelined", prog, nsteps, xnew, cyc);
    run<8>("static smem, pipelined", prog, nsteps, xnew, cyc);
    run<8 | 2>("+ import check", prog, nsteps, xnew, cyc);
    run<8 | 2 | 4>("+ STG", prog, nsteps, xnew, cyc);
    run<1 | 8>("TMA ring, pipelined, no arrive (deadlocks?)", prog, kSPC * 4, xnew, cyc);
    run<1 | 8 | 16>("TMA ring + arrive", prog, nsteps, xnew, cyc);
    run<1 | 8 | 16 | 2 | 4>("full kernel", prog, nsteps, xnew, cyc);
    run<1 | 16 | 2 | 4>("full kernel, unpipelined", prog, nsteps, xnew, cyc);
    run2<0, 0>("restructured, no STG, no import", prog, nsteps, xnew, cyc);
    run2<0, 1>("restructured, import check", prog, nsteps, xnew, cyc);
    run2<1, 1>("restructured, import + STG", prog, nsteps, xnew, cyc);
    run3<0, 0>("branch-free inner loop", prog, nsteps, xnew, cyc);
    run3<0, 1>("+ import check", prog, nsteps, xnew, cyc);
    run3<1, 1>("+ STG", prog, nsteps, xnew, cyc);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
