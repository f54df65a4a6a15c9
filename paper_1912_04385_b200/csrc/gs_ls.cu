// gs_ls.cu -- level-synchronous pipelined Gauss-Seidel sweep (K14, v2).
//
// Same natural-order semantics as the other sweep kernels
// (sym_gauss_seidel, amg.cpp:25-43): x_i = (b_i - sum_{k<i} a_ik x_k^new
// - sum_{k>i} a_ik x_k^old) / a_ii in the forward direction, the mirror image
// backward.  What changes is how the dependency DAG is mapped onto the GPU:
//
//   * GROUPS.  The rows are cut into K contiguous ranges in sweep order, one
//     thread block (one SM) each.  A group's rows are processed by ONE compute
//     warp in global DAG-level order, <= 32 rows (one "step") at a time, with
//     only a __syncwarp between steps: every dependency inside the group is a
//     shared-memory read of a value the same warp wrote one or a few steps
//     earlier.  The per-level cost is a few dependent instructions instead of
//     a cross-SM hop (>= 0.38 us per hop).
//   * PIPELINE.  Dependencies may only cross into the previous group (checked
//     at setup; the level falls back to the other kernels otherwise).  An
//     importer warp polls the previous group's published values in the order
//     they are produced and copies them into a shared-memory halo; the compute
//     warp only checks a shared-memory counter.  The cross-SM latency is paid
//     once per group boundary (pipeline fill), not once per DAG level.
//   * PROGRAM.  Everything that does not depend on the sweep's new values --
//     the row's coefficients pre-multiplied by 1/a_ii and the shared-memory
//     slots of its dependencies -- is compiled at setup into a per-group
//     stream of fixed-size chunks, in processing order, which a loader warp
//     streams into a shared-memory ring with 1-D TMA bulk copies
//     (cp.async.bulk + mbarrier).  The part of each row that depends on the
//     previous iterate, c'_i = (b_i - sum_old a_ik x_k^old) / a_ii, is computed
//     by a fully parallel pre-pass straight into the chunks.
//
// Own-group values live in a ring of W slots indexed by processing position
// (W > the largest position distance of a dependency + 32, checked at setup).
// Results differ from the warp-per-row sweep only by association (the old part
// is summed first, coefficients are pre-scaled by 1/a_ii) and stay within the
// 1e-10 apply bar.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "mprec.cuh"

namespace mg {
namespace {

constexpr int kThreads = 96;  // warp 0: compute, warp 1: importer, warp 2: loader
constexpr int kLsExportBit = 1 << 30;       // record myslot: row is read by the next group
constexpr int kLsSlotMask = kLsExportBit - 1;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "LS_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LS_WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_ls(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// c'_i = (b_i - sum_{old k} a_ik xold_k) * invd_i, written into the row's program slot;
// exported rows (read by the next group's importer) get the kPending sentinel.
__global__ void k_ls_pre(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                         const int* __restrict__ diag, const double* __restrict__ invd, const double* __restrict__ b,
                         const double* __restrict__ xold, int dir, const long long* __restrict__ coff, char* prog,
                         double* xnew) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double old = 0.0;
    if (xold) {
        const int d = __ldg(diag + i);
        const int k0 = dir > 0 ? d + 1 : __ldg(rp + i), k1 = dir > 0 ? __ldg(rp + i + 1) : d;
        for (int k = k0; k < k1; ++k) old += __ldg(v + k) * __ldg(xold + __ldg(ci + k));
    }
    const double cv = (__ldg(b + i) - old) * __ldg(invd + i);
    const long long o = __ldg(coff + i);
    *reinterpret_cast<double*>(prog + (o & ~1ll)) = cv;
    if (o & 1) reinterpret_cast<unsigned long long*>(xnew)[i] = kPending;
}

// Step layout (16-byte aligned; a step never straddles a chunk):
//   int4 {cnt, cls, need, bytes}     rows, dependency class, imports required, step size
//   cnt lane records of RS(cls) bytes, record of lane q at 16 + q * RS:
//     +0  int    sl[4]               shared-memory slots of dependencies 0..3
//     +16 double c                   c'_i (written by the pre-pass)
//     +24 int    row, myslot         output row, own ring slot
//     +32 double e[ND]               a_ij / a_ii (0 for padding)
//     +32+8ND int sl[4..ND)
// The class is the step's widest row rounded up to ND = 2, 4, 8, 16, 32; the
// record size has an odd number of 16-byte units so that the 32 lanes' 16-byte
// loads are bank-conflict free.  A chunk starts with int4 {nsteps, 0, 0, 0}.
__host__ __device__ constexpr int ls_nd(int cls) { return 2 << cls; }
__host__ __device__ constexpr int ls_rs(int cls) {
    return cls == 0 ? 48 : cls == 1 ? 80 : cls == 2 ? 112 : cls == 3 ? 208 : 400;
}

// dependency part of one row: x = c - sum_d e_d x_d (sequential for ND = 2,
// a pairwise tree otherwise: depth log2(ND) + 2 instead of ND)
template <int ND>
__device__ __forceinline__ double ls_dot(const double* e, const double* xv, double c) {
    if (ND == 2) return fma(-e[1], xv[1], fma(-e[0], xv[0], c));
    double p[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) p[d] = e[d] * xv[d];
#pragma unroll
    for (int w = ND / 2; w >= 1; w /= 2)
#pragma unroll
        for (int d = 0; d < w; ++d) p[d] += p[d + w];
    return c - p[0];
}

template <int ND>
__device__ __forceinline__ void ls_slots(const char* rec, int* sl) {
    const int4 q = *reinterpret_cast<const int4*>(rec);
    sl[0] = q.x;
    sl[1] = q.y;
    if (ND > 2) {
        sl[2] = q.z;
        sl[3] = q.w;
    }
#pragma unroll
    for (int d = 4; d < ND; d += 4) {
        const int4 r = reinterpret_cast<const int4*>(rec + 32 + 8 * ND)[(d - 4) / 4];
        sl[d] = r.x;
        sl[d + 1] = r.y;
        sl[d + 2] = r.z;
        sl[d + 3] = r.w;
    }
}

// One thread block per group; ND (the level's widest row, rounded up) is a
// template parameter so the step loop has no class switch.
template <int ND>
__global__ void __launch_bounds__(kThreads, 1) k_gs_ls(const char* __restrict__ prog, const int2* __restrict__ gch,
                                                        const int* __restrict__ imp, const int2* __restrict__ gimp,
                                                        double* xnew, int W, int trash, int ns, long long* stats,
                                                        int push) {
    constexpr int RS = ls_rs(ND == 2 ? 0 : ND == 4 ? 1 : ND == 8 ? 2 : ND == 16 ? 3 : 4);
    extern __shared__ __align__(128) unsigned char sm[];
    char* ring = reinterpret_cast<char*>(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + ns * kLsCH);
    uint64_t* empty = full + ns;
    int* imported = reinterpret_cast<int*>(empty + ns);
    double* xs = reinterpret_cast<double*>(sm + ns * kLsCH + 2 * ns * 8 + 16);
    const int g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2 ch = gch[g];  // first chunk, chunk count
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        *imported = 0;
        xs[W] = 0.0;  // zero slot (padding dependencies)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // cluster push (launched as clusters of 2): the even CTA of a pair stores its
    // exported values straight into the odd CTA's halo (DSMEM), whose importer
    // then only polls shared memory; the halo starts as kPending in every thread
    // block and a cluster barrier orders that before any remote store
    const bool pushed_in = push && (g & 1);  // my halo is written by my cluster peer
    if (pushed_in) {
        const int nimp = gimp[g].y;
        for (int i = threadIdx.x; i < nimp; i += blockDim.x)
            reinterpret_cast<unsigned long long*>(xs + W + 1)[i] = kPending;
    }
    __syncthreads();
    if (push) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp == 2) {  // loader: program chunks -> shared-memory ring (1-D TMA bulk copies)
        if (lane == 0)
            for (int c = 0; c < ch.y; ++c) {
                const int s = c & (ns - 1);
                if (c >= ns) mbar_wait(empty + s, ((c / ns) - 1) & 1);
                mbar_expect_tx(full + s, kLsCH);
                bulk_g2s(ring + s * kLsCH, prog + (int64_t)(ch.x + c) * kLsCH, kLsCH, full + s);
            }
        return;
    }
    if (warp == 1 && pushed_in) {  // importer, cluster push: poll the local halo
        const int nimp = gimp[g].y;
        volatile unsigned long long* halo = reinterpret_cast<volatile unsigned long long*>(xs + W + 1);
        volatile int* vimp = imported;
        int base = 0;
        while (base < nimp) {
            const int idx = base + lane;
            const bool ready = idx < nimp && halo[idx] != kPending;
            const unsigned m = __ballot_sync(0xffffffffu, ready);
            const int pre = min(m == 0xffffffffu ? 32 : __ffs(~m) - 1, nimp - base);
            if (pre > 0) {
                if (lane == 0) {
                    asm volatile("fence.acq_rel.cluster;" ::: "memory");
                    *vimp = base + pre;
                }
                base += pre;
            }
        }
        return;
    }
    if (warp == 1) {  // importer: previous group's values -> halo, in production order
        const int2 gi = gimp[g];
        const int* rows = imp + gi.x;
        const int nimp = gi.y;
        volatile double* halo = xs + W + 1;
        volatile int* vimp = imported;
        int base = 0;
        while (base < nimp) {
            const int idx = base + lane;
            const bool in = idx < nimp;
            unsigned long long raw = kPending;
            if (in) raw = ld_relaxed_ls(xnew + __ldg(rows + idx));
            const bool ready = in && raw != kPending;
            const unsigned m = __ballot_sync(0xffffffffu, ready);
            const int pre = min(m == 0xffffffffu ? 32 : __ffs(~m) - 1, nimp - base);
            if (lane < pre) halo[idx] = __longlong_as_double((long long)raw);
            if (pre > 0) {
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    *vimp = base + pre;
                }
                base += pre;
            }
        }
        return;
    }
    // compute warp.  Software pipeline: at step k the registers of step k
    // (header, slots) are already loaded; the next header and slots are issued
    // right after this step's dependency loads, so the only latencies left on the
    // critical path are LDS(dependencies) -> FMAs -> STS.  The import wait is a
    // warp-uniform loop inside one asm block, padding lanes read a valid record
    // (min(lane, cnt - 1)) and their stores are predicated off: no divergent branch.
    const volatile double* vxs = xs;
    const unsigned imp_a = smem_u32(imported);
    int have = 0;
    long long t_start = 0;
    if (stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    // cluster push target: the peer CTA's halo (shared::cluster address)
    const bool push_out = push && !(g & 1) && g + 1 < int(gridDim.x);
    unsigned peer_halo = 0;
    int nexp = 0;
    if (push_out)
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_halo) : "r"(smem_u32(xs + W + 1)), "r"(1));
    for (int c = 0; c < ch.y; ++c) {
        const int slot = c & (ns - 1);
        mbar_wait(full + slot, (c / ns) & 1);
        const char* st = ring + slot * kLsCH;
        const int nsteps = *reinterpret_cast<const int*>(st);
        st += 16;
        int4 h = *reinterpret_cast<const int4*>(st);
        int sl[ND];
        ls_slots<ND>(st + 16 + min(lane, h.x - 1) * RS, sl);
        for (int k = 0; k < nsteps; ++k) {
            asm volatile(
                "{\n .reg .pred p;\n .reg .s32 r;\n"
                " setp.le.s32 p, %2, %0;\n"
                " @p bra.uni LSD%=;\n"
                "LSW%=:\n ld.volatile.shared.s32 r, [%1];\n setp.lt.s32 p, r, %2;\n @p bra.uni LSW%=;\n"
                " mov.s32 %0, r;\n fence.acq_rel.cta;\n"
                "LSD%=:\n}"
                : "+r"(have)
                : "r"(imp_a), "r"(h.z)
                : "memory");
            const char* rec = st + 16 + min(lane, h.x - 1) * RS;
            // next step's header first: its slots can then be loaded while this
            // step's dependencies are summed (garbage after the chunk's last step)
            const char* stn = st + h.w;
            int4 hn;
            asm volatile("ld.volatile.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(hn.x), "=r"(hn.y), "=r"(hn.z), "=r"(hn.w)
                         : "r"(smem_u32(stn)));
            double xv[ND];
#pragma unroll
            for (int d = 0; d < ND; ++d) MG_DCHECK(sl[d] >= 0 && sl[d] < trash);
            MG_DCHECK(h.x >= 1 && h.x <= 32 && h.w >= 16 && h.w <= kLsCH && h.z >= 0 && h.z <= trash - W - 1);
#pragma unroll
            for (int d = 0; d < ND; ++d) xv[d] = vxs[sl[d]];
            const bool more = k + 1 < nsteps;  // (select, not a branch)
            ls_slots<ND>((more ? stn : st) + 16 + min(lane, (more ? hn.x : h.x) - 1) * RS, sl);
            const double cc = *reinterpret_cast<const double*>(rec + 16);
            const int2 rs = *reinterpret_cast<const int2*>(rec + 24);
            double e[ND];
#pragma unroll
            for (int d = 0; d < ND; d += 2) {
                const double2 q = reinterpret_cast<const double2*>(rec + 32)[d / 2];
                e[d] = q.x;
                e[d + 1] = q.y;
            }
            double x = ls_dot<ND>(e, xv, cc);
            // lane groups (header .y: pairs << 8 | quads << 16): quads on lanes
            // [0, 4 nq), pairs on [4 nq, 4 nq + 2 np); the group's other lanes hold
            // -(sums of further dependencies) with c' = 0
            if (h.y >> 8) {
                const int nq = (h.y >> 16) & 0xff, np2 = 4 * nq + 2 * ((h.y >> 8) & 0xff);
                const double o1 = __shfl_xor_sync(0xffffffffu, x, 1);
                if (lane < np2) x += o1;
                if (nq) {
                    const double o2 = __shfl_xor_sync(0xffffffffu, x, 2);
                    if (lane < 4 * nq) x += o2;
                }
            }
            const int row = lane < h.x ? rs.x : -1;
            MG_DCHECK(lane >= h.x || rs.x < 0 || (rs.y & kLsSlotMask) < W);
            asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(
                             smem_u32(xs + (lane < h.x ? (rs.y & kLsSlotMask) : trash))),
                         "d"(x)
                         : "memory");
            asm volatile(
                "{\n .reg .pred p;\n setp.ge.s32 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(xnew + row),
                "l"(__double_as_longlong(x)), "r"(row)
                : "memory");
            if (push_out) {
                // exported rows arrive in the peer's import order (processing order)
                const bool ex = lane < h.x && (rs.y & kLsExportBit);
                const unsigned m = __ballot_sync(0xffffffffu, ex);
                const int hidx = nexp + __popc(m & ((1u << lane) - 1));
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.s32 p, %2, 0;\n"
                    " @p st.relaxed.cluster.shared::cluster.b64 [%0], %1;\n}" ::"r"(peer_halo + 8u * unsigned(hidx)),
                    "l"(__double_as_longlong(x)), "r"(int(ex))
                    : "memory");
                nexp += __popc(m);
            }
            __syncwarp();
            st = stn;
            h = hn;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
    }
    if (stats && lane == 0) {
        long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        stats[4 * g + 0] = t_start;
        stats[4 * g + 1] = t_end;
        stats[4 * g + 2] = 0;
        stats[4 * g + 3] = 0;
    }
}

// Variable-width records (levels whose widest row has more than 4
// dependencies): the step header's class field is nd4 = ceil(widest row / 4),
// the record of lane q is
//   +0 int4 sl[0..3] | +16 double c' | +24 int row, myslot | +32 double e[0..3]
//   +64 + 48 (g - 1): int4 sl[4g..4g+3], double e[4g..4g+3]    (g = 1 .. nd4 - 1)
// padded to an odd number of 16-byte units (conflict-free lane-strided loads).
// Only the step's own width is loaded and summed (warp-uniform group loop), so
// a few wide rows no longer widen every record of the level.
__host__ __device__ constexpr int ls_rsv(int nd4) {
    return (16 + 48 * nd4) + ((((16 + 48 * nd4) >> 4) & 1) ? 0 : 16);
}

__device__ __forceinline__ double ls_quad(const volatile double* xs, int4 sl, const double* e) {
    const double x0 = xs[sl.x], x1 = xs[sl.y], x2 = xs[sl.z], x3 = xs[sl.w];
    const double2 a = reinterpret_cast<const double2*>(e)[0], b = reinterpret_cast<const double2*>(e)[1];
    return fma(a.x, x0, a.y * x1) + fma(b.x, x2, b.y * x3);
}

// dependency groups 1 .. NQ-1 of a variable-width record (NQ = the step's nd4)
template <int NQ>
__device__ __forceinline__ double lsv_rest(const char* rec, const volatile double* xs) {
    constexpr int M = NQ - 1;
    int4 sq[M];
#pragma unroll
    for (int q = 0; q < M; ++q) sq[q] = *reinterpret_cast<const int4*>(rec + 64 + 48 * q);
    double xv[4 * M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
        xv[4 * q] = xs[sq[q].x];
        xv[4 * q + 1] = xs[sq[q].y];
        xv[4 * q + 2] = xs[sq[q].z];
        xv[4 * q + 3] = xs[sq[q].w];
    }
    double p[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
        const double2 a = reinterpret_cast<const double2*>(rec + 64 + 48 * q + 16)[0];
        const double2 b = reinterpret_cast<const double2*>(rec + 64 + 48 * q + 16)[1];
        p[q] = fma(a.x, xv[4 * q], a.y * xv[4 * q + 1]) + fma(b.x, xv[4 * q + 2], b.y * xv[4 * q + 3]);
    }
#pragma unroll
    for (int w = 1; w < M; w *= 2)
#pragma unroll
        for (int q = 0; q + w < M; q += 2 * w) p[q] += p[q + w];
    return p[0];
}

__global__ void __launch_bounds__(kThreads, 1) k_gs_lsv(const char* __restrict__ prog, const int2* __restrict__ gch,
                                                         const int* __restrict__ imp, const int2* __restrict__ gimp,
                                                         double* xnew, int W, int trash, int ns) {
    extern __shared__ __align__(128) unsigned char sm[];
    char* ring = reinterpret_cast<char*>(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + ns * kLsCH);
    uint64_t* empty = full + ns;
    int* imported = reinterpret_cast<int*>(empty + ns);
    double* xs = reinterpret_cast<double*>(sm + ns * kLsCH + 2 * ns * 8 + 16);
    const int g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2 ch = gch[g];
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        *imported = 0;
        xs[W] = 0.0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 2) {
        if (lane == 0)
            for (int c = 0; c < ch.y; ++c) {
                const int s = c & (ns - 1);
                if (c >= ns) mbar_wait(empty + s, ((c / ns) - 1) & 1);
                mbar_expect_tx(full + s, kLsCH);
                bulk_g2s(ring + s * kLsCH, prog + (int64_t)(ch.x + c) * kLsCH, kLsCH, full + s);
            }
        return;
    }
    if (warp == 1) {
        const int2 gi = gimp[g];
        const int* rows = imp + gi.x;
        const int nimp = gi.y;
        volatile double* halo = xs + W + 1;
        volatile int* vimp = imported;
        int base = 0;
        while (base < nimp) {
            const int idx = base + lane;
            const bool in = idx < nimp;
            unsigned long long raw = kPending;
            if (in) raw = ld_relaxed_ls(xnew + __ldg(rows + idx));
            const bool ready = in && raw != kPending;
            const unsigned m = __ballot_sync(0xffffffffu, ready);
            const int pre = min(m == 0xffffffffu ? 32 : __ffs(~m) - 1, nimp - base);
            if (lane < pre) halo[idx] = __longlong_as_double((long long)raw);
            if (pre > 0) {
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    *vimp = base + pre;
                }
                base += pre;
            }
        }
        return;
    }
    const volatile double* vxs = xs;
    const unsigned imp_a = smem_u32(imported);
    int have = 0;
    for (int c = 0; c < ch.y; ++c) {
        const int slot = c & (ns - 1);
        mbar_wait(full + slot, (c / ns) & 1);
        const char* st = ring + slot * kLsCH;
        const int nsteps = *reinterpret_cast<const int*>(st);
        st += 16;
        int4 h = *reinterpret_cast<const int4*>(st);
        int4 s0 = *reinterpret_cast<const int4*>(st + 16 + min(lane, h.x - 1) * ls_rsv(h.y));
        for (int k = 0; k < nsteps; ++k) {
            asm volatile(
                "{\n .reg .pred p;\n .reg .s32 r;\n"
                " setp.le.s32 p, %2, %0;\n"
                " @p bra.uni LSD%=;\n"
                "LSW%=:\n ld.volatile.shared.s32 r, [%1];\n setp.lt.s32 p, r, %2;\n @p bra.uni LSW%=;\n"
                " mov.s32 %0, r;\n fence.acq_rel.cta;\n"
                "LSD%=:\n}"
                : "+r"(have)
                : "r"(imp_a), "r"(h.z)
                : "memory");
            const char* rec = st + 16 + min(lane, h.x - 1) * ls_rsv(h.y);
            // next step: header first, then (below) its first slot group
            const char* stn = st + h.w;
            int4 hn;
            asm volatile("ld.volatile.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(hn.x), "=r"(hn.y), "=r"(hn.z), "=r"(hn.w)
                         : "r"(smem_u32(stn)));
            MG_DCHECK(s0.x >= 0 && s0.x < trash && s0.y >= 0 && s0.y < trash && s0.z >= 0 && s0.z < trash &&
                      s0.w >= 0 && s0.w < trash);
            MG_DCHECK(h.x >= 1 && h.x <= 32 && h.y >= 1 && h.y <= 8 && h.w >= 16 && h.w <= kLsCH);
            const double x0 = vxs[s0.x], x1 = vxs[s0.y], x2 = vxs[s0.z], x3 = vxs[s0.w];
            const bool more = k + 1 < nsteps;
            const int4 s0n = *reinterpret_cast<const int4*>((more ? stn : st) + 16 +
                                                           min(lane, (more ? hn.x : h.x) - 1) *
                                                               ls_rsv(more ? hn.y : h.y));
            const double cc = *reinterpret_cast<const double*>(rec + 16);
            const int2 rs = *reinterpret_cast<const int2*>(rec + 24);
            const double2 ea = reinterpret_cast<const double2*>(rec + 32)[0], eb = reinterpret_cast<const double2*>(rec + 32)[1];
            // groups 1 .. nd4-1: one warp-uniform switch on the step's width, then
            // straight-line loads (all slots, all values) and a pairwise tree
            double rest;
            switch (h.y) {
                case 1: rest = 0.0; break;
                case 2: rest = lsv_rest<2>(rec, vxs); break;
                case 3: rest = lsv_rest<3>(rec, vxs); break;
                case 4: rest = lsv_rest<4>(rec, vxs); break;
                case 5: rest = lsv_rest<5>(rec, vxs); break;
                case 6: rest = lsv_rest<6>(rec, vxs); break;
                case 7: rest = lsv_rest<7>(rec, vxs); break;
                default: rest = lsv_rest<8>(rec, vxs); break;
            }
            const double acc = (fma(ea.x, x0, ea.y * x1) + fma(eb.x, x2, eb.y * x3)) + rest;
            const double x = cc - acc;
            const int row = lane < h.x ? rs.x : -1;
            asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(
                             smem_u32(xs + (lane < h.x ? (rs.y & kLsSlotMask) : trash))),
                         "d"(x)
                         : "memory");
            asm volatile(
                "{\n .reg .pred p;\n setp.ge.s32 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(xnew + row),
                "l"(__double_as_longlong(x)), "r"(row)
                : "memory");
            __syncwarp();
            st = stn;
            h = hn;
            s0 = s0n;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
    }
}

__global__ void k_ls_testvec(double* b, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = 1.5 + sin(0.37 * i);
}


}  // namespace

int ls_smem_bytes(int W, int hmax, int ns) { return ns * kLsCH + 2 * ns * 8 + 16 + (W + 2 + hmax) * 8; }

// Build the group programs of one sweep direction.  Returns false (and leaves
// s.ok = false) when the level does not fit the scheme: a dependency reaching
// beyond the previous group, or a ring + halo larger than shared memory.
// Host-side program of one sweep direction (built from a host copy of the level).
struct LsBuilt {
    bool ok = false;
    int K = 0, W = 0, hmax = 0, dir = 0, nsteps = 0, nchunks = 0, maxdist = 0, nd = 0, ns = 0, cls = 0;
    std::vector<char> prog;
    std::vector<int2> gch, gimp;
    std::vector<int> imp;
    std::vector<long long> coff;
};

static void ls_build_host(const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<double>& v,
                          const std::vector<int>& lev, const std::vector<double>& invd, int n, int dir, int K,
                          int rec_mode, LsBuilt& out) {
    out = LsBuilt();
    if (n < 64 || K < 1) return;
    K = std::min(K, n / 32);
    if (K < 1) return;
    auto row_of_t = [&](int t) { return dir > 0 ? t : n - 1 - t; };
    auto is_dep = [&](int i, int j) { return dir > 0 ? j < i : j > i; };
    std::vector<int> gstart(K + 1), gid(n);
    for (int g = 0; g <= K; ++g) gstart[g] = int((int64_t)g * n / K);
    for (int g = 0; g < K; ++g)
        for (int t = gstart[g]; t < gstart[g + 1]; ++t) gid[row_of_t(t)] = g;
    for (int i = 0; i < n; ++i)
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (is_dep(i, j) && gid[j] != gid[i] && gid[j] != gid[i] - 1) return;
        }
    auto ndeps = [&](int i) {
        int d = 0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) d += is_dep(i, ci[k]) ? 1 : 0;
        return d;
    };
    std::vector<int> nd(n);
    int maxnd = 0;
    for (int i = 0; i < n; ++i) maxnd = std::max(maxnd, nd[i] = ndeps(i));
    if (maxnd > 32) return;
    // processing order inside each group: (level, dependency count, sweep index) --
    // sorting a level's rows by width keeps wide rows together in few steps
    std::vector<int> seq(n), pos(n);
    for (int g = 0; g < K; ++g) {
        int* q = seq.data() + gstart[g];
        const int m = gstart[g + 1] - gstart[g];
        for (int u = 0; u < m; ++u) q[u] = row_of_t(gstart[g] + u);
        std::stable_sort(q, q + m, [&](int x, int y) { return lev[x] != lev[y] ? lev[x] < lev[y] : nd[x] < nd[y]; });
        for (int u = 0; u < m; ++u) pos[q[u]] = u;
    }
    // import lists (previous group's rows, in its processing order) and halo indices
    std::vector<int> hidx(n, -1), gimp_off(K + 1, 0), imp;
    std::vector<char> exported(n, 0);
    int hmax = 0, maxdist = 0;
    for (int g = 0; g < K; ++g) {
        gimp_off[g] = int(imp.size());
        std::vector<int> need;
        for (int u = gstart[g]; u < gstart[g + 1]; ++u) {
            const int i = seq[u];
            for (int k = rp[i]; k < rp[i + 1]; ++k) {
                const int j = ci[k];
                if (!is_dep(i, j)) continue;
                if (gid[j] == g)
                    maxdist = std::max(maxdist, pos[i] - pos[j]);
                else if (!exported[j]) {
                    exported[j] = 1;
                    need.push_back(j);
                }
            }
        }
        std::sort(need.begin(), need.end(), [&](int x, int y) { return pos[x] < pos[y]; });
        for (size_t q = 0; q < need.size(); ++q) hidx[need[q]] = int(q);
        imp.insert(imp.end(), need.begin(), need.end());
        hmax = std::max(hmax, int(need.size()));
    }
    gimp_off[K] = int(imp.size());
    int W = 64;
    while (W < maxdist + 32) W <<= 1;
    int ns = 0;
    for (int t = kLsMaxNS; t >= 2; t /= 2)
        if (ls_smem_bytes(W, hmax, t) <= 225 * 1024) {
            ns = t;
            break;
        }
    if (ns == 0) return;
    // programs: one dependency class for the whole level (kernel template)
    int cls = 0;
    while (ls_nd(cls) < maxnd) ++cls;
    // variable-width records (k_gs_lsv) for wide levels unless fixed-class forced
    const bool var0 = rec_mode == 2 || (rec_mode == 0 && maxnd > kLsVarMin);
    // lane groups: when most rows fit a smaller class (coarse RS levels: 92-95 %
    // of the rows have <= 8 of up to 15-19 dependencies) the records use that
    // class and each wider row takes TWO or FOUR lanes (dependencies 0..ND-1,
    // ND..2ND-1, ..., summed by xor shuffles).  Quads occupy the first lanes of a
    // step, then pairs, then single rows, so a level still needs one step per 32
    // lanes; this also replaces the variable-width records on levels whose widest
    // row has 17-32 dependencies.  MPREC_LS_PAIRS=0: off.
    const bool pairs_on = [] {  // read per build (tests toggle it)
        const char* e = getenv("MPREC_LS_PAIRS");
        return !(e && e[0] == '0');
    }();
    bool pair = false;
    if (pairs_on && rec_mode == 0 && maxnd > 4) {
        const int cmax = var0 ? 4 : cls;
        for (int c2 = 1; c2 < cmax && !pair; ++c2) {
            if (maxnd > 4 * ls_nd(c2)) continue;
            int wide = 0;
            for (int i = 0; i < n; ++i) wide += nd[i] > ls_nd(c2) ? 1 : 0;
            if (wide * 4 < n) {
                pair = true;
                cls = c2;
            }
        }
    }
    const bool var = var0 && !pair;
    if (var) cls = kLsVar;
    const int trash_slot = W + 1 + hmax;
    std::vector<char> prog;
    std::vector<int2> gch(K);
    std::vector<long long> coff(n);
    int64_t nchunks = 0, nsteps_total = 0;
    for (int g = 0; g < K; ++g) {
        gch[g].x = int(nchunks);
        const int m = gstart[g + 1] - gstart[g];
        const int* q = seq.data() + gstart[g];
        int64_t cbase = 0;
        int off = kLsCH;
        for (int u = 0; u < m;) {
            const int L = lev[q[u]];
            int cnt = 0, nd4 = 1;
            if (var) {
                while (u + cnt < m && cnt < 32 && lev[q[u + cnt]] == L) {
                    const int n4 = std::max(nd4, (nd[q[u + cnt]] + 3) / 4);
                    if (16 + (cnt + 1) * ls_rsv(n4) > kLsCH - 16) break;
                    nd4 = n4;
                    ++cnt;
                }
            } else if (!pair) {
                while (u + cnt < m && cnt < 32 && lev[q[u + cnt]] == L && 16 + (cnt + 1) * ls_rs(cls) <= kLsCH - 16)
                    ++cnt;
            }
            // grouped steps: rows of the level in order until 32 lanes (1, 2 or 4 per row)
            int npair = 0, nquad = 0, lanes = cnt;
            std::vector<int> lane_row, lane_half;
            if (pair) {
                auto lanes_of = [&](int i) { return nd[i] <= ls_nd(cls) ? 1 : nd[i] <= 2 * ls_nd(cls) ? 2 : 4; };
                lanes = 0;
                while (u + cnt < m && lev[q[u + cnt]] == L) {
                    const int nl = lanes_of(q[u + cnt]);
                    // (quads first, then pairs: both stay aligned without padding)
                    if (lanes + nl > 32 || 16 + (lanes + nl) * ls_rs(cls) > kLsCH - 16) break;
                    lanes += nl;
                    nquad += nl == 4;
                    npair += nl == 2;
                    ++cnt;
                }
                // lane layout: quads, then pairs, then single rows
                for (int want : {4, 2, 1})
                    for (int r = 0; r < cnt; ++r)
                        if (lanes_of(q[u + r]) == want)
                            for (int hh = 0; hh < want; ++hh) {
                                lane_row.push_back(r);
                                lane_half.push_back(hh);
                            }
                lanes = int(lane_row.size());
            }
            const int RS = var ? ls_rsv(nd4) : ls_rs(cls), ND = var ? 4 * nd4 : ls_nd(cls), bytes = 16 + lanes * RS;
            if (off + bytes > kLsCH) {
                cbase = nchunks * int64_t(kLsCH);
                prog.resize(size_t(cbase + kLsCH), 0);
                ++nchunks;
                off = 16;
            }
            char* base = prog.data() + cbase + off;
            int need = 0;
            for (int ln = 0; ln < lanes; ++ln) {
                const int r = pair ? lane_row[ln] : ln, half = pair ? lane_half[ln] : 0;
                const int i = q[u + r];
                char* rec = base + 16 + ln * RS;
                int* sl0 = reinterpret_cast<int*>(rec);
                double* cp = reinterpret_cast<double*>(rec + 16);
                int* rsl = reinterpret_cast<int*>(rec + 24);
                double* ep0 = reinterpret_cast<double*>(rec + 32);
                int* sl1 = reinterpret_cast<int*>(rec + 32 + 8 * ND);
                auto slot = [&](int d) -> int& {
                    if (d < 4) return sl0[d];
                    if (var) return reinterpret_cast<int*>(rec + 64 + 48 * (d / 4 - 1))[d % 4];
                    return sl1[d - 4];
                };
                auto coef = [&](int d) -> double& {
                    if (var && d >= 4) return reinterpret_cast<double*>(rec + 64 + 48 * (d / 4 - 1) + 16)[d % 4];
                    return ep0[d];
                };
                *cp = 0.0;
                if (half == 0) {  // first lane of the row's group
                    rsl[0] = i;
                    rsl[1] = (pos[i] & (W - 1)) | (exported[i] ? kLsExportBit : 0);
                    coff[i] = (cbase + off + 16 + ln * RS + 16) | (exported[i] ? 1 : 0);
                } else {  // further lanes of a pair / quad: c' = 0, no store
                    rsl[0] = -1;
                    rsl[1] = trash_slot;
                }
                for (int d = 0; d < std::max(ND, 4); ++d) {
                    if (d < ND) coef(d) = 0.0;
                    if (d < 4 || d < ND) slot(d) = W;
                }
                int d = 0, dd = 0;
                for (int k = rp[i]; k < rp[i + 1]; ++k) {
                    const int j = ci[k];
                    if (!is_dep(i, j)) continue;
                    if (dd++ / ND != half) continue;  // another lane of the row's group
                    coef(d) = v[k] * invd[i];
                    if (gid[j] == g) {
                        slot(d) = pos[j] & (W - 1);
                    } else {
                        slot(d) = W + 1 + hidx[j];
                        need = std::max(need, hidx[j] + 1);
                    }
                    ++d;
                }
            }
            const int hdr[4] = {lanes, var ? nd4 : (cls | (npair << 8) | (nquad << 16)), need, bytes};
            std::memcpy(base, hdr, 16);
            *reinterpret_cast<int*>(prog.data() + cbase) += 1;
            off += bytes;
            u += cnt;
            ++nsteps_total;
        }
        gch[g].y = int(nchunks - gch[g].x);
    }
    std::vector<int2> gimp(K);
    for (int g = 0; g < K; ++g) gimp[g] = make_int2(gimp_off[g], gimp_off[g + 1] - gimp_off[g]);
    out.prog = std::move(prog);
    out.gch = std::move(gch);
    out.gimp = std::move(gimp);
    out.imp = std::move(imp);
    out.coff = std::move(coff);
    out.K = K;
    out.W = W;
    out.hmax = hmax;
    out.dir = dir;
    out.nsteps = int(nsteps_total);
    out.nchunks = int(nchunks);
    out.maxdist = maxdist;
    out.nd = maxnd;
    out.ns = ns;
    out.cls = cls;
    out.ok = true;
}

static void ls_upload(Ctx& c, LsBuilt& b, LsSched& s) {
    s = LsSched();
    if (!b.ok) return;
    s.prog.upload(b.prog.data(), b.prog.size(), c.s);
    s.gch.upload(b.gch.data(), b.K, c.s);
    s.imp.alloc(std::max<size_t>(b.imp.size(), 1));
    if (!b.imp.empty()) s.imp.upload(b.imp.data(), b.imp.size(), c.s);
    s.gimp.upload(b.gimp.data(), b.K, c.s);
    s.coff.upload(b.coff.data(), b.coff.size(), c.s);
    c.sync();
    s.K = b.K;
    s.W = b.W;
    s.hmax = b.hmax;
    s.dir = b.dir;
    s.nsteps = b.nsteps;
    s.nchunks = b.nchunks;
    s.maxdist = b.maxdist;
    s.nd = b.nd;
    s.ns = b.ns;
    s.cls = b.cls;
    s.smem = ls_smem_bytes(b.W, b.hmax, b.ns);
    s.ok = true;
}

// Host copy of a level: one download serves both sweep directions.
struct LsHost {
    int n = 0;
    std::vector<int> rp, ci, levf, levb;
    std::vector<double> v, invd;
};
static void ls_download(Ctx& c, const CsrView& a, const double* invd_dev, const int* glev_f, const int* glev_b,
                        LsHost& h) {
    const int n = a.n;
    h.n = n;
    h.rp.resize(n + 1);
    h.ci.resize(a.nnz);
    h.v.resize(a.nnz);
    h.invd.resize(n);
    MG_CUDA(cudaMemcpyAsync(h.rp.data(), a.rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, c.s));
    MG_CUDA(cudaMemcpyAsync(h.ci.data(), a.ci, sizeof(int) * a.nnz, cudaMemcpyDeviceToHost, c.s));
    MG_CUDA(cudaMemcpyAsync(h.v.data(), a.v, sizeof(double) * a.nnz, cudaMemcpyDeviceToHost, c.s));
    MG_CUDA(cudaMemcpyAsync(h.invd.data(), invd_dev, sizeof(double) * n, cudaMemcpyDeviceToHost, c.s));
    if (glev_f) {
        h.levf.resize(n);
        MG_CUDA(cudaMemcpyAsync(h.levf.data(), glev_f, sizeof(int) * n, cudaMemcpyDeviceToHost, c.s));
    }
    if (glev_b) {
        h.levb.resize(n);
        MG_CUDA(cudaMemcpyAsync(h.levb.data(), glev_b, sizeof(int) * n, cudaMemcpyDeviceToHost, c.s));
    }
    c.sync();
}

bool build_ls_sched(Ctx& c, const CsrView& a, const double* invd_dev, int dir, const int* glev_dev, int K,
                    LsSched& s, int rec_mode) {
    s = LsSched();
    if (a.n < 64) return false;
    LsHost h;
    ls_download(c, a, invd_dev, dir > 0 ? glev_dev : nullptr, dir > 0 ? nullptr : glev_dev, h);
    LsBuilt b;
    ls_build_host(h.rp, h.ci, h.v, dir > 0 ? h.levf : h.levb, h.invd, h.n, dir, K, rec_mode, b);
    ls_upload(c, b, s);
    s.rec_mode = rec_mode;
    return s.ok;
}

// Both directions from one download, the two host builds on two threads.
bool build_ls_pair(Ctx& c, const CsrView& a, const double* invd_dev, const int* glev_f, const int* glev_b, int K,
                   int rec_mode, LsSched& f, LsSched& bw) {
    f = LsSched();
    bw = LsSched();
    if (a.n < 64) return false;
    LsHost h;
    ls_download(c, a, invd_dev, glev_f, glev_b, h);
    LsBuilt bf, bb;
    std::thread t([&] { ls_build_host(h.rp, h.ci, h.v, h.levb, h.invd, h.n, -1, K, rec_mode, bb); });
    ls_build_host(h.rp, h.ci, h.v, h.levf, h.invd, h.n, +1, K, rec_mode, bf);
    t.join();
    if (!bf.ok || !bb.ok) return false;
    ls_upload(c, bf, f);
    ls_upload(c, bb, bw);
    f.rec_mode = bw.rec_mode = rec_mode;
    return true;
}

long long* g_ls_stats = nullptr;  // diagnostics: per-group {start, end, wait ns, waits}

template <int ND>
static void launch_ls(Ctx& c, const LsSched& s, double* xnew) {
    static bool attr = false;
    static int max_clusters = -1;
    if (!attr) {
        MG_CUDA(cudaFuncSetAttribute(k_gs_ls<ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        attr = true;
    }
    // clusters of two thread blocks (DSMEM push across every other group boundary)
    // when all K/2 clusters fit on the device at once.  Opt-in (MPREC_LS_PUSH=1):
    // measured slower at c5 (level 0: 0.77 vs 0.59 ms; the per-step ballot and
    // remote store slow the pushing groups more than the halved boundary
    // latency saves), DESIGN.md §5.1
    static const bool push_on = [] {
        const char* e = getenv("MPREC_LS_PUSH");
        return e && e[0] == '1';
    }();
    bool push = push_on && (s.K % 2 == 0);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(s.K);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = s.smem;
    cfg.stream = c.s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (push) {
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_gs_ls<ND>, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        push = n >= s.K / 2;
    }
    if (!push) cfg.numAttrs = 0;
    MG_CUDA(cudaLaunchKernelEx(&cfg, k_gs_ls<ND>, (const char*)s.prog.p, (const int2*)s.gch.p, (const int*)s.imp.p,
                               (const int2*)s.gimp.p, xnew, s.W, s.W + 1 + s.hmax, s.ns, g_ls_stats, push ? 1 : 0));
    (void)max_clusters;
}

void gs_sweep_ls(Ctx& c, const CsrView& a, const double* invd, const double* b, const double* xold, double* xnew,
                 bool xold_zero, const LsSched& s) {
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 4.0 * a.n + 24.0 * a.n;
    {
        Ctx::Scope sc(&c, MPREC_K_GS, bytes);
        k_ls_pre<<<(a.n + 255) / 256, 256, 0, c.s>>>(a.n, a.rp, a.ci, a.v, a.diag, invd, b, xold_zero ? nullptr : xold,
                                                    s.dir, s.coff.p, s.prog.p, xnew);
        check_launch("gs ls pre");
        switch (s.cls) {
            case kLsVar: {
                static bool attr = false;
                if (!attr) {
                    MG_CUDA(cudaFuncSetAttribute(k_gs_lsv, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
                    attr = true;
                }
                k_gs_lsv<<<s.K, kThreads, s.smem, c.s>>>(s.prog.p, s.gch.p, s.imp.p, s.gimp.p, xnew, s.W,
                                                         s.W + 1 + s.hmax, s.ns);
                break;
            }
            case 0: launch_ls<2>(c, s, xnew); break;
            case 1: launch_ls<4>(c, s, xnew); break;
            case 2: launch_ls<8>(c, s, xnew); break;
            case 3: launch_ls<16>(c, s, xnew); break;
            default: launch_ls<32>(c, s, xnew); break;
        }
        check_launch("gs ls sweep");
    }
}

void gs_level_sweep(Ctx& c, AmgLevel& L, const double* r, const double* xold, double* xnew, int dir, bool zero);

// Diagnostics: build the level-synchronous programs with K groups on level l,
// time them against the level's current sweep kernel and compare the results.
// out[0..9] = ms fwd ls, ms bwd ls, ms fwd cur, ms bwd cur, rel err fwd, rel err bwd,
//             W, hmax, steps fwd, build ok (1/0)
void gs_ls_experiment(Ctx& c, Amg& amg, int l, int K, int reps, double* out) {
    AmgLevel& L = *amg.lv[l];
    for (int q = 0; q < 10; ++q) out[q] = 0.0;
    LsSched sf, sb;
    const int rm = getenv("MPREC_LS_REC") ? atoi(getenv("MPREC_LS_REC")) : 0;
    const bool okf = build_ls_sched(c, L.a, L.invd.p, +1, L.glev_f, K, sf, rm);
    const bool okb = okf && build_ls_sched(c, L.a, L.invd.p, -1, L.glev_b, K, sb, rm);
    out[9] = (okf && okb) ? 1.0 : 0.0;
    if (!okf || !okb) return;
    out[6] = sf.W;
    out[7] = sf.hmax;
    out[8] = sf.nsteps + 1e6 * sf.nd + 1e8 * sf.ns;
    const int n = L.n;
    DBuf<double> bb(n), y1(n), y2(n), xf(n), xb(n);
    k_ls_testvec<<<(n + 255) / 256, 256, 0, c.s>>>(bb.p, n);
    cudaEvent_t e[6];
    for (auto& x : e) cudaEventCreate(&x);
    float t[4] = {0, 0, 0, 0};
    for (int r = 0; r < reps; ++r) {
        fill_pending(c, xf.p, n);
        fill_pending(c, xb.p, n);
        cudaEventRecord(e[0], c.s);
        gs_level_sweep(c, L, bb.p, nullptr, xf.p, +1, true);
        cudaEventRecord(e[1], c.s);
        gs_level_sweep(c, L, bb.p, xf.p, xb.p, -1, false);
        cudaEventRecord(e[2], c.s);
        gs_sweep_ls(c, L.a, L.invd.p, bb.p, nullptr, y1.p, true, sf);
        cudaEventRecord(e[3], c.s);
        gs_sweep_ls(c, L.a, L.invd.p, bb.p, xf.p, y2.p, false, sb);
        cudaEventRecord(e[4], c.s);
        MG_CUDA(cudaEventSynchronize(e[4]));
        float a0, a1, a2, a3;
        cudaEventElapsedTime(&a0, e[0], e[1]);
        cudaEventElapsedTime(&a1, e[1], e[2]);
        cudaEventElapsedTime(&a2, e[2], e[3]);
        cudaEventElapsedTime(&a3, e[3], e[4]);
        if (r > 0 || reps == 1) {
            t[0] += a2;
            t[1] += a3;
            t[2] += a0;
            t[3] += a1;
        }
    }
    const int cntr = reps > 1 ? reps - 1 : 1;
    out[0] = t[0] / cntr;
    out[1] = t[1] / cntr;
    out[2] = t[2] / cntr;
    out[3] = t[3] / cntr;
    if (getenv("MPREC_LS_STATS")) {
        DBuf<long long> st(4 * sf.K);
        g_ls_stats = st.p;
        gs_sweep_ls(c, L.a, L.invd.p, bb.p, nullptr, y1.p, true, sf);
        c.sync();
        g_ls_stats = nullptr;
        auto h = st.to_host(c.s);
        std::vector<int2> gch(sf.K);
        sf.gch.download(gch.data(), sf.K, c.s);
        c.sync();
        long long t0 = h[0];
        for (int g = 0; g < sf.K; ++g) t0 = std::min(t0, h[4 * g]);
        fprintf(stderr, "[ls stats] level n=%d K=%d (group: start end wait_us waits chunks)\n", n, sf.K);
        const int every = atoi(getenv("MPREC_LS_STATS")) >= 2 ? 1 : std::max(1, sf.K / 12);
        for (int g = 0; g < sf.K; g += every)
            fprintf(stderr, "  g%3d: %8.1f %8.1f %8.1f %6lld %5d\n", g, (h[4 * g] - t0) * 1e-3, (h[4 * g + 1] - t0) * 1e-3,
                    h[4 * g + 2] * 1e-3, h[4 * g + 3], gch[g].y);
    }
    auto h1 = y1.to_host(c.s), h2 = y2.to_host(c.s), hf = xf.to_host(c.s), hb = xb.to_host(c.s);
    double n1 = 0, d1 = 0, n2 = 0, d2 = 0;
    for (int i = 0; i < n; ++i) {
        n1 = std::max(n1, std::abs(h1[i] - hf[i]));
        d1 = std::max(d1, std::abs(hf[i]));
        n2 = std::max(n2, std::abs(h2[i] - hb[i]));
        d2 = std::max(d2, std::abs(hb[i]));
    }
    out[4] = (std::isnan(n1) ? 1e300 : n1) / std::max(d1, 1e-300);
    out[5] = (std::isnan(n2) ? 1e300 : n2) / std::max(d2, 1e-300);
    for (auto& x : e) cudaEventDestroy(x);
}

}  // namespace mg
