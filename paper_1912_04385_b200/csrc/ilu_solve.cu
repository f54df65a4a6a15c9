// ilu_solve.cu -- K6: ILU(0) triangular solves (ILU0Factor::apply, ilu0.cpp:41-59)
// on the block factors, dependency-scheduled (no level-set replacement, no
// colouring): y_i = r_i - sum_{k<i} l_ik y_k, then y_i = (y_i - sum_{k>i} u_ik y_k)/u_ii
// in the reference's natural order semantics.
//
// Sync-free: one warp per block row, claimed in dependency order (ascending for
// the forward sweep, descending for the backward sweep) from an atomic counter.
// Output vectors are pre-filled with the kPending signalling NaN; a consumer
// polls the producer's VALUES directly (ld.relaxed.gpu) -- one L2 round trip
// per dependency hop, no separate flag word.  Block values are loaded before
// the wait so that HBM latency overlaps the dependency chain.
#include "mprec.cuh"

namespace mg {

void ilu_factor_run(Ctx& c, const BsrView& lu, DBuf<int>& flags, Pattern* pat);

namespace {

__device__ __forceinline__ double ld_poll(const double* p) {
    unsigned long long v;
    do {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    } while (v == kPending);
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ void st_pub(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}

constexpr int kWarps = 8;

// ---- nb = 8: lane l -> (row r = l & 7, column pair cq = l >> 3 : c = 2cq, 2cq+1)
template <bool kFwd>
__global__ void __launch_bounds__(kWarps * 32) k_ilu8(const int* __restrict__ rp, const int* __restrict__ ci,
                                                      const int* __restrict__ dpos, const double* __restrict__ val,
                                                      const double* __restrict__ rhs, double* y, int nc,
                                                      const int* __restrict__ order, int* counter,
                                                      long long* ts = nullptr) {
    const int lane = threadIdx.x & 31;
    const int r = lane & 7, cq = lane >> 3, c0 = cq * 2;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nc) return;
        const int I = __ldg(order + t);
        const int d = dpos[I];
        const int ka = kFwd ? rp[I] : d + 1;
        const int kb = kFwd ? d : rp[I + 1];
        // diagonal block row r (all 8 columns) -- independent of the chain
        const double* bd = val + (int64_t)d * 64;
        double drow[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) drow[c] = __ldg(bd + c * 8 + r);
        double acc = 0.0;
        int k = ka;
        for (; k + 2 <= kb; k += 2) {
            const int K0 = __ldg(ci + k), K1 = __ldg(ci + k + 1);
            const double* b0 = val + (int64_t)k * 64;
            const double* b1 = b0 + 64;
            const double v00 = __ldg(b0 + c0 * 8 + r), v01 = __ldg(b0 + (c0 + 1) * 8 + r);
            const double v10 = __ldg(b1 + c0 * 8 + r), v11 = __ldg(b1 + (c0 + 1) * 8 + r);
            const double y00 = ld_poll(y + (int64_t)K0 * 8 + c0), y01 = ld_poll(y + (int64_t)K0 * 8 + c0 + 1);
            const double y10 = ld_poll(y + (int64_t)K1 * 8 + c0), y11 = ld_poll(y + (int64_t)K1 * 8 + c0 + 1);
            acc += v00 * y00 + v01 * y01;
            acc += v10 * y10 + v11 * y11;
        }
        for (; k < kb; ++k) {
            const int K = __ldg(ci + k);
            const double* b0 = val + (int64_t)k * 64;
            const double v0 = __ldg(b0 + c0 * 8 + r), v1 = __ldg(b0 + (c0 + 1) * 8 + r);
            const double y0 = ld_poll(y + (int64_t)K * 8 + c0), y1 = ld_poll(y + (int64_t)K * 8 + c0 + 1);
            acc += v0 * y0 + v1 * y1;
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 8);
        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
        double v = rhs[(int64_t)I * 8 + r] - acc;
        if (kFwd) {
            // unit lower triangular diagonal block
#pragma unroll
            for (int c = 0; c < 7; ++c) {
                const double yc = __shfl_sync(0xffffffffu, v, c);
                if (r > c) v -= drow[c] * yc;
            }
        } else {
#pragma unroll
            for (int c = 7; c >= 0; --c) {
                if (r == c) v = v / drow[c];
                const double yc = __shfl_sync(0xffffffffu, v, c);
                if (r < c) v -= drow[c] * yc;
            }
        }
        if (lane < 8) st_pub(y + (int64_t)I * 8 + r, v);
        if (ts && lane == 0) {
            long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            ts[2 * t] = g;
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            ts[2 * t + 1] = (long long)smid * 1000000 + (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5));
        }
    }
}

// ---- generic nb <= 32: lane r handles scalar row r of the block row
template <bool kFwd>
__global__ void __launch_bounds__(kWarps * 32) k_ilu_gen(const int* __restrict__ rp, const int* __restrict__ ci,
                                                         const int* __restrict__ dpos, const double* __restrict__ val,
                                                         const double* __restrict__ rhs, double* y, int nc, int nb,
                                                         const int* __restrict__ order, int* counter) {
    const int lane = threadIdx.x & 31;
    const int nb2 = nb * nb;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nc) return;
        const int I = __ldg(order + t);
        const int d = dpos[I];
        const int ka = kFwd ? rp[I] : d + 1;
        const int kb = kFwd ? d : rp[I + 1];
        double acc = 0.0;
        for (int k = ka; k < kb; ++k) {
            const int K = __ldg(ci + k);
            const double* b = val + (int64_t)k * nb2;
            // warp-convergent wait (see amg_cycle.cu)
            unsigned long long raw = 0;
            bool pend = lane < nb;
            while (__any_sync(0xffffffffu, pend)) {
                if (pend) {
                    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(raw) : "l"(y + (int64_t)K * nb + lane)
                                 : "memory");
                    pend = raw == kPending;
                }
            }
            const double yk = lane < nb ? __longlong_as_double((long long)raw) : 0.0;
            for (int c = 0; c < nb; ++c) {
                const double yc = __shfl_sync(0xffffffffu, yk, c);
                if (lane < nb) acc += __ldg(b + c * nb + lane) * yc;
            }
        }
        const double* bd = val + (int64_t)d * nb2;
        double v = lane < nb ? rhs[(int64_t)I * nb + lane] - acc : 0.0;
        if (kFwd) {
            for (int c = 0; c < nb - 1; ++c) {
                const double yc = __shfl_sync(0xffffffffu, v, c);
                if (lane > c && lane < nb) v -= __ldg(bd + c * nb + lane) * yc;
            }
        } else {
            for (int c = nb - 1; c >= 0; --c) {
                if (lane == c) v = v / __ldg(bd + c * nb + c);
                const double yc = __shfl_sync(0xffffffffu, v, c);
                if (lane < c) v -= __ldg(bd + c * nb + lane) * yc;
            }
        }
        if (lane < nb) st_pub(y + (int64_t)I * nb + lane, v);
    }
}

}  // namespace

void Ilu::factor(Ctx& c) { ilu_factor_run(c, lu, flags, pat); }

void Ilu::apply(Ctx& c, const double* r, double* y) {
    const int64_t nn = (int64_t)lu.nc * lu.nb;
    pat->ensure_sched(c);
    const int* of = pat->fwd.order.p;
    const int* ob = pat->bwd.order.p;
    ybuf.ensure(nn);
    // both sweep outputs start as "pending"
    fill_pending(c, ybuf.p, nn);
    fill_pending(c, y, nn);
    MG_CUDA(cudaMemsetAsync(c.counters.p + 2, 0, sizeof(int) * 2, c.s));
    const int blocks = std::max(1, std::min((lu.nc + kWarps - 1) / kWarps, c.sm_count * 8));
    const double nb2 = double(lu.nb) * lu.nb;
    // forward reads the lower + diagonal blocks, backward the upper + diagonal blocks
    const double lower_blocks = double(lu.nnzb - lu.nc) / 2 + lu.nc;
    const double bytes = lower_blocks * (8.0 * nb2 + 4.0) + 4.0 * (lu.nc + 1) + 16.0 * nn;
    if (lu.nb > 32) throw Error(MPREC_DIMENSION, "nb > 32 not supported by the ILU solve");
    {
        Ctx::Scope sc(&c, MPREC_K_ILU_FWD, bytes);
        if (lu.nb == 8)
            k_ilu8<true><<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, r, ybuf.p, lu.nc, of,
                                                          c.counters.p + 2);
        else
            k_ilu_gen<true><<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, r, ybuf.p, lu.nc, lu.nb,
                                                             of, c.counters.p + 2);
        check_launch("ilu_fwd");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_ILU_BWD, bytes);
        if (lu.nb == 8)
            k_ilu8<false><<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, ybuf.p, y, lu.nc, ob,
                                                           c.counters.p + 3);
        else
            k_ilu_gen<false><<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, ybuf.p, y, lu.nc,
                                                              lu.nb, ob, c.counters.p + 3);
        check_launch("ilu_bwd");
    }
}

}  // namespace mg

namespace mg {
// Diagnostics: one forward ILU sweep recording (globaltimer, sm*1e6+warp) per claimed slot.
void ilu_timeline(Ctx& c, Ilu& ilu, const double* r, double* y, long long* ts_dev, int blocks) {
    const int64_t nn = (int64_t)ilu.lu.nc * ilu.lu.nb;
    ilu.pat->ensure_sched(c);
    ilu.ybuf.ensure(nn);
    fill_pending(c, ilu.ybuf.p, nn);
    MG_CUDA(cudaMemsetAsync(c.counters.p + 2, 0, sizeof(int), c.s));
    if (ilu.lu.nb != 8) throw Error(MPREC_DIMENSION, "timeline diagnostics need nb = 8");
    if (blocks <= 0) blocks = std::max(1, std::min((ilu.lu.nc + kWarps - 1) / kWarps, c.sm_count * 8));
    k_ilu8<true><<<blocks, kWarps * 32, 0, c.s>>>(ilu.lu.rp, ilu.lu.ci, ilu.lu.dpos, ilu.lu.val, r, ilu.ybuf.p,
                                                  ilu.lu.nc, ilu.pat->fwd.order.p, c.counters.p + 2, ts_dev);
    check_launch("ilu_timeline");
    c.sync();
}
}  // namespace mg
