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
#include <algorithm>
#include <cstdlib>

#include "mprec.cuh"

namespace mg {

void ilu_factor_run(Ctx& c, const BsrView& lu, DBuf<int>& flags, Pattern* pat);

namespace {

__device__ __forceinline__ unsigned long long ld_relaxed(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_pub(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}

constexpr int kWarps = 8;

// ---- nb = 8: lane l -> (row r = l & 7, column pair cq = l >> 3 : c = 2cq, 2cq+1)
template <bool kFwd>
__global__ void __launch_bounds__(kWarps * 32, 4) k_ilu8(const int* __restrict__ rp, const int* __restrict__ ci,
                                                      const int* __restrict__ dpos, const double* __restrict__ val,
                                                      const double* __restrict__ rhs, double* y, int nc,
                                                      const int* __restrict__ order, int* counter,
                                                      const double* __restrict__ dinv, long long* ts = nullptr) {
    const int lane = threadIdx.x & 31;
    const int r = lane & 7, cq = lane >> 3, c0 = cq * 2;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nc) return;
        const int I = __ldg(order + t);
        MG_DCHECK(I >= 0 && I < nc);
        const int d = dpos[I];
        const int ka = kFwd ? rp[I] : d + 1;
        const int kb = kFwd ? d : rp[I + 1];
        MG_DCHECK(ka <= kb && (kb - ka) <= 64);
        // row r of the packed inverse diagonal block (strict lower: inv(L_II),
        // upper incl. diagonal: inv(U_II)) -- independent of the chain
        const double* bd = dinv + (int64_t)I * 64;
        double drow[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) drow[c] = __ldg(bd + c * 8 + r);
        // also off the chain: the polls below are volatile asm with a memory
        // clobber, so a load written after them could not be hoisted
        const double rhs_r = rhs[(int64_t)I * 8 + r];
        double acc = 0.0;
        // dependency blocks in groups of 2 (64 registers, 4 CTAs/SM): block values first, then ALL polls
        // issued together, then a warp-convergent re-poll of the pending ones
        for (int kk = ka; kk < kb; kk += 2) {
            double va[2][2];
            unsigned long long raw[2][2];
            int K[2];
            bool pend[2][2];
            bool any = false;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const bool ok = kk + u < kb;
                K[u] = ok ? __ldg(ci + kk + u) : 0;
                const double* bk = val + (int64_t)(ok ? kk + u : ka) * 64;
                va[u][0] = ok ? __ldg(bk + c0 * 8 + r) : 0.0;
                va[u][1] = ok ? __ldg(bk + (c0 + 1) * 8 + r) : 0.0;
                pend[u][0] = pend[u][1] = ok;
            }
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    raw[u][h] = pend[u][h] ? ld_relaxed(y + (int64_t)K[u] * 8 + c0 + h) : 0ull;
                    pend[u][h] = pend[u][h] && raw[u][h] == kPending;
                    any |= pend[u][h];
                }
            while (__any_sync(0xffffffffu, any)) {
                any = false;
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if (pend[u][h]) {
                            raw[u][h] = ld_relaxed(y + (int64_t)K[u] * 8 + c0 + h);
                            pend[u][h] = raw[u][h] == kPending;
                            any |= pend[u][h];
                        }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u)
                acc += va[u][0] * __longlong_as_double((long long)raw[u][0]) +
                       va[u][1] * __longlong_as_double((long long)raw[u][1]);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 8);
        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
        const double v = rhs_r - acc;
        // y_I = inv(L_II) v (forward) or inv(U_II) v (backward): 8 independent
        // shuffles + FMAs instead of an 8-step serial substitution
        double yv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) yv[c] = __shfl_sync(0xffffffffu, v, c);
        double out = kFwd ? v : 0.0;  // y_r itself (a dynamic yv[r] would live in local memory)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (kFwd ? (c < r) : (c >= r)) out += drow[c] * yv[c];
        }
        const double v_out = out;
        if (lane < 8) st_pub(y + (int64_t)I * 8 + r, v_out);
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
        const double rhs_l = lane < nb ? rhs[(int64_t)I * nb + lane] : 0.0;  // before the polls
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
        double v = lane < nb ? rhs_l - acc : 0.0;
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

// packed inverse diagonal blocks: strict lower = inv(unit L_II), upper = inv(U_II)
__global__ void k_ilu_dinv8(const int* __restrict__ dpos, const double* __restrict__ val, int nc, double* dinv) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= nc) return;
    const double* d = val + (int64_t)dpos[I] * 64;
    double m[64], o[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) {
        m[e] = d[e];
        o[e] = 0.0;
    }
    // inv(L) column by column: L unit lower (strict part of m)
    for (int j = 0; j < 8; ++j) {
        double x[8];
        for (int i = 0; i < 8; ++i) x[i] = (i == j) ? 1.0 : 0.0;
        for (int k = 0; k < 8; ++k)
            for (int i = k + 1; i < 8; ++i) x[i] -= m[k * 8 + i] * x[k];
        for (int i = j + 1; i < 8; ++i) o[j * 8 + i] = x[i];
    }
    // inv(U) column by column: U upper incl. diagonal
    for (int j = 0; j < 8; ++j) {
        double x[8];
        for (int i = 0; i < 8; ++i) x[i] = (i == j) ? 1.0 : 0.0;
        for (int k = 7; k >= 0; --k) {
            x[k] /= m[k * 8 + k];
            for (int i = 0; i < k; ++i) x[i] -= m[k * 8 + i] * x[k];
        }
        for (int i = 0; i <= j; ++i) o[j * 8 + i] = x[i];
    }
    double* out = dinv + (int64_t)I * 64;
#pragma unroll
    for (int e = 0; e < 64; ++e) out[e] = o[e];
}

}  // namespace

void Ilu::factor(Ctx& c) {
    ilu_factor_run(c, lu, flags, pat);
    if (lu.nb == 8) {
        dinv.ensure((size_t)lu.nc * 64);
        k_ilu_dinv8<<<(lu.nc + 127) / 128, 128, 0, c.s>>>(lu.dpos, lu.val, lu.nc, dinv.p);
        check_launch("ilu dinv");
        // level-synchronous solve streams (ilu_ls.cu) when the pattern fits them
        // (<= 2 dependency blocks per direction, dependencies within the previous
        // group): MPREC_ILU_LS=<groups> (default 148; 0 = warp-per-block-row kernel)
        const int ls_k = [] {  // read per factorisation (tests toggle it)
            const char* e = getenv("MPREC_ILU_LS");
            return e ? atoi(e) : 148;
        }();
        if (ls_k > 0 && pat && lu.nc >= 4096) {
            if (!ls_fwd.ok) build_ilu_ls(c, *pat, std::min(ls_k, c.sm_count), ls_fwd, ls_bwd);
            if (ls_fwd.ok && ls_bwd.ok) {
                ilu_ls_fill(c, ls_fwd, lu.val, dinv.p);
                ilu_ls_fill(c, ls_bwd, lu.val, dinv.p);
            }
        } else {
            ls_fwd = IluLs();
            ls_bwd = IluLs();
        }
    }
}

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
    if (lu.nb == 8 && ls_fwd.ok && ls_bwd.ok) {
        // algorithmic bytes as for the BSR kernels (factor blocks + vectors); the
        // stream copy of the right-hand side is charged inside the same scope
        {
            Ctx::Scope sc(&c, MPREC_K_ILU_FWD, bytes);
            ilu_ls_solve(c, ls_fwd, true, r, ybuf.p);
        }
        {
            Ctx::Scope sc(&c, MPREC_K_ILU_BWD, bytes);
            ilu_ls_solve(c, ls_bwd, false, ybuf.p, y);
        }
        return;
    }
    {
        Ctx::Scope sc(&c, MPREC_K_ILU_FWD, bytes);
        if (lu.nb == 8)
            k_ilu8<true><<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, r, ybuf.p, lu.nc, of,
                                                          c.counters.p + 2, dinv.p);
        else
            k_ilu_gen<true><<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, r, ybuf.p, lu.nc, lu.nb,
                                                             of, c.counters.p + 2);
        check_launch("ilu_fwd");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_ILU_BWD, bytes);
        if (lu.nb == 8)
            k_ilu8<false><<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, ybuf.p, y, lu.nc, ob,
                                                           c.counters.p + 3, dinv.p);
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
                                                  ilu.lu.nc, ilu.pat->fwd.order.p, c.counters.p + 2, ilu.dinv.p,
                                                  ts_dev);
    check_launch("ilu_timeline");
    c.sync();
}
}  // namespace mg
