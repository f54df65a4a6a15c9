// gs_cluster.cu -- Gauss-Seidel sweep of a whole AMG level inside ONE thread
// block cluster (K14), for levels whose iterate fits the
// cluster's distributed shared memory (16 CTAs x ~200 KB on B200).
//
// Same natural-order semantics and per-row arithmetic as k_gs (warp per row,
// amg.cpp:25-43).  CTA q of the cluster owns rows [q*R, (q+1)*R) and keeps
// their new values in its shared memory (kPending sentinel); its warps claim
// the owned rows in DAG-level order from a shared-memory counter.  A row's
// dependencies are polled in the owner CTA's shared memory: locally (~40
// cycles) or through DSMEM (~215 cycles, B300_MICROARCH.md) instead of an L2
// round trip (~380 ns one way, scripts/micro/hop.cu).  Results also go to
// global memory for the next operation.  Deadlock freedom: every CTA claims in
// level order and all CTAs of a cluster are co-resident, so the lowest
// unfinished level always progresses.
#include <cooperative_groups.h>

#include "mprec.cuh"

namespace cg = cooperative_groups;

namespace mg {
namespace {

constexpr int kClThreads = 1024;

__device__ __forceinline__ void st_pub_cl(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}

// one row's operands, loaded ahead of time (first 32 entries in registers)
struct RowPre {
    int i = -1, k0 = 0, k1 = 0, j = 0;
    double bi = 0.0, dii = 0.0, a = 0.0, xo = 0.0;
};

template <int DIR>
__device__ __forceinline__ RowPre prefetch_row(int t, int nr, int r0, const int* __restrict__ border,
                                               const int* __restrict__ rp, const int* __restrict__ ci,
                                               const double* __restrict__ v, const double* __restrict__ invd,
                                               const double* __restrict__ b, const double* __restrict__ xold,
                                               int lane) {
    RowPre p;
    if (t >= nr) return p;
    p.i = __ldg(border + r0 + t);
    p.k0 = __ldg(rp + p.i);
    p.k1 = __ldg(rp + p.i + 1);
    p.bi = __ldg(b + p.i);
    p.dii = __ldg(invd + p.i);
    const int k = p.k0 + lane;
    p.j = k < p.k1 ? __ldg(ci + k) : p.i;
    p.a = (k < p.k1 && p.j != p.i) ? __ldg(v + k) : 0.0;
    const bool dep = DIR > 0 ? (p.j < p.i) : (p.j > p.i);
    if (k < p.k1 && p.j != p.i && !dep && xold) p.xo = __ldg(xold + p.j);
    return p;
}

template <int DIR>
__global__ void __launch_bounds__(kClThreads, 1) k_gs_cluster(const int* __restrict__ rp, const int* __restrict__ ci,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ invd,
                                                             const double* __restrict__ b,
                                                             const double* __restrict__ xold, double* xnew,
                                                             const int* __restrict__ border, int n, int R) {
    extern __shared__ unsigned long long xs[];
    __shared__ int claim;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned q = cl.block_rank();
    const int lane = threadIdx.x & 31;
    const int r0 = int(q) * R, r1 = min(n, r0 + R), nr = max(0, r1 - r0);
    for (int t = threadIdx.x; t < R; t += blockDim.x) xs[t] = kPending;
    if (threadIdx.x == 0) claim = 0;
    cl.sync();  // every CTA's slice initialised before anyone polls it
    // software pipeline: the next row's operands are in flight while this row waits
    int t = 0;
    if (lane == 0) t = atomicAdd(&claim, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    RowPre cur = prefetch_row<DIR>(t, nr, r0, border, rp, ci, v, invd, b, xold, lane);
    while (cur.i >= 0) {
        if (lane == 0) t = atomicAdd(&claim, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        const RowPre nxt = prefetch_row<DIR>(t, nr, r0, border, rp, ci, v, invd, b, xold, lane);
        const int i = cur.i;
        double acc = 0.0;
        for (int base = cur.k0; base < cur.k1; base += 32) {
            const int k = base + lane;
            const bool valid = k < cur.k1;
            int j;
            double a, xj = 0.0;
            if (base == cur.k0) {
                j = cur.j;
                a = cur.a;
                xj = cur.xo;
            } else {
                j = valid ? __ldg(ci + k) : i;
                a = (valid && j != i) ? __ldg(v + k) : 0.0;
            }
            const bool off = valid && j != i;
            const bool dep = off && (DIR > 0 ? (j < i) : (j > i));
            if (base != cur.k0 && off && !dep && xold) xj = __ldg(xold + j);
            volatile unsigned long long* src = nullptr;
            if (dep) {
                const unsigned owner = unsigned(j / R);
                src = cl.map_shared_rank(xs, owner) + (j - int(owner) * R);
            }
            unsigned long long raw = dep ? *src : 0ull;
            bool pend = dep && raw == kPending;
            while (__any_sync(0xffffffffu, pend)) {
                if (pend) {
                    raw = *src;
                    pend = raw == kPending;
                }
            }
            if (dep) xj = __longlong_as_double((long long)raw);
            acc += a * xj;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            const double xi = (cur.bi - acc) * cur.dii;
            reinterpret_cast<volatile double*>(xs)[i - r0] = xi;
            st_pub_cl(xnew + i, xi);
        }
        cur = nxt;
    }
    cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

}  // namespace

// smallest cluster (1, 2, 4, 8, 16 CTAs) whose shared memory holds the level's
// iterate, or 0 when none does; `min_cs` asks for at least that many CTAs
int gs_cluster_plan(int n, int* rows_per_cta, int min_cs) {
    const int max_rows = (200 * 1024) / int(sizeof(double));
    for (int cs : {1, 2, 4, 8, 16}) {
        if (cs < min_cs) continue;
        const int r = (n + cs - 1) / cs;
        if (r <= max_rows) {
            *rows_per_cta = r;
            return cs;
        }
    }
    return 0;
}

void gs_sweep_cluster(Ctx& c, const CsrView& a, const double* invd, const double* b, const double* xold, double* xnew,
                      int dir, bool xold_zero, const int* border, int csize, int R) {
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 4.0 * a.n + 24.0 * a.n;
    Ctx::Scope sc(&c, MPREC_K_GS, bytes);
    static bool attr = false;
    if (!attr) {
        for (auto fn : {k_gs_cluster<1>, k_gs_cluster<-1>}) {
            MG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            MG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize, 1, 1);
    cfg.blockDim = dim3(kClThreads, 1, 1);
    cfg.dynamicSmemBytes = size_t(R) * sizeof(double);
    cfg.stream = c.s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const double* xo = xold_zero ? nullptr : xold;
    if (dir > 0)
        MG_CUDA(cudaLaunchKernelEx(&cfg, k_gs_cluster<1>, a.rp, a.ci, a.v, invd, b, xo, xnew, border, a.n, R));
    else
        MG_CUDA(cudaLaunchKernelEx(&cfg, k_gs_cluster<-1>, a.rp, a.ci, a.v, invd, b, xo, xnew, border, a.n, R));
    check_launch("gs_sweep_cluster");
}

}  // namespace mg
