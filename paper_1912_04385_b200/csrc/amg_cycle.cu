// amg_cycle.cu -- the V(1,1)-cycle (AMGHierarchy::cycle/apply, amg.cpp:216-238):
// K14 symmetric Gauss-Seidel sweeps, K15 residual / restriction / prolongation
// (CSR SpMV), K13 coarsest solve as a dense GEMV with the precomputed inverse.
//
// Gauss-Seidel keeps the reference's natural-order semantics
// (sym_gauss_seidel, amg.cpp:25-43): the forward sweep uses updated x_k for
// k < i and previous x_k for k > i, the backward sweep the mirror image.  It is
// dependency-scheduled, not replaced: one warp per row, rows claimed in sweep
// order from an atomic counter, the new iterate is written to a fresh buffer
// pre-filled with the kPending sentinel and consumers poll the producer's value
// (double buffering also makes the "old" reads race-free for any pattern).
#include <cub/cub.cuh>
#include <cstdlib>
#include <string>

#include "mprec.cuh"

namespace mg {
namespace {

__device__ __forceinline__ void st_pub(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}

constexpr int kGsWarps = 8;

__device__ __forceinline__ unsigned long long ld_relaxed(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Warp per row.  The wait is warp-CONVERGENT (every lane stays in one
// __any_sync loop): a divergent spin under independent thread scheduling
// serialises the warp's paths and costs ~100x the hop latency.
template <int DIR>
__global__ void __launch_bounds__(kGsWarps * 32) k_gs(const int* __restrict__ rp, const int* __restrict__ ci,
                                                      const double* __restrict__ v, const int* __restrict__ diag,
                                                      const double* __restrict__ b, const double* __restrict__ xold,
                                                      double* xnew, int n, const int* __restrict__ order,
                                                      int* counter, unsigned sleep_ns, const double* __restrict__ invd) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n) return;
        const int i = __ldg(order + t);
        const int k0 = __ldg(rp + i), k1 = __ldg(rp + i + 1);
        // independent of the dependency chain: issue before waiting
        const double bi = __ldg(b + i);
        const double dii = invd ? __ldg(invd + i) : __ldg(v + __ldg(diag + i));
        double acc = 0.0;
        for (int base = k0; base < k1; base += 32) {
            const int k = base + lane;
            const bool valid = k < k1;
            const int j = valid ? __ldg(ci + k) : i;
            const bool off = valid && j != i;
            const double a = off ? __ldg(v + k) : 0.0;
            const bool dep = off && (DIR > 0 ? (j < i) : (j > i));
            double xj = 0.0;
            if (off && !dep && xold) xj = __ldg(xold + j);
            unsigned long long raw = 0;
            bool pend = dep;
            while (__any_sync(0xffffffffu, pend)) {
                if (pend) {
                    raw = ld_relaxed(xnew + j);
                    pend = raw == kPending;
                }
                if (sleep_ns && __any_sync(0xffffffffu, pend)) __nanosleep(sleep_ns);
            }
            if (dep) xj = __longlong_as_double((long long)raw);
            acc += a * xj;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) st_pub(xnew + i, invd ? (bi - acc) * dii : (bi - acc) / dii);
    }
}

// CTA per band of B consecutive rows (doacross).  The band's new
// iterate lives in shared memory (kPending sentinel), so dependencies inside
// the band are resolved by an on-SM poll instead of an L2 round trip; rows of
// the band are claimed by the CTA's warps in global DAG-level order (`border`)
// and bands are claimed in sweep order, hence deadlock-free.  Row arithmetic
// is identical to k_gs (warp per row).  Chosen per AMG level by a setup-time
// measurement (Amg::setup) against the row-per-warp sweep.
template <int DIR>
__global__ void __launch_bounds__(1024) k_gs_cta(const int* __restrict__ rp, const int* __restrict__ ci,
                                                 const double* __restrict__ v, const double* __restrict__ invd,
                                                 const double* __restrict__ b, const double* __restrict__ xold,
                                                 double* xnew, const int* __restrict__ border, int n, int B,
                                                 int nbands, int* counter) {
    extern __shared__ double xs[];
    __shared__ int band_sh, claim_sh;
    const int lane = threadIdx.x & 31;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const int t = atomicAdd(counter, 1);
            band_sh = DIR > 0 ? t : nbands - 1 - t;
            claim_sh = 0;
            if (t >= nbands) band_sh = -1;
        }
        __syncthreads();
        const int band = band_sh;
        if (band < 0) return;
        const int b0 = band * B, b1 = min(n, b0 + B), nrow = b1 - b0;
        for (int q = threadIdx.x; q < nrow; q += blockDim.x)
            reinterpret_cast<unsigned long long*>(xs)[q] = kPending;
        __syncthreads();
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&claim_sh, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= nrow) break;
            const int i = __ldg(border + b0 + t);
            const int k0 = __ldg(rp + i), k1 = __ldg(rp + i + 1);
            const double bi = __ldg(b + i), dii = __ldg(invd + i);
            double acc = 0.0;
            for (int base = k0; base < k1; base += 32) {
                const int k = base + lane;
                const bool valid = k < k1;
                const int j = valid ? __ldg(ci + k) : i;
                const bool off = valid && j != i;
                const double a = off ? __ldg(v + k) : 0.0;
                const bool dep = off && (DIR > 0 ? (j < i) : (j > i));
                const bool local = dep && j >= b0 && j < b1;
                double xj = 0.0;
                if (off && !dep && xold) xj = __ldg(xold + j);
                unsigned long long raw = 0;
                if (dep && !local) raw = ld_relaxed(xnew + j);
                if (local) raw = reinterpret_cast<volatile unsigned long long*>(xs)[j - b0];
                bool pend = dep && raw == kPending;
                while (__any_sync(0xffffffffu, pend)) {
                    if (pend) {
                        raw = local ? reinterpret_cast<volatile unsigned long long*>(xs)[j - b0] : ld_relaxed(xnew + j);
                        pend = raw == kPending;
                    }
                }
                if (dep) xj = __longlong_as_double((long long)raw);
                acc += a * xj;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) {
                const double xi = (bi - acc) * dii;
                reinterpret_cast<volatile double*>(xs)[i - b0] = xi;
                st_pub(xnew + i, xi);
            }
        }
    }
}

__global__ void k_band_key(const int* lev, int n, int B, unsigned long long* key, int* row) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        key[i] = ((unsigned long long)(i / B) << 32) | (unsigned)lev[i];
        row[i] = i;
    }
}

__global__ void k_invd(const double* v, const int* diag, int n, double* invd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) invd[i] = 1.0 / v[diag[i]];
}

// LN lanes per row (chosen per matrix from its mean row length: short P rows
// and 5-point level-0 rows waste most of 8 lanes); mode 0: y = Ax, 1: y = b - Ax,
// 2: y = y + Ax
template <int LN>
__global__ void __launch_bounds__(256) k_csr(const int* __restrict__ rp, const int* __restrict__ ci,
                                             const double* __restrict__ v, const double* __restrict__ x, double* y,
                                             const double* __restrict__ b, int n, int mode) {
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    const int row = int(g / LN), s = int(g % LN);
    double acc = 0.0;
    if (row < n)
        for (int k = __ldg(rp + row) + s; k < __ldg(rp + row + 1); k += LN)
            acc += __ldg(v + k) * __ldg(x + __ldg(ci + k));
#pragma unroll
    for (int o = 1; o < LN; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (row < n && s == 0) y[row] = mode == 0 ? acc : (mode == 1 ? b[row] - acc : y[row] + acc);
}

// y = M x, M row-major n x n, warp per row
__global__ void __launch_bounds__(256) k_gemv(const double* __restrict__ m, int n, const double* __restrict__ x,
                                              double* y) {
    const int lane = threadIdx.x & 31;
    const int row = int((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (row >= n) return;
    const double* mr = m + (int64_t)row * n;
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc += mr[j] * x[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[row] = acc;
}

}  // namespace

void gs_sweep(Ctx& c, const CsrView& a, const double* b, const double* xold, double* xnew, int dir, bool xold_zero,
              const int* order, const double* invd) {
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 4.0 * a.n + 24.0 * a.n;
    Ctx::Scope sc(&c, MPREC_K_GS, bytes);
    int* ctr = c.counters.p + 4;
    MG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int), c.s));
    static const int blk_per_sm = [] {
        const char* e = getenv("MPREC_GS_BLOCKS_PER_SM");
        return e ? atoi(e) : 8;
    }();
    static const unsigned sleep_ns = [] {
        const char* e = getenv("MPREC_POLL_SLEEP");
        return e ? unsigned(atoi(e)) : 0u;
    }();
    const int blocks = std::max(1, std::min((a.n + kGsWarps - 1) / kGsWarps, c.sm_count * blk_per_sm));
    if (dir > 0)
        k_gs<1><<<blocks, kGsWarps * 32, 0, c.s>>>(a.rp, a.ci, a.v, a.diag, b, xold_zero ? nullptr : xold, xnew, a.n,
                                                   order, ctr, sleep_ns, invd);
    else
        k_gs<-1><<<blocks, kGsWarps * 32, 0, c.s>>>(a.rp, a.ci, a.v, a.diag, b, xold_zero ? nullptr : xold, xnew,
                                                    a.n, order, ctr, sleep_ns, invd);
    check_launch("gs_sweep");
}

// rows of every band of B rows in global DAG-level order
void build_band_order(Ctx& c, int n, const int* lev, int B, DBuf<int>& border) {
    DBuf<unsigned long long> key(n), skey(n);
    DBuf<int> row(n);
    border.alloc(std::max(n, 1));
    k_band_key<<<(n + 255) / 256, 256, 0, c.s>>>(lev, n, B, key.p, row.p);
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, skey.p, row.p, border.p, n, 0, 64, c.s);
    DBuf<char> tmp(bytes + 16);
    cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, skey.p, row.p, border.p, n, 0, 64, c.s);
    check_launch("band order");
    c.sync();
}

void gs_sweep_cta(Ctx& c, const CsrView& a, const double* invd, const double* b, const double* xold, double* xnew,
                  int dir, bool xold_zero, const int* border, int B) {
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 4.0 * a.n + 24.0 * a.n;
    Ctx::Scope sc(&c, MPREC_K_GS, bytes);
    int* ctr = c.counters.p + 7;
    MG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int), c.s));
    const int nbands = (a.n + B - 1) / B;
    const size_t smem = size_t(B) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        MG_CUDA(cudaFuncSetAttribute(k_gs_cta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        MG_CUDA(cudaFuncSetAttribute(k_gs_cta<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    static const int threads = [] {
        const char* e = getenv("MPREC_GS_CTA_THREADS");
        return e ? atoi(e) : 1024;
    }();
    const int grid = std::max(1, std::min(nbands, c.sm_count * std::max(1, 2048 / threads)));
    if (dir > 0)
        k_gs_cta<1><<<grid, threads, smem, c.s>>>(a.rp, a.ci, a.v, invd, b, xold_zero ? nullptr : xold, xnew, border, a.n,
                                              B, nbands, ctr);
    else
        k_gs_cta<-1><<<grid, threads, smem, c.s>>>(a.rp, a.ci, a.v, invd, b, xold_zero ? nullptr : xold, xnew, border,
                                               a.n, B, nbands, ctr);
    check_launch("gs_sweep_cta");
}

void compute_invd(Ctx& c, const CsrView& a, double* invd) {
    k_invd<<<(a.n + 255) / 256, 256, 0, c.s>>>(a.v, a.diag, a.n, invd);
    check_launch("invd");
}

void csr_spmv(Ctx& c, const CsrView& a, const double* x, double* y, const double* b, bool add_to_y, int kclass) {
    if (a.n == 0) return;
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 8.0 * a.m + 8.0 * a.n + ((b || add_to_y) ? 8.0 * a.n : 0.0);
    Ctx::Scope sc(&c, kclass, bytes);
    const int mode = add_to_y ? 2 : (b ? 1 : 0);
    const double per_row = double(a.nnz) / std::max(a.n, 1);
    const int ln = per_row <= 3.0 ? 2 : per_row <= 6.0 ? 4 : per_row <= 12.0 ? 8 : 16;
    const int64_t threads = (int64_t)a.n * ln;
    const int grid = int((threads + 255) / 256);
    switch (ln) {
        case 2: k_csr<2><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, y, b, a.n, mode); break;
        case 4: k_csr<4><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, y, b, a.n, mode); break;
        case 8: k_csr<8><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, y, b, a.n, mode); break;
        default: k_csr<16><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, y, b, a.n, mode); break;
    }
    check_launch("csr_spmv");
}

void dense_gemv(Ctx& c, const double* m, int n, const double* x, double* y) {
    if (n == 0) return;
    Ctx::Scope sc(&c, MPREC_K_COARSE, 8.0 * n * n + 16.0 * n);
    const int64_t threads = (int64_t)n * 32;
    k_gemv<<<int((threads + 255) / 256), 256, 0, c.s>>>(m, n, x, y);
    check_launch("dense_gemv");
}

// one Gauss-Seidel direction on level L: band schedule when available
static void level_sweep(Ctx& c, AmgLevel& L, const double* r, const double* xold, double* xnew, int dir, bool zero) {
    const BandSched& bs = dir > 0 ? L.band_fwd : L.band_bwd;
    const LsSched& ls = dir > 0 ? L.ls_fwd : L.ls_bwd;
    if (ls.ok)
        gs_sweep_ls(c, L.a, L.invd.p, r, xold, xnew, zero, ls);
    else if (bs.ok)
        gs_band_sweep(c, bs, L.a.nnz, L.n, r, zero ? nullptr : xold, xnew);
    else if (L.seg)
        gs_sweep_seg(c, L.a, L.invd.p, r, xold, xnew, dir, zero, dir > 0 ? L.seg_fwd : L.seg_bwd);
    else if (L.cl_size > 0)
        gs_sweep_cluster(c, L.a, L.invd.p, r, xold, xnew, dir, zero, dir > 0 ? L.border_f.p : L.border_b.p,
                         L.cl_size, L.cl_R);
    else if (L.cta_B > 0)
        gs_sweep_cta(c, L.a, L.invd.p, r, xold, xnew, dir, zero, dir > 0 ? L.border_f.p : L.border_b.p, L.cta_B);
    else
        gs_sweep(c, L.a, r, xold, xnew, dir, zero, dir > 0 ? L.ofwd : L.obwd, L.invd.p);
}

void gs_level_sweep(Ctx& c, AmgLevel& L, const double* r, const double* xold, double* xnew, int dir, bool zero) {
    level_sweep(c, L, r, xold, xnew, dir, zero);
}

// amg.cpp:216-231
void Amg::cycle(Ctx& c, int l, const double* r, double* x) {
    AmgLevel& L = *lv[l];
    if (l == n_levels() - 1) {
        dense_gemv(c, coarse_inv.p, nco, r, x);
        return;
    }
    AmgLevel& N = *lv[l + 1];
    const int64_t n = L.n;
    // x = 0; sym GS (the level-synchronous programs mark their own exported rows)
    const bool pend = !L.ls_fwd.ok;
    if (pend) fill_pending(c, L.xf.p, n);
    level_sweep(c, L, r, nullptr, L.xf.p, +1, true);
    if (pend) fill_pending(c, x, n);
    level_sweep(c, L, r, L.xf.p, x, -1, false);
    // rc = R (r - A x)
    csr_spmv(c, L.a, x, L.t.p, r, false, MPREC_K_CSR);
    csr_spmv(c, N.r.view(), L.t.p, N.b.p, nullptr, false, MPREC_K_CSR);
    cycle(c, l + 1, N.b.p, N.x.p);
    // x += P ec
    csr_spmv(c, N.p.view(), N.x.p, x, nullptr, true, MPREC_K_CSR);
    // post sym GS
    if (pend) fill_pending(c, L.xf.p, n);
    level_sweep(c, L, r, x, L.xf.p, +1, false);
    if (pend) fill_pending(c, x, n);
    level_sweep(c, L, r, L.xf.p, x, -1, false);
}

// amg.cpp:233-238
void Amg::apply(Ctx& c, const double* r, double* x) { cycle(c, 0, r, x); }

}  // namespace mg

namespace mg {
extern long long* g_band_ts;
// Diagnostics: per-band timeline of one forward band sweep on level l
void gs_band_timeline(Ctx& c, Amg& amg, int l, long long* host_ts, int* nbands) {
    AmgLevel& L = *amg.lv[l];
    if (!L.band_fwd.ok) throw Error(MPREC_SETUP, "no band schedule on this level");
    DBuf<long long> ts(3 * L.band_fwd.nbands + 2 * L.band_fwd.nchunks);
    fill(c, L.b.p, 1.0, L.n);
    fill_pending(c, L.xf.p, L.n);
    g_band_ts = ts.p;
    level_sweep(c, L, L.b.p, nullptr, L.xf.p, +1, true);
    c.sync();
    g_band_ts = nullptr;
    ts.download(host_ts, 3 * L.band_fwd.nbands + 2 * L.band_fwd.nchunks, c.s);
    c.sync();
    *nbands = L.band_fwd.nbands;
}
// Diagnostics: time `reps` forward+backward sweeps on level l of an AMG.
void gs_bench(Ctx& c, Amg& amg, int l, int reps, double* ms_f, double* ms_b, int* nl_f, int* nl_b) {
    AmgLevel& L = *amg.lv[l];
    fill(c, L.b.p, 1.0, L.n);
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    float tf = 0, tb = 0;
    for (int r = 0; r < reps; ++r) {
        fill_pending(c, L.xf.p, L.n);
        fill_pending(c, L.x.p, L.n);
        cudaEventRecord(e0, c.s);
        level_sweep(c, L, L.b.p, nullptr, L.xf.p, +1, true);
        cudaEventRecord(e1, c.s);
        level_sweep(c, L, L.b.p, L.xf.p, L.x.p, -1, false);
        cudaEventRecord(e2, c.s);
        cudaEventSynchronize(e2);
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        tf += a;
        tb += b;
    }
    *ms_f = tf / reps;
    *ms_b = tb / reps;
    *nl_f = L.band_fwd.ok ? -L.band_fwd.nbands : L.own_fwd.nlev;
    *nl_b = L.band_bwd.ok ? -L.band_bwd.nbands : L.own_bwd.nlev;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
}
}  // namespace mg

namespace mg {
// Setup-time choice of the sweep kernel for one level (measure, don't guess):
// row-per-warp (cross-SM hops), CTA bands of 4096 / 8192 rows (on-SM hops) or
// band-segment chains (gs_seg.cu) or a whole level in one thread block cluster
// (gs_cluster.cu).  MPREC_GS_MODE forces one: warp | cta | seg | cluster.
// LS group counts by level size, in order of preference (B200 measurements,
// DESIGN.md §5.1); the next one is tried when a program does not fit.
static std::vector<int> ls_group_counts(int n) {
    if (n >= (1 << 20)) return {74, 148, 37};
    if (n >= 300000) return {148, 74, 37};
    if (n >= 50000) return {74, 148, 37};
    if (n >= 8192) return {37, 16, 8, 4};
    return {16, 8, 4, 2, 1};  // small levels: one warp may beat any pipeline
}

void tune_level_sweep(Ctx& c, AmgLevel& L, const Sched& sf, const Sched& sb) {
    L.cta_B = 0;
    L.seg = false;
    L.ls_fwd = LsSched();
    L.ls_bwd = LsSched();
    std::string force = [] {  // read per setup so tests can force each kernel
        const char* e = getenv("MPREC_GS_MODE");
        return std::string(e ? e : "");
    }();
    // The sweep kernels round a row's sum in different orders (the LS program
    // pre-scales by 1/a_ii and sums the previous iterate's part first), so the
    // kernel choice must not depend on timing: the default is a fixed rule (the
    // first LS program that fits, the cluster kernel on levels whose iterate fits
    // one cluster, else the warp-per-row sweep) and setups are bitwise
    // reproducible.  MPREC_GS_MODE=tune restores the timed search (experiments).
    const bool timed = force == "tune";
    if (timed) force.clear();
    L.cl_size = 0;
    if (force == "warp") return;
    if (force == "ls") {
        if (!L.glev_f || !L.glev_b || !csr_sorted(c, L.a)) return;
        const int K = [] {
            const char* e = getenv("MPREC_GS_LS_K");
            return e ? atoi(e) : 16;
        }();
        const int rec = [] {
            const char* e = getenv("MPREC_GS_LS_REC");  // 0 auto, 1 fixed class, 2 variable width
            return e ? atoi(e) : 0;
        }();
        build_ls_pair(c, L.a, L.invd.p, L.glev_f, L.glev_b, K, rec, L.ls_fwd, L.ls_bwd);
        return;
    }
    // candidates by size (B200 measurements): the band kernels only
    // win on the finest, million-row levels; the cluster kernel needs the whole
    // level's iterate in one cluster's shared memory
    const bool try_cta = !force.empty() || L.n >= (1 << 20);
    const bool try_seg = !force.empty() || L.n >= (2 << 20);
    int cl_R = 0;
    const int cl_size = gs_cluster_plan(L.n, &cl_R);
    const bool try_cl = cl_size > 0 && (force.empty() || force == "cluster");
    if (force == "cluster") {
        if (!try_cl) return;
        L.cl_size = cl_size;
        L.cl_R = cl_R;
        build_band_order(c, L.n, sf.level.p, cl_R, L.border_f);
        build_band_order(c, L.n, sb.level.p, cl_R, L.border_b);
        return;
    }
    const bool try_ls = L.glev_f && L.glev_b && L.n >= 512;
    if (force.empty() && !timed) {
        if (try_ls && csr_sorted(c, L.a))
            for (int K : ls_group_counts(L.n))
                if (build_ls_pair(c, L.a, L.invd.p, L.glev_f, L.glev_b, K, 0, L.ls_fwd, L.ls_bwd)) {
                    if (trace_on()) fprintf(stderr, "[mprec] level n=%d sweep: level-sync K=%d\n", L.n, K);
                    return;
                }
        if (cl_size > 0) {
            L.cl_size = cl_size;
            L.cl_R = cl_R;
            build_band_order(c, L.n, sf.level.p, cl_R, L.border_f);
            build_band_order(c, L.n, sb.level.p, cl_R, L.border_b);
            if (trace_on()) fprintf(stderr, "[mprec] level n=%d sweep: cluster of %d\n", L.n, cl_size);
            return;
        }
        if (trace_on()) fprintf(stderr, "[mprec] level n=%d sweep: row-per-warp\n", L.n);
        return;
    }
    // million-row levels: the level-synchronous program beats the band kernels by
    // 3-4x, so their schedules are not built and timed
    if (force.empty() && !try_cta && !try_seg && !try_cl && !try_ls) return;
    const bool sorted = csr_sorted(c, L.a);
    if (force == "seg") {
        if (!sorted) return;
        const int bsz = [] {
            const char* e = getenv("MPREC_GS_SEG_B");
            return e ? atoi(e) : 8192;
        }();
        build_seg_sched(c, L.a, L.seg_fwd, L.seg_bwd);
        build_seg_bands(c, L.seg_fwd, bsz);
        build_seg_bands(c, L.seg_bwd, bsz);
        L.seg = true;
        return;
    }
    fill(c, L.b.p, 1.0, L.n);
    cudaEvent_t e0, e1;
    MG_CUDA(cudaEventCreate(&e0));
    MG_CUDA(cudaEventCreate(&e1));
    auto time_fwd = [&]() {
        float best = 1e30f;
        for (int rep = 0; rep < 2; ++rep) {
            fill_pending(c, L.xf.p, L.n);
            cudaEventRecord(e0, c.s);
            level_sweep(c, L, L.b.p, nullptr, L.xf.p, +1, true);
            cudaEventRecord(e1, c.s);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        return best;
    };
    const char* names[5] = {"row-per-warp", "cta-band", "band-segment", "cluster", "level-sync"};
    int best_mode = 0, b_best = 0;
    // level-synchronous programs (gs_ls.cu) first: on levels above 50k rows they
    // beat the band kernels by 2-4x, so those are only built and
    // timed when no LS program fits the level.  Group counts by level size, the
    // next candidate tried only when a program does not fit (dependency beyond
    // the previous group, shared memory); both directions built together.
    int ls_K = 0;
    LsSched ls_bf, ls_bb;
    float t_ls = 1e30f;
    if (try_ls && sorted && force.empty()) {
        const std::vector<int> cands = ls_group_counts(L.n);
        const bool first_fit = L.n >= 50000;  // large levels: the first program that fits
        for (int K : cands) {
            if (!build_ls_pair(c, L.a, L.invd.p, L.glev_f, L.glev_b, K, 0, L.ls_fwd, L.ls_bwd)) continue;
            LsSched keep_b = std::move(L.ls_bwd);
            L.ls_bwd = LsSched();
            const float t = time_fwd();
            if (t < t_ls) {
                t_ls = t;
                ls_K = K;
                ls_bf = std::move(L.ls_fwd);
                ls_bb = std::move(keep_b);
            }
            L.ls_fwd = LsSched();
            if (first_fit) break;
        }
    }
    const bool skip_band = ls_K > 0 && L.n >= 50000;
    float t_best = force.empty() ? time_fwd() : 1e30f;
    if ((force.empty() && try_cta && !skip_band) || force == "cta") {
        for (int bsz : {4096, 8192}) {
            if (L.n < 2 * bsz) continue;
            L.cta_B = bsz;
            build_band_order(c, L.n, sf.level.p, bsz, L.border_f);
            const float t = time_fwd();
            if (t < t_best) {
                t_best = t;
                b_best = bsz;
                best_mode = 1;
            }
        }
        L.cta_B = 0;
    }
    int seg_best = 0;
    if (sorted && ((force.empty() && try_seg && !skip_band) || force == "seg")) {
        build_seg_sched(c, L.a, L.seg_fwd, L.seg_bwd);
        L.seg = true;
        for (int bsz : {4096, 8192}) {
            build_seg_bands(c, L.seg_fwd, bsz);
            const float t = time_fwd();
            if (t < t_best) {
                t_best = t;
                best_mode = 2;
                seg_best = bsz;
            }
            if (L.n <= bsz) break;
        }
        L.seg = false;
    }
    int cl_best = 0, cl_best_R = 0;
    if (try_cl) {
        // every feasible cluster size: more CTAs = more warps in flight, fewer local hops
        for (int want : {1, 2, 4, 8, 16}) {
            int r = 0;
            const int cs = gs_cluster_plan(L.n, &r, want);
            if (cs != want) continue;
            L.cl_size = cs;
            L.cl_R = r;
            build_band_order(c, L.n, sf.level.p, r, L.border_f);
            float t = 1e30f;
            try {
                t = time_fwd();
            } catch (const Error&) {  // cluster not schedulable on this device
                cudaGetLastError();
            }
            L.cl_size = 0;
            if (t < t_best) {
                t_best = t;
                best_mode = 3;
                cl_best = cs;
                cl_best_R = r;
            }
        }
    }
    // the level-synchronous program when it is the fastest candidate
    if (ls_K > 0 && t_ls < t_best) {
        t_best = t_ls;
        best_mode = 4;
        L.ls_fwd = std::move(ls_bf);
        L.ls_bwd = std::move(ls_bb);
    } else {
        ls_K = 0;
        L.ls_fwd = LsSched();
        L.ls_bwd = LsSched();
    }
    if (best_mode != 2) {
        L.seg_fwd = SegSched();
        L.seg_bwd = SegSched();
    }
    L.seg = best_mode == 2;
    if (L.seg) {
        build_seg_bands(c, L.seg_fwd, seg_best);
        build_seg_bands(c, L.seg_bwd, seg_best);
    }
    L.cta_B = best_mode == 1 ? b_best : 0;
    if (best_mode == 1) {
        build_band_order(c, L.n, sf.level.p, b_best, L.border_f);
        build_band_order(c, L.n, sb.level.p, b_best, L.border_b);
    } else if (best_mode == 3) {
        L.cl_size = cl_best;
        L.cl_R = cl_best_R;
        build_band_order(c, L.n, sf.level.p, cl_best_R, L.border_f);
        build_band_order(c, L.n, sb.level.p, cl_best_R, L.border_b);
    } else {
        L.border_f.release();
        L.border_b.release();
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (trace_on())
        fprintf(stderr, "[mprec] level n=%d sweep: %s B=%d (%.3f ms fwd)\n", L.n, names[best_mode],
                best_mode == 2 ? seg_best : (best_mode == 3 ? L.cl_size : best_mode == 4 ? ls_K : L.cta_B), t_best);
}
}  // namespace mg
