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

// rows sorted by column with the diagonal present (the LS programs' precondition)
__global__ void k_sorted(const int* rp, const int* ci, const int* diag, int n, int* bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool ok = diag[i] >= rp[i] && diag[i] < rp[i + 1] && ci[diag[i]] == i;
    for (int k = rp[i] + 1; k < rp[i + 1]; ++k) ok = ok && ci[k - 1] < ci[k];
    if (!ok) atomicOr(bad, 1);
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

bool csr_sorted(Ctx& c, const CsrView& a) {
    if (a.n == 0) return true;
    DBuf<int> bad(1);
    MG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.s));
    k_sorted<<<(a.n + 255) / 256, 256, 0, c.s>>>(a.rp, a.ci, a.diag, a.n, bad.p);
    int h = 1;
    MG_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    return h == 0;
}

void compute_invd(Ctx& c, const CsrView& a, double* invd) {
    k_invd<<<(a.n + 255) / 256, 256, 0, c.s>>>(a.v, a.diag, a.n, invd);
    check_launch("invd");
}

// Fused residual + restriction (K15): rc = R (r - A x) in one launch
// (amg.cpp:224-226).  A coarse row's lanes walk its R entries; each entry's fine
// residual t_j = r_j - (A x)_j is recomputed on the fly with exactly the
// association k_csr<LNA> uses for the unfused residual (LNA strided partial sums,
// xor butterfly), and the R row is summed like k_csr<LNR>: bitwise equal to the
// two-launch path.  Each fine row is recomputed once per R entry that refers to
// it (~2x on the RS levels), so it pays only where the level is launch-bound.
template <int LNA, int LNR>
__global__ void __launch_bounds__(256) k_resid_restrict(const int* __restrict__ rp, const int* __restrict__ ci,
                                                        const double* __restrict__ v, const double* __restrict__ x,
                                                        const double* __restrict__ r, const int* __restrict__ rrp,
                                                        const int* __restrict__ rci, const double* __restrict__ rv,
                                                        double* __restrict__ rc, int nc) {
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    const int row = int(g / LNR), s = int(g % LNR);
    double acc = 0.0;
    if (row < nc)
        for (int k = __ldg(rrp + row) + s; k < __ldg(rrp + row + 1); k += LNR) {
            const int j = __ldg(rci + k);
            const int a0 = __ldg(rp + j), a1 = __ldg(rp + j + 1);
            double p[LNA];
#pragma unroll
            for (int s2 = 0; s2 < LNA; ++s2) {
                double ps = 0.0;
                for (int q = a0 + s2; q < a1; q += LNA) ps += __ldg(v + q) * __ldg(x + __ldg(ci + q));
                p[s2] = ps;
            }
#pragma unroll
            for (int o = 1; o < LNA; o <<= 1)
#pragma unroll
                for (int i = 0; i < LNA; i += 2 * o) p[i] = p[i] + p[i + o];
            acc += __ldg(rv + k) * (__ldg(r + j) - p[0]);
        }
#pragma unroll
    for (int o = 1; o < LNR; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (row < nc && s == 0) rc[row] = acc;
}

static int csr_lanes(const CsrView& a) {
    const double per_row = double(a.nnz) / std::max(a.n, 1);
    return per_row <= 3.0 ? 2 : per_row <= 6.0 ? 4 : per_row <= 12.0 ? 8 : 16;
}

template <int LNA>
static void launch_rr(Ctx& c, const CsrView& a, const CsrView& R, const double* x, const double* r, double* rc, int lnr) {
    const int grid = int(((int64_t)R.n * lnr + 255) / 256);
    switch (lnr) {
        case 2: k_resid_restrict<LNA, 2><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, r, R.rp, R.ci, R.v, rc, R.n); break;
        case 4: k_resid_restrict<LNA, 4><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, r, R.rp, R.ci, R.v, rc, R.n); break;
        case 8: k_resid_restrict<LNA, 8><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, r, R.rp, R.ci, R.v, rc, R.n); break;
        default: k_resid_restrict<LNA, 16><<<grid, 256, 0, c.s>>>(a.rp, a.ci, a.v, x, r, R.rp, R.ci, R.v, rc, R.n); break;
    }
}

// rc = R (r - A x)
void csr_resid_restrict(Ctx& c, const CsrView& a, const CsrView& R, const double* x, const double* r, double* rc) {
    if (R.n == 0) return;
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 16.0 * a.n + 12.0 * R.nnz + 4.0 * (R.n + 1) + 8.0 * R.n;
    Ctx::Scope sc(&c, MPREC_K_CSR, bytes);
    const int lnr = csr_lanes(R);
    switch (csr_lanes(a)) {
        case 2: launch_rr<2>(c, a, R, x, r, rc, lnr); break;
        case 4: launch_rr<4>(c, a, R, x, r, rc, lnr); break;
        case 8: launch_rr<8>(c, a, R, x, r, rc, lnr); break;
        default: launch_rr<16>(c, a, R, x, r, rc, lnr); break;
    }
    check_launch("resid+restrict");
}

void csr_spmv(Ctx& c, const CsrView& a, const double* x, double* y, const double* b, bool add_to_y, int kclass) {
    if (a.n == 0) return;
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 8.0 * a.m + 8.0 * a.n + ((b || add_to_y) ? 8.0 * a.n : 0.0);
    Ctx::Scope sc(&c, kclass, bytes);
    const int mode = add_to_y ? 2 : (b ? 1 : 0);
    const int ln = csr_lanes(a);
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

// one Gauss-Seidel direction on level L with the kernel chosen at setup
static void level_sweep(Ctx& c, AmgLevel& L, const double* r, const double* xold, double* xnew, int dir, bool zero) {
    const LsSched& ls = dir > 0 ? L.ls_fwd : L.ls_bwd;
    if (ls.ok)
        gs_sweep_ls(c, L.a, L.invd.p, r, xold, xnew, zero, ls);
    else if (L.cl_size > 0)
        gs_sweep_cluster(c, L.a, L.invd.p, r, xold, xnew, dir, zero, dir > 0 ? L.border_f.p : L.border_b.p,
                         L.cl_size, L.cl_R);
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
    // rc = R (r - A x): one fused launch on the launch-bound (small) levels, two
    // CSR products above (bitwise the same; MPREC_FUSE_RR_MAX = largest fused level)
    static const int fuse_max = [] {
        const char* e = getenv("MPREC_FUSE_RR_MAX");
        return e ? atoi(e) : 100000;
    }();
    if (L.n <= fuse_max) {
        csr_resid_restrict(c, L.a, N.r.view(), x, r, N.b.p);
    } else {
        csr_spmv(c, L.a, x, L.t.p, r, false, MPREC_K_CSR);
        csr_spmv(c, N.r.view(), L.t.p, N.b.p, nullptr, false, MPREC_K_CSR);
    }
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
    *nl_f = L.own_fwd.nlev;
    *nl_b = L.own_bwd.nlev;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
}
}  // namespace mg

namespace mg {
// Setup-time choice of the sweep kernel for one level.  The kernels round a
// row's sum in different orders (the LS programs pre-scale by 1/a_ii and sum the
// previous iterate's part first), so the choice is a fixed rule -- not timing --
// and setups are bitwise reproducible:
//   1. the level-synchronous programs (gs_ls.cu) with the first plan of
//      ls_plans() that fits (B200 measurements);
//   2. else the thread-block-cluster sweep (gs_cluster.cu) when the level's
//      iterate fits one cluster's shared memory;
//   3. else the warp-per-row sweep in topological claim order (k_gs).
// MPREC_GS_MODE=warp | cluster | ls forces one (tests; `ls` with MPREC_GS_LS_K
// groups, default 16, MPREC_GS_LS_NW compute warps per group, default 1, and
// MPREC_GS_LS_ND=0|2|4|8 dependency class, default 0 = from the level).
struct LsPlan {
    int K, nw;
};
// r = rows per DAG level.  Narrow levels run as ONE group (no boundary hops) on
// 1-4 lockstep warps; wide levels as a pipeline of groups.  c5, r02 build
// (scripts/gs_lw_exp.py; ms per forward sweep, previous kernel in brackets):
//   r 1000 / 486 (levels 0, 1): 74 groups x 1 warp    0.48 / 0.55  [0.67 / 0.80]
//   r 170 / 120  (levels 2, 3): 37 / 28 groups x 2    0.96 / 0.73  [1.58 / 1.22]
//   r 87         (level 4):     1 group x 4 warps     0.47         [0.87]
//   r 63         (level 5):     1 x 3                 0.23         [0.43]
//   r 46 / 32    (levels 6, 7): 1 x 2                 0.11 / 0.07  [0.25 / 0.13]
//   r <= 26      (levels 8+):   1 x 1                 0.04 ...     [0.06 ...]
static std::vector<LsPlan> ls_plans(int n, int depth) {
    const double r = double(n) / std::max(depth, 1);
    std::vector<LsPlan> p;
    if (r <= 26) p = {{1, 1}, {4, 1}};
    else if (r <= 50) p = {{1, 2}, {4, 2}, {8, 1}};
    else if (r <= 75) p = {{1, 3}, {4, 2}, {16, 2}};
    else if (r <= 100) p = {{1, 4}, {24, 3}, {37, 2}};
    else if (r <= 140) p = {{28, 2}, {37, 2}, {74, 1}};
    else if (r <= 250) p = {{37, 2}, {56, 2}, {74, 1}};
    else p = {{74, 1}, {148, 1}, {37, 2}};
    for (LsPlan q : {LsPlan{74, 1}, LsPlan{37, 1}, LsPlan{16, 1}, LsPlan{8, 1}, LsPlan{4, 1}, LsPlan{1, 1}}) p.push_back(q);
    return p;
}

void tune_level_sweep(Ctx& c, AmgLevel& L, const Sched& sf, const Sched& sb) {
    L.ls_fwd = LsSched();
    L.ls_bwd = LsSched();
    L.cl_size = 0;
    const std::string force = [] {  // read per setup so tests can force each kernel
        const char* e = getenv("MPREC_GS_MODE");
        return std::string(e ? e : "");
    }();
    if (force == "warp") return;
    auto env_int = [](const char* name, int dflt) {
        const char* e = getenv(name);
        return e ? atoi(e) : dflt;
    };
    if (force == "ls") {
        if (!csr_sorted(c, L.a)) return;
        build_ls_pair(c, L.a, L.invd.p, env_int("MPREC_GS_LS_K", 16), env_int("MPREC_GS_LS_NW", 1),
                      env_int("MPREC_GS_LS_ND", 0), L.ls_fwd, L.ls_bwd);
        return;
    }
    if (force.empty() && L.n >= 512 && csr_sorted(c, L.a)) {
        int lastK = -1, lastnw = -1;
        for (LsPlan q : ls_plans(L.n, std::max(sf.nlev, sb.nlev))) {
            if (q.K == lastK && q.nw == lastnw) continue;
            lastK = q.K;
            lastnw = q.nw;
            if (L.n < 64 * q.K) continue;
            if (build_ls_pair(c, L.a, L.invd.p, q.K, q.nw, 0, L.ls_fwd, L.ls_bwd)) {
                if (trace_on())
                    fprintf(stderr, "[mprec] level n=%d depth %d sweep: level-sync K=%d nw=%d\n", L.n, sf.nlev, q.K, q.nw);
                return;
            }
        }
    }
    int cl_R = 0;
    const int cl_size = gs_cluster_plan(L.n, &cl_R);
    if (cl_size > 0 && (force.empty() || force == "cluster")) {
        L.cl_size = cl_size;
        L.cl_R = cl_R;
        build_band_order(c, L.n, sf.level.p, cl_R, L.border_f);
        build_band_order(c, L.n, sb.level.p, cl_R, L.border_b);
        if (trace_on()) fprintf(stderr, "[mprec] level n=%d sweep: cluster of %d\n", L.n, cl_size);
        return;
    }
    if (trace_on()) fprintf(stderr, "[mprec] level n=%d sweep: row-per-warp\n", L.n);
}
}  // namespace mg
