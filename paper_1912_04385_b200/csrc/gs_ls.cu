// gs_ls.cu -- level-synchronous pipelined Gauss-Seidel sweep (K14).
//
// Same natural-order semantics as the other sweep kernels
// (sym_gauss_seidel, amg.cpp:25-43): x_i = (b_i - sum_{k<i} a_ik x_k^new
// - sum_{k>i} a_ik x_k^old) / a_ii in the forward direction, the mirror image
// backward.  What changes is how the dependency DAG is mapped onto the GPU:
//
//   * GROUPS.  The rows are cut into K contiguous ranges in sweep order, one
//     thread block (one SM) each.  A group's rows are processed by nw compute
//     warps (usually one) in DAG-level order, <= 32 nw rows (one "step") at a
//     time, with only a __syncwarp (nw > 1: a named barrier) between steps:
//     every dependency inside the group is a shared-memory read of a value
//     written one or a few steps earlier.  The per-level cost is a few dozen
//     instructions instead of a cross-SM hop.
//   * PIPELINE.  Dependencies may only cross into the previous group (checked
//     at setup; the level falls back to the other kernels otherwise).  An
//     importer warp polls the previous group's published values and copies
//     them into a shared-memory halo; the compute warps only check a
//     shared-memory counter.  The cross-SM latency is paid once per group
//     boundary (pipeline fill), not once per DAG level.  Narrow levels (few
//     rows per DAG level) run as ONE group on one SM with no boundary at all.
//   * PROGRAM.  Everything that does not depend on the sweep's new values --
//     the row's coefficients pre-multiplied by 1/a_ii and the shared-memory
//     offsets of its dependencies -- is compiled at setup into a per-group
//     stream of fixed-size steps, in processing order, which a loader warp
//     streams into a shared-memory ring with 1-D TMA bulk copies
//     (cp.async.bulk + mbarrier).  The part of each row that depends on the
//     previous iterate, c'_i = (b_i - sum_old a_ik x_k^old) / a_ii, is computed
//     by a fully parallel pre-pass straight into the program.
//
// Own-group values live in a ring of W slots indexed by processing position.
// Results differ from the warp-per-row sweep only by association (the old part
// is summed first, coefficients are pre-scaled by 1/a_ii, wide rows are summed
// through partial nodes) and stay within the 1e-10 apply bar.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "mprec.cuh"

namespace mg {
namespace {


__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
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

__host__ __device__ constexpr int ls_nd(int cls) { return 2 << cls; }

// ---------------------------------------------------------------------------
// Fixed-format warp-steps (k_gs_lw): the program format and the step loop.  A
// lone warp pays ~5-10 cycles per issued instruction, so the step loop is kept
// to ~25-45 instructions (the header-parsed records of the first versions of
// this file cost ~120 per step, 0.2-0.4 us per DAG level):
//   * a step is NW WARP BLOCKS of fixed size (one per compute warp), each an
//     array of 16-byte vectors over the 32 lanes (every load a conflict-free
//     lane-strided LDS.128): ND/2 vectors of coefficients a_ij / a_ii, one tail
//     vector {c', row, packed}, ND 32-bit byte offsets of the dependencies in
//     the value area.  No headers, no variable sizes, a fixed number of steps
//     per chunk (the inner loop is fully unrolled, every program address an
//     immediate); the record of step s + 1 is loaded into registers while step
//     s waits for its dependency values, which are the only loads left on the
//     step-to-step chain.
//   * packed = own byte offset in the value area (17 bits) | imports needed (15).
//   * NODES: a row with more than ND dependencies becomes a two-level tree --
//     partial nodes summing its earliest-available dependencies (scheduled in
//     earlier steps, in otherwise idle lanes, value kept in the ring only) and a
//     final node of <= ND inputs.  The node DAG is re-levelled on the host; no
//     shuffles in the step loop.
//   * the compute warps never touch an mbarrier: a publisher warp waits for the
//     bulk copies and advances a `loaded` chunk counter (checked once per
//     chunk), the compute warps publish `consumed` chunk counters the loader
//     polls before it refills a ring slot.
//   * NW > 1: the compute warps run in lockstep, one named barrier per step
//     (slower per step -- the warps share the SM's one shared-memory pipe: 0.108 /
//     0.135 / 0.185 / 0.243 us for 1-4 warps at ND = 8 -- but one step per DAG
//     level where a level has up to 32 NW nodes).
// Padding lanes and padding steps: zero coefficients, the zero slot, row -1,
// the trash slot.
__host__ __device__ constexpr int lw_wb(int nd) { return nd == 2 ? 1280 : nd == 4 ? 2048 : 3584; }
__host__ __device__ constexpr int lw_tail(int nd) { return (nd / 2) * 512; }
__host__ __device__ constexpr int lw_off(int nd) { return (nd / 2) * 512 + 512; }
__host__ __device__ constexpr int lw_spc(int nd) { return nd == 8 ? 4 : 8; }  // steps per chunk
constexpr int kLwOwnBits = 17;

template <int ND>
struct LwRec {
    double e[ND];
    unsigned off[ND];
    double c;
    int row;
    unsigned packed;
};

template <int ND>
__device__ __forceinline__ void lw_load(unsigned wb, int lane, LwRec<ND>& r) {  // wb: the warp block
    const unsigned a = wb + 16u * unsigned(lane);
#pragma unroll
    for (int v = 0; v < ND / 2; ++v)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.e[2 * v]), "=d"(r.e[2 * v + 1]) : "r"(a + 512 * v));
    unsigned lo, hi;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(lo), "=r"(hi), "=r"(r.row), "=r"(r.packed)
                 : "r"(a + lw_tail(ND)));
    r.c = __hiloint2double(int(hi), int(lo));
    if (ND == 2) {
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                     : "=r"(r.off[0]), "=r"(r.off[1])
                     : "r"(wb + lw_off(ND) + 8u * unsigned(lane)));
    } else {
#pragma unroll
        for (int v = 0; v < ND / 4; ++v)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r.off[4 * v]), "=r"(r.off[4 * v + 1]), "=r"(r.off[4 * v + 2]), "=r"(r.off[4 * v + 3])
                         : "r"(a + lw_off(ND) + 512 * v));
    }
}

// wait until the shared-memory counter at `a` reaches `want` (warp-uniform)
__device__ __forceinline__ void lw_wait(unsigned a, int want, int& have) {
    asm volatile(
        "{\n .reg .pred p;\n .reg .s32 r;\n"
        " setp.le.s32 p, %2, %0;\n"
        " @p bra.uni LWD%=;\n"
        "LWW%=:\n ld.volatile.shared.s32 r, [%1];\n setp.lt.s32 p, r, %2;\n @p bra.uni LWW%=;\n"
        " mov.s32 %0, r;\n fence.acq_rel.cta;\n"
        "LWD%=:\n}"
        : "+r"(have)
        : "r"(a), "r"(want)
        : "memory");
}

template <int ND, int NW>
__global__ void __launch_bounds__((NW + 3) * 32, 1) k_gs_lw(const char* __restrict__ prog, const int2* __restrict__ gch,
                                                             const int* __restrict__ imp, const int2* __restrict__ gimp,
                                                             double* xnew, int W, int hmax, int ns, long long* stats) {
    constexpr int WB = lw_wb(ND), SPC = lw_spc(ND), nw = NW;
    constexpr bool MULTI = NW > 1;
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int stepb = NW * WB, chb = SPC * stepb;
    char* ring = reinterpret_cast<char*>(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + ns * chb);
    int* ctr = reinterpret_cast<int*>(full + ns);  // [0] imported, [1] chunks loaded, [2 + w] chunks consumed by warp w
    double* xs = reinterpret_cast<double*>(sm + ns * chb + ns * 8 + 64);
    const int g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2 ch = gch[g];  // first chunk, chunks
    const int nch = ch.y;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) mbar_init(full + s, 1);
        for (int q = 0; q < 16; ++q) ctr[q] = 0;
        xs[W] = 0.0;  // zero slot (padding dependencies)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == nw + 1) {  // loader: program chunks -> ring, refilling a slot once every compute warp released it
        if (lane == 0) {
            volatile int* cons = ctr + 2;
            for (int c = 0; c < nch; ++c) {
                const int s = c % ns;
                if (c >= ns) {
                    for (int w = 0; w < nw; ++w)
                        while (cons[w] < c - ns + 1) __nanosleep(32);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                mbar_expect_tx(full + s, chb);
                bulk_g2s(ring + s * chb, prog + (int64_t)(ch.x + c) * chb, chb, full + s);
            }
        }
        return;
    }
    if (warp == nw + 2) {  // publisher: completed bulk copies -> `loaded` chunk counter
        if (lane == 0) {
            volatile int* ld = ctr + 1;
            for (int c = 0; c < nch; ++c) {
                mbar_wait(full + (c % ns), (c / ns) & 1);
                __threadfence_block();
                *ld = c + 1;
            }
        }
        return;
    }
    if (warp == nw) {  // importer: previous group's values -> halo, in production order
        const int2 gi = gimp[g];
        const int* rows = imp + gi.x;
        const int nimp = gi.y;
        volatile double* halo = xs + W + 1;
        volatile int* vimp = ctr;
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
    // compute warps
    const unsigned xs_a = smem_u32(xs);
    const unsigned imp_a = smem_u32(ctr), ld_a = imp_a + 4, cons_a = imp_a + 8 + 4 * warp;
    const unsigned ring_a = smem_u32(ring) + unsigned(warp) * WB;
    double* xg = xnew;
    asm volatile("" : "+l"(xg));  // keep the pointer in registers (no constant-bank reload per step)
    int have_imp = 0, have_ld = 0, slot = 0;
    long long t_start = 0, t_first = 0;
    if (stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    LwRec<ND> R;
    for (int c = 0; c < nch; ++c) {
        // this chunk and the next one (its first record is prefetched at this chunk's last step)
        lw_wait(ld_a, min(nch, c + 2), have_ld);
        const unsigned base = ring_a + unsigned(slot) * unsigned(chb);
        slot = slot + 1 == ns ? 0 : slot + 1;
        const unsigned nbase = c + 1 < nch ? ring_a + unsigned(slot) * unsigned(chb) : base;
        if (c == 0) lw_load<ND>(base, lane, R);
#pragma unroll
        for (int k = 0; k < SPC; ++k) {
            lw_wait(imp_a, int(R.packed >> kLwOwnBits), have_imp);
            if (MULTI)
                asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
            else
                __syncwarp();
            double xv[ND];
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                MG_DCHECK(R.off[d] <= 8u * unsigned(W + 1 + hmax) && (R.off[d] & 7u) == 0);
                asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(xv[d]) : "r"(xs_a + R.off[d]) : "memory");
            }
            LwRec<ND> N;
            lw_load<ND>(k + 1 < SPC ? base + unsigned(k + 1) * unsigned(stepb) : nbase, lane, N);
            // x = c' - sum_d e_d x_d as a tree of depth <= 4
            double x;
            if (ND == 2) {
                x = fma(-R.e[1], xv[1], fma(-R.e[0], xv[0], R.c));
            } else if (ND == 4) {
                const double t0 = fma(-R.e[1], xv[1], fma(-R.e[0], xv[0], R.c));
                const double t1 = fma(R.e[3], xv[3], R.e[2] * xv[2]);
                x = t0 - t1;
            } else {
                const double t0 = fma(-R.e[1], xv[1], fma(-R.e[0], xv[0], R.c));
                const double t1 = fma(R.e[3], xv[3], R.e[2] * xv[2]);
                const double t2 = fma(R.e[5], xv[5], R.e[4] * xv[4]);
                const double t3 = fma(R.e[7], xv[7], R.e[6] * xv[6]);
                x = (t0 - t1) - (t2 + t3);
            }
            const unsigned own = R.packed & ((1u << kLwOwnBits) - 1);
            MG_DCHECK(own <= 8u * unsigned(W + 1 + hmax) && (R.row < 0 || own < 8u * unsigned(W)));
            asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(xs_a + own), "d"(x) : "memory");
            asm volatile(
                "{\n .reg .pred p;\n setp.ge.s32 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(xg + R.row),
                "l"(__double_as_longlong(x)), "r"(R.row)
                : "memory");
            R = N;
        }
        if (lane == 0) asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(cons_a), "r"(c + 1) : "memory");
        if (stats && c == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_first));
    }
    if (stats && threadIdx.x == 0) {  // diagnostics: group start, end of its first chunk, end
        long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        stats[4 * g + 0] = t_start;
        stats[4 * g + 1] = t_end;
        stats[4 * g + 2] = t_first - t_start;
        stats[4 * g + 3] = nch * SPC;
    }
}


__global__ void k_ls_testvec(double* b, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = 1.5 + sin(0.37 * i);
}


}  // namespace

struct LsBuilt {
    bool ok = false;
    int K = 0, W = 0, hmax = 0, dir = 0, nsteps = 0, nchunks = 0, maxdist = 0, nd = 0, ns = 0, cls = 0;
    int nw = 0, spc = 0, chb = 0;  // fixed-format warp-steps (k_gs_lw)
    std::vector<char> prog;
    std::vector<int2> gch, gimp;
    std::vector<int> imp;
    std::vector<long long> coff;
};

// Fixed-format warp-step programs (k_gs_lw) of one sweep direction.  nw compute
// warps per group; ndsel 0: dependency class chosen from the level, 1/2/3: ND = 2/4/8.
static void ls_build_lw(const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<double>& v,
                        const std::vector<double>& invd, int n, int dir, int K, int nw, int ndsel, LsBuilt& out) {
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
    std::vector<int> nd(n, 0);
    int maxnd = 0;
    int64_t sumnd = 0;
    for (int i = 0; i < n; ++i) {
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (!is_dep(i, j)) continue;
            if (gid[j] != gid[i] && gid[j] != gid[i] - 1) return;  // beyond the previous group
            ++nd[i];
        }
        maxnd = std::max(maxnd, nd[i]);
        sumnd += nd[i];
    }
    // dependency class: ND >= the widest row when that is <= 4; else 8 (wider rows
    // become trees of partial nodes).  A two-level tree holds ND * ND dependencies.
    int ND = ndsel == 1 ? 2 : ndsel == 2 ? 4 : ndsel == 3 ? 8 : maxnd <= 2 ? 2 : maxnd <= 4 ? 4 : 8;
    if (maxnd > ND * ND) ND = 8;
    if (maxnd > ND * ND) return;
    const int cls = ND == 2 ? 0 : ND == 4 ? 1 : 2;
    // ---- nodes: id < n is row id's final node, id >= n a partial node.  Expanded
    // rows keep their inputs in (xsrc, xcoef): src >= 0 a row's value, src < 0 the
    // partial node n + (-1 - src)
    struct Part {
        int owner, lev, first, cnt;
    };
    std::vector<Part> parts;
    std::vector<int> xfirst(n, -1), xcnt(n, 0), xsrc;
    std::vector<double> xcoef;
    std::vector<int> rlev(n, 0);
    {
        std::vector<std::pair<int, int>> dl;  // (level of the dependency, k)
        for (int t = 0; t < n; ++t) {
            const int i = row_of_t(t);
            int lv = 0;
            if (nd[i] <= ND) {
                for (int k = rp[i]; k < rp[i + 1]; ++k)
                    if (is_dep(i, ci[k])) lv = std::max(lv, rlev[ci[k]] + 1);
                rlev[i] = lv;
                continue;
            }
            dl.clear();
            for (int k = rp[i]; k < rp[i + 1]; ++k)
                if (is_dep(i, ci[k])) dl.emplace_back(rlev[ci[k]], k);
            std::stable_sort(dl.begin(), dl.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            const int m = int(dl.size());
            const int P = (m - ND + (ND - 2)) / (ND - 1);  // partial nodes
            const int direct = ND - P;                     // latest dependencies stay direct
            const int npd = m - direct;                    // dependencies summed by partial nodes
            xfirst[i] = int(xsrc.size());
            int at = 0;
            // layout in xsrc for row i: [final node inputs: P partial refs + direct deps][partial 0 deps][partial 1 deps]...
            const int pbase = int(parts.size());
            for (int p = 0; p < P; ++p) {
                xsrc.push_back(-1 - (pbase + p));
                xcoef.push_back(1.0);
            }
            for (int q = npd; q < m; ++q) {
                xsrc.push_back(ci[dl[q].second]);
                xcoef.push_back(v[dl[q].second] * invd[i]);
                lv = std::max(lv, dl[q].first + 1);
            }
            xcnt[i] = P + direct;
            at = 0;
            for (int p = 0; p < P; ++p) {
                const int cnt = std::min(ND, npd - at);
                Part pn{i, 0, int(xsrc.size()), cnt};
                for (int q = at; q < at + cnt; ++q) {
                    xsrc.push_back(ci[dl[q].second]);
                    xcoef.push_back(-(v[dl[q].second] * invd[i]));  // node value = +sum e x
                    pn.lev = std::max(pn.lev, dl[q].first + 1);
                }
                lv = std::max(lv, pn.lev + 1);
                parts.push_back(pn);
                at += cnt;
            }
            rlev[i] = lv;
            // partial nodes no earlier than two levels before their row: the value
            // only lives in the ring
            for (int p = 0; p < P; ++p) parts[pbase + p].lev = std::max(parts[pbase + p].lev, lv - 2);
        }
    }
    const int np = int(parts.size()), nn = n + np;
    auto node_lev = [&](int id) { return id < n ? rlev[id] : parts[id - n].lev; };
    // ---- processing order inside each group: (node level, id)
    std::vector<int> gnstart(K + 1, 0);
    {
        std::vector<int> cntg(K, 0);
        for (int g = 0; g < K; ++g) cntg[g] = gstart[g + 1] - gstart[g];
        for (const Part& p : parts) ++cntg[gid[p.owner]];
        for (int g = 0; g < K; ++g) gnstart[g + 1] = gnstart[g] + cntg[g];
    }
    std::vector<int> seq(nn), pos(nn);
    {
        std::vector<int> fill(gnstart.begin(), gnstart.end() - 1);
        for (int g = 0; g < K; ++g)
            for (int t = gstart[g]; t < gstart[g + 1]; ++t) seq[fill[g]++] = row_of_t(t);
        for (int p = 0; p < np; ++p) seq[fill[gid[parts[p].owner]]++] = n + p;
        for (int g = 0; g < K; ++g) {
            int* q = seq.data() + gnstart[g];
            const int m = gnstart[g + 1] - gnstart[g];
            std::stable_sort(q, q + m, [&](int a, int b) { return node_lev(a) < node_lev(b); });
            for (int u = 0; u < m; ++u) pos[q[u]] = u;
        }
    }
    // inputs of a node: f(src row or partial id as node id, coefficient)
    auto for_inputs = [&](int id, auto&& f) {
        if (id >= n) {
            const Part& p = parts[id - n];
            for (int q = p.first; q < p.first + p.cnt; ++q) f(xsrc[q], xcoef[q]);
        } else if (xfirst[id] >= 0) {
            for (int q = xfirst[id]; q < xfirst[id] + xcnt[id]; ++q)
                f(xsrc[q] >= 0 ? xsrc[q] : n + (-1 - xsrc[q]), xcoef[q]);
        } else {
            for (int k = rp[id]; k < rp[id + 1]; ++k)
                if (is_dep(id, ci[k])) f(ci[k], v[k] * invd[id]);
        }
    };
    auto node_gid = [&](int id) { return gid[id < n ? id : parts[id - n].owner]; };
    // ---- ring size.  Own-group values live in a ring of W slots indexed by
    // processing position; a dependency further back than the ring holds (a few
    // rows reach hundreds of DAG levels back) is a FAR dependency: the row's value
    // comes back through the group's own importer, from global memory
    const int WB = lw_wb(ND), SPC = lw_spc(ND), cap = 32 * nw;
    const int stepb = nw * WB, chb = SPC * stepb;
    int maxdist = 0, maxlev = 0;
    for (int g = 0; g < K; ++g) {
        for (int u = gnstart[g]; u < gnstart[g + 1]; ++u) {
            const int id = seq[u];
            for_inputs(id, [&](int src, double) {
                if (node_gid(src) == g) maxdist = std::max(maxdist, pos[id] - pos[src]);
            });
        }
        for (int u = gnstart[g], u1; u < gnstart[g + 1]; u = u1) {
            for (u1 = u; u1 < gnstart[g + 1] && node_lev(seq[u1]) == node_lev(seq[u]);) ++u1;
            maxlev = std::max(maxlev, u1 - u);
        }
    }
    const int margin = std::max(cap, maxlev) + 32;
    // (MPREC_GS_LS_WCAP: a smaller ring for tests, so that small systems exercise
    // the far-dependency path)
    const int wcap_env = getenv("MPREC_GS_LS_WCAP") ? atoi(getenv("MPREC_GS_LS_WCAP")) : 0;
    const int wcap = wcap_env >= 256 && (wcap_env & (wcap_env - 1)) == 0 ? wcap_env : (225 * 1024 - 3 * chb) / 8 >= 8192 + 4096 ? 8192 : 4096;
    int W = 64, farthr = INT_MAX;
    while (W < maxdist + margin) W <<= 1;
    if (W > wcap) {
        W = wcap;
        farthr = W - margin;
        if (farthr < 64) return;
    }
    // ---- import lists in CONSUMER order (first step that needs the value): the
    // previous group's rows and the group's own far rows.  An entry a step needs
    // has only entries before it that an earlier-or-equal step needs, all of them
    // produced before that step can run, so the in-order importer cannot deadlock
    std::vector<int> hidx(n, -1), hown(n, -1), gimp_off(K + 1, 0), imp;
    std::vector<char> exported(n, 0);
    int hmax = 0, nfar = 0;
    for (int g = 0; g < K; ++g) {
        gimp_off[g] = int(imp.size());
        int cnt = 0;
        for (int u = gnstart[g]; u < gnstart[g + 1]; ++u) {
            const int id = seq[u];
            bool bad = false;
            for_inputs(id, [&](int src, double) {
                if (node_gid(src) != g) {
                    if (hidx[src] < 0) {
                        hidx[src] = cnt++;
                        exported[src] = 1;
                        imp.push_back(src);
                    }
                } else if (pos[id] - pos[src] > farthr) {
                    if (src >= n) {
                        bad = true;  // (partial nodes sit right before their row: cannot happen)
                    } else if (hown[src] < 0) {
                        hown[src] = cnt++;
                        exported[src] = 1;
                        imp.push_back(src);
                        ++nfar;
                    }
                }
            });
            if (bad) return;
        }
        hmax = std::max(hmax, cnt);
    }
    gimp_off[K] = int(imp.size());
    const int trash_slot = W + 1 + hmax;
    if (8 * trash_slot >= (1 << kLwOwnBits) || hmax >= (1 << (32 - kLwOwnBits))) return;
    int ns = 0;
    for (int t : {8, 6, 4, 3, 2})
        if (t * chb + t * 8 + 64 + (W + 2 + hmax) * 8 <= 225 * 1024) {
            ns = t;
            break;
        }
    if (ns == 0) return;
    // value-area slot of input src of node id in group g
    auto in_slot = [&](int g, int id, int src) {
        if (node_gid(src) != g) return W + 1 + hidx[src];
        if (pos[id] - pos[src] > farthr) return W + 1 + hown[src];
        return pos[src] & (W - 1);
    };
    // ---- steps: a node level's lanes cut into steps of `cap`; groups padded to whole chunks
    std::vector<int2> gch(K);
    int64_t nchunks = 0, nsteps_total = 0;
    for (int g = 0; g < K; ++g) {
        int steps = 0;
        for (int u = gnstart[g], u1; u < gnstart[g + 1]; u = u1) {
            for (u1 = u; u1 < gnstart[g + 1] && node_lev(seq[u1]) == node_lev(seq[u]);) ++u1;
            steps += (u1 - u + cap - 1) / cap;
        }
        const int chunks = (steps + SPC - 1) / SPC;
        gch[g] = make_int2(int(nchunks), chunks);
        nchunks += chunks;
        nsteps_total += steps;
    }
    std::vector<char> prog(size_t(nchunks) * size_t(chb), 0);
    std::vector<long long> coff(n);
    for (int g = 0; g < K; ++g) {
        char* gbase = prog.data() + size_t(gch[g].x) * size_t(chb);
        const int total_steps = gch[g].y * SPC;
        int step = 0;
        auto emit_step = [&](int u0, int u1) {  // nodes seq[u0 .. u1) (possibly none: a padding step)
            char* sbase = gbase + size_t(step) * size_t(stepb);
            for (int w = 0; w < nw; ++w) {
                char* wb = sbase + w * WB;
                int need = 0;
                for (int ln = 0; ln < 32; ++ln) {
                    const int u = u0 + w * 32 + ln;
                    if (u >= u1) break;
                    const int id = seq[u];
                    for_inputs(id, [&](int src, double) {
                        const int sl = in_slot(g, id, src);
                        if (sl > W) need = std::max(need, sl - W);
                    });
                }
                for (int ln = 0; ln < 32; ++ln) {
                    const int u = u0 + w * 32 + ln;
                    double* e = reinterpret_cast<double*>(wb + 16 * ln);  // e[2q], e[2q + 1] at +512 q
                    char* tail = wb + lw_tail(ND) + 16 * ln;
                    auto offp = [&](int d) -> unsigned& {
                        if (ND == 2) return reinterpret_cast<unsigned*>(wb + lw_off(ND) + 8 * ln)[d];
                        return reinterpret_cast<unsigned*>(wb + lw_off(ND) + 512 * (d / 4) + 16 * ln)[d % 4];
                    };
                    auto coef = [&](int d) -> double& { return *(e + (512 / 8) * (d / 2) + (d % 2)); };
                    for (int d = 0; d < ND; ++d) {
                        coef(d) = 0.0;
                        offp(d) = 8u * unsigned(W);
                    }
                    *reinterpret_cast<double*>(tail) = 0.0;
                    int row = -1;
                    unsigned own = 8u * unsigned(trash_slot);
                    if (u < u1) {
                        const int id = seq[u];
                        own = 8u * unsigned(pos[id] & (W - 1));
                        if (id < n) {
                            row = id;
                            coff[id] = int64_t(tail - prog.data()) | (exported[id] ? 1 : 0);
                        }
                        int d = 0;
                        for_inputs(id, [&](int src, double cf) {
                            coef(d) = cf;
                            offp(d) = 8u * unsigned(in_slot(g, id, src));
                            ++d;
                        });
                    }
                    *reinterpret_cast<int*>(tail + 8) = row;
                    *reinterpret_cast<unsigned*>(tail + 12) = own | (unsigned(need) << kLwOwnBits);
                }
            }
            ++step;
        };
        for (int u = gnstart[g], u1; u < gnstart[g + 1]; u = u1) {
            for (u1 = u; u1 < gnstart[g + 1] && node_lev(seq[u1]) == node_lev(seq[u]);) ++u1;
            for (int l0 = u; l0 < u1; l0 += cap) emit_step(l0, std::min(l0 + cap, u1));
        }
        while (step < total_steps) emit_step(0, 0);
    }
    std::vector<int2> gimp(K);
    for (int g = 0; g < K; ++g) gimp[g] = make_int2(gimp_off[g], gimp_off[g + 1] - gimp_off[g]);
    if (getenv("MPREC_LS_TRACE")) {
        int dmax = 0;
        for (int i = 0; i < n; ++i) dmax = std::max(dmax, rlev[i] + 1);
        fprintf(stderr, "[ls lw] n=%d dir=%d K=%d nw=%d ND=%d maxnd=%d mean nd %.2f partial nodes %d node-DAG depth %d "
                        "steps %lld W=%d hmax=%d maxlev=%d far rows %d ns=%d\n",
                n, dir, K, nw, ND, maxnd, double(sumnd) / n, np, dmax, (long long)nsteps_total, W, hmax, maxlev, nfar, ns);
    }
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
    out.nw = nw;
    out.spc = SPC;
    out.chb = chb;
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
    s.nw = b.nw;
    s.spc = b.spc;
    s.chb = b.chb;
    s.smem = b.ns * b.chb + b.ns * 8 + 64 + (b.W + 2 + b.hmax) * 8;
    s.ok = true;
}

// Host copy of a level: one download serves both sweep directions.
struct LsHost {
    int n = 0;
    std::vector<int> rp, ci;
    std::vector<double> v, invd;
};
static void ls_download(Ctx& c, const CsrView& a, const double* invd_dev, LsHost& h) {
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
    c.sync();
}

// Both directions from one download, the two host builds on two threads.
// nd = 0: dependency class from the level, else 2 / 4 / 8.
bool build_ls_pair(Ctx& c, const CsrView& a, const double* invd_dev, int K, int nw, int nd, LsSched& f, LsSched& bw) {
    f = LsSched();
    bw = LsSched();
    if (a.n < 64) return false;
    LsHost h;
    ls_download(c, a, invd_dev, h);
    LsBuilt bf, bb;
    const int ndsel = nd == 2 ? 1 : nd == 4 ? 2 : nd == 8 ? 3 : 0;
    nw = std::min(std::max(nw, 1), 4);  // (kernel instantiations: 1-4 lockstep warps)
    std::thread t([&] { ls_build_lw(h.rp, h.ci, h.v, h.invd, h.n, -1, K, nw, ndsel, bb); });
    ls_build_lw(h.rp, h.ci, h.v, h.invd, h.n, +1, K, nw, ndsel, bf);
    t.join();
    if (!bf.ok || !bb.ok) return false;
    ls_upload(c, bf, f);
    ls_upload(c, bb, bw);
    return true;
}

long long* g_ls_stats = nullptr;  // diagnostics: per-group {start, end, first chunk ns, steps}

template <int ND, int NW>
static void launch_lw(Ctx& c, const LsSched& s, double* xnew) {
    static bool attr = false;
    if (!attr) {
        MG_CUDA(cudaFuncSetAttribute(k_gs_lw<ND, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        attr = true;
    }
    k_gs_lw<ND, NW><<<s.K, (NW + 3) * 32, s.smem, c.s>>>(s.prog.p, s.gch.p, s.imp.p, s.gimp.p, xnew, s.W, s.hmax, s.ns,
                                                        g_ls_stats);
}
template <int ND>
static void launch_lw_nd(Ctx& c, const LsSched& s, double* xnew) {
    switch (s.nw) {
        case 1: launch_lw<ND, 1>(c, s, xnew); break;
        case 2: launch_lw<ND, 2>(c, s, xnew); break;
        case 3: launch_lw<ND, 3>(c, s, xnew); break;
        default: launch_lw<ND, 4>(c, s, xnew); break;
    }
}

void gs_sweep_ls(Ctx& c, const CsrView& a, const double* invd, const double* b, const double* xold, double* xnew,
                 bool xold_zero, const LsSched& s) {
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 4.0 * a.n + 24.0 * a.n;
    Ctx::Scope sc(&c, MPREC_K_GS, bytes);
    k_ls_pre<<<(a.n + 255) / 256, 256, 0, c.s>>>(a.n, a.rp, a.ci, a.v, a.diag, invd, b, xold_zero ? nullptr : xold,
                                                s.dir, s.coff.p, s.prog.p, xnew);
    check_launch("gs ls pre");
    switch (s.cls) {
        case 0: launch_lw_nd<2>(c, s, xnew); break;
        case 1: launch_lw_nd<4>(c, s, xnew); break;
        default: launch_lw_nd<8>(c, s, xnew); break;
    }
    check_launch("gs ls sweep");
}

void gs_level_sweep(Ctx& c, AmgLevel& L, const double* r, const double* xold, double* xnew, int dir, bool zero);

// Diagnostics: build the level-synchronous programs with K groups (MPREC_GS_LS_NW warps, MPREC_GS_LS_ND class) on level l,
// time them against the level's current sweep kernel and compare the results.
// out[0..9] = ms fwd ls, ms bwd ls, ms fwd cur, ms bwd cur, rel err fwd, rel err bwd,
//             W, hmax, steps fwd, build ok (1/0)
void gs_ls_experiment(Ctx& c, Amg& amg, int l, int K, int reps, double* out) {
    AmgLevel& L = *amg.lv[l];
    for (int q = 0; q < 10; ++q) out[q] = 0.0;
    LsSched sf, sb;
    const int nw = getenv("MPREC_GS_LS_NW") ? atoi(getenv("MPREC_GS_LS_NW")) : 1;
    const int nd = getenv("MPREC_GS_LS_ND") ? atoi(getenv("MPREC_GS_LS_ND")) : 0;
    const bool ok = build_ls_pair(c, L.a, L.invd.p, K, nw, nd, sf, sb);
    out[9] = ok ? 1.0 : 0.0;
    if (!ok) return;
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
        fprintf(stderr, "[ls stats] level n=%d K=%d (group: start end first-chunk_us steps chunks)\n", n, sf.K);
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
