// amg_setup_exact.cu -- AMG setup on the device: K7 strength, K8/K9 exact
// Ruge-Stueben C/F splitting, K10 direct interpolation, K11 transpose, K12
// Galerkin SpGEMM, K13 coarsest dense LU + inverse.  Restates
// rs_coarsen / AMGHierarchy::setup (proj/src/amg.cpp:47-214) with results
// bitwise equal to the oracle (file compiled with -fmad=false):
//
//  * strength (amg.cpp:53-68): m_i = max(0, max_{k!=i} -a_ik); j strong iff
//    -a_ij >= theta*m_i; S in CSR order, S^T in ascending row order.
//  * first pass (amg.cpp:70-111): the lazy max-heap on (lambda, -i) with
//    lambda only ever incremented selects, at every step, the undecided node
//    of maximal lambda and lowest index.  It is emulated EXACTLY by one warp
//    over per-lambda hierarchical bitmaps (bucket queue): find the highest
//    non-empty bucket, find-first-set through three bitmap levels, then apply
//    the selection's F-marks and lambda increments with warp-parallel
//    neighbourhood updates (removals and insertions in separate phases so the
//    summary bits stay consistent).  Parallel coarsenings (PMIS/HMIS/CLJP)
//    would change the splitting and are not used.
//  * second/third passes (amg.cpp:113-143) are ascending-i sequential with
//    F->C promotions only.  Promotions can only add C points, so a node that
//    needs no promotion under the current marks never will: a parallel filter
//    finds the candidates, and one warp replays exactly the reference loop on
//    the (few) candidates in ascending order.
//  * interpolation (amg.cpp:145-185) thread per row, same summation order,
//    entries pushed only if w != 0.
//  * Galerkin R(AP) (scalar_matrix.cpp:120-151): per output entry the products
//    are summed from 0.0 in ascending A-column order, symbolic zeros kept.
#include <cub/cub.cuh>
#include <cstdlib>

#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include "mprec.cuh"

namespace mg {
namespace {

enum : signed char { kU = 0, kC = 1, kF = 2 };

// ---------------------------------------------------------------- strength --
__global__ void k_strength_count(const int* rp, const int* ci, const double* v, int n, double theta, double* mrow,
                                 int* scnt, int* stcnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double m = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] != i) {
            const double t = -v[k];
            m = (m < t) ? t : m;  // std::max(m, t)
        }
    mrow[i] = m;
    int cnt = 0;
    if (m > 0.0) {
        const double thr = theta * m;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (j != i && -v[k] >= thr) {
                ++cnt;
                atomicAdd(stcnt + j, 1);
            }
        }
    }
    scnt[i] = cnt;
}

__global__ void k_strength_fill(const int* rp, const int* ci, const double* v, int n, double theta, const double* mrow,
                                const int* srp, int* sci, const int* strp, int* stfill, int* stci) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double m = mrow[i];
    if (!(m > 0.0)) return;
    const double thr = theta * m;
    int o = srp[i];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (j != i && -v[k] >= thr) {
            sci[o++] = j;
            const int pos = atomicAdd(stfill + j, 1);
            stci[strp[j] + pos] = i;
        }
    }
}

// insertion sort of each CSR row by column (carrying optional values)
__global__ void k_sort_rows(const int* rp, int* ci, double* v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = rp[i], b = rp[i + 1];
    for (int p = a + 1; p < b; ++p) {
        const int key = ci[p];
        const double kv = v ? v[p] : 0.0;
        int q = p - 1;
        while (q >= a && ci[q] > key) {
            ci[q + 1] = ci[q];
            if (v) v[q + 1] = v[q];
            --q;
        }
        ci[q + 1] = key;
        if (v) v[q + 1] = kv;
    }
}

// ------------------------------------------------------- RS first pass ------
struct Buckets {
    unsigned long long *l0, *l1, *l2;
    int n0, n1, n2;
    int* cnt;
};

__device__ __forceinline__ void bq_remove(const Buckets& q, int i, int b) {
    const int w0 = i >> 6;
    const unsigned long long bit = 1ull << (i & 63);
    const unsigned long long o0 = atomicAnd(q.l0 + (int64_t)b * q.n0 + w0, ~bit);
    if ((o0 & ~bit) == 0ull) {
        const int w1 = w0 >> 6;
        const unsigned long long bit1 = 1ull << (w0 & 63);
        const unsigned long long o1 = atomicAnd(q.l1 + (int64_t)b * q.n1 + w1, ~bit1);
        if ((o1 & ~bit1) == 0ull) atomicAnd(q.l2 + (int64_t)b * q.n2 + (w1 >> 6), ~(1ull << (w1 & 63)));
    }
    atomicSub(q.cnt + b, 1);
}

__device__ __forceinline__ void bq_insert(const Buckets& q, int i, int b) {
    const int w0 = i >> 6;
    const unsigned long long bit = 1ull << (i & 63);
    const unsigned long long o0 = atomicOr(q.l0 + (int64_t)b * q.n0 + w0, bit);
    if (o0 == 0ull) {
        const int w1 = w0 >> 6;
        const unsigned long long o1 = atomicOr(q.l1 + (int64_t)b * q.n1 + w1, 1ull << (w0 & 63));
        if (o1 == 0ull) atomicOr(q.l2 + (int64_t)b * q.n2 + (w1 >> 6), 1ull << (w1 & 63));
    }
    atomicAdd(q.cnt + b, 1);
}

__global__ void k_rs_init(const int* scnt, const int* stcnt, int n, signed char* mark, int* lam, Buckets q, int* lmax) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int l = stcnt[i];
    lam[i] = l;
    if (scnt[i] == 0 && l == 0) {
        mark[i] = kF;  // unconnected: smoothing handles it alone
        return;
    }
    mark[i] = kU;
    const int w0 = i >> 6;
    atomicOr(q.l0 + (int64_t)l * q.n0 + w0, 1ull << (i & 63));
    atomicAdd(q.cnt + l, 1);
}

__global__ void k_bq_summary(const unsigned long long* lo, unsigned long long* hi, int nlo, int nhi, int nbuckets) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nhi * nbuckets) return;
    const int b = int(t / nhi), w = int(t - (int64_t)b * nhi);
    unsigned long long acc = 0;
    for (int s = 0; s < 64; ++s) {
        const int idx = w * 64 + s;
        if (idx < nlo && lo[(int64_t)b * nlo + idx] != 0ull) acc |= 1ull << s;
    }
    hi[(int64_t)b * nhi + w] = acc;
}

__global__ void k_max_int(const int* a, int n, int* out) {
    int m = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, a[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

constexpr int kRsList = 512;  // per-selection lists kept in smem (overflow spills to global)

// One warp: exact emulation of the lazy-heap greedy (amg.cpp:86-111).
// SMEM: the bucket counts and the two summary levels of the bitmaps live in
// shared memory (copied in at start), so of the per-selection dependent memory
// round trips only the bottom bitmap level and the per-point arrays (mark,
// lambda, increments; L2-resident) go off-chip.  The selection order -- highest
// bucket, lowest index -- and hence the C/F splitting are unchanged.
template <bool SMEM>
__global__ void __launch_bounds__(32) k_rs_select(const int* srp, const int* sci, const int* strp, const int* stci,
                                                  signed char* mark, int* lam, Buckets q, int nbuckets, int* inc,
                                                  int* jlist, int* klist, long long* prof) {
    extern __shared__ unsigned long long bq_sm[];
    long long pf[6] = {0, 0, 0, 0, 0, 0}, tp = clock64(), iters = 0;
#define RS_LAP(k)                          \
    if (prof) {                            \
        const long long tn = clock64();    \
        pf[k] += tn - tp;                  \
        tp = tn;                           \
    }
    const int lane = threadIdx.x;
    __shared__ int nj_sh, nk_sh;
    __shared__ int js0[kRsList], js1[kRsList], kid[kRsList], klam[kRsList];
    if (SMEM) {
        unsigned long long* s1 = bq_sm;
        unsigned long long* s2 = s1 + (size_t)nbuckets * q.n1;
        int* sc = reinterpret_cast<int*>(s2 + (size_t)nbuckets * q.n2);
        for (int t = lane; t < nbuckets * q.n1; t += 32) s1[t] = q.l1[t];
        for (int t = lane; t < nbuckets * q.n2; t += 32) s2[t] = q.l2[t];
        for (int t = lane; t < nbuckets; t += 32) sc[t] = q.cnt[t];
        q.l1 = s1;
        q.l2 = s2;
        q.cnt = sc;
        __syncwarp();
    }
    int hi = nbuckets - 1;
    for (;;) {
        // highest non-empty bucket
        for (;;) {
            const int b = hi - lane;
            const bool ne = b >= 0 && ((volatile int*)q.cnt)[b] > 0;
            const unsigned bal = __ballot_sync(0xffffffffu, ne);
            if (bal) {
                hi -= __ffs(bal) - 1;
                break;
            }
            hi -= 32;
            if (hi < 0) break;
        }
        if (hi < 0) {
            if (prof && lane == 0) {
                for (int k = 0; k < 6; ++k) prof[k] = pf[k];
                prof[6] = iters;
            }
            return;
        }
        ++iters;
        // lowest index in bucket hi: first non-zero top-level word
        int first = 0x7fffffff;
        for (int w = lane; w < q.n2; w += 32)
            if (((volatile unsigned long long*)q.l2)[(int64_t)hi * q.n2 + w] != 0ull) {
                first = w;
                break;
            }
        for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        int i = 0;
        if (lane == 0) {
            const unsigned long long x2 = ((volatile unsigned long long*)q.l2)[(int64_t)hi * q.n2 + first];
            const int w1 = first * 64 + __ffsll((long long)x2) - 1;
            const unsigned long long x1 = ((volatile unsigned long long*)q.l1)[(int64_t)hi * q.n1 + w1];
            const int w0 = w1 * 64 + __ffsll((long long)x1) - 1;
            const unsigned long long x0 = ((volatile unsigned long long*)q.l0)[(int64_t)hi * q.n0 + w0];
            i = w0 * 64 + __ffsll((long long)x0) - 1;
            mark[i] = kC;
            bq_remove(q, i, hi);
            nj_sh = 0;
            nk_sh = 0;
        }
        i = __shfl_sync(0xffffffffu, i, 0);
        __syncwarp();
        RS_LAP(0)
        // phase d: undecided j in S^T_i become F.  The loads a later phase needs
        // (lambda_j, the bounds of S_j) are issued together with mark[j].
        {
            const int a0 = strp[i], a1 = strp[i + 1];
            for (int jj = a0 + lane; jj < a1; jj += 32) {
                const int j = stci[jj];
                const signed char mj = ((volatile signed char*)mark)[j];
                const int lj = lam[j], s0 = srp[j], s1 = srp[j + 1];
                if (mj == kU) {
                    mark[j] = kF;
                    bq_remove(q, j, lj);
                    const int t = atomicAdd(&nj_sh, 1);
                    if (t < kRsList) {
                        js0[t] = s0;
                        js1[t] = s1;
                    } else {
                        jlist[2 * (t - kRsList)] = s0;
                        jlist[2 * (t - kRsList) + 1] = s1;
                    }
                }
            }
        }
        __syncwarp();
        RS_LAP(1)
        const int nj = ((volatile int*)&nj_sh)[0];
        // phase e1: count the increments of every undecided k in S_j; 4 rows at a
        // time, 8 lanes per row (the rows' memory round trips overlap)
        {
            const int grp = lane >> 3, sub = lane & 7;
            for (int t0 = 0; t0 < nj; t0 += 4) {
                const int t = t0 + grp;
                if (t < nj) {
                    const int s0 = t < kRsList ? js0[t] : jlist[2 * (t - kRsList)];
                    const int s1 = t < kRsList ? js1[t] : jlist[2 * (t - kRsList) + 1];
                    for (int kk = s0 + sub; kk < s1; kk += 8) {
                        const int k = sci[kk];
                        const signed char mk = ((volatile signed char*)mark)[k];
                        const int lk = lam[k];
                        if (mk == kU && atomicAdd(inc + k, 1) == 0) {
                            const int u = atomicAdd(&nk_sh, 1);
                            if (u < kRsList) {
                                kid[u] = k;
                                klam[u] = lk;
                            } else {
                                klist[2 * (u - kRsList)] = k;
                                klist[2 * (u - kRsList) + 1] = lk;
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
        RS_LAP(2)
        const int nk = ((volatile int*)&nk_sh)[0];
        // phase e2: removals (all), then insertions at the incremented lambda; a
        // removal and an insertion may share a bitmap word, hence two phases
        int mx = -1;
        int k0 = 0, lk0 = 0, ik0 = 0;  // first 32 candidates stay in registers
        for (int t = lane; t < nk; t += 32) {
            const int k = t < kRsList ? kid[t] : klist[2 * (t - kRsList)];
            const int lk = t < kRsList ? klam[t] : klist[2 * (t - kRsList) + 1];
            if (t < 32) {
                k0 = k;
                lk0 = lk;
                ik0 = ((volatile int*)inc)[k];  // overlaps the removal below
            }
            bq_remove(q, k, lk);
        }
        __syncwarp();
        RS_LAP(3)
        for (int t = lane; t < nk; t += 32) {
            int k = k0, lk = lk0, ik = ik0;
            if (t >= 32) {
                k = t < kRsList ? kid[t] : klist[2 * (t - kRsList)];
                lk = t < kRsList ? klam[t] : klist[2 * (t - kRsList) + 1];
                ik = ((volatile int*)inc)[k];
            }
            const int nl = lk + ik;
            inc[k] = 0;
            lam[k] = nl;
            bq_insert(q, k, nl);
            mx = max(mx, nl);
        }
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        hi = max(hi, mx);
        __syncwarp();
        RS_LAP(4)
    }
#undef RS_LAP
}

// Two-hop adjacency records for the windowed first pass.  A selection of point i
// walks S^T_i and, for every j in it that becomes F, S_j: four dependent loads
// (row pointer -> column list, twice) at L2 latency.  The record of i holds all of
// it -- [0] = |S^T_i|, then per j a block {j, |S_j|, S_j padded to maxS} -- in
// one fixed-size, 128-byte-aligned run (1-4 cache lines, fetched in one round
// trip right after the selection is known).  Levels whose record would exceed
// kRsRecMax ints keep the CSR walk.
constexpr int kRsRecMax = 128;
__global__ void k_rs_records(const int* __restrict__ srp, const int* __restrict__ sci, const int* __restrict__ strp,
                             const int* __restrict__ stci, int n, int B, int RW, int* __restrict__ rec) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int* r = rec + (int64_t)RW * i;
    const int t0 = strp[i], nt = strp[i + 1] - t0;
    r[0] = nt;
    for (int t = 0; t < nt; ++t) {
        const int j = stci[t0 + t], s0 = srp[j], ns = srp[j + 1] - s0;
        int* blk = r + 1 + t * B;
        blk[0] = j;
        blk[1] = ns;
        for (int u = 0; u < ns; ++u) blk[2 + u] = sci[s0 + u];
    }
}

// ---------------------------------------------------------------------------
// Windowed variant of the one-warp greedy.  The selections follow a front (on
// the c4 / c5 levels 98 % of consecutive C points lie within three grid lines),
// and every selection made ~10 dependent L2 round trips (~800 cycles each) on
// the per-point state.  Here the MUTABLE state of a window of WN consecutive
// points around the front -- mark, lambda, the per-selection increment counters
// and the bottom bitmap level of every bucket -- lives in shared memory; the
// window slides with the front (write back, reload: every few thousand
// selections).  Points outside the window are still served from global memory,
// so any selection order is handled; the order itself -- highest bucket, lowest
// index -- and hence the C/F splitting are unchanged.  The read-only strength
// graph goes through the L1 (ld.global.nc): consecutive selections share its
// cache lines.
struct RsWin {
    int wb, wn;                 // window [wb, wb + wn), wb % 64 == 0
    unsigned char* lm;          // [WN] lambda
    unsigned char* st;          // [WN] mark (2 bits) | per-selection increment counter << 2
    unsigned long long* l0;     // [nbuckets][WN / 64]
    int w64;                    // WN / 64
    // shared-space addresses (explicit atom.shared / red.shared: a generic-address
    // atomic that lands in shared memory costs several hundred cycles)
    unsigned l0_a, ic_a, s1_a, s2_a, cnt_a;
};

__device__ __forceinline__ unsigned sm_and32(unsigned a, unsigned v) {
    unsigned o;
    asm volatile("atom.shared.and.b32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ unsigned sm_or32(unsigned a, unsigned v) {
    unsigned o;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ unsigned sm_add32(unsigned a, unsigned v) {
    unsigned o;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ void sm_red_add(unsigned a, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned sm_ld32(unsigned a) {
    unsigned o;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(o) : "r"(a) : "memory");
    return o;
}

__device__ __forceinline__ bool rw_in(const RsWin& w, int x) { return unsigned(x - w.wb) < unsigned(w.wn); }

__device__ __forceinline__ signed char rw_mark(const RsWin& w, const signed char* mark, int x) {
    return rw_in(w, x) ? (signed char)(((volatile unsigned char*)w.st)[x - w.wb] & 3)
                       : ((volatile const signed char*)mark)[x];
}
// (only between selections' counting phases: the point's counter is zero)
__device__ __forceinline__ void rw_set_mark(const RsWin& w, signed char* mark, int x, signed char v) {
    if (rw_in(w, x))
        ((volatile unsigned char*)w.st)[x - w.wb] = (unsigned char)v;
    else
        mark[x] = v;
}
__device__ __forceinline__ int rw_lam(const RsWin& w, const int* lam, int x) {
    return rw_in(w, x) ? int(((volatile unsigned char*)w.lm)[x - w.wb]) : ((volatile const int*)lam)[x];
}
__device__ __forceinline__ void rw_set_lam(const RsWin& w, int* lam, int x, int v) {
    if (rw_in(w, x))
        ((volatile unsigned char*)w.lm)[x - w.wb] = (unsigned char)v;
    else
        lam[x] = v;
}
// fetch-and-increment of the per-selection counter of x (old value)
__device__ __forceinline__ int rw_inc_add(const RsWin& w, int* inc, int x) {
    if (rw_in(w, x)) {
        const int o = x - w.wb, sh = 8 * (o & 3);
        return int((sm_add32(w.ic_a + 4u * unsigned(o >> 2), 4u << sh) >> (sh + 2)) & 0x3fu);
    }
    return atomicAdd(inc + x, 1);
}
// read and clear
__device__ __forceinline__ int rw_inc_take(const RsWin& w, int* inc, int x) {
    if (rw_in(w, x)) {
        const int o = x - w.wb, sh = 8 * (o & 3);
        return int((sm_and32(w.ic_a + 4u * unsigned(o >> 2), ~(0xfcu << sh)) >> (sh + 2)) & 0x3fu);
    }
    const int v = ((volatile int*)inc)[x];
    inc[x] = 0;
    return v;
}
// summary levels (shared memory): clear / set the bit of bottom word w0 in bucket b.
// Idempotent, so a redundant call is harmless.
__device__ __forceinline__ void rw_sum_clear(const RsWin& w, const Buckets& q, int w0, int b) {
    const int w1 = w0 >> 6;
    const unsigned a1 = w.s1_a + 8u * unsigned(b * q.n1 + w1) + 4u * unsigned((w0 >> 5) & 1);
    const unsigned n1 = sm_and32(a1, ~(1u << (w0 & 31))) & ~(1u << (w0 & 31));
    if (n1 == 0u && sm_ld32(a1 ^ 4u) == 0u)
        sm_and32(w.s2_a + 8u * unsigned(b * q.n2 + (w1 >> 6)) + 4u * unsigned((w1 >> 5) & 1), ~(1u << (w1 & 31)));
}
__device__ __forceinline__ void rw_sum_set(const RsWin& w, const Buckets& q, int w0, int b) {
    const int w1 = w0 >> 6;
    const unsigned a1 = w.s1_a + 8u * unsigned(b * q.n1 + w1) + 4u * unsigned((w0 >> 5) & 1);
    if (sm_or32(a1, 1u << (w0 & 31)) == 0u)
        sm_or32(w.s2_a + 8u * unsigned(b * q.n2 + (w1 >> 6)) + 4u * unsigned((w1 >> 5) & 1), 1u << (w1 & 31));
}
__device__ __forceinline__ void rw_remove(const RsWin& w, const Buckets& q, int i, int b) {
    const int w0 = i >> 6;
    if (rw_in(w, i)) {
        // the 64-bit bottom word as two 32-bit halves: whoever empties a half looks at
        // the other one (lanes run their atomics before their loads, so at least one
        // lane sees the word empty)
        const unsigned a = w.l0_a + 8u * unsigned(b * w.w64 + ((i - w.wb) >> 6)) + 4u * unsigned((i >> 5) & 1);
        const unsigned bit = 1u << (i & 31);
        if ((sm_and32(a, ~bit) & ~bit) == 0u && sm_ld32(a ^ 4u) == 0u) rw_sum_clear(w, q, w0, b);
    } else {
        const unsigned long long bit = 1ull << (i & 63);
        const unsigned long long o0 = atomicAnd(q.l0 + (int64_t)b * q.n0 + w0, ~bit);
        if ((o0 & ~bit) == 0ull) rw_sum_clear(w, q, w0, b);
    }
    sm_red_add(w.cnt_a + 4u * unsigned(b), -1);
}
__device__ __forceinline__ void rw_insert(const RsWin& w, const Buckets& q, int i, int b) {
    const int w0 = i >> 6;
    if (rw_in(w, i)) {
        const unsigned a = w.l0_a + 8u * unsigned(b * w.w64 + ((i - w.wb) >> 6)) + 4u * unsigned((i >> 5) & 1);
        if (sm_or32(a, 1u << (i & 31)) == 0u) rw_sum_set(w, q, w0, b);
    } else {
        if (atomicOr(q.l0 + (int64_t)b * q.n0 + w0, 1ull << (i & 63)) == 0ull) rw_sum_set(w, q, w0, b);
    }
    sm_red_add(w.cnt_a + 4u * unsigned(b), 1);
}

// Window move, all kRsWinThreads threads of the block (the helper warps sleep on a
// named barrier between moves): write the old window back, then load the new one.
constexpr int kRsWinThreads = 1024;  // one selecting warp + 31 warps that only move the window
__device__ __forceinline__ void rw_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kRsWinThreads) : "memory"); }

__device__ void rw_move(unsigned char* st, unsigned char* lm, unsigned long long* wl0, int w64, const Buckets& q,
                        signed char* mark, int* lam, int n, int WN, int nbuckets, int owb, int own, int nwb, int tid) {
    // ---- flush [owb, owb + own)
    if (own > 0) {
        const int own4 = own & ~3;
        for (int t = 4 * tid; t < own4; t += 4 * kRsWinThreads) {
            const unsigned s4 = *reinterpret_cast<const unsigned*>(st + t), l4 = *reinterpret_cast<const unsigned*>(lm + t);
            *reinterpret_cast<unsigned*>(mark + owb + t) = s4 & 0x03030303u;
            *reinterpret_cast<int4*>(lam + owb + t) =
                make_int4(int(l4 & 0xffu), int((l4 >> 8) & 0xffu), int((l4 >> 16) & 0xffu), int(l4 >> 24));
        }
        for (int t = own4 + tid; t < own; t += kRsWinThreads) {
            mark[owb + t] = (signed char)(st[t] & 3);
            lam[owb + t] = int(lm[t]);
        }
        const int words = (own + 63) >> 6;
        for (int t = tid; t < nbuckets * words; t += kRsWinThreads) {
            const int b = t / words, x = t - b * words;
            q.l0[(int64_t)b * q.n0 + (owb >> 6) + x] = wl0[b * w64 + x];
        }
        __threadfence();
    }
    rw_bar(3);
    // ---- load [nwb, nwb + nwn)
    if (nwb >= 0) {
        const int nwn = min(WN, n - nwb), nwn4 = nwn & ~3;
        for (int t = 4 * tid; t < nwn4; t += 4 * kRsWinThreads) {
            const unsigned m4 = *reinterpret_cast<volatile const unsigned*>(mark + nwb + t);
            const volatile int* lp = lam + nwb + t;
            const int l0v = lp[0], l1v = lp[1], l2v = lp[2], l3v = lp[3];
            *reinterpret_cast<unsigned*>(st + t) = m4;
            *reinterpret_cast<unsigned*>(lm + t) =
                unsigned(l0v & 0xff) | (unsigned(l1v & 0xff) << 8) | (unsigned(l2v & 0xff) << 16) | (unsigned(l3v & 0xff) << 24);
        }
        for (int t = nwn4 + tid; t < nwn; t += kRsWinThreads) {
            st[t] = (unsigned char)((volatile const signed char*)mark)[nwb + t];
            lm[t] = (unsigned char)((volatile const int*)lam)[nwb + t];
        }
        const int words = (nwn + 63) >> 6;
        for (int t = tid; t < nbuckets * words; t += kRsWinThreads) {
            const int b = t / words, x = t - b * words;
            wl0[b * w64 + x] = ((volatile const unsigned long long*)q.l0)[(int64_t)b * q.n0 + (nwb >> 6) + x];
        }
    }
}

__global__ void __launch_bounds__(kRsWinThreads) k_rs_select_win(const int* __restrict__ srp, const int* __restrict__ sci,
                                                      const int* __restrict__ strp, const int* __restrict__ stci,
                                                      signed char* mark, int* lam, Buckets q, int nbuckets, int* inc,
                                                      int* jlist, int* klist, int n, int WN, long long* prof,
                                                      const int* __restrict__ rec, int recB, int recW) {
    extern __shared__ unsigned long long bq_sm[];
    long long pf[6] = {0, 0, 0, 0, 0, 0}, tp = clock64(), iters = 0, slides = 0, outside = 0;
#define RS_LAP(k)                          \
    if (prof) {                            \
        const long long tn = clock64();    \
        pf[k] += tn - tp;                  \
        tp = tn;                           \
    }
    const int lane = threadIdx.x & 31, tid = threadIdx.x;
    __shared__ int nj_sh, nk_sh;
    __shared__ int cmd[3];  // window move: old base, old size, new base (-1: none, the kernel ends)
    __shared__ int js0[kRsList], js1[kRsList], kid[kRsList], klam[kRsList];
    __shared__ int recs[kRsRecMax], newlist[32];
    // shared memory: summary levels + counts (as k_rs_select<true>), then the window
    unsigned long long* s1 = bq_sm;
    unsigned long long* s2 = s1 + (size_t)nbuckets * q.n1;
    unsigned long long* wl0 = s2 + (size_t)nbuckets * q.n2;
    int* sc = reinterpret_cast<int*>(wl0 + (size_t)nbuckets * (WN / 64));
    unsigned char* wst = reinterpret_cast<unsigned char*>(sc + ((nbuckets + 3) & ~3));
    unsigned char* wlm = wst + WN;
    for (int t = tid; t < nbuckets * q.n1; t += kRsWinThreads) s1[t] = q.l1[t];
    for (int t = tid; t < nbuckets * q.n2; t += kRsWinThreads) s2[t] = q.l2[t];
    for (int t = tid; t < nbuckets; t += kRsWinThreads) sc[t] = q.cnt[t];
    q.l1 = s1;
    q.l2 = s2;
    q.cnt = sc;
    rw_move(wst, wlm, wl0, WN / 64, q, mark, lam, n, WN, nbuckets, 0, 0, 0, tid);
    __syncthreads();
    if (tid >= 32) {  // helper warps: asleep on barrier 1 until the selecting warp moves the window
        for (;;) {
            rw_bar(1);
            const int owb = ((volatile int*)cmd)[0], own = ((volatile int*)cmd)[1], nwb = ((volatile int*)cmd)[2];
            rw_move(wst, wlm, wl0, WN / 64, q, mark, lam, n, WN, nbuckets, owb, own, nwb, tid);
            rw_bar(2);
            if (nwb < 0) return;
        }
    }
    RsWin w;
    w.st = wst;
    w.lm = wlm;
    w.l0 = wl0;
    w.w64 = WN / 64;
    w.l0_a = (unsigned)__cvta_generic_to_shared(wl0);
    w.ic_a = (unsigned)__cvta_generic_to_shared(wst);
    w.s1_a = (unsigned)__cvta_generic_to_shared(s1);
    w.s2_a = (unsigned)__cvta_generic_to_shared(s2);
    w.cnt_a = (unsigned)__cvta_generic_to_shared(sc);
    w.wb = 0;
    w.wn = min(WN, n);
    auto move_window = [&](int nwb) {  // all lanes of the selecting warp
        __syncwarp();
        if (lane == 0) {
            cmd[0] = w.wb;
            cmd[1] = w.wn;
            cmd[2] = nwb;
        }
        __syncwarp();
        rw_bar(1);
        rw_move(wst, wlm, wl0, WN / 64, q, mark, lam, n, WN, nbuckets, w.wb, w.wn, nwb, tid);
        rw_bar(2);
        if (nwb >= 0) {
            w.wb = nwb;
            w.wn = min(WN, n - nwb);
        }
    };
    // the window keeps 5/8 of its points behind the selection when it moves (the
    // selections of the c5 levels hop between ~6 grid lines around a front) and
    // moves when the selection reaches its last 1/20, or lies outside 16 times
    // in a row (isolated far selections are served from global memory)
    const int back = (WN / 8) * 5;
    int hi = nbuckets - 1, miss = 0;
    for (;;) {
        // highest non-empty bucket
        for (;;) {
            const int b = hi - lane;
            const bool ne = b >= 0 && ((volatile int*)q.cnt)[b] > 0;
            const unsigned bal = __ballot_sync(0xffffffffu, ne);
            if (bal) {
                hi -= __ffs(bal) - 1;
                break;
            }
            hi -= 32;
            if (hi < 0) break;
        }
        if (hi < 0) break;
        ++iters;
        // lowest index in bucket hi: first non-zero top-level word (one ballot while
        // the top level has <= 32 words, i.e. up to 8M points), then the descent on
        // every lane (same addresses: broadcasts; no shuffle of the result)
        int first = 0x7fffffff;
        const unsigned long long* l2b = q.l2 + (int64_t)hi * q.n2;
        if (q.n2 <= 32) {
            const bool nz = lane < q.n2 && ((volatile const unsigned long long*)l2b)[lane] != 0ull;
            first = __ffs(__ballot_sync(0xffffffffu, nz)) - 1;
        } else {
            for (int t = lane; t < q.n2; t += 32)
                if (((volatile const unsigned long long*)l2b)[t] != 0ull) {
                    first = t;
                    break;
                }
            for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        }
        int i;
        {
            const unsigned long long x2 = ((volatile const unsigned long long*)l2b)[first];
            const int w1 = first * 64 + __ffsll((long long)x2) - 1;
            const unsigned long long x1 = ((volatile unsigned long long*)q.l1)[(int64_t)hi * q.n1 + w1];
            const int w0 = w1 * 64 + __ffsll((long long)x1) - 1;
            const unsigned long long x0 =
                rw_in(w, w0 * 64) ? ((volatile unsigned long long*)w.l0)[hi * w.w64 + ((w0 * 64 - w.wb) >> 6)]
                                  : ((volatile unsigned long long*)q.l0)[(int64_t)hi * q.n0 + w0];
            i = w0 * 64 + __ffsll((long long)x0) - 1;
        }
        // move the window with the front: when the selection runs into the last
        // quarter, or lies outside twice in a row (an isolated far selection is
        // served from global memory)
        {
            const bool in = rw_in(w, i);
            const bool tail = in && i - w.wb > WN - WN / 20 && w.wb + WN < n;
            miss = in ? 0 : miss + 1;
            if (!in) ++outside;
            if (tail || miss >= 16) {
                move_window(max(0, (i - back) & ~63));
                miss = 0;
                ++slides;
            }
        }
        int rw0 = 0, rw1 = 0, rw2 = 0, rw3 = 0;  // the selection's two-hop record (in flight during lane 0's work)
        if (rec) {
            const int* rp_ = rec + (int64_t)recW * i + lane;
            rw0 = __ldg(rp_);
            if (recW > 32) rw1 = __ldg(rp_ + 32);
            if (recW > 64) rw2 = __ldg(rp_ + 64);
            if (recW > 96) rw3 = __ldg(rp_ + 96);
        }
        if (lane == 0) {
            rw_set_mark(w, mark, i, kC);
            rw_remove(w, q, i, hi);
            nj_sh = 0;
            nk_sh = 0;
        }
        __syncwarp();
        RS_LAP(0)
        if (rec) {
            recs[lane] = rw0;
            if (recW > 32) recs[32 + lane] = rw1;
            if (recW > 64) recs[64 + lane] = rw2;
            if (recW > 96) recs[96 + lane] = rw3;
            __syncwarp();
            // phase d: undecided j in S^T_i become F (one lane per j; |S^T_i| <= 32 here)
            const int nst = ((volatile int*)recs)[0];
            bool newf = false;
            if (lane < nst) {
                const int j = ((volatile int*)recs)[1 + lane * recB];
                if (rw_mark(w, mark, j) == kU) {
                    const int lj = rw_lam(w, lam, j);
                    rw_set_mark(w, mark, j, kF);
                    rw_remove(w, q, j, lj);
                    newf = true;
                }
            }
            const unsigned nm = __ballot_sync(0xffffffffu, newf);
            if (newf) newlist[__popc(nm & ((1u << lane) - 1))] = lane;
            const int nnew = __popc(nm);
            __syncwarp();
            RS_LAP(1)
            // phase e1: count the increments of every undecided k in S_j of the new F
            // points: MS lanes per j (MS = power of two >= maxS), 32 / MS points a round
            const int maxs = recB - 2;
            const int ms = maxs <= 4 ? 4 : maxs <= 8 ? 8 : maxs <= 16 ? 16 : 32;
            const int per = 32 / ms, sub = lane % ms, slot = lane / ms;
            for (int r0 = 0; r0 < nnew; r0 += per) {
                const int sidx = r0 + slot;
                if (sidx < nnew) {
                    const int t = ((volatile int*)newlist)[sidx];
                    const int ns = ((volatile int*)recs)[2 + t * recB];
                    if (sub < ns) {
                        const int k = ((volatile int*)recs)[3 + t * recB + sub];
                        if (rw_mark(w, mark, k) == kU && rw_inc_add(w, inc, k) == 0) {
                            const int lk = rw_lam(w, lam, k);
                            const int u = atomicAdd(&nk_sh, 1);
                            if (u < kRsList) {
                                kid[u] = k;
                                klam[u] = lk;
                            } else {
                                klist[2 * (u - kRsList)] = k;
                                klist[2 * (u - kRsList) + 1] = lk;
                            }
                        }
                    }
                }
            }
            __syncwarp();
            RS_LAP(2)
        } else {
        // phase d: undecided j in S^T_i become F
        {
            const int a0 = __ldg(strp + i), a1 = __ldg(strp + i + 1);
            for (int jj = a0 + lane; jj < a1; jj += 32) {
                const int j = __ldg(stci + jj);
                const signed char mj = rw_mark(w, mark, j);
                if (mj == kU) {
                    const int lj = rw_lam(w, lam, j), s0 = __ldg(srp + j), s1e = __ldg(srp + j + 1);
                    rw_set_mark(w, mark, j, kF);
                    rw_remove(w, q, j, lj);
                    const int t = atomicAdd(&nj_sh, 1);
                    if (t < kRsList) {
                        js0[t] = s0;
                        js1[t] = s1e;
                    } else {
                        jlist[2 * (t - kRsList)] = s0;
                        jlist[2 * (t - kRsList) + 1] = s1e;
                    }
                }
            }
        }
        __syncwarp();
        RS_LAP(1)
        const int nj = ((volatile int*)&nj_sh)[0];
        // phase e1: count the increments of every undecided k in S_j; 4 rows at a
        // time, 8 lanes per row
        {
            const int grp = lane >> 3, sub = lane & 7;
            for (int t0 = 0; t0 < nj; t0 += 4) {
                const int t = t0 + grp;
                if (t < nj) {
                    const int s0 = t < kRsList ? js0[t] : jlist[2 * (t - kRsList)];
                    const int s1e = t < kRsList ? js1[t] : jlist[2 * (t - kRsList) + 1];
                    for (int kk = s0 + sub; kk < s1e; kk += 8) {
                        const int k = __ldg(sci + kk);
                        if (rw_mark(w, mark, k) == kU && rw_inc_add(w, inc, k) == 0) {
                            const int lk = rw_lam(w, lam, k);
                            const int u = atomicAdd(&nk_sh, 1);
                            if (u < kRsList) {
                                kid[u] = k;
                                klam[u] = lk;
                            } else {
                                klist[2 * (u - kRsList)] = k;
                                klist[2 * (u - kRsList) + 1] = lk;
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
        RS_LAP(2)
        }
        const int nk = ((volatile int*)&nk_sh)[0];
        // phase e2: removals (all), then insertions at the incremented lambda; a
        // removal and an insertion may share a bitmap word, hence two phases
        for (int t = lane; t < nk; t += 32) {
            const int k = t < kRsList ? kid[t] : klist[2 * (t - kRsList)];
            const int lk = t < kRsList ? klam[t] : klist[2 * (t - kRsList) + 1];
            rw_remove(w, q, k, lk);
        }
        __syncwarp();
        RS_LAP(3)
        int mx = -1;
        for (int t = lane; t < nk; t += 32) {
            const int k = t < kRsList ? kid[t] : klist[2 * (t - kRsList)];
            const int lk = t < kRsList ? klam[t] : klist[2 * (t - kRsList) + 1];
            const int nl = lk + rw_inc_take(w, inc, k);
            rw_set_lam(w, lam, k, nl);
            rw_insert(w, q, k, nl);
            mx = max(mx, nl);
        }
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        hi = max(hi, mx);
        __syncwarp();
        RS_LAP(4)
    }
    move_window(-1);  // write back; the helper warps leave
    if (prof && lane == 0) {
        for (int k = 0; k < 6; ++k) prof[k] = pf[k];
        prof[6] = iters;
        prof[7] = slides * 1000000ll + outside;
    }
#undef RS_LAP
}

// --------------------------------------------- RS second and third passes --
__device__ __forceinline__ bool in_row(const int* sci, int a, int b, int key) {
    while (a < b) {
        const int m = (a + b) >> 1;
        const int v = sci[m];
        if (v == key) return true;
        if (v < key)
            a = m + 1;
        else
            b = m;
    }
    return false;
}

// candidates of the second pass: F with S_i != {} that would promote now
__global__ void k_rs2_cand(const int* srp, const int* sci, const signed char* mark, int n, int* flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int need = 0;
    if (mark[i] == kF && srp[i + 1] > srp[i]) {
        const int a = srp[i], b = srp[i + 1];
        for (int p = a; p < b && !need; ++p) {
            const int j = sci[p];
            if (mark[j] != kF) continue;
            bool shared = false;
            for (int kk = srp[j]; kk < srp[j + 1]; ++kk) {
                const int k = sci[kk];
                if (mark[k] == kC && in_row(sci, a, b, k)) {
                    shared = true;
                    break;
                }
            }
            if (!shared) need = 1;
        }
    }
    flag[i] = need;
}

// S_i is sorted ascending (CSR order of a canonical matrix), so `in_row` works.
__global__ void __launch_bounds__(32) k_rs2_seq(const int* srp, const int* sci, signed char* mark, const int* cand,
                                                int ncand) {
    const int lane = threadIdx.x;
    __shared__ int cil[4096];
    __shared__ int ncil;
    for (int t = 0; t < ncand; ++t) {
        const int i = cand[t];
        if (((volatile signed char*)mark)[i] != kF) continue;
        const int a = srp[i], b = srp[i + 1];
        if (lane == 0) ncil = 0;
        __syncwarp();
        for (int p = a + lane; p < b; p += 32) {
            const int j = sci[p];
            if (((volatile signed char*)mark)[j] == kC) {
                const int pos = atomicAdd(&ncil, 1);
                if (pos < 4096) cil[pos] = j;
            }
        }
        __syncwarp();
        for (int p = a; p < b; ++p) {
            const int j = sci[p];
            if (((volatile signed char*)mark)[j] != kF) continue;
            const int nci = min(((volatile int*)&ncil)[0], 4096);
            bool shared = false;
            const int ja = srp[j], jb = srp[j + 1];
            for (int kk = ja + lane; kk < jb && !shared; kk += 32) {
                const int k = sci[kk];
                for (int e = 0; e < nci; ++e)
                    if (((volatile int*)cil)[e] == k) {
                        shared = true;
                        break;
                    }
            }
            shared = __any_sync(0xffffffffu, shared);
            if (!shared && lane == 0) {
                mark[j] = kC;
                const int pos = ncil;
                if (pos < 4096) cil[pos] = j;
                ncil = pos + 1;
            }
            __syncwarp();
        }
        __syncwarp();
    }
}

// Windowed replay of the second pass: the candidates come in increasing index
// order and every access lies within two rows' reach of the candidate, so the
// marks (the only mutable state) of a window of kRs2Win points that moves
// forward with the candidates live in shared memory; accesses outside the window
// (none on the c5 levels) go to global memory.  Same decisions as k_rs2_seq.
constexpr int kRs2Win = 128 * 1024, kRs2Threads = 256;
__device__ __forceinline__ void rs2_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kRs2Threads) : "memory"); }

__device__ void rs2_move(unsigned char* wm, signed char* mark, int n, int owb, int own, int nwb, int tid) {
    if (own > 0) {
        const int own4 = own & ~3;
        for (int t = 4 * tid; t < own4; t += 4 * kRs2Threads)
            *reinterpret_cast<unsigned*>(mark + owb + t) = *reinterpret_cast<const unsigned*>(wm + t);
        for (int t = own4 + tid; t < own; t += kRs2Threads) mark[owb + t] = (signed char)wm[t];
        __threadfence();
    }
    rs2_bar(3);
    if (nwb >= 0) {
        const int nwn = min(kRs2Win, n - nwb), nwn4 = nwn & ~3;
        for (int t = 4 * tid; t < nwn4; t += 4 * kRs2Threads)
            *reinterpret_cast<unsigned*>(wm + t) = *reinterpret_cast<volatile const unsigned*>(mark + nwb + t);
        for (int t = nwn4 + tid; t < nwn; t += kRs2Threads) wm[t] = (unsigned char)((volatile signed char*)mark)[nwb + t];
    }
}

template <int PASS>
__global__ void __launch_bounds__(kRs2Threads) k_rs2_seq_win(const int* __restrict__ srp, const int* __restrict__ sci,
                                                             signed char* mark, const int* __restrict__ cand, int ncand,
                                                             int n, const int* __restrict__ rec, int recB, int recW) {
    extern __shared__ unsigned char rs2_sm[];
    unsigned char* wm = rs2_sm;
    const int lane = threadIdx.x & 31, tid = threadIdx.x;
    __shared__ int cil[4096];
    __shared__ int ncil;
    __shared__ int cmd[3];
    __shared__ int recs[kRsRecMax];
    int wb = max(0, (cand[0] - kRs2Win / 4) & ~63), wn = min(kRs2Win, n - wb);
    rs2_move(wm, mark, n, 0, 0, wb, tid);
    __syncthreads();
    if (tid >= 32) {
        for (;;) {
            rs2_bar(1);
            const int owb = ((volatile int*)cmd)[0], own = ((volatile int*)cmd)[1], nwb = ((volatile int*)cmd)[2];
            rs2_move(wm, mark, n, owb, own, nwb, tid);
            rs2_bar(2);
            if (nwb < 0) return;
        }
    }
    auto move_window = [&](int nwb) {
        __syncwarp();
        if (lane == 0) {
            cmd[0] = wb;
            cmd[1] = wn;
            cmd[2] = nwb;
        }
        __syncwarp();
        rs2_bar(1);
        rs2_move(wm, mark, n, wb, wn, nwb, tid);
        rs2_bar(2);
        if (nwb >= 0) {
            wb = nwb;
            wn = min(kRs2Win, n - nwb);
        }
    };
    auto get = [&](int x) -> signed char {
        return unsigned(x - wb) < unsigned(wn) ? (signed char)((volatile unsigned char*)wm)[x - wb]
                                              : ((volatile signed char*)mark)[x];
    };
    auto set_c = [&](int x) {
        if (unsigned(x - wb) < unsigned(wn))
            ((volatile unsigned char*)wm)[x - wb] = (unsigned char)kC;
        else
            mark[x] = kC;
    };
    int pw0 = 0, pw1 = 0, pw2 = 0, pw3 = 0;  // prefetched record words (pass 2)
    for (int t = 0; t < ncand; ++t) {
        const int i = __ldg(cand + t);
        if (i - wb > kRs2Win - kRs2Win / 4 && wb + kRs2Win < n) move_window(max(0, (i - kRs2Win / 4) & ~63));
        if (PASS == 3) {  // third pass (k_rs3_seq): an F point with no C among its strong neighbours becomes C
            bool has_c = false;
            for (int p = __ldg(srp + i) + lane, pe = __ldg(srp + i + 1); p < pe; p += 32)
                if (get(__ldg(sci + p)) == kC) has_c = true;
            has_c = __any_sync(0xffffffffu, has_c);
            if (!has_c && lane == 0) set_c(i);
            __syncwarp();
            continue;
        }
        if (PASS == 2 && rec) {
            // two-hop record of the candidate (S_i and the S_j of its members; built by
            // k_rs_records over S twice): the next candidate's record is requested
            // before this one is replayed, so the replay sees no global latency
            if (t == 0) {
                const int* rp_ = rec + (int64_t)recW * i + lane;
                pw0 = __ldg(rp_);
                if (recW > 32) pw1 = __ldg(rp_ + 32);
                if (recW > 64) pw2 = __ldg(rp_ + 64);
                if (recW > 96) pw3 = __ldg(rp_ + 96);
            }
            __syncwarp();
            recs[lane] = pw0;
            if (recW > 32) recs[32 + lane] = pw1;
            if (recW > 64) recs[64 + lane] = pw2;
            if (recW > 96) recs[96 + lane] = pw3;
            if (t + 1 < ncand) {
                const int* rp_ = rec + (int64_t)recW * __ldg(cand + t + 1) + lane;
                pw0 = __ldg(rp_);
                if (recW > 32) pw1 = __ldg(rp_ + 32);
                if (recW > 64) pw2 = __ldg(rp_ + 64);
                if (recW > 96) pw3 = __ldg(rp_ + 96);
            }
            if (lane == 0) ncil = 0;
            __syncwarp();
            if (get(i) != kF) continue;
            const int ns = ((volatile int*)recs)[0];
            // one lane per member of S_i: the C members seed the list, the F members
            // (their marks cannot change before their own turn) are replayed in order
            const int myj = lane < ns ? ((volatile int*)recs)[1 + lane * recB] : -1;
            const signed char mj = lane < ns ? get(myj) : kU;
            if (mj == kC) {
                const int pos = atomicAdd(&ncil, 1);
                if (pos < 4096) cil[pos] = myj;
            }
            unsigned fmask = __ballot_sync(0xffffffffu, mj == kF);
            __syncwarp();
            while (fmask) {
                const int p = __ffs(fmask) - 1;
                fmask &= fmask - 1;
                const int j = __shfl_sync(0xffffffffu, myj, p);
                const int nci = min(((volatile int*)&ncil)[0], 4096);
                const int nsj = ((volatile int*)recs)[2 + p * recB];
                bool shared = false;
                if (lane < nsj) {
                    const int k = ((volatile int*)recs)[3 + p * recB + lane];
                    for (int e = 0; e < nci; ++e)
                        if (((volatile int*)cil)[e] == k) {
                            shared = true;
                            break;
                        }
                }
                shared = __any_sync(0xffffffffu, shared);
                if (!shared && lane == 0) {
                    set_c(j);
                    const int pos = ncil;
                    if (pos < 4096) cil[pos] = j;
                    ncil = pos + 1;
                }
                __syncwarp();
            }
            __syncwarp();
            continue;
        }
        if (get(i) != kF) continue;
        const int a = __ldg(srp + i), b = __ldg(srp + i + 1);
        if (lane == 0) ncil = 0;
        __syncwarp();
        for (int p = a + lane; p < b; p += 32) {
            const int j = __ldg(sci + p);
            if (get(j) == kC) {
                const int pos = atomicAdd(&ncil, 1);
                if (pos < 4096) cil[pos] = j;
            }
        }
        __syncwarp();
        for (int p = a; p < b; ++p) {
            const int j = __ldg(sci + p);
            if (get(j) != kF) continue;
            const int nci = min(((volatile int*)&ncil)[0], 4096);
            bool shared = false;
            const int ja = __ldg(srp + j), jb = __ldg(srp + j + 1);
            for (int kk = ja + lane; kk < jb && !shared; kk += 32) {
                const int k = __ldg(sci + kk);
                for (int e = 0; e < nci; ++e)
                    if (((volatile int*)cil)[e] == k) {
                        shared = true;
                        break;
                    }
            }
            shared = __any_sync(0xffffffffu, shared);
            if (!shared && lane == 0) {
                set_c(j);
                const int pos = ncil;
                if (pos < 4096) cil[pos] = j;
                ncil = pos + 1;
            }
            __syncwarp();
        }
        __syncwarp();
    }
    move_window(-1);
}

__global__ void k_rs3_cand(const int* srp, const int* sci, const signed char* mark, int n, int* flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int need = 0;
    if (mark[i] == kF && srp[i + 1] > srp[i]) {
        need = 1;
        for (int p = srp[i]; p < srp[i + 1]; ++p)
            if (mark[sci[p]] == kC) {
                need = 0;
                break;
            }
    }
    flag[i] = need;
}

__global__ void __launch_bounds__(32) k_rs3_seq(const int* srp, const int* sci, signed char* mark, const int* cand,
                                                int ncand) {
    const int lane = threadIdx.x;
    for (int t = 0; t < ncand; ++t) {
        const int i = cand[t];
        bool has_c = false;
        for (int p = srp[i] + lane; p < srp[i + 1]; p += 32)
            if (((volatile signed char*)mark)[sci[p]] == kC) has_c = true;
        has_c = __any_sync(0xffffffffu, has_c);
        if (!has_c && lane == 0) mark[i] = kC;
        __syncwarp();
    }
}

__global__ void k_compact(const int* flag, const int* pos, int n, int* list) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) list[pos[i]] = i;
}

__global__ void k_is_c(const signed char* mark, int n, int* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = mark[i] == kC ? 1 : 0;
}

// ---------------------------------------------------------- interpolation --
// mode 0: count entries per row; mode 1: fill (prp = row pointer)
__global__ void k_interp(const int* rp, const int* ci, const double* v, int n, double theta, const double* mrow,
                         const int* scnt, const signed char* mark, const int* cpos, int mode, int* pcnt,
                         const int* prp, int* pci, double* pv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // coarse_id[j] = cpos[j] when mark[j] == C
    if (mark[i] == kC) {
        if (mode == 0)
            pcnt[i] = 1;
        else {
            pci[prp[i]] = cpos[i];
            pv[prp[i]] = 1.0;
        }
        return;
    }
    if (scnt[i] == 0) {
        if (mode == 0) pcnt[i] = 0;
        return;
    }
    const double thr = theta * mrow[i];
    double sum_neg_all = 0.0, sum_pos_all = 0.0, sum_neg_c = 0.0, sum_pos_c = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (j == i) continue;
        const double a = v[k];
        if (a < 0.0)
            sum_neg_all += a;
        else
            sum_pos_all += a;
        if (mark[j] == kC && -a >= thr) {
            if (a < 0.0)
                sum_neg_c += a;
            else
                sum_pos_c += a;
        }
    }
    double aii = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] == i) aii = v[k];
    if (sum_pos_c == 0.0) aii += sum_pos_all;
    const double alpha = sum_neg_c != 0.0 ? sum_neg_all / sum_neg_c : 0.0;
    const double beta = sum_pos_c != 0.0 ? sum_pos_all / sum_pos_c : 0.0;
    int cnt = 0, o = mode ? prp[i] : 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (j == i || !(-v[k] >= thr) || mark[j] != kC) continue;  // j in S_i and coarse
        const double aij = v[k];
        const double w = aij < 0.0 ? -alpha * aij / aii : -beta * aij / aii;
        if (w != 0.0) {
            if (mode) {
                pci[o] = cpos[j];
                pv[o] = w;
                ++o;
            }
            ++cnt;
        }
    }
    if (mode == 0) pcnt[i] = cnt;
}

// -------------------------------------------------------------- transpose --
__global__ void k_col_count(const int* ci, int nnz, int* cnt) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnz) atomicAdd(cnt + ci[k], 1);
}

__global__ void k_transpose_fill(const int* rp, const int* ci, const double* v, int n, const int* trp, int* fillc,
                                 int* tci, double* tv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int c = ci[k];
        const int pos = trp[c] + atomicAdd(fillc + c, 1);
        tci[pos] = i;
        tv[pos] = v[k];
    }
}

// ----------------------------------------------------------------- SpGEMM --
__global__ void k_prod_count(const int* arp, const int* aci, const int* brp, int n, int* m) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int s = 0;
    for (int k = arp[i]; k < arp[i + 1]; ++k) s += brp[aci[k] + 1] - brp[aci[k]];
    m[i] = s;
}

// Warp per output row.  mode 0: unique-column count; mode 1: fill.
__global__ void __launch_bounds__(256) k_spgemm(const int* arp, const int* aci, const double* av, const int* brp,
                                                const int* bci, const double* bv, int n, int cap, int* scol,
                                                double* sval, int* sfirst, int mode, int* cnt, const int* crp,
                                                int* cci, double* cv) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int* col = scol + wid * cap;
    double* val = sval + wid * cap;
    int* first = sfirst + wid * cap;
    for (int64_t row = wid; row < n; row += nw) {
        const int i = int(row);
        int m = 0;
        for (int ka = arp[i]; ka < arp[i + 1]; ++ka) {
            const int j = aci[ka];
            const double a = av[ka];
            const int b0 = brp[j], len = brp[j + 1] - b0;
            for (int t = lane; t < len; t += 32) {
                col[m + t] = bci[b0 + t];
                val[m + t] = a * bv[b0 + t];
            }
            m += len;
        }
        __syncwarp();
        int u = 0;
        for (int p = lane; p < m; p += 32) {
            const int cp = col[p];
            int f = 1;
            for (int q = 0; q < p; ++q)
                if (col[q] == cp) {
                    f = 0;
                    break;
                }
            first[p] = f;
            u += f;
        }
        for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
        __syncwarp();
        if (mode == 0) {
            if (lane == 0) cnt[i] = u;
        } else {
            const int base = crp[i];
            for (int p = lane; p < m; p += 32) {
                if (!first[p]) continue;
                const int cp = col[p];
                int rank = 0;
                double s = 0.0;
                for (int q = 0; q < m; ++q) {
                    const int cq = col[q];
                    if (first[q] && cq < cp) ++rank;
                    if (cq == cp) s += val[q];
                }
                cci[base + rank] = cp;
                cv[base + rank] = s;
            }
        }
        __syncwarp();
    }
}

__global__ void k_diag_pos(const int* rp, const int* ci, int n, int* diag, int* missing) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = -1;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] == i) d = k;
    diag[i] = d;
    if (d < 0) atomicOr(missing, 1);
}

// ------------------------------------------------------------- dense LU -----
__global__ void k_csr_to_dense(const int* rp, const int* ci, const double* v, int n, double* d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) d[(int64_t)ci[k] * n + i] = v[k];
}

// Single CTA: Eigen::PartialPivLU unblocked path, column-major.
__global__ void __launch_bounds__(1024) k_dense_lu(double* a, int n, int* perm, double* scale_out) {
    __shared__ double sv[1024];
    __shared__ int si[1024];
    __shared__ double sbest;
    __shared__ int sp;
    const int t = threadIdx.x;
    // scale = max |a|
    double mx = 0.0;
    for (int64_t e = t; e < (int64_t)n * n; e += 1024) mx = fmax(mx, fabs(a[e]));
    sv[t] = mx;
    __syncthreads();
    for (int s = 512; s > 0; s >>= 1) {
        if (t < s) sv[t] = fmax(sv[t], sv[t + s]);
        __syncthreads();
    }
    if (t == 0) *scale_out = sv[0];
    for (int i = t; i < n; i += 1024) perm[i] = i;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        // first max |a(i,k)|, i >= k
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int i = k + t; i < n; i += 1024) {
            const double x = fabs(a[(int64_t)k * n + i]);
            if (x > best) {
                best = x;
                bi = i;
            }
        }
        sv[t] = best;
        si[t] = bi;
        __syncthreads();
        for (int s = 512; s > 0; s >>= 1) {
            if (t < s) {
                const double o = sv[t + s];
                const int oi = si[t + s];
                if (o > sv[t] || (o == sv[t] && oi < si[t])) {
                    sv[t] = o;
                    si[t] = oi;
                }
            }
            __syncthreads();
        }
        if (t == 0) {
            sbest = sv[0];
            sp = si[0];
        }
        __syncthreads();
        const double bst = sbest;
        const int p = sp;
        if (bst != 0.0) {
            if (p != k) {
                for (int j = t; j < n; j += 1024) {
                    const double x = a[(int64_t)j * n + k];
                    a[(int64_t)j * n + k] = a[(int64_t)j * n + p];
                    a[(int64_t)j * n + p] = x;
                }
                if (t == 0) {
                    const int x = perm[k];
                    perm[k] = perm[p];
                    perm[p] = x;
                }
            }
            __syncthreads();
            const double d = a[(int64_t)k * n + k];
            for (int i = k + 1 + t; i < n; i += 1024) a[(int64_t)k * n + i] = a[(int64_t)k * n + i] / d;
        }
        __syncthreads();
        const int rem = n - k - 1;
        for (int64_t e = t; e < (int64_t)rem * rem; e += 1024) {
            const int jj = k + 1 + int(e / rem), ii = k + 1 + int(e % rem);
            a[(int64_t)jj * n + ii] = a[(int64_t)jj * n + ii] - a[(int64_t)k * n + ii] * a[(int64_t)jj * n + k];
        }
        __syncthreads();
    }
}

// thread per column j of the inverse: oracle DenseLU::solve_inplace(e_j);
// out row-major (out[i*n + j] = inv(i,j)), which is also the coalesced layout.
__global__ void k_dense_inv(const double* lu, const int* perm, int n, double* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    for (int i = 0; i < n; ++i) out[(int64_t)i * n + j] = (perm[i] == j) ? 1.0 : 0.0;
    for (int jj = 0; jj < n; ++jj) {
        const double xj = out[(int64_t)jj * n + j];
        for (int i = jj + 1; i < n; ++i)
            out[(int64_t)i * n + j] = out[(int64_t)i * n + j] - lu[(int64_t)jj * n + i] * xj;
    }
    for (int jj = n - 1; jj >= 0; --jj) {
        const double xj = out[(int64_t)jj * n + j] / lu[(int64_t)jj * n + jj];
        out[(int64_t)jj * n + j] = xj;
        for (int i = 0; i < jj; ++i) out[(int64_t)i * n + j] = out[(int64_t)i * n + j] - lu[(int64_t)jj * n + i] * xj;
    }
}

}  // namespace

// =========================================================== host helpers ==
struct Scratch {
    DBuf<char> tmp;
};

// out[0] = 0, out[i+1] = sum_{k<=i} in[k]; returns out[n]
static int scan(Ctx& c, Scratch& s, const int* in, int* out, int n) {
    MG_CUDA(cudaMemsetAsync(out, 0, sizeof(int), c.s));
    if (n == 0) return 0;
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out + 1, n, c.s);
    s.tmp.ensure(bytes + 16);
    cub::DeviceScan::InclusiveSum(s.tmp.p, bytes, in, out + 1, n, c.s);
    check_launch("scan");
    int total = 0;
    MG_CUDA(cudaMemcpyAsync(&total, out + n, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    return total;
}

static inline int nblk(int64_t n, int t = 256) { return int(std::max<int64_t>(1, (n + t - 1) / t)); }

// C = A * B (scalar_matrix.cpp:120-151), exact
static void spgemm(Ctx& c, Scratch& s, const CsrView& a, const CsrView& b, DCsr& out) {
    const int n = a.n;
    DBuf<int> m(n > 0 ? n : 1), cnt(n > 0 ? n : 1);
    out.n = n;
    out.m = b.m;
    out.rp.alloc(n + 1);
    if (n == 0) {
        MG_CUDA(cudaMemsetAsync(out.rp.p, 0, sizeof(int), c.s));
        out.nnz = 0;
        return;
    }
    k_prod_count<<<nblk(n), 256, 0, c.s>>>(a.rp, a.ci, b.rp, n, m.p);
    int cap = 0;
    {
        DBuf<int> mx(1);
        MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), c.s));
        k_max_int<<<std::min(nblk(n), 1024), 256, 0, c.s>>>(m.p, n, mx.p);
        MG_CUDA(cudaMemcpyAsync(&cap, mx.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
        c.sync();
    }
    cap = std::max(cap, 1);
    // per-warp scratch of `cap` products; keep the total under ~512 MB
    const int64_t budget = int64_t(512) << 20;
    const int64_t wcap = std::max<int64_t>(8, budget / (int64_t(cap) * 16));
    const int warps = int(std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(n, int64_t(c.sm_count) * 16), wcap)));
    const int blocks = (warps + 7) / 8;
    const int64_t nw = int64_t(blocks) * 8;
    DBuf<int> scol(nw * cap), sfirst(nw * cap);
    DBuf<double> sval(nw * cap);
    k_spgemm<<<blocks, 256, 0, c.s>>>(a.rp, a.ci, a.v, b.rp, b.ci, b.v, n, cap, scol.p, sval.p, sfirst.p, 0, cnt.p,
                                      nullptr, nullptr, nullptr);
    check_launch("spgemm count");
    out.nnz = scan(c, s, cnt.p, out.rp.p, n);
    out.ci.alloc(std::max(out.nnz, 1));
    out.v.alloc(std::max(out.nnz, 1));
    k_spgemm<<<blocks, 256, 0, c.s>>>(a.rp, a.ci, a.v, b.rp, b.ci, b.v, n, cap, scol.p, sval.p, sfirst.p, 1, nullptr,
                                      out.rp.p, out.ci.p, out.v.p);
    check_launch("spgemm fill");
    c.sync();
}

// R = P^T (scalar_matrix.cpp:98-105)
static void transpose(Ctx& c, Scratch& s, const DCsr& p, DCsr& r) {
    r.n = p.m;
    r.m = p.n;
    r.nnz = p.nnz;
    DBuf<int> cnt(std::max(r.n, 1)), fillc(std::max(r.n, 1));
    MG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * r.n, c.s));
    MG_CUDA(cudaMemsetAsync(fillc.p, 0, sizeof(int) * r.n, c.s));
    if (p.nnz) k_col_count<<<nblk(p.nnz), 256, 0, c.s>>>(p.ci.p, p.nnz, cnt.p);
    r.rp.alloc(r.n + 1);
    scan(c, s, cnt.p, r.rp.p, r.n);
    r.ci.alloc(std::max(r.nnz, 1));
    r.v.alloc(std::max(r.nnz, 1));
    k_transpose_fill<<<nblk(p.n), 256, 0, c.s>>>(p.rp.p, p.ci.p, p.v.p, p.n, r.rp.p, fillc.p, r.ci.p, r.v.p);
    k_sort_rows<<<nblk(r.n), 256, 0, c.s>>>(r.rp.p, r.ci.p, r.v.p, r.n);
    check_launch("transpose");
}

static void diag_positions(Ctx& c, const CsrView& a, DBuf<int>& diag) {
    diag.alloc(std::max(a.n, 1));
    int* missing = c.counters.p + 8;
    MG_CUDA(cudaMemsetAsync(missing, 0, sizeof(int), c.s));
    k_diag_pos<<<nblk(a.n), 256, 0, c.s>>>(a.rp, a.ci, a.n, diag.p, missing);
    int h = 0;
    MG_CUDA(cudaMemcpyAsync(&h, missing, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    if (h) throw Error(MPREC_SETUP, "AMG: structurally absent diagonal");
}

// rs_coarsen (amg.cpp:47-186): returns nc; fills cf (1 = C) and P
static int rs_coarsen(Ctx& c, Scratch& s, const CsrView& a, double theta, DBuf<signed char>& cf, DCsr& p) {
    const int n = a.n;
    DBuf<double> mrow(n);
    DBuf<int> scnt(n), stcnt(n), srp(n + 1), strp(n + 1), stfill(n);
    MG_CUDA(cudaMemsetAsync(stcnt.p, 0, sizeof(int) * n, c.s));
    MG_CUDA(cudaMemsetAsync(stfill.p, 0, sizeof(int) * n, c.s));
    auto tr_s = std::make_unique<Trace>(&c, "amg strength");
    k_strength_count<<<nblk(n), 256, 0, c.s>>>(a.rp, a.ci, a.v, n, theta, mrow.p, scnt.p, stcnt.p);
    const int ns = scan(c, s, scnt.p, srp.p, n);
    scan(c, s, stcnt.p, strp.p, n);
    DBuf<int> sci(std::max(ns, 1)), stci(std::max(ns, 1));
    k_strength_fill<<<nblk(n), 256, 0, c.s>>>(a.rp, a.ci, a.v, n, theta, mrow.p, srp.p, sci.p, strp.p, stfill.p,
                                              stci.p);
    k_sort_rows<<<nblk(n), 256, 0, c.s>>>(strp.p, stci.p, nullptr, n);
    check_launch("strength");

    tr_s.reset();
    // ---- first pass: bucket queue
    int lmax = 0;
    {
        DBuf<int> mx(1);
        MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), c.s));
        k_max_int<<<std::min(nblk(n), 1024), 256, 0, c.s>>>(stcnt.p, n, mx.p);
        MG_CUDA(cudaMemcpyAsync(&lmax, mx.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
        c.sync();
    }
    const int nbuckets = 2 * lmax + 1;
    Buckets q;
    q.n0 = (n + 63) / 64;
    q.n1 = (q.n0 + 63) / 64;
    q.n2 = (q.n1 + 63) / 64;
    DBuf<unsigned long long> l0((size_t)nbuckets * q.n0), l1((size_t)nbuckets * q.n1), l2((size_t)nbuckets * q.n2);
    DBuf<int> bcnt(nbuckets), lam(n), inc(n), jlist(2 * (size_t)n), klist(2 * (size_t)n);
    MG_CUDA(cudaMemsetAsync(l0.p, 0, l0.bytes(), c.s));
    MG_CUDA(cudaMemsetAsync(bcnt.p, 0, bcnt.bytes(), c.s));
    MG_CUDA(cudaMemsetAsync(inc.p, 0, inc.bytes(), c.s));
    q.l0 = l0.p;
    q.l1 = l1.p;
    q.l2 = l2.p;
    q.cnt = bcnt.p;
    cf.alloc(n);
    signed char* mark = cf.p;
    k_rs_init<<<nblk(n), 256, 0, c.s>>>(scnt.p, stcnt.p, n, mark, lam.p, q, nullptr);
    k_bq_summary<<<nblk((int64_t)q.n1 * nbuckets), 256, 0, c.s>>>(l0.p, l1.p, q.n0, q.n1, nbuckets);
    k_bq_summary<<<nblk((int64_t)q.n2 * nbuckets), 256, 0, c.s>>>(l1.p, l2.p, q.n1, q.n2, nbuckets);
    {
        Trace tr(&c, "amg rs first pass");
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 0.0);
        const size_t smem = sizeof(unsigned long long) * (size_t)nbuckets * (q.n1 + q.n2) + sizeof(int) * nbuckets;
        DBuf<long long> prof;
        if (trace_on()) prof.alloc(8);
        // windowed kernel: summary levels + a window of WN points' state in shared memory
        static const bool win_on = [] {
            const char* e = getenv("MPREC_RS_WINDOW");
            return !(e && e[0] == '0');
        }();
        int WN = 0;
        size_t wsmem = 0;
        if (win_on && nbuckets <= 127) {  // (increment counters: 6 bits)
            const size_t fixed = sizeof(unsigned long long) * (size_t)nbuckets * (q.n1 + q.n2) + 4 * (size_t)((nbuckets + 3) & ~3);
            const size_t budget = [] {  // (MPREC_RS_BUDGET_KB: experiments; more window, less L1 for the strength graph)
                const char* e = getenv("MPREC_RS_BUDGET_KB");
                return size_t(e ? atoi(e) : 208) * 1024;
            }();
            for (int t = 32768; t >= 2048 && !WN; t >>= 1) {
                const size_t need = fixed + (size_t)nbuckets * (t / 64) * 8 + 2 * (size_t)t;
                if (need <= budget) {
                    WN = t;
                    wsmem = need;
                }
            }
        }
        if (WN) {
            static bool attr = false;
            if (!attr) {
                MG_CUDA(cudaFuncSetAttribute(k_rs_select_win, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
                attr = true;
            }
            // two-hop adjacency records when they fit kRsRecMax ints (levels 0-1 of c5)
            DBuf<int> rec;
            int recB = 0, recW = 0;
            {
                int smax = 0;
                DBuf<int> mx2(1);
                MG_CUDA(cudaMemsetAsync(mx2.p, 0, sizeof(int), c.s));
                k_max_int<<<std::min(nblk(n), 1024), 256, 0, c.s>>>(scnt.p, n, mx2.p);
                MG_CUDA(cudaMemcpyAsync(&smax, mx2.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
                c.sync();
                const int B = 2 + smax, RW = (1 + lmax * B + 31) & ~31;
                static const bool rec_on = [] {
                    const char* e = getenv("MPREC_RS_RECORDS");
                    return !(e && e[0] == '0');
                }();
                if (rec_on && RW <= kRsRecMax && lmax <= 32 && smax <= 32) {
                    recB = B;
                    recW = RW;
                    rec.alloc((size_t)RW * n);
                    k_rs_records<<<nblk(n), 256, 0, c.s>>>(srp.p, sci.p, strp.p, stci.p, n, B, RW, rec.p);
                }
            }
            k_rs_select_win<<<1, kRsWinThreads, wsmem, c.s>>>(srp.p, sci.p, strp.p, stci.p, mark, lam.p, q, nbuckets, inc.p, jlist.p,
                                                   klist.p, n, WN, prof.p, rec.p, recB, recW);
        } else if (smem <= 200 * 1024) {
            static bool attr = false;
            if (!attr) {
                MG_CUDA(cudaFuncSetAttribute(k_rs_select<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                attr = true;
            }
            k_rs_select<true><<<1, 32, smem, c.s>>>(srp.p, sci.p, strp.p, stci.p, mark, lam.p, q, nbuckets, inc.p,
                                                    jlist.p, klist.p, prof.p);
        } else {
            k_rs_select<false><<<1, 32, 0, c.s>>>(srp.p, sci.p, strp.p, stci.p, mark, lam.p, q, nbuckets, inc.p,
                                                  jlist.p, klist.p, prof.p);
        }
        check_launch("rs first pass");
        if (trace_on()) {
            long long h[8];
            prof.download(h, 8, c.s);
            c.sync();
            fprintf(stderr, "[mprec] rs select n=%d sel=%lld window %d (slides %lld, selections outside %lld) cycles/sel: find %.0f  d %.0f  e1 %.0f  e2a %.0f  e2b %.0f\n", n,
                    h[6], WN, WN ? h[7] / 1000000 : 0ll, WN ? h[7] % 1000000 : 0ll, h[0] / double(h[6]), h[1] / double(h[6]), h[2] / double(h[6]), h[3] / double(h[6]),
                    h[4] / double(h[6]));
        }
    }
    // ---- second pass
    auto tr2 = std::make_unique<Trace>(&c, "amg rs pass 2");
    DBuf<int> flag(n), fpos(n + 1), list(n);
    k_rs2_cand<<<nblk(n), 256, 0, c.s>>>(srp.p, sci.p, mark, n, flag.p);
    int ncand = scan(c, s, flag.p, fpos.p, n);
    if (trace_on()) fprintf(stderr, "[mprec] rs pass 2: n=%d candidates %d\n", n, ncand);
    if (ncand) {
        k_compact<<<nblk(n), 256, 0, c.s>>>(flag.p, fpos.p, n, list.p);
        static const bool win2_on = [] {
            const char* e = getenv("MPREC_RS_WINDOW");
            return !(e && e[0] == '0');
        }();
        if (win2_on) {
            static bool attr = false;
            if (!attr) {
                MG_CUDA(cudaFuncSetAttribute(k_rs2_seq_win<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRs2Win));
                MG_CUDA(cudaFuncSetAttribute(k_rs2_seq_win<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRs2Win));
                attr = true;
            }
            // S-S two-hop records (the first pass's builder with S in both hops)
            DBuf<int> rec2;
            int rB = 0, rW = 0;
            {
                int smax = 0;
                DBuf<int> mx2(1);
                MG_CUDA(cudaMemsetAsync(mx2.p, 0, sizeof(int), c.s));
                k_max_int<<<std::min(nblk(n), 1024), 256, 0, c.s>>>(scnt.p, n, mx2.p);
                MG_CUDA(cudaMemcpyAsync(&smax, mx2.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
                c.sync();
                const int B = 2 + smax, RW = (1 + smax * B + 31) & ~31;
                const char* e = getenv("MPREC_RS_RECORDS");
                if (!(e && e[0] == '0') && RW <= kRsRecMax && smax <= 32) {
                    rB = B;
                    rW = RW;
                    rec2.alloc((size_t)RW * n);
                    k_rs_records<<<nblk(n), 256, 0, c.s>>>(srp.p, sci.p, srp.p, sci.p, n, B, RW, rec2.p);
                }
            }
            k_rs2_seq_win<2><<<1, kRs2Threads, kRs2Win, c.s>>>(srp.p, sci.p, mark, list.p, ncand, n, rec2.p, rB, rW);
        } else {
            k_rs2_seq<<<1, 32, 0, c.s>>>(srp.p, sci.p, mark, list.p, ncand);
        }
        check_launch("rs second pass");
    }
    tr2.reset();
    auto tr2b = std::make_unique<Trace>(&c, "amg rs pass 3");
    // ---- third pass
    k_rs3_cand<<<nblk(n), 256, 0, c.s>>>(srp.p, sci.p, mark, n, flag.p);
    ncand = scan(c, s, flag.p, fpos.p, n);
    if (ncand) {
        k_compact<<<nblk(n), 256, 0, c.s>>>(flag.p, fpos.p, n, list.p);
        static const bool win3_on = [] {
            const char* e = getenv("MPREC_RS_WINDOW");
            return !(e && e[0] == '0');
        }();
        if (win3_on) {
            static bool attr3 = false;
            if (!attr3) {
                MG_CUDA(cudaFuncSetAttribute(k_rs2_seq_win<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRs2Win));
                attr3 = true;
            }
            k_rs2_seq_win<3><<<1, kRs2Threads, kRs2Win, c.s>>>(srp.p, sci.p, mark, list.p, ncand, n, nullptr, 0, 0);
        } else {
            k_rs3_seq<<<1, 32, 0, c.s>>>(srp.p, sci.p, mark, list.p, ncand);
        }
        check_launch("rs third pass");
    }
    tr2b.reset();
    // ---- coarse ids + direct interpolation
    Trace tr3(&c, "amg interpolation");
    DBuf<int> isc(n), cpos(n + 1), pcnt(n);
    k_is_c<<<nblk(n), 256, 0, c.s>>>(mark, n, isc.p);
    const int nc = scan(c, s, isc.p, cpos.p, n);
    k_interp<<<nblk(n), 256, 0, c.s>>>(a.rp, a.ci, a.v, n, theta, mrow.p, scnt.p, mark, cpos.p, 0, pcnt.p, nullptr,
                                       nullptr, nullptr);
    p.n = n;
    p.m = nc;
    p.rp.alloc(n + 1);
    p.nnz = scan(c, s, pcnt.p, p.rp.p, n);
    p.ci.alloc(std::max(p.nnz, 1));
    p.v.alloc(std::max(p.nnz, 1));
    k_interp<<<nblk(n), 256, 0, c.s>>>(a.rp, a.ci, a.v, n, theta, mrow.p, scnt.p, mark, cpos.p, 1, nullptr, p.rp.p,
                                       p.ci.p, p.v.p);
    check_launch("interp");
    c.sync();
    return nc;
}

// DenseFactor::factor + inverse for the coarsest level (dense_factor.cpp:7-19)
static void coarse_factor(Ctx& c, const CsrView& a, DBuf<double>& lu, DBuf<double>& inv) {
    const int n = a.n;
    if (n > 20000) throw Error(MPREC_SETUP, "AMG coarsest level too large for the dense solve (" + std::to_string(n) + ")");
    lu.alloc(std::max<int64_t>(1, (int64_t)n * n));
    inv.alloc(std::max<int64_t>(1, (int64_t)n * n));
    if (n == 0) return;
    MG_CUDA(cudaMemsetAsync(lu.p, 0, lu.bytes(), c.s));
    k_csr_to_dense<<<nblk(n), 256, 0, c.s>>>(a.rp, a.ci, a.v, n, lu.p);
    DBuf<int> perm(n);
    DBuf<double> scale(1);
    {
        Ctx::Scope sc(&c, MPREC_K_COARSE, 0.0);
        k_dense_lu<<<1, 1024, 0, c.s>>>(lu.p, n, perm.p, scale.p);
        check_launch("dense lu");
    }
    // pivot check |u_ii| <= 1e-14 * max|a|
    double sc = 0.0;
    scale.download(&sc, 1, c.s);
    std::vector<double> h = lu.to_host(c.s, (size_t)n * n);  // synchronises c.s
    for (int i = 0; i < n; ++i)
        if (std::abs(h[(size_t)i * n + i]) <= 1e-14 * sc)
            throw Error(MPREC_SINGULAR_BLOCK, "singular dense-factor pivot block in cell " + std::to_string(i), i);
    k_dense_inv<<<nblk(n, 128), 128, 0, c.s>>>(lu.p, perm.p, n, inv.p);
    check_launch("dense inverse");
    c.sync();
}

// Sweep schedules of one smoothed level (run on the setup's helper thread).
static void build_level_schedules(Ctx& c, AmgLevel& l, Pattern* pat) {
    if (pat) {
        pat->ensure_sched(c);  // (built before the hierarchies when two share it)
        l.ofwd = pat->fwd.order.p;
        l.obwd = pat->bwd.order.p;
        l.glev_f = pat->fwd.level.p;
        l.glev_b = pat->bwd.level.p;
    } else {
        build_sched(c, l.n, l.a.rp, l.a.ci, +1, l.own_fwd);
        build_sched(c, l.n, l.a.rp, l.a.ci, -1, l.own_bwd);
        l.ofwd = l.own_fwd.order.p;
        l.obwd = l.own_bwd.order.p;
        l.glev_f = l.own_fwd.level.p;
        l.glev_b = l.own_bwd.level.p;
    }
    l.invd.alloc(std::max(l.n, 1));
    compute_invd(c, l.a, l.invd.p);
    l.b.ensure(std::max(l.n, 1));
    l.xf.ensure(std::max(l.n, 1));
    tune_level_sweep(c, l, pat ? pat->fwd : l.own_fwd, pat ? pat->bwd : l.own_bwd);
    c.sync();
}

// AMGHierarchy::setup (amg.cpp:188-214)
void Amg::setup(Ctx& c, const CsrView& a0, const AmgParams& p, Pattern* pat) {
    prm = p;
    lv.clear();
    Scratch s;
    auto L0 = std::make_unique<AmgLevel>();
    L0->n = a0.n;
    L0->a = a0;
    if (!a0.diag) {
        diag_positions(c, a0, L0->a_own.diag);
        L0->a.diag = L0->a_own.diag.p;
    }
    lv.push_back(std::move(L0));
    // Sweep schedules (Kahn levels, 1/a_ii, the level-synchronous programs) of a
    // level are built on a helper thread with its own stream as soon as the level
    // is known not to be the coarsest, i.e. while the single-warp RS first pass of
    // the next level runs on this thread's stream (they only read the level).
    // (two helpers, each with its own stream: the coarse levels arrive faster than
    // one thread compiles their programs, and the backlog would end the setup)
    constexpr int kHelpers = 2;
    Ctx cs[kHelpers];
    std::mutex qm;
    std::condition_variable qcv;
    std::deque<std::pair<AmgLevel*, bool>> queue;  // (level, is level 0)
    bool qdone = false;
    std::exception_ptr qerr;
    std::thread helpers[kHelpers];
    for (int hq = 0; hq < kHelpers; ++hq)
        helpers[hq] = std::thread([&, hq] {
            StreamAllocScope alloc_on(cs[hq].s);
            try {
                for (;;) {
                    std::pair<AmgLevel*, bool> job;
                    {
                        std::unique_lock<std::mutex> lk(qm);
                        qcv.wait(lk, [&] { return qdone || !queue.empty(); });
                        if (queue.empty()) break;
                        job = queue.front();
                        queue.pop_front();
                    }
                    build_level_schedules(cs[hq], *job.first, job.second ? pat : nullptr);
                }
                cs[hq].sync();
            } catch (...) {
                std::lock_guard<std::mutex> lk(qm);
                if (!qerr) qerr = std::current_exception();
            }
        });
    auto finish_helper = [&] {
        {
            std::lock_guard<std::mutex> lk(qm);
            qdone = true;
        }
        qcv.notify_all();
        for (auto& t : helpers)
            if (t.joinable()) t.join();
    };
    struct Joiner {  // the helper must not outlive this frame on an exception
        std::function<void()> f;
        ~Joiner() { f(); }
    } joiner{finish_helper};
    while (lv.back()->n > prm.max_coarse && int(lv.size()) < prm.max_levels) {
        AmgLevel& f = *lv.back();
        auto nl = std::make_unique<AmgLevel>();
        const int nc = rs_coarsen(c, s, f.a, prm.theta, f.cf, nl->p);
        if (nc == 0) {
            f.cf.release();
            break;
        }
        if (nc > int(0.95 * f.n))
            throw Error(MPREC_SETUP, "AMG coarsening stagnated at size " + std::to_string(f.n));
        Trace tr(&c, "amg transpose+galerkin");
        transpose(c, s, nl->p, nl->r);
        DCsr ap;
        spgemm(c, s, f.a, nl->p.view(), ap);
        spgemm(c, s, nl->r.view(), ap.view(), nl->a_own);
        nl->n = nc;
        nl->a = nl->a_own.view();
        diag_positions(c, nl->a, nl->a_own.diag);
        nl->a.diag = nl->a_own.diag.p;
        lv.push_back(std::move(nl));
        {
            std::lock_guard<std::mutex> lk(qm);
            queue.emplace_back(lv[lv.size() - 2].get(), lv.size() == 2);
        }
        qcv.notify_one();
    }
    nco = lv.back()->n;
    Trace trc(&c, "amg coarse dense LU+inv");
    coarse_factor(c, lv.back()->a, coarse_lu, coarse_inv);
    {
        Trace tr(&c, "amg sweep schedules (wait)");
        finish_helper();
        if (qerr) std::rethrow_exception(qerr);
    }
    for (auto& l : lv) {
        l->x.ensure(std::max(l->n, 1));
        l->b.ensure(std::max(l->n, 1));
        l->t.ensure(std::max(l->n, 1));
        l->xf.ensure(std::max(l->n, 1));
    }
}

}  // namespace mg
