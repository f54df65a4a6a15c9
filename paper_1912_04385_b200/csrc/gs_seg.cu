// gs_seg.cu -- band-segment Gauss-Seidel sweep (K14).
//
// Same natural-order semantics as k_gs (sym_gauss_seidel, amg.cpp:25-43), a
// different mapping of the dependency DAG onto the machine.
//   * SEGMENTS: maximal runs of <= 32 consecutive rows in which every row
//     couples to its predecessor in sweep order (on a natural-order grid:
//     pieces of grid lines).  A warp owns a segment, lane per row; the chain
//     x_r = c_r - (a_{r,pred} / a_rr) x_pred costs one DFMA (8.4 cycles) per
//     row instead of one cross-SM hop (>= 0.38 us measured).
//   * BANDS: runs of consecutive segments covering <= B rows, one CTA each,
//     the band's iterate in shared memory.  Dependencies inside the band
//     (the next grid lines) are resolved through shared memory; only those
//     crossing a band boundary pay the L2 hop.
// Bands are claimed in sweep order and segments inside a band in Kahn-level
// order of the segment DAG, so a warp only waits on work claimed before it:
// deadlock free.  Every partial sum has a fixed order, so results are
// deterministic; they differ from the warp-per-row sweep only by association
// and stay within the 1e-10 apply bar.  Requires rows sorted by column with a
// stored diagonal (checked at setup).
//
// Measured on B200 while building this (scripts/micro/*.cu): a per-row store
// from one lane costs ~110 ns (same-line serialisation) vs ~14 ns per row with
// group stores; a volatile smem spin per row costs ~70 cycles; a strong L2
// load ~280 cycles, a cross-SM store->load hop ~380 ns.
#include <algorithm>
#include <vector>

#include "mprec.cuh"

namespace mg {
namespace {

constexpr int kExt = 8;       // external dependencies held in registers per row

__device__ __forceinline__ unsigned long long ld_relaxed_s(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// One CTA per BAND (a run of consecutive segments covering <= B rows; the
// band's iterate lives in shared memory).  Warps claim the band's segments in
// Kahn-level order and process one segment each: lane u <-> row r(u) = i0 + u
// (forward) or i1 - 1 - u (backward).  Per row the dependencies other than the
// chain predecessor are gathered in non-blocking poll rounds -- from shared
// memory when inside the band (~30 cycles), from global memory otherwise (one
// L2 hop, only across band boundaries) -- into c_r = (b_r - rest) / a_rr; the
// ready prefix of the segment then advances by x_r = c_r - (a_{r,pred}/a_rr) x_pred,
// one DFMA per row with the coefficients broadcast by shuffles off the
// critical path.  Values are published per group of 8 rows (one coalesced
// store; a store per row from one lane serialises on the cache line).
template <int DIR>
__global__ void __launch_bounds__(512) k_gs_bseg(const int* __restrict__ rp, const int* __restrict__ ci,
                                                const double* __restrict__ v, const int* __restrict__ diag,
                                                const double* __restrict__ invd, const double* __restrict__ b,
                                                const double* __restrict__ xold, double* xnew,
                                                const int* __restrict__ sstart, const int* __restrict__ bord,
                                                const int* __restrict__ bseg0, const int* __restrict__ brow0,
                                                int nbands, int* counter, unsigned sleep_ns, int window,
                                                long long* tl) {
    extern __shared__ unsigned long long xb[];
    __shared__ int band_sh, claim_sh;
    const int lane = threadIdx.x & 31;
    volatile unsigned long long* vxb = xb;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const int t = atomicAdd(counter, 1);
            band_sh = t < nbands ? (DIR > 0 ? t : nbands - 1 - t) : -1;
            claim_sh = 0;
        }
        __syncthreads();
        const int band = band_sh;
        if (band < 0) return;
        const int lo = __ldg(brow0 + band), hi = __ldg(brow0 + band + 1);
        for (int q = threadIdx.x; q < hi - lo; q += blockDim.x) xb[q] = kPending;
        __syncthreads();
        const int kb = __ldg(bseg0 + band), kn = __ldg(bseg0 + band + 1) - kb;
        for (;;) {
            int k = 0;
            if (lane == 0) k = atomicAdd(&claim_sh, 1);
            k = __shfl_sync(0xffffffffu, k, 0);
            if (k >= kn) break;
            const int s = __ldg(bord + kb + k);
            long long tc = 0, tf = 0;
            if (tl) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tc));
            const int i0 = __ldg(sstart + s), i1 = __ldg(sstart + s + 1), nrow = i1 - i0;
            const bool valid = lane < nrow;
            const int r = DIR > 0 ? i0 + lane : i1 - 1 - lane;
            int k0 = 0, k1 = 0, kd = 0;
            double bi = 0.0, dii = 0.0;
            if (valid) {
                k0 = __ldg(rp + r);
                k1 = __ldg(rp + r + 1);
                kd = __ldg(diag + r);
                bi = __ldg(b + r);
                dii = __ldg(invd + r);
            }
            const int kp = kd - DIR;  // chain predecessor position, if stored
            const bool has_pred = valid && lane > 0 && kp >= k0 && kp < k1 && __ldg(ci + kp) == r - DIR;
            const double e = has_pred ? __ldg(v + kp) * dii : 0.0;
            // sorted row: fwd [deps | diag | previous iterate], bwd [previous iterate | diag | deps]
            double nd = 0.0;
            if (valid && xold) {
                const int nb = DIR > 0 ? kd + 1 : k0, ne = DIR > 0 ? k1 : kd;
                for (int q = nb; q < ne; ++q) nd += __ldg(v + q) * __ldg(xold + __ldg(ci + q));
            }
            const int db = DIR > 0 ? k0 : kd + 1, de = DIR > 0 ? kd : k1;  // dependency positions
            int dpos[kExt], sidx[kExt];
            double da[kExt], dx[kExt];
            unsigned pend = 0;
            int kq = db;
#pragma unroll
            for (int q = 0; q < kExt; ++q) {
                if (has_pred && kq == kp) ++kq;
                dpos[q] = 0;
                sidx[q] = -1;
                da[q] = 0.0;
                dx[q] = 0.0;
                if (valid && kq < de) {
                    const int j = __ldg(ci + kq);
                    dpos[q] = j;
                    sidx[q] = (j >= lo && j < hi) ? j - lo : -1;
                    da[q] = __ldg(v + kq);
                    pend |= 1u << q;
                    ++kq;
                }
            }
            int kov = kq;  // overflow dependencies, one per round
            double ov = 0.0, cval = 0.0;
            bool ready = !valid;
            double x = 0.0, mine = 0.0;
            int u = 0, rounds = 0;
            while (u < nrow) {
                ++rounds;
                // only rows close to the chain's ready prefix poll: every resident
                // warp's polls share the SM's shared-memory pipe
                if (!ready && lane < u + window) {
                    if (pend) {
                        unsigned long long raw[kExt];
#pragma unroll
                        for (int q = 0; q < kExt; ++q)
                            if (pend & (1u << q))
                                raw[q] = sidx[q] >= 0 ? vxb[sidx[q]] : ld_relaxed_s(xnew + dpos[q]);
#pragma unroll
                        for (int q = 0; q < kExt; ++q)
                            if ((pend & (1u << q)) && raw[q] != kPending) {
                                dx[q] = __longlong_as_double((long long)raw[q]);
                                pend &= ~(1u << q);
                            }
                    }
                    if (!pend) {
                        if (has_pred && kov == kp) ++kov;
                        if (kov < de) {
                            const int j = __ldg(ci + kov);
                            const unsigned long long raw =
                                (j >= lo && j < hi) ? vxb[j - lo] : ld_relaxed_s(xnew + j);
                            if (raw != kPending) {
                                ov += __ldg(v + kov) * __longlong_as_double((long long)raw);
                                ++kov;
                                if (has_pred && kov == kp) ++kov;
                            }
                        }
                        if (kov >= de) {
                            double sum = 0.0;
#pragma unroll
                            for (int q = 0; q < kExt; ++q) sum += da[q] * dx[q];
                            cval = (bi - (nd + (sum + ov))) * dii;
                            ready = true;
                        }
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, ready);
                const int p = min(nrow, m == 0xffffffffu ? 32 : __ffs(~m) - 1);
                if (tl && u == 0 && p > 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tf));
                if (p == u) {
                    // No progress: spin on ONE value -- the first pending dependency of
                    // the prefix row -- in a few-instruction loop.  A full poll round is
                    // ~200 instructions and every resident warp competes for issue slots,
                    // so full rounds by waiting warps would slow the warps that progress.
                    int wi = -1;
                    int wa = -1;
#pragma unroll
                    for (int q = 0; q < kExt; ++q)
                        if (wa < 0 && wi < 0 && (pend & (1u << q))) {
                            if (sidx[q] >= 0)
                                wi = sidx[q];
                            else
                                wa = dpos[q];
                        }
                    wi = __shfl_sync(0xffffffffu, wi, u);
                    wa = __shfl_sync(0xffffffffu, wa, u);
                    if (wi >= 0) {
                        while (vxb[wi] == kPending)
                            if (sleep_ns) __nanosleep(sleep_ns);
                    } else if (wa >= 0) {
                        while (ld_relaxed_s(xnew + wa) == kPending)
                            if (sleep_ns) __nanosleep(sleep_ns);
                    }
                }
                for (int g = u & ~7; g < p; g += 8) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int st = g + q;
                        const double ct = __shfl_sync(0xffffffffu, cval, st);
                        const double et = __shfl_sync(0xffffffffu, e, st);
                        if (st >= u && st < p) {
                            x = fma(-et, x, ct);
                            if (lane == st) mine = x;
                        }
                    }
                    if (lane >= max(g, u) && lane < min(g + 8, p)) {
                        vxb[r - lo] = (unsigned long long)__double_as_longlong(mine);
                        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(xnew + r),
                                     "l"(__double_as_longlong(mine))
                                     : "memory");
                    }
                }
                u = max(u, p);
            }
            if (tl && lane == 0) {
                long long te;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
                tl[4 * s + 0] = tc;
                tl[4 * s + 1] = tf;
                tl[4 * s + 2] = te;
                tl[4 * s + 3] = rounds;
            }
        }
    }
}

// 1 when every row is strictly sorted by column and stores its diagonal at diag[i]
__global__ void k_sorted(const int* rp, const int* ci, const int* diag, int n, int* bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool ok = diag[i] >= rp[i] && diag[i] < rp[i + 1] && ci[diag[i]] == i;
    for (int k = rp[i] + 1; k < rp[i + 1]; ++k) ok = ok && ci[k - 1] < ci[k];
    if (!ok) atomicOr(bad, 1);
}

// bit 0: row i couples to i-1 (forward chain), bit 1: row i couples to i+1 (backward chain)
__global__ void k_chain_flags(const int* rp, const int* ci, const int* diag, int n, unsigned char* f) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int d = diag[i];
    unsigned char v = 0;
    if (d > rp[i] && ci[d - 1] == i - 1) v |= 1;
    if (d + 1 < rp[i + 1] && ci[d + 1] == i + 1) v |= 2;
    f[i] = v;
}

__global__ void k_seg_id(const int* start, int nseg, int* segid) {
    const int s = blockIdx.x;
    for (int i = start[s] + threadIdx.x; i < start[s + 1]; i += blockDim.x) segid[i] = s;
}

__global__ void k_seg_graph(const int* rp, const int* ci, const int* start, const int* segid, int nseg, int* srp,
                            int* sci, int64_t nnz) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g <= nseg) srp[g] = rp[start[g]];
    for (int64_t k = g; k < nnz; k += (int64_t)gridDim.x * blockDim.x) sci[k] = segid[ci[k]];
}

}  // namespace

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

// Segments are maximal dependency chains (row i couples to its predecessor in
// sweep order) cut to at most 32 rows, so the lockstep chain never delays a
// row behind one it does not depend on.  Claim order: Kahn levels of the
// segment DAG (the row DAG with rows merged per segment).
static void build_one(Ctx& c, const CsrView& a, const std::vector<int>& starts, int dir, SegSched& out) {
    const int nseg = int(starts.size()) - 1;
    out.start.alloc(nseg + 1);
    out.start.upload(starts.data(), nseg + 1, c.s);
    out.hstart = starts;
    DBuf<int> segid(std::max(a.n, 1)), srp(nseg + 1), sci(std::max<int64_t>(a.nnz, 1));
    k_seg_id<<<nseg, 32, 0, c.s>>>(out.start.p, nseg, segid.p);
    const int64_t work = std::max<int64_t>(a.nnz, nseg + 1);
    k_seg_graph<<<int(std::min<int64_t>((work + 255) / 256, 65535)), 256, 0, c.s>>>(a.rp, a.ci, out.start.p, segid.p,
                                                                                   nseg, srp.p, sci.p, a.nnz);
    check_launch("seg graph");
    build_sched(c, nseg, srp.p, sci.p, dir, out.sched);
}

void build_seg_sched(Ctx& c, const CsrView& a, SegSched& fwd, SegSched& bwd) {
    const int n = a.n;
    DBuf<unsigned char> f(std::max(n, 1));
    k_chain_flags<<<(n + 255) / 256, 256, 0, c.s>>>(a.rp, a.ci, a.diag, n, f.p);
    std::vector<unsigned char> h(n);
    f.download(h.data(), n, c.s);
    c.sync();
    std::vector<int> sf, sb;
    sf.reserve(n / 16 + 2);
    sb.reserve(n / 16 + 2);
    // forward: a segment starts at i unless i continues the chain from i-1
    int cur = 0;
    for (int i = 0; i < n; ++i)
        if (i == 0 || !(h[i] & 1) || i - cur == 32) {
            sf.push_back(i);
            cur = i;
        }
    sf.push_back(n);
    // backward (descending sweep): a segment's top row is i unless i chains to i+1
    int top = n - 1;
    for (int i = n - 1; i >= 0; --i)
        if (i == n - 1 || !(h[i] & 2) || top - i == 32) {
            sb.push_back(i + 1);  // end (exclusive) of the segment topped by i
            top = i;
        }
    sb.push_back(0);
    std::reverse(sb.begin(), sb.end());
    build_one(c, a, sf, +1, fwd);
    build_one(c, a, sb, -1, bwd);
}

long long* g_seg_tl = nullptr;  // diagnostics: per-segment timeline (gs_seg_timeline)

// bands of consecutive segments with <= B rows each; inside a band the
// segments are ordered by Kahn level (a topological order of the band)
void build_seg_bands(Ctx& c, SegSched& seg, int B) {
    const int nseg = seg.sched.n;
    std::vector<int> lev(nseg);
    seg.sched.level.download(lev.data(), nseg, c.s);
    c.sync();
    const std::vector<int>& st = seg.hstart;
    std::vector<int> brow0{0}, bseg0{0}, bid(nseg);
    int nb = 0;
    for (int s = 0; s < nseg; ++s) {
        if (st[s + 1] - brow0.back() > B) {
            brow0.push_back(st[s]);
            bseg0.push_back(s);
            ++nb;
        }
        bid[s] = nb;
    }
    brow0.push_back(st[nseg]);
    bseg0.push_back(nseg);
    std::vector<int> ord(nseg);
    for (int s = 0; s < nseg; ++s) ord[s] = s;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return bid[x] != bid[y] ? bid[x] < bid[y] : lev[x] < lev[y]; });
    seg.B = B;
    seg.nbands = int(brow0.size()) - 1;
    seg.bord.alloc(std::max(nseg, 1));
    seg.bord.upload(ord.data(), nseg, c.s);
    seg.bseg0.alloc(seg.nbands + 1);
    seg.bseg0.upload(bseg0.data(), seg.nbands + 1, c.s);
    seg.brow0.alloc(seg.nbands + 1);
    seg.brow0.upload(brow0.data(), seg.nbands + 1, c.s);
    int maxrows = 0;
    for (int q = 0; q < seg.nbands; ++q) maxrows = std::max(maxrows, brow0[q + 1] - brow0[q]);
    seg.band_rows = maxrows;
    c.sync();
}

void gs_sweep_seg(Ctx& c, const CsrView& a, const double* invd, const double* b, const double* xold, double* xnew,
                  int dir, bool xold_zero, const SegSched& seg) {
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 4.0 * a.n + 24.0 * a.n;
    Ctx::Scope sc(&c, MPREC_K_GS, bytes);
    int* ctr = c.counters.p + 9;
    MG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int), c.s));
    static bool attr = false;
    if (!attr) {
        MG_CUDA(cudaFuncSetAttribute(k_gs_bseg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        MG_CUDA(cudaFuncSetAttribute(k_gs_bseg<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    const int warps = [] {
        const char* e = getenv("MPREC_GS_SEG_WARPS");
        return e ? atoi(e) : 16;
    }();
    const unsigned sleep_ns = [] {
        const char* e = getenv("MPREC_GS_SEG_SLEEP");
        return e ? unsigned(atoi(e)) : 0u;
    }();
    const int window = [] {
        const char* e = getenv("MPREC_GS_SEG_WINDOW");
        return e ? atoi(e) : 32;
    }();

    const size_t smem = size_t(std::max(seg.band_rows, 1)) * sizeof(double);
    const int per_sm = std::max(1, int((220 * 1024) / (smem + 1024)));
    const int blocks = std::max(1, std::min(seg.nbands, c.sm_count * std::min(per_sm, 64 / warps)));
    const double* xo = xold_zero ? nullptr : xold;
    if (dir > 0)
        k_gs_bseg<1><<<blocks, warps * 32, smem, c.s>>>(a.rp, a.ci, a.v, a.diag, invd, b, xo, xnew, seg.start.p,
                                                        seg.bord.p, seg.bseg0.p, seg.brow0.p, seg.nbands, ctr, sleep_ns, window, g_seg_tl);
    else
        k_gs_bseg<-1><<<blocks, warps * 32, smem, c.s>>>(a.rp, a.ci, a.v, a.diag, invd, b, xo, xnew, seg.start.p,
                                                         seg.bord.p, seg.bseg0.p, seg.brow0.p, seg.nbands, ctr, sleep_ns, window, g_seg_tl);
    check_launch("gs_sweep_seg");
}

}  // namespace mg


namespace mg {
// Diagnostics: one forward band-segment sweep of level l with a per-segment
// timeline [claim, first rows ready, end, band] indexed by segment.
void gs_seg_timeline(Ctx& c, Amg& amg, int l, long long* host, int* nseg) {
    AmgLevel& L = *amg.lv[l];
    if (!L.seg) throw Error(MPREC_SETUP, "level does not use the band-segment sweep");
    DBuf<long long> ts(4 * (int64_t)L.seg_fwd.sched.n);
    fill(c, L.b.p, 1.0, L.n);
    fill_pending(c, L.xf.p, L.n);
    g_seg_tl = ts.p;
    gs_sweep_seg(c, L.a, L.invd.p, L.b.p, nullptr, L.xf.p, +1, true, L.seg_fwd);
    c.sync();
    g_seg_tl = nullptr;
    ts.download(host, 4 * (int64_t)L.seg_fwd.sched.n, c.s);
    c.sync();
    *nseg = L.seg_fwd.sched.n;
}
}  // namespace mg
