// ilu_ls.cu -- K6 v2: block ILU(0) triangular solves (ILU0Factor::apply,
// ilu0.cpp:41-59) as a level-synchronous pipeline, nb = 8.
//
// The same mapping as the Gauss-Seidel programs (gs_ls.cu), on block rows: K
// contiguous groups of block rows in sweep order, one thread block each; one
// compute warp processes the group's block rows in block-DAG-level order, four
// per step (lane = (block row b, scalar row r)), with only __syncwarp between
// steps; the previous group's values arrive through an importer warp and a
// shared-memory halo.  Per block row
//     v   = rhs_I - sum_{dependency blocks K} B_IK y_K        (B = L or U block)
//     y_I = inv(L_II) v (forward, unit lower)  /  inv(U_II) v (backward)
// with the packed inverses of the diagonal blocks (k_ilu_dinv8).  The block
// values are NOT copied into the program (they are the 10 GB factor): the
// compute warp prefetches the blocks of the step P = 20 steps ahead straight
// from the factor with 1-D TMA bulk copies (one per 512-byte block, completion
// counted on one mbarrier per ring slot) into a shared-memory ring, so HBM
// latency leaves the dependency chain.  The import halo is a ring
// of 256 block rows; the importer is held back by the consumer's progress.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "mprec.cuh"

namespace mg {
namespace {

constexpr int kIB = 4;                   // block rows per step
constexpr int kIStep = 16 + kIB * 24;    // program bytes per step
constexpr int kISPC = kLsCH / kIStep;    // steps per program chunk
constexpr int kIChunk = kISPC * kIStep;  // program chunk bytes
constexpr int kIP = 20;                  // prefetch distance (steps)
constexpr int kIH = 256;                 // halo ring entries (block rows)
constexpr int kIBlk = kIB * 200;         // doubles per prefetched step: 4 x (3 blocks + rhs)
constexpr int kINS = 2;                  // program chunks in the ring
constexpr int kIThreads = 96;

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
        "IL_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra IL_WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_il(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// prefetch the blocks of one step into a ring slot with 1-D TMA bulk copies
// (16 per step, lanes 0..15, completion counted on the slot's mbarrier): per
// block row b, [0, 64) first dependency block, [64, 128) second, [128, 192) packed
// inverse of the diagonal block, [192, 200) right-hand side.  Missing
// dependencies read the zero block; padding block rows read the step's first
// block row.  (16-byte cp.async per lane stalled at issue: 1.5 us per step.)
__device__ __forceinline__ void il_prefetch(const int* rec, int lane, const double* __restrict__ val,
                                            const double* __restrict__ dinv, const double* __restrict__ rhs,
                                            const double* __restrict__ zero, double* slot, uint64_t* bar) {
    if (lane == 0) mbar_expect_tx(bar, kIB * (3 * 512 + 64));
    __syncwarp();
    if (lane < 16) {
        const int cnt = rec[0];
        const int b = lane >> 2, w = lane & 3;
        const int* br = rec + 4 + 6 * min(b, cnt - 1);
        const int I = br[0];
        const double* src;
        unsigned bytes = 512;
        if (w < 2) {
            const int k = br[2 + w];
            src = k >= 0 ? val + int64_t(k) * 64 : zero;
        } else if (w == 2) {
            src = dinv + int64_t(I) * 64;
        } else {
            src = rhs + int64_t(I) * 8;
            bytes = 64;
        }
        bulk_g2s(slot + b * 200 + 64 * w, src, bytes, bar);
    }
}

template <bool kFwd>
__global__ void __launch_bounds__(kIThreads, 1) k_ilu_ls(const char* __restrict__ prog, const int2* __restrict__ gch,
                                                          const int* __restrict__ imp, const int2* __restrict__ gimp,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ dinv,
                                                          const double* __restrict__ rhs,
                                                          const double* __restrict__ zero, double* y, int W,
                                                          long long* stats) {
    extern __shared__ __align__(128) unsigned char sm[];
    char* ring = reinterpret_cast<char*>(sm);                             // program chunks
    double* blk = reinterpret_cast<double*>(sm + kINS * kLsCH);           // prefetched blocks
    uint64_t* full = reinterpret_cast<uint64_t*>(blk + kIP * kIBlk);
    uint64_t* empty = full + kINS;
    uint64_t* slotbar = empty + kINS;                                     // prefetch slots (cp.async arrivals)
    int* imported = reinterpret_cast<int*>(slotbar + kIP);
    volatile int* cons = imported + 1;                                   // consumer's current need
    double* xs = reinterpret_cast<double*>(imported + 4);                 // 8W ring | zero 8 | trash 8 | halo ring
    const int g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2 ch = gch[g];  // first chunk, steps
    const int nsteps = ch.y, nchunks = (nsteps + kISPC - 1) / kISPC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kINS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int s = 0; s < kIP; ++s) mbar_init(slotbar + s, 1);
        *imported = 0;
        *cons = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 16; i += blockDim.x) xs[8 * W + i] = 0.0;
    __syncthreads();
    if (warp == 2) {  // loader: program chunks -> shared-memory ring
        if (lane == 0)
            for (int c = 0; c < nchunks; ++c) {
                const int s = c & (kINS - 1);
                if (c >= kINS) mbar_wait(empty + s, ((c / kINS) - 1) & 1);
                mbar_expect_tx(full + s, kIChunk);
                bulk_g2s(ring + s * kLsCH, prog + (int64_t)(ch.x + c) * kIChunk, kIChunk, full + s);
            }
        return;
    }
    if (warp == 1) {  // importer: previous group's block rows (8 values each), in production order
        const int2 gi = gimp[g];
        const int* rows = imp + gi.x;
        const int nimp = gi.y;
        volatile double* halo = xs + 8 * W + 16;
        volatile int* vimp = imported;
        const int e = lane >> 3, r = lane & 7;
        int base = 0;
        while (base < nimp) {
            // ring back-pressure: entry idx overwrites idx - kIH, which is dead once
            // the consumer's need passed idx - kIH / 2 (checked at setup)
            while (base + 4 > *cons + kIH / 2) {
            }
            const int idx = base + e;
            const bool in = idx < nimp;
            unsigned long long raw = kPending;
            if (in) raw = ld_relaxed_il(y + int64_t(__ldg(rows + idx)) * 8 + r);
            const bool ready = in && raw != kPending;
            const unsigned m = __ballot_sync(0xffffffffu, ready);
            int pre = 0;
            while (pre < 4 && ((m >> (8 * pre)) & 0xffu) == 0xffu) ++pre;
            pre = min(pre, nimp - base);
            if (e < pre) halo[int64_t(idx & (kIH - 1)) * 8 + r] = __longlong_as_double((long long)raw);
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
    // compute warp
    if (nsteps == 0) return;
    long long t_start = 0, t_imp = 0, t_blk = 0;
    if (stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    const int b = lane >> 3, r = lane & 7;
    const unsigned imp_a = smem_u32(imported);
    const volatile double* vxs = xs;
    int have = 0;
    auto rec_of = [&](int s) {
        return reinterpret_cast<const int*>(ring + ((s / kISPC) & (kINS - 1)) * kLsCH + (s % kISPC) * kIStep);
    };
    // prologue: steps 0 .. P-1 (program chunk 0 first)
    mbar_wait(full, 0);
    for (int s = 0; s < kIP; ++s) {
        if (s < nsteps) {
            if (s > 0 && s % kISPC == 0) mbar_wait(full + ((s / kISPC) & (kINS - 1)), ((s / kISPC) / kINS) & 1);
            il_prefetch(rec_of(s), lane, val, dinv, rhs, zero, blk + (s % kIP) * kIBlk, slotbar + s % kIP);
        }
    }
    for (int s = 0; s < nsteps; ++s) {
        const int* rec = rec_of(s);
        const int cnt = rec[0], need = rec[1];
        const int* br = rec + 4 + 6 * min(b, cnt - 1);
        const int I = br[0], myoff = br[1], off0 = br[4], off1 = br[5];
        if (lane == 0) *cons = need;
        long long ta = 0, tb = 0, tc = 0;
        if (stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ta));
        asm volatile(
            "{\n .reg .pred p;\n .reg .s32 r;\n"
            " setp.le.s32 p, %2, %0;\n"
            " @p bra.uni ILD%=;\n"
            "ILW%=:\n ld.volatile.shared.s32 r, [%1];\n setp.lt.s32 p, r, %2;\n @p bra.uni ILW%=;\n"
            " mov.s32 %0, r;\n fence.acq_rel.cta;\n"
            "ILD%=:\n}"
            : "+r"(have)
            : "r"(imp_a), "r"(need)
            : "memory");
        if (stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb));
        mbar_wait(slotbar + s % kIP, (s / kIP) & 1);
        if (stats) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tc));
            t_imp += tb - ta;
            t_blk += tc - tb;
        }
        const double* sb = blk + (s % kIP) * kIBlk + b * 200;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) acc += sb[c * 8 + r] * vxs[off0 + c] + sb[64 + c * 8 + r] * vxs[off1 + c];
        const double v = sb[192 + r] - acc;
        double vc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) vc[c] = __shfl_sync(0xffffffffu, v, (lane & ~7) + c);
        double out = kFwd ? v : 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (kFwd ? (c < r) : (c >= r)) out += sb[128 + c * 8 + r] * vc[c];
        const bool act = b < cnt;
        asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(smem_u32(xs + (act ? myoff + r : 8 * W + 8 + r))),
                     "d"(out)
                     : "memory");
        const int64_t yo = act ? int64_t(I) * 8 + r : -1;
        asm volatile(
            "{\n .reg .pred p;\n setp.ge.s64 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(y + yo),
            "l"(__double_as_longlong(out)), "l"(yo)
            : "memory");
        __syncwarp();
        // release a program chunk once its last step is consumed AND prefetched past
        if (s % kISPC == kISPC - 1 && lane == 0) mbar_arrive(empty + ((s / kISPC) & (kINS - 1)));
        // prefetch step s + P (its program chunk may be the next one)
        const int sp = s + kIP;
        long long td = 0, te = 0;
        if (stats) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(td));
        if (sp < nsteps) {
            if (sp % kISPC == 0) mbar_wait(full + ((sp / kISPC) & (kINS - 1)), ((sp / kISPC) / kINS) & 1);
            il_prefetch(rec_of(sp), lane, val, dinv, rhs, zero, blk + (sp % kIP) * kIBlk, slotbar + sp % kIP);
        }
        if (stats) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
            t_imp += (te - td) << 32;  // prefetch issue time in the high word
        }
    }
    if (stats && lane == 0) {
        long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        stats[4 * g] = t_start;
        stats[4 * g + 1] = t_end;
        stats[4 * g + 2] = t_imp;
        stats[4 * g + 3] = t_blk;
    }
}

}  // namespace

// ---------------------------------------------------------------- setup ------
// Programs of both directions for the block pattern `pat` (levels from its
// Kahn schedules).  Returns false when the pattern does not fit the scheme
// (a block row with more than 2 dependency blocks in one direction, a dependency
// beyond the previous group, or shared memory).
struct IlBuilt {
    bool ok = false;
    int K = 0, W = 0, hmax = 0, nsteps = 0, nchunks = 0;
    std::vector<char> prog;
    std::vector<int2> gch, gimp;
    std::vector<int> imp;
};

static int il_smem(int W, int hmax) {
    return kINS * kLsCH + kIP * kIBlk * 8 + (2 * kINS + kIP) * 8 + 16 + (8 * W + 16 + 8 * std::min(hmax, kIH)) * 8;
}

static void il_build(const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<int>& lev, int n,
                     int dir, int K, IlBuilt& out) {
    out = IlBuilt();
    K = std::min(K, n / 64);
    if (K < 1) return;
    auto row_of_t = [&](int t) { return dir > 0 ? t : n - 1 - t; };
    auto is_dep = [&](int i, int j) { return dir > 0 ? j < i : j > i; };
    std::vector<int> gstart(K + 1), gid(n);
    for (int g = 0; g <= K; ++g) gstart[g] = int((int64_t)g * n / K);
    for (int g = 0; g < K; ++g)
        for (int t = gstart[g]; t < gstart[g + 1]; ++t) gid[row_of_t(t)] = g;
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (!is_dep(i, j)) continue;
            if (++d > 2) return;
            if (gid[j] != gid[i] && gid[j] != gid[i] - 1) return;
        }
    }
    std::vector<int> seq(n), pos(n);
    for (int g = 0; g < K; ++g) {
        int* q = seq.data() + gstart[g];
        const int m = gstart[g + 1] - gstart[g];
        for (int u = 0; u < m; ++u) q[u] = row_of_t(gstart[g] + u);
        std::stable_sort(q, q + m, [&](int x, int y) { return lev[x] < lev[y]; });
        for (int u = 0; u < m; ++u) pos[q[u]] = u;
    }
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
    int W = 16;
    while (W < maxdist + kIB + 4) W <<= 1;
    if (il_smem(W, hmax) > 225 * 1024) return;
    std::vector<int2> gch(K);
    std::vector<std::vector<int>> steps(K);
    int64_t nchunks = 0, nsteps = 0;
    for (int g = 0; g < K; ++g) {
        const int m = gstart[g + 1] - gstart[g];
        const int* q = seq.data() + gstart[g];
        auto& st = steps[g];
        for (int u = 0; u < m;) {
            st.push_back(u);
            int cnt = 0;
            while (u + cnt < m && cnt < kIB && lev[q[u + cnt]] == lev[q[u]]) ++cnt;
            u += cnt;
        }
        st.push_back(m);
        const int ns = int(st.size()) - 1;
        gch[g] = make_int2(int(nchunks), ns);
        nchunks += (ns + kISPC - 1) / kISPC;
        nsteps += ns;
    }
    std::vector<char> prog(size_t(nchunks) * kIChunk, 0);
    const int zero_off = 8 * W, halo_off = 8 * W + 16;
    for (int g = 0; g < K; ++g) {
        const int* q = seq.data() + gstart[g];
        const auto& st = steps[g];
        int run_need = 0;
        for (int k = 0; k + 1 < int(st.size()); ++k) {
            int* rec = reinterpret_cast<int*>(prog.data() + int64_t(gch[g].x + k / kISPC) * kIChunk +
                                              int64_t(k % kISPC) * kIStep);
            const int cnt = st[k + 1] - st[k];
            int need = 0, minneed = 1 << 30;
            rec[0] = cnt;
            for (int bb = 0; bb < kIB; ++bb) {
                int* br = rec + 4 + 6 * bb;
                br[0] = q[st[k]];
                br[1] = 8 * W + 8;
                br[2] = br[3] = -1;
                br[4] = br[5] = zero_off;
                if (bb >= cnt) continue;
                const int i = q[st[k] + bb];
                br[0] = i;
                br[1] = 8 * (pos[i] & (W - 1));
                int d = 0;
                for (int kk = rp[i]; kk < rp[i + 1]; ++kk) {
                    const int j = ci[kk];
                    if (!is_dep(i, j)) continue;
                    br[2 + d] = kk;
                    if (gid[j] == g) {
                        br[4 + d] = 8 * (pos[j] & (W - 1));
                    } else {
                        br[4 + d] = halo_off + 8 * (hidx[j] & (kIH - 1));
                        need = std::max(need, hidx[j] + 1);
                        minneed = std::min(minneed, hidx[j]);
                    }
                    ++d;
                }
            }
            // monotone per group (the importer's ring window follows it), and every
            // entry a step reads must still be in the halo ring
            need = std::max(need, run_need);
            run_need = need;
            rec[1] = need;
            if (minneed != (1 << 30) && need - minneed > kIH / 4) return;
        }
    }
    std::vector<int2> gimp(K);
    for (int g = 0; g < K; ++g) gimp[g] = make_int2(gimp_off[g], gimp_off[g + 1] - gimp_off[g]);
    out.prog = std::move(prog);
    out.gch = std::move(gch);
    out.gimp = std::move(gimp);
    out.imp = std::move(imp);
    out.K = K;
    out.W = W;
    out.hmax = hmax;
    out.nsteps = int(nsteps);
    out.nchunks = int(nchunks);
    out.ok = true;
}

static void il_upload(Ctx& c, IlBuilt& b, IluLs& s) {
    s.prog.upload(b.prog.data(), b.prog.size(), c.s);
    s.gch.upload(b.gch.data(), b.K, c.s);
    s.imp.alloc(std::max<size_t>(b.imp.size(), 1));
    if (!b.imp.empty()) s.imp.upload(b.imp.data(), b.imp.size(), c.s);
    s.gimp.upload(b.gimp.data(), b.K, c.s);
    s.K = b.K;
    s.W = b.W;
    s.hmax = b.hmax;
    s.nsteps = b.nsteps;
    s.smem = il_smem(b.W, b.hmax);
    s.ok = true;
}

bool build_ilu_ls(Ctx& c, Pattern& pat, int K, IluLs& fwd, IluLs& bwd) {
    fwd = IluLs();
    bwd = IluLs();
    const int n = pat.nc;
    if (n < 1024 || int(pat.h_rp.size()) != n + 1) return false;
    pat.ensure_sched(c);
    std::vector<int> lf(n), lb(n);
    MG_CUDA(cudaMemcpyAsync(lf.data(), pat.fwd.level.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c.s));
    MG_CUDA(cudaMemcpyAsync(lb.data(), pat.bwd.level.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c.s));
    c.sync();
    IlBuilt bf, bb;
    std::thread t([&] { il_build(pat.h_rp, pat.h_ci, lb, n, -1, K, bb); });
    il_build(pat.h_rp, pat.h_ci, lf, n, +1, K, bf);
    t.join();
    if (!bf.ok || !bb.ok) return false;
    il_upload(c, bf, fwd);
    il_upload(c, bb, bwd);
    fwd.zero.alloc(64);
    MG_CUDA(cudaMemsetAsync(fwd.zero.p, 0, 64 * sizeof(double), c.s));
    c.sync();
    return true;
}

void ilu_ls_solve(Ctx& c, const IluLs& s, const IluLs& zero_owner, bool fwd, const double* val, const double* dinv,
                  const double* rhs, double* y) {
    static bool attr[2] = {false, false};
    if (!attr[fwd]) {
        if (fwd)
            MG_CUDA(cudaFuncSetAttribute(k_ilu_ls<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        else
            MG_CUDA(cudaFuncSetAttribute(k_ilu_ls<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        attr[fwd] = true;
    }
    static const bool want_stats = getenv("MPREC_ILU_LS_STATS") != nullptr;
    DBuf<long long> st;
    if (want_stats) st.alloc(4 * s.K);
    if (fwd)
        k_ilu_ls<true><<<s.K, kIThreads, s.smem, c.s>>>(s.prog.p, s.gch.p, s.imp.p, s.gimp.p, val, dinv, rhs,
                                                        zero_owner.zero.p, y, s.W, st.p);
    else
        k_ilu_ls<false><<<s.K, kIThreads, s.smem, c.s>>>(s.prog.p, s.gch.p, s.imp.p, s.gimp.p, val, dinv, rhs,
                                                         zero_owner.zero.p, y, s.W, st.p);
    check_launch(fwd ? "ilu ls fwd" : "ilu ls bwd");
    if (want_stats) {
        auto h = st.to_host(c.s);
        long long t0 = h[0];
        for (int g = 0; g < s.K; ++g) t0 = std::min(t0, h[4 * g]);
        fprintf(stderr, "[ilu ls %s] K=%d steps=%d (group: start end import_wait_us block_wait_us)\n", fwd ? "fwd" : "bwd",
                s.K, s.nsteps);
        for (int g = 0; g < s.K; g += std::max(1, s.K / 10))
            fprintf(stderr, "  g%3d %9.1f %9.1f import %9.1f prefetch-issue %9.1f block %9.1f\n", g,
                    (h[4 * g] - t0) * 1e-3, (h[4 * g + 1] - t0) * 1e-3, (h[4 * g + 2] & 0xffffffffll) * 1e-3,
                    (h[4 * g + 2] >> 32) * 1e-3, h[4 * g + 3] * 1e-3);
    }
}

}  // namespace mg
