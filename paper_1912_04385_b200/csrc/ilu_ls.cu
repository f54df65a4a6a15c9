// ilu_ls.cu -- K6 v3: block ILU(0) triangular solves (ILU0Factor::apply,
// ilu0.cpp:41-59) as a level-synchronous pipeline over a SOLVE STREAM, nb = 8.
//
// Mapping (as the Gauss-Seidel programs, gs_ls.cu): K contiguous groups of block
// rows in sweep order, one thread block each.  Four compute warps process the
// group's block rows in block-DAG-level order, up to 16 per step (lane = (block
// row b, scalar row r)), a named barrier between steps; values of the group live
// in a shared-memory ring, the previous group's values arrive through an
// importer warp and a shared-memory halo ring.  Per block row
//     v   = rhs_I - B0 y_K0 - B1 y_K1           (B = the L or U blocks of row I)
//     y_I = inv(L_II) v (forward, unit lower)  /  inv(U_II) v (backward)
// with the packed inverse of the diagonal block (k_ilu_dinv8).
//
// What makes it bandwidth-shaped: at factorisation the row's dependency blocks,
// the packed inverse and a right-hand-side slot are copied into a per-direction
// STREAM in processing order -- one step's data is one contiguous range -- so the
// loader warp moves a whole step with ONE bulk copy (plus one for the step's
// 272-byte metadata).  (The previous version gathered 16 separate 512-byte
// blocks per step straight from the BSR factor: issue-bound, 28 ms per sweep at
// c5.)  The right-hand side is scattered into the stream by a parallel pre-pass
// per apply.  Results differ from the warp-per-block-row kernel (ilu_solve.cu)
// only by association.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "mprec.cuh"

namespace mg {
namespace {

constexpr int kIB = 16;                  // block rows per step
constexpr int kIRec = 200;               // doubles per row record: B0, B1, D, rhs
constexpr int kIMeta = 16 + 16 * kIB;    // metadata bytes per step
constexpr int kISlot = ((kIMeta + kIB * kIRec * 8) + 127) & ~127;  // ring slot bytes
constexpr int kINS = 4;                  // ring slots
constexpr int kIH = 256;                 // halo ring entries (block rows)
constexpr int kICW = 4;                  // compute warps
constexpr int kIThreads = 32 * (kICW + 2);

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

// Step metadata (kIMeta bytes): int4 {cnt, imports needed, 0, 0}, then per row
// slot b < kIB int4 {block row I, own ring slot, dependency slot 0, dependency
// slot 1} (slots in doubles; missing dependency -> the zero slot).
template <bool kFwd>
__global__ void __launch_bounds__(kIThreads, 1) k_ilu_ls(const int4* __restrict__ meta, const char* __restrict__ data,
                                                          const int2* __restrict__ gst, const long long* __restrict__ gdoff,
                                                          const int* __restrict__ scnt, const int* __restrict__ imp,
                                                          const int2* __restrict__ gimp, double* y, int W) {
    extern __shared__ __align__(128) unsigned char sm[];
    char* ring = reinterpret_cast<char*>(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kINS * kISlot);
    uint64_t* empty = full + kINS;
    int* imported = reinterpret_cast<int*>(empty + kINS);
    volatile int* cons = imported + 1;  // consumer's current import need (importer back-pressure)
    double* xs = reinterpret_cast<double*>(imported + 4);  // 8W ring | zero 8 | trash 8 | halo ring 8 kIH
    const int g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int2 gs = gst[g];  // first step, step count
    if (threadIdx.x == 0) {
        for (int s = 0; s < kINS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        *imported = 0;
        *cons = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 16; i += blockDim.x) xs[8 * W + i] = 0.0;
    __syncthreads();
    if (warp == kICW) {  // loader: one bulk copy for the metadata, one for the data of a step
        if (lane == 0) {
            long long off = gdoff[g];
            for (int s = 0; s < gs.y; ++s) {
                const int slot = s % kINS;
                if (s >= kINS) mbar_wait(empty + slot, ((s / kINS) - 1) & 1);
                const int cnt = __ldg(scnt + gs.x + s);
                mbar_expect_tx(full + slot, kIMeta + cnt * kIRec * 8);
                bulk_g2s(ring + slot * kISlot, meta + int64_t(gs.x + s) * (kIMeta / 16), kIMeta, full + slot);
                bulk_g2s(ring + slot * kISlot + kIMeta, data + off, cnt * kIRec * 8, full + slot);
                off += int64_t(cnt) * kIRec * 8;
            }
        }
        return;
    }
    if (warp == kICW + 1) {  // importer: previous group's block rows (8 values each), in production order
        const int2 gi = gimp[g];
        const int* rows = imp + gi.x;
        const int nimp = gi.y;
        volatile double* halo = xs + 8 * W + 16;
        volatile int* vimp = imported;
        const int e = lane >> 3, r = lane & 7;
        int base = 0;
        while (base < nimp) {
            // ring back-pressure: entry idx overwrites idx - kIH, dead once the
            // consumer's need passed idx - kIH / 2 (checked at setup)
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
            MG_DCHECK(e >= pre || idx < nimp);
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
    // compute warps: warp w handles row slots 4w .. 4w+3 of every step
    const int b = warp * 4 + (lane >> 3), r = lane & 7;
    const unsigned imp_a = smem_u32(imported);
    const volatile double* vxs = xs;
    int have = 0;
    for (int s = 0; s < gs.y; ++s) {
        const int slot = s % kINS;
        mbar_wait(full + slot, (s / kINS) & 1);
        const char* st = ring + slot * kISlot;
        const int4 h = *reinterpret_cast<const int4*>(st);
        const int cnt = h.x, need = h.y;
        if (warp == 0 && lane == 0) *cons = need;
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
        const bool act = b < cnt;
        const int4 mr = *reinterpret_cast<const int4*>(st + 16 + 16 * min(b, cnt - 1));
        MG_DCHECK(cnt >= 1 && cnt <= kIB && need >= 0);
        MG_DCHECK(mr.z >= 0 && mr.z <= 8 * W + 16 + 8 * (kIH - 1) && mr.w >= 0 && mr.w <= 8 * W + 16 + 8 * (kIH - 1));
        MG_DCHECK(mr.y >= 0 && (mr.y < 8 * W || mr.y == 8 * W + 8) && mr.x >= 0);
        const double* rec = reinterpret_cast<const double*>(st + kIMeta) + min(b, cnt - 1) * kIRec;
        // four independent FMA chains of 4 (dependency latency, not throughput, bounds a step)
        double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            a[c & 1] = fma(rec[c * 8 + r], vxs[mr.z + c], a[c & 1]);
            a[2 + (c & 1)] = fma(rec[64 + c * 8 + r], vxs[mr.w + c], a[2 + (c & 1)]);
        }
        const double v = rec[192 + r] - ((a[0] + a[1]) + (a[2] + a[3]));
        double vc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) vc[c] = __shfl_sync(0xffffffffu, v, (lane & ~7) + c);
        double o[4] = {kFwd ? v : 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (kFwd ? (c < r) : (c >= r)) o[c & 3] = fma(rec[128 + c * 8 + r], vc[c], o[c & 3]);
        const double out = (o[0] + o[1]) + (o[2] + o[3]);
        asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(smem_u32(xs + (act ? mr.y + r : 8 * W + 8 + r))),
                     "d"(out)
                     : "memory");
        const int64_t yo = act ? int64_t(mr.x) * 8 + r : -1;
        asm volatile(
            "{\n .reg .pred p;\n setp.ge.s64 p, %2, 0;\n @p st.relaxed.gpu.global.b64 [%0], %1;\n}" ::"l"(y + yo),
            "l"(__double_as_longlong(out)), "l"(yo)
            : "memory");
        // the step's rows are read by the next steps of all four warps; the slot is
        // free once every warp is past it
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kICW) : "memory");
        if (warp == 0 && lane == 0) mbar_arrive(empty + slot);
    }
}

// per factorisation: row records (B0, B1, packed inverse) into the stream
__global__ void k_il_fill(int nc, const long long* __restrict__ roff, const int2* __restrict__ kdep,
                          const double* __restrict__ val, const double* __restrict__ dinv, char* data) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int I = int(t >> 5), lane = int(t & 31);
    if (I >= nc) return;
    double* rec = reinterpret_cast<double*>(data + roff[I]);
    const int2 k = kdep[I];
    for (int e = lane; e < 192; e += 32) {
        double v;
        if (e < 64)
            v = k.x >= 0 ? val[int64_t(k.x) * 64 + e] : 0.0;
        else if (e < 128)
            v = k.y >= 0 ? val[int64_t(k.y) * 64 + e - 64] : 0.0;
        else
            v = dinv[int64_t(I) * 64 + e - 128];
        rec[e] = v;
    }
}

// per apply: right-hand side into the row records
__global__ void k_il_rhs(int nc, const long long* __restrict__ roff, const double* __restrict__ rhs, char* data) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int I = int(t >> 3), r = int(t & 7);
    if (I >= nc) return;
    reinterpret_cast<double*>(data + roff[I])[192 + r] = rhs[int64_t(I) * 8 + r];
}

}  // namespace

// ---------------------------------------------------------------- setup ------
// Programs of one direction for the block pattern (levels from its Kahn
// schedules).  Fails (ok = false) when the pattern does not fit the scheme: a
// block row with more than 2 dependency blocks in one direction, a dependency
// beyond the previous group, a halo entry read too far behind the import front,
// or shared memory.
struct IlBuilt {
    bool ok = false;
    int K = 0, W = 0, hmax = 0, nsteps = 0;
    std::vector<int4> meta;        // nsteps x kIMeta / 16
    std::vector<int> scnt;         // rows per step
    std::vector<int2> gst, gimp;   // per group: (first step, steps), (import offset, count)
    std::vector<long long> gdoff;  // per group: data byte offset
    std::vector<int> imp;
    std::vector<long long> roff;   // per block row: byte offset of its record
    std::vector<int2> kdep;        // per block row: BSR indices of its dependency blocks (-1: none)
    int64_t data_bytes = 0;
};

static int il_smem(int W) { return kINS * kISlot + 2 * kINS * 8 + 16 + (8 * W + 16 + 8 * kIH) * 8; }

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
    out.kdep.assign(n, make_int2(-1, -1));
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (!is_dep(i, j)) continue;
            if (d >= 2) return;
            (d == 0 ? out.kdep[i].x : out.kdep[i].y) = k;
            ++d;
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
    if (il_smem(W) > 225 * 1024) return;
    const int zero_slot = 8 * W, trash_slot = 8 * W + 8, halo_slot = 8 * W + 16;
    out.roff.assign(n, 0);
    out.gst.resize(K);
    out.gdoff.resize(K);
    int64_t doff = 0;
    for (int g = 0; g < K; ++g) {
        const int m = gstart[g + 1] - gstart[g];
        const int* q = seq.data() + gstart[g];
        out.gst[g] = make_int2(int(out.scnt.size()), 0);
        out.gdoff[g] = doff;
        int run_need = 0;
        for (int u = 0; u < m;) {
            int cnt = 0;
            while (u + cnt < m && cnt < kIB && lev[q[u + cnt]] == lev[q[u]]) ++cnt;
            const size_t mb = out.meta.size();
            out.meta.resize(mb + kIMeta / 16, make_int4(0, 0, 0, 0));
            int4* mt = out.meta.data() + mb;
            int need = 0, minneed = 1 << 30;
            for (int bb = 0; bb < kIB; ++bb) {
                int4& br = mt[1 + bb];
                br = make_int4(q[u], trash_slot, zero_slot, zero_slot);
                if (bb >= cnt) continue;
                const int i = q[u + bb];
                br.x = i;
                br.y = 8 * (pos[i] & (W - 1));
                out.roff[i] = doff + int64_t(bb) * kIRec * 8;
                int d = 0;
                for (int kk = rp[i]; kk < rp[i + 1]; ++kk) {
                    const int j = ci[kk];
                    if (!is_dep(i, j)) continue;
                    int sl;
                    if (gid[j] == g) {
                        sl = 8 * (pos[j] & (W - 1));
                    } else {
                        sl = halo_slot + 8 * (hidx[j] & (kIH - 1));
                        need = std::max(need, hidx[j] + 1);
                        minneed = std::min(minneed, hidx[j]);
                    }
                    (d == 0 ? br.z : br.w) = sl;
                    ++d;
                }
            }
            // monotone per group (the importer's ring window follows it), and every
            // entry a step reads must still be in the halo ring
            need = std::max(need, run_need);
            run_need = need;
            mt[0] = make_int4(cnt, need, 0, 0);
            if (minneed != (1 << 30) && need - minneed > kIH / 4) return;
            out.scnt.push_back(cnt);
            doff += int64_t(cnt) * kIRec * 8;
            u += cnt;
        }
        out.gst[g].y = int(out.scnt.size()) - out.gst[g].x;
    }
    out.gimp.resize(K);
    for (int g = 0; g < K; ++g) out.gimp[g] = make_int2(gimp_off[g], gimp_off[g + 1] - gimp_off[g]);
    out.imp = std::move(imp);
    out.K = K;
    out.W = W;
    out.hmax = hmax;
    out.nsteps = int(out.scnt.size());
    out.data_bytes = doff;
    out.ok = true;
}

static void il_upload(Ctx& c, IlBuilt& b, IluLs& s) {
    s.meta.upload(b.meta.data(), b.meta.size(), c.s);
    s.scnt.upload(b.scnt.data(), b.scnt.size(), c.s);
    s.gst.upload(b.gst.data(), b.K, c.s);
    s.gdoff.upload(b.gdoff.data(), b.K, c.s);
    s.imp.alloc(std::max<size_t>(b.imp.size(), 1));
    if (!b.imp.empty()) s.imp.upload(b.imp.data(), b.imp.size(), c.s);
    s.gimp.upload(b.gimp.data(), b.K, c.s);
    s.roff.upload(b.roff.data(), b.roff.size(), c.s);
    s.kdep.upload(b.kdep.data(), b.kdep.size(), c.s);
    s.data.alloc(size_t(b.data_bytes));
    s.K = b.K;
    s.W = b.W;
    s.hmax = b.hmax;
    s.nsteps = b.nsteps;
    s.nc = int(b.roff.size());
    s.smem = il_smem(b.W);
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
    c.sync();
    return true;
}

// (Re)fill the solve streams from the factor and the packed inverses.
void ilu_ls_fill(Ctx& c, IluLs& s, const double* val, const double* dinv) {
    const int64_t threads = int64_t(s.nc) * 32;
    k_il_fill<<<int((threads + 255) / 256), 256, 0, c.s>>>(s.nc, s.roff.p, s.kdep.p, val, dinv, s.data.p);
    check_launch("ilu ls fill");
    s.filled = true;
}

void ilu_ls_solve(Ctx& c, IluLs& s, bool fwd, const double* rhs, double* y) {
    static bool attr[2] = {false, false};
    if (!attr[fwd]) {
        if (fwd)
            MG_CUDA(cudaFuncSetAttribute(k_ilu_ls<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        else
            MG_CUDA(cudaFuncSetAttribute(k_ilu_ls<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        attr[fwd] = true;
    }
    if (!s.filled) throw Error(MPREC_SETUP, "ilu ls: stream not filled");
    k_il_rhs<<<int((int64_t(s.nc) * 8 + 255) / 256), 256, 0, c.s>>>(s.nc, s.roff.p, rhs, s.data.p);
    check_launch("ilu ls rhs");
    if (fwd)
        k_ilu_ls<true><<<s.K, kIThreads, s.smem, c.s>>>(s.meta.p, s.data.p, s.gst.p, s.gdoff.p, s.scnt.p, s.imp.p,
                                                        s.gimp.p, y, s.W);
    else
        k_ilu_ls<false><<<s.K, kIThreads, s.smem, c.s>>>(s.meta.p, s.data.p, s.gst.p, s.gdoff.p, s.scnt.p, s.imp.p,
                                                         s.gimp.p, y, s.W);
    check_launch(fwd ? "ilu ls fwd" : "ilu ls bwd");
}

}  // namespace mg
