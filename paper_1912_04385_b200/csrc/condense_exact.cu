// condense_exact.cu -- static condensation of the secondary unknowns
// (condense.cpp:206-258), compiled -fmad=false: the
// reduced system and the back-substituted secondary update are bitwise equal
// to the oracle (oracle.cpp: condense / back_substitute).
//
//   k_cond_lu      warp per cell: partial-pivot LU of J22_c in shared memory
//                  (Eigen unblocked order, DenseLU in the oracle), the
//                  singular-pivot test of condense.cpp:214-219, then the
//                  np+1 right-hand sides [J21_c | r2_c] solved one per lane.
//   k_cond_j12     warp per J12 entry: C_e = -(J12_e X_c), v_e = J12_e x_c.
//   k_cond_merge   warp per reduced block: J11 block + C_e ... summed in
//                  entry order, exactly BlockMatrix::assemble's merge
//                  (block_matrix.cpp:32-69) of the entry list condense builds.
//   k_cond_rhs     b = -r1, then += v_e in J12 list order per block row.
//   k_cond_back    warp per cell: d2_c = J22_c^-1 (-r2_c - J21_c d1_c).
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <vector>

#include "condense.cuh"

namespace mg {
namespace {

constexpr int kCondWarps = 2;  // warps per CTA (2 x 16 KB of shared memory)
constexpr int kMaxSec = 32;    // secondary unknowns per cell (a warp)

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// lu_out: ns*ns column-major per cell at lu_off; x_out: ns x (np+1) per cell at
// sec_off[c]*(np+1) (column np = J22^-1 r2)
__global__ void __launch_bounds__(kCondWarps * 32) k_cond_lu(const int* __restrict__ sec_off,
                                                             const int64_t* __restrict__ lu_off,
                                                             const double* __restrict__ j22,
                                                             const double* __restrict__ j21,
                                                             const double* __restrict__ r2, int nc, int np,
                                                             double* lu_out, int* perm_out, double* x_out,
                                                             int* err) {
    __shared__ double sm_a[kCondWarps][kMaxSec * kMaxSec];
    __shared__ double sm_t[kCondWarps][kMaxSec * kMaxSec];
    __shared__ int sm_p[kCondWarps][kMaxSec];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x * kCondWarps + w;
    if (c >= nc) return;
    const int s0 = sec_off[c], ns = sec_off[c + 1] - s0;
    if (ns == 0) return;
    double* A = sm_a[w];
    int* perm = sm_p[w];
    const double* src = j22 + lu_off[c];
    double scale = 0.0;
    for (int e = lane; e < ns * ns; e += 32) {
        A[e] = src[e];
        scale = fmax(scale, fabs(src[e]));
    }
    scale = warp_max(scale);
    if (lane < ns) perm[lane] = lane;
    __syncwarp();
    // DenseLU::factor (oracle.cpp), lane i owns row i
    for (int k = 0; k < ns; ++k) {
        // pivot: first row with the largest |a_ik|, i >= k
        double best = lane >= k && lane < ns ? fabs(A[k * ns + lane]) : -1.0;
        int p = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            if (ob > best || (ob == best && op < p)) {
                best = ob;
                p = op;
            }
        }
        if (best != 0.0) {
            if (p != k) {
                for (int j = lane; j < ns; j += 32) {
                    const double t = A[j * ns + k];
                    A[j * ns + k] = A[j * ns + p];
                    A[j * ns + p] = t;
                }
                if (lane == 0) {
                    const int t = perm[k];
                    perm[k] = perm[p];
                    perm[p] = t;
                }
            }
            __syncwarp();
            const double d = A[k * ns + k];
            if (lane > k && lane < ns) A[k * ns + lane] = A[k * ns + lane] / d;
        }
        __syncwarp();
        if (lane > k && lane < ns) {
            const double lik = A[k * ns + lane];
            for (int j = k + 1; j < ns; ++j) A[j * ns + lane] = A[j * ns + lane] - lik * A[j * ns + k];
        }
        __syncwarp();
    }
    // condense.cpp:214-219
    const double tol = 1e-14 * (scale > 0.0 ? scale : 1.0);
    const bool bad = lane < ns && fabs(A[lane * ns + lane]) <= tol;
    if (__any_sync(0xffffffffu, bad)) {
        if (lane == 0) atomicMin(err, c);
        return;
    }
    for (int e = lane; e < ns * ns; e += 32) lu_out[lu_off[c] + e] = A[e];
    if (lane < ns) perm_out[s0 + lane] = perm[lane];
    // solve the np+1 right-hand sides, one per lane (DenseLU::solve_inplace)
    double* T = sm_t[w];
    if (lane <= np) {
        double* t = T + lane * ns;
        const double* rhs = lane < np ? j21 + int64_t(s0) * np + int64_t(lane) * ns : r2 + s0;
        for (int i = 0; i < ns; ++i) t[i] = rhs[perm[i]];
        for (int j = 0; j < ns; ++j) {
            const double xj = t[j];
            for (int i = j + 1; i < ns; ++i) t[i] = t[i] - A[j * ns + i] * xj;
        }
        for (int j = ns - 1; j >= 0; --j) {
            t[j] = t[j] / A[j * ns + j];
            const double xj = t[j];
            for (int i = 0; i < j; ++i) t[i] = t[i] - A[j * ns + i] * xj;
        }
        double* out = x_out + int64_t(s0) * (np + 1) + int64_t(lane) * ns;
        for (int i = 0; i < ns; ++i) out[i] = t[i];
    }
}

// C_e = -(J12_e X_c[:, :np]) (np x np, column-major), v_e = J12_e X_c[:, np]
__global__ void __launch_bounds__(256) k_cond_j12(const int* __restrict__ sec_off, const int* __restrict__ ecol,
                                                  const int64_t* __restrict__ eoff, const double* __restrict__ j12,
                                                  const double* __restrict__ x, int ne, int np, double* corr,
                                                  double* vrhs) {
    const int lane = threadIdx.x & 31;
    const int e = int((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (e >= ne) return;
    const int c = ecol[e];
    const int s0 = sec_off[c], ns = sec_off[c + 1] - s0;
    const double* a = j12 + eoff[e];                   // np x ns
    const double* xc = x + int64_t(s0) * (np + 1);     // ns x (np+1)
    for (int o = lane; o < np * (np + 1); o += 32) {
        const int i = o % np, j = o / np;
        double acc = a[i] * xc[int64_t(j) * ns];
        for (int k = 1; k < ns; ++k) acc = acc + a[int64_t(k) * np + i] * xc[int64_t(j) * ns + k];
        if (j < np)
            corr[int64_t(e) * np * np + int64_t(j) * np + i] = -acc;
        else
            vrhs[int64_t(e) * np + i] = acc;
    }
}

__global__ void k_cond_keys(const int* rp, const int* ci, int nc, int nnzb, const int* erow, const int* ecol, int ne,
                            unsigned long long* key, int* id) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nnzb) {
        // row of J11 block t: binary search in rp
        int lo = 0, hi = nc;
        while (hi - lo > 1) {
            const int m = (lo + hi) >> 1;
            if (rp[m] <= t)
                lo = m;
            else
                hi = m;
        }
        key[t] = (unsigned long long)lo * nc + ci[t];
        id[t] = t;
    } else if (t < nnzb + ne) {
        const int e = t - nnzb;
        key[t] = (unsigned long long)erow[e] * nc + ecol[e];
        id[t] = t;
    }
}

__global__ void k_cond_heads(const unsigned long long* skey, int m, int* head) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) head[t] = (t == 0 || skey[t] != skey[t - 1]) ? 1 : 0;
}

// unique key u: segment [seg[u], seg[u+1]) of the sorted entries
__global__ void k_cond_pattern(const unsigned long long* skey, const int* head, const int* pos, int m, int nc,
                               int* ci_out, int* seg, int* rowcnt) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m && head[t]) {
        const int u = pos[t];
        ci_out[u] = int(skey[t] % nc);
        seg[u] = t;
        atomicAdd(rowcnt + int(skey[t] / nc), 1);
    }
}

// reduced block u = first entry, then += each later entry (entry order)
__global__ void __launch_bounds__(256) k_cond_merge(const int* __restrict__ seg, const int* __restrict__ sid, int nu,
                                                    int m, int nnzb, int np, const double* __restrict__ j11,
                                                    const double* __restrict__ corr, double* out) {
    const int lane = threadIdx.x & 31;
    const int u = int((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (u >= nu) return;
    const int a = seg[u], b = (u + 1 < nu) ? seg[u + 1] : m;
    const int nbb = np * np;
    for (int o = lane; o < nbb; o += 32) {
        double acc = 0.0;
        for (int t = a; t < b; ++t) {
            const int id = sid[t];
            const double v = id < nnzb ? j11[int64_t(id) * nbb + o] : corr[int64_t(id - nnzb) * nbb + o];
            acc = (t == a) ? v : acc + v;
        }
        out[int64_t(u) * nbb + o] = acc;
    }
}

// b = -r1; b[r-block] += v_e for the row's entries in list order
__global__ void k_cond_rhs(const double* __restrict__ r1, const int* __restrict__ rrp, const int* __restrict__ rlist,
                           const double* __restrict__ vrhs, int nc, int np, double* b) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= int64_t(nc) * np) return;
    const int r = int(g / np), i = int(g - int64_t(r) * np);
    double acc = -r1[g];
    for (int k = rrp[r]; k < rrp[r + 1]; ++k) acc = acc + vrhs[int64_t(rlist[k]) * np + i];
    b[g] = acc;
}

// d2_c = J22_c^-1 (-r2_c - J21_c d1_c)   (condense.cpp:243-258)
__global__ void __launch_bounds__(kCondWarps * 32) k_cond_back(const int* __restrict__ sec_off,
                                                               const int64_t* __restrict__ lu_off,
                                                               const double* __restrict__ lu,
                                                               const int* __restrict__ perm,
                                                               const double* __restrict__ j21,
                                                               const double* __restrict__ r2,
                                                               const double* __restrict__ d1, int nc, int np,
                                                               double* d2) {
    __shared__ double sm_r[kCondWarps][kMaxSec];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x * kCondWarps + w;
    if (c >= nc) return;
    const int s0 = sec_off[c], ns = sec_off[c + 1] - s0;
    if (ns == 0) return;
    double* r = sm_r[w];
    if (lane < ns) {
        const double* a = j21 + int64_t(s0) * np;  // ns x np column-major
        const double* x = d1 + int64_t(c) * np;
        double acc = a[lane] * x[0];
        for (int k = 1; k < np; ++k) acc = acc + a[int64_t(k) * ns + lane] * x[k];
        r[lane] = -r2[s0 + lane] - acc;
    }
    __syncwarp();
    if (lane == 0) {
        const double* L = lu + lu_off[c];
        double t[kMaxSec];
        for (int i = 0; i < ns; ++i) t[i] = r[perm[s0 + i]];
        for (int j = 0; j < ns; ++j) {
            const double xj = t[j];
            for (int i = j + 1; i < ns; ++i) t[i] = t[i] - L[j * ns + i] * xj;
        }
        for (int j = ns - 1; j >= 0; --j) {
            t[j] = t[j] / L[j * ns + j];
            const double xj = t[j];
            for (int i = 0; i < j; ++i) t[i] = t[i] - L[j * ns + i] * xj;
        }
        for (int i = 0; i < ns; ++i) d2[s0 + i] = t[i];
    }
}

}  // namespace

void condense(Ctx& c, const mprec_global_jacobian& j, Condensed& out) {
    const int nc = j.n_cells, np = j.np;
    if (nc < 1 || np < 1 || !j.row_ptr || !j.col_idx || !j.j11 || !j.sec_off || !j.r1)
        throw Error(MPREC_DIMENSION, "condense: incomplete GlobalJacobian");
    if (np + 1 > 32) throw Error(MPREC_DIMENSION, "condense: more than 31 primary unknowns per cell");
    const int nnzb = j.row_ptr[nc];
    // host-side validation of the index data (the reference's assemble checks)
    std::vector<int> sec(j.sec_off, j.sec_off + nc + 1);
    std::vector<int64_t> luo(nc + 1, 0);
    for (int q = 0; q < nc; ++q) {
        const int ns = sec[q + 1] - sec[q];
        if (ns < 0 || ns > kMaxSec) throw Error(MPREC_DIMENSION, "condense: secondary count per cell out of range");
        luo[q + 1] = luo[q] + int64_t(ns) * ns;
    }
    const int n2 = sec[nc];
    for (int r = 0; r < nc; ++r) {
        bool diag = false;
        for (int k = j.row_ptr[r]; k < j.row_ptr[r + 1]; ++k) {
            if (j.col_idx[k] < 0 || j.col_idx[k] >= nc) throw Error(MPREC_INDEX, "condense: J11 column out of range");
            diag = diag || j.col_idx[k] == r;
        }
        if (!diag) throw Error(MPREC_DIMENSION, "condense: J11 without a diagonal block");
    }
    // J12 entries that contribute (ns of the column cell > 0, condense.cpp:232), in list order
    std::vector<int> er, ec;
    std::vector<int64_t> eoff_all(size_t(j.n_j12) + 1, 0);
    for (int e = 0; e < j.n_j12; ++e) {
        const int r = j.j12_row[e], q = j.j12_col[e];
        if (r < 0 || r >= nc || q < 0 || q >= nc) throw Error(MPREC_INDEX, "condense: J12 cell index out of range");
        eoff_all[e + 1] = eoff_all[e] + int64_t(np) * (sec[q + 1] - sec[q]);
    }
    std::vector<int64_t> eoff;
    for (int e = 0; e < j.n_j12; ++e)
        if (sec[j.j12_col[e] + 1] > sec[j.j12_col[e]]) {
            er.push_back(j.j12_row[e]);
            ec.push_back(j.j12_col[e]);
            eoff.push_back(eoff_all[e]);
        }
    const int ne = int(er.size());
    // per block row: contributing entries in list order (b accumulation order)
    std::vector<int> rrp(nc + 1, 0), rlist(ne);
    for (int e = 0; e < ne; ++e) rrp[er[e] + 1]++;
    for (int r = 0; r < nc; ++r) rrp[r + 1] += rrp[r];
    {
        std::vector<int> fill(rrp.begin(), rrp.end() - 1);
        for (int e = 0; e < ne; ++e) rlist[fill[er[e]]++] = e;
    }

    Trace tr_all(&c, "condense total");
    std::unique_ptr<Trace> tr(new Trace(&c, "condense H2D"));
    out.nc = nc;
    out.np = np;
    out.n2 = n2;
    out.sec_off.upload(sec.data(), nc + 1, c.s);
    out.h_sec = sec;
    out.lu_off.upload(luo.data(), nc + 1, c.s);
    out.j21.upload(j.j21, size_t(n2) * np, c.s);
    out.r2.upload(j.r2, size_t(std::max(n2, 0)), c.s);
    out.lu.alloc(size_t(std::max<int64_t>(luo[nc], 1)));
    out.perm.alloc(size_t(std::max(n2, 1)));
    DBuf<double> j22(size_t(std::max<int64_t>(luo[nc], 1)));
    if (luo[nc]) j22.upload(j.j22, size_t(luo[nc]), c.s);
    DBuf<double> x(size_t(std::max<int64_t>(int64_t(n2) * (np + 1), 1)));
    DBuf<int> rp(nc + 1), ci11(std::max(nnzb, 1));
    rp.upload(j.row_ptr, nc + 1, c.s);
    ci11.upload(j.col_idx, nnzb, c.s);
    DBuf<double> j11(size_t(nnzb) * np * np);
    j11.upload(j.j11, size_t(nnzb) * np * np, c.s);
    const int64_t j12n = eoff_all[j.n_j12];
    DBuf<double> j12d(size_t(std::max<int64_t>(j12n, 1)));
    if (j12n) j12d.upload(j.j12, size_t(j12n), c.s);
    DBuf<double> r1(size_t(nc) * np);
    r1.upload(j.r1, size_t(nc) * np, c.s);
    tr.reset(new Trace(&c, "condense J22 LU + solves"));
    int* err = c.counters.p + 10;
    const int big = 0x7fffffff;
    MG_CUDA(cudaMemcpyAsync(err, &big, sizeof(int), cudaMemcpyHostToDevice, c.s));
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * double(luo[nc] + int64_t(n2) * (2 * np + 2)));
        k_cond_lu<<<(nc + kCondWarps - 1) / kCondWarps, kCondWarps * 32, 0, c.s>>>(
            out.sec_off.p, out.lu_off.p, j22.p, out.j21.p, out.r2.p, nc, np, out.lu.p, out.perm.p, x.p, err);
        check_launch("condense lu");
    }
    int bad = big;
    MG_CUDA(cudaMemcpyAsync(&bad, err, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    if (bad != big) throw Error(MPREC_SINGULAR_BLOCK, "singular secondary block", bad);

    // J12 products
    tr.reset(new Trace(&c, "condense J12 products"));
    DBuf<double> corr(size_t(std::max<int64_t>(int64_t(ne) * np * np, 1))),
        vrhs(size_t(std::max<int64_t>(int64_t(ne) * np, 1)));
    DBuf<int> d_ec(std::max(ne, 1)), d_er(std::max(ne, 1)), d_rrp(nc + 1), d_rlist(std::max(ne, 1));
    DBuf<int64_t> d_eoff(std::max(ne, 1));
    if (ne) {
        d_ec.upload(ec.data(), ne, c.s);
        d_er.upload(er.data(), ne, c.s);
        d_eoff.upload(eoff.data(), ne, c.s);
        d_rlist.upload(rlist.data(), ne, c.s);
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * double(j12n + int64_t(ne) * np * (np + 1)));
        k_cond_j12<<<int((int64_t(ne) * 32 + 255) / 256), 256, 0, c.s>>>(out.sec_off.p, d_ec.p, d_eoff.p, j12d.p, x.p,
                                                                         ne, np, corr.p, vrhs.p);
        check_launch("condense j12");
    }
    d_rrp.upload(rrp.data(), nc + 1, c.s);

    // assembly of the entry list [J11 blocks..., C_e...] (BlockMatrix::assemble)
    tr.reset(new Trace(&c, "condense assembly"));
    const int m = nnzb + ne;
    DBuf<unsigned long long> key(m), skey(m);
    DBuf<int> id(m), sid(m), head(m), pos(m + 1);
    k_cond_keys<<<(m + 255) / 256, 256, 0, c.s>>>(rp.p, ci11.p, nc, nnzb, d_er.p, d_ec.p, ne, key.p, id.p);
    int bits = 1;
    while (bits < 64 && ((unsigned long long)nc * nc) >> bits) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, skey.p, id.p, sid.p, m, 0, bits, c.s);
    DBuf<char> tmp(tb + 16);
    cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, skey.p, id.p, sid.p, m, 0, bits, c.s);
    k_cond_heads<<<(m + 255) / 256, 256, 0, c.s>>>(skey.p, m, head.p);
    size_t tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, head.p, pos.p, m + 1, c.s);
    DBuf<char> tmp2(tb2 + 16);
    // pos has m+1 entries: exclusive scan over head padded with a zero
    DBuf<int> headp(m + 1);
    MG_CUDA(cudaMemsetAsync(headp.p, 0, sizeof(int) * (m + 1), c.s));
    MG_CUDA(cudaMemcpyAsync(headp.p, head.p, sizeof(int) * m, cudaMemcpyDeviceToDevice, c.s));
    cub::DeviceScan::ExclusiveSum(tmp2.p, tb2, headp.p, pos.p, m + 1, c.s);
    int nu = 0;
    MG_CUDA(cudaMemcpyAsync(&nu, pos.p + m, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    DBuf<int> seg(nu), rowcnt(nc);
    out.pat.ci.alloc(nu);
    MG_CUDA(cudaMemsetAsync(rowcnt.p, 0, sizeof(int) * nc, c.s));
    k_cond_pattern<<<(m + 255) / 256, 256, 0, c.s>>>(skey.p, head.p, pos.p, m, nc, out.pat.ci.p, seg.p, rowcnt.p);
    out.pat.rp.alloc(nc + 1);
    {
        DBuf<int> rcp(nc + 1);
        MG_CUDA(cudaMemsetAsync(rcp.p, 0, sizeof(int) * (nc + 1), c.s));
        MG_CUDA(cudaMemcpyAsync(rcp.p, rowcnt.p, sizeof(int) * nc, cudaMemcpyDeviceToDevice, c.s));
        size_t tb3 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb3, rcp.p, out.pat.rp.p, nc + 1, c.s);
        DBuf<char> tmp3(tb3 + 16);
        cub::DeviceScan::ExclusiveSum(tmp3.p, tb3, rcp.p, out.pat.rp.p, nc + 1, c.s);
    }
    out.a_val.alloc(size_t(nu) * np * np);
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * double(int64_t(m) * np * np + int64_t(nu) * np * np));
        k_cond_merge<<<int((int64_t(nu) * 32 + 255) / 256), 256, 0, c.s>>>(seg.p, sid.p, nu, m, nnzb, np, j11.p,
                                                                           corr.p, out.a_val.p);
        check_launch("condense merge");
    }
    out.b.alloc(size_t(nc) * np);
    k_cond_rhs<<<int((int64_t(nc) * np + 255) / 256), 256, 0, c.s>>>(r1.p, d_rrp.p, d_rlist.p, vrhs.p, nc, np, out.b.p);
    check_launch("condense rhs");
    out.pat.nc = nc;
    out.pat.nnzb = nu;
    out.pat.h_rp = out.pat.rp.to_host(c.s, nc + 1);
    out.pat.h_ci = out.pat.ci.to_host(c.s, nu);
    out.pat.h_dpos.assign(nc, -1);
    for (int r = 0; r < nc; ++r)
        for (int k = out.pat.h_rp[r]; k < out.pat.h_rp[r + 1]; ++k)
            if (out.pat.h_ci[k] == r) out.pat.h_dpos[r] = k;
    out.pat.dpos.upload(out.pat.h_dpos.data(), nc, c.s);
    tr.reset();
    c.sync();
}

void back_substitute(Ctx& c, const Condensed& h, const double* d1_dev, double* d2_dev) {
    if (h.n2 == 0) return;
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * double(int64_t(h.n2) * (h.np + 2) + int64_t(h.nc) * h.np));
    k_cond_back<<<(h.nc + kCondWarps - 1) / kCondWarps, kCondWarps * 32, 0, c.s>>>(
        h.sec_off.p, h.lu_off.p, h.lu.p, h.perm.p, h.j21.p, h.r2.p, d1_dev, h.nc, h.np, d2_dev);
    check_launch("back substitute");
}

}  // namespace mg
