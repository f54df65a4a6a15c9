// scaling_exact.cu -- K3: per-cell exact left scaling (the decoupling) and
// K4 sub-system extraction.  Compiled with -fmad=false: every expression is a
// rounded multiply followed by a rounded add/sub in exactly the oracle's order
// (oracle/oracle.cpp invert_block / small_mul / combine_cell), so Ā, b̄, B_PP
// and C_TT are bitwise equal to the oracle -- they feed the AMG strength tests.
//
// Reference: scaling_factors (scaling.cpp:31-46), scale_rhs (:49-61),
// left_scale_cpr (:73-88), left_scale_cptr3 (:107-147); inverted_copy
// (block_matrix.cpp:10-30), row_combine (:201-221), extract_submatrix (:142-170).
#include "mprec.cuh"

namespace mg {
namespace {

constexpr int kMaxNb = 16;

// Eigen::PartialPivLU (unblocked) + inverse of an m x m column-major block,
// pivot tolerance 1e-12 * max|entry|.  Returns false when a pivot fails.
__device__ bool invert_small(const double* b, int m, double* inv, double* lu, int* perm) {
    double scale = 0.0;
    for (int e = 0; e < m * m; ++e) scale = fmax(scale, fabs(b[e]));  // fmax == std::max for non-NaN
    const double tol = 1e-12 * scale;
    for (int e = 0; e < m * m; ++e) lu[e] = b[e];
    for (int i = 0; i < m; ++i) perm[i] = i;
    for (int k = 0; k < m; ++k) {
        int p = k;
        double best = fabs(lu[k * m + k]);
        for (int i = k + 1; i < m; ++i)
            if (fabs(lu[k * m + i]) > best) {
                best = fabs(lu[k * m + i]);
                p = i;
            }
        if (best != 0.0) {
            if (p != k) {
                for (int j = 0; j < m; ++j) {
                    const double t = lu[j * m + k];
                    lu[j * m + k] = lu[j * m + p];
                    lu[j * m + p] = t;
                }
                const int t = perm[k];
                perm[k] = perm[p];
                perm[p] = t;
            }
            const double d = lu[k * m + k];
            for (int i = k + 1; i < m; ++i) lu[k * m + i] = lu[k * m + i] / d;
        }
        for (int j = k + 1; j < m; ++j) {
            const double ukj = lu[j * m + k];
            for (int i = k + 1; i < m; ++i) lu[j * m + i] = lu[j * m + i] - lu[k * m + i] * ukj;
        }
    }
    for (int i = 0; i < m; ++i)
        if (fabs(lu[i * m + i]) <= tol) return false;
    double t[kMaxNb];
    for (int j = 0; j < m; ++j) {
        for (int i = 0; i < m; ++i) t[i] = (perm[i] == j) ? 1.0 : 0.0;
        for (int jj = 0; jj < m; ++jj) {
            const double xj = t[jj];
            for (int i = jj + 1; i < m; ++i) t[i] = t[i] - lu[jj * m + i] * xj;
        }
        for (int jj = m - 1; jj >= 0; --jj) {
            t[jj] = t[jj] / lu[jj * m + jj];
            const double xj = t[jj];
            for (int i = 0; i < jj; ++i) t[i] = t[i] - lu[jj * m + i] * xj;
        }
        for (int i = 0; i < m; ++i) inv[j * m + i] = t[i];
    }
    return true;
}

// rows tl of every block of block row c (and of b) -= W * rows sl
__device__ void combine_cell(const int* rp, double* val, double* b, int c, int nb, const int* tl, int nt,
                             const int* sl, int ns, const double* w) {
    if (nt == 0 || ns == 0) return;
    double upd[2];
    const int nb2 = nb * nb;
    for (int k = rp[c]; k < rp[c + 1]; ++k) {
        double* blk = val + (int64_t)k * nb2;
        for (int col = 0; col < nb; ++col) {
            for (int i = 0; i < nt; ++i) {
                double acc = w[0 * nt + i] * blk[col * nb + sl[0]];
                for (int s = 1; s < ns; ++s) acc = acc + w[s * nt + i] * blk[col * nb + sl[s]];
                upd[i] = acc;
            }
            for (int i = 0; i < nt; ++i) blk[col * nb + tl[i]] = blk[col * nb + tl[i]] - upd[i];
        }
    }
    double* bc = b + (int64_t)c * nb;
    for (int i = 0; i < nt; ++i) {
        double acc = w[0 * nt + i] * bc[sl[0]];
        for (int s = 1; s < ns; ++s) acc = acc + w[s * nt + i] * bc[sl[s]];
        upd[i] = acc;
    }
    for (int i = 0; i < nt; ++i) bc[tl[i]] = bc[tl[i]] - upd[i];
}

// W (nt x ns, column-major) = D_ts * inv(D_ss) from the diagonal block
__device__ void scaling_w(const double* d, int nb, const int* tl, int nt, const int* sl, int ns, const double* inv,
                          double* w) {
    for (int i = 0; i < nt; ++i)
        for (int j = 0; j < ns; ++j) {
            double acc = d[sl[0] * nb + tl[i]] * inv[j * ns + 0];
            for (int k = 1; k < ns; ++k) acc = acc + d[sl[k] * nb + tl[i]] * inv[j * ns + k];
            w[j * nt + i] = acc;
        }
}

// CPR (scaling.cpp:73-88): P rows -= (D_Ph D_hh^-1) * h rows, h = s..., T.
// scalar_diag: DiagMode::Scalar -- D_hh is the diagonal of the cell block
// (block_diagonal_of, block_matrix.cpp:186-193); D_Ph stays the full block.
__global__ void k_scale_cpr(const int* rp, const int* dpos, double* val, double* b, int nc, int nb, int* err,
                            int scalar_diag) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const int ns = nb - 2, P = nb - 2, T = nb - 1, m = ns + 1;
    int sl[kMaxNb], tl[1] = {P}, perm[kMaxNb];
    for (int k = 0; k < ns; ++k) sl[k] = k;
    sl[ns] = T;
    double dss[kMaxNb * kMaxNb], lu[kMaxNb * kMaxNb], inv[kMaxNb * kMaxNb], w[kMaxNb];
    const double* d = val + (int64_t)dpos[c] * nb * nb;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) dss[j * m + i] = (scalar_diag && i != j) ? 0.0 : d[sl[j] * nb + sl[i]];
    if (!invert_small(dss, m, inv, lu, perm)) {
        atomicMin(err + 0, c);
        return;
    }
    scaling_w(d, nb, tl, 1, sl, m, inv, w);
    combine_cell(rp, val, b, c, nb, tl, 1, sl, m, w);
}

// CPTR3 (scaling.cpp:107-147): e = {P,T} rows -= (D_es D_ss^-1) * s rows, then
// T rows -= (D_Tp * (1/D_PP)) * P rows on the once-scaled block row; D_PP of
// the once-scaled row or, with second_scaling_from_original (scaling.cpp:126),
// of the original A (orig).
__global__ void k_scale_cptr3(const int* rp, const int* dpos, double* val, double* b, int nc, int nb, int* err,
                              int second, int scalar_diag, const double* orig) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const int ns = nb - 2, P = nb - 2, T = nb - 1;
    double* d = val + (int64_t)dpos[c] * nb * nb;
    if (ns > 0) {
        int sl[kMaxNb], tl[2] = {P, T}, perm[kMaxNb];
        for (int k = 0; k < ns; ++k) sl[k] = k;
        double dss[kMaxNb * kMaxNb], lu[kMaxNb * kMaxNb], inv[kMaxNb * kMaxNb], w[2 * kMaxNb];
        for (int j = 0; j < ns; ++j)
            for (int i = 0; i < ns; ++i) dss[j * ns + i] = (scalar_diag && i != j) ? 0.0 : d[sl[j] * nb + sl[i]];
        if (!invert_small(dss, ns, inv, lu, perm)) {
            atomicMin(err + 0, c);
            return;
        }
        scaling_w(d, nb, tl, 2, sl, ns, inv, w);
        combine_cell(rp, val, b, c, nb, tl, 2, sl, ns, w);
    }
    if (!second) return;  // CPTR (scaling.cpp:90-105): first scaling only
    const double pp = orig ? orig[(int64_t)dpos[c] * nb * nb + P * nb + P] : d[P * nb + P];
    // inverted_copy of the 1x1 block: tol = 1e-12|pp| -> fails iff |pp| <= tol
    if (fabs(pp) <= 1e-12 * fabs(pp)) {
        atomicMin(err + 1, c);
        return;
    }
    const double w2 = d[P * nb + T] * (1.0 / pp);
    const int tl2[1] = {T}, sl2[1] = {P};
    combine_cell(rp, val, b, c, nb, tl2, 1, sl2, 1, &w2);
}

__global__ void k_extract(const double* val, int nnzb, int nb, int f, double* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnzb) out[k] = val[((int64_t)k * nb + f) * nb + f];
}

// extract_submatrix({P,T},{P,T}) as CSR (2 n_c rows, cell-interleaved P,T)
__global__ void k_extract_pt(const int* rp, const int* ci, const double* val, int nc, int nb, int* erp, int* eci,
                             double* ev) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * nc) return;
    const int c = t >> 1, r = t & 1;
    const int P = nb - 2, fr = r ? nb - 1 : P;
    const int nblk = rp[c + 1] - rp[c];
    int o = 4 * rp[c] + r * 2 * nblk;
    erp[t] = o;
    if (t == 2 * nc - 1) erp[2 * nc] = 4 * rp[nc];
    for (int k = rp[c]; k < rp[c + 1]; ++k)
        for (int q = 0; q < 2; ++q) {
            eci[o] = 2 * ci[k] + q;
            ev[o] = val[((int64_t)k * nb + (q ? nb - 1 : P)) * nb + fr];
            ++o;
        }
}

}  // namespace

void extract_pt(Ctx& c, const BsrView& a, int* erp, int* eci, double* ev) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 40.0 * a.nnzb);
    k_extract_pt<<<(2 * a.nc + 255) / 256, 256, 0, c.s>>>(a.rp, a.ci, a.val, a.nc, a.nb, erp, eci, ev);
    check_launch("extract_pt");
}

void left_scale(Ctx& c, const BsrView& a, double* bbar, int method, int scalar_diag, const double* orig_for_pp) {
    if (method == MPREC_METHOD_ILU0) return;
    if (a.nb < 2) throw Error(MPREC_DIMENSION, "CPR/CPTR3 need P and T unknowns (nb >= 2)");
    if (a.nb > kMaxNb) throw Error(MPREC_DIMENSION, "nb > 16 not supported by the scaling kernel");
    const int big = 0x7fffffff;
    int h_err[2] = {big, big};
    MG_CUDA(cudaMemcpyAsync(c.err.p, h_err, sizeof(h_err), cudaMemcpyHostToDevice, c.s));
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 2.0 * a.nnzb * 8.0 * a.nb * a.nb);
        const int th = 128, g = (a.nc + th - 1) / th;
        if (method == MPREC_METHOD_CPR_AMG || method == MPREC_METHOD_CPR_DIRECT)
            k_scale_cpr<<<g, th, 0, c.s>>>(a.rp, a.dpos, a.val, bbar, a.nc, a.nb, c.err.p, scalar_diag);
        else if (method == MPREC_METHOD_CPTR3_AMG || method == MPREC_METHOD_CPTR3_DIRECT ||
                 method == MPREC_METHOD_CPTR_DIRECT)
            k_scale_cptr3<<<g, th, 0, c.s>>>(a.rp, a.dpos, a.val, bbar, a.nc, a.nb, c.err.p,
                                             method != MPREC_METHOD_CPTR_DIRECT, scalar_diag, orig_for_pp);
        else
            throw Error(MPREC_CONFIG, "unknown method id " + std::to_string(method));
        check_launch("left_scale");
    }
    MG_CUDA(cudaMemcpyAsync(h_err, c.err.p, sizeof(h_err), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    if (h_err[0] != big) {
        const char* what = (method == MPREC_METHOD_CPR_AMG || method == MPREC_METHOD_CPR_DIRECT) ? "D_hh" : "D_ss";
        throw Error(MPREC_SINGULAR_BLOCK, std::string("singular ") + what + " block in cell " + std::to_string(h_err[0]),
                    h_err[0]);
    }
    if (h_err[1] != big)
        throw Error(MPREC_SINGULAR_BLOCK, "singular D_PP block in cell " + std::to_string(h_err[1]), h_err[1]);
}

void extract_field(Ctx& c, const BsrView& a, int f, double* vals) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * a.nnzb);
    k_extract<<<(a.nnzb + 255) / 256, 256, 0, c.s>>>(a.val, a.nnzb, a.nb, f, vals);
    check_launch("extract_field");
}

}  // namespace mg
