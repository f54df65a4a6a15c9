// mprec.cuh -- internal C++ interface of libmprec_gpu.so (device data
// structures and kernel launchers).  The C ABI (include/mprec_gpu.h) is
// implemented on top of this in capi.cu.
#pragma once

#include <memory>

#include "common.cuh"

namespace mg {

// Sentinel written into the output vectors of the dependency-scheduled sweeps
// (ILU(0) solves, Gauss-Seidel) before a sweep: a signalling NaN that IEEE
// arithmetic never produces, so a consumer can poll the value itself.
constexpr unsigned long long kPending = 0xFFF4DEADBEEFCAFEull;

// ---- views -------------------------------------------------------------------
struct BsrView {
    int nc = 0, nb = 0, nnzb = 0;
    const int* rp = nullptr;
    const int* ci = nullptr;
    const int* dpos = nullptr;
    double* val = nullptr;  // column-major nb x nb blocks
};

struct CsrView {
    int n = 0, m = 0, nnz = 0;  // rows, cols, nonzeros
    const int* rp = nullptr;
    const int* ci = nullptr;
    const double* v = nullptr;
    const int* diag = nullptr;  // position of the diagonal entry per row (square only)
};

// Topological claim order of a sweep's dependency DAG (sched.cu).
struct Sched {
    DBuf<int> order;
    DBuf<int> level;  // DAG level (Kahn round) of every row
    int n = 0;
    int nlev = 0;
};
// dir = +1: row i depends on stored k < i; dir = -1: on stored k > i.
void build_sched(Ctx& c, int n, const int* rp, const int* ci, int dir, Sched& out);

// Block pattern shared by A, Ā, the ILU(0) factors and (as a scalar pattern)
// the level-0 operators B_PP / C_TT of both AMG hierarchies.
struct Pattern {
    int nc = 0, nnzb = 0;
    DBuf<int> rp, ci, dpos;
    std::vector<int> h_rp, h_ci, h_dpos;
    Sched fwd, bwd;
    bool sched_built = false;
    void ensure_sched(Ctx& c) {
        if (sched_built) return;
        build_sched(c, nc, rp.p, ci.p, +1, fwd);
        build_sched(c, nc, rp.p, ci.p, -1, bwd);
        sched_built = true;
    }
};

// Owned CSR.
struct DCsr {
    int n = 0, m = 0, nnz = 0;
    DBuf<int> rp, ci, diag;
    DBuf<double> v;
    CsrView view() const { return CsrView{n, m, nnz, rp.p, ci.p, v.p, diag.p}; }
};

// ---- blas.cu -----------------------------------------------------------------
void fill(Ctx& c, double* x, double val, int64_t n);
void fill_pending(Ctx& c, double* x, int64_t n);
void copy(Ctx& c, double* y, const double* x, int64_t n);
// out_dev <- sum a_i b_i (deterministic fixed-order two-level reduction)
void dot(Ctx& c, const double* a, const double* b, int64_t n, double* out_dev);
// out_dev <- ||a||_2
void nrm2(Ctx& c, const double* a, int64_t n, double* out_dev);
// Gram-form MGS sweep (gram.cu): with the basis v_0..v_k (device pointer table
// vt), h = (I + L)^-1 V^T w (h += when accumulate), w -= V h; gt (ld x ld,
// transposed Gram lower part) gains the row of v_k when want_q; pre_norm =
// ||w|| before (when non-null), post_norm = ||w|| after.  Gated on *gate.
// The Krylov basis is stored in chunks of kBasisChunk vectors, tile-major
// ([tile][vector][kBasisTile rows]); tab[c] = chunk c.
constexpr int kBasisTile = 2048;
constexpr int kBasisChunk = 8;
int64_t basis_chunk_doubles(int64_t n);
void gram_set_ptr(Ctx& c, double** tab, int i, double* p);
void basis_put(Ctx& c, double* chunk, int j, const double* x, double a, int64_t n);  // v_j = x / a
void basis_get(Ctx& c, double* y, const double* chunk, int j, int64_t n);
void basis_combine(Ctx& c, const double* const* ct, int k, const double* y, double* z, int64_t n);  // z = V_k y
int gram_part_size(Ctx& c, int kmax);
void gram_orthogonalise(Ctx& c, const double* const* ct, int k, double* w, int64_t n, double* gt, int ld,
                        double* pbuf, double* h, double* pre_norm, double* post_norm, double* reorth_norm,
                        double* part, int* gate);
void gram_sweep(Ctx& c, const double* const* vt, int k, double* w, int64_t n, double* gt, int ld, double* pbuf,
                double* h, bool accumulate, bool want_q, double* pre_norm, double* post_norm, double* part,
                const int* gate);
// gate_dev <- (||w|| < 0.7 * pre_norm) evaluated on device scalars
void set_reorth_gate(Ctx& c, const double* wnorm, const double* prenorm, int* gate);
// out = b - ax ; optional
void sub(Ctx& c, double* out, const double* b, const double* ax, int64_t n);
// out[c] = x[c*stride + f]
void gather_stride(Ctx& c, double* out, const double* x, int nc, int stride, int f);
// y[i] = w[i] + s[i] where s is the scatter of the stage solutions (xs on field fx,
// vs on field fv; either may be null)
void stage_combine(Ctx& c, double* y, const double* w, const double* xs, int fx, const double* vs, int fv,
                   int nc, int nb);
// two-field (P,T) gather / zero-padded scatter of cell-interleaved sub-vectors (CPTR scope)
void gather_pt(Ctx& c, double* out, const double* x, int nc, int nb);
void add2(Ctx& c, double* y, const double* a, const double* b, int64_t n);  // y = a + b
void scatter_pt(Ctx& c, double* y, const double* sub, int nc, int nb);

// ---- bsr.cu ------------------------------------------------------------------
// y = A x  or  y = b - A x  (b != nullptr); flat (scalar-CSR) semantics
void bsr_spmv(Ctx& c, const BsrView& a, const double* x, double* y, const double* b, int kclass);
// z = r - A[:, field f] xs  (xs: one value per cell = the stage solution scattered
// to field f); optionally gather zsub[c] = z[c*nb + g]
void bsr_col_update(Ctx& c, const BsrView& a, int f, const double* xs, const double* r, double* z,
                    double* zsub, int g);

// ---- scaling.cu --------------------------------------------------------------
// In-place left scaling of Ā and b̄ (scaling.cpp:73-147); throws mg::Error
// (SINGULAR_BLOCK with the reference's tag and cell) after synchronising.
// scalar_diag: ScalingOptions::diag_mode == Scalar; orig_for_pp: the original
// A's values when second_scaling_from_original (else nullptr)
void left_scale(Ctx& c, const BsrView& abar, double* bbar, int method, int scalar_diag = 0,
                const double* orig_for_pp = nullptr);
// vals[k] = A_k(f, f)  (extract_submatrix on a single field, pattern = block pattern)
void extract_field(Ctx& c, const BsrView& a, int f, double* vals);
// B_ee (CPTR): CSR with 2 n_c rows, cell-interleaved (P, T); erp[2nc+1], eci/ev[4 nnzb]
void extract_pt(Ctx& c, const BsrView& a, int* erp, int* eci, double* ev);

// ---- ilu.cu ------------------------------------------------------------------
// Level-synchronous block ILU(0) solve programs (ilu_ls.cu, nb = 8).
struct IluLs {
    bool ok = false, filled = false;
    int K = 0, W = 0, hmax = 0, nsteps = 0, smem = 0, nc = 0;
    DBuf<int4> meta;            // per step: header + row metadata (ilu_ls.cu)
    DBuf<int> scnt;             // rows per step
    DBuf<int2> gst, gimp;       // per group: (first step, steps), (import offset, count)
    DBuf<long long> gdoff;      // per group: byte offset of its data
    DBuf<int> imp;              // per group: block rows imported from the previous group
    DBuf<long long> roff;       // per block row: byte offset of its record in `data`
    DBuf<int2> kdep;            // per block row: BSR indices of its two dependency blocks
    DBuf<char> data;            // the solve stream: per row B0, B1, packed inverse, rhs
};
bool build_ilu_ls(Ctx& c, Pattern& pat, int K, IluLs& fwd, IluLs& bwd);
void ilu_ls_fill(Ctx& c, IluLs& s, const double* val, const double* dinv);
void ilu_ls_solve(Ctx& c, IluLs& s, bool fwd, const double* rhs, double* y);

struct Ilu {
    BsrView lu;           // values owned elsewhere (or by `own`)
    DBuf<double> own;     // factor storage when the Ilu owns it
    DBuf<double> ybuf;    // forward-sweep output
    DBuf<int> flags;      // factorisation ready flags
    DBuf<double> dinv;    // nb = 8: packed inverses of the diagonal blocks (apply path)
    IluLs ls_fwd, ls_bwd; // nb = 8: level-synchronous solve programs (when the pattern fits)
    Pattern* pat = nullptr;
    int n = 0;
    // factor in place (values of lu are overwritten by L\U); throws ZERO_PIVOT/SETUP
    void factor(Ctx& c);
    // y = U^-1 L^-1 r  (ilu0.cpp:41-59); y must not alias r
    void apply(Ctx& c, const double* r, double* y);
};

// ---- amg.cu ------------------------------------------------------------------
struct AmgParams {
    double theta = 0.25;
    int max_coarse = 1000;
    int max_levels = 25;
};

// Level-synchronous pipelined sweep schedule (gs_ls.cu): K groups of
// consecutive rows, each a stream of fixed-size program steps processed by nw
// compute warps of one thread block.
struct LsSched {
    bool ok = false;
    int K = 0, W = 0, hmax = 0, dir = 0, nsteps = 0, nchunks = 0, maxdist = 0, smem = 0, nd = 0, ns = 0, cls = 0;
    int nw = 0, spc = 0, chb = 0;  // compute warps per group, steps per chunk, chunk bytes
    DBuf<char> prog;       // K groups' chunks
    DBuf<int2> gch;        // per group: first chunk, chunk count
    DBuf<int> imp;         // per group: rows imported (previous group's, own far rows) in consumer order
    DBuf<int2> gimp;       // per group: offset, count into imp
    DBuf<long long> coff;  // per row: byte offset of its c' slot in prog | export bit
};
// both directions (one download of the level, two host threads); nd = 0: the
// dependency class is chosen from the level, else 2 / 4 / 8
bool build_ls_pair(Ctx& c, const CsrView& a, const double* invd, int K, int nw, int nd, LsSched& fwd, LsSched& bwd);
void gs_sweep_ls(Ctx& c, const CsrView& a, const double* invd, const double* b, const double* xold, double* xnew,
                 bool xold_zero, const LsSched& s);

struct AmgLevel {
    int n = 0;
    const int* glev_f = nullptr;      // global DAG levels of the sweep directions
    const int* glev_b = nullptr;
    LsSched ls_fwd, ls_bwd;           // level-synchronous sweep programs (gs_ls.cu)
    CsrView a;            // level operator (level 0 may be a non-owning view)
    DCsr a_own, p, r;     // p/r: interpolation into the finer level (levels >= 1)
    DBuf<signed char> cf; // C/F splitting of this level (levels < last)
    DBuf<double> x, b, t, xf, xb;  // work vectors
    Sched own_fwd, own_bwd;           // Gauss-Seidel claim orders
    const int* ofwd = nullptr;        // (level 0 may borrow the block pattern's)
    const int* obwd = nullptr;
    DBuf<double> invd;                // 1 / a_ii
    DBuf<int> border_f, border_b;     // cluster sweep: rows per CTA band in global level order
    int cl_size = 0, cl_R = 0;        // cluster sweep (gs_cluster.cu): CTAs, rows per CTA
};

struct Amg {
    AmgParams prm;
    std::vector<std::unique_ptr<AmgLevel>> lv;
    DBuf<double> coarse_inv;  // row-major inverse of the coarsest operator
    DBuf<double> coarse_lu;   // LU factors (diagnostic / parity)
    int nco = 0;
    DCsr a0_copy;             // when the caller's matrix must be owned
    // AMGHierarchy::setup (amg.cpp:188-214). a0 must stay alive; `pat`
    // (optional) supplies level 0's sweep schedules when a0 has its pattern.
    void setup(Ctx& c, const CsrView& a0, const AmgParams& p, Pattern* pat = nullptr);
    // AMGHierarchy::apply (amg.cpp:233-238): x = V(1,1)-cycle(r), zero initial guess.
    void apply(Ctx& c, const double* r, double* x);
    int n_levels() const { return int(lv.size()); }
   private:
    void cycle(Ctx& c, int l, const double* r, double* x);
};

// csr.cu helpers
void csr_spmv(Ctx& c, const CsrView& a, const double* x, double* y, const double* b, bool add_to_y,
              int kclass);
// forward (dir=+1) / backward (dir=-1) Gauss-Seidel sweep, dependency scheduled
// invd (optional): precomputed 1/a_ii (multiply instead of the fp64 division)
void gs_sweep(Ctx& c, const CsrView& a, const double* b, const double* xold, double* xnew, int dir,
              bool xold_zero, const int* order, const double* invd = nullptr);
void dense_gemv(Ctx& c, const double* m_rowmajor, int n, const double* x, double* y);
void compute_invd(Ctx& c, const CsrView& a, double* invd);
void build_band_order(Ctx& c, int n, const int* lev, int B, DBuf<int>& border);
bool csr_sorted(Ctx& c, const CsrView& a);
int gs_cluster_plan(int n, int* rows_per_cta, int min_cs = 1);
void gs_sweep_cluster(Ctx& c, const CsrView& a, const double* invd, const double* b, const double* xold, double* xnew,
                      int dir, bool xold_zero, const int* border, int csize, int R);
void tune_level_sweep(Ctx& c, AmgLevel& L, const Sched& sf, const Sched& sb);

}  // namespace mg
