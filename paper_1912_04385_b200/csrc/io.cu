// io.cu -- ingestion of the reference's on-disk system format straight into a
// device BSR: Matrix Market "coordinate real general"
// (1-based, %.17g) + layout sidecar (`n_unknowns n_cells`, then `<cell> <s|P|T>`
// per unknown) + rhs (one value per line) -- read_matrix_market /
// read_layout / read_vector (proj/src/matrix_io.cpp:40-121) and ingest_external
// (harness.cpp:153-188), and the writers (matrix_io.cpp:31-38, 67-72, 111-114).
//
// Text is parsed on the host (it is text); the scalar triplets are then
// canonicalised and assembled into nb x nb column-major blocks ON THE DEVICE
// (radix sort by (row, col) -- stable, so duplicates are summed in file order
// like the oracle's stable sort -- then block keys, diagonal insertion as in
// BlockMatrix::assemble, and a scatter of the values).
#include <cub/cub.cuh>

#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "mprec.cuh"

namespace mg {
namespace {

struct File {
    FILE* f = nullptr;
    explicit File(const char* p, const char* mode) : f(std::fopen(p, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

[[noreturn]] void io_fail(const std::string& m) { throw Error(MPREC_IO, m); }

// (row*n + col) keys -> sorted, duplicate-summed scalar CSR pieces on the device
__global__ void k_keys(const int* r, const int* c, int nnz, int n, unsigned long long* key) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nnz) key[t] = (unsigned long long)r[t] * (unsigned long long)n + (unsigned long long)c[t];
}

__global__ void k_seg_flags(const unsigned long long* key, int nnz, int* flag) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nnz) flag[t] = (t == 0 || key[t] != key[t - 1]) ? 1 : 0;
}

// one thread per unique entry: sum the duplicates in (stable) file order
__global__ void k_seg_sum(const unsigned long long* key, const double* v, const int* flag, const int* pos, int nnz,
                          unsigned long long* ukey, double* uval) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nnz || !flag[t]) return;
    double s = 0.0;
    int e = t;
    do {
        s += v[e];
        ++e;
    } while (e < nnz && !flag[e]);
    ukey[pos[t]] = key[t];
    uval[pos[t]] = s;
}

// block key per unique entry (uniform layout: cell = index / nb)
__global__ void k_block_keys(const unsigned long long* ukey, int nu, int n, int nb, int nc, unsigned long long* bkey) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nu + nc) {
        if (t < nu) {
            const int i = int(ukey[t] / (unsigned long long)n), j = int(ukey[t] % (unsigned long long)n);
            bkey[t] = (unsigned long long)(i / nb) * (unsigned long long)nc + (unsigned long long)(j / nb);
        } else {
            const int c = t - nu;  // BlockMatrix::assemble: diagonal block always present
            bkey[t] = (unsigned long long)c * (unsigned long long)nc + (unsigned long long)c;
        }
    }
}

__global__ void k_bsr_pattern(const unsigned long long* bkey, const int* flag, const int* pos, int m, int nc,
                              int* ci, int* rowcnt) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m || !flag[t]) return;
    const int r = int(bkey[t] / (unsigned long long)nc), c = int(bkey[t] % (unsigned long long)nc);
    ci[pos[t]] = c;
    atomicAdd(rowcnt + r, 1);
}

__global__ void k_bsr_scatter(const unsigned long long* ukey, const double* uval, int nu, int n, int nb,
                              const int* rp, const int* ci, double* val) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nu) return;
    const int i = int(ukey[t] / (unsigned long long)n), j = int(ukey[t] % (unsigned long long)n);
    const int ri = i / nb, cj = j / nb;
    int lo = rp[ri], hi = rp[ri + 1];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ci[mid] < cj)
            lo = mid + 1;
        else
            hi = mid;
    }
    val[((int64_t)lo * nb + (j % nb)) * nb + (i % nb)] = uval[t];
}

template <class T>
int scan_total(Ctx& c, const T* in, T* out, int n) {
    MG_CUDA(cudaMemsetAsync(out, 0, sizeof(T), c.s));
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out + 1, n, c.s);
    DBuf<char> tmp(bytes + 16);
    cub::DeviceScan::InclusiveSum(tmp.p, bytes, in, out + 1, n, c.s);
    T tot{};
    MG_CUDA(cudaMemcpyAsync(&tot, out + n, sizeof(T), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    return int(tot);
}

}  // namespace

// Parses the three files; returns the uniform layout (n_cells, nb, P/T present)
// and the device BSR (pattern uploaded into `pat`, values into `val`), rhs on host.
void ingest(Ctx& c, const char* mtx, const char* layout, const char* rhs, Pattern& pat, DBuf<double>& val, int* n_cells,
            int* nb_out, std::vector<double>& b) {
    // ---- layout sidecar (matrix_io.cpp:74-91, field_layout.cpp:30-73)
    int nu = 0, nc = 0;
    {
        File f(layout, "r");
        if (!f.f) io_fail(std::string("cannot open '") + layout + "' for reading");
        if (std::fscanf(f.f, "%d %d", &nu, &nc) != 2) io_fail(std::string(layout) + ": bad layout header");
        std::vector<int> cell(nu);
        std::vector<char> tag(nu);
        for (int g = 0; g < nu; ++g) {
            char t[8];
            if (std::fscanf(f.f, "%d %7s", &cell[g], t) != 2) io_fail(std::string(layout) + ": truncated layout");
            tag[g] = t[0];
            if (tag[g] != 's' && tag[g] != 'P' && tag[g] != 'T')
                io_fail(std::string("unknown field tag '") + t[0] + "'");
        }
        if (nc < 1) io_fail(std::string(layout) + ": header cell count disagrees with tag list");
        // uniform layout with P and T in every cell (ingest_external, harness.cpp:162-167)
        int nb = -1, g = 0;
        for (int cc = 0; cc < nc; ++cc) {
            int ns = 0, k0 = g;
            if (g >= nu || cell[g] != cc) io_fail("layout cells must be contiguous and ascending");
            while (g < nu && cell[g] == cc && tag[g] == 's') ++ns, ++g;
            if (!(g < nu && cell[g] == cc && tag[g] == 'P'))
                io_fail("cell " + std::to_string(cc) + " has no pressure unknown");
            ++g;
            if (!(g < nu && cell[g] == cc && tag[g] == 'T'))
                io_fail("cell " + std::to_string(cc) + " has no temperature unknown");
            ++g;
            if (g < nu && cell[g] == cc) io_fail("intra-cell order must be s..., P, T");
            const int sz = g - k0;
            if (nb < 0) nb = sz;
            if (sz != nb) throw Error(MPREC_DIMENSION, "non-uniform layout: the B200 path needs a uniform nb");
        }
        if (g != nu) io_fail(std::string(layout) + ": header cell count disagrees with tag list");
        *n_cells = nc;
        *nb_out = nb;
    }
    const int nb = *nb_out, n = nc * nb;
    // ---- Matrix Market (matrix_io.cpp:40-65)
    std::vector<int> ri, cj;
    std::vector<double> vv;
    {
        File f(mtx, "r");
        if (!f.f) io_fail(std::string("cannot open '") + mtx + "' for reading");
        char line[4096];
        if (!std::fgets(line, sizeof line, f.f)) io_fail(std::string(mtx) + ": empty file");
        char banner[64] = {0}, object[64] = {0}, format[64] = {0}, type[64] = {0}, sym[64] = {0};
        if (std::sscanf(line, "%63s %63s %63s %63s %63s", banner, object, format, type, sym) != 5 ||
            std::strcmp(banner, "%%MatrixMarket") || std::strcmp(object, "matrix") ||
            std::strcmp(format, "coordinate") || std::strcmp(type, "real") || std::strcmp(sym, "general"))
            io_fail(std::string(mtx) + ": expected 'matrix coordinate real general' header");
        do {
            if (!std::fgets(line, sizeof line, f.f)) io_fail(std::string(mtx) + ": bad size line");
        } while (line[0] == '%' || line[0] == '\n');
        int rows = 0, cols = 0, nnz = 0;
        if (std::sscanf(line, "%d %d %d", &rows, &cols, &nnz) != 3) io_fail(std::string(mtx) + ": bad size line");
        if (rows != cols) io_fail(std::string(mtx) + ": block matrix must be square");
        if (rows != n) throw Error(MPREC_DIMENSION, "scalar matrix does not match layout dimension");
        ri.resize(nnz);
        cj.resize(nnz);
        vv.resize(nnz);
        for (int k = 0; k < nnz; ++k) {
            if (std::fscanf(f.f, "%d %d %lf", &ri[k], &cj[k], &vv[k]) != 3)
                io_fail(std::string(mtx) + ": truncated entry list");
            --ri[k];
            --cj[k];
            if (ri[k] < 0 || ri[k] >= n || cj[k] < 0 || cj[k] >= n) throw Error(MPREC_INDEX, "triplet index out of range");
        }
    }
    // ---- rhs (matrix_io.cpp:116-121)
    {
        File f(rhs, "r");
        if (!f.f) io_fail(std::string("cannot open '") + rhs + "' for reading");
        b.clear();
        double x;
        while (std::fscanf(f.f, "%lf", &x) == 1) b.push_back(x);
        if (int64_t(b.size()) != int64_t(n))
            io_fail("rhs dimension " + std::to_string(b.size()) + " does not match matrix dimension " +
                    std::to_string(n));
    }
    // ---- device assembly (from_triplets + BlockMatrix::from_scalar + assemble)
    const int nnz = int(ri.size());
    DBuf<int> dr, dc;
    DBuf<double> dv;
    dr.upload(ri.data(), std::max(nnz, 1), c.s);
    dc.upload(cj.data(), std::max(nnz, 1), c.s);
    dv.upload(vv.data(), std::max(nnz, 1), c.s);
    DBuf<unsigned long long> key(std::max(nnz, 1)), skey(std::max(nnz, 1));
    DBuf<double> sval(std::max(nnz, 1));
    auto nbk = [](int64_t m) { return int(std::max<int64_t>(1, (m + 255) / 256)); };
    k_keys<<<nbk(nnz), 256, 0, c.s>>>(dr.p, dc.p, nnz, n, key.p);
    {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, skey.p, dv.p, sval.p, nnz, 0, 64, c.s);
        DBuf<char> tmp(bytes + 16);
        cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, skey.p, dv.p, sval.p, nnz, 0, 64, c.s);
        check_launch("ingest sort");
    }
    DBuf<int> flag(std::max(nnz, 1)), pos(nnz + 1);
    k_seg_flags<<<nbk(nnz), 256, 0, c.s>>>(skey.p, nnz, flag.p);
    const int nuq = nnz ? scan_total(c, flag.p, pos.p, nnz) : 0;
    DBuf<unsigned long long> ukey(std::max(nuq, 1));
    DBuf<double> uval(std::max(nuq, 1));
    k_seg_sum<<<nbk(nnz), 256, 0, c.s>>>(skey.p, sval.p, flag.p, pos.p, nnz, ukey.p, uval.p);
    // block keys (+ every diagonal block), sorted and de-duplicated
    const int m = nuq + nc;
    DBuf<unsigned long long> bkey(m), sbkey(m);
    k_block_keys<<<nbk(m), 256, 0, c.s>>>(ukey.p, nuq, n, nb, nc, bkey.p);
    {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, bytes, bkey.p, sbkey.p, m, 0, 64, c.s);
        DBuf<char> tmp(bytes + 16);
        cub::DeviceRadixSort::SortKeys(tmp.p, bytes, bkey.p, sbkey.p, m, 0, 64, c.s);
    }
    DBuf<int> bflag(m), bpos(m + 1), rowcnt(nc);
    k_seg_flags<<<nbk(m), 256, 0, c.s>>>(sbkey.p, m, bflag.p);
    const int nnzb = scan_total(c, bflag.p, bpos.p, m);
    MG_CUDA(cudaMemsetAsync(rowcnt.p, 0, rowcnt.bytes(), c.s));
    pat.ci.alloc(nnzb);
    k_bsr_pattern<<<nbk(m), 256, 0, c.s>>>(sbkey.p, bflag.p, bpos.p, m, nc, pat.ci.p, rowcnt.p);
    pat.rp.alloc(nc + 1);
    scan_total(c, rowcnt.p, pat.rp.p, nc);
    val.alloc(size_t(nnzb) * nb * nb);
    MG_CUDA(cudaMemsetAsync(val.p, 0, val.bytes(), c.s));
    k_bsr_scatter<<<nbk(nuq), 256, 0, c.s>>>(ukey.p, uval.p, nuq, n, nb, pat.rp.p, pat.ci.p, val.p);
    check_launch("ingest assemble");
    pat.nc = nc;
    pat.nnzb = nnzb;
    pat.h_rp = pat.rp.to_host(c.s, nc + 1);
    pat.h_ci = pat.ci.to_host(c.s, nnzb);
    pat.h_dpos.assign(nc, -1);
    for (int r = 0; r < nc; ++r)
        for (int k = pat.h_rp[r]; k < pat.h_rp[r + 1]; ++k)
            if (pat.h_ci[k] == r) pat.h_dpos[r] = k;
    pat.dpos.upload(pat.h_dpos.data(), nc, c.s);
    c.sync();
}

// write_block_matrix + write_vector (matrix_io.cpp:31-38, 67-72, 93-97, 111-114)
void write_system(const char* mtx, const char* layout, const char* rhs, int nc, int nb, const std::vector<int>& rp,
                  const std::vector<int>& ci, const std::vector<double>& val, const double* b) {
    const int n = nc * nb;
    {
        File f(mtx, "w");
        if (!f.f) io_fail(std::string("cannot open '") + mtx + "' for writing");
        std::fprintf(f.f, "%%%%MatrixMarket matrix coordinate real general\n%d %d %lld\n", n, n,
                     (long long)rp[nc] * nb * nb);
        for (int cc = 0; cc < nc; ++cc)
            for (int r = 0; r < nb; ++r)
                for (int k = rp[cc]; k < rp[cc + 1]; ++k)
                    for (int q = 0; q < nb; ++q)
                        std::fprintf(f.f, "%d %d %.17g\n", cc * nb + r + 1, ci[k] * nb + q + 1,
                                     val[((size_t)k * nb + q) * nb + r]);
    }
    {
        File f(layout, "w");
        if (!f.f) io_fail(std::string("cannot open '") + layout + "' for writing");
        std::fprintf(f.f, "%d %d\n", n, nc);
        for (int cc = 0; cc < nc; ++cc)
            for (int r = 0; r < nb; ++r) std::fprintf(f.f, "%d %c\n", cc, r < nb - 2 ? 's' : (r == nb - 2 ? 'P' : 'T'));
    }
    if (rhs && b) {
        File f(rhs, "w");
        if (!f.f) io_fail(std::string("cannot open '") + rhs + "' for writing");
        for (int i = 0; i < n; ++i) std::fprintf(f.f, "%.17g\n", b[i]);
    }
}

}  // namespace mg
