// mprec_gen.cpp -- see mprec_gen.h for the contract and the builder decisions.
#include "mprec_gen.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

enum Stream : uint64_t {
    S_PERM = 1,   // permeability normal draw per cell
    S_EPS = 2,    // seed-field noise per cell
    S_FLUX = 3,   // flux block entries per cell
    S_ACCD = 4,   // accumulation diagonal per (cell,row)
    S_ACCO = 5,   // accumulation off-diagonal factor per (cell,row,col)
    S_BANDT = 6,  // reaction band T-column multiplier per (cell,row)
    S_BANDC = 7,  // reaction band component-component factor per (cell,row,col)
    S_XSTAR = 8,  // exact solution per unknown
};

inline uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Portable elementary functions built only from IEEE +,-,*,/ and frexp/ldexp
// (compiled with -ffp-contract=off), so generated systems are bit-identical on
// any x86-64 host regardless of which libm variant the loader picks.
const double kLn2 = 0.6931471805599453094172321;
const double kTwoPi = 6.283185307179586476925287;

double det_log(double x) {  // x > 0, finite
    int e = 0;
    double m = std::frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
    if (m < 0.70710678118654752440) {
        m = m * 2.0;
        e -= 1;
    }
    const double f = (m - 1.0) / (m + 1.0);
    const double f2 = f * f;
    double s = 1.0 / 25.0;
    for (int k = 23; k >= 1; k -= 2) s = 1.0 / double(k) + f2 * s;
    return double(e) * kLn2 + 2.0 * f * s;
}

double det_exp(double x) {
    const double kd = std::floor(x / kLn2 + 0.5);
    const double r = x - kd * kLn2;  // |r| <= ~0.35
    double s = 1.0;
    for (int k = 17; k >= 1; --k) s = 1.0 + r * s / double(k);
    return std::ldexp(s, int(kd));
}

double det_cos2pi(double t) {  // cos(2 pi t), t in [0,1)
    const double q = std::floor(4.0 * t + 0.5);
    const double r = (t - 0.25 * q) * kTwoPi;  // [-pi/4, pi/4]
    const double r2 = r * r;
    double c = 1.0, s = 1.0;  // Taylor series of cos and sin/r
    for (int k = 18; k >= 2; k -= 2) c = 1.0 - r2 * c / double(k * (k - 1));
    for (int k = 19; k >= 3; k -= 2) s = 1.0 - r2 * s / double(k * (k - 1));
    s = s * r;
    switch (int(q) & 3) {
        case 0: return c;
        case 1: return -s;
        case 2: return -c;
        default: return s;
    }
}

struct Rng {
    uint64_t seed;
    uint64_t raw(uint64_t stream, uint64_t idx) const {
        return mix(mix(mix(seed) ^ (stream * 0xD1B54A32D192ED03ULL)) ^ idx);
    }
    // uniform in [0,1)
    double u01(uint64_t stream, uint64_t idx) const {
        return double(raw(stream, idx) >> 11) * 0x1.0p-53;
    }
    double uniform(uint64_t stream, uint64_t idx, double a, double b) const {
        return a + (b - a) * u01(stream, idx);
    }
    // standard normal, Box-Muller on two counter draws
    double normal(uint64_t stream, uint64_t idx) const {
        const double u1 = double((raw(stream, 2 * idx) >> 11) + 1) * 0x1.0p-53;  // (0,1]
        const double u2 = u01(stream, 2 * idx + 1);
        return std::sqrt(-2.0 * det_log(u1)) * det_cos2pi(u2);
    }
};

struct Gen {
    mprec_gen_spec s;
    Rng rng;
    int nb, P, T, nb2;

    explicit Gen(const mprec_gen_spec& spec) : s(spec), rng{spec.seed} {
        nb = s.nb;
        P = nb - 2;
        T = nb - 1;
        nb2 = nb * nb;
    }
    double perm(int c) const {
        return s.perm_sigma > 0.0 ? det_exp(s.perm_sigma * rng.normal(S_PERM, uint64_t(c))) : 1.0;
    }
    double p0(int c) const {
        const int x = c % s.nx, y = c / s.nx;
        const int span = s.nx + s.ny - 2;
        const double lin = span > 0 ? 1.0 - double(x + y) / double(span) : 1.0;
        return lin + 0.1 * rng.normal(S_EPS, uint64_t(c));
    }
    // flux block entry (r,col) of cell c
    double flux(int c, int r, int col) const {
        const uint64_t idx = uint64_t(c) * nb2 + uint64_t(col) * nb + r;
        return col == P ? rng.uniform(S_FLUX, idx, 0.5, 1.5) : rng.uniform(S_FLUX, idx, -0.1, 0.1);
    }
    // off-diagonal block A_cj (column-major into out)
    void offdiag(int c, int j, double kc, double kj, double pc, double pj, double* out) const {
        const double tf = 2.0 * kc * kj / (kc + kj);
        const int u = pc > pj ? c : (pj > pc ? j : std::min(c, j));
        for (int col = 0; col < nb; ++col)
            for (int r = 0; r < nb; ++r) out[col * nb + r] = -(tf * flux(u, r, col));
        out[T * nb + T] = out[T * nb + T] - s.kappa * tf;
    }
    bool in_band(int c) const {
        if (!s.band) return false;
        const int x = c % s.nx, y = c / s.nx;
        return std::abs(x - y) <= 2;
    }
};

}  // namespace

extern "C" {

int mprec_gen_config(int config_id, mprec_gen_spec* out) {
    mprec_gen_spec s{};
    switch (config_id) {
        case 1: s = {40, 40, 3, 1.0, 0.0, 0, 1}; break;
        case 2: s = {200, 200, 4, 1e-3, 2.0, 0, 2}; break;
        case 3: s = {200, 200, 4, 1e3, 2.0, 0, 3}; break;
        case 4: s = {500, 500, 8, 1.0, 1.5, 1, 4}; break;
        case 5: s = {2000, 2000, 8, 1.0, 1.5, 1, 5}; break;
        default: return -1;
    }
    *out = s;
    return 0;
}

int64_t mprec_gen_nnzb(int nx, int ny) {
    return int64_t(nx) * ny + 2 * (int64_t(nx - 1) * ny + int64_t(nx) * (ny - 1));
}

int mprec_gen_pattern(int nx, int ny, int* row_ptr, int* col_idx) {
    if (nx < 1 || ny < 1) return -1;
    int64_t k = 0;
    const int n = nx * ny;
    row_ptr[0] = 0;
    for (int c = 0; c < n; ++c) {
        const int x = c % nx, y = c / nx;
        if (y > 0) col_idx[k++] = c - nx;
        if (x > 0) col_idx[k++] = c - 1;
        col_idx[k++] = c;
        if (x + 1 < nx) col_idx[k++] = c + 1;
        if (y + 1 < ny) col_idx[k++] = c + nx;
        row_ptr[c + 1] = int(k);
    }
    return 0;
}

int mprec_gen_fill(const mprec_gen_spec* spec, const int* rp, const int* ci, double* vals,
                   double* xstar, double* b, int nthreads) {
    if (!spec || spec->nb < 2 || spec->nx < 1 || spec->ny < 1) return -1;
    if (b && (!vals || !xstar)) return -1;
    const Gen g(*spec);
    const int n_cells = spec->nx * spec->ny;
    const int nb = g.nb, nb2 = g.nb2;
    if (nthreads <= 0) nthreads = int(std::max(1u, std::thread::hardware_concurrency()));
    nthreads = std::min(nthreads, std::max(1, n_cells / 64));

    auto work = [&](int c0, int c1) {
        std::vector<double> blk(nb2), d(nb2);
        for (int c = c0; c < c1; ++c) {
            if (xstar)
                for (int r = 0; r < nb; ++r)
                    xstar[int64_t(c) * nb + r] = g.rng.normal(S_XSTAR, uint64_t(c) * nb + r);
            if (!vals) continue;
            const double kc = g.perm(c), pc = g.p0(c);
            // accumulation block
            for (int r = 0; r < nb; ++r) {
                const double dr = 10.0 * g.rng.uniform(S_ACCD, uint64_t(c) * nb + r, 1.0, 2.0);
                for (int col = 0; col < nb; ++col) {
                    const uint64_t idx = uint64_t(c) * nb2 + uint64_t(col) * nb + r;
                    d[col * nb + r] = col == r ? dr : g.rng.uniform(S_ACCO, idx, -0.2, 0.2) * dr;
                }
            }
            int64_t kdiag = -1;
            for (int64_t k = rp[c]; k < rp[c + 1]; ++k) {
                const int j = ci[k];
                if (j == c) {
                    kdiag = k;
                    continue;
                }
                g.offdiag(c, j, kc, g.perm(j), pc, g.p0(j), blk.data());
                double* dst = vals + k * nb2;
                for (int e = 0; e < nb2; ++e) {
                    dst[e] = blk[e];
                    d[e] = d[e] - blk[e];
                }
            }
            if (g.in_band(c)) {
                for (int r = 0; r < nb; ++r)
                    d[g.T * nb + r] *= g.rng.uniform(S_BANDT, uint64_t(c) * nb + r, 10.0, 100.0);
                for (int r = 0; r < nb - 2; ++r)
                    for (int col = 0; col < nb - 2; ++col) {
                        if (r == col) continue;
                        const uint64_t idx = uint64_t(c) * nb2 + uint64_t(col) * nb + r;
                        d[col * nb + r] = g.rng.uniform(S_BANDC, idx, -5.0, 5.0) * d[r * nb + r];
                    }
            }
            if (kdiag >= 0)
                for (int e = 0; e < nb2; ++e) vals[kdiag * nb2 + e] = d[e];
        }
    };
    auto rhs = [&](int c0, int c1) {
        for (int c = c0; c < c1; ++c)
            for (int r = 0; r < nb; ++r) {
                double acc = 0.0;
                for (int64_t k = rp[c]; k < rp[c + 1]; ++k) {
                    const double* blkp = vals + k * nb2;
                    const double* xs = xstar + int64_t(ci[k]) * nb;
                    for (int col = 0; col < nb; ++col) acc += blkp[col * nb + r] * xs[col];
                }
                b[int64_t(c) * nb + r] = acc;
            }
    };
    auto run = [&](auto&& fn) {
        std::vector<std::thread> th;
        const int chunk = (n_cells + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; ++t) {
            const int c0 = t * chunk, c1 = std::min(n_cells, c0 + chunk);
            if (c0 >= c1) break;
            th.emplace_back(fn, c0, c1);
        }
        for (auto& x : th) x.join();
    };
    run(work);
    if (b) run(rhs);
    return 0;
}

}  // extern "C"
