// ilu_factor_exact.cu -- K5: block ILU(0) factorisation, dependency scheduled.
//
// Restates ILU0Factor::factor (ilu0.cpp:7-39) -- scalar IKJ elimination
// restricted to the pattern of the flattened Ā -- on the block pattern
// (SURVEY D4 / §8a A13): scalar row i = (I, r) sees k in the order "all
// columns of lower blocks (I,K), K ascending, in-block column ascending, then
// diagonal-block columns r' < r", and each entry receives its updates in the
// reference's k order, so the factors are bitwise equal to the oracle
// (compiled -fmad=false; division is IEEE).
//
// Schedule: one warp per block row, rows claimed in ascending order from an
// atomic counter (so every row a warp waits for is already owned by a running
// warp), sync-free: a row waits on the ready flag of each lower block's row
// (acquire), then publishes its own flag (release).  Lane l owns block entries
// e = l, l+32, ... (column-major index e = c*nb + r) of every block of its row.
#include "mprec.cuh"

namespace mg {
namespace {

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kWarps = 4;  // warps per block
constexpr int kMaxNb = 16;

__global__ void __launch_bounds__(kWarps * 32) k_ilu_factor(const int* __restrict__ rp, const int* __restrict__ ci,
                                                            const int* __restrict__ dpos, double* val, int nc, int nb,
                                                            int* flags, int epoch, const int* __restrict__ order,
                                                            int* counter, int* zero_flag) {
    __shared__ double fac_sh[kWarps][kMaxNb];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* fac = fac_sh[wid];
    const int nb2 = nb * nb;
    for (;;) {
        int I = 0;
        if (lane == 0) I = atomicAdd(counter, 1);
        I = __shfl_sync(0xffffffffu, I, 0);
        if (I >= nc) return;
        I = order[I];
        const int k0 = rp[I], k1 = rp[I + 1], d = dpos[I];
        // ---- phase 1: lower blocks (I,K), K ascending
        for (int k = k0; k < d; ++k) {
            const int K = ci[k];
            while (ld_acquire(flags + K) != epoch) {
            }
            __syncwarp();
            const int dK = dpos[K];
            const double* bK = val + (int64_t)dK * nb2;
            double* bk = val + (int64_t)k * nb2;
            for (int rk = 0; rk < nb; ++rk) {
                const double piv = __ldcg(bK + rk * nb + rk);
                if (piv == 0.0 && lane == 0) atomicOr(zero_flag, 1);
                // factors of column rk of block (I,K): fac[r] = L(r,rk) / piv
                for (int r = lane; r < nb; r += 32) {
                    const double f = bk[rk * nb + r] / piv;
                    bk[rk * nb + r] = f;
                    fac[r] = f;
                }
                __syncwarp();
                // in-block: entries (r, c > rk) -= fac[r] * U_K(rk, c)
                for (int e = lane; e < nb2; e += 32) {
                    const int c = e / nb, r = e - c * nb;
                    if (c > rk) bk[e] = bk[e] - fac[r] * __ldcg(bK + c * nb + rk);
                }
                // upper blocks (K, J) of row K matched into row I
                for (int kj = dK + 1; kj < rp[K + 1]; ++kj) {
                    const int J = ci[kj];
                    int lo = k0, hi = k1;  // binary search J in row I
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (ci[mid] < J)
                            lo = mid + 1;
                        else
                            hi = mid;
                    }
                    if (lo >= k1 || ci[lo] != J) continue;
                    double* bI = val + (int64_t)lo * nb2;
                    const double* bKJ = val + (int64_t)kj * nb2;
                    for (int e = lane; e < nb2; e += 32) {
                        const int c = e / nb, r = e - c * nb;
                        bI[e] = bI[e] - fac[r] * __ldcg(bKJ + c * nb + rk);
                    }
                }
                __syncwarp();
            }
        }
        // ---- phase 2: diagonal block, right-looking over pivot rows rp_
        double* bd = val + (int64_t)d * nb2;
        for (int q = 0; q < nb - 1; ++q) {
            const double piv = bd[q * nb + q];
            if (piv == 0.0 && lane == 0) atomicOr(zero_flag, 1);
            for (int r = q + 1 + lane; r < nb; r += 32) {
                const double f = bd[q * nb + r] / piv;
                bd[q * nb + r] = f;
                fac[r] = f;
            }
            __syncwarp();
            for (int e = lane; e < nb2; e += 32) {
                const int c = e / nb, r = e - c * nb;
                if (r > q && c > q) bd[e] = bd[e] - fac[r] * bd[c * nb + q];
            }
            for (int kb = d + 1; kb < k1; ++kb) {
                double* bu = val + (int64_t)kb * nb2;
                for (int e = lane; e < nb2; e += 32) {
                    const int c = e / nb, r = e - c * nb;
                    if (r > q) bu[e] = bu[e] - fac[r] * bu[c * nb + q];
                }
            }
            __syncwarp();
        }
        if (lane == 0 && bd[(nb - 1) * nb + nb - 1] == 0.0) atomicOr(zero_flag, 1);
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(flags + I, epoch);
    }
}

__global__ void k_diag(const int* dpos, const double* val, int nc, int nb, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nc * nb) return;
    const int I = i / nb, r = i - I * nb;
    out[i] = val[((int64_t)dpos[I] * nb + r) * nb + r];
}

}  // namespace

// Reference error semantics (ilu0.cpp:27,36): the first failing event in
// scalar row order; row i >= 1 fails its end-of-row check, row 0 fails when
// first used as a pivot (by row 1 when nb >= 2).
static int first_zero_pivot(const std::vector<double>& diag, const Pattern* pat, int nb, const BsrView& lu) {
    const int n = int(diag.size());
    long best_key = -1;
    int best_row = -1;
    auto consider = [&](long key, int row) {
        if (best_key < 0 || key < best_key) {
            best_key = key;
            best_row = row;
        }
    };
    for (int i = 1; i < n; ++i)
        if (diag[i] == 0.0) {
            consider(2L * i, i);
            break;
        }
    if (n > 0 && diag[0] == 0.0) {
        int first_ref = -1;
        if (nb >= 2)
            first_ref = 1;
        else if (pat) {
            for (int I = 1; I < lu.nc && first_ref < 0; ++I)
                for (int k = pat->h_rp[I]; k < pat->h_rp[I + 1]; ++k)
                    if (pat->h_ci[k] == 0) {
                        first_ref = I;
                        break;
                    }
        }
        if (first_ref >= 0) consider(2L * first_ref - 1, 0);
    }
    return best_row;
}

void ilu_factor_run(Ctx& c, const BsrView& lu, DBuf<int>& flags, Pattern* pat) {
    if (lu.nb > kMaxNb) throw Error(MPREC_DIMENSION, "nb > 16 not supported by the ILU kernel");
    pat->ensure_sched(c);
    flags.ensure(lu.nc);
    MG_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * lu.nc, c.s));
    MG_CUDA(cudaMemsetAsync(c.counters.p, 0, sizeof(int) * 2, c.s));
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * lu.nnzb * lu.nb * lu.nb);
        const int blocks = std::max(1, std::min((lu.nc + kWarps - 1) / kWarps, c.sm_count * 16));
        k_ilu_factor<<<blocks, kWarps * 32, 0, c.s>>>(lu.rp, lu.ci, lu.dpos, lu.val, lu.nc, lu.nb, flags.p, 1,
                                                       pat->fwd.order.p, c.counters.p, c.counters.p + 1);
        check_launch("ilu_factor");
    }
    int zero = 0;
    MG_CUDA(cudaMemcpyAsync(&zero, c.counters.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    if (zero) {
        // gather the pivots (rare error path) and apply the reference's ordering
        const int n = lu.nc * lu.nb;
        DBuf<double> dd(n);
        k_diag<<<(n + 255) / 256, 256, 0, c.s>>>(lu.dpos, lu.val, lu.nc, lu.nb, dd.p);
        check_launch("ilu_diag");
        const std::vector<double> diag = dd.to_host(c.s);
        const int row = first_zero_pivot(diag, pat, lu.nb, lu);
        if (row >= 0) throw Error(MPREC_ZERO_PIVOT, "zero pivot in ILU(0) at row " + std::to_string(row), row);
    }
}

}  // namespace mg
