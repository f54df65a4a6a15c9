// bsr.cu -- K1 block SpMV and K2 scoped residual update.
//
// K1 replaces ScalarMatrix::apply on the flattened Ā (scalar_matrix.cpp:79-88,
// the GMRES operator) and BlockMatrix::apply (block_matrix.cpp:103-114, the
// true residual).  HBM-bound: every stored block is streamed exactly once
// (algorithmic bytes = nnzb*(8 nb^2 + 4) + 4(n_c+1) + 16 n), the vector x is
// re-read from L2.  nb = 8: one warp per block row, each lane owns a
// (column, row-pair) of every block, so one warp-wide 16-byte load moves a whole
// 512-byte column-major block; block values use streaming (evict-first) loads so
// that x stays L2-resident.  Other nb: one thread per scalar row.
//
// K2: z = r - Ā[:, f] x_f where the stage solution is zero outside field f
// (stages.cpp:48,55,57): only column f of each block (nb doubles, contiguous
// in column-major storage) is read, and the next stage's gather is fused.
#include "mprec.cuh"

namespace mg {
namespace {

__device__ __forceinline__ double2 ld_stream2(const double* p) {
    double2 v;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// nb = 8: warp per block row.
__global__ void __launch_bounds__(256) k_bsr8(const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ val, const double* __restrict__ x,
                                              double* __restrict__ y, const double* __restrict__ b, int nc) {
    const int lane = threadIdx.x & 31;
    const int I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (I >= nc) return;
    const int c = lane >> 2, rr = (lane & 3) * 2;
    const int k0 = rp[I], k1 = rp[I + 1];
    double a0 = 0.0, a1 = 0.0;
    int k = k0;
    for (; k + 4 <= k1; k += 4) {
        int j[4];
        double2 v[4];
        double xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            j[u] = __ldg(ci + k + u);
            v[u] = ld_stream2(val + (int64_t)(k + u) * 64 + c * 8 + rr);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = __ldg(x + (int64_t)j[u] * 8 + c);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 += v[u].x * xv[u];
            a1 += v[u].y * xv[u];
        }
    }
    for (; k < k1; ++k) {
        const int j = __ldg(ci + k);
        const double2 v = ld_stream2(val + (int64_t)k * 64 + c * 8 + rr);
        const double xv = __ldg(x + (int64_t)j * 8 + c);
        a0 += v.x * xv;
        a1 += v.y * xv;
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if (lane < 4) {
        double2 out;
        if (b) {
            const double2 bb = *reinterpret_cast<const double2*>(b + (int64_t)I * 8 + rr);
            out.x = bb.x - a0;
            out.y = bb.y - a1;
        } else {
            out.x = a0;
            out.y = a1;
        }
        *reinterpret_cast<double2*>(y + (int64_t)I * 8 + rr) = out;
    }
}

// generic nb: thread per scalar row (consecutive threads = rows of one block row)
__global__ void __launch_bounds__(256) k_bsr_gen(const int* __restrict__ rp, const int* __restrict__ ci,
                                                 const double* __restrict__ val, const double* __restrict__ x,
                                                 double* __restrict__ y, const double* __restrict__ b, int nc, int nb) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nc * nb) return;
    const int I = int(t / nb), r = int(t - (int64_t)I * nb);
    double acc = 0.0;
    for (int k = rp[I]; k < rp[I + 1]; ++k) {
        const double* blk = val + (int64_t)k * nb * nb + r;
        const double* xs = x + (int64_t)__ldg(ci + k) * nb;
        for (int c = 0; c < nb; ++c) acc += ld_stream(blk + c * nb) * __ldg(xs + c);
    }
    y[t] = b ? b[t] - acc : acc;
}

// K2, thread per scalar row: z = r - sum_k A_k(row, f) * xs[col(k)]
__global__ void __launch_bounds__(256) k_bsr_col(const int* __restrict__ rp, const int* __restrict__ ci,
                                                 const double* __restrict__ val, int f, const double* __restrict__ xs,
                                                 const double* __restrict__ r, double* __restrict__ z,
                                                 double* __restrict__ zsub, int g, int nc, int nb) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nc * nb) return;
    const int I = int(t / nb), row = int(t - (int64_t)I * nb);
    double acc = 0.0;
    for (int k = rp[I]; k < rp[I + 1]; ++k)
        acc += ld_stream(val + ((int64_t)k * nb + f) * nb + row) * __ldg(xs + __ldg(ci + k));
    const double zv = r[t] - acc;
    z[t] = zv;
    if (zsub && row == g) zsub[I] = zv;
}

}  // namespace

void bsr_spmv(Ctx& c, const BsrView& a, const double* x, double* y, const double* b, int kclass) {
    const double n = double(a.nc) * a.nb;
    const double bytes = double(a.nnzb) * (8.0 * a.nb * a.nb + 4.0) + 4.0 * (a.nc + 1) + 16.0 * n + (b ? 8.0 * n : 0);
    Ctx::Scope sc(&c, kclass, bytes);
    if (a.nb == 8) {
        const int64_t threads = (int64_t)a.nc * 32;
        k_bsr8<<<int((threads + 255) / 256), 256, 0, c.s>>>(a.rp, a.ci, a.val, x, y, b, a.nc);
    } else {
        const int64_t threads = (int64_t)a.nc * a.nb;
        k_bsr_gen<<<int((threads + 255) / 256), 256, 0, c.s>>>(a.rp, a.ci, a.val, x, y, b, a.nc, a.nb);
    }
    check_launch("bsr_spmv");
}

void bsr_col_update(Ctx& c, const BsrView& a, int f, const double* xs, const double* r, double* z, double* zsub,
                    int g) {
    const double n = double(a.nc) * a.nb;
    const double bytes = double(a.nnzb) * (8.0 * a.nb + 4.0) + 4.0 * (a.nc + 1) + 8.0 * a.nc + 16.0 * n +
                         (zsub ? 8.0 * a.nc : 0.0);
    Ctx::Scope sc(&c, MPREC_K_SPMV_COL, bytes);
    const int64_t threads = (int64_t)a.nc * a.nb;
    k_bsr_col<<<int((threads + 255) / 256), 256, 0, c.s>>>(a.rp, a.ci, a.val, f, xs, r, z, zsub, g, a.nc, a.nb);
    check_launch("bsr_col_update");
}

}  // namespace mg
