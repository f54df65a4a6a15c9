// gram.cu -- Arnoldi orthogonalisation of gmres.cpp:39-50 in Gram (inverse
// compact WY) form: two passes over the Krylov basis per MGS sweep instead of
// one fused dot/axpy pass per basis vector.
//
// Modified Gram-Schmidt computes, for i = 0..k in order,
//     h_i = <w - sum_{j<i} h_j v_j, v_i> = <w, v_i> - sum_{j<i} G_ij h_j,
// with G_ij = <v_j, v_i>, i.e. (I + L) h = V^T w where L is the strictly lower
// part of the Gram matrix of the basis -- exactly, for any basis, not only an
// orthogonal one.  So one sweep is
//     pass A   p = V^T w            (one read of the basis, all dots at once)
//     solve    (I + L) h = p        (k^2/2 flops, one thread block)
//     pass B   w <- w - sum_i h_i v_i  (one read of the basis; per element the
//                                      updates are applied in i order, as MGS)
// and the new row of G (<v_j, v_k>, j < k) is computed in the same pass A as
// the dots with w, reading the basis once.  The reference's re-orthogonalisation
// (a second sweep when ||w|| < 0.7 ||w_0||, h += c) is the same three steps gated
// on a device flag.  Traffic per sweep: 16 n (k + 1) bytes + O(n) instead of
// 32 n (k + 1) for the fused per-vector MGS kernel, and 4 launches instead of
// k + 2.  Results differ from the sequential sweep only by rounding (same
// loss-of-orthogonality class as MGS; GMRES iteration counts stay within the
// reference's +-1 bar, tests/test_gpu_parity.py).
#include "mprec.cuh"

namespace mg {
namespace {

constexpr int kGT = 256;             // threads per block
constexpr int kT = kBasisTile;       // rows per tile (basis storage tile)
constexpr int kGV = kBasisChunk;     // basis vectors per storage chunk
constexpr int kGRed = 2 * kGV + 1;
constexpr int kRPT = kT / kGT;       // rows per thread per tile

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Basis storage (capi.cu: Basis): chunk c holds vectors 8c..8c+7 tile-major,
// [tile][8][kT]: the 8 vectors' rows of one tile are one contiguous 128 KB
// region, so both passes stream long contiguous runs (DRAM row-buffer friendly)
// instead of k + 1 interleaved vector streams.
__device__ __forceinline__ const double* tile_base(const double* const* ct, int c, int64_t tile) {
    return ct[c] + tile * (int64_t(kGV) * kT);
}

// Per-block partial sums of p_i = <v_i, w> (i <= k), q_j = <v_j, v_k> (j < k)
// and <w, w>, over a fixed set of tiles (tile = blockIdx.x + t * gridDim.x):
// part[blk * stride + {0..k | k+1..2k+1 | 2k+2}].
template <bool WQ>
__global__ void __launch_bounds__(kGT) k_gram_a(const double* const* __restrict__ ct, int k,
                                                 const double* __restrict__ w, int64_t n, double* __restrict__ part,
                                                 int stride, int want_q, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;
    extern __shared__ double sm[];
    double* acc = sm;
    double* red = acc + stride;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < stride; i += kGT) acc[i] = 0.0;
    const int64_t ntiles = (n + kT - 1) / kT;
    const int ck = k / kGV, jk = k % kGV;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * kT;
        const int nr = int(n - r0 < kT ? n - r0 : kT);
        double wr[kRPT], vr[kRPT];
        const double* vkp = tile_base(ct, ck, tile) + jk * kT;
#pragma unroll
        for (int q = 0; q < kRPT; ++q) {
            const int r = tid + q * kGT;
            wr[q] = r < nr ? w[r0 + r] : 0.0;
            vr[q] = (WQ && r < nr) ? vkp[r] : 0.0;
        }
        for (int c = 0; c <= ck; ++c) {
            const double* base = tile_base(ct, c, tile);
            const int nv = c < ck ? kGV : jk + 1;
            double ap[kGV], aq[kGV], aw = 0.0;
#pragma unroll
            for (int j = 0; j < kGV; ++j) {
                ap[j] = aq[j] = 0.0;
                if (j < nv) {
#pragma unroll
                    for (int q = 0; q < kRPT; ++q) {
                        const int r = tid + q * kGT;
                        const double x = r < nr ? __ldcs(base + j * kT + r) : 0.0;
                        ap[j] += x * wr[q];
                        if (WQ) aq[j] += x * vr[q];
                    }
                }
            }
            if (c == 0)
#pragma unroll
                for (int q = 0; q < kRPT; ++q) aw += wr[q] * wr[q];
            // butterfly reduction of all V partial sums at once (V - 1 + 5 - log2 V
            // shuffles instead of 5 V): after it, lane l holds the warp total of
            // value idx(l) when l has no bits below the last halving offset
            constexpr int V = WQ ? 2 * kGV : kGV;
            double vv[V];
#pragma unroll
            for (int j = 0; j < kGV; ++j) {
                vv[j] = ap[j];
                if (WQ) vv[kGV + j] = aq[j];
            }
            int idx = 0;
#pragma unroll
            for (int cnt = V, o = 16; cnt > 1; cnt /= 2, o /= 2) {
                const bool up = lane & o;
#pragma unroll
                for (int i = 0; i < cnt / 2; ++i) {
                    const double send = up ? vv[i] : vv[i + cnt / 2];
                    const double keep = up ? vv[i + cnt / 2] : vv[i];
                    vv[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
                if (up) idx += cnt / 2;
            }
            // remaining lanes bits below the last offset: plain xor reduction
            constexpr int LOG_V = (V == 16) ? 4 : 3;
#pragma unroll
            for (int o = 16 >> LOG_V; o > 0; o >>= 1) vv[0] += __shfl_xor_sync(0xffffffffu, vv[0], o);
            if (c == 0) aw = warp_sum(aw);
            __syncthreads();  // previous chunk's red consumed
            if ((lane & ((32 >> LOG_V) - 1)) == 0) {
                if (WQ)
                    red[wid * kGRed + idx] = vv[0];
                else {
                    red[wid * kGRed + idx] = vv[0];
                    red[wid * kGRed + kGV + idx] = 0.0;
                }
            }
            if (lane == 0) red[wid * kGRed + 2 * kGV] = aw;
            __syncthreads();
            if (tid < kGRed) {
                double s = 0.0;
                for (int q = 0; q < kGT / 32; ++q) s += red[q * kGRed + tid];
                if (tid < kGV) {
                    if (tid < nv) acc[c * kGV + tid] += s;
                } else if (tid < 2 * kGV) {
                    const int j = c * kGV + tid - kGV;
                    if (j < k) acc[k + 1 + j] += s;
                } else if (c == 0) {
                    acc[2 * k + 2] += s;
                }
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < stride; i += kGT) part[int64_t(blockIdx.x) * stride + i] = acc[i];
}

// Sum the per-block partials in block order; scatter p, the new Gram row (stored
// transposed: gt[j * ld + k] = <v_j, v_k>) and sqrt(<w, w>).
__global__ void k_gram_fin(const double* __restrict__ part, int nblk, int stride, int k, double* p_out, double* gt,
                           int ld, double* norm_out, int want_q, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;
    // one warp per output: lane l sums blocks l, l + 32, ... then a fixed shuffle tree
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= stride) return;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += part[int64_t(b) * stride + i];
    s = warp_sum(s);
    if (lane != 0) return;
    if (i <= k)
        p_out[i] = s;
    else if (i <= 2 * k + 1) {
        const int j = i - (k + 1);
        if (want_q && j < k) gt[int64_t(j) * ld + k] = s;
    } else if (norm_out) {
        *norm_out = sqrt(s);
    }
}

// (I + L) c = p by forward substitution, column by column (h_i accumulates its
// corrections in j order); c overwrites p, h = c or h += c (re-orthogonalisation).
__global__ void k_gram_tri(const double* __restrict__ gt, int ld, int k, double* p, double* h, int accumulate,
                           const int* __restrict__ gate) {
    if (gate && *gate == 0) return;
    extern __shared__ double ps[];
    for (int i = threadIdx.x; i <= k; i += blockDim.x) ps[i] = p[i];
    __syncthreads();
    for (int j = 0; j < k; ++j) {
        const double hj = ps[j];
        const double* col = gt + int64_t(j) * ld;
        for (int i = j + 1 + threadIdx.x; i <= k; i += blockDim.x) ps[i] -= col[i] * hj;
        __syncthreads();
    }
    for (int i = threadIdx.x; i <= k; i += blockDim.x) {
        p[i] = ps[i];
        h[i] = accumulate ? h[i] + ps[i] : ps[i];
    }
}

// mode 0: w <- w - sum_{i<=k} c_i v_i (per element in i order), norm_out =
// ||w||; mode 1: w <- sum_{i<=k} c_i v_i (GMRES solution update, no norm).
// Tile-major: each thread keeps its kRPT rows of the tile in registers while the
// basis chunks of the tile stream by.
__global__ void __launch_bounds__(kGT) k_gram_b(const double* const* __restrict__ ct, int k,
                                                 const double* __restrict__ cvec, double* __restrict__ w, int64_t n,
                                                 double* partials, unsigned* ctr, double* norm_out, int mode,
                                                 const int* __restrict__ gate) {
    if (gate && *gate == 0) return;
    extern __shared__ double sm[];
    double* cs = sm;
    double* red = cs + k + 1;
    for (int i = threadIdx.x; i <= k; i += kGT) cs[i] = cvec[i];
    __syncthreads();
    const int64_t ntiles = (n + kT - 1) / kT;
    const int ck = k / kGV, jk = k % kGV;
    double ss = 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * kT;
        const int nr = int(n - r0 < kT ? n - r0 : kT);
        double x[kRPT];
#pragma unroll
        for (int q = 0; q < kRPT; ++q) {
            const int r = threadIdx.x + q * kGT;
            x[q] = (mode == 0 && r < nr) ? w[r0 + r] : 0.0;
        }
        for (int c = 0; c <= ck; ++c) {
            const double* base = tile_base(ct, c, tile);
            const int nv = c < ck ? kGV : jk + 1;
#pragma unroll
            for (int j = 0; j < kGV; ++j)
                if (j < nv) {
                    const double cj = cs[c * kGV + j];
#pragma unroll
                    for (int q = 0; q < kRPT; ++q) {
                        const int r = threadIdx.x + q * kGT;
                        const double v = r < nr ? __ldcs(base + j * kT + r) : 0.0;
                        if (mode == 0)
                            x[q] -= cj * v;
                        else
                            x[q] += cj * v;
                    }
                }
        }
#pragma unroll
        for (int q = 0; q < kRPT; ++q) {
            const int r = threadIdx.x + q * kGT;
            if (r < nr) {
                w[r0 + r] = x[q];
                ss += x[q] * x[q];
            }
        }
    }
    if (mode != 0) return;
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int q = 0; q < kGT / 32; ++q) s += red[q];
        partials[blockIdx.x] = s;
        __threadfence();
        last = atomicInc(ctr, 0xFFFFFFFFu) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    double s = 0.0;
    for (int b = 0; b < int(gridDim.x); ++b) s += reinterpret_cast<volatile double*>(partials)[b];
    *norm_out = sqrt(s);
    *ctr = 0;
}

// Pass B of the first MGS sweep fused with pass A of the (gated) re-orthogonalisation
// sweep: w' = w - V c, ||w'||, and the per-block partials of p' = V^T w', reading the
// basis ONCE.  The basis values a thread needs twice stay in its REGISTERS: a block
// of 16 warps takes a row sub-tile; warp (vector group vg, row set rs) holds, lane =
// row, the values of <= 32 consecutive basis vectors (vg*32 ..) for its 32 rows.
//   phase 1: per-warp partial of (V c)[row] over its 32 vectors; the NG partials of
//            a row are combined in shared memory in group order: x = w - V c;
//   phase 2: v_j[row] * x[row] for the same 32 register values, reduced over the
//            32 rows of the warp by one butterfly (31 shuffles for 32 sums).
// 32 independent 8-byte loads per thread, 128 KB in flight per SM (one block per
// SM, persistent).  The speculative p' costs no extra memory traffic; the sweep that
// uses it runs only when the gate fires (gmres.cpp:44-50).  Deterministic: per-warp
// accumulators, fixed orders.
constexpr int kBW = 16;  // warps per block

template <int NG>  // vector groups of 32: NG = next power of two >= (k + 1) / 32
__global__ void __launch_bounds__(kBW * 32, 1) k_gram_ba(const double* const* __restrict__ ct, int k,
                                                          const double* __restrict__ cvec, double* __restrict__ w,
                                                          int64_t n, double* __restrict__ part, int stride,
                                                          double* npart, unsigned* ctr, double* norm_out) {
    constexpr int NRS = kBW / NG;  // row sets of 32 rows per sub-tile
    constexpr int R = 32 * NRS;    // rows per sub-tile (divides kT)
    __shared__ double cs[32 * NG];
    __shared__ double xp[NG][R];
    __shared__ double xs[R];
    __shared__ double acc[kBW][32];
    __shared__ double red[kBW];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int vg = wid % NG, rs = wid / NG;
    for (int i = tid; i < 32 * NG; i += blockDim.x) cs[i] = i <= k ? cvec[i] : 0.0;
    acc[wid][lane] = 0.0;
    __syncthreads();
    const int j0 = vg * 32;
    const int nv = max(0, min(32, k + 1 - j0));
    const double* cbase[4];  // the group's 4 storage chunks
#pragma unroll
    for (int q = 0; q < 4; ++q) cbase[q] = (j0 / kGV + q) * kGV <= k ? ct[j0 / kGV + q] : nullptr;
    const int64_t nsub = (n + R - 1) / R;
    double ss = 0.0;
    for (int64_t st = blockIdx.x; st < nsub; st += gridDim.x) {
        const int64_t row = st * R + rs * 32 + lane;
        const bool in = row < n;
        const int64_t tile = (st * R) / kT;
        const int off = int((st * R) % kT) + rs * 32 + lane;
        double v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t)
            v[t] = (t < nv && in) ? __ldcs(cbase[t / kGV] + tile * (int64_t(kGV) * kT) + (t % kGV) * kT + off) : 0.0;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
            a0 = fma(cs[j0 + t], v[t], a0);
            a1 = fma(cs[j0 + t + 1], v[t + 1], a1);
        }
        xp[vg][rs * 32 + lane] = a0 + a1;
        __syncthreads();
        if (vg == 0) {
            double vc = 0.0;
#pragma unroll
            for (int g = 0; g < NG; ++g) vc += xp[g][rs * 32 + lane];
            const double x = in ? w[row] - vc : 0.0;
            xs[rs * 32 + lane] = x;
            if (in) {
                w[row] = x;
                ss += x * x;
            }
        }
        __syncthreads();
        const double x = xs[rs * 32 + lane];
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] *= x;
        int idx = 0;
#pragma unroll
        for (int cnt = 32, o = 16; cnt > 1; cnt /= 2, o /= 2) {
            const bool up = lane & o;
#pragma unroll
            for (int i = 0; i < cnt / 2; ++i) {
                const double send = up ? v[i] : v[i + cnt / 2];
                const double keep = up ? v[i + cnt / 2] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
            if (up) idx += cnt / 2;
        }
        acc[wid][idx] += v[0];
    }
    __syncthreads();
    // per-block partials of p' (row sets summed in order); entries k+1.. unused
    for (int j = tid; j <= k; j += blockDim.x) {
        double sacc = 0.0;
#pragma unroll
        for (int r2 = 0; r2 < NRS; ++r2) sacc += acc[r2 * NG + j / 32][j % 32];
        part[int64_t(blockIdx.x) * stride + j] = sacc;
    }
    // ||w'||: block partials, the last block sums them in block order
    ss = warp_sum(ss);
    if (lane == 0) red[wid] = ss;
    __syncthreads();
    __shared__ bool last;
    if (tid == 0) {
        double sm2 = 0.0;
        for (int v2 = 0; v2 < kBW; ++v2) sm2 += red[v2];
        npart[blockIdx.x] = sm2;
        __threadfence();
        last = atomicInc(ctr, 0xFFFFFFFFu) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || tid != 0) return;
    __threadfence();
    double tot = 0.0;
    for (int b2 = 0; b2 < int(gridDim.x); ++b2) tot += reinterpret_cast<volatile double*>(npart)[b2];
    *norm_out = sqrt(tot);
    *ctr = 0;
}

__global__ void k_set_ptr(double** tab, int i, double* p) { tab[i] = p; }

// vector j of a chunk <- x / a (put) or y <- vector j of a chunk (get)
__global__ void k_basis_put(double* chunk, int j, const double* __restrict__ x, double a, int64_t n) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x)
        chunk[(r / kT) * (int64_t(kGV) * kT) + j * kT + (r % kT)] = x[r] / a;
}
__global__ void k_basis_get(double* y, const double* __restrict__ chunk, int j, int64_t n) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x)
        y[r] = chunk[(r / kT) * (int64_t(kGV) * kT) + j * kT + (r % kT)];
}

inline int tile_grid(Ctx& c, int64_t n, int per_sm) {
    const int64_t ntiles = (n + kT - 1) / kT;
    return int(std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(per_sm) * c.sm_count)));
}

}  // namespace

int64_t basis_chunk_doubles(int64_t n) { return ((n + kT - 1) / kT) * int64_t(kGV) * kT; }

void gram_set_ptr(Ctx& c, double** tab, int i, double* p) {
    k_set_ptr<<<1, 1, 0, c.s>>>(tab, i, p);
    check_launch("gram ptr");
}

void basis_put(Ctx& c, double* chunk, int j, const double* x, double a, int64_t n) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * n);
    k_basis_put<<<grid_for(n, 256), 256, 0, c.s>>>(chunk, j, x, a, n);
    check_launch("basis put");
}

void basis_get(Ctx& c, double* y, const double* chunk, int j, int64_t n) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * n);
    k_basis_get<<<grid_for(n, 256), 256, 0, c.s>>>(y, chunk, j, n);
    check_launch("basis get");
}

int gram_part_size(Ctx& c, int kmax) { return 4 * c.sm_count * (2 * (kmax + 1) + 1); }

void gram_sweep(Ctx& c, const double* const* ct, int k, double* w, int64_t n, double* gt, int ld, double* pbuf,
                double* h, bool accumulate, bool want_q, double* pre_norm, double* post_norm, double* part,
                const int* gate) {
    const int stride = 2 * (k + 1) + 1;
    const int grid_a = tile_grid(c, n, 4);
    {
        Ctx::Scope sc(&c, MPREC_K_MGS, 8.0 * n * (k + 2), gate != nullptr);
        const size_t smem = sizeof(double) * (stride + (kGT / 32) * kGRed);
        static size_t attr = 0;
        if (smem > 48 * 1024 && smem > attr) {
            MG_CUDA(cudaFuncSetAttribute(k_gram_a<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            MG_CUDA(cudaFuncSetAttribute(k_gram_a<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr = smem;
        }
        if (want_q)
            k_gram_a<true><<<grid_a, kGT, smem, c.s>>>(ct, k, w, n, part, stride, 1, gate);
        else
            k_gram_a<false><<<grid_a, kGT, smem, c.s>>>(ct, k, w, n, part, stride, 0, gate);
        check_launch("gram pass A");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * grid_a * stride, gate != nullptr);
        k_gram_fin<<<(stride + 7) / 8, 256, 0, c.s>>>(part, grid_a, stride, k, pbuf, gt, ld, pre_norm,
                                                      want_q ? 1 : 0, gate);
        check_launch("gram fin");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * (k + 1) * (k + 1) / 2, gate != nullptr);
        k_gram_tri<<<1, 512, sizeof(double) * (k + 1), c.s>>>(gt, ld, k, pbuf, h, accumulate ? 1 : 0, gate);
        check_launch("gram tri");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_MGS, 8.0 * n * (k + 3), gate != nullptr);
        const size_t smem = sizeof(double) * (k + 1 + kGT / 32);
        static size_t attr = 0;
        if (smem > 48 * 1024 && smem > attr) {
            MG_CUDA(cudaFuncSetAttribute(k_gram_b, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr = smem;
        }
        const int grid_b = std::min(tile_grid(c, n, 8), kRedBlocks);
        k_gram_b<<<grid_b, kGT, smem, c.s>>>(ct, k, pbuf, w, n, c.red.p, c.red_ctr.p + 8, post_norm, 0, gate);
        check_launch("gram pass B");
    }
}

// One Arnoldi orthogonalisation (gmres.cpp:37-51) with the re-orthogonalisation's
// pass A fused into the first sweep's pass B (k_gram_ba): pass A, (I+L) h = p,
// [w -= V h, ||w||, p' = V^T w], gate, then -- gated -- (I+L) c = p', h += c,
// w -= V c, ||w||.  Three reads of the basis from HBM when the gate fires (four with
// gram_sweep twice), two when it does not.
void gram_orthogonalise(Ctx& c, const double* const* ct, int k, double* w, int64_t n, double* gt, int ld,
                        double* pbuf, double* h, double* pre_norm, double* post_norm, double* reorth_norm,
                        double* part, int* gate) {
    const int stride = 2 * (k + 1) + 1;
    const int grid_a = tile_grid(c, n, 4);
    {
        Ctx::Scope sc(&c, MPREC_K_MGS, 8.0 * n * (k + 2));
        const size_t smem = sizeof(double) * (stride + (kGT / 32) * kGRed);
        static size_t attr = 0;
        if (smem > 48 * 1024 && smem > attr) {
            MG_CUDA(cudaFuncSetAttribute(k_gram_a<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            MG_CUDA(cudaFuncSetAttribute(k_gram_a<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr = smem;
        }
        if (k > 0)
            k_gram_a<true><<<grid_a, kGT, smem, c.s>>>(ct, k, w, n, part, stride, 1, nullptr);
        else
            k_gram_a<false><<<grid_a, kGT, smem, c.s>>>(ct, k, w, n, part, stride, 0, nullptr);
        check_launch("gram pass A");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * grid_a * stride);
        k_gram_fin<<<(stride + 7) / 8, 256, 0, c.s>>>(part, grid_a, stride, k, pbuf, gt, ld, pre_norm, k > 0 ? 1 : 0,
                                                      nullptr);
        check_launch("gram fin");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * (k + 1) * (k + 1) / 2);
        k_gram_tri<<<1, 512, sizeof(double) * (k + 1), c.s>>>(gt, ld, k, pbuf, h, 0, nullptr);
        check_launch("gram tri");
    }
    // fused pass B + speculative pass A' (registers): one persistent block per SM
    int grid_ba = 0;
    {
        // algorithmic: basis once + w read and written
        Ctx::Scope sc(&c, MPREC_K_MGS, 8.0 * n * (k + 3));
        const int ng = k + 1 <= 32 ? 1 : k + 1 <= 64 ? 2 : k + 1 <= 128 ? 4 : k + 1 <= 256 ? 8 : 16;
        if (k + 1 > 512) throw Error(MPREC_DIMENSION, "gram: fused pass supports k < 512");
        const int R = 32 * (kBW / ng);
        grid_ba = int(std::max<int64_t>(1, std::min<int64_t>((n + R - 1) / R, c.sm_count)));
        auto* red = c.red.p;
        auto* ctr = c.red_ctr.p + 8;
        switch (ng) {
            case 1: k_gram_ba<1><<<grid_ba, kBW * 32, 0, c.s>>>(ct, k, pbuf, w, n, part, stride, red, ctr, post_norm); break;
            case 2: k_gram_ba<2><<<grid_ba, kBW * 32, 0, c.s>>>(ct, k, pbuf, w, n, part, stride, red, ctr, post_norm); break;
            case 4: k_gram_ba<4><<<grid_ba, kBW * 32, 0, c.s>>>(ct, k, pbuf, w, n, part, stride, red, ctr, post_norm); break;
            case 8: k_gram_ba<8><<<grid_ba, kBW * 32, 0, c.s>>>(ct, k, pbuf, w, n, part, stride, red, ctr, post_norm); break;
            default: k_gram_ba<16><<<grid_ba, kBW * 32, 0, c.s>>>(ct, k, pbuf, w, n, part, stride, red, ctr, post_norm); break;
        }
        check_launch("gram pass BA");
    }
    set_reorth_gate(c, post_norm, pre_norm, gate);
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * grid_ba * (k + 1), true);
        k_gram_fin<<<(stride + 7) / 8, 256, 0, c.s>>>(part, grid_ba, stride, k, pbuf, gt, ld, nullptr, 0, gate);
        check_launch("gram fin (reorth)");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * (k + 1) * (k + 1) / 2, true);
        k_gram_tri<<<1, 512, sizeof(double) * (k + 1), c.s>>>(gt, ld, k, pbuf, h, 1, gate);
        check_launch("gram tri (reorth)");
    }
    {
        Ctx::Scope sc(&c, MPREC_K_MGS, 8.0 * n * (k + 3), true);
        const size_t smem = sizeof(double) * (k + 1 + kGT / 32);
        static size_t attr = 0;
        if (smem > 48 * 1024 && smem > attr) {
            MG_CUDA(cudaFuncSetAttribute(k_gram_b, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr = smem;
        }
        const int grid_b = std::min(tile_grid(c, n, 8), kRedBlocks);
        k_gram_b<<<grid_b, kGT, smem, c.s>>>(ct, k, pbuf, w, n, c.red.p, c.red_ctr.p + 8, reorth_norm, 0, gate);
        check_launch("gram pass B (reorth)");
    }
}

void basis_combine(Ctx& c, const double* const* ct, int k, const double* y, double* z, int64_t n) {
    if (k <= 0) return;
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * n * (k + 1));
    const size_t smem = sizeof(double) * (k + kGT / 32);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        MG_CUDA(cudaFuncSetAttribute(k_gram_b, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = smem;
    }
    k_gram_b<<<std::min(tile_grid(c, n, 8), kRedBlocks), kGT, smem, c.s>>>(ct, k - 1, y, z, n, nullptr, nullptr,
                                                                           nullptr, 1, nullptr);
    check_launch("basis combine");
}

}  // namespace mg
