// gs_band.cu -- band-scheduled ("doacross") Gauss-Seidel sweeps.
//
// The sync-free row-per-warp sweep pays one cross-SM L2 round trip per DAG
// level (0.6-0.9 us measured, 3-5k levels per AMG level).  Here the rows are
// cut into BANDS of consecutive indices; one warp owns a band and walks its
// LOCAL level sets (levels of the intra-band dependency DAG): intra-band
// dependencies are read from a shared-memory window written by the same warp
// one level earlier (a __syncwarp, not an L2 round trip), and only
// dependencies on earlier bands are polled in global memory (kPending
// sentinel).  Bands are claimed in sweep order, so every polled value belongs
// to a band that is already owned by a running warp (deadlock-free).  Row
// arithmetic is the reference's (sym_gauss_seidel, amg.cpp:25-43): forward
// rows use updated x_k for k < i and previous x_k for k > i.
//
// Schedule records (built once at setup, on the GPU): per band, per local
// level, chunks of <= 32 rows; a chunk record is
//   {int pos0, nrows, E, pad} int row[32] double invd[32]
//   uint code[E][32] double val[E][32]
// with code = type<<30 | index: 0 = shared-window slot, 1 = this band's
// published value (window overflow), 2 = earlier band (poll), 3 = previous
// iterate x_old, 0xFFFFFFFF = padding.  Records are contiguous in processing
// order and streamed into a shared-memory ring with cp.async, D records ahead.
#include <cub/cub.cuh>
#include <cstdlib>

#include "mprec.cuh"

namespace mg {

namespace {

constexpr int kWin = 2048;      // x window (doubles) per band
constexpr int kMaxE = 48;       // max off-diagonal entries per row in a band (else: row-per-warp kernel)
// src codes (uint16): < kWin window slot; kSrcG gathered x_new; kSrcO gathered x_old; kSrcZ padding
constexpr unsigned short kSrcG = 0xFFFF, kSrcO = 0xFFFE, kSrcZ = 0xFFFD;

// record layout (per chunk; uniform size within a band)
//   int hdr[4] {pos0, nr, E, n_ext} | int row[32] | double invd[32] | double val[E][32]
//   | int gidx[E][32] (>=0: x_new[g]; <=-2: x_old[-g-2]; -1: none)
//   | ushort src[E][32] | ushort ext[E*32] (entries that may still be pending) | pad16
__host__ __device__ inline int off_val() { return 16 + 128 + 256; }
__host__ __device__ inline int off_gidx(int e) { return off_val() + e * 256; }
__host__ __device__ inline int off_src(int e) { return off_gidx(e) + e * 128; }
__host__ __device__ inline int off_ext(int e) { return off_src(e) + e * 64; }
__host__ __device__ inline int rec_bytes(int e) { return (off_ext(e) + e * 64 + 15) & ~15; }
// gather area of a ring slot: double b[32], double x[E][32]
__host__ __device__ inline int gather_bytes(int e) { return 256 + e * 256; }

// ---- setup kernels ----------------------------------------------------------
// thread per band: local level = global DAG level - band minimum (so consecutive
// bands process the same global level at the same time), number of levels
__global__ void k_band_levels(const int* glev, int n, int B, int nbands, int* loc, int* nlev) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbands) return;
    const int b0 = b * B, b1 = min(n, b0 + B);
    int mn = 0x7fffffff, mx = -1;
    for (int i = b0; i < b1; ++i) {
        mn = min(mn, glev[i]);
        mx = max(mx, glev[i]);
    }
    for (int i = b0; i < b1; ++i) loc[i] = glev[i] - mn;
    nlev[b] = mx - mn + 1;
}

__global__ void k_band_positions(const int* rp, int n, int B, int nbands, int dir, const int* loc, const int* levbase,
                                 int* lstart, int* pos, int* nchunk) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbands) return;
    const int b0 = b * B, b1 = min(n, b0 + B);
    int* ls = lstart + levbase[b] + b;
    const int nl = levbase[b + 1] - levbase[b];
    for (int L = 0; L <= nl; ++L) ls[L] = 0;
    for (int i = b0; i < b1; ++i) ls[loc[i] + 1]++;
    int chunks = 0;
    for (int L = 0; L < nl; ++L) {
        chunks += (ls[L + 1] + 31) / 32;
        ls[L + 1] += ls[L];
    }
    nchunk[b] = chunks;
    if (dir > 0) {
        for (int i = b0; i < b1; ++i) pos[i] = b0 + ls[loc[i]]++;
    } else {
        for (int i = b1 - 1; i >= b0; --i) pos[i] = b0 + ls[loc[i]]++;
    }
    for (int L = nl; L > 0; --L) ls[L] = ls[L - 1];
    ls[0] = 0;
}

__global__ void k_rowat(const int* pos, int n, int* rowat) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rowat[pos[i]] = i;
}

// thread per band: chunk table {pos0, nrows, E_band, level_end}, band E, sizes
__global__ void k_band_chunks(const int* rp, int n, int B, int nbands, const int* levbase, const int* lstart,
                              const int* chunkbase, const int* rowat, int4* chunks, int* csize) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbands) return;
    const int b0 = b * B;
    const int* ls = lstart + levbase[b] + b;
    const int nl = levbase[b + 1] - levbase[b];
    int c = chunkbase[b];
    int emax = 0;
    for (int L = 0; L < nl; ++L) {
        for (int p = ls[L]; p < ls[L + 1]; p += 32) {
            const int nr = min(32, ls[L + 1] - p);
            for (int q = 0; q < nr; ++q) {
                const int i = rowat[b0 + p + q];
                emax = max(emax, rp[i + 1] - rp[i] - 1);
            }
            chunks[c++] = make_int4(b0 + p, nr, 0, b0 + ls[L + 1]);
        }
    }
    for (int q = chunkbase[b]; q < c; ++q) {
        chunks[q].z = emax;
        csize[q] = rec_bytes(emax);
    }
}

// warp per chunk: write the record
__global__ void k_band_records(const int* rp, const int* ci, const double* v, const int* diag, int n, int B,
                               int dir, const int4* chunks, const long long* coff, int nchunks, const int* pos,
                               const int* rowat, unsigned char* rec) {
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= nchunks) return;
    const int4 ch = chunks[c];
    const int pos0 = ch.x, nr = ch.y, E = ch.z, lev_end = ch.w;
    unsigned char* r = rec + coff[c];
    int* hdr = reinterpret_cast<int*>(r);
    int* rows = reinterpret_cast<int*>(r + 16);
    double* invd = reinterpret_cast<double*>(r + 144);
    double* val = reinterpret_cast<double*>(r + off_val());
    int* gidx = reinterpret_cast<int*>(r + off_gidx(E));
    unsigned short* src = reinterpret_cast<unsigned short*>(r + off_src(E));
    unsigned short* ext = reinterpret_cast<unsigned short*>(r + off_ext(E));
    const bool on = lane < nr;
    const int i = on ? rowat[pos0 + lane] : 0;
    const int band = i / B;
    const int b0 = band * B, b1 = min(n, b0 + B);
    rows[lane] = on ? i : -1;
    invd[lane] = on ? 1.0 / v[diag[i]] : 0.0;
    int e = 0;
    unsigned short my_ext[kMaxE];
    int n_my = 0;
    if (on) {
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (j == i) continue;
            const bool dep = dir > 0 ? (j < i) : (j > i);
            unsigned short sc;
            int g = -1;
            if (!dep) {
                sc = kSrcO;
                g = -j - 2;
            } else if (j >= b0 && j < b1 && pos[j] + kWin >= lev_end) {
                sc = (unsigned short)(pos[j] & (kWin - 1));
            } else {
                sc = kSrcG;  // earlier band (or far in this band): gathered, re-polled if pending
                g = j;
                my_ext[n_my++] = (unsigned short)(e * 32 + lane);
            }
            val[e * 32 + lane] = v[k];
            gidx[e * 32 + lane] = g;
            src[e * 32 + lane] = sc;
            ++e;
        }
    }
    for (; e < E; ++e) {
        val[e * 32 + lane] = 0.0;
        gidx[e * 32 + lane] = -1;
        src[e * 32 + lane] = kSrcZ;
    }
    // compact the (few) possibly-pending entries
    unsigned lt = (1u << lane) - 1u;
    int base = 0;
    for (int t = 0; t < kMaxE; ++t) {
        const bool has = t < n_my;
        const unsigned m = __ballot_sync(0xffffffffu, has);
        if (!m) break;
        if (has) ext[base + __popc(m & lt)] = my_ext[t];
        base += __popc(m);
    }
    if (lane == 0) {
        hdr[0] = pos0;
        hdr[1] = nr;
        hdr[2] = E;
        hdr[3] = base;
    }
}

// ---- the sweep ----------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_relaxed(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_pub(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}
__device__ __forceinline__ void cp16(void* s, const void* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp8(void* s, const void* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ int ld_vol(const int* p) { return *(const volatile int*)p; }

// CTA = 2 warps per band: warp 1 (producer) streams the band's records into a
// ring of R slots with cp.async, then gathers b / x_old / x_new operands into
// the slot and publishes `ready`; warp 0 (consumer) re-polls the few entries
// that were still pending, computes the level and publishes `done`.
template <int R, int L>
__global__ void __launch_bounds__(64) k_gs_band(const long long* __restrict__ coff, const int* __restrict__ band_chunk,
                                                const unsigned char* rec, const int* __restrict__ band_recb,
                                                int nbands, int slot_bytes, int dir, const double* __restrict__ b,
                                                const double* __restrict__ xold, double* xnew, int* counter,
                                                long long* ts, int nogather) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* xw = reinterpret_cast<double*>(smem);
    volatile int* ctl = reinterpret_cast<volatile int*>(smem + kWin * 8);  // [0]=band [1]=ready [2]=done
    unsigned char* ring = smem + kWin * 8 + 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (;;) {
        if (threadIdx.x == 0) {
            const int t = atomicAdd(counter, 1);
            ctl[0] = t;
            ctl[1] = 0;
            ctl[2] = 0;
        }
        __syncthreads();
        const int t = ctl[0];
        if (t >= nbands) return;
        const int band = dir > 0 ? t : nbands - 1 - t;
        const int c0 = band_chunk[band], c1 = band_chunk[band + 1], nch = c1 - c0;
        const unsigned char* brec = rec + coff[c0];
        const int rb = band_recb[band];
        if (warp == 1) {
            // ---------------- producer: software pipeline over chunks
            // iteration k commits {record k+L}, {gathers k}; records are waited
            // with wait_group<2L>, gathers published L behind with wait_group<2L>.
            for (int k = -L; k < nch + L; ++k) {
                const int kr = k + L;
                if (kr >= 0 && kr < nch) {
                    if (kr >= R)
                        while (ld_vol((const int*)&ctl[2]) < kr - R + 1) {
                        }
                    unsigned char* slot = ring + (kr % R) * slot_bytes;
                    const unsigned char* src = brec + (long long)kr * rb;
                    for (int o = lane * 16; o < rb; o += 512) cp16(slot + o, src + o);
                }
                cp_commit();
                cp_wait<2 * L>();  // record k has landed
                __syncwarp();
                if (k >= 0 && k < nch && !nogather) {
                    unsigned char* slot = ring + (k % R) * slot_bytes;
                    const int* hdr = reinterpret_cast<const int*>(slot);
                    const int nr = hdr[1], Ek = hdr[2];
                    double* gb = reinterpret_cast<double*>(slot + rb);
                    double* gx = gb + 32;
                    if (lane < nr) cp8(gb + lane, b + reinterpret_cast<const int*>(slot + 16)[lane]);
                    const int* gidx = reinterpret_cast<const int*>(slot + off_gidx(Ek));
                    for (int e = 0; e < Ek; ++e) {
                        const int g = gidx[e * 32 + lane];
                        if (g >= 0)
                            cp8(gx + e * 32 + lane, xnew + g);
                        else if (g <= -2 && xold)
                            cp8(gx + e * 32 + lane, xold + (-g - 2));
                    }
                }
                cp_commit();
                cp_wait<2 * L>();  // gathers of k - L have landed
                __syncwarp();
                const int kp = k - L;
                if (kp >= 0 && kp < nch && lane == 0) {
                    __threadfence_block();
                    ctl[1] = kp + 1;
                }
                if (ts && band == 0 && lane == 0 && k >= 0 && k < nch) {
                    long long g;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                    ts[3 * nbands + 2 * k] = g;  // producer iteration k end
                }
            }
            cp_wait<0>();
        } else {
            // ---------------- consumer
            if (ts && lane == 0) {
                long long g;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                ts[3 * band] = g;
            }
            for (int k = 0; k < nch; ++k) {
                while (ld_vol((const int*)&ctl[1]) < k + 1) {
                }
                __syncwarp();
                const unsigned char* slot = ring + (k % R) * slot_bytes;
                const int* hdr = reinterpret_cast<const int*>(slot);
                const int pos0 = hdr[0], nr = hdr[1], E = hdr[2], n_ext = hdr[3];
                const double* gb = reinterpret_cast<const double*>(slot + rb);
                double* gx = const_cast<double*>(gb) + 32;
                // entries gathered while possibly still pending: re-poll (warp-convergent)
                const unsigned short* ext = reinterpret_cast<const unsigned short*>(slot + off_ext(E));
                const int* gidx = reinterpret_cast<const int*>(slot + off_gidx(E));
                for (int q0 = 0; q0 < n_ext; q0 += 32) {
                    const int q = q0 + lane;
                    int slotidx = 0;
                    bool pend = false;
                    if (q < n_ext) {
                        slotidx = ext[q];
                        pend = __double_as_longlong(gx[slotidx]) == (long long)kPending;
                    }
                    while (__any_sync(0xffffffffu, pend)) {
                        if (pend) {
                            const unsigned long long raw = ld_relaxed(xnew + gidx[slotidx]);
                            if (raw != kPending) {
                                gx[slotidx] = __longlong_as_double((long long)raw);
                                pend = false;
                            }
                        }
                    }
                }
                __syncwarp();
                const double* val = reinterpret_cast<const double*>(slot + off_val());
                const unsigned short* src = reinterpret_cast<const unsigned short*>(slot + off_src(E));
                double acc = 0.0;
#pragma unroll 4
                for (int e = 0; e < E; ++e) {
                    const unsigned short sc = src[e * 32 + lane];
                    const double a = val[e * 32 + lane];
                    double x;
                    if (sc < kWin)
                        x = xw[sc];
                    else if (sc == kSrcG)
                        x = gx[e * 32 + lane];
                    else if (sc == kSrcO)
                        x = xold ? gx[e * 32 + lane] : 0.0;
                    else
                        x = 0.0;
                    acc += a * x;
                }
                if (lane < nr) {
                    const double xi = (gb[lane] - acc) * reinterpret_cast<const double*>(slot + 144)[lane];
                    xw[(pos0 + lane) & (kWin - 1)] = xi;
                    st_pub(xnew + reinterpret_cast<const int*>(slot + 16)[lane], xi);
                }
                __syncwarp();
                if (lane == 0) ctl[2] = k + 1;
                if (ts && band == 0 && lane == 0) {
                    long long g;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                    ts[3 * nbands + 2 * k + 1] = g;  // consumer chunk k end
                }
            }
            if (ts && lane == 0) {
                long long g;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                ts[3 * band + 1] = g;
                ts[3 * band + 2] = nch;
            }
        }
        __syncthreads();
    }
}

__global__ void k_band_recb(const int* band_chunk, const int* csize, int nbands, int* recb) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nbands) recb[b] = band_chunk[b + 1] > band_chunk[b] ? csize[band_chunk[b]] : 16;
}

__global__ void k_max_int_g(const int* a, int n, int* out) {
    int m = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, a[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_to_ll(const int* a, int n, long long* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i];
}

template <class T>
static T scan_ex(Ctx& c, const T* in, T* out, int n) {  // out[0..n], returns out[n]
    MG_CUDA(cudaMemsetAsync(out, 0, sizeof(T), c.s));
    if (n > 0) {
        size_t bytes = 0;
        cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out + 1, n, c.s);
        DBuf<char> tmp(bytes + 16);
        cub::DeviceScan::InclusiveSum(tmp.p, bytes, in, out + 1, n, c.s);
        check_launch("band scan");
    }
    T tot{};
    MG_CUDA(cudaMemcpyAsync(&tot, out + n, sizeof(T), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    return tot;
}

}  // namespace

bool build_band_sched(Ctx& c, const CsrView& a, int dir, const int* glev, BandSched& s) {
    const int n = a.n;
    s = BandSched{};
    if (n < 4096) return false;
    const int target = (n + 63) / 64;
    s.B = std::max(kWin, (target + kWin - 1) / kWin * kWin);
    s.nbands = (n + s.B - 1) / s.B;
    s.dir = dir;
    auto nb = [](int64_t m) { return int(std::max<int64_t>(1, (m + 127) / 128)); };
    DBuf<int> loc(n), nlev(s.nbands), levbase(s.nbands + 1), pos(n), rowat(n), nchunk(s.nbands);
    k_band_levels<<<nb(s.nbands), 128, 0, c.s>>>(glev, n, s.B, s.nbands, loc.p, nlev.p);
    check_launch("band levels");
    const int totlev = scan_ex(c, nlev.p, levbase.p, s.nbands);
    DBuf<int> lstart(totlev + s.nbands + 1);
    k_band_positions<<<nb(s.nbands), 128, 0, c.s>>>(a.rp, n, s.B, s.nbands, dir, loc.p, levbase.p, lstart.p, pos.p,
                                                     nchunk.p);
    k_rowat<<<nb(n), 128, 0, c.s>>>(pos.p, n, rowat.p);
    s.band_chunk.alloc(s.nbands + 1);
    s.nchunks = scan_ex(c, nchunk.p, s.band_chunk.p, s.nbands);
    s.chunks.alloc(std::max(s.nchunks, 1));
    DBuf<int> csize(std::max(s.nchunks, 1));
    k_band_chunks<<<nb(s.nbands), 128, 0, c.s>>>(a.rp, n, s.B, s.nbands, levbase.p, lstart.p, s.band_chunk.p,
                                                  rowat.p, s.chunks.p, csize.p);
    check_launch("band chunks");
    DBuf<int> mx(1);
    MG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), c.s));
    k_max_int_g<<<std::min(nb(s.nchunks), 1024), 128, 0, c.s>>>(csize.p, s.nchunks, mx.p);
    MG_CUDA(cudaMemcpyAsync(&s.slot_bytes, mx.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    DBuf<long long> cs64(std::max(s.nchunks, 1));
    k_to_ll<<<nb(s.nchunks), 128, 0, c.s>>>(csize.p, s.nchunks, cs64.p);
    s.coff.alloc(s.nchunks + 1);
    const long long total = scan_ex(c, cs64.p, s.coff.p, s.nchunks);
    // ring slot = record + gather area (b[32] + E_max x 32 doubles)
    int emax = 0;
    while (rec_bytes(emax) < s.slot_bytes) ++emax;
    if (emax > kMaxE) return false;  // very wide rows: keep the row-per-warp kernel
    s.rec_max = s.slot_bytes;
    s.slot_bytes = s.rec_max + gather_bytes(emax);
    static const int want = [] {
        const char* e = getenv("MPREC_BAND_DEPTH");
        return e ? atoi(e) : 16;
    }();
    s.depth = want;
    while (s.depth > 4 && kWin * 8 + 16 + s.depth * s.slot_bytes > 200 * 1024) s.depth /= 2;
    s.smem = kWin * 8 + 16 + s.depth * s.slot_bytes;
    if (s.smem > 200 * 1024) return false;
    s.band_recb.alloc(s.nbands);
    k_band_recb<<<nb(s.nbands), 128, 0, c.s>>>(s.band_chunk.p, csize.p, s.nbands, s.band_recb.p);
    s.rec.alloc(size_t(std::max<long long>(total, 16)));
    k_band_records<<<nb(int64_t(s.nchunks) * 32), 128, 0, c.s>>>(a.rp, a.ci, a.v, a.diag, n, s.B, dir, s.chunks.p,
                                                                 s.coff.p, s.nchunks, pos.p, rowat.p, s.rec.p);
    check_launch("band records");
    c.sync();
    s.nlev_total = totlev;
    s.ok = true;
    return true;
}

long long* g_band_ts = nullptr;  // diagnostics: per-band {start, end, chunks}

void gs_band_sweep(Ctx& c, const BandSched& s, int64_t nnz, int n, const double* b, const double* xold, double* xnew) {
    const double bytes = 12.0 * nnz + 4.0 * (n + 1) + 4.0 * n + 24.0 * n;
    Ctx::Scope sc(&c, MPREC_K_GS, bytes);
    int* ctr = c.counters.p + 5;
    MG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int), c.s));
    static bool attr = false;
    if (!attr) {
        MG_CUDA(cudaFuncSetAttribute(k_gs_band<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        MG_CUDA(cudaFuncSetAttribute(k_gs_band<8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        MG_CUDA(cudaFuncSetAttribute(k_gs_band<16, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    static const int nogather = [] {
        const char* e = getenv("MPREC_BAND_NOGATHER");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    const int grid = std::max(1, std::min(s.nbands, c.sm_count * 4));
#define MG_BAND_LAUNCH(R, L)                                                                                  \
    k_gs_band<R, L><<<grid, 64, s.smem, c.s>>>(s.coff.p, s.band_chunk.p, s.rec.p, s.band_recb.p, s.nbands,      \
                                            s.slot_bytes, s.dir, b, xold, xnew, ctr, g_band_ts, nogather)
    if (s.depth >= 16)
        MG_BAND_LAUNCH(16, 6);
    else if (s.depth >= 8)
        MG_BAND_LAUNCH(8, 3);
    else
        MG_BAND_LAUNCH(4, 1);
#undef MG_BAND_LAUNCH
    check_launch("gs_band");
}

}  // namespace mg
