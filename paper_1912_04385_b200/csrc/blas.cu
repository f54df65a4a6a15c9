// blas.cu -- Ctx runtime + vector kernels of the Krylov loop (gmres.cpp:17-100):
// deterministic fixed-order reductions (dot, norm), the re-orthogonalisation
// gate, gathers and the stage combine (the Arnoldi passes are in gram.cu).
//
// Reductions are deterministic: the grid size is a function of n only, each
// block reduces a fixed grid-stride slice through a fixed shared-memory tree,
// and the last block to finish sums the per-block partials in a fixed order.
// Repeated solves are therefore bitwise identical (test_krylov.cpp:92-100).
#include <chrono>
#include <cstdlib>

#include "mprec.cuh"

namespace mg {

// ============================================================== Ctx runtime ==
Ctx::Ctx() {
    MG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int dev = 0;
    MG_CUDA(cudaGetDevice(&dev));
    MG_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
    red.alloc(kRedBlocks * 4);
    red_ctr.alloc(64);
    MG_CUDA(cudaMemsetAsync(red_ctr.p, 0, red_ctr.bytes(), s));
    scal.alloc(4096);
    counters.alloc(64);
    err.alloc(64);
}

Ctx::~Ctx() {
    if (s) cudaStreamSynchronize(s);
    for (auto& p : pending) {
        event_pool.push_back(p.a);
        event_pool.push_back(p.b);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    if (s) cudaStreamDestroy(s);
}

cudaEvent_t Ctx::get_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    MG_CUDA(cudaEventCreate(&e));
    return e;
}

Ctx::Scope::Scope(Ctx* c_, int kc_, double bytes_, bool gated_) : c(c_), kc(kc_), bytes(bytes_), gated(gated_) {
    c->launches++;
    if (gated) c->unresolved_gated++;
    if (c->profile) {
        a = c->get_event();
        cudaEventRecord(a, c->s);
    }
}

Ctx::Scope::~Scope() {
    if (a) {
        cudaEvent_t b = c->get_event();
        cudaEventRecord(b, c->s);
        c->pending.push_back({kc, bytes, a, b, gated});
        if (c->pending.size() > 4096 && c->unresolved_gated == 0) c->harvest();
    } else {
        c->stat[kc].launches++;
        if (gated)
            c->gated_bytes[kc] += bytes;
        else
            c->stat[kc].bytes += bytes;
    }
}

void Ctx::resolve_gate(bool fired) {
    for (auto& p : pending)
        if (p.gated) {
            if (!fired) p.bytes = 0.0;
            p.gated = false;
        }
    for (int k = 0; k < MPREC_K_COUNT; ++k) {
        if (fired) stat[k].bytes += gated_bytes[k];
        gated_bytes[k] = 0.0;
    }
    unresolved_gated = 0;
}

void Ctx::harvest() {
    if (pending.empty()) return;
    MG_CUDA(cudaStreamSynchronize(s));
    for (auto& p : pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        stat[p.kc].ms += ms;
        stat[p.kc].launches++;
        stat[p.kc].bytes += p.bytes;
        event_pool.push_back(p.a);
        event_pool.push_back(p.b);
    }
    pending.clear();
}

bool trace_on() {
    static const bool on = [] {
        const char* e = getenv("MPREC_TRACE");
        return e && e[0] == '1';
    }();
    return on;
}

static double wall() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Trace::Trace(Ctx* c_, const char* w) : what(w), c(c_), t0(0) {
    if (trace_on()) {
        c->sync();
        t0 = wall();
    }
}

Trace::~Trace() {
    if (trace_on()) {
        cudaStreamSynchronize(c->s);
        fprintf(stderr, "[mprec] %-28s %9.3f ms\n", what, 1e3 * (wall() - t0));
    }
}

// ================================================================== kernels ==
namespace {

constexpr int kRT = 256;  // reduction block size

__device__ __forceinline__ double block_sum(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = kRT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    return sh[0];
}

// Final stage of a two-level reduction, run by the last block to arrive.
// mode bit0: sqrt of the sum; bit1: accumulate into *hsum too.
__device__ void finish(double part, double* partials, unsigned* ctr, double* out, double* hsum, int mode,
                       double* sh) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = part;
        __threadfence();
        const unsigned t = atomicInc(ctr, 0xFFFFFFFFu);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double v = 0.0;
    for (int i = threadIdx.x; i < gridDim.x; i += kRT) v += ((volatile double*)partials)[i];
    const double tot = block_sum(v, sh);
    if (threadIdx.x == 0) {
        const double r = (mode & 1) ? sqrt(tot) : tot;
        *out = r;
        if (hsum) *hsum += r;
        *ctr = 0;
    }
}

__global__ void k_fill(double* x, double v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void k_fill_bits(unsigned long long* x, unsigned long long v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void k_copy(double* y, const double* x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i];
}

__global__ void __launch_bounds__(kRT) k_dot(const double* a, const double* b, int64_t n, double* partials,
                                             unsigned* ctr, double* out, int mode) {
    __shared__ double sh[kRT];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kRT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRT)
        s += a[i] * b[i];
    const double part = block_sum(s, sh);
    __syncthreads();
    finish(part, partials, ctr, out, nullptr, mode, sh);
}

__global__ void k_gate(const double* wnorm, const double* prenorm, int* gate) {
    *gate = (*wnorm < 0.7 * *prenorm) ? 1 : 0;
}

__global__ void k_sub(double* out, const double* b, const double* ax, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = b[i] - ax[i];
}

__global__ void k_gather(double* out, const double* x, int nc, int stride, int f) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x)
        out[i] = x[(int64_t)i * stride + f];
}

__global__ void k_combine(double* y, const double* w, const double* xs, int fx, const double* vs, int fv, int nc,
                          int nb) {
    const int64_t n = (int64_t)nc * nb;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = int(i / nb), f = int(i - (int64_t)c * nb);
        double s = 0.0;
        if (xs && f == fx) s = xs[c];
        if (vs && f == fv) s = s + vs[c];
        y[i] = s + w[i];
    }
}

__global__ void k_add2(double* y, const double* a, const double* b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = a[i] + b[i];
}

__global__ void k_gather_pt(double* out, const double* x, int nc, int nb) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < 2 * nc) out[t] = x[(int64_t)(t >> 1) * nb + nb - 2 + (t & 1)];
}

__global__ void k_scatter_pt(double* y, const double* sub, int nc, int nb) {
    const int64_t n = (int64_t)nc * nb;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = int(i / nb), f = int(i - (int64_t)c * nb);
        y[i] = f >= nb - 2 ? sub[2 * c + (f - (nb - 2))] : 0.0;
    }
}

inline int red_grid(int64_t n) {
    int64_t g = (n + kRT - 1) / kRT;
    return int(std::max<int64_t>(1, std::min<int64_t>(g, kRedBlocks)));
}

}  // namespace

void fill(Ctx& c, double* x, double v, int64_t n) {
    if (n <= 0) return;
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * n);
    k_fill<<<grid_for(n, 256, c.sm_count * 8), 256, 0, c.s>>>(x, v, n);
    check_launch("fill");
}

void fill_pending(Ctx& c, double* x, int64_t n) {
    if (n <= 0) return;
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * n);
    k_fill_bits<<<grid_for(n, 256, c.sm_count * 8), 256, 0, c.s>>>((unsigned long long*)x, kPending, n);
    check_launch("fill_pending");
}

void copy(Ctx& c, double* y, const double* x, int64_t n) {
    if (n <= 0) return;
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * n);
    k_copy<<<grid_for(n, 256, c.sm_count * 8), 256, 0, c.s>>>(y, x, n);
    check_launch("copy");
}

void dot(Ctx& c, const double* a, const double* b, int64_t n, double* out) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * n);
    k_dot<<<red_grid(n), kRT, 0, c.s>>>(a, b, n, c.red.p, c.red_ctr.p, out, 0);
    check_launch("dot");
}

void nrm2(Ctx& c, const double* a, int64_t n, double* out) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * n);
    k_dot<<<red_grid(n), kRT, 0, c.s>>>(a, a, n, c.red.p, c.red_ctr.p, out, 1);
    check_launch("nrm2");
}

void set_reorth_gate(Ctx& c, const double* wnorm, const double* prenorm, int* gate) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 0.0);
    k_gate<<<1, 1, 0, c.s>>>(wnorm, prenorm, gate);
    check_launch("gate");
}

void sub(Ctx& c, double* out, const double* b, const double* ax, int64_t n) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 24.0 * n);
    k_sub<<<grid_for(n, 256, c.sm_count * 8), 256, 0, c.s>>>(out, b, ax, n);
    check_launch("sub");
}

void gather_stride(Ctx& c, double* out, const double* x, int nc, int stride, int f) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * nc);
    k_gather<<<grid_for(nc, 256, c.sm_count * 8), 256, 0, c.s>>>(out, x, nc, stride, f);
    check_launch("gather");
}

void stage_combine(Ctx& c, double* y, const double* w, const double* xs, int fx, const double* vs, int fv, int nc,
                   int nb) {
    const int64_t n = (int64_t)nc * nb;
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 16.0 * n + 8.0 * nc * ((xs ? 1 : 0) + (vs ? 1 : 0)));
    k_combine<<<grid_for(n, 256, c.sm_count * 8), 256, 0, c.s>>>(y, w, xs, fx, vs, fv, nc, nb);
    check_launch("combine");
}

}  // namespace mg

namespace mg {
void add2(Ctx& c, double* y, const double* a, const double* b, int64_t n) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 24.0 * n);
    k_add2<<<grid_for(n, 256, c.sm_count * 8), 256, 0, c.s>>>(y, a, b, n);
    check_launch("add2");
}
void gather_pt(Ctx& c, double* out, const double* x, int nc, int nb) {
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 32.0 * nc);
    k_gather_pt<<<(2 * nc + 255) / 256, 256, 0, c.s>>>(out, x, nc, nb);
    check_launch("gather_pt");
}
void scatter_pt(Ctx& c, double* y, const double* sub, int nc, int nb) {
    const int64_t n = (int64_t)nc * nb;
    Ctx::Scope sc(&c, MPREC_K_BLAS1, 8.0 * n + 16.0 * nc);
    k_scatter_pt<<<grid_for(n, 256, c.sm_count * 8), 256, 0, c.s>>>(y, sub, nc, nb);
    check_launch("scatter_pt");
}
}  // namespace mg
