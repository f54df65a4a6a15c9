// common.cuh -- runtime infrastructure of libmprec_gpu.so: errors, device
// buffers, the per-handle stream context, launch accounting and kernel-class
// timing.  Every kernel in this library is launched through Ctx so that launch
// counts and (when profiling) CUDA-event durations are recorded on the stream
// the kernel actually runs on.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "mprec_gpu.h"

namespace mg {

struct Error : std::runtime_error {
    int code;
    int payload;
    Error(int c, const std::string& m, int p = -1) : std::runtime_error(m), code(c), payload(p) {}
};

#define MG_CUDA(expr)                                                                            \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess)                                                                   \
            throw ::mg::Error(MPREC_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// Device-side bounds checks of the sync-free / level-synchronous kernels, compiled
// only into the checked build (libmprec_gpu_checked.so, -DMPREC_CHECKED; the
// pool's compute-sanitizer is unavailable): a failed check prints and traps, the
// launch then fails with cudaErrorLaunchFailure -> MPREC_CUDA.
#ifdef MPREC_CHECKED
#define MG_DCHECK(cond)                                                                         \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("[mprec checked] %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x, #cond);                                                        \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define MG_DCHECK(cond) \
    do {                \
    } while (0)
#endif

inline void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(MPREC_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- stream-ordered allocation scope -------------------------------------------
// cudaMalloc / cudaFree may synchronise the whole device.  While two host
// threads build independent structures on two streams (the AMG hierarchies of
// one setup), each thread allocates and frees stream-ordered on its own stream
// (cudaMallocAsync / cudaFreeAsync), so neither waits for the other's kernels.
inline cudaStream_t& tl_alloc_stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}
struct StreamAllocScope {
    cudaStream_t prev;
    explicit StreamAllocScope(cudaStream_t s) : prev(tl_alloc_stream()) { tl_alloc_stream() = s; }
    ~StreamAllocScope() { tl_alloc_stream() = prev; }
};

// ---- device buffer ---------------------------------------------------------
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    bool async_ = false;  // allocated stream-ordered (StreamAllocScope)
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), async_(o.async_) {
        o.p = nullptr;
        o.n = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            async_ = o.async_;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) {
            if (cudaStream_t s = tl_alloc_stream()) {
                MG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
                async_ = true;
            } else {
                MG_CUDA(cudaMalloc(&p, count * sizeof(T)));
                async_ = false;
            }
        }
        n = count;
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p) {
            cudaStream_t s = tl_alloc_stream();
            if (async_ && s)
                cudaFreeAsync(p, s);
            else
                cudaFree(p);
        }
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    void upload(const T* h, size_t count, cudaStream_t s) {
        ensure(count);
        if (count) MG_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void download(T* h, size_t count, cudaStream_t s) const {
        if (count) MG_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    std::vector<T> to_host(cudaStream_t s, size_t count = size_t(-1)) const {
        if (count == size_t(-1)) count = n;
        std::vector<T> h(count);
        download(h.data(), count, s);
        MG_CUDA(cudaStreamSynchronize(s));
        return h;
    }
};

// ---- per-handle execution context -------------------------------------------
struct KStat {
    double ms = 0.0;
    int64_t launches = 0;
    double bytes = 0.0;
};

struct Ctx {
    cudaStream_t s = nullptr;
    int sm_count = 148;
    bool profile = false;
    int64_t launches = 0;
    KStat stat[MPREC_K_COUNT];
    // pending event pairs (class, bytes, start, stop) harvested at sync points
    struct Pending {
        int kc;
        double bytes;
        cudaEvent_t a, b;
        bool gated;  // launched under a device gate not yet resolved (resolve_gate)
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    DBuf<double> red;      // reduction partials
    DBuf<unsigned> red_ctr;  // last-block counters
    DBuf<double> scal;     // device scalars (norms, dots)
    DBuf<int> counters;    // work-distribution counters
    DBuf<int> err;         // device error slots

    Ctx();
    ~Ctx();
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;

    cudaEvent_t get_event();
    // Bracket a launch of kernel class kc with algorithmic byte count `bytes`.
    // gated: the kernel exits at once unless a device flag is set; its bytes are
    // held back until the host learns the flag (resolve_gate) and charged only
    // when it fired.
    struct Scope {
        Ctx* c;
        int kc;
        double bytes;
        bool gated;
        cudaEvent_t a = nullptr;
        Scope(Ctx* c_, int kc_, double bytes_, bool gated_ = false);
        ~Scope();
    };
    double gated_bytes[MPREC_K_COUNT] = {};  // non-profiling mode: held-back bytes
    int unresolved_gated = 0;
    void resolve_gate(bool fired);
    void harvest();  // fold completed event pairs into stat (synchronizes)
    void sync() {
        MG_CUDA(cudaStreamSynchronize(s));
        if (!pending.empty()) harvest();
    }
    void reset_stats() {
        harvest();
        for (auto& k : stat) k = KStat{};
        launches = 0;
    }
};

// MPREC_TRACE=1: setup phase timings on stderr (synchronising; diagnostics only)
bool trace_on();
struct Trace {
    const char* what;
    Ctx* c;
    double t0;
    Trace(Ctx* c_, const char* w);
    ~Trace();
};

constexpr int kRedBlocks = 1184;  // 8 x 148: partials of the deterministic reductions

inline int grid_for(int64_t work, int threads, int cap = 148 * 32) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return int(g);
}

}  // namespace mg
