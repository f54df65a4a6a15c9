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

inline void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(MPREC_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- deferred frees -----------------------------------------------------------
// cudaFree synchronises the whole device.  While two host threads build
// independent structures on two streams (the AMG hierarchies of one setup),
// each thread parks the blocks it frees in a thread-local pool and reuses them
// for its own later allocations (same thread = same stream, so stream order
// makes the reuse safe); the pool is released when the scope ends.
struct DeferredPool {
    std::vector<std::pair<size_t, void*>> blocks;
};
inline DeferredPool*& tl_deferred_pool() {
    static thread_local DeferredPool* p = nullptr;
    return p;
}
struct DeferFreeScope {
    DeferredPool pool;
    DeferredPool* prev;
    DeferFreeScope() : prev(tl_deferred_pool()) { tl_deferred_pool() = &pool; }
    ~DeferFreeScope() {
        tl_deferred_pool() = prev;
        for (auto& b : pool.blocks) cudaFree(b.second);
    }
};
// a parked block of at least `bytes` (smallest fit), or nullptr
inline void* deferred_take(size_t bytes, size_t* cap) {
    DeferredPool* p = tl_deferred_pool();
    if (!p) return nullptr;
    size_t best = size_t(-1);
    int bi = -1;
    for (int k = 0; k < int(p->blocks.size()); ++k)
        if (p->blocks[k].first >= bytes && p->blocks[k].first < best && p->blocks[k].first <= 2 * bytes + (1 << 20)) {
            best = p->blocks[k].first;
            bi = k;
        }
    if (bi < 0) return nullptr;
    void* ptr = p->blocks[bi].second;
    *cap = p->blocks[bi].first;
    p->blocks[bi] = p->blocks.back();
    p->blocks.pop_back();
    return ptr;
}
inline bool deferred_park(void* ptr, size_t cap) {
    DeferredPool* p = tl_deferred_pool();
    if (!p) return false;
    p->blocks.emplace_back(cap, ptr);
    return true;
}

// ---- device buffer ---------------------------------------------------------
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    size_t cap = 0;  // bytes of the underlying block
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) {
        o.p = nullptr;
        o.n = 0;
        o.cap = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            cap = o.cap;
            o.p = nullptr;
            o.n = 0;
            o.cap = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) {
            const size_t bytes = count * sizeof(T);
            if (void* q = deferred_take(bytes, &cap)) {
                p = static_cast<T*>(q);
            } else {
                MG_CUDA(cudaMalloc(&p, bytes));
                cap = bytes;
            }
        }
        n = count;
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p && !deferred_park(p, cap)) cudaFree(p);
        p = nullptr;
        n = 0;
        cap = 0;
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
    struct Scope {
        Ctx* c;
        int kc;
        double bytes;
        cudaEvent_t a = nullptr;
        Scope(Ctx* c_, int kc_, double bytes_);
        ~Scope();
    };
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
