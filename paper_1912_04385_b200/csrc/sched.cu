// sched.cu -- dependency schedules of the sequential sweeps.
//
// The natural-order sweeps (Gauss-Seidel, amg.cpp:25-43; ILU(0) factor and
// solves, ilu0.cpp) define a DAG: in the forward direction row i depends on
// every stored k < i of row i (backward: k > i).  Warps of the sync-free sweep
// kernels claim rows from an atomic counter; if they claimed rows in index
// order only ~(resident warps / grid width) rows of the wavefront would be in
// flight.  Claiming in topological (level-set) order keeps every claimed row
// at most one level behind the front while preserving deadlock freedom (a row
// is only claimed after all rows it depends on).  The results do not depend on
// the claim order: every row's arithmetic is fixed.
//
// The order is built on the GPU with Kahn's algorithm, one frontier per
// round: round r emits exactly the rows of level r (level(i) = 1 + max level
// of its dependencies), so the number of rounds is the DAG depth (nx+ny-1 on a
// 5-point grid).
#include <cub/cub.cuh>

#include "mprec.cuh"

namespace mg {
namespace {

__global__ void k_indeg(const int* rp, const int* ci, int n, int dir, int* indeg, int* depcnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (dir > 0 ? j < i : j > i) {
            ++d;
            atomicAdd(depcnt + j, 1);
        }
    }
    indeg[i] = d;
}

__global__ void k_dep_fill(const int* rp, const int* ci, int n, int dir, const int* drp, int* fillc, int* dci) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (dir > 0 ? j < i : j > i) dci[drp[j] + atomicAdd(fillc + j, 1)] = i;
    }
}

__global__ void k_zero_flag(const int* indeg, int n, int* flag, int* lev) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        flag[i] = indeg[i] == 0 ? 1 : 0;
        lev[i] = 0;
    }
}

__global__ void k_compact(const int* flag, const int* pos, int n, int* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) out[pos[i]] = i;
}

// st[0] = begin, st[1] = end of the current frontier, st[2] = tail, st[3] = rounds
__global__ void k_round(const int* drp, const int* dci, int* indeg, int* order, int* st, int* lev) {
    const int b = st[0], e = st[1], L = st[3];
    for (int t = b + blockIdx.x * blockDim.x + threadIdx.x; t < e; t += gridDim.x * blockDim.x) {
        const int r = order[t];
        for (int k = drp[r]; k < drp[r + 1]; ++k) {
            const int i = dci[k];
            if (atomicSub(indeg + i, 1) == 1) {
                order[atomicAdd(st + 2, 1)] = i;
                lev[i] = L;
            }
        }
    }
}

__global__ void k_advance(int* st) {
    if (st[1] == st[2]) return;  // done (or stalled)
    st[0] = st[1];
    st[1] = st[2];
    st[3] += 1;
}

}  // namespace

void build_sched(Ctx& c, int n, const int* rp, const int* ci, int dir, Sched& out) {
    out.n = n;
    out.order.alloc(std::max(n, 1));
    out.level.alloc(std::max(n, 1));
    out.nlev = 0;
    if (n == 0) return;
    auto nb = [](int64_t m) { return int(std::max<int64_t>(1, (m + 255) / 256)); };
    DBuf<int> indeg(n), depcnt(n), drp(n + 1), fillc(n), flag(n), pos(n + 1), st(4);
    MG_CUDA(cudaMemsetAsync(depcnt.p, 0, depcnt.bytes(), c.s));
    MG_CUDA(cudaMemsetAsync(fillc.p, 0, fillc.bytes(), c.s));
    k_indeg<<<nb(n), 256, 0, c.s>>>(rp, ci, n, dir, indeg.p, depcnt.p);
    DBuf<char> tmp;
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, depcnt.p, drp.p + 1, n, c.s);
    tmp.alloc(bytes + 16);
    MG_CUDA(cudaMemsetAsync(drp.p, 0, sizeof(int), c.s));
    cub::DeviceScan::InclusiveSum(tmp.p, bytes, depcnt.p, drp.p + 1, n, c.s);
    int ndep = 0;
    MG_CUDA(cudaMemcpyAsync(&ndep, drp.p + n, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    DBuf<int> dci(std::max(ndep, 1));
    k_dep_fill<<<nb(n), 256, 0, c.s>>>(rp, ci, n, dir, drp.p, fillc.p, dci.p);
    k_zero_flag<<<nb(n), 256, 0, c.s>>>(indeg.p, n, flag.p, out.level.p);
    MG_CUDA(cudaMemsetAsync(pos.p, 0, sizeof(int), c.s));
    cub::DeviceScan::InclusiveSum(tmp.p, bytes, flag.p, pos.p + 1, n, c.s);
    k_compact<<<nb(n), 256, 0, c.s>>>(flag.p, pos.p, n, out.order.p);
    int f0 = 0;
    MG_CUDA(cudaMemcpyAsync(&f0, pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    if (f0 == 0) throw Error(MPREC_INTERNAL, "dependency graph has no source (not a DAG)");
    const int init[4] = {0, f0, f0, 1};
    MG_CUDA(cudaMemcpyAsync(st.p, init, sizeof(init), cudaMemcpyHostToDevice, c.s));
    const int grid = c.sm_count * 4;
    int h[4] = {0, 0, 0, 0};
    for (;;) {
        for (int r = 0; r < 64; ++r) {
            k_round<<<grid, 256, 0, c.s>>>(drp.p, dci.p, indeg.p, out.order.p, st.p, out.level.p);
            k_advance<<<1, 1, 0, c.s>>>(st.p);
        }
        check_launch("sched rounds");
        MG_CUDA(cudaMemcpyAsync(h, st.p, sizeof(h), cudaMemcpyDeviceToHost, c.s));
        c.sync();
        if (h[2] >= n || h[0] == h[1]) break;
    }
    if (h[2] != n) throw Error(MPREC_INTERNAL, "dependency schedule incomplete");
    out.nlev = h[3];
}

}  // namespace mg
