// apply.cu -- cluster-mass / active-set update.
//
// apply_moves: the sync apply step and the async boundary
//   reconcile.  Labels are canonicalised to the smallest member
//   id (segmented min by 32-bit atomicMin), then K is rebuilt from scratch
//   with fp64 RED (exact for integer-valued k, which covers every config);
//   a non-integral k switches to a fixed-order segmented sum.
// compute_frontier: AllVertices / VertexNeighbors / ClusterNeighbors
//    as a byte mask scattered over the
//   contributing vertices' neighbour lists by the edge-balanced map
//   (edgemap.cuh: hubs cost the same per edge as leaves), then
//   stream-compacted into sorted ids.
#include <cub/cub.cuh>

#include "edgemap.cuh"
#include "internal.cuh"
#include "prims.cuh"

namespace lcc {
namespace {

__global__ void k_iota(int32_t* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

__global__ void k_fill_k(double* K, const double* __restrict__ k, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        K[i] = k ? k[i] : 1.0;
}

__global__ void k_min_member(const int32_t* __restrict__ L, int32_t* minm, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t l = L[v];
        // members whose label equals their own id are the common case after
        // canonicalisation; a plain compare avoids most atomics
        if (minm[l] > (int32_t)v) atomicMin(minm + l, (int32_t)v);
    }
}

// fp64 RED per vertex: exact (so order free) while every k is an integer --
// k = 1 or an unweighted degree, every BASELINE config.  A non-integral k
// sets *nonint and the host redoes K in a fixed order (mass_fixed_order).
__global__ void k_relabel_mass(const int32_t* __restrict__ L, const int32_t* __restrict__ minm,
                               const double* __restrict__ k, int32_t* C, double* K, int64_t n,
                               unsigned* nonint) {
    bool frac = false;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = minm[L[v]];
        C[v] = c;
        const double x = k ? k[v] : 1.0;
        frac |= x != floor(x) || fabs(x) >= 4503599627370496.0;  // 2^52: sums may round
        atomicAdd(K + c, x);
    }
    if (nonint && __any_sync(__activemask(), frac) && (threadIdx.x & 31) == 0) *nonint = 1u;
}

__global__ void k_gather_k(const int32_t* __restrict__ members, const double* __restrict__ k, int64_t n,
                           double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = k[members[i]];
}

__global__ void k_scatter_mass(const int32_t* __restrict__ ids, const double* __restrict__ sums,
                               const int64_t* __restrict__ nruns, double* K) {
    const int64_t r = *nruns;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r; i += (int64_t)gridDim.x * blockDim.x)
        K[ids[i]] = sums[i];
}

// K[c] = sum of k over the members of c in a fixed order: members sorted by
// (label, id) -- a stable radix sort of the labels over the ids -- then one
// reduce-by-key.  Same inputs, same bits on every run (sync determinism,
// SPEC.md:306) for any real-valued k.
void mass_fixed_order(int64_t n, const int32_t* C, const double* k, double* K, cudaStream_t s) {
    Buf<int32_t> lab(n, s), ids(n, s), ids_in(n, s), runs(n, s);
    Buf<double> kv(n, s), sums(n, s);
    Buf<int64_t> nruns(1, s);
    fill_iota(ids_in.get(), n, s);
    const int bits = std::max(1, bit_width((uint64_t)n));
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, C, lab.get(), ids_in.get(), ids.get(), n, 0, bits, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, C, lab.get(), ids_in.get(), ids.get(), n, 0,
                                                 bits, s));
    }
    k_gather_k<<<grid_for(n, 256), 256, 0, s>>>(ids.get(), k, n, kv.get());
    LCC_LAUNCH_CHECK();
    bytes = 0;
    LCC_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, lab.get(), runs.get(), kv.get(), sums.get(),
                                            nruns.get(), cub::Sum(), n, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), bytes, lab.get(), runs.get(), kv.get(), sums.get(),
                                                nruns.get(), cub::Sum(), n, s));
    }
    LCC_CUDA(cudaMemsetAsync(K, 0, sizeof(double) * n, s));
    k_scatter_mass<<<grid_for(n, 256), 256, 0, s>>>(runs.get(), sums.get(), nruns.get(), K);
    LCC_LAUNCH_CHECK();
}

struct HasEdgesAndFlag {
    const int64_t* indptr;
    const uint8_t* flag;
    __device__ __forceinline__ bool operator()(int32_t v) const {
        return flag[v] && indptr[v + 1] > indptr[v];
    }
};
struct ListDeg {
    const int64_t* indptr;
    const int32_t* list;
    int64_t n;
    __device__ __forceinline__ int64_t operator()(int64_t i) const {
        if (i >= n) return 0;
        const int32_t v = list[i];
        return indptr[v + 1] - indptr[v];
    }
};
// edge functor: mark the neighbour
struct MarkNbr {
    const int32_t* indices;
    uint8_t* mark;
    __device__ __forceinline__ void operator()(int64_t, int64_t e, int64_t) const { mark[__ldg(indices + e)] = 1; }
    __device__ __forceinline__ void flush() const {}
};

__global__ void k_cluster_flags(const uint8_t* __restrict__ moved, const int32_t* __restrict__ Cold,
                                const int32_t* __restrict__ Cnew, int64_t n, uint8_t* src, uint8_t* dst) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (moved[v]) { src[Cold[v]] = 1; dst[Cnew[v]] = 1; }
}

__global__ void k_cluster_contrib(const int32_t* __restrict__ Cold, const int32_t* __restrict__ Cnew,
                                  const uint8_t* __restrict__ src, const uint8_t* __restrict__ dst, int64_t n,
                                  uint8_t* contrib) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        contrib[u] = (src[Cold[u]] || dst[Cnew[u]]) ? 1 : 0;
}

__global__ void k_mark_dst_members(const int32_t* __restrict__ Cnew, const uint8_t* __restrict__ dst, int64_t n,
                                   uint8_t* mark) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        if (dst[Cnew[u]]) mark[u] = 1;
}

}  // namespace

void fill_iota(int32_t* p, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(p, n);
    LCC_LAUNCH_CHECK();
}

void fill_k(double* K, const double* k, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_fill_k<<<grid_for(n, 256), 256, 0, s>>>(K, k, n);
    LCC_LAUNCH_CHECK();
}

void apply_moves(int64_t n, const int32_t* labels_in, int64_t label_range, const double* k,
                 int32_t* C, double* K, cudaStream_t s) {
    if (n <= 0) return;
    Buf<int32_t> minm(label_range, s);
    LCC_CUDA(cudaMemsetAsync(minm.get(), 0x7f, sizeof(int32_t) * label_range, s));
    k_min_member<<<grid_for(n, 256), 256, 0, s>>>(labels_in, minm.get(), n);
    LCC_LAUNCH_CHECK();
    LCC_CUDA(cudaMemsetAsync(K, 0, sizeof(double) * n, s));
    if (!k) {  // k = 1: integer sums, exact in any order
        k_relabel_mass<<<grid_for(n, 256), 256, 0, s>>>(labels_in, minm.get(), k, C, K, n, nullptr);
        LCC_LAUNCH_CHECK();
        return;
    }
    Buf<unsigned> nonint(1, s);
    LCC_CUDA(cudaMemsetAsync(nonint.get(), 0, sizeof(unsigned), s));
    k_relabel_mass<<<grid_for(n, 256), 256, 0, s>>>(labels_in, minm.get(), k, C, K, n, nonint.get());
    LCC_LAUNCH_CHECK();
    unsigned h = 0;
    LCC_CUDA(cudaMemcpyAsync(&h, nonint.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    if (h) mass_fixed_order(n, C, k, K, s);
}

int64_t compute_frontier(const lcc_graph& g, int policy, const uint8_t* moved, const int32_t* C_old,
                         const int32_t* C_new, int32_t* frontier, cudaStream_t s) {
    const int64_t n = g.n;
    if (n == 0) return 0;
    LCC_REQUIRE(policy >= LCC_FRONTIER_ALL && policy <= LCC_FRONTIER_CLUSTER_NBRS, "unknown frontier policy");
    Buf<int64_t> dcnt(1, s);
    // any move at all?  (moved == empty -> empty frontier)
    {
        cub::TransformInputIterator<int64_t, cub::CastOp<int64_t>, const uint8_t*> mv(moved, cub::CastOp<int64_t>());
        device_sum(mv, dcnt.get(), n, s);
        int64_t h = 0;
        LCC_CUDA(cudaMemcpyAsync(&h, dcnt.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
        if (h == 0) return 0;
    }
    if (policy == LCC_FRONTIER_ALL) {
        fill_iota(frontier, n, s);
        return n;
    }
    Buf<uint8_t> mark(n, s);
    LCC_CUDA(cudaMemsetAsync(mark.get(), 0, n, s));
    // contributing vertices (movers, or members of affected clusters) are
    // compacted first so every list entry has degree >= 1 and the edge map's
    // per-tile window stays in shared memory
    Buf<uint8_t> contrib;
    const uint8_t* cflag = moved;
    Buf<uint8_t> flags;
    if (policy == LCC_FRONTIER_CLUSTER_NBRS) {
        flags.alloc(2 * n, s);
        LCC_CUDA(cudaMemsetAsync(flags.get(), 0, 2 * n, s));
        k_cluster_flags<<<grid_for(n, 256), 256, 0, s>>>(moved, C_old, C_new, n, flags.get(), flags.get() + n);
        LCC_LAUNCH_CHECK();
        k_mark_dst_members<<<grid_for(n, 256), 256, 0, s>>>(C_new, flags.get() + n, n, mark.get());
        LCC_LAUNCH_CHECK();
        contrib.alloc(n, s);
        k_cluster_contrib<<<grid_for(n, 256), 256, 0, s>>>(C_old, C_new, flags.get(), flags.get() + n, n, contrib.get());
        LCC_LAUNCH_CHECK();
        cflag = contrib.get();
    }
    Buf<int32_t> clist(n, s);
    select_if(cub::CountingInputIterator<int32_t>(0), clist.get(), dcnt.get(), n,
              HasEdgesAndFlag{g.indptr, cflag}, s);
    int64_t nc = 0;
    LCC_CUDA(cudaMemcpyAsync(&nc, dcnt.get(), sizeof(nc), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    if (nc > 0) {
        Buf<int64_t> off(nc + 1, s);
        cub::TransformInputIterator<int64_t, ListDeg, cub::CountingInputIterator<int64_t>> degs(
            cub::CountingInputIterator<int64_t>(0), ListDeg{g.indptr, clist.get(), nc});
        exclusive_sum(degs, off.get(), nc + 1, s);
        int64_t total = 0;
        LCC_CUDA(cudaMemcpyAsync(&total, off.get() + nc, sizeof(total), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
        edge_balanced(g.indptr, clist.get(), off.get(), nc, total, MarkNbr{g.indices, mark.get()}, s);
    }
    return frontier_from_mask(n, mark.get(), frontier, s);
}

int64_t frontier_from_mask(int64_t n, const uint8_t* mark, int32_t* frontier, cudaStream_t s) {
    if (n <= 0) return 0;
    Buf<int64_t> dcnt(1, s);
    select_flagged(cub::CountingInputIterator<int32_t>(0), mark, frontier, dcnt.get(), n, s);
    int64_t h = 0;
    LCC_CUDA(cudaMemcpyAsync(&h, dcnt.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    return h;
}

}  // namespace lcc
