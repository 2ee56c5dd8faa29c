// apply.cu -- cluster-mass / active-set update.
//
// apply_moves: the sync apply step and the async boundary
//   reconcile.  Labels are canonicalised to the smallest member
//   id (segmented min by 32-bit atomicMin), then K is rebuilt from scratch
//   with fp64 RED (exact for integer-valued k, which covers every config).
// compute_frontier: AllVertices / VertexNeighbors / ClusterNeighbors
//    as a byte mask scattered by warps
//   over the neighbour lists, then stream-compacted into sorted ids.
#include <cub/cub.cuh>

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

__global__ void k_relabel_mass(const int32_t* __restrict__ L, const int32_t* __restrict__ minm,
                               const double* __restrict__ k, int32_t* C, double* K, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = minm[L[v]];
        C[v] = c;
        atomicAdd(K + c, k ? k[v] : 1.0);
    }
}

// one warp per listed vertex: mark all neighbours
__global__ void k_mark_nbrs_of_moved(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                     const uint8_t* __restrict__ moved, int64_t n, uint8_t* mark) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t v = gw; v < n; v += nw) {
        if (!moved[v]) continue;
        for (int64_t e = indptr[v] + lane; e < indptr[v + 1]; e += 32) mark[indices[e]] = 1;
    }
}

__global__ void k_cluster_flags(const uint8_t* __restrict__ moved, const int32_t* __restrict__ Cold,
                                const int32_t* __restrict__ Cnew, int64_t n, uint8_t* src, uint8_t* dst) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (moved[v]) { src[Cold[v]] = 1; dst[Cnew[v]] = 1; }
}

__global__ void k_mark_cluster_nbrs(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                    const int32_t* __restrict__ Cold, const int32_t* __restrict__ Cnew,
                                    const uint8_t* __restrict__ src, const uint8_t* __restrict__ dst,
                                    int64_t n, uint8_t* mark) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t u = gw; u < n; u += nw) {
        const bool d = dst[Cnew[u]];
        const bool sflag = src[Cold[u]];
        if (d && lane == 0) mark[u] = 1;
        if (!(d || sflag)) continue;
        for (int64_t e = indptr[u] + lane; e < indptr[u + 1]; e += 32) mark[indices[e]] = 1;
    }
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
    k_relabel_mass<<<grid_for(n, 256), 256, 0, s>>>(labels_in, minm.get(), k, C, K, n);
    LCC_LAUNCH_CHECK();
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
    if (policy == LCC_FRONTIER_VERTEX_NBRS) {
        k_mark_nbrs_of_moved<<<grid_for(n * 32, 256, 16), 256, 0, s>>>(g.indptr, g.indices, moved, n, mark.get());
        LCC_LAUNCH_CHECK();
    } else {
        Buf<uint8_t> flags(2 * n, s);
        LCC_CUDA(cudaMemsetAsync(flags.get(), 0, 2 * n, s));
        k_cluster_flags<<<grid_for(n, 256), 256, 0, s>>>(moved, C_old, C_new, n, flags.get(), flags.get() + n);
        LCC_LAUNCH_CHECK();
        k_mark_cluster_nbrs<<<grid_for(n * 32, 256, 16), 256, 0, s>>>(g.indptr, g.indices, C_old, C_new,
                                                                     flags.get(), flags.get() + n, n, mark.get());
        LCC_LAUNCH_CHECK();
    }
    select_flagged(cub::CountingInputIterator<int32_t>(0), mark.get(), frontier, dcnt.get(), n, s);
    int64_t h = 0;
    LCC_CUDA(cudaMemcpyAsync(&h, dcnt.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    return h;
}

}  // namespace lcc
