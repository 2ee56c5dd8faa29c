// objective.cu -- cc_objective, closed form over unordered pairs:
//   CC = sum_{intra undirected edges} w - lambda * sum_c (K_c^2 - sum_{v in c} k_v^2) / 2
// evaluated as  intra_dir*0.5 - lam*(sum K^2 - sum k^2)*0.5  (same order as the
// oracle).  Unweighted graphs count intra entries in uint64, so the edge term
// is exact and order independent; K sums are integer valued for every config
// (k = 1 or k = degree) and therefore exact in fp64 below 2^53.
#include <cub/cub.cuh>

#include "edgemap.cuh"
#include "internal.cuh"
#include "prims.cuh"

namespace lcc {
namespace {

template <class WT>
struct IntraEdges {
    const int32_t* indices;
    const void* w;
    const int32_t* C;
    unsigned long long* cnt_out;
    double* w_out;
    unsigned long long cnt = 0;
    double acc = 0.0;
    __device__ __forceinline__ void operator()(int64_t v, int64_t e, int64_t) {
        if (__ldg(C + v) == ld_gather_i32(C + __ldg(indices + e))) {
            ++cnt;
            if (WLoad<WT>::weighted) acc += WLoad<WT>::at(w, e);
        }
    }
    __device__ __forceinline__ void flush() {
        for (int d = 16; d; d >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
            acc += __shfl_xor_sync(0xffffffffu, acc, d);
        }
        if ((threadIdx.x & 31) == 0 && cnt) {
            atomicAdd(cnt_out, cnt);
            if (WLoad<WT>::weighted) atomicAdd(w_out, acc);
        }
    }
};

__global__ void k_mass(const int32_t* __restrict__ C, const double* __restrict__ k, int64_t n, double* K) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(K + C[v], k ? k[v] : 1.0);
}

struct Sq {
    __device__ __forceinline__ double operator()(double x) const { return x * x; }
};
struct KSq {
    const double* k;
    __device__ __forceinline__ double operator()(int64_t v) const { const double x = k ? k[v] : 1.0; return x * x; }
};

template <class WT>
double objective_impl(const lcc_graph& g, const double* k, double lam, const int32_t* C, cudaStream_t s) {
    const int64_t n = g.n;
    if (n == 0) return 0.0;
    Buf<unsigned long long> dcnt(1, s);
    Buf<double> dd(3, s);
    LCC_CUDA(cudaMemsetAsync(dcnt.get(), 0, sizeof(unsigned long long), s));
    LCC_CUDA(cudaMemsetAsync(dd.get(), 0, 3 * sizeof(double), s));
    edge_balanced(g.indptr, nullptr, g.indptr, n, g.nnz,
                  IntraEdges<WT>{g.indices, g.weights, C, dcnt.get(), dd.get()}, s);
    Buf<double> K(n, s);
    LCC_CUDA(cudaMemsetAsync(K.get(), 0, sizeof(double) * n, s));
    k_mass<<<grid_for(n, 256), 256, 0, s>>>(C, k, n, K.get());
    LCC_LAUNCH_CHECK();
    cub::TransformInputIterator<double, Sq, const double*> sq(K.get(), Sq{});
    device_sum(sq, dd.get() + 1, n, s);
    cub::TransformInputIterator<double, KSq, cub::CountingInputIterator<int64_t>> ksq(
        cub::CountingInputIterator<int64_t>(0), KSq{k});
    device_sum(ksq, dd.get() + 2, n, s);
    unsigned long long hc = 0;
    double hd[3];
    LCC_CUDA(cudaMemcpyAsync(&hc, dcnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaMemcpyAsync(hd, dd.get(), sizeof(hd), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    const double intra = WLoad<WT>::weighted ? hd[0] : (double)hc;
    return intra * 0.5 - lam * (hd[1] - hd[2]) * 0.5;
}

// weighted_degrees (graph.py:57-61): the reference's np.add.at walks the
// CSR in order, so each row is summed left to right in fp64 -- one thread
// per row, loads unrolled 8 deep so the dependent adds, not the loads, set
// the pace.  Bit-identical to the reference for fp32 / fp64 weights.
template <class WT>
__global__ void k_wdeg(const int64_t* __restrict__ indptr, const void* __restrict__ w, int64_t n, double* out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = indptr[v], e = indptr[v + 1];
        double acc = 0.0;
        int64_t i = b;
        for (; i + 8 <= e; i += 8) {
            double x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = WLoad<WT>::at(w, i + j);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, x[j]);
        }
        for (; i < e; ++i) acc = __dadd_rn(acc, (double)WLoad<WT>::at(w, i));
        out[v] = acc;
    }
}
__global__ void k_deg(const int64_t* __restrict__ indptr, int64_t n, double* out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        out[v] = (double)(indptr[v + 1] - indptr[v]);
}

}  // namespace

void weighted_degrees(const lcc_graph& g, double* k, cudaStream_t s) {
    if (g.n <= 0) return;
    const unsigned grid = grid_for(g.n, 128);
    switch (g.weights ? g.wtype : LCC_W_NONE) {
        case LCC_W_NONE: k_deg<<<grid, 128, 0, s>>>(g.indptr, g.n, k); break;
        case LCC_W_F32: k_wdeg<float><<<grid, 128, 0, s>>>(g.indptr, g.weights, g.n, k); break;
        case LCC_W_F64: k_wdeg<double><<<grid, 128, 0, s>>>(g.indptr, g.weights, g.n, k); break;
        case LCC_W_U32: k_wdeg<uint32_t><<<grid, 128, 0, s>>>(g.indptr, g.weights, g.n, k); break;
        default: throw Invalid("unknown weight dtype");
    }
    LCC_LAUNCH_CHECK();
}

double cc_objective(const lcc_graph& g, const double* k, double lam, const int32_t* C, cudaStream_t s) {
    switch (g.weights ? g.wtype : LCC_W_NONE) {
        case LCC_W_NONE: return objective_impl<WNone>(g, k, lam, C, s);
        case LCC_W_F32: return objective_impl<float>(g, k, lam, C, s);
        case LCC_W_F64: return objective_impl<double>(g, k, lam, C, s);
        case LCC_W_U32: return objective_impl<uint32_t>(g, k, lam, C, s);
        default: throw Invalid("unknown weight dtype");
    }
}

}  // namespace lcc
