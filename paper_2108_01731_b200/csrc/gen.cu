// gen.cu -- device graph build + R-MAT generator.
//
// build_csr_from_pairs follows the reference's build_graph contract for
// unweighted input (graph.py:98-164): self-loops dropped, duplicate
// unordered pairs merged, both orientations emitted, rows sorted.  (For
// unweighted inputs with the pairs deduplicated first -- SURVEY.md erratum 3
// -- every merged edge keeps w = 1.)
// gen_rmat draws `samples` directed edges by recursive quadrant descent with
// a counter-based splitmix64 stream, so the same graph can be regenerated on
// the host for tests (paper_2108_01731_b200/gen.py: rmat_pairs_host).
#include <cub/cub.cuh>

#include "internal.cuh"
#include "prims.cuh"

namespace lcc {
namespace {

__global__ void k_pair_keys(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t np, int bits,
                            uint64_t* keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = (uint32_t)u[i], b = (uint32_t)v[i];
        if (a == b) keys[i] = ~0ULL;
        else keys[i] = a < b ? ((a << bits) | b) : ((b << bits) | a);
    }
}

__global__ void k_both_dirs(const uint64_t* __restrict__ uk, int64_t m, int bits, uint64_t* out) {
    const uint64_t mask = (1ULL << bits) - 1ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = uk[i] >> bits, hi = uk[i] & mask;
        out[2 * i] = uk[i];
        out[2 * i + 1] = (hi << bits) | lo;
    }
}

__global__ void k_csr_rows(const uint64_t* __restrict__ keys, int64_t R, int bits, int64_t n, int64_t* indptr,
                           int32_t* indices) {
    const uint64_t mask = (1ULL << bits) - 1ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i < R ? (int64_t)(keys[i] >> bits) : n;
        const int64_t prev = i > 0 ? (int64_t)(keys[i - 1] >> bits) : -1;
        for (int64_t r = prev + 1; r <= row; ++r) indptr[r] = i;
        if (i < R) indices[i] = (int32_t)(keys[i] & mask);
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void k_rmat(int scale, int64_t samples, double t1, double t2, double t3, uint64_t seed, int32_t* u,
                       int32_t* v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < samples; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t src = 0, dst = 0;
        for (int l = 0; l < scale; ++l) {
            const uint64_t ctr = (uint64_t)i * (uint64_t)scale + (uint64_t)l + 1ULL;
            const uint64_t z = splitmix64(seed + 0x9E3779B97F4A7C15ULL * ctr);
            const double r = (double)(z >> 11) * 0x1.0p-53;
            const uint32_t bs = r >= t2 ? 1u : 0u;                 // quadrants c, d -> src bit
            const uint32_t bd = (r >= t1 && r < t2) || r >= t3 ? 1u : 0u;  // b, d -> dst bit
            src = (src << 1) | bs;
            dst = (dst << 1) | bd;
        }
        u[i] = (int32_t)src;
        v[i] = (int32_t)dst;
    }
}

// Power-law planted communities (config 5): Chung-Lu draws, intra-community
// with probability 1-mu (community chosen by weight, endpoints by weight inside
// it), else endpoints by weight over the whole graph.  Vertices of a
// community are contiguous ids; vw_prefix is the inclusive-exclusive prefix of
// the vertex weights (vw_prefix[0] = 0), cw_prefix the same per community.
__device__ __forceinline__ double u01(uint64_t seed, uint64_t ctr) {
    return (double)(splitmix64(seed + 0x9E3779B97F4A7C15ULL * ctr) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ int64_t prefix_search(const double* __restrict__ p, int64_t lo, int64_t hi, double x) {
    // largest i in [lo, hi) with p[i] <= x
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (p[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}
__global__ void k_plc(int64_t samples, double mu, const double* __restrict__ vw, int64_t n,
                      const int64_t* __restrict__ cstart, const double* __restrict__ cw, int64_t nc, uint64_t seed,
                      int32_t* u, int32_t* v) {
    const double W = vw[n];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < samples; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t base = (uint64_t)i * 4ULL + 1ULL;
        int64_t a, b;
        if (u01(seed, base) >= mu) {
            const int64_t c = prefix_search(cw, 0, nc, u01(seed, base + 1) * cw[nc]);
            const int64_t s = cstart[c], e = cstart[c + 1];
            const double w0 = vw[s], ws = vw[e] - vw[s];
            a = prefix_search(vw, s, e, w0 + u01(seed, base + 2) * ws);
            b = prefix_search(vw, s, e, w0 + u01(seed, base + 3) * ws);
        } else {
            a = prefix_search(vw, 0, n, u01(seed, base + 2) * W);
            b = prefix_search(vw, 0, n, u01(seed, base + 3) * W);
        }
        u[i] = (int32_t)a;
        v[i] = (int32_t)b;
    }
}

int64_t csr_from_pairs_impl(int64_t n, int64_t np, const int32_t* u, const int32_t* v, Buf<int32_t>* owned_u,
                            Buf<int32_t>* owned_v, int64_t* indptr, int32_t* indices, cudaStream_t s);

}  // namespace

int64_t gen_powerlaw_communities(int64_t n, int64_t samples, double mu, const double* vw_prefix,
                                 const int64_t* cstart, const double* cw_prefix, int64_t nc, uint64_t seed,
                                 int64_t* indptr, int32_t* indices, cudaStream_t s) {
    LCC_REQUIRE(n > 0 && n < (1LL << 31), "vertex count out of range");
    LCC_REQUIRE(nc > 0 && samples >= 0 && mu >= 0.0 && mu <= 1.0, "bad generator parameters");
    Buf<int32_t> u(std::max<int64_t>(samples, 1), s), v(std::max<int64_t>(samples, 1), s);
    if (samples > 0) {
        k_plc<<<grid_for(samples, 256, 16), 256, 0, s>>>(samples, mu, vw_prefix, n, cstart, cw_prefix, nc, seed,
                                                         u.get(), v.get());
        LCC_LAUNCH_CHECK();
    }
    return csr_from_pairs_impl(n, samples, u.get(), v.get(), &u, &v, indptr, indices, s);
}

namespace {
// Keys the pairs, then (when `owned`) frees them before the sorts; double-
// buffered radix sorts keep the peak at two key buffers.
int64_t csr_from_pairs_impl(int64_t n, int64_t np, const int32_t* u, const int32_t* v, Buf<int32_t>* owned_u,
                            Buf<int32_t>* owned_v, int64_t* indptr, int32_t* indices, cudaStream_t s) {
    LCC_REQUIRE(n > 0 && n < (1LL << 31), "vertex count out of range");
    LCC_REQUIRE(np >= 0, "negative pair count");
    const int bits = std::max(1, bit_width((uint64_t)(n - 1)));
    if (np == 0) {
        LCC_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int64_t) * (n + 1), s));
        return 0;
    }
    Buf<uint64_t> k1(np, s), k2(np, s);
    k_pair_keys<<<grid_for(np, 256), 256, 0, s>>>(u, v, np, bits, k1.get());
    LCC_LAUNCH_CHECK();
    if (owned_u) owned_u->release();
    if (owned_v) owned_v->release();
    cub::DoubleBuffer<uint64_t> db(k1.get(), k2.get());
    sort_keys_db(db, np, 2 * bits, s);  // sentinel ~0 keeps the max on these bits too
    uint64_t* sorted = db.Current();
    uint64_t* other = db.Alternate();
    Buf<int64_t> dcnt(1, s);
    {
        size_t bytes = 0;
        LCC_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, sorted, other, dcnt.get(), np, s));
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceSelect::Unique(tmp.get(), bytes, sorted, other, dcnt.get(), np, s));
    }
    int64_t nu = 0;
    uint64_t last = 0;
    LCC_CUDA(cudaMemcpyAsync(&nu, dcnt.get(), sizeof(nu), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    if (nu > 0) {
        LCC_CUDA(cudaMemcpyAsync(&last, other + nu - 1, sizeof(last), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
    }
    const int64_t m = nu - (nu > 0 && last == ~0ULL ? 1 : 0);
    Buf<uint64_t>& uniq = other == k1.get() ? k1 : k2;
    (other == k1.get() ? k2 : k1).release();
    Buf<uint64_t> d1(2 * std::max<int64_t>(m, 1), s), d2(2 * std::max<int64_t>(m, 1), s);
    uint64_t* rows = d1.get();
    if (m > 0) {
        k_both_dirs<<<grid_for(m, 256), 256, 0, s>>>(uniq.get(), m, bits, d1.get());
        LCC_LAUNCH_CHECK();
        uniq.release();
        cub::DoubleBuffer<uint64_t> dd(d1.get(), d2.get());
        sort_keys_db(dd, 2 * m, 2 * bits, s);
        rows = dd.Current();
    }
    k_csr_rows<<<grid_for(2 * m + 1, 256), 256, 0, s>>>(rows, 2 * m, bits, n, indptr, indices);
    LCC_LAUNCH_CHECK();
    LCC_CUDA(cudaStreamSynchronize(s));
    return 2 * m;
}
}  // namespace

int64_t build_csr_from_pairs(int64_t n, int64_t np, const int32_t* u, const int32_t* v, int64_t* indptr,
                             int32_t* indices, cudaStream_t s) {
    return csr_from_pairs_impl(n, np, u, v, nullptr, nullptr, indptr, indices, s);
}

int64_t gen_rmat(int scale, int64_t samples, double a, double b, double c, uint64_t seed, int64_t* indptr,
                 int32_t* indices, cudaStream_t s) {
    LCC_REQUIRE(scale >= 1 && scale <= 30, "scale must lie in [1, 30]");
    LCC_REQUIRE(samples >= 0, "negative sample count");
    LCC_REQUIRE(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0 + 1e-9, "quadrant probabilities must be >= 0 and sum to 1");
    const int64_t n = 1LL << scale;
    Buf<int32_t> u(std::max<int64_t>(samples, 1), s), v(std::max<int64_t>(samples, 1), s);
    const double t1 = a, t2 = a + b, t3 = a + b + c;
    if (samples > 0) {
        k_rmat<<<grid_for(samples, 256, 16), 256, 0, s>>>(scale, samples, t1, t2, t3, seed, u.get(), v.get());
        LCC_LAUNCH_CHECK();
    }
    return csr_from_pairs_impl(n, samples, u.get(), v.get(), &u, &v, indptr, indices, s);
}

}  // namespace lcc
