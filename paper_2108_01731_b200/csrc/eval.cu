// eval.cu -- quality metrics of the reference's eval module,
// adjusted Rand index and NMI over the label/cluster
// contingency table, average precision/recall against (overlapping)
// ground-truth communities, and cluster statistics.
//
// Everything is sort + run-length work on the device:
//   contingency  : 64-bit keys (a_i, b_i) radix-sorted, run-length encoded
//                  -> one (pair, n_ij) per non-zero cell; marginals by the
//                  same encode over a and b alone; a cell finds its
//                  marginals by binary search in the sorted value lists.
//   pair counts  : sum n_ij^2, sum a^2, sum b^2 in uint64 (exact), then the
//                  sklearn pair-confusion ARI in 128-bit integers on the host
//                  (sklearn.metrics.adjusted_rand_score).
//   NMI          : MI = sum n_ij/N log(N n_ij / (a_i b_j)), arithmetic-mean
//                  normalisation of the entropies, with
//                  sklearn's degenerate cases (both single-cluster -> 1,
//                  one single-cluster -> 0).
//   precision /  : keys (community t, C[member]) sorted and run-length
//   recall         encoded; per t the cell with the largest count, ties to
//                  the lowest cluster id, by a max-reduce of
//                  (count << 32 | ~cluster) per community.
// Labels are any int32 values (ordered as signed).  All sums are
// deterministic (CUB reductions, no float atomics).
#include <cub/cub.cuh>
#include <cmath>

#include "internal.cuh"
#include "prims.cuh"

namespace lcc {
namespace {

__device__ __forceinline__ uint32_t okey(int32_t x) { return (uint32_t)x ^ 0x80000000u; }  // signed order

__global__ void k_okeys(const int32_t* __restrict__ x, int64_t n, uint32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = okey(x[i]);
}
__global__ void k_pair_keys(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                            uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = ((uint64_t)okey(a[i]) << 32) | okey(b[i]);
}

// sorted distinct values (order keys) of x[n] and their counts; returns #distinct
int64_t value_counts(const int32_t* x, int64_t n, Buf<uint32_t>& uniq, Buf<int64_t>& cnt, cudaStream_t s) {
    Buf<uint32_t> k0(n, s), k1(n, s);
    k_okeys<<<grid_for(n, 256), 256, 0, s>>>(x, n, k0.get());
    LCC_LAUNCH_CHECK();
    cub::DoubleBuffer<uint32_t> db(k0.get(), k1.get());
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, n, 0, 32, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, db, n, 0, 32, s));
    }
    uniq.alloc(n, s);
    cnt.alloc(n, s);
    Buf<int64_t> druns(1, s);
    bytes = 0;
    LCC_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, db.Current(), uniq.get(), cnt.get(), druns.get(), n, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), bytes, db.Current(), uniq.get(), cnt.get(), druns.get(),
                                                    n, s));
    }
    int64_t runs = 0;
    LCC_CUDA(cudaMemcpyAsync(&runs, druns.get(), sizeof(runs), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    return runs;
}

__device__ __forceinline__ int64_t find_u32(const uint32_t* __restrict__ v, int64_t n, uint32_t x) {
    int64_t lo = 0, hi = n;  // lower bound
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (v[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

struct Sq64 {
    const int64_t* c;
    __device__ __forceinline__ unsigned long long operator()(int64_t i) const {
        return (unsigned long long)c[i] * (unsigned long long)c[i];
    }
};
struct EntropyTerm {
    const int64_t* c;
    double N;
    __device__ __forceinline__ double operator()(int64_t i) const {
        const double p = (double)c[i] / N;
        return -p * log(p);
    }
};
struct MiTerm {
    const uint64_t* cell;
    const int64_t* nij;
    const uint32_t* ua;
    const int64_t* ca;
    int64_t ka;
    const uint32_t* ub;
    const int64_t* cb;
    int64_t kb;
    double logN, N;
    __device__ __forceinline__ double operator()(int64_t i) const {
        const uint64_t key = cell[i];
        const double ai = (double)ca[find_u32(ua, ka, (uint32_t)(key >> 32))];
        const double bj = (double)cb[find_u32(ub, kb, (uint32_t)key)];
        const double n = (double)nij[i];
        return (n / N) * (log(n) + logN - log(ai) - log(bj));
    }
};

// deterministic device sum of f(0..n-1), returned to the host
template <class T, class F>
T sum_map(F f, int64_t n, cudaStream_t s) {
    cub::TransformInputIterator<T, F, cub::CountingInputIterator<int64_t>> in(cub::CountingInputIterator<int64_t>(0), f);
    Buf<T> d(1, s);
    device_sum(in, d.get(), n, s);
    T h{};
    LCC_CUDA(cudaMemcpyAsync(&h, d.get(), sizeof(T), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    return h;
}

// per-community entries: key (t, okey(C[member])); flags members outside [0, n)
__global__ void k_comm_keys(const int64_t* __restrict__ off, int64_t nc, const int32_t* __restrict__ members,
                            int64_t total, const int32_t* __restrict__ C, int64_t n, uint64_t* __restrict__ out,
                            unsigned* bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nc;  // last t with off[t] <= e
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (off[mid] <= e) lo = mid; else hi = mid;
        }
        const int32_t m = members[e];
        uint32_t ck = 0;
        if (m < 0 || m >= n) atomicOr(bad, 1u);
        else ck = okey(C[m]);
        out[e] = ((uint64_t)lo << 32) | ck;
    }
}
struct CommOf {
    const uint64_t* cell;
    __device__ __forceinline__ int64_t operator()(int64_t i) const { return (int64_t)(cell[i] >> 32); }
};
struct CellScore {  // count << 32 | ~cluster key: max = largest count, then lowest cluster id
    const uint64_t* cell;
    const int64_t* cnt;
    __device__ __forceinline__ unsigned long long operator()(int64_t i) const {
        return ((unsigned long long)cnt[i] << 32) | (uint32_t)~(uint32_t)cell[i];
    }
};
struct PrecRec {
    const int64_t* comm;             // community of each best cell
    const unsigned long long* best;  // its score
    const int64_t* off;
    const uint32_t* ucl;
    const int64_t* ccl;
    int64_t kc;
    bool recall;
    __device__ __forceinline__ double operator()(int64_t i) const {
        const unsigned long long b = best[i];
        const double inter = (double)(b >> 32);
        if (recall) {
            const int64_t t = comm[i];
            return inter / (double)(off[t + 1] - off[t]);
        }
        const uint32_t cl = ~(uint32_t)b;
        return inter / (double)ccl[find_u32(ucl, kc, cl)];
    }
};

}  // namespace

void partition_scores(int64_t n, const int32_t* a, const int32_t* b, double* ari, double* nmi, cudaStream_t s) {
    if (n <= 1) {  // sklearn: one or no sample is a perfect match
        *ari = 1.0;
        *nmi = 1.0;
        return;
    }
    Buf<uint32_t> ua, ub;
    Buf<int64_t> ca, cb;
    const int64_t ka = value_counts(a, n, ua, ca, s);
    const int64_t kb = value_counts(b, n, ub, cb, s);
    // contingency cells
    Buf<uint64_t> k0(n, s), k1(n, s);
    k_pair_keys<<<grid_for(n, 256), 256, 0, s>>>(a, b, n, k0.get());
    LCC_LAUNCH_CHECK();
    cub::DoubleBuffer<uint64_t> db(k0.get(), k1.get());
    sort_keys_db(db, n, 64, s);
    Buf<uint64_t> cell(n, s);
    Buf<int64_t> nij(n, s), druns(1, s);
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, db.Current(), cell.get(), nij.get(), druns.get(), n, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), bytes, db.Current(), cell.get(), nij.get(), druns.get(),
                                                    n, s));
    }
    int64_t kc = 0;
    LCC_CUDA(cudaMemcpyAsync(&kc, druns.get(), sizeof(kc), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    const unsigned long long sij = sum_map<unsigned long long>(Sq64{nij.get()}, kc, s);
    const unsigned long long sa = sum_map<unsigned long long>(Sq64{ca.get()}, ka, s);
    const unsigned long long sb = sum_map<unsigned long long>(Sq64{cb.get()}, kb, s);
    // ARI: sklearn's pair-confusion form (entries are twice the pair counts)
    const __int128 N = n;
    const __int128 tp = (__int128)sij - N;
    const __int128 fp = (__int128)sb - (__int128)sij;
    const __int128 fn = (__int128)sa - (__int128)sij;
    const __int128 tn = N * N - fp - fn - (__int128)sij;
    if (fn == 0 && fp == 0) {
        *ari = 1.0;
    } else {
        const __int128 num = 2 * (tp * tn - fn * fp);
        const __int128 den = (tp + fn) * (fn + tn) + (tp + fp) * (fp + tn);
        *ari = (double)((long double)num / (long double)den);
    }
    // NMI (arithmetic mean of the entropies)
    if ((ka == 1 && kb == 1)) {
        *nmi = 1.0;
        return;
    }
    if (ka == 1 || kb == 1) {
        *nmi = 0.0;
        return;
    }
    const double Nd = (double)n;
    const double mi = std::max(0.0, sum_map<double>(MiTerm{cell.get(), nij.get(), ua.get(), ca.get(), ka, ub.get(),
                                                            cb.get(), kb, std::log(Nd), Nd}, kc, s));
    if (mi == 0.0) {
        *nmi = 0.0;
        return;
    }
    const double ha = sum_map<double>(EntropyTerm{ca.get(), Nd}, ka, s);
    const double hb = sum_map<double>(EntropyTerm{cb.get(), Nd}, kb, s);
    *nmi = mi / std::max(0.5 * (ha + hb), 2.220446049250313e-16);
}

void avg_precision_recall(int64_t n, const int32_t* C, int64_t nc, const int64_t* off, const int32_t* members,
                          double* precision, double* recall, cudaStream_t s) {
    LCC_REQUIRE(nc > 0, "empty ground truth");
    LCC_REQUIRE(nc < (1LL << 31), "too many communities");
    int64_t h_off[2] = {0, 0};
    LCC_CUDA(cudaMemcpyAsync(&h_off[0], off, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaMemcpyAsync(&h_off[1], off + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    LCC_REQUIRE(h_off[0] == 0 && h_off[1] >= nc, "community offsets must start at 0; communities are non-empty");
    const int64_t total = h_off[1];
    Buf<uint32_t> ucl;
    Buf<int64_t> ccl;
    const int64_t kcl = value_counts(C, n, ucl, ccl, s);
    Buf<uint64_t> k0(total, s), k1(total, s);
    Buf<unsigned> bad(1, s);
    LCC_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned), s));
    k_comm_keys<<<grid_for(total, 256), 256, 0, s>>>(off, nc, members, total, C, n, k0.get(), bad.get());
    LCC_LAUNCH_CHECK();
    unsigned hbad = 0;
    LCC_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(hbad), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    LCC_REQUIRE(hbad == 0, "ground-truth member id out of range");
    cub::DoubleBuffer<uint64_t> db(k0.get(), k1.get());
    sort_keys_db(db, total, 32 + bit_width((uint64_t)nc), s);
    Buf<uint64_t> cell(total, s);
    Buf<int64_t> cnt(total, s), druns(1, s);
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, db.Current(), cell.get(), cnt.get(), druns.get(), total, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), bytes, db.Current(), cell.get(), cnt.get(), druns.get(),
                                                    total, s));
    }
    int64_t kcells = 0;
    LCC_CUDA(cudaMemcpyAsync(&kcells, druns.get(), sizeof(kcells), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    // best cell per community
    cub::CountingInputIterator<int64_t> it(0);
    cub::TransformInputIterator<int64_t, CommOf, decltype(it)> comm_in(it, CommOf{cell.get()});
    cub::TransformInputIterator<unsigned long long, CellScore, decltype(it)> score_in(it, CellScore{cell.get(), cnt.get()});
    Buf<int64_t> comm(nc, s), druns2(1, s);
    Buf<unsigned long long> best(nc, s);
    bytes = 0;
    LCC_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, comm_in, comm.get(), score_in, best.get(), druns2.get(),
                                            cub::Max(), kcells, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), bytes, comm_in, comm.get(), score_in, best.get(),
                                                druns2.get(), cub::Max(), kcells, s));
    }
    const double ps = sum_map<double>(PrecRec{comm.get(), best.get(), off, ucl.get(), ccl.get(), kcl, false}, nc, s);
    const double rs = sum_map<double>(PrecRec{comm.get(), best.get(), off, ucl.get(), ccl.get(), kcl, true}, nc, s);
    *precision = ps / (double)nc;
    *recall = rs / (double)nc;
}

void cluster_stats(int64_t n, const int32_t* C, int64_t* num, int64_t* mn, int64_t* mx, double* mean, cudaStream_t s) {
    if (n == 0) {
        *num = *mn = *mx = 0;
        *mean = 0.0;
        return;
    }
    Buf<uint32_t> u;
    Buf<int64_t> c;
    const int64_t k = value_counts(C, n, u, c, s);
    Buf<int64_t> d(2, s);
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceReduce::Min(nullptr, bytes, c.get(), d.get(), k, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceReduce::Min(tmp.get(), bytes, c.get(), d.get(), k, s));
    }
    bytes = 0;
    LCC_CUDA(cub::DeviceReduce::Max(nullptr, bytes, c.get(), d.get() + 1, k, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceReduce::Max(tmp.get(), bytes, c.get(), d.get() + 1, k, s));
    }
    int64_t h[2];
    LCC_CUDA(cudaMemcpyAsync(h, d.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    *num = k;
    *mn = h[0];
    *mx = h[1];
    *mean = (double)n / (double)k;
}

}  // namespace lcc
