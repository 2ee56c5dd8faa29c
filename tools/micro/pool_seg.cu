// Micro-benchmarks: (1) stream-ordered pool growth cost, (2) CUB segmented
// sort on many small segments plus a few huge ones.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void fill(uint32_t* k, int64_t n, uint32_t mod) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        k[i] = (uint32_t)((i * 2654435761ull) % mod);
}

int main() {
    cudaStream_t s; CK(cudaStreamCreate(&s));
    cudaMemPool_t pool; CK(cudaDeviceGetDefaultMemPool(&pool, 0));
    uint64_t thr = ~0ull; CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (size_t gb : {1, 4, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaMemPoolTrimTo(pool, 0));
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a, s);
            void* p; CK(cudaMallocAsync(&p, gb << 30, s));
            CK(cudaMemsetAsync(p, 0, gb << 30, s));
            cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            CK(cudaFreeAsync(p, s)); CK(cudaStreamSynchronize(s));
            // reuse from pool
            cudaEventRecord(a, s);
            CK(cudaMallocAsync(&p, gb << 30, s));
            CK(cudaMemsetAsync(p, 0, gb << 30, s));
            cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
            float ms2; cudaEventElapsedTime(&ms2, a, b);
            CK(cudaFreeAsync(p, s)); CK(cudaStreamSynchronize(s));
            printf("pool growth %zu GB: fresh %.2f ms, reused %.2f ms\n", gb, ms, ms2);
        }
    }
    // segmented sort: n keys, segments of random length (mean ~35) + big ones
    const int64_t n = 500000000;
    std::mt19937_64 rng(1);
    std::vector<int> off{0};
    std::geometric_distribution<int> geo(1.0 / 35);
    std::vector<int64_t> bigs = {5000000, 2000000, 1000000, 400000, 400000, 200000};
    size_t bi = 0;
    while (off.back() < n) {
        int64_t len = (bi < bigs.size() && off.size() % 1000000 == 7) ? bigs[bi++] : 1 + geo(rng);
        off.push_back((int)std::min<int64_t>(n, off.back() + len));
    }
    const int segs = (int)off.size() - 1;
    printf("segments %d, big %zu\n", segs, bi);
    int* doff; CK(cudaMalloc(&doff, sizeof(int) * off.size()));
    CK(cudaMemcpy(doff, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
    uint32_t *k1, *k2; CK(cudaMalloc(&k1, 4 * n)); CK(cudaMalloc(&k2, 4 * n));
    for (int rep = 0; rep < 3; ++rep) {
        fill<<<1184, 256, 0, s>>>(k1, n, 14700000u);
        cub::DoubleBuffer<uint32_t> db(k1, k2);
        size_t bytes = 0;
        cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, db, (int)n, segs, doff, doff + 1, s);
        void* tmp; CK(cudaMalloc(&tmp, bytes));
        CK(cudaStreamSynchronize(s));
        cudaEventRecord(a, s);
        CK(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, db, (int)n, segs, doff, doff + 1, s));
        cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("segmented sort %lld keys: %.2f ms\n", (long long)n, ms);
        CK(cudaFree(tmp));
    }
    // same without the big segments (shrink them to 1 element by remapping)
    std::vector<int> off2{0};
    for (int i = 1; i < (int)off.size(); ++i) {
        int64_t len = off[i] - off[i - 1];
        off2.push_back(off2.back() + (int)(len > 65536 ? 1 : len));
    }
    const int n2 = off2.back();
    CK(cudaMemcpy(doff, off2.data(), sizeof(int) * off2.size(), cudaMemcpyHostToDevice));
    for (int rep = 0; rep < 2; ++rep) {
        fill<<<1184, 256, 0, s>>>(k1, n2, 14700000u);
        cub::DoubleBuffer<uint32_t> db(k1, k2);
        size_t bytes = 0;
        cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, db, n2, segs, doff, doff + 1, s);
        void* tmp; CK(cudaMalloc(&tmp, bytes));
        CK(cudaStreamSynchronize(s));
        cudaEventRecord(a, s);
        CK(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, db, n2, segs, doff, doff + 1, s));
        cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("segmented sort %d keys (no big segments): %.2f ms\n", n2, ms);
        CK(cudaFree(tmp));
    }
    // global radix sort of n 64-bit keys over 48 bits for reference
    {
        uint64_t *g1, *g2; CK(cudaMalloc(&g1, 8 * (int64_t)n)); CK(cudaMalloc(&g2, 8 * (int64_t)n));
        CK(cudaMemset(g1, 1, 8 * (int64_t)n));
        cub::DoubleBuffer<uint64_t> db(g1, g2);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, n, 0, 48, s);
        void* tmp; CK(cudaMalloc(&tmp, bytes));
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a, s);
            CK(cub::DeviceRadixSort::SortKeys(tmp, bytes, db, n, 0, 48, s));
            cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("global radix sort %lld u64 keys, 48 bits: %.2f ms\n", (long long)n, ms);
        }
    }
    return 0;
}
