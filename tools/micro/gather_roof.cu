// Gather "roofline" of the best-move access pattern on this GPU.
//
// The best-move round is not bandwidth bound (DRAM 5-9% of peak): every edge
// is a chain index -> label gather -> shared-table insert, and every distinct
// neighbour cluster a mass gather.  This measures what the hardware does for
// those access patterns alone, with the config-4 array sizes, so the kernel
// can be compared against the right ceiling:
//   stream   : coalesced int32 read of an index array (HBM bandwidth)
//   gather1  : idx[e] (streamed) -> C[idx[e]] (random 4-byte gather), C of
//              |C| bytes; reported as G gathers/s
//   chain2   : idx[e] -> C[idx[e]] -> K[C[...]]  (two dependent gathers,
//              the label -> mass chain of a singleton start)
//   smem_ins : per-warp 512-slot open-addressing table, CAS insert of
//              random 32-bit keys (+ RED of a count) -- the table step alone
// All timings with CUDA events, best of 5, after a warm-up; UNROLL loads in
// flight per thread as in the kernels.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_roof tools/micro/gather_roof.cu && /tmp/gather_roof
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (uint32_t)(z ^ (z >> 31));
}
__global__ void k_fill_idx(int32_t* idx, int64_t m, uint32_t range) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        idx[i] = (int32_t)(((uint64_t)mix(i) * range) >> 32);
}
__global__ void k_fill_iota(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}
__global__ void k_stream(const int32_t* __restrict__ idx, int64_t m, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        acc += (uint32_t)__ldg(idx + i);
    if (acc == 0x123456789ull) *out = acc;
}
template <int U>
__global__ void k_gather1(const int32_t* __restrict__ idx, int64_t m, const int32_t* __restrict__ C,
                          unsigned long long* out) {
    unsigned long long acc = 0;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < m; i0 += T * U) {
        int32_t u[U];
#pragma unroll
        for (int j = 0; j < U; ++j) u[j] = i0 + j * T < m ? __ldg(idx + i0 + j * T) : 0;
#pragma unroll
        for (int j = 0; j < U; ++j) u[j] = __ldg(C + u[j]);
#pragma unroll
        for (int j = 0; j < U; ++j) acc += (uint32_t)u[j];
    }
    if (acc == 0x123456789ull) *out = acc;
}
template <int U>
__global__ void k_chain2(const int32_t* __restrict__ idx, int64_t m, const int32_t* __restrict__ C,
                         const uint32_t* __restrict__ K, unsigned long long* out) {
    unsigned long long acc = 0;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < m; i0 += T * U) {
        int32_t u[U];
#pragma unroll
        for (int j = 0; j < U; ++j) u[j] = i0 + j * T < m ? __ldg(idx + i0 + j * T) : 0;
#pragma unroll
        for (int j = 0; j < U; ++j) u[j] = __ldg(C + u[j]);
#pragma unroll
        for (int j = 0; j < U; ++j) acc += __ldg(K + u[j]);
    }
    if (acc == 0x123456789ull) *out = acc;
}
// per-warp 512-slot tables, 8 warps per CTA (cleared every 256 inserts:
// load <= 0.5)
__global__ void __launch_bounds__(256) k_smem_ins(int64_t per_warp, unsigned long long* out) {
    __shared__ int32_t keys[8][512];
    __shared__ uint32_t cnts[8][512];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = lane; q < 512; q += 32) { keys[w][q] = -1; cnts[w][q] = 0; }
    __syncwarp();
    const uint64_t base = ((uint64_t)blockIdx.x * 8 + w) << 32;
    unsigned long long acc = 0;
    for (int64_t r = 0; r < per_warp; r += 256) {
        for (int q = lane; q < 256; q += 32) {
            const int32_t x = (int32_t)(mix(base + r + q) & 0x7fffffff);
            uint32_t h = (uint32_t)(((uint64_t)((uint32_t)x * 0x9E3779B1u) * 512u) >> 32);
            while (true) {
                const int32_t prev = atomicCAS(&keys[w][h], -1, x);
                if (prev == -1 || prev == x) break;
                h = (h + 1) & 511;
            }
            atomicAdd(&cnts[w][h], 1u);
        }
        __syncwarp();
        for (int q = lane; q < 512; q += 32) { acc += cnts[w][q]; keys[w][q] = -1; cnts[w][q] = 0; }
        __syncwarp();
    }
    if (acc == 0x123456789ull) *out = acc;
}

template <class F>
float best_ms(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t m = 521000000;  // config-4 directed entries
    int32_t* idx;
    unsigned long long* out;
    CK(cudaMalloc(&idx, sizeof(int32_t) * m));
    CK(cudaMalloc(&out, 8));
    const unsigned grid = sms * 8, block = 256;
    const float ts = best_ms([&] { k_stream<<<grid, block>>>(idx, m, out); });
    printf("{\"stream_GBps\": %.1f", 4.0 * m / ts / 1e6);
    for (int64_t n : {2000000LL, 16777216LL, 33554432LL, 268435456LL}) {
        int32_t* C;
        uint32_t* K;
        CK(cudaMalloc(&C, sizeof(int32_t) * n));
        CK(cudaMalloc(&K, sizeof(uint32_t) * n));
        k_fill_idx<<<grid, block>>>(idx, m, (uint32_t)n);
        k_fill_iota<<<grid, block>>>(C, n);
        k_fill_iota<<<grid, block>>>((int32_t*)K, n);
        CK(cudaDeviceSynchronize());
        const float t1 = best_ms([&] { k_gather1<8><<<grid, block>>>(idx, m, C, out); });
        const float t2 = best_ms([&] { k_chain2<8><<<grid, block>>>(idx, m, C, K, out); });
        printf(", \"n_%lld\": {\"array_MB\": %.0f, \"gather1_Gps\": %.1f, \"chain2_Gps\": %.1f}", (long long)n,
               4.0 * n / 1e6, m / t1 / 1e6, m / t2 / 1e6);
        cudaFree(C);
        cudaFree(K);
    }
    const int64_t per_warp = 1 << 16;
    const unsigned g2 = sms * 6;
    const float t3 = best_ms([&] { k_smem_ins<<<g2, 256>>>(per_warp, out); });
    printf(", \"smem_insert_Gps\": %.1f}\n", (double)g2 * 8 * per_warp / t3 / 1e6);
    return 0;
}
