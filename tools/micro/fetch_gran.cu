// DRAM fetch granularity of a random 8-byte gather on this GPU.
//
// The config-5 best-move round moves ~105 bytes of DRAM traffic per scanned
// entry for one 8-byte (label, mass) gather (profiles/r02_traffic_cfg5.json):
// how many bytes does ONE L2 miss of a random 8-byte load pull from DRAM, and
// does a load qualifier change it?  Each variant gathers u64 words at hashed
// positions of a 2 GB array (every load a miss) with U loads in flight per
// thread.  Run under
//   ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none
// and divide the kernel's DRAM bytes by its gather count (printed), or alone
// for the G gathers/s of each variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fetch_gran tools/micro/fetch_gran.cu
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int V>
__device__ __forceinline__ unsigned long long ld(const unsigned long long* p) {
    unsigned long long r;
    if constexpr (V == 0) asm volatile("ld.global.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 1) asm volatile("ld.global.L2::64B.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 2) asm volatile("ld.global.L2::128B.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 3) asm volatile("ld.global.L2::256B.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 4) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 5) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 6) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 7) asm volatile("ld.relaxed.gpu.global.L2::64B.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 8) asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(r) : "l"(p));
    if constexpr (V == 9) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}

template <int V, int U>
__global__ void __launch_bounds__(256) k_gather(const unsigned long long* __restrict__ A, uint64_t nwords,
                                                int64_t per_thread, uint64_t salt, unsigned long long* out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long acc = 0;
    for (int64_t i = 0; i < per_thread; i += U) {
        unsigned long long v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint64_t h = mix((t * (uint64_t)per_thread + (uint64_t)(i + j)) ^ salt);
            v[j] = ld<V>(A + (uint64_t)(((unsigned __int128)h * nwords) >> 64));
        }
#pragma unroll
        for (int j = 0; j < U; ++j) acc += v[j];
    }
    if (acc == 0x123456789ull) *out = acc;
}

template <int V>
int run(const char* name, const unsigned long long* A, uint64_t nwords, unsigned long long* out) {
    const int grid = 148 * 8, per = 2048;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_gather<V, 8><<<grid, 256>>>(A, nwords, per, 1, out);  // warm-up
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0));
        k_gather<V, 8><<<grid, 256>>>(A, nwords, per, 2 + r, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    const double g = (double)grid * 256 * per;
    printf("{\"variant\": \"%s\", \"gathers\": %.0f, \"ms\": %.3f, \"G_per_s\": %.2f}\n", name, g, best, g / best / 1e6);
    return 0;
}

int main(int argc, char** argv) {
    const uint64_t bytes = (argc > 1 ? strtoull(argv[1], nullptr, 0) : 2048ull) << 20;
    const uint64_t nwords = bytes / 8;
    unsigned long long *A, *out;
    CK(cudaMalloc(&A, bytes));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(A, 1, bytes));
    printf("array %.0f MB\n", bytes / 1048576.0);
    if (run<0>("ld.global", A, nwords, out)) return 1;
    if (run<1>("ld.global.L2::64B", A, nwords, out)) return 1;
    if (run<2>("ld.global.L2::128B", A, nwords, out)) return 1;
    if (run<3>("ld.global.L2::256B", A, nwords, out)) return 1;
    if (run<4>("ld.relaxed.gpu.global", A, nwords, out)) return 1;
    if (run<5>("ld.global.nc", A, nwords, out)) return 1;
    if (run<6>("ld.global.nc.L1::no_allocate.L2::64B", A, nwords, out)) return 1;
    if (run<7>("ld.relaxed.gpu.global.L2::64B", A, nwords, out)) return 1;
    if (run<8>("ld.global.cv", A, nwords, out)) return 1;
    if (run<9>("ld.global.cg", A, nwords, out)) return 1;
    return 0;
}
