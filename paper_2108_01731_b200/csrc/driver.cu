// driver.cu -- par_best_moves and the multi-level parallel_cc driver
// (Alg. 1, lines 1-19).
//
// Native host orchestration: one best-move iteration = bin partition +
// best-move kernels + (sync) apply / (async) reconcile + frontier, with one
// host read of the mover count per iteration for the early exit (Alg. 1
// line 9).  Levels are kept on an explicit stack so refinement can revisit
// them while unwinding.
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <utility>
#include <vector>

#include "internal.cuh"

#ifndef LCC_PMIN_DEFAULT
#define LCC_PMIN_DEFAULT 1
#endif

namespace lcc {

namespace {
struct EventTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    explicit EventTimer(cudaStream_t st) : s(st) {
        LCC_CUDA(cudaEventCreate(&a));
        LCC_CUDA(cudaEventCreate(&b));
        LCC_CUDA(cudaEventRecord(a, s));
    }
    float stop() {
        LCC_CUDA(cudaEventRecord(b, s));
        LCC_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        LCC_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
    ~EventTimer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

// LCC_TRACE_MOVERS=1 (diagnostic): classify an async iteration's movers.
//   st[0] movers, st[1] moved in the previous iteration too, st[2] alone in
//   the cluster they joined (mass == k_v), st[3] joined a fresh singleton id,
//   st[4] sum of their degrees
__global__ void k_mover_stats(int64_t n, const int64_t* __restrict__ indptr, const double* __restrict__ k,
                              const uint8_t* __restrict__ moved, const uint8_t* __restrict__ prev,
                              const int32_t* __restrict__ D, const double* __restrict__ K2,
                              unsigned long long* st) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || !moved[v]) return;
    const double kv = k ? k[v] : 1.0;
    const int32_t x = D[v];
    atomicAdd(st + 0, 1ull);
    if (prev && prev[v]) atomicAdd(st + 1, 1ull);
    if (K2[x] == kv) atomicAdd(st + 2, 1ull);
    if (x >= n) atomicAdd(st + 3, 1ull);
    atomicAdd(st + 4, (unsigned long long)(indptr[v + 1] - indptr[v]));
}
}  // namespace

int async_min_subrounds() {
    const char* e = getenv("LCC_PMIN");  // tuning knob
    return e ? std::max(1, std::min(64, atoi(e))) : LCC_PMIN_DEFAULT;
}

bool par_best_moves(const lcc_graph& g, const double* k, double lam, const Options& o, bool first_level, int32_t* C,
                    double* K, lcc_stats* st, cudaStream_t s) {
    LCC_REQUIRE(o.num_iter >= 1, "num_iter must be >= 1");
    const int64_t n = g.n;
    if (n == 0) return false;
    const bool as = o.schedule == LCC_ASYNC;
    Buf<int32_t> D(n, s), Cnext(n, s), F(n, s);
    Buf<uint8_t> moved(n, s);
    // VertexNeighbors frontier fused into the round (nbr_mark), else computed after
    const bool fused = o.policy == LCC_FRONTIER_VERTEX_NBRS;
    Buf<uint8_t> mark;
    if (fused && o.num_iter > 1) mark.alloc(n, s);
    // async damping needs last iteration's movers: two flag arrays, swapped
    const char* ed = getenv("LCC_DAMP");
    const bool damping = as && fused && o.num_iter > 1 && !(ed && ed[0] == '0');
    Buf<uint8_t> moved2;
    if (damping) moved2.alloc(n, s);
    uint8_t* mv_cur = moved.get();
    uint8_t* mv_prev = nullptr;
    Buf<double> K2;
    if (as) K2.alloc(2 * n, s);
    int32_t* cur = C;
    int32_t* nxt = Cnext.get();
    const int32_t* frontier = nullptr;  // V' <- V
    int64_t nF = n;
    bool any = false;
    for (int it = 0; it < o.num_iter; ++it) {
        if (frontier && nF == 0) break;
        RoundStats rs;
        int64_t cnt;
        // Asynchronous levels run their last iteration like the others, with the fused
        // marks and the damping that rides on them: without them it was the slowest
        // iteration of its level (config 5 level 0: 96-100 ms against 73).
        // LCC_LASTMARK=0: no marks in the last iteration; 2: marks, no damping.
        static const int lastmark_mode = getenv("LCC_LASTMARK") ? atoi(getenv("LCC_LASTMARK")) : 1;  // 2: marks, no damping
        const bool lastmark = lastmark_mode > 0;
        uint8_t* mk = (fused && (it + 1 < o.num_iter || (as && lastmark && mark.get()))) ? mark.get() : nullptr;
        EventTimer tm(s);
        if (!as) {
            cnt = best_moves_round(g, k, lam, cur, K, frontier, nF, LCC_SYNC, o.deg_threshold, 1, D.get(),
                                   mv_cur, mk, &rs, s);
        } else {
            AsyncDamp damp;
            damp.prev_moved = damping && !(lastmark_mode == 2 && it + 1 == o.num_iter) ? mv_prev : nullptr;
            // seeded, recorded RNG: the damping coin of iteration
            // `it` is a hash of (seed, it); the default seed 0 keeps round 1's salts
            damp.salt = 0x85EBCA6Bu * (uint32_t)(it + 1) ^ (uint32_t)(o.seed * 0x9E3779B97F4A7C15ull >> 32);
            LCC_CUDA(cudaMemcpyAsync(D.get(), cur, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
            LCC_CUDA(cudaMemcpyAsync(K2.get(), K, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
            LCC_CUDA(cudaMemsetAsync(K2.get() + n, 0, sizeof(double) * n, s));
            cnt = best_moves_round(g, k, lam, D.get(), K2.get(), frontier, nF, LCC_ASYNC, o.deg_threshold,
                                   o.async_chunks > 0 ? o.async_chunks
                                   : (first_level && it == 0) ? 0 : -async_min_subrounds(),
                                   nullptr, mv_cur, mk, &rs, s, &damp);
        }
        const float ms = tm.stop();
        if (getenv("LCC_TRACE"))
            fprintf(stderr, "[lcc]     iter %d frontier %lld edges %lld movers %lld launches %lld %.2f ms (kernels %.2f)\n",
                    it, (long long)nF, (long long)rs.edges, (long long)cnt, (long long)rs.launches, ms, rs.ms_kernels);
        if (st) {
            st->rounds += 1;
            st->vertices += rs.vertices;
            st->edges_scanned += rs.edges;
            st->moves += rs.moved;
            st->ms_best_moves += ms;
            st->ms_kernels += rs.ms_kernels;
            st->kernel_launches += rs.launches;
        }
        if (as && cnt && getenv("LCC_TRACE_MOVERS")) {
            Buf<unsigned long long> ms5(5, s);
            LCC_CUDA(cudaMemsetAsync(ms5.get(), 0, 5 * sizeof(unsigned long long), s));
            k_mover_stats<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, g.indptr, k, mv_cur, damping ? mv_prev : nullptr,
                                                                      D.get(), K2.get(), ms5.get());
            unsigned long long h[5];
            LCC_CUDA(cudaMemcpyAsync(h, ms5.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaStreamSynchronize(s));
            fprintf(stderr, "[lcc]       movers %llu: repeat %llu, alone in target %llu, fresh %llu, mean degree %.1f\n", h[0],
                    h[1], h[2], h[3], h[0] ? (double)h[4] / (double)h[0] : 0.0);
        }
        if (cnt == 0) break;  // Alg. 1 line 9
        any = true;
        apply_moves(n, D.get(), 2 * n, k, nxt, K, s);  // sync apply / async reconcile
        if (it + 1 < o.num_iter) {  // the next frontier is only needed by a next iteration
            nF = mk ? frontier_from_mask(n, mk, F.get(), s)
                    : compute_frontier(g, o.policy, mv_cur, cur, nxt, F.get(), s);
            frontier = F.get();
        }
        std::swap(cur, nxt);
        if (damping) {
            mv_prev = mv_cur;
            mv_cur = mv_cur == moved.get() ? moved2.get() : moved.get();
        }
    }
    if (cur != C) LCC_CUDA(cudaMemcpyAsync(C, cur, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    return any;
}

namespace {
// MemAvailable of the host (bytes), or 0 if unknown
size_t host_available() {
    FILE* f = fopen("/proc/meminfo", "r");
    if (!f) return 0;
    char line[256];
    size_t kb = 0;
    while (fgets(line, sizeof(line), f)) {
        if (sscanf(line, "MemAvailable: %zu kB", &kb) == 1) break;
    }
    fclose(f);
    return kb * 1024;
}

// A coarse level owned by the driver.  Levels that are only needed again
// while unwinding can be parked in pinned host memory when the next
// contraction would not fit (config 5: every level of a 1.8B-edge graph is
// ~24 GB and the levels shrink slowly), then restored for their refinement.
struct OwnedGraph {
    Buf<int64_t> indptr;
    Buf<int32_t> indices;
    Buf<double> w;
    Buf<uint32_t> wi;
    Buf<double> k;
    lcc_graph g{};
    char* host = nullptr;
    size_t wbytes() const { return g.wtype == LCC_W_U32 ? 4 : 8; }
    size_t bytes() const { return sizeof(int64_t) * (g.n + 1) + (sizeof(int32_t) + wbytes()) * g.nnz; }
    void park(cudaStream_t s) {
        if (host) return;
        // pinned pages cannot be swapped: keep 16 GB of the host free
        if (host_available() < bytes() + (16ull << 30))
            throw OutOfMemory("parallel_cc: the coarse levels exceed device memory and the host cannot hold "
                              "them either (" + std::to_string(bytes() >> 30) + " GB per level)");
        LCC_CUDA(cudaHostAlloc((void**)&host, std::max<size_t>(bytes(), 1), cudaHostAllocDefault));
        char* p = host;
        LCC_CUDA(cudaMemcpyAsync(p, g.indptr, sizeof(int64_t) * (g.n + 1), cudaMemcpyDeviceToHost, s));
        p += sizeof(int64_t) * (g.n + 1);
        if (g.nnz) {
            LCC_CUDA(cudaMemcpyAsync(p, g.indices, sizeof(int32_t) * g.nnz, cudaMemcpyDeviceToHost, s));
            p += sizeof(int32_t) * g.nnz;
            LCC_CUDA(cudaMemcpyAsync(p, g.weights, wbytes() * g.nnz, cudaMemcpyDeviceToHost, s));
        }
        LCC_CUDA(cudaStreamSynchronize(s));
        indptr.release();
        indices.release();
        w.release();
        wi.release();
        g.indptr = nullptr;
        g.indices = nullptr;
        g.weights = nullptr;
    }
    void unpark(cudaStream_t s) {
        if (!host) return;
        indptr.alloc(g.n + 1, s);
        indices.alloc(std::max<int64_t>(g.nnz, 1), s);
        const char* p = host;
        LCC_CUDA(cudaMemcpyAsync(indptr.get(), p, sizeof(int64_t) * (g.n + 1), cudaMemcpyHostToDevice, s));
        p += sizeof(int64_t) * (g.n + 1);
        void* wp;
        if (g.wtype == LCC_W_U32) { wi.alloc(std::max<int64_t>(g.nnz, 1), s); wp = wi.get(); }
        else { w.alloc(std::max<int64_t>(g.nnz, 1), s); wp = w.get(); }
        if (g.nnz) {
            LCC_CUDA(cudaMemcpyAsync(indices.get(), p, sizeof(int32_t) * g.nnz, cudaMemcpyHostToDevice, s));
            p += sizeof(int32_t) * g.nnz;
            LCC_CUDA(cudaMemcpyAsync(wp, p, wbytes() * g.nnz, cudaMemcpyHostToDevice, s));
        }
        LCC_CUDA(cudaStreamSynchronize(s));
        cudaFreeHost(host);
        host = nullptr;
        g.indptr = indptr.get();
        g.indices = indices.get();
        g.weights = wp;
    }
    ~OwnedGraph() {
        if (host) cudaFreeHost(host);
    }
};
struct Frame {
    int own;  // owner of this level's graph: -1 = the caller's graph, else owned[own]
    const double* k;
    Buf<int32_t> mapping;
};

// device bytes a contraction of g may take (keys x2, values x2, unique keys,
// outputs), vs what is free on the device plus what the library has cached
// sorted: entries going through keys + radix sort (all of them, or only the
// complex rows' on the mostly-singleton fast path); the coarse outputs are
// sized by nnz either way
bool contraction_fits(const lcc_graph& g, int64_t sorted) {
    const double vb = (g.weights && g.wtype != LCC_W_U32) ? 8.0 : 4.0;
    const double need = (double)sorted * (16.0 + 2.0 * vb + 8.0) + (double)g.nnz * (4.0 + vb) + (double)g.n * 64.0;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return true;
    double r, u;
    pool_gb(r, u);
    const double avail = (double)fr + (r - u) * 1073741824.0;  // unmapped + mapped-but-free
    return need < 0.9 * avail;
}
}  // namespace

void parallel_cc(const lcc_graph& g0, const double* k0, double lam, const Options& o, int32_t* C_out,
                 lcc_stats* st, cudaStream_t s) {
    EventTimer total(s);
    std::vector<std::unique_ptr<OwnedGraph>> owned;
    std::vector<Frame> stack;
    lcc_graph g = g0;
    const double* k = k0;
    Buf<int32_t> C;
    Buf<double> K;
    const bool trace = getenv("LCC_TRACE") != nullptr;  // per-phase device times on stderr
    while (true) {
        const int64_t n = g.n;
        EventTimer tl(s);
        C.alloc(std::max<int64_t>(n, 1), s);
        K.alloc(std::max<int64_t>(n, 1), s);
        fill_iota(C.get(), n, s);  // singletons
        fill_k(K.get(), k, n, s);
        if (st) st->levels += 1;
        const bool moved = par_best_moves(g, k, lam, o, stack.empty(), C.get(), K.get(), st, s);
        if (trace) {
            const float ms = tl.stop();
            double r, u;
            pool_gb(r, u);
            fprintf(stderr, "[lcc] level n=%lld nnz=%lld best_moves %.2f ms (pool %.1f/%.1f GB)\n", (long long)n,
                    (long long)g.nnz, ms, r, u);
        }
        if (!moved) break;  // Alg. 1 line 13
        // deeper levels first: park the finer owned levels on the host when
        // this contraction would not fit next to them
        // (LCC_PARK_ALWAYS=1 parks every finer level: tests of the parking path)
        const bool park_always = getenv("LCC_PARK_ALWAYS") && getenv("LCC_PARK_ALWAYS")[0] == '1';
        const int64_t sorted = owned.size() > 1 ? contraction_sort_entries(g, C.get(), s) : g.nnz;
        if (owned.size() > 1 && (park_always || !contraction_fits(g, sorted))) {
            for (size_t i = 0; i + 1 < owned.size(); ++i) {
                if (owned[i]->host) continue;
                owned[i]->park(s);
                if (trace) fprintf(stderr, "[lcc]   parked level %zu (%.1f GB) on the host\n", i + 1,
                                   owned[i]->bytes() / 1073741824.0);
                if (!park_always && contraction_fits(g, sorted)) break;
            }
        }
        EventTimer tc(s);
        // contraction straight into exact-size buffers
        Buf<int32_t> mapping(n, s);
        Buf<double> ck(n, s);
        Coarse cs = compress(g, k, lam, C.get(), K.get(), mapping.get(), ck.get(), s);
        if (trace) fprintf(stderr, "[lcc]   compress -> cn=%lld cnnz=%lld %.2f ms\n", (long long)cs.cn,
                           (long long)cs.cnnz, tc.stop());
        if (cs.cn == n) break;  // no size reduction
        C.release();
        K.release();
        auto og = std::make_unique<OwnedGraph>();
        og->indptr = std::move(cs.indptr);
        og->indices = std::move(cs.indices);
        og->w = std::move(cs.w);
        og->wi = std::move(cs.wi);
        og->k.alloc(std::max<int64_t>(cs.cn, 1), s);
        LCC_CUDA(cudaMemcpyAsync(og->k.get(), ck.get(), sizeof(double) * cs.cn, cudaMemcpyDeviceToDevice, s));
        og->g.n = cs.cn;
        og->g.nnz = cs.cnnz;
        og->g.indptr = og->indptr.get();
        og->g.indices = og->indices.get();
        // integer sums stay integers (LCC_W_U32: exact 32-bit table sums)
        og->g.weights = cs.integral ? (const void*)og->wi.get() : (const void*)og->w.get();
        og->g.wtype = cs.integral ? LCC_W_U32 : LCC_W_F64;
        og->g.total_weight = cs.total_weight;
        stack.push_back(Frame{(int)owned.size() - 1, k, std::move(mapping)});
        g = og->g;
        k = og->k.get();
        owned.push_back(std::move(og));
    }
    // unwind: flatten (+ refine) level by level (Alg. 1 lines 17-18)
    Buf<int32_t> Cres = std::move(C);
    for (auto it = stack.rbegin(); it != stack.rend(); ++it) {
        // the coarse level above this one is finished: free it
        owned[it->own + 1].reset();
        OwnedGraph* fine = it->own >= 0 ? owned[it->own].get() : nullptr;
        if (fine) fine->unpark(s);
        const lcc_graph& gf = fine ? fine->g : g0;
        const int64_t n = gf.n;
        EventTimer tu(s);
        Buf<int32_t> Cf(std::max<int64_t>(n, 1), s);
        Buf<double> Kf(std::max<int64_t>(n, 1), s);
        flatten(n, it->mapping.get(), Cres.get(), it->k, Cf.get(), Kf.get(), s);
        if (o.refine) par_best_moves(gf, it->k, lam, o, false, Cf.get(), Kf.get(), st, s);
        if (trace) fprintf(stderr, "[lcc] unwind n=%lld flatten+refine %.2f ms\n", (long long)n, tu.stop());
        Cres = std::move(Cf);
    }
    if (g0.n > 0)
        LCC_CUDA(cudaMemcpyAsync(C_out, Cres.get(), sizeof(int32_t) * g0.n, cudaMemcpyDeviceToDevice, s));
    const float ms = total.stop();
    if (st) st->ms_total += ms;
}

}  // namespace lcc
