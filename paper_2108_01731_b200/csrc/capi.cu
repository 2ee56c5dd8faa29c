// capi.cu -- the extern "C" boundary declared in include/lcc_b200.h.
// Exceptions never cross it: each call returns an lcc_status and leaves a
// one-line message in a thread-local buffer (lcc_last_error()).
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.cuh"

namespace lcc {
long long& launch_counter() {
    static long long c = 0;  // diagnostics only (bench.py "gpu_launches")
    return c;
}
}  // namespace lcc

namespace {
thread_local std::string g_err;

// Library scratch stays mapped inside a call (memory.cu: an arena of mapped
// virtual memory for blocks >= 1 MB, the stream-ordered pool for small
// ones): fresh device memory costs ~6 ms per GB to map on B200 (measured:
// 16 GB 93 ms, reused 2.3 ms), more than the contraction that needs it.
// When a call returns both are cut back to pool_keep() (default 64 GB,
// LCC_POOL_KEEP_GB); lcc_release_memory() hands everything back on request.
uint64_t pool_keep() {
    static uint64_t keep = [] {
        const char* e = getenv("LCC_POOL_KEEP_GB");  // tuning / memory-tight callers
        return (e ? (uint64_t)atoll(e) : 64ull) << 30;
    }();
    return keep;
}

cudaMemPool_t pool_once() {
    static bool done[64] = {false};
    static cudaMemPool_t pools[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!done[dev]) {
        if (cudaDeviceGetDefaultMemPool(&pools[dev], dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        } else {
            pools[dev] = nullptr;
        }
        done[dev] = true;
    }
    return pools[dev];
}

struct TrimOnExit {
    cudaMemPool_t pool;
    ~TrimOnExit() {
        lcc::trim_cache(pool_keep(), nullptr);
        if (pool) cudaMemPoolTrimTo(pool, pool_keep());
    }
};

template <class F>
lcc_status guard(F&& f) {
    try {
        TrimOnExit trim{pool_once()};
        f();
        g_err.clear();
        return LCC_OK;
    } catch (const lcc::Invalid& e) {
        g_err = e.what();
        return LCC_ERR_INVALID;
    } catch (const lcc::OutOfMemory& e) {
        g_err = e.what();
        return LCC_ERR_OOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LCC_ERR_CUDA;
    }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void check_graph(const lcc_graph* g) {
    LCC_REQUIRE(g != nullptr, "graph is NULL");
    LCC_REQUIRE(g->n >= 0, "negative vertex count");
    LCC_REQUIRE(g->nnz >= 0, "negative entry count");
    LCC_REQUIRE(g->n == 0 || g->indptr != nullptr, "indptr is NULL");
    LCC_REQUIRE(g->nnz == 0 || g->indices != nullptr, "indices is NULL");
    LCC_REQUIRE(g->weights == nullptr || g->wtype == LCC_W_F32 || g->wtype == LCC_W_F64 || g->wtype == LCC_W_U32,
                "unknown weight dtype");
}

void check_params(const lcc_params* p) {
    LCC_REQUIRE(p != nullptr, "params is NULL");
    LCC_REQUIRE(p->lambda >= 0.0 && p->lambda < 1.0, "lambda must lie in [0, 1)");
}

lcc::Options to_opts(const lcc_options* o) {
    lcc::Options r;
    if (o) {
        LCC_REQUIRE(o->schedule == LCC_SYNC || o->schedule == LCC_ASYNC, "unknown schedule");
        LCC_REQUIRE(o->frontier_policy >= 0 && o->frontier_policy <= 2, "unknown frontier policy");
        LCC_REQUIRE(o->num_iter >= 1, "num_iter must be >= 1");
        r.schedule = o->schedule;
        r.policy = o->frontier_policy;
        r.refine = o->refine;
        r.num_iter = o->num_iter;
        r.deg_threshold = o->degree_threshold;
        r.async_chunks = o->async_chunks > 0 ? o->async_chunks : 0;  // 0 = auto
        r.seed = o->seed;
    }
    return r;
}
}  // namespace

extern "C" {

int lcc_abi_version(void) { return LCC_ABI_VERSION; }

lcc_status lcc_release_memory(void) {
    return guard([&] {
        cudaMemPool_t pool = pool_once();
        lcc::trim_cache(0, nullptr);
        LCC_CUDA(cudaDeviceSynchronize());
        if (pool) LCC_CUDA(cudaMemPoolTrimTo(pool, 0));
    });
}
int64_t lcc_kernel_launches(void) { return lcc::launch_counter(); }
const char* lcc_last_error(void) { return g_err.c_str(); }

lcc_status lcc_best_moves_round(const lcc_graph* g, const lcc_params* p, int32_t* C, double* K,
                                const int32_t* frontier, int64_t n_frontier, int32_t schedule,
                                int32_t degree_threshold, int32_t async_chunks, int32_t* D, uint8_t* moved,
                                uint8_t* nbr_mark, int64_t* moved_count, lcc_stats* stats, void* stream) {
    return guard([&] {
        check_graph(g);
        check_params(p);
        LCC_REQUIRE(C && K && moved, "C, K and moved are required");
        LCC_REQUIRE(n_frontier >= 0 && n_frontier <= g->n, "frontier size out of range");
        // frontier == NULL means V' = V only with n_frontier == n; an empty
        // frontier (n_frontier == 0) is an empty round: D = C, no movers
        LCC_REQUIRE(frontier || n_frontier == 0 || n_frontier == g->n,
                    "frontier == NULL needs n_frontier == n (all vertices) or 0 (empty)");
        lcc::RoundStats rs;
        const int64_t cnt = lcc::best_moves_round(*g, p->k, p->lambda, C, K, frontier, n_frontier, schedule,
                                                  degree_threshold, async_chunks > 0 ? async_chunks : 0, D, moved,
                                                  nbr_mark, &rs, S(stream));
        if (moved_count) *moved_count = cnt;
        if (stats) {
            stats->rounds += 1;
            stats->vertices += rs.vertices;
            stats->edges_scanned += rs.edges;
            stats->moves += rs.moved;
            stats->ms_kernels += rs.ms_kernels;
            stats->kernel_launches += rs.launches;
        }
    });
}

lcc_status lcc_frontier_from_mask(int64_t n, const uint8_t* mark, int32_t* frontier, int64_t* n_frontier,
                                  void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0, "negative vertex count");
        LCC_REQUIRE(n == 0 || (mark && frontier), "NULL buffer");
        const int64_t h = lcc::frontier_from_mask(n, mark, frontier, S(stream));
        if (n_frontier) *n_frontier = h;
    });
}

lcc_status lcc_apply_moves(int64_t n, const int32_t* labels_in, int64_t label_range, const double* k, int32_t* C,
                           double* K, void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0 && label_range >= n, "label_range must be >= n");
        LCC_REQUIRE(n == 0 || (labels_in && C && K), "NULL buffer");
        lcc::apply_moves(n, labels_in, label_range, k, C, K, S(stream));
    });
}

lcc_status lcc_compute_frontier(const lcc_graph* g, int32_t policy, const uint8_t* moved, const int32_t* C_old,
                                const int32_t* C_new, int32_t* frontier, int64_t* n_frontier, void* stream) {
    return guard([&] {
        check_graph(g);
        LCC_REQUIRE(moved && frontier, "NULL buffer");
        LCC_REQUIRE(policy != LCC_FRONTIER_CLUSTER_NBRS || (C_old && C_new), "cluster-neighbours needs both labelings");
        const int64_t nf = lcc::compute_frontier(*g, policy, moved, C_old, C_new, frontier, S(stream));
        if (n_frontier) *n_frontier = nf;
    });
}

lcc_status lcc_par_best_moves(const lcc_graph* g, const lcc_params* p, const lcc_options* opts, int32_t* C,
                              double* K, int32_t* any_moved, lcc_stats* stats, void* stream) {
    return guard([&] {
        check_graph(g);
        check_params(p);
        LCC_REQUIRE(g->n == 0 || (C && K), "NULL buffer");
        const bool a = lcc::par_best_moves(*g, p->k, p->lambda, to_opts(opts), true, C, K, stats, S(stream));
        if (any_moved) *any_moved = a ? 1 : 0;
    });
}

lcc_status lcc_par_compress(const lcc_graph* g, const lcc_params* p, const int32_t* C, const double* K,
                            int32_t* mapping, double* ck, int64_t* cindptr, int32_t* cindices, double* cweights,
                            int64_t* cn, int64_t* cnnz, double* internal_offset, double* ctotal_weight,
                            void* stream) {
    return guard([&] {
        check_graph(g);
        check_params(p);
        LCC_REQUIRE(g->n == 0 || (C && K && mapping && ck && cindptr), "NULL buffer");
        LCC_REQUIRE(g->nnz == 0 || (cindices && cweights), "NULL buffer");
        const lcc::Coarse r = lcc::compress(*g, p->k, p->lambda, C, K, mapping, ck, S(stream));
        LCC_CUDA(cudaMemcpyAsync(cindptr, r.indptr.get(), sizeof(int64_t) * (r.cn + 1), cudaMemcpyDeviceToDevice,
                                 S(stream)));
        if (r.cnnz) {
            LCC_CUDA(cudaMemcpyAsync(cindices, r.indices.get(), sizeof(int32_t) * r.cnnz, cudaMemcpyDeviceToDevice,
                                     S(stream)));
            if (r.integral) lcc::widen_u32(r.wi.get(), cweights, r.cnnz, S(stream));
            else LCC_CUDA(cudaMemcpyAsync(cweights, r.w.get(), sizeof(double) * r.cnnz, cudaMemcpyDeviceToDevice,
                                          S(stream)));
        }
        if (cn) *cn = r.cn;
        if (cnnz) *cnnz = r.cnnz;
        if (internal_offset) *internal_offset = r.internal_offset;
        if (ctotal_weight) *ctotal_weight = r.total_weight;
    });
}

lcc_status lcc_par_flatten(int64_t n, const int32_t* mapping, const int32_t* Cc, const double* k, int32_t* C,
                           double* K, void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0, "negative vertex count");
        LCC_REQUIRE(n == 0 || (mapping && Cc && C && K), "NULL buffer");
        lcc::flatten(n, mapping, Cc, k, C, K, S(stream));
    });
}

lcc_status lcc_cc_objective(const lcc_graph* g, const lcc_params* p, const int32_t* C, double* objective,
                            void* stream) {
    return guard([&] {
        check_graph(g);
        check_params(p);
        LCC_REQUIRE(objective, "objective is NULL");
        LCC_REQUIRE(g->n == 0 || C, "C is NULL");
        *objective = lcc::cc_objective(*g, p->k, p->lambda, C, S(stream));
    });
}

lcc_status lcc_weighted_degrees(const lcc_graph* g, double* k, void* stream) {
    return guard([&] {
        check_graph(g);
        LCC_REQUIRE(g->n == 0 || k, "k is NULL");
        lcc::weighted_degrees(*g, k, S(stream));
    });
}

lcc_status lcc_parallel_cc(const lcc_graph* g, const lcc_params* p, const lcc_options* opts, int32_t* C_out,
                           lcc_stats* stats, void* stream) {
    return guard([&] {
        check_graph(g);
        check_params(p);
        LCC_REQUIRE(g->n == 0 || C_out, "C_out is NULL");
        lcc::parallel_cc(*g, p->k, p->lambda, to_opts(opts), C_out, stats, S(stream));
    });
}

lcc_status lcc_gen_rmat(int32_t scale, int64_t samples, double a, double b, double c, uint64_t seed, int64_t* indptr,
                        int32_t* indices, int64_t* nnz, void* stream) {
    return guard([&] {
        LCC_REQUIRE(indptr && (samples == 0 || indices), "NULL buffer");
        const int64_t r = lcc::gen_rmat(scale, samples, a, b, c, seed, indptr, indices, S(stream));
        if (nnz) *nnz = r;
    });
}

lcc_status lcc_gen_powerlaw_communities(int64_t n, int64_t samples, double mu, const double* vw_prefix,
                                        const int64_t* cstart, const double* cw_prefix, int64_t n_communities,
                                        uint64_t seed, int64_t* indptr, int32_t* indices, int64_t* nnz,
                                        void* stream) {
    return guard([&] {
        LCC_REQUIRE(vw_prefix && cstart && cw_prefix && indptr && (samples == 0 || indices), "NULL buffer");
        const int64_t r = lcc::gen_powerlaw_communities(n, samples, mu, vw_prefix, cstart, cw_prefix, n_communities,
                                                        seed, indptr, indices, S(stream));
        if (nnz) *nnz = r;
    });
}

lcc_status lcc_build_csr_from_pairs(int64_t n, int64_t n_pairs, const int32_t* u, const int32_t* v, int64_t* indptr,
                                    int32_t* indices, int64_t* nnz, void* stream) {
    return guard([&] {
        LCC_REQUIRE(indptr && (n_pairs == 0 || (u && v && indices)), "NULL buffer");
        const int64_t r = lcc::build_csr_from_pairs(n, n_pairs, u, v, indptr, indices, S(stream));
        if (nnz) *nnz = r;
    });
}

lcc_status lcc_edge_id_range(int64_t n_edges, const int64_t* u, const int64_t* v, int64_t* min_id, int64_t* max_id,
                             void* stream) {
    return guard([&] {
        LCC_REQUIRE(n_edges >= 0, "negative edge count");
        LCC_REQUIRE(n_edges == 0 || (u && v), "NULL buffer");
        LCC_REQUIRE(min_id && max_id, "NULL output");
        lcc::edge_id_range(n_edges, u, v, min_id, max_id, S(stream));
    });
}

lcc_status lcc_build_graph(int64_t n, int64_t n_edges, const int64_t* u, const int64_t* v, const double* w,
                           int64_t* indptr, int32_t* indices, double* weights, int64_t* m, double* total_weight,
                           int32_t* unit_weights, void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0 && n_edges >= 0, "negative size");
        LCC_REQUIRE(indptr && (n_edges == 0 || (u && v && indices && weights)), "NULL buffer");
        const lcc::BuiltGraph b = lcc::build_graph(n, n_edges, u, v, w, indptr, indices, weights, S(stream));
        if (m) *m = b.m;
        if (total_weight) *total_weight = b.total_weight;
        if (unit_weights) *unit_weights = b.unit ? 1 : 0;
    });
}

lcc_status lcc_coo_merge(int64_t n, int64_t nnz, const int32_t* rows, const int32_t* cols, const void* w,
                         int32_t wtype, int64_t* indptr, int32_t* indices, void* w_out, int64_t* nnz_out,
                         void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0 && nnz >= 0, "negative size");
        LCC_REQUIRE(indptr && (nnz == 0 || (rows && cols && indices && w_out)), "NULL buffer");
        LCC_REQUIRE(wtype == LCC_W_NONE || wtype == LCC_W_U32 || wtype == LCC_W_F64,
                    "coo_merge takes LCC_W_NONE / LCC_W_U32 (uint32 sums) or LCC_W_F64 (double sums)");
        LCC_REQUIRE(wtype == LCC_W_NONE || nnz == 0 || w, "weights are NULL");
        int64_t r;
        if (wtype == LCC_W_F64)
            r = lcc::coo_merge<double>(n, nnz, rows, cols, static_cast<const double*>(w), indptr, indices,
                                       static_cast<double*>(w_out), S(stream));
        else
            r = lcc::coo_merge<uint32_t>(n, nnz, rows, cols,
                                         wtype == LCC_W_NONE ? nullptr : static_cast<const uint32_t*>(w), indptr,
                                         indices, static_cast<uint32_t*>(w_out), S(stream));
        if (nnz_out) *nnz_out = r;
    });
}

lcc_status lcc_partition_scores(int64_t n, const int32_t* a, const int32_t* b, double* ari, double* nmi,
                                void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0, "negative length");
        LCC_REQUIRE(n == 0 || (a && b), "NULL labels");
        LCC_REQUIRE(ari && nmi, "NULL output");
        lcc::partition_scores(n, a, b, ari, nmi, S(stream));
    });
}

lcc_status lcc_avg_precision_recall(int64_t n, const int32_t* C, int64_t n_comm, const int64_t* offsets,
                                    const int32_t* members, double* precision, double* recall, void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0, "negative vertex count");
        LCC_REQUIRE(n_comm > 0, "empty ground truth");
        LCC_REQUIRE(offsets && members && (n == 0 || C), "NULL buffer");
        LCC_REQUIRE(precision && recall, "NULL output");
        lcc::avg_precision_recall(n, C, n_comm, offsets, members, precision, recall, S(stream));
    });
}

lcc_status lcc_cluster_stats(int64_t n, const int32_t* C, int64_t* num_clusters, int64_t* min_size, int64_t* max_size,
                             double* mean_size, void* stream) {
    return guard([&] {
        LCC_REQUIRE(n >= 0, "negative vertex count");
        LCC_REQUIRE(n == 0 || C, "C is NULL");
        LCC_REQUIRE(num_clusters && min_size && max_size && mean_size, "NULL output");
        lcc::cluster_stats(n, C, num_clusters, min_size, max_size, mean_size, S(stream));
    });
}

}  // extern "C"
