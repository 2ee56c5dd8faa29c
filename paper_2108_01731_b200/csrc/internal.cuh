// internal.cuh -- C++ entry points shared between the translation units.
#pragma once
#include "common.cuh"

namespace lcc {

struct RoundStats {
    int64_t vertices = 0;
    int64_t edges = 0;
    int64_t moved = 0;
    int64_t n_small = 0, n_medium = 0, n_large = 0;
    double ms_kernels = 0.0;   // CUDA-event time of the best-move kernels
    int64_t launches = 0;      // best-move kernel launches
};

// best_moves.cu: one best-move iteration over `frontier` (nullptr = all).
//   sync : D <- C, D[v] <- target for movers, moved[] set; C/K untouched.
//   async: C and K (2n entries) updated live; D unused.
// mark (optional, n bytes): zeroed, then every neighbour of a mover is
// flagged -- the VertexNeighbors frontier fused into the round.
// Returns the number of movers (synchronises the stream once).
// damp (async, optional): vertices that moved in the previous iteration
// (prev_moved) defer a move with probability 1/2 -- they stay in the next
// frontier (via mark) and count as pending -- which breaks the 2-cycles
// (swaps) that simultaneous moves create.
struct AsyncDamp {
    const uint8_t* prev_moved = nullptr;
    uint32_t salt = 0;
};
int64_t best_moves_round(const lcc_graph& g, const double* k, double lam, int32_t* C, double* K,
                         const int32_t* frontier, int64_t nF, int schedule, int deg_threshold,
                         int async_chunks, int32_t* D, uint8_t* moved, uint8_t* mark, RoundStats* st,
                         cudaStream_t s, const AsyncDamp* damp = nullptr);

// apply.cu
void apply_moves(int64_t n, const int32_t* labels_in, int64_t label_range, const double* k,
                 int32_t* C, double* K, cudaStream_t s);
int64_t compute_frontier(const lcc_graph& g, int policy, const uint8_t* moved,
                         const int32_t* C_old, const int32_t* C_new, int32_t* frontier,
                         cudaStream_t s);
int64_t frontier_from_mask(int64_t n, const uint8_t* mark, int32_t* frontier, cudaStream_t s);
void fill_iota(int32_t* p, int64_t n, cudaStream_t s);
void fill_k(double* K, const double* k, int64_t n, cudaStream_t s);

// contract.cu
// The coarse CSR is returned in exact-size pool buffers (cindptr[cn+1],
// cindices[cnnz], cw[cnnz]); mapping[n] and ck[n] are caller buffers.
struct Coarse {
    int64_t cn = 0, cnnz = 0;
    double internal_offset = 0.0, total_weight = 0.0;
    Buf<int64_t> indptr;
    Buf<int32_t> indices;
    Buf<double> w;       // float sums (float/double inputs) ...
    Buf<uint32_t> wi;    // ... or exact integer sums (unweighted / uint32 inputs)
    bool integral = false;
};
Coarse compress(const lcc_graph& g, const double* k, double lam, const int32_t* C, const double* K,
                int32_t* mapping, double* ck, cudaStream_t s);
void widen_u32(const uint32_t* in, double* out, int64_t n, cudaStream_t s);
int64_t contraction_sort_entries(const lcc_graph& g, const int32_t* C, cudaStream_t s);
void flatten(int64_t n, const int32_t* mapping, const int32_t* Cc, const double* k, int32_t* C,
             double* K, cudaStream_t s);

// contract.cu: COO entries (row, col, w) -> CSR with duplicate (row, col)
// entries summed, rows sorted by col.  VT = uint32_t (counts / integer
// weights; vals == nullptr means 1 each) or double.  Returns the entry count.
template <class VT>
int64_t coo_merge(int64_t n, int64_t nnz, const int32_t* rows, const int32_t* cols, const VT* vals,
                  int64_t* indptr, int32_t* indices, VT* wout, cudaStream_t s);

// build.cu: build_graph (graph.py:79-164) on the device
struct BuiltGraph {
    int64_t m = 0, nnz = 0;
    double total_weight = 0.0;
    bool unit = true;  // every weight is 1 (the reference's unweighted graph)
};
void edge_id_range(int64_t ne, const int64_t* u, const int64_t* v, int64_t* lo, int64_t* hi, cudaStream_t s);
BuiltGraph build_graph(int64_t n, int64_t ne, const int64_t* u, const int64_t* v, const double* w, int64_t* indptr,
                       int32_t* indices, double* weights, cudaStream_t s);

// objective.cu
double cc_objective(const lcc_graph& g, const double* k, double lam, const int32_t* C,
                    cudaStream_t s);
void weighted_degrees(const lcc_graph& g, double* k, cudaStream_t s);

// gen.cu
int64_t build_csr_from_pairs(int64_t n, int64_t n_pairs, const int32_t* u, const int32_t* v,
                             int64_t* indptr, int32_t* indices, cudaStream_t s);
int64_t gen_rmat(int scale, int64_t samples, double a, double b, double c, uint64_t seed,
                 int64_t* indptr, int32_t* indices, cudaStream_t s);
int64_t gen_powerlaw_communities(int64_t n, int64_t samples, double mu, const double* vw_prefix,
                                 const int64_t* cstart, const double* cw_prefix, int64_t nc, uint64_t seed,
                                 int64_t* indptr, int32_t* indices, cudaStream_t s);

// eval.cu
void partition_scores(int64_t n, const int32_t* a, const int32_t* b, double* ari, double* nmi, cudaStream_t s);
void avg_precision_recall(int64_t n, const int32_t* C, int64_t nc, const int64_t* off, const int32_t* members,
                          double* precision, double* recall, cudaStream_t s);
void cluster_stats(int64_t n, const int32_t* C, int64_t* num, int64_t* mn, int64_t* mx, double* mean, cudaStream_t s);

// driver.cu
struct Options {
    int schedule = LCC_ASYNC, policy = LCC_FRONTIER_VERTEX_NBRS, refine = 1, num_iter = 10;
    int deg_threshold = 1000, async_chunks = 0;  // 0 = auto
    uint64_t seed = 0;  // ParOptions.seed: salts the async damping coin
};
// first_level: the first iteration may run as one wave (P auto); later
// async iterations take at least async_min_subrounds() ordered sub-rounds.
int async_min_subrounds();
bool par_best_moves(const lcc_graph& g, const double* k, double lam, const Options& o, bool first_level, int32_t* C,
                    double* K, lcc_stats* st, cudaStream_t s);
void parallel_cc(const lcc_graph& g, const double* k, double lam, const Options& o, int32_t* C_out,
                 lcc_stats* st, cudaStream_t s);

}  // namespace lcc
