/*
 * lcc_b200.h -- C ABI of the B200-native LambdaCC best-move / contraction path.
 *
 * Every entry point takes plain pointers and sizes.  Graph, label and mass
 * arrays are DEVICE pointers on the current CUDA device unless a name says
 * "host"; `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  All calls are stream-ordered; the ones that return counts to the
 * host synchronise that stream once.  Scratch is taken from the device's
 * stream-ordered pool (cudaMallocAsync); no global state is kept.
 *
 * The reference (arXiv 2108.01731, /root/reference) has no FFI: its hot path
 * is specified as Python functions over `WeightedGraph` (graph.py:23-38).
 * Each entry point below replaces one of those functions; the citation names
 * the SPEC operation it implements.  INTEGRATION.md shows the ctypes binding.
 *
 * Errors: a non-zero lcc_status is returned and lcc_last_error() (thread
 * local) holds a one-line message.  LCC_ERR_INVALID mirrors the reference's
 * GraphError/ValueError (graph.py:19-20; SPEC "errors:" clauses).
 */
#ifndef LCC_B200_H
#define LCC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LCC_ABI_VERSION 3

typedef enum {
    LCC_OK = 0,
    LCC_ERR_INVALID = 1, /* bad argument: maps to GraphError / ValueError  */
    LCC_ERR_CUDA = 2,    /* CUDA runtime / launch failure                   */
    LCC_ERR_OOM = 3      /* device allocation failed                        */
} lcc_status;

/* LCC_W_U32: non-negative integer weights (multi-edge counts, e.g. every
 * coarse level of an unweighted graph), summed exactly in 32-bit integers;
 * requires 2 * total_weight < 2^32.                                          */
/* lcc_graph.flags: LCC_GRAPH_PARTIAL_ROWS -- only some vertices carry their
 * rows (a rank's shard in the vertex-partitioned driver), so the CSR is not
 * symmetric as stored.  Whole graphs pass 0.                                 */
enum { LCC_GRAPH_PARTIAL_ROWS = 1 };
typedef enum { LCC_W_NONE = 0, LCC_W_F32 = 1, LCC_W_F64 = 2, LCC_W_U32 = 3 } lcc_wtype;
/* ParOptions.schedule */
typedef enum { LCC_SYNC = 0, LCC_ASYNC = 1 } lcc_schedule;
/* ParOptions.frontier_policy */
typedef enum {
    LCC_FRONTIER_ALL = 0,
    LCC_FRONTIER_VERTEX_NBRS = 1,
    LCC_FRONTIER_CLUSTER_NBRS = 2
} lcc_frontier_policy;

/* Undirected graph in symmetric CSR form, the device image of the reference
 * WeightedGraph (graph.py:33-38).  weights == NULL (wtype LCC_W_NONE) means
 * every edge weighs 1.  nnz = 2m.                                           */
typedef struct {
    int64_t n;
    int64_t nnz;
    const int64_t* indptr;  /* [n+1]                                       */
    const int32_t* indices; /* [nnz], sorted within each row, no self loops */
    const void* weights;    /* [nnz] float, double or uint32, or NULL      */
    int32_t wtype;          /* lcc_wtype                                    */
    int32_t flags;          /* LCC_GRAPH_* bits (0 for a whole graph)       */
    double total_weight;    /* sum of w over undirected edges               */
} lcc_graph;

/* ClusteringParams: k == NULL means k_v = 1.                */
typedef struct {
    const double* k; /* [n] device, or NULL                                 */
    double lambda;
} lcc_params;

/* ParOptions.                                             */
typedef struct {
    int32_t schedule;         /* lcc_schedule                              */
    int32_t frontier_policy;  /* lcc_frontier_policy                       */
    int32_t refine;           /* 0/1                                        */
    int32_t num_iter;         /* >= 1, default 10                          */
    uint64_t seed;            /* recorded; sync mode is seed-independent    */
    int32_t degree_threshold; /* vertices above it use the block/global
                                 hash path (default 1000)    */
    int32_t async_chunks;     /* async: frontier processed in this many
                                 ordered sub-rounds; 0 = auto              */
} lcc_options;

/* Per-call counters, accumulated (caller zeroes).                           */
typedef struct {
    int64_t rounds;        /* best-move iterations executed              */
    int64_t levels;        /* levels visited by parallel_cc              */
    int64_t vertices;      /* sum of |V'| over rounds                    */
    int64_t edges_scanned; /* sum of deg(v), v in V', over rounds        */
    int64_t moves;         /* sum of moved vertices over rounds          */
    double ms_best_moves;  /* device time of the best-move iterations     */
    double ms_total;       /* device time of the whole call              */
    double ms_kernels;     /* device time of the best-move kernels alone */
    int64_t kernel_launches; /* best-move kernel launches                */
} lcc_stats;

int lcc_abi_version(void);
/* Hand the library's cached device scratch (stream-ordered pool) back to
 * the driver.  Calls keep up to LCC_POOL_KEEP_GB (default 64) GB cached
 * between them: fresh pool memory costs ~6 ms per GB to map.             */
lcc_status lcc_release_memory(void);
const char* lcc_last_error(void);
/* Number of this library's own kernel launches so far in this process
 * (diagnostics; CUB helper kernels are not counted).                       */
int64_t lcc_kernel_launches(void);

/* ---- one best-move iteration -------------------------------------------
 * Alg. 1 lines 6-8, per_vertex_best_target for every v in
 * the frontier.  frontier == NULL means all vertices.
 *   LCC_SYNC : reads C[n], K[n]; writes D[n] (D[v] = C[v] unless v moves,
 *              fresh-singleton targets are n+v) and moved[n] (0/1).
 *   LCC_ASYNC: updates C[n] and K[2n] in place with relaxed atomics
 *              (SPEC.md:261,313); D may be NULL; moved[n] written.
 * nbr_mark (may be NULL, n bytes): zeroed, then nbr_mark[u] = 1 for every
 * neighbour u of a mover -- the VertexNeighbors frontier
 * fused into the round; lcc_frontier_from_mask compacts it.
 * *moved_count (host) receives the number of movers; stats (may be NULL) is
 * accumulated (vertices, edges scanned, movers, best-move kernel time).     */
lcc_status lcc_best_moves_round(const lcc_graph* g, const lcc_params* p,
                                int32_t* C, double* K,
                                const int32_t* frontier, int64_t n_frontier,
                                int32_t schedule, int32_t degree_threshold,
                                int32_t async_chunks,
                                int32_t* D, uint8_t* moved, uint8_t* nbr_mark,
                                int64_t* moved_count, lcc_stats* stats,
                                void* stream);

/* ---- sync apply: canonicalise labels and rebuild masses ----
 * labels_in[n] take values in [0, label_range); writes C[v] = smallest member
 * id of v's cluster and K[x] = sum of k over members (K has n entries).     */
lcc_status lcc_apply_moves(int64_t n, const int32_t* labels_in, int64_t label_range,
                           const double* k, int32_t* C, double* K, void* stream);

/* ---- compute_frontier ---------------------------------
 * Writes the sorted member ids to frontier[n]; *n_frontier (host) = size.   */
lcc_status lcc_compute_frontier(const lcc_graph* g, int32_t policy,
                                const uint8_t* moved, const int32_t* C_old,
                                const int32_t* C_new, int32_t* frontier,
                                int64_t* n_frontier, void* stream);

/* Sorted ids v with mark[v] != 0 -> frontier[n]; *n_frontier (host) = size.
 * With the nbr_mark of lcc_best_moves_round this equals compute_frontier
 * under LCC_FRONTIER_VERTEX_NBRS.                                           */
lcc_status lcc_frontier_from_mask(int64_t n, const uint8_t* mark, int32_t* frontier,
                                  int64_t* n_frontier, void* stream);

/* ---- par_best_moves -----------------------------------
 * Up to opts->num_iter iterations starting from the frontier V' = V.
 * C[n] (canonical labels) and K[n] are updated in place.                   */
lcc_status lcc_par_best_moves(const lcc_graph* g, const lcc_params* p,
                              const lcc_options* opts, int32_t* C, double* K,
                              int32_t* any_moved, lcc_stats* stats, void* stream);

/* ---- par_compress ----------------------------
 * C[n] must be canonical (smallest-member ids) with masses K[n].  Outputs,
 * caller-allocated with these upper bounds: mapping[n], ck[n],
 * cindptr[n+1], cindices[nnz], cweights[nnz] (double).  Host outputs: coarse
 * vertex count, coarse nnz, internal_offset, coarse total weight.          */
lcc_status lcc_par_compress(const lcc_graph* g, const lcc_params* p,
                            const int32_t* C, const double* K,
                            int32_t* mapping, double* ck, int64_t* cindptr,
                            int32_t* cindices, double* cweights,
                            int64_t* cn, int64_t* cnnz, double* internal_offset,
                            double* ctotal_weight, void* stream);

/* ---- par_flatten -----------------------------
 * C[v] = canonical(Cc[mapping[v]]); K[n] rebuilt from k.                    */
lcc_status lcc_par_flatten(int64_t n, const int32_t* mapping, const int32_t* Cc,
                           const double* k, int32_t* C, double* K, void* stream);

/* ---- cc_objective -------------------------------------
 * Unordered-pair LambdaCC objective of clustering C[n] (any labels < n).   */
lcc_status lcc_cc_objective(const lcc_graph* g, const lcc_params* p,
                            const int32_t* C, double* objective, void* stream);

/* ---- weighted_degrees (graph.py:57-61) -----------------
 * k[v] = sum of the weights of v's CSR row, summed left to right in fp64
 * (the reference's np.add.at order: bit-identical).  The k_v of the
 * modularity mapping (modularity_params).                                  */
lcc_status lcc_weighted_degrees(const lcc_graph* g, double* k, void* stream);

/* ---- parallel_cc (Alg. 1) ---------------------
 * Full multi-level clustering.  C_out[n] receives canonical labels.        */
lcc_status lcc_parallel_cc(const lcc_graph* g, const lcc_params* p,
                           const lcc_options* opts, int32_t* C_out,
                           lcc_stats* stats, void* stream);

/* ---- generators / graph build ---------------------
 * R-MAT: samples = edge_factor * 2^scale directed draws by
 * recursive quadrant descent with probabilities (a, b, c, 1-a-b-c), counter-
 * based RNG (splitmix64 of seed, sample, level); then symmetrised, deduped
 * and self-loops dropped into CSR.  indptr[2^scale+1]; indices must hold
 * 2*samples entries.  *nnz (host) receives 2m.                              */
lcc_status lcc_gen_rmat(int32_t scale, int64_t samples, double a, double b,
                        double c, uint64_t seed, int64_t* indptr,
                        int32_t* indices, int64_t* nnz, void* stream);

/* Power-law planted communities (config 5 stand-in): `samples` Chung-Lu draws,
 * intra-community with probability 1-mu (community by weight, endpoints by
 * weight inside it; communities are contiguous id ranges cstart[0..nc]),
 * otherwise endpoints by weight over all vertices.  vw_prefix[n+1] and
 * cw_prefix[nc+1] are exclusive prefix sums of the vertex / community
 * weights (device).  Deduplicated, symmetrised CSR as lcc_gen_rmat.         */
lcc_status lcc_gen_powerlaw_communities(int64_t n, int64_t samples, double mu,
                                        const double* vw_prefix, const int64_t* cstart,
                                        const double* cw_prefix, int64_t n_communities,
                                        uint64_t seed, int64_t* indptr, int32_t* indices,
                                        int64_t* nnz, void* stream);

/* Build symmetric CSR from undirected pairs (u[i], v[i]) on the device:
 * self-loops dropped, duplicate unordered pairs merged (unweighted graphs,
 * so merged edges keep w = 1), both directions emitted, rows sorted.
 * indices must hold 2*n_pairs entries.  *nnz (host) receives 2m.           */
lcc_status lcc_build_csr_from_pairs(int64_t n, int64_t n_pairs, const int32_t* u,
                                    const int32_t* v, int64_t* indptr,
                                    int32_t* indices, int64_t* nnz, void* stream);

/* build_graph (reference graph.py:79-164) on the device.  Edge list
 * (u[i], v[i], w[i]) with int64 ids (w == NULL: all 1.0): self loops dropped,
 * same-orientation parallel edges summed in ascending weight order, the two
 * orientations of a pair averaged, both directions emitted with rows sorted;
 * every fp64 sum in numpy's order, so indptr / indices / weights and
 * *total_weight are bit-identical to the reference's.  Ids must lie in
 * [0, n) (lcc_edge_id_range gives n_seen = max id + 1; the reference's
 * GraphError cases are LCC_ERR_INVALID).  indptr[n+1]; indices and weights
 * must hold 2 * n_edges entries.  *m = undirected edge count (nnz = 2m);
 * *unit_weights = 1 when every weight is 1.                                */
lcc_status lcc_build_graph(int64_t n, int64_t n_edges, const int64_t* u, const int64_t* v,
                           const double* w, int64_t* indptr, int32_t* indices, double* weights,
                           int64_t* m, double* total_weight, int32_t* unit_weights, void* stream);
/* Smallest and largest id over u[] and v[] (device reduce; n_edges == 0
 * gives min 0, max -1).                                                     */
lcc_status lcc_edge_id_range(int64_t n_edges, const int64_t* u, const int64_t* v,
                             int64_t* min_id, int64_t* max_id, void* stream);

/* COO -> CSR with duplicate (row, col) entries summed (the merge step of the
 * sharded contraction: partial coarse rows arriving from several ranks).
 * rows[i] in [0, n), cols[i] >= 0.  wtype LCC_W_NONE (each entry counts 1)
 * or LCC_W_U32: uint32 sums in w_out; LCC_W_F64: double sums.  indptr[n+1];
 * indices / w_out hold up to nnz entries; *nnz_out = merged entries.       */
lcc_status lcc_coo_merge(int64_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                         const void* w, int32_t wtype, int64_t* indptr, int32_t* indices,
                         void* w_out, int64_t* nnz_out, void* stream);

/* ---- eval -----------------------
 * Adjusted Rand index and normalised mutual information (arithmetic-mean
 * normalisation) of two labelings a[n], b[n] (any int32
 * values), over their contingency table; sklearn's degenerate cases
 * (SPEC.md:354-364 `ari`, `nmi`).                                          */
lcc_status lcc_partition_scores(int64_t n, const int32_t* a, const int32_t* b,
                                double* ari, double* nmi, void* stream);
/* avg_precision_recall: ground-truth communities as CSR
 * (offsets[n_comm+1] starting at 0, members[offsets[n_comm]] vertex ids,
 * each community non-empty and duplicate-free; they may overlap).  For each
 * community t the cluster c' of C[n] with the largest |t & c'| (ties to the
 * lowest cluster id); unweighted means of |t&c'|/|c'| and |t&c'|/|t|.
 * n_comm == 0 or a member id outside [0, n) -> LCC_ERR_INVALID.             */
lcc_status lcc_avg_precision_recall(int64_t n, const int32_t* C, int64_t n_comm,
                                    const int64_t* offsets, const int32_t* members,
                                    double* precision, double* recall, void* stream);
/* cluster_stats: number of clusters and min / max / mean
 * cluster size of C[n].                                                     */
lcc_status lcc_cluster_stats(int64_t n, const int32_t* C, int64_t* num_clusters,
                             int64_t* min_size, int64_t* max_size, double* mean_size,
                             void* stream);
#ifdef __cplusplus
}
#endif
#endif /* LCC_B200_H */
