/*
 * lcc_oracle.c -- CPU restatement of the LambdaCC parallel-Louvain hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the timed CPU baseline ("kind": "port") in bench.py.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path (paper_2108_01731_b200/)
 * never links or calls it.
 *
 * What it restates (the reference ships these only as specification):
 *   - per-vertex best target / best-move round (sync "Jacobi" and async)
 *       /root/reference/SPEC.md:258-266, 296-304
 *       move delta: PAPER.md:525-527
 *       tie rule (strict > 0, lowest id): SPEC.md:164; fresh singleton: SPEC.md:230
 *   - sync apply + cluster-mass rebuild
 *   - async live mass updates + boundary reconcile  SPEC.md:313; _atomics.py:37-43
 *   - compute_frontier (All / VertexNeighbors / ClusterNeighbors)  SPEC.md:267-275;
 *       PAPER.md:201-212
 *   - compress (renumber by smallest member, merge by sum, internal_offset)
 *       SPEC.md:196-204, 276-282; edge-merge algorithm graph.py:126-164
 *   - flatten
 *   - cc_objective closed form
 *
 * Canonical conventions shared with the CUDA kernels:
 *   gain(x) = (S_x - t*K_x) - b,  b = (S_c - t*K_c) + t*k_v,  t = lam*k_v
 *   evaluated in exactly that order with no FMA contraction (-ffp-contract=off);
 *   fresh singleton = temporary id n+v, gain -b, loses all ties;
 *   move iff best gain > 0; ties -> lowest cluster id;
 *   after every round labels are canonicalised to the minimum member id.
 *
 * Build: see oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off -shared).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define EMPTY_I32 (-1)

static inline double wt(const double* w, int64_t e) { return w ? w[e] : 1.0; }
static inline double kv_of(const double* k, int64_t v) { return k ? k[v] : 1.0; }

/* ------------------------------------------------------------------ */
/* per-vertex best target, dense scratch S[label] with touched list.  */
/* Returns the chosen label (== C[v] when staying) and the best gain.  */
/* S must be zero on entry and is left zero on exit.                   */
/* ------------------------------------------------------------------ */
static int32_t best_target(int64_t n, const int64_t* indptr, const int32_t* indices,
                           const double* w, const double* k, double lam,
                           const int32_t* C, const double* K, int64_t v,
                           double* S, int32_t* touched, double* gain_out)
{
    const int32_t c = C[v];
    const double kv = kv_of(k, v);
    const double t = lam * kv;
    int64_t nt = 0;
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
        int32_t x = C[indices[e]];
        S[x] += wt(w, e);          /* CSR order: the summation order is fixed */
        touched[nt++] = x;         /* may repeat; repeats score identically   */
    }
    const double Sc = S[c];
    const double b = (Sc - t * K[c]) + t * kv;
    int32_t best = -1;
    double bestg = 0.0;
    for (int64_t i = 0; i < nt; ++i) {
        int32_t x = touched[i];
        if (x == c) continue;
        double a = S[x] - t * K[x];
        double g = a - b;
        if (best < 0 || g > bestg || (g == bestg && x < best)) { best = x; bestg = g; }
    }
    /* fresh singleton: a = 0 - t*0 = 0, gain = 0 - b; id n+v loses ties */
    double gf = 0.0 - b;
    int32_t choice = c;
    double cg = 0.0;
    if (best >= 0) { choice = best; cg = bestg; }
    if (best < 0 || gf > cg) { choice = (int32_t)(n + v); cg = gf; }
    for (int64_t i = 0; i < nt; ++i) S[touched[i]] = 0.0;
    if (!(cg > 0.0)) { choice = c; }
    if (gain_out) *gain_out = (choice == c) ? 0.0 : cg;
    return choice;
}

/* Synchronous round.  D[v] = C[v] for all v, then D[v] = target for v in F.
 * moved[v] = 1 iff D[v] != C[v].  Returns number of moved vertices.
 * F == NULL means all vertices.  Labels in C must be < label_range (>= n;
 * canonical labels are < n).                                                 */
int64_t orc_sync_round(int64_t n, const int64_t* indptr, const int32_t* indices,
                       const double* w, const double* k, double lam,
                       const int32_t* C, const double* K,
                       const int32_t* F, int64_t nF,
                       int32_t* D, uint8_t* moved, double* gains, int threads,
                       int64_t label_range)
{
    if (label_range < n) label_range = n;
    if (threads > 0) omp_set_num_threads(threads);
    memcpy(D, C, sizeof(int32_t) * (size_t)n);
    memset(moved, 0, (size_t)n);
    const int64_t cnt = F ? nF : n;
    int64_t nmoved = 0;
    int64_t maxdeg = 0;
    for (int64_t v = 0; v < n; ++v) {
        int64_t d = indptr[v + 1] - indptr[v];
        if (d > maxdeg) maxdeg = d;
    }
#pragma omp parallel reduction(+ : nmoved)
    {
        double* S = (double*)calloc((size_t)(label_range + 1), sizeof(double));
        int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(maxdeg + 1));
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < cnt; ++i) {
            int64_t v = F ? F[i] : i;
            double g;
            int32_t x = best_target(n, indptr, indices, w, k, lam, C, K, v, S, touched, &g);
            if (gains) gains[v] = g;
            if (x != C[v]) { D[v] = x; moved[v] = 1; nmoved++; }
        }
        free(S); free(touched);
    }
    return nmoved;
}

static inline void atomic_add_double(double* p, double val)
{
    uint64_t* q = (uint64_t*)p;
    uint64_t old = __atomic_load_n(q, __ATOMIC_RELAXED);
    for (;;) {
        double d; memcpy(&d, &old, 8);
        d += val;
        uint64_t nw; memcpy(&nw, &d, 8);
        if (__atomic_compare_exchange_n(q, &old, nw, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) break;
    }
}

/* Asynchronous round with live updates.
 * C (labels, may take values in [0,2n)) and K (size 2n) are updated in place.
 * parallel == 0: sequential Gauss-Seidel in frontier order (deterministic,
 *                equivalent to the single-thread async schedule).
 * parallel != 0: OpenMP parfor with relaxed atomics, the shape of the
 *                reference's numba+_atomics design (nondeterministic).
 * moved[] is zeroed and set for movers.  Returns moved count.                */
int64_t orc_async_round(int64_t n, const int64_t* indptr, const int32_t* indices,
                        const double* w, const double* k, double lam,
                        int32_t* C, double* K, const int32_t* F, int64_t nF,
                        uint8_t* moved, int parallel, int threads)
{
    if (threads > 0) omp_set_num_threads(threads);
    memset(moved, 0, (size_t)n);
    const int64_t cnt = F ? nF : n;
    int64_t maxdeg = 0;
    for (int64_t v = 0; v < n; ++v) {
        int64_t d = indptr[v + 1] - indptr[v];
        if (d > maxdeg) maxdeg = d;
    }
    int64_t nmoved = 0;
    if (!parallel) {
        double* S = (double*)calloc((size_t)(2 * n + 1), sizeof(double));
        int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(maxdeg + 1));
        for (int64_t i = 0; i < cnt; ++i) {
            int64_t v = F ? F[i] : i;
            int32_t c = C[v];
            int32_t x = best_target(n, indptr, indices, w, k, lam, C, K, v, S, touched, NULL);
            if (x != c) {
                double kv = kv_of(k, v);
                K[c] -= kv; K[x] += kv; C[v] = x; moved[v] = 1; nmoved++;
            }
        }
        free(S); free(touched);
        return nmoved;
    }
#pragma omp parallel reduction(+ : nmoved)
    {
        double* S = (double*)calloc((size_t)(2 * n + 1), sizeof(double));
        int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(maxdeg + 1));
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < cnt; ++i) {
            int64_t v = F ? F[i] : i;
            int32_t c = __atomic_load_n(&C[v], __ATOMIC_RELAXED);
            int32_t x = best_target(n, indptr, indices, w, k, lam, C, K, v, S, touched, NULL);
            if (x != c) {
                double kv = kv_of(k, v);
                atomic_add_double(&K[c], -kv);
                atomic_add_double(&K[x], kv);
                __atomic_store_n(&C[v], x, __ATOMIC_RELAXED);
                moved[v] = 1; nmoved++;
            }
        }
        free(S); free(touched);
    }
    return nmoved;
}

/* Canonicalise labels to the minimum member id and rebuild K (size >= n).
 * D holds labels in [0, label_range).                                       */
void orc_canonicalize(int64_t n, const int32_t* D, int64_t label_range,
                      const double* k, int32_t* C, double* K)
{
    int32_t* minm = (int32_t*)malloc(sizeof(int32_t) * (size_t)label_range);
    for (int64_t x = 0; x < label_range; ++x) minm[x] = INT32_MAX;
    for (int64_t v = 0; v < n; ++v) if ((int32_t)v < minm[D[v]]) minm[D[v]] = (int32_t)v;
    for (int64_t v = 0; v < n; ++v) C[v] = minm[D[v]];
    free(minm);
    for (int64_t x = 0; x < n; ++x) K[x] = 0.0;
    for (int64_t v = 0; v < n; ++v) K[C[v]] += kv_of(k, v);
}

/* Frontier.  policy: 0 = AllVertices, 1 = VertexNeighbors, 2 = ClusterNeighbors.
 * Cold = labels before the round, Cnew = labels after (both canonical).
 * Writes sorted ids into F, returns the count.                               */
int64_t orc_frontier(int64_t n, const int64_t* indptr, const int32_t* indices,
                     int policy, const uint8_t* moved,
                     const int32_t* Cold, const int32_t* Cnew, int32_t* F)
{
    int64_t any = 0;
    for (int64_t v = 0; v < n; ++v) any |= moved[v];
    if (!any) return 0;
    if (policy == 0) { for (int64_t v = 0; v < n; ++v) F[v] = (int32_t)v; return n; }
    uint8_t* mark = (uint8_t*)calloc((size_t)n, 1);
    if (policy == 1) {
        for (int64_t v = 0; v < n; ++v)
            if (moved[v])
                for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) mark[indices[e]] = 1;
    } else {
        /* superset reading: neighbours of the old members of
         * every source cluster, plus members and neighbours of the new
         * members of every destination cluster.                               */
        uint8_t* src = (uint8_t*)calloc((size_t)n, 1);
        uint8_t* dst = (uint8_t*)calloc((size_t)n, 1);
        for (int64_t v = 0; v < n; ++v)
            if (moved[v]) { src[Cold[v]] = 1; dst[Cnew[v]] = 1; }
        for (int64_t u = 0; u < n; ++u) {
            int s = src[Cold[u]], d = dst[Cnew[u]];
            if (d) mark[u] = 1;
            if (s || d)
                for (int64_t e = indptr[u]; e < indptr[u + 1]; ++e) mark[indices[e]] = 1;
        }
        free(src); free(dst);
    }
    int64_t nF = 0;
    for (int64_t v = 0; v < n; ++v) if (mark[v]) F[nF++] = (int32_t)v;
    free(mark);
    return nF;
}

typedef struct { int64_t e; int32_t b; int32_t _pad; } ent_t;
static int cmp_ent(const void* p, const void* q)
{
    const ent_t* a = (const ent_t*)p; const ent_t* b = (const ent_t*)q;
    if (a->b != b->b) return a->b < b->b ? -1 : 1;
    return a->e < b->e ? -1 : (a->e > b->e);
}

/* Compress.  C canonical (min-member ids), K masses.
 * Outputs (caller-allocated upper bounds): mapping[n], ck[n], cindptr[n+1],
 * cindices[nnz], cw[nnz].  Returns coarse nnz; *cn = coarse vertex count;
 * *offset = internal_offset; *ctotal = coarse total weight.
 * Each coarse row's entries are sorted by (neighbour, fine CSR position),
 * so merge sums run in CSR order of the fine graph -- the order the GPU's
 * stable radix sort produces.  OpenMP over rows (config 5: 3.6B entries);
 * the result does not depend on the thread count.                          */
int64_t orc_compress(int64_t n, const int64_t* indptr, const int32_t* indices,
                     const double* w, const double* k, double lam,
                     const int32_t* C, const double* K,
                     int32_t* mapping, double* ck, int64_t* cindptr,
                     int32_t* cindices, double* cw,
                     int64_t* cn_out, double* offset, double* ctotal)
{
    int32_t* rank = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int64_t cn = 0;
    for (int64_t x = 0; x < n; ++x) { rank[x] = (int32_t)cn; if (C[x] == (int32_t)x) cn++; }
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) mapping[v] = rank[C[v]];
    for (int64_t x = 0; x < n; ++x) if (C[x] == (int32_t)x) ck[rank[x]] = K[x];
    free(rank);
    /* intra-cluster mass and coarse row lengths */
    double intra = 0.0;
    int64_t* rowcnt = (int64_t*)calloc((size_t)(cn + 1), sizeof(int64_t));
    if (w) {
        /* fp sums: CSR order, sequential (weighted graphs are small here) */
        for (int64_t v = 0; v < n; ++v)
            for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
                int32_t a = mapping[v], b = mapping[indices[e]];
                if (a == b) intra += w[e]; else rowcnt[a]++;
            }
    } else {
        int64_t icnt = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : icnt)
        for (int64_t v = 0; v < n; ++v) {
            const int32_t a = mapping[v];
            int64_t out = 0;
            for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
                if (a == mapping[indices[e]]) icnt++; else out++;
            }
            if (out) __atomic_fetch_add(&rowcnt[a], out, __ATOMIC_RELAXED);
        }
        intra = (double)icnt;
    }
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cn + 1));
    start[0] = 0;
    for (int64_t a = 0; a < cn; ++a) start[a + 1] = start[a] + rowcnt[a];
    int64_t tot = start[cn];
    ent_t* ents = (ent_t*)malloc(sizeof(ent_t) * (size_t)(tot + 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cn + 1));
    memcpy(fill, start, sizeof(int64_t) * (size_t)(cn + 1));
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v) {
        const int32_t a = mapping[v];
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
            const int32_t b = mapping[indices[e]];
            if (a != b) {
                const int64_t p = __atomic_fetch_add(&fill[a], 1, __ATOMIC_RELAXED);
                ents[p].b = b; ents[p].e = e;
            }
        }
    }
    /* per coarse row: sort, merge runs in place, count */
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t a = 0; a < cn; ++a) {
        const int64_t s = start[a], e = start[a + 1];
        if (e - s > 1) qsort(ents + s, (size_t)(e - s), sizeof(ent_t), cmp_ent);
        int64_t o = s;
        for (int64_t i = s; i < e;) {
            const int32_t b = ents[i].b;
            double acc = 0.0;
            while (i < e && ents[i].b == b) { acc += wt(w, ents[i].e); ++i; }
            ents[o].b = b; ents[o].e = 0; ((double*)&ents[o])[0] = acc;  /* (sum kept in the e slot) */
            o++;
        }
        rowcnt[a] = o - s;
    }
    cindptr[0] = 0;
    for (int64_t a = 0; a < cn; ++a) cindptr[a + 1] = cindptr[a] + rowcnt[a];
    double total2 = 0.0;
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t a = 0; a < cn; ++a) {
        const int64_t s = start[a], d = cindptr[a];
        for (int64_t i = 0; i < rowcnt[a]; ++i) {
            cindices[d + i] = ents[s + i].b;
            cw[d + i] = ((const double*)&ents[s + i])[0];
        }
    }
    const int64_t out = cindptr[cn];
    for (int64_t i = 0; i < out; ++i) total2 += cw[i];
    double sk2 = 0.0, sK2 = 0.0;
    for (int64_t v = 0; v < n; ++v) { double kv = kv_of(k, v); sk2 += kv * kv; }
    for (int64_t x = 0; x < cn; ++x) sK2 += ck[x] * ck[x];
    *offset = intra * 0.5 - lam * (sK2 - sk2) * 0.5;
    *ctotal = total2 * 0.5;
    *cn_out = cn;
    free(rowcnt); free(start); free(ents); free(fill);
    return out;
}

/* Flatten: out[v] = Cc[mapping[v]], then canonicalise. */
void orc_flatten(int64_t n, const int32_t* mapping, const int32_t* Cc,
                 const double* k, int32_t* C, double* K)
{
    int32_t* D = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t v = 0; v < n; ++v) D[v] = Cc[mapping[v]];
    orc_canonicalize(n, D, n, k, C, K);
    free(D);
}

/* cc_objective closed form: unordered pairs.
 * obj = intra_dir*0.5 - lam*(sum_c K_c^2 - sum_v k_v^2)*0.5                */
double orc_objective(int64_t n, const int64_t* indptr, const int32_t* indices,
                     const double* w, const double* k, double lam, const int32_t* C)
{
    double intra = 0.0;
    if (w) {
        for (int64_t v = 0; v < n; ++v)
            for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e)
                if (C[v] == C[indices[e]]) intra += w[e];
    } else {  /* exact integer count: any order, all threads */
        int64_t cnt = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : cnt)
        for (int64_t v = 0; v < n; ++v)
            for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e)
                if (C[v] == C[indices[e]]) cnt++;
        intra = (double)cnt;
    }
    double* K = (double*)calloc((size_t)n, sizeof(double));
    double sk2 = 0.0, sK2 = 0.0;
    for (int64_t v = 0; v < n; ++v) { double kv = kv_of(k, v); K[C[v]] += kv; sk2 += kv * kv; }
    for (int64_t x = 0; x < n; ++x) sK2 += K[x] * K[x];
    free(K);
    return intra * 0.5 - lam * (sK2 - sk2) * 0.5;
}
