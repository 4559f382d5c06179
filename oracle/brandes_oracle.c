/*
 * oracle/brandes_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement (plain C, unit edge weights) of the reference's arithmetic
 * for the betweenness-centrality hot path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library;
 * the product path (paper_2008_05718_b200/) never does.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function here
 * against (a) the reference's own known-answer vectors
 * and (b) the JSON fixtures under tests/golden/, which were produced by importing the reference
 * package itself (tests/golden/gen_golden.py) in the build container.
 *
 * What each function follows:
 *   oracle_brandes_single_source  reference pkg/src/hybir/oracle.py:29-67
 *   oracle_brandes_bc             reference pkg/src/hybir/oracle.py:70-82
 *   oracle_masked_relax           reference pkg/src/hybir/relax.py:42-103
 *   oracle_build_levels           reference pkg/src/hybir/relax.py:106-113
 *   oracle_brandes_single_source_w / oracle_brandes_bc_w
 *                                 the same two functions on weighted graphs
 *                                 (positive integer weights, heap Dijkstra)
 *
 * Unit weights turn the reference's heap Dijkstra into a breadth-first
 * search; the heap pops (dist, vertex) pairs, so vertices settle in ascending
 * (dist, id) order and predecessor lists are in ascending id order.  The code
 * below reproduces exactly that order, which makes delta bit-identical to the
 * Python oracle as long as sigma stays below 2^53 (Python divides exact
 * integers with correct rounding; fp64 division of exactly representable
 * integers gives the same quotient).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_UNREACHED (-1)

typedef struct {
    int64_t *queue;   /* n entries */
    int64_t *order;   /* n entries: reached vertices sorted by (dist, id) */
    int64_t *count;   /* n + 2 entries: per-level counters */
} scratch_t;

static int scratch_init(scratch_t *sc, int64_t n) {
    sc->queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    sc->order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    sc->count = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 2));
    return (sc->queue && sc->order && sc->count) ? 0 : -1;
}

static void scratch_free(scratch_t *sc) {
    free(sc->queue);
    free(sc->order);
    free(sc->count);
}

/* Forward + backward pass from one source (oracle.py:29-67).
 * dist: -1 where unreached (the reference uses None, oracle.py:36).
 * Returns the number of reached vertices; *out_levels = eccentricity + 1,
 * *out_sigma_max = largest path count seen (callers assert it is < 2^53
 * before they claim bit-exact sigma). */
static int64_t single_source(int64_t n, const int64_t *offsets, const int32_t *col, int64_t s,
                             int64_t *dist, double *sigma, double *delta, scratch_t *sc,
                             int64_t *out_levels, double *out_sigma_max,
                             int64_t *out_arcs_reached, int64_t *out_dag_arcs) {
    int64_t head = 0, tail = 0, reached, maxd = 0;
    for (int64_t v = 0; v < n; ++v) {
        dist[v] = ORACLE_UNREACHED;
        sigma[v] = 0.0;
        delta[v] = 0.0;
    }
    dist[s] = 0;
    sc->queue[tail++] = s;
    while (head < tail) {
        int64_t v = sc->queue[head++];
        int64_t dv = dist[v];
        for (int64_t k = offsets[v]; k < offsets[v + 1]; ++k) {
            int64_t w = col[k];
            if (dist[w] == ORACLE_UNREACHED) {
                dist[w] = dv + 1;
                if (dv + 1 > maxd) maxd = dv + 1;
                sc->queue[tail++] = w;
            }
        }
    }
    reached = tail;

    /* Settle order of the reference's heap: ascending (dist, id). */
    memset(sc->count, 0, sizeof(int64_t) * (size_t)(maxd + 2));
    for (int64_t v = 0; v < n; ++v)
        if (dist[v] >= 0) sc->count[dist[v] + 1]++;
    for (int64_t d = 0; d <= maxd; ++d) sc->count[d + 1] += sc->count[d];
    for (int64_t v = 0; v < n; ++v)
        if (dist[v] >= 0) sc->order[sc->count[dist[v]]++] = v;

    /* sigma[w] = sum of sigma over predecessors, ascending id (oracle.py:56-61). */
    double smax = 1.0;
    int64_t arcs_reached = 0, dag = 0;
    sigma[s] = 1.0;
    for (int64_t i = 0; i < reached; ++i) {
        int64_t w = sc->order[i];
        arcs_reached += offsets[w + 1] - offsets[w];
        if (w == s) continue;
        double acc = 0.0;
        int64_t dw = dist[w];
        for (int64_t k = offsets[w]; k < offsets[w + 1]; ++k) {
            int64_t v = col[k];
            if (dist[v] == dw - 1) {
                acc += sigma[v];
                ++dag;
            }
        }
        sigma[w] = acc;
        if (acc > smax) smax = acc;
    }

    /* Reverse settle order; each vertex pushes into its predecessors
     * (oracle.py:63-66). */
    for (int64_t i = reached - 1; i >= 0; --i) {
        int64_t u = sc->order[i];
        int64_t du = dist[u];
        double coeff = 1.0 + delta[u];
        double su = sigma[u];
        for (int64_t k = offsets[u]; k < offsets[u + 1]; ++k) {
            int64_t v = col[k];
            if (dist[v] == du - 1) delta[v] += (sigma[v] / su) * coeff;
        }
    }
    if (out_levels) *out_levels = maxd + 1;
    if (out_sigma_max) *out_sigma_max = smax;
    if (out_arcs_reached) *out_arcs_reached = arcs_reached;
    if (out_dag_arcs) *out_dag_arcs = dag;
    return reached;
}

/* stats (may be NULL): [0] reached vertices, [1] levels, [2] arcs incident to
 * reached vertices (A_r), [3] shortest-path DAG arcs (T). */
int oracle_brandes_single_source(int64_t n, const int64_t *offsets, const int32_t *col, int64_t s,
                                 int64_t *dist, double *sigma, double *delta,
                                 double *sigma_max, int64_t *stats) {
    scratch_t sc;
    int64_t levels = 0, ar = 0, dag = 0;
    if (n <= 0 || s < 0 || s >= n) return 2;
    if (scratch_init(&sc, n)) {
        scratch_free(&sc);
        return 1;
    }
    int64_t reached =
        single_source(n, offsets, col, s, dist, sigma, delta, &sc, &levels, sigma_max, &ar, &dag);
    if (stats) {
        stats[0] = reached;
        stats[1] = levels;
        stats[2] = ar;
        stats[3] = dag;
    }
    scratch_free(&sc);
    return 0;
}

/* bc[v] = sum over sources s != v of delta_s[v] (oracle.py:70-82), sources
 * dealt to OpenMP threads; per-thread partial vectors are added in thread
 * order so a fixed thread count gives a fixed result.
 * totals (may be NULL): [0] sum n_r, [1] sum A_r, [2] sum T, [3] max levels;
 * sigma_max (may be NULL): largest path count over all sources. */
int oracle_brandes_bc(int64_t n, const int64_t *offsets, const int32_t *col,
                      const int64_t *sources, int64_t k, double *bc, int nthreads,
                      int64_t *totals, double *sigma_max) {
    if (n <= 0) return 2;
    for (int64_t i = 0; i < k; ++i)
        if (sources[i] < 0 || sources[i] >= n) return 2;
    if (nthreads < 1) nthreads = 1;
    double *partial = (double *)calloc((size_t)nthreads * (size_t)n, sizeof(double));
    int64_t *tot = (int64_t *)calloc((size_t)nthreads * 4, sizeof(int64_t));
    double *smax = (double *)calloc((size_t)nthreads, sizeof(double));
    int failed = 0;
    if (!partial || !tot || !smax) {
        free(partial);
        free(tot);
        free(smax);
        return 1;
    }
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
#endif
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        scratch_t sc;
        int64_t *dist = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
        double *sigma = (double *)malloc(sizeof(double) * (size_t)n);
        double *delta = (double *)malloc(sizeof(double) * (size_t)n);
        int ok = !scratch_init(&sc, n) && dist && sigma && delta;
        if (!ok) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
        }
        double *mine = partial + (size_t)t * (size_t)n;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t i = 0; i < k; ++i) {
            if (!ok) continue;
            int64_t s = sources[i], levels = 0, ar = 0, dag = 0;
            double sm = 0.0;
            int64_t reached = single_source(n, offsets, col, s, dist, sigma, delta, &sc, &levels,
                                            &sm, &ar, &dag);
            for (int64_t v = 0; v < n; ++v)
                if (v != s) mine[v] += delta[v];
            tot[t * 4 + 0] += reached;
            tot[t * 4 + 1] += ar;
            tot[t * 4 + 2] += dag;
            if (levels > tot[t * 4 + 3]) tot[t * 4 + 3] = levels;
            if (sm > smax[t]) smax[t] = sm;
        }
        scratch_free(&sc);
        free(dist);
        free(sigma);
        free(delta);
    }
    for (int64_t v = 0; v < n; ++v) bc[v] = 0.0;
    for (int t = 0; t < nthreads; ++t)
        for (int64_t v = 0; v < n; ++v) bc[v] += partial[(size_t)t * (size_t)n + v];
    if (totals) {
        totals[0] = totals[1] = totals[2] = totals[3] = 0;
        for (int t = 0; t < nthreads; ++t) {
            totals[0] += tot[t * 4 + 0];
            totals[1] += tot[t * 4 + 1];
            totals[2] += tot[t * 4 + 2];
            if (tot[t * 4 + 3] > totals[3]) totals[3] = tot[t * 4 + 3];
        }
    }
    if (sigma_max) {
        *sigma_max = 0.0;
        for (int t = 0; t < nthreads; ++t)
            if (smax[t] > *sigma_max) *sigma_max = smax[t];
    }
    free(partial);
    free(tot);
    free(smax);
    return failed ? 1 : 0;
}

/* ------------------------------------------------------------------------
 * Weighted graphs (positive integer arc weights): the reference's heap Dijkstra
 * itself (oracle.py:44-61).  The heap holds (dist, vertex) pairs compared
 * lexicographically and stale entries are skipped, so vertices settle in
 * ascending (dist, id) order exactly as in the Python code; the backward pass
 * walks that order in reverse (oracle.py:63-66).
 * ------------------------------------------------------------------------ */
typedef struct {
    int64_t d, v;
} heap_item_t;

static int heap_less(heap_item_t a, heap_item_t b) { return a.d < b.d || (a.d == b.d && a.v < b.v); }

static void heap_push(heap_item_t *h, int64_t *size, heap_item_t x) {
    int64_t i = (*size)++;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!heap_less(x, h[p])) break;
        h[i] = h[p];
        i = p;
    }
    h[i] = x;
}

static heap_item_t heap_pop(heap_item_t *h, int64_t *size) {
    heap_item_t top = h[0], x = h[--(*size)];
    int64_t i = 0, n = *size;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && heap_less(h[c + 1], h[c])) ++c;
        if (!heap_less(h[c], x)) break;
        h[i] = h[c];
        i = c;
    }
    if (n > 0) h[i] = x;
    return top;
}

/* heap: capacity n_arcs + 1 entries (every improving relaxation pushes once). */
static int64_t single_source_w(int64_t n, const int64_t *offsets, const int32_t *col,
                               const int64_t *wgt, int64_t s, int64_t *dist, double *sigma,
                               double *delta, int64_t *order, heap_item_t *heap,
                               int64_t *out_maxd, double *out_sigma_max, int64_t *out_arcs_reached,
                               int64_t *out_dag_arcs) {
    int64_t hs = 0, reached = 0, maxd = 0, arcs_reached = 0, dag = 0;
    double smax = 1.0;
    for (int64_t v = 0; v < n; ++v) {
        dist[v] = ORACLE_UNREACHED;
        sigma[v] = 0.0;
        delta[v] = 0.0;
    }
    /* delta doubles as the "settled" flag holder until the backward pass: use order[] marks */
    dist[s] = 0;
    sigma[s] = 1.0;
    heap_push(heap, &hs, (heap_item_t){0, s});
    /* settled[v] is encoded as delta[v] = -1 during the forward pass */
    while (hs > 0) {
        heap_item_t it = heap_pop(heap, &hs);
        int64_t v = it.v, d = it.d;
        if (delta[v] < 0.0 || d != dist[v]) continue;
        delta[v] = -1.0;
        order[reached++] = v;
        if (d > maxd) maxd = d;
        arcs_reached += offsets[v + 1] - offsets[v];
        for (int64_t k = offsets[v]; k < offsets[v + 1]; ++k) {
            int64_t w = col[k];
            int64_t nd = d + wgt[k];
            if (dist[w] == ORACLE_UNREACHED || nd < dist[w]) {
                dist[w] = nd;
                sigma[w] = sigma[v];
                heap_push(heap, &hs, (heap_item_t){nd, w});
            } else if (nd == dist[w]) {
                sigma[w] += sigma[v];
            }
        }
    }
    for (int64_t i = 0; i < reached; ++i) {
        delta[order[i]] = 0.0;
        if (sigma[order[i]] > smax) smax = sigma[order[i]];
    }
    for (int64_t i = reached - 1; i >= 0; --i) {
        int64_t u = order[i];
        int64_t du = dist[u];
        double coeff = 1.0 + delta[u];
        double su = sigma[u];
        for (int64_t k = offsets[u]; k < offsets[u + 1]; ++k) {
            int64_t v = col[k];
            /* v is a predecessor of u iff the arc is tight (the graph is symmetric,
             * so the arc u -> v carries the weight of v -> u) */
            if (dist[v] >= 0 && dist[v] + wgt[k] == du) {
                delta[v] += (sigma[v] / su) * coeff;
                ++dag;
            }
        }
    }
    if (out_maxd) *out_maxd = maxd;
    if (out_sigma_max) *out_sigma_max = smax;
    if (out_arcs_reached) *out_arcs_reached = arcs_reached;
    if (out_dag_arcs) *out_dag_arcs = dag;
    return reached;
}

/* stats: [0] reached, [1] largest distance + 1, [2] A_r, [3] T. */
int oracle_brandes_single_source_w(int64_t n, const int64_t *offsets, const int32_t *col,
                                   const int64_t *wgt, int64_t s, int64_t *dist, double *sigma,
                                   double *delta, double *sigma_max, int64_t *stats) {
    if (n <= 0 || s < 0 || s >= n) return 2;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    heap_item_t *heap = (heap_item_t *)malloc(sizeof(heap_item_t) * (size_t)(offsets[n] + 2));
    if (!order || !heap) {
        free(order), free(heap);
        return 1;
    }
    int64_t maxd = 0, ar = 0, dag = 0;
    int64_t reached = single_source_w(n, offsets, col, wgt, s, dist, sigma, delta, order, heap, &maxd,
                                      sigma_max, &ar, &dag);
    if (stats) {
        stats[0] = reached;
        stats[1] = maxd + 1;
        stats[2] = ar;
        stats[3] = dag;
    }
    free(order), free(heap);
    return 0;
}

int oracle_brandes_bc_w(int64_t n, const int64_t *offsets, const int32_t *col, const int64_t *wgt,
                        const int64_t *sources, int64_t k, double *bc, int nthreads,
                        int64_t *totals, double *sigma_max) {
    if (n <= 0) return 2;
    for (int64_t i = 0; i < k; ++i)
        if (sources[i] < 0 || sources[i] >= n) return 2;
    if (nthreads < 1) nthreads = 1;
    double *partial = (double *)calloc((size_t)nthreads * (size_t)n, sizeof(double));
    int64_t *tot = (int64_t *)calloc((size_t)nthreads * 4, sizeof(int64_t));
    double *smax = (double *)calloc((size_t)nthreads, sizeof(double));
    int failed = 0;
    if (!partial || !tot || !smax) {
        free(partial), free(tot), free(smax);
        return 1;
    }
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
#endif
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        int64_t *dist = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
        int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
        double *sigma = (double *)malloc(sizeof(double) * (size_t)n);
        double *delta = (double *)malloc(sizeof(double) * (size_t)n);
        heap_item_t *heap = (heap_item_t *)malloc(sizeof(heap_item_t) * (size_t)(offsets[n] + 2));
        int ok = dist && order && sigma && delta && heap;
        if (!ok) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
        }
        double *mine = partial + (size_t)t * (size_t)n;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t i = 0; i < k; ++i) {
            if (!ok) continue;
            int64_t s = sources[i], maxd = 0, ar = 0, dag = 0;
            double sm = 0.0;
            int64_t reached = single_source_w(n, offsets, col, wgt, s, dist, sigma, delta, order, heap,
                                              &maxd, &sm, &ar, &dag);
            for (int64_t v = 0; v < n; ++v)
                if (v != s) mine[v] += delta[v];
            tot[t * 4 + 0] += reached;
            tot[t * 4 + 1] += ar;
            tot[t * 4 + 2] += dag;
            if (maxd + 1 > tot[t * 4 + 3]) tot[t * 4 + 3] = maxd + 1;
            if (sm > smax[t]) smax[t] = sm;
        }
        free(dist), free(order), free(sigma), free(delta), free(heap);
    }
    for (int64_t v = 0; v < n; ++v) bc[v] = 0.0;
    for (int t = 0; t < nthreads; ++t)
        for (int64_t v = 0; v < n; ++v) bc[v] += partial[(size_t)t * (size_t)n + v];
    if (totals) {
        totals[0] = totals[1] = totals[2] = totals[3] = 0;
        for (int t = 0; t < nthreads; ++t) {
            totals[0] += tot[t * 4 + 0];
            totals[1] += tot[t * 4 + 1];
            totals[2] += tot[t * 4 + 2];
            if (tot[t * 4 + 3] > totals[3]) totals[3] = tot[t * 4 + 3];
        }
    }
    if (sigma_max) {
        *sigma_max = 0.0;
        for (int t = 0; t < nthreads; ++t)
            if (smax[t] > *sigma_max) *sigma_max = smax[t];
    }
    free(partial), free(tot), free(smax);
    return failed ? 1 : 0;
}

/* Masked multi-seed relaxation for unit weights (relax.py:42-103).
 *   mask      : uint8[n] (NULL = every vertex); arcs with an endpoint outside
 *               the mask are ignored (relax.py:83-84)
 *   seeds     : (seed_v[i], seed_d[i], seed_sigma[i]); a seed with d >= inf or
 *               sigma == 0 is skipped (relax.py:65-66); the smallest d wins and
 *               equal d adds sigma (relax.py:67-71)
 *   dist      : inf where unreached (inf = the reference's inf_distance)
 *   sigma     : base (if the seed distance survived) + sum over tight in-arcs,
 *               the invariant stated at relax.py:8-12
 * Returns 0, 1 (allocation) or 3 (seed outside the mask -> ContractViolation,
 * relax.py:52-55). */
int oracle_masked_relax(int64_t n, const int64_t *offsets, const int32_t *col, const uint8_t *mask,
                        int64_t nseeds, const int64_t *seed_v, const int64_t *seed_d,
                        const double *seed_sigma, int64_t inf, int64_t *dist, double *sigma) {
    if (mask)
        for (int64_t i = 0; i < nseeds; ++i)
            if (!mask[seed_v[i]]) return 3;
    double *base = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *nxt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    uint8_t *queued = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!base || !cur || !nxt || !order || !queued) {
        free(base), free(cur), free(nxt), free(order), free(queued);
        return 1;
    }
    for (int64_t v = 0; v < n; ++v) {
        dist[v] = inf;
        sigma[v] = 0.0;
    }
    for (int64_t i = 0; i < nseeds; ++i) {
        int64_t v = seed_v[i], d = seed_d[i];
        if (d >= inf || seed_sigma[i] == 0.0) continue;
        if (d < dist[v]) {
            dist[v] = d;
            base[v] = seed_sigma[i];
        } else if (d == dist[v]) {
            base[v] += seed_sigma[i];
        }
    }
    /* Level loop.  `cur` is the frontier at level d: every vertex whose
     * tentative distance is d when the loop arrives there, discovered through
     * an arc or seeded.  When a frontier dies out the loop jumps to the
     * smallest seed distance still waiting (seeds sit at staggered levels). */
    int64_t n_order = 0, n_cur = 0, d = 0;
    for (;;) {
        if (n_cur == 0) {
            int64_t best = inf;
            for (int64_t i = 0; i < nseeds; ++i) {
                int64_t v = seed_v[i];
                if (!queued[v] && dist[v] < best) best = dist[v];
            }
            if (best >= inf) break;
            d = best;
            for (int64_t i = 0; i < nseeds; ++i) {
                int64_t v = seed_v[i];
                if (!queued[v] && dist[v] == d) {
                    queued[v] = 1;
                    cur[n_cur++] = v;
                }
            }
        }
        for (int64_t i = 0; i < n_cur; ++i) order[n_order++] = cur[i];
        int64_t n_nxt = 0;
        for (int64_t i = 0; i < n_cur; ++i) {
            int64_t v = cur[i];
            for (int64_t k = offsets[v]; k < offsets[v + 1]; ++k) {
                int64_t w = col[k];
                if (mask && !mask[w]) continue;
                if (queued[w]) continue;
                if (d + 1 < dist[w]) {
                    dist[w] = d + 1;
                    base[w] = 0.0; /* strict improvement drops the seed base (relax.py:87-94) */
                }
                if (dist[w] == d + 1) {
                    queued[w] = 1;
                    nxt[n_nxt++] = w;
                }
            }
        }
        /* seeds whose own distance is exactly d + 1 join the next frontier */
        for (int64_t i = 0; i < nseeds; ++i) {
            int64_t v = seed_v[i];
            if (!queued[v] && dist[v] == d + 1) {
                queued[v] = 1;
                nxt[n_nxt++] = v;
            }
        }
        int64_t *tmp = cur;
        cur = nxt;
        nxt = tmp;
        n_cur = n_nxt;
        d += 1;
    }
    /* sigma in ascending distance order: base + tight in-arcs inside the mask. */
    for (int64_t i = 0; i < n_order; ++i) {
        int64_t w = order[i];
        double acc = base[w];
        for (int64_t k = offsets[w]; k < offsets[w + 1]; ++k) {
            int64_t v = col[k];
            if (mask && !mask[v]) continue;
            if (dist[v] < inf && dist[v] + 1 == dist[w]) acc += sigma[v];
        }
        sigma[w] = acc;
    }
    free(base), free(cur), free(nxt), free(order), free(queued);
    return 0;
}
