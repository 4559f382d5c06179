/*
 * bc_b200.h -- C ABI of the B200 betweenness-centrality engine.
 *
 * The reference (`hybir`) has no FFI: its boundary for this path is the Python
 * call `run_bc(g, cfg) -> RunResult` (reference pkg/src/hybir/engine.py:120-153)
 * plus the inspection entry points `forward_phase` / `backward_phase` /
 * `merge_states` (forward.py:188-196, backward.py:59-67, forward.py:275-284).
 * The functions below are what a binding for that path needs; every one cites
 * the reference interface it stands in for.  INTEGRATION.md shows the ctypes
 * stub a `hybir` maintainer would add.
 *
 * Conventions
 *   - plain pointers and sizes only; the caller owns every buffer it passes;
 *     the library copies the CSR to the device once per handle and never
 *     writes to caller inputs (reference SPEC.md:73: Graph is immutable);
 *   - return value: BC_OK, BC_ERR_INTERNAL (CUDA / allocation failure; maps to
 *     the reference's exit code 1) or BC_ERR_INPUT (bad argument; maps to
 *     `InputError`, exit code 2, reference cli.py:148-160);
 *     `bc_last_error()` returns the message;
 *   - one handle is driven by one host thread (reference is single-threaded);
 *     results are deterministic for a fixed (graph, sources, options);
 *   - unit weights by default; positive integer arc weights (int32) through bc_set_weights.
 *
 * There is no CPU implementation behind these entry points: if the CUDA
 * runtime or a device is missing, `bc_create` fails.
 */
#ifndef BC_B200_H
#define BC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BC_OK 0
#define BC_ERR_INTERNAL 1
#define BC_ERR_INPUT 2

/* Distance sentinel of bc_debug_sources (the Python shim maps it to the
 * reference's `g.inf_distance`, graph.py:34-38). */
#define BC_UNREACHED (-1)

/* Forward-phase algorithm, the reference's `RunConfig.mode` (engine.py:34,43). */
#define BC_MODE_DIRECT 0 /* whole graph = one partition: batched Brandes            */
#define BC_MODE_HYBIR 1  /* border-matrix refinement (forward.py:188-256)            */
#define BC_MODE_BSP 2    /* level-synchronous partitioned baseline (bsp.py:22-142)   */

typedef struct bc_handle bc_handle;

/* Counters of one bc_run* call.  The three traversal totals are the inputs of
 * the algorithmic-bytes formula of SURVEY.md section 8(d):
 * B = 16*arcs_reached + 32*dag_arcs + 72*reached + 20*n*sources. */
typedef struct bc_stats {
    int64_t sources;      /* sources processed                                         */
    int64_t batches;      /* source batches (32 * groups lanes each)                    */
    int64_t max_levels;   /* deepest BFS (eccentricity + 1) over all sources            */
    int64_t reached;      /* sum over sources of reached vertices  (n_r)                */
    int64_t arcs_reached; /* sum over sources of degrees of reached vertices (A_r)      */
    int64_t dag_arcs;     /* sum over sources of shortest-path DAG arcs (T)             */
    int64_t launches;     /* kernels launched by this call                              */
    int64_t h2d_bytes;    /* bytes copied host->device by this call                     */
    int64_t d2h_bytes;    /* bytes copied device->host by this call                     */
    double ms_total;      /* device time of the whole call (CUDA events on the stream)  */
    double ms_forward;    /* ... of the forward level kernels                           */
    double ms_backward;   /* ... of the backward level kernels                          */
    double ms_border;     /* ... of border refinement + sigma composition (hybir mode)  */
    /* per-source report totals, the reference's ForwardReport / BackwardReport
     * (forward.py:52-64, backward.py:33-43) summed over sources */
    int64_t iterations;   /* border refinement iterations                               */
    int64_t comm_events;  /* forward cross-partition transfers                          */
    int64_t sync_events;  /* backward cross-partition sync points                       */
    int64_t comm_bytes;   /* backward payload, 16 B per (sigma, delta) pair (ledger.py:12) */
    int64_t launches_forward;  /* kernels launched between the events that bound ms_forward  */
    int64_t launches_backward; /* ... ms_backward                                           */
    int64_t launches_level;    /* of those, launches of the dense level kernel (both directions) */
    double ms_level;           /* device time of those launches alone (level kernel + its hub pass;
                                  at most 512 launches per call are timed, launches_level_timed)   */
    int64_t launches_level_timed;
    /* batched byte model of those launches: what one launch has to move
     * when the 32 lanes of a group share every adjacency read */
    int64_t level_scan_arcs;    /* arcs scanned per (vertex, group): col_idx word + mask probe, 8 B */
    int64_t level_pairs;        /* (DAG arc, lane) pairs gathered: one fp64 of sigma / coef, 8 B      */
    int64_t level_vertex_lanes; /* fp64 values read or written per (vertex, lane), 8 B each          */
    int64_t level_dense_words;  /* level / visited mask words swept per (vertex, group), 4 B each    */
    int64_t level_entries;      /* (vertex, group) entries of the backward launches: 16 B BC partial */
    int64_t level_model_bytes;  /* the sum in bytes, plus 8 B of row offsets per vertex and launch; 0
                                   unless option "model_counters" is on (one more atomic per work item) */
    int64_t lookahead_batches;  /* batches whose Step 1 ran ahead, beside the previous border phase  */
} bc_stats;

/* Replaces: construction of the device-side view of `Graph`
 * (graph.py:21-61: offsets int64[n+1]; arc_dst as int32 col_idx[n_arcs], arcs
 * sorted by (src, dst), both directions present).  `device` is a CUDA ordinal. */
int bc_create(int64_t n, int64_t n_arcs, const int64_t *offsets, const int32_t *col_idx,
              int device, bc_handle **out);

/* Positive integer arc weights, int32[n_arcs] in CSR arc order (`Graph.arc_weight`,
 * graph.py:21-61; both directions of an edge carry the same weight).  NULL or
 * all-ones selects the unit-weight kernels.  With weights up to 4096 a level is a
 * distance value: the forward sweep is the reference's Dijkstra order (relax.py:75-101,
 * oracle.py:44-61) taken one distance at a time, in every mode.  Larger weights
 * (DIMACS road graphs, graph.py:139-173), or low-degree graphs with weights above 16
 * where a level per distance value is out of reach, take the general-weight sweeps of
 * csrc/bc_sssp.cuh -- label-correcting distances, then path counts and dependencies in
 * dependency-counted order -- in BC_MODE_DIRECT only (option "sssp" overrides the
 * choice).  Same results: dist and sigma exact, delta / BC to 1e-9. */
int bc_set_weights(bc_handle *h, const int32_t *weights);

/* Tuning knobs ("groups": 32-lane source groups per batch; "item_arcs": arcs
 * per warp work item; "reports": 1 = keep per-source report counters;
 * "sparse" / "deep": frontier-queue levels / persistent multi-level sweeps;
 * "hybir_queues": 1 = BC_MODE_HYBIR sweeps of low-degree graphs run on frontier
 * queues with the Step-6 border seeds joining the queue levels, 0 = dense level
 * rows; "row_cache": 1 = sigma / coef row gathers allocate in L1, 0 = bypass
 * L1, -1 (default) = chosen from the degree skew of the graph; "lookahead": 1 =
 * BC_MODE_HYBIR issues Step 1 of the next source batch on a second stream while
 * the border phase of the current batch runs (`pipeline_sources`, engine.py:135-143,
 * 156-161); "l2_fetch": 32 / 64 / 128, L2 fill granularity of the device;
 * "model_counters": 1 = the forward pulls count the arcs they scan, which completes
 * bc_stats.level_model_bytes (bench.py turns it on for one untimed step);
 * "deep_compact": 1 (default) = deep (road-like) graphs sweep over level-ordered path
 * counts with one atomically updated BC vector per batch, 2 = same with per-group BC
 * partials, 0 = row layout everywhere;
 * "relabel": unpartitioned unit-weight runs sweep a copy of the graph renumbered by
 * descending degree (csrc/bc_relabel.cuh; sources and the BC vector keep the caller's ids):
 * 1 = from the first run, 0 = never, -1 (default) = graphs whose largest degree exceeds 16
 * average degrees, once the handle has been given 2048 sources;
 * "sssp": weighted graphs, 1 = general-weight sweeps (csrc/bc_sssp.cuh), 0 = one level
 * per distance value (weights up to 4096), -1 (default) = by weight range;
 * "sssp_delta": step of the near-far distance bound there (0 = 16 mean arc weights);
 * "bwd_push": direction switch of the dependency sweep (csrc/bc_bwd_push.cuh): a backward level
 * is driven by its children (atomic adds into the parents' sums) when the children's arcs
 * times this factor do not exceed the parents' arcs; default 16, 0 = every level parent-driven
 * (sums in CSR arc order: BC reproducible bit for bit from run to run);
 * "push_beta", "push_beta_late", "reorder": see csrc/bc_engine.cu). */
int bc_set_option(bc_handle *h, const char *key, int64_t value);

/* Replaces: `Partition` + `identify_borders` + `compute_border_matrices`
 * (partition.py:26-61,139-154; border_matrix.py:48-67) for k >= 1 parts.
 * assignment[v] in [0, k).  Builds the cut-arc-free CSR, the border lists
 * (ascending vertex id per part, partition.py:148) and, for BC_MODE_HYBIR,
 * the per-part border distance / path-count tables. */
int bc_set_partition(bc_handle *h, int k, const int32_t *assignment);

/* Replaces: the source loop of `run_bc` (engine.py:132-149) including
 * `accumulate_bc` (backward.py:154-158): bc_out[v] = sum over sources s != v of
 * delta_s[v].  Host buffers in, host buffer out (the end-to-end call). */
int bc_run(bc_handle *h, int mode, const int64_t *sources, int64_t n_sources, double *bc_out,
           bc_stats *stats);

/* Same, but accumulates into a caller-owned DEVICE vector bc_dev[n] (+=) on
 * the CUDA stream `stream` (a cudaStream_t; NULL = default stream).  Used by
 * the multi-GPU host code, which all-reduces bc_dev with NCCL afterwards. */
int bc_run_device(bc_handle *h, int mode, const int64_t *sources, int64_t n_sources,
                  double *bc_dev, void *stream, bc_stats *stats);

/* Replaces: the inspection path `forward_phase` + `merge_states` +
 * `backward_phase` (forward.py:188, 275; backward.py:59) for k sources at once.
 * Outputs are [k][n] row-major host arrays: dist (BC_UNREACHED where
 * unreached), sigma (0 where unreached), delta (including delta[s] of the
 * source itself, backward.py:76-77).  Any output pointer may be NULL. */
int bc_debug_sources(bc_handle *h, int mode, const int64_t *sources, int64_t k, int32_t *dist,
                     double *sigma, double *delta);

/* Per-source reports of the last bc_run* / bc_debug_sources call, 8 int64 per
 * source: iterations, comm_events, max_level[0], max_level[1], sync_events,
 * comm_bytes, levels[0], levels[1] (forward.py:52-64, backward.py:33-43;
 * the two-element fields are defined for k = 2 partitions). */
int bc_get_reports(bc_handle *h, int64_t *out, int64_t n_sources);

/* Border inspection for tests (border_matrix.py:25-45, partition.py:47-61):
 * counts[k]; then per part p: borders (vertex ids), bm (int32, BC_UNREACHED =
 * unreachable inside the part) and sm (fp64) as b_p x b_p row-major. */
int bc_get_border_counts(bc_handle *h, int64_t *counts);
int bc_get_border_tables(bc_handle *h, int part, int32_t *borders, int32_t *bm, double *sm);

/* Install the border table of `part` from host arrays (b_p x b_p row-major; bm with
 * BC_UNREACHED = unreachable): the border-table disk cache of the reference
 * (`load_border_matrices`, border_matrix.py:109-125) hands cached tables back
 * through this call instead of recomputing them.  Once every part is set, BC_MODE_HYBIR
 * runs use them as they are. */
int bc_set_border_tables(bc_handle *h, int part, const int32_t *bm, const double *sm);

/* Border frontier of the LAST batch of the last BC_MODE_HYBIR call, the
 * reference's `BorderFrontier` (forward.py:45-48): for each of the first
 * `n_lanes` sources of that batch, refined distance (BC_UNREACHED = inf), path
 * count and arrival count of every border, [B][n_lanes] row-major with
 * borders in part order. */
int bc_get_border_frontier(bc_handle *h, int64_t n_lanes, int32_t *dist, double *sigma,
                           double *arrival);

/* ---- graph-partitioned multi-GPU mode: one rank = one part = one GPU -------
 * The handle is created on the rank's LOCAL graph: its own vertices first, then its halo (the
 * other parts' border vertices its cut arcs reach, with empty rows) and one catch-all vertex
 * per other part for borders it has no arc to; the host code numbers them
 * (paper_2008_05718_b200/partitioned.py: local_graph).  State arrays are therefore sized
 * owned + halo, not n.  The host code (one process per GPU, torch.distributed) drives a batch
 * and moves the exported buffers with NCCL; these calls are the device side of the reference's
 * cross-worker transfers (bsp.py:83-87,128-135, backward.py:121-139, ledger.py:28-31).
 * `assignment` maps every local vertex to its part; border_off[world+1] / border_v list every
 * rank's border vertices in local ids (ascending global ids per rank, partition.py:148). */
int bc_dist_setup(bc_handle *h, int rank, int world, const int32_t *assignment,
                  const int64_t *border_off, const int32_t *border_v);
/* Cut arcs of this rank's own borders: far ends cut_dst[cut_off[j] .. cut_off[j+1]) (local halo
 * ids) of border j -- the arcs `_cross_dependencies` walks (backward.py:46-56). */
int bc_dist_set_cut_arcs(bc_handle *h, const int64_t *cut_off, const int32_t *cut_dst);
/* Start a batch of `count` sources (<= 32 * groups, local ids; -1 = the source is neither owned
 * by this rank nor in its halo: the lane exists, nothing is planted here). */
int bc_dist_begin(bc_handle *h, const int64_t *sources, int64_t count, void *stream);
/* Local work of forward level L (pull from level L-1) / backward level L. */
int bc_dist_forward_level(bc_handle *h, int level, void *stream);
int bc_dist_backward_level(bc_handle *h, int level, int deepest, void *stream);
/* Export this rank's border state of `level`: masks_dev[nb * groups] u32 (what = 0
 * only reads them back into the scan), then values_dev[*count_out] fp64 of
 * what = 1 (sigma, forward) or 2 (coef, backward).  Buffers are device memory. */
int bc_dist_export(bc_handle *h, int level, int what, void *masks_dev, void *values_dev,
                   int64_t value_capacity, int64_t *count_out, void *stream);
/* Import rank `from`'s border state of `level` (forward: masks + sigma, also marks
 * the lanes visited; backward: coef under the masks exported on the way forward). */
int bc_dist_import(bc_handle *h, int level, int what, int from, const void *masks_dev,
                   const void *values_dev, void *stream);
/* Backward exchange at the paper's minimal sync points (backward.py:46-56,121-139).  After the
 * forward phase of a batch, ONE call lists -- level by level -- the (border, lanes) values of
 * this rank that a vertex of another part will pull: counts_out[2 L] entries and
 * counts_out[2 L + 1] fp64 values at level L.  Levels where no rank has an entry need no
 * exchange.  pack / unpack move exactly the listed values of one level through a message of
 * [cap_values fp64][3 x cap_entries int32] (the caps are the maxima over ranks, so every rank
 * sends the same size and one all-gather moves them); nothing in the per-level path reads
 * back to the host. */
int bc_dist_plan_backward(bc_handle *h, int depth, int64_t *counts_out, void *stream);
int bc_dist_pack(bc_handle *h, int level, void *send_dev, int64_t cap_entries, int64_t cap_values,
                 void *stream);
int bc_dist_unpack(bc_handle *h, int level, int from, const void *recv_dev, int64_t cap_entries,
                   int64_t cap_values, int64_t n_entries, void *stream);
/* Unpack every peer's message of one level in ONE launch out of the all-gathered buffer
 * (world x words_per_rank int64 words); the entry counts are read on the device from the
 * all-gathered plan table plan_dev[world][depth][2] (what bc_dist_plan_backward returned, gathered). */
int bc_dist_unpack_all(bc_handle *h, int level, const void *recv_dev, int64_t words_per_rank,
                       int64_t cap_entries, int64_t cap_values, const int64_t *plan_dev, int depth,
                       void *stream);
/* Kernel launches, CUDA-event time of the dense level kernel and its byte model since the last
 * call (drains the device). */
int bc_dist_get_stats(bc_handle *h, bc_stats *stats);
/* live[level][g] (lanes with a non-empty frontier), read / overwrite with the OR over ranks. */
int bc_dist_get_live(bc_handle *h, int level, uint32_t *live_out, void *stream);
int bc_dist_set_live(bc_handle *h, int level, const uint32_t *live, void *stream);
/* bc_dev[v] += BC partials of the vertices this rank owns (others untouched). */
int bc_dist_finish(bc_handle *h, double *bc_dev, void *stream);

/* ---- the paper's border-matrix forward phase across ranks (forward.py:188-256 with one part per
 * GPU).  Every rank keeps ALL parts' border tables and runs the border refinement and the
 * path-count composition redundantly, so the forward phase of a batch costs ONE exchange (the
 * Step-1 seeds) instead of one per level; the backward phase uses bc_dist_backward_level /
 * export / import as above.  Call order per batch: step1 -> (all-reduce the two seed arrays:
 * MIN on distances, MAX on path counts) -> forward -> (all-reduce MAX of the depth) -> set_depth. */
/* Global cut arcs: for border j (rank-major order of bc_dist_setup) the borders
 * cin_src[cin_off[j] .. cin_off[j+1]) on the other side of its cut arcs; cin_w NULL = unit
 * weights.  Builds the cut-free CSR of this rank's part and the border table of its own part. */
int bc_dist_hybir_setup(bc_handle *h, const int64_t *cin_off, const int32_t *cin_src,
                        const int32_t *cin_w);
/* Border table of `part` (b_p x b_p distances and path counts, border_matrix.py:48-67) out of /
 * into device buffers: each rank publishes its own part's table once. */
int bc_dist_hybir_get_table(bc_handle *h, int part, int32_t *bm_dev, double *sm_dev);
int bc_dist_hybir_set_table(bc_handle *h, int part, const int32_t *bm_dev, const double *sm_dev);
/* Entries of the seed arrays: total borders x 32 x groups. */
int64_t bc_dist_hybir_seed_count(bc_handle *h);
/* Step 1 of a batch (BFS inside this rank's part from the sources it owns; source_part[i] = part
 * of source i, whichever rank holds it); writes the border seeds [border][lane] (distance,
 * 0x3fffffff = unreached; path count) into device buffers. */
int bc_dist_hybir_seeds(bc_handle *h, const int64_t *sources, const int32_t *source_part, int64_t count,
                        int32_t *seed_dist_dev, double *seed_sigma_dev, void *stream);
/* Steps 2-5 + path-count composition on the reduced seeds (identical on every rank), then Step 6
 * on this rank's part.  depth_out = levels seen by this rank; iterations_out = refinement
 * iterations summed over the batch's sources. */
int bc_dist_hybir_forward(bc_handle *h, const int32_t *seed_dist_dev, const double *seed_sigma_dev,
                          int *depth_out, int64_t *iterations_out, void *stream);
/* The same forward phase with ONE border table per rank (memory b_p^2 x 12 B instead of the sum
 * over all parts; the min-plus closure and the composition of a part run on its owner only).
 * bc_dist_hybir_shard_tables drops the other parts' tables after bc_dist_hybir_setup.  A batch is
 * then driven step by step, the caller all-reducing the exchange buffers between the steps
 * (xchg_values: B x 32 x groups int32 distances [MIN] in steps 1-2, fp64 path counts [MAX] in steps
 * 4-5; xchg_flags: 32 x groups u32 "lane changed" words [MAX]):
 *   0 begin refinement from the reduced seeds       1 refinement iteration -> exchange buffers
 *   2 merged buffers -> state; *flag_out = some lane is still active (NULL: do not read back)
 *   3 begin composition                              4 composition round -> exchange buffers
 *   5 merged buffers -> state; *flag_out = some path count changed
 *   6 Step 6 on this rank's part; *flag_out = levels seen by this rank */
int bc_dist_hybir_shard_tables(bc_handle *h);
int bc_dist_hybir_border_step(bc_handle *h, int step, void *xchg_values_dev, void *xchg_flags_dev,
                              const int32_t *seed_dist_dev, const double *seed_sigma_dev, int *flag_out,
                              void *stream);
/* Extend this rank's level rows (empty) to the depth of the deepest rank. */
int bc_dist_hybir_set_depth(bc_handle *h, int global_depth, void *stream);

const char *bc_last_error(bc_handle *h);
/* Releases the handle.  Its device blocks go to a per-device cache that the next
 * bc_create / bc_run reuses (run_bc() opens one handle per call, as the
 * reference's run_bc builds its state per call, engine.py:120-131; without the
 * cache every call pays cudaMalloc + cudaFree of the multi-GB batch state). */
void bc_destroy(bc_handle *h);
/* Hands every cached device block back to the CUDA driver. */
void bc_release_cached_memory(void);

#ifdef __cplusplus
}
#endif
#endif /* BC_B200_H */
