// bc_sssp.cuh -- Brandes sweeps for arbitrary positive integer arc weights (
// relax.py:75-101 is the reference's Dijkstra with path-count re-relaxation, oracle.py:29-67 its
// single-source oracle, backward.py:95-103 the dependency rule).
//
// The unit-weight and small-weight kernels (bc_kernels.cuh) take one level per distance value;
// with DIMACS-style weights (10^3 .. 10^6 per arc) a level per distance is millions of launches
// and one mask array each.  This path does not order the work by distance at all:
//
//   A  label-correcting distances, near-far style: a (vertex, source) pair whose distance dropped
//      is dirty; dirty pairs below a threshold push dist + w to their neighbours with a 64-bit
//      atomic min, the others wait.  When a round finds nothing below the threshold, the threshold
//      moves to the smallest waiting distance plus a step (16 mean arc weights); when nothing is
//      dirty the distances are final -- the same array Dijkstra produces.  Every round works out
//      its threshold from what the previous round recorded, so there is no host round trip and
//      no control kernel in between.
//   B  one pass over the arcs counts, per (vertex, source), the arcs that are tight towards it
//      (shortest-path parents, dist[u] + w = dist[v]) and away from it (children).
//   C  path counts in topological order of the shortest-path DAG without sorting it: a
//      (vertex, source) pair is ready when its parent count has dropped to zero; a ready pair
//      adds up its parents' counts in arc order (a pull: no floating-point atomics, the sum
//      does not depend on scheduling) and takes one off the parent count of each child.
//   D  dependencies the same way from the leaves: a pair is ready when its child count is
//      zero, pulls coef = (1 + delta) / sigma from its children (backward.py:95-103 with the
//      division hoisted, as in finalize_backward) and releases its parents.
//
// 32 sources share a warp as everywhere else: per group g, rows [v][32] of dist / sigma / coef /
// counts, one 32-bit lane mask per vertex for "in this round's frontier" and a queue of the
// vertices whose mask is not empty (a vertex enters when its mask goes from zero to non-zero).
// Rounds of C and D are as many as the DAG is deep in arcs; every round is one launch over the
// queue, and a launch whose predecessor produced nothing returns at once (the host launches
// rounds in chunks and reads the flags afterwards, as forward_sweep does).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "bc_kernels.cuh"   // kFull, warp_sum

namespace bcb200 {

constexpr long long kSsspInf = (long long)1 << 62;

struct SsspParams {
    const int64_t *off;
    const int32_t *col;
    const int32_t *wgt;
    int64_t n;
    long long *dist;   // [G][n][32]
    double *sigma;     // [G][n][32]
    double *coef;      // [G][n][32]
    double *delta;     // [G][n][32] or nullptr (inspection runs)
    int *npar;         // [G][n][32] tight arcs into the pair still to be accounted for
    int *nchild;       // [G][n][32] tight arcs out of the pair still to be accounted for
    uint32_t *cur;     // [G][n] lanes in this round's frontier (cleared as they are consumed)
    uint32_t *next;    // [G][n] lanes in the next round's frontier
    uint32_t *leaf;    // [G][n] pairs without children (phase B -> first frontier of phase D)
    // frontier queues: the vertices whose word in cur / next is not zero, in the order they got there
    int32_t *q_cur;    // [G][n]
    int32_t *q_next;   // [G][n]
    int32_t *q_leaf;   // [G][n] (phase B -> first queue of phase D)
    int *q_count;      // [3][G] queue lengths, rotating: this round reads slot qs_in, fills qs_out, clears qs_zero
    int *q_leaf_count; // [G]
    int qs_in, qs_out, qs_zero;
    int G;             // groups the state arrays were sized for (stride of q_count)
    double *bcg;       // [G][n] BC partial of the group
    int *flags;        // flags[r] != 0: round r put something into `next`
    int round;
    // phase A only: threshold[r] = distance bound of round r, far_min[r] = smallest distance a
    // pair above the bound was left waiting with in round r, step = how far the bound moves
    long long *threshold;
    long long *far_min;
    long long step;
    int accumulate;    // phase D: add delta into bcg
    unsigned long long *counters;   // reached pairs, arcs at reached pairs, DAG arcs (bc_stats)
};

constexpr int kSsspWarps = 4;
// A warp takes 32 queue entries at a time: lane i holds vertex myv and its frontier mask (consumed:
// the word is cleared so the mask array is empty when it becomes `next` again).  Scanning the
// whole mask array every round instead (the first version) cost 0.7 us of load latency per
// 32-vertex chunk and warp slot, empty or not: ~100 us per round on a 1024^2 grid with four groups.
constexpr int kSsspChunk = 32;

__device__ __forceinline__ void sssp_take_items(const SsspParams &p, size_t g, int lane, int base, int count,
                                                int32_t &myv, uint32_t &mask) {
    myv = -1;
    mask = 0;
    if (base + lane < count) {
        myv = p.q_cur[g * p.n + base + lane];
        uint32_t *w = p.cur + g * p.n + myv;
        mask = *w;
        *w = 0;
    }
}

// Round prologue: false = the sweep ended before this round.  One thread clears the queue length
// slot nobody uses in this round (it was the input of the previous one).
__device__ __forceinline__ bool sssp_round_begin(const SsspParams &p, size_t g, int &count) {
    if (p.round > 0 && p.flags[p.round - 1] == 0) return false;
    count = p.q_count[p.qs_in * p.G + g];
    if (blockIdx.x == 0 && threadIdx.x == 0) p.q_count[p.qs_zero * p.G + g] = 0;
    return true;
}

// lanes `bits` of vertex w join the next frontier
__device__ __forceinline__ void sssp_push(const SsspParams &p, size_t g, int32_t w, uint32_t bits) {
    if (atomicOr(p.next + g * p.n + w, bits) == 0) {
        const int pos = atomicAdd(p.q_count + p.qs_out * p.G + g, 1);
        p.q_next[g * p.n + pos] = w;
    }
}

// Sparse frontiers (a road network: a couple of sources per frontier vertex) leave most lanes of
// a row-per-vertex visit idle while the warp walks its frontier vertices one after the other, each
// visit a chain of dependent loads.  When a chunk holds fewer than kSsspPairLanes frontier pairs
// per frontier vertex, its pairs are dealt out one per thread instead: every chain runs at once.
constexpr int kSsspPairLanes = 16;

struct ChunkPairs {
    int total;    // frontier pairs in the chunk
    int excl;     // pairs of the vertices before this lane's vertex
    uint32_t mask;
    int32_t myv;  // this lane's vertex
    // pair t of the chunk -> its vertex and source lane (all threads call it)
    __device__ __forceinline__ bool get(int t, int64_t &vertex, int &src_lane) const {
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int cand = lo + step;
            const int e = __shfl_sync(kFull, excl, cand & 31);
            if (e <= t) lo = cand;
        }
        const uint32_t m = __shfl_sync(kFull, mask, lo);
        const int first = __shfl_sync(kFull, excl, lo);
        vertex = __shfl_sync(kFull, myv, lo);
        if (t >= total) return false;
        src_lane = (int)__fns(m, 0, t - first + 1);
        return true;
    }
};

__device__ __forceinline__ ChunkPairs chunk_pairs(uint32_t mask, int32_t myv, int lane) {
    ChunkPairs c;
    const int mine = __popc(mask);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    c.excl = incl - mine;
    c.total = __shfl_sync(kFull, incl, 31);
    c.mask = mask;
    c.myv = myv;
    return c;
}

// A pair's visit is a chain of dependent loads per arc (neighbour id -> its distance -> its value
// or counter); arcs are taken kSsspArcBatch at a time so the chains of a batch overlap.
constexpr int kSsspArcBatch = 4;

struct ArcBatch {
    int32_t w[kSsspArcBatch];
    int32_t wt[kSsspArcBatch];
    long long dw[kSsspArcBatch];
    int cnt;
    __device__ __forceinline__ void load(const SsspParams &p, const long long *dist, int64_t a, int64_t a1, int sl) {
        cnt = (int)min((int64_t)kSsspArcBatch, a1 - a);
#pragma unroll
        for (int j = 0; j < kSsspArcBatch; ++j) {
            w[j] = 0;
            wt[j] = 0;
            if (j < cnt) {
                w[j] = __ldg(p.col + a + j);
                wt[j] = __ldg(p.wgt + a + j);
            }
        }
#pragma unroll
        for (int j = 0; j < kSsspArcBatch; ++j) dw[j] = j < cnt ? dist[(size_t)w[j] * 32 + sl] : kSsspInf;
    }
};

__global__ void fill_i64_kernel(long long *p, size_t count, long long value) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
        p[i] = value;
}

// dist = inf everywhere, frontier masks empty.
__global__ void sssp_init_kernel(long long *dist, uint32_t *cur, uint32_t *next, uint32_t *leaf,
                                 int64_t n) {
    const size_t g = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * 32;
         i += (int64_t)gridDim.x * blockDim.x)
        dist[g * n * 32 + i] = kSsspInf;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        cur[g * n + v] = 0;
        next[g * n + v] = 0;
        leaf[g * n + v] = 0;
    }
}

// Sources: distance 0, in the first frontier of phase A.
__global__ void sssp_seed_kernel(const int64_t *src, int count, int64_t n, long long *dist, uint32_t *cur,
                                 int32_t *q_cur, int *q_count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const size_t g = i >> 5;
    const int lane = i & 31;
    const int64_t v = src[i];
    if (v < 0) return;
    dist[(g * n + v) * 32 + lane] = 0;
    if (atomicOr(cur + g * n + v, 1u << lane) == 0) q_cur[g * n + atomicAdd(q_count + g, 1)] = (int32_t)v;
}

// Phase A, one round: dirty pairs below the round's distance bound relax their arcs; the others
// stay dirty.  flags[r] != 0 while anything is dirty after round r.
__global__ void __launch_bounds__(kSsspWarps * 32) sssp_relax_kernel(const SsspParams p) {
    const size_t g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    long long bound = p.threshold[0];
    int count;
    if (!sssp_round_begin(p, g, count)) return;   // nothing dirty: the distances are final
    if (p.round > 0) {
        bound = p.threshold[p.round - 1];
        // the previous round relaxed nothing: move the bound past the nearest waiting pair
        if (p.flags[p.round - 1] == 1) bound = p.far_min[p.round - 1] + p.step;
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) p.threshold[p.round] = bound;
    }
    long long *dist = p.dist + g * p.n * 32;
    int produced = 0;             // 2: relaxed something, 1: left pairs waiting
    long long waiting = kSsspInf;  // smallest distance left waiting (this lane)
    for (int base = (blockIdx.x * kSsspWarps + (threadIdx.x >> 5)) * 32; base < count;
         base += gridDim.x * kSsspWarps * 32) {
        int32_t myv;
        uint32_t mask;
        sssp_take_items(p, g, lane, base, count, myv, mask);
        unsigned need = __ballot_sync(kFull, mask != 0);
        if (need == 0) continue;
        const ChunkPairs cp = chunk_pairs(mask, myv, lane);
        if (__popc(need) > 1 && cp.total < kSsspPairLanes * __popc(need)) {
            // ---- one dirty pair per thread
            for (int t0 = 0; t0 < cp.total; t0 += 32) {
                int sl;
                int64_t u;
                if (!cp.get(t0 + lane, u, sl)) continue;
                const long long du = dist[u * 32 + sl];
                if (du >= bound) {
                    sssp_push(p, g, (int32_t)u, 1u << sl);   // still dirty next round
                    waiting = min(waiting, du);
                    produced |= 1;
                    continue;
                }
                produced |= 2;
                const int64_t a1 = p.off[u + 1];
                for (int64_t a = p.off[u]; a < a1; a += kSsspArcBatch) {
                    ArcBatch ab;
                    ab.load(p, dist, a, a1, sl);
                    long long old[kSsspArcBatch];
#pragma unroll
                    for (int j = 0; j < kSsspArcBatch; ++j) {
                        old[j] = 0;
                        if (j < ab.cnt && du + ab.wt[j] < ab.dw[j])
                            old[j] = atomicMin(dist + (size_t)ab.w[j] * 32 + sl, du + ab.wt[j]);
                    }
#pragma unroll
                    for (int j = 0; j < kSsspArcBatch; ++j)
                        if (j < ab.cnt && du + ab.wt[j] < ab.dw[j] && du + ab.wt[j] < old[j])
                            sssp_push(p, g, ab.w[j], 1u << sl);
                }
            }
            continue;
        }
        while (need) {
            const int i = __ffs(need) - 1;
            need &= need - 1;
            const int64_t u = __shfl_sync(kFull, myv, i);
            const uint32_t mu = __shfl_sync(kFull, mask, i);
            const bool dirty = (mu >> lane) & 1u;
            const long long du = dirty ? dist[u * 32 + lane] : kSsspInf;
            const bool on = dirty && du < bound;
            const unsigned far = __ballot_sync(kFull, dirty && !on);
            if (far) {
                if (lane == 0) sssp_push(p, g, (int32_t)u, far);   // still dirty next round
                if (dirty && !on) waiting = min(waiting, du);
                produced |= 1;
            }
            if (!__any_sync(kFull, on)) continue;
            produced |= 2;   // (a relaxation round, whether or not a distance dropped)
            const int64_t a0 = p.off[u], a1 = p.off[u + 1];
            for (int64_t base = a0; base < a1; base += 32) {
                int32_t my_w = 0, my_wt = 0;
                if (base + lane < a1) {
                    my_w = __ldg(p.col + base + lane);
                    my_wt = __ldg(p.wgt + base + lane);
                }
                const int cnt = (int)min((int64_t)32, a1 - base);
                for (int j = 0; j < cnt; ++j) {
                    const int32_t w = __shfl_sync(kFull, my_w, j);
                    const int32_t wt = __shfl_sync(kFull, my_wt, j);
                    bool better = false;
                    if (on) {
                        const long long cand = du + wt;
                        long long *d = dist + (size_t)w * 32 + lane;
                        if (cand < *d) better = cand < atomicMin(d, cand);
                    }
                    const unsigned b = __ballot_sync(kFull, better);
                    if (b && lane == 0) sssp_push(p, g, w, b);
                }
            }
        }
    }
    produced = __reduce_or_sync(kFull, (unsigned)produced);
    if (produced & 1) {
        for (int o = 16; o > 0; o >>= 1) waiting = min(waiting, __shfl_xor_sync(kFull, waiting, o));
        if (lane == 0) atomicMin(p.far_min + p.round, waiting);
    }
    // 2 = pairs were relaxed (what they improved is dirty now), 1 = only waiting pairs
    if (produced && lane == 0) atomicMax(p.flags + p.round, (produced & 2) ? 2 : 1);
}

// Phase B: parent / child counts of every reached pair, the first frontiers of phases C (the
// sources: distance 0) and D (pairs without children), sigma = 1 at the sources, and the
// traversal counters of bc_stats.
__global__ void __launch_bounds__(kSsspWarps * 32) sssp_count_kernel(const SsspParams p) {
    const size_t g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t chunk = (int64_t)blockIdx.x * kSsspWarps + (threadIdx.x >> 5);
    const int64_t v0 = chunk * 32;
    if (v0 >= p.n) return;
    const long long *dist = p.dist + g * p.n * 32;
    const int nv = (int)min((int64_t)32, p.n - v0);
    uint32_t src_mask = 0, leaf_mask = 0;   // of vertex v0 + lane
    unsigned long long c_reached = 0, c_arcs = 0, c_dag = 0;
    for (int i = 0; i < nv; ++i) {
        const int64_t v = v0 + i;
        const long long dv = dist[v * 32 + lane];
        const bool on = dv < kSsspInf;
        int np = 0, nc = 0;
        const int64_t a0 = p.off[v], a1 = p.off[v + 1];
        if (__any_sync(kFull, on)) {
            for (int64_t base = a0; base < a1; base += 32) {
                int32_t my_w = 0, my_wt = 0;
                if (base + lane < a1) {
                    my_w = __ldg(p.col + base + lane);
                    my_wt = __ldg(p.wgt + base + lane);
                }
                const int cnt = (int)min((int64_t)32, a1 - base);
                for (int j = 0; j < cnt; ++j) {
                    const int32_t w = __shfl_sync(kFull, my_w, j);
                    const int32_t wt = __shfl_sync(kFull, my_wt, j);
                    if (on) {
                        const long long dw = dist[(size_t)w * 32 + lane];
                        np += dw + wt == dv;
                        nc += dv + wt == dw;
                    }
                }
            }
        }
        p.npar[(g * p.n + v) * 32 + lane] = np;
        p.nchild[(g * p.n + v) * 32 + lane] = nc;
        const unsigned srcs = __ballot_sync(kFull, on && dv == 0);
        const unsigned leaves = __ballot_sync(kFull, on && nc == 0);
        if (lane == i) {
            src_mask = srcs;
            leaf_mask = leaves;
        }
        if (on && dv != 0) {
            ++c_reached;
            c_arcs += (unsigned long long)(a1 - a0);
            c_dag += (unsigned long long)np;
        }
    }
    if (lane < nv) {
        p.cur[g * p.n + v0 + lane] = src_mask;
        p.leaf[g * p.n + v0 + lane] = leaf_mask;
        if (src_mask) p.q_cur[g * p.n + atomicAdd(p.q_count + p.qs_in * p.G + g, 1)] = (int32_t)(v0 + lane);
    }
    {
        // leaves in one reservation per warp
        const unsigned has = __ballot_sync(kFull, leaf_mask != 0);
        int qbase = 0;
        if (lane == 0 && has) qbase = atomicAdd(p.q_leaf_count + g, __popc(has));
        qbase = __shfl_sync(kFull, qbase, 0);
        if (leaf_mask) p.q_leaf[g * p.n + qbase + __popc(has & ((1u << lane) - 1u))] = (int32_t)(v0 + lane);
    }
    c_reached = __reduce_add_sync(kFull, (unsigned)c_reached);
    // (per-lane partials are below 2^32 only for the first; the others go through 64-bit adds)
    for (int o = 16; o > 0; o >>= 1) {
        c_arcs += __shfl_xor_sync(kFull, c_arcs, o);
        c_dag += __shfl_xor_sync(kFull, c_dag, o);
    }
    if (lane == 0 && c_reached) {
        atomicAdd(p.counters + 0, c_reached);
        atomicAdd(p.counters + 1, c_arcs);
        atomicAdd(p.counters + 2, c_dag);
    }
}

// Phase C, one round: ready pairs add up their parents' path counts and release their children.
__global__ void __launch_bounds__(kSsspWarps * 32) sssp_forward_kernel(const SsspParams p) {
    const size_t g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    int count;
    if (!sssp_round_begin(p, g, count)) return;   // the sweep ended before this round
    bool produced = false;
    const long long *dist = p.dist + g * p.n * 32;
    double *sigma = p.sigma + g * p.n * 32;
    int *npar = p.npar + g * p.n * 32;
    for (int base = (blockIdx.x * kSsspWarps + (threadIdx.x >> 5)) * 32; base < count;
         base += gridDim.x * kSsspWarps * 32) {
        int32_t myv;
        uint32_t mask;
        sssp_take_items(p, g, lane, base, count, myv, mask);
        unsigned need = __ballot_sync(kFull, mask != 0);
        if (need == 0) continue;
        const ChunkPairs cp = chunk_pairs(mask, myv, lane);
        if (__popc(need) > 1 && cp.total < kSsspPairLanes * __popc(need)) {
            // ---- one ready pair per thread (same arc order, so the same sums)
            for (int t0 = 0; t0 < cp.total; t0 += 32) {
                int sl;
                int64_t v;
                if (!cp.get(t0 + lane, v, sl)) continue;
                const long long dv = dist[v * 32 + sl];
                double acc = 0.0;
                const int64_t a1 = p.off[v + 1];
                for (int64_t a = p.off[v]; a < a1; a += kSsspArcBatch) {
                    ArcBatch ab;
                    ab.load(p, dist, a, a1, sl);
                    double x[kSsspArcBatch];
                    int left[kSsspArcBatch];
#pragma unroll
                    for (int j = 0; j < kSsspArcBatch; ++j) {
                        const size_t idx = (size_t)ab.w[j] * 32 + sl;
                        x[j] = 0.0;
                        left[j] = 0;
                        if (j < ab.cnt && ab.dw[j] + ab.wt[j] == dv) x[j] = sigma[idx];               // a parent
                        else if (j < ab.cnt && dv + ab.wt[j] == ab.dw[j]) left[j] = atomicSub(npar + idx, 1);  // a child
                    }
#pragma unroll
                    for (int j = 0; j < kSsspArcBatch; ++j) {
                        acc += x[j];   // arc order
                        if (left[j] == 1) {
                            sssp_push(p, g, ab.w[j], 1u << sl);
                            produced = true;
                        }
                    }
                }
                sigma[v * 32 + sl] = dv == 0 ? 1.0 : acc;
            }
            continue;
        }
        while (need) {
            const int i = __ffs(need) - 1;
            need &= need - 1;
            const int64_t v = __shfl_sync(kFull, myv, i);
            const uint32_t mv = __shfl_sync(kFull, mask, i);
            const bool on = (mv >> lane) & 1u;
            const long long dv = on ? dist[v * 32 + lane] : kSsspInf;
            double acc = 0.0;
            const int64_t a0 = p.off[v], a1 = p.off[v + 1];
            for (int64_t base = a0; base < a1; base += 32) {
                int32_t my_w = 0, my_wt = 0;
                if (base + lane < a1) {
                    my_w = __ldg(p.col + base + lane);
                    my_wt = __ldg(p.wgt + base + lane);
                }
                const int cnt = (int)min((int64_t)32, a1 - base);
                for (int j = 0; j < cnt; ++j) {
                    const int32_t w = __shfl_sync(kFull, my_w, j);
                    const int32_t wt = __shfl_sync(kFull, my_wt, j);
                    bool released = false;
                    if (on) {
                        const size_t idx = (size_t)w * 32 + lane;
                        const long long dw = dist[idx];
                        if (dw + wt == dv) acc += sigma[idx];                     // a parent: final since an earlier round
                        else if (dv + wt == dw) released = atomicSub(npar + idx, 1) == 1;  // a child: one parent fewer
                    }
                    const unsigned b = __ballot_sync(kFull, released);
                    if (b) {
                        if (lane == 0) sssp_push(p, g, w, b);
                        produced = true;
                    }
                }
            }
            if (on) sigma[v * 32 + lane] = dv == 0 ? 1.0 : acc;
        }
    }
    if (__any_sync(kFull, produced) && lane == 0) p.flags[p.round] = 1;   // (per thread in the pair branch)
}

// Phase D, one round: ready pairs pull coef from their children, release their parents.
__global__ void __launch_bounds__(kSsspWarps * 32) sssp_backward_kernel(const SsspParams p) {
    const size_t g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    int count;
    if (!sssp_round_begin(p, g, count)) return;   // the sweep ended before this round
    bool produced = false;
    const long long *dist = p.dist + g * p.n * 32;
    const double *sigma = p.sigma + g * p.n * 32;
    double *coef = p.coef + g * p.n * 32;
    int *nchild = p.nchild + g * p.n * 32;
    for (int base = (blockIdx.x * kSsspWarps + (threadIdx.x >> 5)) * 32; base < count;
         base += gridDim.x * kSsspWarps * 32) {
        int32_t myv;
        uint32_t mask;
        sssp_take_items(p, g, lane, base, count, myv, mask);
        unsigned need = __ballot_sync(kFull, mask != 0);
        if (need == 0) continue;
        const ChunkPairs cp = chunk_pairs(mask, myv, lane);
        if (__popc(need) > 1 && cp.total < kSsspPairLanes * __popc(need)) {
            // ---- one ready pair per thread; the BC partial takes the pair's delta with an atomic add
            for (int t0 = 0; t0 < cp.total; t0 += 32) {
                int sl;
                int64_t v;
                if (!cp.get(t0 + lane, v, sl)) continue;
                const size_t me = (size_t)v * 32 + sl;
                const long long dv = dist[me];
                double acc = 0.0;
                const int64_t a1 = p.off[v + 1];
                for (int64_t a = p.off[v]; a < a1; a += kSsspArcBatch) {
                    ArcBatch ab;
                    ab.load(p, dist, a, a1, sl);
                    double x[kSsspArcBatch];
                    int left[kSsspArcBatch];
#pragma unroll
                    for (int j = 0; j < kSsspArcBatch; ++j) {
                        const size_t idx = (size_t)ab.w[j] * 32 + sl;
                        x[j] = 0.0;
                        left[j] = 0;
                        if (j < ab.cnt && dv + ab.wt[j] == ab.dw[j]) x[j] = coef[idx];                   // a child
                        else if (j < ab.cnt && ab.dw[j] + ab.wt[j] == dv) left[j] = atomicSub(nchild + idx, 1);  // a parent
                    }
#pragma unroll
                    for (int j = 0; j < kSsspArcBatch; ++j) {
                        acc += x[j];   // arc order
                        if (left[j] == 1) {
                            sssp_push(p, g, ab.w[j], 1u << sl);
                            produced = true;
                        }
                    }
                }
                const double sv = sigma[me];
                const double d = sv * acc;
                coef[me] = (1.0 + d) / sv;
                if (p.delta) p.delta[g * p.n * 32 + me] = d;
                if (p.accumulate && dv != 0 && d != 0.0) atomicAdd(p.bcg + g * p.n + v, d);
            }
            continue;
        }
        while (need) {
            const int i = __ffs(need) - 1;
            need &= need - 1;
            const int64_t v = __shfl_sync(kFull, myv, i);
            const uint32_t mv = __shfl_sync(kFull, mask, i);
            const bool on = (mv >> lane) & 1u;
            const long long dv = on ? dist[v * 32 + lane] : kSsspInf;
            double acc = 0.0;
            const int64_t a0 = p.off[v], a1 = p.off[v + 1];
            for (int64_t base = a0; base < a1; base += 32) {
                int32_t my_w = 0, my_wt = 0;
                if (base + lane < a1) {
                    my_w = __ldg(p.col + base + lane);
                    my_wt = __ldg(p.wgt + base + lane);
                }
                const int cnt = (int)min((int64_t)32, a1 - base);
                for (int j = 0; j < cnt; ++j) {
                    const int32_t w = __shfl_sync(kFull, my_w, j);
                    const int32_t wt = __shfl_sync(kFull, my_wt, j);
                    bool released = false;
                    if (on) {
                        const size_t idx = (size_t)w * 32 + lane;
                        const long long dw = dist[idx];
                        if (dv + wt == dw) acc += coef[idx];                        // a child: final since an earlier round
                        else if (dw + wt == dv) released = atomicSub(nchild + idx, 1) == 1;  // a parent: one child fewer
                    }
                    const unsigned b = __ballot_sync(kFull, released);
                    if (b) {
                        if (lane == 0) sssp_push(p, g, w, b);
                        produced = true;
                    }
                }
            }
            double contrib = 0.0;
            if (on) {
                const size_t idx = (size_t)v * 32 + lane;
                const double sv = sigma[idx];
                const double d = sv * acc;
                coef[idx] = (1.0 + d) / sv;
                if (p.delta) p.delta[g * p.n * 32 + idx] = d;
                if (dv != 0) contrib = d;   // the source's own dependency is not part of BC (backward.py:154-158)
            }
            if (p.accumulate) {
                const double s = warp_sum(contrib);
                if (lane == 0 && s != 0.0) p.bcg[g * p.n + v] += s;
            }
        }
    }
    if (__any_sync(kFull, produced) && lane == 0) p.flags[p.round] = 1;   // (per thread in the pair branch)
}

// Inspection: rows [v][32] of one group -> [lane][n] arrays (BC_UNREACHED / 0 where unreached).
// *overflow is set when a distance does not fit the int32 inspection array.
__global__ void sssp_extract_kernel(const long long *dist, const double *sigma, const double *delta,
                                    int64_t n, int lanes, int32_t unreached, int32_t *dist_out,
                                    double *sigma_out, double *delta_out, int *overflow) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * 32;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int lane = (int)(i & 31);
        const int64_t v = i >> 5;
        if (lane >= lanes) continue;
        const long long d = dist[i];
        const bool on = d < kSsspInf;
        const size_t o = (size_t)lane * n + v;
        if (on && d > 2147483647LL) *overflow = 1;
        if (dist_out) dist_out[o] = on ? (int32_t)d : unreached;
        if (sigma_out) sigma_out[o] = on ? sigma[i] : 0.0;
        if (delta_out) delta_out[o] = on ? delta[i] : 0.0;
    }
}

}  // namespace bcb200
