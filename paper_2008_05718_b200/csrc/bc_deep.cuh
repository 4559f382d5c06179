// bc_deep.cuh -- persistent sweeps for high-diameter graphs (road networks, grids).
//
// A 2048 x 2048 road-like graph has ~4000 BFS levels whose frontiers hold a few
// thousand vertices per source.  Driven level by level from the host, every
// level costs three launches, a report read-back and a stream synchronise, and
// the kernels are too short to hide any of it.  The two kernels here run MANY
// consecutive thin levels in one cooperative launch: the grid walks a level,
// meets at a grid-wide barrier, and moves to the next one; the host comes back
// only when the run ends (frontier empty, level no longer thin, queue nearly
// full, level budget used) and reads the per-level log once.
//
// Arithmetic is that of fwd_push_thin_kernel / push_post_kernel /
// advance_level_kernel (forward) and bwd_queue_thin_kernel /
// swap_scatter_kernel (backward) in bc_kernels.cuh; reference functions being
// replaced: initial_relax (relax.py:75-101) and process_level vertex-pull
// (backward.py:95-103), for consecutive levels of one source batch.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bc_border.cuh"
#include "bc_kernels.cuh"

namespace bcb200 {

namespace cg = cooperative_groups;

// ---- Step-6 seeds on queue levels --------------------------------------------------------
// Step 6 of the partitioned forward phase (forward.py:232-246) relaxes every part from its
// borders at once: border j joins lane l's traversal at its refined distance D[j][l] with the
// arrival count arr[j][l] (paths whose last arc is a cut arc) as base path count.  On queue
// levels a seed is one more push into the level being produced: add the base count, set the
// lane in next[], append the vertex when nobody else has yet.  The (border, lane) pairs are
// sorted by level once per batch (seed_key_kernel + radix sort + seed_offsets_kernel).
struct SeedPlan {
    const int32_t *idx;        // border * S + lane, sorted by level (nullptr: no seeds)
    const int64_t *off;        // [levels + 1] first seed of each level
    int levels;                // seeds sit at levels [0, levels)
    const double *arr;         // [B][S] arrival counts
    const int32_t *border_v;   // [B] vertex of each border
    int S;
};

__device__ __forceinline__ void inject_seed_entry(const SeedPlan &sp, int64_t s, int64_t n,
                                                  const QueueParams &q, const uint32_t *vis,
                                                  uint32_t *next, double *sigma) {
    const int32_t idx = sp.idx[s];
    const int j = idx / sp.S, lane_all = idx % sp.S;
    const size_t g = (size_t)(lane_all >> 5);
    const int lane = lane_all & 31;
    const uint32_t bit = 1u << lane;
    const int64_t v = sp.border_v[j];
    if (vis[g * n + v] & bit) return;   // cannot happen while D is the exact distance
    atomicAdd(sigma + (g * n + v) * 32 + lane, sp.arr[idx]);
    const uint32_t old = atomicOr(next + g * n + v, bit);
    if (old == 0) {
        const unsigned long long pos = atomicAdd(q.q_count + g, 1ull);
        q.q_v[g * q.cap + pos] = (int32_t)v;
    }
}

// Seeds of one level, between the push kernels and push_post_kernel of that level.
__global__ void inject_seeds_queue_kernel(SeedPlan sp, int level, int64_t n, QueueParams q,
                                          const uint32_t *vis, uint32_t *next, double *sigma) {
    if (level >= sp.levels) return;
    const int64_t e = sp.off[level + 1];
    for (int64_t s = sp.off[level] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < e;
         s += (int64_t)gridDim.x * blockDim.x)
        inject_seed_entry(sp, s, n, q, vis, next, sigma);
}

// Sort key of every (border, lane) pair: its level when it is a Step-6 seed (finite distance,
// non-zero arrival count, lane in use), INT32_MAX otherwise.
__global__ void seed_key_kernel(int B, int S, int lanes, const int32_t *D, const double *arr,
                                int32_t *keys, int32_t *vals) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)B * S) return;
    const bool seed = (int)(idx % S) < lanes && D[idx] < kInf && arr[idx] != 0.0;
    keys[idx] = seed ? D[idx] : 0x7fffffff;
    vals[idx] = (int32_t)idx;
}

// off[L] = first sorted pair whose level is >= L, L = 0 .. levels.
__global__ void seed_offsets_kernel(const int32_t *keys, int64_t count, int levels, int64_t *off) {
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L > levels) return;
    int64_t lo = 0, hi = count;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < L) lo = mid + 1;
        else hi = mid;
    }
    off[L] = lo;
}

// Level of queue entry i of group g: levels own consecutive entry ranges, level_end[L][g] is one
// past the last entry of level L.
__device__ __forceinline__ int level_of_entry(const int64_t *level_end, int depth, int G, size_t g,
                                              int64_t i) {
    int lo = 0, hi = depth - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (level_end[(size_t)mid * G + g] > i) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// (dist, sigma) of the border vertices out of a queue-level sweep (border_gather_kernel for the
// dense level rows): one thread per queue entry, D_out / S_out pre-filled with kInf / 0.
// Path count of lane `bit` of queue entry i (mask m): from the level-ordered value array of a
// compact sweep (qs != nullptr) or from the row of its vertex.
__device__ __forceinline__ double entry_sigma(const double *qs, const uint32_t *q_off, int64_t vcap,
                                              const double *sigma, size_t g, int64_t n, size_t qslot,
                                              int64_t v, uint32_t m, int bit) {
    if (qs != nullptr) return qs[g * (size_t)vcap + q_off[qslot] + __popc(m & ((1u << bit) - 1u))];
    return sigma[(g * n + v) * 32 + bit];
}

__global__ void border_gather_queue_kernel(QueueParams q, const int64_t *level_end, int depth, int G,
                                           int64_t n, const int32_t *border_index,
                                           const double *sigma, int S, int32_t *D_out,
                                           double *S_out, const double *qs, const uint32_t *q_off,
                                           int64_t vcap) {
    const size_t g = blockIdx.y;
    const int64_t end = (int64_t)q.q_count[g];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q.q_v[g * q.cap + i];
        const int j = border_index[v];
        if (j < 0) continue;
        const uint32_t mask = q.q_m[g * q.cap + i];
        uint32_t m = mask;
        const int level = level_of_entry(level_end, depth, G, g, i);
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const size_t at = (size_t)j * S + g * 32 + bit;
            D_out[at] = level;
            S_out[at] = entry_sigma(qs, q_off, vcap, sigma, g, n, g * q.cap + i, v, mask, bit);
        }
    }
}

// Border-table rows out of a queue-level sweep whose lanes are borders first .. first+count-1
// (border_table_kernel for the dense level rows); bm / sm pre-filled with kInf / 0.
__global__ void border_table_queue_kernel(QueueParams q, const int64_t *level_end, int depth, int G,
                                          int64_t n, const int32_t *border_index,
                                          const double *sigma, BorderGeom geo, int first, int count,
                                          int32_t *bm, double *sm, const double *qs,
                                          const uint32_t *q_off, int64_t vcap) {
    const size_t g = blockIdx.y;
    const int64_t end = (int64_t)q.q_count[g];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < end;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q.q_v[g * q.cap + e];
        const int j = border_index[v];
        if (j < 0) continue;
        const uint32_t mask = q.q_m[g * q.cap + e];
        uint32_t m = mask;
        const int level = level_of_entry(level_end, depth, G, g, e);
        const int p = geo.border_p[j];
        const int b = geo.part_off[p + 1] - geo.part_off[p];
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const int lane_all = (int)g * 32 + bit;
            if (lane_all >= count) continue;
            const int i = first + lane_all;   // from-border (the lane's source), same part as j
            const size_t at = (size_t)geo.tab_off[p] + (size_t)(i - geo.part_off[p]) * b + (j - geo.part_off[p]);
            bm[at] = level;
            sm[at] = entry_sigma(qs, q_off, vcap, sigma, g, n, g * q.cap + e, v, mask, bit);
        }
    }
}

// s_pref[g] = sum over j < g of len(j) rounded up to whole warps, g = 0 .. ng (the flattened
// (group, entry) space of a level: every group padded to a multiple of 32 so a warp never
// straddles two groups).  One load per group and a two-stage scan instead of a serial loop per
// thread; ng <= kDeepMaxGroups = 128, every thread of the 256-thread block calls it.
template <typename LenFn>
__device__ __forceinline__ void padded_prefix(int64_t *s_pref, int ng, LenFn len) {
    __shared__ int64_t s_warp_total[4];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int64_t x = (t < ng) ? ((len(t) + 31) & ~(int64_t)31) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (warp < 4 && lane == 31) s_warp_total[warp] = x;
    __syncthreads();
    if (t < ng) {
        int64_t base = 0;
        for (int w = 0; w < warp; ++w) base += s_warp_total[w];
        s_pref[t + 1] = base + x;
    }
    if (t == 0) s_pref[0] = 0;
    __syncthreads();
}

// Shape of the persistent kernels: 1024 resident threads per SM (64 registers each) measured best
// (road-like 2048^2 x 512 sources: 743 / 780 / 878 ms at 1280 / 1536 / 2048 threads per SM, 748 / 849 at
// 768 / 512), and one block of 1024 threads per SM beats four of 256 by ~1 % (709 vs 719 ms: four times
// fewer participants in the grid-wide barriers).
#ifndef BC_DEEP_THREADS
#define BC_DEEP_THREADS 1024
#endif
#ifndef BC_DEEP_MIN_BLOCKS_F
#define BC_DEEP_MIN_BLOCKS_F 1
#endif
#ifndef BC_DEEP_MIN_BLOCKS_B
#define BC_DEEP_MIN_BLOCKS_B 1
#endif
constexpr int kDeepThreads = BC_DEEP_THREADS;
constexpr int kDeepWarps = kDeepThreads / 32;
constexpr int kDeepMaxGroups = 128;   // groups per batch the persistent sweeps accept

struct DeepFwdParams {
    const int64_t *off;
    const int32_t *col;
    int64_t n;
    QueueParams q;             // q_beg / q_end hold the frontier of the first level on entry
    int64_t *q_beg, *q_end, *q_lbeg;   // writable views of the device-resident ranges
    uint32_t *vis;
    uint32_t *next;            // all-zero scratch masks (left all-zero)
    double *sigma;
    uint32_t *live;            // live[level][G]
    unsigned long long *counters;
    unsigned long long *lstat;   // [0] vertices [1] arcs [2] largest degree of the level being produced
    unsigned long long *log;     // [iteration][3 + 2G], the advance_level_kernel report of every level
    int *run_info;               // [0] levels produced by this launch
    int ng, G;
    int first_level;             // level produced by iteration 0
    int max_levels;              // iterations allowed in this launch
    unsigned long long graph_arcs;   // arcs of the graph * groups (push / pull switch)
    unsigned long long push_beta;
    unsigned long long thin_degree;
    unsigned long long max_degree;
    SeedPlan seeds;              // Step-6 border seeds joining at their own level (idx == nullptr: none)
    unsigned long long seed_room;   // queue entries the seeds of one level may add per group
};

// Forward: consecutive top-down levels, one THREAD per frontier entry.
__global__ void __launch_bounds__(kDeepThreads) deep_forward_kernel(const DeepFwdParams p) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t stage[kDeepWarps][kStage];
    __shared__ int64_t s_pref[kDeepMaxGroups + 1];
    __shared__ unsigned long long s_stat[8];
    __shared__ uint32_t s_live[kDeepMaxGroups];
    __shared__ int s_cont;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = p.n;
    int *cont_flag = p.run_info + 1;

    for (int it = 0;; ++it) {
        const int L = p.first_level + it;
        // ---- phase 1: push from the frontier queues.  The (group, entry) space is
        // flattened, every group padded to whole warps, so that all threads stay
        // busy when one group's frontier is short and a warp never straddles groups.
        if (threadIdx.x <= p.ng) {
            int64_t acc = 0;
            for (int g = 0; g < (int)threadIdx.x; ++g) acc += (p.q.q_end[g] - p.q.q_beg[g] + 31) & ~(int64_t)31;
            s_pref[threadIdx.x] = acc;
        }
        __syncthreads();
        unsigned c_t = 0;
        {
            const int64_t total = s_pref[p.ng];
            int g = 0;
            // Appends to a group's queue cost one atomic on q_count[g] per flush, and every warp of
            // the grid hits the same few words: the staging buffer is carried over the iterations
            // of a group and flushed only when it runs full, the group changes or the phase ends.
            int staged = 0;       // warp-uniform
            int staged_g = 0;     // group the staged vertices belong to
            auto flush = [&]() {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(p.q.q_count + staged_g, (unsigned long long)staged);
                base = __shfl_sync(kFull, base, 0);
                const size_t qb = (size_t)staged_g * p.q.cap;
                for (int k = lane; k < staged; k += 32) p.q.q_v[qb + base + k] = stage[warp][k];
                staged = 0;
                __syncwarp();
            };
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;   // f0 only grows
                if (g != staged_g) {
                    if (staged) flush();
                    staged_g = g;
                }
                const int64_t end = p.q.q_end[g];
                const int64_t i = p.q.q_beg[g] + (f0 - s_pref[g]) + lane;
                const uint32_t *gvis = p.vis + (size_t)g * n;
                uint32_t *gnext = p.next + (size_t)g * n;
                double *gsig = p.sigma + (size_t)g * n * 32;
                const size_t qbase = (size_t)g * p.q.cap;
                int32_t u = 0;
                uint32_t mask = 0;
                int64_t a = 0, e = 0;
                if (i < end) {
                    u = p.q.q_v[qbase + i];
                    mask = p.q.q_m[qbase + i];
                    a = p.off[u];
                    e = p.off[u + 1];
                }
                int rounds = (int)(e - a);
                rounds = __reduce_max_sync(kFull, rounds);
                const double *urow = gsig + (size_t)u * 32;
                push_entry_thin(a, e, rounds, mask, p.col, gvis, gnext, gsig, urow, c_t,
                                [&](bool fresh_vertex, int32_t w) {
                                    const unsigned newm = __ballot_sync(kFull, fresh_vertex);
                                    if (newm) {
                                        if (fresh_vertex)
                                            stage[warp][staged + __popc(newm & ((1u << lane) - 1u))] = w;
                                        staged += __popc(newm);
                                        __syncwarp();
                                        if (staged > kStage - 32) flush();
                                    }
                                });
            }
            if (staged) flush();
        }
        {
            // DAG arcs of the level: one global atomic per block
            if (threadIdx.x == 0) s_stat[5] = 0ull;
            __syncthreads();
            const unsigned t = __reduce_add_sync(kFull, c_t);
            if (lane == 0 && t) atomicAdd(&s_stat[5], (unsigned long long)t);
            __syncthreads();
            if (threadIdx.x == 0 && s_stat[5]) atomicAdd(p.counters + 2, s_stat[5]);
        }
        // border seeds of level L: more pushes into the same level (atomics on sigma / next)
        if (p.seeds.idx != nullptr && L < p.seeds.levels) {
            const int64_t se = p.seeds.off[L + 1];
            for (int64_t s = p.seeds.off[L] + gtid; s < se; s += gthreads)
                inject_seed_entry(p.seeds, s, n, p.q, p.vis, p.next, p.sigma);
        }
        grid.sync();

        // ---- phase 2: the entries appended above become level L (same flattening)
        if (threadIdx.x <= p.ng) {
            int64_t acc = 0;
            for (int g = 0; g < (int)threadIdx.x; ++g)
                acc += ((int64_t)p.q.q_count[g] - p.q_lbeg[g] + 31) & ~(int64_t)31;
            s_pref[threadIdx.x] = acc;
        }
        __syncthreads();
        {
            // The level's statistics are five counters shared by the whole grid: every thread
            // keeps its own partial sums over the level, the block adds them up in shared memory
            // and issues ONE set of global atomics per level (a warp-per-iteration atomic on the
            // same five words serialises the whole grid at one L2 slice).
            if (threadIdx.x < 8) s_stat[threadIdx.x] = 0ull;
            for (int k = threadIdx.x; k < p.ng; k += blockDim.x) s_live[k] = 0u;
            __syncthreads();
            const int64_t total = s_pref[p.ng];
            int g = 0;
            unsigned long long nr = 0, ar = 0, nv = 0, fa = 0, md = 0;
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;
                const int64_t end = (int64_t)p.q.q_count[g];
                const int64_t i = p.q_lbeg[g] + (f0 - s_pref[g]) + lane;
                const size_t qbase = (size_t)g * p.q.cap;
                uint32_t any = 0;
                int32_t w = 0;
                if (i < end) {
                    w = p.q.q_v[qbase + i];
                    const uint32_t m = p.next[(size_t)g * n + w];
                    p.q.q_m[qbase + i] = m;
                    p.vis[(size_t)g * n + w] |= m;
                    p.next[(size_t)g * n + w] = 0u;
                    const unsigned long long deg = (unsigned long long)(p.off[w + 1] - p.off[w]);
                    any = m;
                    nr += __popc(m);
                    ar += __popc(m) * deg;
                    nv += 1;
                    fa += deg;
                    md = max(md, deg);
                }
                any = __reduce_or_sync(kFull, any);
                if (lane == 0 && any) atomicOr(&s_live[g], any);
            }
            for (int o = 16; o > 0; o >>= 1) {
                nr += __shfl_xor_sync(kFull, nr, o);
                ar += __shfl_xor_sync(kFull, ar, o);
                nv += __shfl_xor_sync(kFull, nv, o);
                fa += __shfl_xor_sync(kFull, fa, o);
                md = max(md, __shfl_xor_sync(kFull, md, o));
            }
            if (lane == 0 && nv) {
                atomicAdd(&s_stat[0], nr);
                atomicAdd(&s_stat[1], ar);
                atomicAdd(&s_stat[2], nv);
                atomicAdd(&s_stat[3], fa);
                atomicMax(&s_stat[4], md);
            }
            __syncthreads();
            if (threadIdx.x == 0 && s_stat[2]) {
                atomicAdd(p.counters + 0, s_stat[0]);
                atomicAdd(p.counters + 1, s_stat[1]);
                atomicAdd(p.lstat + 0, s_stat[2]);
                atomicAdd(p.lstat + 1, s_stat[3]);
                atomicMax(p.lstat + 2, s_stat[4]);
            }
            for (int k = threadIdx.x; k < p.ng; k += blockDim.x)
                if (s_live[k]) atomicOr(p.live + (size_t)L * p.G + k, s_live[k]);
        }
        grid.sync();

        // ---- phase 3: publish the level, rotate the ranges, decide whether to go on
        if (blockIdx.x == 0) {
            unsigned long long *rep = p.log + (size_t)it * (3 + 2 * p.G);
            const int g = threadIdx.x;
            unsigned long long nverts = p.lstat[0], farcs = p.lstat[1], maxdeg = p.lstat[2];
            uint32_t alive_any = 0;
            unsigned long long used = 0;
            for (int j = 0; j < p.ng; ++j) {
                alive_any |= p.live[(size_t)L * p.G + j];
                used = max(used, p.q.q_count[j]);
            }
            __syncthreads();
            if (g < 3) rep[g] = p.lstat[g];
            if (g < p.G) {
                const unsigned long long c = p.q.q_count[g];
                rep[3 + g] = c;
                rep[3 + p.G + g] = p.live[(size_t)L * p.G + g];
                p.q_beg[g] = p.q_lbeg[g];
                p.q_end[g] = (int64_t)c;
                p.q_lbeg[g] = (int64_t)c;
            }
            __syncthreads();
            if (g == 0) {
                p.lstat[0] = p.lstat[1] = p.lstat[2] = 0;
                const unsigned long long room = min((unsigned long long)n, farcs) + 1 + p.seed_room;
                const bool go = alive_any != 0 && it + 1 < p.max_levels &&
                                farcs * p.push_beta <= p.graph_arcs && maxdeg <= p.max_degree &&
                                farcs <= p.thin_degree * nverts &&
                                (unsigned long long)p.q.cap - used >= room;
                p.run_info[0] = it + 1;
                *cont_flag = go ? 1 : 0;
            }
        }
        grid.sync();
        if (threadIdx.x == 0) s_cont = *(volatile int *)cont_flag;
        __syncthreads();
        if (!s_cont) break;
    }
}

// ---- forward over level-ordered path counts ---------------------------------------------------
// deep_forward_kernel adds path counts into the 256-byte row of the vertex: one random DRAM
// read-modify-write per discovered (vertex, lane) pair plus one random read of the parent's row
// (the rows of a 2048 x 2048 road graph span 17 GB per batch).  Here a level's path counts live in
// the slots of its queue entries (qs[g][q_off[i] + rank of the lane in q_m[i]]), a window of a few
// MB that stays in L2, and a level takes three phases:
//   A  discover: frontier entries walk their arcs, OR the fresh lanes into next[], append new
//      vertices to the queue and record the entry index in pos[g][w]; every frontier entry
//      keeps a bit per arc that found something (q_arc);
//   A2 post: the new entries get their lane masks (next[] -> q_m, vis |=, next = 0), their value
//      slots (zeroed) and the level statistics;
//   B  accumulate: the frontier entries walk the arcs marked in q_arc, look the child's entry up
//      through pos[], and add their own path counts into the child's slots (red.global.add.f64
//      on an L2-resident window; integer-valued, exact in any order).
// The per-(group, vertex) words the phases touch -- visited lanes, lanes being discovered at this
// level, queue entry of the vertex -- sit side by side in one 16-byte record (VertexState), so the
// visited probe of an arc, the OR into the next-level word and the entry index of the child share a
// 32-byte sector: these dense arrays are what is left of the random DRAM traffic.  (Carrying the
// entry's lane mask and value slot in the record as well -- 32 bytes, one hop less per child -- was
// measured and lost: road-like 2048^2, 662 -> 692 ms, the doubled footprint costs more L2 misses on
// the probes than the hop saves.)
// `pos` is never cleared inside a batch: queue indices only grow, so an index below the start of
// the level being produced is a stale one.  The host initialises the records per sweep.
struct __align__(16) VertexState {
    uint32_t vis;    // lanes that reached the vertex
    uint32_t next;   // lanes discovering it at the level being produced (zero between levels)
    uint32_t pos;    // queue entry (index + 1) the vertex got most recently
    uint32_t pos2;   // backward sweep: entries of odd levels write here, of even levels into `pos`
};

__device__ __forceinline__ int32_t nb_at(const int4 &nb, int k) {
    return k == 0 ? nb.x : k == 1 ? nb.y : k == 2 ? nb.z : nb.w;
}

// Degree byte of a queue entry (top byte of q_arc): the degree itself below 240, 255 = look it up
// in the offsets, 0xF0 | d = degree d <= 4 with the neighbour ids in q_nb.
constexpr uint32_t kNbCached = 0xF0u;
__device__ __forceinline__ uint32_t degree_byte(unsigned long long deg) { return deg < 240ull ? (uint32_t)deg : 255u; }
__device__ __forceinline__ bool entry_cached(uint32_t byte) { return byte >= kNbCached && byte != 255u; }
__device__ __forceinline__ uint32_t entry_degree(uint32_t byte) { return entry_cached(byte) ? (byte & 0x0Fu) : byte; }

struct DeepFwdCompactParams {
    const int64_t *off;
    const int32_t *col;
    int64_t n;
    QueueParams q;
    int64_t *q_beg, *q_end, *q_lbeg;
    VertexState *vs;           // [G][n]
    double *qs;                // [G][vcap]
    uint32_t *q_off;           // [G][cap]
    uint32_t *q_arc;           // [G][cap] degree byte (degree_byte / kNbCached) << 24 | arcs 0..23 that reached a fresh lane
    uint32_t *q_a;             // [G][cap] first arc of the entry's vertex (the sweeps then never read the
                               // row offsets of a frontier vertex: one random access and one hop less)
    int4 *q_nb;                // [G][cap] the neighbour ids of an entry's vertex when it has at most four (-1 = none):
                               // left by the discover pass, read in entry order by the accumulate pass and the
                               // backward sweep instead of a random col_idx sector each
    unsigned long long *v_count;   // [G] value slots handed out so far
    int64_t vcap;
    uint32_t *live;
    unsigned long long *counters;
    unsigned long long *lstat;
    unsigned long long *log;
    int *run_info;
    int ng, G;
    int first_level;
    int max_levels;
    unsigned long long graph_arcs;
    unsigned long long push_beta;
    unsigned long long thin_degree;
    unsigned long long max_degree;
    SeedPlan seeds;
    unsigned long long seed_room;
};

#ifdef BC_DEEP_PHASE_TIMING
__device__ unsigned long long g_phase_ns[8];   // dev build: time per phase (A, A2, B) as seen by block 0
#endif
__global__ void __launch_bounds__(kDeepThreads, BC_DEEP_MIN_BLOCKS_F) deep_forward_compact_kernel(const DeepFwdCompactParams p) {
    cg::grid_group grid = cg::this_grid();
#ifdef BC_DEEP_PHASE_TIMING
    unsigned long long t_last;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_last));
#endif
    __shared__ int32_t stage[kDeepWarps][kStage];
    __shared__ int64_t s_pref[kDeepMaxGroups + 1];
    __shared__ int64_t s_beg[kDeepMaxGroups], s_end[kDeepMaxGroups], s_lbeg[kDeepMaxGroups];
    __shared__ unsigned long long s_stat[8];
    __shared__ uint32_t s_live[kDeepMaxGroups];
    __shared__ int s_cont;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = p.n;
    int *cont_flag = p.run_info + 1;

    auto frontier_prefix = [&]() {   // flattened (group, entry) space of the frontier, groups padded to warps
        padded_prefix(s_pref, p.ng, [&](int g) { return s_end[g] - s_beg[g]; });
    };

    for (int it = 0;; ++it) {
        const int L = p.first_level + it;
        for (int k = threadIdx.x; k < p.ng; k += blockDim.x) {
            s_beg[k] = p.q.q_beg[k];
            s_end[k] = p.q.q_end[k];
            s_lbeg[k] = p.q_lbeg[k];
        }
        __syncthreads();
        frontier_prefix();
        // ---- phase A: discover
        {
            const int64_t total = s_pref[p.ng];
            int g = 0;
            int staged = 0, staged_g = 0;   // warp-uniform
            auto flush = [&]() {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(p.q.q_count + staged_g, (unsigned long long)staged);
                base = __shfl_sync(kFull, base, 0);
                const size_t qb = (size_t)staged_g * p.q.cap;
                for (int k = lane; k < staged; k += 32) {
                    const int32_t w = stage[warp][k];
                    p.q.q_v[qb + base + k] = w;
                    p.vs[(size_t)staged_g * n + w].pos = (uint32_t)(base + k) + 1u;
                }
                staged = 0;
                __syncwarp();
            };
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;
                if (g != staged_g) {
                    if (staged) flush();
                    staged_g = g;
                }
                const int64_t end = s_end[g];
                const int64_t i = s_beg[g] + (f0 - s_pref[g]) + lane;
                VertexState *gvs = p.vs + (size_t)g * n;
                const size_t qbase = (size_t)g * p.q.cap;
                uint32_t mask = 0, word = 0;
                int64_t a = 0, e = 0;
                int4 first4 = make_int4(-1, -1, -1, -1);   // neighbours 0..3 of the entry's vertex
                if (i < end) {
                    mask = p.q.q_m[qbase + i];
                    word = p.q_arc[qbase + i];
                    a = p.q_a[qbase + i];
                    e = a + entry_degree(word >> 24);   // (flagged already if the level is being re-run after a relaunch)
                    if ((word >> 24) == 255u) {     // long adjacency: the degree did not fit
                        const int32_t u = p.q.q_v[qbase + i];
                        a = p.off[u];
                        e = p.off[u + 1];
                    }
                }
                int rounds = (int)(e - a);
                rounds = __reduce_max_sync(kFull, rounds);
                uint32_t arcbits = 0;
                for (int r0 = 0; r0 < rounds; r0 += kThinArcs) {
                    int32_t w[kThinArcs];
                    uint32_t fresh[kThinArcs], old[kThinArcs];
#pragma unroll
                    for (int k = 0; k < kThinArcs; ++k) w[k] = (a + r0 + k < e) ? __ldg(p.col + a + r0 + k) : -1;
                    if (r0 == 0) first4 = make_int4(w[0], w[1], w[2], w[3]);
#pragma unroll
                    for (int k = 0; k < kThinArcs; ++k) fresh[k] = (w[k] >= 0) ? (mask & ~gvs[w[k]].vis) : 0u;
#pragma unroll
                    for (int k = 0; k < kThinArcs; ++k) old[k] = fresh[k] ? atomicOr(&gvs[w[k]].next, fresh[k]) : 1u;
#pragma unroll
                    for (int k = 0; k < kThinArcs; ++k) {
                        if (r0 + k >= rounds) break;   // warp-uniform
                        if (fresh[k] && r0 + k < 24) arcbits |= 1u << (r0 + k);
                        const bool fresh_vertex = fresh[k] != 0 && old[k] == 0;
                        const unsigned newm = __ballot_sync(kFull, fresh_vertex);
                        if (newm) {
                            if (fresh_vertex) stage[warp][staged + __popc(newm & ((1u << lane) - 1u))] = w[k];
                            staged += __popc(newm);
                            __syncwarp();
                            if (staged > kStage - 32) flush();
                        }
                    }
                }
                if (i < end) {
                    // a vertex with at most four arcs leaves its neighbour ids with the entry: the
                    // accumulate pass below and the backward sweep read them in entry order instead of
                    // one random col_idx sector each (degree byte 0xF0 | degree marks such an entry)
                    uint32_t byte = word >> 24;
                    if (p.q_nb != nullptr && byte != 255u && entry_degree(byte) <= 4u) {
                        p.q_nb[qbase + i] = first4;
                        byte = kNbCached | entry_degree(byte);
                    }
                    p.q_arc[qbase + i] = (byte << 24) | arcbits;
                }
            }
            if (staged) flush();
        }
        // border seeds of level L: discovered like any other vertex, their counts join in phase B
        if (p.seeds.idx != nullptr && L < p.seeds.levels) {
            const int64_t se = p.seeds.off[L + 1];
            for (int64_t s = p.seeds.off[L] + gtid; s < se; s += gthreads) {
                const int32_t idx = p.seeds.idx[s];
                const int j = idx / p.seeds.S, lane_all = idx % p.seeds.S;
                const size_t g = (size_t)(lane_all >> 5);
                const uint32_t bit = 1u << (lane_all & 31);
                const int64_t v = p.seeds.border_v[j];
                VertexState *rec = p.vs + g * n + v;
                if (rec->vis & bit) continue;   // cannot happen while D is the exact distance
                const uint32_t old = atomicOr(&rec->next, bit);
                if (old == 0) {
                    const unsigned long long at = atomicAdd(p.q.q_count + g, 1ull);
                    p.q.q_v[g * p.q.cap + at] = (int32_t)v;
                    rec->pos = (uint32_t)at + 1u;
                }
            }
        }
        grid.sync();
#ifdef BC_DEEP_PHASE_TIMING
        if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long t_now; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_now)); g_phase_ns[0] += t_now - t_last; t_last = t_now; }
#endif

        // ---- phase A2: the entries appended above become level L
        if (threadIdx.x < 8) s_stat[threadIdx.x] = 0ull;
        for (int k = threadIdx.x; k < p.ng; k += blockDim.x) s_live[k] = 0u;
        padded_prefix(s_pref, p.ng, [&](int g) { return (int64_t)p.q.q_count[g] - s_lbeg[g]; });
        {
            const int64_t total = s_pref[p.ng];
            int g = 0;
            unsigned long long nr = 0, ar = 0, nv = 0, fa = 0, md = 0;
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;
                const int64_t end = (int64_t)p.q.q_count[g];
                const int64_t i = s_lbeg[g] + (f0 - s_pref[g]) + lane;
                const size_t qbase = (size_t)g * p.q.cap;
                uint32_t m = 0;
                if (i < end) {
                    const int32_t w = p.q.q_v[qbase + i];
                    uint2 *vn = reinterpret_cast<uint2 *>(p.vs + (size_t)g * n + w);   // (vis, next)
                    const uint2 cur = *vn;
                    m = cur.y;
                    p.q.q_m[qbase + i] = m;
                    *vn = make_uint2(cur.x | m, 0u);
                    const int64_t w_a = p.off[w];
                    const unsigned long long deg = (unsigned long long)(p.off[w + 1] - w_a);
                    p.q_a[qbase + i] = (uint32_t)w_a;
                    p.q_arc[qbase + i] = degree_byte(deg) << 24;
                    nr += __popc(m);
                    ar += __popc(m) * deg;
                    nv += 1;
                    fa += deg;
                    md = max(md, deg);
                }
                // value slots of the warp's entries: warp prefix of popc + one atomic per warp
                const unsigned pc = __popc(m);
                unsigned incl = pc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                const unsigned wtotal = __shfl_sync(kFull, incl, 31);
                unsigned long long base = 0;
                if (lane == 0 && wtotal) base = atomicAdd(p.v_count + g, (unsigned long long)wtotal);
                base = __shfl_sync(kFull, base, 0);
                if (i < end) {
                    const unsigned long long at = base + incl - pc;
                    p.q_off[qbase + i] = (uint32_t)at;
                    if (at + pc <= (unsigned long long)p.vcap)
                        for (unsigned k = 0; k < pc; ++k) p.qs[(size_t)g * p.vcap + at + k] = 0.0;
                }
                const uint32_t any = __reduce_or_sync(kFull, m);
                if (lane == 0 && any) atomicOr(&s_live[g], any);
            }
            for (int o = 16; o > 0; o >>= 1) {
                nr += __shfl_xor_sync(kFull, nr, o);
                ar += __shfl_xor_sync(kFull, ar, o);
                nv += __shfl_xor_sync(kFull, nv, o);
                fa += __shfl_xor_sync(kFull, fa, o);
                md = max(md, __shfl_xor_sync(kFull, md, o));
            }
            if (lane == 0 && nv) {
                atomicAdd(&s_stat[0], nr);
                atomicAdd(&s_stat[1], ar);
                atomicAdd(&s_stat[2], nv);
                atomicAdd(&s_stat[3], fa);
                atomicMax(&s_stat[4], md);
            }
            __syncthreads();
            if (threadIdx.x == 0 && s_stat[2]) {
                atomicAdd(p.counters + 0, s_stat[0]);
                atomicAdd(p.counters + 1, s_stat[1]);
                atomicAdd(p.lstat + 0, s_stat[2]);
                atomicAdd(p.lstat + 1, s_stat[3]);
                atomicMax(p.lstat + 2, s_stat[4]);
            }
            for (int k = threadIdx.x; k < p.ng; k += blockDim.x)
                if (s_live[k]) atomicOr(p.live + (size_t)L * p.G + k, s_live[k]);
        }
        grid.sync();
#ifdef BC_DEEP_PHASE_TIMING
        if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long t_now; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_now)); g_phase_ns[1] += t_now - t_last; t_last = t_now; }
#endif

        // ---- phase B: the frontier adds its path counts into the new entries' slots
        frontier_prefix();
        unsigned c_t = 0;
        {
            const int64_t total = s_pref[p.ng];
            int g = 0;
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;
                const int64_t i = s_beg[g] + (f0 - s_pref[g]) + lane;
                if (i >= s_end[g]) continue;
                const size_t qbase = (size_t)g * p.q.cap;
                const size_t vbase = (size_t)g * p.vcap;
                const uint32_t mask = p.q.q_m[qbase + i];
                const uint32_t word = p.q_arc[qbase + i];
                int64_t a = p.q_a[qbase + i], e = a + entry_degree(word >> 24);
                if ((word >> 24) == 255u) {
                    const int32_t u = p.q.q_v[qbase + i];
                    a = p.off[u];
                    e = p.off[u + 1];
                }
                const bool cached = p.q_nb != nullptr && entry_cached(word >> 24);     // (set by phase A above)
                int4 nbv = make_int4(-1, -1, -1, -1);
                if (cached) nbv = p.q_nb[qbase + i];
                const uint32_t at_u = p.q_off[qbase + i];
                const VertexState *gvs = p.vs + (size_t)g * n;
                const uint32_t lbeg = (uint32_t)s_lbeg[g];
                auto add_into = [&](int32_t w) {
                    const uint32_t pj = gvs[w].pos;
                    if (pj <= lbeg) return;                 // no entry in the level being produced
                    const uint32_t mj = p.q.q_m[qbase + pj - 1];
                    uint32_t lanes = mask & mj;
                    if (lanes == 0) return;
                    const uint32_t oj = p.q_off[qbase + pj - 1];
                    while (lanes) {
                        const int bit = __ffs(lanes) - 1;
                        lanes &= lanes - 1;
                        const uint32_t lower = (1u << bit) - 1u;
                        atomicAdd(p.qs + vbase + oj + __popc(mj & lower), p.qs[vbase + at_u + __popc(mask & lower)]);
                        ++c_t;
                    }
                };
                if (e - a <= 24) {
                    uint32_t bits = word & 0x00ffffffu;
                    while (bits) {
                        const int k = __ffs(bits) - 1;
                        bits &= bits - 1;
                        add_into(cached ? nb_at(nbv, k) : __ldg(p.col + a + k));
                    }
                } else {
                    for (int64_t b = a; b < e; ++b) add_into(__ldg(p.col + b));
                }
            }
        }
        if (p.seeds.idx != nullptr && L < p.seeds.levels) {
            const int64_t se = p.seeds.off[L + 1];
            for (int64_t s = p.seeds.off[L] + gtid; s < se; s += gthreads) {
                const int32_t idx = p.seeds.idx[s];
                const int j = idx / p.seeds.S, lane_all = idx % p.seeds.S;
                const size_t g = (size_t)(lane_all >> 5);
                const int bit = lane_all & 31;
                const int64_t v = p.seeds.border_v[j];
                const uint32_t pj = p.vs[g * n + v].pos;
                if (pj <= (uint32_t)s_lbeg[g]) continue;
                const uint32_t mj = p.q.q_m[g * p.q.cap + pj - 1];
                if (!((mj >> bit) & 1u)) continue;
                atomicAdd(p.qs + g * (size_t)p.vcap + p.q_off[g * p.q.cap + pj - 1] + __popc(mj & ((1u << bit) - 1u)),
                          p.seeds.arr[idx]);
            }
        }
        {
            if (threadIdx.x == 0) s_stat[5] = 0ull;
            __syncthreads();
            const unsigned t = __reduce_add_sync(kFull, c_t);
            if (lane == 0 && t) atomicAdd(&s_stat[5], (unsigned long long)t);
            __syncthreads();
            if (threadIdx.x == 0 && s_stat[5]) atomicAdd(p.counters + 2, s_stat[5]);
        }
        // ---- publish the level, rotate the ranges, decide whether to go on (block 0; the other
        // blocks only read their shared copies of the ranges in phase B)
        if (blockIdx.x == 0) {
            unsigned long long *rep = p.log + (size_t)it * (3 + 2 * p.G);
            const int g = threadIdx.x;
            unsigned long long nverts = p.lstat[0], farcs = p.lstat[1], maxdeg = p.lstat[2];
            uint32_t alive_any = 0;
            unsigned long long used = 0;
            for (int j = 0; j < p.ng; ++j) {
                alive_any |= p.live[(size_t)L * p.G + j];
                used = max(used, p.q.q_count[j]);
            }
            __syncthreads();
            if (g < 3) rep[g] = p.lstat[g];
            if (g < p.G) {
                const unsigned long long c = p.q.q_count[g];
                rep[3 + g] = c;
                rep[3 + p.G + g] = p.live[(size_t)L * p.G + g];
                p.q_beg[g] = p.q_lbeg[g];
                p.q_end[g] = (int64_t)c;
                p.q_lbeg[g] = (int64_t)c;
            }
            __syncthreads();
            if (g == 0) {
                p.lstat[0] = p.lstat[1] = p.lstat[2] = 0;
                const unsigned long long room = min((unsigned long long)n, farcs) + 1 + p.seed_room;
                const bool go = alive_any != 0 && it + 1 < p.max_levels &&
                                farcs * p.push_beta <= p.graph_arcs && maxdeg <= p.max_degree &&
                                farcs <= p.thin_degree * nverts &&
                                (unsigned long long)p.q.cap - used >= room;
                p.run_info[0] = it + 1;
                *cont_flag = go ? 1 : 0;
            }
        }
        grid.sync();
#ifdef BC_DEEP_PHASE_TIMING
        if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long t_now; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_now)); g_phase_ns[2] += t_now - t_last; t_last = t_now; }
#endif
        if (threadIdx.x == 0) s_cont = *(volatile int *)cont_flag;
        __syncthreads();
        if (!s_cont) break;
    }
}

// Rows from level-ordered values (a compact sweep that has to continue on the row layout): every
// queue entry writes its path counts back into the row of its vertex.
__global__ void decompact_sigma_kernel(QueueParams q, const uint32_t *q_off, const double *qs,
                                       int64_t vcap, int64_t n, double *sigma) {
    const size_t g = blockIdx.y;
    const int64_t end = (int64_t)q.q_count[g];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q.q_v[g * q.cap + i];
        uint32_t m = q.q_m[g * q.cap + i];
        const double *in = qs + g * (size_t)vcap + q_off[g * q.cap + i];
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            sigma[(g * n + v) * 32 + bit] = *in++;
        }
    }
}

// Per-vertex records of a compact sweep: lanes the batch does not use count as visited.
__global__ void compact_init_kernel(VertexState *vs, int64_t n, int batch_count) {
    const size_t g = blockIdx.y;
    const int lanes = min(32, batch_count - (int)g * 32);
    const uint32_t dead = lanes >= 32 ? 0u : ~((1u << lanes) - 1u);
    uint4 *out = reinterpret_cast<uint4 *>(vs + g * n);
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        out[v] = make_uint4(dead, 0u, 0u, 0u);
    }
}

// ... and the visited words out of the vertex records, for the row-based kernels that take over.
__global__ void vis_from_records_kernel(const VertexState *vs, uint32_t *vis, int64_t n) {
    const size_t g = blockIdx.y;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        vis[g * n + v] = vs[g * n + v].vis;
}

// Level 0 of a compact sweep: every set lane of a source entry carries one path.
__global__ void compact_level0_kernel(QueueParams q, uint32_t *q_off, double *qs, int64_t vcap,
                                      unsigned long long *v_count, VertexState *vs, int64_t n,
                                      const int64_t *off, uint32_t *q_a, uint32_t *q_arc) {
    const size_t g = blockIdx.x;
    if (threadIdx.x != 0) return;
    const int64_t end = (int64_t)q.q_count[g];
    uint32_t at = 0;
    for (int64_t i = 0; i < end; ++i) {     // <= 32 entries
        const uint32_t m = q.q_m[g * q.cap + i];
        const int64_t v = q.q_v[g * q.cap + i];
        vs[g * n + v].vis |= m;
        q_a[g * q.cap + i] = (uint32_t)off[v];
        q_arc[g * q.cap + i] = degree_byte((unsigned long long)(off[v + 1] - off[v])) << 24;
        q_off[g * q.cap + i] = at;
        for (int k = 0; k < __popc(m); ++k) qs[g * (size_t)vcap + at + k] = 1.0;
        at += __popc(m);
    }
    v_count[g] = at;
}

struct DeepBwdParams {
    const int64_t *off;
    const int32_t *col;
    int64_t n;
    QueueParams q;               // q_v / q_m / cap
    const int64_t *range_table;  // [level][0: begin, 1: end][G]
    double *sigma;
    double *coef;
    double *delta;               // only with STORE_DELTA
    double *bcg;
    int ng, G;
    int hi, lo;                  // levels hi, hi - 1, ..., lo
    const uint32_t *nbr_first;   // masks of level hi + 1 (nullptr: hi is the deepest level)
    uint32_t *erase_first;       // scratch array holding level hi + 1 (nullptr: dense array, keep)
    uint32_t *scr0, *scr1;       // all-zero scratch arrays (apart from erase_first's content)
    int first_write;             // scratch (0 / 1) that receives level hi
    int accumulate;              // bit 0: BC partials, bit 1: clear sigma (finalize_backward)
};

// Backward: consecutive queue levels, one thread per entry (bwd_queue_thin_kernel),
// with the mask hand-over of swap_scatter_kernel between levels.  On exit the
// masks of level `lo` sit in scratch (first_write + hi - lo) & 1, everything
// else in the scratch arrays is zero again.
template <bool STORE_DELTA>
__global__ void __launch_bounds__(kDeepThreads) deep_backward_kernel(const DeepBwdParams p) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int64_t s_pref[kDeepMaxGroups + 1];
    const int lane = threadIdx.x & 31;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = p.n;
    const uint32_t *nbr = p.nbr_first;
    uint32_t *erase = p.erase_first;
    int widx = p.first_write;
    for (int L = p.hi; L >= p.lo; --L) {
        uint32_t *wr = widx ? p.scr1 : p.scr0;
        const int64_t *beg_t = p.range_table + ((size_t)L * 2 + 0) * p.G;
        const int64_t *end_t = p.range_table + ((size_t)L * 2 + 1) * p.G;
        if (threadIdx.x <= p.ng) {
            int64_t acc = 0;
            for (int g = 0; g < (int)threadIdx.x; ++g) acc += (end_t[g] - beg_t[g] + 31) & ~(int64_t)31;
            s_pref[threadIdx.x] = acc;
        }
        __syncthreads();
        {
            const int64_t total = s_pref[p.ng];
            int g = 0;
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;
                const int64_t i = beg_t[g] + (f0 - s_pref[g]) + lane;
                if (i >= end_t[g]) continue;
                const size_t qbase = (size_t)g * p.q.cap;
                const uint32_t *gn = nbr ? nbr + (size_t)g * n : nullptr;
                double *gsig = p.sigma + (size_t)g * n * 32;
                double *gcoef = p.coef + (size_t)g * n * 32;
                const int64_t v = p.q.q_v[qbase + i];
                const uint32_t m = p.q.q_m[qbase + i];
                wr[(size_t)g * n + v] = m;   // level L becomes the children masks of level L - 1
                if (m != 0)
                    pull_entry_thin<STORE_DELTA>(v, m, p.off[v], p.off[v + 1], p.col, gn, gsig, gcoef,
                                                 STORE_DELTA ? p.delta + (size_t)g * n * 32 : nullptr,
                                                 p.bcg + (size_t)g * n, p.accumulate);
            }
        }
        __syncthreads();   // s_pref is rewritten by the next level
        grid.sync();
        if (erase != nullptr) {
            const int64_t *eb = p.range_table + ((size_t)(L + 1) * 2 + 0) * p.G;
            const int64_t *ee = p.range_table + ((size_t)(L + 1) * 2 + 1) * p.G;
            if (threadIdx.x <= p.ng) {
                int64_t acc = 0;
                for (int g = 0; g < (int)threadIdx.x; ++g) acc += (ee[g] - eb[g] + 31) & ~(int64_t)31;
                s_pref[threadIdx.x] = acc;
            }
            __syncthreads();
            const int64_t total = s_pref[p.ng];
            int g = 0;
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;
                const int64_t i = eb[g] + (f0 - s_pref[g]) + lane;
                if (i < ee[g]) erase[(size_t)g * n + p.q.q_v[(size_t)g * p.q.cap + i]] = 0u;
            }
            __syncthreads();
            grid.sync();
        }
        nbr = wr;
        erase = wr;
        widx ^= 1;
    }
}

// ---- backward over level-ordered values ---------------------------------------------------
// Deep graphs are bound by random DRAM transactions: deep_backward_kernel touches ~10 64-byte
// lines per (vertex, lane) visit (sigma row, coef row, children's coef rows, BC partial, mask
// scratch; ncu: 687 B of DRAM traffic per visit at 2.8 TB/s, profiles/r2_deep_kernels_ncu.md).
// This variant keeps sigma and coef per queue ENTRY, in level order (DeepFwdParams::qs):
//   - an entry reads its sigma and writes its coef at q_off[i] + rank: sequential traffic;
//   - the vertex record maps a vertex to the queue entry it has at the level below (index + 1:
//     every entry writes it while its level is processed, into one of two words chosen by the
//     level's parity so that the probes of the level in flight are not disturbed; an index
//     outside the probed level's range is a stale one, so nothing is ever erased and one
//     grid-wide barrier per level is enough), and a parent finds a
//     child's lanes (q_m[j]) and coef (qc[q_off[j] + rank]) inside the few-MB window of that
//     level, which stays in L2;
//   - BC partials are added with atomics into ONE vector per batch (bc_acc, n doubles: L2
//     resident) instead of a read-modify-write of the 8-byte partial of (group, vertex) in a
//     G x n array: the per-vertex sums then depend on the order the atomics land in (last-bit
//     differences between runs), which is why only deep graphs take this path.
struct DeepBwdCompactParams {
    const int64_t *off;
    const int32_t *col;
    int64_t n;
    QueueParams q;               // q_v / q_m / cap
    const uint32_t *q_off;       // [G][cap] first value slot of an entry
    const int64_t *range_table;  // [level][0: begin, 1: end][G]
    const double *qs;            // [G][vcap] path counts in entry order
    double *qc;                  // [G][vcap] coef in entry order
    int64_t vcap;
    double *bc_acc;              // [n] BC partial of the batch (atomics), or nullptr
    double *bcg;                 // [G][n] per-group partials (used when bc_acc == nullptr)
    int ng, G;
    int hi, lo;                  // levels hi (the deepest level of the batch), hi - 1, ..., lo
    VertexState *vs;             // [G][n] (pos field)
    const uint32_t *q_a;         // first arc / degree of every entry as the forward sweep recorded them
    const uint32_t *q_arc;       // (nullptr when that sweep ran on another CSR: the cut-free one of hybir mode)
    const int4 *q_nb;            // neighbour ids of the entries of vertices with at most four arcs (nullptr with q_a)
};

__global__ void __launch_bounds__(kDeepThreads, BC_DEEP_MIN_BLOCKS_B) deep_backward_compact_kernel(const DeepBwdCompactParams p) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int64_t s_pref[kDeepMaxGroups + 1];
    __shared__ uint32_t s_cb[kDeepMaxGroups], s_ce[kDeepMaxGroups];   // entry range (+1) of the level below
    const int lane = threadIdx.x & 31;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = p.n;
    for (int L = p.hi; L >= p.lo; --L) {
        const bool deepest = L == p.hi;
        const int64_t *beg_t = p.range_table + ((size_t)L * 2 + 0) * p.G;
        const int64_t *end_t = p.range_table + ((size_t)L * 2 + 1) * p.G;
        for (int k = threadIdx.x; k < p.ng; k += blockDim.x) {
            s_cb[k] = deepest ? 1u : (uint32_t)p.range_table[((size_t)(L + 1) * 2 + 0) * p.G + k] + 1u;
            s_ce[k] = deepest ? 0u : (uint32_t)p.range_table[((size_t)(L + 1) * 2 + 1) * p.G + k];
        }
        padded_prefix(s_pref, p.ng, [&](int g) { return end_t[g] - beg_t[g]; });
        const int64_t total = s_pref[p.ng];
        int g = 0;
        for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
            while (f0 >= s_pref[g + 1]) ++g;
            const int64_t i = beg_t[g] + (f0 - s_pref[g]) + lane;
            if (i >= end_t[g]) continue;
            const size_t qbase = (size_t)g * p.q.cap;
            const size_t vbase = (size_t)g * p.vcap;
            VertexState *gvs = p.vs + (size_t)g * n;
            const int64_t v = p.q.q_v[qbase + i];
            const uint32_t m = p.q.q_m[qbase + i];
            const uint32_t at = p.q_off[qbase + i];
            // this entry is what level L - 1 will look for: the two index words alternate by level
            // parity, so the parents' probes of the level below (other word) are not disturbed
            if (L & 1) gvs[v].pos2 = (uint32_t)i + 1u;
            else gvs[v].pos = (uint32_t)i + 1u;
            if (m == 0) continue;
            int64_t a0, a1;
            bool cached = false;
            int4 nbv = make_int4(-1, -1, -1, -1);
            if (p.q_a != nullptr && (p.q_arc[qbase + i] >> 24) != 255u) {
                const uint32_t byte = p.q_arc[qbase + i] >> 24;
                a0 = p.q_a[qbase + i];
                a1 = a0 + entry_degree(byte);
                if (p.q_nb != nullptr && entry_cached(byte)) {
                    nbv = p.q_nb[qbase + i];
                    cached = true;
                }
            } else {
                a0 = p.off[v];
                a1 = p.off[v + 1];
            }
            const uint32_t cb = s_cb[g], ce = s_ce[g];   // a child's entry index + 1 lies in [cb, ce]
            double total_d = 0.0;
            uint32_t rest = m;
            int rank = 0;
            if (a1 - a0 <= kThinArcs || deepest) {
                // children: entry of every neighbour at the level below, its lanes and its first
                // value slot -- kThinArcs arcs at a time, one round trip per stage
                uint32_t cj[kThinArcs], cm[kThinArcs], co[kThinArcs];
#pragma unroll
                for (int k = 0; k < kThinArcs; ++k) {
                    cj[k] = 0;
                    if (!deepest && a0 + k < a1) {
                        const VertexState *child = gvs + (cached ? nb_at(nbv, k) : __ldg(p.col + a0 + k));
                        const uint32_t pj = ((L + 1) & 1) ? child->pos2 : child->pos;
                        if (pj >= cb && pj <= ce) cj[k] = pj;
                    }
                }
#pragma unroll
                for (int k = 0; k < kThinArcs; ++k) {
                    cm[k] = cj[k] ? p.q.q_m[qbase + cj[k] - 1] : 0u;
                    co[k] = cj[k] ? p.q_off[qbase + cj[k] - 1] : 0u;
                }
                while (rest) {
                    const int bit = __ffs(rest) - 1;
                    rest &= rest - 1;
                    const uint32_t lower = (1u << bit) - 1u;
                    double c[kThinArcs];
#pragma unroll
                    for (int k = 0; k < kThinArcs; ++k)
                        c[k] = ((cm[k] >> bit) & 1u) ? p.qc[vbase + co[k] + __popc(cm[k] & lower)] : 0.0;
                    double acc = 0.0;
#pragma unroll
                    for (int k = 0; k < kThinArcs; ++k)
                        if ((cm[k] >> bit) & 1u) acc += c[k];   // ascending arc order
                    const double sv = p.qs[vbase + at + rank];
                    const double d = sv * acc;
                    p.qc[vbase + at + rank] = (1.0 + d) / sv;
                    total_d += d;
                    ++rank;
                }
            } else {
                while (rest) {
                    const int bit = __ffs(rest) - 1;
                    rest &= rest - 1;
                    const uint32_t lower = (1u << bit) - 1u;
                    double acc = 0.0;
                    for (int64_t a = a0; a < a1; ++a) {
                        const VertexState *child = gvs + __ldg(p.col + a);
                        const uint32_t pj = ((L + 1) & 1) ? child->pos2 : child->pos;
                        if (pj < cb || pj > ce) continue;
                        const uint32_t mj = p.q.q_m[qbase + pj - 1];
                        if ((mj >> bit) & 1u) acc += p.qc[vbase + p.q_off[qbase + pj - 1] + __popc(mj & lower)];
                    }
                    const double sv = p.qs[vbase + at + rank];
                    const double d = sv * acc;
                    p.qc[vbase + at + rank] = (1.0 + d) / sv;
                    total_d += d;
                    ++rank;
                }
            }
            if (p.bc_acc != nullptr) {
                if (total_d != 0.0) atomicAdd(p.bc_acc + v, total_d);
            } else {
                p.bcg[(size_t)g * n + v] += total_d;
            }
        }
        __syncthreads();   // the shared ranges are rewritten by the next level
        grid.sync();
    }
}

}  // namespace bcb200
