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
__global__ void border_gather_queue_kernel(QueueParams q, const int64_t *level_end, int depth, int G,
                                           int64_t n, const int32_t *border_index,
                                           const double *sigma, int S, int32_t *D_out,
                                           double *S_out) {
    const size_t g = blockIdx.y;
    const int64_t end = (int64_t)q.q_count[g];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q.q_v[g * q.cap + i];
        const int j = border_index[v];
        if (j < 0) continue;
        uint32_t m = q.q_m[g * q.cap + i];
        const int level = level_of_entry(level_end, depth, G, g, i);
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const size_t at = (size_t)j * S + g * 32 + bit;
            D_out[at] = level;
            S_out[at] = sigma[(g * n + v) * 32 + bit];
        }
    }
}

// Border-table rows out of a queue-level sweep whose lanes are borders first .. first+count-1
// (border_table_kernel for the dense level rows); bm / sm pre-filled with kInf / 0.
__global__ void border_table_queue_kernel(QueueParams q, const int64_t *level_end, int depth, int G,
                                          int64_t n, const int32_t *border_index,
                                          const double *sigma, BorderGeom geo, int first, int count,
                                          int32_t *bm, double *sm) {
    const size_t g = blockIdx.y;
    const int64_t end = (int64_t)q.q_count[g];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < end;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q.q_v[g * q.cap + e];
        const int j = border_index[v];
        if (j < 0) continue;
        uint32_t m = q.q_m[g * q.cap + e];
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
            sm[at] = sigma[(g * n + v) * 32 + bit];
        }
    }
}

constexpr int kDeepThreads = 256;
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
    // level-ordered copy of the path counts (nullptr: off).  Entry i of group g owns the slots
    // q_off[g][i] .. + popc(q_m[i]) of qs[g][..], one per set lane in lane order: the backward
    // sweep of a deep graph then reads sigma (and writes coef) sequentially instead of one random
    // 8-byte access into the 256-byte row of the vertex (deep_backward_compact_kernel).
    double *qs;
    uint32_t *q_off;
    unsigned long long *v_count;   // [G] value slots handed out so far
    int64_t vcap;                  // value slots per group
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
                if (p.qs != nullptr) {
                    // value slots of the warp's entries: warp prefix of popc + one atomic per warp
                    const unsigned pc = __popc(any);
                    unsigned incl = pc;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned t = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += t;
                    }
                    const unsigned total = __shfl_sync(kFull, incl, 31);
                    unsigned long long base = 0;
                    if (lane == 0 && total) base = atomicAdd(p.v_count + g, (unsigned long long)total);
                    base = __shfl_sync(kFull, base, 0);
                    if (i < end) {
                        const unsigned long long at = base + incl - pc;
                        p.q_off[qbase + i] = (uint32_t)at;
                        if (at + pc <= (unsigned long long)p.vcap) {
                            const double *row = p.sigma + ((size_t)g * n + w) * 32;
                            double *out = p.qs + (size_t)g * p.vcap + at;
                            uint32_t m = any;
                            while (m) {
                                const int bit = __ffs(m) - 1;
                                m &= m - 1;
                                *out++ = row[bit];   // final: every push of the level is behind the barrier
                            }
                        }
                    }
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
//   - the scratch array maps a vertex to the queue entry it has at the level below (index + 1),
//     so a parent finds a child's lanes (q_m[j]) and coef (qc[q_off[j] + rank]) inside the
//     few-MB window of that level, which stays in L2;
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
    uint32_t *scr0, *scr1;       // all-zero scratch arrays on entry and on exit
};

__global__ void __launch_bounds__(kDeepThreads) deep_backward_compact_kernel(const DeepBwdCompactParams p) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int64_t s_pref[kDeepMaxGroups + 1];
    const int lane = threadIdx.x & 31;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = p.n;
    const uint32_t *below = nullptr;   // scratch holding entry index + 1 of the level below
    uint32_t *erase = nullptr;
    int widx = 0;
    for (int L = p.hi; L >= p.lo - 1; --L) {
        // iteration L = lo - 1 only erases what level lo left in the scratch array
        if (L >= p.lo) {
            uint32_t *wr = widx ? p.scr1 : p.scr0;
            const int64_t *beg_t = p.range_table + ((size_t)L * 2 + 0) * p.G;
            const int64_t *end_t = p.range_table + ((size_t)L * 2 + 1) * p.G;
            if (threadIdx.x <= p.ng) {
                int64_t acc = 0;
                for (int g = 0; g < (int)threadIdx.x; ++g) acc += (end_t[g] - beg_t[g] + 31) & ~(int64_t)31;
                s_pref[threadIdx.x] = acc;
            }
            __syncthreads();
            const int64_t total = s_pref[p.ng];
            int g = 0;
            for (int64_t f0 = gtid - lane; f0 < total; f0 += gthreads) {
                while (f0 >= s_pref[g + 1]) ++g;
                const int64_t i = beg_t[g] + (f0 - s_pref[g]) + lane;
                if (i >= end_t[g]) continue;
                const size_t qbase = (size_t)g * p.q.cap;
                const size_t vbase = (size_t)g * p.vcap;
                const int64_t v = p.q.q_v[qbase + i];
                const uint32_t m = p.q.q_m[qbase + i];
                const uint32_t at = p.q_off[qbase + i];
                wr[(size_t)g * n + v] = (uint32_t)i + 1u;
                if (m == 0) continue;
                const int64_t a0 = p.off[v], a1 = p.off[v + 1];
                double total_d = 0.0;
                // children: entry (index + 1) of every neighbour at the level below, its lanes and
                // its first value slot -- kThinArcs arcs at a time, one round trip per stage
                uint32_t rest = m;
                int rank = 0;
                if (a1 - a0 <= kThinArcs || below == nullptr) {
                    uint32_t cj[kThinArcs], cm[kThinArcs], co[kThinArcs];
#pragma unroll
                    for (int k = 0; k < kThinArcs; ++k) {
                        cj[k] = 0;
                        if (below != nullptr && a0 + k < a1) cj[k] = below[(size_t)g * n + __ldg(p.col + a0 + k)];
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
                            const uint32_t j = below[(size_t)g * n + __ldg(p.col + a)];
                            if (j == 0) continue;
                            const uint32_t mj = p.q.q_m[qbase + j - 1];
                            if ((mj >> bit) & 1u) acc += p.qc[vbase + p.q_off[qbase + j - 1] + __popc(mj & lower)];
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
            __syncthreads();   // s_pref is rewritten below
        }
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
        if (L >= p.lo) {
            uint32_t *wr = widx ? p.scr1 : p.scr0;
            below = wr;
            erase = wr;
            widx ^= 1;
        }
    }
}

}  // namespace bcb200
