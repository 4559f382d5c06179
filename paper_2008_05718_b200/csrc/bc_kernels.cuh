// bc_kernels.cuh -- sm_100a kernels of the batched Brandes engine.
//
// Data model.  A *group* is 32 BFS
// instances ("lanes") that advance in lock step, one bit per lane:
//   vis [g][v]      u32   lanes that have reached v so far (forward only)
//   lvl[L][g][v]    u32   lanes whose distance to v is exactly L  (this IS dist)
//   sigma[g][v][32] f64   path counts, one 256 B row per vertex
//   coef [g][v][32] f64   (1 + delta) / sigma, the value parents pull backward
// A warp owns a vertex (or a 32-arc-aligned chunk of a hub's adjacency): it
// filters 32 arcs at a time with lanes = arcs (one coalesced col_idx load, one
// 4 B mask probe per arc), stages the arcs that hit in shared memory, then
// switches to lanes = BFS instances and adds the neighbours' 256 B rows, one
// row per hit arc, predicated per lane.
// Pull direction on both phases: no atomics on fp64, sums run in CSR arc
// order, results are bit-reproducible.
//
// Reference arithmetic being replaced: the heap loop of initial_relax
// (reference pkg/src/hybir/relax.py:75-101) for sigma, process_level's
// vertex-pull branch (backward.py:95-103) for delta, accumulate_bc
// (backward.py:154-158) for the BC sum.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bcb200 {

// resident blocks per SM the compiler must allow (register cap = 65536 / (threads * blocks)):
// the forward kernel keeps 40 registers, the backward kernel runs better at 32 registers and
// full occupancy (measured both ways after every change of the gather loop)
#ifndef BC_MIN_BLOCKS_FWD
#define BC_MIN_BLOCKS_FWD 12
#endif
#ifndef BC_MIN_BLOCKS_BWD
#define BC_MIN_BLOCKS_BWD 16
#endif
#ifndef BC_WPB
#define BC_WPB 4
#endif

constexpr int kWarpsPerBlock = BC_WPB;
constexpr unsigned kFull = 0xffffffffu;

// -DBC_PROFILE: dev build that counts what the gather loops do (dumped per launch on stderr)
#ifdef BC_PROFILE
__device__ unsigned long long g_prof[16];
#define PROF_ADD(slot, value)                                                      \
    do {                                                                           \
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_prof[slot], (unsigned long long)(value)); \
    } while (0)
#else
#define PROF_ADD(slot, value) do { } while (0)
#endif

struct LevelParams {
    // graph (full CSR or the cut-arc-free CSR of a partitioning)
    const int64_t *off;
    const int32_t *col;
    // work items: hub chunks first, then vertex ranges (<= 32 vertices each)
    const int32_t *chk_v;
    const int64_t *chk_a0;
    const int64_t *chk_a1;
    int n_chk;
    const int32_t *rng_v0;
    const int32_t *rng_nv;
    int n_rng;
    int64_t n;
    // state, all indexed [group][...]
    uint32_t *vis;
    const uint32_t *nbr;  // forward: lvl[L-1]; backward: lvl[L+1] (nullptr at the deepest level)
    uint32_t *cur;        // lvl[L]: written forward, read backward
    double *sigma;
    double *coef;
    double *delta;  // only with STORE_DELTA
    double *bcg;    // [group][v] per-group BC partial sums
    double *pacc;   // [group][chunk][32] hub partial sums
    uint32_t *pmask;  // [group][chunk]
    // live[L][g] = lanes of group g whose level-L frontier is not empty.  A lane
    // whose frontier died (e.g. an isolated source) is dropped from every later
    // `want`, so exhausted instances stop costing adjacency scans.
    const uint32_t *live_prev;  // forward: live[L-1]; backward: live[L]
    uint32_t *live_cur;         // forward: live[L], OR-ed by this launch
    unsigned long long *counters;  // [0] n_r, [1] A_r, [2] T
    unsigned long long *lstat;     // forward: [0] vertices discovered, [1] their arcs, [2] largest degree,
                                   // [4] arcs scanned by this launch (byte model of the roofline); may be null
    int accumulate_bc;
    int count_scan;   // forward: add the arcs scanned into lstat[4] (one more atomic per item: off on timed runs)
    // forward sweeps of low-degree (deep) graphs without frontier queues: only vertices with a
    // neighbour in the previous level are scanned (mark_candidates_kernel); nullptr = scan all
    uint8_t *cand;   // [group][v]
    // weighted graphs (positive integer arc weights, WEIGHTED kernels only): level = distance,
    // an arc of weight wt ties level L to level L - wt (forward) / L + wt (backward)
    const int32_t *wgt;                  // per arc, CSR order
    const uint32_t *const *lvl_ptrs;     // lvl_ptrs[L] = mask array of level L
    const uint32_t *live_base;           // live[level][G]
    int level, max_level, wmax, G;
};

// Lanes a forward level still has to serve: those with a non-empty frontier in one of the
// last `wmax` levels (wmax = 1 for unit weights: the previous level).
__device__ __forceinline__ uint32_t forward_live(const uint32_t *live_base, int G, size_t g, int level,
                                                 int wmax) {
    uint32_t live = 0;
    for (int j = 1; j <= wmax && j <= level; ++j) live |= live_base[(size_t)(level - j) * G + g];
    return live;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    return x;
}

// Predicated read-only load: one LDG under a predicate, never a branch (the
// compiler turns `if (p) x = __ldg(..)` into divergent control flow here).
// NOALLOC: the line is not kept in L1.  Row gathers of a graph without hubs (Erdos-Renyi) never
// come back to a row while it is still in L1, and allocating them only evicts the level masks:
// -9 % on the whole pass there; on R-MAT the hubs' rows are re-read constantly and bypassing
// L1 costs +13 %, so the host picks the variant per graph (bc_engine.cu, `row_cache`).
template <bool NOALLOC>
__device__ __forceinline__ double ldg_if(const double *ptr, uint32_t pred) {
    double x;
    if (NOALLOC)
        asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.f64 %0, 0d0000000000000000;\n\t"
            "@q ld.global.nc.L1::no_allocate.f64 %0, [%1];\n\t}"
            : "=d"(x)
            : "l"(ptr), "r"(pred));
    else
        asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.f64 %0, 0d0000000000000000;\n\t"
            "@q ld.global.nc.f64 %0, [%1];\n\t}"
            : "=d"(x)
            : "l"(ptr), "r"(pred));
    return x;
}

// Neighbour ids are streamed: every 128-byte line of col_idx is used once by one warp.
__device__ __forceinline__ int32_t ld_col(const int32_t *ptr) {
#ifdef BC_COL_NOALLOC
    int32_t x;
    asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(x) : "l"(ptr));
    return x;
#else
    return __ldg(ptr);
#endif
}

#ifndef BC_STAGED_UNROLL_FWD
#define BC_STAGED_UNROLL_FWD 8
#endif
#ifndef BC_STAGED_UNROLL_BWD
#define BC_STAGED_UNROLL_BWD 4
#endif
constexpr int kStagedMax = BC_STAGED_UNROLL_FWD > BC_STAGED_UNROLL_BWD ? BC_STAGED_UNROLL_FWD : BC_STAGED_UNROLL_BWD;

struct WeightedProbe {
    const int32_t *wgt;
    const uint32_t *const *lvl_ptrs;
    size_t goff;     // group offset into a level array
    int level, max_level;
};

// Mask of the lanes for which arc k ties its endpoint w to the level being computed.
template <bool WEIGHTED, bool BWD>
__device__ __forceinline__ uint32_t probe_arc(int k, int32_t w, const uint32_t *__restrict__ nmask,
                                              const WeightedProbe &wp) {
    if (!WEIGHTED) return __ldg(nmask + w);
    const int wt = __ldg(wp.wgt + k);
    const int ls = BWD ? wp.level + wt : wp.level - wt;
    if (BWD ? ls > wp.max_level : ls < 0) return 0u;
    return __ldg(wp.lvl_ptrs[ls] + wp.goff + w);
}

// Staged row gather of one 32-arc slice: the hit arcs, compacted in arc order into a per-warp
// list in shared memory; every lane then reads one (neighbour, hit mask) entry per arc with a
// broadcast LDS (instead of two shuffles and a find-first-set) and adds the neighbour's row
// under its own bit.  ~6 instructions and two L1 wavefronts per hit arc.
template <bool BWD, bool NOALLOC>
__device__ __forceinline__ void gather_staged(unsigned any, uint32_t hit, int32_t w,
                                              const double *__restrict__ myval, int lane,
                                              double &acc) {
    constexpr int kU = BWD ? BC_STAGED_UNROLL_BWD : BC_STAGED_UNROLL_FWD;  // row loads in flight
#ifdef BC_EXACT_PAD
    __shared__ __align__(16) int2 s_rows[kWarpsPerBlock][32];
#else
    __shared__ int2 s_rows[kWarpsPerBlock][32 + kStagedMax];
#endif
    int2 *lst = s_rows[threadIdx.x >> 5];
    const int nh = __popc(any);
    const uint32_t lbit = 1u << lane;
    if (hit != 0) lst[__popc(any & (lbit - 1u))] = make_int2(w, (int)hit);
#ifdef BC_EXACT_PAD
    if (lane < ((-nh) & (kU - 1))) lst[nh + lane] = make_int2(0, 0);  // pad the last round: predicate off
#else
    if (lane < kU) lst[nh + lane] = make_int2(0, 0);  // pad the last round: predicate off
#endif
    __syncwarp();
    for (int i = 0; i < nh; i += kU) {
        int2 e[kU];
        double x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) e[u] = lst[i + u];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            x[u] = ldg_if<NOALLOC>(myval + (size_t)e[u].x * 32, (uint32_t)e[u].y & lbit);
#pragma unroll
        for (int u = 0; u < kU; ++u) acc += x[u];  // ascending arc order
    }
    __syncwarp();  // the next slice overwrites the list
}

// Scan arcs [0, n_arcs) of one vertex, relative to `col` (and to wp.wgt): 32-bit index
// arithmetic.  `want` (warp-uniform) = instances that still need a value.
//   filter, lanes = arcs: one coalesced col_idx load and one 4 B mask probe per arc,
//     hit = mask[neighbour] & want.  Two loads deep: neighbour ids are fetched two slices
//     ahead and masks one slice ahead, so the probe of the next slice never waits for its own
//     address, and `& want` is applied where the mask is consumed, not where it is loaded;
//   gather, lanes = instances: gather_staged() adds the rows of the arcs that hit, in
//     ascending arc order -- sums are deterministic and independent of the slice shape.
// tcount is a per-lane partial count of (arc, instance) hits (COUNT_T only).
template <bool COUNT_T, bool WEIGHTED = false, bool BWD = false, bool NOALLOC = false>
__device__ __forceinline__ void scan_arcs(int n_arcs, uint32_t want,
                                          const int32_t *__restrict__ col,
                                          const uint32_t *__restrict__ nmask,
                                          const double *__restrict__ val, int lane, double &acc,
                                          uint32_t &got, unsigned &tcount,
                                          const WeightedProbe &wp = WeightedProbe{}) {
    int32_t w_c = 0, w_n = 0;
    uint32_t m_c = 0;
    if (lane < n_arcs) w_c = ld_col(col + lane);
    if (lane + 32 < n_arcs) w_n = ld_col(col + 32 + lane);
    if (lane < n_arcs) m_c = probe_arc<WEIGHTED, BWD>(lane, w_c, nmask, wp);
    const double *myval = val + lane;
    for (int base = 0; base < n_arcs; base += 32) {
        const int32_t w = w_c;
        const uint32_t hit = m_c & want;
        w_c = w_n;
        m_c = 0;
        if (base + 32 + lane < n_arcs) m_c = probe_arc<WEIGHTED, BWD>(base + 32 + lane, w_c, nmask, wp);
        w_n = 0;
        if (base + 64 + lane < n_arcs) w_n = ld_col(col + base + 64 + lane);
        const unsigned any = __ballot_sync(kFull, hit != 0);
        PROF_ADD(0, 1);
        if (any == 0) continue;
        PROF_ADD(1, 1);
        PROF_ADD(2, __popc(any));
        PROF_ADD(3, __popc(want));
#ifdef BC_PROFILE
        {
            const unsigned prof_pairs = __reduce_add_sync(kFull, __popc(hit));
            const unsigned prof_lanes = __popc(__reduce_or_sync(kFull, hit));
            PROF_ADD(4, prof_pairs);
            PROF_ADD(5, prof_lanes);
        }
#endif
        if (COUNT_T) tcount += __popc(hit);  // lanes = arcs here: a per-lane partial
        got |= __reduce_or_sync(kFull, hit);
        gather_staged<BWD, NOALLOC>(any, hit, w, myval, lane, acc);
    }
}

// Forward: lanes in `got` have just been discovered at this level with path
// count acc.  `seen` = vis[v] before the level.
__device__ __forceinline__ void finalize_forward(int64_t v, uint32_t seen, uint32_t got,
                                                 double acc, int lane, uint32_t *vis,
                                                 uint32_t *cur, double *sigma) {
    if ((got >> lane) & 1u) sigma[(size_t)v * 32 + lane] = acc;
    if (lane == 0) {
        cur[v] = got;
        if (got) vis[v] = seen | got;
    }
}

// Backward: lanes in `mine` sit at this level; acc = sum of coef over their
// DAG children.  delta = sigma * acc (backward.py:95-103 with the division
// hoisted: (sigma_v / sigma_u)(1 + delta_u) = sigma_v * coef_u).
// *ptr = 0 once `loaded` (the value just read from *ptr) has arrived.  A store issued while
// the same thread's load of that address is still in flight stalls the memory pipe for the
// whole round trip (measured: the backward sweep went from 18 ms to 51 ms with the store placed
// right behind the load), so the zero is tied to the loaded value.
__device__ __forceinline__ void clear_after_use(double *ptr, double loaded) {
    double zero = 0.0;
    asm volatile("" : "+d"(zero) : "d"(loaded));
    *ptr = zero;
}

// `accumulate`: bit 0 = add delta into the BC partials, bit 1 = clear sigma.
// This is the last read of sigma[v][lane] in a batch, so shallow-graph runs
// clear it on the way out: the top-down push levels add path counts with
// atomics and need zeros under every pair they discover, and clearing the
// pairs a batch reached costs less than a memset of the whole array (5 GB per
// batch on R-MAT scale 20) at the start of the next batch.  On deep graphs the
// extra dirty sector per visit costs more than the memset, so the host leaves
// bit 1 off there.
template <bool STORE_DELTA>
__device__ __forceinline__ void finalize_backward(int64_t v, uint32_t mine, double acc, int lane,
                                                  double *sigma, double *coef,
                                                  double *delta, double *bcg, int accumulate) {
    double contrib = 0.0;
    if ((mine >> lane) & 1u) {
        const size_t idx = (size_t)v * 32 + lane;
        const double sv = sigma[idx];
        const double d = sv * acc;
        coef[idx] = (1.0 + d) / sv;
        if (STORE_DELTA) delta[idx] = d;
        contrib = d;
        if (!STORE_DELTA && (accumulate & 2)) clear_after_use(sigma + idx, sv);
    }
    if (accumulate & 1) {
        const double s = warp_sum(contrib);
        if (lane == 0) bcg[v] += s;
    }
}

// One BFS level, forward (discover level L from level L-1) or backward
// (accumulate level L from level L+1).  grid = (ceil(items / 8), groups).
template <bool BWD, bool STORE_DELTA, bool WEIGHTED = false, bool NOALLOC = false>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, BWD ? BC_MIN_BLOCKS_BWD : BC_MIN_BLOCKS_FWD) level_kernel(const LevelParams p) {
    const size_t g = blockIdx.y;
    // forward: instances still expanding; backward: instances present at this level
    const uint32_t live = (WEIGHTED && !BWD) ? forward_live(p.live_base, p.G, g, p.level, p.wmax)
                                             : p.live_prev[g];
    WeightedProbe wp{};
    if (WEIGHTED) {
        wp.wgt = p.wgt;
        wp.lvl_ptrs = p.lvl_ptrs;
        wp.goff = g * (size_t)p.n;
        wp.level = p.level;
        wp.max_level = p.max_level;
    }
    if (live == 0) return;  // also covers speculative launches past the last level
    const int lane = threadIdx.x & 31;
    const int64_t item = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (item >= (int64_t)p.n_chk + p.n_rng) return;
    uint32_t *vis = p.vis + g * p.n;
    // weighted: the masks come from lvl_ptrs; `nbr` only says whether there is anything to pull
    const uint32_t *nbr = p.nbr ? p.nbr + g * p.n : nullptr;
    uint32_t *cur = p.cur + g * p.n;
    double *sigma = p.sigma + g * p.n * 32;
    double *coef = p.coef + g * p.n * 32;
    double *delta = STORE_DELTA ? p.delta + g * p.n * 32 : nullptr;
    const double *val = BWD ? coef : sigma;

    unsigned c_t = 0;  // per-lane partial count of (arc, instance) hits

    if (item < p.n_chk) {
        // ---- a slice of a hub's adjacency: partial sum into the hub buffers
        const int32_t v = p.chk_v[item];
        const uint32_t want = BWD ? cur[v] : (~vis[v] & live);
        double acc = 0.0;
        uint32_t got = 0;
        if (want != 0 && nbr != nullptr) {
            const int64_t a0 = p.chk_a0[item];
            if (WEIGHTED) wp.wgt += a0;
            scan_arcs<!BWD, WEIGHTED, BWD, NOALLOC>((int)(p.chk_a1[item] - a0), want, p.col + a0, nbr, val,
                                           lane, acc, got, c_t, wp);
        }
        const size_t slot = g * (size_t)p.n_chk + item;
        if (want != 0) p.pacc[slot * 32 + lane] = acc;
        if (lane == 0) p.pmask[slot] = got;
        if (!BWD) {
            const unsigned t = __reduce_add_sync(kFull, c_t);
            if (lane == 0 && t) atomicAdd(p.counters + 2, (unsigned long long)t);
            if (lane == 0 && p.count_scan && p.lstat != nullptr && want != 0 && nbr != nullptr)
                atomicAdd(p.lstat + 4, (unsigned long long)(p.chk_a1[item] - p.chk_a0[item]));
        }
    } else {
        // ---- up to 32 consecutive non-hub vertices, one per lane for the set-up and for what
        // is written per vertex afterwards (level bits, visited bits, counters)
        const int64_t r = item - p.n_chk;
        const int32_t v0 = p.rng_v0[r];
        const int32_t nv = p.rng_nv[r];
        const int64_t a0 = p.off[v0];  // arcs of the item are consecutive: 32-bit offsets from here
        uint32_t mine = 0, seen = 0;
        int rb = 0, deg = 0;
        if (lane < nv) {
            const int64_t v = (int64_t)v0 + lane;
            rb = (int)(p.off[v] - a0);
            deg = (int)(p.off[v + 1] - a0) - rb;
            if (BWD) {
                mine = cur[v];
            } else {
                seen = vis[v];
                mine = ~seen & live;
                if (p.cand != nullptr) {
                    uint8_t *c = p.cand + g * p.n + v;
                    if (*c) *c = 0;      // consumed
                    else mine = 0;       // no neighbour in the previous level
                }
            }
        }
        const int32_t *colp = p.col + a0;
        if (WEIGHTED) wp.wgt += a0;
        uint32_t mygot = 0;  // forward: what this lane's vertex discovered
        unsigned need = __ballot_sync(kFull, mine != 0 && (BWD || deg > 0));
        if (!BWD && p.count_scan && p.lstat != nullptr && need != 0 && nbr != nullptr) {
            // arcs this item scans (one col_idx word + one mask probe each): byte model of the roofline
            const unsigned c_scan = __reduce_add_sync(kFull, (mine != 0) ? (unsigned)deg : 0u);
            if (lane == 0) atomicAdd(p.lstat + 4, (unsigned long long)c_scan);
        }
        while (need) {
            const int i = __ffs(need) - 1;
            need &= need - 1;
            const int64_t v = (int64_t)v0 + i;
            const uint32_t want = __shfl_sync(kFull, mine, i);
            const int vb = __shfl_sync(kFull, rb, i);
            const int vd = __shfl_sync(kFull, deg, i);
            double acc = 0.0;
            uint32_t got = 0;
            if (nbr != nullptr) {
                WeightedProbe wv = wp;
                if (WEIGHTED) wv.wgt += vb;
                scan_arcs<!BWD, WEIGHTED, BWD, NOALLOC>(vd, want, colp + vb, nbr, val, lane, acc, got, c_t, wv);
            }
            if (BWD) {
                finalize_backward<STORE_DELTA>(v, want, acc, lane, sigma, coef, delta,
                                               p.bcg + g * p.n, p.accumulate_bc);
            } else {
                if ((got >> lane) & 1u) sigma[(size_t)v * 32 + lane] = acc;
                if (lane == i) mygot = got;
            }
        }
        if (!BWD) {
            // one coalesced store per array instead of two lane-0 stores per vertex
            if (lane < nv) {
                const int64_t v = (int64_t)v0 + lane;
                cur[v] = mygot;
                if (mygot) vis[v] = seen | mygot;
            }
            // counters, once per item (an item holds <= 32 vertices and <= 2 * item_arcs arcs)
            const unsigned newv = __ballot_sync(kFull, mygot != 0);
            const unsigned t = __reduce_add_sync(kFull, c_t);
            if (newv) {
                const unsigned pc = __popc(mygot);
                const unsigned c_nr = __reduce_add_sync(kFull, pc);
                const unsigned c_ar = __reduce_add_sync(kFull, pc * (unsigned)deg);
                const uint32_t any_new = __reduce_or_sync(kFull, mygot);
                unsigned c_fa = 0, c_md = 0;
                if (p.lstat) {
                    c_fa = __reduce_add_sync(kFull, mygot ? (unsigned)deg : 0u);
                    c_md = __reduce_max_sync(kFull, mygot ? (unsigned)deg : 0u);
                }
                if (lane == 0) {
                    atomicOr(p.live_cur + g, any_new);
                    atomicAdd(p.counters + 0, (unsigned long long)c_nr);
                    atomicAdd(p.counters + 1, (unsigned long long)c_ar);
                    if (p.lstat) {
                        atomicAdd(p.lstat + 0, (unsigned long long)__popc(newv));
                        atomicAdd(p.lstat + 1, (unsigned long long)c_fa);
                        atomicMax(p.lstat + 2, (unsigned long long)c_md);
                    }
                }
            }
            if (lane == 0 && t) atomicAdd(p.counters + 2, (unsigned long long)t);
        }
    }
}

struct HubParams {
    const int64_t *off;
    const int32_t *hub_v;
    const int32_t *hub_c0;  // first chunk of the hub
    const int32_t *hub_nc;  // number of chunks
    int n_hub;
    int n_chk;
    int64_t n;
    uint32_t *vis;
    uint32_t *cur;
    double *sigma;
    double *coef;
    double *delta;
    double *bcg;
    const double *pacc;
    const uint32_t *pmask;
    const uint32_t *live_prev;
    uint32_t *live_cur;
    unsigned long long *counters;
    unsigned long long *lstat;
    int accumulate_bc;
    const uint32_t *live_base;   // weighted forward levels: see forward_live()
    int level, wmax, G;
};

// Adds a hub's chunk partials in chunk order (= arc order) and finalises it.
template <bool BWD, bool STORE_DELTA>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) hub_kernel(const HubParams p) {
    const size_t g = blockIdx.y;
    const uint32_t live = (!BWD && p.wmax > 1) ? forward_live(p.live_base, p.G, g, p.level, p.wmax)
                                               : p.live_prev[g];
    if (live == 0) return;
    const int lane = threadIdx.x & 31;
    const int h = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (h >= p.n_hub) return;
    const int64_t v = p.hub_v[h];
    uint32_t *vis = p.vis + g * p.n;
    uint32_t *cur = p.cur + g * p.n;
    const uint32_t want = BWD ? cur[v] : (~vis[v] & live);
    if (want == 0) {
        if (!BWD && lane == 0) cur[v] = 0;
        return;
    }
    const int c0 = p.hub_c0[h], nc = p.hub_nc[h];
    double acc = 0.0;
    uint32_t got = 0;
    for (int c = 0; c < nc; ++c) {
        const size_t slot = g * (size_t)p.n_chk + c0 + c;
        acc += p.pacc[slot * 32 + lane];
        got |= p.pmask[slot];
    }
    if (BWD) {
        finalize_backward<STORE_DELTA>(v, want, acc, lane, p.sigma + g * p.n * 32,
                                       p.coef + g * p.n * 32,
                                       STORE_DELTA ? p.delta + g * p.n * 32 : nullptr,
                                       p.bcg + g * p.n, p.accumulate_bc);
    } else {
        finalize_forward(v, vis[v], got, acc, lane, vis, cur, p.sigma + g * p.n * 32);
        if (lane == 0 && got) {
            atomicOr(p.live_cur + g, got);
            atomicAdd(p.counters + 0, (unsigned long long)__popc(got));
            atomicAdd(p.counters + 1,
                      (unsigned long long)__popc(got) * (unsigned long long)(p.off[v + 1] - p.off[v]));
            if (p.lstat) {
                atomicAdd(p.lstat + 0, 1ull);
                atomicAdd(p.lstat + 1, (unsigned long long)(p.off[v + 1] - p.off[v]));
                atomicMax(p.lstat + 2, (unsigned long long)(p.off[v + 1] - p.off[v]));
            }
        }
    }
}

// cand[g][w] = 1 for every neighbour w of a vertex in the previous level.  A dense pull level
// scans the arcs of every vertex some lane has not reached; on a road network that is the whole
// graph at each of thousands of levels.  With the candidates marked first (work proportional to
// the frontier) the pull only scans vertices that can be discovered.  One thread per vertex.
__global__ void mark_candidates_kernel(const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                       int64_t n, const uint32_t *__restrict__ prev,
                                       const uint32_t *live_prev, uint8_t *cand) {
    const size_t g = blockIdx.y;
    if (live_prev[g] == 0) return;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        if (prev[g * n + v] == 0) continue;
        for (int64_t a = off[v]; a < off[v + 1]; ++a) cand[g * n + __ldg(col + a)] = 1;
    }
}

// vis[g][v] = lanes of group g that do not exist in this batch (so that
// ~vis never selects them); lvl0[g][v] = 0.
__global__ void init_state_kernel(uint32_t *vis, uint32_t *lvl0, int64_t n, int batch_count) {
    const size_t g = blockIdx.y;
    const int lanes = min(32, batch_count - (int)g * 32);
    const uint32_t dead = lanes >= 32 ? 0u : ~((1u << lanes) - 1u);
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        vis[g * n + v] = dead;
        lvl0[g * n + v] = 0u;
    }
}

// Sources of the batch become level-0 seeds with one path each (relax.py:62-72
// for a single seed (s, 0, 1)).
__global__ void seed_sources_kernel(const int64_t *src, int batch_count, int64_t n, uint32_t *vis,
                                    uint32_t *lvl0, double *sigma, uint32_t *live0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch_count) return;
    const size_t g = i >> 5;
    const int lane = i & 31;
    const int64_t v = src[i];
    atomicOr(live0 + g, 1u << lane);
    if (v < 0) return;   // graph-partitioned runs: the lane's source lives on another rank
    atomicOr(vis + g * n + v, 1u << lane);
    atomicOr(lvl0 + g * n + v, 1u << lane);
    sigma[(g * n + v) * 32 + lane] = 1.0;
}

// sigma = 1 at the sources (rows cleared after begin_batch: see forward_adaptive).
__global__ void source_sigma_kernel(const int64_t *src, int batch_count, int64_t n, double *sigma) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch_count) return;
    const size_t g = i >> 5;
    if (src[i] < 0) return;
    sigma[(g * n + src[i]) * 32 + (i & 31)] = 1.0;
}

// The sources sit at level 0, which the backward sweep does not visit: clear their
// path counts separately (see finalize_backward).
__global__ void clear_source_sigma_kernel(const int64_t *src, int batch_count, int64_t n, double *sigma) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch_count) return;
    const size_t g = i >> 5;
    if (src[i] < 0) return;
    sigma[(g * n + src[i]) * 32 + (i & 31)] = 0.0;
}

// bc[v] += sum over groups, in group order; the per-group partials are reset.
// old_of_new (or nullptr): the partials are indexed by renumbered vertices (bc_relabel.cuh), bc by the caller's.
__global__ void reduce_bc_kernel(double *bc, double *bcg, int64_t n, int groups, const int32_t *old_of_new = nullptr) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        int g = 0;
        for (; g + 4 <= groups; g += 4) {     // four loads in flight, added in group order
            double x[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) x[k] = bcg[(size_t)(g + k) * n + v];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                s += x[k];
                if (x[k] != 0.0) bcg[(size_t)(g + k) * n + v] = 0.0;
            }
        }
        for (; g < groups; ++g) {
            const double x = bcg[(size_t)g * n + v];
            s += x;
            if (x != 0.0) bcg[(size_t)g * n + v] = 0.0;
        }
        if (s != 0.0) bc[old_of_new ? old_of_new[v] : v] += s;
    }
}

// Deep graphs: the batch's BC partial (one vector, filled with atomics by
// deep_backward_compact_kernel) joins the per-group partials of group 0 and is reset.
__global__ void bc_acc_flush_kernel(double *bc_acc, double *bcg0, int64_t n) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const double x = bc_acc[v];
        if (x != 0.0) {
            bcg0[v] += x;
            bc_acc[v] = 0.0;
        }
    }
}

// Inspection: scatter level L of every lane into per-source rows.
__global__ void extract_level_kernel(const uint32_t *lvl, const uint32_t *live_level,
                                     const double *sigma, const double *delta, int64_t n, int level,
                                     int32_t *dist_out, double *sigma_out, double *delta_out) {
    const size_t g = blockIdx.y;
    if (live_level[g] == 0) return;  // the level row of a dead group was never written
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        uint32_t m = lvl[g * n + v];
        while (m) {
            const int lane = __ffs(m) - 1;
            m &= m - 1;
            const size_t row = (g * 32 + lane) * (size_t)n + v;
            const size_t idx = (g * n + v) * 32 + lane;
            if (dist_out) dist_out[row] = level;
            if (sigma_out) sigma_out[row] = sigma[idx];
            if (delta_out) delta_out[row] = delta[idx];
        }
    }
}

// ------------------------------------------------------------------------------------
// Sparse levels: frontier queues and top-down (push) expansion.
//
// A level whose frontier is small is kept as a queue of (vertex, lane mask)
// entries per group instead of a dense mask array, and is produced top-down:
// every frontier vertex pushes along its arcs into the vertices its lanes have
// not seen.  Path counts are added with red.global.add.f64 -- they are
// integer-valued, so the sum is exact in any order and the result stays
// deterministic (sigma is zeroed per batch when push may run).  The host picks
// push or pull per level from the frontier's arc count (direction-optimising
// switch); dense pull levels read a queue level through a scratch mask array.
// ------------------------------------------------------------------------------------

struct QueueParams {
    int32_t *q_v;          // [group][cap] vertex of the entry
    uint32_t *q_m;         // [group][cap] lanes at that vertex
    int64_t cap;           // entries per group
    unsigned long long *q_count;  // [group] entries used so far
    const int64_t *q_beg;  // [group] first entry of the level being read
    const int64_t *q_end;  // [group] one past its last entry
};

constexpr int kStage = 128;  // per-warp shared-memory staging buffer (queue entries)

// A queue entry is walked by one warp (or one thread on thin levels).  Entries of
// vertices with more than kHeavyDeg arcs are left to fwd_push_heavy_kernel, which
// takes one warp per kHeavySlice-arc slice of the adjacency: R-MAT hubs hold tens
// of thousands of arcs and sit in the first levels of almost every source.
constexpr int kHeavyDeg = 2048;
constexpr int kHeavySlice = 256;   // arcs per record: short dependent chains, thousands of warps
struct HeavyRec {
    int64_t qi;     // queue entry (index inside the group's queue)
    int32_t g;      // group
    int32_t slice;  // arcs [slice * kHeavySlice, (slice + 1) * kHeavySlice) of the vertex
};

// Appends the slices of a heavy queue entry (called by one thread).
__device__ __forceinline__ void append_heavy(HeavyRec *heavy, unsigned long long *heavy_count,
                                             int64_t qi, int g, int64_t deg) {
    const int slices = (int)((deg + kHeavySlice - 1) / kHeavySlice);
    const unsigned long long at = atomicAdd(heavy_count, (unsigned long long)slices);
    for (int s = 0; s < slices; ++s) heavy[at + s] = HeavyRec{qi, g, s};
}

// Top-down expansion of level L-1 (a queue) into level L.  Lanes = arcs.
// next[] must be all zero on entry; it holds the new level's masks on exit
// (push_post_kernel moves them into the queue and clears next[] again).
__global__ void __launch_bounds__(kWarpsPerBlock * 32) fwd_push_kernel(
    const int64_t *__restrict__ off, const int32_t *__restrict__ col, int64_t n, QueueParams q,
    const uint32_t *__restrict__ vis, uint32_t *next, double *sigma,
    unsigned long long *counters) {
    __shared__ int32_t stage[kWarpsPerBlock][kStage];
    const size_t g = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t beg = q.q_beg[g], end = q.q_end[g];
    const int64_t stride = (int64_t)gridDim.x * kWarpsPerBlock;
    const uint32_t *gvis = vis + g * n;
    uint32_t *gnext = next + g * n;
    double *gsig = sigma + g * n * 32;
    int staged = 0;      // warp-uniform
    unsigned c_t = 0;
    auto flush = [&]() {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(q.q_count + g, (unsigned long long)staged);
        base = __shfl_sync(kFull, base, 0);
        for (int i = lane; i < staged; i += 32) q.q_v[g * q.cap + base + i] = stage[warp][i];
        staged = 0;
        __syncwarp();
    };
    for (int64_t i = beg + (int64_t)blockIdx.x * kWarpsPerBlock + warp; i < end; i += stride) {
        const int32_t u = q.q_v[g * q.cap + i];
        const uint32_t mask = q.q_m[g * q.cap + i];
        const int64_t b = off[u], e = off[u + 1];
        if (e - b > kHeavyDeg) continue;  // fwd_push_heavy_kernel takes it slice by slice
        const double *urow = gsig + (size_t)u * 32;
        for (int64_t base = b; base < e; base += 32) {
            const int64_t k = base + lane;
            bool fresh_vertex = false;
            int32_t w = 0;
            if (k < e) {
                w = __ldg(col + k);
                uint32_t fresh = mask & ~gvis[w];
                if (fresh) {
                    const uint32_t old = atomicOr(gnext + w, fresh);
                    fresh_vertex = old == 0;
                    double *wrow = gsig + (size_t)w * 32;
                    while (fresh) {
                        const int bit = __ffs(fresh) - 1;
                        fresh &= fresh - 1;
                        atomicAdd(wrow + bit, urow[bit]);   // exact: integer-valued fp64
                        ++c_t;
                    }
                }
            }
            const unsigned newm = __ballot_sync(kFull, fresh_vertex);
            if (newm) {
                if (fresh_vertex) stage[warp][staged + __popc(newm & ((1u << lane) - 1u))] = w;
                staged += __popc(newm);
                __syncwarp();
                if (staged > kStage - 32) flush();
            }
        }
    }
    if (staged) flush();
    const unsigned t = __reduce_add_sync(kFull, c_t);
    if (lane == 0 && t) atomicAdd(counters + 2, (unsigned long long)t);
}

// ---- thread-per-entry work of the thin (low-degree) levels ---------------------------------
// These levels are latency-bound: a thread's work is a chain of dependent random accesses
// (adjacency word -> visited word -> atomic on the next-level word), and with one arc per loop
// trip the chain is 3 round trips PER ARC.  The helpers below take the arcs kThinArcs at a
// time and issue each stage for all of them before anything is consumed, so a whole entry of a
// road-like graph (degree <= 4) costs 3 round trips in all (ncu of the persistent sweeps:
// 5-8 % issue utilisation, long-scoreboard + barrier stalls; profiles/r2_deep_kernels_ncu.md).
constexpr int kThinArcs = 4;

// Top-down push of one frontier entry (u, mask) along its arcs [a, e): new lanes are OR-ed into
// next[w], path counts added with red.global.add.f64 (integer-valued, exact in any order), and
// every vertex that was not in the next level yet is handed to `stage_vertex` under a
// warp-wide ballot (all 32 threads of the warp call this together; `rounds` = largest degree
// in the warp).
template <typename StageFn>
__device__ __forceinline__ void push_entry_thin(int64_t a, int64_t e, int rounds, uint32_t mask,
                                                const int32_t *__restrict__ col,
                                                const uint32_t *__restrict__ gvis, uint32_t *gnext,
                                                double *gsig, const double *urow, unsigned &c_t,
                                                StageFn stage_vertex) {
    // path count of the entry's first lane, fetched beside the adjacency (most entries of a
    // thin level carry one lane)
    const int bit0 = mask ? __ffs(mask) - 1 : 0;
    const double s0 = (a < e) ? urow[bit0] : 0.0;
    for (int r0 = 0; r0 < rounds; r0 += kThinArcs) {
        int32_t w[kThinArcs];
        uint32_t fresh[kThinArcs], old[kThinArcs];
#pragma unroll
        for (int k = 0; k < kThinArcs; ++k) w[k] = (a + r0 + k < e) ? __ldg(col + a + r0 + k) : -1;
#pragma unroll
        for (int k = 0; k < kThinArcs; ++k) fresh[k] = (w[k] >= 0) ? (mask & ~gvis[w[k]]) : 0u;
#pragma unroll
        for (int k = 0; k < kThinArcs; ++k) old[k] = fresh[k] ? atomicOr(gnext + w[k], fresh[k]) : 1u;
#pragma unroll
        for (int k = 0; k < kThinArcs; ++k) {
            uint32_t f = fresh[k];
            if (f == 0) continue;
            double *wrow = gsig + (size_t)w[k] * 32;
            while (f) {
                const int bit = __ffs(f) - 1;
                f &= f - 1;
                atomicAdd(wrow + bit, bit == bit0 ? s0 : urow[bit]);
                ++c_t;
            }
        }
#pragma unroll
        for (int k = 0; k < kThinArcs; ++k) {
            if (r0 + k >= rounds) break;                      // warp-uniform
            stage_vertex(fresh[k] != 0 && old[k] == 0, w[k]);
        }
    }
}

// Backward pull of one queue entry (v, want) over its arcs [a0, a1): per lane of the entry the
// children's coef summed in arc order (process_level vertex-pull, backward.py:95-103), then
// delta, coef and the BC partial -- the arithmetic of scan_arcs + finalize_backward, serial.
template <bool STORE_DELTA>
__device__ __forceinline__ void pull_entry_thin(int64_t v, uint32_t want, int64_t a0, int64_t a1,
                                                const int32_t *__restrict__ col, const uint32_t *gn,
                                                double *gsig, double *gcoef, double *gdelta,
                                                double *gbcg, int accumulate) {
    double total = 0.0;
    const int bit_first = __ffs(want) - 1;
    const double sv_first = gsig[(size_t)v * 32 + bit_first];   // independent of the arc chain
    if (a1 - a0 <= kThinArcs || gn == nullptr) {
        // the whole adjacency in registers: one round trip per stage
        int32_t w[kThinArcs];
        uint32_t nm[kThinArcs];
#pragma unroll
        for (int k = 0; k < kThinArcs; ++k) w[k] = (gn != nullptr && a0 + k < a1) ? __ldg(col + a0 + k) : -1;
#pragma unroll
        for (int k = 0; k < kThinArcs; ++k) nm[k] = (w[k] >= 0) ? __ldg(gn + w[k]) : 0u;
        uint32_t rest = want;
        while (rest) {
            const int bit = __ffs(rest) - 1;
            rest &= rest - 1;
            double c[kThinArcs];
#pragma unroll
            for (int k = 0; k < kThinArcs; ++k)
                c[k] = ((nm[k] >> bit) & 1u) ? gcoef[(size_t)w[k] * 32 + bit] : 0.0;
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < kThinArcs; ++k)
                if ((nm[k] >> bit) & 1u) acc += c[k];            // ascending arc order
            const size_t idx = (size_t)v * 32 + bit;
            const double sv = bit == bit_first ? sv_first : gsig[idx];
            const double d = sv * acc;
            gcoef[idx] = (1.0 + d) / sv;
            if (STORE_DELTA) gdelta[idx] = d;
            else if (accumulate & 2) clear_after_use(gsig + idx, sv);   // see finalize_backward
            total += d;
        }
    } else {
        uint32_t rest = want;
        while (rest) {
            const int bit = __ffs(rest) - 1;
            rest &= rest - 1;
            double acc = 0.0;
            for (int64_t b = a0; b < a1; b += kThinArcs) {
                int32_t w[kThinArcs];
                uint32_t nm[kThinArcs];
                double c[kThinArcs];
#pragma unroll
                for (int k = 0; k < kThinArcs; ++k) w[k] = (b + k < a1) ? __ldg(col + b + k) : -1;
#pragma unroll
                for (int k = 0; k < kThinArcs; ++k) nm[k] = (w[k] >= 0) ? __ldg(gn + w[k]) : 0u;
#pragma unroll
                for (int k = 0; k < kThinArcs; ++k)
                    c[k] = ((nm[k] >> bit) & 1u) ? gcoef[(size_t)w[k] * 32 + bit] : 0.0;
#pragma unroll
                for (int k = 0; k < kThinArcs; ++k)
                    if ((nm[k] >> bit) & 1u) acc += c[k];
            }
            const size_t idx = (size_t)v * 32 + bit;
            const double sv = bit == bit_first ? sv_first : gsig[idx];
            const double d = sv * acc;
            gcoef[idx] = (1.0 + d) / sv;
            if (STORE_DELTA) gdelta[idx] = d;
            else if (accumulate & 2) clear_after_use(gsig + idx, sv);
            total += d;
        }
    }
    if (accumulate & 1) gbcg[v] += total;
}

// Thin variant for levels of low-degree vertices (road-like graphs): one THREAD
// per queue entry walks its few arcs, so a warp advances 32 frontier vertices
// at once instead of leaving 29 of 32 lanes idle on a 3-arc adjacency.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) fwd_push_thin_kernel(
    const int64_t *__restrict__ off, const int32_t *__restrict__ col, int64_t n, QueueParams q,
    const uint32_t *__restrict__ vis, uint32_t *next, double *sigma,
    unsigned long long *counters) {
    __shared__ int32_t stage[kWarpsPerBlock][kStage];
    const size_t g = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t beg = q.q_beg[g], end = q.q_end[g];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint32_t *gvis = vis + g * n;
    uint32_t *gnext = next + g * n;
    double *gsig = sigma + g * n * 32;
    int staged = 0;  // warp-uniform
    unsigned c_t = 0;
    auto flush = [&]() {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(q.q_count + g, (unsigned long long)staged);
        base = __shfl_sync(kFull, base, 0);
        for (int i = lane; i < staged; i += 32) q.q_v[g * q.cap + base + i] = stage[warp][i];
        staged = 0;
        __syncwarp();
    };
    // warp-uniform trip count: every lane of the warp runs the same number of rounds
    for (int64_t i0 = beg + (int64_t)blockIdx.x * blockDim.x + warp * 32; i0 < end; i0 += stride) {
        const int64_t i = i0 + lane;
        int32_t u = 0;
        uint32_t mask = 0;
        int64_t a = 0, e = 0;
        if (i < end) {
            u = q.q_v[g * q.cap + i];
            mask = q.q_m[g * q.cap + i];
            a = off[u];
            e = off[u + 1];
            if (e - a > kHeavyDeg) e = a;  // left to fwd_push_heavy_kernel
        }
        int rounds = (int)(e - a);
        rounds = __reduce_max_sync(kFull, rounds);
        const double *urow = gsig + (size_t)u * 32;
        push_entry_thin(a, e, rounds, mask, col, gvis, gnext, gsig, urow, c_t,
                        [&](bool fresh_vertex, int32_t w) {
                            const unsigned newm = __ballot_sync(kFull, fresh_vertex);
                            if (newm) {
                                if (fresh_vertex) stage[warp][staged + __popc(newm & ((1u << lane) - 1u))] = w;
                                staged += __popc(newm);
                                __syncwarp();
                                if (staged > kStage - 32) flush();
                            }
                        });
    }
    if (staged) flush();
    const unsigned t = __reduce_add_sync(kFull, c_t);
    if (lane == 0 && t) atomicAdd(counters + 2, (unsigned long long)t);
}

// Top-down expansion of the heavy entries of level L-1: one warp per record
// (a kHeavySlice-arc slice of one frontier vertex), same arithmetic as fwd_push_kernel.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) fwd_push_heavy_kernel(
    const int64_t *__restrict__ off, const int32_t *__restrict__ col, int64_t n, QueueParams q,
    const HeavyRec *__restrict__ heavy, int64_t n_heavy, const uint32_t *__restrict__ vis,
    uint32_t *next, double *sigma, unsigned long long *counters) {
    __shared__ int32_t stage[kWarpsPerBlock][kStage];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
    if (r >= n_heavy) return;
    const HeavyRec rec = heavy[r];
    const size_t g = (size_t)rec.g;
    const int32_t u = q.q_v[g * q.cap + rec.qi];
    const uint32_t mask = q.q_m[g * q.cap + rec.qi];
    const int64_t b = off[u] + (int64_t)rec.slice * kHeavySlice;
    const int64_t e = min(off[u + 1], b + kHeavySlice);
    const uint32_t *gvis = vis + g * n;
    uint32_t *gnext = next + g * n;
    double *gsig = sigma + g * n * 32;
    const double *urow = gsig + (size_t)u * 32;
    int staged = 0;  // warp-uniform
    unsigned c_t = 0;
    auto flush = [&]() {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(q.q_count + g, (unsigned long long)staged);
        base = __shfl_sync(kFull, base, 0);
        for (int i = lane; i < staged; i += 32) q.q_v[g * q.cap + base + i] = stage[warp][i];
        staged = 0;
        __syncwarp();
    };
    for (int64_t base = b; base < e; base += 32) {
        const int64_t k = base + lane;
        bool fresh_vertex = false;
        int32_t w = 0;
        if (k < e) {
            w = __ldg(col + k);
            uint32_t fresh = mask & ~gvis[w];
            if (fresh) {
                const uint32_t old = atomicOr(gnext + w, fresh);
                fresh_vertex = old == 0;
                double *wrow = gsig + (size_t)w * 32;
                while (fresh) {
                    const int bit = __ffs(fresh) - 1;
                    fresh &= fresh - 1;
                    atomicAdd(wrow + bit, urow[bit]);   // exact: integer-valued fp64
                    ++c_t;
                }
            }
        }
        const unsigned newm = __ballot_sync(kFull, fresh_vertex);
        if (newm) {
            if (fresh_vertex) stage[warp][staged + __popc(newm & ((1u << lane) - 1u))] = w;
            staged += __popc(newm);
            __syncwarp();
            if (staged > kStage - 32) flush();
        }
    }
    if (staged) flush();
    const unsigned t = __reduce_add_sync(kFull, c_t);
    if (lane == 0 && t) atomicAdd(counters + 2, (unsigned long long)t);
}

// After a push: entries [q_lbeg[g], q_count[g]) are the new level.  Record
// their masks, mark them seen, clear next[], gather the level's statistics.
// lstat: [0] vertices in the level, [1] their arcs, [2] largest degree (all groups).
__global__ void push_post_kernel(const int64_t *__restrict__ off, int64_t n, QueueParams q,
                                 const int64_t *q_lbeg, uint32_t *vis, uint32_t *next,
                                 uint32_t *live_cur, unsigned long long *counters,
                                 unsigned long long *lstat, HeavyRec *heavy) {
    const size_t g = blockIdx.y;
    const int64_t beg = q_lbeg[g], end = (int64_t)q.q_count[g];
    unsigned long long nr = 0, ar = 0, nv = 0, fa = 0, md = 0;
    uint32_t any = 0;
    for (int64_t i = beg + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t w = q.q_v[g * q.cap + i];
        const uint32_t m = next[g * n + w];
        q.q_m[g * q.cap + i] = m;
        vis[g * n + w] |= m;
        next[g * n + w] = 0u;
        const unsigned long long deg = (unsigned long long)(off[w + 1] - off[w]);
        if (deg > (unsigned long long)kHeavyDeg) append_heavy(heavy, lstat + 3, i, (int)g, (int64_t)deg);
        any |= m;
        nr += __popc(m);
        ar += __popc(m) * deg;
        nv += 1;
        fa += deg;
        md = max(md, deg);
    }
    any = __reduce_or_sync(kFull, any);
    for (int o = 16; o > 0; o >>= 1) {
        nr += __shfl_xor_sync(kFull, nr, o);
        ar += __shfl_xor_sync(kFull, ar, o);
        nv += __shfl_xor_sync(kFull, nv, o);
        fa += __shfl_xor_sync(kFull, fa, o);
        md = max(md, __shfl_xor_sync(kFull, md, o));
    }
    if ((threadIdx.x & 31) == 0 && nv) {
        atomicOr(live_cur + g, any);
        atomicAdd(counters + 0, nr);
        atomicAdd(counters + 1, ar);
        atomicAdd(lstat + 0, nv);
        atomicAdd(lstat + 1, fa);
        atomicMax(lstat + 2, md);
    }
}

// End of a push level, one thread per group: publish the level's report for the
// host ([0..2] lstat, then q_count per group, then live per group), reset the
// statistics, and make the level just produced the frontier of the next push
// (device-resident ranges: consecutive push levels need no host uploads).
// report[4 + 2G ..]: running totals of (vertex, lane) pairs reached and of DAG arcs (the traversal
// counters) and the arcs the level's dense pull scanned -- the per-level inputs of the batched
// byte model.
__global__ void advance_level_kernel(unsigned long long *lstat, unsigned long long *q_count,
                                     const uint32_t *live_cur, int64_t *q_beg, int64_t *q_end,
                                     int64_t *q_lbeg, int G, unsigned long long *report,
                                     const unsigned long long *counters) {
    const int g = threadIdx.x;
    if (g < 3) report[g] = lstat[g];
    if (g == 3) report[3 + 2 * G] = lstat[3];   // heavy records of the level just produced
    if (g == 4) report[4 + 2 * G] = counters[0];
    if (g == 5) report[5 + 2 * G] = counters[2];
    if (g == 6) report[6 + 2 * G] = lstat[4];
    __syncthreads();
    if (g < 8) lstat[g] = 0;
    if (g < G) {
        const unsigned long long c = q_count[g];
        report[3 + g] = c;
        report[3 + G + g] = live_cur[g];
        q_beg[g] = q_lbeg[g];
        q_end[g] = (int64_t)c;
        q_lbeg[g] = (int64_t)c;
    }
}

// Backward helper: erase one queue level from `erase_arr` and write another into
// `write_arr` in a single launch (either range may be empty).
__global__ void swap_scatter_kernel(QueueParams q, int64_t n, const int64_t *erase_beg,
                                    const int64_t *erase_end, uint32_t *erase_arr,
                                    const int64_t *write_beg, const int64_t *write_end,
                                    uint32_t *write_arr) {
    const size_t g = blockIdx.y;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    if (erase_arr != nullptr)
        for (int64_t i = erase_beg[g] + tid; i < erase_end[g]; i += step)
            erase_arr[g * n + q.q_v[g * q.cap + i]] = 0u;
    if (write_arr != nullptr)
        for (int64_t i = write_beg[g] + tid; i < write_end[g]; i += step)
            write_arr[g * n + q.q_v[g * q.cap + i]] = q.q_m[g * q.cap + i];
}

// Write (clear = 0) or erase (clear = 1) a queue level in a dense mask array.
__global__ void scatter_queue_kernel(QueueParams q, int64_t n, uint32_t *dense, int clear) {
    const size_t g = blockIdx.y;
    const int64_t beg = q.q_beg[g], end = q.q_end[g];
    for (int64_t i = beg + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x)
        dense[g * n + q.q_v[g * q.cap + i]] = clear ? 0u : q.q_m[g * q.cap + i];
}

// Dense level -> queue (needed when a push level follows a pull level).
__global__ void compact_level_kernel(const uint32_t *__restrict__ lvl, const uint32_t *live_level,
                                     int64_t n, QueueParams q, const int64_t *__restrict__ off,
                                     HeavyRec *heavy, unsigned long long *heavy_count) {
    const size_t g = blockIdx.y;
    if (live_level[g] == 0) return;
    const int lane = threadIdx.x & 31;
    for (int64_t v0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane; v0 < n;
         v0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = v0 + lane;
        const uint32_t m = v < n ? lvl[g * n + v] : 0u;
        const unsigned has = __ballot_sync(kFull, m != 0);
        if (!has) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(q.q_count + g, (unsigned long long)__popc(has));
        base = __shfl_sync(kFull, base, 0);
        if (m) {
            const int64_t qi = (int64_t)base + __popc(has & ((1u << lane) - 1u));
            const size_t at = g * q.cap + qi;
            q.q_v[at] = (int32_t)v;
            q.q_m[at] = m;
            const int64_t deg = off[v + 1] - off[v];
            if (deg > kHeavyDeg) append_heavy(heavy, heavy_count, qi, (int)g, deg);
        }
    }
}

// Backward over a queue level: one warp per entry, same arithmetic as the
// dense kernel (scan_arcs + finalize_backward).
template <bool STORE_DELTA>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) bwd_queue_kernel(
    const int64_t *__restrict__ off, const int32_t *__restrict__ col, int64_t n, QueueParams q,
    const uint32_t *nbr, double *sigma, double *coef, double *delta, double *bcg,
    int accumulate) {
    const size_t g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t beg = q.q_beg[g], end = q.q_end[g];
    const int64_t stride = (int64_t)gridDim.x * kWarpsPerBlock;
    const uint32_t *gn = nbr ? nbr + g * n : nullptr;
    unsigned unused = 0;
    for (int64_t i = beg + (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); i < end;
         i += stride) {
        const int64_t v = q.q_v[g * q.cap + i];
        const uint32_t want = q.q_m[g * q.cap + i];
        double acc = 0.0;
        uint32_t got = 0;
        if (gn != nullptr)
            scan_arcs<false>((int)(off[v + 1] - off[v]), want, col + off[v], gn, coef + g * n * 32, lane,
                             acc, got, unused);
        finalize_backward<STORE_DELTA>(v, want, acc, lane, sigma + g * n * 32, coef + g * n * 32,
                                       STORE_DELTA ? delta + g * n * 32 : nullptr, bcg + g * n,
                                       accumulate);
    }
}

// Thin backward variant: one thread per queue entry; for each lane of the entry
// the thread sums its children's coef in arc order (same arithmetic as
// scan_arcs + finalize_backward, serial instead of warp-wide).
template <bool STORE_DELTA>
__global__ void bwd_queue_thin_kernel(const int64_t *__restrict__ off,
                                      const int32_t *__restrict__ col, int64_t n, QueueParams q,
                                      const uint32_t *nbr, double *sigma, double *coef,
                                      double *delta, double *bcg, int accumulate) {
    const size_t g = blockIdx.y;
    const int64_t beg = q.q_beg[g], end = q.q_end[g];
    const uint32_t *gn = nbr ? nbr + g * n : nullptr;
    double *gsig = sigma + g * n * 32;
    double *gcoef = coef + g * n * 32;
    for (int64_t i = beg + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q.q_v[g * q.cap + i];
        const uint32_t want = q.q_m[g * q.cap + i];
        if (want == 0) continue;
        pull_entry_thin<STORE_DELTA>(v, want, off[v], off[v + 1], col, gn, gsig, gcoef,
                                     STORE_DELTA ? delta + g * n * 32 : nullptr, bcg + g * n, accumulate);
    }
}

// Inspection of a queue level (see extract_level_kernel).
__global__ void extract_queue_kernel(QueueParams q, const double *sigma, const double *delta,
                                     int64_t n, int level, int32_t *dist_out, double *sigma_out,
                                     double *delta_out) {
    const size_t g = blockIdx.y;
    const int64_t beg = q.q_beg[g], end = q.q_end[g];
    for (int64_t i = beg + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q.q_v[g * q.cap + i];
        uint32_t m = q.q_m[g * q.cap + i];
        while (m) {
            const int lane = __ffs(m) - 1;
            m &= m - 1;
            const size_t row = (g * 32 + lane) * (size_t)n + v;
            const size_t idx = (g * n + v) * 32 + lane;
            if (dist_out) dist_out[row] = level;
            if (sigma_out) sigma_out[row] = sigma[idx];
            if (delta_out) delta_out[row] = delta[idx];
        }
    }
}

// key[i] = sum of the degrees of the neighbours of source i (size of its
// 2-hop neighbourhood, used to group like sources).  One warp per source.
__global__ void source_key_kernel(const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                  const int64_t *src, int64_t k, int64_t *key) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= k) return;
    const int64_t s = src[i];
    long long sum = 0;
    for (int64_t a = off[s] + lane; a < off[s + 1]; a += 32) {
        const int64_t w = col[a];
        sum += off[w + 1] - off[w];
    }
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
    if (lane == 0) key[i] = sum;
}

// bc_create: every neighbour id must name a vertex.
__global__ void validate_col_kernel(const int32_t *__restrict__ col, int64_t n_arcs, int64_t n, int *bad) {
    bool any = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_arcs;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t w = col[i];
        any |= w < 0 || w >= n;
    }
    if (__any_sync(kFull, any) && (threadIdx.x & 31) == 0) *bad = 1;
}

__global__ void fill_i32_kernel(int32_t *p, size_t count, int32_t value) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x)
        p[i] = value;
}

}  // namespace bcb200
