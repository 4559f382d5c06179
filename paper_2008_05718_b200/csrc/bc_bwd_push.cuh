// bc_bwd_push.cuh -- child-driven backward levels: the direction switch of the dependency sweep.
//
// The dense backward kernel (level_kernel<BWD>) is parent-driven: every vertex sitting at level L
// in some lane scans ALL its arcs for children at level L + 1 (backward.py:95-103, vertex pull).
// Past the peak of a small-world graph that is the wrong side to drive from: on R-MAT scale 20 the
// vertices at level 3 hold 99.5 % of the arcs while their children at level 4 hold 10 %, and one
// level further down 10 % against 0.04 %.  There the children walk their arcs instead.  With
// S = sum of coef over the children, coef[v] = (1 + sigma S) / sigma = 1 / sigma + S, so:
//   1. bwd_child_init_kernel     every (vertex, lane) pair of level L as if it had no children:
//                                coef = 1 / sigma, sigma cleared (its last read, as in
//                                finalize_backward) -- the freed sigma slot is the accumulator;
//   2. bwd_push_kernel           every (w, lane) at level L + 1 adds coef[w][lane] into the sigma
//                                slot of its parents at level L (red.global.add.f64; the arcs of
//                                32 consecutive vertices are dealt out one per thread) and ORs
//                                the lanes it served into the parent's word of a `recv` mask array
//                                (a list of served pairs was tried first: its counters serialise,
//                                0.13 -> 1.15 ms for the push of R-MAT scale 20's level 4);
//   3. bwd_child_apply_kernel    sweeps `recv`; the served pairs only: coef += S,
//                                delta = S / (1 / sigma) into the BC partial, slot and word back to zero.
// Pairs without children (most of a tail level) cost what the parent-driven kernel moves for them
// and nothing else.  A (vertex, lane) pair sits at exactly one level, so the sums never alias the
// values they read.  Sums arrive in atomic order: results agree with the parent-driven kernel to
// rounding, not bit for bit; option "bwd_push" 0 keeps every level parent-driven.
#pragma once

#include "bc_kernels.cuh"

namespace bcb200 {

constexpr int kBwdPushThreads = 256;
constexpr int kBwdPushWarps = kBwdPushThreads / 32;
// a warp deals out the arcs of its 32 consecutive children one per thread; a child above this
// degree goes to a per-group list instead, one record per slice of its arcs, one block per record
// (bwd_push_heavy_kernel).  With the graph renumbered by degree the large vertices sit next to one
// another: dealt out by their own warp, 32 of them are one warp's serial work.
constexpr int kBwdPushHeavyDegree = 256;
constexpr int kBwdPushSliceArcs = 4096;

// One child arc: w (lanes `mw` at level L + 1) -> x.  Adds coef[w][b] into the accumulator (the
// cleared sigma slot) of x for the lanes b where x sits at level L and marks them in recv[x].
struct BwdPushLists {
    uint4 *heavy;                  // [group][heavy_cap] (vertex, lane mask, slice of its arcs)
    unsigned *heavy_count;         // [group]
    long long heavy_cap;
    uint32_t *recv;                // [group][n] lanes of each parent that were handed a sum; zero between levels
};

__device__ __forceinline__ void bwd_push_arc(int64_t w, uint32_t mw, int64_t x, const uint32_t *gc,
                                             double *gs, const double *gcoef, uint32_t *grecv) {
    uint32_t p = gc[x] & mw;
    if (p == 0) return;
    atomicOr(grecv + x, p);
    const double *src = gcoef + (size_t)w * 32;
    double *dst = gs + (size_t)x * 32;
    while (p) {
        const int b = __ffs(p) - 1;
        p &= p - 1;
        atomicAdd(dst + b, src[b]);
    }
}

// grid = (blocks, groups); a warp takes chunks of 32 consecutive vertices, grid-stride.
__global__ void __launch_bounds__(kBwdPushThreads) bwd_child_init_kernel(const uint32_t *__restrict__ cur, int64_t n,
                                                                  double *sigma, double *coef,
                                                                  const uint32_t *__restrict__ live) {
    const size_t g = blockIdx.y;
    if (live[g] == 0) return;
    const int lane = threadIdx.x & 31;
    const uint32_t *gc = cur + g * n;
    double *gs = sigma + g * n * 32;
    double *gcoef = coef + g * n * 32;
    const int64_t chunks = (n + 31) / 32;
    for (int64_t ch = (int64_t)blockIdx.x * kBwdPushWarps + (threadIdx.x >> 5); ch < chunks;
         ch += (int64_t)gridDim.x * kBwdPushWarps) {
        const int64_t v0 = ch * 32;
        const uint32_t m = (v0 + lane < n) ? gc[v0 + lane] : 0u;
        unsigned any = __ballot_sync(kFull, m != 0);
        while (any) {
            // four vertices per round: all loads issued before the first dependent store
            size_t o[4];
            bool on[4];
            double sv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = any ? __ffs(any) - 1 : 0;
                const bool have = any != 0;
                any &= any - 1;
                const uint32_t mk = __shfl_sync(kFull, m, i);
                on[k] = have && ((mk >> lane) & 1u);
                o[k] = (size_t)(v0 + i) * 32 + lane;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sv[k] = on[k] ? gs[o[k]] : 1.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (on[k]) {
                    gcoef[o[k]] = 1.0 / sv[k];
                    clear_after_use(gs + o[k], sv[k]);
                }
        }
    }
}

// nbr = masks of level L + 1 (the children), cur = masks of level L (the parents).
__global__ void __launch_bounds__(kBwdPushThreads) bwd_push_kernel(const int64_t *__restrict__ off,
                                                            const int32_t *__restrict__ col, int64_t n,
                                                            const uint32_t *__restrict__ nbr,
                                                            const uint32_t *__restrict__ cur, double *sigma,
                                                            const double *coef,
                                                            const uint32_t *__restrict__ live_child,
                                                            const BwdPushLists l) {
    const size_t g = blockIdx.y;
    if (live_child[g] == 0) return;
    const int lane = threadIdx.x & 31;
    const uint32_t *gn = nbr + g * n;
    const uint32_t *gc = cur + g * n;
    double *gs = sigma + g * n * 32;
    const double *gcoef = coef + g * n * 32;
    uint32_t *grecv = l.recv + g * n;
    const int64_t chunks = (n + 31) / 32;
    for (int64_t ch = (int64_t)blockIdx.x * kBwdPushWarps + (threadIdx.x >> 5); ch < chunks;
         ch += (int64_t)gridDim.x * kBwdPushWarps) {
        const int64_t v0 = ch * 32;
        const int64_t w = v0 + lane;
        const uint32_t m = (w < n) ? gn[w] : 0u;
        if (__ballot_sync(kFull, m != 0) == 0) continue;
        long long a0 = 0;
        int deg = 0;
        if (m != 0) {
            a0 = off[w];
            const long long d = off[w + 1] - a0;
            if (d > kBwdPushHeavyDegree) {
                const unsigned ns = (unsigned)((d + kBwdPushSliceArcs - 1) / kBwdPushSliceArcs);
                const unsigned slot = atomicAdd(l.heavy_count + g, ns);
                for (unsigned k = 0; k < ns && (long long)(slot + k) < l.heavy_cap; ++k)
                    l.heavy[g * l.heavy_cap + slot + k] = make_uint4((unsigned)w, m, k, 0u);
            } else {
                deg = (int)d;
            }
        }
        // inclusive scan of the degrees: arc j of the chunk belongs to the first lane with incl > j
        int incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(kFull, incl, 31);
        const int excl = incl - deg;
        for (int base = 0; base < total; base += 32) {
            const int j = base + lane;
            int ow = 0;   // number of lanes whose arcs all come before j
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int t = __shfl_sync(kFull, incl, ow + step - 1);
                if (t <= j) ow += step;
            }
            ow = min(ow, 31);
            const uint32_t mo = __shfl_sync(kFull, m, ow);
            const long long ao = __shfl_sync(kFull, a0, ow);
            const int eo = __shfl_sync(kFull, excl, ow);
            if (j < total) bwd_push_arc(v0 + ow, mo, col[ao + (j - eo)], gc, gs, gcoef, grecv);
        }
    }
}

// The listed slices of heavy children of group blockIdx.y: one block per record, grid-stride.
__global__ void __launch_bounds__(kBwdPushThreads) bwd_push_heavy_kernel(const int64_t *__restrict__ off,
                                                                  const int32_t *__restrict__ col, int64_t n,
                                                                  const uint32_t *__restrict__ cur, double *sigma,
                                                                  const double *coef, const BwdPushLists l) {
    const size_t g = blockIdx.y;
    const unsigned cnt = (unsigned)min((long long)l.heavy_count[g], l.heavy_cap);
    const uint32_t *gc = cur + g * n;
    double *gs = sigma + g * n * 32;
    const double *gcoef = coef + g * n * 32;
    uint32_t *grecv = l.recv + g * n;
    for (unsigned e = blockIdx.x; e < cnt; e += gridDim.x) {
        const uint4 rec = l.heavy[g * l.heavy_cap + e];
        const int64_t w = rec.x;
        const long long a0 = off[w] + (long long)rec.z * kBwdPushSliceArcs;
        const long long a1 = min((long long)off[w + 1], a0 + kBwdPushSliceArcs);
        for (long long a = a0 + threadIdx.x; a < a1; a += kBwdPushThreads)
            bwd_push_arc(w, rec.y, col[a], gc, gs, gcoef, grecv);
    }
}

// Sweeps recv[group][*]: for the served pairs S sits in the sigma slot, 1 / sigma in coef.
__global__ void __launch_bounds__(kBwdPushThreads) bwd_child_apply_kernel(int64_t n, double *sigma, double *coef,
                                                                   double *bcg, uint32_t *recv,
                                                                   const uint32_t *__restrict__ live) {
    const size_t g = blockIdx.y;
    if (live[g] == 0) return;
    const int lane = threadIdx.x & 31;
    uint32_t *gr = recv + g * n;
    double *gs = sigma + g * n * 32;
    double *gcoef = coef + g * n * 32;
    double *gb = bcg + g * n;
    const int64_t chunks = (n + 31) / 32;
    for (int64_t ch = (int64_t)blockIdx.x * kBwdPushWarps + (threadIdx.x >> 5); ch < chunks;
         ch += (int64_t)gridDim.x * kBwdPushWarps) {
        const int64_t v0 = ch * 32;
        const uint32_t m = (v0 + lane < n) ? gr[v0 + lane] : 0u;
        unsigned any = __ballot_sync(kFull, m != 0);
        if (m != 0) gr[v0 + lane] = 0u;
        while (any) {
            const int i = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t mi = __shfl_sync(kFull, m, i);
            double contrib = 0.0;
            if ((mi >> lane) & 1u) {
                const size_t o = (size_t)(v0 + i) * 32 + lane;
                const double S = gs[o];
                const double c0 = gcoef[o];
                gcoef[o] = c0 + S;
                contrib = S / c0;   // delta = sigma * S
                clear_after_use(gs + o, S);
            }
            const double sum = warp_sum(contrib);
            if (lane == 0) gb[v0 + i] += sum;
        }
    }
}

}  // namespace bcb200
