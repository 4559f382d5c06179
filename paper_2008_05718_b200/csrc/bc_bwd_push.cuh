// bc_bwd_push.cuh -- child-driven backward levels: the direction switch of the dependency sweep.
//
// The dense backward kernel (level_kernel<BWD>) is parent-driven: every vertex sitting at level L
// in some lane scans ALL its arcs for children at level L + 1 (backward.py:95-103, vertex pull).
// Past the peak of a small-world graph that is the wrong side to drive from: on R-MAT scale 20 the
// vertices at level 3 hold 99.5 % of the arcs while their children at level 4 hold 10 %, and one
// level further down 10 % against 0.04 %.  There the children walk their arcs instead:
//   1. bwd_push_zero_kernel      coef[v][lane] = 0 for the (vertex, lane) pairs of level L;
//   2. bwd_push_kernel           every (w, lane) at level L + 1 adds coef[w][lane] into
//                                coef[v][lane] of its parents v at level L (red.global.add.f64;
//                                the arcs of 32 consecutive vertices are dealt out one per thread);
//   3. bwd_push_finalize_kernel  delta = sigma * sum, coef = (1 + delta) / sigma, BC partial --
//                                finalize_backward's arithmetic with the sum read from coef.
// A (vertex, lane) pair sits at exactly one level, so the sums of step 2 never alias the values
// they read.  Sums arrive in atomic order: results agree with the parent-driven kernel to rounding
// (1e-16 relative per add), not bit for bit; option "bwd_push" 0 keeps every level parent-driven.
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

// One child arc: w (lanes `mw` at level L + 1) -> x.  Adds coef[w][b] into coef[x][b] for the
// lanes b where x sits at level L.
__device__ __forceinline__ void bwd_push_arc(int64_t w, uint32_t mw, int64_t x, const uint32_t *gc,
                                             double *gcoef) {
    uint32_t p = gc[x] & mw;
    const double *src = gcoef + (size_t)w * 32;
    double *dst = gcoef + (size_t)x * 32;
    while (p) {
        const int b = __ffs(p) - 1;
        p &= p - 1;
        atomicAdd(dst + b, src[b]);
    }
}

// grid = (blocks, groups); a warp takes chunks of 32 consecutive vertices, grid-stride.
__global__ void __launch_bounds__(kBwdPushThreads) bwd_push_zero_kernel(const uint32_t *__restrict__ cur, int64_t n,
                                                                 double *coef, const uint32_t *__restrict__ live) {
    const size_t g = blockIdx.y;
    if (live[g] == 0) return;
    const int lane = threadIdx.x & 31;
    const uint32_t *gc = cur + g * n;
    double *gcoef = coef + g * n * 32;
    const int64_t chunks = (n + 31) / 32;
    for (int64_t ch = (int64_t)blockIdx.x * kBwdPushWarps + (threadIdx.x >> 5); ch < chunks;
         ch += (int64_t)gridDim.x * kBwdPushWarps) {
        const int64_t v0 = ch * 32;
        const uint32_t m = (v0 + lane < n) ? gc[v0 + lane] : 0u;
        unsigned any = __ballot_sync(kFull, m != 0);
        while (any) {
            const int i = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t mi = __shfl_sync(kFull, m, i);
            if ((mi >> lane) & 1u) gcoef[(size_t)(v0 + i) * 32 + lane] = 0.0;
        }
    }
}

// nbr = masks of level L + 1 (the children), cur = masks of level L (the parents).
__global__ void __launch_bounds__(kBwdPushThreads) bwd_push_kernel(const int64_t *__restrict__ off,
                                                            const int32_t *__restrict__ col, int64_t n,
                                                            const uint32_t *__restrict__ nbr,
                                                            const uint32_t *__restrict__ cur, double *coef,
                                                            const uint32_t *__restrict__ live_child,
                                                            uint4 *heavy_list, unsigned *heavy_count,
                                                            int64_t heavy_cap) {
    const size_t g = blockIdx.y;
    if (live_child[g] == 0) return;
    const int lane = threadIdx.x & 31;
    const uint32_t *gn = nbr + g * n;
    const uint32_t *gc = cur + g * n;
    double *gcoef = coef + g * n * 32;
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
                const unsigned slot = atomicAdd(heavy_count + g, ns);
                for (unsigned k = 0; k < ns && (int64_t)(slot + k) < heavy_cap; ++k)
                    heavy_list[g * heavy_cap + slot + k] = make_uint4((unsigned)w, m, k, 0u);
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
            if (j < total) bwd_push_arc(v0 + ow, mo, col[ao + (j - eo)], gc, gcoef);
        }
    }
}

// The listed slices of heavy children of group blockIdx.y: one block per record, grid-stride.
__global__ void __launch_bounds__(kBwdPushThreads) bwd_push_heavy_kernel(const int64_t *__restrict__ off,
                                                                  const int32_t *__restrict__ col, int64_t n,
                                                                  const uint32_t *__restrict__ cur, double *coef,
                                                                  const uint4 *__restrict__ heavy_list,
                                                                  const unsigned *__restrict__ heavy_count,
                                                                  int64_t heavy_cap) {
    const size_t g = blockIdx.y;
    const unsigned cnt = (unsigned)min((long long)heavy_count[g], (long long)heavy_cap);
    const uint32_t *gc = cur + g * n;
    double *gcoef = coef + g * n * 32;
    for (unsigned e = blockIdx.x; e < cnt; e += gridDim.x) {
        const uint4 rec = heavy_list[g * heavy_cap + e];
        const int64_t w = rec.x;
        const long long a0 = off[w] + (long long)rec.z * kBwdPushSliceArcs;
        const long long a1 = min((long long)off[w + 1], a0 + kBwdPushSliceArcs);
        for (long long a = a0 + threadIdx.x; a < a1; a += kBwdPushThreads)
            bwd_push_arc(w, rec.y, col[a], gc, gcoef);
    }
}

// accumulate: finalize_backward's bits (0: add delta into the BC partials, 1: clear sigma).
__global__ void __launch_bounds__(kBwdPushThreads) bwd_push_finalize_kernel(const uint32_t *__restrict__ cur, int64_t n,
                                                                     double *sigma, double *coef, double *bcg,
                                                                     const uint32_t *__restrict__ live,
                                                                     int accumulate) {
    const size_t g = blockIdx.y;
    if (live[g] == 0) return;
    const int lane = threadIdx.x & 31;
    const uint32_t *gc = cur + g * n;
    double *gs = sigma + g * n * 32;
    double *gcoef = coef + g * n * 32;
    double *gb = bcg + g * n;
    const int64_t chunks = (n + 31) / 32;
    for (int64_t ch = (int64_t)blockIdx.x * kBwdPushWarps + (threadIdx.x >> 5); ch < chunks;
         ch += (int64_t)gridDim.x * kBwdPushWarps) {
        const int64_t v0 = ch * 32;
        const uint32_t m = (v0 + lane < n) ? gc[v0 + lane] : 0u;
        unsigned any = __ballot_sync(kFull, m != 0);
        while (any) {
            // four vertices per round: all loads issued before the first dependent store
            int idx[4];
            bool on[4];
            double sv[4], ac[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                idx[k] = any ? __ffs(any) - 1 : 0;
                const bool have = any != 0;
                any &= any - 1;
                const uint32_t mk = __shfl_sync(kFull, m, idx[k]);
                on[k] = have && ((mk >> lane) & 1u);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                sv[k] = 1.0;
                ac[k] = 0.0;
                if (on[k]) {
                    const size_t o = (size_t)(v0 + idx[k]) * 32 + lane;
                    sv[k] = gs[o];
                    ac[k] = gcoef[o];
                }
            }
            double contrib[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                contrib[k] = 0.0;
                if (on[k]) {
                    const size_t o = (size_t)(v0 + idx[k]) * 32 + lane;
                    const double d = sv[k] * ac[k];
                    gcoef[o] = (1.0 + d) / sv[k];
                    contrib[k] = d;
                    if (accumulate & 2) clear_after_use(gs + o, sv[k]);
                }
            }
            if (accumulate & 1) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double s = warp_sum(contrib[k]);
                    // idx[k] repeats 0 only for exhausted slots, whose sum is zero
                    if (lane == 0 && s != 0.0) gb[v0 + idx[k]] += s;
                }
            }
        }
    }
}

}  // namespace bcb200
