// bc_dist.cuh -- border exchange kernels of the graph-partitioned multi-GPU mode.
//
// One rank = one part = one GPU.  A rank holds the CSR rows of its own vertices
// and full-length state arrays; after every level only the *border* vertices'
// new state crosses the NVLink fabric (the paper's exchange points, reference
// PAPER.md:408-458; the level-synchronous schedule is the reference's
// bsp_forward / bsp_backward, bsp.py:22-142, batched over 32 * groups sources):
//   forward  level L : masks lvl[L][g][b] of my borders b, then sigma[b][lane]
//                      for the set lanes, lane-compacted
//   backward level L : coef[b][lane] for the borders that sit at level L
// Masks travel as a dense [border][group] u32 block; values follow in the order
// (border, group, lane) with offsets = exclusive scan of popc(mask), which the
// receiver recomputes from the masks it just received -- no index is sent.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bcb200 {

// masks[j * ng + g] = lvl[g][border_v[j]];  counts = popc (input of the scan)
__global__ void dist_export_masks_kernel(const uint32_t *lvl, const int32_t *border_v, int nb,
                                         int ng, int64_t n, uint32_t *masks, int32_t *counts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * ng) return;
    const int j = i / ng;
    const size_t g = i % ng;
    const uint32_t m = lvl[g * n + border_v[j]];
    masks[i] = m;
    counts[i] = __popc(m);
}

__global__ void dist_count_kernel(const uint32_t *masks, int count, int32_t *counts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) counts[i] = __popc(masks[i]);
}

// values[offsets[i] + r] = val[g][v][lane_r] for the r-th set lane of masks[i]
__global__ void dist_export_values_kernel(const double *val, const int32_t *border_v, int nb,
                                          int ng, int64_t n, const uint32_t *masks,
                                          const int32_t *offsets, double *values) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * ng) return;
    uint32_t m = masks[i];
    if (!m) return;
    const int j = i / ng;
    const size_t g = i % ng;
    const double *row = val + (g * n + border_v[j]) * 32;
    double *out = values + offsets[i];
    while (m) {
        const int lane = __ffs(m) - 1;
        m &= m - 1;
        *out++ = row[lane];
    }
}

// lvl[g][v] = mask (and vis |= mask on the forward phase) for a peer's borders
__global__ void dist_import_masks_kernel(const uint32_t *masks, const int32_t *border_v, int nb,
                                         int ng, int64_t n, uint32_t *lvl, uint32_t *vis) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * ng) return;
    const int j = i / ng;
    const size_t g = i % ng;
    const uint32_t m = masks[i];
    const size_t at = g * n + border_v[j];
    lvl[at] = m;
    if (m && vis) vis[at] |= m;
}

__global__ void dist_import_values_kernel(const double *values, const int32_t *border_v, int nb,
                                          int ng, int64_t n, const uint32_t *masks,
                                          const int32_t *offsets, double *val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * ng) return;
    uint32_t m = masks[i];
    if (!m) return;
    const int j = i / ng;
    const size_t g = i % ng;
    double *row = val + (g * n + border_v[j]) * 32;
    const double *in = values + offsets[i];
    while (m) {
        const int lane = __ffs(m) - 1;
        m &= m - 1;
        row[lane] = *in++;
    }
}

// bc[v] += per-group partials of the vertices this rank owns
__global__ void dist_finish_kernel(double *bc, double *bcg, const int32_t *part, int rank,
                                   int64_t n, int groups) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int g = 0; g < groups; ++g) {
            s += bcg[(size_t)g * n + v];
            bcg[(size_t)g * n + v] = 0.0;
        }
        if (part[v] == rank) bc[v] += s;
    }
}

}  // namespace bcb200
