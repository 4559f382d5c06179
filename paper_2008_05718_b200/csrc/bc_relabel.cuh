// bc_relabel.cuh -- vertices renumbered by descending degree for the dense pull kernels.
//
// The level kernels are bound by L1 (bc_kernels.cuh): every scanned arc probes the 4-byte level
// mask of its far end, every hit gathers a row.  On a skewed graph most arcs end at a few
// thousand hubs, whose mask words are scattered over the whole n x 4 B array when ids are as
// given (one hot word per 128-byte line).  With hubs first the hot words are contiguous (the
// 21,689 vertices above 256 arcs of R-MAT scale 20 hold 63 % of the arc ends: 87 KB per group
// instead of 4 MB), and sorted adjacency lists start with runs of small ids that share lines.
// Measured on the bench workload: 28.5 -> 25.7 ms per 1024 sources (lists left in the old
// order: 26.5; log2-degree buckets: 26.4; hubs first only: 27.0; random ids: 29.8).
//
// The renumbered CSR is a second copy used by unpartitioned unit-weight runs only; sources are
// mapped on the way in and the BC vector on the way out (reduce_bc_kernel), everything else
// (partitions, border tables, inspection, weights, the graph-partitioned ranks) keeps the
// caller's ids.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bcb200 {

__global__ void relabel_degree_kernel(const int64_t *off, int64_t n, int32_t *deg, int32_t *ids) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        deg[v] = (int32_t)(off[v + 1] - off[v]);
        ids[v] = (int32_t)v;
    }
}

// order[new] = old  ->  new_of_old[old] = new; the sorted degrees widened for the offset scan
__global__ void relabel_invert_kernel(const int32_t *order, const int32_t *deg_sorted, int64_t n,
                                      int32_t *new_of_old, int64_t *deg64) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        new_of_old[order[v]] = (int32_t)v;
        deg64[v] = deg_sorted[v];
    }
}

// Arcs in renumbered-source order: key = renumbered far end, value = renumbered source (one warp per
// vertex).  A stable sort by key then groups the arcs by far end with the sources ascending --
// and since every arc has its reverse, the group of w is the sorted adjacency list of w, at
// off_new[w] (a 20-bit radix sort of 31 M pairs instead of a segmented sort of a million lists:
// 1.3 ms instead of 4.5 ms on R-MAT scale 20).
__global__ void relabel_arcs_kernel(const int64_t *off_old, const int32_t *col_old, const int32_t *order,
                                    const int64_t *off_new, const int32_t *new_of_old, int64_t n,
                                    int64_t n_arcs, int64_t *off_new_end, int32_t *key, int32_t *val) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = off_old[order[v]], b = off_old[order[v] + 1], o = off_new[v];
        for (int64_t j = lane; j < b - a; j += 32) {
            key[o + j] = new_of_old[__ldg(col_old + a + j)];
            val[o + j] = (int32_t)v;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *off_new_end = n_arcs;   // the scan is exclusive
}

// The grouping above relies on every arc having its reverse (bc_create's contract).  After the sort the
// group of w must span exactly [off_new[w], off_new[w + 1]): anything else is an asymmetric CSR.
__global__ void relabel_check_kernel(const int32_t *key_sorted, const int64_t *off_new, int64_t n, int *bad) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = off_new[w], b = off_new[w + 1];
        if (b > a && (key_sorted[a] != (int32_t)w || key_sorted[b - 1] != (int32_t)w)) *bad = 1;
    }
}

// renumbered ids of the listed sources
__global__ void relabel_sources_kernel(const int64_t *src, int64_t k, const int32_t *new_of_old, int64_t *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) out[i] = new_of_old[src[i]];
}

}  // namespace bcb200
