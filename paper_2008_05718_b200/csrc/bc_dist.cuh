// bc_dist.cuh -- border exchange kernels of the graph-partitioned multi-GPU mode.
//
// One rank = one part = one GPU.  A rank holds the CSR rows of its own vertices and
// state arrays over its own vertices plus a halo (the other parts' border vertices next to
// them; the host numbers them locally, paper_2008_05718_b200/partitioned.py); after a level
// only the *border* vertices' new state crosses the NVLink fabric (the paper's exchange points, reference
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

// ---- backward exchange plan ("minimal sync points", reference backward.py:46-56,121-139) ------
// A rank has to publish coef of its border vertex b at level L for lane l only if a vertex of
// ANOTHER part at level L - 1 pulls it: some cut arc (b, u) with lvl[L-1][u] holding l.  The plan
// lists those (border, group, lanes) entries level by level once per batch; levels without an
// entry on any rank need no exchange at all, and the others move exactly the listed values.
// One thread per (own border, group) walks the levels.  fill = 0: count entries / values per
// level; fill = 1: write the entries at eoff[L] + cursor and reserve their value slots.
struct DistPlan {
    int32_t *ent_idx;    // border * ng + group (border = index among this rank's borders)
    uint32_t *ent_mask;  // lanes to publish
    int32_t *ent_voff;   // first value slot inside the level's message
    const int32_t *eoff; // [depth + 1] first entry of each level
    int32_t *cnt_e;      // [depth] entries per level (fill = 0) / cursors (fill = 1)
    int32_t *cnt_v;      // [depth] values per level / cursors
};

__global__ void dist_plan_kernel(const uint32_t *const *lvl, const uint32_t *live, int G, int depth,
                                 const int32_t *border_v, int nb, int ng, int64_t n,
                                 const int64_t *cut_off, const int32_t *cut_dst, int fill,
                                 DistPlan plan) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * ng) return;
    const int j = i / ng;
    const size_t g = i % ng;
    const int64_t b = border_v[j];
    const int64_t c0 = cut_off[j], c1 = cut_off[j + 1];
    for (int L = 2; L < depth; ++L) {      // level 1 is pulled by the sources only (level 0: not run)
        if (live[(size_t)L * G + g] == 0) continue;
        const uint32_t m = lvl[L][g * n + b];
        if (m == 0) continue;
        uint32_t parents = 0;
        for (int64_t c = c0; c < c1; ++c) parents |= lvl[L - 1][g * n + cut_dst[c]];
        const uint32_t need = m & parents;
        if (need == 0) continue;
        if (!fill) {
            atomicAdd(plan.cnt_e + L, 1);
            atomicAdd(plan.cnt_v + L, __popc(need));
        } else {
            const int at = plan.eoff[L] + atomicAdd(plan.cnt_e + L, 1);
            plan.ent_idx[at] = i;
            plan.ent_mask[at] = need;
            plan.ent_voff[at] = atomicAdd(plan.cnt_v + L, __popc(need));
        }
    }
}

// Message of one level: [cap_v fp64 values][3 x cap_e int32: idx, mask, value offset].
__global__ void dist_pack_kernel(const double *val, const int32_t *border_v, int ng, int64_t n,
                                 const int32_t *ent_idx, const uint32_t *ent_mask,
                                 const int32_t *ent_voff, int count, double *values, int32_t *head,
                                 int64_t cap_e) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const int i = ent_idx[e];
    uint32_t m = ent_mask[e];
    const int voff = ent_voff[e];
    head[e] = i;
    head[cap_e + e] = (int32_t)m;
    head[2 * cap_e + e] = voff;
    const double *row = val + ((size_t)(i % ng) * n + border_v[i / ng]) * 32;
    double *out = values + voff;
    while (m) {
        const int lane = __ffs(m) - 1;
        m &= m - 1;
        *out++ = row[lane];
    }
}

__global__ void dist_unpack_kernel(double *val, const int32_t *border_v, int ng, int64_t n,
                                   const double *values, const int32_t *head, int64_t cap_e,
                                   int count) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const int i = head[e];
    uint32_t m = (uint32_t)head[cap_e + e];
    const double *in = values + head[2 * cap_e + e];
    double *row = val + ((size_t)(i % ng) * n + border_v[i / ng]) * 32;
    while (m) {
        const int lane = __ffs(m) - 1;
        m &= m - 1;
        row[lane] = *in++;
    }
}

// All peers' messages of one level in one launch: blockIdx.y = sender; its entry count comes from
// the all-gathered plan table plan[sender][level][0] (int64 [world][depth][2], on the device).
__global__ void dist_unpack_all_kernel(double *val, const int32_t *border_v_all, const int64_t *border_off,
                                       int ng, int64_t n, const int64_t *recv, int64_t words_per_rank,
                                       int64_t cap_e, int64_t cap_v, const int64_t *plan, int depth,
                                       int level, int self) {
    const int from = blockIdx.y;
    if (from == self) return;
    const int count = (int)plan[((size_t)from * depth + level) * 2];
    const double *values = reinterpret_cast<const double *>(recv + (size_t)from * words_per_rank);
    const int32_t *head = reinterpret_cast<const int32_t *>(values + cap_v);
    const int32_t *border_v = border_v_all + border_off[from];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
        const int i = head[e];
        uint32_t m = (uint32_t)head[cap_e + e];
        const double *in = values + head[2 * cap_e + e];
        double *row = val + ((size_t)(i % ng) * n + border_v[i / ng]) * 32;
        while (m) {
            const int lane = __ffs(m) - 1;
            m &= m - 1;
            row[lane] = *in++;
        }
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
