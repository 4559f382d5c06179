// engine_dist.cuh -- entry points of the graph-partitioned multi-GPU mode (one rank = one part = one GPU):
// per-level forward / backward work, border export / import, the backward exchange plan (minimal sync
// points, backward.py:46-56,121-139) and the border-matrix forward phase across ranks.
#pragma once
namespace {

// ------------------------------------------------------------------------------------
// graph-partitioned multi-GPU mode
// ------------------------------------------------------------------------------------

int dist_check(bc_handle *h, int level) {
    if (h->dist_rank < 0) return h->fail(BC_ERR_INPUT, "bc_dist_*: call bc_dist_setup first");
    if (h->dist_ng <= 0) return h->fail(BC_ERR_INPUT, "bc_dist_*: no batch in flight (bc_dist_begin)");
    if (level < 0) return h->fail(BC_ERR_INPUT, "bc_dist_*: negative level");
    return BC_OK;
}

// offsets = exclusive scan of counts over `entries` items (CUB), entries + 1 outputs
int dist_scan(bc_handle *h, int entries, cudaStream_t st) {
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, h->dist_counts, h->dist_offsets, entries + 1, st);
    if (need > h->dist_scan_bytes) {
        arena_free(h->dist_scan_tmp);
        h->dist_scan_tmp = nullptr;
        CUDA_TRY(h, arena_malloc(&h->dist_scan_tmp, need));
        h->dist_scan_bytes = need;
    }
    CUDA_TRY(h, cudaMemsetAsync(h->dist_counts + entries, 0, sizeof(int32_t), st));
    CUDA_TRY(h, cub::DeviceScan::ExclusiveSum(h->dist_scan_tmp, need, h->dist_counts, h->dist_offsets,
                                              entries + 1, st));
    ++h->launches;
    return BC_OK;
}

}  // namespace

extern "C" {

int bc_dist_setup(bc_handle *h, int rank, int world, const int32_t *assignment,
                  const int64_t *border_off, const int32_t *border_v) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (world < 1 || rank < 0 || rank >= world || !assignment || !border_off || border_off[0] != 0)
        return h->fail(BC_ERR_INPUT, "bc_dist_setup: bad rank / world / border lists");
    CUDA_TRY(h, cudaSetDevice(h->device));
    h->dist_rank = rank;
    h->dist_world = world;
    h->dist_border_off.assign(border_off, border_off + world + 1);
    const int64_t total = border_off[world];
    int64_t widest = 0;
    for (int r = 0; r < world; ++r) widest = std::max(widest, border_off[r + 1] - border_off[r]);
    for (int64_t i = 0; i < total; ++i)
        if (border_v[i] < 0 || border_v[i] >= h->n)
            return h->fail(BC_ERR_INPUT, "bc_dist_setup: border vertex out of range");
    std::vector<int32_t> bv(border_v, border_v + total);
    if (bv.empty()) bv.push_back(0);
    TRY(upload(h, &h->dist_border_v, bv));
    h->h_part.assign(assignment, assignment + h->n);
    TRY(upload(h, &h->d_part, h->h_part));
    h->dist_entries_cap = widest * std::max(h->groups, 1);
    TRY(dev_alloc(h, &h->dist_counts, (size_t)h->dist_entries_cap + 1));
    TRY(dev_alloc(h, &h->dist_offsets, (size_t)h->dist_entries_cap + 1));
    return BC_OK;
}

int bc_dist_begin(bc_handle *h, const int64_t *sources, int64_t count, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (h->dist_rank < 0) return h->fail(BC_ERR_INPUT, "bc_dist_begin: call bc_dist_setup first");
    if (count < 1 || count > 32 * (int64_t)h->groups || sources == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_begin: need 1 <= count <= 32 * groups sources");
    for (int64_t i = 0; i < count; ++i)
        if (sources[i] < -1 || sources[i] >= h->n)   // -1: the lane's source is not on this rank
            return h->fail(BC_ERR_INPUT, "bc_dist_begin: source out of range");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    TRY(ensure_state(h, h->groups, false));
    TRY(ensure_levels(h, 2));
    if (h->bcg_dirty) {
        CUDA_TRY(h, cudaMemsetAsync(h->bcg, 0, (size_t)h->alloc_groups * (size_t)h->n * sizeof(double), st));
        h->bcg_dirty = false;
    }
    if (h->lstat == nullptr) {
        TRY(dev_alloc(h, &h->lstat, (size_t)8));
        CUDA_TRY(h, cudaMemsetAsync(h->lstat, 0, 8 * sizeof(unsigned long long), st));
        CUDA_TRY(h, cudaMemsetAsync(h->counters, 0, 8 * sizeof(unsigned long long), st));
    }
    if (h->d_src_cap < count) {
        arena_free(h->d_src);
        h->d_src = nullptr;
        CUDA_TRY(h, arena_malloc((void **)&h->d_src, count * sizeof(int64_t)));
        h->d_src_cap = count;
    }
    CUDA_TRY(h, cudaMemcpyAsync(h->d_src, sources, count * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    h->dist_cnt = (int)count;
    h->dist_ng = (int)((count + 31) / 32);
    if ((int64_t)h->dist_ng * (h->dist_entries_cap / std::max(h->groups, 1)) > h->dist_entries_cap)
        return h->fail(BC_ERR_INTERNAL, "bc_dist_begin: scan buffers too small");
    return begin_batch(h, h->d_src, (int)count, h->dist_ng, st);
}

int bc_dist_forward_level(bc_handle *h, int level, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level - 1));
    CUDA_TRY(h, cudaSetDevice(h->device));
    TRY(ensure_levels(h, level + 1));
    return launch_forward(h, h->full, level, h->dist_ng, (cudaStream_t)stream);
}

int bc_dist_backward_level(bc_handle *h, int level, int deepest, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    CUDA_TRY(h, cudaSetDevice(h->device));
    return launch_backward(h, h->full, level, deepest != 0, h->dist_ng, false, true,
                           (cudaStream_t)stream);
}

int bc_dist_export(bc_handle *h, int level, int what, void *masks_dev, void *values_dev,
                   int64_t value_capacity, int64_t *count_out, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    if (level >= (int)h->lvl.size() || masks_dev == nullptr || what < 0 || what > 2)
        return h->fail(BC_ERR_INPUT, "bc_dist_export: bad level / buffer / kind");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int r = h->dist_rank, ng = h->dist_ng;
    const int nb = (int)(h->dist_border_off[r + 1] - h->dist_border_off[r]);
    const int entries = nb * ng;
    int64_t count = 0;
    if (entries > 0) {
        const int32_t *bv = h->dist_border_v + h->dist_border_off[r];
        dist_export_masks_kernel<<<grid1d((size_t)entries), 256, 0, st>>>(
            h->lvl[level], bv, nb, ng, h->n, (uint32_t *)masks_dev, h->dist_counts);
        ++h->launches;
        if (what != 0) {
            TRY(dist_scan(h, entries, st));
            int32_t total = 0;
            CUDA_TRY(h, cudaMemcpyAsync(&total, h->dist_offsets + entries, sizeof total,
                                        cudaMemcpyDeviceToHost, st));
            CUDA_TRY(h, cudaStreamSynchronize(st));
            count = total;
            if (count > value_capacity || (count > 0 && values_dev == nullptr))
                return h->fail(BC_ERR_INPUT, "bc_dist_export: value buffer too small");
            if (count > 0) {
                dist_export_values_kernel<<<grid1d((size_t)entries), 256, 0, st>>>(
                    what == 1 ? h->sigma : h->coef, bv, nb, ng, h->n, (const uint32_t *)masks_dev,
                    h->dist_offsets, (double *)values_dev);
                ++h->launches;
            }
        }
        CUDA_TRY(h, cudaGetLastError());
    }
    if (count_out) *count_out = count;
    return BC_OK;
}

int bc_dist_import(bc_handle *h, int level, int what, int from, const void *masks_dev,
                   const void *values_dev, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    if (from < 0 || from >= h->dist_world || from == h->dist_rank || what < 1 || what > 2 ||
        level >= (int)h->lvl.size())
        return h->fail(BC_ERR_INPUT, "bc_dist_import: bad peer / kind / level");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int ng = h->dist_ng;
    const int nb = (int)(h->dist_border_off[from + 1] - h->dist_border_off[from]);
    const int entries = nb * ng;
    if (entries == 0) return BC_OK;
    if (masks_dev == nullptr) return h->fail(BC_ERR_INPUT, "bc_dist_import: null masks");
    const int32_t *bv = h->dist_border_v + h->dist_border_off[from];
    if (what == 1) {
        dist_import_masks_kernel<<<grid1d((size_t)entries), 256, 0, st>>>(
            (const uint32_t *)masks_dev, bv, nb, ng, h->n, h->lvl[level], h->vis);
        ++h->launches;
    }
    dist_count_kernel<<<grid1d((size_t)entries), 256, 0, st>>>((const uint32_t *)masks_dev, entries,
                                                              h->dist_counts);
    TRY(dist_scan(h, entries, st));
    if (values_dev != nullptr) {
        dist_import_values_kernel<<<grid1d((size_t)entries), 256, 0, st>>>(
            (const double *)values_dev, bv, nb, ng, h->n, (const uint32_t *)masks_dev,
            h->dist_offsets, what == 1 ? h->sigma : h->coef);
        ++h->launches;
    }
    h->launches += 1;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

int bc_dist_get_live(bc_handle *h, int level, uint32_t *live_out, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    if (level >= h->live_cap || live_out == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_get_live: bad level");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(h, cudaMemcpyAsync(live_out, h->live + (size_t)level * h->alloc_groups,
                                h->dist_ng * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    return BC_OK;
}

int bc_dist_set_live(bc_handle *h, int level, const uint32_t *live, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    if (level >= h->live_cap || live == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_set_live: bad level");
    CUDA_TRY(h, cudaSetDevice(h->device));
    CUDA_TRY(h, cudaMemcpyAsync(h->live + (size_t)level * h->alloc_groups, live,
                                h->dist_ng * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                (cudaStream_t)stream));
    return BC_OK;
}

int bc_dist_set_cut_arcs(bc_handle *h, const int64_t *cut_off, const int32_t *cut_dst) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (h->dist_rank < 0 || cut_off == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_set_cut_arcs: call bc_dist_setup first");
    CUDA_TRY(h, cudaSetDevice(h->device));
    const int r = h->dist_rank;
    const int64_t nb = h->dist_border_off[(size_t)r + 1] - h->dist_border_off[(size_t)r];
    if (cut_off[0] != 0) return h->fail(BC_ERR_INPUT, "bc_dist_set_cut_arcs: cut_off[0] must be 0");
    const int64_t total = cut_off[nb];
    for (int64_t c = 0; c < total; ++c)
        if (cut_dst == nullptr || cut_dst[c] < 0 || cut_dst[c] >= h->n)
            return h->fail(BC_ERR_INPUT, "bc_dist_set_cut_arcs: far end out of range");
    std::vector<int64_t> off(cut_off, cut_off + nb + 1);
    std::vector<int32_t> dst(cut_dst, cut_dst + total);
    if (dst.empty()) dst.push_back(0);
    TRY(upload(h, &h->dist_cut_off, off));
    TRY(upload(h, &h->dist_cut_dst, dst));
    return BC_OK;
}

int bc_dist_plan_backward(bc_handle *h, int depth, int64_t *counts_out, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, 0));
    if (depth < 1 || depth > (int)h->lvl.size() || counts_out == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_plan_backward: bad depth / null output");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int r = h->dist_rank, ng = h->dist_ng;
    const int nb = (int)(h->dist_border_off[(size_t)r + 1] - h->dist_border_off[(size_t)r]);
    h->plan_depth = depth;
    h->plan_eoff_h.assign((size_t)depth + 1, 0);
    h->plan_cnt_e_h.assign((size_t)depth, 0);
    h->plan_cnt_v_h.assign((size_t)depth, 0);
    for (int L = 0; L < depth; ++L) counts_out[2 * L] = counts_out[2 * L + 1] = 0;
    if (nb == 0 || h->dist_world == 1) return BC_OK;
    if (h->dist_cut_off == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_plan_backward: call bc_dist_set_cut_arcs first");
    if (h->plan_levels_cap < depth + 1) {
        const int cap = std::max(depth + 1, 2 * h->plan_levels_cap);
        TRY(dev_alloc(h, &h->plan_eoff, (size_t)cap));
        TRY(dev_alloc(h, &h->plan_cnt_e, (size_t)cap));
        TRY(dev_alloc(h, &h->plan_cnt_v, (size_t)cap));
        h->plan_levels_cap = cap;
    }
    TRY(upload_level_ptrs(h, depth, st));
    const int32_t *bv = h->dist_border_v + h->dist_border_off[(size_t)r];
    DistPlan plan{h->plan_idx, h->plan_mask, h->plan_voff, h->plan_eoff, h->plan_cnt_e, h->plan_cnt_v};
    CUDA_TRY(h, cudaMemsetAsync(h->plan_cnt_e, 0, depth * sizeof(int32_t), st));
    CUDA_TRY(h, cudaMemsetAsync(h->plan_cnt_v, 0, depth * sizeof(int32_t), st));
    const unsigned blocks = grid1d((size_t)nb * ng);
    dist_plan_kernel<<<blocks, 256, 0, st>>>(h->d_lvl_ptrs, h->live, h->alloc_groups, depth, bv, nb, ng, h->n,
                                             h->dist_cut_off, h->dist_cut_dst, 0, plan);
    CUDA_TRY(h, cudaMemcpyAsync(h->plan_cnt_e_h.data(), h->plan_cnt_e, depth * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaMemcpyAsync(h->plan_cnt_v_h.data(), h->plan_cnt_v, depth * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));   // the one host round trip of a batch's backward phase
    int64_t total = 0;
    for (int L = 0; L < depth; ++L) {
        h->plan_eoff_h[(size_t)L] = (int32_t)total;
        total += h->plan_cnt_e_h[(size_t)L];
        counts_out[2 * L] = h->plan_cnt_e_h[(size_t)L];
        counts_out[2 * L + 1] = h->plan_cnt_v_h[(size_t)L];
    }
    h->plan_eoff_h[(size_t)depth] = (int32_t)total;
    if (total > h->plan_cap) {
        const int64_t cap = std::max(total, 2 * h->plan_cap);
        TRY(dev_alloc(h, &h->plan_idx, (size_t)cap));
        TRY(dev_alloc(h, &h->plan_mask, (size_t)cap));
        TRY(dev_alloc(h, &h->plan_voff, (size_t)cap));
        h->plan_cap = cap;
    }
    if (total > 0) {
        plan = DistPlan{h->plan_idx, h->plan_mask, h->plan_voff, h->plan_eoff, h->plan_cnt_e, h->plan_cnt_v};
        CUDA_TRY(h, cudaMemcpyAsync(h->plan_eoff, h->plan_eoff_h.data(), (depth + 1) * sizeof(int32_t),
                                    cudaMemcpyHostToDevice, st));
        CUDA_TRY(h, cudaMemsetAsync(h->plan_cnt_e, 0, depth * sizeof(int32_t), st));
        CUDA_TRY(h, cudaMemsetAsync(h->plan_cnt_v, 0, depth * sizeof(int32_t), st));
        dist_plan_kernel<<<blocks, 256, 0, st>>>(h->d_lvl_ptrs, h->live, h->alloc_groups, depth, bv, nb, ng,
                                                 h->n, h->dist_cut_off, h->dist_cut_dst, 1, plan);
    }
    h->launches += 2;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

int bc_dist_pack(bc_handle *h, int level, void *send_dev, int64_t cap_entries, int64_t cap_values,
                 void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    if (level >= h->plan_depth || send_dev == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_pack: no plan for this level / null buffer");
    const int count = h->plan_cnt_e_h[(size_t)level];
    if (count > cap_entries || h->plan_cnt_v_h[(size_t)level] > cap_values)
        return h->fail(BC_ERR_INPUT, "bc_dist_pack: message buffer too small");
    if (count == 0) return BC_OK;
    CUDA_TRY(h, cudaSetDevice(h->device));
    const int r = h->dist_rank;
    const int32_t eo = h->plan_eoff_h[(size_t)level];
    double *values = (double *)send_dev;
    int32_t *head = (int32_t *)(values + cap_values);
    dist_pack_kernel<<<grid1d((size_t)count), 256, 0, (cudaStream_t)stream>>>(
        h->coef, h->dist_border_v + h->dist_border_off[(size_t)r], h->dist_ng, h->n, h->plan_idx + eo,
        h->plan_mask + eo, h->plan_voff + eo, count, values, head, cap_entries);
    ++h->launches;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

int bc_dist_unpack(bc_handle *h, int level, int from, const void *recv_dev, int64_t cap_entries,
                   int64_t cap_values, int64_t n_entries, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    if (from < 0 || from >= h->dist_world || from == h->dist_rank || recv_dev == nullptr ||
        n_entries < 0 || n_entries > cap_entries)
        return h->fail(BC_ERR_INPUT, "bc_dist_unpack: bad peer / buffer / entry count");
    if (n_entries == 0) return BC_OK;
    CUDA_TRY(h, cudaSetDevice(h->device));
    const double *values = (const double *)recv_dev;
    const int32_t *head = (const int32_t *)(values + cap_values);
    dist_unpack_kernel<<<grid1d((size_t)n_entries), 256, 0, (cudaStream_t)stream>>>(
        h->coef, h->dist_border_v + h->dist_border_off[(size_t)from], h->dist_ng, h->n, values, head,
        cap_entries, (int)n_entries);
    ++h->launches;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

int bc_dist_unpack_all(bc_handle *h, int level, const void *recv_dev, int64_t words_per_rank,
                       int64_t cap_entries, int64_t cap_values, const int64_t *plan_dev, int depth,
                       void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    TRY(dist_check(h, level));
    if (recv_dev == nullptr || plan_dev == nullptr || level >= depth || cap_entries < 0 || cap_values < 0 ||
        words_per_rank < cap_values + (3 * cap_entries + 1) / 2)
        return h->fail(BC_ERR_INPUT, "bc_dist_unpack_all: bad buffers / sizes");
    if (cap_entries == 0 || h->dist_world < 2) return BC_OK;
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (h->dist_border_off_dev == nullptr) {
        std::vector<int64_t> off(h->dist_border_off.begin(), h->dist_border_off.end());
        TRY(upload(h, &h->dist_border_off_dev, off));
    }
    const dim3 grid(std::min<unsigned>(grid1d((size_t)cap_entries), 1184), (unsigned)h->dist_world);
    dist_unpack_all_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        h->coef, h->dist_border_v, h->dist_border_off_dev, h->dist_ng, h->n, (const int64_t *)recv_dev,
        words_per_rank, cap_entries, cap_values, plan_dev, depth, level, h->dist_rank);
    ++h->launches;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

int bc_dist_get_stats(bc_handle *h, bc_stats *stats) {
    if (h == nullptr || stats == nullptr) return BC_ERR_INPUT;
    memset(stats, 0, sizeof *stats);
    stats->launches = h->launches;
    stats->launches_level = h->level_launches;
    // CUDA-event time of the dense level-kernel launches since the last call
    double ms = 0;
    int64_t timed = 0;
    for (auto &pr : h->level_events) {
        float t = 0;
        if (cudaEventSynchronize(pr.second) == cudaSuccess &&
            cudaEventElapsedTime(&t, pr.first, pr.second) == cudaSuccess) {
            ms += t;
            ++timed;
        }
        cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
    }
    h->level_events.clear();
    stats->ms_level = ms;
    stats->launches_level_timed = timed;
    // byte model of the dense launches since the last call: running device totals
    if (h->lstat != nullptr && h->counters != nullptr) {
        unsigned long long ls[8] = {0}, cn[8] = {0};
        CUDA_TRY(h, cudaSetDevice(h->device));
        CUDA_TRY(h, cudaDeviceSynchronize());
        CUDA_TRY(h, cudaMemcpy(ls, h->lstat, sizeof ls, cudaMemcpyDeviceToHost));
        CUDA_TRY(h, cudaMemcpy(cn, h->counters, sizeof cn, cudaMemcpyDeviceToHost));
        CUDA_TRY(h, cudaMemset(h->lstat, 0, sizeof ls));
        CUDA_TRY(h, cudaMemset(h->counters, 0, sizeof cn));
        const int64_t vl = (int64_t)(cn[0] + cn[4]), pairs = (int64_t)(cn[2] + cn[6]);
        stats->level_scan_arcs = (int64_t)(ls[4] + ls[1]);   // forward pulls + backward entries' arcs
        stats->level_pairs = 2 * pairs;                        // gathered forward and backward
        stats->level_vertex_lanes = 3 * vl;                    // sigma written; sigma read + coef written
        stats->level_dense_words = h->model_dense_words;
        stats->level_entries = (int64_t)ls[0];
        stats->level_model_bytes = 8 * stats->level_scan_arcs + 8 * stats->level_pairs +
                                   8 * stats->level_vertex_lanes + 4 * stats->level_dense_words +
                                   16 * stats->level_entries + 8 * h->n * stats->launches_level;
        stats->reached = vl;
        stats->dag_arcs = pairs;
        h->model_dense_words = 0;
    }
    h->level_launches = 0;
    return BC_OK;
}

int bc_dist_finish(bc_handle *h, double *bc_dev, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (h->dist_rank < 0 || bc_dev == nullptr || h->bcg == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_finish: nothing to finish");
    CUDA_TRY(h, cudaSetDevice(h->device));
    dist_finish_kernel<<<grid1d((size_t)h->n, 256, 1184), 256, 0, (cudaStream_t)stream>>>(
        bc_dev, h->bcg, h->d_part, h->dist_rank, h->n, h->alloc_groups);
    ++h->launches;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

// ---- border-matrix forward phase across ranks ------------------------------------------------
// Every rank holds all parts' border tables and runs the (cheap, batched) border refinement and
// path-count composition redundantly, so the forward phase of a batch needs ONE exchange: the
// Step-1 border seeds (distance min-reduced, path count max-reduced over the ranks; only the
// rank that owns a lane's source holds finite values).  Step 6 then runs on the rank's own part.

int bc_dist_hybir_setup(bc_handle *h, const int64_t *cin_off, const int32_t *cin_src,
                        const int32_t *cin_w) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (h->dist_rank < 0) return h->fail(BC_ERR_INPUT, "bc_dist_hybir_setup: call bc_dist_setup first");
    if (cin_off == nullptr || (cin_off[h->dist_border_off[(size_t)h->dist_world]] > 0 && cin_src == nullptr))
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_setup: null cut-arc lists");
    if (h->full.wgt != nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_setup: the multi-GPU border exchange is unit-weight");
    std::vector<int32_t> bv((size_t)h->dist_border_off[(size_t)h->dist_world]);
    if (!bv.empty())
        CUDA_TRY(h, cudaMemcpy(bv.data(), h->dist_border_v, bv.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    ExternalBorders ext{h->dist_border_off.data(), bv.data(), cin_off, cin_src, cin_w};
    h->dist_hybir = true;
    std::vector<int32_t> part = h->h_part;
    TRY(install_partition(h, h->dist_world, part.data(), &ext));
    h->tables_ready = false;
    return build_border_tables(h);   // rows of this rank's own part
}

int bc_dist_hybir_get_table(bc_handle *h, int part, int32_t *bm_dev, double *sm_dev) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (!h->dist_hybir || !h->tables_ready || part < 0 || part >= h->k)
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_get_table: no tables / bad part");
    CUDA_TRY(h, cudaSetDevice(h->device));
    const int64_t b = h->h_part_off[(size_t)part + 1] - h->h_part_off[(size_t)part];
    if (b == 0) return BC_OK;
    CUDA_TRY(h, cudaMemcpy(bm_dev, h->bm + h->h_tab_off[(size_t)part], (size_t)(b * b) * sizeof(int32_t),
                           cudaMemcpyDeviceToDevice));
    CUDA_TRY(h, cudaMemcpy(sm_dev, h->sm + h->h_tab_off[(size_t)part], (size_t)(b * b) * sizeof(double),
                           cudaMemcpyDeviceToDevice));
    return BC_OK;
}

int bc_dist_hybir_set_table(bc_handle *h, int part, const int32_t *bm_dev, const double *sm_dev) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (!h->dist_hybir || !h->tables_ready || part < 0 || part >= h->k)
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_set_table: no tables / bad part");
    CUDA_TRY(h, cudaSetDevice(h->device));
    const int64_t b = h->h_part_off[(size_t)part + 1] - h->h_part_off[(size_t)part];
    if (b == 0) return BC_OK;
    CUDA_TRY(h, cudaMemcpy(h->bm + h->h_tab_off[(size_t)part], bm_dev, (size_t)(b * b) * sizeof(int32_t),
                           cudaMemcpyDeviceToDevice));
    CUDA_TRY(h, cudaMemcpy(h->sm + h->h_tab_off[(size_t)part], sm_dev, (size_t)(b * b) * sizeof(double),
                           cudaMemcpyDeviceToDevice));
    return BC_OK;
}

int64_t bc_dist_hybir_seed_count(bc_handle *h) {
    if (h == nullptr || !h->dist_hybir) return -1;
    return (int64_t)h->B * 32 * std::max(h->groups, 1);
}

int bc_dist_hybir_seeds(bc_handle *h, const int64_t *sources, const int32_t *source_part, int64_t count,
                        int32_t *seed_dist_dev, double *seed_sigma_dev, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (!h->dist_hybir) return h->fail(BC_ERR_INPUT, "bc_dist_hybir_seeds: call bc_dist_hybir_setup first");
    if (seed_dist_dev == nullptr || seed_sigma_dev == nullptr || source_part == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_seeds: null buffers");
    for (int64_t i = 0; i < count; ++i)
        if (source_part[i] < 0 || source_part[i] >= h->dist_world)
            return h->fail(BC_ERR_INPUT, "bc_dist_hybir_seeds: source part outside [0, world)");
    cudaStream_t st = (cudaStream_t)stream;
    TRY(bc_dist_begin(h, sources, count, stream));   // state, lanes, level-0 seeds
    const int S = 32 * h->groups;
    TRY(ensure_border_state(h, S));
    std::vector<int32_t> lp((size_t)h->border_S, 0);
    for (int64_t i = 0; i < count; ++i) lp[(size_t)i] = source_part[i];
    CUDA_TRY(h, cudaMemcpyAsync(h->lane_part, lp.data(), h->border_S * sizeof(int32_t),
                                cudaMemcpyHostToDevice, st));
    int depth = 1;
    h->cnt_off = 4;   // Step 1 is a partial traversal: keep it out of the totals
    const int rc = forward_sweep(h, h->intra, h->dist_ng, st, &depth);
    h->cnt_off = 0;
    TRY(rc);
    const size_t bcnt = (size_t)h->B * h->border_S;
    fill_border_kernel<<<grid1d(bcnt, 256, 4736), 256, 0, st>>>(h->D, h->seedD, h->seedS, h->sig, h->arr, bcnt);
    TRY(upload_level_ptrs(h, depth, st));
    if (h->B > 0)
        border_gather_kernel<<<grid1d(bcnt), 256, 0, st>>>(h->d_lvl_ptrs, h->live, h->alloc_groups, depth,
                                                           h->sigma, h->n, border_geom(h), h->border_S,
                                                           h->seedD, h->seedS);
    h->launches += 2;
    CUDA_TRY(h, cudaGetLastError());
    CUDA_TRY(h, cudaMemcpyAsync(seed_dist_dev, h->seedD, bcnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(h, cudaMemcpyAsync(seed_sigma_dev, h->seedS, bcnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    return BC_OK;
}

int bc_dist_hybir_forward(bc_handle *h, const int32_t *seed_dist_dev, const double *seed_sigma_dev,
                          int *depth_out, int64_t *iterations_out, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (!h->dist_hybir || h->dist_ng <= 0)
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_forward: no batch in flight (bc_dist_hybir_seeds)");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bcnt = (size_t)h->B * h->border_S;
    CUDA_TRY(h, cudaMemcpyAsync(h->seedD, seed_dist_dev, bcnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(h, cudaMemcpyAsync(h->seedS, seed_sigma_dev, bcnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
    std::vector<int32_t> iters;
    std::vector<uint32_t> entered;
    int max_seed = -1;
    TRY(refine_and_compose(h, h->dist_cnt, h->dist_ng, st, &iters, &entered, &max_seed));
    // Step 6 on this rank's part: its own source lanes plus every border seed (seeds of other
    // parts' borders only mark those vertices at their level: they have no rows here, and the
    // backward sweep needs exactly those marks to find its cross-part children)
    TRY(begin_batch(h, h->d_src, h->dist_cnt, h->dist_ng, st));
    int depth = 1;
    TRY(forward_sweep(h, h->intra, h->dist_ng, st, &depth, true, h->dist_cnt, max_seed));
    h->dist_depth = depth;
    if (depth_out) *depth_out = depth;
    if (iterations_out) {
        int64_t total = 0;
        for (int i = 0; i < h->dist_cnt; ++i) total += iters[(size_t)i];
        *iterations_out = total;
    }
    return BC_OK;
}

// ---- the same forward phase with ONE border table per rank --------------------------------------
// bc_dist_hybir_forward runs refinement and composition redundantly on every rank, which needs every
// part's table everywhere and does not shrink with the number of GPUs.  With sharded tables a rank
// closes / composes its own part only, and the border state is merged after every iteration:
//   refinement : cut-arc relaxation for all borders (cheap, replicated), min-plus closure of the
//                rank's own part, then all-reduce MIN of the border distances [B][S] and MAX of
//                the per-lane "changed" words;
//   composition: arrival counts for all borders (cheap, replicated), composition for the own
//                part, then all-reduce MAX of the path counts (they only grow) and of "changed".
// The collectives are the caller's (torch.distributed on exchange buffers it owns); the steps:
//   0 begin refinement (seeds already reduced)   1 refinement: compute -> exchange buffers
//   2 refinement: merged buffers -> state, lane step (flag = a lane is still active)
//   3 begin composition                          4 composition: compute -> exchange buffers
//   5 composition: merged -> state, lane round (flag = some count changed)
//   6 Step 6 on the rank's part (flag = levels seen by this rank)
int bc_dist_hybir_shard_tables(bc_handle *h) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (!h->dist_hybir) return h->fail(BC_ERR_INPUT, "bc_dist_hybir_shard_tables: call bc_dist_hybir_setup first");
    CUDA_TRY(h, cudaSetDevice(h->device));
    const int r = h->dist_rank;
    const int64_t b = h->h_part_off[(size_t)r + 1] - h->h_part_off[(size_t)r];
    // keep the own part's table only (bc_dist_hybir_setup built exactly those rows)
    int32_t *bm = nullptr;
    double *sm = nullptr;
    TRY(dev_alloc(h, &bm, (size_t)(b * b)));
    TRY(dev_alloc(h, &sm, (size_t)(b * b)));
    if (b > 0) {
        CUDA_TRY(h, cudaMemcpy(bm, h->bm + h->h_tab_off[(size_t)r], (size_t)(b * b) * sizeof(int32_t),
                               cudaMemcpyDeviceToDevice));
        CUDA_TRY(h, cudaMemcpy(sm, h->sm + h->h_tab_off[(size_t)r], (size_t)(b * b) * sizeof(double),
                               cudaMemcpyDeviceToDevice));
    }
    arena_free(h->bm), arena_free(h->sm);
    h->bm = bm;
    h->sm = sm;
    h->h_tab_off.assign((size_t)h->k, 0);
    h->tab_total = b * b;
    TRY(upload(h, &h->d_tab_off, h->h_tab_off));
    h->dist_sharded = true;
    return BC_OK;
}

int bc_dist_hybir_border_step(bc_handle *h, int step, void *xchg_values_dev, void *xchg_flags_dev,
                              const int32_t *seed_dist_dev, const double *seed_sigma_dev, int *flag_out,
                              void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (!h->dist_hybir || !h->dist_sharded || h->dist_ng <= 0)
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_border_step: sharded tables and a batch in flight needed");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int S = h->border_S, lanes = h->dist_cnt, r = h->dist_rank;
    const BorderGeom geo = border_geom(h);
    const size_t cnt = (size_t)h->B * S;
    const unsigned gb = grid1d(cnt), gl = grid1d((size_t)S, 128);
    int max_b = 0;
    for (int p = 0; p < h->k; ++p) max_b = std::max(max_b, h->h_part_off[p + 1] - h->h_part_off[p]);
    const dim3 mgrid((max_b + kTJ - 1) / kTJ, (S + kTL - 1) / kTL, h->k);
    auto read_flag = [&](const uint32_t *dev) -> int {
        if (flag_out == nullptr) return BC_OK;
        uint32_t v = 0;
        CUDA_TRY(h, cudaMemcpyAsync(&v, dev, sizeof v, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        *flag_out = (int)v;
        return BC_OK;
    };
    if ((step == 1 || step == 2 || step == 4 || step == 5) && (xchg_values_dev == nullptr || xchg_flags_dev == nullptr))
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_border_step: null exchange buffers");
    switch (step) {
    case 0:
        if (seed_dist_dev == nullptr || seed_sigma_dev == nullptr)
            return h->fail(BC_ERR_INPUT, "bc_dist_hybir_border_step: null seeds");
        CUDA_TRY(h, cudaMemcpyAsync(h->seedD, seed_dist_dev, cnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemcpyAsync(h->seedS, seed_sigma_dev, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemcpyAsync(h->D, h->seedD, cnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemsetAsync(h->lane_iters, 0, S * sizeof(int32_t), st));
        CUDA_TRY(h, cudaMemsetAsync(h->lane_changed, 0, S * sizeof(uint32_t), st));
        lane_enter_kernel<<<S, 128, 0, st>>>(geo, S, lanes, h->D, h->lane_part, h->lane_active, h->lane_entered,
                                              h->n_cut);
        ++h->launches;
        break;
    case 1:
        cut_relax_kernel<<<gb, 256, 0, st>>>(geo, S, h->D, h->D2, h->lane_part, h->lane_active, kApplyAll,
                                             h->lane_changed, h->sync_flag);
        std::swap(h->D, h->D2);
        matrix_relax_kernel<<<mgrid, 256, 0, st>>>(geo, S, h->D, h->D2, h->bm, h->lane_part, h->lane_active,
                                                   kApplyAll, h->lane_changed, h->sync_flag, r);
        std::swap(h->D, h->D2);
        h->launches += 2;
        CUDA_TRY(h, cudaMemcpyAsync(xchg_values_dev, h->D, cnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemcpyAsync(xchg_flags_dev, h->lane_changed, S * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        break;
    case 2:
        CUDA_TRY(h, cudaMemcpyAsync(h->D, xchg_values_dev, cnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemcpyAsync(h->lane_changed, xchg_flags_dev, S * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemsetAsync(h->dflags, 0, 4 * sizeof(uint32_t), st));
        lane_step_kernel<<<gl, 128, 0, st>>>(S, h->lane_active, h->lane_changed, h->lane_iters, h->dflags);
        ++h->launches;
        TRY(read_flag(h->dflags));
        break;
    case 3:
        CUDA_TRY(h, cudaMemsetAsync(h->sig, 0, cnt * sizeof(double), st));
        CUDA_TRY(h, cudaMemsetAsync(h->lane_active, 1, S * sizeof(uint32_t), st));
        CUDA_TRY(h, cudaMemsetAsync(h->lane_changed, 0, S * sizeof(uint32_t), st));
        CUDA_TRY(h, cudaMemsetAsync(h->arr, 0, cnt * sizeof(double), st));
        h->dist_round = 0;
        break;
    case 4:
        arrival_kernel<<<gb, 256, 0, st>>>(geo, S, h->D, h->sig, h->arr, h->darr, h->lane_active, h->sync_flag);
        compose_sigma_kernel<<<mgrid, 256, 0, st>>>(geo, S, h->D, h->seedD, h->seedS, h->darr, h->bm, h->sm,
                                                    h->lane_part, h->sig, h->lane_active, h->lane_changed,
                                                    h->dist_round == 0, h->sync_flag, r);
        ++h->dist_round;
        h->launches += 2;
        CUDA_TRY(h, cudaMemcpyAsync(xchg_values_dev, h->sig, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemcpyAsync(xchg_flags_dev, h->lane_changed, S * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        break;
    case 5:
        CUDA_TRY(h, cudaMemcpyAsync(h->sig, xchg_values_dev, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemcpyAsync(h->lane_changed, xchg_flags_dev, S * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, cudaMemsetAsync(h->dflags + 1, 0, sizeof(uint32_t), st));
        lane_round_kernel<<<gl, 128, 0, st>>>(S, h->lane_active, h->lane_changed, h->dflags + 1);
        ++h->launches;
        TRY(read_flag(h->dflags + 1));
        break;
    case 6: {
        int m = -1;
        CUDA_TRY(h, cudaMemcpyAsync(h->d_maxlvl, &m, sizeof m, cudaMemcpyHostToDevice, st));
        if (h->B > 0) {
            max_seed_level_kernel<<<grid1d(cnt, 256, 1184), 256, 0, st>>>(h->D, h->arr, cnt, h->d_maxlvl, 1);
            ++h->launches;
        }
        CUDA_TRY(h, cudaMemcpyAsync(&m, h->d_maxlvl, sizeof m, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        TRY(begin_batch(h, h->d_src, h->dist_cnt, h->dist_ng, st));
        int depth = 1;
        TRY(forward_sweep(h, h->intra, h->dist_ng, st, &depth, true, h->dist_cnt, m));
        h->dist_depth = depth;
        if (flag_out) *flag_out = depth;
        break;
    }
    default:
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_border_step: unknown step");
    }
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

// Levels [local depth, global depth) exist on other ranks only: give them empty mask rows here.
int bc_dist_hybir_set_depth(bc_handle *h, int global_depth, void *stream) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (!h->dist_hybir || global_depth < h->dist_depth)
        return h->fail(BC_ERR_INPUT, "bc_dist_hybir_set_depth: global depth below the local one");
    cudaStream_t st = (cudaStream_t)stream;
    TRY(ensure_levels(h, global_depth + 1));
    const size_t bytes = (size_t)h->alloc_groups * (size_t)h->n * sizeof(uint32_t);
    for (int L = h->dist_depth; L < global_depth; ++L) {
        CUDA_TRY(h, cudaMemsetAsync(h->lvl[(size_t)L], 0, bytes, st));
        CUDA_TRY(h, cudaMemsetAsync(h->live + (size_t)L * h->alloc_groups, 0,
                                    h->alloc_groups * sizeof(uint32_t), st));
    }
    h->dist_depth = global_depth;
    return BC_OK;
}

}  // extern "C"
