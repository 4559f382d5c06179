// engine_border.cuh -- the border phase of the partitioned modes: Step-6 seed plan, border state, border
// refinement + path-count composition (forward.py:99-185), border tables (border_matrix.py:48-67).
#pragma once

namespace {

// ------------------------------------------------------------------------------------
// partitioned forward phase
// ------------------------------------------------------------------------------------

// Frontier-queue sweeps inside the parts: unit weights, a low-degree (deep) graph, and no vertex
// long enough to need the sliced heavy-entry push.
bool partition_queue_sweeps(const bc_handle *h) {
    return h->hybir_queues && h->sparse && h->full.wgt == nullptr && h->n_arcs < 6 * h->n &&
           h->intra_maxdeg <= (int64_t)kHeavyDeg && !h->h_ioff.empty();
}

// Blocks of a kernel that walks every queue entry of a sweep (all levels).
unsigned queue_blocks_all(const std::vector<LevelRep> &reps, int depth) {
    int64_t longest = 1;
    if (depth > 0)
        for (size_t g = 0; g < reps[depth - 1].qe.size(); ++g) longest = std::max(longest, reps[depth - 1].qe[g]);
    return (unsigned)std::min<int64_t>((longest + 255) / 256, 8 * 148);
}

// Queue sweeps of the partitioned modes: one past the last queue entry of every level,
// [level][group], for the kernels that map a queue entry back to its level.
int upload_level_ends(bc_handle *h, const std::vector<LevelRep> &reps, int depth, cudaStream_t st) {
    const size_t G = (size_t)h->alloc_groups;
    std::vector<int64_t> ends((size_t)depth * G, 0);
    for (int L = 0; L < depth; ++L) {
        if (!reps[L].queued) return h->fail(BC_ERR_INTERNAL, "partitioned queue sweep produced a dense level");
        for (size_t g = 0; g < G; ++g)
            ends[(size_t)L * G + g] = g < reps[L].qe.size() ? reps[L].qe[g] : 0;
    }
    if ((int64_t)ends.size() > h->range_table_cap) {
        TRY(dev_alloc(h, &h->range_table, ends.size()));
        h->range_table_cap = (int64_t)ends.size();
    }
    CUDA_TRY(h, cudaMemcpyAsync(h->range_table, ends.data(), ends.size() * sizeof(int64_t),
                                cudaMemcpyHostToDevice, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));   // `ends` goes out of scope
    return BC_OK;
}

// Step-6 seeds of the batch sorted by level (forward.py:232-241): every (border, lane) pair with a
// finite refined distance and a non-zero arrival count.
int build_seed_plan(bc_handle *h, int lanes, int max_seed_level, cudaStream_t st, SeedPlan *plan) {
    const int S = h->border_S;
    const size_t cnt = (size_t)h->B * S;
    *plan = SeedPlan{};
    plan->arr = h->arr;
    plan->border_v = h->d_border_v;
    plan->S = S;
    plan->levels = 0;
    if (cnt == 0 || max_seed_level < 0) return BC_OK;
    if (cnt >= ((size_t)1 << 31)) return h->fail(BC_ERR_INPUT, "too many (border, lane) pairs in one batch");
    if (h->seed_keys == nullptr) {
        TRY(dev_alloc(h, &h->seed_keys, cnt));
        TRY(dev_alloc(h, &h->seed_keys2, cnt));
        TRY(dev_alloc(h, &h->seed_vals, cnt));
        TRY(dev_alloc(h, &h->seed_vals2, cnt));
    }
    const int levels = max_seed_level + 1;
    if (h->seed_off_cap < levels + 1) {
        arena_free(h->seed_off);
        h->seed_off = nullptr;
        TRY(dev_alloc(h, &h->seed_off, (size_t)levels + 1));
        h->seed_off_cap = levels + 1;
    }
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, h->seed_keys, h->seed_keys2, h->seed_vals, h->seed_vals2,
                                    (int)cnt, 0, 32, st);
    if (need > h->seed_tmp_bytes) {
        arena_free(h->seed_tmp);
        h->seed_tmp = nullptr;
        CUDA_TRY(h, arena_malloc(&h->seed_tmp, need));
        h->seed_tmp_bytes = need;
    }
    seed_key_kernel<<<grid1d(cnt), 256, 0, st>>>(h->B, S, lanes, h->D, h->arr, h->seed_keys, h->seed_vals);
    CUDA_TRY(h, cub::DeviceRadixSort::SortPairs(h->seed_tmp, need, h->seed_keys, h->seed_keys2, h->seed_vals,
                                                h->seed_vals2, (int)cnt, 0, 32, st));
    seed_offsets_kernel<<<(levels + 1 + 127) / 128, 128, 0, st>>>(h->seed_keys2, (int64_t)cnt, levels, h->seed_off);
    h->launches += 3;
    CUDA_TRY(h, cudaGetLastError());
    plan->idx = h->seed_vals2;
    plan->off = h->seed_off;
    plan->levels = levels;
    return BC_OK;
}

int ensure_border_state(bc_handle *h, int S) {
    if (h->border_S >= S && h->D != nullptr) return BC_OK;
    free_border_state(h);
    const size_t cnt = (size_t)std::max(h->B, 1) * S;
    TRY(dev_alloc(h, &h->D, cnt));
    TRY(dev_alloc(h, &h->D2, cnt));
    TRY(dev_alloc(h, &h->seedD, cnt));
    TRY(dev_alloc(h, &h->Dfin, cnt));
    TRY(dev_alloc(h, &h->seedS, cnt));
    TRY(dev_alloc(h, &h->sig, cnt));
    TRY(dev_alloc(h, &h->arr, cnt));
    TRY(dev_alloc(h, &h->darr, cnt));
    TRY(dev_alloc(h, &h->sync_flag, cnt));
    TRY(dev_alloc(h, &h->lane_part, (size_t)S));
    TRY(dev_alloc(h, &h->seedD_alt, cnt));
    TRY(dev_alloc(h, &h->seedS_alt, cnt));
    TRY(dev_alloc(h, &h->lane_part_alt, (size_t)S));
    TRY(dev_alloc(h, &h->lane_iters, (size_t)S));
    TRY(dev_alloc(h, &h->lane_active, (size_t)S));
    TRY(dev_alloc(h, &h->lane_entered, (size_t)S));
    TRY(dev_alloc(h, &h->lane_changed, (size_t)S));
    TRY(dev_alloc(h, &h->lane_sync, (size_t)S));
    TRY(dev_alloc(h, &h->lane_bytes, (size_t)S));
    h->border_S = S;
    return BC_OK;
}

// Steps 2-5 of the reference (forward.py:99-142) for every lane of the batch,
// then the path-count composition.  `lanes` real lanes, S allocated lanes.
int refine_and_compose(bc_handle *h, int lanes, int ng, cudaStream_t st,
                       std::vector<int32_t> *iters_out, std::vector<uint32_t> *entered_out,
                       int *max_seed_level) {
    const int S = h->border_S;
    Trace tr;
    const BorderGeom geo = border_geom(h);
    const size_t cnt = (size_t)h->B * S;
    const unsigned gb = grid1d(cnt);
    const unsigned gl = grid1d((size_t)S, 128);
    int max_b = 0;
    for (int p = 0; p < h->k; ++p) max_b = std::max(max_b, h->h_part_off[p + 1] - h->h_part_off[p]);
    (void)ng;
    const dim3 mgrid((max_b + kTJ - 1) / kTJ, (S + kTL - 1) / kTL, h->k);  // every allocated lane is kept defined

    CUDA_TRY(h, cudaMemcpyAsync(h->D, h->seedD, cnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(h, cudaMemsetAsync(h->lane_iters, 0, S * sizeof(int32_t), st));
    CUDA_TRY(h, cudaMemsetAsync(h->lane_changed, 0, S * sizeof(uint32_t), st));
    lane_enter_kernel<<<S, 128, 0, st>>>(geo, S, lanes, h->D, h->lane_part, h->lane_active,
                                          h->lane_entered, h->n_cut);
    ++h->launches;
    if (h->B > 0 && h->n_cut > 0) {
        // Two parts: the reference's bound max(b0, b1) + 2 (forward.py:118,130-133).  k > 2: one
        // iteration settles one more part crossing of the shortest paths, and a path enters a
        // distinct border at every crossing, so the bound is the total border count.
        const int max_iter = (h->k == 2 ? max_b : h->B) + 2;
        // The host looks at the "any lane still active" flag only every `poll` iterations (1, 1,
        // 2, 3, 4, 4, ...): an iteration without active lanes changes nothing (inactive lanes are
        // masked in every kernel and lane_step_kernel counts iterations of active lanes only), so
        // running a few past convergence costs less than a device round trip per iteration.
        int poll = 1, since_poll = 0;
        for (int it = 0;; ++it) {
            if (h->k == 2) {
                cut_relax_kernel<<<gb, 256, 0, st>>>(geo, S, h->D, h->D, h->lane_part, h->lane_active,
                                                     kApplyOther, nullptr, h->sync_flag);
                matrix_relax_kernel<<<mgrid, 256, 0, st>>>(geo, S, h->D, h->D2, h->bm, h->lane_part,
                                                           h->lane_active, kApplyOther, nullptr, h->sync_flag);
                std::swap(h->D, h->D2);
                cut_relax_kernel<<<gb, 256, 0, st>>>(geo, S, h->D, h->D, h->lane_part, h->lane_active,
                                                     kApplySource, h->lane_changed, h->sync_flag);
                matrix_relax_kernel<<<mgrid, 256, 0, st>>>(geo, S, h->D, h->D2, h->bm, h->lane_part,
                                                           h->lane_active, kApplySource,
                                                           h->lane_changed, h->sync_flag);
                std::swap(h->D, h->D2);
                h->launches += 4;
            } else {
                cut_relax_kernel<<<gb, 256, 0, st>>>(geo, S, h->D, h->D2, h->lane_part, h->lane_active,
                                                     kApplyAll, h->lane_changed, h->sync_flag);
                std::swap(h->D, h->D2);
                matrix_relax_kernel<<<mgrid, 256, 0, st>>>(geo, S, h->D, h->D2, h->bm, h->lane_part,
                                                           h->lane_active, kApplyAll, h->lane_changed,
                                                           h->sync_flag);
                std::swap(h->D, h->D2);
                h->launches += 2;
            }
            CUDA_TRY(h, cudaMemsetAsync(h->dflags, 0, 4 * sizeof(uint32_t), st));
            lane_step_kernel<<<gl, 128, 0, st>>>(S, h->lane_active, h->lane_changed, h->lane_iters,
                                                 h->dflags);
            ++h->launches;
            if (++since_poll < poll) continue;
            since_poll = 0;
            poll = std::min(4, 1 + (it + 1) / 2);
            uint32_t any = 0;
            CUDA_TRY(h, cudaMemcpyAsync(&any, h->dflags, sizeof any, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(h, cudaStreamSynchronize(st));
            if (!any) break;
            if (it > max_iter + 4)
                return h->fail(BC_ERR_INTERNAL, "border refinement exceeded the border-count bound");
        }
        if (h->k == 2) {
            // 'step2-final' (forward.py:134-135) for every lane that ran the loop
            cut_relax_kernel<<<gb, 256, 0, st>>>(geo, S, h->D, h->D, h->lane_part, h->lane_entered,
                                                 kApplyOther, nullptr, nullptr);
            ++h->launches;
        }
    }
    tr.mark("border: refinement");
    // path counts at the borders: Jacobi rounds until nothing changes
    CUDA_TRY(h, cudaMemsetAsync(h->sig, 0, cnt * sizeof(double), st));
    if (h->B > 0) {
        // every lane runs the first round; afterwards only those whose counts changed
        CUDA_TRY(h, cudaMemsetAsync(h->lane_active, 1, S * sizeof(uint32_t), st));
        CUDA_TRY(h, cudaMemsetAsync(h->lane_changed, 0, S * sizeof(uint32_t), st));
        CUDA_TRY(h, cudaMemsetAsync(h->arr, 0, cnt * sizeof(double), st));
        int poll = 1, since_poll = 0;   // as above: a round without running lanes is a no-op
        for (int round = 0;; ++round) {
            if (round > 2 * h->B + 8)
                return h->fail(BC_ERR_INTERNAL, "border sigma composition did not settle");
            arrival_kernel<<<gb, 256, 0, st>>>(geo, S, h->D, h->sig, h->arr, h->darr, h->lane_active,
                                               h->sync_flag);   // (sync_flag is free until the reports)
            CUDA_TRY(h, cudaMemsetAsync(h->dflags + 1, 0, sizeof(uint32_t), st));
            compose_sigma_kernel<<<mgrid, 256, 0, st>>>(geo, S, h->D, h->seedD, h->seedS, h->darr,
                                                        h->bm, h->sm, h->lane_part, h->sig,
                                                        h->lane_active, h->lane_changed, round == 0,
                                                        h->sync_flag);
            lane_round_kernel<<<gl, 128, 0, st>>>(S, h->lane_active, h->lane_changed, h->dflags + 1);
            h->launches += 3;
            if (++since_poll < poll) continue;
            since_poll = 0;
            poll = std::min(4, 1 + (round + 1) / 2);
            uint32_t changed = 0;
            CUDA_TRY(h, cudaMemcpyAsync(&changed, h->dflags + 1, sizeof changed,
                                        cudaMemcpyDeviceToHost, st));
            CUDA_TRY(h, cudaStreamSynchronize(st));
            if (!changed) break;
        }
    }
    tr.mark("border: composition");
    int m = -1;
    CUDA_TRY(h, cudaMemcpyAsync(h->d_maxlvl, &m, sizeof m, cudaMemcpyHostToDevice, st));
    if (h->B > 0) {
        max_seed_level_kernel<<<grid1d(cnt, 256, 1184), 256, 0, st>>>(h->D, h->arr, cnt, h->d_maxlvl,
                                                                      h->dist_hybir ? 1 : 0);
        ++h->launches;
    }
    CUDA_TRY(h, cudaMemcpyAsync(&m, h->d_maxlvl, sizeof m, cudaMemcpyDeviceToHost, st));
    if (iters_out) {
        iters_out->assign(S, 0);
        entered_out->assign(S, 0);
        CUDA_TRY(h, cudaMemcpyAsync(iters_out->data(), h->lane_iters, S * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaMemcpyAsync(entered_out->data(), h->lane_entered, S * sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(h, cudaStreamSynchronize(st));
    CUDA_TRY(h, cudaGetLastError());
    *max_seed_level = m;
    return BC_OK;
}

// Border tables (border_matrix.py:48-67): one BFS per border inside its part
// (cut-free CSR), batched 32 * groups borders at a time.
int build_border_tables(bc_handle *h) {
    if (h->tables_ready) return BC_OK;
    cudaStream_t st = nullptr;
    double bytes = 0;
    for (int p = 0; p < h->k; ++p) {
        const double b = h->h_part_off[p + 1] - h->h_part_off[p];
        bytes += 12.0 * b * b;
    }
    if (bytes > kMaxTableBytes) {
        char buf[256];
        snprintf(buf, sizeof buf,
                 "border tables need %.1f GB (sum of b_p^2 x 12 B); use mode 'bsp-baseline' for "
                 "this partition", bytes / 1e9);
        return h->fail(BC_ERR_INPUT, buf);
    }
    h->table_set.clear();   // (a partial set of installed tables is rebuilt from scratch)
    TRY(dev_alloc(h, &h->bm, (size_t)h->tab_total));
    TRY(dev_alloc(h, &h->sm, (size_t)h->tab_total));
    if (h->B == 0) {
        h->tables_ready = true;
        return BC_OK;
    }
    const int groups = (int)std::max<int64_t>(1, std::min<int64_t>(h->groups, (h->B + 31) / 32));
    TRY(ensure_state(h, groups, false));
    TRY(ensure_levels(h, 2));
    std::vector<int64_t> src(h->h_border_v.begin(), h->h_border_v.end());
    ScopedBlock<int64_t> d_borders_blk;
    TRY(upload(h, &d_borders_blk.p, src));
    int64_t *const d_borders = d_borders_blk.p;
    const int per = 32 * groups;
    const BorderGeom geo = border_geom(h);
    // graph-partitioned multi-GPU runs build the rows of their own part only; the other parts'
    // tables arrive through bc_dist_hybir_set_table
    const int b_lo = h->dist_hybir ? h->h_part_off[(size_t)h->dist_rank] : 0;
    const int b_hi = h->dist_hybir ? h->h_part_off[(size_t)h->dist_rank + 1] : h->B;
    const bool qsweep = partition_queue_sweeps(h);
    if (qsweep) {
        // queue sweeps write only the pairs they reach
        fill_i32_kernel<<<grid1d((size_t)h->tab_total, 256, 4736), 256, 0, st>>>(h->bm, (size_t)h->tab_total, kInf);
        CUDA_TRY(h, cudaMemsetAsync(h->sm, 0, (size_t)h->tab_total * sizeof(double), st));
        ++h->launches;
    }
    struct AllowScope {   // the table searches read their path counts through the queue entries
        bc_handle *h;
        bool was;
        ~AllowScope() { h->fwd_compact_allowed = was; }
    } allow_scope{h, h->fwd_compact_allowed};
    h->fwd_compact_allowed = qsweep;
    for (int first = b_lo; first < b_hi; first += per) {
        const int cnt = std::min(per, b_hi - first);
        const int ng = (cnt + 31) / 32;
        TRY(begin_batch(h, d_borders + first, cnt, ng, st, qsweep));
        int depth = 1;
        if (qsweep) {
            std::vector<LevelRep> reps;
            TRY(forward_adaptive(h, h->intra, ng, cnt, src.data() + first, st, &depth, reps, &h->h_ioff, true));
            TRY(upload_level_ends(h, reps, depth, st));
            border_table_queue_kernel<<<dim3(queue_blocks_all(reps, depth), ng), 256, 0, st>>>(
                queue_params(h), h->range_table, depth, h->alloc_groups, h->n, h->d_border_index, h->sigma,
                geo, first, cnt, h->bm, h->sm, reps.back().compact ? h->qs : nullptr, h->q_off, h->q_vcap);
            ++h->launches;
            CUDA_TRY(h, cudaGetLastError());
            continue;
        }
        TRY(forward_sweep(h, h->intra, ng, st, &depth));
        TRY(upload_level_ptrs(h, depth, st));
        const size_t work = (size_t)h->B * ((cnt + 31) / 32 * 32);
        border_table_kernel<<<grid1d(work), 256, 0, st>>>(h->d_lvl_ptrs, h->live, h->alloc_groups,
                                                          depth, h->sigma, h->n, geo, first, cnt,
                                                          h->bm, h->sm);
        ++h->launches;
        CUDA_TRY(h, cudaGetLastError());
    }
    CUDA_TRY(h, cudaStreamSynchronize(st));
    h->tables_ready = true;
    return BC_OK;
}

}  // namespace
