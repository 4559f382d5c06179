// engine_sweeps.cuh -- the sweeps of the unpartitioned ("direct") path and the building blocks every mode
// shares: dense level launches, batch set-up, level-by-level forward / backward sweeps, and the
// direction-optimising sweeps over frontier queues (push / pull per level, persistent runs of thin levels).
// Reference: initial_relax (relax.py:42-103), process_level vertex-pull (backward.py:95-103).
#pragma once

namespace {

// Row gathers keep their lines in L1 only where rows come back soon: graphs with hubs (R-MAT:
// +13 % without).  Without hubs and at a degree that spreads the neighbours over the whole array
// (Erdos-Renyi n = 2^22, degree 32) a row is never re-read in time and allocating it only evicts
// the level masks: the whole pass is 9 % faster with the gathers bypassing L1.
bool rows_bypass_l1(const bc_handle *h, const Csr &c, int L, bool bwd) {
    if (h->row_bypass_mask != 0 && L < 16) return (h->row_bypass_mask >> (L + (bwd ? 16 : 0))) & 1u;
    if (h->row_cache >= 0) return h->row_cache == 0;
    return c.n > 0 && c.n_arcs >= 8 * c.n && c.max_deg * c.n <= 16 * c.n_arcs;
}

// Forward level L on graph c for `ng` groups: pull from the masks `nbr` (level
// L - 1) into the dense array `cur`.
int launch_forward(bc_handle *h, const Csr &c, int L, int ng, cudaStream_t st,
                   const uint32_t *nbr = nullptr, uint32_t *cur = nullptr,
                   unsigned long long *lstat = nullptr) {
    LevelParams p = level_params(h, c);
    p.nbr = nbr ? nbr : h->lvl[L - 1];
    p.cur = cur ? cur : h->lvl[L];
    p.lstat = lstat;
    if (h->dist_rank >= 0 && lstat == nullptr) {
        // graph-partitioned runs: running totals for the byte model (bc_dist_get_stats)
        p.lstat = h->lstat;
        p.count_scan = 1;
        h->model_dense_words += 2 * c.n * ng;
    }
    p.live_prev = h->live + (size_t)(L - 1) * h->alloc_groups;
    p.live_cur = h->live + (size_t)L * h->alloc_groups;
    p.level = L;
    if (h->use_cand && c.wgt == nullptr) {
        mark_candidates_kernel<<<dim3(grid1d((size_t)c.n, 256, 1184), ng), 256, 0, st>>>(
            c.off, c.col, c.n, p.nbr, p.live_prev, h->cand);
        ++h->launches;
        p.cand = h->cand;
    }
    LevelTimer timer(h, st);
    const dim3 grid(blocks_for((int64_t)c.n_chk + c.n_rng), ng);
    if (c.wgt != nullptr)
        level_kernel<false, false, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    else if (rows_bypass_l1(h, c, L, false))
        level_kernel<false, false, false, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    else
        level_kernel<false, false><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    ++h->launches;
    ++h->level_launches;
    if (c.n_hub > 0) {
        HubParams q = hub_params(h, c);
        q.level = L;
        q.cur = p.cur;
        q.lstat = lstat;
        q.live_prev = p.live_prev;
        q.live_cur = p.live_cur;
        hub_kernel<false, false><<<dim3(blocks_for(c.n_hub), ng), kWarpsPerBlock * 32, 0, st>>>(q);
        ++h->launches;
    }
    timer.stop();
    CUDA_TRY(h, cudaGetLastError());
    prof_dump("fwd", L, st);
    return BC_OK;
}

// Backward level L (children at L + 1; `deepest` = no level below).
int launch_backward(bc_handle *h, const Csr &c, int L, bool deepest, int ng, bool store_delta,
                    bool accumulate, cudaStream_t st, uint32_t *cur = nullptr,
                    const uint32_t *nbr = nullptr) {
    LevelParams p = level_params(h, c);
    p.nbr = deepest ? nullptr : (nbr ? nbr : h->lvl[L + 1]);
    p.cur = cur ? cur : h->lvl[L];
    p.live_prev = h->live + (size_t)L * h->alloc_groups;
    p.accumulate_bc = (accumulate ? 1 : 0) | (h->lazy_clear ? 2 : 0);
    p.level = L;
    p.max_level = h->cur_depth - 1;
    if (h->dist_rank >= 0) h->model_dense_words += c.n * ng;
    LevelTimer timer(h, st);
    const dim3 grid(blocks_for((int64_t)c.n_chk + c.n_rng), ng);
    if (c.wgt != nullptr && store_delta)
        level_kernel<true, true, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    else if (c.wgt != nullptr)
        level_kernel<true, false, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    else if (store_delta)
        level_kernel<true, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    else if (rows_bypass_l1(h, c, L, true))
        level_kernel<true, false, false, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    else
        level_kernel<true, false><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    ++h->launches;
    ++h->level_launches;
    if (c.n_hub > 0) {
        HubParams q = hub_params(h, c);
        q.cur = p.cur;
        q.live_prev = p.live_prev;
        q.accumulate_bc = p.accumulate_bc;
        const dim3 hg(blocks_for(c.n_hub), ng);
        if (store_delta)
            hub_kernel<true, true><<<hg, kWarpsPerBlock * 32, 0, st>>>(q);
        else
            hub_kernel<true, false><<<hg, kWarpsPerBlock * 32, 0, st>>>(q);
        ++h->launches;
    }
    timer.stop();
    CUDA_TRY(h, cudaGetLastError());
    prof_dump("bwd", L, st);
    return BC_OK;
}

// Reset the BFS state of a batch and plant the level-0 seeds (sigma = 1).
int begin_batch(bc_handle *h, const int64_t *src_dev, int cnt, int ng, cudaStream_t st,
                bool zero_sigma = false) {
    const int64_t n = h->n;
    // push levels accumulate path counts with atomic adds: they need zeros.  The backward sweep
    // of a non-inspection batch leaves sigma all zero again (finalize_backward), so the memset runs
    // only after something else touched the array.
    // Deep graphs (previous batch above 64 levels) take the memset instead: there the extra dirty
    // sector per (vertex, source) visit costs more than clearing the array.
    h->lazy_clear = zero_sigma && h->last_depth <= 64;
    // Deep graphs keep their path counts in level order (deep_forward_compact_kernel) and never
    // touch the rows: the memset (17 GB per batch on the 2048^2 road graph) is skipped when the
    // sweep is expected to take that path; forward_adaptive clears the rows itself if it does not.
    h->sigma_stale = zero_sigma && !h->lazy_clear && h->fwd_compact_allowed && h->deep && h->deep_compact &&
                     h->sparse && h->full.wgt == nullptr && h->n_arcs < 6 * h->n && ng <= kDeepMaxGroups;
    // sigma_clean_groups: leading groups whose rows are all zero.  A lazily cleared batch only needs
    // zeros under the groups it uses, so a fresh engine clears ng groups, not the whole allocation.
    const int clean = h->sigma_clean_groups;
    const size_t group_bytes = (size_t)n * 32 * sizeof(double);
    h->sigma_clean_groups = 0;   // rows are in use while the batch runs
    h->sigma_clean_after = 0;
    if (zero_sigma && !h->sigma_stale) {
        if (h->lazy_clear) {
            if (ng > clean)
                CUDA_TRY(h, cudaMemsetAsync(h->sigma + (size_t)clean * n * 32, 0, (size_t)(ng - clean) * group_bytes, st));
            h->sigma_clean_after = std::max(clean, ng);
        } else {
            CUDA_TRY(h, cudaMemsetAsync(h->sigma, 0, (size_t)h->alloc_groups * group_bytes, st));
        }
    }
    h->batch_src_dev = src_dev;
    h->batch_cnt = cnt;
    CUDA_TRY(h, cudaMemsetAsync(h->live, 0, (size_t)h->live_cap * h->alloc_groups * sizeof(uint32_t), st));
    init_state_kernel<<<dim3(grid1d((size_t)n, 256, 1184), ng), 256, 0, st>>>(h->vis, h->lvl[0], n, cnt);
    seed_sources_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(src_dev, cnt, n, h->vis, h->lvl[0],
                                                          h->sigma, h->live);
    h->launches += 2;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

// Forward sweep from the level-0 seeds already in lvl[0]; *depth_out = number
// of levels up to the last non-empty one.  Levels are launched speculatively
// in growing chunks (a launch past the last level returns at once) so deep
// graphs do not pay a host round trip per level.
// Seeded mode (Step 6 of the partitioned forward phase): border seeds join at
// their own level after the pull of that level, and stepping continues through
// empty frontiers up to the largest seed level.
int forward_sweep(bc_handle *h, const Csr &c, int ng, cudaStream_t st, int *depth_out,
                  bool seeded = false, int lanes = 0, int max_seed_level = -1) {
    int L = 1, chunk = 4, last_alive = 0;
    std::vector<uint32_t> flags;
    const size_t G = (size_t)h->alloc_groups;
    const size_t lvl_bytes = G * (size_t)h->n * sizeof(uint32_t);
    const int wmax = c.wgt ? h->wmax : 1;
    // low average degree = deep graph: pull only at vertices next to the previous level
    struct CandScope {
        bc_handle *h;
        ~CandScope() { h->use_cand = false; }
    } cand_scope{h};
    if (c.wgt == nullptr && h->n_arcs < 6 * h->n) {
        const size_t bytes = (size_t)h->alloc_groups * (size_t)h->n;
        if (h->cand == nullptr) CUDA_TRY(h, arena_malloc((void **)&h->cand, bytes));
        CUDA_TRY(h, cudaMemsetAsync(h->cand, 0, bytes, st));
        h->use_cand = true;
    }
    for (;;) {
        TRY(ensure_levels(h, L + chunk));
        if (c.wgt) TRY(upload_level_ptrs(h, L + chunk, st));   // weighted levels probe lvl[L - wt]
        for (int j = 0; j < chunk; ++j) {
            if (seeded) CUDA_TRY(h, cudaMemsetAsync(h->lvl[L + j], 0, lvl_bytes, st));
            TRY(launch_forward(h, c, L + j, ng, st));
            if (seeded && L + j <= max_seed_level) {
                const size_t cnt = (size_t)h->B * h->border_S;
                inject_seeds_kernel<<<grid1d(cnt), 256, 0, st>>>(
                    border_geom(h), h->border_S, lanes, h->D, h->arr, L + j, h->n, h->vis,
                    h->lvl[L + j], h->sigma, h->live + (size_t)(L + j) * G,
                    h->dist_hybir ? h->dist_rank : -1);
                ++h->launches;
            }
        }
        flags.assign(chunk * G, 0);
        CUDA_TRY(h, cudaMemcpyAsync(flags.data(), h->live + (size_t)L * G,
                                    chunk * G * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        bool stop = false;
        for (int j = 0; j < chunk; ++j) {
            bool alive = false;
            for (int g = 0; g < ng; ++g) alive |= flags[(size_t)j * G + g] != 0;
            if (alive) last_alive = L + j;
            else if (L + j > max_seed_level && L + j - last_alive >= wmax) {
                // unit weights: the first empty level ends the sweep; weighted: a frontier can
                // jump over up to wmax - 1 empty distance values
                stop = true;
                break;
            }
        }
        if (stop) {
            *depth_out = last_alive + 1;
            return BC_OK;
        }
        L += chunk;
        chunk = std::min(chunk * 2, 64);
    }
}

int backward_sweep(bc_handle *h, const Csr &c, int depth, int ng, bool debug, cudaStream_t st) {
    // Level 0 holds only the sources; their delta is excluded from BC
    // (engine.py:147-148), so it is computed only for inspection.
    const int last = debug ? 0 : 1;
    h->cur_depth = depth;
    if (c.wgt) TRY(upload_level_ptrs(h, depth, st));
    for (int L = depth - 1; L >= last; --L)
        TRY(launch_backward(h, c, L, L == depth - 1, ng, debug, !debug, st));
    return BC_OK;
}


// ------------------------------------------------------------------------------------
// direction-optimising sweeps (dense pull levels + queue / push levels)
// ------------------------------------------------------------------------------------

struct LevelRep {
    int slot = -1;                 // dense mask array h->lvl[slot], or -1
    bool queued = false;           // entries [qb[g], qe[g]) of group g's queue
    std::vector<int64_t> qb, qe;
    unsigned long long nverts = 0, farcs = 0;  // vertices in the level, their arcs (all groups)
    unsigned long long maxdeg = 0;             // largest degree in the level
    long long heavy = 0;   // slice records of its heavy entries in h->heavy (-1: not built)
    // batched byte model; -1 = not recorded (levels of a persistent run)
    long long vlanes = -1;   // (vertex, lane) pairs sitting at this level
    long long pairs = -1;    // (DAG arc, lane) pairs between the previous level and this one
    bool compact = false;    // its path counts also sit in the level-ordered value array (h->qs)
};

QueueParams queue_params(bc_handle *h) {
    QueueParams q{};
    q.q_v = h->q_v;
    q.q_m = h->q_m;
    q.cap = h->q_cap;
    q.q_count = h->q_count;
    q.q_beg = h->d_qbeg;
    q.q_end = h->d_qend;
    return q;
}

int upload_ranges(bc_handle *h, const LevelRep &r, cudaStream_t st) {
    const size_t G = (size_t)h->alloc_groups;
    std::vector<int64_t> b(G, 0), e(G, 0);
    for (size_t g = 0; g < r.qb.size(); ++g) b[g] = r.qb[g], e[g] = r.qe[g];
    CUDA_TRY(h, cudaMemcpyAsync(h->d_qbeg, b.data(), G * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(h, cudaMemcpyAsync(h->d_qend, e.data(), G * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    return BC_OK;
}

inline unsigned queue_blocks(const LevelRep &r, int per_block) {
    int64_t longest = 1;
    for (size_t g = 0; g < r.qb.size(); ++g) longest = std::max(longest, r.qe[g] - r.qb[g]);
    return (unsigned)std::min<int64_t>((longest + per_block - 1) / per_block, 8 * 148);
}

int scatter_level(bc_handle *h, const LevelRep &r, uint32_t *dense, bool clear, int ng, cudaStream_t st) {
    TRY(upload_ranges(h, r, st));
    scatter_queue_kernel<<<dim3(queue_blocks(r, 256), ng), 256, 0, st>>>(queue_params(h), h->n, dense,
                                                                        clear ? 1 : 0);
    ++h->launches;
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

// Forward sweep with the per-level push / pull choice.  One host round trip
// per level (the choice needs the frontier's arc count): a single small read
// of the level report that advance_level_kernel publishes.  Queue ranges stay
// on the device between consecutive push levels.
// `off_host`: host copy of c's offsets (default: the full graph).  `force_push`: every level is a
// queue level (the partitioned sweeps of low-degree graphs; the caller has checked that no
// vertex of c is heavy).  `seeds`: Step-6 border seeds joining the queue levels at their own
// level (needs force_push).
int forward_adaptive(bc_handle *h, const Csr &c, int ng, int cnt, const int64_t *batch_src,
                     cudaStream_t st, int *depth_out, std::vector<LevelRep> &reps,
                     const std::vector<int64_t> *off_host = nullptr, bool force_push = false,
                     const SeedPlan *seeds = nullptr) {
    const size_t G = (size_t)h->alloc_groups;
    const int64_t n = h->n;
    TRY(ensure_queues(h));
    const std::vector<int64_t> &c_off_host = off_host ? *off_host : h->h_off;
    const int64_t seed_room = seeds ? (int64_t)h->B : 0;
    reps.clear();
    reps.emplace_back();
    // level 0: the sources, as a dense array (begin_batch) and as a queue
    std::vector<unsigned long long> qcount(G, 0);
    {
        LevelRep &r0 = reps[0];
        std::vector<HeavyRec> heavy0;
        r0.slot = 0;
        r0.queued = true;
        r0.qb.assign(ng, 0);
        r0.qe.assign(ng, 0);
        // all groups' level-0 entries go up in two pitched copies (32 entries per group at most)
        std::vector<int32_t> qv_all((size_t)ng * 32, 0);
        std::vector<uint32_t> qm_all((size_t)ng * 32, 0);
        for (int g = 0; g < ng; ++g) {
            std::vector<std::pair<int32_t, uint32_t>> ent;
            for (int i = g * 32; i < std::min(cnt, g * 32 + 32); ++i)
                ent.emplace_back((int32_t)batch_src[i], 1u << (i & 31));
            std::sort(ent.begin(), ent.end());
            int32_t *qv = qv_all.data() + (size_t)g * 32;
            uint32_t *qm = qm_all.data() + (size_t)g * 32;
            size_t len = 0;
            for (auto &e : ent) {
                if (len > 0 && qv[len - 1] == e.first) qm[len - 1] |= e.second;
                else qv[len] = e.first, qm[len] = e.second, ++len;
            }
            r0.qe[g] = (int64_t)len;
            qcount[g] = len;
            r0.nverts += len;
            for (size_t qi = 0; qi < len; ++qi) {
                const int32_t v = qv[qi];
                const unsigned long long d = (unsigned long long)(c_off_host[v + 1] - c_off_host[v]);
                r0.farcs += d;
                r0.maxdeg = std::max(r0.maxdeg, d);
                if (d > (unsigned long long)kHeavyDeg)
                    for (int sl = 0; sl < (int)((d + kHeavySlice - 1) / kHeavySlice); ++sl)
                        heavy0.push_back(HeavyRec{(int64_t)qi, g, sl});
            }
        }
        if ((size_t)h->q_cap * sizeof(int32_t) < ((size_t)1 << 31)) {
            CUDA_TRY(h, cudaMemcpy2DAsync(h->q_v, (size_t)h->q_cap * sizeof(int32_t), qv_all.data(),
                                          32 * sizeof(int32_t), 32 * sizeof(int32_t), (size_t)ng,
                                          cudaMemcpyHostToDevice, st));
            CUDA_TRY(h, cudaMemcpy2DAsync(h->q_m, (size_t)h->q_cap * sizeof(uint32_t), qm_all.data(),
                                          32 * sizeof(uint32_t), 32 * sizeof(uint32_t), (size_t)ng,
                                          cudaMemcpyHostToDevice, st));
        } else {   // queue rows further apart than the largest pitch a 2-D copy takes
            for (int g = 0; g < ng; ++g) {
                CUDA_TRY(h, cudaMemcpyAsync(h->q_v + (size_t)g * h->q_cap, qv_all.data() + (size_t)g * 32,
                                            32 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
                CUDA_TRY(h, cudaMemcpyAsync(h->q_m + (size_t)g * h->q_cap, qm_all.data() + (size_t)g * 32,
                                            32 * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            }
        }
        CUDA_TRY(h, cudaMemcpyAsync(h->q_count, qcount.data(), G * sizeof(unsigned long long),
                                    cudaMemcpyHostToDevice, st));
        CUDA_TRY(h, cudaMemsetAsync(h->lstat, 0, 8 * sizeof(unsigned long long), st));
        if (!heavy0.empty())
            CUDA_TRY(h, cudaMemcpyAsync(h->heavy, heavy0.data(), heavy0.size() * sizeof(HeavyRec),
                                        cudaMemcpyHostToDevice, st));
        r0.heavy = (long long)heavy0.size();
        r0.vlanes = cnt;
        r0.pairs = 0;
        CUDA_TRY(h, cudaStreamSynchronize(st));  // the staging vectors go out of scope
    }
    auto upload_lbeg = [&]() -> int {
        std::vector<int64_t> lbeg(G, 0);
        for (size_t g = 0; g < G; ++g) lbeg[g] = (int64_t)qcount[g];
        CUDA_TRY(h, cudaMemcpyAsync(h->d_qlbeg, lbeg.data(), G * sizeof(int64_t),
                                    cudaMemcpyHostToDevice, st));
        return BC_OK;
    };
    // Level-ordered path counts (deep graphs).  The sweep starts in compact mode when level 1 is a
    // thin level the persistent kernel takes; it leaves it (values written back into the rows,
    // every level so far marked row-based) the first time a level has to go through a kernel
    // that works on rows.
    bool compact_mode = false;
    auto rows_from_values = [&]() -> int {      // compact -> row layout for everything produced so far
        CUDA_TRY(h, cudaMemsetAsync(h->sigma, 0, G * (size_t)n * 32 * sizeof(double), st));
        decompact_sigma_kernel<<<dim3(1184, ng), 256, 0, st>>>(queue_params(h), h->q_off, h->qs, h->q_vcap, n,
                                                               h->sigma);
        vis_from_records_kernel<<<dim3(grid1d((size_t)n, 256, 1184), ng), 256, 0, st>>>(h->vs, h->vis, n);
        h->launches += 2;
        CUDA_TRY(h, cudaGetLastError());
        for (LevelRep &x : reps) x.compact = false;
        compact_mode = false;
        h->sigma_stale = false;
        return BC_OK;
    };
    auto rows_for_level0 = [&]() -> int {       // the sweep stays on rows: clear them now, re-plant the sources
        CUDA_TRY(h, cudaMemsetAsync(h->sigma, 0, G * (size_t)n * 32 * sizeof(double), st));
        source_sigma_kernel<<<(h->batch_cnt + 127) / 128, 128, 0, st>>>(h->batch_src_dev, h->batch_cnt, n, h->sigma);
        ++h->launches;
        CUDA_TRY(h, cudaGetLastError());
        h->sigma_stale = false;
        return BC_OK;
    };
    bool pulled = false;    // a pull level has run (the frontier is past its peak)
    int device_level = -1;  // level whose ranges sit in d_qbeg / d_qend (and d_qlbeg = q_count)
    int next_slot = 1;
    const unsigned long long graph_arcs = (unsigned long long)std::max<int64_t>(c.n_arcs, 1) * ng;
    std::vector<unsigned long long> report(8 + 2 * G);
    unsigned long long seen_vl = 0, seen_pairs = 0;   // running totals at the previous level
    for (int L = 1;; ++L) {
        TRY(ensure_live(h, L + 1));
        reps.emplace_back();
        LevelRep &prev = reps[L - 1];
        LevelRep &cur = reps[L];
        int64_t used = 0;
        for (int g = 0; g < ng; ++g) used = std::max<int64_t>(used, (int64_t)qcount[g]);
        const int64_t want_room = (int64_t)std::min<unsigned long long>((unsigned long long)n, prev.farcs) +
                                  (prev.queued ? 0 : (int64_t)prev.nverts) + 1 + seed_room;
        // a queue entry is walked by one warp: keep vertices with very long adjacencies on the
        // dense kernels, which slice them
        // entries above kHeavyDeg arcs are pushed slice by slice from the heavy records of the
        // level (a level that came out of a persistent run has none: pull from it instead)
        const unsigned long long beta = (unsigned long long)(pulled ? h->push_beta_late : h->push_beta);
        bool push = force_push ||
                    (prev.farcs * beta <= graph_arcs &&
                     (prev.maxdeg <= (unsigned long long)kHeavyDeg || prev.heavy >= 0 || !prev.queued));
        if (push && h->q_cap - used < want_room) {
            TRY(grow_queues(h, used + want_room, st, qcount));
            push = h->q_cap - used >= want_room;
            if (!push && force_push)
                return h->fail(BC_ERR_INTERNAL, "frontier queues of a partitioned sweep cannot grow further");
        }
        if (push) {
            if (!prev.queued) {  // dense level -> queue
                prev.qb.assign(qcount.begin(), qcount.begin() + ng);
                compact_level_kernel<<<dim3(grid1d((size_t)n, 256, 1184), ng), 256, 0, st>>>(
                    h->lvl[prev.slot], h->live + (size_t)(L - 1) * G, n, queue_params(h), c.off, h->heavy,
                    h->lstat + 3);
                ++h->launches;
                unsigned long long nheavy = 0;
                CUDA_TRY(h, cudaMemcpyAsync(qcount.data(), h->q_count, G * sizeof(unsigned long long),
                                            cudaMemcpyDeviceToHost, st));
                CUDA_TRY(h, cudaMemcpyAsync(&nheavy, h->lstat + 3, sizeof nheavy, cudaMemcpyDeviceToHost, st));
                CUDA_TRY(h, cudaMemsetAsync(h->lstat + 3, 0, sizeof(unsigned long long), st));
                CUDA_TRY(h, cudaStreamSynchronize(st));
                prev.heavy = (long long)nheavy;
                prev.qe.assign(qcount.begin(), qcount.begin() + ng);
                prev.queued = true;
                device_level = -1;
            }
            if (device_level != L - 1) {
                TRY(upload_ranges(h, prev, st));
                TRY(upload_lbeg());
            }
            const bool thin = prev.farcs <= kThinDegree * prev.nverts;
            const bool deep_run = thin && h->deep && ng <= kDeepMaxGroups &&
                                  prev.maxdeg <= (unsigned long long)kHeavyDeg;
            if (L == 1 && deep_run && h->sigma_stale) TRY(ensure_deep(h));
            if (L == 1 && deep_run && h->sigma_stale && ensure_deep_compact(h) && h->deep_grid_fc > 0) {
                // level 0 in level order: one path per source lane
                compact_init_kernel<<<dim3(grid1d((size_t)n, 256, 1184), ng), 256, 0, st>>>(h->vs, n, cnt);
                compact_level0_kernel<<<ng, 32, 0, st>>>(queue_params(h), h->q_off, h->qs, h->q_vcap, h->v_count,
                                                         h->vs, n, c.off, h->q_a, h->q_arc);
                h->launches += 2;
                reps[0].compact = true;
                compact_mode = true;
            } else if (L == 1 && h->sigma_stale) {
                TRY(rows_for_level0());
            }
            if (compact_mode && !deep_run) TRY(rows_from_values());
            if (deep_run && compact_mode) {
                // ---- a run of thin levels over level-ordered path counts
                TRY(ensure_deep(h));
                TRY(ensure_live(h, L + kDeepLevels + 1));
                DeepFwdCompactParams dp{};
                dp.off = c.off;
                dp.col = c.col;
                dp.n = n;
                dp.q = queue_params(h);
                dp.q_beg = h->d_qbeg;
                dp.q_end = h->d_qend;
                dp.q_lbeg = h->d_qlbeg;
                dp.vs = h->vs;
                dp.qs = h->qs;
                dp.q_off = h->q_off;
                dp.q_arc = h->q_arc;
                dp.q_a = h->q_a;
                dp.q_nb = h->q_nb;
                h->q_a_csr = c.off;
                dp.v_count = h->v_count;
                dp.vcap = h->q_vcap;
                dp.live = h->live;
                dp.counters = h->counters + h->cnt_off;
                dp.lstat = h->lstat;
                dp.log = h->deep_log;
                dp.run_info = h->deep_info;
                dp.ng = ng;
                dp.G = (int)G;
                dp.first_level = L;
                dp.max_levels = kDeepLevels;
                dp.graph_arcs = graph_arcs;
                dp.push_beta = beta;
                dp.thin_degree = kThinDegree;
                dp.max_degree = kHeavyDeg;
                if (seeds) dp.seeds = *seeds;
                dp.seed_room = (unsigned long long)seed_room;
                void *args[] = {&dp};
                CUDA_TRY(h, cudaLaunchCooperativeKernel((void *)deep_forward_compact_kernel, dim3(h->deep_grid_fc),
                                                        dim3(kDeepThreads), args, 0, st));
                ++h->launches;
#ifdef BC_DEEP_PHASE_TIMING
                {
                    unsigned long long ns[8];
                    cudaStreamSynchronize(st);
                    cudaMemcpyFromSymbol(ns, g_phase_ns, sizeof ns);
                    fprintf(stderr, "[phase] forward compact, cumulative ms: A %.1f  A2 %.1f  B+publish %.1f\n",
                            ns[0] / 1e6, ns[1] / 1e6, ns[2] / 1e6);
                }
#endif
                int info[2] = {0, 0};
                CUDA_TRY(h, cudaMemcpyAsync(info, h->deep_info, sizeof info, cudaMemcpyDeviceToHost, st));
                CUDA_TRY(h, cudaStreamSynchronize(st));
                const int done = info[0];
                if (done < 1 || done > kDeepLevels)
                    return h->fail(BC_ERR_INTERNAL, "persistent forward sweep returned no level");
                const size_t rw = 3 + 2 * G;
                std::vector<unsigned long long> log((size_t)done * rw);
                CUDA_TRY(h, cudaMemcpyAsync(log.data(), h->deep_log, log.size() * sizeof(unsigned long long),
                                            cudaMemcpyDeviceToHost, st));
                CUDA_TRY(h, cudaStreamSynchronize(st));
                reps.pop_back();  // `cur` is re-created below, level by level
                for (int j = 0; j < done; ++j) {
                    const unsigned long long *rep = log.data() + (size_t)j * rw;
                    bool alive = false;
                    for (int g = 0; g < ng; ++g) alive |= rep[3 + G + g] != 0;
                    if (!alive) {
                        *depth_out = L + j;
                        return BC_OK;
                    }
                    reps.emplace_back();
                    LevelRep &lr = reps.back();
                    lr.queued = true;
                    lr.qb.assign(qcount.begin(), qcount.begin() + ng);
                    for (size_t g = 0; g < G; ++g) qcount[g] = rep[3 + g];
                    lr.qe.assign(qcount.begin(), qcount.begin() + ng);
                    lr.nverts = rep[0];
                    lr.farcs = rep[1];
                    lr.maxdeg = rep[2];
                    lr.heavy = rep[2] > (unsigned long long)kHeavyDeg ? -1 : 0;
                    lr.compact = true;
                }
                L += done - 1;
                device_level = L;
                continue;
            }
            if (deep_run) {
                // ---- a run of thin levels inside one cooperative launch
                TRY(ensure_deep(h));
                TRY(ensure_live(h, L + kDeepLevels + 1));
                DeepFwdParams dp{};
                dp.off = c.off;
                dp.col = c.col;
                dp.n = n;
                dp.q = queue_params(h);
                dp.q_beg = h->d_qbeg;
                dp.q_end = h->d_qend;
                dp.q_lbeg = h->d_qlbeg;
                dp.vis = h->vis;
                dp.next = h->scrA;
                dp.sigma = h->sigma;
                dp.live = h->live;
                dp.counters = h->counters + h->cnt_off;
                dp.lstat = h->lstat;
                dp.log = h->deep_log;
                dp.run_info = h->deep_info;
                dp.ng = ng;
                dp.G = (int)G;
                dp.first_level = L;
                dp.max_levels = kDeepLevels;
                dp.graph_arcs = graph_arcs;
                dp.push_beta = beta;
                dp.thin_degree = kThinDegree;
                dp.max_degree = kHeavyDeg;
                if (seeds) dp.seeds = *seeds;
                dp.seed_room = (unsigned long long)seed_room;
                void *args[] = {&dp};
                CUDA_TRY(h, cudaLaunchCooperativeKernel((void *)deep_forward_kernel, dim3(h->deep_grid_f),
                                                        dim3(kDeepThreads), args, 0, st));
                ++h->launches;
                int info[2] = {0, 0};
                CUDA_TRY(h, cudaMemcpyAsync(info, h->deep_info, sizeof info, cudaMemcpyDeviceToHost, st));
                CUDA_TRY(h, cudaStreamSynchronize(st));
                const int done = info[0];
                if (done < 1 || done > kDeepLevels)
                    return h->fail(BC_ERR_INTERNAL, "persistent forward sweep returned no level");
                const size_t rw = 3 + 2 * G;
                std::vector<unsigned long long> log((size_t)done * rw);
                CUDA_TRY(h, cudaMemcpyAsync(log.data(), h->deep_log, log.size() * sizeof(unsigned long long),
                                            cudaMemcpyDeviceToHost, st));
                CUDA_TRY(h, cudaStreamSynchronize(st));
                reps.pop_back();  // `cur` is re-created below, level by level
                for (int j = 0; j < done; ++j) {
                    const unsigned long long *rep = log.data() + (size_t)j * rw;
                    bool alive = false;
                    for (int g = 0; g < ng; ++g) alive |= rep[3 + G + g] != 0;
                    if (!alive) {
                        *depth_out = L + j;
                        return BC_OK;
                    }
                    reps.emplace_back();
                    LevelRep &lr = reps.back();
                    lr.queued = true;
                    lr.qb.assign(qcount.begin(), qcount.begin() + ng);
                    for (size_t g = 0; g < G; ++g) qcount[g] = rep[3 + g];
                    lr.qe.assign(qcount.begin(), qcount.begin() + ng);
                    lr.nverts = rep[0];
                    lr.farcs = rep[1];
                    lr.maxdeg = rep[2];
                    lr.heavy = rep[2] > (unsigned long long)kHeavyDeg ? -1 : 0;   // no records built in there
                }
                L += done - 1;
                device_level = L;
                continue;
            }
            if (thin)  // low-degree level: one thread per entry
                fwd_push_thin_kernel<<<dim3(queue_blocks(prev, kWarpsPerBlock * 32), ng),
                                       kWarpsPerBlock * 32, 0, st>>>(
                    c.off, c.col, n, queue_params(h), h->vis, h->scrA, h->sigma,
                    h->counters + h->cnt_off);
            else
                fwd_push_kernel<<<dim3(queue_blocks(prev, kWarpsPerBlock), ng), kWarpsPerBlock * 32, 0, st>>>(
                    c.off, c.col, n, queue_params(h), h->vis, h->scrA, h->sigma,
                    h->counters + h->cnt_off);
            if (prev.heavy > 0) {
                fwd_push_heavy_kernel<<<blocks_for(prev.heavy), kWarpsPerBlock * 32, 0, st>>>(
                    c.off, c.col, n, queue_params(h), h->heavy, (int64_t)prev.heavy, h->vis, h->scrA,
                    h->sigma, h->counters + h->cnt_off);
                ++h->launches;
            }
            if (seeds && L < seeds->levels) {
                inject_seeds_queue_kernel<<<296, 256, 0, st>>>(*seeds, L, n, queue_params(h), h->vis, h->scrA,
                                                              h->sigma);
                ++h->launches;
            }
            push_post_kernel<<<dim3(std::min<unsigned>(grid1d((size_t)std::min<unsigned long long>(
                                                           (unsigned long long)n, prev.farcs + 1 + seed_room)), 1184), ng),
                               256, 0, st>>>(c.off, n, queue_params(h), h->d_qlbeg, h->vis, h->scrA,
                                             h->live + (size_t)L * G, h->counters + h->cnt_off, h->lstat,
                                             h->heavy);
            h->launches += 2;
            cur.queued = true;
            cur.qb.assign(qcount.begin(), qcount.begin() + ng);
            device_level = L;
        } else {
            if (L == 1 && h->sigma_stale) TRY(rows_for_level0());
            if (compact_mode) TRY(rows_from_values());
            const uint32_t *nbr;
            if (prev.slot >= 0) nbr = h->lvl[prev.slot];
            else {
                TRY(scatter_level(h, prev, h->scrB, false, ng, st));
                nbr = h->scrB;
            }
            cur.slot = next_slot++;
            TRY(ensure_pool(h, cur.slot + 1));
            TRY(launch_forward(h, c, L, ng, st, nbr, h->lvl[cur.slot], h->lstat));
            pulled = true;
            if (prev.slot < 0) TRY(scatter_level(h, prev, h->scrB, true, ng, st));
            device_level = -1;
        }
        advance_level_kernel<<<1, (unsigned)std::max<size_t>(G, 32), 0, st>>>(
            h->lstat, h->q_count, h->live + (size_t)L * G, h->d_qbeg, h->d_qend, h->d_qlbeg, (int)G,
            h->report, h->counters + h->cnt_off);
        ++h->launches;
        CUDA_TRY(h, cudaGetLastError());
        CUDA_TRY(h, cudaMemcpyAsync(report.data(), h->report, report.size() * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        bool alive = false;
        for (int g = 0; g < ng; ++g) alive |= report[3 + G + g] != 0;
        if (!alive) {
            reps.pop_back();
            *depth_out = L;
            return BC_OK;
        }
        cur.nverts = report[0];
        cur.farcs = report[1];
        cur.maxdeg = report[2];
        cur.heavy = (long long)report[3 + 2 * G];
        cur.vlanes = (long long)(report[4 + 2 * G] - seen_vl);
        cur.pairs = (long long)(report[5 + 2 * G] - seen_pairs);
        seen_vl = report[4 + 2 * G];
        seen_pairs = report[5 + 2 * G];
        if (!cur.queued) {
            // a dense pull produced this level: arcs scanned (col_idx + mask probe), sigma rows
            // gathered per (hit arc, lane), sigma written per (vertex, lane), vis read + level
            // mask written per (vertex, group)
            h->model_scan += (int64_t)report[6 + 2 * G];
            h->model_pairs += cur.pairs;
            h->model_vlanes += cur.vlanes;
            h->model_dense_words += 2 * n * ng;
        }
        for (size_t g = 0; g < G; ++g) qcount[g] = report[3 + g];
        if (cur.queued) cur.qe.assign(qcount.begin(), qcount.begin() + ng);
    }
}

// Backward sweep over the level representations forward_adaptive produced.
// The ranges of every queue level are uploaded once; a queue level's masks are
// kept in one of two scratch arrays while its parents' level runs.
int backward_adaptive(bc_handle *h, const Csr &c, int depth, std::vector<LevelRep> &reps, int ng,
                      bool debug, cudaStream_t st) {
    const int last = debug ? 0 : 1;
    const size_t G = (size_t)h->alloc_groups;
    const unsigned long long graph_arcs = (unsigned long long)std::max<int64_t>(c.n_arcs, 1) * ng;
    // per-level range table: [level][0: begin, 1: end][group]
    std::vector<int64_t> table((size_t)depth * 2 * G, 0);
    for (int L = 0; L < depth; ++L)
        if (reps[L].queued)
            for (size_t g = 0; g < reps[L].qb.size(); ++g) {
                table[((size_t)L * 2 + 0) * G + g] = reps[L].qb[g];
                table[((size_t)L * 2 + 1) * G + g] = reps[L].qe[g];
            }
    if ((int64_t)table.size() > h->range_table_cap) {
        TRY(dev_alloc(h, &h->range_table, table.size()));
        h->range_table_cap = (int64_t)table.size();
    }
    CUDA_TRY(h, cudaMemcpyAsync(h->range_table, table.data(), table.size() * sizeof(int64_t),
                                cudaMemcpyHostToDevice, st));
    auto beg_of = [&](int L) { return h->range_table + ((size_t)L * 2 + 0) * G; };
    auto end_of = [&](int L) { return h->range_table + ((size_t)L * 2 + 1) * G; };
    uint32_t *scr[2] = {h->scrA, h->scrB};
    {
        // ---- deep graphs: the whole sweep in one cooperative launch over level-ordered values
        bool all_thin = !debug && h->deep && h->deep_compact && h->qs != nullptr && !h->lazy_clear &&
                        ng <= kDeepMaxGroups && depth >= 3;
        for (int L = 1; all_thin && L < depth; ++L) {
            const LevelRep &x = reps[L];
            all_thin = x.queued && x.slot < 0 && x.compact && x.maxdeg <= kQueueMaxDegree &&
                       x.farcs * (unsigned long long)h->push_beta <= graph_arcs &&
                       x.farcs <= kThinDegree * x.nverts;
        }
        bool any_compact = false;
        for (int L = 0; L < depth; ++L) any_compact |= reps[L].compact;
        if (any_compact && !all_thin) {
            // the forward sweep ran on level-ordered values but this sweep works on rows
            CUDA_TRY(h, cudaMemsetAsync(h->sigma, 0, G * (size_t)h->n * 32 * sizeof(double), st));
            decompact_sigma_kernel<<<dim3(1184, ng), 256, 0, st>>>(queue_params(h), h->q_off, h->qs, h->q_vcap,
                                                                   h->n, h->sigma);
            ++h->launches;
            CUDA_TRY(h, cudaGetLastError());
            for (LevelRep &x : reps) x.compact = false;
            h->sigma_stale = false;
        }
        if (all_thin) {
            TRY(ensure_deep(h));
            DeepBwdCompactParams dp{};
            dp.off = c.off;
            dp.col = c.col;
            dp.n = h->n;
            dp.q = queue_params(h);
            dp.q_off = h->q_off;
            dp.range_table = h->range_table;
            dp.qs = h->qs;
            dp.qc = h->coef;             // the coef rows are not used on this path: same size
            dp.vcap = h->q_vcap;
            dp.bc_acc = h->deep_compact == 2 ? nullptr : h->bc_acc;
            dp.bcg = h->bcg;
            dp.ng = ng;
            dp.G = (int)G;
            dp.hi = depth - 1;
            dp.lo = last;
            dp.vs = h->vs;
            if (h->q_a_csr == c.off) {     // the forward sweep walked this very CSR
                dp.q_a = h->q_a;
                dp.q_arc = h->q_arc;
                dp.q_nb = h->q_nb;
            }
            void *args[] = {&dp};
            CUDA_TRY(h, cudaLaunchCooperativeKernel((void *)deep_backward_compact_kernel, dim3(h->deep_grid_c),
                                                    dim3(kDeepThreads), args, 0, st));
            bc_acc_flush_kernel<<<grid1d((size_t)h->n, 256, 1184), 256, 0, st>>>(h->bc_acc, h->bcg, h->n);
            h->launches += 2;
            CUDA_TRY(h, cudaGetLastError());
            return BC_OK;
        }
    }
    int holder = -1, held_level = -1;  // scratch array holding the masks of queue level held_level
    auto swap_scatter = [&](int erase_level, int erase_idx, int write_level, int write_idx) -> int {
        if (erase_idx < 0 && write_idx < 0) return BC_OK;
        unsigned blocks = 1;
        if (erase_idx >= 0) blocks = std::max(blocks, queue_blocks(reps[erase_level], 256));
        if (write_idx >= 0) blocks = std::max(blocks, queue_blocks(reps[write_level], 256));
        swap_scatter_kernel<<<dim3(blocks, ng), 256, 0, st>>>(
            queue_params(h), h->n, erase_idx >= 0 ? beg_of(erase_level) : nullptr,
            erase_idx >= 0 ? end_of(erase_level) : nullptr, erase_idx >= 0 ? scr[erase_idx] : nullptr,
            write_idx >= 0 ? beg_of(write_level) : nullptr, write_idx >= 0 ? end_of(write_level) : nullptr,
            write_idx >= 0 ? scr[write_idx] : nullptr);
        ++h->launches;
        CUDA_TRY(h, cudaGetLastError());
        return BC_OK;
    };
    for (int L = depth - 1; L >= last; --L) {
        LevelRep &r = reps[L];
        const bool deepest = L == depth - 1;
        const uint32_t *nbr = nullptr;
        if (!deepest) {
            LevelRep &below = reps[L + 1];
            if (below.slot >= 0) nbr = h->lvl[below.slot];
            else {
                if (holder < 0 || held_level != L + 1)
                    return h->fail(BC_ERR_INTERNAL, "backward sweep lost the masks of a queue level");
                nbr = scr[holder];
            }
        }
        int cur_holder = -1;  // scratch that already holds level L's masks
        auto queue_thin = [&](const LevelRep &x) {
            return x.slot < 0 && x.farcs * (unsigned long long)h->push_beta <= graph_arcs &&
                   x.maxdeg <= kQueueMaxDegree && x.farcs <= kThinDegree * x.nverts;
        };
        if (h->deep && ng <= kDeepMaxGroups && queue_thin(r) && L - 1 >= last && queue_thin(reps[L - 1])) {
            // ---- a run of thin queue levels inside one cooperative launch
            int lo = L;
            while (lo - 1 >= last && queue_thin(reps[lo - 1])) --lo;
            TRY(ensure_deep(h));
            DeepBwdParams dp{};
            dp.off = c.off;
            dp.col = c.col;
            dp.n = h->n;
            dp.q = queue_params(h);
            dp.range_table = h->range_table;
            dp.sigma = h->sigma;
            dp.coef = h->coef;
            dp.delta = h->delta;
            dp.bcg = h->bcg;
            dp.ng = ng;
            dp.G = (int)G;
            dp.hi = L;
            dp.lo = lo;
            dp.nbr_first = nbr;
            dp.erase_first = (!deepest && reps[L + 1].slot < 0) ? scr[holder] : nullptr;
            dp.scr0 = scr[0];
            dp.scr1 = scr[1];
            dp.first_write = holder == 0 ? 1 : 0;
            dp.accumulate = (debug ? 0 : 1) | (h->lazy_clear ? 2 : 0);
            void *args[] = {&dp};
            if (debug)
                CUDA_TRY(h, cudaLaunchCooperativeKernel((void *)deep_backward_kernel<true>, dim3(h->deep_grid_b),
                                                        dim3(kDeepThreads), args, 0, st));
            else
                CUDA_TRY(h, cudaLaunchCooperativeKernel((void *)deep_backward_kernel<false>, dim3(h->deep_grid_b),
                                                        dim3(kDeepThreads), args, 0, st));
            ++h->launches;
            holder = (dp.first_write + (L - lo)) & 1;   // scratch that now holds level `lo`
            held_level = lo;
            L = lo;
            continue;
        }
        auto model_backward = [&]() {
            // dense backward launch at level L: arcs of the (vertex, group) entries at L scanned,
            // coef gathered per (DAG arc, lane) towards L + 1, sigma read + coef written (+ sigma
            // cleared) per (vertex, lane), level mask read per (vertex, group), BC partial
            // read + written per entry
            h->model_scan += (int64_t)r.farcs;
            if (!deepest && reps[L + 1].pairs >= 0) h->model_pairs += reps[L + 1].pairs;
            if (r.vlanes >= 0) h->model_vlanes += (h->lazy_clear ? 3 : 2) * r.vlanes;
            h->model_dense_words += h->n * ng;
            h->model_entries += (int64_t)r.nverts;
        };
        // direction switch of the dependency sweep (bc_bwd_push.cuh): past the peak the children
        // at L + 1 hold far fewer arcs than their parents at L, so they walk theirs
        bool child_driven = r.slot >= 0 && !deepest && !debug && h->bwd_push > 0 && c.wgt == nullptr &&
                            reps[L + 1].farcs * (unsigned long long)h->bwd_push <= r.farcs;
        if (child_driven) {
            const LevelRep &below = reps[L + 1];
            const uint32_t *live_cur = h->live + (size_t)L * G;
            const uint32_t *live_child = h->live + (size_t)(L + 1) * G;
            uint32_t *cur = h->lvl[r.slot];
            const dim3 sweep_grid(std::min<unsigned>(grid1d((size_t)(h->n + 31) / 32 * 32, kBwdPushThreads), 148 * 16), ng);
            const dim3 push_grid(std::min<unsigned>(grid1d((size_t)(h->n + 31) / 32 * 32, kBwdPushThreads), 148 * 64), ng);
            if (h->bp_cap < 0) {   // slices of the vertices a warp does not deal out itself
                int64_t heavy = 0;
                for (int64_t v = 0; v < h->n; ++v) {
                    const int64_t d = h->h_off[v + 1] - h->h_off[v];
                    if (d > kBwdPushHeavyDegree) heavy += (d + kBwdPushSliceArcs - 1) / kBwdPushSliceArcs;
                }
                h->bp_cap = heavy;
            }
            const bool any_heavy = h->bp_cap > 0 && below.maxdeg > (unsigned long long)kBwdPushHeavyDegree;
            if (h->bp_cap > 0 && h->bp_list == nullptr)
                CUDA_TRY(h, arena_malloc((void **)&h->bp_list, G * (size_t)h->bp_cap * sizeof(uint4)));
            if (h->bp_count == nullptr) CUDA_TRY(h, arena_malloc((void **)&h->bp_count, G * sizeof(unsigned)));
            if (h->bp_recv == nullptr) {   // zero between levels: the apply pass clears what it reads
                CUDA_TRY(h, arena_malloc((void **)&h->bp_recv, G * (size_t)h->n * sizeof(uint32_t)));
                CUDA_TRY(h, cudaMemsetAsync(h->bp_recv, 0, G * (size_t)h->n * sizeof(uint32_t), st));
            }
            BwdPushLists lists{};
            lists.heavy = h->bp_list;
            lists.heavy_count = h->bp_count;
            lists.heavy_cap = h->bp_cap;
            lists.recv = h->bp_recv;
            CUDA_TRY(h, cudaMemsetAsync(h->bp_count, 0, G * sizeof(unsigned), st));
            LevelTimer timer(h, st);
            bwd_child_init_kernel<<<sweep_grid, kBwdPushThreads, 0, st>>>(cur, h->n, h->sigma, h->coef, live_cur);
            bwd_push_kernel<<<push_grid, kBwdPushThreads, 0, st>>>(c.off, c.col, h->n, nbr, cur, h->sigma, h->coef,
                                                                  live_child, lists);
            if (any_heavy) {
                bwd_push_heavy_kernel<<<dim3((unsigned)std::min<int64_t>(h->bp_cap, 148 * 8), ng), kBwdPushThreads, 0, st>>>(
                    c.off, c.col, h->n, cur, h->sigma, h->coef, lists);
                ++h->launches;
            }
            bwd_child_apply_kernel<<<sweep_grid, kBwdPushThreads, 0, st>>>(h->n, h->sigma, h->coef, h->bcg, h->bp_recv,
                                                                          live_cur);
            timer.stop();
            h->launches += 3;
            ++h->level_launches;
            ++h->bwd_push_levels;
            CUDA_TRY(h, cudaGetLastError());
            // byte model: the children's arcs scanned, coef read + added per (DAG arc, lane), the
            // parents' pairs initialised (sigma read + cleared, coef written) and the listed ones
            // updated; two sweeps over the level masks plus the probes' share
            h->model_scan += (int64_t)below.farcs;
            if (below.pairs >= 0) h->model_pairs += 2 * below.pairs;
            if (r.vlanes >= 0) h->model_vlanes += 3 * r.vlanes;
            h->model_dense_words += 3 * h->n * ng;
            h->model_entries += (int64_t)r.nverts;
        } else if (r.slot >= 0) {
            model_backward();
            TRY(launch_backward(h, c, L, deepest, ng, debug, !debug, st, h->lvl[r.slot], nbr));
        } else if (r.farcs * (unsigned long long)h->push_beta <= graph_arcs && r.maxdeg <= kQueueMaxDegree) {
            QueueParams q = queue_params(h);
            q.q_beg = beg_of(L);
            q.q_end = end_of(L);
            const bool thin = r.farcs <= kThinDegree * r.nverts;
            const dim3 grid(queue_blocks(r, thin ? 128 : kWarpsPerBlock), ng);
            if (thin && debug)
                bwd_queue_thin_kernel<true><<<grid, 128, 0, st>>>(
                    c.off, c.col, h->n, q, nbr, h->sigma, h->coef, h->delta, h->bcg, 0);
            else if (thin)
                bwd_queue_thin_kernel<false><<<grid, 128, 0, st>>>(
                    c.off, c.col, h->n, q, nbr, h->sigma, h->coef, h->delta, h->bcg, h->lazy_clear ? 3 : 1);
            else if (debug)
                bwd_queue_kernel<true><<<grid, kWarpsPerBlock * 32, 0, st>>>(
                    c.off, c.col, h->n, q, nbr, h->sigma, h->coef, h->delta, h->bcg, 0);
            else
                bwd_queue_kernel<false><<<grid, kWarpsPerBlock * 32, 0, st>>>(
                    c.off, c.col, h->n, q, nbr, h->sigma, h->coef, h->delta, h->bcg, h->lazy_clear ? 3 : 1);
            ++h->launches;
            CUDA_TRY(h, cudaGetLastError());
        } else {  // a queue level with heavy vertices: run it through the dense kernel (hub slices)
            cur_holder = holder == 0 ? 1 : 0;
            model_backward();
            TRY(swap_scatter(-1, -1, L, cur_holder));
            TRY(launch_backward(h, c, L, deepest, ng, debug, !debug, st, scr[cur_holder], nbr));
        }
        // hand over: level L's masks become the children masks of level L - 1
        const bool need_masks = L - 1 >= last && r.slot < 0;
        int write_idx = -1;
        if (need_masks && cur_holder < 0) write_idx = holder == 0 ? 1 : 0;
        TRY(swap_scatter(held_level, holder, L, write_idx));
        if (cur_holder >= 0 || write_idx >= 0) {
            holder = cur_holder >= 0 ? cur_holder : write_idx;
            held_level = L;
        } else {
            holder = -1;
            held_level = -1;
        }
    }
    if (holder >= 0) TRY(swap_scatter(held_level, holder, -1, -1));  // leave the scratch arrays zero
    return BC_OK;
}

}  // namespace
