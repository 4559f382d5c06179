// engine_run.cuh -- the source loop (engine.py:132-149): batches of 32 x groups sources through forward,
// border phase (hybir), Step 6, backward; Step-1 look-ahead; per-source reports; statistics.
#pragma once

namespace {

// ------------------------------------------------------------------------------------
// the source loop
// ------------------------------------------------------------------------------------

int run_sources(bc_handle *h, int mode, const int64_t *sources_in, int64_t k_all, double *bc_dev,
                cudaStream_t st, bc_stats *stats, bool debug, int32_t *dist_out, double *sigma_out,
                double *delta_out) {
    const int64_t n = h->n;
    Trace tr;
    for (int64_t i = 0; i < k_all; ++i)
        if (sources_in[i] < 0 || sources_in[i] >= n) {
            char buf[128];
            snprintf(buf, sizeof buf, "listed source %lld out of range [0, %lld)",
                     (long long)sources_in[i], (long long)n);
            return h->fail(BC_ERR_INPUT, buf);
        }
    if (mode != BC_MODE_DIRECT && h->k == 1) mode = BC_MODE_DIRECT;  // one part: no borders
    if (general_weights(h)) {
        // weights beyond the level-per-distance kernels: label-correcting distances and
        // dependency-counted sweeps (engine_sssp.cuh)
        if (mode != BC_MODE_DIRECT)
            return h->fail(BC_ERR_INPUT, "arc weights above 4096 (or option sssp = 1): BC_MODE_DIRECT only");
        return run_sources_sssp(h, sources_in, k_all, bc_dev, st, stats, debug, dist_out, sigma_out, delta_out);
    }
    if (h->full.wgt != nullptr && h->wmax > 4096)
        return h->fail(BC_ERR_INPUT, "arc weights above 4096 need the general-weight sweeps (option sssp = -1 or 1)");
    const bool hybir = mode == BC_MODE_HYBIR;
    const bool want_reports = h->reports && mode != BC_MODE_DIRECT;
    if (hybir) TRY(build_border_tables(h));
    drop_level_events(h);   // (table searches, graph-partitioned runs: not this call's launches)

    // Sources without arcs reach nothing: sigma = 1 at the source, delta = 0
    // everywhere.  In direct mode they stay in the result (and the counters)
    // but take no lane on the device.  The inspection path and the partitioned
    // modes keep them so rows and per-source reports line up.
    std::vector<int64_t> active;
    std::vector<int64_t> where;  // index in the caller's list
    active.reserve((size_t)k_all);
    for (int64_t i = 0; i < k_all; ++i)
        if (debug || mode != BC_MODE_DIRECT ||
            h->h_off[sources_in[i] + 1] > h->h_off[sources_in[i]]) {
            active.push_back(sources_in[i]);
            where.push_back(i);
        }
    if (!debug && h->reorder) {
        // Lanes of a group advance together, so a group works best when its
        // sources see the graph alike: order them by the size of their 2-hop
        // neighbourhood (sum of neighbour degrees).  BC is a sum over sources, so
        // the order only moves fp64 rounding; the inspection path keeps the
        // caller's order because its output rows follow it.
        std::vector<int64_t> key(active.size());
        if (!active.empty()) {
            ScopedBlock<int64_t> d_tmp_blk;
            CUDA_TRY(h, arena_malloc((void **)&d_tmp_blk.p, 2 * active.size() * sizeof(int64_t)));
            int64_t *const d_tmp = d_tmp_blk.p;
            CUDA_TRY(h, cudaMemcpyAsync(d_tmp, active.data(), active.size() * sizeof(int64_t),
                                        cudaMemcpyHostToDevice, st));
            source_key_kernel<<<grid1d(active.size() * 32, 256), 256, 0, st>>>(
                h->full.off, h->full.col, d_tmp, (int64_t)active.size(), d_tmp + active.size());
            ++h->launches;
            CUDA_TRY(h, cudaMemcpyAsync(key.data(), d_tmp + active.size(), active.size() * sizeof(int64_t),
                                        cudaMemcpyDeviceToHost, st));
            CUDA_TRY(h, cudaStreamSynchronize(st));
        }
        std::vector<size_t> order(active.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(),
                         [&](size_t a, size_t b) { return key[a] > key[b]; });
        std::vector<int64_t> a2(active.size()), w2(active.size());
        for (size_t i = 0; i < order.size(); ++i) {
            a2[i] = active[order[i]];
            w2[i] = where[order[i]];
        }
        active.swap(a2);
        where.swap(w2);
    }
    tr.mark("run: source ordering");
    const int64_t k = (int64_t)active.size();
    // Unpartitioned unit-weight sweeps of a skewed graph run on the copy renumbered by descending
    // degree (bc_relabel.cuh): sources are renamed here, the BC vector on the way out.
    bool relabelled = !debug && mode == BC_MODE_DIRECT && h->k == 1 && h->dist_rank < 0 && k > 0 &&
                      relabel_wanted(h, k);
    if (!debug && mode == BC_MODE_DIRECT && h->k == 1) h->sources_seen += k;
    if (relabelled) {
        const int rc = ensure_relabelled(h, st);
        if (rc == BC_ERR_INPUT) return rc;   // an arc without its reverse
        if (rc != BC_OK) {
            // no room for the second copy (it needs ~5 x the arc array while it is built): this
            // handle stays on the caller's ids
            cudaGetLastError();
            free_csr(h->relab);
            h->relab_ready = false;
            h->relabel = 0;
            relabelled = false;
        }
    }
    if (relabelled) {
        ScopedBlock<int64_t> d_ids;
        CUDA_TRY(h, arena_malloc((void **)&d_ids.p, 2 * (size_t)k * sizeof(int64_t)));
        CUDA_TRY(h, cudaMemcpyAsync(d_ids.p, active.data(), k * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        relabel_sources_kernel<<<grid1d((size_t)k, 256), 256, 0, st>>>(d_ids.p, k, h->d_new_of_old, d_ids.p + k);
        ++h->launches;
        CUDA_TRY(h, cudaMemcpyAsync(active.data(), d_ids.p + k, k * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        tr.mark("run: renumbered graph");
    }
    const Csr &whole = relabelled ? h->relab : h->full;                       // the unpartitioned graph of this run
    const std::vector<int64_t> &whole_off = relabelled ? h->h_off_relab : h->h_off;
    const int64_t *sources = active.data();
    const int groups = debug ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(h->groups, (k + 31) / 32));
    TRY(ensure_state(h, groups, debug));
    TRY(ensure_levels(h, 2));
    const int S = 32 * groups;
    if (hybir) TRY(ensure_border_state(h, S));
    if (h->d_src_cap < k) {
        arena_free(h->d_src);
        h->d_src = nullptr;
        CUDA_TRY(h, arena_malloc((void **)&h->d_src, std::max<int64_t>(k, 1) * sizeof(int64_t)));
        h->d_src_cap = k;
    }
    tr.mark("run: state allocation");
    // The per-group BC partials are zeroed by reduce_bc_kernel at the end of a run.  After a fresh
    // allocation, or after a run that failed half way (its batches are already in there), clear
    // them here, on the caller's stream.
    if (h->bcg_dirty)
        CUDA_TRY(h, cudaMemsetAsync(h->bcg, 0, (size_t)h->alloc_groups * (size_t)n * sizeof(double), st));
    h->bcg_dirty = !debug;   // until reduce_bc_kernel has run
    // inspection reads sigma / delta rows; everything else may keep deep sweeps in level order
    struct AllowScope {
        bc_handle *h;
        ~AllowScope() { h->fwd_compact_allowed = false; }
    } allow_scope{h};
    h->fwd_compact_allowed = !debug;
    const int64_t launches0 = h->launches;
    const int64_t level_launches0 = h->level_launches;
    h->model_scan = h->model_pairs = h->model_vlanes = h->model_dense_words = h->model_entries = 0;
    int64_t h2d = 0, d2h = 0;
    if (k > 0) {
        CUDA_TRY(h, cudaMemcpyAsync(h->d_src, sources, k * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        h2d += k * sizeof(int64_t);
    }
    CUDA_TRY(h, cudaMemsetAsync(h->counters, 0, 8 * sizeof(unsigned long long), st));
    h->reports_host.assign((size_t)k_all * 8, 0);

    const int lanes_per_batch = S;
    const int64_t n_batches = (k + lanes_per_batch - 1) / lanes_per_batch;
    std::vector<Events> ev((size_t)n_batches);
    int max_depth = 0;
    int64_t launches_f = 0, launches_b = 0;
    int64_t tot_iters = 0, tot_comm = 0, tot_sync = 0, tot_bytes = 0;
    const Csr &fwd_csr = hybir ? h->intra : whole;
    // queue levels / push: the unpartitioned sweeps only (the partitioned modes
    // read dense level rows for borders and reports)
    const bool adaptive = h->sparse && !hybir && !(want_reports && h->k == 2) && h->full.wgt == nullptr;
    // hybir mode on low-degree (deep) graphs: Step 1 and Step 6 run on frontier queues inside the
    // parts (the dense level rows cost levels x n x groups x 4 B there), the border seeds of
    // Step 6 join the queue levels, and the backward sweep reads the same queues
    const bool qsweep = hybir && partition_queue_sweeps(h) && !(want_reports && h->k == 2);
    const bool queued = adaptive || qsweep;   // levels are LevelReps, not h->lvl[L]

    // debug staging: one batch (<= 32 sources) of [lane][n] rows
    ScopedBlock<int32_t> dbg_dist_blk;
    ScopedBlock<double> dbg_sigma_blk, dbg_delta_blk;
    if (debug) {
        if (dist_out) CUDA_TRY(h, arena_malloc((void **)&dbg_dist_blk.p, 32 * (size_t)n * sizeof(int32_t)));
        if (sigma_out) CUDA_TRY(h, arena_malloc((void **)&dbg_sigma_blk.p, 32 * (size_t)n * sizeof(double)));
        if (delta_out) CUDA_TRY(h, arena_malloc((void **)&dbg_delta_blk.p, 32 * (size_t)n * sizeof(double)));
    }
    int32_t *const dbg_dist = dbg_dist_blk.p;
    double *const dbg_sigma = dbg_sigma_blk.p, *const dbg_delta = dbg_delta_blk.p;

    // ---- Step 1 of a hybir batch + its border seeds, on stream `s`, into the given seed buffers.
    // Runs inline on the caller's stream, or -- look-ahead, engine.py:135-143 -- for batch b + 1 on
    // the side stream from a helper thread while the border phase of batch b is in flight: Step 1
    // needs the BFS state only, the border phase the border state only.
    struct Step1Out {
        int depth = 1;
        std::vector<LevelRep> reps;
        int rc = BC_OK;
    };
    auto step1 = [&](int64_t b, cudaStream_t s, int32_t *seedD, double *seedS, int32_t *lane_part,
                     Step1Out &out) -> int {
        const int cnt = (int)std::min<int64_t>(lanes_per_batch, k - b * lanes_per_batch);
        const int ng = (cnt + 31) / 32;
        const int64_t *batch_src = sources + b * lanes_per_batch;
        TRY(begin_batch(h, h->d_src + b * lanes_per_batch, cnt, ng, s, queued));
        h->cnt_off = 4;   // Step 1 is a partial traversal: keep it out of the totals
        const int rc = qsweep ? forward_adaptive(h, h->intra, ng, cnt, batch_src, s, &out.depth, out.reps,
                                                 &h->h_ioff, true)
                              : forward_sweep(h, h->intra, ng, s, &out.depth);
        h->cnt_off = 0;
        TRY(rc);
        const size_t bcnt = (size_t)h->B * h->border_S;
        std::vector<int32_t> lp(h->border_S, 0);
        for (int i = 0; i < cnt; ++i) lp[i] = h->h_part[batch_src[i]];
        CUDA_TRY(h, cudaMemcpyAsync(lane_part, lp.data(), h->border_S * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        CUDA_TRY(h, cudaStreamSynchronize(s));   // `lp` goes out of scope
        fill_seed_kernel<<<grid1d(bcnt, 256, 4736), 256, 0, s>>>(seedD, seedS, bcnt);
        if (qsweep) {
            TRY(upload_level_ends(h, out.reps, out.depth, s));
            if (h->B > 0)
                border_gather_queue_kernel<<<dim3(queue_blocks_all(out.reps, out.depth), ng), 256, 0, s>>>(
                    queue_params(h), h->range_table, out.depth, h->alloc_groups, n, h->d_border_index,
                    h->sigma, h->border_S, seedD, seedS, out.reps.back().compact ? h->qs : nullptr, h->q_off,
                    h->q_vcap);
        } else {
            TRY(upload_level_ptrs(h, out.depth, s));
            if (h->B > 0)
                border_gather_kernel<<<grid1d(bcnt), 256, 0, s>>>(
                    h->d_lvl_ptrs, h->live, h->alloc_groups, out.depth, h->sigma, n, border_geom(h),
                    h->border_S, seedD, seedS);
        }
        h->launches += 2;
        CUDA_TRY(h, cudaGetLastError());
        return BC_OK;
    };
    const bool lookahead = hybir && h->lookahead && !debug && n_batches > 1;
    if (lookahead && h->side_stream == nullptr) {
        CUDA_TRY(h, cudaStreamCreateWithFlags(&h->side_stream, cudaStreamNonBlocking));
        CUDA_TRY(h, cudaEventCreateWithFlags(&h->side_go, cudaEventDisableTiming));
        CUDA_TRY(h, cudaEventCreateWithFlags(&h->side_done, cudaEventDisableTiming));
    }
    Step1Out ahead;            // Step 1 of batch b + 1, filled by the look-ahead thread
    bool ahead_ready = false;
    int64_t lookahead_batches = 0;
    std::thread helper;
    struct Joiner {
        std::thread &t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } joiner{helper};

    for (int64_t b = 0; b < n_batches; ++b) {
        const int cnt = (int)std::min<int64_t>(lanes_per_batch, k - b * lanes_per_batch);
        const int ng = (cnt + 31) / 32;
        const int64_t *batch_src = sources + b * lanes_per_batch;
        Events &e = ev[(size_t)b];
        CUDA_TRY(h, cudaEventCreate(&e.start));
        CUDA_TRY(h, cudaEventCreate(&e.fwd_end));
        CUDA_TRY(h, cudaEventCreate(&e.border_end));
        CUDA_TRY(h, cudaEventCreate(&e.fwd2_end));
        CUDA_TRY(h, cudaEventCreate(&e.bwd_end));
        CUDA_TRY(h, cudaEventRecord(e.start, st));
        const int64_t l_start = h->launches;

        // ---- forward: Step 1 (or the whole BFS when there is no partition)
        int depth = 1;
        std::vector<LevelRep> reps;
        if (!hybir) {
            TRY(begin_batch(h, h->d_src + b * lanes_per_batch, cnt, ng, st, queued));
            if (adaptive) TRY(forward_adaptive(h, fwd_csr, ng, cnt, batch_src, st, &depth, reps, &whole_off));
            else TRY(forward_sweep(h, fwd_csr, ng, st, &depth));
        } else if (ahead_ready) {
            // issued ahead while the previous batch's border phase ran: its seeds sit in the
            // alternate buffers
            std::swap(h->seedD, h->seedD_alt);
            std::swap(h->seedS, h->seedS_alt);
            std::swap(h->lane_part, h->lane_part_alt);
            depth = ahead.depth;
            reps.swap(ahead.reps);
            ahead_ready = false;
        } else {
            Step1Out now;
            TRY(step1(b, st, h->seedD, h->seedS, h->lane_part, now));
            depth = now.depth;
            reps.swap(now.reps);
        }
        CUDA_TRY(h, cudaEventRecord(e.fwd_end, st));
        launches_f += h->launches - l_start;
        tr.mark("batch: forward (Step 1)");

        std::vector<int32_t> iters;
        std::vector<uint32_t> entered;
        if (hybir) {
            if (lookahead && b + 1 < n_batches) {
                // the BFS state is free until Step 6: Step 1 of the next batch takes it now
                CUDA_TRY(h, cudaEventRecord(h->side_go, st));
                CUDA_TRY(h, cudaStreamWaitEvent(h->side_stream, h->side_go, 0));
                ahead = Step1Out{};
                try {
                    helper = std::thread([&, b]() {
                        cudaSetDevice(h->device);
                        ahead.rc = step1(b + 1, h->side_stream, h->seedD_alt, h->seedS_alt, h->lane_part_alt, ahead);
                        if (ahead.rc == BC_OK && cudaEventRecord(h->side_done, h->side_stream) != cudaSuccess)
                            ahead.rc = BC_ERR_INTERNAL;
                    });
                } catch (const std::exception &) {
                    // no thread to be had: the next batch runs its Step 1 inline, as without look-ahead
                }
            }
            // ---- Steps 2-5 + path-count composition on the border tables
            int max_seed = -1;
            const int rc_border = refine_and_compose(h, cnt, ng, st, &iters, &entered, &max_seed);
            SeedPlan plan{};
            int rc_plan = BC_OK;
            if (rc_border == BC_OK && qsweep) rc_plan = build_seed_plan(h, cnt, max_seed, st, &plan);
            if (helper.joinable()) {
                helper.join();
                if (ahead.rc != BC_OK) return ahead.rc;
                // Step 6 below takes the BFS state over: wait for the look-ahead's gather
                CUDA_TRY(h, cudaStreamWaitEvent(st, h->side_done, 0));
                ahead_ready = true;
                ++lookahead_batches;
            }
            TRY(rc_border);
            TRY(rc_plan);
            tr.mark("batch: border phase");
            CUDA_TRY(h, cudaEventRecord(e.border_end, st));
            // ---- Step 6: every part relaxes from its borders at once
            const int64_t l_step6 = h->launches;
            TRY(begin_batch(h, h->d_src + b * lanes_per_batch, cnt, ng, st, qsweep));
            if (qsweep) TRY(forward_adaptive(h, h->intra, ng, cnt, batch_src, st, &depth, reps, &h->h_ioff, true, &plan));
            else TRY(forward_sweep(h, h->intra, ng, st, &depth, true, cnt, max_seed));
            CUDA_TRY(h, cudaEventRecord(e.fwd2_end, st));
            launches_f += h->launches - l_step6;
            tr.mark("batch: Step 6");
        } else {
            CUDA_TRY(h, cudaEventRecord(e.border_end, st));
            CUDA_TRY(h, cudaEventRecord(e.fwd2_end, st));
        }
        max_depth = std::max(max_depth, depth);

        // ---- backward over the whole graph (cross-part children are final by
        // the time their parents' level runs: levels are global)
        const int64_t l_bwd = h->launches;
        if (queued) TRY(backward_adaptive(h, whole, depth, reps, ng, debug, st));
        else TRY(backward_sweep(h, whole, depth, ng, debug, st));
        h->last_depth = depth;
        if (queued && !debug && h->lazy_clear) {
            // the sweep cleared every pair it visited; the sources (level 0) are left
            clear_source_sigma_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(h->d_src + b * lanes_per_batch, cnt, n,
                                                                        h->sigma);
            ++h->launches;
            h->sigma_clean_groups = h->sigma_clean_after;
        }
        CUDA_TRY(h, cudaEventRecord(e.bwd_end, st));
        launches_b += h->launches - l_bwd;
        tr.mark("batch: backward");

        if (want_reports && h->k == 2) {
            // ---- per-source reports (forward.py:52-64, backward.py:33-43, bsp.py:96-103,137-141)
            const size_t G = (size_t)h->alloc_groups;
            const size_t pw = (size_t)depth * h->k * G;
            if (h->presence_words < pw) {
                arena_free(h->presence);
                h->presence = nullptr;
                CUDA_TRY(h, arena_malloc((void **)&h->presence, pw * sizeof(uint32_t)));
                h->presence_words = pw;
            }
            CUDA_TRY(h, cudaMemsetAsync(h->presence, 0, pw * sizeof(uint32_t), st));
            for (int L = 0; L < depth; ++L) {
                level_presence_kernel<<<dim3(grid1d((size_t)n, 256, 296), ng), 256,
                                        h->k * sizeof(uint32_t), st>>>(
                    h->lvl[L], h->live + (size_t)L * G, h->d_part, n, h->k, (int)G,
                    h->presence + (size_t)L * h->k * G);
                ++h->launches;
            }
            std::vector<uint32_t> pres(pw);
            CUDA_TRY(h, cudaMemcpyAsync(pres.data(), h->presence, pw * sizeof(uint32_t),
                                        cudaMemcpyDeviceToHost, st));
            std::vector<int64_t> lsync(h->border_S, 0), lbytes(h->border_S, 0);
            if (hybir && h->B > 0) {
                const size_t bcnt = (size_t)h->B * h->border_S;
                const int W = (depth + 31) / 32 + 1;
                const int wm = h->full.wgt ? h->wmax : 1;
                const size_t words = (size_t)2 * W * wm * h->border_S;
                if (words > ((size_t)1 << 28))
                    return h->fail(BC_ERR_INPUT, "per-source sync reports need too much memory for these weights "
                                                 "and depths; run with reports = 0");
                if (h->sync_bits_words < words) {
                    TRY(dev_alloc(h, &h->sync_bits, words));
                    h->sync_bits_words = words;
                }
                CUDA_TRY(h, cudaMemsetAsync(h->sync_bits, 0, words * sizeof(uint32_t), st));
                TRY(upload_level_ptrs(h, depth, st));
                border_gather_kernel<<<grid1d(bcnt), 256, 0, st>>>(
                    h->d_lvl_ptrs, h->live, h->alloc_groups, depth, h->sigma, n, border_geom(h),
                    h->border_S, h->Dfin, nullptr);
                sync_mark_kernel<<<grid1d(bcnt), 256, 0, st>>>(border_geom(h), h->border_S, h->Dfin,
                                                               h->sync_flag, h->sync_bits, W, wm);
                sync_count_kernel<<<grid1d((size_t)h->border_S, 128), 128, 0, st>>>(
                    h->B, h->border_S, W, wm, h->sync_flag, h->sync_bits, h->lane_sync, h->lane_bytes);
                h->launches += 3;
                CUDA_TRY(h, cudaMemcpyAsync(lsync.data(), h->lane_sync, h->border_S * sizeof(int64_t),
                                            cudaMemcpyDeviceToHost, st));
                CUDA_TRY(h, cudaMemcpyAsync(lbytes.data(), h->lane_bytes, h->border_S * sizeof(int64_t),
                                            cudaMemcpyDeviceToHost, st));
            }
            CUDA_TRY(h, cudaStreamSynchronize(st));
            int64_t border_total = h->B;
            for (int i = 0; i < cnt; ++i) {
                const size_t g = i >> 5;
                const uint32_t bit = 1u << (i & 31);
                int64_t maxl[2] = {0, 0}, nl[2] = {0, 0}, global_levels = 0;
                for (int L = 0; L < depth; ++L) {
                    bool any = false;
                    for (int p = 0; p < 2; ++p)
                        if (pres[((size_t)L * h->k + p) * G + g] & bit) {
                            maxl[p] = L;
                            ++nl[p];
                            any = true;
                        }
                    global_levels += any;
                }
                int64_t *r = &h->reports_host[(size_t)where[b * lanes_per_batch + i] * 8];
                if (hybir) {
                    r[0] = iters[i];
                    r[1] = entered[i] ? 2 * (int64_t)iters[i] + 1 : 0;
                    r[4] = lsync[i];
                    r[5] = lbytes[i];
                } else {
                    // level-synchronous baseline: one exchange per level that has a successor
                    r[0] = global_levels - 1;
                    r[1] = 2 * (global_levels - 1);
                    r[4] = 2 * (global_levels - 1);
                    r[5] = (global_levels - 1) * border_total * 16;
                }
                r[2] = maxl[0];
                r[3] = maxl[1];
                r[6] = nl[0];
                r[7] = nl[1];
                tot_iters += r[0];
                tot_comm += r[1];
                tot_sync += r[4];
                tot_bytes += r[5];
            }
        } else if (hybir) {
            for (int i = 0; i < cnt; ++i) {
                int64_t *r = &h->reports_host[(size_t)where[b * lanes_per_batch + i] * 8];
                r[0] = iters[i];
                tot_iters += r[0];
            }
        }

        if (debug) {
            const size_t rows = (size_t)cnt * (size_t)n;
            const unsigned fb = grid1d(rows, 256, 4736);
            if (dbg_dist) fill_i32_kernel<<<fb, 256, 0, st>>>(dbg_dist, rows, BC_UNREACHED);
            if (dbg_sigma) CUDA_TRY(h, cudaMemsetAsync(dbg_sigma, 0, rows * sizeof(double), st));
            if (dbg_delta) CUDA_TRY(h, cudaMemsetAsync(dbg_delta, 0, rows * sizeof(double), st));
            for (int L = 0; L < depth; ++L) {
                if (queued && reps[L].slot < 0) {
                    TRY(upload_ranges(h, reps[L], st));
                    extract_queue_kernel<<<dim3(queue_blocks(reps[L], 256), 1), 256, 0, st>>>(
                        queue_params(h), h->sigma, h->delta, n, L, dbg_dist, dbg_sigma, dbg_delta);
                } else {
                    extract_level_kernel<<<dim3(grid1d((size_t)n, 256, 1184), 1), 256, 0, st>>>(
                        h->lvl[queued ? reps[L].slot : L], h->live + (size_t)L * h->alloc_groups,
                        h->sigma, h->delta, n, L, dbg_dist, dbg_sigma, dbg_delta);
                }
                ++h->launches;
            }
            CUDA_TRY(h, cudaGetLastError());
            const size_t o = (size_t)b * 32 * (size_t)n;
            if (dbg_dist)
                CUDA_TRY(h, cudaMemcpyAsync(dist_out + o, dbg_dist, rows * sizeof(int32_t),
                                            cudaMemcpyDeviceToHost, st));
            if (dbg_sigma)
                CUDA_TRY(h, cudaMemcpyAsync(sigma_out + o, dbg_sigma, rows * sizeof(double),
                                            cudaMemcpyDeviceToHost, st));
            if (dbg_delta)
                CUDA_TRY(h, cudaMemcpyAsync(delta_out + o, dbg_delta, rows * sizeof(double),
                                            cudaMemcpyDeviceToHost, st));
            CUDA_TRY(h, cudaStreamSynchronize(st));
        }
    }
    if (!debug && bc_dev != nullptr) {
        // (groups beyond the ones this run used hold zeros)
        reduce_bc_kernel<<<grid1d((size_t)n, 256, 4736), 256, 0, st>>>(bc_dev, h->bcg, n, groups,
                                                                       relabelled ? h->d_old_of_new : nullptr);
        ++h->launches;
        CUDA_TRY(h, cudaGetLastError());
        h->bcg_dirty = false;
    }
    unsigned long long cnts[8] = {0};
    CUDA_TRY(h, cudaMemcpyAsync(cnts, h->counters, sizeof cnts, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    d2h += sizeof cnts;
    tr.mark("run: batches");

    double ms_level = 0;
    const bool level_trace = getenv("BC_LEVEL_TRACE") != nullptr;   // dev: one line per timed level launch
    const int64_t level_timed = (int64_t)h->level_events.size();
    for (auto &pr : h->level_events) {
        float t = 0;
        if (cudaEventElapsedTime(&t, pr.first, pr.second) == cudaSuccess) ms_level += t;
        if (level_trace) fprintf(stderr, "[bc level %d] %.3f ms\n", (int)(&pr - h->level_events.data()), t);
        cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
    }
    h->level_events.clear();
    double ms_f = 0, ms_b = 0, ms_border = 0;
    for (Events &e : ev) {
        float a = 0, bo = 0, f2 = 0, bw = 0;
        cudaEventElapsedTime(&a, e.start, e.fwd_end);
        cudaEventElapsedTime(&bo, e.fwd_end, e.border_end);
        cudaEventElapsedTime(&f2, e.border_end, e.fwd2_end);
        cudaEventElapsedTime(&bw, e.fwd2_end, e.bwd_end);
        ms_f += a + f2;
        ms_border += bo;
        ms_b += bw;
    }
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->sources = k_all;
        stats->batches = n_batches;
        stats->max_levels = std::max<int64_t>(max_depth, k_all > 0 ? 1 : 0);
        // sources themselves are reached vertices too (level 0); in hybir mode
        // the totals count Step 6 (arcs inside the parts; cut arcs are not walked)
        stats->reached = (int64_t)cnts[0] + k_all;
        int64_t src_arcs = 0;
        for (int64_t i = 0; i < k; ++i) src_arcs += whole_off[sources[i] + 1] - whole_off[sources[i]];
        stats->arcs_reached = (int64_t)cnts[1] + src_arcs;
        stats->dag_arcs = (int64_t)cnts[2];
        stats->launches = h->launches - launches0;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = d2h;
        stats->ms_total = ms_f + ms_b + ms_border;
        stats->ms_forward = ms_f;
        stats->ms_backward = ms_b;
        stats->ms_border = ms_border;
        stats->iterations = tot_iters;
        stats->comm_events = tot_comm;
        stats->sync_events = tot_sync;
        stats->comm_bytes = tot_bytes;
        stats->launches_forward = launches_f;
        stats->launches_backward = launches_b;
        stats->launches_level = h->level_launches - level_launches0;
        stats->ms_level = ms_level;
        stats->launches_level_timed = level_timed;
        stats->lookahead_batches = lookahead_batches;
        stats->level_scan_arcs = h->model_scan;
        stats->level_pairs = h->model_pairs;
        stats->level_vertex_lanes = h->model_vlanes;
        stats->level_dense_words = h->model_dense_words;
        stats->level_entries = h->model_entries;
        // col_idx word + mask probe per scanned arc; one fp64 per gathered pair and per
        // (vertex, lane) value; 4 B per dense mask word; 16 B of BC partial per backward entry;
        // row offsets once per launch
        // (complete only with option model_counters = 1: the forward pulls count their scanned arcs then)
        stats->level_model_bytes = h->model_counters
                                       ? 8 * h->model_scan + 8 * h->model_pairs + 8 * h->model_vlanes +
                                             4 * h->model_dense_words + 16 * h->model_entries +
                                             8 * h->n * stats->launches_level
                                       : 0;
    }
    return BC_OK;
}

}  // namespace
