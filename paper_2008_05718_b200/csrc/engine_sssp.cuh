// engine_sssp.cuh -- the source loop for graphs with general positive integer arc weights
// (bc_sssp.cuh): batches of 32 x groups sources through label-correcting distances, the tight-arc
// counts, and the two dependency-counted sweeps.  BC_MODE_DIRECT only.
#pragma once

namespace {

constexpr int kSsspFlagCap = 1 << 14;   // rounds per flag epoch

// Weighted graphs leave the level-per-distance kernels when a level per distance value is out of
// reach: weights above 4096, or a deep (low-degree) graph with weights above 16, where the number
// of distance values is the depth times the weights.  Option "sssp" overrides the rule.
bool general_weights(const bc_handle *h) {
    if (h->full.wgt == nullptr) return false;
    if (h->wgt_mode >= 0) return h->wgt_mode == 1;
    return h->wmax > 4096 || (h->wmax > 16 && h->n_arcs < 6 * h->n);
}

int ensure_sssp_state(bc_handle *h, int groups) {
    if (h->sp_groups >= groups) return BC_OK;
    free_sssp_state(h);
    const size_t n = (size_t)h->n;
    CUDA_TRY(h, arena_malloc((void **)&h->sp_dist, groups * n * 32 * sizeof(long long)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_npar, groups * n * 32 * sizeof(int)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_nchild, groups * n * 32 * sizeof(int)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_maskA, groups * n * sizeof(uint32_t)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_maskB, groups * n * sizeof(uint32_t)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_leaf, groups * n * sizeof(uint32_t)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_flags, kSsspFlagCap * sizeof(int)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_bound, 2 * kSsspFlagCap * sizeof(long long)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_queue, 3 * groups * n * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&h->sp_qcount, 4 * (size_t)groups * sizeof(int)));
    h->sp_groups = groups;
    return BC_OK;
}

// Runs `kernel` round after round until a round leaves nothing for the next one; both mask arrays
// are empty at the end.  Rounds are launched in growing chunks: a launch behind the last productive
// round returns at once.  near_far (phase A): the rounds carry a distance bound (bc_sssp.cuh).
template <typename Kernel>
int sssp_rounds(bc_handle *h, Kernel kernel, SsspParams &p, int ng, cudaStream_t st, int64_t *rounds_out,
                bool near_far = false) {
    // one wave of blocks over all groups; a warp takes 32 queue entries per step
    const int64_t warps = (h->n + kSsspChunk - 1) / kSsspChunk;
    const unsigned blocks = (unsigned)std::min<int64_t>((warps + kSsspWarps - 1) / kSsspWarps,
                                                        std::max(h->sp_blocks > 0 ? h->sp_blocks : 296, 148 * 8 / ng));
    const dim3 grid(blocks, (unsigned)ng);
    int64_t rounds = 0;
    int chunk = 8;
    std::vector<int> flags;
    long long bound = p.step;   // first round: the sources (distance 0) are below any positive bound
    for (;;) {
        // one flag epoch: rounds [0, kSsspFlagCap)
        CUDA_TRY(h, cudaMemsetAsync(h->sp_flags, 0, kSsspFlagCap * sizeof(int), st));
        if (near_far) {
            fill_i64_kernel<<<grid1d(kSsspFlagCap, 256), 256, 0, st>>>(p.far_min, kSsspFlagCap, kSsspInf);
            CUDA_TRY(h, cudaMemcpyAsync(p.threshold, &bound, sizeof bound, cudaMemcpyHostToDevice, st));
            CUDA_TRY(h, cudaStreamSynchronize(st));   // `bound` is a stack variable
        }
        int r = 0;
        bool ended = false;
        while (r < kSsspFlagCap && !ended) {
            const int m = std::min(chunk, kSsspFlagCap - r);
            for (int j = 0; j < m; ++j) {
                p.round = r + j;
                kernel<<<grid, kSsspWarps * 32, 0, st>>>(p);
                std::swap(p.cur, p.next);
                std::swap(p.q_cur, p.q_next);
                p.qs_zero = p.qs_in;              // consumed: cleared by the round after next
                p.qs_in = p.qs_out;
                p.qs_out = 3 - p.qs_zero - p.qs_in;
                ++h->launches;
            }
            flags.assign(m, 0);
            CUDA_TRY(h, cudaMemcpyAsync(flags.data(), h->sp_flags + r, m * sizeof(int), cudaMemcpyDeviceToHost, st));
            CUDA_TRY(h, cudaStreamSynchronize(st));
            CUDA_TRY(h, cudaGetLastError());
            for (int j = 0; j < m; ++j)
                if (flags[j] == 0) {
                    // round r + j left nothing behind: the sweep is over, both mask arrays are empty
                    // (the launches behind it returned at once)
                    rounds += j + 1;
                    ended = true;
                    break;
                }
            if (!ended) rounds += m;
            r += m;
            chunk = std::min(chunk * 2, 256);
        }
        if (ended) break;
        if (near_far) {
            // the bound of the next epoch's first round, by the rule the kernel applies
            long long last[2] = {0, 0};
            CUDA_TRY(h, cudaMemcpy(&last[0], p.threshold + kSsspFlagCap - 1, sizeof(long long), cudaMemcpyDeviceToHost));
            CUDA_TRY(h, cudaMemcpy(&last[1], p.far_min + kSsspFlagCap - 1, sizeof(long long), cudaMemcpyDeviceToHost));
            bound = flags.back() == 1 ? last[1] + p.step : last[0];
        }
    }
    if (rounds_out) *rounds_out = rounds;
    return BC_OK;
}

int run_sources_sssp(bc_handle *h, const int64_t *sources_in, int64_t k_all, double *bc_dev, cudaStream_t st,
                     bc_stats *stats, bool debug, int32_t *dist_out, double *sigma_out, double *delta_out) {
    const int64_t n = h->n;
    Trace tr;
    for (int64_t i = 0; i < k_all; ++i)
        if (sources_in[i] < 0 || sources_in[i] >= n) {
            char buf[128];
            snprintf(buf, sizeof buf, "listed source %lld out of range [0, %lld)", (long long)sources_in[i],
                     (long long)n);
            return h->fail(BC_ERR_INPUT, buf);
        }
    drop_level_events(h);
    // sources without arcs reach nothing (as in run_sources): no lane on the device outside inspection
    std::vector<int64_t> active;
    for (int64_t i = 0; i < k_all; ++i)
        if (debug || h->h_off[sources_in[i] + 1] > h->h_off[sources_in[i]]) active.push_back(sources_in[i]);
    const int64_t k = (int64_t)active.size();
    const int groups = debug ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(h->groups, (k + 31) / 32));
    TRY(ensure_state(h, groups, debug));
    TRY(ensure_sssp_state(h, groups));
    if (h->d_src_cap < k) {
        arena_free(h->d_src);
        h->d_src = nullptr;
        CUDA_TRY(h, arena_malloc((void **)&h->d_src, std::max<int64_t>(k, 1) * sizeof(int64_t)));
        h->d_src_cap = k;
    }
    if (h->bcg_dirty)
        CUDA_TRY(h, cudaMemsetAsync(h->bcg, 0, (size_t)h->alloc_groups * (size_t)n * sizeof(double), st));
    h->bcg_dirty = !debug;
    h->sigma_clean_groups = 0;   // this path writes the rows without clearing them afterwards
    const int64_t launches0 = h->launches;
    int64_t h2d = 0, d2h = 0;
    if (k > 0) {
        CUDA_TRY(h, cudaMemcpyAsync(h->d_src, active.data(), k * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        h2d += k * sizeof(int64_t);
    }
    CUDA_TRY(h, cudaMemsetAsync(h->counters, 0, 8 * sizeof(unsigned long long), st));
    h->reports_host.assign((size_t)k_all * 8, 0);

    ScopedBlock<int32_t> dbg_dist_blk;
    ScopedBlock<double> dbg_sigma_blk, dbg_delta_blk;
    ScopedBlock<int> overflow_blk;
    if (debug) {
        if (dist_out) CUDA_TRY(h, arena_malloc((void **)&dbg_dist_blk.p, 32 * (size_t)n * sizeof(int32_t)));
        if (sigma_out) CUDA_TRY(h, arena_malloc((void **)&dbg_sigma_blk.p, 32 * (size_t)n * sizeof(double)));
        if (delta_out) CUDA_TRY(h, arena_malloc((void **)&dbg_delta_blk.p, 32 * (size_t)n * sizeof(double)));
        CUDA_TRY(h, arena_malloc((void **)&overflow_blk.p, sizeof(int)));
        CUDA_TRY(h, cudaMemsetAsync(overflow_blk.p, 0, sizeof(int), st));
    }

    const int S = 32 * groups;
    const int64_t n_batches = (k + S - 1) / S;
    int64_t max_rounds = 0, launches_f = 0, launches_b = 0;
    double ms_f = 0, ms_b = 0;
    Events e;
    CUDA_TRY(h, cudaEventCreate(&e.start));
    CUDA_TRY(h, cudaEventCreate(&e.fwd_end));
    CUDA_TRY(h, cudaEventCreate(&e.bwd_end));
    for (int64_t b = 0; b < n_batches; ++b) {
        const int cnt = (int)std::min<int64_t>(S, k - b * S);
        const int ng = (cnt + 31) / 32;
        CUDA_TRY(h, cudaEventRecord(e.start, st));
        const int64_t l0 = h->launches;
        SsspParams p{};
        p.off = h->full.off;
        p.col = h->full.col;
        p.wgt = h->full.wgt;
        p.n = n;
        p.dist = h->sp_dist;
        p.sigma = h->sigma;
        p.coef = h->coef;
        p.delta = debug ? h->delta : nullptr;
        p.npar = h->sp_npar;
        p.nchild = h->sp_nchild;
        p.cur = h->sp_maskA;
        p.next = h->sp_maskB;
        p.leaf = h->sp_leaf;
        p.bcg = h->bcg;
        p.flags = h->sp_flags;
        p.threshold = h->sp_bound;
        p.far_min = h->sp_bound + kSsspFlagCap;
        // bound step: small = little wasted relaxation but many rounds; 16 mean weights was the best
        // of 1 .. 60 on a 1024^2 road grid with weights up to 10^5 (419 / 221 / 162 / 170 ms)
        p.step = h->sp_delta > 0 ? h->sp_delta : std::max<long long>(1, 16 * (h->wsum / std::max<int64_t>(h->n_arcs, 1)));
        p.accumulate = debug ? 0 : 1;
        p.counters = h->counters;
        const size_t G = (size_t)h->sp_groups;
        p.G = (int)G;
        p.q_cur = h->sp_queue;
        p.q_next = h->sp_queue + G * (size_t)n;
        p.q_leaf = h->sp_queue + 2 * G * (size_t)n;
        p.q_count = h->sp_qcount;
        p.q_leaf_count = h->sp_qcount + 3 * G;
        // queue length slots: a phase starts with its first frontier in slot 0, the others empty
        auto reset_slots = [&]() -> int {
            CUDA_TRY(h, cudaMemsetAsync(p.q_count, 0, 3 * G * sizeof(int), st));
            p.qs_in = 0, p.qs_out = 1, p.qs_zero = 2;
            return BC_OK;
        };
        TRY(reset_slots());
        CUDA_TRY(h, cudaMemsetAsync(p.q_leaf_count, 0, G * sizeof(int), st));
        sssp_init_kernel<<<dim3(grid1d((size_t)n * 32, 256, 2368), ng), 256, 0, st>>>(p.dist, p.cur, p.next, p.leaf, n);
        sssp_seed_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(h->d_src + b * S, cnt, n, p.dist, p.cur, p.q_cur, p.q_count);
        h->launches += 2;
        // ---- A: distances
        int64_t rounds_a = 0, rounds_c = 0, rounds_d = 0;
        TRY(sssp_rounds(h, sssp_relax_kernel, p, ng, st, &rounds_a, true));
        tr.mark("batch: distances");
        // ---- B: tight-arc counts, first frontiers
        const dim3 grid((unsigned)((n + 32 * kSsspWarps - 1) / (32 * kSsspWarps)), (unsigned)ng);
        TRY(reset_slots());
        sssp_count_kernel<<<grid, kSsspWarps * 32, 0, st>>>(p);
        ++h->launches;
        // ---- C: path counts
        TRY(sssp_rounds(h, sssp_forward_kernel, p, ng, st, &rounds_c));
        CUDA_TRY(h, cudaEventRecord(e.fwd_end, st));
        launches_f += h->launches - l0;
        tr.mark("batch: tight-arc counts + path counts");
        // ---- D: dependencies from the leaves
        const int64_t l1 = h->launches;
        // the leaf masks and the leaf queue are the first frontier as they are (both mask arrays and
        // both queues of phase C are empty by now; the leaf buffers are rebuilt by the next batch)
        TRY(reset_slots());
        p.cur = p.leaf;
        p.q_cur = p.q_leaf;
        CUDA_TRY(h, cudaMemcpyAsync(p.q_count, p.q_leaf_count, G * sizeof(int), cudaMemcpyDeviceToDevice, st));
        TRY(sssp_rounds(h, sssp_backward_kernel, p, ng, st, &rounds_d));
        CUDA_TRY(h, cudaEventRecord(e.bwd_end, st));
        launches_b += h->launches - l1;
        tr.mark("batch: dependencies");
        if (tr.on)
            fprintf(stderr, "[bc_b200] rounds: distances %lld, path counts %lld, dependencies %lld\n",
                    (long long)rounds_a, (long long)rounds_c, (long long)rounds_d);
        max_rounds = std::max(max_rounds, rounds_c);
        h->last_depth = (int)std::min<int64_t>(rounds_c, 1 << 30);

        if (debug) {
            sssp_extract_kernel<<<grid1d((size_t)n * 32, 256, 2368), 256, 0, st>>>(
                p.dist, p.sigma, h->delta, n, cnt, BC_UNREACHED, dbg_dist_blk.p, dbg_sigma_blk.p, dbg_delta_blk.p,
                overflow_blk.p);
            ++h->launches;
            const size_t rows = (size_t)cnt * (size_t)n;
            const size_t o = (size_t)b * 32 * (size_t)n;
            if (dist_out)
                CUDA_TRY(h, cudaMemcpyAsync(dist_out + o, dbg_dist_blk.p, rows * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            if (sigma_out)
                CUDA_TRY(h, cudaMemcpyAsync(sigma_out + o, dbg_sigma_blk.p, rows * sizeof(double), cudaMemcpyDeviceToHost, st));
            if (delta_out)
                CUDA_TRY(h, cudaMemcpyAsync(delta_out + o, dbg_delta_blk.p, rows * sizeof(double), cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(h, cudaStreamSynchronize(st));
        float a = 0, bw = 0;
        cudaEventElapsedTime(&a, e.start, e.fwd_end);
        cudaEventElapsedTime(&bw, e.fwd_end, e.bwd_end);
        ms_f += a;
        ms_b += bw;
    }
    if (debug) {
        int overflow = 0;
        CUDA_TRY(h, cudaMemcpyAsync(&overflow, overflow_blk.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        if (overflow && dist_out)
            return h->fail(BC_ERR_INPUT, "a shortest-path distance exceeds the int32 inspection array");
    }
    if (!debug && bc_dev != nullptr) {
        reduce_bc_kernel<<<grid1d((size_t)n, 256, 4736), 256, 0, st>>>(bc_dev, h->bcg, n, groups);
        ++h->launches;
        CUDA_TRY(h, cudaGetLastError());
        h->bcg_dirty = false;
    }
    unsigned long long cnts[8] = {0};
    CUDA_TRY(h, cudaMemcpyAsync(cnts, h->counters, sizeof cnts, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    d2h += sizeof cnts;
    tr.mark("run: batches");
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->sources = k_all;
        stats->batches = n_batches;
        stats->max_levels = std::max<int64_t>(max_rounds, k_all > 0 ? 1 : 0);   // depth of the DAG in arcs
        stats->reached = (int64_t)cnts[0] + k_all;
        int64_t src_arcs = 0;
        for (int64_t i = 0; i < k; ++i) src_arcs += h->h_off[active[i] + 1] - h->h_off[active[i]];
        stats->arcs_reached = (int64_t)cnts[1] + src_arcs;
        stats->dag_arcs = (int64_t)cnts[2];
        stats->launches = h->launches - launches0;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = d2h;
        stats->ms_total = ms_f + ms_b;
        stats->ms_forward = ms_f;
        stats->ms_backward = ms_b;
        stats->launches_forward = launches_f;
        stats->launches_backward = launches_b;
    }
    return BC_OK;
}

}  // namespace
