// bc_engine.cu -- host side of the C ABI declared in include/bc_b200.h.
//
// One handle = one CUDA device = one host thread.  The handle owns the CSR on
// the device, the warp work items derived from it and the per-batch state;
// sources are processed in batches of 32 * groups lanes.  There is no CPU
// code path for the arithmetic: every bc_run* call launches the kernels of
// bc_kernels.cuh or fails.
#include "bc_b200.h"
#include "bc_kernels.cuh"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace bcb200;

namespace {

thread_local std::string g_create_error;

// Device-side CSR plus the work items of the level kernels.
struct Csr {
    int64_t n = 0, n_arcs = 0;
    int64_t *off = nullptr;
    int32_t *col = nullptr;
    bool owns_graph = false;
    int n_chk = 0, n_rng = 0, n_hub = 0;
    int32_t *chk_v = nullptr;
    int64_t *chk_a0 = nullptr, *chk_a1 = nullptr;
    int32_t *rng_v0 = nullptr, *rng_nv = nullptr;
    int32_t *hub_v = nullptr, *hub_c0 = nullptr, *hub_nc = nullptr;
};

struct Events {
    cudaEvent_t start, fwd_end, bwd_end;
};

}  // namespace

struct bc_handle {
    int device = 0;
    int64_t n = 0, n_arcs = 0;
    std::vector<int64_t> h_off;  // host copy of offsets (item building, partition set-up)
    Csr full;
    // options
    int groups = 4;
    int item_arcs = 512;
    int reports = 1;
    // per-batch state
    int alloc_groups = 0;
    uint32_t *vis = nullptr;
    std::vector<uint32_t *> lvl;
    double *sigma = nullptr, *coef = nullptr, *delta = nullptr;
    double *bcg = nullptr;
    double *pacc = nullptr;
    uint32_t *pmask = nullptr;
    int pacc_chunks = 0;
    uint32_t *live = nullptr;  // [level][alloc_groups] lanes with a non-empty frontier
    int live_cap = 0;          // levels
    unsigned long long *counters = nullptr;
    int64_t *d_src = nullptr;
    int64_t d_src_cap = 0;
    double *bc_scratch = nullptr;  // device bc vector of bc_run
    std::string err;
    int64_t launches = 0;

    int fail(int code, const std::string &msg) {
        err = msg;
        return code;
    }
};

#define CUDA_TRY(h, call)                                                                  \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            char buf_[512];                                                                \
            snprintf(buf_, sizeof buf_, "%s failed: %s (%s:%d)", #call,                    \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                          \
            return (h)->fail(BC_ERR_INTERNAL, buf_);                                       \
        }                                                                                  \
    } while (0)

namespace {

template <typename T>
int upload(bc_handle *h, T **dst, const std::vector<T> &src) {
    *dst = nullptr;
    if (src.empty()) return BC_OK;
    CUDA_TRY(h, cudaMalloc((void **)dst, src.size() * sizeof(T)));
    CUDA_TRY(h, cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    return BC_OK;
}

void free_csr(Csr &c) {
    if (c.owns_graph) {
        cudaFree(c.off);
        cudaFree(c.col);
    }
    cudaFree(c.chk_v), cudaFree(c.chk_a0), cudaFree(c.chk_a1);
    cudaFree(c.rng_v0), cudaFree(c.rng_nv);
    cudaFree(c.hub_v), cudaFree(c.hub_c0), cudaFree(c.hub_nc);
    c = Csr();
}

// Cut the vertex set into warp work items: runs of <= 32 consecutive vertices
// holding <= item_arcs arcs, and, for vertices above 2 * item_arcs arcs
// ("hubs"), slices of item_arcs arcs whose partial sums a second kernel adds
// in order.
int build_items(bc_handle *h, Csr &c, const int64_t *off, int item_arcs) {
    std::vector<int32_t> chk_v, rng_v0, rng_nv, hub_v, hub_c0, hub_nc;
    std::vector<int64_t> chk_a0, chk_a1;
    const int64_t hub_deg = 2 * (int64_t)item_arcs;
    int64_t run_v0 = -1, run_arcs = 0;
    int run_nv = 0;
    auto flush = [&]() {
        if (run_nv > 0) {
            rng_v0.push_back((int32_t)run_v0);
            rng_nv.push_back(run_nv);
        }
        run_v0 = -1;
        run_nv = 0;
        run_arcs = 0;
    };
    for (int64_t v = 0; v < c.n; ++v) {
        const int64_t deg = off[v + 1] - off[v];
        if (deg > hub_deg) {
            flush();
            hub_v.push_back((int32_t)v);
            hub_c0.push_back((int32_t)chk_v.size());
            int nc = 0;
            for (int64_t a = off[v]; a < off[v + 1]; a += item_arcs) {
                chk_v.push_back((int32_t)v);
                chk_a0.push_back(a);
                chk_a1.push_back(std::min<int64_t>(a + item_arcs, off[v + 1]));
                ++nc;
            }
            hub_nc.push_back(nc);
            continue;
        }
        if (run_nv == 32 || (run_nv > 0 && run_arcs + deg > item_arcs)) flush();
        if (run_nv == 0) run_v0 = v;
        ++run_nv;
        run_arcs += deg;
    }
    flush();
    c.n_chk = (int)chk_v.size();
    c.n_rng = (int)rng_v0.size();
    c.n_hub = (int)hub_v.size();
    int rc;
    if ((rc = upload(h, &c.chk_v, chk_v))) return rc;
    if ((rc = upload(h, &c.chk_a0, chk_a0))) return rc;
    if ((rc = upload(h, &c.chk_a1, chk_a1))) return rc;
    if ((rc = upload(h, &c.rng_v0, rng_v0))) return rc;
    if ((rc = upload(h, &c.rng_nv, rng_nv))) return rc;
    if ((rc = upload(h, &c.hub_v, hub_v))) return rc;
    if ((rc = upload(h, &c.hub_c0, hub_c0))) return rc;
    if ((rc = upload(h, &c.hub_nc, hub_nc))) return rc;
    return BC_OK;
}

void free_state(bc_handle *h) {
    cudaFree(h->vis);
    for (uint32_t *p : h->lvl) cudaFree(p);
    h->lvl.clear();
    cudaFree(h->sigma), cudaFree(h->coef), cudaFree(h->delta), cudaFree(h->bcg);
    cudaFree(h->pacc), cudaFree(h->pmask);
    cudaFree(h->live);
    h->live = nullptr;
    h->live_cap = 0;
    h->vis = nullptr;
    h->sigma = h->coef = h->delta = h->bcg = h->pacc = nullptr;
    h->pmask = nullptr;
    h->alloc_groups = 0;
    h->pacc_chunks = 0;
}

int ensure_state(bc_handle *h, int groups, int n_chk, bool want_delta) {
    const size_t n = (size_t)h->n;
    if (h->alloc_groups < groups) {
        free_state(h);
        CUDA_TRY(h, cudaMalloc((void **)&h->vis, groups * n * sizeof(uint32_t)));
        CUDA_TRY(h, cudaMalloc((void **)&h->sigma, groups * n * 32 * sizeof(double)));
        CUDA_TRY(h, cudaMalloc((void **)&h->coef, groups * n * 32 * sizeof(double)));
        CUDA_TRY(h, cudaMalloc((void **)&h->bcg, groups * n * sizeof(double)));
        CUDA_TRY(h, cudaMemset(h->bcg, 0, groups * n * sizeof(double)));
        h->alloc_groups = groups;
    }
    if (want_delta && h->delta == nullptr)
        CUDA_TRY(h, cudaMalloc((void **)&h->delta, (size_t)h->alloc_groups * n * 32 * sizeof(double)));
    if (h->pacc_chunks < n_chk || (n_chk > 0 && h->pacc == nullptr)) {
        cudaFree(h->pacc), cudaFree(h->pmask);
        h->pacc = nullptr, h->pmask = nullptr;
        const size_t slots = (size_t)h->alloc_groups * n_chk;
        CUDA_TRY(h, cudaMalloc((void **)&h->pacc, slots * 32 * sizeof(double)));
        CUDA_TRY(h, cudaMalloc((void **)&h->pmask, slots * sizeof(uint32_t)));
        h->pacc_chunks = n_chk;
    }
    if (h->counters == nullptr) {
        CUDA_TRY(h, cudaMalloc((void **)&h->counters, 8 * sizeof(unsigned long long)));
    }
    return BC_OK;
}

int ensure_levels(bc_handle *h, int count) {
    const size_t bytes = (size_t)h->alloc_groups * (size_t)h->n * sizeof(uint32_t);
    while ((int)h->lvl.size() < count) {
        uint32_t *p = nullptr;
        CUDA_TRY(h, cudaMalloc((void **)&p, bytes));
        h->lvl.push_back(p);
    }
    if (h->live_cap < count + 1) {
        const int cap = std::max(count + 1, 2 * h->live_cap);
        const size_t G = (size_t)h->alloc_groups;
        uint32_t *p = nullptr;
        CUDA_TRY(h, cudaMalloc((void **)&p, cap * G * sizeof(uint32_t)));
        CUDA_TRY(h, cudaMemset(p, 0, cap * G * sizeof(uint32_t)));
        if (h->live) {
            CUDA_TRY(h, cudaMemcpy(p, h->live, h->live_cap * G * sizeof(uint32_t),
                                   cudaMemcpyDeviceToDevice));
            cudaFree(h->live);
        }
        h->live = p;
        h->live_cap = cap;
    }
    return BC_OK;
}

LevelParams level_params(bc_handle *h, const Csr &c) {
    LevelParams p{};
    p.off = c.off;
    p.col = c.col;
    p.chk_v = c.chk_v;
    p.chk_a0 = c.chk_a0;
    p.chk_a1 = c.chk_a1;
    p.n_chk = c.n_chk;
    p.rng_v0 = c.rng_v0;
    p.rng_nv = c.rng_nv;
    p.n_rng = c.n_rng;
    p.n = c.n;
    p.vis = h->vis;
    p.sigma = h->sigma;
    p.coef = h->coef;
    p.delta = h->delta;
    p.bcg = h->bcg;
    p.pacc = h->pacc;
    p.pmask = h->pmask;
    p.counters = h->counters;
    return p;
}

HubParams hub_params(bc_handle *h, const Csr &c) {
    HubParams p{};
    p.off = c.off;
    p.hub_v = c.hub_v;
    p.hub_c0 = c.hub_c0;
    p.hub_nc = c.hub_nc;
    p.n_hub = c.n_hub;
    p.n_chk = c.n_chk;
    p.n = c.n;
    p.vis = h->vis;
    p.sigma = h->sigma;
    p.coef = h->coef;
    p.delta = h->delta;
    p.bcg = h->bcg;
    p.pacc = h->pacc;
    p.pmask = h->pmask;
    p.counters = h->counters;
    return p;
}

inline unsigned blocks_for(int64_t items) {
    return (unsigned)((items + kWarpsPerBlock - 1) / kWarpsPerBlock);
}

// Forward level L on graph c for `ng` groups.
int launch_forward(bc_handle *h, const Csr &c, int L, int ng, cudaStream_t st) {
    LevelParams p = level_params(h, c);
    p.nbr = h->lvl[L - 1];
    p.cur = h->lvl[L];
    p.live_prev = h->live + (size_t)(L - 1) * h->alloc_groups;
    p.live_cur = h->live + (size_t)L * h->alloc_groups;
    const dim3 grid(blocks_for((int64_t)c.n_chk + c.n_rng), ng);
    level_kernel<false, false><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    ++h->launches;
    if (c.n_hub > 0) {
        HubParams q = hub_params(h, c);
        q.cur = h->lvl[L];
        q.live_prev = p.live_prev;
        q.live_cur = p.live_cur;
        hub_kernel<false, false><<<dim3(blocks_for(c.n_hub), ng), kWarpsPerBlock * 32, 0, st>>>(q);
        ++h->launches;
    }
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

// Backward level L (children at L + 1; `deepest` = no level below).
int launch_backward(bc_handle *h, const Csr &c, int L, bool deepest, int ng, bool store_delta,
                    bool accumulate, cudaStream_t st) {
    LevelParams p = level_params(h, c);
    p.nbr = deepest ? nullptr : h->lvl[L + 1];
    p.cur = h->lvl[L];
    p.live_prev = h->live + (size_t)L * h->alloc_groups;
    p.accumulate_bc = accumulate ? 1 : 0;
    const dim3 grid(blocks_for((int64_t)c.n_chk + c.n_rng), ng);
    if (store_delta)
        level_kernel<true, true><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    else
        level_kernel<true, false><<<grid, kWarpsPerBlock * 32, 0, st>>>(p);
    ++h->launches;
    if (c.n_hub > 0) {
        HubParams q = hub_params(h, c);
        q.cur = h->lvl[L];
        q.live_prev = p.live_prev;
        q.accumulate_bc = p.accumulate_bc;
        const dim3 hg(blocks_for(c.n_hub), ng);
        if (store_delta)
            hub_kernel<true, true><<<hg, kWarpsPerBlock * 32, 0, st>>>(q);
        else
            hub_kernel<true, false><<<hg, kWarpsPerBlock * 32, 0, st>>>(q);
        ++h->launches;
    }
    CUDA_TRY(h, cudaGetLastError());
    return BC_OK;
}

// Forward sweep from the level-0 seeds already in lvl[0]; returns the number
// of non-empty levels.  Levels are launched speculatively in growing chunks
// (a launch past the last level returns at once) so deep graphs do not pay a
// host round trip per level.
int forward_sweep(bc_handle *h, const Csr &c, int ng, cudaStream_t st, int *depth_out) {
    int L = 1, chunk = 4;
    std::vector<uint32_t> flags;
    for (;;) {
        int rc = ensure_levels(h, L + chunk);
        if (rc) return rc;
        for (int j = 0; j < chunk; ++j)
            if ((rc = launch_forward(h, c, L + j, ng, st))) return rc;
        const size_t G = (size_t)h->alloc_groups;
        flags.assign(chunk * G, 0);
        CUDA_TRY(h, cudaMemcpyAsync(flags.data(), h->live + (size_t)L * G,
                                    chunk * G * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        auto level_alive = [&](int j) {
            for (int g = 0; g < ng; ++g)
                if (flags[(size_t)j * G + g]) return true;
            return false;
        };
        int j = 0;
        while (j < chunk && level_alive(j)) ++j;
        if (j < chunk) {
            *depth_out = L + j;
            return BC_OK;
        }
        L += chunk;
        chunk = std::min(chunk * 2, 64);
    }
}

int run_sources(bc_handle *h, const int64_t *sources, int64_t k, double *bc_dev, cudaStream_t st,
                bc_stats *stats, bool debug, int32_t *dist_out, double *sigma_out,
                double *delta_out) {
    const Csr &c = h->full;
    const int64_t n = h->n;
    for (int64_t i = 0; i < k; ++i)
        if (sources[i] < 0 || sources[i] >= n) {
            char buf[128];
            snprintf(buf, sizeof buf, "listed source %lld out of range [0, %lld)",
                     (long long)sources[i], (long long)n);
            return h->fail(BC_ERR_INPUT, buf);
        }
    // Sources without arcs reach nothing: sigma = 1 at the source, delta = 0
    // everywhere.  They stay in the result (and in the counters) but take no
    // lane on the device.  The inspection path keeps them so rows line up.
    std::vector<int64_t> active;
    active.reserve((size_t)k);
    for (int64_t i = 0; i < k; ++i)
        if (debug || h->h_off[sources[i] + 1] > h->h_off[sources[i]]) active.push_back(sources[i]);
    const int64_t k_all = k;
    k = (int64_t)active.size();
    sources = active.data();
    const int groups = debug ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(h->groups, (k + 31) / 32));
    int rc = ensure_state(h, groups, c.n_chk, debug);
    if (rc) return rc;
    if ((rc = ensure_levels(h, 2))) return rc;
    if (h->d_src_cap < k) {
        cudaFree(h->d_src);
        h->d_src = nullptr;
        CUDA_TRY(h, cudaMalloc((void **)&h->d_src, std::max<int64_t>(k, 1) * sizeof(int64_t)));
        h->d_src_cap = k;
    }
    const int64_t launches0 = h->launches;
    int64_t h2d = 0, d2h = 0;
    if (k > 0) {
        CUDA_TRY(h, cudaMemcpyAsync(h->d_src, sources, k * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        h2d += k * sizeof(int64_t);
    }
    CUDA_TRY(h, cudaMemsetAsync(h->counters, 0, 8 * sizeof(unsigned long long), st));

    const int lanes_per_batch = 32 * groups;
    const int64_t n_batches = (k + lanes_per_batch - 1) / lanes_per_batch;
    std::vector<Events> ev((size_t)n_batches);
    int max_depth = 0;

    // debug staging: one batch (<= 32 sources) of [lane][n] rows
    int32_t *dbg_dist = nullptr;
    double *dbg_sigma = nullptr, *dbg_delta = nullptr;
    if (debug) {
        if (dist_out) CUDA_TRY(h, cudaMalloc((void **)&dbg_dist, 32 * (size_t)n * sizeof(int32_t)));
        if (sigma_out) CUDA_TRY(h, cudaMalloc((void **)&dbg_sigma, 32 * (size_t)n * sizeof(double)));
        if (delta_out) CUDA_TRY(h, cudaMalloc((void **)&dbg_delta, 32 * (size_t)n * sizeof(double)));
    }

    for (int64_t b = 0; b < n_batches; ++b) {
        const int cnt = (int)std::min<int64_t>(lanes_per_batch, k - b * lanes_per_batch);
        const int ng = (cnt + 31) / 32;
        Events &e = ev[(size_t)b];
        CUDA_TRY(h, cudaEventCreate(&e.start));
        CUDA_TRY(h, cudaEventCreate(&e.fwd_end));
        CUDA_TRY(h, cudaEventCreate(&e.bwd_end));
        CUDA_TRY(h, cudaEventRecord(e.start, st));

        CUDA_TRY(h, cudaMemsetAsync(h->live, 0,
                                    (size_t)h->live_cap * h->alloc_groups * sizeof(uint32_t), st));
        init_state_kernel<<<dim3(std::min<int64_t>((n + 255) / 256, 1184), ng), 256, 0, st>>>(
            h->vis, h->lvl[0], n, cnt);
        seed_sources_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(h->d_src + b * lanes_per_batch, cnt, n,
                                                                h->vis, h->lvl[0], h->sigma, h->live);
        h->launches += 2;
        CUDA_TRY(h, cudaGetLastError());

        int depth = 1;
        if ((rc = forward_sweep(h, c, ng, st, &depth))) return rc;
        max_depth = std::max(max_depth, depth);
        CUDA_TRY(h, cudaEventRecord(e.fwd_end, st));

        // Level 0 holds only the sources; their delta is excluded from BC
        // (engine.py:147-148), so it is computed only for inspection.
        const int last = debug ? 0 : 1;
        for (int L = depth - 1; L >= last; --L)
            if ((rc = launch_backward(h, c, L, L == depth - 1, ng, debug, !debug, st))) return rc;
        CUDA_TRY(h, cudaEventRecord(e.bwd_end, st));

        if (debug) {
            const size_t rows = (size_t)cnt * (size_t)n;
            const unsigned fb = (unsigned)std::min<size_t>((rows + 255) / 256, 4736);
            if (dbg_dist) fill_i32_kernel<<<fb, 256, 0, st>>>(dbg_dist, rows, BC_UNREACHED);
            if (dbg_sigma) CUDA_TRY(h, cudaMemsetAsync(dbg_sigma, 0, rows * sizeof(double), st));
            if (dbg_delta) CUDA_TRY(h, cudaMemsetAsync(dbg_delta, 0, rows * sizeof(double), st));
            for (int L = 0; L < depth; ++L) {
                extract_level_kernel<<<dim3(std::min<int64_t>((n + 255) / 256, 1184), 1), 256, 0, st>>>(
                    h->lvl[L], h->sigma, h->delta, n, L, dbg_dist, dbg_sigma, dbg_delta);
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
        reduce_bc_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, st>>>(
            bc_dev, h->bcg, n, h->alloc_groups);
        ++h->launches;
        CUDA_TRY(h, cudaGetLastError());
    }
    unsigned long long cnts[8] = {0};
    CUDA_TRY(h, cudaMemcpyAsync(cnts, h->counters, sizeof cnts, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    d2h += sizeof cnts;
    cudaFree(dbg_dist), cudaFree(dbg_sigma), cudaFree(dbg_delta);

    double ms_total = 0, ms_f = 0, ms_b = 0;
    for (Events &e : ev) {
        float a = 0, bms = 0;
        cudaEventElapsedTime(&a, e.start, e.fwd_end);
        cudaEventElapsedTime(&bms, e.fwd_end, e.bwd_end);
        ms_f += a;
        ms_b += bms;
        cudaEventDestroy(e.start), cudaEventDestroy(e.fwd_end), cudaEventDestroy(e.bwd_end);
    }
    if (!ev.empty()) ms_total = ms_f + ms_b;
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->sources = k_all;
        stats->batches = n_batches;
        stats->max_levels = std::max<int64_t>(max_depth, k_all > 0 ? 1 : 0);
        // sources themselves are reached vertices too (level 0)
        stats->reached = (int64_t)cnts[0] + k_all;
        int64_t src_arcs = 0;
        for (int64_t i = 0; i < k; ++i) src_arcs += h->h_off[sources[i] + 1] - h->h_off[sources[i]];
        stats->arcs_reached = (int64_t)cnts[1] + src_arcs;
        stats->dag_arcs = (int64_t)cnts[2];
        stats->launches = h->launches - launches0;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = d2h;
        stats->ms_total = ms_total;
        stats->ms_forward = ms_f;
        stats->ms_backward = ms_b;
    }
    return BC_OK;
}

}  // namespace

extern "C" {

int bc_create(int64_t n, int64_t n_arcs, const int64_t *offsets, const int32_t *col_idx,
              int device, bc_handle **out) {
    if (out == nullptr) return BC_ERR_INPUT;
    *out = nullptr;
    if (n <= 0) {
        g_create_error = "empty graph";
        return BC_ERR_INPUT;
    }
    if (n >= (int64_t)1 << 31 || offsets == nullptr || (n_arcs > 0 && col_idx == nullptr) ||
        offsets[0] != 0 || offsets[n] != n_arcs) {
        g_create_error = "malformed CSR (need int64 offsets[n+1] with offsets[0]=0, offsets[n]=n_arcs, n < 2^31)";
        return BC_ERR_INPUT;
    }
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || device < 0 || device >= count) {
        g_create_error = std::string("no usable CUDA device ") + std::to_string(device) + ": " +
                         (e != cudaSuccess ? cudaGetErrorString(e) : "ordinal out of range") +
                         " (this engine has no CPU fallback)";
        return BC_ERR_INTERNAL;
    }
    bc_handle *h = new bc_handle();
    h->device = device;
    h->n = n;
    h->n_arcs = n_arcs;
    h->h_off.assign(offsets, offsets + n + 1);
    auto bail = [&](int rc) {
        g_create_error = h->err;
        bc_destroy(h);
        return rc;
    };
    if (cudaSetDevice(device) != cudaSuccess) {
        h->err = "cudaSetDevice failed";
        return bail(BC_ERR_INTERNAL);
    }
    Csr &c = h->full;
    c.n = n;
    c.n_arcs = n_arcs;
    c.owns_graph = true;
    auto body = [&]() -> int {
        CUDA_TRY(h, cudaMalloc((void **)&c.off, (n + 1) * sizeof(int64_t)));
        CUDA_TRY(h, cudaMalloc((void **)&c.col, std::max<int64_t>(n_arcs, 1) * sizeof(int32_t)));
        CUDA_TRY(h, cudaMemcpy(c.off, offsets, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
        if (n_arcs > 0)
            CUDA_TRY(h, cudaMemcpy(c.col, col_idx, n_arcs * sizeof(int32_t), cudaMemcpyHostToDevice));
        return build_items(h, c, offsets, h->item_arcs);
    };
    int rc = body();
    if (rc) return bail(rc);
    *out = h;
    return BC_OK;
}

int bc_set_option(bc_handle *h, const char *key, int64_t value) {
    if (h == nullptr || key == nullptr) return BC_ERR_INPUT;
    cudaSetDevice(h->device);
    const std::string k(key);
    if (k == "groups") {
        if (value < 1 || value > 1024) return h->fail(BC_ERR_INPUT, "groups must be in [1, 1024]");
        h->groups = (int)value;
        return BC_OK;
    }
    if (k == "item_arcs") {
        if (value < 32 || value > (1 << 20) || value % 32)
            return h->fail(BC_ERR_INPUT, "item_arcs must be a multiple of 32 in [32, 2^20]");
        if (value != h->item_arcs) {
            h->item_arcs = (int)value;
            Csr &c = h->full;
            cudaFree(c.chk_v), cudaFree(c.chk_a0), cudaFree(c.chk_a1);
            cudaFree(c.rng_v0), cudaFree(c.rng_nv);
            cudaFree(c.hub_v), cudaFree(c.hub_c0), cudaFree(c.hub_nc);
            c.chk_v = c.rng_v0 = c.rng_nv = c.hub_v = c.hub_c0 = c.hub_nc = nullptr;
            c.chk_a0 = c.chk_a1 = nullptr;
            return build_items(h, c, h->h_off.data(), h->item_arcs);
        }
        return BC_OK;
    }
    if (k == "reports") {
        h->reports = value ? 1 : 0;
        return BC_OK;
    }
    return h->fail(BC_ERR_INPUT, "unknown option '" + k + "'");
}

int bc_set_partition(bc_handle *h, int k, const int32_t *assignment) {
    if (h == nullptr) return BC_ERR_INPUT;
    (void)k;
    (void)assignment;
    return h->fail(BC_ERR_INTERNAL, "bc_set_partition: not built yet");
}

int bc_run_device(bc_handle *h, int mode, const int64_t *sources, int64_t n_sources,
                  double *bc_dev, void *stream, bc_stats *stats) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (n_sources < 0 || (n_sources > 0 && sources == nullptr) || bc_dev == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_run_device: null buffer or negative source count");
    if (mode != BC_MODE_DIRECT) return h->fail(BC_ERR_INPUT, "bc_run_device: mode not built yet");
    CUDA_TRY(h, cudaSetDevice(h->device));
    return run_sources(h, sources, n_sources, bc_dev, (cudaStream_t)stream, stats, false, nullptr,
                       nullptr, nullptr);
}

int bc_run(bc_handle *h, int mode, const int64_t *sources, int64_t n_sources, double *bc_out,
           bc_stats *stats) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (bc_out == nullptr) return h->fail(BC_ERR_INPUT, "bc_run: bc_out is null");
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (h->bc_scratch == nullptr)
        CUDA_TRY(h, cudaMalloc((void **)&h->bc_scratch, (size_t)h->n * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->bc_scratch, 0, (size_t)h->n * sizeof(double)));
    int rc = bc_run_device(h, mode, sources, n_sources, h->bc_scratch, nullptr, stats);
    if (rc) return rc;
    CUDA_TRY(h, cudaMemcpy(bc_out, h->bc_scratch, (size_t)h->n * sizeof(double),
                           cudaMemcpyDeviceToHost));
    if (stats) stats->d2h_bytes += h->n * (int64_t)sizeof(double);
    return BC_OK;
}

int bc_debug_sources(bc_handle *h, int mode, const int64_t *sources, int64_t k, int32_t *dist,
                     double *sigma, double *delta) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (k < 0 || (k > 0 && sources == nullptr))
        return h->fail(BC_ERR_INPUT, "bc_debug_sources: null sources");
    if (mode != BC_MODE_DIRECT) return h->fail(BC_ERR_INPUT, "bc_debug_sources: mode not built yet");
    CUDA_TRY(h, cudaSetDevice(h->device));
    return run_sources(h, sources, k, nullptr, nullptr, nullptr, true, dist, sigma, delta);
}

int bc_get_reports(bc_handle *h, int64_t *out, int64_t n_sources) {
    if (h == nullptr) return BC_ERR_INPUT;
    (void)out;
    (void)n_sources;
    return h->fail(BC_ERR_INTERNAL, "bc_get_reports: not built yet");
}

int bc_get_border_counts(bc_handle *h, int64_t *counts) {
    if (h == nullptr) return BC_ERR_INPUT;
    (void)counts;
    return h->fail(BC_ERR_INTERNAL, "bc_get_border_counts: not built yet");
}

int bc_get_border_tables(bc_handle *h, int part, int32_t *borders, int32_t *bm, double *sm) {
    if (h == nullptr) return BC_ERR_INPUT;
    (void)part, (void)borders, (void)bm, (void)sm;
    return h->fail(BC_ERR_INTERNAL, "bc_get_border_tables: not built yet");
}

const char *bc_last_error(bc_handle *h) {
    return h ? h->err.c_str() : g_create_error.c_str();
}

void bc_destroy(bc_handle *h) {
    if (h == nullptr) return;
    cudaSetDevice(h->device);
    free_state(h);
    free_csr(h->full);
    cudaFree(h->live);
    cudaFree(h->counters);
    cudaFree(h->d_src);
    cudaFree(h->bc_scratch);
    delete h;
}

}  // extern "C"
