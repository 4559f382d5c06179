// bc_engine.cu -- host side of the C ABI declared in include/bc_b200.h.
//
// One handle = one CUDA device = one host thread.  The handle owns the CSR on
// the device, the warp work items derived from it, the partition data (cut-free
// CSR, border lists, border tables) and the per-batch state; sources are
// processed in batches of 32 * groups lanes.  There is no CPU code path for
// the arithmetic: every bc_run* call launches the kernels of bc_kernels.cuh /
// bc_border.cuh or fails.
#include "bc_b200.h"
#include "bc_border.cuh"
#include "bc_deep.cuh"
#include "bc_dist.cuh"
#include "bc_kernels.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

using namespace bcb200;

namespace {

thread_local std::string g_create_error;


// ------------------------------------------------------------------------------------
// Device memory arena.  cudaMalloc / cudaFree of the multi-GB batch state cost
// 15-20 ms per run_bc() call (and cudaFree drains the device); blocks released by
// a handle are kept per device and handed to the next handle that asks for a
// similar size.  bc_release_cached_memory() returns them to the driver, and an
// allocation that fails flushes the cache before it gives up.
// ------------------------------------------------------------------------------------
struct Arena {
    std::mutex mu;
    std::unordered_map<void *, std::pair<int, size_t>> live;   // ptr -> (device, bytes)
    std::multimap<size_t, void *> spare[64];                   // per device, by size
    size_t spare_bytes = 0;

    static size_t round_up(size_t b) {
        const size_t g = b < (1u << 20) ? 512 : (size_t)2 << 20;   // driver granularity for big blocks
        return (std::max<size_t>(b, 1) + g - 1) / g * g;
    }
    void flush_locked(int dev) {
        for (auto &kv : spare[dev]) {
            cudaFree(kv.second);
            spare_bytes -= kv.first;
        }
        spare[dev].clear();
    }
    cudaError_t alloc(void **out, size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        dev &= 63;
        const size_t want = round_up(bytes);
        std::lock_guard<std::mutex> lock(mu);
        auto it = spare[dev].lower_bound(want);
        if (it != spare[dev].end() && it->first <= want + want / 4 + (1u << 16)) {
            *out = it->second;
            live[*out] = {dev, it->first};
            spare_bytes -= it->first;
            spare[dev].erase(it);
            return cudaSuccess;
        }
        cudaError_t e = cudaMalloc(out, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            flush_locked(dev);
            e = cudaMalloc(out, want);
        }
        if (e == cudaSuccess) live[*out] = {dev, want};
        return e;
    }
    void release(void *p) {
        if (p == nullptr) return;
        std::lock_guard<std::mutex> lock(mu);
        auto it = live.find(p);
        if (it == live.end()) {  // not ours
            cudaFree(p);
            return;
        }
        spare[it->second.first].emplace(it->second.second, p);
        spare_bytes += it->second.second;
        live.erase(it);
    }
    void flush_all() {
        std::lock_guard<std::mutex> lock(mu);
        int cur = 0;
        cudaGetDevice(&cur);
        for (int d = 0; d < 64; ++d)
            if (!spare[d].empty()) {
                cudaSetDevice(d);
                flush_locked(d);
            }
        cudaSetDevice(cur);
    }
};
Arena &arena() {
    static Arena *a = new Arena();  // leaked on purpose: the driver may be gone at exit
    return *a;
}
inline cudaError_t arena_malloc(void **out, size_t bytes) { return arena().alloc(out, bytes); }
template <typename T>
inline void arena_free(T *p) { arena().release((void *)p); }

// BC_B200_TRACE=1: host wall clock per stage on stderr (the device is drained at
// every mark, so traced runs are for attribution only, never for a bench number).
struct Trace {
    bool on;
    std::chrono::steady_clock::time_point t;
    Trace() : on(getenv("BC_B200_TRACE") != nullptr), t(std::chrono::steady_clock::now()) {}
    void mark(const char *what) {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[bc_b200] %-28s %8.2f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// Device-side CSR plus the work items of the level kernels.
struct Csr {
    int64_t n = 0, n_arcs = 0;
    int64_t *off = nullptr;
    int32_t *col = nullptr;
    int32_t *wgt = nullptr;   // arc weights (nullptr: unit weights)
    int n_chk = 0, n_rng = 0, n_hub = 0;
    int64_t heavy_slices = 0;   // kHeavySlice-arc slices over all vertices above kHeavyDeg arcs
    int64_t max_deg = 0;        // largest degree (build_items)
    int32_t *chk_v = nullptr;
    int64_t *chk_a0 = nullptr, *chk_a1 = nullptr;
    int32_t *rng_v0 = nullptr, *rng_nv = nullptr;
    int32_t *hub_v = nullptr, *hub_c0 = nullptr, *hub_nc = nullptr;
};

// Events of one batch; destroyed with the vector that holds them, on every exit path.
struct Events {
    cudaEvent_t start = nullptr, fwd_end = nullptr, border_end = nullptr, fwd2_end = nullptr, bwd_end = nullptr;
    Events() = default;
    Events(const Events &) = delete;
    Events &operator=(const Events &) = delete;
    ~Events() {
        for (cudaEvent_t e : {start, fwd_end, border_end, fwd2_end, bwd_end})
            if (e) cudaEventDestroy(e);
    }
};

// Arena block released when the scope ends (error exits included).
template <typename T>
struct ScopedBlock {
    T *p = nullptr;
    ScopedBlock() = default;
    ScopedBlock(const ScopedBlock &) = delete;
    ScopedBlock &operator=(const ScopedBlock &) = delete;
    ~ScopedBlock() { arena_free(p); }
};

constexpr unsigned long long kQueueMaxDegree = 8192;
constexpr unsigned long long kThinDegree = 8;  // average degree up to which a level runs thread-per-entry
constexpr int kDeepLevels = 1024;              // levels one persistent launch may produce

// Border-table feasibility: b_p^2 entries of 12 B per part.
constexpr double kMaxTableBytes = 64e9;

}  // namespace

struct bc_handle {
    int device = 0;
    int64_t n = 0, n_arcs = 0;
    std::vector<int64_t> h_off;   // host copy of the offsets (item building, partition set-up)
    std::vector<int32_t> h_col;   // host copy of col_idx, fetched from the device when a partition is set
    Csr full;
    std::vector<int32_t> h_wgt;   // host copy of the arc weights (empty: unit weights)
    int wmax = 1;                 // largest arc weight
    int cur_depth = 0;        // levels of the batch being swept backward (weighted kernels)
    // options
    int groups = 4;
    int item_arcs = 1024;
    int reports = 1;
    int sparse = 1;        // allow queue levels + top-down push (direction-optimising switch)
    int reorder = 1;       // group sources by the size of their 2-hop neighbourhood
    int row_cache = -1;    // sigma / coef row gathers: 1 = allocate in L1, 0 = bypass L1, -1 = by degree skew
    uint32_t row_bypass_mask = 0;  // dev: bit L = forward level L bypasses L1, bit 16 + L = backward level L
    int push_beta_late = 24;   // same, once a pull level has run: a late pull scans unvisited vertices only
    int push_beta = 4;     // push when frontier arcs * beta <= arcs of the graph
    int deep = 1;          // run consecutive thin levels inside one cooperative launch (bc_deep.cuh)
    int deep_blocks_per_sm = 0;   // 0 = what the occupancy calculator allows
    int deep_grid_f = 0, deep_grid_b = 0;
    unsigned long long *deep_log = nullptr;
    int *deep_info = nullptr;
    // ---- partition ------------------------------------------------------
    int k = 1;
    std::vector<int32_t> h_part;
    int32_t *d_part = nullptr;
    Csr intra;                     // cut arcs removed
    std::vector<int64_t> h_ioff;   // host copy of its offsets (queue sweeps inside the parts)
    int64_t intra_maxdeg = 0;      // largest degree inside a part
    int32_t *d_border_index = nullptr;   // [n] border number of a vertex, -1 for inner vertices
    int hybir_queues = 1;          // partitioned sweeps of low-degree graphs on frontier queues
    // Step-6 seeds sorted by level (queue sweeps)
    int32_t *seed_keys = nullptr, *seed_keys2 = nullptr, *seed_vals = nullptr, *seed_vals2 = nullptr;
    int64_t *seed_off = nullptr;
    int64_t seed_off_cap = 0;
    void *seed_tmp = nullptr;
    size_t seed_tmp_bytes = 0;
    int B = 0;                     // borders over all parts
    int64_t n_cut = 0;
    std::vector<int32_t> h_border_v, h_border_p, h_part_off;
    std::vector<int64_t> h_tab_off;
    int64_t tab_total = 0;
    int32_t *d_border_v = nullptr, *d_border_p = nullptr, *d_part_off = nullptr, *d_cin_src = nullptr;
    int32_t *d_cin_w = nullptr;   // weight of each incoming cut arc
    int64_t *d_tab_off = nullptr, *d_cin_off = nullptr;
    int32_t *bm = nullptr;         // border distance tables
    double *sm = nullptr;          // border path-count tables
    bool tables_ready = false;
    // per-batch border state, [B][S]
    int border_S = 0;
    int32_t *D = nullptr, *D2 = nullptr, *seedD = nullptr, *Dfin = nullptr;
    double *seedS = nullptr, *sig = nullptr, *arr = nullptr, *darr = nullptr;
    int32_t *lane_part = nullptr, *lane_iters = nullptr;
    // look-ahead (engine.py:135-143): Step 1 of the next batch runs on a second stream while the
    // border phase of the current one is in flight and leaves its border seeds here
    int lookahead = 0;
    int32_t *seedD_alt = nullptr, *lane_part_alt = nullptr;
    double *seedS_alt = nullptr;
    cudaStream_t side_stream = nullptr;
    cudaEvent_t side_go = nullptr, side_done = nullptr;
    std::vector<bool> table_set;   // parts whose border table was installed by bc_set_border_tables
    uint32_t *lane_active = nullptr, *lane_entered = nullptr, *lane_changed = nullptr;
    uint32_t *dflags = nullptr;    // [0] any lane active, [1] sigma changed
    int *d_maxlvl = nullptr;
    uint32_t *sync_flag = nullptr, *sync_bits = nullptr;
    int64_t *lane_sync = nullptr, *lane_bytes = nullptr;
    size_t sync_bits_words = 0;
    const uint32_t **d_lvl_ptrs = nullptr;
    int lvl_ptrs_cap = 0;
    uint32_t *presence = nullptr;
    size_t presence_words = 0;
    std::vector<int64_t> reports_host;  // 8 per source of the last run
    // ---- per-batch BFS state ------------------------------------------------
    int alloc_groups = 0;
    uint32_t *vis = nullptr;
    std::vector<uint32_t *> lvl;
    double *sigma = nullptr, *coef = nullptr, *delta = nullptr;
    uint8_t *cand = nullptr;    // [alloc_groups][n] candidate flags of the dense forward sweeps (deep graphs)
    bool use_cand = false;      // set by forward_sweep for the launches of its levels
    bool sigma_clean = false;   // sigma is all zero (kept so by the backward sweeps of adaptive batches)
    bool lazy_clear = false;    // this batch's backward sweep clears sigma behind itself
    int last_depth = 0;         // levels of the previous batch (deep graphs: memset instead)
    double *bcg = nullptr;
    bool bcg_dirty = true;      // partial sums of an unfinished (failed) run are in there: clear first
    double *pacc = nullptr;
    uint32_t *pmask = nullptr;
    int pacc_chunks = 0;
    uint32_t *live = nullptr;  // [level][alloc_groups] lanes with a non-empty frontier
    int live_cap = 0;          // levels
    // sparse levels: per-group frontier queues + two all-zero scratch mask arrays
    int32_t *q_v = nullptr;
    uint32_t *q_m = nullptr;
    int64_t q_cap = 0;
    unsigned long long *q_count = nullptr;
    int64_t *d_qbeg = nullptr, *d_qend = nullptr, *d_qlbeg = nullptr;
    uint32_t *scrA = nullptr, *scrB = nullptr;
    unsigned long long *lstat = nullptr;
    HeavyRec *heavy = nullptr;      // slices of the heavy entries of the current frontier level
    int64_t heavy_cap = 0;
    unsigned long long *report = nullptr;   // per-level report read by the host (forward_adaptive)
    int64_t *range_table = nullptr;        // queue ranges of every level (backward_adaptive)
    int64_t range_table_cap = 0;
    unsigned long long *counters = nullptr;
    int cnt_off = 0;  // 0: traversal counters of the result; 4: scratch (Step 1 of hybir mode)
    int64_t *d_src = nullptr;
    int64_t d_src_cap = 0;
    double *bc_scratch = nullptr;  // device bc vector of bc_run
    // ---- graph-partitioned multi-GPU mode (one rank = one part)
    int dist_rank = -1, dist_world = 0, dist_ng = 0, dist_cnt = 0;
    bool dist_hybir = false;      // border-matrix forward phase across ranks (bc_dist_hybir_*)
    int dist_depth = 0;           // levels of the batch in flight (local, then global)
    std::vector<int64_t> dist_border_off;
    int32_t *dist_border_v = nullptr;   // all ranks' borders, rank-major
    int32_t *dist_counts = nullptr, *dist_offsets = nullptr;
    void *dist_scan_tmp = nullptr;
    size_t dist_scan_bytes = 0;
    int64_t dist_entries_cap = 0;
    // backward exchange plan of the batch in flight (bc_dist_plan_backward)
    int64_t *dist_cut_off = nullptr;    // [own borders + 1] cut arcs of this rank's borders
    int32_t *dist_cut_dst = nullptr;    // their far ends (local vertex ids of the halo)
    int32_t *plan_idx = nullptr, *plan_voff = nullptr, *plan_eoff = nullptr, *plan_cnt_e = nullptr, *plan_cnt_v = nullptr;
    uint32_t *plan_mask = nullptr;
    int64_t plan_cap = 0;
    int plan_levels_cap = 0, plan_depth = 0;
    std::vector<int32_t> plan_eoff_h, plan_cnt_e_h, plan_cnt_v_h;
    std::string err;
    std::atomic<int64_t> launches{0};   // (the look-ahead thread launches too)
    int64_t level_launches = 0;   // dense level kernel only
    // batched byte model of the dense level-kernel launches of the current call
    int64_t model_scan = 0, model_pairs = 0, model_vlanes = 0, model_dense_words = 0, model_entries = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> level_events;   // around those launches (<= 512 per call)

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

#define TRY(expr)                 \
    do {                          \
        int rc_ = (expr);         \
        if (rc_) return rc_;      \
    } while (0)

namespace {

template <typename T>
int upload(bc_handle *h, T **dst, const std::vector<T> &src) {
    arena_free(*dst);
    *dst = nullptr;
    if (src.empty()) return BC_OK;
    CUDA_TRY(h, arena_malloc((void **)dst, src.size() * sizeof(T)));
    CUDA_TRY(h, cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    return BC_OK;
}

template <typename T>
int dev_alloc(bc_handle *h, T **dst, size_t count) {
    arena_free(*dst);
    *dst = nullptr;
    CUDA_TRY(h, arena_malloc((void **)dst, std::max<size_t>(count, 1) * sizeof(T)));
    return BC_OK;
}

void free_items(Csr &c) {
    arena_free(c.chk_v), arena_free(c.chk_a0), arena_free(c.chk_a1);
    arena_free(c.rng_v0), arena_free(c.rng_nv);
    arena_free(c.hub_v), arena_free(c.hub_c0), arena_free(c.hub_nc);
    c.chk_v = c.rng_v0 = c.rng_nv = c.hub_v = c.hub_c0 = c.hub_nc = nullptr;
    c.chk_a0 = c.chk_a1 = nullptr;
    c.n_chk = c.n_rng = c.n_hub = 0;
}

void free_csr(Csr &c) {
    arena_free(c.off);
    arena_free(c.col);
    arena_free(c.wgt);
    free_items(c);
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
    int64_t heavy_slices = 0, max_deg = 0;
    for (int64_t v = 0; v < c.n; ++v) {
        const int64_t deg = off[v + 1] - off[v];
        max_deg = std::max(max_deg, deg);
        if (deg > kHeavyDeg) heavy_slices += (deg + kHeavySlice - 1) / kHeavySlice;
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
    free_items(c);
    c.n_chk = (int)chk_v.size();
    c.n_rng = (int)rng_v0.size();
    c.n_hub = (int)hub_v.size();
    c.heavy_slices = heavy_slices;
    c.max_deg = max_deg;
    TRY(upload(h, &c.chk_v, chk_v));
    TRY(upload(h, &c.chk_a0, chk_a0));
    TRY(upload(h, &c.chk_a1, chk_a1));
    TRY(upload(h, &c.rng_v0, rng_v0));
    TRY(upload(h, &c.rng_nv, rng_nv));
    TRY(upload(h, &c.hub_v, hub_v));
    TRY(upload(h, &c.hub_c0, hub_c0));
    TRY(upload(h, &c.hub_nc, hub_nc));
    return BC_OK;
}

void free_state(bc_handle *h) {
    arena_free(h->vis);
    for (uint32_t *p : h->lvl) arena_free(p);
    h->lvl.clear();
    arena_free(h->sigma), arena_free(h->coef), arena_free(h->delta), arena_free(h->bcg);
    arena_free(h->pacc), arena_free(h->pmask);
    arena_free(h->live);
    h->live = nullptr;
    h->live_cap = 0;
    arena_free(h->q_v), arena_free(h->q_m), arena_free(h->q_count);
    arena_free(h->d_qbeg), arena_free(h->d_qend), arena_free(h->d_qlbeg);
    arena_free(h->scrA), arena_free(h->scrB), arena_free(h->lstat), arena_free(h->report);
    arena_free(h->range_table);
    arena_free(h->deep_log), arena_free(h->deep_info);
    arena_free(h->heavy);
    arena_free(h->cand);
    h->cand = nullptr;
    h->heavy = nullptr;
    h->heavy_cap = 0;
    h->deep_log = nullptr;
    h->deep_info = nullptr;
    h->report = nullptr;
    h->range_table = nullptr;
    h->range_table_cap = 0;
    h->q_v = nullptr;
    h->q_m = h->scrA = h->scrB = nullptr;
    h->q_count = h->lstat = nullptr;
    h->d_qbeg = h->d_qend = h->d_qlbeg = nullptr;
    h->q_cap = 0;
    h->vis = nullptr;
    h->sigma = h->coef = h->delta = h->bcg = h->pacc = nullptr;
    h->pmask = nullptr;
    h->alloc_groups = 0;
    h->pacc_chunks = 0;
}

void free_border_state(bc_handle *h) {
    arena_free(h->D), arena_free(h->D2), arena_free(h->seedD), arena_free(h->Dfin);
    arena_free(h->seedS), arena_free(h->sig), arena_free(h->arr), arena_free(h->darr);
    arena_free(h->seedD_alt), arena_free(h->seedS_alt), arena_free(h->lane_part_alt);
    h->seedD_alt = h->lane_part_alt = nullptr;
    h->seedS_alt = nullptr;
    h->darr = nullptr;
    arena_free(h->seed_keys), arena_free(h->seed_keys2), arena_free(h->seed_vals), arena_free(h->seed_vals2);
    arena_free(h->seed_off), arena_free(h->seed_tmp);
    h->seed_keys = h->seed_keys2 = h->seed_vals = h->seed_vals2 = nullptr;
    h->seed_off = nullptr, h->seed_tmp = nullptr;
    h->seed_off_cap = 0, h->seed_tmp_bytes = 0;
    arena_free(h->lane_part), arena_free(h->lane_iters), arena_free(h->lane_active);
    arena_free(h->lane_entered), arena_free(h->lane_changed);
    arena_free(h->sync_flag), arena_free(h->sync_bits), arena_free(h->lane_sync), arena_free(h->lane_bytes);
    h->D = h->D2 = h->seedD = h->Dfin = h->lane_part = h->lane_iters = nullptr;
    h->seedS = h->sig = h->arr = nullptr;
    h->lane_active = h->lane_entered = h->lane_changed = h->sync_flag = h->sync_bits = nullptr;
    h->lane_sync = h->lane_bytes = nullptr;
    h->border_S = 0;
    h->sync_bits_words = 0;
}

void free_partition(bc_handle *h) {
    free_csr(h->intra);
    free_border_state(h);
    arena_free(h->d_part), arena_free(h->d_border_v), arena_free(h->d_border_p), arena_free(h->d_part_off);
    arena_free(h->d_cin_src), arena_free(h->d_tab_off), arena_free(h->d_cin_off), arena_free(h->d_cin_w);
    h->d_cin_w = nullptr;
    arena_free(h->bm), arena_free(h->sm);
    arena_free(h->d_border_index);
    h->d_border_index = nullptr;
    h->h_ioff.clear();
    h->intra_maxdeg = 0;
    h->d_part = h->d_border_v = h->d_border_p = h->d_part_off = h->d_cin_src = nullptr;
    h->d_tab_off = h->d_cin_off = nullptr;
    h->bm = nullptr;
    h->sm = nullptr;
    h->tables_ready = false;
    h->table_set.clear();
    h->k = 1;
    h->B = 0;
    h->n_cut = 0;
}

int ensure_state(bc_handle *h, int groups, bool want_delta) {
    const size_t n = (size_t)h->n;
    const int n_chk = std::max(h->full.n_chk, h->intra.n_chk);
    if (h->alloc_groups < groups) {
        free_state(h);
        CUDA_TRY(h, arena_malloc((void **)&h->vis, groups * n * sizeof(uint32_t)));
        CUDA_TRY(h, arena_malloc((void **)&h->sigma, groups * n * 32 * sizeof(double)));
        CUDA_TRY(h, arena_malloc((void **)&h->coef, groups * n * 32 * sizeof(double)));
        CUDA_TRY(h, arena_malloc((void **)&h->bcg, groups * n * sizeof(double)));
        h->bcg_dirty = true;   // cleared on the caller's stream by the run that uses it
        h->alloc_groups = groups;
        h->sigma_clean = false;
    }
    if (want_delta && h->delta == nullptr)
        CUDA_TRY(h, arena_malloc((void **)&h->delta, (size_t)h->alloc_groups * n * 32 * sizeof(double)));
    if (h->pacc_chunks < n_chk || (n_chk > 0 && h->pacc == nullptr)) {
        arena_free(h->pacc), arena_free(h->pmask);
        h->pacc = nullptr, h->pmask = nullptr;
        const size_t slots = (size_t)h->alloc_groups * n_chk;
        CUDA_TRY(h, arena_malloc((void **)&h->pacc, slots * 32 * sizeof(double)));
        CUDA_TRY(h, arena_malloc((void **)&h->pmask, slots * sizeof(uint32_t)));
        h->pacc_chunks = n_chk;
    }
    if (h->counters == nullptr)
        CUDA_TRY(h, arena_malloc((void **)&h->counters, 8 * sizeof(unsigned long long)));
    if (h->dflags == nullptr) CUDA_TRY(h, arena_malloc((void **)&h->dflags, 4 * sizeof(uint32_t)));
    if (h->d_maxlvl == nullptr) CUDA_TRY(h, arena_malloc((void **)&h->d_maxlvl, sizeof(int)));
    return BC_OK;
}

int ensure_pool(bc_handle *h, int count) {
    const size_t bytes = (size_t)h->alloc_groups * (size_t)h->n * sizeof(uint32_t);
    while ((int)h->lvl.size() < count) {
        uint32_t *p = nullptr;
        CUDA_TRY(h, arena_malloc((void **)&p, bytes));
        h->lvl.push_back(p);
    }
    return BC_OK;
}

int ensure_live(bc_handle *h, int count) {
    if (h->live_cap < count + 1) {
        const int cap = std::max(count + 1, 2 * h->live_cap);
        const size_t G = (size_t)h->alloc_groups;
        uint32_t *p = nullptr;
        CUDA_TRY(h, arena_malloc((void **)&p, cap * G * sizeof(uint32_t)));
        CUDA_TRY(h, cudaMemset(p, 0, cap * G * sizeof(uint32_t)));
        if (h->live) {
            CUDA_TRY(h, cudaMemcpy(p, h->live, h->live_cap * G * sizeof(uint32_t),
                                   cudaMemcpyDeviceToDevice));
            arena_free(h->live);
        }
        h->live = p;
        h->live_cap = cap;
    }
    return BC_OK;
}

int ensure_levels(bc_handle *h, int count) {
    TRY(ensure_pool(h, count));
    return ensure_live(h, count);
}

int ensure_queues(bc_handle *h) {
    if (h->q_v != nullptr) return BC_OK;
    const size_t G = (size_t)h->alloc_groups, n = (size_t)h->n;
    h->q_cap = (int64_t)(4 * n + 1024);
    TRY(dev_alloc(h, &h->q_v, G * (size_t)h->q_cap));
    TRY(dev_alloc(h, &h->q_m, G * (size_t)h->q_cap));
    TRY(dev_alloc(h, &h->q_count, G));
    CUDA_TRY(h, cudaMemset(h->q_count, 0, G * sizeof(unsigned long long)));
    TRY(dev_alloc(h, &h->d_qbeg, G));
    TRY(dev_alloc(h, &h->d_qend, G));
    TRY(dev_alloc(h, &h->d_qlbeg, G));
    CUDA_TRY(h, cudaMemset(h->d_qbeg, 0, G * sizeof(int64_t)));
    CUDA_TRY(h, cudaMemset(h->d_qend, 0, G * sizeof(int64_t)));
    CUDA_TRY(h, cudaMemset(h->d_qlbeg, 0, G * sizeof(int64_t)));
    TRY(dev_alloc(h, &h->scrA, G * n));
    TRY(dev_alloc(h, &h->scrB, G * n));
    TRY(dev_alloc(h, &h->lstat, (size_t)8));
    TRY(dev_alloc(h, &h->report, 8 + 2 * G));
    h->heavy_cap = (int64_t)G * std::max(h->full.heavy_slices, h->intra.heavy_slices) + 1;
    TRY(dev_alloc(h, &h->heavy, (size_t)h->heavy_cap));
    CUDA_TRY(h, cudaMemset(h->scrA, 0, G * n * sizeof(uint32_t)));
    CUDA_TRY(h, cudaMemset(h->scrB, 0, G * n * sizeof(uint32_t)));
    return BC_OK;
}

// Buffers and grid size of the persistent sweeps (bc_deep.cuh).  The grid must be
// fully resident for the grid-wide barrier, so it comes from the occupancy
// calculator (the backward kernel is the heavier of the two).
int ensure_deep(bc_handle *h) {
    if (h->deep_log != nullptr) return BC_OK;
    const size_t G = (size_t)h->alloc_groups;
    TRY(dev_alloc(h, &h->deep_log, (size_t)kDeepLevels * (3 + 2 * G)));
    TRY(dev_alloc(h, &h->deep_info, (size_t)4));
    int per_sm_f = 0, per_sm_b = 0, per_sm_d = 0, sms = 0;
    CUDA_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_f, deep_forward_kernel, kDeepThreads, 0));
    CUDA_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, deep_backward_kernel<false>,
                                                              kDeepThreads, 0));
    CUDA_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_d, deep_backward_kernel<true>,
                                                              kDeepThreads, 0));
    CUDA_TRY(h, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    per_sm_b = std::min(per_sm_b, per_sm_d);
    if (h->deep_blocks_per_sm > 0) {
        per_sm_f = std::min(per_sm_f, h->deep_blocks_per_sm);
        per_sm_b = std::min(per_sm_b, h->deep_blocks_per_sm);
    }
    if (per_sm_f < 1 || per_sm_b < 1 || sms < 1)
        return h->fail(BC_ERR_INTERNAL, "persistent sweep kernels do not fit on an SM");
    h->deep_grid_f = per_sm_f * sms;
    h->deep_grid_b = per_sm_b * sms;
    return BC_OK;
}

// Queue entries are (vertex, level) pairs: a vertex can sit in up to 32 levels of
// a group (one per lane), so deep graphs outgrow the initial 4n entries.  Grow
// by doubling up to 33n.
int grow_queues(bc_handle *h, int64_t need_cap, cudaStream_t st,
                const std::vector<unsigned long long> &used) {
    const int64_t max_cap = 33 * h->n + 1024 + h->B;
    if (h->q_cap >= max_cap || need_cap <= h->q_cap) return BC_OK;
    const int64_t cap = std::min(max_cap, std::max(need_cap, 2 * h->q_cap));
    const size_t G = (size_t)h->alloc_groups;
    int32_t *nv = nullptr;
    uint32_t *nm = nullptr;
    CUDA_TRY(h, cudaStreamSynchronize(st));
    CUDA_TRY(h, arena_malloc((void **)&nv, G * (size_t)cap * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&nm, G * (size_t)cap * sizeof(uint32_t)));
    for (size_t g = 0; g < G; ++g) {
        const size_t keep = (size_t)std::min<int64_t>(g < used.size() ? (int64_t)used[g] : 0, h->q_cap);   // entries in use
        if (keep == 0) continue;
        CUDA_TRY(h, cudaMemcpy(nv + g * cap, h->q_v + g * h->q_cap, keep * sizeof(int32_t),
                               cudaMemcpyDeviceToDevice));
        CUDA_TRY(h, cudaMemcpy(nm + g * cap, h->q_m + g * h->q_cap, keep * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice));
    }
    arena_free(h->q_v), arena_free(h->q_m);
    h->q_v = nv;
    h->q_m = nm;
    h->q_cap = cap;
    return BC_OK;
}

// Device table of the level-mask pointers (the border gathers walk levels).
int upload_level_ptrs(bc_handle *h, int depth, cudaStream_t st) {
    if (h->lvl_ptrs_cap < depth) {
        arena_free((void *)h->d_lvl_ptrs);
        h->d_lvl_ptrs = nullptr;
        const int cap = std::max(depth, 2 * h->lvl_ptrs_cap);
        CUDA_TRY(h, arena_malloc((void **)&h->d_lvl_ptrs, cap * sizeof(uint32_t *)));
        h->lvl_ptrs_cap = cap;
    }
    CUDA_TRY(h, cudaMemcpyAsync((void *)h->d_lvl_ptrs, h->lvl.data(), depth * sizeof(uint32_t *),
                                cudaMemcpyHostToDevice, st));
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
    p.counters = h->counters + h->cnt_off;
    p.wgt = c.wgt;
    p.cand = nullptr;
    p.lvl_ptrs = h->d_lvl_ptrs;
    p.live_base = h->live;
    p.wmax = c.wgt ? h->wmax : 1;
    p.G = h->alloc_groups;
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
    p.counters = h->counters + h->cnt_off;
    p.live_base = h->live;
    p.wmax = c.wgt ? h->wmax : 1;
    p.G = h->alloc_groups;
    return p;
}

BorderGeom border_geom(bc_handle *h) {
    BorderGeom g{};
    g.k = h->k;
    g.B = h->B;
    g.border_v = h->d_border_v;
    g.border_p = h->d_border_p;
    g.part_off = h->d_part_off;
    g.tab_off = h->d_tab_off;
    g.cin_off = h->d_cin_off;
    g.cin_src = h->d_cin_src;
    g.cin_w = h->d_cin_w;
    return g;
}

inline unsigned blocks_for(int64_t items) {
    return (unsigned)((items + kWarpsPerBlock - 1) / kWarpsPerBlock);
}

inline unsigned grid1d(size_t count, int block = 256, size_t cap = 1u << 30) {
    return (unsigned)std::max<size_t>(1, std::min<size_t>((count + block - 1) / block, cap));
}

#ifdef BC_PROFILE
void prof_dump(const char *what, int L, cudaStream_t st) {
    unsigned long long v[16];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(v, g_prof, sizeof v);
    fprintf(stderr, "[prof] %s L=%d slices=%llu any=%llu hit_arcs=%llu want_lanes=%llu pairs=%llu hit_lanes=%llu\n",
            what, L, v[0], v[1], v[2], v[3], v[4], v[5]);
    memset(v, 0, sizeof v);
    cudaMemcpyToSymbol(g_prof, v, sizeof v);
}
#else
inline void prof_dump(const char *, int, cudaStream_t) {}
#endif

void drop_level_events(bc_handle *h) {
    for (auto &pr : h->level_events) cudaEventDestroy(pr.first), cudaEventDestroy(pr.second);
    h->level_events.clear();
}

// CUDA events around one dense level launch (level kernel + hub pass): bc_stats.ms_level.
struct LevelTimer {
    bc_handle *h;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    LevelTimer(bc_handle *h_, cudaStream_t st_) : h(h_), st(st_) {
        if (h->level_events.size() >= 512) return;
        if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) {
            a = b = nullptr;
            return;
        }
        cudaEventRecord(a, st);
    }
    void stop() {
        if (a == nullptr) return;
        cudaEventRecord(b, st);
        h->level_events.emplace_back(a, b);
        a = b = nullptr;
    }
    ~LevelTimer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

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
    if (zero_sigma && !(h->sigma_clean && h->lazy_clear))
        CUDA_TRY(h, cudaMemsetAsync(h->sigma, 0, (size_t)h->alloc_groups * n * 32 * sizeof(double), st));
    h->sigma_clean = false;
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
            if (thin && h->deep && ng <= kDeepMaxGroups && prev.maxdeg <= (unsigned long long)kHeavyDeg) {
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
        if (r.slot >= 0) {
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
                geo, first, cnt, h->bm, h->sm);
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
    const Csr &fwd_csr = hybir ? h->intra : h->full;
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
                    h->sigma, h->border_S, seedD, seedS);
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
            if (adaptive) TRY(forward_adaptive(h, fwd_csr, ng, cnt, batch_src, st, &depth, reps));
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
                helper = std::thread([&, b]() {
                    cudaSetDevice(h->device);
                    ahead.rc = step1(b + 1, h->side_stream, h->seedD_alt, h->seedS_alt, h->lane_part_alt, ahead);
                    if (ahead.rc == BC_OK && cudaEventRecord(h->side_done, h->side_stream) != cudaSuccess)
                        ahead.rc = BC_ERR_INTERNAL;
                });
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
        if (queued) TRY(backward_adaptive(h, h->full, depth, reps, ng, debug, st));
        else TRY(backward_sweep(h, h->full, depth, ng, debug, st));
        h->last_depth = depth;
        if (queued && !debug && h->lazy_clear) {
            // the sweep cleared every pair it visited; the sources (level 0) are left
            clear_source_sigma_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(h->d_src + b * lanes_per_batch, cnt, n,
                                                                        h->sigma);
            ++h->launches;
            h->sigma_clean = true;
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
        reduce_bc_kernel<<<grid1d((size_t)n, 256, 1184), 256, 0, st>>>(bc_dev, h->bcg, n, h->alloc_groups);
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
    const int64_t level_timed = (int64_t)h->level_events.size();
    for (auto &pr : h->level_events) {
        float t = 0;
        if (cudaEventElapsedTime(&t, pr.first, pr.second) == cudaSuccess) ms_level += t;
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
        for (int64_t i = 0; i < k; ++i) src_arcs += h->h_off[sources[i] + 1] - h->h_off[sources[i]];
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
        stats->level_model_bytes = 8 * h->model_scan + 8 * h->model_pairs + 8 * h->model_vlanes +
                                   4 * h->model_dense_words + 16 * h->model_entries +
                                   8 * h->n * stats->launches_level;
    }
    return BC_OK;
}


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

int check_mode(bc_handle *h, int mode) {
    if (mode != BC_MODE_DIRECT && mode != BC_MODE_HYBIR && mode != BC_MODE_BSP)
        return h->fail(BC_ERR_INPUT, "unknown mode (use BC_MODE_DIRECT, BC_MODE_HYBIR or BC_MODE_BSP)");
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
    Trace tr;
    bc_handle *h = new bc_handle();
    h->device = device;
    h->n = n;
    h->n_arcs = n_arcs;
    h->last_depth = n_arcs < 6 * n ? 1 << 20 : 0;   // low average degree: expect a deep graph (see begin_batch)
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
    auto body = [&]() -> int {
        CUDA_TRY(h, arena_malloc((void **)&c.off, (n + 1) * sizeof(int64_t)));
        CUDA_TRY(h, arena_malloc((void **)&c.col, std::max<int64_t>(n_arcs, 1) * sizeof(int32_t)));
        // the CSR copy is queued first (it runs at PCIe speed from pinned memory) and the
        // host builds its offsets copy and the work items while it is in flight
        CUDA_TRY(h, cudaMemcpyAsync(c.off, offsets, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, 0));
        if (n_arcs > 0)
            CUDA_TRY(h, cudaMemcpyAsync(c.col, col_idx, n_arcs * sizeof(int32_t), cudaMemcpyHostToDevice, 0));
        h->h_off.assign(offsets, offsets + n + 1);
        for (int64_t v = 0; v < n; ++v)
            if (offsets[v + 1] < offsets[v])
                return h->fail(BC_ERR_INPUT, "malformed CSR: offsets decrease at vertex " + std::to_string(v));
        TRY(build_items(h, c, offsets, h->item_arcs));
        // neighbour ids are checked on the device, behind the upload (a bad id would be an
        // out-of-bounds read in every kernel)
        if (n_arcs > 0) {
            ScopedBlock<int> d_bad;
            CUDA_TRY(h, arena_malloc((void **)&d_bad.p, sizeof(int)));
            CUDA_TRY(h, cudaMemsetAsync(d_bad.p, 0, sizeof(int), 0));
            validate_col_kernel<<<grid1d((size_t)n_arcs, 256, 2368), 256>>>(c.col, n_arcs, n, d_bad.p);
            int bad = 0;
            CUDA_TRY(h, cudaMemcpy(&bad, d_bad.p, sizeof bad, cudaMemcpyDeviceToHost));
            if (bad) return h->fail(BC_ERR_INPUT, "malformed CSR: col_idx holds a vertex id outside [0, n)");
        }
        tr.mark("create: CSR upload + work items");
        return BC_OK;
    };
    int rc = body();
    if (rc) return bail(rc);
    *out = h;
    return BC_OK;
}

int bc_set_weights(bc_handle *h, const int32_t *weights) {
    if (h == nullptr) return BC_ERR_INPUT;
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (h->k > 1)
        return h->fail(BC_ERR_INPUT, "bc_set_weights: set the weights before bc_set_partition");
    arena_free(h->full.wgt);
    h->full.wgt = nullptr;
    h->h_wgt.clear();
    h->wmax = 1;
    if (weights == nullptr) return BC_OK;   // back to unit weights
    int64_t wmax = 1;
    for (int64_t a = 0; a < h->n_arcs; ++a) {
        if (weights[a] <= 0) return h->fail(BC_ERR_INPUT, "arc weights must be positive integers");
        wmax = std::max<int64_t>(wmax, weights[a]);
    }
    if (wmax > 4096)
        return h->fail(BC_ERR_INPUT, "arc weights above 4096 are not supported (one level per distance value)");
    if (wmax == 1) return BC_OK;
    CUDA_TRY(h, arena_malloc((void **)&h->full.wgt, std::max<int64_t>(h->n_arcs, 1) * sizeof(int32_t)));
    CUDA_TRY(h, cudaMemcpy(h->full.wgt, weights, h->n_arcs * sizeof(int32_t), cudaMemcpyHostToDevice));
    h->h_wgt.assign(weights, weights + h->n_arcs);
    h->wmax = (int)wmax;
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
            TRY(build_items(h, h->full, h->h_off.data(), h->item_arcs));
            if (h->k > 1) {
                std::vector<int64_t> ioff((size_t)h->n + 1);
                CUDA_TRY(h, cudaMemcpy(ioff.data(), h->intra.off, (h->n + 1) * sizeof(int64_t),
                                       cudaMemcpyDeviceToHost));
                TRY(build_items(h, h->intra, ioff.data(), h->item_arcs));
            }
        }
        return BC_OK;
    }
    if (k == "reports") {
        h->reports = value ? 1 : 0;
        return BC_OK;
    }
    if (k == "sparse") {
        h->sparse = value ? 1 : 0;
        return BC_OK;
    }
    if (k == "reorder") {
        h->reorder = value ? 1 : 0;
        return BC_OK;
    }
    if (k == "row_bypass_mask") {
        h->row_bypass_mask = (uint32_t)value;
        return BC_OK;
    }
    if (k == "row_cache") {
        if (value < -1 || value > 1) return h->fail(BC_ERR_INPUT, "row_cache must be -1 (auto), 0 or 1");
        h->row_cache = (int)value;
        return BC_OK;
    }
    if (k == "deep") {
        h->deep = value ? 1 : 0;
        return BC_OK;
    }
    if (k == "hybir_queues") {
        h->hybir_queues = value ? 1 : 0;
        return BC_OK;
    }
    if (k == "deep_blocks_per_sm") {
        if (value < 0 || value > 32) return h->fail(BC_ERR_INPUT, "deep_blocks_per_sm must be in [0, 32]");
        h->deep_blocks_per_sm = (int)value;
        arena_free(h->deep_log), arena_free(h->deep_info);
        h->deep_log = nullptr;
        h->deep_info = nullptr;
        return BC_OK;
    }
    if (k == "lookahead") {
        h->lookahead = value ? 1 : 0;
        return BC_OK;
    }
    if (k == "l2_fetch") {
        // granularity of L2 fills from HBM (32 / 64 / 128 B; the driver default is 64): random
        // 8-byte accesses of the deep-graph sweeps use a quarter of a 32-byte sector as it is
        if (value != 32 && value != 64 && value != 128)
            return h->fail(BC_ERR_INPUT, "l2_fetch must be 32, 64 or 128");
        CUDA_TRY(h, cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)value));
        return BC_OK;
    }
    if (k == "push_beta_late") {
        if (value < 1) return h->fail(BC_ERR_INPUT, "push_beta_late must be >= 1");
        h->push_beta_late = (int)value;
        return BC_OK;
    }
    if (k == "push_beta") {
        if (value < 1) return h->fail(BC_ERR_INPUT, "push_beta must be >= 1");
        h->push_beta = (int)value;
        return BC_OK;
    }
    return h->fail(BC_ERR_INPUT, "unknown option '" + k + "'");
}

}  // extern "C"

namespace {

// Border geometry supplied by the caller (graph-partitioned multi-GPU runs: a rank holds the CSR
// rows of its own part only, so the borders and cut arcs of the other parts cannot be derived
// from its rows).  Borders are listed part by part, ascending vertex id inside a part.
struct ExternalBorders {
    const int64_t *border_off;   // [k + 1]
    const int32_t *border_v;     // [B]
    const int64_t *cin_off;      // [B + 1] incoming cut arcs per border
    const int32_t *cin_src;      // [n_cut] border index of the arc's source
    const int32_t *cin_w;        // [n_cut] weights, nullptr = all one
};

int install_partition(bc_handle *h, int k, const int32_t *assignment, const ExternalBorders *ext) {
    const int64_t n = h->n;
    for (int64_t v = 0; v < n; ++v)
        if (assignment[v] < 0 || assignment[v] >= k)
            return h->fail(BC_ERR_INPUT, "bc_set_partition: part id outside [0, k)");
    CUDA_TRY(h, cudaSetDevice(h->device));
    std::vector<int32_t> part(assignment, assignment + n);   // `assignment` may alias h->h_part
    free_partition(h);
    h->k = k;
    h->h_part.swap(part);
    assignment = h->h_part.data();
    if (k == 1 && ext == nullptr) return BC_OK;   // (a one-rank partitioned run keeps the empty border set-up)
    if ((int64_t)h->h_col.size() != h->n_arcs) {
        h->h_col.resize((size_t)h->n_arcs);
        if (h->n_arcs > 0)
            CUDA_TRY(h, cudaMemcpy(h->h_col.data(), h->full.col, h->n_arcs * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost));
    }
    const int64_t *off = h->h_off.data();
    const int32_t *col = h->h_col.data();
    // cut-free CSR + border lists (ascending vertex id inside each part)
    std::vector<int64_t> ioff((size_t)n + 1, 0);
    std::vector<int32_t> icol, iwgt;
    icol.reserve((size_t)h->n_arcs);
    const bool weighted = !h->h_wgt.empty();
    if (weighted) iwgt.reserve((size_t)h->n_arcs);
    std::vector<std::vector<int32_t>> borders((size_t)k);
    for (int64_t v = 0; v < n; ++v) {
        bool is_border = false;
        for (int64_t a = off[v]; a < off[v + 1]; ++a) {
            if (assignment[col[a]] == assignment[v]) {
                icol.push_back(col[a]);
                if (weighted) iwgt.push_back(h->h_wgt[(size_t)a]);
            } else is_border = true;
        }
        ioff[(size_t)v + 1] = (int64_t)icol.size();
        if (is_border && ext == nullptr) borders[(size_t)assignment[v]].push_back((int32_t)v);
    }
    if (ext != nullptr)
        for (int p = 0; p < k; ++p)
            borders[(size_t)p].assign(ext->border_v + ext->border_off[p], ext->border_v + ext->border_off[p + 1]);
    h->h_part_off.assign((size_t)k + 1, 0);
    h->h_tab_off.assign((size_t)k, 0);
    h->h_border_v.clear();
    h->h_border_p.clear();
    int64_t tab = 0;
    for (int p = 0; p < k; ++p) {
        h->h_part_off[(size_t)p] = (int32_t)h->h_border_v.size();
        h->h_tab_off[(size_t)p] = tab;
        const int64_t b = (int64_t)borders[(size_t)p].size();
        tab += b * b;
        for (int32_t v : borders[(size_t)p]) {
            if (v < 0 || v >= n || assignment[v] != p)
                return h->fail(BC_ERR_INPUT, "border list names a vertex outside its part");
            h->h_border_v.push_back(v);
            h->h_border_p.push_back(p);
        }
    }
    h->h_part_off[(size_t)k] = (int32_t)h->h_border_v.size();
    h->B = (int)h->h_border_v.size();
    h->tab_total = tab;
    // incoming cut arcs of every border, in arc order (the graph is symmetric)
    std::vector<int64_t> cin_off((size_t)h->B + 1, 0);
    std::vector<int32_t> cin_src, cin_w;
    if (ext != nullptr) {
        cin_off.assign(ext->cin_off, ext->cin_off + h->B + 1);
        const int64_t nc = cin_off[(size_t)h->B];
        cin_src.assign(ext->cin_src, ext->cin_src + nc);
        if (ext->cin_w) cin_w.assign(ext->cin_w, ext->cin_w + nc);
        else cin_w.assign((size_t)nc, 1);
        for (int64_t c = 0; c < nc; ++c)
            if (cin_src[(size_t)c] < 0 || cin_src[(size_t)c] >= h->B)
                return h->fail(BC_ERR_INPUT, "cut arc list names a border outside [0, B)");
    } else {
        std::vector<int32_t> index_of((size_t)n, -1);
        for (int j = 0; j < h->B; ++j) index_of[(size_t)h->h_border_v[(size_t)j]] = j;
        for (int j = 0; j < h->B; ++j) {
            const int64_t v = h->h_border_v[(size_t)j];
            for (int64_t a = off[v]; a < off[v + 1]; ++a)
                if (assignment[col[a]] != assignment[v]) {
                    cin_src.push_back(index_of[(size_t)col[a]]);
                    cin_w.push_back(weighted ? h->h_wgt[(size_t)a] : 1);   // symmetric graph: w(u->v) = w(v->u)
                }
            cin_off[(size_t)j + 1] = (int64_t)cin_src.size();
        }
    }
    h->n_cut = (int64_t)cin_src.size();
    Csr &c = h->intra;
    c.n = n;
    c.n_arcs = (int64_t)icol.size();
    TRY(upload(h, &c.off, ioff));
    if (icol.empty()) icol.push_back(0);
    TRY(upload(h, &c.col, icol));
    if (weighted) {
        if (iwgt.empty()) iwgt.push_back(1);
        TRY(upload(h, &c.wgt, iwgt));
    }
    TRY(build_items(h, c, ioff.data(), h->item_arcs));
    h->intra_maxdeg = 0;
    for (int64_t v = 0; v < n; ++v)
        h->intra_maxdeg = std::max(h->intra_maxdeg, ioff[(size_t)v + 1] - ioff[(size_t)v]);
    h->h_ioff.swap(ioff);
    {
        std::vector<int32_t> index_of((size_t)n, -1);
        for (int j = 0; j < h->B; ++j) index_of[(size_t)h->h_border_v[(size_t)j]] = j;
        TRY(upload(h, &h->d_border_index, index_of));
    }
    TRY(upload(h, &h->d_part, h->h_part));
    TRY(upload(h, &h->d_border_v, h->h_border_v));
    TRY(upload(h, &h->d_border_p, h->h_border_p));
    TRY(upload(h, &h->d_part_off, h->h_part_off));
    TRY(upload(h, &h->d_tab_off, h->h_tab_off));
    TRY(upload(h, &h->d_cin_off, cin_off));
    if (cin_src.empty()) cin_src.push_back(0), cin_w.push_back(1);
    TRY(upload(h, &h->d_cin_src, cin_src));
    TRY(upload(h, &h->d_cin_w, cin_w));
    return BC_OK;
}

}  // namespace

extern "C" {

int bc_set_partition(bc_handle *h, int k, const int32_t *assignment) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (k < 1 || assignment == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_set_partition: need k >= 1 and an assignment");
    h->dist_hybir = false;
    return install_partition(h, k, assignment, nullptr);
}

int bc_run_device(bc_handle *h, int mode, const int64_t *sources, int64_t n_sources,
                  double *bc_dev, void *stream, bc_stats *stats) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (n_sources < 0 || (n_sources > 0 && sources == nullptr) || bc_dev == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_run_device: null buffer or negative source count");
    TRY(check_mode(h, mode));
    CUDA_TRY(h, cudaSetDevice(h->device));
    return run_sources(h, mode, sources, n_sources, bc_dev, (cudaStream_t)stream, stats, false,
                       nullptr, nullptr, nullptr);
}

int bc_run(bc_handle *h, int mode, const int64_t *sources, int64_t n_sources, double *bc_out,
           bc_stats *stats) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (bc_out == nullptr) return h->fail(BC_ERR_INPUT, "bc_run: bc_out is null");
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (h->bc_scratch == nullptr)
        CUDA_TRY(h, arena_malloc((void **)&h->bc_scratch, (size_t)h->n * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->bc_scratch, 0, (size_t)h->n * sizeof(double)));
    TRY(bc_run_device(h, mode, sources, n_sources, h->bc_scratch, nullptr, stats));
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
    TRY(check_mode(h, mode));
    CUDA_TRY(h, cudaSetDevice(h->device));
    return run_sources(h, mode, sources, k, nullptr, nullptr, nullptr, true, dist, sigma, delta);
}

int bc_get_reports(bc_handle *h, int64_t *out, int64_t n_sources) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (out == nullptr || n_sources * 8 != (int64_t)h->reports_host.size())
        return h->fail(BC_ERR_INPUT, "bc_get_reports: source count differs from the last run");
    memcpy(out, h->reports_host.data(), h->reports_host.size() * sizeof(int64_t));
    return BC_OK;
}

int bc_get_border_counts(bc_handle *h, int64_t *counts) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (counts == nullptr) return h->fail(BC_ERR_INPUT, "bc_get_border_counts: null output");
    if (h->k == 1) {
        counts[0] = 0;
        return BC_OK;
    }
    for (int p = 0; p < h->k; ++p) counts[p] = h->h_part_off[(size_t)p + 1] - h->h_part_off[(size_t)p];
    return BC_OK;
}

int bc_get_border_tables(bc_handle *h, int part, int32_t *borders, int32_t *bm, double *sm) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (h->k < 2 || part < 0 || part >= h->k)
        return h->fail(BC_ERR_INPUT, "bc_get_border_tables: no such part");
    CUDA_TRY(h, cudaSetDevice(h->device));
    TRY(build_border_tables(h));
    const int64_t b = h->h_part_off[(size_t)part + 1] - h->h_part_off[(size_t)part];
    if (borders)
        memcpy(borders, h->h_border_v.data() + h->h_part_off[(size_t)part], b * sizeof(int32_t));
    if (b == 0) return BC_OK;
    if (bm) {
        CUDA_TRY(h, cudaMemcpy(bm, h->bm + h->h_tab_off[(size_t)part], b * b * sizeof(int32_t),
                               cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < b * b; ++i)
            if (bm[i] >= kInf) bm[i] = BC_UNREACHED;
    }
    if (sm)
        CUDA_TRY(h, cudaMemcpy(sm, h->sm + h->h_tab_off[(size_t)part], b * b * sizeof(double),
                               cudaMemcpyDeviceToHost));
    return BC_OK;
}

int bc_set_border_tables(bc_handle *h, int part, const int32_t *bm, const double *sm) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (h->k < 2 || part < 0 || part >= h->k || bm == nullptr || sm == nullptr)
        return h->fail(BC_ERR_INPUT, "bc_set_border_tables: no such part / null table");
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (h->bm == nullptr) {
        TRY(dev_alloc(h, &h->bm, (size_t)h->tab_total));
        TRY(dev_alloc(h, &h->sm, (size_t)h->tab_total));
        h->table_set.assign((size_t)h->k, false);
    }
    if ((int)h->table_set.size() != h->k) h->table_set.assign((size_t)h->k, false);
    const int64_t b = h->h_part_off[(size_t)part + 1] - h->h_part_off[(size_t)part];
    if (b > 0) {
        std::vector<int32_t> d(bm, bm + b * b);
        for (int32_t &x : d)
            if (x < 0) x = kInf;   // BC_UNREACHED
        CUDA_TRY(h, cudaMemcpy(h->bm + h->h_tab_off[(size_t)part], d.data(), (size_t)(b * b) * sizeof(int32_t),
                               cudaMemcpyHostToDevice));
        CUDA_TRY(h, cudaMemcpy(h->sm + h->h_tab_off[(size_t)part], sm, (size_t)(b * b) * sizeof(double),
                               cudaMemcpyHostToDevice));
    }
    h->table_set[(size_t)part] = true;
    bool all = true;
    for (bool x : h->table_set) all = all && x;
    h->tables_ready = all;
    return BC_OK;
}

int bc_get_border_frontier(bc_handle *h, int64_t n_lanes, int32_t *dist, double *sigma,
                           double *arrival) {
    if (h == nullptr) return BC_ERR_INPUT;
    if (h->k < 2 || h->D == nullptr || n_lanes < 0 || n_lanes > h->border_S)
        return h->fail(BC_ERR_INPUT, "bc_get_border_frontier: no hybir batch of that width has run");
    CUDA_TRY(h, cudaSetDevice(h->device));
    const size_t cnt = (size_t)h->B * h->border_S;
    std::vector<int32_t> d(cnt);
    std::vector<double> s(cnt), a(cnt);
    if (cnt) {
        CUDA_TRY(h, cudaMemcpy(d.data(), h->D, cnt * sizeof(int32_t), cudaMemcpyDeviceToHost));
        CUDA_TRY(h, cudaMemcpy(s.data(), h->sig, cnt * sizeof(double), cudaMemcpyDeviceToHost));
        CUDA_TRY(h, cudaMemcpy(a.data(), h->arr, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    }
    for (int j = 0; j < h->B; ++j)
        for (int64_t l = 0; l < n_lanes; ++l) {
            const size_t from = (size_t)j * h->border_S + l, to = (size_t)j * n_lanes + l;
            if (dist) dist[to] = d[from] >= kInf ? BC_UNREACHED : d[from];
            if (sigma) sigma[to] = s[from];
            if (arrival) arrival[to] = a[from];
        }
    return BC_OK;
}


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

void bc_release_cached_memory(void) { arena().flush_all(); }

const char *bc_last_error(bc_handle *h) {
    return h ? h->err.c_str() : g_create_error.c_str();
}

void bc_destroy(bc_handle *h) {
    if (h == nullptr) return;
    cudaSetDevice(h->device);
    drop_level_events(h);
    free_state(h);
    free_partition(h);
    free_csr(h->full);
    arena_free(h->counters);
    arena_free(h->dflags);
    arena_free(h->d_maxlvl);
    arena_free(h->d_src);
    arena_free(h->bc_scratch);
    arena_free((void *)h->d_lvl_ptrs);
    arena_free(h->presence);
    arena_free(h->dist_border_v), arena_free(h->dist_counts), arena_free(h->dist_offsets);
    arena_free(h->dist_scan_tmp);
    arena_free(h->dist_cut_off), arena_free(h->dist_cut_dst);
    arena_free(h->plan_idx), arena_free(h->plan_mask), arena_free(h->plan_voff);
    arena_free(h->plan_eoff), arena_free(h->plan_cnt_e), arena_free(h->plan_cnt_v);
    if (h->side_stream) cudaStreamDestroy(h->side_stream);
    if (h->side_go) cudaEventDestroy(h->side_go);
    if (h->side_done) cudaEventDestroy(h->side_done);
    delete h;
}

}  // extern "C"
