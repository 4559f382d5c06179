// engine_state.cuh -- device memory arena, the handle (bc_handle) and its state: CSR + work items, per-batch
// BFS state, frontier queues, border state; allocation / release helpers and the kernel-parameter builders.
// Part of the single translation unit bc_engine.cu (included from there, in this order: engine_state,
// engine_sweeps, engine_border, engine_run, engine_dist).
#pragma once
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
    std::unordered_map<void *, size_t> zeroed;                 // spare block -> leading bytes known to be zero
    size_t spare_bytes = 0;

    static size_t round_up(size_t b) {
        const size_t g = b < (1u << 20) ? 512 : (size_t)2 << 20;   // driver granularity for big blocks
        return (std::max<size_t>(b, 1) + g - 1) / g * g;
    }
    void flush_locked(int dev) {
        for (auto &kv : spare[dev]) {
            cudaFree(kv.second);
            zeroed.erase(kv.second);
            spare_bytes -= kv.first;
        }
        spare[dev].clear();
    }
    // *zero_prefix (optional) = leading bytes of the block its last owner left zeroed (release())
    cudaError_t alloc(void **out, size_t bytes, size_t *zero_prefix = nullptr) {
        if (zero_prefix) *zero_prefix = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        dev &= 63;
        const size_t want = round_up(bytes);
        std::lock_guard<std::mutex> lock(mu);
        auto it = spare[dev].lower_bound(want);
        if (it != spare[dev].end() && it->first <= want + want / 4 + (1u << 16)) {
            *out = it->second;
            auto z = zeroed.find(*out);
            if (z != zeroed.end()) {
                if (zero_prefix) *zero_prefix = z->second;
                zeroed.erase(z);
            }
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
    void release(void *p, size_t zero_prefix = 0) {
        if (p == nullptr) return;
        std::lock_guard<std::mutex> lock(mu);
        auto it = live.find(p);
        if (it == live.end()) {  // not ours
            cudaFree(p);
            return;
        }
        if (zero_prefix) zeroed[p] = std::min(zero_prefix, it->second.second);
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
    // the same graph with vertices renumbered by descending degree (bc_relabel.cuh): built on the
    // first unpartitioned unit-weight run of a skewed graph
    Csr relab;
    bool relab_ready = false;
    int relabel = -1;                     // option "relabel": 1 = always, 0 = never, -1 = skewed graphs, once there is enough work
    int64_t sources_seen = 0;             // sources of the unpartitioned runs so far
    int32_t *d_old_of_new = nullptr;      // device: caller's id of renumbered vertex v
    int32_t *d_new_of_old = nullptr;      // device: renumbered id of the caller's vertex (sources on the way in)
    std::vector<int64_t> h_off_relab;     // host copy of its offsets
    std::vector<int32_t> h_wgt;   // host copy of the arc weights (empty: unit weights)
    int wmax = 1;                 // largest arc weight
    int wgt_mode = -1;            // option "sssp": 1 = general-weight sweeps (bc_sssp.cuh), 0 = one level per distance value, -1 = by weight range
    // general-weight sweeps: rows [G][n][32] of distances and tight-arc counts, frontier masks [G][n]
    long long *sp_dist = nullptr;
    int *sp_npar = nullptr, *sp_nchild = nullptr;
    uint32_t *sp_maskA = nullptr, *sp_maskB = nullptr, *sp_leaf = nullptr;
    int *sp_flags = nullptr;
    long long *sp_bound = nullptr;   // per round: distance bound, smallest waiting distance (phase A)
    int32_t *sp_queue = nullptr;     // three frontier queues [G][n]: this round, next round, leaves
    int *sp_qcount = nullptr;        // their lengths: [3][G] rotating + [G] leaves
    int sp_blocks = 0;               // dev option "sssp_blocks": blocks per group of a round (0 = default)
    long long sp_delta = 0;          // option "sssp_delta": step of the bound (0 = 16 mean arc weights)
    long long wsum = 0;              // sum of the arc weights
    int sp_groups = 0;
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
    // backward: children drive a level when their arcs * bwd_push <= the parents' arcs (0: never).
    // 16 = the far tail only: at 4 the level behind the peak of R-MAT scale 20 switches too and
    // loses (7.3 against 5.0 ms: 155 M scattered fp64 atomics run at 37 G/s)
    int bwd_push = 16;
    int bwd_push_levels = 0;   // levels of the last run that took that path
    int deep = 1;          // run consecutive thin levels inside one cooperative launch (bc_deep.cuh)
    int deep_blocks_per_sm = 0;   // 0 = what the occupancy calculator allows
    int deep_grid_f = 0, deep_grid_b = 0, deep_grid_c = 0, deep_grid_fc = 0;
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
    // child-driven backward levels (bc_bwd_push.cuh): children above kBwdPushHeavyDegree arcs are
    // listed per group and walked by the whole grid
    uint4 *bp_list = nullptr;   // [alloc_groups][bp_cap] (vertex, lane mask, slice of its arcs)
    unsigned *bp_count = nullptr;   // [alloc_groups] heavy records
    uint32_t *bp_recv = nullptr;    // [alloc_groups][n] lanes of each parent that were handed a sum; zero between levels
    int64_t bp_cap = -1;        // slices of all vertices of the graph above that degree (-1: not counted yet)
    uint8_t *cand = nullptr;    // [alloc_groups][n] candidate flags of the dense forward sweeps (deep graphs)
    bool use_cand = false;      // set by forward_sweep for the launches of its levels
    int sigma_clean_groups = 0; // leading groups of sigma that are all zero (kept so by the backward sweeps of adaptive batches)
    int sigma_clean_after = 0;  // its value once the running batch has cleared what it touched
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
    // level-ordered values of the deep sweeps (bc_deep.cuh: DeepFwdParams::qs, deep_backward_compact_kernel)
    int deep_compact = 1;          // option: backward sweeps of deep graphs run on them
    double *qs = nullptr;          // [G][q_vcap] path counts in queue-entry order
    uint32_t *q_off = nullptr;     // [G][q_cap] first value slot of an entry
    unsigned long long *v_count = nullptr;   // [G]
    int64_t q_vcap = 0;
    double *bc_acc = nullptr;      // [n] BC partial of a batch, added with atomics
    VertexState *vs = nullptr;     // [G][n] visited / next-level / queue-entry words of the compact sweeps
    uint32_t *q_arc = nullptr;     // [G][q_cap] degree << 24 | arcs of a frontier entry that reached a fresh lane
    uint32_t *q_a = nullptr;       // [G][q_cap] first arc of the entry's vertex
    int4 *q_nb = nullptr;          // [G][q_cap] neighbour ids of entries whose vertex has at most four arcs (optional)
    const int64_t *q_a_csr = nullptr;   // ... in the CSR with these offsets (the last compact forward sweep's)
    bool fwd_compact_allowed = false;   // set by the caller of a sweep: nobody reads sigma rows afterwards
    bool sigma_stale = false;      // the sigma rows were not cleared for this batch (compact sweep expected)
    const int64_t *batch_src_dev = nullptr;   // sources of the batch in flight (begin_batch)
    int batch_cnt = 0;
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
    bool dist_sharded = false;    // ... with the own part's border table only (bc_dist_hybir_shard_tables)
    int dist_round = 0;           // composition round of the batch in flight (sharded tables)
    int dist_depth = 0;           // levels of the batch in flight (local, then global)
    std::vector<int64_t> dist_border_off;
    int32_t *dist_border_v = nullptr;   // all ranks' borders, rank-major
    int32_t *dist_counts = nullptr, *dist_offsets = nullptr;
    void *dist_scan_tmp = nullptr;
    size_t dist_scan_bytes = 0;
    int64_t dist_entries_cap = 0;
    // backward exchange plan of the batch in flight (bc_dist_plan_backward)
    int64_t *dist_border_off_dev = nullptr;   // device copy of dist_border_off (bc_dist_unpack_all)
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
    int model_counters = 0;   // option: count the arcs the forward pulls scan (level_model_bytes is complete)
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

// state of the general-weight sweeps (engine_sssp.cuh)
void free_sssp_state(bc_handle *h) {
    arena_free(h->sp_dist), arena_free(h->sp_npar), arena_free(h->sp_nchild);
    arena_free(h->sp_maskA), arena_free(h->sp_maskB), arena_free(h->sp_leaf), arena_free(h->sp_flags);
    arena_free(h->sp_bound), arena_free(h->sp_queue), arena_free(h->sp_qcount);
    h->sp_bound = nullptr;
    h->sp_queue = nullptr;
    h->sp_qcount = nullptr;
    h->sp_dist = nullptr;
    h->sp_npar = h->sp_nchild = nullptr;
    h->sp_maskA = h->sp_maskB = h->sp_leaf = nullptr;
    h->sp_flags = nullptr;
    h->sp_groups = 0;
}

void free_state(bc_handle *h) {
    free_sssp_state(h);
    arena_free(h->vis);
    for (uint32_t *p : h->lvl) arena_free(p);
    h->lvl.clear();
    // the path-count rows a finished run left zeroed (begin_batch) stay tagged in the arena: the
    // next handle that gets the block skips that part of its first memset
    arena().release((void *)h->sigma, (size_t)h->sigma_clean_groups * (size_t)h->n * 32 * sizeof(double));
    h->sigma_clean_groups = 0;
    arena_free(h->coef), arena_free(h->delta), arena_free(h->bcg);
    arena_free(h->pacc), arena_free(h->pmask);
    arena_free(h->live);
    h->live = nullptr;
    h->live_cap = 0;
    arena_free(h->q_v), arena_free(h->q_m), arena_free(h->q_count);
    arena_free(h->qs), arena_free(h->q_off), arena_free(h->v_count), arena_free(h->bc_acc);
    arena_free(h->vs), arena_free(h->q_arc), arena_free(h->q_a);
    h->vs = nullptr, h->q_arc = nullptr, h->q_a = nullptr;
    arena_free(h->q_nb);
    h->q_nb = nullptr;
    h->qs = nullptr, h->q_off = nullptr, h->v_count = nullptr, h->bc_acc = nullptr;
    h->q_vcap = 0;
    arena_free(h->d_qbeg), arena_free(h->d_qend), arena_free(h->d_qlbeg);
    arena_free(h->scrA), arena_free(h->scrB), arena_free(h->lstat), arena_free(h->report);
    arena_free(h->range_table);
    arena_free(h->deep_log), arena_free(h->deep_info);
    arena_free(h->heavy);
    arena_free(h->cand);
    h->cand = nullptr;
    arena_free(h->bp_list), arena_free(h->bp_count), arena_free(h->bp_recv);
    h->bp_list = nullptr, h->bp_count = nullptr, h->bp_recv = nullptr;
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
    const int n_chk = std::max(std::max(h->full.n_chk, h->intra.n_chk), h->relab.n_chk);
    if (h->alloc_groups < groups) {
        free_state(h);
        CUDA_TRY(h, arena_malloc((void **)&h->vis, groups * n * sizeof(uint32_t)));
        size_t zero_prefix = 0;
        CUDA_TRY(h, arena().alloc((void **)&h->sigma, groups * n * 32 * sizeof(double), &zero_prefix));
        CUDA_TRY(h, arena_malloc((void **)&h->coef, groups * n * 32 * sizeof(double)));
        CUDA_TRY(h, arena_malloc((void **)&h->bcg, groups * n * sizeof(double)));
        h->bcg_dirty = true;   // cleared on the caller's stream by the run that uses it
        h->alloc_groups = groups;
        h->sigma_clean_groups = (int)std::min<size_t>(groups, zero_prefix / (n * 32 * sizeof(double)));
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
    CUDA_TRY(h, cudaMemset(h->report, 0, (8 + 2 * G) * sizeof(unsigned long long)));
    CUDA_TRY(h, cudaMemset(h->lstat, 0, 8 * sizeof(unsigned long long)));
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
    int per_sm_c = 0;
    CUDA_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_c, deep_backward_compact_kernel,
                                                              kDeepThreads, 0));
    if (h->deep_blocks_per_sm > 0) per_sm_c = std::min(per_sm_c, h->deep_blocks_per_sm);
    h->deep_grid_c = std::max(per_sm_c, 0) * sms;
    int per_sm_fc = 0;
    CUDA_TRY(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_fc, deep_forward_compact_kernel,
                                                              kDeepThreads, 0));
    if (h->deep_blocks_per_sm > 0) per_sm_fc = std::min(per_sm_fc, h->deep_blocks_per_sm);
    h->deep_grid_fc = std::max(per_sm_fc, 0) * sms;
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

// Level-ordered value arrays of the deep sweeps.  Fails softly: without the memory the sweeps
// keep the row layout (returns false).
bool ensure_deep_compact(bc_handle *h) {
    if (!h->deep_compact || h->q_v == nullptr) return false;
    if (h->qs != nullptr) return true;
    const size_t G = (size_t)h->alloc_groups;
    const int64_t vcap = 32 * h->n;
    if (vcap >= ((int64_t)1 << 32) || h->n_arcs >= ((int64_t)1 << 32)) return false;   // 32-bit value / arc offsets
    if (arena_malloc((void **)&h->qs, G * (size_t)vcap * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        h->qs = nullptr;
        h->deep_compact = 0;
        return false;
    }
    if (arena_malloc((void **)&h->q_off, G * (size_t)h->q_cap * sizeof(uint32_t)) != cudaSuccess ||
        arena_malloc((void **)&h->q_arc, G * (size_t)h->q_cap * sizeof(uint32_t)) != cudaSuccess ||
        arena_malloc((void **)&h->q_a, G * (size_t)h->q_cap * sizeof(uint32_t)) != cudaSuccess ||
        arena_malloc((void **)&h->vs, G * (size_t)h->n * sizeof(VertexState)) != cudaSuccess ||
        arena_malloc((void **)&h->v_count, G * sizeof(unsigned long long)) != cudaSuccess ||
        arena_malloc((void **)&h->bc_acc, (size_t)h->n * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        arena_free(h->qs), arena_free(h->q_off), arena_free(h->v_count), arena_free(h->bc_acc);
        arena_free(h->vs), arena_free(h->q_arc), arena_free(h->q_a);
        h->qs = nullptr, h->q_off = nullptr, h->v_count = nullptr, h->bc_acc = nullptr;
        h->vs = nullptr, h->q_arc = nullptr, h->q_a = nullptr;
        h->deep_compact = 0;
        return false;
    }
    cudaMemset(h->v_count, 0, G * sizeof(unsigned long long));
    cudaMemset(h->bc_acc, 0, (size_t)h->n * sizeof(double));
    // (entries of the last level never become a frontier: their arc words are copied, unwritten,
    // when the queues grow)
    cudaMemset(h->q_off, 0, G * (size_t)h->q_cap * sizeof(uint32_t));
    cudaMemset(h->q_arc, 0, G * (size_t)h->q_cap * sizeof(uint32_t));
    cudaMemset(h->q_a, 0, G * (size_t)h->q_cap * sizeof(uint32_t));
    // optional: without it the sweeps read col_idx
    if (arena_malloc((void **)&h->q_nb, G * (size_t)h->q_cap * sizeof(int4)) != cudaSuccess) {
        cudaGetLastError();
        h->q_nb = nullptr;
    } else {
        cudaMemset(h->q_nb, 0, G * (size_t)h->q_cap * sizeof(int4));
    }
    h->q_vcap = vcap;
    return true;
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
    for (uint32_t **arr : {&h->q_off, &h->q_arc, &h->q_a}) {
        if (*arr == nullptr) continue;
        uint32_t *no = nullptr;
        CUDA_TRY(h, arena_malloc((void **)&no, G * (size_t)cap * sizeof(uint32_t)));
        CUDA_TRY(h, cudaMemset(no, 0, G * (size_t)cap * sizeof(uint32_t)));
        for (size_t g = 0; g < G; ++g) {
            const size_t keep = (size_t)std::min<int64_t>(g < used.size() ? (int64_t)used[g] : 0, h->q_cap);
            if (keep == 0) continue;
            CUDA_TRY(h, cudaMemcpy(no + g * cap, *arr + g * h->q_cap, keep * sizeof(uint32_t),
                                   cudaMemcpyDeviceToDevice));
        }
        arena_free(*arr);
        *arr = no;
    }
    if (h->q_nb != nullptr) {
        int4 *nn = nullptr;
        if (arena_malloc((void **)&nn, G * (size_t)cap * sizeof(int4)) != cudaSuccess) {
            cudaGetLastError();
            h->q_a_csr = nullptr;          // entries so far have no neighbour cache any more: sweeps of this batch
            arena_free(h->q_nb);           // (the forward kernel is relaunched with q_nb = nullptr) read col_idx
            h->q_nb = nullptr;
        } else {
            CUDA_TRY(h, cudaMemset(nn, 0, G * (size_t)cap * sizeof(int4)));
            for (size_t g = 0; g < G; ++g) {
                const size_t keep = (size_t)std::min<int64_t>(g < used.size() ? (int64_t)used[g] : 0, h->q_cap);
                if (keep == 0) continue;
                CUDA_TRY(h, cudaMemcpy(nn + g * cap, h->q_nb + g * h->q_cap, keep * sizeof(int4), cudaMemcpyDeviceToDevice));
            }
            arena_free(h->q_nb);
            h->q_nb = nn;
        }
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
    p.count_scan = h->model_counters;
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

// Unpartitioned unit-weight sweeps of a skewed graph run on the renumbered copy.
// Renumbering costs about as much as sweeping 1,700 sources saves (R-MAT scale 20: 4.8 ms against
// 2.8 ms per 1024 sources), so by default it waits until the handle has been given that much work.
constexpr int64_t kRelabelAfterSources = 2048;

bool relabel_wanted(const bc_handle *h, int64_t sources_now) {
    if (h->full.wgt != nullptr || h->n_arcs <= 0 || h->n_arcs >= ((int64_t)1 << 31) - 64) return false;
    if (h->relabel >= 0) return h->relabel == 1;
    // shallow and skewed: largest degree above 16 average degrees (R-MAT yes; Erdos-Renyi, grids, roads no)
    if (!(h->n_arcs >= 6 * h->n && h->full.max_deg * h->n > 16 * h->n_arcs)) return false;
    return h->relab_ready || h->sources_seen + sources_now >= kRelabelAfterSources;
}

int ensure_relabelled(bc_handle *h, cudaStream_t st) {
    if (h->relab_ready) return BC_OK;
    const int64_t n = h->n, m = h->n_arcs;
    Trace tr;
    Csr &c = h->relab;
    free_csr(c);
    c.n = n;
    c.n_arcs = m;
    ScopedBlock<int32_t> deg, ids, deg_sorted, order, key, key2, val;
    ScopedBlock<int64_t> deg64;
    ScopedBlock<char> tmp;
    CUDA_TRY(h, arena_malloc((void **)&deg.p, n * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&ids.p, n * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&deg_sorted.p, n * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&order.p, n * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&deg64.p, n * sizeof(int64_t)));
    CUDA_TRY(h, arena_malloc((void **)&key.p, m * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&key2.p, m * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&val.p, m * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&c.off, (n + 1) * sizeof(int64_t)));
    CUDA_TRY(h, arena_malloc((void **)&c.col, m * sizeof(int32_t)));
    arena_free(h->d_old_of_new), arena_free(h->d_new_of_old);
    h->d_old_of_new = h->d_new_of_old = nullptr;
    CUDA_TRY(h, arena_malloc((void **)&h->d_old_of_new, n * sizeof(int32_t)));
    CUDA_TRY(h, arena_malloc((void **)&h->d_new_of_old, n * sizeof(int32_t)));
    int id_bits = 1;
    while (((int64_t)1 << id_bits) < n) ++id_bits;
    size_t need_sort = 0, need_scan = 0, need_arcs = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, need_sort, deg.p, deg_sorted.p, ids.p, order.p, (int)n, 0, 32, st);
    cub::DeviceScan::ExclusiveSum(nullptr, need_scan, deg64.p, c.off, (int)n, st);
    cub::DeviceRadixSort::SortPairs(nullptr, need_arcs, key.p, key2.p, val.p, c.col, (int)m, 0, id_bits, st);
    const size_t need = std::max(need_sort, std::max(need_scan, need_arcs));
    CUDA_TRY(h, arena_malloc((void **)&tmp.p, std::max<size_t>(need, 1)));
    size_t bytes = need;
    relabel_degree_kernel<<<grid1d((size_t)n, 256, 2368), 256, 0, st>>>(h->full.off, n, deg.p, ids.p);
    // stable: equal degrees keep the caller's order
    CUDA_TRY(h, cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, deg.p, deg_sorted.p, ids.p, order.p, (int)n, 0,
                                                          32, st));
    relabel_invert_kernel<<<grid1d((size_t)n, 256, 2368), 256, 0, st>>>(order.p, deg_sorted.p, n, h->d_new_of_old, deg64.p);
    bytes = need;
    CUDA_TRY(h, cub::DeviceScan::ExclusiveSum(tmp.p, bytes, deg64.p, c.off, (int)n, st));
    // the host cuts the work items from the new offsets while the device renames and sorts the arcs
    h->h_off_relab.resize((size_t)n + 1);
    CUDA_TRY(h, cudaMemcpyAsync(h->h_off_relab.data(), c.off, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    cudaEvent_t got_offsets = nullptr;
    CUDA_TRY(h, cudaEventCreateWithFlags(&got_offsets, cudaEventDisableTiming));
    struct EventScope {
        cudaEvent_t e;
        ~EventScope() { cudaEventDestroy(e); }
    } event_scope{got_offsets};
    CUDA_TRY(h, cudaEventRecord(got_offsets, st));
    relabel_arcs_kernel<<<grid1d((size_t)n * 32, 256, 148 * 64), 256, 0, st>>>(h->full.off, h->full.col, order.p, c.off,
                                                                              h->d_new_of_old, n, m, c.off + n, key.p, val.p);
    bytes = need;
    CUDA_TRY(h, cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key2.p, val.p, c.col, (int)m, 0, id_bits, st));
    CUDA_TRY(h, cudaMemcpyAsync(h->d_old_of_new, order.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    ScopedBlock<int> d_bad;
    CUDA_TRY(h, arena_malloc((void **)&d_bad.p, sizeof(int)));
    CUDA_TRY(h, cudaMemsetAsync(d_bad.p, 0, sizeof(int), st));
    relabel_check_kernel<<<grid1d((size_t)n, 256, 2368), 256, 0, st>>>(key2.p, c.off, n, d_bad.p);
    int bad = 0;
    CUDA_TRY(h, cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    h->launches += 4;
    CUDA_TRY(h, cudaEventSynchronize(got_offsets));
    h->h_off_relab[(size_t)n] = m;
    tr.mark("  renumber: offsets on the host");
    TRY(build_items(h, c, h->h_off_relab.data(), h->item_arcs));
    CUDA_TRY(h, cudaStreamSynchronize(st));   // the scoped blocks are released on return
    CUDA_TRY(h, cudaGetLastError());
    if (bad) {
        free_csr(c);
        return h->fail(BC_ERR_INPUT, "malformed CSR: an arc without its reverse (the graph must be undirected)");
    }
    tr.mark("  renumber: work items + arc sort");
    h->relab_ready = true;
    return BC_OK;
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


}  // namespace
