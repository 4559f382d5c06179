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
#include "bc_bwd_push.cuh"
#include "bc_deep.cuh"
#include "bc_dist.cuh"
#include "bc_kernels.cuh"
#include "bc_relabel.cuh"
#include "bc_sssp.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <stdexcept>
#include <thread>
#include <unordered_map>
#include <vector>

using namespace bcb200;

#include "engine_state.cuh"
#include "engine_sweeps.cuh"
#include "engine_border.cuh"
#include "engine_sssp.cuh"
#include "engine_run.cuh"

namespace {

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
#ifdef BC_CARVEOUT
    // shared-memory carve-out of the dense pull kernels, in percent of the SM's 228 KB
    cudaFuncSetAttribute(level_kernel<false, false, false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, BC_CARVEOUT);
    cudaFuncSetAttribute(level_kernel<true, false, false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, BC_CARVEOUT);
    cudaFuncSetAttribute(level_kernel<false, false, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, BC_CARVEOUT);
    cudaFuncSetAttribute(level_kernel<true, false, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, BC_CARVEOUT);
#endif
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
    int64_t wmax = 1, wsum = 0;
    for (int64_t a = 0; a < h->n_arcs; ++a) {
        if (weights[a] <= 0) return h->fail(BC_ERR_INPUT, "arc weights must be positive integers");
        wmax = std::max<int64_t>(wmax, weights[a]);
        wsum += weights[a];
    }
    h->wsum = wsum;
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
            if (h->relab_ready) TRY(build_items(h, h->relab, h->h_off_relab.data(), h->item_arcs));
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
    if (k == "sssp") {
        if (value < -1 || value > 1) return h->fail(BC_ERR_INPUT, "sssp must be -1 (by weight range), 0 or 1");
        h->wgt_mode = (int)value;
        return BC_OK;
    }
    if (k == "relabel") {
        if (value < -1 || value > 1) return h->fail(BC_ERR_INPUT, "relabel must be -1 (by degree skew), 0 or 1");
        h->relabel = (int)value;
        return BC_OK;
    }
    if (k == "sssp_blocks") {
        h->sp_blocks = (int)std::max<int64_t>(0, std::min<int64_t>(value, 1 << 16));
        return BC_OK;
    }
    if (k == "sssp_delta") {
        if (value < 0) return h->fail(BC_ERR_INPUT, "sssp_delta must be >= 0 (0 = 16 mean arc weights)");
        h->sp_delta = value;
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
    if (k == "model_counters") {
        h->model_counters = value ? 1 : 0;
        return BC_OK;
    }
    if (k == "deep_compact") {
        // 0: row layout everywhere; 1 (default): deep graphs sweep backward over level-ordered
        // values with one atomically-updated BC vector; 2: same, BC kept in per-group partials
        if (value < 0 || value > 2) return h->fail(BC_ERR_INPUT, "deep_compact must be 0, 1 or 2");
        h->deep_compact = (int)value;
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
    if (k == "bwd_push") {
        // child-driven backward levels (bc_bwd_push.cuh): 0 = every level parent-driven, else the
        // factor by which the children's arcs must undercut the parents' arcs
        if (value < 0) return h->fail(BC_ERR_INPUT, "bwd_push must be >= 0");
        h->bwd_push = (int)value;
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

}  // extern "C"

#include "engine_dist.cuh"

extern "C" {

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
    free_csr(h->relab);
    arena_free(h->d_old_of_new), arena_free(h->d_new_of_old);
    arena_free(h->counters);
    arena_free(h->dflags);
    arena_free(h->d_maxlvl);
    arena_free(h->d_src);
    arena_free(h->bc_scratch);
    arena_free((void *)h->d_lvl_ptrs);
    arena_free(h->presence);
    arena_free(h->dist_border_v), arena_free(h->dist_counts), arena_free(h->dist_offsets);
    arena_free(h->dist_scan_tmp);
    arena_free(h->dist_cut_off), arena_free(h->dist_cut_dst), arena_free(h->dist_border_off_dev);
    arena_free(h->plan_idx), arena_free(h->plan_mask), arena_free(h->plan_voff);
    arena_free(h->plan_eoff), arena_free(h->plan_cnt_e), arena_free(h->plan_cnt_v);
    if (h->side_stream) cudaStreamDestroy(h->side_stream);
    if (h->side_go) cudaEventDestroy(h->side_go);
    if (h->side_done) cudaEventDestroy(h->side_done);
    delete h;
}

}  // extern "C"
