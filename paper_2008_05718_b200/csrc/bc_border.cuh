// bc_border.cuh -- kernels of the partitioned ("hybir") forward phase.
//
// Borders of all parts are numbered 0..B-1 part by part (ascending vertex id
// inside a part, reference pkg/src/hybir/partition.py:148).  Per-batch border
// state is laid out [border][lane] with S = 32 * groups lanes per row, so a
// warp touching one border row moves 128 B (int32) or 256 B (fp64) coalesced:
//   D      int32  border distances being refined (kInf = unreached)
//   seedD / seedS Step-1 distance / path count at the source-side borders
//   sig    fp64   path counts at the borders       (forward.py:145-185)
//   arr    fp64   arrival counts (last arc is a cut arc)
// Per-part border tables (border_matrix.py:48-67): bm int32 / sm fp64, b_p x b_p
// row-major, row = from-border, so tab[i][j0..j0+31] is one coalesced read.
//
// Reference arithmetic replaced here: _cut_relax / _matrix_relax and the loop
// of refine_border_distances (forward.py:82-142), _compose_border_sigma
// (forward.py:145-185, as Jacobi rounds of the same recurrence instead of one
// ascending-distance sweep: the dependency graph is a DAG ordered by distance,
// every round settles one more partition crossing, and all values are
// integers in fp64, so the fixpoint is the sweep's result exactly), and the
// seed list of Step 6 (forward.py:232-241).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bcb200 {

constexpr int32_t kInf = 0x3fffffff;

struct BorderGeom {
    int k;                     // parts
    int B;                     // total borders
    const int32_t *border_v;   // [B] vertex id
    const int32_t *border_p;   // [B] part of the border
    const int32_t *part_off;   // [k+1] first border of each part
    const int64_t *tab_off;    // [k] offset of the part's b_p x b_p table
    const int64_t *cin_off;    // [B+1] incoming cut arcs per border
    const int32_t *cin_src;    // [n_cut] source border of each incoming cut arc
    const int32_t *cin_w;      // [n_cut] its weight (1 on unit-weight graphs)
};

// Which (border, lane) pairs a relaxation step applies to (the reference's
// two-sided schedule, forward.py:119-129).
enum Apply : int {
    kApplyAll = 0,     // every part (k > 2: symmetric schedule)
    kApplySource = 1,  // borders in the lane's source part
    kApplyOther = 2    // borders outside the lane's source part
};

__device__ __forceinline__ bool applies(int which, int part, int source_part) {
    return which == kApplyAll || (which == kApplySource) == (part == source_part);
}

// D[j][lane] = kInf, seedS = 0 ... plain fills.
__global__ void fill_border_kernel(int32_t *D, int32_t *seedD, double *seedS, double *sig,
                                   double *arr, size_t count) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        D[i] = kInf;
        seedD[i] = kInf;
        seedS[i] = 0.0;
        sig[i] = 0.0;
        arr[i] = 0.0;
    }
}

// Step-1 border seeds of a batch before the gather: unreached everywhere.
__global__ void fill_seed_kernel(int32_t *seedD, double *seedS, size_t count) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        seedD[i] = kInf;
        seedS[i] = 0.0;
    }
}

// Read (dist, sigma) of every border vertex out of the BFS state: lvl[L][g][v]
// bit = "lane is at distance L".  One thread per (border, lane).
// A group whose lanes all died before level L never wrote lvl[L] (the level
// kernel returns at once), so live[L][g] gates every read of a level row.
__global__ void border_gather_kernel(const uint32_t *const *lvl, const uint32_t *live, int G,
                                     int depth, const double *sigma, int64_t n, BorderGeom geo,
                                     int S, int32_t *D_out, double *S_out) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)geo.B * S) return;
    const int j = (int)(idx / S), lane_all = (int)(idx % S);
    const size_t g = lane_all >> 5;
    const int lane = lane_all & 31;
    const int64_t v = geo.border_v[j];
    int32_t d = kInf;
    for (int L = 0; L < depth; ++L)
        if (((live[(size_t)L * G + g] >> lane) & 1u) && ((lvl[L][g * n + v] >> lane) & 1u)) {
            d = L;
            break;
        }
    D_out[idx] = d;
    if (S_out) S_out[idx] = d < kInf ? sigma[(g * n + v) * 32 + lane] : 0.0;
}

// Rows of the border tables from a BFS batch whose lanes are borders
// first..first+count-1 (each BFS ran inside its own part on the cut-free CSR).
__global__ void border_table_kernel(const uint32_t *const *lvl, const uint32_t *live, int G,
                                    int depth, const double *sigma, int64_t n, BorderGeom geo,
                                    int first, int count, int32_t *bm, double *sm) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lanes = (count + 31) / 32 * 32;
    if (idx >= (size_t)geo.B * lanes) return;
    const int j = (int)(idx / lanes), lane_all = (int)(idx % lanes);
    if (lane_all >= count) return;
    const int i = first + lane_all;          // from-border (BFS source)
    const int p = geo.border_p[i];
    if (geo.border_p[j] != p) return;        // tables hold same-part pairs only
    const size_t g = lane_all >> 5;
    const int lane = lane_all & 31;
    const int64_t v = geo.border_v[j];
    int32_t d = kInf;
    for (int L = 0; L < depth; ++L)
        if (((live[(size_t)L * G + g] >> lane) & 1u) && ((lvl[L][g * n + v] >> lane) & 1u)) {
            d = L;
            break;
        }
    const int b = geo.part_off[p + 1] - geo.part_off[p];
    const size_t at = (size_t)geo.tab_off[p] + (size_t)(i - geo.part_off[p]) * b + (j - geo.part_off[p]);
    bm[at] = d;
    sm[at] = d < kInf ? sigma[(g * n + v) * 32 + lane] : 0.0;
}

// Step 2 / Step 4 (forward.py:82-88): D[j] = min(D[j], D[i] + 1) over incoming
// cut arcs (i -> j).  `which` selects destinations by side; sources are always
// on the other side of a cut arc.  Two-part runs update in place (source and
// destination sets are disjoint); k > 2 reads `Din` and writes `Dout`.
__global__ void cut_relax_kernel(BorderGeom geo, int S, const int32_t *Din, int32_t *Dout,
                                 const int32_t *lane_part, const uint32_t *lane_active, int which,
                                 uint32_t *lane_changed, uint32_t *rowflag) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)geo.B * S) return;   // whole warps: B * S is a multiple of 32
    const int j = (int)(idx / S), lane = (int)(idx % S);
    const int32_t old = Din[idx];
    int32_t best = old;
    if (lane_active[lane] && applies(which, geo.border_p[j], lane_part[lane])) {
        for (int64_t a = geo.cin_off[j]; a < geo.cin_off[j + 1]; ++a) {
            const int32_t di = Din[(size_t)geo.cin_src[a] * S + lane];
            best = min(best, min(di + geo.cin_w[a], kInf));
        }
    }
    if (Dout != Din || best != old) Dout[idx] = best;
    if (best != old && lane_changed) lane_changed[lane] = 1u;
    // rowflag[j][lane / 32]: some lane of the word was lowered.  The closure pass that follows
    // only has to push these rows on: every other row was either pushed by the pass that
    // followed its own change, or set by a closure pass / an intra-part search, and then
    // D[i] + bm[i][j] cannot beat what is there (bm is a metric closure).
    if (rowflag) {
        const unsigned nz = __ballot_sync(0xffffffffu, best != old);
        if ((threadIdx.x & 31) == 0) rowflag[idx >> 5] = nz;
    }
}

// Step 3 / Step 5 (forward.py:91-96): one Jacobi pass of the min-plus closure
// Dout[j] = min(Din[j], min_i Din[i] + bm[i][j]) inside each part -- a min-plus
// "matrix product" b_p x b_p by b_p x S.  Block = 64 borders j x 64 lanes, every
// thread owns a 4 x 4 register tile; the i-loop is tiled through shared memory
// (two 128-bit loads feed 16 fused add-min instructions, VIADDMNMX via
// __viaddmin_s32), so the kernel is bound by integer issue, not by shared-memory
// bandwidth.  The bound: 148 SMs x 128 lanes x 1.9 GHz = 36 T min-plus / s.
constexpr int kTJ = 64;  // borders j per block
constexpr int kTL = 64;  // lanes per block
constexpr int kTI = 32;  // borders i per shared-memory tile
__global__ void __launch_bounds__(256) matrix_relax_kernel(BorderGeom geo, int S,
                                                           const int32_t *Din, int32_t *Dout,
                                                           const int32_t *bm,
                                                           const int32_t *lane_part,
                                                           const uint32_t *lane_active, int which,
                                                           uint32_t *lane_changed,
                                                           const uint32_t *rowflag, int only_part = -1) {
    __shared__ __align__(16) int32_t sD[kTI][kTL];
    __shared__ __align__(16) int32_t sB[kTI][kTJ];
    const int p = blockIdx.z;
    const int b = geo.part_off[p + 1] - geo.part_off[p];
    const int j0 = blockIdx.x * kTJ;
    if (j0 >= b) return;
    const int base = geo.part_off[p];
    if (only_part >= 0 && p != only_part) {
        // graph-partitioned runs with one table per rank: the closure of another part is its
        // owner's work; its rows pass through (Din and Dout are swapped by the caller)
        const int l0 = blockIdx.y * kTL;
        for (int e = threadIdx.x; e < kTJ * kTL; e += blockDim.x) {
            const int j = j0 + e / kTL, l = l0 + e % kTL;
            if (j < b && l < S) Dout[(size_t)(base + j) * S + l] = Din[(size_t)(base + j) * S + l];
        }
        return;
    }
    const int32_t *tab = bm + geo.tab_off[p];
    const int tl = threadIdx.x & 15, tj = threadIdx.x >> 4;   // 16 lane quads x 16 border quads
    const int lane4 = blockIdx.y * kTL + 4 * tl;              // first of this thread's 4 lanes
    const bool lanes_in = lane4 < S;                           // S is a multiple of 32: a quad is in or out
    int32_t best[4][4], old[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int j = j0 + 4 * tj + r;
        int4 v = make_int4(kInf, kInf, kInf, kInf);
        if (j < b && lanes_in) v = *reinterpret_cast<const int4 *>(Din + (size_t)(base + j) * S + lane4);
        old[r][0] = best[r][0] = v.x;
        old[r][1] = best[r][1] = v.y;
        old[r][2] = best[r][2] = v.z;
        old[r][3] = best[r][3] = v.w;
    }
    const int words = S >> 5;   // rowflag words per border row
    for (int i0 = 0; i0 < b; i0 += kTI) {
        // rows the preceding cut-arc step did not lower cannot improve anything: skip the tile
        bool live_tile = rowflag == nullptr;
        if (rowflag != nullptr && threadIdx.x < 2 * kTI) {
            const int i = i0 + (threadIdx.x >> 1), w = blockIdx.y * (kTL / 32) + (threadIdx.x & 1);
            live_tile = i < b && w < words && rowflag[(size_t)(base + i) * words + w] != 0;
        }
        if (!__syncthreads_or(live_tile)) continue;   // (also the barrier that protects the tiles)
#pragma unroll
        for (int k = 0; k < 2; ++k) {                          // 32 x 16 int4 slots of sD
            const int slot = threadIdx.x + 256 * k, row = slot >> 4, c4 = slot & 15;
            const int i = i0 + row, l4 = blockIdx.y * kTL + 4 * c4;
            int4 v = make_int4(kInf, kInf, kInf, kInf);
            if (i < b && l4 < S) v = *reinterpret_cast<const int4 *>(Din + (size_t)(base + i) * S + l4);
            *reinterpret_cast<int4 *>(&sD[row][4 * c4]) = v;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {                          // 32 x 64 entries of sB, coalesced along j
            const int e = threadIdx.x + 256 * k, row = e >> 6, cj = e & 63;
            const int i = i0 + row, j = j0 + cj;
            sB[row][cj] = (i < b && j < b) ? tab[(size_t)i * b + j] : kInf;
        }
        __syncthreads();
#pragma unroll 4
        for (int i = 0; i < kTI; ++i) {
            const int4 d = *reinterpret_cast<const int4 *>(&sD[i][4 * tl]);
            const int4 t = *reinterpret_cast<const int4 *>(&sB[i][4 * tj]);
            const int dd[4] = {d.x, d.y, d.z, d.w}, tt[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int l = 0; l < 4; ++l) best[r][l] = __viaddmin_s32(dd[l], tt[r], best[r][l]);
        }
    }
    if (!lanes_in) return;
    bool on[4], changed[4] = {false, false, false, false};
#pragma unroll
    for (int l = 0; l < 4; ++l) on[l] = lane_active[lane4 + l] && applies(which, p, lane_part[lane4 + l]);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int j = j0 + 4 * tj + r;
        if (j >= b) continue;
        int32_t v[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            v[l] = on[l] ? min(best[r][l], kInf) : old[r][l];
            changed[l] |= v[l] != old[r][l];
        }
        *reinterpret_cast<int4 *>(Dout + (size_t)(base + j) * S + lane4) = make_int4(v[0], v[1], v[2], v[3]);
    }
    if (lane_changed)
#pragma unroll
        for (int l = 0; l < 4; ++l)
            if (changed[l]) lane_changed[lane4 + l] = 1u;
}

// arr[j] = sum of sig[i] over incoming cut arcs (i -> j) that are tight
// (forward.py:170-174), in arc order.
// darr[j] = what the round adds to arr[j]: the composition only has to push the change on.
// rowflag[j][lane / 32] = some lane of that 32-lane word changed (S is a multiple of 32, so a
// warp covers one word of one border): compose_sigma_kernel skips the row tiles nothing
// changed in without reading them.
__global__ void arrival_kernel(BorderGeom geo, int S, const int32_t *D, const double *sig,
                               double *arr, double *darr, const uint32_t *lane_run,
                               uint32_t *rowflag) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)geo.B * S) return;   // whole warps: B * S is a multiple of 32
    const int j = (int)(idx / S), lane = (int)(idx % S);
    double delta = 0.0;
    if (lane_run[lane]) {          // (a lane whose counts settled in an earlier round stays put)
        const int32_t dj = D[idx];
        double a = 0.0;
        if (dj < kInf)
            for (int64_t c = geo.cin_off[j]; c < geo.cin_off[j + 1]; ++c) {
                const size_t at = (size_t)geo.cin_src[c] * S + lane;
                if (D[at] + geo.cin_w[c] == dj) a += sig[at];
            }
        delta = a - arr[idx];
        arr[idx] = a;
    }
    darr[idx] = delta;
    const unsigned nz = __ballot_sync(0xffffffffu, delta != 0.0);
    if ((threadIdx.x & 31) == 0) rowflag[idx >> 5] = nz;
}

// sig[j] = (seed count if j is on the source side and its Step-1 distance is
// still optimal) + sum over same-part borders c with arr[c] != 0 and
// D[c] + bm[c][j] == D[j] of arr[c] * sm[c][j]   (forward.py:176-184).
// Same 64 x 64 block / 4 x 4 register tiling as matrix_relax_kernel.  Delta form: the tight
// (c, j) structure is fixed once the distances are refined, so a round adds
// sum_c darr[c] * sm[c][j] to sig[j], where darr is what the round changed in the arrival
// counts; rows c whose four lanes did not change are skipped, which makes the later rounds
// cheap (each border's arrival count changes in one or two rounds).  Path counts are
// integer-valued, so the sum is exact in any order below 2^53.
__global__ void __launch_bounds__(256) compose_sigma_kernel(
    BorderGeom geo, int S, const int32_t *D, const int32_t *seedD, const double *seedS,
    const double *darr, const int32_t *bm, const double *sm, const int32_t *lane_part,
    double *sig, const uint32_t *lane_run, uint32_t *lane_changed, int first_round,
    const uint32_t *rowflag, int only_part = -1) {
    __shared__ __align__(16) int32_t sD[kTI][kTL];
    __shared__ __align__(16) double sA[kTI][kTL];
    __shared__ __align__(16) int32_t sB[kTI][kTJ];
    __shared__ __align__(16) double sS[kTI][kTJ];
    const int p = blockIdx.z;
    if (only_part >= 0 && p != only_part) return;   // another rank composes that part's counts
    const int b = geo.part_off[p + 1] - geo.part_off[p];
    const int j0 = blockIdx.x * kTJ;
    if (j0 >= b) return;
    const int base = geo.part_off[p];
    const int32_t *tbm = bm + geo.tab_off[p];
    const double *tsm = sm + geo.tab_off[p];
    const int tl = threadIdx.x & 15, tj = threadIdx.x >> 4;
    const int lane4 = blockIdx.y * kTL + 4 * tl;
    const bool lanes_in = lane4 < S;
    // lanes are independent: one whose counts did not change in a round is final, and a block
    // whose 64 lanes are all final has nothing left to do (the rounds a lane needs = the number
    // of part crossings on its shortest paths, which differs from source to source)
    bool run[4] = {false, false, false, false};
    if (lanes_in)
#pragma unroll
        for (int l = 0; l < 4; ++l) run[l] = lane_run[lane4 + l] != 0;
    if (!__syncthreads_or(run[0] || run[1] || run[2] || run[3])) return;
    int32_t dj[4][4];
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int j = j0 + 4 * tj + r;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            dj[r][l] = kInf;
            acc[r][l] = 0.0;
            if (j < b && lanes_in) {
                const size_t at = (size_t)(base + j) * S + lane4 + l;
                dj[r][l] = D[at];
                if (first_round && dj[r][l] < kInf && p == lane_part[lane4 + l] && seedD[at] == dj[r][l])
                    acc[r][l] = seedS[at];
            }
        }
    }
    const int words = S >> 5;   // rowflag words per border row
    for (int i0 = 0; i0 < b; i0 += kTI) {
        // nothing changed in these kTI rows for this block's 64 lanes: skip the tile unread
        bool live_tile = false;
        if (threadIdx.x < 2 * kTI) {
            const int i = i0 + (threadIdx.x >> 1), w = blockIdx.y * (kTL / 32) + (threadIdx.x & 1);
            live_tile = i < b && w < words && rowflag[(size_t)(base + i) * words + w] != 0;
        }
        if (!__syncthreads_or(live_tile)) continue;   // (also the barrier that protects the tiles)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int e = threadIdx.x + 256 * k, row = e >> 6, c = e & 63;
            const int i = i0 + row, lane = blockIdx.y * kTL + c, j = j0 + c;
            const bool lin = i < b && lane < S;
            const size_t at = (size_t)(base + i) * S + lane;
            sD[row][c] = lin ? D[at] : kInf;
            sA[row][c] = lin ? darr[at] : 0.0;
            const bool in = i < b && j < b;
            sB[row][c] = in ? tbm[(size_t)i * b + j] : kInf;
            sS[row][c] = in ? tsm[(size_t)i * b + j] : 0.0;
        }
        __syncthreads();
        for (int i = 0; i < kTI; ++i) {
            const double a[4] = {sA[i][4 * tl], sA[i][4 * tl + 1], sA[i][4 * tl + 2], sA[i][4 * tl + 3]};
            if (a[0] == 0.0 && a[1] == 0.0 && a[2] == 0.0 && a[3] == 0.0) continue;
            const int4 d = *reinterpret_cast<const int4 *>(&sD[i][4 * tl]);
            const int4 t = *reinterpret_cast<const int4 *>(&sB[i][4 * tj]);
            const int dd[4] = {d.x, d.y, d.z, d.w}, tt[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double sv = sS[i][4 * tj + r];
#pragma unroll
                for (int l = 0; l < 4; ++l)
                    if (a[l] != 0.0 && dd[l] + tt[r] == dj[r][l]) acc[r][l] += a[l] * sv;
            }
        }
    }
    if (!lanes_in) return;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int j = j0 + 4 * tj + r;
        if (j >= b) continue;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            if (!run[l] || acc[r][l] == 0.0 || dj[r][l] >= kInf) continue;
            sig[(size_t)(base + j) * S + lane4 + l] += acc[r][l];
            lane_changed[lane4 + l] = 1u;
        }
    }
}

// End of a composition round: lanes that changed run again.
__global__ void lane_round_kernel(int S, uint32_t *lane_run, uint32_t *lane_changed, uint32_t *any_running) {
    const int lane = blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= S) return;
    const uint32_t c = lane_changed[lane];
    lane_run[lane] = c;
    lane_changed[lane] = 0;
    if (c) *any_running = 1u;
}

// Per-lane bookkeeping of the refinement loop (forward.py:113-135).
//   enter: a lane runs the loop iff cut arcs exist and Step 1 reached a border
//   of its source part; after every iteration a lane whose source side did not
//   change stops (forward.py:128).
__global__ void lane_enter_kernel(BorderGeom geo, int S, int lanes, const int32_t *D,
                                  const int32_t *lane_part, uint32_t *lane_active,
                                  uint32_t *lane_entered, int64_t n_cut) {
    const int lane = blockIdx.x;   // one block per lane, threads stride over the part's borders
    if (lane >= S) return;
    int found = 0;
    if (lane < lanes && n_cut > 0) {
        const int p = lane_part[lane];
        for (int j = geo.part_off[p] + threadIdx.x; j < geo.part_off[p + 1]; j += blockDim.x)
            if (D[(size_t)j * S + lane] < kInf) {
                found = 1;
                break;
            }
    }
    const uint32_t on = __syncthreads_or(found) ? 1u : 0u;
    if (threadIdx.x == 0) {
        lane_active[lane] = on;
        lane_entered[lane] = on;
    }
}

__global__ void lane_step_kernel(int S, uint32_t *lane_active, uint32_t *lane_changed,
                                 int32_t *lane_iters, uint32_t *any_active) {
    const int lane = blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= S) return;
    if (lane_active[lane]) {
        lane_iters[lane] += 1;
        if (!lane_changed[lane]) lane_active[lane] = 0;
        else *any_active = 1u;
    }
    lane_changed[lane] = 0;
}

// Largest finite border distance that carries an arrival count: Step 6 must
// keep stepping levels at least that far even through empty frontiers.
// all_finite: every border with a finite distance counts (graph-partitioned runs mark the other
// parts' borders at their level whether or not a cut arc arrives there, see inject_seeds_kernel).
__global__ void max_seed_level_kernel(const int32_t *D, const double *arr, size_t count,
                                      int *out, int all_finite) {
    int m = -1;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x)
        if (D[i] < kInf && (all_finite || arr[i] != 0.0)) m = max(m, D[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m >= 0) atomicMax(out, m);
}

// Step 6 seeds (forward.py:232-241): border j joins level D[j] with base count
// arr[j] when D[j] is finite and arr[j] != 0.  Runs after the pull of level L:
// a border the pull just discovered at L keeps its pulled count and adds the
// base (relax.py:70-71,95-99); one found at a smaller level ignores the seed.
// own_part >= 0 (graph-partitioned runs, one part per rank): borders of the OTHER parts have no
// rows on this rank; they are only marked at their level -- all of them, also those no cut arc
// arrives at -- because the backward exchange plan reads those marks to find the cross-part
// parents of this rank's borders (dist_plan_kernel).
__global__ void inject_seeds_kernel(BorderGeom geo, int S, int lanes, const int32_t *D,
                                    const double *arr, int level, int64_t n, uint32_t *vis,
                                    uint32_t *cur, double *sigma, uint32_t *live_cur, int own_part) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)geo.B * S) return;
    const int lane_all = (int)(idx % S);
    if (lane_all >= lanes || D[idx] != level) return;
    const double base = arr[idx];
    const int j = (int)(idx / S);
    if (base == 0.0 && (own_part < 0 || geo.border_p[j] == own_part)) return;
    const size_t g = lane_all >> 5;
    const uint32_t bit = 1u << (lane_all & 31);
    const int64_t v = geo.border_v[j];
    const size_t at = (g * n + v) * 32 + (lane_all & 31);
    if (cur[g * n + v] & bit) {
        sigma[at] += base;                 // reached through an arc at the same level
    } else if (!(vis[g * n + v] & bit)) {
        atomicOr(vis + g * n + v, bit);    // other lanes of the word may be seeded concurrently
        atomicOr(cur + g * n + v, bit);
        sigma[at] = base;
        atomicOr(live_cur + g, bit);
    }
}

// presence[(L * k + part) * G + g] |= lanes of group g that have a vertex of
// `part` at level L -- the raw material of max_level / levels in the reports
// (forward.py:52-64, backward.py:33-43).
__global__ void level_presence_kernel(const uint32_t *lvl, const uint32_t *live_level,
                                      const int32_t *part, int64_t n, int k, int G,
                                      uint32_t *presence_level) {
    extern __shared__ uint32_t sp[];  // [k]
    const size_t g = blockIdx.y;
    if (live_level[g] == 0) return;  // the level row of a dead group was never written
    for (int i = threadIdx.x; i < k; i += blockDim.x) sp[i] = 0;
    __syncthreads();
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t m = lvl[g * n + v];
        if (m) atomicOr(&sp[part[v]], m);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        if (sp[i]) atomicOr(&presence_level[(size_t)i * G + g], sp[i]);
}

// Backward sync accounting for two parts (backward.py:46-56,121-139).  A tight
// cut arc u -> j makes u's side pull border j; the reference counts one sync
// event per distinct (consumer side, consumer level d[u], producer level d[j])
// and 16 bytes per border child in each such set.  With unit weights d[j] is
// d[u] + 1; with weights a border can serve parents at several levels.
// flag[j][lane] = distinct consumer levels that pull j (its share of the
// payload); level_bits[((side * W + d[u] / 32) * wmax + (w - 1)) * S + lane]
// collects the distinct (consumer level, arc weight) pairs per consumer side.
__global__ void sync_mark_kernel(BorderGeom geo, int S, const int32_t *Dfin, uint32_t *flag,
                                 uint32_t *level_bits, int W, int wmax) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)geo.B * S) return;
    const int j = (int)(idx / S), lane = (int)(idx % S);
    const int32_t dj = Dfin[idx];
    uint32_t f = 0;
    if (dj < kInf) {
        const int consumer = 1 - geo.border_p[j];  // two parts: the other side pulls
        for (int64_t c = geo.cin_off[j]; c < geo.cin_off[j + 1]; ++c) {
            const int w = geo.cin_w[c];
            const int32_t du = Dfin[(size_t)geo.cin_src[c] * S + lane];
            if (du + w != dj) continue;
            bool seen = false;   // an earlier tight arc from the same consumer level
            for (int64_t c2 = geo.cin_off[j]; c2 < c && !seen; ++c2)
                seen = geo.cin_w[c2] == w && Dfin[(size_t)geo.cin_src[c2] * S + lane] == du;
            if (seen) continue;
            ++f;
            atomicOr(&level_bits[(((size_t)consumer * W + (du >> 5)) * wmax + (w - 1)) * S + lane],
                     1u << (du & 31));
        }
    }
    flag[idx] = f;
}

__global__ void sync_count_kernel(int B, int S, int W, int wmax, const uint32_t *flag,
                                  const uint32_t *level_bits, int64_t *sync_events,
                                  int64_t *comm_bytes) {
    const int lane = blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= S) return;
    int64_t children = 0, events = 0;
    for (int j = 0; j < B; ++j) children += flag[(size_t)j * S + lane];
    for (int w = 0; w < 2 * W * wmax; ++w) events += __popc(level_bits[(size_t)w * S + lane]);
    sync_events[lane] = events;
    comm_bytes[lane] = 16 * children;
}

}  // namespace bcb200
