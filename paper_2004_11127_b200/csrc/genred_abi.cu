// genred_abi.cu -- the C ABI of libgenred (include/genred.h): validation, parameter folding,
// launch planning (rows per thread, j-splits), scratch arena, host-pointer staging, dispatch.
//
// Host runtime only: every step of the path itself runs in the kernels of this library
// (pack -> pair loop -> fixed-order merge).  There is no CPU fallback: without a device,
// genred_create fails with GENRED_E_CUDA.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/genred.h"
#include "internal.h"

using namespace genred;

struct genred_ctx {
    int device = 0;
    int num_sms = 148;
    std::string err;
    void *scratch = nullptr;
    size_t scratch_cap = 0;
    size_t scratch_need = 0;                                   // bytes the last call used
    void *stage = nullptr;
    size_t stage_cap = 0;
    void *hstage = nullptr;                                    // pinned host gather buffer (small
    size_t hstage_cap = 0;                                     //   GENRED_MEM_HOST calls)
    genred_plan plan{};
    int64_t launches = 0;
    std::map<std::tuple<int, int, int, int, int>, int> occ;   // (kind, a, b, c, R) -> CTAs/SM
    int *fallback_dev = nullptr;                               // k-NN rows rescanned exactly
    const uint32_t *geo_dev = nullptr;                         // Gaussian Sum bounding box
    int geo_D = 0;
    float geo_s = 0.f;
    unsigned *tile_done = nullptr;                             // split-merge arrival counters (zero at rest)
    int64_t tile_done_cap = 0;
    bool small_fused = true;                                   // genred_set_option("small_fused")
    bool fused_merge = true;                                   // genred_set_option("fused_merge")
    int local_form = 1;                                        // genred_set_option("local_form")
    bool split_major = true;                                   // genred_set_option("split_major")
    const float4 *centers_dev = nullptr;                       // last tile-centred call: per-tile
    int64_t centers_n = 0;                                     //   (centre, r^2 or -1)
    bool profiling = false;
    std::vector<cudaEvent_t> ev;                               // pairs: (start, stop) per launch
    int nprof = 0;
};

namespace {

constexpr double kLog2e = 1.4426950408889634074;
constexpr int kMaxSplit = 64;                // 512-j tile splits (ArgKMin, LSE_GRAD)
constexpr int kMaxSplitPairs = 1024;         // record-pair splits (Sum, LSE): merged by warp finalizes

genred_status fail(genred_ctx *ctx, genred_status st, const std::string &msg) {
    if (ctx) ctx->err = msg;
    return st;
}

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

genred_status validate(const genred_args *a, std::string &msg) {
    if (!a) { msg = "args is NULL"; return GENRED_E_INVALID; }
    if (a->abi_version != GENRED_ABI_VERSION) {
        msg = "abi_version mismatch (expected " + std::to_string(GENRED_ABI_VERSION) + ")";
        return GENRED_E_INVALID;
    }
    if (a->memory != GENRED_MEM_DEVICE && a->memory != GENRED_MEM_HOST) {
        msg = "memory must be GENRED_MEM_DEVICE or GENRED_MEM_HOST"; return GENRED_E_INVALID;
    }
    if (a->M < 0 || a->N < 0) { msg = "M and N must be >= 0"; return GENRED_E_SHAPE; }
    if (a->D < 1 || a->E < 1) { msg = "D and E must be >= 1"; return GENRED_E_SHAPE; }
    if (a->split_j < 0) { msg = "split_j must be >= 0"; return GENRED_E_INVALID; }
    const int f = a->formula, r = a->reduction;
    const bool sum_pair = r == GENRED_SUM &&
        (f == GENRED_GAUSS || f == GENRED_GAUSS_GRADX || f == GENRED_GAUSS_SUM_GRADX || f == GENRED_SQDIST);
    const bool lse_pair = r == GENRED_LSE && f == GENRED_SQDIST;
    const bool argk_pair = r == GENRED_ARGKMIN && f == GENRED_SQDIST;
    const bool smg_pair = r == GENRED_SUM && f == GENRED_LSE_GRAD;
    if (!sum_pair && !lse_pair && !argk_pair && !smg_pair) {
        msg = "unsupported (formula, reduction) pair"; return GENRED_E_UNSUPPORTED;
    }
    if (sum_pair && (a->D > 8 || a->E > 4)) {
        msg = "Sum formulas support 1 <= D <= 8 and 1 <= E <= 4"; return GENRED_E_UNSUPPORTED;
    }
    if ((lse_pair || smg_pair) && (a->D > 8 || a->E != 1)) {
        msg = "log-sum-exp supports 1 <= D <= 8 and E == 1 (scalar formula)"; return GENRED_E_UNSUPPORTED;
    }
    if (argk_pair) {
        if (a->K < 1) { msg = "K must be >= 1"; return GENRED_E_SHAPE; }
        if (a->K > 32) { msg = "ArgKMin supports K <= 32"; return GENRED_E_UNSUPPORTED; }
        if (a->E != 1) { msg = "ArgKMin is scalar-formula only (E == 1)"; return GENRED_E_UNSUPPORTED; }
        if (a->D > 16 && a->K > 28) { msg = "the tensor-core ArgKMin path (D > 16) supports K <= 28"; return GENRED_E_UNSUPPORTED; }
        if (a->D > 16384) { msg = "ArgKMin supports D <= 16384"; return GENRED_E_UNSUPPORTED; }
        if (a->N > (int64_t)INT32_MAX - kTileJ) { msg = "ArgKMin requires N < 2^31"; return GENRED_E_SHAPE; }
        if (a->out_dtype != GENRED_F32) { msg = "ArgKMin distances are fp32 (out_dtype F32)"; return GENRED_E_INVALID; }
    }
    if ((f == GENRED_GAUSS || f == GENRED_GAUSS_GRADX || f == GENRED_GAUSS_SUM_GRADX || lse_pair || smg_pair) &&
        !(isfinite(a->scale) && a->scale > 0.0)) {
        msg = "scale (sigma or eps) must be finite and > 0"; return GENRED_E_INVALID;
    }
    if (a->out_dtype != GENRED_F32 && a->out_dtype != GENRED_F64) {
        msg = "out_dtype must be GENRED_F32 or GENRED_F64"; return GENRED_E_INVALID;
    }
    if (a->n_ranges < 0) { msg = "n_ranges must be >= 0"; return GENRED_E_SHAPE; }
    if (a->n_ranges > 0) {
        if (!(sum_pair || lse_pair || (argk_pair && a->D <= 16))) {
            msg = "block-sparse ranges are supported for Sum, LSE and ArgKMin with D <= 16"; return GENRED_E_UNSUPPORTED;
        }
        if (!a->ranges_i || !a->slices || !a->ranges_j) { msg = "ranges_i / slices / ranges_j is NULL"; return GENRED_E_INVALID; }
        int64_t prev_ie = 0, prev_slice = 0;
        for (int64_t c = 0; c < a->n_ranges; ++c) {
            const int64_t is = a->ranges_i[2 * c], ie = a->ranges_i[2 * c + 1];
            if (is < prev_ie || ie < is || ie > a->M) { msg = "ranges_i must be sorted, disjoint and within [0, M]"; return GENRED_E_SHAPE; }
            prev_ie = ie;
            const int64_t s1 = a->slices[c];
            if (s1 < prev_slice) { msg = "slices must be non-decreasing"; return GENRED_E_SHAPE; }
            int64_t prev_je = 0;
            for (int64_t k = prev_slice; k < s1; ++k) {
                const int64_t js = a->ranges_j[2 * k], je = a->ranges_j[2 * k + 1];
                if (js < prev_je || je < js || je > a->N) { msg = "a cluster's ranges_j must be sorted, disjoint and within [0, N]"; return GENRED_E_SHAPE; }
                prev_je = je;
            }
            prev_slice = s1;
        }
    }
    if (a->M > 0) {
        if (!a->out) { msg = "out is NULL"; return GENRED_E_INVALID; }
        if (a->N > 0 && !a->x) { msg = "x is NULL"; return GENRED_E_INVALID; }
        if (argk_pair && !a->out_idx) { msg = "out_idx is NULL"; return GENRED_E_INVALID; }
        if ((f == GENRED_GAUSS_SUM_GRADX || smg_pair) && !a->out_grad) { msg = "out_grad is NULL"; return GENRED_E_INVALID; }
    }
    if (a->N > 0 && a->M > 0 && !a->y) { msg = "y is NULL"; return GENRED_E_INVALID; }
    const void *fp[] = {a->x, a->y, a->b, a->g, a->out_grad};
    for (const void *p : fp)
        if (p && !aligned(p, 4)) { msg = "fp32 pointers must be 4-byte aligned"; return GENRED_E_INVALID; }
    if (a->out && !aligned(a->out, a->out_dtype == GENRED_F64 ? 8 : 4)) {
        msg = "out is misaligned for its dtype"; return GENRED_E_INVALID;
    }
    if ((a->out_idx && !aligned(a->out_idx, 8)) || (a->lse_state && !aligned(a->lse_state, 8)) ||
        (a->row_shift && !aligned(a->row_shift, 8)) || (a->col_shift && !aligned(a->col_shift, 8))) {
        msg = "out_idx / lse_state / row_shift / col_shift must be 8-byte aligned"; return GENRED_E_INVALID;
    }
    msg.clear();
    return GENRED_OK;
}

int occupancy(genred_ctx *ctx, int kind, int a, int b, int c, int R) {
    auto key = std::make_tuple(kind, a, b, c, R);
    auto it = ctx->occ.find(key);
    if (it != ctx->occ.end()) return it->second;
    int n = 1;
    if (kind == 0) n = sum_occupancy(a, b, c, R);
    else if (kind == 1) n = lse_occupancy(a, R, b != 0);
    else if (kind == 3) n = softmax_grad_occupancy(a, R);
    else n = argk_occupancy(a, b, R);
    ctx->occ[key] = n;
    return n;
}

constexpr int64_t kDirectMaxN = 64;          // Gaussian Sum: N at or below -> direct form, no bbox
constexpr int64_t kDirectMaxM = 16;          // Gaussian Sum: M at or below -> direct form, no bbox
constexpr int64_t kMinSplitPairs = 64;       // shortest record-pair j-split (128 j)
#ifndef GENRED_MIN_WAVES
#define GENRED_MIN_WAVES 4
#endif
constexpr int64_t kMinWaves = GENRED_MIN_WAVES;  // Sum / LSE row-tile kernels: waves of CTAs to aim for
constexpr int64_t kMaxSplitSmm = 2048;       // small-M mode: j-splits (CTAs of a few rows each)
constexpr int64_t kSmmMaxM = 64;             // small-M mode for M at or below
constexpr int64_t kMinSmmPairs = 512;        // small-M mode: shortest j-split (1024 j)
// Tile-centred form of the Gaussian Sum (R18j, tile_order.cu), option local_form = 1: for N and M
// at or above these (the sort's cost, ~N, against the pair loop's M N)
constexpr size_t kL2SplitBytes = (size_t)48 << 20;
constexpr size_t kHostGatherMax = (size_t)1 << 20;   // GENRED_MEM_HOST inputs gathered into one copy   // j-records per split in the split-major order
constexpr int64_t kLocalMinN = 1 << 18;
constexpr int64_t kLocalMinM = 1 << 16;

// Choose the j-split S so that itiles*S CTAs fill whole waves of `slots` concurrent CTAs.  The
// j-axis has `total` units (512-j tiles, or record pairs split in multiples of `grain`); every
// split keeps at least `min_units`.
int choose_split(int64_t itiles, int64_t total, int64_t grain, int64_t min_units, int64_t slots,
                 double *eff_out, int64_t cap = kMaxSplit, double penalty = 0.002) {
    int best = 1;
    double best_score = -1.0, best_eff = 0.0;
    const int smax = (int)std::min<int64_t>(cap, std::max<int64_t>(1, total / min_units));
    for (int S = 1; S <= smax; ++S) {
        const int64_t per = ((total + S - 1) / S + grain - 1) / grain * grain;
        const int64_t Seff = (total + per - 1) / per;
        if (Seff != S) continue;
        const int64_t U = itiles * S;
        const int64_t waves = (U + slots - 1) / slots;
        const double eff = (double)U / (double)(waves * slots);
        // relative penalty: prefer fewer splits at equal efficiency, but never trade a fuller GPU
        // for fewer splits (an absolute penalty made tiny-M launches pick S = 1: one CTA)
        const double score = eff * (1.0 - penalty * S);
        if (score > best_score + 1e-12) { best_score = score; best = S; best_eff = eff; }
    }
    if (eff_out) *eff_out = best_eff;
    return best;
}

struct Plan {
    int R = 1, split = 1;
    int64_t itiles = 0, ntiles = 0, tiles_per_split = 0;
    int64_t npv = 0, pairs_per_split = 0;     // record-pair splits (Sum, LSE)
};

// pair_splits: the Sum and LSE kernels split j at record-pair granularity (kSplitGrain), so small
// and mid-size problems can spread over all SMs; ArgKMin and LSE_GRAD split whole 512-j tiles.
Plan make_plan(genred_ctx *ctx, const genred_args *a, int kind, int rmax, int occ_kind_a,
               int occ_kind_b, int occ_kind_c, bool pair_splits = false) {
    Plan pl;
    pl.ntiles = (a->N + kTileJ - 1) / kTileJ;
    pl.npv = ((a->N + 1) / 2 + kSplitGrain - 1) / kSplitGrain * kSplitGrain;
    const int64_t total = pair_splits ? pl.npv : pl.ntiles;
    const int64_t grain = pair_splits ? kSplitGrain : 1;
    const int64_t min_units = pair_splits ? kMinSplitPairs : 4;
    int rcands[2] = {rmax, 1};
    int ncand = rmax > 1 ? 2 : 1;
    double best = -1.0;
    for (int ci = 0; ci < ncand; ++ci) {
        const int R = rcands[ci];
        const int64_t rows = (int64_t)kConsumerWarps * 32 * R;
        const int64_t itiles = (a->M + rows - 1) / rows;
        const int64_t slots = (int64_t)ctx->num_sms * occupancy(ctx, kind, occ_kind_a, occ_kind_b, occ_kind_c, R);
        int S;
        double eff;
        const int64_t cap = pair_splits ? kMaxSplitPairs : kMaxSplit;
        if (a->split_j > 0) {
            S = (int)std::min<int64_t>(std::min<int64_t>(a->split_j, cap), std::max<int64_t>(1, total / grain));
            const int64_t U = itiles * S, waves = (U + slots - 1) / slots;
            eff = (double)U / (double)(waves * slots);
        } else {
            // (pair splits: a smaller per-split penalty lets small M spread over many splits)
            S = choose_split(itiles, total, grain, min_units, slots, &eff, cap, pair_splits ? 2e-4 : 0.002);
            if (pair_splits && kind == 0 && kMinWaves > 0 && itiles * S < kMinWaves * slots) {
                // At least kMinWaves waves of CTAs: with one (or two) waves the kernel ends with the
                // slowest SM, while later waves let faster SMs take more CTAs.  Measured at 1e5^2
                // (`profiles/r02_split_sweep.txt`): the Gaussian Sum goes 14.28 (6 splits, 1 wave)
                // -> 14.96 (27) pairs/clk/SM, the fused Sum + grad 13.30 (6) -> 13.79 (27), and
                // 3e5^2 14.99 -> 15.24.  Take the best wave efficiency over [S_min, 2 S_min]
                // (ties: fewer splits), if the j-axis allows it.  Sum family only: an LSE CTA
                // restarts its running max per split (more lazy rescales) and measured slower
                // with more splits (1e5^2: 12.94 -> 12.74).
                const int64_t smax = std::min<int64_t>(cap, std::max<int64_t>(1, total / min_units));
                const int64_t s_lo = (kMinWaves * slots + itiles - 1) / itiles;
                double e_best = 0.0;
                int S_best = S;
                for (int64_t S2 = s_lo; S2 <= std::min<int64_t>(smax, 2 * s_lo); ++S2) {
                    const int64_t per = ((total + S2 - 1) / S2 + grain - 1) / grain * grain;
                    if ((total + per - 1) / per != S2) continue;
                    const int64_t U = itiles * S2, waves = (U + slots - 1) / slots;
                    const double e2 = (double)U / (double)(waves * slots);
                    if (e2 > e_best + 1e-9) { e_best = e2; S_best = (int)S2; }
                }
                if (e_best >= 0.9) { S = S_best; eff = e_best; }
            }
        }
        // fewer rows/thread costs issue slots; rows past M in the last row tile are wasted work
        const double util = (double)a->M / (double)(itiles * rows);
        const double score = eff * util * (R == rmax ? 1.0 : 0.9);
        if (score > best || (a->split_j > 0 && R == rmax)) {
            best = score;
            pl.R = R; pl.split = S; pl.itiles = itiles;
            if (a->split_j > 0) break;                          // forced split: always rmax rows
        }
    }
    if (pair_splits) {
        pl.pairs_per_split = ((pl.npv + pl.split - 1) / pl.split + kSplitGrain - 1) / kSplitGrain * kSplitGrain;
        pl.split = (int)((pl.npv + pl.pairs_per_split - 1) / pl.pairs_per_split);
    } else {
        pl.tiles_per_split = (pl.ntiles + pl.split - 1) / pl.split;
        pl.split = (int)((pl.ntiles + pl.tiles_per_split - 1) / pl.tiles_per_split);
    }
    return pl;
}

// Per-row-tile arrival counters of the in-kernel split merge: zeroed once when allocated, by an
// asynchronous memset on the caller's stream `st` (the stream the merging kernel runs on, which
// may be a non-blocking stream: a legacy-stream memset would not be ordered before it); every
// merging CTA resets its counter, so they are zero again whenever the stream is idle.
genred_status ensure_tile_done(genred_ctx *ctx, int64_t n, cudaStream_t st) {
    if (n <= ctx->tile_done_cap) return GENRED_OK;
    const int64_t cap = std::max<int64_t>(n, 1024);
    if (ctx->tile_done) { cudaFree(ctx->tile_done); ctx->tile_done = nullptr; ctx->tile_done_cap = 0; }
    if (cudaMalloc(&ctx->tile_done, cap * sizeof(unsigned)) != cudaSuccess ||
        cudaMemsetAsync(ctx->tile_done, 0, cap * sizeof(unsigned), st) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, GENRED_E_NOMEM, "split-merge counter allocation failed");
    }
    ctx->tile_done_cap = cap;
    return GENRED_OK;
}

genred_status ensure(genred_ctx *ctx, void **buf, size_t *cap, size_t need) {
    if (buf == &ctx->scratch) ctx->scratch_need = need;
    if (need <= *cap) return GENRED_OK;
    size_t n = std::max(need, *cap + *cap / 2);
    n = (n + 255) & ~size_t(255);
    if (*buf) {
        cudaFree(*buf);
        *buf = nullptr;
        *cap = 0;
    }
    if (cudaMalloc(buf, n) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, GENRED_E_NOMEM, "device scratch allocation of " + std::to_string(n) + " bytes failed");
    }
    *cap = n;
    return GENRED_OK;
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int kMaxProfiled = 4096;

// Event pair around the main kernel (benchmark roofline timing); no-op unless profiling.
// With no_record the event is only returned (the launcher records it around its main kernel).
cudaEvent_t prof_event(genred_ctx *ctx, bool start, cudaStream_t st, bool no_record = false) {
    if (!ctx->profiling || ctx->nprof >= kMaxProfiled) return nullptr;
    const size_t k = (size_t)ctx->nprof * 2 + (start ? 0 : 1);
    while (ctx->ev.size() <= k) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        ctx->ev.push_back(e);
    }
    if (!no_record) cudaEventRecord(ctx->ev[k], st);
    if (!start) ctx->nprof++;
    return ctx->ev[k];
}

genred_status cuda_fail(genred_ctx *ctx, cudaError_t e, const char *where) {
    cudaGetLastError();
    return fail(ctx, GENRED_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Block-sparse ranges (Sum family): gather every cluster's j-intervals into a contiguous,
// tile-padded "range-packed" J, then one CTA per (cluster, row tile) streams only its tiles.
// mode: 0..3 the Sum modes of sum_kernel, 4 = LSE
genred_status eval_ranges(genred_ctx *ctx, const genred_args *a, cudaStream_t st, int mode, int rmax) {
    const int64_t M = a->M, N = a->N;
    const int D = a->D, E = a->E;
    const int out_f64 = a->out_dtype == GENRED_F64;
    const int64_t pairs_per_tile = kTileJ / 2;
    std::vector<RangeCopy> copies;
    std::vector<RangeUnit> units;
    int64_t cursor = 0, rows_total = 0;
    for (int64_t c = 0; c < a->n_ranges; ++c) rows_total += a->ranges_i[2 * c + 1] - a->ranges_i[2 * c];
    const int R = (a->n_ranges > 0 && rows_total / a->n_ranges >= 1024) ? rmax : 1;
    const int64_t RT = (int64_t)kConsumerWarps * 32 * R;
    int64_t s0 = 0;
    for (int64_t c = 0; c < a->n_ranges; ++c) {
        const int64_t is = a->ranges_i[2 * c], ie = a->ranges_i[2 * c + 1], s1 = a->slices[c];
        const int64_t tile0 = cursor / pairs_per_tile;
        for (int64_t k = s0; k < s1; ++k) {
            const int64_t js = a->ranges_j[2 * k], je = a->ranges_j[2 * k + 1];
            if (je <= js) continue;
            copies.push_back({cursor, js, je});
            cursor += (je - js + 1) / 2;
        }
        s0 = s1;
        const int64_t pad = (pairs_per_tile - cursor % pairs_per_tile) % pairs_per_tile;
        if (pad) { copies.push_back({cursor, 0, 0}); cursor += pad; }
        const int64_t ntiles = cursor / pairs_per_tile - tile0;
        if (ntiles == 0) continue;
        for (int64_t r = is; r < ie; r += RT) units.push_back({r, std::min(r + RT, ie), tile0, ntiles});
    }
    copies.push_back({cursor, 0, 0});
    const int pk = mode == 5 ? PACK_ARGKMIN : mode == 4 ? (a->b ? PACK_LSE_H : PACK_LSE_HZ)
                 : mode == 3 ? PACK_SQDIST_SUM : (mode == 1 || mode == 2) ? PACK_GAUSS_AUTO_RAW : PACK_GAUSS_AUTO;
    const int RS = pack_record_stride(pk, D, E);
    const size_t jbytes = al256((size_t)std::max<int64_t>(cursor, 1) * RS * 4);
    const size_t cbytes = al256(copies.size() * sizeof(RangeCopy));
    const size_t ubytes = al256(std::max<size_t>(units.size(), 1) * sizeof(RangeUnit));
    genred_status s = ensure(ctx, &ctx->scratch, &ctx->scratch_cap, jbytes + cbytes + ubytes + 256);
    if (s != GENRED_OK) return s;
    char *base = (char *)ctx->scratch;
    float *J = (float *)base;
    RangeCopy *dcopies = (RangeCopy *)(base + jbytes);
    RangeUnit *dunits = (RangeUnit *)(base + jbytes + cbytes);
    uint32_t *geo = (uint32_t *)(base + jbytes + cbytes + ubytes);
    cudaError_t e = cudaMemcpyAsync(dcopies, copies.data(), copies.size() * sizeof(RangeCopy),
                                    cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && !units.empty())
        e = cudaMemcpyAsync(dunits, units.data(), units.size() * sizeof(RangeUnit), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "range table copy");
    // neutral outputs for every row first; cluster rows are overwritten by the kernel
    const int fill_kind = mode == 5 ? 3 : mode == 4 ? 2 : (mode == 2 ? 1 : 0);
    const int fill_C = mode == 1 ? D : E;
    e = launch_fill(fill_kind, M, fill_C, mode == 5 ? a->K : D, a->out, out_f64, a->out_grad, a->out_idx,
                    a->lse_state, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "fill kernel");
    int kernels = 1;
    float sc = 1.0f;
    double scale_grad = 0.0;
    if (mode != 3 && mode != 4 && mode != 5) {
        sc = (float)(sqrt(kLog2e) / a->scale);
        scale_grad = -2.0 / (a->scale * a->scale * (double)sc);
        e = launch_bbox(a->x, M, a->y, N, D, geo, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "bbox kernel");
        kernels++;
    }
    e = launch_pack_ranges(pk, a->y, a->b, N, D, E, sc, dcopies, (int)copies.size(), cursor, J, st, geo);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "range pack kernel");
    kernels++;
    if (mode == 5) {                                  // ArgKMin: units write their rows' lists directly
        ArgkLaunch L;
        L.D = D; L.K = a->K; L.R = R; L.x = a->x; L.J = J; L.M = M; L.split = 1;
        L.pairs_per_split = 0; L.npv = 0;
        L.dist = (float *)a->out; L.idx = a->out_idx; L.j_offset = a->j_offset;
        L.pdist = nullptr; L.pidx = nullptr;
        L.units = dunits; L.n_units = (int64_t)units.size();
        int ctas = 0;
        if (!units.empty()) {
            prof_event(ctx, true, st);
            e = launch_argk(L, st, &ctas);
            prof_event(ctx, false, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "argkmin kernel (ranges)");
            kernels++;
        }
        ctx->launches += kernels;
        ctx->plan.split_j = 1; ctx->plan.rows_per_cta = (int32_t)RT; ctx->plan.ctas = ctas;
        ctx->plan.kernels = kernels; ctx->plan.path = 0;
        ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
        return GENRED_OK;
    }
    if (mode == 4) {
        LseLaunch L;
        L.D = D; L.R = R; L.x = a->x; L.J = J; L.M = M; L.split = 1; L.pairs_per_split = 0;
        L.npv = 0; L.negc = (float)(-kLog2e / a->scale); L.h_zero = a->b == nullptr;
        L.out = a->out; L.out_f64 = out_f64; L.state = a->lse_state;
        L.units = dunits; L.n_units = (int64_t)units.size();
        int ctas = 0;
        if (!units.empty()) {
            prof_event(ctx, true, st);
            e = launch_lse(L, st, &ctas);
            prof_event(ctx, false, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "lse kernel (ranges)");
            kernels++;
        }
        ctx->launches += kernels;
        ctx->plan.split_j = 1; ctx->plan.rows_per_cta = (int32_t)RT; ctx->plan.ctas = ctas;
        ctx->plan.kernels = kernels; ctx->plan.path = 0;
        ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
        return GENRED_OK;
    }
    SumLaunch L;
    L.num_sms = ctx->num_sms;
    L.mode = mode; L.D = D; L.E = E; L.R = R; L.x = a->x; L.J = J; L.g = a->g; L.M = M;
    L.split = 1; L.pairs_per_split = 0; L.npv = 0; L.s = sc;
    L.scale_sum = 1.0; L.scale_grad = scale_grad; L.out = a->out; L.out_f64 = out_f64;
    L.out_grad = a->out_grad; L.part = nullptr; L.geo = geo;
    L.units = dunits; L.n_units = (int64_t)units.size();
    int ctas = 0;
    if (!units.empty()) {
        prof_event(ctx, true, st);
        e = launch_sum(L, st, &ctas);
        prof_event(ctx, false, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "sum kernel (ranges)");
        kernels++;
    }
    ctx->launches += kernels;
    ctx->plan.split_j = 1; ctx->plan.rows_per_cta = (int32_t)RT; ctx->plan.ctas = ctas;
    ctx->plan.kernels = kernels; ctx->plan.path = 0;
    ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
    ctx->geo_dev = mode != 3 ? geo : nullptr;
    ctx->geo_D = D;
    ctx->geo_s = sc;
    return GENRED_OK;
}

// Device-pointer evaluation (the path itself).
genred_status eval_device(genred_ctx *ctx, const genred_args *a, cudaStream_t st) {
    const int f = a->formula, red = a->reduction;
    const int64_t M = a->M, N = a->N;
    const int D = a->D, E = a->E;
    ctx->plan = genred_plan{};
    ctx->plan.tile_j = kTileJ;
    ctx->geo_dev = nullptr;
    if (M == 0) return GENRED_OK;
    const int out_f64 = a->out_dtype == GENRED_F64;
    cudaError_t e;

    if (N == 0) {                                               // neutral outputs (R11)
        int kind, C = 0, K = 0;
        if (red == GENRED_SUM) {
            if (f == GENRED_GAUSS_SUM_GRADX || f == GENRED_LSE_GRAD) { kind = 1; C = E; K = D; }
            else { kind = 0; C = (f == GENRED_GAUSS_GRADX) ? D : E; }
        } else if (red == GENRED_LSE) kind = 2;
        else { kind = 3; K = a->K; }
        e = launch_fill(kind, M, C, K, a->out, out_f64, a->out_grad, a->out_idx, a->lse_state, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "fill kernel");
        ctx->launches += 1;
        ctx->plan.kernels = 1;
        return GENRED_OK;
    }

    if (f == GENRED_LSE_GRAD) {                                   // LSE backward (8(f) row 2)
        const int rmax = sm_rows_per_thread_max(D);
        Plan pl = make_plan(ctx, a, 3, rmax, D, 0, 0, true);
        const int RS = softmax_record_stride(D);
        const int64_t npairs = pl.ntiles * (kTileJ / 2);
        const int C = 1 + D;
        const size_t jbytes = al256((size_t)npairs * RS * 4);
        const size_t pbytes = pl.split > 1 ? al256((size_t)pl.split * M * C * 8) : 0;
        genred_status s = ensure(ctx, &ctx->scratch, &ctx->scratch_cap, jbytes + pbytes);
        if (s != GENRED_OK) return s;
        float *J = (float *)ctx->scratch;
        double *part = pl.split > 1 ? (double *)((char *)ctx->scratch + jbytes) : nullptr;
        e = launch_pack_softmax(a->y, a->b, a->col_shift, N, D, npairs, J, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "pack kernel");
        SmLaunch L;
        L.D = D; L.R = pl.R; L.x = a->x; L.J = J; L.coef = a->g; L.alpha = a->row_shift; L.M = M;
        L.split = pl.split; L.pairs_per_split = pl.pairs_per_split; L.npv = pl.npv;
        L.negc = (float)(-kLog2e / a->scale); L.scale_grad = -2.0 / a->scale;
        L.out = a->out; L.out_f64 = out_f64; L.out_grad = a->out_grad; L.part = part;
        int ctas = 0;
        prof_event(ctx, true, st);
        e = launch_softmax_grad(L, st, &ctas);
        prof_event(ctx, false, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "softmax-grad kernel");
        int kernels = 2;
        if (pl.split > 1) {
            e = launch_sum_finalize(part, pl.split, M, C, 1, a->g, 1, 1.0, L.scale_grad, 2, a->out,
                                    out_f64, a->out_grad, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "finalize kernel");
            kernels++;
        }
        ctx->launches += kernels;
        ctx->plan.split_j = pl.split; ctx->plan.rows_per_cta = kConsumerWarps * 32 * pl.R;
        ctx->plan.ctas = ctas; ctx->plan.kernels = kernels; ctx->plan.path = 0;
        ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
        return GENRED_OK;
    }

    if (red == GENRED_SUM) {
        const int mode = (f == GENRED_GAUSS) ? 0 : (f == GENRED_GAUSS_GRADX) ? 1
                       : (f == GENRED_GAUSS_SUM_GRADX) ? 2 : 3;
        const int rmax = sum_rows_per_thread_max(mode, D, E);
        if (a->n_ranges > 0) return eval_ranges(ctx, a, st, mode, rmax);
        Plan pl = make_plan(ctx, a, 0, rmax, mode, D, E, true);
        // Small M (north star (a), the warp-shuffle finish): when even one-row-per-thread tiles
        // split as far as j allows cannot fill the GPU, CTAs of a few rows whose 256 threads
        // share the rows and split j take over (sum_smm.cu).  Not for tiny N (edge kernel).
        bool smm = false;
        // (A forced split_j keeps the row-tile kernels, so i-shards of one problem with the same
        // split compute their rows bitwise as the unsharded call does.)
        // (Measured at N = 1e7: the small-M CTAs re-stream the j-records per R = 8 rows, so they
        // pay off only while most threads of a one-row-per-thread tile would idle, M <= 64.)
        if (a->split_j <= 0 && N > kDirectMaxN && M <= kSmmMaxM && sum_smm_supported(mode, D, E))
            smm = true;
        if (smm) {
            const int Rs = sum_smm_rows(mode);
            const int64_t groups = (M + Rs - 1) / Rs;
            const int64_t slots = (int64_t)ctx->num_sms * sum_smm_occupancy(mode, D);
            const int S = choose_split(groups, pl.npv, kSplitGrain, kMinSmmPairs, slots, nullptr, kMaxSplitSmm, 2e-4);
            pl.pairs_per_split = ((pl.npv + S - 1) / S + kSplitGrain - 1) / kSplitGrain * kSplitGrain;
            pl.split = (int)((pl.npv + pl.pairs_per_split - 1) / pl.pairs_per_split);
            pl.R = Rs;
        }
        const int pk = mode == 3 ? PACK_SQDIST_SUM
                     : (mode == 1 || mode == 2) ? PACK_GAUSS_AUTO_RAW : PACK_GAUSS_AUTO;
        const int RS = pack_record_stride(pk, D, E);
        const int64_t npairs = pl.ntiles * (kTileJ / 2);
        const int C = (mode == 1) ? D : (mode == 2) ? E + D : E;
        // Tile-centred form (R18j): y in Hilbert order, records centred per 512-j tile; the device
        // takes it where the global box rules the expanded form out (geo.cuh), tile by tile.  The
        // j-splits then cover whole tiles.
        const bool local = (mode == 0 || ((mode == 1 || mode == 2) && E == 1 && kGradBY && pl.R == 4)) &&
                           !smm && D <= 3 && N > kDirectMaxN && M > kDirectMaxM &&
                           N < ((int64_t)1 << 31) &&
                           (ctx->local_form == 2 || (ctx->local_form == 1 && N >= kLocalMinN && M >= kLocalMinM));
        // Large j-record sets (C5: 240 MB, twice the L2): at least enough j-splits for one split's
        // records to fit kL2SplitBytes, and the CTAs ordered split by split, so the resident
        // CTAs share one split's records in L2 instead of re-streaming them from DRAM per wave.
        const bool split_major = ctx->split_major && !smm && (size_t)npairs * RS * 4 > kL2SplitBytes;
        if (split_major && a->split_j <= 0) {
            const int64_t smin = (int64_t)(((size_t)npairs * RS * 4 + kL2SplitBytes - 1) / kL2SplitBytes);
            if (pl.split < smin) {
                // the best wave efficiency over [smin, 2 smin] (ties: fewer splits), as the
                // planner's wave rule: e.g. an 8-way i-shard of C5 (1221 row tiles, 592 slots)
                // goes from 0.94 at 5 splits to 0.98 at 10
                const int64_t slots = (int64_t)ctx->num_sms * occupancy(ctx, 0, mode, D, E, pl.R);
                const int64_t P = local ? kTileJ / 2 : kSplitGrain;
                double e_best = -1.0;
                int64_t pps_best = 0;
                for (int64_t S2 = smin; S2 <= 2 * smin; ++S2) {
                    const int64_t pps = ((pl.npv + S2 - 1) / S2 + P - 1) / P * P;
                    const int64_t Se = (pl.npv + pps - 1) / pps;
                    if (Se < smin) continue;
                    const int64_t U = pl.itiles * Se, waves = (U + slots - 1) / slots;
                    const double e2 = (double)U / (double)(waves * slots);
                    if (e2 > e_best + 1e-9) { e_best = e2; pps_best = pps; }
                }
                if (pps_best == 0)
                    pps_best = ((pl.npv + smin - 1) / smin + kSplitGrain - 1) / kSplitGrain * kSplitGrain;
                pl.pairs_per_split = pps_best;
                pl.split = (int)((pl.npv + pl.pairs_per_split - 1) / pl.pairs_per_split);
            }
        }
        if (local) {
            const int64_t P = kTileJ / 2;
            pl.pairs_per_split = (pl.pairs_per_split + P - 1) / P * P;
            pl.split = (int)((pl.npv + pl.pairs_per_split - 1) / pl.pairs_per_split);
        }
        const size_t jbytes = al256((size_t)npairs * RS * 4);
        const size_t pbytes = pl.split > 1 ? al256((size_t)pl.split * M * C * 8) : 0;
        const size_t lbytes = local ? al256((size_t)pl.ntiles * 16) + 4 * al256((size_t)N * 4) +
                                      al256(tile_order_temp_bytes(N)) : 0;
        genred_status s = ensure(ctx, &ctx->scratch, &ctx->scratch_cap, jbytes + pbytes + 256 + lbytes);
        if (s != GENRED_OK) return s;
        float *J = (float *)ctx->scratch;
        double *part = pl.split > 1 ? (double *)((char *)ctx->scratch + jbytes) : nullptr;
        uint32_t *geo = (uint32_t *)((char *)ctx->scratch + jbytes + pbytes);
        char *lbase = (char *)ctx->scratch + jbytes + pbytes + 256;
        float4 *centers = local ? (float4 *)lbase : nullptr;
        // parameter folding in fp64, rounded once to fp32 (R15, R18)
        float sc = 1.0f;
        double scale_grad = 0.0;
        if (mode != 3) {
            const double sig = a->scale;
            sc = (float)(sqrt(kLog2e) / sig);                   // 2^(-|s x - s y|^2) = e^(-|x-y|^2/sig^2)
            scale_grad = -2.0 / (sig * sig * (double)sc);        // (x - y) = (x' - y') / s
        }
        int kernels = 2;
        // Tiny N (the HBM-bound edge, SURVEY.md 8(d) Cedge): the pair loop is a few FP32 ops per
        // row, so the direct form is free and the bounding-box pass over x (a second full read
        // of x) is skipped; geo = nullptr selects the direct form on the device.
        const bool tiny_n = N <= kDirectMaxN;
        // Few rows (M <= kDirectMaxM): the pair loop is bound by streaming the j-records, so the
        // direct form costs nothing and the bounding-box pass over y (a full read of y) is skipped.
        const bool no_box = tiny_n || M <= kDirectMaxM;
        if (no_box) geo = nullptr;
        // Small problems in ONE launch (C1-like, launch-latency bound; sum_small_kernel): the CTAs
        // build their own direct-form j-records in shared memory (no pack kernel, no bounding
        // box), and the split partials are merged in the same kernel.  Option "small_fused" = 0
        // keeps the pack + pair-loop path (which may take the expanded form).
        {
            const int64_t tile_rows = (int64_t)kConsumerWarps * 32 * pl.R;
            // split <= 8: the split's CTAs form a cluster and merge through distributed shared
            // memory; else the last-CTA merge through global partials (as sum_kernel)
            const bool merge_ok = pl.split == 1 || (pl.split <= 8 && kSmallCluster) ||
                (pl.split <= 32 && ctx->fused_merge && std::min<int64_t>(tile_rows, M) * C * pl.split <= 16384);
            if (!smm && !tiny_n && E == 1 && D <= 4 && std::max(M, N) <= kFusedBoxMax &&
                pl.pairs_per_split <= kSmallMaxPairs && merge_ok && ctx->small_fused) {
                SumLaunch L;
                L.num_sms = ctx->num_sms;
                L.mode = mode; L.D = D; L.E = E; L.R = pl.R; L.x = a->x; L.J = nullptr; L.g = a->g; L.M = M;
                L.split = pl.split; L.pairs_per_split = pl.pairs_per_split; L.npv = pl.npv; L.s = sc;
                L.scale_sum = 1.0; L.scale_grad = scale_grad; L.out = a->out; L.out_f64 = out_f64;
                L.out_grad = a->out_grad; L.part = part; L.geo = nullptr; L.units = nullptr; L.n_units = 0;
                if (pl.split > 8 || (pl.split > 1 && !kSmallCluster)) {
                    s = ensure_tile_done(ctx, pl.itiles, st);
                    if (s != GENRED_OK) return s;
                    L.tile_done = ctx->tile_done;
                }
                int ctas = 0;
                prof_event(ctx, true, st);
                e = launch_sum_small(L, a->y, a->b, N, st, &ctas);
                prof_event(ctx, false, st);
                if (e != cudaSuccess) return cuda_fail(ctx, e, "small sum kernel");
                ctx->launches += 1;
                ctx->plan.split_j = pl.split; ctx->plan.rows_per_cta = (int32_t)tile_rows;
                ctx->plan.ctas = ctas; ctx->plan.kernels = 1; ctx->plan.path = 0;
                ctx->plan.tile_j = (int32_t)(2 * pl.pairs_per_split);
                ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
                ctx->geo_dev = nullptr;
                return GENRED_OK;
            }
        }
        // small problems: the box is reduced inside the pack kernel (one launch fewer)
        const bool boxed_pack = mode != 3 && !no_box && std::max(M, N) <= kFusedBoxMax && !local;
        if (mode != 3 && !no_box && !boxed_pack) {
            e = launch_bbox(a->x, M, a->y, N, D, geo, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "bbox kernel");
            kernels++;
        }
        int ctas = 0;
        if (local) {
            char *q = lbase + al256((size_t)pl.ntiles * 16);
            const size_t nb = al256((size_t)N * 4);
            uint32_t *keys = (uint32_t *)q, *idx = (uint32_t *)(q + nb), *keys_s = (uint32_t *)(q + 2 * nb),
                     *perm = (uint32_t *)(q + 3 * nb);
            int lk = 0;
            e = launch_tile_order(a->y, a->b, N, D, E, sc, geo, keys, idx, keys_s, perm, q + 4 * nb,
                                  tile_order_temp_bytes(N), pl.ntiles, J, centers, st, &lk, mode == 0 ? 0 : 2);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "tile order / pack kernels");
            kernels += lk - 1;
        } else {
            e = boxed_pack ? launch_pack_boxed(pk, a->y, a->b, N, D, E, sc, npairs, J, a->x, M, geo, st)
                           : launch_pack(pk, a->y, a->b, N, D, E, sc, 0.0, npairs, J, st, geo);
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "pack kernel");
        if (tiny_n && mode == 0 && E == 1 && D <= 4 && N <= sum_edge_max_n() &&
            ((uintptr_t)a->x & 15) == 0) {
            // HBM-bound edge: persistent CTAs, bulk-copied x tiles, j-records resident in smem
            prof_event(ctx, true, st);
            e = launch_sum_edge(a->x, J, N, D, RS, M, sc, 1.0, a->out, out_f64, ctx->num_sms, st, &ctas);
            prof_event(ctx, false, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "edge sum kernel");
            ctx->launches += kernels;
            ctx->plan.split_j = 1; ctx->plan.rows_per_cta = sum_edge_tile_rows(); ctx->plan.ctas = ctas;
            ctx->plan.kernels = kernels; ctx->plan.path = 0; ctx->plan.tile_j = (int32_t)N;
            ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
            ctx->geo_dev = nullptr;
            return GENRED_OK;
        }
        SumLaunch L;
        L.num_sms = ctx->num_sms;
        L.mode = mode; L.D = D; L.E = E; L.R = pl.R; L.x = a->x; L.J = J; L.g = a->g; L.M = M;
        L.split = pl.split; L.pairs_per_split = pl.pairs_per_split; L.npv = pl.npv; L.s = sc;
        L.scale_sum = 1.0; L.scale_grad = scale_grad; L.out = a->out; L.out_f64 = out_f64;
        L.out_grad = a->out_grad; L.part = part; L.geo = geo; L.units = nullptr; L.n_units = 0;
        L.centers = centers;
        L.split_major = split_major ? 1 : 0;
        // Few partials per row tile: the last CTA of each row tile merges them (no finalize
        // launch); the merge tail is bounded at 16 K fp64 reads for that CTA.  Only up to 32
        // splits: above that the finalize kernel sums lane-strided (sum_finalize_warp_kernel),
        // and the fused merge must give bitwise its result (i-shards of one problem may take
        // either path).
        const int64_t tile_rows = (int64_t)kConsumerWarps * 32 * pl.R;
        const bool fused_merge = pl.split > 1 && pl.split <= 32 && !smm && ctx->fused_merge &&
                                 std::min<int64_t>(tile_rows, M) * C * pl.split <= 16384;
        if (fused_merge) {
            s = ensure_tile_done(ctx, pl.itiles, st);
            if (s != GENRED_OK) return s;
            L.tile_done = ctx->tile_done;
        }
        int sctas = 0;
        prof_event(ctx, true, st);
        e = smm ? launch_sum_smm(L, st, &sctas) : launch_sum(L, st, &sctas);
        prof_event(ctx, false, st);
        ctas = sctas;
        if (e != cudaSuccess) return cuda_fail(ctx, e, "sum kernel");
        if (pl.split > 1 && !fused_merge) {
            const int cols_sum = (mode == 1) ? 0 : E;
            e = launch_sum_finalize(part, pl.split, M, C, cols_sum, a->g, E, 1.0, scale_grad, mode,
                                    a->out, out_f64, a->out_grad, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "sum finalize kernel");
            kernels++;
        }
        ctx->launches += kernels;
        ctx->plan.split_j = pl.split; ctx->plan.rows_per_cta = smm ? pl.R : kConsumerWarps * 32 * pl.R;
        ctx->plan.ctas = ctas; ctx->plan.kernels = kernels; ctx->plan.path = local ? 3 : 0;
        ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
        ctx->centers_dev = centers;
        ctx->centers_n = local ? pl.ntiles : 0;
        ctx->geo_dev = mode != 3 ? geo : nullptr;
        ctx->geo_D = D;
        ctx->geo_s = sc;
        return GENRED_OK;
    }

    if (red == GENRED_LSE) {
        if (a->n_ranges > 0) return eval_ranges(ctx, a, st, 4, lse_rows_per_thread_max(D));
        Plan pl = make_plan(ctx, a, 1, lse_rows_per_thread_max(D), D, a->b == nullptr ? 1 : 0, 0, true);
        // small M: CTAs of a few rows whose threads split j (see the Sum path)
        const bool smm = a->split_j <= 0 && M <= kSmmMaxM && N > kDirectMaxN;
        if (smm) {
            const int Rs = lse_smm_rows(D);
            const int64_t groups = (M + Rs - 1) / Rs;
            const int S = choose_split(groups, pl.npv, kSplitGrain, kMinSmmPairs, (int64_t)ctx->num_sms * 2,
                                       nullptr, kMaxSplitSmm, 2e-4);
            pl.pairs_per_split = ((pl.npv + S - 1) / S + kSplitGrain - 1) / kSplitGrain * kSplitGrain;
            pl.split = (int)((pl.npv + pl.pairs_per_split - 1) / pl.pairs_per_split);
            pl.R = Rs;
        }
        const int pk = a->b ? PACK_LSE_H : PACK_LSE_HZ;
        // Tile-centred form (R18j): as the Gaussian Sum's, with the LSE's own radius bound
        const bool local = !smm && D <= 3 && pl.R == 4 && N > kDirectMaxN && M > kDirectMaxM &&
                           N < ((int64_t)1 << 31) &&
                           (ctx->local_form == 2 || (ctx->local_form == 1 && N >= kLocalMinN && M >= kLocalMinM));
        if (local) {
            const int64_t P = kTileJ / 2;
            pl.pairs_per_split = (pl.pairs_per_split + P - 1) / P * P;
            pl.split = (int)((pl.npv + pl.pairs_per_split - 1) / pl.pairs_per_split);
        }
        const int RS = local ? lse_local_record_stride(D, a->b == nullptr) : pack_record_stride(pk, D, 1);
        const int64_t npairs = pl.ntiles * (kTileJ / 2);
        const size_t jbytes = al256((size_t)npairs * RS * 4);
        const size_t pbytes = pl.split > 1 ? al256((size_t)pl.split * M * 2 * 8) : 0;
        const size_t lbytes = local ? 256 + al256((size_t)pl.ntiles * 16) + 4 * al256((size_t)N * 4) +
                                      al256(tile_order_temp_bytes(N)) : 0;
        genred_status s = ensure(ctx, &ctx->scratch, &ctx->scratch_cap, jbytes + pbytes + lbytes);
        if (s != GENRED_OK) return s;
        float *J = (float *)ctx->scratch;
        double *part = pl.split > 1 ? (double *)((char *)ctx->scratch + jbytes) : nullptr;
        float4 *centers = nullptr;
        const float sl = (float)sqrt(kLog2e / a->scale);     // s units of the tile-centred form
        int kernels = 2;
        if (local) {
            char *lb = (char *)ctx->scratch + jbytes + pbytes;
            uint32_t *geo = (uint32_t *)lb;
            centers = (float4 *)(lb + 256);
            char *q = lb + 256 + al256((size_t)pl.ntiles * 16);
            const size_t nb = al256((size_t)N * 4);
            e = launch_bbox(a->x, M, a->y, N, D, geo, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "bbox kernel");
            int lk = 0;
            e = launch_tile_order(a->y, a->b, N, D, 1, sl, geo, (uint32_t *)q, (uint32_t *)(q + nb),
                                  (uint32_t *)(q + 2 * nb), (uint32_t *)(q + 3 * nb), q + 4 * nb,
                                  tile_order_temp_bytes(N), pl.ntiles, J, centers, st, &lk, 1, RS, kLog2e,
                                  kLseLocalR2Max);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "tile order / pack kernels");
            kernels += lk;                               // bbox + keys + sort + pack (pack counted in 2)
        } else {
            e = launch_pack(pk, a->y, a->b, N, D, 1, 1.0f, kLog2e, npairs, J, st);
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "pack kernel");
        LseLaunch L;
        L.centers = centers; L.s = sl;
        L.D = D; L.R = pl.R; L.x = a->x; L.J = J; L.M = M; L.split = pl.split;
        L.pairs_per_split = pl.pairs_per_split; L.npv = pl.npv;
        L.negc = (float)(-kLog2e / a->scale);
        L.h_zero = a->b == nullptr;
        L.out = a->out; L.out_f64 = out_f64;
        L.state = pl.split > 1 ? part : a->lse_state;
        int ctas = 0;
        prof_event(ctx, true, st);
        e = smm ? launch_lse_smm(L, st, &ctas) : launch_lse(L, st, &ctas);
        prof_event(ctx, false, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "lse kernel");
        if (pl.split > 1) {
            e = launch_lse_finalize(part, pl.split, M, a->out, out_f64, a->lse_state, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "lse finalize kernel");
            kernels++;
        }
        ctx->launches += kernels;
        ctx->plan.split_j = pl.split; ctx->plan.rows_per_cta = smm ? pl.R : kConsumerWarps * 32 * pl.R;
        ctx->plan.ctas = ctas; ctx->plan.kernels = kernels; ctx->plan.path = local ? 3 : 0;
        ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
        ctx->centers_dev = centers;
        ctx->centers_n = local ? pl.ntiles : 0;
        ctx->geo_dev = nullptr;
        return GENRED_OK;
    }

    // ArgKMin with block-sparse ranges (small D; validated)
    if (a->n_ranges > 0) return eval_ranges(ctx, a, st, 5, argk_rows_per_thread(a->K));

    // ArgKMin, large D: tcgen05 3xTF32 screening + exact re-rank (knn_tc.cu)
    if (D > 16) {
        const size_t need = knn_tc_scratch_bytes(M, N, D, a->K) + 1024;
        genred_status s = ensure(ctx, &ctx->scratch, &ctx->scratch_cap, need);
        if (s != GENRED_OK) return s;
        KnnTcLaunch L;
        L.x = a->x; L.y = a->y; L.M = M; L.N = N; L.D = D; L.K = a->K;
        L.dist = (float *)a->out; L.idx = a->out_idx; L.j_offset = a->j_offset;
        L.scratch = (void *)(((uintptr_t)ctx->scratch + 1023) & ~(uintptr_t)1023);
        L.num_sms = ctx->num_sms;
        L.ev_start = prof_event(ctx, true, nullptr, true);
        L.ev_stop = prof_event(ctx, false, nullptr, true);
        KnnTcInfo info{};
        e = launch_knn_tc(L, st, &info);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "tensor-core k-NN");
        ctx->launches += info.kernels;
        ctx->fallback_dev = info.fallback_count;
        ctx->plan.split_j = 1; ctx->plan.rows_per_cta = 128; ctx->plan.ctas = info.ctas;
        ctx->plan.kernels = info.kernels; ctx->plan.path = 1; ctx->plan.tile_j = 256;
        ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
        return GENRED_OK;
    }

    // ArgKMin, small D, FP32 path
    const int K = a->K;
    const int R = argk_rows_per_thread(K);
    Plan pl = make_plan(ctx, a, 2, R, D, K, 0, true);
    // small M: one row per CTA, its threads split j (see the Sum path)
    const bool smm = a->split_j <= 0 && M <= kSmmMaxM && N > kDirectMaxN;
    if (smm) {
        const int S = choose_split(M, pl.npv, kSplitGrain, kMinSmmPairs, (int64_t)ctx->num_sms, nullptr,
                                   kMaxSplitSmm, 2e-4);
        pl.pairs_per_split = ((pl.npv + S - 1) / S + kSplitGrain - 1) / kSplitGrain * kSplitGrain;
        pl.split = (int)((pl.npv + pl.pairs_per_split - 1) / pl.pairs_per_split);
        pl.R = 1;
    }
    const int RS = pack_record_stride(PACK_ARGKMIN, D, 0);
    const int64_t npairs = pl.ntiles * (kTileJ / 2);
    const size_t jbytes = al256((size_t)npairs * RS * 4);
    const size_t pdb = pl.split > 1 ? al256((size_t)pl.split * M * K * 4) : 0;
    const int G1 = pl.split > 64 ? (pl.split + 63) / 64 : 0;        // two-level merge above 64 lists
    const size_t gdb = G1 ? al256((size_t)G1 * M * K * 4) : 0;
    genred_status s = ensure(ctx, &ctx->scratch, &ctx->scratch_cap, jbytes + 2 * pdb + 2 * gdb);
    if (s != GENRED_OK) return s;
    float *J = (float *)ctx->scratch;
    float *pdist = pl.split > 1 ? (float *)((char *)ctx->scratch + jbytes) : nullptr;
    int32_t *pidx = pl.split > 1 ? (int32_t *)((char *)ctx->scratch + jbytes + pdb) : nullptr;
    float *gdist = G1 ? (float *)((char *)ctx->scratch + jbytes + 2 * pdb) : nullptr;
    int32_t *gidx = G1 ? (int32_t *)((char *)ctx->scratch + jbytes + 2 * pdb + gdb) : nullptr;
    e = launch_pack(PACK_ARGKMIN, a->y, nullptr, N, D, 0, 1.0f, 0.0, npairs, J, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "pack kernel");
    ArgkLaunch L;
    L.D = D; L.K = K; L.R = pl.R; L.x = a->x; L.J = J; L.M = M; L.split = pl.split;
    L.pairs_per_split = pl.pairs_per_split; L.npv = pl.npv;
    L.dist = (float *)a->out; L.idx = a->out_idx; L.j_offset = a->j_offset;
    L.pdist = pdist; L.pidx = pidx;
    int ctas = 0;
    prof_event(ctx, true, st);
    e = smm ? launch_argk_smm(L, st, &ctas) : launch_argk(L, st, &ctas);
    prof_event(ctx, false, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "argkmin kernel");
    int kernels = 2;
    if (G1) {
        e = launch_topk_merge_groups(pdist, pidx, pl.split, M, K, gdist, gidx, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "top-k group merge kernel");
        e = launch_topk_merge_i32(gdist, gidx, G1, M, K, (float *)a->out, a->out_idx, a->j_offset, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "top-k merge kernel");
        kernels += 2;
    } else if (pl.split > 1) {
        e = launch_topk_merge_i32(pdist, pidx, pl.split, M, K, (float *)a->out, a->out_idx,
                                  a->j_offset, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "top-k merge kernel");
        kernels++;
    }
    ctx->launches += kernels;
    ctx->plan.split_j = pl.split; ctx->plan.rows_per_cta = smm ? 1 : kConsumerWarps * 32 * pl.R;
    ctx->plan.ctas = ctas; ctx->plan.kernels = kernels; ctx->plan.path = 0;
    ctx->plan.scratch_bytes = (int64_t)ctx->scratch_need;
    return GENRED_OK;
}

// Byte sizes of every operand, for host-pointer staging.
struct Sizes {
    size_t x, y, b, g, out, grad, idx, state, rs, cs;
};
Sizes operand_sizes(const genred_args *a) {
    Sizes z{};
    const size_t M = (size_t)a->M, N = (size_t)a->N;
    z.x = M * a->D * 4;
    z.y = N * a->D * 4;
    const bool lse = a->reduction == GENRED_LSE, argk = a->reduction == GENRED_ARGKMIN;
    const bool smg = a->formula == GENRED_LSE_GRAD;
    z.b = a->b ? ((lse || smg) ? N * 4 : N * a->E * 4) : 0;
    z.rs = a->row_shift ? M * 8 : 0;
    z.cs = a->col_shift ? N * 8 : 0;
    z.g = a->g ? M * a->E * 4 : 0;
    const size_t es = a->out_dtype == GENRED_F64 ? 8 : 4;
    if (argk) z.out = M * a->K * 4;
    else if (lse || smg) z.out = M * es;
    else if (a->formula == GENRED_GAUSS_GRADX) z.out = M * a->D * es;
    else z.out = M * a->E * es;
    z.grad = (a->formula == GENRED_GAUSS_SUM_GRADX || smg) ? M * a->D * 4 : 0;
    z.idx = argk ? M * a->K * 8 : 0;
    z.state = (lse && a->lse_state) ? M * 16 : 0;
    return z;
}

}  // namespace

extern "C" {

int32_t genred_abi_version(void) { return GENRED_ABI_VERSION; }

#define GENRED_STR2(x) #x
#define GENRED_STR(x) GENRED_STR2(x)
const char *genred_build_info(void) {
    return "libgenred abi=" GENRED_STR(GENRED_ABI_VERSION) " target=sm_100a (compute_100a) nvcc "
           GENRED_STR(__CUDACC_VER_MAJOR__) "." GENRED_STR(__CUDACC_VER_MINOR__);
}

genred_status genred_create(int32_t cuda_device, genred_ctx **out) {
    if (!out) return GENRED_E_INVALID;
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return GENRED_E_CUDA;
    }
    if (cuda_device < 0 || cuda_device >= n) return GENRED_E_INVALID;
    genred_ctx *ctx = new (std::nothrow) genred_ctx();
    if (!ctx) return GENRED_E_NOMEM;
    ctx->device = cuda_device;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(cuda_device);
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
    if (const char *v = getenv("GENRED_SMALL_FUSED")) ctx->small_fused = atoi(v) != 0;
    if (const char *v = getenv("GENRED_FUSED_MERGE")) ctx->fused_merge = atoi(v) != 0;
    if (const char *v = getenv("GENRED_LOCAL_FORM")) ctx->local_form = atoi(v);
    if (const char *v = getenv("GENRED_SPLIT_MAJOR")) ctx->split_major = atoi(v) != 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cuda_device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, cuda_device);
    cudaSetDevice(prev);
    if (major != 10 || minor != 0) {
        delete ctx;
        return GENRED_E_UNSUPPORTED;                            // sm_100a code only
    }
    *out = ctx;
    return GENRED_OK;
}

void genred_destroy(genred_ctx *ctx) {
    if (!ctx) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->stage) cudaFree(ctx->stage);
    if (ctx->hstage) cudaFreeHost(ctx->hstage);
    if (ctx->tile_done) cudaFree(ctx->tile_done);
    for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
    cudaSetDevice(prev);
    delete ctx;
}

const char *genred_last_error(const genred_ctx *ctx) {
    return ctx ? ctx->err.c_str() : "null context";
}

genred_status genred_validate(const genred_args *args, char *msg, size_t msg_len) {
    std::string m;
    genred_status s = validate(args, m);
    if (msg && msg_len) {
        strncpy(msg, m.c_str(), msg_len - 1);
        msg[msg_len - 1] = 0;
    }
    return s;
}

genred_status genred_eval(genred_ctx *ctx, const genred_args *args, void *stream) {
    if (!ctx) return GENRED_E_INVALID;
    std::string m;
    genred_status s = validate(args, m);
    if (s != GENRED_OK) return fail(ctx, s, m);
    ctx->err.clear();
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (args->memory == GENRED_MEM_DEVICE) {
        s = eval_device(ctx, args, st);
    } else {
        // Host pointers: stage through context-owned device buffers, H2D -> eval -> D2H.
        Sizes z = operand_sizes(args);
        size_t off[10], tot = 0;
        size_t sz[10] = {z.x, z.y, z.b, z.g, z.out, z.grad, z.idx, z.state, z.rs, z.cs};
        for (int k = 0; k < 10; ++k) { off[k] = tot; tot += al256(sz[k]); }
        s = ensure(ctx, &ctx->stage, &ctx->stage_cap, tot + 256);
        if (s == GENRED_OK) {
            char *base = (char *)ctx->stage;
            genred_args d = *args;
            d.memory = GENRED_MEM_DEVICE;
            const void *src[6] = {args->x, args->y, args->b, args->g, args->row_shift, args->col_shift};
            const void **dst[6] = {(const void **)&d.x, (const void **)&d.y, (const void **)&d.b,
                                   (const void **)&d.g, (const void **)&d.row_shift,
                                   (const void **)&d.col_shift};
            const int slot[6] = {0, 1, 2, 3, 8, 9};
            // Small inputs (C1-like: launch-latency bound) are gathered on the host into a pinned
            // buffer with the device layout and sent by ONE copy; large ones go one copy each.
            size_t in_bytes = 0, in_end = 0;
            for (int k = 0; k < 6; ++k)
                if (src[k] && sz[slot[k]] > 0) { in_bytes += sz[slot[k]]; in_end = off[slot[k]] + sz[slot[k]]; }
            bool gathered = false;
            if (in_bytes > 0 && in_bytes <= kHostGatherMax) {
                if (ctx->hstage_cap < in_end) {
                    if (ctx->hstage) { cudaFreeHost(ctx->hstage); ctx->hstage = nullptr; ctx->hstage_cap = 0; }
                    const size_t cap = std::max<size_t>(in_end, (size_t)1 << 20);
                    if (cudaMallocHost(&ctx->hstage, cap) == cudaSuccess) ctx->hstage_cap = cap;
                    else { cudaGetLastError(); ctx->hstage = nullptr; }
                }
                if (ctx->hstage) {
                    for (int k = 0; k < 6; ++k) {
                        if (!src[k] || sz[slot[k]] == 0) continue;
                        *dst[k] = base + off[slot[k]];
                        memcpy((char *)ctx->hstage + off[slot[k]], src[k], sz[slot[k]]);
                    }
                    cudaError_t e = cudaMemcpyAsync(base, ctx->hstage, in_end, cudaMemcpyHostToDevice, st);
                    if (e != cudaSuccess) s = cuda_fail(ctx, e, "H2D copy");
                    gathered = true;
                }
            }
            for (int k = 0; k < 6 && s == GENRED_OK && !gathered; ++k) {
                if (!src[k] || sz[slot[k]] == 0) continue;
                *dst[k] = base + off[slot[k]];
                cudaError_t e = cudaMemcpyAsync(base + off[slot[k]], src[k], sz[slot[k]], cudaMemcpyHostToDevice, st);
                if (e != cudaSuccess) s = cuda_fail(ctx, e, "H2D copy");
            }
            d.out = args->out ? base + off[4] : nullptr;
            d.out_grad = args->out_grad ? (float *)(base + off[5]) : nullptr;
            d.out_idx = args->out_idx ? (int64_t *)(base + off[6]) : nullptr;
            d.lse_state = args->lse_state ? (double *)(base + off[7]) : nullptr;
            if (s == GENRED_OK) s = eval_device(ctx, &d, st);
            void *hdst[4] = {args->out, args->out_grad, args->out_idx, args->lse_state};
            const void *dsrc[4] = {d.out, d.out_grad, d.out_idx, d.lse_state};
            size_t dsz[4] = {z.out, z.grad, z.idx, z.state};
            for (int k = 0; k < 4 && s == GENRED_OK; ++k) {
                if (!hdst[k] || dsz[k] == 0) continue;
                cudaError_t e = cudaMemcpyAsync(hdst[k], dsrc[k], dsz[k], cudaMemcpyDeviceToHost, st);
                if (e != cudaSuccess) s = cuda_fail(ctx, e, "D2H copy");
            }
            if (s == GENRED_OK) {
                cudaError_t e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) s = cuda_fail(ctx, e, "stream synchronize");
            }
        }
    }
    if (prev != ctx->device) cudaSetDevice(prev);
    return s;
}

genred_status genred_combine_lse(genred_ctx *ctx, int64_t M, int32_t G, const double *states,
                                 void *out, int32_t out_dtype, double *state_out, void *stream) {
    if (!ctx) return GENRED_E_INVALID;
    if (M < 0 || G < 1) return fail(ctx, GENRED_E_SHAPE, "M >= 0 and G >= 1 required");
    if (M > 0 && (!states || (!out && !state_out))) return fail(ctx, GENRED_E_INVALID, "null pointer");
    if (out_dtype != GENRED_F32 && out_dtype != GENRED_F64) return fail(ctx, GENRED_E_INVALID, "bad out_dtype");
    if (M == 0) return GENRED_OK;
    cudaError_t e = launch_lse_finalize(states, G, M, out, out_dtype == GENRED_F64, state_out,
                                        (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "combine_lse kernel");
    ctx->launches += 1;
    return GENRED_OK;
}

genred_status genred_merge_topk(genred_ctx *ctx, int64_t M, int32_t K, int32_t G, const float *d,
                                const int64_t *idx, float *d_out, int64_t *idx_out, void *stream) {
    if (!ctx) return GENRED_E_INVALID;
    if (M < 0 || K < 1 || G < 1) return fail(ctx, GENRED_E_SHAPE, "M >= 0, K >= 1, G >= 1 required");
    if (G > 64 || K > 1024) return fail(ctx, GENRED_E_UNSUPPORTED, "merge_topk supports G <= 64");
    if (M > 0 && (!d || !idx || !d_out || !idx_out)) return fail(ctx, GENRED_E_INVALID, "null pointer");
    if (M == 0) return GENRED_OK;
    cudaError_t e = launch_topk_merge_i64(d, idx, G, M, K, d_out, idx_out, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "merge_topk kernel");
    ctx->launches += 1;
    return GENRED_OK;
}

genred_status genred_last_plan(const genred_ctx *ctx, genred_plan *plan) {
    if (!ctx || !plan) return GENRED_E_INVALID;
    *plan = ctx->plan;
    plan->fallback_rows = -1;
    if ((ctx->plan.path == 0 || ctx->plan.path == 3) && ctx->geo_dev &&
        geo_expanded_host(ctx->geo_dev, ctx->geo_D, ctx->geo_s))
        plan->path = 2;                                        // expanded form (global box)
    if (ctx->plan.path == 1 && ctx->fallback_dev) {
        int n = -1;
        if (cudaMemcpy(&n, ctx->fallback_dev, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return GENRED_E_CUDA;
        }
        plan->fallback_rows = n;
    }
    return GENRED_OK;
}

int64_t genred_launch_count(const genred_ctx *ctx) { return ctx ? ctx->launches : 0; }

genred_status genred_last_tiles(const genred_ctx *ctx, int64_t *local_tiles, int64_t *tiles) {
    if (!ctx || !local_tiles || !tiles) return GENRED_E_INVALID;
    *local_tiles = 0;
    *tiles = ctx->plan.path == 3 ? ctx->centers_n : 0;
    if (ctx->plan.path != 3 || !ctx->centers_dev || ctx->centers_n == 0) return GENRED_OK;
    std::vector<float4> h((size_t)ctx->centers_n);
    if (cudaMemcpy(h.data(), ctx->centers_dev, h.size() * sizeof(float4), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return GENRED_E_CUDA;
    }
    for (const float4 &c : h) *local_tiles += c.w >= 0.0f;
    return GENRED_OK;
}

genred_status genred_profile(genred_ctx *ctx, int32_t enable) {
    if (!ctx) return GENRED_E_INVALID;
    ctx->profiling = enable != 0;
    ctx->nprof = 0;
    // create the first 1024 (start, stop) pairs now: cudaEventCreate inside a caller's timed
    // region would add host latency to launch-bound calls (C1)
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    while (ctx->profiling && ctx->ev.size() < 2048) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); break; }
        ctx->ev.push_back(e);
    }
    if (prev != ctx->device) cudaSetDevice(prev);
    return GENRED_OK;
}

genred_status genred_set_option(genred_ctx *ctx, const char *name, int64_t value) {
    if (!ctx || !name) return GENRED_E_INVALID;
    const std::string n(name);
    if (n == "small_fused") { ctx->small_fused = value != 0; return GENRED_OK; }
    if (n == "fused_merge") { ctx->fused_merge = value != 0; return GENRED_OK; }
    if (n == "split_major") { ctx->split_major = value != 0; return GENRED_OK; }
    if (n == "local_form") {
        if (value < 0 || value > 2) return fail(ctx, GENRED_E_INVALID, "local_form is 0, 1 or 2");
        ctx->local_form = (int)value;
        return GENRED_OK;
    }
    return fail(ctx, GENRED_E_INVALID, "unknown option '" + n + "'");
}

int32_t genred_profile_read(genred_ctx *ctx, float *ms, int32_t max) {
    if (!ctx || (!ms && max > 0)) return -1;
    int n = std::min(ctx->nprof, (int)max);
    for (int k = 0; k < n; ++k) {
        if (cudaEventSynchronize(ctx->ev[2 * k + 1]) != cudaSuccess ||
            cudaEventElapsedTime(&ms[k], ctx->ev[2 * k], ctx->ev[2 * k + 1]) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
    }
    return n;
}

}  // extern "C"
