// sum_kernel.cu -- Genred Sum reductions on the FP32 + MUFU pipes:
//
//   GAUSS       a_i   = sum_j exp(-|x_i - y_j|^2 / sigma^2) b_j           (Eq. 1)
//   GAUSS_GRADX G_i   = sum_j (-2/sigma^2)(x_i - y_j) e_ij <b_j, g_i>
//   SUM_GRADX   both in one pass (shares the distance and the exponential)
//   SQDIST_SUM  a_i   = sum_j |x_i - y_j|^2 b_j                           (test combination)
//
// Design (B200-first; the paper's GPU Gems "tiled map-reduce", is prior art):
//   * one CTA owns 256*R i-rows, kept in registers (R rows per math thread), and one j-range;
//   * a producer warp streams j-tiles (512 records, pair-interleaved, pre-scaled by
//     s = sqrt(log2 e)/sigma so that exp(-|x-y|^2/sigma^2) = 2^(-|x'-y'|^2)) from HBM/L2 into a
//     4-stage shared-memory ring with cp.async.bulk (TMA engine) completing on mbarriers;
//   * math warps read each record pair once per thread (broadcast LDS.128) and evaluate two j's
//     at a time with packed FADD2/FMUL2/FFMA2 and two MUFU.EX2 (ex2.approx.ftz), so a pair costs
//     3.5 issue slots of FP32 work + 1 MUFU for D=3 (the MUFU pipe, 16/clk/SM, is the bound);
//   * per-tile fp32 partials are promoted to fp64 every 512 j (reading R18 in DESIGN.md);
//   * j-splits (grid = i-tiles x splits) fill all 148 SMs; their fp64 partials are merged in a
//     fixed order by sum_finalize (deterministic, no float atomics).
#include <math.h>
#include <stdlib.h>

#include "device.cuh"
#include "geo.cuh"
#include "internal.h"

namespace genred {

// Rows per thread of the gradient modes for D + E <= 4: 2 rows at 3 CTAs/SM measured 10.74
// pairs/clk/SM against 10.48 for 4 rows at 2 CTAs/SM (fused Sum+grad, M = N = 1e5).
#ifndef GENRED_GRAD_R
#define GENRED_GRAD_R 2
#endif
#ifndef GENRED_GRAD_HH
#define GENRED_GRAD_HH 2
#endif

template <int MODE, int D, int E>
struct SumCfg {
    // record pair: 2D coordinates, then (MODE 0 only) the pair slot of w = -|y'|^2 used by the
    // expanded form, then 2E signal values; padded to a multiple of 16 bytes
    static constexpr int BOFF = (MODE != 3) ? 2 * (D + 1) : 2 * D;
    static constexpr int RS = ((BOFF + 2 * E) + 3) / 4 * 4;       // floats per record pair
    static constexpr int PAIRS = kTileJ / 2;
    static constexpr int TILE_FLOATS = PAIRS * RS;
    static constexpr int NS = (MODE == 1) ? 0 : E;                // sum columns
    static constexpr int NG = (MODE == 1 || MODE == 2) ? D : 0;   // gradient columns
    static constexpr int C = NS + NG;
    static constexpr bool GRAD = NG > 0;
    static constexpr bool EXP = MODE != 3;
    static constexpr int SMEM = JRing<kStages>::smem_bytes(TILE_FLOATS);
};

struct SumParams {
    const float *x, *J, *g;
    const uint32_t *geo;      // Gaussian modes: encoded bounding box (geo.cuh)
    int64_t M;
    int split;
    int64_t pairs_per_split;  // j-split length in record pairs (a multiple of kSplitGrain)
    int64_t npv;              // record pairs to reduce: ceil(N/2) rounded up to kSplitGrain
    float s;
    double scale_sum, scale_grad;
    void *out;
    int out_f64;
    float *out_grad;
    double *part;
    const RangeUnit *units;   // block-sparse ranges: one CTA per unit (rows of one cluster)
    int direct_only;          // MODE 0: exit when the expanded form applies (gauss_tc.cu runs)
};

// Moving 1/8 (1/4) of the exps to the FP32 pipe measured 14.74 (13.73) pairs/clk/SM against
// 14.90 with every exp on MUFU (M = N = 1e6, B200): the packed FFMA2s of the expanded form read
// three register pairs and already load the FP32 pipe close to the MUFU time, so the share is off.
constexpr bool kPolyShare = false;

// The pair loop + epilogue.  XP selects the expanded form of the Gaussian Sum (MODE 0 only):
//   exp(-|x-y|^2/sigma^2) = 2^(-|x'|^2) * 2^(u),  u = 2 x'.y' - |y'|^2,  x' = s (x - c)
// so a pair costs 3 FFMA (u, packed over two j's) + exp + 1 FFMA instead of 7 FP32 ops, which
// leaves the MUFU pipe (16 ex2/clk/SM) as the only bound; the row factor 2^(-|x'|^2) is applied
// in fp64 at the end.
template <int MODE, int D, int E, int R, bool XP>
__device__ __forceinline__ void sum_body(const SumParams &p, JRing<kStages> &ring, int nt, int last_np,
                                         int64_t row0, int64_t row_end, int sp, const Geo &geo) {
    using Cfg = SumCfg<MODE, D, E>;
    constexpr int RS = Cfg::RS, NS = Cfg::NS, NG = Cfg::NG, C = Cfg::C, BOFF = Cfg::BOFF;
    constexpr bool POLY = kPolyShare && XP && R == 4;
    constexpr int HH = (MODE == 1 || MODE == 2) ? GENRED_GRAD_HH : 2;   // record pairs per iteration
    const int ct = threadIdx.x;
    float xr[R][D];
    float gr[R][E];
    double xsq[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        const bool ok = i < row_end;
        xsq[r] = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const float v = ok ? __ldg(p.x + i * D + d) : 0.0f;
            if constexpr (XP) {
                const float xs = ok ? p.s * (v - geo.c[d]) : 0.0f;        // x' = s (x - c)
                xsq[r] += (double)xs * (double)xs;
                xr[r][d] = 2.0f * xs;                                      // exact doubling
            } else {
                xr[r][d] = p.s * v;
            }
        }
#pragma unroll
        for (int e = 0; e < E; ++e)
            gr[r][e] = (Cfg::GRAD && E > 1 && ok && p.g) ? __ldg(p.g + i * E + e) : 1.0f;
    }
    float2 acc[R][NS > 0 ? NS : 1];
    float2 accg[R][NG > 0 ? NG : 1];
    double acc64[R][C];
    // expanded gradient: G_i ~ x'_i S0_i - S_i with S0 = sum_j w_ij, S = sum_j w_ij y'_j; S0 is the
    // Sum itself when MODE == 2 and E == 1 (w = e b), else it has its own accumulator
    constexpr bool OWN_S0 = XP && NG > 0 && !(MODE == 2 && E == 1);
    float2 s0[R];
    double s064[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        s0[r] = make_float2(0.f, 0.f);
        s064[r] = 0.0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int c = 0; c < C; ++c) acc64[r][c] = 0.0;
#pragma unroll
        for (int c = 0; c < (NS > 0 ? NS : 1); ++c) acc[r][c] = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < (NG > 0 ? NG : 1); ++c) accg[r][c] = make_float2(0.f, 0.f);
    }

    for (int k = 0; k < nt; ++k) {
        const float *tile = ring.acquire(k);
        // record pairs of this tile: whole tiles, except the range's last one (a multiple of
        // kSplitGrain, so of HH)
        const int np = k == nt - 1 ? last_np : Cfg::PAIRS;
        for (int pp2 = 0; pp2 < np; pp2 += HH) {
#pragma unroll
        for (int hh = 0; hh < HH; ++hh) {
            const int pp = pp2 + hh;
            float f[RS];
#pragma unroll
            for (int q = 0; q < RS / 4; ++q) {
                const float4 v = lds128(tile + pp * RS + 4 * q);
                f[4 * q + 0] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
            }
            float2 ny[D], bv[E];
#pragma unroll
            for (int d = 0; d < D; ++d) ny[d] = make_float2(f[2 * d], f[2 * d + 1]);
#pragma unroll
            for (int e = 0; e < E; ++e) bv[e] = make_float2(f[BOFF + 2 * e], f[BOFF + 2 * e + 1]);
            if constexpr (XP) {
                const float2 w = make_float2(f[2 * D], f[2 * D + 1]);              // -|y'|^2
                // (a coordinate-major order over the rows, meant to share y'_d through the register
                // reuse cache, measured 0.8% slower for the Sum and no change for the fused
                // gradient: ptxas schedules either way)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 u = fma2(dup2(xr[r][0]), ny[0], w);
#pragma unroll
                    for (int d = 1; d < D; ++d) u = fma2(dup2(xr[r][d]), ny[d], u);   // 2x'.y' - |y'|^2
                    float2 ex;
                    // FP32-pipe exp2 share (kPolyShare, off: see DESIGN.md Sec. 6 measurements)
                    if (POLY && r == R - 1 && hh == 0) ex = ex2_poly2(u);
                    else ex = make_float2(ex2(u.x), ex2(u.y));
                    if constexpr (NG == 0) {
#pragma unroll
                        for (int e = 0; e < E; ++e) acc[r][e] = fma2(ex, bv[e], acc[r][e]);
                    } else {
                        float2 wt;
                        if constexpr (E == 1) {
                            wt = mul2(ex, bv[0]);                       // e b (g_i applied later)
                        } else {
                            float2 bg = mul2(bv[0], dup2(gr[r][0]));
#pragma unroll
                            for (int e = 1; e < E; ++e) bg = fma2(bv[e], dup2(gr[r][e]), bg);
                            wt = mul2(ex, bg);                          // e <b, g_i>
                        }
                        if constexpr (MODE == 2 && E == 1) {
                            acc[r][0] = add2(acc[r][0], wt);           // Sum == S0
                        } else {
                            if constexpr (MODE == 2) {
#pragma unroll
                                for (int e = 0; e < E; ++e) acc[r][e] = fma2(ex, bv[e], acc[r][e]);
                            }
                            s0[r] = add2(s0[r], wt);
                        }
                        // (two scalar FFMAs instead of this 3-register-pair FFMA2 measured 2% slower)
#pragma unroll
                        for (int d = 0; d < D; ++d) accg[r][d] = fma2(wt, ny[d], accg[r][d]);   // w y'
                    }
                }
            } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 dd[D];
#pragma unroll
                for (int d = 0; d < D; ++d) dd[d] = add2(dup2(xr[r][d]), ny[d]);   // x' - y'
                float2 q = mul2(dd[0], dd[0]);
#pragma unroll
                for (int d = 1; d < D; ++d) q = fma2(dd[d], dd[d], q);             // |x'-y'|^2
                if constexpr (!Cfg::EXP) {
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[r][e] = fma2(q, bv[e], acc[r][e]);
                } else {
                    const float2 ex = make_float2(ex2(-q.x), ex2(-q.y));   // e^{-|x-y|^2/sigma^2}
                    if constexpr (MODE == 0) {
#pragma unroll
                        for (int e = 0; e < E; ++e) acc[r][e] = fma2(ex, bv[e], acc[r][e]);
                    } else {
                        float2 w;
                        if constexpr (E == 1) {
                            w = mul2(ex, bv[0]);                   // e_ij b_j (g_i applied later)
                            if constexpr (MODE == 2) acc[r][0] = add2(acc[r][0], w);
                        } else {
                            float2 bg = mul2(bv[0], dup2(gr[r][0]));
#pragma unroll
                            for (int e = 1; e < E; ++e) bg = fma2(bv[e], dup2(gr[r][e]), bg);
                            w = mul2(ex, bg);                      // e_ij <b_j, g_i>
                            if constexpr (MODE == 2) {
#pragma unroll
                                for (int e = 0; e < E; ++e) acc[r][e] = fma2(ex, bv[e], acc[r][e]);
                            }
                        }
#pragma unroll
                        for (int d = 0; d < D; ++d) accg[r][d] = fma2(w, dd[d], accg[r][d]);
                    }
                }
            }
            }
        }
        }
        ring.release(k);
        // promote the tile's fp32 partials to fp64 (every 512 j)
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int c = 0; c < NS; ++c) {
                acc64[r][c] += (double)acc[r][c].x + (double)acc[r][c].y;
                acc[r][c] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int c = 0; c < NG; ++c) {
                acc64[r][NS + c] += (double)accg[r][c].x + (double)accg[r][c].y;
                accg[r][c] = make_float2(0.f, 0.f);
            }
            if constexpr (OWN_S0) {
                s064[r] += (double)s0[r].x + (double)s0[r].y;
                s0[r] = make_float2(0.f, 0.f);
            }
        }
    }

    // ---- epilogue --------------------------------------------------------------------------
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= row_end) continue;
        if constexpr (XP) {
            const double fac = exp2(-xsq[r]);                  // row factor 2^(-|x'|^2)
            if constexpr (NG > 0) {
                // sum_j w_ij (x'_i - y'_j) = x'_i S0_i - S_i  (the kernel's d' convention)
                const double S0 = OWN_S0 ? s064[r] : acc64[r][0];
#pragma unroll
                for (int c = 0; c < NG; ++c)
                    acc64[r][NS + c] = 0.5 * (double)xr[r][c] * S0 - acc64[r][NS + c];
            }
#pragma unroll
            for (int c = 0; c < C; ++c) acc64[r][c] *= fac;
        }
        if (p.split > 1) {
            double *dst = p.part + ((int64_t)sp * p.M + i) * C;
#pragma unroll
            for (int c = 0; c < C; ++c) dst[c] = acc64[r][c];
            continue;
        }
#pragma unroll
        for (int c = 0; c < NS; ++c) {
            const double v = acc64[r][c] * p.scale_sum;
            if (p.out_f64) ((double *)p.out)[i * NS + c] = v;
            else ((float *)p.out)[i * NS + c] = (float)v;
        }
        if constexpr (NG > 0) {
            double gs = p.scale_grad;
            if (E == 1 && p.g) gs *= (double)__ldg(p.g + i);
#pragma unroll
            for (int c = 0; c < NG; ++c) {
                const double v = acc64[r][NS + c] * gs;
                if (MODE == 2) p.out_grad[i * D + c] = (float)v;
                else if (p.out_f64) ((double *)p.out)[i * D + c] = v;
                else ((float *)p.out)[i * D + c] = (float)v;
            }
        }
    }
}

template <int MODE, int D, int E, int R>
__global__ void __launch_bounds__(kThreads, (((MODE == 0 || MODE == 3) && E == 1 && D <= 3 && R == 4) ||
                                            ((MODE == 1 || MODE == 2) && GENRED_GRAD_R == 2 && D + E <= 4 && E == 1 && R == 2)) ? 3 : 2)
sum_kernel(const SumParams p) {
    using Cfg = SumCfg<MODE, D, E>;
    extern __shared__ __align__(128) unsigned char smem_raw[];

    // this CTA's j-range: record pairs [q0, q0 + npc), streamed in tiles of PAIRS
    int64_t row0, row_end, q0, npc;
    int sp;
    if (p.units) {                                     // block-sparse: rows of one cluster
        const RangeUnit u = p.units[blockIdx.x];
        row0 = u.row0; row_end = u.row_end; sp = 0;
        q0 = u.tile0 * Cfg::PAIRS; npc = u.ntiles * Cfg::PAIRS;
    } else {
        const int64_t itile = blockIdx.x / p.split;
        sp = (int)(blockIdx.x % p.split);
        q0 = (int64_t)sp * p.pairs_per_split;
        npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);   // empty: zero partial
        row0 = itile * (int64_t)(kConsumerWarps * 32 * R);
        row_end = p.M;
    }
    const int nt = (int)((npc + Cfg::PAIRS - 1) / Cfg::PAIRS);
    const int last_np = (int)(npc - (int64_t)(nt > 0 ? nt - 1 : 0) * Cfg::PAIRS);
    const uint32_t last_bytes = (uint32_t)last_np * Cfg::RS * 4u;   // a partial last tile is copied partially

    JRing<kStages> ring;
    if constexpr (MODE != 3) {
        const Geo geo = geo_decode(p.geo, D, p.s);     // same decision as the pack kernel
        if (MODE == 0 && p.direct_only && geo.expanded) return;   // gauss_tc.cu took this call
        ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * Cfg::RS, nt, kConsumerWarps, last_bytes);
        if (geo.expanded) sum_body<MODE, D, E, R, true>(p, ring, nt, last_np, row0, row_end, sp, geo);
        else sum_body<MODE, D, E, R, false>(p, ring, nt, last_np, row0, row_end, sp, geo);
    } else {
        ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * Cfg::RS, nt, kConsumerWarps, last_bytes);
        Geo geo{};
        sum_body<MODE, D, E, R, false>(p, ring, nt, last_np, row0, row_end, sp, geo);
    }
}

// ---- host-side dispatch over (MODE, D, E, R) ------------------------------------------------
template <int MODE, int D, int E, int R>
static cudaError_t run_sum(const SumLaunch &a, cudaStream_t st, int *ctas) {
    using Cfg = SumCfg<MODE, D, E>;
    auto kern = sum_kernel<MODE, D, E, R>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Cfg::SMEM);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    SumParams p;
    p.x = a.x; p.J = a.J; p.g = a.g; p.M = a.M; p.split = a.split;
    p.pairs_per_split = a.pairs_per_split; p.npv = a.npv; p.s = a.s;
    p.scale_sum = a.scale_sum; p.scale_grad = a.scale_grad; p.out = a.out; p.out_f64 = a.out_f64;
    p.out_grad = a.out_grad; p.part = a.part; p.geo = a.geo; p.units = a.units;
    p.direct_only = a.direct_only;
    const int64_t rows = (int64_t)kConsumerWarps * 32 * R;
    const int64_t itiles = (a.M + rows - 1) / rows;
    const int64_t grid = a.units ? a.n_units : itiles * a.split;
    if (grid == 0) { *ctas = 0; return cudaSuccess; }
    *ctas = (int)grid;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
}

template <int MODE, int D, int E, int R>
static int occ_sum() {
    using Cfg = SumCfg<MODE, D, E>;
    auto kern = sum_kernel<MODE, D, E, R>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, Cfg::SMEM) != cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

// Largest rows-per-thread that stays spill-free (80 registers for Sum at 3 CTAs/SM, 128 for the
// gradient modes at 2 CTAs/SM).
template <int MODE, int D, int E>
constexpr int sum_rmax() {
    return (MODE == 0 || MODE == 3) ? ((D + E <= 4 || (E == 1 && D <= 4)) ? 4 : 2)
                                    : ((D + E <= 4) ? GENRED_GRAD_R : (D + E <= 6 ? 2 : 1));
}
template <int MODE, int D, int E>
static cudaError_t run_sum_r(const SumLaunch &a, cudaStream_t st, int *ctas) {
    constexpr int RM = sum_rmax<MODE, D, E>();
    return a.R == 1 ? run_sum<MODE, D, E, 1>(a, st, ctas) : run_sum<MODE, D, E, RM>(a, st, ctas);
}
template <int MODE, int D, int E>
static int occ_sum_r(int R) {
    constexpr int RM = sum_rmax<MODE, D, E>();
    return R == 1 ? occ_sum<MODE, D, E, 1>() : occ_sum<MODE, D, E, RM>();
}

template <int MODE, int D>
static cudaError_t run_sum_e(const SumLaunch &a, cudaStream_t st, int *ctas) {
    switch (a.E) {
        case 1: return run_sum_r<MODE, D, 1>(a, st, ctas);
        case 2: return run_sum_r<MODE, D, 2>(a, st, ctas);
        case 3: return run_sum_r<MODE, D, 3>(a, st, ctas);
        case 4: return run_sum_r<MODE, D, 4>(a, st, ctas);
    }
    return cudaErrorInvalidValue;
}
template <int MODE, int D>
static int occ_sum_e(int E, int R) {
    switch (E) {
        case 1: return occ_sum_r<MODE, D, 1>(R);
        case 2: return occ_sum_r<MODE, D, 2>(R);
        case 3: return occ_sum_r<MODE, D, 3>(R);
        case 4: return occ_sum_r<MODE, D, 4>(R);
    }
    return 1;
}

template <int MODE>
static cudaError_t run_sum_d(const SumLaunch &a, cudaStream_t st, int *ctas) {
    switch (a.D) {
        case 1: return run_sum_e<MODE, 1>(a, st, ctas);
        case 2: return run_sum_e<MODE, 2>(a, st, ctas);
        case 3: return run_sum_e<MODE, 3>(a, st, ctas);
        case 4: return run_sum_e<MODE, 4>(a, st, ctas);
        case 5: return run_sum_e<MODE, 5>(a, st, ctas);
        case 6: return run_sum_e<MODE, 6>(a, st, ctas);
        case 7: return run_sum_e<MODE, 7>(a, st, ctas);
        case 8: return run_sum_e<MODE, 8>(a, st, ctas);
    }
    return cudaErrorInvalidValue;
}
template <int MODE>
static int occ_sum_d(int D, int E, int R) {
    switch (D) {
        case 1: return occ_sum_e<MODE, 1>(E, R);
        case 2: return occ_sum_e<MODE, 2>(E, R);
        case 3: return occ_sum_e<MODE, 3>(E, R);
        case 4: return occ_sum_e<MODE, 4>(E, R);
        case 5: return occ_sum_e<MODE, 5>(E, R);
        case 6: return occ_sum_e<MODE, 6>(E, R);
        case 7: return occ_sum_e<MODE, 7>(E, R);
        case 8: return occ_sum_e<MODE, 8>(E, R);
    }
    return 1;
}

cudaError_t launch_sum(const SumLaunch &a, cudaStream_t st, int *ctas) {
    switch (a.mode) {
        case 0: return run_sum_d<0>(a, st, ctas);
        case 1: return run_sum_d<1>(a, st, ctas);
        case 2: return run_sum_d<2>(a, st, ctas);
        case 3: return run_sum_d<3>(a, st, ctas);
    }
    return cudaErrorInvalidValue;
}

template <int MODE>
static int rmax_d_e(int D, int E) {
    int r = 1;
#define GENRED_RM(DD, EE) if (D == DD && E == EE) r = sum_rmax<MODE, DD, EE>();
#define GENRED_RM_E(DD) GENRED_RM(DD, 1) GENRED_RM(DD, 2) GENRED_RM(DD, 3) GENRED_RM(DD, 4)
    GENRED_RM_E(1) GENRED_RM_E(2) GENRED_RM_E(3) GENRED_RM_E(4)
    GENRED_RM_E(5) GENRED_RM_E(6) GENRED_RM_E(7) GENRED_RM_E(8)
#undef GENRED_RM_E
#undef GENRED_RM
    return r;
}

int sum_rows_per_thread_max(int mode, int D, int E) {
    switch (mode) {
        case 0: return rmax_d_e<0>(D, E);
        case 1: return rmax_d_e<1>(D, E);
        case 2: return rmax_d_e<2>(D, E);
        case 3: return rmax_d_e<3>(D, E);
    }
    return 1;
}

int sum_occupancy(int mode, int D, int E, int R) {
    switch (mode) {
        case 0: return occ_sum_d<0>(D, E, R);
        case 1: return occ_sum_d<1>(D, E, R);
        case 2: return occ_sum_d<2>(D, E, R);
        case 3: return occ_sum_d<3>(D, E, R);
    }
    return 1;
}

}  // namespace genred
