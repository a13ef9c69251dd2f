// sum_body.cuh -- the Genred Sum pair loop, shared by sum_kernel.cu (row tiles: one thread per
// row, R rows per thread) and sum_smm.cu (small M: the CTA's threads share R rows).  See
// sum_kernel.cu for the design notes.
#pragma once
#include <math.h>
#include <stdlib.h>

#include "device.cuh"
#include "geo.cuh"
#include "internal.h"

namespace genred {

// Gradient modes with D + E <= 4 (fused Sum+grad, records carrying b' and b' y'), row-pair mode
// (GENRED_GRAD_RP): 4 rows per thread and 16 record pairs per iteration at 3 CTAs/SM (80
// registers; the fp64 tile sums spill to local memory once per 512 j, outside the pair loop)
// measured 13.46 pairs/clk/SM at M = N = 1e5 and 14.07 at 4e5 (8 pairs: 13.34 / 13.91; 2 CTAs/SM:
// 13.03 / 13.41; 4 pairs: 12.42 / 12.94; 6 or 8 rows per thread spill in the loop: 13.22 / 11.82).  The j-packed loop of
// round 1 (4 rows, 4 pairs, 2 CTAs/SM) measured 11.45 / 11.93.  The direct form shares the
// kernel: 8.92 -> 8.77 pairs/clk/SM at 3 CTAs/SM (4e5, sigma = 0.05).
#ifndef GENRED_GRAD_R
#define GENRED_GRAD_R 4
#endif
#ifndef GENRED_GRAD_MINB
#define GENRED_GRAD_MINB 3
#endif
// (Round 2: the row-pair loop's 4 accumulating FFMA2s -- a broadcast scalar and two register
// pairs, 95.8 lane-FMA/clk/SM in tools/hwprobe2.cu, the wall C2 sits at -- split into scalar
// fma.rn.f32 pairs measured 11.18 against 13.78 pairs/clk/SM: issue-bound,
// profiles/r02_grad_scalar_acc.txt.)
// Row-pair packing of the expanded gradient modes (E = 1, records carrying b' and b' y'): the
// packed FFMA2 lanes hold two ROWS and the j-record value is a broadcast scalar operand, instead
// of two j's against a per-row broadcast.  Every FFMA2 then reads one fresh scalar + two register
// pairs (not three pairs), and the row-pair's exponential is reused by the 1 + D accumulations.
#ifndef GENRED_GRAD_RP
#define GENRED_GRAD_RP 1
#endif
// Record pairs per pair-loop iteration of the Sum modes: 4 measured 15.16 pairs/clk/SM against
// 14.98 for 2 and 15.01 for 8 (Gaussian Sum, M = N = 1e6).
#ifndef GENRED_SUM_HH
#define GENRED_SUM_HH 4
#endif
// Gaussian Sum / SqDist Sum, D <= 3, 4 rows per thread: 4 CTAs/SM (64 registers) measured 15.42
// pairs/clk/SM (expanded form, 2e6^2) and 13.40 (direct form, sigma = 0.05) against 15.34 / 13.21
// at 3 CTAs/SM (round 2).
#ifndef GENRED_SUM_MINB
#define GENRED_SUM_MINB 4
#endif
// Tile-centred loops: each tile's table entry (c_k, r_k^2) loaded one tile ahead (fused gradient
// at sigma = 0.05: 13.15 -> 13.61 pairs/clk/SM; Sum and LSE unchanged)
#ifndef GENRED_CEN_PREFETCH
#define GENRED_CEN_PREFETCH 1
#endif
#ifndef GENRED_GRAD_HH
#define GENRED_GRAD_HH 16
#endif
// Row-pair gradient loop: fp32 tile sums promoted to fp64 every GENRED_GRAD_PROMO tiles of 512 j
// (R18: every <= 1024 pairs); each promotion costs conversions on the MUFU pipe.
#ifndef GENRED_GRAD_STAGES
#define GENRED_GRAD_STAGES 4
#endif
#ifndef GENRED_GRAD_PROMO
#define GENRED_GRAD_PROMO 2
#endif

template <int MODE, int D, int E>
struct SumCfg {
    // record pair: 2D coordinates, then (MODE 0 only) the pair slot of w = -|y'|^2 used by the
    // expanded form, then 2E signal values; padded to a multiple of 16 bytes
    static constexpr int BOFF = (MODE != 3) ? 2 * (D + 1) : 2 * D;
    // gradient modes, E = 1: 2D more floats, b_j y'_j (expanded form; zero in direct records)
    static constexpr bool BY = (MODE == 1 || MODE == 2) && E == 1 && kGradBY;
    static constexpr int BYOFF = BOFF + 2 * E;
    static constexpr int RS = ((BOFF + 2 * E + (BY ? 2 * D : 0)) + 3) / 4 * 4;   // floats per record pair
    static constexpr int PAIRS = kTileJ / 2;
    static constexpr int TILE_FLOATS = PAIRS * RS;
    static constexpr int NS = (MODE == 1) ? 0 : E;                // sum columns
    static constexpr int NG = (MODE == 1 || MODE == 2) ? D : 0;   // gradient columns
    static constexpr int C = NS + NG;
    static constexpr bool GRAD = NG > 0;
    static constexpr bool EXP = MODE != 3;
    // ring depth: the row-pair gradient kernels (GENRED_GRAD_STAGES) may run 4 CTAs/SM, whose
    // smem budget holds 3 stages of their 16 KB tiles
    static constexpr int STAGES = ((MODE == 1 || MODE == 2) && E == 1 && D <= 3) ? GENRED_GRAD_STAGES : kStages;
    static constexpr int SMEM = JRing<STAGES>::smem_bytes(TILE_FLOATS);
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
    const RangeUnit *units;   // block-sparse ranges: one unit per (cluster, row tile)
    int64_t n_work;           // work units; the persistent grid walks w = blockIdx.x, + gridDim.x, ...
    unsigned *tile_done;      // split > 1, row tiles only: per-row-tile arrival counters (all zero
                              // between calls); the last CTA of a row tile merges its partials
    double *part_smem = nullptr;   // sum_small_kernel with a cluster merge: this CTA's partials go
                                   // to its own shared memory, [local row][C], not to `part`
    const float4 *centers = nullptr;   // MODE 0 tile-centred form: per 512-j tile (c_k, r_k^2 or -1)
    int split_major = 0;      // row tiles: work unit w -> (split w / itiles, row tile w % itiles)
    int64_t itiles = 0;       // row tiles (split_major)
};

// (Round 1, at 3 CTAs/SM: moving 1/8 (1/4) of the exps to the FP32 pipe measured 14.74 (13.73)
// pairs/clk/SM against 14.90 with every exp on MUFU; at 4 CTAs/SM the 1/8 share pays, above.)
// Expanded Gaussian Sum: a share of the exponentials on the FP32 pipe (ex2_poly2: degree-5
// polynomial + exponent add, 2.3e-7 relative, u in [-24, 6] by the box bound).  At 4 CTAs/SM
// (FP32 pipe ~48% busy, MUFU 97%) one eighth (mode 3: the last row of a thread, every other
// record pair) measured 16.66 pairs/clk/SM against 15.43 without (2e6^2); 1/16 16.21, 3/16 15.93,
// 1/4 15.05 (round 2).  At 3 CTAs/SM in round 1 the share had measured slower.
#ifndef GENRED_POLY_MODE
#define GENRED_POLY_MODE 3
#endif
constexpr bool kPolyShare = GENRED_POLY_MODE != 0;

// The pair loop + epilogue.  XP selects the expanded form of the Gaussian Sum (MODE 0 only):
//   exp(-|x-y|^2/sigma^2) = 2^(-|x'|^2) * 2^(u),  u = 2 x'.y' - |y'|^2,  x' = s (x - c)
// so a pair costs 3 FFMA (u, packed over two j's) + exp + 1 FFMA instead of 7 FP32 ops, which
// leaves the MUFU pipe (16 ex2/clk/SM) as the only bound; the row factor 2^(-|x'|^2) is applied
// in fp64 at the end.
// SMM (small-M mode, north star (a) "a warp-shuffle finish runs when several threads share one
// i"): all 256 threads of the CTA share the same R rows and split each tile's record pairs among
// themselves (thread t takes pairs t, t + 256, ...); at the end the CTA reduces its fp64 partials
// with warp shuffles (fixed butterfly order) and a fixed-order sum over the 8 warps, and thread 0
// runs the epilogue for the R rows.  Used when M is too small to fill the GPU with row tiles.
// A JRing stand-in whose tiles are already resident in shared memory (sum_small_kernel builds the
// CTA's j-records there itself): acquire returns the tile, release is a no-op.
struct SmemTiles {
    const float *base;
    int tile_floats;
    __device__ __forceinline__ const float *acquire(int k) const { return base + k * tile_floats; }
    __device__ __forceinline__ void release(int) const {}
};

template <int MODE, int D, int E, int R, bool XP, bool SMM, class Ring>
__device__ __forceinline__ void sum_body(const SumParams &p, Ring &ring, int nt, int last_np,
                                         int64_t row0, int64_t row_end, int sp, const Geo &geo) {
    using Cfg = SumCfg<MODE, D, E>;
    constexpr int RS = Cfg::RS, NS = Cfg::NS, NG = Cfg::NG, C = Cfg::C, BOFF = Cfg::BOFF;
    constexpr bool POLY = kPolyShare && XP && R == 4;
    constexpr int HH = SMM ? 1 : (MODE == 1 || MODE == 2) ? GENRED_GRAD_HH : GENRED_SUM_HH;   // record pairs per iteration
    constexpr bool RAWD = !XP && Cfg::EXP;           // direct Gaussian modes: raw differences
    const float2 negs2 = dup2(-(p.s * p.s));
    const int ct = threadIdx.x;
    float xr[R][D];
    float gr[R][E];
    double xsq[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = SMM ? row0 + r : row0 + r * (kConsumerWarps * 32) + ct;
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
                // direct Gaussian form: RAW x.  The difference x - y is then exact for nearby
                // coordinates (Sterbenz) and rounded relative to |x - y| otherwise; s x - s y
                // would round each term at ulp(s |x|), which loses the gradient's linear factor
                // when x ~ y (R18d) and the exponent of clouds far from the origin or
                // wide against sigma (R18e).  |x - y|^2 is scaled by s^2 afterwards.
                xr[r][d] = RAWD ? v : p.s * v;
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
    // row-pair mode (GENRED_GRAD_RP): X2[q][d] = (2x'_{2q,d}, 2x'_{2q+1,d}); S0p / Sp the fp32
    // tile sums of e b' and e b' y'_d for the two rows of pair q (lanes x, y)
    constexpr bool RP = GENRED_GRAD_RP && XP && Cfg::BY && !SMM && (R % 2 == 0);
    // (the same packing for the direct-form Gaussian Sum measured 1.7% slower at 3 CTAs/SM and
    // +0.4% at 4: not used)
    constexpr int RQ = RP ? R / 2 : 1;
    float2 X2[RQ][D], S0p[RQ], Sp[RQ][D];
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
        S0p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int d = 0; d < D; ++d) {
            X2[q][d] = RP ? make_float2(xr[2 * q][d], xr[(2 * q + 1) % R][d]) : make_float2(0.f, 0.f);
            Sp[q][d] = make_float2(0.f, 0.f);
        }
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
        if constexpr (RP) {
        for (int pp2 = 0; pp2 < np; pp2 += HH) {
#pragma unroll
        for (int hh = 0; hh < HH; ++hh) {
            float f[RS];
#pragma unroll
            for (int q = 0; q < RS / 4; ++q) {
                const float4 v = lds128(tile + (pp2 + hh) * RS + 4 * q);
                f[4 * q + 0] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int hq = 0; hq < 2 * RQ; ++hq) {     // the record pair's two j's x the row pairs
                const int h = hq / RQ, q = hq % RQ;
                {
                    float2 u = mul2(X2[q][0], dup2(f[h]));                          // 2 x'.y'
#pragma unroll
                    for (int d = 1; d < D; ++d) u = fma2(X2[q][d], dup2(f[2 * d + h]), u);
                    const float2 ex = make_float2(ex2(u.x), ex2(u.y));
                    S0p[q] = fma2(ex, dup2(f[BOFF + h]), S0p[q]);                   // e b'
#pragma unroll
                    for (int d = 0; d < D; ++d)
                        Sp[q][d] = fma2(ex, dup2(f[Cfg::BYOFF + 2 * d + h]), Sp[q][d]);   // e b' y'_d
                }
            }
        }
        }
        } else {
        for (int pp2 = SMM ? ct : 0; pp2 < np; pp2 += SMM ? kThreads : HH) {
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
                    // FP32-pipe exp2 share (GENRED_POLY_MODE above)
                    // share of the exponentials on the FP32 pipe: mode 1 = 1/(R HH), 2 = 1/R,
                    // 3 = 1/(2R), 4 = 3/(4R), 5 = 1/(2R) spread over two rows
                    const bool poly = POLY &&
                        (GENRED_POLY_MODE == 1 ? (r == R - 1 && hh == 0) :
                         GENRED_POLY_MODE == 2 ? (r == R - 1) :
                         GENRED_POLY_MODE == 3 ? (r == R - 1 && (hh & 1) == 0) :
                         GENRED_POLY_MODE == 4 ? (r == R - 1 && hh != HH - 1) :
                         GENRED_POLY_MODE == 5 ? ((r == R - 1 && hh == 0) || (r == R - 2 && hh == HH / 2)) :
                         GENRED_POLY_MODE == 6 ? (hh == 0) : false);
                    if (poly) ex = ex2_poly2(u);
                    else ex = make_float2(ex2(u.x), ex2(u.y));
                    if constexpr (NG == 0) {
#pragma unroll
                        for (int e = 0; e < E; ++e) acc[r][e] = fma2(ex, bv[e], acc[r][e]);
                    } else {
                        float2 wt = make_float2(0.f, 0.f);
                        if constexpr (Cfg::BY) {
                            // S0 += e b, S_d += e (b y')_d: b y' comes with the record
                            float2 &S0r = (MODE == 2) ? acc[r][0] : s0[r];
                            S0r = fma2(ex, bv[0], S0r);
#pragma unroll
                            for (int d = 0; d < D; ++d)
                                accg[r][d] = fma2(ex, make_float2(f[Cfg::BYOFF + 2 * d], f[Cfg::BYOFF + 2 * d + 1]), accg[r][d]);
                        } else if constexpr (E == 1) {
                            wt = mul2(ex, bv[0]);                       // e b (g_i applied later)
                        } else {
                            float2 bg = mul2(bv[0], dup2(gr[r][0]));
#pragma unroll
                            for (int e = 1; e < E; ++e) bg = fma2(bv[e], dup2(gr[r][e]), bg);
                            wt = mul2(ex, bg);                          // e <b, g_i>
                        }
                        if constexpr (!Cfg::BY) {
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
                    float2 ex;                                                 // e^{-|x-y|^2/sigma^2}
                    if constexpr (RAWD) {
                        const float2 t = mul2(q, negs2);                      // -s^2 |x - y|^2
                        ex = make_float2(ex2(t.x), ex2(t.y));
                    } else {
                        ex = make_float2(ex2(-q.x), ex2(-q.y));
                    }
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
        }   // RP
        ring.release(k);
        // promote the tile's fp32 partials to fp64 (every 512 j)
        if constexpr (RP) {
            if (GENRED_GRAD_PROMO > 1 && (k + 1) % GENRED_GRAD_PROMO != 0 && k != nt - 1) continue;
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                const int r0 = 2 * q, r1 = 2 * q + 1;
                double &a0 = OWN_S0 ? s064[r0] : acc64[r0][0];
                double &a1 = OWN_S0 ? s064[r1] : acc64[r1][0];
                a0 += (double)S0p[q].x;
                a1 += (double)S0p[q].y;
                S0p[q] = make_float2(0.f, 0.f);
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    acc64[r0][NS + d] += (double)Sp[q][d].x;
                    acc64[r1][NS + d] += (double)Sp[q][d].y;
                    Sp[q][d] = make_float2(0.f, 0.f);
                }
            }
        }
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

    if constexpr (SMM) {
        // CTA reduction of the per-thread fp64 partials (deterministic), result in thread 0
        constexpr int CO = C + (OWN_S0 ? 1 : 0);
        __shared__ double red[kConsumerWarps][R * CO];
        const int lane = ct & 31, warp = ct >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int c = 0; c < CO; ++c) {
                double v = c < C ? acc64[r][c] : s064[r];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) red[warp][r * CO + c] = v;
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int c = 0; c < CO; ++c) {
                double v = red[0][r * CO + c];
#pragma unroll
                for (int w = 1; w < kConsumerWarps; ++w) v += red[w][r * CO + c];
                if (c < C) acc64[r][c] = v;
                else s064[r] = v;
            }
        }
    }

    // ---- epilogue (small-M mode: thread 0 for the CTA's rows) ---------------------------------
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = SMM ? row0 + r : row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= row_end || (SMM && ct != 0)) continue;
        if constexpr (XP) {
            // row factor 2^(-|x'|^2); in the row-pair mode x' is re-read from X2 (= 2 x', exact),
            // so neither xr nor xsq stays live through the pair loop
            double xs2 = 0.0;
            if constexpr (RP) {
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const double h = 0.5 * (double)((r & 1) ? X2[r >> 1][d].y : X2[r >> 1][d].x);
                    xs2 += h * h;
                }
            } else {
                xs2 = xsq[r];
            }
            const double fac = exp2(-xs2);
            if constexpr (NG > 0) {
                // sum_j w_ij (x'_i - y'_j) = x'_i S0_i - S_i  (the kernel's d' convention)
                const double S0 = OWN_S0 ? s064[r] : acc64[r][0];
#pragma unroll
                for (int c = 0; c < NG; ++c)
                    acc64[r][NS + c] = 0.5 * (double)(RP ? ((r & 1) ? X2[r >> 1][c].y : X2[r >> 1][c].x) : xr[r][c]) * S0
                                       - acc64[r][NS + c];
            }
#pragma unroll
            for (int c = 0; c < C; ++c) acc64[r][c] *= fac;
        }
        if constexpr (RAWD) {                              // raw (x - y): back to the s-scaled convention
#pragma unroll
            for (int c = 0; c < NG; ++c) acc64[r][NS + c] *= (double)p.s;
        }
        if (p.part_smem) {                                 // cluster merge (sum_small_kernel)
#pragma unroll
            for (int c = 0; c < C; ++c) p.part_smem[(i - row0) * C + c] = acc64[r][c];
            continue;
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

// The tile-centred expanded form of the Gaussian Sum (MODE 0, tile_order.cu, R18j).
// y is ordered along a Hilbert curve and each 512-j tile k carries its records around its own
// centre c_k: y'' = s (y - c_k), w = -|y''|^2.  For a row, x'' = s (x - c_k) (from RAW x, so the
// rounding is relative to |x - c_k|), and
//   exp(-|x - y|^2 / sigma^2) = 2^(-|x''|^2) * 2^(u),   u = 2 x''.y'' - |y''|^2,
// the pair loop of sum_body's expanded form (3 FFMA + exp + 1 FFMA per pair, the same FP32-pipe
// exp2 share) with the row factor 2^(-|x''|^2) applied per tile in fp64 when the tile's fp32 sums
// are promoted.  A row farther than r_k + 11.5 from c_k (every term of the tile below 2^-121, the
// deep tail of reading R4c) takes x'' = 0 and factor 0, which also keeps 2^u finite (u <= 68).
// Tiles whose radius fails |y''|^2 <= kExpandedR2Max keep the direct layout and run the direct
// form's loop on raw differences (R18e).
template <int D, int E, int R, class Ring>
__device__ __forceinline__ void sum_body_local(const SumParams &p, Ring &ring, int nt, int last_np,
                                               int64_t row0, int64_t row_end, int sp, int64_t tile0) {
    using Cfg = SumCfg<0, D, E>;
    constexpr int RS = Cfg::RS, BOFF = Cfg::BOFF;
    constexpr bool POLY = kPolyShare && R == 4;
    constexpr int HH = GENRED_SUM_HH;
    const int ct = threadIdx.x;
    const float2 negs2 = dup2(-(p.s * p.s));
    float xw[R][D];                                   // raw x rows
    double acc64[R][E];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
#pragma unroll
        for (int d = 0; d < D; ++d) xw[r][d] = i < row_end ? __ldg(p.x + i * D + d) : 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) acc64[r][e] = 0.0;
    }
#if GENRED_CEN_PREFETCH
    float4 cen_next = nt > 0 ? __ldg(p.centers + tile0) : make_float4(0.f, 0.f, 0.f, -1.f);
#endif
    for (int k = 0; k < nt; ++k) {
#if GENRED_CEN_PREFETCH
        const float4 cen = cen_next;                 // loaded one tile ahead
        if (k + 1 < nt) cen_next = __ldg(p.centers + tile0 + k + 1);
#else
        const float4 cen = __ldg(p.centers + tile0 + k);
#endif
        const float *tile = ring.acquire(k);
        const int np = k == nt - 1 ? last_np : Cfg::PAIRS;
        float2 acc[R][E];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < E; ++e) acc[r][e] = make_float2(0.f, 0.f);
        if (cen.w >= 0.0f) {
            const float cc[3] = {cen.x, cen.y, cen.z};
            const float lim = sqrtf(cen.w) + 11.5f;
            float xl[R][D];                           // 2 x''
            unsigned far = 0u;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float q = 0.0f;
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const float h = p.s * (xw[r][d] - cc[d]);
                    xl[r][d] = 2.0f * h;
                    q = fmaf(h, h, q);
                }
                if (q > lim * lim) {
                    far |= 1u << r;
#pragma unroll
                    for (int d = 0; d < D; ++d) xl[r][d] = 0.0f;
                }
            }
            for (int pp2 = 0; pp2 < np; pp2 += HH) {
#pragma unroll
            for (int hh = 0; hh < HH; ++hh) {
                float f[RS];
#pragma unroll
                for (int q = 0; q < RS / 4; ++q) {
                    const float4 v = lds128(tile + (pp2 + hh) * RS + 4 * q);
                    f[4 * q + 0] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
                }
                const float2 w = make_float2(f[2 * D], f[2 * D + 1]);              // -|y''|^2
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 u = fma2(dup2(xl[r][0]), make_float2(f[0], f[1]), w);
#pragma unroll
                    for (int d = 1; d < D; ++d) u = fma2(dup2(xl[r][d]), make_float2(f[2 * d], f[2 * d + 1]), u);
                    const bool poly = POLY && (r == R - 1 && (hh & 1) == 0);      // GENRED_POLY_MODE 3
                    const float2 ex = poly ? ex2_poly2(u) : make_float2(ex2(u.x), ex2(u.y));
#pragma unroll
                    for (int e = 0; e < E; ++e)
                        acc[r][e] = fma2(ex, make_float2(f[BOFF + 2 * e], f[BOFF + 2 * e + 1]), acc[r][e]);
                }
            }
            }
            ring.release(k);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                // row factor 2^(-|x''|^2) in fp64 from the same x'' (= xl / 2, exact): 2^-n exact,
                // 2^-f (f in [0, 1)) by MUFU.EX2 (2^-22 relative)
                double q64 = 0.0;
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const double hd = 0.5 * (double)xl[r][d];
                    q64 = fma(hd, hd, q64);
                }
                const double n = floor(q64);
                const double fac = ((far >> r) & 1u) ? 0.0 : ldexp((double)ex2(-(float)(q64 - n)), -(int)n);
#pragma unroll
                for (int e = 0; e < E; ++e) acc64[r][e] += fac * ((double)acc[r][e].x + (double)acc[r][e].y);
            }
        } else {
            for (int pp2 = 0; pp2 < np; pp2 += HH) {
#pragma unroll
            for (int hh = 0; hh < HH; ++hh) {
                float f[RS];
#pragma unroll
                for (int q = 0; q < RS / 4; ++q) {
                    const float4 v = lds128(tile + (pp2 + hh) * RS + 4 * q);
                    f[4 * q + 0] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 dd[D];
#pragma unroll
                    for (int d = 0; d < D; ++d) dd[d] = add2(dup2(xw[r][d]), make_float2(f[2 * d], f[2 * d + 1]));
                    float2 q = mul2(dd[0], dd[0]);
#pragma unroll
                    for (int d = 1; d < D; ++d) q = fma2(dd[d], dd[d], q);         // |x - y|^2 (raw)
                    const float2 tq = mul2(q, negs2);
                    const float2 ex = make_float2(ex2(tq.x), ex2(tq.y));
#pragma unroll
                    for (int e = 0; e < E; ++e)
                        acc[r][e] = fma2(ex, make_float2(f[BOFF + 2 * e], f[BOFF + 2 * e + 1]), acc[r][e]);
                }
            }
            }
            ring.release(k);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int e = 0; e < E; ++e) acc64[r][e] += (double)acc[r][e].x + (double)acc[r][e].y;
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= row_end) continue;
        if (p.split > 1) {
            double *dst = p.part + ((int64_t)sp * p.M + i) * E;
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e] = acc64[r][e];
            continue;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double v = acc64[r][e] * p.scale_sum;
            if (p.out_f64) ((double *)p.out)[i * E + e] = v;
            else ((float *)p.out)[i * E + e] = (float)v;
        }
    }
}

// Tile-centred form of the gradient modes (MODE 1 / 2, E = 1, D <= 3, R = 4 rows per thread; R18j
// with R18g's records per tile: y'', b' = b 2^(-|y''|^2), b' y'').  The row-pair loop of sum_body
// (two rows in the FFMA2 lanes) runs on 2x'' = 2s(x - c_k); per row and tile, with
// fac = 2^(-|x''|^2):  S0 += fac S0p,  G += fac (x'' S0p - Sp)  (sum_j w (x'' - y'') is the
// s-scaled x - y in any frame).  Direct tiles run sum_body's raw-difference gradient loop, their
// (x - y) sums scaled by s into the same convention.
template <int MODE, int D, class Ring>
__device__ __forceinline__ void sum_body_local_grad(const SumParams &p, Ring &ring, int nt, int last_np,
                                                    int64_t row0, int64_t row_end, int sp, int64_t tile0) {
    using Cfg = SumCfg<MODE, D, 1>;
    constexpr int R = 4, RQ = 2, RS = Cfg::RS, BOFF = Cfg::BOFF, BYOFF = Cfg::BYOFF;
    constexpr int HH = GENRED_GRAD_HH;
    constexpr int NS = Cfg::NS, C = Cfg::C;
    const int ct = threadIdx.x;
    const float2 negs2 = dup2(-(p.s * p.s));
    double acc64[R][C];            // [sum (MODE 2)][grad D]
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) acc64[r][c] = 0.0;
#if GENRED_CEN_PREFETCH
    float4 cen_next = nt > 0 ? __ldg(p.centers + tile0) : make_float4(0.f, 0.f, 0.f, -1.f);
#endif
    for (int k = 0; k < nt; ++k) {
#if GENRED_CEN_PREFETCH
        const float4 cen = cen_next;                 // loaded one tile ahead
        if (k + 1 < nt) cen_next = __ldg(p.centers + tile0 + k + 1);
#else
        const float4 cen = __ldg(p.centers + tile0 + k);
#endif
        const bool loc = cen.w >= 0.0f;
        const float cc[3] = {cen.x, cen.y, cen.z};
        const float lim = loc ? sqrtf(cen.w) + 11.5f : 0.0f;
        float2 X2[RQ][D];              // 2x'' (centred tile) or raw x (direct tile), row pairs
        unsigned far = 0u;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
            float q = 0.0f;
            float xv[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const float xd = i < row_end ? __ldg(p.x + i * D + d) : 0.0f;
                if (loc) {
                    const float h = p.s * (xd - cc[d]);
                    xv[d] = 2.0f * h;
                    q = fmaf(h, h, q);
                } else {
                    xv[d] = xd;
                }
            }
            if (loc && q > lim * lim) {
                far |= 1u << r;
#pragma unroll
                for (int d = 0; d < D; ++d) xv[d] = 0.0f;
            }
#pragma unroll
            for (int d = 0; d < D; ++d) { if (r & 1) X2[r >> 1][d].y = xv[d]; else X2[r >> 1][d].x = xv[d]; }
        }
        const float *tile = ring.acquire(k);
        const int np = k == nt - 1 ? last_np : Cfg::PAIRS;
        float2 S0p[RQ], Sp[RQ][D];
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
            S0p[q] = make_float2(0.f, 0.f);
#pragma unroll
            for (int d = 0; d < D; ++d) Sp[q][d] = make_float2(0.f, 0.f);
        }
        if (loc) {
            for (int pp2 = 0; pp2 < np; pp2 += HH) {
#pragma unroll
            for (int hh = 0; hh < HH; ++hh) {
                float f[RS];
#pragma unroll
                for (int q = 0; q < RS / 4; ++q) {
                    const float4 v = lds128(tile + (pp2 + hh) * RS + 4 * q);
                    f[4 * q + 0] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
                }
#pragma unroll
                for (int hq = 0; hq < 2 * RQ; ++hq) {
                    const int h = hq / RQ, q = hq % RQ;
                    float2 u = mul2(X2[q][0], dup2(f[h]));                              // 2 x''.y''
#pragma unroll
                    for (int d = 1; d < D; ++d) u = fma2(X2[q][d], dup2(f[2 * d + h]), u);
                    const float2 ex = make_float2(ex2(u.x), ex2(u.y));
                    S0p[q] = fma2(ex, dup2(f[BOFF + h]), S0p[q]);                       // e b'
#pragma unroll
                    for (int d = 0; d < D; ++d) Sp[q][d] = fma2(ex, dup2(f[BYOFF + 2 * d + h]), Sp[q][d]);
                }
            }
            }
        } else {
            for (int pp2 = 0; pp2 < np; pp2 += HH) {
#pragma unroll
            for (int hh = 0; hh < HH; ++hh) {
                float f[RS];
#pragma unroll
                for (int q = 0; q < RS / 4; ++q) {
                    const float4 v = lds128(tile + (pp2 + hh) * RS + 4 * q);
                    f[4 * q + 0] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
                }
#pragma unroll
                for (int hq = 0; hq < 2 * RQ; ++hq) {
                    const int h = hq / RQ, q = hq % RQ;
                    float2 dd[D];
#pragma unroll
                    for (int d = 0; d < D; ++d) dd[d] = add2(X2[q][d], dup2(f[2 * d + h]));   // x - y (raw)
                    float2 q2 = mul2(dd[0], dd[0]);
#pragma unroll
                    for (int d = 1; d < D; ++d) q2 = fma2(dd[d], dd[d], q2);
                    const float2 t = mul2(q2, negs2);
                    const float2 ex = make_float2(ex2(t.x), ex2(t.y));
                    const float2 w = mul2(ex, dup2(f[BOFF + h]));                     // e b
                    S0p[q] = add2(S0p[q], w);
#pragma unroll
                    for (int d = 0; d < D; ++d) Sp[q][d] = fma2(w, dd[d], Sp[q][d]);   // w (x - y)
                }
            }
            }
        }
        ring.release(k);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int q = r >> 1;
            const double s0 = (double)((r & 1) ? S0p[q].y : S0p[q].x);
            if (loc) {
                double q64 = 0.0;
                double xh[D];
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    xh[d] = 0.5 * (double)((r & 1) ? X2[q][d].y : X2[q][d].x);     // x''
                    q64 = fma(xh[d], xh[d], q64);
                }
                const double n = floor(q64);
                const double fac = ((far >> r) & 1u) ? 0.0 : ldexp((double)ex2(-(float)(q64 - n)), -(int)n);
                if constexpr (NS > 0) acc64[r][0] += fac * s0;
#pragma unroll
                for (int d = 0; d < D; ++d)
                    acc64[r][NS + d] += fac * (xh[d] * s0 - (double)((r & 1) ? Sp[q][d].y : Sp[q][d].x));
            } else {
                if constexpr (NS > 0) acc64[r][0] += s0;
#pragma unroll
                for (int d = 0; d < D; ++d)
                    acc64[r][NS + d] += (double)p.s * (double)((r & 1) ? Sp[q][d].y : Sp[q][d].x);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= row_end) continue;
        if (p.split > 1) {
            double *dst = p.part + ((int64_t)sp * p.M + i) * C;
#pragma unroll
            for (int c = 0; c < C; ++c) dst[c] = acc64[r][c];
            continue;
        }
        if constexpr (NS > 0) {
            const double v = acc64[r][0] * p.scale_sum;
            if (p.out_f64) ((double *)p.out)[i] = v;
            else ((float *)p.out)[i] = (float)v;
        }
        double gs = p.scale_grad;
        if (p.g) gs *= (double)__ldg(p.g + i);
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const double v = acc64[r][NS + c] * gs;
            if (MODE == 2) p.out_grad[i * D + c] = (float)v;
            else if (p.out_f64) ((double *)p.out)[i * D + c] = v;
            else ((float *)p.out)[i * D + c] = (float)v;
        }
    }
}

// CTAs per SM the register allocation must allow (the 16 K registers of each SM sub-partition)
template <int MODE, int D, int E, int R, bool SMM>
constexpr int sum_min_blocks() {
    if (SMM) return 2;
    if ((MODE == 0 || MODE == 3) && E == 1 && D <= 3 && R == 4) return GENRED_SUM_MINB;
    if ((MODE == 1 || MODE == 2) && D + E <= 4 && E == 1 && R == GENRED_GRAD_R) return GENRED_GRAD_MINB;
    return 2;
}

// Split-j merge folded into the pair-loop kernel: the CTA that finishes a
// row tile last (arrival counter, release/acquire through __threadfence) sums the tile's S
// partials in split order 0..S-1 -- the order and arithmetic of sum_finalize_kernel, so the
// result is bitwise that of the two-kernel path -- and resets the counter for the next call.
template <int MODE, int D, int E, int R>
__device__ __forceinline__ void sum_tile_merge(const SumParams &p, int64_t itile, int64_t row0, int64_t row_end) {
    using Cfg = SumCfg<MODE, D, E>;
    constexpr int NS = Cfg::NS, NG = Cfg::NG, C = Cfg::C;
    __shared__ int s_last;
    __syncthreads();                                   // every thread's partials are stored
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(p.tile_done + itile, 1u);
        s_last = prev == (unsigned)(p.split - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();                                   // acquire: the other CTAs' partials
    const int64_t rows = min(row_end, row0 + (int64_t)(kConsumerWarps * 32 * R)) - row0;
    for (int64_t t = threadIdx.x; t < rows * C; t += blockDim.x) {
        const int64_t i = row0 + t / C;
        const int c = (int)(t % C);
        double acc = 0.0;
#pragma unroll 8
        for (int q = 0; q < p.split; ++q) acc += __ldcg(p.part + ((int64_t)q * p.M + i) * C + c);   // 8 loads in flight
        if (c < NS) {
            const double v = acc * p.scale_sum;
            if (p.out_f64) ((double *)p.out)[i * NS + c] = v;
            else ((float *)p.out)[i * NS + c] = (float)v;
        } else if constexpr (NG > 0) {
            double v = acc * p.scale_grad;
            if (E == 1 && p.g) v *= (double)__ldg(p.g + i);
            const int dc = c - NS;
            if (MODE == 2) p.out_grad[i * D + dc] = (float)v;
            else if (p.out_f64) ((double *)p.out)[i * D + dc] = v;
            else ((float *)p.out)[i * D + dc] = (float)v;
        }
    }
    if (threadIdx.x == 0) p.tile_done[itile] = 0u;     // ready for the next call on the stream
}

// The grid walks the work units w = blockIdx.x, blockIdx.x + gridDim.x, ...; a unit is (row
// tile, j-split), (row group, j-split) in the small-M mode, or one block-sparse range unit.  The
// launch uses one CTA per unit (measured faster than a persistent grid, see sum_kernel.cu).
template <int MODE, int D, int E, int R, bool SMM = false>
__global__ void __launch_bounds__(kThreads, sum_min_blocks<MODE, D, E, R, SMM>())
sum_kernel(const SumParams p) {
    using Cfg = SumCfg<MODE, D, E>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    for (int64_t w = blockIdx.x; w < p.n_work; w += gridDim.x) {
    if (w != blockIdx.x) __syncthreads();            // the previous unit is done with shared memory
    // this unit's j-range: record pairs [q0, q0 + npc), streamed in tiles of PAIRS
    int64_t row0, row_end, q0, npc;
    int sp;
    if (p.units) {                                     // block-sparse: rows of one cluster
        const RangeUnit u = p.units[w];
        row0 = u.row0; row_end = u.row_end; sp = 0;
        q0 = u.tile0 * Cfg::PAIRS; npc = u.ntiles * Cfg::PAIRS;
    } else if (SMM) {
        // split-major: concurrently running CTAs share a j-range (L2 reuse across row groups)
        const int64_t ngroups = (p.M + R - 1) / R;
        sp = (int)(w / ngroups);
        row0 = (int64_t)(w % ngroups) * R;
        row_end = p.M;
        q0 = (int64_t)sp * p.pairs_per_split;
        npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);
    } else {
        // split-major (large j-record sets): the CTAs resident at any time stream the same j-split,
        // whose records then stay in L2 (one DRAM read per split, not one per wave)
        int64_t itile;
        if (p.split_major) {
            itile = w % p.itiles;
            sp = (int)(w / p.itiles);
        } else {
            itile = w / p.split;
            sp = (int)(w % p.split);
        }
        q0 = (int64_t)sp * p.pairs_per_split;
        npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);   // empty: zero partial
        row0 = itile * (int64_t)(kConsumerWarps * 32 * R);
        row_end = p.M;
    }
    const int nt = (int)((npc + Cfg::PAIRS - 1) / Cfg::PAIRS);
    const int last_np = (int)(npc - (int64_t)(nt > 0 ? nt - 1 : 0) * Cfg::PAIRS);
    const uint32_t last_bytes = (uint32_t)last_np * Cfg::RS * 4u;   // a partial last tile is copied partially

    JRing<Cfg::STAGES> ring;
    if constexpr (MODE != 3) {
        const Geo geo = geo_decode(p.geo, D, p.s);     // same decision as the pack kernel
        ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * Cfg::RS, nt, kConsumerWarps, last_bytes);
        if (geo.expanded) sum_body<MODE, D, E, R, true, SMM>(p, ring, nt, last_np, row0, row_end, sp, geo);
        else {
            bool local = false;
            if constexpr (MODE == 0 && !SMM && D <= 3) {
                if (p.centers && !p.units) {           // tile-centred form (R18j)
                    sum_body_local<D, E, R>(p, ring, nt, last_np, row0, row_end, sp, q0 / Cfg::PAIRS);
                    local = true;
                }
            } else if constexpr ((MODE == 1 || MODE == 2) && E == 1 && D <= 3 && R == 4 && !SMM && Cfg::BY) {
                if (p.centers && !p.units) {
                    sum_body_local_grad<MODE, D>(p, ring, nt, last_np, row0, row_end, sp, q0 / Cfg::PAIRS);
                    local = true;
                }
            }
            if (!local) sum_body<MODE, D, E, R, false, SMM>(p, ring, nt, last_np, row0, row_end, sp, geo);
        }
    } else {
        ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * Cfg::RS, nt, kConsumerWarps, last_bytes);
        Geo geo{};
        sum_body<MODE, D, E, R, false, SMM>(p, ring, nt, last_np, row0, row_end, sp, geo);
    }
    if (!SMM && p.tile_done && !p.units)
        sum_tile_merge<MODE, D, E, R>(p, p.split_major ? w % p.itiles : w / p.split, row0, row_end);
    }
}


// Small problems in ONE launch (max(M, N) <= kFusedBoxMax, C1-like; launch-latency bound): each
// CTA builds the direct-form j-records of its own j-split in shared memory straight from y and b
// (the pack kernel's direct layout: -y raw, w = 0, b; zero records past N), so there is no pack
// launch and no bounding box (the direct form on raw differences, reading R18e, needs none), runs
// the unchanged pair loop on them, and the last CTA of each row tile merges the split partials
// (sum_tile_merge).  The pair arithmetic is that of sum_kernel's direct form.
// Cluster merge (CL = split <= 8): the split's CTAs of one row tile form a thread-block cluster;
// each leaves its fp64 partials in its own shared memory, and after a cluster barrier CTA q of
// the cluster merges rows q, q + S, ... reading every CTA's partials through distributed shared
// memory in split order 0..S-1 (the finalize kernel's order and arithmetic), then writes the
// outputs.  No global partials, no arrival counters, no threadfence round trips.
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double ld_dsmem_f64(const double *local, uint32_t rank) {
    uint32_t a = smem_u32(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}

template <int MODE, int D, int E, int R>
__device__ __forceinline__ void sum_cluster_merge(const SumParams &p, const double *part_s, int rank,
                                                  int64_t row0) {
    using Cfg = SumCfg<MODE, D, E>;
    constexpr int NS = Cfg::NS, NG = Cfg::NG, C = Cfg::C;
    const int64_t rows = min(p.M, row0 + (int64_t)(kConsumerWarps * 32 * R)) - row0;
    for (int64_t t = (int64_t)rank * blockDim.x + threadIdx.x; t < rows * C; t += (int64_t)p.split * blockDim.x) {
        const int64_t i = row0 + t / C;
        const int c = (int)(t % C);
        double acc = 0.0;
        for (int q = 0; q < p.split; ++q) acc += ld_dsmem_f64(part_s + t, (uint32_t)q);
        if (c < NS) {
            const double v = acc * p.scale_sum;
            if (p.out_f64) ((double *)p.out)[i * NS + c] = v;
            else ((float *)p.out)[i * NS + c] = (float)v;
        } else if constexpr (NG > 0) {
            double v = acc * p.scale_grad;
            if (E == 1 && p.g) v *= (double)__ldg(p.g + i);
            const int dc = c - NS;
            if (MODE == 2) p.out_grad[i * D + dc] = (float)v;
            else if (p.out_f64) ((double *)p.out)[i * D + dc] = v;
            else ((float *)p.out)[i * D + dc] = (float)v;
        }
    }
}

template <int MODE, int D, int E, int R>
__global__ void __launch_bounds__(kThreads, 2)
sum_small_kernel(SumParams p, const float *__restrict__ y, const float *__restrict__ b, int64_t N,
                 int cluster_merge) {
    using Cfg = SumCfg<MODE, D, E>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // [cluster partials: kThreads R rows x C fp64][j-records]
    double *part_s = reinterpret_cast<double *>(smem_raw);
    float *recs = reinterpret_cast<float *>(smem_raw + (cluster_merge ? kThreads * R * Cfg::C * 8 : 0));
    const int64_t itile = blockIdx.x / p.split;
    const int sp = (int)(blockIdx.x % p.split);
    const int64_t q0 = (int64_t)sp * p.pairs_per_split;
    const int npc = (int)max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);
    const int64_t row0 = itile * (int64_t)(kConsumerWarps * 32 * R);
    // this thread's x rows: prefetched into L1 now, so the pair loop's loads do not add a second
    // memory round trip after the j-records'
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + threadIdx.x;
        if (i < p.M) asm volatile("prefetch.global.L1 [%0];" ::"l"(p.x + i * D));
    }
    // one pass: thread t builds whole record pairs t, t + 256, ... (zeros past N and in the pad)
    for (int pp = threadIdx.x; pp < npc; pp += kThreads) {
        float rec[Cfg::RS];
#pragma unroll
        for (int k = 0; k < Cfg::RS; ++k) rec[k] = 0.0f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t j = 2 * (q0 + pp) + h;
            if (j >= N) continue;                          // zero record: contributes nothing
#pragma unroll
            for (int d = 0; d < D; ++d) rec[2 * d + h] = -__ldg(y + j * D + d);
#pragma unroll
            for (int e = 0; e < E; ++e) rec[Cfg::BOFF + 2 * e + h] = b ? __ldg(b + j * E + e) : 1.0f;
        }
        float4 *dst = reinterpret_cast<float4 *>(recs + pp * Cfg::RS);
#pragma unroll
        for (int q = 0; q < Cfg::RS / 4; ++q) dst[q] = make_float4(rec[4 * q], rec[4 * q + 1], rec[4 * q + 2], rec[4 * q + 3]);
    }
    __syncthreads();
    const int nt = (npc + Cfg::PAIRS - 1) / Cfg::PAIRS;
    const int last_np = npc - (nt > 0 ? nt - 1 : 0) * Cfg::PAIRS;
    SmemTiles ring{recs, Cfg::TILE_FLOATS};
    Geo geo{};
    geo.expanded = false;
    if (cluster_merge) p.part_smem = part_s;
    sum_body<MODE, D, E, R, false, false>(p, ring, nt, last_np, row0, p.M, sp, geo);
    if (cluster_merge) {
        cluster_barrier();                             // every CTA's partials are in its smem
        sum_cluster_merge<MODE, D, E, R>(p, part_s, sp, row0);
        cluster_barrier();                             // no CTA leaves while others read its smem
    } else if (p.tile_done) {
        sum_tile_merge<MODE, D, E, R>(p, itile, row0, p.M);
    }
}

}  // namespace genred
