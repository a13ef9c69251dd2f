// lse_kernel.cu -- streaming, max-shifted log-sum-exp reduction:
//
//     F_ij = -|x_i - y_j|^2 / eps + h_j ,     a_i = log sum_j exp(F_ij)          (Eq. 1)
//
// evaluated in the log2 domain: v_ij = log2(e) F_ij = negc |x_i - y_j|^2 + h'_j with
// negc = -log2(e)/eps, h' = log2(e) h.  Each row keeps a reference m_i (log2 units) and
// s_i = sum_j 2^(v_ij - m_i) (reading R6 in DESIGN.md):
//   * RAW differences d = x - y (no pre-scaling of coordinates: the query shift of a pre-scaled
//     x costs up to 1.35e-6 in a_i);
//   * t = fma(negc, |d|^2, h'_hi - m) then MUFU.EX2, times c = 2^(h' - h'_hi) when h != 0
//     (reading R6c); two j's per packed FADD2/FFMA2;
//   * lazy rescale: terms are summed per 16-j sub-chunk into a fresh fp32 pair; if that sum
//     exceeds 2^16 (or overflows) the sub-chunk is discarded, m is
//     set to the sub-chunk's exact max v (never m + t), s is rescaled in fp64 and the sub-chunk
//     is recomputed -- rare (a few times per row);
//   * fp32 partials are promoted to fp64 every 128 j; the output is finalised in fp64:
//     a_i = ln2 (m_i + log2 s_i).
// Pipeline and tiling are those of sum_kernel.cu (bulk-copy ring of 512-record j-tiles); the
// small-M variant (lse_smm_kernel) gives each CTA a few rows whose threads split j.
#include <math.h>

#include "device.cuh"
#include "internal.h"

namespace genred {

// Lazy rescale: a sub-chunk is accepted while its fp32 sum of 2 kSub terms 2^(v - m) stays
// <= kSumMax (or is not finite): every accepted term is then < 2^16, so the reference m may lag
// the running max by up to 16 (log2) without overflow or loss of relative precision, and the
// check costs one FMNMX + FSETP per row and sub-chunk instead of a max per pair.
constexpr float kSumMax = 65536.0f;
#ifndef GENRED_LSE_SUB
#define GENRED_LSE_SUB 16
#endif
// 3 CTAs/SM (80 registers; the spills are outside the pair loop) with the row-pair loop:
// C3-like LSE (1e6 x 1e6, eps = 0.05) 13.42 -> 13.60 pairs/clk/SM; the j-packed loop of round 1
// at 2 CTAs/SM measured 12.98 (B200, round 2).
#ifndef GENRED_LSE_MINB
#define GENRED_LSE_MINB 4
#endif
#ifndef GENRED_LSE_MINB_BIG
#define GENRED_LSE_MINB_BIG 2
#endif
// Row-pair packing (as the gradient modes, sum_body.cuh GENRED_GRAD_RP): the packed lanes hold
// two ROWS, the record's -y_d is a broadcast scalar operand, one j at a time.
#ifndef GENRED_LSE_RP
#define GENRED_LSE_RP 1
#endif
constexpr int kSub = GENRED_LSE_SUB;  // record pairs per sub-chunk (2 kSub j)
constexpr int kPromote = 64 / kSub;   // sub-chunks per fp64 promotion (128 j)
static_assert(kSplitGrain % kSub == 0, "j-splits must hold whole sub-chunks");

template <int D, bool HZ>
struct LseCfg {
    // records: 2D coordinates (-y), then for h != 0 the pair of fp32 h'hi and h'lo
    static constexpr int RS = ((2 * D + (HZ ? 0 : 4)) + 3) / 4 * 4;
    static constexpr int PAIRS = kTileJ / 2;
    static constexpr int TILE_FLOATS = PAIRS * RS;
    static constexpr int STAGE_BYTES = TILE_FLOATS * 4;
    static constexpr int SMEM = JRing<kStages>::smem_bytes(TILE_FLOATS);
};

struct LseParams {
    const float4 *centers = nullptr;   // tile-centred form: per 512-j tile (c_k, r_k^2 or -1)
    float s = 0.0f;                    // tile-centred form: sqrt(log2(e) / eps)
    const float *x, *J;
    int64_t M;
    int split;
    int64_t pairs_per_split, npv;      // record-pair j-splits (see SumParams)
    float negc;
    void *out;
    int out_f64;
    double *state;
    const RangeUnit *units;   // block-sparse ranges: one CTA per unit (rows of one cluster)
};

struct LseRescale {
    float m;
    double s64;
    float c1;
};

// Out of line so that its registers do not burden the hot loop.
template <int D, bool HZ, int RS, int NSUB = kSub>
__device__ __noinline__ LseRescale lse_rescale(const float *base, const float (&xr)[D], float negc,
                                               float m_old, double s64, float2 s32) {
    float vmax = -INFINITY;
    for (int q = 0; q < NSUB; ++q) {
        const float *rec = base + q * RS;
        for (int h = 0; h < 2; ++h) {
            float q1 = 0.f;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const float dd = xr[d] + rec[2 * d + h];
                q1 = fmaf(dd, dd, q1);
            }
            float hv = 0.0f;
            if constexpr (!HZ) hv = rec[2 * D + h];
            vmax = fmaxf(vmax, fmaf(q1, negc, hv));
        }
    }
    LseRescale o;
    o.m = fmaxf(vmax, m_old);
    o.s64 = (s64 + (double)s32.x + (double)s32.y) * exp2((double)m_old - (double)o.m);
    float c1 = 0.f;
    for (int q = 0; q < NSUB; ++q) {
        const float *rec = base + q * RS;
        for (int h = 0; h < 2; ++h) {
            float q1 = 0.f;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const float dd = xr[d] + rec[2 * d + h];
                q1 = fmaf(dd, dd, q1);
            }
            float hmv = -o.m, cj = 1.0f;
            if constexpr (!HZ) { hmv = rec[2 * D + h] + (-o.m); cj = rec[2 * D + 2 + h]; }
            c1 = fmaf(ex2(fmaf(q1, negc, hmv)), cj, c1);
        }
    }
    o.c1 = c1;
    return o;
}

template <int D, int R>
constexpr int lse_min_blocks(bool hz) {
    // h = 0: 4 CTAs/SM (64 registers, spills outside the pair loop) measured 13.81 pairs/clk/SM
    // against 13.61 at 3; with h the 3-CTA build is faster (12.03 against 11.78)
    return (D <= 3 && R % 2 == 0) ? (R > 4 ? GENRED_LSE_MINB_BIG : (hz ? GENRED_LSE_MINB : 3)) : 2;
}

template <int D, int R, bool HZ>
__global__ void __launch_bounds__(kThreads, lse_min_blocks<D, R>(HZ)) lse_kernel(const LseParams p) {
    using Cfg = LseCfg<D, HZ>;
    constexpr int RS = Cfg::RS;
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
        npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);
        row0 = itile * (int64_t)(kConsumerWarps * 32 * R);
        row_end = p.M;
    }
    const int nt = (int)((npc + Cfg::PAIRS - 1) / Cfg::PAIRS);
    const int last_np = (int)(npc - (int64_t)(nt > 0 ? nt - 1 : 0) * Cfg::PAIRS);

    JRing<kStages> ring;
    ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * RS, nt, kConsumerWarps, (uint32_t)last_np * RS * 4u);

    const int ct = threadIdx.x;
    const float negc = p.negc;
    const float2 negc2 = dup2(negc);
    float xr[R][D];
    float m[R];
    double s64[R];
    float2 s32[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        const bool ok = i < row_end;
#pragma unroll
        for (int d = 0; d < D; ++d) xr[r][d] = ok ? __ldg(p.x + i * D + d) : 0.0f;
        m[r] = kLseSentinel;
        s64[r] = 0.0;
        s32[r] = make_float2(0.f, 0.f);
    }

    constexpr bool RP = GENRED_LSE_RP && (R % 2 == 0);
    if constexpr (RP) {
    // ---- row-pair mode: lanes = rows (2q, 2q + 1) -------------------------------------------
    constexpr int RQ = R / 2;
    float2 X2[RQ][D], NM2[RQ], S32[RQ];
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
#pragma unroll
        for (int d = 0; d < D; ++d) X2[q][d] = make_float2(xr[2 * q][d], xr[2 * q + 1][d]);
        NM2[q] = make_float2(-m[2 * q], -m[2 * q + 1]);
        S32[q] = make_float2(0.f, 0.f);
    }
    for (int k = 0; k < nt; ++k) {
        const float *tile = ring.acquire(k);
        const int nsc = (k == nt - 1 ? last_np : Cfg::PAIRS) / kSub;     // sub-chunks in this tile
        for (int sc = 0; sc < nsc; ++sc) {
            const float *base = tile + sc * kSub * RS;
            float2 cs[RQ];
#pragma unroll
            for (int q = 0; q < RQ; ++q) cs[q] = make_float2(0.f, 0.f);
#pragma unroll
            for (int pq = 0; pq < kSub; ++pq) {
                float f[RS];
#pragma unroll
                for (int u = 0; u < RS / 4; ++u) {
                    const float4 v = lds128(base + pq * RS + 4 * u);
                    f[4 * u + 0] = v.x; f[4 * u + 1] = v.y; f[4 * u + 2] = v.z; f[4 * u + 3] = v.w;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int q = 0; q < RQ; ++q) {
                        float2 dd = add2(X2[q][0], dup2(f[h]));              // x - y (raw, R6)
                        float2 q2 = mul2(dd, dd);
#pragma unroll
                        for (int d = 1; d < D; ++d) {
                            dd = add2(X2[q][d], dup2(f[2 * d + h]));
                            q2 = fma2(dd, dd, q2);
                        }
                        const float2 hm = HZ ? NM2[q] : add2(NM2[q], dup2(f[2 * D + h]));   // h'_hi - m
                        const float2 t = fma2(q2, negc2, hm);
                        const float2 e = make_float2(ex2(t.x), ex2(t.y));
                        cs[q] = HZ ? add2(cs[q], e) : fma2(e, dup2(f[2 * D + 2 + h]), cs[q]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                if (!(fmaxf(cs[q].x, cs[q].y) <= kSumMax)) {           // rare: per-row rescale
#pragma unroll
                    for (int l = 0; l < 2; ++l) {
                        const int r = 2 * q + l;
                        const float c = l ? cs[q].y : cs[q].x;
                        if (c <= kSumMax) {
                            if (l) S32[q].y += c; else S32[q].x += c;
                            continue;
                        }
                        float xrow[D];
#pragma unroll
                        for (int d = 0; d < D; ++d) xrow[d] = l ? X2[q][d].y : X2[q][d].x;
                        const float sl = l ? S32[q].y : S32[q].x;
                        const LseRescale rs = lse_rescale<D, HZ, RS>(base, xrow, negc, m[r], s64[r],
                                                                     make_float2(sl, 0.f));
                        m[r] = rs.m;
                        s64[r] = rs.s64;
                        if (l) { S32[q].y = rs.c1; NM2[q].y = -rs.m; } else { S32[q].x = rs.c1; NM2[q].x = -rs.m; }
                    }
                } else {
                    S32[q] = add2(S32[q], cs[q]);
                }
            }
            if ((sc + 1) % kPromote == 0) {
#pragma unroll
                for (int q = 0; q < RQ; ++q) {
                    s64[2 * q] += (double)S32[q].x;
                    s64[2 * q + 1] += (double)S32[q].y;
                    S32[q] = make_float2(0.f, 0.f);
                }
            }
        }
        ring.release(k);
    }
#pragma unroll
    for (int q = 0; q < RQ; ++q) {                 // the (at most) partial last promotion
        s32[2 * q] = make_float2(S32[q].x, 0.f);
        s32[2 * q + 1] = make_float2(S32[q].y, 0.f);
    }
    } else {
    for (int k = 0; k < nt; ++k) {
        const float *tile = ring.acquire(k);
        const int nsc = (k == nt - 1 ? last_np : Cfg::PAIRS) / kSub;     // sub-chunks in this tile
        for (int sc = 0; sc < nsc; ++sc) {
            const float *base = tile + sc * kSub * RS;
            float2 cs[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                cs[r] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int q = 0; q < kSub; ++q) {
                float f[RS];
#pragma unroll
                for (int u = 0; u < RS / 4; ++u) {
                    const float4 v = lds128(base + q * RS + 4 * u);
                    f[4 * u + 0] = v.x; f[4 * u + 1] = v.y; f[4 * u + 2] = v.z; f[4 * u + 3] = v.w;
                }
                float2 ny[D];
#pragma unroll
                for (int d = 0; d < D; ++d) ny[d] = make_float2(f[2 * d], f[2 * d + 1]);
                // with h: h'_hi enters the exponent, c = 2^(h'_lo) multiplies the term (R6c)
                float2 hhi = make_float2(0.f, 0.f), hc = make_float2(1.f, 1.f);
                if constexpr (!HZ) {
                    hhi = make_float2(f[2 * D], f[2 * D + 1]);
                    hc = make_float2(f[2 * D + 2], f[2 * D + 3]);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 dd = add2(dup2(xr[r][0]), ny[0]);
                    float2 q2 = mul2(dd, dd);
#pragma unroll
                    for (int d = 1; d < D; ++d) {
                        dd = add2(dup2(xr[r][d]), ny[d]);
                        q2 = fma2(dd, dd, q2);
                    }
                    const float2 hm = HZ ? dup2(-m[r]) : add2(hhi, dup2(-m[r]));   // (h'_hi - m)
                    const float2 t = fma2(q2, negc2, hm);          // v - m, log2 units
                    const float2 e = make_float2(ex2(t.x), ex2(t.y));
                    cs[r] = HZ ? add2(cs[r], e) : fma2(e, hc, cs[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!(fmaxf(cs[r].x, cs[r].y) <= kSumMax)) {          // also catches inf / NaN
                    // rare path (a few times per row): new reference m = exact max of v over the
                    // sub-chunk, fp64 rescale of the accumulated sum, sub-chunk recomputed
                    const LseRescale rs = lse_rescale<D, HZ, RS>(base, xr[r], negc, m[r], s64[r], s32[r]);
                    m[r] = rs.m;
                    s64[r] = rs.s64;
                    s32[r] = make_float2(rs.c1, 0.f);
                } else {
                    s32[r] = add2(s32[r], cs[r]);
                }
            }
            if ((sc + 1) % kPromote == 0) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    s64[r] += (double)s32[r].x + (double)s32[r].y;
                    s32[r] = make_float2(0.f, 0.f);
                }
            }
        }
        ring.release(k);
    }
    }   // RP

#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= row_end) continue;
        const double stot = s64[r] + (double)s32[r].x + (double)s32[r].y;
        if (p.split > 1) {
            p.state[((int64_t)sp * p.M + i) * 2 + 0] = (double)m[r];
            p.state[((int64_t)sp * p.M + i) * 2 + 1] = stot;
            continue;
        }
        const double a = (stot > 0.0) ? 0.69314718055994530942 * ((double)m[r] + log2(stot)) : -INFINITY;
        if (p.out) {
            if (p.out_f64) ((double *)p.out)[i] = a;
            else ((float *)p.out)[i] = (float)a;
        }
        if (p.state) {
            p.state[2 * i + 0] = (double)m[r];
            p.state[2 * i + 1] = stot;
        }
    }
}

// ---- tile-centred form (R18j; records by tile_order.cu) ------------------------------
// y in Hilbert order; a 512-j tile k whose radius (s units, s = sqrt(log2(e)/eps)) is at most
// kLseLocalR2Max carries y'' = s (y - c_k) and w = fl32(h' - |y''|^2) (+ c = 2^(rest) with h),
// so that for x'' = s (x - c_k) (from raw x)
//     v_ij = -|x'' - y''|^2 + h'_j = o_i + (2 x''.y'' + w_j),     o_i = -|x''|^2  (fp64, per tile)
// and a pair costs FADD (w - m') + D FFMA + MUFU.EX2 + 1 accumulate: 5 FP32 lane-ops against
// the raw-difference loop's 8, so MUFU becomes the only bound.  Wider tiles keep the direct
// layout and the raw-difference loop (R6).  Each row keeps its reference M_i in fp64; at a tile
// start the fp32 reference of the tile's frame is m' = fl32(M_i - o_i) and M_i is moved to
// m' + o_i exactly (the fp64 sum is rescaled by 2^(M_old - M_new), a few ulps of m'), so every
// fp32 term 2^(u - m') is relative to M_i.  The lazy rescale (kSumMax) works in the tile frame.
template <int D, bool HZ>
struct LseLocCfg {
    static constexpr int RS = ((2 * D + 2 + (HZ ? 0 : 2)) + 3) / 4 * 4;
    static constexpr int PAIRS = kTileJ / 2;
    static constexpr int TILE_FLOATS = PAIRS * RS;
    static constexpr int SMEM = JRing<kStages>::smem_bytes(TILE_FLOATS);
};
int lse_local_record_stride(int D, bool hz) { return ((2 * D + 2 + (hz ? 0 : 2)) + 3) / 4 * 4; }

// Rare path of the tile-centred loop: exact max of the sub-chunk's values in the tile frame, the
// fp64 sum rescaled, the sub-chunk recomputed (as lse_rescale).  xv: 2 x'' (centred tile) or raw x.
template <int D, bool HZ, int RS>
__device__ __noinline__ LseRescale lse_local_rescale(const float *base, const float (&xv)[D], bool loc, float negc,
                                                     float m_old, double s64, float s32) {
    auto value = [&](const float *rec, int h) {
        if (loc) {
            float u = rec[2 * D + h];
#pragma unroll
            for (int d = 0; d < D; ++d) u = fmaf(xv[d], rec[2 * d + h], u);
            return u;
        }
        float q1 = 0.f;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const float dd = xv[d] + rec[2 * d + h];
            q1 = fmaf(dd, dd, q1);
        }
        return fmaf(q1, negc, HZ ? 0.0f : rec[2 * D + h]);
    };
    float vmax = -INFINITY;
    for (int q = 0; q < kSub; ++q)
        for (int h = 0; h < 2; ++h) vmax = fmaxf(vmax, value(base + q * RS, h));
    LseRescale o;
    o.m = fmaxf(vmax, m_old);
    o.s64 = (s64 + (double)s32) * exp2((double)m_old - (double)o.m);
    float c1 = 0.f;
    for (int q = 0; q < kSub; ++q)
        for (int h = 0; h < 2; ++h) {
            const float *rec = base + q * RS;
            const float cj = HZ ? 1.0f : rec[2 * D + 2 + h];
            c1 = fmaf(ex2(value(rec, h) - o.m), cj, c1);
        }
    o.c1 = c1;
    return o;
}

// (1/8 of the exponentials on the FP32 pipe, as the Sum: 14.54 against 14.63 pairs/clk/SM with
// h = 0 and 14.14 against 14.46 with h at C3's shape -- not used; 3 CTAs/SM the same as 4)
#ifndef GENRED_CEN_PREFETCH
#define GENRED_CEN_PREFETCH 1
#endif
#ifndef GENRED_LSE_POLY
#define GENRED_LSE_POLY 0
#endif
#ifndef GENRED_LSE_LOC_MINB
#define GENRED_LSE_LOC_MINB 4
#endif

template <int D, bool HZ>
__global__ void __launch_bounds__(kThreads, HZ ? GENRED_LSE_LOC_MINB : 3) lse_local_kernel(const LseParams p) {
    using Cfg = LseLocCfg<D, HZ>;
    constexpr int RS = Cfg::RS;
    constexpr int R = 4, RQ = 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int64_t itile = blockIdx.x / p.split;
    const int sp = (int)(blockIdx.x % p.split);
    const int64_t q0 = (int64_t)sp * p.pairs_per_split;             // a multiple of PAIRS
    const int64_t npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);
    const int64_t row0 = itile * (int64_t)(kConsumerWarps * 32 * R);
    const int nt = (int)((npc + Cfg::PAIRS - 1) / Cfg::PAIRS);
    const int last_np = (int)(npc - (int64_t)(nt > 0 ? nt - 1 : 0) * Cfg::PAIRS);
    JRing<kStages> ring;
    ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * RS, nt, kConsumerWarps, (uint32_t)last_np * RS * 4u);

    const int ct = threadIdx.x;
    const float negc = p.negc;
    const float2 negc2 = dup2(negc);
    double Mr[R], s64[R];
#pragma unroll
    for (int r = 0; r < R; ++r) { Mr[r] = (double)kLseSentinel; s64[r] = 0.0; }
    float2 X2[RQ][D], NM2[RQ], S32[RQ];
#pragma unroll
    for (int q = 0; q < RQ; ++q) S32[q] = make_float2(0.f, 0.f);
    const int64_t tile0 = q0 / Cfg::PAIRS;
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
        // this tile's frame: 2 x'' (or raw x), m' = fl32(M - o), M moved to m' + o
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
            double o = 0.0;
            float xv[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const float xd = i < p.M ? __ldg(p.x + i * D + d) : 0.0f;
                if (loc) {
                    const float h = p.s * (xd - cc[d]);
                    xv[d] = 2.0f * h;
                    const double hd = 0.5 * (double)xv[d];           // = h exactly
                    o = fma(-hd, hd, o);
                } else {
                    xv[d] = xd;
                }
            }
            const float mp = (float)(Mr[r] - o);
            const double Mn = (double)mp + o;
            if (s64[r] != 0.0) {
                const double dl = (Mr[r] - Mn) * 0.69314718055994530942;     // ln of 2^(M_old - M_new)
                s64[r] *= fabs(dl) < 1e-4 ? 1.0 + dl * (1.0 + dl * (0.5 + dl * (1.0 / 6.0))) : exp(dl);
            }
            Mr[r] = Mn;
#pragma unroll
            for (int d = 0; d < D; ++d) { if (r & 1) X2[r >> 1][d].y = xv[d]; else X2[r >> 1][d].x = xv[d]; }
            if (r & 1) NM2[r >> 1].y = -mp; else NM2[r >> 1].x = -mp;
        }
        const float *tile = ring.acquire(k);
        const int nsc = (k == nt - 1 ? last_np : Cfg::PAIRS) / kSub;
        for (int sc = 0; sc < nsc; ++sc) {
            const float *base = tile + sc * kSub * RS;
            float2 cs[RQ];
#pragma unroll
            for (int q = 0; q < RQ; ++q) cs[q] = make_float2(0.f, 0.f);
            if (loc) {
#pragma unroll
                for (int pq = 0; pq < kSub; ++pq) {
                    float f[RS];
#pragma unroll
                    for (int u = 0; u < RS / 4; ++u) {
                        const float4 v = lds128(base + pq * RS + 4 * u);
                        f[4 * u + 0] = v.x; f[4 * u + 1] = v.y; f[4 * u + 2] = v.z; f[4 * u + 3] = v.w;
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
#pragma unroll
                        for (int q = 0; q < RQ; ++q) {
                            float2 t = add2(NM2[q], dup2(f[2 * D + h]));                 // w - m'
#pragma unroll
                            for (int d = 0; d < D; ++d) t = fma2(X2[q][d], dup2(f[2 * d + h]), t);   // + 2x''.y''
                            float2 e;
                            if (GENRED_LSE_POLY && q == RQ - 1 && h == 0 && (pq & 1) == 0) {
                                // 1/8 of the exponentials on the FP32 pipe (as the Sum, sum_body.cuh);
                                // t clamped to [-126, 64]: 2^64 still trips the kSumMax check
                                const float2 tc = make_float2(fminf(fmaxf(t.x, -126.0f), 64.0f),
                                                              fminf(fmaxf(t.y, -126.0f), 64.0f));
                                e = ex2_poly2(tc);
                            } else {
                                e = make_float2(ex2(t.x), ex2(t.y));
                            }
                            cs[q] = HZ ? add2(cs[q], e) : fma2(e, dup2(f[2 * D + 2 + h]), cs[q]);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int pq = 0; pq < kSub; ++pq) {
                    float f[RS];
#pragma unroll
                    for (int u = 0; u < RS / 4; ++u) {
                        const float4 v = lds128(base + pq * RS + 4 * u);
                        f[4 * u + 0] = v.x; f[4 * u + 1] = v.y; f[4 * u + 2] = v.z; f[4 * u + 3] = v.w;
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
#pragma unroll
                        for (int q = 0; q < RQ; ++q) {
                            float2 dd = add2(X2[q][0], dup2(f[h]));                       // x - y (raw, R6)
                            float2 q2 = mul2(dd, dd);
#pragma unroll
                            for (int d = 1; d < D; ++d) {
                                dd = add2(X2[q][d], dup2(f[2 * d + h]));
                                q2 = fma2(dd, dd, q2);
                            }
                            const float2 hm = HZ ? NM2[q] : add2(NM2[q], dup2(f[2 * D + h]));
                            const float2 t = fma2(q2, negc2, hm);
                            const float2 e = make_float2(ex2(t.x), ex2(t.y));
                            cs[q] = HZ ? add2(cs[q], e) : fma2(e, dup2(f[2 * D + 2 + h]), cs[q]);
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                if (!(fmaxf(cs[q].x, cs[q].y) <= kSumMax)) {           // rare: per-row rescale
#pragma unroll
                    for (int l = 0; l < 2; ++l) {
                        const int r = 2 * q + l;
                        const float c = l ? cs[q].y : cs[q].x;
                        if (c <= kSumMax) {
                            if (l) S32[q].y += c; else S32[q].x += c;
                            continue;
                        }
                        float xrow[D];
#pragma unroll
                        for (int d = 0; d < D; ++d) xrow[d] = l ? X2[q][d].y : X2[q][d].x;
                        const float m_old = -(l ? NM2[q].y : NM2[q].x);
                        const LseRescale rs = lse_local_rescale<D, HZ, RS>(base, xrow, loc, negc, m_old, s64[r],
                                                                           l ? S32[q].y : S32[q].x);
                        // M = m' + o with this tile's o = -|x''|^2 (recomputed bitwise as at the
                        // tile start; 0 for a direct tile)
                        double o = 0.0;
                        if (loc) {
#pragma unroll
                            for (int d = 0; d < D; ++d) {
                                const double hd = 0.5 * (double)xrow[d];
                                o = fma(-hd, hd, o);
                            }
                        }
                        Mr[r] = (double)rs.m + o;
                        s64[r] = rs.s64;
                        if (l) { S32[q].y = rs.c1; NM2[q].y = -rs.m; } else { S32[q].x = rs.c1; NM2[q].x = -rs.m; }
                    }
                } else {
                    S32[q] = add2(S32[q], cs[q]);
                }
            }
            if ((sc + 1) % kPromote == 0) {
#pragma unroll
                for (int q = 0; q < RQ; ++q) {
                    s64[2 * q] += (double)S32[q].x;
                    s64[2 * q + 1] += (double)S32[q].y;
                    S32[q] = make_float2(0.f, 0.f);
                }
            }
        }
        ring.release(k);
#pragma unroll
        for (int q = 0; q < RQ; ++q) {                 // (a partial last tile's tail promotion)
            s64[2 * q] += (double)S32[q].x;
            s64[2 * q + 1] += (double)S32[q].y;
            S32[q] = make_float2(0.f, 0.f);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= p.M) continue;
        const double stot = s64[r];
        if (p.split > 1) {
            p.state[((int64_t)sp * p.M + i) * 2 + 0] = Mr[r];
            p.state[((int64_t)sp * p.M + i) * 2 + 1] = stot;
            continue;
        }
        const double a = (stot > 0.0) ? 0.69314718055994530942 * (Mr[r] + log2(stot)) : -INFINITY;
        if (p.out) {
            if (p.out_f64) ((double *)p.out)[i] = a;
            else ((float *)p.out)[i] = (float)a;
        }
        if (p.state) {
            p.state[2 * i + 0] = Mr[r];
            p.state[2 * i + 1] = stot;
        }
    }
}

// Small-M mode (north star (a), the warp-shuffle finish; see sum_smm.cu): a CTA owns R rows, its
// 256 threads take the tile's record pairs t, t + 256, ..., each keeping its own streaming
// (m, s) per row with the same lazy rescale (one pair per check), and the CTA merges the 256
// states per row with max / rescaled-sum butterflies and a fixed-order sum over warps.
template <int D, int R, bool HZ>
__global__ void __launch_bounds__(kThreads, 2) lse_smm_kernel(const LseParams p) {
    using Cfg = LseCfg<D, HZ>;
    constexpr int RS = Cfg::RS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int64_t ngroups = (p.M + R - 1) / R;
    const int sp = (int)(blockIdx.x / ngroups);                    // split-major (L2 sharing)
    const int64_t row0 = (int64_t)(blockIdx.x % ngroups) * R;
    const int64_t q0 = (int64_t)sp * p.pairs_per_split;
    const int64_t npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);
    const int nt = (int)((npc + Cfg::PAIRS - 1) / Cfg::PAIRS);
    const int last_np = (int)(npc - (int64_t)(nt > 0 ? nt - 1 : 0) * Cfg::PAIRS);
    JRing<kStages> ring;
    ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * RS, nt, kConsumerWarps, (uint32_t)last_np * RS * 4u);

    const int ct = threadIdx.x;
    const float negc = p.negc;
    const float2 negc2 = dup2(negc);
    float xr[R][D];
    float m[R];
    double s64[R];
    float2 s32[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r;
        const bool ok = i < p.M;
#pragma unroll
        for (int d = 0; d < D; ++d) xr[r][d] = ok ? __ldg(p.x + i * D + d) : 0.0f;
        m[r] = kLseSentinel;
        s64[r] = 0.0;
        s32[r] = make_float2(0.f, 0.f);
    }
    for (int k = 0; k < nt; ++k) {
        const float *tile = ring.acquire(k);
        const int np = k == nt - 1 ? last_np : Cfg::PAIRS;
        for (int pp = ct; pp < np; pp += kThreads) {
            const float *rec = tile + pp * RS;
            float f[RS];
#pragma unroll
            for (int u = 0; u < RS / 4; ++u) {
                const float4 v = lds128(rec + 4 * u);
                f[4 * u + 0] = v.x; f[4 * u + 1] = v.y; f[4 * u + 2] = v.z; f[4 * u + 3] = v.w;
            }
            float2 ny[D];
#pragma unroll
            for (int d = 0; d < D; ++d) ny[d] = make_float2(f[2 * d], f[2 * d + 1]);
            float2 hhi = make_float2(0.f, 0.f), hc = make_float2(1.f, 1.f);
            if constexpr (!HZ) {
                hhi = make_float2(f[2 * D], f[2 * D + 1]);
                hc = make_float2(f[2 * D + 2], f[2 * D + 3]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 dd = add2(dup2(xr[r][0]), ny[0]);
                float2 q2 = mul2(dd, dd);
#pragma unroll
                for (int d = 1; d < D; ++d) {
                    dd = add2(dup2(xr[r][d]), ny[d]);
                    q2 = fma2(dd, dd, q2);
                }
                const float2 hm = HZ ? dup2(-m[r]) : add2(hhi, dup2(-m[r]));
                const float2 t = fma2(q2, negc2, hm);
                const float2 e = make_float2(ex2(t.x), ex2(t.y));
                const float2 cs = HZ ? e : mul2(e, hc);
                if (!(fmaxf(cs.x, cs.y) <= kSumMax)) {
                    const LseRescale rs = lse_rescale<D, HZ, RS, 1>(rec, xr[r], negc, m[r], s64[r], s32[r]);
                    m[r] = rs.m;
                    s64[r] = rs.s64;
                    s32[r] = make_float2(rs.c1, 0.f);
                } else {
                    s32[r] = add2(s32[r], cs);
                }
            }
        }
        ring.release(k);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            s64[r] += (double)s32[r].x + (double)s32[r].y;
            s32[r] = make_float2(0.f, 0.f);
        }
    }
    // CTA merge of the per-thread (m, s) states of each row (deterministic butterflies)
    __shared__ double red[kConsumerWarps][R];
    __shared__ double mrow[R];
    const int lane = ct & 31, warp = ct >> 5;
    double mt[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        mt[r] = s64[r] > 0.0 ? (double)m[r] : -INFINITY;
        double v = mt[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[warp][r] = v;
    }
    __syncthreads();
    if (ct < R) {
        double v = red[0][ct];
        for (int w = 1; w < kConsumerWarps; ++w) v = fmax(v, red[w][ct]);
        mrow[ct] = v;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double c = (s64[r] > 0.0 && mrow[r] > -INFINITY) ? s64[r] * exp2(mt[r] - mrow[r]) : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) red[warp][r] = c;
    }
    __syncthreads();
    if (ct >= R) return;
    const int64_t i = row0 + ct;
    if (i >= p.M) return;
    double stot = red[0][ct];
    for (int w = 1; w < kConsumerWarps; ++w) stot += red[w][ct];
    const double mm = stot > 0.0 ? mrow[ct] : (double)kLseSentinel;
    if (p.split > 1) {
        p.state[((int64_t)sp * p.M + i) * 2 + 0] = mm;
        p.state[((int64_t)sp * p.M + i) * 2 + 1] = stot;
        return;
    }
    const double a = (stot > 0.0) ? 0.69314718055994530942 * (mm + log2(stot)) : -INFINITY;
    if (p.out) {
        if (p.out_f64) ((double *)p.out)[i] = a;
        else ((float *)p.out)[i] = (float)a;
    }
    if (p.state) {
        p.state[2 * i + 0] = mm;
        p.state[2 * i + 1] = stot;
    }
}

template <int D, bool HZ>
static cudaError_t run_lse_smm(const LseLaunch &a, cudaStream_t st, int *ctas) {
    using Cfg = LseCfg<D, HZ>;
    constexpr int R = D <= 4 ? 8 : 4;
    auto kern = lse_smm_kernel<D, R, HZ>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    LseParams p;
    p.x = a.x; p.J = a.J; p.M = a.M; p.split = a.split; p.pairs_per_split = a.pairs_per_split;
    p.npv = a.npv; p.negc = a.negc; p.out = a.out; p.out_f64 = a.out_f64; p.state = a.state;
    p.units = nullptr;
    const int64_t grid = (a.M + R - 1) / R * a.split;
    *ctas = (int)grid;
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
}

int lse_smm_rows(int D) { return D <= 4 ? 8 : 4; }

cudaError_t launch_lse_smm(const LseLaunch &a, cudaStream_t st, int *ctas) {
#define GENRED_SMM(DD) if (a.D == DD) return a.h_zero ? run_lse_smm<DD, true>(a, st, ctas) : run_lse_smm<DD, false>(a, st, ctas);
    GENRED_SMM(1) GENRED_SMM(2) GENRED_SMM(3) GENRED_SMM(4)
    GENRED_SMM(5) GENRED_SMM(6) GENRED_SMM(7) GENRED_SMM(8)
#undef GENRED_SMM
    return cudaErrorInvalidValue;
}

template <int D, int R, bool HZ>
static cudaError_t run_lse(const LseLaunch &a, cudaStream_t st, int *ctas) {
    using Cfg = LseCfg<D, HZ>;
    auto kern = lse_kernel<D, R, HZ>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    LseParams p;
    p.x = a.x; p.J = a.J; p.M = a.M; p.split = a.split; p.pairs_per_split = a.pairs_per_split;
    p.npv = a.npv; p.negc = a.negc; p.out = a.out; p.out_f64 = a.out_f64; p.state = a.state;
    p.units = a.units;
    const int64_t rows = (int64_t)kConsumerWarps * 32 * R;
    const int64_t grid = a.units ? a.n_units : ((a.M + rows - 1) / rows) * a.split;
    *ctas = (int)grid;
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
}

template <int D, bool HZ>
static cudaError_t run_lse_local(const LseLaunch &a, cudaStream_t st, int *ctas) {
    using Cfg = LseLocCfg<D, HZ>;
    auto kern = lse_local_kernel<D, HZ>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    LseParams p;
    p.x = a.x; p.J = a.J; p.M = a.M; p.split = a.split; p.pairs_per_split = a.pairs_per_split;
    p.npv = a.npv; p.negc = a.negc; p.out = a.out; p.out_f64 = a.out_f64; p.state = a.state;
    p.units = nullptr; p.centers = a.centers; p.s = a.s;
    const int64_t rows = (int64_t)kConsumerWarps * 32 * 4;
    const int64_t grid = ((a.M + rows - 1) / rows) * a.split;
    *ctas = (int)grid;
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
}

template <int D, int R>
static int occ_lse(bool hz) {
    using Cfg = LseCfg<D, false>;
    auto kern = hz ? lse_kernel<D, R, true> : lse_kernel<D, R, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, hz ? LseCfg<D, true>::SMEM : Cfg::SMEM) != cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

// Rows per thread (D <= 3: 4 rows at 80 registers, 3 CTAs/SM; else 2 at 2 CTAs/SM).
template <int D>
#ifndef GENRED_LSE_R4
#define GENRED_LSE_R4 1
#endif
#ifndef GENRED_LSE_RBIG
#define GENRED_LSE_RBIG 4
#endif
constexpr int lse_rmax() { return (D <= 3 && GENRED_LSE_R4) ? GENRED_LSE_RBIG : 2; }

int lse_rows_per_thread_max(int D) { return (D <= 3 && GENRED_LSE_R4) ? GENRED_LSE_RBIG : 2; }

template <int D>
static cudaError_t run_lse_r(const LseLaunch &a, cudaStream_t st, int *ctas) {
    constexpr int RM = lse_rmax<D>();
    if (a.R == 1) return a.h_zero ? run_lse<D, 1, true>(a, st, ctas) : run_lse<D, 1, false>(a, st, ctas);
    return a.h_zero ? run_lse<D, RM, true>(a, st, ctas) : run_lse<D, RM, false>(a, st, ctas);
}

cudaError_t launch_lse(const LseLaunch &a, cudaStream_t st, int *ctas) {
    if (a.centers) {                                   // tile-centred form (R = 4, D <= 3)
        if (a.R != 4) return cudaErrorInvalidValue;
        switch (a.D) {
            case 1: return a.h_zero ? run_lse_local<1, true>(a, st, ctas) : run_lse_local<1, false>(a, st, ctas);
            case 2: return a.h_zero ? run_lse_local<2, true>(a, st, ctas) : run_lse_local<2, false>(a, st, ctas);
            case 3: return a.h_zero ? run_lse_local<3, true>(a, st, ctas) : run_lse_local<3, false>(a, st, ctas);
        }
        return cudaErrorInvalidValue;
    }
    switch (a.D) {
        case 1: return run_lse_r<1>(a, st, ctas);
        case 2: return run_lse_r<2>(a, st, ctas);
        case 3: return run_lse_r<3>(a, st, ctas);
        case 4: return run_lse_r<4>(a, st, ctas);
        case 5: return run_lse_r<5>(a, st, ctas);
        case 6: return run_lse_r<6>(a, st, ctas);
        case 7: return run_lse_r<7>(a, st, ctas);
        case 8: return run_lse_r<8>(a, st, ctas);
    }
    return cudaErrorInvalidValue;
}

int lse_occupancy(int D, int R, bool hz) {
#define GENRED_OCC(DD) if (D == DD) return R == 1 ? occ_lse<DD, 1>(hz) : occ_lse<DD, lse_rmax<DD>()>(hz);
    GENRED_OCC(1) GENRED_OCC(2) GENRED_OCC(3) GENRED_OCC(4)
    GENRED_OCC(5) GENRED_OCC(6) GENRED_OCC(7) GENRED_OCC(8)
#undef GENRED_OCC
    return 1;
}

}  // namespace genred
