// softmax_grad_kernel.cu -- the backward of the log-sum-exp reduction (
// PAPER.md:140-147 "backprop through KeOps calls"; the gradient of a reduction is
// another reduction):
//
//     p_ij = exp(-|x_i - y_j|^2 / eps + alpha_i + beta_j)
//     S_i  = sum_j sig_j p_ij ,   G_i = coef_i (-2/eps) sum_j sig_j p_ij (x_i - y_j)
//
// With alpha = -a (the forward LSE), beta = h, sig = coef-free 1: S_i = 1 and G_i = da_i/dx_i.
// With the roles swapped (rows y, reduced axis x, alpha = h, beta = -a, sig = g):
// S_j = dL/dh_j and G_j = dL/dy_j.  The exponent never exceeds ~0 (alpha + beta is a max shift)
// so there is no rescaling; raw differences as in the forward (R6), log2(e) folded into the
// shifts, which are carried as fp32 hi + lo pairs (R6c).  Pipeline and tiling: sum_kernel.cu.
#include <math.h>

#include "device.cuh"
#include "internal.h"

// 3 CTAs/SM (80 registers): 8.06 -> 8.18 pairs/clk/SM at 4e5^2 (4: spills, 5.48; round 2)
#ifndef GENRED_SM_MINB
#define GENRED_SM_MINB 3
#endif
#ifndef GENRED_SM_UNROLL
#define GENRED_SM_UNROLL 2
#endif

namespace genred {

constexpr int kSmUnroll = GENRED_SM_UNROLL;      // record pairs unrolled per pair-loop iteration

template <int D>
struct SmCfg {
    // record pair: 2D coordinates (-y), beta' hi pair, beta' lo pair, sig pair
    static constexpr int RS = ((2 * D + 6) + 3) / 4 * 4;
    static constexpr int PAIRS = kTileJ / 2;
    static constexpr int TILE_FLOATS = PAIRS * RS;
    static constexpr int SMEM = JRing<kStages>::smem_bytes(TILE_FLOATS);
};

struct SmParams {
    const float *x, *J, *coef;
    const double *alpha;
    int64_t M;
    int split;
    int64_t pairs_per_split, npv;      // record-pair j-splits (see SumParams)
    float negc;               // -log2(e)/eps
    double scale_grad;        // -2/eps
    void *out;
    int out_f64;
    float *out_grad;
    double *part;             // split > 1: split x M x (1 + D)
};

template <int D, int R>
__global__ void __launch_bounds__(kThreads, GENRED_SM_MINB) softmax_grad_kernel(const SmParams p) {
    using Cfg = SmCfg<D>;
    constexpr int RS = Cfg::RS, C = 1 + D;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int64_t itile = blockIdx.x / p.split;
    const int sp = (int)(blockIdx.x % p.split);
    const int64_t q0 = (int64_t)sp * p.pairs_per_split;                 // record pairs [q0, q0 + npc)
    const int64_t npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);
    const int nt = (int)((npc + Cfg::PAIRS - 1) / Cfg::PAIRS);
    const int last_np = (int)(npc - (int64_t)(nt > 0 ? nt - 1 : 0) * Cfg::PAIRS);
    JRing<kStages> ring;
    ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * RS, nt, kConsumerWarps, (uint32_t)last_np * RS * 4u);

    const int ct = threadIdx.x;
    const int64_t row0 = itile * (int64_t)(kConsumerWarps * 32 * R);
    const float2 negc2 = dup2(p.negc);
    float xr[R][D];
    float ahi[R], alo[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        const bool ok = i < p.M;
#pragma unroll
        for (int d = 0; d < D; ++d) xr[r][d] = ok ? __ldg(p.x + i * D + d) : 0.0f;
        const double a2 = (ok && p.alpha) ? 1.4426950408889634074 * p.alpha[i] : 0.0;
        ahi[r] = (float)a2;
        alo[r] = (float)(a2 - (double)ahi[r]);
    }
    float2 s0[R], sg[R][D];
    double s064[R], sg64[R][D];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        s0[r] = make_float2(0.f, 0.f);
        s064[r] = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) { sg[r][d] = make_float2(0.f, 0.f); sg64[r][d] = 0.0; }
    }

    for (int k = 0; k < nt; ++k) {
        const float *tile = ring.acquire(k);
        const int np = k == nt - 1 ? last_np : Cfg::PAIRS;
#pragma unroll kSmUnroll
        for (int pp = 0; pp < np; ++pp) {
            float f[RS];
#pragma unroll
            for (int q = 0; q < RS / 4; ++q) {
                const float4 v = lds128(tile + pp * RS + 4 * q);
                f[4 * q + 0] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
            }
            float2 ny[D];
#pragma unroll
            for (int d = 0; d < D; ++d) ny[d] = make_float2(f[2 * d], f[2 * d + 1]);
            const float2 bhi = make_float2(f[2 * D], f[2 * D + 1]);
            const float2 sig = make_float2(f[2 * D + 4], f[2 * D + 5]);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 dd[D];
#pragma unroll
                for (int d = 0; d < D; ++d) dd[d] = add2(dup2(xr[r][d]), ny[d]);   // x - y
                float2 q = mul2(dd[0], dd[0]);
#pragma unroll
                for (int d = 1; d < D; ++d) q = fma2(dd[d], dd[d], q);
                // alpha' + beta': only the hi parts enter the exponent (their sum is exact when
                // they nearly cancel); 2^beta_lo is folded into sig by the pack, 2^alpha_lo is
                // applied to the row's fp64 sums at the end
                const float2 z = add2(bhi, dup2(ahi[r]));
                const float2 t = fma2(q, negc2, z);
                const float2 w = mul2(make_float2(ex2(t.x), ex2(t.y)), sig);
                s0[r] = add2(s0[r], w);
#pragma unroll
                for (int d = 0; d < D; ++d) sg[r][d] = fma2(w, dd[d], sg[r][d]);
            }
        }
        ring.release(k);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            s064[r] += (double)s0[r].x + (double)s0[r].y;
            s0[r] = make_float2(0.f, 0.f);
#pragma unroll
            for (int d = 0; d < D; ++d) {
                sg64[r][d] += (double)sg[r][d].x + (double)sg[r][d].y;
                sg[r][d] = make_float2(0.f, 0.f);
            }
        }
    }

#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= p.M) continue;
        const double flo = exp2((double)alo[r]);                 // the 2^alpha_lo factor
        s064[r] *= flo;
#pragma unroll
        for (int d = 0; d < D; ++d) sg64[r][d] *= flo;
        if (p.split > 1) {
            double *dst = p.part + ((int64_t)sp * p.M + i) * C;
            dst[0] = s064[r];
#pragma unroll
            for (int d = 0; d < D; ++d) dst[1 + d] = sg64[r][d];
            continue;
        }
        if (p.out_f64) ((double *)p.out)[i] = s064[r];
        else ((float *)p.out)[i] = (float)s064[r];
        const double gs = p.scale_grad * (p.coef ? (double)__ldg(p.coef + i) : 1.0);
#pragma unroll
        for (int d = 0; d < D; ++d) p.out_grad[i * D + d] = (float)(gs * sg64[r][d]);
    }
}

template <int D, int R>
static cudaError_t run_sm(const SmLaunch &a, cudaStream_t st, int *ctas) {
    using Cfg = SmCfg<D>;
    auto kern = softmax_grad_kernel<D, R>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    SmParams p;
    p.x = a.x; p.J = a.J; p.coef = a.coef; p.alpha = a.alpha; p.M = a.M; p.split = a.split;
    p.pairs_per_split = a.pairs_per_split; p.npv = a.npv; p.negc = a.negc;
    p.scale_grad = a.scale_grad; p.out = a.out; p.out_f64 = a.out_f64; p.out_grad = a.out_grad;
    p.part = a.part;
    const int64_t rows = (int64_t)kConsumerWarps * 32 * R;
    const int64_t grid = ((a.M + rows - 1) / rows) * a.split;
    *ctas = (int)grid;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
}

template <int D, int R>
static int occ_sm() {
    using Cfg = SmCfg<D>;
    auto kern = softmax_grad_kernel<D, R>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, Cfg::SMEM) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

// rows per thread: 2 for D <= 4 (registers: D + 2 shifts + 2 + 2D accumulators + 1 + D fp64), else 1
#ifndef GENRED_SM_R
#define GENRED_SM_R 4
#endif
int sm_rows_per_thread_max(int D) { return D <= 4 ? GENRED_SM_R : 1; }

#define GENRED_SM_D(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)

cudaError_t launch_softmax_grad(const SmLaunch &a, cudaStream_t st, int *ctas) {
#define GENRED_CASE(DD) \
    if (a.D == DD) return (a.R == 1 || DD > 4) ? run_sm<DD, 1>(a, st, ctas) : run_sm<DD, (DD <= 4 ? GENRED_SM_R : 1)>(a, st, ctas);
    GENRED_SM_D(GENRED_CASE)
#undef GENRED_CASE
    return cudaErrorInvalidValue;
}

int softmax_grad_occupancy(int D, int R) {
#define GENRED_CASE(DD) \
    if (D == DD) return (R == 1 || DD > 4) ? occ_sm<DD, 1>() : occ_sm<DD, (DD <= 4 ? GENRED_SM_R : 1)>();
    GENRED_SM_D(GENRED_CASE)
#undef GENRED_CASE
    return 1;
}

}  // namespace genred

namespace genred {

// records for softmax_grad_kernel: (-y_d pairs, beta' = log2(e) beta as fp32 hi / lo pairs, sig
// pairs); padding records contribute exactly 0 (y = 0, beta' = -inf, sig = 0)
__global__ void pack_softmax_kernel(const float *__restrict__ y, const float *__restrict__ sig,
                                    const double *__restrict__ beta, int64_t N, int D,
                                    int64_t npairs, int RS, float *__restrict__ J) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
         p += (int64_t)gridDim.x * blockDim.x) {
        float *rec = J + p * RS;
        for (int h = 0; h < 2; ++h) {
            const int64_t j = 2 * p + h;
            const bool valid = j < N;
            for (int d = 0; d < D; ++d) rec[2 * d + h] = valid ? -y[j * D + d] : 0.0f;
            const double b2 = (valid && beta) ? 1.4426950408889634074 * beta[j] : 0.0;
            const float hi = valid ? (float)b2 : -INFINITY;
            rec[2 * D + h] = hi;
            rec[2 * D + 2 + h] = 0.0f;                            // (beta_lo: folded into sig)
            // sig' = sig 2^(beta'_lo) in fp64, rounded once: the kernel's exponent uses beta'_hi
            const double lo = valid ? b2 - (double)hi : 0.0;
            rec[2 * D + 4 + h] = valid ? (float)((sig ? (double)sig[j] : 1.0) * exp2(lo)) : 0.0f;
        }
        for (int k = 2 * D + 6; k < RS; ++k) rec[k] = 0.0f;
    }
}

int softmax_record_stride(int D) { return ((2 * D + 6) + 3) / 4 * 4; }

cudaError_t launch_pack_softmax(const float *y, const float *sig, const double *beta, int64_t N,
                                int D, int64_t npairs, float *J, cudaStream_t st) {
    int64_t blocks = (npairs + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    pack_softmax_kernel<<<(unsigned)blocks, 256, 0, st>>>(y, sig, beta, N, D, npairs,
                                                          softmax_record_stride(D), J);
    return cudaGetLastError();
}

}  // namespace genred
