// sum_kernel.cu -- Genred Sum reductions on the FP32 + MUFU pipes:
//
//   GAUSS       a_i   = sum_j exp(-|x_i - y_j|^2 / sigma^2) b_j           (Eq. 1)
//   GAUSS_GRADX G_i   = sum_j (-2/sigma^2)(x_i - y_j) e_ij <b_j, g_i>
//   SUM_GRADX   both in one pass (shares the distance and the exponential)
//   SQDIST_SUM  a_i   = sum_j |x_i - y_j|^2 b_j                           (test combination)
//
// Design (B200-first; the paper's GPU Gems "tiled map-reduce", is prior art):
//   * one CTA owns 256*R i-rows, kept in registers (R rows per math thread), and one j-range of
//     record pairs (a j-split);
//   * j-tiles (512 records, pair-interleaved, pre-scaled by s = sqrt(log2 e)/sigma so that
//     exp(-|x-y|^2/sigma^2) = 2^(-|x'-y'|^2)) stream from HBM/L2 into a 4-stage shared-memory
//     ring with cp.async.bulk (TMA engine) completing on mbarriers; the last warp to release a
//     stage refills it (all 8 warps are math warps, device.cuh JRing);
//   * math warps read each record pair once per thread (broadcast LDS.128) and evaluate two j's
//     at a time with packed FADD2/FMUL2/FFMA2 and two MUFU.EX2 (ex2.approx.ftz): in the expanded
//     form a pair costs 4 FP32 lane-ops + 1 MUFU for D=3 (the MUFU pipe, 16/clk/SM, is the bound);
//   * per-tile fp32 partials are promoted to fp64 every 512 j (reading R18 in DESIGN.md);
//   * record-pair j-splits (grid = i-tiles x splits) fill all 148 SMs; their fp64 partials are
//     merged in a fixed order by sum_finalize (deterministic, no float atomics);
//   * the pair loop itself lives in sum_body.cuh, shared with the small-M kernels (sum_smm.cu).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "sum_body.cuh"

namespace genred {

// ---- host-side dispatch over (MODE, D, E, R) ------------------------------------------------
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

template <int MODE, int D, int E, int R>
static cudaError_t run_sum(const SumLaunch &a, cudaStream_t st, int *ctas) {
    using Cfg = SumCfg<MODE, D, E>;
    auto kern = sum_kernel<MODE, D, E, R>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    SumParams p;
    p.x = a.x; p.J = a.J; p.g = a.g; p.M = a.M; p.split = a.split;
    p.pairs_per_split = a.pairs_per_split; p.npv = a.npv; p.s = a.s;
    p.scale_sum = a.scale_sum; p.scale_grad = a.scale_grad; p.out = a.out; p.out_f64 = a.out_f64;
    p.out_grad = a.out_grad; p.part = a.part; p.geo = a.geo; p.units = a.units;
    p.centers = a.centers;
    p.split_major = a.split_major;
    p.itiles = (a.M + (int64_t)kConsumerWarps * 32 * R - 1) / ((int64_t)kConsumerWarps * 32 * R);
    p.tile_done = a.split > 1 ? a.tile_done : nullptr;
    const int64_t rows = (int64_t)kConsumerWarps * 32 * R;
    const int64_t itiles = (a.M + rows - 1) / rows;
    p.n_work = a.units ? a.n_units : itiles * a.split;
    if (p.n_work == 0) { *ctas = 0; return cudaSuccess; }
    // One CTA per work unit by default.  The kernel also runs persistent (GENRED_PERSIST=1: 148 x
    // occupancy CTAs walking the units), but that measured 11% slower at M = N = 2e6 (3.92e12
    // against 4.37e12 pairs/s, same SASS in the pair loop): the hardware's dynamic CTA launch
    // staggers the units across the SM's resident CTAs, the fixed assignment runs them in lock step.
    static const int occ = occ_sum<MODE, D, E, R>();
    static const int persist = getenv("GENRED_PERSIST") ? atoi(getenv("GENRED_PERSIST")) : 0;
    const int64_t grid = persist ? std::min<int64_t>(p.n_work, (int64_t)a.num_sms * occ) : p.n_work;
    *ctas = (int)grid;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
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

template <int MODE, int D, int R>
static cudaError_t run_sum_small(const SumLaunch &a, const float *y, const float *b, int64_t N,
                                 cudaStream_t st, int *ctas) {
    using Cfg = SumCfg<MODE, D, 1>;
    SumParams p;
    p.x = a.x; p.J = nullptr; p.g = a.g; p.M = a.M; p.split = a.split;
    p.pairs_per_split = a.pairs_per_split; p.npv = a.npv; p.s = a.s;
    p.scale_sum = a.scale_sum; p.scale_grad = a.scale_grad; p.out = a.out; p.out_f64 = a.out_f64;
    p.out_grad = a.out_grad; p.part = a.part; p.geo = nullptr; p.units = nullptr;
    p.tile_done = a.split > 1 ? a.tile_done : nullptr;
    const int64_t rows = (int64_t)kConsumerWarps * 32 * R;
    const int64_t itiles = (a.M + rows - 1) / rows;
    p.n_work = itiles * a.split;
    *ctas = (int)p.n_work;
    if (p.n_work == 0) return cudaSuccess;
    // cluster merge through distributed shared memory for split <= 8 (portable cluster size)
    const int cl = (a.split > 1 && a.split <= 8 && kSmallCluster) ? 1 : 0;
    const int smem = (int)(a.pairs_per_split * Cfg::RS * 4) + (cl ? kThreads * R * Cfg::C * 8 : 0);
    auto kern = sum_small_kernel<MODE, D, 1, R>;
    // the size varies per call: opt in once to the largest this instance can ask for
    // (smem_opt_in caches per kernel, so a smaller first request would stick)
    constexpr int kSmemMax = (int)(kSmallMaxPairs * Cfg::RS * 4) + kThreads * R * Cfg::C * 8;
    if (kSmemMax > 48 * 1024) {
        const cudaError_t e = smem_opt_in((const void *)kern, kSmemMax);
        if (e != cudaSuccess) return e;
    }
    if (!cl) {
        kern<<<(unsigned)p.n_work, kThreads, smem, st>>>(p, y, b, N, 0);
        return cudaGetLastError();
    }
    p.tile_done = nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.n_work);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)a.split;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, y, b, N, 1);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <int MODE, int D>
static cudaError_t run_sum_small_r(const SumLaunch &a, const float *y, const float *b, int64_t N,
                                   cudaStream_t st, int *ctas) {
    constexpr int RM = sum_rmax<MODE, D, 1>();
    return a.R == 1 ? run_sum_small<MODE, D, 1>(a, y, b, N, st, ctas) : run_sum_small<MODE, D, RM>(a, y, b, N, st, ctas);
}

template <int MODE>
static cudaError_t run_sum_small_d(const SumLaunch &a, const float *y, const float *b, int64_t N,
                                   cudaStream_t st, int *ctas) {
    switch (a.D) {
        case 1: return run_sum_small_r<MODE, 1>(a, y, b, N, st, ctas);
        case 2: return run_sum_small_r<MODE, 2>(a, y, b, N, st, ctas);
        case 3: return run_sum_small_r<MODE, 3>(a, y, b, N, st, ctas);
        case 4: return run_sum_small_r<MODE, 4>(a, y, b, N, st, ctas);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_sum_small(const SumLaunch &a, const float *y, const float *b, int64_t N,
                             cudaStream_t st, int *ctas) {
    if (a.E != 1 || a.pairs_per_split > kSmallMaxPairs) return cudaErrorInvalidValue;
    switch (a.mode) {
        case 0: return run_sum_small_d<0>(a, y, b, N, st, ctas);
        case 1: return run_sum_small_d<1>(a, y, b, N, st, ctas);
        case 2: return run_sum_small_d<2>(a, y, b, N, st, ctas);
        case 3: return run_sum_small_d<3>(a, y, b, N, st, ctas);
    }
    return cudaErrorInvalidValue;
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
