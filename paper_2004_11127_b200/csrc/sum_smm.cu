// sum_smm.cu -- small-M mode of the Genred Sum kernels (north star (a): "a warp-shuffle finish
// runs when several threads share one i"; SURVEY.md 8(e) j-shard regime M << N).
//
// With few rows the row-tile grid (one thread per row) cannot fill 148 SMs however the j-axis is
// split, and each CTA would run with most threads idle.  Here every CTA owns R rows only (R = 8
// for the Sum, 2 for the gradient modes); its 256 threads split each j-tile's record pairs, and
// the CTA reduces its fp64 partials with warp shuffles and a fixed-order sum over warps
// (sum_body.cuh, SMM = true).  j-splits (record-pair grains) then spread the work over the GPU;
// their partials merge in sum_finalize like the row-tile kernels'.  Instantiated for E = 1 and
// D <= 4 (the other shapes take the row-tile kernels).
#include <stdlib.h>

#include <algorithm>

#include "sum_body.cuh"

namespace genred {

template <int MODE>
constexpr int smm_rows() { return (MODE == 0 || MODE == 3) ? 8 : 2; }

template <int MODE, int D>
static int occ_smm() {
    constexpr int R = smm_rows<MODE>();
    using Cfg = SumCfg<MODE, D, 1>;
    auto kern = sum_kernel<MODE, D, 1, R, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, Cfg::SMEM) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

template <int MODE, int D>
static cudaError_t run_smm(const SumLaunch &a, cudaStream_t st, int *ctas) {
    constexpr int R = smm_rows<MODE>();
    using Cfg = SumCfg<MODE, D, 1>;
    auto kern = sum_kernel<MODE, D, 1, R, true>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    SumParams p;
    p.x = a.x; p.J = a.J; p.g = a.g; p.M = a.M; p.split = a.split;
    p.pairs_per_split = a.pairs_per_split; p.npv = a.npv; p.s = a.s;
    p.scale_sum = a.scale_sum; p.scale_grad = a.scale_grad; p.out = a.out; p.out_f64 = a.out_f64;
    p.out_grad = a.out_grad; p.part = a.part; p.geo = a.geo; p.units = nullptr;
    p.tile_done = nullptr;
    p.n_work = (a.M + R - 1) / R * a.split;
    if (p.n_work == 0) { *ctas = 0; return cudaSuccess; }
    static const int occ = occ_smm<MODE, D>();                 // GENRED_PERSIST=1: persistent grid
    static const int persist = getenv("GENRED_PERSIST") ? atoi(getenv("GENRED_PERSIST")) : 0;
    const int64_t grid = persist ? std::min<int64_t>(p.n_work, (int64_t)a.num_sms * occ) : p.n_work;
    *ctas = (int)grid;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
}


template <int MODE>
static cudaError_t run_smm_d(const SumLaunch &a, cudaStream_t st, int *ctas) {
    switch (a.D) {
        case 1: return run_smm<MODE, 1>(a, st, ctas);
        case 2: return run_smm<MODE, 2>(a, st, ctas);
        case 3: return run_smm<MODE, 3>(a, st, ctas);
        case 4: return run_smm<MODE, 4>(a, st, ctas);
    }
    return cudaErrorInvalidValue;
}
template <int MODE>
static int occ_smm_d(int D) {
    switch (D) {
        case 1: return occ_smm<MODE, 1>();
        case 2: return occ_smm<MODE, 2>();
        case 3: return occ_smm<MODE, 3>();
        case 4: return occ_smm<MODE, 4>();
    }
    return 1;
}

bool sum_smm_supported(int mode, int D, int E) { return mode >= 0 && mode <= 3 && E == 1 && D >= 1 && D <= 4; }

int sum_smm_rows(int mode) { return (mode == 0 || mode == 3) ? smm_rows<0>() : smm_rows<1>(); }

int sum_smm_occupancy(int mode, int D) {
    switch (mode) {
        case 0: return occ_smm_d<0>(D);
        case 1: return occ_smm_d<1>(D);
        case 2: return occ_smm_d<2>(D);
        case 3: return occ_smm_d<3>(D);
    }
    return 1;
}

cudaError_t launch_sum_smm(const SumLaunch &a, cudaStream_t st, int *ctas) {
    if (!sum_smm_supported(a.mode, a.D, a.E)) return cudaErrorInvalidValue;
    switch (a.mode) {
        case 0: return run_smm_d<0>(a, st, ctas);
        case 1: return run_smm_d<1>(a, st, ctas);
        case 2: return run_smm_d<2>(a, st, ctas);
        case 3: return run_smm_d<3>(a, st, ctas);
    }
    return cudaErrorInvalidValue;
}

}  // namespace genred
