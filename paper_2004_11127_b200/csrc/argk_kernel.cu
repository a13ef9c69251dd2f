// argk_kernel.cu -- ArgKMin over squared distances on the FP32 pipe, small D (
// k-nearest neighbours):
//
//     a_i = the K smallest (|x_i - y_j|^2, j) in lexicographic order (ties -> lowest j, R7)
//
// Same pipeline as sum_kernel.cu (bulk-copy ring of 512-record j-tiles, rows in registers).
// Per j-pair: packed FADD2/FMUL2/FFMA2 distance, one FMNMX + FSETP against the current K-th
// best; a hit (about K ln(N/K) times per row) runs an unrolled compare-swap insertion into the
// register-resident sorted list.  Within one thread j arrives in ascending order, so strict '<'
// realises the (d, j) order; split-j lists are merged lexicographically by topk_merge.
#include <math.h>

#include "device.cuh"
#include "internal.h"

#ifndef GENRED_ARGK_R
#define GENRED_ARGK_R 2
#endif
// record pairs unrolled per iteration: 4 measured 12.88 / 12.52 pairs/clk/SM (K = 1 / 10, M = 1e5,
// N = 1e7) against 12.72 / 11.82 for 2; 4 rows per thread for K <= 4 measured slower (11.93)
#ifndef GENRED_ARGK_UNROLL
#define GENRED_ARGK_UNROLL 4
#endif

namespace genred {

constexpr int kArgkUnroll = GENRED_ARGK_UNROLL;   // record pairs unrolled per pair-loop iteration

template <int D>
struct ArgkCfg {
    // record pair: (-y_d) pairs, then the pair's two j (int32 bits; -1 = padding), so that the
    // same kernel serves range-packed J (block-sparse ranges), whose positions are not j
    static constexpr int RS = ((2 * (D + 1)) + 3) / 4 * 4;
    static constexpr int PAIRS = kTileJ / 2;
    static constexpr int TILE_FLOATS = PAIRS * RS;
    static constexpr int STAGE_BYTES = TILE_FLOATS * 4;
    static constexpr int SMEM = JRing<kStages>::smem_bytes(TILE_FLOATS);
};

// small-M mode: the per-thread K-lists live after the j-ring in dynamic shared memory
template <int D>
constexpr int argk_smm_list_offset() { return (ArgkCfg<D>::SMEM + 15) / 16 * 16; }
template <int D, int KMAX>
constexpr int argk_smm_smem() { return argk_smm_list_offset<D>() + 2 * kThreads * KMAX * 4; }

struct ArgkParams {
    const float *x, *J;
    int64_t M;
    int K;
    int split;
    int64_t pairs_per_split, npv;      // record-pair j-splits (see SumParams)
    float *dist;
    int64_t *idx;
    int64_t j_offset;
    float *pdist;
    int32_t *pidx;
    const RangeUnit *units;            // block-sparse ranges: one CTA per unit, direct output
};

template <int KMAX>
__device__ __forceinline__ void topk_insert(float (&dist)[KMAX], int32_t (&idx)[KMAX], int K,
                                            float cd, int32_t cj, float &kth) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        if (k < K) {
            // (d, j) lexicographic: a displaced entry keeps precedence over later equal d's
            const bool sw = cd < dist[k] || (cd == dist[k] && (uint32_t)cj < (uint32_t)idx[k]);
            const float td = dist[k];
            const int32_t tj = idx[k];
            dist[k] = sw ? cd : td;
            idx[k] = sw ? cj : tj;
            cd = sw ? td : cd;
            cj = sw ? tj : cj;
        }
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
        if (k == K - 1) kth = dist[k];
}

template <int D, int KMAX, int R>
__global__ void __launch_bounds__(kThreads, 2) argk_kernel(const ArgkParams p) {
    using Cfg = ArgkCfg<D>;
    constexpr int RS = Cfg::RS;
    extern __shared__ __align__(128) unsigned char smem_raw[];

    int64_t row0, row_end, q0, npc;                                       // record pairs [q0, q0 + npc)
    int sp;
    if (p.units) {
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
    const int K = p.K;
    float xr[R][D];
    float dist[R][KMAX];
    int32_t idx[R][KMAX];
    float kth[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        const bool ok = i < row_end;
#pragma unroll
        for (int d = 0; d < D; ++d) xr[r][d] = ok ? __ldg(p.x + i * D + d) : 0.0f;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) { dist[r][k] = INFINITY; idx[r][k] = -1; }
        kth[r] = INFINITY;
    }

    for (int k = 0; k < nt; ++k) {
        const float *tile = ring.acquire(k);
        const int np = k == nt - 1 ? last_np : Cfg::PAIRS;
#pragma unroll kArgkUnroll
        for (int pp = 0; pp < np; ++pp) {
            float f[RS];
#pragma unroll
            for (int u = 0; u < RS / 4; ++u) {
                const float4 v = lds128(tile + pp * RS + 4 * u);
                f[4 * u + 0] = v.x; f[4 * u + 1] = v.y; f[4 * u + 2] = v.z; f[4 * u + 3] = v.w;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 dd = add2(dup2(xr[r][0]), make_float2(f[0], f[1]));
                float2 q = mul2(dd, dd);
#pragma unroll
                for (int d = 1; d < D; ++d) {
                    dd = add2(dup2(xr[r][d]), make_float2(f[2 * d], f[2 * d + 1]));
                    q = fma2(dd, dd, q);
                }
                if (fminf(q.x, q.y) < kth[r]) {
                    const int32_t jx = __float_as_int(f[2 * D]), jy = __float_as_int(f[2 * D + 1]);
                    if (q.x < kth[r]) topk_insert<KMAX>(dist[r], idx[r], K, q.x, jx, kth[r]);
                    if (q.y < kth[r]) topk_insert<KMAX>(dist[r], idx[r], K, q.y, jy, kth[r]);
                }
            }
        }
        ring.release(k);
    }

#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = row0 + r * (kConsumerWarps * 32) + ct;
        if (i >= row_end) continue;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            if (k >= K) break;
            if (p.split > 1) {
                const int64_t off = ((int64_t)sp * p.M + i) * K + k;
                p.pdist[off] = dist[r][k];
                p.pidx[off] = idx[r][k];
            } else {
                p.dist[i * K + k] = dist[r][k];
                p.idx[i * K + k] = idx[r][k] < 0 ? -1 : (int64_t)idx[r][k] + p.j_offset;
            }
        }
    }
}

// Small-M mode (north star (a), the warp-shuffle finish; see sum_smm.cu): one row per CTA, the
// 256 threads take the tile's record pairs t, t + 256, ... and keep their own sorted K-list; the
// CTA then merges the 256 lists in K rounds of a lexicographic (d, j) argmin (warp shuffles, then
// the 8 warp winners in a fixed order), so the result is independent of the thread schedule.
template <int D, int KMAX>
__global__ void __launch_bounds__(kThreads, 1) argk_smm_kernel(const ArgkParams p) {
    using Cfg = ArgkCfg<D>;
    constexpr int RS = Cfg::RS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int64_t i = blockIdx.x % p.M;                 // split-major: concurrent CTAs share j-ranges
    const int sp = (int)(blockIdx.x / p.M);
    const int64_t q0 = (int64_t)sp * p.pairs_per_split;
    const int64_t npc = max(min(q0 + p.pairs_per_split, p.npv) - q0, (int64_t)0);
    const int nt = (int)((npc + Cfg::PAIRS - 1) / Cfg::PAIRS);
    const int last_np = (int)(npc - (int64_t)(nt > 0 ? nt - 1 : 0) * Cfg::PAIRS);
    JRing<kStages> ring;
    ring.init(smem_raw, Cfg::TILE_FLOATS, p.J + q0 * RS, nt, kConsumerWarps, (uint32_t)last_np * RS * 4u);

    const int ct = threadIdx.x, lane = ct & 31, warp = ct >> 5;
    const int K = p.K;
    float xr[D];
#pragma unroll
    for (int d = 0; d < D; ++d) xr[d] = __ldg(p.x + i * D + d);
    float dist[KMAX];
    int32_t idx[KMAX];
    float kth = INFINITY;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) { dist[k] = INFINITY; idx[k] = -1; }
    for (int k = 0; k < nt; ++k) {
        const float *tile = ring.acquire(k);
        const int np = k == nt - 1 ? last_np : Cfg::PAIRS;
        for (int pp = ct; pp < np; pp += kThreads) {
            float f[RS];
#pragma unroll
            for (int u = 0; u < RS / 4; ++u) {
                const float4 v = lds128(tile + pp * RS + 4 * u);
                f[4 * u + 0] = v.x; f[4 * u + 1] = v.y; f[4 * u + 2] = v.z; f[4 * u + 3] = v.w;
            }
            float2 dd = add2(dup2(xr[0]), make_float2(f[0], f[1]));
            float2 q = mul2(dd, dd);
#pragma unroll
            for (int d = 1; d < D; ++d) {
                dd = add2(dup2(xr[d]), make_float2(f[2 * d], f[2 * d + 1]));
                q = fma2(dd, dd, q);
            }
            if (fminf(q.x, q.y) < kth) {
                const int32_t jx = __float_as_int(f[2 * D]), jy = __float_as_int(f[2 * D + 1]);
                if (q.x < kth) topk_insert<KMAX>(dist, idx, K, q.x, jx, kth);
                if (q.y < kth) topk_insert<KMAX>(dist, idx, K, q.y, jy, kth);
            }
        }
        ring.release(k);
    }
    // CTA merge of the 256 sorted lists: K rounds of a lexicographic argmin over the list heads
    float *ld = reinterpret_cast<float *>(smem_raw + argk_smm_list_offset<D>());
    int32_t *lj = reinterpret_cast<int32_t *>(ld + kThreads * KMAX);
    __shared__ float wd[kConsumerWarps];
    __shared__ int32_t wj[kConsumerWarps], wt[kConsumerWarps];
    __shared__ int gwin;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) { ld[ct * KMAX + k] = dist[k]; lj[ct * KMAX + k] = idx[k]; }
    __syncthreads();
    int head = 0;
    for (int k = 0; k < K; ++k) {
        float d = head < K ? ld[ct * KMAX + head] : INFINITY;
        int32_t j = head < K ? lj[ct * KMAX + head] : -1;
        int32_t t = ct;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float od = __shfl_xor_sync(0xffffffffu, d, o);
            const int32_t oj = __shfl_xor_sync(0xffffffffu, j, o);
            const int32_t ot = __shfl_xor_sync(0xffffffffu, t, o);
            if (od < d || (od == d && (uint32_t)oj < (uint32_t)j)) { d = od; j = oj; t = ot; }
        }
        if (lane == 0) { wd[warp] = d; wj[warp] = j; wt[warp] = t; }
        __syncthreads();
        if (ct == 0) {
            float bd = wd[0]; int32_t bj = wj[0], bt = wt[0];
            for (int w = 1; w < kConsumerWarps; ++w)
                if (wd[w] < bd || (wd[w] == bd && (uint32_t)wj[w] < (uint32_t)bj)) { bd = wd[w]; bj = wj[w]; bt = wt[w]; }
            gwin = bt;
            if (p.split > 1) {
                const int64_t off = ((int64_t)sp * p.M + i) * K + k;
                p.pdist[off] = bd;
                p.pidx[off] = bj;
            } else {
                p.dist[i * K + k] = bd;
                p.idx[i * K + k] = bj < 0 ? -1 : (int64_t)bj + p.j_offset;
            }
        }
        __syncthreads();
        if (ct == gwin) ++head;
    }
}

template <int KMAX>
constexpr int argk_rows() { return KMAX <= 4 ? GENRED_ARGK_R : 1; }

template <int D, int KMAX>
static cudaError_t run_argk(const ArgkLaunch &a, cudaStream_t st, int *ctas) {
    using Cfg = ArgkCfg<D>;
    constexpr int R = argk_rows<KMAX>();
    auto kern = argk_kernel<D, KMAX, R>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    ArgkParams p;
    p.x = a.x; p.J = a.J; p.M = a.M; p.K = a.K; p.split = a.split;
    p.pairs_per_split = a.pairs_per_split; p.npv = a.npv; p.dist = a.dist; p.idx = a.idx;
    p.j_offset = a.j_offset; p.pdist = a.pdist; p.pidx = a.pidx; p.units = a.units;
    const int64_t rows = (int64_t)kConsumerWarps * 32 * R;
    const int64_t grid = a.units ? a.n_units : ((a.M + rows - 1) / rows) * a.split;
    if (grid == 0) { *ctas = 0; return cudaSuccess; }
    *ctas = (int)grid;
    kern<<<(unsigned)grid, kThreads, Cfg::SMEM, st>>>(p);
    return cudaGetLastError();
}

template <int D, int KMAX>
static int occ_argk() {
    using Cfg = ArgkCfg<D>;
    auto kern = argk_kernel<D, KMAX, argk_rows<KMAX>()>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, Cfg::SMEM) != cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

template <int D>
static cudaError_t run_argk_k(const ArgkLaunch &a, cudaStream_t st, int *ctas) {
    if (a.K <= 1) return run_argk<D, 1>(a, st, ctas);
    if (a.K <= 4) return run_argk<D, 4>(a, st, ctas);
    if (a.K <= 16) return run_argk<D, 16>(a, st, ctas);
    return run_argk<D, 32>(a, st, ctas);
}
template <int D>
static int occ_argk_k(int K) {
    if (K <= 1) return occ_argk<D, 1>();
    if (K <= 4) return occ_argk<D, 4>();
    if (K <= 16) return occ_argk<D, 16>();
    return occ_argk<D, 32>();
}

int argk_rows_per_thread(int K) { return K <= 4 ? GENRED_ARGK_R : 1; }

#define GENRED_ARGK_D(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

cudaError_t launch_argk(const ArgkLaunch &a, cudaStream_t st, int *ctas) {
#define GENRED_CASE(DD) if (a.D == DD) return run_argk_k<DD>(a, st, ctas);
    GENRED_ARGK_D(GENRED_CASE)
#undef GENRED_CASE
    return cudaErrorInvalidValue;
}

template <int D, int KMAX>
static cudaError_t run_argk_smm(const ArgkLaunch &a, cudaStream_t st, int *ctas) {
    auto kern = argk_smm_kernel<D, KMAX>;
    constexpr int smem = argk_smm_smem<D, KMAX>();
    {
        const cudaError_t e = smem_opt_in((const void *)kern, smem);
        if (e != cudaSuccess) return e;
    }
    ArgkParams p;
    p.x = a.x; p.J = a.J; p.M = a.M; p.K = a.K; p.split = a.split;
    p.pairs_per_split = a.pairs_per_split; p.npv = a.npv; p.dist = a.dist; p.idx = a.idx;
    p.j_offset = a.j_offset; p.pdist = a.pdist; p.pidx = a.pidx; p.units = nullptr;
    const int64_t grid = a.M * a.split;
    if (grid == 0) { *ctas = 0; return cudaSuccess; }
    *ctas = (int)grid;
    kern<<<(unsigned)grid, kThreads, smem, st>>>(p);
    return cudaGetLastError();
}

template <int D>
static cudaError_t run_argk_smm_k(const ArgkLaunch &a, cudaStream_t st, int *ctas) {
    if (a.K <= 1) return run_argk_smm<D, 1>(a, st, ctas);
    if (a.K <= 4) return run_argk_smm<D, 4>(a, st, ctas);
    if (a.K <= 16) return run_argk_smm<D, 16>(a, st, ctas);
    return run_argk_smm<D, 32>(a, st, ctas);
}

cudaError_t launch_argk_smm(const ArgkLaunch &a, cudaStream_t st, int *ctas) {
#define GENRED_CASE(DD) if (a.D == DD) return run_argk_smm_k<DD>(a, st, ctas);
    GENRED_ARGK_D(GENRED_CASE)
#undef GENRED_CASE
    return cudaErrorInvalidValue;
}

int argk_occupancy(int D, int K, int R) {
    (void)R;
#define GENRED_CASE(DD) if (D == DD) return occ_argk_k<DD>(K);
    GENRED_ARGK_D(GENRED_CASE)
#undef GENRED_CASE
    return 1;
}

}  // namespace genred
