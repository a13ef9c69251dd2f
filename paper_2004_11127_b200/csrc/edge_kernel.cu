// edge_kernel.cu -- the Gaussian Genred Sum at the HBM-bound edge: N tiny (N <= 64), M huge
// (SURVEY.md Sec. 8(d) row Cedge; Eq. 1).
//
// With a handful of j's the pair loop is a few dozen FP32 operations per row, so the kernel is
// bound by streaming x in (D floats per row) and a out (one float per row).  The generic pair-loop
// kernel spends a CTA per 1024 rows and pays its whole set-up latency (mbarrier init, j-tile
// copy, x loads, store) once per CTA; here instead:
//   * persistent CTAs (a few per SM) keep the N packed j-records in shared memory for the whole
//     launch and walk row tiles c, c + grid, ...;
//   * each 4096-row x tile (contiguous, 4096 * D * 4 bytes) arrives by one cp.async.bulk into a
//     2-stage shared-memory ring completing on mbarriers (2 CTAs per SM: 192 KB in flight per SM
//     at D = 3; the bytes in flight per SM, not the thread count, set the achieved HBM bandwidth);
//   * a thread evaluates its rows from shared memory in the direct form (no bounding-box pass
//     over x, which would be a second full read) and stores a with coalesced writes.
// The j-records are the PACK_GAUSS_AUTO direct records (raw -y_j pairs, w slot, b_j pairs;
// the kernel scales |x - y|^2 by s^2 as sum_body.cuh's direct form, reading R18e).
#include <math.h>

#include <algorithm>

#include "device.cuh"
#include "internal.h"

namespace genred {
namespace edge {

// Round 2: 4096-row tiles in a 2-stage ring (16 rows per thread) measured 0.970 / 0.743 / 0.247
// of HBM at N = 1 / 8 / 32 against 0.949 / 0.720 / 0.246 for 1024-row tiles in 4 stages (2048 x
// 3: 0.965 / 0.729; 1024 x 6: 0.688 at N = 8; 512 x 8: 0.604; 4096 x 3: 0.638;
// profiles/r02_edge_tiles.txt): fewer, larger bulk copies and half the per-tile barriers.
#ifndef GENRED_EDGE_ROWS
#define GENRED_EDGE_ROWS 4096
#endif
constexpr int kRowsPerTile = GENRED_EDGE_ROWS;
constexpr int kThreads = 256;
constexpr int kRows = kRowsPerTile / kThreads;      // rows per thread per tile
#ifndef GENRED_EDGE_STAGES
#define GENRED_EDGE_STAGES 2
#endif
constexpr int kStages = GENRED_EDGE_STAGES;
constexpr int kMaxPairs = 32;                       // N <= 64

template <int D>
__global__ void __launch_bounds__(kThreads)
sum_edge_kernel(const float *__restrict__ x, const float *__restrict__ J, int npairs, int RS,
                int64_t M, float s, double scale, void *out, int out_f64) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *xt = reinterpret_cast<float *>(smem_raw);                         // [kStages][kRowsPerTile*D]
    float *jr = xt + kStages * kRowsPerTile * D;                             // [npairs][RS]
    uint64_t *full = reinterpret_cast<uint64_t *>(jr + kMaxPairs * 12 + 4);
    const int64_t ntiles = (M + kRowsPerTile - 1) / kRowsPerTile;
    const int64_t nfull = M / kRowsPerTile;           // tiles copied whole (16-byte multiple)
    constexpr uint32_t kTileBytes = kRowsPerTile * D * 4;
    const float2 negs2 = dup2(-(s * s));               // as sum_body.cuh's direct form

    if (threadIdx.x == 0) {
        for (int k = 0; k < kStages; ++k) mbar_init(&full[k], 1);
        fence_barrier_init();
    }
    for (int k = threadIdx.x; k < npairs * RS; k += kThreads) jr[k] = J[k];
    __syncthreads();
    // prologue: the first kStages tiles of this CTA (whole tiles only; a partial last tile is
    // read straight from global memory, never past the end of x)
    if (threadIdx.x == 0) {
        for (int k = 0; k < kStages; ++k) {
            const int64_t t = blockIdx.x + (int64_t)k * gridDim.x;
            if (t < nfull) {
                mbar_arrive_expect_tx(&full[k], kTileBytes);
                bulk_g2s(xt + k * kRowsPerTile * D, x + t * kRowsPerTile * D, kTileBytes, &full[k]);
            }
        }
    }
    int k = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int st = k % kStages;
        const int64_t row0 = t * kRowsPerTile;
        float xr[kRows][D];
        if (t < nfull) {
            mbar_wait(&full[st], (k / kStages) & 1);
            const float *xs = xt + st * kRowsPerTile * D;
#pragma unroll
            for (int r = 0; r < kRows; ++r)
#pragma unroll
                for (int d = 0; d < D; ++d) xr[r][d] = xs[(r * kThreads + threadIdx.x) * D + d];
        } else {
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                const int64_t i = row0 + r * kThreads + threadIdx.x;
#pragma unroll
                for (int d = 0; d < D; ++d) xr[r][d] = i < M ? __ldg(x + i * D + d) : 0.0f;
            }
        }
        __syncthreads();                                  // every thread is done with stage st
        if (threadIdx.x == 0) {
            const int64_t tn = t + (int64_t)kStages * gridDim.x;
            if (tn < nfull) {
                mbar_arrive_expect_tx(&full[st], kTileBytes);
                bulk_g2s(xt + st * kRowsPerTile * D, x + tn * kRowsPerTile * D, kTileBytes, &full[st]);
            }
        }
        float2 acc[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int p = 0; p < npairs; ++p) {
            const float *rec = jr + p * RS;
            float2 ny[D];
#pragma unroll
            for (int d = 0; d < D; ++d) ny[d] = make_float2(rec[2 * d], rec[2 * d + 1]);
            const float2 bv = make_float2(rec[2 * D + 2], rec[2 * D + 3]);
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                float2 dd = add2(dup2(xr[r][0]), ny[0]);
                float2 q = mul2(dd, dd);
#pragma unroll
                for (int d = 1; d < D; ++d) {
                    dd = add2(dup2(xr[r][d]), ny[d]);
                    q = fma2(dd, dd, q);                  // |x - y|^2 (raw differences, R18e)
                }
                const float2 t = mul2(q, negs2);                    // -s^2 |x - y|^2
                const float2 e = make_float2(ex2(t.x), ex2(t.y));
                acc[r] = fma2(e, bv, acc[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            const int64_t i = row0 + r * kThreads + threadIdx.x;
            if (i >= M) continue;
            const double v = ((double)acc[r].x + (double)acc[r].y) * scale;
            if (out_f64) ((double *)out)[i] = v;
            else ((float *)out)[i] = (float)v;
        }
    }
}

template <int D>
static cudaError_t run(const float *x, const float *J, int npairs, int RS, int64_t M, float s,
                       double scale, void *out, int out_f64, int num_sms, cudaStream_t st, int *ctas) {
    auto kern = sum_edge_kernel<D>;
    const int smem = kStages * kRowsPerTile * D * 4 + (kMaxPairs * 12 + 4) * 4 + kStages * 8 + 64;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, smem);
        if (e != cudaSuccess) return e;
    }
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    const int64_t ntiles = (M + kRowsPerTile - 1) / kRowsPerTile;
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)num_sms * std::max(occ, 1));
    *ctas = grid;
    kern<<<grid, kThreads, smem, st>>>(x, J, npairs, RS, M, s, scale, out, out_f64);
    return cudaGetLastError();
}

}  // namespace edge

int sum_edge_max_n() { return 2 * edge::kMaxPairs; }
int sum_edge_tile_rows() { return edge::kRowsPerTile; }

cudaError_t launch_sum_edge(const float *x, const float *J, int64_t N, int D, int RS, int64_t M, float s,
                            double scale, void *out, int out_f64, int num_sms, cudaStream_t st, int *ctas) {
    if (M == 0) { *ctas = 0; return cudaSuccess; }
    if (N > 2 * edge::kMaxPairs || RS > 12) return cudaErrorInvalidValue;
    const int npairs = (int)((N + 1) / 2);
    switch (D) {
        case 1: return edge::run<1>(x, J, npairs, RS, M, s, scale, out, out_f64, num_sms, st, ctas);
        case 2: return edge::run<2>(x, J, npairs, RS, M, s, scale, out, out_f64, num_sms, st, ctas);
        case 3: return edge::run<3>(x, J, npairs, RS, M, s, scale, out, out_f64, num_sms, st, ctas);
        case 4: return edge::run<4>(x, J, npairs, RS, M, s, scale, out, out_f64, num_sms, st, ctas);
    }
    return cudaErrorInvalidValue;
}

}  // namespace genred
