// internal.h -- launch interfaces between the C-ABI layer (genred_abi.cu) and the kernel
// translation units.  Not installed; not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <set>
#include <utility>

namespace genred {

// Opt a kernel in to `bytes` of dynamic shared memory on the current device, once per (kernel,
// device): the attribute is per device, so a process driving several GPUs needs it on each.
inline cudaError_t smem_opt_in(const void *kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

constexpr int kTileJ = 512;                 // j-records per shared-memory stage
constexpr int kStages = 4;                  // depth of the bulk-copy ring
constexpr int kConsumerWarps = 8;           // math warps per CTA
constexpr int kThreads = kConsumerWarps * 32;         // all math warps; thread 0 also refills the j-ring
constexpr float kLseSentinel = -3.0e38f;    // finite "minus infinity" reference of an empty LSE state
// j-splits of the Sum and LSE kernels are whole multiples of this many record pairs (32 j): the
// Sum's record-pair unroll and the LSE's 16-pair rescale sub-chunk both divide it.
constexpr int kSplitGrain = 16;
// Gradient modes with E = 1: the j-records also carry b_j y'_j (expanded form), so a pair
// accumulates S0 += e b and S_d += e (b y')_d with 1 + D FFMA2 instead of FMUL2 + FADD2 + D FFMA2.
#ifndef GENRED_GRAD_BY
#define GENRED_GRAD_BY 1
#endif
constexpr bool kGradBY = GENRED_GRAD_BY != 0;
// Record-pair floats of the Gaussian family: [2D coords][w pair][2E signal][2D b y' (gradient
// modes with E = 1, kGradBY)], padded to 16 bytes.
inline int gauss_record_stride(int D, int E, bool grad) {
    const int by = (grad && E == 1 && kGradBY) ? 2 * D : 0;
    return (2 * (D + 1) + 2 * E + by + 3) / 4 * 4;
}

// Record stride (floats) of one j-PAIR in the packed layout: 2*(D+E) rounded up to 4.
inline int record_stride(int D, int E) { return ((2 * (D + E)) + 3) / 4 * 4; }

enum PackKind { PACK_GAUSS = 0, PACK_SQDIST_SUM = 1, PACK_LSE_HZ = 2, PACK_ARGKMIN = 3, PACK_LSE_H = 4,
                PACK_GAUSS_AUTO = 5, PACK_GAUSS_AUTO_RAW = 7 };

// Pack y (N x D) and b (N x E) into the pair-interleaved j-record layout used by every small-D
// kernel: pair p holds (-s*y_d[2p], -s*y_d[2p+1]) for d < D, then (b_e[2p], b_e[2p+1]) for e < E
// (Sum kinds), nothing more (ArgKMin, LSE with h = 0), or (h'hi[2p], h'hi[2p+1], c[2p], c[2p+1])
// with h' = hscale * h, h'hi its fp32 rounding and c = 2^(h' - h'hi) (LSE with h).  Records past N
// (padding up to npairs) hold y = 0 and b = 0 (Sum), or y = +inf and h = -inf (LSE, ArgKMin),
// which contribute nothing.
// PACK_GAUSS_AUTO (Gaussian Sum): decodes the bounding box `geo` (geo.cuh) and writes either the
// expanded records (y' = s (y - c), w = -|y'|^2, b) or the direct ones (-y raw, 0, b): the kernel
// forms raw differences x - y and scales their squared norm by s^2 (readings R18d, R18e).
// PACK_GAUSS_AUTO_RAW (gradient modes): as PACK_GAUSS_AUTO, plus the b y' slots (kGradBY).
cudaError_t launch_pack(int kind, const float *y, const float *b, int64_t N, int D, int E,
                        float s, double hscale, int64_t npairs, float *J, cudaStream_t st,
                        const uint32_t *geo = nullptr);
// Small problems (max(M, N) <= kFusedBoxMax): pack with the bounding box reduced inside the pack
// kernel (every block reduces the whole of x and y, block 0 stores geo), replacing the memset +
// bbox_kernel pair by nothing: one launch fewer on the latency-bound C1 path.
constexpr int64_t kFusedBoxMax = 4096;
cudaError_t launch_pack_boxed(int kind, const float *y, const float *b, int64_t N, int D, int E,
                              float s, int64_t npairs, float *J, const float *x, int64_t M,
                              uint32_t *geo, cudaStream_t st);
// Per-coordinate bounding boxes of y (N x D) and x (M x D) into geo[32] (encoded, geo.cuh).
cudaError_t launch_bbox(const float *x, int64_t M, const float *y, int64_t N, int D, uint32_t *geo,
                        cudaStream_t st);
// Host mirror of the device path decision (reads geo back; synchronises; introspection only).
bool geo_expanded_host(const uint32_t *geo_dev, int D, float s);
int pack_record_stride(int kind, int D, int E);

// Block-sparse ranges ("cluster-wise block-sparsity patterns"): one CTA per unit,
// the rows [row0, row_end) of one i-cluster against the ntiles j-tiles starting at tile0 of the
// range-packed J (the cluster's j-intervals gathered contiguously, padded to whole tiles).
struct RangeUnit {
    int64_t row0, row_end, tile0, ntiles;
};
// One gathered j-interval: destination record pair `dst`, source j-interval [js, je)
// (js = je = 0 marks padding records).
struct RangeCopy {
    int64_t dst, js, je;
};
cudaError_t launch_pack_ranges(int kind, const float *y, const float *b, int64_t N, int D, int E,
                               float s, const RangeCopy *copies, int ncopies, int64_t npairs,
                               float *J, cudaStream_t st, const uint32_t *geo);

struct SumLaunch {
    int mode;                 // 0 SUM, 1 GRADX, 2 SUM_GRADX, 3 SQDIST_SUM
    int D, E, R;              // R = rows per consumer thread
    const float *x, *J, *g;
    const uint32_t *geo;      // MODE 0: encoded bounding box (geo.cuh)
    int64_t M;
    int split;                // number of j-splits (grid = itiles * split)
    int64_t pairs_per_split;  // record pairs per j-split (multiple of kSplitGrain)
    int64_t npv;              // record pairs reduced: ceil(N/2) rounded up to kSplitGrain
    float s;                  // coordinate pre-scale (sqrt(log2e)/sigma, or 1 for SQDIST)
    double scale_sum, scale_grad;
    void *out; int out_f64;   // sum output (SUM / SUM_GRADX / SQDIST_SUM) or gradient (GRADX)
    float *out_grad;          // SUM_GRADX gradient output
    double *part;             // split > 1: split x M x C fp64 partials
    const RangeUnit *units;   // block-sparse ranges (device), or nullptr
    int64_t n_units;
    unsigned *tile_done = nullptr;  // split > 1: zeroed per-row-tile counters -> merge in the kernel
    int num_sms = 148;        // persistent grid: at most num_sms x occupancy CTAs
    // MODE 0, tile-centred form (tile_order.cu, R18j): per 512-j tile (centre, radius^2 or -1 =
    // direct layout); pairs_per_split is then a multiple of kTileJ / 2
    const float4 *centers = nullptr;
    int split_major = 0;      // row-tile CTAs ordered split by split (L2 residency of a split's records)
};
cudaError_t launch_sum(const SumLaunch &a, cudaStream_t st, int *ctas);
// Tile-centred form (tile_order.cu): Hilbert keys of y over its box (geo), a radix sort of
// (key, j), and the per-tile pack (records + centers).  Scratch: keys/idx/keys_s/perm N words
// each, temp = tile_order_temp_bytes(N).  *kernels = kernels launched.
size_t tile_order_temp_bytes(int64_t N);
cudaError_t launch_tile_order(const float *y, const float *b, int64_t N, int D, int E, float s,
                              const uint32_t *geo, uint32_t *keys, uint32_t *idx, uint32_t *keys_s,
                              uint32_t *perm, void *temp, size_t temp_bytes, int64_t ntiles, float *J,
                              float4 *centers, cudaStream_t st, int *kernels, int lse = 0, int RS_lse = 0,
                              double hscale = 0.0, float r2max = 6.0f);
// Small problems in one launch (sum_small_kernel, sum_body.cuh): E = 1, D <= 4, j-splits of at
// most kSmallMaxPairs record pairs (the CTA's records live in shared memory); a.J is unused.
constexpr int64_t kSmallMaxPairs = 512;
#ifndef GENRED_SMALL_CLUSTER
#define GENRED_SMALL_CLUSTER 1
#endif
constexpr bool kSmallCluster = GENRED_SMALL_CLUSTER != 0;   // split <= 8: merge through DSMEM
cudaError_t launch_sum_small(const SumLaunch &a, const float *y, const float *b, int64_t N,
                             cudaStream_t st, int *ctas);
// Small-M mode (sum_smm.cu): CTAs of R = sum_smm_rows(mode) rows whose threads split j; grid =
// ceil(M / R) * split, split-major.  E = 1, D <= 4 only (sum_smm_supported).
bool sum_smm_supported(int mode, int D, int E);
int sum_smm_rows(int mode);
int sum_smm_occupancy(int mode, int D);
cudaError_t launch_sum_smm(const SumLaunch &a, cudaStream_t st, int *ctas);
int sum_occupancy(int mode, int D, int E, int R);
int sum_rows_per_thread_max(int mode, int D, int E);

struct LseLaunch {
    int D, R;
    const float *x, *J;
    int64_t M;
    int split;
    int64_t pairs_per_split;  // record pairs per j-split (multiple of kSplitGrain)
    int64_t npv;              // record pairs reduced: ceil(N/2) rounded up to kSplitGrain
    float negc;               // -log2(e)/eps
    int h_zero;               // h == 0 everywhere (skips a per-pair FADD)
    void *out; int out_f64;   // split == 1: a_i
    double *state;            // split == 1: optional M x 2 state; split > 1: split x M x 2 partials
    const RangeUnit *units = nullptr;   // block-sparse ranges (device), or nullptr
    int64_t n_units = 0;
    // tile-centred form (lse_kernel.cu, R18j): per-tile table of tile_order.cu, s = sqrt(log2 e / eps)
    const float4 *centers = nullptr;
    float s = 0.0f;
};
cudaError_t launch_lse(const LseLaunch &a, cudaStream_t st, int *ctas);
// Record stride (floats per record pair) of the tile-centred LSE layout (tile_order.cu)
int lse_local_record_stride(int D, bool hz);
// Tile radius bound (s units, squared) of the tile-centred LSE: the exponent's fp32 rounding stays
// below ~3 ulp(4) for the dominant terms (1e-6 absolute bar of R6; R18j)
constexpr float kLseLocalR2Max = 0.5f;
// Small-M mode (lse_kernel.cu): CTAs of lse_smm_rows(D) rows whose threads split j; grid =
// ceil(M / R) * split, split-major, 2 CTAs per SM.
int lse_smm_rows(int D);
cudaError_t launch_lse_smm(const LseLaunch &a, cudaStream_t st, int *ctas);
int lse_occupancy(int D, int R, bool hz);
int lse_rows_per_thread_max(int D);

struct ArgkLaunch {
    int D, K, R;
    const float *x, *J;
    int64_t M;
    int split;
    int64_t pairs_per_split, npv;                  // record-pair j-splits (multiple of kSplitGrain)
    float *dist; int64_t *idx; int64_t j_offset;   // split == 1 outputs
    float *pdist; int32_t *pidx;                   // split > 1: split x M x K partials
    const RangeUnit *units = nullptr;              // block-sparse ranges (device), or nullptr
    int64_t n_units = 0;
};
cudaError_t launch_argk(const ArgkLaunch &a, cudaStream_t st, int *ctas);
// Small-M mode (argk_kernel.cu): one row per CTA, threads split j, K-round CTA merge; grid =
// M * split, split-major; partial lists as launch_argk's.
cudaError_t launch_argk_smm(const ArgkLaunch &a, cudaStream_t st, int *ctas);
int argk_occupancy(int D, int K, int R);
int argk_rows_per_thread(int K);

// Softmax-weighted sums / gradients (the LSE backward, softmax_grad_kernel.cu).
struct SmLaunch {
    int D, R;
    const float *x, *J, *coef;
    const double *alpha;
    int64_t M;
    int split;
    int64_t pairs_per_split, npv;  // record-pair j-splits (multiple of kSplitGrain)
    float negc;
    double scale_grad;
    void *out; int out_f64;
    float *out_grad;
    double *part;
};
cudaError_t launch_softmax_grad(const SmLaunch &a, cudaStream_t st, int *ctas);
int softmax_grad_occupancy(int D, int R);
int sm_rows_per_thread_max(int D);
int softmax_record_stride(int D);
cudaError_t launch_pack_softmax(const float *y, const float *sig, const double *beta, int64_t N,
                                int D, int64_t npairs, float *J, cudaStream_t st);

// Large-D ArgKMin on the tensor cores (knn_tc.cu): 3xTF32 tcgen05 screening + exact re-rank.
struct KnnTcLaunch {
    const float *x, *y;
    int64_t M, N;
    int D, K;
    float *dist;
    int64_t *idx;
    int64_t j_offset;
    void *scratch;                     // knn_tc_scratch_bytes(M, N, D, K) bytes, 1024-aligned
    int num_sms;
    cudaEvent_t ev_start, ev_stop;     // optional: recorded around the tcgen05 kernel
};
struct KnnTcInfo {
    int kernels;
    int ctas;
    int *fallback_count;               // device int: rows rescanned exactly
};
int knn_tc_group();
size_t knn_tc_scratch_bytes(int64_t M, int64_t N, int D, int K);
cudaError_t launch_knn_tc(const KnnTcLaunch &a, cudaStream_t st, KnnTcInfo *info);


// Gaussian Sum at the HBM-bound edge (edge_kernel.cu): N <= sum_edge_max_n(), D <= 4, E = 1,
// x 16-byte aligned; J = the PACK_GAUSS_AUTO direct records (geo = nullptr).
int sum_edge_max_n();
int sum_edge_tile_rows();   // x rows per bulk-copied tile of the edge kernel
cudaError_t launch_sum_edge(const float *x, const float *J, int64_t N, int D, int RS, int64_t M, float s,
                            double scale, void *out, int out_f64, int num_sms, cudaStream_t st, int *ctas);

// Deterministic (fixed-order) merges of split-j partials.
cudaError_t launch_sum_finalize(const double *part, int split, int64_t M, int C, int cols_sum,
                                const float *g, int E, double scale_sum, double scale_grad,
                                int mode, void *out, int out_f64, float *out_grad, cudaStream_t st);
cudaError_t launch_lse_finalize(const double *part, int split, int64_t M, void *out, int out_f64,
                                double *state_out, cudaStream_t st);
cudaError_t launch_topk_merge_i32(const float *pd, const int32_t *pi, int split, int64_t M, int K,
                                  float *dist, int64_t *idx, int64_t j_offset, cudaStream_t st);
// First level of a two-level merge for split > 64: groups of 64 lists -> ceil(split / 64) lists
// in the same (split-major) partial layout.
cudaError_t launch_topk_merge_groups(const float *pd, const int32_t *pi, int split, int64_t M, int K,
                                     float *gd, int32_t *gi, cudaStream_t st);
cudaError_t launch_topk_merge_i64(const float *pd, const int64_t *pi, int G, int64_t M, int K,
                                  float *dist, int64_t *idx, cudaStream_t st);
cudaError_t launch_fill(int kind, int64_t M, int C, int K, void *out, int out_f64, float *out_grad,
                        int64_t *idx, double *state, cudaStream_t st);

}  // namespace genred
