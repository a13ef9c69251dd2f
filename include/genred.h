/*
 * genred.h -- C ABI of libgenred, the B200 (sm_100a) Genred hot path.
 *
 * The paper's problem statement (Sec. 2, Eq. 1): given parameters p, i-variables
 * x_i (i = 1..M), j-variables y_j (j = 1..N), a formula F and a reduction, evaluate
 *
 *        a_i = Reduction_{j=1..N} F(p, x_i, y_j)          "with a linear memory footprint".
 *
 * libgenred evaluates Eq. (1) for a FIXED formula set (the Gaussian kernel
 * product Scal<Exp<Minus<SqDist<X,Y>>>,B>; its gradient; the squared
 * distance) and the reductions Sum, log-sum-exp and ArgKMin.  Nothing of
 * size M*N is ever allocated: library scratch is O((M+N)*(D+E)).
 *
 * Conventions (every entry point):
 *   - Data pointers are fp32 row-major contiguous unless stated; by default they are DEVICE
 *     pointers (GENRED_MEM_DEVICE).  With GENRED_MEM_HOST, x/y/b/g/out/out_idx/lse_state are
 *     HOST pointers: the call stages them through context-owned device buffers (H2D, compute,
 *     D2H on `stream`) and returns only after the results are in host memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Ownership: the caller owns every pointer and the stream.  The library reads x, y, b, g and
 *     writes only out, out_idx, out_grad and lse_state.  Device-mode calls are asynchronous:
 *     they return after enqueue and the buffers must stay live until the stream passes.
 *   - Errors: return codes only (no abort, no C++ exception crosses the ABI).  Validation is
 *     synchronous and happens before any launch; on error nothing is written.  The message of
 *     the last failure on a context is returned by genred_last_error().  Asynchronous device
 *     faults surface at the caller's next synchronisation.
 *   - NaN / Inf inputs propagate under IEEE semantics and are not checked.
 *   - A context is used by one host thread at a time; distinct contexts are independent.
 *   - Calls on one context must be STREAM-SERIALISED: its scratch arena and its split-merge
 *     arrival counters (one per row tile, zero at rest, reset by the merging CTA) are shared by
 *     every call, so two calls in flight at once on different streams -- or concurrent replays
 *     of a captured graph -- would interleave on them and give wrong results.  For concurrency
 *     use one context per stream.
 *   - CUDA graphs: once a context's scratch arena has grown to the largest problem (one warm-up
 *     call), device-mode genred_eval neither synchronises nor allocates, so it can be captured
 *     on `stream`.  Captured launches use that arena: while the graph lives, calls on the same
 *     context must not need a larger arena nor run concurrently on another stream.
 */
#ifndef GENRED_H
#define GENRED_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GENRED_ABI_VERSION 3

typedef struct genred_ctx genred_ctx;

typedef enum {
    GENRED_OK = 0,
    GENRED_E_INVALID = 1,      /* bad argument value / null pointer / misalignment */
    GENRED_E_UNSUPPORTED = 2,  /* (formula, reduction, D, E, K) not in the supported set */
    GENRED_E_SHAPE = 3,        /* negative sizes, D/E/K out of range */
    GENRED_E_NOMEM = 4,        /* scratch allocation failed */
    GENRED_E_CUDA = 5          /* a CUDA runtime call or launch failed (message has the reason) */
} genred_status;

/* Formulas F (readings R1, R2, R5, R10 in DESIGN.md; LSE_GRAD: SURVEY 8(f) row 2):
 *   GAUSS           F_ij = exp(-|x_i - y_j|^2 / sigma^2) * b_j                 (E outputs)
 *   GAUSS_GRADX     F_ij = d/dx_i of the above, contracted with the cotangent g_i:
 *                   (-2/sigma^2) (x_i - y_j) exp(-|x_i-y_j|^2/sigma^2) <b_j, g_i>  (D outputs)
 *   GAUSS_SUM_GRADX both of the above in one pass (out: M x E sum, out_grad: M x D gradient)
 *   SQDIST          F_ij = |x_i - y_j|^2; under LSE: F_ij = -|x_i - y_j|^2 / eps + h_j,
 *                   with h = b (N values, E = 1; NULL means h = 0).
 *   LSE_GRAD        the backward of the LSE reduction: with
 *                   p_ij = exp(-|x_i - y_j|^2/eps + alpha_i + beta_j) (alpha = row_shift,
 *                   beta = col_shift, fp64, NULL = 0; b = sig (N), g = coef (M), NULL = 1):
 *                   out = S_i = sum_j sig_j p_ij (M values) and
 *                   out_grad = coef_i (-2/eps) sum_j sig_j p_ij (x_i - y_j) (M x D, fp32).
 *                   alpha = -a (the forward LSE), beta = h gives S = 1 and out_grad = da/dx;
 *                   rows y, reduced x, alpha = h, beta = -a, sig = g gives dL/dh and dL/dy.
 *                   Not max-shifted: the caller keeps alpha_i + beta_j - |x-y|^2/eps <= ~80.    */
typedef enum {
    GENRED_GAUSS = 0,
    GENRED_GAUSS_GRADX = 1,
    GENRED_SQDIST = 2,
    GENRED_GAUSS_SUM_GRADX = 3,
    GENRED_LSE_GRAD = 4
} genred_formula;

/* Reductions:
 *   SUM      a_i = sum_j F_ij
 *   LSE      a_i = log sum_j exp(F_ij)   (natural log; max-shifted, streaming)
 *   ARGKMIN  the K smallest (F_ij, j) in lexicographic order (ties -> lowest j), ascending.   */
typedef enum { GENRED_SUM = 0, GENRED_LSE = 1, GENRED_ARGKMIN = 2 } genred_reduction;

typedef enum { GENRED_F32 = 0, GENRED_F64 = 1 } genred_dtype;

typedef enum { GENRED_MEM_DEVICE = 0, GENRED_MEM_HOST = 1 } genred_memory;

/* Supported (formula, reduction) pairs and shapes:
 *   (GAUSS, SUM), (GAUSS_GRADX, SUM), (GAUSS_SUM_GRADX, SUM): 1 <= D <= 8, 1 <= E <= 4
 *   (SQDIST, SUM): 1 <= D <= 8, 1 <= E <= 4 (closed-form test combination)
 *   (SQDIST, LSE), (LSE_GRAD, SUM): 1 <= D <= 8, E == 1
 *   (SQDIST, ARGKMIN): E == 1 and either 1 <= D <= 16, 1 <= K <= 32 (FP32 path), or
 *                      17 <= D <= 16384, 1 <= K <= 28 (tcgen05 3xTF32 screening + exact fp64
 *                      re-rank of the K' best candidates, PAPER.md:97 k-NN)
 * Anything else -> GENRED_E_UNSUPPORTED.                                                        */
typedef struct {
    int32_t abi_version;     /* must equal GENRED_ABI_VERSION */
    int32_t formula;         /* genred_formula */
    int32_t reduction;       /* genred_reduction */
    int32_t memory;          /* genred_memory: DEVICE (default 0) or HOST pointers */
    int64_t M, N;            /* rows of x (i-variables) and of y (j-variables); >= 0 */
    int32_t D, E, K;         /* point dimension, signal dimension, K of ArgKMin (else ignored) */
    int32_t split_j;         /* 0 = automatic; >= 1 forces the number of j-splits (tests) */
    double  scale;           /* sigma (GAUSS*) or eps (SQDIST+LSE); finite and > 0; ignored otherwise */
    const float *x;          /* M x D */
    const float *y;          /* N x D */
    const float *b;          /* N x E signal (GAUSS*, SQDIST+SUM; NULL means b = 1 with E = 1),
                                or h (N values) for SQDIST+LSE (NULL means h = 0)           */
    const float *g;          /* M x E cotangent for *_GRADX (NULL means g = 1) */
    void    *out;            /* SUM: M x E | GAUSS_GRADX: M x D | LSE: M | ARGKMIN: M x K
                                squared distances (always fp32 for ARGKMIN)                   */
    int32_t  out_dtype;      /* genred_dtype of `out` (SUM/GRADX/LSE); F64 recommended for LSE */
    int32_t  pad0;
    float   *out_grad;       /* GAUSS_SUM_GRADX only: M x D fp32 gradient */
    int64_t *out_idx;        /* ARGKMIN: M x K, 0-based j (+ j_offset); pad -1 (d = +inf) if K > N */
    double  *lse_state;      /* optional, LSE only: M x 2 (m_i in log2 units, s_i) so that
                                a_i = ln2 * (m_i + log2 s_i); input of genred_combine_lse      */
    int64_t  j_offset;       /* added to every reported index (j-sharded evaluation) */
    const double *row_shift; /* LSE_GRAD: alpha (M values) */
    const double *col_shift; /* LSE_GRAD: beta (N values) */
    /* Block-sparse ranges ("cluster-wise block-sparsity patterns"; KeOps'
     * ranges_i / slices_i / redranges_j convention).  HOST int64 arrays, used when n_ranges > 0
     * (Sum reductions of GAUSS, GAUSS_GRADX, GAUSS_SUM_GRADX, SQDIST; (SQDIST, LSE); and
     * (SQDIST, ARGKMIN) with D <= 16, whose indices are the original j):
     *   ranges_i[2c], ranges_i[2c+1]   rows [is, ie) of cluster c; clusters sorted, disjoint
     *   slices[c]                     end of cluster c's intervals in ranges_j (cumulative)
     *   ranges_j[2k], ranges_j[2k+1]  j-interval [js, je); a cluster's intervals sorted, disjoint
     * a_i reduces over the union of its cluster's j-intervals; rows outside every cluster get the
     * neutral value (0, -inf for LSE, (+inf, -1) for ArgKMin).  split_j is ignored. */
    int64_t n_ranges;
    const int64_t *ranges_i;
    const int64_t *slices;
    const int64_t *ranges_j;
} genred_args;

/* Library-level information. */
int32_t     genred_abi_version(void);
const char *genred_build_info(void);                 /* compile flags, target arch */

/* Context: one per CUDA device; owns the scratch arena (packed j-records, split-j partials,
 * host-mode staging buffers), grown geometrically, freed by genred_destroy. */
genred_status genred_create(int32_t cuda_device, genred_ctx **out);
void          genred_destroy(genred_ctx *ctx);
const char   *genred_last_error(const genred_ctx *ctx);

/* Host-only argument check (no GPU needed): returns the status genred_eval would return from
 * validation, and writes a message into msg[0..msg_len) (may be NULL). */
genred_status genred_validate(const genred_args *args, char *msg, size_t msg_len);

/* Evaluate Eq. (1) for `args` on `stream` (see conventions above). */
genred_status genred_eval(genred_ctx *ctx, const genred_args *args, void *stream);

/* Merge G partial log-sum-exp states (G x M x 2 doubles, as written to lse_state) of one set of
 * rows, e.g. from G j-shards: (m, s)_1 (+) (m, s)_2 = (m*, s_1 2^(m_1-m*) + s_2 2^(m_2-m*)),
 * m* = max(m_1, m_2) (reduction_monoids merge).  Writes a_i (natural log) to
 * `out` (M values, dtype) and, if state_out != NULL, the merged state (M x 2).  Device pointers. */
genred_status genred_combine_lse(genred_ctx *ctx, int64_t M, int32_t G, const double *states,
                                 void *out, int32_t out_dtype, double *state_out, void *stream);

/* Merge G sorted K-lists per row (G x M x K distances and indices, each list ascending in (d, j))
 * into the K smallest under (d, j) lexicographic order (ArgKMin merge).
 * Device pointers. */
genred_status genred_merge_topk(genred_ctx *ctx, int64_t M, int32_t K, int32_t G,
                                const float *d, const int64_t *idx,
                                float *d_out, int64_t *idx_out, void *stream);

/* Introspection for tests and the benchmark. */
typedef struct {
    int32_t split_j;         /* j-splits used by the last genred_eval */
    int32_t rows_per_cta;    /* i-rows owned by one CTA */
    int32_t ctas;            /* CTAs launched by the main kernel */
    int32_t tile_j;          /* j-records per shared-memory stage */
    int32_t kernels;         /* kernels launched by the last call */
    int32_t path;            /* 0 = FP32/MUFU small-D path, 1 = tcgen05 tensor path, 2 = Gaussian
                                Sum expanded form with the FP32-pipe exp2 share (synchronises),
                                3 = Gaussian Sum tile-centred form (y in Hilbert order, records
                                centred per 512-j tile; genred_last_tiles counts its tiles) */
    int64_t scratch_bytes;   /* device scratch the last call used (the context may hold more) */
    int64_t fallback_rows;   /* tensor path: rows whose 3xTF32 screening failed the margin
                                certificate and were rescanned exactly (synchronises; else -1) */
} genred_plan;
genred_status genred_last_plan(const genred_ctx *ctx, genred_plan *plan);

/* Tile-centred form of the last call (plan.path == 3; R18j): the number of 512-j tiles
 * and how many of them ran the tile-centred expanded form (the others, wider than the radius bound
 * kExpandedR2Max in sigma units, ran the direct form).  Synchronises (reads the per-tile table).
 * Other paths: both 0. */
genred_status genred_last_tiles(const genred_ctx *ctx, int64_t *local_tiles, int64_t *tiles);

/* Total kernels launched by this context since creation (evidence for the bench's
 * gpu_launches claim). */
int64_t genred_launch_count(const genred_ctx *ctx);

/* Live timing of the dominant kernel for the benchmark's roofline: while enabled, every
 * genred_eval records a pair of CUDA events (owned by the context) on its stream around its
 * main pair-loop kernel, for up to 4096 launches.  genred_profile(ctx, 0) disables and clears.
 * genred_profile_read waits for the recorded events and writes up to `max` durations (ms) in
 * launch order; it returns the number written (or -1 on a CUDA error). */
genred_status genred_profile(genred_ctx *ctx, int32_t enable);
int32_t       genred_profile_read(genred_ctx *ctx, float *ms, int32_t max);

/* Planner switches of a context (defaults read once from the environment at genred_create, so a
 * call does not scan the environment).  Names:
 *   "small_fused"  1 (default; env GENRED_SMALL_FUSED): problems with max(M, N) <= 4096, E = 1,
 *                  D <= 4 run as ONE kernel (CTAs build their own direct-form j-records, split
 *                  partials merged through distributed shared memory in a cluster, or by the last
 *                  CTA); 0 keeps the pack + pair-loop kernels (which may take the expanded form).
 *   "fused_merge"  1 (default; env GENRED_FUSED_MERGE): the last CTA of a row tile merges the
 *                  split partials inside the pair-loop kernel when they are few; 0 always launches
 *                  the finalize kernel.
 *   "local_form"   Gaussian Sum (D <= 3, row tiles): 1 (default; env GENRED_LOCAL_FORM) orders y
 *                  along a Hilbert curve and centres the j-records per 512-j tile when
 *                  N >= 2^18 and M >= 2^16 (the expanded form for clouds wider than the global
 *                  box allows, R18j); 2 does so at any size above the tiny-problem paths; 0 never.
 *                  The j-splits then cover whole tiles.
 * Returns GENRED_E_INVALID for an unknown name; affects later calls on this context only. */
genred_status genred_set_option(genred_ctx *ctx, const char *name, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* GENRED_H */
