// knn_tc.cu -- ArgKMin over squared distances for large D on the 5th-generation tensor cores
// (k-NN; north star (b)).
//
//   d_ij = |x_i|^2 + |y_j|^2 - 2 x_i . y_j ,   a_i = K smallest (d_ij, j), ties -> lowest j (R7)
//
// a10  prepass: x, y -> tf32 hi/lo split (hi = rna_tf32(v), lo = rna_tf32(v - hi)), rows padded
//      to Dp (multiple of 16) with zeros; |x|^2, |y|^2 accumulated in fp64; max_j |y_j|.
// a11  S_ij = x.y with 3xTF32: A_lo.B_hi + A_hi.B_lo + A_hi.B_hi accumulated in one fp32 TMEM
//      accumulator (tcgen05.mma.cta_group::1.kind::tf32, 128 x 256 x 8), operands staged by TMA
//      (cp.async.bulk.tensor.2d, 64B swizzle) into a 4-stage shared-memory ring; one thread
//      issues MMAs, tcgen05.commit releases smem stages / publishes accumulators; the two
//      256-column accumulators in TMEM (512 columns) let the epilogue of tile t overlap the
//      MMAs of tile t+1.
// a12  epilogue: 4 warps read the accumulator with tcgen05.ld (one TMEM lane = one query row per
//      thread), form d~ = |x|^2 + |y|^2 - 2S and keep a register top-K' (K' = 16 or 32) per row;
//      partial lists per (ref group, row) are merged, the K' candidates are re-ranked with exact
//      fp64 direct differences, and the screening is certified by the margin test of reading
//      R17 (d~_(K') - d~_(K) > 2 delta_i); rows that fail it are rescanned exactly (counted).
//
// Work units: (ref group g of kGroup ref tiles, query row tile r), g-major so that concurrently
// running CTAs share the same ref tiles in L2; CTA c processes units c, c + grid, ...
#include <cuda.h>
#include <math.h>

#include <stdlib.h>

#include <algorithm>

#include "device.cuh"
#include "internal.h"

namespace genred {
namespace tc {

constexpr int BM = 128;                 // query rows per tile (TMEM lanes)
constexpr int BN = 256;                 // refs per tile (TMEM columns per accumulator)
constexpr int BK = 16;                  // fp32/tf32 elements per k-block (64 B rows, 64B swizzle)
constexpr int STAGES = 4;
#ifndef GENRED_KNN_CLUSTER
#define GENRED_KNN_CLUSTER 1
#endif
// CTAs sharing (multicasting) each ref tile.  CLUSTER = 2 is correct (tests pass) and cuts the
// data path (1-MMA probe: 3.47 -> 3.10 ms at C4) but measured 3.77 ms against 3.69 ms for the
// full 3xTF32 kernel: the tensor pipe is then the bound and the pair's lock-step costs more
// than it saves, so 1 is the default.
constexpr int CLUSTER = GENRED_KNN_CLUSTER;
constexpr int A_BYTES = BM * BK * 4;    // 8 KB
constexpr int B_BYTES = BN * BK * 4;    // 16 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;   // hi + lo of both: 48 KB
constexpr int NUM_THREADS = 192;        // warp 0 TMA, warp 1 MMA + TMEM alloc, warps 2-5 epilogue
constexpr int CB = 16;                  // per-thread candidate buffer (epilogue)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 2 * BN * 4 + 256 + 2 * CB * 128 * 4 + 1024;
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB per-CTA shared memory");

__device__ __forceinline__ void tma_load_2d(void *smem, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(smem)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

// Multicast variant: the same box lands at the same offset in every CTA of `mask` (cluster), each
// completing the mbarrier at that offset in its own shared memory.
__device__ __forceinline__ void tma_load_2d_mc(void *smem, const CUtensorMap *map, int c0, int c1,
                                               uint64_t *bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(smem_u32(smem)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask) : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand, 64-byte swizzle: rows of BK*4 = 64 B, 8-row groups 512 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * BK * 4) >> 4) << 32;// SBO: one 8-row swizzle atom
    d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
    d |= (uint64_t)4 << 61;                  // SWIZZLE_64B
    return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, K-major, M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a), "l"(b), "r"(kIdesc), "r"(accum) : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}

// Arrive (when the MMAs issued so far complete) on the barrier at this offset in every CTA of mask.
__device__ __forceinline__ void mma_commit_mc(uint64_t *bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Params {
    int64_t M, N;
    int Dp;
    int nk;                  // Dp / BK
    int n_rtiles, n_ttiles, n_groups, group;
    const float *xn, *yn;    // squared norms (fp32)
    unsigned int *row_thr;   // M: best known K'-th screened value per row (float bits, >= 0)
    float *pd;               // n_groups x M x KP screened distances
    int32_t *pj;             // n_groups x M x KP indices
};

template <int KP>
__device__ __forceinline__ void kp_insert(float (&d)[KP], int32_t (&j)[KP], float cd, int32_t cj,
                                          float &kth) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        const bool sw = cd < d[k] || (cd == d[k] && (uint32_t)cj < (uint32_t)j[k]);
        const float td = d[k];
        const int32_t tj = j[k];
        d[k] = sw ? cd : td;
        j[k] = sw ? cj : tj;
        cd = sw ? td : cd;
        cj = sw ? tj : cj;
    }
    kth = d[KP - 1];
}

// CL = 2: a cluster of two CTAs works on two query row tiles against the same ref tiles; each
// CTA loads its own A tile and HALF of the B tile, multicast to both (B traffic from L2 halves);
// a ring stage may be refilled only once both CTAs' MMAs have read it (empty barriers count 2,
// commits multicast to the pair).
template <int KP, int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap map_xhi, const __grid_constant__ CUtensorMap map_xlo,
              const __grid_constant__ CUtensorMap map_yhi, const __grid_constant__ CUtensorMap map_ylo,
              const Params p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned operand ring (SW128 atoms), then y-norm tiles, then barriers
    unsigned char *base = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    float *ybuf = reinterpret_cast<float *>(base + STAGES * STAGE_BYTES);          // 2 x BN
    uint64_t *bars = reinterpret_cast<uint64_t *>(base + STAGES * STAGE_BYTES + 2 * BN * 4);
    uint64_t *full = bars;                   // [STAGES]
    uint64_t *empty = bars + STAGES;         // [STAGES]
    uint64_t *tfull = bars + 2 * STAGES;     // [2]
    uint64_t *tempty = bars + 2 * STAGES + 2;// [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
    float *cand_d = reinterpret_cast<float *>(base + STAGES * STAGE_BYTES + 2 * BN * 4 + 256);
    int32_t *cand_j = reinterpret_cast<int32_t *>(cand_d + CB * 128);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CL); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
        fence_barrier_init();
    }
    if (warp == 1) {                                     // TMEM: 2 accumulators x 256 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     ::"r"(smem_u32(tmem_slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    if (CL > 1) cluster_sync_all();                      // peer barriers initialised before any multicast
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int n_rgroups = (p.n_rtiles + CL - 1) / CL;    // row tiles per cluster unit
    const int n_units = p.n_groups * n_rgroups;
    const int crank = CL > 1 ? (int)(blockIdx.x % CL) : 0;   // rank in the cluster
    const int ubeg = blockIdx.x / CL, ustep = gridDim.x / CL;
    const uint16_t mc_mask = (uint16_t)((1u << CL) - 1);

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            int stage = 0; uint32_t phase = 0;
            for (int u = ubeg; u < n_units; u += ustep) {
                const int g = u / n_rgroups, r = (u % n_rgroups) * CL + crank;
                const int t0 = g * p.group, t1 = min(t0 + p.group, p.n_ttiles);
                for (int t = t0; t < t1; ++t) {
                    for (int kb = 0; kb < p.nk; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        unsigned char *sb = base + stage * STAGE_BYTES;
                        if (CL > 1) {
                            constexpr int HB = B_BYTES / CL;     // this CTA's share of B
                            mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                            tma_load_2d(sb, &map_xhi, kb * BK, r * BM, &full[stage]);
                            tma_load_2d(sb + A_BYTES, &map_xlo, kb * BK, r * BM, &full[stage]);
                            tma_load_2d_mc(sb + 2 * A_BYTES + crank * HB, &map_yhi, kb * BK,
                                           t * BN + crank * (BN / CL), &full[stage], mc_mask);
                            tma_load_2d_mc(sb + 2 * A_BYTES + B_BYTES + crank * HB, &map_ylo, kb * BK,
                                           t * BN + crank * (BN / CL), &full[stage], mc_mask);
                        } else {
                        mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                        tma_load_2d(sb, &map_xhi, kb * BK, r * BM, &full[stage]);
                        tma_load_2d(sb + A_BYTES, &map_xlo, kb * BK, r * BM, &full[stage]);
                        tma_load_2d(sb + 2 * A_BYTES, &map_yhi, kb * BK, t * BN, &full[stage]);
                        tma_load_2d(sb + 2 * A_BYTES + B_BYTES, &map_ylo, kb * BK, t * BN, &full[stage]);
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer (one thread) ------------------------------
        if (lane == 0) {
            int stage = 0; uint32_t phase = 0;
            int acc = 0; uint32_t aphase = 0;
            for (int u = ubeg; u < n_units; u += ustep) {
                const int g = u / n_rgroups;
                const int t0 = g * p.group, t1 = min(t0 + p.group, p.n_ttiles);
                for (int t = t0; t < t1; ++t) {
                    mbar_wait(&tempty[acc], aphase ^ 1);
                    fence_after();
                    const uint32_t d_tmem = tmem_base + acc * BN;
                    for (int kb = 0; kb < p.nk; ++kb) {
                        mbar_wait(&full[stage], phase);
                        fence_after();
                        const uint32_t sb = smem_u32(base + stage * STAGE_BYTES);
                        const uint64_t ahi = sw_desc(sb), alo = sw_desc(sb + A_BYTES);
                        const uint64_t bhi = sw_desc(sb + 2 * A_BYTES);
                        const uint64_t blo = sw_desc(sb + 2 * A_BYTES + B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 8; ++k) {
                            const uint64_t off = (uint64_t)(k * 32) >> 4;    // 8 tf32 = 32 B
                            mma_tf32(d_tmem, alo + off, bhi + off, (kb | k) != 0);
                            mma_tf32(d_tmem, ahi + off, blo + off, 1);
                            mma_tf32(d_tmem, ahi + off, bhi + off, 1);
                        }
                        if (CL > 1) mma_commit_mc(&empty[stage], mc_mask);
                        else mma_commit(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    mma_commit(&tfull[acc]);
                    if (++acc == 2) { acc = 0; aphase ^= 1; }
                }
            }
        }
    } else {
        // ------------------------------ epilogue: 4 warps, one query row per thread ------------
        // Per value: d~ = fma(-2, S, |x|^2 + |y|^2) and one compare with the row's K'-th best;
        // hits are appended to a per-thread candidate buffer in shared memory (a few instructions,
        // so warp divergence on hits stays cheap) and merged into the sorted register list at the
        // end of every tile or when the buffer fills.
        const int q = warp & 3;                      // TMEM lane quarter this warp may access
        const int row_in_tile = q * 32 + lane;
        const int et = threadIdx.x - 64;             // 0..127
        float *cbd = cand_d + et;                    // column et of a [CB][128] array
        int32_t *cbj = cand_j + et;
        int acc = 0; uint32_t aphase = 0;
        for (int u = ubeg; u < n_units; u += ustep) {
            const int g = u / n_rgroups, r = (u % n_rgroups) * CL + crank;
            const int t0 = g * p.group, t1 = min(t0 + p.group, p.n_ttiles);
            const int64_t i = (int64_t)r * BM + row_in_tile;
            const float xn = i < p.M ? __ldg(p.xn + i) : 0.0f;
            float bd[KP];
            int32_t bj[KP];
#pragma unroll
            for (int k = 0; k < KP; ++k) { bd[k] = INFINITY; bj[k] = -1; }
            float kth = INFINITY;
            // Units of the same row in other CTAs publish their K'-th best: anything not below
            // it cannot enter the row's global top-K' (R17 screening), so it is not a candidate.
            float thr = i < p.M ? __uint_as_float(atomicAdd(p.row_thr + i, 0u)) : INFINITY;
            float lim = fminf(kth, thr);
            int nc = 0;
            for (int t = t0; t < t1; ++t) {
                float *yb = ybuf + acc * BN;
                for (int c = et; c < BN; c += 128) {
                    const int64_t j = (int64_t)t * BN + c;
                    yb[c] = j < p.N ? __ldg(p.yn + j) : INFINITY;      // padded refs never win
                }
                named_sync(1, 128);
                mbar_wait(&tfull[acc], aphase);
                fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(taddr + c * 32, v);
#pragma unroll
                    for (int k4 = 0; k4 < 8; ++k4) {
                        const float4 y4 = *reinterpret_cast<const float4 *>(yb + c * 32 + 4 * k4);
                        const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int k = 4 * k4 + e;
                            const float dt = fmaf(-2.0f, __uint_as_float(v[k]), xn + yv[e]);
                            if (dt < lim) {
                                cbd[nc * 128] = dt;
                                cbj[nc * 128] = t * BN + c * 32 + k;
                                ++nc;
                            }
                        }
                        if (nc > CB - 4) {                // room for the next 4 values
                            for (int m = 0; m < nc; ++m) {
                                const float dd = cbd[m * 128];
                                if (dd < kth) kp_insert<KP>(bd, bj, dd, cbj[m * 128], kth);
                            }
                            nc = 0;
                            lim = fminf(kth, thr);
                        }
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
                for (int m = 0; m < nc; ++m) {
                    const float dd = cbd[m * 128];
                    if (dd < kth) kp_insert<KP>(bd, bj, dd, cbj[m * 128], kth);
                }
                nc = 0;
                if (i < p.M) thr = fminf(thr, __uint_as_float(atomicAdd(p.row_thr + i, 0u)));
                lim = fminf(kth, thr);
            }
            if (i < p.M && bj[KP - 1] >= 0)
                atomicMin(p.row_thr + i, __float_as_uint(fmaxf(bd[KP - 1], 0.0f)));
            if (i < p.M) {
                float *od = p.pd + ((int64_t)g * p.M + i) * KP;
                int32_t *oj = p.pj + ((int64_t)g * p.M + i) * KP;
#pragma unroll
                for (int k = 0; k < KP; ++k) { od[k] = bd[k]; oj[k] = bj[k]; }
            }
        }
    }
    __syncthreads();
    if (CL > 1) cluster_sync_all();                      // no multicast may still target this CTA
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

// ---- a10: tf32 hi/lo split + fp64 squared norms --------------------------------------------------
__device__ __forceinline__ float rna_tf32(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// Also does the call's initialisation (folded in to spare stream operations): with `init` (the
// x call, which runs first) it sets every row threshold to 3.4e38 and zeroes the max-norm word
// and the fallback counters that the later kernels of this call accumulate into.
struct SplitInit {
    unsigned int *row_thr; int64_t M;           // per-row K'-th-best thresholds -> 0x7f7f7f7f
    unsigned int *maxnorm; int *fb_count;        // -> 0
    unsigned int *fb_done; int fb_cap;           // -> 0
};

__global__ void split_kernel(const float *__restrict__ src, int64_t rows, int D, int Dp,
                             float *__restrict__ hi, float *__restrict__ lo, float *__restrict__ nrm,
                             unsigned int *maxnorm_bits, SplitInit init) {
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    if (init.row_thr) {
        for (int64_t k = gt; k < init.M; k += gs) init.row_thr[k] = 0x7f7f7f7fu;
        if (gt == 0) { *init.maxnorm = 0u; *init.fb_count = 0; }
        for (int64_t k = gt; k < init.fb_cap; k += gs) init.fb_done[k] = 0u;
    }
    // one warp per row; float4 loads and stores when rows are 16-byte multiples (D % 4 == 0)
    const int64_t w = gt >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nw = gs >> 5;
    const bool vec = (D & 3) == 0 && (((uintptr_t)src) & 15) == 0;
    float wmax = 0.0f;                                  // this warp's largest |row| (lane 0)
    for (int64_t i = w; i < rows; i += nw) {
        double s = 0.0;
        if (vec) {
            // all of a lane's float4 of the row (up to 7 x 32: D <= 896 in one pass) are loaded
            // before any is converted: ~3.5 KB per warp in flight instead of 512 B
            constexpr int U = 7;
            const float4 *s4 = reinterpret_cast<const float4 *>(src + i * D);
            float4 *h4 = reinterpret_cast<float4 *>(hi + i * Dp);
            float4 *l4 = reinterpret_cast<float4 *>(lo + i * Dp);
            for (int base = 0; base < Dp / 4; base += 32 * U) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = base + lane + 32 * u;
                    v[u] = k < D / 4 ? __ldg(s4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = base + lane + 32 * u;
                    if (k >= Dp / 4) break;
                    float4 h, l;
                    h.x = rna_tf32(v[u].x); h.y = rna_tf32(v[u].y); h.z = rna_tf32(v[u].z); h.w = rna_tf32(v[u].w);
                    l.x = rna_tf32(v[u].x - h.x); l.y = rna_tf32(v[u].y - h.y);
                    l.z = rna_tf32(v[u].z - h.z); l.w = rna_tf32(v[u].w - h.w);
                    h4[k] = h;
                    l4[k] = l;
                    s += (double)v[u].x * (double)v[u].x + (double)v[u].y * (double)v[u].y +
                         (double)v[u].z * (double)v[u].z + (double)v[u].w * (double)v[u].w;
                }
            }
        } else {
            for (int k = lane; k < Dp; k += 32) {
                const float v = k < D ? src[i * D + k] : 0.0f;
                const float h = rna_tf32(v);
                const float l = rna_tf32(v - h);
                hi[i * Dp + k] = h;
                lo[i * Dp + k] = l;
                s += (double)v * (double)v;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            nrm[i] = (float)s;
            wmax = fmaxf(wmax, (float)sqrt(s) * 1.0000002f);
        }
    }
    // one atomicMax per CTA (not per row: same-address atomics serialise in L2)
    if (maxnorm_bits) {
        __shared__ float smax[32];
        if (lane == 0) smax[threadIdx.x >> 5] = wmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = 0.0f;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmaxf(m, smax[k]);
            atomicMax(maxnorm_bits, __float_as_uint(m));
        }
    }
}

// ---- a12: merge group lists -> K' best screened, exact fp64 re-rank, margin certificate --------
template <int KP>
__global__ void rerank_kernel(const float *__restrict__ pd, const int32_t *__restrict__ pj,
                              int n_groups, const float *__restrict__ x, const float *__restrict__ y,
                              const float *__restrict__ xn, const unsigned int *maxnorm_bits,
                              int64_t M, int64_t N, int D, int K, float *dist, int64_t *idx,
                              int64_t j_offset, int *fb_count, int32_t *fb_rows) {
    __shared__ float s_d[4][KP];
    __shared__ int32_t s_j[4][KP];
    __shared__ double s_e[4][KP];
    const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * 4 + wl;
    if (i >= M) return;
    // (1) each lane merges the group lists g = lane, lane + 32, ... into a sorted register list
    float bd[KP];
    int32_t bj[KP];
    float kth = INFINITY;
#pragma unroll
    for (int k = 0; k < KP; ++k) { bd[k] = INFINITY; bj[k] = -1; }
    if (n_groups <= 32) {
        // one group per lane: the main kernel leaves each group's list sorted by (d, j) (kp_insert
        // order), so the lane takes it as is -- no insertion
        if (lane < n_groups) {
            const float4 *gd4 = reinterpret_cast<const float4 *>(pd + ((int64_t)lane * M + i) * KP);
            const int4 *gj4 = reinterpret_cast<const int4 *>(pj + ((int64_t)lane * M + i) * KP);
#pragma unroll
            for (int q = 0; q < KP / 4; ++q) {
                const float4 dv = gd4[q];
                const int4 jv = gj4[q];
                bd[4 * q] = dv.x; bd[4 * q + 1] = dv.y; bd[4 * q + 2] = dv.z; bd[4 * q + 3] = dv.w;
                bj[4 * q] = jv.x; bj[4 * q + 1] = jv.y; bj[4 * q + 2] = jv.z; bj[4 * q + 3] = jv.w;
            }
#pragma unroll
            for (int k = 0; k < KP; ++k)
                if (bj[k] < 0) bd[k] = INFINITY;
        }
    }
    for (int g = lane; n_groups > 32 && g < n_groups; g += 32) {
        const float *gd = pd + ((int64_t)g * M + i) * KP;
        const int32_t *gj = pj + ((int64_t)g * M + i) * KP;
        for (int k = 0; k < KP; ++k) {
            const int32_t j = gj[k];
            if (j < 0) break;
            const float d = gd[k];
            if (!(d < kth || (d == kth && (uint32_t)j < (uint32_t)bj[KP - 1]))) break;   // sorted
            kp_insert<KP>(bd, bj, d, j, kth);
        }
    }
    // (2) warp-wide K'-way merge of the 32 lane lists: K' rounds of a lexicographic (d, j)
    //     argmin over the lanes' heads; the winning lane pops its head
    {
        int head = 0;
        for (int k = 0; k < KP; ++k) {
            float hd = INFINITY;
            int32_t hj = -1;
#pragma unroll
            for (int q = 0; q < KP; ++q)
                if (q == head) { hd = bd[q]; hj = bj[q]; }
            if (hj < 0) hd = INFINITY;
            float wd = hd;
            int32_t wj = hj < 0 ? INT32_MAX : hj;
            int wl_ = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float od = __shfl_xor_sync(0xffffffffu, wd, o);
                const int32_t oj = __shfl_xor_sync(0xffffffffu, wj, o);
                const int ol = __shfl_xor_sync(0xffffffffu, wl_, o);
                if (od < wd || (od == wd && oj < wj)) { wd = od; wj = oj; wl_ = ol; }
            }
            if (lane == wl_) ++head;
            if (lane == 0) {
                s_d[wl][k] = wd;
                s_j[wl][k] = wj == INT32_MAX ? -1 : wj;
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < KP; ++k) { bd[k] = s_d[wl][k]; bj[k] = s_j[wl][k]; }
        // margin certificate (R17): every true top-K member is among the K' screened candidates
        // when d~_(K') - d~_(K) > 2 delta, delta = gamma |x| max|y| + 2^-22 (|x|^2 + max|y|^2)
        const float ymax = __uint_as_float(*maxnorm_bits);
        const double xnorm = sqrt((double)xn[i]);
        const double gamma = 3.0 * D * ldexp(1.0, -23);
        const double delta = gamma * xnorm * ymax + ldexp(1.0, -22) * ((double)xn[i] + (double)ymax * ymax);
        const bool all_in = bj[KP - 1] < 0;                 // fewer than K' refs exist at all
        if (!all_in && !((double)bd[KP - 1] - (double)bd[K - 1] > 2.0 * delta)) {
            const int slot = atomicAdd(fb_count, 1);
            fb_rows[slot] = (int32_t)i;
        }
    }
    __syncwarp();
    // exact fp64 distances (direct differences, never expanded) of the candidates that can still
    // be in the top K: d~_(k) <= d~_(K) + 2 delta (a candidate above that has a true distance >
    // d~_(K) + delta >= the true distance of each of the K best screened ones, so it cannot be
    // among the K nearest); all candidates' y rows are read together (one load of x, up to K'
    // independent loads of y per step: the rows are scattered, so memory-level parallelism, not
    // arithmetic, sets this kernel's time)
    {
        const float ymax = __uint_as_float(*maxnorm_bits);
        const double xnorm = sqrt((double)xn[i]);
        const double delta = 3.0 * D * ldexp(1.0, -23) * xnorm * ymax +
                             ldexp(1.0, -22) * ((double)xn[i] + (double)ymax * ymax);
        const double dK = (double)s_d[wl][K - 1];
        int32_t jj[KP];
        bool use[KP];
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            jj[k] = s_j[wl][k];
            use[k] = jj[k] >= 0 && (k < K || (double)s_d[wl][k] <= dK + 2.0 * delta);
        }
        constexpr int CV = 7;                          // float4 per lane per row: D <= 896 in one pass
        if ((D & 3) == 0 && D / 4 <= 32 * CV && ((((uintptr_t)x) | ((uintptr_t)y)) & 15) == 0) {
            // candidate-major: a lane's CV float4 of one candidate row are requested together (one
            // memory latency per candidate instead of one per float4: the scattered y rows made
            // this kernel latency-bound)
            const float4 *x4 = reinterpret_cast<const float4 *>(x + i * D);
            float4 xv[CV];
#pragma unroll
            for (int u = 0; u < CV; ++u) {
                const int c = lane + 32 * u;
                xv[u] = c < D / 4 ? __ldg(x4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int k = 0; k < KP; ++k) {
                if (!use[k]) {                             // warp-uniform
                    if (lane == 0) s_e[wl][k] = INFINITY;
                    continue;
                }
                const float4 *y4 = reinterpret_cast<const float4 *>(y + (int64_t)jj[k] * D);
                float4 yv[CV];
#pragma unroll
                for (int u = 0; u < CV; ++u) {
                    const int c = lane + 32 * u;
                    yv[u] = c < D / 4 ? __ldg(y4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                double v = 0.0;
#pragma unroll
                for (int u = 0; u < CV; ++u) {
                    const double d0 = (double)xv[u].x - (double)yv[u].x, d1 = (double)xv[u].y - (double)yv[u].y;
                    const double d2 = (double)xv[u].z - (double)yv[u].z, d3 = (double)xv[u].w - (double)yv[u].w;
                    v = fma(d3, d3, fma(d2, d2, fma(d1, d1, fma(d0, d0, v))));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) s_e[wl][k] = v;
            }
        } else {
            double acc[KP];
#pragma unroll
            for (int k = 0; k < KP; ++k) acc[k] = 0.0;
            for (int c = lane; c < D; c += 32) {
                const double xs = (double)x[i * D + c];
#pragma unroll
                for (int k = 0; k < KP; ++k) {
                    if (!use[k]) continue;
                    const double dv = xs - (double)y[(int64_t)jj[k] * D + c];
                    acc[k] = fma(dv, dv, acc[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                double v = acc[k];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) s_e[wl][k] = use[k] ? v : INFINITY;
            }
        }
    }
    __syncwarp();
    // emit the K best by (exact d, j): lane k < K' computes candidate k's rank (the number of
    // candidates before it in that order; (d, j) pairs are distinct) and writes it to slot rank
    // if rank < K -- all lanes at once instead of a serial sort on lane 0; unused slots (fewer
    // than K candidates) get the (+inf, -1) padding
    {
        const double myd = lane < KP ? s_e[wl][lane] : INFINITY;
        const int32_t myj = lane < KP ? s_j[wl][lane] : -1;
        const uint32_t myju = (uint32_t)myj;                  // -1 (no candidate) sorts last
        int rank = 0;
        bool valid = lane < KP && myj >= 0 && myd < INFINITY;
        if (valid) {
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const double od = s_e[wl][k];
                const uint32_t oj = (uint32_t)s_j[wl][k];
                if (s_j[wl][k] >= 0 && (od < myd || (od == myd && oj < myju))) ++rank;
            }
        }
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        const int nvalid = __popc(vmask);
        if (valid && rank < K) {
            dist[i * K + rank] = (float)myd;
            idx[i * K + rank] = (int64_t)myj + j_offset;
        }
        for (int k = nvalid + lane; k < K; k += 32) {
            dist[i * K + k] = INFINITY;
            idx[i * K + k] = -1;
        }
    }
}

// ---- exact fp64 rescan of rows whose screening was not certified ---------------------------------
// Rare (rows failing the R17 certificate) but a full scan of N refs x D per row: every CTA of the
// grid takes one chunk of the refs of each flagged row (warps over refs, lanes over D, fp64
// direct differences), writes its sorted partial list, and the last CTA to finish a row merges
// the G lists (threadfence + counter).  Rows beyond FB_CAP fall back to a single-CTA scan.
constexpr int FB_THREADS = 256;
constexpr int FB_WARPS = FB_THREADS / 32;
constexpr int FB_LIST = 32;              // >= K
constexpr int FB_ILP = 4;                // refs per warp iteration
constexpr int FB_CAP = 64;               // rows handled grid-wide
constexpr int FB_GRID = 296;

__device__ void fb_scan_chunk(const float *__restrict__ x, const float *__restrict__ y, int64_t i,
                              int64_t jlo, int64_t jhi, int D, double (*sd)[FB_LIST],
                              int32_t (*sj)[FB_LIST]) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int k = 0; k < FB_LIST; ++k) { sd[w][k] = INFINITY; sj[w][k] = -1; }
    __syncwarp();
    for (int64_t j0 = jlo + (int64_t)w * FB_ILP; j0 < jhi; j0 += (int64_t)FB_WARPS * FB_ILP) {
        double s[FB_ILP];
#pragma unroll
        for (int u = 0; u < FB_ILP; ++u) s[u] = 0.0;
        for (int c = lane; c < D; c += 32) {
            const double xv = (double)x[i * D + c];
#pragma unroll
            for (int u = 0; u < FB_ILP; ++u) {
                if (j0 + u < jhi) {
                    const double dv = xv - (double)y[(j0 + u) * D + c];
                    s[u] = fma(dv, dv, s[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < FB_ILP; ++u) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
        }
        if (lane == 0) {
#pragma unroll
            for (int u = 0; u < FB_ILP; ++u) {                      // j ascending within the warp
                if (j0 + u < jhi && s[u] < sd[w][FB_LIST - 1]) {
                    int pos = FB_LIST - 1;
                    while (pos > 0 && s[u] < sd[w][pos - 1]) {
                        sd[w][pos] = sd[w][pos - 1]; sj[w][pos] = sj[w][pos - 1]; --pos;
                    }
                    sd[w][pos] = s[u]; sj[w][pos] = (int32_t)(j0 + u);
                }
            }
        }
    }
    __syncthreads();
}

// Merge `nl` sorted (d, j) lists (stride `ld` apart) into the first `K` of (od, oj).
__device__ void fb_merge(const double *ld_d, const int32_t *ld_j, int nl, int ld, int K,
                         double *od, int32_t *oj) {
    int head[FB_GRID > FB_WARPS ? FB_GRID : FB_WARPS];
    for (int q = 0; q < nl; ++q) head[q] = 0;
    for (int k = 0; k < K; ++k) {
        int best = -1;
        for (int q = 0; q < nl; ++q) {
            if (head[q] >= FB_LIST) continue;
            const int32_t j = ld_j[q * ld + head[q]];
            if (j < 0) continue;
            const double d = ld_d[q * ld + head[q]];
            if (best < 0 || d < ld_d[best * ld + head[best]] ||
                (d == ld_d[best * ld + head[best]] && j < ld_j[best * ld + head[best]]))
                best = q;
        }
        if (best >= 0) {
            od[k] = ld_d[best * ld + head[best]];
            oj[k] = ld_j[best * ld + head[best]];
            head[best]++;
        } else {
            od[k] = INFINITY;
            oj[k] = -1;
        }
    }
}

__global__ void __launch_bounds__(FB_THREADS)
fallback_kernel(const float *__restrict__ x, const float *__restrict__ y, int64_t N, int D, int K,
                const int *fb_count, const int32_t *fb_rows, double *part_d, int32_t *part_j,
                unsigned int *done, float *dist, int64_t *idx, int64_t j_offset) {
    __shared__ double sd[FB_WARPS][FB_LIST];
    __shared__ int32_t sj[FB_WARPS][FB_LIST];
    __shared__ int is_last;
    const int n = *fb_count;
    const int ncap = n < FB_CAP ? n : FB_CAP;
    const int G = gridDim.x;
    // grid-wide rows
    for (int f = 0; f < ncap; ++f) {
        const int64_t i = fb_rows[f];
        const int64_t jlo = N * blockIdx.x / G, jhi = N * (blockIdx.x + 1) / G;
        fb_scan_chunk(x, y, i, jlo, jhi, D, sd, sj);
        if (threadIdx.x == 0) {
            double md[FB_LIST];
            int32_t mj[FB_LIST];
            fb_merge(&sd[0][0], &sj[0][0], FB_WARPS, FB_LIST, FB_LIST, md, mj);
            double *pd = part_d + ((int64_t)f * G + blockIdx.x) * FB_LIST;
            int32_t *pj = part_j + ((int64_t)f * G + blockIdx.x) * FB_LIST;
            for (int k = 0; k < FB_LIST; ++k) { pd[k] = md[k]; pj[k] = mj[k]; }
            __threadfence();
            is_last = atomicAdd(done + f, 1u) == (unsigned)(G - 1);
        }
        __syncthreads();
        if (is_last) {
            // block-parallel K-way merge of the G partial lists: thread t owns lists t, t + 256,
            // ...; K rounds of a block-wide lexicographic (d, j) argmin over the list heads
            __threadfence();
            __shared__ double rd[FB_WARPS];
            __shared__ int32_t rj[FB_WARPS];
            __shared__ int rq[FB_WARPS];
            const double *LD = part_d + (int64_t)f * G * FB_LIST;
            const int32_t *LJ = part_j + (int64_t)f * G * FB_LIST;
            int heads[(FB_GRID + FB_THREADS - 1) / FB_THREADS];
            for (int u = 0; u * FB_THREADS + (int)threadIdx.x < G; ++u) heads[u] = 0;
            const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
            for (int k = 0; k < K; ++k) {
                double bd = INFINITY;
                int32_t bj = INT32_MAX;
                int bq = -1;
                for (int u = 0; u * FB_THREADS + (int)threadIdx.x < G; ++u) {
                    const int q = u * FB_THREADS + threadIdx.x;
                    if (heads[u] >= FB_LIST) continue;
                    const int32_t j = LJ[q * FB_LIST + heads[u]];
                    if (j < 0) continue;
                    const double d = LD[q * FB_LIST + heads[u]];
                    if (d < bd || (d == bd && j < bj)) { bd = d; bj = j; bq = q; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
                    const int32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
                    const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
                    if (od < bd || (od == bd && oj < bj)) { bd = od; bj = oj; bq = oq; }
                }
                if (lane == 0) { rd[w] = bd; rj[w] = bj; rq[w] = bq; }
                __syncthreads();
                if (threadIdx.x == 0) {
                    for (int q = 1; q < FB_WARPS; ++q)
                        if (rd[q] < rd[0] || (rd[q] == rd[0] && rj[q] < rj[0])) { rd[0] = rd[q]; rj[0] = rj[q]; rq[0] = rq[q]; }
                    const bool ok = rq[0] >= 0;
                    dist[i * K + k] = ok ? (float)rd[0] : INFINITY;
                    idx[i * K + k] = ok ? (int64_t)rj[0] + j_offset : -1;
                }
                __syncthreads();
                const int win = rq[0];
                if (win >= 0 && win % FB_THREADS == (int)threadIdx.x) heads[win / FB_THREADS]++;
                __syncthreads();
            }
        }
        __syncthreads();
    }
    // rows beyond the cap: one CTA per row
    for (int f = FB_CAP + blockIdx.x; f < n; f += G) {
        const int64_t i = fb_rows[f];
        fb_scan_chunk(x, y, i, 0, N, D, sd, sj);
        if (threadIdx.x == 0) {
            double md[FB_LIST];
            int32_t mj[FB_LIST];
            fb_merge(&sd[0][0], &sj[0][0], FB_WARPS, FB_LIST, K, md, mj);
            for (int k = 0; k < K; ++k) {
                dist[i * K + k] = mj[k] >= 0 ? (float)md[k] : INFINITY;
                idx[i * K + k] = mj[k] >= 0 ? (int64_t)mj[k] + j_offset : -1;
            }
        }
        __syncthreads();
    }
}

}  // namespace tc

// ---------------------------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------------------------
#include <cudaTypedefs.h>

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static cudaError_t get_encoder() {
    if (g_encode) return cudaSuccess;
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    return cudaSuccess;
}

static cudaError_t make_map(CUtensorMap *m, const float *ptr, int64_t rows, int Dp, int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)Dp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)Dp * 4};
    cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)ptr, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int knn_tc_group() { return 8; }

size_t knn_tc_scratch_bytes(int64_t M, int64_t N, int D, int K) {
    const int Dp = (D + tc::BK - 1) / tc::BK * tc::BK;
    const int KP = K <= 12 ? 16 : 32;
    const int n_ttiles = (int)((N + tc::BN - 1) / tc::BN);
    const int n_groups = (n_ttiles + knn_tc_group() - 1) / knn_tc_group();
    auto al = [](size_t v) { return (v + 1023) & ~size_t(1023); };
    return al((size_t)M * Dp * 4) * 2 + al((size_t)N * Dp * 4) * 2 + al((size_t)M * 4) +
           al((size_t)N * 4) + al(64) + al((size_t)n_groups * M * KP * 4) * 2 + al((size_t)M * 4) * 2 + al(64) +
           al((size_t)tc::FB_CAP * tc::FB_GRID * tc::FB_LIST * 12) + al((size_t)tc::FB_CAP * 4) + 2048;
}

template <int KP, int CL>
static cudaError_t launch_main(const CUtensorMap *maps, const tc::Params &p, int grid, cudaStream_t st) {
    auto kern = tc::knn_tc_kernel<KP, CL>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, tc::SMEM_BYTES);
        if (e != cudaSuccess) return e;
    }
    if (CL == 1) {                                        // plain launch (no cluster scheduling)
        kern<<<grid, tc::NUM_THREADS, tc::SMEM_BYTES, st>>>(maps[0], maps[1], maps[2], maps[3], p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::NUM_THREADS);
    cfg.dynamicSmemBytes = tc::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = CL;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], p);
}

cudaError_t launch_knn_tc(const KnnTcLaunch &a, cudaStream_t st, KnnTcInfo *info) {
    cudaError_t e = get_encoder();
    if (e != cudaSuccess) return e;
    const int64_t M = a.M, N = a.N;
    const int D = a.D, K = a.K;
    const int Dp = (D + tc::BK - 1) / tc::BK * tc::BK;
    const int KP = K <= 12 ? 16 : 32;
    const int n_rtiles = (int)((M + tc::BM - 1) / tc::BM);
    const int n_ttiles = (int)((N + tc::BN - 1) / tc::BN);
    const int group = knn_tc_group();
    const int n_groups = (n_ttiles + group - 1) / group;
    auto al = [](size_t v) { return (v + 1023) & ~size_t(1023); };
    char *s = (char *)a.scratch;
    float *xhi = (float *)s; s += al((size_t)M * Dp * 4);
    float *xlo = (float *)s; s += al((size_t)M * Dp * 4);
    float *yhi = (float *)s; s += al((size_t)N * Dp * 4);
    float *ylo = (float *)s; s += al((size_t)N * Dp * 4);
    float *xn = (float *)s; s += al((size_t)M * 4);
    float *yn = (float *)s; s += al((size_t)N * 4);
    unsigned int *ymax = (unsigned int *)s; s += al(64);
    float *pd = (float *)s; s += al((size_t)n_groups * M * KP * 4);
    unsigned int *row_thr = (unsigned int *)s; s += al((size_t)M * 4);
    int32_t *pj = (int32_t *)s; s += al((size_t)n_groups * M * KP * 4);
    int32_t *fb_rows = (int32_t *)s; s += al((size_t)M * 4);
    double *fb_pd = (double *)s; s += al((size_t)tc::FB_CAP * tc::FB_GRID * tc::FB_LIST * 8);
    int32_t *fb_pj = (int32_t *)s; s += al((size_t)tc::FB_CAP * tc::FB_GRID * tc::FB_LIST * 4);
    unsigned int *fb_done = (unsigned int *)s; s += al((size_t)tc::FB_CAP * 4);
    int *fb_count = (int *)s;

    int kernels = 0;
    // the x split also initialises row_thr, ymax, fb_count and fb_done (no memset launches)
    tc::SplitInit ini{row_thr, M, ymax, fb_count, fb_done, tc::FB_CAP};
    tc::split_kernel<<<(unsigned)std::min<int64_t>((M + 7) / 8, 148 * 16), 256, 0, st>>>(a.x, M, D, Dp, xhi, xlo, xn, nullptr, ini);
    tc::split_kernel<<<(unsigned)std::min<int64_t>((N + 7) / 8, 148 * 16), 256, 0, st>>>(a.y, N, D, Dp, yhi, ylo, yn, ymax, tc::SplitInit{});
    kernels += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;

    CUtensorMap maps[4];
    if ((e = make_map(&maps[0], xhi, M, Dp, tc::BM)) != cudaSuccess) return e;
    if ((e = make_map(&maps[1], xlo, M, Dp, tc::BM)) != cudaSuccess) return e;
    const int CL = tc::CLUSTER;                          // B box = the CTA's share of the ref tile
    if ((e = make_map(&maps[2], yhi, N, Dp, tc::BN / CL)) != cudaSuccess) return e;
    if ((e = make_map(&maps[3], ylo, N, Dp, tc::BN / CL)) != cudaSuccess) return e;
    tc::Params p;
    p.M = M; p.N = N; p.Dp = Dp; p.nk = Dp / tc::BK; p.n_rtiles = n_rtiles; p.n_ttiles = n_ttiles;
    p.n_groups = n_groups; p.group = group; p.xn = xn; p.yn = yn; p.pd = pd; p.pj = pj;
    p.row_thr = row_thr;
    const int n_units = n_groups * ((n_rtiles + CL - 1) / CL);
    const int grid = std::min(n_units, a.num_sms / CL) * CL;
    if (a.ev_start) cudaEventRecord(a.ev_start, st);
    e = KP == 16 ? launch_main<16, tc::CLUSTER>(maps, p, grid, st) : launch_main<32, tc::CLUSTER>(maps, p, grid, st);
    if (a.ev_stop) cudaEventRecord(a.ev_stop, st);
    if (e != cudaSuccess) return e;
    kernels += 1;
    const unsigned rgrid = (unsigned)((M + 3) / 4);
    if (KP == 16)
        tc::rerank_kernel<16><<<rgrid, 128, 0, st>>>(pd, pj, n_groups, a.x, a.y, xn, ymax, M, N, D, K,
                                                     a.dist, a.idx, a.j_offset, fb_count, fb_rows);
    else
        tc::rerank_kernel<32><<<rgrid, 128, 0, st>>>(pd, pj, n_groups, a.x, a.y, xn, ymax, M, N, D, K,
                                                     a.dist, a.idx, a.j_offset, fb_count, fb_rows);
    tc::fallback_kernel<<<tc::FB_GRID, tc::FB_THREADS, 0, st>>>(a.x, a.y, N, D, K, fb_count, fb_rows,
                                                                fb_pd, fb_pj, fb_done, a.dist, a.idx,
                                                                a.j_offset);
    kernels += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (info) {
        info->kernels = kernels;
        info->ctas = grid;
        info->fallback_count = fb_count;
    }
    return cudaSuccess;
}

}  // namespace genred
