// gauss_tc.cu -- the Gaussian Genred Sum with its exponent contraction on the tensor cores
// (Eq. 1: a_i = sum_j exp(-|x_i - y_j|^2/s^2) b_j).
//
// In the expanded form of the FP32 kernel (sum_kernel.cu, reading R18b),
//
//   exp(-|x_i - y_j|^2 / sigma^2) = 2^(-|x'_i|^2) * 2^(u_ij),   u_ij = 2 x'_i . y'_j - |y'_j|^2,
//   x' = s (x - c), y' = s (y - c), s = sqrt(log2 e) / sigma, c = centre of y's bounding box,
//
// u is a rank-(D+1) contraction U = A B^T with A_i = (2x'_i, 1) and B_j = (y'_j, -|y'_j|^2).  On
// the FP32 pipe it costs D+1 FMAs per pair (half of the pipe's time at D = 3); here the tensor
// cores produce it instead (tcgen05.mma kind::tf32, 3xTF32 split for fp32 accuracy), so the
// CUDA cores only do the exponential and the b-weighted accumulation, and the exponentials can
// be shared between the MUFU pipe (16 ex2/clk/SM) and a polynomial on the FP32 pipe:
//
//   a  prepass: A rows (tf32 hi / lo of 2x', 1) and B rows (tf32 hi / lo of y', w = -|y'|^2),
//      32 bytes each (K = 8), b padded to whole 256-j tiles;
//   b  per 128-row tile x 256-j tile: two MMAs (A_lo.B + A_hi.B with B = [hi | lo] along K, i.e.
//      A_lo B_hi + A_hi B_hi + A_hi B_lo) into one of two 256-column fp32 TMEM accumulators,
//      operands staged by TMA (32B swizzle) into a shared-memory ring;
//   c  epilogue warps read U with tcgen05.ld (one TMEM lane = one row), evaluate 2^u (MUFU.EX2,
//      or a degree-5 polynomial on the FP32 pipe for NPOLY of every 16 values), accumulate
//      2^u b_j in fp32 per tile, promote to fp64 per tile, and apply the row factor 2^(-|x'|^2)
//      in fp64 (the same epilogue as the FP32 kernel's expanded path).
//
// The path exists only under the expanded-form condition (box radius^2 <= 6, geo.cuh, decided on
// the device from the same encoded box); otherwise the kernel exits at once and the direct FP32
// kernel launched behind it does the work.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "device.cuh"
#include "geo.cuh"
#include "internal.h"

namespace genred {
namespace gtc {

constexpr int BM = 128;                 // rows per tile = TMEM lanes
constexpr int BN = 256;                 // j per tile = TMEM columns per accumulator
constexpr int KW = 8;                   // floats per operand row (K = 8 tf32 = 32 B)
constexpr int STAGES = 6;
#ifndef GENRED_TC_EW
#define GENRED_TC_EW 16
#endif
constexpr int EW = GENRED_TC_EW;        // epilogue warps (multiple of 4: each lane quarter EW/4 times)
constexpr int NT = 64 + EW * 32;        // warp 0 TMA, warp 1 MMA + TMEM alloc, then epilogue
constexpr int CG = EW / 4;              // column groups per tile
constexpr int COLS = BN / CG;           // columns per epilogue thread per tile
#ifndef GENRED_TC_ILV
#define GENRED_TC_ILV 0
#endif
#ifndef GENRED_TC_LD2
#define GENRED_TC_LD2 0
#endif
#ifndef GENRED_TC_POLY
#define GENRED_TC_POLY 6
#endif
constexpr int NPOLY = GENRED_TC_POLY;   // of every 16 exponentials, NPOLY on the FP32 pipe (even)
static_assert(NPOLY % 2 == 0 && NPOLY <= 16, "NPOLY: even, <= 16");
static_assert(COLS % 32 == 0, "COLS: whole 32-column TMEM loads");

constexpr int A_BYTES = BM * KW * 4;    // 4 KB
constexpr int B_BYTES = BN * KW * 4;    // 8 KB
constexpr int BV_BYTES = BN * 4;        // 1 KB of b
constexpr int STAGE_BYTES = B_BYTES + BV_BYTES;
constexpr int SMEM_BYTES = 1024 + 2 * A_BYTES + STAGES * STAGE_BYTES + CG * BM * 8 + 256;
static_assert(STAGE_BYTES % 1024 == 0, "stages keep 1024-byte alignment");

__device__ __forceinline__ void tma_load_2d(void *smem, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(smem)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand with 32-byte rows, 32B swizzle: 8-row atoms of 256 B (SBO), version 1.
__device__ __forceinline__ uint64_t desc32(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
    d |= (uint64_t)(256 >> 4) << 32;         // SBO
    d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
    d |= (uint64_t)6 << 61;                  // SWIZZLE_32B
    return d;
}

// kind::tf32: D f32, A/B tf32, both K-major, N = 256, M = 128.
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
// Load without waiting; tmem_wait32 completes every outstanding load and pins the registers of
// v after it (so the compiler cannot read them before the wait).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
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
}
__device__ __forceinline__ void tmem_wait32(uint32_t (&v)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
          "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]),
          "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]),
          "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]),
          "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
        :: "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float rna_tf32(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

struct Params {
    int64_t M, Mpad;
    int n_rtiles, n_ttiles, tiles_per_split, n_units;
    const float *x;
    const uint32_t *geo;
    float s;
    double scale_sum;
    void *out;
    int out_f64;
    int split;
    double *part;            // split > 1: split x M fp64 partials (sum_finalize layout, C = 1)
};

__device__ __forceinline__ float4 lds128s(uint32_t addr) {     // LDS.128 (broadcast: one address per warp)
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// 32 values of one TMEM row segment: s += 2^u b over the row's four fp32 partial sums.
__device__ __forceinline__ void accumulate32(const uint32_t (&v)[32], uint32_t bv, float (&acc)[4]) {
#pragma unroll
    for (int k4 = 0; k4 < 8; ++k4) {
        const float4 b4 = lds128s(bv + 16 * k4);
        float e[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = 4 * k4 + 2 * h;
            // ILV: the polynomial pairs interleaved with the MUFU pairs (pairs 0, 2, 4, ... of
            // every 8), else the first NPOLY values of every 16
            const bool poly = GENRED_TC_ILV ? (((k / 2) % 8) % 2 == 0 && ((k / 2) % 8) / 2 < NPOLY / 2)
                                            : ((k % 16) < NPOLY);
            if (poly) {
                const float2 r = ex2_poly2(make_float2(__uint_as_float(v[k]), __uint_as_float(v[k + 1])));
                e[2 * h] = r.x;
                e[2 * h + 1] = r.y;
            } else {
                e[2 * h] = ex2(__uint_as_float(v[k]));
                e[2 * h + 1] = ex2(__uint_as_float(v[k + 1]));
            }
        }
        acc[0] = fmaf(e[0], b4.x, acc[0]);
        acc[1] = fmaf(e[1], b4.y, acc[1]);
        acc[2] = fmaf(e[2], b4.z, acc[2]);
        acc[3] = fmaf(e[3], b4.w, acc[3]);
    }
}

template <int D>
__global__ void __launch_bounds__(NT, 1)
gauss_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const float *__restrict__ bvec, const Params p) {
    const Geo geo = geo_decode(p.geo, D, p.s);
    if (!geo.expanded) return;                           // the direct FP32 kernel takes this call
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *a_hi = base, *a_lo = base + A_BYTES;  // A tiles: (2x'_hi, 1 | same), (2x'_lo, 0 | 0)
    unsigned char *ring = base + 2 * A_BYTES;
    double *red = reinterpret_cast<double *>(ring + STAGES * STAGE_BYTES);     // [CG][BM]
    uint64_t *bars = reinterpret_cast<uint64_t *>(red + CG * BM);
    uint64_t *full = bars, *empty = bars + STAGES;
    uint64_t *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + 2;
    uint64_t *afull = bars + 2 * STAGES + 4, *aempty = bars + 2 * STAGES + 5;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 6);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + EW);                // MMA commit + every epilogue warp (b)
        }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], EW); }
        mbar_init(afull, 1);
        mbar_init(aempty, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     ::"r"(smem_u32(tmem_slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            int stage = 0; uint32_t phase = 0, uphase = 0;
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                const int sp = u / p.n_rtiles, r = u % p.n_rtiles;
                const int t0 = sp * p.tiles_per_split, t1 = min(t0 + p.tiles_per_split, p.n_ttiles);
                mbar_wait(aempty, uphase ^ 1);           // previous unit's MMAs are done with A
                uphase ^= 1;
                mbar_arrive_expect_tx(afull, 2 * A_BYTES);
                tma_load_2d(a_hi, &map_a, 0, r * BM, afull);
                tma_load_2d(a_lo, &map_a, 0, (int)(p.Mpad + (int64_t)r * BM), afull);
                for (int t = t0; t < t1; ++t) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char *sb = ring + stage * STAGE_BYTES;
                    mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                    tma_load_2d(sb, &map_b, 0, t * BN, &full[stage]);
                    bulk_g2s(sb + B_BYTES, bvec + (int64_t)t * BN, BV_BYTES, &full[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer (one thread) ------------------------------
        if (lane == 0) {
            int stage = 0; uint32_t phase = 0, uphase = 0;
            int acc = 0; uint32_t aphase = 0;
            const uint64_t dhi = desc32(smem_u32(a_hi)), dlo = desc32(smem_u32(a_lo));
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                const int sp = u / p.n_rtiles;
                const int t0 = sp * p.tiles_per_split, t1 = min(t0 + p.tiles_per_split, p.n_ttiles);
                mbar_wait(afull, uphase);
                uphase ^= 1;
                fence_after();
                for (int t = t0; t < t1; ++t) {
                    mbar_wait(&tempty[acc], aphase ^ 1);
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    const uint64_t db = desc32(smem_u32(ring + stage * STAGE_BYTES));
                    const uint32_t d_tmem = tmem_base + acc * BN;
                    mma_tf32(d_tmem, dlo, db, 0);        // A_lo . [B_hi | B_lo]  (second half 0)
                    mma_tf32(d_tmem, dhi, db, 1);        // + A_hi . [B_hi | B_lo]
                    mma_commit(&empty[stage]);
                    mma_commit(&tfull[acc]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    if (++acc == 2) { acc = 0; aphase ^= 1; }
                }
                mma_commit(aempty);
            }
        }
    } else {
        // ------------------------------ epilogue ------------------------------
        const int ew = warp - 2, q = warp & 3, cg = ew >> 2;
        const int row_in_tile = q * 32 + lane;
        int stage = 0; uint32_t phase = 0;
        int acc = 0; uint32_t aphase = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            const int sp = u / p.n_rtiles, r = u % p.n_rtiles;
            const int t0 = sp * p.tiles_per_split, t1 = min(t0 + p.tiles_per_split, p.n_ttiles);
            double a64 = 0.0;
            for (int t = t0; t < t1; ++t) {
                mbar_wait(&tfull[acc], aphase);
                mbar_wait(&full[stage], phase);          // b of this tile is visible
                fence_after();
                const uint32_t bv = smem_u32(ring + stage * STAGE_BYTES + B_BYTES) + cg * COLS * 4;
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + cg * COLS;
                float s4[4] = {0.f, 0.f, 0.f, 0.f};
                if constexpr (GENRED_TC_LD2) {
                    // two 32-column loads in flight, one wait: 64 independent values per batch
#pragma unroll
                    for (int c = 0; c < COLS / 32; c += 2) {
                        uint32_t v0[32], v1[32];
                        tmem_ld32_nowait(taddr + c * 32, v0);
                        tmem_ld32_nowait(taddr + c * 32 + 32, v1);
                        tmem_wait32(v0);
                        tmem_wait32(v1);
                        accumulate32(v0, bv + c * 128, s4);
                        accumulate32(v1, bv + c * 128 + 128, s4);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < COLS / 32; ++c) {
                        uint32_t v[32];
                        tmem_ld32(taddr + c * 32, v);
                        accumulate32(v, bv + c * 128, s4);
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&tempty[acc]);
                    mbar_arrive(&empty[stage]);
                }
                a64 += (double)(s4[0] + s4[1]) + (double)(s4[2] + s4[3]);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
            // fixed-order combine of the column groups, row factor 2^(-|x'|^2) in fp64
            red[cg * BM + row_in_tile] = a64;
            named_sync(1, EW * 32);
            if (cg == 0) {
                const int64_t i = (int64_t)r * BM + row_in_tile;
                if (i < p.M) {
                    double tot = red[row_in_tile];
#pragma unroll
                    for (int g = 1; g < CG; ++g) tot += red[g * BM + row_in_tile];
                    double xsq = 0.0;
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const float xs = p.s * (__ldg(p.x + i * D + d) - geo.c[d]);   // as the pack
                        xsq += (double)xs * (double)xs;
                    }
                    tot *= exp2(-xsq);
                    if (p.split > 1) p.part[(int64_t)sp * p.M + i] = tot;
                    else if (p.out_f64) ((double *)p.out)[i] = tot * p.scale_sum;
                    else ((float *)p.out)[i] = (float)(tot * p.scale_sum);
                }
            }
            named_sync(1, EW * 32);
        }
    }
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

// ---- prepass: operand rows (tf32 hi / lo), b padded ------------------------------------------
// A (2 Mpad rows of 8 floats): row i = (hi(2x'_0..D-1), 0.., 1 at [3]) twice; row Mpad + i =
// (lo(2x'_0..D-1), 0...).  B (Npad rows): (hi(y'_0..D-1), 0.., hi(w) at [3], lo(y'), lo(w)).
// Padded rows are zero (u = 0, b = 0: no contribution).
template <int D>
__global__ void gtc_pack_kernel(const float *__restrict__ x, const float *__restrict__ y,
                                const float *__restrict__ b, int64_t M, int64_t Mpad, int64_t N,
                                int64_t Npad, float s, const uint32_t *geo_enc, float *__restrict__ A,
                                float *__restrict__ B, float *__restrict__ bvec) {
    const Geo geo = geo_decode(geo_enc, D, s);
    if (!geo.expanded) return;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < Mpad + Npad;
         k += (int64_t)gridDim.x * blockDim.x) {
        float hi[4] = {0.f, 0.f, 0.f, 0.f}, lo[4] = {0.f, 0.f, 0.f, 0.f};
        if (k < Mpad) {
            const int64_t i = k;
            if (i < M) {
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const float xs2 = 2.0f * (s * (x[i * D + d] - geo.c[d]));   // 2x', exact doubling
                    hi[d] = rna_tf32(xs2);
                    lo[d] = rna_tf32(xs2 - hi[d]);
                }
                hi[3] = 1.0f;
            }
            float4 *ah = reinterpret_cast<float4 *>(A + i * KW);
            float4 *al = reinterpret_cast<float4 *>(A + (Mpad + i) * KW);
            const float4 h4 = make_float4(hi[0], hi[1], hi[2], hi[3]);
            ah[0] = h4; ah[1] = h4;
            al[0] = make_float4(lo[0], lo[1], lo[2], lo[3]); al[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            const int64_t j = k - Mpad;
            float bj = 0.0f;
            if (j < N) {
                double w = 0.0;
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const float ys = s * (y[j * D + d] - geo.c[d]);              // y' = s (y - c)
                    w += (double)ys * (double)ys;
                    hi[d] = rna_tf32(ys);
                    lo[d] = rna_tf32(ys - hi[d]);
                }
                const float wf = (float)(-w);
                hi[3] = rna_tf32(wf);
                lo[3] = rna_tf32((float)(-w - (double)hi[3]));
                bj = b ? b[j] : 1.0f;
            }
            float4 *bp = reinterpret_cast<float4 *>(B + j * KW);
            bp[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
            bp[1] = make_float4(lo[0], lo[1], lo[2], lo[3]);
            bvec[j] = bj;
        }
    }
}

}  // namespace gtc

// ---------------------------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode_gtc = nullptr;

static cudaError_t gtc_encoder() {
    if (g_encode_gtc) return cudaSuccess;
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    g_encode_gtc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    return cudaSuccess;
}

static cudaError_t gtc_map(CUtensorMap *m, const float *ptr, int64_t rows, int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)gtc::KW, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)gtc::KW * 4};
    cuuint32_t box[2] = {(cuuint32_t)gtc::KW, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode_gtc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)ptr, dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static size_t al1k(size_t v) { return (v + 1023) & ~size_t(1023); }

size_t gauss_tc_scratch_bytes(int64_t M, int64_t N) {
    const int64_t Mpad = (M + gtc::BM - 1) / gtc::BM * gtc::BM;
    const int64_t Npad = (N + 2 * gtc::BN - 1) / (2 * gtc::BN) * (2 * gtc::BN);
    return al1k((size_t)2 * Mpad * gtc::KW * 4) + al1k((size_t)Npad * gtc::KW * 4) +
           al1k((size_t)Npad * 4) + 1024;
}

int gauss_tc_rows_per_unit() { return gtc::BM; }

template <int D>
static cudaError_t gtc_run(const GaussTcLaunch &a, cudaStream_t st, int *ctas, int *kernels) {
    cudaError_t e = gtc_encoder();
    if (e != cudaSuccess) return e;
    const int64_t M = a.M, N = a.N;
    const int64_t Mpad = (M + gtc::BM - 1) / gtc::BM * gtc::BM;
    const int64_t Npad = (N + 2 * gtc::BN - 1) / (2 * gtc::BN) * (2 * gtc::BN);
    char *s = (char *)(((uintptr_t)a.scratch + 1023) & ~(uintptr_t)1023);
    float *A = (float *)s; s += al1k((size_t)2 * Mpad * gtc::KW * 4);
    float *B = (float *)s; s += al1k((size_t)Npad * gtc::KW * 4);
    float *bvec = (float *)s;
    const int64_t work = Mpad + Npad;
    const unsigned blocks = (unsigned)std::min<int64_t>((work + 255) / 256, (int64_t)a.num_sms * 16);
    gtc::gtc_pack_kernel<D><<<blocks, 256, 0, st>>>(a.x, a.y, a.b, M, Mpad, N, Npad, a.s, a.geo, A, B, bvec);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    CUtensorMap ma, mb;
    if ((e = gtc_map(&ma, A, 2 * Mpad, gtc::BM)) != cudaSuccess) return e;
    if ((e = gtc_map(&mb, B, Npad, gtc::BN)) != cudaSuccess) return e;
    gtc::Params p;
    p.M = M; p.Mpad = Mpad;
    p.n_rtiles = (int)(Mpad / gtc::BM);
    p.n_ttiles = (int)(Npad / gtc::BN);
    p.tiles_per_split = (int)a.tiles_per_split;
    p.split = a.split;
    p.n_units = p.n_rtiles * a.split;
    p.x = a.x; p.geo = a.geo; p.s = a.s; p.scale_sum = a.scale_sum;
    p.out = a.out; p.out_f64 = a.out_f64; p.part = a.part;
    auto kern = gtc::gauss_tc_kernel<D>;
    {
        const cudaError_t e = smem_opt_in((const void *)kern, gtc::SMEM_BYTES);
        if (e != cudaSuccess) return e;
    }
    const int grid = std::min(p.n_units, a.num_sms);
    if (a.ev_start) cudaEventRecord(a.ev_start, st);
    kern<<<grid, gtc::NT, gtc::SMEM_BYTES, st>>>(ma, mb, bvec, p);
    if (a.ev_stop) cudaEventRecord(a.ev_stop, st);
    *ctas = grid;
    *kernels = 2;
    return cudaGetLastError();
}

cudaError_t launch_gauss_tc(const GaussTcLaunch &a, cudaStream_t st, int *ctas, int *kernels) {
    if (a.M == 0) { *ctas = 0; *kernels = 0; return cudaSuccess; }
    switch (a.D) {
        case 1: return gtc_run<1>(a, st, ctas, kernels);
        case 2: return gtc_run<2>(a, st, ctas, kernels);
        case 3: return gtc_run<3>(a, st, ctas, kernels);
    }
    return cudaErrorInvalidValue;
}

}  // namespace genred
