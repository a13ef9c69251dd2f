// device.cuh -- sm_100a device primitives used by the Genred kernels: mbarrier, 1-D bulk copy
// (TMA engine, cp.async.bulk -> SASS UBLKCP), MUFU ex2, packed f32x2 arithmetic.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace genred {

__device__ __forceinline__ float ex2(float x) {          // MUFU.EX2, 2^x, flush-to-zero
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float max3(float a, float b, float c) {   // FMNMX3
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 dup2(float a) { return make_float2(a, a); }

// 2^u for u in [-24, 6] (the expanded path's range, geo.cuh) on the FP32 pipe: u = n + f with
// n = rint(u) from the 1.5*2^23 shifter, f in [-1/2, 1/2], a degree-5 near-minimax polynomial
// (max relative error 7.5e-8; 2.3e-7 through fp32 Horner, on par with MUFU.EX2), and n added
// to the exponent field with one integer LEA.  Two values per packed FADD2/FFMA2.
__device__ __forceinline__ float2 ex2_poly2(float2 u) {
    const float2 shifter = dup2(12582912.0f);
    const float2 t = add2(u, shifter);
    const float2 n = add2(t, dup2(-12582912.0f));
    const float2 f = fma2(n, dup2(-1.0f), u);                       // u - n, exact
    float2 q = fma2(dup2(1.327647129073739e-03f), f, dup2(9.675541892647743e-03f));
    q = fma2(q, f, dup2(5.550713092088699e-02f));
    q = fma2(q, f, dup2(2.402212023735046e-01f));
    q = fma2(q, f, dup2(6.931469440460205e-01f));
    q = fma2(q, f, dup2(1.000000119209290e+00f));
    return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier (shared::cta) -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// ---- 1-D bulk copy global -> shared through the TMA engine, completing on an mbarrier -----
// bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float4 lds128(const float *p) {
    return *reinterpret_cast<const float4 *>(p);
}

}  // namespace genred

// Stage release: the LAST warp to finish a tile refills its stage (an acq_rel shared-memory
// counter per stage, then fence.proxy.async before the bulk copy), instead of thread 0 waiting
// on an mbarrier for every warp: +0.7% Gaussian Sum, +1.6% LSE, +0.5% fused Sum+grad (B200).
#ifndef GENRED_RING_LAST_WARP
#define GENRED_RING_LAST_WARP 1
#endif

namespace genred {

// ---- j-tile ring shared by the FP32/MUFU pair-loop kernels ---------------------------------
// STAGES shared-memory buffers of `bytes` each, filled by cp.async.bulk (TMA engine) and
// completing on `full` mbarriers.  No dedicated producer warp: thread 0 issues the prologue
// loads, and the last warp to release a stage refills it with the tile STAGES ahead.  All warps
// of the CTA are math warps, so a 256-thread CTA keeps 2 (or 3) CTAs per SM within the
// per-SM-partition register budget (16K registers / SMSP).
template <int STAGES>
struct JRing {
    float *tiles;
    uint64_t *full, *empty;
    const float *src;          // first tile of this CTA's j-range
    int nt;                    // tiles in the range
    int tile_floats;
    uint32_t bytes;
    uint32_t last_bytes;       // bytes of the range's last tile (a partial tile when N is small)
    int nw;                    // warps that release each stage

    __device__ __forceinline__ uint32_t tile_bytes(int k) const { return k == nt - 1 ? last_bytes : bytes; }

    __device__ __forceinline__ void init(unsigned char *smem, int tile_floats_, const float *src_,
                                         int nt_, int nwarps, uint32_t last_bytes_ = 0) {
        tile_floats = tile_floats_;
        bytes = (uint32_t)tile_floats_ * 4u;
        last_bytes = last_bytes_ ? last_bytes_ : bytes;
        tiles = reinterpret_cast<float *>(smem);
        full = reinterpret_cast<uint64_t *>(smem + (size_t)STAGES * bytes);
        empty = full + STAGES;
        src = src_;
        nt = nt_;
        nw = nwarps;
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(&full[s], 1);
#if GENRED_RING_LAST_WARP
                reinterpret_cast<uint32_t *>(empty)[s] = 0;                // stage release counters
#else
                mbar_init(&empty[s], nwarps);
#endif
            }
            fence_barrier_init();
            for (int k = 0; k < STAGES && k < nt; ++k) {
                mbar_arrive_expect_tx(&full[k], tile_bytes(k));
                bulk_g2s(tiles + k * tile_floats, src + (int64_t)k * tile_floats, tile_bytes(k), &full[k]);
            }
        }
        __syncthreads();
    }
    __device__ __forceinline__ const float *acquire(int k) {
        const int s = k % STAGES;
        mbar_wait(&full[s], (k / STAGES) & 1);
        return tiles + s * tile_floats;
    }
    __device__ __forceinline__ void release(int k) {
        const int s = k % STAGES;
        __syncwarp();
#if GENRED_RING_LAST_WARP
        // the last warp to finish tile k refills its stage (no warp waits for stragglers)
        if ((threadIdx.x & 31) == 0) {
            uint32_t *cnt = reinterpret_cast<uint32_t *>(empty);           // [STAGES] counters
            uint32_t old;
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old) : "r"(smem_u32(cnt + s)) : "memory");
            if (old == (uint32_t)nw - 1) {
                cnt[s] = 0;
                if (k + STAGES < nt) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const uint32_t nb = tile_bytes(k + STAGES);
                    mbar_arrive_expect_tx(&full[s], nb);
                    bulk_g2s(tiles + s * tile_floats, src + (int64_t)(k + STAGES) * tile_floats, nb, &full[s]);
                }
            }
        }
#else
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        if (threadIdx.x == 0 && k + STAGES < nt) {
            mbar_wait(&empty[s], (k / STAGES) & 1);          // every warp is done with tile k
            const uint32_t nb = tile_bytes(k + STAGES);
            mbar_arrive_expect_tx(&full[s], nb);
            bulk_g2s(tiles + s * tile_floats, src + (int64_t)(k + STAGES) * tile_floats, nb, &full[s]);
        }
#endif
    }
    static constexpr int smem_bytes(int tile_floats_) { return STAGES * tile_floats_ * 4 + 2 * STAGES * 8; }
};

}  // namespace genred
