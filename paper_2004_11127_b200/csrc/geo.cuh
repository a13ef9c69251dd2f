// geo.cuh -- data geometry for the Gaussian Sum's expanded-form path (see sum_kernel.cu).
//
// The bounding box of x and y (per coordinate, over both clouds) is reduced on the device into
// order-preserving uint encodings; every kernel that needs it decodes the same box with the
// same code, so the centre c and the path decision are bitwise identical in the pack kernel and
// in the pair-loop kernel without any host round trip.
#pragma once
#include <stdint.h>

namespace genred {

// |s (p - c)|^2 <= R2max for every point p keeps u = |x'|^2 - |x'-y'|^2 in [-4 R2max, R2max]
// (no overflow / underflow of 2^u, no range clamp needed in the polynomial exp2) and bounds the
// fp32 rounding of the expanded exponent by 3 ulp(18) ~ 3e-6 (R18b in DESIGN.md).
constexpr float kExpandedR2Max = 6.0f;

__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t e) {
    return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}

struct Geo {
    float c[8];
    bool expanded;
};

// lohi[0..7] / [8..15] = encoded per-coordinate minima / INVERTED maxima (~code, so that one
// 0xff initialisation and atomicMin serve both) of y, [16..23] / [24..31] those of x.  The centre comes from y alone, so every i-shard of the same problem (same y, different
// x rows) gets the same centre and, when its rows fit the same radius, bitwise the same
// arithmetic as the single-GPU run; the radius test covers both clouds.
// lohi == nullptr: no box was reduced (tiny N, see genred_abi.cu) -> the direct form.
__device__ __forceinline__ Geo geo_decode(const uint32_t *lohi, int D, float s) {
    Geo g;
    if (!lohi) {
#pragma unroll
        for (int d = 0; d < 8; ++d) g.c[d] = 0.0f;
        g.expanded = false;
        return g;
    }
    float r2 = 0.0f;
    bool ok = true;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
        g.c[d] = 0.0f;
        if (d < D) {
            const float lo = ord2f(lohi[d]), hi = ord2f(~lohi[8 + d]);       // maxima stored inverted
            const float xlo = ord2f(lohi[16 + d]), xhi = ord2f(~lohi[24 + d]);
            ok = ok && isfinite(lo) && isfinite(hi) && isfinite(xlo) && isfinite(xhi);
            const float c = 0.5f * lo + 0.5f * hi;
            const float h = fmaxf(fmaxf(hi - c, c - lo), fmaxf(xhi - c, c - xlo)) * 1.0001f;
            const float sh = s * h;
            r2 = fmaf(sh, sh, r2);
            g.c[d] = c;
        }
    }
    g.expanded = ok && r2 <= kExpandedR2Max;
    return g;
}

}  // namespace genred
