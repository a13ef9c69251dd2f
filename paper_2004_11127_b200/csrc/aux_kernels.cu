// aux_kernels.cu -- the HBM-streaming steps around the pair loop:
//   * j-record packing (the paper's X/Y/B "data loaders"),
//   * deterministic fixed-order merges of split-j partials (a8) and the public combine entry
//     points (monoid merges),
//   * neutral outputs for an empty reduction axis.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <cmath>

#include "device.cuh"
#include "geo.cuh"
#include "internal.h"

namespace genred {

// One block = one 512-j tile = 256 record pairs: the tile's y (and b / h) rows are staged into
// shared memory with coalesced loads, each thread builds its record pair there, and the block
// writes the tile's records (contiguous in J) with coalesced 16-byte stores.
__global__ void __launch_bounds__(256) pack_kernel(int kind, const float *__restrict__ y,
                                                   const float *__restrict__ b, int64_t N, int D, int E,
                                                   float s, double hscale, int64_t npairs, int RS,
                                                   float *__restrict__ J, const uint32_t *geo_enc,
                                                   const float *__restrict__ bx = nullptr, int64_t bM = 0,
                                                   uint32_t *geo_out = nullptr) {
    extern __shared__ float4 pack_smem4[];
    __shared__ uint32_t sgeo[32];
    float *sm = reinterpret_cast<float *>(pack_smem4);
    const float NEG_INF = -INFINITY;
    const bool gauss = kind == PACK_GAUSS_AUTO || kind == PACK_GAUSS_AUTO_RAW;
    const bool raw = kind == PACK_GAUSS_AUTO_RAW;           // + the b y' slots (gradient modes)
    const bool sumk = kind == PACK_GAUSS || kind == PACK_SQDIST_SUM;
    const int EB = (gauss || sumk) ? (b ? E : 0) : (kind == PACK_LSE_H ? 1 : 0);   // staged b / h columns
    float *ys = sm;                           // [512][D]
    float *bs = ys + kTileJ * D;              // [512][EB]
    float *outs = bs + kTileJ * EB;           // [256][RS]  (16-byte aligned: 512 (D + EB) floats)
    Geo geo{};
    if (geo_out) {
        // fused bounding box (small problems): the same encoded minima / inverted maxima that
        // bbox_kernel reduces, computed by every block over all of y (words 0..15) and x (16..31)
        __shared__ float blo[2][8][8], bhi[2][8][8];
        // both clouds in one loop, 4 rows of each per thread and iteration with every load issued
        // before the min/max: one memory round trip per 1024 rows instead of one per 256
        float lo[2][8], hi[2][8];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int d = 0; d < 8; ++d) { lo[q][d] = INFINITY; hi[q][d] = -INFINITY; }
        const int64_t rmax = max(N, bM);
        for (int64_t r0 = threadIdx.x; r0 < rmax; r0 += 4 * (int64_t)blockDim.x) {
            float v[2][4][8];
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t r = r0 + u * (int64_t)blockDim.x;
                    const bool ok = r < (q == 0 ? N : bM);
                    const float *src = q == 0 ? y : bx;
#pragma unroll
                    for (int d = 0; d < 8; ++d)
                        v[q][u][d] = (d < D && ok) ? __ldg(src + r * D + d) : NAN;   // NaN: ignored by fminf/fmaxf
                }
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int d = 0; d < 8; ++d) {
                        lo[q][d] = fminf(lo[q][d], v[q][u][d]);
                        hi[q][d] = fmaxf(hi[q][d], v[q][u][d]);
                    }
        }
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int d = 0; d < 8; ++d)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    lo[q][d] = fminf(lo[q][d], __shfl_xor_sync(0xffffffffu, lo[q][d], o));
                    hi[q][d] = fmaxf(hi[q][d], __shfl_xor_sync(0xffffffffu, hi[q][d], o));
                }
        const int warp = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int d = 0; d < 8; ++d) { blo[q][warp][d] = lo[q][d]; bhi[q][warp][d] = hi[q][d]; }
        }
        __syncthreads();
        if (threadIdx.x < 16) {
            const int q = threadIdx.x >> 3, d = threadIdx.x & 7;
            float l = blo[q][0][d], h = bhi[q][0][d];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { l = fminf(l, blo[q][w][d]); h = fmaxf(h, bhi[q][w][d]); }
            // an empty side leaves (+inf, -inf): decodes as non-finite -> the direct form,
            // as the 0xff-initialised words of the bbox_kernel path do
            sgeo[16 * q + d] = f2ord(l);
            sgeo[16 * q + 8 + d] = ~f2ord(h);
        }
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x < 32) geo_out[threadIdx.x] = sgeo[threadIdx.x];
        geo_enc = sgeo;
    }
    if (gauss) {
        geo = geo_decode(geo_enc, D, s);      // expanded or direct per the bounding box
    }
    const int t = threadIdx.x;
    for (int64_t blk = blockIdx.x; blk * 256 < npairs; blk += gridDim.x) {
        const int64_t j0 = blk * kTileJ;
        const int nj = (int)max((int64_t)0, min((int64_t)kTileJ, N - j0));
        for (int k = t; k < nj * D; k += 256) ys[k] = __ldg(y + j0 * D + k);
        for (int k = t; k < nj * EB; k += 256) bs[k] = __ldg(b + j0 * EB + k);
        __syncthreads();
        float *rec = outs + t * RS;
        for (int k = 0; k < RS; ++k) rec[k] = 0.0f;
        for (int h = 0; h < 2; ++h) {
            const int jj = 2 * t + h;
            const bool valid = jj < nj;
            if (gauss) {
                // [2D coords][w pair][2E signal]; padding: y = 0, w = 0, b = 0
                double w = 0.0;
                for (int d = 0; d < D; ++d) {
                    const float v = valid ? ys[jj * D + d] : 0.0f;
                    float r;
                    if (geo.expanded) {
                        r = valid ? s * (v - geo.c[d]) : 0.0f;        // y' = s (y - c)
                        w += (double)r * (double)r;
                    } else {
                        r = valid ? -v : 0.0f;              // direct: raw -y (R18d, R18e)
                    }
                    rec[2 * d + h] = r;
                }
                rec[2 * D + h] = geo.expanded ? (float)(-w) : 0.0f;   // w = -|y'|^2
                for (int e = 0; e < E; ++e)
                    rec[2 * D + 2 + 2 * e + h] = valid ? (b ? bs[jj * E + e] : 1.0f) : 0.0f;
                if (raw && E == 1 && kGradBY && geo.expanded) {
                    // gradient records (expanded form): the j factor 2^w is folded into the
                    // signal, b' = b 2^(-|y'|^2) (fp64, one rounding), and the records carry
                    // b' y' -- the pair loop's exponent is then u = 2 x'.y' alone (no w term)
                    const double bj = valid ? (b ? (double)bs[jj] : 1.0) : 0.0;
                    const float bp = (float)(bj * exp2(-w));
                    rec[2 * D + h] = 0.0f;
                    rec[2 * D + 2 + h] = bp;
                    for (int d = 0; d < D; ++d) rec[2 * D + 4 + 2 * d + h] = bp * rec[2 * d + h];
                } else if (raw && E == 1 && kGradBY) {
                    for (int d = 0; d < D; ++d) rec[2 * D + 4 + 2 * d + h] = 0.0f;   // direct form
                }
                continue;
            }
            for (int d = 0; d < D; ++d) {
                const float v = valid ? ys[jj * D + d] : 0.0f;
                // Sum kinds: -s y (padding 0, b = 0); LSE / ArgKMin: -y (padding at +inf distance)
                rec[2 * d + h] = sumk ? (valid ? -(s * v) : 0.0f) : (valid ? -v : NEG_INF);
            }
            if (kind == PACK_ARGKMIN) {            // the j of each half, as int32 bits (-1: padding)
                rec[2 * D + h] = __int_as_float(valid ? (int)(j0 + jj) : -1);
            } else if (sumk) {
                for (int e = 0; e < E; ++e)
                    rec[2 * D + 2 * e + h] = valid ? (b ? bs[jj * E + e] : 1.0f) : 0.0f;
            } else if (kind == PACK_LSE_H) {
                // h' = log2(e) h split into an fp32 hi part, which enters the exponent, and the
                // factor c = 2^(h'_lo) of the term: |h| ~ 1e4 biases stay exact to fp32 rounding.
                const double hv = valid ? hscale * (double)bs[jj] : 0.0;
                const float hi = valid ? (float)hv : NEG_INF;
                rec[2 * D + h] = hi;
                rec[2 * D + 2 + h] = valid ? (float)exp2(hv - (double)hi) : 0.0f;   // c = 2^(h'_lo)
            }
        }
        __syncthreads();
        const int nrec = (int)min((int64_t)256, npairs - blk * 256);
        float4 *dst = reinterpret_cast<float4 *>(J + blk * 256 * RS);
        const float4 *src4 = reinterpret_cast<const float4 *>(outs);
        for (int k = t; k < nrec * RS / 4; k += 256) dst[k] = src4[k];
        __syncthreads();
    }
}

static int pack_smem_bytes(int kind, int D, int E, int RS, bool has_b) {
    const bool gauss = kind == PACK_GAUSS_AUTO || kind == PACK_GAUSS_AUTO_RAW;
    const bool sumk = kind == PACK_GAUSS || kind == PACK_SQDIST_SUM;
    const int EB = (gauss || sumk) ? (has_b ? E : 0) : (kind == PACK_LSE_H ? 1 : 0);
    return (kTileJ * (D + EB) + 256 * RS) * 4;
}

int pack_record_stride(int kind, int D, int E) {
    if (kind == PACK_GAUSS_AUTO) return record_stride(D + 1, E);
    if (kind == PACK_GAUSS_AUTO_RAW) return gauss_record_stride(D, E, true);
    if (kind == PACK_ARGKMIN) return record_stride(D + 1, 0);      // + the j pair
    if (kind == PACK_LSE_HZ) return record_stride(D, 0);
    if (kind == PACK_LSE_H) return record_stride(D, 2);
    return record_stride(D, E);
}

cudaError_t launch_pack(int kind, const float *y, const float *b, int64_t N, int D, int E, float s,
                        double hscale, int64_t npairs, float *J, cudaStream_t st, const uint32_t *geo) {
    const int RS = pack_record_stride(kind, D, E);
    const int smem = pack_smem_bytes(kind, D, E, RS, b != nullptr);
    if (smem > 48 * 1024) {                       // every kind / D / E fits in 96 KB
        const cudaError_t e = smem_opt_in((const void *)pack_kernel, 96 * 1024);
        if (e != cudaSuccess) return e;
    }
    int64_t blocks = (npairs + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    pack_kernel<<<(unsigned)blocks, 256, smem, st>>>(kind, y, b, N, D, E, s, hscale, npairs, RS, J, geo);
    return cudaGetLastError();
}

cudaError_t launch_pack_boxed(int kind, const float *y, const float *b, int64_t N, int D, int E,
                              float s, int64_t npairs, float *J, const float *x, int64_t M,
                              uint32_t *geo, cudaStream_t st) {
    const int RS = pack_record_stride(kind, D, E);
    const int smem = pack_smem_bytes(kind, D, E, RS, b != nullptr);
    if (smem > 48 * 1024) {
        const cudaError_t e = smem_opt_in((const void *)pack_kernel, 96 * 1024);
        if (e != cudaSuccess) return e;
    }
    int64_t blocks = (npairs + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    pack_kernel<<<(unsigned)blocks, 256, smem, st>>>(kind, y, b, N, D, E, s, 0.0, npairs, RS, J,
                                                      nullptr, x, M, geo);
    return cudaGetLastError();
}

// ---- range-packed j-records (block-sparse ranges) -----------------------------------------------
// Record pair p belongs to the gathered interval k with copies[k].dst <= p < copies[k+1].dst; its
// two j's are js + 2 (p - dst) + {0, 1}, valid while < je.  Invalid halves and padding pairs hold
// zero-contribution records (b = 0).  Layouts as pack_kernel (GAUSS_AUTO or SQDIST_SUM).
__global__ void pack_ranges_kernel(int kind, const float *__restrict__ y, const float *__restrict__ b,
                                   int64_t N, int D, int E, float s, const RangeCopy *__restrict__ copies,
                                   int ncopies, int64_t npairs, int RS, float *__restrict__ J,
                                   const uint32_t *geo_enc) {
    const bool gauto = kind == PACK_GAUSS_AUTO || kind == PACK_GAUSS_AUTO_RAW;
    const Geo geo = gauto ? geo_decode(geo_enc, D, s) : Geo{};
    const int boff = gauto ? 2 * (D + 1) : 2 * D;
    const bool lse = kind == PACK_LSE_HZ || kind == PACK_LSE_H || kind == PACK_ARGKMIN;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
         p += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = ncopies - 1;                          // last copy with dst <= p
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (copies[mid].dst <= p) lo = mid; else hi = mid - 1;
        }
        const RangeCopy c = copies[lo];
        float *rec = J + p * RS;
        if (lse) {          // LSE records: (-y) pairs [+ h' hi/lo pairs]; invalid: y = +inf, h = -inf
                            // ArgKMin records: (-y) pairs + the original j pair (int32 bits, -1 invalid)
            for (int h = 0; h < 2; ++h) {
                const int64_t j = c.js + 2 * (p - c.dst) + h;
                const bool valid = j < c.je && j < N;
                for (int d = 0; d < D; ++d) rec[2 * d + h] = valid ? -y[j * D + d] : -INFINITY;
                if (kind == PACK_ARGKMIN) rec[2 * D + h] = __int_as_float(valid ? (int)j : -1);
                if (kind == PACK_LSE_H) {
                    const double hv = valid ? 1.4426950408889634074 * (double)b[j] : 0.0;
                    const float hi = valid ? (float)hv : -INFINITY;
                    rec[2 * D + h] = hi;
                    rec[2 * D + 2 + h] = valid ? (float)exp2(hv - (double)hi) : 0.0f;   // c = 2^(h'_lo)
                }
            }
            for (int k = 2 * D + (kind == PACK_LSE_H ? 4 : kind == PACK_ARGKMIN ? 2 : 0); k < RS; ++k) rec[k] = 0.0f;
            continue;
        }
        for (int h = 0; h < 2; ++h) {
            const int64_t j = c.js + 2 * (p - c.dst) + h;
            const bool valid = j < c.je && j < N;
            double w = 0.0;
            for (int d = 0; d < D; ++d) {
                const float v = valid ? y[j * D + d] : 0.0f;
                float r;
                if (gauto && geo.expanded) {
                    r = valid ? s * (v - geo.c[d]) : 0.0f;
                    w += (double)r * (double)r;
                } else {
                    r = valid ? (gauto ? -v : -(s * v)) : 0.0f;   // Gaussian direct: raw -y
                }
                rec[2 * d + h] = r;
            }
            if (gauto) rec[2 * D + h] = geo.expanded ? (float)(-w) : 0.0f;
            for (int e = 0; e < E; ++e)
                rec[boff + 2 * e + h] = valid ? (b ? b[j * E + e] : 1.0f) : 0.0f;
            if (kind == PACK_GAUSS_AUTO_RAW && E == 1 && kGradBY) {   // b' = b 2^w, b' y' (as pack_kernel)
                if (geo.expanded) {
                    const double bj = valid ? (b ? (double)b[j] : 1.0) : 0.0;
                    const float bp = (float)(bj * exp2(-w));
                    rec[2 * D + h] = 0.0f;
                    rec[boff + h] = bp;
                    for (int d = 0; d < D; ++d) rec[boff + 2 + 2 * d + h] = bp * rec[2 * d + h];
                } else {
                    for (int d = 0; d < D; ++d) rec[boff + 2 + 2 * d + h] = 0.0f;
                }
            }
        }
        const int used = boff + 2 * E + ((kind == PACK_GAUSS_AUTO_RAW && E == 1 && kGradBY) ? 2 * D : 0);
        for (int k = used; k < RS; ++k) rec[k] = 0.0f;
    }
}

cudaError_t launch_pack_ranges(int kind, const float *y, const float *b, int64_t N, int D, int E,
                               float s, const RangeCopy *copies, int ncopies, int64_t npairs,
                               float *J, cudaStream_t st, const uint32_t *geo) {
    const int RS = pack_record_stride(kind, D, E);
    int64_t blocks = (npairs + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    pack_ranges_kernel<<<(unsigned)blocks, 256, 0, st>>>(kind, y, b, N, D, E, s, copies, ncopies,
                                                         npairs, RS, J, geo);
    return cudaGetLastError();
}

// ---- per-coordinate bounding box of x and y (order-preserving uint encodings, geo.cuh) -------
// blockIdx.y = 0: y into geo[0..15]; blockIdx.y = 1: x into geo[16..31]
// Row-wise pass over y (blockIdx.y == 0) or x (1): a warp reads 32 consecutive rows per load
// instruction (coalesced); four rows per thread per iteration keep 4 D loads in flight.
__global__ void bbox_kernel(const float *__restrict__ x, int64_t M, const float *__restrict__ y,
                            int64_t N, int D, uint32_t *geo) {
    float lo[8], hi[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) { lo[d] = INFINITY; hi[d] = -INFINITY; }
    const float *src = blockIdx.y == 0 ? y : x;
    const int64_t rows = blockIdx.y == 0 ? N : M;
    const int off = blockIdx.y == 0 ? 0 : 16;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; t + 3 * stride < rows; t += 4 * stride) {
        float v[4][8];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int d = 0; d < 8; ++d) v[q][d] = d < D ? __ldg(src + (t + q * stride) * D + d) : 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int d = 0; d < 8; ++d)
                if (d < D) { lo[d] = fminf(lo[d], v[q][d]); hi[d] = fmaxf(hi[d], v[q][d]); }
    }
    for (; t < rows; t += stride) {
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            if (d < D) {
                const float v = __ldg(src + t * D + d);
                lo[d] = fminf(lo[d], v);
                hi[d] = fmaxf(hi[d], v);
            }
        }
    }
#pragma unroll
    for (int d = 0; d < 8; ++d) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    }
    // block reduction through shared memory, then one atomic per coordinate and block (per-warp
    // atomics on the same 2D words serialise at L2)
    __shared__ float slo[8][8], shi[8][8];
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int dd = 0; dd < 8; ++dd) { slo[warp][dd] = lo[dd]; shi[warp][dd] = hi[dd]; }
    }
    __syncthreads();
    if (threadIdx.x < D) {
        const int dd = threadIdx.x;
        float l = slo[0][dd], h = shi[0][dd];
        for (int w = 1; w < nw; ++w) { l = fminf(l, slo[w][dd]); h = fmaxf(h, shi[w][dd]); }
        if (l <= h) {
            atomicMin(geo + off + dd, f2ord(l));
            atomicMin(geo + off + 8 + dd, ~f2ord(h));          // maxima stored inverted (geo.cuh)
        }
    }
}

cudaError_t launch_bbox(const float *x, int64_t M, const float *y, int64_t N, int D, uint32_t *geo,
                        cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    // every word starts at the largest code: minima reduce with atomicMin, and so do the maxima,
    // stored inverted (one memset instead of four)
    e = cudaMemsetAsync(geo, 0xff, 32 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    int64_t blocks = (std::max(M, N) + 1023) / 1024;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    bbox_kernel<<<dim3((unsigned)blocks, 2), 256, 0, st>>>(x, M, y, N, D, geo);
    return cudaGetLastError();
}

bool geo_expanded_host(const uint32_t *geo_dev, int D, float s) {
    uint32_t h[32];
    if (cudaMemcpy(h, geo_dev, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    auto dec = [](uint32_t e) {
        uint32_t u = (e & 0x80000000u) ? (e & 0x7fffffffu) : ~e;
        float f;
        memcpy(&f, &u, 4);
        return f;
    };
    float r2 = 0.0f;
    bool ok = true;
    for (int d = 0; d < D; ++d) {
        const float lo = dec(h[d]), hi = dec(~h[8 + d]), xlo = dec(h[16 + d]), xhi = dec(~h[24 + d]);
        ok = ok && std::isfinite(lo) && std::isfinite(hi) && std::isfinite(xlo) && std::isfinite(xhi);
        const float c = 0.5f * lo + 0.5f * hi;
        const float hh = fmaxf(fmaxf(hi - c, c - lo), fmaxf(xhi - c, c - xlo)) * 1.0001f;
        const float sh = s * hh;
        r2 = fmaf(sh, sh, r2);
    }
    return ok && r2 <= kExpandedR2Max;
}

// ---- Sum / gradient: out = scale * sum_{split} part[split] in split order ----------------------
__device__ __forceinline__ void sum_finalize_store(double acc, int64_t i, int C, int c, int cols_sum,
                                                   const float *__restrict__ g, int E, double scale_sum,
                                                   double scale_grad, int mode, void *out, int out_f64,
                                                   float *out_grad);

// Many splits (small-M mode): one warp per output, lanes sum strided partials in a fixed order
// and a fixed butterfly finishes (deterministic), instead of one thread walking all S partials.
__global__ void sum_finalize_warp_kernel(const double *__restrict__ part, int split, int64_t M, int C,
                                         int cols_sum, const float *__restrict__ g, int E,
                                         double scale_sum, double scale_grad, int mode, void *out,
                                         int out_f64, float *out_grad) {
    const int64_t total = M * C;
    const int lane = threadIdx.x & 31;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < total;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t i = t / C;
        const int c = (int)(t % C);
        double acc = 0.0;
        for (int q = lane; q < split; q += 32) acc += part[((int64_t)q * M + i) * C + c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) sum_finalize_store(acc, i, C, c, cols_sum, g, E, scale_sum, scale_grad, mode, out, out_f64, out_grad);
    }
}

__global__ void sum_finalize_kernel(const double *__restrict__ part, int split, int64_t M, int C,
                                    int cols_sum, const float *__restrict__ g, int E,
                                    double scale_sum, double scale_grad, int mode, void *out,
                                    int out_f64, float *out_grad) {
    const int64_t total = M * C;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / C;
        const int c = (int)(t % C);
        double acc = 0.0;
        for (int q = 0; q < split; ++q) acc += part[((int64_t)q * M + i) * C + c];
        sum_finalize_store(acc, i, C, c, cols_sum, g, E, scale_sum, scale_grad, mode, out, out_f64, out_grad);
    }
}

__device__ __forceinline__ void sum_finalize_store(double acc, int64_t i, int C, int c, int cols_sum,
                                                   const float *__restrict__ g, int E, double scale_sum,
                                                   double scale_grad, int mode, void *out, int out_f64,
                                                   float *out_grad) {
    {
        if (c < cols_sum) {
            double v = acc * scale_sum;
            if (out_f64) ((double *)out)[i * cols_sum + c] = v;
            else ((float *)out)[i * cols_sum + c] = (float)v;
        } else {
            // gradient column: scale (and the cotangent when it was factored out, E == 1)
            double v = acc * scale_grad;
            if (E == 1 && g) v *= (double)g[i];
            const int dcol = c - cols_sum;
            const int Dg = C - cols_sum;
            if (mode == 2) out_grad[i * Dg + dcol] = (float)v;
            else if (out_f64) ((double *)out)[i * Dg + dcol] = v;
            else ((float *)out)[i * Dg + dcol] = (float)v;
        }
    }
}

cudaError_t launch_sum_finalize(const double *part, int split, int64_t M, int C, int cols_sum,
                                const float *g, int E, double scale_sum, double scale_grad,
                                int mode, void *out, int out_f64, float *out_grad, cudaStream_t st) {
    if (split > 32) {
        int64_t blocks = (M * C * 32 + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        if (blocks < 1) blocks = 1;
        sum_finalize_warp_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, split, M, C, cols_sum, g, E,
                                                                   scale_sum, scale_grad, mode, out,
                                                                   out_f64, out_grad);
        return cudaGetLastError();
    }
    int64_t blocks = (M * C + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    sum_finalize_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, split, M, C, cols_sum, g, E,
                                                          scale_sum, scale_grad, mode, out,
                                                          out_f64, out_grad);
    return cudaGetLastError();
}

// ---- log-sum-exp: (m, s) states in log2 units; merge = max-rescale ------------
__global__ void lse_finalize_kernel(const double *__restrict__ part, int split, int64_t M, void *out,
                                    int out_f64, double *state_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        double mstar = -INFINITY;
        for (int q = 0; q < split; ++q) {
            const double s = part[((int64_t)q * M + i) * 2 + 1];
            const double m = part[((int64_t)q * M + i) * 2 + 0];
            if (s > 0.0 && m > mstar) mstar = m;
        }
        double S = 0.0;
        if (mstar > -INFINITY) {
            for (int q = 0; q < split; ++q) {
                const double m = part[((int64_t)q * M + i) * 2 + 0];
                const double s = part[((int64_t)q * M + i) * 2 + 1];
                if (s > 0.0) S += s * exp2(m - mstar);
            }
        }
        const double a = (S > 0.0) ? 0.69314718055994530942 * (mstar + log2(S)) : -INFINITY;
        if (out) {
            if (out_f64) ((double *)out)[i] = a;
            else ((float *)out)[i] = (float)a;
        }
        if (state_out) {
            state_out[2 * i + 0] = (S > 0.0) ? mstar : (double)kLseSentinel;
            state_out[2 * i + 1] = S;
        }
    }
}

// Many splits: one warp per row; the max and the rescaled sum run lane-strided in a fixed order
// and finish with fixed butterflies (deterministic).
__global__ void lse_finalize_warp_kernel(const double *__restrict__ part, int split, int64_t M, void *out,
                                         int out_f64, double *state_out) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < M;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double mstar = -INFINITY;
        for (int q = lane; q < split; q += 32) {
            const double s = part[((int64_t)q * M + i) * 2 + 1];
            const double m = part[((int64_t)q * M + i) * 2 + 0];
            if (s > 0.0 && m > mstar) mstar = m;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mstar = fmax(mstar, __shfl_xor_sync(0xffffffffu, mstar, o));
        double S = 0.0;
        if (mstar > -INFINITY) {
            for (int q = lane; q < split; q += 32) {
                const double m = part[((int64_t)q * M + i) * 2 + 0];
                const double s = part[((int64_t)q * M + i) * 2 + 1];
                if (s > 0.0) S += s * exp2(m - mstar);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
        if (lane != 0) continue;
        const double a = (S > 0.0) ? 0.69314718055994530942 * (mstar + log2(S)) : -INFINITY;
        if (out) {
            if (out_f64) ((double *)out)[i] = a;
            else ((float *)out)[i] = (float)a;
        }
        if (state_out) {
            state_out[2 * i + 0] = (S > 0.0) ? mstar : (double)kLseSentinel;
            state_out[2 * i + 1] = S;
        }
    }
}

cudaError_t launch_lse_finalize(const double *part, int split, int64_t M, void *out, int out_f64,
                                double *state_out, cudaStream_t st) {
    if (split > 32) {
        int64_t blocks = (M * 32 + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        if (blocks < 1) blocks = 1;
        lse_finalize_warp_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, split, M, out, out_f64, state_out);
        return cudaGetLastError();
    }
    int64_t blocks = (M + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    lse_finalize_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, split, M, out, out_f64, state_out);
    return cudaGetLastError();
}

// ---- ArgKMin: G sorted K-lists per row -> K smallest under (d, j) lexicographic order ---------
template <typename IDX>
__global__ void topk_merge_kernel(const float *__restrict__ pd, const IDX *__restrict__ pi, int G,
                                  int64_t M, int K, float *dist, int64_t *idx, int64_t j_offset) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        int head[64];
        for (int q = 0; q < G; ++q) head[q] = 0;
        for (int k = 0; k < K; ++k) {
            int best = -1;
            float bd = INFINITY;
            int64_t bj = -1;
            for (int q = 0; q < G; ++q) {
                if (head[q] >= K) continue;
                const int64_t off = ((int64_t)q * M + i) * K + head[q];
                const int64_t j = (int64_t)pi[off];
                if (j < 0) continue;                      // list exhausted (padding)
                const float d = pd[off];
                if (best < 0 || d < bd || (d == bd && j < bj)) { best = q; bd = d; bj = j; }
            }
            if (best >= 0) {
                head[best]++;
                dist[i * K + k] = bd;
                idx[i * K + k] = bj + j_offset;
            } else {
                dist[i * K + k] = INFINITY;
                idx[i * K + k] = -1;
            }
        }
    }
}

cudaError_t launch_topk_merge_i32(const float *pd, const int32_t *pi, int split, int64_t M, int K,
                                  float *dist, int64_t *idx, int64_t j_offset, cudaStream_t st) {
    int64_t blocks = (M + 127) / 128;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    topk_merge_kernel<int32_t><<<(unsigned)blocks, 128, 0, st>>>(pd, pi, split, M, K, dist, idx,
                                                                 j_offset);
    return cudaGetLastError();
}

// Merge lists [64 g, 64 g + 64) of row i into list g (lexicographic (d, j), as topk_merge).
__global__ void topk_merge_groups_kernel(const float *__restrict__ pd, const int32_t *__restrict__ pi,
                                         int split, int64_t M, int K, float *gd, int32_t *gi) {
    const int G1 = (split + 63) / 64;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M * G1;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int g = (int)(t / M);
        const int64_t i = t % M;
        const int q0 = 64 * g, nq = min(64, split - q0);
        int head[64];
        for (int q = 0; q < nq; ++q) head[q] = 0;
        for (int k = 0; k < K; ++k) {
            int best = -1;
            float bd = INFINITY;
            int32_t bj = -1;
            for (int q = 0; q < nq; ++q) {
                if (head[q] >= K) continue;
                const int64_t off = ((int64_t)(q0 + q) * M + i) * K + head[q];
                const int32_t j = pi[off];
                if (j < 0) continue;
                const float d = pd[off];
                if (best < 0 || d < bd || (d == bd && (uint32_t)j < (uint32_t)bj)) { best = q; bd = d; bj = j; }
            }
            const int64_t o = ((int64_t)g * M + i) * K + k;
            if (best >= 0) { head[best]++; gd[o] = bd; gi[o] = bj; }
            else { gd[o] = INFINITY; gi[o] = -1; }
        }
    }
}

cudaError_t launch_topk_merge_groups(const float *pd, const int32_t *pi, int split, int64_t M, int K,
                                     float *gd, int32_t *gi, cudaStream_t st) {
    const int64_t work = M * ((split + 63) / 64);
    int64_t blocks = (work + 127) / 128;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    topk_merge_groups_kernel<<<(unsigned)blocks, 128, 0, st>>>(pd, pi, split, M, K, gd, gi);
    return cudaGetLastError();
}

cudaError_t launch_topk_merge_i64(const float *pd, const int64_t *pi, int G, int64_t M, int K,
                                  float *dist, int64_t *idx, cudaStream_t st) {
    int64_t blocks = (M + 127) / 128;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    topk_merge_kernel<int64_t><<<(unsigned)blocks, 128, 0, st>>>(pd, pi, G, M, K, dist, idx, 0);
    return cudaGetLastError();
}

// ---- neutral outputs for N == 0: Sum -> 0, LSE -> -inf, ArgKMin -> (+inf, -1) -------------------
__global__ void fill_kernel(int kind, int64_t M, int C, int K, void *out, int out_f64,
                            float *out_grad, int64_t *idx, double *state) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (kind == 0) {                                  // SUM / GRADX
            for (int c = 0; c < C; ++c) {
                if (out_f64) ((double *)out)[i * C + c] = 0.0;
                else ((float *)out)[i * C + c] = 0.0f;
            }
        } else if (kind == 1) {                           // SUM_GRADX: C = E sum cols, K = D
            for (int c = 0; c < C; ++c) {
                if (out_f64) ((double *)out)[i * C + c] = 0.0;
                else ((float *)out)[i * C + c] = 0.0f;
            }
            for (int d = 0; d < K; ++d) out_grad[i * K + d] = 0.0f;
        } else if (kind == 2) {                           // LSE
            if (out_f64) ((double *)out)[i] = -INFINITY;
            else ((float *)out)[i] = -INFINITY;
            if (state) { state[2 * i] = (double)kLseSentinel; state[2 * i + 1] = 0.0; }
        } else {                                          // ARGKMIN
            for (int k = 0; k < K; ++k) {
                ((float *)out)[i * K + k] = INFINITY;
                idx[i * K + k] = -1;
            }
        }
    }
}

cudaError_t launch_fill(int kind, int64_t M, int C, int K, void *out, int out_f64, float *out_grad,
                        int64_t *idx, double *state, cudaStream_t st) {
    int64_t blocks = (M + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(kind, M, C, K, out, out_f64, out_grad, idx, state);
    return cudaGetLastError();
}

}  // namespace genred
