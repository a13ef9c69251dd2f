// aux_kernels.cu -- the HBM-streaming steps around the pair loop:
//   * j-record packing (the paper's X/Y/B "data loaders"),
//   * deterministic fixed-order merges of split-j partials (a8) and the public combine entry
//     points (monoid merges),
//   * neutral outputs for an empty reduction axis.
#include <math.h>

#include "device.cuh"
#include "internal.h"

namespace genred {

__global__ void pack_kernel(int kind, const float *__restrict__ y, const float *__restrict__ b,
                            int64_t N, int D, int E, float s, double hscale, int64_t npairs, int RS,
                            float *__restrict__ J) {
    const float NEG_INF = -INFINITY;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
         p += (int64_t)gridDim.x * blockDim.x) {
        float *rec = J + p * RS;
        for (int h = 0; h < 2; ++h) {
            const int64_t j = 2 * p + h;
            const bool valid = j < N;
            for (int d = 0; d < D; ++d) {
                float v = valid ? y[j * D + d] : 0.0f;
                float r;
                if (kind == PACK_GAUSS || kind == PACK_SQDIST_SUM) r = valid ? -(s * v) : 0.0f;
                else r = valid ? -v : NEG_INF;          // LSE / ARGKMIN: padded y at +inf distance
                rec[2 * d + h] = r;
            }
            if (kind == PACK_GAUSS || kind == PACK_SQDIST_SUM) {
                for (int e = 0; e < E; ++e)
                    rec[2 * D + 2 * e + h] = valid ? (b ? b[j * E + e] : 1.0f) : 0.0f;
            } else if (kind == PACK_LSE_H) {
                // h' = log2(e) h as an fp32 hi + lo pair (fp64 product), so that
                // (h'_hi - m) + h'_lo keeps |h| ~ 1e4 biases exact to fp32 rounding of t.
                const double hv = valid ? hscale * (double)b[j] : 0.0;
                const float hi = valid ? (float)hv : NEG_INF;
                rec[2 * D + h] = hi;
                rec[2 * D + 2 + h] = valid ? (float)(hv - (double)hi) : 0.0f;
            }
        }
        const int used = (kind == PACK_ARGKMIN || kind == PACK_LSE_HZ) ? 2 * D
                       : (kind == PACK_LSE_H ? 2 * D + 4 : 2 * (D + E));
        for (int k = used; k < RS; ++k) rec[k] = 0.0f;
    }
}

int pack_record_stride(int kind, int D, int E) {
    if (kind == PACK_ARGKMIN || kind == PACK_LSE_HZ) return record_stride(D, 0);
    if (kind == PACK_LSE_H) return record_stride(D, 2);
    return record_stride(D, E);
}

cudaError_t launch_pack(int kind, const float *y, const float *b, int64_t N, int D, int E, float s,
                        double hscale, int64_t npairs, float *J, cudaStream_t st) {
    const int RS = pack_record_stride(kind, D, E);
    int64_t blocks = (npairs + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    pack_kernel<<<(unsigned)blocks, 256, 0, st>>>(kind, y, b, N, D, E, s, hscale, npairs, RS, J);
    return cudaGetLastError();
}

// ---- Sum / gradient: out = scale * sum_{split} part[split] in split order ----------------------
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

cudaError_t launch_lse_finalize(const double *part, int split, int64_t M, void *out, int out_f64,
                                double *state_out, cudaStream_t st) {
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
