// Host-side cost of genred_eval (C ABI, no Python): enqueue time per call for a C1-sized
// Gaussian Sum (M = N = 1000), plus the device time per call when the host is not the limit.
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "genred.h"
int main() {
    const int n = 1000;
    std::vector<float> hx(n * 3), hy(n * 3), hb(n);
    for (int i = 0; i < n * 3; ++i) { hx[i] = (i * 37 % 1000) / 1000.f; hy[i] = (i * 91 % 1000) / 1000.f; }
    for (int i = 0; i < n; ++i) hb[i] = (i % 7) / 7.f;
    float *x, *y, *b, *o;
    cudaMalloc(&x, n * 12); cudaMalloc(&y, n * 12); cudaMalloc(&b, n * 4); cudaMalloc(&o, n * 4);
    cudaMemcpy(x, hx.data(), n * 12, cudaMemcpyHostToDevice);
    cudaMemcpy(y, hy.data(), n * 12, cudaMemcpyHostToDevice);
    cudaMemcpy(b, hb.data(), n * 4, cudaMemcpyHostToDevice);
    genred_ctx *ctx = nullptr;
    if (genred_create(0, &ctx) != GENRED_OK) { printf("create failed\n"); return 1; }
    genred_args a = {};
    a.abi_version = GENRED_ABI_VERSION; a.formula = GENRED_GAUSS; a.reduction = GENRED_SUM;
    a.M = n; a.N = n; a.D = 3; a.E = 1; a.K = 1; a.scale = 0.5; a.x = x; a.y = y; a.b = b; a.out = o;
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int i = 0; i < 100; ++i) genred_eval(ctx, &a, st);
    cudaStreamSynchronize(st);
    for (int rep = 0; rep < 3; ++rep) {
        const int K = 200;
        auto t0 = std::chrono::high_resolution_clock::now();
        for (int i = 0; i < K; ++i) genred_eval(ctx, &a, st);
        auto t1 = std::chrono::high_resolution_clock::now();
        cudaStreamSynchronize(st);
        auto t2 = std::chrono::high_resolution_clock::now();
        printf("C ABI: enqueue us/call %.2f, wall us/call %.2f\n",
               std::chrono::duration<double, std::micro>(t1 - t0).count() / K,
               std::chrono::duration<double, std::micro>(t2 - t0).count() / K);
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // bare launch cost of an empty-ish kernel for comparison: a 1-float memset
    auto t0 = std::chrono::high_resolution_clock::now();
    for (int i = 0; i < 200; ++i) cudaMemsetAsync(o, 0, 4, st);
    auto t1 = std::chrono::high_resolution_clock::now();
    cudaStreamSynchronize(st);
    printf("cudaMemsetAsync enqueue us/call %.2f\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 200);
    genred_plan pl; genred_last_plan(ctx, &pl);
    printf("plan split %d kernels %d ctas %d\n", pl.split_j, pl.kernels, pl.ctas);
    genred_destroy(ctx);
    return 0;
}
