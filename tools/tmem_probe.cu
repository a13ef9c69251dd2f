// Probe: tcgen05.ld (TMEM -> registers) throughput per SM, 4 / 8 / 16 warps per CTA, 1 CTA/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
__device__ __forceinline__ uint32_t smem_u32(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll 1
    for (int c = 0; c < 512 / (NW / 4); c += 32) {
      const uint32_t col = (uint32_t)((warp >> 2) * (512 / (NW / 4)) + c);
      uint32_t v[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
        : "r"(base + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      #pragma unroll
      for (int q = 0; q < 32; ++q) acc += __uint_as_float(v[q]);
    }
  }
  if (acc == 1.2345f) out[0] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot) : "memory");
}
template <int NW> int run(int nsm) {
  float* d; CK(cudaMalloc(&d, 4));
  int iters = 2000;
  k<NW><<<nsm, NW * 32>>>(d, 10); CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<NW><<<nsm, NW * 32>>>(d, iters); cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  double bytes = (double)nsm * iters * 128.0 * 512 * 4;     // every lane x column read once per iter
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("tmem ld warps=%2d  %.3f ms  %.1f B/clk/SM (at max clock)\n", NW, ms, bytes / (ms * 1e-3) / nsm / (clk * 1e3));
  return 0;
}
int main() { int n; cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0); run<4>(n); run<8>(n); run<16>(n); return 0; }
