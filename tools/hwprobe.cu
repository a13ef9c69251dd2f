// Step-0 hardware probe: per-clock throughput of FFMA, FFMA2, FADD2,
// MUFU.EX2 and the Gaussian pair mix on sm_100a. Standalone; not part of libgenred.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ unsigned long long g_clk[2], g_ns[2];
__device__ __forceinline__ unsigned long long gtimer(){unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;":"=l"(t)); return t;}
__device__ __forceinline__ float ex2f(float x){float y; asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(y):"f"(x)); return y;}

#define ITERS 4096
__global__ void __launch_bounds__(512,2) k_ffma(float* out, float b, float c){
  float a[8]; for(int k=0;k<8;k++) a[k]=threadIdx.x*1e-3f+k;
  if(blockIdx.x==0&&threadIdx.x==0){g_clk[0]=clock64(); g_ns[0]=gtimer();}
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=fmaf(a[k],b,c);
  }
  if(blockIdx.x==0&&threadIdx.x==0){g_clk[1]=clock64(); g_ns[1]=gtimer();}
  float s=0; for(int k=0;k<8;k++) s+=a[k]; if(s==1.2345f) out[0]=s;
}
__global__ void __launch_bounds__(512,2) k_ffma2(float* out, float b, float c){
  float2 a[8]; for(int k=0;k<8;k++) a[k]=make_float2(threadIdx.x*1e-3f+k, k*0.5f);
  float2 bb=make_float2(b,b*0.5f), cc=make_float2(c,c*0.25f);
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=__ffma2_rn(a[k],bb,cc);
  }
  float s=0; for(int k=0;k<8;k++) s+=a[k].x+a[k].y; if(s==1.2345f) out[0]=s;
}
__global__ void __launch_bounds__(512,2) k_fadd2(float* out, float b, float c){
  float2 a[8]; for(int k=0;k<8;k++) a[k]=make_float2(threadIdx.x*1e-3f+k, k*0.5f);
  float2 bb=make_float2(b,b*0.5f);
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=__fadd2_rn(a[k],bb);
  }
  float s=0; for(int k=0;k<8;k++) s+=a[k].x+a[k].y; if(s==1.2345f) out[0]=s;
}
__global__ void __launch_bounds__(512,2) k_mufu(float* out, float b, float c){
  float a[8]; for(int k=0;k<8;k++) a[k]=-(threadIdx.x*1e-3f+k);
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=-ex2f(a[k]);
  }
  float s=0; for(int k=0;k<8;k++) s+=a[k]; if(s==1.2345f) out[0]=s;
}
// Gaussian pair mix, direct form, FFMA2-packed over j-pairs; 4 rows x 2 j per step -> 8 pairs.
__global__ void __launch_bounds__(512,2) k_pair(float* out, float b, float c){
  float2 x0[4],x1[4],x2[4],acc[4];
  for(int r=0;r<4;r++){float v=threadIdx.x*1e-4f+r*0.1f; x0[r]=make_float2(v,v); x1[r]=make_float2(v*0.5f,v*0.5f); x2[r]=make_float2(v*0.25f,v*0.25f); acc[r]=make_float2(0,0);}
  float2 y0=make_float2(b,c), y1=make_float2(c,b), y2=make_float2(b*c,b), bw=make_float2(c,c);
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for(int r=0;r<4;r++){
      float2 d0=__fadd2_rn(x0[r],y0), d1=__fadd2_rn(x1[r],y1), d2=__fadd2_rn(x2[r],y2);
      float2 q=__fmul2_rn(d0,d0); q=__ffma2_rn(d1,d1,q); q=__ffma2_rn(d2,d2,q);
      float2 e=make_float2(ex2f(-q.x),ex2f(-q.y));
      acc[r]=__ffma2_rn(e,bw,acc[r]);
    }
    y0.x+=1e-7f; y1.y+=1e-7f; y2.x-=1e-7f;   // loop-carried so nothing hoists (3 extra FADD / 8 pairs)
  }
  float s=0; for(int r=0;r<4;r++) s+=acc[r].x+acc[r].y; if(s==1.2345f) out[0]=s;
}

template<typename K> int run(const char* name, K kern, double ops_per_thread_iter, int nsm){
  float* d; CK(cudaMalloc(&d,4));
  int blocks=nsm*2, threads=512;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks,threads>>>(d,0.999f,1e-3f); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); kern<<<blocks,threads>>>(d,0.999f,1e-3f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  unsigned long long clk[2],ns[2]; cudaMemcpyFromSymbol(clk,g_clk,16); cudaMemcpyFromSymbol(ns,g_ns,16);
  double total=ops_per_thread_iter*ITERS*(double)blocks*threads;
  printf("%-8s %9.3f ms  %.3e ops/s\n",name,ms,total/(ms*1e-3));
  cudaFree(d); return 0;
}
int main(){
  cudaDeviceProp p; cudaGetDeviceProperties(&p,0);
  printf("device %s SMs %d smem/SM %zu L2 %d clock(kHz) %d\n",p.name,p.multiProcessorCount,p.sharedMemPerMultiprocessor,p.l2CacheSize,p.clockRate);
  int n=p.multiProcessorCount;
  // measure clock with ffma kernel
  run("ffma",k_ffma,8,n);
  unsigned long long clk[2],ns[2]; cudaMemcpyFromSymbol(clk,g_clk,16); cudaMemcpyFromSymbol(ns,g_ns,16);
  double mhz=(double)(clk[1]-clk[0])/((double)(ns[1]-ns[0])*1e-3);
  printf("sm_clock_mhz_during_ffma %.1f\n",mhz);
  run("ffma2(lane-ops x2)",k_ffma2,16,n);
  run("fadd2(lane-ops x2)",k_fadd2,16,n);
  run("mufu.ex2",k_mufu,8,n);
  run("pair",k_pair,8,n);
  printf("divide ops/s by (%d SMs * clock) for per-clk/SM rates\n",n);
  return 0;
}
