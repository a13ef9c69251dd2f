// Step-0 probe #2: MUFU.EX2 rate and FFMA2 issue cost by operand pattern, and their overlap.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
__device__ __forceinline__ float ex2f(float x){float y; asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(y):"f"(x)); return y;}
#define IT 32768
// MUFU only: 8 independent chains
__global__ void __launch_bounds__(256,3) k_mufu(float* out, float s){
  float a[8]; for(int k=0;k<8;k++) a[k]=-(threadIdx.x*1e-4f+k*0.01f);
  for(int i=0;i<IT;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=-ex2f(a[k]*s);
  }
  float t=0; for(int k=0;k<8;k++) t+=a[k]; if(t==1.2345f) out[0]=t;
}
// MUFU only, no FMUL in the chain (negation folded): a = ex2(-a)
__global__ void __launch_bounds__(256,3) k_mufu2(float* out, float s){
  float a[8]; for(int k=0;k<8;k++) a[k]=(threadIdx.x*1e-4f+k*0.01f)*s;
  for(int i=0;i<IT;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=ex2f(-a[k]);
  }
  float t=0; for(int k=0;k<8;k++) t+=a[k]; if(t==1.2345f) out[0]=t;
}
// FFMA2 with three distinct register pairs (no reuse): a_k = fma(a_k, b_k, c_k)
__global__ void __launch_bounds__(256,3) k_ffma2_3reg(float* out, float s){
  float2 a[6], b[6], c[6];
  for(int k=0;k<6;k++){ a[k]=make_float2(threadIdx.x*1e-4f+k, k*0.5f); b[k]=make_float2(s*k, s); c[k]=make_float2(s, s*0.5f*k);}
  for(int i=0;i<IT;i++){
    #pragma unroll
    for(int k=0;k<6;k++) a[k]=__ffma2_rn(a[k], b[k], c[k]);
    #pragma unroll
    for(int k=0;k<6;k++) c[k]=__ffma2_rn(c[k], b[(k+1)%6], a[k]);
  }
  float t=0; for(int k=0;k<6;k++) t+=a[k].x+a[k].y+c[k].x; if(t==1.2345f) out[0]=t;
}
// FFMA2 with a broadcast SCALAR first operand and two register pairs (the row-pair loops'
// accumulation pattern: acc_k = fma2(e_k pair, scalar, acc_k))
__global__ void __launch_bounds__(256,3) k_ffma2_scalar(float* out, float s){
  float2 a[6], c[6]; float b[6];
  for(int k=0;k<6;k++){ a[k]=make_float2(threadIdx.x*1e-4f+k, k*0.5f); b[k]=s*k; c[k]=make_float2(s, s*0.5f*k);}
  for(int i=0;i<IT;i++){
    #pragma unroll
    for(int k=0;k<6;k++) a[k]=__ffma2_rn(c[k], make_float2(b[k],b[k]), a[k]);
    #pragma unroll
    for(int k=0;k<6;k++) c[k]=__ffma2_rn(a[k], make_float2(b[(k+1)%6],b[(k+1)%6]), c[k]);
  }
  float t=0; for(int k=0;k<6;k++) t+=a[k].x+a[k].y+c[k].x; if(t==1.2345f) out[0]=t;
}
// FFMA2 with an immediate third operand: a_k = fma(a_k, b_k, imm)
__global__ void __launch_bounds__(256,3) k_ffma2_imm(float* out, float s){
  float2 a[8], b[8];
  for(int k=0;k<8;k++){ a[k]=make_float2(threadIdx.x*1e-4f+k, k*0.5f); b[k]=make_float2(s*k*0.1f, s*0.3f);}
  for(int i=0;i<IT;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=__ffma2_rn(a[k], b[k], make_float2(0.25f,0.25f));
  }
  float t=0; for(int k=0;k<8;k++) t+=a[k].x+a[k].y; if(t==1.2345f) out[0]=t;
}
// FFMA (scalar) three distinct registers
__global__ void __launch_bounds__(256,3) k_ffma_3reg(float* out, float s){
  float a[8], b[8], c[8];
  for(int k=0;k<8;k++){ a[k]=threadIdx.x*1e-4f+k; b[k]=s*k; c[k]=s*0.5f*k;}
  for(int i=0;i<IT;i++){
    #pragma unroll
    for(int k=0;k<8;k++) a[k]=fmaf(a[k], b[k], c[k]);
    #pragma unroll
    for(int k=0;k<8;k++) c[k]=fmaf(c[k], b[(k+1)%8], a[k]);
  }
  float t=0; for(int k=0;k<8;k++) t+=a[k]+c[k]; if(t==1.2345f) out[0]=t;
}
// mix: per 2 values: 4 FFMA2 (imm form) + 2 MUFU  (FP32 lane-ops 8 : exps 2 -> ratio 4:1)
__global__ void __launch_bounds__(256,3) k_mix(float* out, float s){
  float2 a[4]; float m[8];
  for(int k=0;k<4;k++) a[k]=make_float2(threadIdx.x*1e-4f+k, k*0.5f);
  for(int k=0;k<8;k++) m[k]=(threadIdx.x*1e-4f+k*0.01f)*s;
  for(int i=0;i<IT;i++){
    #pragma unroll
    for(int k=0;k<4;k++){
      a[k]=__ffma2_rn(a[k], make_float2(s,s), make_float2(0.25f,0.25f));
      a[k]=__ffma2_rn(a[k], make_float2(0.5f,0.5f), make_float2(s,0.125f));
      a[k]=__ffma2_rn(a[k], make_float2(s,s), make_float2(0.25f,0.25f));
      a[k]=__ffma2_rn(a[k], make_float2(0.5f,0.5f), make_float2(s,0.125f));
      m[2*k]=ex2f(-m[2*k]); m[2*k+1]=ex2f(-m[2*k+1]);
    }
  }
  float t=0; for(int k=0;k<4;k++) t+=a[k].x+a[k].y+m[2*k]+m[2*k+1]; if(t==1.2345f) out[0]=t;
}
template<typename K> int run(const char* name, K kern, double ops_per_iter, int nsm, const char* unit){
  float* d; CK(cudaMalloc(&d,4));
  int blocks=nsm*3*4, threads=256;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks,threads>>>(d,0.999f); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); kern<<<blocks,threads>>>(d,0.999f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double total=ops_per_iter*IT*(double)blocks*threads;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-14s %9.3f ms  %.4e %s/s  = %.2f %s/clk/SM at max clock\n",name,ms,total/(ms*1e-3),unit,total/(ms*1e-3)/(nsm*clk*1e3),unit);
  cudaFree(d); return 0;
}
int main(){
  cudaDeviceProp p; cudaGetDeviceProperties(&p,0);
  int n=p.multiProcessorCount;
  run("mufu(+fmul)",k_mufu,8,n,"ex2");
  run("mufu",k_mufu2,8,n,"ex2");
  run("ffma2_3reg",k_ffma2_3reg,24,n,"lane-fma");
  run("ffma2_imm",k_ffma2_imm,16,n,"lane-fma");
  run("ffma2_scalar+2pairs",k_ffma2_scalar,24,n,"lane-fma");
  run("ffma_3reg",k_ffma_3reg,16,n,"lane-fma");
  run("mix 4ffma2:2mufu",k_mix,8,n,"ex2");
  return 0;
}
