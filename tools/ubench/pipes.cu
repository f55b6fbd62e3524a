// Micro-benchmark: throughput/latency of FFMA, FFMA2, FADD2, FSETP+FSEL on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 d;asm volatile("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(d):"l"(a),"l"(b),"l"(c));return d;}
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 d;asm volatile("add.rn.f32x2 %0,%1,%2;":"=l"(d):"l"(a),"l"(b));return d;}
template<int MODE, int ILP>
__global__ void k(float* out, int iters, float s){
  float x[ILP]; u64 y[ILP];
  for(int i=0;i<ILP;i++){ x[i]=threadIdx.x*1e-3f+i; y[i]=((u64)__float_as_uint(x[i])<<32)|__float_as_uint(x[i]+1);}
  u64 sv = ((u64)__float_as_uint(s)<<32)|__float_as_uint(s);
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<ILP;i++){
      if(MODE==0) x[i]=__fmaf_rn(x[i],s,0.5f);
      if(MODE==1) y[i]=fma2(y[i],sv,y[(i+1)%ILP]);
      if(MODE==2) y[i]=add2(y[i],sv);
      if(MODE==3) x[i]= fabsf(x[i]) < fabsf(s) ? s : x[i]*0.999f;
      if(MODE==4) x[i]=__fadd_rn(x[i],s);
    }
  }
  float acc=0; for(int i=0;i<ILP;i++) acc+=x[i]+__uint_as_float((unsigned)y[i]);
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
template<int MODE,int ILP> void run(const char* name, float* d, int blocks, int threads){
  int iters=4096; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE,ILP><<<blocks,threads>>>(d,16,1.0001f);
  cudaEventRecord(a); k<MODE,ILP><<<blocks,threads>>>(d,iters,1.0001f); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  double ops=(double)blocks*threads*iters*ILP; // per-lane ops (FFMA2 counts 1 instr)
  printf("%-28s blocks=%5d thr=%4d : %8.1f G warp-instr/s per SM-cycle-ish: %.3f instr/clk/SM (at 1.9GHz)\n",name,blocks,threads, ops/32/ms/1e6, ops/32/(ms*1e-3)/148/1.9e9);
}
int main(){
  float* d; cudaMalloc(&d, 148*64*1024*4);
  for (int occ : {1, 4, 16}) {
    int blocks=148*occ, thr=128;
    printf("--- %d warps/SM\n", occ*4);
    run<0,8>("FFMA ilp8",d,blocks,thr);
    run<4,8>("FADD ilp8",d,blocks,thr);
    run<1,8>("FFMA2 ilp8",d,blocks,thr);
    run<2,8>("FADD2 ilp8",d,blocks,thr);
    run<3,8>("FSETP+FSEL+FMUL ilp8",d,blocks,thr);
    run<0,1>("FFMA ilp1 (latency)",d,blocks,thr);
    run<1,1>("FFMA2 ilp1 (latency)",d,blocks,thr);
  }
  return 0;
}
