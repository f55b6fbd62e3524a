// Pipe-mix micro-benchmark on sm_100a: which instruction mixes dual-issue.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 d;asm volatile("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(d):"l"(a),"l"(b),"l"(c));return d;}
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 d;asm volatile("add.rn.f32x2 %0,%1,%2;":"=l"(d):"l"(a),"l"(b));return d;}
__device__ __forceinline__ float fsel_abs(float l, float r){float d; asm volatile("{.reg .pred p; setp.lt.f32 p, %1, %2; selp.f32 %0, %3, %4, p;}":"=f"(d):"f"(fabsf(r)),"f"(fabsf(l)),"f"(r),"f"(l)); return d;}
template<int MODE>
__global__ void k(float* out, int iters, float s){
  const int ILP=8;
  u64 y[ILP]; float x[ILP];
  for(int i=0;i<ILP;i++){ x[i]=threadIdx.x*1e-3f+i; y[i]=((u64)__float_as_uint(x[i])<<32)|__float_as_uint(x[i]+1);}
  u64 sv = ((u64)__float_as_uint(s)<<32)|__float_as_uint(s);
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<ILP;i++){
      if(MODE==0){ y[i]=fma2(y[i],sv,sv); }                                   // FFMA2 only
      if(MODE==1){ y[i]=fma2(y[i],sv,sv); y[(i+4)%ILP]=add2(y[(i+4)%ILP],sv);} // FFMA2+FADD2
      if(MODE==2){ y[i]=fma2(y[i],sv,sv); x[i]=fsel_abs(x[i], s);}            // FFMA2+FSETP/FSEL
      if(MODE==3){ x[i]=fsel_abs(x[i], s);}                                   // FSETP/FSEL only
      if(MODE==4){ y[i]=fma2(y[i],sv,sv); x[i]=__fmaf_rn(x[i],s,0.5f);}       // FFMA2+FFMA
      if(MODE==5){ y[i]=add2(y[i],sv); x[i]=fsel_abs(x[i], s);}               // FADD2+FSETP/FSEL
    }
  }
  float acc=0; for(int i=0;i<ILP;i++) acc+=x[i]+__uint_as_float((unsigned)y[i]);
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
template<int MODE> void run(const char* name, float* d){
  int blocks=148*16, thr=128, iters=2048;
  k<MODE><<<blocks,thr>>>(d,16,1.0001f);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<MODE><<<blocks,thr>>>(d,iters,1.0001f); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double iterations=(double)blocks*thr/32*iters*8; // per-warp loop bodies x ILP
  double cyc=ms*1e-3*1.92e9*148*4; // SMSP-cycles (assume 1.92 GHz)
  printf("%-24s %.3f SMSP-cycles per (warp x element)\n",name, cyc/iterations);
}
int main(){ float* d; cudaMalloc(&d, 148*16*128*4);
  run<0>("FFMA2",d); run<1>("FFMA2+FADD2",d); run<2>("FFMA2+FSETP/FSEL",d); run<3>("FSETP/FSEL",d);
  run<4>("FFMA2+FFMA",d); run<5>("FADD2+FSETP/FSEL",d); return 0; }
