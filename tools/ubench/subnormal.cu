// Do packed f32x2 ops preserve subnormals like their scalar forms?
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void k(const float* in, float* out) {
  float a = in[0], b = in[1], c = in[2];
  u64 A = ((u64)__float_as_uint(a) << 32) | __float_as_uint(a);
  u64 B = ((u64)__float_as_uint(b) << 32) | __float_as_uint(b);
  u64 Cc = ((u64)__float_as_uint(c) << 32) | __float_as_uint(c);
  u64 r1, r2, r3;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r1) : "l"(A), "l"(B));
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r2) : "l"(A), "l"(B), "l"(Cc));
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r3) : "l"(A), "l"(B));
  out[0] = __uint_as_float((unsigned)r1); out[1] = __fadd_rn(a, b);
  out[2] = __uint_as_float((unsigned)r2); out[3] = __fmaf_rn(a, b, c);
  out[4] = __uint_as_float((unsigned)r3); out[5] = __fmul_rn(a, b);
}
int main() {
  float cases[][3] = {{1e-39f, 2e-39f, 0.f}, {3e-39f, 1.0f, 1e-39f}, {2.35e-38f, -1e-39f, 0.f}, {1e-39f, 0.5f, 0.f}};
  float *din, *dout; cudaMalloc(&din, 12); cudaMalloc(&dout, 24);
  for (auto& cs : cases) {
    float out[6]; cudaMemcpy(din, cs, 12, cudaMemcpyHostToDevice);
    k<<<1,1>>>(din, dout); cudaMemcpy(out, dout, 24, cudaMemcpyDeviceToHost);
    printf("a=%g b=%g c=%g | add2 %g add %g | fma2 %g fma %g | mul2 %g mul %g\n", cs[0], cs[1], cs[2], out[0], out[1], out[2], out[3], out[4], out[5]);
  }
  return 0;
}
