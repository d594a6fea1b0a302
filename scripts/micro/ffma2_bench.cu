// Microbenchmark: FFMA (scalar, const operand) vs FFMA2 (packed f32x2) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
struct P { float c[64]; unsigned long long c2[64]; };
template <int MODE>
__global__ void k(float* out, const __grid_constant__ P p, int iters) {
  float a[16]; unsigned long long b[8];
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 1e-7f + i;
  for (int i = 0; i < 8; i++) b[i] = ((unsigned long long)__float_as_uint(a[2*i]) << 32) | __float_as_uint(a[2*i+1]);
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int j = 0; j < 16; j++) {
      if (MODE == 0) {
        #pragma unroll
        for (int i = 0; i < 16; i++) a[i] = fmaf(a[i], p.c[j], p.c[j + 16]);
      } else if (MODE == 1) {
        #pragma unroll
        for (int i = 0; i < 8; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(b[i]) : "l"(p.c2[j]), "l"(p.c2[j + 16]));
      } else {
        #pragma unroll
        for (int i = 0; i < 16; i++) a[i] = fmaf(a[i], a[(i + 1) & 15], a[(i + 3) & 15]);
      }
    }
  }
  float s = 0; for (int i = 0; i < 16; i++) s += a[i];
  for (int i = 0; i < 8; i++) s += __uint_as_float((unsigned)b[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  P p; for (int i = 0; i < 64; i++) { p.c[i] = 0.999f; p.c2[i] = 0x3f7fbe773f7fbe77ull; }
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int iters = 2000; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"FFMA c[] operand", "FFMA2 (f32x2) UR operands", "FFMA 3-reg"};
  for (int mode = 0; mode < 3; mode++) for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    if (mode == 0) k<0><<<148 * 8, 256>>>(out, p, iters);
    if (mode == 1) k<1><<<148 * 8, 256>>>(out, p, iters);
    if (mode == 2) k<2><<<148 * 8, 256>>>(out, p, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = 148.0 * 8 * 256 * iters * 16 * 16;  // FMA operations (FFMA2 counts 2)
    if (rep) printf("%-28s %8.3f ms  %7.2f TFMA/s  (%6.1f TFLOP/s)\n", names[mode], ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  return 0;
}
