#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
// throughput of FFMA, FFMA2 (fma.rn.f32x2), FHFMA (fma.rn.f32.bf16) per SM
template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  uint32_t xw = __float_as_uint(s) ^ threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {
        asm volatile("fma.rn.f32 %0, %0, %2, %3;\n\tfma.rn.f32 %1, %1, %2, %3;" : "+f"(a[i]), "+f"(a[i+1]) : "f"(s), "f"(a[15-i]));
      } else if (MODE == 1) {
        uint64_t p, w, c;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(a[i]), "f"(a[i+1]));
        asm volatile("mov.b64 %0, {%1, %1};" : "=l"(w) : "f"(s));
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(a[15-i]), "f"(a[14-i]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p) : "l"(w), "l"(c));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a[i]), "=f"(a[i+1]) : "l"(p));
      } else {
        asm volatile("{.reg .b16 xl, xh;\n\tmov.b32 {xl, xh}, %2;\n\tfma.rn.f32.bf16 %0, xl, xh, %0;\n\tfma.rn.f32.bf16 %1, xh, xl, %1;}" : "+f"(a[i]), "+f"(a[i+1]) : "r"(xw));
      }
    }
  }
  float t = 0; for (int i = 0; i < 16; ++i) t += a[i];
  if (t == 1234.5f) out[threadIdx.x] = t;
}
int main() {
  float* o; cudaMalloc(&o, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int mode = 0; mode < 3; ++mode) for (int threads : {256, 512, 1024}) {
    auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
    f<<<148, threads>>>(o, 100, 1.0001f);
    cudaEventRecord(e0);
    f<<<148, threads>>>(o, iters, 1.0001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double macs = 148.0 * threads * iters * 16;  // scalar MACs
    // fma.rn.f32x2 does 2 MACs per instr on 8 instrs x2 -> 16 MACs per it per thread as well
    if (mode == 1) macs *= 2;  // 8 f32x2 instrs per it = 16 MACs... adjust below
    printf("mode %d threads %d: %.3f ms, %.2f TMAC/s (per SM per clk @1.965: %.1f)\n", mode, threads, ms,
           (mode==1? macs/2 : macs) / ms / 1e9, (mode==1? macs/2: macs) / (ms*1e-3) / 148 / 1.965e9);
  }
  return 0;
}
