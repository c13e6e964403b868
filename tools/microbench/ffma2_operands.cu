// FFMA2 (fma.rn.f32x2) issue model on B200: MAC/clk/SM for packed FMAs whose operands come from
// vector registers, a uniform register (warp-uniform weight) or the reuse cache, with and without
// interleaved ALU byte permutes (the bf16 -> fp32 widening of the DW core). Answers: what bounds
// the DW core at ~7.5 channel-pixels/clk/SM (53 % of the FMA pipe)?
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void f2(uint64_t& d, uint64_t a, uint64_t b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ uint32_t prmt(uint32_t x, uint32_t sel) {
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "n"(0x1044));
  return r;
}

// MODE 0: a, b, c all vector; 12 accumulators, 4 x values, 3 w values (per-lane)
// MODE 1: b warp-uniform (loop-invariant from params -> uniform / constant operand)
// MODE 2: as 0 + 1 PRMT per FFMA2
// MODE 3: as 0 + 2 PRMT per FFMA2 (the DW core's widening ratio is ~0.55 PRMT per FFMA2)
// MODE 4: as 1 + 1 PRMT per FFMA2
// MODE 5: as 0 but each w used by 4 back-to-back FFMA2 (reuse-cache friendly)
struct P {
  uint64_t w[16];
};
template <int MODE>
__global__ void k(const __grid_constant__ P p, int iters, uint64_t* out) {
  uint64_t acc[12], x[4], w[3];
  const uint32_t t = threadIdx.x;
  for (int i = 0; i < 12; ++i) acc[i] = (uint64_t)(t + i) * 0x3f8000003f800000ull;
  for (int i = 0; i < 4; ++i) x[i] = 0x3f8000013f800001ull + t * i;
  for (int i = 0; i < 3; ++i) w[i] = (MODE == 1 || MODE == 4) ? p.w[i] : 0x3f7fffff3f7fffffull ^ (t << 3) ^ i;
  uint32_t r = t * 2654435761u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const int xi = (MODE == 5) ? (i & 3) : (i % 4), wi = (MODE == 5) ? (i >> 2) : (i % 3);
      f2(acc[i], x[xi], w[wi]);
      if (MODE == 2 || MODE == 3 || MODE == 4) r = prmt(r, 0) ^ (uint32_t)i;
      if (MODE == 3) r = prmt(r, 0) + 1u;
    }
  }
  uint64_t s = r;
  for (int i = 0; i < 12; ++i) s ^= acc[i];
  if (s == 0x1234) out[t] = s;
}

int main() {
  uint64_t* o;
  cudaMalloc(&o, 1 << 16);
  P p;
  for (int i = 0; i < 16; ++i) p.w[i] = 0x3f7ff0003f7ff000ull + i;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"3 vector operands", "uniform weight operand", "vector + 1 PRMT/FFMA2",
                         "vector + 2 PRMT/FFMA2", "uniform + 1 PRMT/FFMA2", "vector, weight reused x4"};
  auto run = [&](auto kern, int mode) {
    for (int threads : {256, 512, 1024}) {
      const int iters = 4000;
      kern<<<148, threads>>>(p, 10, o);
      cudaEventRecord(e0);
      kern<<<148, threads>>>(p, iters, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double macs = 148.0 * threads * iters * 12 * 2;
      printf("mode %d %-28s threads %4d: %.1f MAC/clk/SM @1.965 GHz\n", mode, names[mode], threads,
             macs / (ms * 1e-3) / 148 / 1.965e9);
    }
  };
  run(k<0>, 0);
  run(k<1>, 1);
  run(k<2>, 2);
  run(k<3>, 3);
  run(k<4>, 4);
  run(k<5>, 5);
  return 0;
}
