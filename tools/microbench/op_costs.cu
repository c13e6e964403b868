// Issue cost of the DW core's non-FMA instructions on B200, alone and interleaved 1:1 with FFMA2
// (fma.rn.f32x2): cycles per warp instruction per SM sub-partition (SMSP), 1024 threads per SM,
// 12 independent dependency chains per thread. Decides which ALU work the DW core can afford
// next to its FMAs.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b) {
  uint32_t d;
  if constexpr (OP == 0) asm volatile("prmt.b32 %0, %1, %2, 0x1044;" : "=r"(d) : "r"(a), "r"(b));
  if constexpr (OP == 1) asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  if constexpr (OP == 2) asm volatile("lop3.b32 %0, %1, %2, %1, 0x6a;" : "=r"(d) : "r"(a), "r"(b));
  if constexpr (OP == 3) asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.b32 %0, %1, %2, p;}" : "=r"(d) : "r"(a), "r"(b));
  if constexpr (OP == 4) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b)));
  if constexpr (OP == 5) asm volatile("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  if constexpr (OP == 6) asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  if constexpr (OP == 7) asm volatile("shl.b32 %0, %1, 16;" : "=r"(d) : "r"(a));
  if constexpr (OP == 8) asm volatile("and.b32 %0, %1, 0xFFFF0000;" : "=r"(d) : "r"(a));
  if constexpr (OP == 9) asm volatile("fma.rn.f32 %0, %1, %2, %1;" : "=f"(*reinterpret_cast<float*>(&d)) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b)));
  if constexpr (OP == 10) {
    float f = __uint_as_float(a);
    asm volatile("{.reg .b16 l, h; mov.b32 {l, h}, %1; fma.rn.f32.bf16 %0, l, h, %0;}" : "+f"(f) : "r"(b));
    d = __float_as_uint(f);
  }
  if constexpr (OP == 11) asm volatile("min.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  if constexpr (OP == 12) asm volatile("mov.b32 %0, %1;" : "=r"(d) : "r"(a));  // placeholder (usually elided)
  return d;
}

template <int OP, bool WITH_F2>
__global__ void k(int iters, const uint32_t* __restrict__ in, uint32_t* out) {
  const uint32_t t = threadIdx.x;
  uint32_t r[12];
  uint64_t acc[12], x;
  for (int i = 0; i < 12; ++i) {
    r[i] = in[(t * 13 + i) & 1023];
    acc[i] = ((uint64_t)in[(t + i * 7) & 1023] << 32) | in[(t * 3 + i) & 1023];
  }
  x = ((uint64_t)in[(t + 5) & 1023] << 32) | in[(t + 9) & 1023];
  const uint32_t b = in[(t * 11) & 1023];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      r[i] = op<OP>(r[i], b);
      if constexpr (WITH_F2) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(x), "l"(acc[(i + 5) % 12]));
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < 12; ++i) s ^= r[i] ^ (uint32_t)acc[i];
  if (s == 0x12345) out[t] = s;
}

int main() {
  uint32_t *o, *in;
  cudaMalloc(&o, 1 << 16);
  cudaMalloc(&in, 4096);
  uint32_t h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 0x3f800000u + i * 977u;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"PRMT", "IADD", "LOP3", "SETP+SEL", "F2FP cvt.bf16x2", "HMNMX2 max.bf16x2", "IMAD mul.lo",
                         "shl 16", "and 0xffff0000", "FFMA", "FHFMA fma.f32.bf16", "IMNMX min.s32"};
  auto run = [&](auto kern, const char* name, bool f2) {
    const int iters = 2000, threads = 1024;
    kern<<<148, threads>>>(10, in, o);
    cudaEventRecord(e0);
    kern<<<148, threads>>>(iters, in, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * 1.965e9;
    const double per_smsp_instr = (double)iters * 12 * (threads / 32) / 4;  // op instrs per SMSP
    printf("%-22s %-9s %.2f cycles per op (per SMSP)\n", name, f2 ? "+FFMA2" : "alone", cyc / per_smsp_instr);
  };
#define RUN(I)                             \
  run(k<I, false>, names[I], false);       \
  run(k<I, true>, names[I], true);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9) RUN(10) RUN(11)
  run(k<12, true>, "FFMA2 only (mov)", true);
  return 0;
}
