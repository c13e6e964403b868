// Feasibility of a tensor-core depthwise stage on sm_100a:
//  (1) tcgen05.mma kind::f16 SS issue rate for M = 128 and small N (a depthwise tap = X[128 px x 16 ch]
//      times a diagonal 16 x 16 weight block: 128 x 16 useful MACs per MMA), with A start addresses
//      shifted by whole 16-byte pixels and SBO = a halo-row pitch (not the 128 of a dense tile);
//  (2) tcgen05.ld 32x32b throughput (the DW result has to come back out of TMEM for the epilogue).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2404_19331_b200/csrc
//        -I ../../include --expt-relaxed-constexpr -o dw_mma_rate dw_mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "common.cuh"
using namespace fcm;

__device__ __forceinline__ uint64_t desc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}

// one thread issues ITER x 36 MMAs (M = 128, N, K = 16) into TMEM; cycles per MMA
__global__ void __launch_bounds__(128, 1) mma_rate(int N, int iters, int sbo, int shift, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 100 * 1024 / 16; i += blockDim.x) sts128(smem_u32(sm) + 16 * i, 0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc_rt(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  __syncthreads();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(1, 1, 128, N);
    const uint32_t abase = smem_u32(sm), bbase = smem_u32(sm) + 64 * 1024;
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const uint32_t aoff = ((tap / 3) * sbo + (tap % 3) * shift) + g * 2 * 8192;
          const uint64_t ad = desc_ns(abase + aoff, 8192, sbo);
          const uint64_t bd = desc_ns(bbase + (g * 9 + tap) * 512, 256, 128);
          mma_ss<MmaKind::F16>(tb + ((g * N) & 511), ad, bd, idesc, tap != 0 || it != 0);
        }
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_rt(tb, 512);
}

// Same, but the commit / wait is only every 8 iterations (pipelined issue)
__global__ void __launch_bounds__(128, 1) mma_rate_nowait(int N, int iters, int sbo, int shift, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 100 * 1024 / 16; i += blockDim.x) sts128(smem_u32(sm) + 16 * i, 0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc_rt(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  __syncthreads();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(1, 1, 128, N);
    const uint32_t abase = smem_u32(sm), bbase = smem_u32(sm) + 64 * 1024;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const uint32_t aoff = ((tap / 3) * sbo + (tap % 3) * shift) + g * 2 * 8192;
          const uint64_t ad = desc_ns(abase + aoff, 8192, sbo);
          const uint64_t bd = desc_ns(bbase + (g * 9 + tap) * 512, 256, 128);
          mma_ss<MmaKind::F16>(tb + (((it & 1) * 256 + g * N) & 511), ad, bd, idesc, tap != 0);
        }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_rt(tb, 512);
}

// TMEM -> registers: NW warps (warp w reads lane quadrant w % 4), x16 loads of 32 columns each
template <int X>
__global__ void __launch_bounds__(512, 1) tmem_ld_rate(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc_rt(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[16];
    const uint32_t col = ((it * 16) + (warp >> 2) * 128) & 511;
    if (X == 16) {
      tmem_ld16(tb + col, r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += r[i];
    } else {
      uint32_t q[32];
      tmem_ld32(tb + (col & ~31), q);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += q[i];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_rt(tslot, 512);
}


// Correctness of the formulation: output tile 16 rows x 8 cols (M = 128), 64 channels (4 groups of 16),
// 3x3 stride 1. X halo 18 x 10 pixels in the TMA SW128 layout ([pix][128 B], 16-B chunk c of pixel p at
// p*128 + ((c ^ (p & 7)) * 16)). Tap (dy, dx) = A view starting at pixel dy*10 + dx, SBO = 10*128 B.
// B(tap, g) = diag(w[tap][16g..16g+15]) as a 16 x 16 K-major no-swizzle operand (LBO 128, SBO 256).
// mode bit 0: set the descriptor's matrix base offset ((start >> 7) & 7).
__global__ void __launch_bounds__(128, 1) dw_mma_check(const uint16_t* x, const uint16_t* w, float* y, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* xs = sm;                 // 180 px * 128 B = 23040 B
  uint8_t* bs = sm + 24 * 1024;     // 9 taps * 4 groups * 512 B = 18 KB
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 180 * 8; i += blockDim.x) {
    const int p = i >> 3, c = i & 7;
    const uint4 v = reinterpret_cast<const uint4*>(x)[p * 8 + c];
    sts128(smem_u32(xs) + p * 128 + ((c ^ (p & 7)) * 16), v.x, v.y, v.z, v.w);
  }
  for (int i = threadIdx.x; i < 9 * 4 * 256; i += blockDim.x) {  // element (tap, g, n, k)
    const int t = i / 1024, g = (i / 256) & 3, n = (i / 16) & 15, k = i & 15;
    const uint16_t v = (n == k) ? w[t * 64 + g * 16 + n] : 0;
    const int off = (t * 4 + g) * 512 + (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
    *reinterpret_cast<uint16_t*>(bs + off) = v;
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc_rt(&tslot, 64);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(1, 1, 128, 16);
    for (int g = 0; g < 4; ++g)
      for (int t = 0; t < 9; ++t) {
        const uint32_t start = smem_u32(xs) + ((t / 3) * 10 + (t % 3)) * 128 + g * 32;
        uint64_t ad = 0;
        ad |= (uint64_t)((start >> 4) & 0x3FFF);
        ad |= (uint64_t)1 << 16;
        ad |= (uint64_t)(1280 >> 4) << 32;
        ad |= (uint64_t)1 << 46;
        if (mode & 1) ad |= (uint64_t)((start >> 7) & 7) << 49;
        ad |= (uint64_t)2 << 61;
        const uint64_t bd = desc_ns(smem_u32(bs) + (t * 4 + g) * 512, 128, 256);
        mma_ss<MmaKind::F16>(tb + g * 16, ad, bd, idesc, t != 0);
      }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[16];
  for (int g = 0; g < 4; ++g) {
    tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + g * 16, r);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) y[(warp * 32 + lane) * 64 + g * 16 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_rt(tb, 64);
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16); }
static float bf2f(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

static int run_check() {
  std::vector<uint16_t> hx(180 * 64), hw(9 * 64);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 32768.0f - 1.0f; };
  for (auto& v : hx) v = f2bf(rnd());
  for (auto& v : hw) v = f2bf(rnd());
  uint16_t *dx, *dw; float* dy;
  cudaMalloc(&dx, hx.size() * 2); cudaMalloc(&dw, hw.size() * 2); cudaMalloc(&dy, 128 * 64 * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(dw_mma_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dy, 0, 128 * 64 * 4);
    dw_mma_check<<<1, 128, 48 * 1024>>>(dx, dw, dy, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("check error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> hy(128 * 64);
    cudaMemcpy(hy.data(), dy, hy.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int c = 0; c < 64; ++c) {
        const int r = m / 8, q = m % 8;
        double ref = 0;
        for (int t = 0; t < 9; ++t) ref += (double)bf2f(hx[((r + t / 3) * 10 + q + t % 3) * 64 + c]) * bf2f(hw[t * 64 + c]);
        maxerr = fmax(maxerr, fabs(ref - hy[m * 64 + c]));
      }
    printf("dw-as-mma check, base offset %s: max abs err %.3g\n", mode ? "set" : "zero", maxerr);
  }
  return 0;
}

// Issue-cost check: the A / B descriptors of all 36 MMAs are a uniform base descriptor plus
// compile-time offsets (what a production kernel can do), so the lone issuing thread only adds
// immediates; NB = B operands per tap (N / 16 diag blocks)
template <int N, int SBO, bool SW>
__global__ void __launch_bounds__(128, 1) mma_rate_const(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 100 * 1024 / 16; i += blockDim.x) sts128(smem_u32(sm) + 16 * i, 0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc_rt(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  __syncthreads();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc(1, 1, 128, N);
    const uint32_t abase = smem_u32(sm), bbase = smem_u32(sm) + 64 * 1024;
    uint64_t a0 = 0;
    a0 |= (uint64_t)((abase >> 4) & 0x3FFF);
    a0 |= (uint64_t)1 << 16;
    a0 |= (uint64_t)(SBO >> 4) << 32;
    a0 |= (uint64_t)1 << 46;
    if (SW) a0 |= (uint64_t)2 << 61;
    const uint64_t b0 = desc_ns(bbase, 128, 256);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          constexpr int dummy = 0;
          const uint64_t ad = a0 + (uint64_t)((((tap / 3) * SBO + (tap % 3) * 128 + g * 32) >> 4) + dummy);
          const uint64_t bd = b0 + (uint64_t)(((g * 9 + tap) * 512) >> 4);
          mma_ss<MmaKind::F16>(tb + (((it & 1) * 256 + g * N) & 511), ad, bd, idesc, tap != 0);
        }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_rt(tb, 512);
}

template <int N, int SBO, bool SW>
static void run_const(unsigned long long* d, int iters) {
  unsigned long long h[148];
  cudaFuncSetAttribute(mma_rate_const<N, SBO, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 101 * 1024);
  mma_rate_const<N, SBO, SW><<<148, 128, 101 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[i];
  cyc /= 148.0 * iters * 36;
  printf("const-desc N=%3d sbo=%d sw128=%d: %.2f cyc/MMA (floor %.1f), useful diag MAC/clk/SM %.1f\n", N, SBO, (int)SW,
         cyc, 128.0 * N / 256, 128.0 * 16 / cyc);
}

int main() {
  run_check();
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  unsigned long long h[148];
  const int smem = 101 * 1024;
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_rate_nowait, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  run_const<16, 1280, true>(d, iters);
  run_const<16, 2304, true>(d, iters);
  run_const<16, 128, false>(d, iters);
  run_const<8, 1280, true>(d, iters);
  run_const<32, 1280, true>(d, iters);
  run_const<64, 1280, true>(d, iters);
  run_const<128, 1280, true>(d, iters);
  for (int pass = 0; pass < 2; ++pass)
    for (int N : {8, 16, 32, 64, 128, 256}) {
      for (int sbo_shift = 0; sbo_shift < 2; ++sbo_shift) {
        const int sbo = sbo_shift ? 160 : 128, shift = sbo_shift ? 16 : 0;
        if (pass == 0) mma_rate<<<148, 128, smem>>>(N, iters, sbo, shift, d);
        else mma_rate_nowait<<<148, 128, smem>>>(N, iters, sbo, shift, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < 148; ++i) cyc += h[i];
        cyc /= 148.0 * iters * 36;
        printf("%s N=%3d sbo=%d shift=%d: %.2f cyc/MMA (floor %.1f), useful diag MAC/clk/SM %.1f\n",
               pass ? "pipelined" : "wait/36  ", N, sbo, shift, cyc, 128.0 * N / 256, 128.0 * 16 / cyc);
      }
    }
  for (int nw : {4, 8, 16}) {
    for (int x : {16, 32}) {
      if (x == 16) tmem_ld_rate<16><<<148, nw * 32>>>(4000, d, sink);
      else tmem_ld_rate<32><<<148, nw * 32>>>(4000, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i];
      cyc /= 148.0;
      const double bytes = 4000.0 * nw * 32 * x * 4;
      printf("tmem ld x%d, %2d warps: %.1f B/clk/SM\n", x, nw, bytes / cyc);
    }
  }
  return 0;
}
