// TMA 4-D halo-box load throughput: 1 producer thread per CTA, ring of S stages, a consumer warp
// that releases each stage as soon as it lands. grid = 148 persistent CTAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"
using namespace fcm;
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap tm, int S, int bytes, int ntile, int tx, int ty,
                                            int nchunk, int th, int tw, int halo) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + S * ((bytes + 1023) & ~1023));
  uint64_t* empty = full + S;
  const int stride = (bytes + 1023) & ~1023;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int total = ntile * nchunk;
  if (threadIdx.x == 0) {
    int it = 0;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x)
      for (int kc = 0; kc < nchunk; ++kc, ++it) {
        int s = it % S;
        mbar_wait(empty + s, ((it / S) & 1) ^ 1);
        mbar_arrive_expect_tx(full + s, bytes);
        int txi = t % tx, r = t / tx, tyi = r % ty, n = r / ty;
        tma_load_4d(sm + s * stride, &tm, full + s, kc * 64, txi * tw - halo, tyi * th - halo, n);
      }
  } else if (threadIdx.x == 32) {
    int it = 0;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x)
      for (int kc = 0; kc < nchunk; ++kc, ++it) {
        int s = it % S;
        mbar_wait(full + s, (it / S) & 1);
        mbar_arrive(empty + s);
      }
  }
  (void)total;
}
int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc = (PFN)p;
  struct Cfg { const char* name; int N, H, W, C, th, tw, k; };
  std::vector<Cfg> cfgs = {{"b0 112x112x32 16x8", 256, 112, 112, 32, 16, 8, 3},
                           {"b0 as C=64 tensor", 128, 112, 112, 64, 16, 8, 3},
                           {"b11 14x14x576 14x7", 256, 14, 14, 576, 14, 7, 3},
                           {"b5 28x28x192 14x7", 256, 28, 28, 192, 14, 7, 3},
                           {"b5 28x28x192 14x8", 256, 28, 28, 192, 14, 8, 3},
                           {"56x56x144 14x8", 256, 56, 56, 144, 14, 8, 3},
                           {"56x56x144 8x16", 256, 56, 56, 144, 8, 16, 3},
                           {"56x56x128 no halo 8x16", 256, 56, 56, 128, 8, 16, 1}};
  for (auto& c : cfgs) {
    size_t elems = (size_t)c.N * c.H * c.W * c.C;
    void* x; cudaMalloc(&x, elems * 2); cudaMemset(x, 0, elems * 2);
    int thi = c.th + c.k - 1, twi = c.tw + c.k - 1;
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)c.C, (cuuint64_t)c.W, (cuuint64_t)c.H, (cuuint64_t)c.N};
    cuuint64_t str[3] = {(cuuint64_t)c.C * 2, (cuuint64_t)c.W * c.C * 2, (cuuint64_t)c.H * c.W * c.C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)twi, (cuuint32_t)thi, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); continue; }
    int bytes = thi * twi * 128;
    int tx = (c.W + c.tw - 1) / c.tw, ty = (c.H + c.th - 1) / c.th, nt = tx * ty * c.N, nch = (c.C + 63) / 64;
    for (int S : {2, 4, 8}) {
      int smem = S * ((bytes + 1023) & ~1023) + 2048;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k<<<148, 64, smem>>>(tm, S, bytes, nt, tx, ty, nch, c.th, c.tw, c.k / 2);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i) k<<<148, 64, smem>>>(tm, S, bytes, nt, tx, ty, nch, c.th, c.tw, c.k / 2);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      double real = (double)elems * 2;  // compulsory bytes
      double fill = (double)nt * nch * bytes;
      printf("%-26s S=%d box %dx%dx128B: %.1f us  compulsory %.0f GB/s  smem-fill %.0f GB/s  err=%s\n", c.name, S, thi, twi,
             ms * 1e3, real / ms / 1e6, fill / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(x);
  }
}
