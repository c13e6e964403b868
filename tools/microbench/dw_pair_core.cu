// Isolated column-pair DW core throughput: NW warps per CTA, 1 CTA/SM, each warp runs `iters`
// items over a 18x10x128B smem tile (bf16, 3x3 s1), storing to an A-layout smem buffer.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "common.cuh"
using namespace fcm;
template <int SEG, int SLOTS>
__global__ void k(int iters, uint32_t* out, int nw, int rowb, int maxr, int nvalid, int tw) {
  extern __shared__ uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  __syncthreads();
  uint64_t W[9];
  // per-lane weights (a lane owns its own channels, as in the kernels): not warp-uniform
  const float lf = 0.001f * (threadIdx.x & 31);
  for (int q = 0; q < 9; ++q) W[q] = f2_pack(0.1f * q + lf, 0.2f * q - lf);
  uint64_t bias = f2_pack(0.5f + lf, 0.25f - lf);
  const uint32_t xt = smem_u32(sm), ab = smem_u32(sm + 24 * 1024);
  const uint32_t hi2 = 0x40c040c0u;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int grp = SLOTS == 2 ? lane >> 4 : 0, wd = SLOTS == 2 ? lane & 15 : lane;
    const int x0 = 2 * ((warp + it) & 3), y0 = (((warp >> 2) & 1) * 2 + grp) % 2 * SEG;
    const uint32_t src = xt + ((0 * 10 + x0) * 32 + wd) * 4 + (SLOTS == 2 ? grp * 10 * 128 * SEG : 0);
    const uint32_t a0 = ab + (wd >> 2) * kAlbo + (wd & 3) * 4 + (uint32_t)(y0 * 8 + x0) * 16;
    const uint32_t dead = ab + 40000 + lane * 4;
    const bool c1 = x0 + 1 < tw;
    const uint32_t rstep = (uint32_t)tw * 16;
    dw3_pair<FCM_BF16, 1, SEG>(src, 128, rowb, y0, maxr, W, bias, [&](int r, uint64_t p0, uint64_t p1) {
      const uint32_t ad = a0 + r * rstep;
      const bool rok = r < nvalid;
      sts32(rok ? ad : dead, pack_act<FCM_BF16, 2>(p0, hi2));
      sts32(rok && c1 ? ad + 16 : dead, pack_act<FCM_BF16, 2>(p1, hi2));
    });
  }
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) out[warp] = (uint32_t)(t1 - t0);
}
int main() {
  uint32_t* o; cudaMallocManaged(&o, 64 * 4);
  for (int nw : {8, 16}) {
    int iters = 2000;
    auto run = [&](auto kern, int seg) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
      kern<<<148, nw * 32, 48 * 1024>>>(iters, o, nw, 10 * 128, 17, 16, 16);
      cudaDeviceSynchronize();
      double cyc = o[0];
      double words = (double)iters * seg * 2;  // per lane
      printf("SEG %2d warps %2d: %.1f cycles/item, %.2f cycles per word-row per warp; SM rate %.2f ch-px/clk (%s)\n",
             seg, nw, cyc / iters, cyc / words, nw * 32.0 * words * 2 / cyc, cudaGetErrorString(cudaGetLastError()));
    };
    run(k<8, 1>, 8);
    run(k<8, 2>, 8);
  }
}
