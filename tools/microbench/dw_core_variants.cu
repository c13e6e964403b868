// DW-core variants for the bf16 3x3 s1 DWPW producer stage (round 2): channel-pixels per clock
// per SM on an smem-resident X tile, each warp running `iters` items and storing the packed
// (RELU6) results to an smem A buffer, 1 CTA per SM, NW warps.
//   V0  current `dw3_pair`: lane = 32-bit channel word, 2 output columns, per-lane fp32 weights
//       (three vector 64-bit FFMA2 operands)
//   V1  lane = channel word, 4 output columns: each weight operand is reused by 4 FFMA2s back to back
//   V2  lane = output pixel, a warp owns one 8-channel octet (TMA inner box = 16 B): 3 LDS.128 per
//       input row, the fp32 weights come from the kernel-parameter constant bank at a warp-uniform
//       index (LDCU -> uniform-register FFMA2 operand)
//   V3  dw3_cols_h, 2 columns: lane = channel word, mixed FHFMA taps straight from the packed words
//       (no bf16 -> fp32 widening), scale / bias / RELU6 in the sink
//   V4  dw3_cols_h, 4 columns
//   V6  V5 with a CTA barrier after every item (all DW warps in lock-step, as in the kernel's
//       C_in-chunk phases)
//   V5  V3 with the kernel's runtime geometry: row pitch and output row step are kernel arguments,
//       stores predicated per item (as in dwpw_tc_kernel)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include "common.cuh"
using namespace fcm;

struct WP {
  uint64_t w[8 * 4 * 10];  // [octet][word][9 taps + bias] fp32 pairs
};

template <int SEG>
__device__ __forceinline__ void quad_core(uint32_t src, int row_bytes, const uint64_t (&W)[9], uint64_t bias,
                                          uint32_t a0, uint32_t rstep, uint32_t hi2) {
  constexpr int NCW = 6, WR = SEG + 2;
  uint64_t acc[SEG][4];
#pragma unroll
  for (int ii = 0; ii < WR; ++ii) {
    uint64_t x[NCW];
#pragma unroll
    for (int j = 0; j < NCW; ++j) x[j] = word_to_f2<FCM_BF16>(lds32(src + ii * row_bytes + j * 128));
#pragma unroll
    for (int r = 0; r < SEG; ++r) {
      const int i = ii - r;
      if (i < 0 || i > 2) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = f2_fma(x[c + j], W[i * 3 + j], (i == 0 && j == 0) ? bias : acc[r][c]);
      if (i == 2) {
#pragma unroll
        for (int c = 0; c < 4; ++c) sts32(a0 + r * rstep + c * 16, pack_act<FCM_BF16, 2>(acc[r][c], hi2));
      }
    }
  }
}

template <int V, int SEG>
__global__ void k(const __grid_constant__ WP wp, int iters, uint32_t* out, int rb = 40 * 128, int maxr = 19,
                  int rstep = 512, int nvalid_rt = 64) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u ^ ((i * 2654435761u) & 0x00ff00ffu);
  __syncthreads();
  const uint32_t xt = smem_u32(sm), ab = smem_u32(sm + 120 * 1024);
  const uint32_t hi2 = 0x40c040c0u;
  const float lf = 0.001f * lane;
  long long t0 = clock64();
  if constexpr (V == 5 || V == 6) {
    uint32_t W[9];
    for (int q = 0; q < 9; ++q) W[q] = 0x3dcc3dccu + q * 0x00010001u + lane;
    const uint64_t sc2 = f2_pack(1.0f + lf, 0.9f - lf), bi2 = f2_pack(0.5f + lf, 0.25f - lf);
    for (int it = 0; it < iters; ++it) {
      const int x0 = 2 * ((warp + it) & 7), y0 = SEG > 8 ? 0 : ((warp >> 3) + it) & 1;
      const uint32_t src = xt + ((y0 * 40 + x0) * 32 + lane) * 4;
      const uint32_t a0 = ab + (lane >> 2) * kAlbo + (lane & 3) * 4 + (uint32_t)(y0 * 32 + x0) * 16;
      const int nvalid = nvalid_rt - y0;
      const bool c1 = x0 + 1 < 40;
      dw3_cols_h<FCM_BF16, 1, SEG, 2, 128>(src, rb, W, [&](int r, int c, float lo, float hi) {
        const uint32_t v = epi_act2<FCM_BF16, 2>(lo, hi, sc2, bi2, hi2);
        if (c == 0 ? nvalid > 0 : c1) sts32(a0 + r * rstep + c * 16, v);
      });
      if constexpr (V == 6) __syncthreads();
    }
  } else if constexpr (V == 3 || V == 4) {
    constexpr int NC = V == 3 ? 2 : 4;
    uint32_t W[9];
    for (int q = 0; q < 9; ++q) W[q] = 0x3dcc3dccu + q * 0x00010001u + lane;
    const uint64_t sc2 = f2_pack(1.0f + lf, 0.9f - lf), bi2 = f2_pack(0.5f + lf, 0.25f - lf);
    for (int it = 0; it < iters; ++it) {
      const int x0 = NC * ((warp + it) & 7), y0 = SEG > 8 ? 0 : ((warp >> 3) + it) & 1;
      const uint32_t src = xt + ((y0 * 40 + x0) * 32 + lane) * 4;
      const uint32_t a0 = ab + (lane >> 2) * kAlbo + (lane & 3) * 4 + (uint32_t)(y0 * 32 + x0) * 16;
      dw3_cols_h<FCM_BF16, 1, SEG, NC, 128>(src, 40 * 128, W, [&](int r, int c, float lo, float hi) {
        sts32(a0 + r * 512 + c * 16, epi_act2<FCM_BF16, 2>(lo, hi, sc2, bi2, hi2));
      });
    }
  } else if constexpr (V == 0 || V == 1) {
    uint64_t W[9];
    for (int q = 0; q < 9; ++q) W[q] = f2_pack(0.1f * q + lf, 0.2f * q - lf);
    const uint64_t bias = f2_pack(0.5f + lf, 0.25f - lf);
    // X tile [rows 20][cols 40][32 words]
    for (int it = 0; it < iters; ++it) {
      const int x0 = (V == 0 ? 2 : 4) * ((warp + it) & 7), y0 = SEG > 8 ? 0 : ((warp >> 3) + it) & 1;
      const uint32_t src = xt + ((y0 * 40 + x0) * 32 + lane) * 4;
      const uint32_t a0 = ab + (lane >> 2) * kAlbo + (lane & 3) * 4 + (uint32_t)(y0 * 32 + x0) * 16;
      if constexpr (V == 0) {
        dw3_pair<FCM_BF16, 1, SEG>(src, 128, 40 * 128, y0, 19, W, bias, [&](int r, uint64_t p0, uint64_t p1) {
          sts32(a0 + r * 512, pack_act<FCM_BF16, 2>(p0, hi2));
          sts32(a0 + r * 512 + 16, pack_act<FCM_BF16, 2>(p1, hi2));
        });
      } else {
        quad_core<SEG>(src, 40 * 128, W, bias, a0, 512, hi2);
      }
    }
  } else {
    // X tile per octet: [oct 8][rows 12][cols 40][16 B] = 61 KB. All input rows of the item are
    // loaded once (3 shifted LDS.128 per row); the 4 words of the octet are then processed one at a
    // time so that only that word's 10 weight pairs occupy uniform registers.
    constexpr int WR = SEG + 2;
    for (int it = 0; it < iters; ++it) {
      const int oct = it & 7;  // warp-uniform by construction (loop counter)
      const int y0 = (it >> 3) & 1;
      const uint32_t src = xt + ((oct * 12 + y0) * 40 + lane) * 16;
      const uint32_t a0 = ab + (oct & 1) * 8 * kAlbo + (uint32_t)(y0 * 32 + lane) * 16;
      uint32_t raw[WR][3][4];
#pragma unroll
      for (int ii = 0; ii < WR; ++ii)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const uint4 q = lds128(src + ii * 40 * 16 + j * 16);
          raw[ii][j][0] = q.x; raw[ii][j][1] = q.y; raw[ii][j][2] = q.z; raw[ii][j][3] = q.w;
        }
      uint32_t packed[SEG][4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint64_t* W = wp.w + (oct * 4 + w) * 10;
        uint64_t acc[SEG];
#pragma unroll
        for (int ii = 0; ii < WR; ++ii) {
          uint64_t x[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) x[j] = word_to_f2<FCM_BF16>(raw[ii][j][w]);
#pragma unroll
          for (int r = 0; r < SEG; ++r) {
            const int i = ii - r;
            if (i < 0 || i > 2) continue;
#pragma unroll
            for (int j = 0; j < 3; ++j) acc[r] = f2_fma(x[j], W[i * 3 + j], (i == 0 && j == 0) ? W[9] : acc[r]);
            if (i == 2) packed[r][w] = pack_act<FCM_BF16, 2>(acc[r], hi2);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < SEG; ++r) sts128(a0 + r * 512, packed[r][0], packed[r][1], packed[r][2], packed[r][3]);
    }
  }
  long long t1 = clock64();
  if (lane == 0) atomicMax(out + warp, (uint32_t)(t1 - t0));
}

int main() {
  uint32_t* o;
  cudaMallocManaged(&o, 64 * 4);
  WP wp;
  for (int i = 0; i < 8 * 4 * 10; ++i) {
    float a = 0.01f * (i % 37), b = -0.02f * (i % 11);
    uint32_t ua, ub; memcpy(&ua, &a, 4); memcpy(&ub, &b, 4);
    wp.w[i] = (uint64_t)ua | ((uint64_t)ub << 32);
  }
  auto run = [&](auto kern, const char* name, int nw, double chpx_per_item) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 1024;
    for (int rep = 0; rep < 2; ++rep) {
      for (int i = 0; i < 64; ++i) o[i] = 0;
      kern<<<148, nw * 32, 160 * 1024>>>(wp, iters, o, 40 * 128, 19, 512, 64);
      cudaError_t e = cudaDeviceSynchronize();
      double cyc = 0;
      for (int w = 0; w < nw; ++w) cyc = cyc > o[w] ? cyc : o[w];
      if (rep == 1)
        printf("%-34s warps %2d: %8.0f cycles, %.1f cycles/item, SM rate %.2f ch-px/clk (%s)\n", name, nw, cyc,
               cyc / iters, nw * chpx_per_item * iters / cyc, cudaGetErrorString(e));
    }
  };
  for (int nw : {8, 12, 16}) {
    run(k<0, 8>, "V0 pair (lane=word, 2 col), SEG 8", nw, 2 * 8 * 64);
    run(k<0, 14>, "V0 pair (lane=word, 2 col), SEG 14", nw, 2 * 14 * 64);
    run(k<0, 4>, "V0 pair (lane=word, 2 col), SEG 4", nw, 2 * 4 * 64);
    run(k<1, 4>, "V1 quad (lane=word, 4 col), SEG 4", nw, 4 * 4 * 64);
    run(k<1, 6>, "V1 quad (lane=word, 4 col), SEG 6", nw, 4 * 6 * 64);
    run(k<1, 8>, "V1 quad (lane=word, 4 col), SEG 8", nw, 4 * 8 * 64);
    run(k<2, 4>, "V2 pixel (lane=px, UR W), SEG 4", nw, 32 * 4 * 8);
    run(k<3, 8>, "V3 FHFMA pair, SEG 8", nw, 2 * 8 * 64);
    run(k<3, 14>, "V3 FHFMA pair, SEG 14", nw, 2 * 14 * 64);
    run(k<5, 14>, "V5 FHFMA pair runtime geometry, SEG 14", nw, 2 * 14 * 64);
    run(k<5, 8>, "V5 FHFMA pair runtime geometry, SEG 8", nw, 2 * 8 * 64);
    run(k<6, 14>, "V6 = V5 + barrier per item, SEG 14", nw, 2 * 14 * 64);
    run(k<3, 4>, "V3 FHFMA pair, SEG 4", nw, 2 * 4 * 64);
    run(k<4, 4>, "V4 FHFMA quad, SEG 4", nw, 4 * 4 * 64);
    run(k<4, 8>, "V4 FHFMA quad, SEG 8", nw, 4 * 8 * 64);
    run(k<2, 6>, "V2 pixel (lane=px, UR W), SEG 6", nw, 32 * 6 * 8);
  }
  return 0;
}
