// FP32 paths on the CUDA cores (FFMA) -- the north_star's "CUDA-core fallback for thin layers"
// and the paper's own FP32 kernels. fp32 keeps 1e-5 relative accuracy, which a single
// TF32 tensor-core pass cannot (R10b). Same structure as the tensor-core FCMs:
// the intermediate T lives only in shared memory.
#include "common.cuh"
#include "host.h"

namespace fcm {

// ------------------------------------------------------------------ LBL PW (fp32 FFMA GEMM)
// Y[M,N] = eps(X[M,K] . Wp[N,K]^T). 64x64 output tile per CTA, 4x4 per thread, K chunks of 16.
__global__ void __launch_bounds__(256) pw_simt_kernel(const float* __restrict__ x, const float* __restrict__ wp,
                                                      Epi ep, float* __restrict__ y, int M, int K, int N) {
  __shared__ float xs[16][64 + 4];
  __shared__ float ws[16][64 + 4];
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i / 16, kk = i % 16;
      xs[kk][r] = (m0 + r < M && k0 + kk < K) ? x[(size_t)(m0 + r) * K + k0 + kk] : 0.f;
      ws[kk][r] = (n0 + r < N && k0 + kk < K) ? wp[(size_t)(n0 + r) * K + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = xs[kk][ty * 4 + i]; b[i] = ws[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = n0 + tx * 4 + j;
    if (n >= N) continue;
    const float sc = ep.scale ? ep.scale[n] : 1.f, bi = ep.bias ? ep.bias[n] : 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m < M) y[(size_t)m * N + n] = epi_f(acc[i][j], sc, bi, ep.act);
    }
  }
}

__device__ __forceinline__ float dw_tap_sum(const float* __restrict__ x, const float* __restrict__ wdw, int n, int H,
                                            int W, int C, int c, int yo, int xo, int k, int s, int pt, int pl) {
  float acc = 0.f;
  for (int i = 0; i < k; ++i) {
    const int yi = yo * s - pt + i;
    if (yi < 0 || yi >= H) continue;
    for (int j = 0; j < k; ++j) {
      const int xi = xo * s - pl + j;
      if (xi < 0 || xi >= W) continue;
      acc = fmaf(x[(((size_t)n * H + yi) * W + xi) * C + c], wdw[(i * k + j) * C + c], acc);
    }
  }
  return acc;
}

// ------------------------------------------------------------------ FCM DWPW (fp32)
// CTA = 8x8 output pixels x 64 output channels; C_in streams in chunks of 32 through the smem
// commBuffer T[32][64]; PW partial sums stay in registers (OS).
__global__ void __launch_bounds__(256) dwpw_simt_kernel(const float* __restrict__ x, const float* __restrict__ wdw,
                                                        Epi ed, const float* __restrict__ wp, Epi ep,
                                                        float* __restrict__ y, int N, int H, int W, int C, int Ho,
                                                        int Wo, int Cout, int k, int s, int pt, int pl, int tiles_x,
                                                        int tiles_y) {
  __shared__ float ts[32][64 + 4];
  __shared__ float ws[32][64 + 4];
  int t = blockIdx.x;
  const int txi = t % tiles_x;
  t /= tiles_x;
  const int tyi = t % tiles_y;
  const int n = t / tiles_y;
  const int n0 = blockIdx.y * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int c0 = 0; c0 < C; c0 += 32) {
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int p = i % 64, cc = i / 64;
      const int c = c0 + cc;
      const int yo = tyi * 8 + p / 8, xo = txi * 8 + p % 8;
      float v = 0.f;
      if (c < C && yo < Ho && xo < Wo) {
        const float a = dw_tap_sum(x, wdw, n, H, W, C, c, yo, xo, k, s, pt, pl);
        const float sc = ed.scale ? ed.scale[c] : 1.f, bi = ed.bias ? ed.bias[c] : 0.f;
        v = epi_f(a, sc, bi, ed.act);
      }
      ts[cc][p] = v;
      const int co = n0 + p;
      ws[cc][p] = (c < C && co < Cout) ? wp[(size_t)co * C + c] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < 32; ++cc) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = ts[cc][ty * 4 + i]; b[i] = ws[cc][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int co = n0 + tx * 4 + j;
    if (co >= Cout) continue;
    const float sc = ep.scale ? ep.scale[co] : 1.f, bi = ep.bias ? ep.bias[co] : 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int p = ty * 4 + i;
      const int yo = tyi * 8 + p / 8, xo = txi * 8 + p % 8;
      if (yo < Ho && xo < Wo) y[(((size_t)n * Ho + yo) * Wo + xo) * Cout + co] = epi_f(acc[i][j], sc, bi, ep.act);
    }
  }
}

// ------------------------------------------------------------------ FCM PWDW_R (fp32)
// CTA = 8x8 DW output pixels x 32 intermediate channels. T is computed over the halo tile
// (recomputed overlap) into smem, zero outside the image, then the DW reads it.
__global__ void __launch_bounds__(256) pwdw_simt_kernel(const float* __restrict__ x, const float* __restrict__ wp,
                                                        Epi ep, const float* __restrict__ wdw, Epi ed,
                                                        float* __restrict__ y, int N, int H, int W, int C, int Ho,
                                                        int Wo, int Cmid, int k, int s, int pt, int pl, int tiles_x,
                                                        int tiles_y) {
  extern __shared__ float tsm[];  // [R][33]
  int t = blockIdx.x;
  const int txi = t % tiles_x;
  t /= tiles_x;
  const int tyi = t % tiles_y;
  const int n = t / tiles_y;
  const int cm0 = blockIdx.y * 32;
  const int hin = 7 * s + k, win = 7 * s + k;
  const int R = hin * win;
  const int y_in0 = tyi * 8 * s - pt, x_in0 = txi * 8 * s - pl;
  for (int i = threadIdx.x; i < R * 32; i += 256) {
    const int cc = i % 32, r = i / 32;
    const int yi = y_in0 + r / win, xi = x_in0 + r % win;
    const int cm = cm0 + cc;
    float v = 0.f;
    if (cm < Cmid && yi >= 0 && yi < H && xi >= 0 && xi < W) {
      const float* xp = x + (((size_t)n * H + yi) * W + xi) * C;
      const float* wr = wp + (size_t)cm * C;
      float a = 0.f;
      for (int ci = 0; ci < C; ++ci) a = fmaf(xp[ci], wr[ci], a);
      const float sc = ep.scale ? ep.scale[cm] : 1.f, bi = ep.bias ? ep.bias[cm] : 0.f;
      v = epi_f(a, sc, bi, ep.act);
    }
    tsm[r * 33 + cc] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 32; i += 256) {
    const int cc = i % 32, p = i / 32;
    const int cm = cm0 + cc;
    const int yo = tyi * 8 + p / 8, xo = txi * 8 + p % 8;
    if (cm >= Cmid || yo >= Ho || xo >= Wo) continue;
    float a = 0.f;
    for (int ii = 0; ii < k; ++ii)
      for (int jj = 0; jj < k; ++jj)
        a = fmaf(tsm[((p / 8) * s + ii) * win * 33 + ((p % 8) * s + jj) * 33 + cc], wdw[(ii * k + jj) * Cmid + cm], a);
    const float sc = ed.scale ? ed.scale[cm] : 1.f, bi = ed.bias ? ed.bias[cm] : 0.f;
    y[(((size_t)n * Ho + yo) * Wo + xo) * Cmid + cm] = epi_f(a, sc, bi, ed.act);
  }
}

int launch_pw_simt(const float* x, const float* wp, const Epi& ep, float* y, int M, int K, int N, cudaStream_t st) {
  dim3 grid((M + 63) / 64, (N + 63) / 64);
  pw_simt_kernel<<<grid, 256, 0, st>>>(x, wp, ep, y, M, K, N);
  return check_launch("pw_simt_kernel");
}

int launch_dwpw_simt(const float* x, const float* wdw, const Epi& ed, const float* wp, const Epi& ep, float* y,
                     const Geo& g, cudaStream_t st) {
  const int tiles_x = (g.Wo + 7) / 8, tiles_y = (g.Ho + 7) / 8;
  dim3 grid(tiles_x * tiles_y * g.N, (g.Cout + 63) / 64);
  dwpw_simt_kernel<<<grid, 256, 0, st>>>(x, wdw, ed, wp, ep, y, g.N, g.H, g.W, g.C, g.Ho, g.Wo, g.Cout, g.k, g.s,
                                         g.pt, g.pl, tiles_x, tiles_y);
  return check_launch("dwpw_simt_kernel");
}

int launch_pwdw_simt(const float* x, const float* wp, const Epi& ep, const float* wdw, const Epi& ed, float* y,
                     const Geo& g, cudaStream_t st) {
  const int tiles_x = (g.Wo + 7) / 8, tiles_y = (g.Ho + 7) / 8;
  const int hin = 7 * g.s + g.k;
  const size_t smem = (size_t)hin * hin * 33 * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(pwdw_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(tiles_x * tiles_y * g.N, (g.Cout + 31) / 32);
  pwdw_simt_kernel<<<grid, 256, smem, st>>>(x, wp, ep, wdw, ed, y, g.N, g.H, g.W, g.C, g.Ho, g.Wo, g.Cout, g.k, g.s,
                                            g.pt, g.pl, tiles_x, tiles_y);
  return check_launch("pwdw_simt_kernel");
}

}  // namespace fcm
