// Shared device-side pieces of the FCM kernels: dtype traits (a lane handles one 32-bit word
// of channels), the Conv-Norm-Act epilogue and the depthwise column core.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "fcm.h"
#include "ptx.cuh"

namespace fcm {

// Device copy of fcm_epilogue (passed by value as a kernel argument).
struct Epi {
  int act;
  const float* scale;
  const float* bias;
  const int32_t* bias_q;
  const int32_t* mult_q;
  const int32_t* shift_q;
  int zp_in, zp_out, qmin, qmax;
};

// ---------------------------------------------------------------------------- dtype traits
// VEC = channels per 32-bit word; acc_t = accumulator type (fp32, or exact int32 for int8).
template <int DT> struct Tr;

template <> struct Tr<FCM_F32> {
  using T = float;
  using acc_t = float;
  static constexpr int VEC = 1, ES = 4;
  __device__ static void unpack(uint32_t w, acc_t (&o)[1]) { o[0] = __uint_as_float(w); }
};
template <> struct Tr<FCM_BF16> {
  using T = __nv_bfloat16;
  using acc_t = float;
  static constexpr int VEC = 2, ES = 2;
  __device__ static void unpack(uint32_t w, acc_t (&o)[2]) {
    o[0] = __uint_as_float(w << 16);
    o[1] = __uint_as_float(w & 0xFFFF0000u);
  }
};
template <> struct Tr<FCM_F16> {
  using T = __half;
  using acc_t = float;
  static constexpr int VEC = 2, ES = 2;
  __device__ static void unpack(uint32_t w, acc_t (&o)[2]) {
    __half2 h = *reinterpret_cast<__half2*>(&w);
    float2 f = __half22float2(h);
    o[0] = f.x;
    o[1] = f.y;
  }
};
template <> struct Tr<FCM_S8> {
  using T = int8_t;
  using acc_t = int32_t;
  static constexpr int VEC = 4, ES = 1;
  __device__ static void unpack(uint32_t w, acc_t (&o)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = static_cast<int32_t>(w << (24 - 8 * i)) >> 24;
  }
};

// ---------------------------------------------------------------------------- epilogue
__device__ __forceinline__ float act_f(float v, int act) {
  if (act == FCM_ACT_RELU) return fmaxf(v, 0.f);
  if (act == FCM_ACT_RELU6) return fminf(fmaxf(v, 0.f), 6.f);
  return v;
}

// Per-channel epilogue constants held in registers.
struct EpiC {
  float sc, bi;         // float paths
  int32_t bq, m, sh;    // int8 path
};

template <int DT>
__device__ __forceinline__ EpiC load_epi(const Epi& e, int c, bool valid) {
  EpiC r{0.f, 0.f, 0, 0, 1};
  if (!valid) return r;
  if constexpr (DT == FCM_S8) {
    r.bq = e.bias_q ? __ldg(e.bias_q + c) : 0;
    r.m = __ldg(e.mult_q + c);
    r.sh = __ldg(e.shift_q + c);
  } else {
    r.sc = e.scale ? __ldg(e.scale + c) : 1.f;
    r.bi = e.bias ? __ldg(e.bias + c) : 0.f;
  }
  return r;
}

__device__ __forceinline__ int32_t requant_i8(int32_t acc, const EpiC& c, int zp, int qmin, int qmax) {
  long long p = static_cast<long long>(acc + c.bq) * static_cast<long long>(c.m) + (1LL << (c.sh - 1));
  int32_t r = static_cast<int32_t>(p >> c.sh) + zp;
  return min(max(r, qmin), qmax);
}

// Apply the epilogue to VEC accumulators of one 32-bit word and pack to storage.
template <int DT>
__device__ __forceinline__ uint32_t epi_pack(const typename Tr<DT>::acc_t (&a)[Tr<DT>::VEC],
                                             const EpiC (&c)[Tr<DT>::VEC], const Epi& e) {
  if constexpr (DT == FCM_F32) {
    return __float_as_uint(act_f(fmaf(a[0], c[0].sc, c[0].bi), e.act));
  } else if constexpr (DT == FCM_BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(act_f(fmaf(a[0], c[0].sc, c[0].bi), e.act),
                                             act_f(fmaf(a[1], c[1].sc, c[1].bi), e.act));
    return *reinterpret_cast<uint32_t*>(&h);
  } else if constexpr (DT == FCM_F16) {
    __half2 h = __floats2half2_rn(act_f(fmaf(a[0], c[0].sc, c[0].bi), e.act),
                                  act_f(fmaf(a[1], c[1].sc, c[1].bi), e.act));
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w |= (static_cast<uint32_t>(requant_i8(a[i], c[i], e.zp_out, e.qmin, e.qmax)) & 0xFFu) << (8 * i);
    return w;
  }
}

// Float epilogue of a single fp32 accumulator (tensor-core paths).
__device__ __forceinline__ float epi_f(float a, float sc, float bi, int act) { return act_f(fmaf(a, sc, bi), act); }

// ---------------------------------------------------------------------------- DW weights
template <int DT, int K>
struct DwW {
  typename Tr<DT>::acc_t w[K][K][Tr<DT>::VEC];
};

// Load this lane's VEC channels [c, c+VEC) of Wdw[k][k][C]; zero outside [0, C).
template <int DT, int K>
__device__ __forceinline__ void load_dw_weights(DwW<DT, K>& W, const typename Tr<DT>::T* wdw, int C, int c) {
  using TT = typename Tr<DT>::T;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int v = 0; v < Tr<DT>::VEC; ++v) {
        const int cc = c + v;
        if (cc < C) {
          TT t = wdw[(i * K + j) * C + cc];
          if constexpr (DT == FCM_S8) W.w[i][j][v] = static_cast<int32_t>(t);
          else if constexpr (DT == FCM_F32) W.w[i][j][v] = t;
          else if constexpr (DT == FCM_BF16) W.w[i][j][v] = __bfloat162float(t);
          else W.w[i][j][v] = __half2float(t);
        } else {
          W.w[i][j][v] = 0;
        }
      }
}

// ---------------------------------------------------------------------------- DW column core
// One output column of a tile: rows [0, nrows) at stride S over a K x K window that slides down
// the staged input. `src` points at the lane's 32-bit word of input pixel (row 0, col x*S) in
// shared memory; consecutive input columns are `col_words` words apart and consecutive input
// rows `row_words` apart. sink(y, acc) receives the VEC accumulators of output row y.
// Each input word is read from shared memory once per column and reused for K (or K/S) taps.
template <int DT, int K, int S, class Sink>
__device__ __forceinline__ void dw_column(const uint32_t* src, int col_words, int row_words, int nrows,
                                         const DwW<DT, K>& W, Sink&& sink) {
  using A = typename Tr<DT>::acc_t;
  constexpr int V = Tr<DT>::VEC;
  A win[K][K][V];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) Tr<DT>::unpack(src[i * row_words + j * col_words], win[i][j]);
  for (int y = 0; y < nrows; ++y) {
    if (y > 0) {
#pragma unroll
      for (int i = 0; i < K - S; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j)
#pragma unroll
          for (int v = 0; v < V; ++v) win[i][j][v] = win[i + S][j][v];
      const uint32_t* r = src + (y * S) * row_words;
#pragma unroll
      for (int i = K - S; i < K; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j) Tr<DT>::unpack(r[i * row_words + j * col_words], win[i][j]);
    }
    A acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0;
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] += win[i][j][v] * W.w[i][j][v];
    sink(y, acc);
  }
}

// Byte offset of (row m, 32-bit word `wd` in 0..31) in a K-major SWIZZLE_128B operand tile.
__device__ __forceinline__ uint32_t sw128_off(int m, int wd) {
  return (m >> 3) * 1024 + (m & 7) * 128 + ((((wd >> 2) ^ (m & 7))) << 4) + ((wd & 3) << 2);
}

}  // namespace fcm
