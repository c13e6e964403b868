// Shared device-side pieces of the FCM kernels: dtype traits (a lane handles one 32-bit word
// of channels), the Conv-Norm-Act epilogue and the depthwise column core.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <type_traits>

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
  const void* residual;  // optional: same shape / dtype as the output, added after the activation
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
// Activation as a clamp [lo, hi] (NONE: (-inf, inf), RELU: [0, inf), RELU6: [0, 6]); branch-free.
__device__ __forceinline__ float act_lo(int act) { return act == FCM_ACT_NONE ? -INFINITY : 0.f; }
__device__ __forceinline__ float act_hi(int act) { return act == FCM_ACT_RELU6 ? 6.f : INFINITY; }
// SiLU v * sigmoid(v) = v / (1 + e^-v) (fast exp; e^-v -> inf gives -0) and the exact (erf) GELU.
__device__ __forceinline__ float silu_f(float v) {
  float e, r;  // 2^(-v log2 e) and the approximate reciprocal (2 MUFU ops; rcp(inf) = 0 -> -0)
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-1.4426950408889634f * v));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
  return v * r;
}
__device__ __forceinline__ float gelu_f(float v) { return 0.5f * v * (1.f + erff(v * 0.70710678118654752f)); }
__device__ __forceinline__ float act_f(float v, int act) {
  if (act == FCM_ACT_SILU) return silu_f(v);
  if (act == FCM_ACT_GELU) return gelu_f(v);
  return fminf(fmaxf(v, act_lo(act)), act_hi(act));
}
template <int ACT>
__device__ __forceinline__ float act_t(float v) {
  if constexpr (ACT == FCM_ACT_SILU) return silu_f(v);
  else if constexpr (ACT == FCM_ACT_GELU) return gelu_f(v);
  else if constexpr (ACT == FCM_ACT_RELU6) return fminf(fmaxf(v, 0.f), 6.f);
  else if constexpr (ACT == FCM_ACT_RELU) return fmaxf(v, 0.f);
  else return v;
}
// One output element of a float path: act(acc*scale + bias) (+ residual r).
__device__ __forceinline__ float epi_fr(float a, float sc, float bi, int act, float r) { return act_f(fmaf(a, sc, bi), act) + r; }
// Residual element i of a float-dtype tensor as fp32.
template <int DT>
__device__ __forceinline__ float res_at(const void* r, size_t i) {
  if constexpr (DT == FCM_F32) return __ldg(static_cast<const float*>(r) + i);
  else if constexpr (DT == FCM_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(r)[i]);
  else if constexpr (DT == FCM_F16) return __half2float(static_cast<const __half*>(r)[i]);
  else return 0.f;
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

// Per-column epilogue constants staged once per CTA in shared memory (broadcast reads through
// explicit ld.shared). float: scale[ncap], bias[ncap]; int8: bias_q, mult_q, shift_q [ncap].
struct EpiS {
  uint32_t base;  // shared-space byte address
  int ncap;
  int fast;       // int8: every staged shift >= 33 (the one-mad.hi requantisation applies to all columns)
  __device__ __forceinline__ float sc(int n) const { return __uint_as_float(lds32(base + 4 * n)); }
  __device__ __forceinline__ float bi(int n) const { return __uint_as_float(lds32(base + 4 * (ncap + n))); }
  __device__ __forceinline__ int32_t bq(int n) const { return (int32_t)lds32(base + 4 * n); }
  __device__ __forceinline__ int32_t mq(int n) const { return (int32_t)lds32(base + 4 * (ncap + n)); }
  __device__ __forceinline__ int32_t sh(int n) const { return (int32_t)lds32(base + 4 * (2 * ncap + n)); }
};

// Fill the constant arrays for columns [0, ncap) (zeros past N). Each thread first issues up to
// 4 independent global loads per array, then the shared stores (no load/store serialisation).
template <int DT>
__device__ __forceinline__ EpiS stage_consts(const Epi& e, int N, int ncap, uint8_t* area) {
  const uint32_t base = smem_u32(area);
  const int nt = blockDim.x;
  bool fast = true;
  for (int i0 = threadIdx.x; i0 < ncap; i0 += 4 * nt) {
    uint32_t a[4], b[4], c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * nt;
      const bool v = i < N;
      if constexpr (DT == FCM_S8) {
        a[u] = (v && e.bias_q) ? (uint32_t)__ldg(e.bias_q + i) : 0u;
        b[u] = v ? (uint32_t)__ldg(e.mult_q + i) : 0u;
        c[u] = v ? (uint32_t)__ldg(e.shift_q + i) : 1u;
        fast = fast && (!v || (int32_t)c[u] >= 33);
      } else {
        a[u] = __float_as_uint(v ? (e.scale ? __ldg(e.scale + i) : 1.f) : 0.f);
        b[u] = __float_as_uint((v && e.bias) ? __ldg(e.bias + i) : 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * nt;
      if (i < ncap) {
        sts32(base + 4 * i, a[u]);
        sts32(base + 4 * (ncap + i), b[u]);
        if constexpr (DT == FCM_S8) sts32(base + 4 * (2 * ncap + i), c[u]);
      }
    }
  }
  // block-wide: every caller stages its constants with all threads at kernel entry
  const int f = DT == FCM_S8 ? __syncthreads_and(fast) : 0;
  return EpiS{base, ncap, f};
}
template <int DT> constexpr int consts_bytes(int ncap) { return (DT == FCM_S8 ? 12 : 8) * ncap; }

template <int DT>
__device__ __forceinline__ EpiC epic(const EpiS& cs, int c) {
  if constexpr (DT == FCM_S8) return EpiC{0.f, 0.f, cs.bq(c), cs.mq(c), cs.sh(c)};
  else return EpiC{cs.sc(c), cs.bi(c), 0, 0, 1};
}

// ---------------------------------------------------------------------------- DW segment core
// Output rows [y0, y0+nrows) of one output column of a staged tile. `src` points at the lane's
// 32-bit word of input pixel (row 0, col x*S) in shared memory; input columns are `col_words`
// words apart, rows `row_words` apart; input rows are clamped to `max_row` (the tile's last
// staged row: rows computed past the tile are never stored). Rows are produced R at a time from
// a K x K window that slides down the column, so each staged word is read about once and the
// R x VEC accumulation chains are independent (ILP). Tap order (i, j) is fixed, so every
// kernel that uses this core produces bit-identical DW results.
template <int DT, int K> constexpr int dw_rows_per_step() { return (K == 3 && Tr<DT>::VEC <= 2) ? 4 : 1; }

template <int DT, int K, int S, class Sink>
__device__ __forceinline__ void dw_segment(uint32_t src, int col_bytes, int row_bytes, int y0, int nrows,
                                           int max_row, const DwW<DT, K>& W, Sink&& sink) {
  using A = typename Tr<DT>::acc_t;
  constexpr int V = Tr<DT>::VEC;
  constexpr int R = dw_rows_per_step<DT, K>();
  constexpr int WR = (R - 1) * S + K;  // window rows
  A win[WR][K][V];
  int r0 = y0 * S;  // input row of window row 0
#pragma unroll
  for (int i = 0; i < WR; ++i) {
    const uint32_t rp = src + min(r0 + i, max_row) * row_bytes;
#pragma unroll
    for (int j = 0; j < K; ++j) Tr<DT>::unpack(lds32(rp + j * col_bytes), win[i][j]);
  }
  for (int y = 0; y < nrows; y += R) {
    if (y > 0) {
      r0 += R * S;
      constexpr int KEEP = WR - R * S > 0 ? WR - R * S : 0;
#pragma unroll
      for (int i = 0; i < KEEP; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j)
#pragma unroll
          for (int v = 0; v < V; ++v) win[i][j][v] = win[i + R * S][j][v];
#pragma unroll
      for (int i = KEEP; i < WR; ++i) {
        const uint32_t rp = src + min(r0 + i, max_row) * row_bytes;
#pragma unroll
        for (int j = 0; j < K; ++j) Tr<DT>::unpack(lds32(rp + j * col_bytes), win[i][j]);
      }
    }
    A acc[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[r][v] = 0;
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[r][v] += win[r * S + i][j][v] * W.w[i][j][v];
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (y + r < nrows) sink(y0 + y + r, acc[r]);
  }
}

// ---------------------------------------------------------------------------- paired-FP32 DW core
// bf16 / fp16 with K = 3: a lane's 32-bit word holds 2 channels, kept as an fp32 pair in a 64-bit
// register and accumulated with the sm_100 packed FFMA2 (fma.rn.f32x2: two IEEE fp32 FMAs per
// instruction, identical results to two FFMAs). A segment of SEG output rows is fully unrolled:
// no window-shift moves, SEG x 1 independent accumulation chains.
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
template <int DT>
__device__ __forceinline__ uint64_t word_to_f2(uint32_t w) {
  if constexpr (DT == FCM_BF16) {
    // two byte permutes (ALU pipe; `w << 16` would become an IMAD on the FMA pipe the FFMA2s use)
    uint32_t lo, hi;
    asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(lo) : "r"(w));
    asm("prmt.b32 %0, %1, 0, 0x3244;" : "=r"(hi) : "r"(w));
    return f2_pack(__uint_as_float(lo), __uint_as_float(hi));
  } else {
    __half2 h = *reinterpret_cast<__half2*>(&w);
    float2 f = __half22float2(h);
    return f2_pack(f.x, f.y);
  }
}

template <int DT, int K>
struct DwW2 {
  uint64_t w[K][K];
};

template <int DT, int K>
__device__ __forceinline__ void load_dw_weights2_smem(DwW2<DT, K>& W, const uint32_t* wsm, int cwords, int cw) {
  const uint32_t a = smem_u32(wsm) + 4 * cw;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) W.w[i][j] = word_to_f2<DT>(lds32(a + 4 * (i * K + j) * cwords));
}

template <int DT, int K>
__device__ __forceinline__ void load_dw_weights2(DwW2<DT, K>& W, const void* wdw, int C, int c) {
  const uint32_t* g = static_cast<const uint32_t*>(wdw);
  const int cw = c / 2;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) W.w[i][j] = (c < C) ? word_to_f2<DT>(__ldg(g + (i * K + j) * (C / 2) + cw)) : 0ull;
}

// Output rows y0 .. y0+SEG-1 (all computed; input rows clamped to max_row); sink(r, acc) gets the
// compile-time row offset r and the fp32 pair accumulator.
template <int DT, int K, int S, int SEG, class Sink>
__device__ __forceinline__ void dw_seg2(uint32_t src, int col_bytes, int row_bytes, int y0, int max_row,
                                        const DwW2<DT, K>& W, Sink&& sink) {
  constexpr int WR = (SEG - 1) * S + K;
  uint64_t win[WR][K];
#pragma unroll
  for (int i = 0; i < WR; ++i) {
    const uint32_t rp = src + min(y0 * S + i, max_row) * row_bytes;
#pragma unroll
    for (int j = 0; j < K; ++j) win[i][j] = word_to_f2<DT>(lds32(rp + j * col_bytes));
  }
#pragma unroll
  for (int r = 0; r < SEG; ++r) {
    uint64_t acc = 0ull;
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) acc = f2_fma(win[r * S + i][j], W.w[i][j], acc);
    sink(r, acc);
  }
}

// Mixed-precision FMA on sm_100: fp32 accumulator += bf16/f16 x bf16/f16 taken straight from the
// halves of packed 32-bit words (SASS FHFMA with .H0/.H1 selectors) -- no unpacking. Exact: the
// product of two bf16/f16 values is exact in fp32, so the result equals fmaf on converted values.
template <int DT>
__device__ __forceinline__ void hfma2_acc(float& a0, float& a1, uint32_t x, uint32_t w) {
  if constexpr (DT == FCM_BF16)
    asm("{.reg .b16 xl, xh, wl, wh;\n\tmov.b32 {xl, xh}, %2;\n\tmov.b32 {wl, wh}, %3;\n\t"
        "fma.rn.f32.bf16 %0, xl, wl, %0;\n\tfma.rn.f32.bf16 %1, xh, wh, %1;}"
        : "+f"(a0), "+f"(a1) : "r"(x), "r"(w));
  else
    asm("{.reg .b16 xl, xh, wl, wh;\n\tmov.b32 {xl, xh}, %2;\n\tmov.b32 {wl, wh}, %3;\n\t"
        "fma.rn.f32.f16 %0, xl, wl, %0;\n\tfma.rn.f32.f16 %1, xh, wh, %1;}"
        : "+f"(a0), "+f"(a1) : "r"(x), "r"(w));
}

template <int K>
struct DwWh {
  uint32_t w[K][K];  // packed channel pairs
};

template <int K>
__device__ __forceinline__ void load_dw_weights_h_smem(DwWh<K>& W, const uint32_t* wsm, int cwords, int cw) {
  const uint32_t a = smem_u32(wsm) + 4 * cw;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) W.w[i][j] = lds32(a + 4 * (i * K + j) * cwords);
}

template <int K>
__device__ __forceinline__ void load_dw_weights_h(DwWh<K>& W, const void* wdw, int C, int c) {
  const uint32_t* g = static_cast<const uint32_t*>(wdw);
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) W.w[i][j] = (c < C) ? __ldg(g + (i * K + j) * (C / 2) + c / 2) : 0u;
}

// Same contract as dw_seg2 (rows y0..y0+SEG-1, input rows clamped to max_row), with the window and
// the weights kept as packed words; sink(r, acc) receives the fp32 pair packed in a uint64.
template <int DT, int K, int S, int SEG, class Sink>
__device__ __forceinline__ void dw_segh(uint32_t src, int col_bytes, int row_bytes, int y0, int max_row,
                                        const DwWh<K>& W, Sink&& sink) {
  constexpr int WR = (SEG - 1) * S + K;
  uint32_t win[WR][K];
#pragma unroll
  for (int i = 0; i < WR; ++i) {
    const uint32_t rp = src + min(y0 * S + i, max_row) * row_bytes;
#pragma unroll
    for (int j = 0; j < K; ++j) win[i][j] = lds32(rp + j * col_bytes);
  }
#pragma unroll
  for (int r = 0; r < SEG; ++r) {
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) hfma2_acc<DT>(a0, a1, win[r * S + i][j], W.w[i][j]);
    sink(r, f2_pack(a0, a1));
  }
}

// Division by a runtime-invariant divisor d >= 1 without the ~15-instruction integer divide:
// q = (umulhi(n, m) + n) >> l with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1 (exact for
// 0 <= n < 2^31). The magic pair is computed on the host and passed as a kernel parameter.
struct FDiv {
  uint32_t m, l;
};
inline FDiv make_fdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  return FDiv{static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - d)) / d + 1), l};
}
__device__ __forceinline__ int fdiv(int n, FDiv f) {
  return static_cast<int>((__umulhi(static_cast<uint32_t>(n), f.m) + static_cast<uint32_t>(n)) >> f.l);
}

// Activation bounds as a packed pair (both halves = the bound, rounded to DT; all three bounds
// -inf / 0 / 6 / +inf are exact in bf16 and f16).
template <int DT>
__device__ __forceinline__ uint32_t bound2(float v) {
  uint32_t h;
  if constexpr (DT == FCM_BF16) asm("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(h) : "f"(v));
  else asm("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(h) : "f"(v));
  return h;
}

// Epilogue of an fp32 pair -> packed bf16x2 / f16x2 word (scale/bias as pairs, then the activation
// clamp on the packed result: rounding is monotonic and the bounds are representable, so
// clamp(round(v)) == round(clamp(v)) -- two packed min/max instead of four fp32 ones).
template <int DT>
__device__ __forceinline__ uint32_t epi2_pack(uint64_t acc, uint64_t sc, uint64_t bi, uint32_t lo2, uint32_t hi2) {
  float a, b;
  f2_unpack(f2_fma(acc, sc, bi), a, b);
  uint32_t h;
  if constexpr (DT == FCM_BF16)
    asm("{cvt.rn.bf16x2.f32 %0, %2, %1;\n\tmax.bf16x2 %0, %0, %3;\n\tmin.bf16x2 %0, %0, %4;}"
        : "=r"(h) : "f"(a), "f"(b), "r"(lo2), "r"(hi2));
  else
    asm("{cvt.rn.f16x2.f32 %0, %2, %1;\n\tmax.f16x2 %0, %0, %3;\n\tmin.f16x2 %0, %0, %4;}"
        : "=r"(h) : "f"(a), "f"(b), "r"(lo2), "r"(hi2));
  return h;
}

// Load this lane's DW weights from a shared-memory copy of Wdw laid out [k*k][C/VEC words].
template <int DT, int K>
__device__ __forceinline__ void load_dw_weights_smem(DwW<DT, K>& W, const uint32_t* wsm, int cwords, int cw) {
  const uint32_t a = smem_u32(wsm) + 4 * cw;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) Tr<DT>::unpack(lds32(a + 4 * (i * K + j) * cwords), W.w[i][j]);
}

// Copy Wdw [k*k][C] (global) into shared memory as [k*k][cwords] 32-bit words, zero-padding
// channel words >= C/VEC up to cwords.
template <int DT>
__device__ __forceinline__ void stage_dw_weights(const void* wdw, int k, int C, int cwords, uint32_t* wsm) {
  const uint32_t* g = static_cast<const uint32_t*>(wdw);
  const int cw_real = C / Tr<DT>::VEC;
  const int n = k * k * cwords, nt = blockDim.x;
  const uint32_t base = smem_u32(wsm);
  for (int i0 = threadIdx.x; i0 < n; i0 += 4 * nt) {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * nt;
      const int t = i / cwords, w = i - t * cwords;
      v[u] = (i < n && w < cw_real) ? __ldg(g + t * cw_real + w) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * nt < n) sts32(base + 4 * (i0 + u * nt), v[u]);
  }
}

// Byte offset of (row m, 32-bit word `wd` in 0..31) in a K-major SWIZZLE_128B operand tile.
__device__ __forceinline__ uint32_t sw128_off(int m, int wd) {
  return (m >> 3) * 1024 + (m & 7) * 128 + ((((wd >> 2) ^ (m & 7))) << 4) + ((wd & 3) << 2);
}

// ---------------------------------------------------------------------------- column-pair FFMA2 DW core
// bf16 / f16, 3x3. A lane owns one 32-bit word (2 channels) of TWO adjacent output columns
// (x0, x0+1) over SEG output rows. Input rows stream through once: each row's 3+S words are read
// (ld.shared), widened to fp32 pairs, and fed as packed FFMA2 (fma.rn.f32x2, two IEEE fp32 FMAs
// per instruction) into the <= 3 x 2 output accumulators that use the row. The folded-BN scale
// is pre-multiplied into the fp32 weights and the accumulator starts at the bias (reading R3:
// per-channel affine Norm), so the epilogue is the rounding + activation clamp only. Tap order
// (i, j) is fixed: every kernel using this core gives bit-identical DW results.
// Per output word: (3+S)((SEG-1)S+3)/(2 SEG) loads, 9 FFMA2, 1-2 packs.
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

template <int DT, int S, int SEG, class Sink>
__device__ __forceinline__ void dw3_pair(uint32_t src, int col_bytes, int row_bytes, int y0, int max_row,
                                         const uint64_t (&W)[9], uint64_t bias, Sink&& sink) {
  constexpr int NCW = 3 + S;              // input words per row feeding 2 output columns
  constexpr int WR = (SEG - 1) * S + 3;   // input rows of the segment
  constexpr int PD = 2;                   // software pipelining: rows loaded ahead of their use
  uint64_t acc[SEG][2];
  uint32_t raw[WR][NCW];
  auto load_row = [&](int ii) {
    const uint32_t rp = src + min(y0 * S + ii, max_row) * row_bytes;
#pragma unroll
    for (int j = 0; j < NCW; ++j) raw[ii][j] = lds32(rp + j * col_bytes);
  };
#pragma unroll
  for (int ii = 0; ii < PD && ii < WR; ++ii) load_row(ii);
#pragma unroll
  for (int ii = 0; ii < WR; ++ii) {
    if (ii + PD < WR) load_row(ii + PD);
    uint64_t x[NCW];
#pragma unroll
    for (int j = 0; j < NCW; ++j) x[j] = word_to_f2<DT>(raw[ii][j]);
#pragma unroll
    for (int r = 0; r < SEG; ++r) {
      const int i = ii - r * S;  // kernel row of this input row for output row r
      if (i < 0 || i > 2) continue;
      // tap-outer / column-inner: the two columns' FFMA2s share the weight operand back to back
      // (operand-reuse cache: fewer register-file reads; each accumulator still sees taps in the
      // same (i, j) order, so results are unchanged)
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          acc[r][c] = f2_fma(x[c * S + j], W[i * 3 + j], (i == 0 && j == 0) ? bias : acc[r][c]);
      if (i == 2) sink(r, acc[r][0], acc[r][1]);
    }
  }
}

// ---------------------------------------------------------------------------- column-group FHFMA DW core
// bf16 / f16, 3x3. Same lane mapping as dw3_pair (a lane owns one 32-bit word = 2 channels of NC
// adjacent output columns over SEG rows, input rows streamed once), but the taps are the mixed
// fp32 += bf16 x bf16 FMA (fma.rn.f32.bf16 / .f16, SASS FHFMA with .H0/.H1 half selectors): the
// packed words feed the FMA directly, so there is no bf16 -> fp32 widening. Measured on B200
// (tools/microbench/ffma2_operands.cu): every ALU-pipe instruction (PRMT, LOP3, ...) costs about as
// much issue time as one FFMA2, so the widening (2 PRMT per input word) made up ~40 % of dw3_pair's
// pipe time. FHFMA does 32 MACs per warp instruction at the FFMA rate (~125 MAC/clk/SM, fma_rates.cu).
// Products of two bf16 / f16 values are exact in fp32, so each tap is one correctly rounded fp32
// FMA -- the same arithmetic as widening first. Weights are the raw packed DW weights; the
// accumulators start at 0 and the caller applies the per-channel scale / bias (R3) in its sink.
// sink(r, c, acc) gets output row r, column c (compile-time) and the fp32 pair as (lo, hi).
// `src` addresses the item's first input row (row y0 * S of the staged tile, this lane's word);
// rows are COLB bytes per pixel apart and `row_bytes` apart. All (SEG - 1) S + 3 input rows must
// lie inside the staged tile: callers shift a ragged last segment up (y0 = th - SEG) and recompute
// the overlap instead of clamping row indices, so the row addresses are plain increments.
template <int DT, int S, int SEG, int NC, int COLB, class Sink>
__device__ __forceinline__ void dw3_cols_h(uint32_t src, int row_bytes, const uint32_t (&W)[9], Sink&& sink) {
  constexpr int NCW = (NC - 1) * S + 3;   // input words per row feeding NC output columns
  constexpr int WR = (SEG - 1) * S + 3;   // input rows of the segment
  constexpr int PD = 2;                   // rows loaded ahead of their use
  float acc[SEG][NC][2];
  uint32_t raw[WR][NCW];
  auto load_row = [&](int ii) {
    const uint32_t rp = src + ii * row_bytes;
#pragma unroll
    for (int j = 0; j < NCW; ++j) raw[ii][j] = lds32(rp + j * COLB);
  };
#pragma unroll
  for (int ii = 0; ii < PD && ii < WR; ++ii) load_row(ii);
#pragma unroll
  for (int ii = 0; ii < WR; ++ii) {
    if (ii + PD < WR) load_row(ii + PD);
#pragma unroll
    for (int r = 0; r < SEG; ++r) {
      const int i = ii - r * S;
      if (i < 0 || i > 2) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (i == 0 && j == 0) acc[r][c][0] = acc[r][c][1] = 0.f;
          hfma2_acc<DT>(acc[r][c][0], acc[r][c][1], raw[ii][c * S + j], W[i * 3 + j]);
        }
      if (i == 2) {
#pragma unroll
        for (int c = 0; c < NC; ++c) sink(r, c, acc[r][c][0], acc[r][c][1]);
      }
    }
  }
}

// Rolled form of dw3_cols_h for a RUNTIME number of output rows: output row r is computed whole
// in iteration r from a 3-row window of staged input words (S = 1: rows r..r+2, one new row per
// iteration, window period 3; S = 2: rows 2r..2r+2, two new rows per iteration, the even row
// shared with the next output row, period 2; measured: a 4-buffer variant loading one row ahead
// was 3 % slower). The loop body is unrolled by the window period so
// the window rotates through static registers. Same taps in the same (i, j) order per output as
// dw3_cols_h (bit-identical results). Code size: one period (~3 x 50 instructions) instead of a
// fully unrolled segment (~750 for 14 rows) -- the SM instruction cache is shared with the other
// warp roles of the fused kernels and a fully unrolled segment per SEG x activation variant made
// the DW warps instruction-fetch bound (ncu: 40 % no_instruction stalls).
#ifndef FCM_DW_SPLIT  // measured: no gain in DWPW (b8 30.3 -> 31.2 us), kept as a development switch
#define FCM_DW_SPLIT 0
#endif
template <int DT, int S, int NC, int COLB, class Sink>
__device__ __forceinline__ void dw3_cols_roll(uint32_t src, int row_bytes, int nrows, const uint32_t (&W)[9],
                                              Sink&& sink) {
  constexpr int NCW = (NC - 1) * S + 3;
  auto load = [&](uint32_t (&dst)[NCW], int row) {
    const uint32_t rp = src + row * row_bytes;
#pragma unroll
    for (int j = 0; j < NCW; ++j) dst[j] = lds32(rp + j * COLB);
  };
  auto out_row = [&](int r, const uint32_t (&x0)[NCW], const uint32_t (&x1)[NCW], const uint32_t (&x2)[NCW]) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
#if FCM_DW_SPLIT
      // one partial sum per filter row (three 3-deep FHFMA chains instead of one 9-deep chain per
      // output half: the DW warps are latency-bound at two warps per SM sub-partition), summed
      // with two packed adds: (p0 + p1) + p2
      float a[3] = {0.f, 0.f, 0.f}, b[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 3; ++j) hfma2_acc<DT>(a[0], b[0], x0[c * S + j], W[j]);
#pragma unroll
      for (int j = 0; j < 3; ++j) hfma2_acc<DT>(a[1], b[1], x1[c * S + j], W[3 + j]);
#pragma unroll
      for (int j = 0; j < 3; ++j) hfma2_acc<DT>(a[2], b[2], x2[c * S + j], W[6 + j]);
      const uint64_t one2 = 0x3F8000003F800000ull;
      const uint64_t s = f2_fma(f2_pack(a[2], b[2]), one2, f2_fma(f2_pack(a[0], b[0]), one2, f2_pack(a[1], b[1])));
      float lo, hi;
      f2_unpack(s, lo, hi);
      sink(r, c, lo, hi);
#else
      float a = 0.f, b = 0.f;
#pragma unroll
      for (int j = 0; j < 3; ++j) hfma2_acc<DT>(a, b, x0[c * S + j], W[j]);
#pragma unroll
      for (int j = 0; j < 3; ++j) hfma2_acc<DT>(a, b, x1[c * S + j], W[3 + j]);
#pragma unroll
      for (int j = 0; j < 3; ++j) hfma2_acc<DT>(a, b, x2[c * S + j], W[6 + j]);
      sink(r, c, a, b);
#endif
    }
  };
  if constexpr (S == 1) {
    uint32_t B0[NCW], B1[NCW], B2[NCW];
    load(B0, 0);
    load(B1, 1);
    for (int r = 0; r < nrows; r += 3) {
      load(B2, r + 2);
      out_row(r, B0, B1, B2);
      if (r + 1 >= nrows) break;
      load(B0, r + 3);
      out_row(r + 1, B1, B2, B0);
      if (r + 2 >= nrows) break;
      load(B1, r + 4);
      out_row(r + 2, B2, B0, B1);
    }
  } else {
    uint32_t E0[NCW], E1[NCW], O[NCW];
    load(E0, 0);
    for (int r = 0; r < nrows; r += 2) {
      load(O, 2 * r + 1);
      load(E1, 2 * r + 2);
      out_row(r, E0, O, E1);
      if (r + 1 >= nrows) break;
      load(O, 2 * r + 3);
      load(E0, 2 * r + 4);
      out_row(r + 1, E1, O, E0);
    }
  }
}

// fp32 3x3 column-pair core (the fp32 DWPW's DW stage): a lane owns one fp32 channel of two
// adjacent output columns; each tap is one packed fma.rn.f32x2 over (x[col0 tap], x[col1 tap]) with
// the weight duplicated in both halves -- per column the same IEEE fp32 fma chain, in the same
// (i, j) order, as the scalar core. Rolled 3-row window as in dw3_cols_roll. sink(r, c, acc).
template <int S, int COLB, class Sink>
__device__ __forceinline__ void dw3_pair_f32(uint32_t src, int row_bytes, int nrows, const uint64_t (&W2)[9],
                                             Sink&& sink) {
  constexpr int NCW = S + 3;  // input words of a row feeding the two output columns
  auto load = [&](float (&dst)[NCW], int row) {
    const uint32_t rp = src + row * row_bytes;
#pragma unroll
    for (int j = 0; j < NCW; ++j) dst[j] = __uint_as_float(lds32(rp + j * COLB));
  };
  auto out_row = [&](int r, const float (&x0)[NCW], const float (&x1)[NCW], const float (&x2)[NCW]) {
    uint64_t acc = 0ull;  // (+0, +0)
#pragma unroll
    for (int j = 0; j < 3; ++j) acc = f2_fma(f2_pack(x0[j], x0[S + j]), W2[j], acc);
#pragma unroll
    for (int j = 0; j < 3; ++j) acc = f2_fma(f2_pack(x1[j], x1[S + j]), W2[3 + j], acc);
#pragma unroll
    for (int j = 0; j < 3; ++j) acc = f2_fma(f2_pack(x2[j], x2[S + j]), W2[6 + j], acc);
    float a, b;
    f2_unpack(acc, a, b);
    sink(r, 0, a);
    sink(r, 1, b);
  };
  if constexpr (S == 1) {
    float B0[NCW], B1[NCW], B2[NCW];
    load(B0, 0);
    load(B1, 1);
    for (int r = 0; r < nrows; r += 3) {
      load(B2, r + 2);
      out_row(r, B0, B1, B2);
      if (r + 1 >= nrows) break;
      load(B0, r + 3);
      out_row(r + 1, B1, B2, B0);
      if (r + 2 >= nrows) break;
      load(B1, r + 4);
      out_row(r + 2, B2, B0, B1);
    }
  } else {
    float E0[NCW], E1[NCW], O[NCW];
    load(E0, 0);
    for (int r = 0; r < nrows; r += 2) {
      load(O, 2 * r + 1);
      load(E1, 2 * r + 2);
      out_row(r, E0, O, E1);
      if (r + 1 >= nrows) break;
      load(O, 2 * r + 3);
      load(E0, 2 * r + 4);
      out_row(r + 1, E1, O, E0);
    }
  }
}

// Activation dispatch: one instantiation per activation (the runtime value picks it once).
template <class F>
__device__ __forceinline__ void with_act(int act, F&& f) {
  if (act == FCM_ACT_RELU6) f(std::integral_constant<int, 2>());
  else if (act == FCM_ACT_RELU) f(std::integral_constant<int, 1>());
  else if (act == FCM_ACT_SILU) f(std::integral_constant<int, 3>());
  else if (act == FCM_ACT_GELU) f(std::integral_constant<int, 4>());
  else f(std::integral_constant<int, 0>());
}

// with_act, or the RELU6 variant alone when the kernel is compiled for it
template <bool R6, class F>
__device__ __forceinline__ void with_act_r6(int act, F&& f) {
  if constexpr (R6) f(std::integral_constant<int, 2>());
  else with_act(act, static_cast<F&&>(f));
}

// fp32 pair (lo, hi) -> folded-BN affine (one FFMA2) -> packed bf16x2 / f16x2 with the activation
template <int DT, int ACT>
__device__ __forceinline__ uint32_t epi_act2(float lo, float hi, uint64_t sc2, uint64_t bi2, uint32_t hi_c) {
  float a, b;
  f2_unpack(f2_fma(f2_pack(lo, hi), sc2, bi2), a, b);
  uint32_t h;
  if constexpr (ACT >= FCM_ACT_SILU) {  // SiLU / GELU in fp32, then one rounding
    a = act_t<ACT>(a);
    b = act_t<ACT>(b);
    if constexpr (DT == FCM_BF16) asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    else asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
  } else if constexpr (DT == FCM_BF16) {
    if constexpr (ACT == 0) asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    else asm("cvt.rn.relu.bf16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    if constexpr (ACT == 2) asm("min.bf16x2 %0, %0, %1;" : "+r"(h) : "r"(hi_c));
  } else {
    if constexpr (ACT == 0) asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    else asm("cvt.rn.relu.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    if constexpr (ACT == 2) asm("min.f16x2 %0, %0, %1;" : "+r"(h) : "r"(hi_c));
  }
  return h;
}

// fp32 pair -> packed bf16x2 / f16x2 with the activation: ACT 0 none, 1 relu (free in the
// convert), 2 relu6 (relu convert + one packed min; 6 is exact in both formats).
template <int DT, int ACT>
__device__ __forceinline__ uint32_t pack_act(uint64_t acc, uint32_t hi2) {
  float a, b;
  f2_unpack(acc, a, b);
  uint32_t h;
  if constexpr (DT == FCM_BF16) {
    if constexpr (ACT == 0) asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    else asm("cvt.rn.relu.bf16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    if constexpr (ACT == 2) asm("min.bf16x2 %0, %0, %1;" : "+r"(h) : "r"(hi2));
  } else {
    if constexpr (ACT == 0) asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    else asm("cvt.rn.relu.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
    if constexpr (ACT == 2) asm("min.f16x2 %0, %0, %1;" : "+r"(h) : "r"(hi2));
  }
  return h;
}

// ---------------------------------------------------------------------------- int8 column-pair FFMA2 DW core
// int8, 3x3. Exact in fp32: every product |x w| <= 128 * 127 and every partial sum of the 9 taps
// (|acc| < 9 * 128 * 128 < 2^18) is an integer below 2^24, so FFMA2 accumulation is bit-exact
// whatever the order (SURVEY §8(c) "Exactness bound for fp32-accumulated int8 DW"). The int32
// bias is NOT folded into the fp32 accumulator (any int32 bias_q is allowed): callers start the
// accumulators at 0 and add bias_q in int32 after f2_to_i2. A lane owns one 32-bit word (4 channels) of
// two adjacent output columns: per input word one
// XOR + 4 byte permutes build 2^23 + (x + 128) as fp32 bit patterns, one FFMA2 pair subtracts
// 2^23 + 128 (exact), and the channel pairs (0,1), (2,3) feed packed FFMA2s.
__device__ __forceinline__ void i8word_to_f2x2(uint32_t w, uint64_t& lo, uint64_t& hi) {
  const uint32_t u = w ^ 0x80808080u;
  uint32_t b0, b1, b2, b3;
  asm("prmt.b32 %0, %1, 0x4B000000, 0x7440;" : "=r"(b0) : "r"(u));
  asm("prmt.b32 %0, %1, 0x4B000000, 0x7441;" : "=r"(b1) : "r"(u));
  asm("prmt.b32 %0, %1, 0x4B000000, 0x7442;" : "=r"(b2) : "r"(u));
  asm("prmt.b32 %0, %1, 0x4B000000, 0x7443;" : "=r"(b3) : "r"(u));
  const uint64_t one2 = f2_pack(1.f, 1.f), nb2 = f2_pack(-8388736.f, -8388736.f);
  lo = f2_fma(f2_pack(__uint_as_float(b0), __uint_as_float(b1)), one2, nb2);
  hi = f2_fma(f2_pack(__uint_as_float(b2), __uint_as_float(b3)), one2, nb2);
}

template <int S, int SEG, class Sink>
__device__ __forceinline__ void dw3_pair_i8(uint32_t src, int col_bytes, int row_bytes, int y0, int max_row,
                                            const uint64_t (&W)[9][2], const uint64_t (&bias)[2], Sink&& sink) {
  constexpr int NCW = 3 + S;
  constexpr int WR = (SEG - 1) * S + 3;
  constexpr int PD = 2;
  uint64_t acc[SEG][2][2];
  uint32_t raw[WR][NCW];
  auto load_row = [&](int ii) {
    const uint32_t rp = src + min(y0 * S + ii, max_row) * row_bytes;
#pragma unroll
    for (int j = 0; j < NCW; ++j) raw[ii][j] = lds32(rp + j * col_bytes);
  };
#pragma unroll
  for (int ii = 0; ii < PD && ii < WR; ++ii) load_row(ii);
#pragma unroll
  for (int ii = 0; ii < WR; ++ii) {
    if (ii + PD < WR) load_row(ii + PD);
    uint64_t x[NCW][2];
#pragma unroll
    for (int j = 0; j < NCW; ++j) i8word_to_f2x2(raw[ii][j], x[j][0], x[j][1]);
#pragma unroll
    for (int r = 0; r < SEG; ++r) {
      const int i = ii - r * S;
      if (i < 0 || i > 2) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            acc[r][c][h] = f2_fma(x[c * S + j][h], W[i * 3 + j][h], (i == 0 && j == 0) ? bias[h] : acc[r][c][h]);
      if (i == 2) sink(r, acc[r]);
    }
  }
}

// Per-channel int8 requantiser in the form the FFMA2 core's epilogue uses. For sh >= 33 the
// rounding term 2^(sh-1) has no low-word bits, so (acc M + 2^(sh-1)) >> sh ==
// (mulhi(acc, M) + 2^(sh-33)) >> (sh-32) exactly (floor((n + f) / 2^k) = floor(n / 2^k) for integer
// n, 0 <= f < 1): one mad.hi + one shift. Smaller shifts take the 64-bit form.
struct RqI8 {
  int32_t m, c, s;  // multiplier, addend, shift (fast form: c = 2^(sh-33), s = sh - 32; else c = -1, s = sh)
};
__device__ __forceinline__ RqI8 make_rq(int32_t m, int32_t sh) {
  return sh >= 33 ? RqI8{m, 1 << (sh - 33), sh - 32} : RqI8{m, -1, sh};
}
__device__ __forceinline__ int32_t rq_apply(int32_t a, const RqI8& q) {
  if (q.c >= 0) {
    int32_t h;
    asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(h) : "r"(a), "r"(q.m), "r"(q.c));
    return h >> q.s;
  }
  const long long p = static_cast<long long>(a) * q.m + (1LL << (q.s - 1));
  return static_cast<int32_t>(p >> q.s);
}
// fp32 pair holding exact integers |v| < 2^22 -> int32 pair (magic-number rounding: the bits of
// v + 1.5 * 2^23 are 0x4B400000 + v).
__device__ __forceinline__ void f2_to_i2(uint64_t v, int32_t& a, int32_t& b) {
  float x, y;
  f2_unpack(f2_fma(v, f2_pack(1.f, 1.f), f2_pack(12582912.f, 12582912.f)), x, y);
  a = static_cast<int32_t>(__float_as_uint(x) - 0x4B400000u);
  b = static_cast<int32_t>(__float_as_uint(y) - 0x4B400000u);
}

// Stage the 3x3 DW weights of C channels for dw3_cols_h: the raw packed weight words [9][cwords]
// (uint32, 2 channels each) followed by the per-word folded-BN scale pairs [cwords] and bias pairs
// [cwords] (fp32 pairs as uint64), all zero past C. dw3h_bytes(cwords) bytes.
constexpr int dw3h_bytes(int cwords) { return 52 * cwords; }
template <int DT>
__device__ __forceinline__ void stage_dw3_h(const void* wdw, const Epi& e, int C, int cwords, uint32_t* wsm) {
  const uint32_t* g = static_cast<const uint32_t*>(wdw);
  const int cw_real = C / 2;
  for (int i = threadIdx.x; i < 9 * cwords; i += blockDim.x) {
    const int t = i / cwords, w = i - t * cwords;
    wsm[i] = w < cw_real ? __ldg(g + t * cw_real + w) : 0u;
  }
  uint64_t* sb = reinterpret_cast<uint64_t*>(wsm + 9 * cwords);
  for (int w = threadIdx.x; w < cwords; w += blockDim.x) {
    const bool v = w < cw_real;
    const float s0 = v ? (e.scale ? __ldg(e.scale + 2 * w) : 1.f) : 0.f;
    const float s1 = v ? (e.scale ? __ldg(e.scale + 2 * w + 1) : 1.f) : 0.f;
    const float b0 = (v && e.bias) ? __ldg(e.bias + 2 * w) : 0.f;
    const float b1 = (v && e.bias) ? __ldg(e.bias + 2 * w + 1) : 0.f;
    sb[w] = f2_pack(s0, s1);
    sb[cwords + w] = f2_pack(b0, b1);
  }
}
// This lane's word `cw` of the staged weights: 9 packed taps + scale / bias pairs.
__device__ __forceinline__ void load_dw3_h(const uint32_t* wsm, int cwords, int cw, uint32_t (&W)[9], uint64_t& sc2,
                                           uint64_t& bi2) {
  const uint32_t a = smem_u32(wsm) + 4 * cw;
#pragma unroll
  for (int q = 0; q < 9; ++q) W[q] = lds32(a + 4 * q * cwords);
  const uint32_t sa = smem_u32(wsm) + 36 * cwords + 8 * cw;
  sc2 = lds64(sa);
  bi2 = lds64(sa + 8 * cwords);
}

// K-major operand without swizzle (UMMA "interleave" layout): row m of 16-byte channel chunk q at
// m * 16 + q * kAlbo. kAlbo = 2064 (not 2048) puts the 8 chunks of one row in distinct bank
// groups, so a warp's 32 words of one pixel store without bank conflicts. 8-row core matrices are
// 128 B contiguous (SBO = 128).
constexpr int kAlbo = 2064;
constexpr int kAbytes = 17408;  // 8 * kAlbo rounded up to 1 KB (also >= one 128 x 128 B SW128 tile)
__device__ __forceinline__ uint64_t smem_desc_interleave(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;  // LBO: next 16-byte K chunk
  d |= static_cast<uint64_t>(128 >> 4) << 32;            // SBO: next 8-row group
  d |= static_cast<uint64_t>(1) << 46;                   // version (sm_100)
  return d;                                              // layout type 0 = SWIZZLE_NONE
}
__device__ __forceinline__ uint64_t smem_desc_interleave(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(kAlbo >> 4) << 16;        // LBO: next 16-byte K chunk
  d |= static_cast<uint64_t>(128 >> 4) << 32;          // SBO: next 8-row group
  d |= static_cast<uint64_t>(1) << 46;                 // version (sm_100)
  return d;                                            // layout type 0 = SWIZZLE_NONE
}

// Ring-buffer position for the single-thread producer / consumer loops: slot index and mbarrier
// phase advanced incrementally (a runtime `it % n` / `it / n` is a ~25-instruction dependent chain
// on the critical path of a lone issuing thread).
struct Ring {
  int i, n;
  uint32_t ph;
  __device__ __forceinline__ explicit Ring(int n_) : i(0), n(n_), ph(0) {}
  __device__ __forceinline__ void next() {
    if (++i == n) {
      i = 0;
      ph ^= 1u;
    }
  }
};

}  // namespace fcm
