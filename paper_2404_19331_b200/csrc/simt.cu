// CUDA-core (SIMT) paths, templated on the dtype:
//  * fp32 everywhere for PW / DWPW / PWDW_R -- the north_star's "CUDA-core fallback for thin
//    layers" and the paper's own FP32 kernels: fp32 keeps 1e-5 relative accuracy, which a
//    single TF32 tensor-core pass cannot (R10b);
//  * any dtype whose NHWC channel pitch is not a multiple of 16 bytes (e.g. int8 C = 24 / 40 in
//    EfficientNet-B0), which TMA cannot address.
// Same structure as the tensor-core FCMs: the intermediate T lives only in shared memory and is
// rounded / requantised to the feature-map dtype before the second convolution.
#include <cstdint>

#include "common.cuh"
#include "host.h"

namespace fcm {

template <int DT>
__device__ __forceinline__ typename Tr<DT>::acc_t to_acc(typename Tr<DT>::T v) {
  if constexpr (DT == FCM_S8) return static_cast<int32_t>(v);
  else if constexpr (DT == FCM_F32) return v;
  else if constexpr (DT == FCM_BF16) return __bfloat162float(v);
  else return __half2float(v);
}

template <int DT>
__device__ __forceinline__ typename Tr<DT>::acc_t mac(typename Tr<DT>::acc_t a, typename Tr<DT>::acc_t b,
                                                     typename Tr<DT>::acc_t c) {
  if constexpr (DT == FCM_S8) return a * b + c;
  else return fmaf(a, b, c);
}

// Conv-Norm-Act of one accumulator -> storage value; `oidx` = the element's index in the output
// (for the optional residual, float paths; SIZE_MAX on intermediate T writes).
template <int DT>
__device__ __forceinline__ typename Tr<DT>::T epi1(typename Tr<DT>::acc_t a, const EpiC& c, const Epi& e,
                                                   size_t oidx = SIZE_MAX) {
  if constexpr (DT == FCM_S8) {
    return static_cast<int8_t>(requant_i8(a, c, e.zp_out, e.qmin, e.qmax));
  } else {
    const float r = (e.residual && oidx != SIZE_MAX) ? res_at<DT>(e.residual, oidx) : 0.f;
    const float v = epi_fr(a, c.sc, c.bi, e.act, r);
    if constexpr (DT == FCM_F32) return v;
    else if constexpr (DT == FCM_BF16) return __float2bfloat16_rn(v);
    else return __float2half_rn(v);
  }
}

// ------------------------------------------------------------------ LBL PW
// Y[M,N] = eps(X[M,K] . Wp[N,K]^T). 64x64 output tile per CTA, 4x4 per thread, K chunks of 16.
// VEC (row pitches of X / Wp a multiple of 8 bytes and N a multiple of 4): operands staged with
// 8-byte loads and the 4 consecutive outputs of a thread written as one vector store, instead
// of element-wise (byte-wise for int8) global accesses.
template <int DT>
__device__ __forceinline__ void store4(typename Tr<DT>::T* y, const typename Tr<DT>::T (&v)[4]) {
  if constexpr (DT == FCM_S8) {
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) w |= (static_cast<uint32_t>(static_cast<uint8_t>(v[j])) << (8 * j));
    *reinterpret_cast<uint32_t*>(y) = w;
  } else if constexpr (DT == FCM_F32) {
    *reinterpret_cast<float4*>(y) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    uint2 w;
    w.x = static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(&v[0])) |
          (static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(&v[1])) << 16);
    w.y = static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(&v[2])) |
          (static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(&v[3])) << 16);
    *reinterpret_cast<uint2*>(y) = w;
  }
}

// int8 with 8-byte pitches: the K chunk stays packed (4 int8 per word) and every word pair is
// one __dp4a (4 exact int32 MACs per instruction instead of one IMAD each).
__device__ __forceinline__ void pw_simt_i8_dp4a(const int8_t* __restrict__ x, const int8_t* __restrict__ wp,
                                                const Epi& ep, int8_t* __restrict__ y, int M, int K, int N) {
  __shared__ uint32_t xw[4][64 + 4];
  __shared__ uint32_t ww[4][64 + 4];
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  int32_t acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    {  // 2 x 64 rows x 2 groups of 8 bytes = 256 loads: one per thread
      const int i = threadIdx.x;
      const int which = i >> 7, rem = i & 127, r = rem >> 1, gi = rem & 1, kk = gi * 8;
      const int row = (which ? n0 : m0) + r;
      uint2 g = make_uint2(0u, 0u);
      if (row < (which ? N : M) && k0 + kk < K)
        g = __ldg(reinterpret_cast<const uint2*>((which ? wp : x) + (size_t)row * K + k0 + kk));
      uint32_t(*dst)[64 + 4] = which ? ww : xw;
      dst[2 * gi][r] = g.x;
      dst[2 * gi + 1][r] = g.y;
    }
    __syncthreads();
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      int a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = (int)xw[kq][ty * 4 + i]; b[i] = (int)ww[kq][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dp4a(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int nb = n0 + tx * 4;
  if (nb >= N) return;
  EpiC c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = load_epi<FCM_S8>(ep, nb + j, true);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w |= (static_cast<uint32_t>(requant_i8(acc[i][j], c[j], ep.zp_out, ep.qmin, ep.qmax)) & 0xFFu) << (8 * j);
    *reinterpret_cast<uint32_t*>(y + (size_t)m * N + nb) = w;
  }
}

template <int DT, bool VEC>
__global__ void __launch_bounds__(256) pw_simt_kernel(const typename Tr<DT>::T* __restrict__ x,
                                                      const typename Tr<DT>::T* __restrict__ wp, Epi ep,
                                                      typename Tr<DT>::T* __restrict__ y, int M, int K, int N) {
  pdl_launch();
  pdl_wait();
  if constexpr (DT == FCM_S8 && VEC) {
    pw_simt_i8_dp4a(x, wp, ep, y, M, K, N);
    return;
  }
  using A = typename Tr<DT>::acc_t;
  using TT = typename Tr<DT>::T;
  constexpr int V = Tr<DT>::VEC;          // elements per 32-bit word
  constexpr int EPG = 2 * V;              // elements per 8-byte group
  __shared__ A xs[16][64 + 4];
  __shared__ A ws[16][64 + 4];
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  A acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    if constexpr (VEC) {
      constexpr int GPR = 16 / EPG;       // 8-byte groups per row of the K chunk
      for (int i = threadIdx.x; i < 2 * 64 * GPR; i += 256) {
        const int which = i / (64 * GPR), rem = i - which * 64 * GPR;
        const int r = rem / GPR, gi = rem - r * GPR, kk = gi * EPG;
        const int row = (which ? n0 : m0) + r;
        const bool ok = row < (which ? N : M) && k0 + kk < K;
        uint2 g = make_uint2(0u, 0u);
        if (ok) g = __ldg(reinterpret_cast<const uint2*>((which ? wp : x) + (size_t)row * K + k0 + kk));
        A u0[V], u1[V];
        Tr<DT>::unpack(g.x, u0);
        Tr<DT>::unpack(g.y, u1);
        A(*dst)[64 + 4] = which ? ws : xs;
#pragma unroll
        for (int e = 0; e < V; ++e) {
          dst[kk + e][r] = u0[e];
          dst[kk + V + e][r] = u1[e];
        }
      }
    } else {
      for (int i = threadIdx.x; i < 64 * 16; i += 256) {
        const int r = i / 16, kk = i % 16;
        xs[kk][r] = (m0 + r < M && k0 + kk < K) ? to_acc<DT>(x[(size_t)(m0 + r) * K + k0 + kk]) : A(0);
        ws[kk][r] = (n0 + r < N && k0 + kk < K) ? to_acc<DT>(wp[(size_t)(n0 + r) * K + k0 + kk]) : A(0);
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      A a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = xs[kk][ty * 4 + i]; b[i] = ws[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = mac<DT>(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  if constexpr (VEC) {
    const int nb = n0 + tx * 4;
    if (nb >= N) return;
    EpiC c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = load_epi<DT>(ep, nb + j, true);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m >= M) continue;
      TT v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = epi1<DT>(acc[i][j], c[j], ep, (size_t)m * N + nb + j);
      store4<DT>(y + (size_t)m * N + nb, v);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      const EpiC c = load_epi<DT>(ep, n, true);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m < M) y[(size_t)m * N + n] = epi1<DT>(acc[i][j], c, ep, (size_t)m * N + n);
      }
    }
  }
}

template <int DT>
__device__ __forceinline__ typename Tr<DT>::acc_t dw_tap_sum(const typename Tr<DT>::T* __restrict__ x,
                                                            const typename Tr<DT>::T* __restrict__ wdw, int n, int H,
                                                            int W, int C, int c, int yo, int xo, int k, int s, int pt,
                                                            int pl) {
  typename Tr<DT>::acc_t acc = 0;
  for (int i = 0; i < k; ++i) {
    const int yi = yo * s - pt + i;
    if (yi < 0 || yi >= H) continue;
    for (int j = 0; j < k; ++j) {
      const int xi = xo * s - pl + j;
      if (xi < 0 || xi >= W) continue;
      acc = mac<DT>(to_acc<DT>(x[(((size_t)n * H + yi) * W + xi) * C + c]), to_acc<DT>(wdw[(i * k + j) * C + c]), acc);
    }
  }
  return acc;
}

// ------------------------------------------------------------------ LBL DW (NHWC, any pitch)
template <int DT>
__global__ void dw_nhwc_simt_kernel(const typename Tr<DT>::T* __restrict__ x, const typename Tr<DT>::T* __restrict__ wdw,
                                    Epi ep, typename Tr<DT>::T* __restrict__ y, int H, int W, int C, int Ho, int Wo,
                                    int k, int s, int pt, int pl, long long total) {
  pdl_launch();
  pdl_wait();
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = idx % C;
    long long r = idx / C;
    const int xo = r % Wo;
    r /= Wo;
    const int yo = r % Ho;
    const int n = r / Ho;
    const auto a = dw_tap_sum<DT>(x, wdw, n, H, W, C, c, yo, xo, k, s, pt, pl);
    y[idx] = epi1<DT>(a, load_epi<DT>(ep, c, true), ep);
  }
}

// ------------------------------------------------------------------ FCM DWPW
// CTA = 8x8 output pixels x 64 output channels; C_in streams in chunks of 32 through the smem
// commBuffer T[32][64]; PW partial sums stay in registers (OS).
template <int DT>
__global__ void __launch_bounds__(256) dwpw_simt_kernel(const typename Tr<DT>::T* __restrict__ x,
                                                        const typename Tr<DT>::T* __restrict__ wdw, Epi ed,
                                                        const typename Tr<DT>::T* __restrict__ wp, Epi ep,
                                                        typename Tr<DT>::T* __restrict__ y, int N, int H, int W, int C,
                                                        int Ho, int Wo, int Cout, int k, int s, int pt, int pl,
                                                        int tiles_x, int tiles_y) {
  pdl_launch();
  pdl_wait();
  using A = typename Tr<DT>::acc_t;
  __shared__ A ts[32][64 + 4];
  __shared__ A ws[32][64 + 4];
  int t = blockIdx.x;
  const int txi = t % tiles_x;
  t /= tiles_x;
  const int tyi = t % tiles_y;
  const int n = t / tiles_y;
  const int n0 = blockIdx.y * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  A acc[4][4] = {};
  for (int c0 = 0; c0 < C; c0 += 32) {
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int p = i % 64, cc = i / 64;
      const int c = c0 + cc;
      const int yo = tyi * 8 + p / 8, xo = txi * 8 + p % 8;
      A v = 0;
      if (c < C && yo < Ho && xo < Wo) {
        const A a = dw_tap_sum<DT>(x, wdw, n, H, W, C, c, yo, xo, k, s, pt, pl);
        v = to_acc<DT>(epi1<DT>(a, load_epi<DT>(ed, c, true), ed));  // T in the FM dtype
      }
      ts[cc][p] = v;
      const int co = n0 + p;
      ws[cc][p] = (c < C && co < Cout) ? to_acc<DT>(wp[(size_t)co * C + c]) : A(0);
    }
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < 32; ++cc) {
      A a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = ts[cc][ty * 4 + i]; b[i] = ws[cc][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = mac<DT>(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int co = n0 + tx * 4 + j;
    if (co >= Cout) continue;
    const EpiC c = load_epi<DT>(ep, co, true);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int p = ty * 4 + i;
      const int yo = tyi * 8 + p / 8, xo = txi * 8 + p % 8;
      if (yo < Ho && xo < Wo) {
        const size_t o = (((size_t)n * Ho + yo) * Wo + xo) * Cout + co;
        y[o] = epi1<DT>(acc[i][j], c, ep, o);
      }
    }
  }
}

// ------------------------------------------------------------------ FCM PWDW_R
// CTA = 8x8 DW output pixels x 32 intermediate channels. T is computed over the halo tile
// (recomputed overlap) into smem, zero (the zero point) outside the image, then the DW reads it.
template <int DT>
__global__ void __launch_bounds__(256) pwdw_simt_kernel(const typename Tr<DT>::T* __restrict__ x,
                                                        const typename Tr<DT>::T* __restrict__ wp, Epi ep,
                                                        const typename Tr<DT>::T* __restrict__ wdw, Epi ed,
                                                        typename Tr<DT>::T* __restrict__ y, int N, int H, int W, int C,
                                                        int Ho, int Wo, int Cmid, int k, int s, int pt, int pl,
                                                        int tiles_x, int tiles_y) {
  pdl_launch();
  pdl_wait();
  using A = typename Tr<DT>::acc_t;
  extern __shared__ __align__(16) unsigned char tsm_raw[];  // [R][33] acc_t
  A* tsm = reinterpret_cast<A*>(tsm_raw);
  int t = blockIdx.x;
  const int txi = t % tiles_x;
  t /= tiles_x;
  const int tyi = t % tiles_y;
  const int n = t / tiles_y;
  const int cm0 = blockIdx.y * 32;
  const int win = 7 * s + k;
  const int R = win * win;
  const int y_in0 = tyi * 8 * s - pt, x_in0 = txi * 8 * s - pl;
  for (int i = threadIdx.x; i < R * 32; i += 256) {
    const int cc = i % 32, r = i / 32;
    const int yi = y_in0 + r / win, xi = x_in0 + r % win;
    const int cm = cm0 + cc;
    A v = 0;
    if (cm < Cmid && yi >= 0 && yi < H && xi >= 0 && xi < W) {
      const typename Tr<DT>::T* xp = x + (((size_t)n * H + yi) * W + xi) * C;
      const typename Tr<DT>::T* wr = wp + (size_t)cm * C;
      A a = 0;
      for (int ci = 0; ci < C; ++ci) a = mac<DT>(to_acc<DT>(xp[ci]), to_acc<DT>(wr[ci]), a);
      v = to_acc<DT>(epi1<DT>(a, load_epi<DT>(ep, cm, true), ep));
      if constexpr (DT == FCM_S8) v -= ed.zp_in;  // (T - zp_T): out-of-image taps contribute 0
    }
    tsm[r * 33 + cc] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 32; i += 256) {
    const int cc = i % 32, p = i / 32;
    const int cm = cm0 + cc;
    const int yo = tyi * 8 + p / 8, xo = txi * 8 + p % 8;
    if (cm >= Cmid || yo >= Ho || xo >= Wo) continue;
    A a = 0;
    for (int ii = 0; ii < k; ++ii)
      for (int jj = 0; jj < k; ++jj)
        a = mac<DT>(tsm[((p / 8) * s + ii) * win * 33 + ((p % 8) * s + jj) * 33 + cc],
                    to_acc<DT>(wdw[(ii * k + jj) * Cmid + cm]), a);
    y[(((size_t)n * Ho + yo) * Wo + xo) * Cmid + cm] = epi1<DT>(a, load_epi<DT>(ed, cm, true), ed);
  }
}

// ------------------------------------------------------------------ launchers
#define FCM_DT_SWITCH(dt, F)                        \
  switch (dt) {                                     \
    case FCM_F32: return F(FCM_F32);                \
    case FCM_BF16: return F(FCM_BF16);              \
    case FCM_F16: return F(FCM_F16);                \
    case FCM_S8: return F(FCM_S8);                  \
  }                                                 \
  return set_error(FCM_E_INVAL, "bad dtype");

int launch_pw_simt(int dt, const void* x, const void* wp, const Epi& ep, void* y, int M, int K, int N,
                   cudaStream_t st) {
  dim3 grid((M + 63) / 64, (N + 63) / 64);
  const int es = elem_size(dt);
  const bool vec = ((size_t)K * es) % 8 == 0 && N % 4 == 0;
#define L_PW(D)                                                                                                 \
  ((vec ? launch_k(pw_simt_kernel<D, true>, dim3(grid), dim3(256), 0, st, static_cast<const Tr<D>::T*>(x),    \
                   static_cast<const Tr<D>::T*>(wp), ep, static_cast<Tr<D>::T*>(y), M, K, N)                   \
        : launch_k(pw_simt_kernel<D, false>, dim3(grid), dim3(256), 0, st, static_cast<const Tr<D>::T*>(x),   \
                   static_cast<const Tr<D>::T*>(wp), ep, static_cast<Tr<D>::T*>(y), M, K, N)),                 \
   check_launch("pw_simt_kernel"))
  FCM_DT_SWITCH(dt, L_PW)
#undef L_PW
}

int launch_dw_simt(int dt, const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  const long long total = (long long)g.N * g.Ho * g.Wo * g.C;
  const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)device_props().sms * 16);
#define L_DW(D)                                                                                            \
  (launch_k(dw_nhwc_simt_kernel<D>, dim3(blocks), dim3(256), 0, st, static_cast<const Tr<D>::T*>(x), static_cast<const Tr<D>::T*>(wdw), \
                                                   ep, static_cast<Tr<D>::T*>(y), g.H, g.W, g.C, g.Ho, g.Wo, g.k, g.s,  \
                                                   g.pt, g.pl, total),                                     \
   check_launch("dw_nhwc_simt_kernel"))
  FCM_DT_SWITCH(dt, L_DW)
#undef L_DW
}

int launch_dwpw_simt(int dt, const void* x, const void* wdw, const Epi& ed, const void* wp, const Epi& ep, void* y,
                     const Geo& g, cudaStream_t st) {
  const int tiles_x = (g.Wo + 7) / 8, tiles_y = (g.Ho + 7) / 8;
  dim3 grid(tiles_x * tiles_y * g.N, (g.Cout + 63) / 64);
#define L_DWPW(D)                                                                                          \
  (launch_k(dwpw_simt_kernel<D>, dim3(grid), dim3(256), 0, st, static_cast<const Tr<D>::T*>(x), static_cast<const Tr<D>::T*>(wdw), ed, \
                                             static_cast<const Tr<D>::T*>(wp), ep, static_cast<Tr<D>::T*>(y), g.N, g.H,   \
                                             g.W, g.C, g.Ho, g.Wo, g.Cout, g.k, g.s, g.pt, g.pl, tiles_x, tiles_y),  \
   check_launch("dwpw_simt_kernel"))
  FCM_DT_SWITCH(dt, L_DWPW)
#undef L_DWPW
}

template <int DT>
static int launch_pwdw_simt_t(const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                              const Geo& g, cudaStream_t st) {
  const int tiles_x = (g.Wo + 7) / 8, tiles_y = (g.Ho + 7) / 8;
  const int hin = 7 * g.s + g.k;
  const size_t smem = (size_t)hin * hin * 33 * sizeof(typename Tr<DT>::acc_t);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(pwdw_simt_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(tiles_x * tiles_y * g.N, (g.Cout + 31) / 32);
  using TT = typename Tr<DT>::T;
  launch_k(pwdw_simt_kernel<DT>, dim3(grid), dim3(256), smem, st, static_cast<const TT*>(x), static_cast<const TT*>(wp), ep,
                                                static_cast<const TT*>(wdw), ed, static_cast<TT*>(y), g.N, g.H, g.W,
                                                g.C, g.Ho, g.Wo, g.Cout, g.k, g.s, g.pt, g.pl, tiles_x, tiles_y);
  return check_launch("pwdw_simt_kernel");
}

int launch_pwdw_simt(int dt, const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                     const Geo& g, cudaStream_t st) {
#define L_PWDW(D) launch_pwdw_simt_t<D>(x, wp, ep, wdw, ed, y, g, st)
  FCM_DT_SWITCH(dt, L_PWDW)
#undef L_PWDW
}

}  // namespace fcm
