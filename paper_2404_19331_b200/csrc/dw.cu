// Layer-by-layer depthwise convolution (fcm_dw; the paper's LBL DW kernel) and the
// offline PW weight packing kernel.
//
// NHWC path: one CTA per (output tile th x tw, 128-byte channel group). The input halo tile
// ((th-1)s+k) x ((tw-1)s+k) x 128 B is staged in shared memory by ONE TMA load whose
// out-of-bounds fill provides the zero padding (overlapping halos are re-loaded per
// tile -- on B200 they are L2 hits). Lane = one 32-bit word of channels (conflict-free smem
// reads); warps own output columns and slide a k x k register window down them, so each
// staged word is read once per column. Output stores are 128 B per warp instruction.
#include "common.cuh"
#include "host.h"

#include <cstring>

namespace fcm {

// TMA = false: the pixel pitch C * b is not a multiple of 16 bytes (e.g. int8 C = 728), which TMA
// cannot address; all threads stage the same halo tile with 8- or 4-byte cp.async (zero-filled
// outside the image and past C) and the compute below is unchanged.
template <int DT, int K, int S, bool TMA>
__global__ void __launch_bounds__(128) dw_nhwc_kernel(const __grid_constant__ CUtensorMap tmx,
                                                      const typename Tr<DT>::T* __restrict__ wdw, Epi ep,
                                                      typename Tr<DT>::T* __restrict__ y, int C, int Ho, int Wo,
                                                      int pt, int pl, int th, int tw, int tiles_x, int tiles_y, int pb,
                                                      const uint8_t* __restrict__ xr, int H, int W, int chunk) {
  pdl_launch();
  pdl_wait();
  constexpr int V = Tr<DT>::VEC;
  constexpr int KC = 32 * V;  // channels per 128-byte group
  extern __shared__ __align__(128) uint32_t xs[];
  __shared__ uint64_t bar;
  const int th_in = (th - 1) * S + K, tw_in = (tw - 1) * S + K;
  int t = blockIdx.x;
  const int tx = t % tiles_x;
  t /= tiles_x;
  const int ty = t % tiles_y;
  const int n = t / tiles_y;
  const int c0 = blockIdx.y * KC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pwd = pb >> 2;  // staged 32-bit words per pixel (128 B, or C * ES when C is narrower)
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      tma_prefetch_desc(&tmx);
      mbar_init(&bar, 1);
      fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, th_in * tw_in * pb);
      tma_load_4d(xs, &tmx, &bar, c0, tx * tw * S - pl, ty * th * S - pt, n);
    }
  } else {
    constexpr int ES = Tr<DT>::ES;
    const int cpp = pb / chunk, cbytes = C * ES, gy0 = ty * th * S - pt, gx0 = tx * tw * S - pl;
    const uint32_t base = smem_u32(xs);
    for (int i = threadIdx.x; i < th_in * tw_in * cpp; i += blockDim.x) {
      const int p = i / cpp, q = i - p * cpp;
      const int iy = p / tw_in, ix = p - iy * tw_in;
      const int gy = gy0 + iy, gx = gx0 + ix, boff = c0 * ES + q * chunk;
      const bool v = gy >= 0 && gy < H && gx >= 0 && gx < W && boff < cbytes;
      const uint8_t* src = v ? xr + ((static_cast<size_t>(n) * H + gy) * W + gx) * cbytes + boff : xr;
      if (chunk == 8) cp_async_ca<8>(base + p * pb + q * 8, src, v ? 8 : 0);
      else cp_async_ca<4>(base + p * pb + q * 4, src, v ? 4 : 0);
    }
  }
  auto wait_x = [&]() {
    if constexpr (TMA) {
      mbar_wait(&bar, 0);
    } else {
      cp_async_wait_all();
      __syncthreads();
    }
  };
  const int y0 = ty * th, x0 = tx * tw;
  const int nrows = min(th, Ho - y0);
  uint32_t* yw = reinterpret_cast<uint32_t*>(y);
  constexpr bool kPair = (DT == FCM_BF16 || DT == FCM_F16) && K == 3;
  if constexpr (kPair) {
    // same paired-FP32 core and segment length as the fused kernels (bit-identical DW); a partly
    // filled channel group packs 2 or 4 output columns per warp (gs lanes per pixel)
    constexpr int kSeg = (S == 1) ? 16 : 8;
    const int cw_valid = min(32, (C - c0) / V);
    const int gs = cw_valid > 16 ? 32 : (cw_valid > 8 ? 16 : 8);
    const int npix = 32 / gs, grp = lane / gs, wd = lane - grp * gs;
    const int cl = c0 + wd * V;
    const bool cval = wd < cw_valid;
    DwWh<K> W2;
    load_dw_weights_h<K>(W2, wdw, C, cval ? cl : C);
    const uint64_t sc2 = f2_pack(cval ? (ep.scale ? ep.scale[cl] : 1.f) : 0.f, cval ? (ep.scale ? ep.scale[cl + 1] : 1.f) : 0.f);
    const uint64_t bi2 = f2_pack(cval && ep.bias ? ep.bias[cl] : 0.f, cval && ep.bias ? ep.bias[cl + 1] : 0.f);
    const uint32_t hi_c = bound2<DT>(act_hi(ep.act));
    wait_x();
    const int nseg = (nrows + kSeg - 1) / kSeg;
    const int ncolg = (tw + npix - 1) / npix;
    // same epilogue as the fused kernels' DW stage (epi_act2): LBL and fused DW are bit-identical
    with_act(ep.act, [&](auto actc) {
      constexpr int ACT = decltype(actc)::value;
      for (int item = warp; item < ncolg * nseg; item += 4) {
        const int cg = item / nseg, seg = item - cg * nseg;
        const int col = cg * npix + grp;
        const int x = x0 + col;
        const bool live = col < tw && x < Wo && cval;
        const int ys = seg * kSeg;
        const uint32_t src = smem_u32(xs) + (((live ? col : 0) * S) * pwd + wd) * 4;
        uint32_t* dst = yw + (((static_cast<size_t>(n) * Ho + (y0 + ys)) * Wo + (live ? x : 0)) * C + cl) / V;
        const size_t rstride = (size_t)Wo * C / V;
        const int nvalid = live ? nrows - ys : 0;
        dw_segh<DT, K, S, kSeg>(src, pb, tw_in * pb, ys, th_in - 1, W2, [&](int r, uint64_t acc) {
          float lo, hi;
          f2_unpack(acc, lo, hi);
          if (r < nvalid) dst[r * rstride] = epi_act2<DT, ACT>(lo, hi, sc2, bi2, hi_c);
        });
      }
    });
    return;
  } else if constexpr (DT == FCM_S8 && K == 3) {
    // int8 column-pair FFMA2 core (exact, see dw3_pair_i8); a lane owns one word (4 channels) of
    // two adjacent output columns; lane groups for partly filled 128-channel groups as above
#ifndef FCM_I8SEG
#define FCM_I8SEG 8
#endif
    constexpr int kSeg = (S == 1) ? FCM_I8SEG : 4;
    const int cw_valid = min(32, (C - c0) / 4);
    const int gs = cw_valid > 16 ? 32 : (cw_valid > 8 ? 16 : 8);
    const int npix = 32 / gs, grp = lane / gs, wd = lane - grp * gs;
    const int cl = c0 + wd * 4;
    const bool cval = wd < cw_valid;
    // the accumulators start at 0 and bias_q is added in int32 after the exact fp32 -> int32
    // conversion: the fp32 path is exact only below 2^22 (the 9 products: < 2^18), bias_q is any int32
    const uint64_t bias[2] = {0ull, 0ull};
    uint64_t W[9][2];
    int32_t bq[4];
    RqI8 rq[4];
    {
      const uint32_t* g = reinterpret_cast<const uint32_t*>(wdw);
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const uint32_t w = cval ? __ldg(g + t * (C / 4) + cl / 4) : 0u;
        float f[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) f[v] = static_cast<float>(static_cast<int32_t>(w << (24 - 8 * v)) >> 24);
        W[t][0] = f2_pack(f[0], f[1]);
        W[t][1] = f2_pack(f[2], f[3]);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        bq[v] = (cval && ep.bias_q) ? __ldg(ep.bias_q + cl + v) : 0;
        rq[v] = make_rq(cval ? __ldg(ep.mult_q + cl + v) : 0, cval ? __ldg(ep.shift_q + cl + v) : 40);
      }
    }
    const int zp = ep.zp_out, qmin = ep.qmin, qmax = ep.qmax;
    wait_x();
    const int nseg = (nrows + kSeg - 1) / kSeg;
    const int ncolp = (tw + 1) / 2;
    const int ncolg = (ncolp + npix - 1) / npix;
    const size_t rstride = (size_t)Wo * C / 4;
    for (int item = warp; item < ncolg * nseg; item += 4) {
      const int cg = item / nseg, seg = item - cg * nseg;
      const int cp = cg * npix + grp;
      const int col = 2 * cp, x = x0 + col;
      const bool live0 = cp < ncolp && x < Wo && cval;
      const bool live1 = live0 && col + 1 < tw && x + 1 < Wo;
      const int ys = seg * kSeg;
      const uint32_t src = smem_u32(xs) + (((live0 ? col : 0) * S) * pwd + wd) * 4;
      uint32_t* dst = yw + (((static_cast<size_t>(n) * Ho + (y0 + ys)) * Wo + (live0 ? x : 0)) * C + cl) / 4;
      const int nvalid = live0 ? nrows - ys : 0;
      dw3_pair_i8<S, kSeg>(src, pb, tw_in * pb, ys, th_in - 1, W, bias, [&](int r, const uint64_t (&a)[2][2]) {
        if (r < nvalid) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            int32_t v[4];
            f2_to_i2(a[c][0], v[0], v[1]);
            f2_to_i2(a[c][1], v[2], v[3]);
            int32_t o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = min(rq_apply(v[q] + bq[q], rq[q]) + zp, qmax);
            uint32_t word;
            if (qmin == -128) {  // saturating pack gives the lower clamp
              asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(word) : "r"(o[3]), "r"(o[2]));
              asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %0;" : "+r"(word) : "r"(o[1]), "r"(o[0]));
            } else if (qmin == 0) {  // RELU / RELU6 with zp_out = 0
              asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(word) : "r"(o[3]), "r"(o[2]));
              asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %0;" : "+r"(word) : "r"(o[1]), "r"(o[0]));
            } else {
              word = 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) word |= (static_cast<uint32_t>(max(o[q], qmin)) & 0xFFu) << (8 * q);
            }
            if (c == 0 || live1) dst[r * rstride + c * (C / 4)] = word;
          }
        }
      });
    }
    return;
  } else if constexpr (DT == FCM_S8 && K >= 5) {
    // int8 5x5 / 7x7: weights stay packed (one word = 4 channels per tap, K^2 registers) and are
    // widened at use; each output row re-reads its K x K input words from shared memory. Exact
    // int32 accumulation (register pressure, not speed: these layers are rare)
    const int cw_valid = min(32, (C - c0) / 4);
    const int gs = cw_valid > 16 ? 32 : (cw_valid > 8 ? 16 : 8);
    const int npix = 32 / gs, grp = lane / gs, wd = lane - grp * gs;
    const int cl = c0 + wd * 4;
    const bool cval = wd < cw_valid;
    uint32_t Wp[K][K];
    {
      const uint32_t* g = reinterpret_cast<const uint32_t*>(wdw);
#pragma unroll
      for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j) Wp[i][j] = cval ? __ldg(g + (i * K + j) * (C / 4) + cl / 4) : 0u;
    }
    EpiC ec[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) ec[v] = load_epi<DT>(ep, cl + v, cval);
    wait_x();
    for (int cb = warp * npix; cb < tw; cb += 4 * npix) {
      const int col = cb + grp;
      const int x = x0 + col;
      const bool live = col < tw && x < Wo && cval;
      const uint32_t src = smem_u32(xs) + (((live ? col : cb) * S) * pwd + wd) * 4;
      for (int yy = 0; yy < nrows; ++yy) {
        int32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const uint32_t rp = src + min(yy * S + i, th_in - 1) * (tw_in * pb);
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const uint32_t xw = lds32(rp + j * pb);
#pragma unroll
            for (int v = 0; v < 4; ++v)
              acc[v] += (static_cast<int32_t>(xw << (24 - 8 * v)) >> 24) *
                        (static_cast<int32_t>(Wp[i][j] << (24 - 8 * v)) >> 24);
          }
        }
        if (live) {
          const size_t pix = (static_cast<size_t>(n) * Ho + (y0 + yy)) * Wo + x;
          yw[(pix * C + cl) / 4] = epi_pack<DT>(acc, ec, ep);
        }
      }
    }
  } else {
    // lane groups as in the pair core: a channel group with fewer valid words than lanes (e.g.
    // int8 C = 32 -> 8 words) packs 2 or 4 output columns into one warp instead of idling lanes
    const int cw_valid = min(32, (C - c0 + V - 1) / V);
    const int gs = cw_valid > 16 ? 32 : (cw_valid > 8 ? 16 : 8);
    const int npix = 32 / gs, grp = lane / gs, wd = lane - grp * gs;
    const int cl = c0 + wd * V;
    DwW<DT, K> W;
    load_dw_weights<DT, K>(W, wdw, C, cl);
    EpiC ec[V];
#pragma unroll
    for (int v = 0; v < V; ++v) ec[v] = load_epi<DT>(ep, cl + v, cl + v < C);
    wait_x();
    for (int cb = warp * npix; cb < tw; cb += 4 * npix) {
      const int col = cb + grp;
      const int x = x0 + col;
      const bool live = col < tw && x < Wo;
      const uint32_t src = smem_u32(xs) + (((live ? col : cb) * S) * pwd + wd) * 4;
      dw_segment<DT, K, S>(src, pb, tw_in * pb, 0, nrows, th_in - 1, W,
                           [&](int yy, const typename Tr<DT>::acc_t(&acc)[V]) {
                             if (live && cl < C) {
                               const size_t pix = (static_cast<size_t>(n) * Ho + (y0 + yy)) * Wo + x;
                               yw[(pix * C + cl) / V] = epi_pack<DT>(acc, ec, ep);
                             }
                           });
    }
  }
}

// NCHW: plane-per-(n,c) direct convolution through the read-only cache (layout accepted for
// completeness; the fused paths are NHWC).
template <int DT>
__global__ void dw_nchw_kernel(const typename Tr<DT>::T* __restrict__ x, const typename Tr<DT>::T* __restrict__ wdw,
                               Epi ep, typename Tr<DT>::T* __restrict__ y, int C, int H, int W, int Ho, int Wo, int k,
                               int s, int pt, int pl, long long total) {
  pdl_launch();
  pdl_wait();
  using TT = typename Tr<DT>::T;
  using A = typename Tr<DT>::acc_t;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int xo = idx % Wo;
    long long r = idx / Wo;
    const int yo = r % Ho;
    r /= Ho;
    const int c = r % C;
    const long long plane = r;  // n*C + c
    A acc = 0;
    for (int i = 0; i < k; ++i) {
      const int yi = yo * s - pt + i;
      if (yi < 0 || yi >= H) continue;
      for (int j = 0; j < k; ++j) {
        const int xi = xo * s - pl + j;
        if (xi < 0 || xi >= W) continue;
        TT xv = x[(plane * H + yi) * W + xi];
        TT wv = wdw[(i * k + j) * C + c];
        if constexpr (DT == FCM_S8) acc += static_cast<int32_t>(xv) * static_cast<int32_t>(wv);
        else if constexpr (DT == FCM_F32) acc = fmaf(xv, wv, acc);
        else if constexpr (DT == FCM_BF16) acc = fmaf(__bfloat162float(xv), __bfloat162float(wv), acc);
        else acc = fmaf(__half2float(xv), __half2float(wv), acc);
      }
    }
    EpiC e = load_epi<DT>(ep, c, true);
    if constexpr (DT == FCM_S8) y[idx] = static_cast<int8_t>(requant_i8(acc, e, ep.zp_out, ep.qmin, ep.qmax));
    else if constexpr (DT == FCM_F32) y[idx] = epi_f(acc, e.sc, e.bi, ep.act);
    else if constexpr (DT == FCM_BF16) y[idx] = __float2bfloat16_rn(epi_f(acc, e.sc, e.bi, ep.act));
    else y[idx] = __float2half_rn(epi_f(acc, e.sc, e.bi, ep.act));
  }
}

// Offline PW packing: canonical [C_in][C_out] -> K-major [C_out][C_in].
template <typename TT>
__global__ void pack_pw_kernel(const TT* __restrict__ w, TT* __restrict__ p, int cin, int cout) {
  // no early trigger: weights are what a following libfcm kernel may stage before its own PDL wait
  pdl_wait();
  __shared__ TT tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx over cout, by over cin
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int ci = by + i, co = bx + threadIdx.x;
    if (ci < cin && co < cout) tile[i][threadIdx.x] = w[(size_t)ci * cout + co];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int co = bx + i, ci = by + threadIdx.x;
    if (ci < cin && co < cout) p[(size_t)co * cin + ci] = tile[threadIdx.x][i];
  }
}

// ------------------------------------------------------------------------------- launchers
static bool dw_tc_i8_enabled() {  // FCM_DW_I8_TC=0: the CUDA-core int8 DW (development comparison)
  static const bool on = [] { const char* e = getenv("FCM_DW_I8_TC"); return !e || atoi(e) != 0; }();
  return on;
}

template <int DT, int K, int S>
static int launch_dw_t(const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  // int8, stride 1, k in {3, 5}, 16-byte pixel pitch, maps that fill its 16 x 8 output tiles: the
  // tensor-core DW (tc.cu dw_tc_i8_kernel). Measured on B200 (EfficientNet-B0 / MobileNetV1 int8):
  // 1.2-1.4x faster than this kernel on 112^2..14^2 maps, slower on 7^2 maps (38 % of the tile's
  // rows live) and for 5x5 with C > 512 (one CTA per SM, the 25-tap MMA chain per tile)
  if constexpr (DT == FCM_S8 && S == 1 && (K == 3 || K == 5))
    if (g.C % 16 == 0 && g.Wo >= 14 && g.Ho >= 14 && (K == 3 || g.C <= 512) && dw_tc_i8_enabled())
      return launch_dw_tc_i8(x, wdw, ep, y, g, st);
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  const int th = g.th, tw = g.tw;
  const int th_in = (th - 1) * S + K, tw_in = (tw - 1) * S + K;
  const int cbytes = g.C * ES;
  const bool tma = cbytes % 16 == 0;
  if (tma && (th_in > 256 || tw_in > 256)) return set_error(FCM_E_INFEASIBLE, "dw tile halo exceeds the TMA box limit (256)");
  CUtensorMap tm;
  // channel box: one 128-byte group, or the whole pixel when C is narrower -- no out-of-bounds
  // fill traffic and 4x less shared memory for e.g. int8 C = 32. Without TMA (pitch not a
  // multiple of 16 B) the narrow pixel is staged at its 16-byte-rounded width.
  const int pb = cbytes < 128 ? (cbytes + 15) / 16 * 16 : 128;
  if (tma) {
    const uint64_t dims[4] = {(uint64_t)g.C, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N};
    const uint64_t strides[3] = {(uint64_t)g.C * ES, (uint64_t)g.W * g.C * ES, (uint64_t)g.H * g.W * g.C * ES};
    const uint32_t box[4] = {(uint32_t)(pb / ES), (uint32_t)tw_in, (uint32_t)th_in, 1};
    if (!encode_tmap(&tm, tmap_dtype(DT), 4, x, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
      return set_error(FCM_E_CUDA, "cuTensorMapEncodeTiled failed for the DW input");
  } else {
    memset(&tm, 0, sizeof(tm));
  }
  const int tiles_x = (g.Wo + tw - 1) / tw, tiles_y = (g.Ho + th - 1) / th;
  // + 2 columns of slack: the int8 column-pair core reads S extra input words past the last
  // column of an odd-width tile (its second output column is dead, never stored)
  const size_t smem = (size_t)th_in * tw_in * pb + 256;
  if (smem > (size_t)device_props().smem_optin) return set_error(FCM_E_INFEASIBLE, "dw tile exceeds shared memory");
  auto kern = tma ? dw_nhwc_kernel<DT, K, S, true> : dw_nhwc_kernel<DT, K, S, false>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(tiles_x * tiles_y * g.N, (g.C + KC - 1) / KC);
  using TT = typename Tr<DT>::T;
  launch_k(kern, dim3(grid), dim3(128), smem, st, tm, static_cast<const TT*>(wdw), ep, static_cast<TT*>(y), g.C, g.Ho, g.Wo, g.pt, g.pl,
           th, tw, tiles_x, tiles_y, pb, static_cast<const uint8_t*>(x), g.H, g.W, cbytes % 8 == 0 ? 8 : 4);
  return check_launch("dw_nhwc_kernel");
}

template <int DT>
static int launch_dw_dt(const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  if (g.k == 3 && g.s == 1) return launch_dw_t<DT, 3, 1>(x, wdw, ep, y, g, st);
  if (g.k == 3 && g.s == 2) return launch_dw_t<DT, 3, 2>(x, wdw, ep, y, g, st);
  if (g.k == 5 && g.s == 1) return launch_dw_t<DT, 5, 1>(x, wdw, ep, y, g, st);
  if (g.k == 5 && g.s == 2) return launch_dw_t<DT, 5, 2>(x, wdw, ep, y, g, st);
  if (g.k == 7 && g.s == 1) return launch_dw_t<DT, 7, 1>(x, wdw, ep, y, g, st);
  if (g.k == 7 && g.s == 2) return launch_dw_t<DT, 7, 2>(x, wdw, ep, y, g, st);
  return set_error(FCM_E_UNSUPPORTED, "dw: only k in {3,5,7} and stride in {1,2} are built");
}

int launch_dw(int dt, const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  switch (dt) {
    case FCM_F32: return launch_dw_dt<FCM_F32>(x, wdw, ep, y, g, st);
    case FCM_BF16: return launch_dw_dt<FCM_BF16>(x, wdw, ep, y, g, st);
    case FCM_F16: return launch_dw_dt<FCM_F16>(x, wdw, ep, y, g, st);
    case FCM_S8: return launch_dw_dt<FCM_S8>(x, wdw, ep, y, g, st);
  }
  return set_error(FCM_E_INVAL, "bad dtype");
}

template <int DT>
static int launch_dw_nchw_t(const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  using TT = typename Tr<DT>::T;
  const long long total = (long long)g.N * g.C * g.Ho * g.Wo;
  const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)device_props().sms * 16);
  launch_k(dw_nchw_kernel<DT>, dim3(blocks), dim3(256), 0, st, static_cast<const TT*>(x), static_cast<const TT*>(wdw), ep,
                                             static_cast<TT*>(y), g.C, g.H, g.W, g.Ho, g.Wo, g.k, g.s, g.pt, g.pl,
                                             total);
  return check_launch("dw_nchw_kernel");
}

int launch_dw_nchw(int dt, const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  switch (dt) {
    case FCM_F32: return launch_dw_nchw_t<FCM_F32>(x, wdw, ep, y, g, st);
    case FCM_BF16: return launch_dw_nchw_t<FCM_BF16>(x, wdw, ep, y, g, st);
    case FCM_F16: return launch_dw_nchw_t<FCM_F16>(x, wdw, ep, y, g, st);
    case FCM_S8: return launch_dw_nchw_t<FCM_S8>(x, wdw, ep, y, g, st);
  }
  return set_error(FCM_E_INVAL, "bad dtype");
}

int launch_pack_pw(int dt, int cin, int cout, const void* w, void* packed, cudaStream_t st) {
  dim3 grid((cout + 31) / 32, (cin + 31) / 32), block(32, 8);
  switch (elem_size(dt)) {
    case 4: launch_k(pack_pw_kernel<uint32_t>, dim3(grid), dim3(block), 0, st, (const uint32_t*)w, (uint32_t*)packed, cin, cout); break;
    case 2: launch_k(pack_pw_kernel<uint16_t>, dim3(grid), dim3(block), 0, st, (const uint16_t*)w, (uint16_t*)packed, cin, cout); break;
    default: launch_k(pack_pw_kernel<uint8_t>, dim3(grid), dim3(block), 0, st, (const uint8_t*)w, (uint8_t*)packed, cin, cout); break;
  }
  return check_launch("pack_pw_kernel");
}

}  // namespace fcm
