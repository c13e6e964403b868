// Tensor-core (tcgen05 / TMEM / TMA) kernels: LBL PW, FCM DWPW, FCM PWDW_R.
//
// All three are persistent (grid <= #SMs), warp-specialised CTAs in the shape of Listing 1
// re-cast for sm_100a:
//   Listing-1 part 1 commBuffer  -> a K-major SWIZZLE_128B smem tile that is directly the
//                                   tcgen05 A operand (DWPW) / a padded smem T tile (PWDW_R)
//   part 2 weight prefetch       -> a TMA producer warp (mbarrier ring, `stages` deep)
//   part 3 conv1 -> commBuffer   -> DW warps (DWPW) / MMA + TMEM epilogue warps (PWDW_R)
//   "Synchronize"                -> mbarrier phases (no __syncthreads in the steady state)
//   part 4 conv2 -> OFMs         -> MMA warp + epilogue warps (DWPW) / DW warps (PWDW_R)
// Accumulators live in TMEM, double-buffered so the epilogue of tile i overlaps tile i+1.
// One 32-bit word of channels per lane; a K chunk is one 128-byte row (64 bf16 / 128 int8).
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "host.h"
#include "tiles.h"

namespace fcm {

template <int DT> struct TcKind;
template <> struct TcKind<FCM_BF16> { static constexpr MmaKind kind = MmaKind::F16; static constexpr uint32_t cf = 1, ab = 1; };
template <> struct TcKind<FCM_F16> { static constexpr MmaKind kind = MmaKind::F16; static constexpr uint32_t cf = 1, ab = 0; };
template <> struct TcKind<FCM_S8> { static constexpr MmaKind kind = MmaKind::I8; static constexpr uint32_t cf = 2, ab = 1; };
// fp32 PW: kind::tf32 with the 3xTF32 split (x = x_hi + x_lo, w = w_hi + w_lo; x_hi.w_hi + x_hi.w_lo
// + x_lo.w_hi, the dropped x_lo.w_lo term is ~2^-22 relative: reading R10b's 1e-5 is met)
template <> struct TcKind<FCM_F32> { static constexpr MmaKind kind = MmaKind::TF32; static constexpr uint32_t cf = 1, ab = 2; };
// K elements per tcgen05.mma instruction (32 bytes of each operand row)

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Pack two fp32 into bf16x2 / f16x2 (RNE), optionally with the free ReLU of cvt.relu.
template <int DT, bool kRelu>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t d;
  if constexpr (DT == FCM_BF16) {
    if constexpr (kRelu) asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    else asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  } else {
    if constexpr (kRelu) asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    else asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  }
  return d;
}

// A packed bf16x2 / f16x2 word -> its two fp32 values (lo, hi).
template <int DT>
__device__ __forceinline__ float2 word2f(uint32_t w) {
  if constexpr (DT == FCM_BF16) return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  else return __half22float2(*reinterpret_cast<const __half2*>(&w));
}

// Epilogue of 16 accumulator columns [n_base, n_base+16) of one row -> packed storage words.
// Constants come from smem as 128-bit broadcast loads (n_base is a multiple of 16).
// RES (bf16 / f16): ra / rb = the 8 packed words of the residual (shortcut) for these 16 columns,
// added after the activation. The activation variants are dispatched once per
// call, so a kernel only fetches the code it runs (the DWPW epilogue shares the SM's instruction
// cache with the DW stage's hot loop; measured: a per-element activation switch with erf inlined 16x
// cost the DW warps 2x in instruction-fetch stalls).
// SMOOTH = false: the kernel is compiled for NONE / RELU / RELU6 only (no SiLU / GELU code)
template <int DT, bool RES = false, bool SMOOTH = true>
__device__ __forceinline__ void epi16(const uint32_t* r, const EpiS& cs, const Epi& e, int n_base,
                                      uint32_t (&out)[8], uint4 ra = uint4{}, uint4 rb = uint4{}) {
  if constexpr (DT == FCM_S8) {
    if (cs.fast) {  // CTA-uniform: all shifts >= 33 -> one mad.hi + shift per value (identical results)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint4 bq = lds128(cs.base + 4 * (n_base + 4 * w));
        const uint4 mq = lds128(cs.base + 4 * (cs.ncap + n_base + 4 * w));
        const uint4 sh = lds128(cs.base + 4 * (2 * cs.ncap + n_base + 4 * w));
        const int32_t b4[4] = {(int32_t)bq.x, (int32_t)bq.y, (int32_t)bq.z, (int32_t)bq.w};
        const int32_t m4[4] = {(int32_t)mq.x, (int32_t)mq.y, (int32_t)mq.z, (int32_t)mq.w};
        const int32_t s4[4] = {(int32_t)sh.x, (int32_t)sh.y, (int32_t)sh.z, (int32_t)sh.w};
        uint32_t word = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int32_t h;
          asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(h) : "r"(static_cast<int32_t>(r[4 * w + i]) + b4[i]), "r"(m4[i]),
              "r"(1 << (s4[i] - 33)));
          word |= (static_cast<uint32_t>(min(max((h >> (s4[i] - 32)) + e.zp_out, e.qmin), e.qmax)) & 0xFFu) << (8 * i);
        }
        out[w] = word;
      }
      return;
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint4 bq = lds128(cs.base + 4 * (n_base + 4 * w));
      const uint4 mq = lds128(cs.base + 4 * (cs.ncap + n_base + 4 * w));
      const uint4 sh = lds128(cs.base + 4 * (2 * cs.ncap + n_base + 4 * w));
      const uint32_t b4[4] = {bq.x, bq.y, bq.z, bq.w}, m4[4] = {mq.x, mq.y, mq.z, mq.w}, s4[4] = {sh.x, sh.y, sh.z, sh.w};
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        EpiC c{0.f, 0.f, (int32_t)b4[i], (int32_t)m4[i], (int32_t)s4[i]};
        const int32_t q = requant_i8(static_cast<int32_t>(r[4 * w + i]), c, e.zp_out, e.qmin, e.qmax);
        word |= (static_cast<uint32_t>(q) & 0xFFu) << (8 * i);
      }
      out[w] = word;
    }
  } else {
    float sc[16], bi[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 a = lds128(cs.base + 4 * (n_base + 4 * q));
      const uint4 b = lds128(cs.base + 4 * (cs.ncap + n_base + 4 * q));
      sc[4 * q] = __uint_as_float(a.x); sc[4 * q + 1] = __uint_as_float(a.y);
      sc[4 * q + 2] = __uint_as_float(a.z); sc[4 * q + 3] = __uint_as_float(a.w);
      bi[4 * q] = __uint_as_float(b.x); bi[4 * q + 1] = __uint_as_float(b.y);
      bi[4 * q + 2] = __uint_as_float(b.z); bi[4 * q + 3] = __uint_as_float(b.w);
    }
    if (SMOOTH && e.act > FCM_ACT_RELU6) {
      // SiLU / GELU (+ residual): the activation dispatched once per call (one variant's code is
      // fetched; a rolled loop would move r / out to local memory)
      with_act(e.act, [&](auto actc) {
        constexpr int ACT = decltype(actc)::value;
        const uint32_t rw[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          float v0 = act_t<ACT>(fmaf(__uint_as_float(r[2 * w]), sc[2 * w], bi[2 * w]));
          float v1 = act_t<ACT>(fmaf(__uint_as_float(r[2 * w + 1]), sc[2 * w + 1], bi[2 * w + 1]));
          if constexpr (RES) {
            const float2 s = word2f<DT>(rw[w]);
            v0 += s.x;
            v1 += s.y;
          }
          out[w] = pack2<DT, false>(v0, v1);
        }
      });
      return;
    }
    const float hi_c = act_hi(e.act);
    if constexpr (RES) {
      const uint32_t rw[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
      if (e.act == FCM_ACT_NONE) {
        // (the inverted-residual projection) packed: v = fma(acc, scale, bias) then + shortcut, two
        // FFMA2 per column pair -- the same two roundings as the scalar form below
        const uint64_t one2 = 0x3F8000003F800000ull;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const float2 sf = word2f<DT>(rw[w]);
          const uint64_t v = f2_fma(f2_fma(f2_pack(__uint_as_float(r[2 * w]), __uint_as_float(r[2 * w + 1])),
                                           f2_pack(sc[2 * w], sc[2 * w + 1]), f2_pack(bi[2 * w], bi[2 * w + 1])),
                                    one2, f2_pack(sf.x, sf.y));
          float v0, v1;
          f2_unpack(v, v0, v1);
          out[w] = pack2<DT, false>(v0, v1);
        }
        return;
      }
      const float lo_c = act_lo(e.act);
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const float2 s = word2f<DT>(rw[w]);
        out[w] = pack2<DT, false>(
            fminf(fmaxf(fmaf(__uint_as_float(r[2 * w]), sc[2 * w], bi[2 * w]), lo_c), hi_c) + s.x,
            fminf(fmaxf(fmaf(__uint_as_float(r[2 * w + 1]), sc[2 * w + 1], bi[2 * w + 1]), lo_c), hi_c) + s.y);
      }
    } else {
      // packed: one FFMA2 per column pair, cvt.rn(.relu) pack, min for RELU6 (bit-identical to the
      // scalar fma / min / round: 6 is exact in bf16 / f16, rounding is monotonic)
      auto pk = [&](auto actc) {
        constexpr int ACT = decltype(actc)::value;
        const uint32_t hc = ACT == FCM_ACT_RELU6 ? bound2<DT>(hi_c) : 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w)
          out[w] = epi_act2<DT, ACT>(__uint_as_float(r[2 * w]), __uint_as_float(r[2 * w + 1]),
                                     f2_pack(sc[2 * w], sc[2 * w + 1]), f2_pack(bi[2 * w], bi[2 * w + 1]), hc);
      };
      if (e.act == FCM_ACT_NONE) pk(std::integral_constant<int, FCM_ACT_NONE>());
      else if (e.act == FCM_ACT_RELU) pk(std::integral_constant<int, FCM_ACT_RELU>());
      else pk(std::integral_constant<int, FCM_ACT_RELU6>());
    }
  }
}

// One 16-column epilogue step of a float (bf16 / f16) output with the runtime activation / residual
// choice; r points at 16 consecutive accumulator words.
template <int DT, bool SMOOTH = true>
__device__ __forceinline__ void epi16_any(const uint32_t* r, const EpiS& cs, const Epi& e, int n_base,
                                          uint32_t (&out)[8], bool res, uint4 ra, uint4 rb) {
  if constexpr (DT == FCM_S8) {
    epi16<DT>(r, cs, e, n_base, out);
  } else {
    if (res) epi16<DT, true, SMOOTH>(r, cs, e, n_base, out, ra, rb);
    else epi16<DT, false, SMOOTH>(r, cs, e, n_base, out);
  }
}

// Residual (shortcut) words of 32 consecutive bf16 / f16 output columns, loaded one 32-column
// chunk ahead of their use so the epilogue never waits a global round trip.
struct Res32 {
  uint4 v[4];
};
__device__ __forceinline__ uint4 ldg_nc128(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// columns [col, col + 32) of the row at element offset `rowoff`; 8-column pieces at or past
// `lim` (the row's valid width) and rows with !ok read as 0
__device__ __forceinline__ void res32_load(const void* r, size_t rowoff, int col, int lim, bool ok, Res32& o) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    o.v[p] = make_uint4(0u, 0u, 0u, 0u);
    if (ok && col + 8 * p < lim) o.v[p] = ldg_nc128(static_cast<const uint16_t*>(r) + rowoff + col + 8 * p);
  }
}

// Byte offset of 16-byte vector `vi` (0..7) of row m in a SWIZZLE_128B tile (1024-B aligned).
__device__ __forceinline__ uint32_t sw128_vec(int m, int vi) {
  return (m >> 3) * 1024 + (m & 7) * 128 + ((vi ^ (m & 7)) << 4);
}

// Epilogue of one TMEM accumulator tile (128 lanes x BN columns) by NEPI warps (4 or 8; warp w
// reads lane quadrant w%4 and every (NEPI/4)-th 16-column subchunk). Each 128-byte chunk of
// output columns is converted into a SWIZZLE_128B staging tile (two buffers, alternating) and
// written by ONE TMA store issued by thread 0: full-line, coalesced HBM writes; rows / columns
// outside the tensor are clipped by the TMA unit.
template <int DT, int NEPI, class StoreFn>
__device__ __forceinline__ void epilogue_tile(uint32_t tacc, int BN, int n0, int N, const EpiS& cs, const Epi& e,
                                              uint8_t* stage, int& sbuf, StoreFn&& store) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int CPC = 128 / ES;  // output columns per 128-byte chunk
  constexpr int SUB = CPC / 16;  // 16-column subchunks per chunk
  constexpr int G = NEPI / 4;    // warps sharing a lane quadrant
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, h = warp >> 2;
  const int m = q * 32 + lane;
  const int valid = min(BN, N - n0);
  const int nch = (valid + CPC - 1) / CPC;
  for (int cc = 0; cc < nch; ++cc, ++sbuf) {
    uint8_t* buf = stage + (sbuf & 1) * 16384;
    if (threadIdx.x == 0) bulk_wait_read<1>();
    named_bar_sync(1, NEPI * 32);
    for (int j = h; j < SUB; j += G) {
      const int c0 = cc * CPC + j * 16;
      if (c0 >= BN) break;
      uint32_t r[16];
      tmem_ld16(tacc + ((uint32_t)(q * 32) << 16) + c0, r);
      tmem_ld_wait();
      uint32_t o[8];
      epi16_any<DT>(r, cs, e, n0 + c0, o, false, uint4{}, uint4{});
#pragma unroll
      for (int v = 0; v < ES; ++v)
        sts128(smem_u32(buf) + sw128_vec(m, j * ES + v), o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
    }
    fence_proxy_async_smem();
    named_bar_sync(1, NEPI * 32);
    if (threadIdx.x == 0) {
      store(buf, n0 + cc * CPC);
      bulk_commit();
    }
  }
}

// Warp-private epilogue (PW): warp w owns TMEM lane quadrant q = w % 4 (32 output rows) and the
// 128-byte column chunks hs, hs + G, ... ; it converts its 32 x CPC block into a private SW128
// staging buffer (4 KB) and its lane 0 issues the TMA store of a (CPC x 32-row) box -- no
// CTA-wide barriers in the epilogue.
// row0 / M: global output row of TMEM lane 0 and the row count (for the optional residual).
template <int DT, class StoreFn>
__device__ __forceinline__ void epilogue_tile_warp(uint32_t tacc, int BN, int n0, int N, const EpiS& cs, const Epi& e,
                                                   uint8_t* wstage, int& sbuf, int hs, int G, long row0, int M,
                                                   StoreFn&& store) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int CPC = 128 / ES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;
  const long grow = row0 + q * 32 + lane;
  const bool hasres = ES == 2 && e.residual != nullptr;
  const bool rrow = hasres && grow < M;
  const int valid = min(BN, N - n0);
  const int nch = (valid + CPC - 1) / CPC;
  for (int cc = hs; cc < nch; cc += G, ++sbuf) {
    uint8_t* buf = wstage;  // one 4 KB buffer per warp: wait until its previous store has read it
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
#pragma unroll 1
    for (int c32 = 0; c32 < CPC; c32 += 32) {
      const int c0 = cc * CPC + c32;
      if (c0 >= BN) break;
      if constexpr (ES == 4) {
        // fp32 output (3xTF32 PW): v = act(acc * scale + bias) (+ residual), 32 columns = one
        // 128-byte chunk
        uint32_t r[32];
        tmem_ld32(tacc + ((uint32_t)(q * 32) << 16) + c0, r);
        const float* rp = e.residual ? static_cast<const float*>(e.residual) + (size_t)grow * N + n0 + c0 : nullptr;
        tmem_ld_wait();
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 sc = lds128(cs.base + 4 * (n0 + c0 + 4 * v));
          const uint4 bi = lds128(cs.base + 4 * (cs.ncap + n0 + c0 + 4 * v));
          float4 rs = make_float4(0.f, 0.f, 0.f, 0.f);
          if (rp && grow < M && n0 + c0 + 4 * v < N) {
            const uint4 w = ldg_nc128(rp + 4 * v);
            rs = make_float4(__uint_as_float(w.x), __uint_as_float(w.y), __uint_as_float(w.z), __uint_as_float(w.w));
          }
          const float* a = reinterpret_cast<const float*>(&r[4 * v]);
          sts128(smem_u32(buf) + sw128_vec(lane, v),
                 __float_as_uint(act_f(fmaf(a[0], __uint_as_float(sc.x), __uint_as_float(bi.x)), e.act) + rs.x),
                 __float_as_uint(act_f(fmaf(a[1], __uint_as_float(sc.y), __uint_as_float(bi.y)), e.act) + rs.y),
                 __float_as_uint(act_f(fmaf(a[2], __uint_as_float(sc.z), __uint_as_float(bi.z)), e.act) + rs.z),
                 __float_as_uint(act_f(fmaf(a[3], __uint_as_float(sc.w), __uint_as_float(bi.w)), e.act) + rs.w));
        }
        continue;
      }
      if (ES == 2 && (hasres || e.act > FCM_ACT_RELU6)) {
        // SiLU / GELU / residual: 16 columns per TMEM load, the residual words
        // issued before it (register budget 18 warps x 96; the 16 epilogue warps hide the latency)
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          uint4 rw[2] = {make_uint4(0u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u)};
          const int col = n0 + c0 + 16 * hh;
          if (hasres) {
            const uint16_t* rp = static_cast<const uint16_t*>(e.residual) + (size_t)grow * N + col;
            if (rrow && col < N) rw[0] = ldg_nc128(rp);
            if (rrow && col + 8 < N) rw[1] = ldg_nc128(rp + 8);
          }
          uint32_t r[16];
          tmem_ld16(tacc + ((uint32_t)(q * 32) << 16) + c0 + 16 * hh, r);
          tmem_ld_wait();
          uint32_t o[8];
          epi16_any<DT>(r, cs, e, col, o, hasres, rw[0], rw[1]);
          const int vi0 = (c32 + 16 * hh) * ES / 16;
#pragma unroll
          for (int v = 0; v < ES; ++v)
            sts128(smem_u32(buf) + sw128_vec(lane, vi0 + v), o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
        }
        continue;
      }
      uint32_t r[32];
      tmem_ld32(tacc + ((uint32_t)(q * 32) << 16) + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t o[8];
        epi16<DT>(&r[16 * hh], cs, e, n0 + c0 + 16 * hh, o);
        const int vi0 = (c32 + 16 * hh) * ES / 16;
#pragma unroll
        for (int v = 0; v < ES; ++v)
          sts128(smem_u32(buf) + sw128_vec(lane, vi0 + v), o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      store(buf, n0 + cc * CPC, q * 32);
      bulk_commit();
    }
  }
}

// =====================================================================================
// LBL PW: Y[M,N] = eps(X[M,K] . Wp[N,K]^T). Warps 0-15 epilogue, 16 TMA producer, 17 MMA.
// The 16 epilogue warps form `ng` groups that take alternate tiles (tile l -> group l % ng), each
// with its own pair of TMEM accumulators, so the epilogues of ng tiles run concurrently: a tile
// needs only 4 x nch warps (nch = 128-byte column chunks), and a single group would leave the
// rest idle while its TMEM round trips serialise.
// =====================================================================================
template <int DT>
__global__ void __launch_bounds__(DT == FCM_F32 ? 640 : 576, 1)
    pw_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                 const __grid_constant__ CUtensorMap tmy, Epi ep, int M, int N, int K, int BN, int nbn, FDiv fnbn,
                 int stages, int ng, int nbuf, uint32_t tmem_cols, int ncap, int resB, unsigned long long* trace,
                 int dbg) {
  pdl_launch();
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  constexpr MmaKind KIND = TcKind<DT>::kind;
  constexpr int KSTEP = 32 / Tr<DT>::ES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  // kSplit (fp32, 3xTF32): every stage also holds x_lo and w_lo; two converter warps (18, 19) split
  // the landed tiles in place (hi = the value with its low 13 mantissa bits cleared, exact in tf32)
  constexpr bool kSplit = DT == FCM_F32;
  constexpr int AST = kSplit ? 32768 : 16384;    // A stage: x (-> x_hi) [+ x_lo]
  const int BST = BN * 128 * (kSplit ? 2 : 1);   // B stage: w (-> w_hi) [+ w_lo]
  uint8_t* stage = smem;                         // 16 warps x 4 KB output staging
  uint8_t* abuf = smem + 65536;
  uint8_t* bbuf = abuf + stages * AST;           // resB: all nk chunks of this CTA's B slice, else a ring
  const int nk = (K + KC - 1) / KC;
  uint8_t* cst = bbuf + (resB ? nk * BN * 128 : stages * BST);
  uint64_t* full = reinterpret_cast<uint64_t*>(cst + consts_bytes<DT>(ncap));
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 8;
  uint64_t* bfull = tempty + 8;
  uint64_t* cfull = bfull + 1;                   // kSplit: stage converted
  uint32_t* tslot = reinterpret_cast<uint32_t*>(cfull + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const EpiS cs = stage_consts<DT>(ep, N, ncap, cst);
  const int spg = 4 / ng;  // warps per TMEM lane quadrant in one group
  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmb);
    tma_prefetch_desc(&tmy);
    for (int s = 0; s < stages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int a = 0; a < nbuf * ng; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 4 * spg); }
    mbar_init(bfull, 1);
    for (int s = 0; s < stages && kSplit; ++s) mbar_init(cfull + s, 2);
    fence_barrier_init();
  }
  if (warp == 17) tmem_alloc_rt(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // previous kernel's outputs (our inputs) complete; our outputs free to overwrite
  const uint32_t tbase = *tslot;
  const int nbm = (M + 127) / 128;
  const int total = nbm * nbn;
  auto stamp = [&](int local, int ev) {
    if (trace && blockIdx.x == 0 && local < 64) trace[local * 16 + ev] = clock64();
  };
  // tile l of this CTA -> accumulator (group l % ng, its nbuf buffers in turn) and its phase
  auto acc_of = [&](int l, int& acc, uint32_t& ph) {
    const int g = l % ng, j = l / ng;
    acc = nbuf * g + (nbuf == 2 ? (j & 1) : 0);
    ph = (nbuf == 2 ? (j >> 1) : j) & 1;
  };

  if (warp == 16) {
    if (lane == 0) {
      Ring rs(stages);
      int lt = 0;
      if (resB) {
        // the grid is a multiple of nbn, so this CTA's C_out slice never changes: load it once
        // (a per-tile reload has every SM re-reading the same few KB of L2 each tile)
        mbar_arrive_expect_tx(bfull, nk * BN * 128);
        const int nb0 = blockIdx.x - fdiv(blockIdx.x, fnbn) * nbn;
        for (int kc = 0; kc < nk; ++kc) tma_load_2d(bbuf + kc * BN * 128, &tmb, bfull, kc * KC, nb0 * BN);
      }
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
        const int tm = fdiv(t, fnbn);
        const int m0 = tm * 128, n0 = (t - tm * nbn) * BN;
        for (int kc = 0; kc < nk; ++kc, rs.next()) {
          mbar_wait(empty + rs.i, rs.ph ^ 1);
          if (kc == 0) stamp(lt, 8);
          mbar_arrive_expect_tx(full + rs.i, 16384 + (resB ? 0 : BN * 128));
          tma_load_2d(abuf + rs.i * AST, &tma, full + rs.i, kc * KC, m0);
          if (!resB) tma_load_2d(bbuf + rs.i * BST, &tmb, full + rs.i, kc * KC, n0);
        }
      }
    }
  } else if (warp == 17) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, BN);
      Ring rs(stages);
      int local = 0;
      if (resB) mbar_wait(bfull, 0);
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        int acc;
        uint32_t ph;
        acc_of(local, acc, ph);
        mbar_wait(tempty + acc, ph ^ 1);
        stamp(local, 0);
        tc_fence_after();
        const uint32_t d = tbase + acc * BN;
        for (int kc = 0; kc < nk; ++kc, rs.next()) {
          mbar_wait(kSplit ? cfull + rs.i : full + rs.i, rs.ph);
          if (kc == 0) stamp(local, 1);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(abuf + rs.i * AST));
          const uint64_t bd = smem_desc_sw128(smem_u32(resB ? bbuf + kc * BN * 128 : bbuf + rs.i * BST));
          const int ksteps = min(4, (K - kc * KC + KSTEP - 1) / KSTEP);  // skip all-zero K steps
          if constexpr (kSplit) {
            const uint64_t adl = ad + (16384 >> 4), bdl = bd + ((BN * 128) >> 4);  // x_lo, w_lo
            for (int k = 0; k < ksteps; ++k) {
              mma_ss<KIND>(d, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
              mma_ss<KIND>(d, ad + 2 * k, bdl + 2 * k, idesc, 1);
              mma_ss<KIND>(d, adl + 2 * k, bd + 2 * k, idesc, 1);
            }
          } else {
            for (int k = 0; k < ksteps; ++k) mma_ss<KIND>(d, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
          }
          mma_commit(empty + rs.i);
        }
        mma_commit(tfull + acc);
        stamp(local, 2);
      }
    }
  } else if (warp >= 18) {
    // kSplit converters: x -> (x_hi in place, x_lo), w -> (w_hi in place, w_lo) per landed stage
    if constexpr (kSplit) {
      const int ct = threadIdx.x - 18 * 32;
      Ring rs(stages);
      for (int t = blockIdx.x; t < total; t += gridDim.x)
        for (int kc = 0; kc < nk; ++kc, rs.next()) {
          mbar_wait(full + rs.i, rs.ph);
          auto split = [&](uint32_t hi_base, uint32_t lo_base, int nvec) {
            for (int v = ct; v < nvec; v += 64) {
              const uint4 x = lds128(hi_base + 16 * v);
              const uint4 h = make_uint4(x.x & 0xFFFFE000u, x.y & 0xFFFFE000u, x.z & 0xFFFFE000u, x.w & 0xFFFFE000u);
              sts128(hi_base + 16 * v, h.x, h.y, h.z, h.w);
              sts128(lo_base + 16 * v, __float_as_uint(__uint_as_float(x.x) - __uint_as_float(h.x)),
                     __float_as_uint(__uint_as_float(x.y) - __uint_as_float(h.y)),
                     __float_as_uint(__uint_as_float(x.z) - __uint_as_float(h.z)),
                     __float_as_uint(__uint_as_float(x.w) - __uint_as_float(h.w)));
            }
          };
          const uint32_t a = smem_u32(abuf + rs.i * AST), b = smem_u32(bbuf + rs.i * BST);
          split(a, a + 16384, 1024);
          split(b, b + BN * 128, BN * 8);
          fence_proxy_async_smem();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive(cfull + rs.i);
        }
    }
  } else {
    // epilogue warp: lane quadrant q = warp % 4, group g, slot hs within the group
    const int h = warp >> 2, g = h / spg, hs = h - g * spg;
    int sbuf = 0;
    for (int local = g, t = blockIdx.x + g * gridDim.x; t < total; t += ng * gridDim.x, local += ng) {
      int acc;
      uint32_t ph;
      acc_of(local, acc, ph);
      const int tm = fdiv(t, fnbn);
      const int m0 = tm * 128, n0 = (t - tm * nbn) * BN;
      group_wait(tfull + acc, ph, hs == 0 && (warp & 3) == 0, 2 + g, 4 * spg * 32);
      if (threadIdx.x == 0) stamp(local, 3);
      tc_fence_after();
      if (!(dbg & 32))
        epilogue_tile_warp<DT>(tbase + acc * BN, BN, n0, N, cs, ep, stage + warp * 4096, sbuf, hs, spg, m0, M,
                               [&](const uint8_t* buf, int c, int r) {
                                 if (!(dbg & 16)) tma_store_2d(&tmy, buf, c, m0 + r);
                               });
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (threadIdx.x == 0) stamp(local, 5);
    }
    if (lane == 0) bulk_wait_all();
  }
  __syncthreads();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, tmem_cols);
  }
}

// =====================================================================================
// FCM DWPW. Warps 0-3 PW epilogue, 4..4+NDW-1 DW producers of the A operand (commBuffer),
// then one TMA warp and one MMA warp. One tile = nb x th x tw output pixels (MB <= 2 MMA row
// blocks of 128: M <= 256 for the bf16/f16 3x3 pair core, else <= 128) x one C_out slice of BN
// channels; the C_in (=K) dimension streams through in 128-byte chunks, so the intermediate
// "contains all channels" in time, not space. The PW epilogue stores straight from
// registers (a lane owns one output pixel: its BN channels are contiguous in NHWC).
// =====================================================================================
// DW warps per DWPW CTA
#ifndef FCM_DWPW_NDW
#define FCM_DWPW_NDW 8
#endif
// 1: a relay warp turns "X stage full + A slot free" into one named-barrier release of all DW
// warps per C_in chunk; 0: every DW warp waits on the two mbarriers itself (no lock-step)
#ifndef FCM_DWPW_RELAY
#define FCM_DWPW_RELAY 1
#endif
// output columns per DW item of the bf16/f16 3x3 core (a lane owns one channel word of NC adjacent
// columns): 4 gives each warp 8 independent accumulation chains per row (2 -> 4 was 2-3x faster on
// the 14 x 14 tiles, whose few items left one latency-bound warp per phase on the critical path)
#ifndef FCM_DWPW_NC
#define FCM_DWPW_NC 4
#endif
constexpr int kDwpwNC = FCM_DWPW_NC;
template <int DT, int K> constexpr int dwpw_ndw() { return FCM_DWPW_NDW; }
// relay waits: plain try_wait polling (FCM_RELAY_SLEEP=1: sleep back-off, development experiment)
#if defined(FCM_RELAY_SLEEP) && FCM_RELAY_SLEEP
#define RELAY_WAIT(b, p) mbar_wait_sleep<32>(b, p)
#else
#define RELAY_WAIT(b, p) mbar_wait(b, p)
#endif
constexpr int kDwpwNA = 2;  // default A-operand (commBuffer) ring depth
struct DwDivs {
  FDiv hp;              // column pairs per image
  FDiv nsg[3];          // ceil(th / SEG) for the SEG of each lane-group width
  int nsgi;             // the same counts, byte gi (<= 255)
  FDiv nsplit, tx, ty;  // tile decode
  FDiv thw, tw;         // epilogue: MMA row m -> (image, row, col) of the tile
  int seg_sel;          // SEG per lane-group width: byte g (g = 0, 1, 2 for 32, 16, 8 lanes per slot)
};
template <int DT, int K> constexpr bool dwpw_pair() { return (DT == FCM_BF16 || DT == FCM_F16) && K == 3; }
template <int DT, int K> constexpr int dwpw_wbytes(int nk) {
  return dwpw_pair<DT, K>() ? dw3h_bytes(nk * 32) : K * K * nk * 32 * 4;
}

// R6: the DW activation is RELU6 and the PW one NONE / RELU / RELU6 (one compiled DW epilogue
// variant, no SiLU / GELU code in the PW epilogue: measured 7 % faster DWPW on MobileNetV2 b2 than
// the runtime dispatch, whose variants share the instruction cache with the other warp roles);
// otherwise the activations are dispatched at run time
template <int DT, int K, int S, bool R6 = false>
__global__ void __launch_bounds__((4 + dwpw_ndw<DT, K>() + 4) * 32, 1)
    dwpw_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
                   void* __restrict__ tmy_base, const typename Tr<DT>::T* __restrict__ wdw, Epi ed,
                   Epi ep, int N, int Cin, int Ho, int Wo, int Cout, int pt, int pl, int nb, int th, int tw,
                   int tiles_x, int tiles_y, int nsplit, int BN, int XS, int BS, uint32_t tmem_cols, int ncap, int resB,
                   DwDivs dv, int na, int nacc, int MB, int albo, int dbg, unsigned long long* trace) {
  pdl_launch();
  constexpr int V = Tr<DT>::VEC;
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  constexpr MmaKind KIND = TcKind<DT>::kind;
  constexpr int KSTEP = 32 / Tr<DT>::ES;
  constexpr int kDwpwNDW = dwpw_ndw<DT, K>();
  constexpr int WARP_TX = 4 + kDwpwNDW, WARP_TB = 5 + kDwpwNDW, WARP_MMA = 6 + kDwpwNDW, WARP_RELAY = 7 + kDwpwNDW;
  // relay: one warp turns "X stage landed (TMA mbarrier) and A slot free (MMA commit mbarrier)"
  // into a named-barrier release of the DW warps (bar.sync ~ tens of cycles vs ~200 per
  // mbarrier try_wait round trip on the DW warps' critical path); barriers 2/3 alternate phases
  constexpr uint32_t kGoThreads = (kDwpwNDW + 1) * 32;
  const int th_in = (th - 1) * S + K, tw_in = (tw - 1) * S + K;
  const int xbytes = nb * th_in * tw_in * 128;
  const int xstride = (xbytes + 1023) & ~1023;
  const int nk = (Cin + KC - 1) / KC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr bool kPair = dwpw_pair<DT, K>();
  // A slot: pair core = no-swizzle K-major rows (MB x 128 rows, LBO = albo); else SW128, 128 rows
  // fp32 (3xTF32): the commBuffer holds T_hi and T_lo (the DW warps write both), the resident PW
  // weights W and W_lo (split in place once per CTA by the DW warps)
  constexpr bool kSplit = DT == FCM_F32;
  const int aslot = kPair ? ((8 * albo + 1023) & ~1023) : (kSplit ? 32768 : 16384);
  uint8_t* abuf = smem;                          // na x aslot A operand (commBuffer) ring
  uint8_t* xbuf = abuf + na * aslot;             // XS x X halo chunks (TMA -> DW)
  uint8_t* bbuf = xbuf + XS * xstride;           // BS x PW weight chunks (TMA -> MMA); resB: BS = nk, loaded once
  uint8_t* cst = bbuf + BS * BN * 128 * (kSplit ? 2 : 1);
  uint8_t* dcst = cst + consts_bytes<DT>(ncap);                 // DW epilogue constants [nk*KC]
  uint32_t* wsm = reinterpret_cast<uint32_t*>(dcst + consts_bytes<DT>(nk * KC));  // DW weights
  uint64_t* fullX = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(wsm) + dwpw_wbytes<DT, K>(nk));
  uint64_t* emptyX = fullX + XS;
  uint64_t* fullB = emptyX + XS;
  uint64_t* emptyB = fullB + BS;
  uint64_t* afull = emptyB + BS;
  uint64_t* aempty = afull + na;
  uint64_t* tfull = aempty + na;
  uint64_t* tempty = tfull + nacc;
  uint64_t* bconv = tempty + nacc;               // kSplit: resident weights split
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bconv + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const EpiS cs = stage_consts<DT>(ep, Cout, ncap, cst);
  const EpiS dcs = stage_consts<DT>(ed, Cin, nk * KC, dcst);
  // kPair: raw packed weight words [9][nk*32] + scale / bias pairs (stage_dw3_h)
  if constexpr (kPair) stage_dw3_h<DT>(wdw, ed, Cin, nk * 32, wsm);
  else stage_dw_weights<DT>(wdw, K, Cin, nk * 32, wsm);
  for (int i = threadIdx.x; i < na * aslot / 16; i += blockDim.x) sts128(smem_u32(abuf) + 16 * i, 0, 0, 0, 0);
  if (warp == WARP_TX && lane == 0) {
    tma_prefetch_desc(&tmx);
    tma_prefetch_desc(&tmb);
    for (int s = 0; s < XS; ++s) { mbar_init(fullX + s, 1); mbar_init(emptyX + s, kDwpwNDW); }
    for (int s = 0; s < BS; ++s) { mbar_init(fullB + s, 1); mbar_init(emptyB + s, 1); }
    for (int a = 0; a < na; ++a) { mbar_init(afull + a, kDwpwNDW); mbar_init(aempty + a, 1); }
    for (int a = 0; a < nacc; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 4); }
    mbar_init(bconv, kDwpwNDW);
    fence_barrier_init();
  }
  if (warp == WARP_MMA) tmem_alloc_rt(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // previous kernel's outputs (our inputs) complete; our outputs free to overwrite
  const uint32_t tbase = *tslot;
  const int spatial = ((N + nb - 1) / nb) * tiles_y * tiles_x;
  const int total = spatial * nsplit;
  // development tracing (FCM_TRACE): clock64 stamps of CTA 0's first 64 tiles
#ifdef FCM_TRACE_STAMPS
  __shared__ unsigned long long tr_sm[64 * 12];  // stamps land in smem (cheap), copied out at exit
  for (int i = threadIdx.x; i < 64 * 12; i += blockDim.x) tr_sm[i] = 0;
  __syncthreads();
#endif
  auto stamp = [&](int local, int ev) {
#if defined(FCM_TRACE_STAMPS) && !defined(FCM_TRACE_CHUNK)
    if (trace && blockIdx.x == 0 && local < 64) tr_sm[local * 12 + ev] = clock64();
#endif
  };
  // chunk-level variant (FCM_TRACE_CHUNK, tools/trace_chunks.py): one row per C_in-chunk phase
  auto cstamp = [&](int idx, int ev) {
#if defined(FCM_TRACE_STAMPS) && defined(FCM_TRACE_CHUNK)
    if (trace && blockIdx.x == 0 && idx < 64) tr_sm[idx * 12 + ev] = clock64();
#endif
  };
  // tile t -> (C_out split, image group, tile row, tile col) with host-computed magic divisors
  auto decode = [&](int t, int& ns, int& nbi, int& tyi, int& txi) {
    int sp = fdiv(t, dv.nsplit);
    ns = t - sp * nsplit;
    int q = fdiv(sp, dv.tx);
    txi = sp - q * tiles_x;
    nbi = fdiv(q, dv.ty);
    tyi = q - nbi * tiles_y;
  };

  if (warp == WARP_TX) {
    if (lane == 0) {
      Ring rx(XS);
      int local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        int ns, nbi, tyi, txi;
        decode(t, ns, nbi, tyi, txi);
        for (int kc = 0; kc < nk; ++kc, rx.next()) {
          mbar_wait_sleep<128>(emptyX + rx.i, rx.ph ^ 1);
          if (kc == 0) stamp(local, 8);
          if (kc == nk - 1) stamp(local, 9);
          if (dbg & 8) {  // development: skip the X load (timing attribution only)
            mbar_arrive(fullX + rx.i);
            continue;
          }
          cstamp(local * nk + kc, 8);
          mbar_arrive_expect_tx(fullX + rx.i, xbytes);
          tma_load_4d(xbuf + rx.i * xstride, &tmx, fullX + rx.i, kc * KC, txi * tw * S - pl, tyi * th * S - pt, nbi * nb);
        }
      }
    }
  } else if (warp == WARP_TB) {
    if (lane == 0) {
      if (resB) {  // grid is a multiple of nsplit: this CTA's C_out slice is fixed
        const int ns = blockIdx.x - fdiv(blockIdx.x, dv.nsplit) * nsplit;
        for (int kc = 0; kc < nk; ++kc) {
          mbar_arrive_expect_tx(fullB + kc, BN * 128);
          tma_load_2d(bbuf + kc * BN * 128, &tmb, fullB + kc, kc * KC, ns * BN);
        }
      }
      Ring rb(BS);
      for (int t = blockIdx.x; t < total && !resB; t += gridDim.x) {
        const int ns = t - fdiv(t, dv.nsplit) * nsplit;
        for (int kc = 0; kc < nk; ++kc, rb.next()) {
          mbar_wait_sleep<128>(emptyB + rb.i, rb.ph ^ 1);
          mbar_arrive_expect_tx(fullB + rb.i, BN * 128);
          tma_load_2d(bbuf + rb.i * BN * 128, &tmb, fullB + rb.i, kc * KC, ns * BN);
        }
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, BN);
      Ring ra(na), rb(BS), rt(nacc);
      int local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local, rt.next()) {
        const int acc = rt.i;
        mbar_wait_sleep<128>(tempty + acc, rt.ph ^ 1);
        stamp(local, 0);
        tc_fence_after();
        const uint32_t d = tbase + acc * (MB * BN);
        for (int kc = 0; kc < nk; ++kc, ra.next(), rb.next()) {
          const int a = ra.i, sb = resB ? kc : rb.i;
          mbar_wait_sleep<64>(afull + a, ra.ph);
          cstamp(local * nk + kc, 6);
          if (kc == 0) stamp(local, 1);
          mbar_wait(fullB + sb, resB ? 0 : rb.ph);
          if (kSplit && local == 0 && kc == 0) mbar_wait(bconv, 0);
          tc_fence_after();
          // kPair: A (the commBuffer) in the no-swizzle K-major layout, a K step = 2 chunks of albo,
          // row block h starts 128 rows (2 KB) further
          const uint64_t ad = kPair ? smem_desc_interleave(smem_u32(abuf + a * aslot), albo)
                                    : smem_desc_sw128(smem_u32(abuf + a * aslot));
          const uint32_t astep = kPair ? (2 * albo) >> 4 : 2;
          const uint64_t bd = smem_desc_sw128(smem_u32(bbuf + sb * BN * 128));
          const int ksteps = min(4, (Cin - kc * KC + KSTEP - 1) / KSTEP);  // skip all-zero K steps
          // fully unrolled (MB <= 2, ksteps <= 4) with the descriptors formed up front: a rolled loop
          // serialises the per-MMA vector -> uniform register moves (~160 cycles per MMA measured)
          if (!(dbg & 256)) {
            uint64_t adk[2][4], bdk[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              bdk[k] = bd + 2 * k;
              adk[0][k] = ad + astep * k;
              adk[1][k] = ad + (2048 >> 4) + astep * k;
            }
            if constexpr (kSplit) {  // T_hi.W_hi + T_hi.W_lo + T_lo.W_hi (MB == 1)
              const uint64_t alo = 16384 >> 4, blo = (uint64_t)((nk * BN * 128) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (k < ksteps) {
                  mma_ss<KIND>(d, adk[0][k], bdk[k], idesc, (kc | k) != 0);
                  mma_ss<KIND>(d, adk[0][k], bdk[k] + blo, idesc, 1);
                  mma_ss<KIND>(d, adk[0][k] + alo, bdk[k], idesc, 1);
                }
            } else {
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  if (h < MB && k < ksteps) mma_ss<KIND>(d + h * BN, adk[h][k], bdk[k], idesc, (kc | k) != 0);
            }
          }
          mma_commit(aempty + a);
          cstamp(local * nk + kc, 7);
          if (!resB) mma_commit(emptyB + sb);
        }
        mma_commit(tfull + acc);
        stamp(local, 2);
      }
    }
  } else if (warp == WARP_RELAY) {
    Ring rx(XS), ra(na);
    int p = 0;
    for (int t = blockIdx.x; t < total && FCM_DWPW_RELAY; t += gridDim.x)
      for (int kc = 0; kc < nk; ++kc, rx.next(), ra.next(), ++p) {
        RELAY_WAIT(fullX + rx.i, rx.ph);
        if (lane == 0) cstamp(p, 0);
        RELAY_WAIT(aempty + ra.i, ra.ph ^ 1);
        if (lane == 0) cstamp(p, 1);
        named_bar_arrive(2 + (p & 1), kGoThreads);
      }
  } else if (warp >= 4) {
    // ---------------- DW warps: X halo chunk (smem) -> DW -> eps_dw -> A operand (commBuffer)
    constexpr int kSeg = 8;
    const int dw = warp - 4;
    const int nseg = (th + kSeg - 1) / kSeg;
    const uint32_t hi_c = kPair ? bound2<DT>(act_hi(ed.act)) : 0u;
    uint32_t W9[9];
    uint64_t sc2 = 0ull, bi2 = 0ull;
    int kc_w = -1;
    Ring rx(XS), ra(na);
    int local = 0, phase = 0;
    if constexpr (kSplit) {
      // resident fp32 PW weights (the launcher requires resB): W -> W_hi in place, W_lo after the
      // nk chunks (same SW128 positions), once per CTA; the MMA warp waits on bconv
      for (int c = 0; c < nk; ++c) mbar_wait(fullB + c, 0);
      const uint32_t b0 = smem_u32(bbuf), lo = (uint32_t)(nk * BN * 128);
      for (int v = dw * 32 + lane; v < nk * BN * 8; v += kDwpwNDW * 32) {
        const uint4 x = lds128(b0 + 16 * v);
        const uint4 h = make_uint4(x.x & 0xFFFFE000u, x.y & 0xFFFFE000u, x.z & 0xFFFFE000u, x.w & 0xFFFFE000u);
        sts128(b0 + 16 * v, h.x, h.y, h.z, h.w);
        sts128(b0 + lo + 16 * v, __float_as_uint(__uint_as_float(x.x) - __uint_as_float(h.x)),
               __float_as_uint(__uint_as_float(x.y) - __uint_as_float(h.y)),
               __float_as_uint(__uint_as_float(x.z) - __uint_as_float(h.z)),
               __float_as_uint(__uint_as_float(x.w) - __uint_as_float(h.w)));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bconv);
    }
    // start of a C_in-chunk phase: X stage full and A slot free (relay barrier or own mbarrier waits)
    auto go = [&]() {
      if constexpr (FCM_DWPW_RELAY) {
        named_bar_sync(2 + (phase & 1), kGoThreads);
      } else {
        mbar_wait(fullX + rx.i, rx.ph);
        mbar_wait(aempty + ra.i, ra.ph ^ 1);
      }
    };
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      for (int kc = 0; kc < nk; ++kc, rx.next(), ra.next(), ++phase) {
        const int sx = rx.i, a = ra.i;
        const uint32_t st = smem_u32(xbuf + sx * xstride);
        const uint32_t abase = smem_u32(abuf + a * aslot);
        if constexpr (kPair) {
          // lane groups: a partially filled chunk (C_in not a multiple of 64) packs 2 or 4 column
          // pairs into one warp (slots of 2^gsl lanes) instead of idling the empty lanes
          const int cw_valid = min(32, (Cin - kc * KC) >> 1);
          const int gi = cw_valid > 16 ? 0 : (cw_valid > 8 ? 1 : 2);
          const int gsl = 5 - gi, npl = gi;
          const int grp = lane >> gsl, wd = lane & ((1 << gsl) - 1);
          if (kc != kc_w) {  // this chunk's weights + scale / bias (once per CTA when nk == 1)
            load_dw3_h(wsm, nk * 32, kc * 32 + wd, W9, sc2, bi2);
            kc_w = kc;
          }
          const uint32_t lane_off = (wd >> 2) * albo + (wd & 3) * 4;
          constexpr int NC = kDwpwNC;
          const int hp = (tw + NC - 1) / NC;   // column groups per image row
          const int ncp = nb * hp;
          if (dw == 0 && lane == 0 && kc == 0) stamp(local, 10);
          if (dw == 0 && lane == 0) cstamp(phase, 2);
          go();
          if (dw == 0 && lane == 0) cstamp(phase, 3);
          if (dw == 0 && lane == 0 && kc == 0) stamp(local, 11);
          // item = (group of NC columns, segment of SEG rows); SEG (<= th) chosen on the host per
          // lane-group width. A ragged last segment / column group is shifted back inside the tile
          // (y0 = th - SEG, x0 = tw - NC): the overlap is recomputed with identical values, so every
          // item reads only staged rows (columns past a tile narrower than NC are not stored)
          const int seg_sel = (dv.seg_sel >> (8 * gi)) & 0xFF;
          const FDiv fnsg = gi == 0 ? dv.nsg[0] : (gi == 1 ? dv.nsg[1] : dv.nsg[2]);  // no dynamic param index (-> stack)
          {
            const int SEG = seg_sel;  // rows per item (runtime: the rolled core has one code path)
            with_act_r6<R6>(ed.act, [&](auto actc) {
              constexpr int ACT = decltype(actc)::value;
              const int nsg = (dv.nsgi >> (8 * gi)) & 0xFF;  // ceil(th / SEG), host-computed
              const int nit = ncp * nsg;
              const uint32_t rstep = (uint32_t)tw * 16;
              for (int base = dw << npl; base < nit && !(dbg & 1); base += kDwpwNDW << npl) {
                const int item = base + grp;
                const bool live = item < nit;
                const int iv = live ? item : 0;
                const int cp = fdiv(iv, fnsg), seg = iv - cp * nsg;
                const int b = fdiv(cp, dv.hp);
                const int x0 = max(0, min(NC * (cp - b * hp), tw - NC));
                const int y0 = min(seg * SEG, th - SEG);
                const uint32_t src = st + ((((b * th_in) + y0 * S) * tw_in + x0 * S) * 32 + wd) * 4;
                const int ncv = live ? min(NC, tw - x0) : 0;  // columns this lane stores
                const uint32_t a0 = abase + lane_off + (uint32_t)((b * th + y0) * tw + x0) * 16;
                dw3_cols_roll<DT, S, NC, 128>(src, tw_in * 128, SEG, W9, [&](int r, int c, float lo, float hi) {
                  const uint32_t v = epi_act2<DT, ACT>(lo, hi, sc2, bi2, hi_c);
                  if (c < ncv) sts32(a0 + r * rstep + c * 16, v);
                });
              }
            });
          }
        } else {
         bool done = false;
         if constexpr (DT == FCM_S8 && K == 3) {
          // int8: the exact column-pair FFMA2 core of the LBL DW (dw3_pair_i8), same lane groups;
          // a lane owns one word (4 channels) of two adjacent columns, rows stored to the SW128 A
          // tile. Chunks with <= 8 valid words (C_in = 32) stay on the per-column core (faster there).
          const int cw_valid = min(32, (Cin - kc * KC + 3) / 4);
          if (cw_valid > 8) {
          done = true;
          const int gs = cw_valid > 16 ? 32 : (cw_valid > 8 ? 16 : 8);
          const int npix = 32 / gs, grp = lane / gs, wd = lane - grp * gs;
          const int cl = kc * KC + wd * 4;
          // accumulators start at 0; bias_q is added in int32 after the exact conversion (as in dw.cu)
          const uint64_t bias[2] = {0ull, 0ull};
          uint64_t Wf[9][2];
          int32_t bq[4];
          RqI8 rq[4];
          {
            const uint32_t wa = smem_u32(wsm) + 4 * (kc * 32 + wd);
#pragma unroll
            for (int t9 = 0; t9 < 9; ++t9) {
              const uint32_t w = lds32(wa + 4 * t9 * nk * 32);
              float f[4];
#pragma unroll
              for (int v = 0; v < 4; ++v) f[v] = static_cast<float>(static_cast<int32_t>(w << (24 - 8 * v)) >> 24);
              Wf[t9][0] = f2_pack(f[0], f[1]);
              Wf[t9][1] = f2_pack(f[2], f[3]);
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const EpiC e = epic<DT>(dcs, cl + v);
              bq[v] = e.bq;
              rq[v] = make_rq(e.m, e.sh < 1 ? 40 : e.sh);
            }
          }
          const int zp = ed.zp_out, qmin = ed.qmin, qmax = ed.qmax;
          go();
          const int ncolp = (tw + 1) >> 1;
          const int ncg = (nb * ncolp + npix - 1) / npix;
          for (int item = dw; item < ncg * nseg; item += kDwpwNDW) {
            const int cg = item / nseg, seg = item - cg * nseg;
            const int cpr = cg * npix + grp;
            const bool live = cpr < nb * ncolp;
            const int cpi = live ? cpr : cg * npix;
            const int b = cpi / ncolp, x0 = 2 * (cpi - b * ncolp);
            const int y0 = seg * kSeg;
            const int nvalid = live ? th - y0 : 0;
            const bool c1 = x0 + 1 < tw;
            const uint32_t src = st + (((b * th_in) * tw_in + x0 * S) * 32 + wd) * 4;
            dw3_pair_i8<S, kSeg>(src, 128, tw_in * 128, y0, th_in - 1, Wf, bias, [&](int r, const uint64_t (&acc)[2][2]) {
              if (r < nvalid) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                  int32_t v[4];
                  f2_to_i2(acc[c][0], v[0], v[1]);
                  f2_to_i2(acc[c][1], v[2], v[3]);
                  uint32_t word = 0;
#pragma unroll
                  for (int q = 0; q < 4; ++q)
                    word |= (static_cast<uint32_t>(min(max(rq_apply(v[q] + bq[q], rq[q]) + zp, qmin), qmax)) & 0xFFu) << (8 * q);
                  const int m = (b * th + y0 + r) * tw + x0 + c;
                  if (c == 0 || c1) sts32(abase + sw128_off(m, wd), cl < Cin ? word : 0u);
                }
              }
            });
          }
          }
         }
         if constexpr (DT == FCM_F32 && K == 3) {
          // fp32 3x3: column-pair FFMA2 core (a lane = one channel of two adjacent output columns),
          // T written as T_hi / T_lo for the 3xTF32 PW; the same lane groups as the other cores
          done = true;
          const int cw_valid = min(32, Cin - kc * KC);
          const int gs = cw_valid > 16 ? 32 : (cw_valid > 8 ? 16 : 8);
          const int npix = 32 / gs, grp = lane / gs, wd = lane - grp * gs;
          const int cl = kc * KC + wd;
          uint64_t W2[9];
          {
            const uint32_t wa = smem_u32(wsm) + 4 * (kc * 32 + wd);
#pragma unroll
            for (int t9 = 0; t9 < 9; ++t9) {
              const float w = __uint_as_float(lds32(wa + 4 * t9 * nk * 32));
              W2[t9] = f2_pack(w, w);
            }
          }
          const EpiC ec = epic<DT>(dcs, cl);
          go();
          const int ncolp = (tw + 1) >> 1;
          const int ncg = (nb * ncolp + npix - 1) / npix;
          for (int item = dw; item < ncg * nseg; item += kDwpwNDW) {
            const int cg = item / nseg, seg = item - cg * nseg;
            const int cpr = cg * npix + grp;
            const bool live = cpr < nb * ncolp;
            const int cpi = live ? cpr : cg * npix;
            const int b = cpi / ncolp, x0 = 2 * (cpi - b * ncolp);
            const int y0 = seg * kSeg;
            const int nrows = live ? min(kSeg, th - y0) : 0;
            const bool c1 = x0 + 1 < tw;
            const uint32_t src = st + ((((b * th_in) + y0 * S) * tw_in + x0 * S) * 32 + wd) * 4;
            dw3_pair_f32<S, 128>(src, tw_in * 128, nrows, W2, [&](int r, int c, float a) {
              if (c == 1 && !c1) return;
              const int m = (b * th + y0 + r) * tw + x0 + c;
              const float v = cl < Cin ? act_f(fmaf(a, ec.sc, ec.bi), ed.act) : 0.f;
              const uint32_t word = __float_as_uint(v), hi = word & 0xFFFFE000u;
              sts32(abase + sw128_off(m, wd), hi);
              sts32(abase + 16384 + sw128_off(m, wd), __float_as_uint(v - __uint_as_float(hi)));
            });
          }
         }
         if (!done) {
          DwW<DT, K> W;
          // lane groups (as in the pair core): a partly filled channel chunk packs 2 or 4 output
          // columns into one warp; lanes past the valid words compute with zero weights and their
          // (finite) words meet zero PW weight rows, so they never reach the output
          const int cw_valid = min(32, (Cin - kc * KC + V - 1) / V);
          const int gs = cw_valid > 16 ? 32 : (cw_valid > 8 ? 16 : 8);
          const int npix = 32 / gs, grp = lane / gs, wd = lane - grp * gs;
          const int cl = kc * KC + wd * V;
          load_dw_weights_smem<DT, K>(W, wsm, nk * 32, kc * 32 + wd);
          EpiC ec[V];
#pragma unroll
          for (int v = 0; v < V; ++v) ec[v] = epic<DT>(dcs, cl + v);
          go();
          const int ncolg = (nb * tw + npix - 1) / npix;
          for (int item = dw; item < ncolg * nseg; item += kDwpwNDW) {
            const int cg = item / nseg, seg = item - cg * nseg;
            const int colr = cg * npix + grp;
            const bool live = colr < nb * tw;
            const int col = live ? colr : cg * npix;
            const int b = col / tw, x = col - b * tw;
            const int y0 = seg * kSeg;
            const uint32_t src = st + (((b * th_in) * tw_in + x * S) * 32 + wd) * 4;
            dw_segment<DT, K, S>(src, 128, tw_in * 128, y0, min(kSeg, th - y0), th_in - 1, W,
                                 [&](int yy, const typename Tr<DT>::acc_t(&acc)[V]) {
                                   const int m = (b * th + yy) * tw + x;
                                   const uint32_t word = (cl < Cin) ? epi_pack<DT>(acc, ec, ed) : 0u;
                                   if constexpr (kSplit) {  // T_hi (exact in tf32) and T_lo = T - T_hi
                                     const uint32_t hi = word & 0xFFFFE000u;
                                     if (live) {
                                       sts32(abase + sw128_off(m, wd), hi);
                                       sts32(abase + 16384 + sw128_off(m, wd),
                                             __float_as_uint(__uint_as_float(word) - __uint_as_float(hi)));
                                     }
                                   } else {
                                     if (live) sts32(abase + sw128_off(m, wd), word);
                                   }
                                 });
          }
         }
        }
        if (!(dbg & 64)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(afull + a);
          mbar_arrive(emptyX + sx);
        }
        if (dw == 0 && lane == 0 && kc == nk - 1) stamp(local, 7);
        if (dw == 0 && lane == 0) cstamp(phase, 4);
        if (dw == kDwpwNDW - 1 && lane == 0) cstamp(phase, 5);
      }
    }
  } else {
    // ---------------- epilogue warps 0-3: TMEM -> eps_pw -> global (lane = one output pixel)
    int local = 0;
    Ring rt(nacc);
    const int q = warp & 3;
    const int tpx = nb * th * tw;
    uint8_t* yb = static_cast<uint8_t*>(tmy_base);
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local, rt.next()) {
      const int acc = rt.i;
      int ns, nbi, tyi, txi;
      decode(t, ns, nbi, tyi, txi);
      const int valid = min(BN, Cout - ns * BN);
      // the <= 2 output pixels of this lane (row blocks h): NHWC offsets and validity
      size_t po0, po1;
      bool pok0, pok1;
      auto pix = [&](int h, size_t& po, bool& pok) {
        const int m = h * 128 + q * 32 + lane;
        const int b = fdiv(m, dv.thw), rem = m - b * (th * tw);
        const int yy = fdiv(rem, dv.tw), xx = rem - yy * tw;
        const int n = nbi * nb + b, yo = tyi * th + yy, xo = txi * tw + xx;
        pok = h < MB && m < tpx && n < N && yo < Ho && xo < Wo;
        po = pok ? (((size_t)n * Ho + yo) * Wo + xo) * Cout + (size_t)ns * BN : 0;
      };
      pix(0, po0, pok0);
      pix(1, po1, pok1);
      // residual (shortcut) words one 32-column step ahead; the first step's before the TMEM wait
      const bool hasres = ES == 2 && ep.residual != nullptr;
      Res32 rnext;
      if (hasres) res32_load(ep.residual, po0, 0, valid, pok0, rnext);
      group_wait_sleep(tfull + acc, rt.ph, warp == 0, 4, 128);
      if (threadIdx.x == 0) stamp(local, 3);
      tc_fence_after();
      for (int h = 0; h < MB && !(dbg & 2); ++h) {
        const bool ok = h ? pok1 : pok0;
        const size_t poh = h ? po1 : po0;
        uint8_t* dst = yb + poh * ES;
        const uint32_t tq = tbase + acc * (MB * BN) + h * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
        for (int c0 = 0; c0 < valid; c0 += 32) {
          Res32 rcur;
          if (hasres) {
            rcur = rnext;
            if (c0 + 32 < valid) res32_load(ep.residual, poh, c0 + 32, valid, ok, rnext);
            else if (h + 1 < MB) res32_load(ep.residual, po1, 0, valid, pok1, rnext);
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int cb = c0 + 16 * hh;  // 16 columns = 2 x 8-column (16 B bf16 / 8 B int8) pieces
            if (cb >= valid) break;
            uint32_t r[16];
            tmem_ld16(tq + cb, r);
            tmem_ld_wait();
            if constexpr (ES == 4) {  // fp32 output: act(acc * scale + bias) (+ residual), 4 x 16 B
              if (ok) {
                const float* rp = ep.residual ? static_cast<const float*>(ep.residual) + poh + cb : nullptr;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  if (cb + 4 * j < valid) {
                    const uint4 sc = lds128(cs.base + 4 * (ns * BN + cb + 4 * j));
                    const uint4 bi = lds128(cs.base + 4 * (cs.ncap + ns * BN + cb + 4 * j));
                    uint4 rs = make_uint4(0u, 0u, 0u, 0u);
                    if (rp) rs = ldg_nc128(rp + 4 * j);
                    const float* a = reinterpret_cast<const float*>(&r[4 * j]);
                    stg128(dst + cb * 4 + 16 * j,
                           __float_as_uint(act_f(fmaf(a[0], __uint_as_float(sc.x), __uint_as_float(bi.x)), ep.act) + __uint_as_float(rs.x)),
                           __float_as_uint(act_f(fmaf(a[1], __uint_as_float(sc.y), __uint_as_float(bi.y)), ep.act) + __uint_as_float(rs.y)),
                           __float_as_uint(act_f(fmaf(a[2], __uint_as_float(sc.z), __uint_as_float(bi.z)), ep.act) + __uint_as_float(rs.z)),
                           __float_as_uint(act_f(fmaf(a[3], __uint_as_float(sc.w), __uint_as_float(bi.w)), ep.act) + __uint_as_float(rs.w)));
                  }
              }
              continue;
            }
            uint32_t o[8];
            // (the residual: the shortcut input at the same NHWC position)
            epi16_any<DT, !R6>(r, cs, ep, ns * BN + cb, o, hasres, rcur.v[2 * hh], rcur.v[2 * hh + 1]);
            if (ok) {
              if constexpr (ES == 2) {
                stg128(dst + cb * 2, o[0], o[1], o[2], o[3]);
                if (cb + 8 < valid) stg128(dst + cb * 2 + 16, o[4], o[5], o[6], o[7]);
              } else {
                if (cb + 8 < valid) stg128(dst + cb, o[0], o[1], o[2], o[3]);
                else stg64(dst + cb, o[0], o[1]);
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (threadIdx.x == 0) stamp(local, 5);
    }
  }
  __syncthreads();
#ifdef FCM_TRACE_STAMPS
  if (trace && blockIdx.x == 0)
    for (int i = threadIdx.x; i < 64 * 12; i += blockDim.x) trace[(i / 12) * 16 + i % 12] = tr_sm[i];
#endif
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, tmem_cols);
  }
}

// =====================================================================================
// FCM PWDW_R. One tile = DW output tile (nb x th x tw) x TD intermediate channels (one 128-byte
// group). The PW runs over the tile's T HALO (R = nb*th_in*tw_in <= 256 rows, 1-2 M=128 MMAs):
// T pixels in the overlap are recomputed by every tile that needs them (the "_R"). T
// outside the image is written as 0 (DW pads T, reading R6).
// Warps 0-3: T producers (TMEM -> eps_pw -> smem T tile), warps 4-11: DW consumers (T -> DW ->
// eps_dw -> OFM), warp 12: TMA, warp 13: MMA. TMEM and the T tile are both double-buffered, so
// the PW of tile i+1, its epilogue and the DW of tile i proceed concurrently.
// =====================================================================================
constexpr int kPwdwNDW = 8;
// T-producer warps (TMEM -> T): 8 (two per TMEM lane quadrant) for 3x3, 4 for 5x5 (registers).
template <int K> constexpr int pwdw_ntp() { return K == 3 ? 8 : 4; }
// rows per DW item of the PWDW_R consumers (must match kSeg in the kernel)
template <int DT, int K, int S> constexpr int pwdw_seg() {
  return ((DT == FCM_BF16 || DT == FCM_F16) && K == 3) ? (S == 1 ? 16 : 8) : 8;
}
struct PwdwDivs {
  FDiv nslice, tx, ty, tw, nseg;  // tile decode + DW item decode
  FDiv hp, nsg;                   // pair core: column groups per image, ceil(th / seg)
  int seg;                        // pair core segment length
  FDiv thw_in, tw_in;             // T producers: halo row r -> (image, row, column)
  FDiv rot;                       // slice rotation period (spatial tiles per round of the grid)
  int nsgi;                       // ceil(th / seg)
};
template <int DT, int K> constexpr bool pwdw_pair() { return (DT == FCM_BF16 || DT == FCM_F16) && K == 3; }
template <int DT, int K> constexpr int pwdw_wbytes(int nslice) {
  return pwdw_pair<DT, K>() ? dw3h_bytes(nslice * 32) : K * K * nslice * 128;
}

template <int DT, int K, int S, bool R6 = false>  // R6: both activations RELU6 (as in dwpw_tc_kernel)
__global__ void __launch_bounds__((pwdw_ntp<K>() + kPwdwNDW + 2) * 32, 1)
    pwdw_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
                   const typename Tr<DT>::T* __restrict__ wdw, Epi ep, Epi ed, uint8_t* __restrict__ y, int N, int H,
                   int W, int Cin, int Ho, int Wo, int Cmid, int pt, int pl, int nb, int th, int tw, int tiles_x,
                   int tiles_y, int stages, int depth, uint32_t tmem_cols, int ncap, int resB, PwdwDivs dv,
                   int xb, int dbg, unsigned long long* trace) {
  pdl_launch();
  constexpr int ES = Tr<DT>::ES;
  constexpr int V = Tr<DT>::VEC;
  constexpr int KC = 128 / ES;
  constexpr int TD = 128 / ES;           // intermediate channels per tile
  constexpr int PITCH = 128 + 16;        // bytes per T row in smem (padded: conflict-free)
  constexpr int PW = PITCH / 4;
  constexpr MmaKind KIND = TcKind<DT>::kind;
  constexpr int KSTEP = 32 / Tr<DT>::ES;
  constexpr int NTP = pwdw_ntp<K>();
  constexpr int WARP_TMA = NTP + kPwdwNDW, WARP_MMA = NTP + 1 + kPwdwNDW;
  const int th_in = (th - 1) * S + K, tw_in = (tw - 1) * S + K;
  const int R = nb * th_in * tw_in;
  const int MB = (R + 127) / 128;
  // X halo rows of xb bytes (32 / 64 / 128: a C_in below 64 channels is staged at its own width,
  // not as 128-byte rows that are mostly out-of-bounds fill)
  const int xbytes = R * xb;
  const int astride = MB * 128 * xb;
  const int stage_bytes = astride + (resB ? 0 : TD * 128);
  const int tbytes = ((R * PITCH) + 1023) & ~1023;
  const int nslice = (Cmid + TD - 1) / TD;
  const int nk = (Cin + KC - 1) / KC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* tsm = smem + stages * stage_bytes;  // `depth` T buffers
  // resB 1: all PW weight slices x nk chunks resident; 2: only this CTA's slice (grid a multiple of
  // nslice, no slice rotation: the CTA's slice is fixed)
  const int nres = resB == 1 ? nslice : 1;
  uint8_t* bres = tsm + depth * tbytes;
  uint8_t* cst = bres + (resB ? nk * nres * TD * 128 : 0);
  uint8_t* dcst = cst + consts_bytes<DT>(ncap);
  uint32_t* wsm = reinterpret_cast<uint32_t*>(dcst + consts_bytes<DT>(ncap));
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(wsm) + pwdw_wbytes<DT, K>(nslice));
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 4;
  uint64_t* Tfull = tempty + 4;
  uint64_t* Tempty = Tfull + 4;
  uint64_t* bfull = Tempty + 4;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const EpiS cs = stage_consts<DT>(ep, Cmid, ncap, cst);
  const EpiS dcs = stage_consts<DT>(ed, Cmid, ncap, dcst);
  // pair core: raw packed weight words [9][nslice*32] + scale / bias pairs (stage_dw3_h)
  if constexpr (pwdw_pair<DT, K>()) stage_dw3_h<DT>(wdw, ed, Cmid, nslice * 32, wsm);
  else stage_dw_weights<DT>(wdw, K, Cmid, nslice * 32, wsm);
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch_desc(&tmx);
    tma_prefetch_desc(&tmb);
    for (int s = 0; s < stages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int a = 0; a < depth; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, NTP);  // one arrive per warp (after __syncwarp): TMEM reads only
      // the T tile (generic-proxy smem written by the producers, read by the DW consumers) is handed
      // over with every thread's own arrive: an explicit release by each writer / reader
      mbar_init(Tfull + a, NTP * 32);
      mbar_init(Tempty + a, kPwdwNDW * 32);
    }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == WARP_MMA) tmem_alloc_rt(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // previous kernel's outputs (our inputs) complete; our outputs free to overwrite
  const uint32_t tbase = *tslot;
  const int spatial = ((N + nb - 1) / nb) * tiles_y * tiles_x;
  const int total = spatial * nslice;
  const uint32_t acc_cols = MB * TD;

  // development tracing (FCM_TRACE): clock64 stamps of CTA 0's first 64 tiles
  auto stamp = [&](int local, int ev) {
    if (trace && blockIdx.x == 0 && local < 64) trace[local * 16 + ev] = clock64();
  };
  // tile t -> (spatial tile sp, C_mid slice): the slices of one spatial tile are consecutive tiles
  // (their X halo is one L2 fetch), rotated by sp / (grid / nslice) so that every CTA cycles
  // through the slices (a partly filled last slice is cheaper; a fixed slice per CTA left the
  // full-slice CTAs on the critical path)
  auto decode = [&](int t, int& sl, int& nbi, int& tyi, int& txi) {
    int sp = fdiv(t, dv.nslice);
    sl = t - sp * nslice;
    const int rot = fdiv(sp, dv.rot);
    sl += rot - fdiv(rot, dv.nslice) * nslice;
    if (sl >= nslice) sl -= nslice;
    int q = fdiv(sp, dv.tx);
    txi = sp - q * tiles_x;
    nbi = fdiv(q, dv.ty);
    tyi = q - nbi * tiles_y;
  };

  if (warp == WARP_TMA) {
    if (lane == 0) {
      const uint32_t tx = xbytes + (resB ? 0 : TD * 128);
      int it = 0;
      if (resB) {  // resident weight slices: loaded once per CTA
        mbar_arrive_expect_tx(bfull, nk * nres * TD * 128);
        for (int kc = 0; kc < nk; ++kc)
          for (int s2 = 0; s2 < nres; ++s2)
            tma_load_2d(bres + (kc * nres + s2) * TD * 128, &tmb, bfull, kc * KC,
                        (resB == 1 ? s2 : blockIdx.x % nslice) * TD);
      }
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int sl, nbi, tyi, txi;
        decode(t, sl, nbi, tyi, txi);
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          mbar_wait(empty + s, ((it / stages) & 1) ^ 1);
          if (kc == 0) stamp(it / nk, 8);
          uint8_t* st = smem + s * stage_bytes;
          if (dbg & 8) {
            mbar_arrive(full + s);
            continue;
          }
          mbar_arrive_expect_tx(full + s, tx);
          tma_load_4d(st, &tmx, full + s, kc * KC, txi * tw * S - pl, tyi * th * S - pt, nbi * nb);
          if (!resB) tma_load_2d(st + astride, &tmb, full + s, kc * KC, sl * TD);
        }
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, TD);
      int it = 0, local = 0;
      if (resB) mbar_wait(bfull, 0);
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int acc = local % depth;
        int sl, nbi, tyi, txi;
        decode(t, sl, nbi, tyi, txi);
        mbar_wait(tempty + acc, ((local / depth) & 1) ^ 1);
        stamp(local, 0);
        tc_fence_after();
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          mbar_wait(full + s, (it / stages) & 1);
          if (kc == 0) stamp(local, 1);
          tc_fence_after();
          uint8_t* st = smem + s * stage_bytes;
          const uint64_t bd =
              smem_desc_sw128(smem_u32(resB ? bres + (kc * nres + (resB == 1 ? sl : 0)) * TD * 128 : st + astride));
          for (int mb = 0; mb < MB; ++mb) {
            const uint64_t ad = smem_desc_swz(smem_u32(st + mb * 128 * xb), xb);
            const uint32_t d = tbase + acc * acc_cols + mb * TD;
            const int ksteps = min(xb / 32, (Cin - kc * KC + KSTEP - 1) / KSTEP);  // skip all-zero K steps
            for (int k = 0; k < ksteps; ++k) mma_ss<KIND>(d, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
          }
          mma_commit(empty + s);
        }
        mma_commit(tfull + acc);
        stamp(local, 2);
      }
    }
  } else if (warp < NTP) {
    // ---------------- T producers: TMEM (PW accumulators over the halo) -> eps_pw -> T (0 outside)
    constexpr int G = NTP / 4;      // warps per TMEM lane quadrant; each owns TD/G contiguous columns
    constexpr int CPW = TD / G;     // 32 or 64 (bf16), 64 or 128 (int8)
    constexpr int NU = CPW / 32;    // 32-column TMEM loads per M block
    const int q = warp & 3, h = warp >> 2;
    int local = 0;
    Ring rt(depth);
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local, rt.next()) {
      const int acc = rt.i;
      int sl, nbi, tyi, txi;
      decode(t, sl, nbi, tyi, txi);
      uint8_t* tb = tsm + acc * tbytes;
      if (warp == 0) {
        mbar_wait(tfull + acc, rt.ph);
        if (lane == 0) stamp(local, 3);
        mbar_wait(Tempty + acc, rt.ph ^ 1);
        if (lane == 0) stamp(local, 4);
      }
      named_bar_sync(2, NTP * 32);
      tc_fence_after();
      // eps_pw of 16 accumulator columns -> 8 T words: the packed bf16 / f16 fast path (FFMA2 affine,
      // cvt.rn(.relu) pack, min for RELU6 -- identical to the scalar fma / min / round) for the
      // clamp activations, the generic epilogue for SiLU / GELU and int8
      auto produce = [&](auto actc) {
        constexpr int ACT = decltype(actc)::value;
        const uint32_t hi_c = (ES == 2 && ACT == FCM_ACT_RELU6) ? bound2<DT>(6.f) : 0u;
        for (int mb = 0; mb < MB && !(dbg & 2); ++mb) {
          const int r = mb * 128 + q * 32 + lane;
          const int b = fdiv(r, dv.thw_in), rr = r - b * th_in * tw_in;
          const int ry = fdiv(rr, dv.tw_in);
          const int yi = tyi * th * S - pt + ry, xi = txi * tw * S - pl + (rr - ry * tw_in);
          const int n = nbi * nb + b;
          const bool inside = (r < R) && (n < N) && (yi >= 0) && (yi < H) && (xi >= 0) && (xi < W);
#pragma unroll 1
          for (int u = 0; u < NU; ++u) {
            if (sl * TD + h * CPW + 32 * u >= Cmid) break;  // columns past C_mid: never read by the DW
            uint32_t rg[32];
            tmem_ld32(tbase + ((uint32_t)(q * 32) << 16) + acc * acc_cols + mb * TD + h * CPW + 32 * u, rg);
            tmem_ld_wait();  // one round trip per 32 columns
            if (r < R) {
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int c0 = h * CPW + 32 * u + 16 * hh;
                uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                if (inside) {
                  if constexpr (ES == 2 && ACT <= FCM_ACT_RELU6) {
                    const uint32_t cb = cs.base + 4 * (sl * TD + c0);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                      const uint4 sc = lds128(cb + 16 * q4), bi = lds128(cb + 4 * cs.ncap + 16 * q4);
                      const uint32_t* a4 = &rg[16 * hh + 4 * q4];
                      o[2 * q4] = epi_act2<DT, ACT>(__uint_as_float(a4[0]), __uint_as_float(a4[1]),
                                                    f2_pack(__uint_as_float(sc.x), __uint_as_float(sc.y)),
                                                    f2_pack(__uint_as_float(bi.x), __uint_as_float(bi.y)), hi_c);
                      o[2 * q4 + 1] = epi_act2<DT, ACT>(__uint_as_float(a4[2]), __uint_as_float(a4[3]),
                                                        f2_pack(__uint_as_float(sc.z), __uint_as_float(sc.w)),
                                                        f2_pack(__uint_as_float(bi.z), __uint_as_float(bi.w)), hi_c);
                    }
                  } else {
                    epi16_any<DT>(&rg[16 * hh], cs, ep, sl * TD + c0, o, false, uint4{}, uint4{});
                  }
                }
                const uint32_t dst = smem_u32(tb) + r * PITCH + c0 * ES;
#pragma unroll
                for (int v = 0; v < ES; ++v) sts128(dst + 16 * v, o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
              }
            }
          }
        }
      };
      if constexpr (R6) {
        produce(std::integral_constant<int, FCM_ACT_RELU6>());
      } else if constexpr (ES == 2) {
        if (ep.act == FCM_ACT_RELU6) produce(std::integral_constant<int, FCM_ACT_RELU6>());
        else if (ep.act == FCM_ACT_RELU) produce(std::integral_constant<int, FCM_ACT_RELU>());
        else if (ep.act == FCM_ACT_NONE) produce(std::integral_constant<int, FCM_ACT_NONE>());
        else produce(std::integral_constant<int, 99>());
      } else {
        produce(std::integral_constant<int, 99>());
      }
      tc_fence_before();
      mbar_arrive(Tfull + acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (warp == 0 && lane == 0) stamp(local, 5);
    }
  } else {
    // ---------------- DW consumers: T tile -> DW -> eps_dw -> OFM (128 B per warp store)
    constexpr bool kPair = (DT == FCM_BF16 || DT == FCM_F16) && K == 3;
    constexpr int kSeg = pwdw_seg<DT, K, S>();
    const int dw = warp - NTP;
    const int nseg = (th + kSeg - 1) / kSeg;
    const int nitems = nb * tw * nseg;
    const uint32_t hi_c = bound2<DT>(act_hi(ed.act));
    uint32_t* yw = reinterpret_cast<uint32_t*>(y);
    uint32_t W9[9];
    uint64_t sc2 = 0ull, bi2 = 0ull;
    int sl_w = -1;
    // the activation is dispatched once for the whole role (not per tile)
    auto role = [&](auto actc) {
    constexpr int ACT = decltype(actc)::value;
    Ring rt(depth);
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local, rt.next()) {
      const int tbi = rt.i;
      int sl, nbi, tyi, txi;
      decode(t, sl, nbi, tyi, txi);
      const int c = sl * TD + lane * V;
      const uint32_t tsa = smem_u32(tsm + tbi * tbytes);
      const int y0t = tyi * th;
      const int nrows_t = min(th, Ho - y0t);
      if constexpr (kPair) {
        // column-group core (as in DWPW): a lane owns one channel word of NC adjacent output
        // columns x SEG rows; stores go straight to the NHWC OFM (128 B per warp and pixel)
        // lane groups: a partly filled last slice (C_mid not a multiple of 64) packs 2 or 4 items
        // into one warp (slots of 16 / 8 lanes) instead of computing idle channel words
        const int cw_valid = min(32, (Cmid - sl * TD) / V);
        const int gi = cw_valid > 16 ? 0 : (cw_valid > 8 ? 1 : 2);
        const int gsl = 5 - gi, grp = lane >> gsl, wd = lane & ((1 << gsl) - 1);
        if (sl != sl_w) {  // this slice's weights / scale / bias (once per CTA with resident slices)
          load_dw3_h(wsm, nslice * 32, sl * 32 + wd, W9, sc2, bi2);
          sl_w = sl;
        }
        const int cw = sl * TD + wd * V;
        const bool cval = cw < Cmid;
        constexpr int NC = kDwpwNC;
        const int hp = (tw + NC - 1) / NC;
        group_wait(Tfull + tbi, rt.ph, dw == 0, 3, kPwdwNDW * 32);
        if (dw == 0 && lane == 0) stamp(local, 6);
        const int SEG = dv.seg, nsg = dv.nsgi;  // rows per item (runtime, rolled core), segments
        const int nit = nb * hp * nsg;
        const uint32_t rstride = (uint32_t)Wo * Cmid / V, cstride = (uint32_t)Cmid / V;
        for (int base = dw << gi; base < nit && !(dbg & 1); base += kPwdwNDW << gi) {
          const int item = base + grp;
          if (item >= nit) continue;
          // ragged last segment / column group shifted back inside the tile (SEG <= th): the
          // overlap is recomputed and stored twice with identical values
          const int cp = fdiv(item, dv.nsg), seg = item - cp * nsg;
          const int b = fdiv(cp, dv.hp);
          const int x0 = max(0, min(NC * (cp - b * hp), tw - NC));
          const int n = nbi * nb + b, xo = txi * tw + x0;
          const int y0 = min(seg * SEG, th - SEG);
          if (n >= N || xo >= Wo || y0 >= nrows_t) continue;
          const uint32_t src = tsa + ((((b * th_in) + y0 * S) * tw_in + x0 * S) * PW + wd) * 4;
          const int nvalid = nrows_t - y0;
          const int ncv = cval ? min(min(NC, tw - x0), Wo - xo) : 0;  // columns stored
          uint32_t* dst = yw + ((((size_t)n * Ho + (y0t + y0)) * Wo + xo) * Cmid + cw) / V;
          dw3_cols_roll<DT, S, NC, PITCH>(src, tw_in * PITCH, SEG, W9, [&](int r, int cc, float lo, float hi) {
            if (r < nvalid && cc < ncv)
              dst[(uint32_t)r * rstride + (uint32_t)cc * cstride] = epi_act2<DT, ACT>(lo, hi, sc2, bi2, hi_c);
          });
        }
      } else {
        DwW<DT, K> Wd;
        load_dw_weights_smem<DT, K>(Wd, wsm, nslice * 32, sl * 32 + lane);
        EpiC ec[V];
#pragma unroll
        for (int v = 0; v < V; ++v) ec[v] = epic<DT>(dcs, c + v);
        group_wait(Tfull + tbi, rt.ph, dw == 0, 3, kPwdwNDW * 32);
        for (int item = dw; item < nitems; item += kPwdwNDW) {
          const int col = fdiv(item, dv.nseg), seg = item - col * nseg;
          const int b = fdiv(col, dv.tw), x = col - b * tw;
          const int n = nbi * nb + b, xo = txi * tw + x;
          const int y0 = seg * kSeg;
          if (n >= N || xo >= Wo || y0 >= nrows_t) continue;
          const uint32_t src = tsa + (((b * th_in) * tw_in + x * S) * PW + lane) * 4;
          dw_segment<DT, K, S>(src, PITCH, tw_in * PITCH, y0, min(kSeg, nrows_t - y0), th_in - 1, Wd,
                               [&](int yy, const typename Tr<DT>::acc_t(&a)[V]) {
                                 if (c < Cmid) {
                                   const size_t pix = ((size_t)n * Ho + (y0t + yy)) * Wo + xo;
                                   yw[(pix * Cmid + c) / V] = epi_pack<DT>(a, ec, ed);
                                 }
                               });
        }
      }
      mbar_arrive(Tempty + tbi);
      if (dw == 0 && lane == 0) stamp(local, 7);
    }
    };
    if constexpr (kPair) with_act_r6<R6>(ed.act, role);
    else role(std::integral_constant<int, 0>());
  }
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, tmem_cols);
  }
}

// ------------------------------------------------------------------------------- launchers
// FCM_DEBUG_FLAGS (env, development only): bit 0 skip DW math, bit 1 skip PW epilogue, bit 2 DW
// (bits 4/5: LBL PW skips its TMA store / its whole epilogue)
// warps do not wait for the TMA. Results are wrong when set; used to attribute time to roles.
static int debug_flags() {
  static int f = [] { const char* e = getenv("FCM_DEBUG_FLAGS"); return e ? atoi(e) : 0; }();
  return f;
}

// FCM_TRACE=<file> (development only): clock64 stamps of CTA 0 appended to <file> after each launch.
static unsigned long long* trace_buf() {
  static unsigned long long* buf = nullptr;
  static bool on = getenv("FCM_TRACE") != nullptr;
  if (on && !buf) {
    cudaMalloc(&buf, 64 * 16 * sizeof(unsigned long long));
    cudaMemset(buf, 0, 64 * 16 * sizeof(unsigned long long));
  }
  return on ? buf : nullptr;
}
static void trace_dump(const char* tag) {
  unsigned long long* b = trace_buf();
  if (!b) return;
  unsigned long long h[64 * 16];
  cudaDeviceSynchronize();
  cudaMemcpy(h, b, sizeof(h), cudaMemcpyDeviceToHost);
  FILE* f = fopen(getenv("FCM_TRACE"), "a");
  if (!f) return;
  fprintf(f, "# %s\n", tag);
  for (int t = 0; t < 64; ++t) {
    for (int e = 0; e < 12; ++e) fprintf(f, "%llu ", h[t * 16 + e]);
    fprintf(f, "\n");
  }
  fclose(f);
  cudaMemset(b, 0, sizeof(h));
}

static uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}
static inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

template <int DT>
static int pick_bn(int N, int nsplit, int& nb_out) {
  return fcm::pick_bn(N, nsplit, 128 / Tr<DT>::ES, nb_out);
}

static bool out_tmap_2d(CUtensorMap* m, int dt, void* y, int M, int N) {
  const int ES = elem_size(dt);
  const uint64_t dims[2] = {(uint64_t)N, (uint64_t)M};
  const uint64_t str[1] = {(uint64_t)N * ES};
  const uint32_t box[2] = {(uint32_t)(128 / ES), 32};  // one warp's 32 rows
  return encode_tmap(m, tmap_dtype(dt), 2, y, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int DT>
static int launch_pw_t(const void* x, const void* wp, const Epi& ep, void* y, int M, int K, int N, int nsplit_req,
                       cudaStream_t st) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  int nbn = 0;
  int BN = pick_bn<DT>(N, nsplit_req, nbn);
  if (DT == FCM_F32 && BN > 128) BN = pick_bn<DT>(N, (N + 127) / 128, nbn);  // 3xTF32 stages hold x, x_lo, w, w_lo
  CUtensorMap ta, tb, ty;
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
    const uint64_t str[1] = {(uint64_t)K * ES};
    const uint32_t box[2] = {(uint32_t)KC, 128};
    if (!encode_tmap(&ta, tmap_dtype(DT), 2, x, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PW A) failed");
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    const uint64_t str[1] = {(uint64_t)K * ES};
    const uint32_t box[2] = {(uint32_t)KC, (uint32_t)BN};
    if (!encode_tmap(&tb, tmap_dtype(DT), 2, wp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PW B) failed");
  }
  if (!out_tmap_2d(&ty, DT, y, M, N)) return set_error(FCM_E_CUDA, "tensor map (PW Y) failed");
  const int ncap = round_up(nbn * BN, 16);
  const int fixed = 1024 + 65536 + consts_bytes<DT>(ncap) + 512;
  const int budget = device_props().smem_optin - fixed;
  const int nk = (K + KC - 1) / KC;
  const int total = ((M + 127) / 128) * nbn;
  int grid = std::min(total, device_props().sms);
  // resident B: the CTA keeps its whole C_out slice of the weights in smem (grid a multiple of nbn
  // so the slice is fixed) when that still leaves >= 4 A stages
  const int resgrid = (grid / nbn) * nbn;
  const bool resB = DT != FCM_F32 && resgrid > 0 && budget - nk * BN * 128 >= 4 * 16384 && resgrid >= grid * 15 / 16;
  int stages;
  size_t smem;
  if (resB) {
    grid = resgrid;
    stages = std::min(std::max(2 * nk, 4), std::min(8, (budget - nk * BN * 128) / 16384));
    smem = (size_t)fixed + (size_t)stages * 16384 + (size_t)nk * BN * 128;
  } else {
    const int stage_bytes = (16384 + BN * 128) * (DT == FCM_F32 ? 2 : 1);
    stages = std::min(std::max(2 * nk, 4), std::min(8, budget / stage_bytes));
    if (stages < 2) return set_error(FCM_E_INFEASIBLE, "pw: not enough shared memory for 2 stages");
    smem = (size_t)fixed + (size_t)stages * stage_bytes;
  }
  // epilogue groups: 4 x nch warps per tile, so 4 / nch tiles can drain concurrently (2 TMEM
  // accumulators per group)
  // 3 chunks: two groups (slots of 2 warps per quadrant, 2 + 1 chunks) with one accumulator each;
  // the MMA still alternates between two accumulators (one per group)
  const int nchk = (BN * Tr<DT>::ES + 127) / 128;
  int ng = nchk >= 4 ? 1 : 4 / nchk;
  if (ng == 3) ng = 2;
  int nbuf = 2;
  if (nchk == 3 && 2 * BN <= 512) { ng = 2; nbuf = 1; }
  while (ng > 1 && nbuf * ng * BN > 512) ng /= 2;
  auto kern = pw_tc_kernel<DT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_k(kern, dim3(grid), dim3(DT == FCM_F32 ? 640 : 576), smem, st, ta, tb, ty, ep, M, N, K, BN, nbn, make_fdiv(nbn), stages, ng, nbuf,
           pow2_cols(nbuf * ng * BN),
                                ncap, resB ? 1 : 0, trace_buf(), debug_flags());
  const int rc = check_launch("pw_tc_kernel");
  trace_dump("pw");
  return rc;
}

int launch_pw_tc(int dt, const void* x, const void* wp, const Epi& ep, void* y, int M, int K, int N, int nsplit,
                 cudaStream_t st) {
  switch (dt) {
    case FCM_F32: return launch_pw_t<FCM_F32>(x, wp, ep, y, M, K, N, nsplit, st);
    case FCM_BF16: return launch_pw_t<FCM_BF16>(x, wp, ep, y, M, K, N, nsplit, st);
    case FCM_F16: return launch_pw_t<FCM_F16>(x, wp, ep, y, M, K, N, nsplit, st);
    case FCM_S8: return launch_pw_t<FCM_S8>(x, wp, ep, y, M, K, N, nsplit, st);
  }
  return set_error(FCM_E_UNSUPPORTED, "pw tensor-core path: dtype");
}

// Segment length of the column-pair DW items per lane-group width (1, 2 or 4 slots per warp):
// the fewest input rows per DW warp (rounds x rows per item, + 2 rows of per-item overhead).
template <int K, int S>
static DwDivs dwpw_divs(const Geo& g, int ndw, int nsplit) {
  const int hp = (g.tw + kDwpwNC - 1) / kDwpwNC;  // column groups per image row (pair core)
  int sel = 0;
  DwDivs d{};
  for (int gi = 0; gi < 3; ++gi) {
    const int slots = 1 << gi;
    int best = 1, bcost = 1 << 30;
    for (int seg = std::min(g.th, 32); seg >= std::max(1, (g.th + 254) / 255); --seg) {  // any length (rolled core); ragged ones shift up; <= 255 segments (byte field)
      const int nit = g.nb * hp * ((g.th + seg - 1) / seg);
      const int rounds = ((nit + slots - 1) / slots + ndw - 1) / ndw;
      const int cost = rounds * ((seg - 1) * S + K + 2);
      if (cost < bcost) { bcost = cost; best = seg; }
    }
    sel |= best << (8 * gi);
    d.nsg[gi] = make_fdiv((g.th + best - 1) / best);
    d.nsgi |= ((g.th + best - 1) / best) << (8 * gi);
  }
  const int tiles_x = (g.Wo + g.tw - 1) / g.tw, tiles_y = (g.Ho + g.th - 1) / g.th;
  d.hp = make_fdiv(hp);
  d.nsplit = make_fdiv(nsplit);
  d.tx = make_fdiv(tiles_x);
  d.ty = make_fdiv(tiles_y);
  d.thw = make_fdiv(g.th * g.tw);
  d.tw = make_fdiv(g.tw);
  d.seg_sel = sel;
  return d;
}

template <int DT, int K, int S>
static int launch_dwpw_t(const void* x, const void* wdw, const Epi& ed, const void* wp, const Epi& ep, void* y,
                         const Geo& g, int nsplit_req, cudaStream_t st) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  constexpr bool kPair = dwpw_pair<DT, K>();
  const int th_in = (g.th - 1) * S + K, tw_in = (g.tw - 1) * S + K;
  const int tpx = g.nb * g.th * g.tw;
  if (tpx > (kPair ? 256 : 128))
    return set_error(FCM_E_INFEASIBLE, "dwpw: tile has more pixels than the MMA rows (256 pair core, else 128)");
  if (th_in > 256 || tw_in > 256 || g.nb > 256) return set_error(FCM_E_INFEASIBLE, "dwpw: halo box > 256");
  const int MB = (tpx + 127) / 128;            // MMA row blocks of 128
  static const int albo_pad = [] { const char* e = getenv("FCM_ALBO_PAD"); return e ? atoi(e) : 16; }();  // dev
  const int albo = 16 * 128 * MB + albo_pad;    // interleave LBO (padded: conflict-free DW stores)
  int nsplit = 0;
  const int BN = pick_bn<DT>(g.Cout, nsplit_req, nsplit);
  if (2 * MB * BN > 512) return set_error(FCM_E_INFEASIBLE, "dwpw: 2 x (tile rows / 128) x C_out slice > 512 TMEM columns");
  CUtensorMap tx, tb;
  {
    const uint64_t dims[4] = {(uint64_t)g.C, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N};
    const uint64_t str[3] = {(uint64_t)g.C * ES, (uint64_t)g.W * g.C * ES, (uint64_t)g.H * g.W * g.C * ES};
    const uint32_t box[4] = {(uint32_t)KC, (uint32_t)tw_in, (uint32_t)th_in, (uint32_t)g.nb};
    if (!encode_tmap(&tx, tmap_dtype(DT), 4, x, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE))
      return set_error(FCM_E_CUDA, "tensor map (DWPW X) failed");
  }
  {
    const uint64_t dims[2] = {(uint64_t)g.C, (uint64_t)g.Cout};
    const uint64_t str[1] = {(uint64_t)g.C * ES};
    const uint32_t box[2] = {(uint32_t)KC, (uint32_t)BN};
    if (!encode_tmap(&tb, tmap_dtype(DT), 2, wp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (DWPW B) failed");
  }
  const int ncap = round_up(nsplit * BN, 16);
  const int nk = (g.C + KC - 1) / KC;
  static const int na_env = [] { const char* e = getenv("FCM_NA"); return e ? atoi(e) : 0; }();  // dev override
  const int na = na_env ? na_env : kDwpwNA;
  const int nacc = 2;
  constexpr int kSp = DT == FCM_F32 ? 2 : 1;  // fp32 3xTF32: T_hi / T_lo slots, W / W_lo resident
  const int aslot = kPair ? ((8 * albo + 1023) & ~1023) : 16384 * kSp;
  const int fixed = 1024 + na * aslot + consts_bytes<DT>(ncap) + consts_bytes<DT>(nk * KC) + dwpw_wbytes<DT, K>(nk) + 512;
  const int xstride = ((g.nb * th_in * tw_in * 128) + 1023) & ~1023;
  const int tiles_x = (g.Wo + g.tw - 1) / g.tw, tiles_y = (g.Ho + g.th - 1) / g.th;
  const int total = ((g.N + g.nb - 1) / g.nb) * tiles_x * tiles_y * nsplit;
  int grid = std::min(total, device_props().sms);
  int BS = 2;
  static const int xs_cap = [] { const char* e = getenv("FCM_XS_MAX"); return e ? atoi(e) : 6; }();  // dev override
#ifdef FCM_TRACE_STAMPS
  const int smem_cap = device_props().smem_optin - 64 * 12 * 8;  // the trace build's static stamp buffer
#else
  const int smem_cap = device_props().smem_optin;
#endif
  int XS = std::min(xs_cap, (smem_cap - fixed - BS * BN * 128) / xstride);
  if (XS < 2) return set_error(FCM_E_INFEASIBLE, "dwpw: tile too large for 2 X stages");
  // resident weights: grid a multiple of nsplit fixes each CTA's C_out slice; keep all nk chunks
  // unless that leaves fewer than min(XS, kXsMin) X stages: the X halo chunk is the latency-critical
  // load (a 14 x 14 x 64-channel box takes ~1-2.5k cycles to land; with 2 stages in flight the DW
  // phases wait on it), the weights are L2 hits either way
  static const int xs_min = [] { const char* e = getenv("FCM_XS_MIN"); return e ? atoi(e) : 4; }();
  const int resgrid = (grid / nsplit) * nsplit;
  const int xs_res = std::min(xs_cap, (smem_cap - fixed - nk * BN * 128 * kSp) / xstride);
  const bool resB = nk <= 16 && resgrid > 0 && resgrid >= grid * 15 / 16 && xs_res >= 2 &&
                    (DT == FCM_F32 || xs_res >= std::min(XS, xs_min));
  if (DT == FCM_F32 && !resB)  // the fp32 split keeps all weight chunks resident
    return set_error(FCM_E_INFEASIBLE, "dwpw fp32 (3xTF32): the C_in x C_out slice does not fit shared memory");
  if (resB) {
    grid = resgrid;
    BS = nk;
    XS = xs_res;
  }
  const size_t smem = (size_t)fixed + (size_t)BS * BN * 128 * (resB ? kSp : 1) + (size_t)XS * xstride;
  auto kern = dwpw_tc_kernel<DT, K, S>;
  if constexpr (dwpw_pair<DT, K>())
    if (ed.act == FCM_ACT_RELU6 && ep.act <= FCM_ACT_RELU6) kern = dwpw_tc_kernel<DT, K, S, true>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  using TT = typename Tr<DT>::T;
  DwDivs dv = dwpw_divs<K, S>(g, dwpw_ndw<DT, K>(), nsplit);
  static const bool verbose = getenv("FCM_VERBOSE") != nullptr;  // development: launch configuration
  if (verbose)
    fprintf(stderr, "dwpw: grid %d XS %d BS %d resB %d BN %d nsplit %d MB %d seg_sel %06x smem %zu\n", grid, XS, BS,
            (int)resB, BN, nsplit, MB, dv.seg_sel, smem);
  launch_k(kern, dim3(grid), dim3((4 + dwpw_ndw<DT, K>() + 4) * 32), smem, st, tx, tb, y, static_cast<const TT*>(wdw), ed, ep, g.N, g.C,
                                                              g.Ho, g.Wo, g.Cout, g.pt, g.pl, g.nb, g.th, g.tw,
                                                              tiles_x, tiles_y, nsplit, BN, XS, BS,
                                                              pow2_cols(nacc * MB * BN), ncap, resB ? 1 : 0, dv, na,
                                                              nacc, MB, albo, debug_flags(), trace_buf());
  const int rc = check_launch("dwpw_tc_kernel");
  trace_dump("dwpw");
  return rc;
}

template <int DT>
static int launch_dwpw_dt(const void* x, const void* wdw, const Epi& ed, const void* wp, const Epi& ep, void* y,
                          const Geo& g, int ns, cudaStream_t st) {
  if (g.k == 3 && g.s == 1) return launch_dwpw_t<DT, 3, 1>(x, wdw, ed, wp, ep, y, g, ns, st);
  if (g.k == 3 && g.s == 2) return launch_dwpw_t<DT, 3, 2>(x, wdw, ed, wp, ep, y, g, ns, st);
  if (g.k == 5 && g.s == 1) return launch_dwpw_t<DT, 5, 1>(x, wdw, ed, wp, ep, y, g, ns, st);
  if (g.k == 5 && g.s == 2) return launch_dwpw_t<DT, 5, 2>(x, wdw, ed, wp, ep, y, g, ns, st);
  return set_error(FCM_E_UNSUPPORTED, "dwpw: only k in {3,5}, stride in {1,2}");
}

int launch_dwpw_tc(int dt, const void* x, const void* wdw, const Epi& ed, const void* wp, const Epi& ep, void* y,
                   const Geo& g, int ns, cudaStream_t st) {
  switch (dt) {
    case FCM_F32: return launch_dwpw_dt<FCM_F32>(x, wdw, ed, wp, ep, y, g, ns, st);
    case FCM_BF16: return launch_dwpw_dt<FCM_BF16>(x, wdw, ed, wp, ep, y, g, ns, st);
    case FCM_F16: return launch_dwpw_dt<FCM_F16>(x, wdw, ed, wp, ep, y, g, ns, st);
    case FCM_S8: return launch_dwpw_dt<FCM_S8>(x, wdw, ed, wp, ep, y, g, ns, st);
  }
  return set_error(FCM_E_UNSUPPORTED, "dwpw tensor-core path: dtype");
}

// PWDW_R tile decode + DW item decode; the pair core's segment length is the one with the fewest
// input rows per DW warp (rounds x rows per item, + 2 rows of per-item overhead).
template <int DT, int K, int S>
static PwdwDivs pwdw_divs(const Geo& g, int nslice, int tiles_x, int tiles_y, int grid, int resB) {
  const int hp = (g.tw + kDwpwNC - 1) / kDwpwNC;
  int best = 1, bcost = 1 << 30;
  for (int seg = std::min(g.th, 32); seg >= 1; --seg) {  // any length (rolled core); ragged ones shift up
    const int nit = g.nb * hp * ((g.th + seg - 1) / seg);
    const int rounds = (nit + kPwdwNDW - 1) / kPwdwNDW;
    const int cost = rounds * ((seg - 1) * S + K + 2);
    if (cost < bcost) { bcost = cost; best = seg; }
  }
  return PwdwDivs{make_fdiv(nslice), make_fdiv(tiles_x), make_fdiv(tiles_y), make_fdiv(g.tw),
                  make_fdiv((g.th + pwdw_seg<DT, K, S>() - 1) / pwdw_seg<DT, K, S>()), make_fdiv(hp),
                  make_fdiv((g.th + best - 1) / best), best,
                  make_fdiv(((g.th - 1) * S + K) * ((g.tw - 1) * S + K)), make_fdiv((g.tw - 1) * S + K),
                  make_fdiv(resB == 2 ? (1 << 30) : std::max(1, grid / nslice)), (g.th + best - 1) / best};
}

template <int DT, int K, int S>
static int launch_pwdw_t(const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                         const Geo& g, cudaStream_t st) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  constexpr int TD = 128 / ES;
  const int th_in = (g.th - 1) * S + K, tw_in = (g.tw - 1) * S + K;
  const int R = g.nb * th_in * tw_in;
  if (R > 512) return set_error(FCM_E_INFEASIBLE, "pwdw_r: halo tile has more than 512 pixels");
  const int MB = (R + 127) / 128;
  // X box width: the pixel's C_in bytes rounded up to 32 / 64, else 128-byte channel chunks
  const int xb = g.C * ES <= 32 ? 32 : (g.C * ES <= 64 ? 64 : 128);
  CUtensorMap tx, tb;
  {
    const uint64_t dims[4] = {(uint64_t)g.C, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N};
    const uint64_t str[3] = {(uint64_t)g.C * ES, (uint64_t)g.W * g.C * ES, (uint64_t)g.H * g.W * g.C * ES};
    const uint32_t box[4] = {(uint32_t)(xb / ES), (uint32_t)tw_in, (uint32_t)th_in, (uint32_t)g.nb};
    const CUtensorMapSwizzle sw = xb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                            : (xb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    if (!encode_tmap(&tx, tmap_dtype(DT), 4, x, dims, str, box, sw))
      return set_error(FCM_E_CUDA, "tensor map (PWDW X) failed");
  }
  {
    const uint64_t dims[2] = {(uint64_t)g.C, (uint64_t)g.Cout};
    const uint64_t str[1] = {(uint64_t)g.C * ES};
    const uint32_t box[2] = {(uint32_t)KC, (uint32_t)TD};
    if (!encode_tmap(&tb, tmap_dtype(DT), 2, wp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PWDW B) failed");
  }
  const int tbytes = ((R * (128 + 16)) + 1023) & ~1023;
  const int ncap = round_up(g.Cout, TD);
  const int nslice = ncap / TD;
  const int nk = (g.C + KC - 1) / KC;
  const int depth = std::min(3, 512 / (MB * TD));  // TMEM accumulators = T buffers in flight
  const int fixed = 1024 + 2 * consts_bytes<DT>(ncap) + pwdw_wbytes<DT, K>(nslice) + 512;
  const int tiles_x = (g.Wo + g.tw - 1) / g.tw, tiles_y = (g.Ho + g.th - 1) / g.th;
  const int total = ((g.N + g.nb - 1) / g.nb) * tiles_x * tiles_y * nslice;
  int grid = std::min(total, device_props().sms);
  // resident weights: all nk x nslice weight tiles loaded once per CTA when they take <= 64 KB and
  // fit (mode 1); else this CTA's own slice with the grid a multiple of nslice (mode 2); else one
  // B tile per X stage
  auto plan = [&](int res, int& stages, int& dep) {
    const int sb = MB * 128 * xb + (res ? 0 : TD * 128);
    const int extra = res == 1 ? nk * nslice * TD * 128 : (res == 2 ? nk * TD * 128 : 0);
    for (dep = depth; dep >= 2; --dep) {
      stages = std::min(4, (device_props().smem_optin - fixed - extra - dep * tbytes) / sb);
      if (stages >= 2) return (size_t)fixed + extra + (size_t)dep * tbytes + (size_t)stages * sb;
    }
    stages = 0;
    return (size_t)0;
  };
  int stages = 0, dep = 0;
  int resB = 0;
  size_t smem = 0;
  const int resgrid = (grid / nslice) * nslice;
  if (nk * nslice * TD * 128 <= 64 * 1024 && (smem = plan(1, stages, dep)) && stages >= 2) {
    resB = 1;
  } else if (resgrid > 0 && resgrid >= grid * 15 / 16 && (smem = plan(2, stages, dep)) && stages >= 2) {
    resB = 2;
    grid = resgrid;
  } else {
    smem = plan(0, stages, dep);
  }
  if (stages < 2) return set_error(FCM_E_INFEASIBLE, "pwdw_r: tile too large for 2 smem stages");
  auto kern = pwdw_tc_kernel<DT, K, S>;
  if constexpr (pwdw_pair<DT, K>())
    if (ed.act == FCM_ACT_RELU6 && ep.act == FCM_ACT_RELU6) kern = pwdw_tc_kernel<DT, K, S, true>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  using TT = typename Tr<DT>::T;
  launch_k(kern, dim3(grid), dim3((pwdw_ntp<K>() + kPwdwNDW + 2) * 32), smem, st, tx, tb, static_cast<const TT*>(wdw), ep, ed,
                                                     static_cast<uint8_t*>(y), g.N, g.H, g.W, g.C, g.Ho, g.Wo, g.Cout,
                                                     g.pt, g.pl, g.nb, g.th, g.tw, tiles_x, tiles_y, stages, dep,
                                                     pow2_cols(dep * MB * TD), ncap, resB,
                                                     pwdw_divs<DT, K, S>(g, nslice, tiles_x, tiles_y, grid, resB), xb,
                                                     debug_flags(), trace_buf());
  const int rc = check_launch("pwdw_tc_kernel");
  trace_dump("pwdw");
  return rc;
}

template <int DT>
static int launch_pwdw_dt(const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                          const Geo& g, cudaStream_t st) {
  if (g.k == 3 && g.s == 1) return launch_pwdw_t<DT, 3, 1>(x, wp, ep, wdw, ed, y, g, st);
  if (g.k == 3 && g.s == 2) return launch_pwdw_t<DT, 3, 2>(x, wp, ep, wdw, ed, y, g, st);
  if (g.k == 5 && g.s == 1) return launch_pwdw_t<DT, 5, 1>(x, wp, ep, wdw, ed, y, g, st);
  if (g.k == 5 && g.s == 2) return launch_pwdw_t<DT, 5, 2>(x, wp, ep, wdw, ed, y, g, st);
  return set_error(FCM_E_UNSUPPORTED, "pwdw_r: only k in {3,5}, stride in {1,2}");
}

int launch_pwdw_tc(int dt, const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                   const Geo& g, cudaStream_t st) {
  switch (dt) {
    case FCM_BF16: return launch_pwdw_dt<FCM_BF16>(x, wp, ep, wdw, ed, y, g, st);
    case FCM_F16: return launch_pwdw_dt<FCM_F16>(x, wp, ep, wdw, ed, y, g, st);
    case FCM_S8: return launch_pwdw_dt<FCM_S8>(x, wp, ep, wdw, ed, y, g, st);
  }
  return set_error(FCM_E_UNSUPPORTED, "pwdw_r tensor-core path: dtype");
}

// =====================================================================================
// FCM PWPW: Y = eps2(T . W2), T = eps1(X . W1) rounded to
// the feature-map dtype, for one 128-row tile at a time. T never leaves the CTA: GEMM1
// accumulates in TMEM, the 4 epilogue warps write T as the SW128 K-major A operand of GEMM2
// (zero / zero-point padded past C_mid, whose W2 columns are TMA zero fill), GEMM2 runs over
// C_out slices of BN2 <= 192 columns into two alternating TMEM accumulators. Warps 0-3 produce T
// (epilogue 1), warps 4-15 drain GEMM2 (epilogue 2: three warps per lane quadrant), 16 TMA of X / W1,
// 17 MMA, 18 TMA of W2 (resident when it fits: loaded once per CTA),
// so T of tile t+1 is produced while the slices of tile t drain. C_mid <= 128.
// =====================================================================================
template <int DT>
__global__ void __launch_bounds__(608, 1)
    pwpw_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb1,
                   const __grid_constant__ CUtensorMap tmb2, const __grid_constant__ CUtensorMap tmy, Epi ep1,
                   Epi ep2, int M, int K1, int Cmid, int N, int BN1, int BN2, int nbn2, int stages, int w2slots,
                   int resW2, uint32_t tmem_cols, int ncap1, int ncap2, int dbg) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  constexpr MmaKind KIND = TcKind<DT>::kind;
  constexpr int KSTEP = 32 / Tr<DT>::ES;
  pdl_launch();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int nk1 = (K1 + KC - 1) / KC, nk2 = (Cmid + KC - 1) / KC;
  const int sA = 16384 + BN1 * 128;              // X chunk + W1 chunk per stage
  uint8_t* ring = smem;                          // stages x sA
  uint8_t* tbuf = ring + stages * sA;            // T: nk2 x 16 KB SW128 chunks (128 rows)
  uint8_t* w2buf = tbuf + nk2 * 16384;           // w2slots x BN2 x 128: W2 chunk ring, or all chunks (resW2)
  uint8_t* stage = w2buf + w2slots * BN2 * 128;        // 12 epilogue-2 warps x 4 KB output staging
  uint8_t* cst1 = stage + 12 * 4096;
  uint8_t* cst2 = cst1 + consts_bytes<DT>(ncap1);
  uint64_t* full = reinterpret_cast<uint64_t*>(cst2 + consts_bytes<DT>(ncap2));
  uint64_t* empty = full + stages;
  uint64_t* w2full = empty + stages;
  uint64_t* w2empty = w2full + w2slots;
  uint64_t* acc1full = w2empty + w2slots;
  uint64_t* tready = acc1full + 1;
  uint64_t* tfree = tready + 1;
  uint64_t* acc2full = tfree + 1;
  uint64_t* acc2empty = acc2full + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acc2empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const EpiS cs1 = stage_consts<DT>(ep1, Cmid, ncap1, cst1);
  const EpiS cs2 = stage_consts<DT>(ep2, N, ncap2, cst2);
  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmb1);
    tma_prefetch_desc(&tmb2);
    tma_prefetch_desc(&tmy);
    for (int i = 0; i < stages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    for (int i = 0; i < w2slots; ++i) { mbar_init(w2full + i, 1); mbar_init(w2empty + i, 1); }
    mbar_init(acc1full, 1);
    mbar_init(tready, 128);  // every epilogue thread releases its own T writes
    mbar_init(tfree, 1);
    for (int i = 0; i < 2; ++i) { mbar_init(acc2full + i, 1); mbar_init(acc2empty + i, 12); }
    fence_barrier_init();
  }
  if (warp == 17) tmem_alloc_rt(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tbase = *tslot;
  const uint32_t tacc1 = tbase, tacc2 = tbase + 128;  // acc1: <= 128 columns, acc2: 2 x BN2 columns
  const int nbm = (M + 127) / 128;

  if (warp == 16) {
    if (lane == 0) {
      Ring rs(stages);
      for (int t = blockIdx.x; t < nbm; t += gridDim.x) {
        for (int kc = 0; kc < nk1; ++kc, rs.next()) {
          mbar_wait(empty + rs.i, rs.ph ^ 1);
          mbar_arrive_expect_tx(full + rs.i, sA);
          tma_load_2d(ring + rs.i * sA, &tma, full + rs.i, kc * KC, t * 128);
          tma_load_2d(ring + rs.i * sA + 16384, &tmb1, full + rs.i, kc * KC, 0);
        }
      }
    }
  } else if (warp == 18) {
    if (lane == 0) {
      if (resW2) {
        for (int j = 0; j < nbn2; ++j)
          for (int kc = 0; kc < nk2; ++kc) {
            const int sl = j * nk2 + kc;
            mbar_arrive_expect_tx(w2full + sl, BN2 * 128);
            tma_load_2d(w2buf + sl * BN2 * 128, &tmb2, w2full + sl, kc * KC, j * BN2);
          }
      } else {
        Ring rw(w2slots);
        for (int t = blockIdx.x; t < nbm; t += gridDim.x)
          for (int j = 0; j < nbn2; ++j)
            for (int kc = 0; kc < nk2; ++kc, rw.next()) {
              mbar_wait(w2empty + rw.i, rw.ph ^ 1);
              mbar_arrive_expect_tx(w2full + rw.i, BN2 * 128);
              tma_load_2d(w2buf + rw.i * BN2 * 128, &tmb2, w2full + rw.i, kc * KC, j * BN2);
            }
      }
    }
  } else if (warp == 17) {
    if (lane == 0) {
      const uint32_t idesc1 = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, BN1);
      const uint32_t idesc2 = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, BN2);
      Ring rs(stages), rw(w2slots), ra(2);
      uint32_t ph_t = 0;
      for (int t = blockIdx.x; t < nbm; t += gridDim.x) {
        // GEMM1: acc1 = X . W1^T over the C_in chunks (acc1 was drained: tready of the last tile)
        for (int kc = 0; kc < nk1; ++kc, rs.next()) {
          mbar_wait(full + rs.i, rs.ph);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(ring + rs.i * sA));
          const uint64_t bd = smem_desc_sw128(smem_u32(ring + rs.i * sA + 16384));
          const int ksteps = min(4, (K1 - kc * KC + KSTEP - 1) / KSTEP);
          for (int k = 0; k < ksteps && !(dbg & 256); ++k)
            mma_ss<KIND>(tacc1, ad + 2 * k, bd + 2 * k, idesc1, (kc | k) != 0);
          mma_commit(empty + rs.i);
        }
        mma_commit(acc1full);
        // GEMM2 over the C_out slices, A = the T tile in smem
        mbar_wait(tready, ph_t);
        ph_t ^= 1;
        tc_fence_after();
        for (int j = 0; j < nbn2; ++j, ra.next()) {
          mbar_wait(acc2empty + ra.i, ra.ph ^ 1);
          tc_fence_after();
          const uint32_t d2 = tacc2 + ra.i * BN2;
          for (int kc = 0; kc < nk2; ++kc, rw.next()) {
            const int sl = resW2 ? j * nk2 + kc : rw.i;
            mbar_wait(w2full + sl, resW2 ? 0 : rw.ph);
            tc_fence_after();
            const uint64_t ad = smem_desc_sw128(smem_u32(tbuf + kc * 16384));
            const uint64_t bd = smem_desc_sw128(smem_u32(w2buf + sl * BN2 * 128));
            const int ksteps = min(4, (Cmid - kc * KC + KSTEP - 1) / KSTEP);
            for (int k = 0; k < ksteps && !(dbg & 256); ++k)
              mma_ss<KIND>(d2, ad + 2 * k, bd + 2 * k, idesc2, (kc | k) != 0);
            if (!resW2) mma_commit(w2empty + rw.i);
          }
          mma_commit(acc2full + ra.i);
        }
        mma_commit(tfree);  // every GEMM2 of this tile has read T
      }
    }
  } else if (warp < 4) {
    // epilogue 1, warps 0-3 (lane quadrant q = warp): acc1 -> eps1 -> T (SW128 K-major, FM dtype)
    const int q = warp;
    const int m = q * 32 + lane;
    uint32_t ph_a1 = 0, ph_f = 0;
    bool first = true;
    for (int t = blockIdx.x; t < nbm; t += gridDim.x) {
      if (warp == 0) {
        mbar_wait(acc1full, ph_a1);
        if (!first) mbar_wait(tfree, ph_f);  // GEMM2 of the previous tile has finished reading T
      }
      named_bar_sync(2, 128);
      ph_a1 ^= 1;
      if (!first) ph_f ^= 1;
      first = false;
      tc_fence_after();
      for (int c0 = 0; c0 < nk2 * KC; c0 += 16) {
        uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // columns past the GEMM1 width: zeros (never stale TMEM)
        if (c0 < BN1) {
          uint32_t r[16];
          tmem_ld16(tacc1 + ((uint32_t)(q * 32) << 16) + c0, r);
          tmem_ld_wait();
          epi16_any<DT>(r, cs1, ep1, c0, o, false, uint4{}, uint4{});
        }
        const int kc = c0 / KC, vi0 = (c0 % KC) * ES / 16;
#pragma unroll
        for (int v = 0; v < ES; ++v)
          sts128(smem_u32(tbuf + kc * 16384) + sw128_vec(m, vi0 + v), o[4 * v], o[4 * v + 1], o[4 * v + 2],
                 o[4 * v + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(tready);
    }
  } else if (warp < 16) {
    // epilogue 2, warps 4-15: three warps per lane quadrant split a slice's 128-byte column chunks
    const int w2i = warp - 4, hs = w2i >> 2;
    Ring ra(2);
    int sbuf = 0;
    for (int t = blockIdx.x; t < nbm; t += gridDim.x) {
      for (int j = 0; j < nbn2; ++j, ra.next()) {
        group_wait(acc2full + ra.i, ra.ph, warp == 4, 3, 12 * 32);
        tc_fence_after();
        epilogue_tile_warp<DT>(tacc2 + ra.i * BN2, BN2, j * BN2, N, cs2, ep2, stage + w2i * 4096, sbuf, hs, 3,
                               (long)t * 128, M,
                               [&](const uint8_t* buf, int c, int rr) { tma_store_2d(&tmy, buf, c, t * 128 + rr); });
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc2empty + ra.i);
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  __syncthreads();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, tmem_cols);
  }
}

template <int DT>
static int launch_pwpw_t(const void* x, const void* w1, const Epi& ep1, const void* w2, const Epi& ep2, void* y, int M,
                         int K1, int Cmid, int N, cudaStream_t st) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  if (Cmid > 128) return set_error(FCM_E_UNSUPPORTED, "pwpw: C_mid > 128 (T must fit one M=128 x N<=128 accumulator)");
  const int BN1 = round_up(Cmid, 16);
  int nbn2 = (N + 191) / 192;  // BN2 <= 192: acc1 (128) + 2 x BN2 TMEM columns <= 512
  int BN2 = round_up((N + nbn2 - 1) / nbn2, 16);
  nbn2 = (N + BN2 - 1) / BN2;
  CUtensorMap ta, tb1, tb2, ty;
  {
    const uint64_t dims[2] = {(uint64_t)K1, (uint64_t)M};
    const uint64_t str[1] = {(uint64_t)K1 * ES};
    const uint32_t box[2] = {(uint32_t)KC, 128};
    if (!encode_tmap(&ta, tmap_dtype(DT), 2, x, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PWPW X) failed");
  }
  {
    const uint64_t dims[2] = {(uint64_t)K1, (uint64_t)Cmid};
    const uint64_t str[1] = {(uint64_t)K1 * ES};
    const uint32_t box[2] = {(uint32_t)KC, (uint32_t)BN1};
    if (!encode_tmap(&tb1, tmap_dtype(DT), 2, w1, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PWPW W1) failed");
  }
  {
    const uint64_t dims[2] = {(uint64_t)Cmid, (uint64_t)N};
    const uint64_t str[1] = {(uint64_t)Cmid * ES};
    const uint32_t box[2] = {(uint32_t)KC, (uint32_t)BN2};
    if (!encode_tmap(&tb2, tmap_dtype(DT), 2, w2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PWPW W2) failed");
  }
  if (!out_tmap_2d(&ty, DT, y, M, N)) return set_error(FCM_E_CUDA, "tensor map (PWPW Y) failed");
  const int nk2 = (Cmid + KC - 1) / KC;
  const int ncap1 = round_up(nk2 * KC, 16), ncap2 = round_up(nbn2 * BN2, 16);
  const int sA = 16384 + BN1 * 128;
  // W2 resident (all nbn2 x nk2 chunks loaded once per CTA) when that still leaves >= 3 stages
  const int base = 1024 + nk2 * 16384 + 12 * 4096 + consts_bytes<DT>(ncap1) + consts_bytes<DT>(ncap2) + 1024;
  const int nres = nbn2 * nk2;
  const bool resW2 = nres <= 24 && base + nres * BN2 * 128 + 3 * sA <= device_props().smem_optin;
  const int w2slots = resW2 ? nres : 2;
  const int fixed = base + w2slots * BN2 * 128;
  const int stages = std::min(6, (device_props().smem_optin - fixed) / sA);
  if (stages < 2) return set_error(FCM_E_INFEASIBLE, "pwpw: not enough shared memory for 2 stages");
  const size_t smem = (size_t)fixed + (size_t)stages * sA;
  const int nbm = (M + 127) / 128;
  const int grid = std::min(nbm, device_props().sms);
  auto kern = pwpw_tc_kernel<DT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_k(kern, dim3(grid), dim3(608), smem, st, ta, tb1, tb2, ty, ep1, ep2, M, K1, Cmid, N, BN1, BN2, nbn2, stages,
           w2slots, resW2 ? 1 : 0, pow2_cols(128 + 2 * BN2), ncap1, ncap2, debug_flags());
  return check_launch("pwpw_tc_kernel");
}

int launch_pwpw_tc(int dt, const void* x, const void* w1, const Epi& ep1, const void* w2, const Epi& ep2, void* y,
                   int M, int K1, int Cmid, int N, cudaStream_t st) {
  switch (dt) {
    case FCM_BF16: return launch_pwpw_t<FCM_BF16>(x, w1, ep1, w2, ep2, y, M, K1, Cmid, N, st);
    case FCM_F16: return launch_pwpw_t<FCM_F16>(x, w1, ep1, w2, ep2, y, M, K1, Cmid, N, st);
    case FCM_S8: return launch_pwpw_t<FCM_S8>(x, w1, ep1, w2, ep2, y, M, K1, Cmid, N, st);
  }
  return set_error(FCM_E_UNSUPPORTED, "pwpw tensor-core path: dtype");
}


// =====================================================================================
// LBL int8 DW on the tensor cores (stride 1, k in {3, 5}). A depthwise tap is a matrix product
// with a DIAGONAL weight block: for output pixels m (rows) and channels c of a 32-channel group,
//   O[m, c] += X[m shifted by the tap, c] * w[tap, c]  =  (A_tap . diag(w_tap))[m, c]
// with A_tap = the staged X halo tile viewed from the tap's offset. The X tile is TMA-loaded in the
// 128-byte-swizzled K-major layout (a pixel = one 128-byte row of 128 int8 channels); an output
// tile of 16 rows x 8 columns is M = 128 MMA rows whose 8-row core-matrix groups are the output
// rows, so the tap view is the same tile descriptor started (dy * tw_in + dx) rows further with
// SBO = tw_in * 128 B (no data movement; verified: tools/microbench/dw_mma_rate.cu). One
// tcgen05.mma kind::i8 (M 128, N 32, K 32) per tap and 32-channel group accumulates exact int32 in
// TMEM; 4 epilogue warps requantise (int32 bias, fixed-point multiplier, zero point, clamp:
// reading R1) and store 128-bit rows. 32 of the 1024 MACs per weight column are useful, but the
// tensor pipe still retires ~85 useful int8 MACs/clk/SM (MMA floor ~48 cycles, measured) against
// ~17 for the CUDA-core int8 DW, and it leaves the CUDA cores to the epilogue.
// Persistent: CTA (i, chunk) keeps the chunk's diagonal weight blocks (k^2 x 4 KB) resident and
// loops over spatial tiles; 2-stage X ring, 2 TMEM accumulators; warp 0 TMA, warp 1 MMA, warps
// 2-9 epilogue (TMEM lane quadrant = warp % 4, two warps per quadrant: the requantisation is the
// CUDA-core work per output and bounds the kernel).
// =====================================================================================
constexpr int kDwTcTh = 16, kDwTcTw = 8;  // output tile (M = 128)
#ifndef FCM_I8TC_FAST
#define FCM_I8TC_FAST 0
#endif

// K-major operand, rows of xb = 32 / 64 / 128 bytes with the matching swizzle, 8-row groups SBO apart
__device__ __forceinline__ uint64_t desc_swz_sbo(uint32_t saddr, int xb, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(xb == 128 ? 2 : (xb == 64 ? 4 : 6)) << 61;
  return d;
}
__device__ __forceinline__ uint64_t desc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}

// 16 int32 accumulators of consecutive channels -> 4 packed int8 words: bias, requantisation (the
// mad.hi fast form when the shift is >= 33, else the 64-bit form; identical results), zero point,
// clamp. Constants from the staged per-channel arrays (broadcast loads: every lane reads the same
// channel).
__device__ __forceinline__ void epi16_i8_fast(const uint32_t* r, const EpiS& cs, const Epi& e, int n_base,
                                              uint32_t (&out)[4]) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint4 bq = lds128(cs.base + 4 * (n_base + 4 * w));
    const uint4 mq = lds128(cs.base + 4 * (cs.ncap + n_base + 4 * w));
    const uint4 sh = lds128(cs.base + 4 * (2 * cs.ncap + n_base + 4 * w));
    const int32_t b4[4] = {(int32_t)bq.x, (int32_t)bq.y, (int32_t)bq.z, (int32_t)bq.w};
    const int32_t m4[4] = {(int32_t)mq.x, (int32_t)mq.y, (int32_t)mq.z, (int32_t)mq.w};
    const int32_t s4[4] = {(int32_t)sh.x, (int32_t)sh.y, (int32_t)sh.z, (int32_t)sh.w};
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int32_t q = rq_apply(static_cast<int32_t>(r[4 * w + i]) + b4[i], make_rq(m4[i], s4[i]));
      word |= (static_cast<uint32_t>(min(max(q + e.zp_out, e.qmin), e.qmax)) & 0xFFu) << (8 * i);
    }
    out[w] = word;
  }
}

template <int K>
__global__ void __launch_bounds__(320, K == 3 ? 2 : 1)  // 2 CTAs per SM for 3x3 (smem, TMEM, registers)
    dw_tc_i8_kernel(const __grid_constant__ CUtensorMap tmx, const int8_t* __restrict__ wdw, Epi ep,
                    int8_t* __restrict__ y, int N, int C, int Ho, int Wo, int pt, int pl, int tiles_x, int tiles_y,
                    FDiv ftx, FDiv fty, int xb) {
  pdl_launch();
  constexpr int TH = kDwTcTh, TW = kDwTcTw;
  constexpr int THI = TH + K - 1, TWI = TW + K - 1;
  // X rows of xb bytes: 128-channel chunks, or the pixel's own 32 / 64 bytes when C is narrower
  // (the matching 32 / 64 / 128-byte swizzle on both the TMA box and the MMA descriptor)
  const int XB = (THI * TWI * xb + 1023) & ~1023;  // one X stage
  constexpr int BB = K * K * 4 * 1024;                   // diagonal weight blocks of the chunk
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* xs = smem;              // 2 x XB
  uint8_t* bs = xs + 2 * XB;       // BB
  uint8_t* cst = bs + BB;          // int8 epilogue constants of the chunk (128 channels)
  uint64_t* full = reinterpret_cast<uint64_t*>(cst + consts_bytes<FCM_S8>(128));
  uint64_t* empty = full + 2;
  uint64_t* tfull = empty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cbase = blockIdx.y * 128;
  const int cval = min(128, C - cbase);
  const int ng = (cval + 31) >> 5;  // 32-channel groups with weights (MMAs past them are skipped)
  // chunk constants and diagonal B blocks (weights are not produced by the previous kernel)
  Epi e2 = ep;
  if (e2.bias_q) e2.bias_q += cbase;
  e2.mult_q += cbase;
  e2.shift_q += cbase;
  const EpiS cs = stage_consts<FCM_S8>(e2, cval, 128, cst);
  for (int i = threadIdx.x; i < BB / 16; i += blockDim.x) sts128(smem_u32(bs) + 16 * i, 0, 0, 0, 0);
  __syncthreads();
  // B(tap, g)[n][k] = (n == k) ? w[tap][cbase + 32 g + n] : 0, K-major no-swizzle: 8-row x 16-byte
  // core matrices, LBO 128 (next 16 K bytes), SBO 256 (next 8 rows); 1 KB per (tap, group)
  for (int i = threadIdx.x; i < K * K * 128; i += blockDim.x) {
    const int t = i >> 7, c = i & 127, g = c >> 5, n = c & 31;
    const int8_t v = c < cval ? __ldg(wdw + (size_t)t * C + cbase + c) : int8_t(0);
    const uint32_t off = (t * 4 + g) * 1024 + (n >> 3) * 256 + (n >> 4) * 128 + (n & 7) * 16 + (n & 15);
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(smem_u32(bs) + off), "h"((unsigned short)(uint8_t)v) : "memory");
  }
  fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmx);
    for (int i = 0; i < 2; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_rt(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tbase = *tslot;
  const int total = N * tiles_y * tiles_x;
  auto decode = [&](int t, int& n, int& ty, int& tx) {
    const int q = fdiv(t, ftx);
    tx = t - q * tiles_x;
    n = fdiv(q, fty);
    ty = q - n * tiles_y;
  };
  if (warp == 0) {
    if (lane == 0) {
      Ring rs(2);
      for (int t = blockIdx.x; t < total; t += gridDim.x, rs.next()) {
        int n, ty, tx;
        decode(t, n, ty, tx);
        mbar_wait_sleep<128>(empty + rs.i, rs.ph ^ 1);
        mbar_arrive_expect_tx(full + rs.i, THI * TWI * xb);
        tma_load_4d(xs + rs.i * XB, &tmx, full + rs.i, cbase, tx * TW - pl, ty * TH - pt, n);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(TcKind<FCM_S8>::cf, TcKind<FCM_S8>::ab, 128, 32);
      const uint64_t b0 = desc_ns(smem_u32(bs), 128, 256);
      Ring rs(2), ra(2);
      for (int t = blockIdx.x; t < total; t += gridDim.x, rs.next(), ra.next()) {
        mbar_wait_sleep<128>(tempty + ra.i, ra.ph ^ 1);
        mbar_wait_sleep<64>(full + rs.i, rs.ph);
        tc_fence_after();
        const uint64_t a0 = desc_swz_sbo(smem_u32(xs + rs.i * XB), xb, TWI * xb);
        const uint32_t d = tbase + ra.i * 128;
        const uint32_t xr = (uint32_t)xb >> 4;  // one pixel row, in 16-byte descriptor units
#pragma unroll
        for (int tap = 0; tap < K * K; ++tap)
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if (g < ng)
              mma_ss<MmaKind::I8>(d + g * 32, a0 + (uint64_t)(((tap / K) * TWI + tap % K) * xr + g * 2),
                                  b0 + (uint64_t)(((tap * 4 + g) * 1024) >> 4), idesc, tap != 0);
        mma_commit(empty + rs.i);
        mma_commit(tfull + ra.i);
      }
    }
  } else {
    // epilogue (8 warps): lane = one output pixel (row m = 32 q + lane of the 16 x 8 tile); the two
    // warps of a TMEM lane quadrant take 64 channels each
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int m = q * 32 + lane;
    const int r = m >> 3, c = m & 7;
    Ring ra(2);
    for (int t = blockIdx.x; t < total; t += gridDim.x, ra.next()) {
      int n, ty, tx;
      decode(t, n, ty, tx);
      const int yo = ty * TH + r, xo = tx * TW + c;
      const bool ok = yo < Ho && xo < Wo;
      int8_t* dst = y + (((size_t)n * Ho + yo) * Wo + xo) * C + cbase;
      group_wait_sleep(tfull + ra.i, ra.ph, warp == 2, 1, 256);
      tc_fence_after();
      const uint32_t tq = tbase + ra.i * 128 + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c32 = half * 64; c32 < half * 64 + 64; c32 += 32) {
        if (c32 >= cval) break;
        uint32_t acc[32];
        tmem_ld32(tq + c32, acc);
        tmem_ld_wait();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#if FCM_I8TC_FAST
          uint32_t o[4];
          epi16_i8_fast(&acc[16 * hh], cs, ep, c32 + 16 * hh, o);
#else
          uint32_t o[8];
          epi16<FCM_S8>(&acc[16 * hh], cs, ep, c32 + 16 * hh, o);
#endif
          if (ok && c32 + 16 * hh < cval) stg128(dst + c32 + 16 * hh, o[0], o[1], o[2], o[3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + ra.i);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, 256);
  }
}

template <int K>
static int launch_dw_tc_i8_t(const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  constexpr int THI = kDwTcTh + K - 1, TWI = kDwTcTw + K - 1;
  const int xb = g.C <= 32 ? 32 : (g.C <= 64 ? 64 : 128);
  CUtensorMap tm;
  const uint64_t dims[4] = {(uint64_t)g.C, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N};
  const uint64_t str[3] = {(uint64_t)g.C, (uint64_t)g.W * g.C, (uint64_t)g.H * g.W * g.C};
  const uint32_t box[4] = {(uint32_t)xb, (uint32_t)TWI, (uint32_t)THI, 1u};
  const CUtensorMapSwizzle sw = xb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                          : (xb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  if (!encode_tmap(&tm, tmap_dtype(FCM_S8), 4, x, dims, str, box, sw))
    return set_error(FCM_E_CUDA, "tensor map (int8 tensor-core DW X) failed");
  const int tiles_x = (g.Wo + kDwTcTw - 1) / kDwTcTw, tiles_y = (g.Ho + kDwTcTh - 1) / kDwTcTh;
  const int spatial = g.N * tiles_x * tiles_y, nchunk = (g.C + 127) / 128;
  const int xst = (THI * TWI * xb + 1023) & ~1023;
  const size_t smem = 1024 + 2 * (size_t)xst + K * K * 4 * 1024 + consts_bytes<FCM_S8>(128) + 128;
  if (smem > (size_t)device_props().smem_optin) return set_error(FCM_E_INFEASIBLE, "int8 tensor-core DW: smem");
  const int per_sm = smem * 2 <= (size_t)device_props().smem_optin ? 2 : 1;  // TMEM: 256 columns per CTA
  const int gx = std::max(1, std::min(spatial, (device_props().sms * per_sm + nchunk - 1) / nchunk));
  auto kern = dw_tc_i8_kernel<K>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_k(kern, dim3(gx, nchunk), dim3(320), smem, st, tm, static_cast<const int8_t*>(wdw), ep,
           static_cast<int8_t*>(y), g.N, g.C, g.Ho, g.Wo, g.pt, g.pl, tiles_x, tiles_y, make_fdiv(tiles_x),
           make_fdiv(tiles_y), xb);
  return check_launch("dw_tc_i8_kernel");
}

int launch_dw_tc_i8(const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st) {
  if (g.s != 1 || g.C % 16 != 0) return set_error(FCM_E_UNSUPPORTED, "int8 tensor-core DW: stride 1, C % 16 == 0");
  if (g.k == 3) return launch_dw_tc_i8_t<3>(x, wdw, ep, y, g, st);
  if (g.k == 5) return launch_dw_tc_i8_t<5>(x, wdw, ep, y, g, st);
  return set_error(FCM_E_UNSUPPORTED, "int8 tensor-core DW: k in {3, 5}");
}

}  // namespace fcm
