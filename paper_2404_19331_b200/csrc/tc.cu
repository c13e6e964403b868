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

#include "common.cuh"
#include "host.h"

namespace fcm {

template <int DT> struct TcKind;
template <> struct TcKind<FCM_BF16> { static constexpr MmaKind kind = MmaKind::F16; static constexpr uint32_t cf = 1, ab = 1; };
template <> struct TcKind<FCM_F16> { static constexpr MmaKind kind = MmaKind::F16; static constexpr uint32_t cf = 1, ab = 0; };
template <> struct TcKind<FCM_S8> { static constexpr MmaKind kind = MmaKind::I8; static constexpr uint32_t cf = 2, ab = 1; };

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Epilogue of 16 accumulator columns of one output row -> packed storage words.
// Returns the number of 32-bit words written into out[] (16 / VEC).
template <int DT>
__device__ __forceinline__ void epi16(const uint32_t (&r)[16], const Epi& e, int n_base, int N, uint32_t (&out)[8]) {
  if constexpr (DT == FCM_S8) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int n = n_base + 4 * w + i;
        int32_t q = 0;
        if (n < N) {
          EpiC c{0.f, 0.f, e.bias_q ? __ldg(e.bias_q + n) : 0, __ldg(e.mult_q + n), __ldg(e.shift_q + n)};
          q = requant_i8(static_cast<int32_t>(r[4 * w + i]), c, e.zp_out, e.qmin, e.qmax);
        }
        word |= (static_cast<uint32_t>(q) & 0xFFu) << (8 * i);
      }
      out[w] = word;
    }
  } else {
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      float v[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int n = n_base + 2 * w + i;
        float sc = 1.f, bi = 0.f;
        if (n < N) {
          sc = e.scale ? __ldg(e.scale + n) : 1.f;
          bi = e.bias ? __ldg(e.bias + n) : 0.f;
        }
        v[i] = epi_f(__uint_as_float(r[2 * w + i]), sc, bi, e.act);
      }
      if constexpr (DT == FCM_BF16) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[0], v[1]);
        out[w] = *reinterpret_cast<uint32_t*>(&h);
      } else {
        __half2 h = __floats2half2_rn(v[0], v[1]);
        out[w] = *reinterpret_cast<uint32_t*>(&h);
      }
    }
  }
}

// Store the 16 outputs of columns [n_base, n_base+16) of row `row_ptr` (16-byte vectors,
// skipping vectors past N). N*ES is a multiple of 16 (validated).
template <int DT>
__device__ __forceinline__ void store16(uint8_t* row_ptr, const uint32_t (&o)[8], int n_base, int N) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int EPV = 16 / ES;  // elements per 16-byte vector
  constexpr int NV = 16 / EPV;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (n_base + v * EPV < N)
      *reinterpret_cast<uint4*>(row_ptr + (size_t)(n_base + v * EPV) * ES) =
          make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
  }
}

// =====================================================================================
// LBL PW: Y[M,N] = eps(X[M,K] . Wp[N,K]^T). Warps 0-3 epilogue, 4 TMA, 5 MMA.
// =====================================================================================
template <int DT>
__global__ void __launch_bounds__(192, 1)
    pw_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, Epi ep,
                 uint8_t* __restrict__ y, int M, int N, int K, int BN, int nbn, int stages, uint32_t tmem_cols) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  constexpr MmaKind KIND = TcKind<DT>::kind;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* abuf = smem;
  uint8_t* bbuf = smem + stages * 16384;
  uint64_t* full = reinterpret_cast<uint64_t*>(bbuf + stages * BN * 128);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmb);
    for (int s = 0; s < stages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 128); }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc_rt(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int nk = (K + KC - 1) / KC;
  const int nbm = (M + 127) / 128;
  const int total = nbm * nbn;
  const uint32_t stage_tx = 16384 + BN * 128;

  if (warp == 4) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m0 = (t / nbn) * 128, n0 = (t % nbn) * BN;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait(empty + s, ph ^ 1);
          mbar_arrive_expect_tx(full + s, stage_tx);
          tma_load_2d(abuf + s * 16384, &tma, full + s, kc * KC, m0);
          tma_load_2d(bbuf + s * BN * 128, &tmb, full + s, kc * KC, n0);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, BN);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(tempty + acc, ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + acc * BN;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          mbar_wait(full + s, (it / stages) & 1);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(abuf + s * 16384));
          const uint64_t bd = smem_desc_sw128(smem_u32(bbuf + s * BN * 128));
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ss<KIND>(d, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
          mma_commit(empty + s);
        }
        mma_commit(tfull + acc);
      }
    }
  } else {
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const int m0 = (t / nbn) * 128, n0 = (t % nbn) * BN;
      mbar_wait(tfull + acc, (local >> 1) & 1);
      tc_fence_after();
      const int row = m0 + warp * 32 + lane;
      uint8_t* rp = y + (size_t)row * N * ES;
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + acc * BN + c0, r);
        tmem_ld_wait();
        if (n0 + c0 < N && row < M) {
          uint32_t o[8];
          epi16<DT>(r, ep, n0 + c0, N, o);
          store16<DT>(rp, o, n0 + c0, N);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty + acc);
    }
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, tmem_cols);
  }
}

// =====================================================================================
// FCM DWPW. Warps 0-3 PW epilogue, 4..4+NDW-1 DW producers of the A operand (commBuffer),
// then one TMA warp and one MMA warp. One tile = nb x th x tw output pixels (<= 128 rows of
// the MMA) x one C_out slice of BN channels; the C_in (=K) dimension streams through in
// 128-byte chunks, so the intermediate "contains all channels" in time, not space.
// =====================================================================================
constexpr int kDwpwNDW = 8;

template <int DT, int K, int S>
__global__ void __launch_bounds__((4 + kDwpwNDW + 2) * 32, 1)
    dwpw_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
                   const typename Tr<DT>::T* __restrict__ wdw, Epi ed, Epi ep, uint8_t* __restrict__ y, int N,
                   int Cin, int Ho, int Wo, int Cout, int pt, int pl, int nb, int th, int tw, int tiles_x,
                   int tiles_y, int nsplit, int BN, int stages, uint32_t tmem_cols) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int V = Tr<DT>::VEC;
  constexpr int KC = 128 / ES;
  constexpr MmaKind KIND = TcKind<DT>::kind;
  constexpr int WARP_TMA = 4 + kDwpwNDW, WARP_MMA = 5 + kDwpwNDW;
  const int th_in = (th - 1) * S + K, tw_in = (tw - 1) * S + K;
  const int xbytes = nb * th_in * tw_in * 128;
  const int xstride = (xbytes + 1023) & ~1023;
  const int stage_bytes = xstride + 16384 + BN * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* afull = full + stages;
  uint64_t* empty = afull + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch_desc(&tmx);
    tma_prefetch_desc(&tmb);
    for (int s = 0; s < stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(afull + s, kDwpwNDW * 32);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 128); }
    fence_barrier_init();
  }
  if (warp == WARP_MMA) tmem_alloc_rt(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int nk = (Cin + KC - 1) / KC;
  const int spatial = ((N + nb - 1) / nb) * tiles_y * tiles_x;
  const int total = spatial * nsplit;

  if (warp == WARP_TMA) {
    if (lane == 0) {
      const uint32_t tx = xbytes + BN * 128;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int ns = t % nsplit;
        int sp = t / nsplit;
        const int txi = sp % tiles_x;
        sp /= tiles_x;
        const int tyi = sp % tiles_y;
        const int nbi = sp / tiles_y;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          mbar_wait(empty + s, ((it / stages) & 1) ^ 1);
          uint8_t* st = smem + s * stage_bytes;
          mbar_arrive_expect_tx(full + s, tx);
          tma_load_4d(st, &tmx, full + s, kc * KC, txi * tw * S - pl, tyi * th * S - pt, nbi * nb);
          tma_load_2d(st + xstride + 16384, &tmb, full + s, kc * KC, ns * BN);
        }
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, BN);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(tempty + acc, ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + acc * BN;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait(full + s, ph);
          mbar_wait(afull + s, ph);
          tc_fence_after();
          uint8_t* st = smem + s * stage_bytes;
          const uint64_t ad = smem_desc_sw128(smem_u32(st + xstride));
          const uint64_t bd = smem_desc_sw128(smem_u32(st + xstride + 16384));
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ss<KIND>(d, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
          mma_commit(empty + s);
        }
        mma_commit(tfull + acc);
      }
    }
  } else if (warp >= 4) {
    // ---------------- DW warps: X halo chunk (smem) -> DW -> eps_dw -> A operand (commBuffer)
    const int dw = warp - 4;
    const int ncols = nb * tw;
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = it % stages;
        const int c = kc * KC + lane * V;
        DwW<DT, K> W;
        load_dw_weights<DT, K>(W, wdw, Cin, c);
        EpiC ec[V];
#pragma unroll
        for (int v = 0; v < V; ++v) ec[v] = load_epi<DT>(ed, c + v, c + v < Cin);
        mbar_wait(full + s, (it / stages) & 1);
        uint8_t* st = smem + s * stage_bytes;
        const uint32_t* xs = reinterpret_cast<const uint32_t*>(st);
        uint8_t* abase = st + xstride;
        for (int col = dw; col < ncols; col += kDwpwNDW) {
          const int b = col / tw, x = col - b * tw;
          const uint32_t* src = xs + ((b * th_in) * tw_in + x * S) * 32 + lane;
          dw_column<DT, K, S>(src, 32, tw_in * 32, th, W, [&](int yy, const typename Tr<DT>::acc_t(&a)[V]) {
            const int m = (b * th + yy) * tw + x;
            const uint32_t word = (c < Cin) ? epi_pack<DT>(a, ec, ed) : 0u;
            *reinterpret_cast<uint32_t*>(abase + sw128_off(m, lane)) = word;
          });
        }
        fence_proxy_async_smem();
        mbar_arrive(afull + s);
      }
    }
  } else {
    // ---------------- epilogue warps 0-3: TMEM -> eps_pw -> OFM
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const int ns = t % nsplit;
      int sp = t / nsplit;
      const int txi = sp % tiles_x;
      sp /= tiles_x;
      const int tyi = sp % tiles_y;
      const int nbi = sp / tiles_y;
      const int m = warp * 32 + lane;
      const int b = m / (th * tw), r = m - b * th * tw;
      const int yy = r / tw, xx = r - yy * tw;
      const int n = nbi * nb + b, yo = tyi * th + yy, xo = txi * tw + xx;
      const bool valid = (b < nb) && (n < N) && (yo < Ho) && (xo < Wo);
      uint8_t* rp = y + (((size_t)n * Ho + yo) * Wo + xo) * Cout * ES;
      const int n0 = ns * BN;
      mbar_wait(tfull + acc, (local >> 1) & 1);
      tc_fence_after();
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t rr[16];
        tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + acc * BN + c0, rr);
        tmem_ld_wait();
        if (valid && n0 + c0 < Cout) {
          uint32_t o[8];
          epi16<DT>(rr, ep, n0 + c0, Cout, o);
          store16<DT>(rp, o, n0 + c0, Cout);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty + acc);
    }
  }
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, tmem_cols);
  }
}

// =====================================================================================
// FCM PWDW_R. Warps 0-7: PW epilogue into the smem T tile, then DW from it; warp 8 TMA,
// warp 9 MMA. One tile = DW output tile (nb x th x tw) x TD intermediate channels (one
// 128-byte group). The PW runs over the tile's T HALO (R = nb*th_in*tw_in <= 256 rows,
// 1-2 M=128 MMAs): T pixels in the overlap are recomputed by every tile that needs them
// (the "_R"). T outside the image is written as 0 (DW pads T, reading R6).
// =====================================================================================
template <int DT, int K, int S>
__global__ void __launch_bounds__(320, 1)
    pwdw_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
                   const typename Tr<DT>::T* __restrict__ wdw, Epi ep, Epi ed, uint8_t* __restrict__ y, int N, int H,
                   int W, int Cin, int Ho, int Wo, int Cmid, int pt, int pl, int nb, int th, int tw, int tiles_x,
                   int tiles_y, int stages, uint32_t tmem_cols) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int V = Tr<DT>::VEC;
  constexpr int KC = 128 / ES;
  constexpr int TD = 128 / ES;           // intermediate channels per tile
  constexpr int PITCH = 128 + 16;        // bytes per T row in smem (padded: conflict-free)
  constexpr MmaKind KIND = TcKind<DT>::kind;
  const int th_in = (th - 1) * S + K, tw_in = (tw - 1) * S + K;
  const int R = nb * th_in * tw_in;
  const int MB = (R + 127) / 128;
  const int xbytes = R * 128;
  const int astride = MB * 16384;
  const int stage_bytes = astride + TD * 128;
  const int tbytes = ((R * PITCH) + 1023) & ~1023;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* tsm = smem + stages * stage_bytes;  // 2 T buffers
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + 2 * tbytes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmx);
    tma_prefetch_desc(&tmb);
    for (int s = 0; s < stages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 256); }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc_rt(tslot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int nk = (Cin + KC - 1) / KC;
  const int nslice = (Cmid + TD - 1) / TD;
  const int spatial = ((N + nb - 1) / nb) * tiles_y * tiles_x;
  const int total = spatial * nslice;
  const uint32_t acc_cols = MB * TD;

  auto decode = [&](int t, int& sl, int& nbi, int& tyi, int& txi) {
    sl = t % nslice;
    int sp = t / nslice;
    txi = sp % tiles_x;
    sp /= tiles_x;
    tyi = sp % tiles_y;
    nbi = sp / tiles_y;
  };

  if (warp == 8) {
    if (lane == 0) {
      const uint32_t tx = xbytes + TD * 128;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int sl, nbi, tyi, txi;
        decode(t, sl, nbi, tyi, txi);
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          mbar_wait(empty + s, ((it / stages) & 1) ^ 1);
          uint8_t* st = smem + s * stage_bytes;
          mbar_arrive_expect_tx(full + s, tx);
          tma_load_4d(st, &tmx, full + s, kc * KC, txi * tw * S - pl, tyi * th * S - pt, nbi * nb);
          tma_load_2d(st + astride, &tmb, full + s, kc * KC, sl * TD);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(TcKind<DT>::cf, TcKind<DT>::ab, 128, TD);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(tempty + acc, ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % stages;
          mbar_wait(full + s, (it / stages) & 1);
          tc_fence_after();
          uint8_t* st = smem + s * stage_bytes;
          const uint64_t bd = smem_desc_sw128(smem_u32(st + astride));
          for (int mb = 0; mb < MB; ++mb) {
            const uint64_t ad = smem_desc_sw128(smem_u32(st + mb * 16384));
            const uint32_t d = tbase + acc * acc_cols + mb * TD;
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_ss<KIND>(d, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
          }
          mma_commit(empty + s);
        }
        mma_commit(tfull + acc);
      }
    }
  } else {
    const int q = warp & 3, mbw = warp >> 2;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      int sl, nbi, tyi, txi;
      decode(t, sl, nbi, tyi, txi);
      uint8_t* tb = tsm + acc * tbytes;
      // ---- phase 1: TMEM (PW accumulators over the halo) -> eps_pw -> T tile (zero outside image)
      mbar_wait(tfull + acc, (local >> 1) & 1);
      tc_fence_after();
      if (mbw < MB) {
        const int r = mbw * 128 + q * 32 + lane;
        const int b = r / (th_in * tw_in), rr = r - b * th_in * tw_in;
        const int yi = tyi * th * S - pt + rr / tw_in, xi = txi * tw * S - pl + rr % tw_in;
        const int n = nbi * nb + b;
        const bool inside = (r < R) && (n < N) && (yi >= 0) && (yi < H) && (xi >= 0) && (xi < W);
        for (int c0 = 0; c0 < TD; c0 += 16) {
          uint32_t rg[16];
          tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + acc * acc_cols + mbw * TD + c0, rg);
          tmem_ld_wait();
          if (r < R) {
            uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (inside) epi16<DT>(rg, ep, sl * TD + c0, Cmid, o);
            uint8_t* dst = tb + r * PITCH + c0 * ES;
            constexpr int NV = 16 * ES / 16;
#pragma unroll
            for (int v = 0; v < NV; ++v)
              *reinterpret_cast<uint4*>(dst + 16 * v) = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty + acc);
      named_bar_sync(1, 256);
      // ---- phase 2: DW over the T tile -> eps_dw -> OFM
      const int c = sl * TD + lane * V;
      DwW<DT, K> Wd;
      load_dw_weights<DT, K>(Wd, wdw, Cmid, c);
      EpiC ec[V];
#pragma unroll
      for (int v = 0; v < V; ++v) ec[v] = load_epi<DT>(ed, c + v, c + v < Cmid);
      const uint32_t* tw32 = reinterpret_cast<const uint32_t*>(tb);
      constexpr int PW = PITCH / 4;
      uint32_t* yw = reinterpret_cast<uint32_t*>(y);
      for (int col = warp; col < nb * tw; col += 8) {
        const int b = col / tw, x = col - b * tw;
        const int n = nbi * nb + b, xo = txi * tw + x;
        if (n >= N || xo >= Wo) continue;
        const int y0 = tyi * th;
        const int nrows = min(th, Ho - y0);
        const uint32_t* src = tw32 + ((b * th_in) * tw_in + x * S) * PW + lane;
        dw_column<DT, K, S>(src, PW, tw_in * PW, nrows, Wd, [&](int yy, const typename Tr<DT>::acc_t(&a)[V]) {
          if (c < Cmid) {
            const size_t pix = ((size_t)n * Ho + (y0 + yy)) * Wo + xo;
            yw[(pix * Cmid + c) / V] = epi_pack<DT>(a, ec, ed);
          }
        });
      }
    }
  }
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc_rt(tbase, tmem_cols);
  }
}

// ------------------------------------------------------------------------------- launchers
static uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}
static inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

template <int DT>
static int launch_pw_t(const void* x, const void* wp, const Epi& ep, void* y, int M, int K, int N, cudaStream_t st) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  const int nbn = (N + 255) / 256;
  const int BN = round_up((N + nbn - 1) / nbn, 16);
  CUtensorMap ta, tb;
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
  const int stage_bytes = 16384 + BN * 128;
  const int budget = device_props().smem_optin - 2048;
  int stages = std::min(8, budget / stage_bytes);
  if (stages < 2) return set_error(FCM_E_INFEASIBLE, "pw: not enough shared memory for 2 stages");
  const size_t smem = 1024 + (size_t)stages * stage_bytes + (2 * stages + 4) * 8 + 16;
  auto kern = pw_tc_kernel<DT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int total = ((M + 127) / 128) * nbn;
  const int grid = std::min(total, device_props().sms);
  kern<<<grid, 192, smem, st>>>(ta, tb, ep, static_cast<uint8_t*>(y), M, N, K, BN, nbn, stages, pow2_cols(2 * BN));
  return check_launch("pw_tc_kernel");
}

int launch_pw_tc(int dt, const void* x, const void* wp, const Epi& ep, void* y, int M, int K, int N, cudaStream_t st) {
  switch (dt) {
    case FCM_BF16: return launch_pw_t<FCM_BF16>(x, wp, ep, y, M, K, N, st);
    case FCM_F16: return launch_pw_t<FCM_F16>(x, wp, ep, y, M, K, N, st);
    case FCM_S8: return launch_pw_t<FCM_S8>(x, wp, ep, y, M, K, N, st);
  }
  return set_error(FCM_E_UNSUPPORTED, "pw tensor-core path: dtype");
}

template <int DT, int K, int S>
static int launch_dwpw_t(const void* x, const void* wdw, const Epi& ed, const void* wp, const Epi& ep, void* y,
                         const Geo& g, int nsplit, cudaStream_t st) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  const int th_in = (g.th - 1) * S + K, tw_in = (g.tw - 1) * S + K;
  if (g.nb * g.th * g.tw > 128) return set_error(FCM_E_INFEASIBLE, "dwpw: tile has more than 128 pixels");
  if (th_in > 256 || tw_in > 256 || g.nb > 256) return set_error(FCM_E_INFEASIBLE, "dwpw: halo box > 256");
  if (nsplit <= 0) nsplit = (g.Cout + 255) / 256;
  const int BN = round_up((g.Cout + nsplit - 1) / nsplit, 16);
  if (BN > 256) return set_error(FCM_E_INFEASIBLE, "dwpw: C_out slice > 256 (raise n_split)");
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
  const int xbytes = g.nb * th_in * tw_in * 128;
  const int stage_bytes = ((xbytes + 1023) & ~1023) + 16384 + BN * 128;
  const int budget = device_props().smem_optin - 2048;
  const int stages = std::min(4, budget / stage_bytes);
  if (stages < 2) return set_error(FCM_E_INFEASIBLE, "dwpw: tile too large for 2 smem stages");
  const size_t smem = 1024 + (size_t)stages * stage_bytes + (3 * stages + 4) * 8 + 16;
  auto kern = dwpw_tc_kernel<DT, K, S>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles_x = (g.Wo + g.tw - 1) / g.tw, tiles_y = (g.Ho + g.th - 1) / g.th;
  const int total = ((g.N + g.nb - 1) / g.nb) * tiles_x * tiles_y * nsplit;
  const int grid = std::min(total, device_props().sms);
  using TT = typename Tr<DT>::T;
  kern<<<grid, (4 + kDwpwNDW + 2) * 32, smem, st>>>(tx, tb, static_cast<const TT*>(wdw), ed, ep,
                                                     static_cast<uint8_t*>(y), g.N, g.C, g.Ho, g.Wo, g.Cout, g.pt,
                                                     g.pl, g.nb, g.th, g.tw, tiles_x, tiles_y, nsplit, BN, stages,
                                                     pow2_cols(2 * BN));
  return check_launch("dwpw_tc_kernel");
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
    case FCM_BF16: return launch_dwpw_dt<FCM_BF16>(x, wdw, ed, wp, ep, y, g, ns, st);
    case FCM_F16: return launch_dwpw_dt<FCM_F16>(x, wdw, ed, wp, ep, y, g, ns, st);
    case FCM_S8: return launch_dwpw_dt<FCM_S8>(x, wdw, ed, wp, ep, y, g, ns, st);
  }
  return set_error(FCM_E_UNSUPPORTED, "dwpw tensor-core path: dtype");
}

template <int DT, int K, int S>
static int launch_pwdw_t(const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                         const Geo& g, cudaStream_t st) {
  constexpr int ES = Tr<DT>::ES;
  constexpr int KC = 128 / ES;
  constexpr int TD = 128 / ES;
  const int th_in = (g.th - 1) * S + K, tw_in = (g.tw - 1) * S + K;
  const int R = g.nb * th_in * tw_in;
  if (R > 256) return set_error(FCM_E_INFEASIBLE, "pwdw_r: halo tile has more than 256 pixels");
  const int MB = (R + 127) / 128;
  CUtensorMap tx, tb;
  {
    const uint64_t dims[4] = {(uint64_t)g.C, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N};
    const uint64_t str[3] = {(uint64_t)g.C * ES, (uint64_t)g.W * g.C * ES, (uint64_t)g.H * g.W * g.C * ES};
    const uint32_t box[4] = {(uint32_t)KC, (uint32_t)tw_in, (uint32_t)th_in, (uint32_t)g.nb};
    if (!encode_tmap(&tx, tmap_dtype(DT), 4, x, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PWDW X) failed");
  }
  {
    const uint64_t dims[2] = {(uint64_t)g.C, (uint64_t)g.Cout};
    const uint64_t str[1] = {(uint64_t)g.C * ES};
    const uint32_t box[2] = {(uint32_t)KC, (uint32_t)TD};
    if (!encode_tmap(&tb, tmap_dtype(DT), 2, wp, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return set_error(FCM_E_CUDA, "tensor map (PWDW B) failed");
  }
  const int stage_bytes = MB * 16384 + TD * 128;
  const int tbytes = ((R * (128 + 16)) + 1023) & ~1023;
  const int budget = device_props().smem_optin - 2048 - 2 * tbytes;
  const int stages = std::min(4, budget / stage_bytes);
  if (stages < 2) return set_error(FCM_E_INFEASIBLE, "pwdw_r: tile too large for 2 smem stages");
  const size_t smem = 1024 + (size_t)stages * stage_bytes + 2 * tbytes + (2 * stages + 4) * 8 + 16;
  auto kern = pwdw_tc_kernel<DT, K, S>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles_x = (g.Wo + g.tw - 1) / g.tw, tiles_y = (g.Ho + g.th - 1) / g.th;
  const int total = ((g.N + g.nb - 1) / g.nb) * tiles_x * tiles_y * ((g.Cout + TD - 1) / TD);
  const int grid = std::min(total, device_props().sms);
  using TT = typename Tr<DT>::T;
  kern<<<grid, 320, smem, st>>>(tx, tb, static_cast<const TT*>(wdw), ep, ed, static_cast<uint8_t*>(y), g.N, g.H, g.W,
                                g.C, g.Ho, g.Wo, g.Cout, g.pt, g.pl, g.nb, g.th, g.tw, tiles_x, tiles_y, stages,
                                pow2_cols(2 * MB * TD));
  return check_launch("pwdw_tc_kernel");
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

}  // namespace fcm
