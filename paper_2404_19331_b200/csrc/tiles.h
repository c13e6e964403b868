// Default output-tile choice per kernel family (used when the caller passes no fcm_tile and by
// the planner's candidate grid). Host-only.
#pragma once
#include <algorithm>

#include "host.h"

namespace fcm {

inline int halo(int t, int k, int s) { return (t - 1) * s + k; }

// Column block width of the tensor-core PW stage: one block when N <= 256 (padded to the MMA
// granule of 16; the TMA store clips the tail), otherwise a multiple of the 128-byte store chunk
// (cpc columns) so that blocks never overlap. nb_out = number of blocks.
inline int pick_bn(int N, int nsplit, int cpc, int& nb_out) {
  if (nsplit <= 0) nsplit = (N + 255) / 256;
  int bn = (nsplit == 1) ? (N + 15) / 16 * 16 : ((N + nsplit - 1) / nsplit + cpc - 1) / cpc * cpc;
  bn = std::min(bn, 256);
  nb_out = (N + bn - 1) / bn;
  return bn;
}

// LBL DW: one 128-byte channel group x th x tw outputs per CTA.
inline void default_dw_tile(Geo& g, int es = 0) {
  // 8 x 16 (s1) / 4 x 16 (s2) output pixels of one 128-byte channel group; a narrower pixel
  // (C * es < 128 B, staged at its own width) gets proportionally more pixels per CTA
  const int pb = es > 0 ? std::min(128, g.C * es) : 128;
  const int f = std::max(1, 128 / std::max(pb, 1));
  const int fh = f >= 4 ? 2 : 1, fw = f / fh >= 2 ? 2 : 1;
  g.th = std::min((g.s == 1 ? 8 : 4) * fh, g.Ho);
  g.tw = std::min(16 * fw, g.Wo);
  g.nb = 1;
}

// Cost of one DWPW tiling: DW rows computed (incl. ragged edges) + half the staged halo + a
// fixed per-tile (per C_in-chunk phase) overhead, all x number of tiles. The overhead constant
// (96 pixel-equivalents) reflects the measured hand-off cost of a phase on B200 (~800 cycles vs
// ~1000 cycles of DW work per 128 pixels x 64 channels).
inline long dwpw_tile_cost(const Geo& g, int nb, int th, int tw) {
  const int th_in = halo(th, g.k, g.s), tw_in = halo(tw, g.k, g.s);
  const long tiles = (long)((g.N + nb - 1) / nb) * ((g.Ho + th - 1) / th) * ((g.Wo + tw - 1) / tw);
  return tiles * (2L * nb * th * tw + (long)nb * th_in * tw_in + 96);
}

// Largest DWPW tile (MMA rows): 256 (two M=128 blocks) for the bf16/f16 3x3 pair core when
// 2 x 2 x C_out fits the 512 TMEM columns, else 128.
inline bool dwpw_pair_dt(int dt, const Geo& g) { return (dt == FCM_BF16 || dt == FCM_F16) && g.k == 3; }
inline int dwpw_mmax(int dt, const Geo& g) { return (dwpw_pair_dt(dt, g) && g.Cout <= 128) ? 256 : 128; }

inline bool dwpw_tile_ok(const Geo& g, int nb, int th, int tw, int mmax = 128) {
  const int th_in = halo(th, g.k, g.s), tw_in = halo(tw, g.k, g.s);
  if (nb * th * tw > mmax || th_in > 256 || tw_in > 256) return false;
  // mirror of launch_dwpw_t's layout: A ring 2 x (8 chunks x (rows x 16 B + 16)) + B ring
  // 2 x BN x 128 + constants / DW weights (<= 40K) + at least 2 X stages
  const int mb = (nb * th * tw + 127) / 128;
  const int aslot = ((8 * (16 * 128 * mb + 16)) + 1023) & ~1023;
  const int bn = std::min(256, (g.Cout + 15) / 16 * 16);
  const int xstride = ((nb * th_in * tw_in * 128) + 1023) & ~1023;
  return 1024 + 2 * aslot + 2 * bn * 128 + 40960 + 1536 + 2 * xstride <= 232448;
}

// Pair-core (bf16/f16 3x3) DWPW tile time in "DW row" units: a C_in-chunk phase costs the
// slowest DW warp's rows (rounds x (SEG + 2) over 8 warps, best SEG of 8/7/4) plus ~10 rows of
// hand-off; tiles run in waves of #SMs.
inline long dwpw_pair_cost(const Geo& g, int nb, int th, int tw, int sms = 148) {
  const long tiles = (long)((g.N + nb - 1) / nb) * ((g.Ho + th - 1) / th) * ((g.Wo + tw - 1) / tw);
  const int hp = (tw + 1) / 2;
  long best = -1;
  for (int seg = std::min(th, 32); seg >= 1; --seg) {
    const int items = nb * hp * ((th + seg - 1) / seg);
    const long t = (long)((items + 7) / 8) * ((seg - 1) * g.s + 3 + 2);
    if (best < 0 || t < best) best = t;
  }
  const int halo_px = nb * halo(th, g.k, g.s) * halo(tw, g.k, g.s);  // TMA / smem fill of the halo tile
  return ((tiles + sms - 1) / sms) * (best + 10 + halo_px / 64);
}

inline void default_dwpw_tile(Geo& g, int mmax = 128, bool pair = false) {
  long best = -1;
  int bn = 1, bh = 1, bw = 1;
  for (int tw = 1; tw <= std::min(g.Wo, 64); ++tw)
    for (int th = 1; th <= std::min(g.Ho, mmax / tw); ++th) {
      const int nbmax = (th == g.Ho && tw == g.Wo) ? std::max(1, std::min(g.N, mmax / (th * tw))) : 1;
      for (int nb = 1; nb <= nbmax; ++nb) {
        if (!dwpw_tile_ok(g, nb, th, tw, mmax)) continue;
        if (pair && tw < std::min(4, g.Wo)) continue;  // thin columns: halo re-reads dominate
        const long c = pair ? dwpw_pair_cost(g, nb, th, tw) : dwpw_tile_cost(g, nb, th, tw);
        if (best < 0 || c < best) { best = c; bn = nb; bh = th; bw = tw; }
      }
    }
  g.nb = bn; g.th = bh; g.tw = bw;
}

// PWDW_R: halo tile R = nb*th_in*tw_in <= 256 rows (two M=128 MMAs). Cost = PW rows computed
// (incl. recomputed halo) + DW rows + per-tile overhead.
inline long pwdw_tile_cost(const Geo& g, int nb, int th, int tw) {
  const int th_in = halo(th, g.k, g.s), tw_in = halo(tw, g.k, g.s);
  const long tiles = (long)((g.N + nb - 1) / nb) * ((g.Ho + th - 1) / th) * ((g.Wo + tw - 1) / tw);
  return tiles * ((long)nb * th_in * tw_in + nb * th * tw + 32);
}

// rmax: MMA rows of the halo tile the default / planner tiles use (the kernel takes up to 512 for
// bf16 / f16: 4 row blocks x 64 T columns x 2 TMEM buffers; measured plans search those)
inline bool pwdw_tile_ok(const Geo& g, int nb, int th, int tw, int rmax = 256) {
  const int th_in = halo(th, g.k, g.s), tw_in = halo(tw, g.k, g.s);
  return nb * th_in * tw_in <= rmax && th_in <= 256 && tw_in <= 256;
}

// Shared memory of the tensor-core PWDW_R kernel at its minimum configuration (2 X/B stages, 2 T
// buffers, non-resident B), as its launcher computes it: fixed part = barriers + PW/DW epilogue
// constants for all C_mid + DW weights of all C_mid slices (grows with C_mid).
inline bool pwdw_smem_fits(int dt, const Geo& g, int smem_optin = 232448) {
  const int es = dt == FCM_F32 ? 4 : (dt == FCM_S8 ? 1 : 2);
  const int td = 128 / es;
  const int r = g.nb * halo(g.th, g.k, g.s) * halo(g.tw, g.k, g.s);
  const long mb = (r + 127) / 128, tbytes = ((long)r * 144 + 1023) / 1024 * 1024;
  const long ncap = (long)(g.Cout + td - 1) / td * td, nslice = ncap / td;
  const long consts = (dt == FCM_S8 ? 12 : 8) * ncap;
  const bool pair = (dt == FCM_BF16 || dt == FCM_F16) && g.k == 3;
  const long wbytes = pair ? 52 * nslice * 32 : (long)g.k * g.k * nslice * 128;  // dw3h_bytes
  const long fixed = 1024 + 2 * consts + wbytes + 512;
  const long xb = (long)g.C * es <= 32 ? 32 : ((long)g.C * es <= 64 ? 64 : 128);  // X box bytes / pixel
  return 2 * mb * td <= 512 && fixed + 2 * tbytes + 2 * (mb * 128 * xb + td * 128) <= smem_optin;
}

inline void default_pwdw_tile(Geo& g) {
  long best = -1;
  int bn = 1, bh = 1, bw = 1;
  for (int tw = 1; tw <= std::min(g.Wo, 64); ++tw)
    for (int th = 1; th <= std::min(g.Ho, 64); ++th) {
      const int nbmax = (th == g.Ho && tw == g.Wo) ? std::max(1, g.N) : 1;
      for (int nb = 1; nb <= nbmax; ++nb) {
        if (!pwdw_tile_ok(g, nb, th, tw)) break;
        const long c = pwdw_tile_cost(g, nb, th, tw);
        if (best < 0 || c < best) { best = c; bn = nb; bh = th; bw = tw; }
      }
    }
  g.nb = bn; g.th = bh; g.tw = bw;
}

}  // namespace fcm
