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
inline void default_dw_tile(Geo& g) {
  g.th = std::min(g.s == 1 ? 8 : 4, g.Ho);
  g.tw = std::min(16, g.Wo);
  g.nb = 1;
}

// Cost of one DWPW tiling: DW rows computed (incl. ragged edges) + half the staged halo + a
// fixed per-tile overhead, all x number of tiles. Candidates respect M <= 128, box <= 256 and a
// 2-stage smem budget.
inline long dwpw_tile_cost(const Geo& g, int nb, int th, int tw) {
  const int th_in = halo(th, g.k, g.s), tw_in = halo(tw, g.k, g.s);
  const long tiles = (long)((g.N + nb - 1) / nb) * ((g.Ho + th - 1) / th) * ((g.Wo + tw - 1) / tw);
  return tiles * (2L * nb * th * tw + (long)nb * th_in * tw_in + 32);
}

inline bool dwpw_tile_ok(const Geo& g, int nb, int th, int tw) {
  const int th_in = halo(th, g.k, g.s), tw_in = halo(tw, g.k, g.s);
  if (nb * th * tw > 128 || th_in > 256 || tw_in > 256) return false;
  // mirror of launch_dwpw_t's layout: staging 32K + A ring 2x16K + B ring 2x(BN<=256)x128
  // + constants / DW weights (<= 24K) + at least 2 X stages
  const int xstride = ((nb * th_in * tw_in * 128) + 1023) & ~1023;
  return 1024 + 32768 + 2 * 16384 + 2 * 256 * 128 + 24576 + 1536 + 2 * xstride <= 232448;
}

inline void default_dwpw_tile(Geo& g) {
  long best = -1;
  int bn = 1, bh = 1, bw = 1;
  for (int tw = 1; tw <= std::min(g.Wo, 64); ++tw)
    for (int th = 1; th <= std::min(g.Ho, 128 / tw); ++th) {
      const int nbmax = (th == g.Ho && tw == g.Wo) ? std::max(1, std::min(g.N, 128 / (th * tw))) : 1;
      for (int nb = 1; nb <= nbmax; ++nb) {
        if (!dwpw_tile_ok(g, nb, th, tw)) continue;
        const long c = dwpw_tile_cost(g, nb, th, tw);
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

inline bool pwdw_tile_ok(const Geo& g, int nb, int th, int tw) {
  const int th_in = halo(th, g.k, g.s), tw_in = halo(tw, g.k, g.s);
  return nb * th_in * tw_in <= 256 && th_in <= 256 && tw_in <= 256;
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
