// FusePlanner (fcm_plan): PAPER.md §IV re-derived for B200. Host-only.
//
// Two modes:
//  "paper"  the paper's estimators verbatim -- Eq. 1 Overlap, Eq. 2 PwGMA, Eq. 3 DwGMA, Eq. 4
//           PwDwGMA and the DWPW equation constructed "similarly" -- minimised over a
//           tile grid under the paper's two constraints (tiles fit on chip, #OFM tiles >= #SMs),
//           fuse iff the FCM minimum is LESS than the LBL minima. Grid and readings:
//           DESIGN.md §6 (R13-R22); mirrored exactly by oracle/planner.py.
//  "b200"   (default) the kernels this library actually runs: each layer / pair is costed with
//           the tile the kernel would use, as predicted time = max(HBM bytes / BW, L2->SM bytes /
//           BW, DW MACs / DW rate, PW MACs / tensor rate) + launch overhead. HBM bytes are the
//           compulsory bytes (the intermediate of an FCM is never counted); L2->SM bytes come from
//           the exact unit enumeration (oracle/counting.py *_units). Fuse iff strictly faster.
// A chain DP then picks non-overlapping fusions, later fusion winning exact ties.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "fcm.h"
#include "host.h"
#include "json.h"
#include "tiles.h"

namespace fcm {
namespace plan {

using json::Value;
typedef long long ll;

static ll cdiv(ll a, ll b) { return (a + b - 1) / b; }

struct Layer {
  std::string id, kind;
  ll H, W, C, Cout, k = 1, s = 1, pt = 0, pl = 0, pb = 0, pr = 0, Ho, Wo;
  ll res = 0;        // 1: the output epilogue adds a residual (shortcut) of the output's shape
  ll extra_out = 0;  // consumers outside the edge list (a residual shortcut reads this output)
};

struct Gpu {
  ll sms = 148, smem = 232448, l2 = 126LL << 20;
  // calibrated on B200 against the measured per-launch times of the MobileNetV2 bf16 b256 plan
  // (profiles/r02/layers.json, tests/test_planner_time_model.py): the kernels reach ~0.5 of the HBM
  // peak on their compulsory bytes, the bf16 DW stage ~0.16 of the FFMA peak, each PWDW_R T value
  // (PW output over the halo: TMEM -> epilogue -> smem) costs about 2 DW MACs, ~8 us per launch
  double hbm_gbs = 6534.5, l2_gbs = 20000, tc_tmacs = 832, ffma_tmacs = 37.2, dw_eff = 0.16, launch_us = 8.0;
  double hbm_eff = 0.5, t_cost = 2.0;
  // int8 DW efficiency (of the FFMA peak), measured on B200: LBL FFMA2 core ~0.17, inside the fused
  // kernels ~0.085 (profiles/r01_ncu_summary.md)
  double dw_eff_i8 = 0.17, dw_eff_i8_fused = 0.085;
};

// ---------------------------------------------------------------------------- Eq. 1-4 (verbatim)
static ll overlap(ll ch, ll cw, ll th, ll tw, ll fh, ll fw, ll s) {
  return (cdiv(cw, tw) - 1) * std::max(fw - s, 0LL) * ch + (cdiv(ch, th) - 1) * std::max(fh - s, 0LL) * cw;
}

static std::vector<ll> cand(ll n) {
  std::set<ll> c = {1, 2, 4, 8, 16, 32, 64, n};
  for (ll d = 1; d <= std::min(n, 64LL); ++d)
    if (n % d == 0) c.insert(d);
  std::vector<ll> r;
  for (ll v : c)
    if (v >= 1 && v <= n) r.push_back(v);
  return r;
}

static std::vector<ll> dcand(ll d) {
  std::set<ll> c = {d};
  for (ll v = 32; v <= d; v += 32) c.insert(v);
  return std::vector<ll>(c.begin(), c.end());
}

struct Best {
  bool ok = false;
  ll gma = 0, th = 0, tw = 0, td = 0;
  std::string kind;
};

static Best paper_dw(const Layer& l, ll N, ll b, const Gpu& g, ll min_tiles) {
  Best best;
  for (ll td : dcand(l.C))
    for (ll th : cand(l.Ho))
      for (ll tw : cand(l.Wo)) {
        if ((th * tw * td) % 32) continue;
        if (N * cdiv(l.Ho, th) * cdiv(l.Wo, tw) * cdiv(l.C, td) < min_tiles) continue;
        const ll thi = std::min((th - 1) * l.s + l.k, l.H), twi = std::min((tw - 1) * l.s + l.k, l.W);
        if ((thi * twi * td + th * tw * td + l.k * l.k * td) * b > g.smem) continue;
        const ll ov = overlap(l.H, l.W, th * l.s, tw * l.s, l.k, l.k, l.s);
        const ll gma = 2 * l.C * N * ov + N * l.H * l.W * l.C + N * l.Ho * l.Wo * l.C +
                       cdiv(N * l.Ho * l.Wo, th * tw) * l.k * l.k * l.C;
        if (!best.ok || gma < best.gma) best = {true, gma, th, tw, td, "dw"};
      }
  return best;
}

static Best paper_pw(const Layer& l, ll N, ll b, const Gpu& g, ll min_tiles) {
  Best best;
  for (ll td : dcand(l.Cout))
    for (ll th : cand(l.H))
      for (ll tw : cand(l.W)) {
        if ((th * tw * td) % 32) continue;
        if (N * cdiv(l.H, th) * cdiv(l.W, tw) * cdiv(l.Cout, td) < min_tiles) continue;
        if ((th * tw * l.C + th * tw * td + td * l.C) * b > g.smem) continue;
        const ll gma = cdiv(l.C * l.Cout, td * l.C) * N * l.H * l.W * l.C + N * l.H * l.W * l.Cout +
                       cdiv(N * l.H * l.W * l.Cout, th * tw * td) * l.C * l.Cout;
        if (!best.ok || gma < best.gma) best = {true, gma, th, tw, td, "pw"};
      }
  return best;
}

// PW (C -> Cm) then DW (k, s) over T: Eq. 4 (+ DwOFM store in "consistent" accounting)
static Best paper_pwdw(const Layer& p, const Layer& d, ll N, ll b, const Gpu& g, ll min_tiles) {
  Best best;
  const ll Cin = p.C, Cm = p.Cout;
  for (ll td : dcand(Cm))
    for (ll th : cand(d.Ho))
      for (ll tw : cand(d.Wo)) {
        if ((th * tw * td) % 32) continue;
        if (N * cdiv(d.Ho, th) * cdiv(d.Wo, tw) * cdiv(Cm, td) < min_tiles) continue;
        const ll thi = std::min((th - 1) * d.s + d.k, d.H), twi = std::min((tw - 1) * d.s + d.k, d.W);
        if ((thi * twi * Cin + th * tw * td + td * Cin + d.k * d.k * td + thi * twi * td) * b > g.smem) continue;
        const ll ov = overlap(d.H, d.W, th * d.s, tw * d.s, d.k, d.k, d.s);
        const ll rep = std::max(cdiv(Cin * Cm, td * Cin), cdiv(d.k * d.k * Cm, d.k * d.k * td));
        const ll gma = (2 * Cin * N * ov + N * d.H * d.W * Cin) * rep + cdiv(N * d.Ho * d.Wo * Cm, th * tw * td) * Cin * Cm +
                       cdiv(N * d.Ho * d.Wo, th * tw) * d.k * d.k * Cm + N * d.Ho * d.Wo * Cm;
        const std::string kind = (th == d.Ho && tw == d.Wo) ? "pwdw" : "pwdw_r";
        if (!best.ok || gma < best.gma || (gma == best.gma && kind == "pwdw" && best.kind == "pwdw_r"))
          best = {true, gma, th, tw, td, kind};
      }
  return best;
}

// DW (k, s on Cin) then PW (Cin -> Co): construction rule of P:211 (reading R13)
static Best paper_dwpw(const Layer& d, const Layer& p, ll N, ll b, const Gpu& g, ll min_tiles) {
  Best best;
  const ll Cin = d.C, Co = p.Cout;
  for (ll td : dcand(Co))
    for (ll th : cand(d.Ho))
      for (ll tw : cand(d.Wo)) {
        if ((th * tw * td) % 32) continue;
        if (N * cdiv(d.Ho, th) * cdiv(d.Wo, tw) * cdiv(Co, td) < min_tiles) continue;
        const ll thi = std::min((th - 1) * d.s + d.k, d.H), twi = std::min((tw - 1) * d.s + d.k, d.W);
        if ((thi * twi * Cin + th * tw * td + d.k * d.k * Cin + Cin * td + th * tw * Cin) * b > g.smem) continue;
        const ll ov = overlap(d.H, d.W, th * d.s, tw * d.s, d.k, d.k, d.s);
        const ll nw = cdiv(Cin * Co, Cin * td);
        const ll gma = (2 * Cin * N * ov + N * d.H * d.W * Cin) * nw + cdiv(N * d.Ho * d.Wo, th * tw) * nw * d.k * d.k * Cin +
                       cdiv(N * d.Ho * d.Wo * Co, th * tw * td) * Cin * Co + N * d.Ho * d.Wo * Co;
        if (!best.ok || gma < best.gma) best = {true, gma, th, tw, td, "dwpw"};
      }
  return best;
}

// The "#OFM tiles >= #SMs" constraint is waived when no tiling can satisfy it (tiny
// layers, e.g. batch-1 14x14x16): reading R17.
template <class F>
static Best with_sm_rule(F f, ll sms) {
  Best r = f(sms);
  return r.ok ? r : f(1);
}

// ---------------------------------------------------------------------------- exact unit counts
// Distinct in-image input rows read by output rows [a, b) of a k-tap, stride-s, pad-p window.
static ll touched(ll a, ll b, ll k, ll s, ll p, ll n) {
  if (k >= s) {
    const ll lo = std::max(a * s - p, 0LL), hi = std::min((b - 1) * s - p + k, n);
    return std::max(hi - lo, 0LL);
  }
  ll c = 0;
  for (ll y = a; y < b; ++y)
    for (ll i = 0; i < k; ++i) {
      const ll r = y * s - p + i;
      c += (r >= 0 && r < n);
    }
  return c;
}

struct Units {
  ll ifm = 0, w = 0, ofm = 0, halo = 0;
  ll total() const { return ifm + w + ofm; }
};

// unit = (nb images) x (th x tw output tile) x (channel slice of width `sl`)
// kind 'dw': slice over C of the DW; 'dwpw': slice over Cout; 'pwdw': slice over Cm.
static Units units(const std::string& kind, ll N, const Layer& d, ll Cin, ll Cx, ll nb, ll th, ll tw, ll sl) {
  Units u;
  const ll Cs = (kind == "dw") ? Cin : Cx;
  std::vector<ll> ty, tx;
  for (ll y0 = 0; y0 < d.Ho; y0 += th) ty.push_back(touched(y0, std::min(y0 + th, d.Ho), d.k, d.s, d.pt, d.H));
  for (ll x0 = 0; x0 < d.Wo; x0 += tw) tx.push_back(touched(x0, std::min(x0 + tw, d.Wo), d.k, d.s, d.pl, d.W));
  for (ll n0 = 0; n0 < N; n0 += nb) {
    const ll nbe = std::min(nb, N - n0);
    for (ll ny : ty)
      for (ll nx : tx)
        for (ll c0 = 0; c0 < Cs; c0 += sl) {
          const ll ce = std::min(sl, Cs - c0);
          const ll px = nbe * ny * nx;
          if (kind == "dw") {
            u.ifm += px * ce;
            u.w += d.k * d.k * ce;
          } else if (kind == "dwpw") {
            u.ifm += px * Cin;
            u.w += d.k * d.k * Cin + Cin * ce;
          } else {
            u.ifm += px * Cin;
            u.w += Cin * ce + d.k * d.k * ce;
            u.halo += px * ce;
          }
        }
  }
  u.ofm = N * d.Ho * d.Wo * Cs;
  return u;
}

// PW kernel: row blocks of `bm` pixels x column blocks of `bn` output channels
static Units pw_units(ll M, ll Cin, ll Cout, ll bm, ll bn) {
  Units u;
  const ll nbn = cdiv(Cout, bn);
  u.ifm = nbn * M * Cin;
  u.w = cdiv(M, bm) * Cout * Cin;
  u.ofm = M * Cout;
  return u;
}

// ---------------------------------------------------------------------------- B200 costing
struct Cost {
  bool ok = false;
  std::string op;
  double us = 0;
  ll dram = 0, l2 = 0, dw_macs = 0, pw_macs = 0, red_macs = 0, t_vals = 0;
  ll nb = 1, th = 0, tw = 0, nsplit = 0;
  ll gma = -1, p_th = 0, p_tw = 0, p_td = 0;  // paper mode: Eq. value (bytes) and its argmin tile
  // paper mode keeps the paper's decision even for a pair the fused kernels cannot run
  // (k not in {3, 5}, or no kernel tile fits): such an entry is reported "executable": false and
  // runs as its two layer-by-layer kernels
  bool exec = true;
};

static double t_us(const Cost& c, int dt, const Gpu& g) {
  const double hbm = c.dram / (g.hbm_gbs * g.hbm_eff * 1e3);
  const double l2 = c.l2 / (g.l2_gbs * 1e3);
  const double eff = dt == FCM_S8 ? (c.op == "dw" ? g.dw_eff_i8 : g.dw_eff_i8_fused) : g.dw_eff;
  const double dw = (c.dw_macs + g.t_cost * c.t_vals) / (g.ffma_tmacs * 1e6 * eff);
  const double tcr = (dt == FCM_F32) ? g.ffma_tmacs : (dt == FCM_S8 ? 2.0 : 1.0) * g.tc_tmacs;
  const double pw = c.pw_macs / (tcr * 1e6);
  return std::max(std::max(hbm, l2), std::max(dw, pw)) + g.launch_us;
}

static Geo geo_of(const Layer& d, ll N, ll Cout) {
  Geo g{};
  g.N = (int)N; g.H = (int)d.H; g.W = (int)d.W; g.C = (int)d.C; g.Ho = (int)d.Ho; g.Wo = (int)d.Wo;
  g.Cout = (int)Cout; g.k = (int)d.k; g.s = (int)d.s; g.pt = (int)d.pt; g.pl = (int)d.pl; g.nb = 1;
  return g;
}

// A 16-byte-misaligned NHWC channel pitch runs on the CUDA-core kernels (csrc/simt.cu), as does
// fp32 for every PW-containing kernel.
static bool aligned16(ll c, ll b) { return (c * b) % 16 == 0; }

static Cost b200_dw(const Layer& d, ll N, int dt, ll b, const Gpu& gp) {
  Cost c;
  c.ok = true;
  c.op = "dw";
  Geo g = geo_of(d, N, d.C);
  default_dw_tile(g, (int)b);
  if ((d.C * b) % 4) { g.th = 1; g.tw = 1; }  // element-wise SIMT kernel: unit = one pixel
  c.th = g.th; c.tw = g.tw;
  const Units u = units("dw", N, d, d.C, d.C, 1, g.th, g.tw, aligned16(d.C, b) ? 128 / b : d.C);
  c.l2 = u.total() * b;
  c.dram = (N * (d.H * d.W * d.C + d.Ho * d.Wo * d.C) + d.k * d.k * d.C) * b;
  c.dw_macs = N * d.Ho * d.Wo * d.C * d.k * d.k;
  c.us = t_us(c, dt, gp);
  return c;
}

static Cost b200_pw(const Layer& p, ll N, int dt, ll b, const Gpu& gp) {
  Cost c;
  c.ok = true;
  c.op = "pw";
  const ll M = N * p.H * p.W;
  ll bm = 128, bn;
  if (dt == FCM_F32 || !aligned16(p.C, b) || !aligned16(p.Cout, b)) {
    bm = 64; bn = 64;
  } else {
    int nb_out = 0;
    bn = pick_bn((int)p.Cout, 0, (int)(128 / b), nb_out);
  }
  c.th = bm; c.nsplit = cdiv(p.Cout, bn);
  const Units u = pw_units(M, p.C, p.Cout, bm, bn);
  c.l2 = u.total() * b;
  c.dram = (M * (p.C + p.Cout + p.res * p.Cout) + p.C * p.Cout) * b;
  c.pw_macs = M * p.C * p.Cout;
  c.us = t_us(c, dt, gp);
  return c;
}

static Cost b200_dwpw(const Layer& d, const Layer& p, ll N, int dt, ll b, const Gpu& gp) {
  Cost c;
  c.op = "dwpw";
  const ll Co = p.Cout;
  Geo g = geo_of(d, N, Co);
  ll bn;
  if (dt == FCM_F32 || !aligned16(d.C, b) || !aligned16(Co, b)) {
    g.nb = 1; g.th = 8; g.tw = 8; bn = 64;
  } else {
    const int mmax = dwpw_mmax(dt, g);
    default_dwpw_tile(g, mmax, dwpw_pair_dt(dt, g));
    int nb_out = 0;
    bn = pick_bn((int)Co, 0, (int)(128 / b), nb_out);
    if (!dwpw_tile_ok(g, g.nb, g.th, g.tw, mmax)) return c;
  }
  c.ok = true;
  c.nb = g.nb; c.th = g.th; c.tw = g.tw; c.nsplit = cdiv(Co, bn);
  const Units u = units("dwpw", N, d, d.C, Co, g.nb, g.th, g.tw, bn);
  c.l2 = u.total() * b;
  c.dram = (N * (d.H * d.W * d.C + d.Ho * d.Wo * Co * (1 + p.res)) + d.k * d.k * d.C + d.C * Co) * b;
  c.dw_macs = N * d.Ho * d.Wo * d.C * d.k * d.k * c.nsplit;
  c.pw_macs = N * d.Ho * d.Wo * d.C * Co;
  c.us = t_us(c, dt, gp);
  return c;
}

static Cost b200_pwdw(const Layer& p, const Layer& d, ll N, int dt, ll b, const Gpu& gp) {
  Cost c;
  c.op = "pwdw_r";
  const ll Cin = p.C, Cm = p.Cout;
  Geo g = geo_of(d, N, Cm);
  g.C = (int)Cin;
  ll td;
  if (dt == FCM_F32 || !aligned16(Cin, b) || !aligned16(Cm, b)) {
    g.nb = 1; g.th = 8; g.tw = 8; td = 32;
  } else {
    default_pwdw_tile(g);
    td = 128 / b;
    if (!pwdw_tile_ok(g, g.nb, g.th, g.tw) || !pwdw_smem_fits(dt, g)) return c;
  }
  c.ok = true;
  c.nb = g.nb; c.th = g.th; c.tw = g.tw; c.nsplit = cdiv(Cm, td);
  const Units u = units("pwdw", N, d, Cin, Cm, g.nb, g.th, g.tw, td);
  c.l2 = u.total() * b;
  c.dram = (N * (d.H * d.W * Cin + d.Ho * d.Wo * Cm) + Cin * Cm + d.k * d.k * Cm) * b;
  c.dw_macs = N * d.Ho * d.Wo * Cm * d.k * d.k;
  c.pw_macs = u.halo * Cin;
  c.t_vals = u.halo;  // T values produced over the halo tiles (epilogue + smem writes)
  c.red_macs = (u.halo - N * d.H * d.W * Cm) * Cin;
  if (g.th == d.Ho && g.tw == d.Wo) c.op = "pwdw";
  c.us = t_us(c, dt, gp);
  return c;
}

// ---------------------------------------------------------------------------- driver
static std::string entry_json(const Cost& c, const std::vector<std::string>& ids, ll lbl_dram, double red_ratio,
                              const std::string& mode) {
  std::string s = "{\"op\":" + json::quote(c.op == "pwdw" ? "pwdw_r" : c.op) + ",\"kind\":" + json::quote(c.op) +
                  ",\"layers\":[";
  for (size_t i = 0; i < ids.size(); ++i) s += (i ? "," : "") + json::quote(ids[i]);
  s += "],\"tile\":{\"tile_n\":" + json::num(c.nb) + ",\"tile_h\":" + json::num(c.th) + ",\"tile_w\":" +
       json::num(c.tw) + ",\"n_split\":" + json::num(c.nsplit) + "}";
  s += ",\"dram_bytes\":" + json::num(c.dram) + ",\"l2_bytes\":" + json::num(c.l2) + ",\"lbl_dram_bytes\":" +
       json::num(lbl_dram) + ",\"dw_macs\":" + json::num(c.dw_macs) + ",\"pw_macs\":" + json::num(c.pw_macs) +
       ",\"redundant_macs\":" + json::num(c.red_macs) + ",\"redundancy\":" + json::num(red_ratio) +
       ",\"pred_us\":" + json::num(c.us) + ",\"executable\":" + (c.exec ? "true" : "false");
  if (mode == "paper")
    s += ",\"gma_bytes\":" + json::num(c.gma) + ",\"paper_tile\":{\"th\":" + json::num(c.p_th) + ",\"tw\":" +
         json::num(c.p_tw) + ",\"td\":" + json::num(c.p_td) + "}";
  return s + "}";
}

// integer field of a model / GPU object: range-checked before the cast (no UB on huge values)
static ll geti(const Value& v, const char* key, double def) {
  const double d = v.num(key, def);
  if (!(d >= -(double)(1LL << 40) && d <= (double)(1LL << 40)) || d != std::floor(d))
    throw std::runtime_error(std::string("field '") + key + "' must be an integer of magnitude < 2^40");
  return (ll)d;
}

static Layer parse_layer(const Value& v) {
  Layer l;
  l.id = v.str("id", "");
  l.kind = v.str("kind", "");
  l.res = geti(v, "residual", 0) != 0;
  l.extra_out = geti(v, "extra_consumers", 0);
  l.H = geti(v, "h", 0);
  l.W = geti(v, "w", 0);
  if (l.kind == "dw") {
    l.C = l.Cout = geti(v, "c", 0);
    l.k = geti(v, "k", 3);
    l.s = geti(v, "stride", 1);
    const Value* p = v.get("pads");
    const ll dp = l.k / 2;
    l.pt = l.pl = l.pb = l.pr = dp;
    if (p && p->kind == Value::Arr && p->a.size() == 4) {
      ll q[4];
      for (int i = 0; i < 4; ++i) {
        const double d = p->a[i].n;
        if (p->a[i].kind != Value::Num || !(d >= 0 && d <= 64) || d != std::floor(d))
          throw std::runtime_error("layer " + l.id + ": pads must be integers in [0, 64]");
        q[i] = (ll)d;
      }
      l.pt = q[0]; l.pl = q[1]; l.pb = q[2]; l.pr = q[3];
    }
    if (l.H + l.pt + l.pb < l.k || l.W + l.pl + l.pr < l.k)
      throw std::runtime_error("layer " + l.id + ": the k x k window does not fit the padded input");
    l.Ho = (l.H + l.pt + l.pb - l.k) / l.s + 1;
    l.Wo = (l.W + l.pl + l.pr - l.k) / l.s + 1;
  } else if (l.kind == "pw") {
    l.C = geti(v, "c_in", 0);
    l.Cout = geti(v, "c_out", 0);
    l.Ho = l.H;
    l.Wo = l.W;
  } else {
    throw std::runtime_error("layer " + l.id + ": kind must be dw or pw");
  }
  if (l.id.empty() || l.H < 1 || l.W < 1 || l.C < 1 || l.Cout < 1 || l.k < 1 || l.s < 1 || l.Ho < 1 || l.Wo < 1)
    throw std::runtime_error("layer " + l.id + ": bad dims");
  return l;
}

static std::string run(const char* model_json, const char* gpu_json) {
  const Value m = json::Parser(model_json).parse();
  if (m.kind != Value::Obj) throw std::runtime_error("model JSON must be an object");
  const std::string dts = m.str("dtype", "bf16");
  const int dt = dts == "f32" ? FCM_F32 : dts == "f16" ? FCM_F16 : dts == "s8" ? FCM_S8 : FCM_BF16;
  if (dts != "f32" && dts != "f16" && dts != "s8" && dts != "bf16") throw std::runtime_error("bad dtype " + dts);
  const ll b = elem_size(dt);
  const ll N = geti(m, "batch", 1);
  const std::string mode = m.str("mode", "b200");
  if (mode != "b200" && mode != "paper") throw std::runtime_error("mode must be b200 or paper");
  Gpu gp;
  if (gpu_json) {
    const Value g = json::Parser(gpu_json).parse();
    gp.sms = geti(g, "num_sms", (double)gp.sms);
    gp.smem = geti(g, "smem_bytes", (double)gp.smem);
    gp.l2 = geti(g, "l2_bytes", (double)gp.l2);
    gp.hbm_gbs = g.num("hbm_gbs", gp.hbm_gbs);
    gp.l2_gbs = g.num("l2_gbs", gp.l2_gbs);
    gp.tc_tmacs = g.num("tc_tmacs", gp.tc_tmacs);
    gp.ffma_tmacs = g.num("ffma_tmacs", gp.ffma_tmacs);
    gp.dw_eff = g.num("dw_eff", gp.dw_eff);
    gp.dw_eff_i8 = g.num("dw_eff_i8", gp.dw_eff_i8);
    gp.dw_eff_i8_fused = g.num("dw_eff_i8_fused", gp.dw_eff_i8_fused);
    gp.launch_us = g.num("launch_us", gp.launch_us);
    gp.hbm_eff = g.num("hbm_eff", gp.hbm_eff);
    gp.t_cost = g.num("t_cost", gp.t_cost);
  }
  const Value* lv = m.get("layers");
  if (!lv || lv->kind != Value::Arr || lv->a.empty()) throw std::runtime_error("model needs a non-empty layers array");
  std::vector<Layer> L;
  for (auto& v : lv->a) L.push_back(parse_layer(v));
  const size_t n = L.size();
  // edges -> producer/consumer counts; default: a chain in list order
  std::vector<int> outdeg(n, 0), indeg(n, 0);
  for (size_t i = 0; i < n; ++i) outdeg[i] = (int)L[i].extra_out;  // residual shortcuts (single-consumer rule)
  std::vector<char> link(n, 0);  // link[i]: edge L[i-1] -> L[i]
  const Value* ev = m.get("edges");
  auto idx = [&](const std::string& id) -> int {
    for (size_t i = 0; i < n; ++i)
      if (L[i].id == id) return (int)i;
    throw std::runtime_error("edge names unknown layer " + id);
  };
  if (ev && ev->kind == Value::Arr) {
    for (auto& e : ev->a) {
      if (e.kind != Value::Arr || e.a.size() != 2) throw std::runtime_error("edges must be [from, to] pairs");
      const int a = idx(e.a[0].s), c = idx(e.a[1].s);
      outdeg[a]++;
      indeg[c]++;
      const Layer &pa = L[a], &pc = L[c];
      if (pa.Ho != pc.H || pa.Wo != pc.W || pa.Cout != pc.C)
        throw std::runtime_error("edge " + pa.id + "->" + pc.id + ": shape mismatch");
      if (c == a + 1) link[c] = 1;
    }
  } else {
    for (size_t i = 1; i < n; ++i) {
      outdeg[i - 1]++; indeg[i]++; link[i] = 1;
      if (L[i - 1].Ho != L[i].H || L[i - 1].Wo != L[i].W || L[i - 1].Cout != L[i].C)
        throw std::runtime_error("chain " + L[i - 1].id + "->" + L[i].id + ": shape mismatch");
    }
  }
  // per-layer LBL
  std::vector<Cost> lbl(n);
  for (size_t i = 0; i < n; ++i) {
    const Layer& l = L[i];
    if (mode == "paper") {
      Best bst = with_sm_rule([&](ll mt) { return l.kind == "dw" ? paper_dw(l, N, b, gp, mt) : paper_pw(l, N, b, gp, mt); }, gp.sms);
      Cost c = l.kind == "dw" ? b200_dw(l, N, dt, b, gp) : b200_pw(l, N, dt, b, gp);
      if (!bst.ok) {
        // no tile of the grid fits on chip: the layer runs untiled, GMA = IFM + W + OFM (the
        // single-tile closed form of Eq. 2 / Eq. 3)
        const ll w = l.kind == "dw" ? l.k * l.k * l.C : l.C * l.Cout;
        bst = {true, N * l.H * l.W * l.C + w + N * l.Ho * l.Wo * l.Cout, l.Ho, l.Wo, l.Cout, l.kind};
      }
      c.gma = bst.gma * b;
      c.p_th = bst.th; c.p_tw = bst.tw; c.p_td = bst.td;
      lbl[i] = c;
    } else {
      lbl[i] = l.kind == "dw" ? b200_dw(l, N, dt, b, gp) : b200_pw(l, N, dt, b, gp);
    }
  }
  // pair candidates (i-1, i)
  std::vector<Cost> fc(n), fall(n);
  for (size_t i = 1; i < n; ++i) {
    if (!link[i] || outdeg[i - 1] != 1 || indeg[i] != 1) continue;
    const Layer &a = L[i - 1], &c = L[i];
    // the fused kernels are built for k in {3, 5} (fcm_dw also has k = 7): no FCM candidate
    // otherwise in b200 mode (paper mode keeps the paper's decision)
    const Layer& dwl = a.kind == "dw" ? a : c;
    const bool k_ok = dwl.kind != "dw" || dwl.k == 3 || dwl.k == 5;
    if (mode != "paper" && !k_ok) continue;
    Cost f;
    if (a.kind == "dw" && c.kind == "pw") {
      if (mode == "paper") {
        Best bst = with_sm_rule([&](ll mt) { return paper_dwpw(a, c, N, b, gp, mt); }, gp.sms);
        if (!bst.ok) continue;
        f = b200_dwpw(a, c, N, dt, b, gp);
        f.exec = f.ok && k_ok;
        f.ok = true;
        f.dram = (N * (a.H * a.W * a.C + a.Ho * a.Wo * c.Cout * (1 + c.res)) + a.k * a.k * a.C + a.C * c.Cout) * b;
        f.gma = bst.gma * b; f.p_th = bst.th; f.p_tw = bst.tw; f.p_td = bst.td;
      } else {
        f = b200_dwpw(a, c, N, dt, b, gp);
      }
    } else if (a.kind == "pw" && c.kind == "dw") {
      if (mode == "paper") {
        Best bst = with_sm_rule([&](ll mt) { return paper_pwdw(a, c, N, b, gp, mt); }, gp.sms);
        if (!bst.ok) continue;
        f = b200_pwdw(a, c, N, dt, b, gp);
        f.exec = f.ok && k_ok;
        f.ok = true;
        f.dram = (N * (c.H * c.W * a.C + c.Ho * c.Wo * a.Cout) + a.C * a.Cout + c.k * c.k * a.Cout) * b;
        f.op = bst.kind;
        f.gma = bst.gma * b; f.p_th = bst.th; f.p_tw = bst.tw; f.p_td = bst.td;
      } else {
        f = b200_pwdw(a, c, N, dt, b, gp);
      }
    } else {
      continue;  // (DW,DW) never fuses; (PW,PW) is a NEXT item
    }
    if (!f.ok) continue;
    fall[i] = f;
    // fuse only if strictly better than the two LBL layers
    const bool better = (mode == "paper") ? f.gma < lbl[i - 1].gma + lbl[i].gma : f.us < lbl[i - 1].us + lbl[i].us;
    if (better) fc[i] = f;
  }
  // chain DP: dp[i] = best cost of layers [0, i)
  std::vector<double> dp(n + 1, 0.0);
  std::vector<int> take(n + 1, 0);
  auto cost_of = [&](const Cost& c) { return mode == "paper" ? (double)c.gma : c.us; };
  for (size_t i = 1; i <= n; ++i) {
    dp[i] = dp[i - 1] + cost_of(lbl[i - 1]);
    take[i] = 1;
    if (i >= 2 && fc[i - 1].ok) {
      const double v = dp[i - 2] + cost_of(fc[i - 1]);
      if (v <= dp[i]) { dp[i] = v; take[i] = 2; }
    }
  }
  std::vector<std::string> ents;
  ll tot_dram = 0, tot_lbl = 0, n_fused = 0;
  double tot_us = 0;
  for (ll i = (ll)n; i > 0;) {
    if (take[i] == 2) {
      const Cost& f = fc[i - 1];
      const ll lbl_d = lbl[i - 2].dram + lbl[i - 1].dram;
      double rr = 0;
      if (f.op == "pwdw_r" || f.op == "pwdw") {
        const double nominal = (double)(f.pw_macs - f.red_macs) + (double)f.dw_macs;
        rr = f.red_macs > 0 ? f.red_macs / (nominal + f.red_macs) : 0.0;
      }
      ents.push_back(entry_json(f, {L[i - 2].id, L[i - 1].id}, lbl_d, rr, mode));
      tot_dram += f.dram; tot_lbl += lbl_d; tot_us += f.us; ++n_fused;
      i -= 2;
    } else {
      const Cost& c = lbl[i - 1];
      ents.push_back(entry_json(c, {L[i - 1].id}, c.dram, 0.0, mode));
      tot_dram += c.dram; tot_lbl += c.dram; tot_us += c.us;
      i -= 1;
    }
  }
  std::reverse(ents.begin(), ents.end());
  std::string out = "{\"mode\":" + json::quote(mode) + ",\"dtype\":" + json::quote(dts) + ",\"batch\":" + json::num(N) +
                    ",\"gpu\":{\"num_sms\":" + json::num(gp.sms) + ",\"smem_bytes\":" + json::num(gp.smem) +
                    ",\"hbm_gbs\":" + json::num(gp.hbm_gbs) + "},\"entries\":[";
  for (size_t i = 0; i < ents.size(); ++i) out += (i ? "," : "") + ents[i];
  out += "],\"candidates\":{\"lbl\":[";
  for (size_t i = 0; i < n; ++i) out += (i ? "," : "") + entry_json(lbl[i], {L[i].id}, lbl[i].dram, 0.0, mode);
  out += "],\"fcm\":[";
  bool first = true;
  for (size_t i = 1; i < n; ++i) {
    if (!fall[i].ok) continue;
    std::string e = entry_json(fall[i], {L[i - 1].id, L[i].id}, lbl[i - 1].dram + lbl[i].dram, 0.0, mode);
    e.back() = ',';
    e += std::string("\"accepted\":") + (fc[i].ok ? "true" : "false") + "}";
    out += (first ? "" : ",") + e;
    first = false;
  }
  out += "]},\"totals\":{\"dram_bytes\":" + json::num(tot_dram) + ",\"lbl_dram_bytes\":" + json::num(tot_lbl) +
         ",\"pred_us\":" + json::num(tot_us) + ",\"fused_pairs\":" + json::num(n_fused) + ",\"conv_layers\":" +
         json::num((ll)n) + "}}";
  return out;
}

}  // namespace plan
}  // namespace fcm

extern "C" int fcm_plan(const char* model_json, const char* gpu_json, char* out, size_t cap, size_t* needed) {
  if (!model_json) return fcm::set_error(FCM_E_INVAL, "fcm_plan: model_json is NULL");
  std::string s;
  try {
    s = fcm::plan::run(model_json, gpu_json);
  } catch (const std::exception& e) {
    return fcm::set_error(FCM_E_INVAL, std::string("fcm_plan: ") + e.what());
  }
  const size_t n = s.size() + 1;
  if (needed) *needed = n;
  if (!out || cap < n) return fcm::set_error(FCM_E_BUFSZ, "fcm_plan: output buffer too small");
  std::memcpy(out, s.c_str(), n);
  return FCM_OK;
}
