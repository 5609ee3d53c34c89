// laydown.cpp — host side of the hot path, run once per problem.
//
//  * 2D cyclic track laydown with corrected azimuths (App. A.1; P:129
//    "the CPU executes 2D ray tracing to generate the requisite data for 3D").
//  * 2D reflective links by integer boundary-grid-point arithmetic (App. A.2) and
//    the 2D cycles they form.
//  * 2D segmentation by marching the pin lattice cell by cell, with the
//    epsilon-merge of App. A.7 (readings Q22, Q22b).
//  * Gauss-Legendre polar nodes, per-(a, n) corrected polar angles, z-stacks with
//    cyclic phases (App. A.3-A.4, Eq. 5, reading Q7b), 3D links by index arithmetic.
//
// Written independently of oracle/ (which matches links geometrically and segments
// by brute force); tests compare the two.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <numeric>

#include "host.h"

namespace moc {

namespace {
const double kPi = 3.14159265358979323846;
const double kPhaseFrac = 0.6180339887498949;  // reading Q7b

struct EndPt {
  int face;
  int idx;
};

// Boundary grid points of track q of a first-quadrant family with (nx, ny) tracks
// per edge (App. A.2): faces 0 x-, 1 x+, 2 y-, 3 y+.
void quadrant_track_ends(int nx, int ny, int q, EndPt& st, EndPt& en) {
  if (q < ny) {
    int j = ny - 1 - q;
    st = {0, j};
    if (ny - j - 1 < nx) en = {3, ny - j - 1};
    else en = {1, j + nx};
  } else {
    int i = q - ny;
    st = {2, i};
    if (i + ny < nx) en = {3, i + ny};
    else en = {1, nx - i - 1};
  }
}

EndPt mirror(EndPt e, int nx) {
  if (e.face == 0) return {1, e.idx};
  if (e.face == 1) return {0, e.idx};
  return {e.face, nx - 1 - e.idx};
}

void gauss_legendre_desc(int N, std::vector<double>& mu, std::vector<double>& w) {
  // Newton on P_N from Tricomi's initial guesses; nodes returned descending.
  mu.resize(N);
  w.resize(N);
  for (int i = 0; i < N; ++i) {
    double x = std::cos(kPi * (4.0 * i + 3.0) / (4.0 * N + 2.0));
    double dpn = 1.0;
    for (int it = 0; it < 200; ++it) {
      double pm1 = 1.0, p = x;  // P_0, P_1
      for (int k = 1; k < N; ++k) {
        double pn = ((2 * k + 1) * x * p - k * pm1) / (k + 1);
        pm1 = p;
        p = pn;
      }
      dpn = N * (pm1 - x * p) / (1.0 - x * x);
      double step = p / dpn;
      x -= step;
      if (std::fabs(step) <= 1e-17) break;
    }
    double pm1 = 1.0, p = x;
    for (int k = 1; k < N; ++k) {
      double pn = ((2 * k + 1) * x * p - k * pm1) / (k + 1);
      pm1 = p;
      p = pn;
    }
    dpn = N * (pm1 - x * p) / (1.0 - x * x);
    mu[i] = x;
    w[i] = 2.0 / ((1.0 - x * x) * dpn * dpn);
  }
  std::vector<int> o(N);
  std::iota(o.begin(), o.end(), 0);
  std::sort(o.begin(), o.end(), [&](int a, int b) { return mu[a] > mu[b]; });
  std::vector<double> m2(N), w2(N);
  for (int i = 0; i < N; ++i) {
    m2[i] = mu[o[i]];
    w2[i] = w[o[i]];
  }
  mu.swap(m2);
  w.swap(w2);
}

// merge state machine of App. A.7 over raw pieces (same rule as otf.h)
struct Merger {
  std::vector<uint32_t>& reg;
  std::vector<double>& send;
  int64_t pj = -1;
  double pend = 0, pstart = 0;
  bool lead = false;
  void raw(uint32_t r, double a0, double a1) {
    double len = a1 - a0;
    if (pj < 0) {
      pj = r;
      pstart = a0;
      pend = a1;
      lead = len < kEpsL;
    } else if (len < kEpsL) {
      pend = a1;
    } else if (lead) {
      pj = r;
      pend = a1;
      lead = false;
    } else {
      reg.push_back((uint32_t)pj);
      send.push_back(pend);
      pj = r;
      pstart = a0;
      pend = a1;
    }
  }
  void finish(double L) {
    reg.push_back((uint32_t)pj);
    send.push_back(L);
  }
};

}  // namespace

int64_t Geometry::region_at(int cx, int cy, double x, double y) const {
  int c = cy * nx + cx;
  int ty = cell_type[c];
  double ddx = x - (cx + 0.5) * px, ddy = y - (cy + 0.5) * py;
  double d2 = ddx * ddx + ddy * ddy;
  int nr = n_rings[ty];
  int local = nr;
  for (int q = 0; q < nr; ++q) {
    double r = radii[(size_t)ty * max_rings + q];
    if (d2 < r * r) {
      local = q;
      break;
    }
  }
  return prefix[c] + local;
}

// Analytic FSR volumes (S:83-85 'analytic_volume'): ring q of a cell is the annulus
// pi (r_q^2 - r_{q-1}^2), the moderator the cell minus the outer circle, times the layer
// height (rings lie inside their cell; App. A.6 numbering j = r * NL + layer).
void Geometry::analytic_volumes(double* vol) const {
  const double pi = 3.14159265358979323846;
  for (int c = 0; c < nx * ny; ++c) {
    const int ty = cell_type[c], nr = n_rings[ty];
    double prev = 0.0;
    for (int q = 0; q <= nr; ++q) {
      double area;
      if (q < nr) {
        const double rq = radii[(size_t)ty * max_rings + q];
        area = pi * (rq * rq - prev * prev);
        prev = rq;
      } else {
        area = px * py - pi * prev * prev;
      }
      const int64_t r = prefix[c] + q;
      for (int l = 0; l < NL; ++l) vol[r * NL + l] = area * (planes[l + 1] - planes[l]);
    }
  }
}

int Geometry::mat_of_fsr(int64_t j) const {
  int64_t r = j / NL;
  int l = (int)(j % NL);
  int64_t c = std::upper_bound(prefix.begin(), prefix.end(), r) - prefix.begin() - 1;
  int ty = cell_type[c];
  int local = (int)(r - prefix[c]);
  return material[((size_t)ty * (max_rings + 1) + local) * n_zones + zone_of_layer[l]];
}

// 2D segmentation of one track by marching lattice cells; raw pieces are the cell
// crossings split at ring crossings whose chord exceeds eps_L (App. A.7).
static void segment_track(const Geometry& g, double x0, double y0, double ux, double uy, double L,
                          std::vector<uint32_t>& reg, std::vector<double>& send) {
  Merger mg{reg, send};
  int cx = ux > 0 ? (int)std::floor(x0 / g.px) : (int)std::ceil(x0 / g.px) - 1;
  int cy = (int)std::floor(y0 / g.py);  // uy > 0 for all tracks (phi in (0, pi))
  cx = std::min(std::max(cx, 0), g.nx - 1);
  cy = std::min(std::max(cy, 0), g.ny - 1);
  double u = 0.0;
  double cross[64];
  int guard = 0;
  while (true) {
    double ux_exit = ux > 0 ? ((cx + 1) * g.px - x0) / ux : (cx * g.px - x0) / ux;
    double uy_exit = ((cy + 1) * g.py - y0) / uy;
    double ue = std::min(std::min(ux_exit, uy_exit), L);
    int ty = g.cell_type[cy * g.nx + cx];
    int nc = 0;
    double wx = (cx + 0.5) * g.px - x0, wy = (cy + 0.5) * g.py - y0;
    double proj = wx * ux + wy * uy;
    double d2 = wx * wx + wy * wy - proj * proj;
    for (int q = 0; q < g.n_rings[ty]; ++q) {
      double r = g.radii[(size_t)ty * g.max_rings + q];
      if (d2 >= r * r) continue;
      double half = std::sqrt(r * r - d2);
      if (2.0 * half <= kEpsL) continue;
      double u1 = proj - half, u2 = proj + half;
      if (u1 > u && u1 < ue) cross[nc++] = u1;
      if (u2 > u && u2 < ue) cross[nc++] = u2;
    }
    std::sort(cross, cross + nc);
    double a0 = u;
    for (int q = 0; q <= nc; ++q) {
      double a1 = q < nc ? cross[q] : ue;
      double um = 0.5 * (a0 + a1);
      mg.raw((uint32_t)g.region_at(cx, cy, x0 + um * ux, y0 + um * uy), a0, a1);
      a0 = a1;
    }
    u = ue;
    if (u >= L) break;
    if (ux_exit <= uy_exit) cx += ux > 0 ? 1 : -1;
    if (uy_exit <= ux_exit) cy += 1;
    if (cx < 0 || cx >= g.nx || cy < 0 || cy >= g.ny || ++guard > 10 * (g.nx + g.ny) + 16)
      throw Error(MOC_E_TRACE, "2D segmentation left the lattice before the track end");
  }
  mg.finish(L);
}

void build_laydown(const Geometry& g, const moc_track_params& tp, Laydown& L) {
  L = Laydown();
  L.M = tp.num_azim;
  L.N = tp.num_polar;
  L.dr = tp.radial_spacing;
  L.dzs = tp.axial_spacing;
  const int M = L.M, N = L.N, Q = M / 4, F = M / 2;
  if (M < 4 || M % 4 != 0) throw Error(MOC_E_PARAM, "num_azim must be a positive multiple of 4");
  if (N < 2 || N % 2 != 0) throw Error(MOC_E_PARAM, "num_polar must be even and >= 2");
  if (!(L.dr > 0) || L.dr > std::min(g.W, g.Y)) throw Error(MOC_E_PARAM, "radial_spacing must be in (0, min(W, Y)]");
  if (!(L.dzs > 0) || L.dzs > g.Z) throw Error(MOC_E_PARAM, "axial_spacing must be in (0, Z]");
  // ---- App. A.1: corrected azimuths, spacings, weights
  L.phi.assign(F, 0);
  L.delta.assign(F, 0);
  L.omega.assign(F, 0);
  L.nxa.assign(F, 0);
  L.nya.assign(F, 0);
  for (int a = 0; a < Q; ++a) {
    double want = 2.0 * kPi / M * (a + 0.5);
    int nxa = (int)std::floor(g.W * std::sin(want) / L.dr) + 1;
    int nya = (int)std::floor(g.Y * std::cos(want) / L.dr) + 1;
    double ph = std::atan((g.Y * nxa) / (g.W * nya));
    int ac = F - 1 - a;
    L.phi[a] = ph;
    L.phi[ac] = kPi - ph;
    L.nxa[a] = L.nxa[ac] = nxa;
    L.nya[a] = L.nya[ac] = nya;
    L.delta[a] = L.delta[ac] = (g.W / nxa) * std::sin(ph);
  }
  for (int a = 0; a < Q; ++a) {
    double b0 = a == 0 ? 0.0 : 0.5 * (L.phi[a - 1] + L.phi[a]);
    double b1 = a == Q - 1 ? 0.5 * kPi : 0.5 * (L.phi[a] + L.phi[a + 1]);
    L.omega[a] = L.omega[F - 1 - a] = (b1 - b0) / (2.0 * kPi);
  }
  // ---- 2D tracks (family-major, within a family by perpendicular offset)
  L.fam_off.assign(F + 1, 0);
  for (int a = 0; a < F; ++a) L.fam_off[a + 1] = L.fam_off[a] + L.nxa[a] + L.nya[a];
  const int64_t T2 = L.fam_off[F];
  L.t_a.resize(T2);
  L.t_x0.resize(T2);
  L.t_y0.resize(T2);
  L.t_x1.resize(T2);
  L.t_y1.resize(T2);
  L.t_len.resize(T2);
  L.t_ux.resize(T2);
  L.t_uy.resize(T2);
  L.t_fstart.resize(T2);
  L.t_fend.resize(T2);
  std::vector<EndPt> est(T2), een(T2);
  for (int a = 0; a < F; ++a) {
    const bool mir = a >= Q;
    const int asrc = mir ? F - 1 - a : a;
    const int nxa = L.nxa[a], nya = L.nya[a];
    const double dx = g.W / nxa, dy = g.Y / nya;
    const double cph = std::cos(L.phi[asrc]), sph = std::sin(L.phi[asrc]);
    for (int q = 0; q < nxa + nya; ++q) {
      int64_t t = L.fam_off[a] + q;
      EndPt s0, e0;
      quadrant_track_ends(nxa, nya, q, s0, e0);
      double xs = s0.face == 0 ? 0.0 : dx * (s0.idx + 0.5);
      double ys = s0.face == 0 ? dy * (s0.idx + 0.5) : 0.0;
      if (mir) {
        s0 = mirror(s0, nxa);
        e0 = mirror(e0, nxa);
        xs = g.W - xs;
      }
      double ux = mir ? -cph : cph, uy = sph;
      double tx = ux > 0 ? (g.W - xs) / ux : (0.0 - xs) / ux;
      double tyy = (g.Y - ys) / uy;
      double len = std::min(tx, tyy);
      int fend_geo = tx < tyy ? (ux > 0 ? 1 : 0) : 3;
      if (fend_geo != e0.face) throw Error(MOC_E_TRACE, "2D track end face disagrees with grid arithmetic");
      L.t_a[t] = a;
      L.t_x0[t] = xs;
      L.t_y0[t] = ys;
      L.t_ux[t] = ux;
      L.t_uy[t] = uy;
      L.t_len[t] = len;
      double x1 = xs + len * ux, y1 = ys + len * uy;
      if (e0.face == 0) x1 = 0.0;
      if (e0.face == 1) x1 = g.W;
      if (e0.face == 3) y1 = g.Y;
      L.t_x1[t] = x1;
      L.t_y1[t] = y1;
      L.t_fstart[t] = (int8_t)s0.face;
      L.t_fend[t] = (int8_t)e0.face;
      est[t] = s0;
      een[t] = e0;
    }
  }
  // ---- App. A.2: geometric links through boundary grid points
  // table[family][face][idx] = q*2 + (is_start ? 1 : 0)
  L.t_glf.resize(T2);
  L.t_glb.resize(T2);
  L.t_glf_fwd.resize(T2);
  L.t_glb_fwd.resize(T2);
  std::vector<std::vector<int64_t>> tab((size_t)F * 4);
  for (int a = 0; a < F; ++a) {
    tab[a * 4 + 0].assign(L.nya[a], -1);
    tab[a * 4 + 1].assign(L.nya[a], -1);
    tab[a * 4 + 2].assign(L.nxa[a], -1);
    tab[a * 4 + 3].assign(L.nxa[a], -1);
    for (int q = 0; q < L.nxa[a] + L.nya[a]; ++q) {
      int64_t t = L.fam_off[a] + q;
      tab[a * 4 + est[t].face][est[t].idx] = 2 * (int64_t)q + 1;
      tab[a * 4 + een[t].face][een[t].idx] = 2 * (int64_t)q;
    }
  }
  for (int a = 0; a < F; ++a) {
    int ac = F - 1 - a;
    for (int q = 0; q < L.nxa[a] + L.nya[a]; ++q) {
      int64_t t = L.fam_off[a] + q;
      int64_t e = tab[ac * 4 + een[t].face][een[t].idx];
      int64_t b = tab[ac * 4 + est[t].face][est[t].idx];
      if (e < 0 || b < 0) throw Error(MOC_E_TRACE, "2D link target missing");
      L.t_glf[t] = L.fam_off[ac] + e / 2;
      L.t_glf_fwd[t] = (int8_t)(e & 1);
      L.t_glb[t] = L.fam_off[ac] + b / 2;
      L.t_glb_fwd[t] = (int8_t)(b & 1);
    }
  }
  // ---- cycles: lowest-id track traversed forward
  L.t_cyc.assign(T2, -1);
  L.t_lt.assign(T2, 0);
  L.t_sig.assign(T2, 0);
  L.cycle_len.assign(F, -1.0);
  L.n_cycles = 0;
  for (int64_t t0 = 0; t0 < T2; ++t0) {
    if (L.t_cyc[t0] >= 0) continue;
    int64_t cur = t0;
    bool fwd = true;
    double cum = 0;
    std::vector<int64_t> mem;
    do {
      if (L.t_cyc[cur] >= 0) throw Error(MOC_E_TRACE, "2D cycle revisits a track");
      L.t_cyc[cur] = L.n_cycles;
      L.t_sig[cur] = fwd ? 1 : -1;
      L.t_lt[cur] = fwd ? cum : cum + L.t_len[cur];
      cum += L.t_len[cur];
      mem.push_back(cur);
      int64_t nxt = fwd ? L.t_glf[cur] : L.t_glb[cur];
      bool nf = (fwd ? L.t_glf_fwd[cur] : L.t_glb_fwd[cur]) != 0;
      cur = nxt;
      fwd = nf;
    } while (!(cur == t0 && fwd));
    for (int64_t m : mem) {
      int a = L.t_a[m];
      if (L.cycle_len[a] < 0) L.cycle_len[a] = cum;
      else if (std::fabs(L.cycle_len[a] - cum) > 1e-9 * cum) throw Error(MOC_E_TRACE, "unequal cycle lengths");
    }
    ++L.n_cycles;
  }
  // ---- 2D segmentation
  L.t_seg.assign(T2 + 1, 0);
  {
    std::vector<std::vector<uint32_t>> r(T2);
    std::vector<std::vector<double>> s(T2);
    std::string err;
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t t = 0; t < T2; ++t) {
      try {
        segment_track(g, L.t_x0[t], L.t_y0[t], L.t_ux[t], L.t_uy[t], L.t_len[t], r[t], s[t]);
      } catch (const Error& e) {
#pragma omp critical
        err = e.what() + std::string(" (2D track ") + std::to_string(t) + ")";
      }
    }
    if (!err.empty()) throw Error(MOC_E_TRACE, err);
    for (int64_t t = 0; t < T2; ++t) L.t_seg[t + 1] = L.t_seg[t] + (int64_t)r[t].size();
    L.seg_region.resize(L.t_seg[T2]);
    L.seg_send.resize(L.t_seg[T2]);
    for (int64_t t = 0; t < T2; ++t) {
      std::copy(r[t].begin(), r[t].end(), L.seg_region.begin() + L.t_seg[t]);
      std::copy(s[t].begin(), s[t].end(), L.seg_send.begin() + L.t_seg[t]);
    }
  }
  // ---- App. A.3-A.4: polar quadrature and per-(a, n) corrected angles
  gauss_legendre_desc(N, L.mu, L.wgl);
  size_t AN = (size_t)F * N;
  L.an_theta.assign(AN, 0);
  L.an_cot.assign(AN, 0);
  L.an_tan.assign(AN, 0);
  L.an_invsin.assign(AN, 0);
  L.an_dz.assign(AN, 0);
  L.an_w.assign(AN, 0);
  L.an_aperp.assign(AN, 0);
  for (int a = 0; a < F; ++a) {
    const double LC = L.cycle_len[a];
    for (int n = 0; n < N / 2; ++n) {
      double th_want = std::acos(L.mu[n]);
      int nz = (int)std::floor(g.Z * std::sin(th_want) / L.dzs) + 1;
      int nl = (int)std::floor(LC * std::cos(th_want) / L.dzs) + 1;
      double dz = g.Z / nz, dl = LC / nl;
      double th = std::atan(dl / dz);
      size_t up = (size_t)a * N + n, lo = (size_t)a * N + (N - 1 - n);
      double s = std::sin(th), c = std::cos(th);
      L.an_theta[up] = th;
      L.an_theta[lo] = kPi - th;
      L.an_cot[up] = c / s;
      L.an_cot[lo] = -(c / s);
      L.an_tan[up] = s / c;
      L.an_tan[lo] = -(s / c);
      L.an_invsin[up] = L.an_invsin[lo] = 1.0 / s;
      L.an_dz[up] = L.an_dz[lo] = dz;
      L.an_aperp[up] = L.an_aperp[lo] = L.delta[a] * dz * s;  // App. A.5
    }
    for (int n = 0; n < N; ++n) L.an_w[(size_t)a * N + n] = 4.0 * kPi * L.omega[a] * (0.5 * L.wgl[n]);
  }
  // ---- z-stacks: members whose line meets (0, Z) with positive length over s in (0, L_t)
  const int64_t S = T2 * N;
  L.st_z0.assign(S, 0);
  L.st_cnt.assign(S, 0);
  L.st_first.assign(S + 1, 0);
  int64_t degenerate = 0;
  for (int64_t t = 0; t < T2; ++t) {
    const int a = L.t_a[t];
    for (int n = 0; n < N; ++n) {
      const int nu = n < N / 2 ? n : N - 1 - n;
      const size_t an = (size_t)a * N + n, anu = (size_t)a * N + nu;
      double ph = L.t_sig[t] * (L.t_lt[t] * L.an_cot[anu] - kPhaseFrac * L.an_dz[anu]);
      if (n >= N / 2) ph = -ph;
      const double c = L.an_cot[an], D = L.an_dz[an], Lt = L.t_len[t];
      double lo, hi;
      if (c > 0) {
        lo = (-Lt * c - ph) / D;
        hi = (g.Z - ph) / D;
      } else {
        lo = (-ph) / D;
        hi = (g.Z - Lt * c - ph) / D;
      }
      if (std::fabs(lo - std::nearbyint(lo)) < 1e-9 || std::fabs(hi - std::nearbyint(hi)) < 1e-9) ++degenerate;
      int64_t mlo = (int64_t)std::floor(lo) + 1, mhi = (int64_t)std::ceil(hi) - 1;
      int64_t s = t * N + n;
      L.st_cnt[s] = std::max<int64_t>(0, mhi - mlo + 1);
      L.st_z0[s] = ph + (double)mlo * D;
    }
  }
  if (degenerate)
    throw Error(MOC_E_TRACE, std::to_string(degenerate) + " z-stack members touch a box edge within 1e-9 dz");
  for (int64_t s = 0; s < S; ++s) L.st_first[s + 1] = L.st_first[s] + L.st_cnt[s];
  L.n3 = L.st_first[S];
  // raw piece count estimate (#2D segments spanned + #planes crossed) for sizing
  int64_t raw = 0;
  const OtfView v = otf_view_host(g, L);
  L.st_raw.assign(S, 0);
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : raw)
  for (int64_t s = 0; s < S; ++s) {
    int64_t t = s / N;
    int n = (int)(s % N);
    size_t an = (size_t)L.t_a[t] * N + n;
    int64_t raw_s = 0;
    for (int64_t i = 0; i < L.st_cnt[s]; ++i) {
      TrackGeo tg{L.st_z0[s] + (double)i * L.an_dz[an], L.an_cot[an], L.an_tan[an], L.an_invsin[an],
                  L.t_len[t], g.Z, L.t_seg[t], L.t_seg[t + 1]};
      double s_in, s_out;
      otf_clip(tg, s_in, s_out);
      int64_t k0 = otf_seg_after(v, tg.sb, tg.se, s_in), k1 = otf_seg_upto(v, tg.sb, tg.se, s_out);
      double z_in = tg.z0 + s_in * tg.cot, z_out = tg.z0 + s_out * tg.cot;
      int l0 = otf_layer_up(v, std::min(z_in, z_out)), l1 = otf_layer_down(v, std::max(z_in, z_out));
      raw_s += (k1 - k0 + 1) + std::max(0, l1 - l0);
    }
    L.st_raw[s] = raw_s;
    raw += raw_s;
  }
  L.n_raw3 = raw;
  L.done = true;
}

OtfView otf_view_host(const Geometry& g, const Laydown& L) {
  return OtfView{L.seg_send.data(), L.seg_region.data(), g.planes.data(), g.NL};
}

TrackGeo track_geo(const Geometry& g, const Laydown& L, int64_t track, int64_t* stack_out) {
  int64_t s = std::upper_bound(L.st_first.begin(), L.st_first.end(), track) - L.st_first.begin() - 1;
  int64_t t = s / L.N;
  int n = (int)(s % L.N);
  size_t an = (size_t)L.t_a[t] * L.N + n;
  int64_t i = track - L.st_first[s];
  if (stack_out) *stack_out = s;
  return TrackGeo{L.st_z0[s] + (double)i * L.an_dz[an], L.an_cot[an], L.an_tan[an], L.an_invsin[an],
                  L.t_len[t], g.Z, L.t_seg[t], L.t_seg[t + 1]};
}

// App. A.4 3D links by index arithmetic.  Returns the target slot or -1 (vacuum).
int64_t link_slot(const Geometry& g, const Laydown& L, int64_t track, int dir) {
  int64_t s;
  TrackGeo tg = track_geo(g, L, track, &s);
  const int N = L.N;
  const int64_t t = s / N;
  const int n = (int)(s % N);
  const int a = L.t_a[t];
  double s_in, s_out;
  otf_clip(tg, s_in, s_out);
  const bool up = tg.cot > 0;
  int64_t t2;
  int n2, dir2;
  double z_exit, s2;
  if (dir == 0) {
    if (s_out < tg.L) {  // axial exit through z+ (up) or z- (down)
      int face = up ? 5 : 4;
      if (!g.bc[face]) return -1;
      t2 = t;
      n2 = N - 1 - n;
      dir2 = 0;
      z_exit = up ? g.Z : 0.0;
      s2 = s_out;
    } else {
      int face = L.t_fend[t];
      if (!g.bc[face]) return -1;
      t2 = L.t_glf[t];
      bool ef = L.t_glf_fwd[t] != 0;
      n2 = ef ? n : N - 1 - n;
      dir2 = ef ? 0 : 1;
      z_exit = tg.z0 + tg.L * tg.cot;
      s2 = ef ? 0.0 : L.t_len[t2];
    }
  } else {
    if (s_in > 0.0) {  // axial exit through z- (up track going back) or z+
      int face = up ? 4 : 5;
      if (!g.bc[face]) return -1;
      t2 = t;
      n2 = N - 1 - n;
      dir2 = 1;
      z_exit = up ? 0.0 : g.Z;
      s2 = s_in;
    } else {
      int face = L.t_fstart[t];
      if (!g.bc[face]) return -1;
      t2 = L.t_glb[t];
      bool ef = L.t_glb_fwd[t] != 0;
      n2 = ef ? N - 1 - n : n;
      dir2 = ef ? 0 : 1;
      z_exit = tg.z0;
      s2 = ef ? 0.0 : L.t_len[t2];
    }
  }
  const int a2 = L.t_a[t2];
  const size_t an2 = (size_t)a2 * N + n2;
  const int64_t st2 = t2 * N + n2;
  const double x = (z_exit - L.st_z0[st2] - s2 * L.an_cot[an2]) / L.an_dz[an2];
  const double xr = std::nearbyint(x);
  if (std::fabs(x - xr) > 1e-6 || xr < 0 || xr >= (double)L.st_cnt[st2])
    throw Error(MOC_E_TRACE, "3D link of track " + std::to_string(track) + " dir " + std::to_string(dir) +
                                 " does not land on a stack member (residual " + std::to_string(x - xr) + ")");
  (void)a;
  return 2 * (L.st_first[st2] + (int64_t)xr) + dir2;
}

void links3d(const Geometry& g, const Laydown& L, int64_t* link) {
  std::string err;
#pragma omp parallel for schedule(static, 1024)
  for (int64_t tr = 0; tr < L.n3; ++tr) {
    for (int d = 0; d < 2; ++d) {
      try {
        link[2 * tr + d] = link_slot(g, L, tr, d);
      } catch (const Error& e) {
#pragma omp critical
        err = e.what();
        link[2 * tr + d] = -2;
      }
    }
  }
  if (!err.empty()) throw Error(MOC_E_TRACE, err);
}

}  // namespace moc
