// moc_oracle.cpp — plain, slow, fp64 CPU oracle for the OTF 3D MOC sweep of
// arXiv 2503.17743 and the power iteration around it.
//
// TEST INFRASTRUCTURE ONLY (see moc_oracle.h).  Shares no code with the product.
//
// Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
// "App. A.x" = SURVEY.md Appendix A (the laydown spec the paper is silent on),
// "Qn" = SURVEY.md §8(c) readings (listed again in DESIGN.md).
//
// What is deliberately NOT used here: the paper's OTF formulas Eqs. 5-11
// (P:70-120).  3D segments are found by brute force: each 3D track is an
// explicit 3D line clipped to the box, its crossing parameters are the union
// of its projection's 2D segment boundaries and the axial planes, sorted,
// epsilon-merged, and classified by midpoint.  Links are
// found by geometric matching of exit/entry points, not by index arithmetic.
//
// Parity pins: see tests/test_oracle_*.py and DESIGN.md §"Oracle pins".

#include "moc_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <omp.h>

namespace {

const double kEpsL = 1e-6;                  // App. A.7 epsilon_L (cm)
const double kPi = 3.14159265358979323846;  // pi
// Stack phase offset as a fraction of dz (reading Q7b): the golden-ratio
// fraction instead of 1/2 keeps 3D track ends off the box edges in symmetric layouts.
const double kPhaseFrac = 0.6180339887498949;

struct Err {
  std::string msg;
};

// ---------------------------------------------------------------------------
// epsilon-merge of a sorted boundary list (App. A.7; readings Q22, Q22b):
// every raw segment shorter than eps joins the preceding merged segment; the
// leading run of short raw segments joins the first long one (so the merged
// list read backwards is the merge of the reversed raw list).  Returns merged
// intervals.
// ---------------------------------------------------------------------------
void merge_segments(const std::vector<double>& b, std::vector<std::pair<double, double>>& out) {
  out.clear();
  bool lead = true;  // everything merged so far is a run of short raw segments
  for (size_t q = 0; q + 1 < b.size(); ++q) {
    double a0 = b[q], a1 = b[q + 1];
    double len = a1 - a0;
    if (out.empty()) {
      out.push_back({a0, a1});
      lead = len < kEpsL;
    } else if (len < kEpsL) {
      out.back().second = a1;
    } else if (lead) {
      out.back().second = a1;  // leading short run merges forward
      lead = false;
    } else {
      out.push_back({a0, a1});
    }
  }
}

uint64_t fnv1a_u32_seq(const std::vector<int64_t>& ids) {
  uint64_t h = 14695981039346656037ull;
  for (int64_t v : ids) {
    uint32_t u = (uint32_t)v;
    for (int b = 0; b < 4; ++b) {
      h ^= (uint64_t)((u >> (8 * b)) & 0xffu);
      h *= 1099511628211ull;
    }
  }
  return h;
}

// Gauss-Legendre nodes/weights on [-1,1] by Newton iteration on P_N.
// Returned with mu descending (n = 0 is the smallest polar angle theta).
void gauss_legendre(int N, std::vector<double>& mu, std::vector<double>& w) {
  mu.assign(N, 0.0);
  w.assign(N, 0.0);
  for (int i = 0; i < N; ++i) {
    double x = std::cos(kPi * (i + 0.75) / (N + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= N; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      // p1 = P_N(x), p0 = P_{N-1}(x)
      double dp = N * (x * p1 - p0) / (x * x - 1.0);
      double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    double p0 = 1.0, p1 = x;
    for (int k = 2; k <= N; ++k) {
      double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    double dp = N * (x * p1 - p0) / (x * x - 1.0);
    mu[i] = x;
    w[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  // sort descending in mu
  std::vector<int> idx(N);
  for (int i = 0; i < N; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return mu[a] > mu[b]; });
  std::vector<double> m2(N), w2(N);
  for (int i = 0; i < N; ++i) {
    m2[i] = mu[idx[i]];
    w2[i] = w[idx[i]];
  }
  mu = m2;
  w = w2;
}

struct Track2 {
  int a;
  double x0, y0, x1, y1, L, ux, uy;
  int f_start, f_end;
  int64_t sb, se;          // segment range [sb, se)
  int64_t glf, glb;        // geometric link targets (all faces reflective)
  int glf_fwd, glb_fwd;    // target entered forward?
  int64_t cyc;
  double lt;               // cycle arc length of the s = 0 point
  int sig;                 // +1 forward in its cycle, -1 backward
};

struct PointKey {
  uint64_t key;
  int64_t id;
  bool operator<(const PointKey& o) const { return key < o.key || (key == o.key && id < o.id); }
};

uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t cell_key(int64_t qx, int64_t qy, int64_t qz) {
  return mix64((uint64_t)qx * 0x100000001b3ull ^ mix64((uint64_t)qy + 0x51ull) ^ mix64((uint64_t)qz * 7 + 3));
}

const double kQuant = 1e6;  // point-matching grid: 1e-6 cm cells, neighbours probed

struct Oracle {
  // --- problem copy ---
  int nx = 0, ny = 0;
  double px = 0, py = 0;
  std::vector<int32_t> cell_type;
  int n_types = 0, max_rings = 0;
  std::vector<int32_t> n_rings;
  std::vector<double> radii;
  int NL = 0;
  std::vector<double> planes;
  int n_zones = 0;
  std::vector<int32_t> zone_of_layer;
  std::vector<int32_t> material;
  int bc[6] = {1, 1, 1, 1, 1, 1};
  int n_mat = 0, G = 0;
  std::vector<double> sigt, sigs, nusf, chi;
  int M = 0, N = 0;
  double dr = 0, dzs = 0;
  // --- derived ---
  double W = 0, Y = 0, Z = 0;
  std::vector<int64_t> prefix;  // region prefix per cell
  int64_t n_regions = 0, n_fsr = 0;
  std::vector<double> phi_a, delta_a, omega_a;
  std::vector<int32_t> nx_a, ny_a;
  std::vector<Track2> t2;
  std::vector<int64_t> seg_region;
  std::vector<double> seg_send;
  int64_t n_cycles = 0;
  std::vector<double> cycle_len_a;  // per family
  std::vector<double> mu, wgl;
  // per (a, n)
  std::vector<double> theta, dz, wgt, aperp, sth, cth;
  // stacks (t, n)
  std::vector<double> z0b;
  std::vector<int64_t> cnt, first;
  int64_t n3 = 0;
  int64_t n_degenerate = 0;
  // segment cache (optional)
  bool cached = false;
  std::vector<int64_t> c_off;
  std::vector<int32_t> c_fsr;
  std::vector<double> c_len;
  std::vector<double> vol_track;
  bool have_vol = false;
  std::vector<int64_t> link3;
  bool have_links = false;

  int64_t region_of(double x, double y) const {
    int cx = (int)std::floor(x / px), cy = (int)std::floor(y / py);
    cx = std::min(std::max(cx, 0), nx - 1);
    cy = std::min(std::max(cy, 0), ny - 1);
    int c = cy * nx + cx;
    int ty = cell_type[c];
    double ddx = x - (cx + 0.5) * px, ddy = y - (cy + 0.5) * py;
    double d2 = ddx * ddx + ddy * ddy;
    int local = n_rings[ty];
    for (int q = 0; q < n_rings[ty]; ++q) {
      double r = radii[(size_t)ty * max_rings + q];
      if (d2 < r * r) {
        local = q;
        break;
      }
    }
    return prefix[c] + local;
  }
  int layer_of(double z) const {
    for (int l = 0; l < NL; ++l)
      if (z < planes[l + 1]) return l;
    return NL - 1;
  }
  int mat_of_fsr(int64_t j) const {
    int64_t r = j / NL;
    int l = (int)(j % NL);
    // find cell of region r
    int64_t c = std::upper_bound(prefix.begin(), prefix.end(), r) - prefix.begin() - 1;
    int ty = cell_type[c];
    int local = (int)(r - prefix[c]);
    return material[((size_t)ty * (max_rings + 1) + local) * n_zones + zone_of_layer[l]];
  }

  // --------------------------------------------------------------- 2D laydown
  void laydown2d() {
    if (M < 4 || M % 4 != 0) throw Err{"num_azim must be a positive multiple of 4"};
    if (dr <= 0 || dr > std::min(W, Y)) throw Err{"radial spacing must be in (0, min(W,Y)]"};
    int Q = M / 4;
    phi_a.assign(M / 2, 0);
    delta_a.assign(M / 2, 0);
    omega_a.assign(M / 2, 0);
    nx_a.assign(M / 2, 0);
    ny_a.assign(M / 2, 0);
    for (int a = 0; a < Q; ++a) {
      // App. A.1: desired angle, integer counts, corrected angle
      double phs = 2.0 * kPi / M * (a + 0.5);
      int nxa = (int)std::floor(W * std::sin(phs) / dr) + 1;
      int nya = (int)std::floor(Y * std::cos(phs) / dr) + 1;
      double ph = std::atan((Y * nxa) / (W * nya));
      double ddx = W / nxa;
      int ac = M / 2 - 1 - a;
      phi_a[a] = ph;
      phi_a[ac] = kPi - ph;
      nx_a[a] = nx_a[ac] = nxa;
      ny_a[a] = ny_a[ac] = nya;
      delta_a[a] = delta_a[ac] = ddx * std::sin(ph);
    }
    // weights from angular bisectors in the first quadrant (App. A.1)
    for (int a = 0; a < Q; ++a) {
      double blo = (a == 0) ? 0.0 : 0.5 * (phi_a[a - 1] + phi_a[a]);
      double bhi = (a == Q - 1) ? 0.5 * kPi : 0.5 * (phi_a[a] + phi_a[a + 1]);
      omega_a[a] = omega_a[M / 2 - 1 - a] = (bhi - blo) / (2.0 * kPi);
    }
    // tracks, family-major
    t2.clear();
    for (int a = 0; a < M / 2; ++a) {
      int asrc = (a < Q) ? a : (M / 2 - 1 - a);
      bool mirror = (a >= Q);
      double ph = phi_a[asrc];
      double cph = std::cos(ph), sph = std::sin(ph);
      int nxa = nx_a[a], nya = ny_a[a];
      double ddx = W / nxa, ddy = Y / nya;
      struct S {
        double u, x, y;
      };
      std::vector<S> st;
      for (int j = 0; j < nya; ++j) {
        double y = ddy * (j + 0.5);
        st.push_back({0.0 * sph - y * cph, 0.0, y});
      }
      for (int i = 0; i < nxa; ++i) {
        double x = ddx * (i + 0.5);
        st.push_back({x * sph - 0.0 * cph, x, 0.0});
      }
      std::sort(st.begin(), st.end(), [](const S& p, const S& q) { return p.u < q.u; });
      for (const S& s : st) {
        Track2 t{};
        t.a = a;
        double x0 = mirror ? (W - s.x) : s.x;
        double y0 = s.y;
        double ux = mirror ? -cph : cph, uy = sph;
        t.x0 = x0;
        t.y0 = y0;
        t.ux = ux;
        t.uy = uy;
        double tx = (ux > 0) ? (W - x0) / ux : (0.0 - x0) / ux;
        double ty = (Y - y0) / uy;
        if (tx < ty) {
          t.L = tx;
          t.f_end = (ux > 0) ? 1 : 0;
        } else {
          t.L = ty;
          t.f_end = 3;
        }
        t.x1 = x0 + t.L * ux;
        t.y1 = y0 + t.L * uy;
        if (t.f_end == 1) t.x1 = W;
        if (t.f_end == 0) t.x1 = 0.0;
        if (t.f_end == 3) t.y1 = Y;
        if (y0 == 0.0)
          t.f_start = 2;
        else
          t.f_start = (x0 == 0.0) ? 0 : 1;
        t2.push_back(t);
      }
    }
  }

  // brute-force 2D segmentation of one line: every lattice line and every circle (App. A.7)
  void segment_line(double x0, double y0, double ux, double uy, double L, std::vector<int64_t>& reg,
                    std::vector<double>& send) const {
    std::vector<double> b;
    std::vector<std::pair<double, double>> mg;
    Track2 t{};
    t.x0 = x0;
    t.y0 = y0;
    t.ux = ux;
    t.uy = uy;
    t.L = L;
    {
      b.clear();
      b.push_back(0.0);
      b.push_back(t.L);
      for (int i = 0; i <= nx; ++i) {
        double u = (i * px - t.x0) / t.ux;
        if (u > 0.0 && u < t.L) b.push_back(u);
      }
      for (int j = 0; j <= ny; ++j) {
        double u = (j * py - t.y0) / t.uy;
        if (u > 0.0 && u < t.L) b.push_back(u);
      }
      for (int cy = 0; cy < ny; ++cy)
        for (int cx = 0; cx < nx; ++cx) {
          int ty = cell_type[cy * nx + cx];
          double ccx = (cx + 0.5) * px, ccy = (cy + 0.5) * py;
          double wx = ccx - t.x0, wy = ccy - t.y0;
          double proj = wx * t.ux + wy * t.uy;
          double d2 = wx * wx + wy * wy - proj * proj;
          for (int q = 0; q < n_rings[ty]; ++q) {
            double r = radii[(size_t)ty * max_rings + q];
            if (d2 >= r * r) continue;
            double half = std::sqrt(r * r - d2);
            if (2.0 * half <= kEpsL) continue;  // chord must exceed epsilon_L
            double u1 = proj - half, u2 = proj + half;
            if (u1 > 0.0 && u1 < t.L) b.push_back(u1);
            if (u2 > 0.0 && u2 < t.L) b.push_back(u2);
          }
        }
      std::sort(b.begin(), b.end());
      merge_segments(b, mg);
      reg.clear();
      send.clear();
      for (auto& iv : mg) {
        double um = 0.5 * (iv.first + iv.second);
        reg.push_back(region_of(t.x0 + um * t.ux, t.y0 + um * t.uy));
        send.push_back(iv.second);
      }
      send.back() = t.L;
    }
  }
  void segment2d() {
    seg_region.clear();
    seg_send.clear();
    std::vector<int64_t> reg;
    std::vector<double> send;
    for (auto& t : t2) {
      segment_line(t.x0, t.y0, t.ux, t.uy, t.L, reg, send);
      t.sb = (int64_t)seg_region.size();
      seg_region.insert(seg_region.end(), reg.begin(), reg.end());
      seg_send.insert(seg_send.end(), send.begin(), send.end());
      t.se = (int64_t)seg_region.size();
    }
  }

  // geometric 2D links: reflect the exit direction on the exit face and find the
  // track whose start (forward) or end (backward) is at the same point with that
  // direction.
  void links2d() {
    std::vector<PointKey> pk;
    auto qk = [&](double x, double y) {
      return cell_key(std::llround(x * kQuant), std::llround(y * kQuant), 0);
    };
    for (int64_t t = 0; t < (int64_t)t2.size(); ++t) {
      pk.push_back({qk(t2[t].x0, t2[t].y0), 2 * t});      // entry forward at start
      pk.push_back({qk(t2[t].x1, t2[t].y1), 2 * t + 1});  // entry backward at end
    }
    std::sort(pk.begin(), pk.end());
    auto find = [&](double x, double y, double dx, double dy, int64_t& tgt, int& fwd) {
      int64_t qx = std::llround(x * kQuant), qy = std::llround(y * kQuant);
      double best = 1e-8;
      tgt = -1;
      for (int ox = -1; ox <= 1; ++ox)
        for (int oy = -1; oy <= 1; ++oy) {
          uint64_t k = cell_key(qx + ox, qy + oy, 0);
          auto it = std::lower_bound(pk.begin(), pk.end(), PointKey{k, INT64_MIN});
          for (; it != pk.end() && it->key == k; ++it) {
            int64_t tt = it->id / 2;
            bool f = (it->id % 2) == 0;
            double ex = f ? t2[tt].x0 : t2[tt].x1, ey = f ? t2[tt].y0 : t2[tt].y1;
            double ddx = f ? t2[tt].ux : -t2[tt].ux, ddy = f ? t2[tt].uy : -t2[tt].uy;
            double dist = std::hypot(ex - x, ey - y);
            if (dist < best && std::fabs(ddx - dx) < 1e-9 && std::fabs(ddy - dy) < 1e-9) {
              best = dist;
              tgt = tt;
              fwd = f ? 1 : 0;
            }
          }
        }
    };
    for (int64_t t = 0; t < (int64_t)t2.size(); ++t) {
      Track2& T = t2[t];
      // forward exit at (x1, y1), direction (ux, uy)
      double dx = T.ux, dy = T.uy;
      if (T.f_end <= 1) dx = -dx; else dy = -dy;
      find(T.x1, T.y1, dx, dy, T.glf, T.glf_fwd);
      // backward exit at (x0, y0), direction (-ux, -uy)
      dx = -T.ux;
      dy = -T.uy;
      if (T.f_start <= 1) dx = -dx; else dy = -dy;
      find(T.x0, T.y0, dx, dy, T.glb, T.glb_fwd);
      if (T.glf < 0 || T.glb < 0) throw Err{"2D link not found for track " + std::to_string(t)};
    }
  }

  void cycles2d() {
    std::vector<char> vis(t2.size(), 0);
    cycle_len_a.assign(M / 2, -1.0);
    n_cycles = 0;
    for (int64_t t0 = 0; t0 < (int64_t)t2.size(); ++t0) {
      if (vis[t0]) continue;
      int64_t cur = t0;
      bool fwd = true;
      double cum = 0.0;
      std::vector<int64_t> members;
      while (true) {
        if (vis[cur]) throw Err{"2D cycle revisits a track"};
        vis[cur] = 1;
        members.push_back(cur);
        Track2& T = t2[cur];
        T.cyc = n_cycles;
        T.sig = fwd ? 1 : -1;
        T.lt = fwd ? cum : cum + T.L;
        cum += T.L;
        int64_t nxt = fwd ? T.glf : T.glb;
        int nf = fwd ? T.glf_fwd : T.glb_fwd;
        cur = nxt;
        fwd = nf != 0;
        if (cur == t0) {
          if (!fwd) throw Err{"2D cycle returns to its first track backward"};
          break;
        }
      }
      for (int64_t m : members) {
        int a = t2[m].a;
        if (cycle_len_a[a] < 0) cycle_len_a[a] = cum;
        else if (std::fabs(cycle_len_a[a] - cum) > 1e-9 * cum) throw Err{"unequal cycle lengths in a family"};
      }
      ++n_cycles;
    }
  }

  // ------------------------------------------------------------- 3D stacks
  void stacks3d() {
    gauss_legendre(N, mu, wgl);
    theta.assign((size_t)(M / 2) * N, 0);
    dz.assign(theta.size(), 0);
    wgt.assign(theta.size(), 0);
    aperp.assign(theta.size(), 0);
    sth.assign(theta.size(), 0);
    cth.assign(theta.size(), 0);
    for (int a = 0; a < M / 2; ++a) {
      double LC = cycle_len_a[a];
      for (int n = 0; n < N / 2; ++n) {
        double ths = std::acos(mu[n]);
        int nz = (int)std::floor(Z * std::sin(ths) / dzs) + 1;
        int nl = (int)std::floor(LC * std::cos(ths) / dzs) + 1;
        double Dz = Z / nz, Dl = LC / nl;
        double th = std::atan(Dl / Dz);
        size_t u = (size_t)a * N + n, l = (size_t)a * N + (N - 1 - n);
        theta[u] = th;
        theta[l] = kPi - th;
        dz[u] = dz[l] = Dz;
      }
      for (int n = 0; n < N; ++n) {
        size_t u = (size_t)a * N + n;
        sth[u] = std::sin(theta[u]);
        cth[u] = std::cos(theta[u]);
        wgt[u] = 4.0 * kPi * omega_a[a] * (wgl[n] / 2.0);        // App. A.5
        aperp[u] = delta_a[a] * dz[u] * sth[u];
      }
    }
    size_t ns = t2.size() * (size_t)N;
    z0b.assign(ns, 0);
    cnt.assign(ns, 0);
    first.assign(ns + 1, 0);
    n_degenerate = 0;
    auto near_int = [](double x) { return std::fabs(x - std::round(x)) < 1e-9; };
    for (size_t t = 0; t < t2.size(); ++t) {
      const Track2& T = t2[t];
      for (int n = 0; n < N; ++n) {
        size_t an = (size_t)T.a * N + n;
        int nu = (n < N / 2) ? n : (N - 1 - n);
        size_t anu = (size_t)T.a * N + nu;
        double cot_u = cth[anu] / sth[anu];
        double ph = T.sig * (T.lt * cot_u - kPhaseFrac * dz[anu]);  // App. A.4 phase (reading Q7b)
        if (n >= N / 2) ph = -ph;
        double c = cth[an] / sth[an];
        double D = dz[an];
        double lo, hi;
        if (c > 0) {
          lo = (-T.L * c - ph) / D;
          hi = (Z - ph) / D;
        } else {
          lo = (-ph) / D;
          hi = (Z - T.L * c - ph) / D;
        }
        if (near_int(lo) || near_int(hi)) ++n_degenerate;
        int64_t mlo = (int64_t)std::floor(lo) + 1, mhi = (int64_t)std::ceil(hi) - 1;
        size_t s = t * N + n;
        cnt[s] = std::max<int64_t>(0, mhi - mlo + 1);
        z0b[s] = ph + mlo * D;
      }
    }
    for (size_t s = 0; s < ns; ++s) first[s + 1] = first[s] + cnt[s];
    n3 = first[ns];
  }

  // ------------------------------------------------------- 3D explicit trace
  struct Geo3 {
    int64_t t;
    int n;
    double z0, s, c;  // sin, cos
    double uin, uout, uhi, ua, ub;
  };
  void geo3(int64_t id, Geo3& g) const {
    int64_t s = std::upper_bound(first.begin(), first.end(), id) - first.begin() - 1;
    g.t = s / N;
    g.n = (int)(s % N);
    int64_t i = id - first[s];
    size_t an = (size_t)t2[g.t].a * N + g.n;
    g.z0 = z0b[s] + i * dz[an];
    g.s = sth[an];
    g.c = cth[an];
    g.uhi = t2[g.t].L / g.s;
    if (g.c > 0) {
      g.ua = (0.0 - g.z0) / g.c;
      g.ub = (Z - g.z0) / g.c;
    } else {
      g.ua = (Z - g.z0) / g.c;
      g.ub = (0.0 - g.z0) / g.c;
    }
    g.uin = std::max(0.0, g.ua);
    g.uout = std::min(g.uhi, g.ub);
  }
  void trace3d(int64_t id, std::vector<int64_t>& fsr, std::vector<double>& len, std::vector<double>& b,
               std::vector<std::pair<double, double>>& mg) const {
    Geo3 g;
    geo3(id, g);
    const Track2& T = t2[g.t];
    b.clear();
    b.push_back(g.uin);
    for (int64_t k = T.sb; k + 1 < T.se; ++k) {
      double u = seg_send[k] / g.s;
      if (u > g.uin && u < g.uout) b.push_back(u);
    }
    for (int l = 1; l < NL; ++l) {
      double u = (planes[l] - g.z0) / g.c;
      if (u > g.uin && u < g.uout) b.push_back(u);
    }
    b.push_back(g.uout);
    std::sort(b.begin(), b.end());
    merge_segments(b, mg);
    fsr.clear();
    len.clear();
    for (auto& iv : mg) {
      double um = 0.5 * (iv.first + iv.second);
      double sm = um * g.s;
      int64_t k = std::upper_bound(seg_send.begin() + T.sb, seg_send.begin() + T.se, sm) - seg_send.begin();
      if (k >= T.se) k = T.se - 1;
      int l = layer_of(g.z0 + um * g.c);
      fsr.push_back(seg_region[k] * NL + l);
      len.push_back(iv.second - iv.first);
    }
  }

  void build_cache() {
    const char* env = std::getenv("ORACLE_SEG_CACHE_GB");
    double budget = env ? std::atof(env) : 12.0;
    // count first
    std::vector<int64_t> ns(n3);
#pragma omp parallel
    {
      std::vector<int64_t> f;
      std::vector<double> l, b;
      std::vector<std::pair<double, double>> mg;
#pragma omp for schedule(dynamic, 256)
      for (int64_t id = 0; id < n3; ++id) {
        trace3d(id, f, l, b, mg);
        ns[id] = (int64_t)f.size();
      }
    }
    c_off.assign(n3 + 1, 0);
    for (int64_t id = 0; id < n3; ++id) c_off[id + 1] = c_off[id] + ns[id];
    double gb = c_off[n3] * 12.0 / 1e9;
    if (gb > budget) {
      cached = false;
      return;
    }
    c_fsr.resize(c_off[n3]);
    c_len.resize(c_off[n3]);
#pragma omp parallel
    {
      std::vector<int64_t> f;
      std::vector<double> l, b;
      std::vector<std::pair<double, double>> mg;
#pragma omp for schedule(dynamic, 256)
      for (int64_t id = 0; id < n3; ++id) {
        trace3d(id, f, l, b, mg);
        for (size_t q = 0; q < f.size(); ++q) {
          c_fsr[c_off[id] + q] = (int32_t)f[q];
          c_len[c_off[id] + q] = l[q];
        }
      }
    }
    cached = true;
  }

  double weight_c(int64_t id) const {
    int64_t s = std::upper_bound(first.begin(), first.end(), id) - first.begin() - 1;
    int64_t t = s / N;
    int n = (int)(s % N);
    size_t an = (size_t)t2[t].a * N + n;
    return wgt[an] * aperp[an];
  }

  void volumes() {
    if (have_vol) return;
    int nth = omp_get_max_threads();
    std::vector<std::vector<double>> part(nth, std::vector<double>(n_fsr, 0.0));
#pragma omp parallel
    {
      std::vector<int64_t> f;
      std::vector<double> l, b;
      std::vector<std::pair<double, double>> mg;
      std::vector<double>& v = part[omp_get_thread_num()];
#pragma omp for schedule(static)
      for (int64_t id = 0; id < n3; ++id) {
        trace3d(id, f, l, b, mg);
        int64_t s = std::upper_bound(first.begin(), first.end(), id) - first.begin() - 1;
        size_t an = (size_t)t2[s / N].a * N + (s % N);
        double w = wgt[an] / (2.0 * kPi) * aperp[an];  // App. A.5
        for (size_t q = 0; q < f.size(); ++q) v[f[q]] += w * l[q];
      }
    }
    vol_track.assign(n_fsr, 0.0);
    for (int th = 0; th < nth; ++th)
      for (int64_t j = 0; j < n_fsr; ++j) vol_track[j] += part[th][j];
    have_vol = true;
  }

  // geometric 3D links (independent of the A.4 index arithmetic)
  void links3d() {
    if (have_links) return;
    std::vector<PointKey> pk((size_t)2 * n3);
    auto entry = [&](int64_t slot, double& x, double& y, double& z, double& dx, double& dy, double& dzz) {
      Geo3 g;
      geo3(slot / 2, g);
      const Track2& T = t2[g.t];
      bool fwd = (slot % 2) == 0;
      double u = fwd ? g.uin : g.uout;
      double sg = u * g.s;
      x = T.x0 + sg * T.ux;
      y = T.y0 + sg * T.uy;
      z = g.z0 + u * g.c;
      dx = g.s * T.ux;
      dy = g.s * T.uy;
      dzz = g.c;
      if (!fwd) {
        dx = -dx;
        dy = -dy;
        dzz = -dzz;
      }
    };
#pragma omp parallel for schedule(static)
    for (int64_t slot = 0; slot < 2 * n3; ++slot) {
      double x, y, z, a, b, c;
      entry(slot, x, y, z, a, b, c);
      pk[slot] = {cell_key(std::llround(x * kQuant), std::llround(y * kQuant), std::llround(z * kQuant)), slot};
    }
    std::sort(pk.begin(), pk.end());
    link3.assign((size_t)2 * n3, -1);
    int64_t missing = 0;
#pragma omp parallel for schedule(static) reduction(+ : missing)
    for (int64_t slot = 0; slot < 2 * n3; ++slot) {
      Geo3 g;
      geo3(slot / 2, g);
      const Track2& T = t2[g.t];
      bool fwd = (slot % 2) == 0;
      double u = fwd ? g.uout : g.uin;
      double sg = u * g.s;
      double x = T.x0 + sg * T.ux, y = T.y0 + sg * T.uy, z = g.z0 + u * g.c;
      double dx = g.s * T.ux, dy = g.s * T.uy, dzz = g.c;
      if (!fwd) {
        dx = -dx;
        dy = -dy;
        dzz = -dzz;
      }
      int face;
      if (fwd) face = (g.uhi < g.ub) ? T.f_end : (g.c > 0 ? 5 : 4);
      else face = (0.0 > g.ua) ? T.f_start : (g.c > 0 ? 4 : 5);
      if (face <= 1) dx = -dx;
      else if (face <= 3) dy = -dy;
      else dzz = -dzz;
      if (bc[face] == 0) {
        link3[slot] = -1;
        continue;
      }
      int64_t qx = std::llround(x * kQuant), qy = std::llround(y * kQuant), qz = std::llround(z * kQuant);
      double best = 1e-8;
      int64_t tgt = -1;
      for (int ox = -1; ox <= 1; ++ox)
        for (int oy = -1; oy <= 1; ++oy)
          for (int oz = -1; oz <= 1; ++oz) {
            uint64_t k = cell_key(qx + ox, qy + oy, qz + oz);
            auto it = std::lower_bound(pk.begin(), pk.end(), PointKey{k, INT64_MIN});
            for (; it != pk.end() && it->key == k; ++it) {
              double ex, ey, ez, ea, eb, ec;
              entry(it->id, ex, ey, ez, ea, eb, ec);
              double dist = std::sqrt((ex - x) * (ex - x) + (ey - y) * (ey - y) + (ez - z) * (ez - z));
              if (dist < best && std::fabs(ea - dx) < 1e-9 && std::fabs(eb - dy) < 1e-9 &&
                  std::fabs(ec - dzz) < 1e-9) {
                best = dist;
                tgt = it->id;
              }
            }
          }
      if (tgt < 0) ++missing;
      link3[slot] = tgt;
    }
    if (missing) throw Err{"3D links: " + std::to_string(missing) + " reflective exits without a matching entry"};
    have_links = true;
  }
};

void copy_problem(Oracle& o, const or_problem* p) {
  o.nx = p->nx;
  o.ny = p->ny;
  o.px = p->pitch_x;
  o.py = p->pitch_y;
  o.cell_type.assign(p->cell_type, p->cell_type + (size_t)p->nx * p->ny);
  o.n_types = p->n_types;
  o.max_rings = p->max_rings;
  o.n_rings.assign(p->n_rings, p->n_rings + p->n_types);
  if (p->max_rings > 0) o.radii.assign(p->radii, p->radii + (size_t)p->n_types * p->max_rings);
  o.NL = p->n_layers;
  o.planes.assign(p->planes, p->planes + p->n_layers + 1);
  o.n_zones = p->n_zones;
  o.zone_of_layer.assign(p->zone_of_layer, p->zone_of_layer + p->n_layers);
  o.material.assign(p->material, p->material + (size_t)p->n_types * (p->max_rings + 1) * p->n_zones);
  for (int f = 0; f < 6; ++f) o.bc[f] = p->bc[f];
  o.n_mat = p->n_mat;
  o.G = p->G;
  o.sigt.assign(p->sigma_t, p->sigma_t + (size_t)p->n_mat * p->G);
  o.sigs.assign(p->sigma_s, p->sigma_s + (size_t)p->n_mat * p->G * p->G);
  o.nusf.assign(p->nu_sigma_f, p->nu_sigma_f + (size_t)p->n_mat * p->G);
  o.chi.assign(p->chi, p->chi + (size_t)p->n_mat * p->G);
  o.M = p->num_azim;
  o.N = p->num_polar;
  o.dr = p->radial_spacing;
  o.dzs = p->axial_spacing;
}

void set_err(char* err, int64_t n, const std::string& s) {
  if (err && n > 0) {
    std::snprintf(err, (size_t)n, "%s", s.c_str());
  }
}

}  // namespace

extern "C" {

void* or_create(const or_problem* p, char* err, int64_t errlen) {
  Oracle* o = new Oracle();
  try {
    copy_problem(*o, p);
    if (o->planes[0] != 0.0) throw Err{"planes[0] must be 0"};
    for (int l = 0; l < o->NL; ++l)
      if (!(o->planes[l + 1] > o->planes[l])) throw Err{"axial planes must be strictly increasing"};
    if (o->N < 2 || o->N % 2) throw Err{"num_polar must be even and >= 2"};
    o->W = o->nx * o->px;
    o->Y = o->ny * o->py;
    o->Z = o->planes[o->NL];
    o->prefix.assign((size_t)o->nx * o->ny + 1, 0);
    for (int c = 0; c < o->nx * o->ny; ++c) o->prefix[c + 1] = o->prefix[c] + o->n_rings[o->cell_type[c]] + 1;
    o->n_regions = o->prefix[(size_t)o->nx * o->ny];
    o->n_fsr = o->n_regions * o->NL;
    for (int m = 0; m < o->n_mat; ++m)
      for (int g = 0; g < o->G; ++g)
        if (!(o->sigt[(size_t)m * o->G + g] > 0)) throw Err{"sigma_t must be > 0"};
    o->laydown2d();
    o->segment2d();
    o->links2d();
    o->cycles2d();
    o->stacks3d();
  } catch (const Err& e) {
    set_err(err, errlen, e.msg);
    delete o;
    return nullptr;
  }
  return o;
}

void or_destroy(void* h) { delete (Oracle*)h; }

void or_get_counts(void* h, or_counts* c) {
  Oracle* o = (Oracle*)h;
  c->n_fsr = o->n_fsr;
  c->n_regions = o->n_regions;
  c->n_tracks2d = (int64_t)o->t2.size();
  c->n_segs2d = (int64_t)o->seg_region.size();
  c->n_stacks = (int64_t)o->t2.size() * o->N;
  c->n_tracks3d = o->n3;
  c->n_cycles = o->n_cycles;
  c->n_degenerate = o->n_degenerate;
}

void or_get_tracks2d(void* h, int32_t* azim, double* xy0, double* xy1, double* length, int64_t* seg_off,
                     int64_t* link_fwd, int32_t* link_fwd_enters_fwd, int64_t* link_bwd,
                     int32_t* link_bwd_enters_fwd, int64_t* cycle, double* ltilde, int32_t* sigma) {
  Oracle* o = (Oracle*)h;
  for (size_t t = 0; t < o->t2.size(); ++t) {
    const Track2& T = o->t2[t];
    azim[t] = T.a;
    xy0[2 * t] = T.x0;
    xy0[2 * t + 1] = T.y0;
    xy1[2 * t] = T.x1;
    xy1[2 * t + 1] = T.y1;
    length[t] = T.L;
    seg_off[t] = T.sb;
    seg_off[t + 1] = T.se;
    link_fwd[t] = o->bc[T.f_end] ? T.glf : -1;
    link_fwd_enters_fwd[t] = T.glf_fwd;
    link_bwd[t] = o->bc[T.f_start] ? T.glb : -1;
    link_bwd_enters_fwd[t] = T.glb_fwd;
    cycle[t] = T.cyc;
    ltilde[t] = T.lt;
    sigma[t] = T.sig;
  }
}

void or_get_segments2d(void* h, int64_t* region, double* s_end) {
  Oracle* o = (Oracle*)h;
  for (size_t k = 0; k < o->seg_region.size(); ++k) {
    region[k] = o->seg_region[k];
    s_end[k] = o->seg_send[k];
  }
}

void or_get_azim(void* h, double* phi, int32_t* nx, int32_t* ny, double* delta, double* omega) {
  Oracle* o = (Oracle*)h;
  for (int a = 0; a < o->M / 2; ++a) {
    phi[a] = o->phi_a[a];
    nx[a] = o->nx_a[a];
    ny[a] = o->ny_a[a];
    delta[a] = o->delta_a[a];
    omega[a] = o->omega_a[a];
  }
}

void or_get_polar(void* h, double* theta, double* dz, double* wgt, double* aperp) {
  Oracle* o = (Oracle*)h;
  for (size_t u = 0; u < o->theta.size(); ++u) {
    theta[u] = o->theta[u];
    dz[u] = o->dz[u];
    wgt[u] = o->wgt[u];
    aperp[u] = o->aperp[u];
  }
}

void or_get_polar_gl(void* h, double* mu, double* w) {
  Oracle* o = (Oracle*)h;
  for (int n = 0; n < o->N; ++n) {
    mu[n] = o->mu[n];
    w[n] = o->wgl[n];
  }
}

void or_get_stacks(void* h, double* z0, int64_t* count, int64_t* first) {
  Oracle* o = (Oracle*)h;
  for (size_t s = 0; s < o->cnt.size(); ++s) {
    z0[s] = o->z0b[s];
    count[s] = o->cnt[s];
    first[s] = o->first[s];
  }
  first[o->cnt.size()] = o->first[o->cnt.size()];
}

int64_t or_trace3d(void* h, int64_t track, int64_t* fsr, double* len, int64_t cap) {
  Oracle* o = (Oracle*)h;
  std::vector<int64_t> f;
  std::vector<double> l, b;
  std::vector<std::pair<double, double>> mg;
  o->trace3d(track, f, l, b, mg);
  if ((int64_t)f.size() > cap) return -(int64_t)f.size();
  for (size_t q = 0; q < f.size(); ++q) {
    fsr[q] = f[q];
    len[q] = l[q];
  }
  return (int64_t)f.size();
}

void or_track_checksums(void* h, int64_t first, int64_t n, int32_t* nseg, uint64_t* hash, double* suml,
                        double* chord, uint64_t* rhash) {
  Oracle* o = (Oracle*)h;
#pragma omp parallel
  {
    std::vector<int64_t> f;
    std::vector<double> l, b;
    std::vector<std::pair<double, double>> mg;
#pragma omp for schedule(dynamic, 64)
    for (int64_t q = 0; q < n; ++q) {
      int64_t id = first + q;
      o->trace3d(id, f, l, b, mg);
      nseg[q] = (int32_t)f.size();
      hash[q] = fnv1a_u32_seq(f);
      if (rhash) {  // the same FNV-1a-64 over the ids in reverse order (backward travel)
        std::vector<int64_t> fr(f.rbegin(), f.rend());
        rhash[q] = fnv1a_u32_seq(fr);
      }
      double s = 0;
      for (double x : l) s += x;
      suml[q] = s;
      Oracle::Geo3 g;
      o->geo3(id, g);
      chord[q] = g.uout - g.uin;
    }
  }
}

int64_t or_total_segments3d(void* h) {
  Oracle* o = (Oracle*)h;
  int64_t tot = 0;
#pragma omp parallel reduction(+ : tot)
  {
    std::vector<int64_t> f;
    std::vector<double> l, b;
    std::vector<std::pair<double, double>> mg;
#pragma omp for schedule(dynamic, 256)
    for (int64_t id = 0; id < o->n3; ++id) {
      o->trace3d(id, f, l, b, mg);
      tot += (int64_t)f.size();
    }
  }
  return tot;
}

int or_links3d(void* h, int64_t* link, char* err, int64_t errlen) {
  Oracle* o = (Oracle*)h;
  try {
    o->links3d();
  } catch (const Err& e) {
    set_err(err, errlen, e.msg);
    return -1;
  }
  for (int64_t s = 0; s < 2 * o->n3; ++s) link[s] = o->link3[s];
  return 0;
}

void or_volumes(void* h, double* vol_track, double* vol_analytic) {
  Oracle* o = (Oracle*)h;
  o->volumes();
  for (int64_t j = 0; j < o->n_fsr; ++j) vol_track[j] = o->vol_track[j];
  if (vol_analytic) {
    for (int64_t j = 0; j < o->n_fsr; ++j) {
      int64_t r = j / o->NL;
      int l = (int)(j % o->NL);
      int64_t c = std::upper_bound(o->prefix.begin(), o->prefix.end(), r) - o->prefix.begin() - 1;
      int ty = o->cell_type[c];
      int local = (int)(r - o->prefix[c]);
      double area;
      if (local < o->n_rings[ty]) {
        double ro = o->radii[(size_t)ty * o->max_rings + local];
        double ri = local > 0 ? o->radii[(size_t)ty * o->max_rings + local - 1] : 0.0;
        area = kPi * (ro * ro - ri * ri);
      } else {
        double rl = o->n_rings[ty] > 0 ? o->radii[(size_t)ty * o->max_rings + o->n_rings[ty] - 1] : 0.0;
        area = o->px * o->py - kPi * rl * rl;
      }
      vol_analytic[j] = area * (o->planes[l + 1] - o->planes[l]);
    }
  }
}

void or_fsr_material(void* h, int32_t* mat) {
  Oracle* o = (Oracle*)h;
  for (int64_t j = 0; j < o->n_fsr; ++j) mat[j] = o->mat_of_fsr(j);
}

double or_attenuate(double psi_in, double q_over_sigma, double sigma_t, double s, double* delta_psi) {
  // Eq. 3: psi_out = psi_in e^{-s Sigma} + (Q/Sigma)(1 - e^{-s Sigma})
  double F = -std::expm1(-sigma_t * s);
  double d = (psi_in - q_over_sigma) * F;
  if (delta_psi) *delta_psi = d;
  return psi_in - d;
}

void or_source(int G, const double* phi, const double* sigma_t, const double* sigma_s, const double* nu_sigma_f,
               const double* chi, double k, double* qtilde) {
  // Q_g = (1/4pi)[chi_g/k sum_g' nuSf_g' phi_g' + sum_g' Ss_{g'->g} phi_g'];  qtilde = Q/Sigma_t
  double F = 0;
  for (int g = 0; g < G; ++g) F += nu_sigma_f[g] * phi[g];
  for (int g = 0; g < G; ++g) {
    double s = chi[g] * F / k;
    for (int gp = 0; gp < G; ++gp) s += sigma_s[gp * G + g] * phi[gp];
    qtilde[g] = s / (4.0 * kPi * sigma_t[g]);
  }
}

int or_solve(void* h, int fixed_iters, int max_iter, double tol_k, double tol_src, double* k_out, double* k_hist,
             double* res_hist, double* phi_out, double* leakage_out, double* production_out,
             double* absorption_out, char* err, int64_t errlen) {
  Oracle* o = (Oracle*)h;
  try {
    o->volumes();
    o->links3d();
    if (!o->cached) o->build_cache();
  } catch (const Err& e) {
    set_err(err, errlen, e.msg);
    return -1;
  }
  const int G = o->G;
  const int64_t J = o->n_fsr;
  std::vector<int32_t> mat(J);
  for (int64_t j = 0; j < J; ++j) mat[j] = o->mat_of_fsr(j);
  for (int64_t j = 0; j < J; ++j)
    if (!(o->vol_track[j] > 0)) {
      set_err(err, errlen, "FSR " + std::to_string(j) + " has zero track volume");
      return -1;
    }
  std::vector<double> phi((size_t)J * G, 1.0), qt((size_t)J * G), Fold(J), Fnew(J);
  std::vector<double> psi_in((size_t)2 * o->n3 * G, 0.0), psi_out((size_t)2 * o->n3 * G, 0.0);
  std::vector<double> cw(o->n3);
  for (int64_t id = 0; id < o->n3; ++id) cw[id] = o->weight_c(id);
  auto fission = [&](const std::vector<double>& ph, std::vector<double>& F) {
    for (int64_t j = 0; j < J; ++j) {
      double f = 0;
      for (int g = 0; g < G; ++g) f += o->nusf[(size_t)mat[j] * G + g] * ph[(size_t)j * G + g];
      F[j] = f;
    }
  };
  double k = 1.0;
  fission(phi, Fold);
  int nth = omp_get_max_threads();
  std::vector<std::vector<double>> tal(nth, std::vector<double>((size_t)J * G));
  int it = 0;
  double leak = 0;
  int limit = fixed_iters > 0 ? fixed_iters : max_iter;
  for (it = 0; it < limit; ++it) {
    // source update (reading Q2): qtilde = Q / Sigma_t, Q per steradian
    for (int64_t j = 0; j < J; ++j) {
      int m = mat[j];
      or_source(G, &phi[(size_t)j * G], &o->sigt[(size_t)m * G], &o->sigs[(size_t)m * G * G],
                &o->nusf[(size_t)m * G], &o->chi[(size_t)m * G], k, &qt[(size_t)j * G]);
    }
    for (auto& v : tal) std::fill(v.begin(), v.end(), 0.0);
    // transport sweep, Alg. 1 order, forward then backward per track (Q24)
#pragma omp parallel
    {
      std::vector<double>& T = tal[omp_get_thread_num()];
      std::vector<int64_t> f;
      std::vector<double> l, b;
      std::vector<std::pair<double, double>> mg;
      std::vector<double> psi(G);
#pragma omp for schedule(static, 64)
      for (int64_t id = 0; id < o->n3; ++id) {
        const int32_t* fs;
        const double* ls;
        int64_t nsg;
        std::vector<int32_t> f32;
        if (o->cached) {
          fs = &o->c_fsr[o->c_off[id]];
          ls = &o->c_len[o->c_off[id]];
          nsg = o->c_off[id + 1] - o->c_off[id];
        } else {
          o->trace3d(id, f, l, b, mg);
          f32.assign(f.begin(), f.end());
          fs = f32.data();
          ls = l.data();
          nsg = (int64_t)f.size();
        }
        double c = cw[id];
        for (int dir = 0; dir < 2; ++dir) {
          int64_t slot = 2 * id + dir;
          for (int g = 0; g < G; ++g) psi[g] = psi_in[(size_t)slot * G + g];
          for (int64_t q = 0; q < nsg; ++q) {
            int64_t qq = dir == 0 ? q : nsg - 1 - q;
            int64_t j = fs[qq];
            double L = ls[qq];
            int m = mat[j];
            for (int g = 0; g < G; ++g) {
              double F = -std::expm1(-o->sigt[(size_t)m * G + g] * L);   // Eq. 3
              double d = (psi[g] - qt[(size_t)j * G + g]) * F;
              psi[g] -= d;
              T[(size_t)j * G + g] += c * d;                                // Eq. 4 (Q1, Q2)
            }
          }
          for (int g = 0; g < G; ++g) psi_out[(size_t)slot * G + g] = psi[g];
        }
      }
    }
    // scalar flux (Q2): phi = 4 pi qtilde + T / (Sigma_t V)
    std::vector<double> phin((size_t)J * G);
    for (int64_t j = 0; j < J; ++j)
      for (int g = 0; g < G; ++g) {
        double t = 0;
        for (int th = 0; th < nth; ++th) t += tal[th][(size_t)j * G + g];
        double st = o->sigt[(size_t)mat[j] * G + g];
        phin[(size_t)j * G + g] = 4.0 * kPi * qt[(size_t)j * G + g] + t / (st * o->vol_track[j]);
      }
    fission(phin, Fnew);
    double pn = 0, po = 0;
    for (int64_t j = 0; j < J; ++j) {
      pn += o->vol_track[j] * Fnew[j];
      po += o->vol_track[j] * Fold[j];
    }
    if (!(pn > 0) || !(po > 0)) {
      set_err(err, errlen, "zero fission source");
      return -1;
    }
    double knew = k * pn / po;
    double sc = 1.0 / pn;  // normalisation sum V F = 1 (Q12)
    for (auto& v : phin) v *= sc;
    for (int64_t j = 0; j < J; ++j)
      for (int g = 0; g < G; ++g) {
        double v = phin[(size_t)j * G + g];
        if (!(v >= 0) || std::isnan(v)) {
          set_err(err, errlen, "negative or NaN flux in FSR " + std::to_string(j));
          return -1;
        }
      }
    // Jacobi boundary hand-off (Q9)
    std::fill(psi_in.begin(), psi_in.end(), 0.0);
    leak = 0;
    for (int64_t s = 0; s < 2 * o->n3; ++s) {
      int64_t t = o->link3[s];
      if (t >= 0) {
        for (int g = 0; g < G; ++g) psi_in[(size_t)t * G + g] = psi_out[(size_t)s * G + g] * sc;
      } else {
        double e = 0;
        for (int g = 0; g < G; ++g) e += psi_out[(size_t)s * G + g] * sc;
        leak += cw[s / 2] * e;
      }
    }
    fission(phin, Fnew);
    double r2 = 0;
    int64_t nf = 0;
    for (int64_t j = 0; j < J; ++j)
      if (Fnew[j] > 0) {
        double d = (Fnew[j] - Fold[j]) / Fnew[j];
        r2 += d * d;
        ++nf;
      }
    double res = nf ? std::sqrt(r2 / nf) : 0.0;
    double dk = std::fabs(knew - k);
    k = knew;
    phi.swap(phin);
    Fold = Fnew;
    if (k_hist) k_hist[it] = k;
    if (res_hist) res_hist[it] = res;
    if (fixed_iters <= 0 && dk < tol_k && res < tol_src) {
      ++it;
      break;
    }
  }
  *k_out = k;
  for (size_t q = 0; q < phi.size(); ++q) phi_out[q] = phi[q];
  double prod = 0, absn = 0;
  for (int64_t j = 0; j < J; ++j) {
    int m = mat[j];
    for (int g = 0; g < G; ++g) {
      double sa = o->sigt[(size_t)m * G + g];
      for (int gp = 0; gp < G; ++gp) sa -= o->sigs[((size_t)m * G + g) * G + gp];
      absn += o->vol_track[j] * sa * phi[(size_t)j * G + g];
      prod += o->vol_track[j] * o->nusf[(size_t)m * G + g] * phi[(size_t)j * G + g];
    }
  }
  if (leakage_out) *leakage_out = leak;
  if (production_out) *production_out = prod;
  if (absorption_out) *absorption_out = absn;
  return it;
}

double or_time_sample_sweep(void* h, int64_t stride, int nthreads, int64_t* integrations) {
  Oracle* o = (Oracle*)h;
  const int G = o->G;
  const int64_t J = o->n_fsr;
  std::vector<int32_t> mat(J);
  for (int64_t j = 0; j < J; ++j) mat[j] = o->mat_of_fsr(j);
  std::vector<double> qt((size_t)J * G, 1.0 / (4.0 * kPi));
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  std::vector<std::vector<double>> tal(nthreads, std::vector<double>((size_t)J * G, 0.0));
  int64_t nint = 0;
  auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(nthreads) reduction(+ : nint)
  {
    std::vector<double>& T = tal[omp_get_thread_num()];
    std::vector<int64_t> f;
    std::vector<double> l, b;
    std::vector<std::pair<double, double>> mg;
    std::vector<double> psi(G);
#pragma omp for schedule(dynamic, 16)
    for (int64_t id = 0; id < o->n3; id += stride) {
      o->trace3d(id, f, l, b, mg);
      double c = o->weight_c(id);
      for (int dir = 0; dir < 2; ++dir) {
        for (int g = 0; g < G; ++g) psi[g] = 0.0;
        int64_t nsg = (int64_t)f.size();
        for (int64_t q = 0; q < nsg; ++q) {
          int64_t qq = dir == 0 ? q : nsg - 1 - q;
          int64_t j = f[qq];
          int m = mat[j];
          for (int g = 0; g < G; ++g) {
            double F = -std::expm1(-o->sigt[(size_t)m * G + g] * l[qq]);
            double d = (psi[g] - qt[(size_t)j * G + g]) * F;
            psi[g] -= d;
            T[(size_t)j * G + g] += c * d;
          }
        }
      }
      nint += 2 * (int64_t)f.size() * G;
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  *integrations = nint;
  return std::chrono::duration<double>(t1 - t0).count();
}

int or_num_threads(void) { return omp_get_max_threads(); }

int64_t or_segment_line(void* h, double x0, double y0, double ux, double uy, double L, int64_t* region,
                        double* s_end, int64_t cap) {
  Oracle* o = (Oracle*)h;
  std::vector<int64_t> reg;
  std::vector<double> send;
  o->segment_line(x0, y0, ux, uy, L, reg, send);
  if ((int64_t)reg.size() > cap) return -(int64_t)reg.size();
  for (size_t q = 0; q < reg.size(); ++q) {
    region[q] = reg[q];
    s_end[q] = send[q];
  }
  return (int64_t)reg.size();
}

int64_t or_region_of(void* h, double x, double y) { return ((Oracle*)h)->region_of(x, y); }


}  // extern "C"
