// capi.cpp — problem-level entry points of libmoc3d.so (include/moc3d.h).
// Geometry/material setup, host laydown (A1/A2), debug exports and
// the paper's scalar formulas (Eqs. 5-7, 9-10, 13) and host scheduling rules
// (§4.2, §4.3).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include <omp.h>

#include "host.h"

using namespace moc;

#define MOC_TRY(p, ...)                           \
  try {                                           \
    __VA_ARGS__;                                  \
    return MOC_OK;                                \
  } catch (const Error& e) {                      \
    if (p) (p)->impl.err = e.what();              \
    return e.code;                                \
  } catch (const std::bad_alloc&) {               \
    if (p) (p)->impl.err = "host out of memory";  \
    return MOC_E_CAPACITY;                        \
  } catch (const std::exception& e) {             \
    if (p) (p)->impl.err = e.what();              \
    return MOC_E_INVALID_ARG;                     \
  }

// S:30-35 material rules (shared by moc_set_materials and moc_solver_update_materials)
void moc::check_materials(int n_mat, int G, const double* sigma_t, const double* sigma_s, const double* nu_sigma_f,
                          const double* chi) {
  for (int i = 0; i < n_mat; ++i) {
    double cs = 0, fs = 0;
    for (int g = 0; g < G; ++g) {
      if (!(sigma_t[(size_t)i * G + g] > 0)) throw Error(MOC_E_PARAM, "sigma_t must be > 0");
      if (!(nu_sigma_f[(size_t)i * G + g] >= 0) || !(chi[(size_t)i * G + g] >= 0))
        throw Error(MOC_E_PARAM, "nu_sigma_f and chi must be >= 0");
      for (int h = 0; h < G; ++h)
        if (!(sigma_s[((size_t)i * G + g) * G + h] >= 0)) throw Error(MOC_E_PARAM, "sigma_s must be >= 0");
      cs += chi[(size_t)i * G + g];
      fs += nu_sigma_f[(size_t)i * G + g];
    }
    if (fs > 0 && std::fabs(cs - 1.0) > 1e-9) throw Error(MOC_E_PARAM, "chi of a fissile material must sum to 1");
  }
}

extern "C" {

int moc_problem_create(moc_problem** out) {
  if (!out) return MOC_E_INVALID_ARG;
  try {
    *out = new moc_problem();
  } catch (...) {
    return MOC_E_CAPACITY;
  }
  return MOC_OK;
}

void moc_problem_destroy(moc_problem* p) { delete p; }

const char* moc_last_error(const moc_problem* p) { return p ? p->impl.err.c_str() : "NULL problem"; }

int moc_set_materials(moc_problem* p, int32_t n_mat, int32_t G, const double* sigma_t, const double* sigma_s,
                      const double* nu_sigma_f, const double* chi) {
  if (!p) return MOC_E_INVALID_ARG;
  MOC_TRY(p, {
    if (n_mat <= 0 || G <= 0 || !sigma_t || !sigma_s || !nu_sigma_f || !chi)
      throw Error(MOC_E_INVALID_ARG, "materials: bad sizes or NULL arrays");
    if (G > 8) throw Error(MOC_E_PARAM, "at most 8 energy groups are supported");
    Materials& m = p->impl.mat;
    m.n_mat = n_mat;
    m.G = G;
    m.sigma_t.assign(sigma_t, sigma_t + (size_t)n_mat * G);
    m.sigma_s.assign(sigma_s, sigma_s + (size_t)n_mat * G * G);
    m.nu_sigma_f.assign(nu_sigma_f, nu_sigma_f + (size_t)n_mat * G);
    m.chi.assign(chi, chi + (size_t)n_mat * G);
    check_materials(n_mat, G, sigma_t, sigma_s, nu_sigma_f, chi);
    m.set = true;
  })
}

int moc_set_geometry(moc_problem* p, const moc_geometry_desc* d) {
  if (!p || !d) return MOC_E_INVALID_ARG;
  MOC_TRY(p, {
    Geometry g;
    if (d->nx <= 0 || d->ny <= 0 || !(d->pitch_x > 0) || !(d->pitch_y > 0) || !d->cell_type || d->n_types <= 0 ||
        !d->n_rings || d->n_layers <= 0 || !d->planes || d->n_zones <= 0 || !d->zone_of_layer || !d->material)
      throw Error(MOC_E_INVALID_ARG, "geometry: bad sizes or NULL arrays");
    if (d->max_rings < 0 || d->max_rings > 16) throw Error(MOC_E_PARAM, "max_rings must be in [0, 16]");
    g.nx = d->nx;
    g.ny = d->ny;
    g.px = d->pitch_x;
    g.py = d->pitch_y;
    g.cell_type.assign(d->cell_type, d->cell_type + (size_t)d->nx * d->ny);
    g.n_types = d->n_types;
    g.max_rings = d->max_rings;
    g.n_rings.assign(d->n_rings, d->n_rings + d->n_types);
    if (d->max_rings > 0) {
      if (!d->radii) throw Error(MOC_E_INVALID_ARG, "radii is NULL");
      g.radii.assign(d->radii, d->radii + (size_t)d->n_types * d->max_rings);
    }
    g.NL = d->n_layers;
    g.planes.assign(d->planes, d->planes + d->n_layers + 1);
    g.n_zones = d->n_zones;
    g.zone_of_layer.assign(d->zone_of_layer, d->zone_of_layer + d->n_layers);
    g.material.assign(d->material, d->material + (size_t)d->n_types * (d->max_rings + 1) * d->n_zones);
    for (int f = 0; f < 6; ++f) {
      if (d->bc[f] != 0 && d->bc[f] != 1) throw Error(MOC_E_INVALID_ARG, "bc must be 0 (vacuum) or 1 (reflective)");
      g.bc[f] = d->bc[f];
    }
    if (g.planes[0] != 0.0) throw Error(MOC_E_MESH, "planes[0] must be 0");
    for (int l = 0; l < g.NL; ++l)
      if (!(g.planes[l + 1] > g.planes[l])) throw Error(MOC_E_MESH, "axial planes must be strictly increasing");
    for (int l = 0; l < g.NL; ++l)
      if (g.zone_of_layer[l] < 0 || g.zone_of_layer[l] >= g.n_zones) throw Error(MOC_E_MESH, "zone_of_layer out of range");
    for (int c = 0; c < g.nx * g.ny; ++c)
      if (g.cell_type[c] < 0 || g.cell_type[c] >= g.n_types) throw Error(MOC_E_REFERENCE, "cell_type out of range");
    for (int t = 0; t < g.n_types; ++t) {
      if (g.n_rings[t] < 0 || g.n_rings[t] > g.max_rings) throw Error(MOC_E_GEOMETRY, "n_rings out of range");
      double prev = 0;
      for (int q = 0; q < g.n_rings[t]; ++q) {
        double r = g.radii[(size_t)t * g.max_rings + q];
        if (!(r > prev)) throw Error(MOC_E_GEOMETRY, "ring radii must be positive and ascending");
        if (!(r < 0.5 * std::min(g.px, g.py))) throw Error(MOC_E_GEOMETRY, "ring overlaps the cell boundary");
        prev = r;
      }
    }
    const Materials& m = p->impl.mat;
    for (size_t i = 0; i < g.material.size(); ++i)
      if (g.material[i] < 0 || (m.set && g.material[i] >= m.n_mat)) throw Error(MOC_E_REFERENCE, "unknown material index");
    g.W = g.nx * g.px;
    g.Y = g.ny * g.py;
    g.Z = g.planes[g.NL];
    g.prefix.assign((size_t)g.nx * g.ny + 1, 0);
    for (int c = 0; c < g.nx * g.ny; ++c) g.prefix[c + 1] = g.prefix[c] + g.n_rings[g.cell_type[c]] + 1;
    g.n_regions = g.prefix[(size_t)g.nx * g.ny];
    g.n_fsr = g.n_regions * g.NL;
    g.set = true;
    p->impl.geo = std::move(g);
    p->impl.lay = Laydown();
  })
}

int moc_num_fsrs(const moc_problem* p, int64_t* J) {
  if (!p || !J) return MOC_E_INVALID_ARG;
  if (!p->impl.geo.set) return MOC_E_STATE;
  *J = p->impl.geo.n_fsr;
  return MOC_OK;
}

int moc_fsr_of_point(const moc_problem* p, double x, double y, double z, int64_t* fsr) {
  if (!p || !fsr) return MOC_E_INVALID_ARG;
  const Geometry& g = p->impl.geo;
  if (!g.set) return MOC_E_STATE;
  if (!(x >= 0 && x <= g.W && y >= 0 && y <= g.Y && z >= 0 && z <= g.Z)) return MOC_E_GEOMETRY;
  int cx = std::min((int)std::floor(x / g.px), g.nx - 1);
  int cy = std::min((int)std::floor(y / g.py), g.ny - 1);
  int l = 0;
  while (l < g.NL - 1 && z >= g.planes[l + 1]) ++l;  // half-open slabs, top slab closed
  *fsr = g.region_at(cx, cy, x, y) * g.NL + l;
  return MOC_OK;
}

int moc_generate_tracks(moc_problem* p, const moc_track_params* tp) {
  if (!p || !tp) return MOC_E_INVALID_ARG;
  MOC_TRY(p, {
    if (!p->impl.geo.set) throw Error(MOC_E_STATE, "set the geometry before generating tracks");
    build_laydown(p->impl.geo, *tp, p->impl.lay);
  })
}

int moc_get_track_stats(const moc_problem* p, moc_track_stats* st) {
  if (!p || !st) return MOC_E_INVALID_ARG;
  const Laydown& L = p->impl.lay;
  if (!L.done) return MOC_E_STATE;
  st->n_fsr = p->impl.geo.n_fsr;
  st->n_regions = p->impl.geo.n_regions;
  st->n_tracks2d = L.T2();
  st->n_segs2d = (int64_t)L.seg_region.size();
  st->n_stacks = L.S();
  st->n_tracks3d = L.n3;
  st->n_cycles = L.n_cycles;
  st->n_segs3d_raw = L.n_raw3;
  return MOC_OK;
}

int moc_get_tracks2d(const moc_problem* p, int32_t* azim, double* xy0, double* xy1, double* length,
                     int64_t* seg_off, int64_t* link_fwd, int32_t* link_fwd_enters_fwd, int64_t* link_bwd,
                     int32_t* link_bwd_enters_fwd) {
  if (!p) return MOC_E_INVALID_ARG;
  const Laydown& L = p->impl.lay;
  const Geometry& g = p->impl.geo;
  if (!L.done) return MOC_E_STATE;
  for (int64_t t = 0; t < L.T2(); ++t) {
    if (azim) azim[t] = L.t_a[t];
    if (xy0) {
      xy0[2 * t] = L.t_x0[t];
      xy0[2 * t + 1] = L.t_y0[t];
    }
    if (xy1) {
      xy1[2 * t] = L.t_x1[t];
      xy1[2 * t + 1] = L.t_y1[t];
    }
    if (length) length[t] = L.t_len[t];
    if (link_fwd) link_fwd[t] = g.bc[L.t_fend[t]] ? L.t_glf[t] : -1;
    if (link_fwd_enters_fwd) link_fwd_enters_fwd[t] = L.t_glf_fwd[t];
    if (link_bwd) link_bwd[t] = g.bc[L.t_fstart[t]] ? L.t_glb[t] : -1;
    if (link_bwd_enters_fwd) link_bwd_enters_fwd[t] = L.t_glb_fwd[t];
  }
  if (seg_off)
    for (int64_t t = 0; t <= L.T2(); ++t) seg_off[t] = L.t_seg[t];
  return MOC_OK;
}

int moc_get_segments2d(const moc_problem* p, int64_t* region, double* s_end) {
  if (!p || !region || !s_end) return MOC_E_INVALID_ARG;
  const Laydown& L = p->impl.lay;
  if (!L.done) return MOC_E_STATE;
  for (size_t k = 0; k < L.seg_region.size(); ++k) {
    region[k] = L.seg_region[k];
    s_end[k] = L.seg_send[k];
  }
  return MOC_OK;
}

int moc_get_stacks(const moc_problem* p, double* z0, int64_t* count, int64_t* first) {
  if (!p) return MOC_E_INVALID_ARG;
  const Laydown& L = p->impl.lay;
  if (!L.done) return MOC_E_STATE;
  for (int64_t s = 0; s < L.S(); ++s) {
    if (z0) z0[s] = L.st_z0[s];
    if (count) count[s] = L.st_cnt[s];
  }
  if (first)
    for (int64_t s = 0; s <= L.S(); ++s) first[s] = L.st_first[s];
  return MOC_OK;
}

int moc_get_polar(const moc_problem* p, double* theta, double* dz, double* weight, double* aperp) {
  if (!p) return MOC_E_INVALID_ARG;
  const Laydown& L = p->impl.lay;
  if (!L.done) return MOC_E_STATE;
  for (size_t u = 0; u < L.an_theta.size(); ++u) {
    if (theta) theta[u] = L.an_theta[u];
    if (dz) dz[u] = L.an_dz[u];
    if (weight) weight[u] = L.an_w[u];
    if (aperp) aperp[u] = L.an_aperp[u];
  }
  return MOC_OK;
}

int moc_get_links3d(const moc_problem* p, int64_t* link) {
  if (!p || !link) return MOC_E_INVALID_ARG;
  moc_problem* q = const_cast<moc_problem*>(p);
  MOC_TRY(q, {
    if (!p->impl.lay.done) throw Error(MOC_E_STATE, "tracks not generated");
    links3d(p->impl.geo, p->impl.lay, link);
  })
}

int moc_trace_track_3d(const moc_problem* p, int64_t track3d, int64_t* fsr, double* len, int64_t cap, int64_t* nseg) {
  if (!p || !nseg) return MOC_E_INVALID_ARG;
  const Laydown& L = p->impl.lay;
  if (!L.done) return MOC_E_STATE;
  if (track3d < 0 || track3d >= L.n3) return MOC_E_INVALID_ARG;
  TrackGeo tg = track_geo(p->impl.geo, L, track3d, nullptr);
  OtfView v = otf_view_host(p->impl.geo, L);
  int64_t n = 0;
  otf_walk_fwd(v, tg, [&](int64_t, int, double) { ++n; });
  *nseg = n;
  if (cap < n) return MOC_E_INVALID_ARG;
  int64_t q = 0;
  otf_walk_fwd(v, tg, [&](int64_t k, int ly, double l) {
    if (fsr) fsr[q] = (int64_t)v.seg_region[k] * v.NL + ly;
    if (len) len[q] = l;
    ++q;
  });
  return MOC_OK;
}

// SURVEY §8(b) moc_get_fsr_volumes on the problem handle: track-estimated volumes from the
// host OTF walk over every 3D track (App. A.5: V_j = sum W/(2 pi) A_perp L), OpenMP with
// per-thread sums merged in thread order; analytic volumes S:83-85.
static void host_track_volumes(const Geometry& g, const Laydown& L, double* vol) {
  const int64_t J = g.n_fsr;
  const OtfView v = otf_view_host(g, L);
  const int nth = omp_get_max_threads();
  std::vector<std::vector<double>> part(nth, std::vector<double>((size_t)J, 0.0));
#pragma omp parallel num_threads(nth)
  {
    std::vector<double>& V = part[omp_get_thread_num()];
#pragma omp for schedule(static)
    for (int64_t s = 0; s < L.S(); ++s) {
      const int64_t t = s / L.N;
      const size_t an = (size_t)L.t_a[t] * L.N + (size_t)(s % L.N);
      const double w = L.an_w[an] / (2.0 * 3.14159265358979323846) * L.an_aperp[an];
      for (int64_t id = L.st_first[s]; id < L.st_first[s + 1]; ++id) {
        const TrackGeo tg = track_geo(g, L, id, nullptr);
        otf_walk_fwd(v, tg, [&](int64_t k, int ly, double len) { V[(size_t)(v.seg_region[k] * v.NL + ly)] += w * len; });
      }
    }
  }
  for (int64_t j = 0; j < J; ++j) {
    double a = 0.0;
    for (int th = 0; th < nth; ++th) a += part[th][j];
    vol[j] = a;
  }
}

int moc_problem_fsr_volumes(const moc_problem* p, double* vol_track, double* vol_analytic) {
  if (!p || (!vol_track && !vol_analytic)) return MOC_E_INVALID_ARG;
  moc_problem* q = const_cast<moc_problem*>(p);
  MOC_TRY(q, {
    if (!p->impl.lay.done) throw Error(MOC_E_STATE, "tracks not generated");
    if (vol_analytic) p->impl.geo.analytic_volumes(vol_analytic);
    if (vol_track) host_track_volumes(p->impl.geo, p->impl.lay, vol_track);
  })
}

/* host-side backward walk (test hook: the backward list must mirror the forward one) */
int moc_trace_track_3d_backward(const moc_problem* p, int64_t track3d, int64_t* fsr, double* len, int64_t cap,
                                int64_t* nseg) {
  if (!p || !nseg) return MOC_E_INVALID_ARG;
  const Laydown& L = p->impl.lay;
  if (!L.done) return MOC_E_STATE;
  if (track3d < 0 || track3d >= L.n3) return MOC_E_INVALID_ARG;
  TrackGeo tg = track_geo(p->impl.geo, L, track3d, nullptr);
  OtfView v = otf_view_host(p->impl.geo, L);
  int64_t q = 0;
  otf_walk_bwd(v, tg, [&](int64_t k, int ly, double l) {
    if (q < cap) {
      if (fsr) fsr[q] = (int64_t)v.seg_region[k] * v.NL + ly;
      if (len) len[q] = l;
    }
    ++q;
  });
  *nseg = q;
  return q <= cap ? MOC_OK : MOC_E_INVALID_ARG;
}

int moc_partition_stacks(const moc_problem* p, int32_t world, int32_t* owner, double* cost) {
  if (!p || !owner || world < 1) return MOC_E_INVALID_ARG;
  moc_problem* q = const_cast<moc_problem*>(p);
  MOC_TRY(q, {
    if (!p->impl.lay.done) throw Error(MOC_E_STATE, "tracks not generated");
    std::vector<int32_t> o;
    std::vector<double> c;
    partition_stacks(p->impl.lay, world, o, &c);
    std::copy(o.begin(), o.end(), owner);
    if (cost) std::copy(c.begin(), c.end(), cost);
  })
}

int moc_halo_plan(const moc_problem* p, int32_t world, const int32_t* owner, int32_t rank, int32_t peer,
                  int64_t* slots, int64_t cap, int64_t* n) {
  if (!p || !owner || !n || rank < 0 || peer < 0 || rank >= world || peer >= world) return MOC_E_INVALID_ARG;
  moc_problem* q = const_cast<moc_problem*>(p);
  MOC_TRY(q, {
    const Laydown& L = p->impl.lay;
    if (!L.done) throw Error(MOC_E_STATE, "tracks not generated");
    std::vector<int64_t> link(2 * (size_t)L.n3);
    links3d(p->impl.geo, L, link.data());
    std::vector<int32_t> own(owner, owner + L.S());
    std::vector<std::vector<int64_t>> send, recv;
    halo_plans(L, link.data(), own, rank, world, send, recv);
    *n = (int64_t)send[peer].size();
    if (slots && cap >= *n) std::copy(send[peer].begin(), send[peer].end(), slots);
  })
}

int moc_rank_layout(const moc_problem* p, int32_t world, const int32_t* owner, int32_t rank, int64_t* sizes,
                    int64_t* slot_first, int64_t* link, int64_t* recv_slots, int64_t* send_counts,
                    int64_t* recv_counts) {
  if (!p || !owner || !sizes || rank < 0 || rank >= world) return MOC_E_INVALID_ARG;
  moc_problem* q = const_cast<moc_problem*>(p);
  MOC_TRY(q, {
    const Laydown& L = p->impl.lay;
    if (!L.done) throw Error(MOC_E_STATE, "tracks not generated");
    std::vector<int64_t> lk(2 * (size_t)L.n3);
    links3d(p->impl.geo, L, lk.data());
    std::vector<int32_t> own(owner, owner + L.S());
    RankLayout rl;
    rank_layout(L, lk.data(), own, rank, world, rl);
    sizes[0] = rl.T3_local;
    sizes[1] = rl.n_send;
    sizes[2] = (int64_t)rl.recv_slots.size();
    if (slot_first) std::copy(rl.slot_first.begin(), rl.slot_first.end(), slot_first);
    if (link) std::copy(rl.link.begin(), rl.link.end(), link);
    if (recv_slots) std::copy(rl.recv_slots.begin(), rl.recv_slots.end(), recv_slots);
    if (send_counts) std::copy(rl.send_counts.begin(), rl.send_counts.end(), send_counts);
    if (recv_counts) std::copy(rl.recv_counts.begin(), rl.recv_counts.end(), recv_counts);
  })
}

// ---- Eq. 5: z_i(s) = z_0(0) + i dz + s cot(theta)
double moc_z_of(double z0, double dz, int64_t i, double theta, double s) {
  return z0 + (double)i * dz + s * (std::cos(theta) / std::sin(theta));
}

// ---- Eqs. 6-7, clamping left to the caller
void moc_intersecting_range(double z0_sstart, double z0_send, double dz, double zmin, double zmax, int64_t* i_start,
                            int64_t* i_end) {
  double zhi = std::max(z0_sstart, z0_send), zlo = std::min(z0_sstart, z0_send);
  *i_start = (int64_t)std::ceil((zmin - zhi) / dz);
  *i_end = (int64_t)std::floor((zmax - zlo) / dz);
}

// ---- Eqs. 9-10
void moc_full_crossing_range(double z0_sstart, double z0_send, double dz, double zmin, double zmax, int64_t* i_in,
                             int64_t* i_out) {
  double zhi = std::max(z0_sstart, z0_send), zlo = std::min(z0_sstart, z0_send);
  *i_in = (int64_t)std::ceil((zmin - zlo) / dz);
  *i_out = (int64_t)std::floor((zmax - zhi) / dz);
}

// ---- Eq. 13: Z-STACK[i][j][k] = stack[z[i] + j*c + k]
int64_t moc_flat_index(const int64_t* offsets, int64_t c, int64_t i, int64_t j, int64_t k) {
  return offsets[i] + j * c + k;
}

// ---- §4.3: sort descending by segment count, chunk, reverse every other chunk
int moc_serpentine_order(const int64_t* counts, int64_t n, int64_t chunk, int64_t* order) {
  if (!counts || !order || n < 0 || chunk <= 0) return MOC_E_INVALID_ARG;
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return counts[a] > counts[b]; });
  for (int64_t c0 = 0, ci = 0; c0 < n; c0 += chunk, ++ci)
    if (ci & 1) std::reverse(idx.begin() + c0, idx.begin() + std::min(n, c0 + chunk));
  std::copy(idx.begin(), idx.end(), order);
  return MOC_OK;
}

// ---- §4.2: descending by memory, accumulate until the threshold is reached
int moc_partition_exp_otf(const int64_t* est, int64_t n, double budget, double fraction, int32_t* preload) {
  if (!est || !preload || n < 0 || !(budget > 0) || !(fraction > 0) || fraction > 1) return MOC_E_INVALID_ARG;
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return est[a] > est[b]; });
  std::fill(preload, preload + n, 0);
  double cum = 0, lim = budget * fraction;
  for (int64_t q = 0; q < n; ++q) {
    if (cum + (double)est[idx[q]] > lim) break;
    cum += (double)est[idx[q]];
    preload[idx[q]] = 1;
  }
  return MOC_OK;
}

}  // extern "C"
