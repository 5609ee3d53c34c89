// host.h — internal host-side data of libmoc3d.so (not part of the ABI).
//
// Problem = materials + extruded pin-lattice geometry + the laydown
// produced on the host: cyclic 2D tracks and their
// 2D segments, per-(a, n) polar data, z-stacks and the 3D link table.
#pragma once
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/moc3d.h"
#include "otf.h"

namespace moc {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Materials {
  int n_mat = 0, G = 0;
  std::vector<double> sigma_t, sigma_s, nu_sigma_f, chi;  // row-major as in the ABI
  bool set = false;
};

// sigma_t > 0, sigma_s / nu_sigma_f / chi >= 0, chi of a fissile material sums to 1
void check_materials(int n_mat, int G, const double* sigma_t, const double* sigma_s, const double* nu_sigma_f,
                     const double* chi);

struct Geometry {
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
  // derived
  double W = 0, Y = 0, Z = 0;
  std::vector<int64_t> prefix;  // region prefix per cell [nx*ny + 1]
  int64_t n_regions = 0, n_fsr = 0;
  bool set = false;

  int64_t region_at(int cx, int cy, double x, double y) const;  // ring test inside cell (cx, cy)
  int mat_of_fsr(int64_t j) const;
  void analytic_volumes(double* vol) const;  // [n_fsr]
};

struct Laydown {
  int M = 0, N = 0;
  double dr = 0, dzs = 0;
  // per azimuthal family a in [0, M/2)
  std::vector<double> phi, delta, omega;
  std::vector<int32_t> nxa, nya;
  std::vector<int64_t> fam_off;  // [M/2 + 1]
  // 2D tracks
  std::vector<int32_t> t_a;
  std::vector<double> t_x0, t_y0, t_x1, t_y1, t_len, t_ux, t_uy;
  std::vector<int8_t> t_fstart, t_fend;
  std::vector<int64_t> t_glf, t_glb;      // geometric links (every face reflective)
  std::vector<int8_t> t_glf_fwd, t_glb_fwd;
  std::vector<int64_t> t_seg;             // [T2 + 1]
  std::vector<int64_t> t_cyc;
  std::vector<double> t_lt;               // cycle arc length of s = 0
  std::vector<int8_t> t_sig;              // +1 forward in its cycle, -1 backward
  std::vector<double> cycle_len;          // per family
  int64_t n_cycles = 0;
  // 2D segments
  std::vector<uint32_t> seg_region;
  std::vector<double> seg_send;
  // polar: GL nodes, and per (a, n) corrected angles
  std::vector<double> mu, wgl;
  std::vector<double> an_theta, an_cot, an_tan, an_invsin, an_dz, an_w, an_aperp;
  // z-stacks (t, n) in Alg. 1 order
  std::vector<double> st_z0;
  std::vector<int64_t> st_cnt, st_first;  // first [S + 1]
  int64_t n3 = 0;
  int64_t n_raw3 = 0;                     // sum of raw piece counts (cost estimate)
  std::vector<int64_t> st_raw;            // raw piece count per stack
  bool done = false;

  int64_t T2() const { return (int64_t)t_len.size(); }
  int64_t S() const { return (int64_t)st_cnt.size(); }
};

struct ProblemImpl {
  Materials mat;
  Geometry geo;
  Laydown lay;
  std::string err;
};

// laydown.cpp
void build_laydown(const Geometry& g, const moc_track_params& tp, Laydown& L);
void links3d(const Geometry& g, const Laydown& L, int64_t* link);  // index arithmetic (App. A.4)
int64_t link_slot(const Geometry& g, const Laydown& L, int64_t track, int dir);
TrackGeo track_geo(const Geometry& g, const Laydown& L, int64_t track, int64_t* stack_out);
OtfView otf_view_host(const Geometry& g, const Laydown& L);

// partition.cpp: contiguous cost-balanced split of the stacks, ordered by
// (polar pair, 2D cycle, position along the cycle), over `world` ranks; and the
// boundary-psi halo plan (target slots this rank writes that `peer` owns).
void partition_stacks(const Laydown& L, int world, std::vector<int32_t>& owner, std::vector<double>* cost);
void halo_plan(const Laydown& L, const int64_t* link, const std::vector<int32_t>& owner, int rank, int peer,
               std::vector<int64_t>& slots);
void halo_plans(const Laydown& L, const int64_t* link, const std::vector<int32_t>& owner, int rank, int world,
                std::vector<std::vector<int64_t>>& send, std::vector<std::vector<int64_t>>& recv);
struct RankLayout {
  int64_t T3_local = 0, n_send = 0;
  std::vector<int64_t> slot_first;               // [S + 1] local first track of each stack
  std::vector<int64_t> link;                     // [2 T3_local] local target slot (-1 vacuum)
  std::vector<int64_t> recv_slots;               // local slots of received psi, peer-major
  std::vector<int64_t> send_counts, recv_counts; // [world] slots per peer
};
void rank_layout(const Laydown& L, const int64_t* link, const std::vector<int32_t>& owner, int rank, int world,
                 RankLayout& out);

}  // namespace moc

struct moc_problem {
  moc::ProblemImpl impl;
};
