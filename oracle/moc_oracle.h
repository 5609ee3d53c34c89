/*
 * moc_oracle.h — C interface of the fp64 CPU oracle for the 3D MOC OTF sweep.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * The product (paper_2503_17743_b200/, include/) never includes this header
 * and this oracle never includes product code: the two share nothing but the
 * seeded input generator in problems/ (which holds none of the method's
 * arithmetic).
 *
 * What it computes: a plain explicit 3D MOC k-eigenvalue
 * solver in double precision — the same cyclic track laydown,
 * brute-force 2D and 3D segmentation (no Eqs. 6-11), geometric (hash-matched)
 * reflective links, Jacobi power iteration with Eq. 3 evaluated with expm1.
 *
 * Conventions: lengths cm, cross sections 1/cm.  Faces: 0 x-, 1 x+, 2 y-,
 * 3 y+, 4 z-, 5 z+; bc value 0 = vacuum, 1 = reflective.  A "slot" is
 * 2*track3d + dir (dir 0 = forward along increasing 2D s, 1 = backward).
 */
#ifndef MOC_ORACLE_H
#define MOC_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  /* pin lattice */
  int32_t nx, ny;
  double pitch_x, pitch_y;
  const int32_t* cell_type;    /* [ny*nx], row-major from (x_min, y_min) */
  int32_t n_types;
  int32_t max_rings;
  const int32_t* n_rings;      /* [n_types] */
  const double* radii;         /* [n_types][max_rings], ascending per type */
  /* axial mesh (global), planes[0] must be 0 */
  int32_t n_layers;
  const double* planes;        /* [n_layers+1] */
  int32_t n_zones;
  const int32_t* zone_of_layer;/* [n_layers] */
  const int32_t* material;     /* [n_types][max_rings+1][n_zones]; local ring index, last = moderator */
  int32_t bc[6];
  /* materials */
  int32_t n_mat, G;
  const double* sigma_t;       /* [n_mat][G] */
  const double* sigma_s;       /* [n_mat][G from][G to] */
  const double* nu_sigma_f;    /* [n_mat][G] */
  const double* chi;           /* [n_mat][G] */
  /* quadrature / tracking */
  int32_t num_azim, num_polar;
  double radial_spacing, axial_spacing;
} or_problem;

typedef struct {
  int64_t n_fsr, n_regions, n_tracks2d, n_segs2d, n_stacks, n_tracks3d;
  int64_t n_cycles;
  int64_t n_degenerate;  /* stack-membership tests within 1e-9 of an integer (should be 0) */
} or_counts;

void* or_create(const or_problem* p, char* err, int64_t errlen);
void or_destroy(void* h);
void or_get_counts(void* h, or_counts* c);

/* 2D laydown: per 2D track: family a, start/end points, length, segment range,
 * link target of the forward exit (and whether it is entered forward) and of
 * the backward exit; -1 = vacuum. */
void or_get_tracks2d(void* h, int32_t* azim, double* xy0, double* xy1, double* length,
                     int64_t* seg_off, int64_t* link_fwd, int32_t* link_fwd_enters_fwd,
                     int64_t* link_bwd, int32_t* link_bwd_enters_fwd,
                     int64_t* cycle, double* ltilde, int32_t* sigma);
void or_get_segments2d(void* h, int64_t* region, double* s_end);
/* per (family a): phi, n_x, n_y, spacing delta_a, weight omega_a */
void or_get_azim(void* h, double* phi, int32_t* nx, int32_t* ny, double* delta, double* omega);
/* per (a, n): theta, dz, weight W_{a,n}, A_perp */
void or_get_polar(void* h, double* theta, double* dz, double* wgt, double* aperp);
void or_get_polar_gl(void* h, double* mu, double* w);
/* stacks in Alg. 1 order (t, n): z0 of member 0, member count, first 3D track id */
void or_get_stacks(void* h, double* z0, int64_t* count, int64_t* first);
/* explicit 3D segmentation of one track; returns #segments (or -needed if cap too small) */
int64_t or_trace3d(void* h, int64_t track, int64_t* fsr, double* len, int64_t cap);
/* per-track n_seg, FNV-1a-64 hash of the FSR id sequence (uint32 LE), sum of lengths, chord */
void or_track_checksums(void* h, int64_t first, int64_t n, int32_t* nseg, uint64_t* hash, double* suml,
                        double* chord, uint64_t* rhash /* reversed-order hash or NULL */);
int64_t or_total_segments3d(void* h);
/* 3D links by geometric matching: link[slot] = target slot or -1 (vacuum) */
int or_links3d(void* h, int64_t* link, char* err, int64_t errlen);
void or_volumes(void* h, double* vol_track, double* vol_analytic);
void or_fsr_material(void* h, int32_t* mat);

/* Power iteration.  fixed_iters>0: exactly that many
 * iterations; else until |dk|<tol_k and residual<tol_src or max_iter.
 * Returns #iterations.  phi: [n_fsr][G] normalised so sum_j V_j F_j = 1. */
int or_solve(void* h, int fixed_iters, int max_iter, double tol_k, double tol_src,
             double* k_out, double* k_hist, double* res_hist, double* phi_out,
             double* leakage_out, double* production_out, double* absorption_out,
             char* err, int64_t errlen);

/* CPU baseline timing on a bounded sample: sweep every `stride`-th 3D track (both
 * directions) once with psi_in = 0 and a flat source; returns seconds, and the
 * number of segment-group integrations done (2 * nseg * G per track). */
double or_time_sample_sweep(void* h, int64_t stride, int nthreads, int64_t* integrations);
int or_num_threads(void);

/* brute-force 2D segmentation of an arbitrary line (pin P7); returns #segments */
int64_t or_segment_line(void* h, double x0, double y0, double ux, double uy, double L, int64_t* region,
                        double* s_end, int64_t cap);
int64_t or_region_of(void* h, double x, double y);

/* Standalone formulas for pins. */
double or_attenuate(double psi_in, double q_over_sigma, double sigma_t, double s, double* delta_psi);
void or_source(int G, const double* phi, const double* sigma_t, const double* sigma_s,
               const double* nu_sigma_f, const double* chi, double k, double* qtilde);

#ifdef __cplusplus
}
#endif
#endif
