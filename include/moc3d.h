/*
 * moc3d.h — C ABI of libmoc3d.so, the B200-native OTF 3D MOC transport sweep
 * (arXiv 2503.17743) and the power iteration that wraps it.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (reference text),
 * SURVEY §x = /root/repo/SURVEY.md, Qn = reading n in DESIGN.md §2.
 *
 * Conventions (all entry points):
 *   - Return value: MOC_OK (0) on success, a negative MOC_E_* code on error; the
 *     message is available from moc_last_error()/moc_solver_last_error() until
 *     the next call on the same handle.  No C++ exception crosses the ABI.
 *   - Units: cm and 1/cm.  Host arrays are fp64 unless stated; every input array
 *     is COPIED on entry — the caller keeps ownership and may free it on return.
 *   - Output arrays are caller-allocated host buffers whose sizes come from the
 *     query calls (moc_num_fsrs, moc_get_track_stats).
 *   - Handles own all host and device memory they allocate.  A handle is not
 *     thread-safe; distinct handles are independent.
 *   - Device work is stream-ordered on the stream given to moc_solver_create
 *     (pass torch.cuda.current_stream().cuda_stream, or NULL for the legacy stream).
 *   - Faces: 0 x-, 1 x+, 2 y-, 3 y+, 4 z-, 5 z+ ; bc 0 = vacuum, 1 = reflective.
 *   - 3D track id: Alg. 1 order: 2D track t outer, polar n, stack member i.
 *     Slot = 2*track + dir, dir 0 = forward (increasing 2D s), 1 = backward.
 */
#ifndef MOC3D_H
#define MOC3D_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
  MOC_OK = 0,
  MOC_E_INVALID_ARG = -1, /* NULL / out-of-range argument                                  */
  MOC_E_GEOMETRY = -2,    /* radii overlap the cell, point out of domain       */
  MOC_E_REFERENCE = -3,   /* unknown material index                                  */
  MOC_E_MESH = -4,        /* axial planes not strictly increasing / planes[0] != 0   */
  MOC_E_PARAM = -5,       /* num_azim % 4, spacing > domain, G > 8, odd num_polar    */
  MOC_E_TRACE = -6,       /* segmentation stall, 3D link landing off a stack member */
  MOC_E_CAPACITY = -7,    /* device memory exhausted                                */
  MOC_E_EIGEN = -8,       /* k <= 0 or zero fission source                    */
  MOC_E_NUMERIC = -9,     /* NaN / negative scalar flux                              */
  MOC_E_NOCONV = -10,     /* max_iter reached without convergence                    */
  MOC_E_CUDA = -11,       /* CUDA runtime error                                              */
  MOC_E_NCCL = -12,       /* multi-GPU exchange failed: NCCL could not be loaded (libnccl.so.2)
                             or returned an error (message names the call and ncclResult), or
                             the caller's exchange callback returned non-zero               */
  MOC_E_STATE = -13       /* call order (e.g. tracks not generated)                          */
};

typedef struct moc_problem moc_problem;
typedef struct moc_solver moc_solver;

/* ---------------------------------------------------------------- problem
 * Geometry/material setup ("geometric modelling").       */
int moc_problem_create(moc_problem** out);
void moc_problem_destroy(moc_problem* p);
const char* moc_last_error(const moc_problem* p);

/* Multigroup materials.  sigma_t [n_mat][G], sigma_s [n_mat][G from][G to],
 * nu_sigma_f [n_mat][G], chi [n_mat][G].  Requires sigma_t > 0, G in [1, 8];
 * chi must sum to 1 +- 1e-9 for fissile materials (MOC_E_PARAM otherwise). */
int moc_set_materials(moc_problem* p, int32_t n_mat, int32_t G, const double* sigma_t,
                      const double* sigma_s, const double* nu_sigma_f, const double* chi);

/* Axially extruded pin lattice ("axially extruded geometry").
 * Cells are nx*ny rectangles of pitch (pitch_x, pitch_y), row-major from (x_min, y_min).
 * Cell type c has n_rings[c] concentric circles (radii[c*max_rings + q], ascending,
 * < min(pitch)/2) centred in the cell; local region q < n_rings is the q-th ring
 * (innermost first), local region n_rings[c] is the moderator outside the last circle.
 * material[(c*(max_rings+1) + q)*n_zones + zone] is the material of local region q
 * in axial zone `zone`; zone_of_layer[l] maps axial layer l (between planes[l] and
 * planes[l+1]; planes[0] must be 0) to its zone.
 * FSR numbering: region r = prefix(cell) + local, j = r*n_layers + layer. */
typedef struct {
  int32_t nx, ny;
  double pitch_x, pitch_y;
  const int32_t* cell_type;     /* [ny*nx]            */
  int32_t n_types, max_rings;
  const int32_t* n_rings;       /* [n_types]          */
  const double* radii;          /* [n_types*max_rings] (may be NULL if max_rings == 0) */
  int32_t n_layers;
  const double* planes;         /* [n_layers+1]       */
  int32_t n_zones;
  const int32_t* zone_of_layer; /* [n_layers]         */
  const int32_t* material;      /* [n_types*(max_rings+1)*n_zones] */
  int32_t bc[6];
} moc_geometry_desc;
int moc_set_geometry(moc_problem* p, const moc_geometry_desc* g);
int moc_num_fsrs(const moc_problem* p, int64_t* J);
/* FSR containing (x, y, z) (axial slabs half-open, top slab closed). */
int moc_fsr_of_point(const moc_problem* p, double x, double y, double z, int64_t* fsr);

/* 2D cyclic laydown + 2D segmentation (A1) and z-stacks + 3D links (A2), on the host
 * ("the CPU executes 2D ray tracing").  num_azim % 4 == 0,
 * num_polar even, spacings > 0. */
typedef struct {
  int32_t num_azim, num_polar;
  double radial_spacing, axial_spacing;
} moc_track_params;
int moc_generate_tracks(moc_problem* p, const moc_track_params* tp);

typedef struct {
  int64_t n_fsr, n_regions, n_tracks2d, n_segs2d, n_stacks, n_tracks3d, n_cycles;
  int64_t n_segs3d_raw; /* upper bound: #2D segments spanned + #axial planes crossed */
} moc_track_stats;
int moc_get_track_stats(const moc_problem* p, moc_track_stats* st);

/* Debug/parity exports of the laydown (caller-allocated, sizes from moc_get_track_stats).
 * tracks2d: azim[T2], xy0[2*T2], xy1[2*T2], length[T2], seg_off[T2+1],
 *           link_fwd/link_bwd[T2] (target 2D track or -1 vacuum), *_enters_fwd[T2]. */
int moc_get_tracks2d(const moc_problem* p, int32_t* azim, double* xy0, double* xy1, double* length,
                     int64_t* seg_off, int64_t* link_fwd, int32_t* link_fwd_enters_fwd,
                     int64_t* link_bwd, int32_t* link_bwd_enters_fwd);
int moc_get_segments2d(const moc_problem* p, int64_t* region, double* s_end);
/* per stack (t, n) in Alg. 1 order: z of member 0 at s = 0, member count, first 3D id [S+1] */
int moc_get_stacks(const moc_problem* p, double* z0, int64_t* count, int64_t* first);
/* per (a, n): corrected polar angle, axial spacing dz, weight W, perpendicular area A_perp */
int moc_get_polar(const moc_problem* p, double* theta, double* dz, double* weight, double* aperp);
/* 3D link table by index arithmetic: link[slot] = target slot or -1. */
int moc_get_links3d(const moc_problem* p, int64_t* link);

/* FSR volumes [J] on the problem (SURVEY §8(b) moc_get_fsr_volumes; host computation, no
 * GPU): vol_track = the track estimate V_j = sum_{a,n} W_{a,n}/(2 pi) A_perp sum L from the
 * host OTF walk over every 3D track (App. A.5), vol_analytic = area x layer height
 * (S:83-85).  Either pointer may be NULL (not both).  The solver's moc_get_fsr_volumes
 * returns the same track estimate from the device walk. */
int moc_problem_fsr_volumes(const moc_problem* p, double* vol_track, double* vol_analytic);

/* OTF 3D segments of one track (S:231 trace_segments_otf; Eqs. 5, 8, 11) computed on
 * the host with the same walk the device kernel runs.  Returns #segments in *nseg;
 * if cap < *nseg nothing is written and MOC_E_INVALID_ARG is returned. */
int moc_trace_track_3d(const moc_problem* p, int64_t track3d, int64_t* fsr, double* len,
                       int64_t cap, int64_t* nseg);

/* Eqs. 5-7 and 9-10 as stated, for tests and cost estimates.
 * intersecting_range: i_start = ceil((zmin - max(z0s, z0e))/dz), i_end = floor((zmax - min(z0s, z0e))/dz);
 * full_crossing_range: i_in = ceil((zmin - min)/dz), i_out = floor((zmax - max)/dz). */
double moc_z_of(double z0, double dz, int64_t i, double theta, double s);
void moc_intersecting_range(double z0_sstart, double z0_send, double dz, double zmin, double zmax,
                            int64_t* i_start, int64_t* i_end);
void moc_full_crossing_range(double z0_sstart, double z0_send, double dz, double zmin, double zmax,
                             int64_t* i_in, int64_t* i_out);
/* Eq. 13 flattened Z-STACK accessor: stack[z[i] + j*c + k]. */
int64_t moc_flat_index(const int64_t* offsets, int64_t c, int64_t i, int64_t j, int64_t k);

/* Paper §4.2 / §4.3 host scheduling rules.
 * serpentine: sort by count descending (stable), reverse every odd chunk. */
int moc_serpentine_order(const int64_t* counts, int64_t n, int64_t chunk, int64_t* order_out);
/* EXP/OTF partition: descending by estimate, accumulate while <= fraction*budget. */
int moc_partition_exp_otf(const int64_t* estimates, int64_t n, double budget, double fraction,
                          int32_t* preload_out);

/* Multi-GPU decomposition, host side and deterministic on every rank:
 * owner[S] = rank sweeping each stack (contiguous cost-balanced pieces of the stacks ordered
 * by polar pair, 2D cycle, position along the cycle); cost[world] (or NULL) = raw segment
 * count per rank.  halo: target slots `rank` writes that `peer` owns, in source-slot order
 * (the receiver derives the same list); *n = count, nothing written if cap < *n. */
int moc_partition_stacks(const moc_problem* p, int32_t world, int32_t* owner, double* cost);
int moc_halo_plan(const moc_problem* p, int32_t world, const int32_t* owner, int32_t rank, int32_t peer,
                  int64_t* slots, int64_t cap, int64_t* n);
/* The layout the solver uses on `rank` (boundary psi owned by the sweeping rank): sizes[3] =
 * {T3_local, n_send, n_recv}; then (each optional, NULL = skip) slot_first[S+1] (local first
 * track of each stack), link[2 T3_local] (local target slot: < 2 T3_local owned, else the
 * halo-send tail in peer blocks; -1 vacuum), recv_slots[n_recv] (local slots of received
 * psi, peer-major), send_counts[world], recv_counts[world].  Call once with NULL arrays
 * to size them. */
int moc_rank_layout(const moc_problem* p, int32_t world, const int32_t* owner, int32_t rank, int64_t* sizes,
                    int64_t* slot_first, int64_t* link, int64_t* recv_slots, int64_t* send_counts,
                    int64_t* recv_counts);

/* ---------------------------------------------------------------- solver */
/* Multi-GPU: one process per GPU, `world` ranks.  Each rank sweeps its
 * contiguous cost-balanced share of the z-stacks; every iteration the fp32 FSR tally
 * [J][Gp] (+ the leakage in one tail element) is sum-all-reduced and the outgoing boundary
 * psi of cut-crossing links is exchanged with the owning ranks.
 *   backend MOC_COMM_NCCL: the library owns an NCCL communicator built from nccl_id
 *     (rank 0 calls moc_nccl_unique_id and the caller broadcasts the 128 bytes, e.g. with
 *     torch.distributed); the all-reduce and the grouped send/recv run on the solver's
 *     stream inside moc_iterate / moc_solve, which then capture each iteration in a CUDA
 *     graph (no host synchronisation between iterations).  NCCL is loaded at run time
 *     (dlopen libnccl.so.2; torch has it in-process): no link dependency.
 *   backend MOC_COMM_CALLER: the caller performs the exchange, either by driving
 *     moc_iteration_sweep / moc_iteration_finish itself or by registering a host callback
 *     with moc_solver_set_exchange (used with gloo on one GPU, for tests). */
enum { MOC_COMM_CALLER = 0, MOC_COMM_NCCL = 1 };
typedef struct {
  int32_t rank, world;      /* world == 1: single GPU                                 */
  int32_t backend;          /* MOC_COMM_CALLER or MOC_COMM_NCCL                       */
  uint8_t nccl_id[128];     /* ncclUniqueId (backend MOC_COMM_NCCL), same on every rank */
} moc_comm_desc;

/* ncclGetUniqueId into id[128] (rank 0; MOC_E_NCCL if NCCL cannot be loaded). */
int moc_nccl_unique_id(uint8_t* id);

/* Sweep schedules.  MOC_SCHED_STACK_COLLECTIVE is the product path (opts == NULL selects
 * it); the others are kept as measured baselines.  Schedule 0 accumulates the tally in a
 * per-unit u32 fixed point and misses the per-element flux criterion at convergence in
 * low-flux FSRs (2e-3 on the converged cfg3 assembly). */
enum {
  MOC_SCHED_TRACK_BANDS = 0,       /* persistent cost-sorted stack-band units, one thread per 3D track */
  MOC_SCHED_ALG2 = 1,              /* Alg. 2 grid-stride over 3D tracks in Alg. 1 order (paper baseline) */
  MOC_SCHED_SERPENTINE = 2,        /* Alg. 2 over tracks sorted by segment count + §4.3 serpentine */
  MOC_SCHED_STACK_COLLECTIVE = 3   /* one warp per band of a z-stack, lanes own (2D segment, layer)
                                      cells, exponentials shared per cell, register tallies:
                                      P:68, Eqs. 6-11; SURVEY §8(f) NEXT-2 */
};
typedef struct {
  int32_t schedule;     /* MOC_SCHED_* */
  int32_t threads, blocks;  /* Alg. 2 launch shape (P:146 default 512 x 512); 0 = default */
  int32_t deterministic;    /* reserved (0) */
  int32_t tile_cells;       /* schedule 0: cap on FSR cells per shared-memory tally chunk
                               (0 = as many as fit; small values force many chunks, for tests) */
  int32_t exp_mode;         /* schedule 0 only (else MOC_E_PARAM): 0 = pure on-the-fly (OTF); 1 = EXP/OTF hybrid of §4.2:
                               work units sorted by segment count descending are preloaded as stored
                               segments while the cumulative size stays within exp_fraction of the
                               budget, the rest is traced on the fly */
  int32_t exp_budget_mb;    /* EXP budget in MiB (0 = free device memory after allocation) */
  double exp_fraction;      /* fraction of the budget (0 = the paper's 0.8) */
  int32_t sc_lanes_per_cell; /* schedule 3: lanes per (2D segment, layer) cell, 1/2/4/8 (0 = per stack) */
  int32_t sc_psi_cap;        /* schedule 3: cap on the boundary-psi band capacity per warp in
                                members (0 = fill the shared memory of the stack's CTAs per SM) */
  int32_t v2_lane_stride;    /* schedule 0: force the member stride between the lanes of a warp to
                                1, 2, 4 or 8 (0 = per unit from the stack's dz; for tests) */
  int32_t no_graph;          /* 1: launch every iteration's kernels individually instead of
                                replaying a captured CUDA graph (debugging / A-B) */
  int32_t gauss_seidel;      /* schedule 3, 5-7 groups, one GPU (not in the
                                paper): one boundary-psi buffer updated in place, so a track whose
                                linked predecessor was swept earlier in the same sweep starts from
                                its fresh outgoing psi (asynchronous Gauss-Seidel along the 3D
                                links) instead of last iteration's (Jacobi, Q9).  Halves the psi
                                memory; the iterates differ (parity at convergence only), order
                                and therefore results are not bitwise reproducible run to run */
  int32_t sc_ctas_per_sm;    /* schedule 3: CTAs per SM of the sweep for every stack, 3, 4 or 5
                                (else MOC_E_PARAM); 0 = per stack, the most CTAs per SM (more
                                resident warps, smaller shared-memory psi bands) that do not cut
                                the stack into more bands than 3 CTAs per SM do */
} moc_solver_opts;

/* Upload the laydown to `device`, allocate HBM state (boundary psi double buffer,
 * FSR arrays), compute track-based FSR volumes and exact per-track segment counts on
 * the device.  comm == NULL means one GPU; with world > 1 this rank sweeps its
 * contiguous cost-balanced share of the stacks.
 * MOC_E_CAPACITY: device memory exhausted, more than 255 axial layers, an axial mesh too
 * fine for the shared-memory tally tile, or (5-8 groups) more than 2^26 FSRs, the limit
 * of the 1D texture the sweep gathers FSR sources through.  The small per-problem tables
 * (cross sections, axial planes) live in the device's constant bank and are re-uploaded
 * by whichever solver runs next on the device (one solver active per device at a time). */
int moc_solver_create(moc_solver** out, moc_problem* p, int device, void* cuda_stream,
                      const moc_comm_desc* comm, const moc_solver_opts* opts);
int moc_solver_destroy(moc_solver* s);
const char* moc_solver_last_error(const moc_solver* s);

/* Run n_iter power iterations (A3..A8 on the device).  Initial state phi = 1, k = 1,
 * psi = 0 (Q11).  world > 1 needs backend MOC_COMM_NCCL or a registered exchange callback
 * (else MOC_E_STATE).  Each iteration is one CUDA-graph replay (captured on first use per
 * Jacobi buffer parity) unless opts.no_graph or a host callback is involved.  Writes the
 * final k and fission-source residual; synchronises the stream once at the end to read
 * them (16 bytes D2H). */
int moc_iterate(moc_solver* s, int32_t n_iter, double* k_out, double* residual_out);

typedef struct { double tol_k, tol_src; int32_t max_iter, check_every; } moc_solve_opts;
typedef struct { double k; double residual; int32_t iterations; int32_t converged; } moc_result;
/* Iterate until |dk| < tol_k and residual < tol_src.  MOC_E_NOCONV if max_iter hit. */
int moc_solve(moc_solver* s, const moc_solve_opts* o, moc_result* r);
int moc_reset(moc_solver* s); /* back to phi = 1, k = 1, psi = 0 */

/* Replace the cross sections of a live solver (same n_mat, G; host fp64 arrays laid out
 * as in moc_set_materials), e.g. for multiphysics feedback between outer iterations.
 * Stream-ordered host->device copy (the flux state is kept). */
int moc_solver_update_materials(moc_solver* s, const double* sigma_t, const double* sigma_s,
                                const double* nu_sigma_f, const double* chi);

/* Results (host, caller-owned). phi [J][G] normalised to sum_j V_j F_j = 1. */
int moc_get_scalar_flux(moc_solver* s, double* phi);
/* FSR volumes [J] (cm^3): vol_track = the track estimate V_j = sum_{a,n} W_{a,n}/(2 pi)
 * A_perp sum L over every 3D segment in j (App. A.5, device walk); vol_analytic = ring /
 * moderator area x layer height.  Either pointer may be NULL (not both). */
int moc_get_fsr_volumes(moc_solver* s, double* vol_track, double* vol_analytic);
int moc_get_history(moc_solver* s, double* k_hist, double* res_hist, int32_t cap, int32_t* n);
int moc_get_balance(moc_solver* s, double* production, double* absorption, double* leakage);

/* Device OTF walk per 3D track: merged segment count and FNV-1a-64 hash of the FSR id
 * sequence (uint32 little-endian bytes), plus the sum of lengths (parity vs oracle). */
int moc_device_trace_checksums(moc_solver* s, int64_t first, int64_t n, int32_t* nseg,
                               uint64_t* hash, double* suml);

/* One sweep of the schedule-3 (stack-collective) kernel in checksum mode: for every slot
 * (2*track + dir) the number of 3D segments the kernel applied Eq. 3 to and the FNV-1a-64
 * hash of their FSR ids in travel order (dir 1 = the reverse of dir 0).  nseg/hash are
 * [2*n_tracks3d] host arrays.  The sweep reads the current state and writes only scratch
 * state (the next psi buffer and the tally, both rewritten by the next iteration); k,
 * phi and the current psi are unchanged.  MOC_E_STATE unless schedule == 3. */
int moc_sweep_checksums(moc_solver* s, int32_t* nseg, uint64_t* hash);

/* Device probe of the sweep's Eq. 3 arithmetic: for host fp32 arrays of length n
 * returns dpsi = (psi - q)(1 - e^{-sigma_t len}) and psi_out = psi - dpsi exactly as the sweep
 * kernel evaluates them (ex2.approx on sigma_t log2(e) len, one FFMA).  For accuracy tests. */
int moc_attenuation_probe(int device, int64_t n, const float* psi, const float* q, const float* sigma_t,
                          const float* len, float* psi_out, float* dpsi);

typedef struct {
  int64_t n_segs3d;          /* exact merged 3D segment count (device walk) */
  int64_t n_integrations;    /* per sweep: 2 * n_segs3d * G */
  double sweep_ms_last;      /* CUDA-event time of the last sweep kernel */
  double iter_ms_last;       /* CUDA-event time of the last full iteration */
  int64_t launches_per_iter; /* kernels launched per iteration */
  double setup_ms;           /* moc_solver_create wall time */
  int64_t device_bytes;      /* HBM allocated by this handle */
  int64_t exp_segments;      /* merged 3D segments preloaded by the EXP option (0 = pure OTF) */
  int64_t exp_bytes;         /* bytes of the EXP record store */
  int64_t emitted_last;      /* merged segment-direction applications of Eq. 3-4 in the last
                                iteration's sweep on this rank (integrity counter: equals
                                2 * n_segs3d on one GPU); -1 if it could not be read */
  int64_t sc_units[3];       /* schedule 3: work units swept at 3, 4 and 5 CTAs per SM (one
                                sweep launch per non-empty group) */
} moc_timings;
int moc_get_timings(moc_solver* s, moc_timings* t);

/* Multi-GPU plumbing: device pointers of this rank's tally (fp32 [J][Gp],
 * to be sum-all-reduced by the caller after each sweep) and of the halo send/recv
 * buffers for cut-crossing boundary psi. */
typedef struct {
  void* tally; int64_t tally_elems;
  void* halo_send; void* halo_recv; int64_t halo_elems;
} moc_comm_buffers;
int moc_solver_comm_buffers(moc_solver* s, moc_comm_buffers* b);
/* per-peer element counts (floats) of this rank's halo send / recv buffers, [world] each,
 * in peer order (the layout all_to_all expects) */
int moc_solver_halo_counts(moc_solver* s, int64_t* send_elems, int64_t* recv_elems);

/* Fine-grained iteration steps for the multi-GPU driver: sweep (A3-A6) then, after the
 * caller's allreduce of the tally / halo exchange, finish (A7). */
int moc_iteration_sweep(moc_solver* s);
int moc_iteration_finish(moc_solver* s);

/* Backend MOC_COMM_CALLER with world > 1: host callback that performs the exchange on the
 * buffers of moc_solver_comm_buffers (the stream is synchronised before the call); with it
 * registered, moc_iterate / moc_solve run multi-rank.  Return 0 on success (else the
 * iteration fails with MOC_E_NCCL).  fn == NULL unregisters. */
typedef int (*moc_exchange_fn)(void* ctx);
int moc_solver_set_exchange(moc_solver* s, moc_exchange_fn fn, void* ctx);

#ifdef __cplusplus
}
#endif
#endif
