// sweep_v2.cuh — persistent, cost-sorted stack-band OTF sweep for sm_100a
// (the paper's §4.3 load balancing rebuilt for Blackwell;
// §4.2 EXP preloading as an option).
//
// Work unit = (z-stack (t, n), band of <= 256 consecutive members).  One CTA of 256
// threads takes units from a global atomic counter (units sorted by exact segment
// count, descending — P:228 "sorting ... in descending order according to segment
// count" — so the tail is short).  Per unit the CTA
//   1. stages t's 2D segments (s_end f64, region u32) in shared memory: the only
//      geometry the OTF walk reads ("retain exclusively the 2D segments");
//   2. derives the band's tally window: for every 2D segment k the band occupies a
//      contiguous layer range [lo_k, lo_k + w_k) (Eq. 5 is linear in i and s), so the
//      unit's FSR cells (k, layer) are packed by an exclusive scan of w_k, and cut
//      into chunks of consecutive k whose cells fit the shared-memory tile;
//   3. each thread walks one track on the fly (otf.h rules, resumable at chunk
//      boundaries), forward chunk by chunk, then backward through the chunks in
//      reverse, applying Eq. 3 per merged segment and group and accumulating dpsi into
//      the chunk's tile.  Units preloaded by the EXP option replay stored 8-byte
//      records {2D segment, layer, material, length} in both directions instead (on
//      B200 this measured slower than regenerating the geometry: DESIGN.md §5).
//      Tally accumulation uses native u32 shared atomics (ATOMS.ADD) in 2^21-scaled
//      fixed point: r = fma(dpsi, scale, 1.5*2^23) has bits 0x4B400000 +
//      round(dpsi*scale); the tile sums raw bits plus a per-cell segment count and the
//      flush subtracts count * 0x4B400000 (mod 2^32).  scale = 2^21 / bound with bound
//      >= max |dpsi| over the unit (dpsi = (psi - q)(1 - e^-tau), psi stays between the
//      incoming psi and the sources under the 2D track), so terms and sums are exact-range;
//   4. after each chunk, flushes its cells: c_{a,n} * sum -> tally[j][g] with
//      red.global.add.v4.f32, re-zeroing them for the next chunk.
// Shared-memory float atomics compile to a CAS loop on sm_100a (measured 9.9 vs 54
// lanes/clk/SM for u32 ATOMS, profiles/micro_r1.jsonl) — hence the fixed point.
#pragma once

namespace {

#ifndef MOC_V2_CTAS_PER_SM
#define MOC_V2_CTAS_PER_SM 4
#endif
#ifndef MOC_V2_THREADS
#define MOC_V2_THREADS 256
#endif
constexpr int kV2Threads = MOC_V2_THREADS;  // one stack band of up to this many members per CTA
constexpr int kV2MinBlocks = MOC_V2_CTAS_PER_SM;  // CTAs per SM the register/smem budget targets
constexpr int kMaxK = 512;                    // max 2D segments per 2D track (host-checked)
constexpr int kMaxPlanes = 256;               // axial planes staged in shared memory (host-checked)
constexpr uint32_t kMagicBits = 0x4B400000u;  // bits of 1.5 * 2^23
constexpr float kMagic = 12582912.0f;         // 1.5 * 2^23
constexpr float kFixOne = 2097152.0f;         // 2^21: max |term| in fixed point
constexpr uint64_t kNoExp = ~0ull;
// tile words receive bits(dpsi' + 1.5 * 2^23) - 0x4B400000 (offset-free fixed-point codes:
// an IADD per group instead of a per-cell count atomic removing the offset at the flush)
static_assert(kMaxPlanes == sizeof(c_planes) / sizeof(double), "c_planes sized for kMaxPlanes");
// epsilon_L in the constant bank: DSETP reads it as an operand, where the immediate form
// would cost two uniform moves per raw piece (same value as otf.h kEpsL)
__constant__ double c_epsL = kEpsL;

// per-kernel shared tables; the per-unit tables share the dynamic buffer with the tile
__shared__ double sh_planes[kMaxPlanes];  // axial planes
__shared__ __align__(16) float sh_sig[kMaxMat * kMaxG];  // sigma_t * log2(e), [m][GP]
__shared__ float sh_iscale[kMaxG];
__shared__ float sh_scale[kMaxG];
__shared__ unsigned sh_max[kMaxG];

// Per 2D segment k of the unit's 2D track, one 16-byte record per walk direction: the
// crossing the walk meets next in k (forward table: s at the end of k; backward table:
// s at its start) with k's FSR and tile-cell offsets, so a radial step is one LDS.128.
struct __align__(16) KSeg {
  double s;
  int kx;  // region(k) * NL: FSR j = kx + layer
  int ky;  // first tile cell of k - lo_k: cell = ky + layer
};

// Dynamic shared memory of one CTA: the per-unit tables from the bottom (TF[nk] at offset
// 0, so a radial step's address is one shift from the buffer base | TB[nk] | base[nk+1] |
// chunk[nk+1]), then the tile [cap][cell_words] u32 at a per-solver offset (tile_off >= the
// largest unit's tables; GP group words + the segment count, the odd stride keeping lanes
// in different cells on different banks).  The tile never moves and stays zero between
// flushes.
__host__ __device__ constexpr int unit_table_bytes(int nk) { return 32 * nk + ((8 * (nk + 1) + 15) & ~15); }
// (Round-1 A/B variants that measured slower -- staged chunk sources, tile copies, packed
// fp32 pairs, F2I codes, texture radial records, constant-bank planes, lane skew,
// interleaved units, early advance, branch-free advance -- were removed from this file;
// they live at git tag round1-v2-ab-options, their timings in DESIGN.md.)
// tile cell stride in u32 words: the G group words rounded up to an odd count, so lanes in
// consecutive cells hit distinct banks
__host__ __device__ constexpr int cell_words(int G, int GP) { return G | 1; }
__host__ __device__ constexpr int tile_cell_bytes(int G, int GP) { return 4 * cell_words(G, GP); }
__host__ __device__ constexpr int cell_bytes(int G, int GP) { return tile_cell_bytes(G, GP); }
__host__ __device__ constexpr int cap_max_cells(int G, int GP) { return ((224000 / kV2MinBlocks) / cell_bytes(G, GP)) & ~7; }

// members i0, i0 + step, ..., i0 + (n - 1) step of one z-stack (step > 1 interleaves
// sibling units over one range, spreading a warp's lanes further apart in z)
struct Unit {
  uint32_t stack, i0, n, step;
};

// merged segment record: meta = kk | layer << 10 | material << 18, plus the 3D length
struct __align__(8) Rec {
  uint32_t meta;
  float L;
};
__device__ __forceinline__ uint32_t rec_meta(int kk, int l, int m) {
  return (uint32_t)kk | ((uint32_t)l << 10) | ((uint32_t)m << 18);
}

struct V2Args {
  DevData d;
  const Unit* units;
  const uint64_t* unit_exp;  // record-store offset (in records) per unit, kNoExp = OTF
  uint32_t n_units;
  uint32_t* counter;
  const uint32_t* link;
  const uint8_t* mat;
  const float* qt;      // [J][GP]; for G < GP slot G carries the FSR's material index bits
  cudaTextureObject_t qtex;  // qt as a float4 texture (GP = 8: the gather on the TEX pipe)
  const float* qmax_t;  // [T2][GP] max qtilde over the FSRs under 2D track t
  const float* psi_in;
  float* psi_out;
  float* tally;         // fp32 [J][GP]
  double* sc;
  const Rec* store;     // EXP record store
  const uint32_t* cost; // exact merged segments per track (EXP replay length)
  int tile_off;         // byte offset of the tile in the dynamic buffer (multiple of 16)
  int cap_cells;        // tile capacity in cells (multiple of 8)
  double h_lane;        // thinnest axial layer / 3 (lane_lg_of)
  int lane_lg;          // forced log2 lane stride, -1 = per unit (lane_lg_of)
  int* err;
  const uint32_t* slot_first;  // per stack: first psi / link slot pair of its members on this rank
};

// Stack member (within the unit's band) walked by thread tid, for a lane stride of
// 2^lg members: groups of 2^lg warps cover 32 * 2^lg consecutive members, lane i of a
// warp taking every 2^lg-th.  Neighbouring z-members have nearly equal 3D lengths (busy
// SIMT lanes: lane efficiency 0.90 contiguous vs 0.76 spread over the band on cfg4,
// tools/lane_eff.py) but cross the same FSR at the same time (same-address shared
// atomics serialise); the stride trades the two.  lane_lg_of picks it per unit from the
// stack's member spacing dz: the smallest 2^lg (<= warps per CTA) with 2^lg dz >= h_min / 3 (about
// 3 lanes per layer thickness) while 2^lg warps stay busy on the band's n members
// (A/B over the divisor and forced strides on cfg4 / cfg5: profiles/README.md).
__device__ __forceinline__ int lane_lg_of(double dz, double h_lane, int forced, int n) {
  if (forced >= 0) return forced;
  int lg = 0;
  // 2^(lg+1) warps busy, and 2^(lg+1) warps must exist in the CTA
  while ((64 << lg) <= kV2Threads && (double)(1 << lg) * dz < h_lane && (64 << lg) <= n + 31) ++lg;
  return lg;
}
__device__ __forceinline__ int member_of(int tid, int lg) {
  const int w = tid >> 5, lane = tid & 31;
  return ((w >> lg) << (5 + lg)) + (lane << lg) + (w & ((1 << lg) - 1));
}

// a value the compiler must keep in a register rather than re-derive at every use (it
// otherwise recomputes shared-window bases from SR_CgaCtaId inside the hot loop)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float e) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(e)
               : "memory");
}

// Eq. 3 for one segment and group: returns dpsi = (psi - qtilde)(1 - e^{-tau}) with
// tau = sigma_t L evaluated as 2^{-(sigma_t log2 e) L} (ex2.approx.ftz) and the
// difference folded into one FFMA: dpsi = d - d * E.
__device__ __forceinline__ float attenuation_dpsi(float psi, float q, float sig_log2e, float L) {
  const float E = ex2_approx(-sig_log2e * L);
  const float dd = psi - q;
  return fmaf(-dd, E, dd);
}

template <int GP>
__device__ __forceinline__ void load_q(const float* qt, int64_t j, float* q) {
  if constexpr (GP == 8) {
    // one 256-bit load per FSR record (LDG.E.ENL2.256): half the load instructions and L1
    // data-pipe wavefronts of two LDG.128 — the L1 data pipe is the sweep's busiest unit
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(q[0]), "=f"(q[1]), "=f"(q[2]), "=f"(q[3]), "=f"(q[4]), "=f"(q[5]), "=f"(q[6]), "=f"(q[7])
        : "l"(qt + j * GP));
  } else if constexpr (GP % 4 == 0) {
#pragma unroll
    for (int h = 0; h < GP / 4; ++h) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(qt + j * GP) + h);
      q[4 * h] = x.x;
      q[4 * h + 1] = x.y;
      q[4 * h + 2] = x.z;
      q[4 * h + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int h = 0; h < GP; ++h) q[h] = __ldg(qt + j * GP + h);
  }
}

// first k in [0, nk-1] with T[k].s > s  /  >= s  (otf_seg_after / otf_seg_upto on the
// forward table, whose s is the cumulative end of each 2D segment)
__device__ __forceinline__ int kseg_after(const KSeg* T, int nk, double s) {
  int lo = 0, hi = nk - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (T[mid].s > s) hi = mid; else lo = mid + 1;
  }
  return lo;
}
__device__ __forceinline__ int kseg_upto(const KSeg* T, int nk, double s) {
  int lo = 0, hi = nk - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (T[mid].s >= s) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// Eq. 3 + Eq. 4 for one merged segment in all groups.  psi is carried in the unit's
// fixed-point units (psi' = psi * scale_g, scale_g = 2^21 / bound_g), so the tally term
// dpsi' = (psi' - q scale_g)(1 - e^{-tau}) is already scaled and its fixed-point code is
// one FADD with the 1.5 * 2^23 magic: per group FMUL, MUFU.EX2, 2 FFMA, 2 FADD, ATOMS.
// Storage is in float2 pairs; for odd G the last pair's upper half is a dead lane (scale 0,
// psi 0).
template <int G, int GP>
struct Physics {
  static constexpr int NP = (G + 1) / 2;
  float2 psi2[NP];
  float2 scl2[NP];
  const uint8_t* mat;
  const float* qt;
  cudaTextureObject_t qtex;
  int cb;        // first cell of the current chunk (tile cell 0)
  int tile_off;  // byte offset of the tile in the dynamic buffer
  uint32_t tsa;  // shared address of the tile minus cb cells (cell pc at tsa + pc * 4 cell_words)
  uint32_t ssa;  // shared address of sh_sig
  uint32_t psa;  // shared address of sh_planes
  uint32_t nem;  // emissions (the tile has no per-cell count)

  // axial plane i: an LDS.64 from the register-held shared base
  __device__ __forceinline__ double plane(int i) const {
    double z;
    asm("ld.shared.f64 %0, [%1];" : "=d"(z) : "r"(psa + 8u * (uint32_t)i));
    return z;
  }
#ifdef MOC_DEBUG_WALK
  int dbg_lo, dbg_hi, dbg_dir;
#endif

  __device__ __forceinline__ float& psi(int g) { return (g & 1) ? psi2[g >> 1].y : psi2[g >> 1].x; }
  __device__ __forceinline__ float& scl(int g) { return (g & 1) ? scl2[g >> 1].y : scl2[g >> 1].x; }

  __device__ __forceinline__ void emit(int pc, int m, const float* q, float Lf) {
#ifdef MOC_DEBUG_WALK
    if (pc < dbg_lo || pc >= dbg_hi) {
      printf("bad emit: blk %d tid %d dir %d pc %d chunk [%d,%d) m %d L %g\n", blockIdx.x, threadIdx.x, dbg_dir, pc,
             dbg_lo, dbg_hi, m, Lf);
      return;
    }
#endif
    // 32-bit shared-window addresses held in registers (tile base pre-offset by the
    // chunk's first cell; Sigma_t table base): one IMAD / LEA per emit instead of the
    // compiler re-deriving both generic->shared bases (S2UR CgaCtaId, ULEA, LDC) each time
    const uint32_t ca = tsa + (uint32_t)pc * (4u * cell_words(G, GP));
    // Sigma_t from the constant bank (LDC through the constant cache, off the L1 data pipe;
    // lanes mostly share the material, else the load replays per distinct address)
    float sg[GP];
#pragma unroll
    for (int h = 0; h < GP; ++h) sg[h] = h < G ? c_sigt2[m * kMaxG + h] : 0.f;
    ++nem;
#define MOC_TILE_ADD(g, v) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(ca + 4u * (g)), "r"((v) - kMagicBits))
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float E = ex2_approx(-sg[g] * Lf);
      const float dd = fmaf(-q[g], scl(g), psi(g));
      const float dl = fmaf(-dd, E, dd);  // (psi' - q')(1 - E)
      psi(g) -= dl;
      MOC_TILE_ADD(g, __float_as_uint(dl + kMagic));
    }
#undef MOC_TILE_ADD
  }
};

// On-the-fly walk state (same piece and merge rules as otf.h, reading Q22b).  The
// next radial and axial crossings are cached (s_rad with k's offsets kx / ky from one
// KSeg load, s_ax) and refreshed after each step.  Pending merged segment: pc = its
// tile cell (-1 = none; cells of 2D segment k are [base_k, base_k+1), so chunk
// membership is a compare on pc), pm / pq = material and source loaded when it was set
// (one raw piece ahead of use).  carry = sliver length not yet attached to a long
// piece; fkl = first sliver (k | l << 16) seen while nothing is pending (all-sliver
// tracks only, else -1).
template <int G, int GP>
struct WalkState {
  double s, s_end, s_rad, s_ax;
  int k, l, kx, ky, pc, pm, fkl, done;
  float pL, carry;
  float pq[GP];

  __device__ __forceinline__ void load(const KSeg& e) {
    const int4 v = *reinterpret_cast<const int4*>(&e);  // one LDS.128
    s_rad = __hiloint2double(v.y, v.x);
    kx = v.z;
    ky = v.w;
  }
  // radial step to 2D segment k in the hot loop: one LDS.128
  __device__ __forceinline__ void step(const KSeg* T, int kk) { load(T[kk]); }
  // make raw piece (k, l) the pending segment: its cell, source and material
  __device__ __forceinline__ void set_pending(int jx, int cy, int ll, const uint8_t* mat, const float* qt,
                                              cudaTextureObject_t qtex) {
    pc = cy + ll;
    const int64_t j = (int64_t)(jx + ll);
    if constexpr (GP == 8) {
      // the source gather through the texture pipe (its own L1TEX data path; the LSU
      // data pipe carries the tally atomics; the solver refuses problems whose sources
      // exceed a 1D texture, > 2^26 FSRs at GP = 8)
      const float4 a = tex1Dfetch<float4>(qtex, (int)(2 * j)), b = tex1Dfetch<float4>(qtex, (int)(2 * j + 1));
      pq[0] = a.x; pq[1] = a.y; pq[2] = a.z; pq[3] = a.w;
      pq[4] = b.x; pq[5] = b.y; pq[6] = b.z; pq[7] = b.w;
    } else {
      load_q<GP>(qt, j, pq);
    }
    if constexpr (G < GP) pm = __float_as_int(pq[G]);  // material index rides in the pad slot
    else pm = mat[j];
  }
  template <class PH>
  __device__ __forceinline__ void emit_to(PH& ph, float L) {
    ph.emit(pc, pm, pq, L);
  }
};

// forward OTF: advance until the pending segment's cell is >= c_hi (a later chunk) or
// the track ends.  UP: the track climbs (cot > 0).
template <int G, int GP, bool UP>
__device__ __forceinline__ void walk_fwd_chunk(WalkState<G, GP>& w, Physics<G, GP>& ph, const KSeg* TF, double z0,
                                               double tn, double isn, int c_hi) {
  while (true) {
    if (w.pc >= c_hi) return;
    if (w.done) {
      if (w.pc >= 0) {
        w.emit_to(ph, w.pL);
        w.pc = -1;
        w.fkl = -1;  // the track is finished: no all-sliver emission follows
      } else if (w.fkl >= 0) {  // all-sliver track: one segment at its first piece
        const KSeg e = TF[w.fkl & 0xffff];
        if (e.ky + (w.fkl >> 16) >= c_hi) return;
        w.set_pending(e.kx, e.ky, w.fkl >> 16, ph.mat, ph.qt, ph.qtex);
        w.emit_to(ph, w.carry);
        w.pc = -1;
        w.fkl = -1;
      }
      return;
    }
    const bool rad = w.s_rad <= w.s_ax;
    double sn = rad ? w.s_rad : w.s_ax;
    const bool last = sn >= w.s_end;
    sn = last ? w.s_end : sn;
    const double L3d = (sn - w.s) * isn;
    const float L3 = (float)L3d;
    if (L3d < c_epsL) {
      if (w.pc >= 0) {
        w.pL += L3;  // a sliver merges into the segment before it
      } else {
        w.carry += L3;  // a leading sliver run merges forward
        if (w.fkl < 0) w.fkl = w.k | (w.l << 16);
      }
    } else {
      if (w.pc >= 0) w.emit_to(ph, w.pL);
      w.pL = L3 + w.carry;
      w.carry = 0.f;
      w.set_pending(w.kx, w.ky, w.l, ph.mat, ph.qt, ph.qtex);
    }
    if (last) {
      w.done = 1;
    } else {
      w.s = sn;
      if (rad) {
        ++w.k;
        w.step(TF, w.k);
      } else {
        w.l += UP ? 1 : -1;
        w.s_ax = (ph.plane(w.l + (UP ? 1 : 0)) - z0) * tn;
      }
    }
  }
}

// backward OTF: retreat until the pending segment's cell is < c_lo (an earlier chunk)
// or the track start.  Short raw pieces are carried into the next long one, so the
// merged list is the reverse of the forward one (reading Q22b).
template <int G, int GP, bool UP>
__device__ __forceinline__ void walk_bwd_chunk(WalkState<G, GP>& w, Physics<G, GP>& ph, const KSeg* TF,
                                               const KSeg* TB, double z0, double tn, double isn, int c_lo) {
  while (true) {
    if ((unsigned)w.pc < (unsigned)c_lo) return;
    if (w.done) {
      if (w.pc >= 0) {
        w.emit_to(ph, w.pL + w.carry);
        w.pc = -1;
        w.fkl = -1;  // the track is finished: no all-sliver emission follows
      } else if (w.fkl >= 0) {  // all-sliver track: emitted in the chunk of its first piece
        const KSeg e = TF[w.fkl & 0xffff];
        if (e.ky + (w.fkl >> 16) < c_lo) return;
        w.set_pending(e.kx, e.ky, w.fkl >> 16, ph.mat, ph.qt, ph.qtex);
        w.emit_to(ph, w.carry);
        w.pc = -1;
        w.fkl = -1;
      }
      return;
    }
    const bool rad = w.s_rad >= w.s_ax;
    double sp = rad ? w.s_rad : w.s_ax;
    const bool last = sp <= w.s_end;
    sp = last ? w.s_end : sp;
    const double L3d = (w.s - sp) * isn;
    const float L3 = (float)L3d;
    if (L3d < c_epsL) {
      w.carry += L3;
      if (w.pc < 0) w.fkl = w.k | (w.l << 16);  // the forward-first sliver wins
    } else {
      if (w.pc >= 0) w.emit_to(ph, w.pL);
      w.pL = L3 + w.carry;
      w.carry = 0.f;
      w.set_pending(w.kx, w.ky, w.l, ph.mat, ph.qt, ph.qtex);
    }
    if (last) {
      w.done = 1;
    } else {
      w.s = sp;
      if (rad) {
        --w.k;
        w.step(TB, w.k);
      } else {
        w.l -= UP ? 1 : -1;
        w.s_ax = (ph.plane(w.l + (UP ? 0 : 1)) - z0) * tn;
      }
    }
  }
}

// Replay of a record stream (stride kV2Threads between a thread's consecutive records)
// in direction dq = +1 (forward) or -1 (backward).  Records are loaded kRecAhead ahead
// (HBM latency) and the next record's source one ahead, so the chain record -> table ->
// source never stalls the Eq. 3 work of the current record.
constexpr int kRecAhead = 2;  // (2 / 3 / 4 measured 23.9 / 24.5 / 24.4 ms on cfg4)
template <int GP>
struct Replay {
  const Rec* rs;
  const KSeg* TF;
  int q, dq;     // next record index to load; step (records outside [0, nrec) are not read)
  int nrec;      // this thread's records
  int left;      // records still to apply
  Rec buf[kRecAhead];  // buf[0] = next to apply
  int cpc;       // tile cell of buf[0]
  float cq[GP];  // source of buf[0]

  __device__ __forceinline__ Rec load_next() {
    Rec x{0u, 0.f};
    if ((unsigned)q < (unsigned)nrec) x = rs[(size_t)q * kV2Threads];
    q += dq;
    return x;
  }
  __device__ __forceinline__ void prepare(const float* qt) {
    if (left > 0) {
      const int kk = buf[0].meta & 1023, l = (buf[0].meta >> 10) & 255;
      const KSeg e = TF[kk];
      cpc = e.ky + l;
      load_q<GP>(qt, (int64_t)(e.kx + l), cq);
    }
  }
  __device__ __forceinline__ void start(int q0, int n, const float* qt) {
    q = q0;
    nrec = n;
    left = n;
#pragma unroll
    for (int i = 0; i < kRecAhead; ++i) buf[i] = load_next();
    prepare(qt);
  }
  __device__ __forceinline__ void advance(const float* qt) {
#pragma unroll
    for (int i = 0; i + 1 < kRecAhead; ++i) buf[i] = buf[i + 1];
    buf[kRecAhead - 1] = load_next();
    --left;
    prepare(qt);
  }
};

// apply records while they belong to the chunk [k_lo, k_hi)
template <int G, int GP>
__device__ __forceinline__ void replay_chunk(Replay<GP>& r, Physics<G, GP>& ph, int k_lo, int k_hi) {
  while (r.left > 0) {
    const Rec cur = r.buf[0];
    const int kk = cur.meta & 1023;
    if (kk < k_lo || kk >= k_hi) return;
    const int m = cur.meta >> 18, pc = r.cpc;
    float q[GP];
#pragma unroll
    for (int h = 0; h < GP; ++h) q[h] = r.cq[h];
    r.advance(ph.qt);  // look-ahead loads overlap the physics below
    ph.emit(pc, m, q, cur.L);
  }
}

// one direction of one track through one chunk
template <int G, int GP, bool UP>
__device__ __forceinline__ void walk_chunk(int dir, WalkState<G, GP>& w, Physics<G, GP>& ph, const KSeg* TF,
                                           const KSeg* TB, double z0, double tn, double isn, int c_lo, int c_hi) {
  if (dir == 0) walk_fwd_chunk<G, GP, UP>(w, ph, TF, z0, tn, isn, c_hi);
  else walk_bwd_chunk<G, GP, UP>(w, ph, TF, TB, z0, tn, isn, c_lo);
}

// largest k in [k_lo, k_hi) with base[k] <= c (the 2D segment owning tile cell c)
__device__ __forceinline__ int k_of_cell(const int* base, int k_lo, int k_hi, int c) {
  int lo = k_lo, hi = k_hi - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (base[mid] <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// EXP = false: on-the-fly sweep of the units past the preloaded prefix (the replay path
// is not compiled in, which keeps the register budget for the walk); EXP = true: replay
// of the preloaded units (§4.2), no walk code.  The two run back to back on the stream.
template <int G, int GP, bool EXP>
__global__ void __launch_bounds__(kV2Threads, kV2MinBlocks) k_sweep_v2(V2Args a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int cap = a.cap_cells;
  uint32_t* const cells = reinterpret_cast<uint32_t*>(dsm + a.tile_off);  // [cap][kCW]
  constexpr int kCW = cell_words(G, GP);
  __shared__ uint32_t s_unit;
  __shared__ int s_nchunk;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kV2Threads / 32;
  const DevData& d = a.d;
  for (int q = tid; q < kMaxMat * GP; q += blockDim.x) {
    const int m = q / GP, g = q - m * GP;
    sh_sig[q] = g < G ? c_sigt2[m * kMaxG + g] : 0.f;
  }
  for (int q = tid; q <= d.NL; q += blockDim.x) sh_planes[q] = d.planes[q];
  // the tile starts zeroed; each flush re-zeroes exactly the cells it consumed
  for (int q = tid; q < cap * kCW; q += blockDim.x) cells[q] = 0u;
  const float ps = (float)a.sc[SC_PSI_SCALE];
  const OtfView v{nullptr, nullptr, sh_planes, d.NL};
  double leak = 0.0;
  uint64_t nemit = 0;  // merged segment-direction emissions flushed by this thread

  while (true) {
    __syncthreads();
    if (tid == 0) s_unit = atomicAdd(a.counter, 1u);
    __syncthreads();
    const uint32_t u = s_unit;
    if (u >= a.n_units) break;
    const Unit U = a.units[u];
    const uint64_t exp_off = EXP ? a.unit_exp[u] : kNoExp;
    const int s = (int)U.stack;
    const int t = s / d.N, n = s - t * d.N;
    const int an = d.t_a[t] * d.N + n;
    const int64_t sb = d.t_seg[t];
    const int nk = (int)(d.t_seg[t + 1] - sb);
    const double dz = d.an_dz[an], cot = d.an_cot[an];
    const double z0b = d.st_z0[s];
    const double zf = z0b + (double)U.i0 * dz, zl = z0b + (double)(U.i0 + (U.n - 1) * U.step) * dz;
    // per-unit tables at the top of the dynamic buffer, the tile below them
    KSeg* const TF = reinterpret_cast<KSeg*>(dsm);
    KSeg* const TB = TF + nk;
    int* const base = reinterpret_cast<int*>(TB + nk);
    int* const chunk = base + nk + 1;
    // 1-2. stage the 2D segments, per-k layer windows of the band
    for (int kk = tid; kk < nk; kk += blockDim.x) {
      const double s1 = d.seg_send[sb + kk];
      const double s0 = kk ? d.seg_send[sb + kk - 1] : 0.0;
      const int kx = (int)d.seg_region[sb + kk] * d.NL;
      double zlo = cot > 0 ? zf + s0 * cot : zf + s1 * cot;
      double zhi = cot > 0 ? zl + s1 * cot : zl + s0 * cot;
      zlo = zlo > 0.0 ? zlo : 0.0;
      zhi = zhi < d.Z ? zhi : d.Z;
      int lo = 0, w = 0;
      if (zlo <= zhi) {
        lo = otf_layer_down(v, zlo);
        w = otf_layer_up(v, zhi) - lo + 1;
      }
      TF[kk] = KSeg{s1, kx, lo};  // ky completed after the scan
      TB[kk] = KSeg{s0, kx, lo};
      base[kk] = w;
    }
    if (tid < kMaxG) sh_max[tid] = 0u;
    __syncthreads();
    // 3. one track per thread (member_of: neighbouring members share a warp); its incoming
    //    psi loads are issued here so their HBM latency overlaps the scan below
    const int p = member_of(tid, lane_lg_of(dz * U.step, a.h_lane, a.lane_lg, (int)U.n));
    const bool active = p < (int)U.n;
    const uint32_t id = d.st_first[s] + U.i0 + (uint32_t)p * U.step;     // global track id (costs)
    const uint32_t sid = a.slot_first[s] + U.i0 + (uint32_t)p * U.step;  // this rank's numbering (psi, links)
    float fpsi[GP], bpsi[GP];
    if (active) {
      load_q<GP>(a.psi_in, (int64_t)(2 * sid), fpsi);
      load_q<GP>(a.psi_in, (int64_t)(2 * sid + 1), bpsi);
    } else {
#pragma unroll
      for (int g = 0; g < GP; ++g) fpsi[g] = bpsi[g] = 0.f;
    }
    if (warp == 0) {
      int carry = 0;
      for (int b0 = 0; b0 < nk; b0 += 32) {
        const int kk = b0 + lane;
        const int w = kk < nk ? base[kk] : 0;
        int x = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (kk < nk) {
          const int b = carry + x - w;
          base[kk] = b;
          const int ky = b - TF[kk].ky;
          TF[kk].ky = ky;
          TB[kk].ky = ky;
        }
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) base[nk] = carry;
      __syncwarp();
      // greedy chunks of consecutive k whose cells fit the tile: chunk [k0, k1) ends at
      // the first k1 with base[k1 + 1] - base[k0] > cap, found 32 k at a time by ballot
      int nc = 0, k0 = 0;
      while (k0 < nk) {
        const int b0 = base[k0];
        int k1 = nk;
        for (int kb = k0; kb < nk; kb += 32) {
          const int kk = kb + lane;
          const unsigned over = __ballot_sync(0xffffffffu, kk < nk && base[kk + 1] - b0 > cap);
          if (over) {
            k1 = kb + __ffs(over) - 1;
            break;
          }
        }
        if (k1 == k0) {  // a single 2D segment's window exceeds the tile
          if (lane == 0) atomicAdd(a.err, 1);
          k1 = nk;
        }
        if (lane == 0) chunk[nc] = k0;
        ++nc;
        k0 = k1;
      }
      if (lane == 0) {
        chunk[nc] = nk;
        s_nchunk = nc;
      }
    }
    Physics<G, GP> ph;
    ph.nem = 0u;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float m = fmaxf(fpsi[g], bpsi[g]) * ps;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) atomicMax(&sh_max[g], __float_as_uint(m));
    }
    __syncthreads();
    if (tid < G) {
      const float b = fmaxf(__uint_as_float(sh_max[tid]), a.qmax_t[(size_t)t * GP + tid]) * 1.0001f;
      sh_scale[tid] = b > 0.f ? kFixOne / b : 0.f;
      sh_iscale[tid] = b > 0.f ? b / kFixOne : 0.f;
    }
    __syncthreads();
    const int nchunk = s_nchunk;
#pragma unroll
    for (int g = 0; g < 2 * Physics<G, GP>::NP; ++g) ph.scl(g) = g < G ? sh_scale[g] : 0.f;
    ph.mat = a.mat;
    ph.qt = a.qt;
    ph.qtex = a.qtex;
    ph.tile_off = a.tile_off;
    const uint32_t tile_sa = (uint32_t)__cvta_generic_to_shared(dsm) + (uint32_t)a.tile_off;
    ph.ssa = opaque_u32((uint32_t)__cvta_generic_to_shared(sh_sig));
    ph.psa = opaque_u32((uint32_t)__cvta_generic_to_shared(sh_planes));
    const double tn = d.an_tan[an], isn = d.an_invsin[an], Lt = d.t_len[t];
    const double z0 = z0b + (double)(U.i0 + (uint32_t)p * U.step) * dz;
    const bool up = cot > 0;
    const float cw = d.an_c[an];
    constexpr bool otf = !EXP;
    double s_in = 0, s_out = 0;
    if constexpr (otf) {
      TrackGeo tg;
      tg.z0 = z0;
      tg.cot = cot;
      tg.tan = tn;
      tg.invsin = isn;
      tg.L = Lt;
      tg.Z = d.Z;
      tg.sb = 0;
      tg.se = nk;
      otf_clip(tg, s_in, s_out);
    }
#pragma unroll 1
    for (int dir = 0; dir < 2; ++dir) {
      {
        float pin[GP] = {};  // re-read (an L1/L2 hit): holding both directions' psi costs spills
        if (active) load_q<GP>(a.psi_in, (int64_t)(2 * sid + dir), pin);
#pragma unroll
        for (int g = 0; g < 2 * Physics<G, GP>::NP; ++g) ph.psi(g) = active && g < G ? pin[g] * ps * ph.scl(g) : 0.f;
      }
      WalkState<G, GP> w;
      Replay<GP> r;
      if constexpr (otf) {
        w.done = !active;
        w.carry = 0.f;
        w.pc = -1;
        w.pm = 0;
        w.fkl = -1;
        w.pL = 0.f;
        if (dir == 0) {
          w.s = s_in;
          w.s_end = s_out;
          if (s_in > 0.0) {
            w.l = up ? 0 : d.NL - 1;
            w.k = kseg_after(TF, nk, s_in);
          } else {
            w.l = up ? otf_layer_up(v, z0) : otf_layer_down(v, z0);
            w.k = 0;
          }
          w.load(TF[w.k]);
          w.s_ax = (sh_planes[up ? w.l + 1 : w.l] - z0) * tn;
        } else {
          w.s = s_out;
          w.s_end = s_in;
          if (s_out < Lt) {
            w.l = up ? d.NL - 1 : 0;
            w.k = kseg_upto(TF, nk, s_out);
          } else {
            const double z_out = z0 + Lt * cot;
            w.l = up ? otf_layer_down(v, z_out) : otf_layer_up(v, z_out);
            w.k = nk - 1;
          }
          w.load(TB[w.k]);
          w.s_ax = (sh_planes[up ? w.l : w.l + 1] - z0) * tn;
        }
      } else {
        // EXP: this thread's preloaded records, first to last or last to first
        const int nrec = active ? (int)a.cost[id] : 0;
        r.rs = a.store + exp_off + tid;
        r.TF = TF;
        r.dq = dir == 0 ? 1 : -1;
        r.start(dir == 0 ? 0 : nrec - 1, nrec, a.qt);
      }
#pragma unroll 1
      for (int ci = 0; ci < nchunk; ++ci) {
        const int c = dir == 0 ? ci : nchunk - 1 - ci;
        const int k_lo = chunk[c], k_hi = chunk[c + 1];
        const int cb = base[k_lo], ce = base[k_hi];
        ph.cb = cb;
        ph.tsa = opaque_u32(tile_sa - (uint32_t)cb * (4u * kCW));
#ifdef MOC_DEBUG_WALK
        ph.dbg_lo = cb;
        ph.dbg_hi = ce;
        ph.dbg_dir = dir;
#endif
        if constexpr (!otf) replay_chunk(r, ph, k_lo, k_hi);
        else if (up) walk_chunk<G, GP, true>(dir, w, ph, TF, TB, z0, tn, isn, cb, ce);
        else walk_chunk<G, GP, false>(dir, w, ph, TF, TB, z0, tn, isn, cb, ce);
        // the forward pass's last chunk is the backward pass's first: keep accumulating
        // (tile atomics commute) and flush both directions' sums once
        if (dir == 0 && ci == nchunk - 1) continue;
        __syncthreads();
        // 4. flush the chunk: c_{a,n} * fixed-point sums -> global tally (fp32 vector
        //    reductions), re-zeroing every consumed cell.  Each warp takes a contiguous
        //    eighth of the chunk's cells, lane-strided, so a lane's 2D segment k (for the
        //    cell's FSR) advances by a step or two per cell from one binary search.
        const int per = (ce - cb + nw - 1) / nw;  // nw is a compile-time constant
        float fsc[G];  // fixed point -> c_{a,n} * dpsi, per group
#pragma unroll
        for (int g = 0; g < G; ++g) fsc[g] = sh_iscale[g] * cw;
        const int x0 = warp * per + lane, x1 = min(ce - cb, (warp + 1) * per);
        int kc = x0 < x1 ? k_of_cell(base, k_lo, k_hi, cb + x0) : k_lo;
        for (int x = x0; x < x1; x += 32) {
          uint32_t* cp = cells + (size_t)x * kCW;
          uint32_t any = 0u;
          uint32_t sum[GP];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            sum[g] = cp[g];
            any |= sum[g];
          }
          if (!any) continue;
          while (base[kc + 1] <= cb + x) ++kc;
          const KSeg e = TF[kc];
          const int64_t j = (int64_t)(e.kx - e.ky) + cb + x;  // FSR of cell cb + x = ky + layer
          uint32_t raw[GP];
#pragma unroll
          for (int g = 0; g < GP; ++g) {
            raw[g] = g < G ? sum[g] : 0u;  // pad words are never written
            if (g < G) cp[g] = 0u;
          }
          float val[GP];
#pragma unroll
          for (int g = 0; g < GP; ++g) val[g] = g < G ? (float)(int)raw[g] * fsc[g] : 0.f;
          float* dst = a.tally + j * GP;
          if constexpr (GP % 4 == 0) {
#pragma unroll
            for (int h = 0; h < GP / 4; ++h)
              red_add_v4(dst + 4 * h, val[4 * h], val[4 * h + 1], val[4 * h + 2], val[4 * h + 3]);
          } else {
#pragma unroll
            for (int g = 0; g < G; ++g) atomicAdd(dst + g, val[g]);
          }
        }
        __syncthreads();
      }
      if (active) {
        const uint32_t out = a.link[2 * sid + dir];
        if (out != 0xffffffffu) {
          if constexpr (GP == 8 && G < GP) {
            // one 256-bit store of the whole slot (the pad word of psi is never read)
            float v[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) v[g] = g < G ? ph.psi(g) * sh_iscale[g] : 0.f;
            asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(a.psi_out + (size_t)out * GP),
                         "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                         : "memory");
          } else {
#pragma unroll
            for (int g = 0; g < G; ++g) a.psi_out[(size_t)out * GP + g] = ph.psi(g) * sh_iscale[g];
          }
        } else {
          float e = 0.f;
#pragma unroll
          for (int g = 0; g < G; ++g) e += ph.psi(g) * sh_iscale[g];
          leak += (double)(cw * e);
        }
      }
    }
    nemit += ph.nem;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    leak += __shfl_xor_sync(0xffffffffu, leak, o);
    nemit += __shfl_xor_sync(0xffffffffu, nemit, o);
  }
  if (lane == 0 && leak != 0.0) atomicAdd(&a.sc[SC_LEAK], leak);
  if (lane == 0 && nemit) atomicAdd(&a.sc[SC_NEMIT], (double)nemit);
}

// EXP preload ("the device function for generating characteristic lines is
// executed, and these data are stored on the GPU"): walk every track of a preloaded
// unit once and store its merged segments as records, lane-interleaved per unit.
__global__ void k_exp_generate(DevData d, const Unit* units, const uint64_t* unit_exp, uint32_t n_units,
                               const uint8_t* mat, Rec* store, double h_lane, int lane_lg) {
  const OtfView v = dev_view(d);
  for (uint32_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    if (unit_exp[u] == kNoExp) continue;
    const Unit U = units[u];
    const int p = member_of(threadIdx.x, lane_lg_of(d.an_dz[d.t_a[U.stack / d.N] * d.N + U.stack % d.N] * U.step,
                                                    h_lane, lane_lg, (int)U.n));
    if (p >= (int)U.n) continue;
    int s, an;
    const uint32_t id = d.st_first[U.stack] + U.i0 + (uint32_t)p * U.step;
    TrackGeo g = dev_track(d, id, s, an);
    Rec* rs = store + unit_exp[u] + threadIdx.x;
    int q = 0;
    otf_walk_fwd(v, g, [&](int64_t k, int l, double len) {
      const int64_t j = (int64_t)v.seg_region[k] * v.NL + l;
      rs[(size_t)q * kV2Threads] = Rec{rec_meta((int)(k - g.sb), l, mat[j]), (float)len};
      ++q;
    });
  }
}

// max qtilde over the layers of each radial region, then over the regions under each
// 2D track: the per-unit fixed-point bound's source part (see k_sweep_v2 step 3).
template <int G, int GP>
__global__ void k_region_qmax(int64_t n_regions, int NL, const float* qt, float* rmax) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_regions * G;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / G;
    const int g = (int)(q - r * G);
    float m = 0.f;
    for (int l = 0; l < NL; ++l) m = fmaxf(m, fabsf(qt[(r * NL + l) * GP + g]));  // |q|: robust bound
    rmax[r * GP + g] = m;
  }
}

template <int G, int GP>
__global__ void k_track_qmax(int64_t T2, const int64_t* t_seg, const uint32_t* seg_region, const float* rmax,
                             float* qmax_t) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < T2 * G; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = q / G;
    const int g = (int)(q - t * G);
    float m = 0.f;
    for (int64_t k = t_seg[t]; k < t_seg[t + 1]; ++k) m = fmaxf(m, rmax[(int64_t)seg_region[k] * GP + g]);
    qmax_t[t * GP + g] = m;
  }
}

// probe of the sweep's Eq. 3 arithmetic (tests: accuracy of the exponential path)
__global__ void k_attenuation_probe(int64_t n, const float* psi, const float* q, const float* sig, const float* len,
                                    float* psi_out, float* dpsi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = attenuation_dpsi(psi[i], q[i], sig[i] * 1.4426950408889634f, len[i]);
    dpsi[i] = d;
    psi_out[i] = psi[i] - d;
  }
}

__global__ void k_unit_cost(const Unit* units, uint32_t n_units, const uint32_t* st_first, const uint32_t* cost,
                            uint32_t* key, uint32_t* maxq) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n_units; u += gridDim.x * blockDim.x) {
    const Unit U = units[u];
    const uint32_t f = st_first[U.stack] + U.i0;
    uint32_t c = 0, mx = 0;
    for (uint32_t i = 0; i < U.n; ++i) {
      c += cost[f + i * U.step];
      mx = max(mx, cost[f + i * U.step]);
    }
    key[u] = c;
    maxq[u] = mx;
  }
}

}  // namespace
