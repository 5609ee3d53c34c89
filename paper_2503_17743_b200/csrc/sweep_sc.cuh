// sweep_sc.cuh — stack-collective OTF sweep with exponential reuse (
// the paper's per-z-stack tracing, Eqs. 6-11, rebuilt for sm_100a).
//
// Every member of a z-stack (t, n) is the same line z = z0 + i dz + s cot(theta) shifted
// by i dz (Eq. 5).  In the (s, z) plane of the stack, the FSRs crossed by its members are
// the rectangles "cell (k, l)" = [s_k, s_k+1] x [P_l, P_l+1] (2D segment k x axial layer l),
// and which members cross which cell, and with which 3D length, follows from index
// arithmetic (Eqs. 6-7, 9-10): a member crossing cell (k, l) from its left face to its
// right face has L = (s_k+1 - s_k)/sin(theta) (Eq. 8), one from its bottom plane to its top
// plane L = (P_l+1 - P_l)/|cos(theta)| (Eq. 11, reading Q3) — the same for every such
// member, so their exponentials are evaluated once per cell; only the "corner" pieces
// (entering through one kind of face and leaving through the other) have member-dependent
// lengths, linear in i.
//
// Work decomposition (one warp = one work unit = a band of B consecutive members of one
// stack, one direction after the other):
//   * the band's boundary psi lives in shared memory (two 16-byte halves per member, SoA);
//   * the warp walks the 2D segments k (columns) in travel order; in each column lane
//     (cell c, r) owns cell (k, L_lo + c) — R lanes per cell, C = 32/R cells per warp — and
//     applies Eq. 3 to that cell's members (those with member index = r mod R) with the
//     tally of Eq. 4 accumulated in REGISTERS (no shared-memory atomics);
//   * a member's pieces inside one column are ordered by "sub-phase" q = layer - entry
//     layer: sub-phase 0 = pieces entered through the column's left face, q >= 1 = pieces
//     entered through a plane after q-1 earlier pieces in the column; sub-phases are
//     separated by __syncwarp(), so every member's pieces are applied in travel order;
//   * at the end of the column each cell's tally (summed over its R lanes) is added to the
//     FSR tally with two red.global.add.v4.f32.
// Full classes (left->right, bottom->top) use per-cell E = 2^(-sigma' L) and the
// aggregated update psi' = psi E + q (1 - E), T += (sum psi - n q)(1 - E): two FP32
// operations per member and group.  Corner pieces: E per member (FMUL + MUFU.EX2) and the
// 4-op update of the per-track kernel.
//
// Frames.  Each (unit, direction) is mapped to a canonical frame in which the members
// climb (z' increasing along s') and columns are visited in increasing s': the forward
// direction of a descending stack mirrors z (z' = Z - z), the backward direction mirrors s
// (s' = L_t - s) and, for an ascending stack, z.  Member index arithmetic (which member is
// in which cell) uses one fp64 expression U(x) = ceil((x - base_k)/dz) per boundary, the
// same on every lane, so each member is in exactly one cell per sub-phase.
//
// Segment canonicalisation (App. A.7, readings Q22/Q22b).  Rounding can only misplace a
// member whose crossing lies within ~1e-13 cm of a cell corner, and then the misplaced
// piece has (near) zero length.  Raw pieces shorter than eps_L are exactly the ones the
// walk (otf.h) merges into a neighbour, and they are dropped here: the member's FSR-id
// sequence equals the walk's merged sequence (a merge keeps the neighbour's id), lengths
// differ by < eps_L per merge.  The only candidates are the shortest member of each corner
// range; when its fp32 length is below a guard, the walk's own fp64 expression (forward
// walk, otf.h) decides.
#pragma once

namespace {

#ifndef MOC_SC_WARPS
#define MOC_SC_WARPS 4
#endif
constexpr int kScWarps = MOC_SC_WARPS;       // independent warps (units) per CTA
constexpr int kScThreads = 32 * kScWarps;
// CTAs per SM: the kernel is instantiated for 3, 4 and 5 (register caps 168 / 128 / 102;
// the shared-memory psi band capacity shrinks as CTAs are added) and each stack is swept
// by the instance with the most CTAs that does not cut it into more bands (solver.cu)
constexpr int kScMinBlocksList[3] = {3, 4, 5};
constexpr float kScSliverGuard = 4e-5f;      // fp32 corner length below which fp64 decides

// debug statistics build (-DMOC_SC_STATS): per-sweep counts of the work decomposition
#ifdef MOC_SC_STATS
__device__ unsigned long long g_sc_stats[16];
#define SC_STAT(i, v) atomicAdd(&g_sc_stats[i], (unsigned long long)(v))
#else
#define SC_STAT(i, v) ((void)0)
#endif

// doubles per canonical plane copy in dynamic shared memory (NL + 1 planes, even count so
// the psi bands that follow stay 16-byte aligned)
__host__ __device__ constexpr int sc_plane_stride(int NL) { return (NL + 2) & ~1; }

// 5 CTAs per SM (stacks whose bands are not limited by shared memory): static plane copies
// and a shared staging area through which cell l + 1's source and material (sigma_t from
// the per-CTA table) reach the corner pieces of cell l (4 KB per CTA for G < 8; fewer
// registers and instructions, the 102-register cap spills otherwise).  3 and 4 CTAs per SM: the planes sized for NL in dynamic shared memory
// and shuffles instead of the staging, every KB to the psi bands
__host__ __device__ constexpr bool sc_stage_smem(int minb) { return minb >= 5; }
// staging per warp: [2][32 lanes] float4 (q[0..6] + the material index) for G < 8, else
// [4][32 lanes] (q[0..7], sigma_t log2(e)[0..7])
template <int G>
constexpr size_t sc_stage_bytes() { return (size_t)kScWarps * 32 * (G < 8 ? 32 : 64); }

// bounds-checked debug build (-DMOC_SC_CHECK, tests run against it with MOC3D_LIB): every
// shared-memory psi / hash index, plane index, FSR index and link target of the sweep is
// checked and an out-of-range one traps (the kernel fails, the run reports a CUDA error)
#ifdef MOC_SC_CHECK
#define SC_CHECK(c) \
  do {              \
    if (!(c)) __trap(); \
  } while (0)
#else
#define SC_CHECK(c) ((void)0)
#endif

struct ScUnit {
  uint32_t stack, i0, n;  // members i0 .. i0+n-1 of the stack
  uint32_t lgR;           // bits 0-7: R = 1 << lgR lanes per cell; bits 16-31: slot skew (5 CTAs)
};

struct ScArgs {
  DevData d;
  const ScUnit* units;
  uint32_t n_units;
  uint32_t* counter;
  const uint32_t* link;
  const uint8_t* mat;
  const float* qt;           // [J][GP]; for G < GP slot G carries the FSR's material index bits
  cudaTextureObject_t qtex;  // qt as a float4 texture (GP == 8)
  const float* psi_in;
  float* psi_out;
  float* tally;              // fp32 [J][GP]
  double* sc;
  int pcap;                  // psi capacity per warp (members)
  double inv_hmin;           // 1 / thinnest axial layer (rounded up)
  double h_fast;             // columns with rho < h_fast take the one-crossing fast path
  int* err;
  unsigned long long* hash;  // HASH: per slot FNV-1a of the emitted FSR ids, in travel order
  int32_t* nseg;             // HASH: per slot emitted segment count
  int gs;                    // Gauss-Seidel (NEXT-4): psi_in == psi_out, slot pad word = write epoch
  const uint32_t* slot_first;  // per stack: first boundary-psi / link slot pair of its members on this rank
  uint64_t n_slots;            // boundary-psi slots per buffer (bounds checks)
  uint64_t n_fsr;              // FSRs (bounds checks)
};

template <int G>
struct ScH {
  static constexpr int NH = (G + 3) / 4;  // 16-byte halves of a member's psi
};

// forward-walk length of the raw piece (member z0, physical column k, physical layer lp):
// the exact fp64 expressions of otf.h / the per-track walk (entry = max of the candidate
// crossings, exit = min), so the sliver decision is the walk's own
__device__ __forceinline__ double sc_walk_len(const DevData& d, const double* P, int64_t sb, int k, int lp,
                                              double z0, double tn, double isn, double Lt, bool up) {
  double s_in, s_out;
  if (up) {
    s_in = (0.0 - z0) * tn;
    s_out = (d.Z - z0) * tn;
  } else {
    s_in = (d.Z - z0) * tn;
    s_out = (0.0 - z0) * tn;
  }
  s_in = s_in > 0.0 ? s_in : 0.0;
  s_out = s_out < Lt ? s_out : Lt;
  if (s_out < s_in) s_out = s_in;
  const double sa = k ? d.seg_send[sb + k - 1] : 0.0;
  const double sbd = d.seg_send[sb + k];
  const double pe = up ? P[lp] : P[lp + 1];
  const double px = up ? P[lp + 1] : P[lp];
  const double se = (pe - z0) * tn, sx = (px - z0) * tn;
  double lo = sa > se ? sa : se;
  lo = lo > s_in ? lo : s_in;
  double hi = sbd < sx ? sbd : sx;
  hi = hi < s_out ? hi : s_out;
  return (hi - lo) * isn;
}

__device__ __forceinline__ uint64_t sc_fnv(uint64_t h, uint32_t u) {
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    h ^= (uint64_t)((u >> (8 * b)) & 0xffu);
    h *= 1099511628211ull;
  }
  return h;
}

template <int G, int GP, bool HASH, bool SK = false>
struct ScCell {
  static constexpr int NH = ScH<G>::NH;
  float4* psl;  // psi halves [NH][pcap]
  int pcap;
  int nb;       // members in the band (bounds checks)
  float q[8], sg[8], T[8];
  uint32_t j;
  uint64_t* hh;  // HASH state per member
  int* hc;
  uint32_t nem;
  uint32_t skew = 0;  // SK: shared-memory slot of member m = m + (m skew) >> 16 (sc_configure)
  __device__ __forceinline__ int slot(int m) const {
    if constexpr (SK) return m + (int)(((uint32_t)m * skew) >> 16);
    else return m;
  }

  __device__ __forceinline__ void load(int m, float* v) const {
    SC_CHECK(m >= 0 && m < nb && slot(nb - 1) < pcap);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const float4 x = psl[h * pcap + slot(m)];
      v[4 * h] = x.x;
      v[4 * h + 1] = x.y;
      v[4 * h + 2] = x.z;
      v[4 * h + 3] = x.w;
    }
  }
  __device__ __forceinline__ void store(int m, const float* v) {
    SC_CHECK(m >= 0 && m < nb && slot(nb - 1) < pcap);
#pragma unroll
    for (int h = 0; h < NH; ++h) psl[h * pcap + slot(m)] = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
  }
  __device__ __forceinline__ void emit_hash(int m) {
    if constexpr (HASH) {
      SC_CHECK(m >= 0 && m < nb);
      hh[m] = sc_fnv(hh[m], j);
      hc[m] += 1;
    }
  }

  // members m = a1, a1 + R, ... < b (all = r mod R) in a bank-rotated order (the lanes of
  // a quarter-warp start on distinct 16-byte bank groups: member m -> group m mod 8), one
  // member per trip: a single inlined copy of the member body, because the sweep's hot
  // code must stay inside the 32 KB instruction cache (ncu: three copies per class put
  // 99 % of the executed instructions in 30 KB and cost 6 % over this form; 46 KB cost
  // 35 %); returns the count
  template <int STAT_TRIP, int STAT_CALL, class F1>
  __device__ __forceinline__ int visit(int a, int b, int r, int lgR, int c, F1&& f1) {
    const int R = 1 << lgR;
    const int a1 = a + ((r - a) & (R - 1));
    if (a1 >= b) return 0;
    const int n = ((b - 1 - a1) >> lgR) + 1;
    int idx = ((((c << lgR) + r - slot(a1)) & 7) >> lgR);
    // a range shorter than the rotation: fold the start back into it (idx mod n for n >= 4),
    // so lanes whose bank group is not in their range spread over it instead of all starting
    // on its first member (consecutive cells' ranges start on nearly the same bank group)
    if (idx >= n) idx -= n;
    if (idx >= n) idx = 0;
    // iterate the member index itself (no per-trip index -> member shift), wrapping from
    // the range end to a1, until back at the start
    const int m0 = a1 + (idx << lgR), me = a1 + (n << lgR);
    int m = m0;
#pragma unroll 1
    do {
      f1(m);
      m += R;
      m = m == me ? a1 : m;
    } while (m != m0);
#ifdef MOC_SC_STATS
    {
      const unsigned am = __activemask();
      const int mx = __reduce_max_sync(am, (unsigned)n);
      if ((threadIdx.x & 31) == __ffs(am) - 1) SC_STAT(STAT_TRIP, mx), SC_STAT(STAT_CALL, 1);
    }
#endif
    return n;
  }


  // shared-E class (Eq. 8 / Eq. 11 pieces of one cell, all of length L):
  // psi' = psi E + q (1 - E); T += (sum psi - n q)(1 - E)
  __device__ __forceinline__ void full(int a, int b, int r, int lgR, int c, float L) {
    if (a >= b) return;
    float E[8], F[8], qc[8], S[8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      E[g] = ex2_approx(-sg[g] * L);  // 2^(-sigma_t log2(e) L)
      F[g] = 1.f - E[g];
      qc[g] = q[g] * F[g];
      S[g] = 0.f;
    }
    // packed FP32 over group pairs (FFMA2 / FADD2, each lane rounded as FFMA / FADD: the
    // same results as the one-group form), an odd G's last group scalar: 20 instructions
    // per member instead of 27
    static_assert(NH == 2 || G <= 4, "psi halves layout");
    constexpr int NPF = G / 2;  // full pairs; an odd G's last group is scalar
    float2 E2[4], Q2[4], S2[4];
#pragma unroll
    for (int p = 0; p < NPF; ++p) {
      E2[p] = make_float2(E[2 * p], E[2 * p + 1]);
      Q2[p] = make_float2(qc[2 * p], qc[2 * p + 1]);
      S2[p] = make_float2(0.f, 0.f);
    }
    float Sl = 0.f;
    const int n = visit<6, 8>(
        a, b, r, lgR, c,
        [&](int m) {
          SC_CHECK(m >= 0 && m < nb && slot(nb - 1) < pcap);
          float2* const p2 = reinterpret_cast<float2*>(psl);
          float2 x[4];
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const float4 t = psl[h * pcap + slot(m)];
            x[2 * h] = make_float2(t.x, t.y);
            x[2 * h + 1] = make_float2(t.z, t.w);
          }
#pragma unroll
          for (int p = 0; p < NPF; ++p) {
            S2[p] = __fadd2_rn(S2[p], x[p]);
            x[p] = __ffma2_rn(x[p], E2[p], Q2[p]);
          }
          if constexpr (G & 1) {
            float& xl = (G - 1) & 1 ? x[(G - 1) / 2].y : x[(G - 1) / 2].x;
            Sl += xl;
            xl = fmaf(xl, E[G - 1], qc[G - 1]);
          }
#pragma unroll
          for (int p = 0; p < 2 * NH; ++p)
            if (2 * p < G) p2[2 * ((p >> 1) * pcap + slot(m)) + (p & 1)] = x[p];
          emit_hash(m);
        });
#pragma unroll
    for (int p = 0; p < NPF; ++p) S[2 * p] = S2[p].x, S[2 * p + 1] = S2[p].y;
    if constexpr (G & 1) S[G - 1] = Sl;
    const float fn = (float)n;
#pragma unroll
    for (int g = 0; g < G; ++g) T[g] = fmaf(fmaf(-fn, q[g], S[g]), F[g], T[g]);
    nem += n;
    SC_STAT(3, n);
  }

  // members full in this cell in two consecutive columns (same layer, same lanes): both
  // updates in one visit, Eq. 3 with this column's (E, q (1 - E)) then the next column's
  // (E', q' (1 - E')); this column's tally as full(), the next column's partial sum Sn and
  // count nn carried to it (addff).  Hash: this cell's id j, then the next cell's j2.
  __device__ __forceinline__ void fullff(int a, int b, int r, int lgR, int c, float L, const float* q2,
                                         const float* sg2, float L2, uint32_t j2, float* Sn, int& nn) {
    nn = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) Sn[g] = 0.f;
    if (a >= b) return;
    constexpr int NPF = G / 2;
    float E[8], F[8], qc[8], Eb[8], qcb[8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      E[g] = ex2_approx(-sg[g] * L);
      F[g] = 1.f - E[g];
      qc[g] = q[g] * F[g];
      Eb[g] = ex2_approx(-sg2[g] * L2);
      qcb[g] = q2[g] * (1.f - Eb[g]);
    }
    float2 E2[4], Q2[4], S2[4], Eb2[4], Qb2[4], Sb2[4];
#pragma unroll
    for (int p = 0; p < NPF; ++p) {
      E2[p] = make_float2(E[2 * p], E[2 * p + 1]);
      Q2[p] = make_float2(qc[2 * p], qc[2 * p + 1]);
      Eb2[p] = make_float2(Eb[2 * p], Eb[2 * p + 1]);
      Qb2[p] = make_float2(qcb[2 * p], qcb[2 * p + 1]);
      S2[p] = Sb2[p] = make_float2(0.f, 0.f);
    }
    float Sl = 0.f, Sbl = 0.f;
    const int n = visit<6, 8>(
        a, b, r, lgR, c,
        [&](int m) {
          SC_CHECK(m >= 0 && m < nb && slot(nb - 1) < pcap);
          float2* const p2 = reinterpret_cast<float2*>(psl);
          float2 x[4];
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const float4 t = psl[h * pcap + slot(m)];
            x[2 * h] = make_float2(t.x, t.y);
            x[2 * h + 1] = make_float2(t.z, t.w);
          }
#pragma unroll
          for (int p = 0; p < NPF; ++p) {
            S2[p] = __fadd2_rn(S2[p], x[p]);
            x[p] = __ffma2_rn(x[p], E2[p], Q2[p]);
            Sb2[p] = __fadd2_rn(Sb2[p], x[p]);
            x[p] = __ffma2_rn(x[p], Eb2[p], Qb2[p]);
          }
          if constexpr (G & 1) {
            float& xl = (G - 1) & 1 ? x[(G - 1) / 2].y : x[(G - 1) / 2].x;
            Sl += xl;
            xl = fmaf(xl, E[G - 1], qc[G - 1]);
            Sbl += xl;
            xl = fmaf(xl, Eb[G - 1], qcb[G - 1]);
          }
#pragma unroll
          for (int p = 0; p < 2 * NH; ++p)
            if (2 * p < G) p2[2 * ((p >> 1) * pcap + slot(m)) + (p & 1)] = x[p];
          if constexpr (HASH) {
            emit_hash(m);
            hh[m] = sc_fnv(hh[m], j2);
            hc[m] += 1;
          }
        });
    float S[8];
#pragma unroll
    for (int p = 0; p < NPF; ++p) {
      S[2 * p] = S2[p].x, S[2 * p + 1] = S2[p].y;
      Sn[2 * p] = Sb2[p].x, Sn[2 * p + 1] = Sb2[p].y;
    }
    if constexpr (G & 1) S[G - 1] = Sl, Sn[G - 1] = Sbl;
    const float fn = (float)n;
#pragma unroll
    for (int g = 0; g < G; ++g) T[g] = fmaf(fmaf(-fn, q[g], S[g]), F[g], T[g]);
    nn = n;
    nem += 2 * n;
    SC_STAT(3, 2 * n);
  }
  // the carried part of this cell's tally: (1 - E)(Sn - nn q) of the members fullff swept
  __device__ __forceinline__ void addff(const float* Sn, int nn, float L) {
    if (nn == 0) return;
    const float fn = (float)nn;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float F = 1.f - ex2_approx(-sg[g] * L);
      T[g] = fmaf(fmaf(-fn, q[g], Sn[g]), F, T[g]);
    }
  }

  // corner class: length d(m) * ti with d = d0 + |m - anchor| dz (anchor = shortest member);
  // per member Eq. 3: dpsi = (psi - q)(1 - E), psi -= dpsi, T += dpsi
  __device__ __forceinline__ void corner(int a, int b, int r, int lgR, int c, int anchor, float d0, float dzf,
                                         float ti) {
    if (a >= b) return;
    const int n = visit<7, 9>(
        a, b, r, lgR, c,
        [&](int m) {
          const float L = fmaf((float)abs(m - anchor), dzf, d0) * ti;
          float v[4 * NH];
          load(m, v);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float E = ex2_approx(-sg[g] * L);
            const float dd = v[g] - q[g];
            const float dl = fmaf(-dd, E, dd);
            v[g] -= dl;
            T[g] += dl;
          }
          store(m, v);
          emit_hash(m);
        });
    nem += n;
    SC_STAT(4, n);
  }

  // fast-path corner class (rho < h_min): members entering cell l through its left face
  // and leaving through its top plane P_u into cell l + 1, whose right face they reach
  // before the next plane.  Piece 1 (cell l): d1(m) = P_u - z_m = d1a + (b - 1 - m) dz;
  // piece 2 (cell l + 1, only if l + 1 is inside the domain): d2(m) = z_m + rho - P_u =
  // d2a + (m - a) dz; 3D length = d * ti.  A sliver piece (the walk merges it, App. A.7)
  // gets length 0 (E = 1: no change) and is not emitted.  fetch2 gives cell l + 1's source
  // and sigma_t log2(e) (q2, sg2); T2 = its tally share.
  template <class Fetch2>
  __device__ __forceinline__ void corner2(int a, int b, int r, int lgR, int c, float d1a, float d2a, float dzf,
                                          float ti, bool nxt, int skip1, int skip2, Fetch2&& fetch2,
                                          uint32_t j2, float* T2) {
    if (a >= b) return;
    float q2[8], sg2[8];
    fetch2(q2, sg2);
    const float t2 = nxt ? ti : 0.f;  // no second piece above the domain top
    auto one = [&](int m, float* v) {
      const float L1 = m == skip1 ? 0.f : fmaf((float)(b - 1 - m), dzf, d1a) * ti;
      const float L2 = m == skip2 ? 0.f : fmaf((float)(m - a), dzf, d2a) * t2;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float E1 = ex2_approx(-sg[g] * L1);
        const float e1 = v[g] - q[g];
        const float l1 = fmaf(-e1, E1, e1);
        v[g] -= l1;
        T[g] += l1;
        const float E2 = ex2_approx(-sg2[g] * L2);
        const float e2 = v[g] - q2[g];
        const float l2 = fmaf(-e2, E2, e2);
        v[g] -= l2;
        T2[g] += l2;
      }
    };
    auto emit = [&](int m) {
      if constexpr (HASH) {
        if (m != skip1) emit_hash(m);
        if (nxt && m != skip2) {
          hh[m] = sc_fnv(hh[m], j2);
          hc[m] += 1;
        }
      }
    };
    const int n = visit<7, 9>(
        a, b, r, lgR, c,
        [&](int m) {
          float v[4 * NH];
          load(m, v);
          one(m, v);
          store(m, v);
          emit(m);
        });
    // emitted pieces: n first + (n second, if inside the domain), minus this lane's slivers
    nem += nxt ? 2 * n : n;
    if (skip1 >= 0 && (skip1 & ((1 << lgR) - 1)) == r) --nem;
    if (nxt && skip2 >= 0 && (skip2 & ((1 << lgR) - 1)) == r) --nem;
    SC_STAT(4, 2 * n);
  }
};

template <int G, int GP, bool HASH, int MINB>
__global__ void __launch_bounds__(kScThreads, MINB) k_sweep_sc(ScArgs a) {
  // shared memory: the canonical planes (as given, and mirrored z' = Z - z), the warps' psi
  // bands, then the cell staging (sc_stage_smem) or, HASH, the per-member hash state
  extern __shared__ __align__(16) float4 dsm_sc[];
  __shared__ __align__(16) float4 shS4[kMaxMat * 2];  // sigma_t log2(e) per material, 8 groups
  constexpr int NH = ScH<G>::NH;
  const DevData& d = a.d;
  const int NL = d.NL;
  double* shP0;
  double* shP1;
  float4* band4;
  if constexpr (sc_stage_smem(MINB)) {  // static plane copies (fixed addresses, fewer registers)
    __shared__ double shPs[2][kMaxPlanes + 1];
    shP0 = shPs[0];
    shP1 = shPs[1];
    band4 = dsm_sc;
  } else {  // plane copies at the head of the dynamic shared memory, sized for NL
    shP0 = reinterpret_cast<double*>(dsm_sc);
    shP1 = shP0 + sc_plane_stride(NL);
    band4 = dsm_sc + sc_plane_stride(NL);  // 2 x stride doubles = stride float4
  }
  for (int q = threadIdx.x; q <= NL; q += blockDim.x) {
    shP0[q] = d.planes[q];
    shP1[q] = d.Z - d.planes[NL - q];
  }
  for (int q = threadIdx.x; q < kMaxMat * 8; q += blockDim.x) {
    const int m = q >> 3, g = q & 7;
    reinterpret_cast<float*>(shS4)[q] = g < G ? c_sigt2[m * kMaxG + g] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pcap = a.pcap;
  float4* const psl = band4 + (size_t)warp * NH * pcap;
  // per-warp cell staging (sc_stage_bytes) after the bands, only where shared memory is not
  // the band limit (sc_stage_smem)
  float4* const stg = band4 + (size_t)kScWarps * NH * pcap + (size_t)warp * 32 * (G < 8 ? 2 : 4);
  float4* const hbase = band4 + (size_t)kScWarps * NH * pcap;
  uint64_t* const hh = HASH ? reinterpret_cast<uint64_t*>(hbase) + (size_t)warp * pcap : nullptr;
  int* const hc =
      HASH ? reinterpret_cast<int*>(reinterpret_cast<uint64_t*>(hbase) + (size_t)kScWarps * pcap) + (size_t)warp * pcap
           : nullptr;
  const float ps = (float)a.sc[SC_PSI_SCALE];
  const uint32_t ep = (uint32_t)a.sc[SC_ITER] + 1u;  // this sweep's epoch (Gauss-Seidel slots)
  double leak = 0.0;
  uint64_t nemit = 0;

  while (true) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(a.counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= a.n_units) break;
    const ScUnit U = a.units[u];
    const int s = (int)U.stack;
    const int t = s / d.N, n = s - t * d.N;
    const int an = d.t_a[t] * d.N + n;
    const int64_t sb = d.t_seg[t];
    const int nk = (int)(d.t_seg[t + 1] - sb);
    const double dz = d.an_dz[an], cot = d.an_cot[an], tn = d.an_tan[an], isn = d.an_invsin[an];
    const double Lt = d.t_len[t], z0b = d.st_z0[s];
    const double c = fabs(cot), invD = 1.0 / dz;
    const float ti = (float)(isn * fabs(tn));  // 3D length per unit of z: 1/|cos(theta)|
    const float dzf = (float)dz;
    const int B = (int)U.n, lgRu = (int)(U.lgR & 0xffu);
    const uint32_t skw = U.lgR >> 16;  // the band's shared-memory slot skew (5 CTAs per SM)
    auto slot_of = [&](int m) {
      if constexpr (MINB == 5 && !HASH) return m + (int)(((uint32_t)m * skw) >> 16);
      else return m;
    };
    // largest R for a column: keep >= 3 members of a full cell per lane (hmin / dz members
    // per cell), below which the per-lane cell setup outweighs the split member work
    int lgRcap = lgRu;
    while (lgRcap < 3 && a.inv_hmin * (double)(6 << lgRcap) * dz <= 1.0) ++lgRcap;
    const bool up = cot > 0;
    const uint32_t id0 = a.slot_first[s] + U.i0;  // this rank's track numbering (psi, links)
    const float cw = d.an_c[an];

    for (int dir = 0; dir < 2; ++dir) {
      const bool ms = dir == 1;
      const bool mz = up == (dir == 1);
      const double* P = mz ? shP1 : shP0;
      // canonical member m <-> physical member i0 + (mz ? B-1-m : m)
      for (int m = lane; m < B; m += 32) {
        const uint32_t id = id0 + (uint32_t)(mz ? B - 1 - m : m);
        float v[8];
        load_q<GP>(a.psi_in, (int64_t)(2 * id + dir), v);
        // lazy normalisation: psi written in an earlier iteration is scaled on read; in
        // Gauss-Seidel mode a slot already rewritten in this sweep (pad word = this epoch)
        // is in the current units
        float sc_ = ps;
        if constexpr (GP == 8 && G < 8) {
          if (a.gs && __float_as_uint(v[7]) == ep) sc_ = 1.f;
        }
#pragma unroll
        for (int h = 0; h < NH; ++h)
          psl[h * pcap + slot_of(m)] = make_float4(v[4 * h] * sc_, 4 * h + 1 < G ? v[4 * h + 1] * sc_ : 0.f,
                                          4 * h + 2 < G ? v[4 * h + 2] * sc_ : 0.f, 4 * h + 3 < G ? v[4 * h + 3] * sc_ : 0.f);
        if constexpr (HASH) {
          hh[m] = kFnvInit;
          hc[m] = 0;
        }
      }
      // canonical height of member 0 at s' = 0
      const double zc0 = (mz ? d.Z - z0b - (double)(U.i0 + (uint32_t)B - 1) * dz : z0b + (double)U.i0 * dz) -
                         (ms ? Lt * c : 0.0);
      // band layer window [L_lo, L_hi]: both ends only rise along the canonical walk
      // (base and top = base of the next column + (B - 1) dz are non-decreasing)
      int L_lo = 0, L_hi = 0;
      // P[L_lo + 1] and P[L_hi + 1] kept in registers (+inf above the top layer): the
      // window ends move in few columns, so the common case needs no shared-memory load
      const double kInf = __longlong_as_double(0x7ff0000000000000ll);
      double PnLo = NL > 1 ? P[1] : kInf, PnHi = PnLo;
      if (lane == 0) SC_STAT(0, 1);
      __syncwarp();
      ScCell<G, GP, HASH, MINB == 5 && !HASH> cell;
      cell.skew = skw;
      cell.psl = psl;
      cell.pcap = pcap;
      cell.nb = B;
      cell.hh = hh;
      cell.hc = hc;
      cell.nem = 0;
      // column data prefetched 32 columns at a time (lane i holds column kk0 + i: its 2D
      // segment's two ends and region, one coalesced load each) and broadcast by shuffles
      double pf_sa = 0.0, pf_sb = 0.0;
      uint32_t pf_rg = 0;
      // two-column visits (fullff): this column's fused members were swept in the previous
      // one (fzr); their member range [fzA, fzB) and carried tally part (fzS, fzN)
      bool fzr = false;
      int fzA = 0, fzB = 0, fzN = 0;
      float fzS[8];
#pragma unroll 1
      for (int kk = 0; kk < nk; ++kk) {
        const int k = ms ? nk - 1 - kk : kk;
        if ((kk & 31) == 0) {
          const int kq = kk + lane;
          if (kq < nk) {
            const int kx = ms ? nk - 1 - kq : kq;
            pf_sa = kx ? d.seg_send[sb + kx - 1] : 0.0;
            pf_sb = d.seg_send[sb + kx];
            pf_rg = d.seg_region[sb + kx];
          }
        }
        const double s_a = __shfl_sync(0xffffffffu, pf_sa, kk & 31);
        const double s_b = __shfl_sync(0xffffffffu, pf_sb, kk & 31);
        const uint32_t region = __shfl_sync(0xffffffffu, pf_rg, kk & 31);
        const double S = kk == 0 ? 0.0 : (ms ? Lt - s_b : s_a);
        const double w = s_b - s_a;
        const double base = zc0 + S * c, rho = w * c;
        if (base >= d.Z) break;  // every member of the band has left through the top
        const double top = base + (double)(B - 1) * dz + rho;
        if (top <= 0.0) continue;  // no member has entered yet
        while (PnLo <= base) {
          ++L_lo;
          PnLo = L_lo < NL - 1 ? P[L_lo + 1] : kInf;
        }
        if (L_hi < L_lo) {
          L_hi = L_lo;
          PnHi = PnLo;
        }
        while (PnHi < top) {
          ++L_hi;
          PnHi = L_hi < NL - 1 ? P[L_hi + 1] : kInf;
        }
        // lanes per cell for this column: the unit's R, raised while the column's cells
        // still fit (a band entering or leaving the domain touches few layers: its members
        // are then split over R = 2, 4, 8 lanes per cell instead of idling lanes)
        int lgR = lgRu;
        while (lgR < lgRcap && (32 >> (lgR + 1)) >= L_hi - L_lo + 1) ++lgR;
        const int R = 1 << lgR, C = 32 >> lgR;
        const int ci = lane >> lgR, r = lane & (R - 1);
        int Lh = L_hi;
        if (Lh - L_lo + 1 > C) {
          if (lane == 0) atomicAdd(a.err, 1);
          Lh = L_lo + C - 1;
        }
        const int l = L_lo + ci;
        const bool act = l <= Lh;
        if (lane == 0) SC_STAT(1, 1), SC_STAT(2, Lh - L_lo + 1);
        auto Uf = [&](double x) {
          const int v = __double2int_ru((x - base) * invD);
          return min(max(v, 0), B);
        };
        const float Lf = (float)(w * isn);
#pragma unroll
        for (int g = 0; g < 8; ++g) cell.T[g] = 0.f;
        float T2[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) T2[g] = 0.f;
        double Pl = 0, Pu = 0;
        int uPl = 0, uPu = 0, uPlR = 0, uPuR = 0, lp = 0;
        int mi = 0;  // the cell's material
        if (act) {
          lp = mz ? NL - 1 - l : l;
          cell.j = region * (uint32_t)NL + (uint32_t)lp;
          SC_CHECK(l >= 0 && l < NL && lp >= 0 && lp < NL && (uint64_t)cell.j < a.n_fsr);
          float qv[8];
          if constexpr (GP == 8) {
            const float4 x0 = tex1Dfetch<float4>(a.qtex, (int)(2 * cell.j)), x1 = tex1Dfetch<float4>(a.qtex, (int)(2 * cell.j + 1));
            qv[0] = x0.x; qv[1] = x0.y; qv[2] = x0.z; qv[3] = x0.w;
            qv[4] = x1.x; qv[5] = x1.y; qv[6] = x1.z; qv[7] = x1.w;
          } else {
            load_q<GP>(a.qt, (int64_t)cell.j, qv);
          }
          if constexpr (G < GP) mi = __float_as_int(qv[G]);
          else mi = a.mat[cell.j];
          const float4 s0 = shS4[2 * mi], s1 = shS4[2 * mi + 1];
          cell.sg[0] = s0.x; cell.sg[1] = s0.y; cell.sg[2] = s0.z; cell.sg[3] = s0.w;
          cell.sg[4] = s1.x; cell.sg[5] = s1.y; cell.sg[6] = s1.z; cell.sg[7] = s1.w;
#pragma unroll
          for (int g = 0; g < 8; ++g) cell.q[g] = g < G ? qv[g] : 0.f;
          Pl = P[l];
          Pu = P[l + 1];
          uPlR = Uf(Pl - rho);
          uPuR = Uf(Pu - rho);
          uPl = Uf(Pl);
          uPu = Uf(Pu);
        }
        const bool fast = rho < a.h_fast;  // every member crosses at most one plane here
        // fuse with the next column when it is in this prefetch block, also takes the fast
        // path and keeps the band window (so the same lane owns each layer in both): the
        // same expressions the next column evaluates, so both agree bit for bit.  Only at 3
        // CTAs per SM: there it cuts the shared-memory wavefronts by 22 % (ncu) and the time
        // by 2.6 %; at 4 CTAs it measured slower, at 5 the registers would spill
        bool fzs = false;
        double base2 = 0.0, rho2 = 0.0;
        float Lf2 = 0.f;
        uint32_t region2 = 0;
        if constexpr (MINB == 3) {
          const int kn = (kk + 1) & 31;
          const double sa2 = __shfl_sync(0xffffffffu, pf_sa, kn), sb2 = __shfl_sync(0xffffffffu, pf_sb, kn);
          region2 = __shfl_sync(0xffffffffu, pf_rg, kn);
          if (fast && !fzr && kk + 1 < nk && kn != 0) {
            const double S2 = ms ? Lt - sb2 : sa2;
            const double w2 = sb2 - sa2;
            base2 = zc0 + S2 * c;
            rho2 = w2 * c;
            const double top2 = base2 + (double)(B - 1) * dz + rho2;
            fzs = rho2 < a.h_fast && base2 < d.Z && top2 > 0.0 && PnLo > base2 && PnHi >= top2;
            Lf2 = (float)(w2 * isn);
          }
        }
        if (fast) {
          if (!act) {  // finite values for lanes without a cell, shuffled to corner pieces (read only with zero lengths)
#pragma unroll
            for (int g = 0; g < 8; ++g) cell.q[g] = cell.sg[g] = 0.f;
          }
          // cell l + 1's source and sigma_t for the corner pieces entering it: through the
          // warp's staging area, or by shuffles from its lanes (lane + R) after the full class
          float q2s[8], sg2s[8];
          // the full class (Eq. 8), with the two-column visits of a fused column pair
          auto full_class = [&]() {
            const int e1 = min(uPu, uPuR);
            if (fzr) {  // the fused members [fzA, fzB) were swept with the previous column
              cell.full(uPl, min(fzA, e1), r, lgR, ci, Lf);
              cell.full(max(fzB, uPl), e1, r, lgR, ci, Lf);
              cell.addff(fzS, fzN, Lf);
            } else if (fzs) {
              // the next column's cell in this layer: source, material, Sigma_t
              const uint32_t j2 = region2 * (uint32_t)NL + (uint32_t)lp;
              SC_CHECK((uint64_t)j2 < a.n_fsr);
              float q2f[8], sg2f[8];
              {
                float qv[8];
                int mi2;
                if constexpr (GP == 8) {
                  const float4 x0 = tex1Dfetch<float4>(a.qtex, (int)(2 * j2)), x1 = tex1Dfetch<float4>(a.qtex, (int)(2 * j2 + 1));
                  qv[0] = x0.x; qv[1] = x0.y; qv[2] = x0.z; qv[3] = x0.w;
                  qv[4] = x1.x; qv[5] = x1.y; qv[6] = x1.z; qv[7] = x1.w;
                } else {
                  load_q<GP>(a.qt, (int64_t)j2, qv);
                }
                if constexpr (G < GP) mi2 = __float_as_int(qv[G]);
                else mi2 = a.mat[j2];
                const float4 s0 = shS4[2 * mi2], s1 = shS4[2 * mi2 + 1];
                sg2f[0] = s0.x; sg2f[1] = s0.y; sg2f[2] = s0.z; sg2f[3] = s0.w;
                sg2f[4] = s1.x; sg2f[5] = s1.y; sg2f[6] = s1.z; sg2f[7] = s1.w;
#pragma unroll
                for (int g = 0; g < 8; ++g) q2f[g] = g < G ? qv[g] : 0.f;
              }
              const int uPuR2 = min(max(__double2int_ru((Pu - rho2 - base2) * invD), 0), B);
              const int ffb = max(min(e1, uPuR2), uPl);
              cell.fullff(uPl, ffb, r, lgR, ci, Lf, q2f, sg2f, Lf2, j2, fzS, fzN);
              cell.full(ffb, e1, r, lgR, ci, Lf);
              fzA = uPl;
              fzB = ffb;
            } else {
              cell.full(uPl, e1, r, lgR, ci, Lf);
            }
          };
          if constexpr (sc_stage_smem(MINB)) {
            stg[lane] = make_float4(cell.q[0], cell.q[1], cell.q[2], cell.q[3]);
            if constexpr (G < 8) {  // the material index in the free eighth word: Sigma_t from shS4
              stg[32 + lane] = make_float4(cell.q[4], cell.q[5], cell.q[6], __int_as_float(act ? mi : 0));
            } else {
              stg[32 + lane] = make_float4(cell.q[4], cell.q[5], cell.q[6], cell.q[7]);
              stg[64 + lane] = make_float4(cell.sg[0], cell.sg[1], cell.sg[2], cell.sg[3]);
              stg[96 + lane] = make_float4(cell.sg[4], cell.sg[5], cell.sg[6], cell.sg[7]);
            }
            __syncwarp();
          } else {
            // members entering through the left face in layer l: full (Eq. 8)
            if (act) full_class();
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              q2s[g] = g < G ? __shfl_sync(0xffffffffu, cell.q[g], (lane + R) & 31) : 0.f;
              sg2s[g] = g < G ? __shfl_sync(0xffffffffu, cell.sg[g], (lane + R) & 31) : 0.f;
            }
          }
          auto fetch2 = [&](float* q2, float* sg2) {
            if constexpr (sc_stage_smem(MINB)) {
              const float4* st2 = stg + ((lane + R) & 31);
              const float4 x0 = st2[0], x1 = st2[32];
              float4 y0, y1;
              if constexpr (G < 8) {
                const int mi2 = __float_as_int(x1.w);
                y0 = shS4[2 * mi2];
                y1 = shS4[2 * mi2 + 1];
              } else {
                y0 = st2[64];
                y1 = st2[96];
              }
              q2[0] = x0.x; q2[1] = x0.y; q2[2] = x0.z; q2[3] = x0.w;
              q2[4] = x1.x; q2[5] = x1.y; q2[6] = x1.z; q2[7] = G < 8 ? 0.f : x1.w;
              sg2[0] = y0.x; sg2[1] = y0.y; sg2[2] = y0.z; sg2[3] = y0.w;
              sg2[4] = y1.x; sg2[5] = y1.y; sg2[6] = y1.z; sg2[7] = y1.w;
            } else {
#pragma unroll
              for (int g = 0; g < 8; ++g) q2[g] = q2s[g], sg2[g] = sg2s[g];
            }
          };
          if (act) {
            // members entering through the left face in layer l: full (Eq. 8) ...
            if constexpr (sc_stage_smem(MINB)) full_class();
            // ... and corners, left -> top in l, bottom -> right in l + 1
            const int a0 = max(uPl, uPuR), b0 = uPu;
            if (a0 < b0) {
              const bool nxt = l + 1 < NL;
              const int lp2 = mz ? lp - 1 : lp + 1;
              SC_CHECK(!nxt || (lp2 >= 0 && lp2 < NL && l + 1 <= Lh));
              const double d1 = Pu - (base + (double)(b0 - 1) * dz);  // shortest piece 1: member b0 - 1
              const double d2 = base + (double)a0 * dz + rho - Pu;    // shortest piece 2: member a0
              int skip1 = -1, skip2 = -1;
              if ((float)d1 * ti < kScSliverGuard) {
                const int mphys = mz ? B - 1 - (b0 - 1) : b0 - 1;
                const double z0 = z0b + (double)(U.i0 + (uint32_t)mphys) * dz;
                if (sc_walk_len(d, shP0, sb, k, lp, z0, tn, isn, Lt, up) < kEpsL) skip1 = b0 - 1;
              }
              if (nxt && (float)d2 * ti < kScSliverGuard) {
                const int mphys = mz ? B - 1 - a0 : a0;
                const double z0 = z0b + (double)(U.i0 + (uint32_t)mphys) * dz;
                if (sc_walk_len(d, shP0, sb, k, lp2, z0, tn, isn, Lt, up) < kEpsL) skip2 = a0;
              }
              cell.corner2(a0, b0, r, lgR, ci, (float)d1, (float)d2, dzf, ti, nxt, skip1, skip2, fetch2,
                           region * (uint32_t)NL + (uint32_t)lp2, T2);
            }
            // members entering through the domain bottom (canonical z' = 0) in this column
            if (l == 0 && uPlR < uPl) {
              int a1 = uPlR;
              const double dbot = base + (double)a1 * dz + rho - Pl;
              if ((float)dbot * ti < kScSliverGuard) {
                const int mphys = mz ? B - 1 - a1 : a1;
                const double z0 = z0b + (double)(U.i0 + (uint32_t)mphys) * dz;
                if (sc_walk_len(d, shP0, sb, k, lp, z0, tn, isn, Lt, up) < kEpsL) ++a1;
              }
              if (a1 < uPl)
                cell.corner(a1, uPl, r, lgR, ci, a1, (float)(base + (double)a1 * dz + rho - Pl), dzf, ti);
            }
          }
          // cell l + 1's shares of the corner pieces -> the lanes of cell l + 1
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float x = __shfl_up_sync(0xffffffffu, T2[g], R);
            if (ci > 0) cell.T[g] += x;
          }
        } else {
          int uprev = uPl;
          if (act) {
            // sub-phase 0: members entering through the left face in layer l
            cell.full(uPl, min(uPu, uPuR), r, lgR, ci, Lf);
            int a0 = max(uPl, uPuR), b0 = uPu;
            if (a0 < b0) {
              // left -> top corners: the shortest is the highest member (anchor b0 - 1)
              const double dtop = Pu - (base + (double)(b0 - 1) * dz);
              if ((float)dtop * ti < kScSliverGuard) {
                const int mphys = mz ? B - 1 - (b0 - 1) : b0 - 1;
                const double z0 = z0b + (double)(U.i0 + (uint32_t)mphys) * dz;
                if (sc_walk_len(d, shP0, sb, k, lp, z0, tn, isn, Lt, up) < kEpsL) --b0;
              }
              cell.corner(a0, b0, r, lgR, ci, b0 - 1, (float)(Pu - (base + (double)(b0 - 1) * dz)), dzf, ti);
            }
          }
          // sub-phases q >= 1: pieces entered through the plane below layer l after q - 1
          // earlier pieces of the member in this column (at most 1 + rho / h_min of them)
          const int Q = 1 + (int)(rho * a.inv_hmin);
#pragma unroll 1
          for (int q = 1; q <= Q; ++q) {
            if (lane == 0) SC_STAT(5, 1);
            __syncwarp();
            const int e = l - q;  // entry layer (-1: through the domain bottom)
            if (act && e >= -1) {
              const int hi = uprev;  // Uf(P[e + 1])
              SC_CHECK(e <= NL);
              const int ue = e >= 0 ? Uf(P[e]) : 0;
              uprev = ue;
              const int lo = max(ue, uPlR);
              // bottom -> right corners: the shortest is the lowest member (anchor lo)
              int a1 = lo;
              const int b1 = min(hi, uPuR);
              if (a1 < b1) {
                const double dbot = base + (double)a1 * dz + rho - Pl;
                if ((float)dbot * ti < kScSliverGuard) {
                  const int mphys = mz ? B - 1 - a1 : a1;
                  const double z0 = z0b + (double)(U.i0 + (uint32_t)mphys) * dz;
                  if (sc_walk_len(d, shP0, sb, k, lp, z0, tn, isn, Lt, up) < kEpsL) ++a1;
                }
                if (a1 < b1)
                  cell.corner(a1, b1, r, lgR, ci, a1, (float)(base + (double)a1 * dz + rho - Pl), dzf, ti);
              }
              // bottom -> top (full axial, Eq. 11)
              cell.full(max(lo, uPuR), hi, r, lgR, ci, (float)(Pu - Pl) * ti);
            }
          }
        }
        // the cell's tally: sum over its R lanes, c_{a,n} * T -> FSR tally
        for (int o = 1; o < R; o <<= 1)
#pragma unroll
          for (int g = 0; g < G; ++g) cell.T[g] += __shfl_xor_sync(0xffffffffu, cell.T[g], o);
        if (act && r == 0) {
          float v[8];
          bool any = false;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            v[g] = g < G ? cell.T[g] * cw : 0.f;
            any |= v[g] != 0.f;
          }
          if (any) {
            float* dst = a.tally + (size_t)cell.j * GP;
            if constexpr (GP % 4 == 0) {
#pragma unroll
              for (int h = 0; h < GP / 4; ++h) red_add_v4(dst + 4 * h, v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
            } else {
#pragma unroll
              for (int g = 0; g < G; ++g) atomicAdd(dst + g, v[g]);
            }
          }
        }
        fzr = fzs;
        __syncwarp();
      }
      nemit += cell.nem;
      // outgoing psi of every member (each left through the top or the far end)
      for (int m = lane; m < B; m += 32) {
        const uint32_t id = id0 + (uint32_t)(mz ? B - 1 - m : m);
        float v[8];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const float4 x = psl[h * pcap + slot_of(m)];
          v[4 * h] = x.x;
          v[4 * h + 1] = x.y;
          v[4 * h + 2] = x.z;
          v[4 * h + 3] = x.w;
        }
#pragma unroll
        for (int g = G; g < 8; ++g) v[g] = 0.f;
        if constexpr (GP == 8 && G < 8) {
          if (a.gs) v[7] = __uint_as_float(ep);  // written in this sweep: current units
        }
        SC_CHECK(2 * (uint64_t)id + dir < a.n_slots);
        const uint32_t out = a.link[2 * id + dir];
        SC_CHECK(out == 0xffffffffu || out < a.n_slots);
        if (out != 0xffffffffu) {
          float* dst = a.psi_out + (size_t)out * GP;
          if constexpr (GP == 8) {
            asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(v[0]), "f"(v[1]),
                         "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                         : "memory");
          } else {
#pragma unroll
            for (int g = 0; g < G; ++g) dst[g] = v[g];
          }
        } else {
          float e = 0.f;
#pragma unroll
          for (int g = 0; g < G; ++g) e += v[g];
          leak += (double)(cw * e);
        }
        if constexpr (HASH) {
          a.hash[2 * id + dir] = hh[m];
          a.nseg[2 * id + dir] = hc[m];
        }
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    leak += __shfl_xor_sync(0xffffffffu, leak, o);
    nemit += __shfl_xor_sync(0xffffffffu, nemit, o);
  }
  if (lane == 0 && leak != 0.0) atomicAdd(&a.sc[SC_LEAK], leak);
  if (lane == 0 && nemit) atomicAdd(&a.sc[SC_NEMIT], (double)nemit);
}

__global__ void k_sc_unit_cost(const ScUnit* units, uint32_t n_units, const uint32_t* st_first, const uint32_t* cost,
                               uint32_t* key) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n_units; u += gridDim.x * blockDim.x) {
    const ScUnit U = units[u];
    const uint32_t f = st_first[U.stack] + U.i0;
    uint32_t c = 0;
    for (uint32_t i = 0; i < U.n; ++i) c += cost[f + i];
    key[u] = c;
  }
}

}  // namespace
