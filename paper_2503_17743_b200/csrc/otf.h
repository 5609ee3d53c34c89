// otf.h — on-the-fly 3D segment generation for one 3D track.
//
// A 3D track is member i of the z-stack (t, n): it projects onto 2D track t, has
// the corrected polar angle theta_{a,n}, and height z(s) = z0 + s cot(theta) along
// the 2D arc length s, with z0 = z_0(0) + i dz (Eq. 5).  Its 3D segments
// are generated from t's preloaded 2D segments (cumulative ends s_end[k], radial
// region r_k) and the global axial mesh: the next crossing is the nearer
// of the next 2D boundary and the next axial plane, and the 3D length is the 2D
// advance divided by sin(theta) (Eq. 8) — which for a piece bounded by two
// planes equals (z_max - z_min)/|cos(theta)| (Eq. 11 with |cos|, reading Q3).
// FSR j = r_k * n_layers + layer (App. A.6).
//
// Raw pieces shorter than eps_L = 1e-6 cm are merged exactly as the oracle does
// (App. A.7, readings Q22/Q22b): into the preceding piece, a leading run into the
// first long piece.  The backward walk emits the exact reverse of the forward list.
//
// Used by the host debug trace (moc_trace_track_3d), the device cost/volume/
// checksum kernels and the sweep kernels — one walk, two compilers.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define MOC_HD __host__ __device__ __forceinline__
#else
#define MOC_HD inline
#endif

namespace moc {

constexpr double kEpsL = 1e-6;  // App. A.7 epsilon_L (cm)

struct OtfView {
  const double* seg_send;      // [N2] cumulative 2D segment end s (fp64)
  const uint32_t* seg_region;  // [N2] radial region r of each 2D segment
  const double* planes;        // [NL+1] axial planes, planes[0] = 0, planes[NL] = Z
  int32_t NL;
};

struct TrackGeo {
  double z0;               // z at s = 0 of this member (Eq. 5 with s = 0)
  double cot, tan, invsin; // of the corrected polar angle
  double L;                // 2D track length
  double Z;                // domain height
  int64_t sb, se;          // 2D segment range [sb, se)
};

// Entry/exit parameters (2D arc length) of the 3D chord inside [0, Z].
MOC_HD void otf_clip(const TrackGeo& g, double& s_in, double& s_out) {
  if (g.cot > 0) {
    s_in = (0.0 - g.z0) * g.tan;
    s_out = (g.Z - g.z0) * g.tan;
  } else {
    s_in = (g.Z - g.z0) * g.tan;
    s_out = (0.0 - g.z0) * g.tan;
  }
  s_in = s_in > 0.0 ? s_in : 0.0;
  s_out = s_out < g.L ? s_out : g.L;
  if (s_out < s_in) s_out = s_in;
}

// largest l in [0, NL-1] with planes[l] <= z  (moving up from z)
MOC_HD int otf_layer_up(const OtfView& v, double z) {
  int lo = 0, hi = v.NL - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (v.planes[mid] <= z) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// smallest l in [0, NL-1] with planes[l+1] >= z  (moving down from z)
MOC_HD int otf_layer_down(const OtfView& v, double z) {
  int lo = 0, hi = v.NL - 1;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (v.planes[mid + 1] >= z) hi = mid; else lo = mid + 1;
  }
  return lo;
}
// first k in [sb, se-1] with seg_send[k] > s
MOC_HD int64_t otf_seg_after(const OtfView& v, int64_t sb, int64_t se, double s) {
  int64_t lo = sb, hi = se - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (v.seg_send[mid] > s) hi = mid; else lo = mid + 1;
  }
  return lo;
}
// first k in [sb, se-1] with seg_send[k] >= s
MOC_HD int64_t otf_seg_upto(const OtfView& v, int64_t sb, int64_t se, double s) {
  int64_t lo = sb, hi = se - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (v.seg_send[mid] >= s) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// Forward walk (increasing s).  emit(int64_t k, int layer, double len) per merged
// segment: k indexes the view's 2D segment arrays, FSR j = seg_region[k] * NL + layer.
template <class Emit>
MOC_HD int otf_walk_fwd(const OtfView& v, const TrackGeo& g, Emit&& emit) {
  double s_in, s_out;
  otf_clip(g, s_in, s_out);
  const bool up = g.cot > 0;
  int l;
  int64_t k;
  if (s_in > 0.0) {
    l = up ? 0 : v.NL - 1;
    k = otf_seg_after(v, g.sb, g.se, s_in);
  } else {
    l = up ? otf_layer_up(v, g.z0) : otf_layer_down(v, g.z0);
    k = g.sb;
  }
  double s = s_in;
  int64_t pk = -1;
  int pl = 0;
  double pL = 0.0;
  bool lead = false;
  int n = 0;
  while (true) {
    const double s_rad = v.seg_send[k];
    const double s_ax = ((up ? v.planes[l + 1] : v.planes[l]) - g.z0) * g.tan;
    double s_next = s_rad < s_ax ? s_rad : s_ax;
    s_next = s_next < s_out ? s_next : s_out;
    const double L3 = (s_next - s) * g.invsin;
    if (pk < 0) {
      pk = k;
      pl = l;
      pL = L3;
      lead = L3 < kEpsL;
    } else if (L3 < kEpsL) {
      pL += L3;
    } else if (lead) {
      pk = k;
      pl = l;
      pL += L3;
      lead = false;
    } else {
      emit(pk, pl, pL);
      ++n;
      pk = k;
      pl = l;
      pL = L3;
    }
    if (s_next >= s_out) break;
    if (s_rad <= s_ax) ++k; else l += up ? 1 : -1;
    s = s_next;
  }
  emit(pk, pl, pL);
  return n + 1;
}

// Backward walk (decreasing s): emits the reverse of otf_walk_fwd's list.
template <class Emit>
MOC_HD int otf_walk_bwd(const OtfView& v, const TrackGeo& g, Emit&& emit) {
  double s_in, s_out;
  otf_clip(g, s_in, s_out);
  const bool up = g.cot > 0;
  int l;
  int64_t k;
  if (s_out < g.L) {
    l = up ? v.NL - 1 : 0;
    k = otf_seg_upto(v, g.sb, g.se, s_out);
  } else {
    const double z_out = g.z0 + g.L * g.cot;
    l = up ? otf_layer_down(v, z_out) : otf_layer_up(v, z_out);
    k = g.se - 1;
  }
  double s = s_out;
  int64_t pk = -1, lk = -1;
  int pl = 0, ll = 0;
  double pL = 0.0, carry = 0.0;
  int n = 0;
  while (true) {
    const double s_rad = k > g.sb ? v.seg_send[k - 1] : 0.0;
    const double s_ax = ((up ? v.planes[l] : v.planes[l + 1]) - g.z0) * g.tan;
    double s_prev = s_rad > s_ax ? s_rad : s_ax;
    s_prev = s_prev > s_in ? s_prev : s_in;
    const double L3 = (s - s_prev) * g.invsin;
    if (L3 < kEpsL) {
      carry += L3;
      lk = k;
      ll = l;
    } else {
      if (pk >= 0) {
        emit(pk, pl, pL);
        ++n;
      }
      pk = k;
      pl = l;
      pL = L3 + carry;
      carry = 0.0;
    }
    if (s_prev <= s_in) break;
    if (s_rad >= s_ax) --k; else l -= up ? 1 : -1;
    s = s_prev;
  }
  if (pk >= 0) {
    emit(pk, pl, pL + carry);
  } else {
    emit(lk, ll, carry);
  }
  return n + 1;
}

// FNV-1a-64 over uint32 little-endian FSR ids (checksum definition).
MOC_HD uint64_t fnv1a_step(uint64_t h, uint32_t u) {
  for (int b = 0; b < 4; ++b) {
    h ^= (uint64_t)((u >> (8 * b)) & 0xffu);
    h *= 1099511628211ull;
  }
  return h;
}
constexpr uint64_t kFnvInit = 14695981039346656037ull;

}  // namespace moc
