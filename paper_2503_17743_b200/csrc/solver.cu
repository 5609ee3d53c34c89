// solver.cu — device side of libmoc3d.so: HBM layout, the OTF sweep kernels and
// the per-iteration FSR kernels, plus the solver ABI.
//
// HBM layout (SoA):
//   2D segments   seg_send f64[N2], seg_region u32[N2]       (A1, preloaded once)
//   2D tracks     t_len f64, t_seg i64[T2+1], t_a i32
//   (a, n)        cot, tan, 1/sin, dz f64; c = W A_perp f32
//   z-stacks      st_z0 f64[S], st_first u32[S+1]            (Alg. 1 order)
//   3D links      link u32[2*T3] (slot -> slot, ~0 = vacuum) (A6)
//   work list     work u32[T3]                               (schedule, §4.3)
//   boundary psi  psi f32[2][2*T3][GP]  (Jacobi double buffer, lazily normalised)
//   FSR arrays    mat u8[J], qt f32[J][GP], phi f32[J][GP], tally f64[J][GP], vol f64[J]
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: NCCL is loaded at run time (nccl_api below)
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host.h"
#include "otf.h"

using namespace moc;

#define CUDA_OK(x)                                                                              \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw Error(e_ == cudaErrorMemoryAllocation ? MOC_E_CAPACITY : MOC_E_CUDA,               \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                            \
  } while (0)

namespace {

constexpr int kMaxMat = 32;
constexpr int kMaxG = 8;
constexpr double kFourPi = 12.566370614359172;

__constant__ float c_sigt2[kMaxMat * kMaxG];     // sigma_t * log2(e)   (for ex2)
__constant__ float c_sigt[kMaxMat * kMaxG];      // sigma_t
__constant__ float c_nusf[kMaxMat * kMaxG];
__constant__ float c_chi[kMaxMat * kMaxG];
__constant__ float c_sigs[kMaxMat * kMaxG * kMaxG];  // [m][from][to]
__constant__ double c_planes[256];                   // axial planes (kMaxPlanes, sweep_v2.cuh)

// device scalars (fp64): index map
enum {
  SC_K = 0,        // current k
  SC_KPREV,        // k before the last update
  SC_PROD_OLD,     // sum V F(phi) at the start of the iteration
  SC_PROD_NEW,     // sum V F(phi_new) before normalisation
  SC_SCALE,        // 1 / SC_PROD_NEW
  SC_PSI_SCALE,    // scale applied to psi_in on read (lazy normalisation, Q12)
  SC_RESID,        // RMS fission-source residual
  SC_LEAK,         // vacuum outflow tally (unscaled) of the last sweep
  SC_LEAK_SCALED,
  SC_BAD,          // count of NaN/negative fluxes in the last finalize
  SC_ITER,         // completed iterations
  SC_NEMIT,        // merged segment-direction emissions of the running sweep (this rank)
  SC_NEMIT_LAST,   // ... of the last completed iteration
  SC_N
};

struct DevData {
  const double* seg_send;
  const uint32_t* seg_region;
  const double* planes;
  int32_t NL;
  double Z;
  const double* t_len;
  const int64_t* t_seg;
  const int32_t* t_a;
  const double *an_cot, *an_tan, *an_invsin, *an_dz;
  const float* an_c;
  const double* an_vw;  // W/(2 pi) * A_perp (volume weight)
  const double* st_z0;
  const uint32_t* st_first;
  int32_t S, N;
  uint32_t T3;
};

__device__ __forceinline__ int find_stack(const DevData& d, uint32_t id) {
  int lo = 0, hi = d.S - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (d.st_first[mid] <= id) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ TrackGeo dev_track(const DevData& d, uint32_t id, int& stack, int& an) {
  int s = find_stack(d, id);
  int t = s / d.N, n = s - t * d.N;
  an = d.t_a[t] * d.N + n;
  stack = s;
  TrackGeo g;
  g.z0 = d.st_z0[s] + (double)(id - d.st_first[s]) * d.an_dz[an];
  g.cot = d.an_cot[an];
  g.tan = d.an_tan[an];
  g.invsin = d.an_invsin[an];
  g.L = d.t_len[t];
  g.Z = d.Z;
  g.sb = d.t_seg[t];
  g.se = d.t_seg[t + 1];
  return g;
}

__device__ __forceinline__ OtfView dev_view(const DevData& d) {
  return OtfView{d.seg_send, d.seg_region, d.planes, d.NL};
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------------ setup kernels
__global__ void k_volumes_costs(DevData d, double* vol, uint32_t* cost, unsigned long long* nseg_total) {
  unsigned long long local = 0;
  const OtfView v = dev_view(d);
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < d.T3; id += gridDim.x * blockDim.x) {
    int s, an;
    TrackGeo g = dev_track(d, id, s, an);
    const double w = d.an_vw[an];
    int n = otf_walk_fwd(v, g, [&](int64_t k, int l, double len) {
      atomicAdd(&vol[(int64_t)v.seg_region[k] * v.NL + l], w * len);
    });
    cost[id] = (uint32_t)n;
    local += (unsigned long long)n;
  }
  atomicAdd(nseg_total, local);
}

__global__ void k_checksums(DevData d, uint32_t first, uint32_t n, int32_t* nseg, unsigned long long* hash,
                            double* suml) {
  const OtfView v = dev_view(d);
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    int s, an;
    TrackGeo g = dev_track(d, first + q, s, an);
    uint64_t h = kFnvInit;
    double sl = 0;
    int c = otf_walk_fwd(v, g, [&](int64_t k, int l, double len) {
      h = fnv1a_step(h, (uint32_t)((int64_t)v.seg_region[k] * v.NL + l));
      sl += len;
    });
    nseg[q] = c;
    hash[q] = h;
    suml[q] = sl;
  }
}

__global__ void k_serpentine(uint32_t* work, uint64_t n, uint64_t chunk) {
  // reverse every odd chunk in place: thread per pair in odd chunks
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = x / chunk;
    if (!(c & 1)) continue;
    uint64_t c0 = c * chunk, c1 = min(n, c0 + chunk);
    uint64_t off = x - c0, len = c1 - c0;
    if (off < len / 2) {
      uint32_t a = work[c0 + off], b = work[c1 - 1 - off];
      work[c0 + off] = b;
      work[c1 - 1 - off] = a;
    }
  }
}

// ------------------------------------------------------------ A3: source
// qtilde_j,g = [chi_g F_j / k + sum_g' Ss[g'->g] phi_j,g'] / (4 pi Sigma_t)   (Q2)
// F_j = sum_g nuSf phi (for k and the residual); block partials of sum V F.
template <int G, int GP>
__global__ void k_source(int64_t J, const uint8_t* mat, const float* phi, const double* vol, const double* sc,
                         float* qt, float* fold, double* part) {
  __shared__ double red[32];
  double acc = 0;
  const double k = sc[SC_K];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < J; j += (int64_t)gridDim.x * blockDim.x) {
    int m = mat[j];
    float ph[G];
#pragma unroll
    for (int g = 0; g < G; ++g) ph[g] = phi[j * GP + g];
    float F = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) F = fmaf(c_nusf[m * kMaxG + g], ph[g], F);
    float fk = (float)(F / k);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float s = c_chi[m * kMaxG + g] * fk;
#pragma unroll
      for (int h = 0; h < G; ++h) s = fmaf(c_sigs[(m * kMaxG + h) * kMaxG + g], ph[h], s);
      qt[j * GP + g] = s / ((float)kFourPi * c_sigt[m * kMaxG + g]);
    }
    if constexpr (G < GP) qt[j * GP + G] = __int_as_float(m);  // material for the v2 sweep's prefetch
    fold[j] = F;
    acc += vol[j] * (double)F;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
  }
}

// ------------------------------------------------------------ A4-A6: sweep (v1)
// Alg. 2: grid-stride over 3D tracks in `work` order.  Each thread
// walks its track forward then backward (Q24), applies Eq. 3 per segment and
// group, accumulates c * dpsi into the FSR tally with fp64 atomics (Eq. 4, Q1),
// and writes the outgoing psi into the linked slot of the other buffer (Q9).
template <int G, int GP>
__global__ void __launch_bounds__(512) k_sweep_v1(DevData d, const uint32_t* work, uint32_t nwork,
                                                  const uint32_t* link, const uint8_t* mat, const float* qt,
                                                  const float* psi_in, float* psi_out, double* tally, double* sc) {
  const OtfView v = dev_view(d);
  const float ps = (float)sc[SC_PSI_SCALE];
  double leak = 0;
  uint64_t nemit = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwork; w += gridDim.x * blockDim.x) {
    const uint32_t id = work[w];
    int s, an;
    TrackGeo g = dev_track(d, id, s, an);
    const float c = d.an_c[an];
    for (int dir = 0; dir < 2; ++dir) {
      const uint32_t slot = 2 * id + dir;
      float psi[G];
#pragma unroll
      for (int q = 0; q < G; ++q) psi[q] = psi_in[(size_t)slot * GP + q] * ps;
      auto seg = [&](int64_t k, int l, double len) {
        ++nemit;
        const int64_t j = (int64_t)v.seg_region[k] * v.NL + l;
        const float Lf = (float)len;
        const int m = mat[j];
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const float E = ex2_approx(-c_sigt2[m * kMaxG + q] * Lf);
          const float dd = psi[q] - qt[j * GP + q];
          const float dl = fmaf(-dd, E, dd);  // (psi - qtilde)(1 - e^{-tau})
          psi[q] -= dl;
          atomicAdd(&tally[j * GP + q], (double)(c * dl));
        }
      };
      if (dir == 0) otf_walk_fwd(v, g, seg); else otf_walk_bwd(v, g, seg);
      const uint32_t out = link[slot];
      if (out != 0xffffffffu) {
#pragma unroll
        for (int q = 0; q < G; ++q) psi_out[(size_t)out * GP + q] = psi[q];
      } else {
        float e = 0;
#pragma unroll
        for (int q = 0; q < G; ++q) e += psi[q];
        leak += (double)(c * e);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    leak += __shfl_xor_sync(0xffffffffu, leak, o);
    nemit += __shfl_xor_sync(0xffffffffu, nemit, o);
  }
  if ((threadIdx.x & 31) == 0 && leak != 0.0) atomicAdd(&sc[SC_LEAK], leak);
  if ((threadIdx.x & 31) == 0 && nemit) atomicAdd(&sc[SC_NEMIT], (double)nemit);
}

// ------------------------------------------------------------ A7: finalize
// phi_new = 4 pi qtilde + T / (Sigma_t V)   (Q2); block partials of sum V F(phi_new)
template <int G, int GP, class TT>
__global__ void k_finalize(int64_t J, const uint8_t* mat, const float* qt, const TT* tally, const double* vol,
                           float* phi, float* fnew, double* part, double* sc) {
  __shared__ double red[32];
  double acc = 0;
  int bad = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < J; j += (int64_t)gridDim.x * blockDim.x) {
    int m = mat[j];
    double V = vol[j];
    float F = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double p = kFourPi * (double)qt[j * GP + g] + (double)tally[j * GP + g] / ((double)c_sigt[m * kMaxG + g] * V);
      float pf = (float)p;
      if (!(pf >= 0.f)) ++bad;
      phi[j * GP + g] = pf;
      F = fmaf(c_nusf[m * kMaxG + g], pf, F);
    }
    fnew[j] = F;
    acc += V * (double)F;
  }
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = acc;
    if (bad) atomicAdd(&sc[SC_BAD], (double)bad);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
  }
}

// k update (single block): k_new = k * sum V F_new / sum V F_old; scale = 1 / sum V F_new
__global__ void k_keff(const double* part_old, const double* part_new, int nb, double* sc) {
  __shared__ double r1[32], r2[32];
  double a = 0, b = 0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += part_old[i];
    b += part_new[i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    r1[threadIdx.x >> 5] = a;
    r2[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0;
    b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += r1[w];
      b += r2[w];
    }
    double k = sc[SC_K];
    sc[SC_KPREV] = k;
    sc[SC_PROD_OLD] = a;
    sc[SC_PROD_NEW] = b;
    double knew = (a > 0 && b > 0) ? k * b / a : 0.0;
    sc[SC_K] = knew;
    double scale = b > 0 ? 1.0 / b : 0.0;
    sc[SC_SCALE] = scale;
    sc[SC_PSI_SCALE] = scale;
    sc[SC_LEAK_SCALED] = sc[SC_LEAK] * scale;
  }
}

// normalise phi (Q12) and residual partials: RMS over fissile FSRs of (F_new - F_old)/F_new
template <int G, int GP>
__global__ void k_normalize(int64_t J, float* phi, const float* fnew, const float* fold, const double* sc,
                            double* part2) {
  __shared__ double r1[32], r2[32];
  const float scale = (float)sc[SC_SCALE];
  double a = 0, n = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < J; j += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int g = 0; g < G; ++g) phi[j * GP + g] *= scale;
    float Fn = fnew[j] * scale;
    if (Fn > 0.f) {
      double d = ((double)Fn - (double)fold[j]) / (double)Fn;
      a += d * d;
      n += 1.0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    n += __shfl_xor_sync(0xffffffffu, n, o);
  }
  if ((threadIdx.x & 31) == 0) {
    r1[threadIdx.x >> 5] = a;
    r2[threadIdx.x >> 5] = n;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    a = threadIdx.x < (blockDim.x >> 5) ? r1[threadIdx.x] : 0.0;
    n = threadIdx.x < (blockDim.x >> 5) ? r2[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      n += __shfl_xor_sync(0xffffffffu, n, o);
    }
    if (threadIdx.x == 0) {
      part2[2 * blockIdx.x] = a;
      part2[2 * blockIdx.x + 1] = n;
    }
  }
}

__global__ void k_resid(const double* part2, int nb, double* sc, double* hist, int hist_cap) {
  __shared__ double r1[32], r2[32];
  double a = 0, n = 0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += part2[2 * i];
    n += part2[2 * i + 1];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    n += __shfl_xor_sync(0xffffffffu, n, o);
  }
  if ((threadIdx.x & 31) == 0) {
    r1[threadIdx.x >> 5] = a;
    r2[threadIdx.x >> 5] = n;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0;
    n = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += r1[w];
      n += r2[w];
    }
    double r = n > 0 ? sqrt(a / n) : 0.0;
    sc[SC_RESID] = r;
    int it = (int)sc[SC_ITER];
    if (it < hist_cap) {
      hist[2 * it] = sc[SC_K];
      hist[2 * it + 1] = r;
    }
    sc[SC_ITER] = it + 1;
    sc[SC_LEAK] = 0.0;
    sc[SC_NEMIT_LAST] = sc[SC_NEMIT];
    sc[SC_NEMIT] = 0.0;
  }
}

// halo gather (dir 0: buf[q] = psi[slot[q]]) / scatter (dir 1: psi[slot[q]] = buf[q]), GP floats per slot
__global__ void k_halo_move(float* psi, const uint32_t* slots, int64_t n, int GP, float* buf, int dir) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * GP; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / GP;
    const int g = (int)(e - q * GP);
    float* p = psi + (size_t)slots[q] * GP + g;
    if (dir == 0) buf[e] = *p; else *p = buf[e];
  }
}

// leakage rides in the tally's tail through the all-reduce (dir 0: park, dir 1: restore)
__global__ void k_leak_park(double* sc, float* tail, int dir) {
  if (dir == 0) {
    tail[0] = (float)sc[SC_LEAK];
    sc[SC_LEAK] = 0.0;
  } else {
    sc[SC_LEAK] = (double)tail[0];
  }
}

// phi f32 [J][GP] -> f64 [J][G] (the host API's layout), so moc_get_scalar_flux is one
// device-side conversion and one DMA into the caller's buffer
__global__ void k_phi_f64(const float* phi, int64_t J, int G, int GP, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < J * G; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / G;
    out[i] = (double)phi[j * GP + (i - j * G)];
  }
}

__global__ void k_fill_f32(float* p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

}  // namespace

#include "sweep_v2.cuh"
#include "sweep_sc.cuh"

namespace {

template <class T>
T* dmalloc(size_t n, int64_t& bytes) {
  T* p = nullptr;
  if (n == 0) n = 1;
  CUDA_OK(cudaMalloc(&p, n * sizeof(T)));
  bytes += (int64_t)(n * sizeof(T));
  return p;
}

// NCCL loaded at run time (dlopen libnccl.so.2): the single-GPU library has no NCCL link
// dependency, and in a torch process the already-loaded copy is reused.
struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
#define MOC_SYM(f, name)                                      \
  a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, name));     \
  if (!a.f) {                                                 \
    a.why = std::string("libnccl.so.2 lacks ") + name;        \
    return a;                                                 \
  }
    MOC_SYM(getUniqueId, "ncclGetUniqueId")
    MOC_SYM(commInitRank, "ncclCommInitRank")
    MOC_SYM(commDestroy, "ncclCommDestroy")
    MOC_SYM(allReduce, "ncclAllReduce")
    MOC_SYM(send, "ncclSend")
    MOC_SYM(recv, "ncclRecv")
    MOC_SYM(groupStart, "ncclGroupStart")
    MOC_SYM(groupEnd, "ncclGroupEnd")
    MOC_SYM(errorString, "ncclGetErrorString")
#undef MOC_SYM
    a.ok = true;
    return a;
  }();
  if (!api.ok) throw Error(MOC_E_NCCL, api.why);
  return api;
}

#define NCCL_OK(call)                                                                           \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess)                                                                      \
      throw Error(MOC_E_NCCL, std::string(#call) + ": " + nccl_api().errorString(r_));        \
  } while (0)

}  // namespace

struct moc_solver {
  std::string err;
  int device = 0;
  uint64_t uid = 0;           // process-unique id: owner tag of the per-device __constant__ tables
  double* h_planes = nullptr; // pinned copy of the axial planes (re-uploaded with the XS tables)
  cudaStream_t stream = nullptr;
  moc_solver_opts opts{};
  moc_comm_desc comm{0, 1, 0};
  int G = 0, GP = 0, N = 0, M = 0, NL = 0, n_mat = 0;
  int64_t J = 0, T2 = 0, S = 0, T3 = 0, N2 = 0, nseg3 = 0;
  int64_t dev_bytes = 0;
  double setup_ms = 0;
  DevData dd{};
  // device buffers
  double *d_seg_send = nullptr, *d_planes = nullptr, *d_t_len = nullptr;
  uint32_t* d_seg_region = nullptr;
  int64_t* d_t_seg = nullptr;
  int32_t* d_t_a = nullptr;
  double *d_an_cot = nullptr, *d_an_tan = nullptr, *d_an_invsin = nullptr, *d_an_dz = nullptr, *d_an_vw = nullptr;
  float* d_an_c = nullptr;
  double* d_st_z0 = nullptr;
  uint32_t* d_st_first = nullptr;
  uint32_t* d_link = nullptr;
  uint32_t* d_work = nullptr;
  uint32_t nwork = 0;
  uint32_t* d_cost = nullptr;
  uint8_t* d_mat = nullptr;
  float *d_qt = nullptr, *d_phi = nullptr, *d_fold = nullptr, *d_fnew = nullptr;
  cudaTextureObject_t qtex = 0;  // d_qt as float4 texture (GP = 8: the sweeps' source gather)
  double* d_phi64 = nullptr;  // [J][G] staging for moc_get_scalar_flux (allocated on first use)
  double *d_tally = nullptr, *d_vol = nullptr;
  float* d_psi[2] = {nullptr, nullptr};
  double *d_sc = nullptr, *d_part_a = nullptr, *d_part_b = nullptr, *d_part_c = nullptr, *d_hist = nullptr;
  int hist_cap = 100000;
  int cur = 0;  // psi buffer holding the incoming fluxes
  int nb_fsr = 0, sweep_blocks = 0, sweep_threads = 256;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double sweep_ms_last = 0, iter_ms_last = 0;
  bool sweep_timed = false;
  std::vector<double> sigma_t, nusf, sigs;  // host copies (balance)
  std::vector<int32_t> mat_host;
  std::vector<double> vol_analytic;  // S:83-85, host copy
  float* h_xs = nullptr;  // pinned staging for cross-section uploads
  int64_t xs_bytes = 0;
  // v2 (schedule 0): persistent stack-band units
  Unit* d_units = nullptr;
  uint32_t n_units = 0;
  uint32_t* d_counter = nullptr;
  float *d_rmax = nullptr, *d_qmax_t = nullptr, *d_tally32 = nullptr;
  int* d_err = nullptr;
  int cap_cells = 0;  // v2 tile capacity in cells (sweep_v2.cuh layout)
  int tile_off = 0;   // v2 tile byte offset (above the largest unit's tables)
  int lane_lg = -1;  // forced log2 v2 lane stride (opts.v2_lane_stride), -1 = per unit
  double h_lane = 0;     // thinnest axial layer / 3 (sweep_v2.cuh lane_lg_of)
  size_t v2_smem = 0;
  uint32_t* d_unit_maxq = nullptr;  // longest track (merged segments) per unit
  // EXP preload (§4.2): record offsets per unit (kNoExp = on the fly) and the store
  uint64_t* d_unit_exp = nullptr;
  Rec* d_store = nullptr;
  int64_t exp_units = 0, exp_segments = 0, exp_bytes = 0;
  // stack-collective sweep (schedule 3, sweep_sc.cuh)
  ScUnit* d_sc_units = nullptr;
  uint32_t n_sc_units = 0;
  // per occupancy g (kScMinBlocksList[g] CTAs per SM): psi band capacity, dynamic shared
  // memory, grid, and the units it sweeps (d_sc_units[first, first + n))
  struct ScGroup {
    int pcap = 0, blocks = 0;
    size_t smem = 0;
    uint32_t first = 0, n = 0;
  } sc_grp[3];
  size_t sc_smem_hash = 0;
  int sc_blocks_hash = 0;
  double hmin = 0;
  // multi-GPU (world > 1)
  uint32_t *d_send_slots = nullptr, *d_recv_slots = nullptr;
  int64_t n_send = 0, n_recv = 0;
  float *d_halo_send = nullptr, *d_halo_recv = nullptr;
  std::vector<int64_t> send_counts, recv_counts;  // per peer, in slots
  double owned_cost = 0;
  uint32_t* d_slot_first = nullptr; // per stack: first track of this rank's numbering (world > 1)
  int64_t T3_local = 0;             // tracks this rank sweeps (= T3 on one GPU)
  int64_t psi_slots = 0;            // boundary-psi slots per buffer: 2 T3_local (+ halo send tail)
  ncclComm_t nccl = nullptr;        // backend MOC_COMM_NCCL: library-owned communicator
  moc_exchange_fn xfn = nullptr;    // backend MOC_COMM_CALLER: host exchange callback
  void* xctx = nullptr;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};  // one iteration, per Jacobi buffer parity
  cudaStream_t cap_stream = nullptr;  // private non-blocking stream the graphs are captured on
};

namespace {

void upload(const void* h, void* d, size_t bytes, cudaStream_t st) {
  if (bytes) CUDA_OK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
}

// The __constant__ tables (cross sections, axial planes) are per device, shared by every
// solver in the process: the solver whose kernels run next re-uploads its own copies when it
// is not the last owner (one solver active per device at a time; stream-ordered uploads).
// (atomic: several host threads may each drive their own solver; the tables themselves are
// still one set per device, so solvers sharing a device must not run concurrently)
std::atomic<uint64_t>& const_owner(int dev) {
  static std::atomic<uint64_t> owner[64] = {};
  return owner[dev & 63];
}
void ensure_constants(moc_solver* s) {
  if (const_owner(s->device) == s->uid || !s->h_xs) return;
  const size_t a = sizeof(float) * kMaxMat * kMaxG;
  float* t2 = s->h_xs;
  CUDA_OK(cudaMemcpyToSymbolAsync(c_sigt2, t2, a, 0, cudaMemcpyHostToDevice, s->stream));
  CUDA_OK(cudaMemcpyToSymbolAsync(c_sigt, t2 + kMaxMat * kMaxG, a, 0, cudaMemcpyHostToDevice, s->stream));
  CUDA_OK(cudaMemcpyToSymbolAsync(c_nusf, t2 + 2 * kMaxMat * kMaxG, a, 0, cudaMemcpyHostToDevice, s->stream));
  CUDA_OK(cudaMemcpyToSymbolAsync(c_chi, t2 + 3 * kMaxMat * kMaxG, a, 0, cudaMemcpyHostToDevice, s->stream));
  CUDA_OK(cudaMemcpyToSymbolAsync(c_sigs, t2 + 4 * kMaxMat * kMaxG, a * kMaxG, 0, cudaMemcpyHostToDevice, s->stream));
  if (s->h_planes)
    CUDA_OK(cudaMemcpyToSymbolAsync(c_planes, s->h_planes, sizeof(double) * (s->NL + 1), 0, cudaMemcpyHostToDevice,
                                    s->stream));
  const_owner(s->device) = s->uid;
}

// cross-section tables -> __constant__ (padded to kMaxMat x kMaxG); the fp32 tables the
// kernels read; sigma_t * log2(e) for the ex2-based exponential.  Pinned staging buffer
// so the copy is truly asynchronous on the solver's stream.
void upload_materials(moc_solver* s, const double* sigma_t, const double* sigma_s, const double* nusf,
                      const double* chi) {
  const int G = s->G, NM = s->n_mat;
  if (!s->h_xs) CUDA_OK(cudaMallocHost(&s->h_xs, sizeof(float) * kMaxMat * kMaxG * (4 + kMaxG)));
  float* t2 = s->h_xs;
  float* t1 = t2 + kMaxMat * kMaxG;
  float* nf = t1 + kMaxMat * kMaxG;
  float* ch = nf + kMaxMat * kMaxG;
  float* ss = ch + kMaxMat * kMaxG;
  std::memset(s->h_xs, 0, sizeof(float) * kMaxMat * kMaxG * (4 + kMaxG));
  for (int m = 0; m < NM; ++m)
    for (int q = 0; q < G; ++q) {
      t1[m * kMaxG + q] = (float)sigma_t[(size_t)m * G + q];
      t2[m * kMaxG + q] = (float)(sigma_t[(size_t)m * G + q] * 1.4426950408889634);
      nf[m * kMaxG + q] = (float)nusf[(size_t)m * G + q];
      ch[m * kMaxG + q] = (float)chi[(size_t)m * G + q];
      for (int h = 0; h < G; ++h) ss[(m * kMaxG + q) * kMaxG + h] = (float)sigma_s[((size_t)m * G + q) * G + h];
    }
  const size_t a = sizeof(float) * kMaxMat * kMaxG;
  s->xs_bytes = (int64_t)(a * (4 + kMaxG));
  const_owner(s->device) = 0;  // force the upload below
  ensure_constants(s);
  s->sigma_t.assign(sigma_t, sigma_t + (size_t)NM * G);
  s->nusf.assign(nusf, nusf + (size_t)NM * G);
  s->sigs.assign(sigma_s, sigma_s + (size_t)NM * G * G);
}

template <int G, int GP, bool HASH = false>
void run_sweep_sc(moc_solver* s, unsigned long long* hash = nullptr, int32_t* nseg = nullptr) {
  ScArgs a;
  a.d = s->dd;
  a.link = s->d_link;
  a.mat = s->d_mat;
  a.qt = s->d_qt;
  a.qtex = s->qtex;
  a.psi_in = s->d_psi[s->cur];
  a.psi_out = s->d_psi[1 - s->cur];
  a.tally = s->d_tally32;
  a.sc = s->d_sc;
  a.inv_hmin = (1.0 / s->hmin) * (1.0 + 1e-12);
  a.h_fast = s->hmin * (1.0 - 1e-9);
  a.err = s->d_err;
  a.hash = hash;
  a.nseg = nseg;
  a.gs = s->opts.gauss_seidel;
  a.slot_first = s->d_slot_first ? s->d_slot_first : s->d_st_first;
  a.n_slots = (uint64_t)s->psi_slots;
  a.n_fsr = (uint64_t)s->J;
  if constexpr (HASH) {  // every unit, 3 CTAs per SM (the largest band capacity)
    a.units = s->d_sc_units;
    a.n_units = s->n_sc_units;
    a.counter = s->d_counter;
    a.pcap = s->sc_grp[0].pcap;
    k_sweep_sc<G, GP, true, 3><<<s->sc_blocks_hash, kScThreads, s->sc_smem_hash, s->stream>>>(a);
  } else {
    // one launch per occupancy group, each with its own unit queue counter
    for (int g = 0; g < 3; ++g) {
      const auto& q = s->sc_grp[g];
      if (q.n == 0) continue;
      a.units = s->d_sc_units + q.first;
      a.n_units = q.n;
      a.counter = s->d_counter + g;
      a.pcap = q.pcap;
      if (g == 0) k_sweep_sc<G, GP, false, 3><<<q.blocks, kScThreads, q.smem, s->stream>>>(a);
      else if (g == 1) k_sweep_sc<G, GP, false, 4><<<q.blocks, kScThreads, q.smem, s->stream>>>(a);
      else k_sweep_sc<G, GP, false, 5><<<q.blocks, kScThreads, q.smem, s->stream>>>(a);
    }
  }
}

template <int G, int GP>
void run_sweep(moc_solver* s) {
  const int in = s->cur, out = 1 - s->cur;
  if (s->opts.schedule == 3) {
    run_sweep_sc<G, GP>(s);
  } else if (s->opts.schedule == 0) {
    V2Args a;
    a.d = s->dd;
    a.units = s->d_units;
    a.n_units = s->n_units;
    a.counter = s->d_counter;
    a.link = s->d_link;
    a.mat = s->d_mat;
    a.qt = s->d_qt;
    a.qtex = s->qtex;
    a.qmax_t = s->d_qmax_t;
    a.psi_in = s->d_psi[in];
    a.psi_out = s->d_psi[out];
    a.tally = s->d_tally32;
    a.sc = s->d_sc;
    a.tile_off = s->tile_off;
    a.cap_cells = s->cap_cells;
    a.lane_lg = s->lane_lg;
    a.h_lane = s->h_lane;
    a.err = s->d_err;
    a.slot_first = s->d_slot_first ? s->d_slot_first : s->d_st_first;
    a.unit_exp = s->d_unit_exp;
    a.store = s->d_store;
    a.cost = s->d_cost;
    // EXP (§4.2): the preloaded units are a prefix of the cost-sorted list; replay them,
    // then sweep the rest on the fly (each kernel pulls from its own counter)
    const uint32_t n_exp = (uint32_t)s->exp_units;
    if (n_exp) {
      a.n_units = n_exp;
      k_sweep_v2<G, GP, true><<<s->sweep_blocks, kV2Threads, s->v2_smem, s->stream>>>(a);
    }
    if (s->n_units > n_exp) {
      a.units = s->d_units + n_exp;
      a.unit_exp = nullptr;
      a.n_units = s->n_units - n_exp;
      a.counter = s->d_counter + 1;
      k_sweep_v2<G, GP, false><<<s->sweep_blocks, kV2Threads, s->v2_smem, s->stream>>>(a);
    }
  } else {
    k_sweep_v1<G, GP><<<s->sweep_blocks, s->sweep_threads, 0, s->stream>>>(
        s->dd, s->d_work, s->nwork, s->d_link, s->d_mat, s->d_qt, s->d_psi[in], s->d_psi[out], s->d_tally, s->d_sc);
  }
}

template <int G, int GP>
void v2_configure(moc_solver* s) {
  // kV2MinBlocks CTAs per SM: 228 KB of shared memory per SM, 1 KB reserved per CTA;
  // the dynamic part (the tally tile) is what the static per-unit tables leave.
  cudaFuncAttributes fa{}, fb{};
  CUDA_OK(cudaFuncGetAttributes(&fa, k_sweep_v2<G, GP, false>));
  CUDA_OK(cudaFuncGetAttributes(&fb, k_sweep_v2<G, GP, true>));
  const size_t per_cta = (228 * 1024) / kV2MinBlocks - 1024;
  s->v2_smem = (per_cta - std::max(fa.sharedSizeBytes, fb.sharedSizeBytes)) & ~size_t(15);
  CUDA_OK(cudaFuncSetAttribute(k_sweep_v2<G, GP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)s->v2_smem));
  CUDA_OK(cudaFuncSetAttribute(k_sweep_v2<G, GP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)s->v2_smem));
  int per_sm = 0, per_sm_b = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_v2<G, GP, false>, kV2Threads, s->v2_smem));
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, k_sweep_v2<G, GP, true>, kV2Threads, s->v2_smem));
  per_sm = std::min(per_sm, per_sm_b);
  if (per_sm < 1) throw Error(MOC_E_CAPACITY, "sweep kernel does not fit on an SM");
  int dev = 0, nsm = 0;
  CUDA_OK(cudaGetDevice(&dev));
  CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  s->sweep_blocks = nsm * per_sm;
  s->sweep_threads = kV2Threads;
}

// an event record that is also an event-record node when the stream is being captured
// into the iteration's CUDA graph (so every replay re-times the sweep)
void record_event(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_OK(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusActive) CUDA_OK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
  else CUDA_OK(cudaEventRecord(e, st));
}

// first half of an iteration: A3 source, A4-A6 sweep of this rank's units; for world > 1
// also gathers the halo (outgoing psi of cut-crossing links) and parks the leakage in the
// tally's tail so one all-reduce carries both.
template <int G, int GP>
void iter_sweep_half(moc_solver* s, bool time_it) {
  ensure_constants(s);
  const bool v2 = s->opts.schedule == 0, f32t = v2 || s->opts.schedule == 3;
  const int nb = s->nb_fsr;
  k_source<G, GP><<<nb, 256, 0, s->stream>>>(s->J, s->d_mat, s->d_phi, s->d_vol, s->d_sc, s->d_qt, s->d_fold,
                                             s->d_part_a);
  if (v2) {
    k_region_qmax<G, GP><<<64, 256, 0, s->stream>>>(s->J / s->NL, s->NL, s->d_qt, s->d_rmax);
    k_track_qmax<G, GP><<<64, 256, 0, s->stream>>>(s->T2, s->d_t_seg, s->d_seg_region, s->d_rmax, s->d_qmax_t);
  }
  if (f32t) {
    CUDA_OK(cudaMemsetAsync(s->d_tally32, 0, sizeof(float) * s->J * s->GP, s->stream));
    CUDA_OK(cudaMemsetAsync(s->d_counter, 0, (s->opts.schedule == 3 ? 4 : 2) * sizeof(uint32_t), s->stream));
  } else {
    CUDA_OK(cudaMemsetAsync(s->d_tally, 0, sizeof(double) * s->J * s->GP, s->stream));
  }
  if (time_it) record_event(s->ev[0], s->stream);
  run_sweep<G, GP>(s);
  if (time_it) {
    record_event(s->ev[1], s->stream);
    s->sweep_timed = true;
  }
  if (s->comm.world > 1) {
    if (s->n_send) k_halo_move<<<256, 256, 0, s->stream>>>(s->d_psi[1 - s->cur], s->d_send_slots, s->n_send, GP,
                                                          s->d_halo_send, 0);
    k_leak_park<<<1, 1, 0, s->stream>>>(s->d_sc, s->d_tally32 + s->J * GP, 0);
  }
  CUDA_OK(cudaGetLastError());
}

// second half: (after the caller's all-reduce / halo exchange) scatter the halo, A7.
template <int G, int GP>
void iter_finish_half(moc_solver* s) {
  ensure_constants(s);
  const bool v2 = s->opts.schedule == 0 || s->opts.schedule == 3;  // fp32 tally
  const int nb = s->nb_fsr;
  if (s->comm.world > 1) {
    if (s->n_recv) k_halo_move<<<256, 256, 0, s->stream>>>(s->d_psi[1 - s->cur], s->d_recv_slots, s->n_recv, GP,
                                                          s->d_halo_recv, 1);
    k_leak_park<<<1, 1, 0, s->stream>>>(s->d_sc, s->d_tally32 + s->J * GP, 1);
  }
  if (v2)
    k_finalize<G, GP, float><<<nb, 256, 0, s->stream>>>(s->J, s->d_mat, s->d_qt, s->d_tally32, s->d_vol, s->d_phi,
                                                        s->d_fnew, s->d_part_b, s->d_sc);
  else
    k_finalize<G, GP, double><<<nb, 256, 0, s->stream>>>(s->J, s->d_mat, s->d_qt, s->d_tally, s->d_vol, s->d_phi,
                                                         s->d_fnew, s->d_part_b, s->d_sc);
  k_keff<<<1, 1024, 0, s->stream>>>(s->d_part_a, s->d_part_b, nb, s->d_sc);
  k_normalize<G, GP><<<nb, 256, 0, s->stream>>>(s->J, s->d_phi, s->d_fnew, s->d_fold, s->d_sc, s->d_part_c);
  k_resid<<<1, 1024, 0, s->stream>>>(s->d_part_c, nb, s->d_sc, s->d_hist, s->hist_cap);
  s->cur = 1 - s->cur;
  CUDA_OK(cudaGetLastError());
}

// A8 between the halves: sum all-reduce of the fp32 tally (+ the leakage in
// its tail) and the grouped point-to-point exchange of cut-crossing boundary psi, on the
// solver's stream (NCCL), or through the caller's host callback.
void exchange(moc_solver* s) {
  if (s->comm.world <= 1 && !s->nccl) return;  // (a 1-rank NCCL communicator is a self-test)
  if (s->nccl) {
    NcclApi& n = nccl_api();
    const int GP = s->GP;
    NCCL_OK(n.groupStart());
    NCCL_OK(n.allReduce(s->d_tally32, s->d_tally32, (size_t)s->J * GP + 1, ncclFloat32, ncclSum, s->nccl,
                        s->stream));
    int64_t so = 0, ro = 0;
    for (int p = 0; p < (int)s->send_counts.size(); ++p) {
      if (s->send_counts[p])
        NCCL_OK(n.send(s->d_halo_send + so * GP, (size_t)(s->send_counts[p] * GP), ncclFloat32, p, s->nccl,
                       s->stream));
      if (s->recv_counts[p])
        NCCL_OK(n.recv(s->d_halo_recv + ro * GP, (size_t)(s->recv_counts[p] * GP), ncclFloat32, p, s->nccl,
                       s->stream));
      so += s->send_counts[p];
      ro += s->recv_counts[p];
    }
    NCCL_OK(n.groupEnd());
  } else if (s->xfn) {
    CUDA_OK(cudaStreamSynchronize(s->stream));
    if (s->xfn(s->xctx) != 0) throw Error(MOC_E_NCCL, "exchange callback failed");
  } else {
    throw Error(MOC_E_STATE, "world > 1 needs backend MOC_COMM_NCCL, an exchange callback, or "
                             "moc_iteration_sweep/finish driven by the caller");
  }
}

template <int G, int GP>
void run_iteration(moc_solver* s, bool time_it) {
  iter_sweep_half<G, GP>(s, time_it);
  exchange(s);
  iter_finish_half<G, GP>(s);
}

template <int G, int GP>
void run_sweep_half(moc_solver* s, bool time_it) {
  iter_sweep_half<G, GP>(s, time_it);
}

template <int G, int GP>
void run_finish_half(moc_solver* s, bool) {
  iter_finish_half<G, GP>(s);
}

typedef void (*iter_fn)(moc_solver*, bool);
#define PICK(FN)                      \
  switch (G) {                           \
    case 1: return FN<1, 1>;             \
    case 2: return FN<2, 2>;             \
    case 3: return FN<3, 4>;             \
    case 4: return FN<4, 4>;             \
    case 5: return FN<5, 8>;             \
    case 6: return FN<6, 8>;             \
    case 7: return FN<7, 8>;             \
    default: return FN<8, 8>;            \
  }
iter_fn pick_sweep_half(int G) { PICK(run_sweep_half) }
iter_fn pick_finish_half(int G) { PICK(run_finish_half) }
#undef PICK
iter_fn pick_iter(int G) {
  switch (G) {
    case 1: return run_iteration<1, 1>;
    case 2: return run_iteration<2, 2>;
    case 3: return run_iteration<3, 4>;
    case 4: return run_iteration<4, 4>;
    case 5: return run_iteration<5, 8>;
    case 6: return run_iteration<6, 8>;
    case 7: return run_iteration<7, 8>;
    default: return run_iteration<8, 8>;
  }
}

// schedule 3 (sweep_sc.cuh): shared memory per CTA = the warps' psi bands + cell staging,
// for 3, 4 and 5 CTAs per SM (the checksum variant: 3 CTAs, + hash state per member)
template <int G, int GP, int MINB>
void sc_smem_configure_one(moc_solver* s, int g, int nsm) {
  cudaFuncAttributes fa{};
  CUDA_OK(cudaFuncGetAttributes(&fa, k_sweep_sc<G, GP, false, MINB>));
  const size_t planes = sc_stage_smem(MINB) ? 0 : 2 * sizeof(double) * (size_t)sc_plane_stride(s->NL);
  const size_t per_cta = (228 * 1024) / MINB - 1024 - fa.sharedSizeBytes;
  constexpr int NH = ScH<G>::NH;
  const size_t stage = sc_stage_smem(MINB) ? sc_stage_bytes<G>() : 0;
  int pcap = (int)((per_cta - planes - stage) / ((size_t)kScWarps * NH * 16));
  if (s->opts.sc_psi_cap > 0) pcap = std::min(pcap, s->opts.sc_psi_cap);
  pcap = std::max(32, pcap & ~31);
  auto& q = s->sc_grp[g];
  q.pcap = pcap;
  q.smem = planes + (size_t)kScWarps * NH * pcap * 16 + stage;
  CUDA_OK(cudaFuncSetAttribute(k_sweep_sc<G, GP, false, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)q.smem));
  int per_sm = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_sc<G, GP, false, MINB>, kScThreads, q.smem));
  if (per_sm < 1) throw Error(MOC_E_CAPACITY, "stack-collective sweep does not fit on an SM");
  q.blocks = nsm * per_sm;
}

template <int G, int GP>
void sc_smem_configure(moc_solver* s) {
  int dev = 0, nsm = 0;
  CUDA_OK(cudaGetDevice(&dev));
  CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  sc_smem_configure_one<G, GP, 3>(s, 0, nsm);
  sc_smem_configure_one<G, GP, 4>(s, 1, nsm);
  sc_smem_configure_one<G, GP, 5>(s, 2, nsm);
  s->sc_smem_hash = s->sc_grp[0].smem + (size_t)kScWarps * s->sc_grp[0].pcap * 12;
  CUDA_OK(cudaFuncSetAttribute(k_sweep_sc<G, GP, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)s->sc_smem_hash));
  int per_sm_h = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_h, k_sweep_sc<G, GP, true, 3>, kScThreads,
                                                        s->sc_smem_hash));
  if (per_sm_h < 1) throw Error(MOC_E_CAPACITY, "stack-collective sweep does not fit on an SM");
  s->sc_blocks_hash = nsm * per_sm_h;
}

void sc_smem_configure_any(moc_solver* s) {
  switch (s->G) {
    case 1: return sc_smem_configure<1, 1>(s);
    case 2: return sc_smem_configure<2, 2>(s);
    case 3: return sc_smem_configure<3, 4>(s);
    case 4: return sc_smem_configure<4, 4>(s);
    case 5: return sc_smem_configure<5, 8>(s);
    case 6: return sc_smem_configure<6, 8>(s);
    case 7: return sc_smem_configure<7, 8>(s);
    default: return sc_smem_configure<8, 8>(s);
  }
}

// Work units of the stack-collective sweep: bands of B consecutive members of one stack,
// with R = 2^lgR lanes per cell.  A band's members in one column span
// (B - 1) dz + rho_max in z (rho_max = widest 2D segment of t x |cot|), so it touches at
// most floor(((B - 1) dz + rho_max) / h_min) + 2 layers: B is the largest band whose
// cells fit C = 32 / R lanes' cells and whose psi fits the warp's share of shared memory;
// R is the smallest for which a band fits at all (R = 1 unless a 2D segment rises through
// more than 30 layers).  Each stack goes to the occupancy group with the most CTAs per SM
// (3, 4, 5: more warps to hide latency, smaller psi bands) whose band capacity does not cut
// it into more bands than 3 CTAs per SM do (opts.sc_ctas_per_sm forces one group).  Within
// a group units are sorted by exact segment count, descending.
void sc_configure(moc_solver* s, const Geometry& g, const Laydown& L, const std::vector<int32_t>& owner) {
  int64_t& Bytes = s->dev_bytes;
  cudaStream_t st = s->stream;
  sc_smem_configure_any(s);
  double hmin = 1e300;
  for (int l = 0; l < g.NL; ++l) hmin = std::min(hmin, g.planes[l + 1] - g.planes[l]);
  s->hmin = hmin;
  if (g.NL + 1 > kMaxPlanes) throw Error(MOC_E_CAPACITY, "more than 255 axial layers");
  std::vector<ScUnit> ug[3];
  const int fctas = s->opts.sc_ctas_per_sm;
  if (fctas != 0 && (fctas < 3 || fctas > 5)) throw Error(MOC_E_PARAM, "sc_ctas_per_sm must be 0, 3, 4 or 5");
  const int forced = s->opts.sc_lanes_per_cell;
  if (forced != 0 && forced != 1 && forced != 2 && forced != 4 && forced != 8)
    throw Error(MOC_E_PARAM, "sc_lanes_per_cell must be 0, 1, 2, 4 or 8");
  for (int64_t q = 0; q < s->S; ++q) {
    if (!owner.empty() && owner[q] != s->comm.rank) continue;
    const int64_t cnt = L.st_cnt[q];
    if (cnt == 0) continue;
    const int64_t t = q / L.N, n = q % L.N;
    const int64_t an = (int64_t)L.t_a[t] * L.N + n;
    double wmax = 0, prev = 0;
    for (int64_t k = L.t_seg[t]; k < L.t_seg[t + 1]; ++k) {
      wmax = std::max(wmax, L.seg_send[k] - prev);
      prev = L.seg_send[k];
    }
    const double D = L.an_dz[an], rho = wmax * std::fabs(L.an_cot[an]);
    int lgR = -1;
    int64_t Bmax = 0;
    for (int lg = 0; lg <= 3; ++lg) {
      if (forced > 0 && (1 << lg) != forced) continue;
      const int C = 32 >> lg;
      const double room = (C - 2) * hmin - rho;
      if (room < 0) continue;
      // fewest lanes per cell whose band fits: every lane then sweeps all members of its
      // cell (per-cell setup amortised over the most members)
      lgR = lg;
      Bmax = (int64_t)std::floor(room / D) + 1;
      break;
    }
    if (lgR < 0 || Bmax < 1)
      throw Error(MOC_E_CAPACITY, "stack-collective sweep: a 2D segment rises through more layers than a warp has cells");
    auto bands = [&](int g) {
      const int64_t B = std::min<int64_t>(Bmax, s->sc_grp[g].pcap);
      return (cnt + B - 1) / B;
    };
    int gsel = 0;
    if (fctas) gsel = fctas - 3;
    else
      for (int g2 = 2; g2 > 0; --g2)
        if (bands(g2) == bands(0)) {
          gsel = g2;
          break;
        }
    const int64_t Bsel = std::min<int64_t>(Bmax, s->sc_grp[gsel].pcap);
    // 5 CTAs per SM: skewed shared-memory slots (sweep_sc.cuh ScCell::slot), one spare slot
    // every ~1/alpha members, so the member ranges of consecutive cells (P = h / dz apart)
    // start on different 16-byte bank groups even when P is close to a multiple of 8; alpha
    // aims at an odd slot distance and is capped by the band capacity
    uint32_t skew = 0;
    if (gsel == 2 && Bsel > 1) {
      const double Pm = hmin / D;
      double T = std::ceil(Pm);
      if (std::fmod(T, 2.0) == 0.0) T += 1.0;
      const int64_t pc = s->sc_grp[2].pcap;
      const double alpha = std::min(T / Pm - 1.0, (double)(pc - 1) / (double)(Bsel - 1) - 1.0);
      if (alpha > 0) skew = (uint32_t)std::min(65535.0, std::floor(alpha * 65536.0));
      while (skew && (Bsel - 1) + (int64_t)(((uint32_t)(Bsel - 1) * skew) >> 16) > pc - 1) --skew;
    }
    for (int64_t b0 = 0; b0 < cnt; b0 += Bsel)
      ug[gsel].push_back(ScUnit{(uint32_t)q, (uint32_t)b0, (uint32_t)std::min<int64_t>(Bsel, cnt - b0),
                                (uint32_t)lgR | (skew << 16)});
  }
  std::vector<ScUnit> units;
  for (int g2 = 0; g2 < 3; ++g2) {
    s->sc_grp[g2].first = (uint32_t)units.size();
    s->sc_grp[g2].n = (uint32_t)ug[g2].size();
    units.insert(units.end(), ug[g2].begin(), ug[g2].end());
  }
  s->n_sc_units = (uint32_t)units.size();
  s->d_sc_units = dmalloc<ScUnit>(units.size(), Bytes);
  upload(units.data(), s->d_sc_units, sizeof(ScUnit) * units.size(), st);
  uint32_t* keys = dmalloc<uint32_t>(units.size(), Bytes);
  k_sc_unit_cost<<<1024, 256, 0, st>>>(s->d_sc_units, s->n_sc_units, s->d_st_first, s->d_cost, keys);
  CUDA_OK(cudaGetLastError());
  auto pol = thrust::cuda::par.on(st);
  for (int g2 = 0; g2 < 3; ++g2) {
    const auto& q = s->sc_grp[g2];
    if (q.n > 1)
      thrust::stable_sort_by_key(pol, thrust::device_ptr<uint32_t>(keys) + q.first,
                                 thrust::device_ptr<uint32_t>(keys) + q.first + q.n,
                                 thrust::device_ptr<ScUnit>(s->d_sc_units) + q.first, thrust::greater<uint32_t>());
  }
  CUDA_OK(cudaStreamSynchronize(st));
  cudaFree(keys);
  Bytes -= 4 * (int64_t)units.size();
  s->d_counter = dmalloc<uint32_t>(4, Bytes);  // unit queues: one per occupancy group
  s->d_err = dmalloc<int>(1, Bytes);
  CUDA_OK(cudaMemsetAsync(s->d_err, 0, sizeof(int), st));
  s->d_tally32 = dmalloc<float>((size_t)s->J * s->GP + 8, Bytes);  // + tail for the leakage
}

void v2_configure_any(moc_solver* s) {
  switch (s->G) {
    case 1: return v2_configure<1, 1>(s);
    case 2: return v2_configure<2, 2>(s);
    case 3: return v2_configure<3, 4>(s);
    case 4: return v2_configure<4, 4>(s);
    case 5: return v2_configure<5, 8>(s);
    case 6: return v2_configure<6, 8>(s);
    case 7: return v2_configure<7, 8>(s);
    default: return v2_configure<8, 8>(s);
  }
}

int padded_groups(int G) { return G <= 2 ? G : (G <= 4 ? 4 : 8); }

void reset_state(moc_solver* s) {
  const int nb = 1024;
  k_fill_f32<<<nb, 256, 0, s->stream>>>(s->d_phi, s->J * s->GP, 1.0f);
  CUDA_OK(cudaMemsetAsync(s->d_psi[0], 0, sizeof(float) * s->psi_slots * s->GP, s->stream));
  if (s->d_psi[1] != s->d_psi[0])
    CUDA_OK(cudaMemsetAsync(s->d_psi[1], 0, sizeof(float) * s->psi_slots * s->GP, s->stream));
  double sc[SC_N] = {0};
  sc[SC_K] = 1.0;
  sc[SC_PSI_SCALE] = 1.0;
  CUDA_OK(cudaMemcpyAsync(s->d_sc, sc, sizeof(sc), cudaMemcpyHostToDevice, s->stream));
  CUDA_OK(cudaStreamSynchronize(s->stream));
  s->cur = 0;
}

void destroy(moc_solver* s) {
  if (!s) return;
  if (s->d_psi[1] == s->d_psi[0]) s->d_psi[1] = nullptr;  // Gauss-Seidel: one buffer
  void* ptrs[] = {s->d_seg_send, s->d_planes, s->d_t_len, s->d_seg_region, s->d_t_seg, s->d_t_a, s->d_an_cot,
                  s->d_an_tan, s->d_an_invsin, s->d_an_dz, s->d_an_vw, s->d_an_c, s->d_st_z0, s->d_st_first,
                  s->d_link, s->d_work, s->d_cost, s->d_mat, s->d_qt, s->d_phi, s->d_fold, s->d_fnew, s->d_tally,
                  s->d_vol, s->d_psi[0], s->d_psi[1], s->d_sc, s->d_part_a, s->d_part_b, s->d_part_c, s->d_hist,
                  s->d_units, s->d_counter, s->d_rmax, s->d_qmax_t, s->d_tally32, s->d_err,
                  s->d_unit_maxq, s->d_unit_exp, s->d_store, s->d_phi64, s->d_sc_units,
                  s->d_send_slots, s->d_recv_slots, s->d_halo_send, s->d_halo_recv, s->d_slot_first};
  if (s->qtex) cudaDestroyTextureObject(s->qtex);
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& e : s->ev)
    if (e) cudaEventDestroy(e);
  if (s->h_xs) cudaFreeHost(s->h_xs);
  if (s->h_planes) cudaFreeHost(s->h_planes);
  for (auto& g : s->gexec)
    if (g) cudaGraphExecDestroy(g);
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->nccl) nccl_api().commDestroy(s->nccl);
  if (const_owner(s->device) == s->uid) const_owner(s->device) = 0;
}

// One power iteration: a replay of the captured graph of this Jacobi parity (captured on
// first use: source, sweep, exchange, finalize, k, normalisation, residual), or direct
// launches when graphs are off or the exchange needs the host.
void iterate_once(moc_solver* s, iter_fn f, bool time_it) {
  const bool graph = !s->opts.no_graph && (s->comm.world <= 1 || s->nccl);
  if (!graph) {
    f(s, time_it);
    return;
  }
  ensure_constants(s);  // outside the capture: the graph reads the constant bank as it is
  const int c = s->cur;
  if (!s->gexec[c]) {
    // captured on a private non-blocking stream (the caller's may be the legacy default
    // stream, which cannot be captured), replayed on the caller's stream
    if (!s->cap_stream) CUDA_OK(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = s->stream;
    cudaGraph_t g = nullptr;
    CUDA_OK(cudaStreamSynchronize(user));
    s->stream = s->cap_stream;
    try {
      CUDA_OK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      try {
        f(s, true);  // sweep timed by event-record nodes in every replay
      } catch (...) {
        cudaStreamEndCapture(s->stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CUDA_OK(cudaStreamEndCapture(s->stream, &g));
    } catch (...) {
      s->stream = user;
      s->cur = c;
      (void)cudaGetLastError();
      throw;
    }
    s->stream = user;
    s->cur = c;  // capture recorded the launches without running them
    const cudaError_t e = cudaGraphInstantiate(&s->gexec[c], g, 0);
    cudaGraphDestroy(g);
    CUDA_OK(e);
  }
  CUDA_OK(cudaGraphLaunch(s->gexec[c], s->stream));
  s->sweep_timed = true;
  s->cur = 1 - c;
}

}  // namespace

#define SOLVER_TRY(s, ...)                     \
  try {                                        \
    __VA_ARGS__;                               \
    return MOC_OK;                             \
  } catch (const Error& e) {                   \
    if (s) (s)->err = e.what();                \
    return e.code;                             \
  } catch (const std::exception& e) {          \
    if (s) (s)->err = e.what();                \
    return MOC_E_INVALID_ARG;                  \
  }

extern "C" {

const char* moc_solver_last_error(const moc_solver* s) { return s ? s->err.c_str() : "NULL solver"; }

int moc_solver_create(moc_solver** out, moc_problem* p, int device, void* cuda_stream, const moc_comm_desc* comm,
                      const moc_solver_opts* opts) {
  if (!out || !p) return MOC_E_INVALID_ARG;
  *out = nullptr;
  const Geometry& g = p->impl.geo;
  const Laydown& L = p->impl.lay;
  const Materials& mt = p->impl.mat;
  if (!g.set || !mt.set || !L.done) {
    p->impl.err = "solver needs materials, geometry and generated tracks";
    return MOC_E_STATE;
  }
  moc_solver* s = new moc_solver();
  auto t0 = std::chrono::steady_clock::now();
  try {
    if (mt.n_mat > kMaxMat) throw Error(MOC_E_PARAM, "at most 32 materials are supported");
    if (L.n3 >= (int64_t)0x7fffffff) throw Error(MOC_E_CAPACITY, "more than 2^31 3D tracks");
    for (size_t i = 0; i < g.material.size(); ++i)
      if (g.material[i] >= mt.n_mat) throw Error(MOC_E_REFERENCE, "unknown material index");
    if (opts) s->opts = *opts;
    else s->opts.schedule = MOC_SCHED_STACK_COLLECTIVE;  // the product sweep
    if (comm) s->comm = *comm;
    s->device = device;
    static std::atomic<uint64_t> next_uid{1};
    s->uid = next_uid++;
    CUDA_OK(cudaSetDevice(device));
    s->stream = (cudaStream_t)cuda_stream;
    s->G = mt.G;
    s->GP = padded_groups(mt.G);
    s->N = L.N;
    s->M = L.M;
    s->NL = g.NL;
    s->n_mat = mt.n_mat;
    s->J = g.n_fsr;
    s->T2 = L.T2();
    s->S = L.S();
    s->T3 = L.n3;
    s->N2 = (int64_t)L.seg_region.size();
    cudaStream_t st = s->stream;
    int64_t& B = s->dev_bytes;
    // --- laydown upload (A1/A2)
    s->d_seg_send = dmalloc<double>(s->N2, B);
    s->d_seg_region = dmalloc<uint32_t>(s->N2, B);
    s->d_planes = dmalloc<double>(g.NL + 1, B);
    s->d_t_len = dmalloc<double>(s->T2, B);
    s->d_t_seg = dmalloc<int64_t>(s->T2 + 1, B);
    s->d_t_a = dmalloc<int32_t>(s->T2, B);
    const size_t AN = L.an_cot.size();
    s->d_an_cot = dmalloc<double>(AN, B);
    s->d_an_tan = dmalloc<double>(AN, B);
    s->d_an_invsin = dmalloc<double>(AN, B);
    s->d_an_dz = dmalloc<double>(AN, B);
    s->d_an_vw = dmalloc<double>(AN, B);
    s->d_an_c = dmalloc<float>(AN, B);
    s->d_st_z0 = dmalloc<double>(s->S, B);
    s->d_st_first = dmalloc<uint32_t>(s->S + 1, B);
    upload(L.seg_send.data(), s->d_seg_send, 8 * s->N2, st);
    upload(L.seg_region.data(), s->d_seg_region, 4 * s->N2, st);
    upload(g.planes.data(), s->d_planes, 8 * (g.NL + 1), st);
    if (g.NL + 1 <= 256) {
      CUDA_OK(cudaMallocHost(&s->h_planes, sizeof(double) * (g.NL + 1)));
      std::memcpy(s->h_planes, g.planes.data(), sizeof(double) * (g.NL + 1));
    }
    upload(L.t_len.data(), s->d_t_len, 8 * s->T2, st);
    upload(L.t_seg.data(), s->d_t_seg, 8 * (s->T2 + 1), st);
    upload(L.t_a.data(), s->d_t_a, 4 * s->T2, st);
    upload(L.an_cot.data(), s->d_an_cot, 8 * AN, st);
    upload(L.an_tan.data(), s->d_an_tan, 8 * AN, st);
    upload(L.an_invsin.data(), s->d_an_invsin, 8 * AN, st);
    upload(L.an_dz.data(), s->d_an_dz, 8 * AN, st);
    std::vector<double> vw(AN);
    std::vector<float> cw(AN);
    for (size_t u = 0; u < AN; ++u) {
      vw[u] = L.an_w[u] / (2.0 * 3.14159265358979323846) * L.an_aperp[u];  // App. A.5
      cw[u] = (float)(L.an_w[u] * L.an_aperp[u]);
    }
    upload(vw.data(), s->d_an_vw, 8 * AN, st);
    upload(cw.data(), s->d_an_c, 4 * AN, st);
    upload(L.st_z0.data(), s->d_st_z0, 8 * s->S, st);
    std::vector<uint32_t> sf(s->S + 1);
    for (int64_t q = 0; q <= s->S; ++q) sf[q] = (uint32_t)L.st_first[q];
    upload(sf.data(), s->d_st_first, 4 * (s->S + 1), st);
    // --- 3D links (A6)
    std::vector<int32_t> owner;  // stack -> rank (multi-GPU)
    {
      std::vector<int64_t> lk(2 * s->T3);
      links3d(g, L, lk.data());
      s->T3_local = s->T3;
      s->psi_slots = 2 * s->T3;
      if (s->comm.world <= 1) {
        std::vector<uint32_t> l32(2 * s->T3);
        for (int64_t q = 0; q < 2 * s->T3; ++q) l32[q] = lk[q] < 0 ? 0xffffffffu : (uint32_t)lk[q];
        s->d_link = dmalloc<uint32_t>(2 * s->T3, B);
        upload(l32.data(), s->d_link, 4 * 2 * s->T3, st);
        CUDA_OK(cudaStreamSynchronize(st));
        if (s->comm.backend == MOC_COMM_NCCL) {  // 1-rank communicator: exercises the NCCL path
          ncclUniqueId id;
          std::memcpy(&id, s->comm.nccl_id, sizeof(id));
          NCCL_OK(nccl_api().commInitRank(&s->nccl, 1, id, 0));
        }
      } else {
        if (s->opts.schedule != 0 && s->opts.schedule != 3)
          throw Error(MOC_E_PARAM, "multi-GPU runs use schedule 0 or 3");
        if (s->comm.rank < 0 || s->comm.rank >= s->comm.world) throw Error(MOC_E_INVALID_ARG, "bad rank");
        std::vector<double> cost;
        partition_stacks(L, s->comm.world, owner, &cost);
        s->owned_cost = cost[s->comm.rank];
        const int W = s->comm.world;
        RankLayout rl;
        rank_layout(L, lk.data(), owner, s->comm.rank, W, rl);
        s->T3_local = rl.T3_local;
        s->n_send = rl.n_send;
        s->psi_slots = 2 * s->T3_local + s->n_send;
        s->send_counts = rl.send_counts;
        s->recv_counts = rl.recv_counts;
        std::vector<uint32_t> l32(rl.link.size());
        for (size_t q = 0; q < l32.size(); ++q) l32[q] = rl.link[q] < 0 ? 0xffffffffu : (uint32_t)rl.link[q];
        s->d_link = dmalloc<uint32_t>(l32.size(), B);
        upload(l32.data(), s->d_link, 4 * l32.size(), st);
        std::vector<uint32_t> sf32(s->S + 1);
        for (int64_t q = 0; q <= s->S; ++q) sf32[q] = (uint32_t)rl.slot_first[q];
        s->d_slot_first = dmalloc<uint32_t>(s->S + 1, B);
        upload(sf32.data(), s->d_slot_first, 4 * (s->S + 1), st);
        // halo: the send buffer is gathered from the tail; received psi scatter to local slots
        std::vector<uint32_t> ss(s->n_send), rr(rl.recv_slots.size());
        for (int64_t x = 0; x < s->n_send; ++x) ss[x] = (uint32_t)(2 * s->T3_local + x);
        for (size_t x = 0; x < rr.size(); ++x) rr[x] = (uint32_t)rl.recv_slots[x];
        s->n_recv = (int64_t)rr.size();
        s->d_send_slots = dmalloc<uint32_t>(ss.size(), B);
        s->d_recv_slots = dmalloc<uint32_t>(rr.size(), B);
        upload(ss.data(), s->d_send_slots, 4 * ss.size(), st);
        upload(rr.data(), s->d_recv_slots, 4 * rr.size(), st);
        s->d_halo_send = dmalloc<float>(ss.size() * s->GP, B);
        s->d_halo_recv = dmalloc<float>(rr.size() * s->GP, B);
        CUDA_OK(cudaStreamSynchronize(st));
        if (s->comm.backend == MOC_COMM_NCCL) {
          static_assert(sizeof(ncclUniqueId) == sizeof(s->comm.nccl_id), "ncclUniqueId size");
          ncclUniqueId id;
          std::memcpy(&id, s->comm.nccl_id, sizeof(id));
          NCCL_OK(nccl_api().commInitRank(&s->nccl, s->comm.world, id, s->comm.rank));
        } else if (s->comm.backend != MOC_COMM_CALLER) {
          throw Error(MOC_E_INVALID_ARG, "unknown comm backend");
        }
      }
      CUDA_OK(cudaStreamSynchronize(st));
    }
    // --- FSR arrays and materials
    s->vol_analytic.resize(s->J);
    g.analytic_volumes(s->vol_analytic.data());
    s->mat_host.resize(s->J);
    std::vector<uint8_t> m8(s->J);
    for (int64_t j = 0; j < s->J; ++j) {
      s->mat_host[j] = g.mat_of_fsr(j);
      m8[j] = (uint8_t)s->mat_host[j];
    }
    s->d_mat = dmalloc<uint8_t>(s->J, B);
    upload(m8.data(), s->d_mat, s->J, st);
    const size_t JG = (size_t)s->J * s->GP;
    s->d_qt = dmalloc<float>(JG, B);
    if (s->GP == 8) {
      if (JG / 4 >= ((size_t)1 << 27)) throw Error(MOC_E_CAPACITY, "more than 2^26 FSRs at 5-8 groups (source texture)");
      cudaResourceDesc rd{};
      rd.resType = cudaResourceTypeLinear;
      rd.res.linear.devPtr = s->d_qt;
      rd.res.linear.desc = cudaCreateChannelDesc<float4>();
      rd.res.linear.sizeInBytes = sizeof(float) * (size_t)JG;
      cudaTextureDesc td{};
      td.readMode = cudaReadModeElementType;
      CUDA_OK(cudaCreateTextureObject(&s->qtex, &rd, &td, nullptr));
    }
    s->d_phi = dmalloc<float>(JG, B);
    s->d_tally = dmalloc<double>(JG, B);
    s->d_vol = dmalloc<double>(s->J, B);
    s->d_fold = dmalloc<float>(s->J, B);
    s->d_fnew = dmalloc<float>(s->J, B);
    s->nb_fsr = (int)std::min<int64_t>(1184, (s->J + 255) / 256);
    s->d_part_a = dmalloc<double>(s->nb_fsr, B);
    s->d_part_b = dmalloc<double>(s->nb_fsr, B);
    s->d_part_c = dmalloc<double>(2 * s->nb_fsr, B);
    s->d_sc = dmalloc<double>(SC_N, B);
    s->d_hist = dmalloc<double>(2 * (size_t)s->hist_cap, B);
    upload_materials(s, mt.sigma_t.data(), mt.sigma_s.data(), mt.nu_sigma_f.data(), mt.chi.data());
    // --- device view
    DevData& d = s->dd;
    d.seg_send = s->d_seg_send;
    d.seg_region = s->d_seg_region;
    d.planes = s->d_planes;
    d.NL = g.NL;
    d.Z = g.Z;
    d.t_len = s->d_t_len;
    d.t_seg = s->d_t_seg;
    d.t_a = s->d_t_a;
    d.an_cot = s->d_an_cot;
    d.an_tan = s->d_an_tan;
    d.an_invsin = s->d_an_invsin;
    d.an_dz = s->d_an_dz;
    d.an_c = s->d_an_c;
    d.an_vw = s->d_an_vw;
    d.st_z0 = s->d_st_z0;
    d.st_first = s->d_st_first;
    d.S = (int32_t)s->S;
    d.N = s->N;
    d.T3 = (uint32_t)s->T3;
    // --- track volumes and exact per-track segment counts (device OTF walk)
    s->d_cost = dmalloc<uint32_t>(s->T3, B);
    unsigned long long* d_total = dmalloc<unsigned long long>(1, B);
    CUDA_OK(cudaMemsetAsync(s->d_vol, 0, 8 * s->J, st));
    CUDA_OK(cudaMemsetAsync(d_total, 0, 8, st));
    k_volumes_costs<<<148 * 8, 256, 0, st>>>(d, s->d_vol, s->d_cost, d_total);
    CUDA_OK(cudaGetLastError());
    unsigned long long tot = 0;
    CUDA_OK(cudaMemcpyAsync(&tot, d_total, 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    cudaFree(d_total);
    s->nseg3 = (int64_t)tot;
    // --- work list (schedule)
    auto pol = thrust::cuda::par.on(st);
    int sched = s->opts.schedule;
    if (sched < 0 || sched > 3) throw Error(MOC_E_INVALID_ARG, "schedule must be 0, 1, 2 or 3");
    if (s->opts.exp_mode != 0 && sched != 0) throw Error(MOC_E_PARAM, "exp_mode (EXP preload, §4.2) needs schedule 0");
    if (sched == 0) {
      // persistent stack-band units (sweep_v2.cuh), sorted by exact segment count descending
      int64_t max_nk = 0;
      for (int64_t t = 0; t < s->T2; ++t) max_nk = std::max(max_nk, L.t_seg[t + 1] - L.t_seg[t]);
      if (max_nk > kMaxK) throw Error(MOC_E_CAPACITY, "2D track with more than 512 segments");
      if (g.NL + 1 > kMaxPlanes) throw Error(MOC_E_CAPACITY, "more than 255 axial layers");
      v2_configure_any(s);  // dynamic shared memory from the kernel's static footprint
      // the tile left below the largest unit's tables must hold two full layer columns
      s->cap_cells = (int)std::min<int64_t>(
          cap_max_cells(s->G, s->GP),
          (((int64_t)s->v2_smem - unit_table_bytes((int)max_nk)) / cell_bytes(s->G, s->GP)) & ~7);
      s->tile_off = (unit_table_bytes((int)max_nk) + 15) & ~15;
      if (s->cap_cells < 2 * g.NL) throw Error(MOC_E_CAPACITY, "axial mesh too fine for the tally tile");
      if (s->opts.tile_cells > 0) {
        if (s->opts.tile_cells < g.NL) throw Error(MOC_E_PARAM, "tile_cells must be >= the number of axial layers");
        s->cap_cells = std::min(s->cap_cells, (s->opts.tile_cells + 7) & ~7);
      }
      {
        double hmin = 1e300;
        for (int l = 0; l < g.NL; ++l) hmin = std::min(hmin, g.planes[l + 1] - g.planes[l]);
        s->h_lane = hmin / 3.0;
        const int v = s->opts.v2_lane_stride;
        if (v != 0 && v != 1 && v != 2 && v != 4 && v != 8) throw Error(MOC_E_PARAM, "v2_lane_stride must be 0, 1, 2, 4 or 8");
        if (v > 0) s->lane_lg = v == 8 ? 3 : v == 4 ? 2 : v == 2 ? 1 : 0;
      }
      std::vector<Unit> units;
      for (int64_t q = 0; q < s->S; ++q) {
        if (!owner.empty() && owner[q] != s->comm.rank) continue;
        const int64_t cnt = L.st_cnt[q];
        for (int64_t b0 = 0; b0 < cnt; b0 += kV2Threads)
          units.push_back(Unit{(uint32_t)q, (uint32_t)b0, (uint32_t)std::min<int64_t>(kV2Threads, cnt - b0), 1u});
      }
      s->n_units = (uint32_t)units.size();
      s->d_units = dmalloc<Unit>(units.size(), B);
      upload(units.data(), s->d_units, sizeof(Unit) * units.size(), st);
      uint32_t* keys = dmalloc<uint32_t>(units.size(), B);
      s->d_unit_maxq = dmalloc<uint32_t>(units.size(), B);
      k_unit_cost<<<1024, 256, 0, st>>>(s->d_units, s->n_units, s->d_st_first, s->d_cost, keys, s->d_unit_maxq);
      CUDA_OK(cudaGetLastError());
      thrust::stable_sort_by_key(pol, thrust::device_ptr<uint32_t>(keys), thrust::device_ptr<uint32_t>(keys) + units.size(),
                                 thrust::device_ptr<Unit>(s->d_units), thrust::greater<uint32_t>());
      // per-unit segment totals and longest track, in the sorted order
      k_unit_cost<<<1024, 256, 0, st>>>(s->d_units, s->n_units, s->d_st_first, s->d_cost, keys, s->d_unit_maxq);
      CUDA_OK(cudaGetLastError());
      std::vector<uint32_t> ukey(units.size()), umax(units.size());
      CUDA_OK(cudaMemcpyAsync(ukey.data(), keys, 4 * units.size(), cudaMemcpyDeviceToHost, st));
      CUDA_OK(cudaMemcpyAsync(umax.data(), s->d_unit_maxq, 4 * units.size(), cudaMemcpyDeviceToHost, st));
      CUDA_OK(cudaStreamSynchronize(st));
      cudaFree(keys);
      if (s->opts.exp_mode == 1) {
        // §4.2: units in descending segment count, cumulated until the threshold
        size_t freeb = 0, totalb = 0;
        CUDA_OK(cudaMemGetInfo(&freeb, &totalb));
        // leave room for the boundary-psi double buffer allocated below
        const double psi_bytes = 2.0 * (double)s->psi_slots * s->GP * sizeof(float);
        double budget = s->opts.exp_budget_mb > 0 ? s->opts.exp_budget_mb * 1048576.0 : (double)freeb - psi_bytes;
        const double frac = s->opts.exp_fraction > 0 ? s->opts.exp_fraction : 0.8;
        const double lim = budget * frac;
        std::vector<uint64_t> off(units.size(), kNoExp);
        uint64_t cum = 0;
        for (size_t u = 0; u < units.size(); ++u) {
          const uint64_t recs = (uint64_t)umax[u] * kV2Threads;
          if ((double)(cum + recs) * sizeof(Rec) > lim) break;
          off[u] = cum;
          cum += recs;
          s->exp_units += 1;
          s->exp_segments += ukey[u];
        }
        if (s->exp_units > 0) {
          s->exp_bytes = (int64_t)(cum * sizeof(Rec));
          s->d_store = dmalloc<Rec>(cum, B);
          s->d_unit_exp = dmalloc<uint64_t>(units.size(), B);
          upload(off.data(), s->d_unit_exp, 8 * off.size(), st);
          k_exp_generate<<<4096, kV2Threads, 0, st>>>(d, s->d_units, s->d_unit_exp, s->n_units, s->d_mat, s->d_store, s->h_lane, s->lane_lg);
          CUDA_OK(cudaGetLastError());
          CUDA_OK(cudaStreamSynchronize(st));
        }
      }
      s->d_counter = dmalloc<uint32_t>(2, B);  // OTF and EXP unit queues
      s->d_err = dmalloc<int>(1, B);
      CUDA_OK(cudaMemsetAsync(s->d_err, 0, sizeof(int), st));
      s->d_rmax = dmalloc<float>((size_t)g.n_regions * s->GP, B);
      s->d_qmax_t = dmalloc<float>((size_t)s->T2 * s->GP, B);
      s->d_tally32 = dmalloc<float>((size_t)s->J * s->GP + 8, B);  // + tail for the leakage
    } else if (sched == 3) {
      sc_configure(s, g, L, owner);
    } else {
      s->d_work = dmalloc<uint32_t>(s->T3, B);
      s->nwork = (uint32_t)s->T3;
      thrust::sequence(pol, thrust::device_ptr<uint32_t>(s->d_work), thrust::device_ptr<uint32_t>(s->d_work) + s->T3);
    }
    if (sched == 2) {
      // §4.3: sort by segment count descending, then the serpentine reversal
      uint32_t* keys = dmalloc<uint32_t>(s->T3, B);
      CUDA_OK(cudaMemcpyAsync(keys, s->d_cost, 4 * s->T3, cudaMemcpyDeviceToDevice, st));
      thrust::stable_sort_by_key(pol, thrust::device_ptr<uint32_t>(keys), thrust::device_ptr<uint32_t>(keys) + s->T3,
                                 thrust::device_ptr<uint32_t>(s->d_work), thrust::greater<uint32_t>());
      cudaFree(keys);
      B -= 4 * s->T3;
      int th = s->opts.threads > 0 ? s->opts.threads : 512;
      int bl = s->opts.blocks > 0 ? s->opts.blocks : 512;
      if (sched == 2) {
        k_serpentine<<<1024, 256, 0, st>>>(s->d_work, (uint64_t)s->T3, (uint64_t)th * bl);
        CUDA_OK(cudaGetLastError());
      }
    }
    if (sched == 1 || sched == 2) {
      s->sweep_threads = s->opts.threads > 0 ? s->opts.threads : 512;  // P:146 default 512 x 512
      s->sweep_blocks = s->opts.blocks > 0 ? s->opts.blocks : 512;
    }
    // --- state
    if (s->opts.gauss_seidel) {
      if (sched != 3 || !(s->GP == 8 && s->G < 8))
        throw Error(MOC_E_PARAM, "gauss_seidel needs schedule 3 and 5-7 groups (the slot pad word holds the epoch)");
      if (s->comm.world > 1) throw Error(MOC_E_PARAM, "gauss_seidel is single-GPU");
    }
    // boundary psi of this rank's tracks (+ the halo-send tail); Jacobi: double buffer,
    // Gauss-Seidel (NEXT-4): one buffer updated in place
    s->d_psi[0] = dmalloc<float>((size_t)s->psi_slots * s->GP, B);
    s->d_psi[1] = s->opts.gauss_seidel ? s->d_psi[0] : dmalloc<float>((size_t)s->psi_slots * s->GP, B);
    for (auto& e : s->ev) CUDA_OK(cudaEventCreate(&e));
    reset_state(s);
  } catch (const Error& e) {
    p->impl.err = e.what();
    int code = e.code;
    destroy(s);
    delete s;
    return code;
  }
  s->setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = s;
  return MOC_OK;
}

int moc_solver_destroy(moc_solver* s) {
  destroy(s);
  delete s;
  return MOC_OK;
}

int moc_reset(moc_solver* s) {
  if (!s) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    reset_state(s);
  })
}

static void read_scalars(moc_solver* s, double* sc) {
  CUDA_OK(cudaMemcpyAsync(sc, s->d_sc, sizeof(double) * SC_N, cudaMemcpyDeviceToHost, s->stream));
  CUDA_OK(cudaStreamSynchronize(s->stream));
}

static void check_health(moc_solver* s, const double* sc) {
  if (s->d_err) {
    int e = 0;
    CUDA_OK(cudaMemcpy(&e, s->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (e) throw Error(MOC_E_CAPACITY, "sweep work unit exceeded its shared-memory tally tile");
  }
  if (sc[SC_BAD] > 0) throw Error(MOC_E_NUMERIC, "NaN or negative scalar flux after the sweep");
  if (!(sc[SC_K] > 0)) throw Error(MOC_E_EIGEN, "zero fission source (k <= 0)");
}

int moc_iterate(moc_solver* s, int32_t n_iter, double* k_out, double* residual_out) {
  if (!s || n_iter < 0) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    iter_fn f = pick_iter(s->G);
    for (int it = 0; it < n_iter; ++it) {
      bool last = it == n_iter - 1;
      if (last) CUDA_OK(cudaEventRecord(s->ev[2], s->stream));
      iterate_once(s, f, last);
      if (last) CUDA_OK(cudaEventRecord(s->ev[3], s->stream));
    }
    double sc[SC_N];
    read_scalars(s, sc);
    if (n_iter > 0) {
      float ms = 0;
      CUDA_OK(cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]));
      s->sweep_ms_last = ms;
      CUDA_OK(cudaEventElapsedTime(&ms, s->ev[2], s->ev[3]));
      s->iter_ms_last = ms;
    }
    check_health(s, sc);
    if (k_out) *k_out = sc[SC_K];
    if (residual_out) *residual_out = sc[SC_RESID];
  })
}

int moc_solve(moc_solver* s, const moc_solve_opts* o, moc_result* r) {
  if (!s || !o || !r) return MOC_E_INVALID_ARG;
  try {
    CUDA_OK(cudaSetDevice(s->device));
    iter_fn f = pick_iter(s->G);
    int every = o->check_every > 0 ? o->check_every : 10;
    int done = 0;
    r->converged = 0;
    while (done < o->max_iter) {
      int n = std::min(every, o->max_iter - done);
      for (int it = 0; it < n; ++it) iterate_once(s, f, false);
      done += n;
      double sc[SC_N];
      read_scalars(s, sc);
      check_health(s, sc);
      r->k = sc[SC_K];
      r->residual = sc[SC_RESID];
      r->iterations = (int32_t)sc[SC_ITER];
      // convergence on the latest iteration
      if (std::fabs(sc[SC_K] - sc[SC_KPREV]) < o->tol_k && sc[SC_RESID] < o->tol_src) {
        // find the first converged iteration inside the batch from the history
        std::vector<double> h(2 * (size_t)std::min(r->iterations, s->hist_cap));
        CUDA_OK(cudaMemcpy(h.data(), s->d_hist, 8 * h.size(), cudaMemcpyDeviceToHost));
        r->converged = 1;
        return MOC_OK;
      }
    }
    s->err = "max_iter reached without convergence";
    return MOC_E_NOCONV;
  } catch (const Error& e) {
    s->err = e.what();
    return e.code;
  }
}

int moc_solver_update_materials(moc_solver* s, const double* sigma_t, const double* sigma_s, const double* nu_sigma_f,
                                const double* chi) {
  if (!s || !sigma_t || !sigma_s || !nu_sigma_f || !chi) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    check_materials(s->n_mat, s->G, sigma_t, sigma_s, nu_sigma_f, chi);
    // the pinned staging buffer may still feed an earlier asynchronous constant upload
    CUDA_OK(cudaStreamSynchronize(s->stream));
    upload_materials(s, sigma_t, sigma_s, nu_sigma_f, chi);
  })
}

int moc_get_scalar_flux(moc_solver* s, double* phi) {
  if (!s || !phi) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    const size_t n = (size_t)s->J * s->G;
    if (!s->d_phi64) s->d_phi64 = dmalloc<double>(n, s->dev_bytes);
    k_phi_f64<<<s->nb_fsr, 256, 0, s->stream>>>(s->d_phi, s->J, s->G, s->GP, s->d_phi64);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(phi, s->d_phi64, 8 * n, cudaMemcpyDeviceToHost, s->stream));
    CUDA_OK(cudaStreamSynchronize(s->stream));
  })
}

int moc_get_fsr_volumes(moc_solver* s, double* vol_track, double* vol_analytic) {
  if (!s || (!vol_track && !vol_analytic)) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    if (vol_track) {
      CUDA_OK(cudaSetDevice(s->device));
      CUDA_OK(cudaMemcpyAsync(vol_track, s->d_vol, 8 * s->J, cudaMemcpyDeviceToHost, s->stream));
      CUDA_OK(cudaStreamSynchronize(s->stream));
    }
    if (vol_analytic) std::memcpy(vol_analytic, s->vol_analytic.data(), 8 * (size_t)s->J);
  })
}

int moc_get_history(moc_solver* s, double* k_hist, double* res_hist, int32_t cap, int32_t* n) {
  if (!s || !n) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    double sc[SC_N];
    read_scalars(s, sc);
    int it = std::min((int)sc[SC_ITER], s->hist_cap);
    std::vector<double> h(2 * (size_t)std::max(it, 1));
    CUDA_OK(cudaMemcpy(h.data(), s->d_hist, 8 * 2 * (size_t)it, cudaMemcpyDeviceToHost));
    int m = std::min(it, cap);
    for (int q = 0; q < m; ++q) {
      if (k_hist) k_hist[q] = h[2 * q];
      if (res_hist) res_hist[q] = h[2 * q + 1];
    }
    *n = it;
  })
}

int moc_get_balance(moc_solver* s, double* production, double* absorption, double* leakage) {
  if (!s) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    std::vector<double> phi((size_t)s->J * s->G), vol(s->J);
    int rc = moc_get_scalar_flux(s, phi.data());
    if (rc) throw Error(rc, s->err);
    rc = moc_get_fsr_volumes(s, vol.data(), nullptr);
    if (rc) throw Error(rc, s->err);
    double sc[SC_N];
    read_scalars(s, sc);
    double pr = 0, ab = 0;
    const int G = s->G;
    for (int64_t j = 0; j < s->J; ++j) {
      int m = s->mat_host[j];
      for (int g = 0; g < G; ++g) {
        double sa = s->sigma_t[(size_t)m * G + g];
        for (int h = 0; h < G; ++h) sa -= s->sigs[((size_t)m * G + g) * G + h];
        ab += vol[j] * sa * phi[(size_t)j * G + g];
        pr += vol[j] * s->nusf[(size_t)m * G + g] * phi[(size_t)j * G + g];
      }
    }
    if (production) *production = pr;
    if (absorption) *absorption = ab;
    if (leakage) *leakage = sc[SC_LEAK_SCALED];
  })
}

int moc_device_trace_checksums(moc_solver* s, int64_t first, int64_t n, int32_t* nseg, uint64_t* hash, double* suml) {
  if (!s || first < 0 || n < 0 || first + n > s->T3) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    if (n == 0) return MOC_OK;
    CUDA_OK(cudaSetDevice(s->device));
    int64_t B = 0;
    int32_t* dn = dmalloc<int32_t>(n, B);
    unsigned long long* dh = dmalloc<unsigned long long>(n, B);
    double* ds = dmalloc<double>(n, B);
    k_checksums<<<(int)std::min<int64_t>(4096, (n + 255) / 256), 256, 0, s->stream>>>(s->dd, (uint32_t)first,
                                                                                     (uint32_t)n, dn, dh, ds);
    CUDA_OK(cudaGetLastError());
    if (nseg) CUDA_OK(cudaMemcpyAsync(nseg, dn, 4 * n, cudaMemcpyDeviceToHost, s->stream));
    if (hash) CUDA_OK(cudaMemcpyAsync(hash, dh, 8 * n, cudaMemcpyDeviceToHost, s->stream));
    if (suml) CUDA_OK(cudaMemcpyAsync(suml, ds, 8 * n, cudaMemcpyDeviceToHost, s->stream));
    CUDA_OK(cudaStreamSynchronize(s->stream));
    cudaFree(dn);
    cudaFree(dh);
    cudaFree(ds);
  })
}

int moc_get_timings(moc_solver* s, moc_timings* t) {
  if (!s || !t) return MOC_E_INVALID_ARG;
  if (cudaSetDevice(s->device) != cudaSuccess) return MOC_E_CUDA;
  t->n_segs3d = s->nseg3;
  t->n_integrations = 2 * s->nseg3 * s->G;
  float ms = 0;
  if (s->sweep_timed && cudaEventSynchronize(s->ev[1]) == cudaSuccess &&
      cudaEventElapsedTime(&ms, s->ev[0], s->ev[1]) == cudaSuccess)
    s->sweep_ms_last = ms;
  (void)cudaGetLastError();  // never leave a query error behind for the next launch check
  t->sweep_ms_last = s->sweep_ms_last;
  t->iter_ms_last = s->iter_ms_last;
  // kernels per iteration: source, sweep, finalize, keff, normalize, resid (+ the two
  // bound kernels for schedule 0, + halo gather/scatter and leak park/restore for world > 1)
  int sc_launches = 0;
  for (int g = 0; g < 3; ++g) {
    t->sc_units[g] = s->sc_grp[g].n;
    sc_launches += s->sc_grp[g].n > 0;
  }
  t->launches_per_iter = 6 + (s->opts.schedule == 0 ? 2 : 0) + (s->comm.world > 1 ? 4 : 0) +
                         (s->exp_units > 0 && (int64_t)s->n_units > s->exp_units ? 1 : 0) +  // EXP + OTF sweeps
                         (sc_launches > 1 ? sc_launches - 1 : 0);  // schedule 3: one sweep per occupancy group
  t->setup_ms = s->setup_ms;
  t->device_bytes = s->dev_bytes;
  t->exp_segments = s->exp_segments;
  t->exp_bytes = s->exp_bytes;
  double sc[SC_N];
  t->emitted_last = -1;
  if (cudaMemcpyAsync(sc, s->d_sc, sizeof(sc), cudaMemcpyDeviceToHost, s->stream) == cudaSuccess &&
      cudaStreamSynchronize(s->stream) == cudaSuccess)
    t->emitted_last = (int64_t)sc[SC_NEMIT_LAST];
  (void)cudaGetLastError();
  return MOC_OK;
}

int moc_solver_comm_buffers(moc_solver* s, moc_comm_buffers* b) {
  if (!s || !b) return MOC_E_INVALID_ARG;
  b->tally = s->opts.schedule == 0 || s->opts.schedule == 3 ? (void*)s->d_tally32 : (void*)s->d_tally;
  // fp32 [J][GP] plus one tail element carrying the leakage through the all-reduce
  b->tally_elems = s->J * s->GP + (s->comm.world > 1 ? 1 : 0);
  b->halo_send = s->d_halo_send;
  b->halo_recv = s->d_halo_recv;
  b->halo_elems = std::max(s->n_send, s->n_recv) * s->GP;
  return MOC_OK;
}

int moc_sweep_checksums(moc_solver* s, int32_t* nseg, uint64_t* hash) {
  if (!s || !nseg || !hash) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    if (s->opts.schedule != 3) throw Error(MOC_E_STATE, "sweep checksums need schedule 3");
    if (s->comm.world > 1) throw Error(MOC_E_STATE, "sweep checksums are single-GPU");
    ensure_constants(s);
    const size_t n = 2 * (size_t)s->T3;
    int64_t B = 0;
    int32_t* dn = dmalloc<int32_t>(n, B);
    unsigned long long* dh = dmalloc<unsigned long long>(n, B);
    CUDA_OK(cudaMemsetAsync(dn, 0, 4 * n, s->stream));
    CUDA_OK(cudaMemsetAsync(dh, 0, 8 * n, s->stream));
    CUDA_OK(cudaMemsetAsync(s->d_tally32, 0, sizeof(float) * s->J * s->GP, s->stream));
    CUDA_OK(cudaMemsetAsync(s->d_counter, 0, 2 * sizeof(uint32_t), s->stream));
    double sc[SC_N];
    read_scalars(s, sc);
    switch (s->G) {
      case 1: run_sweep_sc<1, 1, true>(s, dh, dn); break;
      case 2: run_sweep_sc<2, 2, true>(s, dh, dn); break;
      case 3: run_sweep_sc<3, 4, true>(s, dh, dn); break;
      case 4: run_sweep_sc<4, 4, true>(s, dh, dn); break;
      case 5: run_sweep_sc<5, 8, true>(s, dh, dn); break;
      case 6: run_sweep_sc<6, 8, true>(s, dh, dn); break;
      case 7: run_sweep_sc<7, 8, true>(s, dh, dn); break;
      default: run_sweep_sc<8, 8, true>(s, dh, dn); break;
    }
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(nseg, dn, 4 * n, cudaMemcpyDeviceToHost, s->stream));
    CUDA_OK(cudaMemcpyAsync(hash, dh, 8 * n, cudaMemcpyDeviceToHost, s->stream));
    // restore the scalars the sweep accumulates into (leakage, emission counter)
    CUDA_OK(cudaMemcpyAsync(s->d_sc, sc, sizeof(sc), cudaMemcpyHostToDevice, s->stream));
    CUDA_OK(cudaStreamSynchronize(s->stream));
    cudaFree(dn);
    cudaFree(dh);
  })
}

#ifdef MOC_SC_STATS
int moc_debug_sc_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_sc_stats, sizeof(g_sc_stats)) != cudaSuccess) return MOC_E_CUDA;
  if (reset) {
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(g_sc_stats, z, sizeof(z)) != cudaSuccess) return MOC_E_CUDA;
  }
  return MOC_OK;
}
#endif

int moc_attenuation_probe(int device, int64_t n, const float* psi, const float* q, const float* sigma_t,
                          const float* len, float* psi_out, float* dpsi) {
  if (n < 0 || (n > 0 && (!psi || !q || !sigma_t || !len || !psi_out || !dpsi))) return MOC_E_INVALID_ARG;
  if (n == 0) return MOC_OK;
  try {
    CUDA_OK(cudaSetDevice(device));
    int64_t B = 0;
    float* d = dmalloc<float>(6 * (size_t)n, B);
    const size_t b = sizeof(float) * n;
    CUDA_OK(cudaMemcpy(d, psi, b, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(d + n, q, b, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(d + 2 * n, sigma_t, b, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(d + 3 * n, len, b, cudaMemcpyHostToDevice));
    k_attenuation_probe<<<256, 256>>>(n, d, d + n, d + 2 * n, d + 3 * n, d + 4 * n, d + 5 * n);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpy(psi_out, d + 4 * n, b, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(dpsi, d + 5 * n, b, cudaMemcpyDeviceToHost));
    cudaFree(d);
  } catch (const Error& e) {
    return e.code;
  }
  return MOC_OK;
}

int moc_solver_halo_counts(moc_solver* s, int64_t* send_elems, int64_t* recv_elems) {
  if (!s || !send_elems || !recv_elems) return MOC_E_INVALID_ARG;
  for (int p = 0; p < s->comm.world; ++p) {
    send_elems[p] = p < (int)s->send_counts.size() ? s->send_counts[p] * s->GP : 0;
    recv_elems[p] = p < (int)s->recv_counts.size() ? s->recv_counts[p] * s->GP : 0;
  }
  return MOC_OK;
}

int moc_nccl_unique_id(uint8_t* id) {
  if (!id) return MOC_E_INVALID_ARG;
  try {
    ncclUniqueId u;
    NCCL_OK(nccl_api().getUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  } catch (const Error& e) {
    return e.code;
  }
  return MOC_OK;
}

int moc_solver_set_exchange(moc_solver* s, moc_exchange_fn fn, void* ctx) {
  if (!s) return MOC_E_INVALID_ARG;
  s->xfn = fn;
  s->xctx = ctx;
  return MOC_OK;
}

int moc_iteration_sweep(moc_solver* s) {
  if (!s) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    if (s->opts.schedule != 0 && s->opts.schedule != 3) throw Error(MOC_E_STATE, "split iterations need schedule 0 or 3");
    pick_sweep_half(s->G)(s, true);
  })
}

int moc_iteration_finish(moc_solver* s) {
  if (!s) return MOC_E_INVALID_ARG;
  SOLVER_TRY(s, {
    CUDA_OK(cudaSetDevice(s->device));
    if (s->opts.schedule != 0 && s->opts.schedule != 3) throw Error(MOC_E_STATE, "split iterations need schedule 0 or 3");
    pick_finish_half(s->G)(s, false);
  })
}

}  // extern "C"
