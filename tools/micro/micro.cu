// M0 microbenchmarks for the MOC sweep design decisions.
// Measures per-SM throughput of the instructions the OTF sweep's inner loop is
// built from: MUFU.EX2, FFMA, DFMA, shared-memory atomics (conflict-free and
// same-address), plain shared RMW, and global RED into an L2-resident array.
// Output: one JSON object per line on stdout.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];

__global__ void k_ex2(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float r0, r1, r2, r3;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(a0));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(a1));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(a2));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r3) : "f"(a3));
    a0 = -r0; a1 = -r1; a2 = -r2; a3 = -r3;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

__global__ void k_ffma(float* out, int iters) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 0.999f, 0.001f);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// Blackwell packed fp32 (FFMA2): 8 independent chains of fma.rn.f32x2 per thread.
__global__ void k_ffma2(float* out, int iters) {
  unsigned long long a[8];
  for (int j = 0; j < 8; ++j) { float2 f = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f); a[j] = *(unsigned long long*)&f; }
  float2 cm = make_float2(0.999f, 0.998f), ca = make_float2(0.001f, 0.002f);
  unsigned long long m = *(unsigned long long*)&cm, c = *(unsigned long long*)&ca;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(m), "l"(c));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  float s = 0; for (int j = 0; j < 8; ++j) { float2 f = *(float2*)&a[j]; s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FFMA2 interleaved 1:1 with integer adds: are packed ops issue-limited or pipe-limited?
__global__ void k_ffma2_iadd(float* out, int iters) {
  unsigned long long a[4];
  unsigned b[4];
  for (int j = 0; j < 4; ++j) { float2 f = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f); a[j] = *(unsigned long long*)&f; b[j] = threadIdx.x + j; }
  float2 cm = make_float2(0.999f, 0.998f), ca = make_float2(0.001f, 0.002f);
  unsigned long long m = *(unsigned long long*)&cm, c = *(unsigned long long*)&ca;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(m), "l"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(b[j]) : "r"(j + 1));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  float s = 0; for (int j = 0; j < 4; ++j) { float2 f = *(float2*)&a[j]; s += f.x + f.y + b[j]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 0.999, 0.001);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  double s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mode 0: each lane its own word (stride 1 -> conflict-free)
// mode 1: 4 lanes share an address (same-address conflicts)
// mode 2: all 32 lanes same address
// mode 3: lanes stride 8 words (8-way bank conflict)
template <int MODE>
__global__ void k_atoms(float* out, int iters) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0.f;
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int addr;
  if (MODE == 0) addr = warp * 32 + lane;
  else if (MODE == 1) addr = warp * 32 + (lane >> 2);
  else if (MODE == 2) addr = warp * 32;
  else addr = (warp * 32 * 8 + lane * 8) & 8191;
  float v = 1.0f + lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) atomicAdd(&sm[(addr + u * 1024) & 8191], v);
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[threadIdx.x];
}

// plain read-modify-write of a float4 per lane (no atomics), conflict-free layout
__global__ void k_rmw4(float* out, int iters) {
  extern __shared__ float4 sm4[];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm4[i] = make_float4(0, 0, 0, 0);
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4 v = make_float4(1, 2, 3, 4);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int a = (warp * 32 + lane + u * 512) & 2047;
      float4 x = sm4[a];
      x.x += v.x; x.y += v.y; x.z += v.z; x.w += v.w;
      sm4[a] = x;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  float4 r = sm4[threadIdx.x & 2047];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r.x + r.y + r.z + r.w;
}

// global RED.ADD.F32 to pseudo-random addresses inside an n-word array
__global__ void k_redg(float* arr, unsigned n, int iters) {
  unsigned x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&arr[(x >> 4) % n], 1.0f);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

__global__ void k_redg_v4(float* arr, unsigned n4, int iters) {
  unsigned x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    float* p = arr + 4 * ((x >> 4) % n4);
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

__global__ void k_redg_f64(double* arr, unsigned n, int iters) {
  unsigned x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    atomicAdd(&arr[(x >> 4) % n], 1.0);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}


template <int MODE>
__global__ void k_atoms_i32(float* out, int iters) {
  extern __shared__ unsigned smu[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) smu[i] = 0u;
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int addr;
  if (MODE == 0) addr = warp * 32 + lane;
  else if (MODE == 1) addr = warp * 32 + (lane >> 2);
  else if (MODE == 2) addr = warp * 32;
  else addr = (warp * 32 * 8 + lane * 8) & 8191;
  unsigned v = 1u + lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) atomicAdd(&smu[(addr + u * 1024) & 8191], v);
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)smu[threadIdx.x];
}

__global__ void k_atoms_u64(float* out, int iters) {
  extern __shared__ unsigned long long smq[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) smq[i] = 0ull;
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int addr = warp * 32 + lane;
  unsigned long long v = 1ull + lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) atomicAdd(&smq[(addr + u * 1024) & 4095], v);
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)smq[threadIdx.x];
}

__global__ void k_f2i(float* out, int iters) {
  float a[8]; int acc = 0;
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc ^= __float2int_rn(a[j]); a[j] += 1.0f; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

static int nsm;
static double report(const char* name, float ms, double ops, int blocks) {
  unsigned long long cyc[1024];
  cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * (blocks < 1024 ? blocks : 1024));
  double mc = 0; int nb = blocks < 1024 ? blocks : 1024;
  for (int i = 0; i < nb; ++i) mc += (double)cyc[i];
  mc /= nb;
  double per_s = ops / (ms * 1e-3);
  double mhz = mc / (ms * 1e3);  // rough: avg block cycles / elapsed us (1 block/SM resident)
  printf("{\"bench\": \"%s\", \"ops_per_s\": %.4e, \"ms\": %.4f, \"ops_per_sm_clk_at_est_clock\": %.3f, \"est_mhz\": %.1f}\n",
         name, per_s, ms, per_s / (nsm * mhz * 1e6), mhz);
  return per_s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  nsm = p.multiProcessorCount;
  int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"smem_optin\": %zu, \"regs_per_sm\": %d, \"mem_bytes\": %zu}\n",
         p.name, nsm, l2, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.totalGlobalMem);
  float* out; CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int B = nsm * 4, T = 256;
  // ex2
  { int it = 20000; k_ex2<<<B, T>>>(out, 10); cudaEventRecord(e0); k_ex2<<<B, T>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("mufu_ex2", ms, 4.0 * it * B * T, B); }
  { int it = 20000; k_ffma<<<B, T>>>(out, 10); cudaEventRecord(e0); k_ffma<<<B, T>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("ffma", ms, 8.0 * it * B * T, B); }
  { int it = 20000; k_ffma2<<<B, T>>>(out, 10); cudaEventRecord(e0); k_ffma2<<<B, T>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("ffma2_fp32_fmas", ms, 16.0 * it * B * T, B);
    report("ffma2_warp_insts_x32", ms, 8.0 * it * B * T, B); }
  { int it = 20000; k_ffma2_iadd<<<B, T>>>(out, 10); cudaEventRecord(e0); k_ffma2_iadd<<<B, T>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("ffma2_plus_iadd_thread_insts", ms, 8.0 * it * B * T, B); }
  { int it = 5000; k_dfma<<<B, T>>>((double*)out, 10); cudaEventRecord(e0); k_dfma<<<B, T>>>((double*)out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("dfma", ms, 8.0 * it * B * T, B); }
  size_t sm = 8192 * 4;
  {
    int it = 5000;
#define RUN_ATOMS(M, NAME) k_atoms<M><<<B, T, sm>>>(out, 10); cudaEventRecord(e0); k_atoms<M><<<B, T, sm>>>(out, it); cudaEventRecord(e1); \
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report(NAME, ms, 4.0 * it * B * T, B);
    RUN_ATOMS(0, "atoms_f32_conflict_free")
    RUN_ATOMS(1, "atoms_f32_4lanes_same_addr")
    RUN_ATOMS(2, "atoms_f32_32lanes_same_addr")
    RUN_ATOMS(3, "atoms_f32_8way_bank_conflict")
  }

  {
    int it = 5000;
#define RUN_ATOMSI(M, NAME) k_atoms_i32<M><<<B, T, sm>>>(out, 10); cudaEventRecord(e0); k_atoms_i32<M><<<B, T, sm>>>(out, it); cudaEventRecord(e1); \
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report(NAME, ms, 4.0 * it * B * T, B);
    RUN_ATOMSI(0, "atoms_u32_conflict_free")
    RUN_ATOMSI(1, "atoms_u32_4lanes_same_addr")
    RUN_ATOMSI(2, "atoms_u32_32lanes_same_addr")
    RUN_ATOMSI(3, "atoms_u32_8way_bank_conflict")
    k_atoms_u64<<<B, T, sm>>>(out, 10); cudaEventRecord(e0); k_atoms_u64<<<B, T, sm>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("atoms_u64_conflict_free", ms, 4.0 * it * B * T, B);
    k_f2i<<<B, T>>>(out, 10); cudaEventRecord(e0); k_f2i<<<B, T>>>(out, 20000); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("f2i_rn", ms, 8.0 * 20000 * B * T, B);
  }
  { int it = 5000; k_rmw4<<<B, T, sm>>>(out, 10); cudaEventRecord(e0); k_rmw4<<<B, T, sm>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report("smem_rmw_float4_lane_elems", ms, 4.0 * 4 * it * B * T, B); }
  // global reds into 12 MB (L2 resident) and 1 GB (DRAM)
  float* arr; CK(cudaMalloc(&arr, 1ull << 30));
  CK(cudaMemset(arr, 0, 1ull << 30));
  unsigned sizes[2] = {3u << 20, 1u << 28};
  const char* nm[2] = {"redg_f32_12MB", "redg_f32_1GB"};
  const char* nm4[2] = {"redg_v4f32_12MB(lane-elems)", "redg_v4f32_1GB(lane-elems)"};
  const char* nm64[2] = {"redg_f64_12MB", "redg_f64_1GB"};
  for (int s = 0; s < 2; ++s) {
    int it = 2000;
    k_redg<<<B, T>>>(arr, sizes[s], 10); cudaEventRecord(e0); k_redg<<<B, T>>>(arr, sizes[s], it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report(nm[s], ms, 1.0 * it * B * T, B);
    k_redg_v4<<<B, T>>>(arr, sizes[s] / 4, 10); cudaEventRecord(e0); k_redg_v4<<<B, T>>>(arr, sizes[s] / 4, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report(nm4[s], ms, 4.0 * it * B * T, B);
    k_redg_f64<<<B, T>>>((double*)arr, sizes[s] / 2, 10); cudaEventRecord(e0); k_redg_f64<<<B, T>>>((double*)arr, sizes[s] / 2, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); report(nm64[s], ms, 1.0 * it * B * T, B);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
