// SDDMM micro-lab (standalone; not part of the library).  Decomposes the time
// of the chunked cp.async SDDMM into its load and chain parts on three shapes:
//   config-2 L0 (1024 x 3072, 24 nnz/row), config-2 L2 (10 x 512, 312/row),
//   config-4 L1 (8192 x 8192, 69/row); batch 1024, fp32.
// MODE 0 = full kernel, 1 = loads only, 2 = chain only (smem not refilled).
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --fmad=false
//        scripts/sddmm_lab.cu -o /tmp/sddmm_lab
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(unsigned dst, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(g));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void waitg() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// TILE nonzeros per CTA (one chain per thread), CH columns per chunk, ST stages
template <int TILE, int CH, int ST, int MODE, int SD = 4>
__global__ void __launch_bounds__(TILE) lab_pipe(const int* row_ptr, const int* col_idx,
                                                 const int* row_of, int nnz, const float* dy,
                                                 const float* x, int n, float* out) {
  constexpr int VPR = CH / 4, LDS = CH + 4, SLOTS = TILE / SD;
  constexpr int STAGE = (TILE + SLOTS) * LDS;
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  const int p0 = blockIdx.x * TILE, p = p0 + tid;
  const bool active = p < nnz;
  const int pl = min(p, nnz - 1);
  const int row = row_of[pl];
  const int r0 = row_of[p0];
  const int slot = row - r0;
  const int rlast = row_of[min(p0 + TILE, nnz) - 1];
  const int nst = rlast - r0 + 1;
  const int v = tid % VPR;
  const float* xs[VPR];
  unsigned xd[VPR];
#pragma unroll
  for (int k = 0; k < VPR; ++k) {
    const int r = tid / VPR + k * (TILE / VPR);
    xs[k] = x + (size_t)col_idx[min(p0 + r, nnz - 1)] * n + v * 4;
    xd[k] = (unsigned)((r * LDS + v * 4) * 4);
  }
  constexpr int DC = (SLOTS * VPR + TILE - 1) / TILE;
  const float* ds[DC];
  unsigned dd[DC];
  bool dok[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    const int e = tid + c * TILE;
    dok[c] = e < nst * VPR;
    ds[c] = dy + (size_t)(r0 + (dok[c] ? e / VPR : 0)) * n + v * 4;
    dd[c] = (unsigned)(((TILE + e / VPR) * LDS + v * 4) * 4);
  }
  const unsigned sb = smem_u32(sm);
  const int nch = n / CH;
  auto issue = [&](int ch) {
    if (MODE == 2 && ch >= ST) return;
    const unsigned st = sb + (unsigned)(ch % ST) * STAGE * 4;
    const int t0 = ch * CH;
#pragma unroll
    for (int k = 0; k < VPR; ++k) cp16(st + xd[k], xs[k] + t0);
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (dok[c]) cp16(st + dd[c], ds[c] + t0);
  };
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    issue(s);
    commit();
  }
  float acc = -0.0f;
  float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int ch = 0; ch < nch; ++ch) {
    waitg<ST - 2>();
    __syncthreads();
    if (ch + ST - 1 < nch) issue(ch + ST - 1);
    commit();
    const float* s = sm + (ch % ST) * STAGE;
    const float* xr = s + tid * LDS;
    const float* dr = s + (TILE + slot) * LDS;
    if (MODE == 1) {
      acc = __fadd_rn(acc, xr[0] * dr[0]);
    } else if (MODE == 3) {  // tolerance experiment: 4 FFMA accumulators (t mod 4)
#pragma unroll
      for (int u = 0; u < VPR; ++u) {
        const float4 a = *reinterpret_cast<const float4*>(xr + u * 4);
        const float4 b = *reinterpret_cast<const float4*>(dr + u * 4);
        a4.x = fmaf(b.x, a.x, a4.x);
        a4.y = fmaf(b.y, a.y, a4.y);
        a4.z = fmaf(b.z, a.z, a4.z);
        a4.w = fmaf(b.w, a.w, a4.w);
      }
    } else {
#pragma unroll
      for (int u = 0; u < VPR; ++u) {
        const float4 a = *reinterpret_cast<const float4*>(xr + u * 4);
        const float4 b = *reinterpret_cast<const float4*>(dr + u * 4);
        acc = __fadd_rn(acc, __fmul_rn(b.x, a.x));
        acc = __fadd_rn(acc, __fmul_rn(b.y, a.y));
        acc = __fadd_rn(acc, __fmul_rn(b.z, a.z));
        acc = __fadd_rn(acc, __fmul_rn(b.w, a.w));
      }
    }
  }
  waitg<0>();
  if (MODE == 3) acc = (a4.x + a4.y) + (a4.z + a4.w);
  if (active) out[p] = acc;
}

// Register-staged variant: 16-byte LDG into registers NR chunks ahead, then
// STS into a 2-stage smem ring (no LDGSTS).  MODE 0 full, 1 loads only.
template <int TILE, int CH, int NR, int MODE, int SD>
__global__ void __launch_bounds__(TILE) lab_reg(const int* row_of, const int* col_idx, int nnz,
                                                const float* __restrict__ dy,
                                                const float* __restrict__ x, int n, float* out) {
  constexpr int VPR = CH / 4, LDS = CH + 4, SLOTS = TILE / SD;
  constexpr int STAGE = (TILE + SLOTS) * LDS;
  constexpr int DC = (SLOTS * VPR + TILE - 1) / TILE;
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  const int p0 = blockIdx.x * TILE, p = p0 + tid;
  const bool active = p < nnz;
  const int pl = min(p, nnz - 1);
  const int row = row_of[pl];
  const int r0 = row_of[p0];
  const int slot = row - r0;
  const int rlast = row_of[min(p0 + TILE, nnz) - 1];
  const int nst = rlast - r0 + 1;
  const int v = tid % VPR;
  const float4* xs[VPR];
  int xd[VPR];
#pragma unroll
  for (int k = 0; k < VPR; ++k) {
    const int r = tid / VPR + k * (TILE / VPR);
    xs[k] = reinterpret_cast<const float4*>(x + (size_t)col_idx[min(p0 + r, nnz - 1)] * n + v * 4);
    xd[k] = r * LDS + v * 4;
  }
  const float4* ds[DC];
  int dd[DC];
  bool dok[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    const int e = tid + c * TILE;
    dok[c] = e < nst * VPR;
    ds[c] = reinterpret_cast<const float4*>(dy + (size_t)(r0 + (dok[c] ? e / VPR : 0)) * n + v * 4);
    dd[c] = (TILE + e / VPR) * LDS + v * 4;
  }
  const int nch = n / CH;
  float4 rx[NR][VPR], rd[NR][DC];
  auto load = [&](int ch, float4(&ax)[VPR], float4(&ad)[DC]) {
    const int q = ch * (CH / 4);
#pragma unroll
    for (int k = 0; k < VPR; ++k) ax[k] = __ldcg(xs[k] + q);
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (dok[c]) ad[c] = __ldcg(ds[c] + q);
  };
  auto store = [&](int stg, const float4(&ax)[VPR], const float4(&ad)[DC]) {
    float* st = sm + stg * STAGE;
#pragma unroll
    for (int k = 0; k < VPR; ++k) *reinterpret_cast<float4*>(st + xd[k]) = ax[k];
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (dok[c]) *reinterpret_cast<float4*>(st + dd[c]) = ad[c];
  };
#pragma unroll
  for (int r = 0; r < NR; ++r)
    if (r < nch) load(r, rx[r], rd[r]);
  float acc = -0.0f;
  for (int base = 0; base < nch; base += NR) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int ch = base + r;
      if (ch < nch) {
        store(ch & 1, rx[r], rd[r]);
        if (ch + NR < nch) load(ch + NR, rx[r], rd[r]);
        __syncthreads();
        const float* s = sm + (ch & 1) * STAGE;
        const float* xr = s + tid * LDS;
        const float* dr = s + (TILE + slot) * LDS;
        if (MODE == 1) {
          acc = __fadd_rn(acc, xr[0] * dr[0]);
        } else {
#pragma unroll
          for (int u = 0; u < VPR; ++u) {
            const float4 a = *reinterpret_cast<const float4*>(xr + u * 4);
            const float4 b = *reinterpret_cast<const float4*>(dr + u * 4);
            acc = __fadd_rn(acc, __fmul_rn(b.x, a.x));
            acc = __fadd_rn(acc, __fmul_rn(b.y, a.y));
            acc = __fadd_rn(acc, __fmul_rn(b.z, a.z));
            acc = __fadd_rn(acc, __fmul_rn(b.w, a.w));
          }
        }
      }
    }
  }
  if (active) out[p] = acc;
}

// Direct-load variant: no shared memory; each thread streams its own x row
// and its d_out row through L1 with 16-byte __ldg, R loads ahead.
template <int R>
__global__ void __launch_bounds__(128) lab_ldg(const int* row_of, const int* col_idx, int nnz,
                                               const float* __restrict__ dy,
                                               const float* __restrict__ x, int n, float* out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)col_idx[p] * n);
  const float4* dr = reinterpret_cast<const float4*>(dy + (size_t)row_of[p] * n);
  const int nv = n / 4;
  float4 xa[R], da[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    xa[r] = __ldg(xr + r);
    da[r] = __ldg(dr + r);
  }
  float acc = -0.0f;
  for (int v = 0; v < nv; v += R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float4 a = xa[r], b = da[r];
      if (v + R + r < nv) {
        xa[r] = __ldg(xr + v + R + r);
        da[r] = __ldg(dr + v + R + r);
      }
      acc = __fadd_rn(acc, __fmul_rn(b.x, a.x));
      acc = __fadd_rn(acc, __fmul_rn(b.y, a.y));
      acc = __fadd_rn(acc, __fmul_rn(b.z, a.z));
      acc = __fadd_rn(acc, __fmul_rn(b.w, a.w));
    }
  }
  out[p] = acc;
}

// Register-only chain: how fast can 1024 dependent mul/add steps go per chain
// with loads fully removed (values synthesised from the index).
__global__ void lab_chain(int nnz, int n, float* out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  float a = 1.0f + p * 1e-7f, b = 0.5f, acc = -0.0f;
  for (int t = 0; t < n; t += 4) {
    acc = __fadd_rn(acc, __fmul_rn(a, b));
    a = __fadd_rn(a, 1e-7f);  // independent of acc
    acc = __fadd_rn(acc, __fmul_rn(a, b));
    a = __fadd_rn(a, 1e-7f);
    acc = __fadd_rn(acc, __fmul_rn(a, b));
    a = __fadd_rn(a, 1e-7f);
    acc = __fadd_rn(acc, __fmul_rn(a, b));
    a = __fadd_rn(a, 1e-7f);
  }
  out[p] = acc;
}

struct Shape {
  const char* name;
  int m, k, r;
};

template <typename F>
float time_us(F f, int reps = 20) {
  // reps launches captured in one CUDA graph (stream launches would round
  // each kernel up to the ~2 us dependency-polling period, launch_gap_lab.cu)
  static cudaStream_t s = nullptr;
  if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaStream_t legacy = 0;
  (void)legacy;
  for (int i = 0; i < 3; ++i) f(s);
  CK(cudaStreamSynchronize(s));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < reps; ++i) f(s);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(g));
  return ms * 1e3f / (5 * reps);
}

template <int TILE, int CH, int ST, int MODE, int SD = 4>
float run_pipe(const Shape& s, int nnz, const int* rp, const int* ci, const int* ro, const float* dy,
               const float* x, int n, float* out) {
  constexpr int SLOTS = TILE / SD;
  const size_t bytes = (size_t)ST * (TILE + SLOTS) * (CH + 4) * 4;
  auto k = lab_pipe<TILE, CH, ST, MODE, SD>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  const int grid = (nnz + TILE - 1) / TILE;
  return time_us([&](cudaStream_t st) { k<<<grid, TILE, bytes, st>>>(rp, ci, ro, nnz, dy, x, n, out); });
}

template <int TILE, int CH, int NR, int MODE, int SD>
float run_reg(int nnz, const int* ro, const int* ci, const float* dy, const float* x, int n, float* out) {
  constexpr int SLOTS = TILE / SD;
  const size_t bytes = (size_t)2 * (TILE + SLOTS) * (CH + 4) * 4;
  auto k = lab_reg<TILE, CH, NR, MODE, SD>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  const int grid = (nnz + TILE - 1) / TILE;
  return time_us([&](cudaStream_t st) { k<<<grid, TILE, bytes, st>>>(ro, ci, nnz, dy, x, n, out); });
}

int main() {
  const int n = 1024;
  Shape shapes[] = {{"c2.L0 1024x3072 r24", 1024, 3072, 24},
                    {"c2.L2 10x512 r312", 10, 512, 312},
                    {"c2.L1 512x1024 r18", 512, 1024, 18},
                    {"c4.L1 8192x8192 r69", 8192, 8192, 69}};
  std::mt19937 rng(1);
  for (const Shape& s : shapes) {
    std::vector<int> rp(s.m + 1), ci, ro;
    std::vector<int> cols(s.k);
    for (int c = 0; c < s.k; ++c) cols[c] = c;
    for (int i = 0; i < s.m; ++i) {
      std::shuffle(cols.begin(), cols.end(), rng);
      std::vector<int> row(cols.begin(), cols.begin() + s.r);
      std::sort(row.begin(), row.end());
      for (int c : row) {
        ci.push_back(c);
        ro.push_back(i);
      }
      rp[i + 1] = (int)ci.size();
    }
    const int nnz = (int)ci.size();
    int *d_rp, *d_ci, *d_ro;
    float *d_dy, *d_x, *d_out;
    CK(cudaMalloc(&d_rp, rp.size() * 4));
    CK(cudaMalloc(&d_ci, ci.size() * 4));
    CK(cudaMalloc(&d_ro, ro.size() * 4));
    CK(cudaMalloc(&d_dy, (size_t)s.m * n * 4));
    CK(cudaMalloc(&d_x, (size_t)s.k * n * 4));
    CK(cudaMalloc(&d_out, (size_t)nnz * 4));
    CK(cudaMemcpy(d_rp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), ci.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ro, ro.data(), ro.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_dy, 0, (size_t)s.m * n * 4));
    CK(cudaMemset(d_x, 0, (size_t)s.k * n * 4));
    printf("%s nnz=%d (%.1f MB x-gather)\n", s.name, nnz, nnz * 4.0 * n / 1e6);
#define P(T, C, S)                                                                          \
  printf("  pipe<%d,%d,%d>: full %.2f  loads %.2f  chain %.2f us\n", T, C, S,               \
         run_pipe<T, C, S, 0>(s, nnz, d_rp, d_ci, d_ro, d_dy, d_x, n, d_out),              \
         run_pipe<T, C, S, 1>(s, nnz, d_rp, d_ci, d_ro, d_dy, d_x, n, d_out),              \
         run_pipe<T, C, S, 2>(s, nnz, d_rp, d_ci, d_ro, d_dy, d_x, n, d_out))
#define Q(T, C, S, D)                                                                       \
  printf("  pipe<%d,%d,%d> SD=%d: full %.2f  split4 %.2f loads %.2f  chain %.2f us\n", T, C, S, D, \
         run_pipe<T, C, S, 0, D>(s, nnz, d_rp, d_ci, d_ro, d_dy, d_x, n, d_out),              \
         run_pipe<T, C, S, 3, D>(s, nnz, d_rp, d_ci, d_ro, d_dy, d_x, n, d_out),              \
         run_pipe<T, C, S, 1, D>(s, nnz, d_rp, d_ci, d_ro, d_dy, d_x, n, d_out),              \
         run_pipe<T, C, S, 2, D>(s, nnz, d_rp, d_ci, d_ro, d_dy, d_x, n, d_out))
#define R(T, C, N, D)                                                                  \
  printf("  reg<%d,%d,NR=%d> SD=%d: full %.2f  loads %.2f us\n", T, C, N, D,                \
         run_reg<T, C, N, 0, D>(nnz, d_ro, d_ci, d_dy, d_x, n, d_out),                      \
         run_reg<T, C, N, 1, D>(nnz, d_ro, d_ci, d_dy, d_x, n, d_out))
    if (s.m == 8192) R(64, 32, 3, 8);
    if (s.m == 10 || s.m == 512) {
      Q(32, 32, 8, 4);
      Q(64, 32, 4, 4);
      Q(64, 64, 4, 4);
      continue;
    }
    if (s.m == 8192) {
      Q(128, 32, 2, 4);
      continue;
    }
    if (s.m == 1024) {
      Q(64, 32, 4, 4);
      Q(64, 32, 2, 4);
      Q(64, 64, 2, 4);
      Q(64, 32, 3, 4);
      Q(64, 32, 6, 8);
      Q(32, 32, 8, 4);
      Q(32, 32, 4, 4);
      Q(32, 64, 2, 4);
      Q(32, 64, 4, 4);
      Q(128, 32, 2, 4);
      Q(96, 32, 4, 8);
      continue;
    }
    P(128, 64, 2);
    P(128, 32, 2);
    if (s.m <= 1024) {
      P(64, 64, 2);
      P(64, 64, 4);
      P(64, 32, 4);
      P(64, 32, 8);
      P(64, 16, 8);
      P(32, 64, 4);
      P(32, 32, 8);
      P(32, 32, 16);
      P(32, 16, 16);
    }
    for (int R : {4, 8})
      printf("  ldg R=%d: %.2f us\n", R,
             R == 4 ? time_us([&](cudaStream_t st) { lab_ldg<4><<<(nnz + 127) / 128, 128, 0, st>>>(d_ro, d_ci, nnz, d_dy, d_x, n, d_out); })
                    : time_us([&](cudaStream_t st) { lab_ldg<8><<<(nnz + 127) / 128, 128, 0, st>>>(d_ro, d_ci, nnz, d_dy, d_x, n, d_out); }));
    for (int bs : {128})
      printf("  chain-only regs (block %d): %.2f us\n", bs,
             time_us([&](cudaStream_t st) { lab_chain<<<(nnz + bs - 1) / bs, bs, 0, st>>>(nnz, n, d_out); }));
    cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_ro); cudaFree(d_dy); cudaFree(d_x); cudaFree(d_out);
  }
  return 0;
}
