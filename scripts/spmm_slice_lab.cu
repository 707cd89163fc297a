// Slice-resident SpMM micro-lab (standalone; not part of the library).
// Y[:, slice] = W * X[:, slice] with the whole X[:, slice] (k x BS floats)
// staged once in shared memory, so every nonzero reads its x segment from
// smem instead of gathering it from L2.  Grid = (B / BS) slices x RS row
// splits.  Thread = (row, 4-column quad); rows processed in CSR order, each
// output element summed in ascending p with separate mul / add roundings.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --fmad=false
//        scripts/spmm_slice_lab.cu -o /tmp/spmm_slice_lab
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

// BS batch columns per slice; LDX padded smem row (floats)
template <int BS, int THREADS>
__global__ void __launch_bounds__(THREADS)
    spmm_slice(const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
               const float* __restrict__ vals, int m, int k, const float* __restrict__ x,
               int ld, float* __restrict__ y, int rs) {
  constexpr int Q = BS / 4;             // quads per row
  constexpr int RPP = THREADS / Q;      // rows per pass
  constexpr int LDX = BS + ((BS == 32 || BS == 4) ? 0 : 4);  // padding breaks row-bank aliasing
  extern __shared__ __align__(16) float xs[];
  const int slice = blockIdx.x / rs, split = blockIdx.x % rs;
  const int c0 = slice * BS;
  // stage X[:, c0:c0+BS]
  for (int e = threadIdx.x; e < k * Q; e += THREADS) {
    const int j = e / Q, q = e % Q;
    cp16(smem_u32(xs + j * LDX + q * 4), x + (size_t)j * ld + c0 + q * 4);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n");
  __syncthreads();
  const int r_lo = (int)((int64_t)m * split / rs), r_hi = (int)((int64_t)m * (split + 1) / rs);
  const int q = threadIdx.x % Q;
  for (int i = r_lo + threadIdx.x / Q; i < r_hi; i += RPP) {
    const int p0 = __ldg(row_ptr + i), p1 = __ldg(row_ptr + i + 1);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int p = p0;
    for (; p + 1 < p1; p += 2) {
      const int j0 = __ldg(col_idx + p), j1 = __ldg(col_idx + p + 1);
      const float w0 = __ldg(vals + p), w1 = __ldg(vals + p + 1);
      const float4 a = *reinterpret_cast<const float4*>(xs + j0 * LDX + q * 4);
      const float4 b = *reinterpret_cast<const float4*>(xs + j1 * LDX + q * 4);
      acc.x = __fadd_rn(acc.x, __fmul_rn(w0, a.x));
      acc.y = __fadd_rn(acc.y, __fmul_rn(w0, a.y));
      acc.z = __fadd_rn(acc.z, __fmul_rn(w0, a.z));
      acc.w = __fadd_rn(acc.w, __fmul_rn(w0, a.w));
      acc.x = __fadd_rn(acc.x, __fmul_rn(w1, b.x));
      acc.y = __fadd_rn(acc.y, __fmul_rn(w1, b.y));
      acc.z = __fadd_rn(acc.z, __fmul_rn(w1, b.z));
      acc.w = __fadd_rn(acc.w, __fmul_rn(w1, b.w));
    }
    if (p < p1) {
      const int j0 = __ldg(col_idx + p);
      const float w0 = __ldg(vals + p);
      const float4 a = *reinterpret_cast<const float4*>(xs + j0 * LDX + q * 4);
      acc.x = __fadd_rn(acc.x, __fmul_rn(w0, a.x));
      acc.y = __fadd_rn(acc.y, __fmul_rn(w0, a.y));
      acc.z = __fadd_rn(acc.z, __fmul_rn(w0, a.z));
      acc.w = __fadd_rn(acc.w, __fmul_rn(w0, a.w));
    }
    *reinterpret_cast<float4*>(y + (size_t)i * ld + c0 + q * 4) = acc;
  }
}

// reference: one thread per output element, same order
__global__ void spmm_ref(const int* row_ptr, const int* col_idx, const float* vals, int m,
                         const float* x, int ld, int n, float* y) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * n) return;
  const int i = (int)(e / n), t = (int)(e % n);
  float acc = 0.f;
  for (int p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
    acc = __fadd_rn(acc, __fmul_rn(vals[p], x[(size_t)col_idx[p] * ld + t]));
  y[(size_t)i * ld + t] = acc;
}

static float* g_flush = nullptr;
static bool g_flushed = false;
template <typename F>
float time_us(F f, int reps = 50) {
  if (g_flushed) {  // L2 flushed before every launch, each launch timed alone
    if (!g_flush) CK(cudaMalloc(&g_flush, 512u << 20));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) f();
    float tot = 0.f;
    for (int i = 0; i < 20; ++i) {
      CK(cudaMemsetAsync(g_flush, i, 512u << 20));
      CK(cudaEventRecord(a));
      f();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      tot += ms;
    }
    CK(cudaGetLastError());
    return tot * 1e3f / 20;
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  return ms * 1e3f / reps;
}

struct Shape {
  const char* name;
  int m, k, r;
};

template <int BS, int TH>
void run(const Shape& s, const int* rp, const int* ci, const float* v, const float* x, float* y,
         const float* yref, int n, int rs) {
  constexpr int LDX = BS + ((BS == 32 || BS == 4) ? 0 : 4);
  const size_t smem = (size_t)s.k * LDX * 4;
  if (smem > 227 * 1024) return;
  auto kern = spmm_slice<BS, TH>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (n / BS) * rs;
  CK(cudaMemset(y, 0, (size_t)s.m * n * 4));
  const float us = time_us([&] { kern<<<grid, TH, smem>>>(rp, ci, v, s.m, s.k, x, n, y, rs); });
  // exact compare
  std::vector<float> a((size_t)s.m * n), b((size_t)s.m * n);
  CK(cudaMemcpy(a.data(), y, a.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), yref, b.size() * 4, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (size_t i = 0; i < a.size(); ++i) bad += memcmp(&a[i], &b[i], 4) != 0;
  printf("  slice BS=%2d th=%d rs=%d grid=%4d smem=%3zu KB: %8.2f us  mismatches %zu\n", BS, TH,
         rs, grid, smem / 1024, us, bad);
}

int main(int argc, char** argv) {
  // optional: m k r n [flushed]  (e.g. the config-3 point 8192 8192 8 512 1)
  const int n = argc >= 5 ? atoi(argv[4]) : 1024;
  g_flushed = argc >= 6 && atoi(argv[5]) != 0;
  std::vector<Shape> shapes;
  if (argc >= 5) {
    shapes.push_back({"argv", atoi(argv[1]), atoi(argv[2]), atoi(argv[3])});
  } else {
    shapes = {{"c2.L0 1024x3072 r24", 1024, 3072, 24},
                    {"c2.L1 512x1024 r18", 512, 1024, 18},
                    {"c2.L2 10x512 r312", 10, 512, 312},
                    {"c4.L1 8192x8192 r69", 8192, 8192, 69},
                    {"c4.L0 8192x3072 r47", 8192, 3072, 47}};
  }
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  for (const Shape& s : shapes) {
    std::vector<int> rp(s.m + 1), ci;
    std::vector<int> cols(s.k);
    for (int c = 0; c < s.k; ++c) cols[c] = c;
    for (int i = 0; i < s.m; ++i) {
      std::shuffle(cols.begin(), cols.end(), rng);
      std::vector<int> row(cols.begin(), cols.begin() + s.r);
      std::sort(row.begin(), row.end());
      for (int c : row) ci.push_back(c);
      rp[i + 1] = (int)ci.size();
    }
    const int nnz = (int)ci.size();
    std::vector<float> hv(nnz), hx((size_t)s.k * n);
    for (auto& f : hv) f = nd(rng);
    for (auto& f : hx) f = nd(rng);
    int *d_rp, *d_ci;
    float *d_v, *d_x, *d_y, *d_yref;
    CK(cudaMalloc(&d_rp, rp.size() * 4));
    CK(cudaMalloc(&d_ci, ci.size() * 4));
    CK(cudaMalloc(&d_v, hv.size() * 4));
    CK(cudaMalloc(&d_x, hx.size() * 4));
    CK(cudaMalloc(&d_y, (size_t)s.m * n * 4));
    CK(cudaMalloc(&d_yref, (size_t)s.m * n * 4));
    CK(cudaMemcpy(d_rp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), ci.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_v, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_x, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
    const int64_t tot = (int64_t)s.m * n;
    spmm_ref<<<(unsigned)((tot + 255) / 256), 256>>>(d_rp, d_ci, d_v, s.m, d_x, n, n, d_yref);
    CK(cudaDeviceSynchronize());
    printf("%s nnz=%d (x-gather %.1f MB)\n", s.name, nnz, nnz * 4.0 * n / 1e6);
    for (int rs : {1, 2, 4}) {
      run<4, 512>(s, d_rp, d_ci, d_v, d_x, d_y, d_yref, n, rs);
      run<4, 1024>(s, d_rp, d_ci, d_v, d_x, d_y, d_yref, n, rs);
      run<4, 256>(s, d_rp, d_ci, d_v, d_x, d_y, d_yref, n, rs);
      run<8, 256>(s, d_rp, d_ci, d_v, d_x, d_y, d_yref, n, rs);
      run<16, 256>(s, d_rp, d_ci, d_v, d_x, d_y, d_yref, n, rs);
      run<32, 256>(s, d_rp, d_ci, d_v, d_x, d_y, d_yref, n, rs);
      run<16, 512>(s, d_rp, d_ci, d_v, d_x, d_y, d_yref, n, rs);
    }
    cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_v); cudaFree(d_x); cudaFree(d_y); cudaFree(d_yref);
  }
  return 0;
}
