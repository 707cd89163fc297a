// L2 -> SM bandwidth on this GPU (standalone; writes JSON to stdout).
//   stream : coalesced 16-byte loads over a 64 MB buffer that stays in L2
//   rows128: each warp reads whole 128-byte row segments of random rows of a
//            (8 independent loads in flight per thread)
//            32 MB [8192 x 1024] fp32 matrix (the SpMM / SDDMM gather shape)
//   rows64 : the same with 64-byte segments
// Every variant reads the buffer a few times per launch; the first launch
// warms L2, the timed ones are back to back.  Bytes = bytes requested by the
// SMs (sector granular), so the result is the L2 -> SM delivery rate.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/l2_peak.cu -o /tmp/l2_peak
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void stream_kernel(const float4* __restrict__ a, size_t n4, int reps, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldcg(a + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 123.456f) out[0] = acc;
}

// SEG bytes per row segment; a warp reads 512 / SEG segments per instruction.
// UNR independent loads per thread are in flight per iteration (the
// addresses never depend on loaded data), so the rate is not latency-bound.
template <int SEG, int UNR>
__global__ void rows_kernel(const float* __restrict__ x, int rows, int ld, int iters,
                            const int* __restrict__ perm, float* out) {
  constexpr int LPS = SEG / 16;  // lanes per segment
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  unsigned r = (unsigned)perm[gw % rows];
  const int seg = lane / LPS;
  for (int it = 0; it < iters; it += UNR) {
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      // 32 / LPS segments per warp-instruction, each from a pseudo-random row
      const unsigned ru = r * (2654435761u * (u + 1)) + 977u * seg;
      const int row = (int)(ru % (unsigned)rows);
      const int col = (((it + u) * 7 + seg) % (ld * 4 / SEG)) * (SEG / 4) + (lane % LPS) * 4;
      v[u] = __ldcg(reinterpret_cast<const float4*>(x + (size_t)row * ld + col));
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    r = r * 1103515245u + 12345u;
  }
  if (acc == 123.456f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  // stream
  const size_t n = 16u << 20;  // 64 MB
  float4* buf;
  cudaMalloc(&buf, n * 4);
  cudaMemset(buf, 0, n * 4);
  const int reps = 8;
  stream_kernel<<<148 * 8, 256>>>(buf, n / 4, reps, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stream_kernel<<<148 * 8, 256>>>(buf, n / 4, reps, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double stream_gbs = 5.0 * reps * n * 4 / (ms * 1e-3) / 1e9;
  // gathers
  const int rows = 8192, ld = 1024;
  float* x;
  cudaMalloc(&x, (size_t)rows * ld * 4);
  cudaMemset(x, 0, (size_t)rows * ld * 4);
  int* perm;
  cudaMalloc(&perm, rows * 4);
  int* hp = new int[rows];
  for (int i = 0; i < rows; ++i) hp[i] = (int)((i * 2654435761u) % rows);
  cudaMemcpy(perm, hp, rows * 4, cudaMemcpyHostToDevice);
  const int iters = 2048, blocks = 148 * 8, threads = 256;
  const double gather_bytes = 5.0 * (double)blocks * threads * iters * 16;
  double g128, g64;
  rows_kernel<128, 8><<<blocks, threads>>>(x, rows, ld, iters, perm, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) rows_kernel<128, 8><<<blocks, threads>>>(x, rows, ld, iters, perm, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  g128 = gather_bytes / (ms * 1e-3) / 1e9;
  rows_kernel<64, 8><<<blocks, threads>>>(x, rows, ld, iters, perm, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) rows_kernel<64, 8><<<blocks, threads>>>(x, rows, ld, iters, perm, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  g64 = gather_bytes / (ms * 1e-3) / 1e9;
  cudaError_t e = cudaGetLastError();
  printf("{\"l2_stream_gbs\": %.1f, \"l2_gather_rows128_gbs\": %.1f, \"l2_gather_rows64_gbs\": %.1f, "
         "\"note\": \"L2-resident buffers (64 MB stream, 32 MB matrix), ld.global.cg, "
         "148x8 CTAs x 256 threads, back-to-back launches\", \"cuda\": \"%s\"}\n",
         stream_gbs, g128, g64, cudaGetErrorString(e));
  return 0;
}
