// cp.async (LDGSTS) helpers shared by the staged-ring kernels (sm_100a).
#pragma once
#include "common.cuh"

namespace smb {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(gmem));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(unsigned dst, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(dst), "l"(gmem),
               "n"(BYTES), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Staged rows of the cp.async rings: unpadded lines of LDS elements (a
// multiple of 128 bytes) starting on 128-byte boundaries, 16-byte vector v of
// row r at slot v ^ (r & 7).  Threads reading 16 bytes of their own rows are
// then bank-conflict free, and a warp's 128-byte row copy lands in one smem
// line (a padded 144-byte row straddles two, and the LSU splits the copy:
// 1.5x the L2 sectors, measured with ncu).
template <int LDS, int VW>
__device__ __forceinline__ int swz(int r, int v) {
  return r * LDS + ((v ^ (r & 7)) * VW);
}
// first 128-byte boundary of the dynamic shared memory (allocations add 128)
__device__ __forceinline__ unsigned char* align128(unsigned char* p) {
  return p + ((128u - (smem_u32(p) & 127u)) & 127u);
}

// 16-byte shared-memory read as a volatile asm: a batch of these stays a
// batch (ptxas otherwise sinks each read next to its first use to save
// registers, exposing the LDS latency once per vector)
__device__ __forceinline__ float4 lds16(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ double2 lds16(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

// Copy `bytes` (<= 16) of a 16-byte vector; VEC: one cp.async with zero fill,
// else element-wise (unaligned operands).
template <typename T, bool VEC>
__device__ __forceinline__ void copy_vec(unsigned dst, const T* src, int valid_elems) {
  constexpr int VW = 16 / sizeof(T);
  if constexpr (VEC) {
    cp_async16(dst, src, valid_elems * (int)sizeof(T));
  } else {
#pragma unroll
    for (int j = 0; j < VW; ++j)
      cp_async_small<sizeof(T)>(dst + j * sizeof(T), j < valid_elems ? src + j : src,
                                j < valid_elems ? (int)sizeof(T) : 0);
  }
}

}  // namespace smb
