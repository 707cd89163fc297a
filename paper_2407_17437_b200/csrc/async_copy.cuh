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
