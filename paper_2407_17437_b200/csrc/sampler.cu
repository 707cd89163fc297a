// Seeded uniform sparsity-pattern sampler on the device (sm_100a) -- the
// "scale mode" counterpart of the reference's host sampler
// (sparsity.py:183-216: multivariate-hypergeometric row counts, then
// rng.choice of the columns of every row, sorted).  Both draw a pattern
// uniformly from all nnz-subsets of the m x k grid; the reference's exact
// numpy stream cannot be parallelised, so parity mode keeps the host sampler
// (bit-identical patterns) and this sampler defines its own stream:
//
//   u_i   = Philox4x32-10(key = seed, counter = (i, stream_id)), 64 bits
//   pos_i = floor(u_i * G / 2^64),  G = m * k grid positions
//   pattern = the first nnz DISTINCT positions of pos_0, pos_1, ...
//             (sequential sampling without replacement by rejection), or,
//             when nnz > G / 2, every position except the first G - nnz
//             distinct ones (the complement is the smaller draw)
//   row = pos / k, col = pos % k, CSR in row-major order.
//
// The result depends only on (m, k, nnz, seed, stream_id), not on launch
// shapes or on how many candidates were generated: the device draws
// N >= needed candidates, sorts (position, index) pairs, keeps the first
// index of every position, re-sorts the survivors by index and takes the
// first `needed`; if fewer than `needed` distinct positions came up, N grows
// and the same sequence is extended.  oracle/pattern_oracle.c restates this
// specification on the CPU (hash set over the same Philox stream) and the
// tests compare the two bit for bit.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace smb {
namespace {

__host__ __device__ __forceinline__ void philox_round(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
  c[0] = n0;
  c[1] = lo1;
  c[2] = n2;
  c[3] = lo0;
}

// 64 uniform bits for candidate i of stream `sid` under `seed`
__host__ __device__ __forceinline__ uint64_t philox_u64(uint64_t seed, uint64_t sid, uint64_t i) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)sid, (uint32_t)(sid >> 32)};
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ((uint64_t)c[1] << 32) | c[0];
}

__global__ void candidates_kernel(uint64_t seed, uint64_t sid, uint64_t grid_size, int64_t n,
                                  uint64_t* pos, uint64_t* idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    pos[i] = __umul64hi(philox_u64(seed, sid, (uint64_t)i), grid_size);
    idx[i] = (uint64_t)i;
  }
}

// first occurrence of each position in the position-sorted list (the radix
// sort is stable and the indices went in ascending, so the first of a run
// carries the smallest candidate index)
__global__ void first_flags_kernel(const uint64_t* pos, int64_t n, uint8_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    flag[i] = (i == 0 || pos[i] != pos[i - 1]) ? 1 : 0;
}

// sorted positions -> col_idx and per-row counts
__global__ void positions_to_csr_kernel(const uint64_t* pos, int64_t nnz, int64_t k,
                                        int32_t* col_idx, int32_t* row_count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const uint64_t p = pos[i];
    col_idx[i] = (int32_t)(p % (uint64_t)k);
    atomicAdd(&row_count[p / (uint64_t)k], 1);
  }
}

// complement mode: mark the excluded positions, then keep the rest
__global__ void mark_positions_kernel(const uint64_t* pos, int64_t n, uint8_t* excluded) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    excluded[pos[i]] = 1;
}

__global__ void invert_flags_kernel(uint8_t* f, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    f[i] = f[i] ? 0 : 1;
}

__global__ void iota_kernel(uint64_t* a, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    a[i] = (uint64_t)i;
}

int bits_for(uint64_t v) {  // bits needed to hold values < v
  int b = 1;
  while (b < 64 && (uint64_t(1) << b) < v) ++b;
  return b;
}

// a growing set of device buffers freed on scope exit
struct Scratch {
  std::vector<void*> ptrs;
  template <typename T>
  T* get(size_t count) {
    void* p = nullptr;
    if (cudaMalloc(&p, count * sizeof(T) + 16) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

unsigned grid_for(int64_t n) { return (unsigned)imax(1, imin(148 * 8, ceil_div(n, 256))); }

}  // namespace
}  // namespace smb

using namespace smb;

extern "C" uint64_t smb_philox_u64(uint64_t seed, uint64_t stream_id, uint64_t i) {
  return philox_u64(seed, stream_id, i);
}

extern "C" int smb_sample_pattern(int64_t m, int64_t k, int64_t nnz, uint64_t seed,
                                  uint64_t stream_id, int32_t* row_ptr, int32_t* col_idx,
                                  void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 0 && k >= 0 && nnz >= 0, "smb_sample_pattern: negative dimension");
  SMB_REQUIRE(m < (int64_t(1) << 31) && k < (int64_t(1) << 31),
              "smb_sample_pattern: dimension too large");
  const uint64_t G = (uint64_t)m * (uint64_t)k;
  SMB_REQUIRE((uint64_t)nnz <= G, "smb_sample_pattern: nnz exceeds the grid size");
  SMB_REQUIRE(nnz < (int64_t(1) << 31), "smb_sample_pattern: too many nonzeros");
  SMB_REQUIRE(row_ptr != nullptr && (nnz == 0 || col_idx != nullptr),
              "smb_sample_pattern: null output");
  cudaStream_t st = as_stream(stream);
  const bool complement = nnz > 0 && (uint64_t)nnz * 2 > G;
  // complement mode enumerates the grid (a byte per position)
  SMB_REQUIRE(!complement || G <= (uint64_t(1) << 32),
              "smb_sample_pattern: dense patterns need m * k <= 2^32");
  const int64_t need = complement ? (int64_t)(G - (uint64_t)nnz) : nnz;
  Scratch s;
  int32_t* counts = s.get<int32_t>((size_t)m + 1);
  if (!counts) return (set_error("smb_sample_pattern: out of memory"), SMB_ERR_CUDA);
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * (m + 1), st);
  uint64_t* chosen = nullptr;  // the `need` first distinct positions, ascending
  if (need > 0) {
    // candidates: the expected count that yields `need` distinct positions
    // (coupon-collector: -G ln(1 - need / G)) plus a margin; doubled if short
    const double g = (double)G, r = (double)need / g;
    double want = (r < 1e-6 ? (double)need * (1.0 + r) : -g * std::log1p(-r));
    int64_t n = (int64_t)(want * 1.02 + 8.0 * std::sqrt(want) + 64.0);
    const int pbits = bits_for(G);
    for (int attempt = 0;; ++attempt) {
      Scratch t;
      uint64_t* pos = t.get<uint64_t>(n);
      uint64_t* idx = t.get<uint64_t>(n);
      uint64_t* pos2 = t.get<uint64_t>(n);
      uint64_t* idx2 = t.get<uint64_t>(n);
      uint8_t* flag = t.get<uint8_t>(n);
      int64_t* n_distinct = t.get<int64_t>(1);
      if (!pos || !idx || !pos2 || !idx2 || !flag || !n_distinct)
        return (set_error("smb_sample_pattern: out of memory"), SMB_ERR_CUDA);
      candidates_kernel<<<grid_for(n), 256, 0, st>>>(seed, stream_id, G, n, pos, idx);
      size_t tb = 0, tb2 = 0, tb3 = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, pos, pos2, idx, idx2, n, 0, pbits, st);
      cub::DeviceSelect::Flagged(nullptr, tb2, idx2, flag, idx, n_distinct, n, st);
      cub::DeviceRadixSort::SortPairs(nullptr, tb3, idx, idx2, pos, pos2, n, 0, bits_for(n), st);
      void* tmp = t.get<uint8_t>(std::max(tb, std::max(tb2, tb3)));
      if (!tmp) return (set_error("smb_sample_pattern: out of memory"), SMB_ERR_CUDA);
      // (position, index) sorted by position; first index of every position
      cub::DeviceRadixSort::SortPairs(tmp, tb, pos, pos2, idx, idx2, n, 0, pbits, st);
      first_flags_kernel<<<grid_for(n), 256, 0, st>>>(pos2, n, flag);
      cub::DeviceSelect::Flagged(tmp, tb2, idx2, flag, idx, n_distinct, n, st);
      cub::DeviceSelect::Flagged(tmp, tb2, pos2, flag, pos, n_distinct, n, st);
      int64_t nd = 0;
      cudaMemcpyAsync(&nd, n_distinct, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess)
        return (set_error("smb_sample_pattern: %s", cudaGetErrorString(cudaGetLastError())),
                SMB_ERR_CUDA);
      if (nd >= need) {
        // survivors back in candidate order; the first `need` are the draw
        cub::DeviceRadixSort::SortPairs(tmp, tb3, idx, idx2, pos, pos2, nd, 0, bits_for(n), st);
        chosen = s.get<uint64_t>(need);
        size_t tb4 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb4, pos2, chosen, need, 0, pbits, st);
        void* tmp4 = t.get<uint8_t>(tb4);
        if (!chosen || !tmp4)
          return (set_error("smb_sample_pattern: out of memory"), SMB_ERR_CUDA);
        cub::DeviceRadixSort::SortKeys(tmp4, tb4, pos2, chosen, need, 0, pbits, st);
        if (cudaStreamSynchronize(st) != cudaSuccess)
          return (set_error("smb_sample_pattern: %s", cudaGetErrorString(cudaGetLastError())),
                  SMB_ERR_CUDA);
        break;
      }
      SMB_REQUIRE(attempt < 16, "smb_sample_pattern: candidate stream exhausted");
      n *= 2;  // extend the same candidate sequence
    }
  }
  if (!complement) {
    if (nnz > 0)
      positions_to_csr_kernel<<<grid_for(nnz), 256, 0, st>>>(chosen, nnz, k, col_idx, counts);
  } else {
    // keep every position the draw did not exclude
    uint8_t* keep = s.get<uint8_t>(G);
    uint64_t* all = s.get<uint64_t>(G);
    uint64_t* kept = s.get<uint64_t>(nnz);
    int64_t* nk = s.get<int64_t>(1);
    if (!keep || !all || !kept || !nk)
      return (set_error("smb_sample_pattern: out of memory"), SMB_ERR_CUDA);
    cudaMemsetAsync(keep, 0, G, st);
    if (need > 0) mark_positions_kernel<<<grid_for(need), 256, 0, st>>>(chosen, need, keep);
    invert_flags_kernel<<<grid_for((int64_t)G), 256, 0, st>>>(keep, (int64_t)G);
    iota_kernel<<<grid_for((int64_t)G), 256, 0, st>>>(all, (int64_t)G);
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, all, keep, kept, nk, (int64_t)G, st);
    void* tmp = s.get<uint8_t>(tb);
    if (!tmp) return (set_error("smb_sample_pattern: out of memory"), SMB_ERR_CUDA);
    cub::DeviceSelect::Flagged(tmp, tb, all, keep, kept, nk, (int64_t)G, st);
    positions_to_csr_kernel<<<grid_for(nnz), 256, 0, st>>>(kept, nnz, k, col_idx, counts);
  }
  // row_ptr = exclusive scan of the row counts (counts[m] = 0 -> row_ptr[m] = nnz)
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, row_ptr, m + 1, st);
  void* tmp = s.get<uint8_t>(tb);
  if (!tmp) return (set_error("smb_sample_pattern: out of memory"), SMB_ERR_CUDA);
  cub::DeviceScan::ExclusiveSum(tmp, tb, counts, row_ptr, m + 1, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return (set_error("smb_sample_pattern: %s", cudaGetErrorString(cudaGetLastError())),
            SMB_ERR_CUDA);
  return check_launch("smb_sample_pattern", 4);
}
