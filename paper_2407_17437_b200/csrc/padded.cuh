// Quad-padded sparse segments (host-side setup shared by the column-chain and
// panel kernels).
//
// A segment (a CSR row, or a CSC column) of s pairs is padded to a multiple of
// 4 with pads that point at an all-zero operand row and carry the value -0.0:
// a pad's product is -0.0 and acc + (-0.0) == acc bit for bit for every acc
// (-0.0 and NaN included), so kernels walk whole 16-byte quads of (index,
// value) pairs with no masks.  The padded values are a copy refreshed from the
// layer's values after every update (padded_refresh_kernel).
#pragma once
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace smb {

struct Padded {
  std::vector<int32_t> ptr;    // [segments + 1], multiples of 4
  std::vector<int32_t> idx;    // operand rows (pads: zero_row)
  std::vector<int32_t> src;    // source value index of every slot (-1: pad)
  std::vector<int32_t> order;  // per part: its segments, longest first
  std::vector<int32_t> split;  // [parts + 1]: segment ranges balanced by slots
};

// seg / idx: the CSR (or CSC) structure; value_of[s] = the value index of
// pair s (null: s itself)
inline Padded pad_segments(const std::vector<int32_t>& seg, const std::vector<int32_t>& idx,
                           const int32_t* value_of, int zero_row) {
  Padded out;
  const int rows = (int)seg.size() - 1;
  out.ptr.resize((size_t)rows + 1);
  out.ptr[0] = 0;
  for (int r = 0; r < rows; ++r) out.ptr[r + 1] = out.ptr[r] + ((seg[r + 1] - seg[r] + 3) & ~3);
  out.idx.assign((size_t)out.ptr[rows], zero_row);
  out.src.assign((size_t)out.ptr[rows], -1);
  for (int r = 0; r < rows; ++r)
    for (int s = seg[r]; s < seg[r + 1]; ++s) {
      out.idx[out.ptr[r] + (s - seg[r])] = idx[s];
      out.src[out.ptr[r] + (s - seg[r])] = value_of ? value_of[s] : s;
    }
  return out;
}

// `parts` contiguous segment ranges of about equal padded size, and within
// each the segments longest first (a warp's concurrent segments then end
// together)
inline void split_and_order(Padded& pd, int parts) {
  const int rows = (int)pd.ptr.size() - 1;
  const int64_t z = pd.ptr[rows];
  pd.split.assign((size_t)parts + 1, 0);
  for (int q = 1; q < parts; ++q) {
    const int64_t target = z * q / parts;
    const int r =
        (int)(std::lower_bound(pd.ptr.begin(), pd.ptr.end(), (int32_t)target) - pd.ptr.begin());
    pd.split[q] = std::max(pd.split[q - 1], std::min(r, rows));
  }
  pd.split[parts] = rows;
  pd.order.clear();
  for (int q = 0; q < parts; ++q) {
    std::vector<int32_t> rr;
    for (int r = pd.split[q]; r < pd.split[q + 1]; ++r) rr.push_back(r);
    std::stable_sort(rr.begin(), rr.end(), [&](int32_t a, int32_t b) {
      return pd.ptr[a + 1] - pd.ptr[a] > pd.ptr[b + 1] - pd.ptr[b];
    });
    pd.order.insert(pd.order.end(), rr.begin(), rr.end());
  }
}

template <typename T>
inline bool to_host(std::vector<T>& v, const T* d, int64_t n) {
  v.resize((size_t)n);
  return n == 0 || cudaMemcpy(v.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost) == cudaSuccess;
}

// pval[s] = values[src[s]], or -0.0 for a pad
__global__ void padded_refresh_kernel(const int32_t* __restrict__ src,
                                      const float* __restrict__ values, float* __restrict__ pval,
                                      int64_t n);

}  // namespace smb
