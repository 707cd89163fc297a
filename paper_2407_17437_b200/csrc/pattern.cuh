// Device-side SparsityPattern (tensor_core.py:97-152): the static CSR
// structure shared by a layer's weights, gradient and velocity, plus the
// derived indices the kernels need, built once per layer.
#pragma once
#include "common.cuh"

struct smb_pattern {
  int64_t m = 0, k = 0, nnz = 0;
  const int32_t* row_ptr = nullptr;  // borrowed, [m+1]
  const int32_t* col_idx = nullptr;  // borrowed, [nnz]
  int32_t* col_ptr = nullptr;        // owned, [k+1]   CSC column pointers
  int32_t* row_idx = nullptr;        // owned, [nnz]   CSC rows, ascending per column
  int32_t* perm = nullptr;           // owned, [nnz]   CSC slot -> CSR value index
  int32_t* tile_row0 = nullptr;      // owned, [ngrains] row of nonzero g*kTileGrain
  int64_t ngrains = 0;               // ceil(nnz / kTileGrain)
  int64_t ntiles = 0;                // ceil(nnz / kSddmmTile)
  // most rows spanned by any tile of 32 / 64 / 128 / 512 consecutive nonzeros
  // (aligned; first row .. row of the last nonzero)
  int64_t span32 = 0, span64 = 0, span128 = 0, span512 = 0;
  // L2-blocked nonzero order for the SDDMM of very wide layers (m, k >= 16384):
  // the nonzeros grouped by (row band, column band) blocks of about one wave
  // of resident warps, CSR order inside a block (sddmm_tma.cu).  ord_p[q] is
  // the CSR index of the q-th nonzero in that order, ord_row[q] its row.
  int32_t* ord_p = nullptr;    // owned, [nnz] or null
  int32_t* ord_row = nullptr;  // owned, [nnz] or null
  float* acc_ws = nullptr;     // owned, [nnz] or null: chain sums carried between batch phases
  int bands = 0;
};

namespace smb {
constexpr int kSddmmTile = 128;  // nonzeros per SDDMM CTA (one per thread)
constexpr int kTileGrain = 32;   // granularity of the tile -> first-row table
constexpr int64_t kBlockedMinDim = 16384;  // layers that get the L2-blocked SDDMM order
constexpr int64_t kBlockNnz = 104000;      // ~ 148 SMs x 22 resident warps x 32 nonzeros
}

namespace smb {
// Row of nonzero p inside a tile starting at row r0, through a shared window
// s_rp[0..W] = row_ptr[r0 .. r0+W]; global binary search when the tile spans
// more than W rows (long runs of empty rows).
template <int W>
__device__ __forceinline__ int64_t tile_row_of(int64_t p, int32_t r0, const int32_t* s_rp,
                                               const int32_t* row_ptr, int64_t m) {
  if (p < (int64_t)s_rp[W]) {
    int lo = 0, hi = W;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)s_rp[mid] <= p) lo = mid; else hi = mid;
    }
    return r0 + lo;
  }
  int64_t lo = r0 + W, hi = m;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)row_ptr[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

// SDDMM + update with TMA gather4 staging (sddmm_tma.cu), fp32
bool sddmm_tma_supported(const smb_pattern* pat, const void* d_out, int64_t ld_d, const void* x,
                         int64_t ld_x, int64_t n);
int launch_sddmm_tma(const smb_pattern* pat, const float* d_out, int64_t ld_d, const float* x,
                     int64_t ld_x, int64_t n, const float* values, float* values_out,
                     float* velocity, float* grad_out, const OptConsts<float>& opt,
                     cudaStream_t st);
// the batch is so wide that x and d_out overflow L2 many times over: walk
// the nonzeros in the pattern's blocked order (when it has one)
bool sddmm_use_blocked_order(const smb_pattern* pat, int64_t n);
}  // namespace smb
