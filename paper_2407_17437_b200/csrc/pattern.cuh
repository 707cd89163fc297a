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
};

namespace smb {
constexpr int kSddmmTile = 128;  // nonzeros per SDDMM CTA (one per thread)
constexpr int kTileGrain = 32;   // granularity of the tile -> first-row table
}
