// Pattern handle: device validation of the CSR structure
// (tensor_core._validate_structure, tensor_core.py:78-94), a deterministic
// CSR -> CSC transpose index (replaces the O(nblocks * nnz) rescan of
// _kernels.spmm_t_kernel, _kernels.py:40-59) and the SDDMM tile index.
#include <vector>

#include <cmath>

#include "pattern.cuh"

namespace smb {
namespace {

// error bits of the validation kernel
enum : int {
  kBadRowPtrEnds = 1,
  kBadRowPtrOrder = 2,
  kBadColRange = 4,
  kBadColOrder = 8,
};

__global__ void validate_kernel(const int32_t* row_ptr, const int32_t* col_idx, int64_t m,
                                int64_t k, int64_t nnz, int* flags) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int32_t a = row_ptr[i], b = row_ptr[i + 1];
    if (b < a) { bad |= kBadRowPtrOrder; continue; }
    if (a < 0 || b > nnz) { bad |= kBadRowPtrEnds; continue; }
    int32_t prev = -1;
    for (int32_t p = a; p < b; ++p) {
      const int32_t c = col_idx[p];
      if (c < 0 || c >= k) bad |= kBadColRange;
      if (c <= prev) bad |= kBadColOrder;
      prev = c;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (row_ptr[0] != 0 || row_ptr[m] != nnz) bad |= kBadRowPtrEnds;
  }
  if (bad) atomicOr(flags, bad);
}

__global__ void count_cols_kernel(const int32_t* col_idx, int64_t nnz, int32_t* counts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += stride)
    atomicAdd(&counts[col_idx[p]], 1);
}

// Single-block exclusive scan: out[0] = 0, out[i+1] = sum(in[0..i]).
__global__ void exclusive_scan_kernel(const int32_t* in, int64_t n, int32_t* out) {
  __shared__ int64_t partial[1024];
  const int tid = threadIdx.x;
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t lo = imin(n, tid * per), hi = imin(n, lo + per);
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += in[i];
  partial[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int64_t v = partial[i];
      partial[i] = run;
      run += v;
    }
  }
  __syncthreads();
  int64_t run = partial[tid];
  if (tid == 0) out[0] = 0;
  for (int64_t i = lo; i < hi; ++i) {
    run += in[i];
    out[i + 1] = (int32_t)run;
  }
}

__global__ void scatter_csc_kernel(const int32_t* row_ptr, const int32_t* col_idx, int64_t m,
                                   const int32_t* col_ptr, int32_t* cursor, int32_t* tmp_row,
                                   int32_t* tmp_perm) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int32_t c = col_idx[p];
      const int32_t slot = col_ptr[c] + atomicAdd(&cursor[c], 1);
      tmp_row[slot] = (int32_t)i;
      tmp_perm[slot] = p;
    }
  }
}

// One warp per column: the atomic scatter left each column's entries in
// arbitrary order; place entry e at (#entries with a smaller row).  Rows are
// unique inside a column, so the result is the ascending-row order the
// reference's spmm_t accumulation follows, independent of scheduling.
__global__ void rank_sort_columns_kernel(const int32_t* col_ptr, int64_t k, const int32_t* tmp_row,
                                         const int32_t* tmp_perm, int32_t* row_idx,
                                         int32_t* perm) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < k;
       c += warps) {
    const int32_t a = col_ptr[c], b = col_ptr[c + 1];
    for (int32_t e = a + lane; e < b; e += 32) {
      const int32_t r = tmp_row[e];
      int32_t rank = 0;
      for (int32_t f = a; f < b; ++f) rank += (tmp_row[f] < r);
      row_idx[a + rank] = r;
      perm[a + rank] = tmp_perm[e];
    }
  }
}

__global__ void tile_rows_kernel(const int32_t* row_ptr, int64_t m, int64_t ngrains,
                                 int32_t* tile_row0) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ngrains) return;
  const int64_t p = t * kTileGrain;
  // last row i with row_ptr[i] <= p (skips empty rows)
  int64_t lo = 0, hi = m;  // invariant: row_ptr[lo] <= p < row_ptr[hi] (row_ptr[m] = nnz > p)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (row_ptr[mid] <= p) lo = mid; else hi = mid;
  }
  tile_row0[t] = (int32_t)lo;
}

int grid_for(int64_t work, int threads) {
  int64_t b = ceil_div(work, threads);
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return (int)b;
}

void free_pattern(smb_pattern* p) {
  if (!p) return;
  cudaFree(p->col_ptr);
  cudaFree(p->row_idx);
  cudaFree(p->perm);
  cudaFree(p->tile_row0);
  cudaFree(p->ord_p);
  cudaFree(p->ord_row);
  cudaFree(p->acc_ws);
  delete p;
}

}  // namespace
}  // namespace smb

using namespace smb;

extern "C" int smb_pattern_create(const int32_t* row_ptr, const int32_t* col_idx, int64_t m,
                                  int64_t k, int64_t nnz, int validate, void* stream,
                                  smb_pattern** out) {
  clear_error();
  SMB_REQUIRE(out != nullptr, "smb_pattern_create: null output handle");
  *out = nullptr;
  SMB_REQUIRE(m >= 0 && k >= 0 && nnz >= 0, "matrix dimensions must be non-negative");
  SMB_REQUIRE(m < (int64_t(1) << 31) && k < (int64_t(1) << 31) && nnz < (int64_t(1) << 31),
              "dimensions and nnz must stay below 2**31 (32-bit indices)");
  SMB_REQUIRE(row_ptr != nullptr && (nnz == 0 || col_idx != nullptr),
              "smb_pattern_create: null index array");
  cudaStream_t st = as_stream(stream);
  smb_pattern* p = new smb_pattern();
  p->m = m;
  p->k = k;
  p->nnz = nnz;
  p->row_ptr = row_ptr;
  p->col_idx = col_idx;
  p->ntiles = ceil_div(nnz, kSddmmTile);
  p->ngrains = ceil_div(nnz, kTileGrain);

  auto fail_cuda = [&](const char* what) {
    set_error("smb_pattern_create: %s: %s", what, cudaGetErrorString(cudaGetLastError()));
    free_pattern(p);
    return SMB_ERR_CUDA;
  };

  if (validate) {
    int* d_flags = nullptr;
    if (cudaMalloc(&d_flags, sizeof(int)) != cudaSuccess) return fail_cuda("cudaMalloc");
    cudaMemsetAsync(d_flags, 0, sizeof(int), st);
    validate_kernel<<<grid_for(m, 256), 256, 0, st>>>(row_ptr, col_idx, m, k, nnz, d_flags);
    int flags = 0;
    cudaMemcpyAsync(&flags, d_flags, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d_flags);
    count_launches(1);
    if (e != cudaSuccess) return fail_cuda("validation");
    if (flags) {
      free_pattern(p);
      if (flags & kBadRowPtrEnds) set_error("row_ptr must start at 0 and end at nnz");
      else if (flags & kBadRowPtrOrder) set_error("row_ptr must be non-decreasing");
      else if (flags & kBadColRange) set_error("column indices out of range");
      else set_error("column indices must be strictly increasing within each row");
      return SMB_ERR_INVALID;
    }
  }

  if (cudaMalloc(&p->col_ptr, sizeof(int32_t) * (k + 1)) != cudaSuccess ||
      cudaMalloc(&p->row_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1)) != cudaSuccess ||
      cudaMalloc(&p->perm, sizeof(int32_t) * (nnz > 0 ? nnz : 1)) != cudaSuccess ||
      cudaMalloc(&p->tile_row0, sizeof(int32_t) * (p->ngrains > 0 ? p->ngrains : 1)) != cudaSuccess)
    return fail_cuda("cudaMalloc");

  int32_t *counts = nullptr, *tmp_row = nullptr, *tmp_perm = nullptr;
  if (cudaMalloc(&counts, sizeof(int32_t) * (k > 0 ? k : 1)) != cudaSuccess ||
      cudaMalloc(&tmp_row, sizeof(int32_t) * (nnz > 0 ? nnz : 1)) != cudaSuccess ||
      cudaMalloc(&tmp_perm, sizeof(int32_t) * (nnz > 0 ? nnz : 1)) != cudaSuccess) {
    cudaFree(counts); cudaFree(tmp_row); cudaFree(tmp_perm);
    return fail_cuda("cudaMalloc");
  }
  uint64_t launches = 0;
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * (k > 0 ? k : 1), st);
  if (nnz > 0) {
    count_cols_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(col_idx, nnz, counts);
    ++launches;
  }
  exclusive_scan_kernel<<<1, 1024, 0, st>>>(counts, k, p->col_ptr);
  ++launches;
  if (nnz > 0) {
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * (k > 0 ? k : 1), st);
    scatter_csc_kernel<<<grid_for(m, 128), 128, 0, st>>>(row_ptr, col_idx, m, p->col_ptr, counts,
                                                          tmp_row, tmp_perm);
    rank_sort_columns_kernel<<<grid_for(k * 32, 256), 256, 0, st>>>(p->col_ptr, k, tmp_row,
                                                                      tmp_perm, p->row_idx,
                                                                      p->perm);
    tile_rows_kernel<<<(unsigned)ceil_div(p->ngrains, 256), 256, 0, st>>>(row_ptr, m, p->ngrains,
                                                                          p->tile_row0);
    launches += 3;
  }
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(counts);
  cudaFree(tmp_row);
  cudaFree(tmp_perm);
  count_launches(launches);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return fail_cuda("index build");
  if (nnz > 0) {
    // row spans of 32- .. 512-nonzero tiles: the tile of grains [g, g + G)
    // covers rows tile_row0[g] .. row of its last nonzero <= tile_row0[g + G]
    // (or m - 1)
    const int64_t ng = p->ngrains;
    std::vector<int32_t> t0(ng);
    if (cudaMemcpy(t0.data(), p->tile_row0, sizeof(int32_t) * ng, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
      return fail_cuda("tile index readback");
    auto span = [&](int64_t grains) {
      int64_t s = 0;
      for (int64_t g = 0; g < ng; g += grains) {
        const int64_t last = (g + grains < ng) ? t0[g + grains] : m - 1;
        s = imax(s, last - t0[g] + 1);
      }
      return s;
    };
    p->span32 = span(1);
    p->span64 = span(64 / kTileGrain);
    p->span128 = span(128 / kTileGrain);
    p->span512 = span(512 / kTileGrain);
  }
  if (m >= kBlockedMinDim && k >= kBlockedMinDim && nnz >= 4 * kBlockNnz) {
    // L2-blocked order: b x b (row band, column band) blocks of ~kBlockNnz
    // nonzeros (about one wave of resident SDDMM warps), stable counting sort
    // of the CSR order by block
    std::vector<int32_t> rp(m + 1), ci(nnz);
    if (cudaMemcpy(rp.data(), row_ptr, sizeof(int32_t) * (m + 1), cudaMemcpyDeviceToHost) !=
            cudaSuccess ||
        cudaMemcpy(ci.data(), col_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost) !=
            cudaSuccess)
      return fail_cuda("blocked order readback");
    // (measured at config 5, B = 4096: 3 / 4 / 5 / 7 / 10 bands -> 6.27 / 6.05 /
    // 6.05 / 6.16 / 9.56 ms; CSR order 7.02 ms)
    const int b = (int)imin(16, imax(2, llround(std::sqrt((double)nnz / (double)kBlockNnz))));
    const int nblk = b * b;
    std::vector<int64_t> start(nblk + 1, 0);
    auto block_of = [&](int64_t r, int64_t c) {
      return (int)((r * b) / m) * b + (int)((c * b) / k);
    };
    for (int64_t r = 0; r < m; ++r)
      for (int32_t q = rp[r]; q < rp[r + 1]; ++q) start[block_of(r, ci[q]) + 1]++;
    for (int i = 0; i < nblk; ++i) start[i + 1] += start[i];
    std::vector<int32_t> op(nnz), orow(nnz);
    for (int64_t r = 0; r < m; ++r)
      for (int32_t q = rp[r]; q < rp[r + 1]; ++q) {
        const int64_t dst = start[block_of(r, ci[q])]++;
        op[dst] = q;
        orow[dst] = (int32_t)r;
      }
    if (cudaMalloc(&p->ord_p, sizeof(int32_t) * nnz) != cudaSuccess ||
        cudaMalloc(&p->ord_row, sizeof(int32_t) * nnz) != cudaSuccess ||
        cudaMalloc(&p->acc_ws, sizeof(float) * nnz) != cudaSuccess ||
        cudaMemcpy(p->ord_p, op.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaMemcpy(p->ord_row, orow.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice) !=
            cudaSuccess)
      return fail_cuda("blocked order");
    p->bands = b;
  }
  *out = p;
  return SMB_OK;
}

extern "C" int smb_pattern_destroy(smb_pattern* p) {
  clear_error();
  free_pattern(p);
  return SMB_OK;
}

extern "C" int smb_pattern_csc(const smb_pattern* p, int32_t* col_ptr, int32_t* row_idx,
                               int32_t* perm, void* stream) {
  clear_error();
  SMB_REQUIRE(p != nullptr, "smb_pattern_csc: null handle");
  cudaStream_t st = as_stream(stream);
  if (col_ptr)
    cudaMemcpyAsync(col_ptr, p->col_ptr, sizeof(int32_t) * (p->k + 1), cudaMemcpyDeviceToDevice, st);
  if (row_idx && p->nnz)
    cudaMemcpyAsync(row_idx, p->row_idx, sizeof(int32_t) * p->nnz, cudaMemcpyDeviceToDevice, st);
  if (perm && p->nnz)
    cudaMemcpyAsync(perm, p->perm, sizeof(int32_t) * p->nnz, cudaMemcpyDeviceToDevice, st);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("smb_pattern_csc: %s", cudaGetErrorString(e));
    return SMB_ERR_CUDA;
  }
  return SMB_OK;
}
