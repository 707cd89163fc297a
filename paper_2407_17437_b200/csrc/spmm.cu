// Row-split CSR SpMM (forward) and CSC SpMM (transposed) for sm_100a.
//
// Both products have the same shape of work: every output row r is
//     out[r, :] = sum_{s in segment(r), ascending} val(s) * dense[idx(s), :]
// with (segment, idx, val) = (CSR row, col_idx, values) for Y = W X
// (_kernels.py:25-37) and (CSC column, row_idx, values[perm]) for dX = W^T dY
// (_kernels.py:40-59; ascending source row == the reference's row-order scan).
//
// Mapping: one warp owns (output row, 32*W-column chunk of the batch); each
// lane owns W consecutive batch columns and keeps them in registers for the
// whole segment, so accumulation order per element is exactly the
// reference's (ascending s, mul and add rounded separately).  The warp reads
// 32 (idx, val) pairs with one coalesced load and broadcasts them with
// shuffles; the dense rows are gathered as 512-byte coalesced vectors
// through the read-only path, U rows in flight per warp.
#include "pattern.cuh"

namespace smb {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kUnroll = 8;

template <typename T, int W>
struct Frag {
  T v[W];
};

template <typename T, int W>
__device__ __forceinline__ void load_frag(Frag<T, W>& f, const T* p, int valid) {
  if constexpr (W > 1) {
    using V = typename Vec16<T>::type;
    static_assert(sizeof(V) == W * sizeof(T), "vector width");
    if (valid == W) {
      V v = ldg_vec(reinterpret_cast<const V*>(p));
#pragma unroll
      for (int j = 0; j < W; ++j) f.v[j] = VecOps<T>::get(v, j);
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < W; ++j) f.v[j] = (j < valid) ? __ldg(p + j) : T(0);
}

template <typename T, int W>
__device__ __forceinline__ void store_frag(const Frag<T, W>& f, T* p, int valid) {
  if constexpr (W > 1) {
    using V = typename Vec16<T>::type;
    if (valid == W) {
      V v;
#pragma unroll
      for (int j = 0; j < W; ++j) VecOps<T>::set(v, j, f.v[j]);
      *reinterpret_cast<V*>(p) = v;
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < W; ++j)
    if (j < valid) p[j] = f.v[j];
}

enum EpiKind { kEpiBiasAct = 0, kEpiMask = 1 };

template <typename T>
struct EpiArgs {
  const T* bias;   // kEpiBiasAct: per-row bias or null
  int relu;        // kEpiBiasAct: apply np.maximum(y, 0)
  const T* mask;   // kEpiMask: out *= (mask > 0), or null
  int64_t ld_mask;
};

template <typename T, int W, int EPI, bool PERM>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    segment_spmm_kernel(const int32_t* __restrict__ seg_ptr, const int32_t* __restrict__ idx,
                        const int32_t* __restrict__ perm, const T* __restrict__ vals,
                        int64_t n_rows, const T* __restrict__ dense, int64_t ld_dense,
                        int64_t n, int64_t n_chunks, T* __restrict__ out, int64_t ld_out,
                        EpiArgs<T> epi) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (gw >= n_rows * n_chunks) return;
  const int64_t row = gw / n_chunks;
  const int64_t chunk = gw - row * n_chunks;
  const int64_t col0 = chunk * (32 * W) + (int64_t)lane * W;
  const int valid = (int)imax(0, imin(W, n - col0));

  Frag<T, W> acc;
#pragma unroll
  for (int j = 0; j < W; ++j) acc.v[j] = T(0);

  const int32_t s_begin = seg_ptr[row];
  const int32_t s_end = seg_ptr[row + 1];
  const T* dcol = dense + col0;

  for (int32_t s0 = s_begin; s0 < s_end; s0 += 32) {
    const int cnt = min(32, s_end - s0);
    int my_idx = 0;
    T my_val = T(0);
    if (lane < cnt) {
      my_idx = idx[s0 + lane];
      my_val = PERM ? vals[perm[s0 + lane]] : vals[s0 + lane];
    }
    for (int q = 0; q < cnt; q += kUnroll) {
      Frag<T, W> xs[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int src = __shfl_sync(0xffffffffu, my_idx, (q + u) & 31);
        if (q + u < cnt && valid > 0) load_frag<T, W>(xs[u], dcol + (int64_t)src * ld_dense, valid);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const T v = __shfl_sync(0xffffffffu, my_val, (q + u) & 31);
        if (q + u < cnt) {
#pragma unroll
          for (int j = 0; j < W; ++j) acc.v[j] = add_rn(acc.v[j], mul_rn(v, xs[u].v[j]));
        }
      }
    }
  }
  if (valid == 0) return;

  if constexpr (EPI == kEpiBiasAct) {
    if (epi.bias != nullptr) {
      const T b = epi.bias[row];
#pragma unroll
      for (int j = 0; j < W; ++j) acc.v[j] = add_rn(acc.v[j], b);
    }
    if (epi.relu) {
#pragma unroll
      for (int j = 0; j < W; ++j) acc.v[j] = relu_np(acc.v[j]);
    }
  } else {
    if (epi.mask != nullptr) {
      Frag<T, W> mk;
      load_frag<T, W>(mk, epi.mask + row * epi.ld_mask + col0, valid);
#pragma unroll
      for (int j = 0; j < W; ++j) acc.v[j] = mask_np(acc.v[j], mk.v[j]);
    }
  }
  store_frag<T, W>(acc, out + row * ld_out + col0, valid);
}

template <typename T, int EPI, bool PERM>
int launch_segment_spmm(const int32_t* seg_ptr, const int32_t* idx, const int32_t* perm,
                        const T* vals, int64_t n_rows, const T* dense, int64_t ld_dense,
                        int64_t n, T* out, int64_t ld_out, EpiArgs<T> epi, cudaStream_t st,
                        const char* name) {
  if (n_rows == 0 || n == 0) return SMB_OK;
  constexpr int VW = Vec16<T>::N;
  const bool vec_ok = aligned16(dense) && aligned16(out) && ld_dense % VW == 0 &&
                      ld_out % VW == 0 &&
                      (EPI != kEpiMask || epi.mask == nullptr ||
                       (aligned16(epi.mask) && epi.ld_mask % VW == 0));
  // Wide vectors need enough warps to fill 148 SMs; with few rows or a
  // narrow batch use one column per lane so the work spreads over more warps.
  const bool wide = vec_ok && n_rows * ceil_div(n, 32 * VW) >= 148 * 16;
  if (wide) {
    const int64_t n_chunks = ceil_div(n, 32 * VW);
    const int64_t warps = n_rows * n_chunks;
    const int64_t blocks = ceil_div(warps, kWarpsPerBlock);
    segment_spmm_kernel<T, VW, EPI, PERM><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, st>>>(
        seg_ptr, idx, perm, vals, n_rows, dense, ld_dense, n, n_chunks, out, ld_out, epi);
  } else {
    const int64_t n_chunks = ceil_div(n, 32);
    const int64_t warps = n_rows * n_chunks;
    const int64_t blocks = ceil_div(warps, kWarpsPerBlock);
    segment_spmm_kernel<T, 1, EPI, PERM><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, st>>>(
        seg_ptr, idx, perm, vals, n_rows, dense, ld_dense, n, n_chunks, out, ld_out, epi);
  }
  return check_launch(name);
}

template <typename T>
int spmm_impl(const int32_t* row_ptr, const int32_t* col_idx, const void* values, int64_t m,
              int64_t k, const void* dense, int64_t ld_dense, int64_t n, const void* bias,
              int epilogue, void* out, int64_t ld_out, void* stream) {
  (void)k;
  EpiArgs<T> epi{static_cast<const T*>(bias), epilogue == SMB_EPI_RELU, nullptr, 0};
  return launch_segment_spmm<T, kEpiBiasAct, false>(
      row_ptr, col_idx, nullptr, static_cast<const T*>(values), m, static_cast<const T*>(dense),
      ld_dense, n, static_cast<T*>(out), ld_out, epi, as_stream(stream), "smb_spmm");
}

template <typename T>
int spmm_t_impl(const int32_t* col_ptr, const int32_t* row_idx, const int32_t* perm,
                const void* values, int64_t m, int64_t k, const void* dense, int64_t ld_dense,
                int64_t n, const void* mask, int64_t ld_mask, void* out, int64_t ld_out,
                void* stream) {
  (void)m;
  EpiArgs<T> epi{nullptr, 0, static_cast<const T*>(mask), ld_mask};
  return launch_segment_spmm<T, kEpiMask, true>(
      col_ptr, row_idx, perm, static_cast<const T*>(values), k, static_cast<const T*>(dense),
      ld_dense, n, static_cast<T*>(out), ld_out, epi, as_stream(stream), "smb_spmm_t");
}

}  // namespace
}  // namespace smb

using namespace smb;

extern "C" int smb_spmm(int dtype, const int32_t* row_ptr, const int32_t* col_idx,
                        const void* values, int64_t m, int64_t k, const void* dense,
                        int64_t ld_dense, int64_t n, const void* bias, int epilogue, void* out,
                        int64_t ld_out, void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 0 && k >= 0 && n >= 0, "smb_spmm: negative dimension");
  SMB_REQUIRE(ld_dense >= n && ld_out >= n, "smb_spmm: leading dimension smaller than n");
  SMB_REQUIRE(epilogue == SMB_EPI_NONE || epilogue == SMB_EPI_RELU, "smb_spmm: bad epilogue %d",
              epilogue);
  SMB_REQUIRE(m == 0 || (row_ptr && out), "smb_spmm: null pointer");
  if (dtype == SMB_F32)
    return spmm_impl<float>(row_ptr, col_idx, values, m, k, dense, ld_dense, n, bias, epilogue,
                            out, ld_out, stream);
  if (dtype == SMB_F64)
    return spmm_impl<double>(row_ptr, col_idx, values, m, k, dense, ld_dense, n, bias, epilogue,
                             out, ld_out, stream);
  set_error("smb_spmm: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}

extern "C" int smb_spmm_t(int dtype, const smb_pattern* pat, const void* values,
                          const void* dense, int64_t ld_dense, int64_t n, const void* mask,
                          int64_t ld_mask, void* out, int64_t ld_out, void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_spmm_t: null pattern");
  SMB_REQUIRE(n >= 0, "smb_spmm_t: negative dimension");
  SMB_REQUIRE(ld_dense >= n && ld_out >= n, "smb_spmm_t: leading dimension smaller than n");
  SMB_REQUIRE(mask == nullptr || ld_mask >= n, "smb_spmm_t: mask leading dimension");
  SMB_REQUIRE(pat->k == 0 || out != nullptr, "smb_spmm_t: null output");
  if (dtype == SMB_F32)
    return spmm_t_impl<float>(pat->col_ptr, pat->row_idx, pat->perm, values, pat->m, pat->k,
                              dense, ld_dense, n, mask, ld_mask, out, ld_out, stream);
  if (dtype == SMB_F64)
    return spmm_t_impl<double>(pat->col_ptr, pat->row_idx, pat->perm, values, pat->m, pat->k,
                               dense, ld_dense, n, mask, ld_mask, out, ld_out, stream);
  set_error("smb_spmm_t: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}
