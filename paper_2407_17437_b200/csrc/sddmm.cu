// SDDMM weight gradient fused with the optimizer update (sm_100a).
//
// grad[p] = sum_t d_out[i, t] * x[j, t] for the p-th stored (i, j), summed
// sequentially over t with separately rounded multiply/add exactly like
// _kernels.sddmm_kernel (_kernels.py:62-75), then (optionally) the momentum /
// Nesterov / GD update of values and velocity in the sparse_combine order of
// SparseLinearLayer.optimize (nn.py:187-197).  Extra CTAs of the same launch
// compute grad_bias = row_sums(d_out) in numpy's pairwise order (nn.py:184)
// and update bias / velocity_bias (_step_vector, nn.py:118-131).  No dense
// m x k gradient and no mask is ever formed.
//
// Mapping: one CTA = 128 consecutive nonzeros (one per thread) of the CSR
// order; the batch is walked in 32-column chunks through a 3-stage cp.async
// pipeline that stages, per chunk, the 128 gathered x rows and the (few)
// d_out rows the tile touches.  Rows are padded to 32+16/sizeof(T) elements
// so each thread's 16-byte LDS of its own x row and the broadcast LDS of its
// d_out row are bank-conflict free.  Each thread runs one sequential
// accumulation chain (required for bit-exactness), 4 (fp32) columns per LDS.
#include "pattern.cuh"

namespace smb {
namespace {

constexpr int kTile = kSddmmTile;  // nonzeros per CTA == threads per CTA
constexpr int kChunk = 32;         // batch columns per pipeline stage
constexpr int kSlots = 32;         // staged d_out rows per tile
constexpr int kStages = 3;

template <typename T>
struct SddmmCfg {
  static constexpr int VW = 16 / sizeof(T);   // elements per 16 B
  static constexpr int LDS = kChunk + VW;     // padded smem row (elements)
  static constexpr int VPR = kChunk / VW;     // 16 B vectors per staged row
  static constexpr size_t stage_elems = size_t(kTile + kSlots) * LDS;
  static constexpr size_t smem_bytes = kStages * stage_elems * sizeof(T);
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Stage one 32-column chunk of a row (x row of a nonzero, or a d_out row).
template <typename T, bool VEC>
__device__ __forceinline__ void stage_row_part(T* dst_row, const T* src_row, int64_t t0, int64_t n,
                                               int v, bool row_valid) {
  using C = SddmmCfg<T>;
  if constexpr (VEC) {
    const int64_t c0 = t0 + (int64_t)v * C::VW;
    int valid = row_valid ? (int)imax(0, imin(C::VW, n - c0)) : 0;
    const T* src = valid > 0 ? src_row + c0 : src_row;
    cp_async16(dst_row + v * C::VW, src, valid * (int)sizeof(T));
  } else {
#pragma unroll
    for (int j = 0; j < C::VW; ++j) {
      const int64_t c = t0 + (int64_t)v * C::VW + j;
      const bool ok = row_valid && c < n;
      cp_async_small<sizeof(T)>(dst_row + v * C::VW + j, ok ? src_row + c : src_row,
                                ok ? (int)sizeof(T) : 0);
    }
  }
}

template <typename T>
__device__ void bias_rows(int64_t row0, int64_t m, const T* __restrict__ d_out, int64_t ld_d,
                          int64_t n, T* bias, T* vbias, T* grad_bias_out,
                          const OptConsts<T>& opt) {
  const int64_t row = row0 + threadIdx.x;
  if (row >= m) return;
  const T g = pairwise_sum(d_out + row * ld_d, n);
  if (grad_bias_out) grad_bias_out[row] = g;
  if (opt.kind != SMB_OPT_NONE && bias) {
    T dummy = T(0);
    apply_update(opt, g, bias + row, vbias ? vbias + row : &dummy);
  }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kTile)
    sddmm_update_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                        const int32_t* __restrict__ tile_row0, int64_t m, int64_t nnz,
                        int64_t nz_tiles, const T* __restrict__ d_out, int64_t ld_d,
                        const T* __restrict__ x, int64_t ld_x, int64_t n, T* values, T* velocity,
                        T* grad_out, T* bias, T* vbias, T* grad_bias_out, OptConsts<T> opt) {
  using C = SddmmCfg<T>;
  if ((int64_t)blockIdx.x >= nz_tiles) {
    bias_rows<T>(((int64_t)blockIdx.x - nz_tiles) * kTile, m, d_out, ld_d, n, bias, vbias,
                 grad_bias_out, opt);
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  __shared__ int32_t s_col[kTile];
  __shared__ int32_t s_rp[kTile + 1];

  const int tid = threadIdx.x;
  const int64_t p0 = (int64_t)blockIdx.x * kTile;
  const int64_t p = p0 + tid;
  const bool active = p < nnz;
  const int32_t r0 = tile_row0[blockIdx.x];

  // row of p: binary search in a shared window of row_ptr[r0 .. r0+kTile]
  s_col[tid] = active ? col_idx[p] : 0;
  s_rp[tid] = (r0 + tid <= m) ? row_ptr[r0 + tid] : INT32_MAX;
  if (tid == 0) s_rp[kTile] = (r0 + kTile <= m) ? row_ptr[r0 + kTile] : INT32_MAX;
  __syncthreads();
  int64_t row;
  if (p < (int64_t)s_rp[kTile]) {
    int lo = 0, hi = kTile;  // s_rp[lo] <= p < s_rp[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)s_rp[mid] <= p) lo = mid; else hi = mid;
    }
    row = r0 + lo;
  } else {  // tile spans more than kTile rows (empty rows): global search
    int64_t lo = r0 + kTile, hi = m;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)row_ptr[mid] <= p) lo = mid; else hi = mid;
    }
    row = lo;
  }
  const int slot = (int)imin(row - r0, kSlots);  // kSlots == "not staged"
  const int n_staged = (int)imin(kSlots, m - r0);

  const int64_t n_chunks = (n + kChunk - 1) / kChunk;
  auto issue = [&](int64_t ch) {
    T* xs = smem + (ch % kStages) * C::stage_elems;
    T* ds = xs + kTile * C::LDS;
    const int64_t t0 = ch * kChunk;
    for (int e = tid; e < kTile * C::VPR; e += kTile) {
      const int r = e / C::VPR, v = e % C::VPR;
      stage_row_part<T, VEC>(xs + r * C::LDS, x + (int64_t)s_col[r] * ld_x, t0, n, v,
                             p0 + r < nnz);
    }
    for (int e = tid; e < n_staged * C::VPR; e += kTile) {
      const int r = e / C::VPR, v = e % C::VPR;
      stage_row_part<T, VEC>(ds + r * C::LDS, d_out + (int64_t)(r0 + r) * ld_d, t0, n, v, true);
    }
  };

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < n_chunks) issue(s);
    cp_async_commit();
  }

  // -0.0 is the exact additive identity, so acc = -0 + a0*b0 == a0*b0 and the
  // chain below is the reference's  acc = a0*b0; acc += a_t*b_t  verbatim.
  T acc = T(-0.0);
  const T* drow = d_out + row * ld_d;
  for (int64_t ch = 0; ch < n_chunks; ++ch) {
    if (ch + kStages - 1 < n_chunks) issue(ch + kStages - 1);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncthreads();
    if (active) {
      const T* xs = smem + (ch % kStages) * C::stage_elems;
      const T* xr = xs + tid * C::LDS;
      const T* dr = xs + (kTile + slot) * C::LDS;
      const int64_t t0 = ch * kChunk;
      const int cnt = (int)imin(kChunk, n - t0);
      if (cnt == kChunk) {
#pragma unroll
        for (int v = 0; v < C::VPR; ++v) {
          using V = typename Vec16<T>::type;
          const V xv = *reinterpret_cast<const V*>(xr + v * C::VW);
          V dv;
          if (slot < kSlots) dv = *reinterpret_cast<const V*>(dr + v * C::VW);
          else {
#pragma unroll
            for (int j = 0; j < C::VW; ++j) VecOps<T>::set(dv, j, drow[t0 + v * C::VW + j]);
          }
#pragma unroll
          for (int j = 0; j < C::VW; ++j)
            acc = add_rn(acc, mul_rn(VecOps<T>::get(dv, j), VecOps<T>::get(xv, j)));
        }
      } else {
        for (int j = 0; j < cnt; ++j) {
          const T dv = slot < kSlots ? dr[j] : drow[t0 + j];
          acc = add_rn(acc, mul_rn(dv, xr[j]));
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if (!active) return;
  const T g = (n == 0) ? T(0) : acc;  // tensor_core.py:283-284: zero batch -> zeros
  if (grad_out) grad_out[p] = g;
  if (opt.kind != SMB_OPT_NONE) {
    T dummy = T(0);
    apply_update(opt, g, values + p, velocity ? velocity + p : &dummy);
  }
}

template <typename T>
int sddmm_update_impl(const smb_pattern* pat, const void* d_out, int64_t ld_d, const void* x,
                      int64_t ld_x, int64_t n, void* values, void* velocity, void* grad_out,
                      void* bias, void* vbias, void* grad_bias_out, int opt_kind, double mu,
                      double eta, void* stream, const char* name) {
  using C = SddmmCfg<T>;
  const OptConsts<T> opt = make_opt<T>(opt_kind, mu, eta);
  const bool want_bias = (grad_bias_out != nullptr) || (opt_kind != SMB_OPT_NONE && bias);
  const int64_t bias_tiles = want_bias ? ceil_div(pat->m, kTile) : 0;
  const int64_t grid = pat->ntiles + bias_tiles;
  if (grid == 0) return SMB_OK;
  const bool vec = aligned16(x) && aligned16(d_out) && ld_x % C::VW == 0 && ld_d % C::VW == 0;
  cudaStream_t st = as_stream(stream);
  auto run = [&](auto kernel) {
    static thread_local bool configured = false;  // per (T, VEC) instantiation
    if (!configured) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)C::smem_bytes);
      configured = true;
    }
    kernel<<<(unsigned)grid, kTile, C::smem_bytes, st>>>(
        pat->row_ptr, pat->col_idx, pat->tile_row0, pat->m, pat->nnz, pat->ntiles,
        static_cast<const T*>(d_out), ld_d, static_cast<const T*>(x), ld_x, n,
        static_cast<T*>(values), static_cast<T*>(velocity), static_cast<T*>(grad_out),
        static_cast<T*>(bias), static_cast<T*>(vbias), static_cast<T*>(grad_bias_out), opt);
  };
  if (vec) run(sddmm_update_kernel<T, true>);
  else run(sddmm_update_kernel<T, false>);
  return check_launch(name);
}

}  // namespace
}  // namespace smb

using namespace smb;

extern "C" int smb_sddmm(int dtype, const smb_pattern* pat, const void* a, int64_t lda,
                         const void* b, int64_t ldb, int64_t n, void* out_values, void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_sddmm: null pattern");
  SMB_REQUIRE(n >= 0 && lda >= n && ldb >= n, "smb_sddmm: bad batch width / leading dimension");
  SMB_REQUIRE(pat->nnz == 0 || out_values != nullptr, "smb_sddmm: null output");
  if (dtype == SMB_F32)
    return sddmm_update_impl<float>(pat, a, lda, b, ldb, n, nullptr, nullptr, out_values, nullptr,
                                    nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0, stream,
                                    "smb_sddmm");
  if (dtype == SMB_F64)
    return sddmm_update_impl<double>(pat, a, lda, b, ldb, n, nullptr, nullptr, out_values,
                                     nullptr, nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0, stream,
                                     "smb_sddmm");
  set_error("smb_sddmm: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}

extern "C" int smb_sddmm_update(int dtype, const smb_pattern* pat, const void* d_out,
                                int64_t ld_dout, const void* x, int64_t ld_x, int64_t n,
                                void* values, void* velocity, void* grad_out, void* bias,
                                void* velocity_bias, void* grad_bias_out, int opt_kind, double mu,
                                double eta, void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_sddmm_update: null pattern");
  SMB_REQUIRE(n >= 0 && ld_dout >= n && ld_x >= n,
              "smb_sddmm_update: bad batch width / leading dimension");
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_sddmm_update: bad optimizer kind %d", opt_kind);
  SMB_REQUIRE(opt_kind == SMB_OPT_NONE || values != nullptr || pat->nnz == 0,
              "smb_sddmm_update: null values");
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) ||
                  velocity != nullptr || pat->nnz == 0,
              "smb_sddmm_update: momentum needs a velocity buffer");
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) || bias == nullptr ||
                  velocity_bias != nullptr,
              "smb_sddmm_update: momentum needs a bias velocity buffer");
  if (dtype == SMB_F32)
    return sddmm_update_impl<float>(pat, d_out, ld_dout, x, ld_x, n, values, velocity, grad_out,
                                    bias, velocity_bias, grad_bias_out, opt_kind, mu, eta, stream,
                                    "smb_sddmm_update");
  if (dtype == SMB_F64)
    return sddmm_update_impl<double>(pat, d_out, ld_dout, x, ld_x, n, values, velocity, grad_out,
                                     bias, velocity_bias, grad_bias_out, opt_kind, mu, eta,
                                     stream, "smb_sddmm_update");
  set_error("smb_sddmm_update: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}
