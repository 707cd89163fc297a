// Fused backward of one sparse layer (sm_100a): the transposed SpMM
//   d_x[c, :] = (sum_{i ascending} W[i, c] * d_out[i, :]) * (x[c, :] > 0)
// (_kernels.spmm_t_kernel, _kernels.py:40-59, fused with ReLU.backward of the
// layer below, nn.py:89-91) and the SDDMM weight gradient + optimizer update
//   grad[p] = sum_t d_out[i, t] * x[c, t];  W, V <- sparse_combine sequence
// (_kernels.sddmm_kernel, _kernels.py:62-75; nn.py:183, 187-197), walked
// together in CSC order.
//
// Why: at wide layers both kernels are bound by the L2 -> SM delivery of one
// B-wide row per nonzero (spmm_t gathers d_out rows in CSC order, the SDDMM
// gathers x rows in CSR order).  In CSC order the two products need the SAME
// gathered rows -- d_out[row_idx[q], :] for every stored q of the tile's
// columns -- plus one x row per column, so one staging pass feeds both and
// the layer's backward moves half the bytes (config 4).
//
// Mapping: CTA = a column tile (whole consecutive columns, <= kBwdTile
// nonzeros, <= kBwdCols columns; pattern.cu builds the table once).  Thread
// q owns the SDDMM chain of the tile's q-th CSC slot.  The batch is walked in
// CH-column chunks through a ring of shared-memory stages filled with 16-byte
// cp.async copies (the gathered d_out rows, one per slot, and the tile's x
// rows); per chunk every thread advances its chain over CH columns, then the
// tile's (column, batch column) outputs of the transposed product are summed
// over the column's slots -- ascending rows, the staged rows, the pre-update
// weights kept in shared memory -- masked by the staged x and stored.
// Rounding and order are exactly smb_spmm_t's and smb_sddmm_update's.
//
// Measured on B200 (scripts/probe_bwd_fused.py, 8192 x 8192): the staging
// itself runs near the L2 gather rate (d = 0.01, B = 1024: 315 us for the
// copies alone, 9 TB/s), but the whole kernel takes 674 us against 454 us
// for smb_spmm_t + smb_sddmm_update_into -- every staged element is written
// to and read twice from shared memory, and the transposed product's chains
// (a column long) sit on a few warps per CTA, so the SM's 128 B/clk
// shared-memory port, not L2, bounds it.  The training step therefore keeps
// the two separate kernels; this entry point stays as a bit-exact,
// tested alternative ("Fused backward").
#include <type_traits>

#include "async_copy.cuh"
#include "pattern.cuh"

namespace smb {
namespace {

template <typename T, int CH, int ST, int COLS>
struct BwdCfg {
  static constexpr int VW = 16 / sizeof(T);
  static constexpr int VPR = CH / VW;     // 16-byte vectors per staged row
  static constexpr int LDS = CH + VW;     // padded smem row (elements)
  static constexpr int ROWS = kBwdTile + COLS;
  static constexpr size_t stage_elems = size_t(ROWS) * LDS;
  static constexpr size_t smem_bytes = ST * stage_elems * sizeof(T);
  static_assert(kBwdTile % VPR == 0, "tile / vector split");
  static_assert((ST & (ST - 1)) == 0, "power-of-two ring");
};

template <typename T, int CH, int ST, int COLS, bool MASK, bool VEC>
__global__ void __launch_bounds__(kBwdTile)
    bwd_fused_kernel(const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
                     const int32_t* __restrict__ perm, const int32_t* __restrict__ ctile,
                     const T* __restrict__ d_out, int64_t ld_d, const T* __restrict__ x,
                     int64_t ld_x, int n32, T* __restrict__ d_x, int64_t ld_dx, const T* values,
                     T* values_out, T* velocity, T* grad_out, OptConsts<T> opt) {
  using C = BwdCfg<T, CH, ST, COLS>;
  constexpr int VW = C::VW, VPR = C::VPR, LDS = C::LDS;
  constexpr unsigned kStageBytes = (unsigned)(C::stage_elems * sizeof(T));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  __shared__ int32_t s_cp[COLS + 1];  // tile-local column pointers
  __shared__ int32_t s_row[kBwdTile];
  __shared__ T s_w[kBwdTile];             // pre-update weights, CSC order
  const int tid = threadIdx.x;
  const int j0 = ctile[blockIdx.x], j1 = ctile[blockIdx.x + 1];
  const int nc = j1 - j0;  // <= COLS
  const int q0 = col_ptr[j0];
  if (tid <= nc) s_cp[tid] = col_ptr[j0 + tid] - q0;
  const int nq = col_ptr[j1] - q0;  // <= kBwdTile
  const bool active = tid < nq;
  const int my_perm = active ? perm[q0 + tid] : 0;
  s_row[tid] = active ? row_idx[q0 + tid] : 0;  // row 0: a valid read nobody sums
  __syncthreads();
  // column of my slot: the last c with s_cp[c] <= tid
  int c_lo = 0, c_hi = nc;
  while (c_hi - c_lo > 1) {
    const int mid = (c_lo + c_hi) >> 1;
    if (s_cp[mid] <= tid) c_lo = mid; else c_hi = mid;
  }
  const int my_c = c_lo;
  // ---- fixed copy slots (computed once) ----
  // gathered d_out rows: slot row r = tid / VPR + k * (kBwdTile / VPR), vector v
  const int v = tid % VPR;
  // (slots past nq copy nothing: a shared dummy source row would turn every
  // CTA's padding copies into one L2 hot spot)
  const T* dsrc[VPR];
  unsigned ddst[VPR];
  bool dok[VPR];
#pragma unroll
  for (int k = 0; k < VPR; ++k) {
    const int r = tid / VPR + k * (kBwdTile / VPR);
    dok[k] = r < nq;
    dsrc[k] = d_out + (int64_t)s_row[r] * ld_d + v * VW;
    ddst[k] = (unsigned)((r * LDS + v * VW) * sizeof(T));
  }
  // x rows of the tile's columns (rows past nc are not copied)
  constexpr int XC = (COLS * VPR + kBwdTile - 1) / kBwdTile;
  constexpr bool kXGuard = (COLS * VPR) % kBwdTile != 0;
  const T* xsrc[XC];
  unsigned xdst[XC];
  bool xcopy[XC];
  bool xok[XC];
#pragma unroll
  for (int c = 0; c < XC; ++c) {
    const int e = tid + c * kBwdTile;
    const int xr = e / VPR;
    xcopy[c] = e < COLS * VPR;
    xok[c] = xr < nc;
    xsrc[c] = x + (int64_t)(j0 + (xok[c] ? xr : 0)) * ld_x + v * VW;
    xdst[c] = (unsigned)(((kBwdTile + xr) * LDS + v * VW) * sizeof(T));
  }
  const unsigned sbase = smem_u32(smem);
  const int n_fast = n32 / CH;           // chunks summed without bounds
  const int n_full = VEC ? n_fast : 0;   // chunks copied without bounds
  const int n_chunks = (n32 + CH - 1) / CH;
  auto issue_full = [&](int ch) {
    const unsigned st = sbase + (unsigned)(ch & (ST - 1)) * kStageBytes;
    const int t0 = ch * CH;
#pragma unroll
    for (int k = 0; k < VPR; ++k)
      if (dok[k]) cp_async16(st + ddst[k], dsrc[k] + t0);
#pragma unroll
    for (int c = 0; c < XC; ++c)
      if ((!kXGuard || xcopy[c]) && xok[c]) cp_async16(st + xdst[c], xsrc[c] + t0);
  };
  auto issue_part = [&](int ch) {
    const unsigned st = sbase + (unsigned)(ch & (ST - 1)) * kStageBytes;
    const int t0 = ch * CH;
    const int valid = max(0, min(VW, n32 - (t0 + v * VW)));
#pragma unroll
    for (int k = 0; k < VPR; ++k)
      if (dok[k]) copy_vec<T, VEC>(st + ddst[k], dsrc[k] + t0, valid);
#pragma unroll
    for (int c = 0; c < XC; ++c)
      if (xcopy[c] && xok[c]) copy_vec<T, VEC>(st + xdst[c], xsrc[c] + t0, valid);
  };
  pdl_wait();  // d_out / x are earlier kernels' outputs
  // the pre-update weights (a concurrent kernel may write values_out)
  s_w[tid] = active ? values[my_perm] : T(0);
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < n_full) issue_full(s);
    else if (s < n_chunks) issue_part(s);
    cp_async_commit();
  }
  T acc = T(-0.0);  // SDDMM chain (see sddmm.cu: -0 is the exact identity)
  using V = typename Vec16<T>::type;
  // one chunk: the SDDMM chains over its `cnt` columns, then the transposed
  // product's outputs of the tile's columns for those batch columns
  auto chunk = [&](int ch, int cnt) {
    const T* ds = smem + (ch & (ST - 1)) * C::stage_elems;
    const T* dr = ds + tid * LDS;
    const T* xr = ds + (kBwdTile + my_c) * LDS;
    if (cnt == CH) {
#pragma unroll
      for (int u = 0; u < VPR; ++u) {
        const V dv = *reinterpret_cast<const V*>(dr + u * VW);
        const V xv = *reinterpret_cast<const V*>(xr + u * VW);
#pragma unroll
        for (int j = 0; j < VW; ++j)
          acc = add_rn(acc, mul_rn(VecOps<T>::get(dv, j), VecOps<T>::get(xv, j)));
      }
    } else {
      for (int j = 0; j < cnt; ++j) acc = add_rn(acc, mul_rn(dr[j], xr[j]));
    }
    const int t0 = ch * CH;
    for (int o = tid; o < nc * CH; o += kBwdTile) {
      const int c = o / CH, t = o % CH;
      if (t >= cnt) continue;
      const int qa = s_cp[c], qb = s_cp[c + 1];
      // software-pipelined walk of the column's slots: one group of G staged
      // operands / weights is loaded while the previous group's chain runs
      // (two register sets, no copies between them)
      constexpr int G = 8;
      T s = T(0);
      int qq = qa;
      if (qb - qa >= G) {
        T a0[G], w0[G], a1[G], w1[G];
        auto load = [&](T (&av)[G], T (&wv)[G], int at) {
#pragma unroll
          for (int i = 0; i < G; ++i) {
            av[i] = ds[(at + i) * LDS + t];
            wv[i] = s_w[at + i];
          }
        };
        auto sum = [&](const T (&av)[G], const T (&wv)[G]) {
#pragma unroll
          for (int i = 0; i < G; ++i) s = add_rn(s, mul_rn(wv[i], av[i]));
        };
        load(a0, w0, qq);
        qq += G;
        for (;;) {
          if (qq + G > qb) { sum(a0, w0); break; }
          load(a1, w1, qq);
          qq += G;
          sum(a0, w0);
          if (qq + G > qb) { sum(a1, w1); break; }
          load(a0, w0, qq);
          qq += G;
          sum(a1, w1);
        }
      }
      for (; qq < qb; ++qq) s = add_rn(s, mul_rn(s_w[qq], ds[qq * LDS + t]));
      if (MASK) s = mask_np(s, ds[(kBwdTile + c) * LDS + t]);
      d_x[(int64_t)(j0 + c) * ld_dx + t0 + t] = s;
    }
  };
  int ch = 0;
  for (; ch < n_fast; ++ch) {
    cp_async_wait<ST - 2>();
    __syncthreads();  // chunk ch landed (and s_w on the first pass); stage ch-1 free
    const int nx = ch + ST - 1;
    if (nx < n_full) issue_full(nx);
    else if (nx < n_chunks) issue_part(nx);
    cp_async_commit();
    chunk(ch, CH);
  }
  if (ch < n_chunks) {  // ragged last chunk
    cp_async_wait<0>();
    __syncthreads();
    chunk(ch, n32 - ch * CH);
  }
  cp_async_wait<0>();
  pdl_trigger();
  if (!active) return;
  const T g = (n32 == 0) ? T(0) : acc;  // tensor_core.py:283-284: zero batch -> zeros
  if (grad_out) grad_out[my_perm] = g;
  if (opt.kind != SMB_OPT_NONE) {
    T w = s_w[tid];
    T vv = velocity ? velocity[my_perm] : T(0);
    apply_update(opt, g, &w, &vv);
    values_out[my_perm] = w;
    if (velocity) velocity[my_perm] = vv;
  }
}

}  // namespace

template <typename T>
int backward_fused_impl(const smb_pattern* pat, const void* d_out, int64_t ld_d, const void* x,
                        int64_t ld_x, int64_t n, int mask, void* d_x, int64_t ld_dx,
                        const void* values, void* values_out, void* velocity, void* grad_out,
                        int opt_kind, double mu, double eta, void* stream) {
  constexpr int VW = 16 / sizeof(T);
  if (pat->k == 0) return SMB_OK;
  const bool vec = aligned16(d_out) && aligned16(x) && ld_d % VW == 0 && ld_x % VW == 0;
  const OptConsts<T> opt = make_opt<T>(opt_kind, mu, eta);
  cudaStream_t st = as_stream(stream);
  auto run = [&](auto ch_tag, auto cols_tag) {
    constexpr int CH = decltype(ch_tag)::value;
    constexpr int COLS = decltype(cols_tag)::value;
    constexpr int ST = 2;
    using C = BwdCfg<T, CH, ST, COLS>;
    auto go = [&](auto kernel) {
      ensure_smem(kernel, C::smem_bytes);
      launch_k(kernel, dim3((unsigned)pat->n_ctiles), dim3(kBwdTile), C::smem_bytes, st,
               pat->col_ptr, pat->row_idx, pat->perm, pat->ctile, static_cast<const T*>(d_out),
               ld_d, static_cast<const T*>(x), ld_x, (int)n, static_cast<T*>(d_x), ld_dx,
               static_cast<const T*>(values), static_cast<T*>(values_out),
               static_cast<T*>(velocity), static_cast<T*>(grad_out), opt);
    };
    if (mask && vec)
      go(bwd_fused_kernel<T, CH, ST, COLS, true, true>);
    else if (vec)
      go(bwd_fused_kernel<T, CH, ST, COLS, false, true>);
    else if (mask)
      go(bwd_fused_kernel<T, CH, ST, COLS, true, false>);
    else
      go(bwd_fused_kernel<T, CH, ST, COLS, false, false>);
  };
  constexpr int CH = sizeof(T) == 4 ? 32 : 16;
  if (pat->bwd_cols == kBwdColsLong)
    run(std::integral_constant<int, CH>(), std::integral_constant<int, kBwdColsLong>());
  else
    run(std::integral_constant<int, CH>(), std::integral_constant<int, kBwdCols>());
  return check_launch("smb_backward_fused");
}

}  // namespace smb

using namespace smb;

extern "C" int smb_backward_fused_supported(int dtype, const smb_pattern* pat) {
  clear_error();
  if (pat == nullptr || (dtype != SMB_F32 && dtype != SMB_F64)) return 0;
  return (pat->k == 0 || pat->n_ctiles > 0) ? 1 : 0;
}

extern "C" int smb_backward_fused(int dtype, const smb_pattern* pat, const void* d_out,
                                  int64_t ld_dout, const void* x, int64_t ld_x, int64_t n,
                                  int mask, void* d_x, int64_t ld_dx, const void* values,
                                  void* values_out, void* velocity, void* grad_out, int opt_kind,
                                  double mu, double eta, void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_backward_fused: null pattern");
  SMB_REQUIRE(pat->k == 0 || pat->n_ctiles > 0,
              "smb_backward_fused: a column holds %lld > %d nonzeros (use smb_spmm_t + "
              "smb_sddmm_update_into)",
              (long long)pat->max_col, kBwdTile);
  SMB_REQUIRE(n >= 0 && n < (int64_t(1) << 31) && ld_dout >= n && ld_x >= n && ld_dx >= n,
              "smb_backward_fused: bad batch width / leading dimension");
  SMB_REQUIRE(pat->k == 0 || d_x != nullptr, "smb_backward_fused: null d_x");
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_backward_fused: bad optimizer kind %d", opt_kind);
  SMB_REQUIRE(pat->nnz == 0 || values != nullptr, "smb_backward_fused: null values");
  SMB_REQUIRE(opt_kind == SMB_OPT_NONE || values_out != nullptr || pat->nnz == 0,
              "smb_backward_fused: null output values");
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) ||
                  velocity != nullptr || pat->nnz == 0,
              "smb_backward_fused: momentum needs a velocity buffer");
  if (dtype == SMB_F32)
    return backward_fused_impl<float>(pat, d_out, ld_dout, x, ld_x, n, mask, d_x, ld_dx, values,
                                      values_out, velocity, grad_out, opt_kind, mu, eta, stream);
  if (dtype == SMB_F64)
    return backward_fused_impl<double>(pat, d_out, ld_dout, x, ld_x, n, mask, d_x, ld_dx, values,
                                       values_out, velocity, grad_out, opt_kind, mu, eta, stream);
  set_error("smb_backward_fused: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}
