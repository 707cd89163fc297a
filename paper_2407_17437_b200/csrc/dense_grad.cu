// Weight gradient + update of a small dense layer (sm_100a): the
// ER-saturated output layer of every BASELINE config (m <= 32 rows).
//
//   grad[i, c] = sum_t d_out[i, t] * x[c, t]      (DenseLinearLayer.backward,
//                                                  nn.py:241-255: d @ x.T)
//   then the optimizer update of W[i, c] / V[i, c] (_step_vector on the dense
//   weights, nn.py:118-131, 260-264), or grad written out (data parallel).
//
// Each gradient element is ONE sequential chain over the batch with multiply
// and add rounded separately -- the SDDMM chain of a full pattern
// (_kernels.py:62-75), so it is deterministic and bit-identical to
// smb_sddmm over an all-ones pattern; the reference's numpy BLAS order is
// unspecified (tolerance parity there).  Replaces a cuBLAS SIMT GEMM plus a
// separate update launch.
//
// Mapping: CTA = 64 columns c (one x row per thread) x one group of MR output
// rows.  The batch is walked in 32-column chunks through a 4-stage cp.async
// ring holding the CTA's 64 x rows (swizzled 128-byte lines, async_copy.cuh:
// each thread's 16-byte read of its own row is bank-conflict free) and the
// group's d_out rows (read as broadcasts); every thread runs MR independent chains, so the
// FADD latency is hidden inside the thread.  x is streamed from HBM once per
// row group.
#include <type_traits>

#include "async_copy.cuh"

namespace smb {
namespace {

constexpr int kDgCols = 64;    // columns c per CTA (threads)
constexpr int kDgChunk = 32;   // batch columns per stage
constexpr int kDgStages = 4;

template <typename T>
struct DgCfg {
  static constexpr int VW = 16 / sizeof(T);
  static constexpr int LDS = kDgChunk;       // swizzled row (swz)
  static constexpr int VPR = kDgChunk / VW;  // 16-byte vectors per staged row
  static_assert(VPR % 8 == 0, "swizzle spans 8 vectors");
};

template <typename T, int MR, bool VEC>
__global__ void __launch_bounds__(kDgCols)
    dense_grad_kernel(const T* __restrict__ d, int64_t ld_d, int m, const T* __restrict__ x,
                      int64_t ld_x, int64_t k, int64_t n, T* __restrict__ w, int64_t ld_w,
                      T* __restrict__ vel, T* __restrict__ grad_out, OptConsts<T> opt) {
  using C = DgCfg<T>;
  using V = typename Vec16<T>::type;
  constexpr int VW = C::VW, LDS = C::LDS, VPR = C::VPR;
  constexpr int ROWS = kDgCols + MR;  // staged rows per stage: x rows, then d rows
  constexpr unsigned kStage = (unsigned)(ROWS * LDS * sizeof(T));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(align128(smem_raw));
  const int tid = threadIdx.x;
  const int row0 = blockIdx.x * MR;
  const int nr = (int)imin(MR, m - row0);
  const int64_t c0 = (int64_t)blockIdx.y * kDgCols;
  const int64_t c = c0 + tid;
  const bool active = c < k;

  // copy slots: x vectors e = tid + 64 q (row e / VPR, part e % VPR), d vectors
  constexpr int XV = kDgCols * VPR / kDgCols;  // = VPR per thread
  const T* xsrc[XV];
  unsigned xdst[XV];
  bool xok[XV];
#pragma unroll
  for (int q = 0; q < XV; ++q) {
    const int e = tid + kDgCols * q, r = e / VPR, v = e % VPR;
    xok[q] = c0 + r < k;
    xsrc[q] = x + (xok[q] ? c0 + r : 0) * ld_x + v * VW;
    xdst[q] = (unsigned)(swz<LDS, VW>(r, v) * sizeof(T));
  }
  constexpr int DV = (MR * VPR + kDgCols - 1) / kDgCols;
  const T* dsrc[DV];
  unsigned ddst[DV];
  bool dok[DV];
#pragma unroll
  for (int q = 0; q < DV; ++q) {
    const int e = tid + kDgCols * q, r = e / VPR, v = e % VPR;
    dok[q] = r < nr;
    dsrc[q] = d + (int64_t)(row0 + (dok[q] ? r : 0)) * ld_d + v * VW;
    ddst[q] = (unsigned)(swz<LDS, VW>(kDgCols + r, v) * sizeof(T));
  }
  // update operands (independent of the previous kernel's output)
  T w_pre[MR], v_pre[MR];
  const bool upd = active && opt.kind != SMB_OPT_NONE;
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    w_pre[r] = (upd && r < nr) ? w[(int64_t)(row0 + r) * ld_w + c] : T(0);
    v_pre[r] = (upd && vel && r < nr) ? vel[(int64_t)(row0 + r) * ld_w + c] : T(0);
  }
  pdl_wait();  // d_out / x are earlier kernels' outputs
  const int n32 = (int)n;
  const int n_chunks = (n32 + kDgChunk - 1) / kDgChunk;
  const unsigned sbase = smem_u32(sm);
  auto issue = [&](int ch) {
    const unsigned st = sbase + (unsigned)(ch % kDgStages) * kStage;
    const int t0 = ch * kDgChunk;
#pragma unroll
    for (int q = 0; q < XV; ++q) {
      const int e = tid + kDgCols * q, v = e % VPR;
      const int valid = (int)imax(0, imin(VW, n32 - (t0 + v * VW)));
      if (xok[q]) copy_vec<T, VEC>(st + xdst[q], xsrc[q] + t0, valid);
    }
#pragma unroll
    for (int q = 0; q < DV; ++q) {
      const int e = tid + kDgCols * q, v = e % VPR;
      const int valid = (int)imax(0, imin(VW, n32 - (t0 + v * VW)));
      if (dok[q] && e < MR * VPR) copy_vec<T, VEC>(st + ddst[q], dsrc[q] + t0, valid);
    }
  };
#pragma unroll
  for (int s = 0; s < kDgStages - 1; ++s) {
    if (s < n_chunks) issue(s);
    cp_async_commit();
  }
  T acc[MR];
#pragma unroll
  for (int r = 0; r < MR; ++r) acc[r] = T(-0.0);  // exact additive identity
  for (int ch = 0; ch < n_chunks; ++ch) {
    cp_async_wait<kDgStages - 2>();
    __syncthreads();  // chunk ch landed; stage (ch - 1) % S is free
    if (ch + kDgStages - 1 < n_chunks) issue(ch + kDgStages - 1);
    cp_async_commit();
    const T* st = sm + (ch % kDgStages) * (kStage / sizeof(T));
    const int cnt = min(kDgChunk, n32 - ch * kDgChunk);
    if (cnt == kDgChunk) {
#pragma unroll
      for (int u = 0; u < VPR; ++u) {
        const V xv = *reinterpret_cast<const V*>(st + swz<LDS, VW>(tid, u));
#pragma unroll
        for (int r = 0; r < MR; ++r) {
          const V dv = *reinterpret_cast<const V*>(st + swz<LDS, VW>(kDgCols + r, u));
#pragma unroll
          for (int j = 0; j < VW; ++j)
            acc[r] = add_rn(acc[r], mul_rn(VecOps<T>::get(dv, j), VecOps<T>::get(xv, j)));
        }
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        const T xv = st[swz<LDS, VW>(tid, j / VW) + j % VW];
#pragma unroll
        for (int r = 0; r < MR; ++r)
          acc[r] = add_rn(acc[r], mul_rn(st[swz<LDS, VW>(kDgCols + r, j / VW) + j % VW], xv));
      }
    }
  }
  cp_async_wait<0>();
  pdl_trigger();
  if (!active) return;
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    if (r >= nr) break;
    const T g = n32 == 0 ? T(0) : acc[r];
    if (grad_out) grad_out[(int64_t)(row0 + r) * k + c] = g;
    if (upd) {
      apply_update(opt, g, &w_pre[r], &v_pre[r]);
      w[(int64_t)(row0 + r) * ld_w + c] = w_pre[r];
      if (vel) vel[(int64_t)(row0 + r) * ld_w + c] = v_pre[r];
    }
  }
}

}  // namespace
}  // namespace smb

using namespace smb;

extern "C" int smb_dense_grad_update(int dtype, const void* d_out, int64_t ld_d, int64_t m,
                                     const void* x, int64_t ld_x, int64_t k, int64_t n,
                                     void* w, int64_t ld_w, void* velocity, void* grad_out,
                                     int opt_kind, double mu, double eta, void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 1 && m <= 32, "smb_dense_grad_update: needs 1 <= m <= 32");
  SMB_REQUIRE(k >= 0 && n >= 0 && n <= INT32_MAX && ld_d >= n && ld_x >= n && ld_w >= k,
              "smb_dense_grad_update: bad shape");
  SMB_REQUIRE(opt_kind == SMB_OPT_NONE || opt_kind == SMB_OPT_GD ||
                  opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV,
              "smb_dense_grad_update: unknown optimizer kind %d", opt_kind);
  if (k == 0) return SMB_OK;
  SMB_REQUIRE(opt_kind == SMB_OPT_NONE || w, "smb_dense_grad_update: null weights");
  SMB_REQUIRE(opt_kind != SMB_OPT_NONE || grad_out, "smb_dense_grad_update: null grad_out");
  SMB_REQUIRE(n == 0 || (d_out && x), "smb_dense_grad_update: null operand");
  SMB_REQUIRE(opt_kind == SMB_OPT_NONE || opt_kind == SMB_OPT_GD || velocity,
              "smb_dense_grad_update: momentum needs a velocity");
  return dispatch_dtype(dtype, "smb_dense_grad_update", [&](auto tag) {
    using T = decltype(tag);
    constexpr int VW = 16 / (int)sizeof(T);
    const OptConsts<T> opt = make_opt<T>(opt_kind, mu, eta);
    const bool vec = aligned16(d_out) && aligned16(x) && ld_d % VW == 0 && ld_x % VW == 0;
    const int64_t cb = ceil_div(k, kDgCols);
    // rows per thread: as many as keep >= 2 CTAs per SM (the x tile is then
    // read once per row group, mostly from L2)
    auto go = [&](auto mr_tag) {
      constexpr int MR = decltype(mr_tag)::value;
      const dim3 grid((unsigned)ceil_div(m, MR), (unsigned)cb);
      const size_t smem = (size_t)kDgStages * (kDgCols + MR) * DgCfg<T>::LDS * sizeof(T) + 128;
      auto launch = [&](auto kernel) {
        ensure_smem(kernel, smem);
        launch_k(kernel, grid, dim3(kDgCols), smem, as_stream(stream),
                 static_cast<const T*>(d_out), ld_d, (int)m, static_cast<const T*>(x), ld_x, k,
                 n, static_cast<T*>(w), ld_w, static_cast<T*>(velocity),
                 static_cast<T*>(grad_out), opt);
      };
      if (vec) launch(dense_grad_kernel<T, MR, true>);
      else launch(dense_grad_kernel<T, MR, false>);
    };
#ifdef SMB_DG_FORCE_MR  // tuning sweeps (scripts/build_variant.sh)
    if (true) go(std::integral_constant<int, SMB_DG_FORCE_MR>{});
    else
#endif
    if (m == 10 && cb >= 296) go(std::integral_constant<int, 10>{});
    else if (cb * ceil_div(m, 16) >= 296) go(std::integral_constant<int, 16>{});
    else if (cb * ceil_div(m, 8) >= 296) go(std::integral_constant<int, 8>{});
    else if (cb * ceil_div(m, 4) >= 296 || m > 16) go(std::integral_constant<int, 4>{});
    else go(std::integral_constant<int, 2>{});
    return check_launch("smb_dense_grad_update");
  });
}
