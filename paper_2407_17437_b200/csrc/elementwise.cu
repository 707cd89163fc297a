// Memory-bound glue of the training step: sparse_combine (axpby), the
// optimizer update of flat segments, numpy-order row sums (+ bias update),
// the softmax cross-entropy step, ReLU forward/backward and the device batch
// gather.
#include "common.cuh"
#include "tma.cuh"

#include <type_traits>

namespace smb {
namespace {

int grid_1d(int64_t work, int threads, int cap_per_sm = 16) {
  int64_t b = ceil_div(work, threads);
  if (b < 1) b = 1;
  const int64_t cap = 148LL * cap_per_sm;
  return (int)(b > cap ? cap : b);
}

// ---- sparse_combine: s = T(alpha) s + T(beta) t  (_kernels.py:78-83) ------
template <typename T>
__global__ void axpby_kernel(T alpha, T* __restrict__ s, T beta, const T* __restrict__ t,
                             int64_t count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    s[i] = add_rn(mul_rn(alpha, s[i]), mul_rn(beta, t[i]));
}

// ---- optimizer update of a flat (param, velocity, grad) segment -----------
template <typename T>
__global__ void optimizer_kernel(T* __restrict__ w, T* __restrict__ v, const T* __restrict__ g,
                                 int64_t count, OptConsts<T> o) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    T dummy = T(0);
    apply_update(o, g[i], w + i, v ? v + i : &dummy);
  }
}

// ---- masked-dense baseline update (DenseLinearLayer.optimize with a mask,
// nn.py:258-264; grad masked as in backward, nn.py:255-256):
//   g' = g*mask; v = v*mask; _step_vector(w, g', v); w = w*mask
// one pass; multiplying by an exact 0/1 keeps numpy's signed zeros.
template <typename T>
__device__ __forceinline__ void masked_update_one(const OptConsts<T>& o, T* w, T* v, T g, T mk) {
  T ww = *w, vv = v ? *v : T(0);
  g = mul_rn(g, mk);
  if (v) vv = mul_rn(vv, mk);
  apply_update(o, g, &ww, &vv);
  *w = mul_rn(ww, mk);
  if (v) *v = vv;
}

template <typename T, bool VEC>
__global__ void masked_optimizer_kernel(T* __restrict__ w, T* __restrict__ v,
                                        const T* __restrict__ g, const T* __restrict__ mask,
                                        int64_t count, OptConsts<T> o) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (VEC) {
    using V = typename Vec16<T>::type;
    constexpr int VW = Vec16<T>::N;
    for (int64_t i = t0; i < count / VW; i += stride) {
      V wv = reinterpret_cast<const V*>(w)[i];
      V vv = v ? reinterpret_cast<const V*>(v)[i] : V{};
      const V gv = __ldg(reinterpret_cast<const V*>(g) + i);
      const V mv = __ldg(reinterpret_cast<const V*>(mask) + i);
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        T a = VecOps<T>::get(wv, j), b = VecOps<T>::get(vv, j);
        masked_update_one(o, &a, v ? &b : nullptr, VecOps<T>::get(gv, j), VecOps<T>::get(mv, j));
        VecOps<T>::set(wv, j, a);
        VecOps<T>::set(vv, j, b);
      }
      reinterpret_cast<V*>(w)[i] = wv;
      if (v) reinterpret_cast<V*>(v)[i] = vv;
    }
  } else {
    for (int64_t i = t0; i < count; i += stride)
      masked_update_one(o, w + i, v ? v + i : nullptr, g[i], mask[i]);
  }
}

// ---- several (param, velocity, grad, mask) segments in one launch: the
// data-parallel update pass after the gradient all-reduce.  Segment i covers
// elements [start[i], start[i+1]) of the concatenation (up to 32 segments).
// Same arithmetic as optimizer_kernel / masked_optimizer_kernel per element.
struct OptSegment {
  void* param;
  void* velocity;      // may be null (GD)
  const void* grad;
  const void* mask;    // may be null (no mask)
  int64_t start;       // first element in the concatenation
};

template <typename T>
__global__ void multi_optimizer_kernel(const OptSegment* __restrict__ segs, int nseg, int64_t total,
                                       OptConsts<T> o) {
  __shared__ OptSegment s_seg[32];
  __shared__ int64_t s_end[32];
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    s_seg[i] = segs[i];
    s_end[i] = (i + 1 < nseg) ? segs[i + 1].start : total;
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int si = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    while (e >= s_end[si]) ++si;  // segments ascend with e
    const OptSegment& sg = s_seg[si];
    const int64_t j = e - sg.start;
    T* w = static_cast<T*>(sg.param) + j;
    T* v = sg.velocity ? static_cast<T*>(sg.velocity) + j : nullptr;
    const T g = static_cast<const T*>(sg.grad)[j];
    if (sg.mask) {
      masked_update_one(o, w, v, g, static_cast<const T*>(sg.mask)[j]);
    } else {
      T dummy = T(0);
      apply_update(o, g, w, v ? v : &dummy);
    }
  }
}

// ---- warp per row: pairwise row sum (tensor_core.py:353-356) and the bias
// optimizer update (_step_vector, nn.py:118-131) --------------------------
constexpr int kRowWarps = 8;
constexpr int kWarpLeafCap = 260;  // warp_pairwise_leaves(n) for n <= 16384

template <typename T>
__global__ void __launch_bounds__(kRowWarps * 32)
    bias_rows_kernel(const T* __restrict__ d, int64_t ld, int64_t m, int64_t n, T* bias, T* vbias,
                     T* grad, OptConsts<T> opt) {
  __shared__ T leaf[kRowWarps][kWarpLeafCap];
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowWarps + warp;
  if (row >= m) return;
  T g;
  if (n <= 16384) {
    g = warp_pairwise_sum(d + row * ld, (int)n, leaf[warp]);
  } else {
    g = pairwise_sum(d + row * ld, n);  // sequential fallback for very wide batches
  }
  if (lane != 0) return;
  if (grad) grad[row] = g;
  if (opt.kind != SMB_OPT_NONE && bias) {
    T dummy = T(0);
    apply_update(opt, g, bias + row, vbias ? vbias + row : &dummy);
  }
}

// ---- softmax cross-entropy step (nn.py:385-417, train.py:399) -------------
// One thread per sample column: z = y - max, e = exp(z) (double, rounded),
// s = sum_c e (sequential, numpy's axis-0 order), d = (e/s - t) / divisor.
// The per-column loss log(s) - sum_c z*t is reduced per CTA in a fixed tree
// and across CTAs by the last CTA to finish (ticket), which then also runs
// the last layer's bias row sums / update and advances the step counter.
template <typename T, bool ROWS>
__global__ void __launch_bounds__(ROWS ? 1024 : 128)
    softmax_step_kernel(const T* __restrict__ y, int64_t ld_y, const T* __restrict__ t,
                        int64_t ld_t, int64_t classes, int64_t n, T divisor, T* dy, int64_t ld_dy,
                        double* loss_out, double* loss_parts, unsigned* ticket, T* bias, T* vbias,
                        T* grad_bias, OptConsts<T> opt, int32_t* counter, int32_t modulo,
                        int stage_rows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_warp[32];
  __shared__ bool s_last;
  // dynamic smem: [warps x pairwise leaves][classes x n staged d_y block]
  T* stage_dst =
      reinterpret_cast<T*>(smem_raw) + (blockDim.x >> 5) * warp_pairwise_leaves((int)n);
  pdl_wait();  // y is the previous kernel's output
  double local = 0.0;
  // bias state of row `warp` (the first row this warp sums), loaded now
  T pb_w = T(0), pb_v = T(0);
  if ((threadIdx.x & 31) == 0 && (int64_t)(threadIdx.x >> 5) < classes && bias &&
      opt.kind != SMB_OPT_NONE) {
    pb_w = bias[threadIdx.x >> 5];
    if (vbias) pb_v = vbias[threadIdx.x >> 5];
  }
  for (int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; col < n;
       col += (int64_t)gridDim.x * blockDim.x) {
    T s = T(0), zt = T(0);
    constexpr int kRegC = 16;  // the column kept in registers for <= 16 classes
    T er[kRegC], tr[kRegC];
    if (classes <= kRegC) {
      // all loads of the column issued back to back (one memory round trip)
#pragma unroll
      for (int c = 0; c < kRegC; ++c) {
        er[c] = c < classes ? y[c * ld_y + col] : T(0);
        tr[c] = c < classes ? t[c * ld_t + col] : T(0);
      }
      T mx = er[0];
#pragma unroll
      for (int c = 1; c < kRegC; ++c)
        if (c < classes) mx = (er[c] > mx || er[c] != er[c]) ? er[c] : mx;
#pragma unroll
      for (int c = 0; c < kRegC; ++c) {
        if (c < classes) {
          const T z = sub_rn(er[c], mx);
          er[c] = exp_full(z);
          s = add_rn(s, er[c]);
          zt = add_rn(zt, mul_rn(z, tr[c]));
        }
      }
    } else {
      T mx = y[col];
      for (int64_t c = 1; c < classes; ++c) {
        const T v = y[c * ld_y + col];
        mx = (v > mx || v != v) ? v : mx;
      }
      for (int64_t c = 0; c < classes; ++c) {
        const T z = sub_rn(y[c * ld_y + col], mx);
        const T e = exp_full(z);
        dy[c * ld_dy + col] = e;
        s = add_rn(s, e);
        zt = add_rn(zt, mul_rn(z, t[c * ld_t + col]));
      }
    }
    auto emit = [&](int64_t c, T e, T tc) {
      const T g = div_rn(sub_rn(div_rn(e, s), tc), divisor);
      dy[c * ld_dy + col] = g;
      // single CTA: keep the block in shared memory for the bias row sums
      if (stage_rows && gridDim.x == 1) stage_dst[c * n + col] = g;
    };
    if (classes <= kRegC) {
#pragma unroll
      for (int c = 0; c < kRegC; ++c)
        if (c < classes) emit(c, er[c], tr[c]);
    } else {
      for (int64_t c = 0; c < classes; ++c) emit(c, dy[c * ld_dy + col], t[c * ld_t + col]);
    }
    local += static_cast<double>(sub_rn(log_full(s), zt));
  }
  pdl_trigger();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (!ROWS) {
    // nothing after the columns: no loss wanted, no counter to advance
    if (loss_out == nullptr && counter == nullptr) return;
  }
  // fixed-order block reduction of the loss
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if (lane == 0) s_warp[warp] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += s_warp[w];
    if (gridDim.x == 1) {
      s_last = true;
      if (loss_out) *loss_out = b;
    } else {
      loss_parts[blockIdx.x] = b;
      __threadfence();
      s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!s_last) return;
  if (gridDim.x > 1) __threadfence();
  if (threadIdx.x == 0 && gridDim.x > 1) {
    double tot = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) tot += loss_parts[b];
    if (loss_out) *loss_out = tot;
    *ticket = 0u;  // ready for the next launch / graph replay
  }
  if (counter && threadIdx.x == 0) {
    const int32_t v = *counter + 1;
    *counter = (modulo > 0 && v >= modulo) ? 0 : v;
  }
  if constexpr (!ROWS) {
    return;  // column-only variant: no bias side compiled in
  }
  if (grad_bias == nullptr && !(opt.kind != SMB_OPT_NONE && bias)) return;
  // stage_rows: the whole classes x n block of d_y fits the dynamic smem the
  // host reserved -> one coalesced pass, then the sums read shared memory
  T* leaf = reinterpret_cast<T*>(smem_raw) + warp * warp_pairwise_leaves((int)n);
  T* staged = stage_dst;
  if (stage_rows && gridDim.x == 1) {
    __syncthreads();  // the single CTA wrote the block while computing it
  } else if (stage_rows) {
    // 8 independent loads in flight per thread (a plain loop serialises one
    // L2 round trip per element)
    const int n32 = (int)n, total = (int)classes * n32, nt = blockDim.x;
    for (int base = threadIdx.x; base < total; base += 8 * nt) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = base + u * nt;
        v[u] = e < total ? dy[(int64_t)(e / n32) * ld_dy + e % n32] : T(0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = base + u * nt;
        if (e < total) staged[e] = v[u];
      }
    }
    __syncthreads();
  }
  for (int64_t c = warp; c < classes; c += (blockDim.x >> 5)) {
    const T* src = stage_rows ? staged + c * n : dy + c * ld_dy;
    const T g = warp_pairwise_sum(src, (int)n, leaf);
    if (lane == 0) {
      if (grad_bias) grad_bias[c] = g;
      if (opt.kind != SMB_OPT_NONE && bias) {
        T w = c == warp ? pb_w : bias[c];
        T v = c == warp ? pb_v : (vbias ? vbias[c] : T(0));
        apply_update(opt, g, &w, &v);
        bias[c] = w;
        if (vbias) vbias[c] = v;
      }
    }
  }
}

// ---- ReLU (nn.py:86-91) ------------------------------------------------------
template <typename T>
__global__ void relu_kernel(const T* __restrict__ x, int64_t ld_x, int64_t m, int64_t n,
                            T* __restrict__ y, int64_t ld_y) {
  const int64_t total = m * n, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / n, j = e - (e / n) * n;
    y[i * ld_y + j] = relu_np(x[i * ld_x + j]);
  }
}

template <typename T>
__global__ void relu_backward_kernel(const T* __restrict__ d, int64_t ld_d,
                                     const T* __restrict__ xc, int64_t ld_x, int64_t m, int64_t n,
                                     T* __restrict__ out, int64_t ld_out) {
  const int64_t total = m * n, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / n, j = e - (e / n) * n;
    out[i * ld_out + j] = mask_np(d[i * ld_d + j], xc[i * ld_x + j]);
  }
}

// ---- device batch gather (train.py:390-396) ----------------------------------
// dst[f, j] = src[perm[base + j], f]: a CTA moves 32 samples x 128 features,
// reading whole 512-byte sample segments (16-byte vectors) and writing
// 128-byte batch rows, transposing through padded shared memory.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256)
    gather_columns_kernel(const T* __restrict__ src, int64_t features,
                          const int32_t* __restrict__ perm, const int32_t* __restrict__ step_counter,
                          int64_t base, int32_t step_offset, int32_t modulo, int64_t batch,
                          T* __restrict__ dst, int64_t ld_dst) {
  constexpr int FT = 128;  // features per tile
  __shared__ T tile[32][FT + 1];
  __shared__ int32_t s_idx[32];
  pdl_wait();  // the step counter may be the previous kernel's output
  int64_t b0 = base;
  if (step_counter) {
    int64_t k = (int64_t)(*step_counter) + step_offset;
    if (modulo > 0) k %= modulo;
    b0 = k * batch;
  }
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t f0 = (int64_t)blockIdx.y * FT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  if (ty == 0) s_idx[tx] = (j0 + tx < batch) ? perm[b0 + j0 + tx] : -1;
  __syncthreads();
  if (VEC) {
    constexpr int VW = 16 / sizeof(T);
    using V = typename Vec16<T>::type;
    // each sample row segment: FT/VW vectors; 256 threads cover 32 rows.
    // All of a thread's loads are issued before any is used (one HBM round
    // trip per CTA instead of one per vector: 10 -> ~4 us for the config-2
    // batch of 1024 x 3072 fp32)
    constexpr int NV = 32 * (FT / VW) / 256;
    V xv[NV];
    bool full[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int e = threadIdx.x + 256 * q;
      const int r = e / (FT / VW), v = e % (FT / VW);
      const int32_t sidx = s_idx[r];
      const int64_t f = f0 + (int64_t)v * VW;
      full[q] = sidx >= 0 && f + VW <= features;
      if (full[q]) xv[q] = __ldg(reinterpret_cast<const V*>(src + (int64_t)sidx * features + f));
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int e = threadIdx.x + 256 * q;
      const int r = e / (FT / VW), v = e % (FT / VW);
      if (full[q]) {
#pragma unroll
        for (int j = 0; j < VW; ++j) tile[r][v * VW + j] = VecOps<T>::get(xv[q], j);
      } else {
        const int32_t sidx = s_idx[r];
        const int64_t f = f0 + (int64_t)v * VW;
        if (sidx < 0 || f >= features) continue;
        const T* p = src + (int64_t)sidx * features + f;
        for (int j = 0; f + j < features; ++j) tile[r][v * VW + j] = p[j];
      }
    }
  } else {
    for (int r = ty; r < 32; r += 8) {
      const int32_t sidx = s_idx[r];
      if (sidx < 0) continue;
      for (int c = tx; c < FT && f0 + c < features; c += 32)
        tile[r][c] = src[(int64_t)sidx * features + f0 + c];
    }
  }
  __syncthreads();
  if (j0 + tx >= batch) return;
  for (int c = ty; c < FT && f0 + c < features; c += 8)
    dst[(f0 + c) * ld_dst + j0 + tx] = tile[tx][c];
}

}  // namespace

template <typename T>
int launch_bias_rows(const T* d, int64_t ld, int64_t m, int64_t n, T* bias, T* vbias, T* grad,
                     const OptConsts<T>& opt, cudaStream_t st) {
  if (m == 0) return SMB_OK;
  launch_k(bias_rows_kernel<T>, dim3((unsigned)ceil_div(m, kRowWarps)), dim3(kRowWarps * 32), 0, st,
      d, ld, m, n, bias, vbias, grad, opt);
  return check_launch("bias_rows");
}
template int launch_bias_rows<float>(const float*, int64_t, int64_t, int64_t, float*, float*,
                                     float*, const OptConsts<float>&, cudaStream_t);
template int launch_bias_rows<double>(const double*, int64_t, int64_t, int64_t, double*, double*,
                                      double*, const OptConsts<double>&, cudaStream_t);

}  // namespace smb

using namespace smb;

extern "C" int smb_axpby(int dtype, double alpha, void* s, double beta, const void* t,
                         int64_t count, void* stream) {
  clear_error();
  SMB_REQUIRE(count >= 0, "smb_axpby: negative count");
  if (count == 0) return SMB_OK;
  SMB_REQUIRE(s && t, "smb_axpby: null pointer");
  return dispatch_dtype(dtype, "smb_axpby", [&](auto tag) {
    using T = decltype(tag);
    axpby_kernel<T><<<grid_1d(count, 256), 256, 0, as_stream(stream)>>>(
        static_cast<T>(alpha), static_cast<T*>(s), static_cast<T>(beta),
        static_cast<const T*>(t), count);
    return check_launch("smb_axpby");
  });
}

extern "C" int smb_optimizer_step(int dtype, void* param, void* velocity, const void* grad,
                                  int64_t count, int opt_kind, double mu, double eta,
                                  void* stream) {
  clear_error();
  SMB_REQUIRE(count >= 0, "smb_optimizer_step: negative count");
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_optimizer_step: bad optimizer kind %d", opt_kind);
  if (count == 0 || opt_kind == SMB_OPT_NONE) return SMB_OK;
  SMB_REQUIRE(param && grad, "smb_optimizer_step: null pointer");
  SMB_REQUIRE(opt_kind == SMB_OPT_GD || velocity, "smb_optimizer_step: momentum needs velocity");
  return dispatch_dtype(dtype, "smb_optimizer_step", [&](auto tag) {
    using T = decltype(tag);
    optimizer_kernel<T><<<grid_1d(count, 256), 256, 0, as_stream(stream)>>>(
        static_cast<T*>(param), static_cast<T*>(velocity), static_cast<const T*>(grad), count,
        make_opt<T>(opt_kind, mu, eta));
    return check_launch("smb_optimizer_step");
  });
}

extern "C" int smb_masked_optimizer_step(int dtype, void* param, void* velocity,
                                         const void* grad, const void* mask, int64_t count,
                                         int opt_kind, double mu, double eta, void* stream) {
  clear_error();
  SMB_REQUIRE(count >= 0, "smb_masked_optimizer_step: negative count");
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_masked_optimizer_step: bad optimizer kind %d", opt_kind);
  if (count == 0 || opt_kind == SMB_OPT_NONE) return SMB_OK;
  SMB_REQUIRE(param && grad && mask, "smb_masked_optimizer_step: null pointer");
  SMB_REQUIRE(opt_kind == SMB_OPT_GD || velocity,
              "smb_masked_optimizer_step: momentum needs velocity");
  return dispatch_dtype(dtype, "smb_masked_optimizer_step", [&](auto tag) {
    using T = decltype(tag);
    constexpr int VW = Vec16<T>::N;
    const bool vec = count % VW == 0 && aligned16(param) && aligned16(grad) &&
                     aligned16(mask) && (velocity == nullptr || aligned16(velocity));
    const OptConsts<T> o = make_opt<T>(opt_kind, mu, eta);
    cudaStream_t st = as_stream(stream);
    if (vec)
      masked_optimizer_kernel<T, true><<<grid_1d(count / VW, 256), 256, 0, st>>>(
          static_cast<T*>(param), static_cast<T*>(velocity), static_cast<const T*>(grad),
          static_cast<const T*>(mask), count, o);
    else
      masked_optimizer_kernel<T, false><<<grid_1d(count, 256), 256, 0, st>>>(
          static_cast<T*>(param), static_cast<T*>(velocity), static_cast<const T*>(grad),
          static_cast<const T*>(mask), count, o);
    return check_launch("smb_masked_optimizer_step");
  });
}

extern "C" int smb_optimizer_step_multi(int dtype, const void* segments, int n_segments,
                                        int64_t total, int opt_kind, double mu, double eta,
                                        void* stream) {
  clear_error();
  SMB_REQUIRE(n_segments >= 0 && n_segments <= 32, "smb_optimizer_step_multi: 0..32 segments");
  SMB_REQUIRE(total >= 0, "smb_optimizer_step_multi: negative total");
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_optimizer_step_multi: bad optimizer kind %d", opt_kind);
  if (total == 0 || n_segments == 0 || opt_kind == SMB_OPT_NONE) return SMB_OK;
  SMB_REQUIRE(segments != nullptr, "smb_optimizer_step_multi: null segment table");
  return dispatch_dtype(dtype, "smb_optimizer_step_multi", [&](auto tag) {
    using T = decltype(tag);
    multi_optimizer_kernel<T><<<grid_1d(total, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const OptSegment*>(segments), n_segments, total,
        make_opt<T>(opt_kind, mu, eta));
    return check_launch("smb_optimizer_step_multi");
  });
}

extern "C" int smb_row_sums(int dtype, const void* dense, int64_t m, int64_t n, int64_t ld,
                            void* out, void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 0 && n >= 0 && ld >= n, "smb_row_sums: bad shape");
  SMB_REQUIRE(m == 0 || out != nullptr, "smb_row_sums: null output");
  return dispatch_dtype(dtype, "smb_row_sums", [&](auto tag) {
    using T = decltype(tag);
    return launch_bias_rows<T>(static_cast<const T*>(dense), ld, m, n, nullptr, nullptr,
                               static_cast<T*>(out), make_opt<T>(SMB_OPT_NONE, 0, 0),
                               as_stream(stream));
  });
}

extern "C" int smb_bias_grad_update(int dtype, const void* d_out, int64_t ld, int64_t m,
                                    int64_t n, void* bias, void* velocity_bias,
                                    void* grad_bias_out, int opt_kind, double mu, double eta,
                                    void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 0 && n >= 0 && ld >= n, "smb_bias_grad_update: bad shape");
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_bias_grad_update: bad optimizer kind %d", opt_kind);
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) || bias == nullptr ||
                  velocity_bias != nullptr,
              "smb_bias_grad_update: momentum needs a bias velocity buffer");
  return dispatch_dtype(dtype, "smb_bias_grad_update", [&](auto tag) {
    using T = decltype(tag);
    return launch_bias_rows<T>(static_cast<const T*>(d_out), ld, m, n, static_cast<T*>(bias),
                               static_cast<T*>(velocity_bias), static_cast<T*>(grad_bias_out),
                               make_opt<T>(opt_kind, mu, eta), as_stream(stream));
  });
}

extern "C" size_t smb_softmax_ce_workspace_bytes(int64_t n) {
  return 256 + sizeof(double) * (size_t)ceil_div(n > 0 ? n : 1, 128);
}

static int softmax_launch(int dtype, const void* y, int64_t ld_y, const void* t, int64_t ld_t,
                          int64_t classes, int64_t n, double divisor, void* d_y, int64_t ld_dy,
                          double* loss_out, void* bias, void* vbias, void* grad_bias,
                          int opt_kind, double mu, double eta, int32_t* counter, int32_t modulo,
                          void* workspace, void* stream) {
  SMB_REQUIRE(classes >= 1 && n >= 0, "softmax: bad shape");
  SMB_REQUIRE(ld_y >= n && ld_t >= n && ld_dy >= n, "softmax: leading dimension");
  SMB_REQUIRE(divisor != 0.0, "softmax: zero divisor");
  SMB_REQUIRE(n <= (int64_t(1) << 30), "softmax: batch too wide");
  return dispatch_dtype(dtype, "smb_softmax_ce", [&](auto tag) {
    using T = decltype(tag);
    // multi-CTA (128 columns each) needs the workspace (ticket + per-CTA
    // loss partials); without it one CTA loops over all columns
    // One 1024-thread CTA whenever the classes x n block of d_y fits shared
    // memory (it then stays on chip for the bias row sums: no cross-CTA
    // ticket, no global round trip); else 128-column CTAs + last-CTA epilogue
    // (needs the workspace).
    const bool rows = grad_bias != nullptr || (opt_kind != SMB_OPT_NONE && bias != nullptr);
    const size_t block = sizeof(T) * (size_t)(classes * n);
    const size_t leaves1 = sizeof(T) * 32 * (size_t)warp_pairwise_leaves((int)n);
    // (without a bias side the step is a pure per-column map: many CTAs)
    const bool single = !workspace || (rows && leaves1 + block <= 180 * 1024 && n <= 64 * 1024);
    const int threads = single ? 1024 : 128;
    const unsigned grid = single ? 1u : (unsigned)ceil_div(n > 0 ? n : 1, threads);
    unsigned* ticket = workspace ? static_cast<unsigned*>(workspace) : nullptr;
    double* parts = workspace ? reinterpret_cast<double*>(static_cast<char*>(workspace) + 256)
                              : nullptr;
    size_t dyn = rows ? sizeof(T) * (threads / 32) * (size_t)warp_pairwise_leaves((int)n) : 0;
    const int stage = rows && dyn + block <= 180 * 1024;
    if (stage) dyn += block;
    // column-only instance (128-thread bound: no spills) for multi-CTA launches
    auto kern = (rows || single) ? softmax_step_kernel<T, true> : softmax_step_kernel<T, false>;
    if (dyn > 40 * 1024) ensure_smem(kern, dyn);
    launch_k(kern, dim3(grid), dim3(threads), dyn, as_stream(stream), static_cast<const T*>(y),
             ld_y, static_cast<const T*>(t), ld_t, classes, n, static_cast<T>(divisor),
             static_cast<T*>(d_y), ld_dy, loss_out, parts, ticket, static_cast<T*>(bias),
             static_cast<T*>(vbias), static_cast<T*>(grad_bias), make_opt<T>(opt_kind, mu, eta),
             counter, modulo, stage);
    return check_launch("smb_softmax_ce");
  });
}

extern "C" int smb_softmax_ce_grad(int dtype, const void* y, int64_t ld_y, const void* t,
                                   int64_t ld_t, int64_t classes, int64_t n, double divisor,
                                   void* d_y, int64_t ld_dy, double* loss_out, void* stream) {
  clear_error();
  return softmax_launch(dtype, y, ld_y, t, ld_t, classes, n, divisor, d_y, ld_dy, loss_out,
                        nullptr, nullptr, nullptr, SMB_OPT_NONE, 0, 0, nullptr, 0, nullptr,
                        stream);
}

extern "C" int smb_softmax_ce_step(int dtype, const void* y, int64_t ld_y, const void* t,
                                   int64_t ld_t, int64_t classes, int64_t n, double divisor,
                                   void* d_y, int64_t ld_dy, double* loss_out, void* bias,
                                   void* velocity_bias, void* grad_bias_out, int opt_kind,
                                   double mu, double eta, int32_t* step_counter, int32_t modulo,
                                   void* workspace, void* stream) {
  clear_error();
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_softmax_ce_step: bad optimizer kind %d", opt_kind);
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) || bias == nullptr ||
                  velocity_bias != nullptr,
              "smb_softmax_ce_step: momentum needs a bias velocity buffer");
  return softmax_launch(dtype, y, ld_y, t, ld_t, classes, n, divisor, d_y, ld_dy, loss_out, bias,
                        velocity_bias, grad_bias_out, opt_kind, mu, eta, step_counter, modulo,
                        workspace, stream);
}

extern "C" int smb_relu(int dtype, const void* x, int64_t ld_x, int64_t m, int64_t n, void* y,
                        int64_t ld_y, void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 0 && n >= 0 && ld_x >= n && ld_y >= n, "smb_relu: bad shape");
  if (m * n == 0) return SMB_OK;
  return dispatch_dtype(dtype, "smb_relu", [&](auto tag) {
    using T = decltype(tag);
    relu_kernel<T><<<grid_1d(m * n, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const T*>(x), ld_x, m, n, static_cast<T*>(y), ld_y);
    return check_launch("smb_relu");
  });
}

extern "C" int smb_relu_backward(int dtype, const void* d_out, int64_t ld_d, const void* x_cached,
                                 int64_t ld_x, int64_t m, int64_t n, void* out, int64_t ld_out,
                                 void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 0 && n >= 0 && ld_d >= n && ld_x >= n && ld_out >= n,
              "smb_relu_backward: bad shape");
  if (m * n == 0) return SMB_OK;
  return dispatch_dtype(dtype, "smb_relu_backward", [&](auto tag) {
    using T = decltype(tag);
    relu_backward_kernel<T><<<grid_1d(m * n, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const T*>(d_out), ld_d, static_cast<const T*>(x_cached), ld_x, m, n,
        static_cast<T*>(out), ld_out);
    return check_launch("smb_relu_backward");
  });
}

namespace smb {
namespace {
// d_x[j, t] = sum_{i < m, ascending} W[i, j] * d_out[i, t]  (* (mask[j, t] > 0))
// for an output layer of m <= kDenseTMaxRows rows (DenseLinearLayer.backward,
// nn.py:241-255, + ReLU.backward of the layer below, nn.py:89-91).  CTA =
// 256 batch columns x kDenseTRows rows of d_x: every thread keeps its column
// of d_out (m values) in registers, the CTA's W block sits in shared memory,
// and each d_x / mask element is touched once, coalesced.
constexpr int kDenseTMaxRows = 32;
constexpr int kDenseTRows = 16;

// M: the row count when known at compile time (10 = the classes of every
// BASELINE config; no predicated-off work), 0 = any m <= kDenseTMaxRows
template <typename T, bool MASK, int M>
__global__ void __launch_bounds__(256)
    dense_t_kernel(const T* __restrict__ w, int64_t ld_w, int m_rt, int64_t k,
                   const T* __restrict__ d, int64_t ld_d, int64_t n, const T* __restrict__ mask,
                   int64_t ld_mask, T* __restrict__ dx, int64_t ld_dx) {
  constexpr int MR = M > 0 ? M : kDenseTMaxRows;  // unrolled row count
  const int m = M > 0 ? M : m_rt;
  __shared__ T s_w[MR][kDenseTRows];
  const int64_t j0 = (int64_t)blockIdx.y * kDenseTRows;
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  for (int e = threadIdx.x; e < m * kDenseTRows; e += 256) {
    const int i = e / kDenseTRows, jj = e % kDenseTRows;
    s_w[i][jj] = (j0 + jj < k) ? w[(int64_t)i * ld_w + j0 + jj] : T(0);
  }
  pdl_wait();  // d_out / mask are earlier kernels' outputs
  T dv[MR];
#pragma unroll
  for (int i = 0; i < MR; ++i) dv[i] = (i < m && t < n) ? d[(int64_t)i * ld_d + t] : T(0);
  __syncthreads();
  if (t >= n) return;
  const int rows = (int)imin(kDenseTRows, k - j0);
  // the mask column block first: kDenseTRows independent loads in flight
  T mk[kDenseTRows];
#pragma unroll
  for (int jj = 0; jj < kDenseTRows; ++jj)
    mk[jj] = (MASK && jj < rows) ? mask[(j0 + jj) * ld_mask + t] : T(1);
#pragma unroll
  for (int jj = 0; jj < kDenseTRows; ++jj) {
    if (jj >= rows) break;
    T acc = T(0);
#pragma unroll
    for (int i = 0; i < MR; ++i)
      if (M > 0 || i < m) acc = add_rn(acc, mul_rn(s_w[i][jj], dv[i]));
    if (MASK) acc = mask_np(acc, mk[jj]);
    dx[(j0 + jj) * ld_dx + t] = acc;
  }
}

// fp32 with 16-byte aligned columns: the same sums, one CTA per (512-column
// block, run of rows) -- thread = 4 columns, its d_out columns (m float4s) in
// registers for the whole run, the W^T slice of the run in shared memory
// (read as broadcast float4s).  Used without a mask; the masked form streams
// the mask through a bulk-copy ring (next kernel).  The 16-row CTAs above
// spent most of their life in the prologue (W block, d_out loads, barrier).
constexpr int kDtvThreads = 128;
constexpr int kDtvCols = 4 * kDtvThreads;
constexpr int kDtvAhead = 8;

template <bool MASK, int M>
__global__ void __launch_bounds__(kDtvThreads)
    dense_t_vec_kernel(const float* __restrict__ w, int64_t ld_w, int m_rt, int64_t k,
                       int64_t run, const float* __restrict__ d, int64_t ld_d, int64_t n,
                       const float* __restrict__ mask, int64_t ld_mask, float* __restrict__ dx,
                       int64_t ld_dx) {
  constexpr int MR = M > 0 ? M : kDenseTMaxRows;
  constexpr int MP = (MR + 3) & ~3;  // shared row of W^T padded to float4s
  const int m = M > 0 ? M : m_rt;
  extern __shared__ __align__(16) float s_wt[];  // [run][MP]
  const int64_t j0 = (int64_t)blockIdx.y * run;
  const int rows = (int)imin(run, k - j0);
  const int64_t t = ((int64_t)blockIdx.x * kDtvThreads + threadIdx.x) * 4;
  for (int e = threadIdx.x; e < MP * rows; e += kDtvThreads) {
    const int i = e / rows, jj = e % rows;
    s_wt[jj * MP + i] = i < m ? w[(int64_t)i * ld_w + j0 + jj] : 0.f;
  }
  pdl_wait();  // d_out / mask are earlier kernels' outputs
  const bool live = t < n;  // (n % 4 == 0: a live thread owns 4 columns)
  float4 dv[MR];
#pragma unroll
  for (int i = 0; i < MR; ++i)
    dv[i] = (live && (M > 0 || i < m)) ? *reinterpret_cast<const float4*>(d + (int64_t)i * ld_d + t)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 mk[kDtvAhead];
  if (MASK) {
#pragma unroll
    for (int u = 0; u < kDtvAhead; ++u)
      if (live && u < rows) mk[u] = __ldg(reinterpret_cast<const float4*>(mask + (j0 + u) * ld_mask + t));
  }
  __syncthreads();
  if (!live) return;
  for (int r0 = 0; r0 < rows; r0 += kDtvAhead) {
#pragma unroll
    for (int u = 0; u < kDtvAhead; ++u) {
      const int r = r0 + u;
      if (r >= rows) break;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4* wr = reinterpret_cast<const float4*>(s_wt + r * MP);
#pragma unroll
      for (int i4 = 0; i4 < MP / 4; ++i4) {
        const float4 wq = wr[i4];
        const float wv[4] = {wq.x, wq.y, wq.z, wq.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = 4 * i4 + e;
          if (i < MR && (M > 0 || i < m)) {
            acc.x = add_rn(acc.x, mul_rn(wv[e], dv[i].x));
            acc.y = add_rn(acc.y, mul_rn(wv[e], dv[i].y));
            acc.z = add_rn(acc.z, mul_rn(wv[e], dv[i].z));
            acc.w = add_rn(acc.w, mul_rn(wv[e], dv[i].w));
          }
        }
      }
      if (MASK) {
        const float4 q = mk[u];
        acc.x = mask_np(acc.x, q.x);
        acc.y = mask_np(acc.y, q.y);
        acc.z = mask_np(acc.z, q.z);
        acc.w = mask_np(acc.w, q.w);
        if (r + kDtvAhead < rows)
          mk[u] = __ldg(reinterpret_cast<const float4*>(mask + (j0 + r + kDtvAhead) * ld_mask + t));
      }
      *reinterpret_cast<float4*>(dx + (j0 + r) * ld_dx + t) = acc;
    }
  }
}

// The masked form (the hot one: the step's ReLU backward of the layer below)
// with the mask rows streamed by 1-D bulk copies into a shared-memory ring
// instead of registers: 5 stages x 8 rows x 2 KB in flight per CTA, two CTAs
// per SM.  With the register ring above (8 float4 loads per thread, 123
// registers, 16 warps per SM) config 5 read + wrote at ~3.4 TB/s, 36% of
// DRAM in ncu.
constexpr int kDtrRows = 8;
constexpr int kDtrStages = 5;
constexpr int64_t kDtrRingBytes = (int64_t)kDtrStages * kDtrRows * kDtvCols * 4;

template <int M>
__global__ void __launch_bounds__(kDtvThreads)
    dense_t_ring_kernel(const float* __restrict__ w, int64_t ld_w, int m_rt, int64_t k,
                        int64_t run, const float* __restrict__ d, int64_t ld_d, int64_t n,
                        const float* __restrict__ mask, int64_t ld_mask, float* __restrict__ dx,
                        int64_t ld_dx) {
  constexpr int MR = M > 0 ? M : kDenseTMaxRows;
  constexpr int MP = (MR + 3) & ~3;
  const int m = M > 0 ? M : m_rt;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw);           // [stages][rows][kDtvCols]
  float* s_wt = reinterpret_cast<float*>(smem_raw + kDtrRingBytes);  // [run][MP]
  __shared__ __align__(8) unsigned long long full[kDtrStages];
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * kDtvCols;
  const unsigned row_bytes = 4u * (unsigned)imin(kDtvCols, n - c0);  // (n % 4 == 0)
  const int64_t j0 = (int64_t)blockIdx.y * run;
  const int rows = (int)imin(run, k - j0);
  const int64_t t = c0 + 4 * tid;
  const bool live = t < n;
  if (tid == 0) {
    for (int s = 0; s < kDtrStages; ++s) bulk::mbar_init(bulk::smem_u32(&full[s]), 1);
    bulk::fence_init();
  }
  for (int e = tid; e < MP * rows; e += kDtvThreads) {
    const int i = e / rows, jj = e % rows;
    s_wt[jj * MP + i] = i < m ? w[(int64_t)i * ld_w + j0 + jj] : 0.f;
  }
  pdl_wait();  // d_out / mask are earlier kernels' outputs
  float4 dv[MR];
#pragma unroll
  for (int i = 0; i < MR; ++i)
    dv[i] = (live && (M > 0 || i < m)) ? *reinterpret_cast<const float4*>(d + (int64_t)i * ld_d + t)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();  // barriers initialised, W^T slice staged
  const int nst = (rows + kDtrRows - 1) / kDtrRows;
  auto issue = [&](int st) {
    const int slot = st % kDtrStages;
    const int rb = st * kDtrRows;
    const int nr = min(kDtrRows, rows - rb);
    const unsigned bar = bulk::smem_u32(&full[slot]);
    bulk::arrive_expect_tx(bar, (unsigned)nr * row_bytes);
    for (int rr = 0; rr < nr; ++rr)
      bulk::g2s(bulk::smem_u32(ring + (slot * kDtrRows + rr) * kDtvCols),
                mask + (j0 + rb + rr) * ld_mask + c0, row_bytes, bar);
  };
  if (tid == 0)
    for (int st = 0; st < kDtrStages && st < nst; ++st) issue(st);
  for (int st = 0; st < nst; ++st) {
    const int slot = st % kDtrStages;
    bulk::wait(bulk::smem_u32(&full[slot]), (unsigned)((st / kDtrStages) & 1));
    const int rb = st * kDtrRows;
    const int nr = min(kDtrRows, rows - rb);
    if (live) {
#pragma unroll
      for (int rr = 0; rr < kDtrRows; ++rr) {
        if (rr >= nr) break;
        const int r = rb + rr;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4* wr = reinterpret_cast<const float4*>(s_wt + r * MP);
#pragma unroll
        for (int i4 = 0; i4 < MP / 4; ++i4) {
          const float4 wq = wr[i4];
          const float wv[4] = {wq.x, wq.y, wq.z, wq.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 4 * i4 + e;
            if (i < MR && (M > 0 || i < m)) {
              acc.x = add_rn(acc.x, mul_rn(wv[e], dv[i].x));
              acc.y = add_rn(acc.y, mul_rn(wv[e], dv[i].y));
              acc.z = add_rn(acc.z, mul_rn(wv[e], dv[i].z));
              acc.w = add_rn(acc.w, mul_rn(wv[e], dv[i].w));
            }
          }
        }
        const float4 q =
            *reinterpret_cast<const float4*>(ring + (slot * kDtrRows + rr) * kDtvCols + 4 * tid);
        acc.x = mask_np(acc.x, q.x);
        acc.y = mask_np(acc.y, q.y);
        acc.z = mask_np(acc.z, q.z);
        acc.w = mask_np(acc.w, q.w);
        *reinterpret_cast<float4*>(dx + (j0 + r) * ld_dx + t) = acc;
      }
    }
    __syncthreads();  // every thread has read the stage: refill it
    if (tid == 0 && st + kDtrStages < nst) issue(st + kDtrStages);
  }
}
}  // namespace
}  // namespace smb

namespace smb {
namespace {
// y[i, t] = bias[i] + sum_s part[s][i][t], part[s][i][t] = sum_{j in slice s,
// ascending} W[i, j] * x[j, t] (fused multiply-add): the forward of a small
// dense output layer (m <= kDenseTMaxRows; DenseLinearLayer.forward,
// nn.py:241-255, numpy BLAS -- tolerance parity) as a deterministic split-K
// pass.  CTA = 128 batch columns x one K slice (thread per column, the W
// slice in shared memory), 8 x loads in flight per thread; a second launch
// sums the slices in ascending order.  Replaces a cuBLAS SIMT GEMM that ran
// 30-35 us on the 10 x 8192 x 1024 config-4 shape.
constexpr int kDfCols = 128;

constexpr int64_t kDfMaxSlice = 768;  // 768 x 32 x 8 B = 192 KB of shared memory

struct DenseFwdPlan {
  int64_t slices, ks, col_blocks;
};
inline DenseFwdPlan dense_fwd_plan(int64_t k, int64_t n, int cw = 4) {
  DenseFwdPlan p;
  p.col_blocks = ceil_div(n > 0 ? n : 1, kDfCols * cw);
  // ~1024 CTAs (7 resident per SM, 16 x loads of 16 bytes in flight per
  // thread keep HBM busy; 256 CTAs left config 5's 134 MB x at 25% of HBM),
  // slices of >= 64 rows so the partial sums stay small next to x
  int64_t s = ceil_div(1024, p.col_blocks);
  s = imax(1, imin(s, ceil_div(k > 0 ? k : 1, cw > 1 ? 64 : 32)));
  p.ks = ceil_div(ceil_div(k > 0 ? k : 1, s), 32) * 32;
  // the W^T slice lives in shared memory (ks x 32 padded rows x 8 bytes at
  // most): cap the slice so it fits the 227 KB opt-in limit for every m,
  // dtype and width (the workspace size uses the same plan)
  p.ks = imin(p.ks, kDfMaxSlice);
  p.slices = ceil_div(k > 0 ? k : 1, p.ks);
  return p;
}

// CW columns per thread: 16 / sizeof(T) with 16-byte x loads (aligned x),
// else 1
template <typename T, int M, int CW>
__global__ void __launch_bounds__(kDfCols)
    dense_fwd_part_kernel(const T* __restrict__ w, int64_t ld_w, int m_rt, int64_t k, int64_t ks,
                          const T* __restrict__ x, int64_t ld_x, int64_t n, T* __restrict__ part) {
  constexpr int MR = M > 0 ? M : kDenseTMaxRows;
  constexpr int VW = 16 / sizeof(T);
  constexpr int MP = (MR + VW - 1) / VW * VW;  // smem row padded to 16-byte vectors
  using V = typename Vec16<T>::type;
  const int m = M > 0 ? M : m_rt;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_w = reinterpret_cast<T*>(smem_raw);  // [ks][MP]: W^T of the slice
  const int64_t j0 = (int64_t)blockIdx.y * ks;
  const int len = (int)imin(ks, k - j0);
  for (int e = threadIdx.x; e < MP * len; e += kDfCols) {
    const int i = e / len, jj = e % len;
    s_w[jj * MP + i] = i < m ? w[(int64_t)i * ld_w + j0 + jj] : T(0);
  }
  pdl_wait();  // x is the previous kernel's output
  __syncthreads();
  const int64_t t = ((int64_t)blockIdx.x * kDfCols + threadIdx.x) * CW;
  if (t >= n) return;
  const bool full = t + CW <= n;  // (CW > 1: n % CW == 0 is required by the host)
  T acc[MR][CW];
#pragma unroll
  for (int i = 0; i < MR; ++i)
#pragma unroll
    for (int c = 0; c < CW; ++c) acc[i][c] = T(0);
  const T* xp = x + j0 * ld_x + t;
  constexpr int U = CW > 1 ? 16 : 8;  // x loads in flight per thread
  auto fma_row = [&](int jj, const T(&xv)[CW]) {
    const V* wr = reinterpret_cast<const V*>(s_w + jj * MP);  // broadcast 16-byte reads
#pragma unroll
    for (int q = 0; q < MP / VW; ++q) {
      const V wv = wr[q];
#pragma unroll
      for (int r = 0; r < VW; ++r) {
        const int i = q * VW + r;
        if (i < MR && (M > 0 || i < m)) {
          const T wi = VecOps<T>::get(wv, r);
#pragma unroll
          for (int c = 0; c < CW; ++c) acc[i][c] = fma(wi, xv[c], acc[i][c]);
        }
      }
    }
  };
  auto load = [&](int jj, T(&xv)[CW]) {
    if constexpr (CW > 1) {
      const V v = *reinterpret_cast<const V*>(xp + (int64_t)jj * ld_x);
#pragma unroll
      for (int c = 0; c < CW; ++c) xv[c] = VecOps<T>::get(v, c);
    } else {
      xv[0] = xp[(int64_t)jj * ld_x];
    }
  };
  (void)full;
  int jj = 0;
  for (; jj + U <= len; jj += U) {
    T xv[U][CW];
#pragma unroll
    for (int u = 0; u < U; ++u) load(jj + u, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) fma_row(jj + u, xv[u]);
  }
  for (; jj < len; ++jj) {
    T xv[CW];
    load(jj, xv);
    fma_row(jj, xv);
  }
  pdl_trigger();
  T* pp = part + (int64_t)blockIdx.y * m * n + t;
#pragma unroll
  for (int i = 0; i < MR; ++i)
    if (M > 0 || i < m) {
#pragma unroll
      for (int c = 0; c < CW; ++c) pp[(int64_t)i * n + c] = acc[i][c];
    }
}

// y[i, t] = bias[i] + sum of the slices' partials: a CTA = 32 consecutive
// outputs x 32 slice groups; group g sums slices g, g + 32, ... in order
// (coalesced over the outputs), then the 32 group sums are added in a fixed
// pairwise tree (deterministic).
constexpr int kDfSumG = 32;

template <typename T>
__global__ void __launch_bounds__(32 * kDfSumG)
    dense_fwd_sum_kernel(const T* __restrict__ part, int64_t slices, int64_t m, int64_t n,
                         const T* __restrict__ bias, T* __restrict__ y, int64_t ld_y) {
  __shared__ T s_acc[kDfSumG][33];
  pdl_wait();
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + c;
  const int64_t mn = m * n;
  T acc = T(0);
  if (e < mn) {
    int64_t s = g;
    for (; s + 3 * kDfSumG < slices; s += 4 * kDfSumG) {  // 4 loads in flight
      const T v0 = part[s * mn + e], v1 = part[(s + kDfSumG) * mn + e],
              v2 = part[(s + 2 * kDfSumG) * mn + e], v3 = part[(s + 3 * kDfSumG) * mn + e];
      acc += v0;
      acc += v1;
      acc += v2;
      acc += v3;
    }
    for (; s < slices; s += kDfSumG) acc += part[s * mn + e];
  }
  s_acc[g][c] = acc;
  __syncthreads();
  for (int h = kDfSumG / 2; h >= 1; h >>= 1) {
    if (g < h) s_acc[g][c] += s_acc[g + h][c];
    __syncthreads();
  }
  if (g == 0 && e < mn) {
    const int64_t i = e / n, t = e - i * n;
    y[i * ld_y + t] = (bias ? bias[i] : T(0)) + s_acc[0][c];
  }
}
}  // namespace
}  // namespace smb

extern "C" size_t smb_dense_forward_workspace_bytes(int64_t m, int64_t k, int64_t n) {
  int64_t slices = 0;
  for (int cw : {1, 2, 4}) slices = imax(slices, dense_fwd_plan(k, n, cw).slices);
  return (size_t)(slices * (m > 0 ? m : 1) * (n > 0 ? n : 1)) * sizeof(double);
}

extern "C" int smb_dense_forward_small(int dtype, const void* w, int64_t ld_w, int64_t m,
                                       int64_t k, const void* x, int64_t ld_x, int64_t n,
                                       const void* bias, void* y, int64_t ld_y, void* workspace,
                                       void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 1 && m <= kDenseTMaxRows, "smb_dense_forward_small: needs 1 <= m <= %d",
              kDenseTMaxRows);
  SMB_REQUIRE(k >= 0 && n >= 0 && ld_y >= n && (k == 0 || (ld_w >= k && ld_x >= n)),
              "smb_dense_forward_small: bad shape");
  if (n == 0) return SMB_OK;
  SMB_REQUIRE(y && workspace && (k == 0 || (w && x)), "smb_dense_forward_small: null pointer");
  return dispatch_dtype(dtype, "smb_dense_forward_small", [&](auto tag) {
    using T = decltype(tag);
    T* part = static_cast<T*>(workspace);
    constexpr int VW = 16 / (int)sizeof(T);
    // 16-byte x loads (VW columns per thread) unless that leaves too few CTAs
    // (small k): then one column per thread
    bool vec = aligned16(x) && ld_x % VW == 0 && n % VW == 0;
    if (vec) {
      const DenseFwdPlan pv = dense_fwd_plan(k, n, VW);
      vec = pv.col_blocks * pv.slices >= 148;
    }
    const DenseFwdPlan p = dense_fwd_plan(k, n, vec ? VW : 1);
    if (k == 0) {  // y = bias
      cudaMemsetAsync(part, 0, sizeof(T) * m * n, as_stream(stream));
    } else {
      const dim3 grid((unsigned)p.col_blocks, (unsigned)p.slices);
      const int vw = 16 / (int)sizeof(T);
      const int mr = ((m == 10 ? 10 : kDenseTMaxRows) + vw - 1) / vw * vw;  // padded row
      const size_t smem = sizeof(T) * (size_t)p.ks * mr;
      auto go = [&](auto kernel) {
        ensure_smem(kernel, smem);
        launch_k(kernel, grid, dim3(kDfCols), smem, as_stream(stream),
                 static_cast<const T*>(w), ld_w, (int)m, k, p.ks, static_cast<const T*>(x),
                 ld_x, n, part);
      };
      if (m == 10 && vec)
        go(dense_fwd_part_kernel<T, 10, VW>);
      else if (m == 10)
        go(dense_fwd_part_kernel<T, 10, 1>);
      else if (vec)
        go(dense_fwd_part_kernel<T, 0, VW>);
      else
        go(dense_fwd_part_kernel<T, 0, 1>);
    }
    launch_k(dense_fwd_sum_kernel<T>, dim3((unsigned)ceil_div(m * n, 32)), dim3(32 * kDfSumG), 0,
             as_stream(stream), static_cast<const T*>(part), k == 0 ? int64_t(1) : p.slices,
             m, n, static_cast<const T*>(bias), static_cast<T*>(y), ld_y);
    return check_launch("smb_dense_forward_small");
  });
}

extern "C" int smb_dense_backward_input(int dtype, const void* w, int64_t ld_w, int64_t m,
                                        int64_t k, const void* d_out, int64_t ld_d, int64_t n,
                                        const void* mask, int64_t ld_mask, void* d_x,
                                        int64_t ld_dx, void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 1 && m <= kDenseTMaxRows, "smb_dense_backward_input: needs 1 <= m <= %d",
              kDenseTMaxRows);
  SMB_REQUIRE(k >= 0 && n >= 0 && ld_w >= k && ld_d >= n && ld_dx >= n &&
                  (mask == nullptr || ld_mask >= n),
              "smb_dense_backward_input: bad shape");
  if (k == 0 || n == 0) return SMB_OK;
  SMB_REQUIRE(w && d_out && d_x, "smb_dense_backward_input: null pointer");
  return dispatch_dtype(dtype, "smb_dense_backward_input", [&](auto tag) {
    using T = decltype(tag);
    if constexpr (std::is_same<T, float>::value) {
      const bool vec = n % 4 == 0 && ld_d % 4 == 0 && ld_dx % 4 == 0 && aligned16(d_out) &&
                       aligned16(d_x) && (mask == nullptr || (ld_mask % 4 == 0 && aligned16(mask)));
      if (vec) {
        // ~8 CTAs of 4 warps per SM over the column blocks x runs of rows
        const int64_t cb = ceil_div(n, kDtvCols);
        const int64_t groups = imax(1, (148 * 8) / cb);
        const int64_t cap = m == 10 ? 1024 : 384;  // W^T slice <= 48 KB of shared memory
        const int64_t run = imin(cap, imax(16, ceil_div(k, groups)));
        const int mp = m == 10 ? 12 : ((kDenseTMaxRows + 3) & ~3);
        const dim3 grid((unsigned)cb, (unsigned)ceil_div(k, run));
        const size_t smem = (size_t)run * mp * sizeof(float);
        auto gov = [&](auto kernel) {
          launch_k(kernel, grid, dim3(kDtvThreads), smem, as_stream(stream),
                   static_cast<const float*>(w), ld_w, (int)m, k, run,
                   static_cast<const float*>(d_out), ld_d, n, static_cast<const float*>(mask),
                   ld_mask, static_cast<float*>(d_x), ld_dx);
        };
        if (mask) {
          // bulk-copy ring: two CTAs per SM, W^T slices of <= ~24 KB
          const int64_t rcap = m == 10 ? 512 : 192;
          const int64_t rgroups = imax(ceil_div(k, rcap), ceil_div(2 * 148, cb));
          const int64_t rrun = ceil_div(k, rgroups);
          const size_t rsmem = (size_t)kDtrRingBytes + (size_t)rrun * mp * sizeof(float);
          auto gor = [&](auto kernel) {
            ensure_smem(kernel, rsmem);
            launch_k(kernel, dim3((unsigned)cb, (unsigned)ceil_div(k, rrun)), dim3(kDtvThreads),
                     rsmem, as_stream(stream), static_cast<const float*>(w), ld_w, (int)m, k, rrun,
                     static_cast<const float*>(d_out), ld_d, n, static_cast<const float*>(mask),
                     ld_mask, static_cast<float*>(d_x), ld_dx);
          };
          if (m == 10)
            gor(dense_t_ring_kernel<10>);
          else
            gor(dense_t_ring_kernel<0>);
        } else if (m == 10) {
          gov(dense_t_vec_kernel<false, 10>);
        } else {
          gov(dense_t_vec_kernel<false, 0>);
        }
        return check_launch("smb_dense_backward_input");
      }
    }
    const dim3 grid((unsigned)ceil_div(n, 256), (unsigned)ceil_div(k, kDenseTRows));
    auto go = [&](auto kernel) {
      launch_k(kernel, grid, dim3(256), 0, as_stream(stream), static_cast<const T*>(w), ld_w,
               (int)m, k, static_cast<const T*>(d_out), ld_d, n, static_cast<const T*>(mask),
               ld_mask, static_cast<T*>(d_x), ld_dx);
    };
    if (mask && m == 10)
      go(dense_t_kernel<T, true, 10>);
    else if (m == 10)
      go(dense_t_kernel<T, false, 10>);
    else if (mask)
      go(dense_t_kernel<T, true, 0>);
    else
      go(dense_t_kernel<T, false, 0>);
    return check_launch("smb_dense_backward_input");
  });
}

static int gather_launch(int dtype, const void* src, int64_t n_samples, int64_t features,
                         const int32_t* perm, const int32_t* step_counter, int64_t base,
                         int32_t step_offset, int32_t modulo, int64_t batch, void* dst,
                         int64_t ld_dst, void* stream);

extern "C" int smb_gather_columns(int dtype, const void* src, int64_t n_samples, int64_t features,
                                  const int32_t* perm, const int32_t* step_counter, int64_t base,
                                  int64_t batch, void* dst, int64_t ld_dst, void* stream) {
  return gather_launch(dtype, src, n_samples, features, perm, step_counter, base, 0, 0, batch,
                       dst, ld_dst, stream);
}

extern "C" int smb_gather_columns_ahead(int dtype, const void* src, int64_t n_samples,
                                        int64_t features, const int32_t* perm,
                                        const int32_t* step_counter, int32_t step_offset,
                                        int32_t modulo, int64_t batch, void* dst, int64_t ld_dst,
                                        void* stream) {
  clear_error();
  SMB_REQUIRE(step_counter != nullptr, "smb_gather_columns_ahead: null step counter");
  SMB_REQUIRE(step_offset >= 0 && modulo >= 0, "smb_gather_columns_ahead: bad offset / modulo");
  return gather_launch(dtype, src, n_samples, features, perm, step_counter, 0, step_offset,
                       modulo, batch, dst, ld_dst, stream);
}

static int gather_launch(int dtype, const void* src, int64_t n_samples, int64_t features,
                         const int32_t* perm, const int32_t* step_counter, int64_t base,
                         int32_t step_offset, int32_t modulo, int64_t batch, void* dst,
                         int64_t ld_dst, void* stream) {
  clear_error();
  SMB_REQUIRE(n_samples >= 0 && features >= 0 && batch >= 0 && ld_dst >= batch,
              "smb_gather_columns: bad shape");
  SMB_REQUIRE(step_counter != nullptr || (base >= 0 && base + batch <= n_samples),
              "smb_gather_columns: batch [%lld, %lld) outside the %lld samples", (long long)base,
              (long long)(base + batch), (long long)n_samples);
  if (batch == 0 || features == 0) return SMB_OK;
  return dispatch_dtype(dtype, "smb_gather_columns", [&](auto tag) {
    using T = decltype(tag);
    dim3 grid((unsigned)ceil_div(batch, 32), (unsigned)ceil_div(features, 128));
    const bool vec = aligned16(src) && (features * (int64_t)sizeof(T)) % 16 == 0;
#ifndef SMB_GATHER_PAD
#define SMB_GATHER_PAD 24576
#endif
    // The gather AHEAD runs beside the training step's kernels; in the
    // chain-kernel step beside the chain, whose CTAs fill 128 SMs with 204 KB
    // of shared memory each.  A 24 KB shared-memory reservation (unused) keeps
    // the gather's CTAs off those SMs, on the 20 the chain leaves free: the
    // chain is no longer slowed by them (config 2: 60.8 -> 58.4 us per step
    // with the L2 flush, 19.0 -> 19.2 M samples/s back to back; 6 / 12 / 16 /
    // 28 KB: 59.4 / 59.4 / 59.5 / 58.5 us).
    const size_t pad = step_counter != nullptr ? SMB_GATHER_PAD : 0;
    if (vec)
      launch_k(gather_columns_kernel<T, true>, grid, dim3(256), pad, as_stream(stream),
               static_cast<const T*>(src), features, perm, step_counter, base, step_offset,
               modulo, batch, static_cast<T*>(dst), ld_dst);
    else
      launch_k(gather_columns_kernel<T, false>, grid, dim3(256), 0, as_stream(stream),
               static_cast<const T*>(src), features, perm, step_counter, base, step_offset,
               modulo, batch, static_cast<T*>(dst), ld_dst);
    return check_launch("smb_gather_columns");
  });
}

namespace smb {
__global__ void step_counter_kernel(int32_t* counter, int32_t modulo) {
  const int32_t v = *counter + 1;
  *counter = (modulo > 0 && v >= modulo) ? 0 : v;
}
}  // namespace smb

extern "C" int smb_step_counter_advance(int32_t* counter, int32_t modulo, void* stream) {
  clear_error();
  SMB_REQUIRE(counter != nullptr, "smb_step_counter_advance: null counter");
  step_counter_kernel<<<1, 1, 0, as_stream(stream)>>>(counter, modulo);
  return check_launch("smb_step_counter_advance");
}
