// Memory-bound glue of the training step: sparse_combine (axpby), the
// optimizer update of flat segments, numpy-order row sums, softmax
// cross-entropy gradient, ReLU forward/backward, the device batch gather and
// the CUDA-graph step counter.
#include "common.cuh"

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

// ---- numpy pairwise row sums (tensor_core.py:353-356) ----------------------
template <typename T>
__global__ void row_sums_kernel(const T* __restrict__ a, int64_t m, int64_t n, int64_t ld,
                                T* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = pairwise_sum(a + i * ld, n);
}

// ---- softmax cross-entropy gradient (nn.py:385-417, train.py:399) ---------
// One thread per sample column; a single CTA so the optional batch loss is
// reduced in a fixed order.
template <typename T>
__global__ void softmax_ce_kernel(const T* __restrict__ y, int64_t ld_y, const T* __restrict__ t,
                                  int64_t ld_t, int64_t classes, int64_t n, T divisor,
                                  T* __restrict__ dy, int64_t ld_dy, double* loss_out) {
  __shared__ double part[1024];
  double local = 0.0;
  for (int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; col < n;
       col += (int64_t)gridDim.x * blockDim.x) {
    // z = y - y.max(axis=0)
    T mx = y[col];
    for (int64_t c = 1; c < classes; ++c) {
      const T v = y[c * ld_y + col];
      mx = (v > mx || v != v) ? v : mx;
    }
    // e.sum(axis=0): sequential over classes (numpy axis-0 reduce order)
    T s = T(0);
    double zt = 0.0;
    for (int64_t c = 0; c < classes; ++c) {
      const T z = sub_rn(y[c * ld_y + col], mx);
      const T e = static_cast<T>(exp(static_cast<double>(z)));
      s = add_rn(s, e);
      zt += static_cast<double>(z) * static_cast<double>(t[c * ld_t + col]);
    }
    for (int64_t c = 0; c < classes; ++c) {
      const T z = sub_rn(y[c * ld_y + col], mx);
      const T e = static_cast<T>(exp(static_cast<double>(z)));
      const T pr = div_rn(e, s);
      dy[c * ld_dy + col] = div_rn(sub_rn(pr, t[c * ld_t + col]), divisor);
    }
    local += log(static_cast<double>(s)) - zt;
  }
  if (loss_out == nullptr) return;
  part[threadIdx.x] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) tot += part[i];
    *loss_out = tot;
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
// dst[f, j] = src[perm[base + j], f]: 32 samples x 32 features per tile,
// coalesced on both sides through a padded shared-memory transpose.
template <typename T>
__global__ void gather_columns_kernel(const T* __restrict__ src, int64_t features,
                                      const int32_t* __restrict__ perm,
                                      const int32_t* __restrict__ step_counter, int64_t base,
                                      int64_t batch, T* __restrict__ dst, int64_t ld_dst) {
  __shared__ T tile[32][33];
  __shared__ int32_t s_idx[32];
  const int64_t b0 = step_counter ? (int64_t)(*step_counter) * batch : base;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t f0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (ty == 0) s_idx[tx] = (j0 + tx < batch) ? perm[b0 + j0 + tx] : -1;
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int32_t sidx = s_idx[r];
    if (sidx >= 0 && f0 + tx < features) tile[r][tx] = src[(int64_t)sidx * features + f0 + tx];
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    if (f0 + r < features && j0 + tx < batch) dst[(f0 + r) * ld_dst + j0 + tx] = tile[tx][r];
  }
}

__global__ void step_counter_kernel(int32_t* counter, int32_t modulo) {
  const int32_t v = *counter + 1;
  *counter = (modulo > 0 && v >= modulo) ? 0 : v;
}

template <typename T>
int dispatch_dtype(int dtype, const char* name, T&& fn) {
  if (dtype == SMB_F32) return fn(float{});
  if (dtype == SMB_F64) return fn(double{});
  set_error("%s: unsupported dtype %d", name, dtype);
  return SMB_ERR_INVALID;
}

}  // namespace
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

extern "C" int smb_row_sums(int dtype, const void* dense, int64_t m, int64_t n, int64_t ld,
                            void* out, void* stream) {
  clear_error();
  SMB_REQUIRE(m >= 0 && n >= 0 && ld >= n, "smb_row_sums: bad shape");
  if (m == 0) return SMB_OK;
  return dispatch_dtype(dtype, "smb_row_sums", [&](auto tag) {
    using T = decltype(tag);
    row_sums_kernel<T><<<(unsigned)ceil_div(m, 128), 128, 0, as_stream(stream)>>>(
        static_cast<const T*>(dense), m, n, ld, static_cast<T*>(out));
    return check_launch("smb_row_sums");
  });
}

extern "C" int smb_softmax_ce_grad(int dtype, const void* y, int64_t ld_y, const void* t,
                                   int64_t ld_t, int64_t classes, int64_t n, double divisor,
                                   void* d_y, int64_t ld_dy, double* loss_out, void* stream) {
  clear_error();
  SMB_REQUIRE(classes >= 1 && n >= 0, "smb_softmax_ce_grad: bad shape");
  SMB_REQUIRE(ld_y >= n && ld_t >= n && ld_dy >= n, "smb_softmax_ce_grad: leading dimension");
  SMB_REQUIRE(divisor != 0.0, "smb_softmax_ce_grad: zero divisor");
  return dispatch_dtype(dtype, "smb_softmax_ce_grad", [&](auto tag) {
    using T = decltype(tag);
    // one CTA keeps the optional loss reduction in a fixed order
    softmax_ce_kernel<T><<<1, 1024, 0, as_stream(stream)>>>(
        static_cast<const T*>(y), ld_y, static_cast<const T*>(t), ld_t, classes, n,
        static_cast<T>(divisor), static_cast<T*>(d_y), ld_dy, loss_out);
    return check_launch("smb_softmax_ce_grad");
  });
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

extern "C" int smb_gather_columns(int dtype, const void* src, int64_t n_samples, int64_t features,
                                  const int32_t* perm, const int32_t* step_counter, int64_t base,
                                  int64_t batch, void* dst, int64_t ld_dst, void* stream) {
  clear_error();
  SMB_REQUIRE(n_samples >= 0 && features >= 0 && batch >= 0 && ld_dst >= batch,
              "smb_gather_columns: bad shape");
  SMB_REQUIRE(step_counter != nullptr || (base >= 0 && base + batch <= n_samples),
              "smb_gather_columns: batch [%lld, %lld) outside the %lld samples", (long long)base,
              (long long)(base + batch), (long long)n_samples);
  if (batch == 0 || features == 0) return SMB_OK;
  return dispatch_dtype(dtype, "smb_gather_columns", [&](auto tag) {
    using T = decltype(tag);
    dim3 grid((unsigned)ceil_div(batch, 32), (unsigned)ceil_div(features, 32));
    gather_columns_kernel<T><<<grid, dim3(32, 8), 0, as_stream(stream)>>>(
        static_cast<const T*>(src), features, perm, step_counter, base, batch,
        static_cast<T*>(dst), ld_dst);
    return check_launch("smb_gather_columns");
  });
}

extern "C" int smb_step_counter_advance(int32_t* counter, int32_t modulo, void* stream) {
  clear_error();
  SMB_REQUIRE(counter != nullptr, "smb_step_counter_advance: null counter");
  step_counter_kernel<<<1, 1, 0, as_stream(stream)>>>(counter, modulo);
  return check_launch("smb_step_counter_advance");
}
