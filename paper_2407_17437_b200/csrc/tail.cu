// Fused output-layer tail of the training step (sm_100a):
//
//     y   = W h + b                  SparseLinearLayer.forward   nn.py:169-176
//     d_y = (softmax(y) - t) / B     softmax_ce_gradient, / B    nn.py:411-417, train.py:399
//     loss = sum_col log(sum e) - z.t                            nn.py:397-408
//     d_h = (W^T d_y) * (h > 0)      spmm_transposed + ReLU.bwd  nn.py:185, 89-91
//
// Every batch column is independent in all three products, so one CTA owns
// kTailCols = 8 batch columns end to end and the three launches of the
// unfused step (spmm, softmax step, transposed spmm) become one; at B = 1024
// that is 128 CTAs.  Before any arithmetic the CTA stages, with batched
// independent loads, everything it reads: the [k x 8] slab of h, W's CSR
// arrays, W's CSC (row, value) entries with the values permuted into CSC
// order, and the [m x 8] targets.  The three phases then run from shared
// memory, each product first computed (and rounded) by all threads in
// parallel into a [nnz x 8] buffer, then summed in the reference's order by
// one thread per output element -- the sequential chains no longer wait on
// dependent index -> operand loads:
//   1. logits: thread (r, col) adds CSR row r's products in ascending column
//      (separately rounded multiply and add, zero-initialised:
//      _kernels.py:25-37), + bias;
//   2. 8 threads: column softmax-CE exactly as softmax_step_kernel computes it;
//   3. d_h: thread (c, col) adds CSC column c's products in ascending row
//      (_kernels.py:40-59), times the ReLU mask of h.
// The per-CTA loss partials are summed in CTA order by the last CTA to
// finish (ticket), which also advances the device step counter.  The bias
// row sums of d_y and d_h (nn.py:184) are not here: they cross columns and
// run beside the critical path (smb_bias_grad_update on a side stream).
#include "pattern.cuh"

namespace smb {
namespace {

constexpr int kTailCols = 8;                 // batch columns per CTA
constexpr int kTailThreads = 512;
constexpr int kTailMaxClasses = 32;
constexpr int kTailPad = 8;             // s_idx / s_val tail padding
constexpr int kTailHs = kTailCols + 1;  // padded h-slab row (fewer bank conflicts)

// one CSC entry, read with a single 8 / 16-byte shared-memory load
template <typename T>
struct alignas(2 * sizeof(T) > 8 ? 16 : 8) CscEntry {
  int32_t row;
  T val;
};

template <typename T>
struct TailLayout {
  size_t h, val, ent, prod, y, dy, t, idx, rp, cp, total;
  size_t o = 0;
  __host__ __device__ size_t take(size_t bytes) {
    const size_t at = o;
    o += (bytes + 15) & ~size_t(15);
    return at;
  }
  __host__ __device__ TailLayout(int64_t m, int64_t k, int64_t nnz) {
    h = take(sizeof(T) * k * kTailHs);
    val = take(sizeof(T) * (nnz + kTailPad));
    ent = take(sizeof(CscEntry<T>) * nnz);
    prod = take(sizeof(T) * nnz * kTailCols);
    y = take(sizeof(T) * m * kTailCols);
    dy = take(sizeof(T) * m * kTailCols);
    t = take(sizeof(T) * m * kTailCols);
    idx = take(sizeof(int32_t) * (nnz + kTailPad));
    rp = take(sizeof(int32_t) * (m + 1));
    cp = take(sizeof(int32_t) * (k + 1));
    total = o;
  }
};

template <typename T>
__global__ void __launch_bounds__(kTailThreads)
    tail_step_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                     const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
                     const int32_t* __restrict__ perm, const T* __restrict__ vals, int m, int k,
                     int nnz, const T* __restrict__ h, int64_t ld_h, int mask,
                     const T* __restrict__ bias, const T* __restrict__ t, int64_t ld_t, int64_t n,
                     T divisor, T* __restrict__ y, int64_t ld_y, T* __restrict__ dy,
                     int64_t ld_dy, T* __restrict__ dh, int64_t ld_dh, double* loss_out,
                     double* loss_parts, unsigned* ticket, int32_t* counter, int32_t modulo) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const TailLayout<T> L(m, k, nnz);
  T* s_h = reinterpret_cast<T*>(smem_raw + L.h);
  T* s_val = reinterpret_cast<T*>(smem_raw + L.val);
  CscEntry<T>* s_ent = reinterpret_cast<CscEntry<T>*>(smem_raw + L.ent);
  T* s_p = reinterpret_cast<T*>(smem_raw + L.prod);  // [nnz][kTailCols] products
  T* s_y = reinterpret_cast<T*>(smem_raw + L.y);
  T* s_dy = reinterpret_cast<T*>(smem_raw + L.dy);
  T* s_t = reinterpret_cast<T*>(smem_raw + L.t);
  int32_t* s_idx = reinterpret_cast<int32_t*>(smem_raw + L.idx);
  int32_t* s_rp = reinterpret_cast<int32_t*>(smem_raw + L.rp);
  int32_t* s_cp = reinterpret_cast<int32_t*>(smem_raw + L.cp);
  __shared__ double s_loss;
  __shared__ bool s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5, nt = blockDim.x;
  const int lc = lane % kTailCols;  // batch column within the CTA
  const int64_t col0 = (int64_t)blockIdx.x * kTailCols;
  const int ncols = (int)imin(kTailCols, n - col0);
  const bool valid = lc < ncols;

  // ---- stage: every thread issues its loads in batches of 4 before storing
  // (a load->store loop would serialise one memory round trip per element)
  {
    const int total = k * kTailCols;
    for (int base = tid; base < total; base += 4 * nt) {
      T v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + u * nt, c = e % kTailCols;
        v[u] = (e < total && c < ncols) ? __ldg(h + (e / kTailCols) * ld_h + col0 + c) : T(0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + u * nt;
        if (e < total) s_h[(e / kTailCols) * kTailHs + e % kTailCols] = v[u];
      }
    }
  }
  for (int e = tid; e < m * kTailCols; e += nt) {
    const int r = e / kTailCols, c = e % kTailCols;
    s_t[e] = c < ncols ? t[r * ld_t + col0 + c] : T(0);
  }
  for (int base = tid; base < nnz; base += 4 * nt) {
    int ix[4], rx[4], px[4];
    T vx[4], cx[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = base + u * nt;
      if (i < nnz) {
        ix[u] = col_idx[i];
        rx[u] = row_idx[i];
        px[u] = perm[i];
        vx[u] = vals[i];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (base + u * nt < nnz) cx[u] = vals[px[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = base + u * nt;
      if (i < nnz) {
        s_idx[i] = ix[u];
        s_val[i] = vx[u];
        s_ent[i] = CscEntry<T>{rx[u], cx[u]};
      }
    }
  }
  if (tid < kTailPad) {
    s_idx[nnz + tid] = 0;
    s_val[nnz + tid] = T(0);
  }
  for (int i = tid; i <= m; i += nt) s_rp[i] = row_ptr[i];
  for (int i = tid; i <= k; i += nt) s_cp[i] = col_ptr[i];
  __syncthreads();

  // ---- 1. logits y[r, col] = sum_s val(s) h[idx(s), col] (+ bias) ----------
  // (a) every product, rounded on its own, by all threads in parallel;
  // (b) one thread per (row, column) adds them in ascending s -- the same
  //     separately rounded multiply-then-add sequence as _kernels.py:25-37
  for (int e = tid; e < nnz * kTailCols; e += nt) {
    const int s = e / kTailCols, c = e % kTailCols;
    s_p[e] = mul_rn(s_val[s], s_h[s_idx[s] * kTailHs + c]);
  }
  __syncthreads();
  for (int e = tid; e < m * kTailCols; e += nt) {
    const int r = e / kTailCols, c = e % kTailCols;
    const int s0 = s_rp[r], s1 = s_rp[r + 1];
    T acc = T(0);
#pragma unroll 8
    for (int s = s0; s < s1; ++s) acc = add_rn(acc, s_p[s * kTailCols + c]);
    if (bias != nullptr) acc = add_rn(acc, bias[r]);
    s_y[e] = acc;
    if (y != nullptr && c < ncols) y[r * ld_y + col0 + c] = acc;
  }
  __syncthreads();

  // ---- 2. softmax-CE of each column (softmax_step_kernel's arithmetic) -----
  if (warp == 0) {
    double local = 0.0;
    if (lane < kTailCols) {
      if (valid) {
        T mx = s_y[lc];
        for (int c = 1; c < m; ++c) {
          const T v = s_y[c * kTailCols + lc];
          mx = (v > mx || v != v) ? v : mx;
        }
        T s = T(0), zt = T(0);
        for (int c = 0; c < m; ++c) {
          const T z = sub_rn(s_y[c * kTailCols + lc], mx);
          const T e = exp_full(z);
          s_dy[c * kTailCols + lc] = e;
          s = add_rn(s, e);
          zt = add_rn(zt, mul_rn(z, s_t[c * kTailCols + lc]));
        }
        for (int c = 0; c < m; ++c) {
          const T g = div_rn(sub_rn(div_rn(s_dy[c * kTailCols + lc], s), s_t[c * kTailCols + lc]),
                             divisor);
          s_dy[c * kTailCols + lc] = g;
          dy[c * ld_dy + col0 + lc] = g;
        }
        local = static_cast<double>(sub_rn(log_full(s), zt));
      } else {
        for (int c = 0; c < m; ++c) s_dy[c * kTailCols + lc] = T(0);
      }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if (lane == 0) s_loss = local;
  }
  __syncthreads();

  // ---- 3. d_h[c, col] = sum_{r ascending} W[r, c] d_y[r, col], * (h > 0) --
  // products in CSC order by all threads, then ascending-row sums
  for (int e = tid; e < nnz * kTailCols; e += nt) {
    const CscEntry<T> en = s_ent[e / kTailCols];
    s_p[e] = mul_rn(en.val, s_dy[en.row * kTailCols + e % kTailCols]);
  }
  __syncthreads();
  for (int e = tid; e < k * kTailCols; e += nt) {
    const int c = e / kTailCols, b = e % kTailCols;
    const int p0 = s_cp[c], p1 = s_cp[c + 1];
    T acc = T(0);
    for (int p = p0; p < p1; ++p) acc = add_rn(acc, s_p[p * kTailCols + b]);
    if (mask) acc = mask_np(acc, s_h[c * kTailHs + b]);
    if (b < ncols) dh[c * ld_dh + col0 + b] = acc;
  }

  // ---- loss across CTAs (fixed order) + step counter ------------------------
  if (tid == 0) {
    if (gridDim.x == 1) {
      if (loss_out) *loss_out = s_loss;
      s_last = true;
    } else {
      loss_parts[blockIdx.x] = s_loss;
      __threadfence();
      s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  if (gridDim.x > 1) {
    __threadfence();
    double tot = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) tot += loss_parts[b];
    if (loss_out) *loss_out = tot;
    *ticket = 0u;  // ready for the next launch / graph replay
  }
  if (counter) {
    const int32_t v = *counter + 1;
    *counter = (modulo > 0 && v >= modulo) ? 0 : v;
  }
}

template <typename T>
size_t tail_smem(const smb_pattern* pat) {
  return TailLayout<T>(pat->m, pat->k, pat->nnz).total;
}

constexpr size_t kTailSmemCap = 200 * 1024;

}  // namespace
}  // namespace smb

using namespace smb;

extern "C" int smb_tail_step_supported(int dtype, const smb_pattern* pat) {
  if (pat == nullptr || pat->m < 1 || pat->m > kTailMaxClasses || pat->k < 1) return 0;
  const size_t bytes = dtype == SMB_F32 ? tail_smem<float>(pat)
                       : dtype == SMB_F64 ? tail_smem<double>(pat) : kTailSmemCap + 1;
  return bytes <= kTailSmemCap ? 1 : 0;
}

extern "C" size_t smb_tail_step_workspace_bytes(int64_t n) {
  return 256 + sizeof(double) * (size_t)ceil_div(n > 0 ? n : 1, kTailCols);
}

extern "C" int smb_tail_step(int dtype, const smb_pattern* pat, const void* values, const void* h,
                             int64_t ld_h, int mask, const void* bias, const void* t,
                             int64_t ld_t, int64_t n, double divisor, void* y, int64_t ld_y,
                             void* d_y, int64_t ld_dy, void* d_h, int64_t ld_dh, double* loss_out,
                             int32_t* step_counter, int32_t modulo, void* workspace,
                             void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_tail_step: null pattern");
  SMB_REQUIRE(smb_tail_step_supported(dtype, pat),
              "smb_tail_step: layer %lld x %lld (nnz %lld) outside the fused tail's limits",
              (long long)pat->m, (long long)pat->k, (long long)pat->nnz);
  SMB_REQUIRE(n >= 1 && n <= (int64_t(1) << 30), "smb_tail_step: bad batch width");
  SMB_REQUIRE(ld_h >= n && ld_t >= n && ld_dy >= n && ld_dh >= n && (y == nullptr || ld_y >= n),
              "smb_tail_step: leading dimension");
  SMB_REQUIRE(divisor != 0.0, "smb_tail_step: zero divisor");
  SMB_REQUIRE(values && h && t && d_y && d_h, "smb_tail_step: null pointer");
  const unsigned grid = (unsigned)ceil_div(n, kTailCols);
  SMB_REQUIRE(grid == 1 || workspace != nullptr, "smb_tail_step: workspace required");
  unsigned* ticket = workspace ? static_cast<unsigned*>(workspace) : nullptr;
  double* parts =
      workspace ? reinterpret_cast<double*>(static_cast<char*>(workspace) + 256) : nullptr;
  auto launch = [&](auto tag) {
    using T = decltype(tag);
    const size_t bytes = tail_smem<T>(pat);
    auto kern = tail_step_kernel<T>;
    ensure_smem(kern, bytes);
    kern<<<grid, kTailThreads, bytes, as_stream(stream)>>>(
        pat->row_ptr, pat->col_idx, pat->col_ptr, pat->row_idx, pat->perm,
        static_cast<const T*>(values), (int)pat->m, (int)pat->k, (int)pat->nnz,
        static_cast<const T*>(h), ld_h, mask, static_cast<const T*>(bias),
        static_cast<const T*>(t), ld_t, n, T(divisor), static_cast<T*>(y), ld_y,
        static_cast<T*>(d_y), ld_dy, static_cast<T*>(d_h), ld_dh, loss_out, parts, ticket,
        step_counter, modulo);
    return check_launch("smb_tail_step");
  };
  return dtype == SMB_F32 ? launch(float{}) : launch(double{});
}
