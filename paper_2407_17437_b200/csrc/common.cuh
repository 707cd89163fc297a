// Shared helpers for the sm_100a sparse-MLP kernels: exact (separately rounded)
// arithmetic, vector types, error plumbing for the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "../../include/sparsemlp_b200.h"

namespace smb {

// ---------------------------------------------------------------------------
// error state (thread-local message, process-wide launch counter)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
void clear_error();
void count_launches(uint64_t n);

#define SMB_REQUIRE(cond, ...)            \
  do {                                    \
    if (!(cond)) {                        \
      ::smb::set_error(__VA_ARGS__);      \
      return SMB_ERR_INVALID;             \
    }                                     \
  } while (0)

// Check the launch that just happened; counts it for smb_launch_count().
int check_launch(const char* what, uint64_t launches = 1);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// fn(T{}) for the value dtype code (SMB_F32 / SMB_F64)
template <typename F>
inline int dispatch_dtype(int dtype, const char* name, F&& fn) {
  if (dtype == SMB_F32) return fn(float{});
  if (dtype == SMB_F64) return fn(double{});
  set_error("%s: unsupported dtype %d", name, dtype);
  return SMB_ERR_INVALID;
}

// Opt a kernel into `bytes` of dynamic shared memory, once per kernel per
// process (device-wide attribute; cheap registry keyed by the entry point).
void ensure_dynamic_smem(const void* kernel, size_t bytes);
template <typename K>
inline void ensure_smem(K* kernel, size_t bytes) {
  ensure_dynamic_smem(reinterpret_cast<const void*>(kernel), bytes);
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+).  Every kernel is launched with
// programmatic stream serialisation allowed: the next kernel on a stream may
// be scheduled while the previous one drains, runs its independent prologue
// (indices, values, bias -- never the previous kernel's output), then
// pdl_wait()s, which returns once the previous grid has completed and its
// writes are visible.  Producers pdl_trigger() when their main loop is done.
// Both are no-ops when the launch carries no programmatic dependency (first
// kernel after an event wait, eager launches on other streams, ...).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// exact arithmetic: multiply and add rounded separately, never contracted.
// (The library is also compiled with --fmad=false as a second guard.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// np.maximum(y, 0): NaN propagates, -0.0 -> +0.0 (verified against numpy 2.3)
template <typename T>
__device__ __forceinline__ T relu_np(T y) {
  return (y > T(0) || y != y) ? y : T(0);
}

// d * (x > 0) with numpy's bool->float promotion: d*1 or d*0 (keeps -0 / NaN)
template <typename T>
__device__ __forceinline__ T mask_np(T d, T x) {
  return mul_rn(d, x > T(0) ? T(1) : T(0));
}

// full-accuracy (non-intrinsic) exp / log in the value type: expf is within
// 2 ulp like numpy's own float32 exp (documented max 2.52 ulp), so the
// softmax is tolerance-exact, not bit-exact, against the reference
__device__ __forceinline__ float exp_full(float x) { return expf(x); }
__device__ __forceinline__ double exp_full(double x) { return exp(x); }
__device__ __forceinline__ float log_full(float x) { return logf(x); }
__device__ __forceinline__ double log_full(double x) { return log(x); }

// 16-byte vector of T
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int N = 4;
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int N = 2;
};

template <typename T>
struct VecOps;
template <>
struct VecOps<float> {
  using V = float4;
  __device__ __forceinline__ static float get(const V& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
  __device__ __forceinline__ static void set(V& v, int i, float x) {
    if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
  }
  __device__ __forceinline__ static V zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  // acc += s * v, lane-wise, separately rounded
  __device__ __forceinline__ static void axpy(V& acc, float s, const V& v) {
    acc.x = add_rn(acc.x, mul_rn(s, v.x));
    acc.y = add_rn(acc.y, mul_rn(s, v.y));
    acc.z = add_rn(acc.z, mul_rn(s, v.z));
    acc.w = add_rn(acc.w, mul_rn(s, v.w));
  }
};
template <>
struct VecOps<double> {
  using V = double2;
  __device__ __forceinline__ static double get(const V& v, int i) { return i == 0 ? v.x : v.y; }
  __device__ __forceinline__ static void set(V& v, int i, double x) {
    if (i == 0) v.x = x; else v.y = x;
  }
  __device__ __forceinline__ static V zero() { return make_double2(0.0, 0.0); }
  __device__ __forceinline__ static void axpy(V& acc, double s, const V& v) {
    acc.x = add_rn(acc.x, mul_rn(s, v.x));
    acc.y = add_rn(acc.y, mul_rn(s, v.y));
  }
};

// Gather loads through the read-only path (L1-allocating: measured 1.5x
// faster on B200 than ld.global.nc.L1::no_allocate for the SpMM gathers).
template <typename V>
__device__ __forceinline__ V ldg_vec(const V* p) {
  return __ldg(p);
}
template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) {
  return __ldg(p);
}

__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Optimizer constants exactly as the reference forms them:
//   sparse_combine(opt.mu, V, 1.0, G)            -> alpha = T(mu), beta = T(1)
//   sparse_combine(1.0, W, -eta * opt.mu, V)     -> T(-eta*mu) (float64 product)
//   sparse_combine(1.0, W, -eta, G)              -> T(-eta)
// (nn.py:189-197, tensor_core.py:304-305; _step_vector nn.py:121-131)
template <typename T>
struct OptConsts {
  int kind;
  T mu;
  T c_v;  // T(-eta * mu)
  T c_g;  // T(-eta)
};

template <typename T>
inline OptConsts<T> make_opt(int kind, double mu, double eta) {
  OptConsts<T> o;
  o.kind = kind;
  o.mu = static_cast<T>(mu);
  o.c_v = static_cast<T>(-eta * mu);
  o.c_g = static_cast<T>(-eta);
  return o;
}

// One element of the update, in the reference's exact operation order.
// 1*x is exact, so fl(1*w) + fl(c*v) == add_rn(w, mul_rn(c, v)).
template <typename T>
__device__ __forceinline__ void apply_update(const OptConsts<T>& o, T g, T* w, T* v) {
  if (o.kind == SMB_OPT_GD) {
    *w = add_rn(*w, mul_rn(o.c_g, g));
  } else if (o.kind == SMB_OPT_MOMENTUM) {
    T vv = add_rn(mul_rn(o.mu, *v), g);
    *v = vv;
    *w = add_rn(*w, mul_rn(o.c_g, vv));
  } else if (o.kind == SMB_OPT_NESTEROV) {
    T vv = add_rn(mul_rn(o.mu, *v), g);
    *v = vv;
    T ww = add_rn(*w, mul_rn(o.c_v, vv));
    *w = add_rn(ww, mul_rn(o.c_g, g));
  }
}

// numpy's pairwise summation (loops_utils.h pairwise_sum, PW_BLOCKSIZE=128)
// of a[0..n) with unit stride, as used by ndarray.sum(axis=-1) on contiguous
// rows (tensor_core.row_sums).  Sequential per thread; the leaves use the
// 8-accumulator unrolled loop.  Verified bit-identical to numpy 2.3 for
// n in [1, 5000].
template <typename T>
__device__ T pairwise_leaf(const T* a, int64_t n) {
  if (n < 8) {
    T res = T(0);
    for (int64_t i = 0; i < n; ++i) res = add_rn(res, a[i]);
    return res;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  const int64_t lim = n - (n % 8);
  for (; i < lim; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = add_rn(r[j], a[i + j]);
  }
  T res = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])),
                 add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
  for (; i < n; ++i) res = add_rn(res, a[i]);
  return res;
}

template <typename T>
__device__ T pairwise_sum(const T* a, int64_t n) {
  // explicit-stack version of:
  //   n <= 128: leaf;  else n2 = n/2 - (n/2)%8; return ps(a, n2) + ps(a+n2, n-n2)
  // Depth is log2(n/128) + 1 <= 40 for 64-bit n; 48 frames is plenty.
  struct Frame {
    int64_t off, n;
    int state;  // 0: expand, 1: left done
    T left;
  };
  Frame st[48];
  int sp = 0;
  st[0] = {0, n, 0, T(0)};
  T ret = T(0);
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_leaf(a + f.off, f.n);
      --sp;
      // propagate
      while (sp >= 0) {
        Frame& p = st[sp];
        if (p.state == 0) {
          p.left = ret;
          p.state = 1;
          int64_t n2 = p.n / 2;
          n2 -= n2 % 8;
          st[++sp] = {p.off + n2, p.n - n2, 0, T(0)};
          break;
        } else {
          ret = add_rn(p.left, ret);
          --sp;
        }
      }
    } else {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      st[sp + 1] = {f.off, n2, 0, T(0)};
      ++sp;
    }
  }
  return ret;
}

// ---------------------------------------------------------------------------
// Warp-cooperative numpy pairwise sum (same tree, same roundings as
// pairwise_sum above).  The leaves of the split tree are computed 4 at a time
// by 8-lane groups (lane j of a group owns accumulator r[j]); lane 0 then
// combines the leaf values in the recursion order.  `leaf_buf` is per-warp
// scratch (shared memory) of at least warp_pairwise_leaves(n) elements.  All
// 32 lanes must call; the result is returned on every lane.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int warp_pairwise_leaves(int n) { return n / 64 + 2; }

// n = 128 * L, L a power of two >= 2: every leaf holds exactly 128 elements
// and numpy's split (n2 = n / 2 rounded down to a multiple of 8) halves the
// leaf range at every level, so the combine is a balanced tree over the L
// leaves.  Four leaves per round (8 lanes per leaf, lane j = accumulator j),
// the next round's 16 loads per lane issued before this round is summed;
// the tree runs level by level in shared memory with all lanes.
template <typename T>
__device__ T warp_pairwise_sum_pow2(const T* a, int L, T* leaf_buf) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, j = lane & 7;
  const int rounds = (L + 3) >> 2;
  T v[16], w[16];
  auto load = [&](T(&x)[16], int leaf) {
    const T* p = a + leaf * 128 + j;
    const bool ok = leaf < L;
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = ok ? p[8 * k] : T(0);
  };
  load(v, grp);
  for (int r = 0; r < rounds; ++r) {
    if (r + 1 < rounds) load(w, 4 * (r + 1) + grp);
    T acc = v[0];  // accumulator j of the leaf: a[j], += a[8k + j] in k order
#pragma unroll
    for (int k = 1; k < 16; ++k) acc = add_rn(acc, v[k]);
    // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
    T t = __shfl_down_sync(0xffffffffu, acc, 1);
    if ((j & 1) == 0) acc = add_rn(acc, t);
    t = __shfl_down_sync(0xffffffffu, acc, 2);
    if ((j & 3) == 0) acc = add_rn(acc, t);
    t = __shfl_down_sync(0xffffffffu, acc, 4);
    if (j == 0 && 4 * r + grp < L) leaf_buf[4 * r + grp] = add_rn(acc, t);
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = w[k];
  }
  __syncwarp();
  for (int h = L >> 1; h >= 1; h >>= 1) {  // level: h sums of adjacent pairs
    T x0 = T(0), x1 = T(0);
    if (lane < h) x0 = add_rn(leaf_buf[2 * lane], leaf_buf[2 * lane + 1]);
    if (lane + 32 < h) x1 = add_rn(leaf_buf[2 * lane + 64], leaf_buf[2 * lane + 65]);
    __syncwarp();
    if (lane < h) leaf_buf[lane] = x0;
    if (lane + 32 < h) leaf_buf[lane + 32] = x1;
    __syncwarp();
  }
  const T ret = leaf_buf[0];
  __syncwarp();
  return ret;
}

template <typename T>
__device__ T warp_pairwise_sum(const T* a, int n, T* leaf_buf) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, j = lane & 7;
  if (n <= 0) return T(0);
  if (n >= 256 && n <= 16384 && (n & 127) == 0 && ((n >> 7) & ((n >> 7) - 1)) == 0)
    return warp_pairwise_sum_pow2(a, n >> 7, leaf_buf);
  int st_off[32], st_len[32];
  int sp = 0, leaf = 0;
  int cur_off = 0, cur_len = n;
  bool done = false;
  while (!done) {
    // gather up to 4 leaves in DFS (left-to-right) order
    int b_off[4] = {0, 0, 0, 0}, b_len[4] = {0, 0, 0, 0};
    int nb = 0;
    while (nb < 4 && !done) {
      while (cur_len > 128) {
        int n2 = cur_len / 2;
        n2 -= n2 % 8;
        st_off[sp] = cur_off + n2;
        st_len[sp] = cur_len - n2;
        ++sp;
        cur_len = n2;
      }
      b_off[nb] = cur_off;
      b_len[nb] = cur_len;
      ++nb;
      if (sp == 0) {
        done = true;
      } else {
        --sp;
        cur_off = st_off[sp];
        cur_len = st_len[sp];
      }
    }
    const int off = grp == 0 ? b_off[0] : grp == 1 ? b_off[1] : grp == 2 ? b_off[2] : b_off[3];
    const int len = grp < nb ? (grp == 0 ? b_len[0] : grp == 1 ? b_len[1] : grp == 2 ? b_len[2] : b_len[3]) : 0;
    const T* p = a + off;
    const int lim = len - (len % 8);
    // the whole leaf (<= 128 elements, <= 16 per lane) is loaded up front so
    // a batch of 4 leaves costs one memory round trip, then summed in order
    T v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = (8 * k + j < lim) ? p[8 * k + j] : T(0);
    T tail[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const int i = (len >= 8 ? lim : 0) + k;
      tail[k] = (j == 0 && i < len) ? p[i] : T(0);
    }
    T r = v[0];
#pragma unroll
    for (int k = 1; k < 16; ++k)
      if (8 * k < lim) r = add_rn(r, v[k]);
    T t = __shfl_down_sync(0xffffffffu, r, 1);
    if ((j & 1) == 0) r = add_rn(r, t);
    t = __shfl_down_sync(0xffffffffu, r, 2);
    if ((j & 3) == 0) r = add_rn(r, t);
    t = __shfl_down_sync(0xffffffffu, r, 4);
    if (j == 0 && grp < nb) {
      T res;
      const int rest = len >= 8 ? len - lim : len;
      res = len >= 8 ? add_rn(r, t) : T(0);
#pragma unroll
      for (int k = 0; k < 7; ++k)
        if (k < rest) res = add_rn(res, tail[k]);
      if (n <= 128) leaf_buf[0] = res; else leaf_buf[leaf + grp] = res;
    }
    leaf += nb;
  }
  __syncwarp();
  T ret = leaf_buf[0];
  if (n > 128 && lane == 0) {
    // combine in recursion order: value(node) = value(left) + value(right)
    int st_n[32], st_state[32];
    T st_left[32];
    int k = 0, idx = 0, cur = n;
    for (;;) {
      while (cur > 128) {
        st_n[k] = cur;
        st_state[k] = 0;
        ++k;
        int n2 = cur / 2;
        n2 -= n2 % 8;
        cur = n2;
      }
      ret = leaf_buf[idx++];
      bool next = false;
      while (!next) {
        if (k == 0) break;
        if (st_state[k - 1] == 0) {
          st_left[k - 1] = ret;
          st_state[k - 1] = 1;
          int n2 = st_n[k - 1] / 2;
          n2 -= n2 % 8;
          cur = st_n[k - 1] - n2;
          next = true;
        } else {
          ret = add_rn(st_left[k - 1], ret);
          --k;
        }
      }
      if (!next) break;
    }
  }
  ret = __shfl_sync(0xffffffffu, ret, 0);
  __syncwarp();
  return ret;
}

}  // namespace smb
