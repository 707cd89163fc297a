// Row-split CSR SpMM (forward) and CSC SpMM (transposed) for sm_100a.
//
// Both products have the same shape of work: every output row r is
//     out[r, :] = sum_{s in segment(r), ascending} val(s) * dense[idx(s), :]
// with (segment, idx, val) = (CSR row, col_idx, values) for Y = W X
// (_kernels.py:25-37) and (CSC column, row_idx, values[perm]) for dX = W^T dY
// (_kernels.py:40-59; ascending source row == the reference's row-order scan).
//
// Mapping: one CTA owns one output row (gridDim.y splits very wide batches);
// its warps own consecutive 32*W-column chunks of the batch and each lane
// keeps W consecutive columns in registers for the whole segment, so the
// accumulation order per element is exactly the reference's (ascending s,
// multiply and add rounded separately).  Each warp reads 32 (idx, val) pairs
// with one coalesced load and broadcasts them with shuffles; the dense rows
// are gathered as 128/512-byte coalesced vectors through the read-only path
// with a U-deep refill-on-consume register ring per warp.
//
// Epilogues (fused, one pass over the output row):
//   forward   + bias[r], np.maximum(., 0)                     nn.py:173, 86-87
//   backward  * (mask > 0)  (ReLU.backward of the layer below)  nn.py:89-91
//             and, when one CTA covers the whole row, grad_bias[r] =
//             row_sums(out[r, :]) in numpy's pairwise order (nn.py:184) with
//             the bias optimizer update (_step_vector, nn.py:118-131).
#include "pattern.cuh"

namespace smb {
namespace {

template <typename T, int W>
struct Frag {
  T v[W];
};

// W consecutive elements as 16-byte vectors (W a multiple of the vector width)
template <typename T, int W>
__device__ __forceinline__ void load_frag_full(Frag<T, W>& f, const T* p) {
  if constexpr (W == 1) {
    f.v[0] = ldg_stream(p);
  } else {
    using V = typename Vec16<T>::type;
    constexpr int VW = Vec16<T>::N;
    static_assert(W % VW == 0, "vector width");
#pragma unroll
    for (int h = 0; h < W / VW; ++h) {
      const V v = ldg_vec(reinterpret_cast<const V*>(p) + h);
#pragma unroll
      for (int j = 0; j < VW; ++j) f.v[h * VW + j] = VecOps<T>::get(v, j);
    }
  }
}

template <typename T, int W>
__device__ __forceinline__ void load_frag(Frag<T, W>& f, const T* p, int valid) {
  if (valid == W) {
    load_frag_full<T, W>(f, p);
    return;
  }
#pragma unroll
  for (int j = 0; j < W; ++j) f.v[j] = (j < valid) ? __ldg(p + j) : T(0);
}

template <typename T, int W>
__device__ __forceinline__ void store_frag(const Frag<T, W>& f, T* p, int valid) {
  if constexpr (W > 1) {
    using V = typename Vec16<T>::type;
    constexpr int VW = Vec16<T>::N;
    if (valid == W) {
#pragma unroll
      for (int h = 0; h < W / VW; ++h) {
        V v;
#pragma unroll
        for (int j = 0; j < VW; ++j) VecOps<T>::set(v, j, f.v[h * VW + j]);
        reinterpret_cast<V*>(p)[h] = v;
      }
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
  const T* bias;  // forward: per-row bias or null
  int relu;       // forward: apply np.maximum(y, 0)
  const T* mask;  // backward: out *= (mask > 0), or null
  int64_t ld_mask;
  // backward row-sum stage (only when the CTA covers the whole row)
  int rowsum;
  T* rb_bias;   // bias of the layer whose output gradient this is (updated)
  T* rb_vbias;  // its velocity
  T* rb_grad;   // grad_bias out (may be null)
  OptConsts<T> opt;
};

// at most 8 warps per CTA: a 256-thread bound leaves up to 255 registers per
// thread, so the U-deep prefetch ring stays in flight (with a 64-register cap
// the compiler sinks the ring's loads next to their uses)
template <int W>
constexpr int max_threads_for() { return 256; }

// A CTA holds rows_per_cta rows x (nwarps / rows_per_cta) warps per row; its
// warps own consecutive 32*W-column chunks of the batch.  Launch order is
// blockIdx.x fastest, so all rows of one column slice (blockIdx.y) run
// before the next slice: when the dense operand is wider than L2, the slice
// width is chosen so the slice's rows stay L2-resident while every output
// row gathers from them (launch_rows).
template <typename T, int W, int U, int EPI, bool PERM, bool MULTI = false, bool ROWSUM = false>
__global__ void __launch_bounds__(max_threads_for<W>())
    row_spmm_kernel(const int32_t* __restrict__ seg_ptr, const int32_t* __restrict__ idx,
                    const int32_t* __restrict__ perm, const T* __restrict__ vals,
                    const T* __restrict__ dense, int64_t ld_dense, int64_t n,
                    T* __restrict__ out, int64_t ld_out, EpiArgs<T> epi, int rows_per_cta,
                    int64_t n_rows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp_in_cta = threadIdx.x >> 5;
  // MULTI: several rows per CTA (never with the fused row-sum epilogue)
  const int nwarps = MULTI ? (blockDim.x >> 5) / rows_per_cta : (blockDim.x >> 5);  // per row
  const int warp = MULTI ? warp_in_cta % nwarps : warp_in_cta;
  const int64_t row =
      MULTI ? (int64_t)blockIdx.x * rows_per_cta + warp_in_cta / nwarps : (int64_t)blockIdx.x;
  if (MULTI && row >= n_rows) return;
  const int64_t chunk = (int64_t)blockIdx.y * nwarps + warp;
  const int64_t col0 = chunk * (32 * W) + (int64_t)lane * W;
  const int valid = (int)imax(0, imin(W, n - col0));

  Frag<T, W> acc;
#pragma unroll
  for (int j = 0; j < W; ++j) acc.v[j] = T(0);

  const int32_t s_begin = seg_ptr[row];
  const int32_t s_end = seg_ptr[row + 1];
  // lanes past the batch read column 0 (in bounds, never stored): every ring
  // refill can then be unconditional -- a predicated refill compiles to a
  // load plus a predicated move that stalls on the load right away
  const T* dcol = dense + (valid > 0 ? col0 : 0);
  const uint32_t ldu = (uint32_t)ld_dense;  // row offsets as one IMAD.WIDE.U32
  // warp-uniform: every lane of this warp owns W valid columns
  const bool full_chunk = (chunk + 1) * (32 * W) <= n;

  // The segment is walked in groups of 32 (idx, val) pairs (one coalesced
  // load per group, broadcast by shuffles; the NEXT group is always loaded a
  // group ahead).  A U-deep register ring of dense-row fragments runs
  // continuously across groups: the slot consumed at position s is refilled
  // with position s + U (U divides 32, so a position's slot is s % U in every
  // group).
  const int len = s_end - s_begin;
  auto load_group = [&](int g, int& gi, T& gv) {
    const int32_t s = s_begin + g * 32 + lane;
    gi = 0;
    gv = T(0);
    if (s < s_end) {
      gi = idx[s];
      gv = PERM ? vals[perm[s]] : vals[s];
    }
  };
  // three groups in registers: current, next (refill targets) and the one
  // after, whose load then has a whole group's time to land
  int idx_c, idx_n, idx_nn;
  T val_c, val_n, val_nn;
  load_group(0, idx_c, val_c);
  load_group(1, idx_n, val_n);
  load_group(2, idx_nn, val_nn);
  // epilogue operands that do not depend on the product: issue them now
  T bias_r = T(0);
  if constexpr (EPI == kEpiBiasAct) {
    if (epi.bias != nullptr) bias_r = epi.bias[row];
  }
  Frag<T, W> mk;
  T rb_w = T(0), rb_v = T(0);  // bias state of the fused row-sum update
  if constexpr (EPI == kEpiMask) {
    if (epi.mask != nullptr && valid > 0)
      load_frag<T, W>(mk, epi.mask + row * epi.ld_mask + col0, valid);
    if (epi.rowsum && threadIdx.x == 0 && epi.opt.kind != SMB_OPT_NONE && epi.rb_bias) {
      rb_w = epi.rb_bias[row];
      if (epi.rb_vbias) rb_v = epi.rb_vbias[row];
    }
  }
  // everything above reads data older than the previous kernel on this
  // stream; the dense operand below is that kernel's output
  pdl_wait();
  // lanes with 0 < valid < W (the batch tail) need element-wise loads
  const bool lane_full = valid == W || valid == 0;
  auto refill = [&](Frag<T, W>& f, int src) {
    const T* p = dcol + (size_t)(uint32_t)src * ldu;
    if (lane_full) load_frag_full<T, W>(f, p);
    else load_frag<T, W>(f, p, valid);
  };
  Frag<T, W> xs[U];
#pragma unroll
  for (int u = 0; u < U; ++u) refill(xs[u], __shfl_sync(0xffffffffu, idx_c, u));
  const int ngroups = (len + 31) / 32;
  for (int g = 0; g < ngroups; ++g) {
    const int cnt = min(32, len - g * 32);
    if (cnt == 32 && full_chunk) {
      // fast path: fully unrolled, unconditional refills (positions past the
      // row end carry index 0 and are never consumed)
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const T v = __shfl_sync(0xffffffffu, val_c, q);
#pragma unroll
        for (int j = 0; j < W; ++j) acc.v[j] = add_rn(acc.v[j], mul_rn(v, xs[q % U].v[j]));
        const uint32_t nxt = (uint32_t)(q + U < 32 ? __shfl_sync(0xffffffffu, idx_c, q + U)
                                                   : __shfl_sync(0xffffffffu, idx_n, q + U - 32));
        load_frag_full<T, W>(xs[q % U], dcol + (size_t)nxt * ldu);
      }
    } else {
      for (int q0 = 0; q0 < cnt; q0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = q0 + u;
          const T v = __shfl_sync(0xffffffffu, val_c, q & 31);
          const int pos = q + U;  // refill target, possibly in the next group
          const int nc = __shfl_sync(0xffffffffu, idx_c, pos & 31);
          const int nn = __shfl_sync(0xffffffffu, idx_n, pos & 31);
          if (q < cnt) {
#pragma unroll
            for (int j = 0; j < W; ++j) acc.v[j] = add_rn(acc.v[j], mul_rn(v, xs[u].v[j]));
            refill(xs[u], pos < 32 ? nc : nn);
          }
        }
      }
    }
    idx_c = idx_n;
    val_c = val_n;
    idx_n = idx_nn;
    val_n = val_nn;
    load_group(g + 3, idx_nn, val_nn);
  }
  pdl_trigger();

  if constexpr (EPI == kEpiBiasAct) {
    if (valid == 0) return;
    if (epi.bias != nullptr) {
#pragma unroll
      for (int j = 0; j < W; ++j) acc.v[j] = add_rn(acc.v[j], bias_r);
    }
    if (epi.relu) {
#pragma unroll
      for (int j = 0; j < W; ++j) acc.v[j] = relu_np(acc.v[j]);
    }
    store_frag<T, W>(acc, out + row * ld_out + col0, valid);
  } else {
    if (valid > 0) {
      if (epi.mask != nullptr) {
#pragma unroll
        for (int j = 0; j < W; ++j) acc.v[j] = mask_np(acc.v[j], mk.v[j]);
      }
      store_frag<T, W>(acc, out + row * ld_out + col0, valid);
    }
    // (the row-sum stage is its own instantiation: compiled into every
    // transposed launch it cost config 4's SpMM-T 2.4%, 142.2 vs 138.9 us)
    if constexpr (!ROWSUM) {
      return;
    } else {
    if (!epi.rowsum) return;
    // whole row in this CTA: stage it, pairwise-sum it, update this row's bias
    T* s_row = reinterpret_cast<T*>(smem_raw);
    T* leaf_buf = s_row + ((n + 3) & ~int64_t(3));
#pragma unroll
    for (int j = 0; j < W; ++j)
      if (j < valid) s_row[col0 + j] = acc.v[j];
    __syncthreads();
    if (warp == 0) {
      const T g = warp_pairwise_sum(s_row, (int)n, leaf_buf);
      if (lane == 0) {
        if (epi.rb_grad) epi.rb_grad[row] = g;
        if (epi.opt.kind != SMB_OPT_NONE && epi.rb_bias) {
          apply_update(epi.opt, g, &rb_w, &rb_v);
          epi.rb_bias[row] = rb_w;
          if (epi.rb_vbias) epi.rb_vbias[row] = rb_v;
        }
      }
    }
    }
  }
}

// Single batch column (n == 1: batch-1 inference, bench.py:366-399): one
// warp per output row.  The 32 lanes gather 32 products val(s) * x[idx(s)]
// at once (coalesced index / value loads, one gathered x element each), park
// them in shared memory and lane 0 adds them in ascending s -- the same
// separately rounded multiply-then-add sequence as the batched kernel.
constexpr int kSpmvWarps = 8;

template <typename T, int EPI, bool PERM>
__global__ void __launch_bounds__(kSpmvWarps * 32)
    row_spmv_kernel(const int32_t* __restrict__ seg_ptr, const int32_t* __restrict__ idx,
                    const int32_t* __restrict__ perm, const T* __restrict__ vals,
                    const T* __restrict__ dense, int64_t ld_dense, int64_t n_rows,
                    T* __restrict__ out, int64_t ld_out, EpiArgs<T> epi) {
  __shared__ T s_p[kSpmvWarps][32];
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kSpmvWarps + warp;
  if (row >= n_rows) return;
  const int32_t s0 = seg_ptr[row], s1 = seg_ptr[row + 1];
  T acc = T(0);
  for (int32_t g = s0; g < s1; g += 32) {
    const int32_t s = g + lane;
    T p = T(0);
    if (s < s1) {
      const T v = PERM ? vals[perm[s]] : vals[s];
      p = mul_rn(v, __ldg(dense + (int64_t)idx[s] * ld_dense));
    }
    s_p[warp][lane] = p;
    __syncwarp();
    if (lane == 0) {
      const int cnt = min(32, s1 - g);
      for (int j = 0; j < cnt; ++j) acc = add_rn(acc, s_p[warp][j]);
    }
    __syncwarp();
  }
  if (lane != 0) return;
  if constexpr (EPI == kEpiBiasAct) {
    if (epi.bias != nullptr) acc = add_rn(acc, epi.bias[row]);
    if (epi.relu) acc = relu_np(acc);
  } else {
    if (epi.mask != nullptr) acc = mask_np(acc, epi.mask[row * epi.ld_mask]);
  }
  out[row * ld_out] = acc;
}

// Few long rows over a wide batch, one column per lane (the output layer at
// config 2: 10 rows x ~310 nonzeros x B = 1024).  One warp per CTA; the loop
// body consumes three 32-nonzero groups held in three register arrays, and
// refills each array (operands, values and indices) three groups ahead right
// after consuming it -- any move the compiler adds to rotate the registers
// then sits three groups after its load, not one.  Order and rounding are
// row_spmm_kernel's.  No fused row sums (the host keeps those elsewhere).
// One warp walks segment `row` for one 32-column batch chunk (lane = column)
// and returns the ascending-order sum (see row_spmm_deep_kernel).  Executes
// pdl_wait() once the segment's indices / values are in flight, before the
// first read of `dense` (the previous kernel's output).
template <typename T, bool PERM>
__device__ __forceinline__ T deep_row_chain(const int32_t* __restrict__ seg_ptr,
                                            const int32_t* __restrict__ idx,
                                            const int32_t* __restrict__ perm,
                                            const T* __restrict__ vals, const T* dcol,
                                            uint32_t ldu, int64_t row, int lane) {
  const int32_t s_begin = seg_ptr[row], s_end = seg_ptr[row + 1];
  const int len = s_end - s_begin;
  const int ngroups = (len + 31) / 32;
  auto ld_idx = [&](int g) -> int {  // index of position (g, lane); 0 past the row
    const int32_t s = s_begin + g * 32 + lane;
    return s < s_end ? idx[s] : 0;
  };
  auto ld_val = [&](int g) -> T {
    const int32_t s = s_begin + g * 32 + lane;
    return s < s_end ? (PERM ? vals[perm[s]] : vals[s]) : T(0);
  };
  auto gather = [&](T (&x)[32], int gi) {  // operands of a group from its indices
#pragma unroll
    for (int q = 0; q < 32; ++q)
      x[q] = ldg_stream(dcol + (size_t)(uint32_t)__shfl_sync(0xffffffffu, gi, q) * ldu);
  };
  T acc = T(0);
  auto consume = [&](const T (&x)[32], T v, int cnt) {
    if (cnt == 32) {
#pragma unroll
      for (int q = 0; q < 32; ++q) acc = add_rn(acc, mul_rn(__shfl_sync(0xffffffffu, v, q), x[q]));
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const T vq = __shfl_sync(0xffffffffu, v, q);
        if (q < cnt) acc = add_rn(acc, mul_rn(vq, x[q]));
      }
    }
  };
  T xa[32], xb[32], xc[32];
  T va = ld_val(0), vb = ld_val(1), vc = ld_val(2);
  const int i0 = ld_idx(0), i1 = ld_idx(1), i2 = ld_idx(2);
  pdl_wait();  // the dense operand is the previous kernel's output
  gather(xa, i0);
  gather(xb, i1);
  gather(xc, i2);
  int ia = ld_idx(3), ib = ld_idx(4), ic = ld_idx(5);
  int g = 0;
  for (; g + 3 <= ngroups; g += 3) {
    consume(xa, va, 32 * (g + 1) <= len ? 32 : len - 32 * g);
    gather(xa, ia);
    va = ld_val(g + 3);
    ia = ld_idx(g + 6);
    consume(xb, vb, 32 * (g + 2) <= len ? 32 : len - 32 * (g + 1));
    gather(xb, ib);
    vb = ld_val(g + 4);
    ib = ld_idx(g + 7);
    consume(xc, vc, 32 * (g + 3) <= len ? 32 : len - 32 * (g + 2));
    gather(xc, ic);
    vc = ld_val(g + 5);
    ic = ld_idx(g + 8);
  }
  // up to two remaining groups, in array order
  if (g < ngroups) consume(xa, va, min(32, len - 32 * g));
  if (g + 1 < ngroups) consume(xb, vb, min(32, len - 32 * (g + 1)));
  return acc;
}

// Few long rows, one column per lane, "parallel products + serial sum": CTA
// = one row x 32 batch columns, 8 warps.  The row is walked in segments of
// kPpSeg nonzeros: all warps compute the segment's products
// val(s) * x[idx(s), col] (each rounded on its own) into one of two
// shared-memory buffers while warp 0 adds the previous segment's products in
// ascending s -- the same separately rounded multiply-then-add sequence, but
// the serial chain no longer waits on index -> operand loads.
constexpr int kPpWarps = 8;
template <typename T>
__host__ __device__ constexpr int pp_seg() { return sizeof(T) == 4 ? 128 : 64; }  // 32 KB x2

template <typename T, int EPI, bool PERM>
__global__ void __launch_bounds__(32 * kPpWarps)
    row_spmm_pp_kernel(const int32_t* __restrict__ seg_ptr, const int32_t* __restrict__ idx,
                       const int32_t* __restrict__ perm, const T* __restrict__ vals,
                       const T* __restrict__ dense, int64_t ld_dense, int64_t n,
                       T* __restrict__ out, int64_t ld_out, EpiArgs<T> epi) {
  constexpr int kPpSeg = pp_seg<T>();
  __shared__ T s_p[2][kPpSeg][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = blockIdx.x;
  const int64_t col = (int64_t)blockIdx.y * 32 + lane;
  const bool valid = col < n;
  const T* dcol = dense + (valid ? col : 0);
  const uint32_t ldu = (uint32_t)ld_dense;
  const int32_t s_begin = seg_ptr[row], s_end = seg_ptr[row + 1];
  const int len = s_end - s_begin;
  const int nseg = (len + kPpSeg - 1) / kPpSeg;
  T bias_r = T(0), mk = T(0);
  if constexpr (EPI == kEpiBiasAct) {
    if (epi.bias != nullptr) bias_r = epi.bias[row];
  } else {
    if (epi.mask != nullptr && valid) mk = epi.mask[row * epi.ld_mask + col];
  }
  // products of segment sg: warp w takes positions w*16 .. w*16+15 (kPpSeg =
  // 8 warps x 16); lane q < 16 holds (idx, val) of position q, broadcast by
  // shuffles
  constexpr int PW = kPpSeg / kPpWarps;
  auto load_iv = [&](int sg, int& gi, T& gv) {
    const int q = lane % PW;
    const int32_t s = s_begin + sg * kPpSeg + warp * PW + q;
    gi = 0;
    gv = T(0);
    if (s < s_end) {
      gi = idx[s];
      gv = PERM ? vals[perm[s]] : vals[s];
    }
  };
  auto products = [&](int sg, int gi, T gv) {
    T (*buf)[32] = s_p[sg & 1];
    T xv[PW];
#pragma unroll
    for (int q = 0; q < PW; ++q)
      xv[q] = ldg_stream(dcol + (size_t)(uint32_t)__shfl_sync(0xffffffffu, gi, q) * ldu);
#pragma unroll
    for (int q = 0; q < PW; ++q) buf[warp * PW + q][lane] = mul_rn(__shfl_sync(0xffffffffu, gv, q), xv[q]);
  };
  int gi;
  T gv;
  load_iv(0, gi, gv);
  pdl_wait();  // the dense operand is the previous kernel's output
  if (nseg > 0) products(0, gi, gv);
  if (nseg > 1) load_iv(1, gi, gv);
  __syncthreads();
  T acc = T(0);
  for (int sg = 0; sg < nseg; ++sg) {
    // warps 1..7 (and warp 0 first) produce segment sg + 1 while warp 0 sums sg
    if (sg + 1 < nseg) {
      products(sg + 1, gi, gv);
      if (sg + 2 < nseg) load_iv(sg + 2, gi, gv);
    }
    if (warp == 0) {
      const T (*buf)[32] = s_p[sg & 1];
      const int cnt = min(kPpSeg, len - sg * kPpSeg);
      if (cnt == kPpSeg) {
#pragma unroll 16
        for (int q = 0; q < kPpSeg; ++q) acc = add_rn(acc, buf[q][lane]);
      } else {
        for (int q = 0; q < cnt; ++q) acc = add_rn(acc, buf[q][lane]);
      }
    }
    __syncthreads();  // segment sg consumed, sg + 1 produced
  }
  pdl_trigger();
  if (warp != 0 || !valid) return;
  if constexpr (EPI == kEpiBiasAct) {
    if (epi.bias != nullptr) acc = add_rn(acc, bias_r);
    if (epi.relu) acc = relu_np(acc);
  } else {
    if (epi.mask != nullptr) acc = mask_np(acc, mk);
  }
  out[row * ld_out + col] = acc;
}

template <typename T, int EPI, bool PERM>
__global__ void __launch_bounds__(32)
    row_spmm_deep_kernel(const int32_t* __restrict__ seg_ptr, const int32_t* __restrict__ idx,
                         const int32_t* __restrict__ perm, const T* __restrict__ vals,
                         const T* __restrict__ dense, int64_t ld_dense, int64_t n,
                         T* __restrict__ out, int64_t ld_out, EpiArgs<T> epi) {
  const int lane = threadIdx.x;
  const int64_t row = blockIdx.x;
  const int64_t col = (int64_t)blockIdx.y * 32 + lane;
  const bool valid = col < n;
  T bias_r = T(0), mk = T(0);
  if constexpr (EPI == kEpiBiasAct) {
    if (epi.bias != nullptr) bias_r = epi.bias[row];
  } else {
    if (epi.mask != nullptr && valid) mk = epi.mask[row * epi.ld_mask + col];
  }
  T acc = deep_row_chain<T, PERM>(seg_ptr, idx, perm, vals, dense + (valid ? col : 0),
                                  (uint32_t)ld_dense, row, lane);
  pdl_trigger();
  if (!valid) return;
  if constexpr (EPI == kEpiBiasAct) {
    if (epi.bias != nullptr) acc = add_rn(acc, bias_r);
    if (epi.relu) acc = relu_np(acc);
  } else {
    if (epi.mask != nullptr) acc = mask_np(acc, mk);
  }
  out[row * ld_out + col] = acc;
}


// L2 budget for the slice of the gathered dense operand (B200: 126 MB L2;
// leave room for the output stream, indices and values)
constexpr int64_t kL2SliceBytes = 48ll << 20;

template <typename T, int W, int U, int EPI, bool PERM>
bool launch_rows(const int32_t* seg_ptr, const int32_t* idx, const int32_t* perm, const T* vals,
                 int64_t n_rows, int64_t dense_rows, const T* dense, int64_t ld_dense, int64_t n,
                 T* out, int64_t ld_out, EpiArgs<T> epi, cudaStream_t st) {
  const int64_t chunks = ceil_div(n, 32 * W);
  // The fused row-sum needs the whole row in one CTA; take that shape when
  // there are enough rows to fill the GPU, else narrow CTAs (<= 8 warps) and
  // the separate warp-per-row bias kernel.
  const int64_t dense_bytes = dense_rows * n * (int64_t)sizeof(T);
  const bool fuse = EPI == kEpiMask && epi.rowsum && n_rows >= 2 * 148 &&
                    chunks <= max_threads_for<W>() / 32 && dense_bytes <= kL2SliceBytes;
  // unfused: narrow CTAs (as few as 1 warp) when rows are few, so the warps
  // of a short, wide layer still spread over all 148 SMs
  int warps = (int)imin(8, chunks);
  while (warps > 1 && n_rows * ceil_div(chunks, warps) < 2 * 148) warps >>= 1;
  // dense operand wider than L2: column slices of `warps` chunks whose rows
  // fit the L2 budget (all output rows gather from one slice before the next
  // starts), the CTA filled with rows_per_cta rows of that slice (config 5:
  // 65536 x 4096 fp32 = 1 GB gathered per SpMM)
  int rpc = 1;
  if (!fuse && dense_bytes > kL2SliceBytes) {
    const int64_t slice_cols = imax(32 * W, kL2SliceBytes / (dense_rows * (int64_t)sizeof(T)));
    const int wmax = (int)imax(1, imin(8, slice_cols / (32 * W)));
    while (warps > wmax) warps >>= 1;
    rpc = 8 / warps;
    if (n_rows < 148 * 2 * rpc) rpc = 1;
  }
  if (fuse) warps = (int)chunks;
  const int64_t gy = ceil_div(chunks, warps);
  size_t dyn = 0;
  if (fuse) dyn = sizeof(T) * (size_t)(((n + 3) & ~int64_t(3)) + warp_pairwise_leaves((int)n));
  epi.rowsum = fuse ? 1 : 0;
  auto kern = fuse      ? row_spmm_kernel<T, W, U, EPI, PERM, false, EPI == kEpiMask>
              : rpc > 1 ? row_spmm_kernel<T, W, U, EPI, PERM, true>
                        : row_spmm_kernel<T, W, U, EPI, PERM, false>;
  if (dyn > 40 * 1024)
    ensure_smem(kern, dyn);
  launch_k(kern, dim3((unsigned)ceil_div(n_rows, rpc), (unsigned)gy), dim3(warps * rpc * 32), dyn,
           st, seg_ptr, idx, perm, vals, dense, ld_dense, n, out, ld_out, epi, rpc, n_rows);
  return epi.rowsum != 0;
}

// n_rows x n outputs; *rowsum_done tells whether the fused row-sum ran
template <typename T, int EPI, bool PERM>
int launch_segment_spmm(const int32_t* seg_ptr, const int32_t* idx, const int32_t* perm,
                        const T* vals, int64_t n_rows, int64_t dense_rows, const T* dense,
                        int64_t ld_dense, int64_t n, T* out, int64_t ld_out, EpiArgs<T> epi,
                        cudaStream_t st, const char* name, bool* rowsum_done,
                        double avg_len = -1.0) {
  if (rowsum_done) *rowsum_done = false;
  if (n_rows == 0 || n == 0) return SMB_OK;
  if (n == 1 && !epi.rowsum) {  // one batch column: warp-per-row SpMV
    launch_k(row_spmv_kernel<T, EPI, PERM>, dim3((unsigned)ceil_div(n_rows, kSpmvWarps)),
             dim3(kSpmvWarps * 32), 0, st, seg_ptr, idx, perm, vals, dense, ld_dense, n_rows, out,
             ld_out, epi);
    return check_launch(name);
  }
  constexpr int VW = Vec16<T>::N;
  const bool vec_ok = aligned16(dense) && aligned16(out) && ld_dense % VW == 0 &&
                      ld_out % VW == 0 &&
                      (EPI != kEpiMask || epi.mask == nullptr ||
                       (aligned16(epi.mask) && epi.ld_mask % VW == 0));
  // One 16-byte vector per lane when the warp count fills 148 SMs (measured
  // on B200 against 2 x 16 B lanes: 1.1-1.6x faster from config 2 to config 3
  // sizes -- lower register pressure, more resident warps); with few rows one
  // column per lane spreads each row over many more warps.
  auto enough = [&](int w) { return n >= 32 * w && n_rows * ceil_div(n, 32 * w) >= 148 * 8; };
  bool done;
  if (avg_len >= 0 && avg_len <= 32 && vec_ok && enough(2 * VW))
    // short segments (<= 32 nonzeros on average; known when the pattern is):
    // two vectors per lane with a 2-deep ring halve the warps per row and
    // the per-column index / shuffle work (config 2: 1.2-1.3x); long
    // segments keep one vector and a 4-deep ring (1.2-1.5x better there)
    done = launch_rows<T, 2 * VW, 2, EPI, PERM>(seg_ptr, idx, perm, vals, n_rows, dense_rows,
                                                dense, ld_dense, n, out, ld_out, epi, st);
  else if (vec_ok && enough(VW))
    done = launch_rows<T, VW, 4, EPI, PERM>(seg_ptr, idx, perm, vals, n_rows, dense_rows, dense,
                                            ld_dense, n, out, ld_out, epi, st);
  // one column per lane: ring depth by shape (measured on B200: many short
  // rows prefer a shallow ring -- more resident warps -- while a few long
  // rows over a wide batch need the deep one)
  else if (n_rows >= 148)
    done = launch_rows<T, 1, 8, EPI, PERM>(seg_ptr, idx, perm, vals, n_rows, dense_rows, dense,
                                           ld_dense, n, out, ld_out, epi, st);
  else if (!(EPI == kEpiMask && epi.rowsum) && n < 512) {
    // few long rows, narrow batch: parallel products + serial sum
    launch_k(row_spmm_pp_kernel<T, EPI, PERM>, dim3((unsigned)n_rows, (unsigned)ceil_div(n, 32)),
             dim3(32 * kPpWarps), 0, st, seg_ptr, idx, perm, vals, dense, ld_dense, n, out, ld_out,
             epi);
    done = false;
  } else if (!(EPI == kEpiMask && epi.rowsum)) {
    launch_k(row_spmm_deep_kernel<T, EPI, PERM>, dim3((unsigned)n_rows, (unsigned)ceil_div(n, 32)),
             dim3(32), 0, st, seg_ptr, idx, perm, vals, dense, ld_dense, n, out, ld_out, epi);
    done = false;
  } else if (n < 512)
    done = launch_rows<T, 1, 16, EPI, PERM>(seg_ptr, idx, perm, vals, n_rows, dense_rows, dense,
                                            ld_dense, n, out, ld_out, epi, st);
  else
    done = launch_rows<T, 1, 32, EPI, PERM>(seg_ptr, idx, perm, vals, n_rows, dense_rows, dense,
                                            ld_dense, n, out, ld_out, epi, st);
  if (rowsum_done) *rowsum_done = done;
  return check_launch(name);
}

}  // namespace

// warp-per-row reduction + bias update (elementwise.cu), used when the fused
// epilogue cannot cover a row (batches wider than 32 warps x 32 x W columns)
template <typename T>
int launch_bias_rows(const T* d, int64_t ld, int64_t m, int64_t n, T* bias, T* vbias, T* grad,
                     const OptConsts<T>& opt, cudaStream_t st);

template <typename T>
int spmm_t_fused_impl(const smb_pattern* pat, const void* values, const void* dense,
                      int64_t ld_dense, int64_t n, const void* mask, int64_t ld_mask, void* out,
                      int64_t ld_out, void* bias, void* vbias, void* grad_bias_out, int opt_kind,
                      double mu, double eta, void* stream, bool csc_values = false) {
  const bool want_rows =
      grad_bias_out != nullptr || (opt_kind != SMB_OPT_NONE && bias != nullptr);
  EpiArgs<T> epi{};
  epi.mask = static_cast<const T*>(mask);
  epi.ld_mask = ld_mask;
  epi.rowsum = want_rows ? 1 : 0;
  epi.rb_bias = static_cast<T*>(bias);
  epi.rb_vbias = static_cast<T*>(vbias);
  epi.rb_grad = static_cast<T*>(grad_bias_out);
  epi.opt = make_opt<T>(opt_kind, mu, eta);
  bool done = false;
  cudaStream_t st = as_stream(stream);
  const double avg = pat->k > 0 ? (double)pat->nnz / (double)pat->k : -1.0;
  int rc = csc_values
               ? launch_segment_spmm<T, kEpiMask, false>(
                     pat->col_ptr, pat->row_idx, nullptr, static_cast<const T*>(values), pat->k,
                     pat->m, static_cast<const T*>(dense), ld_dense, n, static_cast<T*>(out), ld_out, epi,
                     st, "smb_spmm_t_csc", &done, avg)
               : launch_segment_spmm<T, kEpiMask, true>(
                     pat->col_ptr, pat->row_idx, pat->perm, static_cast<const T*>(values), pat->k,
                     pat->m, static_cast<const T*>(dense), ld_dense, n, static_cast<T*>(out), ld_out, epi,
                     st, "smb_spmm_t", &done, avg);
  if (rc != SMB_OK || !want_rows || done) return rc;
  return launch_bias_rows<T>(static_cast<const T*>(out), ld_out, pat->k, n, epi.rb_bias,
                             epi.rb_vbias, epi.rb_grad, epi.opt, st);
}

}  // namespace smb

using namespace smb;

namespace {
template <typename T>
int spmm_impl(const int32_t* row_ptr, const int32_t* col_idx, const void* values, int64_t m,
              int64_t k, const void* dense, int64_t ld_dense, int64_t n, const void* bias,
              int epilogue, void* out, int64_t ld_out, void* stream, double avg_len = -1.0) {
  EpiArgs<T> epi{};
  epi.bias = static_cast<const T*>(bias);
  epi.relu = epilogue == SMB_EPI_RELU;
  return launch_segment_spmm<T, kEpiBiasAct, false>(
      row_ptr, col_idx, nullptr, static_cast<const T*>(values), m, k,
      static_cast<const T*>(dense),
      ld_dense, n, static_cast<T*>(out), ld_out, epi, as_stream(stream), "smb_spmm", nullptr,
      avg_len);
}

int spmm_t_checks(const smb_pattern* pat, int64_t ld_dense, int64_t n, const void* mask,
                  int64_t ld_mask, void* out, int64_t ld_out) {
  SMB_REQUIRE(pat != nullptr, "smb_spmm_t: null pattern");
  SMB_REQUIRE(n >= 0, "smb_spmm_t: negative dimension");
  SMB_REQUIRE(ld_dense >= n && ld_out >= n, "smb_spmm_t: leading dimension smaller than n");
  SMB_REQUIRE(mask == nullptr || ld_mask >= n, "smb_spmm_t: mask leading dimension");
  SMB_REQUIRE(pat->k == 0 || out != nullptr, "smb_spmm_t: null output");
  SMB_REQUIRE(pat->k < (int64_t(1) << 31), "smb_spmm_t: too many columns");
  return SMB_OK;
}
}  // namespace

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
  SMB_REQUIRE(m < (int64_t(1) << 31), "smb_spmm: too many rows");
  if (dtype == SMB_F32)
    return spmm_impl<float>(row_ptr, col_idx, values, m, k, dense, ld_dense, n, bias, epilogue,
                            out, ld_out, stream);
  if (dtype == SMB_F64)
    return spmm_impl<double>(row_ptr, col_idx, values, m, k, dense, ld_dense, n, bias, epilogue,
                             out, ld_out, stream);
  set_error("smb_spmm: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}

extern "C" int smb_spmm_p(int dtype, const smb_pattern* pat, const void* values,
                          const void* dense, int64_t ld_dense, int64_t n, const void* bias,
                          int epilogue, void* out, int64_t ld_out, void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_spmm_p: null pattern");
  SMB_REQUIRE(n >= 0, "smb_spmm_p: negative dimension");
  SMB_REQUIRE(ld_dense >= n && ld_out >= n, "smb_spmm_p: leading dimension smaller than n");
  SMB_REQUIRE(epilogue == SMB_EPI_NONE || epilogue == SMB_EPI_RELU, "smb_spmm_p: bad epilogue %d",
              epilogue);
  SMB_REQUIRE(pat->m == 0 || out != nullptr, "smb_spmm_p: null output");
  const double avg = pat->m > 0 ? (double)pat->nnz / (double)pat->m : -1.0;
  if (dtype == SMB_F32)
    return spmm_impl<float>(pat->row_ptr, pat->col_idx, values, pat->m, pat->k, dense, ld_dense,
                            n, bias, epilogue, out, ld_out, stream, avg);
  if (dtype == SMB_F64)
    return spmm_impl<double>(pat->row_ptr, pat->col_idx, values, pat->m, pat->k, dense, ld_dense,
                             n, bias, epilogue, out, ld_out, stream, avg);
  set_error("smb_spmm_p: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}

extern "C" int smb_spmm_t(int dtype, const smb_pattern* pat, const void* values,
                          const void* dense, int64_t ld_dense, int64_t n, const void* mask,
                          int64_t ld_mask, void* out, int64_t ld_out, void* stream) {
  clear_error();
  const int rc = spmm_t_checks(pat, ld_dense, n, mask, ld_mask, out, ld_out);
  if (rc != SMB_OK) return rc;
  if (dtype == SMB_F32)
    return spmm_t_fused_impl<float>(pat, values, dense, ld_dense, n, mask, ld_mask, out, ld_out,
                                    nullptr, nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0, stream);
  if (dtype == SMB_F64)
    return spmm_t_fused_impl<double>(pat, values, dense, ld_dense, n, mask, ld_mask, out, ld_out,
                                     nullptr, nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0, stream);
  set_error("smb_spmm_t: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}

extern "C" int smb_spmm_t_csc(int dtype, const smb_pattern* pat, const void* values_csc,
                              const void* dense, int64_t ld_dense, int64_t n, const void* mask,
                              int64_t ld_mask, void* out, int64_t ld_out, void* stream) {
  clear_error();
  const int rc = spmm_t_checks(pat, ld_dense, n, mask, ld_mask, out, ld_out);
  if (rc != SMB_OK) return rc;
  if (dtype == SMB_F32)
    return spmm_t_fused_impl<float>(pat, values_csc, dense, ld_dense, n, mask, ld_mask, out,
                                    ld_out, nullptr, nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0,
                                    stream, true);
  if (dtype == SMB_F64)
    return spmm_t_fused_impl<double>(pat, values_csc, dense, ld_dense, n, mask, ld_mask, out,
                                     ld_out, nullptr, nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0,
                                     stream, true);
  set_error("smb_spmm_t_csc: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}

namespace smb {
namespace {
template <typename T>
__global__ void values_to_csc_kernel(const int32_t* __restrict__ perm, const T* __restrict__ src,
                                     T* __restrict__ dst, int64_t nnz) {
  pdl_wait();  // src is the update kernel's output
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += stride)
    dst[q] = src[perm[q]];
  pdl_trigger();
}
}  // namespace
}  // namespace smb

extern "C" int smb_values_to_csc(int dtype, const smb_pattern* pat, const void* values,
                                 void* values_csc, void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_values_to_csc: null pattern");
  if (pat->nnz == 0) return SMB_OK;
  SMB_REQUIRE(values != nullptr && values_csc != nullptr, "smb_values_to_csc: null values");
  SMB_REQUIRE(values != values_csc, "smb_values_to_csc: in-place permutation");
  const unsigned grid = (unsigned)imin(ceil_div(pat->nnz, 256), 148 * 8);
  if (dtype == SMB_F32)
    launch_k(values_to_csc_kernel<float>, dim3(grid), dim3(256), 0, as_stream(stream), pat->perm,
             static_cast<const float*>(values), static_cast<float*>(values_csc), pat->nnz);
  else if (dtype == SMB_F64)
    launch_k(values_to_csc_kernel<double>, dim3(grid), dim3(256), 0, as_stream(stream), pat->perm,
             static_cast<const double*>(values), static_cast<double*>(values_csc), pat->nnz);
  else {
    set_error("smb_values_to_csc: unsupported dtype %d", dtype);
    return SMB_ERR_INVALID;
  }
  return check_launch("smb_values_to_csc");
}

extern "C" int smb_spmm_t_bias(int dtype, const smb_pattern* pat, const void* values,
                               const void* dense, int64_t ld_dense, int64_t n, const void* mask,
                               int64_t ld_mask, void* out, int64_t ld_out, void* bias,
                               void* velocity_bias, void* grad_bias_out, int opt_kind, double mu,
                               double eta, void* stream) {
  clear_error();
  const int rc = spmm_t_checks(pat, ld_dense, n, mask, ld_mask, out, ld_out);
  if (rc != SMB_OK) return rc;
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_spmm_t_bias: bad optimizer kind %d", opt_kind);
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) ||
                  bias == nullptr || velocity_bias != nullptr,
              "smb_spmm_t_bias: momentum needs a bias velocity buffer");
  if (dtype == SMB_F32)
    return spmm_t_fused_impl<float>(pat, values, dense, ld_dense, n, mask, ld_mask, out, ld_out,
                                    bias, velocity_bias, grad_bias_out, opt_kind, mu, eta,
                                    stream);
  if (dtype == SMB_F64)
    return spmm_t_fused_impl<double>(pat, values, dense, ld_dense, n, mask, ld_mask, out, ld_out,
                                     bias, velocity_bias, grad_bias_out, opt_kind, mu, eta,
                                     stream);
  set_error("smb_spmm_t_bias: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}
