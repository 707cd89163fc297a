// Column-chain step kernel (sm_100a): the batch-column-parallel middle of one
// training step in ONE launch.
//
// After the first layer's forward product, everything up to the input
// gradient of layer 1 is independent per batch column (sample):
//
//   forward   a_l = act(W_l a_{l-1} + b_l)          l = 1..L-1   nn.py:169-176, 86-87
//   loss      d_L = (softmax(a_{L-1}) - t) / B                    nn.py:385-417, train.py:399
//   backward  d_{l-1} = (W_l^T d_l) * (a_{l-1} > 0)  l = L-1..1   nn.py:178-185, 89-91
//
// (layer indices 0-based as in engine.py: W_0 is the first layer).  Each of
// these was its own latency-bound launch (config 2: two SpMMs, the output
// layer, the softmax step and two transposed SpMMs, ~28 us of kernels for
// 36 K nonzeros).  Here a thread-block cluster owns 32 batch columns
// (lane = column) and its C CTAs split the output rows of every product; the
// dense operand of a product (all rows of a_{l-1} or d_l for the cluster's 32
// columns) is staged in shared memory by TMA as [rows][32] fp32, 128 bytes per
// row, so lane c reading element (r, c) is conflict-free for any r.  Between
// products the CTAs write their rows to global memory (the step needs every
// activation and gradient there anyway: masks, SDDMMs, bias row sums), meet at
// a cluster barrier (release/acquire), and re-load the full operand with one
// 2-D tensor copy per 256 rows.  The index/value segments of each CTA's rows
// (CSR for the forward products, CSC for the transposed ones) are staged once
// at launch with cp.async, before the programmatic-dependency wait, so they
// overlap the previous kernel's tail; the inner loop reads 4 (index, value)
// pairs with two broadcast 16-byte shared loads and gathers 4 operand
// elements.
//
// Arithmetic is exactly the separate kernels' (and the reference's): each
// output element sums its segment in ascending source index from 0 with
// multiply and add rounded separately (_kernels.py:25-59), then bias / ReLU
// (np.maximum) or the ReLU mask; the softmax column code and the fixed-order
// loss reduction are those of softmax_step_kernel (elementwise.cu), whose
// 128-column CTAs are 4 of this kernel's column groups.
#include "async_copy.cuh"
#include "pattern.cuh"
#include "tma.cuh"

#include <climits>
#include <algorithm>
#include <cstring>
#include <vector>

namespace smb {
namespace {

constexpr int kChainMaxL = 6;
constexpr int kChainWarps = 16;
constexpr int kChainThreads = 32 * kChainWarps;
constexpr int kBoxRows = 256;
constexpr int kChainMaxClasses = 16;
constexpr int kChainMaxC = 8;

// one staged sparse product (a forward layer or a transposed one)
struct ChainPhase {
  const int32_t* ptr;  // segment pointers (row_ptr / col_ptr), [rows + 1]
  const int32_t* idx;  // col_idx / row_idx
  const float* val;    // CSR values / CSC-ordered values
  const float* bias;   // forward: per-row bias, or null
  float* out;          // [rows x ld]
  int rows;            // output rows
  int nnz;
  int split[kChainMaxC + 1];  // the cluster's CTAs' row ranges (balanced by nonzeros)
  int act;             // forward: np.maximum(., 0); backward: ReLU mask of the layer below
  int meta_off;        // shared-memory byte offset of the staged segment
  int ptr_words;       // staged pointer words (multiple of 4)
  int nz_words;        // staged index words = value words (multiple of 4)
  int epi_off;         // forward: staged bias slice; backward: mask bits (byte offset)
  const int32_t* order;  // [rows]: each CTA's rows, longest segment first
  int order_off;       // shared-memory byte offset of the staged order slice
  int in_map;          // tensor map that reloads the operand into region A, -1: none
  int in_boxes;        // 256-row boxes of that reload
  int in_box_rows;
  int wide;            // long rows: one row per warp, one column per lane
};

struct ChainParams {
  CUtensorMap maps[2 * kChainMaxL];
  ChainPhase ph[2 * kChainMaxL];
  int n;
  int64_t ld;
  int classes;
  float* dy_top;  // d_{L-1}
  const float* t;
  int64_t ld_t;
  float divisor;
  double* loss;
  double* parts;
  unsigned* ticket;
  int ngroups;
  int off_A, off_D, off_LG;
  unsigned long long* prof;  // diagnostics: per-CTA phase timestamps, or null
};

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// every thread of every CTA of the cluster: prior global and distributed
// shared-memory writes are visible to the cluster's later reads (TMA
// included: the generic -> async proxy fence precedes the release)
__device__ __forceinline__ void cluster_exchange() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ int lds_s32(const int32_t* p) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ float lds_f32(const float* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ float lds_f32x1(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f32x4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c, int r,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c), "r"(r), "r"(bar)
      : "memory");
}

enum ChainKind { kFwd = 0, kFwdLast = 1, kBwd = 2 };

// What one warp needs to run its rows of one product.
struct RowTask {
  const int32_t* sp;  // staged pointers; row r at sp[r - pr0]
  int pr0;
  int a0;             // staged nonzero s at si[s - a0] / sv[s - a0]
  const int32_t* si;
  const float* sv;
  const int32_t* order;  // the CTA's rows, longest segment first
  int nrows;
  const float* X;     // operand [rows][32]
  const float* sbias;  // forward: staged bias, row r at sbias[r - pr0]
  const unsigned* mbits;  // backward: ReLU mask bits, row r at mbits[r - r0]
  int r0;
  int act;
  float* out;
  int64_t ld;
  int n;              // batch width (valid columns)
  int c0;             // first column of the cluster's group
  unsigned lg;        // forward-last: shared address of the logits block
  unsigned C;
  unsigned long long* dbg;
};

// The CTA's rows of one product.  A warp runs up to 4 rows at a time, one
// per 8-lane group; lane l8 of a group owns columns 4*l8 .. 4*l8+3 (16-byte
// operand reads: the 8 lanes of a group read one 128-byte operand row, the
// 4 groups 4 rows -- conflict-free).  Rows are taken longest first, so the
// rows a warp runs together have about the same length.  Each element sums its
// segment in ascending s from 0, multiply and add rounded separately; then
// the epilogue (bias + ReLU, or the ReLU mask of the layer below) and one
// 16-byte store per lane.
template <int K>
__device__ __forceinline__ void run_rows(const RowTask& w, int warp, int lane) {
  const int g = lane >> 3, l8 = lane & 7;
  const int cq = 4 * l8;  // first of this lane's 4 columns in the group
  const float* Xl = w.X + cq;
  int dk = 0;
  auto dstamp = [&]() {
    if (w.dbg != nullptr && lane == 0 && warp == 0 && dk < 12) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      w.dbg[dk] = t;
    }
    ++dk;
  };
  dstamp();
  // slot (sorted row) warp + 16 g + 64 t: a CTA with at most 16 rows gives
  // every warp its own row
  for (int base = warp; base < w.nrows; base += 4 * kChainWarps) {
    const int slot = base + kChainWarps * g;
    const bool has = slot < w.nrows;
    const int r = has ? w.order[slot] : -1;
    int s = 0, e = 0;
    if (has) {
      s = w.sp[r - w.pr0] - w.a0;
      e = w.sp[r + 1 - w.pr0] - w.a0;
    }
    const int trip = __reduce_max_sync(0xffffffffu, e - s);
    dstamp();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    // software pipeline over rounds of 4 elements: the indices / values of
    // round i+2 and the operands of round i+1 are in flight while round i is
    // summed (volatile shared loads keep each batch together)
    const int32_t* ci = w.si - w.a0;
    const float* cv = w.sv - w.a0;
    const unsigned xb = smem_u32(Xl);
    const int eg = e + w.a0;  // global index of the row end
    auto meta = [&](int jb, int (&c)[4], float (&v)[4]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool p = jb + u < eg;
        const int jj = p ? jb + u : w.a0;  // (staged word 0 when past the end)
        c[u] = lds_s32(ci + jj);
        v[u] = lds_f32(cv + jj);
      }
    };
    auto operands = [&](int jb, const int (&c)[4], float4 (&x)[4]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int cc = jb + u < eg ? c[u] : 0;  // row 0: in range whatever was read
        x[u] = lds_f32x4(xb + (unsigned)cc * 128u);
      }
    };
    int c0[4], c1[4];
    float v0[4], v1[4];
    float4 x0[4];
    const int jg = s + w.a0;  // global nonzero index of the row start
    meta(jg, c0, v0);
    meta(jg + 4, c1, v1);
    operands(jg, c0, x0);
    for (int i = 0; i < trip; i += 4) {
      const int j = jg + i;
      float4 x1[4];
      operands(j + 4, c1, x1);
      int c2[4];
      float v2[4];
      meta(j + 8, c2, v2);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j + u < eg) {
          acc.x = add_rn(acc.x, mul_rn(v0[u], x0[u].x));
          acc.y = add_rn(acc.y, mul_rn(v0[u], x0[u].y));
          acc.z = add_rn(acc.z, mul_rn(v0[u], x0[u].z));
          acc.w = add_rn(acc.w, mul_rn(v0[u], x0[u].w));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v0[u] = v1[u];
        x0[u] = x1[u];
        c1[u] = c2[u];
        v1[u] = v2[u];
      }
    }
    dstamp();
    if (!has) continue;
    if constexpr (K == kBwd) {
      if (w.act) {
        const unsigned bits = w.mbits[r - w.r0] >> cq;
        acc.x = mul_rn(acc.x, (bits & 1u) ? 1.f : 0.f);
        acc.y = mul_rn(acc.y, (bits & 2u) ? 1.f : 0.f);
        acc.z = mul_rn(acc.z, (bits & 4u) ? 1.f : 0.f);
        acc.w = mul_rn(acc.w, (bits & 8u) ? 1.f : 0.f);
      }
    } else {
      if (w.sbias != nullptr) {
        const float b = w.sbias[r - w.pr0];
        acc.x = add_rn(acc.x, b);
        acc.y = add_rn(acc.y, b);
        acc.z = add_rn(acc.z, b);
        acc.w = add_rn(acc.w, b);
      }
      if constexpr (K == kFwd) {
        if (w.act) {
          acc.x = relu_np(acc.x);
          acc.y = relu_np(acc.y);
          acc.z = relu_np(acc.z);
          acc.w = relu_np(acc.w);
        }
      }
    }
    const int col = w.c0 + cq;
    float* o = w.out + (int64_t)r * w.ld + col;
    if (col + 3 < w.n) {
      *reinterpret_cast<float4*>(o) = acc;
    } else {
      if (col < w.n) o[0] = acc.x;
      if (col + 1 < w.n) o[1] = acc.y;
      if (col + 2 < w.n) o[2] = acc.z;
    }
    if constexpr (K == kFwdLast) {
      // the logits of the cluster's columns into every CTA's logit block
      const unsigned a = w.lg + (unsigned)(r * 32 + cq) * 4u;
      for (unsigned t = 0; t < w.C; ++t) {
        unsigned remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(a), "r"(t));
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote),
                     "f"(acc.x), "f"(acc.y), "f"(acc.z), "f"(acc.w)
                     : "memory");
      }
    }
  }
}

__device__ __forceinline__ int4 lds_s32x4(const int32_t* p) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ float4 lds_f32v4(const float* p) {
  return lds_f32x4(smem_u32(p));
}

// Long rows (the output layer's ~300-nonzero rows at config 2): one row per
// warp, one column per lane, so a lane's chain costs ~5 instructions per
// element instead of ~15 (quads of (index, value) pairs by broadcast 16-byte
// loads two quads ahead, the 4 operands of the next quad one quad ahead).
template <int K>
__device__ __forceinline__ void run_rows_wide(const RowTask& w, int warp, int lane) {
  const int32_t* ci = w.si - w.a0;
  const float* cv = w.sv - w.a0;
  const unsigned xl = smem_u32(w.X) + 4u * (unsigned)lane;
  for (int slot = warp; slot < w.nrows; slot += kChainWarps) {
    const int r = w.order[slot];
    int j = w.sp[r - w.pr0];
    const int e = w.sp[r + 1 - w.pr0];
    float acc = 0.f;
    for (; j < e && (j & 3); ++j)
      acc = add_rn(acc, mul_rn(lds_f32(cv + j), lds_f32x1(xl + 128u * (unsigned)lds_s32(ci + j))));
    const int nq = (e - j) >> 2;
    if (nq > 0) {
      const int last = j + 4 * (nq - 1);
      const int jb = j;
      auto at = [&](int i) { return min(jb + 4 * i, last); };
      auto xq = [&](const int4 c) {
        return make_float4(lds_f32x1(xl + 128u * (unsigned)c.x), lds_f32x1(xl + 128u * (unsigned)c.y),
                           lds_f32x1(xl + 128u * (unsigned)c.z), lds_f32x1(xl + 128u * (unsigned)c.w));
      };
      int4 c1 = lds_s32x4(ci + at(1));
      float4 v0 = lds_f32v4(cv + at(0)), v1 = lds_f32v4(cv + at(1));
      float4 x0 = xq(lds_s32x4(ci + at(0)));
      for (int i = 0; i < nq; ++i) {
        const float4 x1 = xq(c1);
        const int4 c2 = lds_s32x4(ci + at(i + 2));
        const float4 v2 = lds_f32v4(cv + at(i + 2));
        acc = add_rn(acc, mul_rn(v0.x, x0.x));
        acc = add_rn(acc, mul_rn(v0.y, x0.y));
        acc = add_rn(acc, mul_rn(v0.z, x0.z));
        acc = add_rn(acc, mul_rn(v0.w, x0.w));
        v0 = v1;
        x0 = x1;
        v1 = v2;
        c1 = c2;
      }
      j += 4 * nq;
    }
    for (; j < e; ++j)
      acc = add_rn(acc, mul_rn(lds_f32(cv + j), lds_f32x1(xl + 128u * (unsigned)lds_s32(ci + j))));
    if constexpr (K == kBwd) {
      if (w.act) acc = mul_rn(acc, ((w.mbits[r - w.r0] >> lane) & 1u) ? 1.f : 0.f);
    } else {
      if (w.sbias != nullptr) acc = add_rn(acc, w.sbias[r - w.pr0]);
      if constexpr (K == kFwd) {
        if (w.act) acc = relu_np(acc);
      }
    }
    const int col = w.c0 + lane;
    if (col < w.n) w.out[(int64_t)r * w.ld + col] = acc;
    if constexpr (K == kFwdLast) {
      const unsigned a = w.lg + (unsigned)(r * 32 + lane) * 4u;
      for (unsigned t = 0; t < w.C; ++t) {
        unsigned remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(a), "r"(t));
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(acc) : "memory");
      }
    }
  }
}

template <int L>
__global__ void __launch_bounds__(kChainThreads, 1) chain_kernel(const __grid_constant__ ChainParams P) {
  constexpr int NF = L - 1, NPH = 2 * (L - 1);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long s_bar[NPH + 1];  // + the staging barrier
  __shared__ int s_bnd[NPH][2];
  // the phase descriptors in shared memory: read from the (3 KB) parameter
  // block inside the loops, they miss the constant cache
  __shared__ __align__(16) ChainPhase s_ph[NPH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  static_assert(sizeof(ChainPhase) % 4 == 0, "phase descriptor words");
  static_assert(NPH <= kChainWarps, "one warp per phase descriptor");
  // (one address per load: lanes reading different parameter words would
  // serialise in the constant cache)
  if (lane == 0 && warp < NPH) {
    constexpr int kW = (int)sizeof(ChainPhase) / 4;
    const int* src = reinterpret_cast<const int*>(&P.ph[warp]);
    int* dst = reinterpret_cast<int*>(&s_ph[warp]);
#pragma unroll
    for (int k = 0; k < kW; ++k) dst[k] = src[k];
  }
  const unsigned q = cluster_rank(), C = cluster_size();
  const int group = (int)(blockIdx.x / C);
  const int c0 = group * 32;
  const int valid = (int)imin(32, (int64_t)P.n - c0);
  const int col = c0 + lane;
  const bool ok = lane < valid;
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* A = reinterpret_cast<float*>(base + P.off_A);
  float* D = reinterpret_cast<float*>(base + P.off_D);
  float* LG = reinterpret_cast<float*>(base + P.off_LG);
  const unsigned bar0 = smem_u32(&s_bar[0]);

  unsigned long long* prof = P.prof ? P.prof + (size_t)blockIdx.x * 32 : nullptr;
  int nprof = 0;
  auto stamp = [&]() {
    if (prof != nullptr && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      prof[nprof] = t;
    }
    ++nprof;
  };
  stamp();
  if (tid == 0) {
#pragma unroll
    for (int p = 0; p < NPH; ++p) mbar_init(bar0 + 8 * p, 1);
    mbar_init(bar0 + 8 * NPH, NPH);  // one arrival per phase's staging thread
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  stamp();
  // every phase's segment bounds for this CTA's rows, loaded in parallel
  if (tid < 2 * NPH) {
    const ChainPhase& f = s_ph[tid >> 1];
    s_bnd[tid >> 1][tid & 1] = f.ptr[f.split[q + (tid & 1)]];
  }
  // the targets of the softmax columns (older than the previous kernel)
  float tr[kChainMaxClasses];
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < kChainMaxClasses; ++c)
      tr[c] = (c < P.classes && ok) ? P.t[c * P.ld_t + col] : 0.f;
  }
  __syncthreads();
  stamp();
  // stage every phase's pointer / index / value segment, row order and bias
  // slice for this CTA's rows with 1-D bulk copies (thread p issues phase
  // p's; the last < 4 words of a segment are copied by plain loads, so no
  // copy reads past an array).  Static data and values older than the
  // previous kernel: before the programmatic-dependency wait.
  const unsigned stage_bar = bar0 + 8 * NPH;
  if (tid < NPH) {
    const int p = tid;
    const ChainPhase& f = s_ph[p];
    const int r0 = f.split[q], r1 = f.split[q + 1];
    const int pr0 = r0 & ~3;
    const int a0 = s_bnd[p][0] & ~3;
    const int a1 = s_bnd[p][1];
    int32_t* sp = reinterpret_cast<int32_t*>(base + f.meta_off);
    int32_t* si = sp + f.ptr_words;
    float* sv = reinterpret_cast<float*>(si + f.nz_words);
    unsigned bytes = 0;
    auto seg = [&](void* dst, const void* src, int words) {
      const int body = words & ~3;
      if (body > 0) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_u32(dst)), "l"(src), "r"(4 * body), "r"(stage_bar)
            : "memory");
        bytes += 4u * (unsigned)body;
      }
      for (int k = body; k < words; ++k)
        static_cast<int32_t*>(dst)[k] = static_cast<const int32_t*>(src)[k];
    };
    seg(sp, f.ptr + pr0, r1 + 1 - pr0);
    seg(si, f.idx + a0, a1 - a0);
    seg(sv, f.val + a0, a1 - a0);
    seg(base + f.order_off, f.order + pr0, r1 - pr0);
    if (p < NF && f.bias != nullptr) seg(base + f.epi_off, f.bias + pr0, r1 - pr0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(stage_bar),
                 "r"(bytes)
                 : "memory");
  }
  stamp();

  auto reload = [&](int p) {
    const ChainPhase& f = s_ph[p];
    if (tid == 0 && f.in_map >= 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const unsigned bar = bar0 + 8 * p;
      mbar_expect_tx(bar, (unsigned)(f.in_boxes * f.in_box_rows * 128));
      for (int b = 0; b < f.in_boxes; ++b)
        tma_load_2d(smem_u32(A) + (unsigned)(b * f.in_box_rows * 128), &P.maps[f.in_map], c0,
                    b * f.in_box_rows, bar);
    }
  };
  // the first operand (the first layer's output) is the previous kernel's
  pdl_wait();
  reload(0);
  mbar_wait(stage_bar, 0);
  __syncthreads();  // staged segments (and their plain-copied tails) visible
  stamp();

  double loss_local = 0.0;
#pragma unroll
  for (int p = 0; p < NPH; ++p) {
    const ChainPhase& f = s_ph[p];
    if (p == NF) {
      // softmax cross-entropy gradient of the cluster's 32 columns from the
      // logits every CTA received (so the first transposed product needs no
      // exchange); the rank-0 CTA writes d_{L-1}.  softmax_step_kernel's
      // column code (elementwise.cu).
      if (warp == 0) {
        const int classes = P.classes;
        float er[kChainMaxClasses];
#pragma unroll
        for (int c = 0; c < kChainMaxClasses; ++c) er[c] = c < classes ? LG[c * 32 + lane] : 0.f;
        float mx = er[0];
#pragma unroll
        for (int c = 1; c < kChainMaxClasses; ++c)
          if (c < classes) mx = (er[c] > mx || er[c] != er[c]) ? er[c] : mx;
        float s = 0.f, zt = 0.f;
#pragma unroll
        for (int c = 0; c < kChainMaxClasses; ++c) {
          if (c < classes) {
            const float z = sub_rn(er[c], mx);
            er[c] = exp_full(z);
            s = add_rn(s, er[c]);
            zt = add_rn(zt, mul_rn(z, tr[c]));
          }
        }
#pragma unroll
        for (int c = 0; c < kChainMaxClasses; ++c) {
          if (c < classes) {
            const float g = div_rn(sub_rn(div_rn(er[c], s), tr[c]), P.divisor);
            D[c * 32 + lane] = ok ? g : 0.f;
            if (q == 0 && ok) P.dy_top[c * P.ld + col] = g;
          }
        }
        loss_local = ok ? static_cast<double>(sub_rn(log_full(s), zt)) : 0.0;
      }
      __syncthreads();
      stamp();
    }
    const float* X = p == NF ? D : A;
    if (f.in_map >= 0) {
      mbar_wait(bar0 + 8 * p, 0);
      stamp();
    }
    const int r0 = f.split[q], r1 = f.split[q + 1];
    if (p < NF) {
      // the ReLU mask of the transposed product of this layer (its rows are
      // this operand's rows): one ballot word per row of that product's
      // range, taken while the operand is on chip
      const ChainPhase& b = s_ph[2 * L - 3 - p];
      if (b.act) {
        unsigned* mb = reinterpret_cast<unsigned*>(base + b.epi_off);
        const int b0 = b.split[q], b1 = b.split[q + 1];
        for (int r = b0 + warp; r < b1; r += kChainWarps) {
          const unsigned bits = __ballot_sync(0xffffffffu, A[r * 32 + lane] > 0.f);
          if (lane == 0) mb[r - b0] = bits;
        }
      }
    }
    stamp();
    RowTask w;
    w.dbg = (prof != nullptr && p == NF - 1) ? prof + 20 : nullptr;
    w.sp = reinterpret_cast<const int32_t*>(base + f.meta_off);
    w.pr0 = r0 & ~3;
    w.a0 = s_bnd[p][0] & ~3;
    w.si = w.sp + f.ptr_words;
    w.sv = reinterpret_cast<const float*>(w.si + f.nz_words);
    w.order = reinterpret_cast<const int32_t*>(base + f.order_off) + (r0 - (r0 & ~3));
    w.nrows = r1 - r0;
    w.X = X;
    w.sbias = (p < NF && f.bias != nullptr) ? reinterpret_cast<const float*>(base + f.epi_off)
                                            : nullptr;
    w.mbits = reinterpret_cast<const unsigned*>(base + f.epi_off);
    w.r0 = r0;
    w.act = f.act;
    w.out = f.out;
    w.ld = P.ld;
    w.n = P.n;
    w.c0 = c0;
    w.lg = smem_u32(LG);
    w.C = C;
    if (f.wide) {
      if (p < NF - 1) run_rows_wide<kFwd>(w, warp, lane);
      else if (p == NF - 1) run_rows_wide<kFwdLast>(w, warp, lane);
      else run_rows_wide<kBwd>(w, warp, lane);
    } else {
      if (p < NF - 1) run_rows<kFwd>(w, warp, lane);
      else if (p == NF - 1) run_rows<kFwdLast>(w, warp, lane);
      else run_rows<kBwd>(w, warp, lane);
    }
    stamp();
    if (p + 1 < NPH) {
      // the next product needs every CTA's rows: exchange through L2 (and
      // the logits through distributed shared memory)
      cluster_exchange();
      stamp();
      reload(p + 1);
    }
  }
  pdl_trigger();
  // the loss: the warp sums of the cluster's columns, then -- last group to
  // arrive -- softmax_step_kernel's order: per 128-column CTA the sum of its 4
  // warps from 0.0, then the CTAs in order from 0.0
  if (warp == 0 && q == 0 && P.loss != nullptr) {
    double local = loss_local;
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if (lane == 0) {
      P.parts[group] = local;
      __threadfence();
      if (atomicAdd(P.ticket, 1u) == (unsigned)P.ngroups - 1) {
        __threadfence();
        double tot = 0.0;
        for (int b = 0; b < (P.ngroups + 3) / 4; ++b) {
          double bs = 0.0;
          for (int w = 0; w < 4; ++w)
            bs += (4 * b + w < P.ngroups) ? __ldcg(P.parts + 4 * b + w) : 0.0;
          tot += bs;
        }
        *P.loss = tot;
        *P.ticket = 0u;
      }
    }
  }
}

}  // namespace
}  // namespace smb

struct smb_chain_plan {
  int L = 0, C = 1, ngroups = 0;
  int64_t n = 0, ld = 0;
  int classes = 0;
  size_t smem = 0;
  smb::ChainParams proto;  // everything but the per-step pointers and maps
  std::vector<int64_t> rows;  // m of every layer
  std::vector<int> relu;      // activation after every layer
  int32_t* order_dev = nullptr;  // every phase's row order (owned)
  ~smb_chain_plan() {
    if (order_dev) cudaFree(order_dev);
  }
};

using smb::ChainParams;
using smb::ChainPhase;

extern "C" size_t smb_chain_workspace_bytes(int64_t n) {
  return 256 + sizeof(double) * (size_t)smb::ceil_div(n > 0 ? n : 1, 32);
}

extern "C" int smb_chain_plan_create(int nlayers, const smb_pattern* const* patterns,
                                     const int* relu, int64_t n, int64_t ld,
                                     smb_chain_plan** out) {
  using namespace smb;
  clear_error();
  SMB_REQUIRE(out != nullptr && patterns != nullptr && relu != nullptr,
              "smb_chain_plan_create: null argument");
  *out = nullptr;
  SMB_REQUIRE(nlayers >= 2 && nlayers <= kChainMaxL,
              "chain: unsupported (%d layers; 2..%d)", nlayers, kChainMaxL);
  SMB_REQUIRE(n >= 1 && ld >= n && ld % 4 == 0 && n < (1 << 30),
              "chain: unsupported batch (n=%lld ld=%lld)", (long long)n, (long long)ld);
  SMB_REQUIRE(encode_fn() != nullptr, "chain: unsupported (no tensor-map encoder)");
  for (int l = 0; l < nlayers; ++l) {
    SMB_REQUIRE(patterns[l] != nullptr, "chain: null pattern");
    if (l > 0)
      SMB_REQUIRE(patterns[l]->k == patterns[l - 1]->m, "chain: layer %d input width mismatch", l);
    SMB_REQUIRE(patterns[l]->m < (1 << 24) && patterns[l]->k < (1 << 24) &&
                    patterns[l]->nnz < (1ll << 31),
                "chain: unsupported layer size");
  }
  const int classes = (int)patterns[nlayers - 1]->m;
  SMB_REQUIRE(classes >= 1 && classes <= kChainMaxClasses,
              "chain: unsupported (%d classes; at most %d)", classes, kChainMaxClasses);
  SMB_REQUIRE(relu[nlayers - 1] == 0, "chain: the last layer feeds the softmax (no activation)");

  auto* plan = new smb_chain_plan();
  const int L = nlayers;
  plan->L = L;
  plan->n = n;
  plan->ld = ld;
  plan->classes = classes;
  plan->ngroups = (int)ceil_div(n, 32);
  // CTAs per cluster: 8 while that keeps one wave of 1-CTA-per-SM clusters
  // (at most 132 CTAs are placed at cluster size 4), else 4 -- wider batches
  // run several waves of clusters
  const int C = (int64_t)plan->ngroups * 8 <= 132 ? 8 : 4;
  plan->C = C;
  for (int l = 0; l < L; ++l) {
    plan->rows.push_back(patterns[l]->m);
    plan->relu.push_back(relu[l] != 0);
  }
  cudaDeviceSynchronize();  // setup: host copies of the segment pointers
  ChainParams& P = plan->proto;
  memset(&P, 0, sizeof(P));
  size_t off = 0;
  int max_in_rows = 0;
  std::vector<int32_t> order_host;
  std::vector<size_t> order_at(2 * kChainMaxL, 0);
  auto fill = [&](int p, const smb_pattern* pat, bool fwd, int in_rows, int in_map) -> bool {
    ChainPhase& f = P.ph[p];
    const int rows = (int)(fwd ? pat->m : pat->k);
    std::vector<int32_t> ptr((size_t)rows + 1);
    if (cudaMemcpy(ptr.data(), fwd ? pat->row_ptr : pat->col_ptr, sizeof(int32_t) * (rows + 1),
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      return false;
    // the CTAs' row ranges, balanced by nonzeros
    const int64_t z = ptr[rows];
    f.split[0] = 0;
    for (int q = 1; q < C; ++q) {
      const int64_t target = z * q / C;
      const int r = (int)(std::lower_bound(ptr.begin(), ptr.end(), (int32_t)target) - ptr.begin());
      f.split[q] = std::max(f.split[q - 1], std::min(r, rows));
    }
    f.split[C] = rows;
    // each CTA's rows, longest segment first (a warp's 4 rows then take about
    // the same number of steps)
    order_at[p] = order_host.size();
    for (int q = 0; q < C; ++q) {
      std::vector<int32_t> rr;
      for (int r = f.split[q]; r < f.split[q + 1]; ++r) rr.push_back(r);
      std::stable_sort(rr.begin(), rr.end(), [&](int32_t a, int32_t b) {
        return ptr[a + 1] - ptr[a] > ptr[b + 1] - ptr[b];
      });
      order_host.insert(order_host.end(), rr.begin(), rr.end());
    }
    while (order_host.size() % 4) order_host.push_back(0);  // 16-byte aligned phases
    int pw = 0, nw = 0, ew = 0, ow = 0;
    for (int q = 0; q < C; ++q) {
      const int r0 = f.split[q], r1 = f.split[q + 1], pr0 = r0 & ~3;
      pw = std::max(pw, ((r1 + 1 - pr0) + 3) & ~3);
      nw = std::max(nw, ((ptr[r1] - (ptr[r0] & ~3)) + 3) & ~3);
      // forward: the bias slice from pr0; backward: one mask word per row
      ew = std::max(ew, fwd ? (((r1 - pr0) + 3) & ~3) : (((r1 - r0) + 3) & ~3));
      ow = std::max(ow, ((r1 - pr0) + 3) & ~3);
    }
    f.rows = rows;
    f.nnz = (int)pat->nnz;
    // rows of >= 48 nonzeros on average run one per warp (lane = column)
    f.wide = rows > 0 && z >= (int64_t)48 * rows;
    f.ptr = fwd ? pat->row_ptr : pat->col_ptr;
    f.idx = fwd ? pat->col_idx : pat->row_idx;
    f.meta_off = (int)off;
    f.ptr_words = pw;
    f.nz_words = nw;
    off += (size_t)4 * (pw + 2 * (size_t)nw);
    f.epi_off = (int)off;
    off += (size_t)4 * ew;
    f.order_off = (int)off;
    off += (size_t)4 * ow;
    f.in_map = in_map;
    f.in_box_rows = std::min(kBoxRows, std::max(in_rows, 1));
    f.in_boxes = (int)ceil_div(in_rows, f.in_box_rows);
    if (in_map >= 0) max_in_rows = std::max(max_in_rows, f.in_boxes * f.in_box_rows);
    return true;
  };
  bool okc = true;
  // forward phases p = l - 1 for layers l = 1..L-1: operand a_{l-1} (map l-1)
  for (int l = 1; l < L; ++l) {
    okc = okc && fill(l - 1, patterns[l], true, (int)patterns[l]->k, l - 1);
    P.ph[l - 1].act = relu[l] != 0;
  }
  // backward phases p = L-1+j for layers l = L-1-j: operand d_l (region D
  // for the top layer, else map (L-1) + (l-1)); mask = relu of layer l-1
  for (int j = 0; j < L - 1; ++j) {
    const int l = L - 1 - j;
    okc = okc && fill(L - 1 + j, patterns[l], false, (int)patterns[l]->m,
                      j == 0 ? -1 : (L - 1) + (l - 1));
    P.ph[L - 1 + j].act = relu[l - 1] != 0;
  }
  if (okc && cudaMalloc(&plan->order_dev, sizeof(int32_t) * order_host.size()) == cudaSuccess &&
      cudaMemcpy(plan->order_dev, order_host.data(), sizeof(int32_t) * order_host.size(),
                 cudaMemcpyHostToDevice) == cudaSuccess) {
    for (int p = 0; p < 2 * (L - 1); ++p) P.ph[p].order = plan->order_dev + order_at[p];
  } else {
    okc = false;
  }
  if (!okc) {
    delete plan;
    set_error("chain: setting up the segment tables failed");
    return SMB_ERR_CUDA;
  }
  off = (off + 1023) & ~size_t(1023);
  P.off_A = (int)off;
  off += (size_t)max_in_rows * 128;
  P.off_D = (int)off;
  off += (size_t)kChainMaxClasses * 128;
  P.off_LG = (int)off;
  off += (size_t)kChainMaxClasses * 128;
  plan->smem = off + 1024;  // alignment slack
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (plan->smem + 2048 > (size_t)optin) {
    const size_t need = plan->smem;
    delete plan;
    set_error("chain: unsupported (%zu bytes of shared memory > %d)", need, optin);
    return SMB_ERR_INVALID;
  }
  P.n = (int)n;
  P.ld = ld;
  P.classes = classes;
  P.ngroups = plan->ngroups;
  *out = plan;
  return SMB_OK;
}

extern "C" int smb_chain_plan_destroy(smb_chain_plan* plan) {
  delete plan;
  return SMB_OK;
}

extern "C" int smb_chain_plan_profile(smb_chain_plan* plan, void* stamps) {
  using namespace smb;
  clear_error();
  SMB_REQUIRE(plan != nullptr, "smb_chain_plan_profile: null plan");
  plan->proto.prof = static_cast<unsigned long long*>(stamps);
  return SMB_OK;
}

extern "C" int smb_chain_plan_info(const smb_chain_plan* plan, int64_t* info4) {
  using namespace smb;
  clear_error();
  SMB_REQUIRE(plan != nullptr && info4 != nullptr, "smb_chain_plan_info: null argument");
  info4[0] = plan->C;
  info4[1] = plan->ngroups;
  info4[2] = (int64_t)plan->smem;
  info4[3] = plan->L;
  return SMB_OK;
}

namespace {
bool map_rows32(CUtensorMap* map, const void* ptr, int64_t rows, int64_t n, int64_t ld,
                int box_rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return smb::encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int L>
void launch_chain(const smb_chain_plan* plan, const ChainParams& P, cudaStream_t st) {
  auto kern = smb::chain_kernel<L>;
  smb::ensure_smem(kern, plan->smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(plan->ngroups * plan->C));
  cfg.blockDim = dim3(smb::kChainThreads);
  cfg.dynamicSmemBytes = plan->smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)plan->C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, P);
}
}  // namespace

extern "C" int smb_chain_run(const smb_chain_plan* plan, const void* const* values,
                             const void* const* values_csc, const void* const* bias,
                             void* const* acts, void* const* dys, const void* t, int64_t ld_t,
                             double divisor, double* loss_out, void* workspace, void* stream) {
  using namespace smb;
  clear_error();
  SMB_REQUIRE(plan != nullptr && values != nullptr && values_csc != nullptr && bias != nullptr &&
                  acts != nullptr && dys != nullptr && t != nullptr,
              "smb_chain_run: null argument");
  SMB_REQUIRE(ld_t >= plan->n, "smb_chain_run: leading dimension of t smaller than n");
  SMB_REQUIRE(divisor != 0.0, "smb_chain_run: zero divisor");
  SMB_REQUIRE(loss_out == nullptr || workspace != nullptr,
              "smb_chain_run: the loss needs the workspace");
  const int L = plan->L;
  for (int l = 0; l < L; ++l) {
    SMB_REQUIRE(acts[l] != nullptr && dys[l] != nullptr && aligned16(acts[l]) && aligned16(dys[l]),
                "smb_chain_run: activation / gradient buffers must be 16-byte aligned");
    if (l > 0)
      SMB_REQUIRE(values[l] != nullptr && values_csc[l] != nullptr && aligned16(values[l]) &&
                      aligned16(values_csc[l]) && aligned16(bias[l]),
                  "smb_chain_run: value / bias buffers must be 16-byte aligned");
  }
  ChainParams P = plan->proto;
  for (int l = 1; l < L; ++l) {
    ChainPhase& f = P.ph[l - 1];
    f.val = static_cast<const float*>(values[l]);
    f.bias = static_cast<const float*>(bias[l]);
    f.out = static_cast<float*>(acts[l]);
    if (!map_rows32(&P.maps[l - 1], acts[l - 1], plan->rows[l - 1], plan->n, plan->ld,
                    f.in_box_rows)) {
      set_error("chain: tensor map encoding failed");
      return SMB_ERR_CUDA;
    }
  }
  for (int j = 0; j < L - 1; ++j) {
    const int l = L - 1 - j;
    ChainPhase& f = P.ph[L - 1 + j];
    f.val = static_cast<const float*>(values_csc[l]);
    f.bias = nullptr;
    f.out = static_cast<float*>(dys[l - 1]);
    if (f.in_map >= 0 &&
        !map_rows32(&P.maps[f.in_map], dys[l], plan->rows[l], plan->n, plan->ld, f.in_box_rows)) {
      set_error("chain: tensor map encoding failed");
      return SMB_ERR_CUDA;
    }
  }
  P.dy_top = static_cast<float*>(dys[L - 1]);
  P.t = static_cast<const float*>(t);
  P.ld_t = ld_t;
  P.divisor = static_cast<float>(divisor);
  P.loss = loss_out;
  P.ticket = workspace ? static_cast<unsigned*>(workspace) : nullptr;
  P.parts = workspace ? reinterpret_cast<double*>(static_cast<char*>(workspace) + 256) : nullptr;
  cudaStream_t st = as_stream(stream);
  switch (L) {
    case 2: launch_chain<2>(plan, P, st); break;
    case 3: launch_chain<3>(plan, P, st); break;
    case 4: launch_chain<4>(plan, P, st); break;
    case 5: launch_chain<5>(plan, P, st); break;
    default: launch_chain<6>(plan, P, st); break;
  }
  return check_launch("smb_chain_run");
}
