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
// 36 K nonzeros).  Here a thread-block cluster owns 32 batch columns and its C
// CTAs split the output rows of every product (balanced by nonzeros).  The
// dense operand of a product (all rows of a_{l-1} or d_l for the cluster's 32
// columns) is staged in shared memory by TMA as [rows][32] fp32, 128 bytes
// per row, plus one all-zero row.  Between products the CTAs write their rows
// to global memory (the step needs every activation and gradient there
// anyway: masks, SDDMMs, bias row sums), meet at a cluster barrier
// (release/acquire), and re-load the full operand with 2-D tensor copies; the
// output layer's logits go to every CTA of the cluster through distributed
// shared memory.
//
// Segments are PADDED to whole quads of 4 (index, value) pairs: a pad points
// at the operand's zero row with value -0.0, so its product is -0.0 and
// acc + (-0.0) == acc bit for bit for every acc (including -0.0 and NaN): the
// inner loop has no masks, no head or tail.  The padded index arrays are
// built once per plan; the padded value copies are refreshed from the
// layer's values after every update (smb_chain_refresh, the counterpart of
// smb_values_to_csc).  Each CTA's padded segments are staged with 1-D bulk
// copies before the programmatic-dependency wait.
//
// Mapping: a warp runs up to 4 rows at a time, one per 8-lane group; lane l8
// of a group owns columns 4 l8 .. 4 l8 + 3, so a group reads one 128-byte
// operand row per element (16-byte loads, conflict-free); rows are taken
// longest first so a warp's rows end together.  Layers with long rows (the
// output layer: ~300 nonzeros per row at config 2) run one row per warp with
// one column per lane instead.
//
// Arithmetic is exactly the separate kernels' (and the reference's): each
// output element sums its segment in ascending source index from 0 with
// multiply and add rounded separately (_kernels.py:25-59), then bias / ReLU
// (np.maximum) or the ReLU mask; the softmax column code and the fixed-order
// loss reduction are those of softmax_step_kernel (elementwise.cu), whose
// 128-column CTAs are 4 of this kernel's column groups.
#include "async_copy.cuh"
#include "pattern.cuh"
#include "padded.cuh"
#include "tma.cuh"

#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

namespace smb {
namespace {

constexpr int kChainMaxL = 6;
constexpr int kChainWarps = 16;
constexpr int kChainThreads = 32 * kChainWarps;
constexpr int kChainMaxClasses = 16;
constexpr int kChainMaxC = 8;

// one staged sparse product (a forward layer or a transposed one)
struct ChainPhase {
  const int32_t* ptr;    // padded segment pointers [rows + 1] (multiples of 4)
  const int32_t* idx;    // padded operand rows (pads: zero_row)
  const float* val;      // padded values (pads: -0.0)
  const int32_t* order;  // [rows]: each CTA's rows, longest segment first
  const float* bias;     // forward: per-row bias, or null
  float* out;            // [rows x ld]
  int rows;              // output rows
  int nnzp;              // padded segment total
  int split[kChainMaxC + 1];  // the cluster's CTAs' row ranges (balanced by nonzeros)
  int segb[kChainMaxC + 1];   // their padded segment bounds
  int act;               // forward: np.maximum(., 0); backward: ReLU mask of the layer below
  int zero_row;          // the operand's all-zero row
  int meta_off;          // shared-memory byte offset of the staged segment
  int ptr_words;         // staged pointer words (multiple of 4)
  int nz_words;          // staged index words = value words (multiple of 4; + the no-op quad)
  int epi_off;           // forward: staged bias slice; backward: mask bits (byte offset)
  int order_off;         // staged order slice (byte offset)
  int in_map;            // tensor map that reloads the operand into region A, -1: region D
  int in_boxes;          // boxes of that reload
  int in_box_rows;
  int wide;              // long rows: one row per warp, one column per lane
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
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c, int r,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c), "r"(r), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                         unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// volatile shared loads: a batch of them stays a batch (ptxas otherwise sinks
// each load next to its first use)
__device__ __forceinline__ float lds_f32(unsigned a) {
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
__device__ __forceinline__ int4 lds_s32x4(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

enum ChainKind { kFwd = 0, kFwdLast = 1, kBwd = 2 };

// What one warp needs to run its rows of one product (shared addresses).
struct RowTask {
  const int32_t* sp;     // staged padded pointers; row r at sp[r - pr0]
  int pr0;
  int a0;                // staged padded slot s at local index s - a0
  unsigned si, sv;       // staged indices / values
  int dummy;             // local index of the no-op quad
  const int32_t* order;  // the CTA's rows, longest segment first
  int nrows;
  unsigned X;            // operand [rows][32] (+ zero row)
  const float* sbias;    // forward: staged bias, row r at sbias[r - pr0]
  const unsigned* mbits;  // backward: ReLU mask bits, row r at mbits[r - r0]
  int r0;
  int act;
  float* out;
  int64_t ld;
  int n;                 // batch width (valid columns)
  int c0;                // first column of the cluster's group
  unsigned lg;           // forward-last: shared address of the logits block
  unsigned C;
};

template <int K, int W>
__device__ __forceinline__ void epilogue(const RowTask& w, int r, int cq, float (&acc)[W]) {
  if constexpr (K == kBwd) {
    if (w.act) {
      const unsigned bits = w.mbits[r - w.r0] >> cq;
#pragma unroll
      for (int u = 0; u < W; ++u) acc[u] = mul_rn(acc[u], ((bits >> u) & 1u) ? 1.f : 0.f);
    }
  } else {
    if (w.sbias != nullptr) {
      const float b = w.sbias[r - w.pr0];
#pragma unroll
      for (int u = 0; u < W; ++u) acc[u] = add_rn(acc[u], b);
    }
    if constexpr (K == kFwd) {
      if (w.act) {
#pragma unroll
        for (int u = 0; u < W; ++u) acc[u] = relu_np(acc[u]);
      }
    }
  }
  const int col = w.c0 + cq;
  float* o = w.out + (int64_t)r * w.ld + col;
  if constexpr (W == 4) {
    if (col + 3 < w.n) {
      *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (col + u < w.n) o[u] = acc[u];
    }
  } else {
    if (col < w.n) o[0] = acc[0];
  }
  if constexpr (K == kFwdLast) {
    // the logits of the cluster's columns into every CTA's logit block
    const unsigned a = w.lg + (unsigned)(r * 32 + cq) * 4u;
    for (unsigned t = 0; t < w.C; ++t) {
      unsigned remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(a), "r"(t));
      if constexpr (W == 4) {
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote),
                     "f"(acc[0]), "f"(acc[1]), "f"(acc[2]), "f"(acc[3])
                     : "memory");
      } else {
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(acc[0]) : "memory");
      }
    }
  }
}

// The CTA's rows of one product, 4 rows per warp at a time (8-lane groups, 4
// columns per lane).  Software pipeline over quads: the indices / values of
// quad k+2 and the 4 operand rows of quad k+1 are in flight while quad k is
// summed.  A group whose row has no quads left reads the no-op quad.
template <int K>
__device__ __forceinline__ void run_rows(const RowTask& w, int warp, int lane) {
  const int g = lane >> 3, l8 = lane & 7;
  const int cq = 4 * l8;
  const unsigned xb = w.X + 4u * (unsigned)cq;
  // slot (sorted row) warp + 16 g + 64 t: a CTA with at most 16 rows gives
  // every warp its own row
  for (int base = warp; base < w.nrows; base += 4 * kChainWarps) {
    const int slot = base + kChainWarps * g;
    const bool has = slot < w.nrows;
    const int r = has ? w.order[slot] : 0;
    const int qb = has ? w.sp[r - w.pr0] - w.a0 : w.dummy;
    const int nq = has ? (w.sp[r + 1 - w.pr0] - w.a0 - qb) >> 2 : 0;
    const int trip = __reduce_max_sync(0xffffffffu, nq);
    auto qa = [&](int k) { return (unsigned)(k < nq ? qb + 4 * k : w.dummy) * 4u; };
    auto opnd = [&](const int4 c, float4 (&x)[4]) {
      x[0] = lds_f32x4(xb + (unsigned)c.x * 128u);
      x[1] = lds_f32x4(xb + (unsigned)c.y * 128u);
      x[2] = lds_f32x4(xb + (unsigned)c.z * 128u);
      x[3] = lds_f32x4(xb + (unsigned)c.w * 128u);
    };
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    int4 c1 = lds_s32x4(w.si + qa(1));
    float4 v0 = lds_f32x4(w.sv + qa(0)), v1 = lds_f32x4(w.sv + qa(1));
    float4 x0[4];
    opnd(lds_s32x4(w.si + qa(0)), x0);
    for (int k = 0; k < trip; ++k) {
      float4 x1[4];
      opnd(c1, x1);
      const int4 c2 = lds_s32x4(w.si + qa(k + 2));
      const float4 v2 = lds_f32x4(w.sv + qa(k + 2));
      const float vv[4] = {v0.x, v0.y, v0.z, v0.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[0] = add_rn(acc[0], mul_rn(vv[u], x0[u].x));
        acc[1] = add_rn(acc[1], mul_rn(vv[u], x0[u].y));
        acc[2] = add_rn(acc[2], mul_rn(vv[u], x0[u].z));
        acc[3] = add_rn(acc[3], mul_rn(vv[u], x0[u].w));
      }
      v0 = v1;
      v1 = v2;
      c1 = c2;
#pragma unroll
      for (int u = 0; u < 4; ++u) x0[u] = x1[u];
    }
    if (has) epilogue<K, 4>(w, r, cq, acc);
  }
}

// Long rows (the output layer's ~300-nonzero rows at config 2): one row per
// warp, one column per lane, ~5 instructions per element.
template <int K>
__device__ __forceinline__ void run_rows_wide(const RowTask& w, int warp, int lane) {
  const unsigned xl = w.X + 4u * (unsigned)lane;
  for (int slot = warp; slot < w.nrows; slot += kChainWarps) {
    const int r = w.order[slot];
    const int qb = w.sp[r - w.pr0] - w.a0;
    const int nq = (w.sp[r + 1 - w.pr0] - w.a0 - qb) >> 2;
    auto qa = [&](int k) { return (unsigned)(k < nq ? qb + 4 * k : w.dummy) * 4u; };
    auto opnd = [&](const int4 c) {
      return make_float4(lds_f32(xl + (unsigned)c.x * 128u), lds_f32(xl + (unsigned)c.y * 128u),
                         lds_f32(xl + (unsigned)c.z * 128u), lds_f32(xl + (unsigned)c.w * 128u));
    };
    float acc[1] = {0.f};
    int4 c1 = lds_s32x4(w.si + qa(1));
    float4 v0 = lds_f32x4(w.sv + qa(0)), v1 = lds_f32x4(w.sv + qa(1));
    float4 x0 = opnd(lds_s32x4(w.si + qa(0)));
    for (int k = 0; k < nq; ++k) {
      const float4 x1 = opnd(c1);
      const int4 c2 = lds_s32x4(w.si + qa(k + 2));
      const float4 v2 = lds_f32x4(w.sv + qa(k + 2));
      acc[0] = add_rn(acc[0], mul_rn(v0.x, x0.x));
      acc[0] = add_rn(acc[0], mul_rn(v0.y, x0.y));
      acc[0] = add_rn(acc[0], mul_rn(v0.z, x0.z));
      acc[0] = add_rn(acc[0], mul_rn(v0.w, x0.w));
      v0 = v1;
      v1 = v2;
      x0 = x1;
      c1 = c2;
    }
    epilogue<K, 1>(w, r, lane, acc);
  }
}

template <int L>
__global__ void __launch_bounds__(kChainThreads, 1) chain_kernel(const __grid_constant__ ChainParams P) {
  constexpr int NF = L - 1, NPH = 2 * (L - 1);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long s_bar[NPH + 1];  // + the staging barrier
  __shared__ int s_bnd[NPH][2];
  // the phase descriptors in shared memory (indexed loads of the 3 KB
  // parameter block miss the constant cache)
  __shared__ __align__(16) ChainPhase s_ph[NPH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  static_assert(sizeof(ChainPhase) % 4 == 0, "phase descriptor words");
  static_assert(NPH < kChainWarps, "one warp per phase descriptor");
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
  float* E = LG + kChainMaxClasses * 32;  // exp(z) per class
  float* S = E + kChainMaxClasses * 32;   // s per column
  float* TT = S + 32;                     // targets
  const unsigned bar0 = smem_u32(&s_bar[0]);
  const unsigned stage_bar = bar0 + 8 * NPH;

  unsigned long long* prof = P.prof ? P.prof + (size_t)blockIdx.x * 32 : nullptr;
  int nprof = 0;
  auto stamp = [&]() {
    if (prof != nullptr && tid == 0) {
      // SM cycles (globaltimer ticks too coarsely for sub-microsecond phases)
      prof[nprof] = clock64();
    }
    ++nprof;
  };
  stamp();
  // the targets of the softmax columns (older than the previous kernel), one
  // class per warp: issued first, stored to shared memory further down
  const float t_col = (warp < P.classes && ok) ? P.t[warp * P.ld_t + col] : 0.f;
  if (tid == 0) {
#pragma unroll
    for (int p = 0; p < NPH; ++p) mbar_init(bar0 + 8 * p, 1);
    mbar_init(stage_bar, NPH);  // one arrival per phase's staging thread
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // barriers initialised
  // the operand of the first product (the first layer's output, the previous
  // kernel's): its tensor copies go out first, so they overlap the staging
  // below (one thread waits for the previous grid; every other thread's
  // wait comes after the staging)
  auto issue_operand = [&](const ChainPhase& f, int p) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const unsigned bar = bar0 + 8 * p;
    mbar_expect_tx(bar, (unsigned)(f.in_boxes * f.in_box_rows * 128));
    for (int b = 0; b < f.in_boxes; ++b)
      tma_load_2d(smem_u32(A) + (unsigned)(b * f.in_box_rows * 128), &P.maps[f.in_map], c0,
                  b * f.in_box_rows, bar);
  };
  if (warp == kChainWarps - 1 && lane == 0 && P.ph[0].in_map >= 0) {
    pdl_wait();
    issue_operand(P.ph[0], 0);
  }
  // The descriptors (lane-parallel copy of the parameters: indexed loads of
  // the 3 KB parameter block miss the constant cache, so each field is read
  // once, by one lane).  Then stage every phase's padded pointers / indices /
  // values, row order and bias slice for this CTA's rows with 1-D bulk
  // copies: lane 0 of warp p issues phase p's from the shared copy (read
  // from the parameters by lane 0 alone this took 1.3 us, 0.6 now); a
  // pointer / order / bias slice is rounded up to 16-byte chunks where the
  // array allows, its last < 4 words otherwise copied by plain loads.  Static
  // data and values older than the previous kernel: before the
  // programmatic-dependency wait.
  if (warp < NPH) {
    constexpr int kW = (int)sizeof(ChainPhase) / 4;
    const int* src = reinterpret_cast<const int*>(&P.ph[warp]);
    int* dst = reinterpret_cast<int*>(&s_ph[warp]);
    for (int k = lane; k < kW; k += 32) dst[k] = src[k];
    __syncwarp();
  }
  if (warp < NPH && lane == 0) {
    const int p = warp;
    const ChainPhase& f = s_ph[p];
    const int r0 = f.split[q], r1 = f.split[q + 1];
    const int pr0 = r0 & ~3;
    const int a0 = f.segb[q], a1 = f.segb[q + 1];
    s_bnd[p][0] = a0;
    s_bnd[p][1] = a1;
    int32_t* sp = reinterpret_cast<int32_t*>(base + f.meta_off);
    int32_t* si = sp + f.ptr_words;
    float* sv = reinterpret_cast<float*>(si + f.nz_words);
    unsigned bytes = 0;
    auto seg = [&](void* dst, const void* src, int words, int avail) {
      const int up = (words + 3) & ~3;
      const int body = up <= avail ? up : (words & ~3);
      if (body > 0) {
        bulk_g2s(smem_u32(dst), src, 4u * (unsigned)body, stage_bar);
        bytes += 4u * (unsigned)body;
      }
      for (int k = body; k < words; ++k)
        static_cast<int32_t*>(dst)[k] = static_cast<const int32_t*>(src)[k];
    };
    seg(sp, f.ptr + pr0, r1 + 1 - pr0, f.rows + 1 - pr0);
    seg(si, f.idx + a0, a1 - a0, f.nnzp - a0);
    seg(sv, f.val + a0, a1 - a0, f.nnzp - a0);
    seg(base + f.order_off, f.order + pr0, r1 - pr0, ((f.rows + 3) & ~3) - pr0);
    if (p < NF && f.bias != nullptr) seg(base + f.epi_off, f.bias + pr0, r1 - pr0, f.rows - pr0);
    // the no-op quad after the segment: the zero row, -0.0
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      si[a1 - a0 + k] = f.zero_row;
      sv[a1 - a0 + k] = -0.f;
    }
    mbar_expect_tx(stage_bar, bytes);
  }
  // the targets (loaded above); the zero row of the first transposed
  // product's operand
  if (warp < P.classes) TT[warp * 32 + lane] = t_col;
  if (warp == kChainWarps - 1) D[P.classes * 32 + lane] = 0.f;
  stamp();

  auto reload = [&](int p) {
    if (tid == 0 && s_ph[p].in_map >= 0) issue_operand(s_ph[p], p);
  };
  pdl_wait();  // (global writes below may overwrite what the previous kernel read)
  mbar_wait(stage_bar, 0);
  __syncthreads();  // staged segments (and their plain-copied parts) visible
  stamp();

  double loss_local = 0.0;
#pragma unroll
  for (int p = 0; p < NPH; ++p) {
    const ChainPhase& f = s_ph[p];
    if (p == NF) {
      // softmax cross-entropy gradient of the cluster's 32 columns from the
      // logits every CTA received (so the first transposed product needs no
      // exchange), parallel over classes: warp c computes e_c = exp(z_c),
      // warp 0 sums s and z.t in class order (the loss term), warp c forms
      // d_c = (e_c / s - t_c) / divisor; the rank-0 CTA writes d_{L-1}
      const int classes = P.classes;
      if (warp < classes) {
        float mx = LG[lane];
        for (int c = 1; c < classes; ++c) {
          const float v = LG[c * 32 + lane];
          mx = (v > mx || v != v) ? v : mx;
        }
        E[warp * 32 + lane] = exp_full(sub_rn(LG[warp * 32 + lane], mx));
      }
      __syncthreads();
      if (warp == 0) {
        float mx = LG[lane];
        for (int c = 1; c < classes; ++c) {
          const float v = LG[c * 32 + lane];
          mx = (v > mx || v != v) ? v : mx;
        }
        float sum = 0.f, zt = 0.f;
        for (int c = 0; c < classes; ++c) {
          sum = add_rn(sum, E[c * 32 + lane]);
          zt = add_rn(zt, mul_rn(sub_rn(LG[c * 32 + lane], mx), TT[c * 32 + lane]));
        }
        S[lane] = sum;
        loss_local = ok ? static_cast<double>(sub_rn(log_full(sum), zt)) : 0.0;
      }
      __syncthreads();
      if (warp < classes) {
        const float g =
            div_rn(sub_rn(div_rn(E[warp * 32 + lane], S[lane]), TT[warp * 32 + lane]), P.divisor);
        D[warp * 32 + lane] = ok ? g : 0.f;
        if (q == 0 && ok) P.dy_top[warp * P.ld + col] = g;
      }
      __syncthreads();
      stamp();
    }
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
        const unsigned ab = smem_u32(A) + 4u * (unsigned)lane;
        for (int r = b0 + warp; r < b1; r += 4 * kChainWarps) {
          float a[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            a[u] = lds_f32(ab + 128u * (unsigned)min(r + u * kChainWarps, b1 - 1));
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned bits = __ballot_sync(0xffffffffu, a[u] > 0.f);
            if (lane == 0 && r + u * kChainWarps < b1) mb[r + u * kChainWarps - b0] = bits;
          }
        }
      }
    }
    stamp();
    RowTask w;
    w.sp = reinterpret_cast<const int32_t*>(base + f.meta_off);
    w.pr0 = r0 & ~3;
    w.a0 = s_bnd[p][0];
    w.si = smem_u32(w.sp + f.ptr_words);
    w.sv = w.si + 4u * (unsigned)f.nz_words;
    w.dummy = s_bnd[p][1] - s_bnd[p][0];
    w.order = reinterpret_cast<const int32_t*>(base + f.order_off) + (r0 - (r0 & ~3));
    w.nrows = r1 - r0;
    w.X = p == NF ? smem_u32(D) : smem_u32(A);
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

__global__ void padded_refresh_kernel(const int32_t* __restrict__ src,
                                      const float* __restrict__ values, float* __restrict__ pval,
                                      int64_t n) {
  pdl_wait();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = src[s];
    pval[s] = k >= 0 ? values[k] : -0.f;
  }
  pdl_trigger();
}
}  // namespace smb

struct smb_chain_plan {
  int L = 0, C = 1, ngroups = 0;
  int64_t n = 0, ld = 0;
  int classes = 0;
  size_t smem = 0;
  smb::ChainParams proto;        // everything but the per-step pointers and maps
  std::vector<int64_t> rows;     // m of every layer
  std::vector<int> relu;         // activation after every layer
  std::vector<int64_t> src_off;  // per layer: [fwd | bwd] padded slots in src / pval
  std::vector<int64_t> src_len;
  void* dev = nullptr;           // owned: pointers, indices, orders, src maps, values
  int32_t* src = nullptr;
  float* pval = nullptr;
  ~smb_chain_plan() {
    if (dev) cudaFree(dev);
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
                    patterns[l]->nnz < (1ll << 29),
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
  cudaDeviceSynchronize();  // setup: host copies of the structure
  ChainParams& P = plan->proto;
  memset(&P, 0, sizeof(P));
  // padded products: forward phase l-1 (CSR of layer l), backward phase
  // 2L-2-l (CSC of layer l)
  std::vector<Padded> pads(2 * (L - 1));
  bool okc = true;
  for (int l = 1; l < L && okc; ++l) {
    const smb_pattern* pat = patterns[l];
    std::vector<int32_t> rp, ci, cp, ri, pm;
    okc = to_host(rp, pat->row_ptr, pat->m + 1) && to_host(ci, pat->col_idx, pat->nnz) &&
          to_host(cp, pat->col_ptr, pat->k + 1) && to_host(ri, pat->row_idx, pat->nnz) &&
          to_host(pm, pat->perm, pat->nnz);
    if (!okc) break;
    pads[l - 1] = pad_segments(rp, ci, nullptr, (int)pat->k);
    pads[2 * L - 2 - l] = pad_segments(cp, ri, pm.data(), (int)pat->m);
  }
  if (!okc) {
    delete plan;
    set_error("chain: reading the pattern structure failed");
    return SMB_ERR_CUDA;
  }
  // one device block: per phase ptr | idx | order (int32, 16-byte aligned
  // pieces), then per layer the src map, then the padded values
  std::vector<int32_t> blob;
  auto put = [&](const std::vector<int32_t>& v) {
    const size_t at = blob.size();
    blob.insert(blob.end(), v.begin(), v.end());
    while (blob.size() % 4) blob.push_back(0);
    return at;
  };
  std::vector<size_t> at_ptr(2 * (L - 1)), at_idx(2 * (L - 1)), at_order(2 * (L - 1));
  size_t off = 0;
  int max_in_rows = 0;
  for (int p = 0; p < 2 * (L - 1); ++p) {
    ChainPhase& f = P.ph[p];
    const bool fwd = p < L - 1;
    const int l = fwd ? p + 1 : 2 * L - 2 - p;
    const smb_pattern* pat = patterns[l];
    Padded& pd = pads[p];
    const int rows = (int)pd.ptr.size() - 1;
    const int in_rows = (int)(fwd ? pat->k : pat->m);
    // the CTAs' row ranges, balanced by (padded) nonzeros
    const int64_t z = pd.ptr[rows];
    f.split[0] = 0;
    for (int q = 1; q < C; ++q) {
      const int64_t target = z * q / C;
      const int r = (int)(std::lower_bound(pd.ptr.begin(), pd.ptr.end(), (int32_t)target) -
                          pd.ptr.begin());
      f.split[q] = std::max(f.split[q - 1], std::min(r, rows));
    }
    f.split[C] = rows;
    for (int q = 0; q <= C; ++q) f.segb[q] = pd.ptr[f.split[q]];
    // each CTA's rows, longest segment first
    for (int q = 0; q < C; ++q) {
      std::vector<int32_t> rr;
      for (int r = f.split[q]; r < f.split[q + 1]; ++r) rr.push_back(r);
      std::stable_sort(rr.begin(), rr.end(), [&](int32_t a, int32_t b) {
        return pd.ptr[a + 1] - pd.ptr[a] > pd.ptr[b + 1] - pd.ptr[b];
      });
      pd.order.insert(pd.order.end(), rr.begin(), rr.end());
    }
    int pw = 0, nw = 0, ew = 0, ow = 0;
    for (int q = 0; q < C; ++q) {
      const int r0 = f.split[q], r1 = f.split[q + 1], pr0 = r0 & ~3;
      pw = std::max(pw, ((r1 + 1 - pr0) + 3) & ~3);
      nw = std::max(nw, pd.ptr[r1] - pd.ptr[r0] + 4);  // + the no-op quad
      // forward: the bias slice from pr0; backward: one mask word per row
      ew = std::max(ew, fwd ? (((r1 - pr0) + 3) & ~3) : (((r1 - r0) + 3) & ~3));
      ow = std::max(ow, ((r1 - pr0) + 3) & ~3);
    }
    f.rows = rows;
    f.nnzp = (int)z;
    f.act = fwd ? (relu[l] != 0) : (relu[l - 1] != 0);
    f.zero_row = in_rows;
    f.wide = rows > 0 && z >= (int64_t)48 * rows;  // long rows: one per warp
    f.meta_off = (int)off;
    f.ptr_words = pw;
    f.nz_words = nw;
    off += (size_t)4 * (pw + 2 * (size_t)nw);
    f.epi_off = (int)off;
    off += (size_t)4 * ew;
    f.order_off = (int)off;
    off += (size_t)4 * ow;
    // operand reload: boxes of <= 256 rows covering the rows AND the zero
    // row after them (out-of-bounds rows of a box are zero-filled)
    f.in_map = fwd ? l - 1 : (p == L - 1 ? -1 : (L - 1) + (l - 1));
    const int need = in_rows + 1;
    f.in_boxes = (int)ceil_div(need, 256);
    f.in_box_rows = (int)ceil_div(need, f.in_boxes);
    if (f.in_map >= 0) max_in_rows = std::max(max_in_rows, f.in_boxes * f.in_box_rows);
    at_ptr[p] = put(pd.ptr);
    at_idx[p] = put(pd.idx);
    at_order[p] = put(pd.order);
  }
  // per layer: the src map of [forward | backward] padded slots
  plan->src_off.assign(L, 0);
  plan->src_len.assign(L, 0);
  const size_t src_at = blob.size();
  std::vector<size_t> at_pval_f(L, 0), at_pval_b(L, 0);
  size_t src_words = 0;
  for (int l = 1; l < L; ++l) {
    const Padded& pf = pads[l - 1];
    const Padded& pb = pads[2 * L - 2 - l];
    plan->src_off[l] = (int64_t)src_words;
    at_pval_f[l] = src_words;
    blob.insert(blob.end(), pf.src.begin(), pf.src.end());
    src_words += pf.src.size();
    while (src_words % 4) {
      blob.push_back(-1);
      ++src_words;
    }
    at_pval_b[l] = src_words;
    blob.insert(blob.end(), pb.src.begin(), pb.src.end());
    src_words += pb.src.size();
    while (src_words % 4) {
      blob.push_back(-1);
      ++src_words;
    }
    plan->src_len[l] = (int64_t)src_words - plan->src_off[l];
  }
  const size_t total_words = blob.size() + src_words;  // + the padded values
  if (cudaMalloc(&plan->dev, 4 * std::max<size_t>(total_words, 4)) != cudaSuccess ||
      cudaMemcpy(plan->dev, blob.data(), 4 * blob.size(), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    delete plan;
    set_error("chain: allocating the padded structure failed");
    return SMB_ERR_CUDA;
  }
  int32_t* d = static_cast<int32_t*>(plan->dev);
  plan->src = d + src_at;
  plan->pval = reinterpret_cast<float*>(d + blob.size());
  for (int p = 0; p < 2 * (L - 1); ++p) {
    ChainPhase& f = P.ph[p];
    const bool fwd = p < L - 1;
    const int l = fwd ? p + 1 : 2 * L - 2 - p;
    f.ptr = d + at_ptr[p];
    f.idx = d + at_idx[p];
    f.order = d + at_order[p];
    f.val = plan->pval + (fwd ? at_pval_f[l] : at_pval_b[l]);
  }
  off = (off + 1023) & ~size_t(1023);
  P.off_A = (int)off;
  off += (size_t)max_in_rows * 128;
  P.off_D = (int)off;
  off += (size_t)(kChainMaxClasses + 1) * 128;  // + the zero row
  P.off_LG = (int)off;                          // logits, exp(z), s, targets
  off += (size_t)(3 * kChainMaxClasses + 1) * 128;
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

extern "C" int smb_chain_refresh(const smb_chain_plan* plan, int layer, const void* values,
                                 void* stream) {
  using namespace smb;
  clear_error();
  SMB_REQUIRE(plan != nullptr && values != nullptr, "smb_chain_refresh: null argument");
  SMB_REQUIRE(layer >= 1 && layer < plan->L, "smb_chain_refresh: layer %d out of 1..%d", layer,
              plan->L - 1);
  const int64_t nslots = plan->src_len[layer];
  if (nslots == 0) return SMB_OK;
  const int64_t o = plan->src_off[layer];
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(nslots, 256), 4 * 148);
  launch_k(padded_refresh_kernel, dim3(grid), dim3(256), 0, as_stream(stream), plan->src + o,
           static_cast<const float*>(values), plan->pval + o, nslots);
  return check_launch("smb_chain_refresh");
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

extern "C" int smb_chain_run(const smb_chain_plan* plan, const void* const* bias,
                             void* const* acts, void* const* dys, const void* t, int64_t ld_t,
                             double divisor, double* loss_out, void* workspace, void* stream) {
  using namespace smb;
  clear_error();
  SMB_REQUIRE(plan != nullptr && bias != nullptr && acts != nullptr && dys != nullptr &&
                  t != nullptr,
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
      SMB_REQUIRE(bias[l] == nullptr || aligned16(bias[l]),
                  "smb_chain_run: bias buffers must be 16-byte aligned");
  }
  ChainParams P = plan->proto;
  for (int l = 1; l < L; ++l) {
    ChainPhase& f = P.ph[l - 1];
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
