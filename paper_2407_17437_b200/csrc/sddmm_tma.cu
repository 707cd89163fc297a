// SDDMM + update with TMA row gathers (sm_100a).
//
// The same per-chain arithmetic as sddmm.cu (grad[p] = sum_t d_out[i,t] *
// x[j,t], one sequential chain per nonzero, multiply and add rounded
// separately, _kernels.py:62-75; then the sparse_combine update sequence of
// nn.py:187-197), with the staging done by the Tensor Memory Accelerator
// instead of per-thread cp.async:
//
//   * one warp per CTA owns 32 consecutive nonzeros (CSR order, or the
//     pattern's L2-blocked order) and a private ring of 2 stages; a stage holds
//     the 32 gathered x-row segments of one 32-column batch chunk plus the
//     (up to DS) d_out rows the warp's nonzeros span;
//   * 9 lanes fill a stage with ONE `cp.async.bulk.tensor.2d.tile::gather4`
//     each (4 arbitrary rows x 128 bytes per instruction, SASS
//     UTMALDG.2D.GATHER4) and the stage's mbarrier counts the bytes in
//     (complete_tx); the other lanes issue no copy instructions at all, so the
//     MIO queue that throttled the LDGSTS version (ncu: mio_throttle the top
//     stall at config 4) only carries the chains' shared-memory reads;
//   * the tensor maps use the 128-byte swizzle: 16-byte chunk u of staged row
//     r sits at chunk u ^ (r mod 8), so the 8 lanes of a quarter-warp reading
//     chunk u of their own rows hit 8 different bank groups (conflict-free
//     without padding, unlike the 144-byte padded rows of cp.async staging
//     that split sectors on the global side).
//
// The kernel is bound by instruction issue and by how many warps (rings) an
// SM holds, so both were trimmed (config-4 hidden layer, graph-timed):
//   215 us  first version: one chunk loop with `staged` tested inside (ptxas
//           predicated the fallback's 32 global d_out loads into the staged
//           path: issue slots spent on masked-off instructions), one copy site
//           choosing its tensor map per lane;
//   178 us  the chunk loop instantiated per staging mode, one copy site per
//           tensor map (uniform map operand);
//   161 us  the chunk loop unrolled over the ring stages (every shared-memory
//           address a register plus an immediate);
//   149 us  no static shared memory and no alignment slack: 9.4 KB per CTA,
//           21 resident warps per SM instead of 18.
// The copy issue is still ~90 of the ~200 instructions per chunk: the gather4
// row coordinates are data (col_idx), so ptxas moves them into uniform
// registers through an ELECT / R2UR.BROADCAST loop, ~10 issue slots per copy
// (a single elected lane holding every coordinate needs as many: the R2URs
// and the UMOVs that line up the operand registers).  Measured and dropped:
// two chains per lane sharing each staged d_out chunk (K = 2: half the warps
// per SM, 221 us), 8 staged d_out rows (DS = 8: 162 us), 3 stages (204 us),
// 2-4 warps per CTA.
//
// Valid for fp32 with 16-byte aligned operands and leading dimensions
// (sddmm_tma_supported); the caller falls back to sddmm.cu otherwise.
#include <cuda.h>

#include <type_traits>

#include "pattern.cuh"
#include "tma.cuh"

namespace smb {
namespace {

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
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
// 4 rows (r0..r3) x 32 fp32 columns starting at column c of a 2-D tensor map
__device__ __forceinline__ void tma_gather4(unsigned dst, const CUtensorMap* map, int c, int r0,
                                            int r1, int r2, int r3, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

// K chains per lane (K = 1, 2): lane l owns the K consecutive nonzeros
// K*l .. K*l+K-1 of the warp's 32*K, which mostly lie in one row of the
// pattern, so the lane reads each staged d_out chunk once for all of them
// (per pair: 4 bytes of x written by the TMA + 4 read + 4/K of d_out read from
// shared memory, the resource the one-chain kernel saturates together with
// the issue slots).  Nonzero K*l+e is staged at shared-memory row 32*e + l:
// every quarter-warp still reads 8 consecutive 128-byte rows, conflict-free
// under the 128-byte swizzle.  The chunk loop is unrolled over the S ring
// stages, so every shared-memory address is a register plus an immediate.
template <int S, bool ORD, int K, int DS>
__global__ void __launch_bounds__(32)
    sddmm_tmak_kernel(const __grid_constant__ CUtensorMap xmap,
                      const __grid_constant__ CUtensorMap dmap,
                      const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                      const int32_t* __restrict__ tile_row0, const int32_t* __restrict__ ord_p,
                      const int32_t* __restrict__ ord_row, int64_t m, int64_t nnz,
                      const float* __restrict__ d_out, int64_t ld_d, int n, const float* values,
                      float* values_out, float* velocity, float* grad_out, OptConsts<float> opt,
                      int tb, int te, float* acc_io) {
  // This launch sums the batch columns [tb, te) of every chain (a phase);
  // phases run in column order, the partial sums carried in acc_io (indexed
  // like the values) between them, so each chain's order over the batch is
  // unchanged.  tb == 0 starts the chains, te == n finishes them (update).
  constexpr int kTile = 32 * K;
  constexpr int kXBytes = kTile * 128;
  constexpr int kDBytes = DS * 128;
  static_assert(kTile % kTileGrain == 0 && DS % 4 == 0 && DS <= 8 && 4 * K + DS / 4 <= 32, "");
  // No static shared memory: the dynamic block then starts at the CTA's
  // 1024-byte aligned window base (checked), so the ring needs no alignment
  // slack and the barriers / row window live behind it -- 9.5 KB per CTA at
  // K = 1, 21 resident warps per SM instead of 18.
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int kRing = S * (kXBytes + kDBytes);
  unsigned long long* s_full = reinterpret_cast<unsigned long long*>(smem_raw + kRing);
  int64_t* s_slot_row = reinterpret_cast<int64_t*>(smem_raw + kRing + 8 * S);
  int32_t* s_rp = reinterpret_cast<int32_t*>(smem_raw + kRing + 8 * S + 8 * DS);
  const int lane = threadIdx.x;
  const unsigned base = smem_addr(smem_raw);  // x blocks, then d blocks
  if (base & 1023u) __trap();
  const unsigned dbase = base + S * kXBytes;
  const unsigned char* gbase = smem_raw;
  const unsigned bar0 = smem_addr(s_full);
  const int64_t pw = (int64_t)blockIdx.x * kTile;
  const int nw = (int)imax(0, imin(kTile, nnz - pw));
  bool act[K];
  int64_t p[K];
  int32_t col[K];
#pragma unroll
  for (int e = 0; e < K; ++e) {
    act[e] = K * lane + e < nw;
    p[e] = ORD ? (act[e] ? (int64_t)ord_p[pw + K * lane + e] : 0) : pw + K * lane + e;
  }
  int32_t r0 = 0;
  if constexpr (!ORD) {
    r0 = tile_row0[(int64_t)blockIdx.x * (kTile / kTileGrain)];
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const int i = lane + 32 * e;
      s_rp[i] = (r0 + i <= m) ? row_ptr[r0 + i] : INT32_MAX;
    }
    if (lane == 0) s_rp[kTile] = (r0 + kTile <= m) ? row_ptr[r0 + kTile] : INT32_MAX;
  }
#pragma unroll
  for (int e = 0; e < K; ++e) col[e] = act[e] ? col_idx[p[e]] : 0;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (nw == 0) return;
  int64_t row[K];
  int slot[K];
  int n_slots;
  int64_t slot_row[DS];
  if constexpr (ORD) {
    // d_out slots = runs of equal rows in the warp's nonzero order
    bool head[K];
    unsigned heads[K];
#pragma unroll
    for (int e = 0; e < K; ++e)
      row[e] = act[e] ? (int64_t)ord_row[pw + K * lane + e] : (int64_t)ord_row[pw];
    const int64_t prev_lane = __shfl_up_sync(0xffffffffu, row[K - 1], 1);
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const int64_t prev = e == 0 ? prev_lane : row[e - 1];
      head[e] = act[e] && ((lane == 0 && e == 0) || row[e] != prev);
      heads[e] = __ballot_sync(0xffffffffu, head[e]);
    }
    // runs started before this lane, then inside it
    int before = 0;
    n_slots = 0;
#pragma unroll
    for (int e = 0; e < K; ++e) {
      before += __popc(heads[e] & ((1u << lane) - 1u));
      n_slots += __popc(heads[e]);
    }
#pragma unroll
    for (int e = 0; e < K; ++e) {
      before += head[e] ? 1 : 0;
      slot[e] = before - 1;
    }
    if (lane < DS) s_slot_row[lane] = row[0];  // filler: any valid row
    __syncwarp();
#pragma unroll
    for (int e = 0; e < K; ++e)
      if (head[e] && slot[e] < DS) s_slot_row[slot[e]] = row[e];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < DS; ++q) slot_row[q] = s_slot_row[q];
  } else {
#pragma unroll
    for (int e = 0; e < K; ++e)
      row[e] = tile_row_of<kTile>(act[e] ? p[e] : pw, r0, s_rp, row_ptr, m);
    const int64_t row_first = __shfl_sync(0xffffffffu, row[0], 0);
    int64_t row_last = row_first;
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const int64_t r = __shfl_sync(0xffffffffu, row[e], (nw - 1) / K);
      if ((nw - 1) % K == e) row_last = r;
    }
    n_slots = (int)(row_last - row_first + 1);
#pragma unroll
    for (int e = 0; e < K; ++e) slot[e] = (int)(row[e] - row_first);
#pragma unroll
    for (int q = 0; q < DS; ++q) slot_row[q] = imin(row_first + imin(q, n_slots - 1), m - 1);
  }
  const bool staged = n_slots <= DS;  // warp-uniform
  const int n_chunks = (te - tb + 31) / 32;
  // copy roles: lane g < 8K gathers the shared-memory rows 4g..4g+3 (nonzero
  // K*l+e sits at row 32e + l), lanes 8K.. the staged d_out rows
  int gr[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int src = 4 * (lane & 7) + q;
    int v = 0;
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const int c = __shfl_sync(0xffffffffu, col[e], src);
      if ((lane >> 3) == e) v = c;
    }
    gr[q] = v;
  }
#pragma unroll
  for (int g = 0; g < DS / 4; ++g)
    if (lane == 8 * K + g) {
#pragma unroll
      for (int q = 0; q < 4; ++q) gr[q] = (int)slot_row[4 * g + q];
    }
  const bool dcopier = staged && lane >= 8 * K && lane < 8 * K + DS / 4;
  const unsigned tx_bytes = kXBytes + (staged ? kDBytes : 0);
  pdl_wait();  // d_out / x are earlier kernels' outputs
  const bool has_opt = opt.kind != SMB_OPT_NONE;
  float w_pre[K], v_pre[K], acc[K];
#pragma unroll
  for (int e = 0; e < K; ++e) {
    const bool upd = act[e] && has_opt && te >= n;
    w_pre[e] = upd ? values[p[e]] : 0.f;
    v_pre[e] = (upd && velocity) ? velocity[p[e]] : 0.f;
    // -0.0f: exact additive identity (sddmm.cu)
    acc[e] = (tb > 0 && act[e]) ? acc_io[p[e]] : -0.0f;
  }
  auto issue = [&](int ch, int s) {
    const unsigned bar = bar0 + 8 * s;
    if (lane == 0) mbar_arrive_expect_tx(bar, tx_bytes);
    __syncwarp();
    if (lane < 8 * K)
      tma_gather4(base + (unsigned)(s * kXBytes + lane * 512), &xmap, tb + ch * 32, gr[0], gr[1],
                  gr[2], gr[3], bar);
    else if (dcopier)
      tma_gather4(dbase + (unsigned)(s * kDBytes + (lane - 8 * K) * 512), &dmap, tb + ch * 32,
                  gr[0], gr[1], gr[2], gr[3], bar);
  };
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (s < n_chunks) issue(s, s);
  const int xsw = lane & 7;  // swizzle of this lane's x rows (row 32e + l, 1024-aligned blocks)
  const unsigned char* xl = gbase + lane * 128;
  // kSame (warp-uniform): every lane's K nonzeros lie in one row, so the lane
  // reads one d_out chunk for all of them with no per-lane test
  auto run = [&](auto staged_c, auto same_c) {
    constexpr bool kStaged = decltype(staged_c)::value;
    constexpr bool kSame = decltype(same_c)::value;
    // staged d_out rows: row `slot` of the stage's d block; the block starts
    // at a multiple of DS rows, so the swizzle of a row (address bits 7-9) is
    // slot ^ (s * DS mod 8) for slot < DS.  Unstaged: the rows in global memory
    auto dst_sw = [](int s) { return (s * DS) & 7; };
    const unsigned char* dl[K];
    const float* drow[K];
    int dsw[K];
#pragma unroll
    for (int e = 0; e < K; ++e) {
      dl[e] = gbase + S * kXBytes + (kStaged ? slot[e] : 0) * 128;
      dsw[e] = slot[e] & 7;
      drow[e] = d_out + row[e] * ld_d;
    }
    for (int ch0 = 0; ch0 < n_chunks; ch0 += S) {
      const unsigned parity = (unsigned)((ch0 / S) & 1);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int ch = ch0 + s;
        if (ch >= n_chunks) break;
        mbar_wait(bar0 + 8 * s, parity);
        const int t0 = tb + ch * 32;
        const int cnt = min(32, te - t0);
        if (cnt == 32) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            float4 xv[K], dv[K];
#pragma unroll
            for (int e = 0; e < K; ++e) {
              xv[e] = *reinterpret_cast<const float4*>(xl + s * kXBytes + e * 4096 +
                                                       16 * (u ^ xsw));
              if constexpr (kStaged) {
                if (e == 0 || (!kSame && slot[e] != slot[e - 1]))
                  dv[e] = *reinterpret_cast<const float4*>(dl[e] + s * kDBytes +
                                                           16 * (u ^ dsw[e] ^ dst_sw(s)));
                else
                  dv[e] = dv[e - 1];
              } else {
                // 16-byte aligned: sddmm_tma_supported
                dv[e] = *reinterpret_cast<const float4*>(drow[e] + t0 + 4 * u);
              }
            }
#pragma unroll
            for (int e = 0; e < K; ++e) {
              acc[e] = add_rn(acc[e], mul_rn(dv[e].x, xv[e].x));
              acc[e] = add_rn(acc[e], mul_rn(dv[e].y, xv[e].y));
              acc[e] = add_rn(acc[e], mul_rn(dv[e].z, xv[e].z));
              acc[e] = add_rn(acc[e], mul_rn(dv[e].w, xv[e].w));
            }
          }
        } else {
          for (int j = 0; j < cnt; ++j) {
            const int u = j >> 2, q = j & 3;
#pragma unroll
            for (int e = 0; e < K; ++e) {
              const float xv = reinterpret_cast<const float*>(xl + s * kXBytes + e * 4096 +
                                                              16 * (u ^ xsw))[q];
              const float dv =
                  kStaged ? reinterpret_cast<const float*>(dl[e] + s * kDBytes +
                                                           16 * (u ^ dsw[e] ^ dst_sw(s)))[q]
                          : drow[e][t0 + j];
              acc[e] = add_rn(acc[e], mul_rn(dv, xv));
            }
          }
        }
        __syncwarp();  // every lane has read stage s: refill it
        if (ch + S < n_chunks) issue(ch + S, s);
      }
    }
  };
  bool same = true;
#pragma unroll
  for (int e = 1; e < K; ++e) same = same && slot[e] == slot[0];
  same = K > 1 && __all_sync(0xffffffffu, same);
  if (!staged)
    run(std::false_type{}, std::false_type{});
  else if (same)
    run(std::true_type{}, std::true_type{});
  else
    run(std::true_type{}, std::false_type{});
  pdl_trigger();
#pragma unroll
  for (int e = 0; e < K; ++e) {
    if (!act[e]) continue;
    if (te < n) {  // more phases follow
      acc_io[p[e]] = acc[e];
      continue;
    }
    const float g = (n == 0) ? 0.f : acc[e];  // tensor_core.py:283-284: zero batch -> zeros
    if (grad_out) grad_out[p[e]] = g;
    if (has_opt) {
      apply_update(opt, g, &w_pre[e], &v_pre[e]);
      values_out[p[e]] = w_pre[e];
      if (velocity) velocity[p[e]] = v_pre[e];
    }
  }
}

// rows x cols fp32 row-major with leading dimension ld; box = 1 row x 32 cols
bool make_row_map(CUtensorMap* map, const float* ptr, int64_t rows, int64_t cols, int64_t ld) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {32, 1};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time dependency on libcuda)
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

bool sddmm_use_blocked_order(const smb_pattern* pat, int64_t n) {
  // x + d_out at least 4x the 126 MB L2 (at 2x -- config 5, B = 512 -- the
  // blocked order measured 526 vs 514 us: the row segments mostly hit L2)
  return pat->ord_p != nullptr && (pat->m + pat->k) * n * (int64_t)sizeof(float) > (512ll << 20);
}

// The TMA variant applies to fp32, 16-byte aligned operands whose leading
// dimensions are multiples of 4 elements, and rows < 2^31.
bool sddmm_tma_supported(const smb_pattern* pat, const void* d_out, int64_t ld_d, const void* x,
                         int64_t ld_x, int64_t n) {
  return encode_fn() != nullptr && aligned16(d_out) && aligned16(x) && ld_d % 4 == 0 &&
         ld_x % 4 == 0 && n >= 1 && n < (int64_t(1) << 31) && pat->m < (int64_t(1) << 31) &&
         pat->k < (int64_t(1) << 31) && pat->nnz > 0;
}

int launch_sddmm_tma(const smb_pattern* pat, const float* d_out, int64_t ld_d, const float* x,
                     int64_t ld_x, int64_t n, const float* values, float* values_out,
                     float* velocity, float* grad_out, const OptConsts<float>& opt,
                     cudaStream_t st) {
  CUtensorMap xmap, dmap;
  if (!make_row_map(&xmap, x, pat->k, n, ld_x) || !make_row_map(&dmap, d_out, pat->m, n, ld_d)) {
    set_error("sddmm (TMA): tensor map encoding failed");
    return SMB_ERR_CUDA;
  }
// lab knobs (scripts/build_variant.sh): chains per lane, ring stages, staged
// d_out rows in CSR order / in the blocked order (a warp spans more rows there)
#ifndef SMB_TMA_PHASE_COLS
#define SMB_TMA_PHASE_COLS 256
#endif
#ifndef SMB_TMA_DS_ORD
#define SMB_TMA_DS_ORD 8
#endif
#ifndef SMB_TMA_K
#define SMB_TMA_K 1
#endif
#ifndef SMB_TMA_S
#define SMB_TMA_S 2
#endif
#ifndef SMB_TMA_DS
#define SMB_TMA_DS 4
#endif
  constexpr int K = SMB_TMA_K, S = SMB_TMA_S, DS = SMB_TMA_DS;
  int tb = 0, te = (int)n;
  auto gok = [&](auto kernel, int ds, int stages = SMB_TMA_S) {
    // ring + barriers + slot rows + row window (sddmm_tmak_kernel)
    const size_t smem =
        (size_t)stages * (32 * K * 128 + ds * 128) + 8 * stages + 8 * ds + 4 * (32 * K + 1);
    ensure_smem(kernel, smem);
    launch_k(kernel, dim3((unsigned)ceil_div(pat->nnz, 32 * K)), dim3(32), smem, st, xmap, dmap,
             pat->row_ptr, pat->col_idx, pat->tile_row0, pat->ord_p, pat->ord_row, pat->m,
             pat->nnz, d_out, ld_d, (int)n, values, values_out, velocity, grad_out, opt, tb, te,
             pat->acc_ws);
  };
  if (sddmm_use_blocked_order(pat, n)) {
    // x and d_out overflow L2 many times over (config 5 at B = 4096: 1 GB
    // each).  One launch over the whole batch kept 27% of its gathers in L2
    // and read 30 GB from HBM for 2.2 GB of operands (ncu): resident warps
    // are at every stage of their chains, so a block's working set is its
    // band rows x the whole batch.  Phases of kPhaseCols columns bound it to
    // band rows x kPhaseCols x 4 bytes x 2 (27 MB at 13,300-row bands).
    constexpr int kPhaseCols = SMB_TMA_PHASE_COLS;
    for (tb = 0; tb < (int)n; tb = te) {
      te = (kPhaseCols > 0 && pat->acc_ws) ? (int)imin(n, tb + kPhaseCols) : (int)n;
      gok(sddmm_tmak_kernel<S, true, K, SMB_TMA_DS_ORD>, SMB_TMA_DS_ORD);
    }
  } else if (pat->nnz < 16 * pat->m)
    // short rows: a warp's 32 nonzeros span more than 4 rows
    gok(sddmm_tmak_kernel<S, false, K, 8>, 8);
  else
    gok(sddmm_tmak_kernel<S, false, K, DS>, DS);
  return check_launch("smb_sddmm_update (TMA)");
}

}  // namespace smb
