// SDDMM + update with TMA row gathers (sm_100a).
//
// The same per-chain arithmetic as sddmm.cu (grad[p] = sum_t d_out[i,t] *
// x[j,t], one sequential chain per nonzero, multiply and add rounded
// separately, _kernels.py:62-75; then the sparse_combine update sequence of
// nn.py:187-197), with the staging done by the Tensor Memory Accelerator
// instead of per-thread cp.async:
//
//   * each warp owns 32 consecutive nonzeros (CSR order) and a private ring
//     of S stages; a stage holds the 32 gathered x-row segments of one
//     32-column batch chunk plus up to 4 d_out rows the warp's nonzeros span;
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
// Measured (ncu, config-4 hidden layer): the chains now leave the SM issue
// bound (78% of peak instruction throughput), and 30% of the issued
// instructions are the copy issue itself: the gather4 row coordinates are
// data (col_idx), so ptxas moves them into uniform registers through an
// ELECT / R2UR.BROADCAST loop per instruction.  Issuing all 9 copies from one
// lane with the same coordinates is slower (232 vs 211 us: one thread then
// serialises the 9 loops); one warp per CTA with a 2-stage ring (22 resident
// warps per SM) beat 2-4 warps per CTA and 3-8 stages.
//
// Valid for fp32 with 16-byte aligned operands and leading dimensions
// (sddmm_tma_supported); the caller falls back to sddmm.cu otherwise.
#include <cuda.h>

#include <type_traits>

#include "pattern.cuh"
#include "tma.cuh"

namespace smb {
namespace {

constexpr int kTmaXBytes = 32 * 128;  // x rows of one stage (1024-byte aligned blocks)
// d_out rows staged per stage: 4 (one gather4) in CSR order, 8 (two) in the
// blocked order, where a warp's 32 nonzeros span more rows
// shared memory of one warp's ring: S x-blocks, then S d-blocks, rounded to
// the 1024-byte swizzle atom (the hardware swizzle follows address bits
// 7-9, so 512-byte aligned gather4 destinations are fine)
template <int S, int DS>
__host__ __device__ constexpr int warp_ring_bytes() {
  return (S * (kTmaXBytes + DS * 128) + 1023) / 1024 * 1024;
}

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

// ORD: the warps walk the pattern's L2-blocked nonzero order (ord_p /
// ord_row, pattern.cu) instead of CSR order: a wave of resident warps then
// gathers the x and d_out rows of one (row band, column band) block, so each
// row segment is fetched from HBM about once per block instead of once per
// wave (config 5 at B = 4096: x and d_out are 1 GB each).  The chains, their
// order over the batch and the update are unchanged; results land at the
// nonzero's CSR index.
template <int S, int WPC, bool ORD, int DS = ORD ? 8 : 4>
__global__ void __launch_bounds__(32 * WPC)
    sddmm_tma_kernel(const __grid_constant__ CUtensorMap xmap,
                     const __grid_constant__ CUtensorMap dmap, const int32_t* __restrict__ row_ptr,
                     const int32_t* __restrict__ col_idx, const int32_t* __restrict__ tile_row0,
                     const int32_t* __restrict__ ord_p, const int32_t* __restrict__ ord_row,
                     int64_t m, int64_t nnz, const float* __restrict__ d_out, int64_t ld_d, int n,
                     const float* values, float* values_out, float* velocity, float* grad_out,
                     OptConsts<float> opt) {
  constexpr int kTile = 32 * WPC;  // nonzeros per CTA (a multiple of the tile_row0 grain)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int32_t s_rp[kTile + 1];
  __shared__ __align__(8) unsigned long long s_full[WPC][S];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // dynamic smem rounded up to 1024 bytes (the 128-byte swizzle atom)
  const unsigned raw = smem_addr(smem_raw);
  const unsigned base = ((raw + 1023u) & ~1023u) + (unsigned)(warp * warp_ring_bytes<S, DS>());
  const unsigned dbase = base + S * kTmaXBytes;
  const unsigned char* gbase = smem_raw + (base - raw);
  const int64_t p0 = (int64_t)blockIdx.x * kTile;
  const int64_t pw = p0 + warp * 32;
  const int nw = (int)imax(0, imin(32, nnz - pw));
  const bool active = lane < nw;
  // p: the CSR index of this lane's nonzero
  const int64_t p = ORD ? (active ? (int64_t)ord_p[pw + lane] : 0) : pw + lane;
  int32_t r0 = 0;
  if constexpr (!ORD) {
    r0 = tile_row0[(int64_t)blockIdx.x * (kTile / kTileGrain)];
    s_rp[tid] = (r0 + tid <= m) ? row_ptr[r0 + tid] : INT32_MAX;
    if (tid == 0) s_rp[kTile] = (r0 + kTile <= m) ? row_ptr[r0 + kTile] : INT32_MAX;
  }
  const int32_t my_col = active ? col_idx[p] : 0;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(smem_addr(&s_full[warp][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // the only CTA-wide barrier (row window + barrier init)
  if (nw == 0) return;
  int64_t row;
  int slot, n_slots;
  constexpr int kTmaDSlots = DS;
  constexpr int kTmaDBytes = DS * 128;
  int64_t slot_row[kTmaDSlots];
  if constexpr (ORD) {
    // d_out slots = runs of equal rows among the warp's nonzeros (rows are
    // non-decreasing inside a block)
    row = active ? (int64_t)ord_row[pw + lane] : (int64_t)ord_row[pw];
    const int64_t prev = __shfl_up_sync(0xffffffffu, row, 1);
    const unsigned runs = __ballot_sync(0xffffffffu, active && (lane == 0 || row != prev));
    slot = __popc(runs & (0xffffffffu >> (31 - lane))) - 1;
    n_slots = __popc(runs);
    unsigned rest = runs;
#pragma unroll
    for (int q = 0; q < kTmaDSlots; ++q) {
      const int src = rest ? __ffs(rest) - 1 : 0;
      const int64_t r = __shfl_sync(0xffffffffu, row, src);
      slot_row[q] = rest ? r : (q > 0 ? slot_row[q - 1] : r);
      rest &= rest - 1;
    }
  } else {
    row = tile_row_of<kTile>(active ? p : pw, r0, s_rp, row_ptr, m);
    const int64_t row_first = __shfl_sync(0xffffffffu, row, 0);
    const int64_t row_last = __shfl_sync(0xffffffffu, row, nw - 1);
    n_slots = (int)(row_last - row_first + 1);
    slot = (int)(row - row_first);
#pragma unroll
    for (int q = 0; q < kTmaDSlots; ++q) slot_row[q] = imin(row_first + imin(q, n_slots - 1), m - 1);
  }
  const bool staged = n_slots <= kTmaDSlots;  // warp-uniform
  const int n_chunks = (n + 31) / 32;
  // copy roles: lane g < 8 gathers x rows 4g..4g+3, lane 8 the d_out rows
  int gr[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int src = (lane < 8) ? 4 * lane + q : 0;
    gr[q] = __shfl_sync(0xffffffffu, my_col, src);
  }
  // lanes 8 (and 9) gather the staged d_out rows 0-3 (4-7)
#pragma unroll
  for (int g = 0; g < DS / 4; ++g)
    if (lane == 8 + g) {
#pragma unroll
      for (int q = 0; q < 4; ++q) gr[q] = (int)slot_row[4 * g + q];
    }
  const bool copier = lane < 8 || (staged && lane < 8 + DS / 4);
  const unsigned tx_bytes = 32 * 128 + (staged ? kTmaDSlots * 128 : 0);
  pdl_wait();  // d_out / x are earlier kernels' outputs
  const bool upd = active && opt.kind != SMB_OPT_NONE;
  float w_pre = upd ? values[p] : 0.f;
  float v_pre = (upd && velocity) ? velocity[p] : 0.f;
  // two copy sites so that each one's tensor map is a uniform operand (the
  // row coordinates are data: ptxas moves them to uniform registers in an
  // ELECT / R2UR loop, one pass per copying lane)
  auto issue = [&](int ch) {
    const int s = ch % S;
    const unsigned bar = smem_addr(&s_full[warp][s]);
    if (lane == 0) mbar_arrive_expect_tx(bar, tx_bytes);
    __syncwarp();
    if (lane < 8)
      tma_gather4(base + (unsigned)(s * kTmaXBytes + lane * 512), &xmap, ch * 32, gr[0], gr[1],
                  gr[2], gr[3], bar);
    else if (copier)
      tma_gather4(dbase + (unsigned)(s * kTmaDBytes + (lane - 8) * 512), &dmap, ch * 32, gr[0],
                  gr[1], gr[2], gr[3], bar);
  };
  for (int c = 0; c < S && c < n_chunks; ++c) issue(c);
  float acc = -0.0f;  // exact additive identity (sddmm.cu)
  const float* drow = d_out + row * ld_d;
  const int xsw = lane & 7;  // swizzle of this lane's x row (1024-aligned x blocks)
  // the chunk loop is instantiated per staging mode (warp-uniform): as one
  // loop with `staged` tested inside, ptxas predicated the 32 global d_out
  // loads of the fallback into the staged path (issue slots spent on
  // masked-off instructions)
  auto run = [&](auto staged_c) {
  constexpr bool kStaged = decltype(staged_c)::value;
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int s = ch % S;
    mbar_wait(smem_addr(&s_full[warp][s]), (unsigned)((ch / S) & 1));
    const float* xr = reinterpret_cast<const float*>(gbase + s * kTmaXBytes + lane * 128);
    const unsigned doff = S * kTmaXBytes + s * kTmaDBytes + slot * 128;
    const float* dr = reinterpret_cast<const float*>(gbase + doff);
    const int dsw = (int)(((base + doff) >> 7) & 7);  // swizzle of this lane's d_out row
    const int t0 = ch * 32;
    const int cnt = min(32, n - t0);
    if (cnt == 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 xv = *reinterpret_cast<const float4*>(xr + 4 * (u ^ xsw));
        float4 dv;
        if constexpr (kStaged) {
          dv = *reinterpret_cast<const float4*>(dr + 4 * (u ^ dsw));
        } else {
          dv = make_float4(drow[t0 + 4 * u], drow[t0 + 4 * u + 1], drow[t0 + 4 * u + 2],
                           drow[t0 + 4 * u + 3]);
        }
        acc = add_rn(acc, mul_rn(dv.x, xv.x));
        acc = add_rn(acc, mul_rn(dv.y, xv.y));
        acc = add_rn(acc, mul_rn(dv.z, xv.z));
        acc = add_rn(acc, mul_rn(dv.w, xv.w));
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        const int u = j >> 2, e = j & 3;
        const float xv = xr[4 * (u ^ xsw) + e];
        const float dv = kStaged ? dr[4 * (u ^ dsw) + e] : drow[t0 + j];
        acc = add_rn(acc, mul_rn(dv, xv));
      }
    }
    __syncwarp();  // every lane has read stage s: refill it
    if (ch + S < n_chunks) issue(ch + S);
  }
  };
  if (staged)
    run(std::true_type{});
  else
    run(std::false_type{});
  pdl_trigger();
  if (!active) return;
  const float g = (n == 0) ? 0.f : acc;  // tensor_core.py:283-284: zero batch -> zeros
  if (grad_out) grad_out[p] = g;
  if (upd) {
    apply_update(opt, g, &w_pre, &v_pre);
    values_out[p] = w_pre;
    if (velocity) velocity[p] = v_pre;
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
  auto go = [&](auto kernel, int s, int wpc, int ring) {
    const size_t smem = (size_t)wpc * ring + 1024;
    ensure_smem(kernel, smem);
    launch_k(kernel, dim3((unsigned)ceil_div(pat->nnz, 32 * wpc)), dim3(32 * wpc), smem, st,
             xmap, dmap, pat->row_ptr, pat->col_idx, pat->tile_row0, pat->ord_p, pat->ord_row,
             pat->m, pat->nnz, d_out, ld_d, (int)n, values, values_out, velocity, grad_out, opt);
  };
  if (sddmm_use_blocked_order(pat, n))
    go(sddmm_tma_kernel<2, 1, true>, 2, 1, warp_ring_bytes<2, 8>());
  else
    go(sddmm_tma_kernel<2, 1, false>, 2, 1, warp_ring_bytes<2, 4>());
  return check_launch("smb_sddmm_update (TMA)");
}

}  // namespace smb
