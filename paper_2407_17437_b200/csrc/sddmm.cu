// SDDMM weight gradient fused with the optimizer update (sm_100a).
//
// grad[p] = sum_t d_out[i, t] * x[j, t] for the p-th stored (i, j), summed
// sequentially over t with separately rounded multiply/add exactly like
// _kernels.sddmm_kernel (_kernels.py:62-75), then (optionally) the momentum /
// Nesterov / GD update of values and velocity in the sparse_combine order of
// SparseLinearLayer.optimize (nn.py:187-197).  No dense m x k gradient and no
// mask is ever formed.  The bias side (grad_bias = row_sums(d_out), nn.py:184,
// and its _step_vector update) runs in the warp-per-row kernel of
// elementwise.cu -- or, on the fused training step, in the epilogue of the
// transposed SpMM / softmax kernel that produced d_out.
//
// Mapping: one CTA = TILE (128 or 512) consecutive nonzeros of the CSR order,
// one per thread, each running ONE sequential accumulation chain (required
// for bit-exactness; the FADD latency is hidden by having 16 warps of
// independent chains per SM).  The batch is walked in 32/64-column chunks
// through a STAGES-deep ring in shared memory, filled with 16-byte cp.async
// (LDGSTS) copies of the gathered x rows and of the few d_out rows the tile
// touches; one barrier per chunk.  Every thread owns a fixed set of copy
// slots (row base pointer + smem offset computed once), so a copy costs ~4
// instructions.  Staged rows are unpadded, 128-byte aligned lines whose
// 16-byte vectors are XOR-swizzled (vector v of row r at slot v ^ (r & 7)), so
// each thread's 16-byte LDS of its own x row is bank-conflict free.  (Rows
// padded to 144 bytes were conflict free too, but a 128-byte copy into a line
// straddling two 128-byte smem lines is split by the LSU: ncu counted 24 L2
// sectors per 16-sector warp copy, 162 MB instead of 106 MB for the config-2
// layer-0 SDDMM.)
// (A TMA variant -- one cp.async.bulk per 128-byte row, producer warp +
// mbarrier ring -- measured 4x slower on B200: 128-byte bulk copies are
// request-rate bound at ~1.1 TB/s.  See DESIGN.md.)
#include "async_copy.cuh"
#include "pattern.cuh"

namespace smb {
namespace {

// TILE nonzeros per CTA, CH batch columns per pipeline stage
template <typename T, int TILE, int CH, int ST, int SD = 4>
struct SddmmCfg {
  static constexpr int kChunk = CH;
  static constexpr int VW = 16 / sizeof(T);  // elements per 16 B
  static constexpr int LDS = kChunk;         // smem row (elements), swizzled
  static constexpr int VPR = kChunk / VW;    // 16 B vectors per staged row
  static_assert(VPR % 8 == 0, "swizzle spans 8 vectors");
  // staged d_out rows per tile: TILE/4 (rows of >= 4 nonzeros on average),
  // or TILE (SD = 1) for very sparse layers whose tiles span ~1 row per nonzero
  static constexpr int SLOTS = TILE / SD;
  // ring of STAGES stages (stage = chunk % STAGES); defaults:
  //   fp32 512-tile x 32 cols x 2 stages = 184 KB (1 CTA, 16 warps / SM),
  //   fp32 128-tile x 64 cols x 2 stages =  87 KB (2 CTAs / SM),
  //   fp64 128-tile x 16 cols x 4 stages =  92 KB
  static constexpr int STAGES = ST;
  static constexpr size_t stage_elems = size_t(TILE + SLOTS) * LDS;
  // + 128: the ring starts at the first 128-byte boundary of dynamic smem
  static constexpr size_t smem_bytes = STAGES * stage_elems * sizeof(T) + 128;
  static_assert(TILE % VPR == 0, "tile / vector split");
};

// ALL: every tile's d_out rows fit the SLOTS staging rows (checked on the
// host from the pattern's tile spans), so the hot loop has no fallback path.
template <typename T, int TILE, int CH, int ST, int SD, bool VEC, bool ALL>
__global__ void __launch_bounds__(TILE)
    sddmm_pipe_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                      const int32_t* __restrict__ tile_row0, int64_t m, int64_t nnz,
                      const T* __restrict__ d_out, int64_t ld_d, const T* __restrict__ x,
                      int64_t ld_x, int64_t n, const T* values, T* values_out, T* velocity,
                      T* grad_out, OptConsts<T> opt) {
  using C = SddmmCfg<T, TILE, CH, ST, SD>;
  constexpr int S = C::STAGES, VW = C::VW, VPR = C::VPR, LDS = C::LDS;
  constexpr int kChunk = C::kChunk;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(align128(smem_raw));
  __shared__ int32_t s_col[TILE];
  __shared__ int32_t s_rp[TILE + 1];
  const int tid = threadIdx.x;
  const int64_t p0 = (int64_t)blockIdx.x * TILE;
  const int64_t p = p0 + tid;
  const int n_active = (int)imin(TILE, nnz - p0);
  const bool active = tid < n_active;
  const int32_t r0 = tile_row0[(int64_t)blockIdx.x * (TILE / kTileGrain)];
  s_col[tid] = active ? col_idx[p] : 0;
  s_rp[tid] = (r0 + tid <= m) ? row_ptr[r0 + tid] : INT32_MAX;
  if (tid == 0) s_rp[TILE] = (r0 + TILE <= m) ? row_ptr[r0 + TILE] : INT32_MAX;
  __syncthreads();
  const int64_t row = tile_row_of<TILE>(p, r0, s_rp, row_ptr, m);
  const int slot = (int)imin(row - r0, C::SLOTS);  // SLOTS == "not staged"
  // only the rows this tile actually touches (r0 .. row of its last nonzero)
  const int64_t last_row = tile_row_of<TILE>(p0 + n_active - 1, r0, s_rp, row_ptr, m);
  const int n_staged = (int)imin(C::SLOTS, last_row - r0 + 1);
  // batch widths are far below 2^31: all chunk / column arithmetic is 32-bit
  const int n32 = (int)n;
  const int n_chunks = (n32 + kChunk - 1) / kChunk;

  // ---- fixed copy slots of this thread (computed once) ----
  // x rows: vector v = tid % VPR of rows tid/VPR + k*TILE/VPR, k < VPR
  const int v = tid % VPR;
  const T* xsrc[VPR];
  unsigned xdst[VPR];
  int xok[VPR];
  // (rows past n_active copy x row 0 -- s_col = 0 -- on full chunks: a
  // valid read nobody sums, so the full-chunk copies carry no predicate)
#pragma unroll
  for (int k = 0; k < VPR; ++k) {
    const int r = tid / VPR + k * (TILE / VPR);
    xok[k] = r < n_active;
    xsrc[k] = x + (int64_t)s_col[r] * ld_x + v * VW;
    xdst[k] = (unsigned)(swz<LDS, VW>(r, v) * sizeof(T));
  }
  // d_out rows of the tile: SLOTS*VPR copies, DC per thread; copy e = tid +
  // c*TILE stages vector v of slot row e/VPR (TILE % VPR == 0 keeps v fixed)
  constexpr int DC = (C::SLOTS * VPR + TILE - 1) / TILE;
  // copies past the rows the tile spans are skipped: issuing them (all from
  // row r0) cost config 4 / 5 ~5-10% in redundant L2 requests to hot lines
  bool dcopy[DC];
  const T* dsrc[DC];
  unsigned ddst[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    const int e = tid + c * TILE;
    dcopy[c] = e < n_staged * VPR;
    dsrc[c] = d_out + (int64_t)(r0 + (dcopy[c] ? e / VPR : 0)) * ld_d + v * VW;
    ddst[c] = (unsigned)(swz<LDS, VW>(TILE + e / VPR, v) * sizeof(T));
  }
  const unsigned sbase = smem_u32(smem);
  constexpr unsigned kStageBytes = (unsigned)(C::stage_elems * sizeof(T));
  pdl_wait();  // d_out / x are earlier kernels' outputs
  // the update's operands, loaded now so they arrive during the chain instead
  // of costing one more memory round trip after it
  const bool upd = active && opt.kind != SMB_OPT_NONE;
  T w_pre = upd ? values[p] : T(0);
  T v_pre = (upd && velocity) ? velocity[p] : T(0);

  // full chunks (copied without bounds when VEC) run a lean main loop; a
  // ragged last chunk (n % CH != 0) is copied and summed after it
  const int n_fast = n32 / kChunk;
  const int n_full = VEC ? n_fast : 0;
  auto issue_full = [&](int ch) {
    const unsigned st = sbase + (unsigned)(ch % S) * kStageBytes;
    const int t0 = ch * kChunk;
#pragma unroll
    for (int k = 0; k < VPR; ++k) cp_async16(st + xdst[k], xsrc[k] + t0);
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (dcopy[c]) cp_async16(st + ddst[c], dsrc[c] + t0);
  };
  auto issue_part = [&](int ch) {
    const unsigned st = sbase + (unsigned)(ch % S) * kStageBytes;
    const int t0 = ch * kChunk;
    // elements of this thread's vector inside [0, n)
    const int valid = max(0, min(VW, n32 - (t0 + v * VW)));
#pragma unroll
    for (int k = 0; k < VPR; ++k) copy_vec<T, VEC>(st + xdst[k], xsrc[k] + t0, xok[k] ? valid : 0);
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (dcopy[c]) copy_vec<T, VEC>(st + ddst[c], dsrc[c] + t0, valid);
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < n_full) issue_full(s);
    else if (s < n_chunks) issue_part(s);
    cp_async_commit();
  }
  // -0.0 is the exact additive identity, so acc = -0 + a0*b0 == a0*b0 and the
  // chain below is the reference's  acc = a0*b0; acc += a_t*b_t  verbatim.
  T acc = T(-0.0);
  // inactive threads sum zero-filled rows (never stored) from slot 0
  const int rslot = active ? slot : 0;
  const T* drow = d_out + (active ? row : r0) * ld_d;
  using V = typename Vec16<T>::type;
  // smem offsets of this thread's x-row / d_out-row vectors w < 8 (the
  // swizzle permutes the vectors inside each aligned group of 8)
  int xo[8], dof[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    xo[w] = swz<LDS, VW>(tid, w);
    dof[w] = swz<LDS, VW>(TILE + rslot, w);
  }
  // chunk ch landed for everyone (then stage (ch-1) % S is free: refill it)
  auto landed = [&](int ch) {
    cp_async_wait<S - 2>();
    __syncthreads();
    const int nx = ch + S - 1;
    if (nx < n_full) issue_full(nx);
    else if (nx < n_chunks) issue_part(nx);
    cp_async_commit();
  };
  // vectors g*8 .. g*8+7 of chunk ch: this thread's x row and d_out row
  auto load8 = [&](int ch, int g, V* xv, V* dv) {
    const T* xs = smem + (ch % S) * C::stage_elems;
    const int t0 = ch * kChunk;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      xv[w] = lds16(xs + xo[w] + g * 8 * VW);
      if (ALL || rslot < C::SLOTS) {
        dv[w] = lds16(xs + dof[w] + g * 8 * VW);
      } else {
#pragma unroll
        for (int j = 0; j < VW; ++j) VecOps<T>::set(dv[w], j, drow[t0 + (g * 8 + w) * VW + j]);
      }
    }
  };
  auto sum8 = [&](const V* xv, const V* dv) {
#pragma unroll
    for (int w = 0; w < 8; ++w)
#pragma unroll
      for (int j = 0; j < VW; ++j)
        acc = add_rn(acc, mul_rn(VecOps<T>::get(dv[w], j), VecOps<T>::get(xv[w], j)));
  };
  int ch = 0;
  if constexpr (VPR == 8) {
    // Chunk ch's shared-memory reads are issued before chunk ch-1's chain
    // runs (two register sets, loop unrolled by two): ptxas otherwise sinks
    // every read next to its first use and the chain stalls on the LDS
    // latency once per vector.
    V xa[8], da[8], xb[8], db[8];
    if (n_fast > 0) {
      landed(0);
      load8(0, 0, xa, da);
    }
    for (ch = 1; ch + 1 < n_fast; ch += 2) {
      landed(ch);
      load8(ch, 0, xb, db);
      sum8(xa, da);
      landed(ch + 1);
      load8(ch + 1, 0, xa, da);
      sum8(xb, db);
    }
    if (ch < n_fast) {
      landed(ch);
      load8(ch, 0, xb, db);
      sum8(xa, da);
      sum8(xb, db);
    } else if (n_fast > 0) {
      sum8(xa, da);
    }
    ch = n_fast;
  } else {
    for (; ch < n_fast; ++ch) {
      landed(ch);
#pragma unroll
      for (int g = 0; g < VPR / 8; ++g) {
        V xv[8], dv[8];
        load8(ch, g, xv, dv);
        sum8(xv, dv);
      }
    }
  }
  if (ch < n_chunks) {  // ragged last chunk (no further copies to issue)
    cp_async_wait<0>();
    __syncthreads();
    const T* xs = smem + (ch % S) * C::stage_elems;
    const int t0 = ch * kChunk;
    const int cnt = n32 - t0;
    for (int j = 0; j < cnt; ++j) {
      const T dv = (ALL || rslot < C::SLOTS) ? xs[swz<LDS, VW>(TILE + rslot, j / VW) + j % VW]
                                             : drow[t0 + j];
      acc = add_rn(acc, mul_rn(dv, xs[swz<LDS, VW>(tid, j / VW) + j % VW]));
    }
  }
  cp_async_wait<0>();
  pdl_trigger();
  if (!active) return;
  const T g = (n == 0) ? T(0) : acc;  // tensor_core.py:283-284: zero batch -> zeros
  if (grad_out) grad_out[p] = g;
  if (upd) {
    // pre-update value read from `values` (above), the result written to
    // `values_out` (== values for the in-place update)
    apply_update(opt, g, &w_pre, &v_pre);
    values_out[p] = w_pre;
    if (velocity) velocity[p] = v_pre;
  }
}

// Warp-independent variant for many-wave layers: each warp owns 32
// consecutive nonzeros of a 128-nonzero tile and stages, in its own
// shared-memory ring, their x rows and the (<= kWarpDSlots) d_out rows they
// span; it waits on its own cp.async groups + __syncwarp, so warps never
// meet at a CTA barrier.  Warps whose 32 nonzeros span more rows read d_out
// from global memory.  Same per-chain order / rounding as sddmm_pipe_kernel.
constexpr int kWarpDSlots = 4;

template <typename T, int CH, int S>
struct SddmmWarpCfg {
  static constexpr int VW = 16 / sizeof(T);
  static constexpr int LDS = CH;  // swizzled 128-byte-aligned rows (see sddmm_pipe_kernel)
  static constexpr int VPR = CH / VW;
  static_assert(VPR % 8 == 0, "swizzle spans 8 vectors");
  static constexpr size_t warp_elems = size_t(S) * (32 + kWarpDSlots) * LDS;
  static constexpr size_t smem_bytes = 4 * warp_elems * sizeof(T) + 128;  // 4 warps per CTA
};

template <typename T, int CH, int S>
__global__ void __launch_bounds__(128)
    sddmm_warp_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                      const int32_t* __restrict__ tile_row0, int64_t m, int64_t nnz,
                      const T* __restrict__ d_out, int64_t ld_d, const T* __restrict__ x,
                      int64_t ld_x, int64_t n, const T* values, T* values_out, T* velocity,
                      T* grad_out, OptConsts<T> opt) {
  using C = SddmmWarpCfg<T, CH, S>;
  constexpr int VW = C::VW, LDS = C::LDS, VPR = C::VPR;
  static_assert(kWarpDSlots * VPR <= 32, "one d_out copy per lane");
  constexpr unsigned kStageBytes = (unsigned)((32 + kWarpDSlots) * LDS * sizeof(T));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int32_t s_rp[kSddmmTile + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* wsm = reinterpret_cast<T*>(align128(smem_raw)) + warp * C::warp_elems;
  const int64_t p0 = (int64_t)blockIdx.x * kSddmmTile;
  const int64_t pw = p0 + warp * 32;             // first nonzero of this warp
  const int nw = (int)imax(0, imin(32, nnz - pw));  // nonzeros of this warp
  const int64_t p = pw + lane;
  const bool active = lane < nw;
  const int32_t r0 = tile_row0[(int64_t)blockIdx.x * (kSddmmTile / kTileGrain)];
  s_rp[tid] = (r0 + tid <= m) ? row_ptr[r0 + tid] : INT32_MAX;
  if (tid == 0) s_rp[kSddmmTile] = (r0 + kSddmmTile <= m) ? row_ptr[r0 + kSddmmTile] : INT32_MAX;
  const int32_t my_col = active ? col_idx[p] : 0;
  __syncthreads();  // the only CTA-wide barrier (row window)
  if (nw == 0) return;
  const int64_t row = tile_row_of<kSddmmTile>(active ? p : pw, r0, s_rp, row_ptr, m);
  const int64_t row_first = __shfl_sync(0xffffffffu, row, 0);
  const int64_t row_last = __shfl_sync(0xffffffffu, row, nw - 1);
  const int span = (int)(row_last - row_first + 1);
  const bool staged = span <= kWarpDSlots;  // warp-uniform
  const int slot = (int)(row - row_first);
  const int n32 = (int)n;
  const int n_chunks = (n32 + CH - 1) / CH;
  // copy slots: x vectors e = lane + 32 k (k < VPR): row e / VPR, part e % VPR
  const T* xsrc[VPR];
  unsigned xdst[VPR];
  int xok[VPR];
#pragma unroll
  for (int k = 0; k < VPR; ++k) {
    const int e = lane + 32 * k, r = e / VPR, v = e % VPR;
    const int32_t c = __shfl_sync(0xffffffffu, my_col, r);
    xok[k] = r < nw ? 16 : 0;
    xsrc[k] = x + (int64_t)c * ld_x + v * VW;
    xdst[k] = (unsigned)(swz<LDS, VW>(r, v) * sizeof(T));
  }
  // d_out rows: vector e = lane (kWarpDSlots * VPR <= 32 for CH <= 32 fp32)
  const bool dcopy = staged && lane < span * VPR;
  const T* dsrc = d_out + (row_first + (dcopy ? lane / VPR : 0)) * ld_d + (lane % VPR) * VW;
  const unsigned ddst = (unsigned)(swz<LDS, VW>(32 + lane / VPR, lane % VPR) * sizeof(T));
  const unsigned sbase = smem_u32(wsm);
  pdl_wait();  // d_out / x are earlier kernels' outputs
  const bool upd = active && opt.kind != SMB_OPT_NONE;  // update operands loaded early
  T w_pre = upd ? values[p] : T(0);
  T v_pre = (upd && velocity) ? velocity[p] : T(0);
  auto issue = [&](int ch) {
    const unsigned st = sbase + (unsigned)(ch % S) * kStageBytes;
    const int t0 = ch * CH;
    if (t0 + CH <= n32) {
#pragma unroll
      for (int k = 0; k < VPR; ++k) cp_async16(st + xdst[k], xsrc[k] + t0, xok[k]);
      if (dcopy) cp_async16(st + ddst, dsrc + t0, 16);
      return;
    }
    const int valid = max(0, min(VW, n32 - (t0 + (lane % VPR) * VW)));
#pragma unroll
    for (int k = 0; k < VPR; ++k) {
      const int vk = max(0, min(VW, n32 - (t0 + ((lane + 32 * k) % VPR) * VW)));
      cp_async16(st + xdst[k], xsrc[k] + t0, xok[k] ? vk * (int)sizeof(T) : 0);
    }
    if (dcopy) cp_async16(st + ddst, dsrc + t0, valid * (int)sizeof(T));
  };
#pragma unroll
  for (int c = 0; c < S - 1; ++c) {
    if (c < n_chunks) issue(c);
    cp_async_commit();
  }
  T acc = T(-0.0);
  const T* drow = d_out + row * ld_d;
  using V = typename Vec16<T>::type;
  for (int ch = 0; ch < n_chunks; ++ch) {
    cp_async_wait<S - 2>();
    __syncwarp();  // chunk ch landed for the whole warp; stage (ch-1) % S is free
    if (ch + S - 1 < n_chunks) issue(ch + S - 1);
    cp_async_commit();
    if (active) {
      const T* xs = wsm + (ch % S) * (kStageBytes / sizeof(T));
      const int t0 = ch * CH;
      const int cnt = min(CH, n32 - t0);
      if (cnt == CH) {
#pragma unroll
        for (int u = 0; u < VPR; ++u) {
          const V xv = *reinterpret_cast<const V*>(xs + swz<LDS, VW>(lane, u));
          V dv;
          if (staged) {
            dv = *reinterpret_cast<const V*>(xs + swz<LDS, VW>(32 + slot, u));
          } else {
#pragma unroll
            for (int j = 0; j < VW; ++j) VecOps<T>::set(dv, j, drow[t0 + u * VW + j]);
          }
#pragma unroll
          for (int j = 0; j < VW; ++j)
            acc = add_rn(acc, mul_rn(VecOps<T>::get(dv, j), VecOps<T>::get(xv, j)));
        }
      } else {
        for (int j = 0; j < cnt; ++j) {
          const T dv = staged ? xs[swz<LDS, VW>(32 + slot, j / VW) + j % VW] : drow[t0 + j];
          acc = add_rn(acc, mul_rn(dv, xs[swz<LDS, VW>(lane, j / VW) + j % VW]));
        }
      }
    }
    __syncwarp();  // every lane done reading this stage before it is refilled
  }
  cp_async_wait<0>();
  pdl_trigger();
  if (!active) return;
  const T g = (n == 0) ? T(0) : acc;  // tensor_core.py:283-284: zero batch -> zeros
  if (grad_out) grad_out[p] = g;
  if (upd) {
    apply_update(opt, g, &w_pre, &v_pre);
    values_out[p] = w_pre;
    if (velocity) velocity[p] = v_pre;
  }
}

// Lean one-warp tile kernel for few-wave fp32 layers (config 2: 1-5 warps per
// SM).  With so few warps an SM's issue slots are idle and each warp runs at
// its own instruction rate, so the time of a chain is the instruction count
// of its chunk loop: sddmm_pipe_kernel spends ~270 instructions per 32-column
// chunk (dynamic ring-stage arithmetic, 64-bit source address adds, full /
// ragged issue branches, a CTA barrier) for 64 multiplies and adds.  Here the
// chunk loop is unrolled over the S ring stages, so stage addresses and the
// copies' column offsets are immediates, the source pointers advance once per
// S chunks, and the warp synchronises with __syncwarp.  Same chains, order
// and rounding; tiles must span <= DS rows (host check) and operands be
// 16-byte aligned.
template <int S, int DS>
__global__ void __launch_bounds__(32)
    sddmm_lean_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                      const int32_t* __restrict__ tile_row0, int64_t m, int64_t nnz,
                      const float* __restrict__ d_out, int64_t ld_d, const float* __restrict__ x,
                      int64_t ld_x, int n, const float* values, float* values_out,
                      float* velocity, float* grad_out, OptConsts<float> opt) {
  static_assert(S % 2 == 0 && DS % 4 == 0, "two register sets alternate over the stages");
  constexpr int kStageFloats = (32 + DS) * 32;
  constexpr unsigned kStageBytes = kStageFloats * 4;
  constexpr int DC = DS / 4;  // d_out copies per lane and chunk
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* smem = reinterpret_cast<float*>(align128(smem_raw));
  __shared__ int32_t s_col[32];
  __shared__ int32_t s_rp[33];
  const int lane = threadIdx.x;
  const int64_t p0 = (int64_t)blockIdx.x * 32;
  const int64_t p = p0 + lane;
  const int n_active = (int)imin(32, nnz - p0);
  const bool active = lane < n_active;
  const int32_t r0 = tile_row0[blockIdx.x];
  s_col[lane] = active ? col_idx[p] : 0;
  s_rp[lane] = (r0 + lane <= m) ? row_ptr[r0 + lane] : INT32_MAX;
  if (lane == 0) s_rp[32] = (r0 + 32 <= m) ? row_ptr[r0 + 32] : INT32_MAX;
  __syncwarp();
  const int64_t row = tile_row_of<32>(active ? p : p0, r0, s_rp, row_ptr, m);
  const int slot = (int)(row - r0);  // < DS (host check)
  const int64_t last_row = tile_row_of<32>(p0 + n_active - 1, r0, s_rp, row_ptr, m);
  const int n_staged = (int)imin(DS, last_row - r0 + 1);
  // copy slots of this lane: vector v of x rows lane/8 + 4k and of d_out rows lane/8 + 4c
  const int v = lane & 7, rq = lane >> 3;
  const float* xp[8];
  unsigned xdst[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int r = rq + 4 * k;
    xp[k] = x + (int64_t)s_col[r] * ld_x + v * 4;
    xdst[k] = (unsigned)(swz<32, 4>(r, v) * 4);
  }
  bool dcopy[DC];
  const float* dp[DC];
  unsigned ddst[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) {
    const int r = rq + 4 * c;
    dcopy[c] = r < n_staged;
    dp[c] = d_out + (int64_t)(r0 + (dcopy[c] ? r : 0)) * ld_d + v * 4;
    ddst[c] = (unsigned)(swz<32, 4>(32 + r, v) * 4);
  }
  const unsigned sbase = smem_u32(smem);
  pdl_wait();  // d_out / x are earlier kernels' outputs
  const bool upd = active && opt.kind != SMB_OPT_NONE;
  float w_pre = upd ? values[p] : 0.f;
  float v_pre = (upd && velocity) ? velocity[p] : 0.f;
  const int n_full = n / 32;
  const int n_chunks = (n + 31) / 32;
  // chunk `ch` into ring stage `stage`; `off` = its first column relative to
  // the advancing source pointers (an immediate at every call site)
  auto issue = [&](int ch, int stage, int off) {
    const unsigned st = sbase + (unsigned)stage * kStageBytes;
    if (ch < n_full) {
#pragma unroll
      for (int k = 0; k < 8; ++k) cp_async16(st + xdst[k], xp[k] + off);
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (dcopy[c]) cp_async16(st + ddst[c], dp[c] + off);
    } else if (ch < n_chunks) {  // the ragged last chunk: zero-filled past n
      const int valid = max(0, min(4, n - (ch * 32 + v * 4)));
#pragma unroll
      for (int k = 0; k < 8; ++k) cp_async16(st + xdst[k], xp[k] + off, valid * 4);
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (dcopy[c]) cp_async16(st + ddst[c], dp[c] + off, valid * 4);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(s, s, s * 32);
  // this lane's x row / d_out row vectors inside a stage
  int xo[8], dof[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    xo[w] = swz<32, 4>(lane, w);
    dof[w] = swz<32, 4>(32 + slot, w);
  }
  float acc = -0.0f;  // exact additive identity (sddmm_pipe_kernel)
  float4 xr[2][8], dr[2][8];
  auto sum8 = [&](const float4* xv, const float4* dv) {
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      acc = add_rn(acc, mul_rn(dv[w].x, xv[w].x));
      acc = add_rn(acc, mul_rn(dv[w].y, xv[w].y));
      acc = add_rn(acc, mul_rn(dv[w].z, xv[w].z));
      acc = add_rn(acc, mul_rn(dv[w].w, xv[w].w));
    }
  };
  // Chunk ch's shared-memory reads are issued before chunk ch-1's chain runs
  // (two register sets; chunk parity == stage parity because S is even).
  for (int ch0 = 0; ch0 < n_full; ch0 += S) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int ch = ch0 + s;
      if (ch >= n_full) break;
      cp_async_wait<S - 2>();
      __syncwarp();  // chunk ch landed for every lane; stage (s - 1) % S is free
      issue(ch + S - 1, (s + S - 1) % S, (s + S - 1) * 32);
      const float* xs = smem + s * kStageFloats;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        xr[s & 1][w] = lds16(xs + xo[w]);
        dr[s & 1][w] = lds16(xs + dof[w]);
      }
      if (ch > 0) sum8(xr[(s & 1) ^ 1], dr[(s & 1) ^ 1]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) xp[k] += S * 32;
#pragma unroll
    for (int c = 0; c < DC; ++c) dp[c] += S * 32;
  }
  if (n_full > 0) {
    if ((n_full - 1) & 1) sum8(xr[1], dr[1]);
    else sum8(xr[0], dr[0]);
  }
  cp_async_wait<0>();
  if (n_full < n_chunks) {  // ragged last chunk
    __syncwarp();
    const float* xs = smem + (n_full % S) * kStageFloats;
    const int cnt = n - n_full * 32;
    for (int j = 0; j < cnt; ++j)
      acc = add_rn(acc, mul_rn(xs[swz<32, 4>(32 + slot, j / 4) + j % 4],
                               xs[swz<32, 4>(lane, j / 4) + j % 4]));
  }
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

}  // namespace

template <typename T>
int launch_bias_rows(const T* d, int64_t ld, int64_t m, int64_t n, T* bias, T* vbias, T* grad,
                     const OptConsts<T>& opt, cudaStream_t st);

// ring shapes of the few-wave (config-2) tile kernels; compile-time knobs
// for tuning sweeps (scripts/build_variant.sh)
#ifndef SMB_SD_MID_STAGES
#define SMB_SD_MID_STAGES 8
#endif
#ifndef SMB_SD_SMALL_STAGES
#define SMB_SD_SMALL_STAGES 4
#endif
#ifndef SMB_SD_SMALL_CHUNK
#define SMB_SD_SMALL_CHUNK 32
#endif

template <typename T>
int sddmm_update_impl(const smb_pattern* pat, const void* d_out, int64_t ld_d, const void* x,
                      int64_t ld_x, int64_t n, const void* values, void* values_out,
                      void* velocity, void* grad_out, void* bias, void* vbias,
                      void* grad_bias_out, int opt_kind, double mu, double eta, void* stream,
                      const char* name, bool concurrent = false) {
  const OptConsts<T> opt = make_opt<T>(opt_kind, mu, eta);
  cudaStream_t st = as_stream(stream);
  if (pat->ntiles > 0) {
    constexpr int VW = 16 / sizeof(T);
    const bool vec = aligned16(x) && aligned16(d_out) && ld_x % VW == 0 && ld_d % VW == 0;
    auto go = [&](auto kernel, int tile, size_t bytes) {
      ensure_smem(kernel, bytes);
      launch_k(kernel, dim3((unsigned)ceil_div(pat->nnz, tile)), dim3(tile), bytes, st,
               pat->row_ptr, pat->col_idx, pat->tile_row0, pat->m, pat->nnz,
               static_cast<const T*>(d_out), ld_d, static_cast<const T*>(x), ld_x, n,
               static_cast<const T*>(values), static_cast<T*>(values_out),
               static_cast<T*>(velocity), static_cast<T*>(grad_out), opt);
    };
    // every tile's d_out rows staged -> fallback-free kernel (a 256 / 512-tile's
    // span is bounded by its enclosing 512-tile's)
    auto all_for = [&](int tile, int sd) {
      const int64_t span = tile == 32    ? pat->span32
                           : tile == 64  ? pat->span64
                           : tile == 128 ? pat->span128
                                         : pat->span512;
      return span <= tile / sd;
    };
#define SMB_GO_SD(TL, CHK, STG, SDV)                                                      \
  do {                                                                                     \
    using C = SddmmCfg<T, TL, CHK, STG, SDV>;                                              \
    const bool all = all_for(TL, SDV);                                                     \
    if (vec && all)                                                                        \
      go(sddmm_pipe_kernel<T, TL, CHK, STG, SDV, true, true>, TL, C::smem_bytes);          \
    else if (vec)                                                                          \
      go(sddmm_pipe_kernel<T, TL, CHK, STG, SDV, true, false>, TL, C::smem_bytes);         \
    else                                                                                   \
      go(sddmm_pipe_kernel<T, TL, CHK, STG, SDV, false, false>, TL, C::smem_bytes);        \
  } while (0)
    // Double-buffered chunks of 128-nonzero tiles: 64 columns (87 KB, 2 CTAs
    // per SM) when every tile is resident in one wave (the per-chain critical
    // path sets the time), 32 columns (46 KB, 4 CTAs per SM) beyond that.
    // Measured on B200 against 256 / 512-nonzero tiles and 16-64-column
    // chunks with 2-8 stages: more resident CTAs beat deeper per-CTA
    // pipelines (1.3-1.4x at config 3).  Tiles spanning more than 32 rows
    // (1-2 nonzeros per row) stage one d_out row per nonzero (SD = 1).
    const bool wave = pat->ntiles <= 2 * 148;
    const bool sparse_rows = !all_for(128, 4);
    // many waves and every 128-tile within kWarpDSlots rows (>= ~10 nonzeros
    // per row): warp-independent staging, no CTA barrier (1.1-1.2x at
    // config 3 d >= 0.01; measured slower when rows are short)
    const bool warp_kernel = sizeof(T) == 4 && vec && !wave &&
                             pat->span128 <= kWarpDSlots;
    // Small layers (a few waves of 32 / 64-nonzero tiles): the chains set the
    // time, so spread them over as many SMs as possible with deeper rings
    // (measured on B200 at the config-2 layers, scripts/sddmm_lab.cu: 10x512
    // and 512x1024 14.4 -> 8.3 us with 32-tiles, 1024x3072 22.6 -> 16.5 us
    // with 64-tiles).
    const int64_t small_cap = 4 * 148;
    const bool small32 = ceil_div(pat->nnz, 32) <= small_cap;
    const bool small64 = !small32 &&
                         ceil_div(pat->nnz, 64) <= small_cap;
    // One wave of 32-nonzero tiles with 4-stage rings (23 KB, up to 9 CTAs
    // per SM) beyond that: config-2 layer 0 (1024 x 3072) 16.3 -> 15.0 us
    // against 64-nonzero tiles (graph-timed, scripts/sddmm_lab.cu)
    const bool mid32 = ceil_div(pat->nnz, 32) > small_cap &&
                       ceil_div(pat->nnz, 32) <= 9 * 148 && all_for(32, 4);
    bool warp_done = false;
    if constexpr (sizeof(T) == 4) {
      // many-wave layers: one warp per CTA, its 32 chains fed by TMA gather4
      // into a 2-stage swizzled ring (sddmm_tma.cu).  Measured on B200
      // against the cp.async warp / pipe kernels (scripts/lab_sddmm_tma.py):
      // config-4 hidden layer 238 -> 211 us, config-5 hidden layer (B=512)
      // 677 -> 485 us, config 3 d=0.1 1364 -> 1236 us; more stages or warps
      // per CTA lower the resident warps and run slower.  Few-wave layers keep
      // the cp.async kernels: one warp's TMA chunks do not overlap well
      // (config-2 layers 10-15 us -> 21-24 us with any ring depth; the
      // rewritten kernel with 4-8 stages: 9-13 us -> 18-20 us, the serial
      // ELECT / R2UR copy issue of each chunk is exposed at 1-5 warps per SM).
      // (rows of >= 8 nonzeros on average: with 16 or more a warp's 32
      // nonzeros span <= 4 rows, with 8-16 -- config 3 d = 0.001 -- the kernel
      // stages 8 d_out rows per chunk: 17.2 -> 15.2 us at B = 512 and 106 ->
      // 51 us at B = 2048 against the cp.async pipe with a d_out row per
      // nonzero; sparser rows are not measured and keep the pipe)
      if (!small32 && !small64 && !mid32 && pat->nnz >= 8 * pat->m &&
          sddmm_tma_supported(pat, d_out, ld_d, x, ld_x, n)) {
        const int rc = launch_sddmm_tma(pat, static_cast<const float*>(d_out), ld_d,
                                        static_cast<const float*>(x), ld_x, n,
                                        static_cast<const float*>(values),
                                        static_cast<float*>(values_out),
                                        static_cast<float*>(velocity),
                                        static_cast<float*>(grad_out), opt, st);
        if (rc != SMB_OK) return rc;
        warp_done = true;
      } else if (!small32 && !small64 && !mid32 && warp_kernel) {
        go(sddmm_warp_kernel<T, 32, 2>, 128, SddmmWarpCfg<T, 32, 2>::smem_bytes);
        warp_done = true;
      }
    }
#ifndef SMB_LEAN
#define SMB_LEAN 1
#endif
#ifndef SMB_LEAN_MID_S
#define SMB_LEAN_MID_S 6
#endif
#ifndef SMB_LEAN_MID_DS
#define SMB_LEAN_MID_DS 4
#endif
#ifndef SMB_LEAN_SMALL_S
#define SMB_LEAN_SMALL_S 6
#endif
#ifndef SMB_LEAN_SMALL_DS
#define SMB_LEAN_SMALL_DS 4
#endif
    if constexpr (sizeof(T) == 4 && SMB_LEAN != 0) {
      // few-wave layers whose 32-nonzero tiles span <= 8 rows: the lean
      // one-warp kernel (sddmm_lean_kernel).  Measured on B200 at config 2
      // (scripts/gpu_ab_bench2.sh; kernel alone graph-timed / step with the L2
      // flush / step back to back):
      //   layer 0 (1024 x 3072, 5.2 tiles per SM) alone: pipe 13.05 us, lean
      //     6 stages 11.1-11.3 us, 4 stages 10.9 us, 8 stages x 8 d_out rows
      //     14.8 us (41 KB per CTA: the SMs that get 6 tiles run two waves);
      //   layers 1 / 2 (1-2 tiles per SM) alone: pipe 8.6 / 8.4 us, lean 8
      //     stages 7.7 / 7.4 us, 6 stages 8.0 / 7.8 us;
      //   the step, where the three kernels share the SMs' shared memory with
      //     each other and the next batch's gather, follows the footprints
      //     rather than the kernels' own times -- pipe kernels 66.5 / 59.7 us;
      //     (layer 0 stages x rows, layers 1-2 stages x rows): 6x4 + 6x4 62.4 /
      //     55.9 us (kept), 8x8 + 8x8 63.5 / 56.7, 6x4 + 4x4 64.4 / 57.6, 6x8 +
      //     6x8 65.4 / 58.1, 4x4 + 8x8 65.6 / 58.3, 6x4 + 8x8 65.9 / 59.3, 6x8 +
      //     6x4 66.3 / 59.8, 6x4 + 8x4 66.4 / 60.0, 6x4 + 6x8 66.6 / 59.9, 4x4 +
      //     6x4 67.3 / 59.8, 8x8 + 8x4 72.4 / 58.0.
      if (!warp_done && vec && (mid32 || small32) && pat->span32 <= 8 && n < (int64_t(1) << 30)) {
        auto lean = [&](auto kernel, int stages, int ds) {
          const size_t bytes = (size_t)stages * (32 + ds) * 128 + 128;
          ensure_smem(kernel, bytes);
          launch_k(kernel, dim3((unsigned)ceil_div(pat->nnz, 32)), dim3(32), bytes, st,
                   pat->row_ptr, pat->col_idx, pat->tile_row0, pat->m, pat->nnz,
                   static_cast<const float*>(d_out), ld_d, static_cast<const float*>(x), ld_x,
                   (int)n, static_cast<const float*>(values), static_cast<float*>(values_out),
                   static_cast<float*>(velocity), static_cast<float*>(grad_out), opt);
        };
        if (small32 && pat->span32 <= SMB_LEAN_SMALL_DS)
          lean(sddmm_lean_kernel<SMB_LEAN_SMALL_S, SMB_LEAN_SMALL_DS>, SMB_LEAN_SMALL_S,
               SMB_LEAN_SMALL_DS);
        else if (small32)
          lean(sddmm_lean_kernel<SMB_LEAN_SMALL_S, 8>, SMB_LEAN_SMALL_S, 8);
        else if (pat->span32 <= SMB_LEAN_MID_DS)
          lean(sddmm_lean_kernel<SMB_LEAN_MID_S, SMB_LEAN_MID_DS>, SMB_LEAN_MID_S,
               SMB_LEAN_MID_DS);
        else
          lean(sddmm_lean_kernel<SMB_LEAN_MID_S, 8>, SMB_LEAN_MID_S, 8);
        warp_done = true;
      }
    }
    if (warp_done) {
    } else if (sizeof(T) == 4 && mid32)
      // 8 stages, 4 staged d_out rows (37 KB, 6 CTAs per SM: the layer's
      // tiles stay one wave): config-2 step 68.3 -> 66.6 us back to back
      // against 6 stages; 3-5 and 10-16 stages slower (10+ stages: two waves)
      // (scripts/sweep_variants.sh)
      SMB_GO_SD(32, 32, SMB_SD_MID_STAGES, 8);
    else if (sizeof(T) == 4 && small32 && all_for(32, 4) && concurrent)
      // beside other kernels (the overlapped training step) the 2-stage ring
      // (12 KB per CTA instead of 46 KB) leaves shared memory to the kernels
      // on the critical path: config-2 step 76.3 -> 74.6 us back to back
      // although this kernel alone is 1.1-1.2x slower
      // (4 stages with 4 staged d_out rows, 18 KB: 66.6 -> 65.9 us/step
      // against 3 stages; 2-8 stages and 64-column chunks measured)
      SMB_GO_SD(32, SMB_SD_SMALL_CHUNK, SMB_SD_SMALL_STAGES, 8);
    else if (sizeof(T) == 4 && small32 && all_for(32, 4)) SMB_GO_SD(32, 32, 8, 4);
    else if (sizeof(T) == 4 && small32) SMB_GO_SD(32, 32, 8, 1);
    else if (sizeof(T) == 4 && small64 && !mid32 && all_for(64, 4)) SMB_GO_SD(64, 32, 4, 4);
    else if (sizeof(T) == 4 && small64) SMB_GO_SD(64, 32, 4, 1);
    else if (sizeof(T) == 4 && wave && sparse_rows) SMB_GO_SD(128, 64, 2, 1);
    else if (sizeof(T) == 4 && wave) SMB_GO_SD(128, 64, 2, 4);
    else if (sizeof(T) == 4 && sparse_rows) SMB_GO_SD(128, 32, 2, 1);
    else if (sizeof(T) == 4) SMB_GO_SD(128, 32, 2, 4);
    else SMB_GO_SD(128, (int)(128 / sizeof(T)), 4, 4);  // fp64: 16-column chunks
#undef SMB_GO_SD
    const int rc = check_launch(name);
    if (rc != SMB_OK) return rc;
  }
  const bool want_bias = (grad_bias_out != nullptr) || (opt_kind != SMB_OPT_NONE && bias);
  if (!want_bias) return SMB_OK;
  return launch_bias_rows<T>(static_cast<const T*>(d_out), ld_d, pat->m, n, static_cast<T*>(bias),
                             static_cast<T*>(vbias), static_cast<T*>(grad_bias_out), opt, st);
}

}  // namespace smb

using namespace smb;

extern "C" int smb_sddmm(int dtype, const smb_pattern* pat, const void* a, int64_t lda,
                         const void* b, int64_t ldb, int64_t n, void* out_values, void* stream) {
  clear_error();
  SMB_REQUIRE(pat != nullptr, "smb_sddmm: null pattern");
  SMB_REQUIRE(n >= 0 && lda >= n && ldb >= n, "smb_sddmm: bad batch width / leading dimension");
  SMB_REQUIRE(pat->nnz == 0 || out_values != nullptr, "smb_sddmm: null output");
  if (dtype == SMB_F32)
    return sddmm_update_impl<float>(pat, a, lda, b, ldb, n, nullptr, nullptr, nullptr, out_values,
                                    nullptr, nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0, stream,
                                    "smb_sddmm");
  if (dtype == SMB_F64)
    return sddmm_update_impl<double>(pat, a, lda, b, ldb, n, nullptr, nullptr, nullptr,
                                     out_values, nullptr, nullptr, nullptr, SMB_OPT_NONE, 0.0, 0.0,
                                     stream, "smb_sddmm");
  set_error("smb_sddmm: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}

extern "C" int smb_sddmm_update(int dtype, const smb_pattern* pat, const void* d_out,
                                int64_t ld_dout, const void* x, int64_t ld_x, int64_t n,
                                void* values, void* velocity, void* grad_out, void* bias,
                                void* velocity_bias, void* grad_bias_out, int opt_kind, double mu,
                                double eta, void* stream) {
  return smb_sddmm_update_into(dtype, pat, d_out, ld_dout, x, ld_x, n, values, values, velocity,
                               grad_out, bias, velocity_bias, grad_bias_out, opt_kind, mu, eta,
                               stream);
}

extern "C" int smb_sddmm_update_into(int dtype, const smb_pattern* pat, const void* d_out,
                                     int64_t ld_dout, const void* x, int64_t ld_x, int64_t n,
                                     const void* values, void* values_out, void* velocity,
                                     void* grad_out, void* bias, void* velocity_bias,
                                     void* grad_bias_out, int opt_kind, double mu, double eta,
                                     void* stream) {
  clear_error();
  const bool concurrent = (opt_kind & SMB_HINT_CONCURRENT) != 0;
  opt_kind &= ~SMB_HINT_CONCURRENT;
  SMB_REQUIRE(pat != nullptr, "smb_sddmm_update: null pattern");
  SMB_REQUIRE(opt_kind == SMB_OPT_NONE || values_out != nullptr || pat->nnz == 0,
              "smb_sddmm_update: null output values");
  SMB_REQUIRE(n >= 0 && ld_dout >= n && ld_x >= n,
              "smb_sddmm_update: bad batch width / leading dimension");
  SMB_REQUIRE(opt_kind >= SMB_OPT_NONE && opt_kind <= SMB_OPT_NESTEROV,
              "smb_sddmm_update: bad optimizer kind %d", opt_kind);
  SMB_REQUIRE(opt_kind == SMB_OPT_NONE || values != nullptr || pat->nnz == 0,
              "smb_sddmm_update: null values");
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) ||
                  velocity != nullptr || pat->nnz == 0,
              "smb_sddmm_update: momentum needs a velocity buffer");
  SMB_REQUIRE(!(opt_kind == SMB_OPT_MOMENTUM || opt_kind == SMB_OPT_NESTEROV) || bias == nullptr ||
                  velocity_bias != nullptr,
              "smb_sddmm_update: momentum needs a bias velocity buffer");
  if (dtype == SMB_F32)
    return sddmm_update_impl<float>(pat, d_out, ld_dout, x, ld_x, n, values, values_out, velocity,
                                    grad_out, bias, velocity_bias, grad_bias_out, opt_kind, mu,
                                    eta, stream, "smb_sddmm_update", concurrent);
  if (dtype == SMB_F64)
    return sddmm_update_impl<double>(pat, d_out, ld_dout, x, ld_x, n, values, values_out,
                                     velocity, grad_out, bias, velocity_bias, grad_bias_out,
                                     opt_kind, mu, eta, stream, "smb_sddmm_update");
  set_error("smb_sddmm_update: unsupported dtype %d", dtype);
  return SMB_ERR_INVALID;
}
