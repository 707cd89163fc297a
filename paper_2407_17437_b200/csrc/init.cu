// Device Xavier-uniform init, bit-identical to sparsity.xavier_init
// (sparsity.py:223-237) for numpy's PCG64 stream.
//
// numpy's PCG64 is PCG XSL-RR 128/64: state <- state * M + inc (mod 2^128),
// output = rotr64(hi ^ lo, hi >> 58) of the NEW state.  Generator.uniform(low,
// high) draws next_double = (x >> 11) * 2^-53 and returns low + (high-low) *
// next_double in float64 (here low = -a, high - low = 2a exactly); xavier_init
// then casts to the value dtype.  Every thread jumps its own copy of the
// generator ahead with the O(log n) LCG jump (Brown, "Random number generation
// with arbitrary strides"), so the stream is produced fully in parallel.
#include "common.cuh"

namespace smb {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const uint64_t x = hi ^ lo;
  const unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int kPerThread = 32;

template <typename T>
__global__ void xavier_kernel(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                              uint64_t offset, int64_t count, double limit, T* __restrict__ out) {
  const int64_t first = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kPerThread;
  if (first >= count) return;
  const u128 inc = ((u128)i_hi << 64) | i_lo;
  u128 st = pcg_advance(((u128)s_hi << 64) | s_lo, inc, offset + (uint64_t)first);
  const u128 mult = pcg_mult();
  const double scale = __dmul_rn(2.0, limit);  // high - low = a - (-a), exact
  const int64_t last = imin(count, first + kPerThread);
  for (int64_t p = first; p < last; ++p) {
    st = st * mult + inc;
    const double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
    out[p] = static_cast<T>(__dadd_rn(-limit, __dmul_rn(scale, u)));
  }
}

}  // namespace
}  // namespace smb

using namespace smb;

extern "C" int smb_xavier_pcg64(int dtype, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                uint64_t inc_lo, uint64_t offset, int64_t count, double limit,
                                void* out, void* stream) {
  clear_error();
  SMB_REQUIRE(count >= 0, "smb_xavier_pcg64: negative count");
  if (count == 0) return SMB_OK;
  SMB_REQUIRE(out != nullptr, "smb_xavier_pcg64: null output");
  const int64_t threads = ceil_div(count, kPerThread);
  const unsigned blocks = (unsigned)ceil_div(threads, 128);
  if (dtype == SMB_F32) {
    xavier_kernel<float><<<blocks, 128, 0, as_stream(stream)>>>(
        state_hi, state_lo, inc_hi, inc_lo, offset, count, limit, static_cast<float*>(out));
  } else if (dtype == SMB_F64) {
    xavier_kernel<double><<<blocks, 128, 0, as_stream(stream)>>>(
        state_hi, state_lo, inc_hi, inc_lo, offset, count, limit, static_cast<double*>(out));
  } else {
    set_error("smb_xavier_pcg64: unsupported dtype %d", dtype);
    return SMB_ERR_INVALID;
  }
  return check_launch("smb_xavier_pcg64");
}
