/*
 * csr_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the four CSR kernels of the reference package
 * sparsemlp (pkg/src/sparsemlp/_kernels.py), used by tests/ as the parity
 * oracle for the CUDA path and by bench.py as the reference arm / CPU
 * baseline ("port").  Each function follows its reference kernel in
 * ARITHMETIC ORDER (ascending source index, multiply and add rounded
 * separately: built with -ffp-contract=off, never -ffast-math) and in
 * PARALLEL STRUCTURE (one task per output row / block / entry, split
 * statically over host threads like numba's prange), so its cost model tracks
 * the reference's CPU path as well as its results.
 *
 * Pinned against the reference itself: tests/golden/ holds outputs of the
 * reference run in the build container (tests/golden/make_golden.py) and
 * tests/test_oracle_golden.py checks this file against them bit for bit.
 */
#include <pthread.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#define ORC_API __attribute__((visibility("default")))
#define MAX_THREADS 256

static int g_threads = 0;

ORC_API int orc_max_threads(void) {
  if (g_threads <= 0) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    g_threads = n < 1 ? 1 : (n > MAX_THREADS ? MAX_THREADS : (int)n);
  }
  return g_threads;
}

ORC_API void orc_set_threads(int n) {
  if (n > 0) g_threads = n > MAX_THREADS ? MAX_THREADS : n;
}

/* static partition of [0, n) over the thread count, like prange */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
struct task { range_fn fn; void* ctx; int64_t lo, hi; };

static void* run_task(void* p) {
  struct task* t = (struct task*)p;
  t->fn(t->ctx, t->lo, t->hi);
  return NULL;
}

static void par_for(int64_t n, range_fn fn, void* ctx) {
  int nt = orc_max_threads();
  if (nt > n) nt = (int)(n > 0 ? n : 1);
  if (nt <= 1) { fn(ctx, 0, n); return; }
  pthread_t th[MAX_THREADS];
  struct task tk[MAX_THREADS];
  for (int i = 0; i < nt; ++i) {
    tk[i].fn = fn; tk[i].ctx = ctx;
    tk[i].lo = n * i / nt; tk[i].hi = n * (i + 1) / nt;
  }
  for (int i = 1; i < nt; ++i) pthread_create(&th[i], NULL, run_task, &tk[i]);
  run_task(&tk[0]);
  for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
}

/* ---- spmm: _kernels.py:25-37 (out zero-initialised, tensor_core.py:237) ----
 * out[i, j] += v * dense[c, j] over p in row i ascending; one task per row. */
#define DEF_SPMM(T, SUF)                                                               \
  struct spmm_ctx_##SUF { const int32_t *rp, *ci; const T *v, *d; int64_t n; T* out; }; \
  static void spmm_rows_##SUF(void* vc, int64_t lo, int64_t hi) {                      \
    struct spmm_ctx_##SUF* c = (struct spmm_ctx_##SUF*)vc;                             \
    for (int64_t i = lo; i < hi; ++i) {                                                \
      T* o = c->out + i * c->n;                                                        \
      for (int64_t j = 0; j < c->n; ++j) o[j] = (T)0;                                  \
      for (int32_t p = c->rp[i]; p < c->rp[i + 1]; ++p) {                              \
        const T v = c->v[p];                                                           \
        const T* d = c->d + (int64_t)c->ci[p] * c->n;                                  \
        for (int64_t j = 0; j < c->n; ++j) { const T prod = v * d[j]; o[j] = o[j] + prod; } \
      }                                                                                \
    }                                                                                  \
  }                                                                                    \
  ORC_API void orc_spmm_##SUF(const int32_t* row_ptr, const int32_t* col_idx,          \
                              const T* values, int64_t m, const T* dense, int64_t n,   \
                              T* out) {                                                \
    struct spmm_ctx_##SUF c = {row_ptr, col_idx, values, dense, n, out};               \
    par_for(m, spmm_rows_##SUF, &c);                                                   \
  }
DEF_SPMM(float, f32)
DEF_SPMM(double, f64)

/* ---- spmm_t: _kernels.py:40-59 (nblocks = min(threads, ncols),
 * tensor_core.py:253).  Block b owns output rows [b*k/nb, (b+1)*k/nb) and
 * scans the whole matrix in row order, so out[c, :] accumulates in ascending
 * source row regardless of nblocks. */
#define DEF_SPMM_T(T, SUF)                                                             \
  struct spmmt_ctx_##SUF {                                                             \
    const int32_t *rp, *ci; const T *v, *d; int64_t m, k, n, nb; T* out; };            \
  static void spmmt_blocks_##SUF(void* vc, int64_t blo, int64_t bhi) {                 \
    struct spmmt_ctx_##SUF* c = (struct spmmt_ctx_##SUF*)vc;                           \
    for (int64_t b = blo; b < bhi; ++b) {                                              \
      const int64_t lo = b * c->k / c->nb, hi = (b + 1) * c->k / c->nb;                \
      for (int64_t i = 0; i < c->m; ++i) {                                             \
        for (int32_t p = c->rp[i]; p < c->rp[i + 1]; ++p) {                            \
          const int64_t col = c->ci[p];                                                \
          if (lo <= col && col < hi) {                                                 \
            const T v = c->v[p];                                                       \
            const T* d = c->d + i * c->n;                                              \
            T* o = c->out + col * c->n;                                                \
            for (int64_t j = 0; j < c->n; ++j) { const T prod = v * d[j]; o[j] = o[j] + prod; } \
          }                                                                            \
        }                                                                              \
      }                                                                                \
    }                                                                                  \
  }                                                                                    \
  ORC_API void orc_spmm_t_##SUF(const int32_t* row_ptr, const int32_t* col_idx,        \
                                const T* values, int64_t m, int64_t k, const T* dense, \
                                int64_t n, T* out, int64_t nblocks) {                  \
    memset(out, 0, sizeof(T) * (size_t)(k * n));                                      \
    struct spmmt_ctx_##SUF c = {row_ptr, col_idx, values, dense, m, k, n, nblocks, out}; \
    par_for(nblocks, spmmt_blocks_##SUF, &c);                                          \
  }
DEF_SPMM_T(float, f32)
DEF_SPMM_T(double, f64)

/* ---- sddmm: _kernels.py:62-75.  acc = a[i,0]*b[j,0]; acc += a[i,t]*b[j,t]
 * for t = 1..kk-1; one task per row.  kk == 0 -> zeros (tensor_core.py:283). */
#define DEF_SDDMM(T, SUF)                                                              \
  struct sddmm_ctx_##SUF { const int32_t *rp, *ci; const T *a, *b; int64_t kk; T* out; }; \
  static void sddmm_rows_##SUF(void* vc, int64_t lo, int64_t hi) {                     \
    struct sddmm_ctx_##SUF* c = (struct sddmm_ctx_##SUF*)vc;                           \
    for (int64_t i = lo; i < hi; ++i) {                                                \
      const T* ar = c->a + i * c->kk;                                                  \
      for (int32_t p = c->rp[i]; p < c->rp[i + 1]; ++p) {                              \
        if (c->kk == 0) { c->out[p] = (T)0; continue; }                                \
        const T* br = c->b + (int64_t)c->ci[p] * c->kk;                                \
        T acc = ar[0] * br[0];                                                         \
        for (int64_t t = 1; t < c->kk; ++t) { const T prod = ar[t] * br[t]; acc = acc + prod; } \
        c->out[p] = acc;                                                               \
      }                                                                                \
    }                                                                                  \
  }                                                                                    \
  ORC_API void orc_sddmm_##SUF(const int32_t* row_ptr, const int32_t* col_idx,         \
                               int64_t m, const T* a, const T* b, int64_t kk,          \
                               T* out_values) {                                        \
    struct sddmm_ctx_##SUF c = {row_ptr, col_idx, a, b, kk, out_values};               \
    par_for(m, sddmm_rows_##SUF, &c);                                                  \
  }
DEF_SDDMM(float, f32)
DEF_SDDMM(double, f64)

/* ---- axpby: _kernels.py:78-83, alpha/beta already in the value dtype ----- */
#define DEF_AXPBY(T, SUF)                                                              \
  struct axpby_ctx_##SUF { T alpha, beta; T* s; const T* t; };                         \
  static void axpby_range_##SUF(void* vc, int64_t lo, int64_t hi) {                    \
    struct axpby_ctx_##SUF* c = (struct axpby_ctx_##SUF*)vc;                           \
    for (int64_t p = lo; p < hi; ++p) {                                                \
      const T x = c->alpha * c->s[p];                                                  \
      const T y = c->beta * c->t[p];                                                   \
      c->s[p] = x + y;                                                                 \
    }                                                                                  \
  }                                                                                    \
  ORC_API void orc_axpby_##SUF(T alpha, T* s, T beta, const T* t, int64_t n) {         \
    struct axpby_ctx_##SUF c = {alpha, beta, s, t};                                    \
    par_for(n, axpby_range_##SUF, &c);                                                 \
  }
DEF_AXPBY(float, f32)
DEF_AXPBY(double, f64)

/* ---- numpy pairwise summation (row_sums, tensor_core.py:353-356) --------- */
#define DEF_PAIRWISE(T, SUF)                                                           \
  static T pairwise_##SUF(const T* a, int64_t n) {                                     \
    if (n < 8) {                                                                       \
      T res = (T)0;                                                                    \
      for (int64_t i = 0; i < n; ++i) res = res + a[i];                                \
      return res;                                                                      \
    }                                                                                  \
    if (n <= 128) {                                                                    \
      T r[8];                                                                          \
      for (int j = 0; j < 8; ++j) r[j] = a[j];                                         \
      int64_t i;                                                                       \
      for (i = 8; i < n - (n % 8); i += 8)                                             \
        for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];                            \
      T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));       \
      for (; i < n; ++i) res = res + a[i];                                             \
      return res;                                                                      \
    }                                                                                  \
    int64_t n2 = n / 2;                                                                \
    n2 -= n2 % 8;                                                                      \
    return pairwise_##SUF(a, n2) + pairwise_##SUF(a + n2, n - n2);                     \
  }                                                                                    \
  struct rows_ctx_##SUF { const T* a; int64_t n; T* out; };                            \
  static void rows_range_##SUF(void* vc, int64_t lo, int64_t hi) {                     \
    struct rows_ctx_##SUF* c = (struct rows_ctx_##SUF*)vc;                             \
    for (int64_t i = lo; i < hi; ++i) c->out[i] = pairwise_##SUF(c->a + i * c->n, c->n); \
  }                                                                                    \
  ORC_API void orc_row_sums_##SUF(const T* a, int64_t m, int64_t n, T* out) {          \
    struct rows_ctx_##SUF c = {a, n, out};                                             \
    par_for(m, rows_range_##SUF, &c);                                                  \
  }
DEF_PAIRWISE(float, f32)
DEF_PAIRWISE(double, f64)
