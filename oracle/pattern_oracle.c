/*
 * pattern_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the device pattern sampler's specification
 * (paper_2407_17437_b200/csrc/sampler.cu, "scale mode"): candidates
 * pos_i = floor(Philox4x32-10(seed, (i, stream_id)) * G / 2^64) over the
 * G = m * k grid, the pattern = the first nnz distinct candidates (or, when
 * nnz > G / 2, every position except the first G - nnz distinct ones),
 * CSR in row-major order.  Written independently of the CUDA code: a
 * sequential walk of the candidate stream with an open-addressing hash set
 * instead of the device's sort / select passes.  The reference's own host
 * sampler (sparsity.py:183-216) draws from the same distribution -- a
 * uniformly random nnz-subset of the grid -- with numpy's stream; tests/
 * check the distribution against it statistically.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

static void philox_round(uint32_t c[4], uint32_t k0, uint32_t k1) {
  uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
  uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
  c[1] = (uint32_t)p1;
  c[3] = (uint32_t)p0;
  c[0] = n0;
  c[2] = n2;
}

ORC_API uint64_t orc_philox_u64(uint64_t seed, uint64_t sid, uint64_t i) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)sid, (uint32_t)(sid >> 32)};
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ((uint64_t)c[1] << 32) | c[0];
}

static uint64_t mulhi64(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* the first `need` distinct candidates, ascending; returns 0 on success */
static int first_distinct(uint64_t G, int64_t need, uint64_t seed, uint64_t sid, uint64_t* out) {
  uint64_t cap = 1;
  while (cap < (uint64_t)need * 2 + 16) cap <<= 1;
  uint64_t* table = malloc(cap * sizeof(uint64_t)); /* stores pos + 1; 0 = empty */
  if (!table) return -1;
  memset(table, 0, cap * sizeof(uint64_t));
  int64_t got = 0;
  for (uint64_t i = 0; got < need; ++i) {
    uint64_t p = mulhi64(orc_philox_u64(seed, sid, i), G);
    uint64_t h = (p * 0x9E3779B97F4A7C15ull) & (cap - 1);
    for (;;) {
      if (table[h] == 0) {
        table[h] = p + 1;
        out[got++] = p;
        break;
      }
      if (table[h] == p + 1) break; /* seen: rejected */
      h = (h + 1) & (cap - 1);
    }
  }
  free(table);
  qsort(out, (size_t)need, sizeof(uint64_t), cmp_u64);
  return 0;
}

ORC_API int orc_sample_pattern(int64_t m, int64_t k, int64_t nnz, uint64_t seed, uint64_t sid,
                               int32_t* row_ptr, int32_t* col_idx) {
  uint64_t G = (uint64_t)m * (uint64_t)k;
  if (nnz < 0 || (uint64_t)nnz > G) return -1;
  int complement = nnz > 0 && (uint64_t)nnz * 2 > G;
  int64_t need = complement ? (int64_t)(G - (uint64_t)nnz) : nnz;
  uint64_t* drawn = malloc((size_t)(need > 0 ? need : 1) * sizeof(uint64_t));
  if (!drawn || first_distinct(G, need, seed, sid, drawn)) return -1;
  for (int64_t r = 0; r <= m; ++r) row_ptr[r] = 0;
  int64_t q = 0;
  if (!complement) {
    for (int64_t e = 0; e < nnz; ++e) {
      col_idx[e] = (int32_t)(drawn[e] % (uint64_t)k);
      row_ptr[drawn[e] / (uint64_t)k + 1]++;
    }
  } else {
    int64_t d = 0;
    for (uint64_t p = 0; p < G; ++p) {
      if (d < need && drawn[d] == p) { ++d; continue; }
      col_idx[q++] = (int32_t)(p % (uint64_t)k);
      row_ptr[p / (uint64_t)k + 1]++;
    }
  }
  for (int64_t r = 0; r < m; ++r) row_ptr[r + 1] += row_ptr[r];
  free(drawn);
  return 0;
}
