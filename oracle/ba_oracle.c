/* TEST INFRASTRUCTURE: plain-C restatement of the reference's Barabasi-Albert
 * generator, graphrl.generate_ba (pkg/src/graphrl/graphs.py:125-157), used
 * where the reference's own pure-Python loop (216 s at BA(2M,16)) is too
 * slow: the --impl reference arm of bench.py builds its input graph with it,
 * so that process never maps the product library libs2v.so.  The edge
 * arrays are pinned byte for byte against the reference by
 * tests/test_oracle.py (tests/golden/generators.json).
 *
 * Draw sequence restated from numpy 2.x:
 *   default_rng(seed) -> PCG64 (128-bit LCG, XSL-RR output), state taken
 *     from numpy's SeedSequence by the caller (bit_generator.state);
 *   Generator.integers(0, len) with len < 2^32 -> Lemire's bounded method on
 *     the buffered 32-bit stream (low half of a 64-bit output first, the
 *     high half kept for the next call).
 * Algorithm (graphs.py:137-156): a d-clique, node d joins all of it, every
 * later node draws repeated[integers(len(repeated))] until d distinct
 * targets; edges (t, node) appended in ascending t.  Output: the sorted
 * (u < v) int64 edge array of Graph(n, edges). */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
  u128 s, inc;
  int have_hi;
  uint32_t hi;
} pcg_t;

static uint64_t pcg_out(pcg_t *g) {
  const u128 mul = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
  g->s = g->s * mul + g->inc;
  const uint64_t x = (uint64_t)(g->s >> 64) ^ (uint64_t)g->s;
  const unsigned r = (unsigned)(g->s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}

static uint32_t pcg_u32(pcg_t *g) {
  if (g->have_hi) {
    g->have_hi = 0;
    return g->hi;
  }
  const uint64_t w = pcg_out(g);
  g->hi = (uint32_t)(w >> 32);
  g->have_hi = 1;
  return (uint32_t)w;
}

static uint32_t lemire(pcg_t *g, uint32_t n) { /* integers(0, n), 1 <= n < 2^32 */
  if (n == 1) return 0;
  uint64_t m = (uint64_t)pcg_u32(g) * n;
  if ((uint32_t)m < n) {
    const uint32_t floor = (uint32_t)(-n) % n;
    while ((uint32_t)m < floor) m = (uint64_t)pcg_u32(g) * n;
  }
  return (uint32_t)(m >> 32);
}

static int cmp_i32(const void *a, const void *b) {
  const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* pcg = {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger};
 * edges NULL: return the edge count; else fill [E][2] int64 sorted. */
int64_t s2vo_generate_ba(int64_t n, int64_t d, const uint64_t *pcg, int64_t *edges) {
  if (d < 1 || n <= d) return -1;
  const int64_t E = d * (d - 1) / 2 + d * (n - d);
  if (!edges) return E;
  if (2 * E >= (int64_t)UINT32_MAX) return -1;
  pcg_t g = {((u128)pcg[0] << 64) | pcg[1], ((u128)pcg[2] << 64) | pcg[3], (int)pcg[4],
             (uint32_t)pcg[5]};
  int32_t *rep = (int32_t *)malloc(sizeof(int32_t) * 2 * E);
  int64_t *deg = (int64_t *)calloc(n + 1, sizeof(int64_t));
  int32_t *pick = (int32_t *)malloc(sizeof(int32_t) * d);
  if (!rep || !deg || !pick) {
    free(rep), free(deg), free(pick);
    return -1;
  }
  int64_t nr = 0;
  for (int64_t i = 0; i < d; i++)
    for (int64_t j = i + 1; j < d; j++) rep[nr++] = (int32_t)i, rep[nr++] = (int32_t)j;
  for (int64_t v = d; v < n; v++) {
    int64_t c = 0;
    if (v == d) {
      for (; c < d; c++) pick[c] = (int32_t)c;
    } else {
      while (c < d) {
        const int32_t t = rep[lemire(&g, (uint32_t)nr)];
        int64_t q = 0;
        while (q < c && pick[q] != t) q++;
        if (q == c) pick[c++] = t;
      }
      qsort(pick, (size_t)d, sizeof(int32_t), cmp_i32);
    }
    for (int64_t q = 0; q < d; q++) rep[nr++] = pick[q], rep[nr++] = (int32_t)v;
  }
  /* rep holds every edge as (u, v) with u < v: clique pairs, then (t, node).
   * Sort lexicographically with a counting sort on u (v ascends within a u:
   * clique v's ascend, and later edges of u come from increasing nodes). */
  for (int64_t e = 0; e < E; e++) deg[rep[2 * e] + 1]++;
  for (int64_t u = 0; u < n; u++) deg[u + 1] += deg[u];
  for (int64_t e = 0; e < E; e++) {
    const int64_t p = deg[rep[2 * e]]++;
    edges[2 * p] = rep[2 * e];
    edges[2 * p + 1] = rep[2 * e + 1];
  }
  free(rep), free(deg), free(pick);
  return E;
}
