// Native graph ingestion (host code): a Barabasi-Albert generator that
// reproduces the reference's numpy draw sequence bit for bit.
//
// Replaces generate_ba (pkg/src/graphrl/graphs.py:125-157), which draws each
// target with Generator.integers(len(repeated)) on a PCG64 stream.  numpy's
// bounded draw for ranges < 2^32 is Lemire's method on the bit generator's
// buffered 32-bit output (PCG64 next_uint32: low half of a 64-bit draw, high
// half kept for the next call); that is reproduced here from the bit
// generator state numpy's SeedSequence produced (passed in by the host).
// Output: the E = C(d,2) + d(n-d) edges (u < v), lexicographically sorted,
// exactly Graph(n, edges).edge_array of the reference.
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Pcg64 {
  unsigned __int128 state, inc;
  int has32;
  uint32_t u32;
  uint64_t next64() {
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  // jump ahead by delta steps (PCG's LCG advance, O(log delta))
  void advance(unsigned __int128 delta) {
    unsigned __int128 cur_mult =
        ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    unsigned __int128 cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
      if (delta & 1) {
        acc_mult *= cur_mult;
        acc_plus = acc_plus * cur_mult + cur_plus;
      }
      cur_plus = (cur_mult + 1) * cur_plus;
      cur_mult *= cur_mult;
      delta >>= 1;
    }
    state = acc_mult * state + acc_plus;
  }
  double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    uint64_t n = next64();
    has32 = 1;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
  // Generator.integers(0, n) for 1 <= n <= 2^32 - 1 (numpy random_bounded_uint64_fill)
  uint64_t bounded(uint64_t n) {
    uint32_t rng = (uint32_t)(n - 1);
    if (rng == 0) return 0;
    uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      uint32_t th = (UINT32_MAX - rng) % excl;
      while (left < th) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return m >> 32;
  }
};

}  // namespace

extern "C" {

// pcg: {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}.
// edges_out: NULL to query the edge count, else [E][2] int64.  Returns E or -1.
int64_t s2v_generate_ba(int64_t n, int64_t d, const void *pcg, void *edges_out) {
  if (d < 1 || n <= d) return -1;
  const int64_t E = d * (d - 1) / 2 + d * (n - d);
  if (!edges_out) return E;
  const uint64_t *p = (const uint64_t *)pcg;
  Pcg64 g;
  g.state = ((unsigned __int128)p[0] << 64) | p[1];
  g.inc = ((unsigned __int128)p[2] << 64) | p[3];
  g.has32 = (int)p[4];
  g.u32 = (uint32_t)p[5];
  if (2 * E >= (int64_t)UINT32_MAX) return -1;
  std::vector<int32_t> eu, ev;
  eu.reserve(E);
  ev.reserve(E);
  std::vector<int32_t> repeated;
  repeated.reserve(2 * E);
  for (int64_t i = 0; i < d; i++)
    for (int64_t j = i + 1; j < d; j++) {
      eu.push_back((int32_t)i);
      ev.push_back((int32_t)j);
      repeated.push_back((int32_t)i);
      repeated.push_back((int32_t)j);
    }
  std::vector<int32_t> chosen(d);
  for (int64_t node = d; node < n; node++) {
    int64_t cnt = 0;
    if (node == d) {
      for (int64_t t = 0; t < d; t++) chosen[cnt++] = (int32_t)t;
    } else {
      while (cnt < d) {
        int32_t t = repeated[g.bounded(repeated.size())];
        bool dup = false;
        for (int64_t q = 0; q < cnt; q++)
          if (chosen[q] == t) {
            dup = true;
            break;
          }
        if (!dup) chosen[cnt++] = t;
      }
      // sorted(chosen): insertion sort (d is small)
      for (int64_t a = 1; a < cnt; a++) {
        int32_t x = chosen[a];
        int64_t b = a - 1;
        while (b >= 0 && chosen[b] > x) {
          chosen[b + 1] = chosen[b];
          b--;
        }
        chosen[b + 1] = x;
      }
    }
    for (int64_t q = 0; q < cnt; q++) {
      eu.push_back(chosen[q]);
      ev.push_back((int32_t)node);
      repeated.push_back(chosen[q]);
      repeated.push_back((int32_t)node);
    }
  }
  // stable counting sort by u: v's of a fixed u already appear ascending
  std::vector<int64_t> start(n + 1, 0);
  for (int64_t e = 0; e < E; e++) start[eu[e] + 1]++;
  for (int64_t u = 0; u < n; u++) start[u + 1] += start[u];
  int64_t *out = (int64_t *)edges_out;
  for (int64_t e = 0; e < E; e++) {
    int64_t pos = start[eu[e]]++;
    out[2 * pos] = eu[e];
    out[2 * pos + 1] = ev[e];
  }
  return E;
}

// R-MAT (Graph500 quadrant descent, no label permutation), the definition of
// paper_2105_08764_b200.graphs.generate_rmat (BASELINE cfg5; the reference has
// no R-MAT generator): edge_factor * 2^scale draws in chunks of `chunk`; per
// chunk and level one Generator.random(m) vector (next_double); symmetrised,
// self-loops dropped, duplicates removed; output sorted (u < v).
// edges_out must hold edge_factor * 2^scale pairs.  Returns E or -1.
int64_t s2v_generate_rmat(int scale, int64_t edge_factor, const void *pcg, double a, double b,
                          double c, int64_t chunk, void *edges_out) {
  if (scale < 1 || scale > 30 || edge_factor < 1 || chunk < 1) return -1;
  const uint64_t *p = (const uint64_t *)pcg;
  Pcg64 g;
  g.state = ((unsigned __int128)p[0] << 64) | p[1];
  g.inc = ((unsigned __int128)p[2] << 64) | p[3];
  g.has32 = (int)p[4];
  g.u32 = (uint32_t)p[5];
  const int64_t n = (int64_t)1 << scale;
  const int64_t total = edge_factor * n;
  const double ab = a + b, abc = a + b + c;
  // Draw j of a chunk (level-major: j = level*m + i) is the (j+1)-th output
  // after the chunk's starting state, so the draws split across threads by
  // jumping the generator ahead; the sequence is identical to one thread's.
  std::vector<int64_t> keys;
  keys.reserve(total);
  std::vector<int64_t> u, v;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 64) nt = 64;
  for (int64_t done = 0; done < total; done += chunk) {
    const int64_t m = std::min(chunk, total - done);
    u.assign(m, 0);
    v.assign(m, 0);
    const int64_t per = (m + nt - 1) / nt;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; t++) {
      const int64_t i0 = t * per, i1 = std::min<int64_t>(m, i0 + per);
      if (i0 >= i1) break;
      th.emplace_back([&, i0, i1]() {
        for (int level = 0; level < scale; level++) {
          Pcg64 gl = g;
          gl.advance((unsigned __int128)level * m + i0);
          const int64_t bit = (int64_t)1 << (scale - 1 - level);
          for (int64_t i = i0; i < i1; i++) {
            const double r = gl.next_double();
            const bool right = (r >= a && r < ab) || (r >= abc);
            const bool down = r >= ab;
            if (down) u[i] += bit;
            if (right) v[i] += bit;
          }
        }
      });
    }
    for (auto &x : th) x.join();
    g.advance((unsigned __int128)scale * m);
    for (int64_t i = 0; i < m; i++) {
      if (u[i] == v[i]) continue;
      const int64_t lo = std::min(u[i], v[i]), hi = std::max(u[i], v[i]);
      keys.push_back(lo * n + hi);
    }
  }
  // LSD radix sort of the keys (< 2^(2*scale)), 11 bits per pass
  {
    std::vector<int64_t> tmp(keys.size());
    const int bits = 2 * scale;
    for (int shift = 0; shift < bits; shift += 11) {
      std::vector<int64_t> cnt(2049, 0);
      for (int64_t k : keys) cnt[((k >> shift) & 2047) + 1]++;
      for (int q = 0; q < 2048; q++) cnt[q + 1] += cnt[q];
      for (int64_t k : keys) tmp[cnt[(k >> shift) & 2047]++] = k;
      keys.swap(tmp);
    }
  }
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  int64_t *out = (int64_t *)edges_out;
  for (size_t i = 0; i < keys.size(); i++) {
    out[2 * i] = keys[i] / n;
    out[2 * i + 1] = keys[i] % n;
  }
  return (int64_t)keys.size();
}

// Symmetric CSR of a sorted unique (u < v) edge list: one pass in edge order
// appends v to row u and u to row v, which leaves every row ascending (all
// (x, w) edges with x < w precede the (w, y) edges).  row_ptr[n+1] int64,
// cols[2E] int32.
int s2v_build_csr(int64_t n, const int64_t *edges, int64_t E, int64_t *row_ptr, int32_t *cols) {
  std::fill(row_ptr, row_ptr + n + 1, 0);
  for (int64_t e = 0; e < E; e++) {
    row_ptr[edges[2 * e] + 1]++;
    row_ptr[edges[2 * e + 1] + 1]++;
  }
  for (int64_t i = 0; i < n; i++) row_ptr[i + 1] += row_ptr[i];
  std::vector<int64_t> fill(row_ptr, row_ptr + n);
  for (int64_t e = 0; e < E; e++) {
    const int64_t x = edges[2 * e], y = edges[2 * e + 1];
    cols[fill[x]++] = (int32_t)y;
    cols[fill[y]++] = (int32_t)x;
  }
  return 0;
}

}  // extern "C"
