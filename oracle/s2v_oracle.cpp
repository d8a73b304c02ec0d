// s2v_oracle.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A plain C++ restatement of the reference's structure2vec forward pass in the
// exact floating-point operation order the reference produces under
// numpy 2.3 / scipy 1.18 / OpenBLAS 0.3.30 (SkylakeX sgemm kernel).  It is the
// bit-exact checker the GPU kernels are compared against at any graph size.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
// it.  It is pinned against golden vectors produced by the reference itself
// (oracle/make_golden.py -> tests/golden/, checked by tests/test_oracle.py).
//
// Reference algorithm followed (paths relative to /root/reference):
//   degrees            pkg/src/graphrl/state.py:140-143   (row sums of residual CSR)
//   w, e1, e2          pkg/src/graphrl/policy.py:157-161
//   layer loop         pkg/src/graphrl/policy.py:163-174  (spmm state.py:157-162)
//   g = sum(embed)     pkg/src/graphrl/policy.py:199      (numpy pairwise sum)
//   u2, relu, theta7   pkg/src/graphrl/policy.py:202-207
//
// Operation-order contract:
//   spmm   : acc=+0; for u in N(v) ascending, edge alive: acc = fl(acc + h[u,k])
//   matmul : acc=+0; for p in 0..K-1: acc = fma(theta[k,p], x[p], acc)
//   einsum : s=+0;   for j in 0..2K-1: s = fl(s + fl(r[j]*t7[j]))
//   sum    : numpy pairwise_sum (8 strided accumulators, <=128-element leaves)
//   relu   : np.maximum(x, 0) == (x >= 0 || isnan(x)) ? x : 0
//
// Layout: node-major h[v*K + k].  CSR: row_ptr int64[n+1], cols int32[nnz],
// neighbour lists sorted ascending.  Entry (v,u) is alive iff !sol[v] && !sol[u]
// (the reference zeroes solution rows and columns, state.py:89-105,173-208).
//
// Build (oracle/Makefile): g++ -O2 -mfma -ffp-contract=off -pthread.  Threads
// split the node range only; every output's own operation order is sequential.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

template <class F>
void parallel_for(int64_t n, F fn) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (n < 4096) nt = 1;
  if (nt == 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; t++) {
    int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([=] { fn(lo, hi); });
  }
  for (auto &x : th) x.join();
}

inline float fmaT(float a, float b, float c) { return std::fmaf(a, b, c); }
inline double fmaT(double a, double b, double c) { return std::fma(a, b, c); }

template <class T>
inline T relu(T x) { return (x >= T(0) || x != x) ? x : T(0); }

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src)
template <class T>
T pairwise(const T *a, int64_t n, int64_t stride) {
  if (n < 8) {
    T res = T(0);
    for (int64_t i = 0; i < n; i++) res = res + a[i * stride];
    return res;
  } else if (n <= 128) {
    T r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j * stride];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = r[j] + a[(i + j) * stride];
    T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res = res + a[i * stride];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(a, n2, stride) + pairwise(a + n2 * stride, n - n2, stride);
}

void degrees(int64_t n, const int64_t *row_ptr, const int32_t *cols, const uint8_t *sol,
             int32_t *deg) {
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t v = lo; v < hi; v++) {
      int32_t d = 0;
      if (!sol[v])
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) d += !sol[cols[e]];
      deg[v] = d;
    }
  });
}

template <class T>
int embed(int64_t n, const int64_t *row_ptr, const int32_t *cols, const uint8_t *sol,
          const T *t1, const T *t2, const T *t3, const T *t4, int K, int L, T *h_out) {
  std::vector<int32_t> deg(n);
  std::vector<T> e12((size_t)n * K), h_prev((size_t)n * K, T(0));
  degrees(n, row_ptr, cols, sol, deg.data());
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    std::vector<T> w(K);
    for (int64_t v = lo; v < hi; v++) {
      T dv = T(deg[v]), sv = sol[v] ? T(1) : T(0);
      for (int p = 0; p < K; p++) w[p] = relu(T(t2[p] * dv));
      for (int k = 0; k < K; k++) {
        T acc = T(0);
        for (int p = 0; p < K; p++) acc = fmaT(t3[k * K + p], w[p], acc);
        T e1 = t1[k] * sv;
        e12[v * K + k] = e1 + acc;
      }
    }
  });
  for (int layer = 0; layer < L; layer++) {
    parallel_for(n, [&](int64_t lo, int64_t hi) {
      std::vector<T> m(K);
      for (int64_t v = lo; v < hi; v++) {
        for (int k = 0; k < K; k++) m[k] = T(0);
        if (!sol[v])
          for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) {
            int32_t u = cols[e];
            if (sol[u]) continue;
            const T *hu = h_prev.data() + (int64_t)u * K;
            for (int k = 0; k < K; k++) m[k] = m[k] + hu[k];
          }
        for (int k = 0; k < K; k++) {
          T acc = T(0);
          for (int p = 0; p < K; p++) acc = fmaT(t4[k * K + p], m[p], acc);
          T z = e12[v * K + k] + acc;
          h_out[v * K + k] = relu(z);
        }
      }
    });
    if (layer + 1 < L) std::memcpy(h_prev.data(), h_out, sizeof(T) * (size_t)n * K);
  }
  return 0;
}

template <class T>
void colsum(int64_t n, int K, const T *h, T *g) {
  for (int k = 0; k < K; k++) g[k] = T(0) + pairwise(h + k, n, K);
}

template <class T>
void scores(int64_t n, int K, const T *h, const uint8_t *cand, const T *t6, const T *t7,
            const T *u1, T *out) {
  T s0 = T(0);
  for (int j = 0; j < K; j++) {
    T prod = relu(u1[j]) * t7[j];
    s0 = s0 + prod;
  }
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    std::vector<T> x(K);
    for (int64_t v = lo; v < hi; v++) {
      T c = cand[v] ? T(1) : T(0);
      for (int p = 0; p < K; p++) x[p] = h[v * K + p] * c;
      T s = s0;
      for (int k = 0; k < K; k++) {
        T acc = T(0);
        for (int p = 0; p < K; p++) acc = fmaT(t6[k * K + p], x[p], acc);
        T prod = relu(acc) * t7[K + k];
        s = s + prod;
      }
      out[v] = s;
    }
  });
}

}  // namespace

extern "C" {

void s2vo_degrees(int64_t n, const int64_t *row_ptr, const int32_t *cols,
                  const uint8_t *sol, int32_t *deg) {
  degrees(n, row_ptr, cols, sol, deg);
}

int s2vo_embed_f32(int64_t n, const int64_t *rp, const int32_t *c, const uint8_t *s,
                   const float *t1, const float *t2, const float *t3, const float *t4,
                   int K, int L, float *h) {
  return embed<float>(n, rp, c, s, t1, t2, t3, t4, K, L, h);
}
int s2vo_embed_f64(int64_t n, const int64_t *rp, const int32_t *c, const uint8_t *s,
                   const double *t1, const double *t2, const double *t3, const double *t4,
                   int K, int L, double *h) {
  return embed<double>(n, rp, c, s, t1, t2, t3, t4, K, L, h);
}
void s2vo_colsum_f32(int64_t n, int K, const float *h, float *g) { colsum<float>(n, K, h, g); }
void s2vo_colsum_f64(int64_t n, int K, const double *h, double *g) { colsum<double>(n, K, h, g); }
void s2vo_scores_f32(int64_t n, int K, const float *h, const uint8_t *cand, const float *t6,
                     const float *t7, const float *u1, float *out) {
  scores<float>(n, K, h, cand, t6, t7, u1, out);
}
void s2vo_scores_f64(int64_t n, int K, const double *h, const uint8_t *cand, const double *t6,
                     const double *t7, const double *u1, double *out) {
  scores<double>(n, K, h, cand, t6, t7, u1, out);
}

}  // extern "C"
