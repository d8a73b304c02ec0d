// Forward kernels of the structure2vec-DQN policy (sm_100a).
//
// Replaces (paths relative to /root/reference):
//   w, e1, e2                       pkg/src/graphrl/policy.py:157-161
//   layer loop (spmm + all-reduce   pkg/src/graphrl/policy.py:163-174,
//     + theta4 + relu)              pkg/src/graphrl/state.py:157-162
//   g = embed.sum(axis=2)           pkg/src/graphrl/policy.py:199-200
//   u2 / relu / theta7 / mask       pkg/src/graphrl/policy.py:202-207,221-224
//   top-d / argmax keys             pkg/src/graphrl/inference.py:61-73, agent.py:163-169
//
// Every floating-point result follows the reference's operation order exactly
// (SURVEY.md 3.4): sequential neighbour sums in ascending id, sequential FMA
// chains for the theta projections, numpy pairwise sums, mul-then-add for the
// theta7 contraction.  The library is compiled with -fmad=false.
#include <map>
#include <mutex>
#include <vector>

#include "s2v_common.cuh"

namespace s2v {

// ---------------------------------------------------------------------------
// e12 table over (sol, residual degree)
// ---------------------------------------------------------------------------
template <class T>
__global__ void e12_table_kernel(const T *__restrict__ t1, const T *__restrict__ t2,
                                 const T *__restrict__ t3, int K, int max_deg,
                                 T *__restrict__ table) {
  const int64_t total = (int64_t)(max_deg + 2) * K;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx / K), k = (int)(idx - (int64_t)row * K);
    const bool in_sol = row == max_deg + 1;
    const T deg = in_sol ? T(0) : T(row);
    T acc = T(0);
    for (int p = 0; p < K; p++) acc = fmaT(t3[k * K + p], relu(mulT(t2[p], deg)), acc);
    const T e1 = mulT(t1[k], in_sol ? T(1) : T(0));
    table[idx] = addT(e1, acc);
  }
}

// ---------------------------------------------------------------------------
// Embedding round, generic K / dtype: one warp per local row.
// ---------------------------------------------------------------------------
template <class T, int KPL>  // KPL = k values per lane (K <= 32*KPL)
__global__ void __launch_bounds__(256) round_generic_kernel(
    s2v_shard sh, const T *__restrict__ theta4, const T *__restrict__ table, int K, int max_deg,
    const T *__restrict__ h_in, T *__restrict__ h_out, T *__restrict__ m_out) {
  extern __shared__ unsigned char smem_raw[];
  T *th = reinterpret_cast<T *>(smem_raw);  // [K][K+1]
  T *mbuf = th + K * (K + 1);               // [8][K]
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x)
    th[(idx / K) * (K + 1) + (idx % K)] = theta4[idx];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T *m = mbuf + warp * K;
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  for (int64_t r = blockIdx.x * 8LL + warp; r < nrows; r += gridDim.x * 8LL) {
    const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
    const bool s = sh.sol[r] != 0;
    T acc[KPL];
#pragma unroll
    for (int t = 0; t < KPL; t++) acc[t] = T(0);
    if (h_in && !s) {
      for (int64_t e = sh.row_ptr[r]; e < sh.row_ptr[r + 1]; e++) {
        const uint32_t c = sh.cols[e];
        if (c & S2V_DEAD) continue;
        const T *src = h_in + (int64_t)c * K;
#pragma unroll
        for (int t = 0; t < KPL; t++) {
          const int k = lane + 32 * t;
          if (k < K) acc[t] = addT(acc[t], src[k]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < KPL; t++) {
      const int k = lane + 32 * t;
      if (k < K) {
        m[k] = acc[t];
        if (m_out) m_out[r * K + k] = acc[t];
      }
    }
    __syncwarp();
    const T *e12 = table + (int64_t)(s ? max_deg + 1 : sh.rdeg[r]) * K;
    const int64_t phys = (b * sh.world + sh.rank) * sh.rows_max + i;
#pragma unroll
    for (int t = 0; t < KPL; t++) {
      const int k = lane + 32 * t;
      if (k < K) {
        T z = T(0);
        for (int p = 0; p < K; p++) z = fmaT(th[k * (K + 1) + p], m[p], z);
        h_out[phys * K + k] = relu(addT(e12[k], z));
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Embedding round, K = 64 fp32 fast path.
//
// CTA = 256 threads processes tiles of 32 consecutive local rows.
//  gather : 16 half-warps, each owns 2 rows; lane l of a half-warp holds
//           m[4l..4l+3] (one float4 of the 256-byte neighbour row) and walks
//           the row's neighbours in ascending order with 4 rows in flight.
//  project: m tile [32][64] and theta4^T [64][64] in shared memory; each
//           thread produces 2 rows x 4 k (float4 store), FMA chain p=0..63.
// Rows of the tile are taken from a dynamic tile counter so that hub tiles
// (low ids in BA graphs) start first and never hold up the tail.
// ---------------------------------------------------------------------------
constexpr int kTileRows = 32;

__device__ __forceinline__ float4 ldg_f4(const float *p) {
  return __ldg(reinterpret_cast<const float4 *>(p));
}

__device__ __forceinline__ void add4(float4 &a, const float4 &b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}

// Sequential alive-neighbour sum of one row; 16 lanes, float4 each.
__device__ __forceinline__ float4 gather_row64(const int64_t e0, const int64_t e1,
                                               const uint32_t *__restrict__ cols,
                                               const float *__restrict__ h_in, int sub) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t e = e0;
  // 8 neighbours per step: indices loaded cooperatively, rows issued before
  // any add so 8 x 256 B are in flight per half-warp.
  for (; e + 8 <= e1; e += 8) {
    uint32_t c[8];
#pragma unroll
    for (int q = 0; q < 8; q++) c[q] = __ldg(cols + e + q);
    float4 v[8];
#pragma unroll
    for (int q = 0; q < 8; q++)
      v[q] = (c[q] & S2V_DEAD) ? make_float4(0.f, 0.f, 0.f, 0.f)
                               : ldg_f4(h_in + (int64_t)c[q] * 64 + sub * 4);
#pragma unroll
    for (int q = 0; q < 8; q++)
      if (!(c[q] & S2V_DEAD)) add4(acc, v[q]);
  }
  for (; e < e1; e++) {
    uint32_t c = __ldg(cols + e);
    if (!(c & S2V_DEAD)) add4(acc, ldg_f4(h_in + (int64_t)c * 64 + sub * 4));
  }
  return acc;
}

__global__ void __launch_bounds__(256, 2) round64_kernel(
    s2v_shard sh, const float *__restrict__ theta4, const float *__restrict__ table, int max_deg,
    const float *__restrict__ h_in, float *__restrict__ h_out, float *__restrict__ m_out,
    int *__restrict__ tile_counter) {
  __shared__ __align__(16) float thT[64][64 + 4];           // thT[p][k] = theta4[k][p]
  __shared__ __align__(16) float ms[kTileRows][64 + 4];     // m tile
  __shared__ int s_tile;
  for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x)
    thT[idx % 64][idx / 64] = theta4[idx];
  const int tid = threadIdx.x;
  const int hw = tid >> 4, sub = tid & 15;  // half-warp id, lane in half-warp
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t ntiles = (nrows + kTileRows - 1) / kTileRows;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    const int64_t r0 = tile * kTileRows;
    // ---- gather: each half-warp handles rows hw and hw+16 of the tile
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int lr = hw + 16 * q;
      const int64_t r = r0 + lr;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (h_in && r < nrows && !sh.sol[r])
        acc = gather_row64(sh.row_ptr[r], sh.row_ptr[r + 1], sh.cols, h_in, sub);
      *reinterpret_cast<float4 *>(&ms[lr][sub * 4]) = acc;
      if (m_out && r < nrows) *reinterpret_cast<float4 *>(m_out + r * 64 + sub * 4) = acc;
    }
    __syncthreads();
    // ---- projection: thread -> rows {rp, rp+16}, k in [4*kq, 4*kq+4)
    const int kq = tid & 15, rp = tid >> 4;
    float z[2][4];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int c = 0; c < 4; c++) z[a][c] = 0.f;
#pragma unroll 8
    for (int p = 0; p < 64; p++) {
      const float4 t = *reinterpret_cast<const float4 *>(&thT[p][kq * 4]);
      const float m0 = ms[rp][p], m1 = ms[rp + 16][p];
      z[0][0] = __fmaf_rn(t.x, m0, z[0][0]);
      z[0][1] = __fmaf_rn(t.y, m0, z[0][1]);
      z[0][2] = __fmaf_rn(t.z, m0, z[0][2]);
      z[0][3] = __fmaf_rn(t.w, m0, z[0][3]);
      z[1][0] = __fmaf_rn(t.x, m1, z[1][0]);
      z[1][1] = __fmaf_rn(t.y, m1, z[1][1]);
      z[1][2] = __fmaf_rn(t.z, m1, z[1][2]);
      z[1][3] = __fmaf_rn(t.w, m1, z[1][3]);
    }
#pragma unroll
    for (int a = 0; a < 2; a++) {
      const int64_t r = r0 + rp + 16 * a;
      if (r >= nrows) continue;
      const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
      const int trow = sh.sol[r] ? max_deg + 1 : sh.rdeg[r];
      const float4 e = *reinterpret_cast<const float4 *>(table + (int64_t)trow * 64 + kq * 4);
      float4 o;
      o.x = relu(__fadd_rn(e.x, z[a][0]));
      o.y = relu(__fadd_rn(e.y, z[a][1]));
      o.z = relu(__fadd_rn(e.z, z[a][2]));
      o.w = relu(__fadd_rn(e.w, z[a][3]));
      const int64_t phys = (b * sh.world + sh.rank) * sh.rows_max + i;
      *reinterpret_cast<float4 *>(h_out + phys * 64 + kq * 4) = o;
    }
  }
}

// ---------------------------------------------------------------------------
// numpy pairwise column sums over the N nodes of each slot.
// Plan (host, cached per N): "roots" = maximal subtrees of numpy's recursion
// with <= kRootMax elements, plus the post-order program of the tree above
// them.  Leaf kernel: one CTA per (root, slot), one thread per k.
// ---------------------------------------------------------------------------
constexpr int64_t kRootMax = 1024;

struct PairwiseCtx {
  const void *h;
  int64_t N, rows_max, base, extra;
  int32_t P, b, K;
};

template <class T>
__device__ __forceinline__ T load_node(const PairwiseCtx &c, int64_t u, int k) {
  const int64_t big = c.extra * (c.base + 1);
  const int64_t r = u < big ? u / (c.base + 1) : c.extra + (u - big) / c.base;
  const int64_t start = r * c.base + (r < c.extra ? r : c.extra);
  const int64_t phys = ((int64_t)c.b * c.P + r) * c.rows_max + (u - start);
  return reinterpret_cast<const T *>(c.h)[phys * c.K + k];
}

// numpy pairwise_sum leaf (n <= 128): 8 strided accumulators + sequential tail.
template <class T>
__device__ __forceinline__ T pairwise_leaf(const PairwiseCtx &c, int64_t u0, int64_t n, int k) {
  if (n < 8) {
    T res = T(0);
    for (int64_t i = 0; i < n; i++) res = addT(res, load_node<T>(c, u0 + i, k));
    return res;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = load_node<T>(c, u0 + j, k);
  int64_t i;
  for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = addT(r[j], load_node<T>(c, u0 + i + j, k));
  }
  T res = addT(addT(addT(r[0], r[1]), addT(r[2], r[3])), addT(addT(r[4], r[5]), addT(r[6], r[7])));
  for (; i < n; i++) res = addT(res, load_node<T>(c, u0 + i, k));
  return res;
}

// numpy pairwise_sum of n elements, recursion unrolled onto an explicit stack
// (split n2 = n/2 - (n/2)%8, left + right).
template <class T>
__device__ T pairwise_dev(const PairwiseCtx &c, int64_t u0, int64_t n, int k) {
  struct Frame {
    int64_t u0, n;
    int stage;
    T left;
  };
  Frame st[24];
  int sp = 0;
  st[0].u0 = u0;
  st[0].n = n;
  st[0].stage = 0;
  T ret = T(0);
  for (;;) {
    Frame &f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_leaf<T>(c, f.u0, f.n, k);
      if (sp == 0) return ret;
      sp--;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.stage == 0) {
      f.stage = 1;
      Frame &ch = st[++sp];
      ch.u0 = f.u0;
      ch.n = n2;
      ch.stage = 0;
    } else if (f.stage == 1) {
      f.left = ret;
      f.stage = 2;
      Frame &ch = st[++sp];
      ch.u0 = f.u0 + n2;
      ch.n = f.n - n2;
      ch.stage = 0;
    } else {
      ret = addT(f.left, ret);
      if (sp == 0) return ret;
      sp--;
    }
  }
}

template <class T>
__global__ void colsum_roots_kernel(PairwiseCtx c, const int64_t *__restrict__ roots,
                                    int nroots, T *__restrict__ root_sums) {
  c.b = blockIdx.y;
  const int root = blockIdx.x;
  for (int k = threadIdx.x; k < c.K; k += blockDim.x) {
    T v = pairwise_dev<T>(c, roots[2 * root], roots[2 * root + 1], k);
    root_sums[((int64_t)c.b * nroots + root) * c.K + k] = v;
  }
}

// prog: post-order over roots; entry >= 0 pushes root_sums[entry], -1 pops
// right then left and pushes left + right.
template <class T>
__global__ void colsum_top_kernel(const int32_t *__restrict__ prog, int nprog, int nroots,
                                  int K, const T *__restrict__ root_sums, T *__restrict__ g) {
  const int b = blockIdx.x;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    T stack[48];
    int sp = 0;
    for (int i = 0; i < nprog; i++) {
      int op = prog[i];
      if (op >= 0) {
        stack[sp++] = root_sums[((int64_t)b * nroots + op) * K + k];
      } else {
        T rgt = stack[--sp];
        T lft = stack[--sp];
        stack[sp++] = addT(lft, rgt);
      }
    }
    g[(int64_t)b * K + k] = addT(T(0), stack[0]);
  }
}

struct PairwisePlan {
  int64_t *d_roots = nullptr;  // [nroots][2] (start, len)
  int32_t *d_prog = nullptr;
  int nroots = 0, nprog = 0;
};

static void build_plan(int64_t u0, int64_t n, std::vector<int64_t> &roots,
                       std::vector<int32_t> &prog) {
  if (n <= kRootMax) {
    prog.push_back((int32_t)(roots.size() / 2));
    roots.push_back(u0);
    roots.push_back(n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  build_plan(u0, n2, roots, prog);
  build_plan(u0 + n2, n - n2, roots, prog);
  prog.push_back(-1);
}

static int get_plan(int64_t N, PairwisePlan **out) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, PairwisePlan> cache;
  int dev = 0;
  S2V_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, N);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<int64_t> roots;
    std::vector<int32_t> prog;
    build_plan(0, N, roots, prog);
    PairwisePlan p;
    p.nroots = (int)(roots.size() / 2);
    p.nprog = (int)prog.size();
    S2V_CUDA_CHECK(cudaMalloc(&p.d_roots, sizeof(int64_t) * roots.size()));
    S2V_CUDA_CHECK(cudaMalloc(&p.d_prog, sizeof(int32_t) * prog.size()));
    S2V_CUDA_CHECK(cudaMemcpy(p.d_roots, roots.data(), sizeof(int64_t) * roots.size(),
                              cudaMemcpyHostToDevice));
    S2V_CUDA_CHECK(cudaMemcpy(p.d_prog, prog.data(), sizeof(int32_t) * prog.size(),
                              cudaMemcpyHostToDevice));
    it = cache.emplace(key, p).first;
  }
  *out = &it->second;
  return S2V_OK;
}

// ---------------------------------------------------------------------------
// Scores + selection keys, generic: one warp per local row.
// ---------------------------------------------------------------------------
constexpr int kTopK = 8;
constexpr int kScoreRowsPerBlock = 256;

__device__ __forceinline__ void insert_top(Key (&top)[kTopK], const Key &k) {
  if (!key_gt(k, top[kTopK - 1])) return;
  int pos = kTopK - 1;
  while (pos > 0 && key_gt(k, top[pos - 1])) {
    top[pos] = top[pos - 1];
    pos--;
  }
  top[pos] = k;
}

// Block-wide merge of per-thread top lists held by lane 0 of each warp... kept
// simple: every thread owns a list; lists are merged through shared memory.
__device__ void block_merge_top(Key (&top)[kTopK], Key *s_keys /*[blockDim*8]*/,
                                Key *out) {
  const int tid = threadIdx.x;
  for (int q = 0; q < kTopK; q++) s_keys[tid * kTopK + q] = top[q];
  __syncthreads();
  for (int stride = blockDim.x / 2; stride > 0; stride >>= 1) {
    if (tid < stride) {
      for (int q = 0; q < kTopK; q++) insert_top(top, s_keys[(tid + stride) * kTopK + q]);
      for (int q = 0; q < kTopK; q++) s_keys[tid * kTopK + q] = top[q];
    }
    __syncthreads();
  }
  if (tid == 0)
    for (int q = 0; q < kTopK; q++) out[q] = top[q];
}

template <class T>
__global__ void __launch_bounds__(256) score_generic_kernel(
    s2v_shard sh, int K, const T *__restrict__ h, const T *__restrict__ u1,
    const T *__restrict__ theta6, const T *__restrict__ theta7,
    const uint8_t *__restrict__ cand_override, int mode, T *__restrict__ scores,
    Key *__restrict__ block_keys, int64_t *__restrict__ counts) {
  extern __shared__ unsigned char smem_raw[];
  T *th = reinterpret_cast<T *>(smem_raw);  // [K][K+1]
  T *xbuf = th + K * (K + 1);               // [8][K]
  T *pbuf = xbuf + 8 * K;                   // [8][K]
  Key *s_keys = reinterpret_cast<Key *>(pbuf + 8 * K);
  __shared__ T s_s0;
  __shared__ unsigned long long s_count;
  const int b = blockIdx.y;
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x)
    th[(idx / K) * (K + 1) + (idx % K)] = theta6[idx];
  if (threadIdx.x == 0) {
    T s0 = T(0);
    for (int j = 0; j < K; j++) s0 = addT(s0, mulT(relu(u1[(int64_t)b * K + j]), theta7[j]));
    s_s0 = s0;
    s_count = 0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T *x = xbuf + warp * K;
  T *pr = pbuf + warp * K;
  Key top[kTopK];
#pragma unroll
  for (int q = 0; q < kTopK; q++) top[q] = null_key();
  unsigned long long cnt = 0;
  const int64_t i0 = (int64_t)blockIdx.x * kScoreRowsPerBlock;
  const int64_t i1 = min(i0 + kScoreRowsPerBlock, sh.num_rows);
  for (int64_t i = i0 + warp; i < i1; i += 8) {
    const int64_t r = (int64_t)b * sh.num_rows + i;
    const bool c = (cand_override ? cand_override[r] : sh.cand[r]) != 0;
    const int64_t phys = ((int64_t)b * sh.world + sh.rank) * sh.rows_max + i;
    for (int k = lane; k < K; k += 32) x[k] = mulT(h[phys * K + k], c ? T(1) : T(0));
    __syncwarp();
    for (int k = lane; k < K; k += 32) {
      T acc = T(0);
      for (int p = 0; p < K; p++) acc = fmaT(th[k * (K + 1) + p], x[p], acc);
      pr[k] = mulT(relu(acc), theta7[K + k]);
    }
    __syncwarp();
    if (lane == 0) {
      T s = s_s0;
      for (int k = 0; k < K; k++) s = addT(s, pr[k]);
      scores[r] = s;
      const bool finite = isfinite((double)s);
      if (c && finite) cnt++;
      if (c && (finite || mode == 1)) insert_top(top, make_key((double)s, sh.row_start + i));
    }
    __syncwarp();
  }
  if (cnt) atomicAdd(&s_count, cnt);
  block_merge_top(top, s_keys, block_keys + ((int64_t)b * gridDim.x + blockIdx.x) * kTopK);
  if (threadIdx.x == 0 && s_count)
    atomicAdd((unsigned long long *)&counts[b], s_count);
}

__global__ void topk_merge_kernel(const Key *__restrict__ block_keys, int nblk, int d,
                                  Key *__restrict__ top_out) {
  extern __shared__ unsigned char smem_raw[];
  Key *s_keys = reinterpret_cast<Key *>(smem_raw);
  const int b = blockIdx.x;
  Key top[kTopK];
#pragma unroll
  for (int q = 0; q < kTopK; q++) top[q] = null_key();
  for (int64_t idx = threadIdx.x; idx < (int64_t)nblk * kTopK; idx += blockDim.x)
    insert_top(top, block_keys[(int64_t)b * nblk * kTopK + idx]);
  __shared__ Key s_out[kTopK];
  block_merge_top(top, s_keys, s_out);
  __syncthreads();
  if (threadIdx.x < d) top_out[(int64_t)b * d + threadIdx.x] = s_out[threadIdx.x];
}

template <class T>
static int embed_round_t(const s2v_shard *sh, const void *theta4, const void *table, int K,
                         int max_deg, const void *h_in, void *h_out, void *m_out,
                         cudaStream_t st) {
  const int64_t nrows = (int64_t)sh->batch * sh->num_rows;
  if (nrows == 0) return S2V_OK;
  if (sizeof(T) == 4 && K == 64) {
    static thread_local int *counter = nullptr;
    if (!counter) S2V_CUDA_CHECK(cudaMalloc(&counter, sizeof(int)));
    S2V_CUDA_CHECK(cudaMemsetAsync(counter, 0, sizeof(int), st));
    int64_t ntiles = (nrows + kTileRows - 1) / kTileRows;
    int grid = (int)std::min<int64_t>(ntiles, kNumSMs * 2);
    round64_kernel<<<grid, 256, 0, st>>>(*sh, (const float *)theta4, (const float *)table,
                                         max_deg, (const float *)h_in, (float *)h_out,
                                         (float *)m_out, counter);
    S2V_LAUNCH_CHECK();
    return S2V_OK;
  }
  if (K > 256) return fail(S2V_EINVAL, "embed_dim %d > 256 unsupported", K);
  size_t smem = sizeof(T) * ((size_t)K * (K + 1) + 8 * (size_t)K);
  int grid = (int)std::min<int64_t>((nrows + 7) / 8, kNumSMs * 8);
#define S2V_LAUNCH_ROUND(KPL)                                                               \
  do {                                                                                      \
    auto kern = round_generic_kernel<T, KPL>;                                               \
    S2V_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                        (int)smem));                                        \
    kern<<<grid, 256, smem, st>>>(*sh, (const T *)theta4, (const T *)table, K, max_deg,     \
                                  (const T *)h_in, (T *)h_out, (T *)m_out);                 \
  } while (0)
  if (K <= 32)
    S2V_LAUNCH_ROUND(1);
  else if (K <= 64)
    S2V_LAUNCH_ROUND(2);
  else if (K <= 128)
    S2V_LAUNCH_ROUND(4);
  else
    S2V_LAUNCH_ROUND(8);
#undef S2V_LAUNCH_ROUND
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // namespace s2v

using namespace s2v;

extern "C" {

int s2v_e12_table(s2v_dtype dt, const void *theta1, const void *theta2, const void *theta3,
                  int K, int max_deg, void *table, void *stream) {
  if (K < 1 || max_deg < 0) return fail(S2V_EINVAL, "bad e12 table args");
  int64_t total = (int64_t)(max_deg + 2) * K;
  int grid = (int)std::min<int64_t>((total + 255) / 256, kNumSMs * 8);
  if (dt == S2V_F32)
    e12_table_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(
        (const float *)theta1, (const float *)theta2, (const float *)theta3, K, max_deg,
        (float *)table);
  else
    e12_table_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
        (const double *)theta1, (const double *)theta2, (const double *)theta3, K, max_deg,
        (double *)table);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_embed_round(s2v_dtype dt, const s2v_shard *sh, const void *theta4, const void *table,
                    int K, int max_deg, const void *h_in, void *h_out, void *m_out,
                    void *stream) {
  cudaStream_t st = as_stream(stream);
  if (dt == S2V_F32)
    return embed_round_t<float>(sh, theta4, table, K, max_deg, h_in, h_out, m_out, st);
  return embed_round_t<double>(sh, theta4, table, K, max_deg, h_in, h_out, m_out, st);
}

size_t s2v_colsum_workspace(const s2v_shard *sh, int K, int elem_bytes) {
  // upper bound on roots: ceil(N / (kRootMax/2)) + 1
  int64_t nroots = sh->num_nodes / (kRootMax / 2) + 2;
  return (size_t)nroots * sh->batch * K * elem_bytes;
}

int s2v_colsum(s2v_dtype dt, const s2v_shard *sh, int K, const void *h, void *g,
               void *workspace, size_t workspace_bytes, void *stream) {
  PairwisePlan *plan = nullptr;
  int rc = get_plan(sh->num_nodes, &plan);
  if (rc) return rc;
  size_t need = (size_t)plan->nroots * sh->batch * K * (dt == S2V_F32 ? 4 : 8);
  if (workspace_bytes < need) return fail(S2V_EINVAL, "colsum workspace too small");
  PairwiseCtx c;
  c.h = h;
  c.N = sh->num_nodes;
  c.rows_max = sh->rows_max;
  c.P = sh->world;
  c.base = sh->num_nodes / sh->world;
  c.extra = sh->num_nodes % sh->world;
  c.K = K;
  c.b = 0;
  cudaStream_t st = as_stream(stream);
  dim3 grid(plan->nroots, sh->batch);
  int threads = K < 32 ? 32 : (K > 256 ? 256 : K);
  if (dt == S2V_F32) {
    colsum_roots_kernel<float><<<grid, threads, 0, st>>>(c, plan->d_roots, plan->nroots,
                                                         (float *)workspace);
    colsum_top_kernel<float><<<sh->batch, threads, 0, st>>>(
        plan->d_prog, plan->nprog, plan->nroots, K, (const float *)workspace, (float *)g);
  } else {
    colsum_roots_kernel<double><<<grid, threads, 0, st>>>(c, plan->d_roots, plan->nroots,
                                                          (double *)workspace);
    colsum_top_kernel<double><<<sh->batch, threads, 0, st>>>(
        plan->d_prog, plan->nprog, plan->nroots, K, (const double *)workspace, (double *)g);
  }
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_score_blocks(const s2v_shard *sh) {
  int64_t n = (sh->num_rows + kScoreRowsPerBlock - 1) / kScoreRowsPerBlock;
  return (int)(n < 1 ? 1 : n);
}

int s2v_score(s2v_dtype dt, const s2v_shard *sh, int K, const void *h, const void *u1,
              const void *theta6, const void *theta7, const uint8_t *cand_override, int mode,
              void *scores, uint64_t *block_keys, int64_t *counts, void *stream) {
  if (K > 256) return fail(S2V_EINVAL, "embed_dim %d > 256 unsupported", K);
  cudaStream_t st = as_stream(stream);
  S2V_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(int64_t) * sh->batch, st));
  dim3 grid(s2v_score_blocks(sh), sh->batch);
  size_t elem = dt == S2V_F32 ? 4 : 8;
  size_t smem = elem * ((size_t)K * (K + 1) + 16 * (size_t)K) + sizeof(Key) * 256 * kTopK;
  if (dt == S2V_F32) {
    auto kern = score_generic_kernel<float>;
    S2V_CUDA_CHECK(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 256, smem, st>>>(*sh, K, (const float *)h, (const float *)u1,
                                  (const float *)theta6, (const float *)theta7, cand_override,
                                  mode, (float *)scores, (Key *)block_keys, counts);
  } else {
    auto kern = score_generic_kernel<double>;
    S2V_CUDA_CHECK(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 256, smem, st>>>(*sh, K, (const double *)h, (const double *)u1,
                                  (const double *)theta6, (const double *)theta7,
                                  cand_override, mode, (double *)scores, (Key *)block_keys,
                                  counts);
  }
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_topk_merge(const s2v_shard *sh, const uint64_t *block_keys, int d, uint64_t *top,
                   void *stream) {
  if (d < 1 || d > kTopK) return fail(S2V_EINVAL, "top-d merge supports 1 <= d <= 8, got %d", d);
  int nblk = s2v_score_blocks(sh);
  size_t smem = sizeof(Key) * 256 * kTopK;
  S2V_CUDA_CHECK(cudaFuncSetAttribute(topk_merge_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  topk_merge_kernel<<<sh->batch, 256, smem, as_stream(stream)>>>((const Key *)block_keys, nblk,
                                                                  d, (Key *)top);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // extern "C"
