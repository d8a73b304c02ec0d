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
#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <vector>

#include "s2v_common.cuh"
#include "s2v_gather.cuh"

namespace s2v {

// ---------------------------------------------------------------------------
// e12 table over (sol, residual degree)
// ---------------------------------------------------------------------------
template <class T>
__global__ void e12_table_kernel(const T *__restrict__ t1, const T *__restrict__ t2,
                                 const T *__restrict__ t3, int K, int max_deg,
                                 T *__restrict__ table) {
  extern __shared__ unsigned char smem_raw[];
  T *th3T = reinterpret_cast<T *>(smem_raw);  // [K][K+1]: th3T[p][k] = theta3[k][p]
  T *th2 = th3T + K * (K + 1);                // [K]
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x)
    th3T[(idx % K) * (K + 1) + idx / K] = t3[idx];
  for (int p = threadIdx.x; p < K; p += blockDim.x) th2[p] = t2[p];
  __syncthreads();
  const int64_t total = (int64_t)(max_deg + 2) * K;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx / K), k = (int)(idx - (int64_t)row * K);
    const bool in_sol = row == max_deg + 1;
    const T deg = in_sol ? T(0) : T(row);
    T acc = T(0);
    for (int p = 0; p < K; p++) acc = fmaT(th3T[p * (K + 1) + k], relu(mulT(th2[p], deg)), acc);
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
// CTA = 256 threads processes tiles of 32 local rows taken in descending
// degree order (sh.order) from a dynamic tile counter, so rows of a tile have
// similar neighbour counts and hub tiles start first.
//  gather : 16 half-warps, each owns 2 rows of the tile; lane l of a
//           half-warp holds m[4l..4l+3] (one float4 of the 256-byte neighbour
//           row).  Neighbour ids are fetched 16 at a time (one per lane,
//           coalesced) and broadcast with shuffles; rows are loaded in
//           batches of 8 (all loads issued before the ascending-order adds).
//           Rows of low physical id (BA hubs: most gathers) are loaded with
//           an L2 evict_last policy, the rest evict_first.
//  project: m tile [32][64] and theta4^T [64][64] in shared memory; each
//           thread produces 2 rows x 4 k (float4 store), FMA chain p=0..63,
//           then z = e12[deg] + chain, relu.
// ---------------------------------------------------------------------------
//  TABLE  : round 2 at P = 1 reads neighbour rows from the per-degree table
//           of round-1 outputs (h1_table_kernel) instead of h1: h1[u] depends
//           only on (sol[u], rdeg[u]) and an alive neighbour has sol = 0, so
//           h1[u] == h1_table[rdeg[u]] bit for bit and the same ascending
//           adds give the same sums; the 2.4 MB table stays in L1/L2, so the
//           round reads the CSR and rdeg instead of 16 GB of neighbour rows.
constexpr int kTileRows = 32;
// tiles whose rows all have at most this many entries gather one row per
// 8-lane group (all 32 rows of the tile in flight at once) instead of one row
// per half-warp, two rows at a time.  Measured on cfg3 (round ms): 0 (off)
// 2.43, 16: 2.41, 32: 2.28, 64: 2.24, 128: 2.237, 512: 2.234, 4096: 2.232 —
// more rows in flight beats the longer per-row chains at every degree below
// the hub cut, so the default is the hub degree (every non-hub tile).
// S2V_SPARSE_MAX overrides it (0 turns the mode off) for A/B runs.
constexpr int kSparseMax = S2V_HUB_DEGREE;

// h1_table[t][k] = the round-1 output of a row whose e12 row is t: the
// round kernel's epilogue with m = 0 (FMA chain over zeros, + e12, relu).
// The chain over m = 0 is the same for every row t, so each block first
// runs the 64 chains once into shared memory.
__global__ void h1_table_kernel(const float *__restrict__ theta4,
                                const float *__restrict__ table, int rows,
                                float *__restrict__ h1) {
  __shared__ float z0[64];
  if (threadIdx.x < 64) {
    float z = 0.f;
    for (int p = 0; p < 64; p++) z = __fmaf_rn(theta4[threadIdx.x * 64 + p], 0.f, z);
    z0[threadIdx.x] = z;
  }
  __syncthreads();
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)rows * 64;
       idx += (int64_t)gridDim.x * blockDim.x)
    h1[idx] = relu(__fadd_rn(table[idx], z0[idx & 63]));
}

template <bool TABLE>
__global__ void __launch_bounds__(256, 4) round64_kernel(
    s2v_shard sh, const float *__restrict__ theta4, const float *__restrict__ table, int max_deg,
    const float *__restrict__ h_in, float *__restrict__ h_out, float *__restrict__ m_out,
    int *__restrict__ tile_counter, uint32_t hot_rows, float *const *__restrict__ peers,
    int npeers, const int32_t *__restrict__ deg_src, int sparse_max, int pf) {
  // deg_src (TABLE): residual degree by physical row -- every rank's rows
  // at P > 1 (s2v_trow + exchange), this shard's rdeg at P = 1
  __shared__ __align__(16) float thT[64][64 + 4];        // thT[p][k] = theta4[k][p]
  __shared__ __align__(16) float ms[kTileRows][64 + 4];  // m tile
  __shared__ int32_t s_rows[kTileRows];
  __shared__ int64_t s_e0[kTileRows], s_e1[kTileRows];  // neighbour range, empty if in S
  __shared__ int32_t s_trow[kTileRows];                 // e12 table row (sol, rdeg)
  // next tile fetched one tile ahead: its index (atomic) and its rows' ids
  // (cp.async, no registers held) overlap the current tile's projection
  __shared__ int32_t s_raw[2][kTileRows];
  __shared__ int s_tiles[2];
  bool have_theta = false;  // staged with the first tile (idle CTAs skip it)
  const int tid = threadIdx.x;
  const int hw = tid >> 4, sub = tid & 15;  // half-warp id, lane in half-warp
  const unsigned hmask = (tid & 16) ? 0xFFFF0000u : 0x0000FFFFu;
  const int hbase = tid & 16;
  const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
  // rows visited: the active list when set (residual rows only), else every
  // row in processing order; hub rows at the head go to hub_round64_kernel
  const int32_t *list = sh.active ? sh.active : sh.order;
  const int64_t nrows = sh.active ? sh.active_n[0] : (int64_t)sh.batch * sh.num_rows;
  const int64_t first = sh.active ? sh.active_n[1] : (sh.order ? sh.n_hub : 0);
  const int64_t ntiles = (nrows - first + kTileRows - 1) / kTileRows;
  // row ids of tile t into s_raw[buf] (thread tid < kTileRows: row tid)
  auto prefetch_rows = [&](int64_t t, int buf) {
    const int64_t q = first + t * kTileRows + tid;
    if (t < ntiles && q < nrows && list)
      cp_async4(&s_raw[buf][tid], list + q);
    else
      s_raw[buf][tid] = (t < ntiles && q < nrows) ? (int32_t)q : -1;
  };
  if (tid == 0) s_tiles[0] = atomicAdd(tile_counter, 1);
  __syncthreads();
  if (tid < kTileRows) prefetch_rows(s_tiles[0], 0);
  int cur = 0;
  for (;;) {
    cp_async_wait_all();
    __syncthreads();
    const int64_t tile = s_tiles[cur];
    if (tile >= ntiles) break;
    if (tid == 0) s_tiles[cur ^ 1] = atomicAdd(tile_counter, 1);
    if (!have_theta) {  // visible to the projection after the gather's barrier
      for (int idx = tid; idx < 64 * 64; idx += blockDim.x) thT[idx % 64][idx / 64] = theta4[idx];
      have_theta = true;
    }
    if (tid < kTileRows) {
      // one pass loads every row's range, membership in S and e12 row
      const int64_t q = first + tile * kTileRows + tid;
      const int32_t r = s_raw[cur][tid];
      s_rows[tid] = r;
      int64_t e0 = 0, e1 = 0;
      int trow = 0;
      if (r >= 0) {
        const bool in_s = sh.sol[r] != 0;
        trow = in_s ? max_deg + 1 : sh.rdeg[r];
        if (h_in && !in_s) {
          // the active list's compact CSR is indexed by list position
          e0 = sh.active_ptr ? sh.active_ptr[q] : sh.row_ptr[r];
          e1 = sh.active_ptr ? sh.active_ptr[q + 1] : sh.row_ptr[r + 1];
        }
      }
      s_e0[tid] = e0;
      s_e1[tid] = e1;
      s_trow[tid] = trow;
    }
    // sparse tile (every row <= kSparseMax entries, the bulk of a late
    // episode and of R-MAT): one 8-lane group per row, all 32 rows of the
    // tile at once instead of two rows in turn per half-warp
    const bool sparse =
        __syncthreads_and(tid >= kTileRows || s_e1[tid] - s_e0[tid] <= sparse_max);
    if (sparse) {
      const int lr = tid >> 3, l8 = tid & 7;
      const unsigned qmask = 0xFFu << (tid & 24);
      const int qbase = tid & 24;
      const int64_t r = s_rows[lr];
      const int64_t e0 = s_e0[lr], e1 = s_e1[lr];
      const uint32_t *cl = sh.active_ptr ? sh.active_cols : sh.cols;
      const uint8_t *sol_of = sh.active_ptr ? (sh.active_sol ? sh.active_sol : sh.sol) : nullptr;
      const uint32_t hot_lo =
          TABLE ? 0u : (uint32_t)(r >= 0 ? (r / sh.num_rows) * sh.world * sh.rows_max : 0);
      float4 a0, a1;
      gather_row64_g8<TABLE>(e0, e1, cl, h_in, l8, qmask, qbase, hot_rows, pol_hot, pol_cold,
                             deg_src, sol_of, hot_lo, a0, a1, TABLE ? 0 : pf);
      *reinterpret_cast<float4 *>(&ms[lr][4 * l8]) = a0;
      *reinterpret_cast<float4 *>(&ms[lr][32 + 4 * l8]) = a1;
      if (m_out && r >= 0) {
        *reinterpret_cast<float4 *>(m_out + r * 64 + 4 * l8) = a0;
        *reinterpret_cast<float4 *>(m_out + r * 64 + 32 + 4 * l8) = a1;
      }
    } else {
    // ---- gather: each half-warp handles rows hw and hw+16 of the tile
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int lr = hw + 16 * q;
      const int64_t r = s_rows[lr];
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (s_e1[lr] > s_e0[lr])
        acc = gather_row64<TABLE>(
            s_e0[lr], s_e1[lr], sh.active_ptr ? sh.active_cols : sh.cols, h_in, sub, hmask, hbase,
            hot_rows, pol_hot, pol_cold, deg_src,
            sh.active_ptr ? (sh.active_sol ? sh.active_sol : sh.sol) : nullptr,
            TABLE ? 0u : (uint32_t)((r / sh.num_rows) * sh.world * sh.rows_max));
      *reinterpret_cast<float4 *>(&ms[lr][sub * 4]) = acc;
      if (m_out && r >= 0) *reinterpret_cast<float4 *>(m_out + r * 64 + sub * 4) = acc;
    }
    }
    __syncthreads();
    if (tid < kTileRows) prefetch_rows(s_tiles[cur ^ 1], cur ^ 1);
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
      const int64_t r = s_rows[rp + 16 * a];
      if (r < 0) continue;
      const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
      const int trow = s_trow[rp + 16 * a];
      const float4 e = *reinterpret_cast<const float4 *>(table + (int64_t)trow * 64 + kq * 4);
      float4 o;
      o.x = relu(__fadd_rn(e.x, z[a][0]));
      o.y = relu(__fadd_rn(e.y, z[a][1]));
      o.z = relu(__fadd_rn(e.z, z[a][2]));
      o.w = relu(__fadd_rn(e.w, z[a][3]));
      const int64_t phys = (b * sh.world + sh.rank) * sh.rows_max + i;
      stg_f4_pol(h_out + phys * 64 + kq * 4, o, pol_cold);
      // fused halo exchange: the same row straight into every peer's buffer
      for (int q = 0; q < npeers; q++)
        if (peers[q] != h_out) *reinterpret_cast<float4 *>(peers[q] + phys * 64 + kq * 4) = o;
    }
    cur ^= 1;
  }
}

// One CTA per hub row (the first sh.n_hub rows of sh.order): cooperative
// gather (hub_gather_row64), then the same e12 + theta4 chain + relu epilogue
// computed by 64 threads.  Runs on a side stream concurrently with
// round64_kernel, which handles every other row.
template <bool TABLE>
__global__ void __launch_bounds__(256, 1) hub_round64_kernel(
    s2v_shard sh, const float *__restrict__ theta4, const float *__restrict__ table, int max_deg,
    const float *__restrict__ h_in, float *__restrict__ h_out, float *__restrict__ m_out,
    int *__restrict__ counter, uint32_t hot_rows, float *const *__restrict__ peers, int npeers,
    const int32_t *__restrict__ deg_src) {
  extern __shared__ __align__(16) float hub_smem[];
  float *ring = hub_smem;                              // [2][120][64]
  float(*thT)[65] = reinterpret_cast<float(*)[65]>(hub_smem + 2 * kHubBatch * 64);
  float *mrow = hub_smem + 2 * kHubBatch * 64 + 64 * 65;
  __shared__ int s_q;
  const int tid = threadIdx.x, sub = tid & 15;
  const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
  bool have_theta = false;  // staged with the first row (idle CTAs skip it)
  for (;;) {
    __syncthreads();
    if (tid == 0) s_q = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t q = s_q;
    if (q >= (sh.active ? sh.active_n[1] : sh.n_hub)) break;
    if (!have_theta) {  // visible to the epilogue after the gather's barriers
      for (int idx = tid; idx < 64 * 64; idx += 256) thT[idx % 64][idx / 64] = theta4[idx];
      have_theta = true;
    }
    const int64_t r = sh.active ? sh.active[q] : sh.order[q];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h_in && !sh.sol[r]) {
      if (sh.active_ptr)
        acc = hub_gather_row64<TABLE>(sh.active_ptr[q], sh.active_ptr[q + 1], sh.active_cols,
                                      h_in, ring, hot_rows, pol_hot, pol_cold, deg_src,
                                      sh.active_sol ? sh.active_sol : sh.sol);
      else
        acc = hub_gather_row64<TABLE>(sh.row_ptr[r], sh.row_ptr[r + 1], sh.cols, h_in, ring,
                                      hot_rows, pol_hot, pol_cold, deg_src);
    }
    if (tid < 16) {
      *reinterpret_cast<float4 *>(mrow + sub * 4) = acc;
      if (m_out) *reinterpret_cast<float4 *>(m_out + r * 64 + sub * 4) = acc;
    }
    __syncthreads();
    if (tid < 64) {
      float z = 0.f;
      for (int p = 0; p < 64; p++) z = __fmaf_rn(thT[p][tid], mrow[p], z);
      const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
      const int trow = sh.sol[r] ? max_deg + 1 : sh.rdeg[r];
      const int64_t phys = (b * sh.world + sh.rank) * sh.rows_max + i;
      const float o = relu(__fadd_rn(table[(int64_t)trow * 64 + tid], z));
      h_out[phys * 64 + tid] = o;
      for (int q = 0; q < npeers; q++)
        if (peers[q] != h_out) peers[q][phys * 64 + tid] = o;
    }
  }
}

// side stream + events for the hub kernels (per thread / device)
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
  int *counter = nullptr;
  int device = -1;
};

static int side_stream(SideStream **out) {
  static thread_local SideStream ss;
  int dev = 0;
  S2V_CUDA_CHECK(cudaGetDevice(&dev));
  if (ss.device != dev) {
    S2V_CUDA_CHECK(cudaStreamCreateWithFlags(&ss.stream, cudaStreamNonBlocking));
    S2V_CUDA_CHECK(cudaEventCreateWithFlags(&ss.ready, cudaEventDisableTiming));
    S2V_CUDA_CHECK(cudaEventCreateWithFlags(&ss.done, cudaEventDisableTiming));
    S2V_CUDA_CHECK(cudaMalloc(&ss.counter, sizeof(int)));
    ss.device = dev;
  }
  *out = &ss;
  return S2V_OK;
}

// Launch `launch_hub(side_stream, counter)` concurrently with the work the
// caller enqueues next on `st`; returns after making `st` wait for it.
template <class F>
static int with_hub_kernel(const s2v_shard *sh, cudaStream_t st, F launch_hub,
                           SideStream **ss_out) {
  *ss_out = nullptr;
  if (!sh->order || sh->n_hub <= 0) return S2V_OK;
  SideStream *ss = nullptr;
  int rc = side_stream(&ss);
  if (rc) return rc;
  S2V_CUDA_CHECK(cudaEventRecord(ss->ready, st));
  S2V_CUDA_CHECK(cudaStreamWaitEvent(ss->stream, ss->ready, 0));
  S2V_CUDA_CHECK(cudaMemsetAsync(ss->counter, 0, sizeof(int), ss->stream));
  launch_hub(ss->stream, ss->counter);
  S2V_LAUNCH_CHECK();
  S2V_CUDA_CHECK(cudaEventRecord(ss->done, ss->stream));
  *ss_out = ss;
  return S2V_OK;
}

constexpr size_t kHubSmem = sizeof(float) * (2 * kHubBatch * 64 + 64 * 65 + 64);

// ---------------------------------------------------------------------------
// numpy pairwise column sums over the N nodes of each slot (policy.py:199).
//
// numpy's pairwise_sum(a, n): n < 8 sequential; n <= 128 eight strided
// accumulators r[j] (r[j] = a[j] + a[j+8] + ... sequentially) combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then a sequential tail; else split at
// n2 = n/2 - (n/2)%8 and return left + right.  The recursion tree depends on
// N only, so the host enumerates it once per N (cached): leaves in order and
// internal nodes grouped by height.  Then
//   leaf kernel : one thread per (leaf, k, j) runs accumulator chain r[j]
//                 (16 independent loads in flight), j = 0 combines + tail;
//   level kernel: one launch per height, vals[node] = vals[left] + vals[right].
// ---------------------------------------------------------------------------
struct PairwiseCtx {
  const void *h;
  int64_t N, rows_max, base, extra;
  int32_t P, b, K;
  // residual mode: rows with rdeg = 0 read dead[sol ? K : 0 .. + K).  P = 1
  // classifies from the shard's rdeg / sol; P > 1 from trow, every rank's
  // e12 table row by physical row (s2v_trow + the round-2 exchange):
  // 0 = rdeg 0 outside S, max_deg + 1 = in S, anything else alive
  const void *dead;
  const int32_t *rdeg;
  const uint8_t *sol;
  const int32_t *trow;
  int32_t max_deg;
  // incremental residual mode: last[row] = the row's class at the previous
  // call (0 live, 1/2 dead); a leaf dead now and then keeps its value
  uint8_t *last;
  int full;
  // incremental forward: only leaves flagged here (rows whose value changed)
  // are recomputed, the rest keep their cached sums
  const uint8_t *leaf_dirty;
};

__device__ __forceinline__ int64_t phys_node(const PairwiseCtx &c, int64_t u);

// residual class of global node u of slot c.b: 0 alive, 1 dead (sol 0), 2 in S
__device__ __forceinline__ uint8_t dead_code(const PairwiseCtx &c, int64_t u) {
  if (c.trow) {
    const int32_t t = c.trow[phys_node(c, u)];
    return t == 0 ? 1 : (t == c.max_deg + 1 ? 2 : 0);
  }
  const int64_t r = (int64_t)c.b * c.N + u;
  return c.rdeg[r] == 0 ? (c.sol[r] ? 2 : 1) : 0;
}

__device__ __forceinline__ int64_t phys_node(const PairwiseCtx &c, int64_t u) {
  if (c.P == 1) return (int64_t)c.b * c.rows_max + u;
  const int64_t big = c.extra * (c.base + 1);
  const int64_t r = u < big ? u / (c.base + 1) : c.extra + (u - big) / c.base;
  const int64_t start = r * c.base + (r < c.extra ? r : c.extra);
  return ((int64_t)c.b * c.P + r) * c.rows_max + (u - start);
}

template <class T>
__device__ __forceinline__ T load_node(const PairwiseCtx &c, int64_t u, int k) {
  if (c.dead) {
    const uint8_t code = dead_code(c, u);
    if (code) return reinterpret_cast<const T *>(c.dead)[(code - 1) * c.K + k];
  }
  int64_t phys;
  if (c.P == 1) {
    phys = (int64_t)c.b * c.rows_max + u;
  } else {
    const int64_t big = c.extra * (c.base + 1);
    const int64_t r = u < big ? u / (c.base + 1) : c.extra + (u - big) / c.base;
    const int64_t start = r * c.base + (r < c.extra ? r : c.extra);
    phys = ((int64_t)c.b * c.P + r) * c.rows_max + (u - start);
  }
  return reinterpret_cast<const T *>(c.h)[phys * c.K + k];
}

// grid (nleaves, ceil(K/32), B), block (32 k, 8 j)
template <class T>
__global__ void __launch_bounds__(256) colsum_leaf_kernel(PairwiseCtx c,
                                                          const int64_t *__restrict__ leaves,
                                                          int64_t nvals, T *__restrict__ vals) {
  __shared__ T part[8][32];
  c.b = blockIdx.z;
  const int leaf = blockIdx.x;
  const int kl = threadIdx.x, j = threadIdx.y;
  const int k = blockIdx.y * 32 + kl;
  const int64_t u0 = leaves[2 * leaf], n = leaves[2 * leaf + 1];
  const bool ok = k < c.K;
  if (n >= 8 && ok) {
    const int64_t stop = n - (n % 8);
    T r = load_node<T>(c, u0 + j, k);
    for (int64_t i = 8 + j; i < stop; i += 8) r = addT(r, load_node<T>(c, u0 + i, k));
    part[j][kl] = r;
  }
  __syncthreads();
  if (j == 0 && ok) {
    T res;
    int64_t i;
    if (n < 8) {
      res = T(0);
      i = 0;
    } else {
      res = addT(addT(addT(part[0][kl], part[1][kl]), addT(part[2][kl], part[3][kl])),
                 addT(addT(part[4][kl], part[5][kl]), addT(part[6][kl], part[7][kl])));
      i = n - (n % 8);
    }
    for (; i < n; i++) res = addT(res, load_node<T>(c, u0 + i, k));
    vals[((int64_t)c.b * nvals + leaf) * c.K + k] = res;
  }
}

// K = 64: one block of 512 threads per (leaf, slot), k = tid & 63 and
// accumulator j = tid >> 6.  In residual mode the leaf's rows are classified
// once into shared memory (0 = read h, 1/2 = dead row with sol 0/1), so the
// 64 x 8 chains read rdeg/sol from HBM once per row and h only for live rows.
template <class T>
__global__ void __launch_bounds__(512) colsum_leaf64_kernel(PairwiseCtx c,
                                                            const int64_t *__restrict__ leaves,
                                                            int64_t nvals, T *__restrict__ vals) {
  __shared__ T part[8][64];
  __shared__ T s_dead[2][64];
  __shared__ uint8_t s_code[128];
  c.b = blockIdx.y;
  const int leaf = blockIdx.x, tid = threadIdx.x;
  const int k = tid & 63, j = tid >> 6;
  const int64_t u0 = leaves[2 * leaf], n = leaves[2 * leaf + 1];
  const T *h = reinterpret_cast<const T *>(c.h);
  const bool res = c.dead != nullptr;
  if (res) {
    bool live = false;
    if (tid < n) {
      const int64_t r = (int64_t)c.b * c.N + u0 + tid;
      const uint8_t code = dead_code(c, u0 + tid);
      s_code[tid] = code;
      live = code == 0;
      if (c.last) {  // a row only ever goes live -> dead (rdeg never grows)
        live |= c.last[r] == 0;
        c.last[r] = code;
      }
    }
    if (tid < 128) s_dead[tid >> 6][k] = reinterpret_cast<const T *>(c.dead)[tid];
    // every row dead now and at the previous call (or, with leaf flags, no
    // row changed): the cached value stands
    const bool redo = c.leaf_dirty ? (c.full || c.leaf_dirty[leaf]) : (live || c.full || !c.last);
    if (!__syncthreads_or(redo)) return;
  }
  // generic pointer to row i's value: a dead row's lives in shared memory
  auto src = [&](int64_t i) -> const T * {
    if (res) {
      const int code = s_code[i];
      if (code) return &s_dead[code - 1][k];
    }
    return h + phys_node(c, u0 + i) * 64 + k;
  };
  auto val = [&](int64_t i) -> T { return *src(i); };
  if (n >= 8) {
    // all 16 loads of the chain issued before the sequential adds
    const int stop = (int)(n - (n % 8));
    T v[16];
#pragma unroll
    for (int t = 0; t < 16; t++) v[t] = (8 * t + j < stop) ? *src(8 * t + j) : T(0);
    T r = v[0];
#pragma unroll
    for (int t = 1; t < 16; t++)
      if (8 * t + j < stop) r = addT(r, v[t]);
    part[j][k] = r;
  }
  __syncthreads();
  if (j == 0) {
    T out;
    int64_t i;
    if (n < 8) {
      out = T(0);
      i = 0;
    } else {
      out = addT(addT(addT(part[0][k], part[1][k]), addT(part[2][k], part[3][k])),
                 addT(addT(part[4][k], part[5][k]), addT(part[6][k], part[7][k])));
      i = n - (n % 8);
    }
    for (; i < n; i++) out = addT(out, val(i));
    vals[((int64_t)c.b * nvals + leaf) * 64 + k] = out;
  }
}

// K = 64, 4 leaves per block of 256 threads: thread (leaf, k) runs all 8
// accumulator chains of its column itself, so every row of the leaf is one
// independent coalesced 256-byte load across the leaf's 64 threads (deep
// memory-level parallelism, 8 waves at 2^22 rows instead of 55).  Residual
// and incremental modes as colsum_leaf64_kernel.
constexpr int kLeavesPerBlock = 4;

template <class T>
__global__ void __launch_bounds__(256) colsum_leaf64x4_kernel(PairwiseCtx c,
                                                              const int64_t *__restrict__ leaves,
                                                              int nleaves, int64_t nvals,
                                                              T *__restrict__ vals) {
  __shared__ T s_dead[2][64];
  __shared__ uint8_t s_code[kLeavesPerBlock][128];
  __shared__ int s_live[kLeavesPerBlock];
  c.b = blockIdx.y;
  const int tid = threadIdx.x, k = tid & 63, ll = tid >> 6;
  const int leaf = blockIdx.x * kLeavesPerBlock + ll;
  const bool ok = leaf < nleaves;
  const int64_t u0 = ok ? leaves[2 * leaf] : 0, n = ok ? leaves[2 * leaf + 1] : 0;
  const T *h = reinterpret_cast<const T *>(c.h);
  const bool res = c.dead != nullptr;
  if (res) {
    if (tid < kLeavesPerBlock) {
      const int lf = blockIdx.x * kLeavesPerBlock + tid;
      s_live[tid] = (c.full || !c.last) ? 1
                    : (c.leaf_dirty && lf < nleaves && c.leaf_dirty[lf]) ? 1 : 0;
    }
    if (tid < 128) s_dead[tid >> 6][k] = reinterpret_cast<const T *>(c.dead)[tid];
    __syncthreads();
    bool live = false;
#pragma unroll
    for (int h2 = 0; h2 < 2; h2++) {  // the leaf's 64 threads classify its <= 128 rows
      const int i = k + 64 * h2;
      if (i < n) {
        const int64_t r = (int64_t)c.b * c.N + u0 + i;
        const uint8_t code = dead_code(c, u0 + i);
        s_code[ll][i] = code;
        live |= code == 0;
        if (c.last) {  // a row only ever goes live -> dead (rdeg never grows)
          live |= c.last[r] == 0;
          c.last[r] = code;
        }
      }
    }
    if (live && !c.leaf_dirty) s_live[ll] = 1;
    __syncthreads();
    if (!s_live[ll]) return;  // all dead now and at the previous call / unchanged
  }
  if (!ok) return;
  auto src = [&](int64_t i) -> const T * {
    if (res) {
      const int code = s_code[ll][i];
      if (code) return &s_dead[code - 1][k];
    }
    return h + phys_node(c, u0 + i) * 64 + k;
  };
  T out;
  int64_t i = 0;
  if (n < 8) {
    out = T(0);
  } else {
    const int stop = (int)(n - (n % 8));
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = *src(j);
    for (int base = 8; base < stop; base += 8) {
      T v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = *src(base + j);
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = addT(r[j], v[j]);
    }
    out = addT(addT(addT(r[0], r[1]), addT(r[2], r[3])), addT(addT(r[4], r[5]), addT(r[6], r[7])));
    i = stop;
  }
  for (; i < n; i++) out = addT(out, *src(i));
  vals[((int64_t)c.b * nvals + leaf) * 64 + k] = out;
}

// Every internal node of height >= first_level in one CTA (the top of the
// tree: few nodes per height), heights separated by __syncthreads.
template <class T>
__global__ void __launch_bounds__(1024) colsum_top_kernel(const int32_t *__restrict__ left,
                                                          const int32_t *__restrict__ right,
                                                          const int *__restrict__ lvl, int nlvl,
                                                          int nleaves, int64_t nvals, int K,
                                                          T *__restrict__ vals) {
  T *v = vals + (int64_t)blockIdx.x * nvals * K;
  for (int l = 0; l < nlvl; l++) {
    const int a = lvl[l], bnd = lvl[l + 1];
    for (int e = threadIdx.x; e < (bnd - a) * K; e += blockDim.x) {
      const int q = a + e / K, k = e % K;
      v[(int64_t)(nleaves + q) * K + k] =
          addT(v[(int64_t)left[q] * K + k], v[(int64_t)right[q] * K + k]);
    }
    __syncthreads();
  }
}

// vals[b][base + q] = vals[b][left[q]] + vals[b][right[q]] for q in [0, count)
template <class T>
__global__ void colsum_level_kernel(const int32_t *__restrict__ left,
                                    const int32_t *__restrict__ right, int count, int base,
                                    int64_t nvals, int K, T *__restrict__ vals) {
  const int b = blockIdx.y;
  T *v = vals + (int64_t)b * nvals * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)count * K;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(e / K), k = (int)(e - (int64_t)q * K);
    v[(int64_t)(base + q) * K + k] = addT(v[(int64_t)left[q] * K + k], v[(int64_t)right[q] * K + k]);
  }
}

template <class T>
__global__ void colsum_out_kernel(int root, int64_t nvals, int K, const T *__restrict__ vals,
                                  T *__restrict__ g) {
  const int b = blockIdx.x;
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    g[(int64_t)b * K + k] = addT(T(0), vals[((int64_t)b * nvals + root) * K + k]);
}

struct PairwisePlan {
  int64_t *d_leaves = nullptr;  // [nleaves][2] (start, len)
  int32_t *d_left = nullptr, *d_right = nullptr;  // internal nodes, by height
  int nleaves = 0, ninternal = 0, root = 0;
  std::vector<int> level_start;  // internal index ranges per height
  int *d_level_start = nullptr;  // the same ranges on the device
};

// returns (node id, height); ids < nleaves are leaves, internal nodes get
// provisional ids in creation order and are renumbered by height afterwards
static std::pair<int, int> plan_rec(int64_t u0, int64_t n, std::vector<int64_t> &leaves,
                                    std::vector<std::array<int, 3>> &internal) {
  if (n <= 128) {
    leaves.push_back(u0);
    leaves.push_back(n);
    return {(int)(leaves.size() / 2 - 1), 0};
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  auto l = plan_rec(u0, n2, leaves, internal);
  auto r = plan_rec(u0 + n2, n - n2, leaves, internal);
  int h = std::max(l.second, r.second) + 1;
  internal.push_back({l.first | (l.second ? (1 << 30) : 0), r.first | (r.second ? (1 << 30) : 0),
                      h});
  return {(int)internal.size() - 1, h};
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
    std::vector<int64_t> leaves;
    std::vector<std::array<int, 3>> internal;  // {left, right, height}; bit 30 = internal
    auto rootp = plan_rec(0, N, leaves, internal);
    PairwisePlan p;
    p.nleaves = (int)(leaves.size() / 2);
    p.ninternal = (int)internal.size();
    // renumber internal nodes by height (stable): id = nleaves + rank
    std::vector<int> order(internal.size());
    for (size_t q = 0; q < order.size(); q++) order[q] = (int)q;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return internal[a][2] < internal[b][2]; });
    std::vector<int> newid(internal.size());
    for (size_t q = 0; q < order.size(); q++) newid[order[q]] = p.nleaves + (int)q;
    auto resolve = [&](int x) { return (x & (1 << 30)) ? newid[x & ~(1 << 30)] : x; };
    std::vector<int32_t> left(internal.size()), right(internal.size());
    int cur_h = -1;
    for (size_t q = 0; q < order.size(); q++) {
      const auto &nd = internal[order[q]];
      left[q] = resolve(nd[0]);
      right[q] = resolve(nd[1]);
      if (nd[2] != cur_h) {
        p.level_start.push_back((int)q);
        cur_h = nd[2];
      }
    }
    p.level_start.push_back((int)internal.size());
    S2V_CUDA_CHECK(cudaMalloc(&p.d_level_start, sizeof(int) * p.level_start.size()));
    S2V_CUDA_CHECK(cudaMemcpy(p.d_level_start, p.level_start.data(),
                              sizeof(int) * p.level_start.size(), cudaMemcpyHostToDevice));
    p.root = rootp.second ? newid[rootp.first] : rootp.first;
    S2V_CUDA_CHECK(cudaMalloc(&p.d_leaves, sizeof(int64_t) * leaves.size()));
    S2V_CUDA_CHECK(cudaMemcpy(p.d_leaves, leaves.data(), sizeof(int64_t) * leaves.size(),
                              cudaMemcpyHostToDevice));
    if (!internal.empty()) {
      S2V_CUDA_CHECK(cudaMalloc(&p.d_left, sizeof(int32_t) * left.size()));
      S2V_CUDA_CHECK(cudaMalloc(&p.d_right, sizeof(int32_t) * right.size()));
      S2V_CUDA_CHECK(cudaMemcpy(p.d_left, left.data(), sizeof(int32_t) * left.size(),
                                cudaMemcpyHostToDevice));
      S2V_CUDA_CHECK(cudaMemcpy(p.d_right, right.data(), sizeof(int32_t) * right.size(),
                                cudaMemcpyHostToDevice));
    }
    it = cache.emplace(key, std::move(p)).first;
  }
  *out = &it->second;
  return S2V_OK;
}

// flags[leaf of u] = 1 for every row u of the list (leaf starts ascending)
__global__ void mark_leaves_kernel(const int64_t *__restrict__ leaves, int nleaves,
                                   const int32_t *__restrict__ rows,
                                   const int64_t *__restrict__ nrows, uint8_t *__restrict__ flags) {
  const int64_t n = nrows[0];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = rows[j];
    int lo = 0, hi = nleaves - 1;  // last leaf with start <= u
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (leaves[2 * mid] <= u)
        lo = mid;
      else
        hi = mid - 1;
    }
    flags[lo] = 1;
  }
}

template <class T>
static int colsum_t(const s2v_shard *sh, int K, const void *h, void *g, void *workspace,
                    size_t workspace_bytes, cudaStream_t st, const T *dead = nullptr,
                    uint8_t *last = nullptr, int full = 1, const int32_t *dirty_rows = nullptr,
                    const int64_t *ndirty = nullptr, uint8_t *flags = nullptr,
                    const int32_t *trow = nullptr, int max_deg = 0) {
  PairwisePlan *plan = nullptr;
  int rc = get_plan(sh->num_nodes, &plan);
  if (rc) return rc;
  const int64_t nvals = (int64_t)plan->nleaves + plan->ninternal;
  if (workspace_bytes < (size_t)nvals * sh->batch * K * sizeof(T))
    return fail(S2V_EINVAL, "colsum workspace too small");
  T *vals = (T *)workspace;
  PairwiseCtx c;
  c.h = h;
  c.N = sh->num_nodes;
  c.rows_max = sh->rows_max;
  c.P = sh->world;
  c.base = sh->num_nodes / sh->world;
  c.extra = sh->num_nodes % sh->world;
  c.K = K;
  c.b = 0;
  c.dead = dead;
  c.rdeg = sh->rdeg;
  c.sol = sh->sol;
  c.trow = trow;
  c.max_deg = max_deg;
  c.last = last;
  c.full = full;
  c.leaf_dirty = nullptr;
  if (last && K != 64) return fail(S2V_EINVAL, "incremental colsum needs K = 64");
  if (dirty_rows) {
    if (!last || !flags || sh->batch != 1) return fail(S2V_EINVAL, "bad dirty-row colsum args");
    S2V_CUDA_CHECK(cudaMemsetAsync(flags, 0, plan->nleaves, st));
    mark_leaves_kernel<<<kNumSMs * 2, 256, 0, st>>>(plan->d_leaves, plan->nleaves, dirty_rows,
                                                    ndirty, flags);
    S2V_LAUNCH_CHECK();
    c.leaf_dirty = flags;
  }
  if (K == 64) {
    static const bool x4 = [] {
      const char *e = getenv("S2V_COLSUM_X4");
      return !(e && e[0] == '0');
    }();
    if (x4)
      colsum_leaf64x4_kernel<T>
          <<<dim3((plan->nleaves + kLeavesPerBlock - 1) / kLeavesPerBlock, sh->batch), 256, 0,
             st>>>(c, plan->d_leaves, plan->nleaves, nvals, vals);
    else
      colsum_leaf64_kernel<T><<<dim3(plan->nleaves, sh->batch), 512, 0, st>>>(c, plan->d_leaves,
                                                                              nvals, vals);
  } else {
    dim3 lgrid(plan->nleaves, (K + 31) / 32, sh->batch);
    colsum_leaf_kernel<T><<<lgrid, dim3(32, 8), 0, st>>>(c, plan->d_leaves, nvals, vals);
  }
  S2V_LAUNCH_CHECK();
  const int nlv = (int)plan->level_start.size() - 1;
  int lv = 0;
  // wide heights: one launch each; the rest (<= 64 nodes per height): one CTA
  for (; lv < nlv; lv++) {
    const int a = plan->level_start[lv], bnd = plan->level_start[lv + 1];
    const int count = bnd - a;
    if (count <= 64) break;
    int64_t work = (int64_t)count * K;
    int blocks = (int)std::min<int64_t>((work + 255) / 256, kNumSMs * 8);
    colsum_level_kernel<T><<<dim3(blocks, sh->batch), 256, 0, st>>>(
        plan->d_left + a, plan->d_right + a, count, plan->nleaves + a, nvals, K, vals);
    S2V_LAUNCH_CHECK();
  }
  if (lv < nlv) {
    colsum_top_kernel<T><<<sh->batch, 1024, 0, st>>>(plan->d_left, plan->d_right,
                                                     plan->d_level_start + lv, nlv - lv,
                                                     plan->nleaves, nvals, K, vals);
    S2V_LAUNCH_CHECK();
  }
  colsum_out_kernel<T><<<sh->batch, 64, 0, st>>>(plan->root, nvals, K, vals, (T *)g);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

// ---------------------------------------------------------------------------
// Scores + selection keys, generic: one warp per local row.
// ---------------------------------------------------------------------------
constexpr int kTopK = 8;
constexpr int kScoreRowsPerBlock = 2048;

__device__ __forceinline__ void insert_top(Key (&top)[kTopK], const Key &k) {
  if (!key_gt(k, top[kTopK - 1])) return;
  int pos = kTopK - 1;
  while (pos > 0 && key_gt(k, top[pos - 1])) {
    top[pos] = top[pos - 1];
    pos--;
  }
  top[pos] = k;
}

// Merge the per-thread top lists of threads [0, n) (n a power of two, all
// threads of the block call this) through shared memory into out[0..8).
__device__ void block_merge_top(Key (&top)[kTopK], Key *s_keys /*[n*8]*/, Key *out,
                                int n = -1) {
  const int tid = threadIdx.x;
  if (n < 0) n = blockDim.x;
  if (tid < n)
    for (int q = 0; q < kTopK; q++) s_keys[tid * kTopK + q] = top[q];
  __syncthreads();
  for (int stride = n / 2; stride > 0; stride >>= 1) {
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
  // rows dealt to blocks in chunks of kScoreRowsPerBlock, round-robin
  for (int64_t c0 = (int64_t)blockIdx.x * kScoreRowsPerBlock; c0 < sh.num_rows;
       c0 += (int64_t)gridDim.x * kScoreRowsPerBlock)
  for (int64_t i = c0 + warp, c1 = min(c0 + kScoreRowsPerBlock, sh.num_rows); i < c1; i += 8) {
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

// K = 64 fp32 scorer: 128-row tiles.  The next tile's rows are copied into a
// row-major staging buffer by cp.async (no registers held) while the current
// tile is projected; each thread then moves the rows it copied into the
// transposed xT[p][row].  u2 = theta6 h as an 8-row x 4-k register-tiled FMA
// chain (p = 0..63 per output, the order numpy's sgemm uses; 3 shared loads
// per 32 FMAs), then one thread per row runs the sequential theta7
// contraction (mul then add, j = 0..127).  The candidate mask of
// q_forward's theta6 (h * cand) is applied to u2 instead of h: for a
// non-candidate row every x_p is +-0 (finite h) or NaN, so every chain of
// fl(h * 0) gives exactly +0 -- or NaN if the row holds a non-finite value
// -- which is what the masked chain computes, bit for bit.
constexpr int kScoreTile = 128;
constexpr size_t kScoreSmem = sizeof(float) * (64 * 68 + kScoreTile * 64 + kScoreTile * 68);

__global__ void __launch_bounds__(256, 2) score64_kernel(
    s2v_shard sh, const float *__restrict__ h, const float *__restrict__ u1,
    const float *__restrict__ theta6, const float *__restrict__ theta7,
    const uint8_t *__restrict__ cand_override, int mode, float *__restrict__ scores,
    Key *__restrict__ block_keys, int64_t *__restrict__ counts,
    float *__restrict__ prod_cache = nullptr, int emit = 1) {
  // prod_cache (nullable, [rows][64]): keep each row's fl(relu(u2) * theta7)
  // terms for score_sum64_kernel; emit = 0: only fill the cache
  extern __shared__ __align__(16) float score_smem[];
  float(*th6T)[68] = reinterpret_cast<float(*)[68]>(score_smem);  // th6T[p][k] = theta6[k][p]
  float *stage = score_smem + 64 * 68;                             // [128 rows][64], cp.async
  // xT[p][row] (4-row groups XOR-swizzled by (p >> 2) & 7); after the
  // projection the same storage holds prod[row][k] = fl(relu(u2) * theta7),
  // and at the end the key lists
  float *xT = stage + kScoreTile * 64;
  float(*prod)[68] = reinterpret_cast<float(*)[68]>(xT);
  __shared__ float s_t7[64];
  __shared__ uint8_t s_c[kScoreTile], s_nf[kScoreTile];
  __shared__ int32_t s_i[kScoreTile];
  __shared__ float s_s0;
  __shared__ unsigned long long s_count;
  Key *s_keys = reinterpret_cast<Key *>(xT);
  const int b = blockIdx.y, tid = threadIdx.x;
  // 128-row tiles are dealt to blocks round-robin (tile t -> block t mod
  // gridDim.x), so a short active list still spreads over every block
  const int64_t lim = sh.active ? sh.active_n[0] : sh.num_rows;
  if ((int64_t)blockIdx.x * kScoreTile >= lim) {
    // no tile for this block: no rows, no keys
    if (tid < kTopK) block_keys[((int64_t)b * gridDim.x + blockIdx.x) * kTopK + tid] = null_key();
    return;
  }
  const int64_t i0 = (int64_t)blockIdx.x * kScoreTile;
  const int64_t tstride = (int64_t)gridDim.x * kScoreTile;
  const int64_t i1 = lim;
  const int64_t base_r = (int64_t)b * sh.num_rows;
  const int64_t base_phys = ((int64_t)b * sh.world + sh.rank) * sh.rows_max;
  // copy role: chunk e = tid + 256 q (q = 0..7) is row (tid >> 4) + 16 q,
  // float4 column c16 = tid & 15
  const int c16 = tid & 15, crow = tid >> 4;
  auto issue = [&](int64_t t0) {
    if (t0 < i1) {
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const int row = crow + 16 * q;
        const int64_t j = t0 + row;
        if (j < i1) {
          const int64_t i = sh.active ? sh.active[j] : j;
          cp_async16(stage + row * 64 + c16 * 4, h + (base_phys + i) * 64 + c16 * 4);
        }
      }
    }
    cp_async_commit();
  };
  issue(i0);
  for (int idx = tid; idx < 64 * 64; idx += 256) th6T[idx % 64][idx / 64] = theta6[idx];
  if (tid < 64) s_t7[tid] = theta7[64 + tid];
  if (tid == 0) {
    float s0 = 0.f;
    for (int j = 0; j < 64; j++) s0 = __fadd_rn(s0, __fmul_rn(relu(u1[b * 64 + j]), theta7[j]));
    s_s0 = s0;
    s_count = 0;
  }
  Key top[kTopK];
#pragma unroll
  for (int q = 0; q < kTopK; q++) top[q] = null_key();
  unsigned long long cnt = 0;
  // compute role: rows rq*8 .. rq*8+7, k = kq*4 .. kq*4+3
  const int kq = tid & 15, rq = tid >> 4;
  for (int64_t t0 = i0; t0 < i1; t0 += tstride) {
    // this tile's row ids and candidate flags (one thread per row)
    if (tid < kScoreTile) {
      const int64_t j = t0 + tid;
      int32_t i = -1;
      uint8_t c = 0;
      if (j < i1) {
        i = (int32_t)(sh.active ? sh.active[j] : j);
        c = cand_override ? cand_override[base_r + i] : sh.cand[base_r + i];
      }
      s_i[tid] = i;
      s_c[tid] = c;
    }
    cp_async_wait<0>();
    __syncthreads();  // (also: the previous tile's prod / keys fully consumed)
    // rows this thread copied -> xT; a row's non-finite flag over its 16 lanes
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int row = crow + 16 * q;
      const float4 v = *reinterpret_cast<const float4 *>(stage + row * 64 + c16 * 4);
      const int rsw = row ^ ((c16 & 7) << 2);
      xT[(c16 * 4 + 0) * kScoreTile + rsw] = v.x;
      xT[(c16 * 4 + 1) * kScoreTile + rsw] = v.y;
      xT[(c16 * 4 + 2) * kScoreTile + rsw] = v.z;
      xT[(c16 * 4 + 3) * kScoreTile + rsw] = v.w;
      unsigned nf = !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
      nf |= __shfl_xor_sync(0xffffffffu, nf, 1);
      nf |= __shfl_xor_sync(0xffffffffu, nf, 2);
      nf |= __shfl_xor_sync(0xffffffffu, nf, 4);
      nf |= __shfl_xor_sync(0xffffffffu, nf, 8);
      if (c16 == 0) s_nf[row] = (uint8_t)nf;
    }
    __syncthreads();
    issue(t0 + tstride);  // the stage is free again
    float acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
      for (int c = 0; c < 4; c++) acc[a][c] = 0.f;
    const float *tb = &th6T[0][kq * 4];
    // rows rq*8 .. +3 and rq*8+4 .. +7 of p sit at xT[p][(rq*8) ^ (g << 2)]
    // and at that offset ^ 4, g = (p >> 2) & 7
    const float *xb[8];
#pragma unroll
    for (int g = 0; g < 8; g++) xb[g] = xT + ((rq * 8) ^ (g << 2));
#pragma unroll 1
    for (int p0 = 0; p0 < 64; p0 += 32) {  // (32-way unroll: g is a constant)
#pragma unroll
      for (int u = 0; u < 32; u++) {
        const int p = p0 + u, g = (u >> 2) & 7;
        const float4 t = *reinterpret_cast<const float4 *>(tb + p * 68);
        const float4 xa = *reinterpret_cast<const float4 *>(xb[g] + p * kScoreTile);
        const float4 xc = *reinterpret_cast<const float4 *>(xb[g ^ 1] + p * kScoreTile);
        const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xc.x, xc.y, xc.z, xc.w};
#pragma unroll
        for (int a = 0; a < 8; a++) {
          acc[a][0] = __fmaf_rn(t.x, xv[a], acc[a][0]);
          acc[a][1] = __fmaf_rn(t.y, xv[a], acc[a][1]);
          acc[a][2] = __fmaf_rn(t.z, xv[a], acc[a][2]);
          acc[a][3] = __fmaf_rn(t.w, xv[a], acc[a][3]);
        }
      }
    }
    __syncthreads();  // xT fully consumed before prod overwrites it
    const float4 t7 = *reinterpret_cast<const float4 *>(&s_t7[kq * 4]);
#pragma unroll
    for (int a = 0; a < 8; a++) {
      const int row = rq * 8 + a;
      // q_forward's theta6 (h * cand): a non-candidate row's chains are +0
      // (NaN if the row is not finite)
      const bool c = s_c[row] != 0;
      const float z = s_nf[row] ? __int_as_float(0x7fffffff) : 0.f;
      const float4 pv = make_float4(__fmul_rn(relu(c ? acc[a][0] : z), t7.x),
                                    __fmul_rn(relu(c ? acc[a][1] : z), t7.y),
                                    __fmul_rn(relu(c ? acc[a][2] : z), t7.z),
                                    __fmul_rn(relu(c ? acc[a][3] : z), t7.w));
      *reinterpret_cast<float4 *>(&prod[row][kq * 4]) = pv;
      const int32_t i = s_i[row];
      if (prod_cache && i >= 0)
        *reinterpret_cast<float4 *>(prod_cache + (int64_t)i * 64 + kq * 4) = pv;
    }
    __syncthreads();
    if (emit && tid < kScoreTile && t0 + tid < i1) {
      float sc = s_s0;
#pragma unroll
      for (int k4 = 0; k4 < 16; k4++) {
        const float4 v = *reinterpret_cast<const float4 *>(&prod[tid][4 * k4]);
        sc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(sc, v.x), v.y), v.z), v.w);
      }
      const int64_t i = s_i[tid];
      scores[base_r + i] = sc;
      const bool c = s_c[tid] != 0;
      const bool finite = isfinite(sc);
      if (c && finite) cnt++;
      if (c && (finite || mode == 1)) insert_top(top, make_key((double)sc, sh.row_start + i));
    }
  }
  cp_async_wait<0>();
  if (cnt) atomicAdd(&s_count, cnt);
  __syncthreads();  // prod fully consumed before the key lists reuse it
  block_merge_top(top, s_keys, block_keys + ((int64_t)b * gridDim.x + blockIdx.x) * kTopK,
                  kScoreTile);
  if (tid == 0 && s_count) atomicAdd((unsigned long long *)&counts[b], s_count);
}

// Scores of the active list from cached theta7 terms (incremental forward):
// score = s0 + sum_k prod_cache[row][k], the same sequential adds as
// score64_kernel, with s0 from this evaluation's u1.  A candidate's cached
// terms are current: its h_L is unchanged unless it was in the frontier,
// whose rows were refreshed by score64_kernel(emit = 0) first.  One thread
// per row, rows dealt round-robin; per-block top-8 keys and counts as
// score64_kernel (scores are not written).
__global__ void __launch_bounds__(256) score_sum64_kernel(s2v_shard sh,
                                                          const float *__restrict__ u1,
                                                          const float *__restrict__ theta7,
                                                          const float *__restrict__ prod_cache,
                                                          int mode, Key *__restrict__ block_keys,
                                                          int64_t *__restrict__ counts) {
  __shared__ Key s_keys[256 * kTopK];
  __shared__ float s_s0;
  __shared__ unsigned long long s_count;
  const int tid = threadIdx.x;
  if (tid == 0) {
    float s0 = 0.f;
    for (int j = 0; j < 64; j++) s0 = __fadd_rn(s0, __fmul_rn(relu(u1[j]), theta7[j]));
    s_s0 = s0;
    s_count = 0;
  }
  __syncthreads();
  Key top[kTopK];
#pragma unroll
  for (int q = 0; q < kTopK; q++) top[q] = null_key();
  unsigned long long cnt = 0;
  const int64_t n = sh.active_n[0];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + tid; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = sh.active[j];
    if (!sh.cand[i]) continue;
    const float4 *pc = reinterpret_cast<const float4 *>(prod_cache + (int64_t)i * 64);
    float sc = s_s0;
#pragma unroll
    for (int q = 0; q < 16; q++) {
      const float4 v = pc[q];
      sc = __fadd_rn(sc, v.x);
      sc = __fadd_rn(sc, v.y);
      sc = __fadd_rn(sc, v.z);
      sc = __fadd_rn(sc, v.w);
    }
    const bool finite = isfinite(sc);
    if (finite) cnt++;
    if (finite || mode == 1) insert_top(top, make_key((double)sc, sh.row_start + i));
  }
  if (cnt) atomicAdd(&s_count, cnt);
  block_merge_top(top, s_keys, block_keys + (int64_t)blockIdx.x * kTopK);
  if (tid == 0 && s_count) atomicAdd((unsigned long long *)&counts[0], s_count);
}

// Per-row selection keys from the scores (mode 0: candidates with a finite
// score; mode 1: every candidate), for the d > 8 path.
template <class T>
__global__ void score_keys_kernel(s2v_shard sh, const T *__restrict__ scores,
                                  const uint8_t *__restrict__ cand, int mode,
                                  Key *__restrict__ keys) {
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = r % sh.num_rows;
    const double s = (double)scores[r];
    const bool ok = cand[r] && (isfinite(s) || mode == 1);
    keys[r] = ok ? make_key(s, sh.row_start + i) : null_key();
  }
}

// Per-block top-8 among keys strictly below ceiling[b].
__global__ void topk_below_kernel(s2v_shard sh, const Key *__restrict__ keys,
                                  const Key *__restrict__ ceiling, Key *__restrict__ block_keys) {
  __shared__ Key s_keys[256 * kTopK];
  const int b = blockIdx.y;
  const Key ceil = ceiling[b];
  Key top[kTopK];
#pragma unroll
  for (int q = 0; q < kTopK; q++) top[q] = null_key();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sh.num_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Key k = keys[(int64_t)b * sh.num_rows + i];
    if (key_gt(ceil, k)) insert_top(top, k);
  }
  block_merge_top(top, s_keys, block_keys + ((int64_t)b * gridDim.x + blockIdx.x) * kTopK);
}

__global__ void topk_merge_kernel(const Key *__restrict__ block_keys, int nblk, int d,
                                  Key *__restrict__ top_out,
                                  const int64_t *__restrict__ active_n) {
  extern __shared__ unsigned char smem_raw[];
  Key *s_keys = reinterpret_cast<Key *>(smem_raw);
  const int b = blockIdx.x;
  Key top[kTopK];
#pragma unroll
  for (int q = 0; q < kTopK; q++) top[q] = null_key();
  const Key *src = block_keys + (int64_t)b * nblk * kTopK;
  // active-row list: only its first blocks hold keys (the rest are empty)
  int used = nblk;
  if (active_n) {
    const int64_t act_blk = (active_n[0] + kScoreTile - 1) / kScoreTile;  // blocks with a tile
    if (act_blk < used) used = (int)act_blk;
  }
  const int64_t total = (int64_t)used * kTopK;
  int64_t idx = threadIdx.x;
  for (; idx + 3 * blockDim.x < total; idx += 4 * blockDim.x) {
    Key k0 = src[idx], k1 = src[idx + blockDim.x], k2 = src[idx + 2 * blockDim.x],
        k3 = src[idx + 3 * blockDim.x];
    insert_top(top, k0);
    insert_top(top, k1);
    insert_top(top, k2);
    insert_top(top, k3);
  }
  for (; idx < total; idx += blockDim.x) insert_top(top, src[idx]);
  __shared__ Key s_out[kTopK];
  block_merge_top(top, s_keys, s_out);
  __syncthreads();
  if (threadIdx.x < d) top_out[(int64_t)b * d + threadIdx.x] = s_out[threadIdx.x];
}

template <class T>
static int embed_round_t(const s2v_shard *sh, const void *theta4, const void *table, int K,
                         int max_deg, const void *h_in, void *h_out, void *m_out,
                         cudaStream_t st, float *const *peers = nullptr, int npeers = 0,
                         bool from_table = false, const int32_t *deg_phys = nullptr) {
  const int64_t nrows = (int64_t)sh->batch * sh->num_rows;
  if (nrows == 0) return S2V_OK;
  if (from_table && !(sizeof(T) == 4 && K == 64 && (sh->world == 1 || deg_phys)))
    return fail(S2V_EINVAL, "degree-table rounds need K = 64 fp32 (and every rank's degrees "
                            "at P > 1)");
  const int32_t *deg_src = deg_phys ? deg_phys : sh->rdeg;
  if (sh->active && !(sizeof(T) == 4 && K == 64 && sh->batch == 1 &&
                      (sh->world == 1 || !sh->active_ptr || sh->active_sol)))
    return fail(S2V_EINVAL, "active-row lists need K = 64 fp32, B = 1 (compact CSR at P > 1: "
                            "active_sol)");
  if (sizeof(T) == 4 && K == 64) {
    static thread_local int *counter = nullptr;
    if (!counter) S2V_CUDA_CHECK(cudaMalloc(&counter, sizeof(int)));
    S2V_CUDA_CHECK(cudaMemsetAsync(counter, 0, sizeof(int), st));
    int64_t ntiles = (nrows + kTileRows - 1) / kTileRows;
    int grid = (int)std::min<int64_t>(ntiles, kNumSMs * 4);
    // rows kept in L2 with evict_last: the lowest physical ids -- the BA hubs,
    // 48 MB of rows source 31% of all gathers at BA(2M,16) (measured best of
    // 0/48/80/110 MB; S2V_HOT_MB overrides).  A persisting L2 carve-out
    // (cudaLimitPersistingL2CacheSize + access-policy window of 48/80/100 MB)
    // measured no better with these hints and worse without.
    uint32_t hot_rows;
    static const uint32_t hot_env = [] {
      const char *e = getenv("S2V_HOT_MB");
      return (uint32_t)(e ? atoi(e) : 48);
    }();
    hot_rows = (uint32_t)(((uint64_t)hot_env << 20) / 256);
    SideStream *ss = nullptr;
    auto hub_kern = from_table ? &hub_round64_kernel<true> : &hub_round64_kernel<false>;
    auto kern = from_table ? &round64_kernel<true> : &round64_kernel<false>;
    S2V_CUDA_CHECK(cudaFuncSetAttribute(hub_kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kHubSmem));
    int rc = with_hub_kernel(sh, st, [&](cudaStream_t hs, int *hub_counter) {
      int hgrid = (int)std::min<int64_t>(sh->n_hub, kNumSMs);
      hub_kern<<<hgrid, 256, kHubSmem, hs>>>(
          *sh, (const float *)theta4, (const float *)table, max_deg, (const float *)h_in,
          (float *)h_out, (float *)m_out, hub_counter, hot_rows, peers, npeers, deg_src);
    }, &ss);
    if (rc) return rc;
    static const int sparse_max = [] {
      const char *e = getenv("S2V_SPARSE_MAX");
      return e ? atoi(e) : kSparseMax;
    }();
    kern<<<grid, 256, 0, st>>>(*sh, (const float *)theta4, (const float *)table, max_deg,
                               (const float *)h_in, (float *)h_out, (float *)m_out, counter,
                               hot_rows, peers, npeers, deg_src, sparse_max, g8_prefetch());
    S2V_LAUNCH_CHECK();
    if (ss) S2V_CUDA_CHECK(cudaStreamWaitEvent(st, ss->done, 0));
    S2V_LAUNCH_CHECK();
    return S2V_OK;
  }
  if (npeers) return fail(S2V_EINVAL, "fused peer rounds need K = 64 fp32");
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

// dead rows' embedding: rows sol ? max_deg+1 : 0 of the h1 table, packed
template <class T>
__global__ void dead_rows_kernel(const T *__restrict__ h1_table, int K, int max_deg,
                                 T *__restrict__ dead) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    dead[k] = h1_table[k];
    dead[K + k] = h1_table[(int64_t)(max_deg + 1) * K + k];
  }
}

// ed[e] = degree of entry e's neighbour (removed entries keep their bit):
// the table row round 2 gathers for that entry
__global__ void edge_degree_kernel(const uint32_t *__restrict__ cols,
                                   const int32_t *__restrict__ deg, int64_t nnz,
                                   uint32_t *__restrict__ ed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cols[e];
    ed[e] = (c & S2V_DEAD) ? c : (uint32_t)__ldg(deg + c);
  }
}

}  // namespace s2v

using namespace s2v;

extern "C" {

int s2v_e12_table(s2v_dtype dt, const void *theta1, const void *theta2, const void *theta3,
                  int K, int max_deg, void *table, void *stream) {
  if (K < 1 || max_deg < 0) return fail(S2V_EINVAL, "bad e12 table args");
  int64_t total = (int64_t)(max_deg + 2) * K;
  int grid = (int)std::min<int64_t>((total + 255) / 256, kNumSMs * 8);
  if (K > 256) return fail(S2V_EINVAL, "embed_dim %d > 256 unsupported", K);
  size_t elem = dt == S2V_F32 ? 4 : 8;
  size_t smem = elem * ((size_t)K * (K + 1) + K);
  if (dt == S2V_F32) {
    S2V_CUDA_CHECK(cudaFuncSetAttribute(e12_table_kernel<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    e12_table_kernel<float><<<grid, 256, smem, as_stream(stream)>>>(
        (const float *)theta1, (const float *)theta2, (const float *)theta3, K, max_deg,
        (float *)table);
  } else {
    S2V_CUDA_CHECK(cudaFuncSetAttribute(e12_table_kernel<double>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    e12_table_kernel<double><<<grid, 256, smem, as_stream(stream)>>>(
        (const double *)theta1, (const double *)theta2, (const double *)theta3, K, max_deg,
        (double *)table);
  }
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_embed_round_peers(s2v_dtype dt, const s2v_shard *sh, const void *theta4,
                          const void *table, int K, int max_deg, const void *h_in, void *h_out,
                          void *const *peer_outs, int npeers, void *m_out, void *stream) {
  if (dt != S2V_F32 || K != 64)
    return fail(S2V_EINVAL, "fused peer rounds need K = 64 fp32");
  return embed_round_t<float>(sh, theta4, table, K, max_deg, h_in, h_out, m_out,
                              as_stream(stream), (float *const *)peer_outs, npeers);
}

int s2v_h1_table(s2v_dtype dt, const void *theta4, const void *table, int K, int max_deg,
                 void *h1_table, void *stream) {
  if (dt != S2V_F32 || K != 64) return fail(S2V_EINVAL, "h1 table needs K = 64 fp32");
  if (max_deg < 0) return fail(S2V_EINVAL, "bad h1 table args");
  const int rows = max_deg + 2;
  h1_table_kernel<<<(int)std::min<int64_t>(((int64_t)rows * 64 + 255) / 256, kNumSMs * 4), 256, 0,
                    as_stream(stream)>>>(
      (const float *)theta4, (const float *)table, rows, (float *)h1_table);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_embed_round2_table(s2v_dtype dt, const s2v_shard *sh, const void *theta4,
                           const void *table, int K, int max_deg, const void *h1_table,
                           const int32_t *deg_phys, void *h_out, void *const *peer_outs,
                           int npeers, void *m_out, void *stream) {
  if (dt != S2V_F32) return fail(S2V_EINVAL, "degree-table rounds need K = 64 fp32");
  static const bool edge_pass = [] {
    const char *e = getenv("S2V_EDGE_DEG");
    return !(e && e[0] == '0');
  }();
  // a table too large for L1 reuse (hub degrees nearly unique per hub: R-MAT
  // scale 22 has a 41 MB table) is read from L2 either way; there the
  // dependent degree lookup per neighbour is the cost, so it moves into a
  // separate streaming pass (measured: 3.86 -> 3.0 + 0.43 ms at R-MAT scale
  // 22; at BA(2M,16), 2.4 MB table, the in-gather lookup is 0.2 ms faster)
  const bool big_table = (int64_t)(max_deg + 2) * 256 > (8ll << 20);
  // (whole-graph rounds only: an active list or frontier visits few rows,
  // and the pass would touch every entry)
  if (edge_pass && big_table && K == 64 && !sh->active && sh->nnz > 0 &&
      (sh->world == 1 || deg_phys)) {
    // stream pass: every entry's neighbour degree (random 4-byte reads with
    // full memory-level parallelism), then a plain round over those table
    // indices -- the round's gather loses its dependent degree lookup
    static thread_local uint32_t *ed = nullptr;
    static thread_local int64_t cap = 0;
    static thread_local int ed_dev = -1;
    int dev = 0;
    S2V_CUDA_CHECK(cudaGetDevice(&dev));
    if (sh->nnz > cap || dev != ed_dev) {
      if (ed && dev == ed_dev) S2V_CUDA_CHECK(cudaFree(ed));
      S2V_CUDA_CHECK(cudaMalloc(&ed, sizeof(uint32_t) * sh->nnz));
      cap = sh->nnz;
      ed_dev = dev;
    }
    cudaStream_t st = as_stream(stream);
    edge_degree_kernel<<<(int)std::min<int64_t>((sh->nnz + 255) / 256, kNumSMs * 8), 256, 0,
                         st>>>(sh->cols, deg_phys ? deg_phys : sh->rdeg, sh->nnz, ed);
    S2V_LAUNCH_CHECK();
    s2v_shard e = *sh;
    e.cols = ed;
    return embed_round_t<float>(&e, theta4, table, K, max_deg, h1_table, h_out, m_out, st,
                                (float *const *)peer_outs, npeers, false, nullptr);
  }
  return embed_round_t<float>(sh, theta4, table, K, max_deg, h1_table, h_out, m_out,
                              as_stream(stream), (float *const *)peer_outs, npeers, true,
                              deg_phys);
}

// trow[phys row] = sol ? max_deg + 1 : rdeg for this rank's rows
__global__ void trow_kernel(s2v_shard sh, int max_deg, int32_t *__restrict__ trow) {
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
    trow[(b * sh.world + sh.rank) * sh.rows_max + i] = sh.sol[r] ? max_deg + 1 : sh.rdeg[r];
  }
}

int s2v_trow(const s2v_shard *sh, int max_deg, int32_t *trow_phys, void *stream) {
  const int64_t nrows = (int64_t)sh->batch * sh->num_rows;
  if (nrows == 0) return S2V_OK;
  trow_kernel<<<(int)std::min<int64_t>((nrows + 255) / 256, kNumSMs * 8), 256, 0,
                as_stream(stream)>>>(*sh, max_deg, trow_phys);
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
  // leaves have > 56 elements unless N < 128; nodes = 2 * leaves - 1
  int64_t nleaves = sh->num_nodes / 56 + 2;
  return (size_t)(2 * nleaves) * sh->batch * K * elem_bytes;
}

int s2v_colsum(s2v_dtype dt, const s2v_shard *sh, int K, const void *h, void *g,
               void *workspace, size_t workspace_bytes, void *stream) {
  if (dt == S2V_F32)
    return colsum_t<float>(sh, K, h, g, workspace, workspace_bytes, as_stream(stream));
  return colsum_t<double>(sh, K, h, g, workspace, workspace_bytes, as_stream(stream));
}

size_t s2v_colsum_residual_workspace(const s2v_shard *sh, int K, int elem_bytes) {
  // tree values, the two dead-row embeddings, one flag byte per leaf
  return s2v_colsum_workspace(sh, K, elem_bytes) + 2 * (size_t)K * elem_bytes +
         (size_t)(sh->num_nodes / 56 + 2) + 16;
}

int s2v_colsum_residual(s2v_dtype dt, const s2v_shard *sh, int K, const void *h,
                        const void *h1_table, int max_deg, void *g, void *workspace,
                        size_t workspace_bytes, uint8_t *last, int full,
                        const int32_t *dirty_rows, const int64_t *ndirty,
                        const int32_t *trow_phys, void *stream) {
  if (sh->world != 1 && !trow_phys)
    return fail(S2V_EINVAL, "residual colsum at P > 1 needs every rank's e12 rows (trow)");
  if (max_deg < 0 || !h1_table) return fail(S2V_EINVAL, "bad residual colsum args");
  cudaStream_t st = as_stream(stream);
  const size_t elem = dt == S2V_F32 ? 4 : 8;
  const size_t need = s2v_colsum_workspace(sh, K, (int)elem);
  if (workspace_bytes < s2v_colsum_residual_workspace(sh, K, (int)elem))
    return fail(S2V_EINVAL, "residual colsum workspace too small");
  void *dead = (char *)workspace + need;  // after the tree values
  uint8_t *flags = (uint8_t *)dead + 2 * K * elem;
  if (dt == S2V_F32) {
    dead_rows_kernel<float><<<1, 64, 0, st>>>((const float *)h1_table, K, max_deg, (float *)dead);
    S2V_LAUNCH_CHECK();
    return colsum_t<float>(sh, K, h, g, workspace, need, st, (const float *)dead, last, full,
                           dirty_rows, ndirty, flags, sh->world > 1 ? trow_phys : nullptr, max_deg);
  }
  dead_rows_kernel<double><<<1, 64, 0, st>>>((const double *)h1_table, K, max_deg,
                                             (double *)dead);
  S2V_LAUNCH_CHECK();
  return colsum_t<double>(sh, K, h, g, workspace, need, st, (const double *)dead, last, full,
                          dirty_rows, ndirty, flags, sh->world > 1 ? trow_phys : nullptr, max_deg);
}

int s2v_score_blocks(const s2v_shard *sh) {
  // one resident wave of score64_kernel (2 CTAs per SM) at most; rows are
  // dealt round-robin
  int64_t n = (sh->num_rows + kScoreRowsPerBlock - 1) / kScoreRowsPerBlock;
  if (n > kNumSMs * 2) n = kNumSMs * 2;
  return (int)(n < 1 ? 1 : n);
}

int s2v_score(s2v_dtype dt, const s2v_shard *sh, int K, const void *h, const void *u1,
              const void *theta6, const void *theta7, const uint8_t *cand_override, int mode,
              void *scores, uint64_t *block_keys, int64_t *counts, void *stream) {
  if (K > 256) return fail(S2V_EINVAL, "embed_dim %d > 256 unsupported", K);
  if (sh->active && !(dt == S2V_F32 && K == 64 && sh->batch == 1))
    return fail(S2V_EINVAL, "active-row lists need K = 64 fp32, B = 1");
  cudaStream_t st = as_stream(stream);
  S2V_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(int64_t) * sh->batch, st));
  dim3 grid(s2v_score_blocks(sh), sh->batch);
  size_t elem = dt == S2V_F32 ? 4 : 8;
  size_t smem = elem * ((size_t)K * (K + 1) + 16 * (size_t)K) + sizeof(Key) * 256 * kTopK;
  if (dt == S2V_F32 && K == 64) {
    S2V_CUDA_CHECK(cudaFuncSetAttribute(score64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kScoreSmem));
    score64_kernel<<<grid, 256, kScoreSmem, st>>>(*sh, (const float *)h, (const float *)u1,
                                         (const float *)theta6, (const float *)theta7,
                                         cand_override, mode, (float *)scores, (Key *)block_keys,
                                         counts);
  } else if (dt == S2V_F32) {
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

int s2v_score_cached(const s2v_shard *sh, const float *h, const float *u1, const float *theta6,
                     const float *theta7, int mode, float *prod_cache, const int32_t *rows,
                     const int64_t *nrows, float *scores, uint64_t *block_keys, int64_t *counts,
                     void *stream) {
  if (!sh->active || sh->batch != 1 || !prod_cache)
    return fail(S2V_EINVAL, "cached scores need an active-row list, B = 1");
  cudaStream_t st = as_stream(stream);
  S2V_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(int64_t), st));
  const int nblk = s2v_score_blocks(sh);
  if (!rows) {  // every active row: scores, keys, and the cache
    S2V_CUDA_CHECK(cudaFuncSetAttribute(score64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kScoreSmem));
    score64_kernel<<<dim3(nblk, 1), 256, kScoreSmem, st>>>(*sh, h, u1, theta6, theta7, nullptr, mode,
                                                  scores, (Key *)block_keys, counts, prod_cache, 1);
    S2V_LAUNCH_CHECK();
    return S2V_OK;
  }
  s2v_shard fr = *sh;  // refresh the cached terms of the frontier rows
  fr.active = rows;
  fr.active_n = nrows;
  fr.active_ptr = nullptr;
  fr.active_cols = nullptr;
  S2V_CUDA_CHECK(cudaFuncSetAttribute(score64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kScoreSmem));
  score64_kernel<<<dim3(nblk, 1), 256, kScoreSmem, st>>>(fr, h, u1, theta6, theta7, nullptr, mode, scores,
                                                (Key *)block_keys, counts, prod_cache, 0);
  S2V_LAUNCH_CHECK();
  score_sum64_kernel<<<nblk, 256, 0, st>>>(*sh, u1, theta7, prod_cache, mode, (Key *)block_keys,
                                           counts);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_score_keys(const s2v_shard *sh, const void *scores, const uint8_t *cand, int mode,
                   uint64_t *keys_all, void *stream) {
  int64_t rows = (int64_t)sh->batch * sh->num_rows;
  if (rows == 0) return S2V_OK;
  int grid = (int)std::min<int64_t>((rows + 255) / 256, kNumSMs * 8);
  score_keys_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(*sh, (const float *)scores, cand,
                                                                mode, (Key *)keys_all);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_score_keys_f64(const s2v_shard *sh, const void *scores, const uint8_t *cand, int mode,
                       uint64_t *keys_all, void *stream) {
  int64_t rows = (int64_t)sh->batch * sh->num_rows;
  if (rows == 0) return S2V_OK;
  int grid = (int)std::min<int64_t>((rows + 255) / 256, kNumSMs * 8);
  score_keys_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
      *sh, (const double *)scores, cand, mode, (Key *)keys_all);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_topk_below(const s2v_shard *sh, const uint64_t *keys_all, const uint64_t *ceiling,
                   uint64_t *block_keys, void *stream) {
  dim3 grid(s2v_score_blocks(sh), sh->batch);
  topk_below_kernel<<<grid, 256, 0, as_stream(stream)>>>(*sh, (const Key *)keys_all,
                                                         (const Key *)ceiling, (Key *)block_keys);
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
  topk_merge_kernel<<<sh->batch, 256, smem, as_stream(stream)>>>(
      (const Key *)block_keys, nblk, d, (Key *)top, sh->active ? sh->active_n : nullptr);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // extern "C"
