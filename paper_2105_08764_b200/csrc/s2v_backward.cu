// Hand-written DQN backward + Adam (sm_100a).
//
// Replaces (paths relative to /root/reference):
//   loss_and_gradients   pkg/src/graphrl/policy.py:232-315
//     head grads at the action nodes         policy.py:256-283
//     dg all-reduce + broadcast              policy.py:285-288
//     layer loop: dz, theta grads, dm, spmm_t policy.py:290-304, state.py:164-169
//     theta2 grad                            policy.py:305-306
//     fp64 gradient pack                     policy.py:308-314
//   adam_step            pkg/src/graphrl/policy.py:339-359
//
// Parity bar for gradients/losses is 1e-4 relative, so the
// K x K reductions use per-CTA partial sums in the parameter dtype and a
// fixed-order fp64 reduction over CTAs: deterministic, hence bit-identical
// replicas on every rank.  Adam follows the reference's element-wise fp32
// rounding sequence exactly.
#include <cstdlib>

#include "s2v_common.cuh"
#include "s2v_gather.cuh"

namespace s2v {

constexpr int kBwdTile = 16;     // rows per tile
constexpr int kBwdThreads = 256;

inline int bwd_blocks(const s2v_shard &sh) {
  int64_t rows = (int64_t)sh.batch * sh.num_rows;
  int64_t tiles = (rows + kBwdTile - 1) / kBwdTile;
  int64_t nb = tiles < kNumSMs * 2 ? tiles : kNumSMs * 2;
  return (int)(nb < 1 ? 1 : nb);
}

__device__ __forceinline__ int64_t phys_of_row(const s2v_shard &sh, int64_t r) {
  if (sh.world == 1 && sh.rows_max == sh.num_rows) return r;  // P = 1: identity
  const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
  return (b * sh.world + sh.rank) * sh.rows_max + i;
}

// grad_h[r] = dg[b] (+ dact[b] at the action row of slot b)
template <class T>
__global__ void grad_h_init_kernel(s2v_shard sh, int K, const T *__restrict__ dg,
                                   const int64_t *__restrict__ actions,
                                   const T *__restrict__ dact, T *__restrict__ grad_h) {
  const int64_t total = (int64_t)sh.batch * sh.num_rows * K;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / K;
    const int k = (int)(idx - r * K);
    const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
    T v = dg[b * K + k];
    if (actions[b] == sh.row_start + i) v = addT(v, dact[b * K + k]);
    grad_h[idx] = v;
  }
}

// K = 64 fp32: one float4 per thread, slot from the grid's y (no integer
// division per element); a thread's column quad is fixed (stride % 16 == 0)
__global__ void grad_h_init64_kernel(s2v_shard sh, const float *__restrict__ dg,
                                     const int64_t *__restrict__ actions,
                                     const float *__restrict__ dact, float *__restrict__ grad_h) {
  const int b = blockIdx.y, c4 = threadIdx.x & 15;
  const float4 g = reinterpret_cast<const float4 *>(dg + (int64_t)b * 64)[c4];
  const int64_t act = actions[b] - sh.row_start;  // local row of the action, if owned
  const int64_t n4 = sh.num_rows * 16;
  float4 *out = reinterpret_cast<float4 *>(grad_h + (int64_t)b * sh.num_rows * 64);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4;
       q += (int64_t)gridDim.x * blockDim.x) {
    float4 v = g;
    if ((q >> 4) == act) {
      const float4 a = reinterpret_cast<const float4 *>(dact + (int64_t)b * 64)[c4];
      v.x = __fadd_rn(v.x, a.x);
      v.y = __fadd_rn(v.y, a.y);
      v.z = __fadd_rn(v.z, a.z);
      v.w = __fadd_rn(v.w, a.w);
    }
    out[q] = v;
  }
}

// Layer backward over tiles of kBwdTile local rows.
//   dz = grad_h * (h_l > 0); dzsum += dz; P4 += dz (x) m_l; dm = theta4^T dz
template <class T>
__global__ void __launch_bounds__(kBwdThreads) layer_backward_kernel(
    s2v_shard sh, int K, const T *__restrict__ theta4, const T *__restrict__ grad_h,
    const T *__restrict__ h_l, const T *__restrict__ m_l, T *__restrict__ dzsum,
    T *__restrict__ partial, int first, T *__restrict__ dm_out) {
  extern __shared__ unsigned char smem_raw[];
  T *th = reinterpret_cast<T *>(smem_raw);  // [K][K+1] theta4
  T *dz_s = th + K * (K + 1);               // [tile][K]
  T *m_s = dz_s + kBwdTile * K;             // [tile][K]
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x)
    th[(idx / K) * (K + 1) + (idx % K)] = theta4[idx];
  const int KK = K * K;
  const int per = (KK + blockDim.x - 1) / blockDim.x;  // outputs per thread (<= 64)
  T acc[64];
  for (int t = 0; t < per && t < 64; t++) {
    int o = threadIdx.x + t * blockDim.x;
    acc[t] = (!first && o < KK) ? partial[(int64_t)blockIdx.x * KK + o] : T(0);
  }
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t ntiles = (nrows + kBwdTile - 1) / kBwdTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kBwdTile;
    __syncthreads();
    for (int e = threadIdx.x; e < kBwdTile * K; e += blockDim.x) {
      const int lr = e / K, k = e - lr * K;
      const int64_t r = r0 + lr;
      T dz = T(0), m = T(0);
      if (r < nrows) {
        const T hv = h_l[phys_of_row(sh, r) * K + k];
        dz = (hv > T(0)) ? grad_h[r * K + k] : T(0);
        dzsum[r * K + k] = first ? dz : addT(dzsum[r * K + k], dz);
        if (m_l) m = m_l[r * K + k];
      }
      dz_s[e] = dz;
      m_s[e] = m;
    }
    __syncthreads();
    if (m_l) {
      for (int t = 0; t < per && t < 64; t++) {
        const int o = threadIdx.x + t * blockDim.x;
        if (o >= KK) break;
        const int k = o / K, j = o - k * K;
        T a = acc[t];
        for (int lr = 0; lr < kBwdTile; lr++) a = fmaT(dz_s[lr * K + k], m_s[lr * K + j], a);
        acc[t] = a;
      }
    }
    if (dm_out) {
      for (int e = threadIdx.x; e < kBwdTile * K; e += blockDim.x) {
        const int lr = e / K, j = e - lr * K;
        const int64_t r = r0 + lr;
        if (r >= nrows) continue;
        T a = T(0);
        for (int k = 0; k < K; k++) a = fmaT(th[k * (K + 1) + j], dz_s[lr * K + k], a);
        dm_out[phys_of_row(sh, r) * K + j] = a;
      }
    }
  }
  for (int t = 0; t < per && t < 64; t++) {
    int o = threadIdx.x + t * blockDim.x;
    if (o < KK) partial[(int64_t)blockIdx.x * KK + o] = acc[t];
  }
}

// out[r] = sum over alive neighbours (ascending) of src[phys]; one warp per row.
template <class T>
__global__ void gather_kernel(s2v_shard sh, int K, const T *__restrict__ src,
                              T *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < nrows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    for (int k0 = 0; k0 < K; k0 += 32) {
      const int k = k0 + lane;
      T a = T(0);
      if (!sh.sol[r])
        for (int64_t e = sh.row_ptr[r]; e < sh.row_ptr[r + 1]; e++) {
          const uint32_t c = sh.cols[e];
          if (c & S2V_DEAD) continue;
          if (k < K) a = addT(a, src[(int64_t)c * K + k]);
        }
      if (k < K) out[r * K + k] = a;
    }
  }
}

// Partials of dtheta1 [K], dtheta2 [K], dtheta3 [K][K] from dzsum.
template <class T>
__global__ void __launch_bounds__(kBwdThreads) param_grads_kernel(
    s2v_shard sh, int K, const T *__restrict__ theta2, const T *__restrict__ theta3,
    const T *__restrict__ dzsum, T *__restrict__ partial, T *__restrict__ t2c) {
  extern __shared__ unsigned char smem_raw[];
  T *th3 = reinterpret_cast<T *>(smem_raw);  // [K][K+1]
  T *dz_s = th3 + K * (K + 1);               // [tile][K]
  T *w_s = dz_s + kBwdTile * K;              // [tile][K]
  T *aux = w_s + kBwdTile * K;               // [tile][2]: sol, deg
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x)
    th3[(idx / K) * (K + 1) + (idx % K)] = theta3[idx];
  const int LEN = 2 * K + K * K;
  const int per = (LEN + blockDim.x - 1) / blockDim.x;
  T acc[72];
  for (int t = 0; t < per && t < 72; t++) acc[t] = T(0);
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t ntiles = (nrows + kBwdTile - 1) / kBwdTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kBwdTile;
    __syncthreads();
    for (int e = threadIdx.x; e < kBwdTile * K; e += blockDim.x) {
      const int lr = e / K, k = e - lr * K;
      const int64_t r = r0 + lr;
      T dz = T(0), w = T(0);
      if (r < nrows) {
        dz = dzsum[r * K + k];
        const T deg = sh.sol[r] ? T(0) : T(sh.rdeg[r]);
        w = relu(mulT(theta2[k], deg));
        if (k == 0) {
          aux[2 * lr] = sh.sol[r] ? T(1) : T(0);
          aux[2 * lr + 1] = deg;
        }
      } else if (k == 0) {
        aux[2 * lr] = T(0);
        aux[2 * lr + 1] = T(0);
      }
      dz_s[e] = dz;
      w_s[e] = w;
    }
    __syncthreads();
    for (int t = 0; t < per && t < 72; t++) {
      const int o = threadIdx.x + t * blockDim.x;
      if (o >= LEN) break;
      T a = acc[t];
      if (o < K) {  // dtheta1[k] = sum dz * sol
        for (int lr = 0; lr < kBwdTile; lr++) a = fmaT(dz_s[lr * K + o], aux[2 * lr], a);
      } else if (o < 2 * K) {  // dtheta2[j] = sum (theta3^T dz)_j * (w_j > 0) * deg
        const int j = o - K;
        for (int lr = 0; lr < kBwdTile; lr++) {
          const bool pos = w_s[lr * K + j] > T(0);
          if (!pos && !t2c) continue;
          T dw = T(0);
          for (int k = 0; k < K; k++) dw = fmaT(th3[k * (K + 1) + j], dz_s[lr * K + k], dw);
          if (pos) a = fmaT(dw, aux[2 * lr + 1], a);
          if (t2c && r0 + lr < nrows) {  // einsum term fl(fl(dw * (w > 0)) * deg)
            const int64_t r = r0 + lr, b = r / sh.num_rows, v = r - b * sh.num_rows;
            constexpr int G = 32 / sizeof(T);
            const int ng = (K + G - 1) / G;
            t2c[((b * ng + j / G) * sh.num_rows + v) * G + j % G] =
                mulT(mulT(dw, pos ? T(1) : T(0)), aux[2 * lr + 1]);
          }
        }
      } else {  // dtheta3[k][j] = sum dz_k w_j
        const int q = o - 2 * K, k = q / K, j = q - k * K;
        for (int lr = 0; lr < kBwdTile; lr++) a = fmaT(dz_s[lr * K + k], w_s[lr * K + j], a);
      }
      acc[t] = a;
    }
  }
  for (int t = 0; t < per && t < 72; t++) {
    int o = threadIdx.x + t * blockDim.x;
    if (o < LEN) partial[(int64_t)blockIdx.x * LEN + o] = acc[t];
  }
}

// dtheta2 in numpy's einsum order (policy.py:305-306,
// np.einsum("bkv,bv->k", dw_acc * (w > 0), deg)).  numpy 2.3's two-operand
// reduction with an outstride-0 inner loop over v
// (float/double_sum_of_products_contig_contig_outstride0_two, SSE baseline:
// LANES = 16 / sizeof(T) lanes, 4-vector unroll applied in the order
// v3, v2, v1, v0, mul then add, a zero-filled tail of LANES-wide vectors,
// lanes combined as (a0 + a1) + (a2 + a3)) gives, for each (b, k), LANES
// sequential chains over v; the per-b results are then added in b order.
// The cancellation in this 4M-term sum at BA(2M,16) (|sum| << sum |term|)
// makes it order-sensitive, so the device follows the same order
// (pinned by tests/test_gpu_fullsize.py; emulated in oracle/port.py).
// One CTA per (slot b, group of G = 32 / sizeof(T) columns): 3-stage cp.async
// ring of kEinRows-row chunks of the chain layout, one warp runs the chains.
constexpr int kEinRows = 1024;
constexpr int kEinStages = 3;

template <class T>
__global__ void __launch_bounds__(256) theta2_einsum_kernel(const T *__restrict__ t2c,
                                                            int64_t rows, int K,
                                                            T *__restrict__ tot) {
  constexpr int G = 32 / sizeof(T), LANES = 16 / sizeof(T), BLK = 4 * LANES;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *ring = reinterpret_cast<T *>(smem_raw);  // [kEinStages][kEinRows][G]
  const int ng = (K + G - 1) / G;
  const int b = blockIdx.x / ng, grp = blockIdx.x - b * ng;
  const T *src = t2c + ((int64_t)b * ng + grp) * rows * G;
  const int64_t nchunks = (rows + kEinRows - 1) / kEinRows;
  auto issue = [&](int64_t c) {
    if (c < nchunks) {
      const int64_t base = c * kEinRows;
      const int64_t n16 = ((rows - base < kEinRows ? rows - base : kEinRows) * G * sizeof(T)) / 16;
      T *dst = ring + (c % kEinStages) * kEinRows * G;
      for (int64_t e = threadIdx.x; e < n16; e += blockDim.x)
        cp_async16(reinterpret_cast<char *>(dst) + 16 * e,
                   reinterpret_cast<const char *>(src + base * G) + 16 * e);
    }
    cp_async_commit();
  };
  for (int c = 0; c < kEinStages - 1; c++) issue(c);
  const int t = threadIdx.x;
  const int lane = t / G, kin = t - lane * G;  // chain (kin, lane) in warp 0
  const bool chain = t < G * LANES;
  T acc = T(0);
  const int64_t nfull = rows / BLK * BLK;  // rows in full 4-vector blocks
  for (int64_t c = 0; c < nchunks; c++) {
    issue(c + kEinStages - 1);
    cp_async_wait<kEinStages - 1>();
    __syncthreads();
    if (chain) {
      const T *s = ring + (c % kEinStages) * kEinRows * G;
      const int64_t base = c * kEinRows;
      const int64_t end = base + kEinRows < rows ? base + kEinRows : rows;
      const int64_t fend = end < nfull ? end : nfull;
      for (int64_t v0 = base; v0 < fend; v0 += BLK) {
        const T *blk = s + (v0 - base) * G;
#pragma unroll
        for (int j = 3; j >= 0; j--) acc = addT(blk[(j * LANES + lane) * G + kin], acc);
      }
      for (int64_t v0 = fend > base ? fend : base; v0 < end; v0 += LANES) {  // tail
        const int64_t v = v0 + lane;
        acc = addT(v < end ? s[(v - base) * G + kin] : T(0), acc);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if (t < 32) {  // all of warp 0 (the chains, plus idle lanes for fp64)
    // lanes of column kin sit in threads kin, kin + G, kin + 2G, ...
    const unsigned full = 0xffffffffu;
    T a1 = __shfl_down_sync(full, acc, G), a2 = T(0), a3 = T(0);
    if (LANES == 4) {
      a2 = __shfl_down_sync(full, acc, 2 * G);
      a3 = __shfl_down_sync(full, acc, 3 * G);
    }
    if (chain && lane == 0 && grp * G + kin < K) {
      const T r = LANES == 4 ? addT(addT(acc, a1), addT(a2, a3)) : addT(acc, a1);
      tot[(int64_t)b * K + grp * G + kin] = r;
    }
  }
}

// out[k] = sum over slots b, in b order, of the per-slot chain results
template <class T>
__global__ void theta2_finish_kernel(const T *__restrict__ tot, int B, int K, double *out) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    T s = T(0);
    for (int b = 0; b < B; b++) s = addT(s, tot[(int64_t)b * K + k]);
    out[k] = (double)s;
  }
}

template <class T>
__global__ void reduce_partials_kernel(const T *__restrict__ partials, int nparts, int len,
                                       double *__restrict__ out) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < len; o += gridDim.x * blockDim.x) {
    // same sequential order; 16 loads in flight ahead of the dependent adds
    // (one L2 trip per part made a B = 32 reduce 32 us)
    double s = 0.0;
    int p = 0;
    for (; p + 16 <= nparts; p += 16) {
      T v[16];
#pragma unroll
      for (int q = 0; q < 16; q++) v[q] = partials[(int64_t)(p + q) * len + o];
#pragma unroll
      for (int q = 0; q < 16; q++) s += (double)v[q];
    }
    for (; p < nparts; p++) s += (double)partials[(int64_t)p * len + o];
    out[o] = s;
  }
}

// Q head at the action node of each slot (owner rank only).  head_out[b] =
// [dtheta5 (K*K), dtheta6 (K*K), dtheta7 (2K), sq_err] in fp64.
template <class T>
__global__ void head_backward_kernel(s2v_shard sh, int K, const T *__restrict__ h_L,
                                     const T *__restrict__ g, const int64_t *__restrict__ actions,
                                     const T *__restrict__ targets, const T *__restrict__ t5,
                                     const T *__restrict__ t6, const T *__restrict__ t7,
                                     double *__restrict__ head_out, T *__restrict__ dg,
                                     T *__restrict__ dact) {
  extern __shared__ unsigned char smem_raw[];
  T *hv = reinterpret_cast<T *>(smem_raw);  // [K]
  T *gb = hv + K;                           // [K]
  T *pre = gb + K;                          // [2K]
  T *dpre = pre + 2 * K;                    // [2K]
  __shared__ T s_delta;
  __shared__ int s_owned;
  const int b = blockIdx.x;
  const int LEN = 2 * K * K + 2 * K + 1;
  double *out = head_out + (int64_t)b * LEN;
  const int64_t a = actions[b];
  if (threadIdx.x == 0) s_owned = (a >= sh.row_start && a < sh.row_start + sh.num_rows);
  __syncthreads();
  if (!s_owned) {
    for (int o = threadIdx.x; o < LEN; o += blockDim.x) out[o] = 0.0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      dg[(int64_t)b * K + k] = T(0);
      dact[(int64_t)b * K + k] = T(0);
    }
    return;
  }
  const int64_t phys = ((int64_t)b * sh.world + sh.rank) * sh.rows_max + (a - sh.row_start);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    hv[k] = h_L[phys * K + k];
    gb[k] = g[(int64_t)b * K + k];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * K; k += blockDim.x) {
    T acc = T(0);
    if (k < K)
      for (int p = 0; p < K; p++) acc = fmaT(t5[k * K + p], gb[p], acc);
    else
      for (int p = 0; p < K; p++) acc = fmaT(t6[(k - K) * K + p], hv[p], acc);
    pre[k] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    T q = T(0);
    for (int j = 0; j < 2 * K; j++) q = addT(q, mulT(relu(pre[j]), t7[j]));
    T err = q - targets[b];
    out[LEN - 1] = (double)err * (double)err;
    s_delta = (T(2) * err) / T(sh.batch);
  }
  __syncthreads();
  const T delta = s_delta;
  for (int j = threadIdx.x; j < 2 * K; j += blockDim.x) {
    dpre[j] = pre[j] > T(0) ? mulT(delta, t7[j]) : T(0);
    out[2 * K * K + j] = (double)mulT(delta, relu(pre[j]));
  }
  __syncthreads();
  for (int o = threadIdx.x; o < 2 * K * K; o += blockDim.x) {
    if (o < K * K) {
      const int k = o / K, p = o - k * K;
      out[o] = (double)mulT(dpre[k], gb[p]);
    } else {
      const int q = o - K * K, k = q / K, p = q - k * K;
      out[o] = (double)mulT(dpre[K + k], hv[p]);
    }
  }
  for (int p = threadIdx.x; p < K; p += blockDim.x) {
    T a5 = T(0), a6 = T(0);
    for (int k = 0; k < K; k++) {
      a5 = fmaT(t5[k * K + p], dpre[k], a5);
      a6 = fmaT(t6[k * K + p], dpre[K + k], a6);
    }
    dg[(int64_t)b * K + p] = a5;
    dact[(int64_t)b * K + p] = a6;
  }
}

// Adam (policy.py:339-359) with numpy's NEP-50 rounding: every Python scalar
// is cast to the array dtype, every op rounded separately.
template <class T>
__global__ void adam_kernel(T *__restrict__ p, const T *__restrict__ g, T *__restrict__ m,
                            T *__restrict__ v, int64_t n, T b1, T omb1, T b2, T omb2, T eps,
                            T lr, T b1c, T b2c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T gi = g[i];
    const T mi = addT(mulT(b1, m[i]), mulT(omb1, gi));
    const T vi = addT(mulT(b2, v[i]), mulT(mulT(omb2, gi), gi));
    m[i] = mi;
    v[i] = vi;
    const T mh = mi / b1c;
    const T vh = vi / b2c;
    const T upd = mulT(lr, mh) / addT(sqrt(vh), eps);
    p[i] = p[i] - upd;
  }
}

// Device-resident tau loop (train_step): gradients straight from the fp64
// pack of s2v_reduce_partials, rounded to T as the host's astype would, and
// adam_step's all-or-nothing non-finite rejection (policy.py:346-349):
// iteration `it` is skipped, with every later one, once any gradient of it
// or of an earlier iteration is non-finite (bad[0..it]).
template <class T>
__global__ void grad_check_kernel(const double *__restrict__ pack, int64_t n, int32_t *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite((double)(T)pack[i])) *bad = 1;
}

template <class T>
__global__ void adam_pack_kernel(T *__restrict__ p, const double *__restrict__ pack,
                                 T *__restrict__ m, T *__restrict__ v, int64_t n, T b1, T omb1,
                                 T b2, T omb2, T eps, T lr, T b1c, T b2c,
                                 const int32_t *__restrict__ bad, int it) {
  for (int j = 0; j <= it; j++)
    if (bad[j]) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T gi = (T)pack[i];
    const T mi = addT(mulT(b1, m[i]), mulT(omb1, gi));
    const T vi = addT(mulT(b2, v[i]), mulT(mulT(omb2, gi), gi));
    m[i] = mi;
    v[i] = vi;
    const T mh = mi / b1c;
    const T vh = vi / b2c;
    const T upd = mulT(lr, mh) / addT(sqrt(vh), eps);
    p[i] = p[i] - upd;
  }
}

// ---------------------------------------------------------------------------
// K = 64 fp32 fast paths (tiles of 64 rows, 4x4 register tiles).
// ---------------------------------------------------------------------------
constexpr int kT64 = 64;

__device__ __forceinline__ float4 f4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ void st4(float *p, const float4 &v) {
  *reinterpret_cast<float4 *>(p) = v;
}

// dz = grad_h * (h_l > 0); dzsum (+)= dz; P4 (+)= dz^T m; dm = dz theta4
// (dm[row][j] = sum_k theta4[k][j] dz[row][k]).  Dynamic smem: 3 x [64][68].
__global__ void __launch_bounds__(256, 2) layer_backward64_kernel(
    s2v_shard sh, const float *__restrict__ theta4, const float *__restrict__ grad_h,
    const float *__restrict__ h_l, const float *__restrict__ m_l, float *__restrict__ dzsum,
    float *__restrict__ partial, int first, float *__restrict__ dm_out) {
  extern __shared__ __align__(16) float smem_f[];
  float(*th4)[68] = reinterpret_cast<float(*)[68]>(smem_f);
  float(*dzs)[68] = reinterpret_cast<float(*)[68]>(smem_f + 64 * 68);
  float(*ms)[68] = reinterpret_cast<float(*)[68]>(smem_f + 2 * 64 * 68);
  // dz transposed, dzT[k][row] with 4-row groups XOR-swizzled by (k>>2)&7:
  // the dm product reads 4 rows of one k as one float4
  float *dzT = smem_f + 3 * 64 * 68;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < 64 * 64; idx += 256) th4[idx / 64][idx % 64] = theta4[idx];
  const int lo = tid & 15, hi = tid >> 4;
  float p4[4][4];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int c = 0; c < 4; c++)
      p4[a][c] = first ? 0.f : partial[(int64_t)blockIdx.x * 4096 + (4 * lo + a) * 64 + 4 * hi + c];
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t ntiles = (nrows + kT64 - 1) / kT64;
  // register double buffer: the next tile's grad_h / h_l / dzsum / m_l
  // loads are issued right after the current tile is staged in shared
  // memory, so they fly during its dzT m and dz theta4 products
  float4 G[kT64 / 16], H[kT64 / 16], O[kT64 / 16], M[kT64 / 16];
  auto load_tile = [&](int64_t t) {
#pragma unroll
    for (int q = 0; q < kT64 / 16; q++) {  // every load in flight before any use
      const int e = tid + q * 256, row = e >> 4, c4 = e & 15;
      const int64_t r = t * kT64 + row;
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      G[q] = H[q] = O[q] = M[q] = z4;
      if (t < ntiles && r < nrows) {
        G[q] = f4(grad_h + r * 64 + 4 * c4);
        H[q] = f4(h_l + phys_of_row(sh, r) * 64 + 4 * c4);
        if (!first) O[q] = f4(dzsum + r * 64 + 4 * c4);
        if (m_l) M[q] = f4(m_l + r * 64 + 4 * c4);
      }
    }
  };
  load_tile(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kT64;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kT64 / 16; q++) {
      const int e = tid + q * 256, row = e >> 4, c4 = e & 15;
      const int64_t r = r0 + row;
      float4 dz;
      dz.x = H[q].x > 0.f ? G[q].x : 0.f;
      dz.y = H[q].y > 0.f ? G[q].y : 0.f;
      dz.z = H[q].z > 0.f ? G[q].z : 0.f;
      dz.w = H[q].w > 0.f ? G[q].w : 0.f;
      if (r < nrows)
        st4(dzsum + r * 64 + 4 * c4, make_float4(O[q].x + dz.x, O[q].y + dz.y, O[q].z + dz.z,
                                                 O[q].w + dz.w));
      st4(&dzs[row][4 * c4], dz);
      st4(&ms[row][4 * c4], M[q]);
      if (dm_out) {
        const int rsw = row ^ ((c4 & 7) << 2);
        dzT[(4 * c4 + 0) * 64 + rsw] = dz.x;
        dzT[(4 * c4 + 1) * 64 + rsw] = dz.y;
        dzT[(4 * c4 + 2) * 64 + rsw] = dz.z;
        dzT[(4 * c4 + 3) * 64 + rsw] = dz.w;
      }
    }
    load_tile(tile + gridDim.x);
    __syncthreads();
    if (m_l) {
#pragma unroll 4
      for (int row = 0; row < kT64; row++) {
        const float4 d = f4(&dzs[row][4 * lo]);
        const float4 m = f4(&ms[row][4 * hi]);
        const float dv[4] = {d.x, d.y, d.z, d.w}, mvv[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int c = 0; c < 4; c++) p4[a][c] = __fmaf_rn(dv[a], mvv[c], p4[a][c]);
      }
    }
    if (dm_out) {
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[a][c] = 0.f;
#pragma unroll 4
      for (int k = 0; k < 64; k++) {
        const float4 t = f4(&th4[k][4 * lo]);
        const float4 d4 = f4(&dzT[k * 64 + ((4 * hi) ^ (((k >> 2) & 7) << 2))]);
        const float dv4[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const float d = dv4[a];
          acc[a][0] = __fmaf_rn(t.x, d, acc[a][0]);
          acc[a][1] = __fmaf_rn(t.y, d, acc[a][1]);
          acc[a][2] = __fmaf_rn(t.z, d, acc[a][2]);
          acc[a][3] = __fmaf_rn(t.w, d, acc[a][3]);
        }
      }
#pragma unroll
      for (int a = 0; a < 4; a++) {
        const int64_t r = r0 + 4 * hi + a;
        if (r < nrows)
          st4(dm_out + phys_of_row(sh, r) * 64 + 4 * lo,
              make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]));
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int c = 0; c < 4; c++)
      partial[(int64_t)blockIdx.x * 4096 + (4 * lo + a) * 64 + 4 * hi + c] = p4[a][c];
}

// Layer backward on the 5th-generation tensor cores (default K = 64 fp32
// path; S2V_BWD_TC=0 selects the FFMA kernel above).
//
// Both contractions of a tile are GEMM-shaped and carry the 1e-4 gradient
// bar, not bitwise, so they run as tcgen05.mma kind::tf32
// on split operands: x = hi + lo with hi = x with the low 13 mantissa bits
// cleared and lo = x - hi (exact), every hi/lo cross term formed -- fp32-
// class products.  The splits are stacked along M and N so every MMA is
// M = 128:
//   dm^T [j'][row'] = sum_k thT [j'][k] dzS [row'][k]       (policy.py:300-303)
//       A = thT: theta4^T hi (j' < 64) | lo (j' >= 64)        M = 128, K = 64,
//       resident in TMEM for the whole kernel (tcgen05.mma with A from
//       TMEM: no shared-memory operand traffic for it, 1.50 -> 1.44 ms)
//       B = dzS: dz hi (row' < 32) | lo (row' >= 32)          N = 64
//       dm[row][j] = sum of the 4 quadrants (j | j+64) x (row | row+32)
//   dtheta4 [k'][j'] += sum_row dzT [k'][row] mT [j'][row]  (policy.py:296-297)
//       A = dz^T hi | lo (M = 128), B = m^T hi | lo (N = 128), K = rows
// The tensor cores' fp32 accumulation truncates when the accumulator
// dwarfs the products, so dtheta4 is accumulated in TMEM for kDrain tiles
// only and then drained into an IEEE fp32 accumulator in shared memory
// (double-buffered TMEM: the MMAs of the next group run meanwhile); over a
// whole CTA (13.5K rows at BA(2M,16)) TMEM-only accumulation measured
// 1.7e-4 off the reference's dtheta4, the drained one matches the FFMA path.
// tcgen05 tf32 operands must be K-major (the MN-major encodings read back
// zeros on B200, probed), so the staging warps write dz twice (rows x k and
// k x rows core matrices).  Core matrix = 8 M/N-rows x 16 bytes of K; the
// strides between core matrices are padded (dzS: K-chunk 65 x 16 B; dzT /
// mT: 8-row group 9 x 16 B) so a warp's staging stores hit 32 distinct banks.
//
// Warp roles (640 threads = 5 warps per SM sub-partition at 96 registers,
// 1 CTA per SM, 32-row tiles, tile = blockIdx.x + i * gridDim.x, kStages
// operand stages):
//   warps 4-19 (staging): global loads of grad_h / h_l / dzsum / m_l three
//     tiles ahead in registers (warp = 4 rows x 128 contiguous bytes);
//     dz = grad_h * (h_l > 0); dzsum += dz to HBM; dzS / dzT / mT hi|lo into
//     operand stage i % kStages; arrive opfull[s]
//   warp 4, lane 0 (MMA issue, after its staging of the tile): 8 + 4 MMAs
//     per tile once all staging warps arrived; commits opfree[s] (stage
//     reusable), d1full[b] (dm accumulator complete) and, every kDrain
//     tiles, d2full[g] (dtheta4 group accumulator complete)
//   warps 0-3 (epilogue, TMEM lanes 32 w + [0, 32)): dm^T via tcgen05.ld,
//     quadrant sums through shared memory, coalesced dm stores; dtheta4
//     group drains; finally the dtheta4 partial of the CTA.
// ---------------------------------------------------------------------------
constexpr int kTR = 32;                       // rows per tile
constexpr int kTcThreads = 640;               // 20 warps: 5 per SM sub-partition
constexpr int kStages = 2;                    // operand stages (and register prefetch depth):
                                              // 2 leaves ~120 KB of the SM's 256 KB to L1,
                                              // 3 (194 KB shared) measured 1.29 vs 1.10 ms
constexpr int kDrain = 8;                     // tiles per TMEM dtheta4 group
constexpr uint32_t kLboS = 65 * 16;           // dzS K-chunk stride
constexpr uint32_t kSboT = 9 * 16;            // dzT / mT 8-row (M/N) group stride
constexpr uint32_t kLboT = 16 * kSboT;        // dzT / mT K-chunk (4 rows) stride
constexpr uint32_t kZsBytes = 16640;          // 15 kLboS + 8 x 128, rounded to 128
constexpr uint32_t kZtBytes = 8 * kLboT;      // 18432
constexpr uint32_t kStageBytes = kZsBytes + 2 * kZtBytes;
constexpr uint32_t kEpiBytes = 32 * 132 * 4;  // dm^T row sums [32 rows][132]
constexpr uint32_t kAccBytes = 64 * 65 * 4;   // dtheta4 fp32 accumulator [64 k][65]
constexpr size_t kTcSmem = 128 + kStages * kStageBytes + kEpiBytes + kAccBytes;

__device__ __forceinline__ float tf32_hi(float v) {
  return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
}

// SWIZZLE_NONE K-major shared-memory matrix descriptor (sm_100 version 1):
// start, leading (K-chunk) and stride (8-row group) byte offsets
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// A operand from TMEM (columns = K elements of each lane's row), B from smem
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}

// 32 consecutive fp32 TMEM columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1) layer_backward64_tc_kernel(
    s2v_shard sh, const float *__restrict__ theta4, const float *__restrict__ grad_h,
    const float *__restrict__ h_l, const float *__restrict__ m_l, float *__restrict__ dzsum,
    float *__restrict__ partial, int first, float *__restrict__ dm_out) {
  extern __shared__ uint8_t tc_raw[];
  // 128-byte aligned base, derived by pointer arithmetic on the shared array
  // (not an integer cast) so every access below compiles to STS / LDS
  uint8_t *base = tc_raw + ((128u - ((uint32_t)__cvta_generic_to_shared(tc_raw) & 127u)) & 127u);
  auto stage_ptr = [&](int s) { return base + (uint32_t)s * kStageBytes; };
  float *epi = reinterpret_cast<float *>(base + kStages * kStageBytes);  // [32][132]
  float *acc = epi + kEpiBytes / 4;                                           // [64][65]
  __shared__ __align__(8) uint64_t bars[2 * kStages + 8];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool want_dm = dm_out != nullptr, want_p4 = m_l != nullptr;
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
  auto opfull = [&](int s) { return bar0 + 8 * s; };
  auto opfree = [&](int s) { return bar0 + 8 * (kStages + s); };
  auto d1full = [&](int b) { return bar0 + 8 * (2 * kStages + b); };
  auto d1free = [&](int b) { return bar0 + 8 * (2 * kStages + 2 + b); };
  auto d2full = [&](int b) { return bar0 + 8 * (2 * kStages + 4 + b); };
  auto d2free = [&](int b) { return bar0 + 8 * (2 * kStages + 6 + b); };
  for (int idx = tid; idx < 64 * 65; idx += kTcThreads) acc[idx] = 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(opfull(s), 512);
      mbar_init(opfree(s), 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(d1full(b), 1);
      mbar_init(d1free(b), 128);
      mbar_init(d2full(b), 1);
      mbar_init(d2free(b), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;  // D1: cols [64 b, +64); D2: cols 128 + [128 g, +128)
  // A of dm^T resident in TMEM (cols [384, 448)): lane j' holds thT[j'][0..63]
  if (warp < 4) {
    const int jp = 32 * warp + lane;
#pragma unroll
    for (int c = 0; c < 4; c++) {
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; q++) {
        const float x = theta4[(16 * c + q) * 64 + (jp & 63)], hx = tf32_hi(x);
        v[q] = jp < 64 ? hx : x - hx;
      }
      tmem_st16(tmem + ((uint32_t)(32 * warp) << 16) + 384 + 16 * c, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t ntiles = (nrows + kTR - 1) / kTR;
  const int n_my = blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto tile_row0 = [&](int i) { return (blockIdx.x + (int64_t)i * gridDim.x) * kTR; };

  if (warp >= 4) {
    // ---------------- staging: warp -> rows 4 (w / 2) + [0, 4), float4 columns
    // 8 (w % 2) + [0, 8); lane -> row + (lane / 8), float4 c4 = ... + lane % 8
    const int w = warp - 4;
    const int row = 4 * (w >> 1) + (lane >> 3), c4 = 8 * (w & 1) + (lane & 7);
    const int kc = 4 * c4;  // first k (or j) of the float4
    const uint32_t idesc1 = (1u << 4) | (2u << 7) | (2u << 10) | (8u << 17) | (8u << 24);
    const uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | (16u << 17) | (8u << 24);
    float4 G[kStages], H[kStages], O[kStages], M[kStages];
    auto load = [&](int i, float4 &g, float4 &hv, float4 &o, float4 &mv) {
      const int64_t r = tile_row0(i) + row;
      g = hv = o = mv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < n_my && r < nrows) {
        g = f4(grad_h + r * 64 + kc);
        hv = f4(h_l + phys_of_row(sh, r) * 64 + kc);
        if (!first) o = f4(dzsum + r * 64 + kc);
        if (want_p4) mv = f4(m_l + r * 64 + kc);
      }
    };
#pragma unroll
    for (int u = 0; u < kStages; u++) load(u, G[u], H[u], O[u], M[u]);
    // core-matrix offsets (floats) of this thread's elements
    const uint32_t o_zs = (uint32_t)c4 * (kLboS / 4) + (row >> 3) * 32 + (row & 7) * 4;
    const uint32_t o_zt = (row >> 2) * (kLboT / 4) + (row & 3);
#pragma unroll 1
    for (int i0 = 0; i0 < n_my; i0 += kStages) {
#pragma unroll
      for (int u = 0; u < kStages; u++) {
        const int i = i0 + u;
        if (i >= n_my) break;
        const int s = u;  // = i % kStages (i0 is a multiple of kStages)
        const int64_t r = tile_row0(i) + row;
        const float4 g = G[u], hv = H[u], o = O[u], mv = M[u];
        float dz[4] = {hv.x > 0.f ? g.x : 0.f, hv.y > 0.f ? g.y : 0.f, hv.z > 0.f ? g.z : 0.f,
                       hv.w > 0.f ? g.w : 0.f};
        if (r < nrows)
          st4(dzsum + r * 64 + kc,
              make_float4(o.x + dz[0], o.y + dz[1], o.z + dz[2], o.w + dz[3]));
        float dh[4], dl[4], mh[4], ml[4];
        const float m4[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          dh[q] = tf32_hi(dz[q]);
          dl[q] = dz[q] - dh[q];
          mh[q] = tf32_hi(m4[q]);
          ml[q] = m4[q] - mh[q];
        }
        load(i + kStages, G[u], H[u], O[u], M[u]);  // this set is consumed: refill
        if (i >= kStages) mbar_wait(opfree(s), ((i / kStages) - 1) & 1);
        uint8_t *sp = stage_ptr(s);
        float *zs = reinterpret_cast<float *>(sp);
        float *zt = reinterpret_cast<float *>(sp + kZsBytes);
        float *mt = reinterpret_cast<float *>(sp + kZsBytes + kZtBytes);
        // dzS [row'][k]: hi at row' = row, lo at row' = row + 32 (4 groups of 8 on)
        st4(zs + o_zs, make_float4(dh[0], dh[1], dh[2], dh[3]));
        st4(zs + o_zs + 4 * 32, make_float4(dl[0], dl[1], dl[2], dl[3]));
        // dzT [k'][row] / mT [j'][row]: lo at k' + 64 (8 groups of 8 on)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int kk = kc + q;
          const uint32_t off = o_zt + (kk >> 3) * (kSboT / 4) + (kk & 7) * 4;
          zt[off] = dh[q];
          zt[off + 8 * (kSboT / 4)] = dl[q];
          if (want_p4) {
            mt[off] = mh[q];
            mt[off + 8 * (kSboT / 4)] = ml[q];
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(opfull(s));
        // one staging thread issues the tile's MMAs once every staging warp
        // has arrived (the epilogue warps never delay the MMA issue; a
        // dynamic last-arriver issue measured slower: 1.69 vs 1.50 ms)
        if (warp == 4 && lane == 0) {
          const int b = i & 1, grp = i / kDrain, gb = grp & 1;
          const bool g_first = i % kDrain == 0, g_last = i % kDrain == kDrain - 1 || i == n_my - 1;
          mbar_wait(opfull(s), (i / kStages) & 1);
          if (i >= 2 && want_dm) mbar_wait(d1free(b), ((i >> 1) - 1) & 1);
          if (want_p4 && g_first && grp >= 2) mbar_wait(d2free(gb), ((grp >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sp = (uint32_t)__cvta_generic_to_shared(stage_ptr(s));
          const uint32_t s_zs = sp, s_zt = sp + kZsBytes, s_mt = sp + kZsBytes + kZtBytes;
          if (want_dm) {
#pragma unroll
            for (int ks = 0; ks < 8; ks++)  // K = 8 of k per MMA
              mma_tf32_ts(tmem + 64 * b, tmem + 384 + 8 * ks,
                          umma_desc(s_zs + ks * 2 * kLboS, kLboS, 128), idesc1, ks ? 1u : 0u);
          }
          if (want_p4) {
#pragma unroll
            for (int ks = 0; ks < 4; ks++)  // K = 8 rows per MMA
              mma_tf32(tmem + 128 + 128 * gb, umma_desc(s_zt + ks * 2 * kLboT, kLboT, kSboT),
                       umma_desc(s_mt + ks * 2 * kLboT, kLboT, kSboT), idesc2,
                       (!g_first || ks) ? 1u : 0u);
          }
          mma_commit(opfree(s));
          mma_commit(d1full(b));
          if (want_p4 && g_last) mma_commit(d2full(gb));
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (warps 0-3: TMEM lanes 32 w + [0, 32)), one
    // tile behind the MMAs
    const int jp = 32 * warp + lane;  // j' of dm^T, k' of dtheta4
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
#pragma unroll 1
    for (int i = 0; i < n_my; i++) {
      const int b = i & 1, grp = i / kDrain, gb = grp & 1;
      const bool g_last = i % kDrain == kDrain - 1 || i == n_my - 1;
      mbar_wait(d1full(b), (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (want_dm) {
        {
          float hi[32], lo[32];
          tmem_ld32(tmem + lane_base + 64 * b, hi);       // row' = row (dz hi)
          tmem_ld32(tmem + lane_base + 64 * b + 32, lo);  // row' = row + 32 (dz lo)
          asm volatile("tcgen05.fence::before_thread_sync;");
          mbar_arrive(d1free(b));
          named_sync(1, 128);  // the previous tile's epi reads are done
#pragma unroll
          for (int rr = 0; rr < 32; rr++) epi[rr * 132 + jp] = hi[rr] + lo[rr];
        }
        named_sync(1, 128);
        // dm[row][j] = epi[row][j] + epi[row][j + 64]: thread -> row tid / 4,
        // columns 16 (tid % 4) + [0, 16)
        const int rr = tid >> 2, j0 = 16 * (tid & 3);
        const int64_t r = tile_row0(i) + rr;
        if (r < nrows) {
          float *dst = dm_out + phys_of_row(sh, r) * 64 + j0;
          const float *e = epi + rr * 132 + j0;
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 a = f4(e + 4 * q), c = f4(e + 64 + 4 * q);
            st4(dst + 4 * q, make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w));
          }
        }
      }
      if (want_p4 && g_last) {  // drain the group's dtheta4 into the fp32 accumulator
        mbar_wait(d2full(gb), (grp >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        // u[k'][j] = D2[k'][j] + D2[k'][j + 64]; acc[k][j] += u[k][j], then
        // += u[k + 64][j]: warps 0-1 (k' < 64) first, warps 2-3 after a
        // barrier -- a fixed order, so partials are bit-reproducible
#pragma unroll 1
        for (int ph = 0; ph < 2; ph++) {
          if ((warp >> 1) == ph) {
#pragma unroll 1
            for (int h = 0; h < 2; h++) {
              float a[32], c[32];
              tmem_ld32(tmem + lane_base + 128 + 128 * gb + 32 * h, a);
              tmem_ld32(tmem + lane_base + 128 + 128 * gb + 64 + 32 * h, c);
#pragma unroll
              for (int q = 0; q < 32; q++) acc[(jp & 63) * 65 + 32 * h + q] += a[q] + c[q];
            }
          }
          named_sync(2, 128);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(d2free(gb));
      }
    }
  }
  // ---------------- dtheta4 partial of this CTA: acc[k][j] + acc[k + 64][j]
  __syncthreads();
  for (int idx = tid; idx < 4096; idx += kTcThreads) {
    float *dst = partial + (int64_t)blockIdx.x * 4096 + idx;
    *dst = (first ? 0.f : *dst) + acc[(idx >> 6) * 65 + (idx & 63)];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// dtheta1 [64], dtheta2 [64], dtheta3 [64][64] partials from dzsum.
// Dynamic smem: th3 [64][68], dzs [64][68], ws [64][68], red [16][64], aux.
// dtheta3 = sum_rows dz[row] w[row]^T with w[row][j] = fl(theta2[j] deg) or
// 0 -- relu(theta2[j] deg) = relu(theta2[j]) deg exactly in real arithmetic
// (deg >= 0), so dtheta3[k][j] = relu(theta2[j]) * u[k], u[k] = sum_rows
// dz[row][k] deg[row]: 64 FMA per row instead of the 4,096 of the outer
// product.  Each term differs from the reference's fl(fl(theta2 deg) dz) by
// at most one rounding of the product -- the same order of error as any
// other summation order of this sum, well inside the 1e-4 bar.

__global__ void __launch_bounds__(256, 2) param_grads64_kernel(
    s2v_shard sh, const float *__restrict__ theta2, const float *__restrict__ theta3,
    const float *__restrict__ dzsum, float *__restrict__ partial, float *__restrict__ t2c) {
  extern __shared__ __align__(16) float smem_f[];
  float(*th3)[68] = reinterpret_cast<float(*)[68]>(smem_f);
  float(*dzs)[68] = reinterpret_cast<float(*)[68]>(smem_f + 64 * 68);
  float(*ws)[68] = reinterpret_cast<float(*)[68]>(smem_f + 2 * 64 * 68);
  float(*red)[64] = reinterpret_cast<float(*)[64]>(smem_f + 3 * 64 * 68);
  float *s_sol = smem_f + 3 * 64 * 68 + 16 * 64;
  float *s_deg = s_sol + 64;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < 64 * 64; idx += 256) th3[idx / 64][idx % 64] = theta3[idx];
  const int lo = tid & 15, hi = tid >> 4;
  float p2[4], p1 = 0.f, pu = 0.f;
#pragma unroll
  for (int a = 0; a < 4; a++) p2[a] = 0.f;
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t ntiles = (nrows + kT64 - 1) / kT64;
  // register double buffer: the next tile's dz sums and (S bit, degree) are
  // loaded while the current tile's products run
  float4 D[kT64 * 16 / 256];
  uint8_t nsol = 0;
  int32_t ndeg = 0;
  auto load_tile = [&](int64_t t) {
#pragma unroll
    for (int q = 0; q < kT64 * 16 / 256; q++) {
      const int e = tid + q * 256, row = e >> 4, c4 = e & 15;
      const int64_t r = t * kT64 + row;
      D[q] = (t < ntiles && r < nrows) ? f4(dzsum + r * 64 + 4 * c4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid < kT64) {
      const int64_t r = t * kT64 + tid;
      const bool ok = t < ntiles && r < nrows;
      nsol = ok ? sh.sol[r] : 0;
      ndeg = ok ? sh.rdeg[r] : 0;
    }
  };
  load_tile(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    if (tid < kT64) {
      s_sol[tid] = nsol ? 1.f : 0.f;
      s_deg[tid] = nsol ? 0.f : (float)ndeg;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kT64 * 16 / 256; q++) {
      const int e = tid + q * 256;
      const int row = e >> 4, c4 = e & 15;
      const float4 d = D[q];
      st4(&dzs[row][4 * c4], d);
      const float deg = s_deg[row];
      float4 w;
      w.x = relu(theta2[4 * c4 + 0] * deg);
      w.y = relu(theta2[4 * c4 + 1] * deg);
      w.z = relu(theta2[4 * c4 + 2] * deg);
      w.w = relu(theta2[4 * c4 + 3] * deg);
      st4(&ws[row][4 * c4], w);
    }
    __syncthreads();
    load_tile(tile + gridDim.x);
    // dtheta2[j] += deg (w_j > 0) (theta3^T dz)_j   rows 4hi+a, j = 4lo+c
    {
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[a][c] = 0.f;
      // dz rows read as float4 along k (4 k per load: 8 shared loads per 64
      // FMA instead of 5 per 16); each output stays the chain k = 0..63
#pragma unroll 2
      for (int k0 = 0; k0 < 64; k0 += 4) {
        float dv[4][4];
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const float4 d4 = f4(&dzs[4 * hi + a][k0]);
          dv[a][0] = d4.x;
          dv[a][1] = d4.y;
          dv[a][2] = d4.z;
          dv[a][3] = d4.w;
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const float4 t = f4(&th3[k0 + i][4 * lo]);
#pragma unroll
          for (int a = 0; a < 4; a++) {
            acc[a][0] = __fmaf_rn(t.x, dv[a][i], acc[a][0]);
            acc[a][1] = __fmaf_rn(t.y, dv[a][i], acc[a][1]);
            acc[a][2] = __fmaf_rn(t.z, dv[a][i], acc[a][2]);
            acc[a][3] = __fmaf_rn(t.w, dv[a][i], acc[a][3]);
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 4; a++) {
        const int row = 4 * hi + a;
        const float deg = s_deg[row];
#pragma unroll
        for (int c = 0; c < 4; c++)
          if (ws[row][4 * lo + c] > 0.f) p2[c] = __fmaf_rn(acc[a][c], deg, p2[c]);
        const int64_t r = tile * kT64 + row;
        if (t2c && r < nrows) {
          // the einsum terms fl(fl(dw_acc * (w > 0)) * deg) of policy.py:305-306
          // in the chain layout [b][k / 8][v][8] read by theta2_einsum_kernel
          const int64_t b = r / sh.num_rows, v = r - b * sh.num_rows;
          float t[4];
#pragma unroll
          for (int c = 0; c < 4; c++)
            t[c] = __fmul_rn(__fmul_rn(acc[a][c], ws[row][4 * lo + c] > 0.f ? 1.f : 0.f), deg);
          st4(t2c + ((b * 8 + (lo >> 1)) * sh.num_rows + v) * 8 + 4 * (lo & 1),
              make_float4(t[0], t[1], t[2], t[3]));
        }
      }
    }
    // dtheta1[k] += dz[row][k] sol[row]: every thread, rows g (mod 4) of
    // column k (tid = 64 g + k), four partials summed in g order at the end
    // (one warp pair walking all rows serially held the other six warps at
    // the next barrier)
#pragma unroll 4
    for (int row = tid >> 6; row < kT64; row += 4) {
      const float d = dzs[row][tid & 63];
      p1 = __fmaf_rn(d, s_sol[row], p1);
      pu = __fmaf_rn(d, s_deg[row], pu);  // u[k] of dtheta3 (above)
    }
  }
  __syncthreads();
  // reduce p2 over the 16 row groups (hi), then write the partial row
#pragma unroll
  for (int c = 0; c < 4; c++) red[hi][4 * lo + c] = p2[c];
  __syncthreads();
  float *out = partial + (int64_t)blockIdx.x * (2 * 64 + 4096);
  float s2 = 0.f;
  if (tid < 64)
    for (int q = 0; q < 16; q++) s2 += red[q][tid];
  __syncthreads();
  red[tid >> 6][tid & 63] = p1;
  red[4 + (tid >> 6)][tid & 63] = pu;
  __syncthreads();
  if (tid < 64) {
    out[tid] = ((red[0][tid] + red[1][tid]) + red[2][tid]) + red[3][tid];
    out[64 + tid] = s2;
    red[8][tid] = ((red[4][tid] + red[5][tid]) + red[6][tid]) + red[7][tid];
  }
  __syncthreads();
  for (int idx = tid; idx < 4096; idx += 256)  // dtheta3 partial [k][j]
    out[128 + idx] = __fmul_rn(red[8][idx >> 6], relu(theta2[idx & 63]));
}

// spmm_t for K = 64 fp32: half-warp per row in descending-degree order.
__global__ void __launch_bounds__(256) gather64_kernel(s2v_shard sh,
                                                       const float *__restrict__ src,
                                                       float *__restrict__ out,
                                                       uint32_t hot_rows) {
  const int tid = threadIdx.x, sub = tid & 15;
  const unsigned hmask = (tid & 16) ? 0xFFFF0000u : 0x0000FFFFu;
  const int hbase = tid & 16;
  const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t nhw = ((int64_t)gridDim.x * blockDim.x) >> 4;
  const int64_t first = sh.order ? sh.n_hub : 0;  // hub rows: hub_gather64_kernel
  // two-deep software pipeline over this half-warp's rows q, q+nhw, ...:
  // the row id two rows ahead and the range / S bit of the next row are
  // loaded before the current row's gather, so they arrive during it
  auto row_of = [&](int64_t qq) -> int64_t {
    return qq < nrows ? (sh.order ? (int64_t)sh.order[qq] : qq) : -1;
  };
  int64_t q = first + (((int64_t)blockIdx.x * blockDim.x + tid) >> 4);
  int64_t rA = row_of(q), rB = row_of(q + nhw);
  int64_t a0 = 0, a1 = 0;
  if (rA >= 0 && !sh.sol[rA]) {
    a0 = sh.row_ptr[rA];
    a1 = sh.row_ptr[rA + 1];
  }
  for (; q < nrows; q += nhw) {
    const int64_t rC = row_of(q + 2 * nhw);
    int64_t b0 = 0, b1 = 0;
    if (rB >= 0 && !sh.sol[rB]) {
      b0 = sh.row_ptr[rB];
      b1 = sh.row_ptr[rB + 1];
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a1 > a0)
      acc = gather_row64(a0, a1, sh.cols, src, sub, hmask, hbase, hot_rows, pol_hot, pol_cold,
                         nullptr, nullptr,
                         (uint32_t)((rA / sh.num_rows) * sh.world * sh.rows_max));
    st4(out + rA * 64 + 4 * sub, acc);
    rA = rB;
    rB = rC;
    a0 = b0;
    a1 = b1;
  }
}

// spmm_t, tiled like round64_kernel: 32-row tiles in descending-degree
// order from an atomic counter, the next tile's index and row ids fetched
// during the current tile's gathers (cp.async), two rows per half-warp.
constexpr int kGTile = 32;

__global__ void __launch_bounds__(256, 4) gather64_tiles_kernel(s2v_shard sh,
                                                                const float *__restrict__ src,
                                                                float *__restrict__ out,
                                                                uint32_t hot_rows,
                                                                int *__restrict__ tile_counter,
                                                                int sparse_max, int pf) {
  __shared__ int32_t s_raw[2][kGTile];
  __shared__ int64_t s_e0[kGTile], s_e1[kGTile];
  __shared__ int32_t s_rows[kGTile];
  __shared__ int s_tiles[2];
  const int tid = threadIdx.x, hw = tid >> 4, sub = tid & 15;
  const unsigned hmask = (tid & 16) ? 0xFFFF0000u : 0x0000FFFFu;
  const int hbase = tid & 16;
  const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const int64_t first = sh.order ? sh.n_hub : 0;  // hub rows: hub_gather64_kernel
  const int64_t ntiles = (nrows - first + kGTile - 1) / kGTile;
  auto prefetch_rows = [&](int64_t t, int buf) {
    const int64_t q = first + t * kGTile + tid;
    if (t < ntiles && q < nrows && sh.order)
      cp_async4(&s_raw[buf][tid], sh.order + q);
    else
      s_raw[buf][tid] = (t < ntiles && q < nrows) ? (int32_t)q : -1;
  };
  if (tid == 0) s_tiles[0] = atomicAdd(tile_counter, 1);
  __syncthreads();
  if (tid < kGTile) prefetch_rows(s_tiles[0], 0);
  int cur = 0;
  for (;;) {
    cp_async_wait_all();
    __syncthreads();
    const int64_t tile = s_tiles[cur];
    if (tile >= ntiles) break;
    if (tid == 0) s_tiles[cur ^ 1] = atomicAdd(tile_counter, 1);
    if (tid < kGTile) {
      const int32_t r = s_raw[cur][tid];
      s_rows[tid] = r;
      int64_t e0 = 0, e1 = 0;
      if (r >= 0 && !sh.sol[r]) {
        e0 = sh.row_ptr[r];
        e1 = sh.row_ptr[r + 1];
      }
      s_e0[tid] = e0;
      s_e1[tid] = e1;
    }
    // tiles whose rows all have <= sparse_max entries: one 8-lane group per
    // row, every row of the tile in flight at once (as round64_kernel)
    const bool sparse =
        __syncthreads_and(tid >= kGTile || s_e1[tid] - s_e0[tid] <= sparse_max);
    if (tid < kGTile) prefetch_rows(s_tiles[cur ^ 1], cur ^ 1);
    if (sparse) {
      const int lr = tid >> 3, l8 = tid & 7;
      const int64_t r = s_rows[lr];
      if (r >= 0) {
        float4 a0, a1;
        gather_row64_g8(s_e0[lr], s_e1[lr], sh.cols, src, l8, 0xFFu << (tid & 24), tid & 24,
                        hot_rows, pol_hot, pol_cold, nullptr, nullptr,
                        (uint32_t)((r / sh.num_rows) * sh.world * sh.rows_max), a0, a1, pf);
        st4(out + r * 64 + 4 * l8, a0);
        st4(out + r * 64 + 32 + 4 * l8, a1);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int lr = hw + 16 * q;
        const int64_t r = s_rows[lr];
        if (r < 0) continue;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (s_e1[lr] > s_e0[lr])
          acc = gather_row64<false, true>(
              s_e0[lr], s_e1[lr], sh.cols, src, sub, hmask, hbase, hot_rows, pol_hot, pol_cold,
              nullptr, nullptr, (uint32_t)((r / sh.num_rows) * sh.world * sh.rows_max));
        st4(out + r * 64 + 4 * sub, acc);
      }
    }
    cur ^= 1;
  }
}

// spmm_t of the hub rows: one CTA per row, cooperative gather.
__global__ void __launch_bounds__(256, 1) hub_gather64_kernel(s2v_shard sh,
                                                              const float *__restrict__ src,
                                                              float *__restrict__ out,
                                                              int *__restrict__ counter,
                                                              uint32_t hot_rows) {
  extern __shared__ __align__(16) float hub_smem[];
  __shared__ int s_q;
  const int tid = threadIdx.x, sub = tid & 15;
  const uint64_t pol_hot = l2_policy_last(), pol_cold = l2_policy_first();
  for (;;) {
    __syncthreads();
    if (tid == 0) s_q = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t q = s_q;
    if (q >= sh.n_hub) break;
    const int64_t r = sh.order[q];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!sh.sol[r])
      acc = hub_gather_row64(sh.row_ptr[r], sh.row_ptr[r + 1], sh.cols, src, hub_smem, hot_rows,
                             pol_hot, pol_cold);
    if (tid < 16) st4(out + r * 64 + sub * 4, acc);
  }
}

static int hub_gather_launch(const s2v_shard *sh, const float *src, float *out,
                             uint32_t hot_rows, cudaStream_t st, cudaStream_t *side,
                             cudaEvent_t *done) {
  static thread_local cudaStream_t hs = nullptr;
  static thread_local cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  static thread_local int *counter = nullptr;
  static thread_local int dev_of = -1;
  int dev = 0;
  S2V_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev_of != dev) {
    S2V_CUDA_CHECK(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
    S2V_CUDA_CHECK(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
    S2V_CUDA_CHECK(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
    S2V_CUDA_CHECK(cudaMalloc(&counter, sizeof(int)));
    dev_of = dev;
  }
  const size_t smem = sizeof(float) * 2 * kHubBatch * 64;
  S2V_CUDA_CHECK(cudaFuncSetAttribute(hub_gather64_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  S2V_CUDA_CHECK(cudaEventRecord(ev_ready, st));
  S2V_CUDA_CHECK(cudaStreamWaitEvent(hs, ev_ready, 0));
  S2V_CUDA_CHECK(cudaMemsetAsync(counter, 0, sizeof(int), hs));
  int grid = (int)std::min<int64_t>(sh->n_hub, kNumSMs);
  hub_gather64_kernel<<<grid, 256, smem, hs>>>(*sh, src, out, counter, hot_rows);
  S2V_LAUNCH_CHECK();
  S2V_CUDA_CHECK(cudaEventRecord(ev_done, hs));
  *side = hs;
  *done = ev_done;
  return S2V_OK;
}

template <class T>
static int layer_backward_t(const s2v_shard *sh, int K, const void *theta4, const void *grad_h,
                            const void *h_l, const void *m_l, void *dzsum, void *partial,
                            int first, void *dm_out, cudaStream_t st) {
  // tcgen05 path by default for K = 64 fp32; S2V_BWD_TC=0 selects the FFMA
  // kernel (kept as the cross-check of the tensor-core path)
  static const bool use_tc = [] {
    const char *e = getenv("S2V_BWD_TC");
    return !(e && e[0] == '0');
  }();
  if (sizeof(T) == 4 && K == 64 && use_tc) {
    S2V_CUDA_CHECK(cudaFuncSetAttribute(layer_backward64_tc_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kTcSmem));
    layer_backward64_tc_kernel<<<bwd_blocks(*sh), kTcThreads, kTcSmem, st>>>(
        *sh, (const float *)theta4, (const float *)grad_h, (const float *)h_l,
        (const float *)m_l, (float *)dzsum, (float *)partial, first, (float *)dm_out);
    S2V_LAUNCH_CHECK();
    return S2V_OK;
  }
  if (sizeof(T) == 4 && K == 64) {
    const size_t smem = sizeof(float) * (3 * 64 * 68 + 64 * 64);
    S2V_CUDA_CHECK(cudaFuncSetAttribute(layer_backward64_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    layer_backward64_kernel<<<bwd_blocks(*sh), 256, smem, st>>>(
        *sh, (const float *)theta4, (const float *)grad_h, (const float *)h_l,
        (const float *)m_l, (float *)dzsum, (float *)partial, first, (float *)dm_out);
    S2V_LAUNCH_CHECK();
    return S2V_OK;
  }
  if (K * K > 64 * kBwdThreads) return fail(S2V_EINVAL, "embed_dim %d too large for backward", K);
  size_t smem = sizeof(T) * ((size_t)K * (K + 1) + 2 * kBwdTile * (size_t)K);
  auto kern = layer_backward_kernel<T>;
  S2V_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<bwd_blocks(*sh), kBwdThreads, smem, st>>>(*sh, K, (const T *)theta4, (const T *)grad_h,
                                                   (const T *)h_l, (const T *)m_l, (T *)dzsum,
                                                   (T *)partial, first, (T *)dm_out);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // namespace s2v

using namespace s2v;

extern "C" {

int s2v_backward_blocks(const s2v_shard *sh) { return bwd_blocks(*sh); }

int s2v_grad_h_init(s2v_dtype dt, const s2v_shard *sh, int K, const void *dg,
                    const int64_t *actions, const void *dact, void *grad_h, void *stream) {
  int64_t total = (int64_t)sh->batch * sh->num_rows * K;
  if (total == 0) return S2V_OK;
  int grid = (int)std::min<int64_t>((total + 255) / 256, kNumSMs * 8);
  if (dt == S2V_F32 && K == 64) {
    const int gx = (int)std::max<int64_t>(
        1, std::min<int64_t>((sh->num_rows * 16 + 255) / 256, kNumSMs * 8 / sh->batch + 1));
    grad_h_init64_kernel<<<dim3(gx, sh->batch), 256, 0, as_stream(stream)>>>(
        *sh, (const float *)dg, actions, (const float *)dact, (float *)grad_h);
  } else if (dt == S2V_F32)
    grad_h_init_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(
        *sh, K, (const float *)dg, actions, (const float *)dact, (float *)grad_h);
  else
    grad_h_init_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
        *sh, K, (const double *)dg, actions, (const double *)dact, (double *)grad_h);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_layer_backward(s2v_dtype dt, const s2v_shard *sh, int K, const void *theta4,
                       const void *grad_h, const void *h_l, const void *m_l, void *dzsum,
                       void *partial, int first, void *dm_out, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (dt == S2V_F32)
    return layer_backward_t<float>(sh, K, theta4, grad_h, h_l, m_l, dzsum, partial, first,
                                   dm_out, st);
  return layer_backward_t<double>(sh, K, theta4, grad_h, h_l, m_l, dzsum, partial, first, dm_out,
                                  st);
}

int s2v_gather(s2v_dtype dt, const s2v_shard *sh, int K, const void *src, void *out,
               void *stream) {
  int64_t rows = (int64_t)sh->batch * sh->num_rows;
  if (rows == 0) return S2V_OK;
  if (dt == S2V_F32 && K == 64) {
    const uint32_t hot = (uint32_t)((48ull << 20) / 256);
    cudaStream_t st = as_stream(stream), side = nullptr;
    cudaEvent_t done = nullptr;
    if (sh->order && sh->n_hub > 0) {
      int rc = hub_gather_launch(sh, (const float *)src, (float *)out, hot, st, &side, &done);
      if (rc) return rc;
    }
    static const bool tiles = [] {
      const char *e = getenv("S2V_GATHER_TILES");
      return !(e && e[0] == '0');
    }();
    if (tiles) {
      static thread_local int *counter = nullptr;
      static thread_local int counter_dev = -1;
      int dev = 0;
      S2V_CUDA_CHECK(cudaGetDevice(&dev));
      if (counter_dev != dev) {
        S2V_CUDA_CHECK(cudaMalloc(&counter, sizeof(int)));
        counter_dev = dev;
      }
      S2V_CUDA_CHECK(cudaMemsetAsync(counter, 0, sizeof(int), st));
      const int64_t ntiles = (rows + kGTile - 1) / kGTile;
      static const int sparse_max = [] {
        const char *e = getenv("S2V_SPARSE_MAX");
        return e ? atoi(e) : S2V_HUB_DEGREE;
      }();
      gather64_tiles_kernel<<<(int)std::min<int64_t>(std::max<int64_t>(ntiles, 1), kNumSMs * 4),
                              256, 0, st>>>(*sh, (const float *)src, (float *)out, hot, counter,
                                            sparse_max, g8_prefetch());
    } else {
      gather64_kernel<<<kNumSMs * 8, 256, 0, st>>>(*sh, (const float *)src, (float *)out, hot);
    }
    S2V_LAUNCH_CHECK();
    if (done) S2V_CUDA_CHECK(cudaStreamWaitEvent(st, done, 0));
    return S2V_OK;
  }
  int grid = (int)std::min<int64_t>((rows * 32 + 255) / 256, kNumSMs * 16);
  if (dt == S2V_F32)
    gather_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(*sh, K, (const float *)src,
                                                              (float *)out);
  else
    gather_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(*sh, K, (const double *)src,
                                                               (double *)out);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_param_grads(s2v_dtype dt, const s2v_shard *sh, int K, const void *theta2,
                    const void *theta3, const void *dzsum, void *partials, void *t2c,
                    void *stream) {
  if (2 * K + K * K > 72 * kBwdThreads) return fail(S2V_EINVAL, "embed_dim %d too large", K);
  size_t elem = dt == S2V_F32 ? 4 : 8;
  size_t smem = elem * ((size_t)K * (K + 1) + 2 * kBwdTile * (size_t)K + 2 * kBwdTile);
  cudaStream_t st = as_stream(stream);
  if (dt == S2V_F32 && K == 64) {
    const size_t smem64 = sizeof(float) * (3 * 64 * 68 + 16 * 64 + 128);
    S2V_CUDA_CHECK(cudaFuncSetAttribute(param_grads64_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem64));
    param_grads64_kernel<<<bwd_blocks(*sh), 256, smem64, st>>>(
        *sh, (const float *)theta2, (const float *)theta3, (const float *)dzsum,
        (float *)partials, (float *)t2c);
  } else if (dt == S2V_F32) {
    auto kern = param_grads_kernel<float>;
    S2V_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<bwd_blocks(*sh), kBwdThreads, smem, st>>>(*sh, K, (const float *)theta2,
                                                     (const float *)theta3,
                                                     (const float *)dzsum, (float *)partials,
                                                     (float *)t2c);
  } else {
    auto kern = param_grads_kernel<double>;
    S2V_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<bwd_blocks(*sh), kBwdThreads, smem, st>>>(*sh, K, (const double *)theta2,
                                                     (const double *)theta3,
                                                     (const double *)dzsum, (double *)partials,
                                                     (double *)t2c);
  }
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

size_t s2v_theta2_terms_bytes(s2v_dtype dt, const s2v_shard *sh, int K) {
  const size_t elem = dt == S2V_F32 ? 4 : 8, G = 32 / elem;
  return (size_t)sh->batch * sh->num_rows * ((K + G - 1) / G) * G * elem;
}

int s2v_theta2_einsum(s2v_dtype dt, const s2v_shard *sh, int K, const void *t2c, void *tot,
                      double *out, void *stream) {
  if (K < 1) return fail(S2V_EINVAL, "embed_dim %d", K);
  cudaStream_t st = as_stream(stream);
  const size_t elem = dt == S2V_F32 ? 4 : 8, G = 32 / elem;
  const int ng = (int)((K + G - 1) / G);
  const int grid = sh->batch * ng;
  const size_t smem = (size_t)kEinStages * kEinRows * 32;
  if (dt == S2V_F32) {
    S2V_CUDA_CHECK(cudaFuncSetAttribute(theta2_einsum_kernel<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    theta2_einsum_kernel<float><<<grid, 256, smem, st>>>((const float *)t2c, sh->num_rows, K,
                                                         (float *)tot);
    S2V_LAUNCH_CHECK();
    theta2_finish_kernel<float><<<1, 128, 0, st>>>((const float *)tot, sh->batch, K, out);
  } else {
    S2V_CUDA_CHECK(cudaFuncSetAttribute(theta2_einsum_kernel<double>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    theta2_einsum_kernel<double><<<grid, 256, smem, st>>>((const double *)t2c, sh->num_rows, K,
                                                          (double *)tot);
    S2V_LAUNCH_CHECK();
    theta2_finish_kernel<double><<<1, 128, 0, st>>>((const double *)tot, sh->batch, K, out);
  }
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_reduce_partials(s2v_dtype dt, const void *partials, int nparts, int len, double *out,
                        void *stream) {
  int grid = (len + 255) / 256;
  if (dt == S2V_F32)
    reduce_partials_kernel<float><<<grid, 256, 0, as_stream(stream)>>>((const float *)partials,
                                                                       nparts, len, out);
  else
    reduce_partials_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
        (const double *)partials, nparts, len, out);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_head_backward(s2v_dtype dt, const s2v_shard *sh, int K, const void *h_L, const void *g,
                      const int64_t *actions, const void *targets, const void *theta5,
                      const void *theta6, const void *theta7, double *head_out, void *dg,
                      void *dact, void *stream) {
  size_t elem = dt == S2V_F32 ? 4 : 8;
  size_t smem = elem * 6 * (size_t)K;
  cudaStream_t st = as_stream(stream);
  if (dt == S2V_F32)
    head_backward_kernel<float><<<sh->batch, 128, smem, st>>>(
        *sh, K, (const float *)h_L, (const float *)g, actions, (const float *)targets,
        (const float *)theta5, (const float *)theta6, (const float *)theta7, head_out,
        (float *)dg, (float *)dact);
  else
    head_backward_kernel<double><<<sh->batch, 128, smem, st>>>(
        *sh, K, (const double *)h_L, (const double *)g, actions, (const double *)targets,
        (const double *)theta5, (const double *)theta6, (const double *)theta7, head_out,
        (double *)dg, (double *)dact);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_adam(s2v_dtype dt, void *params, const void *grads, void *m, void *v, int64_t n,
             double beta1, double omb1, double beta2, double omb2, double eps, double lr,
             double b1c, double b2c, void *stream) {
  if (n == 0) return S2V_OK;
  int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 4);
  if (dt == S2V_F32)
    adam_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(
        (float *)params, (const float *)grads, (float *)m, (float *)v, n, (float)beta1,
        (float)omb1, (float)beta2, (float)omb2, (float)eps, (float)lr, (float)b1c, (float)b2c);
  else
    adam_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
        (double *)params, (const double *)grads, (double *)m, (double *)v, n, beta1, omb1,
        beta2, omb2, eps, lr, b1c, b2c);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_adam_pack(s2v_dtype dt, void *params, const double *pack, void *m, void *v, int64_t n,
                  double beta1, double omb1, double beta2, double omb2, double eps, double lr,
                  double b1c, double b2c, int32_t *bad, int it, void *stream) {
  if (n == 0) return S2V_OK;
  if (it < 0) return fail(S2V_EINVAL, "bad iteration index");
  cudaStream_t st = as_stream(stream);
  int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 4);
  if (dt == S2V_F32) {
    grad_check_kernel<float><<<grid, 256, 0, st>>>(pack, n, bad + it);
    adam_pack_kernel<float><<<grid, 256, 0, st>>>(
        (float *)params, pack, (float *)m, (float *)v, n, (float)beta1, (float)omb1,
        (float)beta2, (float)omb2, (float)eps, (float)lr, (float)b1c, (float)b2c, bad, it);
  } else {
    grad_check_kernel<double><<<grid, 256, 0, st>>>(pack, n, bad + it);
    adam_pack_kernel<double><<<grid, 256, 0, st>>>((double *)params, pack, (double *)m,
                                                   (double *)v, n, beta1, omb1, beta2, omb2, eps,
                                                   lr, b1c, b2c, bad, it);
  }
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // extern "C"
