// Residual-graph state kernels: shard initialisation and group application of
// picks.  Integer-only, hence exact.
//
// Replaces (paths relative to /root/reference):
//   PartitionedState.__init__ residual mask / degrees   pkg/src/graphrl/state.py:89-111
//   PartitionedState.apply_action                       pkg/src/graphrl/state.py:173-208
//   _solve_batch group loop with mid-group skip         pkg/src/graphrl/inference.py:125-146
#include <algorithm>
#include <cstdarg>
#include <mutex>

#include "s2v_common.cuh"

namespace s2v {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

// Balanced block partition (state.py:36-53): first N % P ranks get one extra row.
struct PartitionMap {
  int64_t base, extra;
  int32_t P;
  __device__ __forceinline__ int32_t owner(int64_t u) const {
    int64_t big = extra * (base + 1);
    return u < big ? (int32_t)(u / (base + 1)) : (int32_t)(extra + (u - big) / base);
  }
  __device__ __forceinline__ int64_t start(int32_t r) const {
    return (int64_t)r * base + (r < extra ? r : extra);
  }
};

static PartitionMap make_map(const s2v_shard &sh) {
  PartitionMap m;
  m.base = sh.num_nodes / sh.world;
  m.extra = sh.num_nodes % sh.world;
  m.P = sh.world;
  return m;
}

__device__ __forceinline__ int64_t phys_of(const s2v_shard &sh, const PartitionMap &pm,
                                           int32_t b, int64_t u) {
  int32_t r = pm.owner(u);
  return ((int64_t)b * sh.world + r) * sh.rows_max + (u - pm.start(r));
}

// Entry alive iff neither endpoint is in S.  Eight lanes per local row
// (four rows per warp in flight: a BA row of ~32 entries is 4 steps, and the
// row_ptr -> cols -> sol[nbr] chain of each row overlaps three others);
// cols_src (nullable) is the read-only structure's column array, copied into
// sh.cols with the dead bits in the same pass (no separate clone).
// sol bytes -> bitmap (1 bit per physical row): the neighbour test of
// shard_init_kernel then reads a 256 KB (BA(2M,16)) array that stays in L1
__global__ void sol_bits_kernel(const uint8_t *__restrict__ sol_phys, int64_t n,
                                uint32_t *__restrict__ bits) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < (n + 31) / 32;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int j = 0; j < 32 && 32 * w + j < n; j++) v |= (sol_phys[32 * w + j] ? 1u : 0u) << j;
    bits[w] = v;
  }
}

// Rows with more than kInitLong entries (BA / R-MAT hubs: up to ~10^5) are
// not walked by one 8-lane group, 32 entries per dependent trip to HBM (a
// 9,400-entry BA(2M,16) hub alone took ~300 us, the whole kernel's time):
// shard_init_kernel appends them to a list and shard_init_long_kernel gives
// each one a CTA, 1,024 entries per trip.
constexpr int64_t kInitLong = 1024;

// Coarse S summary for shard_init_kernel's neighbour test: bit t of word j
// is set iff a node of [(32 j + t) << lg, +2^lg) is in S (lg >= 3, 32 KB for
// up to 2^(18 + lg) physical rows).  It lives in shared memory, where 32
// random lookups cost a few bank wavefronts instead of up to 32 L1 lines,
// and only a set summary bit sends the test to the exact bitmap -- the 64M
// random bitmap lookups of BA(2M,16) were the kernel's L1-bound time.
constexpr int kSumWords = 8192;

__global__ void sol_summary_kernel(const uint32_t *__restrict__ bits, int64_t n, int lg,
                                   uint32_t *__restrict__ summary) {
  const int64_t nwords = (n + 31) / 32;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < kSumWords;
       j += gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int t = 0; t < 32; t++) {
      const int64_t lo = ((int64_t)(32 * j + t)) << lg, hi = lo + ((int64_t)1 << lg);
      bool any = false;
      for (int64_t w = lo >> 5; w < nwords && (w << 5) < hi && !any; w++) {
        uint32_t m = bits[w];
        if (lg < 5) m = (m >> (lo & 31)) & ((1u << (1 << lg)) - 1u);
        any = m != 0;
      }
      v |= (any ? 1u : 0u) << t;
    }
    summary[j] = v;
  }
}

__global__ void shard_init_kernel(s2v_shard sh, const uint32_t *__restrict__ cols_src,
                                  const uint8_t *__restrict__ sol_phys,
                                  const uint32_t *__restrict__ sol_bits,
                                  int64_t *__restrict__ long_rows, int *__restrict__ long_n,
                                  const uint32_t *__restrict__ summary, int lg) {
  extern __shared__ uint32_t s_sum[];  // [kSumWords]
  for (int j = threadIdx.x; j < kSumWords / 4; j += blockDim.x)
    reinterpret_cast<uint4 *>(s_sum)[j] = reinterpret_cast<const uint4 *>(summary)[j];
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  const uint32_t *src = cols_src ? cols_src : sh.cols;
  // per-warp running count of alive entries, flushed once per slot (one
  // atomic per warp and slot instead of one per row)
  int64_t acc_b = -1;
  unsigned long long acc = 0;
  const int64_t wstride = ((gridDim.x * (int64_t)blockDim.x) >> 5) * 4;
  // the next iteration's row range and S byte are loaded one iteration
  // ahead, so each row costs one dependent trip to HBM (its columns)
  auto row_info = [&](int64_t r, int64_t &e0, int64_t &e1, uint8_t &s) {
    e0 = e1 = 0;
    s = 0;
    if (r < nrows) {
      int64_t b = 0, i = r;
      if (sh.batch > 1) {
        b = r / sh.num_rows;
        i = r - b * sh.num_rows;
      }
      s = sol_phys[(b * sh.world + sh.rank) * sh.rows_max + i];
      e0 = sh.row_ptr[r];
      e1 = sh.row_ptr[r + 1];
    }
  };
  int64_t w0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 4;
  int64_t n_e0, n_e1;
  uint8_t n_s;
  row_info(w0 + grp, n_e0, n_e1, n_s);
  for (; w0 < nrows; w0 += wstride) {  // warp-uniform loop: rows w0 + grp
    const int64_t r = w0 + grp;
    const bool ok = r < nrows;
    int64_t b = 0;
    if (ok && sh.batch > 1) b = r / sh.num_rows;
    const int64_t e0 = n_e0, e1 = n_e1;
    const uint8_t s = n_s;
    row_info(r + wstride, n_e0, n_e1, n_s);
    int cnt = 0;
    bool mine = ok;
    if (ok) {
      if (e1 - e0 > kInitLong) {  // shard_init_long_kernel's row
        mine = false;
        if (sub == 0) long_rows[atomicAdd(long_n, 1)] = r;
      }
      // four 8-entry steps per iteration: a BA row's ~32 column loads, then
      // its bitmap lookups, all in flight together
      for (int64_t e = e0 + sub; mine && e < e1; e += 32) {
        uint32_t c[4];
#pragma unroll
        for (int q = 0; q < 4; q++) c[q] = e + 8 * q < e1 ? src[e + 8 * q] & ~S2V_DEAD : 0u;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (e + 8 * q >= e1) break;
          const uint32_t cs = c[q] >> lg;
          const bool dead = s || (((s_sum[cs >> 5] >> (cs & 31)) & 1u) &&
                                  ((__ldg(sol_bits + (c[q] >> 5)) >> (c[q] & 31)) & 1u));
          sh.cols[e + 8 * q] = c[q] | (dead ? S2V_DEAD : 0u);
          cnt += !dead;
        }
      }
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (mine && sub == 0) {
      sh.rdeg[r] = cnt;
      sh.sol[r] = s;
      sh.cand[r] = (cnt > 0 && !s) ? 1 : 0;
    }
    // slot counts: the warp's rows share a slot unless a slot boundary
    // falls inside the 4 rows (then per-row atomics)
    const int64_t b0 = __shfl_sync(0xffffffffu, b, 0);
    if (__all_sync(0xffffffffu, !ok || b == b0)) {
      unsigned long long c4 = (ok && sub == 0) ? (unsigned long long)cnt : 0ull;
      c4 += __shfl_xor_sync(0xffffffffu, c4, 8);
      c4 += __shfl_xor_sync(0xffffffffu, c4, 16);
      if (lane == 0) {
        if (b0 != acc_b) {
          if (acc) atomicAdd((unsigned long long *)&sh.residual[acc_b], acc);
          acc_b = b0;
          acc = 0;
        }
        acc += c4;
      }
    } else if (ok && sub == 0 && cnt) {
      atomicAdd((unsigned long long *)&sh.residual[b], (unsigned long long)cnt);
    }
  }
  if (lane == 0 && acc) atomicAdd((unsigned long long *)&sh.residual[acc_b], acc);
}

// One CTA per listed long row: entries tid + 256 j, four per thread in
// flight, the same dead-bit rule and column copy as shard_init_kernel
__global__ void __launch_bounds__(256) shard_init_long_kernel(
    s2v_shard sh, const uint32_t *__restrict__ cols_src, const uint8_t *__restrict__ sol_phys,
    const uint32_t *__restrict__ sol_bits, const int64_t *__restrict__ long_rows,
    const int *__restrict__ long_n) {
  __shared__ int s_cnt;
  const uint32_t *src = cols_src ? cols_src : sh.cols;
  const int n = *long_n;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int64_t r = long_rows[k];
    int64_t b = 0, i = r;
    if (sh.batch > 1) {
      b = r / sh.num_rows;
      i = r - b * sh.num_rows;
    }
    const uint8_t s = sol_phys[(b * sh.world + sh.rank) * sh.rows_max + i];
    const int64_t e1 = sh.row_ptr[r + 1];
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int cnt = 0;
    for (int64_t e = sh.row_ptr[r] + threadIdx.x; e < e1; e += 4 * 256) {
      uint32_t c[4];
#pragma unroll
      for (int q = 0; q < 4; q++) c[q] = e + 256 * q < e1 ? src[e + 256 * q] & ~S2V_DEAD : 0u;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (e + 256 * q >= e1) break;
        const bool dead = s || ((__ldg(sol_bits + (c[q] >> 5)) >> (c[q] & 31)) & 1u);
        sh.cols[e + 256 * q] = c[q] | (dead ? S2V_DEAD : 0u);
        cnt += !dead;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (threadIdx.x == 0) {
      sh.rdeg[r] = s_cnt;
      sh.sol[r] = s;
      sh.cand[r] = (s_cnt > 0 && !s) ? 1 : 0;
      if (s_cnt) atomicAdd((unsigned long long *)&sh.residual[b], (unsigned long long)s_cnt);
    }
    __syncthreads();  // s_cnt is reset for the next row
  }
}

// S of every physical row after a group apply: the applied picks (global
// node ids, identical on every rank) enter S
__global__ void sol_mark_kernel(s2v_shard sh, PartitionMap pm, const int64_t *__restrict__ picks,
                                const uint8_t *__restrict__ applied, int d,
                                uint8_t *__restrict__ sol_all) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sh.batch * d) return;
  const int64_t v = picks[t];
  if (v >= 0 && v < sh.num_nodes && applied[t]) sol_all[phys_of(sh, pm, t / d, v)] = 1;
}

// Is the edge (row r, neighbour phys q) present and alive?  Row cols are
// ascending in node id, hence in physical row.
__device__ __forceinline__ bool row_has_alive(const s2v_shard &sh, int64_t r, uint32_t q) {
  int64_t lo = sh.row_ptr[r], hi = sh.row_ptr[r + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    uint32_t c = sh.cols[mid] & ~S2V_DEAD;
    if (c < q)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < sh.row_ptr[r + 1] && sh.cols[lo] == q;  // dead entries carry the bit
}

// Phase 1 (owner side): rdeg of every locally owned pick and its alive
// adjacency to the other picks of the same group.
__global__ void apply_phase1_kernel(s2v_shard sh, PartitionMap pm, const int64_t *picks, int d,
                                    int64_t *info, int validate, int32_t *err_out) {
  const int b = blockIdx.x;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    int64_t v = picks[(int64_t)b * d + j];
    int64_t *out = info + 2 * ((int64_t)b * d + j);
    out[0] = 0;
    out[1] = 0;
    if (v < 0 || v < sh.row_start || v >= sh.row_start + sh.num_rows) continue;
    int64_t r = (int64_t)b * sh.num_rows + (v - sh.row_start);
    if (validate && j == 0) {
      int code = sh.sol[r] ? 1 : (!sh.cand[r] ? 2 : 0);
      if (code) err_out[b] = code;
    }
    out[0] = sh.rdeg[r];
    uint64_t mask = 0;
    for (int i = 0; i < d && i < 64; i++) {
      int64_t w = picks[(int64_t)b * d + i];
      if (i == j || w < 0) continue;
      if (row_has_alive(sh, r, (uint32_t)phys_of(sh, pm, b, w))) mask |= 1ull << i;
    }
    out[1] = (int64_t)mask;
  }
}

// Replay of the mid-group skip rule (inference.py:127-146) from phase-1
// info: pick j > 0 stays a candidate iff rdeg(v_j) minus the number of
// earlier accepted picks it shares an alive edge with is > 0.  Returns the
// accepted mask and the global number of removed entries (2 * rdeg at apply).
__device__ uint64_t replay_group(const int64_t *picks, int d, const int64_t *info, int b,
                                 long long *removed_global, int first_forced) {
  uint64_t amask = 0;
  long long rem = 0;
  for (int j = 0; j < d && j < 64; j++) {
    const int64_t v = picks[(int64_t)b * d + j];
    if (v < 0) continue;
    int64_t deg = info[2 * ((int64_t)b * d + j)];
    const uint64_t adj = (uint64_t)info[2 * ((int64_t)b * d + j) + 1];
    if (j > 0) deg -= __popcll(adj & amask);
    if ((j == 0 && first_forced) || deg > 0) {
      amask |= 1ull << j;
      rem += 2 * deg;
    }
  }
  *removed_global = rem;
  return amask;
}

// Phase 2 (every rank): replay, then remove the accepted picks' rows (owner)
// and columns (every rank) in parallel.  Entries are killed with atomicOr so
// an edge between two accepted picks is counted exactly once; rdeg is
// decremented atomically.  grid = (chunks, B).
__global__ void apply_phase2_kernel(s2v_shard sh, const int64_t *picks, int d,
                                    const int64_t *info, uint8_t *applied, int64_t *removed,
                                    int first_forced) {
  const int b = blockIdx.y;
  __shared__ uint64_t s_amask;
  __shared__ unsigned long long s_local;
  if (threadIdx.x == 0) {
    long long rem = 0;
    s_amask = replay_group(picks, d, info, b, &rem, first_forced);
    s_local = 0;
    if (blockIdx.x == 0) {
      removed[b] = rem;
      for (int j = 0; j < d; j++)
        applied[(int64_t)b * d + j] = (j < 64 && ((s_amask >> j) & 1ull)) ? 1 : 0;
    }
  }
  __syncthreads();
  const uint64_t amask = s_amask;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (int j = 0; j < d && j < 64; j++) {
    if (!((amask >> j) & 1ull)) continue;
    const int64_t v = picks[(int64_t)b * d + j];
    if (v >= sh.row_start && v < sh.row_start + sh.num_rows) {
      const int64_t r = (int64_t)b * sh.num_rows + (v - sh.row_start);
      for (int64_t e = sh.row_ptr[r] + tid; e < sh.row_ptr[r + 1]; e += stride) {
        const uint32_t old = atomicOr(sh.cols + e, S2V_DEAD);
        if (!(old & S2V_DEAD)) {
          local++;
          atomicSub(sh.rdeg + r, 1);
        }
      }
      if (tid == 0) {
        sh.sol[r] = 1;
        sh.cand[r] = 0;
      }
    }
    const int64_t cb = (int64_t)b * sh.num_nodes + v;
    for (int64_t q = sh.col_ptr[cb] + tid; q < sh.col_ptr[cb + 1]; q += stride) {
      const int64_t e = sh.col_ent[q];
      const uint32_t old = atomicOr(sh.cols + e, S2V_DEAD);
      if (!(old & S2V_DEAD)) {
        local++;
        atomicSub(sh.rdeg + sh.col_row[q], 1);
      }
    }
  }
  if (local) atomicAdd(&s_local, local);
  __syncthreads();
  if (threadIdx.x == 0 && s_local)
    atomicAdd((unsigned long long *)&sh.residual[b], (unsigned long long)(-(long long)s_local));
}

// Phase 3: candidacy of the rows touched by the accepted picks
// (state.py:206-208 recomputes all row sums; only these rows can change).
__global__ void apply_phase3_kernel(s2v_shard sh, const int64_t *picks, int d,
                                    const uint8_t *applied) {
  const int b = blockIdx.y;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < d && j < 64; j++) {
    if (!applied[(int64_t)b * d + j]) continue;
    const int64_t v = picks[(int64_t)b * d + j];
    const int64_t cb = (int64_t)b * sh.num_nodes + v;
    for (int64_t q = sh.col_ptr[cb] + tid; q < sh.col_ptr[cb + 1]; q += stride) {
      const int32_t row = sh.col_row[q];
      sh.cand[row] = (sh.rdeg[row] > 0 && !sh.sol[row]) ? 1 : 0;
    }
  }
}


// ---------------------------------------------------------------------------
// Active-row list compaction (B = 1, P = 1): keep rows with rdeg > 0, stable.
// 4096 list entries per CTA (16 consecutive per thread): count, then scatter
// at the prefix of the CTA counts, then copy back.  Optionally the compact
// CSR of the kept rows: row_ptr over list positions (prefix of rdeg -- the
// alive entries of a row), then one warp per row copies its alive entries.
// ws: [nchunks rows][nchunks hub rows][nchunks entries][rows, hub rows, entries]
// ---------------------------------------------------------------------------
constexpr int kCompactPer = 16;
constexpr int kCompactChunk = 256 * kCompactPer;

__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t *s_red /*[8]*/) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  int64_t t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_red[w];
  return t;
}

// exclusive prefix of v over the block (256 threads)
__device__ __forceinline__ int64_t block_exscan_i64(int64_t v, int64_t *s_warp /*[8]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  int64_t before = 0;
  for (int w = 0; w < warp; w++) before += s_warp[w];
  return before + incl - v;
}

__global__ void __launch_bounds__(256) active_count_kernel(const int32_t *__restrict__ rdeg,
                                                           const int32_t *__restrict__ list,
                                                           const int64_t *__restrict__ n,
                                                           int64_t *__restrict__ ws, int nchunks) {
  __shared__ int64_t s_red[8];
  const int64_t cnt = n[0], nh = n[1];
  const int64_t j0 = (int64_t)blockIdx.x * kCompactChunk + threadIdx.x * kCompactPer;
  int64_t a = 0, h = 0, e = 0;
#pragma unroll
  for (int t = 0; t < kCompactPer; t++) {
    const int64_t j = j0 + t;
    if (j < cnt) {
      const int32_t d = rdeg[list[j]];
      if (d > 0) {
        a++;
        e += d;
        if (j < nh) h++;
      }
    }
  }
  a = block_sum_i64(a, s_red);
  h = block_sum_i64(h, s_red);
  e = block_sum_i64(e, s_red);
  if (threadIdx.x == 0) {
    ws[blockIdx.x] = a;
    ws[nchunks + blockIdx.x] = h;
    ws[2 * nchunks + blockIdx.x] = e;
  }
}

__global__ void __launch_bounds__(256) active_scatter_kernel(
    const int32_t *__restrict__ rdeg, const int32_t *__restrict__ list,
    const int64_t *__restrict__ n, int64_t *__restrict__ ws, int nchunks,
    int32_t *__restrict__ out, int64_t *__restrict__ row_ptr_out) {
  __shared__ int64_t s_red[8];
  const int tid = threadIdx.x;
  int64_t off = 0, eoff = 0;
  for (int c = tid; c < (int)blockIdx.x; c += 256) {
    off += ws[c];
    eoff += ws[2 * nchunks + c];
  }
  off = block_sum_i64(off, s_red);
  eoff = block_sum_i64(eoff, s_red);
  if (blockIdx.x == 0) {  // new totals, read by the copy-back kernel
    int64_t a = 0, h = 0, e = 0;
    for (int c = tid; c < nchunks; c += 256) {
      a += ws[c];
      h += ws[nchunks + c];
      e += ws[2 * nchunks + c];
    }
    a = block_sum_i64(a, s_red);
    h = block_sum_i64(h, s_red);
    e = block_sum_i64(e, s_red);
    if (tid == 0) {
      ws[3 * nchunks] = a;
      ws[3 * nchunks + 1] = h;
      ws[3 * nchunks + 2] = e;
    }
  }
  const int64_t cnt = n[0];
  const int64_t j0 = (int64_t)blockIdx.x * kCompactChunk + tid * kCompactPer;
  int32_t rows[kCompactPer], degs[kCompactPer];
  int64_t mine = 0, mine_e = 0;
#pragma unroll
  for (int t = 0; t < kCompactPer; t++) {
    const int64_t j = j0 + t;
    rows[t] = j < cnt ? list[j] : -1;
    degs[t] = rows[t] >= 0 ? rdeg[rows[t]] : 0;
    if (degs[t] > 0) {
      mine++;
      mine_e += degs[t];
    }
  }
  int64_t pos = off + block_exscan_i64(mine, s_red);
  int64_t epos = eoff + block_exscan_i64(mine_e, s_red);
#pragma unroll
  for (int t = 0; t < kCompactPer; t++)
    if (degs[t] > 0) {
      out[pos] = rows[t];
      if (row_ptr_out) row_ptr_out[pos] = epos;
      pos++;
      epos += degs[t];
    }
}

__global__ void active_copy_kernel(const int32_t *__restrict__ tmp, const int64_t *__restrict__ ws,
                                   int nchunks, int32_t *__restrict__ list,
                                   int64_t *__restrict__ n, int64_t *__restrict__ row_ptr_out) {
  const int64_t cnt = ws[3 * nchunks];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt;
       j += (int64_t)gridDim.x * blockDim.x)
    list[j] = tmp[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    n[0] = cnt;
    n[1] = ws[3 * nchunks + 1];
    if (row_ptr_out) row_ptr_out[cnt] = ws[3 * nchunks + 2];
  }
}

// one warp per kept row: its alive entries, in order, at row_ptr_out[j]
__global__ void __launch_bounds__(256) active_fill_kernel(s2v_shard sh,
                                                          const int32_t *__restrict__ list,
                                                          const int64_t *__restrict__ n,
                                                          const int64_t *__restrict__ row_ptr_out,
                                                          uint32_t *__restrict__ cols_out) {
  const int lane = threadIdx.x & 31;
  const int64_t cnt = n[0];
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < cnt;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t r = list[j];
    int64_t o = row_ptr_out[j];
    const int64_t e1 = sh.row_ptr[r + 1];
    for (int64_t e = sh.row_ptr[r]; e < e1; e += 32) {
      const bool in = e + lane < e1;
      const uint32_t c = in ? sh.cols[e + lane] : S2V_DEAD;
      const bool alive = !(c & S2V_DEAD);
      const unsigned m = __ballot_sync(0xffffffffu, alive);
      if (alive) cols_out[o + __popc(m & ((1u << lane) - 1))] = c;
      o += __popc(m);
    }
  }
}


// ---------------------------------------------------------------------------
// Block-diagonal batch assembly: dst[seg.dst + i] = src[i] + seg.add for
// every segment (one grid row per segment), for 4- or 8-byte integers.
// ---------------------------------------------------------------------------
template <class T>
__global__ void segment_copy_kernel(const s2v_segment *__restrict__ segs, T *__restrict__ dst) {
  const s2v_segment sg = segs[blockIdx.y];
  const T *src = reinterpret_cast<const T *>(sg.src);
  const T add = (T)sg.add;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < sg.len;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[sg.dst_off + i] = src[i] + add;
}

}  // namespace s2v

using namespace s2v;

extern "C" {

const char *s2v_last_error(void) { return g_last_error.c_str(); }
const char *s2v_version(void) { return "libs2v 0.1 sm_100a"; }

int s2v_set_device(int device) {
  S2V_CUDA_CHECK(cudaSetDevice(device));
  return S2V_OK;
}

int s2v_shard_init(const s2v_shard *sh, const uint32_t *cols_src, const uint8_t *sol_phys,
                   void *stream) {
  if (!sh || sh->batch < 1 || sh->world < 1) return fail(S2V_EINVAL, "bad shard");
  cudaStream_t st = as_stream(stream);
  S2V_CUDA_CHECK(cudaMemsetAsync(sh->residual, 0, sizeof(int64_t) * sh->batch, st));
  int64_t rows = (int64_t)sh->batch * sh->num_rows;
  if (rows == 0) return S2V_OK;
  const int64_t nphys = (int64_t)sh->batch * sh->world * sh->rows_max;
  // grow-only scratch per thread and device (no stream-ordered pool
  // allocation on this path: the pool trims at synchronisations and regrows)
  static thread_local struct {
    int dev = -1;
    uint32_t *p = nullptr;
    size_t bytes = 0;
  } scratch;
  int dev = 0;
  S2V_CUDA_CHECK(cudaGetDevice(&dev));
  // sol bitmap, then the long-row list (at most nnz / kInitLong rows) and
  // its count
  const size_t bits_bytes = (4 * (size_t)((nphys + 31) / 32) + 7) & ~(size_t)7;
  const size_t list_n = (size_t)(sh->nnz / kInitLong + 1);
  const size_t need = bits_bytes + 8 * list_n + 8 + 16 + 4 * kSumWords;
  if (scratch.dev != dev || scratch.bytes < need) {
    if (scratch.p && scratch.dev == dev) {
      S2V_CUDA_CHECK(cudaStreamSynchronize(st));
      cudaFree(scratch.p);
    }
    scratch.p = nullptr;
    S2V_CUDA_CHECK(cudaMalloc((void **)&scratch.p, need));
    scratch.dev = dev;
    scratch.bytes = need;
  }
  uint32_t *bits = scratch.p;
  int64_t *long_rows = reinterpret_cast<int64_t *>(reinterpret_cast<char *>(scratch.p) + bits_bytes);
  int *long_n = reinterpret_cast<int *>(long_rows + list_n);
  uint32_t *summary = reinterpret_cast<uint32_t *>(
      (reinterpret_cast<uintptr_t>(long_n + 2) + 15) & ~(uintptr_t)15);  // uint4 loads
  int lg = 3;
  while (((int64_t)kSumWords * 32 << lg) < nphys) lg++;
  S2V_CUDA_CHECK(cudaMemsetAsync(long_n, 0, sizeof(int), st));
  sol_bits_kernel<<<(unsigned)std::min<int64_t>(((nphys + 31) / 32 + 255) / 256, kNumSMs * 8),
                    256, 0, st>>>(sol_phys, nphys, bits);
  S2V_LAUNCH_CHECK();
  sol_summary_kernel<<<kSumWords / 256, 256, 0, st>>>(bits, nphys, lg, summary);
  S2V_LAUNCH_CHECK();
  // one resident wave (the loop is grid-strided and pipelined per warp)
  static const int per_sm = [] {
    int n = 0;
    cudaFuncSetAttribute(shard_init_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         4 * kSumWords);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, shard_init_kernel, 256, 4 * kSumWords);
    return n > 0 ? n : 4;
  }();
  int64_t blocks = (rows * 8 + 255) / 256;
  if (blocks > (int64_t)kNumSMs * per_sm) blocks = (int64_t)kNumSMs * per_sm;
  shard_init_kernel<<<(unsigned)blocks, 256, 4 * kSumWords, st>>>(
      *sh, cols_src, sol_phys, bits, long_rows, long_n, summary, lg);
  S2V_LAUNCH_CHECK();
  if (sh->nnz > kInitLong) {
    shard_init_long_kernel<<<(unsigned)std::min<int64_t>(sh->nnz / kInitLong, kNumSMs * 4), 256,
                             0, st>>>(*sh, cols_src, sol_phys, bits, long_rows, long_n);
    S2V_LAUNCH_CHECK();
  }
  return S2V_OK;
}

int s2v_apply_phase1(const s2v_shard *sh, const int64_t *picks, int d, int64_t *info,
                     int validate, int32_t *err_out, void *stream) {
  if (d < 1 || d > 64) return fail(S2V_EINVAL, "group size d=%d outside [1, 64]", d);
  cudaStream_t st = as_stream(stream);
  if (validate && err_out)
    S2V_CUDA_CHECK(cudaMemsetAsync(err_out, 0, sizeof(int32_t) * sh->batch, st));
  apply_phase1_kernel<<<sh->batch, 64, 0, st>>>(*sh, make_map(*sh), picks, d, info,
                                                validate && err_out, err_out);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_apply_phase2(const s2v_shard *sh, const int64_t *picks, int d, const int64_t *info,
                     uint8_t *applied, int64_t *removed, int first_forced, void *stream) {
  if (d < 1 || d > 64) return fail(S2V_EINVAL, "group size d=%d outside [1, 64]", d);
  dim3 grid(16, sh->batch);
  apply_phase2_kernel<<<grid, 256, 0, as_stream(stream)>>>(*sh, picks, d, info, applied, removed,
                                                           first_forced);
  S2V_LAUNCH_CHECK();
  apply_phase3_kernel<<<grid, 256, 0, as_stream(stream)>>>(*sh, picks, d, applied);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_sol_mark(const s2v_shard *sh, const int64_t *picks, const uint8_t *applied, int d,
                 uint8_t *sol_all, void *stream) {
  if (d < 1 || d > 64) return fail(S2V_EINVAL, "group size d=%d outside [1, 64]", d);
  const int n = sh->batch * d;
  sol_mark_kernel<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(*sh, make_map(*sh), picks,
                                                                   applied, d, sol_all);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int64_t s2v_active_workspace(int64_t cap) {
  return 3 * ((cap + kCompactChunk - 1) / kCompactChunk) + 3;
}

int s2v_active_compact(const s2v_shard *sh, int32_t *list, int64_t *n, int32_t *tmp,
                       int64_t *ws, int64_t cap, int64_t *row_ptr_out, uint32_t *cols_out,
                       void *stream) {
  // (the list holds local rows and the CSR physical neighbour rows: any P;
  // at P > 1 the rounds reading the CSR need shard.active_sol)
  if (sh->batch != 1) return fail(S2V_EINVAL, "active-row lists need B = 1");
  if ((row_ptr_out == nullptr) != (cols_out == nullptr))
    return fail(S2V_EINVAL, "compact CSR needs both row_ptr_out and cols_out");
  if (cap <= 0) return S2V_OK;
  cudaStream_t st = as_stream(stream);
  const int nchunks = (int)((cap + kCompactChunk - 1) / kCompactChunk);
  active_count_kernel<<<nchunks, 256, 0, st>>>(sh->rdeg, list, n, ws, nchunks);
  S2V_LAUNCH_CHECK();
  active_scatter_kernel<<<nchunks, 256, 0, st>>>(sh->rdeg, list, n, ws, nchunks, tmp, row_ptr_out);
  S2V_LAUNCH_CHECK();
  const int cgrid = (int)std::min<int64_t>((cap + 255) / 256, kNumSMs * 4);
  active_copy_kernel<<<cgrid, 256, 0, st>>>(tmp, ws, nchunks, list, n, row_ptr_out);
  S2V_LAUNCH_CHECK();
  if (cols_out) {
    const int fgrid = (int)std::min<int64_t>((cap + 7) / 8, kNumSMs * 8);
    active_fill_kernel<<<fgrid, 256, 0, st>>>(*sh, list, n, row_ptr_out, cols_out);
    S2V_LAUNCH_CHECK();
  }
  return S2V_OK;
}

int s2v_segment_copy(int elem_bytes, const s2v_segment *segs, int nseg, int64_t max_len,
                     void *dst, void *stream) {
  if (nseg <= 0 || max_len <= 0) return S2V_OK;
  if (elem_bytes != 4 && elem_bytes != 8) return fail(S2V_EINVAL, "segment copy: 4 or 8 bytes");
  if (nseg > 65535) return fail(S2V_EINVAL, "segment copy: at most 65535 segments");
  dim3 grid((unsigned)std::min<int64_t>((max_len + 255) / 256, 1024), (unsigned)nseg);
  if (elem_bytes == 4)
    segment_copy_kernel<int32_t><<<grid, 256, 0, as_stream(stream)>>>(segs, (int32_t *)dst);
  else
    segment_copy_kernel<int64_t><<<grid, 256, 0, as_stream(stream)>>>(segs, (int64_t *)dst);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // extern "C"
