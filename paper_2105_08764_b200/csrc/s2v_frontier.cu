// Incremental forward for the tail of an episode (B = 1; P = 1 by CSR walks
// from the frontier rows, P > 1 by all-gathered bitmaps, below).
//
// Late in an adaptive episode (inference.py:107-147) the residual graph is a
// forest of small components and each evaluation applies one or two picks.
// A pick v changes the round-1 rows of v and of its alive neighbours (their
// residual degree drops, state.py:173-208); a round-l output h_l[x] reads
// the h_{l-1} rows of x's alive neighbours, so it can only change within
// l-1 further hops.  The *frontier* D holds, level by level, the rows whose
// h_l may differ from the previous evaluation:
//   D_1 = picks + their alive neighbours                     (before apply)
//   D_l = D_{l-1} + alive neighbours of the rows new in D_{l-1} (after apply)
// in one array (BFS order, deduplicated by an epoch stamp per row), level l
// being the prefix [0, E[l]).  Round l then recomputes only D_l -- every
// other row's h_l is bit-identical to the value kept from the previous
// evaluation -- and the global sum / scores are refreshed for D_L only.  If
// the frontier outgrows `cap`, the active-row list is copied into D for
// every level and the evaluation recomputes every active row.
//
// meta (int64): [0] rows appended, [1] epoch, [2] overflow, [3] unused,
//               [4 + 2l], [5 + 2l] = {E[l], 0} for l = 0..L (an s2v_shard
//               active_n pair: rows of level l, no hub rows).
#include <algorithm>

#include "s2v_common.cuh"

namespace s2v {

__device__ __forceinline__ void frontier_add(int32_t u, int32_t epoch, int32_t *__restrict__ D,
                                             int64_t *__restrict__ meta,
                                             int32_t *__restrict__ mark) {
  if (atomicExch(&mark[u], epoch) != epoch) {
    const unsigned long long at = atomicAdd((unsigned long long *)&meta[0], 1ull);
    D[at] = u;
  }
}

__global__ void frontier_begin_kernel(int64_t *meta, int levels) {
  meta[0] = 0;
  meta[1] += 1;
  meta[2] = 0;
  for (int l = 0; l <= levels; l++) {
    meta[4 + 2 * l] = 0;
    meta[5 + 2 * l] = 0;
  }
}

// one block per pick: the pick and its alive neighbours (removed-entry bits
// of the full CSR, read before the group is applied)
__global__ void __launch_bounds__(256) frontier_seed_kernel(s2v_shard sh,
                                                            const int64_t *__restrict__ picks,
                                                            int32_t *__restrict__ D,
                                                            int64_t *__restrict__ meta,
                                                            int32_t *__restrict__ mark) {
  const int64_t v = picks[blockIdx.x];
  if (v < 0 || v >= sh.num_rows) return;
  const int32_t epoch = (int32_t)meta[1];
  if (threadIdx.x == 0) frontier_add((int32_t)v, epoch, D, meta, mark);
  const int64_t e1 = sh.row_ptr[v + 1];
  for (int64_t e = sh.row_ptr[v] + threadIdx.x; e < e1; e += blockDim.x) {
    const uint32_t c = sh.cols[e];
    if (!(c & S2V_DEAD)) frontier_add((int32_t)c, epoch, D, meta, mark);
  }
}

// level l: alive neighbours (after the apply) of the rows new at level l-1;
// one warp per frontier row
__global__ void __launch_bounds__(256) frontier_expand_kernel(s2v_shard sh, int level,
                                                              int32_t *__restrict__ D,
                                                              int64_t *__restrict__ meta,
                                                              int32_t *__restrict__ mark,
                                                              int64_t cap) {
  if (meta[2]) return;  // overflowed: the evaluation recomputes every row
  const int lane = threadIdx.x & 31;
  const int32_t epoch = (int32_t)meta[1];
  const int64_t f0 = level >= 2 ? meta[4 + 2 * (level - 2)] : 0;
  const int64_t f1 = meta[4 + 2 * (level - 1)];
  for (int64_t j = f0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); j < f1;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t x = D[j];
    const int64_t e1 = sh.row_ptr[x + 1];
    for (int64_t e = sh.row_ptr[x] + lane; e < e1; e += 32) {
      const uint32_t c = sh.cols[e];
      if (!(c & S2V_DEAD)) frontier_add((int32_t)c, epoch, D, meta, mark);
    }
  }
}

__global__ void frontier_close_kernel(int64_t *meta, int level, int64_t cap) {
  const int64_t n = meta[0];
  meta[4 + 2 * level] = n;
  if (n > cap) meta[2] = 1;
}

// overflow: every level = the whole active list
__global__ void frontier_fallback_kernel(int32_t *__restrict__ D, int64_t *__restrict__ meta,
                                         int levels, const int32_t *__restrict__ act,
                                         const int64_t *__restrict__ act_n) {
  if (!meta[2]) return;
  const int64_t n = act_n[0];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    D[j] = act[j];
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int l = 0; l <= levels; l++) meta[4 + 2 * l] = n;
}


// ---------------------------------------------------------------------------
// P > 1: the frontier crosses ranks (a pick's neighbours, and theirs, may be
// anyone's rows), so the BFS runs on bitmaps over every rank's physical rows
// (B = 1): each rank marks the alive neighbours of its own rows into `mbits`,
// the ranks all-gather and OR them (s2v_frontier_bits_merge, identical on
// every rank), and each rank appends the new rows that are its own to the
// same D / meta level prefixes as P = 1, so rounds, scores and the fallback
// are unchanged.  The marking never stops on a local overflow: other ranks'
// levels depend on it.
__device__ __forceinline__ void set_bit(uint32_t *bits, uint32_t p) {
  atomicOr(bits + (p >> 5), 1u << (p & 31));
}

__device__ __forceinline__ bool get_bit(const uint32_t *bits, int64_t p) {
  return (bits[p >> 5] >> (p & 31)) & 1u;
}

__global__ void zero_words_kernel(uint32_t *__restrict__ a, uint32_t *__restrict__ b, int64_t w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < w;
       i += (int64_t)gridDim.x * blockDim.x) {
    a[i] = 0u;
    if (b) b[i] = 0u;
  }
}

// one block per pick owned by this rank: the pick and its alive neighbours
__global__ void __launch_bounds__(256) bits_seed_kernel(s2v_shard sh,
                                                        const int64_t *__restrict__ picks,
                                                        uint32_t *__restrict__ mbits) {
  const int64_t v = picks[blockIdx.x];
  if (v < sh.row_start || v >= sh.row_start + sh.num_rows) return;
  const int64_t i = v - sh.row_start;
  if (threadIdx.x == 0) set_bit(mbits, (uint32_t)(sh.rank * sh.rows_max + i));
  const int64_t e1 = sh.row_ptr[i + 1];
  for (int64_t e = sh.row_ptr[i] + threadIdx.x; e < e1; e += blockDim.x) {
    const uint32_t c = sh.cols[e];
    if (!(c & S2V_DEAD)) set_bit(mbits, c);
  }
}

// alive neighbours of this rank's rows whose bit is set in `newbits`; one
// warp per 32-row word (rows without a set bit cost one word read)
__global__ void __launch_bounds__(256) bits_expand_kernel(s2v_shard sh,
                                                          const uint32_t *__restrict__ newbits,
                                                          uint32_t *__restrict__ mbits) {
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)sh.rank * sh.rows_max;
  const int64_t nw = (sh.num_rows + 31) / 32;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    for (int q = 0; q < 32; q++) {
      const int64_t i = 32 * w + q;
      if (i >= sh.num_rows || !get_bit(newbits, base + i)) continue;
      const int64_t e1 = sh.row_ptr[i + 1];
      for (int64_t e = sh.row_ptr[i] + lane; e < e1; e += 32) {
        const uint32_t c = sh.cols[e];
        if (!(c & S2V_DEAD)) set_bit(mbits, c);
      }
    }
  }
}

// X = OR over ranks of gathered[r]; newbits = X & ~gbits; gbits |= X
__global__ void bits_merge_kernel(int P, int64_t w, const uint32_t *__restrict__ gathered,
                                  uint32_t *__restrict__ gbits, uint32_t *__restrict__ newbits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < w;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = 0u;
    for (int r = 0; r < P; r++) x |= gathered[(int64_t)r * w + i];
    const uint32_t g = gbits[i];
    newbits[i] = x & ~g;
    gbits[i] = g | x;
  }
}

// this rank's rows new at this level (bit in newbits) -> D (epoch-deduped)
__global__ void bits_append_kernel(s2v_shard sh, const uint32_t *__restrict__ newbits,
                                   int32_t *__restrict__ D, int64_t *__restrict__ meta,
                                   int32_t *__restrict__ mark) {
  const int32_t epoch = (int32_t)meta[1];
  const int64_t base = (int64_t)sh.rank * sh.rows_max;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < sh.num_rows;
       i += (int64_t)gridDim.x * blockDim.x)
    if (get_bit(newbits, base + i)) frontier_add((int32_t)i, epoch, D, meta, mark);
}

// global node ids of the set bits (the dirty rows of the global sum)
__global__ void bits_nodes_kernel(int64_t N, int P, int64_t rows_max,
                                  const uint32_t *__restrict__ gbits, int32_t *__restrict__ nodes,
                                  int64_t *__restrict__ n) {
  const int64_t base = N / P, extra = N % P;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < (int64_t)P * rows_max;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!get_bit(gbits, p)) continue;
    const int64_t r = p / rows_max, i = p - r * rows_max;
    const int64_t start = r * base + (r < extra ? r : extra);
    const unsigned long long at = atomicAdd((unsigned long long *)n, 1ull);
    nodes[at] = (int32_t)(start + i);
  }
}

}  // namespace s2v

using namespace s2v;

extern "C" {

int s2v_frontier_seed(const s2v_shard *sh, const int64_t *picks, int d, int levels, int32_t *D,
                      int64_t *meta, int32_t *mark, int64_t cap, void *stream) {
  if (sh->batch != 1 || sh->world != 1) return fail(S2V_EINVAL, "frontier needs B = 1, P = 1");
  if (d < 1 || levels < 1) return fail(S2V_EINVAL, "bad frontier args");
  cudaStream_t st = as_stream(stream);
  frontier_begin_kernel<<<1, 1, 0, st>>>(meta, levels);
  S2V_LAUNCH_CHECK();
  frontier_seed_kernel<<<d, 256, 0, st>>>(*sh, picks, D, meta, mark);
  S2V_LAUNCH_CHECK();
  frontier_close_kernel<<<1, 1, 0, st>>>(meta, 1, cap);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_frontier_expand(const s2v_shard *sh, int levels, int32_t *D, int64_t *meta, int32_t *mark,
                        int64_t cap, const int32_t *act, const int64_t *act_n, int64_t act_cap,
                        void *stream) {
  if (sh->batch != 1 || sh->world != 1) return fail(S2V_EINVAL, "frontier needs B = 1, P = 1");
  cudaStream_t st = as_stream(stream);
  for (int l = 2; l <= levels; l++) {
    frontier_expand_kernel<<<kNumSMs * 2, 256, 0, st>>>(*sh, l, D, meta, mark, cap);
    S2V_LAUNCH_CHECK();
    frontier_close_kernel<<<1, 1, 0, st>>>(meta, l, cap);
    S2V_LAUNCH_CHECK();
  }
  const int g = (int)std::min<int64_t>((act_cap + 255) / 256, kNumSMs * 4);
  frontier_fallback_kernel<<<std::max(g, 1), 256, 0, st>>>(D, meta, levels, act, act_n);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int64_t s2v_frontier_meta_size(int levels) { return 4 + 2 * (int64_t)(levels + 1); }

int64_t s2v_frontier_bits_words(const s2v_shard *sh) {
  return ((int64_t)sh->world * sh->rows_max + 31) / 32;
}

int s2v_frontier_bits_seed(const s2v_shard *sh, const int64_t *picks, int d, int levels,
                           int64_t *meta, uint32_t *mbits, uint32_t *gbits, void *stream) {
  if (sh->batch != 1) return fail(S2V_EINVAL, "frontier needs B = 1");
  if (d < 1 || levels < 1) return fail(S2V_EINVAL, "bad frontier args");
  cudaStream_t st = as_stream(stream);
  const int64_t w = s2v_frontier_bits_words(sh);
  frontier_begin_kernel<<<1, 1, 0, st>>>(meta, levels);
  S2V_LAUNCH_CHECK();
  zero_words_kernel<<<(int)std::min<int64_t>((w + 255) / 256, kNumSMs * 4), 256, 0, st>>>(
      mbits, gbits, w);
  S2V_LAUNCH_CHECK();
  bits_seed_kernel<<<d, 256, 0, st>>>(*sh, picks, mbits);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_frontier_bits_expand(const s2v_shard *sh, const uint32_t *newbits, uint32_t *mbits,
                             void *stream) {
  if (sh->batch != 1) return fail(S2V_EINVAL, "frontier needs B = 1");
  cudaStream_t st = as_stream(stream);
  const int64_t w = s2v_frontier_bits_words(sh);
  zero_words_kernel<<<(int)std::min<int64_t>((w + 255) / 256, kNumSMs * 4), 256, 0, st>>>(
      mbits, nullptr, w);
  S2V_LAUNCH_CHECK();
  const int64_t nw = (sh->num_rows + 31) / 32;
  bits_expand_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((nw * 32 + 255) / 256,
                                                                   kNumSMs * 8)),
                       256, 0, st>>>(*sh, newbits, mbits);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_frontier_bits_merge(const s2v_shard *sh, const uint32_t *gathered, uint32_t *gbits,
                            uint32_t *newbits, int level, int levels, int32_t *D, int64_t *meta,
                            int32_t *mark, int64_t cap, const int32_t *act, const int64_t *act_n,
                            int64_t act_cap, void *stream) {
  if (sh->batch != 1) return fail(S2V_EINVAL, "frontier needs B = 1");
  cudaStream_t st = as_stream(stream);
  const int64_t w = s2v_frontier_bits_words(sh);
  bits_merge_kernel<<<(int)std::min<int64_t>((w + 255) / 256, kNumSMs * 4), 256, 0, st>>>(
      sh->world, w, gathered, gbits, newbits);
  S2V_LAUNCH_CHECK();
  bits_append_kernel<<<(int)std::max<int64_t>(
                           1, std::min<int64_t>((sh->num_rows + 255) / 256, kNumSMs * 4)),
                       256, 0, st>>>(*sh, newbits, D, meta, mark);
  S2V_LAUNCH_CHECK();
  frontier_close_kernel<<<1, 1, 0, st>>>(meta, level, cap);
  S2V_LAUNCH_CHECK();
  if (level == levels) {
    const int g = (int)std::min<int64_t>((act_cap + 255) / 256, kNumSMs * 4);
    frontier_fallback_kernel<<<std::max(g, 1), 256, 0, st>>>(D, meta, levels, act, act_n);
    S2V_LAUNCH_CHECK();
  }
  return S2V_OK;
}

int s2v_frontier_bits_nodes(const s2v_shard *sh, const uint32_t *gbits, int32_t *nodes,
                            int64_t *n, void *stream) {
  cudaStream_t st = as_stream(stream);
  S2V_CUDA_CHECK(cudaMemsetAsync(n, 0, 2 * sizeof(int64_t), st));
  const int64_t tot = (int64_t)sh->world * sh->rows_max;
  bits_nodes_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256,
                                                                  kNumSMs * 4)),
                      256, 0, st>>>(sh->num_nodes, sh->world, sh->rows_max, gbits, nodes, n);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}


}  // extern "C"
