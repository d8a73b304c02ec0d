// Incremental forward for the tail of an episode (B = 1, P = 1).
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

}  // extern "C"
