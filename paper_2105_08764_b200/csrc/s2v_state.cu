// Residual-graph state kernels: shard initialisation and group application of
// picks.  Integer-only, hence exact.
//
// Replaces (paths relative to /root/reference):
//   PartitionedState.__init__ residual mask / degrees   pkg/src/graphrl/state.py:89-111
//   PartitionedState.apply_action                       pkg/src/graphrl/state.py:173-208
//   _solve_batch group loop with mid-group skip         pkg/src/graphrl/inference.py:125-146
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

// One warp per local row: entry alive iff neither endpoint is in S.
__global__ void shard_init_kernel(s2v_shard sh, const uint8_t *__restrict__ sol_phys) {
  const int lane = threadIdx.x & 31;
  const int64_t nrows = (int64_t)sh.batch * sh.num_rows;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < nrows;
       r += (gridDim.x * (int64_t)blockDim.x) >> 5) {
    const int64_t b = r / sh.num_rows, i = r - b * sh.num_rows;
    const uint8_t s = sol_phys[(b * sh.world + sh.rank) * sh.rows_max + i];
    int cnt = 0;
    for (int64_t e = sh.row_ptr[r] + lane; e < sh.row_ptr[r + 1]; e += 32) {
      uint32_t c = sh.cols[e] & ~S2V_DEAD;
      bool dead = s || sol_phys[c];
      sh.cols[e] = c | (dead ? S2V_DEAD : 0u);
      cnt += !dead;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
      sh.rdeg[r] = cnt;
      sh.sol[r] = s;
      sh.cand[r] = (cnt > 0 && !s) ? 1 : 0;
      if (cnt) atomicAdd((unsigned long long *)&sh.residual[b], (unsigned long long)cnt);
    }
  }
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

// Phase 2 (every rank): replay the skip rule identically, then apply the
// accepted picks to this rank's rows (row v if owned) and columns (entries
// whose neighbour is v).  One CTA per slot; picks are applied in order.
__global__ void apply_phase2_kernel(s2v_shard sh, const int64_t *picks, int d,
                                    const int64_t *info, uint8_t *applied, int64_t *removed) {
  const int b = blockIdx.x;
  __shared__ unsigned long long s_removed_local;
  __shared__ uint64_t s_applied_mask;
  if (threadIdx.x == 0) {
    uint64_t amask = 0;
    long long rem_global = 0;
    for (int j = 0; j < d; j++) {
      int64_t v = picks[(int64_t)b * d + j];
      bool ok = false;
      if (v >= 0) {
        int64_t deg = info[2 * ((int64_t)b * d + j)];
        uint64_t adj = (uint64_t)info[2 * ((int64_t)b * d + j) + 1];
        if (j > 0) deg -= __popcll(adj & amask);
        ok = (j == 0) || deg > 0;
        if (ok) rem_global += 2 * deg;
      }
      if (ok && j < 64) amask |= 1ull << j;
      applied[(int64_t)b * d + j] = ok ? 1 : 0;
    }
    s_applied_mask = amask;
    s_removed_local = 0;
    removed[b] = rem_global;
  }
  __syncthreads();
  const uint64_t amask = s_applied_mask;
  unsigned long long local = 0;
  for (int j = 0; j < d && j < 64; j++) {
    if (!((amask >> j) & 1ull)) continue;
    const int64_t v = picks[(int64_t)b * d + j];
    // row v (owner only)
    if (v >= sh.row_start && v < sh.row_start + sh.num_rows) {
      const int64_t r = (int64_t)b * sh.num_rows + (v - sh.row_start);
      for (int64_t e = sh.row_ptr[r] + threadIdx.x; e < sh.row_ptr[r + 1]; e += blockDim.x) {
        uint32_t c = sh.cols[e];
        if (!(c & S2V_DEAD)) {
          sh.cols[e] = c | S2V_DEAD;
          local++;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        sh.rdeg[r] = 0;
        sh.sol[r] = 1;
        sh.cand[r] = 0;
      }
    }
    // column v: each local row holds at most one entry whose neighbour is v
    const int64_t cb = (int64_t)b * sh.num_nodes + v;
    for (int64_t k = sh.col_ptr[cb] + threadIdx.x; k < sh.col_ptr[cb + 1]; k += blockDim.x) {
      int64_t e = sh.col_ent[k];
      uint32_t c = sh.cols[e];
      if (!(c & S2V_DEAD)) {
        sh.cols[e] = c | S2V_DEAD;
        local++;
        int32_t row = sh.col_row[k];
        int32_t nd = sh.rdeg[row] - 1;
        sh.rdeg[row] = nd;
        sh.cand[row] = (nd > 0 && !sh.sol[row]) ? 1 : 0;
      }
    }
    __syncthreads();
  }
  if (local) atomicAdd(&s_removed_local, local);
  __syncthreads();
  if (threadIdx.x == 0) sh.residual[b] -= (int64_t)s_removed_local;
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

int s2v_shard_init(const s2v_shard *sh, const uint8_t *sol_phys, void *stream) {
  if (!sh || sh->batch < 1 || sh->world < 1) return fail(S2V_EINVAL, "bad shard");
  cudaStream_t st = as_stream(stream);
  S2V_CUDA_CHECK(cudaMemsetAsync(sh->residual, 0, sizeof(int64_t) * sh->batch, st));
  int64_t rows = (int64_t)sh->batch * sh->num_rows;
  if (rows == 0) return S2V_OK;
  int64_t blocks = (rows * 32 + 255) / 256;
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  shard_init_kernel<<<(unsigned)blocks, 256, 0, st>>>(*sh, sol_phys);
  S2V_LAUNCH_CHECK();
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
                     uint8_t *applied, int64_t *removed, void *stream) {
  if (d < 1 || d > 64) return fail(S2V_EINVAL, "group size d=%d outside [1, 64]", d);
  apply_phase2_kernel<<<sh->batch, 256, 0, as_stream(stream)>>>(*sh, picks, d, info, applied,
                                                                removed);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // extern "C"
