// Device-side build of one graph's shard structure (replaces the host
// numpy work of the round-1 state build: 8.4 s at BA(2M,16), BENCH r1).
//
// Reference: PartitionedState's CSR build and column lookup,
// pkg/src/graphrl/state.py:89-105 (local rows of the global CSR) and
// state.py:115-122 (_col_order / _col_ptr: for every global column v, the
// local entries in that column, rows ascending).  Same arrays as before,
// bit for bit: cols0 (neighbour -> physical row at P > 1), col_ptr,
// col_ent (stable argsort of the neighbour ids), col_row (their local rows),
// order (stable argsort by descending degree) and the hub count.
// The two stable sorts are cub radix sorts (setup path, not the hot path).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "s2v_common.cuh"

namespace s2v {
namespace {

// phys_rows (state.py restated in paper_2105_08764_b200/state.py): global
// node u -> r * rows_max + (u - start_r) under partition_rows' block split
__device__ __forceinline__ int64_t phys_of_node(int64_t u, int64_t n, int P, int64_t rows_max) {
  const int64_t base = n / P, extra = n % P, big = extra * (base + 1);
  const int64_t r = u < big ? u / (base + 1) : extra + (u - big) / (base > 0 ? base : 1);
  const int64_t start = r * base + (r < extra ? r : extra);
  return r * rows_max + (u - start);
}

__global__ void cols_phys_kernel(const int32_t *__restrict__ nbr, int64_t nnz, int64_t n, int P,
                                 int64_t rows_max, int32_t *__restrict__ cols0,
                                 int32_t *__restrict__ hist, int64_t *__restrict__ iota) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = nbr[e];
    cols0[e] = P > 1 ? (int32_t)phys_of_node(v, n, P, rows_max) : v;
    atomicAdd(hist + v, 1);
    iota[e] = e;
  }
}

// per row: local row id of every entry, descending-degree sort key, iota
__global__ void rows_kernel(const int64_t *__restrict__ row_ptr, int64_t rows, int32_t max_deg,
                            int32_t *__restrict__ entry_row, uint32_t *__restrict__ deg_key,
                            int32_t *__restrict__ iota_rows, int32_t hub_degree,
                            unsigned long long *__restrict__ n_hub) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
    for (int64_t e = e0; e < e1; e++) entry_row[e] = (int32_t)r;
    const int32_t d = (int32_t)(e1 - e0);
    deg_key[r] = (uint32_t)(max_deg - d);  // ascending key = descending degree
    iota_rows[r] = (int32_t)r;
    if (d > hub_degree) atomicAdd(n_hub, 1ull);
  }
}

__global__ void max_deg_kernel(const int64_t *__restrict__ row_ptr, int64_t rows,
                               int *__restrict__ out) {
  int m = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int)(row_ptr[r + 1] - row_ptr[r]));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void widen_kernel(const int32_t *__restrict__ hist, int64_t n,
                             int64_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hist[i];
}

__global__ void gather_rows_kernel(const int64_t *__restrict__ col_ent,
                                   const int32_t *__restrict__ entry_row, int64_t nnz,
                                   int32_t *__restrict__ col_row) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    col_row[e] = entry_row[col_ent[e]];
}

inline int grid_for(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, kNumSMs * 16));
}

// (setup path, once per graph: the stream-ordered pool is trimmed at the
// final synchronisation; hot paths use grow-only cudaMalloc scratch instead)
template <class T>
int dev_alloc(T **p, size_t count, cudaStream_t st) {
  S2V_CUDA_CHECK(cudaMallocAsync((void **)p, std::max<size_t>(count, 1) * sizeof(T), st));
  return S2V_OK;
}

}  // namespace
}  // namespace s2v

using namespace s2v;

extern "C" {

int s2v_shard_structure(int64_t n, int P, int64_t rows_max, int64_t rows,
                        const int64_t *row_ptr, const int32_t *nbr, int64_t nnz, int32_t *cols0,
                        int64_t *col_ptr, int64_t *col_ent, int32_t *col_row, int32_t *order,
                        int64_t *n_hub_out, int32_t *max_deg_out, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (n < 0 || rows < 0 || nnz < 0 || P < 1) return fail(S2V_EINVAL, "bad shard dimensions");
  if (nnz >= ((int64_t)1 << 31) || n >= ((int64_t)1 << 31))
    return fail(S2V_EINVAL, "shard too large for 32-bit column ids");
  int rc = S2V_OK;
  int32_t *hist = nullptr, *entry_row = nullptr, *keys_out = nullptr, *iota_rows = nullptr;
  uint32_t *deg_key = nullptr, *deg_key_out = nullptr;
  int64_t *iota = nullptr;
  int *dmax = nullptr;
  unsigned long long *nhub = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0, need = 0;
  int h_max = 0;
  unsigned long long h_hub = 0;
#define S2V_TRY(x)        \
  do {                    \
    rc = (x);             \
    if (rc) goto cleanup; \
  } while (0)
  S2V_TRY(dev_alloc(&hist, (size_t)n + 1, st));
  S2V_TRY(dev_alloc(&entry_row, (size_t)nnz, st));
  S2V_TRY(dev_alloc(&keys_out, (size_t)nnz, st));
  S2V_TRY(dev_alloc(&iota, (size_t)nnz, st));
  S2V_TRY(dev_alloc(&iota_rows, (size_t)rows, st));
  S2V_TRY(dev_alloc(&deg_key, (size_t)rows, st));
  S2V_TRY(dev_alloc(&deg_key_out, (size_t)rows, st));
  S2V_TRY(dev_alloc(&dmax, 1, st));
  S2V_TRY(dev_alloc(&nhub, 1, st));
  if (cudaMemsetAsync(hist, 0, sizeof(int32_t) * (n + 1), st) ||
      cudaMemsetAsync(dmax, 0, sizeof(int), st) ||
      cudaMemsetAsync(nhub, 0, sizeof(unsigned long long), st)) {
    rc = fail(S2V_ECUDA, "memset failed");
    goto cleanup;
  }
  max_deg_kernel<<<grid_for(rows), 256, 0, st>>>(row_ptr, rows, dmax);
  if (cudaMemcpyAsync(&h_max, dmax, sizeof(int), cudaMemcpyDeviceToHost, st) ||
      cudaStreamSynchronize(st)) {
    rc = fail(S2V_ECUDA, "max degree read-back failed");
    goto cleanup;
  }
  if (nnz)
    cols_phys_kernel<<<grid_for(nnz), 256, 0, st>>>(nbr, nnz, n, P, rows_max, cols0, hist,
                                                     iota);
  if (rows)
    rows_kernel<<<grid_for(rows), 256, 0, st>>>(row_ptr, rows, h_max, entry_row, deg_key,
                                                 iota_rows, S2V_HUB_DEGREE, nhub);
  // col_ptr = exclusive scan of the column histogram (n + 1 entries)
  widen_kernel<<<grid_for(n + 1), 256, 0, st>>>(hist, n + 1, col_ptr);
  cub::DeviceScan::ExclusiveSum(nullptr, need, col_ptr, col_ptr, n + 1, st);
  tmp_bytes = std::max(tmp_bytes, need);
  cub::DeviceRadixSort::SortPairs(nullptr, need, nbr, keys_out, iota, col_ent, (int)nnz, 0, 32,
                                  st);
  tmp_bytes = std::max(tmp_bytes, need);
  cub::DeviceRadixSort::SortPairs(nullptr, need, deg_key, deg_key_out, iota_rows, order,
                                  (int)rows, 0, 32, st);
  tmp_bytes = std::max(tmp_bytes, need);
  S2V_TRY(dev_alloc((uint8_t **)&tmp, tmp_bytes, st));
  need = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, need, col_ptr, col_ptr, n + 1, st);
  if (nnz) {
    // stable by column: entries of one column stay in ascending entry
    // (= ascending local row) order, as np.argsort(kind="stable")
    need = tmp_bytes;
    cub::DeviceRadixSort::SortPairs(tmp, need, nbr, keys_out, iota, col_ent, (int)nnz, 0, 32, st);
    gather_rows_kernel<<<grid_for(nnz), 256, 0, st>>>(col_ent, entry_row, nnz, col_row);
  }
  if (rows) {
    need = tmp_bytes;
    cub::DeviceRadixSort::SortPairs(tmp, need, deg_key, deg_key_out, iota_rows, order, (int)rows,
                                    0, 32, st);
  }
  if (cudaMemcpyAsync(&h_hub, nhub, sizeof(h_hub), cudaMemcpyDeviceToHost, st) ||
      cudaStreamSynchronize(st)) {
    rc = fail(S2V_ECUDA, "shard structure build failed: %s", cudaGetErrorString(cudaGetLastError()));
    goto cleanup;
  }
  if (n_hub_out) *n_hub_out = (int64_t)h_hub;
  if (max_deg_out) *max_deg_out = h_max;
cleanup:
#undef S2V_TRY
  for (void *p : {(void *)hist, (void *)entry_row, (void *)keys_out, (void *)iota,
                  (void *)iota_rows, (void *)deg_key, (void *)deg_key_out, (void *)dmax,
                  (void *)nhub, tmp})
    if (p) cudaFreeAsync(p, st);
  return rc;
}

}  // extern "C"
