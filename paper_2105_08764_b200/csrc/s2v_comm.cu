// NCCL collectives behind the C ABI.  Replaces the reference's in-process
// thread rendezvous (pkg/src/graphrl/collective.py:100-146) for the device
// data path: the per-round halo all-gather of embeddings (in place, one call
// per batch slot inside an NCCL group), and small all-reduces of integer
// selection info / fp64 gradient packs.  Host-side bookkeeping collectives
// stay in Python (torch.distributed / thread rendezvous).
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>

#include "s2v_common.cuh"

using namespace s2v;

namespace {

// out[i] = ((g[0][i] + g[1][i]) + g[2][i]) + ...: the reference's all-reduce
// order (collective.py:114-116: out = slots[0].astype(...); out += other for
// the later ranks), so every rank computes the same bits as the reference.
template <class T>
__global__ void sum_ranks_typed_kernel(int P, int64_t n, const T *__restrict__ g,
                                       T *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    T acc = g[i];
    for (int r = 1; r < P; r++) acc = acc + g[(int64_t)r * n + i];
    out[i] = acc;
  }
}

}  // namespace

typedef CUresult (*PFN_addr_range)(CUdeviceptr *, size_t *, CUdeviceptr);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <class F>
static int driver_fn(const char *name, F *out) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  S2V_CUDA_CHECK(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess)
    return fail(S2V_ECUDA, "driver entry point %s unavailable", name);
  *out = (F)fn;
  return S2V_OK;
}

extern "C" {

int s2v_comm_unique_id(void *out, size_t len) {
  if (len < sizeof(ncclUniqueId)) return fail(S2V_EINVAL, "unique id buffer too small");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(S2V_ECOMM, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out, &id, sizeof(id));
  return S2V_OK;
}

int s2v_comm_init(const void *unique_id, int world, int rank, void **comm) {
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, world, id, rank);
  if (r != ncclSuccess) return fail(S2V_ECOMM, "ncclCommInitRank: %s", ncclGetErrorString(r));
  *comm = c;
  return S2V_OK;
}

int s2v_comm_destroy(void *comm) {
  if (comm) ncclCommDestroy((ncclComm_t)comm);
  return S2V_OK;
}

int s2v_comm_allgather(void *comm, const void *send, void *recv, size_t bytes, void *stream) {
  ncclResult_t r =
      ncclAllGather(send, recv, bytes, ncclUint8, (ncclComm_t)comm, as_stream(stream));
  if (r != ncclSuccess) return fail(S2V_ECOMM, "ncclAllGather: %s", ncclGetErrorString(r));
  return S2V_OK;
}

// Grouped in-place all-gathers of `nslots` equal chunks: slot b gathers
// `bytes` from every rank into recv + b*slot_stride (rank r at r*bytes).
int s2v_comm_allgather_slots(void *comm, void *recv, size_t bytes, size_t slot_stride,
                             int nslots, int rank, void *stream) {
  ncclGroupStart();
  for (int b = 0; b < nslots; b++) {
    char *base = (char *)recv + (size_t)b * slot_stride;
    ncclResult_t r = ncclAllGather(base + (size_t)rank * bytes, base, bytes, ncclUint8,
                                   (ncclComm_t)comm, as_stream(stream));
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return fail(S2V_ECOMM, "ncclAllGather: %s", ncclGetErrorString(r));
    }
  }
  ncclResult_t r = ncclGroupEnd();
  if (r != ncclSuccess) return fail(S2V_ECOMM, "ncclGroupEnd: %s", ncclGetErrorString(r));
  return S2V_OK;
}

// ---- CUDA IPC + stream memory operations: the peer-memory transport ------
// Ranks that are processes (torchrun) map each other's halo buffers with
// cudaIpc* and order producer/consumer with flags written and waited on by
// the streams themselves (cuStreamWriteValue32 / cuStreamWaitValue32, reached
// through cudaGetDriverEntryPoint so libs2v needs no link-time libcuda).  The
// round kernel then pushes every output row straight into every peer's
// buffer (s2v_embed_round_peers): the halo exchange is fused into the kernel.
int s2v_ipc_export(const void *ptr, void *handle_out, uint64_t *offset_out) {
  static PFN_addr_range range = nullptr;
  if (!range) {
    int rc = driver_fn("cuMemGetAddressRange", &range);
    if (rc) return rc;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return fail(S2V_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  S2V_CUDA_CHECK(cudaIpcGetMemHandle(&h, (void *)base));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (uint64_t)((CUdeviceptr)ptr - base);
  return S2V_OK;
}

int s2v_ipc_import(const void *handle, void **base_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  S2V_CUDA_CHECK(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return S2V_OK;
}

int s2v_ipc_close(void *base) {
  S2V_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  return S2V_OK;
}

int s2v_stream_write_u32(void *addr, uint32_t value, void *stream) {
  static PFN_write32 w = nullptr;
  if (!w) {
    int rc = driver_fn("cuStreamWriteValue32", &w);
    if (rc) return rc;
  }
  if (w((CUstream)stream, (CUdeviceptr)addr, value, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    return fail(S2V_ECOMM, "cuStreamWriteValue32 failed");
  return S2V_OK;
}

int s2v_stream_wait_u32(void *addr, uint32_t value, void *stream) {
  static PFN_wait32 w = nullptr;
  if (!w) {
    int rc = driver_fn("cuStreamWaitValue32", &w);
    if (rc) return rc;
  }
  if (w((CUstream)stream, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    return fail(S2V_ECOMM, "cuStreamWaitValue32 failed");
  return S2V_OK;
}

// Plain async copy (device<->device across peers, or host<->device), used by
// the in-process thread-group transport (collective._LocalDeviceComm).
int s2v_memcpy_async(void *dst, const void *src, size_t bytes, void *stream) {
  S2V_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  return S2V_OK;
}

int s2v_sum_ranks_typed(int kind, int P, int64_t n, const void *gathered, void *out,
                        void *stream) {
  if (n <= 0) return S2V_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 1024);
  cudaStream_t st = as_stream(stream);
  if (kind == 0)
    sum_ranks_typed_kernel<int64_t><<<grid, 256, 0, st>>>(P, n, (const int64_t *)gathered,
                                                          (int64_t *)out);
  else if (kind == 1)
    sum_ranks_typed_kernel<double><<<grid, 256, 0, st>>>(P, n, (const double *)gathered,
                                                         (double *)out);
  else if (kind == 2)
    sum_ranks_typed_kernel<float><<<grid, 256, 0, st>>>(P, n, (const float *)gathered,
                                                        (float *)out);
  else
    return fail(S2V_EINVAL, "sum_ranks: unknown kind %d", kind);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_enable_peer_access(int peer_device) {
  int cur = 0;
  S2V_CUDA_CHECK(cudaGetDevice(&cur));
  if (peer_device == cur) return S2V_OK;
  int can = 0;
  S2V_CUDA_CHECK(cudaDeviceCanAccessPeer(&can, cur, peer_device));
  if (!can) return fail(S2V_ECOMM, "device %d cannot access peer device %d", cur, peer_device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return S2V_OK;
  }
  S2V_CUDA_CHECK(e);
  return S2V_OK;
}

// Rank-ordered all-reduce over NCCL: all-gather every rank's count elements
// into scratch [P][count], then the ascending-rank sum (sum_ranks) into buf.
int s2v_comm_allreduce_ordered(void *comm, void *buf, size_t count, int kind, void *scratch,
                               void *stream) {
  int P = 0, rank = 0;
  ncclCommCount((ncclComm_t)comm, &P);
  ncclCommUserRank((ncclComm_t)comm, &rank);
  const size_t bytes = count * (kind == 2 ? 4 : 8);
  ncclResult_t r = ncclAllGather(buf, scratch, bytes, ncclUint8, (ncclComm_t)comm,
                                 as_stream(stream));
  if (r != ncclSuccess) return fail(S2V_ECOMM, "ncclAllGather: %s", ncclGetErrorString(r));
  return s2v_sum_ranks_typed(kind, P, (int64_t)count, scratch, buf, stream);
}

int s2v_comm_allreduce(void *comm, void *buf, size_t count, int kind, void *stream) {
  ncclDataType_t t = kind == 0 ? ncclInt64 : (kind == 1 ? ncclFloat64 : ncclFloat32);
  ncclResult_t r = ncclAllReduce(buf, buf, count, t, ncclSum, (ncclComm_t)comm,
                                 as_stream(stream));
  if (r != ncclSuccess) return fail(S2V_ECOMM, "ncclAllReduce: %s", ncclGetErrorString(r));
  return S2V_OK;
}

}  // extern "C"
