// NCCL collectives behind the C ABI.  Replaces the reference's in-process
// thread rendezvous (pkg/src/graphrl/collective.py:100-146) for the device
// data path: the per-round halo all-gather of embeddings (in place, one call
// per batch slot inside an NCCL group), and small all-reduces of integer
// selection info / fp64 gradient packs.  Host-side bookkeeping collectives
// stay in Python (torch.distributed / thread rendezvous).
#include <nccl.h>

#include "s2v_common.cuh"

using namespace s2v;

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

// Plain async copy (device<->device across peers, or host<->device), used by
// the in-process thread-group transport (collective._LocalDeviceComm).
int s2v_memcpy_async(void *dst, const void *src, size_t bytes, void *stream) {
  S2V_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  return S2V_OK;
}

int s2v_comm_allreduce(void *comm, void *buf, size_t count, int kind, void *stream) {
  ncclDataType_t t = kind == 0 ? ncclInt64 : (kind == 1 ? ncclFloat64 : ncclFloat32);
  ncclResult_t r = ncclAllReduce(buf, buf, count, t, ncclSum, (ncclComm_t)comm,
                                 as_stream(stream));
  if (r != ncclSuccess) return fail(S2V_ECOMM, "ncclAllReduce: %s", ncclGetErrorString(r));
  return S2V_OK;
}

}  // extern "C"
