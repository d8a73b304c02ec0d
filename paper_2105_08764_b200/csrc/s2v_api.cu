// Handle-level C ABI: context, graph and state handles
// whose device memory the library owns, so a caller of the reference's API
// binds plain host arrays -- no torch, no device pointers -- and drives the
// hot path with one call per reference operation:
//
//   s2v_ctx_create / s2v_ctx_destroy      one per GPU (run_workers' rank)
//   s2v_graph_upload / s2v_graph_destroy  Graph.csr_arrays -> device shard
//                                          structure (state.py:89-105,115-122)
//   s2v_state_create / s2v_state_destroy  PartitionedState(graphs, part,
//                                          solutions)      (state.py:56-111)
//   s2v_embed                             embed_forward    (policy.py:144-185)
//   s2v_global_sum                        embed.sum + q_fwd all-reduce
//                                                           (policy.py:199-200)
//   s2v_score_topk                        q_forward + masked_scores + the
//                                          top-d of select_top_d
//                                          (policy.py:188-224, inference.py:61-73)
//   s2v_apply                             the group apply with the mid-group
//                                          skip rule (inference.py:125-146,
//                                          state.py:173-208)
//   s2v_loss_grad                         loss_and_gradients (policy.py:232-315)
//   s2v_adam_update                       adam_step        (policy.py:339-359)
//   s2v_copy_out                          the numpy views tests read (embed,
//                                          sol, cand, rdeg, residual, scores)
//
// Every entry point orchestrates the same kernels, in the same order, as the
// Python mirror (paper_2105_08764_b200/policy.py, state.py), so results are
// the same bits.
//
// Node-sharded P > 1 (one context per rank, every s2v_* call collective, as
// run_workers' threads call the reference's API, collective.py:143-195):
// each rank owns the block partition_rows(N, P)[rank] of every graph
// (state.py:36-53); after every round the ranks all-gather their rows of h
// (the halo exchange of policy.py:168), and the global sums -- dg, the
// gradient pack, the group-apply info -- are rank-ordered all-reduces
// (collective.py:100-117).  Two transports: NCCL (s2v_ctx_create with an
// ncclUniqueId; one process or thread per GPU) and an in-process group
// (s2v_group_create + s2v_ctx_create_in_group; thread ranks on any devices,
// including one shared GPU) that copies peers' chunks on the streams and
// orders them with CUDA events plus a host rendezvous.
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "s2v_common.cuh"

// in-process rank group: host rendezvous + per-rank buffer pointers and
// stream events published for the peers
struct s2v_group {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<void *> ptr;
  std::vector<cudaEvent_t> ready, done;
  explicit s2v_group(int w) : world(w), ptr(w), ready(w), done(w) {}
  // false after a timeout (a rank stopped calling collectives): the group
  // stays broken, every later collective fails (collective.py:134-139)
  bool barrier() {
    std::unique_lock<std::mutex> l(mu);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(l, std::chrono::seconds(300), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

namespace {
using namespace s2v;
// the halo and all-reduce transport of a context at P > 1
struct Transport {
  virtual ~Transport() {}
  // in place: slot b's chunk of rank r at buf + b*stride + r*chunk
  virtual int allgather_slots(void *buf, size_t chunk, size_t stride, int nslots,
                              cudaStream_t s) = 0;
};

struct NcclTransport : Transport {
  void *comm = nullptr;
  int rank = 0;
  ~NcclTransport() override {
    if (comm) s2v_comm_destroy(comm);
  }
  int allgather_slots(void *buf, size_t chunk, size_t stride, int nslots,
                      cudaStream_t s) override {
    return s2v_comm_allgather_slots(comm, buf, chunk, stride, nslots, rank, s);
  }
};

struct LocalTransport : Transport {
  s2v_group *g = nullptr;
  int rank = 0;
  cudaEvent_t ready = nullptr, done = nullptr;
  ~LocalTransport() override {
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
  }
  int allgather_slots(void *buf, size_t chunk, size_t stride, int nslots,
                      cudaStream_t s) override {
    // publish: this rank's chunks are complete once `ready` fires
    S2V_CUDA_CHECK(cudaEventRecord(ready, s));
    g->ptr[rank] = buf;
    g->ready[rank] = ready;
    if (!g->barrier()) return fail(S2V_ECOMM, "collective timed out (a rank stopped)");
    // pull every peer's chunks on this stream, after its producer
    for (int q = 0; q < g->world; q++) {
      if (q == rank) continue;
      S2V_CUDA_CHECK(cudaStreamWaitEvent(s, g->ready[q], 0));
      for (int b = 0; b < nslots; b++) {
        const size_t off = (size_t)b * stride + (size_t)q * chunk;
        S2V_CUDA_CHECK(cudaMemcpyAsync((char *)buf + off, (const char *)g->ptr[q] + off, chunk,
                                       cudaMemcpyDefault, s));
      }
    }
    // no rank reuses its buffer before every peer's pull of it is done
    S2V_CUDA_CHECK(cudaEventRecord(done, s));
    g->done[rank] = done;
    if (!g->barrier()) return fail(S2V_ECOMM, "collective timed out (a rank stopped)");
    for (int q = 0; q < g->world; q++)
      if (q != rank) S2V_CUDA_CHECK(cudaStreamWaitEvent(s, g->done[q], 0));
    if (!g->barrier()) return fail(S2V_ECOMM, "collective timed out (a rank stopped)");
    return S2V_OK;
  }
};
}  // namespace

struct s2v_ctx {
  int device = 0;
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  Transport *tr = nullptr;
  void *scratch = nullptr;  // all-reduce / key exchange staging, grow-only
  size_t scratch_bytes = 0;
  ~s2v_ctx() {
    delete tr;
    if (scratch) cudaFree(scratch);
  }
};

struct s2v_graph {
  int64_t n = 0, nnz = 0, n_hub = 0;
  int32_t max_deg = 0;          // over every node of the graph (the e12 table)
  int P = 1;                    // the context's partition of this graph
  int64_t row_start = 0, rows = 0, rows_max = 0;
  int64_t *row_ptr = nullptr, *col_ptr = nullptr, *col_ent = nullptr;
  int32_t *cols0 = nullptr, *col_row = nullptr, *order = nullptr;
};

namespace {

using namespace s2v;

// grow-only device buffer owned by a state
struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want) {
    if (want <= bytes && p) return S2V_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    S2V_CUDA_CHECK(cudaMalloc(&p, want ? want : 16));
    bytes = want ? want : 16;
    return S2V_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T *as() const {
    return reinterpret_cast<T *>(p);
  }
};

inline size_t dt_size(s2v_dtype dt) { return dt == S2V_F32 ? 4 : 8; }

inline int use_ctx(const s2v_ctx *ctx) {
  if (!ctx) return fail(S2V_EINVAL, "null context");
  S2V_CUDA_CHECK(cudaSetDevice(ctx->device));
  return S2V_OK;
}

__global__ void widen_i32_kernel(const int32_t *__restrict__ a, int64_t *__restrict__ b, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

int ctx_scratch(s2v_ctx *ctx, size_t want) {
  if (want <= ctx->scratch_bytes && ctx->scratch) return S2V_OK;
  if (ctx->scratch) {
    S2V_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    cudaFree(ctx->scratch);
  }
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  S2V_CUDA_CHECK(cudaMalloc(&ctx->scratch, want));
  ctx->scratch_bytes = want;
  return S2V_OK;
}

// in-place rank-ordered sum of count elements (kind 0 int64, 1 fp64, 2 fp32)
// over the context's ranks: every rank's vector into row [rank] of the
// scratch, all-gathered, then summed rank 0, 1, ... (collective.py:114-116)
int ctx_allreduce(s2v_ctx *ctx, void *buf, int64_t count, int kind) {
  if (ctx->world == 1 || count <= 0) return S2V_OK;
  const size_t nb = (size_t)count * (kind == 2 ? 4 : 8);
  int rc = ctx_scratch(ctx, nb * ctx->world);
  if (rc) return rc;
  cudaStream_t s = ctx->stream;
  S2V_CUDA_CHECK(cudaMemcpyAsync((char *)ctx->scratch + nb * ctx->rank, buf, nb,
                                 cudaMemcpyDeviceToDevice, s));
  if ((rc = ctx->tr->allgather_slots(ctx->scratch, nb, nb * ctx->world, 1, s))) return rc;
  return s2v_sum_ranks_typed(kind, ctx->world, count, ctx->scratch, buf, s);
}

// the block partition_rows(n, P)[rank] (state.py:36-53)
inline void partition_of(int64_t n, int P, int rank, int64_t *start, int64_t *rows) {
  const int64_t base = n / P, extra = n % P;
  *start = (int64_t)rank * base + std::min<int64_t>(rank, extra);
  *rows = base + (rank < extra ? 1 : 0);
}

}  // namespace

struct s2v_state {
  s2v_ctx *ctx = nullptr;
  int B = 0;
  int64_t n = 0;
  int64_t rows = 0, rows_max = 0;  // this rank's rows per slot; padded rows per rank
  int32_t max_deg = 0;
  s2v_shard sh{};
  DevBuf row_ptr, col_ptr, col_ent, cols, col_row, order, rdeg, sol, cand, residual;
  // workspaces
  DevBuf theta, table, h1t, h[2], colsum_ws, g, u1, scores, bkeys, out;
  DevBuf picks, info, applied, removed, err;
  DevBuf tape_h, tape_m, grad_h, dzsum, dm, p4, pp, head, dg, dact, t2c, t2tot, pack, act,
      targets;
  const void *h_last = nullptr;  // last embedding written by s2v_embed
  int hK = 0;
  s2v_dtype hdt = S2V_F32;
  bool have_scores = false;
  ~s2v_state() {
    for (DevBuf *b : {&row_ptr, &col_ptr, &col_ent, &cols, &col_row, &order, &rdeg, &sol, &cand,
                      &residual, &theta, &table, &h1t, &h[0], &h[1], &colsum_ws, &g, &u1,
                      &scores, &bkeys, &out, &picks, &info, &applied, &removed, &err, &tape_h,
                      &tape_m, &grad_h, &dzsum, &dm, &p4, &pp, &head, &dg, &dact, &t2c, &t2tot,
                      &pack, &act, &targets})
      b->release();
  }
};

namespace {

// theta1..theta7 packed as param_shapes(K) (policy.py:43-113): offsets in
// elements
struct ThetaOffsets {
  int64_t t1, t2, t3, t4, t5, t6, t7, total;
  explicit ThetaOffsets(int K) {
    const int64_t k = K, kk = k * k;
    t1 = 0;
    t2 = k;
    t3 = 2 * k;
    t4 = 2 * k + kk;
    t5 = 2 * k + 2 * kk;
    t6 = 2 * k + 3 * kk;
    t7 = 2 * k + 4 * kk;
    total = 4 * k + 4 * kk;
  }
};

int upload_theta(s2v_state *st, s2v_dtype dt, const void *theta, int K) {
  ThetaOffsets o(K);
  const size_t bytes = (size_t)o.total * dt_size(dt);
  int rc = st->theta.ensure(bytes);
  if (rc) return rc;
  S2V_CUDA_CHECK(cudaMemcpyAsync(st->theta.p, theta, bytes, cudaMemcpyHostToDevice,
                                 st->ctx->stream));
  return S2V_OK;
}

inline const char *th_ptr(const s2v_state *st, s2v_dtype dt, int64_t off) {
  return st->theta.as<const char>() + off * dt_size(dt);
}

// bytes of one embedding buffer in the gathered layout [B][P][rows_max][K]
// (= [B][N][K] at P = 1)
inline size_t full_bytes(const s2v_state *st, int K, size_t es) {
  return (size_t)st->B * st->ctx->world * st->rows_max * K * es;
}

// at P > 1: every rank's rows of h into every rank's buffer (policy.py:168)
int halo_gather(s2v_state *st, void *h, int K, size_t es) {
  s2v_ctx *c = st->ctx;
  if (c->world == 1) return S2V_OK;
  const size_t chunk = (size_t)st->rows_max * K * es;
  return c->tr->allgather_slots(h, chunk, chunk * c->world, st->B, c->stream);
}

// _forward_rounds (paper_2105_08764_b200/policy.py): e12 table, round 2
// from the per-degree h1 table (K = 64 fp32, L >= 2, P = 1), the rest as
// plain rounds, each followed at P > 1 by the halo all-gather.  tape: every
// layer's h into tape_h [L][full] and the neighbour sums of layers >= 1 into
// tape_m [L][B*rows*K]; round 1 then runs (the backward reads h1), as in the
// Python mirror.
int forward(s2v_state *st, s2v_dtype dt, int K, int L, bool tape) {
  cudaStream_t s = st->ctx->stream;
  const s2v_shard *sh = &st->sh;
  ThetaOffsets o(K);
  const size_t es = dt_size(dt);
  const size_t hbytes = full_bytes(st, K, es);
  const size_t mbytes = (size_t)st->B * st->rows * K * es;
  const int md = st->max_deg;
  int rc = st->table.ensure((size_t)(md + 2) * K * es);
  if (rc) return rc;
  rc = s2v_e12_table(dt, th_ptr(st, dt, o.t1), th_ptr(st, dt, o.t2), th_ptr(st, dt, o.t3), K, md,
                     st->table.p, s);
  if (rc) return rc;
  const bool deg_table = K == 64 && dt == S2V_F32 && L >= 2 && st->ctx->world == 1;
  if (deg_table) {
    if ((rc = st->h1t.ensure((size_t)(md + 2) * K * 4))) return rc;
    if ((rc = s2v_h1_table(dt, th_ptr(st, dt, o.t4), st->table.p, K, md, st->h1t.p, s)))
      return rc;
  }
  if (tape) {
    if ((rc = st->tape_h.ensure(hbytes * L)) ||
        (rc = st->tape_m.ensure(std::max<size_t>(mbytes, 16) * L)))
      return rc;
  } else if ((rc = st->h[0].ensure(hbytes)) || (rc = st->h[1].ensure(hbytes))) {
    return rc;
  }
  const size_t mstride = std::max<size_t>(mbytes, 16);
  const void *h_prev = nullptr;
  for (int layer = 0; layer < L; layer++) {
    void *h_out = tape ? st->tape_h.as<char>() + hbytes * layer : st->h[layer % 2].p;
    void *m_out = (tape && layer > 0) ? st->tape_m.as<char>() + mstride * layer : nullptr;
    if (deg_table && layer == 0 && !tape) continue;  // only round 2 reads h1: the table
    if (deg_table && layer == 1) {
      rc = s2v_embed_round2_table(dt, sh, th_ptr(st, dt, o.t4), st->table.p, K, md, st->h1t.p,
                                  nullptr, h_out, nullptr, 0, m_out, s);
    } else {
      rc = s2v_embed_round(dt, sh, th_ptr(st, dt, o.t4), st->table.p, K, md, h_prev, h_out,
                           m_out, s);
    }
    if (rc || (rc = halo_gather(st, h_out, K, es))) return rc;
    h_prev = h_out;
  }
  st->h_last = h_prev;
  st->hK = K;
  st->hdt = dt;
  return S2V_OK;
}

int colsum_of(s2v_state *st, const void *h, int K, s2v_dtype dt) {
  const size_t wsb = s2v_colsum_workspace(&st->sh, K, (int)dt_size(dt));
  int rc = st->colsum_ws.ensure(wsb);
  if (rc) return rc;
  if ((rc = st->g.ensure((size_t)st->B * K * dt_size(dt)))) return rc;
  return s2v_colsum(dt, &st->sh, K, h, st->g.p, st->colsum_ws.p, wsb, st->ctx->stream);
}

// block-diagonal assembly of one structure array over the batch
template <class T>
int assemble(s2v_state *st, DevBuf &dst, int64_t total, const std::vector<s2v_segment> &segs) {
  int rc = dst.ensure((size_t)std::max<int64_t>(total, 1) * sizeof(T));
  if (rc) return rc;
  int64_t longest = 0;
  for (const auto &sg : segs) longest = std::max(longest, sg.len);
  if (!longest) return S2V_OK;
  s2v_segment *d = nullptr;
  S2V_CUDA_CHECK(cudaMalloc(&d, sizeof(s2v_segment) * segs.size()));
  cudaMemcpy(d, segs.data(), sizeof(s2v_segment) * segs.size(), cudaMemcpyHostToDevice);
  rc = s2v_segment_copy((int)sizeof(T), d, (int)segs.size(), longest, dst.p, st->ctx->stream);
  cudaStreamSynchronize(st->ctx->stream);
  cudaFree(d);
  return rc;
}

}  // namespace

extern "C" {

static int new_ctx(int device, int rank, int world, s2v_ctx **out) {
  if (!out) return fail(S2V_EINVAL, "null output handle");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(S2V_EINVAL, "rank %d outside [0, %d)", rank, world);
  S2V_CUDA_CHECK(cudaSetDevice(device));
  s2v_ctx *c = new s2v_ctx();
  c->device = device;
  c->rank = rank;
  c->world = world;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(S2V_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
  }
  *out = c;
  return S2V_OK;
}

// world = 1: a single-rank context (nccl_id ignored).  world > 1: rank of a
// node-sharded group joined through NCCL (nccl_id: the ncclUniqueId bytes
// of s2v_comm_unique_id, shared by the caller; one rank per GPU).
int s2v_ctx_create(int device, int rank, int world, const void *nccl_id, s2v_ctx **out) {
  if (world > 1 && !nccl_id)
    return fail(S2V_EINVAL, "world > 1 needs an NCCL unique id (or s2v_ctx_create_in_group)");
  s2v_ctx *c = nullptr;
  int rc = new_ctx(device, rank, world, &c);
  if (rc) return rc;
  if (world > 1) {
    auto *t = new NcclTransport();
    t->rank = rank;
    c->tr = t;
    if ((rc = s2v_comm_init(nccl_id, world, rank, &t->comm))) {
      t->comm = nullptr;
      s2v_ctx_destroy(c);
      return rc;
    }
  }
  *out = c;
  return S2V_OK;
}

int s2v_group_create(int world, s2v_group **out) {
  if (!out || world < 1) return fail(S2V_EINVAL, "bad group arguments");
  *out = new s2v_group(world);
  return S2V_OK;
}

int s2v_group_destroy(s2v_group *g) {
  delete g;
  return S2V_OK;
}

// rank `rank` of an in-process group (one thread per rank, any devices)
int s2v_ctx_create_in_group(int device, int rank, s2v_group *group, s2v_ctx **out) {
  if (!group) return fail(S2V_EINVAL, "null group");
  s2v_ctx *c = nullptr;
  int rc = new_ctx(device, rank, group->world, &c);
  if (rc) return rc;
  if (group->world > 1) {
    auto *t = new LocalTransport();
    t->g = group;
    t->rank = rank;
    c->tr = t;
    if (cudaEventCreateWithFlags(&t->ready, cudaEventDisableTiming) ||
        cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming)) {
      s2v_ctx_destroy(c);
      return fail(S2V_ECUDA, "cudaEventCreate failed");
    }
    // peers' buffers on other GPUs: direct NVLink copies where possible
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    for (int d = 0; d < ndev; d++) {
      int ok = 0;
      if (d != device && cudaDeviceCanAccessPeer(&ok, device, d) == cudaSuccess && ok)
        cudaDeviceEnablePeerAccess(d, 0);
    }
    cudaGetLastError();  // (already-enabled peers are fine)
  }
  *out = c;
  return S2V_OK;
}

int s2v_ctx_destroy(s2v_ctx *ctx) {
  if (!ctx) return S2V_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return S2V_OK;
}

int s2v_ctx_sync(s2v_ctx *ctx) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  S2V_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return S2V_OK;
}

// row_ptr [n+1] / cols [row_ptr[n]]: the graph's symmetric CSR with
// ascending neighbour lists (Graph.csr_arrays), host memory.  At P > 1 every
// rank passes the whole graph and keeps its block of rows (state.py:89-105).
int s2v_graph_upload(s2v_ctx *ctx, int64_t n, const int64_t *row_ptr, const int32_t *cols,
                     s2v_graph **out) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!out || !row_ptr || n < 0) return fail(S2V_EINVAL, "bad graph arguments");
  if (row_ptr[0] != 0 || row_ptr[n] < 0 || (row_ptr[n] && !cols))
    return fail(S2V_EINVAL, "bad CSR row_ptr");
  const int P = ctx->world;
  if (P > n) return fail(S2V_EINVAL, "more workers (%d) than nodes (%lld)", P, (long long)n);
  int64_t start = 0, nrows = n;
  partition_of(n, P, ctx->rank, &start, &nrows);
  const int64_t lo = row_ptr[start], nnz = row_ptr[start + nrows] - lo;
  int32_t gmax = 0;  // the e12 table covers every node's degree
  for (int64_t u = 0; u < n; u++)
    gmax = std::max<int32_t>(gmax, (int32_t)(row_ptr[u + 1] - row_ptr[u]));
  s2v_graph *g = new s2v_graph();
  g->n = n;
  g->nnz = nnz;
  g->P = P;
  g->row_start = start;
  g->rows = nrows;
  g->rows_max = (n + P - 1) / P;
  cudaStream_t s = ctx->stream;
  std::vector<int64_t> rp_local;
  if (P > 1) {
    rp_local.resize(nrows + 1);
    for (int64_t i = 0; i <= nrows; i++) rp_local[i] = row_ptr[start + i] - lo;
  }
  int32_t *nbr = nullptr;
  auto bail = [&](int code) {
    if (nbr) cudaFree(nbr);
    s2v_graph_destroy(g);
    return code;
  };
  if (cudaMalloc(&g->row_ptr, 8 * (nrows + 1)) || cudaMalloc(&g->col_ptr, 8 * (n + 1)) ||
      cudaMalloc(&g->cols0, 4 * std::max<int64_t>(nnz, 1)) ||
      cudaMalloc(&g->col_ent, 8 * std::max<int64_t>(nnz, 1)) ||
      cudaMalloc(&g->col_row, 4 * std::max<int64_t>(nnz, 1)) ||
      cudaMalloc(&g->order, 4 * std::max<int64_t>(nrows, 1)) ||
      cudaMalloc(&nbr, 4 * std::max<int64_t>(nnz, 1)))
    return bail(fail(S2V_ECUDA, "graph upload: out of device memory"));
  if (cudaMemcpyAsync(g->row_ptr, P > 1 ? rp_local.data() : row_ptr, 8 * (nrows + 1),
                      cudaMemcpyHostToDevice, s) ||
      (nnz && cudaMemcpyAsync(nbr, cols + lo, 4 * nnz, cudaMemcpyHostToDevice, s)))
    return bail(fail(S2V_ECUDA, "graph upload: copy failed"));
  int32_t md = 0;
  rc = s2v_shard_structure(n, P, g->rows_max, nrows, g->row_ptr, nbr, nnz, g->cols0, g->col_ptr,
                           g->col_ent, g->col_row, g->order, &g->n_hub, &md, s);
  if (rc) return bail(rc);
  S2V_CUDA_CHECK(cudaStreamSynchronize(s));  // (rp_local is a host temporary)
  g->max_deg = gmax;
  cudaFree(nbr);
  *out = g;
  return S2V_OK;
}

int s2v_graph_destroy(s2v_graph *g) {
  if (!g) return S2V_OK;
  for (void *p : {(void *)g->row_ptr, (void *)g->col_ptr, (void *)g->cols0, (void *)g->col_ent,
                  (void *)g->col_row, (void *)g->order})
    if (p) cudaFree(p);
  delete g;
  return S2V_OK;
}

// graphs[B] with equal node counts; sol: host [B][N] 0/1 bytes over every
// node (NULL = empty S); at P > 1 each rank keeps its rows
int s2v_state_create(s2v_ctx *ctx, s2v_graph *const *graphs, int B, const uint8_t *sol,
                     s2v_state **out) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!out || !graphs || B < 1) return fail(S2V_EINVAL, "need at least one graph");
  const int64_t n = graphs[0]->n;
  for (int b = 0; b < B; b++)
    if (!graphs[b] || graphs[b]->n != n)
      return fail(S2V_EINVAL, "all graphs in a batch must have the same node count");
  for (int b = 0; b < B; b++)
    if (graphs[b]->P != ctx->world)
      return fail(S2V_EINVAL, "graph uploaded under a different rank count");
  const int P = ctx->world;
  const int64_t rows = graphs[0]->rows, rows_max = graphs[0]->rows_max;
  s2v_state *st = new s2v_state();
  st->ctx = ctx;
  st->B = B;
  st->n = n;
  st->rows = rows;
  st->rows_max = rows_max;
  std::vector<int64_t> e(B + 1, 0);
  int64_t n_hub = 0;
  for (int b = 0; b < B; b++) {
    e[b + 1] = e[b] + graphs[b]->nnz;
    st->max_deg = std::max(st->max_deg, graphs[b]->max_deg);
    n_hub += graphs[b]->n_hub;
  }
  const int64_t nnz = e[B];
  std::vector<s2v_segment> rp, cp, cl, ce, cr, od;
  int64_t hub_off = 0, rest_off = n_hub;
  // block-diagonal over slots: local rows b*rows.., global columns b*N..,
  // physical neighbour rows b*P*rows_max..
  const int64_t slot_phys = (int64_t)P * rows_max;
  for (int b = 0; b < B; b++) {
    const s2v_graph *g = graphs[b];
    rp.push_back({g->row_ptr, b * rows, rows + (b == B - 1 ? 1 : 0), e[b]});
    cp.push_back({g->col_ptr, b * n, n + (b == B - 1 ? 1 : 0), e[b]});
    cl.push_back({g->cols0, e[b], g->nnz, b * slot_phys});
    ce.push_back({g->col_ent, e[b], g->nnz, e[b]});
    cr.push_back({g->col_row, e[b], g->nnz, b * rows});
    // hub rows of every slot first, then the remaining rows of every slot
    od.push_back({g->order, hub_off, g->n_hub, b * rows});
    hub_off += g->n_hub;
  }
  for (int b = 0; b < B; b++) {
    const s2v_graph *g = graphs[b];
    od.push_back({g->order + g->n_hub, rest_off, rows - g->n_hub, b * rows});
    rest_off += rows - g->n_hub;
  }
  if ((rc = assemble<int64_t>(st, st->row_ptr, B * rows + 1, rp)) ||
      (rc = assemble<int64_t>(st, st->col_ptr, B * n + 1, cp)) ||
      (rc = assemble<int32_t>(st, st->cols, nnz, cl)) ||
      (rc = assemble<int64_t>(st, st->col_ent, nnz, ce)) ||
      (rc = assemble<int32_t>(st, st->col_row, nnz, cr)) ||
      (rc = assemble<int32_t>(st, st->order, B * rows, od)) ||
      (rc = st->rdeg.ensure(4 * std::max<int64_t>(B * rows, 1))) ||
      (rc = st->sol.ensure(std::max<int64_t>(B * rows, 1))) ||
      (rc = st->cand.ensure(std::max<int64_t>(B * rows, 1))) ||
      (rc = st->residual.ensure(8 * B))) {
    delete st;
    return rc;
  }
  s2v_shard &sh = st->sh;
  sh.num_nodes = n;
  sh.batch = B;
  sh.world = P;
  sh.rank = ctx->rank;
  sh.row_start = graphs[0]->row_start;
  sh.num_rows = rows;
  sh.rows_max = rows_max;
  sh.nnz = nnz;
  sh.row_ptr = st->row_ptr.as<int64_t>();
  sh.cols = st->cols.as<uint32_t>();
  sh.col_ptr = st->col_ptr.as<int64_t>();
  sh.col_ent = st->col_ent.as<int64_t>();
  sh.col_row = st->col_row.as<int32_t>();
  sh.rdeg = st->rdeg.as<int32_t>();
  sh.sol = st->sol.as<uint8_t>();
  sh.cand = st->cand.as<uint8_t>();
  sh.residual = st->residual.as<int64_t>();
  sh.order = st->order.as<int32_t>();
  sh.n_hub = n_hub;
  // S of every node in the physical layout [B][P][rows_max] (the neighbour
  // test of s2v_shard_init)
  const int64_t nphys = B * slot_phys;
  std::vector<uint8_t> sol_phys;
  if (sol && P > 1) {
    sol_phys.assign(nphys, 0);
    for (int b = 0; b < B; b++)
      for (int r = 0; r < P; r++) {
        int64_t s0 = 0, nr = 0;
        partition_of(n, P, r, &s0, &nr);
        memcpy(sol_phys.data() + b * slot_phys + r * rows_max, sol + b * n + s0, nr);
      }
  }
  uint8_t *sol_d = nullptr;
  if (cudaMalloc(&sol_d, std::max<int64_t>(nphys, 1)) ||
      (sol ? cudaMemcpy(sol_d, P > 1 ? sol_phys.data() : sol, nphys, cudaMemcpyHostToDevice)
           : cudaMemset(sol_d, 0, std::max<int64_t>(nphys, 1)))) {
    if (sol_d) cudaFree(sol_d);
    delete st;
    return fail(S2V_ECUDA, "state create: solution upload failed");
  }
  rc = s2v_shard_init(&sh, nullptr, sol_d, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(sol_d);
  if (rc) {
    delete st;
    return rc;
  }
  *out = st;
  return S2V_OK;
}

int s2v_state_destroy(s2v_state *st) {
  if (!st) return S2V_OK;
  cudaSetDevice(st->ctx->device);
  cudaStreamSynchronize(st->ctx->stream);
  delete st;
  return S2V_OK;
}

// the state's shard view, for the low-level entry points of this header
int s2v_state_shard(const s2v_state *st, s2v_shard *out) {
  if (!st || !out) return fail(S2V_EINVAL, "null argument");
  *out = st->sh;
  return S2V_OK;
}

// embed_forward: theta packed theta1..theta7 (host, dtype dt), L rounds;
// the final embedding stays in the state (s2v_copy_out(..., S2V_OUT_EMBED)).
int s2v_embed(s2v_ctx *ctx, s2v_state *st, s2v_dtype dt, const void *theta, int K, int L) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!st || !theta || K < 1 || L < 1) return fail(S2V_EINVAL, "bad embed arguments");
  if ((rc = upload_theta(st, dt, theta, K))) return rc;
  st->have_scores = false;
  return forward(st, dt, K, L, false);
}

// g[B][K] (host, dtype of the last s2v_embed): numpy's pairwise sum over the
// N nodes of every slot of the last embedding.
int s2v_global_sum(s2v_ctx *ctx, s2v_state *st, void *g_host) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!st || !st->h_last) return fail(S2V_EINVAL, "s2v_embed has not run on this state");
  if ((rc = colsum_of(st, st->h_last, st->hK, st->hdt))) return rc;
  S2V_CUDA_CHECK(cudaMemcpyAsync(g_host, st->g.p, (size_t)st->B * st->hK * dt_size(st->hdt),
                                 cudaMemcpyDeviceToHost, ctx->stream));
  S2V_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return S2V_OK;
}

// Scores of the last embedding (u1 = g theta5^T on the device; bit-exact
// with numpy's order for B = 1 and B >= 32, s2v_u1_exact), then the top-d
// (d <= 8) selection keys {orderable score, ~node} per slot, descending,
// ties to the lowest node (keys_out [B][d][2], host) and the candidate
// counts (ncand_out [B], host).  Solve semantics (mode 0).
int s2v_score_topk(s2v_ctx *ctx, s2v_state *st, int d, uint64_t *keys_out, int64_t *ncand_out) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!st || !st->h_last) return fail(S2V_EINVAL, "s2v_embed has not run on this state");
  if (d < 0 || d > 8) return fail(S2V_EINVAL, "d = %d outside [0, 8]", d);
  const int K = st->hK, B = st->B;
  const s2v_dtype dt = st->hdt;
  cudaStream_t s = ctx->stream;
  ThetaOffsets o(K);
  if ((rc = colsum_of(st, st->h_last, K, dt))) return rc;
  if ((rc = st->u1.ensure((size_t)B * K * dt_size(dt)))) return rc;
  if ((rc = s2v_u1(dt, B, K, st->g.p, th_ptr(st, dt, o.t5), st->u1.p, s))) return rc;
  const int nblk = s2v_score_blocks(&st->sh);
  const int P = ctx->world;
  // (P > 1: the rank exchange merges d >= 1 keys; d = 0 reads the counts)
  const int dx = P > 1 ? std::max(d, 1) : d;
  const size_t klen = (size_t)B * (1 + 2 * dx);
  if ((rc = st->scores.ensure((size_t)B * st->rows * dt_size(dt))) ||
      (rc = st->bkeys.ensure((size_t)B * nblk * 8 * 16)) ||
      (rc = st->out.ensure((size_t)B * (1 + 8 * 2) * 8 * (P > 1 ? 2 : 1))))
    return rc;
  if ((rc = s2v_score(dt, &st->sh, K, st->h_last, st->u1.p, th_ptr(st, dt, o.t6),
                      th_ptr(st, dt, o.t7), nullptr, 0, st->scores.p, st->bkeys.as<uint64_t>(),
                      st->out.as<int64_t>(), s)))
    return rc;
  if (dx > 0 && (rc = s2v_topk_merge(&st->sh, st->bkeys.as<uint64_t>(), dx,
                                      reinterpret_cast<uint64_t *>(st->out.as<int64_t>() + B), s)))
    return rc;
  const int64_t *res = st->out.as<int64_t>();
  if (P > 1) {  // every rank's counts and top-d keys, merged (inference.py:111-118)
    const size_t kb = klen * 8;
    if ((rc = ctx_scratch(ctx, kb * P))) return rc;
    S2V_CUDA_CHECK(cudaMemcpyAsync((char *)ctx->scratch + kb * ctx->rank, st->out.p, kb,
                                   cudaMemcpyDeviceToDevice, s));
    if ((rc = ctx->tr->allgather_slots(ctx->scratch, kb, kb * P, 1, s))) return rc;
    int64_t *merged = st->out.as<int64_t>() + (size_t)B * (1 + 8 * 2);
    if ((rc = s2v_merge_rank_keys(P, B, dx, (const int64_t *)ctx->scratch, merged, s))) return rc;
    res = merged;
  }
  st->have_scores = true;
  std::vector<int64_t> host(klen);
  S2V_CUDA_CHECK(cudaMemcpyAsync(host.data(), res, host.size() * 8, cudaMemcpyDeviceToHost, s));
  S2V_CUDA_CHECK(cudaStreamSynchronize(s));
  if (ncand_out) memcpy(ncand_out, host.data(), 8 * B);
  if (keys_out && d) memcpy(keys_out, host.data() + B, 16 * (size_t)B * d);
  return S2V_OK;
}

// One group of picks per slot (host [B][d], -1 padded, d <= 64): the
// group's first pick is applied unconditionally (it must be a candidate:
// S2V_EACTION "already in the solution" / "not a candidate" before anything
// is applied), later picks only while still candidates.  applied [B][d]
// (host, may be NULL), residual [B] alive local entries after (host, may be
// NULL).
int s2v_apply(s2v_ctx *ctx, s2v_state *st, const int64_t *picks, int d, uint8_t *applied,
              int64_t *residual) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!st || !picks || d < 1 || d > 64) return fail(S2V_EINVAL, "bad apply arguments");
  const int B = st->B;
  cudaStream_t s = ctx->stream;
  for (int b = 0; b < B; b++)
    for (int j = 0; j < d; j++) {
      const int64_t v = picks[(size_t)b * d + j];
      if (v < -1 || v >= st->n) return fail(S2V_EACTION, "node %lld out of range", (long long)v);
    }
  if ((rc = st->picks.ensure(8 * (size_t)B * d)) || (rc = st->info.ensure(16 * (size_t)B * d)) ||
      (rc = st->applied.ensure((size_t)B * d)) || (rc = st->removed.ensure(8 * B)) ||
      (rc = st->err.ensure(16 * (size_t)B)))
    return rc;
  S2V_CUDA_CHECK(cudaMemcpyAsync(st->picks.p, picks, 8 * (size_t)B * d, cudaMemcpyHostToDevice, s));
  if ((rc = s2v_apply_phase1(&st->sh, st->picks.as<int64_t>(), d, st->info.as<int64_t>(), 1,
                             st->err.as<int32_t>(), s)))
    return rc;
  std::vector<int64_t> err(B);
  // the first pick's owner validates it; at P > 1 every rank learns the
  // verdict (int64 sum: only the owner's code is non-zero)
  int64_t *err64 = reinterpret_cast<int64_t *>(st->err.as<char>() + 8 * (size_t)B);
  widen_i32_kernel<<<(B + 127) / 128, 128, 0, s>>>(st->err.as<int32_t>(), err64, B);
  S2V_LAUNCH_CHECK();
  if ((rc = ctx_allreduce(ctx, err64, B, 0))) return rc;
  S2V_CUDA_CHECK(cudaMemcpyAsync(err.data(), err64, 8 * B, cudaMemcpyDeviceToHost, s));
  S2V_CUDA_CHECK(cudaStreamSynchronize(s));
  for (int b = 0; b < B; b++) {
    if (err[b] == 1)
      return fail(S2V_EACTION, "node %lld is already in the solution",
                  (long long)picks[(size_t)b * d]);
    if (err[b] == 2)
      return fail(S2V_EACTION, "node %lld is not a candidate", (long long)picks[(size_t)b * d]);
  }
  // the later picks' skip rule reads every rank's info (state.py:195-208)
  if (d > 1 && (rc = ctx_allreduce(ctx, st->info.p, 2 * (int64_t)B * d, 0))) return rc;
  if ((rc = s2v_apply_phase2(&st->sh, st->picks.as<int64_t>(), d, st->info.as<int64_t>(),
                             st->applied.as<uint8_t>(), st->removed.as<int64_t>(), 1, s)))
    return rc;
  st->h_last = nullptr;  // the embedding belongs to the previous state
  st->have_scores = false;
  if (applied)
    S2V_CUDA_CHECK(cudaMemcpyAsync(applied, st->applied.p, (size_t)B * d, cudaMemcpyDeviceToHost,
                                   s));
  if (residual)
    S2V_CUDA_CHECK(cudaMemcpyAsync(residual, st->residual.p, 8 * B, cudaMemcpyDeviceToHost, s));
  S2V_CUDA_CHECK(cudaStreamSynchronize(s));
  return S2V_OK;
}

// loss_and_gradients (policy.py:232-315): actions [B] (host int64), targets
// [B] (host, dtype dt), theta packed (host) -> grads packed like theta
// (host, dtype dt) and the mean squared error.
int s2v_loss_grad(s2v_ctx *ctx, s2v_state *st, s2v_dtype dt, const void *theta, int K, int L,
                  const int64_t *actions, const void *targets, void *grads, double *loss) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!st || !theta || !actions || !targets || K < 1 || L < 1)
    return fail(S2V_EINVAL, "bad loss_grad arguments");
  const int B = st->B;
  const int64_t n = st->n;
  for (int b = 0; b < B; b++) {
    if (actions[b] < 0 || actions[b] >= n)
      return fail(S2V_EINVAL, "action node index out of range");
    const double t = dt == S2V_F32 ? (double)((const float *)targets)[b]
                                   : ((const double *)targets)[b];
    if (!std::isfinite(t)) return fail(S2V_EINVAL, "targets must be finite");
  }
  cudaStream_t s = ctx->stream;
  const s2v_shard *sh = &st->sh;
  const size_t es = dt_size(dt);
  ThetaOffsets o(K);
  if ((rc = upload_theta(st, dt, theta, K))) return rc;
  if ((rc = forward(st, dt, K, L, true))) return rc;
  st->h_last = nullptr;  // the tape is not an s2v_embed result
  st->have_scores = false;
  const size_t hbytes = full_bytes(st, K, es);               // gathered layout
  const size_t lbytes = (size_t)B * st->rows * K * es;        // this rank's rows
  const size_t mstride = std::max<size_t>(lbytes, 16);
  auto H = [&](int l) { return st->tape_h.as<char>() + hbytes * l; };
  auto Mt = [&](int l) { return st->tape_m.as<char>() + mstride * l; };
  const int nblk = s2v_backward_blocks(sh);
  const int64_t head_len = 2 * (int64_t)K * K + 2 * K + 1, plen = 2 * (int64_t)K + K * K;
  const int64_t npack = o.total + 1;
  if ((rc = st->act.ensure(8 * B)) || (rc = st->targets.ensure(es * B)) ||
      (rc = st->head.ensure(8 * B * head_len)) || (rc = st->dg.ensure(es * B * K)) ||
      (rc = st->dact.ensure(es * B * K)) || (rc = st->grad_h.ensure(mstride)) ||
      (rc = st->dzsum.ensure(mstride)) || (rc = st->dm.ensure(hbytes)) ||
      (rc = st->p4.ensure(es * nblk * K * K)) || (rc = st->pp.ensure(es * nblk * plen)) ||
      (rc = st->t2tot.ensure(es * B * K)) || (rc = st->pack.ensure(8 * npack)))
    return rc;
  S2V_CUDA_CHECK(cudaMemcpyAsync(st->act.p, actions, 8 * B, cudaMemcpyHostToDevice, s));
  S2V_CUDA_CHECK(cudaMemcpyAsync(st->targets.p, targets, es * B, cudaMemcpyHostToDevice, s));
  // g of h_L, the Q head at the action nodes, dg broadcast to every row
  if ((rc = colsum_of(st, H(L - 1), K, dt))) return rc;
  if ((rc = s2v_head_backward(dt, sh, K, H(L - 1), st->g.p, st->act.as<int64_t>(), st->targets.p,
                              th_ptr(st, dt, o.t5), th_ptr(st, dt, o.t6), th_ptr(st, dt, o.t7),
                              st->head.as<double>(), st->dg.p, st->dact.p, s)))
    return rc;
  // q_bwd: the adjoint of g reaches every rank's rows (policy.py:262-268)
  if ((rc = ctx_allreduce(ctx, st->dg.p, (int64_t)B * K, dt == S2V_F32 ? 2 : 1))) return rc;
  if (ctx->world > 1)  // (rank padding rows of the gathered dm are never read)
    S2V_CUDA_CHECK(cudaMemsetAsync(st->dm.p, 0, hbytes, s));
  if ((rc = s2v_grad_h_init(dt, sh, K, st->dg.p, st->act.as<int64_t>(), st->dact.p,
                            st->grad_h.p, s)))
    return rc;
  for (int layer = L - 1; layer >= 0; layer--) {
    const bool last = layer == 0;
    if ((rc = s2v_layer_backward(dt, sh, K, th_ptr(st, dt, o.t4), st->grad_h.p, H(layer),
                                 layer > 0 ? Mt(layer) : nullptr, st->dzsum.p, st->p4.p,
                                 layer == L - 1 ? 1 : 0, last ? nullptr : st->dm.p, s)))
      return rc;
    if (last) break;
    // embed_bwd: every rank's rows of dm (policy.py:290-300)
    if ((rc = halo_gather(st, st->dm.p, K, es)) ||
        (rc = s2v_gather(dt, sh, K, st->dm.p, st->grad_h.p, s)))
      return rc;
  }
  const size_t t2b = s2v_theta2_terms_bytes(dt, sh, K);
  void *t2c = st->grad_h.p;  // free by now
  if (t2b > mstride) {
    if ((rc = st->t2c.ensure(t2b))) return rc;
    t2c = st->t2c.p;
  }
  double *pack = st->pack.as<double>();
  if ((rc = s2v_param_grads(dt, sh, K, th_ptr(st, dt, o.t2), th_ptr(st, dt, o.t3), st->dzsum.p,
                            st->pp.p, t2c, s)) ||
      (rc = s2v_reduce_partials(dt, st->pp.p, nblk, (int)plen, pack, s)) ||
      (rc = s2v_theta2_einsum(dt, sh, K, t2c, st->t2tot.p, pack + K, s)) ||
      (rc = s2v_reduce_partials(dt, st->p4.p, nblk, K * K, pack + plen, s)) ||
      (rc = s2v_reduce_partials(S2V_F64, st->head.p, B, (int)head_len, pack + plen + K * K, s)) ||
      // one packed fp64 gradient all-reduce (policy.py:311-315)
      (rc = ctx_allreduce(ctx, pack, npack, 1)))
    return rc;
  std::vector<double> host(npack);
  S2V_CUDA_CHECK(cudaMemcpyAsync(host.data(), pack, 8 * npack, cudaMemcpyDeviceToHost, s));
  S2V_CUDA_CHECK(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < o.total; i++) {
    if (dt == S2V_F32)
      ((float *)grads)[i] = (float)host[i];
    else
      ((double *)grads)[i] = host[i];
  }
  if (loss) *loss = host[o.total] / B;
  return S2V_OK;
}

// adam_step in place on host arrays of n elements (dtype dt); step = the
// new step count t >= 1.  A non-finite gradient rejects the step with
// S2V_ENONFINITE before anything is touched (policy.py:346-349).
int s2v_adam_update(s2v_ctx *ctx, s2v_dtype dt, void *params, const void *grads, void *m,
                    void *v, int64_t n, int step, double lr, double beta1, double beta2,
                    double eps) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (n < 0 || step < 1) return fail(S2V_EINVAL, "bad adam arguments");
  for (int64_t i = 0; i < n; i++) {
    const double gi = dt == S2V_F32 ? (double)((const float *)grads)[i]
                                    : ((const double *)grads)[i];
    if (!std::isfinite(gi)) return fail(S2V_ENONFINITE, "non-finite gradient; step rejected");
  }
  const size_t bytes = (size_t)n * dt_size(dt);
  char *d = nullptr;
  S2V_CUDA_CHECK(cudaMalloc(&d, 4 * std::max<size_t>(bytes, 16)));
  cudaStream_t s = ctx->stream;
  cudaMemcpyAsync(d, params, bytes, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d + bytes, grads, bytes, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d + 2 * bytes, m, bytes, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d + 3 * bytes, v, bytes, cudaMemcpyHostToDevice, s);
  rc = s2v_adam(dt, d, d + bytes, d + 2 * bytes, d + 3 * bytes, n, beta1, 1 - beta1, beta2,
                1 - beta2, eps, lr, 1.0 - std::pow(beta1, step), 1.0 - std::pow(beta2, step), s);
  if (!rc) {
    cudaMemcpyAsync(params, d, bytes, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(m, d + 2 * bytes, bytes, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(v, d + 3 * bytes, bytes, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = fail(S2V_ECUDA, "adam read-back failed");
  }
  cudaFree(d);
  return rc;
}

// Host copies of state arrays: S2V_OUT_EMBED [B][N][K] (last s2v_embed,
// node-major, every node), S2V_OUT_SOL / S2V_OUT_CAND [B][rows] uint8,
// S2V_OUT_RDEG [B][rows] int32, S2V_OUT_RESIDUAL [B] int64 (alive local
// entries), S2V_OUT_SCORES [B][rows] (last s2v_score_topk; -inf off the
// candidate set is applied by the caller as masked_scores does) -- rows =
// this rank's block (N at P = 1), as the reference's per-rank views.
int s2v_copy_out(s2v_ctx *ctx, const s2v_state *st, int what, void *host) {
  int rc = use_ctx(ctx);
  if (rc) return rc;
  if (!st || !host) return fail(S2V_EINVAL, "null argument");
  const int64_t bn = (int64_t)st->B * st->rows;
  const void *src = nullptr;
  size_t bytes = 0;
  switch (what) {
    case 0: {
      if (!st->h_last) return fail(S2V_EINVAL, "s2v_embed has not run on this state");
      // gathered rows [B][P][rows_max][K] -> node order [B][N][K]
      const size_t row = (size_t)st->hK * dt_size(st->hdt);
      const int P = ctx->world;
      for (int b = 0; b < st->B; b++)
        for (int r = 0; r < P; r++) {
          int64_t s0 = 0, nr = 0;
          partition_of(st->n, P, r, &s0, &nr);
          S2V_CUDA_CHECK(cudaMemcpyAsync(
              (char *)host + ((size_t)b * st->n + s0) * row,
              (const char *)st->h_last + ((size_t)b * P + r) * st->rows_max * row, nr * row,
              cudaMemcpyDeviceToHost, ctx->stream));
        }
      S2V_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      return S2V_OK;
    }
    case 1: src = st->sol.p; bytes = bn; break;
    case 2: src = st->cand.p; bytes = bn; break;
    case 3: src = st->rdeg.p; bytes = 4 * bn; break;
    case 4: src = st->residual.p; bytes = 8 * (size_t)st->B; break;
    case 5:
      if (!st->have_scores) return fail(S2V_EINVAL, "s2v_score_topk has not run on this state");
      src = st->scores.p;
      bytes = (size_t)bn * dt_size(st->hdt);
      break;
    default: return fail(S2V_EINVAL, "unknown copy_out selector %d", what);
  }
  S2V_CUDA_CHECK(cudaMemcpyAsync(host, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  S2V_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return S2V_OK;
}

}  // extern "C"
