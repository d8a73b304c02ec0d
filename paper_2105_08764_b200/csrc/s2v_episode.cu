// Device-resident selection loop pieces: the exact u1
// product, the adaptive d rule with top-d picks, and the per-evaluation
// trace -- so a whole policy evaluation + group apply runs without a host
// round trip and can be captured in a CUDA graph.
//
// Replaces (paths relative to /root/reference):
//   u1 = g @ theta5.T                      pkg/src/graphrl/policy.py:201
//   SelectionSchedule.d_for / select_top_d pkg/src/graphrl/inference.py:54-73,116-124
//   active = residual_counts > 0           pkg/src/graphrl/inference.py:147
#include <algorithm>

#include "s2v_common.cuh"

namespace s2v {

// u1[b][k] = sum_p theta5[k][p] g[b][p] in numpy/OpenBLAS (SkylakeX) order:
//  B == 1 : sgemv -- two 4-lane FMA accumulators over p blocks of 4
//           (block parity selects the accumulator), then (a0 + a1) per lane
//           and ((l0 + l1) + (l2 + l3));  K % 8 == 0, K >= 16
//  B >= 32: sgemm -- one sequential FMA chain per output
// (identified against numpy 2.3 / OpenBLAS 0.3.30; pinned by the GPU tests,
// whose oracle computes u1 with numpy itself).
__global__ void u1_kernel(int B, int K, const float *__restrict__ g,
                          const float *__restrict__ t5, float *__restrict__ u1) {
  const int b = blockIdx.x;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float *gb = g + (int64_t)b * K;
    const float *row = t5 + (int64_t)k * K;
    float out;
    if (B == 1) {
      float a[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      for (int p = 0; p < K; p++) {
        const int u = (p >> 2) & 1, l = p & 3;
        a[u][l] = __fmaf_rn(row[p], gb[p], a[u][l]);
      }
      float v[4];
      for (int l = 0; l < 4; l++) v[l] = __fadd_rn(a[0][l], a[1][l]);
      out = __fadd_rn(__fadd_rn(v[0], v[1]), __fadd_rn(v[2], v[3]));
    } else {
      float acc = 0.f;
      for (int p = 0; p < K; p++) acc = __fmaf_rn(row[p], gb[p], acc);
      out = acc;
    }
    u1[(int64_t)b * K + k] = out;
  }
}

// Adaptive d and picks per slot (inference.py:116-124): d = first schedule
// entry with count > frac * N (fp64 product, as Python), else fallback;
// d = min(d, count); picks = the first d keys (descending score, lowest id on
// ties).  keys: [B][dmax][2] {orderable score, ~node}; out: picks [B][dmax].
struct Schedule {
  double frac[8];
  int d[8];
  int n;
  int fallback;
};

__global__ void select_kernel(int B, int dmax, int64_t N, Schedule sched,
                              const int64_t *__restrict__ counts,
                              const uint64_t *__restrict__ keys, const uint8_t *__restrict__ active,
                              int64_t *__restrict__ picks, int32_t *__restrict__ evaluated,
                              int32_t *__restrict__ error) {
  // one block: an active slot with no candidates raises the reference's
  // InvalidActionError("empty candidate set") BEFORE any apply
  // (inference.py:119-122), so then no slot gets a pick this evaluation
  __shared__ int s_err;
  if (threadIdx.x == 0) s_err = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x)
    if (active[b] && counts[b] == 0) s_err = 1;
  __syncthreads();
  const bool err = s_err != 0;
  if (err && threadIdx.x == 0) *error = 1;  // sticky: the host zeroes it per call / chunk
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    int d = 0;
    if (active[b] && !err) {
      const int64_t c = counts[b];
      d = sched.fallback;
      for (int i = 0; i < sched.n; i++)
        if ((double)c > sched.frac[i] * (double)N) {
          d = sched.d[i];
          break;
        }
      if ((int64_t)d > c) d = (int)c;
    }
    evaluated[b] = active[b] && !err ? 1 : 0;
    for (int j = 0; j < dmax; j++)
      picks[(int64_t)b * dmax + j] =
          j < d ? (int64_t)(~keys[((int64_t)b * dmax + j) * 2 + 1]) : (int64_t)-1;
  }
}

// After the group apply: append this evaluation to the trace and refresh
// active = residual > 0 (P = 1: local residual is global).
__global__ void trace_kernel(int B, int dmax, const int64_t *__restrict__ picks,
                             const uint8_t *__restrict__ applied,
                             const int32_t *__restrict__ evaluated,
                             const int64_t *__restrict__ residual, uint8_t *__restrict__ active,
                             int64_t *__restrict__ trace_picks, uint8_t *__restrict__ trace_applied,
                             int32_t *__restrict__ trace_eval) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    for (int j = 0; j < dmax; j++) {
      trace_picks[(int64_t)b * dmax + j] = picks[(int64_t)b * dmax + j];
      trace_applied[(int64_t)b * dmax + j] = applied[(int64_t)b * dmax + j];
    }
    trace_eval[b] = evaluated[b];
    active[b] = residual[b] > 0 ? 1 : 0;
  }
}

// P > 1 device loop: the ranks' (counts, top-d keys) gathered as
// [P][B*(1 + 2d)] int64 -> the global counts and top-d keys, same layout,
// identically on every rank (merge_rank_keys' order: key, then ~node).
__global__ void merge_rank_keys_kernel(int P, int B, int d, const int64_t *__restrict__ g,
                                       int64_t *__restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int64_t len = (int64_t)B * (1 + 2 * d);
  int64_t cnt = 0;
  Key top[8];
  for (int q = 0; q < 8; q++) top[q] = null_key();
  for (int r = 0; r < P; r++) {
    const int64_t *src = g + r * len;
    cnt += src[b];
    const Key *k = reinterpret_cast<const Key *>(src + B) + (int64_t)b * d;
    for (int j = 0; j < d; j++) {
      const Key x = k[j];
      if (!key_gt(x, top[d - 1])) continue;
      int pos = d - 1;
      while (pos > 0 && key_gt(x, top[pos - 1])) {
        top[pos] = top[pos - 1];
        pos--;
      }
      top[pos] = x;
    }
  }
  out[b] = cnt;
  Key *o = reinterpret_cast<Key *>(out + B) + (int64_t)b * d;
  for (int j = 0; j < d; j++) o[j] = top[j];
}

// out[i] = sum over ranks of g[r][i], ascending rank order
__global__ void sum_ranks_kernel(int P, int64_t n, const int64_t *__restrict__ g,
                                 int64_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = 0;
    for (int r = 0; r < P; r++) s += g[r * n + i];
    out[i] = s;
  }
}

__global__ void sub_i64_kernel(int64_t *__restrict__ a, const int64_t *__restrict__ b, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] -= b[i];
}

}  // namespace s2v

using namespace s2v;

extern "C" {

int s2v_u1(s2v_dtype dt, int B, int K, const void *g, const void *theta5, void *u1,
           void *stream) {
  if (dt != S2V_F32) return fail(S2V_EINVAL, "device u1 is fp32 only");
  if (!((B == 1 && K % 8 == 0 && K >= 16) || B >= 32))
    return fail(S2V_EINVAL, "no exact device order for u1 with B=%d K=%d", B, K);
  u1_kernel<<<B, 64, 0, as_stream(stream)>>>(B, K, (const float *)g, (const float *)theta5,
                                             (float *)u1);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_u1_exact(int B, int K) { return (B == 1 && K % 8 == 0 && K >= 16) || B >= 32; }

int s2v_select(int B, int dmax, int64_t N, const double *fracs, const int *ds, int nthr,
               int fallback, const int64_t *counts, const uint64_t *keys, const uint8_t *active,
               int64_t *picks, int32_t *evaluated, int32_t *error, void *stream) {
  if (nthr > 8) return fail(S2V_EINVAL, "at most 8 schedule thresholds");
  Schedule sc;
  sc.n = nthr;
  sc.fallback = fallback;
  for (int i = 0; i < nthr; i++) {
    sc.frac[i] = fracs[i];
    sc.d[i] = ds[i];
  }
  select_kernel<<<1, 128, 0, as_stream(stream)>>>(B, dmax, N, sc, counts, keys, active, picks,
                                                  evaluated, error);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_trace(int B, int dmax, const int64_t *picks, const uint8_t *applied,
              const int32_t *evaluated, const int64_t *residual, uint8_t *active,
              int64_t *trace_picks, uint8_t *trace_applied, int32_t *trace_eval, void *stream) {
  trace_kernel<<<1, 128, 0, as_stream(stream)>>>(B, dmax, picks, applied, evaluated, residual,
                                                 active, trace_picks, trace_applied, trace_eval);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_eval_chain(const s2v_shard *sh, const s2v_eval_plan *p, int c, void *stream) {
  if (sh->world != 1 || sh->active) return fail(S2V_EINVAL, "eval chain: P = 1, no active list");
  const int K = p->K, B = sh->batch, d = p->dmax;
  if (d < 1 || d > 8 || p->L < 1) return fail(S2V_EINVAL, "eval chain: bad plan");
  const float *th = p->theta;
  const float *t4 = th + 2 * K + K * K, *t5 = t4 + K * K, *t6 = t5 + K * K, *t7 = t6 + K * K;
  int rc;
  // rounds (policy._forward_rounds, inference: ping-pong buffers)
  const float *h_prev = nullptr;
  for (int layer = 0; layer < p->L; layer++) {
    float *h_out = p->h[layer % 2];
    if (p->h1_table && layer == 0) continue;  // nothing reads h1 but round 2
    if (p->h1_table && layer == 1)
      rc = s2v_embed_round2_table(S2V_F32, sh, t4, p->table, K, p->max_deg, p->h1_table, nullptr,
                                  h_out, nullptr, 0, nullptr, stream);
    else
      rc = s2v_embed_round(S2V_F32, sh, t4, p->table, K, p->max_deg, h_prev, h_out, nullptr,
                           stream);
    if (rc) return rc;
    h_prev = h_out;
  }
  // global sum, u1, scores, top-d keys (policy._score)
  if ((rc = s2v_colsum(S2V_F32, sh, K, h_prev, p->g, p->colsum_ws, p->colsum_ws_bytes, stream)))
    return rc;
  if ((rc = s2v_u1(S2V_F32, B, K, p->g, t5, p->u1, stream))) return rc;
  if ((rc = s2v_score(S2V_F32, sh, K, h_prev, p->u1, t6, t7, nullptr, 0, p->scores,
                      p->block_keys, p->out, stream)))
    return rc;
  uint64_t *top = (uint64_t *)(p->out + B);
  if ((rc = s2v_topk_merge(sh, p->block_keys, d, top, stream))) return rc;
  // d rule + picks, group apply, trace (inference.DeviceEpisode._launch_one)
  if ((rc = s2v_select(B, d, sh->num_nodes, p->fracs, p->ds, p->nthr, p->fallback, p->out, top,
                       p->active, p->picks, p->evaluated, p->error, stream)))
    return rc;
  if ((rc = s2v_apply_phase1(sh, p->picks, d, p->info, 0, nullptr, stream))) return rc;
  if ((rc = s2v_apply_phase2(sh, p->picks, d, p->info, p->applied, p->removed, 1, stream)))
    return rc;
  return s2v_trace(B, d, p->picks, p->applied, p->evaluated, sh->residual, p->active,
                   p->t_picks + (int64_t)c * B * d, p->t_applied + (int64_t)c * B * d,
                   p->t_eval + (int64_t)c * B, stream);
}

int s2v_merge_rank_keys(int P, int B, int d, const int64_t *gathered, int64_t *out,
                        void *stream) {
  if (P < 1 || B < 1 || d < 1 || d > 8) return fail(S2V_EINVAL, "bad key merge args");
  merge_rank_keys_kernel<<<(B + 63) / 64, 64, 0, as_stream(stream)>>>(P, B, d, gathered, out);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_sum_ranks(int P, int64_t n, const int64_t *gathered, int64_t *out, void *stream) {
  if (n <= 0) return S2V_OK;
  sum_ranks_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, as_stream(stream)>>>(
      P, n, gathered, out);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

int s2v_sub_i64(int64_t *a, const int64_t *b, int n, void *stream) {
  if (n <= 0) return S2V_OK;
  sub_i64_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(a, b, n);
  S2V_LAUNCH_CHECK();
  return S2V_OK;
}

}  // extern "C"
