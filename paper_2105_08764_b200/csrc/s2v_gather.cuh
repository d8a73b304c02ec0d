// Gather helpers shared by the forward round and the backward spmm_t
// (K = 64 fp32): one half-warp per row, lane l holds the float4 m[4l..4l+3];
// neighbour ids fetched 16 at a time (one per lane) and broadcast with
// shuffles, rows loaded in batches of 8 with an L2 evict_last policy for hub
// rows (low physical ids) and evict_first for the rest, added in ascending id.
#pragma once
#include "s2v_common.cuh"

namespace s2v {

__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ float4 ldg_f4_pol(const float *ptr, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(ptr), "l"(pol));
  return v;
}

__device__ __forceinline__ void stg_f4_pol(float *ptr, const float4 &v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

__device__ __forceinline__ uint32_t ldg_u32_pol(const uint32_t *ptr, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}

// 4-byte global -> shared copy without a register round trip
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ void add4(float4 &a, const float4 &b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}

// Neighbour id -> source row.  TABLE = false: the neighbour's own row of
// h_in.  TABLE = true (round 2 at P = 1): h_in is the 1-row-per-degree table
// of round-1 outputs and the source row is the neighbour's residual degree
// (an alive neighbour is never in S, so its round-1 row is table[rdeg]).
// sol_of (compact CSR of an active list): an entry built alive has died
// since iff its neighbour entered S.
template <bool TABLE>
__device__ __forceinline__ uint32_t source_row(uint32_t c, const int32_t *__restrict__ deg_of,
                                               const uint8_t *__restrict__ sol_of) {
  if (c & S2V_DEAD) return c;
  if (sol_of && sol_of[c]) return S2V_DEAD;
  if (!TABLE) return c;
  return (uint32_t)__ldg(deg_of + c);
}

// Sequential alive-neighbour sum of one row by one half-warp (lanes `sub`
// 0..15 of mask `hmask`), float4 per lane.
// PF: prefetch the second half of each 16-neighbour group into L2 while the
// first half's rows are in flight (spmm_t: 4.22 -> 3.84 ms per B = 2 launch;
// the forward round, at its 64-register budget, does not gain from it)
template <bool TABLE = false, bool PF = false>
__device__ __forceinline__ float4 gather_row64(int64_t e, const int64_t e1,
                                               const uint32_t *__restrict__ cols,
                                               const float *__restrict__ h_in, int sub,
                                               unsigned hmask, int hbase, uint32_t hot_rows,
                                               uint64_t pol_hot, uint64_t pol_cold,
                                               const int32_t *__restrict__ deg_of = nullptr,
                                               const uint8_t *__restrict__ sol_of = nullptr,
                                               uint32_t hot_lo = 0) {
  // hot rows: [hot_lo, hot_lo + hot_rows) -- the low ids (BA hubs) of the
  // row's own slot of a block-diagonal batch
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (; e < e1; e += 16) {
    const int cnt = (e1 - e) < 16 ? (int)(e1 - e) : 16;
    const uint32_t mine = source_row<TABLE>(
        sub < cnt ? ldg_u32_pol(cols + e + sub, pol_cold) : S2V_DEAD, deg_of, sol_of);
#pragma unroll
    for (int half = 0; half < 2; half++) {
      if (half * 8 >= cnt) break;
      uint32_t c[8];
#pragma unroll
      for (int q = 0; q < 8; q++) c[q] = __shfl_sync(hmask, mine, hbase + half * 8 + q);
      float4 v[8];
#pragma unroll
      for (int q = 0; q < 8; q++) {
        if (c[q] & S2V_DEAD) {
          v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          const float *src = h_in + (int64_t)c[q] * 64 + sub * 4;
          v[q] = ldg_f4_pol(src, c[q] - hot_lo < hot_rows ? pol_hot : pol_cold);
        }
      }
      if (PF && half == 0 && cnt > 8) {
        // the second half's rows into L2 while these 8 are in flight (no
        // registers held): lane l prefetches the line of row 8 + (l & 7)
        // holding its half of the 256-byte row
        const uint32_t cn = __shfl_sync(hmask, mine, hbase + 8 + (sub & 7));
        if (!(cn & S2V_DEAD) && !TABLE)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(h_in + (int64_t)cn * 64 + (sub >> 3) * 32));
      }
#pragma unroll
      for (int q = 0; q < 8; q++)
        if (!(c[q] & S2V_DEAD)) add4(acc, v[q]);
    }
  }
  return acc;
}


// Sequential alive-neighbour sum of one row by an 8-lane group (lanes l8 =
// 0..7 of mask qmask / base qbase): lane l8 holds the float4s l8 and l8 + 8
// of the 64-float row (a0, a1); neighbour ids 8 at a time (one per lane),
// rows 4 at a time (8 float4 per lane in flight), added in ascending order --
// the same sums, bit for bit, as gather_row64.  Four rows per warp instead of
// one: a tile's 32 rows are all in flight at once.
template <bool TABLE = false>
__device__ __forceinline__ void gather_row64_g8(const int64_t e0, const int64_t e1,
                                                const uint32_t *__restrict__ cols,
                                                const float *__restrict__ h_in, int l8,
                                                unsigned qmask, int qbase, uint32_t hot_rows,
                                                uint64_t pol_hot, uint64_t pol_cold,
                                                const int32_t *__restrict__ deg_of,
                                                const uint8_t *__restrict__ sol_of,
                                                uint32_t hot_lo, float4 &a0, float4 &a1,
                                                int pf = 0) {
  a0 = make_float4(0.f, 0.f, 0.f, 0.f);
  a1 = a0;
  const int cnt = (int)(e1 - e0);
  auto col_of = [&](int e) {
    return e + l8 < cnt ? ldg_u32_pol(cols + e0 + e + l8, pol_cold) : S2V_DEAD;
  };
  // TABLE: a neighbour's table row needs its id, then its degree -- two
  // dependent trips to L2 before the (L1-resident) table rows.  Pipelined:
  // the ids two groups ahead and the degrees one group ahead are in flight
  // while this group's table rows are added (round 2: 1585 -> 1545 us cold).
  // Neighbour rows of h: the ids one group ahead (spmm_t 3.76 -> 3.65 ms per
  // B = 2 launch; the forward round is unchanged at 2.22 ms).
  uint32_t id_next = 0, col_next2 = 0;
  if (TABLE) {
    id_next = source_row<TABLE>(col_of(0), deg_of, sol_of);
    col_next2 = col_of(8);
  } else {
    id_next = col_of(0);
    if (pf & 2) col_next2 = col_of(8);
  }
  for (int e8 = 0; e8 < cnt; e8 += 8) {
    uint32_t id;
    if (TABLE) {
      id = id_next;
      id_next = source_row<TABLE>(col_next2, deg_of, sol_of);
      col_next2 = col_of(e8 + 16);
    } else if (pf & 2) {  // ids two groups ahead: the next group's are here
      id = source_row<TABLE>(id_next, deg_of, sol_of);
      id_next = col_next2;
      col_next2 = col_of(e8 + 16);
    } else {
      id = source_row<TABLE>(id_next, deg_of, sol_of);
      id_next = col_of(e8 + 8);
    }
    // pf bit 0: rows 4..7 toward L2 while 0..3 load (bit 2: first group
    // only); bit 1: the next group's 8 rows toward L2 (its ids are already
    // in id_next), so 16 rows per group are in flight without registers
    if ((pf & 1) && (!(pf & 4) || e8 == 0) && l8 >= 4 && !(id & S2V_DEAD)) {
      const float *src = h_in + (int64_t)id * 64;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 32));
    }
    if (!TABLE && (pf & 2) && !(id_next & S2V_DEAD)) {
      const float *src = h_in + (int64_t)id_next * 64;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 32));
    }
#pragma unroll
    for (int g = 0; g < 2; g++) {  // neighbours e8 + 4g .. + 3
      if (e8 + 4 * g >= cnt) break;
      uint32_t c[4];
#pragma unroll
      for (int q = 0; q < 4; q++) c[q] = __shfl_sync(qmask, id, qbase + 4 * g + q);
      float4 v0[4], v1[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (c[q] & S2V_DEAD) {
          v0[q] = v1[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          const float *src = h_in + (int64_t)c[q] * 64;
          const uint64_t pol = c[q] - hot_lo < hot_rows ? pol_hot : pol_cold;
          v0[q] = ldg_f4_pol(src + 4 * l8, pol);
          v1[q] = ldg_f4_pol(src + 32 + 4 * l8, pol);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; q++)
        if (!(c[q] & S2V_DEAD)) {
          add4(a0, v0[q]);
          add4(a1, v1[q]);
        }
    }
  }
}

// gather_row64_g8's L2 prefetch mode (bits of pf): 1 = rows 4..7 of each
// 8-id group while rows 0..3 load (round 2.306 -> 2.288 ms at cfg3, spmm_t
// 3.84 -> 3.76 ms per B = 2 launch); 2 (default) = the next group's 8 rows,
// ids two groups ahead (cfg3 step 9.30-9.34 -> 9.10-9.27 ms, two boxes;
// prefetching two groups ahead measured 10.76 ms: the prefetched lines are
// evicted before use); 4 = bit 0 on the first group only; 0 = off.
// S2V_G8_PF overrides it for A/B runs
inline int g8_prefetch() {
  static const int v = [] {
    const char *e = getenv("S2V_G8_PF");
    return e ? atoi(e) : 2;
  }();
  return v;
}

// CTA-cooperative sequential gather of one hub row (degree > S2V_HUB_DEGREE):
// half-warps 1..15 stage 8 neighbour rows each (kHubBatch = 120 per batch)
// into a double-buffered shared ring while half-warp 0 adds the previous
// batch in ascending order, so one chain gets 120 rows in flight instead of
// 8.  Removed entries are staged as +0 (value-equal to skipping them, as the
// reference adds 0 * h).  The result is valid in half-warp 0.
constexpr int kHubLoaders = 15;
constexpr int kHubBatch = kHubLoaders * 8;

template <bool TABLE>
__device__ __forceinline__ void hub_stage(int64_t e_batch, const int64_t e1,
                                          const uint32_t *__restrict__ cols,
                                          const float *__restrict__ src, float *buf /*[120][64]*/,
                                          int hw, int sub, unsigned hmask, int hbase,
                                          uint32_t hot_rows, uint64_t pol_hot, uint64_t pol_cold,
                                          const int32_t *__restrict__ deg_of,
                                          const uint8_t *__restrict__ sol_of) {
  if (hw == 0) return;
  const int64_t base = e_batch + (int64_t)(hw - 1) * 8;
  const uint32_t mine = source_row<TABLE>(
      (sub < 8 && base + sub < e1) ? ldg_u32_pol(cols + base + sub, pol_cold) : S2V_DEAD,
      deg_of, sol_of);
  float4 v[8];
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const uint32_t c = __shfl_sync(hmask, mine, hbase + q);
    v[q] = (c & S2V_DEAD) ? make_float4(0.f, 0.f, 0.f, 0.f)
                          : ldg_f4_pol(src + (int64_t)c * 64 + sub * 4,
                                       c < hot_rows ? pol_hot : pol_cold);
  }
#pragma unroll
  for (int q = 0; q < 8; q++)
    *reinterpret_cast<float4 *>(buf + ((hw - 1) * 8 + q) * 64 + sub * 4) = v[q];
}

template <bool TABLE = false>
__device__ __forceinline__ float4 hub_gather_row64(const int64_t e0, const int64_t e1,
                                                   const uint32_t *__restrict__ cols,
                                                   const float *__restrict__ src,
                                                   float *ring /*[2][120][64]*/, uint32_t hot_rows,
                                                   uint64_t pol_hot, uint64_t pol_cold,
                                                   const int32_t *__restrict__ deg_of = nullptr,
                                                   const uint8_t *__restrict__ sol_of = nullptr) {
  const int tid = threadIdx.x, hw = tid >> 4, sub = tid & 15;
  const unsigned hmask = (tid & 16) ? 0xFFFF0000u : 0x0000FFFFu;
  const int hbase = tid & 16;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t nb = (e1 - e0 + kHubBatch - 1) / kHubBatch;
  if (nb > 0)
    hub_stage<TABLE>(e0, e1, cols, src, ring, hw, sub, hmask, hbase, hot_rows, pol_hot, pol_cold,
                     deg_of, sol_of);
  __syncthreads();
  for (int64_t b = 0; b < nb; b++) {
    if (b + 1 < nb)
      hub_stage<TABLE>(e0 + (b + 1) * kHubBatch, e1, cols, src,
                       ring + ((b + 1) & 1) * kHubBatch * 64, hw, sub, hmask, hbase, hot_rows,
                       pol_hot, pol_cold, deg_of, sol_of);
    if (hw == 0) {
      const float *cur = ring + (b & 1) * kHubBatch * 64;
      const int64_t left = e1 - e0 - b * kHubBatch;
      const int cnt = left < kHubBatch ? (int)left : kHubBatch;
      for (int q = 0; q < cnt; q++) add4(acc, *reinterpret_cast<const float4 *>(cur + q * 64 + sub * 4));
    }
    __syncthreads();
  }
  return acc;
}

}  // namespace s2v
