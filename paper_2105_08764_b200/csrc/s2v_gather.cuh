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

__device__ __forceinline__ void add4(float4 &a, const float4 &b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}

// Sequential alive-neighbour sum of one row by one half-warp (lanes `sub`
// 0..15 of mask `hmask`), float4 per lane.
__device__ __forceinline__ float4 gather_row64(int64_t e, const int64_t e1,
                                               const uint32_t *__restrict__ cols,
                                               const float *__restrict__ h_in, int sub,
                                               unsigned hmask, int hbase, uint32_t hot_rows,
                                               uint64_t pol_hot, uint64_t pol_cold) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (; e < e1; e += 16) {
    const int cnt = (e1 - e) < 16 ? (int)(e1 - e) : 16;
    const uint32_t mine = sub < cnt ? ldg_u32_pol(cols + e + sub, pol_cold) : S2V_DEAD;
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
          v[q] = ldg_f4_pol(src, c[q] < hot_rows ? pol_hot : pol_cold);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; q++)
        if (!(c[q] & S2V_DEAD)) add4(acc, v[q]);
    }
  }
  return acc;
}


}  // namespace s2v
