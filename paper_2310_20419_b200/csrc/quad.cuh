// quad.cuh -- exact L2 of one pair by a quad of lanes on the chain-blocked
// store copy (k_chain_layout in scan.cu): lane k of the quad sums fp32 chain
// k (metric.hpp:15-24), so the result is bit-identical to rnnd::l2_sq.
// Shared by the push walks (scan.cu) and the Gram-filtered walk (gram.cu).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace rnndg {

// 256-bit read-only loads of chain-blocked blocks.  ld256: the streamed
// row of a pair (the candidate), L1::no_allocate so it does not evict the
// rows that are re-read; ld256w: the row shared by many pairs (a provisional
// kept entry), normal L1 allocation.  C3 1M: 2.25 s -> 2.18 s per build
// (both rows no_allocate 2.20 s, w rows evict_last 2.18 s).  Short rows
// (C2 d = 128, C4 d = 96) stay in L1 across rounds: there the streamed row
// is allocated too (kNA = false; C4 1M 0.97 -> 0.93 s, C2 0.79 -> 0.77 s).
template <bool kNA = true>
__device__ __forceinline__ void ld256(const float* p, float (&r)[8]) {
  if (kNA)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                   "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                   "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld256w(const float* p, float (&r)[8]) {
  asm volatile("ld.global.nc.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                 "=f"(r[6]), "=f"(r[7])
               : "l"(p));
}

// the same loads at a compile-time byte offset from the pointer (the address
// operand takes [reg + imm], so an unrolled loop bumps one register per row
// instead of computing an address per load)
template <bool kNA, int kOff>
__device__ __forceinline__ void ld256o(const float* p, float (&r)[8]) {
  if (kNA)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8+%9];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                   "=f"(r[6]), "=f"(r[7])
                 : "l"(p), "n"(kOff));
  else
    asm volatile("ld.global.nc.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8+%9];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                   "=f"(r[6]), "=f"(r[7])
                 : "l"(p), "n"(kOff));
}

__device__ __forceinline__ void prefetch_row_l2(const float* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void chain_step(const float (&va)[8], const float (&vb)[8], float& s) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float t = __fsub_rn(va[i], vb[i]);
    s = __fadd_rn(s, __fmul_rn(t, t));
  }
}

// A quad computes d(a, b) on chain-blocked rows, lane k = chain k; the exact
// total is returned in the quad's chain-0 lane.  All 32 lanes must call.
// `a` is the streamed row, `b` the row shared across pairs (l2 is
// bit-symmetric, so the order of the operands never changes a result).
// Loads run two blocks ahead of the arithmetic.
template <bool kNA = true>
__device__ __forceinline__ float quad_l2(const float* __restrict__ a, const float* __restrict__ b,
                                         uint32_t k, uint32_t nblk, uint32_t ntail) {
  float s = 0.f;
  const float* pa = a + 8 * k;
  const float* pb = b + 8 * k;
  float a0[8], b0[8], a1[8], b1[8];
  uint32_t blk = 0;
  if (nblk >= 2) {
    ld256<kNA>(pa, a0);
    ld256w(pb, b0);
    ld256<kNA>(pa + 32, a1);
    ld256w(pb + 32, b1);
    const float* qa = pa + 64;
    const float* qb = pb + 64;
    for (blk = 2; blk + 1 < nblk; blk += 2, qa += 64, qb += 64) {
      chain_step(a0, b0, s);
      ld256o<kNA, 0>(qa, a0);
      ld256o<false, 0>(qb, b0);
      chain_step(a1, b1, s);
      ld256o<kNA, 128>(qa, a1);
      ld256o<false, 128>(qb, b1);
    }
    chain_step(a0, b0, s);
    chain_step(a1, b1, s);
  }
  for (; blk < nblk; ++blk) {
    ld256<kNA>(pa + 32 * blk, a0);
    ld256w(pb + 32 * blk, b0);
    chain_step(a0, b0, s);
  }
  const float s_next = __shfl_down_sync(0xffffffffu, s, 1);
  const float pair = __fadd_rn(s, s_next);                    // s0+s1 | s2+s3
  const float pair2 = __shfl_down_sync(0xffffffffu, pair, 2);
  float sum = __fadd_rn(pair, pair2);                         // chain-0 lane
  if (ntail && k == 0) {
    const float* ta = a + 32 * nblk;
    const float* tb = b + 32 * nblk;
    for (uint32_t t = 0; t < ntail; ++t) {
      const float df = __fsub_rn(__ldg(ta + t), __ldg(tb + t));
      sum = __fadd_rn(sum, __fmul_rn(df, df));
    }
  }
  return sum;
}

struct Row {
  const float* xp;
  uint32_t stride, nblk, ntail;
  __device__ const float* operator()(uint64_t key) const {
    return xp + uint64_t(key_id(key)) * stride;
  }
};

}  // namespace rnndg
