// common.cuh -- shared device helpers for the B200 RNN-Descent builder.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rnndg {

// ---------------------------------------------------------------- entries
//
// One list entry is a single u64 "key":
//     bits 63..32  float bits of the cached squared distance (always >= +0,
//                  so unsigned order == float order)
//     bits 31..1   neighbour id (ids < 2^31)
//     bit  0       fresh flag ("new" in NN-Descent terms, graph.hpp:11-18)
// Ascending key order is exactly `nearer` (dist, then id; graph.hpp:21-23):
// ids are unique within a list, so the flag bit never decides an order.
// 8 bytes per entry instead of the reference's 12-byte NeighborEntry.
constexpr uint64_t kTomb = ~0ull;  // deleted slot marker (sorts last)
// "distance pending": a redirected entry whose exact distance is not computed
// at redirect time (gram.cu computes it while streaming the row at the next
// scan of the list; materialize_pending() everywhere else).  The bits are a
// NaN above +inf, so pending entries sort after every real one, by id.
constexpr uint32_t kPendBits = 0x7F800001u;
constexpr uint32_t kNone = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t make_key(float dist, uint32_t id,
                                                     uint32_t fresh) {
  uint32_t db;
#ifdef __CUDA_ARCH__
  db = __float_as_uint(dist);
#else
  __builtin_memcpy(&db, &dist, 4);
#endif
  return (uint64_t(db) << 32) | (uint64_t(id) << 1) | uint64_t(fresh & 1u);
}
__host__ __device__ __forceinline__ uint64_t pending_key(uint32_t id) {
  return (uint64_t(kPendBits) << 32) | (uint64_t(id) << 1) | 1ull;
}
__host__ __device__ __forceinline__ bool key_pending(uint64_t k) {
  return uint32_t(k >> 32) == kPendBits;
}
__host__ __device__ __forceinline__ uint32_t key_id(uint64_t k) {
  return uint32_t(k) >> 1;
}
__host__ __device__ __forceinline__ uint32_t key_fresh(uint64_t k) {
  return uint32_t(k) & 1u;
}
__host__ __device__ __forceinline__ uint32_t key_dbits(uint64_t k) {
  return uint32_t(k >> 32);
}
__device__ __forceinline__ float key_dist(uint64_t k) {
  return __uint_as_float(uint32_t(k >> 32));
}

// ------------------------------------------------------------ SplitMix64
// rng.hpp:13-35; bounded() is the 128-bit multiply-shift (rng.hpp:26-28).
struct SplitMix64 {
  uint64_t s;
  __host__ __device__ explicit SplitMix64(uint64_t seed) : s(seed) {}
  __host__ __device__ __forceinline__ uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  __device__ __forceinline__ uint64_t bounded(uint64_t bound) {
    return __umul64hi(next(), bound);
  }
};

// mix_seed, rng.hpp:39-42
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed,
                                                     uint64_t stream) {
  SplitMix64 g(seed ^ (0xD1B54A32D192ED03ULL * (stream + 1)));
  return g.next();
}

// ------------------------------------------------------------ exact L2
//
// metric.hpp:15-24 fixes the summation order: four fp32 partial sums over
// interleaved lanes (element i -> lane i % 4 of the 4-aligned prefix), each
// `s += (a-b)*(a-b)` as a separate multiply and add (no FMA), combined
// ((s0+s1)+(s2+s3)), then the tail left to right.  The _rn intrinsics pin
// every operation to IEEE round-to-nearest with no contraction, independent
// of -fmad; denormals are preserved (no -ftz).  Result is bit-identical to
// rnnd::l2_sq on every input.
__device__ __forceinline__ void l2_step4(float4 x, float4 y, float& s0,
                                         float& s1, float& s2, float& s3) {
  float t0 = __fsub_rn(x.x, y.x);
  float t1 = __fsub_rn(x.y, y.y);
  float t2 = __fsub_rn(x.z, y.z);
  float t3 = __fsub_rn(x.w, y.w);
  s0 = __fadd_rn(s0, __fmul_rn(t0, t0));
  s1 = __fadd_rn(s1, __fmul_rn(t1, t1));
  s2 = __fadd_rn(s2, __fmul_rn(t2, t2));
  s3 = __fadd_rn(s3, __fmul_rn(t3, t3));
}

__device__ __forceinline__ float l2_finish(float s0, float s1, float s2,
                                           float s3) {
  return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}

// `a` may point anywhere (global or shared: plain loads); `b` must be a
// global row (read-only path).  `kVec4` when both rows are 16-byte aligned
// and the row length is a multiple of 4 (true for every row when d % 4 == 0).
template <bool kVec4>
__device__ __forceinline__ float l2_exact(const float* __restrict__ a,
                                          const float* __restrict__ b,
                                          uint32_t d) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  uint32_t i = 0;
  if (kVec4) {
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    const uint32_t d4 = d >> 2;
#pragma unroll 4
    for (uint32_t q = 0; q < d4; ++q) l2_step4(a4[q], __ldg(b4 + q), s0, s1, s2, s3);
    i = d4 << 2;
  } else {
    for (; i + 4 <= d; i += 4) {
      float4 x = make_float4(a[i], a[i + 1], a[i + 2], a[i + 3]);
      float4 y = make_float4(__ldg(b + i), __ldg(b + i + 1), __ldg(b + i + 2), __ldg(b + i + 3));
      l2_step4(x, y, s0, s1, s2, s3);
    }
  }
  float sum = l2_finish(s0, s1, s2, s3);
  for (; i < d; ++i) {
    float t = __fsub_rn(a[i], __ldg(b + i));
    sum = __fadd_rn(sum, __fmul_rn(t, t));
  }
  return sum;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

}  // namespace rnndg
