// tma_pairs.cu -- feasibility microbenchmark for a smem-staged distance stage:
// per "round" a CTA bulk-copies (cp.async.bulk, TMA engine) the rows of M
// random candidates and D random provisional entries of a 1M x 960 store
// into shared memory (double-buffered: the next round's rows land while this
// round computes), then evaluates the M x D exact-L2 pairs from shared
// memory, a quad of lanes per pair (lane = fp32 chain), packed FP32 for the
// differences and squares.  Reports pair evaluations per SM-cycle, the
// figure the scan kernel (k_scan_spec) reaches at ~1/127.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tma_pairs tma_pairs.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

constexpr uint32_t kD = 960;            // dim
constexpr uint32_t kRowBytes = kD * 4;  // 3840
constexpr uint32_t kNblk = kD / 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <bool kPacked>
__device__ __forceinline__ void step8(const float4& a0, const float4& a1, const float4& b0,
                                      const float4& b1, float& s) {
  const float va[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
  const float vb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
  if (kPacked) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unsigned long long a, b, t, m;
      asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(va[2 * i]), "f"(va[2 * i + 1]));
      asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(vb[2 * i]), "f"(vb[2 * i + 1]));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(a), "l"(b));
      asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(m) : "l"(t));
      float m0, m1;
      asm("mov.b64 {%0,%1}, %2;" : "=f"(m0), "=f"(m1) : "l"(m));
      s = __fadd_rn(s, m0);
      s = __fadd_rn(s, m1);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float t = __fsub_rn(va[i], vb[i]);
      s = __fadd_rn(s, __fmul_rn(t, t));
    }
  }
}

// smem layout: 2 stages x (M + D) rows, 2 mbarriers
template <int W, int M, int D, bool kPacked>
__global__ void __launch_bounds__(32 * W) k_pairs(const float* __restrict__ x, uint32_t n,
                                                  const uint32_t* __restrict__ idx, uint32_t rounds,
                                                  float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int R = M + D;
  float* rows = reinterpret_cast<float*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * R * kRowBytes);
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t* my = idx + uint64_t(blockIdx.x) * rounds * R;
  auto issue = [&](uint32_t r) {
    const uint32_t st = r & 1;
    mbar_expect_tx(&bar[st], R * kRowBytes);
    for (int j = 0; j < R; ++j)
      bulk_g2s(rows + (st * R + j) * kD, x + uint64_t(my[r * R + j]) * kD, kRowBytes, &bar[st]);
  };
  if (tid == 0) issue(0);
  float acc = 0.f;
  for (uint32_t r = 0; r < rounds; ++r) {
    const uint32_t st = r & 1;
    // next round's rows into the other stage (its previous contents were
    // consumed before the trailing barrier of round r - 1)
    if (tid == 0 && r + 1 < rounds) issue(r + 1);
    mbar_wait(&bar[st], (r >> 1) & 1);
    const float* base = rows + st * R * kD;
    for (uint32_t p0 = 0; p0 < uint32_t(M * D); p0 += 8 * W) {
      const uint32_t p = p0 + 8 * wid + quad;
      if (p0 + 8 * wid >= uint32_t(M * D)) break;  // warp-uniform
      const uint32_t pp = p < uint32_t(M * D) ? p : p0 + 8 * wid;
      const float* a = base + (pp / D) * kD + 8 * chain;       // candidate
      const float* b = base + (M + pp % D) * kD + 8 * chain;   // provisional entry
      float s = 0.f;
#pragma unroll 2
      for (uint32_t blk = 0; blk < kNblk; ++blk) {
        const float4* pa = reinterpret_cast<const float4*>(a + 32 * blk);
        const float4* pb = reinterpret_cast<const float4*>(b + 32 * blk);
        step8<kPacked>(pa[0], pa[1], pb[0], pb[1], s);
      }
      const float s1 = __shfl_down_sync(0xffffffffu, s, 1);
      const float pr = __fadd_rn(s, s1);
      const float p2 = __shfl_down_sync(0xffffffffu, pr, 2);
      if (p < uint32_t(M * D) && chain == 0) acc += __fadd_rn(pr, p2);
    }
    __syncthreads();  // stage st consumed: it may be refilled (round r + 2)
  }
  if (acc == 1234.5f) out[blockIdx.x * blockDim.x + tid] = acc;
}

// lane per pair: row-major rows, slot j at j * (kRowBytes + 16) (the 16-byte
// skew spreads the slots over the banks); each lane accumulates the four
// chains of its pair as two packed pairs {s0,s1}, {s2,s3} -- the reference
// SSE loop (metric.hpp:47-65) one float4 at a time, fully packed.
constexpr uint32_t kSlot = kRowBytes + 16;
template <int W, int M, int D>
__global__ void __launch_bounds__(32 * W) k_lanes(const float* __restrict__ x, uint32_t n,
                                                  const uint32_t* __restrict__ idx, uint32_t rounds,
                                                  float* __restrict__ out, unsigned long long nz) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int R = M + D;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * R * kSlot);
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t* my = idx + uint64_t(blockIdx.x) * rounds * R;
  auto issue = [&](uint32_t r) {
    const uint32_t st = r & 1;
    mbar_expect_tx(&bar[st], R * kRowBytes);
    for (int j = 0; j < R; ++j)
      bulk_g2s(smem + (st * R + j) * kSlot, x + uint64_t(my[r * R + j]) * kD, kRowBytes, &bar[st]);
  };
  if (tid == 0) issue(0);
  float acc = 0.f;
  for (uint32_t r = 0; r < rounds; ++r) {
    const uint32_t st = r & 1;
    if (tid == 0 && r + 1 < rounds) issue(r + 1);
    mbar_wait(&bar[st], (r >> 1) & 1);
    const unsigned char* base = smem + st * R * kSlot;
    for (uint32_t p0 = 0; p0 < uint32_t(M * D); p0 += 32 * W) {
      const uint32_t p = p0 + tid;
      if (p0 + 32 * (tid >> 5) >= uint32_t(M * D)) break;  // warp-uniform
      const uint32_t pp = p < uint32_t(M * D) ? p : p0;
      const float4* a = reinterpret_cast<const float4*>(base + (pp / D) * kSlot);
      const float4* b = reinterpret_cast<const float4*>(base + (M + pp % D) * kSlot);
      unsigned long long s01 = 0, s23 = 0;
#pragma unroll 4
      for (uint32_t e = 0; e < kD / 4; ++e) {
        const float4 va = a[e], vb = b[e];
        unsigned long long a01, a23, b01, b23, t01, t23, m01, m23;
        asm("mov.b64 %0, {%1,%2};" : "=l"(a01) : "f"(va.x), "f"(va.y));
        asm("mov.b64 %0, {%1,%2};" : "=l"(a23) : "f"(va.z), "f"(va.w));
        asm("mov.b64 %0, {%1,%2};" : "=l"(b01) : "f"(vb.x), "f"(vb.y));
        asm("mov.b64 %0, {%1,%2};" : "=l"(b23) : "f"(vb.z), "f"(vb.w));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t01) : "l"(a01), "l"(b01));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t23) : "l"(a23), "l"(b23));
        asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m01) : "l"(t01), "l"(nz));
        asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m23) : "l"(t23), "l"(nz));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s01) : "l"(s01), "l"(m01));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s23) : "l"(s23), "l"(m23));
      }
      float s0, s1, s2, s3;
      asm("mov.b64 {%0,%1}, %2;" : "=f"(s0), "=f"(s1) : "l"(s01));
      asm("mov.b64 {%0,%1}, %2;" : "=f"(s2), "=f"(s3) : "l"(s23));
      if (p < uint32_t(M * D)) acc += __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
    }
    __syncthreads();
  }
  if (acc == 1234.5f) out[blockIdx.x * blockDim.x + tid] = acc;
}

template <int W, int M, int D>
void run_lanes(const float* x, uint32_t n, uint32_t* idx, uint32_t rounds, float* out, int sms,
               int clk_khz) {
  auto k = k_lanes<W, M, D>;
  const size_t smem = 2 * (M + D) * kSlot + 16;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * W, smem));
  const int grid = sms * per_sm;
  const unsigned long long nz = 0x8000000080000000ull;
  k<<<grid, 32 * W, smem>>>(x, n, idx, rounds, out, nz);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 32 * W, smem>>>(x, n, idx, rounds, out, nz);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double evals = double(grid) * rounds * M * D;
  const double cyc = ms * 1e-3 * clk_khz * 1e3;
  printf("lanes W=%d M=%2d D=%d ctas/SM=%d smem=%zu: %.2f ms, %.1f SM-cycles/eval\n", W, M, D,
         per_sm, smem, ms, cyc * sms / evals);
}

template <int W, int M, int D, bool kPacked>
void run(const float* x, uint32_t n, uint32_t* idx, uint32_t rounds, float* out, int sms, int clk_khz) {
  auto k = k_pairs<W, M, D, kPacked>;
  const size_t smem = 2 * (M + D) * kRowBytes + 16;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * W, smem));
  const int grid = sms * per_sm;
  k<<<grid, 32 * W, smem>>>(x, n, idx, rounds, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 32 * W, smem>>>(x, n, idx, rounds, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double evals = double(grid) * rounds * M * D;
  const double cyc = ms * 1e-3 * clk_khz * 1e3;
  const double bytes = double(grid) * rounds * (M + D) * kRowBytes;
  printf("W=%d M=%2d D=%d packed=%d ctas/SM=%d smem=%zu: %.2f ms, %.1f SM-cycles/eval, row fetch %.1f TB/s\n",
         W, M, D, int(kPacked), per_sm, smem, ms, cyc * sms / evals, bytes / (ms * 1e-3) / 1e12);
}

int main() {
  const uint32_t n = 1000000;
  int sms, clk;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  float* x;
  CK(cudaMalloc(&x, size_t(n) * kRowBytes));
  CK(cudaMemset(x, 0, size_t(n) * kRowBytes));
  const uint32_t rounds = 200;
  const size_t nidx = size_t(sms) * 4 * rounds * 40;
  std::vector<uint32_t> h(nidx);
  uint64_t s = 88172645463325252ull;
  for (auto& v : h) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    v = uint32_t(s % (getenv("SUB") ? uint32_t(atoi(getenv("SUB"))) : n));
  }
  uint32_t* idx;
  CK(cudaMalloc(&idx, nidx * 4));
  CK(cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
  float* out;
  CK(cudaMalloc(&out, 1 << 24));
  run_lanes<1, 11, 3>(x, n, idx, rounds, out, sms, clk);
  run_lanes<2, 11, 3>(x, n, idx, rounds, out, sms, clk);
  run_lanes<2, 21, 3>(x, n, idx, rounds, out, sms, clk);
  run_lanes<4, 21, 3>(x, n, idx, rounds, out, sms, clk);
  run_lanes<1, 5, 3>(x, n, idx, rounds, out, sms, clk);
  run_lanes<2, 5, 3>(x, n, idx, rounds, out, sms, clk);
  run<4, 11, 3, false>(x, n, idx, rounds, out, sms, clk);
  run<4, 11, 3, true>(x, n, idx, rounds, out, sms, clk);
  run<8, 11, 3, true>(x, n, idx, rounds, out, sms, clk);
  run<4, 24, 3, true>(x, n, idx, rounds, out, sms, clk);
  run<8, 24, 3, true>(x, n, idx, rounds, out, sms, clk);
  run<8, 24, 3, false>(x, n, idx, rounds, out, sms, clk);
  run<16, 24, 3, true>(x, n, idx, rounds, out, sms, clk);
  run<4, 5, 3, true>(x, n, idx, rounds, out, sms, clk);
  run<8, 5, 3, true>(x, n, idx, rounds, out, sms, clk);
  return 0;
}
