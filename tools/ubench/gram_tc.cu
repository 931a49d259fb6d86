// gram_tc.cu -- check of the tcgen05 Gram plumbing (tc.cuh): the centred
// Gram matrix of 128 rows (d = 960) from the bf16 hi/lo split with three
// MMAs per 16-wide k step, against a double-precision host Gram.  Prints the
// worst error relative to |a||b| (the bound gram.cu relies on) and the time
// of one 128-row tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../paper_2310_20419_b200/csrc gram_tc.cu -o gram_tc
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

using namespace rnndg;

constexpr int kRows = 128;
#ifndef CHUNK
#define CHUNK 64
#endif
constexpr int kChunk = CHUNK;  // 64: SWIZZLE_128B rows, 32: SWIZZLE_64B rows

__global__ void __launch_bounds__(128, 1) k_gram(const float* __restrict__ x, const float* __restrict__ u,
                                                 int d, float* __restrict__ g, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* H = smem;
  uint8_t* L = smem + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (wid == 0) tc::tmem_alloc<128>(&tbase);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = tbase;
  constexpr uint32_t idesc = tc::idesc_bf16_f32<128, 128>();
  uint32_t phase = 0;
  const int nch = (d + kChunk - 1) / kChunk;
  for (int rep = 0; rep < reps; ++rep) {
    for (int ch = 0; ch < nch; ++ch) {
      // 128 rows x 8 units of 8 elements: 1024 items, 8 per thread
      for (int it = tid; it < kRows * (kChunk / 8); it += 128) {
        const int r = it / (kChunk / 8), c = it % (kChunk / 8);
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int k = ch * kChunk + c * 8 + e;
          v[e] = k < d ? __fsub_rn(x[size_t(r) * d + k], u[k]) : 0.f;
        }
        uint32_t h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) tc::split2(v[2 * e], v[2 * e + 1], h[e], l[e]);
        const uint32_t off = kChunk == 64 ? tc::sw128_off(r, c) : tc::sw64_off(r, c);
        *reinterpret_cast<uint4*>(H + off) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(L + off) = make_uint4(l[0], l[1], l[2], l[3]);
      }
      tc::fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc::tc_fence_after();
        const uint32_t ha = tc::smem_u32(H), la = tc::smem_u32(L);
#pragma unroll
        for (int k = 0; k < kChunk / 16; ++k) {
          const uint64_t dh = kChunk == 64 ? tc::sw128_desc(ha + 32 * k) : tc::sw64_desc(ha + 32 * k);
          const uint64_t dl = kChunk == 64 ? tc::sw128_desc(la + 32 * k) : tc::sw64_desc(la + 32 * k);
          const uint32_t acc = (ch | k) ? 1u : 0u;
          tc::mma_bf16(tm, dh, dh, idesc, acc);
          tc::mma_bf16(tm, dh, dl, idesc, 1u);
          tc::mma_bf16(tm, dl, dh, idesc, 1u);
        }
        tc::mma_commit(&bar);
      }
      tc::mbar_wait(&bar, phase);
      phase ^= 1u;
      tc::tc_fence_after();
    }
  }
  // row tid, columns 0..127
  for (int cb = 0; cb < 4; ++cb) {
    float v[32];
    tc::tmem_ld32(tm + (uint32_t(32 * wid) << 16) + uint32_t(32 * cb), v);
    for (int j = 0; j < 32; ++j) g[tid * kRows + 32 * cb + j] = v[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc<128>(tm);
}

int main() {
  const int d = 960;
  std::vector<float> x(size_t(kRows) * d), u(d);
  srand(1);
  for (int k = 0; k < d; ++k) u[k] = float(rand()) / RAND_MAX;
  for (int r = 0; r < kRows; ++r)
    for (int k = 0; k < d; ++k) {
      float s = (r % 3 == 0) ? 1e-3f : 0.05f;
      x[size_t(r) * d + k] = u[k] + s * (float(rand()) / RAND_MAX - 0.5f);
    }
  float *dx, *du, *dg;
  cudaMalloc(&dx, x.size() * 4);
  cudaMalloc(&du, d * 4);
  cudaMalloc(&dg, kRows * kRows * 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(du, u.data(), d * 4, cudaMemcpyHostToDevice);
  const int smem = 32768 + 1024;
  cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_gram<<<1, 128, smem>>>(dx, du, d, dg, 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> g(kRows * kRows);
  cudaMemcpy(g.data(), dg, g.size() * 4, cudaMemcpyDeviceToHost);
  // host Gram of the fp32-centred rows in double
  std::vector<double> c(size_t(kRows) * d), nrm(kRows);
  for (int r = 0; r < kRows; ++r) {
    double s = 0;
    for (int k = 0; k < d; ++k) {
      float t = x[size_t(r) * d + k] - u[k];
      c[size_t(r) * d + k] = t;
      s += double(t) * t;
    }
    nrm[r] = std::sqrt(s);
  }
  double worst = 0, worst_abs = 0;
  int bad = 0;
  for (int i = 0; i < kRows; ++i)
    for (int j = 0; j < kRows; ++j) {
      double s = 0;
      for (int k = 0; k < d; ++k) s += c[size_t(i) * d + k] * c[size_t(j) * d + k];
      const double err = std::fabs(double(g[i * kRows + j]) - s);
      const double rel = err / (nrm[i] * nrm[j]);
      if (rel > worst) worst = rel;
      if (err > worst_abs) worst_abs = err;
      if (!(rel < 1e-3)) ++bad;
      if (i < 2 && j < 3) printf("G[%d][%d] = %.9g (ref %.9g)\n", i, j, g[i * kRows + j], s);
    }
  printf("max |G - ref| / (|a||b|) = %.3e  (max abs %.3e), entries over 1e-3: %d\n", worst,
         worst_abs, bad);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  k_gram<<<1, 128, smem>>>(dx, du, d, dg, 100);
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  printf("chunk %d: one CTA, unpipelined: %.2f us per 128x128x960 tile (3 MMA sets)\n", kChunk, ms * 1e3 / 100);
  return bad ? 2 : 0;
}
