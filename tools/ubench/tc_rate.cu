// tc_rate.cu -- issue rate of tcgen05.mma.kind::f16 (bf16 -> fp32) from one
// thread, back to back into one TMEM accumulator, for the shapes and
// operand swizzles gram.cu could use.  One CTA per SM, all SMs; prints
// cycles per MMA and the implied share of the dense bf16 peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../paper_2310_20419_b200/csrc tc_rate.cu -o tc_rate
#include <cstdio>

#include "tc.cuh"

using namespace rnndg;

template <uint32_t N, bool kSW64>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, wid = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3F803F80u;
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (wid == 0) tc::tmem_alloc<256>(&tbase);
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid == 0) {
    constexpr uint32_t idesc = tc::idesc_bf16_f32<128, N>();
    const uint32_t a = tc::smem_u32(smem), b = a + 32768;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t k = uint32_t(i & 1) * 32;
      const uint64_t da = kSW64 ? tc::sw64_desc(a + k) : tc::sw128_desc(a + k);
      const uint64_t db = kSW64 ? tc::sw64_desc(b + k) : tc::sw128_desc(b + k);
      tc::mma_bf16(tbase, da, db, idesc, i ? 1u : 0u);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    atomicAdd(cyc, (unsigned long long)(t1 - t0));
  }
  tc::tc_fence_before();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc<256>(tbase);
}

template <uint32_t N, bool kSW64>
void run(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(k_rate<N, kSW64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  k_rate<N, kSW64><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = double(h) / sms / iters;
  const double flop = 2.0 * 128 * N * 16;
  printf("M128 N%-3u K16 %s: %s %.1f cycles per MMA, %.0f flop/clk/SM (dense peak ~7700)\n", N,
         kSW64 ? "SW64 " : "SW128", e == cudaSuccess ? "" : cudaGetErrorString(e), cyc, flop / cyc);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>(sms);
  run<128, false>(sms);
  run<256, false>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  run<80, false>(sms);
  return 0;
}
