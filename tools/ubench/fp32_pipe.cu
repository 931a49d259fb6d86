// fp32_pipe.cu -- microbenchmark: issue rate of the exact-L2 inner step
// (t = a - b; s = s + t * t, each IEEE round-to-nearest, no FMA) on the
// FP32 pipe, unpacked (FADD/FMUL) vs packed f32x2 (FADD2/FMUL2).
// Operands come from registers, so this is the pipe bound of the distance
// stage, with no memory traffic.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void upk(unsigned long long v, float& x, float& y) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}

// 8 independent chains per thread, unpacked
__global__ void k_unpacked(const float* in, float* out, unsigned long long) {
  float a[8], b[8], s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = in[threadIdx.x + i];
    b[i] = in[threadIdx.x + 8 + i];
    s[i] = 0.f;
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float t = __fsub_rn(a[i], b[(i + it) & 7]);
      s[i] = __fadd_rn(s[i], __fmul_rn(t, t));
    }
  }
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// 8 independent packed chain pairs (16 chains) per thread
__global__ void k_packed(const float* in, float* out, unsigned long long nz) {
  unsigned long long a[8], b[8], s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = pk(in[threadIdx.x + i], in[threadIdx.x + 16 + i]);
    b[i] = pk(in[threadIdx.x + 8 + i], in[threadIdx.x + 24 + i]);
    s[i] = 0ull;
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned long long t, m;
      asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(a[i]), "l"(b[(i + it) & 7]));
      asm volatile("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m) : "l"(t), "l"(nz));
      asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(s[i]) : "l"(s[i]), "l"(m));
    }
  }
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float x, y;
    upk(s[i], x, y);
    r += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// packed with the candidate broadcast into both halves: (v - w1, v - w2)
__global__ void k_packed_bcast(const float* in, float* out, unsigned long long nz) {
  float v[8];
  unsigned long long w[8], s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = in[threadIdx.x + i];
    w[i] = pk(in[threadIdx.x + 8 + i], in[threadIdx.x + 24 + i]);
    s[i] = 0ull;
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned long long t, m;
      const float x = v[(i + it) & 7];
      asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(x, x)), "l"(w[i]));
      asm volatile("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m) : "l"(t), "l"(nz));
      asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(s[i]) : "l"(s[i]), "l"(m));
    }
  }
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float x, y;
    upk(s[i], x, y);
    r += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <typename K>
float run(K kern, const float* in, float* out, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned long long nz = 0x8000000080000000ull;  // (-0.0f, -0.0f)
  kern<<<blocks, threads>>>(in, out, nz);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(in, out, nz);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *in, *out;
  cudaMalloc(&in, 4096 * sizeof(float));
  cudaMalloc(&out, 64 << 20);
  cudaMemset(in, 0, 4096 * sizeof(float));
  for (int threads : {256, 512, 1024}) {
    const int blocks = sms * (2048 / threads);
    const double elems = double(blocks) * threads * ITERS * 8;  // element steps (3 ops)
    float mu = run(k_unpacked, in, out, blocks, threads);
    float mp = run(k_packed, in, out, blocks, threads);
    float mb = run(k_packed_bcast, in, out, blocks, threads);
    // lane-element-steps per SM-cycle at the nominal max clock
    const double cyc = double(clk) * 1e3;
    printf("threads %d: unpacked %.3f ms = %.1f elem/clk/SM | packed %.3f ms = %.1f | bcast %.3f ms = %.1f\n",
           threads, mu, elems / (mu * 1e-3) / cyc / sms, mp, 2 * elems / (mp * 1e-3) / cyc / sms, mb,
           2 * elems / (mb * 1e-3) / cyc / sms);
  }
  return 0;
}
