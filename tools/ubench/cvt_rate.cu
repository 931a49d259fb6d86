// cvt_rate.cu -- issue cost of the fp16 -> fp32 paths on sm_100a: HADD2.F32
// (cvt.f32.f16), bit-shift rebuild (bf16-style), and the fp32 chain step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 cvt_rate.cu -o cvt_rate
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ uint64_t h2f2(uint32_t h) {
  uint64_t v;
  asm volatile("{\n\t.reg .f16 lo, hi;\n\t.reg .f32 a, b;\n\t"
      "mov.b32 {lo, hi}, %1;\n\tcvt.f32.f16 a, lo;\n\tcvt.f32.f16 b, hi;\n\t"
      "mov.b64 %0, {a, b};\n\t}" : "=l"(v) : "r"(h));
  return v;
}
__device__ __forceinline__ uint64_t b2f2(uint32_t h) {
  uint64_t v;
  const uint32_t lo = h << 16, hi = h & 0xffff0000u;
  asm volatile("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(lo), "r"(hi));
  return v;
}

template <int MODE>
__global__ void k(const uint32_t* in, float* out, int iters) {
  uint32_t a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = in[threadIdx.x + i]; b[i] = in[threadIdx.x + 8 + i]; }
  uint64_t acc = 0;
  float s = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        uint64_t t;
        asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(h2f2(a[i])), "l"(h2f2(b[i])));
        asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(t));
      } else if (MODE == 1) {
        uint64_t t;
        asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(b2f2(a[i])), "l"(b2f2(b[i])));
        asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(t));
      } else {
        // exact path: 2 elements per i (same element count as the packed modes)
        float x0 = __uint_as_float(a[i]), y0 = __uint_as_float(b[i]);
        float x1 = __uint_as_float(a[i] ^ 0x10), y1 = __uint_as_float(b[i] ^ 0x10);
        float t0 = __fsub_rn(x0, y0), t1 = __fsub_rn(x1, y1);
        s = __fadd_rn(s, __fmul_rn(t0, t0));
        s = __fadd_rn(s, __fmul_rn(t1, t1));
      }
      a[i] += 0x00010001u;
    }
  }
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc));
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + y + s;
}

int main() {
  uint32_t* in; float* out;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0x3c, 4096 * 4);
  cudaMalloc(&out, 148 * 16 * 1024 * 4);
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  const int iters = 4096;
  const char* names[] = {"fp16 cvt (HADD2.F32) + FADD2 + FFMA2", "bf16 shift + FADD2 + FFMA2", "fp32 exact FADD/FMUL/FADD"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(t0);
      if (m == 0) k<0><<<148 * 8, 256>>>(in, out, iters);
      if (m == 1) k<1><<<148 * 8, 256>>>(in, out, iters);
      if (m == 2) k<2><<<148 * 8, 256>>>(in, out, iters);
      cudaEventRecord(t1); cudaEventSynchronize(t1);
      float ms; cudaEventElapsedTime(&ms, t0, t1);
      const double elems = double(148 * 8 * 256) * iters * 16;  // element pairs
      if (rep) printf("%-40s %.3f ms  %.1f element-pairs/clk/SM (at 1.965 GHz)\n", names[m], ms,
                      elems / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
