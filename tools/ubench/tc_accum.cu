// tc_accum.cu -- how tcgen05.mma (kind::f16, bf16 inputs, fp32 accumulator)
// rounds its additions.  Each case sets one row of A and one row of B so
// that D[0][0] gets chosen products; the other rows are zero.  Prints the
// result against the exact sum, in units of the result's ulp.  This is the
// hardware model behind the error band of gram.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../paper_2310_20419_b200/csrc tc_accum.cu -o tc_accum
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "tc.cuh"

using namespace rnndg;

// one 128x64 bf16 tile for A and for B per k step (we use only K = 16 of the
// 64: the first MMA of each step); steps accumulate into D
__global__ void k_accum(const uint16_t* __restrict__ a_rows, const uint16_t* __restrict__ b_rows,
                        int steps, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = smem;
  uint8_t* B = smem + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, wid = tid >> 5;
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
  for (int i = tid; i < 32768 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  uint32_t phase = 0;
  for (int st = 0; st < steps; ++st) {
    __syncthreads();
    if (tid < 8) {  // row 0, units 0..1 (k 0..15) of A and B
      // unit c covers k = 8c .. 8c+7
      const int c = tid & 1;
      const bool isb = tid >= 4;
      if ((tid & 3) < 2) {
        const uint16_t* src = (isb ? b_rows : a_rows) + st * 16 + 8 * c;
        uint4 v;
        memcpy(&v, src, 16);
        *reinterpret_cast<uint4*>((isb ? B : A) + tc::sw128_off(0, c)) = v;
      }
    }
    tc::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
      tc::mma_bf16(tm, tc::sw128_desc(tc::smem_u32(A)), tc::sw128_desc(tc::smem_u32(B)), idesc,
                   st ? 1u : 0u);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1u;
    tc::tc_fence_after();
  }
  if (wid == 0) {
    float v[32];
    tc::tmem_ld32(tm, v);
    if (tid == 0) out[0] = v[0];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc<128>(tm);
}

static uint16_t bf(float x) {  // exact for the values used
  uint32_t u;
  memcpy(&u, &x, 4);
  return uint16_t(u >> 16);
}

struct Case {
  const char* name;
  std::vector<float> a, b;  // 16 * steps each
};

int main() {
  uint16_t *da, *db;
  float* dout;
  cudaMalloc(&da, 16 * 256 * 2);
  cudaMalloc(&db, 16 * 256 * 2);
  cudaMalloc(&dout, 4);
  const int smem = 32768 + 1024;
  cudaFuncSetAttribute(k_accum, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<Case> cases;
  auto add = [&](const char* nm, int steps, auto fa) {
    Case c{nm, std::vector<float>(16 * steps, 0.f), std::vector<float>(16 * steps, 0.f)};
    for (int s = 0; s < steps; ++s)
      for (int k = 0; k < 16; ++k) fa(s, k, c.a[16 * s + k], c.b[16 * s + k]);
    cases.push_back(c);
  };
  const float t = std::ldexp(1.f, -13), t2 = std::ldexp(1.f, -12);  // t*t2 = 2^-25
  // acc 1 (step 0), then 16 products of 2^-25 in one MMA
  add("acc=1 then 16 x 2^-25 in one MMA", 2, [&](int s, int k, float& a, float& b) {
    if (s == 0) { a = k == 0 ? 1.f : 0.f; b = k == 0 ? 1.f : 0.f; }
    else { a = t; b = t2; }
  });
  // one MMA: 1 + 15 x 2^-25
  add("one MMA: 1 + 15 x 2^-25", 1, [&](int s, int k, float& a, float& b) {
    a = k == 0 ? 1.f : t; b = k == 0 ? 1.f : t2;
  });
  // acc 1, then 1 product of 2^-25 per MMA, 16 MMAs
  add("acc=1 then 2^-25 per MMA x 16", 17, [&](int s, int k, float& a, float& b) {
    if (s == 0) { a = k == 0 ? 1.f : 0.f; b = k == 0 ? 1.f : 0.f; }
    else { a = k == 0 ? t : 0.f; b = k == 0 ? t2 : 0.f; }
  });
  // acc 1, then 1 product of 3*2^-25 per MMA, 16 MMAs
  add("acc=1 then 3*2^-25 per MMA x 16", 17, [&](int s, int k, float& a, float& b) {
    if (s == 0) { a = k == 0 ? 1.f : 0.f; b = k == 0 ? 1.f : 0.f; }
    else { a = k == 0 ? 3.f * t : 0.f; b = k == 0 ? t2 : 0.f; }
  });
  // acc 1, then 2^-24 + 2^-25 in one MMA (round to nearest would give 1+2^-23)
  add("acc=1 then 2^-24+2^-25 in one MMA", 2, [&](int s, int k, float& a, float& b) {
    if (s == 0) { a = k == 0 ? 1.f : 0.f; b = k == 0 ? 1.f : 0.f; }
    else { a = k < 2 ? t : 0.f; b = k == 0 ? 2.f * t2 : (k == 1 ? t2 : 0.f); }
  });
  // 16 products: 1, -1 + tiny cancellations
  add("one MMA: 1 - (1-2^-24)... (1 + 2^-20 - 1)", 1, [&](int s, int k, float& a, float& b) {
    a = k == 0 ? 1.f : (k == 1 ? -1.f : (k == 2 ? std::ldexp(1.f, -10) : 0.f));
    b = k == 0 ? 1.f : (k == 1 ? 1.f : (k == 2 ? std::ldexp(1.f, -10) : 0.f));
  });
  // 16 products each 1 + 2^-7 squared-ish: many terms near equal magnitude
  add("one MMA: 16 x (1+2^-7)(1+2^-7)", 1, [&](int s, int k, float& a, float& b) {
    a = 1.f + std::ldexp(1.f, -7); b = 1.f + std::ldexp(1.f, -7);
  });
  // acc 2^24-ish then small: acc = 1, add -2^-25 x 16 (subtraction direction)
  add("acc=1 then 16 x (-2^-25) in one MMA", 2, [&](int s, int k, float& a, float& b) {
    if (s == 0) { a = k == 0 ? 1.f : 0.f; b = k == 0 ? 1.f : 0.f; }
    else { a = -t; b = t2; }
  });
  // 1 + 2^-9 * 2^-15 products: 16 x 2^-24 (each exactly half an ulp of 1)
  add("acc=1 then 16 x 2^-24 in one MMA", 2, [&](int s, int k, float& a, float& b) {
    if (s == 0) { a = k == 0 ? 1.f : 0.f; b = k == 0 ? 1.f : 0.f; }
    else { a = t; b = 2.f * t2; }
  });
  // 180 MMAs each of 16 equal products, magnitude 1/16: running sum grows
  add("180 MMAs of 16 x (1+2^-7)^2/16", 180, [&](int s, int k, float& a, float& b) {
    a = 0.25f * (1.f + std::ldexp(1.f, -7)); b = 0.25f * (1.f + std::ldexp(1.f, -7));
  });
  for (auto& c : cases) {
    const int steps = int(c.a.size() / 16);
    std::vector<uint16_t> ha(c.a.size()), hb(c.b.size());
    double exact = 0;
    for (size_t i = 0; i < c.a.size(); ++i) {
      ha[i] = bf(c.a[i]);
      hb[i] = bf(c.b[i]);
      float ra, rb;
      uint32_t ua = uint32_t(ha[i]) << 16, ub = uint32_t(hb[i]) << 16;
      memcpy(&ra, &ua, 4);
      memcpy(&rb, &ub, 4);
      exact += double(ra) * double(rb);
    }
    cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
    k_accum<<<1, 128, smem>>>(da, db, steps, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    float got;
    cudaMemcpy(&got, dout, 4, cudaMemcpyDeviceToHost);
    const float rn = float(exact);
    const double ulp = std::ldexp(1.0, std::ilogb(double(rn)) - 23);
    printf("%-44s got %.10g exact %.12g  err %+.3f ulp (RN %+.3f)\n", c.name, got, exact,
           (double(got) - exact) / ulp, (double(rn) - exact) / ulp);
  }
  return 0;
}
