// flat_pairs.cu -- ceiling of the exact-L2 pair evaluation when it is taken
// out of the per-list walk: a flat array of tasks evaluated by a lean kernel
// at full occupancy, with register tiles of TW provisional rows x TV
// candidate rows per quad (every loaded block is used TV resp. TW times).
//
// Task set: G "lists", each with D provisional rows and N candidate rows drawn
// at random from a 1M x 960 store in the chain-blocked layout; all D x N pairs
// of a list are evaluated (what a speculative round does).  A quad of lanes
// per tile, a lane per fp32 chain, 256-bit loads, two blocks in flight -- the
// arithmetic of quad_l2 (csrc/quad.cuh), bit-exact by construction.
// Reports pair evaluations per second and SM-cycles per evaluation
// (k_scan_spec reaches ~127 inside its walk).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o flat_pairs flat_pairs.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                           \
  do {                                                                  \
    cudaError_t e = (x);                                                \
    if (e != cudaSuccess) {                                             \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                          \
    }                                                                   \
  } while (0)

constexpr uint32_t kD = 960;
constexpr uint32_t kNblk = kD / 32;

template <bool kNA>
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

__device__ __forceinline__ void chain_step(const float (&va)[8], const float (&vb)[8], float& s) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#ifdef FFMA_IMM
    float t, m;
    asm("fma.rn.f32 %0, %1, 0f3F800000, %2;" : "=f"(t) : "f"(va[i]), "f"(-vb[i]));
    asm("fma.rn.f32 %0, %1, %1, 0f80000000;" : "=f"(m) : "f"(t));
    asm("fma.rn.f32 %0, %1, 0f3F800000, %2;" : "=f"(s) : "f"(m), "f"(s));
#else
    const float t = __fsub_rn(va[i], vb[i]);
    s = __fadd_rn(s, __fmul_rn(t, t));
#endif
  }
}

struct Tasks {
  const uint32_t* wid;  // G x D provisional row ids
  const uint32_t* vid;  // G x N candidate row ids
  uint32_t G, D, N;
  float* out;           // G x N x D distances
};

// One quad per TW x TV tile.  kDepth blocks in flight per row.
template <int TW, int TV, int kDepth, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks)
k_tiles(const float* __restrict__ xp, Tasks t, unsigned int* work) {
  const uint32_t lane = threadIdx.x & 31u, quad = lane >> 2, chain = lane & 3u;
  const uint32_t wt = t.D / TW, vt = t.N / TV;     // tiles per list along w and v
  const uint64_t ntile = uint64_t(t.G) * wt * vt;
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(work, 8u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= ntile) break;
    uint64_t ti = uint64_t(base) + quad;
    if (ti >= ntile) ti = ntile - 1;
    // tile order: v-tile major, then w-tile (a list's w rows stay hot in L1)
    const uint32_t g = uint32_t(ti / (wt * vt));
    const uint32_t r = uint32_t(ti % (wt * vt));
    const uint32_t vi = r / wt, wi = r % wt;
    const float* pw[TW];
    const float* pv[TV];
#pragma unroll
    for (int i = 0; i < TW; ++i)
      pw[i] = xp + uint64_t(t.wid[uint64_t(g) * t.D + wi * TW + i]) * kD + 8 * chain;
#pragma unroll
    for (int j = 0; j < TV; ++j)
      pv[j] = xp + uint64_t(t.vid[uint64_t(g) * t.N + vi * TV + j]) * kD + 8 * chain;
    float s[TW][TV];
#pragma unroll
    for (int i = 0; i < TW; ++i)
#pragma unroll
      for (int j = 0; j < TV; ++j) s[i][j] = 0.f;
    float bw[kDepth][TW][8], bv[kDepth][TV][8];
#pragma unroll
    for (int dd = 0; dd < kDepth; ++dd) {
#pragma unroll
      for (int j = 0; j < TV; ++j) ld256<true>(pv[j] + 32 * dd, bv[dd][j]);
#pragma unroll
      for (int i = 0; i < TW; ++i) ld256<false>(pw[i] + 32 * dd, bw[dd][i]);
    }
    for (uint32_t blk = kDepth; blk < kNblk; blk += kDepth) {
#pragma unroll
      for (int dd = 0; dd < kDepth; ++dd) {
#pragma unroll
        for (int i = 0; i < TW; ++i)
#pragma unroll
          for (int j = 0; j < TV; ++j) chain_step(bv[dd][j], bw[dd][i], s[i][j]);
        if (blk + dd < kNblk) {
#pragma unroll
          for (int j = 0; j < TV; ++j) ld256<true>(pv[j] + 32 * (blk + dd), bv[dd][j]);
#pragma unroll
          for (int i = 0; i < TW; ++i) ld256<false>(pw[i] + 32 * (blk + dd), bw[dd][i]);
        }
      }
    }
    // kNblk = 30 is a multiple of kDepth in {1, 2, 3}: drain
#pragma unroll
    for (int dd = 0; dd < kDepth; ++dd)
#pragma unroll
      for (int i = 0; i < TW; ++i)
#pragma unroll
        for (int j = 0; j < TV; ++j) chain_step(bv[dd][j], bw[dd][i], s[i][j]);
#pragma unroll
    for (int i = 0; i < TW; ++i)
#pragma unroll
      for (int j = 0; j < TV; ++j) {
        float x = s[i][j];
        const float x1 = __shfl_down_sync(0xffffffffu, x, 1);
        const float p = __fadd_rn(x, x1);
        const float p2 = __shfl_down_sync(0xffffffffu, p, 2);
        const float sum = __fadd_rn(p, p2);
        if (chain == 0 && uint64_t(base) + quad < ntile)
          t.out[(uint64_t(g) * t.N + vi * TV + j) * t.D + wi * TW + i] = sum;
      }
  }
}

__global__ void k_fill(float* x, uint64_t n) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z ^= z >> 29;
    x[i] = float(z & 0xFFFF) * (1.f / 65536.f);
  }
}

static uint64_t rng_state = 12345;
static uint32_t rnd(uint32_t bound) {
  rng_state = rng_state * 6364136223846793005ULL + 1442695040888963407ULL;
  return uint32_t((rng_state >> 33) % bound);
}

template <int TW, int TV, int kDepth, int kMinBlocks>
static double run(const char* name, const float* xp, Tasks t, unsigned int* work, int sms,
                  double clk_hz, std::vector<float>* ref) {
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k_tiles<TW, TV, kDepth, kMinBlocks>));
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tiles<TW, TV, kDepth, kMinBlocks>, 256,
                                                   0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaMemset(work, 0, 4));
    CK(cudaEventRecord(e0));
    k_tiles<TW, TV, kDepth, kMinBlocks><<<sms * nb, 256>>>(xp, t, work);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double evals = double(t.G) * t.D * t.N;
  const double cyc = best * 1e-3 * clk_hz * sms / evals;
  // bit-exactness across tilings: compare with the 1x1 result
  std::vector<float> h(size_t(t.G) * t.D * t.N);
  CK(cudaMemcpy(h.data(), t.out, h.size() * 4, cudaMemcpyDeviceToHost));
  const char* same = "";
  if (ref->empty()) *ref = h;
  else same = memcmp(ref->data(), h.data(), h.size() * 4) ? " MISMATCH" : " bit-equal";
  printf("%-28s regs %3d  %2d CTAs/SM  %8.3f ms  %.3e evals/s  %6.1f SM-cyc/eval%s\n", name,
         fa.numRegs, nb, best, evals / (best * 1e-3), cyc, same);
  fflush(stdout);
  return cyc;
}

#include <cstring>

int main(int argc, char** argv) {
  const uint64_t n = 1000000;
  const uint32_t G = argc > 1 ? atoi(argv[1]) : 200000;
  const uint32_t D = 4, N = argc > 2 ? atoi(argv[2]) : 24;
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const double clk = clk_khz * 1e3;
  float* xp;
  CK(cudaMalloc(&xp, n * kD * 4));
  k_fill<<<p.multiProcessorCount * 8, 256>>>(xp, n * kD);
  std::vector<uint32_t> hw(size_t(G) * D), hv(size_t(G) * N);
  for (auto& w : hw) w = rnd(uint32_t(n));
  for (auto& v : hv) v = rnd(uint32_t(n));
  uint32_t *dw, *dv;
  float* out;
  unsigned int* work;
  CK(cudaMalloc(&dw, hw.size() * 4));
  CK(cudaMalloc(&dv, hv.size() * 4));
  CK(cudaMalloc(&out, size_t(G) * D * N * 4));
  CK(cudaMalloc(&work, 4));
  CK(cudaMemcpy(dw, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice));
  Tasks t{dw, dv, G, D, N, out};
  printf("%s, %d SMs, %.0f MHz; %u lists x %u x %u pairs\n", p.name, p.multiProcessorCount,
         clk / 1e6, G, D, N);
  std::vector<float> ref;
  const int sms = p.multiProcessorCount;
  run<1, 1, 2, 1>("1x1 depth2", xp, t, work, sms, clk, &ref);
  run<1, 1, 2, 4>("1x1 depth2 (>=4 CTAs)", xp, t, work, sms, clk, &ref);
  run<1, 1, 1, 1>("1x1 depth1", xp, t, work, sms, clk, &ref);
  run<1, 1, 3, 1>("1x1 depth3", xp, t, work, sms, clk, &ref);
  run<2, 1, 2, 1>("2x1 depth2", xp, t, work, sms, clk, &ref);
  run<4, 1, 2, 1>("4x1 depth2", xp, t, work, sms, clk, &ref);
  run<4, 1, 1, 1>("4x1 depth1", xp, t, work, sms, clk, &ref);
  run<2, 2, 2, 1>("2x2 depth2", xp, t, work, sms, clk, &ref);
  run<2, 2, 1, 1>("2x2 depth1", xp, t, work, sms, clk, &ref);
  run<2, 2, 1, 3>("2x2 depth1 (>=3 CTAs)", xp, t, work, sms, clk, &ref);
  run<4, 2, 1, 1>("4x2 depth1", xp, t, work, sms, clk, &ref);
  run<4, 2, 2, 1>("4x2 depth2", xp, t, work, sms, clk, &ref);
  run<2, 4, 1, 1>("2x4 depth1", xp, t, work, sms, clk, &ref);
  run<4, 4, 1, 1>("4x4 depth1", xp, t, work, sms, clk, &ref);
  return 0;
}
