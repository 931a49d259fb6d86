// datagen.cpp -- seeded synthetic inputs (libdatagen.so: test/bench input
// generator, NOT part of the product library librnndg.so) for the five BASELINE.json configs.
//
// The paper's datasets (SIFT1M, GIST1M, Deep1M, SIFT20M)
// are not available; these generators stand in with the shapes, sizes and
// value distributions BASELINE.json describes.  Row i is a pure function of
// (config, seed, i): any row range can be produced independently, so the CPU
// baseline's bounded sample is an exact prefix of the GPU workload and held-out
// queries are simply rows n..n+nq-1 of the same stream.
//
// Randomness: the reference's own SplitMix64 / mix_seed (rng.hpp:13-42),
// restated here.  Gaussians by Box-Muller in double, stored as float32.
// Compiled with -ffp-contract=off; per-row arithmetic order is fixed, so the
// output bytes do not depend on the thread count.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include <omp.h>


namespace {

struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  uint64_t bounded(uint64_t b) {
    return uint64_t((static_cast<__uint128_t>(next()) * b) >> 64);
  }
  double unit() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
  double gauss() {
    double u1 = 1.0 - unit();  // (0, 1]
    double u2 = unit();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

uint64_t mix_seed(uint64_t seed, uint64_t stream) {
  Rng g(seed ^ (0xD1B54A32D192ED03ULL * (stream + 1)));
  return g.next();
}

constexpr uint64_t kClusterSalt = 0xC1A55E5ULL;

struct Spec {
  uint32_t d;
  uint32_t comps;
};

Spec spec_of(int cfg) {
  switch (cfg) {
    case 1 /* C1 */: return {128, 64};
    case 2 /* C2 */: return {128, 1000};
    case 3 /* C3 */: return {960, 500};
    case 4 /* C4 */: return {96, 2000};
    case 5 /* C5 */: return {96, 10000};
    default: return {0, 0};
  }
}

// C1: 64-component isotropic GMM, centres ~ N(0,1)^128, sigma 0.3.
void gen_gmm(uint64_t seed, uint64_t row0, uint64_t nrows, const Spec& sp,
             float* out) {
  std::vector<float> centres(size_t(sp.comps) * sp.d);
  for (uint32_t k = 0; k < sp.comps; ++k) {
    Rng r(mix_seed(seed ^ kClusterSalt, k));
    for (uint32_t j = 0; j < sp.d; ++j) centres[size_t(k) * sp.d + j] = float(r.gauss());
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < int64_t(nrows); ++i) {
    Rng r(mix_seed(seed, row0 + uint64_t(i)));
    const float* c = centres.data() + size_t(r.bounded(sp.comps)) * sp.d;
    float* o = out + size_t(i) * sp.d;
    for (uint32_t j = 0; j < sp.d; ++j) o[j] = float(double(c[j]) + 0.3 * r.gauss());
  }
}

// C2: SIFT-like.  1,000 clusters of non-negative histogram-like vectors:
// centre_j = 120 * U^2 (skewed to small counts), a per-cluster mask zeroes
// ~35% of dimensions, per-vector noise sigma 12, rounded and clipped to
// [0, 255].  Clipping adds zeros: ~40% of coordinates end up 0.
void gen_siftlike(uint64_t seed, uint64_t row0, uint64_t nrows, const Spec& sp,
                  float* out) {
  std::vector<float> centres(size_t(sp.comps) * sp.d);
  std::vector<uint8_t> mask(size_t(sp.comps) * sp.d);
  for (uint32_t k = 0; k < sp.comps; ++k) {
    Rng r(mix_seed(seed ^ kClusterSalt, k));
    for (uint32_t j = 0; j < sp.d; ++j) {
      double u = r.unit();
      centres[size_t(k) * sp.d + j] = float(120.0 * u * u);
      mask[size_t(k) * sp.d + j] = r.unit() < 0.35 ? 1 : 0;
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < int64_t(nrows); ++i) {
    Rng r(mix_seed(seed, row0 + uint64_t(i)));
    size_t k = size_t(r.bounded(sp.comps));
    const float* c = centres.data() + k * sp.d;
    const uint8_t* m = mask.data() + k * sp.d;
    float* o = out + size_t(i) * sp.d;
    for (uint32_t j = 0; j < sp.d; ++j) {
      double g = r.gauss();
      double v = m[j] ? 0.0 : std::nearbyint(double(c[j]) + 12.0 * g);
      o[j] = float(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
    }
  }
}

// C3: GIST-like.  500 clusters; x = centre + B_k z, centre ~ U[0.15, 0.85]^960,
// B_k a 960x40 Gaussian basis (entries N(0, 0.03^2)), z_c ~ N(0, 1/(1+c/8))
// (decaying spectrum, intrinsic dimension ~40), clipped to [0, 1].
constexpr uint32_t kGistRank = 40;
void gen_gistlike(uint64_t seed, uint64_t row0, uint64_t nrows, const Spec& sp,
                  float* out) {
  const uint32_t d = sp.d;
  std::vector<float> centres(size_t(sp.comps) * d);
  std::vector<float> basis(size_t(sp.comps) * kGistRank * d);  // [k][c][j]
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < int64_t(sp.comps); ++k) {
    Rng r(mix_seed(seed ^ kClusterSalt, uint64_t(k)));
    for (uint32_t j = 0; j < d; ++j)
      centres[size_t(k) * d + j] = float(0.15 + 0.7 * r.unit());
    float* b = basis.data() + size_t(k) * kGistRank * d;
    for (size_t q = 0; q < size_t(kGistRank) * d; ++q) b[q] = float(0.03 * r.gauss());
  }
  float lam[kGistRank];
  for (uint32_t c = 0; c < kGistRank; ++c) lam[c] = float(1.0 / std::sqrt(1.0 + c / 8.0));
#pragma omp parallel
  {
    std::vector<float> acc(d);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < int64_t(nrows); ++i) {
      Rng r(mix_seed(seed, row0 + uint64_t(i)));
      size_t k = size_t(r.bounded(sp.comps));
      float z[kGistRank];
      for (uint32_t c = 0; c < kGistRank; ++c) z[c] = float(r.gauss()) * lam[c];
      const float* ctr = centres.data() + k * d;
      const float* b = basis.data() + k * kGistRank * d;
      std::memcpy(acc.data(), ctr, sizeof(float) * d);
      for (uint32_t c = 0; c < kGistRank; ++c) {
        const float zc = z[c];
        const float* bc = b + size_t(c) * d;
        for (uint32_t j = 0; j < d; ++j) acc[j] += bc[j] * zc;
      }
      float* o = out + size_t(i) * d;
      for (uint32_t j = 0; j < d; ++j) {
        float v = acc[j];
        o[j] = v < 0.f ? 0.f : (v > 1.f ? 1.f : v);
      }
    }
  }
}

// C4/C5: Deep-like.  Unit centres (normalised N(0, I)), x = centre + 0.05 g,
// renormalised to unit length (von Mises-Fisher-style mixture).
void gen_deeplike(uint64_t seed, uint64_t row0, uint64_t nrows, const Spec& sp,
                  float* out) {
  const uint32_t d = sp.d;
  std::vector<float> centres(size_t(sp.comps) * d);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < int64_t(sp.comps); ++k) {
    Rng r(mix_seed(seed ^ kClusterSalt, uint64_t(k)));
    double norm = 0.0;
    float* c = centres.data() + size_t(k) * d;
    for (uint32_t j = 0; j < d; ++j) {
      double g = r.gauss();
      c[j] = float(g);
      norm += g * g;
    }
    double inv = 1.0 / std::sqrt(norm);
    for (uint32_t j = 0; j < d; ++j) c[j] = float(double(c[j]) * inv);
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < int64_t(nrows); ++i) {
    Rng r(mix_seed(seed, row0 + uint64_t(i)));
    const float* c = centres.data() + size_t(r.bounded(sp.comps)) * d;
    double tmp[1024];
    double norm = 0.0;
    for (uint32_t j = 0; j < d; ++j) {
      tmp[j] = double(c[j]) + 0.05 * r.gauss();
      norm += tmp[j] * tmp[j];
    }
    double inv = 1.0 / std::sqrt(norm);
    float* o = out + size_t(i) * d;
    for (uint32_t j = 0; j < d; ++j) o[j] = float(tmp[j] * inv);
  }
}

}  // namespace

extern "C" {

uint32_t dg_synth_dim(int cfg) { return spec_of(cfg).d; }

int dg_synth(int cfg, uint64_t seed, uint64_t row0, uint64_t nrows, float* out) {
  Spec sp = spec_of(cfg);
  if (sp.d == 0 || (nrows && !out)) return 1;
  switch (cfg) {
    case 1 /* C1 */: gen_gmm(seed, row0, nrows, sp, out); break;
    case 2 /* C2 */: gen_siftlike(seed, row0, nrows, sp, out); break;
    case 3 /* C3 */: gen_gistlike(seed, row0, nrows, sp, out); break;
    case 4 /* C4 */:
    case 5 /* C5 */: gen_deeplike(seed, row0, nrows, sp, out); break;
    default: return 1;
  }
  return 0;
}

}  // extern "C"
