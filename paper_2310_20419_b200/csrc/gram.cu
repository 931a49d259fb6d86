// gram.cu -- the distance stage for lists of at most 128 entries on the
// tensor cores: each list's rows are read ONCE per scan; a Gram filter
// decides the walk's comparisons; exact fp32 L2 only where the result must
// be bit-exact.
//
// scan_vertex (builder.cpp:41-69) sorts u's list by (dist, id) and walks it:
// candidate v is removed by the first kept w (old/old pairs skipped) with
// v.dist >= l2_sq(v, w), and the redirect (w, v, l2_sq(v, w)) is appended to
// w's list.  Per tile of lists:
//
//  1. Producers stream every row of the list once (the SURVEY 8(d)
//     algorithmic bytes), centre it on u's row (x' = x - u, fp32) and split
//     it into bf16 hi + lo (x' = hi + lo + e, |e| <= 2^-16 |x'|) into
//     128-byte-swizzled shared-memory stages.  While doing so they finish
//     the exact rnnd::l2_sq(x, u) of every row -- x' is exactly the
//     reference's (a - b) term, so the four fp32 chains of metric.hpp:15-24
//     only need a square and an add per element (chain-blocked store, see
//     quad.cuh).  That is the exact cached distance of every entry whose
//     distance is still pending (item 5).
//  2. One thread issues three tcgen05 MMAs per 16-wide k step
//     (hi.hi^T + hi.lo^T + lo.hi^T): the Gram matrix G ~= X' X'^T of the
//     whole tile accumulates in TMEM (128 x 128 fp32).
//  3. d~(v,w) = G_vv + G_ww - 2 G_vw.  Error bound: the split drops
//     <= 3.1 * 2^-16 |x'_v,k x'_w,k| per term; the accumulator truncates
//     (round toward zero) once per MMA instruction with the 16 products
//     summed before it (tools/ubench/tc_accum.cu on this B200: 1 + 15 x
//     2^-25 in one MMA -> 1 + 3 ulp, 2^-25 per MMA x 16 -> 1), so with two
//     truncations per instruction budgeted the accumulation error is
//     <= 2 (3K/16) 2^-23 sum|x'_v,k x'_w,k| + 2^-21 sum|...| (terms that
//     fall below the alignment window).  By Cauchy-Schwarz
//     |G_vw - x'_v.x'_w| <= beta |x'_v||x'_w|, beta = 9.1e-5 at K = 960,
//     |d~ - d| <= 2 beta (|x'_v|^2 + |x'_w|^2), plus rnnd::l2_sq's own
//     rounding (4 chains of K/4 positive terms).  With a 1.25 safety factor
//       eps = 2.65e-4 (G_vv + G_ww) + 1e-25   (d = 960; launch_gram)
//     the absolute term covering bf16/fp32 underflow.  d~ + eps < v.dist is
//     an occlusion for certain, d~ - eps > v.dist certainly none; anything
//     else (non-finite G included) is decided by the exact distance.
//     Centring on u makes |x'_v|^2 ~= d(u,v) = v.dist, so the band is
//     ~0.05% of the threshold.  tools/ubench/gram_tc.cu measured
//     7.9e-6 |a||b| on d = 960 rows.
//  4. Epilogue: rows are ranked by (dist, id) (the reference's sort,
//     builder.cpp:47), occluder / band bit masks are built per row in list
//     order, band comparisons the walk can reach are decided exactly (a
//     quad per pair, quad.cuh), then the walk: one thread per list finds
//     the kept set on bit masks, and every row derives its own pair_checks /
//     flag_skips / removed / touched counts and output in parallel.
//  5. A removed v is redirected to its occluder w as a record whose distance
//     is PENDING (common.cuh kPendBits): the apply phase merges it by id
//     (has_target, builder.cpp:22-26), and the exact l2_sq(v, w) is produced
//     by item 1 when w's list is next scanned (every inserted entry is
//     fresh, so that list is active in the next pass).  Lists scanned by the
//     other kernels, reverse phases and every caller-visible read
//     materialise pending distances first (build.cu materialize_pending).
//
// Lists are packed into 128-row tiles by size class (8 lists of <= 16 rows,
// 4 of <= 32, 2 of <= 64, 1 of <= 128).  One persistent CTA per SM:
//   warps 0-7   producers: rows -> centre -> bf16 hi/lo -> SW128 smem stages,
//               exact distances of the rows
//   warp 12     MMA issuer (one thread): 12 tcgen05.mma per 64-wide k chunk
//   warps 8-11  epilogue: TMEM -> ranks -> masks -> band pairs -> walks
// with mbarrier rings between them (4 operand stages, 2 TMEM accumulators).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ctx.hpp"
#include "quad.cuh"
#include "scan.cuh"
#include "tc.cuh"

namespace rnndg {

namespace {

constexpr int kGP = 8;  // producer warps
constexpr int kGE = 4;  // epilogue warps (one per TMEM lane quarter)
constexpr int kGThreads = 32 * (kGP + kGE + 1);
constexpr int kMmaWarp = kGP + kGE;
constexpr int kNS = 4;                    // operand stages
constexpr uint32_t kTileBytes = 16384;    // 128 rows x 64 bf16
constexpr uint32_t kTmemCols = 256;       // two 128-column fp32 accumulators
constexpr uint32_t kChunk = 64;           // k elements per stage
constexpr uint32_t kAQ = 1024;            // band comparisons resolved per round

// RNNDG_TRACE: cycles per role / phase, summed over CTAs (prof[...])
enum GramProf : int {
  kPfProdWait = 0,  // producers waiting for a free operand stage
  kPfProdTotal,     // producer loop
  kPfEpiWait,       // epilogue waiting for an accumulator
  kPfMask,          // ranks + TMEM -> masks
  kPfAmb,           // band comparisons (exact)
  kPfWalk,          // walks + outputs
  kPfEpiTotal,
  kPfAmbPairs,      // band comparisons evaluated
  kPfTiles,
  kPfNum
};

struct GramArgs {
  const uint32_t* gq;  // class queues gq[c * nv + i] (local vertex ids)
  const unsigned long long* ctr_in;
  unsigned int* work;  // work[6]: next tile (work[4] is the hub kernel's)
  uint64_t nv, v0;
  const uint64_t* off;
  const uint32_t* cnt;
  uint64_t* keys;
  Row row;
  uint32_t nch;
  uint32_t* post_cnt;
  uint32_t* pend_src;
  uint64_t* pend_key;
  unsigned long long* bcnt;
  unsigned long long* ctr;
  float eps_rel;  // band half-width per unit of G_vv + G_ww
  unsigned long long* prof;  // kPfNum slots, or null
};

struct GramMeta {  // one per accumulator stage
  int tile;        // -1: no more tiles
  uint32_t cls, nl, first;
  uint32_t lu[8];
  uint32_t lU[8];
  uint64_t lbase[8];
  uint64_t key[128];  // storage order; pending distances filled by the producers
  uint32_t rid[128];  // row (global id); kNone for padding rows
  uint32_t cid[128];  // centre row: the list's own vertex (global id)
};

struct GramSmem {
  uint8_t stage[kNS][2][kTileBytes];  // hi, lo; at the 1024-aligned base
  GramMeta meta[2];
  float diag[128];
  uint32_t occ[128][4];  // by list position: occluders (bit = position)
  uint32_t aq[kAQ];      // band pairs: tile row t << 8 | tile row j
  uint64_t kept[8][2];   // per list: kept positions
  uint64_t fmask[8][2];  //           fresh positions
  uint32_t tch[8][4];    //           touched positions
  uint8_t pos[128];      // tile row -> list position (tile index space)
  uint8_t perm[128];     // list position -> tile row
  uint32_t naq;
  uint32_t tmem_base;
  uint64_t full[kNS], empty[kNS], acc_full[2], acc_empty[2], meta_full[2], meta_empty[2],
      keys_full[2];
};

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// one lane polls the mbarrier, the warp follows
__device__ __forceinline__ void warp_wait(uint64_t* b, uint32_t parity) {
  if (lane_id() == 0) tc::mbar_wait(b, parity);
  __syncwarp();
}

__device__ __forceinline__ void set_bit4(uint32_t (&w)[4], uint32_t pos) {
  const uint32_t b = 1u << (pos & 31u), k = pos >> 5;
  w[0] |= k == 0 ? b : 0u;
  w[1] |= k == 1 ? b : 0u;
  w[2] |= k == 2 ? b : 0u;
  w[3] |= k == 3 ? b : 0u;
}

// bits [0, t) of a 128-bit mask held as two u64 words
__device__ __forceinline__ uint64_t below_lo(uint32_t t) {
  return t >= 64 ? ~0ull : ((1ull << t) - 1ull);
}
__device__ __forceinline__ uint64_t below_hi(uint32_t t) {
  return t <= 64 ? 0ull : ((1ull << (t - 64)) - 1ull);
}
__device__ __forceinline__ uint64_t bit_lo(uint32_t t) { return t < 64 ? (1ull << t) : 0ull; }
__device__ __forceinline__ uint64_t bit_hi(uint32_t t) {
  return t < 64 ? 0ull : (1ull << (t - 64));
}

__global__ void __launch_bounds__(kGThreads, 1) k_scan_gram(GramArgs g) {
  extern __shared__ __align__(1024) uint8_t gram_raw[];
  // 1024-byte aligned (SW128 operand tiles); offset arithmetic on the shared
  // array keeps every access an LDS/STS rather than a generic LD/ST
  GramSmem& sm = *reinterpret_cast<GramSmem*>(
      gram_raw + ((1024u - (tc::smem_u32(gram_raw) & 1023u)) & 1023u));
  const uint32_t tid = threadIdx.x, wid = tid >> 5, lane = lane_id();
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&sm.full[s], 32 * kGP);
      tc::mbar_init(&sm.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&sm.acc_full[a], 1);
      tc::mbar_init(&sm.acc_empty[a], kGE);
      tc::mbar_init(&sm.meta_full[a], 1);
      tc::mbar_init(&sm.meta_empty[a], 1);
      tc::mbar_init(&sm.keys_full[a], 32 * kGP);
    }
    tc::mbar_fence_init();
  }
  if (wid == kMmaWarp) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const Row row = g.row;

  if (wid < kGP) {
    // ------------------------------------------------------------ producers
    const uint32_t p = tid;
    const uint32_t c8 = p & 7u, r0 = p >> 3, hb = c8 >> 2;
    // the d % 4 tail follows the chain blocks (quad.cuh layout): its unit
    const uint32_t tail_e = 32u * row.nblk, tail_c8 = (tail_e % kChunk) / 8u;
    uint32_t s = 0, ps = 0;
    long long pf_wait = 0;
    const long long pf_t0 = clock64();
    for (uint32_t it = 0;; ++it) {
      const uint32_t a = it & 1u, pa = (it >> 1) & 1u;
      GramMeta& m = sm.meta[a];
      if (p == 0) {
        tc::mbar_wait(&sm.meta_empty[a], pa ^ 1u);
        uint32_t rem = atomicAdd(g.work + 6, 1u);
        int tile = -1;
        for (int c = 3; c >= 0; --c) {  // longest lists first
          const uint32_t nc = uint32_t(g.ctr_in[kGram0 + c]);
          const uint32_t P = 8u >> c;
          const uint32_t tiles = (nc + P - 1) / P;
          if (rem < tiles) {
            tile = int(rem);
            m.cls = uint32_t(c);
            m.first = rem * P;
            m.nl = min(P, nc - rem * P);
            break;
          }
          rem -= tiles;
        }
        m.tile = tile;
      }
      named_bar(1, 32 * kGP);
      if (m.tile < 0) {
        if (p == 0) tc::mbar_arrive(&sm.meta_full[a]);
        break;
      }
      const uint32_t cls = m.cls, nl = m.nl;
      if (p < nl) {
        const uint32_t u = g.gq[uint64_t(cls) * g.nv + m.first + p];
        m.lu[p] = u;
        m.lbase[p] = g.off[u];
        m.lU[p] = g.cnt[u];
      }
      named_bar(1, 32 * kGP);
      if (p < 128) {
        const uint32_t R = 16u << cls, sl = p / R, j = p % R;
        if (sl < nl && j < m.lU[sl]) {
          const uint64_t k = g.keys[m.lbase[sl] + j];
          m.key[p] = k;
          m.rid[p] = key_id(k);
          m.cid[p] = uint32_t(g.v0 + m.lu[sl]);
        } else {
          m.key[p] = kTomb;
          m.rid[p] = kNone;
          m.cid[p] = kNone;
        }
      }
      named_bar(1, 32 * kGP);
      if (p == 0) tc::mbar_arrive(&sm.meta_full[a]);
      // operand chunks: thread p covers 16-byte unit c8 of rows r0 + 32 i
      uint32_t rid[4], cid[4];
      float sch[4] = {0.f, 0.f, 0.f, 0.f};  // chain (c8 & 3) of row i, in the hb = 0 lane
      float stl[4][3] = {};                  // squared tail terms (tail unit's lane)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        rid[i] = m.rid[r0 + 32 * i];
        cid[i] = m.cid[r0 + 32 * i];
      }
      for (uint32_t ch = 0; ch < g.nch; ++ch) {
        const uint32_t e0 = ch * kChunk + c8 * 8u;
        const bool in = e0 < row.stride;
        const bool is_tail = row.ntail && e0 == tail_e;
        float xv[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (in && rid[i] != kNone) {
            ld256<true>(row.xp + uint64_t(rid[i]) * row.stride + e0, xv[i]);
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) xv[i][e] = 0.f;
          }
        }
        {
          const long long w0 = clock64();
          warp_wait(&sm.empty[s], ps ^ 1u);
          pf_wait += clock64() - w0;
        }
        uint8_t* H = sm.stage[s][0];
        uint8_t* L = sm.stage[s][1];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          // the centre row is shared by the list's rows: L1 hits after the first
          float cv[8];
          if (in && rid[i] != kNone) {
            ld256w(row.xp + uint64_t(cid[i]) * row.stride + e0, cv);
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) cv[e] = 0.f;
          }
          float t[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) t[e] = __fsub_rn(xv[i][e], cv[e]);
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) tc::split2(t[2 * e], t[2 * e + 1], h[e], l[e]);
          const uint32_t off = tc::sw128_off(r0 + 32 * i, c8);
          *reinterpret_cast<uint4*>(H + off) = make_uint4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<uint4*>(L + off) = make_uint4(l[0], l[1], l[2], l[3]);
          // exact l2_sq(x, u): chain k = c8 & 3 of block 2ch + hb; the
          // running sum passes hb = 0 -> hb = 1 -> hb = 0 (block order)
          float sq[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) sq[e] = __fmul_rn(t[e], t[e]);
          if (is_tail) {
#pragma unroll
            for (int e = 0; e < 3; ++e) stl[i][e] = sq[e];
#pragma unroll
            for (int e = 0; e < 8; ++e) sq[e] = 0.f;  // +0: exact no-op on a chain
          }
          float acc = sch[i];
          if (hb == 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = __fadd_rn(acc, sq[e]);
          }
          const float mid = __shfl_up_sync(0xffffffffu, acc, 4);
          if (hb == 1) {
            acc = mid;
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = __fadd_rn(acc, sq[e]);
          }
          const float back = __shfl_down_sync(0xffffffffu, acc, 4);
          if (hb == 0) sch[i] = back;
        }
        tc::fence_async_smem();
        tc::mbar_arrive(&sm.full[s]);
        if (++s == kNS) {
          s = 0;
          ps ^= 1u;
        }
      }
      // ((s0 + s1) + (s2 + s3)) at the row group's lane 0, then the tail in
      // order (metric.hpp:15-24); pending distances become exact keys
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float pr = __fadd_rn(sch[i], __shfl_down_sync(0xffffffffu, sch[i], 1));
        float tot = __fadd_rn(pr, __shfl_down_sync(0xffffffffu, pr, 2));
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          const float te = __shfl_down_sync(0xffffffffu, stl[i][e], tail_c8);
          if (uint32_t(e) < row.ntail) tot = __fadd_rn(tot, te);
        }
        const uint32_t r = r0 + 32 * i;
        if (c8 == 0 && rid[i] != kNone) {
          const uint64_t k = m.key[r];
          if (key_pending(k)) m.key[r] = make_key(tot, rid[i], key_fresh(k));
        }
      }
      tc::mbar_arrive(&sm.keys_full[a]);
    }
    if (g.prof && p == 0) {
      atomicAdd(&g.prof[kPfProdWait], (unsigned long long)pf_wait);
      atomicAdd(&g.prof[kPfProdTotal], (unsigned long long)(clock64() - pf_t0));
    }
  } else if (wid == kMmaWarp) {
    // ----------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = tc::idesc_bf16_f32<128, 128>();
    uint32_t s = 0, ps = 0;
    for (uint32_t it = 0;; ++it) {
      const uint32_t a = it & 1u, pa = (it >> 1) & 1u;
      warp_wait(&sm.meta_full[a], pa);
      if (sm.meta[a].tile < 0) break;
      warp_wait(&sm.acc_empty[a], pa ^ 1u);
      tc::tc_fence_after();
      const uint32_t d = tmem + a * 128u;
      for (uint32_t ch = 0; ch < g.nch; ++ch) {
        warp_wait(&sm.full[s], ps);
        tc::tc_fence_after();
        if (lane == 0) {
          const uint32_t ha = tc::smem_u32(sm.stage[s][0]), la = tc::smem_u32(sm.stage[s][1]);
#pragma unroll
          for (uint32_t k = 0; k < kChunk / 16; ++k) {
            const uint64_t dh = tc::sw128_desc(ha + 32 * k), dl = tc::sw128_desc(la + 32 * k);
            tc::mma_bf16(d, dh, dh, idesc, (ch | k) ? 1u : 0u);
            tc::mma_bf16(d, dh, dl, idesc, 1u);
            tc::mma_bf16(d, dl, dh, idesc, 1u);
          }
          tc::mma_commit(&sm.empty[s]);
        }
        __syncwarp();
        if (++s == kNS) {
          s = 0;
          ps ^= 1u;
        }
      }
      if (lane == 0) tc::mma_commit(&sm.acc_full[a]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const uint32_t e = tid - 32 * kGP, ew = e >> 5;  // tile row e = TMEM lane e
    unsigned long long removed = 0, checks = 0, skips = 0, touched = 0, namb = 0;
    long long pf[kPfNum] = {};
    const long long pe0 = clock64();
    for (uint32_t it = 0;; ++it) {
      const uint32_t a = it & 1u, pa = (it >> 1) & 1u;
      long long tp = clock64();
      warp_wait(&sm.meta_full[a], pa);
      GramMeta& m = sm.meta[a];
      if (m.tile < 0) break;
      warp_wait(&sm.acc_full[a], pa);
      warp_wait(&sm.keys_full[a], pa);
      tc::tc_fence_after();
      {
        const long long tq = clock64();
        pf[kPfEpiWait] += tq - tp;
        tp = tq;
      }
      const uint32_t tb = tmem + a * 128u + ((32u * ew) << 16);
      const uint32_t cls = m.cls, R = 16u << cls, sl_e = e / R, s0 = sl_e * R;
      const uint32_t nl = m.nl;
      const uint32_t Ue = sl_e < nl ? m.lU[sl_e] : 0u;
      const bool real = e - s0 < Ue;
      float v[32];
      tc::tmem_ld32(tb + 32u * ew, v);  // the warp's diagonal block
      float dg = v[0];
#pragma unroll
      for (int j = 1; j < 32; ++j)
        if (uint32_t(j) == lane) dg = v[j];
      sm.diag[e] = dg;
      const uint64_t ke = m.key[e];
      // list position of row e: its rank by (dist, id) within its list
      uint32_t pe = e;
      if (real) {
        uint32_t r = 0;
        for (uint32_t j = s0; j < s0 + Ue; ++j) r += m.key[j] < ke ? 1u : 0u;
        pe = s0 + r;
        sm.perm[pe] = uint8_t(e);
      }
      sm.pos[e] = uint8_t(pe);
      if (e == 0) sm.naq = 0;
      if (e < 8) sm.tch[e][0] = sm.tch[e][1] = sm.tch[e][2] = sm.tch[e][3] = 0u;
      named_bar(2, 32 * kGE);
      // occluder / band masks of row e over the rows ahead of it in its list
      const float thr = key_dist(ke);
      uint32_t oc[4] = {0u, 0u, 0u, 0u}, am[4] = {0u, 0u, 0u, 0u};
      {
        const uint32_t lo = ((32u * ew) & ~(R - 1u)) >> 5;
        const uint32_t hi = ((32u * ew + 31u) | (R - 1u)) >> 5;
        for (uint32_t cb = lo; cb <= hi; ++cb) {
          tc::tmem_ld32(tb + 32u * cb, v);
          if (!real) continue;
#pragma unroll 4
          for (int jj = 0; jj < 32; ++jj) {
            const uint32_t j = 32u * cb + uint32_t(jj);
            if (j - s0 >= Ue || j == e) continue;
            if (!(m.key[j] < ke)) continue;
            const float dj = sm.diag[j];
            const float sn = __fadd_rn(fabsf(dg), fabsf(dj));
            const float dd = __fsub_rn(__fadd_rn(dg, dj), __fmul_rn(2.f, v[jj]));
            const float eps = __fadd_rn(__fmul_rn(sn, g.eps_rel), 1e-25f);
            const uint32_t pj = sm.pos[j];
            if (__fadd_rn(dd, eps) < thr)
              set_bit4(oc, pj);
            else if (!(__fsub_rn(dd, eps) > thr))
              set_bit4(am, pj);
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.acc_empty[a]);
      if (real) {
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) sm.occ[pe][w4] = oc[w4];
      }
      {
        const long long tq = clock64();
        pf[kPfMask] += tq - tp;
        tp = tq;
      }
      // band comparisons a walk may reach (not old/old) decided exactly, a
      // quad per pair, in rounds of at most kAQ pairs
      {
        const bool fe = key_fresh(ke);
        bool more = real;
        uint32_t w4 = 0;
        for (;;) {
          if (more) {
            more = false;
            for (; w4 < 4; ++w4) {
              uint32_t q = w4 == 0 ? am[0] : (w4 == 1 ? am[1] : (w4 == 2 ? am[2] : am[3]));
              while (q) {
                const uint32_t b = uint32_t(__ffs(q)) - 1u;
                const uint32_t j = sm.perm[32u * w4 + b];
                if (fe || key_fresh(m.key[j])) {  // old/old pairs are never compared
                  const uint32_t qi = atomicAdd(&sm.naq, 1u);
                  if (qi >= kAQ) {
                    more = true;
                    break;
                  }
                  sm.aq[qi] = (e << 8) | j;
                }
                q &= q - 1u;
              }
              if (w4 == 0) am[0] = q;
              if (w4 == 1) am[1] = q;
              if (w4 == 2) am[2] = q;
              if (w4 == 3) am[3] = q;
              if (more) break;
            }
          }
          named_bar(2, 32 * kGE);
          const uint32_t na = min(sm.naq, kAQ);
          if (na == 0) break;  // uniform: every thread read the same count
          pf[kPfAmbPairs] += (e == 0) ? na : 0u;
          namb += (e == 0) ? na : 0u;
          for (uint32_t b0 = 8u * ew; b0 < na; b0 += 8u * kGE) {
            const uint32_t qi = b0 + (lane >> 2);
            const uint32_t rec = sm.aq[qi < na ? qi : b0];
            const uint32_t t = rec >> 8, j = rec & 0xFFu;
            const float d = quad_l2<false>(row.xp + uint64_t(m.rid[t]) * row.stride,
                                           row.xp + uint64_t(m.rid[j]) * row.stride, lane & 3u,
                                           row.nblk, row.ntail);
            if (qi < na && (lane & 3u) == 0 && key_dist(m.key[t]) >= d) {
              const uint32_t pj = sm.pos[j];
              atomicOr(&sm.occ[sm.pos[t]][pj >> 5], 1u << (pj & 31u));
            }
          }
          named_bar(2, 32 * kGE);
          if (e == 0) sm.naq = 0;
          named_bar(2, 32 * kGE);
        }
      }
      {
        const long long tq = clock64();
        pf[kPfAmb] += tq - tp;
        tp = tq;
      }
      // walk, part 1: the kept set of each list, one thread per list
      // (lists spread over the four warps), on the occluder bits only
      const uint64_t* occ64 = reinterpret_cast<const uint64_t*>(&sm.occ[0][0]);
      {
        const uint32_t wsl = (e & 31u) * kGE + ew;
        if ((e & 31u) < 2 && wsl < nl) {
          const uint32_t b0 = wsl * R, U = m.lU[wsl];
          uint64_t k0 = 0, k1 = 0, f0 = 0, f1 = 0;
          for (uint32_t t = b0; t < b0 + U; ++t) {
            const bool f = key_fresh(m.key[sm.perm[t]]);
            const uint64_t c0 = f ? k0 : (k0 & f0), c1 = f ? k1 : (k1 & f1);
            const uint64_t tb0 = bit_lo(t), tb1 = bit_hi(t);
            if (((c0 & occ64[2 * t]) | (c1 & occ64[2 * t + 1])) == 0ull) {
              k0 |= tb0;
              k1 |= tb1;
            }
            if (f) {
              f0 |= tb0;
              f1 |= tb1;
            }
          }
          sm.kept[wsl][0] = k0;
          sm.kept[wsl][1] = k1;
          sm.fmask[wsl][0] = f0;
          sm.fmask[wsl][1] = f1;
          g.post_cnt[m.lu[wsl]] = uint32_t(__popcll(k0) + __popcll(k1));
        }
      }
      named_bar(2, 32 * kGE);
      // walk, part 2: position e's own checks / skips and its output
      if (real) {
        const uint32_t t = e;  // the list position handled by this thread
        const uint32_t te = sm.perm[t];
        const uint64_t kt = m.key[te];
        const bool f = key_fresh(kt);
        const uint64_t K0 = sm.kept[sl_e][0] & below_lo(t), K1 = sm.kept[sl_e][1] & below_hi(t);
        const uint64_t F0 = sm.fmask[sl_e][0], F1 = sm.fmask[sl_e][1];
        const uint64_t c0 = f ? K0 : (K0 & F0), c1 = f ? K1 : (K1 & F1);
        const uint64_t x0 = c0 & occ64[2 * t], x1 = c1 & occ64[2 * t + 1];
        uint64_t tc0, tc1;
        if (x0 | x1) {
          // first occluder in list order: every kept entry before it was
          // checked (or skipped as old/old) and passed
          const uint32_t oi = x0 ? uint32_t(__ffsll(x0)) - 1u : 63u + uint32_t(__ffsll(x1));
          const uint64_t bl0 = below_lo(oi), bl1 = below_hi(oi);
          checks += 1u + __popcll(c0 & bl0) + __popcll(c1 & bl1);
          skips += __popcll(K0 & ~c0 & bl0) + __popcll(K1 & ~c1 & bl1);
          tc0 = (c0 & bl0) | bit_lo(oi) | bit_lo(t);
          tc1 = (c1 & bl1) | bit_hi(oi) | bit_hi(t);
          ++removed;
          // redirect (w, v, pending distance), by the candidate's slot
          const uint32_t w_id = m.rid[sm.perm[oi]];
          const uint64_t slot = m.lbase[sl_e] + (te - s0);
          g.pend_src[slot] = w_id;
          g.pend_key[slot] = pending_key(m.rid[te]);
          if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
        } else {
          const uint32_t nc = __popcll(c0) + __popcll(c1);
          checks += nc;
          skips += __popcll(K0 & ~c0) + __popcll(K1 & ~c1);
          tc0 = c0 | (nc ? bit_lo(t) : 0ull);
          tc1 = c1 | (nc ? bit_hi(t) : 0ull);
          // kept, flagged old (builder.cpp:68), at its rank among the kept
          g.keys[m.lbase[sl_e] + (__popcll(K0) + __popcll(K1))] = kt & ~1ull;
        }
        if (uint32_t(tc0)) atomicOr(&sm.tch[sl_e][0], uint32_t(tc0));
        if (uint32_t(tc0 >> 32)) atomicOr(&sm.tch[sl_e][1], uint32_t(tc0 >> 32));
        if (uint32_t(tc1)) atomicOr(&sm.tch[sl_e][2], uint32_t(tc1));
        if (uint32_t(tc1 >> 32)) atomicOr(&sm.tch[sl_e][3], uint32_t(tc1 >> 32));
      }
      named_bar(2, 32 * kGE);
      if (e < nl)
        touched += __popc(sm.tch[e][0]) + __popc(sm.tch[e][1]) + __popc(sm.tch[e][2]) +
                   __popc(sm.tch[e][3]);
      named_bar(2, 32 * kGE);
      if (e == 0) tc::mbar_arrive(&sm.meta_empty[a]);
      pf[kPfWalk] += clock64() - tp;
      pf[kPfTiles] += e == 0 ? 1 : 0;
    }
    if (g.prof && e == 0) {
      pf[kPfEpiTotal] = clock64() - pe0;
      for (int i = 2; i < kPfNum; ++i) atomicAdd(&g.prof[i], (unsigned long long)pf[i]);
    }
    for (int o = 16; o; o >>= 1) {
      removed += __shfl_xor_sync(0xffffffffu, removed, o);
      checks += __shfl_xor_sync(0xffffffffu, checks, o);
      skips += __shfl_xor_sync(0xffffffffu, skips, o);
      touched += __shfl_xor_sync(0xffffffffu, touched, o);
      namb += __shfl_xor_sync(0xffffffffu, namb, o);
    }
    if (lane == 0) {
      if (removed) atomicAdd(&g.ctr[kRemoved], removed);
      if (checks) atomicAdd(&g.ctr[kPairChecks], checks);
      if (skips) atomicAdd(&g.ctr[kFlagSkips], skips);
      if (touched) atomicAdd(&g.ctr[kTouched], touched);
      if (namb) {
        atomicAdd(&g.ctr[kGramAmb], namb);
        atomicAdd(&g.ctr[kGramExact], namb);
        atomicAdd(&g.ctr[kEvalPairs], namb);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (wid == kMmaWarp) tc::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

// 0 = off (every short list on k_scan_spec); otherwise lists of at most
// this many entries (<= 128) take the Gram-filtered walk.  Default off until
// the kernel beats k_scan_spec end to end (C3 1M: 2.51 s on vs 1.94 s off).
uint32_t gram_cap() {
  static const uint32_t v = [] {
    const char* e = std::getenv("RNNDG_GRAM");
    const int x = e ? std::atoi(e) : 0;
    return uint32_t(x <= 0 ? 0 : (x > 128 ? 128 : x));
  }();
  return v;
}

void launch_gram(rnndg_ctx* c, unsigned int* work) {
  const ScanConfig cfg = scan_config(c);
  GramArgs a{};
  a.gq = c->gram_q.p;
  a.ctr_in = c->counters.p;
  a.work = work;
  a.nv = c->nv;
  a.v0 = c->v0;
  a.off = c->off.p;
  a.cnt = c->cnt.p;
  a.keys = c->key.p;
  a.row = Row{c->xp.p, cfg.stride, cfg.nblk, cfg.ntail};
  a.nch = (cfg.stride + kChunk - 1) / kChunk;
  a.post_cnt = c->post_cnt.p;
  a.pend_src = c->pend_src.p;
  a.pend_key = c->pend_key.p;
  a.bcnt = c->partitioned ? nullptr : c->bcnt.p;
  a.ctr = c->counters.p;
  a.prof = nullptr;
  if (c->trace) {
    a.prof = c->gram_prof.ensure(kPfNum);
    RNNDG_CUDA(cudaMemsetAsync(a.prof, 0, kPfNum * sizeof(unsigned long long), c->stream));
  }
  // error band of the filter (header): 1.25 x the bound for K = nch * 64,
  // two truncations per MMA instruction (3K/16 instructions per entry)
  const double K = double(a.nch) * kChunk;
  const double beta = 2.0 * (3.0 * K / 16.0) * 0x1p-23 + 0x1p-21 + 3.1 * 0x1p-16;
  a.eps_rel = float(1.25 * (2.0 * beta + 2.0 * (K / 4.0 + 3.0) * 0x1p-24 + 1e-6));
  const size_t smem = sizeof(GramSmem) + 1024;
  static unsigned long long attr_set = 0;  // per device
  if (!(attr_set >> (c->device & 63) & 1ull)) {
    RNNDG_CUDA(cudaFuncSetAttribute(k_scan_gram, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
    attr_set |= 1ull << (c->device & 63);
  }
  RNNDG_LAUNCH(c, k_scan_gram, unsigned(sm_count(c)), kGThreads, smem, a);
}

// RNNDG_TRACE: where the Gram kernel's cycles went in the last pass
void gram_trace(rnndg_ctx* c) {
  if (!gram_cap() || !c->gram_prof.p) return;
  unsigned long long h[kPfNum];
  RNNDG_CUDA(cudaMemcpy(h, c->gram_prof.p, sizeof(h), cudaMemcpyDeviceToHost));
  const double ctas = double(sm_count(c));
  auto mc = [&](int i) { return double(h[i]) / ctas * 1e-6; };  // Mcycles per CTA
  std::fprintf(stderr,
               "[rnndg] gram: tiles=%llu prod %.2f Mcyc (wait %.2f) | epi %.2f Mcyc: wait %.2f "
               "mask %.2f amb %.2f (%llu pairs) walk %.2f\n",
               h[kPfTiles], mc(kPfProdTotal), mc(kPfProdWait), mc(kPfEpiTotal), mc(kPfEpiWait),
               mc(kPfMask), mc(kPfAmb), h[kPfAmbPairs], mc(kPfWalk));
}

}  // namespace rnndg
