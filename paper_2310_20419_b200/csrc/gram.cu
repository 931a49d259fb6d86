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
// 4 of <= 32, 2 of <= 64, 1 of <= 128).  Two persistent 256-thread CTAs per
// SM, each with its own 128-column TMEM accumulator, alternate between two
// phases per tile, so one CTA's epilogue overlaps the other's streaming:
//   stream    warp w owns tile rows 16w .. 16w+15 (one list in every size
//             class, so one centre row): their 64-element chunks (two
//             chain blocks, 256 B per row) arrive by cp.async in a 3-stage
//             ring and are converted IN PLACE into two SWIZZLE_64B bf16
//             hi/lo operand sub-tiles (each warp's raw rows sit exactly
//             where its own operand rows go); each lane keeps the chain sum
//             of its (row, chain) pairs; the warp arrives on the stage's
//             mbarrier and warp 0 issues the chunk's 12 MMAs once all eight
//             arrived -- no CTA-wide barrier per chunk
//   epilogue  TMEM -> ranks -> masks -> band pairs (a warp per pair) ->
//             walks -> outputs, on all 8 warps (two per TMEM lane quarter,
//             splitting the columns)
// (A warp-specialised single-CTA version, producers / MMA / epilogue warps
// with mbarrier rings, ran its epilogue on 4 warps only and was latency-bound
// there: 2.5 s per C3 1M build.)
#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ctx.hpp"
#include "quad.cuh"
#include "scan.cuh"
#include "tc.cuh"

namespace rnndg {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kCtasPerSm = 2;
constexpr uint32_t kChunk = 64;      // k elements per ring stage: two chain blocks
constexpr uint32_t kSub = 32;        // k elements per SW64 operand sub-tile
constexpr int kNR = 3;               // ring stages (raw fp32 chunk -> bf16 operands in place)
constexpr int kLA = 1;               // chunks in flight ahead of the one being converted
constexpr uint32_t kOpBytes = 8192;  // 128 rows x 32 bf16 (SWIZZLE_64B)
constexpr uint32_t kTmemCols = 256;  // HH^T at columns 0..127, HL^T at 128..255
constexpr uint32_t kAQ = 512;        // band comparisons resolved per round

// RNNDG_TRACE: cycles per phase (thread 0 of every CTA), summed over CTAs
enum GramProf : int {
  kPfStream = 0,  // tile set-up + chunk loop
  kPfMmaWait,     // waiting for the last MMAs of the tile
  kPfMask,        // ranks + TMEM -> masks
  kPfAmb,         // band comparisons (exact)
  kPfWalk,        // walks + outputs
  kPfTotal,
  kPfAmbPairs,    // band comparisons evaluated
  kPfTiles,
  kPfIssue,     // stream, warp 1: next chunk's copies (incl. waiting for a free stage)
  kPfCpWait,    //   waiting for this chunk's copies
  kPfConv,      //   conversion .. arrival
  kPfMmaIssue,  // warp 0: waiting for all warps' chunk, then issuing the MMAs
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
  int l2pf;                  // bulk L2 prefetch of a tile's rows at its start
  float fast_rel;            // band of warp_l2_fast against rnnd::l2_sq (relative)
};

struct GramSmem {
  // ring stage: a 64-element chunk of every row, raw fp32, converted in
  // place into two SW64 operand sub-tiles (sub-tile s: hi at [16K s, +8K),
  // lo at [16K s + 8K, +8K)).  Warp w's 16 raw rows (256 B each) sit in the
  // four 1 KB pieces its own operand rows occupy (rows 4r..4r+3 in piece r:
  // sub-tile r / 2, hi for even r, lo for odd), so a warp converts in place
  // without touching another warp's data.  1024-aligned base; the
  // epilogue's pair scratch reuses it.
  uint8_t ring[kNR][4 * kOpBytes];
  float craw[kNR][kWarps][kChunk];  // centre row of each warp's list
  uint64_t key[128];             // storage order; pending distances filled in
  uint32_t rid[128];             // row (global id); kNone for padding rows
  uint32_t lu[8], lU[8];
  uint64_t lbase[8];
  float diag[128];
  uint32_t rank[128];
  uint32_t occ[128][4];          // by list position: occluders (bit = position)
  uint32_t aq[kAQ];              // band pairs: tile row t << 8 | tile row j
  uint64_t kept[8][2];           // per list: kept positions
  uint64_t fmask[8][2];          //           fresh positions
  uint32_t tch[8][4];            //           touched positions
  uint8_t pos[128];              // tile row -> list position (tile index space)
  uint8_t perm[128];             // list position -> tile row
  int tile;
  uint32_t cls, nl, first, naq, tmem_base;
  uint64_t st_full[kNR], st_free[kNR], acc_ready;
};

static_assert(offsetof(GramSmem, craw) == offsetof(GramSmem, ring) + sizeof(GramSmem::ring),
              "the epilogue scratch spans ring and craw");
static_assert(sizeof(GramSmem::ring) + sizeof(GramSmem::craw) >=
                  (128u * 129u + kWarps * 1024u) * sizeof(float),
              "staged HL^T + pair scratch must fit the idle ring");

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void set_bit4(uint32_t (&w)[4], uint32_t pos) {
  const uint32_t b = 1u << (pos & 31u), k = pos >> 5;
  w[0] |= k == 0 ? b : 0u;
  w[1] |= k == 1 ? b : 0u;
  w[2] |= k == 2 ? b : 0u;
  w[3] |= k == 3 ? b : 0u;
}

// bits [0, t) / bit t of a 128-bit mask held as two u64 words
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

// exact rnnd::l2_sq of rows ra, rb by one warp: every lane loads and squares
// its share of the differences (all loads in flight at once) into `sq`, then
// lanes 0..3 sum the four chains in the reference's order (metric.hpp:15-24)
__device__ __forceinline__ float warp_l2(const Row& row, uint32_t ra, uint32_t rb, float* sq) {
  const uint32_t lane = lane_id();
  const float4* a = reinterpret_cast<const float4*>(row.xp + uint64_t(ra) * row.stride);
  const float4* b = reinterpret_cast<const float4*>(row.xp + uint64_t(rb) * row.stride);
  const uint32_t n4 = row.stride / 4;
#pragma unroll 4
  for (uint32_t i = lane; i < n4; i += 32) {
    const float4 x = __ldg(a + i), y = __ldg(b + i);
    const float t0 = __fsub_rn(x.x, y.x), t1 = __fsub_rn(x.y, y.y);
    const float t2 = __fsub_rn(x.z, y.z), t3 = __fsub_rn(x.w, y.w);
    reinterpret_cast<float4*>(sq)[i] =
        make_float4(__fmul_rn(t0, t0), __fmul_rn(t1, t1), __fmul_rn(t2, t2), __fmul_rn(t3, t3));
  }
  __syncwarp();
  float s = 0.f;
  if (lane < 4)
    for (uint32_t blk = 0; blk < row.nblk; ++blk) {
      const float* p = sq + 32 * blk + 8 * lane;
#pragma unroll
      for (int j = 0; j < 8; ++j) s = __fadd_rn(s, p[j]);
    }
  const float pr = __fadd_rn(s, __shfl_down_sync(0xffffffffu, s, 1));
  float tot = __fadd_rn(pr, __shfl_down_sync(0xffffffffu, pr, 2));
  if (lane == 0)
    for (uint32_t t = 0; t < row.ntail; ++t) tot = __fadd_rn(tot, sq[32 * row.nblk + t]);
  __syncwarp();
  return __shfl_sync(0xffffffffu, tot, 0);
}

// |x_a - x_b|^2 by a whole warp in any order: per-lane sequential sums of
// <= 4 ceil(stride / 128) squares, then a 5-level tree.  Relative error
// against the real value <= (4 ceil(stride/128) + 8) 2^-24 (launch_gram,
// GramArgs::fast_rel) -- far inside the Gram band, so only comparisons
// within ~3e-5 of the threshold still need the reference-ordered sum.
__device__ __forceinline__ float warp_l2_fast(const Row& row, uint32_t ra, uint32_t rb) {
  const uint32_t lane = lane_id();
  const float4* a = reinterpret_cast<const float4*>(row.xp + uint64_t(ra) * row.stride);
  const float4* b = reinterpret_cast<const float4*>(row.xp + uint64_t(rb) * row.stride);
  const uint32_t n4 = row.stride / 4;
  float s = 0.f;
#pragma unroll 4
  for (uint32_t i = lane; i < n4; i += 32) {
    const float4 x = __ldg(a + i), y = __ldg(b + i);
    const float t0 = __fsub_rn(x.x, y.x), t1 = __fsub_rn(x.y, y.y);
    const float t2 = __fsub_rn(x.z, y.z), t3 = __fsub_rn(x.w, y.w);
    s = __fadd_rn(s, __fmul_rn(t0, t0));
    s = __fadd_rn(s, __fmul_rn(t1, t1));
    s = __fadd_rn(s, __fmul_rn(t2, t2));
    s = __fadd_rn(s, __fmul_rn(t3, t3));
  }
  for (int o = 16; o; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}

__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_scan_gram(GramArgs g) {
  extern __shared__ __align__(1024) uint8_t gram_raw[];
  // 1024-byte aligned operand tiles; offset arithmetic on the shared array
  // keeps every access an LDS/STS rather than a generic LD/ST
  GramSmem& sm = *reinterpret_cast<GramSmem*>(
      gram_raw + ((1024u - (tc::smem_u32(gram_raw) & 1023u)) & 1023u));
  const uint32_t tid = threadIdx.x, wid = tid >> 5, lane = lane_id();
  if (tid == 0) {
    for (int st = 0; st < kNR; ++st) {
      tc::mbar_init(&sm.st_full[st], kWarps);
      tc::mbar_init(&sm.st_free[st], 1);
    }
    tc::mbar_init(&sm.acc_ready, 1);
    tc::mbar_fence_init();
  }
  if (wid == 0) tc::tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const Row row = g.row;
  constexpr uint32_t idesc256 = tc::idesc_bf16_f32<128, 256>();
  // epilogue mapping: TMEM lane quarter q, column half h; tile row e
  const uint32_t q = wid & 3u, h = wid >> 2, e = 32u * q + lane;
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0, namb = 0;
  long long pf[kPfNum] = {};
  const long long p0 = clock64();
  uint32_t gch = 0;  // chunks streamed so far (ring stage and phase)

  for (uint32_t it = 0;; ++it) {
    long long tp = clock64();
    // ------------------------------------------------------------ tile set-up
    if (tid == 0) {
      uint32_t rem = atomicAdd(g.work + 6, 1u);
      int tile = -1;
      for (int c = 3; c >= 0; --c) {  // longest lists first
        const uint32_t nc = uint32_t(g.ctr_in[kGram0 + c]);
        const uint32_t P = 8u >> c;
        const uint32_t tiles = (nc + P - 1) / P;
        if (rem < tiles) {
          tile = int(rem);
          sm.cls = uint32_t(c);
          sm.first = rem * P;
          sm.nl = min(P, nc - rem * P);
          break;
        }
        rem -= tiles;
      }
      sm.tile = tile;
    }
    __syncthreads();
    if (sm.tile < 0) break;
    const uint32_t cls = sm.cls, nl = sm.nl, R = 16u << cls;
    if (tid < nl) {
      const uint32_t u = g.gq[uint64_t(cls) * g.nv + sm.first + tid];
      sm.lu[tid] = u;
      sm.lbase[tid] = g.off[u];
      sm.lU[tid] = g.cnt[u];
    }
    __syncthreads();
    if (tid < 128) {
      const uint32_t sl = tid / R, j = tid % R;
      if (sl < nl && j < sm.lU[sl]) {
        const uint64_t k = g.keys[sm.lbase[sl] + j];
        sm.key[tid] = k;
        sm.rid[tid] = key_id(k);
      } else {
        sm.key[tid] = kTomb;
        sm.rid[tid] = kNone;
      }
    }
    if (tid < 8) sm.tch[tid][0] = sm.tch[tid][1] = sm.tch[tid][2] = sm.tch[tid][3] = 0u;
    __syncthreads();

    // --------------------------------------------------------------- stream
    // Warp w streams tile rows 16w .. 16w+15 -- one list per warp in every
    // size class, so one centre row -- on its own: cp.async of its rows into
    // its slice of the ring, conversion, an arrival on op_full.  Warp 0 also
    // issues the chunk's MMAs once all eight warps arrived.  No CTA-wide
    // barrier inside the chunk loop.
    const uint32_t wrow = 16u * wid;
    const uint32_t wlist = wrow / R;
    const uint32_t ctr_row = wlist < nl ? uint32_t(g.v0 + sm.lu[wlist]) : kNone;
    const uint32_t nch = g.nch;
    // whole rows into L2 up front: DRAM reads them page-contiguously, the
    // per-chunk cp.async then hit L2 (RNNDG_GRAM_L2PF=0 turns this off)
    if (g.l2pf && lane < 17) {
      const uint32_t rr = lane < 16 ? sm.rid[wrow + lane] : ctr_row;
      if (rr != kNone) prefetch_row_l2(row.xp + uint64_t(rr) * row.stride, row.stride * 4u);
    }
    // chunk ci of this tile is global chunk gch + ci: stage (gch + ci) % kNR,
    // use (gch + ci) / kNR.  16-byte cp.async: lane (row j = lane/16 + 2k,
    // piece lane%16), k = 0..7, and lanes 0-15 the centre row.  (One bulk
    // copy per row chunk instead ran 1.4x slower: TMA issue-bound.)
    const uint32_t cp_p = lane & 15u;
    uint32_t cprid[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) cprid[k] = sm.rid[wrow + (lane >> 4) + 2 * k];
    auto raw_row = [&](uint8_t* stage, uint32_t j) {  // warp's raw row j (256 B)
      const uint32_t r = j >> 2;
      return stage + ((r >> 1) << 14) + ((r & 1u) << 13) + (wid << 10) + ((j & 3u) << 8);
    };
    auto issue = [&](uint32_t ci) {
      if (ci < nch) {
        const uint32_t gi = gch + ci, st = gi % kNR, use = gi / kNR;
        // the MMAs of the stage's previous chunk are done with it
        if (lane == 0) tc::mbar_wait(&sm.st_free[st], (use & 1u) ^ 1u);
        __syncwarp();
        const uint32_t e0 = ci * kChunk + cp_p * 4u;
        if (e0 < row.stride) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (cprid[k] != kNone)
              cp_async16(raw_row(sm.ring[st], (lane >> 4) + 2 * k) + 16 * cp_p,
                         row.xp + uint64_t(cprid[k]) * row.stride + e0);
          if (lane < 16 && ctr_row != kNone)
            cp_async16(&sm.craw[st][wid][cp_p * 4], row.xp + uint64_t(ctr_row) * row.stride + e0);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (uint32_t k = 0; k < uint32_t(kLA); ++k) issue(k);
    // conversion: lane handles (row 16 wid + j, chain c) for p = lane + 32 i,
    // j = p / 4, c = p % 4: unit c of both 32-element blocks of the chunk,
    // so its chain sum runs in-lane in block order.  Padding rows convert
    // stale data (their Gram rows / columns are never read); elements past
    // the row stride are zeroed.
    const uint32_t cv_c = lane & 3u;
    float sch[2] = {0.f, 0.f};  // chain cv_c of the two rows
    float stl[2][3] = {};       // squared tail terms (unit 0 of block nblk)
    for (uint32_t ch = 0; ch < nch; ++ch) {
      long long c0 = clock64();
      issue(ch + kLA);
      long long c1 = clock64();
      cp_async_wait<kLA>();
      __syncwarp();  // this warp's copies of chunk ch landed
      long long c2 = clock64();
      pf[kPfIssue] += c1 - c0;
      pf[kPfCpWait] += c2 - c1;
      const uint32_t gi = gch + ch, st = gi % kNR, use = gi / kNR;
      uint8_t* stage = sm.ring[st];
      uint64_t t[2][2][4];  // [row item][block][pair]
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        const float4* cs = reinterpret_cast<const float4*>(&sm.craw[st][wid][32 * bb + cv_c * 8]);
        const float4 c0 = cs[0], c1 = cs[1];
        const uint64_t cp0 = tc::pk2(c0.x, c0.y), cp1 = tc::pk2(c0.z, c0.w);
        const uint64_t cp2 = tc::pk2(c1.x, c1.y), cp3 = tc::pk2(c1.z, c1.w);
        const bool in = ch * kChunk + 32u * bb + cv_c * 8u < row.stride;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const uint32_t j = (lane + 32u * i) >> 2;
          const float4* xs = reinterpret_cast<const float4*>(raw_row(stage, j) + 128 * bb + 32 * cv_c);
          const float4 x0 = xs[0], x1 = xs[1];
          t[i][bb][0] = tc::sub2(tc::pk2(x0.x, x0.y), cp0);
          t[i][bb][1] = tc::sub2(tc::pk2(x0.z, x0.w), cp1);
          t[i][bb][2] = tc::sub2(tc::pk2(x1.x, x1.y), cp2);
          t[i][bb][3] = tc::sub2(tc::pk2(x1.z, x1.w), cp3);
          if (!in) t[i][bb][0] = t[i][bb][1] = t[i][bb][2] = t[i][bb][3] = 0ull;
        }
      }
      __syncwarp();  // every lane read its raw data: the operands overwrite it
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint32_t r = wrow + ((lane + 32u * i) >> 2);
        const uint32_t off = tc::sw64_off(r, cv_c);
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          uint32_t hh[4], ll[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float a0, a1;
            tc::upk2(t[i][bb][k], a0, a1);
            tc::split2(a0, a1, hh[k], ll[k]);
          }
          uint8_t* sub = stage + 2 * kOpBytes * bb;
          *reinterpret_cast<uint4*>(sub + off) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
          *reinterpret_cast<uint4*>(sub + kOpBytes + off) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
          // exact l2_sq(x, u): chain cv_c of block 2 ch + bb; the d % 4 tail
          // (unit 0 of block nblk) is added after the chains are combined
          float q[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) tc::upk2(tc::sqr2(t[i][bb][k]), q[2 * k], q[2 * k + 1]);
          const uint32_t blk = 2 * ch + uint32_t(bb);
          if (blk < row.nblk) {
#pragma unroll
            for (int k = 0; k < 8; ++k) sch[i] = __fadd_rn(sch[i], q[k]);
          } else if (blk == row.nblk && cv_c == 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k) stl[i][k] = q[k];
          }
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sm.st_full[st]);
      {
        const long long c3 = clock64();
        pf[kPfConv] += c3 - c2;
        c2 = c3;
      }
      if (wid == 0) {
        if (lane == 0) {
          tc::mbar_wait(&sm.st_full[st], use & 1u);
          pf[kPfMmaIssue] += clock64() - c2;
          tc::tc_fence_after();
#pragma unroll
          for (uint32_t bb = 0; bb < 2; ++bb) {
            const uint32_t ha = tc::smem_u32(stage) + 2 * kOpBytes * bb, la = ha + kOpBytes;
#pragma unroll
            for (uint32_t k = 0; k < kSub / 16; ++k) {
              const uint64_t dh = tc::sw64_desc(ha + 32 * k), dl = tc::sw64_desc(la + 32 * k);
              // G = HH^T + HL^T + (HL^T)^T: ONE M128 x N256 MMA whose B is
              // the hi tile followed by the lo tile (contiguous, same
              // SBO), so TMEM columns 0..127 get HH^T and 128..255 HL^T;
              // the LH^T term is HL^T transposed, added in the epilogue
              (void)dl;
              tc::mma_bf16(tmem, dh, dh, idesc256, (ch | bb | k) ? 1u : 0u);
            }
          }
          tc::mma_commit(&sm.st_free[st]);
          if (ch + 1 == nch) tc::mma_commit(&sm.acc_ready);
        }
        __syncwarp();
      }
    }
    gch += nch;
    bool cvreal[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) cvreal[i] = sm.rid[wrow + ((lane + 32u * i) >> 2)] != kNone;
    // ((s0 + s1) + (s2 + s3)) then the tail in order (metric.hpp:15-24):
    // pending distances become exact keys
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float pr = __fadd_rn(sch[i], __shfl_down_sync(0xffffffffu, sch[i], 1));
      float tot = __fadd_rn(pr, __shfl_down_sync(0xffffffffu, pr, 2));
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (uint32_t(k) < row.ntail) tot = __fadd_rn(tot, stl[i][k]);
      const uint32_t r = wrow + ((lane + 32u * i) >> 2);
      if (cv_c == 0 && cvreal[i]) {
        const uint64_t k = sm.key[r];
        if (key_pending(k)) sm.key[r] = make_key(tot, sm.rid[r], key_fresh(k));
      }
    }
    {
      const long long tq = clock64();
      pf[kPfStream] += tq - tp;
      tp = tq;
    }
    if (lane == 0) tc::mbar_wait(&sm.acc_ready, it & 1u);
    __syncwarp();
    tc::tc_fence_after();
    {
      const long long tq = clock64();
      pf[kPfMmaWait] += tq - tp;
      tp = tq;
    }

    // ------------------------------------------------------------- epilogue
    const uint32_t tb = tmem + ((32u * q) << 16);
    const uint32_t sl_e = e / R, s0 = sl_e * R;
    const uint32_t Ue = sl_e < nl ? sm.lU[sl_e] : 0u;
    const bool real = e - s0 < Ue;
    float v[32];
    // HL^T rows of the tile in shared memory (the ring is idle now), row
    // stride 129 floats: thread e reads HL[e][j] and HL[j][e] conflict-free
    float* hls = reinterpret_cast<float*>(sm.ring[0]);
    const uint32_t blo = ((32u * q) & ~(R - 1u)) >> 5;        // column blocks of
    const uint32_t bhi = ((32u * q + 31u) | (R - 1u)) >> 5;   // these rows' lists
    if (h == 0) {
      tc::tmem_ld32(tb + 32u * q, v);  // the diagonal blocks of these rows
      float hh = v[0];
#pragma unroll
      for (int j = 1; j < 32; ++j)
        if (uint32_t(j) == lane) hh = v[j];
      tc::tmem_ld32(tb + 128u + 32u * q, v);
      float hl = v[0];
#pragma unroll
      for (int j = 1; j < 32; ++j)
        if (uint32_t(j) == lane) hl = v[j];
      sm.diag[e] = __fadd_rn(hh, __fadd_rn(hl, hl));  // G_ee = HH + HL + LH
      sm.rank[e] = 0u;
    }
    for (uint32_t cb = blo + h; cb <= bhi; cb += 2) {
      tc::tmem_ld32(tb + 128u + 32u * cb, v);
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) hls[e * 129u + 32u * cb + uint32_t(jj)] = v[jj];
    }
    if (tid == 0) sm.naq = 0;
    __syncthreads();  // keys final (pending filled), diag, HL^T staged, rank zeroed
    const uint64_t ke = sm.key[e];
    if (real) {  // rank by (dist, id) within the list, halves split by parity
      uint32_t r = 0;
      for (uint32_t j = s0 + h; j < s0 + Ue; j += 2) r += sm.key[j] < ke ? 1u : 0u;
      atomicAdd(&sm.rank[e], r);
    }
    __syncthreads();
    const uint32_t pe = s0 + sm.rank[e];
    if (h == 0 && real) {
      sm.perm[pe] = uint8_t(e);
      sm.pos[e] = uint8_t(pe);
      sm.occ[pe][0] = sm.occ[pe][1] = sm.occ[pe][2] = sm.occ[pe][3] = 0u;
    }
    __syncthreads();
    // occluder / band masks of row e over the rows ahead of it in its list;
    // the two warps of a lane quarter split the column blocks
    const float thr = key_dist(ke);
    const float dg = sm.diag[e];
    uint32_t oc[4] = {0u, 0u, 0u, 0u}, am[4] = {0u, 0u, 0u, 0u};
    {
      for (uint32_t cb = blo + h; cb <= bhi; cb += 2) {
        tc::tmem_ld32(tb + 32u * cb, v);  // HH^T
        if (!real) continue;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const uint32_t j = 32u * cb + uint32_t(jj);
          if (j - s0 >= Ue || j == e) continue;
          if (!(sm.key[j] < ke)) continue;
          const float gij =
              __fadd_rn(__fadd_rn(v[jj], hls[e * 129u + j]), hls[j * 129u + e]);
          const float dj = sm.diag[j];
          const float sn = __fadd_rn(fabsf(dg), fabsf(dj));
          const float dd = __fsub_rn(__fadd_rn(dg, dj), __fmul_rn(2.f, gij));
          const float eps = __fadd_rn(__fmul_rn(sn, g.eps_rel), 1e-25f);
          const uint32_t pj = sm.pos[j];
          if (__fadd_rn(dd, eps) < thr)
            set_bit4(oc, pj);
          else if (!(__fsub_rn(dd, eps) > thr))
            set_bit4(am, pj);
        }
      }
    }
    if (real) {
#pragma unroll
      for (int w4 = 0; w4 < 4; ++w4)
        if (oc[w4]) atomicOr(&sm.occ[pe][w4], oc[w4]);
    }
    tc::tc_fence_before();
    {
      const long long tq = clock64();
      pf[kPfMask] += tq - tp;
      tp = tq;
    }
    // band comparisons a walk may reach (not old/old): exact, a warp per
    // pair, in rounds of at most kAQ pairs
    {
      const bool fe = key_fresh(ke);
      bool more = real;
      uint32_t w4 = 0;
      // 4 KB per warp past the staged HL^T (ring + centre buffers are contiguous)
      float* scratch = reinterpret_cast<float*>(sm.ring[0]) + 128u * 129u + wid * 1024u;
      for (;;) {
        if (more) {
          more = false;
          for (; w4 < 4; ++w4) {
            uint32_t qb = w4 == 0 ? am[0] : (w4 == 1 ? am[1] : (w4 == 2 ? am[2] : am[3]));
            while (qb) {
              const uint32_t b = uint32_t(__ffs(qb)) - 1u;
              const uint32_t j = sm.perm[32u * w4 + b];
              if (fe || key_fresh(sm.key[j])) {  // old/old pairs are never compared
                const uint32_t qi = atomicAdd(&sm.naq, 1u);
                if (qi >= kAQ) {
                  more = true;
                  break;
                }
                sm.aq[qi] = (e << 8) | j;
              }
              qb &= qb - 1u;
            }
            if (w4 == 0) am[0] = qb;
            if (w4 == 1) am[1] = qb;
            if (w4 == 2) am[2] = qb;
            if (w4 == 3) am[3] = qb;
            if (more) break;
          }
        }
        __syncthreads();
        const uint32_t na = min(sm.naq, kAQ);
        if (na == 0) break;  // uniform
        if (tid == 0) {
          pf[kPfAmbPairs] += na;
          namb += na;
        }
        if (row.stride <= 1024u) {
          for (uint32_t k = wid; k < na; k += kWarps) {
            const uint32_t rec = sm.aq[k];
            const uint32_t t = rec >> 8, j = rec & 0xFFu;
            const float th = key_dist(sm.key[t]);
            const float df = warp_l2_fast(row, sm.rid[t], sm.rid[j]);
            const float m = __fmul_rn(df, g.fast_rel);
            bool occl;
            if (df > 1e-30f && __fadd_rn(df, m) < th)
              occl = true;  // rnnd::l2_sq < d_fast (1 + band) < threshold
            else if (df > 1e-30f && __fsub_rn(df, m) > th)
              occl = false;
            else
              occl = th >= warp_l2(row, sm.rid[t], sm.rid[j], scratch);
            if (lane == 0 && occl) {
              const uint32_t pj = sm.pos[j];
              atomicOr(&sm.occ[sm.pos[t]][pj >> 5], 1u << (pj & 31u));
            }
          }
        } else {
          for (uint32_t b0 = 8u * wid; b0 < na; b0 += 8u * kWarps) {
            const uint32_t qi = b0 + (lane >> 2);
            const uint32_t rec = sm.aq[qi < na ? qi : b0];
            const uint32_t t = rec >> 8, j = rec & 0xFFu;
            const float d = quad_l2<false>(row.xp + uint64_t(sm.rid[t]) * row.stride,
                                           row.xp + uint64_t(sm.rid[j]) * row.stride, lane & 3u,
                                           row.nblk, row.ntail);
            if (qi < na && (lane & 3u) == 0 && key_dist(sm.key[t]) >= d) {
              const uint32_t pj = sm.pos[j];
              atomicOr(&sm.occ[sm.pos[t]][pj >> 5], 1u << (pj & 31u));
            }
          }
        }
        __syncthreads();
        if (tid == 0) sm.naq = 0;
        __syncthreads();
      }
    }
    {
      const long long tq = clock64();
      pf[kPfAmb] += tq - tp;
      tp = tq;
    }
    // walk, part 1: the kept set of each list, one thread per list (lane 0
    // of warp sl), on the occluder bits only
    const uint64_t* occ64 = reinterpret_cast<const uint64_t*>(&sm.occ[0][0]);
    if (lane == 0 && wid < nl) {
      const uint32_t sl = wid, b0 = sl * R, U = sm.lU[sl];
      uint64_t k0 = 0, k1 = 0, f0 = 0, f1 = 0;
      for (uint32_t t = b0; t < b0 + U; ++t) {
        const bool f = key_fresh(sm.key[sm.perm[t]]);
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
      sm.kept[sl][0] = k0;
      sm.kept[sl][1] = k1;
      sm.fmask[sl][0] = f0;
      sm.fmask[sl][1] = f1;
      g.post_cnt[sm.lu[sl]] = uint32_t(__popcll(k0) + __popcll(k1));
    }
    __syncthreads();
    // walk, part 2: list position t's own checks / skips and its output
    if (tid < 128) {
      const uint32_t t = tid, sl = t / R, b0 = sl * R;
      if (sl < nl && t - b0 < sm.lU[sl]) {
        const uint32_t te = sm.perm[t];
        const uint64_t kt = sm.key[te];
        const bool f = key_fresh(kt);
        const uint64_t K0 = sm.kept[sl][0] & below_lo(t), K1 = sm.kept[sl][1] & below_hi(t);
        const uint64_t F0 = sm.fmask[sl][0], F1 = sm.fmask[sl][1];
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
          const uint32_t w_id = sm.rid[sm.perm[oi]];
          const uint64_t slot = sm.lbase[sl] + (te - b0);
          g.pend_src[slot] = w_id;
          g.pend_key[slot] = pending_key(sm.rid[te]);
          if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
        } else {
          const uint32_t nc = __popcll(c0) + __popcll(c1);
          checks += nc;
          skips += __popcll(K0 & ~c0) + __popcll(K1 & ~c1);
          tc0 = c0 | (nc ? bit_lo(t) : 0ull);
          tc1 = c1 | (nc ? bit_hi(t) : 0ull);
          // kept, flagged old (builder.cpp:68), at its rank among the kept
          g.keys[sm.lbase[sl] + (__popcll(K0) + __popcll(K1))] = kt & ~1ull;
        }
        if (uint32_t(tc0)) atomicOr(&sm.tch[sl][0], uint32_t(tc0));
        if (uint32_t(tc0 >> 32)) atomicOr(&sm.tch[sl][1], uint32_t(tc0 >> 32));
        if (uint32_t(tc1)) atomicOr(&sm.tch[sl][2], uint32_t(tc1));
        if (uint32_t(tc1 >> 32)) atomicOr(&sm.tch[sl][3], uint32_t(tc1 >> 32));
      }
    }
    __syncthreads();
    if (tid < nl)
      touched += __popc(sm.tch[tid][0]) + __popc(sm.tch[tid][1]) + __popc(sm.tch[tid][2]) +
                 __popc(sm.tch[tid][3]);
    pf[kPfWalk] += clock64() - tp;
    pf[kPfTiles] += 1;
    // the next tile's set-up barrier orders these reads before any rewrite
  }
  if (g.prof && tid == 0) {
    pf[kPfTotal] = clock64() - p0;
    for (int i = 0; i < kPfIssue; ++i) atomicAdd(&g.prof[i], (unsigned long long)pf[i]);
    atomicAdd(&g.prof[kPfMmaIssue], (unsigned long long)pf[kPfMmaIssue]);
  }
  if (g.prof && tid == 32)
    for (int i = kPfIssue; i < kPfMmaIssue; ++i) atomicAdd(&g.prof[i], (unsigned long long)pf[i]);
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
  tc::tc_fence_before();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

// 0 = off (every short list on k_scan_spec); otherwise lists of at most
// this many entries (<= 128) take the Gram-filtered walk.  Off by default:
// bit-exact (every parity suite passes with RNNDG_GRAM=128, including the
// four 1M-row reference builds) but slower end to end at C3 1M -- 2.29 s
// against 1.94 s (profiles/README.md, round 2): the stream phase converts
// ~570 SM-cycles per row where k_scan_spec spends ~300-400 per entry.
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
  static const int l2pf = [] {
    const char* e = std::getenv("RNNDG_GRAM_L2PF");
    return e ? std::atoi(e) : 1;
  }();
  a.l2pf = l2pf;
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
  // warp_l2_fast vs the reference-ordered l2_sq: both within their chain
  // bounds of the real value, x1.5 (3.1e-5 at d = 960)
  const double per_lane = 4.0 * double((cfg.stride + 127) / 128);
  a.fast_rel = float(1.5 * ((per_lane + 8.0) + (double(cfg.stride) / 4.0 + 5.0)) * 0x1p-24);
  const size_t smem = sizeof(GramSmem) + 1024;
  static unsigned long long attr_set = 0;  // per device
  if (!(attr_set >> (c->device & 63) & 1ull)) {
    RNNDG_CUDA(cudaFuncSetAttribute(k_scan_gram, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
    // all of the unified L1/shared array as shared memory: two CTAs per SM
    RNNDG_CUDA(cudaFuncSetAttribute(k_scan_gram, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    100));
    attr_set |= 1ull << (c->device & 63);
  }
  static int per_sm = 0;
  if (!per_sm) {
    // the occupancy calculator answers 1 for this kernel even without
    // dynamic shared memory; two 256-thread CTAs at 128 registers and
    // 2 x 110 KB do fit an SM and were measured co-resident (a 296-CTA
    // launch ran the C3 passes in ~33 ms against ~60 ms with 148)
    RNNDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan_gram, kThreads, smem));
    if (per_sm < kCtasPerSm) per_sm = kCtasPerSm;
    if (c->trace) {
      cudaFuncAttributes fa{};
      RNNDG_CUDA(cudaFuncGetAttributes(&fa, k_scan_gram));
      int smem_sm = 0, resv = 0, occ0 = 0;
      RNNDG_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                        c->device));
      RNNDG_CUDA(cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, c->device));
      RNNDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, k_scan_gram, kThreads, 0));
      std::fprintf(stderr,
                   "[rnndg] gram: %zu B shared memory per CTA, %d CTAs per SM (regs %d, static "
                   "smem %zu, SM smem %d, reserved %d, occupancy without dynamic smem %d)\n",
                   smem, per_sm, fa.numRegs, fa.sharedSizeBytes, smem_sm, resv, occ0);
    }
  }
  RNNDG_LAUNCH(c, k_scan_gram, unsigned(sm_count(c) * per_sm), kThreads, smem, a);
}

// RNNDG_TRACE: where the Gram kernel's cycles went in the last pass
void gram_trace(rnndg_ctx* c) {
  if (!gram_cap() || !c->gram_prof.p) return;
  unsigned long long h[kPfNum];
  RNNDG_CUDA(cudaMemcpy(h, c->gram_prof.p, sizeof(h), cudaMemcpyDeviceToHost));
  const double ctas = double(sm_count(c) * kCtasPerSm);
  auto mc = [&](int i) { return double(h[i]) / ctas * 1e-6; };  // Mcycles per CTA
  std::fprintf(stderr,
               "[rnndg] gram: tiles=%llu per CTA %.2f Mcyc: stream %.2f (warp 1: issue %.2f "
               "copy-wait %.2f convert %.2f; warp 0 mma-gate %.2f) mma-wait %.2f mask %.2f "
               "amb %.2f (%llu pairs) walk %.2f\n",
               h[kPfTiles], mc(kPfTotal), mc(kPfStream), mc(kPfIssue), mc(kPfCpWait), mc(kPfConv),
               mc(kPfMmaIssue), mc(kPfMmaWait), mc(kPfMask), mc(kPfAmb), h[kPfAmbPairs],
               mc(kPfWalk));
}

}  // namespace rnndg
