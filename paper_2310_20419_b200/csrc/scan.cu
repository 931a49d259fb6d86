// scan.cu -- the distance stage (scan_vertex, builder.cpp:41-69) on sm_100a.
//
// Formulation.  The reference walk is "pull": candidate v (ascending
// (dist, id)) tests the kept list K in order and the first w with
// v.dist >= d(v,w) removes it.  We run the equivalent "push": walk the sorted
// list; the first still-alive candidate is kept (every earlier kept entry has
// already been tested against it), then it is tested against every alive
// candidate after it.  A pair (v, w) counts iff w was kept before v and v was
// still alive -- exactly the reference's pairs -- so pair_checks, flag_skips
// (old/old pairs passed over), removed and each redirect (w, v, d(v,w)) come
// out identical.  k_scan_spec runs D = 4 such steps per round: the first four
// alive candidates are provisionally kept and every pair with them is
// evaluated at once; pairs with a provisional entry that turns out occluded
// are evaluated but not counted.
//
// Mapping.  One CTA per active vertex (persistent CTAs, dynamic queues).  A
// round's pairs are compacted into a task list and evaluated 8 per warp at a
// time: one quad of lanes per pair, one lane per fp32 chain.  The store is
// kept on the device in a chain-blocked layout (k_chain_layout) so lane k
// reads chain k's next 8 elements with one 256-bit load (LDG.E.ENL2.256) and
// a quad reads a full 128-byte line.  The chains are combined exactly as
// ((s0+s1)+(s2+s3)) and the d % 4 tail is added in order (metric.hpp:15-24):
// bit-identical to rnnd::l2_sq.  A vertex's rows are pulled into L2 with one
// bulk prefetch per row (cp.async.bulk.prefetch.L2, UBLKPF) when it starts.
//
//   k_scan_spec<2, false, 3>   lists <= hub_threshold() (256): keys + alive
//                              list in smem, 6 CTAs of 64 threads per SM;
//                              D = 3 speculative rounds and old-run rounds
//   k_scan_hub<32, C, 4>       hub lists, on a second stream concurrently:
//                              clusters of C = 2 1024-thread CTAs (4 / 8 in
//                              the tail passes); lists over
//                              big_hub_threshold() (1024) walked by all CTAs
//                              of a cluster (longest first), the rest by one
//   k_scan_spec<32, true, 4>   hub lists, one 1024-thread CTA each (rows
//                              shorter than 2 KB, or RNNDG_HUB=0)
// Variants measured slower and removed (smem-staged rows, TMA-sliced rows, a
// pull walk, a warp-specialised double-buffered kernel, fused multi-distance
// tasks, early exit, deeper register pipelines): profiles/README.md.
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "ctx.hpp"
#include "scan.cuh"
#include "quad.cuh"

namespace rnndg {

namespace {

constexpr int kPushWarps = 2;    // default push scan: one 64-thread CTA per short list
constexpr int kLongWarps = 32;   // one 1024-thread CTA per long list
constexpr int kSpec = 4;         // provisional kept entries per push round (hub lists)
constexpr int kShortSpec = 3;    // ... and for short lists (RNNDG_SPEC)
constexpr size_t kNaMinRowBytes = 2048;  // rows this long stream L1::no_allocate
constexpr uint64_t kTail4Hubs = 3000;    // hub lists per pass for clusters of 4
constexpr uint64_t kTail8Hubs = 400;     // ... and of 8

// Chain-blocked row layout: element e < d4 = d - d % 4 lives at
//   32 * (e / 32) + 8 * (e % 4) + (e % 32) / 4
// i.e. per 32-element block, chain k's 8 elements are contiguous.  Padding
// slots are +0 (adding (0-0)^2 = +0 to a chain sum is exact); the d % 4 tail
// follows the blocks.  The row stride is a multiple of 8 floats (32 bytes).
__global__ void k_chain_layout(const float* __restrict__ x, uint64_t n, uint32_t d,
                               uint32_t stride, float* __restrict__ xp) {
  const uint32_t d4 = d & ~3u;
  const uint32_t nblk = (d4 + 31) / 32;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * stride;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / stride;
    const uint32_t s = uint32_t(i % stride);
    float v = 0.f;
    if (s < nblk * 32) {
      const uint32_t b = s / 32, k = (s % 32) / 8, j = s % 8;
      const uint32_t e = 32 * b + 4 * j + k;
      if (e < d4) v = x[r * d + e];
    } else {
      const uint32_t t = s - nblk * 32;
      if (t < d - d4) v = x[r * d + d4 + t];
    }
    xp[i] = v;
  }
}

struct ScanArgs {
  const uint64_t* act_small;  // short active lists, locality order (low 32 bits = vertex)
  const int* nsmall;
  const uint32_t* act_list;   // act_list[n ..): long active lists
  uint64_t n;
  const unsigned long long* ctr_in;
  unsigned int* work;
  const uint64_t* off;
  const uint32_t* cnt;
  uint64_t* keys;
  Row row;
  uint32_t* alive_g;
  uint8_t* touch;
  uint32_t* post_cnt;
  uint32_t* pend_src;
  uint64_t* pend_key;
  unsigned long long* bcnt;
  unsigned long long* ctr;
  int l2pf;      // bulk-prefetch a list's rows into L2 when its walk starts
  int coop_all;  // hubs per cluster below which every hub is walked cooperatively
  int run_max;   // longest leading run of old entries kept in one round (0: off)
  int run_tasks; // task budget of an old-run round per 64 threads
  int run_min;   // shortest run taken as an old-run round (0: D + 1)
  int pend;      // redirect records with pending distances (the Gram walk is on)
  int skip_small; // act_small is walked by bsp.cu: only the long short lists here
  uint64_t v0;   // first owned vertex (partitioned contexts)
};

__device__ __forceinline__ void flush_counters(unsigned long long* ctr, unsigned long long removed,
                                               unsigned long long checks,
                                               unsigned long long skips,
                                               unsigned long long touched) {
  for (int o = 16; o; o >>= 1) {
    touched += __shfl_xor_sync(0xffffffffu, touched, o);
    removed += __shfl_xor_sync(0xffffffffu, removed, o);
    checks += __shfl_xor_sync(0xffffffffu, checks, o);
    skips += __shfl_xor_sync(0xffffffffu, skips, o);
  }
  if (lane_id() == 0) {
    if (touched) atomicAdd(&ctr[kTouched], touched);
    if (removed) atomicAdd(&ctr[kRemoved], removed);
    if (checks) atomicAdd(&ctr[kPairChecks], checks);
    if (skips) atomicAdd(&ctr[kFlagSkips], skips);
  }
}

// Order-preserving block-wide compaction index of `pred`; total in `total`.
// kTrail = false drops the trailing barrier that lets `wcnt` be reused at
// once; callers then alternate between two wcnt arrays.
template <int W, bool kTrail = true>
__device__ __forceinline__ uint32_t block_rank(bool pred, uint32_t* wcnt, uint32_t& total) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (lane == 0) wcnt[wid] = __popc(m);
  __syncthreads();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const uint32_t c = wcnt[w];
    before += uint32_t(w) < wid ? c : 0u;
    tot += c;
  }
  total = tot;
  if (kTrail) __syncthreads();
  return before + __popc(m & ((1u << lane) - 1u));
}

template <int W, bool kTrail = true>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t c, uint32_t* wcnt,
                                                    uint32_t& total) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= uint32_t(o)) x += y;
  }
  if (lane == 31) wcnt[wid] = x;
  __syncthreads();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const uint32_t v = wcnt[w];
    before += uint32_t(w) < wid ? v : 0u;
    tot += v;
  }
  total = tot;
  if (kTrail) __syncthreads();
  return before + x - c;
}

// The push walk with D steps per round.  The first D alive candidates
// w_1..w_D are provisionally kept and every later candidate is evaluated
// against all of them in the same round (one task per needed pair).  The
// fates of w_2..w_D are then resolved in list order (w_j is kept iff no kept
// w_i, i < j, occludes it), and each candidate walks w_1..w_D in order,
// counting only pairs with kept entries and stopping at its first occluder --
// the reference's exact sequence of skips and checks (builder.cpp:50-64).
// Pairs evaluated against a w_j that turns out occluded are not counted.
template <int W, bool kLong, int D, bool kNA = true>
__global__ void __launch_bounds__(32 * W, 1) k_scan_spec(ScanArgs g) {
  constexpr uint32_t NT = 32 * W;
  constexpr uint32_t kCap = kLong ? 1 : kScanUcap;
  constexpr uint32_t kTasks = NT * D;
  __shared__ uint64_t keys_sh[kCap];
  __shared__ uint32_t alive_sh[kCap];
  __shared__ uint8_t touch_sh[kCap];  // touched flags of a short list
  __shared__ uint32_t tq[kTasks];  // task: list position of the candidate
  __shared__ uint8_t tw[kTasks];   //       which provisional entry (0 .. D-1)
  __shared__ float tres[kTasks];   //       their distance
  __shared__ uint32_t wcnt[W], wcnt2[W];  // scan / rank partials (alternating, no trailing barriers)
  __shared__ uint32_t s_a, s_kept;
  __shared__ uint32_t s_tb[D];     // task base of candidates 1 .. D-1
  __shared__ uint32_t s_nm[D];     // their need masks
  __shared__ uint32_t s_fr[2];     // fresh alive entries at a round's start (by parity)
  __shared__ uint32_t s_run;       // old-run rounds: window length,
  __shared__ uint32_t s_rp[32];    //   its list positions
  __shared__ uint64_t s_rk[32];    //   and keys
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3;
  const Row row = g.row;
  const uint32_t row_bytes = row.stride * 4u;
  // short lists: the long ones (act_list[0 ..)) first, then the rest
  const uint32_t nls = kLong ? 0u : uint32_t(g.ctr_in[kLongShortCount]);
  const uint32_t nq = kLong ? uint32_t(g.ctr_in[kLargeCount])
                            : nls + (g.skip_small ? 0u : uint32_t(*g.nsmall));
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0, evals = 0;

  for (;;) {
    if (tid == 0) {
      s_a = atomicAdd(g.work + (kLong ? 1 : 0), 1u);
      s_fr[0] = 0;
    }
    __syncthreads();
    const uint32_t a = s_a;
    if (a >= nq) break;
    const uint32_t u = kLong ? g.act_list[g.n + a]
                             : (a < nls ? g.act_list[a] : uint32_t(g.act_small[a - nls]));
    const uint64_t base = g.off[u];
    const uint32_t U = g.cnt[u];
    uint64_t* L = g.keys + base;
    // touched flags (counter only): shared memory for short lists, the
    // pass-zeroed global scratch for long ones
    uint8_t* T = kLong ? g.touch + base : touch_sh;
    const uint64_t* K = kLong ? L : keys_sh;
    uint32_t* A = kLong ? g.alive_g + base : alive_sh;
    uint32_t fr0 = 0;
    for (uint32_t j = tid; j < U; j += NT) {
      const uint64_t k = L[j];
      if (!kLong) {
        keys_sh[j] = k;
        touch_sh[j] = 0;
      }
      A[j] = j;
      fr0 += key_fresh(k);
      if (g.l2pf) prefetch_row_l2(row(k), row_bytes);
    }
    fr0 = __reduce_add_sync(0xffffffffu, fr0);
    if (lane == 0 && fr0) atomicAdd(&s_fr[0], fr0);
    __syncthreads();
    if (!kLong && g.pend && U && key_pending(keys_sh[U - 1])) {
      // redirected entries whose distance is pending (gram.cu) sort last:
      // exact l2_sq(u, v) by the CTA's quads, then the list re-sorted in
      // shared memory (bitonic over the next power of two, kTomb padding)
      uint32_t p0 = U;
      if (tid == 0) s_run = U;  // scratch here: first pending position
      __syncthreads();
      for (uint32_t j = tid; j < U; j += NT)
        if (key_pending(keys_sh[j])) atomicMin(&s_run, j);
      __syncthreads();
      p0 = s_run;
      const float* xu = row.xp + (g.v0 + u) * uint64_t(row.stride);
      for (uint32_t b0 = p0; b0 < U; b0 += NT / 4) {
        const uint32_t j = b0 + (tid >> 2);
        const uint32_t js = j < U ? j : p0;
        const uint64_t kv = keys_sh[js];
        const float d = quad_l2<kNA>(row(kv), xu, chain, row.nblk, row.ntail);
        __syncthreads();
        if (j < U && chain == 0) keys_sh[j] = make_key(d, key_id(kv), key_fresh(kv));
        __syncthreads();
      }
      uint32_t m = 2;
      while (m < U) m <<= 1;
      for (uint32_t j = U + tid; j < m; j += NT) keys_sh[j] = kTomb;
      __syncthreads();
      for (uint32_t k = 2; k <= m; k <<= 1)
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
          for (uint32_t i = tid; i < m; i += NT) {
            const uint32_t l = i ^ jj;
            if (l > i) {
              const uint64_t x = keys_sh[i], y = keys_sh[l];
              const bool up = (i & k) == 0;
              if (up ? (x > y) : (x < y)) {
                keys_sh[i] = y;
                keys_sh[l] = x;
              }
            }
          }
          __syncthreads();
        }
    }
    uint32_t na = U, nk = 0;
    uint32_t rb = 0;  // round parity: s_fr[rb] = fresh alive now, s_fr[rb ^ 1] = next round's
    while (na) {
      const uint32_t ftot = s_fr[rb];
      if (tid == 0) s_fr[rb ^ 1] = 0;  // visible to the batches after the next barrier
      if (g.run_max) {
        // Old-run round.  The alive entries ahead of the first fresh one are
        // all old: each was tested against every earlier kept entry already,
        // and old/old pairs are skipped (builder.cpp:53-56), so the whole
        // run is kept at once -- no provisional fates to resolve -- and only
        // the fresh candidates after it need distances, one per run entry.
        // Used when the run is longer than D and its tasks fit the task
        // arrays; otherwise the speculative round below.
        if (wid == 0) {
          const bool old = lane < na && !key_fresh(K[A[lane]]);
          const unsigned m = ~__ballot_sync(0xffffffffu, old);
          uint32_t run = m ? uint32_t(__ffs(m)) - 1u : 32u;
          if (run > uint32_t(g.run_max)) run = uint32_t(g.run_max);
          const uint32_t fb = ftot < NT ? ftot : NT;  // fresh candidates per batch, at most
          const uint32_t budget = min(kTasks, uint32_t(g.run_tasks) * (NT / 64));
          const uint32_t cap = budget / (fb ? fb : 1u);
          if (run > cap) run = cap;
          if (lane < run) {
            s_rp[lane] = A[lane];
            s_rk[lane] = K[A[lane]];
          }
          if (lane == 0) s_run = run;
        }
        __syncthreads();
        const uint32_t wr = s_run;
        if (wr >= (g.run_min ? uint32_t(g.run_min) : uint32_t(D) + 1)) {
          if (tid == 0) skips += uint64_t(wr) * (wr - 1) / 2;  // run entries among themselves
          uint32_t nn = 0;
          for (uint32_t b0 = wr; b0 < na; b0 += NT) {
            const uint32_t ai = b0 + tid;
            const bool valid = ai < na;
            const uint32_t q = valid ? A[ai] : 0u;
            const uint64_t vk = valid ? K[q] : 0ull;
            const bool vf = valid && key_fresh(vk);
            uint32_t ntask;
            const uint32_t tb = block_excl_scan<W, false>(vf ? wr : 0u, wcnt, ntask);
            evals += tid == 0 ? ntask : 0u;
            if (vf)
              for (uint32_t i = 0; i < wr; ++i) {
                tq[tb + i] = q;
                tw[tb + i] = uint8_t(i);
              }
            if (valid && !vf) skips += wr;
            __syncthreads();
            for (uint32_t t0 = 0; t0 < ntask; t0 += 8 * W) {
              const uint32_t twp = t0 + 8 * wid;
              if (twp >= ntask) continue;  // warp-uniform
              const uint32_t ti = twp + quad;
              const bool has = ti < ntask;
              const uint32_t ts = has ? ti : twp;
              const float dist = quad_l2<kNA>(row(K[tq[ts]]), row(s_rk[tw[ts]]), chain, row.nblk,
                                              row.ntail);
              if (has && chain == 0) tres[ti] = dist;
            }
            __syncthreads();
            bool gone = false;
            if (vf) {
              for (uint32_t i = 0; i < wr; ++i) {
                const float d = tres[tb + i];
                ++checks;
                T[q] = 1;
                T[s_rp[i]] = 1;
                if (key_dist(vk) >= d) {
                  gone = true;
                  ++removed;
                  const uint32_t w_id = key_id(s_rk[i]);
                  g.pend_src[base + q] = w_id;
                  g.pend_key[base + q] = g.pend ? pending_key(key_id(vk)) : make_key(d, key_id(vk), 1u);
                  if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
                  break;
                }
              }
            }
            const bool stay = valid && !gone;
            const unsigned fm = __ballot_sync(0xffffffffu, stay && vf);
            if (lane == 0 && fm) atomicAdd(&s_fr[rb ^ 1], uint32_t(__popc(fm)));
            uint32_t nstay;
            const uint32_t r = block_rank<W, false>(stay, wcnt2, nstay);
            if (stay) A[nn + r] = q;
            nn += nstay;
          }
          if (tid == 0)
            for (uint32_t i = 0; i < wr; ++i) L[nk + i] = s_rk[i];  // old already
          nk += wr;
          na = nn;
          rb ^= 1u;
          __syncthreads();
          continue;
        }
      }
      const uint32_t De = na < uint32_t(D) ? na : uint32_t(D);
      uint64_t wk[D];
      uint32_t wp[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        wp[i] = uint32_t(i) < De ? A[i] : A[0];
        wk[i] = K[wp[i]];
      }
      __syncthreads();  // all threads have read A[0 .. De) / K[p]
      uint32_t nn = 0;  // survivors so far, compacted in place into A[0 ..)
      uint32_t kept = 1u;  // bit i: w_{i+1} kept (known after the first batch)
      for (uint32_t b0 = 1; b0 < na; b0 += NT) {
        const uint32_t ai = b0 + tid;
        const bool valid = ai < na;
        const uint32_t q = valid ? A[ai] : 0u;
        const uint64_t vk = valid ? K[q] : 0ull;
        const bool vf = key_fresh(vk);
        // candidate ai is tested against w_1 .. w_min(D, ai)
        const uint32_t lim = valid ? (ai < De ? ai : De) : 0u;
        uint32_t nm = 0;
#pragma unroll
        for (int i = 0; i < D; ++i)
          if (uint32_t(i) < lim && (key_fresh(wk[i]) || vf)) nm |= 1u << i;
        uint32_t ntask;
        const uint32_t tb = block_excl_scan<W, false>(__popc(nm), wcnt, ntask);
        evals += tid == 0 ? ntask : 0u;
        {
          uint32_t t = tb;
#pragma unroll
          for (int i = 0; i < D; ++i)
            if (nm >> i & 1u) {
              tq[t] = q;
              tw[t] = uint8_t(i);
              ++t;
            }
        }
        if (ai < uint32_t(D)) {  // provisional entries (first batch only)
          s_tb[ai] = tb;
          s_nm[ai] = valid ? nm : 0u;
        }
        __syncthreads();
        for (uint32_t t0 = 0; t0 < ntask; t0 += 8 * W) {
          const uint32_t twp = t0 + 8 * wid;
          if (twp >= ntask) continue;  // warp-uniform
          const uint32_t ti = twp + quad;
          const bool has = ti < ntask;
          const uint32_t ts = has ? ti : twp;
          const uint64_t vkey = K[tq[ts]];
          const float* xv = row(vkey);
          const uint32_t wsel = tw[ts];
          uint64_t wkey = wk[0];
#pragma unroll
          for (int i = 1; i < D; ++i)
            if (wsel == uint32_t(i)) wkey = wk[i];
          const float dist = quad_l2<kNA>(xv, row(wkey), chain, row.nblk, row.ntail);
          if (has && chain == 0) tres[ti] = dist;
        }
        __syncthreads();
        if (b0 == 1) {
          // fates of w_2 .. w_De, in list order
          if (tid == 0) {
            uint32_t kb = 1u;
            for (uint32_t j = 1; j < De; ++j) {
              const float dj = key_dist(wk[j]);
              uint32_t t = s_tb[j];
              bool occl = false;
              for (uint32_t i = 0; i < j; ++i) {
                if (!(s_nm[j] >> i & 1u)) continue;
                const float d = tres[t++];
                if ((kb >> i & 1u) && dj >= d) {
                  occl = true;
                  break;
                }
              }
              if (!occl) kb |= 1u << j;
            }
            s_kept = kb;
          }
          __syncthreads();
          kept = s_kept;
        }
        // walk w_1 .. w_lim in order over the kept ones
        bool gone = false;
        uint32_t by = 0;
        float dvw = 0.f;
        {
          uint32_t t = tb;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            if (uint32_t(i) >= lim || gone) continue;
            const bool nd = nm >> i & 1u;
            const float d = nd ? tres[t] : 0.f;
            if (nd) ++t;
            if (!(kept >> i & 1u)) continue;  // not in the reference's kept list
            if (!nd) {
              ++skips;
              continue;
            }
            ++checks;
            T[q] = 1;
            T[wp[i]] = 1;
            if (key_dist(vk) >= d) {
              gone = true;
              by = uint32_t(i);
              dvw = d;
            }
          }
        }
        if (gone) {
          ++removed;
          uint64_t wkey = wk[0];
#pragma unroll
          for (int i = 1; i < D; ++i)
            if (by == uint32_t(i)) wkey = wk[i];
          const uint32_t w_id = key_id(wkey);
          g.pend_src[base + q] = w_id;
          g.pend_key[base + q] = g.pend ? pending_key(key_id(vk)) : make_key(dvw, key_id(vk), 1u);
          if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);  // null when sharded
        }
        // survivors stay alive; kept provisional entries leave the alive list
        const bool stay = valid && !gone && !(ai < De && (kept >> ai & 1u));
        const unsigned fm = __ballot_sync(0xffffffffu, stay && vf);
        if (lane == 0 && fm) atomicAdd(&s_fr[rb ^ 1], uint32_t(__popc(fm)));
        uint32_t nstay;
        const uint32_t r = block_rank<W, false>(stay, wcnt2, nstay);
        if (stay) A[nn + r] = q;
        nn += nstay;
      }
      __syncthreads();  // compacted alive list and survivor counts complete
      // kept entries, flagged old (builder.cpp:68), in list order
      if (tid == 0) {
#pragma unroll
        for (int i = 0; i < D; ++i)
          if (uint32_t(i) < De && (kept >> i & 1u)) L[nk++] = wk[i] & ~1ull;
      } else {
#pragma unroll
        for (int i = 0; i < D; ++i)
          if (uint32_t(i) < De && (kept >> i & 1u)) ++nk;
      }
      na = nn;
      rb ^= 1u;
    }
    if (tid == 0) g.post_cnt[u] = nk;
    for (uint32_t j = tid; j < U; j += NT) touched += T[j];
    __syncthreads();
  }
  flush_counters(g.ctr, removed, checks, skips, touched);
  if (tid == 0 && evals) {
    atomicAdd(&g.ctr[kEvalPairs], evals);
    if (kLong) atomicAdd(&g.ctr[kEvalHub], evals);
  }
}

// ------------------------------------------------------------ hub clusters
// k_scan_spec's walk for hub lists, spread over a thread-block cluster of C
// CTAs (one hub per cluster, persistent over the hub queue).  The single
// 1024-thread CTA per hub left the passes after each reverse phase bound by
// the largest hub's walk (one CTA's quads against a 5-10k-entry list).
//
// CTA r owns the list positions p with p % C == r and keeps its own alive
// list (ascending positions) in its slice of global scratch alive_g[base ..).
// A round: every CTA publishes its first D alive positions and its alive
// count in shared memory; after one cluster barrier every CTA merges the C*D
// heads over DSMEM into the same w_1..w_D (the D smallest alive positions of
// the whole list), pops the ones it owns, and tests its remaining alive
// candidates -- all of which come after w_D in list order -- against them.
// The fates of w_2..w_D (pairs among the w's only) are evaluated by every CTA
// redundantly, so each knows the kept mask without another exchange; the
// owner of w_j does w_j's bookkeeping (counters, redirect).  Kept entries of
// round r are written to L[nk..] by rank 0 after the next round's barrier,
// when no CTA reads round r's keys any more.  The head buffers are
// double-buffered by round parity, so one cluster barrier per round suffices.
// Pairs, counters and redirects are exactly k_scan_spec's.
template <int W, int D>
struct HubSmem {
  static constexpr uint32_t kTasks = 32 * W * D + D * (D - 1) / 2;
  uint32_t tq[kTasks];
  uint8_t tw[kTasks];
  float tres[kTasks];
  uint32_t wcnt[W];
  uint32_t head[2][32];   // first alive positions, pos << 1 | fresh
  uint32_t na[2], nfr[2]; // alive and fresh-alive counts (published)
  uint32_t frc[2];        // this CTA's fresh alive entries at a round's start (by parity)
  uint32_t a, tot, kept, npk, run;
  uint32_t wp[32];        // the merged first positions (pos << 1 | fresh)
  uint32_t tb[D], nm[D];  // fate tasks of w_2 .. w_D
  uint64_t rk[32];        // old-run window keys
  uint64_t pk[32];        // kept keys of the previous round (rank 0)
};

struct HubCounters {
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0, evals = 0;
};

// The walk of one hub list u by `cs` cooperating CTAs (cs == C, the cluster,
// for lists longer than big_hub_threshold(); cs == 1, this CTA alone,
// otherwise).  rank = this CTA's rank among them.
template <int W, int D, bool kNA>
__device__ __forceinline__ void hub_walk(const ScanArgs& g, uint32_t u, uint32_t cs, uint32_t rank,
                                         HubSmem<W, D>& sm, HubCounters& hc) {
  namespace cg = cooperative_groups;
  constexpr uint32_t NT = 32 * W;
  constexpr uint32_t kInf = 0xFFFFFFFFu;
  cg::cluster_group cl = cg::this_cluster();
  const bool coop = cs > 1;
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3;
  const Row row = g.row;
  const uint32_t row_bytes = row.stride * 4u;
  const uint64_t base = g.off[u];
  const uint32_t U = g.cnt[u];
  uint64_t* L = g.keys + base;
  uint8_t* T = g.touch + base;
  // rank r owns positions p % cs == r: U / cs of them, plus one while r < U % cs
  uint32_t* A = g.alive_g + base + rank * (U / cs) + (rank < U % cs ? rank : U % cs);
  uint32_t na = U / cs + (rank < U % cs ? 1u : 0u);
  uint32_t fr0 = 0;
  for (uint32_t i = tid; i < na; i += NT) {
    const uint32_t p = rank + i * cs;
    A[i] = p;
    const uint64_t k = L[p];
    fr0 += key_fresh(k);
    if (g.l2pf) prefetch_row_l2(row(k), row_bytes);
  }
  if (tid == 0) {
    sm.npk = 0;
    sm.frc[0] = 0;
  }
  __syncthreads();
  fr0 = __reduce_add_sync(0xffffffffu, fr0);
  if (lane == 0 && fr0) atomicAdd(&sm.frc[0], fr0);
  __syncthreads();
  // heads published per CTA: the first H alive positions of every CTA hold
  // the first H of the whole list (old-run windows are at most H long)
  const uint32_t H = 64 / (cs < 2 ? 2u : cs) < 32u ? 64 / (cs < 2 ? 2u : cs) : 32u;
  uint32_t nk = 0, ao = 0;
  for (uint32_t rnd = 0;; ++rnd) {
    const uint32_t buf = rnd & 1u;
    // fresh alive entries of this CTA (kept current by the survivor ballots)
    const uint32_t nfr = sm.frc[buf];
    if (tid == 0) sm.frc[buf ^ 1] = 0;
    if (tid < H) {
      uint32_t h = kInf;
      if (tid < na) {
        const uint32_t p = A[ao + tid];
        h = p << 1 | key_fresh(L[p]);
      }
      sm.head[buf][tid] = h;
    }
    if (tid == 0) {
      sm.na[buf] = na;
      sm.nfr[buf] = nfr;
    }
    if (coop)
      cl.sync();
    else
      __syncthreads();
    if (rank == 0 && tid == 0)
      for (uint32_t i = 0; i < sm.npk; ++i) L[nk - sm.npk + i] = sm.pk[i];
    if (wid == 0) {
      // the H smallest of the cs*H published heads in order, the total alive
      // and fresh-alive counts, and the old run at the head of the list
      uint32_t h0 = kInf, h1 = kInf, cnt = 0, fcnt = 0;
      if (coop) {
        if (lane < cs * H) h0 = cl.map_shared_rank(&sm.head[buf][0], lane / H)[lane % H];
        if (lane + 32 < cs * H)
          h1 = cl.map_shared_rank(&sm.head[buf][0], (lane + 32) / H)[(lane + 32) % H];
        if (lane < cs) {
          cnt = *cl.map_shared_rank(&sm.na[buf], lane);
          fcnt = *cl.map_shared_rank(&sm.nfr[buf], lane);
        }
      } else {
        if (lane < H) h0 = sm.head[buf][lane];
        if (lane == 0) {
          cnt = sm.na[buf];
          fcnt = sm.nfr[buf];
        }
      }
      const uint32_t tot = __reduce_add_sync(0xffffffffu, cnt);
      const uint32_t ftot = __reduce_add_sync(0xffffffffu, fcnt);
      uint32_t run = 0;
      bool in_run = g.run_max != 0;
      for (uint32_t i = 0; i < H; ++i) {
        const uint32_t m = __reduce_min_sync(0xffffffffu, h0 < h1 ? h0 : h1);
        if (h0 == m) h0 = kInf;
        if (h1 == m) h1 = kInf;
        if (lane == 0) sm.wp[i] = m;
        in_run = in_run && m != kInf && !(m & 1u);
        run += in_run ? 1u : 0u;
        if (i + 1 >= uint32_t(D) && !in_run) break;  // warp-uniform
      }
      if (run > uint32_t(g.run_max)) run = uint32_t(g.run_max);
      const uint32_t fb = ftot < NT ? ftot : NT;  // fresh candidates per CTA batch, at most
      const uint32_t cap = min(NT * D, uint32_t(g.run_tasks) * (NT / 64)) / (fb ? fb : 1u);
      if (run > cap) run = cap;
      if (lane == 0) {
        sm.tot = tot;
        sm.run = run;
      }
    }
    __syncthreads();
    const uint32_t tot = sm.tot;
    if (tot == 0) break;
    const uint32_t wr = sm.run;
    if (wr >= (g.run_min ? uint32_t(g.run_min) : uint32_t(D) + 1)) {
      // Old-run round (k_scan_spec's): the run is kept whole, only fresh
      // candidates are tested against it; the owner pops its run entries.
      uint32_t own = 0;
      for (uint32_t i = 0; i < wr; ++i) own += (sm.wp[i] >> 1) % cs == rank ? 1u : 0u;
      if (tid < wr) sm.rk[tid] = L[sm.wp[tid] >> 1];
      if (rank == 0 && tid == 0) hc.skips += uint64_t(wr) * (wr - 1) / 2;
      ao += own;
      na -= own;
      __syncthreads();
      uint32_t nn = 0;
      for (uint32_t b0 = 0; b0 < na; b0 += NT) {
        const uint32_t ai = b0 + tid;
        const bool valid = ai < na;
        const uint32_t q = valid ? A[ao + ai] : 0u;
        const uint64_t vk = valid ? L[q] : 0ull;
        const bool vf = valid && key_fresh(vk);
        uint32_t ntask;
        const uint32_t tb = block_excl_scan<W>(vf ? wr : 0u, sm.wcnt, ntask);
        hc.evals += tid == 0 ? ntask : 0u;
        if (vf)
          for (uint32_t i = 0; i < wr; ++i) {
            sm.tq[tb + i] = q;
            sm.tw[tb + i] = uint8_t(i);
          }
        if (valid && !vf) hc.skips += wr;
        __syncthreads();
        for (uint32_t t0 = 0; t0 < ntask; t0 += 8 * W) {
          const uint32_t twp = t0 + 8 * wid;
          if (twp >= ntask) continue;  // warp-uniform
          const uint32_t ti = twp + quad;
          const bool has = ti < ntask;
          const uint32_t ts = has ? ti : twp;
          const float dist = quad_l2<kNA>(row(L[sm.tq[ts]]), row(sm.rk[sm.tw[ts]]), chain,
                                          row.nblk, row.ntail);
          if (has && chain == 0) sm.tres[ti] = dist;
        }
        __syncthreads();
        bool gone = false;
        if (vf) {
          for (uint32_t i = 0; i < wr; ++i) {
            const float d = sm.tres[tb + i];
            ++hc.checks;
            T[q] = 1;
            T[sm.wp[i] >> 1] = 1;
            if (key_dist(vk) >= d) {
              gone = true;
              ++hc.removed;
              const uint32_t w_id = key_id(sm.rk[i]);
              g.pend_src[base + q] = w_id;
              g.pend_key[base + q] = g.pend ? pending_key(key_id(vk)) : make_key(d, key_id(vk), 1u);
              if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
              break;
            }
          }
        }
        const bool stay = valid && !gone;
        const unsigned fm = __ballot_sync(0xffffffffu, stay && vf);
        if (lane == 0 && fm) atomicAdd(&sm.frc[buf ^ 1], uint32_t(__popc(fm)));
        uint32_t nstay;
        const uint32_t r = block_rank<W>(stay, sm.wcnt, nstay);
        if (stay) A[nn + r] = q;
        nn += nstay;
        __syncthreads();
      }
      if (rank == 0 && tid == 0) {
        for (uint32_t i = 0; i < wr; ++i) sm.pk[i] = sm.rk[i];  // old already
        sm.npk = wr;
      }
      nk += wr;
      na = nn;
      ao = 0;
      continue;
    }
    const uint32_t De = tot < uint32_t(D) ? tot : uint32_t(D);
    uint64_t wk[D];
    uint32_t wp[D];
    uint32_t own = 0;  // w's owned by this CTA: its first `own` alive entries
#pragma unroll
    for (int i = 0; i < D; ++i) {
      wp[i] = (uint32_t(i) < De ? sm.wp[i] : sm.wp[0]) >> 1;
      wk[i] = L[wp[i]];
      own += (uint32_t(i) < De && wp[i] % cs == rank) ? 1u : 0u;
    }
    ao += own;
    na -= own;
    // fate tasks: w_j against w_i, i < j, where a flag is fresh
    if (tid == 0) {
      uint32_t t = 0;
      for (uint32_t j = 1; j < uint32_t(D); ++j) {
        uint32_t nm = 0;
        if (j < De)
          for (uint32_t i = 0; i < j; ++i)
            if (key_fresh(wk[i]) || key_fresh(wk[j])) nm |= 1u << i;
        sm.tb[j] = t;
        sm.nm[j] = nm;
        for (uint32_t i = 0; i < j; ++i)
          if (nm >> i & 1u) {
            sm.tq[t] = wp[j];
            sm.tw[t] = uint8_t(i);
            ++t;
          }
      }
      sm.tb[0] = t;  // number of fate tasks
    }
    __syncthreads();
    const uint32_t nf = sm.tb[0];
    uint32_t nn = 0;  // survivors, compacted into A[0 ..)
    uint32_t kept = 1u;
    for (uint32_t b0 = 0; b0 == 0 || b0 < na; b0 += NT) {
      const uint32_t ai = b0 + tid;
      const bool valid = ai < na;
      const uint32_t q = valid ? A[ao + ai] : 0u;
      const uint64_t vk = valid ? L[q] : 0ull;
      const bool vf = key_fresh(vk);
      uint32_t nm = 0;
#pragma unroll
      for (int i = 0; i < D; ++i)
        if (valid && uint32_t(i) < De && (key_fresh(wk[i]) || vf)) nm |= 1u << i;
      uint32_t ntask;
      const uint32_t pre = b0 == 0 ? nf : 0u;
      const uint32_t tb = pre + block_excl_scan<W>(__popc(nm), sm.wcnt, ntask);
      ntask += pre;
      hc.evals += tid == 0 ? ntask : 0u;
      {
        uint32_t t = tb;
#pragma unroll
        for (int i = 0; i < D; ++i)
          if (nm >> i & 1u) {
            sm.tq[t] = q;
            sm.tw[t] = uint8_t(i);
            ++t;
          }
      }
      __syncthreads();
      for (uint32_t t0 = 0; t0 < ntask; t0 += 8 * W) {
        const uint32_t twp = t0 + 8 * wid;
        if (twp >= ntask) continue;  // warp-uniform
        const uint32_t ti = twp + quad;
        const bool has = ti < ntask;
        const uint32_t ts = has ? ti : twp;
        const float* xv = row(L[sm.tq[ts]]);
        const uint32_t wsel = sm.tw[ts];
        uint64_t wkey = wk[0];
#pragma unroll
        for (int i = 1; i < D; ++i)
          if (wsel == uint32_t(i)) wkey = wk[i];
        const float dist = quad_l2<kNA>(xv, row(wkey), chain, row.nblk, row.ntail);
        if (has && chain == 0) sm.tres[ti] = dist;
      }
      __syncthreads();
      if (b0 == 0) {
        // fates of w_2 .. w_De in list order; the owner of w_j books its walk
        // exactly as k_scan_spec's candidate ai == j
        if (tid == 0) {
          uint32_t kb = 1u;
          for (uint32_t j = 1; j < De; ++j) {
            const float dj = key_dist(wk[j]);
            const bool mine = wp[j] % cs == rank;
            uint32_t t = sm.tb[j];
            bool occl = false;
            uint32_t by = 0;
            float dvw = 0.f;
            for (uint32_t i = 0; i < j && !occl; ++i) {
              const bool nd = sm.nm[j] >> i & 1u;
              const float d = nd ? sm.tres[t] : 0.f;
              if (nd) ++t;
              if (!(kb >> i & 1u)) continue;
              if (!nd) {
                if (mine) ++hc.skips;
                continue;
              }
              if (mine) {
                ++hc.checks;
                T[wp[j]] = 1;
                T[wp[i]] = 1;
              }
              if (dj >= d) {
                occl = true;
                by = i;
                dvw = d;
              }
            }
            if (!occl) {
              kb |= 1u << j;
            } else if (mine) {
              ++hc.removed;
              const uint32_t w_id = key_id(wk[by]);
              g.pend_src[base + wp[j]] = w_id;
              g.pend_key[base + wp[j]] = g.pend ? pending_key(key_id(wk[j])) : make_key(dvw, key_id(wk[j]), 1u);
              if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
            }
          }
          sm.kept = kb;
        }
        __syncthreads();
        kept = sm.kept;
      }
      bool gone = false;
      uint32_t by = 0;
      float dvw = 0.f;
      {
        uint32_t t = tb;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          if (uint32_t(i) >= De || !valid || gone) continue;
          const bool nd = nm >> i & 1u;
          const float d = nd ? sm.tres[t] : 0.f;
          if (nd) ++t;
          if (!(kept >> i & 1u)) continue;
          if (!nd) {
            ++hc.skips;
            continue;
          }
          ++hc.checks;
          T[q] = 1;
          T[wp[i]] = 1;
          if (key_dist(vk) >= d) {
            gone = true;
            by = uint32_t(i);
            dvw = d;
          }
        }
      }
      if (gone) {
        ++hc.removed;
        uint64_t wkey = wk[0];
#pragma unroll
        for (int i = 1; i < D; ++i)
          if (by == uint32_t(i)) wkey = wk[i];
        const uint32_t w_id = key_id(wkey);
        g.pend_src[base + q] = w_id;
        g.pend_key[base + q] = g.pend ? pending_key(key_id(vk)) : make_key(dvw, key_id(vk), 1u);
        if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
      }
      const bool stay = valid && !gone;
      const unsigned fm = __ballot_sync(0xffffffffu, stay && vf);
      if (lane == 0 && fm) atomicAdd(&sm.frc[buf ^ 1], uint32_t(__popc(fm)));
      uint32_t nstay;
      const uint32_t r = block_rank<W>(stay, sm.wcnt, nstay);
      if (stay) A[nn + r] = q;
      nn += nstay;
      __syncthreads();
    }
    const uint32_t km = kept & ((1u << De) - 1u);
    if (rank == 0 && tid == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int i = 0; i < D; ++i)
        if (km >> i & 1u) sm.pk[t++] = wk[i] & ~1ull;
      sm.npk = t;
    }
    nk += __popc(km);
    na = nn;
    ao = 0;
  }
  if (rank == 0 && tid == 0) g.post_cnt[u] = nk;
  for (uint32_t j = rank + tid * cs; j < U; j += NT * cs) hc.touched += T[j];
  __syncthreads();
}

// Launched as clusters of C CTAs.  Phase 1: each cluster walks the big hubs
// (queue act_list[2n - 1 - a], a < kBigCount) cooperatively, one at a time.
// Phase 2: every CTA walks the remaining hub lists (act_list[n + a], a <
// kLargeCount) on its own, like k_scan_spec<32, true, 4>.
__device__ __forceinline__ void flush_hub(const ScanArgs& g, const HubCounters& hc) {
  flush_counters(g.ctr, hc.removed, hc.checks, hc.skips, hc.touched);
  if (threadIdx.x == 0 && hc.evals) {
    atomicAdd(&g.ctr[kEvalPairs], hc.evals);
    atomicAdd(&g.ctr[kEvalHub], hc.evals);
  }
}

template <int W, int C, int D, bool kNA = true>
__global__ void __launch_bounds__(32 * W, 1) k_scan_hub(ScanArgs g) {
  namespace cg = cooperative_groups;
  static_assert(C * D <= 64, "head merge holds two heads per lane");
  __shared__ HubSmem<W, D> sm;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  const uint32_t tid = threadIdx.x;
  const uint32_t nbig = uint32_t(g.ctr_in[kBigCount]);
  const uint32_t nmid = uint32_t(g.ctr_in[kLargeCount]);
  // few hubs in all (the tail passes): every hub is walked cooperatively,
  // the big ones (largest first, k_sort_big) before the rest
  const bool coop_all = nbig + nmid <= uint32_t(g.coop_all) * (gridDim.x / C);
  const uint32_t ncoop = nbig + (coop_all ? nmid : 0u);
  HubCounters hc;
  for (;;) {
    if (rank == 0 && tid == 0) sm.a = atomicAdd(g.work + 1, 1u);
    cl.sync();
    const uint32_t a = *cl.map_shared_rank(&sm.a, 0);
    cl.sync();  // rank 0's sm.a is read before it moves on
    if (a >= ncoop) break;
    const uint32_t u = a < nbig ? g.act_list[2 * g.n - 1 - a] : g.act_list[g.n + (a - nbig)];
    hub_walk<W, D, kNA>(g, u, C, rank, sm, hc);
  }
  if (coop_all) return flush_hub(g, hc);
  // no DSMEM access past this point: CTAs may run (and exit) independently
  for (;;) {
    if (tid == 0) sm.a = atomicAdd(g.work + 4, 1u);
    __syncthreads();
    const uint32_t a = sm.a;
    __syncthreads();
    if (a >= nmid) break;
    hub_walk<W, D, kNA>(g, g.act_list[g.n + a], 1, 0, sm, hc);
  }
  flush_hub(g, hc);
}

// Big-hub queue act_list[2n - nbig .. 2n) sorted by length, longest at
// act_list[2n - 1] (taken first): one CTA, bitonic sort in shared memory of
// (length, vertex) keys.  Skipped when the queue exceeds kSortBig entries
// (throughput passes, where the order does not set the critical path).
constexpr uint32_t kSortBig = 4096;
__global__ void __launch_bounds__(1024) k_sort_big(uint32_t* __restrict__ act_list, uint64_t n,
                                                  const uint32_t* __restrict__ cnt,
                                                  const unsigned long long* __restrict__ ctr) {
  __shared__ uint64_t k[kSortBig];
  const uint32_t nb = uint32_t(ctr[kBigCount]);
  if (nb < 2 || nb > kSortBig) return;
  uint32_t m = 1;
  while (m < nb) m <<= 1;
  uint32_t* q = act_list + 2 * n - nb;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
    k[i] = i < nb ? (uint64_t(cnt[q[i]]) << 32 | q[i]) : ~0ull;
  __syncthreads();
  for (uint32_t s = 2; s <= m; s <<= 1)
    for (uint32_t j = s >> 1; j; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & s) == 0;
          const uint64_t a = k[i], b = k[l];
          if ((a > b) == up) {
            k[i] = b;
            k[l] = a;
          }
        }
      }
      __syncthreads();
    }
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) q[i] = uint32_t(k[i]);
}

// Cached distances of the random initial lists (graph.cpp:53-61), a quad per
// (u, id) pair on the chain-blocked rows.  key[p] holds the raw Floyd sample
// of pair p = ul * S + j (not yet shifted past the pivot u, rng.hpp:68-70).
__global__ void __launch_bounds__(256) k_init_dists(uint64_t nv, uint64_t v0, uint32_t S,
                                                   Row row, uint64_t* __restrict__ key) {
  const uint32_t lane = lane_id(), quad = lane >> 2, chain = lane & 3;
  const uint64_t total = nv * S;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t p0 = warp * 8; p0 < total; p0 += nwarps * 8) {
    const uint64_t p = p0 + quad;
    const bool has = p < total;
    const uint64_t ps = has ? p : p0;
    const uint64_t u = v0 + ps / S;
    uint32_t id = uint32_t(key[ps]);
    if (id >= u) ++id;
    const float dist = quad_l2(row.xp + uint64_t(id) * row.stride, row.xp + u * row.stride, chain,
                               row.nblk, row.ntail);
    if (has && chain == 0) key[ps] = make_key(dist, id, 1u);
  }
}

// NN-Descent local join (nndescent.cpp:72-80) for vertices [u0, u1): a quad
// per pair on the chain-blocked rows.  Pair p of vertex u (flat index
// poff[u] + local) is fresh x fresh (i < j) for local < f(f-1)/2, else
// fresh x old; both directed proposals (a <- b, b <- a) are written.
__global__ void __launch_bounds__(256)
    k_nd_join(uint64_t u0, uint64_t u1, const uint64_t* __restrict__ poff,
              const uint32_t* __restrict__ F, const uint32_t* __restrict__ fcnt,
              const uint32_t* __restrict__ O, const uint32_t* __restrict__ ocnt, uint32_t sample,
              uint32_t cap, Row row, uint32_t* __restrict__ pdst, uint64_t* __restrict__ pkey) {
  const uint32_t lane = lane_id(), quad = lane >> 2, chain = lane & 3;
  const uint64_t p_base = poff[u0], total = poff[u1] - p_base;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t q0 = warp * 8; q0 < total; q0 += nwarps * 8) {
    const uint64_t q = q0 + quad;
    const bool has = q < total;
    const uint64_t p = p_base + (has ? q : q0);
    // vertex: last u in [u0, u1) with poff[u] <= p
    uint64_t lo = u0, hi = u1;
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (poff[mid] <= p)
        lo = mid;
      else
        hi = mid;
    }
    const uint64_t u = lo;
    const uint32_t fc = fcnt[u];
    const uint64_t local = p - poff[u];
    const uint64_t tri = uint64_t(fc) * (fc ? fc - 1 : 0) / 2;
    uint32_t a, b;
    if (local < tri) {
      uint32_t i = 0;
      uint64_t r = local;
      while (r >= fc - 1 - i) {
        r -= fc - 1 - i;
        ++i;
      }
      a = F[u * sample + i];
      b = F[u * sample + i + 1 + uint32_t(r)];
    } else {
      const uint64_t r = local - tri;
      const uint32_t oc = ocnt[u];
      a = F[u * sample + uint32_t(r / oc)];
      b = O[u * cap + uint32_t(r % oc)];
    }
    const float d = quad_l2(row.xp + uint64_t(a) * row.stride, row.xp + uint64_t(b) * row.stride,
                            chain, row.nblk, row.ntail);
    if (has && chain == 0) {
      pdst[2 * q] = a;
      pkey[2 * q] = make_key(d, b, 1u);
      pdst[2 * q + 1] = b;
      pkey[2 * q + 1] = make_key(d, a, 1u);
    }
  }
}

}  // namespace

ScanConfig scan_config(rnndg_ctx* c) {
  ScanConfig cfg{};
  const uint32_t d = c->d;
  const uint32_t d4 = d & ~3u;
  cfg.nblk = (d4 + 31) / 32;
  cfg.ntail = d - d4;
  cfg.stride = cfg.nblk * 32 + (cfg.ntail ? 8 : 0);
  return cfg;
}

void launch_init_dists(rnndg_ctx* c, uint32_t S) {
  const ScanConfig cfg = scan_config(c);
  prepare_chain_layout(c);
  const uint64_t total = c->nv * S;
  if (!total) return;
  const Row row{c->xp.p, cfg.stride, cfg.nblk, cfg.ntail};
  const uint64_t groups = (total + 7) / 8;  // 8 pairs per warp
  uint64_t blocks = (groups + 7) / 8;       // 8 warps per block
  const uint64_t cap = uint64_t(sm_count(c)) * 8;
  if (blocks > cap) blocks = cap;
  RNNDG_LAUNCH(c, k_init_dists, unsigned(blocks), 256, 0, c->nv, c->v0, S, row, c->key.p);
}

void launch_nnd_join(rnndg_ctx* c, uint64_t u0, uint64_t u1, uint64_t npairs) {
  if (!npairs) return;
  const ScanConfig cfg = scan_config(c);
  prepare_chain_layout(c);
  const Row row{c->xp.p, cfg.stride, cfg.nblk, cfg.ntail};
  uint64_t blocks = (npairs + 63) / 64;  // 8 warps x 8 pairs
  const uint64_t cap = uint64_t(sm_count(c)) * 8;
  if (blocks > cap) blocks = cap;
  RNNDG_LAUNCH(c, k_nd_join, unsigned(blocks), 256, 0, u0, u1, c->nd_poff.p, c->nd_F.p,
               c->nd_fcnt.p, c->nd_O.p, c->nd_ocnt.p, c->nd_sample, c->nd_stride, row, c->nd_pdst.p,
               c->nd_pkey.p);
}

void prepare_chain_layout(rnndg_ctx* c) {
  const ScanConfig cfg = scan_config(c);
  if (c->xp_src == c->x && c->xp_stride == cfg.stride && c->xp.p) return;
  const uint64_t total = c->n * cfg.stride;
  c->xp.ensure(total);
  const uint64_t blocks = (total + 255) / 256;
  const unsigned grid = unsigned(blocks < (1u << 20) ? blocks : (1u << 20));
  RNNDG_LAUNCH(c, k_chain_layout, grid, 256, 0, c->x, c->n, c->d, cfg.stride, c->xp.p);
  c->xp_src = c->x;
  c->xp_stride = cfg.stride;
}

// provisional kept entries per push round of the short-list kernel:
// RNNDG_SPEC = 2 | 3 | 4 (default 3; the two-step k_scan_block it could select
// in round 1 was removed).  C3 1M before old-run rounds: 2 -> 2.89 s, 3 -> 2.78 s,
// 4 -> 2.77 s, 6 -> 3.37 s; with them: 2 -> 2.048 s, 3 -> 2.026 s, 4 ->
// 2.051 s (hub walks keep 4: 3 there costs 2.045 s).
int spec_mode() {
  static const int v = [] {
    const char* e = std::getenv("RNNDG_SPEC");
    const int x = e ? std::atoi(e) : kShortSpec;
    return x == 2 || x == 3 || x == 4 ? x : kShortSpec;
  }();
  return v;
}

// Hub lists on thread-block clusters of 1024-thread CTAs: returns the CTAs
// per cluster (2 or 4), or 0 for one k_scan_spec CTA per hub.  RNNDG_HUB
// forces 0 / 2 / 4; by default clusters of 2 for rows of >= 2 KB and one CTA
// per hub for short rows.  C3 1M (big-hub threshold 1024): 2 -> 2.25 s,
// 4 -> 2.26 s, 0 -> 2.42 s; clusters of 8 x 16 warps 2.38 s, 8 x 8 warps
// 2.41 s, 4 x 4 warps 2.36 s.  C2 1M (d = 128): 0 -> 0.755 s, 2 -> 0.769 s
// (the hub kernel's extra spills cost more than the shorter tail passes
// save when a pair is only four blocks).
int hub_cluster_size(rnndg_ctx* c) {
  static const int forced = [] {
    const char* e = std::getenv("RNNDG_HUB");
    if (!e) return -1;
    const int v = std::atoi(e);
    return v == 0 || v == 4 ? v : 2;
  }();
  if (spec_mode() == 0) return 0;
  if (forced >= 0) return forced;
  return scan_config(c).stride * sizeof(float) >= kNaMinRowBytes ? 2 : 0;
}

// Cluster size for this pass's hub kernel, when clusters are on (default
// schedule): pairs while hub lists are many, larger clusters for the tail
// passes whose few hubs set the critical path.  The hub count only falls
// between bulk rebuilds, so the previous pass's count bounds this one's.
// RNNDG_HUB_TAIL=0 keeps pairs throughout.  C3 1M: pairs throughout 2.149 s;
// clusters of 4 / 8 up to 600 / 64 hubs 2.137 s, 1500 / 200 2.128 s,
// 3000 / 400 2.125 s, 6000 / 800 2.126 s, 10000 / 1500 2.147 s.
int hub_cluster_for_pass(rnndg_ctx* c, int mode) {
  static const int tail = [] {
    const char* e = std::getenv("RNNDG_HUB_TAIL");
    return e ? std::atoi(e) : 1;
  }();
  if (mode != 2 || !tail || c->bulk_fresh) return mode;
  if (c->hubs_prev <= kTail8Hubs) return 8;
  if (c->hubs_prev <= kTail4Hubs) return 4;
  return 2;
}

// Launches both scan kernels; the long-list kernel runs on the side stream
// and is joined back before returning.  work[0] / work[1] are the queues
// (work[4] the hub kernel's second queue, work[6] the Gram tiles),
// work[2] the number of short active lists.
void launch_scan(rnndg_ctx* c, unsigned int* work) {
  const ScanConfig cfg = scan_config(c);
  prepare_chain_layout(c);
  ScanArgs a{};
  a.act_small = c->act_small.p;
  a.nsmall = reinterpret_cast<const int*>(work + 2);
  a.act_list = c->act_list.p;
  a.n = c->nv;  // long lists are queued at act_list[nv ..)
  a.ctr_in = c->counters.p;
  a.work = work;
  a.off = c->off.p;
  a.cnt = c->cnt.p;
  a.keys = c->key.p;  // lists are scanned in place (sorted invariant)
  a.row = Row{c->xp.p, cfg.stride, cfg.nblk, cfg.ntail};
  a.alive_g = c->kpos_g.p;
  a.touch = c->touch.p;
  a.post_cnt = c->post_cnt.p;
  a.pend_src = c->pend_src.p;
  a.pend_key = c->pend_key.p;
  a.bcnt = c->partitioned ? nullptr : c->bcnt.p;
  a.ctr = c->counters.p;
  // RNNDG_L2PF=0 drops the bulk L2 prefetch of a list's rows (C3 1M: 2.15 s
  // with it, 2.19 s without)
  static const int l2pf = [] {
    const char* e = std::getenv("RNNDG_L2PF");
    return e ? std::atoi(e) : 1;
  }();
  a.l2pf = l2pf;
  // a pass with at most RNNDG_COOP_ALL (default 4) hub lists per cluster walks
  // every hub cooperatively (0: only the big ones)
  static const int coop_all = [] {
    const char* e = std::getenv("RNNDG_COOP_ALL");
    return e ? std::atoi(e) : 4;
  }();
  a.coop_all = coop_all;
  // old-run rounds (RNNDG_RUN = longest run kept per round, <= 32; 0 = off).
  // C3 1M: off 2.141 s, 16 2.115 s, 32 2.123 s
  static const int run_max = [] {
    const char* e = std::getenv("RNNDG_RUN");
    const int v = e ? std::atoi(e) : 16;
    return v < 0 ? 0 : (v > 32 ? 32 : v);
  }();
  a.run_max = run_max;
  static const int run_tasks = [] {
    const char* e = std::getenv("RNNDG_RUN_TASKS");
    const int v = e ? std::atoi(e) : 256;
    return v < 1 ? 1 : v;
  }();
  a.run_tasks = run_tasks;
  // C3 1M: runs of >= 2 entries 2.022 s, >= 3 2.022 s, >= D + 1 2.025 s,
  // >= 6 2.053 s
  static const int run_min = [] {
    const char* e = std::getenv("RNNDG_RUN_MIN");
    const int v = e ? std::atoi(e) : 2;
    return v < 0 ? 0 : v;
  }();
  a.run_min = run_min;
  a.pend = gram_cap() ? 1 : 0;
  a.v0 = c->v0;
  // two-warp CTAs for short lists (4-warp CTAs measured slower,
  // profiles/README.md)
  constexpr int short_w = kPushWarps;
  // the first pass over the random initial lists removes ~80% of the
  // entries, so most provisional entries would be occluded: two per round
  // there (C3 1M pass 0: 25.1 -> 21 ms)
  const int spec = c->init_fresh && spec_mode() == 3 ? 2 : spec_mode();
  c->init_fresh = false;
  // streamed rows L1::no_allocate only for long rows (see ld256)
  const bool na = cfg.stride * sizeof(float) >= kNaMinRowBytes;
  auto kshort = na ? k_scan_spec<short_w, false, 3, true> : k_scan_spec<short_w, false, 3, false>;
  if (spec == 4)
    kshort = na ? k_scan_spec<short_w, false, 4, true> : k_scan_spec<short_w, false, 4, false>;
  if (spec == 2)
    kshort = na ? k_scan_spec<short_w, false, 2, true> : k_scan_spec<short_w, false, 2, false>;
  const unsigned threads_short = 32u * unsigned(short_w);
  const size_t smem = 0;
  int per_sm = 0;
  // shared-memory carveout in percent (RNNDG_CARVEOUT; -2 = leave the
  // driver's choice): the scan kernels need ~51 KB (short) / 37 KB (hub) of
  // shared memory per SM, the rest serves as L1 for the re-read rows.  C3 1M:
  // driver default 2.18 s, 20-25% 2.15 s, 30-50% 2.16-2.18 s, 0% collapses
  // occupancy.
  static const int carve = [] {
    const char* e = std::getenv("RNNDG_CARVEOUT");
    return e ? std::atoi(e) : 25;
  }();
  if (carve >= -1) {
    RNNDG_CUDA(cudaFuncSetAttribute(kshort, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  }
  RNNDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kshort, threads_short, smem));
  if (c->trace && !c->scan_cfg_logged) {
    std::fprintf(stderr, "[rnndg] scan: short W=%d spec=%d ctas/SM=%d\n", short_w, spec, per_sm);
    c->scan_cfg_logged = true;
  }
  if (const char* e = std::getenv("RNNDG_CTAS_PER_SM")) {  // tuning: cap resident CTAs
    const int v = std::atoi(e);
    if (v > 0 && v < per_sm) per_sm = v;
  }
  const unsigned grid = unsigned(sm_count(c)) * unsigned(per_sm > 0 ? per_sm : 1);
  // fork: the side stream waits for everything issued so far on the main one
  RNNDG_CUDA(cudaEventRecord(c->ev_fork, c->stream));
  RNNDG_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  // hub lists: one 1024-thread CTA per list, persistent over the hub queue,
  // one CTA per SM (CTAs that find the queue empty exit at once and free
  // their SM for the short-list kernel).  A quarter of the SMs (the r01
  // start) left the hub passes after each reverse phase hub-bound: 1M build
  // 2.77 s -> 2.53 s.  RNNDG_LONG_DIV: grid = SMs / div; RNNDG_LONG_W: 8 | 16
  // | 32 warps per hub CTA (32 best).
  static const unsigned long_div = [] {
    const char* e = std::getenv("RNNDG_LONG_DIV");
    const int v = e ? std::atoi(e) : 1;
    return unsigned(v >= 1 && v <= 16 ? v : 1);
  }();
  static const int long_w = [] {
    const char* e = std::getenv("RNNDG_LONG_W");
    const int v = e ? std::atoi(e) : kLongWarps;
    return v == 8 || v == 16 ? v : kLongWarps;
  }();
  const unsigned long_grid = unsigned(sm_count(c)) * unsigned(kLongWarps / long_w) / long_div;
  const int hub_mode = hub_cluster_for_pass(c, hub_cluster_size(c));
  c->bulk_fresh = false;
  if (hub_mode != 0) {
    auto khub = k_scan_hub<kLongWarps, 2, kSpec>;
    if (hub_mode == 4) khub = k_scan_hub<kLongWarps, 4, kSpec>;
    if (hub_mode == 8) khub = k_scan_hub<kLongWarps, 8, kSpec>;
    if (!na) khub = hub_mode == 4 ? k_scan_hub<kLongWarps, 4, kSpec, false>
                                  : k_scan_hub<kLongWarps, 2, kSpec, false>;
    const int hc = !na && hub_mode == 8 ? 2 : hub_mode, hw = kLongWarps;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = unsigned(hc);
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.gridDim = dim3(unsigned(hc) * 64u);
    cfg.blockDim = dim3(32u * unsigned(hw));
    cfg.stream = c->side;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    if (carve >= -1)
      RNNDG_CUDA(cudaFuncSetAttribute(khub, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    // co-resident clusters, per kernel variant (queried once each)
    static thread_local const void* cached_fn[8] = {};
    static thread_local int cached_clusters[8] = {};
    int max_clusters = 0;
    int slot = 0;
    for (; slot < 8 && cached_fn[slot]; ++slot)
      if (cached_fn[slot] == reinterpret_cast<const void*>(khub)) {
        max_clusters = cached_clusters[slot];
        break;
      }
    if (!max_clusters) {
      RNNDG_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, khub, &cfg));
      if (max_clusters < 1) max_clusters = 1;
      if (slot < 8) {
        cached_fn[slot] = reinterpret_cast<const void*>(khub);
        cached_clusters[slot] = max_clusters;
      }
      if (c->trace)
        std::fprintf(stderr, "[rnndg] scan: hub clusters C=%d W=%d, %d co-resident\n", hc, hw,
                     max_clusters);
    }
    cfg.gridDim = dim3(unsigned(max_clusters) * unsigned(hc));
    k_sort_big<<<1, 1024, 0, c->side>>>(c->act_list.p, c->nv, c->cnt.p, c->counters.p);
    ++c->launches;
    RNNDG_CUDA(cudaLaunchKernelEx(&cfg, khub, a));
  } else if (long_w == 8)
    k_scan_spec<8, true, kSpec><<<long_grid, 32 * 8, 0, c->side>>>(a);
  else if (long_w == 16)
    k_scan_spec<16, true, kSpec><<<long_grid, 32 * 16, 0, c->side>>>(a);
  else
    k_scan_spec<kLongWarps, true, kSpec><<<long_grid, 32 * kLongWarps, 0, c->side>>>(a);
  ++c->launches;
  RNNDG_CUDA(cudaGetLastError());
  if (c->trace) RNNDG_CUDA(cudaEventRecord(c->ev_scan[0], c->side));
  if (gram_cap()) {
    launch_gram(c, work);
    if (c->trace) RNNDG_CUDA(cudaEventRecord(c->ev_scan[2], c->stream));
  }
  // RNNDG_BSP: lists of <= bsp_max_len() entries (act_small) are walked round
  // by round across lists (bsp.cu) on a third stream; the short-list kernel
  // keeps the longer ones (act_list[0 .. nls))
  static const int bsp_stream = [] {
    const char* e = std::getenv("RNNDG_BSP_STREAM");
    return e ? std::atoi(e) : 1;
  }();
  bool used_side2 = false;
  if (rowwalk_cap(c)) {
    // short rows: lists of <= rowwalk_cap() entries are walked out of shared
    // memory, one warp per list (rowwalk.cu), ahead of the short-list kernel
    RNNDG_CUDA(cudaStreamWaitEvent(c->side2, c->ev_fork, 0));
    launch_rowwalk(c, work, c->side2, spec);
    used_side2 = true;
  }
  if (bsp_rounds()) {
    a.skip_small = 1;
    if (bsp_stream) {
      RNNDG_CUDA(cudaStreamWaitEvent(c->side2, c->ev_fork, 0));
      if (bsp_stream == 2) launch_bsp(c, work, c->side2, spec, l2pf);
    } else {
      launch_bsp(c, work, c->stream, spec, l2pf);
    }
  }
  RNNDG_LAUNCH(c, kshort, grid, threads_short, smem, a);
  if (bsp_rounds() && bsp_stream == 1) launch_bsp(c, work, c->side2, spec, l2pf);
  if (c->trace) RNNDG_CUDA(cudaEventRecord(c->ev_scan[1], c->stream));
  RNNDG_CUDA(cudaEventRecord(c->ev_join, c->side));
  RNNDG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  if ((bsp_rounds() && bsp_stream) || used_side2) {
    RNNDG_CUDA(cudaEventRecord(c->ev_join2, c->side2));
    RNNDG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join2, 0));
  }
}

}  // namespace rnndg
