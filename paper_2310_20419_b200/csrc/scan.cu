// scan.cu -- the distance stage (scan_vertex, builder.cpp:41-69) on sm_100a.
//
// Formulation.  The reference walk is "pull": candidate v (ascending
// (dist, id)) tests the kept list K in order and the first w with
// v.dist >= d(v,w) removes it.  We run the equivalent "push": walk the sorted
// list; the first still-alive candidate is kept (every earlier kept entry has
// already been tested against it), then it is tested against every alive
// candidate after it.  A pair (v, w) is evaluated iff w was kept before v and
// v was still alive -- exactly the reference's pairs -- so pair_checks,
// flag_skips (old/old pairs passed over), removed and each redirect
// (w, v, d(v,w)) come out identical, with no speculative distance work.
//
// Mapping.  One CTA per active vertex (persistent CTAs, dynamic queue).  A
// push step's tests are compacted into a task list and evaluated 8 per warp
// at a time: one quad of lanes per pair, one lane per fp32 chain.  The store
// is kept on the device in a chain-blocked layout (k_chain_layout) so lane k
// reads chain k's next 8 elements with one 256-bit load (LDG.E.ENL2.256) and
// a quad reads a full 128-byte line.  The chains are combined exactly as
// ((s0+s1)+(s2+s3)) and the d % 4 tail is added in order (metric.hpp:15-24):
// bit-identical to rnnd::l2_sq.  A vertex's rows are pulled into L2 with one
// bulk prefetch per row (cp.async.bulk.prefetch.L2, UBLKPF) when it starts.
//
// Spreading a step over a CTA (instead of one warp) shortens each vertex's
// lifetime, so fewer vertices are in flight and their rows stay in L2 between
// push steps (ncu: a warp-per-vertex scan re-read rows from HBM at every step).
//
//   k_scan_spec<2, false, 4>   lists <= kScanUcap; keys + alive list in smem
//   k_scan_spec<32, true, 4>   longer lists (hubs that collect redirects), on
//                              a second stream concurrently
// (k_scan_block: the same walk with two steps per round; RNNDG_SPEC=0)
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ctx.hpp"
#include "scan.cuh"

namespace rnndg {

namespace {

constexpr int kShortWarps = 4;   // staged / sliced experiments: 128-thread CTAs
constexpr int kPushWarps = 2;    // default push scan: one 64-thread CTA per short list
constexpr int kLongWarps = 32;   // one 1024-thread CTA per long list
constexpr int kSpec = 4;         // provisional kept entries per push round

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

__device__ __forceinline__ void ld256(const float* p, float (&r)[8]) {
  asm volatile("ld.global.nc.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                 "=f"(r[6]), "=f"(r[7])
               : "l"(p));
}

__device__ __forceinline__ void prefetch_row_l2(const float* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void chain_step(const float (&va)[8], const float (&vb)[8], float& s) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float t = __fsub_rn(va[i], vb[i]);
    s = __fadd_rn(s, __fmul_rn(t, t));
  }
}

// A quad computes d(a, b) on chain-blocked rows, lane k = chain k; the exact
// total is returned in the quad's chain-0 lane.  All 32 lanes must call.
// Loads run two blocks ahead of the arithmetic.
__device__ __forceinline__ float quad_l2(const float* __restrict__ a, const float* __restrict__ b,
                                         uint32_t k, uint32_t nblk, uint32_t ntail) {
  float s = 0.f;
  const float* pa = a + 8 * k;
  const float* pb = b + 8 * k;
  float a0[8], b0[8], a1[8], b1[8];
  uint32_t blk = 0;
  if (nblk >= 2) {
    ld256(pa, a0);
    ld256(pb, b0);
    ld256(pa + 32, a1);
    ld256(pb + 32, b1);
    for (blk = 2; blk + 1 < nblk; blk += 2) {
      chain_step(a0, b0, s);
      ld256(pa + 32 * blk, a0);
      ld256(pb + 32 * blk, b0);
      chain_step(a1, b1, s);
      ld256(pa + 32 * (blk + 1), a1);
      ld256(pb + 32 * (blk + 1), b1);
    }
    chain_step(a0, b0, s);
    chain_step(a1, b1, s);
  }
  for (; blk < nblk; ++blk) {
    ld256(pa + 32 * blk, a0);
    ld256(pb + 32 * blk, b0);
    chain_step(a0, b0, s);
  }
  const float s_next = __shfl_down_sync(0xffffffffu, s, 1);
  const float pair = __fadd_rn(s, s_next);                    // s0+s1 | s2+s3
  const float pair2 = __shfl_down_sync(0xffffffffu, pair, 2);
  float sum = __fadd_rn(pair, pair2);                         // chain-0 lane
  if (ntail && k == 0) {
    const float* ta = a + 32 * nblk;
    const float* tb = b + 32 * nblk;
    for (uint32_t t = 0; t < ntail; ++t) {
      const float df = __fsub_rn(__ldg(ta + t), __ldg(tb + t));
      sum = __fadd_rn(sum, __fmul_rn(df, df));
    }
  }
  return sum;
}

// Same as quad_l2 on generic pointers (rows staged in shared memory or in
// global memory): two 128-bit loads per block and operand.
__device__ __forceinline__ float quad_l2_any(const float* a, const float* b, uint32_t k,
                                             uint32_t nblk, uint32_t ntail) {
  float s = 0.f;
  const float4* pa = reinterpret_cast<const float4*>(a + 8 * k);
  const float4* pb = reinterpret_cast<const float4*>(b + 8 * k);
#pragma unroll 4
  for (uint32_t blk = 0; blk < nblk; ++blk) {
    const float4 a0 = pa[8 * blk], a1 = pa[8 * blk + 1];
    const float4 b0 = pb[8 * blk], b1 = pb[8 * blk + 1];
    const float va[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float vb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    chain_step(va, vb, s);
  }
  const float s_next = __shfl_down_sync(0xffffffffu, s, 1);
  const float pair = __fadd_rn(s, s_next);
  const float pair2 = __shfl_down_sync(0xffffffffu, pair, 2);
  float sum = __fadd_rn(pair, pair2);
  if (ntail && k == 0) {
    const float* ta = a + 32 * nblk;
    const float* tb = b + 32 * nblk;
    for (uint32_t t = 0; t < ntail; ++t) {
      const float df = __fsub_rn(ta[t], tb[t]);
      sum = __fadd_rn(sum, __fmul_rn(df, df));
    }
  }
  return sum;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` in bytes
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Row {
  const float* xp;
  uint32_t stride, nblk, ntail;
  __device__ const float* operator()(uint64_t key) const {
    return xp + uint64_t(key_id(key)) * stride;
  }
};

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
  uint32_t nslots;       // row slots in dynamic shared memory (kStage)
  uint32_t slot_floats;  // slot stride
  uint8_t* touch;
  uint32_t* post_cnt;
  uint32_t* pend_src;
  uint64_t* pend_key;
  unsigned long long* bcnt;
  unsigned long long* ctr;
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
template <int W>
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
  __syncthreads();
  return before + __popc(m & ((1u << lane) - 1u));
}

// One CTA of W warps scans one vertex at a time (persistent, dynamic queue).
// A push step walks the alive candidates in batches of 32*W: the needed pairs
// of a batch are compacted into a task list and evaluated 8*W at a time (a
// quad per pair, a lane per chain), so a step with up to 8*W needed pairs
// costs one distance latency.  kLong: lists longer than kScanUcap, whose keys
// and alive list stay in global memory (queue act_list[n ..), work[1]);
// otherwise keys and alive list live in shared memory (queue act_small,
// work[0]).
template <int W, bool kLong, bool kStage>
__global__ void __launch_bounds__(32 * W, 1) k_scan_block(ScanArgs g) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  float* slots = reinterpret_cast<float*>(dyn_smem);
  constexpr uint32_t NT = 32 * W;
  constexpr uint32_t kCap = kLong ? 1 : kScanUcap;
  __shared__ uint64_t keys_sh[kCap];
  __shared__ uint32_t alive_sh[kCap];
  __shared__ uint32_t tq[2 * NT];  // task: list position of the candidate
  __shared__ uint64_t tk[2 * NT];  //       its key
  __shared__ float tres[2 * NT];   //       its distance to the kept entry
  __shared__ uint8_t tsel[2 * NT]; //       which kept entry (0: w1, 1: w2)
  __shared__ uint32_t wcnt[W];
  __shared__ uint32_t s_a, s_w2kept;
  __shared__ uint64_t bar;
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3;
  const Row row = g.row;  // local copy (no generic pointers into param space)
  const uint32_t row_bytes = row.stride * 4u;
  const uint32_t nq = kLong ? uint32_t(g.ctr_in[kLargeCount]) : uint32_t(*g.nsmall);
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0;
  uint32_t parity = 0;
  if (kStage && tid == 0) {
    mbar_init(&bar, 1);
    fence_proxy_async();
  }

  for (;;) {
    if (tid == 0) s_a = atomicAdd(g.work + (kLong ? 1 : 0), 1u);
    __syncthreads();
    const uint32_t a = s_a;
    if (a >= nq) break;
    const uint32_t u = kLong ? g.act_list[g.n + a] : uint32_t(g.act_small[a]);
    const uint64_t base = g.off[u];
    const uint32_t U = g.cnt[u];
    uint64_t* L = g.keys + base;
    uint8_t* T = g.touch + base;
    // kLong: keys are read from L directly; the kept entries of a step are
    // written to L[nk..] with nk <= p < every alive position
    const uint64_t* K = kLong ? L : keys_sh;
    uint32_t* A = kLong ? g.alive_g + base : alive_sh;
    // kStage: the nearest min(U, nslots) rows go to shared-memory slots with
    // one TMA bulk copy each; the rest are read through L2 (bulk prefetch)
    const uint32_t nst = kStage ? (U < g.nslots ? U : g.nslots) : 0u;
    for (uint32_t j = tid; j < U; j += NT) {
      const uint64_t k = L[j];
      if (!kLong) keys_sh[j] = k;
      A[j] = j;
      if (j >= nst) prefetch_row_l2(row(k), row_bytes);
    }
    __syncthreads();
    if (kStage) {
      if (tid == 0 && nst) {
        fence_proxy_async();  // earlier generic reads of the slots are done
        mbar_arrive_expect_tx(&bar, nst * row_bytes);
        for (uint32_t j = 0; j < nst; ++j)
          tma_load(slots + size_t(j) * g.slot_floats, row(K[j]), row_bytes, &bar);
      }
      if (nst) {
        mbar_wait(&bar, parity);
        parity ^= 1u;
      }
    }
    auto rowp = [&](uint32_t pos, uint64_t key) -> const float* {
      return pos < nst ? slots + size_t(pos) * g.slot_floats : row(key);
    };
    uint32_t na = U, nk = 0;
    while (na) {
      // Two push steps at once: w1 = first alive candidate (kept: every
      // earlier kept entry has already been tested against it) and w2 = the
      // second, provisionally kept.  Pairs with w2 are evaluated
      // speculatively and counted only for candidates that survive w1, and
      // only if w2 itself survives w1 -- exactly the reference's pairs.
      const uint32_t p1 = A[0];
      const uint64_t wk1 = K[p1];
      const bool wf1 = key_fresh(wk1);
      const float* xw1 = rowp(p1, wk1);
      const bool two = na >= 2;
      const uint32_t p2 = two ? A[1] : p1;
      const uint64_t wk2 = K[p2];
      const bool wf2 = key_fresh(wk2);
      const float* xw2 = rowp(p2, wk2);
      __syncthreads();  // all threads have read A[0..1] / K[p]
      if (tid == 0) L[nk] = wk1 & ~1ull;  // flagged old (builder.cpp:68)
      ++nk;
      uint32_t nn = 0;  // survivors so far, compacted in place into A[0 ..)
      bool w2kept = false;
      for (uint32_t b0 = 1; b0 < na; b0 += NT) {
        const uint32_t ai = b0 + tid;
        const bool valid = ai < na;
        const uint32_t q = valid ? A[ai] : 0u;
        const uint64_t vk = valid ? K[q] : 0ull;
        const bool vf = key_fresh(vk);
        const bool need1 = valid && (wf1 || vf);  // builder.cpp:53-56
        const bool need2 = valid && ai >= 2 && (wf2 || vf);
        uint32_t n1, n2;
        const uint32_t t1 = block_rank<W>(need1, wcnt, n1);
        const uint32_t t2 = n1 + block_rank<W>(need2, wcnt, n2);
        if (need1) {
          tq[t1] = q;
          tk[t1] = vk;
          tsel[t1] = 0;
        }
        if (need2) {
          tq[t2] = q;
          tk[t2] = vk;
          tsel[t2] = 1;
        }
        const uint32_t ntask = n1 + n2;
        __syncthreads();
        for (uint32_t t0 = 0; t0 < ntask; t0 += 8 * W) {
          const uint32_t tw = t0 + 8 * wid;
          if (tw >= ntask) continue;  // warp-uniform
          const uint32_t ti = tw + quad;
          const bool has = ti < ntask;
          const uint32_t ts = has ? ti : tw;
          const float* xv = rowp(tq[ts], tk[ts]);
          const float* xw = tsel[ts] ? xw2 : xw1;
          const float dist = kStage ? quad_l2_any(xv, xw, chain, row.nblk, row.ntail)
                                    : quad_l2(xv, xw, chain, row.nblk, row.ntail);
          if (has && chain == 0) tres[ti] = dist;
        }
        __syncthreads();
        // resolve w1 for every candidate; the fate of w2 (candidate ai == 1)
        // is known in the first batch
        bool gone = false, by2 = false;
        float dvw = 0.f;
        if (need1) {
          dvw = tres[t1];
          ++checks;
          T[q] = 1;
          T[p1] = 1;
          gone = key_dist(vk) >= dvw;
        } else if (valid) {
          ++skips;
        }
        if (ai == 1) s_w2kept = (valid && !gone) ? 1u : 0u;
        __syncthreads();
        w2kept = two && s_w2kept;
        if (valid && !gone && ai >= 2 && w2kept) {
          if (need2) {
            const float d2 = tres[t2];
            ++checks;
            T[q] = 1;
            T[p2] = 1;
            if (key_dist(vk) >= d2) {
              gone = true;
              by2 = true;
              dvw = d2;
            }
          } else {
            ++skips;
          }
        }
        if (gone) {
          ++removed;
          const uint32_t w_id = key_id(by2 ? wk2 : wk1);
          g.pend_src[base + q] = w_id;
          g.pend_key[base + q] = make_key(dvw, key_id(vk), 1u);
          if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);  // null when sharded
        }
        // survivors stay alive; a kept w2 leaves the alive list
        const bool stay = valid && !gone && !(ai == 1 && w2kept);
        uint32_t nstay;
        const uint32_t r = block_rank<W>(stay, wcnt, nstay);
        // every thread of the batch has read its A[ai] (block_rank syncs)
        if (stay) A[nn + r] = q;
        nn += nstay;
        __syncthreads();
      }
      if (w2kept) {
        if (tid == 0) L[nk] = wk2 & ~1ull;
        ++nk;
      }
      na = nn;
    }
    if (tid == 0) g.post_cnt[u] = nk;
    for (uint32_t j = tid; j < U; j += NT) touched += T[j];
    __syncthreads();
  }
  flush_counters(g.ctr, removed, checks, skips, touched);
}

// ------------------------------------------------------------ speculative
// Order-preserving block-wide exclusive scan of per-thread counts c.
template <int W>
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
  __syncthreads();
  return before + x - c;
}

// k_scan_block with D push steps per round.  The first D alive candidates
// w_1..w_D are provisionally kept and every later candidate is evaluated
// against all of them in the same round (one task per needed pair).  The
// fates of w_2..w_D are then resolved in list order (w_j is kept iff no kept
// w_i, i < j, occludes it), and each candidate walks w_1..w_D in order,
// counting only pairs with kept entries and stopping at its first occluder --
// the reference's exact sequence of skips and checks (builder.cpp:50-64).
// Pairs evaluated against a w_j that turns out occluded are not counted.
template <int W, bool kLong, int D>
__global__ void __launch_bounds__(32 * W, 1) k_scan_spec(ScanArgs g) {
  constexpr uint32_t NT = 32 * W;
  constexpr uint32_t kCap = kLong ? 1 : kScanUcap;
  constexpr uint32_t kTasks = NT * D;
  __shared__ uint64_t keys_sh[kCap];
  __shared__ uint32_t alive_sh[kCap];
  __shared__ uint32_t tq[kTasks];  // task: list position of the candidate
  __shared__ uint8_t tw[kTasks];   //       which provisional entry (0 .. D-1)
  __shared__ float tres[kTasks];   //       their distance
  __shared__ uint32_t wcnt[W];
  __shared__ uint32_t s_a, s_kept;
  __shared__ uint32_t s_tb[D];     // task base of candidates 1 .. D-1
  __shared__ uint32_t s_nm[D];     // their need masks
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3;
  const Row row = g.row;
  const uint32_t row_bytes = row.stride * 4u;
  const uint32_t nq = kLong ? uint32_t(g.ctr_in[kLargeCount]) : uint32_t(*g.nsmall);
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0;

  for (;;) {
    if (tid == 0) s_a = atomicAdd(g.work + (kLong ? 1 : 0), 1u);
    __syncthreads();
    const uint32_t a = s_a;
    if (a >= nq) break;
    const uint32_t u = kLong ? g.act_list[g.n + a] : uint32_t(g.act_small[a]);
    const uint64_t base = g.off[u];
    const uint32_t U = g.cnt[u];
    uint64_t* L = g.keys + base;
    uint8_t* T = g.touch + base;
    const uint64_t* K = kLong ? L : keys_sh;
    uint32_t* A = kLong ? g.alive_g + base : alive_sh;
    for (uint32_t j = tid; j < U; j += NT) {
      const uint64_t k = L[j];
      if (!kLong) keys_sh[j] = k;
      A[j] = j;
      prefetch_row_l2(row(k), row_bytes);
    }
    __syncthreads();
    uint32_t na = U, nk = 0;
    while (na) {
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
        const uint32_t tb = block_excl_scan<W>(__popc(nm), wcnt, ntask);
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
          const float dist = quad_l2(xv, row(wkey), chain, row.nblk, row.ntail);
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
          g.pend_key[base + q] = make_key(dvw, key_id(vk), 1u);
          if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);  // null when sharded
        }
        // survivors stay alive; kept provisional entries leave the alive list
        const bool stay = valid && !gone && !(ai < De && (kept >> ai & 1u));
        uint32_t nstay;
        const uint32_t r = block_rank<W>(stay, wcnt, nstay);
        if (stay) A[nn + r] = q;
        nn += nstay;
        __syncthreads();
      }
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
    }
    if (tid == 0) g.post_cnt[u] = nk;
    for (uint32_t j = tid; j < U; j += NT) touched += T[j];
    __syncthreads();
  }
  flush_counters(g.ctr, removed, checks, skips, touched);
}

// ------------------------------------------------------------- sliced
// Short lists, rows staged per push round.  Each warp owns 8 pairs of a round
// (one per quad) and streams their candidate rows through shared memory in
// slices of kSliceBlk 32-float blocks with 1-D TMA bulk copies, double
// buffered on two per-warp mbarriers; the kept row is staged once per step
// per CTA.  A round therefore waits for ~2 memory latencies instead of one
// per block, which shortens each vertex's lifetime and keeps its rows in L2
// between push steps.
constexpr uint32_t kSliceBlk = 4;
constexpr uint32_t kSliceRow = kSliceBlk * 32 + 4;  // floats; +16 B spreads banks

template <int W>
__global__ void __launch_bounds__(32 * W) k_scan_sliced(ScanArgs g) {
  constexpr uint32_t NT = 32 * W;
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  __shared__ uint64_t keys_sh[kScanUcap];
  __shared__ uint32_t alive_sh[kScanUcap];
  __shared__ uint32_t tq[NT];
  __shared__ uint64_t tk[NT];
  __shared__ float tres[NT];
  __shared__ uint32_t wcnt[W];
  __shared__ uint32_t s_a;
  __shared__ __align__(8) uint64_t wbar;
  __shared__ __align__(8) uint64_t vbar[W][2];
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3;
  const Row row = g.row;
  const uint32_t row_bytes = row.stride * 4u;
  const uint32_t nblk = row.nblk;
  const uint32_t nsl = (nblk + kSliceBlk - 1) / kSliceBlk;
  float* wbuf = reinterpret_cast<float*>(dyn_smem);                       // row.stride floats
  float* vbuf = wbuf + ((row.stride + 31) & ~31u) + size_t(wid) * 2 * 8 * kSliceRow;
  const uint32_t nq = uint32_t(*g.nsmall);
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0;
  uint32_t wpar = 0, vpar0 = 0, vpar1 = 0;
  if (tid == 0) mbar_init(&wbar, 1);
  if (lane == 0) {
    mbar_init(&vbar[wid][0], 1);
    mbar_init(&vbar[wid][1], 1);
  }
  fence_proxy_async();
  __syncthreads();

  // lane 0 of the warp: stage slice sl of the 8 (or fewer) task rows into buf
  auto issue_slice = [&](uint32_t sl, uint32_t b, uint32_t tw, uint32_t nt_w) {
    const uint32_t b0 = sl * kSliceBlk;
    const uint32_t nb = nblk - b0 < kSliceBlk ? nblk - b0 : kSliceBlk;
    const uint32_t bytes = nb * 128u;
    fence_proxy_async();
    mbar_arrive_expect_tx(&vbar[wid][b], bytes * nt_w);
    for (uint32_t q = 0; q < nt_w; ++q)
      tma_load(vbuf + size_t(b * 8 + q) * kSliceRow, row(tk[tw + q]) + 32 * b0, bytes,
               &vbar[wid][b]);
  };

  for (;;) {
    if (tid == 0) s_a = atomicAdd(g.work, 1u);
    __syncthreads();
    const uint32_t a = s_a;
    if (a >= nq) break;
    const uint32_t u = uint32_t(g.act_small[a]);
    const uint64_t base = g.off[u];
    const uint32_t U = g.cnt[u];
    uint64_t* L = g.keys + base;
    uint8_t* T = g.touch + base;
    for (uint32_t j = tid; j < U; j += NT) {
      const uint64_t k = L[j];
      keys_sh[j] = k;
      alive_sh[j] = j;
      prefetch_row_l2(row(k), row_bytes);
    }
    __syncthreads();
    uint32_t na = U, nk = 0;
    while (na) {
      const uint32_t p = alive_sh[0];
      const uint64_t wk = keys_sh[p];
      const bool wf = key_fresh(wk);
      __syncthreads();  // all threads read alive_sh[0]; previous wbuf readers done
      if (tid == 0) {
        L[nk] = wk & ~1ull;  // flagged old (builder.cpp:68)
        if (na > 1) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&wbar, row_bytes);
          tma_load(wbuf, row(wk), row_bytes, &wbar);
        }
      }
      ++nk;
      if (na > 1) {
        mbar_wait(&wbar, wpar);
        wpar ^= 1u;
      }
      uint32_t nn = 0;
      for (uint32_t b0 = 1; b0 < na; b0 += NT) {
        const uint32_t ai = b0 + tid;
        const bool valid = ai < na;
        const uint32_t q = valid ? alive_sh[ai] : 0u;
        const uint64_t vk = valid ? keys_sh[q] : 0ull;
        const bool need = valid && (wf || key_fresh(vk));  // builder.cpp:53-56
        skips += (valid && !need) ? 1 : 0;
        uint32_t ntask;
        const uint32_t t = block_rank<W>(need, wcnt, ntask);
        if (need) {
          tq[t] = q;
          tk[t] = vk;
        }
        checks += need ? 1 : 0;
        __syncthreads();
        for (uint32_t t0 = 0; t0 < ntask; t0 += 8 * W) {
          const uint32_t tw = t0 + 8 * wid;
          if (tw >= ntask) continue;  // warp-uniform
          const uint32_t nt_w = ntask - tw < 8 ? ntask - tw : 8;
          if (lane == 0) {
            issue_slice(0, 0, tw, nt_w);
            if (nsl > 1) issue_slice(1, 1, tw, nt_w);
          }
          float sacc = 0.f;
          for (uint32_t sl = 0; sl < nsl; ++sl) {
            const uint32_t b = sl & 1;
            if (b == 0) {
              mbar_wait(&vbar[wid][0], vpar0);
              vpar0 ^= 1u;
            } else {
              mbar_wait(&vbar[wid][1], vpar1);
              vpar1 ^= 1u;
            }
            const uint32_t bb = sl * kSliceBlk;
            const uint32_t nb = nblk - bb < kSliceBlk ? nblk - bb : kSliceBlk;
            const float* vs = vbuf + size_t(b * 8 + quad) * kSliceRow + 8 * chain;
            const float* ws = wbuf + 32 * bb + 8 * chain;
            for (uint32_t i = 0; i < nb; ++i) {
              const float4 v0 = *reinterpret_cast<const float4*>(vs + 32 * i);
              const float4 v1 = *reinterpret_cast<const float4*>(vs + 32 * i + 4);
              const float4 w0 = *reinterpret_cast<const float4*>(ws + 32 * i);
              const float4 w1 = *reinterpret_cast<const float4*>(ws + 32 * i + 4);
              const float va[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
              const float vb[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
              chain_step(va, vb, sacc);
            }
            __syncwarp();
            if (lane == 0 && sl + 2 < nsl) issue_slice(sl + 2, b, tw, nt_w);
          }
          const float s_next = __shfl_down_sync(0xffffffffu, sacc, 1);
          const float pair = __fadd_rn(sacc, s_next);
          const float pair2 = __shfl_down_sync(0xffffffffu, pair, 2);
          float dist = __fadd_rn(pair, pair2);
          const uint32_t ti = tw + quad;
          const bool has = quad < nt_w;
          if (has && chain == 0) {
            if (row.ntail) {
              const float* ta = row(tk[ti]) + 32 * nblk;
              const float* tb = wbuf + 32 * nblk;
              for (uint32_t x = 0; x < row.ntail; ++x) {
                const float df = __fsub_rn(__ldg(ta + x), tb[x]);
                dist = __fadd_rn(dist, __fmul_rn(df, df));
              }
            }
            tres[ti] = dist;
            T[tq[ti]] = 1;
            T[p] = 1;
          }
        }
        __syncthreads();
        bool gone = false;
        if (need) {
          const float dvw = tres[t];
          gone = key_dist(vk) >= dvw;
          if (gone) {
            ++removed;
            const uint32_t w_id = key_id(wk);
            g.pend_src[base + q] = w_id;
            g.pend_key[base + q] = make_key(dvw, key_id(vk), 1u);
            if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);  // null when sharded
          }
        }
        uint32_t nstay;
        const uint32_t r = block_rank<W>(valid && !gone, wcnt, nstay);
        if (valid && !gone) alive_sh[nn + r] = q;
        nn += nstay;
        __syncthreads();
      }
      na = nn;
    }
    if (tid == 0) g.post_cnt[u] = nk;
    for (uint32_t j = tid; j < U; j += NT) touched += T[j];
    __syncthreads();
  }
  flush_counters(g.ctr, removed, checks, skips, touched);
}

// ------------------------------------------------------------------ pull
// The reference's own ("pull") walk with a shared-memory row pool: a kept row
// is tested by every later candidate, so kept rows stay in smem slots for the
// whole scan of the vertex; candidate rows are TMA-loaded once.  HBM traffic
// is therefore about one read per touched row (the algorithmic 4·d·T_p).
// Candidates are processed in chunks of kCB; a wave evaluates, for every
// pending candidate, its next kKSeg needed kept entries (and, in the first
// wave of a chunk, every pair inside the chunk).  Warp 0 replays the
// reference walk: lane b walks candidate b's kept segment up to its first
// occluder (exact counters and redirect), lane 0 then resolves the
// intra-chunk part in order.  Pairs past an occluder are speculation.
constexpr uint32_t kCB = 8;
constexpr uint32_t kKSeg = 16;
constexpr uint32_t kPullTasks = kCB * kKSeg + kCB * (kCB - 1) / 2;
constexpr uint32_t kPullMaxSlots = 256;
constexpr uint16_t kNoSlot = 0xFFFF;
enum : uint8_t { kStPending = 0, kStKept = 1, kStRemoved = 2 };

template <int W>
__global__ void __launch_bounds__(32 * W) k_scan_pull(ScanArgs g) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  float* slots = reinterpret_cast<float*>(dyn_smem);
  __shared__ uint64_t keys_sh[kScanUcap];
  __shared__ uint16_t rslot[kScanUcap];
  __shared__ uint16_t kpos[kScanUcap];
  __shared__ uint16_t fslot[kPullMaxSlots];
  __shared__ uint16_t ta[kPullTasks], tb[kPullTasks], tinfo[kPullTasks];
  __shared__ float tres[kPullTasks];
  __shared__ float dint[kCB][kCB];
  __shared__ uint16_t lpos[2 * kPullTasks];
  __shared__ uint32_t cpos[kCB], cfront[kCB], cgen[kCB], cintra[kCB], tstart[kCB];
  __shared__ uint8_t cstate[kCB];
  __shared__ uint32_t s_a, s_nk, s_nfree, s_nt, s_loads, s_done;
  __shared__ __align__(8) uint64_t bar;
  constexpr uint32_t NT = 32 * W;
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3;
  const Row row = g.row;
  const uint32_t row_bytes = row.stride * 4u;
  const uint32_t nslots = g.nslots, sfl = g.slot_floats;
  const uint32_t nq = uint32_t(*g.nsmall);
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0;
  uint32_t parity = 0;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_proxy_async();
  }
  __syncthreads();

  for (;;) {
    if (tid == 0) s_a = atomicAdd(g.work, 1u);
    __syncthreads();
    const uint32_t a = s_a;
    if (a >= nq) break;
    const uint32_t u = uint32_t(g.act_small[a]);
    const uint64_t base = g.off[u];
    const uint32_t U = g.cnt[u];
    uint64_t* L = g.keys + base;
    uint8_t* T = g.touch + base;
    for (uint32_t j = tid; j < U; j += NT) {
      const uint64_t k = L[j];
      keys_sh[j] = k;
      rslot[j] = kNoSlot;
      if (j >= nslots) prefetch_row_l2(row(k), row_bytes);
    }
    for (uint32_t j = tid; j < nslots; j += NT) fslot[j] = uint16_t(nslots - 1 - j);
    if (tid == 0) {
      s_nfree = nslots;
      s_nk = 0;
    }
    __syncthreads();
    auto rowp = [&](uint32_t pos) -> const float* {
      const uint16_t sl = rslot[pos];
      return sl != kNoSlot ? slots + size_t(sl) * sfl : row(keys_sh[pos]);
    };

    for (uint32_t pos = 0; pos < U; pos += kCB) {
      const uint32_t nb = U - pos < kCB ? U - pos : kCB;
      if (tid < nb) {
        cpos[tid] = pos + tid;
        cstate[tid] = kStPending;
        cfront[tid] = 0;
        cintra[tid] = 0;
      }
      __syncthreads();
      const uint32_t k_old = s_nk;
      bool first = true;
      for (;;) {
        // ---- task generation (warp 0: lane b owns candidate b)
        if (wid == 0) {
          const uint32_t b = lane;
          const bool mine = b < nb && cstate[b] == kStPending;
          const uint32_t vp = b < nb ? cpos[b] : 0u;
          const bool vf = b < nb && key_fresh(keys_sh[vp]);
          uint32_t nin = 0, nkt = 0, kend = 0;
          if (b < nb && first)
            for (uint32_t b2 = 0; b2 < b; ++b2) nin += (vf || key_fresh(keys_sh[cpos[b2]])) ? 1 : 0;
          if (mine) {
            uint32_t k = cfront[b];
            while (k < k_old && nkt < kKSeg) {
              nkt += (vf || key_fresh(keys_sh[kpos[k]])) ? 1 : 0;
              ++k;
            }
            kend = k;
          }
          // exclusive prefix of (nin + nkt) over the lanes
          uint32_t mycnt = nin + nkt, incl = mycnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += v;
          }
          const uint32_t off0 = incl - mycnt;
          uint32_t t = off0;
          if (b < nb && first)
            for (uint32_t b2 = 0; b2 < b; ++b2)
              if (vf || key_fresh(keys_sh[cpos[b2]])) {
                ta[t] = uint16_t(vp);
                tb[t] = uint16_t(cpos[b2]);
                tinfo[t] = uint16_t(1 + b * kCB + b2);
                ++t;
              }
          if (b < nb) tstart[b] = t;
          if (mine) {
            for (uint32_t k = cfront[b]; k < kend; ++k) {
              const uint32_t wp = kpos[k];
              if (vf || key_fresh(keys_sh[wp])) {
                ta[t] = uint16_t(vp);
                tb[t] = uint16_t(wp);
                tinfo[t] = 0;
                ++t;
              }
            }
            cgen[b] = kend;
          }
          const uint32_t nt = __shfl_sync(0xffffffffu, incl, 31);
          // rows this wave touches that are not resident: one thread assigns
          // free slots and stages them with TMA
          if (lane == 0) {
            uint32_t loads = 0;
            for (uint32_t x = 0; x < 2 * nt; ++x) {
              const uint32_t pp = (x & 1) ? tb[x >> 1] : ta[x >> 1];
              if (rslot[pp] != kNoSlot || s_nfree == 0) continue;
              rslot[pp] = fslot[--s_nfree];
              lpos[loads++] = uint16_t(pp);
            }
            if (loads) {
              fence_proxy_async();
              mbar_arrive_expect_tx(&bar, loads * row_bytes);
              for (uint32_t i = 0; i < loads; ++i) {
                const uint32_t pp = lpos[i];
                tma_load(slots + size_t(rslot[pp]) * sfl, row(keys_sh[pp]), row_bytes, &bar);
              }
            }
            s_loads = loads;
            s_nt = nt;
          }
        }
        __syncthreads();
        const uint32_t nt = s_nt;
        if (s_loads) {
          mbar_wait(&bar, parity);
          parity ^= 1u;
        }
        // ---- evaluate: a quad per pair, 8 pairs per warp per round
        for (uint32_t t0 = 0; t0 < nt; t0 += 8 * W) {
          const uint32_t tw = t0 + 8 * wid;
          if (tw >= nt) continue;  // warp-uniform
          const uint32_t ti = tw + quad;
          const bool has = ti < nt;
          const uint32_t ts = has ? ti : tw;
          const float dist = quad_l2_any(rowp(ta[ts]), rowp(tb[ts]), chain, row.nblk, row.ntail);
          if (has && chain == 0) {
            tres[ti] = dist;
            const uint32_t info = tinfo[ti];
            if (info) dint[(info - 1) / kCB][(info - 1) % kCB] = dist;
          }
        }
        __syncthreads();
        // ---- replay the reference walk (warp 0)
        if (wid == 0) {
          const uint32_t b = lane;
          if (b < nb && cstate[b] == kStPending) {
            const uint32_t vp = cpos[b];
            const uint64_t vk = keys_sh[vp];
            const bool vf = key_fresh(vk);
            const float vd = key_dist(vk);
            uint32_t t = tstart[b];
            bool gone = false;
            for (uint32_t k = cfront[b]; k < cgen[b]; ++k) {
              const uint32_t wp = kpos[k];
              const uint64_t wk = keys_sh[wp];
              if (!vf && !key_fresh(wk)) {
                ++skips;
                continue;
              }
              const float dvw = tres[t++];
              ++checks;
              T[vp] = 1;
              T[wp] = 1;
              if (vd >= dvw) {
                gone = true;
                cstate[b] = kStRemoved;
                ++removed;
                const uint32_t w_id = key_id(wk);
                g.pend_src[base + vp] = w_id;
                g.pend_key[base + vp] = make_key(dvw, key_id(vk), 1u);
                if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);  // null when sharded
                break;
              }
            }
            if (!gone) cfront[b] = cgen[b];
          }
          __syncwarp();
          if (lane == 0) {
            // intra-chunk part, in candidate order: earlier chunk candidates
            // that were kept come after K_old in the kept list
            bool all_final = true;
            for (uint32_t b2 = 0; b2 < nb; ++b2) {
              if (cstate[b2] != kStPending) continue;
              if (cfront[b2] < k_old) {
                all_final = false;
                continue;
              }
              const uint32_t vp = cpos[b2];
              const uint64_t vk = keys_sh[vp];
              const bool vf = key_fresh(vk);
              const float vd = key_dist(vk);
              bool gone = false, blocked = false;
              for (uint32_t b3 = cintra[b2]; b3 < b2; ++b3) {
                const uint8_t s3 = cstate[b3];
                if (s3 == kStPending) {
                  blocked = true;
                  break;
                }
                cintra[b2] = b3 + 1;
                if (s3 == kStRemoved) continue;
                const uint32_t wp = cpos[b3];
                const uint64_t wk = keys_sh[wp];
                if (!vf && !key_fresh(wk)) {
                  ++skips;
                  continue;
                }
                const float dvw = dint[b2][b3];
                ++checks;
                T[vp] = 1;
                T[wp] = 1;
                if (vd >= dvw) {
                  gone = true;
                  cstate[b2] = kStRemoved;
                  ++removed;
                  const uint32_t w_id = key_id(wk);
                  g.pend_src[base + vp] = w_id;
                  g.pend_key[base + vp] = make_key(dvw, key_id(vk), 1u);
                  if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);  // null when sharded
                  break;
                }
              }
              if (gone) continue;
              if (blocked) {
                all_final = false;
                continue;
              }
              cstate[b2] = kStKept;
            }
            s_done = all_final ? 1u : 0u;
            if (all_final) {
              for (uint32_t b2 = 0; b2 < nb; ++b2) {
                const uint32_t pp = cpos[b2];
                if (cstate[b2] == kStKept) {
                  kpos[s_nk++] = uint16_t(pp);
                } else if (rslot[pp] != kNoSlot) {
                  fslot[s_nfree++] = rslot[pp];
                  rslot[pp] = kNoSlot;
                }
              }
            }
          }
        }
        first = false;
        __syncthreads();
        if (s_done) break;
      }
    }
    // survivors, flagged old, become the post-scan list (builder.cpp:68)
    const uint32_t nk = s_nk;
    for (uint32_t k = tid; k < nk; k += NT) L[k] = keys_sh[kpos[k]] & ~1ull;
    if (tid == 0) g.post_cnt[u] = nk;
    for (uint32_t j = tid; j < U; j += NT) touched += T[j];
    __syncthreads();
  }
  flush_counters(g.ctr, removed, checks, skips, touched);
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
    const float dist = quad_l2(row.xp + u * row.stride, row.xp + uint64_t(id) * row.stride, chain,
                               row.nblk, row.ntail);
    if (has && chain == 0) key[ps] = make_key(dist, id, 1u);
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

// Launches both scan kernels; the long-list kernel runs on the side stream
// and is joined back before returning.  work[0] / work[1] are the queues,
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
  // row slots: stride padded to an odd multiple of 16 B (quads of two CTAs'
  // rows land in different bank groups); ~100 KB per CTA for long rows
  // (2 CTAs per SM), ~48 KB for short rows
  a.slot_floats = cfg.stride + 4;
  const size_t slot_bytes = size_t(a.slot_floats) * 4;
  const size_t budget = slot_bytes >= 2048 ? 96 * 1024 : 48 * 1024;
  size_t ns = budget / slot_bytes;
  if (ns > kScanUcap) ns = kScanUcap;
  a.nslots = uint32_t(ns);
  // shared-memory staging of the nearest rows is an experiment (RNNDG_STAGE=1):
  // at 2 CTAs per SM it measured slower than reading rows through L2
  static const bool stage = [] {
    const char* e = std::getenv("RNNDG_STAGE");
    return e && e[0] == '1';
  }();
  if (!stage) a.nslots = 0;
  size_t smem = stage ? ns * slot_bytes : 0;
  // experiment (RNNDG_SLICED=1): rows streamed through per-warp shared-memory
  // slices with TMA; measured slower than direct 256-bit loads through L2
  static const bool sliced = [] {
    const char* e = std::getenv("RNNDG_SLICED");
    return e && e[0] == '1';
  }();
  // default: push walk, rows through L2 (k_scan_block).  RNNDG_SCAN=pull
  // selects the pull walk with a shared-memory row pool (k_scan_pull), which
  // measured ~2x slower at d = 960 (too few CTAs per SM to hide its chunk
  // loads); kept as an experiment
  static const bool push = [] {
    const char* e = std::getenv("RNNDG_SCAN");
    return !(e && e[0] == 'p' && e[1] == 'u' && e[2] == 'l');
  }();
  // pull tuning knobs (experiments): RNNDG_PULL_W = warps per CTA (4|8),
  // RNNDG_PULL_KB = shared-memory row pool per CTA in KB
  static const int pull_w = [] {
    const char* e = std::getenv("RNNDG_PULL_W");
    return e && e[0] == '4' ? 4 : 8;
  }();
  static const int pull_kb = [] {
    const char* e = std::getenv("RNNDG_PULL_KB");
    return e ? std::atoi(e) : 0;
  }();
  // warps per CTA of the push kernel (RNNDG_SHORT_W = 1 | 2 | 4 | 8).  Two
  // warps with an unconstrained register budget (147 regs, 6 CTAs/SM) beat
  // four warps (-6%) and register-capped variants with more CTAs per SM
  // (profiles/README.md, r01 tuning).
  static const int short_w = [] {
    const char* e = std::getenv("RNNDG_SHORT_W");
    const int v = e ? std::atoi(e) : kPushWarps;
    return v == 1 || v == 2 || v == 4 || v == 8 ? v : kPushWarps;
  }();
  auto kpush = short_w == 1   ? k_scan_block<1, false, false>
               : short_w == 2 ? k_scan_block<2, false, false>
               : short_w == 4 ? k_scan_block<4, false, false>
                              : k_scan_block<8, false, false>;
  // provisional kept entries per push round: RNNDG_SPEC = 2 | 3 | 4 (default
  // 4, k_scan_spec) or 0 (k_scan_block, two steps per round).  At C3 1M:
  // 2 -> 2.89 s, 3 -> 2.78 s, 4 -> 2.77 s, 6 -> 3.37 s per build.
  static const int spec = [] {
    const char* e = std::getenv("RNNDG_SPEC");
    const int v = e ? std::atoi(e) : kSpec;
    return v == 0 || v == 2 || v == 3 ? v : kSpec;
  }();
  if (spec == 2) kpush = short_w == 4 ? k_scan_spec<4, false, 2> : k_scan_spec<2, false, 2>;
  if (spec == 3) kpush = short_w == 4 ? k_scan_spec<4, false, 3> : k_scan_spec<2, false, 3>;
  if (spec == kSpec) kpush = short_w == 4 ? k_scan_spec<4, false, kSpec>
                                          : k_scan_spec<2, false, kSpec>;
  auto kshort = stage ? k_scan_block<kShortWarps, false, true>
                      : (sliced ? k_scan_sliced<kShortWarps>
                                : (push ? kpush
                                        : (pull_w == 4 ? k_scan_pull<4> : k_scan_pull<8>)));
  unsigned threads_short = 32 * (stage || sliced ? kShortWarps : (push ? short_w : pull_w));
  if (!push && !stage && !sliced) {
    const size_t pbudget = pull_kb > 0 ? size_t(pull_kb) * 1024
                                       : (slot_bytes >= 2048 ? 150 * 1024 : 96 * 1024);
    size_t pns = pbudget / slot_bytes;
    if (pns > kPullMaxSlots) pns = kPullMaxSlots;
    a.nslots = uint32_t(pns);
    smem = pns * slot_bytes;
  }
  size_t smem_sl = 0;
  if (!stage && sliced) {
    smem_sl = (size_t((cfg.stride + 31) & ~31u) + size_t(kShortWarps) * 2 * 8 * kSliceRow) * 4;
    smem = smem_sl;
  }
  if (smem > 0) {
    RNNDG_CUDA(cudaFuncSetAttribute(kshort, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    RNNDG_CUDA(cudaFuncSetAttribute(kshort, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared));
  }
  int per_sm = 0;
  RNNDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kshort, threads_short, smem));
  if (c->trace && !c->scan_cfg_logged) {
    std::fprintf(stderr, "[rnndg] scan: stage=%d sliced=%d slots=%u smem=%zu B ctas/SM=%d\n",
                 int(stage), int(sliced), a.nslots, smem, per_sm);
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
  if (spec == 0)
    k_scan_block<kLongWarps, true, false><<<long_grid, 32 * kLongWarps, 0, c->side>>>(a);
  else if (long_w == 8)
    k_scan_spec<8, true, kSpec><<<long_grid, 32 * 8, 0, c->side>>>(a);
  else if (long_w == 16)
    k_scan_spec<16, true, kSpec><<<long_grid, 32 * 16, 0, c->side>>>(a);
  else
    k_scan_spec<kLongWarps, true, kSpec><<<long_grid, 32 * kLongWarps, 0, c->side>>>(a);
  ++c->launches;
  RNNDG_CUDA(cudaGetLastError());
  RNNDG_LAUNCH(c, kshort, grid, threads_short, smem, a);
  RNNDG_CUDA(cudaEventRecord(c->ev_join, c->side));
  RNNDG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
}

}  // namespace rnndg
