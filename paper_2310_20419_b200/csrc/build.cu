// build.cu -- the RNN-Descent update loop on sm_100a (everything except the
// distance stage, which lives in scan.cu).
//
// Reference: /root/reference/proj/src/builder.cpp (update_parallel :88-139,
// add_reverse_edges :222-251, out_prune :141-150, in_prune :152-192, final
// sort :283-285) and graph.cpp random_init :47-63.
//
// Invariant: every list of the current graph is sorted ascending by key
// (= `nearer`, dist then id).  The state is a set per vertex, so ordering is
// free to choose; keeping it sorted means
//   * the scan needs no per-pass sort (builder.cpp:48 is a no-op),
//   * out_prune is a truncation, the final sort is a no-op,
//   * append-if-absent is a binary search: every cached distance is the exact
//     l2 of its two endpoints (init, redirect and reverse all store
//     l2_sq(row a, row b), which is bit-symmetric), so a proposal (w, v, d)
//     is already in w's list iff an entry with the same (dist, id) exists.
//
// One update pass (one stream, one host sync for the rebuilt CSR size):
//   k_mark_active       active = >= 1 fresh entry; inactive vertices are exact
//                       no-ops contributing U(U-1)/2 flag skips (builder.cpp:53-56)
//   locality order      3-hop min-id label over the graph, radix sort, select
//                       (processing order only; results are order-independent)
//   scan (scan.cu)      push-formulated occlusion scan, redirects bucketed by w
//   bucket sort         CUB segmented sort of each source's proposals
//   k_apply_count       dedupe (adjacent equal keys) + binary-search membership
//   k_merge             merge post-scan list and new entries into the next CSR
#define CCCL_IGNORE_DEPRECATED_API
#include <cub/device/device_radix_sort.cuh>
#include <vector>
#include <thread>
#include <cstring>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ctx.hpp"
#include "scan.cuh"
#include "quad.cuh"

namespace rnndg {

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kBlock = 32 * kWarpsPerBlock;
constexpr int kLabelRounds = 3;

struct ToU64 {
  __host__ __device__ uint64_t operator()(uint32_t v) const { return v; }
};

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void warp_add_counter(unsigned long long* ctr,
                                                 unsigned long long v) {
  v = warp_sum(v);
  if (lane_id() == 0 && v) atomicAdd(ctr, v);
}

// first index in [0, m) with a[i] >= key
__device__ __forceinline__ uint32_t lower_bound(const uint64_t* a, uint32_t m, uint64_t key) {
  uint32_t lo = 0, hi = m;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

#define WARP_LOOP(var, count)                                                      \
  const uint64_t warp_ = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; \
  const uint64_t nwarps_ = (uint64_t(gridDim.x) * blockDim.x) >> 5;             \
  for (uint64_t var = warp_; var < (count); var += nwarps_)

// ------------------------------------------------------------- random init
// graph.cpp:47-63.  One thread per vertex runs Floyd's sampling (rng.hpp:46-72;
// the emitted-set test is a linear scan, which is exactly the reference's
// S <= 64 branch and equivalent to its hash-set branch) and leaves the raw
// samples in the keys; k_init_dists (scan.cu) shifts them past the pivot and
// computes the S cached distances.
__global__ void k_random_init(uint64_t n, uint64_t v0, uint64_t nv, uint32_t S, uint64_t seed,
                              uint64_t* __restrict__ key) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t ul = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; ul < nv; ul += stride) {
    const uint64_t u = v0 + ul;  // global id: the stream and the pivot are global
    uint64_t* out = key + ul * S;
    SplitMix64 rng(mix_seed(seed, u));
    const uint32_t domain = uint32_t(n - 1);  // exclude u
    uint32_t m = 0;
    for (uint32_t j = domain - S; j < domain; ++j) {
      uint32_t t = uint32_t(rng.bounded(uint64_t(j) + 1));
      bool hit = false;
      for (uint32_t q = 0; q < m; ++q)
        if (uint32_t(out[q]) == t) {
          hit = true;
          break;
        }
      out[m++] = hit ? j : t;
    }
  }
}

__global__ void k_fill_offsets(uint64_t n, uint32_t S, uint64_t* off, uint32_t* cnt) {
  uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u <= n) off[u] = u * S;
  if (u < n) cnt[u] = S;
}

// upper bounds of the size classes 0 .. kSizeClasses - 2 (the last class runs
// up to the cap)
struct ClassBounds {
  uint32_t b[kSizeClasses - 1];
};

// ------------------------------------------------------------ mark active
// active = the list holds a fresh entry (builder.cpp:53-56: otherwise every
// pair is old/old and the scan only counts skips).  One warp per list
// (coalesced key reads, ballot), persistent warps; counters reduced per warp
// and added once per warp at the end.  Lists longer than ucap go to the hub
// queues: act_list[n + i] (<= big_cap) and act_list[2n - 1 - i] (> big_cap);
// short active lists are selected later (locality_order).
__global__ void __launch_bounds__(256) k_mark_active(uint64_t n, const uint64_t* __restrict__ off,
                                                    const uint32_t* __restrict__ cnt,
                                                    const uint64_t* __restrict__ key,
                                                    uint8_t* __restrict__ active,
                                                    uint32_t* __restrict__ act_list,
                                                    uint32_t* __restrict__ post_cnt,
                                                                          unsigned long long* __restrict__ ctr,
                                                    uint32_t ucap, uint32_t big_cap,
                                                    uint32_t ls_cap, uint32_t gcap,
                                                    ClassBounds gb,
                                                    uint32_t* __restrict__ gq,
                                                    uint64_t* __restrict__ mat_b,
                                                    uint64_t* __restrict__ mat_e) {
  constexpr uint32_t kQBuf = 16;
  __shared__ uint32_t qbuf[8][kSizeClasses][kQBuf];  // per warp and size class (lane 0's)
  uint32_t qn[kSizeClasses] = {};
  const uint32_t lane = lane_id();
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long skips = 0, aentries = 0, nact = 0, maxlen = 0;
  for (uint64_t u = warp; u < n; u += nwarps) {
    const uint64_t b = off[u];
    const uint32_t U = cnt[u];
    bool act = false;
    for (uint32_t j0 = 0; j0 < U && !act; j0 += 32) {
      const uint32_t j = j0 + lane;
      act = __any_sync(0xffffffffu, j < U && key_fresh(key[b + j]));
    }
    if (lane != 0) continue;
    if (mat_b && act && U > ucap && key_pending(key[b + U - 1])) {
      // an active hub list ending in pending entries (they sort last):
      // queued for resolve_pending before the scan (the Gram walk and the
      // short-list kernel resolve their own lists' pending entries)
      const uint32_t x = atomicAdd(reinterpret_cast<unsigned int*>(&ctr[kMatCount]), 1u);
      mat_b[x] = b;
      mat_e[x] = b + U;
      mat_e[n + x] = u;  // the list's vertex
    }
    uint8_t flag = 0;
    if (act) {
      aentries += U;
      nact += 1;
      maxlen = U > maxlen ? U : maxlen;
      flag = U > ucap ? 2 : (U > ls_cap ? 3 : 1);
      if (U <= gcap) {  // Gram-filtered walk (gram.cu) / shared-memory walk
        // (rowwalk.cu), queued by size class: buffered per warp, one atomic per
        // kQBuf lists (a million single-address atomics cost 0.5 ms per pass)
        int gc = 0;
#pragma unroll
        for (int i = 0; i < kSizeClasses - 1; ++i) gc += U > gb.b[i] ? 1 : 0;
        uint32_t* qb = qbuf[threadIdx.x >> 5][gc];
        qb[qn[gc]++] = uint32_t(u);
        if (qn[gc] == kQBuf) {
          const uint32_t x =
              atomicAdd(reinterpret_cast<unsigned int*>(&ctr[kGram0 + gc]), uint32_t(kQBuf));
          for (uint32_t i = 0; i < kQBuf; ++i) gq[uint64_t(gc) * n + x + i] = qb[i];
          qn[gc] = 0;
        }
        flag = 4;
      } else if (flag == 3) {  // long short list: queued ahead of the others, act_list[i]
        const uint32_t x = atomicAdd(reinterpret_cast<unsigned int*>(&ctr[kLongShortCount]), 1u);
        act_list[x] = uint32_t(u);
      } else if (U > ucap && U > big_cap) {  // a hub list (never both queues)
        const uint32_t x = atomicAdd(reinterpret_cast<unsigned int*>(&ctr[kBigCount]), 1u);
        act_list[2 * n - 1 - x] = uint32_t(u);
      } else if (U > ucap) {
        const uint32_t x = atomicAdd(reinterpret_cast<unsigned int*>(&ctr[kLargeCount]), 1u);
        act_list[n + x] = uint32_t(u);
      }
    } else {
      post_cnt[u] = U;
      skips += (unsigned long long)U * (U ? U - 1 : 0) / 2;
    }
    active[u] = flag;
  }
  if (lane == 0) {
    for (int gc = 0; gc < kSizeClasses; ++gc)
      if (qn[gc]) {
        const uint32_t x = atomicAdd(reinterpret_cast<unsigned int*>(&ctr[kGram0 + gc]), qn[gc]);
        for (uint32_t i = 0; i < qn[gc]; ++i)
          gq[uint64_t(gc) * n + x + i] = qbuf[threadIdx.x >> 5][gc][i];
      }
    if (skips) atomicAdd(&ctr[kFlagSkips], skips);
    if (aentries) atomicAdd(&ctr[kActiveEntries], aentries);
    if (nact) atomicAdd(&ctr[kActiveCount], nact);
    if (maxlen) atomicMax(&ctr[kMaxLen], maxlen);
  }
}

// ---------------------------------------------------------- locality order
// label(u) <- min(label(u), label of every out-neighbour), kLabelRounds times:
// the minimum id within 3 hops.  Vertices of one neighbourhood share a label,
// so scanning in (label, id) order keeps concurrently scanned lists
// overlapping and their rows resident in L2.  Results do not depend on it.
__global__ void k_label_step(uint64_t n, const uint64_t* __restrict__ off,
                             const uint32_t* __restrict__ cnt,
                             const uint64_t* __restrict__ key,
                             const uint32_t* __restrict__ lab_in,
                             uint32_t* __restrict__ lab_out, int identity) {
  const uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint32_t m = lab_in ? lab_in[u] : uint32_t(u);
  if (identity) {
    lab_out[u] = uint32_t(u);
    return;
  }
  const uint64_t b = off[u];
  const uint32_t U = cnt[u];
  for (uint32_t j = 0; j < U; ++j) {
    const uint32_t v = key_id(key[b + j]);
    const uint32_t l = lab_in ? lab_in[v] : v;
    m = l < m ? l : m;
  }
  lab_out[u] = m;
}

__global__ void k_order_keys(uint64_t n, const uint32_t* __restrict__ label,
                             uint64_t* __restrict__ okey) {
  const uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u < n) okey[u] = (uint64_t(label[u]) << 32) | u;
}

// longest lists first (ties by index): the persistent scan's tail is short
__global__ void k_len_keys(uint64_t n, const uint32_t* __restrict__ cnt,
                           uint64_t* __restrict__ okey) {
  const uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u < n) okey[u] = (uint64_t(0xFFFFFFFFu - cnt[u]) << 32) | u;
}

struct IsShortActive {
  const uint8_t* active;
  __host__ __device__ bool operator()(uint64_t k) const { return active[uint32_t(k)] == 1; }
};

// ------------------------------------------------------------------ apply
// Scatter emitted redirects into per-source buckets.
__global__ void k_pend_scatter(uint64_t span, const uint32_t* __restrict__ pend_src,
                               const uint64_t* __restrict__ pend_key,
                               const uint64_t* __restrict__ boff,
                               unsigned long long* __restrict__ bcur,
                               uint64_t* __restrict__ bkey) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < span;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = pend_src[e];
    if (s == kNone) continue;
    const uint64_t pos = boff[s] + atomicAdd(&bcur[s], 1ull);
    bkey[pos] = pend_key[e];
  }
}

// Append-if-absent decisions (builder.cpp:117-136 / :236-243), one warp per
// vertex, on a bucket sorted by key.  A proposal is dropped when it equals the
// previous proposal (duplicate redirects carry bit-identical keys, so keeping
// one equals the reference's sort + unique) or when the post list already
// holds its id (has_target, builder.cpp:22-26).  by_id = 0: every key is exact
// (reverse proposals on materialised lists), so the id test is a binary
// search for the same (dist, id); by_id = 1: redirect records carry pending
// distances (gram.cu) or the cached distances came from the caller, so the
// warp compares ids against the whole post list, 32 at a time.  brank =
// exclusive rank among kept proposals.
__global__ void __launch_bounds__(kBlock)
    k_apply_count(uint64_t n, const uint64_t* __restrict__ off,
                  const uint64_t* __restrict__ key, const uint32_t* __restrict__ post_cnt,
                  const uint64_t* __restrict__ boff, const uint64_t* __restrict__ bkey,
                  uint8_t* __restrict__ bflag, uint32_t* __restrict__ brank,
                  uint32_t* __restrict__ new_cnt, unsigned long long* __restrict__ ctr,
                  int count_inserted, int by_id) {
  const uint32_t lane = lane_id();
  unsigned long long inserted = 0;
  WARP_LOOP(u, n) {
    const uint64_t b0 = boff[u], b1 = boff[u + 1];
    const uint32_t pc = post_cnt[u];
    if (b0 == b1) {
      if (lane == 0) new_cnt[u] = pc;
      continue;
    }
    const uint64_t* P = key + off[u];
    uint32_t ins = 0;
    for (uint64_t xb = b0; xb < b1; xb += 32) {
      const uint64_t xi = xb + lane;
      const uint64_t k = xi < b1 ? bkey[xi] : kTomb;
      const bool dup = xi < b1 && xi > b0 && bkey[xi - 1] == k;
      bool present = false;
      if (by_id) {
        const uint32_t id = key_id(k);
        for (uint32_t j0 = 0; j0 < pc; j0 += 32) {
          const uint32_t pid = j0 + lane < pc ? key_id(P[j0 + lane]) : kNone;
#pragma unroll 8
          for (int q = 0; q < 32; ++q) present |= __shfl_sync(0xffffffffu, pid, q) == id;
        }
      } else if (xi < b1 && !dup) {
        const uint32_t pos = lower_bound(P, pc, k & ~1ull);
        present = pos < pc && (P[pos] >> 1) == (k >> 1);
      }
      const bool keep = xi < b1 && !dup && !present;
      if (xi < b1) bflag[xi] = keep ? 0 : 1;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (xi < b1) brank[xi] = ins + __popc(m & ((1u << lane) - 1));
      ins += __popc(m);
    }
    if (lane == 0) new_cnt[u] = pc + ins;
    inserted += lane == 0 ? ins : 0;
  }
  if (lane == 0 && inserted && count_inserted) atomicAdd(&ctr[kInserted], inserted);
}

// Next CSR = merge(post list, kept proposals), both sorted by key, so the
// output stays sorted.  Element positions come from binary searches.
__global__ void __launch_bounds__(kBlock)
    k_merge(uint64_t n, const uint64_t* __restrict__ off, const uint64_t* __restrict__ key,
            const uint32_t* __restrict__ post_cnt, const uint64_t* __restrict__ boff,
            const uint64_t* __restrict__ bkey, const uint8_t* __restrict__ bflag,
            const uint32_t* __restrict__ brank, const uint64_t* __restrict__ off_b,
            uint64_t* __restrict__ key_b) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint64_t* P = key + off[u];
    const uint32_t pc = post_cnt[u];
    uint64_t* dst = key_b + off_b[u];
    const uint64_t b0 = boff[u], b1 = boff[u + 1];
    const uint32_t nb = uint32_t(b1 - b0);
    const uint64_t* Bk = bkey + b0;
    if (nb == 0) {
      for (uint32_t j = lane; j < pc; j += 32) dst[j] = P[j];
      continue;
    }
    const uint32_t ins = uint32_t(off_b[u + 1] - off_b[u]) - pc;
    for (uint32_t j = lane; j < pc; j += 32) {
      const uint64_t k = P[j];
      const uint32_t lb = lower_bound(Bk, nb, k);
      const uint32_t r = lb < nb ? brank[b0 + lb] : ins;
      dst[j + r] = k;
    }
    for (uint32_t x = lane; x < nb; x += 32) {
      if (bflag[b0 + x]) continue;
      const uint64_t k = Bk[x];
      dst[brank[b0 + x] + lower_bound(P, pc, k)] = k;
    }
  }
}

// Dense CSR for the host: entry j of list u goes to doff[u] + j, unpacked
// into id / dist / fresh (graph.hpp NeighborEntry fields).
__global__ void __launch_bounds__(kBlock)
    k_export(uint64_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ cnt,
             const uint64_t* __restrict__ key, const uint64_t* __restrict__ doff,
             uint32_t* __restrict__ ids, float* __restrict__ dists,
             uint8_t* __restrict__ fresh) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint64_t* P = key + off[u];
    const uint64_t w = doff[u];
    const uint32_t U = cnt[u];
    for (uint32_t j = lane; j < U; j += 32) {
      const uint64_t k = P[j];
      ids[w + j] = key_id(k);
      dists[w + j] = __uint_as_float(uint32_t(k >> 32));
      fresh[w + j] = uint8_t(k & 1u);
    }
  }
}

// Copy lists without tombstones (order, hence sortedness, is preserved).
__global__ void __launch_bounds__(kBlock)
    k_compact(uint64_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ cnt,
              const uint64_t* __restrict__ key, const uint64_t* __restrict__ off_b,
              uint64_t* __restrict__ key_b) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint64_t* P = key + off[u];
    const uint32_t pc = cnt[u];
    uint64_t* dst = key_b + off_b[u];
    uint32_t w = 0;
    for (uint32_t j0 = 0; j0 < pc; j0 += 32) {
      const uint32_t j = j0 + lane;
      const uint64_t k = j < pc ? P[j] : kTomb;
      const bool live = k != kTomb;
      const unsigned m = __ballot_sync(0xffffffffu, live);
      if (live) dst[w + __popc(m & ((1u << lane) - 1))] = k;
      w += __popc(m);
    }
  }
}

// ----------------------------------------------------------- reverse phase
// add_reverse_edges, builder.cpp:228-243: every edge u->v proposes v->u with
// the same cached distance, flagged fresh, appended when absent.
__global__ void __launch_bounds__(kBlock)
    k_count_targets(uint64_t n, const uint64_t* __restrict__ off,
                    const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ key,
                    unsigned long long* __restrict__ bcnt) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint64_t b = off[u];
    const uint32_t U = cnt[u];
    for (uint32_t j = lane; j < U; j += 32) atomicAdd(&bcnt[key_id(key[b + j])], 1ull);
  }
}

// mode 0: reverse proposal key (dist, u, fresh); mode 1: in-edge key
// (dist bits << 32 | source) with the edge slot as payload (in_prune).
__global__ void __launch_bounds__(kBlock)
    k_scatter_targets(uint64_t n, const uint64_t* __restrict__ off,
                      const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ key,
                      const uint64_t* __restrict__ boff, unsigned long long* __restrict__ bcur,
                      uint64_t* __restrict__ bkey, uint32_t* __restrict__ bpay, int mode) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint64_t b = off[u];
    const uint32_t U = cnt[u];
    for (uint32_t j = lane; j < U; j += 32) {
      const uint64_t k = key[b + j];
      const uint32_t t = key_id(k);
      const uint64_t pos = boff[t] + atomicAdd(&bcur[t], 1ull);
      if (mode == 0) {
        bkey[pos] = make_key(key_dist(k), uint32_t(u), 1u);
      } else {
        bkey[pos] = (uint64_t(key_dbits(k)) << 32) | uint64_t(u);
        bpay[pos] = uint32_t(b + j);
      }
    }
  }
}

// segment ends: [begin, begin + len) where len = cnt or bucket size, or empty
// when the segment has <= R entries (R = 0: every non-empty segment)
__global__ void k_seg_end(uint64_t n, const uint64_t* __restrict__ begin,
                          const uint32_t* __restrict__ cnt,
                          const uint64_t* __restrict__ boff, uint32_t R,
                          uint64_t* __restrict__ seg_end) {
  uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint64_t len = cnt ? cnt[u] : boff[u + 1] - boff[u];
  seg_end[u] = begin[u] + (len > R ? len : 0);
}

// out_prune, builder.cpp:141-150: a list longer than R keeps its R nearest;
// lists are sorted, so that is a truncation.
__global__ void k_out_trunc(uint64_t n, uint32_t* __restrict__ cnt, uint32_t R) {
  uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u < n && cnt[u] > R) cnt[u] = R;
}

// in_prune, builder.cpp:162-176: in-edges of each target sorted by
// (dist, source); ranks >= R are deleted from their source lists.
__global__ void __launch_bounds__(kBlock)
    k_in_mark(uint64_t n, const uint64_t* __restrict__ boff,
              const uint32_t* __restrict__ bpay_s, uint64_t* __restrict__ key, uint32_t R) {
  const uint32_t lane = lane_id();
  WARP_LOOP(t, n) {
    const uint64_t b0 = boff[t], b1 = boff[t + 1];
    if (b1 - b0 <= R) continue;
    for (uint64_t r = b0 + R + lane; r < b1; r += 32) key[bpay_s[r]] = kTomb;
  }
}

__global__ void __launch_bounds__(kBlock)
    k_count_live(uint64_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                 const uint64_t* __restrict__ key, uint32_t* __restrict__ out) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint64_t b = off[u];
    const uint32_t U = cnt[u];
    uint32_t live = 0;
    for (uint32_t j = lane; j < U; j += 32) live += key[b + j] != kTomb;
    live = uint32_t(warp_sum(live));
    if (lane == 0) out[u] = live;
  }
}

// ------------------------------------------------------------ sharding
// Records exchanged between vertex owners are (dst, key)
// pairs: dst a global vertex id, key an entry key addressed to dst's list.

// redirects emitted by the scan (slot-indexed) -> compact records
__global__ void k_pend_records(uint64_t span, const uint32_t* __restrict__ pend_src,
                               const uint64_t* __restrict__ pend_key,
                               unsigned long long* __restrict__ cursor,
                               uint32_t* __restrict__ rdst, uint64_t* __restrict__ rkey) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < span;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = pend_src[e];
    if (s == kNone) continue;
    const uint64_t at = atomicAdd(cursor, 1ull);
    rdst[at] = s;
    rkey[at] = pend_key[e];
  }
}

// mode 0: reverse proposals (target, (dist, src, fresh)); mode 1: in-edges
// (target, (dist, src, 0)) -- src global
__global__ void __launch_bounds__(kBlock)
    k_edge_records(uint64_t nv, uint64_t v0, const uint64_t* __restrict__ off,
                   const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ key,
                   unsigned long long* __restrict__ cursor, uint32_t* __restrict__ rdst,
                   uint64_t* __restrict__ rkey, int mode) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, nv) {
    const uint64_t b = off[u];
    const uint32_t U = cnt[u];
    uint64_t at = 0;
    if (lane == 0 && U) at = atomicAdd(cursor, (unsigned long long)U);
    at = __shfl_sync(0xffffffffu, at, 0);
    for (uint32_t j = lane; j < U; j += 32) {
      const uint64_t k = key[b + j];
      rdst[at + j] = key_id(k);
      rkey[at + j] = make_key(key_dist(k), uint32_t(v0 + u), mode == 0 ? 1u : 0u);
    }
  }
}

// received records -> per-owned-vertex buckets
__global__ void k_rec_count(uint64_t nr, uint64_t v0, const uint32_t* __restrict__ rdst,
                            unsigned long long* __restrict__ bcnt) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nr;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(&bcnt[rdst[i] - v0], 1ull);
}

__global__ void k_rec_scatter(uint64_t nr, uint64_t v0, const uint32_t* __restrict__ rdst,
                              const uint64_t* __restrict__ rkey,
                              const uint64_t* __restrict__ boff,
                              unsigned long long* __restrict__ bcur, uint64_t* __restrict__ bkey) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nr;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t u = rdst[i] - v0;
    bkey[boff[u] + atomicAdd(&bcur[u], 1ull)] = rkey[i];
  }
}

// in_prune at the target's owner: bucket sorted by (dist, source); ranks >= R
// become deletion records (source, (dist, target, 0))
__global__ void __launch_bounds__(kBlock)
    k_inedge_select(uint64_t nv, uint64_t v0, const uint64_t* __restrict__ boff,
                    const uint64_t* __restrict__ bkey, uint32_t R,
                    unsigned long long* __restrict__ cursor, uint32_t* __restrict__ rdst,
                    uint64_t* __restrict__ rkey) {
  const uint32_t lane = lane_id();
  WARP_LOOP(t, nv) {
    const uint64_t b0 = boff[t], b1 = boff[t + 1];
    if (b1 - b0 <= R) continue;
    const uint64_t m = b1 - b0 - R;
    uint64_t at = 0;
    if (lane == 0) at = atomicAdd(cursor, (unsigned long long)m);
    at = __shfl_sync(0xffffffffu, at, 0);
    for (uint64_t r = lane; r < m; r += 32) {
      const uint64_t k = bkey[b0 + R + r];
      rdst[at + r] = key_id(k);
      rkey[at + r] = make_key(key_dist(k), uint32_t(v0 + t), 0u);
    }
  }
}

// deletion records at the source's owner: locate the (dist, target) entry.
// Positions are resolved for every record before any tombstone is written
// (a tombstone inside a sorted list would break concurrent binary searches).
__global__ void k_rec_locate(uint64_t nr, uint64_t v0, const uint32_t* __restrict__ rdst,
                             const uint64_t* __restrict__ rkey, const uint64_t* __restrict__ off,
                             const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ key,
                             uint64_t* __restrict__ slot) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nr;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t u = rdst[i] - v0;
    const uint64_t* P = key + off[u];
    const uint64_t k = rkey[i] & ~1ull;
    const uint32_t pos = lower_bound(P, cnt[u], k);
    slot[i] = (pos < cnt[u] && (P[pos] >> 1) == (k >> 1)) ? off[u] + pos : ~0ull;
  }
}

__global__ void k_tomb_slots(uint64_t nr, const uint64_t* __restrict__ slot,
                             uint64_t* __restrict__ key) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nr;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (slot[i] != ~0ull) key[slot[i]] = kTomb;
}

// per-destination-part counts of records sorted by dst: counts[p] = number of
// dst in [bounds[p], bounds[p+1])
__global__ void k_part_counts(uint64_t nr, const uint32_t* __restrict__ rdst,
                              const uint64_t* __restrict__ bounds, uint32_t parts,
                              unsigned long long* __restrict__ counts) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= parts) return;
  auto lb = [&](uint64_t v) {
    uint64_t lo = 0, hi = nr;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (rdst[mid] < v)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  counts[p] = lb(bounds[p + 1]) - lb(bounds[p]);
}

// ---- direct routing of staged records (rnndg_shard_route / rnndg_shard_push)
constexpr uint32_t kMaxParts = 64;
struct PushArgs {
  uint32_t* dst[kMaxParts];   // receive buffers of every part's owner (peer-mapped
  uint64_t* key[kMaxParts];   //   over NVLink when the owner is another device)
  uint64_t at[kMaxParts];     // where this shard's segment starts in them
  uint64_t bounds[kMaxParts + 1];
  uint32_t parts;
};

__device__ __forceinline__ uint32_t part_of(const uint64_t* bounds, uint32_t parts, uint32_t v) {
  uint32_t lo = 0, hi = parts;  // bounds[lo] <= v < bounds[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (bounds[mid] <= v)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// records per destination part, unsorted records (warp-aggregated by part)
__global__ void __launch_bounds__(256)
    k_route_counts(uint64_t nr, const uint32_t* __restrict__ rdst, PushArgs a,
                   unsigned long long* __restrict__ counts) {
  __shared__ unsigned long long s_cnt[kMaxParts];
  if (threadIdx.x < kMaxParts) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x; i0 < nr;
       i0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const bool has = i < nr;
    const uint32_t p = has ? part_of(a.bounds, a.parts, rdst[i]) : kMaxParts;
    const unsigned peers = __match_any_sync(0xffffffffu, p);
    if (has && lane_id() == uint32_t(__ffs(peers)) - 1u)
      atomicAdd(&s_cnt[p], (unsigned long long)__popc(peers));
  }
  __syncthreads();
  if (threadIdx.x < a.parts && s_cnt[threadIdx.x]) atomicAdd(&counts[threadIdx.x], s_cnt[threadIdx.x]);
}

// every staged record stored straight into its owner's receive buffers: the
// position inside this shard's segment comes from a local cursor per part
// (one atomic per warp and part), the stores go to peer memory
__global__ void __launch_bounds__(256)
    k_route_push(uint64_t nr, const uint32_t* __restrict__ rdst, const uint64_t* __restrict__ rkey,
                 PushArgs a, unsigned long long* __restrict__ cursor) {
  for (uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x; i0 < nr;
       i0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const bool has = i < nr;
    const uint32_t d = has ? rdst[i] : 0u;
    const uint32_t p = has ? part_of(a.bounds, a.parts, d) : kMaxParts;
    const unsigned peers = __match_any_sync(0xffffffffu, p);
    const uint32_t leader = uint32_t(__ffs(peers)) - 1u;
    unsigned long long at = 0;
    if (has && lane_id() == leader) at = atomicAdd(&cursor[p], (unsigned long long)__popc(peers));
    at = __shfl_sync(0xffffffffu, at, leader);
    if (has) {
      const uint64_t pos = a.at[p] + at + __popc(peers & ((1u << lane_id()) - 1u));
      a.dst[p][pos] = d;
      a.key[p][pos] = rkey[i];
    }
  }
}


// ------------------------------------------------------------- host glue

// one thread per item unless `cap` is given (then the kernel must be grid-stride)
unsigned grid_for(uint64_t items, unsigned block, unsigned cap = 0x7fffffffu) {
  uint64_t g = (items + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return unsigned(g);
}

unsigned warp_grid(rnndg_ctx* c, uint64_t items) {
  // one warp per item, persistent: at most 16 blocks per SM
  uint64_t need = (items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  uint64_t cap = uint64_t(sm_count(c)) * 16;
  if (need < 1) need = 1;
  return unsigned(need < cap ? need : cap);
}

void* cub_temp(rnndg_ctx* c, size_t bytes) { return c->cub_tmp.ensure(bytes); }

// exclusive scan of n counts into n+1 u64 offsets (out[n] = total; the input
// array must have n+1 readable slots, the last one's value is irrelevant)
void scan_u32(rnndg_ctx* c, const uint32_t* in, uint64_t* out, uint64_t n) {
  cub::TransformInputIterator<uint64_t, ToU64, const uint32_t*> it(in, ToU64{});
  size_t bytes = 0;
  RNNDG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, out, int64_t(n + 1), c->stream));
  void* tmp = cub_temp(c, bytes);
  RNNDG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, it, out, int64_t(n + 1), c->stream));
  c->launches += 1;
}

void scan_u64(rnndg_ctx* c, const unsigned long long* in, uint64_t* out, uint64_t n) {
  size_t bytes = 0;
  const uint64_t* ip = reinterpret_cast<const uint64_t*>(in);
  RNNDG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, ip, out, int64_t(n + 1), c->stream));
  void* tmp = cub_temp(c, bytes);
  RNNDG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, ip, out, int64_t(n + 1), c->stream));
  c->launches += 1;
}

// ------------------------------------------------------ segmented sort
// Segments [begin[u], end[u]) of keys_in sorted ascending into keys_out.
// Nearly all segments (redirect buckets, initial lists) hold a few dozen
// keys: one warp per segment sorts up to 32 keys in registers and up to 256
// in shared memory; longer segments are queued and sorted by one CTA each
// (in shared memory up to 4096 keys, in place in global memory beyond).  All
// with the "flip" bitonic network (every compare-exchange puts the minimum
// at the lower index), so a non-power-of-two segment is padded with virtual
// +inf keys.  Replaces cub::DeviceSegmentedSort (2.5% of a C3 1M build).
constexpr uint32_t kSegWarpCap = 256;
constexpr uint32_t kSegBlockCap = 4096;

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(v), m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(v >> 32), m);
  return (uint64_t(hi) << 32) | lo;
}

__device__ __forceinline__ void cmp_swap(uint64_t* a, uint32_t lo, uint32_t hi) {
  const uint64_t x = a[lo], y = a[hi];
  if (y < x) {
    a[lo] = y;
    a[hi] = x;
  }
}

// one flip-bitonic network over m (power of two) slots of buf; pairs whose
// upper index is >= lim are skipped (virtual +inf).  `t0`, `dt`: this
// thread's share of the m/2 pairs; `sync` separates the steps.
template <typename Sync>
__device__ __forceinline__ void bitonic_flip(uint64_t* buf, uint32_t m, uint32_t lim, uint32_t t0,
                                             uint32_t dt, Sync sync) {
  for (uint32_t k = 2; k <= m; k <<= 1) {
    const uint32_t half = k >> 1;
    for (uint32_t t = t0; t < m / 2; t += dt) {
      const uint32_t blk = t / half, o = t % half;
      const uint32_t lo = blk * k + o, hi = blk * k + k - 1 - o;
      if (hi < lim) cmp_swap(buf, lo, hi);
    }
    sync();
    for (uint32_t j = half >> 1; j; j >>= 1) {
      for (uint32_t t = t0; t < m / 2; t += dt) {
        const uint32_t lo = (t / j) * 2 * j + t % j, hi = lo + j;
        if (hi < lim) cmp_swap(buf, lo, hi);
      }
      sync();
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_seg_sort_warp(const uint64_t* __restrict__ kin,
                                                         uint64_t* __restrict__ kout,
                                                         uint64_t nseg,
                                                         const uint64_t* __restrict__ begin,
                                                         const uint64_t* __restrict__ end,
                                                         uint32_t* __restrict__ big,
                                                         const unsigned long long* nseg_dev) {
  __shared__ uint64_t sh[kWarpsPerBlock][kSegWarpCap];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  if (nseg_dev && *nseg_dev < nseg) nseg = *nseg_dev;  // segments counted on the device
  for (uint64_t s = warp; s < nseg; s += nwarps) {
    const uint64_t b = begin[s];
    const uint32_t len = uint32_t(end[s] - b);
    if (len <= 1) {  // most buckets of a late pass are empty
      if (len == 1 && lane == 0) kout[b] = kin[b];
    } else if (len <= 32) {
      uint64_t v = lane < len ? kin[b + lane] : ~0ull;
      for (uint32_t k = 2; k <= 32; k <<= 1) {
        uint64_t p = shfl_xor_u64(v, int(k - 1));
        bool lower = (lane & (k >> 1)) == 0;
        v = lower ? (p < v ? p : v) : (p < v ? v : p);
        for (uint32_t j = k >> 2; j; j >>= 1) {
          p = shfl_xor_u64(v, int(j));
          lower = (lane & j) == 0;
          v = lower ? (p < v ? p : v) : (p < v ? v : p);
        }
      }
      if (lane < len) kout[b + lane] = v;
    } else if (len <= kSegWarpCap) {
      uint32_t m = 64;
      while (m < len) m <<= 1;
      uint64_t* buf = sh[wib];
      for (uint32_t i = lane; i < m; i += 32) buf[i] = i < len ? kin[b + i] : ~0ull;
      __syncwarp();
      bitonic_flip(buf, m, m, lane, 32u, [] { __syncwarp(); });
      for (uint32_t i = lane; i < len; i += 32) kout[b + i] = buf[i];
      __syncwarp();
    } else if (lane == 0) {
      const uint32_t x = atomicAdd(big, 1u);
      big[1 + x] = uint32_t(s);
    }
  }
}

__global__ void __launch_bounds__(1024) k_seg_sort_block(const uint64_t* __restrict__ kin,
                                                        uint64_t* __restrict__ kout,
                                                        const uint64_t* __restrict__ begin,
                                                        const uint64_t* __restrict__ end,
                                                        const uint32_t* __restrict__ big) {
  __shared__ uint64_t sh[kSegBlockCap];
  const uint32_t nb = big[0];
  for (uint32_t x = blockIdx.x; x < nb; x += gridDim.x) {
    const uint32_t s = big[1 + x];
    const uint64_t b = begin[s];
    const uint32_t len = uint32_t(end[s] - b);
    uint32_t m = 2;
    while (m < len) m <<= 1;
    const bool in_smem = m <= kSegBlockCap;
    uint64_t* buf = in_smem ? sh : kout + b;
    for (uint32_t i = threadIdx.x; i < (in_smem ? m : len); i += blockDim.x)
      buf[i] = i < len ? kin[b + i] : ~0ull;
    __syncthreads();
    bitonic_flip(buf, m, in_smem ? m : len, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    if (in_smem)
      for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) kout[b + i] = sh[i];
    __syncthreads();
  }
}

void seg_sort_keys(rnndg_ctx* c, const uint64_t* keys_in, uint64_t* keys_out, uint64_t span,
                   uint64_t nseg, const uint64_t* begin, const uint64_t* end,
                   const unsigned long long* nseg_dev = nullptr) {
  if (span == 0 || nseg == 0) return;
  static const bool use_cub = [] {
    const char* e = std::getenv("RNNDG_CUBSORT");
    return e && e[0] == '1';
  }();
  if (!use_cub) {
    uint32_t* big = c->seg_big.ensure(nseg + 1);
    RNNDG_CUDA(cudaMemsetAsync(big, 0, sizeof(uint32_t), c->stream));
    RNNDG_LAUNCH(c, k_seg_sort_warp, nseg_dev ? unsigned(sm_count(c)) * 8u : warp_grid(c, nseg),
                 kBlock, 0, keys_in, keys_out, nseg, begin, end, big, nseg_dev);
    RNNDG_LAUNCH(c, k_seg_sort_block, unsigned(sm_count(c)), 1024, 0, keys_in, keys_out, begin,
                 end, big);
    return;
  }
  if (nseg_dev) {  // CUB needs the count on the host
    unsigned long long h = 0;
    RNNDG_CUDA(cudaMemcpyAsync(&h, nseg_dev, 8, cudaMemcpyDeviceToHost, c->stream));
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
    nseg = std::min<uint64_t>(nseg, h);
    if (nseg == 0) return;
  }
  if (span > uint64_t(INT32_MAX)) throw CudaError("segmented sort span exceeds 2^31");
  size_t bytes = 0;
  RNNDG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, keys_in, keys_out, int(span),
                                                int(nseg), begin, end, c->stream));
  void* tmp = cub_temp(c, bytes);
  RNNDG_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, keys_in, keys_out, int(span),
                                                int(nseg), begin, end, c->stream));
  c->launches += 3;
}

void seg_sort_pairs(rnndg_ctx* c, const uint64_t* kin, uint64_t* kout, const uint32_t* vin,
                    uint32_t* vout, uint64_t span, uint64_t nseg, const uint64_t* begin,
                    const uint64_t* end) {
  if (span == 0 || nseg == 0) return;
  if (span > uint64_t(INT32_MAX)) throw CudaError("segmented sort span exceeds 2^31");
  size_t bytes = 0;
  RNNDG_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, kin, kout, vin, vout,
                                                 int(span), int(nseg), begin, end, c->stream));
  void* tmp = cub_temp(c, bytes);
  RNNDG_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp, bytes, kin, kout, vin, vout, int(span),
                                                 int(nseg), begin, end, c->stream));
  c->launches += 3;
}

uint64_t read_u64(rnndg_ctx* c, const uint64_t* dev) {
  uint64_t v = 0;
  RNNDG_CUDA(cudaMemcpyAsync(&v, dev, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  return v;
}

template <class T>
void zero(rnndg_ctx* c, T* p, uint64_t count, int value = 0) {
  if (count) RNNDG_CUDA(cudaMemsetAsync(p, value, count * sizeof(T), c->stream));
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  RNNDG_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

void ensure_scratch(rnndg_ctx* c) {
  const uint64_t n = c->nv, span = c->span ? c->span : 1;
  c->active.ensure(n);
  c->act_list.ensure(2 * n);
  c->post_cnt.ensure(n + 1);
  c->cnt_b.ensure(n + 1);
  c->seg_end.ensure(n);
  c->bcnt.ensure(n + 1);
  c->bcur.ensure(n);
  c->boff.ensure(n + 1);
  c->counters.ensure(kNumCounters);
  c->work.ensure(16);
  c->label.ensure(2 * n);
  c->okey.ensure(2 * n);
  c->act_small.ensure(n);
  c->gram_q.ensure(kSizeClasses * n + 1);
  c->key_s.ensure(span);
  c->pend_src.ensure(span);
  c->pend_key.ensure(span);
  c->touch.ensure(span);
  c->kpos_g.ensure(span);
  c->bkey.ensure(span);
  c->bkey_s.ensure(span);
  c->bflag.ensure(span);
  c->brank.ensure(span);
}

// Sort each bucket [boff[u], boff[u+1]) of bkey into bkey_s.
void sort_buckets(rnndg_ctx* c, uint64_t total) {
  if (total == 0) return;
  seg_sort_keys(c, c->bkey.p, c->bkey_s.p, total, c->nv, c->boff.p, c->boff.p + 1);
}

// Build graph B = merge(current lists with post_cnt, sorted buckets) and make
// it the current graph.  New counts must be in c->cnt_b.
void merge_and_swap(rnndg_ctx* c, const uint32_t* post_cnt) {
  const uint64_t n = c->nv;
  c->off_b.ensure(n + 1);
  scan_u32(c, c->cnt_b.p, c->off_b.p, n);
  const uint64_t total = read_u64(c, c->off_b.p + n);
  c->key_b.ensure(total ? total : 1);
  RNNDG_LAUNCH(c, k_merge, warp_grid(c, n), kBlock, 0, n, c->off.p, c->key.p, post_cnt,
               c->boff.p, c->bkey_s.p, c->bflag.p, c->brank.p, c->off_b.p, c->key_b.p);
  c->off.swap(c->off_b);
  c->key.swap(c->key_b);
  c->cnt.swap(c->cnt_b);
  c->span = total;
}

// lists longer than this go to the hub kernel (RNNDG_UCAP, at most
// kScanUcap, the short kernel's shared-memory capacity).  C3 1M with one CTA
// per hub: 512 -> 2.51 s, 256 -> 2.46 s, 128 -> 2.56 s, 64 -> 3.25 s; with
// the current kernels: 192 -> 2.051 s, 256 -> 1.999 s, 320 -> 1.989 s,
// 384 -> 1.976 s, 448 -> 1.985 s, 512 -> 2.011 s.
uint32_t hub_threshold() {
  static const uint32_t v = [] {
    const char* e = std::getenv("RNNDG_UCAP");
    const int x = e ? std::atoi(e) : 384;
    return uint32_t(x >= 32 && x <= int(kScanUcap) ? x : 384);
  }();
  return v;
}

// short lists longer than this are scanned first (their walks are the
// longest of the short-list kernel, so starting them last would leave them
// as the tail of the small passes); RNNDG_LS, 0 = plain index order.  C3 1M:
// off 1.975 s, 32 1.962 s, 48 1.955 s, 64 1.954 s, 96 1.955 s, 128 1.956 s,
// 200 1.958 s
uint32_t long_short_threshold() {
  static const uint32_t v = [] {
    const char* e = std::getenv("RNNDG_LS");
    const long x = e ? std::atol(e) : 64;
    return x <= 0 ? 0xFFFFFFFFu : uint32_t(x);
  }();
  return v;
}

// hub lists longer than this are walked by a whole thread-block cluster
// (k_scan_hub phase 1); shorter hubs by one CTA each (RNNDG_BIG_HUB; 0 = no
// cooperative walks)
uint32_t big_hub_threshold(rnndg_ctx* c) {
  // the one-CTA-per-hub schedules have no cooperative phase
  if (hub_cluster_size(c) == 0) return 0xFFFFFFFFu;
  static const uint32_t v = [] {
    const char* e = std::getenv("RNNDG_BIG_HUB");
    const long x = e ? std::atol(e) : 1024;
    return x <= 0 ? 0xFFFFFFFFu : uint32_t(x < 256 ? 256 : x);
  }();
  return v;
}

// Order of the short active lists into c->act_small (RNNDG_ORDER, default
// vertex index); count into work[2] (read by the scan kernel).
void locality_order(rnndg_ctx* c) {
  const uint64_t n = c->nv;
  if (n == 0) {
    zero(c, c->work.p + 2, 1);
    return;
  }
  // RNNDG_ORDER: 0 = vertex index (default), 1 = locality labels (3 label
  // rounds + radix sort; no faster scan at C3 1M once hubs use every SM, and
  // 40 ms per build of its own), 2 = longest list first
  static const int mode = [] {
    const char* e = std::getenv("RNNDG_ORDER");
    return e ? std::atoi(e) : 0;
  }();
  uint32_t* la = c->label.p;
  uint32_t* lb = c->label.p + n;
  uint64_t* ok = c->okey.p;
  uint64_t* ok2 = c->okey.p + n;
  size_t bytes = 0;
  if (mode == 0) {
    // vertex index order: select straight from the index sequence
    int* nsel0 = reinterpret_cast<int*>(c->work.p + 2);
    cub::CountingInputIterator<uint64_t> idx(0);
    RNNDG_CUDA(cub::DeviceSelect::If(nullptr, bytes, idx, c->act_small.p, nsel0, int64_t(n),
                                     IsShortActive{c->active.p}, c->stream));
    RNNDG_CUDA(cub::DeviceSelect::If(cub_temp(c, bytes), bytes, idx, c->act_small.p, nsel0,
                                     int64_t(n), IsShortActive{c->active.p}, c->stream));
    c->launches += 2;
    return;
  } else {
    if (mode == 2) {
      RNNDG_LAUNCH(c, k_len_keys, grid_for(n, 256), 256, 0, n, c->cnt.p, ok);
    } else {
      // a shard's lists point at vertices it does not own: order by index there
      RNNDG_LAUNCH(c, k_label_step, grid_for(n, 256), 256, 0, n, c->off.p, c->cnt.p, c->key.p,
                   nullptr, la, int(c->partitioned));
      for (int r = 1; r < kLabelRounds && !c->partitioned; ++r) {
        RNNDG_LAUNCH(c, k_label_step, grid_for(n, 256), 256, 0, n, c->off.p, c->cnt.p,
                     c->key.p, la, lb, 0);
        std::swap(la, lb);
      }
      RNNDG_LAUNCH(c, k_order_keys, grid_for(n, 256), 256, 0, n, la, ok);
    }
    RNNDG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, ok, ok2, int64_t(n), 0, 64,
                                              c->stream));
    RNNDG_CUDA(cub::DeviceRadixSort::SortKeys(cub_temp(c, bytes), bytes, ok, ok2, int64_t(n), 0,
                                              64, c->stream));
    c->launches += 8;
  }
  int* nsel = reinterpret_cast<int*>(c->work.p + 2);
  bytes = 0;
  RNNDG_CUDA(cub::DeviceSelect::If(nullptr, bytes, ok2, c->act_small.p, nsel, int64_t(n),
                                   IsShortActive{c->active.p}, c->stream));
  RNNDG_CUDA(cub::DeviceSelect::If(cub_temp(c, bytes), bytes, ok2, c->act_small.p, nsel,
                                   int64_t(n), IsShortActive{c->active.p}, c->stream));
  c->launches += 2;
}

}  // namespace

int sm_count(rnndg_ctx* c) {
  static thread_local int cached_dev = -1, cached = 0;
  if (cached_dev != c->device) {
    RNNDG_CUDA(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, c->device));
    cached_dev = c->device;
  }
  return cached;
}

void op_random_init(rnndg_ctx* c, uint32_t S, uint64_t seed) {
  const uint64_t n = c->n, nv = c->nv;
  if (n < 2) throw ParamError("random_init: need at least 2 vectors");
  if (S < 1 || S > n - 1) throw ParamError("random_init: S out of [1, n-1]");
  c->span = nv * S;
  c->off.ensure(nv + 1);
  c->cnt.ensure(nv + 1);
  c->key.ensure(c->span ? c->span : 1);
  RNNDG_LAUNCH(c, k_fill_offsets, grid_for(nv + 1, 256), 256, 0, nv, S, c->off.p, c->cnt.p);
  if (nv) {
    // ids here; the S cached distances per vertex with the scan's quad L2 on
    // the chain-blocked rows (coalesced 128-byte lines per quad)
    RNNDG_LAUNCH(c, k_random_init, grid_for(nv, 128), 128, 0, n, c->v0, nv, S, seed,
                 c->key.p);
    launch_init_dists(c, S);
  }
  c->has_graph = true;
  c->pending = false;
  c->has_distances = true;
  c->exact_dists = true;
  c->bulk_fresh = true;
  c->init_fresh = true;
  op_sort_lists(c);  // establish the sorted-list invariant
}

// ------------------------------------------------------ pending distances
// Redirected entries arrive with a pending distance (gram.cu item 5).  The
// Gram walk computes them while streaming the list; everywhere else they are
// resolved here: exact l2_sq(u, v) by a quad per pending entry (quad.cuh,
// bit-identical to rnnd::l2_sq), then the list re-sorted.  [mat_b[u],
// mat_e[u]) is the list of u when it needs it, else empty.
__global__ void __launch_bounds__(kBlock)
    k_mark_pending(uint64_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                   const uint64_t* __restrict__ key, uint64_t* __restrict__ mat_b,
                   uint64_t* __restrict__ mat_e, unsigned long long* __restrict__ count) {
  for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
       u += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = off[u];
    const uint32_t U = cnt[u];
    if (U && key_pending(key[b + U - 1])) {
      const unsigned long long x = atomicAdd(count, 1ull);
      mat_b[x] = b;
      mat_e[x] = b + U;
      mat_e[n + x] = u;
    }
  }
}

__global__ void __launch_bounds__(kBlock)
    k_resolve_pending(uint64_t n, uint64_t v0, const uint64_t* __restrict__ mat_b,
                      const uint64_t* __restrict__ mat_e, const unsigned long long* __restrict__ count,
                      uint64_t* __restrict__ key, Row row) {
  __shared__ uint32_t q[kWarpsPerBlock][32];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5, quad = lane >> 2, chain = lane & 3;
  const uint64_t nq = *count;
  WARP_LOOP(x, nq) {
    const uint64_t b = mat_b[x], e = mat_e[x], u = mat_e[n + x];
    const float* xu = row.xp + (v0 + u) * row.stride;
    for (uint64_t j0 = b; j0 < e; j0 += 32) {
      const bool pend = j0 + lane < e && key_pending(key[j0 + lane]);
      const unsigned m = __ballot_sync(0xffffffffu, pend);
      if (pend) q[wib][__popc(m & ((1u << lane) - 1u))] = uint32_t(j0 + lane - b);
      __syncwarp();
      const uint32_t np = __popc(m);
      for (uint32_t k0 = 0; k0 < np; k0 += 8) {
        const uint32_t k = k0 + quad;
        const uint64_t slot = b + q[wib][k < np ? k : k0];
        const uint64_t kv = key[slot];
        const float d = quad_l2<false>(row.xp + uint64_t(key_id(kv)) * row.stride, xu, chain,
                                       row.nblk, row.ntail);
        if (k < np && chain == 0) key[slot] = make_key(d, key_id(kv), key_fresh(kv));
      }
      __syncwarp();
    }
  }
}

// after k_resolve_merge: queue entries it finished become empty ranges,
// the ones it flagged (tail too long) keep theirs for resolve_pending
__global__ void __launch_bounds__(kBlock)
    k_flagged_only(uint64_t n, uint64_t* __restrict__ mat_b, uint64_t* __restrict__ mat_e,
                   const unsigned long long* __restrict__ count) {
  const uint64_t nq = *count;
  for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < nq;
       x += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t u = mat_e[n + x];
    if (u >> 63) {
      mat_e[n + x] = u & ~(1ull << 63);
    } else {
      mat_e[x] = mat_b[x];
    }
  }
}

// Hub lists with pending entries, one CTA per list: the pending tail (it
// sorts last) is resolved by the CTA's quads, sorted in shared memory and
// merged with the sorted prefix by ranks -- O(U) instead of a full segmented
// sort of a list of thousands.  Tails longer than kMergeCap are left for
// the segmented sort (flagged by setting mat_e[n + x] |= 1 << 63).
constexpr uint32_t kMergeCap = 2048;
constexpr int kMergeThreads = 256;

__global__ void __launch_bounds__(kMergeThreads)
    k_resolve_merge(uint64_t n, uint64_t v0, const uint64_t* __restrict__ mat_b,
                    uint64_t* __restrict__ mat_e, const unsigned long long* __restrict__ count,
                    uint64_t* __restrict__ key, uint64_t* __restrict__ scratch, Row row) {
  __shared__ uint64_t tail[kMergeCap];
  __shared__ uint32_t s_p0;
  const uint32_t tid = threadIdx.x, lane = lane_id(), quad = tid >> 2, chain = lane & 3;
  const uint64_t nq = *count;
  for (uint64_t x = blockIdx.x; x < nq; x += gridDim.x) {
    const uint64_t b = mat_b[x], U = mat_e[x] - b, u = mat_e[n + x];
    uint64_t* L = key + b;
    if (tid == 0) {  // first pending position: pending keys are the largest
      uint64_t lo = 0, hi = U;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (key_pending(L[mid])) hi = mid; else lo = mid + 1;
      }
      s_p0 = uint32_t(lo);
    }
    __syncthreads();
    const uint32_t p0 = s_p0, p = uint32_t(U) - p0;
    if (p > kMergeCap) {  // rare: the segmented sort after this kernel
      if (tid == 0) mat_e[n + x] = u | (1ull << 63);
      __syncthreads();
      continue;
    }
    for (uint32_t i = tid; i < p; i += kMergeThreads) tail[i] = L[p0 + i];
    __syncthreads();
    const float* xu = row.xp + (v0 + u) * uint64_t(row.stride);
    for (uint32_t b0 = 0; b0 < p; b0 += kMergeThreads / 4) {
      const uint32_t i = b0 + quad;
      const uint64_t kv = tail[i < p ? i : 0];
      const float d = quad_l2<false>(row.xp + uint64_t(key_id(kv)) * row.stride, xu, chain,
                                     row.nblk, row.ntail);
      if (i < p && chain == 0) tail[i] = make_key(d, key_id(kv), key_fresh(kv));
    }
    uint32_t m = 1;
    while (m < p) m <<= 1;
    for (uint32_t i = p + tid; i < m; i += kMergeThreads) tail[i] = kTomb;
    __syncthreads();
    for (uint32_t k = 2; k <= m; k <<= 1)
      for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
        for (uint32_t i = tid; i < m; i += kMergeThreads) {
          const uint32_t l = i ^ jj;
          if (l > i) {
            const uint64_t a = tail[i], c = tail[l];
            if (((i & k) == 0) ? (a > c) : (a < c)) {
              tail[i] = c;
              tail[l] = a;
            }
          }
        }
        __syncthreads();
      }
    // merge by ranks into the scratch slice, then back
    uint64_t* S = scratch + b;
    for (uint32_t j = tid; j < p0; j += kMergeThreads) {
      const uint64_t kj = L[j];
      uint32_t lo = 0, hi = p;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tail[mid] < kj) lo = mid + 1; else hi = mid;
      }
      S[j + lo] = kj;
    }
    for (uint32_t i = tid; i < p; i += kMergeThreads) {
      const uint64_t kt = tail[i];
      uint64_t lo = 0, hi = p0;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (L[mid] < kt) lo = mid + 1; else hi = mid;
      }
      S[i + lo] = kt;
    }
    __syncthreads();
    for (uint64_t j = tid; j < U; j += kMergeThreads) L[j] = S[j];
    __syncthreads();
  }
}

namespace {
void resolve_pending(rnndg_ctx* c, const unsigned long long* count);
void resolve_pending_hubs(rnndg_ctx* c, const unsigned long long* count);
}  // namespace

// Scan phase of a pass: counters zeroed, active vertices marked, locality
// order, distance stage.  Redirects end up in pend_src/pend_key by slot.
void op_scan_phase(rnndg_ctx* c) {
  const uint64_t n = c->nv;
  ensure_scratch(c);
  unsigned long long* ctr = c->counters.p;
  zero(c, ctr, kNumCounters);
  zero(c, c->work.p, 16);
  zero(c, c->pend_src.p, c->span, 0xFF);
  zero(c, c->touch.p, c->span);
  zero(c, c->bcnt.p, n + 1);
  zero(c, c->bcur.p, n);
  RNNDG_CUDA(cudaEventRecord(c->ev[0], c->stream));
  // size classes of the per-class queues: the Gram walk's tiles, or the
  // shared-memory walk's regions
  uint32_t cls[kSizeClasses] = {16, 32, 64, 128, 128, 128, 128, 128};
  if (!gram_cap() && rowwalk_cap(c)) rowwalk_classes(c, cls);
  ClassBounds gb;
  for (int i = 0; i < kSizeClasses - 1; ++i) gb.b[i] = cls[i];
  if (n)
    RNNDG_LAUNCH(c, k_mark_active, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
                 c->active.p, c->act_list.p, c->post_cnt.p, ctr, hub_threshold(),
                 big_hub_threshold(c), bsp_rounds() ? bsp_max_len() : long_short_threshold(),
                 gram_cap() ? gram_cap() : rowwalk_cap(c), gb, c->gram_q.p,
                 c->pending ? c->mat_b.ensure(n) : nullptr,
                 c->pending ? c->mat_e.ensure(2 * n) : nullptr);
  if (c->pending && n) {
    prepare_chain_layout(c);
    resolve_pending_hubs(c, c->counters.p + kMatCount);
  }
  locality_order(c);
  RNNDG_CUDA(cudaEventRecord(c->ev[1], c->stream));
  launch_scan(c, c->work.p);
  RNNDG_CUDA(cudaEventRecord(c->ev[2], c->stream));
}

// Apply phase of a single-context pass: bucket the redirects by source,
// append-if-absent, merge into the next CSR.
void op_apply_local(rnndg_ctx* c) {
  const uint64_t n = c->nv;
  unsigned long long* ctr = c->counters.p;
  scan_u64(c, c->bcnt.p, c->boff.p, n);
  RNNDG_LAUNCH(c, k_pend_scatter, grid_for(c->span, 256, 148 * 64), 256, 0, c->span,
               c->pend_src.p, c->pend_key.p, c->boff.p, c->bcur.p, c->bkey.p);
  sort_buckets(c, c->span);
  RNNDG_LAUNCH(c, k_apply_count, warp_grid(c, n), kBlock, 0, n, c->off.p, c->key.p,
               c->post_cnt.p, c->boff.p, c->bkey_s.p, c->bflag.p, c->brank.p, c->cnt_b.p, ctr, 1,
               int(gram_cap() != 0 || !c->exact_dists));
  // redirect records carry pending distances when the Gram walk is on
  if (gram_cap()) c->pending = true;
  merge_and_swap(c, c->post_cnt.p);
}

void op_read_counters(rnndg_ctx* c, rnndg_counts* out, double* t_scan, double* t_sort,
                      double* t_apply, uint64_t* touched, uint64_t* active_entries) {
  RNNDG_CUDA(cudaEventRecord(c->ev[3], c->stream));
  unsigned long long h[kNumCounters];
  RNNDG_CUDA(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  if (out) {
    out->removed = h[kRemoved];
    out->inserted = h[kInserted];
    out->flag_skips = h[kFlagSkips];
    out->pair_checks = h[kPairChecks];
  }
  if (t_sort) *t_sort += elapsed_ms(c->ev[0], c->ev[1]) * 1e-3;
  if (t_scan) *t_scan += elapsed_ms(c->ev[1], c->ev[2]) * 1e-3;
  if (t_apply) *t_apply += elapsed_ms(c->ev[2], c->ev[3]) * 1e-3;
  if (touched) *touched += h[kTouched];
  c->hubs_prev = h[kLargeCount] + h[kBigCount];
  if (active_entries) *active_entries += h[kActiveEntries];
  if (c->trace)
    std::fprintf(stderr,
                 "[rnndg] pass active=%llu large=%llu maxlen=%llu entries=%llu checks=%llu "
                 "evals=%llu hub_evals=%llu removed=%llu inserted=%llu touched=%llu "
                 "order=%.3fms scan=%.3fms apply=%.3fms hubk=%.3fms shortk=%.3fms "
                 "gram=%llu/%llu/%llu/%llu amb=%llu exact=%llu gramk=%.3fms\n",
                 h[kActiveCount], h[kLargeCount] + h[kBigCount], h[kMaxLen], h[kActiveEntries], h[kPairChecks],
                 h[kEvalPairs], h[kEvalHub],
                 h[kRemoved], h[kInserted], h[kTouched], elapsed_ms(c->ev[0], c->ev[1]),
                 elapsed_ms(c->ev[1], c->ev[2]), elapsed_ms(c->ev[2], c->ev[3]),
                 elapsed_ms(c->ev[1], c->ev_scan[0]), elapsed_ms(c->ev[1], c->ev_scan[1]),
                 h[kGram0], h[kGram1], h[kGram2], h[kGram3], h[kGramAmb], h[kGramExact],
                 gram_cap() ? elapsed_ms(c->ev[1], c->ev_scan[2]) : 0.f);
  if (c->trace) gram_trace(c);
}

namespace {

// memcpy of a large host range on several threads (pinned staging -> the
// caller's pageable arrays)
void par_copy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kChunk = size_t(8) << 20;
  const unsigned hw = std::thread::hardware_concurrency();
  const size_t nt = std::min<size_t>(hw ? hw : 1, std::min<size_t>(16, bytes / kChunk + 1));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + nt - 1) / nt;
  for (size_t t = 0; t < nt; ++t) {
    const size_t a = t * per, b = std::min(bytes, a + per);
    if (a >= b) break;
    th.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
  }
  for (auto& x : th) x.join();
}

}  // namespace

// Graph export (rnnd::AdjacencyGraph as CSR): compacted on the device, copied
// to a pinned staging area in one pass at PCIe speed, then into the caller's
// arrays by a multi-threaded memcpy.
uint64_t op_export(rnndg_ctx* c, uint64_t* offsets, uint32_t* ids, float* dists,
                   uint8_t* fresh) {
  materialize_pending(c);
  const uint64_t n = c->nv;
  c->ex_off.ensure(n + 1);
  scan_u32(c, c->cnt.p, c->ex_off.p, n);
  uint64_t m = 0;
  RNNDG_CUDA(cudaMemcpyAsync(&m, c->ex_off.p + n, 8, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  if (!(offsets || ids || dists || fresh)) return m;
  const size_t b_off = offsets ? (n + 1) * 8 : 0, b_ids = ids ? m * 4 : 0,
               b_d = dists ? m * 4 : 0, b_f = fresh ? m : 0;
  const size_t total = b_off + b_ids + b_d + b_f;
  if (total > c->host_stage_bytes) {
    if (c->host_stage) RNNDG_CUDA(cudaFreeHost(c->host_stage));
    c->host_stage = nullptr;
    c->host_stage_bytes = 0;
    RNNDG_CUDA(cudaHostAlloc(&c->host_stage, total, cudaHostAllocDefault));
    c->host_stage_bytes = total;
  }
  char* st = static_cast<char*>(c->host_stage);
  if (m && (ids || dists || fresh)) {
    c->ex_ids.ensure(m);
    c->ex_dists.ensure(m);
    c->ex_fresh.ensure(m);
    RNNDG_LAUNCH(c, k_export, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
                 c->ex_off.p, c->ex_ids.p, c->ex_dists.p, c->ex_fresh.p);
    if (ids)
      RNNDG_CUDA(cudaMemcpyAsync(st + b_off, c->ex_ids.p, b_ids, cudaMemcpyDeviceToHost,
                                 c->stream));
    if (dists)
      RNNDG_CUDA(cudaMemcpyAsync(st + b_off + b_ids, c->ex_dists.p, b_d, cudaMemcpyDeviceToHost,
                                 c->stream));
    if (fresh)
      RNNDG_CUDA(cudaMemcpyAsync(st + b_off + b_ids + b_d, c->ex_fresh.p, b_f,
                                 cudaMemcpyDeviceToHost, c->stream));
  }
  if (offsets)
    RNNDG_CUDA(cudaMemcpyAsync(st, c->ex_off.p, b_off, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  if (offsets) par_copy(offsets, st, b_off);
  if (m && ids) par_copy(ids, st + b_off, b_ids);
  if (m && dists) par_copy(dists, st + b_off + b_ids, b_d);
  if (m && fresh) par_copy(fresh, st + b_off + b_ids + b_d, b_f);
  return m;
}

void op_update_pass(rnndg_ctx* c, rnndg_counts* out, double* t_scan, double* t_sort,
                    double* t_apply, uint64_t* touched, uint64_t* active_entries) {
  op_scan_phase(c);
  op_apply_local(c);
  op_read_counters(c, out, t_scan, t_sort, t_apply, touched, active_entries);
}

namespace {

void out_prune(rnndg_ctx* c, uint32_t R) {
  RNNDG_LAUNCH(c, k_out_trunc, grid_for(c->nv, 256), 256, 0, c->nv, c->cnt.p, R);
}

void in_prune(rnndg_ctx* c, uint32_t R) {
  const uint64_t n = c->nv;
  zero(c, c->bcnt.p, n + 1);
  zero(c, c->bcur.p, n);
  RNNDG_LAUNCH(c, k_count_targets, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
               c->bcnt.p);
  scan_u64(c, c->bcnt.p, c->boff.p, n);
  const uint64_t m = read_u64(c, c->boff.p + n);
  if (c->span >= (1ull << 32)) throw CudaError("in_prune: edge slots exceed 2^32");
  c->bkey.ensure(m ? m : 1);
  c->bkey_s.ensure(m ? m : 1);
  c->bpay.ensure(m ? m : 1);
  c->bpay_s.ensure(m ? m : 1);
  RNNDG_LAUNCH(c, k_scatter_targets, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p,
               c->key.p, c->boff.p, c->bcur.p, c->bkey.p, c->bpay.p, 1);
  RNNDG_LAUNCH(c, k_seg_end, grid_for(n, 256), 256, 0, n, c->boff.p, nullptr, c->boff.p, R,
               c->seg_end.p);
  seg_sort_pairs(c, c->bkey.p, c->bkey_s.p, c->bpay.p, c->bpay_s.p, m, n, c->boff.p,
                 c->seg_end.p);
  RNNDG_LAUNCH(c, k_in_mark, warp_grid(c, n), kBlock, 0, n, c->boff.p, c->bpay_s.p, c->key.p, R);
  RNNDG_LAUNCH(c, k_count_live, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
               c->cnt_b.p);
  c->off_b.ensure(n + 1);
  scan_u32(c, c->cnt_b.p, c->off_b.p, n);
  const uint64_t total = read_u64(c, c->off_b.p + n);
  c->key_b.ensure(total ? total : 1);
  RNNDG_LAUNCH(c, k_compact, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
               c->off_b.p, c->key_b.p);
  c->off.swap(c->off_b);
  c->key.swap(c->key_b);
  c->cnt.swap(c->cnt_b);
  c->span = total;
}

}  // namespace

void op_reverse(rnndg_ctx* c, uint32_t R, int order) {
  if (R < 1) throw ParamError("add_reverse_edges: R must be >= 1");
  if (!c->has_distances) throw ParamError("add_reverse_edges: graph has no distances");
  materialize_pending(c);
  c->bulk_fresh = true;
  const uint64_t n = c->nv;
  ensure_scratch(c);
  // 1. reversals bucketed by their source (= target of the forward edge)
  zero(c, c->bcnt.p, n + 1);
  zero(c, c->bcur.p, n);
  RNNDG_LAUNCH(c, k_count_targets, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
               c->bcnt.p);
  scan_u64(c, c->bcnt.p, c->boff.p, n);
  const uint64_t m = read_u64(c, c->boff.p + n);
  c->bkey.ensure(m ? m : 1);
  c->bkey_s.ensure(m ? m : 1);
  c->bflag.ensure(m ? m : 1);
  c->brank.ensure(m ? m : 1);
  RNNDG_LAUNCH(c, k_scatter_targets, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p,
               c->key.p, c->boff.p, c->bcur.p, c->bkey.p, nullptr, 0);
  sort_buckets(c, m);
  // 2. append-if-absent (no duplicates among reversals: edges are unique)
  RNNDG_LAUNCH(c, k_apply_count, warp_grid(c, n), kBlock, 0, n, c->off.p, c->key.p, c->cnt.p,
               c->boff.p, c->bkey_s.p, c->bflag.p, c->brank.p, c->cnt_b.p, c->counters.p, 0,
               int(!c->exact_dists));
  merge_and_swap(c, c->cnt.p);
  ensure_scratch(c);  // span grew
  // 3. degree caps (builder.cpp:244-250)
  if (order == RNNDG_OUT_THEN_IN) {
    out_prune(c, R);
    in_prune(c, R);
  } else {
    in_prune(c, R);
    out_prune(c, R);
  }
}

namespace {
// exact distances of the pending entries of the lists marked in mat_b /
// mat_e, then those lists re-sorted in place
void resolve_pending(rnndg_ctx* c, const unsigned long long* count) {
  const uint64_t n = c->nv;
  const ScanConfig cfg = scan_config(c);
  RNNDG_LAUNCH(c, k_resolve_pending, unsigned(sm_count(c)) * 8u, kBlock, 0, n, c->v0, c->mat_b.p,
               c->mat_e.p, count, c->key.p, Row{c->xp.p, cfg.stride, cfg.nblk, cfg.ntail});
  seg_sort_keys(c, c->key.p, c->key.p, c->span, n, c->mat_b.p, c->mat_e.p, count);
}

// the hub lists queued by k_mark_active (few, long, short pending tails)
void resolve_pending_hubs(rnndg_ctx* c, const unsigned long long* count) {
  const uint64_t n = c->nv;
  const ScanConfig cfg = scan_config(c);
  c->key_s.ensure(c->span ? c->span : 1);
  RNNDG_LAUNCH(c, k_resolve_merge, unsigned(sm_count(c)) * 4u, kMergeThreads, 0, n, c->v0,
               c->mat_b.p, c->mat_e.p, count, c->key.p, c->key_s.p,
               Row{c->xp.p, cfg.stride, cfg.nblk, cfg.ntail});
  // tails too long for the merge (flagged): quad resolve + segmented sort
  RNNDG_LAUNCH(c, k_flagged_only, grid_for(n, kBlock), kBlock, 0, n, c->mat_b.p, c->mat_e.p,
               count);
  resolve_pending(c, count);
}
}  // namespace

void materialize_pending(rnndg_ctx* c) {
  if (!c->pending || !c->has_graph) return;
  const uint64_t n = c->nv;
  if (n) {
    prepare_chain_layout(c);
    unsigned long long* count = c->counters.p + kMatCount;
    zero(c, count, 1);
    RNNDG_LAUNCH(c, k_mark_pending, grid_for(n, kBlock), kBlock, 0, n, c->off.p, c->cnt.p,
                 c->key.p, c->mat_b.ensure(n), c->mat_e.ensure(2 * n), count);
    resolve_pending(c, count);
  }
  c->pending = false;
}

void op_sort_lists(rnndg_ctx* c) {
  materialize_pending(c);
  const uint64_t n = c->nv;
  ensure_scratch(c);
  RNNDG_LAUNCH(c, k_seg_end, grid_for(n, 256), 256, 0, n, c->off.p, c->cnt.p, nullptr, 0u,
               c->seg_end.p);
  seg_sort_keys(c, c->key.p, c->key_s.p, c->span, n, c->off.p, c->seg_end.p);
  c->key.swap(c->key_s);
}

// ------------------------------------------------------- sharding ops
void op_set_partition(rnndg_ctx* c, uint64_t v_begin, uint64_t v_end) {
  if (v_begin > v_end || v_end > c->n) throw ParamError("set_partition: bad vertex range");
  c->v0 = v_begin;
  c->nv = v_end - v_begin;
  c->partitioned = true;
  c->has_graph = false;
  c->pending = false;
}

uint64_t records_staged(rnndg_ctx* c) {
  unsigned long long h = 0;
  RNNDG_CUDA(cudaMemcpyAsync(&h, c->rec_cursor.p, 8, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  c->rec_n = h;
  return h;
}

void ensure_records(rnndg_ctx* c, uint64_t cap) {
  c->rec_dst.ensure(cap ? cap : 1);
  c->rec_key.ensure(cap ? cap : 1);
  c->rec_dst2.ensure(cap ? cap : 1);
  c->rec_key2.ensure(cap ? cap : 1);
  c->rec_cursor.ensure(1);
  zero(c, c->rec_cursor.p, 1);
}

// one pass's scan on the owned lists; redirects staged as records
uint64_t op_shard_scan(rnndg_ctx* c, rnndg_counts* partial) {
  op_scan_phase(c);
  ensure_records(c, c->span);
  if (c->span)
    RNNDG_LAUNCH(c, k_pend_records, grid_for(c->span, 256, 148 * 64), 256, 0, c->span,
                 c->pend_src.p, c->pend_key.p, c->rec_cursor.p, c->rec_dst.p, c->rec_key.p);
  // counters of the scan phase (removed, flag_skips, pair_checks)
  op_read_counters(c, partial, &c->shard_scan_s, nullptr, nullptr, &c->shard_touched,
                   &c->shard_active);
  ++c->shard_passes;
  return records_staged(c);
}

// stage reverse proposals (kind 1) or in-edges (kind 2) of the owned lists
uint64_t op_shard_stage(rnndg_ctx* c, int kind) {
  materialize_pending(c);
  // one record per entry: the span (list capacities) bounds their number, so
  // no count has to come back to the host to size the buffers
  ensure_records(c, c->span);
  if (c->nv)
    RNNDG_LAUNCH(c, k_edge_records, warp_grid(c, c->nv), kBlock, 0, c->nv, c->v0, c->off.p,
                 c->cnt.p, c->key.p, c->rec_cursor.p, c->rec_dst.p, c->rec_key.p,
                 kind == RNNDG_X_PROPOSAL ? 0 : 1);
  return records_staged(c);
}

// staged records sorted by destination into caller device buffers, with the
// count per destination part ([bounds[p], bounds[p+1]) ids)
void op_shard_export(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint32_t* dst_dev,
                     uint64_t* key_dev, uint64_t* counts) {
  const uint64_t nr = c->rec_n;
  if (nr) {
    if (nr > uint64_t(INT32_MAX)) throw CudaError("export: too many records");
    size_t bytes = 0;
    RNNDG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, c->rec_dst.p, c->rec_dst2.p,
                                               c->rec_key.p, c->rec_key2.p, int(nr), 0, 32,
                                               c->stream));
    RNNDG_CUDA(cub::DeviceRadixSort::SortPairs(cub_temp(c, bytes), bytes, c->rec_dst.p,
                                               c->rec_dst2.p, c->rec_key.p, c->rec_key2.p, int(nr),
                                               0, 32, c->stream));
    c->launches += 4;
    RNNDG_CUDA(cudaMemcpyAsync(dst_dev, c->rec_dst2.p, nr * 4, cudaMemcpyDeviceToDevice, c->stream));
    RNNDG_CUDA(cudaMemcpyAsync(key_dev, c->rec_key2.p, nr * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  c->part_bounds.ensure(parts + 1);
  c->part_counts.ensure(parts);
  RNNDG_CUDA(cudaMemcpyAsync(c->part_bounds.p, bounds, (parts + 1) * 8, cudaMemcpyHostToDevice,
                             c->stream));
  RNNDG_LAUNCH(c, k_part_counts, (parts + 127) / 128, 128, 0, nr, c->rec_dst2.p,
               c->part_bounds.p, parts, c->part_counts.p);
  RNNDG_CUDA(cudaMemcpyAsync(counts, c->part_counts.p, parts * 8, cudaMemcpyDeviceToHost,
                             c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
}

// Direct routing (the fused exchange of SURVEY 8(e)): instead of sorting the
// staged records by destination and handing them to a transport, count them
// per owner (op_shard_route), and -- once the caller has laid out every
// owner's receive buffer from all shards' counts -- store each record
// straight into its owner's buffer from the kernel (op_shard_push; the
// buffers are peer-mapped when the owner is another GPU, so the stores travel
// over NVLink).  No sort, no staging copy, no collective.
namespace {
PushArgs push_args(const uint64_t* bounds, uint32_t parts) {
  if (parts == 0 || parts > kMaxParts) throw ParamError("shard routing: 1 .. 64 parts");
  PushArgs a{};
  a.parts = parts;
  for (uint32_t p = 0; p <= parts; ++p) a.bounds[p] = bounds[p];
  return a;
}
}  // namespace

void op_shard_route(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint64_t* counts) {
  const uint64_t nr = c->rec_n;
  PushArgs a = push_args(bounds, parts);
  c->part_counts.ensure(2 * kMaxParts);
  zero(c, c->part_counts.p, 2 * kMaxParts);
  if (nr)
    RNNDG_LAUNCH(c, k_route_counts, grid_for(nr, 256, unsigned(sm_count(c)) * 8u), 256, 0, nr,
                 c->rec_dst.p, a, c->part_counts.p);
  static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "");
  RNNDG_CUDA(cudaMemcpyAsync(counts, c->part_counts.p, parts * 8, cudaMemcpyDeviceToHost,
                             c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
}

void op_shard_push(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint32_t* const* dst_ptrs,
                   uint64_t* const* key_ptrs, const uint64_t* offsets) {
  const uint64_t nr = c->rec_n;
  if (nr) {
    PushArgs a = push_args(bounds, parts);
    for (uint32_t p = 0; p < parts; ++p) {
      a.dst[p] = dst_ptrs[p];
      a.key[p] = key_ptrs[p];
      a.at[p] = offsets[p];
    }
    c->part_counts.ensure(2 * kMaxParts);
    unsigned long long* cursor = c->part_counts.p + kMaxParts;
    zero(c, cursor, kMaxParts);
    RNNDG_LAUNCH(c, k_route_push, grid_for(nr, 256, unsigned(sm_count(c)) * 8u), 256, 0, nr,
                 c->rec_dst.p, c->rec_key.p, a, cursor);
  }
  // the owners read the records next, on their own streams
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  c->rec_n = 0;
}

// received records -> owned lists.  kind: redirects (append-if-absent,
// counted as inserted), reverse proposals (append-if-absent), in-edges
// (select deletions, staged for export), deletions (apply).
uint64_t op_shard_import(rnndg_ctx* c, int kind, const uint32_t* dst_dev, const uint64_t* key_dev,
                         uint64_t nr, uint32_t R, rnndg_counts* partial) {
  const uint64_t n = c->nv;
  ensure_scratch(c);
  // only an INEDGE import stages records; nothing is left to export after
  // the others (rnndg_shard_export then reports zero records)
  if (kind != RNNDG_X_INEDGE) c->rec_n = 0;
  if (kind == RNNDG_X_DELETE) {
    if (nr) {
      c->rec_key2.ensure(nr);
      RNNDG_LAUNCH(c, k_rec_locate, grid_for(nr, 256, 148 * 64), 256, 0, nr, c->v0, dst_dev,
                   key_dev, c->off.p, c->cnt.p, c->key.p, c->rec_key2.p);
      RNNDG_LAUNCH(c, k_tomb_slots, grid_for(nr, 256, 148 * 64), 256, 0, nr, c->rec_key2.p,
                   c->key.p);
    }
    RNNDG_LAUNCH(c, k_count_live, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
                 c->cnt_b.p);
    c->off_b.ensure(n + 1);
    scan_u32(c, c->cnt_b.p, c->off_b.p, n);
    const uint64_t total = read_u64(c, c->off_b.p + n);
    c->key_b.ensure(total ? total : 1);
    RNNDG_LAUNCH(c, k_compact, warp_grid(c, n), kBlock, 0, n, c->off.p, c->cnt.p, c->key.p,
                 c->off_b.p, c->key_b.p);
    c->off.swap(c->off_b);
    c->key.swap(c->key_b);
    c->cnt.swap(c->cnt_b);
    c->span = total;
    return 0;
  }
  // bucket by owned destination
  zero(c, c->bcnt.p, n + 1);
  zero(c, c->bcur.p, n);
  c->bkey.ensure(nr ? nr : 1);
  c->bkey_s.ensure(nr ? nr : 1);
  c->bflag.ensure(nr ? nr : 1);
  c->brank.ensure(nr ? nr : 1);
  if (nr)
    RNNDG_LAUNCH(c, k_rec_count, grid_for(nr, 256, 148 * 64), 256, 0, nr, c->v0, dst_dev, c->bcnt.p);
  scan_u64(c, c->bcnt.p, c->boff.p, n);
  if (nr)
    RNNDG_LAUNCH(c, k_rec_scatter, grid_for(nr, 256, 148 * 64), 256, 0, nr, c->v0, dst_dev,
                 key_dev, c->boff.p, c->bcur.p, c->bkey.p);
  sort_buckets(c, nr);
  if (kind == RNNDG_X_INEDGE) {
    ensure_records(c, nr);
    RNNDG_LAUNCH(c, k_inedge_select, warp_grid(c, n), kBlock, 0, n, c->v0, c->boff.p,
                 c->bkey_s.p, R, c->rec_cursor.p, c->rec_dst.p, c->rec_key.p);
    return records_staged(c);
  }
  // redirects / proposals: append-if-absent into the (post-scan) lists
  unsigned long long* ctr = c->counters.p;
  zero(c, ctr, kNumCounters);
  const uint32_t* post = kind == RNNDG_X_PENDING ? c->post_cnt.p : c->cnt.p;
  RNNDG_LAUNCH(c, k_apply_count, warp_grid(c, n), kBlock, 0, n, c->off.p, c->key.p, post,
               c->boff.p, c->bkey_s.p, c->bflag.p, c->brank.p, c->cnt_b.p, ctr,
               kind == RNNDG_X_PENDING ? 1 : 0,
               int((kind == RNNDG_X_PENDING && gram_cap()) || !c->exact_dists));
  merge_and_swap(c, post);
  if (kind == RNNDG_X_PENDING && gram_cap()) c->pending = true;
  if (partial) {
    unsigned long long h[kNumCounters];
    RNNDG_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
    *partial = rnndg_counts{0, h[kInserted], 0, 0};
  }
  return 0;
}

void op_shard_out_prune(rnndg_ctx* c, uint32_t R) {
  if (c->nv) RNNDG_LAUNCH(c, k_out_trunc, grid_for(c->nv, 256), 256, 0, c->nv, c->cnt.p, R);
}

// ------------------------------------------------------ NN-Descent baseline
// nndescent.cpp, in the canonical deferred form the oracle restates
// (oracle/rnnd_oracle.c ro_nnd_pass): per pass, snapshot every pool, join
// every pair of the snapshot lists (launch_nnd_join), then make each pool the
// `cap` nearest distinct entries of (pool + proposals) -- a segmented sort of
// the union per vertex, deduplicated by id (an id has one key per pool: l2
// is bit-symmetric) and truncated.  Proposals are produced and applied in
// vertex chunks to bound memory; applying the union chunk by chunk gives the
// same pools as applying it at once.
namespace {

constexpr uint64_t kNndChunkPairs = uint64_t(24) << 20;  // pairs per join chunk

// random_init lists (stride S, sorted) -> pools (stride cap)
__global__ void __launch_bounds__(kBlock)
    k_nd_from_lists(uint64_t n, uint32_t cap, const uint64_t* __restrict__ off,
                    const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ key,
                    uint64_t* __restrict__ pool, uint32_t* __restrict__ pcnt) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint32_t U = cnt[u];
    for (uint32_t j = lane; j < U; j += 32) pool[u * cap + j] = key[off[u] + j];
    if (lane == 0) pcnt[u] = U;
  }
}

// nndescent.cpp:60-70: the nearest `sample` fresh entries join as fresh and
// turn old; entries old before the pass join as old.  Keeps a copy of the
// pool (the new-entry count) and the pair count of the vertex.
__global__ void k_nd_snapshot(uint64_t n, uint32_t cap, uint32_t sample,
                              uint64_t* __restrict__ pool, const uint32_t* __restrict__ pcnt,
                              uint32_t* __restrict__ F, uint32_t* __restrict__ fcnt,
                              uint32_t* __restrict__ O, uint32_t* __restrict__ ocnt,
                              uint64_t* __restrict__ pool0, uint32_t* __restrict__ pcnt0,
                              uint32_t* __restrict__ npairs) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n; u += stride) {
    uint64_t* P = pool + u * cap;
    const uint32_t m = pcnt[u];
    uint32_t fc = 0, oc = 0;
    for (uint32_t j = 0; j < m; ++j) {
      const uint64_t k = P[j];
      if (key_fresh(k) && fc < sample) {
        F[u * sample + fc++] = key_id(k);
        P[j] = k & ~1ull;
      } else if (!key_fresh(k)) {
        O[u * cap + oc++] = key_id(k);
      }
      pool0[u * cap + j] = k;
    }
    fcnt[u] = fc;
    ocnt[u] = oc;
    pcnt0[u] = m;
    npairs[u] = fc * (fc ? fc - 1 : 0) / 2 + fc * oc;
  }
}

__global__ void k_nd_count_dst(uint64_t m, const uint32_t* __restrict__ dst,
                               unsigned long long* __restrict__ cnt) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride)
    atomicAdd(&cnt[dst[i]], 1ull);
}

// segment v = pool v (first) + its proposals; lengths into len (n + 1 slots)
__global__ void k_nd_seg_len(uint64_t n, const uint32_t* __restrict__ pcnt,
                             const unsigned long long* __restrict__ bcnt,
                             unsigned long long* __restrict__ len) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    len[v] = pcnt[v] + bcnt[v];
}

__global__ void __launch_bounds__(kBlock)
    k_nd_seg_fill(uint64_t n, uint32_t cap, const uint64_t* __restrict__ pool,
                  const uint32_t* __restrict__ pcnt, const uint64_t* __restrict__ boff,
                  uint64_t* __restrict__ seg, unsigned long long* __restrict__ cur) {
  const uint32_t lane = lane_id();
  WARP_LOOP(v, n) {
    const uint32_t m = pcnt[v];
    for (uint32_t j = lane; j < m; j += 32) seg[boff[v] + j] = pool[v * cap + j];
    if (lane == 0) cur[v] = m;
  }
}

__global__ void k_nd_scatter(uint64_t m, const uint32_t* __restrict__ dst,
                             const uint64_t* __restrict__ key, const uint64_t* __restrict__ boff,
                             unsigned long long* __restrict__ cur, uint64_t* __restrict__ seg) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint32_t v = dst[i];
    seg[boff[v] + atomicAdd(&cur[v], 1ull)] = key[i];
  }
}

// sorted union -> pool: drop repeated ids (the existing entry's even key
// sorts before a proposal's odd one), keep the first cap (insert_candidate,
// nndescent.cpp:39-49)
__global__ void __launch_bounds__(kBlock)
    k_nd_merge(uint64_t n, uint32_t cap_ref, uint32_t stride, const uint64_t* __restrict__ boff,
               const uint64_t* __restrict__ seg, const uint32_t* __restrict__ pcnt0,
               uint64_t* __restrict__ pool, uint32_t* __restrict__ pcnt) {
  const uint32_t lane = lane_id();
  WARP_LOOP(v, n) {
    const uint64_t* S = seg + boff[v];
    const uint32_t len = uint32_t(boff[v + 1] - boff[v]);
    uint64_t* P = pool + v * stride;
    // a pool above the cap (init fills min(sample, n-1)) keeps its size:
    // insert_candidate pops one entry per insertion (nndescent.cpp:46-47)
    const uint32_t cap = pcnt0[v] > cap_ref ? pcnt0[v] : cap_ref;
    uint32_t w = 0;
    uint64_t prev = ~0ull;  // previous element's key (id compare via >> 1)
    for (uint32_t j0 = 0; j0 < len && w < cap; j0 += 32) {
      const uint32_t j = j0 + lane;
      const uint64_t k = j < len ? S[j] : ~0ull;
      uint64_t before = __shfl_up_sync(0xffffffffu, k, 1);
      if (lane == 0) before = prev;
      const bool keep = j < len && (k >> 1) != (before >> 1);
      const unsigned mk = __ballot_sync(0xffffffffu, keep);
      const uint32_t r = w + __popc(mk & ((1u << lane) - 1u));
      if (keep && r < cap) P[r] = k;
      w += __popc(mk);
      prev = __shfl_sync(0xffffffffu, k, 31);
    }
    if (lane == 0) pcnt[v] = w < cap ? w : cap;
  }
}

// entries of the new pool whose id was not in the pool before the pass
__global__ void __launch_bounds__(kBlock)
    k_nd_count_new(uint64_t n, uint32_t cap, const uint64_t* __restrict__ pool,
                   const uint32_t* __restrict__ pcnt, const uint64_t* __restrict__ pool0,
                   const uint32_t* __restrict__ pcnt0, unsigned long long* __restrict__ ctr) {
  const uint32_t lane = lane_id();
  unsigned long long fresh = 0;
  WARP_LOOP(v, n) {
    const uint64_t* P0 = pool0 + v * cap;
    const uint32_t m0 = pcnt0[v];
    for (uint32_t j = lane; j < pcnt[v]; j += 32) {
      const uint64_t k = pool[v * cap + j] & ~1ull;
      const uint32_t at = lower_bound(P0, m0, k);
      if (!(at < m0 && (P0[at] >> 1) == (k >> 1))) ++fresh;
    }
  }
  warp_add_counter(ctr, fresh);
}

// nndescent.cpp:88-99: the K nearest pool entries, flagged old, as the graph
__global__ void __launch_bounds__(kBlock)
    k_nd_finalize(uint64_t n, uint32_t cap, uint32_t K, const uint64_t* __restrict__ pool,
                  const uint32_t* __restrict__ pcnt, uint64_t* __restrict__ off,
                  uint32_t* __restrict__ cnt, uint64_t* __restrict__ key) {
  const uint32_t lane = lane_id();
  WARP_LOOP(u, n) {
    const uint32_t t = pcnt[u] < K ? pcnt[u] : K;
    for (uint32_t j = lane; j < t; j += 32) key[u * K + j] = pool[u * cap + j] & ~1ull;
    if (lane == 0) {
      off[u] = u * K;
      cnt[u] = t;
      if (u + 1 == n) off[n] = n * K;
    }
  }
}

}  // namespace

void op_nnd_init(rnndg_ctx* c, uint32_t K, uint32_t sample, uint32_t iters, uint32_t pool,
                 uint64_t seed) {
  const uint64_t n = c->n;
  if (c->partitioned) throw ParamError("nndescent: not available on a partitioned context");
  // NnDescent::NnDescent, nndescent.cpp:11-22
  if (n < 2) throw ParamError("nndescent: need at least 2 vectors");
  if (K < 1 || K > n - 1) throw ParamError("nndescent: K out of [1, n-1]");
  if (sample < 1) throw ParamError("nndescent: sample must be >= 1");
  if (iters < 1) throw ParamError("nndescent: iters must be >= 1");
  const uint32_t cap = std::max(pool ? pool : 2 * K, K);
  c->nd_K = K;
  c->nd_cap = cap;
  c->nd_sample = sample;
  c->nd_iters = iters;
  // init, :24-37: the random_init sampler with s = min(sample, n - 1) ids
  const uint32_t s = uint32_t(std::min<uint64_t>(sample, n - 1));
  c->nd_stride = std::max(cap, s);  // pools may start above the cap
  op_random_init(c, s, seed);
  c->nd_pool.ensure(n * c->nd_stride);
  c->nd_pcnt.ensure(n);
  RNNDG_LAUNCH(c, k_nd_from_lists, warp_grid(c, n), kBlock, 0, n, c->nd_stride, c->off.p,
               c->cnt.p, c->key.p, c->nd_pool.p, c->nd_pcnt.p);
  c->nd_ready = true;
}

uint64_t op_nnd_pass(rnndg_ctx* c) {
  if (!c->nd_ready) throw ParamError("nndescent: call init first");
  const uint64_t n = c->n;
  const uint32_t cap = c->nd_stride, sample = c->nd_sample;  // cap: the pool stride here
  c->nd_pool0.ensure(n * cap);
  c->nd_pcnt0.ensure(n);
  c->nd_F.ensure(n * sample);
  c->nd_fcnt.ensure(n);
  c->nd_O.ensure(n * cap);
  c->nd_ocnt.ensure(n);
  c->nd_np.ensure(n + 1);
  c->nd_poff.ensure(n + 1);
  RNNDG_LAUNCH(c, k_nd_snapshot, grid_for(n, 128), 128, 0, n, cap, sample, c->nd_pool.p,
               c->nd_pcnt.p, c->nd_F.p, c->nd_fcnt.p, c->nd_O.p, c->nd_ocnt.p, c->nd_pool0.p,
               c->nd_pcnt0.p, c->nd_np.p);
  scan_u32(c, c->nd_np.p, c->nd_poff.p, n);
  std::vector<uint64_t> poff(n + 1);
  RNNDG_CUDA(cudaMemcpyAsync(poff.data(), c->nd_poff.p, (n + 1) * 8, cudaMemcpyDeviceToHost,
                             c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  c->nd_bcnt.ensure(n + 1);
  c->nd_cur.ensure(n);
  c->nd_boff.ensure(n + 1);
  // pairs per join chunk (RNNDG_NND_CHUNK overrides, e.g. to test chunking)
  static const uint64_t chunk_pairs = [] {
    const char* e = std::getenv("RNNDG_NND_CHUNK");
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 ? uint64_t(v) : kNndChunkPairs;
  }();
  for (uint64_t u0 = 0; u0 < n;) {
    // the largest vertex range whose pairs fit one chunk (at least one vertex)
    uint64_t u1 = u0 + 1;
    {
      uint64_t lo = u0 + 1, hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi + 1) / 2;
        if (poff[mid] - poff[u0] <= chunk_pairs)
          lo = mid;
        else
          hi = mid - 1;
      }
      u1 = lo;
    }
    const uint64_t npairs = poff[u1] - poff[u0];
    if (npairs) {
      const uint64_t m = 2 * npairs;
      c->nd_pdst.ensure(m);
      c->nd_pkey.ensure(m);
      launch_nnd_join(c, u0, u1, npairs);
      zero(c, c->nd_bcnt.p, n + 1);
      RNNDG_LAUNCH(c, k_nd_count_dst, grid_for(m, 256, 148 * 64), 256, 0, m, c->nd_pdst.p,
                   c->nd_bcnt.p);
      RNNDG_LAUNCH(c, k_nd_seg_len, grid_for(n, 256, 148 * 64), 256, 0, n, c->nd_pcnt.p,
                   c->nd_bcnt.p, c->nd_bcnt.p);
      scan_u64(c, c->nd_bcnt.p, c->nd_boff.p, n);
      const uint64_t total = read_u64(c, c->nd_boff.p + n);
      c->nd_seg.ensure(total);
      c->nd_seg_s.ensure(total);
      RNNDG_LAUNCH(c, k_nd_seg_fill, warp_grid(c, n), kBlock, 0, n, cap, c->nd_pool.p,
                   c->nd_pcnt.p, c->nd_boff.p, c->nd_seg.p, c->nd_cur.p);
      RNNDG_LAUNCH(c, k_nd_scatter, grid_for(m, 256, 148 * 64), 256, 0, m, c->nd_pdst.p,
                   c->nd_pkey.p, c->nd_boff.p, c->nd_cur.p, c->nd_seg.p);
      seg_sort_keys(c, c->nd_seg.p, c->nd_seg_s.p, total, n, c->nd_boff.p, c->nd_boff.p + 1);
      RNNDG_LAUNCH(c, k_nd_merge, warp_grid(c, n), kBlock, 0, n, c->nd_cap, cap, c->nd_boff.p,
                   c->nd_seg_s.p, c->nd_pcnt0.p, c->nd_pool.p, c->nd_pcnt.p);
    }
    u0 = u1;
  }
  unsigned long long* ctr = c->counters.p;
  c->counters.ensure(kNumCounters);
  ctr = c->counters.p;
  zero(c, ctr, 1);
  RNNDG_LAUNCH(c, k_nd_count_new, warp_grid(c, n), kBlock, 0, n, cap, c->nd_pool.p,
               c->nd_pcnt.p, c->nd_pool0.p, c->nd_pcnt0.p, ctr);
  unsigned long long h = 0;
  RNNDG_CUDA(cudaMemcpyAsync(&h, ctr, 8, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  return h;
}

void op_nnd_finalize(rnndg_ctx* c) {
  if (!c->nd_ready) throw ParamError("nndescent: call init first");
  const uint64_t n = c->n;
  const uint32_t K = c->nd_K;
  c->off.ensure(n + 1);
  c->cnt.ensure(n + 1);
  c->key.ensure(n * K);
  c->span = n * K;
  RNNDG_LAUNCH(c, k_nd_finalize, warp_grid(c, n), kBlock, 0, n, c->nd_stride, K, c->nd_pool.p,
               c->nd_pcnt.p, c->off.p, c->cnt.p, c->key.p);
  c->has_graph = true;
  c->pending = false;
  c->has_distances = true;
  c->exact_dists = true;
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
}

#undef WARP_LOOP

}  // namespace rnndg
