// eval.cu -- the evaluator half of the hot path on sm_100a: beam search
// (search.cpp:40-132), exact brute-force ground truth (dataset.cpp:175-205),
// batched exact L2 (metric.hpp:47-65), rng_strategy (builder.cpp:196-212) and
// degree statistics (graph.cpp:76-100).
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_segmented_sort.cuh>

#include "common.cuh"
#include "ctx.hpp"

namespace rnndg {

namespace {

// ----------------------------------------------------------------- search
//
// One warp per query.  The pool holds up to L (dist, id) keys ascending plus
// an `expanded` byte per slot.  The seen set (search.cpp:46) is an
// open-addressing hash table of ids sized from L and the degree cap, in
// global memory per block (L2-resident, cleared per query: O(L * degree),
// not O(n));
// a query that fills it past 3/4 stops and is re-run with a per-block n-bit
// map (kTab = false), so the result never depends on the table size.  The
// pool after any batch of consider() calls is top-L(pool ∪ new) under
// (dist, id) (search.cpp:49-59), so a batch of up to 32 neighbours is
// evaluated in parallel (one lane per neighbour, exact L2) and inserted one
// by one with a warp-parallel position search.  Entry ids come from
// sample_distinct(SplitMix64(seed), n, count) (search.cpp:64-68), computed
// once per call by k_sample_entries.
struct SearchArgs {
  const float* x;
  uint32_t d;
  uint64_t n;
  const uint64_t* off;
  const uint32_t* cnt;
  const uint64_t* key;
  const float* queries;
  uint64_t nq;
  uint32_t L, K, k;
  int fixed;
  uint32_t entry_vertex;
  const uint32_t* entries;
  uint32_t nentries;
  uint32_t* seen;       // bitmap mode: per block words_per_map words
  uint64_t words_per_map;
  uint32_t tab_log2;    // hash mode: open-addressing table of 2^tab_log2 ids
  uint32_t* gtab;       //   per block in global memory (null: in shared memory)
  uint64_t* gpool;      // per block L keys when the pool does not fit smem
  uint8_t* gexp;        // per block L flags
  uint32_t* out_ids;
  float* out_dists;
  unsigned long long* out_visited;
  unsigned long long* out_comps;
};

constexpr uint32_t kTabEmpty = 0xFFFFFFFFu;

// insert id into the seen set; true when it was not there yet
template <bool kTab>
__device__ __forceinline__ bool seen_insert(uint32_t* seen, uint32_t tab_log2, uint32_t id) {
  if (!kTab) {
    const uint32_t bit = 1u << (id & 31u);
    return !(atomicOr(&seen[id >> 5], bit) & bit);
  }
  const uint32_t mask = (1u << tab_log2) - 1u;
  uint32_t h = (id * 2654435761u) >> (32u - tab_log2);
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    const uint32_t prev = atomicCAS(&seen[h], kTabEmpty, id);
    if (prev == kTabEmpty) return true;
    if (prev == id) return false;
    h = (h + 1u) & mask;
  }
  // table full: the query overflows (comps passes 3/4 of the table) and is
  // re-run with the bitmap, so this answer is never used
  return true;
}

template <bool kVec4, bool kTab>
__device__ void consider_batch(const float* __restrict__ x, uint32_t d, uint32_t L,
                               const float* q,
                               const uint32_t* cand, uint32_t m, uint32_t* seen,
                               uint32_t tab_log2, uint64_t* pool, uint8_t* expd,
                               uint32_t& psize, unsigned long long& comps) {
  const uint32_t lane = lane_id();
  for (uint32_t c0 = 0; c0 < m; c0 += 32) {
    const uint32_t c = c0 + lane;
    bool fresh = false;
    uint64_t ck = 0;
    if (c < m) {
      const uint32_t id = cand[c];
      if (seen_insert<kTab>(seen, tab_log2, id)) {
        fresh = true;
        const float dist = l2_exact<kVec4>(q, x + uint64_t(id) * d, d);
        ck = (uint64_t(__float_as_uint(dist)) << 32) | id;
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, fresh);
    comps += __popc(mask);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint64_t key = __shfl_sync(0xffffffffu, ck, src);
      if (psize == L && !(key < pool[psize - 1])) continue;  // rejected
      // upper_bound position: number of pool keys <= key (keys are unique)
      uint32_t pos = 0;
      for (uint32_t p0 = 0; p0 < psize; p0 += 32) {
        const uint32_t p = p0 + lane;
        pos += __popc(__ballot_sync(0xffffffffu, p < psize && pool[p] < key));
      }
      const uint32_t last = psize < L ? psize : L - 1;  // new last index
      // shift [pos, last) right by one, from the top down in warp-wide steps
      for (int32_t hi = int32_t(last) - 1; hi >= int32_t(pos); hi -= 32) {
        const int32_t p = hi - int32_t(lane);
        uint64_t pk = 0;
        uint8_t pe = 0;
        const bool mv = p >= int32_t(pos);
        if (mv) {
          pk = pool[p];
          pe = expd[p];
        }
        __syncwarp();
        if (mv) {
          pool[p + 1] = pk;
          expd[p + 1] = pe;
        }
        __syncwarp();
      }
      if (lane == 0) {
        pool[pos] = key;
        expd[pos] = 0;
      }
      __syncwarp();
      if (psize < L) ++psize;
    }
  }
}

// kTab: hash-table seen set (queries[qi] for qi in `only` when given: the
// bitmap re-run of the queries that overflowed their table)
template <bool kVec4, bool kTab>
__global__ void k_search(SearchArgs a, const uint32_t* only, uint32_t nonly) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t lane = lane_id();
  float* q = reinterpret_cast<float*>(smem);
  const size_t qbytes = (size_t(a.d) * 4 + 15) & ~size_t(15);
  uint64_t* pool;
  uint8_t* expd;
  size_t used = qbytes;
  if (a.gpool) {
    pool = a.gpool + uint64_t(blockIdx.x) * a.L;
    expd = a.gexp + uint64_t(blockIdx.x) * a.L;
  } else {
    pool = reinterpret_cast<uint64_t*>(smem + qbytes);
    expd = reinterpret_cast<uint8_t*>(pool + a.L);
    used += (size_t(a.L) * 9 + 15) & ~size_t(15);
  }
  const uint64_t seen_words = kTab ? (uint64_t(1) << a.tab_log2) : a.words_per_map;
  uint32_t* seen = kTab ? (a.gtab ? a.gtab + uint64_t(blockIdx.x) * seen_words
                                  : reinterpret_cast<uint32_t*>(smem + used))
                        : a.seen + uint64_t(blockIdx.x) * a.words_per_map;
  const uint64_t nrun = only ? nonly : a.nq;
  for (uint64_t qr = blockIdx.x; qr < nrun; qr += gridDim.x) {
    const uint64_t qi = only ? only[qr] : qr;
    for (uint64_t w = lane; w < seen_words; w += 32) seen[w] = kTab ? kTabEmpty : 0u;
    for (uint32_t j = lane; j < a.d; j += 32) q[j] = a.queries[qi * a.d + j];
    __syncwarp();
    uint32_t psize = 0;
    unsigned long long comps = 0, visited = 0;
    __shared__ uint32_t entry_buf[1];
    if (lane == 0) entry_buf[0] = a.entry_vertex;
    __syncwarp();
    if (a.fixed)
      consider_batch<kVec4, kTab>(a.x, a.d, a.L, q, entry_buf, 1, seen, a.tab_log2, pool, expd,
                                  psize, comps);
    else
      consider_batch<kVec4, kTab>(a.x, a.d, a.L, q, a.entries, a.nentries, seen, a.tab_log2, pool,
                                  expd, psize, comps);
    bool overflow = false;
    for (;;) {
      // every considered id is in the seen set: past 3/4 of the table the
      // query is abandoned and re-run with the bitmap
      if (kTab && comps > (3ull << a.tab_log2) / 4) {
        overflow = true;
        break;
      }
      uint32_t at = psize;
      for (uint32_t p0 = 0; p0 < psize; p0 += 32) {
        const uint32_t p = p0 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, p < psize && !expd[p]);
        if (m) {
          at = p0 + __ffs(m) - 1;
          break;
        }
      }
      if (at == psize) break;
      __syncwarp();
      if (lane == 0) expd[at] = 1;
      ++visited;
      const uint32_t v = uint32_t(pool[at]);
      const uint32_t deg = a.cnt[v];
      // select_nearest (graph.cpp:65-74): lists are kept nearest-first when
      // the graph has distances, and in stored order otherwise, so the K
      // nearest are the first min(K, deg) entries.
      const uint32_t take = (a.K == 0 || deg <= a.K) ? deg : a.K;
      const uint64_t* lst = a.key + a.off[v];
      // ids of this expansion, 32 at a time through shared scratch in regs
      for (uint32_t j0 = 0; j0 < take; j0 += 32) {
        const uint32_t j = j0 + lane;
        uint32_t id = j < take ? key_id(lst[j]) : 0u;
        // stage through a register shuffle: each lane consumes its own id
        __shared__ uint32_t ids_buf[32];
        __syncwarp();
        ids_buf[lane] = id;
        __syncwarp();
        const uint32_t m = take - j0 < 32 ? take - j0 : 32;
        consider_batch<kVec4, kTab>(a.x, a.d, a.L, q, ids_buf, m, seen, a.tab_log2, pool, expd,
                                    psize, comps);
      }
    }
    const uint32_t take = a.k < psize ? a.k : psize;
    for (uint32_t j = lane; j < a.k; j += 32) {
      const bool have = j < take;
      a.out_ids[qi * a.k + j] = have ? uint32_t(pool[j]) : kNone;
      a.out_dists[qi * a.k + j] =
          have ? __uint_as_float(uint32_t(pool[j] >> 32)) : __int_as_float(0x7f800000);
    }
    if (lane == 0) {
      a.out_visited[qi] = overflow ? ~0ull : visited;
      a.out_comps[qi] = comps;
    }
    __syncwarp();
  }
}

__global__ void k_sum_u32(const uint32_t* __restrict__ v, uint64_t n, unsigned long long* out) {
  unsigned long long m = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    m += v[i];
  for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  if (lane_id() == 0 && m) atomicAdd(out, m);
}

// sample_distinct(SplitMix64(seed), n, count) with no exclusion (rng.hpp:46-72)
__global__ void k_sample_entries(uint64_t n, uint32_t count, uint64_t seed,
                                 uint32_t* out, uint32_t* bitmap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  SplitMix64 rng(seed);
  const uint32_t domain = uint32_t(n);
  uint32_t m = 0;
  for (uint32_t j = domain - count; j < domain; ++j) {
    const uint32_t t = uint32_t(rng.bounded(uint64_t(j) + 1));
    bool hit;
    if (bitmap) {
      hit = (bitmap[t >> 5] >> (t & 31)) & 1u;
    } else {
      hit = false;
      for (uint32_t q = 0; q < m; ++q)
        if (out[q] == t) {
          hit = true;
          break;
        }
    }
    const uint32_t v = hit ? j : t;
    if (bitmap) bitmap[v >> 5] |= 1u << (v & 31);
    out[m++] = v;
  }
}

// ------------------------------------------------------------ brute force
// Exact k nearest by (dist, id) (dataset.cpp:183-203: a max-heap on
// std::pair<float, uint32_t>, i.e. ties to the lower id).  One block per
// query: each thread keeps a sorted private top-k, then k rounds of a
// block-wide minimum merge the private lists.
constexpr int kBfThreads = 256;
constexpr int kBfMaxK = 64;

template <bool kVec4>
__global__ void __launch_bounds__(kBfThreads)
    k_brute_force(const float* __restrict__ x, uint64_t n, uint32_t d,
                  const float* __restrict__ queries, uint64_t nq, uint32_t k,
                  uint32_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* q = reinterpret_cast<float*>(smem);
  __shared__ unsigned long long red[kBfThreads / 32];
  uint64_t best[kBfMaxK];
  for (uint64_t qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) q[j] = queries[qi * d + j];
    __syncthreads();
    uint32_t m = 0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const float dist = l2_exact<kVec4>(q, x + i * d, d);
      const uint64_t key = (uint64_t(__float_as_uint(dist)) << 32) | i;
      if (m == k && key >= best[k - 1]) continue;
      uint32_t at = m < k ? m : k - 1;
      while (at > 0 && best[at - 1] > key) {
        best[at] = best[at - 1];
        --at;
      }
      best[at] = key;
      if (m < k) ++m;
    }
    uint32_t head = 0;
    for (uint32_t r = 0; r < k; ++r) {
      unsigned long long mine = head < m ? best[head] : ~0ull;
      unsigned long long v = mine;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
      }
      if (lane_id() == 0) red[threadIdx.x >> 5] = v;
      __syncthreads();
      unsigned long long g = red[0];
      for (int w = 1; w < kBfThreads / 32; ++w) g = red[w] < g ? red[w] : g;
      if (mine == g && mine != ~0ull) ++head;  // keys are unique
      if (threadIdx.x == 0) out[qi * k + r] = uint32_t(g);
      __syncthreads();
    }
  }
}

// -------------------------------------------------------------- l2 pairs
template <bool kVec4>
__global__ void k_l2_pairs(const float* __restrict__ x, uint32_t d,
                           const uint32_t* __restrict__ a,
                           const uint32_t* __restrict__ b, uint64_t np,
                           float* __restrict__ out) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < np;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = l2_exact<kVec4>(x + uint64_t(a[i]) * d, x + uint64_t(b[i]) * d, d);
}

// ---------------------------------------------------------- rng_strategy
// builder.cpp:196-212 on one sorted candidate list (plain Algorithm 3: every
// pair is checked, no flags).  One warp; kept entries compacted in place.
template <bool kVec4>
__global__ void k_rng_strategy(const float* __restrict__ x, uint32_t d,
                               uint64_t* keys, uint32_t m, uint32_t* nkept) {
  const uint32_t lane = lane_id();
  uint32_t nk = 0;
  for (uint32_t i = 0; i < m; ++i) {
    const uint64_t vk = keys[i];
    const float vd = key_dist(vk);
    const float* xv = x + uint64_t(key_id(vk)) * d;
    bool keep = true;
    for (uint32_t k0 = 0; k0 < nk && keep; k0 += 32) {
      const uint32_t kk = k0 + lane;
      bool occ = false;
      if (kk < nk) occ = vd >= l2_exact<kVec4>(xv, x + uint64_t(key_id(keys[kk])) * d, d);
      keep = __ballot_sync(0xffffffffu, occ) == 0;
    }
    __syncwarp();
    if (keep) {
      if (lane == 0) keys[nk] = vk;
      ++nk;
    }
    __syncwarp();
  }
  if (lane == 0) *nkept = nk;
}

// ---------------------------------------------------------- degree stats
__global__ void k_degree(uint64_t n, const uint64_t* __restrict__ off,
                         const uint32_t* __restrict__ cnt,
                         const uint64_t* __restrict__ key, uint32_t cap,
                         unsigned int* __restrict__ indeg,
                         unsigned long long* __restrict__ out) {
  for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
       u += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t deg = cnt[u];
    const uint32_t take = (cap == 0 || deg <= cap) ? deg : cap;
    atomicAdd(&out[0], (unsigned long long)take);
    atomicMax(&out[1], (unsigned long long)take);
    for (uint32_t j = 0; j < take; ++j) atomicAdd(&indeg[key_id(key[off[u] + j])], 1u);
  }
}

__global__ void k_max_u32(uint64_t n, const unsigned int* __restrict__ v,
                          unsigned long long* __restrict__ out) {
  for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
       u += uint64_t(gridDim.x) * blockDim.x)
    atomicMax(out, (unsigned long long)v[u]);
}

template <class T>
T* upload(rnndg_ctx* c, DevBuf<T>& buf, const T* host, uint64_t count) {
  T* p = buf.ensure(count ? count : 1);
  if (count)
    RNNDG_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return p;
}

}  // namespace

void op_search(rnndg_ctx* c, const float* queries, uint64_t nq, uint32_t L,
               uint32_t K, uint32_t k, int entry_mode, uint32_t entry_vertex,
               uint32_t entry_count, uint64_t seed, uint32_t* ids, float* dists,
               uint64_t* visited, uint64_t* dist_comps) {
  materialize_pending(c);
  const uint64_t n = c->n;
  if (nq == 0) throw ParamError("batch_search: no queries");
  if (n == 0) throw ParamError("search: empty graph");
  if (L < 1) throw ParamError("search: L must be >= 1");
  if (k < 1 || k > L) throw ParamError("search: k out of [1, L]");
  if (entry_mode == RNNDG_ENTRY_FIXED && entry_vertex >= n)
    throw ParamError("search: entry vertex out of range");
  // select_nearest: lists are kept nearest-first when distances are cached
  // (sorted-list invariant, build.cu) and in stored order otherwise

  SearchArgs a{};
  a.x = c->x;
  a.d = c->d;
  a.n = n;
  a.off = c->off.p;
  a.cnt = c->cnt.p;
  a.key = c->key.p;
  a.nq = nq;
  a.L = L;
  a.K = K;
  a.k = k;
  a.fixed = entry_mode == RNNDG_ENTRY_FIXED;
  a.entry_vertex = entry_vertex;
  a.queries = upload(c, c->q_dev, queries, nq * c->d);

  const uint64_t words = (n + 31) / 32;
  unsigned grid = unsigned(nq < uint64_t(sm_count(c)) * 8 ? nq : uint64_t(sm_count(c)) * 8);
  if (!a.fixed) {
    uint32_t count = entry_count ? uint32_t(entry_count < n ? entry_count : n)
                                 : uint32_t(L < n ? L : n);
    uint32_t* ent = c->entry_dev.ensure(count);
    uint32_t* bitmap = nullptr;
    if (count > 64) {  // the sampler's membership map (n bits, once per call)
      bitmap = c->sample_bits.ensure(words);
      RNNDG_CUDA(cudaMemsetAsync(bitmap, 0, words * 4, c->stream));
    }
    RNNDG_LAUNCH(c, k_sample_entries, 1, 32, 0, n, count, seed, ent, bitmap);
    a.entries = ent;
    a.nentries = count;
  }
  uint32_t* oid = c->ids_dev.ensure(nq * k);
  float* odist = c->dists_dev.ensure(nq * k);
  unsigned long long* st = c->qstat_dev.ensure(2 * nq + 1);
  a.out_ids = oid;
  a.out_dists = odist;
  a.out_visited = st;
  a.out_comps = st + nq;
  // seen-set table: ~4 x the distances a query is expected to evaluate
  // (entries + L expansions x the mean out-degree, or K), at least 2^12
  // ids, per block in global memory (L2-resident; cleared per query).  A
  // query past 3/4 of it is re-run with the bitmap, so the mean is enough.
  uint64_t degsum = uint64_t(K) * c->nv;
  if (!K) {
    unsigned long long* dm = st + 2 * nq;
    RNNDG_CUDA(cudaMemsetAsync(dm, 0, 8, c->stream));
    RNNDG_LAUNCH(c, k_sum_u32, unsigned(sm_count(c)) * 4u, 256, 0, c->cnt.p, c->nv, dm);
    RNNDG_CUDA(cudaMemcpyAsync(&degsum, dm, 8, cudaMemcpyDeviceToHost, c->stream));
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  }
  const uint64_t meandeg = c->nv ? (degsum + c->nv - 1) / c->nv : 1;
  const uint64_t expect = (a.fixed ? 1ull : uint64_t(a.nentries)) + uint64_t(L) * (meandeg + 1);
  uint32_t lg = 12;
  while (lg < 26 && (uint64_t(1) << lg) < 4 * expect) ++lg;
  // RNNDG_SEARCH_TAB: force the table size (tests drive the bitmap re-run)
  static const int force_lg = [] {
    const char* e = std::getenv("RNNDG_SEARCH_TAB");
    return e ? std::atoi(e) : 0;
  }();
  // at most ~512 MB of tables for the whole grid; queries that need more
  // take the bitmap re-run
  while (lg > 12 && (uint64_t(4) << lg) * grid > (uint64_t(512) << 20)) --lg;
  if (force_lg >= 4 && force_lg <= 26) lg = uint32_t(force_lg);
  a.tab_log2 = lg;
  a.gtab = c->seen_bits.ensure((uint64_t(1) << lg) * grid);
  const size_t qbytes = (size_t(c->d) * 4 + 15) & ~size_t(15);
  const size_t pbytes = (size_t(L) * 9 + 15) & ~size_t(15);
  size_t smem = qbytes + pbytes;
  DevBuf<uint64_t> gpool;
  DevBuf<uint8_t> gexp;
  if (smem > 160 * 1024) {
    gpool.ensure(uint64_t(L) * grid);
    gexp.ensure(uint64_t(L) * grid);
    a.gpool = gpool.p;
    a.gexp = gexp.p;
    smem = qbytes;
  }
  auto launch = [&](auto kern, unsigned g, size_t sm, const uint32_t* only, uint32_t nonly) {
    // the attribute is raised once per kernel to the largest size used so far
    static size_t set_for[4] = {0, 0, 0, 0};
    static const void* fn[4] = {nullptr, nullptr, nullptr, nullptr};
    int slot = 0;
    while (slot < 3 && fn[slot] && fn[slot] != reinterpret_cast<const void*>(kern)) ++slot;
    fn[slot] = reinterpret_cast<const void*>(kern);
    if (sm > set_for[slot]) {
      RNNDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      set_for[slot] = sm;
    }
    RNNDG_LAUNCH(c, kern, g, 32, sm, a, only, nonly);
  };
  if (c->d % 4 == 0)
    launch(k_search<true, true>, grid, smem, nullptr, 0u);
  else
    launch(k_search<false, true>, grid, smem, nullptr, 0u);
  std::vector<unsigned long long> h(2 * nq);
  RNNDG_CUDA(cudaMemcpyAsync(h.data(), st, 2 * nq * 8, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  // queries that overflowed their table: again with an n-bit map each
  std::vector<uint32_t> redo;
  for (uint64_t i = 0; i < nq; ++i)
    if (h[i] == ~0ull) redo.push_back(uint32_t(i));
  if (!redo.empty()) {
    const unsigned g2 = unsigned(redo.size() < 64 ? redo.size() : 64);
    DevBuf<uint32_t> only, bits;
    only.ensure(redo.size());
    RNNDG_CUDA(cudaMemcpyAsync(only.p, redo.data(), redo.size() * 4, cudaMemcpyHostToDevice,
                               c->stream));
    a.seen = bits.ensure(words * g2);  // <= 64 blocks x n bits, this call only
    a.words_per_map = words;
    const size_t sm2 = a.gpool ? qbytes : qbytes + pbytes;
    if (c->d % 4 == 0)
      launch(k_search<true, false>, g2, sm2, only.p, uint32_t(redo.size()));
    else
      launch(k_search<false, false>, g2, sm2, only.p, uint32_t(redo.size()));
    RNNDG_CUDA(cudaMemcpyAsync(h.data(), st, 2 * nq * 8, cudaMemcpyDeviceToHost, c->stream));
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  }
  RNNDG_CUDA(cudaMemcpyAsync(ids, oid, nq * k * 4, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaMemcpyAsync(dists, odist, nq * k * 4, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  for (uint64_t i = 0; i < nq; ++i) {
    if (visited) visited[i] = h[i];
    if (dist_comps) dist_comps[i] = h[nq + i];
  }
}

void op_brute_force(rnndg_ctx* c, const float* queries, uint64_t nq, uint32_t k,
                    uint32_t* ids) {
  if (k < 1 || k > c->n) throw ParamError("brute_force_gt: k out of range");
  if (k > uint32_t(kBfMaxK)) throw ParamError("brute_force: k > 64 not supported on device");
  const float* q = upload(c, c->q_dev, queries, nq * c->d);
  uint32_t* oid = c->ids_dev.ensure(nq * k);
  const size_t smem = size_t(c->d) * 4;
  const unsigned grid = unsigned(nq < 65535 ? nq : 65535);
  if (c->d % 4 == 0) {
    RNNDG_CUDA(cudaFuncSetAttribute(k_brute_force<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    RNNDG_LAUNCH(c, k_brute_force<true>, grid, kBfThreads, smem, c->x, c->n, c->d, q, nq, k, oid);
  } else {
    RNNDG_CUDA(cudaFuncSetAttribute(k_brute_force<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    RNNDG_LAUNCH(c, k_brute_force<false>, grid, kBfThreads, smem, c->x, c->n, c->d, q, nq, k, oid);
  }
  RNNDG_CUDA(cudaMemcpyAsync(ids, oid, nq * k * 4, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
}

void op_l2_pairs(rnndg_ctx* c, const uint32_t* a, const uint32_t* b, uint64_t np,
                 float* out) {
  if (np == 0) return;
  DevBuf<uint32_t> da, db;
  DevBuf<float> dout;
  da.ensure(np);
  db.ensure(np);
  dout.ensure(np);
  RNNDG_CUDA(cudaMemcpyAsync(da.p, a, np * 4, cudaMemcpyHostToDevice, c->stream));
  RNNDG_CUDA(cudaMemcpyAsync(db.p, b, np * 4, cudaMemcpyHostToDevice, c->stream));
  const unsigned grid = unsigned((np + 255) / 256 < 65535 ? (np + 255) / 256 : 65535);
  if (c->d % 4 == 0)
    RNNDG_LAUNCH(c, k_l2_pairs<true>, grid, 256, 0, c->x, c->d, da.p, db.p, np, dout.p);
  else
    RNNDG_LAUNCH(c, k_l2_pairs<false>, grid, 256, 0, c->x, c->d, da.p, db.p, np, dout.p);
  RNNDG_CUDA(cudaMemcpyAsync(out, dout.p, np * 4, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
}

uint32_t op_rng_strategy(rnndg_ctx* c, uint32_t u, const uint32_t* cand_ids,
                         const float* cand_dists, uint32_t ncand,
                         uint32_t* kept_ids, float* kept_dists) {
  if (ncand == 0) return 0;
  std::vector<uint64_t> hk(ncand);
  for (uint32_t i = 0; i < ncand; ++i) {
    if (cand_ids[i] >= c->n) throw ParamError("rng_strategy: candidate id out of range");
    hk[i] = make_key(cand_dists[i], cand_ids[i], 0u);
  }
  DevBuf<uint64_t> kin, kout;
  DevBuf<uint64_t> segs;
  DevBuf<uint32_t> nk;
  kin.ensure(ncand);
  kout.ensure(ncand);
  segs.ensure(2);
  nk.ensure(1);
  const uint64_t hs[2] = {0, ncand};
  RNNDG_CUDA(cudaMemcpyAsync(kin.p, hk.data(), ncand * 8, cudaMemcpyHostToDevice, c->stream));
  RNNDG_CUDA(cudaMemcpyAsync(segs.p, hs, 16, cudaMemcpyHostToDevice, c->stream));
  size_t bytes = 0;
  RNNDG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, kin.p, kout.p, int(ncand), 1,
                                                segs.p, segs.p + 1, c->stream));
  void* tmp = c->cub_tmp.ensure(bytes);
  RNNDG_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, kin.p, kout.p, int(ncand), 1,
                                                segs.p, segs.p + 1, c->stream));
  c->launches += 3;
  // builder.cpp:201: a candidate equal to u is an error, raised when the
  // sorted walk reaches it; every candidate is walked, so any occurrence
  for (uint32_t i = 0; i < ncand; ++i)
    if (cand_ids[i] == u) throw ParamError("rng_strategy: candidate equals u");
  if (c->d % 4 == 0)
    RNNDG_LAUNCH(c, k_rng_strategy<true>, 1, 32, 0, c->x, c->d, kout.p, ncand, nk.p);
  else
    RNNDG_LAUNCH(c, k_rng_strategy<false>, 1, 32, 0, c->x, c->d, kout.p, ncand, nk.p);
  uint32_t m = 0;
  RNNDG_CUDA(cudaMemcpyAsync(&m, nk.p, 4, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaMemcpyAsync(hk.data(), kout.p, ncand * 8, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  for (uint32_t i = 0; i < m; ++i) {
    kept_ids[i] = key_id(hk[i]);
    uint32_t db = key_dbits(hk[i]);
    std::memcpy(&kept_dists[i], &db, 4);
  }
  return m;
}

void op_degree_stats(rnndg_ctx* c, uint32_t cap, uint64_t out[3]) {
  DevBuf<unsigned int> indeg;
  DevBuf<unsigned long long> o;
  indeg.ensure(c->n);
  o.ensure(3);
  RNNDG_CUDA(cudaMemsetAsync(indeg.p, 0, c->n * 4, c->stream));
  RNNDG_CUDA(cudaMemsetAsync(o.p, 0, 24, c->stream));
  const unsigned grid = unsigned((c->n + 255) / 256 < 4096 ? (c->n + 255) / 256 : 4096);
  RNNDG_LAUNCH(c, k_degree, grid ? grid : 1, 256, 0, c->n, c->off.p, c->cnt.p, c->key.p, cap,
               indeg.p, o.p);
  RNNDG_LAUNCH(c, k_max_u32, grid ? grid : 1, 256, 0, c->n, indeg.p, o.p + 2);
  unsigned long long h[3];
  RNNDG_CUDA(cudaMemcpyAsync(h, o.p, 24, cudaMemcpyDeviceToHost, c->stream));
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  out[0] = h[0];
  out[1] = h[1];
  out[2] = h[2];
}

}  // namespace rnndg
