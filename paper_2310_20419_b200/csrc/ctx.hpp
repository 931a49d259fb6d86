// ctx.hpp -- the rnndg_ctx definition and device buffer plumbing (host side).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "rnndg.h"

namespace rnndg {

// A failed CUDA call or an internal invariant: surfaces as RNNDG_EINTERNAL.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// rnnd::ParamError analogue (common.hpp:21-23): RNNDG_EPARAM.
struct ParamError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
// rnnd::DataError analogue (common.hpp:16-18): RNNDG_EDATA.
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define RNNDG_CUDA(call)                                                     \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      throw ::rnndg::CudaError(std::string(#call) + ": " +                   \
                               cudaGetErrorString(e_) + " at " + __FILE__ +  \
                               ":" + std::to_string(__LINE__));              \
  } while (0)

// Grow-only device allocation.  ensure() discards contents when it grows.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  T* ensure(size_t n) {
    if (n <= cap && p) return p;
    release();
    size_t want = n < 16 ? 16 : n + n / 8;  // headroom against regrowth
    RNNDG_CUDA(cudaMalloc(&p, want * sizeof(T)));
    cap = want;
    return p;
  }
  void swap(DevBuf& o) {
    std::swap(p, o.p);
    std::swap(cap, o.cap);
  }
};

constexpr int kSizeClasses = 8;  // per-class list queues (k_mark_active)

// Device-side counters of one pass (reduced with atomics).
enum Counter : int {
  kRemoved = 0,
  kInserted,
  kFlagSkips,
  kPairChecks,
  kTouched,
  kActiveEntries,
  kActiveCount,
  kLargeCount,
  kMaxLen,
  kEvalPairs,  // distances evaluated by the scan (incl. speculative ones)
  kEvalHub,    // ... of which by the hub-list kernel
  kBigCount,   // hub lists longer than big_hub_threshold() (cluster-cooperative)
  kLongShortCount,  // short lists longer than long_short_threshold() (queued first)
  kGram0,      // lists of <= 16 / 32 / 64 / 128 entries queued for the Gram-filtered
  kGram1,      //   walk (gram.cu), one counter per size class
  kGram2,
  kGram3,
  kClass4,     // ... and four more size classes for the shared-memory walk
  kClass5,     //   (rowwalk.cu queues lists in up to kSizeClasses classes)
  kClass6,
  kClass7,
  kGramAmb,    // Gram-filter comparisons inside the error band (decided exactly)
  kGramExact,  // exact distances evaluated by the Gram-filtered walk
  kMatCount,   // lists queued for resolve_pending (build.cu)
  kNumCounters
};

}  // namespace rnndg

struct rnndg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // concurrent long-list scan
  cudaStream_t side2 = nullptr; // concurrent round-synchronous walk (bsp.cu)
  cudaEvent_t ev_join2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::string err;
  uint64_t launches = 0;
  // pinned host staging for graph export (grown on demand, freed in destroy)
  void* host_stage = nullptr;
  size_t host_stage_bytes = 0;

  // VectorStore (vector_store.hpp:12-20), row-major n x d fp32
  rnndg::DevBuf<float> x_own;
  const float* x = nullptr;
  uint64_t n = 0;  // rows of the store (global vertex count)
  uint32_t d = 0;
  // lists held by this context: vertices [v0, v0 + nv) (SURVEY 8(e) ownership
  // ranges; nv = n, v0 = 0 unless rnndg_set_partition was called)
  uint64_t v0 = 0, nv = 0;
  bool partitioned = false;

  // Graph "A": lists at key[off[u] .. off[u] + cnt[u]).  off is monotone and
  // may leave gaps between lists (capacity layout); span = off[n].
  rnndg::DevBuf<uint64_t> off, off_b;
  rnndg::DevBuf<uint32_t> cnt, cnt_b;
  rnndg::DevBuf<uint64_t> key, key_b, key_s;
  uint64_t span = 0;
  bool has_graph = false;
  bool has_distances = true;
  // every cached dist is the exact l2 of its endpoints (true for graphs built
  // here; false after rnndg_set_graph with caller-provided distances)
  bool exact_dists = true;
  // some list may hold redirected entries whose distance is pending
  // (common.cuh kPendBits); materialize_pending() resolves them
  bool pending = false;

  // pass scratch
  rnndg::DevBuf<uint8_t> active, touch, bflag;
  rnndg::DevBuf<uint32_t> label, brank;
  rnndg::DevBuf<uint64_t> okey, act_small;
  rnndg::DevBuf<uint32_t> act_list, pend_src, bpay, bpay_s;
  rnndg::DevBuf<uint64_t> pend_key, bkey, bkey_s, seg_end, boff;
  rnndg::DevBuf<uint32_t> seg_big;  // segmented sort: count + segments longer than a warp sorts
  rnndg::DevBuf<unsigned long long> bcnt, bcur;
  rnndg::DevBuf<uint32_t> post_cnt;
  rnndg::DevBuf<unsigned long long> counters;
  rnndg::DevBuf<unsigned int> work;
  // NN-Descent baseline (build.cu, nndescent section): pools of capacity
  // nd_cap per vertex (dense n x cap keys, sorted), the pass snapshot and
  // the proposal / segment scratch of a join chunk
  uint32_t nd_K = 0, nd_cap = 0, nd_stride = 0, nd_sample = 0, nd_iters = 0;
  bool nd_ready = false;
  rnndg::DevBuf<uint64_t> nd_pool, nd_pool0, nd_poff, nd_pkey, nd_seg, nd_seg_s, nd_boff;
  rnndg::DevBuf<uint32_t> nd_pcnt, nd_pcnt0, nd_F, nd_fcnt, nd_O, nd_ocnt, nd_np, nd_pdst;
  rnndg::DevBuf<unsigned long long> nd_bcnt, nd_cur;
  // dense CSR staging for rnndg_get_graph (device-side compaction)
  rnndg::DevBuf<uint64_t> ex_off;
  rnndg::DevBuf<uint32_t> ex_ids;
  rnndg::DevBuf<float> ex_dists;
  rnndg::DevBuf<uint8_t> ex_fresh;
  rnndg::DevBuf<uint32_t> kpos_g;  // scan scratch for lists > kScanUcap
  rnndg::DevBuf<uint32_t> gram_q;  // Gram-walk queues, 4 size classes x nv
  // lists whose pending distances are resolved: [mat_b[x], mat_e[x]), vertex mat_e[nv + x]
  rnndg::DevBuf<uint64_t> mat_b, mat_e;
  rnndg::DevBuf<unsigned long long> gram_prof;  // RNNDG_TRACE cycle counters (gram.cu)
  // sharding: staged (dst, key) records, per-part counts
  rnndg::DevBuf<uint32_t> rec_dst, rec_dst2;
  rnndg::DevBuf<uint64_t> rec_key, rec_key2, part_bounds;
  rnndg::DevBuf<unsigned long long> rec_cursor, part_counts;
  uint64_t rec_n = 0;
  // round-synchronous walk (bsp.cu): worklists, per-list state, round counters,
  // the flat task array with its results, per-warp scratch of the last round
  rnndg::DevBuf<uint32_t> bsp_wl, bsp_state;
  rnndg::DevBuf<unsigned int> bsp_ctl;
  rnndg::DevBuf<uint2> bsp_tasks, bsp_itasks;
  rnndg::DevBuf<float> bsp_res, bsp_ires;
  // chain-blocked copy of the store for the distance stage (scan.cu)
  rnndg::DevBuf<float> xp;
  const float* xp_src = nullptr;
  uint32_t xp_stride = 0;
  rnndg::DevBuf<unsigned char> cub_tmp;

  // eval scratch
  rnndg::DevBuf<float> q_dev;
  rnndg::DevBuf<uint32_t> ids_dev, entry_dev, seen_bits, sample_bits;
  rnndg::DevBuf<float> dists_dev;
  rnndg::DevBuf<unsigned long long> qstat_dev;

  std::vector<rnndg_counts> pass_counts;
  bool trace = false;  // RNNDG_TRACE=1: per-pass line on stderr
  bool scan_cfg_logged = false;
  // hub lists in the previous update pass (~0: unknown) and whether the lists
  // were rebuilt in bulk since (random init, reverse phase, imported graph):
  // picks the hub-cluster size of the next scan
  uint64_t hubs_prev = ~0ull;
  bool bulk_fresh = true;
  bool init_fresh = false;  // lists are the random initial lists (all fresh)
  // shard scans since the last rnndg_shard_totals(reset): distance-stage time
  // and the SURVEY 8(d) units, for the sharded bench roofline
  double shard_scan_s = 0.0;
  uint64_t shard_touched = 0, shard_active = 0, shard_passes = 0;
  // timing events
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_scan[3] = {};  // trace only: hub kernel end (side), short kernel end (main), Gram kernel end (main)
};

namespace rnndg {

// launch bookkeeping: every kernel of this library goes through this
#define RNNDG_LAUNCH(ctx, kernel, grid, block, smem, ...)                     \
  do {                                                                      \
    kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);         \
    ++(ctx)->launches;                                                      \
    RNNDG_CUDA(cudaGetLastError());                                         \
  } while (0)

// build.cu
void op_random_init(rnndg_ctx* c, uint32_t S, uint64_t seed);
void op_update_pass(rnndg_ctx* c, rnndg_counts* out, double* t_scan,
                    double* t_sort, double* t_apply, uint64_t* touched,
                    uint64_t* active_entries);
void op_scan_phase(rnndg_ctx* c);
void op_apply_local(rnndg_ctx* c);
void op_read_counters(rnndg_ctx* c, rnndg_counts* out, double* t_scan, double* t_sort,
                      double* t_apply, uint64_t* touched, uint64_t* active_entries);
void op_reverse(rnndg_ctx* c, uint32_t R, int order);
void op_sort_lists(rnndg_ctx* c);
// exact distances for pending entries (all lists), lists re-sorted
void materialize_pending(rnndg_ctx* c);
void op_set_partition(rnndg_ctx* c, uint64_t v_begin, uint64_t v_end);
uint64_t op_shard_scan(rnndg_ctx* c, rnndg_counts* partial);
// NN-Descent baseline (nndescent.cpp, canonical deferred join)
void op_nnd_init(rnndg_ctx* c, uint32_t K, uint32_t sample, uint32_t iters, uint32_t pool,
                 uint64_t seed);
uint64_t op_nnd_pass(rnndg_ctx* c);
void op_nnd_finalize(rnndg_ctx* c);
void op_load_fvecs(rnndg_ctx* c, const char* path, uint64_t* n, uint32_t* d);
// dense CSR (graph.hpp view) of the owned lists into host arrays (any may be
// null); returns the edge count
uint64_t op_export(rnndg_ctx* c, uint64_t* offsets, uint32_t* ids, float* dists,
                   uint8_t* fresh);
uint64_t op_shard_stage(rnndg_ctx* c, int kind);
void op_shard_export(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint32_t* dst_dev,
                     uint64_t* key_dev, uint64_t* counts);
void op_shard_route(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint64_t* counts);
void op_shard_push(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint32_t* const* dst_ptrs,
                   uint64_t* const* key_ptrs, const uint64_t* offsets);
uint64_t op_shard_import(rnndg_ctx* c, int kind, const uint32_t* dst_dev, const uint64_t* key_dev,
                         uint64_t nr, uint32_t R, rnndg_counts* partial);
void op_shard_out_prune(rnndg_ctx* c, uint32_t R);
int sm_count(rnndg_ctx* c);

// eval.cu
void op_search(rnndg_ctx* c, const float* queries, uint64_t nq, uint32_t L,
               uint32_t K, uint32_t k, int entry_mode, uint32_t entry_vertex,
               uint32_t entry_count, uint64_t seed, uint32_t* ids, float* dists,
               uint64_t* visited, uint64_t* dist_comps);
void op_brute_force(rnndg_ctx* c, const float* queries, uint64_t nq, uint32_t k,
                    uint32_t* ids);
void op_l2_pairs(rnndg_ctx* c, const uint32_t* a, const uint32_t* b,
                 uint64_t npairs, float* out);
uint32_t op_rng_strategy(rnndg_ctx* c, uint32_t u, const uint32_t* cand_ids,
                         const float* cand_dists, uint32_t ncand,
                         uint32_t* kept_ids, float* kept_dists);
void op_degree_stats(rnndg_ctx* c, uint32_t cap, uint64_t out[3]);

}  // namespace rnndg
