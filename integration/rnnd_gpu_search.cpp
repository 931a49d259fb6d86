// rnnd_gpu_search.cpp -- drop-in replacement for the reference's search.cpp,
// plus rnnd::brute_force_gt (dataset.cpp:175-205), on the B200 through the C
// ABI in include/rnndg.h:
//
//   search.hpp:37-38        search          -> rnndg_search, one query
//   search.hpp:45-50        batch_search    -> rnndg_search, all queries at once
//   vector_store.hpp:52-53  brute_force_gt  -> rnndg_brute_force
//
// Link it INSTEAD of src/search.cpp; dataset.cpp stays, compiled with
// -Dbrute_force_gt=brute_force_gt_cpu so that its own brute force does not
// clash (integration/Makefile).  Same parameter validation and messages as
// search.cpp:29-38 / dataset.cpp:176-179.  Results are the reference's: ids,
// dists, visited and dist_comps per query (tests/test_gpu_dropin.py).
// `threads` is ignored (one warp per query on the device); the device's
// brute force supports k <= 64.
#include <chrono>
#include <span>
#include <vector>

#include "rnnd/search.hpp"
#include "rnnd/vector_store.hpp"
#include "rnndg.h"
#include "rnndg_shim.hpp"

namespace rnnd {

namespace {

// search.cpp:29-38
void validate(const AdjacencyGraph& g, const VectorStore& store, size_t qdim,
              const SearchParams& p) {
  if (g.size() == 0) throw ParamError("search: empty graph");
  if (g.size() != store.n) throw ParamError("search: store size mismatch");
  if (qdim != store.d) throw ParamError("search: dimension mismatch");
  if (p.L < 1) throw ParamError("search: L must be >= 1");
  if (p.k < 1 || p.k > p.L) throw ParamError("search: k out of [1, L]");
  if (p.entry == EntryMode::kFixedVertex && p.entry_vertex >= g.size())
    throw ParamError("search: entry vertex out of range");
}

std::vector<SearchResult> run(const AdjacencyGraph& g, const VectorStore& store,
                              const float* queries, size_t nq, const SearchParams& p) {
  shim::bind_store(store);
  shim::bind_graph(g);
  std::vector<uint32_t> ids(nq * p.k);
  std::vector<float> dists(nq * p.k);
  std::vector<uint64_t> vis(nq), comps(nq);
  shim::check(rnndg_search(shim::ctx().h, queries, nq, p.L, p.K, p.k,
                           p.entry == EntryMode::kFixedVertex ? RNNDG_ENTRY_FIXED
                                                              : RNNDG_ENTRY_RANDOM,
                           p.entry_vertex, p.entry_count, p.seed, ids.data(), dists.data(),
                           vis.data(), comps.data()));
  std::vector<SearchResult> out(nq);
  for (size_t q = 0; q < nq; ++q) {
    auto& r = out[q];
    // fewer than k reachable: the device pads with kNone (search.cpp returns
    // only what the pool holds)
    for (uint32_t j = 0; j < p.k; ++j) {
      const uint32_t id = ids[q * p.k + j];
      if (id == 0xFFFFFFFFu) break;
      r.ids.push_back(id);
      r.dists.push_back(dists[q * p.k + j]);
    }
    r.visited = vis[q];
    r.dist_comps = comps[q];
  }
  return out;
}

}  // namespace

SearchResult search(const AdjacencyGraph& g, const VectorStore& store,
                    std::span<const float> query, const SearchParams& params) {
  validate(g, store, query.size(), params);
  return run(g, store, query.data(), 1, params)[0];
}

std::vector<SearchResult> batch_search(const AdjacencyGraph& g, const VectorStore& store,
                                       const VectorStore& queries, const SearchParams& params,
                                       int /*threads*/, BatchTiming* timing) {
  if (queries.n == 0) throw ParamError("batch_search: no queries");
  if (queries.d != store.d) throw ParamError("batch_search: dimension mismatch");
  validate(g, store, queries.d, params);
  const auto t0 = std::chrono::steady_clock::now();
  auto res = run(g, store, queries.data.data(), queries.n, params);
  const double wall =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (timing) {
    timing->wall_seconds = wall;
    timing->qps = wall > 0 ? double(queries.n) / wall : 0.0;
  }
  return res;
}

GroundTruth brute_force_gt(const VectorStore& base, const VectorStore& queries, size_t k,
                           int /*threads*/) {
  // dataset.cpp:176-179
  if (base.d != queries.d) throw DataError("brute_force_gt: dimension mismatch");
  if (k < 1 || k > base.n) throw ParamError("brute_force_gt: k out of range");
  GroundTruth gt;
  gt.k = k;
  gt.ids.assign(queries.n * k, 0);
  if (queries.n == 0) return gt;
  shim::bind_store(base);
  shim::check(rnndg_brute_force(shim::ctx().h, queries.data.data(), queries.n, uint32_t(k),
                                gt.ids.data()));
  return gt;
}

}  // namespace rnnd
