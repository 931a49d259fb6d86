// rnnd_gpu_builder.cpp -- drop-in replacement for the reference's builder.cpp.
//
// Defines the four public functions of include/rnnd/builder.hpp with the
// reference's exact signatures, running them on the B200 through the C ABI in
// include/rnndg.h.  Link it INSTEAD of src/builder.cpp: the rest of the
// reference library (graph.cpp, dataset.cpp, search.cpp, eval.cpp, ...) and
// its callers (CLI, acceptance suite, unit tests) are unchanged.
//
//   builder.hpp:55-56  rng_strategy       -> rnndg_rng_strategy
//   builder.hpp:69-70  update_neighbors   -> rnndg_set_graph + rnndg_update_pass
//   builder.hpp:77-78  add_reverse_edges  -> rnndg_set_graph + rnndg_reverse
//   builder.hpp:84-86  build              -> rnndg_build
//
// `threads` is accepted and ignored: the device always runs the deferred,
// canonical pass the reference runs for threads > 1 (builder.cpp:88-139).
// Error codes map back to the reference's exception classes.
#include <cstring>
#include <string>
#include <vector>

#include "rnnd/builder.hpp"
#include "rnndg.h"

namespace rnnd {

namespace {

struct Ctx {
  rnndg_ctx* h = nullptr;
  const VectorStore* store = nullptr;
  const float* data = nullptr;
  size_t n = 0, d = 0;
  Ctx() {
    if (rnndg_create(&h, 0) != RNNDG_OK) throw std::runtime_error("rnndg: no CUDA device");
  }
  ~Ctx() { rnndg_destroy(h); }
};

Ctx& ctx() {
  thread_local Ctx c;
  return c;
}

void check(int rc) {
  if (rc == RNNDG_OK) return;
  std::string msg = rnndg_last_error(ctx().h);
  if (rc == RNNDG_EPARAM) throw ParamError(msg);
  if (rc == RNNDG_EDATA) throw DataError(msg);
  throw std::runtime_error(msg);
}

// The store is uploaded on every call: the caller may mutate or reallocate
// it between calls (a cached pointer is not an identity).
void bind_store(const VectorStore& s) {
  Ctx& c = ctx();
  check(rnndg_set_data(c.h, s.data.data(), s.n, uint32_t(s.d)));
  c.store = &s;
  c.data = s.data.data();
  c.n = s.n;
  c.d = s.d;
}

void upload(const AdjacencyGraph& g) {
  const size_t n = g.size();
  std::vector<uint64_t> off(n + 1, 0);
  for (size_t u = 0; u < n; ++u) off[u + 1] = off[u] + g.adj[u].size();
  std::vector<uint32_t> ids(off[n]);
  std::vector<float> dists(off[n]);
  std::vector<uint8_t> fresh(off[n]);
  for (size_t u = 0; u < n; ++u)
    for (size_t j = 0; j < g.adj[u].size(); ++j) {
      const auto& e = g.adj[u][j];
      ids[off[u] + j] = e.id;
      dists[off[u] + j] = e.dist;
      fresh[off[u] + j] = e.fresh ? 1 : 0;
    }
  check(rnndg_set_graph(ctx().h, n, off.data(), ids.data(), dists.data(), fresh.data()));
}

void download(AdjacencyGraph& g) {
  uint64_t n = 0, m = 0;
  check(rnndg_graph_size(ctx().h, &n, &m));
  std::vector<uint64_t> off(n + 1);
  std::vector<uint32_t> ids(m ? m : 1);
  std::vector<float> dists(m ? m : 1);
  std::vector<uint8_t> fresh(m ? m : 1);
  check(rnndg_get_graph(ctx().h, off.data(), ids.data(), dists.data(), fresh.data()));
  g.adj.assign(n, {});
  for (uint64_t u = 0; u < n; ++u) {
    auto& l = g.adj[u];
    l.reserve(off[u + 1] - off[u]);
    for (uint64_t j = off[u]; j < off[u + 1]; ++j) l.push_back({ids[j], dists[j], fresh[j] != 0});
  }
  g.has_distances = true;
}

// add_reverse_edges needs no vectors; a 1-d dummy store of the right size
// satisfies the context when the caller has not bound one
void bind_any(size_t n) {
  Ctx& c = ctx();
  static thread_local std::vector<float> zeros;
  zeros.assign(n ? n : 1, 0.0f);
  check(rnndg_set_data(c.h, zeros.data(), n ? n : 1, 1));
  c.store = nullptr;
  c.data = zeros.data();
  c.n = n;
  c.d = 1;
}

}  // namespace

std::vector<NeighborEntry> rng_strategy(const VectorStore& store, uint32_t u,
                                        std::vector<NeighborEntry> candidates) {
  bind_store(store);
  const uint32_t m = uint32_t(candidates.size());
  std::vector<uint32_t> ids(m ? m : 1), kid(m ? m : 1);
  std::vector<float> ds(m ? m : 1), kd(m ? m : 1);
  for (uint32_t i = 0; i < m; ++i) {
    ids[i] = candidates[i].id;
    ds[i] = candidates[i].dist;
  }
  uint32_t nk = 0;
  check(rnndg_rng_strategy(ctx().h, u, ids.data(), ds.data(), m, kid.data(), kd.data(), &nk));
  std::vector<NeighborEntry> kept(nk);
  for (uint32_t i = 0; i < nk; ++i) kept[i] = {kid[i], kd[i], true};
  // rng_strategy returns the candidates' own entries; restore their flags
  for (auto& e : kept)
    for (auto& c : candidates)
      if (c.id == e.id) {
        e.fresh = c.fresh;
        break;
      }
  return kept;
}

EditCounts update_neighbors(AdjacencyGraph& g, const VectorStore& store, int /*threads*/) {
  if (!g.has_distances) throw ParamError("update_neighbors: graph has no distances");
  bind_store(store);
  upload(g);
  rnndg_counts c{};
  check(rnndg_update_pass(ctx().h, &c));
  download(g);
  EditCounts e;
  e.removed = c.removed;
  e.inserted = c.inserted;
  e.flag_skips = c.flag_skips;
  e.pair_checks = c.pair_checks;
  return e;
}

void add_reverse_edges(AdjacencyGraph& g, uint32_t R, int /*threads*/, PruneOrder order) {
  if (R < 1) throw ParamError("add_reverse_edges: R must be >= 1");
  if (!g.has_distances) throw ParamError("add_reverse_edges: graph has no distances");
  bind_any(g.size());
  upload(g);
  check(rnndg_reverse(ctx().h, R,
                      order == PruneOrder::kOutThenIn ? RNNDG_OUT_THEN_IN : RNNDG_IN_THEN_OUT));
  download(g);
}

namespace {
struct ProgressThunk {
  const BuildProgressFn* fn;
};
void progress_cb(uint32_t t1, uint32_t T1, const rnndg_counts* o, double el, void* user) {
  EditCounts e;
  e.removed = o->removed;
  e.inserted = o->inserted;
  e.flag_skips = o->flag_skips;
  e.pair_checks = o->pair_checks;
  (*static_cast<ProgressThunk*>(user)->fn)(t1, T1, e, el);
}
}  // namespace

AdjacencyGraph build(const VectorStore& store, const BuildParams& p, BuildStats* stats,
                     const BuildProgressFn& progress) {
  bind_store(store);
  rnndg_build_stats st{};
  ProgressThunk thunk{&progress};
  check(rnndg_build(ctx().h, p.S, p.R, p.T1, p.T2, p.seed,
                    p.prune_order == PruneOrder::kOutThenIn ? RNNDG_OUT_THEN_IN
                                                            : RNNDG_IN_THEN_OUT,
                    &st, progress ? progress_cb : nullptr, &thunk));
  AdjacencyGraph g;
  download(g);
  if (stats) {
    stats->seconds = st.seconds;
    stats->update_passes = st.update_passes;
    stats->reverse_phases = st.reverse_phases;
    stats->edits.removed = st.edits.removed;
    stats->edits.inserted = st.edits.inserted;
    stats->edits.flag_skips = st.edits.flag_skips;
    stats->edits.pair_checks = st.edits.pair_checks;
  }
  return g;
}

}  // namespace rnnd
