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
// canonical pass the reference runs for threads > 1 (builder.cpp:88-139);
// with threads == 1 the reference runs update_serial (:71-86), whose
// order-dependent redirects give a different graph -- not reproduced here.
// Error codes map back to the reference's exception classes; the store and
// graph uploads are cached per thread (rnndg_shim.hpp).
#include <cstring>
#include <string>
#include <vector>

#include "rnnd/builder.hpp"
#include "rnndg.h"
#include "rnndg_shim.hpp"

namespace rnnd {

using shim::bind_any;
using shim::bind_store;
using shim::check;
using shim::ctx;
using shim::download;
using shim::upload;

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
