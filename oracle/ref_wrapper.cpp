// ref_wrapper.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles the
// reference sources where they lie (/root/reference/proj/src/*.cpp, with the
// reference's own flags: C++20 -O3 -ffp-contract=off -fopenmp, zlib) together
// with this file into oracle/_ref/librnnd_ref.so.  Used to pin the C oracle
// (tests/) and as bench.py's `--impl reference` CPU arm.  Nothing here is
// reference source; it only calls the reference's public API.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

#include "rnnd/builder.hpp"
#include "rnnd/graph.hpp"
#include "rnnd/nndescent.hpp"
#include "rnnd/search.hpp"
#include "rnnd/vector_store.hpp"

using namespace rnnd;

namespace {
VectorStore make_store(const float* data, uint64_t n, uint32_t d) {
  VectorStore s;
  s.n = n;
  s.d = d;
  s.data.assign(data, data + n * d);
  return s;
}
}  // namespace

extern "C" {

struct ref_ctx {
  VectorStore store;
  AdjacencyGraph g;
};

ref_ctx* ref_new(const float* data, uint64_t n, uint32_t d) {
  auto* c = new ref_ctx;
  c->store = make_store(data, n, d);
  c->g = AdjacencyGraph(n);
  return c;
}

void ref_free(ref_ctx* c) { delete c; }

int ref_max_threads() { return omp_get_max_threads(); }

uint64_t ref_edges(ref_ctx* c) { return c->g.edge_count(); }

int ref_random_init(ref_ctx* c, uint32_t S, uint64_t seed) {
  try {
    c->g = random_init(c->store, S, seed);
    return 0;
  } catch (const ParamError&) {
    return 1;
  } catch (...) {
    return 3;
  }
}

// one update pass; threads as in the reference (1 = serial variant)
int ref_update(ref_ctx* c, int threads, uint64_t counts[4]) {
  try {
    EditCounts e = update_neighbors(c->g, c->store, threads);
    counts[0] = e.removed;
    counts[1] = e.inserted;
    counts[2] = e.flag_skips;
    counts[3] = e.pair_checks;
    return 0;
  } catch (const ParamError&) {
    return 1;
  } catch (...) {
    return 3;
  }
}

int ref_reverse(ref_ctx* c, uint32_t R, int threads, int order) {
  try {
    add_reverse_edges(c->g, R, threads,
                      order == 0 ? PruneOrder::kOutThenIn : PruneOrder::kInThenOut);
    return 0;
  } catch (const ParamError&) {
    return 1;
  } catch (...) {
    return 3;
  }
}

// full rnnd::build; stats_out = {seconds, update_passes, reverse_phases,
// removed, inserted, flag_skips, pair_checks}
int ref_build(ref_ctx* c, uint32_t S, uint32_t R, uint32_t T1, uint32_t T2,
              uint64_t seed, int threads, int order, double stats_out[7]) {
  try {
    BuildParams p;
    p.S = S;
    p.R = R;
    p.T1 = T1;
    p.T2 = T2;
    p.seed = seed;
    p.threads = threads;
    p.prune_order = order == 0 ? PruneOrder::kOutThenIn : PruneOrder::kInThenOut;
    BuildStats st;
    c->g = build(c->store, p, &st);
    if (stats_out) {
      stats_out[0] = st.seconds;
      stats_out[1] = st.update_passes;
      stats_out[2] = st.reverse_phases;
      stats_out[3] = double(st.edits.removed);
      stats_out[4] = double(st.edits.inserted);
      stats_out[5] = double(st.edits.flag_skips);
      stats_out[6] = double(st.edits.pair_checks);
    }
    return 0;
  } catch (const ParamError&) {
    return 1;
  } catch (...) {
    return 3;
  }
}

void ref_export(ref_ctx* c, uint64_t* offsets, uint32_t* ids, float* dists,
                uint8_t* fresh) {
  uint64_t off = 0;
  for (size_t u = 0; u < c->g.size(); ++u) {
    if (offsets) offsets[u] = off;
    for (auto& e : c->g.adj[u]) {
      if (ids) ids[off] = e.id;
      if (dists) dists[off] = e.dist;
      if (fresh) fresh[off] = e.fresh ? 1 : 0;
      ++off;
    }
  }
  if (offsets) offsets[c->g.size()] = off;
}

void ref_import(ref_ctx* c, const uint64_t* offsets, const uint32_t* ids,
                const float* dists, const uint8_t* fresh) {
  for (size_t u = 0; u < c->g.size(); ++u) {
    auto& l = c->g.adj[u];
    l.clear();
    for (uint64_t j = offsets[u]; j < offsets[u + 1]; ++j)
      l.push_back({ids[j], dists[j], fresh[j] != 0});
  }
  c->g.has_distances = true;
}

// serialised index via rnnd::save_index; returns size, copies if buf
uint64_t ref_index_bytes(ref_ctx* c, uint8_t* buf, uint64_t cap) {
  auto path = (std::filesystem::temp_directory_path() /
               ("rnnd_ref_idx_" + std::to_string(reinterpret_cast<uintptr_t>(c))))
                  .string();
  save_index(c->g, path);
  std::ifstream in(path, std::ios::binary);
  std::vector<char> b((std::istreambuf_iterator<char>(in)),
                      std::istreambuf_iterator<char>());
  std::filesystem::remove(path);
  if (buf && cap >= b.size()) std::memcpy(buf, b.data(), b.size());
  return b.size();
}

// rnnd::batch_search; ids/dists are nq*k (short results padded with
// UINT32_MAX / +inf); returns wall seconds (<0 on error)
double ref_batch_search(ref_ctx* c, const float* queries, uint64_t nq,
                        uint32_t L, uint32_t K, uint32_t k, uint64_t seed,
                        int threads, uint32_t* ids, float* dists,
                        uint64_t* visited, uint64_t* dist_comps) {
  try {
    VectorStore qs = make_store(queries, nq, uint32_t(c->store.d));
    SearchParams p;
    p.L = L;
    p.K = K;
    p.k = k;
    p.seed = seed;
    BatchTiming t;
    auto res = batch_search(c->g, c->store, qs, p, threads, &t);
    for (uint64_t q = 0; q < nq; ++q) {
      for (uint32_t j = 0; j < k; ++j) {
        bool have = j < res[q].ids.size();
        ids[q * k + j] = have ? res[q].ids[j] : UINT32_MAX;
        dists[q * k + j] = have ? res[q].dists[j] : __builtin_inff();
      }
      if (visited) visited[q] = res[q].visited;
      if (dist_comps) dist_comps[q] = res[q].dist_comps;
    }
    return t.wall_seconds;
  } catch (...) {
    return -1.0;
  }
}

int ref_brute_force(const float* base, uint64_t n, uint32_t d,
                    const float* queries, uint64_t nq, uint32_t k, int threads,
                    uint32_t* ids) {
  try {
    VectorStore b = make_store(base, n, d);
    VectorStore q = make_store(queries, nq, d);
    GroundTruth gt = brute_force_gt(b, q, k, threads);
    std::memcpy(ids, gt.ids.data(), sizeof(uint32_t) * gt.ids.size());
    return 0;
  } catch (...) {
    return 3;
  }
}

// NnDescent (nndescent.cpp) with threads = 1 (deterministic): the pools after
// init (pool_* arrays, dense n x cap, counts in pool_cnt) and the graph after
// `iters` join passes + finalize (CSR).  1 on ParamError.
int ref_nndescent(const float* data, uint64_t n, uint32_t d, uint32_t K, uint32_t sample,
                  uint32_t iters, uint32_t pool, uint64_t seed, uint32_t cap,
                  uint32_t* pool_cnt, uint32_t* pool_ids, float* pool_dists,
                  uint64_t* offsets, uint32_t* ids, float* dists) {
  try {
    VectorStore st = make_store(data, n, d);
    NnDescentParams p;
    p.K = K;
    p.sample = sample;
    p.iters = iters;
    p.pool = pool;
    p.seed = seed;
    p.threads = 1;
    NnDescent nnd(st, p);
    nnd.init();
    for (uint64_t u = 0; u < n; ++u) {
      const auto& pl = nnd.pools()[u];
      pool_cnt[u] = uint32_t(pl.size());
      for (size_t j = 0; j < pl.size() && j < cap; ++j) {
        pool_ids[u * cap + j] = pl[j].id;
        pool_dists[u * cap + j] = pl[j].dist;
      }
    }
    for (uint32_t it = 0; it < iters; ++it) nnd.join_pass();
    AdjacencyGraph g = nnd.finalize();
    uint64_t w = 0;
    for (uint64_t u = 0; u < n; ++u) {
      offsets[u] = w;
      for (const auto& e : g.adj[u]) {
        ids[w] = e.id;
        dists[w] = e.dist;
        ++w;
      }
    }
    offsets[n] = w;
    return 0;
  } catch (const ParamError&) {
    return 1;
  } catch (...) {
    return 3;
  }
}

// load_fvecs / load_ivecs (dataset.cpp:82-119): 0 and (n, d) on success,
// 2 (DataError) with the message copied into err, 3 otherwise
int ref_load_vecs(const char* path, int ivecs, uint64_t* n, uint64_t* d, char* err,
                  uint64_t err_cap) {
  try {
    if (ivecs) {
      GroundTruth gt = load_ivecs(path);
      *n = gt.rows();
      *d = gt.k;
    } else {
      VectorStore st = load_fvecs(path);
      *n = st.n;
      *d = st.d;
    }
    return 0;
  } catch (const DataError& e) {
    std::snprintf(err, err_cap, "%s", e.what());
    return 2;
  } catch (...) {
    return 3;
  }
}

}  // extern "C"
