// dropin_check.cpp -- exercises the C++ drop-ins (rnnd_gpu_builder.cpp,
// rnnd_gpu_search.cpp) through the reference's own API, for
// tests/test_gpu_dropin.py to compare with the unmodified reference
// (oracle/_ref): build -> save_index bytes, batch_search, search of one
// query, brute_force_gt, on the reference's synth_uniform data.
//
// usage: dropin_check n d seed nq L K k T1 T2 out.bin
// out.bin: u64 index size, index bytes, then per query u64 visited,
// u64 dist_comps, k u32 ids, k f32 dists; then nq x k u32 ground truth;
// then the single search of query 0 (u64 visited, u64 comps, k ids).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "rnnd/builder.hpp"
#include "rnnd/graph.hpp"
#include "rnnd/search.hpp"
#include "rnnd/vector_store.hpp"

using namespace rnnd;

int main(int argc, char** argv) {
  if (argc != 11) {
    std::fprintf(stderr, "usage: dropin_check n d seed nq L K k T1 T2 out.bin\n");
    return 2;
  }
  const size_t n = std::strtoull(argv[1], nullptr, 10), d = std::strtoull(argv[2], nullptr, 10);
  const uint64_t seed = std::strtoull(argv[3], nullptr, 10);
  const size_t nq = std::strtoull(argv[4], nullptr, 10);
  SearchParams sp;
  sp.L = uint32_t(std::atoi(argv[5]));
  sp.K = uint32_t(std::atoi(argv[6]));
  sp.k = uint32_t(std::atoi(argv[7]));
  BuildParams bp;
  bp.T1 = uint32_t(std::atoi(argv[8]));
  bp.T2 = uint32_t(std::atoi(argv[9]));
  const VectorStore base = synth_uniform(n, d, seed);
  const VectorStore queries = synth_uniform(nq, d, seed + 1);
  BuildStats st;
  AdjacencyGraph g = build(base, bp, &st);
  const std::string idx = std::string(argv[10]) + ".index";
  save_index(g, idx);
  std::ifstream fi(idx, std::ios::binary);
  std::vector<char> bytes((std::istreambuf_iterator<char>(fi)), std::istreambuf_iterator<char>());
  auto res = batch_search(g, base, queries, sp);
  auto gt = brute_force_gt(base, queries, sp.k);
  auto one = search(g, base, queries.row(0), sp);
  std::ofstream fo(argv[10], std::ios::binary);
  const uint64_t sz = bytes.size();
  fo.write(reinterpret_cast<const char*>(&sz), 8);
  fo.write(bytes.data(), std::streamsize(sz));
  for (const auto& r : res) {
    fo.write(reinterpret_cast<const char*>(&r.visited), 8);
    fo.write(reinterpret_cast<const char*>(&r.dist_comps), 8);
    std::vector<uint32_t> ids(sp.k, 0xFFFFFFFFu);
    std::vector<float> ds(sp.k, 0.f);
    for (size_t j = 0; j < r.ids.size() && j < sp.k; ++j) {
      ids[j] = r.ids[j];
      ds[j] = r.dists[j];
    }
    fo.write(reinterpret_cast<const char*>(ids.data()), 4 * sp.k);
    fo.write(reinterpret_cast<const char*>(ds.data()), 4 * sp.k);
  }
  fo.write(reinterpret_cast<const char*>(gt.ids.data()), std::streamsize(4 * gt.ids.size()));
  fo.write(reinterpret_cast<const char*>(&one.visited), 8);
  fo.write(reinterpret_cast<const char*>(&one.dist_comps), 8);
  std::vector<uint32_t> oid(sp.k, 0xFFFFFFFFu);
  for (size_t j = 0; j < one.ids.size() && j < sp.k; ++j) oid[j] = one.ids[j];
  fo.write(reinterpret_cast<const char*>(oid.data()), 4 * sp.k);
  std::printf("dropin_check: %zu edges, %llu pair checks, %.3f s build\n", g.edge_count(),
              (unsigned long long)st.edits.pair_checks, st.seconds);
  return 0;
}
