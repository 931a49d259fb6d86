// api.cu -- the extern "C" boundary (include/rnndg.h).  Each entry point
// validates like the reference function it replaces, maps exceptions to the
// reference's error classes, and runs the work on the context's device.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"

using namespace rnndg;

namespace {

template <class Fn>
int guarded(rnndg_ctx* c, Fn fn) {
  if (!c) return RNNDG_EPARAM;
  try {
    RNNDG_CUDA(cudaSetDevice(c->device));
    fn();
    c->err.clear();
    return RNNDG_OK;
  } catch (const rnndg::ParamError& e) {
    c->err = e.what();
    return RNNDG_EPARAM;
  } catch (const rnndg::DataError& e) {
    c->err = e.what();
    return RNNDG_EDATA;
  } catch (const std::exception& e) {
    c->err = e.what();
    return RNNDG_EINTERNAL;
  }
}

void need_data(rnndg_ctx* c) {
  if (!c->x || c->n == 0) throw ParamError("no vector data: call rnndg_set_data first");
}
void need_graph(rnndg_ctx* c) {
  need_data(c);
  if (!c->has_graph) throw ParamError("no graph on the context");
}
// whole-graph entry points index [0, n) arrays: not on a vertex shard
// (rnndg_set_partition); the shard protocol has its own rnndg_shard_* calls
void need_whole(rnndg_ctx* c, const char* what) {
  if (c->partitioned)
    throw ParamError(std::string(what) + ": not available on a partitioned context");
}

// zlib crc32 (graph.cpp:41-43): IEEE 802.3, reflected polynomial 0xEDB88320
uint32_t crc32_ieee(const uint8_t* p, size_t size) {
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < size; ++i) c = table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// device CSR (capacity layout) -> host (counts, keys) in list order
}  // namespace

extern "C" {

int rnndg_create(rnndg_ctx** out, int device) {
  if (!out) return RNNDG_EPARAM;
  *out = nullptr;
  auto* c = new rnndg_ctx;
  c->device = device;
  try {
    int ndev = 0;
    RNNDG_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ParamError("rnndg_create: no such device");
    RNNDG_CUDA(cudaSetDevice(device));
    RNNDG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    RNNDG_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    RNNDG_CUDA(cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking));
    RNNDG_CUDA(cudaEventCreateWithFlags(&c->ev_join2, cudaEventDisableTiming));
    RNNDG_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    RNNDG_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    for (auto& e : c->ev) RNNDG_CUDA(cudaEventCreate(&e));
    for (auto& e : c->ev_scan) RNNDG_CUDA(cudaEventCreate(&e));
    const char* tr = std::getenv("RNNDG_TRACE");
    c->trace = tr && tr[0] == '1';
  } catch (const ParamError&) {
    delete c;
    return RNNDG_EPARAM;
  } catch (...) {
    delete c;
    return RNNDG_EINTERNAL;
  }
  *out = c;
  return RNNDG_OK;
}

int rnndg_destroy(rnndg_ctx* c) {
  if (!c) return RNNDG_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_scan)
    if (e) cudaEventDestroy(e);
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->side2) cudaStreamSynchronize(c->side2);
  if (c->ev_join2) cudaEventDestroy(c->ev_join2);
  if (c->side2) cudaStreamDestroy(c->side2);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->host_stage) cudaFreeHost(c->host_stage);
  delete c;
  return RNNDG_OK;
}

const char* rnndg_last_error(const rnndg_ctx* c) { return c ? c->err.c_str() : "null context"; }

uint64_t rnndg_kernel_launches(const rnndg_ctx* c) { return c ? c->launches : 0; }

int rnndg_set_data(rnndg_ctx* c, const float* rows, uint64_t n, uint32_t d) {
  return guarded(c, [&] {
    if (!rows || n == 0 || d == 0) throw ParamError("set_data: empty store");
    if (n >= (1ull << 31)) throw ParamError("set_data: n must be < 2^31");
    c->x_own.ensure(n * d);
    RNNDG_CUDA(cudaMemcpyAsync(c->x_own.p, rows, n * d * 4, cudaMemcpyHostToDevice, c->stream));
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
    c->x = c->x_own.p;
    c->n = n;
    c->d = d;
    c->v0 = 0;
    c->nv = n;
    c->partitioned = false;
    c->has_graph = false;
    c->pending = false;
    c->xp_src = nullptr;  // chain-blocked copy is stale
  });
}

int rnndg_nnd_init(rnndg_ctx* c, uint32_t K, uint32_t sample, uint32_t iters, uint32_t pool,
                   uint64_t seed) {
  return guarded(c, [&] {
    need_data(c);
    op_nnd_init(c, K, sample, iters, pool, seed);
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int rnndg_nnd_pass(rnndg_ctx* c, uint64_t* new_entries) {
  return guarded(c, [&] {
    need_data(c);
    const uint64_t m = op_nnd_pass(c);
    if (new_entries) *new_entries = m;
  });
}

int rnndg_nnd_pools(rnndg_ctx* c, uint32_t* cap_out, uint32_t* cnt, uint32_t* ids, float* dists,
                    uint8_t* fresh) {
  return guarded(c, [&] {
    need_data(c);
    if (!c->nd_ready) throw ParamError("nndescent: call init first");
    const uint64_t n = c->n, cap = c->nd_stride;
    if (cap_out) *cap_out = c->nd_stride;
    if (cnt)
      RNNDG_CUDA(cudaMemcpyAsync(cnt, c->nd_pcnt.p, n * 4, cudaMemcpyDeviceToHost, c->stream));
    if (ids || dists || fresh) {
      std::vector<uint64_t> keys(n * cap);
      RNNDG_CUDA(cudaMemcpyAsync(keys.data(), c->nd_pool.p, n * cap * 8, cudaMemcpyDeviceToHost,
                                 c->stream));
      RNNDG_CUDA(cudaStreamSynchronize(c->stream));
      for (uint64_t i = 0; i < n * cap; ++i) {
        const uint64_t k = keys[i];
        if (ids) ids[i] = key_id(k);
        if (dists) {
          const uint32_t b = key_dbits(k);
          std::memcpy(&dists[i], &b, 4);
        }
        if (fresh) fresh[i] = uint8_t(key_fresh(k));
      }
    }
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int rnndg_nnd_finalize(rnndg_ctx* c) {
  return guarded(c, [&] {
    need_data(c);
    op_nnd_finalize(c);
  });
}

int rnndg_nnd_build(rnndg_ctx* c, uint32_t K, uint32_t sample, uint32_t iters, uint32_t pool,
                    uint64_t seed, rnndg_build_stats* stats) {
  return guarded(c, [&] {
    need_data(c);
    c->xp_src = nullptr;  // the chain-blocked copy is rebuilt inside the timed build
    cudaEvent_t e0, e1;
    RNNDG_CUDA(cudaEventCreate(&e0));
    RNNDG_CUDA(cudaEventCreate(&e1));
    RNNDG_CUDA(cudaEventRecord(e0, c->stream));
    const uint64_t l0 = c->launches;
    op_nnd_init(c, K, sample, iters, pool, seed);
    for (uint32_t it = 0; it < iters; ++it) op_nnd_pass(c);
    op_nnd_finalize(c);
    RNNDG_CUDA(cudaEventRecord(e1, c->stream));
    RNNDG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    RNNDG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (stats) {
      *stats = rnndg_build_stats{};
      stats->seconds = ms * 1e-3;
      stats->update_passes = iters;
      stats->kernel_launches = c->launches - l0;
    }
  });
}

int rnndg_load_fvecs(rnndg_ctx* c, const char* path, uint64_t* n, uint32_t* d) {
  return guarded(c, [&] {
    if (!path) throw ParamError("load_fvecs: path required");
    op_load_fvecs(c, path, n, d);
  });
}

int rnndg_set_data_device(rnndg_ctx* c, const float* rows_dev, uint64_t n, uint32_t d) {
  return guarded(c, [&] {
    if (!rows_dev || n == 0 || d == 0) throw ParamError("set_data: empty store");
    if (n >= (1ull << 31)) throw ParamError("set_data: n must be < 2^31");
    if (d % 4 == 0 && (reinterpret_cast<uintptr_t>(rows_dev) & 15))
      throw ParamError("set_data_device: rows must be 16-byte aligned");
    c->x_own.release();
    c->x = rows_dev;
    c->n = n;
    c->d = d;
    c->v0 = 0;
    c->nv = n;
    c->partitioned = false;
    c->has_graph = false;
    c->pending = false;
    c->xp_src = nullptr;
  });
}

int rnndg_random_init(rnndg_ctx* c, uint32_t S, uint64_t seed) {
  return guarded(c, [&] {
    need_data(c);
    op_random_init(c, S, seed);
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int rnndg_update_pass(rnndg_ctx* c, rnndg_counts* out) {
  return guarded(c, [&] {
    need_graph(c);
    need_whole(c, "update_neighbors");
    if (!c->has_distances) throw ParamError("update_neighbors: graph has no distances");
    rnndg_counts cc{};
    op_update_pass(c, &cc, nullptr, nullptr, nullptr, nullptr, nullptr);
    materialize_pending(c);  // the caller's graph carries exact distances
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
    if (out) *out = cc;
  });
}

int rnndg_reverse(rnndg_ctx* c, uint32_t R, int order) {
  return guarded(c, [&] {
    need_graph(c);
    need_whole(c, "add_reverse_edges");
    op_reverse(c, R, order);
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int rnndg_sort_lists(rnndg_ctx* c) {
  return guarded(c, [&] {
    need_graph(c);
    need_whole(c, "sort_lists");
    op_sort_lists(c);
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int rnndg_build(rnndg_ctx* c, uint32_t S, uint32_t R, uint32_t T1, uint32_t T2,
                uint64_t seed, int order, rnndg_build_stats* stats,
                rnndg_progress_fn progress, void* user) {
  return guarded(c, [&] {
    need_data(c);
    need_whole(c, "build");
    // builder.cpp:255-258
    if (c->n < 2) throw ParamError("build: need at least 2 vectors");
    if (S < 1 || S > c->n - 1) throw ParamError("build: S out of [1, n-1]");
    if (R < 1) throw ParamError("build: R must be >= 1");
    if (T1 < 1 || T2 < 1) throw ParamError("build: T1 and T2 must be >= 1");
    rnndg_build_stats st{};
    const uint64_t launches0 = c->launches;
    c->pass_counts.clear();
    RNNDG_CUDA(cudaEventRecord(c->ev[4], c->stream));
    c->xp_src = nullptr;  // the chain-blocked store copy is rebuilt inside the timed build
    op_random_init(c, S, seed);
    for (uint32_t t1 = 1; t1 <= T1; ++t1) {
      rnndg_counts outer{};
      for (uint32_t t2 = 0; t2 < T2; ++t2) {
        rnndg_counts pc{};
        op_update_pass(c, &pc, &st.scan_seconds, &st.sort_seconds, &st.apply_seconds,
                       &st.touched, &st.active_entries);
        c->pass_counts.push_back(pc);
        outer.removed += pc.removed;
        outer.inserted += pc.inserted;
        outer.flag_skips += pc.flag_skips;
        outer.pair_checks += pc.pair_checks;
        ++st.update_passes;
      }
      if (t1 != T1) {
        RNNDG_CUDA(cudaEventRecord(c->ev[6], c->stream));
        op_reverse(c, R, order);
        RNNDG_CUDA(cudaEventRecord(c->ev[7], c->stream));
        RNNDG_CUDA(cudaEventSynchronize(c->ev[7]));
        float ms = 0.f;
        RNNDG_CUDA(cudaEventElapsedTime(&ms, c->ev[6], c->ev[7]));
        st.reverse_seconds += ms * 1e-3;
        ++st.reverse_phases;
      }
      st.edits.removed += outer.removed;
      st.edits.inserted += outer.inserted;
      st.edits.flag_skips += outer.flag_skips;
      st.edits.pair_checks += outer.pair_checks;
      if (progress) {
        RNNDG_CUDA(cudaEventRecord(c->ev[5], c->stream));
        RNNDG_CUDA(cudaEventSynchronize(c->ev[5]));
        float ms = 0.f;
        RNNDG_CUDA(cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]));
        progress(t1, T1, &outer, ms * 1e-3, user);
      }
    }
    // builder.cpp:283-285 sorts every list nearest-first: the device lists
    // are sorted (build.cu invariant) once the last pass's pending redirect
    // distances are resolved
    materialize_pending(c);
    RNNDG_CUDA(cudaEventRecord(c->ev[5], c->stream));
    RNNDG_CUDA(cudaEventSynchronize(c->ev[5]));
    float ms = 0.f;
    RNNDG_CUDA(cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]));
    st.seconds = ms * 1e-3;
    st.kernel_launches = c->launches - launches0;
    st.scan_launches = st.update_passes;
    if (stats) *stats = st;
  });
}

int rnndg_pass_counts(const rnndg_ctx* c, rnndg_counts* out, uint32_t cap) {
  if (!c) return RNNDG_EPARAM;
  const uint32_t m = uint32_t(std::min<size_t>(cap, c->pass_counts.size()));
  for (uint32_t i = 0; i < m; ++i) out[i] = c->pass_counts[i];
  return RNNDG_OK;
}

int rnndg_graph_size(rnndg_ctx* c, uint64_t* n, uint64_t* edges) {
  return guarded(c, [&] {
    need_graph(c);
    const uint64_t m = op_export(c, nullptr, nullptr, nullptr, nullptr);
    if (n) *n = c->nv;
    if (edges) *edges = m;
  });
}

int rnndg_get_graph(rnndg_ctx* c, uint64_t* offsets, uint32_t* ids, float* dists,
                    uint8_t* fresh) {
  return guarded(c, [&] {
    need_graph(c);
    op_export(c, offsets, ids, dists, fresh);  // compacted on the device
  });
}

int rnndg_set_graph(rnndg_ctx* c, uint64_t n, const uint64_t* offsets, const uint32_t* ids,
                    const float* dists, const uint8_t* fresh) {
  return guarded(c, [&] {
    need_data(c);
    if (n != c->nv) throw DataError("set_graph: graph size does not match the store");
    if (!offsets) throw ParamError("set_graph: offsets required");
    if (offsets[0] != 0) throw DataError("set_graph: bad offsets");
    for (uint64_t u = 0; u < n; ++u)
      if (offsets[u + 1] < offsets[u]) throw DataError("set_graph: bad offsets");
    const uint64_t m = offsets[n];
    if (m && !ids) throw ParamError("set_graph: ids required");
    std::vector<uint64_t> keys(m ? m : 1);
    std::vector<uint32_t> cnt(n);
    std::vector<uint32_t> scratch;
    for (uint64_t u = 0; u < n; ++u) {
      const uint64_t a = offsets[u], b = offsets[u + 1];
      if (b - a >= (1ull << 32)) throw DataError("set_graph: list too long");
      cnt[u] = uint32_t(b - a);
      scratch.assign(ids + a, ids + b);
      for (uint64_t j = a; j < b; ++j) {
        if (ids[j] >= c->n) throw DataError("set_graph: id out of range");
        if (ids[j] == c->v0 + u) throw DataError("set_graph: self-loop");
        float dv = dists ? dists[j] : 0.0f;
        if (dists && !(dv >= 0.0f)) throw DataError("set_graph: distance must be >= 0");
        if (dv == 0.0f) dv = 0.0f;  // canonical +0
        keys[j] = make_key(dv, ids[j], fresh ? (fresh[j] ? 1u : 0u) : 0u);
      }
      std::sort(scratch.begin(), scratch.end());
      if (std::adjacent_find(scratch.begin(), scratch.end()) != scratch.end())
        throw DataError("set_graph: duplicate edge");
    }
    c->off.ensure(n + 1);
    c->cnt.ensure(n + 1);
    c->key.ensure(m ? m : 1);
    RNNDG_CUDA(cudaMemcpyAsync(c->off.p, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, c->stream));
    RNNDG_CUDA(cudaMemcpyAsync(c->cnt.p, cnt.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
    if (m) RNNDG_CUDA(cudaMemcpyAsync(c->key.p, keys.data(), m * 8, cudaMemcpyHostToDevice, c->stream));
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
    c->span = m;
    c->has_graph = true;
    c->pending = false;
    c->has_distances = dists != nullptr;
    c->exact_dists = false;  // caller-provided distances: id-based membership
    // graphs with cached distances keep every list sorted by (dist, id)
    // (build.cu invariant); a graph loaded without distances keeps its stored
    // order, which select_nearest then uses (graph.cpp:65-74)
    if (c->has_distances) op_sort_lists(c);
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int rnndg_index_bytes(rnndg_ctx* c, uint8_t* buf, uint64_t* size) {
  return guarded(c, [&] {
    need_graph(c);
    need_whole(c, "index_bytes");
    const uint64_t m = op_export(c, nullptr, nullptr, nullptr, nullptr);
    const uint64_t total = 16 + (c->nv + 1) * 8 + m * 4 + 4;
    if (size) *size = total;
    if (!buf) return;
    std::vector<uint64_t> offs(c->nv + 1);
    std::vector<uint32_t> ids(m ? m : 1);
    op_export(c, offs.data(), ids.data(), nullptr, nullptr);
    // graph.cpp:102-126: "RNND", u32 version 1, u64 n, u64 offsets[n+1],
    // u32 ids, u32 CRC-32 of everything before; little-endian
    uint8_t* p = buf;
    auto put32 = [&](uint32_t v) {
      for (int i = 0; i < 4; ++i) *p++ = uint8_t(v >> (8 * i));
    };
    auto put64 = [&](uint64_t v) {
      put32(uint32_t(v));
      put32(uint32_t(v >> 32));
    };
    std::memcpy(p, "RNND", 4);
    p += 4;
    put32(1);
    put64(c->nv);
    for (uint64_t u = 0; u <= c->nv; ++u) put64(offs[u]);
    for (uint64_t j = 0; j < m; ++j) put32(ids[j]);
    put32(crc32_ieee(buf, size_t(p - buf)));
  });
}

int rnndg_degree_stats(rnndg_ctx* c, uint32_t cap, uint64_t out[3]) {
  return guarded(c, [&] {
    need_graph(c);
    need_whole(c, "degree_stats");
    op_degree_stats(c, cap, out);
  });
}

int rnndg_search(rnndg_ctx* c, const float* queries, uint64_t nq, uint32_t L, uint32_t K,
                 uint32_t k, int entry_mode, uint32_t entry_vertex, uint32_t entry_count,
                 uint64_t seed, uint32_t* ids, float* dists, uint64_t* visited,
                 uint64_t* dist_comps) {
  return guarded(c, [&] {
    need_graph(c);
    need_whole(c, "search");
    op_search(c, queries, nq, L, K, k, entry_mode, entry_vertex, entry_count, seed, ids,
              dists, visited, dist_comps);
  });
}

int rnndg_brute_force(rnndg_ctx* c, const float* queries, uint64_t nq, uint32_t k,
                      uint32_t* ids) {
  return guarded(c, [&] {
    need_data(c);
    op_brute_force(c, queries, nq, k, ids);
  });
}

int rnndg_rng_strategy(rnndg_ctx* c, uint32_t u, const uint32_t* cand_ids,
                       const float* cand_dists, uint32_t ncand, uint32_t* kept_ids,
                       float* kept_dists, uint32_t* nkept) {
  return guarded(c, [&] {
    need_data(c);
    const uint32_t m = op_rng_strategy(c, u, cand_ids, cand_dists, ncand, kept_ids, kept_dists);
    if (nkept) *nkept = m;
  });
}

int rnndg_l2_pairs(rnndg_ctx* c, const uint32_t* a, const uint32_t* b, uint64_t npairs,
                   float* out) {
  return guarded(c, [&] {
    need_data(c);
    for (uint64_t i = 0; i < npairs; ++i)
      if (a[i] >= c->n || b[i] >= c->n) throw ParamError("l2_pairs: id out of range");
    op_l2_pairs(c, a, b, npairs, out);
  });
}

int rnndg_set_partition(rnndg_ctx* c, uint64_t v_begin, uint64_t v_end) {
  return guarded(c, [&] {
    need_data(c);
    op_set_partition(c, v_begin, v_end);
  });
}

int rnndg_shard_scan(rnndg_ctx* c, rnndg_counts* partial, uint64_t* nrecords) {
  return guarded(c, [&] {
    need_graph(c);
    if (!c->has_distances) throw ParamError("update_neighbors: graph has no distances");
    rnndg_counts cc{};
    const uint64_t m = op_shard_scan(c, &cc);
    if (partial) *partial = cc;
    if (nrecords) *nrecords = m;
  });
}

int rnndg_shard_totals(rnndg_ctx* c, double* scan_seconds, uint64_t* touched,
                       uint64_t* active_entries, uint64_t* passes, int reset) {
  return guarded(c, [&] {
    if (scan_seconds) *scan_seconds = c->shard_scan_s;
    if (touched) *touched = c->shard_touched;
    if (active_entries) *active_entries = c->shard_active;
    if (passes) *passes = c->shard_passes;
    if (reset) {
      c->shard_scan_s = 0.0;
      c->shard_touched = c->shard_active = c->shard_passes = 0;
    }
  });
}

int rnndg_shard_stage(rnndg_ctx* c, int kind, uint64_t* nrecords) {
  return guarded(c, [&] {
    need_graph(c);
    if (kind != RNNDG_X_PROPOSAL && kind != RNNDG_X_INEDGE)
      throw ParamError("shard_stage: kind must be PROPOSAL or INEDGE");
    const uint64_t m = op_shard_stage(c, kind);
    if (nrecords) *nrecords = m;
  });
}

int rnndg_shard_export(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint32_t* dst_dev,
                       uint64_t* key_dev, uint64_t* counts) {
  return guarded(c, [&] {
    need_graph(c);
    if (!bounds || parts == 0 || !counts) throw ParamError("shard_export: bounds/counts required");
    op_shard_export(c, bounds, parts, dst_dev, key_dev, counts);
  });
}

int rnndg_shard_route(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts, uint64_t* counts) {
  return guarded(c, [&] {
    need_graph(c);
    if (!bounds || !counts) throw ParamError("shard_route: bounds/counts required");
    op_shard_route(c, bounds, parts, counts);
  });
}

int rnndg_shard_push(rnndg_ctx* c, const uint64_t* bounds, uint32_t parts,
                     uint32_t* const* dst_ptrs, uint64_t* const* key_ptrs,
                     const uint64_t* offsets) {
  return guarded(c, [&] {
    need_graph(c);
    if (!bounds || !dst_ptrs || !key_ptrs || !offsets)
      throw ParamError("shard_push: bounds/buffers/offsets required");
    op_shard_push(c, bounds, parts, dst_ptrs, key_ptrs, offsets);
  });
}

int rnndg_shard_import(rnndg_ctx* c, int kind, const uint32_t* dst_dev, const uint64_t* key_dev,
                       uint64_t nrecords, uint32_t R, rnndg_counts* partial, uint64_t* nstaged) {
  return guarded(c, [&] {
    need_graph(c);
    if (kind < RNNDG_X_PENDING || kind > RNNDG_X_DELETE) throw ParamError("shard_import: bad kind");
    if (kind == RNNDG_X_INEDGE && R < 1) throw ParamError("add_reverse_edges: R must be >= 1");
    rnndg_counts cc{};
    const uint64_t m = op_shard_import(c, kind, dst_dev, key_dev, nrecords, R, &cc);
    if (partial) *partial = cc;
    if (nstaged) *nstaged = m;
  });
}

int rnndg_shard_out_prune(rnndg_ctx* c, uint32_t R) {
  return guarded(c, [&] {
    need_graph(c);
    if (R < 1) throw ParamError("add_reverse_edges: R must be >= 1");
    op_shard_out_prune(c, R);
    RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
