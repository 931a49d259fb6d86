// multi.cu -- the vertex-sharded build behind the C ABI, in one process:
// rnndg_sharded_* (include/rnndg.h).  No torch, no Python.
//
// Shard i is an rnndg_ctx on CUDA device devs[i] owning the contiguous
// vertex range [b_i, b_i+1) (rnndg_set_partition); every shard holds the
// whole store.  Per update pass each shard scans its own lists and stages its
// redirects as (dst, key) records.  The exchange is fused into the producing
// side: every shard counts its records per owner
// (rnndg_shard_route), the host lays out each owner's receive buffer from the
// P x P counts, and one kernel per shard stores every record straight into
// its owner's buffer (rnndg_shard_push) -- peer-mapped memory over NVLink /
// NVSwitch between distinct B200s (peer access enabled at creation), plain
// device memory when shards share a GPU -- with no sort by destination, no
// staging copy and no collective; then the owner applies them
// (rnndg_shard_import).  RNNDG_MULTI_EXCHANGE=copy selects the older path
// (records sorted by destination, cudaMemcpyPeerAsync per segment).  A
// reverse phase exchanges proposals, in-edges and deletions the same way
// (builder.cpp:222-251).  Every step is set-canonical, so the graph and every
// pass count equal rnndg_build's (tests/test_gpu_multi.py) -- the protocol of
// paper_2310_20419_b200/sharded.py without the collective.  Each phase runs
// on one host thread per shard, so the shards' kernels overlap across
// devices; the phases are separated by joins (the exchange is a data
// dependency between passes).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>
#include <string>
#include <vector>

#include "ctx.hpp"
#include "rnndg.h"

struct rnndg_sharded {
  std::vector<int> devs;
  std::vector<rnndg_ctx*> ctx;
  std::vector<cudaStream_t> copy;  // per shard: receive-side copy stream
  // per shard device buffers: send (export) and receive (import) records
  std::vector<uint32_t*> sdst, rdst;
  std::vector<uint64_t*> skey, rkey;
  std::vector<uint64_t> scap_d, scap_k, rcap_d, rcap_k, nstaged;
  std::vector<uint64_t> bounds;
  std::vector<rnndg_counts> pass_counts;
  uint64_t n = 0;
  std::string err;
};

namespace {

using rnndg::CudaError;
using rnndg::DataError;
using rnndg::ParamError;

template <class Fn>
int sguard(rnndg_sharded* h, Fn fn) {
  if (!h) return RNNDG_EPARAM;
  try {
    fn();
    h->err.clear();
    return RNNDG_OK;
  } catch (const ParamError& e) {
    h->err = e.what();
    return RNNDG_EPARAM;
  } catch (const DataError& e) {
    h->err = e.what();
    return RNNDG_EDATA;
  } catch (const std::exception& e) {
    h->err = e.what();
    return RNNDG_EINTERNAL;
  }
}

// a shard call that failed: its message, tagged with the shard
void chk(rnndg_sharded* h, size_t i, int rc) {
  if (rc == RNNDG_OK) return;
  const std::string msg = std::string(rnndg_last_error(h->ctx[i]));
  if (rc == RNNDG_EPARAM) throw ParamError(msg);
  if (rc == RNNDG_EDATA) throw DataError(msg);
  throw CudaError("shard " + std::to_string(i) + ": " + msg);
}

template <class T>
T* grow(int dev, T* p, uint64_t& cap, uint64_t want) {
  if (want <= cap && p) return p;
  RNNDG_CUDA(cudaSetDevice(dev));
  if (p) RNNDG_CUDA(cudaFree(p));
  cap = want < 16 ? 16 : want + want / 8;
  T* q = nullptr;
  RNNDG_CUDA(cudaMalloc(&q, cap * sizeof(T)));
  return q;
}

// fn(s) for every shard, one host thread per shard (the calls block on their
// device; the devices then work concurrently).  The first failure is rethrown.
template <class Fn>
void par_shards(rnndg_sharded* h, Fn fn) {
  const size_t P = h->ctx.size();
  if (P == 1) {
    fn(size_t(0));
    return;
  }
  std::vector<std::exception_ptr> errs(P);
  std::vector<std::thread> th;
  th.reserve(P);
  for (size_t s = 0; s < P; ++s)
    th.emplace_back([&, s] {
      try {
        fn(s);
      } catch (...) {
        errs[s] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

bool copy_exchange() {
  const char* e = std::getenv("RNNDG_MULTI_EXCHANGE");
  return e && std::strcmp(e, "copy") == 0;
}

void import_all(rnndg_sharded* h, int kind, uint32_t R, const std::vector<uint64_t>& tot,
                std::vector<rnndg_counts>* partial) {
  par_shards(h, [&](size_t r) {
    rnndg_counts pc{};
    uint64_t ns = 0;
    chk(h, r, rnndg_shard_import(h->ctx[r], kind, tot[r] ? h->rdst[r] : nullptr,
                                 tot[r] ? h->rkey[r] : nullptr, tot[r], R, &pc, &ns));
    h->nstaged[r] = ns;
    if (partial) (*partial)[r] = pc;
  });
}

// every shard's staged records to their owners; then `kind` applied on each
// receiving shard.  `partial[r]` gets shard r's import counts.
void exchange(rnndg_sharded* h, int kind, uint32_t R, std::vector<rnndg_counts>* partial) {
  const size_t P = h->ctx.size();
  std::vector<std::vector<uint64_t>> counts(P, std::vector<uint64_t>(P, 0));
  std::vector<uint64_t> tot(P, 0);
  if (!copy_exchange()) {
    // fused: count per owner, lay out the receive buffers, store into them
    par_shards(h, [&](size_t s) {
      chk(h, s, rnndg_shard_route(h->ctx[s], h->bounds.data(), uint32_t(P), counts[s].data()));
    });
    for (size_t r = 0; r < P; ++r) {
      for (size_t s = 0; s < P; ++s) tot[r] += counts[s][r];
      h->rdst[r] = grow(h->devs[r], h->rdst[r], h->rcap_d[r], tot[r]);
      h->rkey[r] = grow(h->devs[r], h->rkey[r], h->rcap_k[r], tot[r]);
    }
    par_shards(h, [&](size_t s) {
      std::vector<uint64_t> at(P, 0);  // shard s's segment in owner r's buffer
      for (size_t r = 0; r < P; ++r)
        for (size_t q = 0; q < s; ++q) at[r] += counts[q][r];
      chk(h, s, rnndg_shard_push(h->ctx[s], h->bounds.data(), uint32_t(P), h->rdst.data(),
                                 h->rkey.data(), at.data()));
    });
    import_all(h, kind, R, tot, partial);
    return;
  }
  par_shards(h, [&](size_t s) {
    h->sdst[s] = grow(h->devs[s], h->sdst[s], h->scap_d[s], h->nstaged[s]);
    h->skey[s] = grow(h->devs[s], h->skey[s], h->scap_k[s], h->nstaged[s]);
    chk(h, s, rnndg_shard_export(h->ctx[s], h->bounds.data(), uint32_t(P), h->sdst[s], h->skey[s],
                                 counts[s].data()));
  });
  for (size_t r = 0; r < P; ++r) {
    for (size_t s = 0; s < P; ++s) tot[r] += counts[s][r];
    h->rdst[r] = grow(h->devs[r], h->rdst[r], h->rcap_d[r], tot[r]);
    h->rkey[r] = grow(h->devs[r], h->rkey[r], h->rcap_k[r], tot[r]);
    RNNDG_CUDA(cudaSetDevice(h->devs[r]));
    uint64_t at = 0;
    for (size_t s = 0; s < P; ++s) {
      uint64_t lo = 0;
      for (size_t q = 0; q < r; ++q) lo += counts[s][q];
      const uint64_t m = counts[s][r];
      if (!m) continue;
      RNNDG_CUDA(cudaMemcpyPeerAsync(h->rdst[r] + at, h->devs[r], h->sdst[s] + lo, h->devs[s],
                                     m * sizeof(uint32_t), h->copy[r]));
      RNNDG_CUDA(cudaMemcpyPeerAsync(h->rkey[r] + at, h->devs[r], h->skey[s] + lo, h->devs[s],
                                     m * sizeof(uint64_t), h->copy[r]));
      at += m;
    }
  }
  // the shards' library streams read the records next
  for (size_t r = 0; r < P; ++r) {
    RNNDG_CUDA(cudaSetDevice(h->devs[r]));
    RNNDG_CUDA(cudaStreamSynchronize(h->copy[r]));
  }
  import_all(h, kind, R, tot, partial);
}

void in_prune(rnndg_sharded* h, uint32_t R) {
  par_shards(h, [&](size_t s) {
    chk(h, s, rnndg_shard_stage(h->ctx[s], RNNDG_X_INEDGE, &h->nstaged[s]));
  });
  exchange(h, RNNDG_X_INEDGE, R, nullptr);  // stages the deletions
  exchange(h, RNNDG_X_DELETE, R, nullptr);
}

}  // namespace

extern "C" {

int rnndg_sharded_create(rnndg_sharded** out, const int* devs, int nshards) {
  if (!out || !devs || nshards < 1) return RNNDG_EPARAM;
  auto* h = new rnndg_sharded();
  *out = h;
  return sguard(h, [&] {
    int ndev = 0;
    RNNDG_CUDA(cudaGetDeviceCount(&ndev));
    for (int i = 0; i < nshards; ++i)
      if (devs[i] < 0 || devs[i] >= ndev) throw ParamError("sharded_create: no such device");
    h->devs.assign(devs, devs + nshards);
    for (int i = 0; i < nshards; ++i) {
      rnndg_ctx* c = nullptr;
      if (rnndg_create(&c, devs[i]) != RNNDG_OK) throw CudaError("sharded_create: context");
      h->ctx.push_back(c);
      cudaStream_t st;
      RNNDG_CUDA(cudaSetDevice(devs[i]));
      RNNDG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      h->copy.push_back(st);
    }
    // NVLink / NVSwitch peer access between distinct devices
    for (int a = 0; a < nshards; ++a)
      for (int b = 0; b < nshards; ++b) {
        if (devs[a] == devs[b]) continue;
        int can = 0;
        RNNDG_CUDA(cudaDeviceCanAccessPeer(&can, devs[a], devs[b]));
        if (can) {
          RNNDG_CUDA(cudaSetDevice(devs[a]));
          const cudaError_t e = cudaDeviceEnablePeerAccess(devs[b], 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) RNNDG_CUDA(e);
          (void)cudaGetLastError();
        }
      }
    const size_t P = size_t(nshards);
    h->sdst.assign(P, nullptr);
    h->rdst.assign(P, nullptr);
    h->skey.assign(P, nullptr);
    h->rkey.assign(P, nullptr);
    h->scap_d.assign(P, 0);
    h->scap_k.assign(P, 0);
    h->rcap_d.assign(P, 0);
    h->rcap_k.assign(P, 0);
    h->nstaged.assign(P, 0);
  });
}

int rnndg_sharded_destroy(rnndg_sharded* h) {
  if (!h) return RNNDG_EPARAM;
  for (size_t i = 0; i < h->ctx.size(); ++i) {
    cudaSetDevice(h->devs[i]);
    if (h->sdst[i]) cudaFree(h->sdst[i]);
    if (h->skey[i]) cudaFree(h->skey[i]);
    if (h->rdst[i]) cudaFree(h->rdst[i]);
    if (h->rkey[i]) cudaFree(h->rkey[i]);
    cudaStreamDestroy(h->copy[i]);
    rnndg_destroy(h->ctx[i]);
  }
  delete h;
  return RNNDG_OK;
}

const char* rnndg_sharded_last_error(const rnndg_sharded* h) {
  return h ? h->err.c_str() : "null handle";
}

int rnndg_sharded_set_data(rnndg_sharded* h, const float* rows, uint64_t n, uint32_t d) {
  return sguard(h, [&] {
    const size_t P = h->ctx.size();
    if (n < P) throw ParamError("sharded_set_data: fewer vectors than shards");
    h->bounds.resize(P + 1);
    for (size_t r = 0; r <= P; ++r) h->bounds[r] = (n * r) / P;  // sharded.py ownership_bounds
    par_shards(h, [&](size_t s) {
      chk(h, s, rnndg_set_data(h->ctx[s], rows, n, d));
      chk(h, s, rnndg_set_partition(h->ctx[s], h->bounds[s], h->bounds[s + 1]));
    });
    h->n = n;
  });
}

int rnndg_sharded_build(rnndg_sharded* h, uint32_t S, uint32_t R, uint32_t T1, uint32_t T2,
                        uint64_t seed, int order, rnndg_build_stats* stats) {
  return sguard(h, [&] {
    const size_t P = h->ctx.size();
    if (h->n == 0) throw ParamError("no vector data: call rnndg_sharded_set_data first");
    // builder.cpp:255-258
    if (h->n < 2) throw ParamError("build: need at least 2 vectors");
    if (S < 1 || S > h->n - 1) throw ParamError("build: S out of [1, n-1]");
    if (R < 1) throw ParamError("build: R must be >= 1");
    if (T1 < 1 || T2 < 1) throw ParamError("build: T1 and T2 must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    rnndg_build_stats st{};
    h->pass_counts.clear();
    par_shards(h, [&](size_t s) { chk(h, s, rnndg_random_init(h->ctx[s], S, seed)); });
    for (uint32_t t1 = 1; t1 <= T1; ++t1) {
      for (uint32_t t2 = 0; t2 < T2; ++t2) {
        rnndg_counts pc{};
        std::vector<rnndg_counts> sc(P);
        par_shards(h, [&](size_t s) {
          chk(h, s, rnndg_shard_scan(h->ctx[s], &sc[s], &h->nstaged[s]));
        });
        for (const auto& c : sc) {
          pc.removed += c.removed;
          pc.flag_skips += c.flag_skips;
          pc.pair_checks += c.pair_checks;
        }
        std::vector<rnndg_counts> imp(P);
        exchange(h, RNNDG_X_PENDING, 0, &imp);
        for (const auto& c : imp) pc.inserted += c.inserted;
        h->pass_counts.push_back(pc);
        st.edits.removed += pc.removed;
        st.edits.inserted += pc.inserted;
        st.edits.flag_skips += pc.flag_skips;
        st.edits.pair_checks += pc.pair_checks;
        ++st.update_passes;
      }
      if (t1 != T1) {
        par_shards(h, [&](size_t s) {
          chk(h, s, rnndg_shard_stage(h->ctx[s], RNNDG_X_PROPOSAL, &h->nstaged[s]));
        });
        exchange(h, RNNDG_X_PROPOSAL, 0, nullptr);
        if (order == RNNDG_OUT_THEN_IN) {
          par_shards(h, [&](size_t s) { chk(h, s, rnndg_shard_out_prune(h->ctx[s], R)); });
          in_prune(h, R);
        } else {
          in_prune(h, R);
          par_shards(h, [&](size_t s) { chk(h, s, rnndg_shard_out_prune(h->ctx[s], R)); });
        }
        ++st.reverse_phases;
      }
    }
    for (size_t s = 0; s < P; ++s) {  // (lists leave sorted through rnndg_get_graph)
      RNNDG_CUDA(cudaSetDevice(h->devs[s]));
      RNNDG_CUDA(cudaDeviceSynchronize());
    }
    st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (size_t s = 0; s < P; ++s) st.kernel_launches += rnndg_kernel_launches(h->ctx[s]);
    if (stats) *stats = st;
  });
}

int rnndg_sharded_pass_counts(rnndg_sharded* h, rnndg_counts* out, uint32_t cap,
                              uint32_t* npasses) {
  return sguard(h, [&] {
    if (npasses) *npasses = uint32_t(h->pass_counts.size());
    for (uint32_t i = 0; out && i < cap && i < h->pass_counts.size(); ++i) out[i] = h->pass_counts[i];
  });
}

int rnndg_sharded_graph_size(rnndg_sharded* h, uint64_t* n, uint64_t* edges) {
  return sguard(h, [&] {
    uint64_t m = 0;
    for (size_t s = 0; s < h->ctx.size(); ++s) {
      uint64_t ns = 0, ms = 0;
      chk(h, s, rnndg_graph_size(h->ctx[s], &ns, &ms));
      m += ms;
    }
    if (n) *n = h->n;
    if (edges) *edges = m;
  });
}

int rnndg_sharded_get_graph(rnndg_sharded* h, uint64_t* offsets, uint32_t* ids, float* dists,
                            uint8_t* fresh) {
  return sguard(h, [&] {
    if (!offsets) throw ParamError("sharded_get_graph: offsets required");
    uint64_t at = 0;
    offsets[0] = 0;
    for (size_t s = 0; s < h->ctx.size(); ++s) {
      uint64_t ns = 0, ms = 0;
      chk(h, s, rnndg_graph_size(h->ctx[s], &ns, &ms));
      std::vector<uint64_t> off(ns + 1);
      chk(h, s, rnndg_get_graph(h->ctx[s], off.data(), ids ? ids + at : nullptr,
                                dists ? dists + at : nullptr, fresh ? fresh + at : nullptr));
      const uint64_t v0 = h->bounds[s];
      for (uint64_t u = 0; u < ns; ++u) offsets[v0 + u + 1] = at + off[u + 1];
      at += ms;
    }
  });
}

}  // extern "C"
