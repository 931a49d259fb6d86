/*
 * rnndg.h -- C ABI of the B200-native RNN-Descent graph builder.
 *
 * The reference `rnnd` artifact exposes its hot path as free C++ functions in
 * namespace rnnd (no plugin registry, no FFI); each entry point below replaces
 * one of them and keeps its argument meaning, defaults and error behaviour:
 *
 *   rnndg_random_init   <- rnnd::random_init        graph.hpp:45, graph.cpp:47-63
 *   rnndg_update_pass   <- rnnd::update_neighbors   builder.hpp:69-70, builder.cpp:214-220
 *                          (always the deferred threads>1 variant, builder.cpp:88-139)
 *   rnndg_reverse       <- rnnd::add_reverse_edges  builder.hpp:77-78, builder.cpp:222-251
 *   rnndg_build         <- rnnd::build              builder.hpp:84-86, builder.cpp:253-289
 *   rnndg_search        <- rnnd::batch_search       search.hpp:45-50, search.cpp:105-132
 *                          (rnnd::search = nq == 1, search.hpp:37-38)
 *   rnndg_brute_force   <- rnnd::brute_force_gt     vector_store.hpp:52-53, dataset.cpp:175-205
 *   rnndg_rng_strategy  <- rnnd::rng_strategy       builder.hpp:55-56, builder.cpp:196-212
 *   rnndg_degree_stats  <- rnnd::degree_stats       graph.hpp:58, graph.cpp:76-100
 *   rnndg_index_bytes   <- rnnd::save_index bytes   graph.hpp:67-71, graph.cpp:102-126
 *   rnndg_l2_pairs      <- rnnd::l2_sq              metric.hpp:47-65 (batched)
 *
 * All paths are relative to /root/reference/proj.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Host pointers unless a name says _dev.
 *   - Return codes mirror the reference's exception classes (common.hpp:16-23,
 *     CLI mapping rnnd_cli.cpp:408-417): RNNDG_OK, RNNDG_EPARAM (ParamError),
 *     RNNDG_EDATA (DataError), RNNDG_EINTERNAL (CUDA / NCCL / internal).
 *     rnndg_last_error() returns the message of the last failure on a context.
 *   - One context per host thread; calls on one context are serialised.  The
 *     context owns its device buffers and stream.
 *   - Arithmetic is bit-exact with the reference: squared L2 with four
 *     interleaved fp32 lanes, ((s0+s1)+(s2+s3)), tail in order, no FMA
 *     (metric.hpp:15-24).  Every graph this library builds is therefore
 *     identical, entry for entry, to rnnd::build with threads > 1.
 */
#ifndef RNNDG_H
#define RNNDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RNNDG_OK 0
#define RNNDG_EPARAM 1
#define RNNDG_EDATA 2
#define RNNDG_EINTERNAL 3

/* PruneOrder, builder.hpp:13 */
#define RNNDG_OUT_THEN_IN 0
#define RNNDG_IN_THEN_OUT 1

/* EntryMode, search.hpp:13 */
#define RNNDG_ENTRY_RANDOM 0
#define RNNDG_ENTRY_FIXED 1

typedef struct rnndg_ctx rnndg_ctx;

/* EditCounts, builder.hpp:25-38 */
typedef struct {
  uint64_t removed;
  uint64_t inserted;
  uint64_t flag_skips;
  uint64_t pair_checks;
} rnndg_counts;

/* BuildStats, builder.hpp:40-45, plus device-side measurements */
typedef struct {
  double seconds;         /* random_init .. final sort, CUDA events */
  uint32_t update_passes;
  uint32_t reverse_phases;
  rnndg_counts edits;
  double scan_seconds;    /* distance stage (scan kernels) only */
  double sort_seconds;    /* per-vertex list sorts */
  double apply_seconds;   /* pending bucket + append-if-absent + CSR rebuild */
  double reverse_seconds; /* reverse phases incl. both prunes */
  uint64_t touched;       /* sum of touched list entries (SURVEY 8(d) T_p) */
  uint64_t active_entries;/* sum of |U| over active vertices (A_p) */
  uint64_t scan_launches; /* kernels launched by the build */
  uint64_t kernel_launches;
} rnndg_build_stats;

/* Called after each outer round (BuildProgressFn, builder.hpp:48-49). */
typedef void (*rnndg_progress_fn)(uint32_t t1, uint32_t T1,
                                  const rnndg_counts* outer, double elapsed_s,
                                  void* user);

/* ---- context ---- */
int rnndg_create(rnndg_ctx** out, int device);
int rnndg_destroy(rnndg_ctx* ctx);
const char* rnndg_last_error(const rnndg_ctx* ctx);
/* number of this library's kernels launched on the context so far */
uint64_t rnndg_kernel_launches(const rnndg_ctx* ctx);

/* ---- NN-Descent baseline (nndescent.hpp:12-52) ----
 * Canonical deferred join (see oracle/rnnd_oracle.c ro_nnd_pass): every pool
 * is snapshotted, all pairs joined, and each pool becomes the `cap` nearest
 * distinct entries of pool + proposals.  The reference's parallel join is
 * order-dependent (per-vertex locks); this form is deterministic.
 * Parameters and errors as NnDescentParams / NnDescent::NnDescent
 * (nndescent.cpp:11-22); cap = max(pool ? pool : 2K, K). */
int rnndg_nnd_init(rnndg_ctx* ctx, uint32_t K, uint32_t sample, uint32_t iters,
                   uint32_t pool, uint64_t seed);            /* NnDescent + init() */
int rnndg_nnd_pass(rnndg_ctx* ctx, uint64_t* new_entries);  /* join_pass() */
/* pools, dense n x stride: cnt[n], ids / dists / fresh [n * stride] (any
 * may be null); *cap_out = stride = max(cap, min(sample, n - 1)) -- init
 * fills min(sample, n-1) entries even above the cap, and such a pool keeps
 * its size (insert_candidate pops one entry per insertion) */
int rnndg_nnd_pools(rnndg_ctx* ctx, uint32_t* cap_out, uint32_t* cnt, uint32_t* ids,
                    float* dists, uint8_t* fresh);
int rnndg_nnd_finalize(rnndg_ctx* ctx);                       /* finalize() -> graph */
/* build_nndescent (nndescent.cpp:101-119): init, iters passes, finalize;
 * stats->seconds (CUDA events), update_passes = iters */
int rnndg_nnd_build(rnndg_ctx* ctx, uint32_t K, uint32_t sample, uint32_t iters,
                    uint32_t pool, uint64_t seed, rnndg_build_stats* stats);

/* ---- data (VectorStore, vector_store.hpp:12-20) ---- */
/* copies n x d row-major fp32 host rows to the device (H2D) */
int rnndg_set_data(rnndg_ctx* ctx, const float* rows, uint64_t n, uint32_t d);
/* borrows rows already resident on the context's device.  The library
   works on its own CUDA stream: the caller must have completed the work that
   produced the rows (e.g. synchronise its stream) before this call. */
int rnndg_set_data_device(rnndg_ctx* ctx, const float* rows_dev, uint64_t n,
                          uint32_t d);
/* replaces rnnd::load_fvecs (dataset.cpp:82-95) + rnndg_set_data: reads an
 * .fvecs file in chunks through pinned staging buffers, validates it with the
 * reference's checks and messages (parse_vecs, dataset.cpp:55-78; non-finite
 * values, :89) and streams it to the device with async H2D copies.  Errors
 * are RNNDG_EDATA with "<path>: <reason>". */
int rnndg_load_fvecs(rnndg_ctx* ctx, const char* path, uint64_t* n, uint32_t* d);

/* ---- hot path ---- */
int rnndg_random_init(rnndg_ctx* ctx, uint32_t S, uint64_t seed);
int rnndg_update_pass(rnndg_ctx* ctx, rnndg_counts* out);
int rnndg_reverse(rnndg_ctx* ctx, uint32_t R, int prune_order);
/* sort every list ascending (dist, id), builder.cpp:283-285 */
int rnndg_sort_lists(rnndg_ctx* ctx);
int rnndg_build(rnndg_ctx* ctx, uint32_t S, uint32_t R, uint32_t T1,
                uint32_t T2, uint64_t seed, int prune_order,
                rnndg_build_stats* stats, rnndg_progress_fn progress,
                void* user);
/* per-pass counters of the last build: T1*T2 entries */
int rnndg_pass_counts(const rnndg_ctx* ctx, rnndg_counts* out, uint32_t cap);

/* ---- graph state (AdjacencyGraph, graph.hpp:25-40) ---- */
int rnndg_graph_size(rnndg_ctx* ctx, uint64_t* n, uint64_t* edges);
/* CSR copy-out; any of ids/dists/fresh may be NULL.  offsets has n+1 slots. */
int rnndg_get_graph(rnndg_ctx* ctx, uint64_t* offsets, uint32_t* ids,
                    float* dists, uint8_t* fresh);
/* replace the graph (validated: ids < n, no self-loops, no duplicates) */
int rnndg_set_graph(rnndg_ctx* ctx, uint64_t n, const uint64_t* offsets,
                    const uint32_t* ids, const float* dists,
                    const uint8_t* fresh);
/* serialized RNND index; returns size through *size; writes when buf */
int rnndg_index_bytes(rnndg_ctx* ctx, uint8_t* buf, uint64_t* size);
/* graph.cpp:76-100: out = {edges, max_out, max_in} under cap (0 = none) */
int rnndg_degree_stats(rnndg_ctx* ctx, uint32_t cap, uint64_t out[3]);

/* ---- evaluation ---- */
/* Batched beam search, search.cpp:40-94 per query.  ids/dists are nq*k
 * (short results padded with UINT32_MAX / +inf); visited / dist_comps are
 * per query and may be NULL. */
int rnndg_search(rnndg_ctx* ctx, const float* queries, uint64_t nq,
                 uint32_t L, uint32_t K, uint32_t k, int entry_mode,
                 uint32_t entry_vertex, uint32_t entry_count, uint64_t seed,
                 uint32_t* ids, float* dists, uint64_t* visited,
                 uint64_t* dist_comps);
int rnndg_brute_force(rnndg_ctx* ctx, const float* queries, uint64_t nq,
                      uint32_t k, uint32_t* ids);
/* rng_strategy on one candidate list; returns the kept count via *nkept.
 * RNNDG_EPARAM when a candidate equals u (builder.cpp:201). */
int rnndg_rng_strategy(rnndg_ctx* ctx, uint32_t u, const uint32_t* cand_ids,
                       const float* cand_dists, uint32_t ncand,
                       uint32_t* kept_ids, float* kept_dists, uint32_t* nkept);
/* l2_sq(row(a[i]), row(b[i])) for i < npairs, exact contract */
int rnndg_l2_pairs(rnndg_ctx* ctx, const uint32_t* a, const uint32_t* b,
                   uint64_t npairs, float* out);

/* ---- sharded build ----
 * Vertex ownership by contiguous ranges; the store is replicated on every
 * rank.  One context owns vertices [v_begin, v_end).  A host-side driver
 * (paper_2310_20419_b200/sharded.py) runs the protocol and moves records
 * between owners with an all-to-all (NCCL, gloo or in-process):
 *   pass:     shard_scan -> export -> all-to-all -> import(PENDING)
 *   reverse:  stage(PROPOSAL) -> export -> all-to-all -> import(PROPOSAL);
 *             out_prune; stage(INEDGE) -> ... -> import(INEDGE, R) stages the
 *             deletions -> export -> ... -> import(DELETE)
 * A record is (dst: global vertex id, key: list entry for dst's list).
 * Every step is set-canonical, so the sharded graph equals the unsharded one
 * entry for entry. */
#define RNNDG_X_PENDING 0  /* redirect (w, v, d(v,w)) -> owner(w) */
#define RNNDG_X_PROPOSAL 1 /* reverse proposal (v, u, d) -> owner(v) */
#define RNNDG_X_INEDGE 2   /* in-edge (t, s, d) -> owner(t) */
#define RNNDG_X_DELETE 3   /* in_prune deletion (s, t, d) -> owner(s) */

int rnndg_set_partition(rnndg_ctx* ctx, uint64_t v_begin, uint64_t v_end);
/* mark + scan of the owned lists; `partial` gets removed / flag_skips /
 * pair_checks of this shard; the redirects are staged as records */
int rnndg_shard_scan(rnndg_ctx* ctx, rnndg_counts* partial, uint64_t* nrecords);
/* totals of this shard's scans since the last reset: distance-stage seconds
 * (CUDA events), touched entries T and active entries A, pass
 * count.  No reference counterpart (measurement only). */
int rnndg_shard_totals(rnndg_ctx* ctx, double* scan_seconds, uint64_t* touched,
                       uint64_t* active_entries, uint64_t* passes, int reset);
/* stage reverse proposals or in-edges of the owned lists */
int rnndg_shard_stage(rnndg_ctx* ctx, int kind, uint64_t* nrecords);
/* staged records sorted by dst into DEVICE buffers (nrecords each) and the
 * number of records per destination part (bounds: parts+1 vertex ids) */
int rnndg_shard_export(rnndg_ctx* ctx, const uint64_t* bounds, uint32_t parts,
                       uint32_t* dst_dev, uint64_t* key_dev, uint64_t* counts);
/* Direct routing of the staged records (the fused exchange; the
 * pending push of builder.cpp:102-105 across shards): rnndg_shard_route
 * counts them per destination part (no sort); once the caller has laid out
 * every owner's receive buffer from all shards' counts, rnndg_shard_push
 * stores each record straight into its owner's DEVICE buffers
 * dst_ptrs[p] / key_ptrs[p] from the kernel, starting at offsets[p] (this
 * shard's segment; order inside it is unspecified, the import is a set
 * operation).  The buffers may live on another GPU with peer access enabled:
 * the stores then travel over NVLink.  Returns after the stores are
 * complete; at most 64 parts. */
int rnndg_shard_route(rnndg_ctx* ctx, const uint64_t* bounds, uint32_t parts, uint64_t* counts);
int rnndg_shard_push(rnndg_ctx* ctx, const uint64_t* bounds, uint32_t parts,
                     uint32_t* const* dst_ptrs, uint64_t* const* key_ptrs,
                     const uint64_t* offsets);
/* apply received records (DEVICE buffers); INEDGE stages deletions and
 * returns their number in *nstaged; PENDING reports `inserted`.  The records
 * are read on the library's stream: the caller completes the transfer that
 * produced them (e.g. synchronises the stream of its collective) first. */
int rnndg_shard_import(rnndg_ctx* ctx, int kind, const uint32_t* dst_dev,
                       const uint64_t* key_dev, uint64_t nrecords, uint32_t R,
                       rnndg_counts* partial, uint64_t* nstaged);
int rnndg_shard_out_prune(rnndg_ctx* ctx, uint32_t R);

/* ---- vertex-sharded build in one process (builder.cpp:253-289 over
 * shards; csrc/multi.cu) ----
 * Shard i runs on CUDA device devs[i] (repeats allowed: several shards may
 * share a GPU) and owns a contiguous vertex range; records move between
 * shards by peer copies (NVLink / NVSwitch between B200s).  The graph and
 * every pass count equal rnndg_build's. */
typedef struct rnndg_sharded rnndg_sharded;
int rnndg_sharded_create(rnndg_sharded** out, const int* devs, int nshards);
int rnndg_sharded_destroy(rnndg_sharded* h);
const char* rnndg_sharded_last_error(const rnndg_sharded* h);
int rnndg_sharded_set_data(rnndg_sharded* h, const float* rows, uint64_t n, uint32_t d);
/* fills seconds, update_passes, reverse_phases, edits, kernel_launches */
int rnndg_sharded_build(rnndg_sharded* h, uint32_t S, uint32_t R, uint32_t T1, uint32_t T2,
                        uint64_t seed, int order, rnndg_build_stats* stats);
int rnndg_sharded_pass_counts(rnndg_sharded* h, rnndg_counts* out, uint32_t cap,
                              uint32_t* npasses);
int rnndg_sharded_graph_size(rnndg_sharded* h, uint64_t* n, uint64_t* edges);
/* the whole graph, lists in vertex order (CSR; any of ids/dists/fresh may be NULL) */
int rnndg_sharded_get_graph(rnndg_sharded* h, uint64_t* offsets, uint32_t* ids, float* dists,
                            uint8_t* fresh);

#ifdef __cplusplus
}
#endif
#endif /* RNNDG_H */
