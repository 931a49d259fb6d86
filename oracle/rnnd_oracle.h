/*
 * rnnd_oracle.h -- CPU ORACLE for the RNN-Descent hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * `rnnd` artifact (/root/reference/proj) used as the checker for the CUDA
 * product.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product library never links it.
 *
 * Parity pin: tests/test_oracle_*.py check this file against every golden
 * value in the reference's own unit tests (test_metric.cpp, test_builder.cpp,
 * test_graph.cpp, test_search.cpp, test_dataset.cpp, test_eval.cpp) and, when
 * oracle/_ref was built from the reference sources, byte-for-byte against
 * rnnd::build(threads>=2) itself (tests/golden/ holds fixtures made that way).
 */
#ifndef RNND_ORACLE_H
#define RNND_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ro_graph ro_graph;

/* ---- primitives (rng.hpp:13-72, metric.hpp:26-45) ---- */
uint64_t ro_splitmix_next(uint64_t* state);
uint64_t ro_splitmix_bounded(uint64_t* state, uint64_t bound);
float ro_splitmix_unit_float(uint64_t* state);
uint64_t ro_mix_seed(uint64_t seed, uint64_t stream);
/* writes `count` ids; exclude >= n means no exclusion */
void ro_sample_distinct(uint64_t* state, uint32_t n, uint32_t count,
                        uint32_t exclude, uint32_t* out);
float ro_l2_sq(const float* a, const float* b, size_t d);
void ro_synth_uniform(uint64_t n, uint64_t d, uint64_t seed, float* out);
uint32_t ro_crc32(const uint8_t* data, size_t size);

/* ---- graph state ---- */
ro_graph* ro_graph_new(uint64_t n);
void ro_graph_free(ro_graph* g);
uint64_t ro_graph_n(const ro_graph* g);
uint64_t ro_graph_edges(const ro_graph* g);
/* CSR export in stored list order; any output pointer may be NULL */
void ro_graph_export(const ro_graph* g, uint64_t* offsets, uint32_t* ids,
                     float* dists, uint8_t* fresh);
/* replaces all lists */
void ro_graph_import(ro_graph* g, const uint64_t* offsets, const uint32_t* ids,
                     const float* dists, const uint8_t* fresh);
/* sort every list ascending (dist, id) -- builder.cpp:283-285 */
void ro_graph_sort_lists(ro_graph* g);

/* ---- algorithms (builder.cpp, graph.cpp) ---- */
/* return 0 ok, 1 param error */
int ro_random_init(ro_graph* g, const float* data, uint32_t d, uint32_t S,
                   uint64_t seed);
/* counts[4] = removed, inserted, flag_skips, pair_checks.  Deferred
 * (threads > 1) variant, builder.cpp:88-139. */
void ro_update_pass(ro_graph* g, const float* data, uint32_t d,
                    uint64_t counts[4]);
/* builder.cpp:71-86, threads == 1 variant (reported only) */
void ro_update_pass_serial(ro_graph* g, const float* data, uint32_t d,
                           uint64_t counts[4]);
/* order 0 = out-then-in, 1 = in-then-out.  builder.cpp:222-251 */
int ro_add_reverse_edges(ro_graph* g, uint32_t R, int order);
/* full build, builder.cpp:253-289.  pass_counts (may be NULL) receives
 * T1*T2*4 u64 (per-pass counts).  serial != 0 uses the threads==1 variant. */
int ro_build(ro_graph* g, const float* data, uint32_t d, uint32_t S, uint32_t R,
             uint32_t T1, uint32_t T2, uint64_t seed, int order, int serial,
             uint64_t* pass_counts);
/* builder.cpp:196-212; returns kept count, -1 if a candidate equals u */
int ro_rng_strategy(const float* data, uint32_t d, uint32_t u,
                    const uint32_t* cand_ids, const float* cand_dists,
                    uint32_t ncand, uint32_t* kept_ids, float* kept_dists);

/* ---- evaluation (search.cpp, dataset.cpp, eval.cpp, graph.cpp) ---- */
/* entry_mode 0 = random sample, 1 = fixed vertex.  returns #results or -1 */
int ro_search(const ro_graph* g, const float* data, uint32_t d,
              const float* query, uint32_t L, uint32_t K, uint32_t k,
              int entry_mode, uint32_t entry_vertex, uint32_t entry_count,
              uint64_t seed, int has_distances, uint32_t* ids, float* dists,
              uint64_t* visited, uint64_t* dist_comps);
void ro_brute_force(const float* base, uint64_t n, uint32_t d,
                    const float* queries, uint64_t nq, uint32_t k,
                    uint32_t* ids_out);
/* degree stats (graph.cpp:76-100); out[0]=edges out[1]=max_out out[2]=max_in */
void ro_degree_stats(const ro_graph* g, uint32_t cap, int has_distances,
                     uint64_t out[3]);
/* serialised index (graph.cpp:102-126); returns byte size, writes if buf */
uint64_t ro_index_bytes(const ro_graph* g, uint8_t* buf);

/* NN-Descent baseline (nndescent.cpp), canonical deferred join.  Pools are
 * held as the lists of an ro_graph.  init validates like the constructor
 * (nndescent.cpp:11-22; returns 1 on a parameter error) and fills the pools
 * (:24-37); pass runs one deferred join (see rnnd_oracle.c) and returns the
 * number of new pool entries; finalize keeps the K nearest (:88-99). */
int ro_nnd_init(ro_graph* pools, const float* data, uint32_t d, uint32_t K,
                uint32_t sample, uint32_t iters, uint32_t pool, uint64_t seed);
uint64_t ro_nnd_pass(ro_graph* pools, const float* data, uint32_t d, uint32_t sample,
                     uint32_t cap);
void ro_nnd_finalize(const ro_graph* pools, uint32_t K, ro_graph* out);

#ifdef __cplusplus
}
#endif
#endif
