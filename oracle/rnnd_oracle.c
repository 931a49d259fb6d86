/*
 * rnnd_oracle.c -- CPU ORACLE (test infrastructure, not product).
 *
 * Plain-C restatement of the reference rnnd artifact's RNN-Descent path.
 * Every function cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Compiled with -ffp-contract=off like the reference
 * (CMakeLists.txt:16-17) so float32 arithmetic is exactly as written.
 * See rnnd_oracle.h for who may use this file.
 */
#include "rnnd_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */

/* SplitMix64::next, rng.hpp:19-24 */
uint64_t ro_splitmix_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* SplitMix64::bounded, rng.hpp:26-28 (128-bit multiply-shift) */
uint64_t ro_splitmix_bounded(uint64_t* s, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)ro_splitmix_next(s) * bound) >> 64);
}

/* SplitMix64::unit_float, rng.hpp:31 */
float ro_splitmix_unit_float(uint64_t* s) {
  return (float)(ro_splitmix_next(s) >> 40) * (1.0f / 16777216.0f);
}

/* mix_seed, rng.hpp:39-42 */
uint64_t ro_mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t st = seed ^ (0xD1B54A32D192ED03ULL * (stream + 1));
  return ro_splitmix_next(&st);
}

/* sample_distinct, rng.hpp:46-72.  Both reference branches (linear find for
 * count <= 64, hash set above) implement the same Floyd rule: draw
 * t = bounded(j+1), emit j if t was already emitted, else t. */
void ro_sample_distinct(uint64_t* s, uint32_t n, uint32_t count,
                        uint32_t exclude, uint32_t* out) {
  const uint32_t domain = exclude < n ? n - 1 : n;
  uint32_t m = 0;
  uint8_t* seen = NULL;
  if (count > 64) seen = (uint8_t*)calloc(domain ? domain : 1, 1);
  for (uint32_t j = domain - count; j < domain; ++j) {
    uint32_t t = (uint32_t)ro_splitmix_bounded(s, (uint64_t)j + 1);
    int hit = 0;
    if (seen) {
      hit = seen[t];
    } else {
      for (uint32_t q = 0; q < m; ++q)
        if (out[q] == t) { hit = 1; break; }
    }
    uint32_t v = hit ? j : t;
    if (seen) seen[v] = 1;
    out[m++] = v;
  }
  free(seen);
  if (exclude < n)
    for (uint32_t q = 0; q < m; ++q)
      if (out[q] >= exclude) ++out[q];
}

/* --------------------------------------------------------------- metric */

/* l2_sq_scalar, metric.hpp:26-45: four interleaved lanes, combined
 * ((s0+s1)+(s2+s3)), then the tail left to right, no FMA. */
float ro_l2_sq(const float* a, const float* b, size_t d) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  size_t i = 0;
  for (; i + 4 <= d; i += 4) {
    float d0 = a[i] - b[i];
    float d1 = a[i + 1] - b[i + 1];
    float d2 = a[i + 2] - b[i + 2];
    float d3 = a[i + 3] - b[i + 3];
    s0 += d0 * d0;
    s1 += d1 * d1;
    s2 += d2 * d2;
    s3 += d3 * d3;
  }
  float sum = (s0 + s1) + (s2 + s3);
  for (; i < d; ++i) {
    float t = a[i] - b[i];
    sum += t * t;
  }
  return sum;
}

/* synth_uniform, dataset.cpp:134-143 */
void ro_synth_uniform(uint64_t n, uint64_t d, uint64_t seed, float* out) {
  uint64_t s = seed;
  for (uint64_t i = 0; i < n * d; ++i) out[i] = ro_splitmix_unit_float(&s);
}

/* zlib crc32 (IEEE 802.3, reflected 0xEDB88320) as used at graph.cpp:41-43 */
uint32_t ro_crc32(const uint8_t* p, size_t size) {
  static uint32_t table[256];
  static int init = 0;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = 1;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < size; ++i) c = table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

/* ---------------------------------------------------------------- graph */

/* NeighborEntry, graph.hpp:14-18 */
typedef struct {
  uint32_t id;
  float dist;
  uint8_t fresh;
} entry_t;

typedef struct {
  entry_t* e;
  uint32_t size, cap;
} list_t;

struct ro_graph {
  uint64_t n;
  list_t* adj; /* AdjacencyGraph::adj, graph.hpp:25-40 */
};

static void list_push(list_t* l, entry_t x) {
  if (l->size == l->cap) {
    l->cap = l->cap ? l->cap * 2 : 8;
    l->e = (entry_t*)realloc(l->e, sizeof(entry_t) * l->cap);
  }
  l->e[l->size++] = x;
}

/* nearer, graph.hpp:21-23 */
static int nearer(const entry_t* a, const entry_t* b) {
  return a->dist != b->dist ? a->dist < b->dist : a->id < b->id;
}

static int cmp_nearer(const void* x, const void* y) {
  const entry_t *a = (const entry_t*)x, *b = (const entry_t*)y;
  if (nearer(a, b)) return -1;
  if (nearer(b, a)) return 1;
  return 0;
}

ro_graph* ro_graph_new(uint64_t n) {
  ro_graph* g = (ro_graph*)calloc(1, sizeof(ro_graph));
  g->n = n;
  g->adj = (list_t*)calloc(n ? n : 1, sizeof(list_t));
  return g;
}

void ro_graph_free(ro_graph* g) {
  if (!g) return;
  for (uint64_t u = 0; u < g->n; ++u) free(g->adj[u].e);
  free(g->adj);
  free(g);
}

uint64_t ro_graph_n(const ro_graph* g) { return g->n; }

uint64_t ro_graph_edges(const ro_graph* g) {
  uint64_t m = 0;
  for (uint64_t u = 0; u < g->n; ++u) m += g->adj[u].size;
  return m;
}

void ro_graph_export(const ro_graph* g, uint64_t* offsets, uint32_t* ids,
                     float* dists, uint8_t* fresh) {
  uint64_t off = 0;
  for (uint64_t u = 0; u < g->n; ++u) {
    if (offsets) offsets[u] = off;
    const list_t* l = &g->adj[u];
    for (uint32_t j = 0; j < l->size; ++j, ++off) {
      if (ids) ids[off] = l->e[j].id;
      if (dists) dists[off] = l->e[j].dist;
      if (fresh) fresh[off] = l->e[j].fresh;
    }
  }
  if (offsets) offsets[g->n] = off;
}

void ro_graph_import(ro_graph* g, const uint64_t* offsets, const uint32_t* ids,
                     const float* dists, const uint8_t* fresh) {
  for (uint64_t u = 0; u < g->n; ++u) {
    list_t* l = &g->adj[u];
    l->size = 0;
    for (uint64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
      entry_t x = {ids[j], dists ? dists[j] : 0.0f,
                   (uint8_t)(fresh ? fresh[j] : 0)};
      list_push(l, x);
    }
  }
}

void ro_graph_sort_lists(ro_graph* g) {
  for (uint64_t u = 0; u < g->n; ++u)
    if (g->adj[u].size > 1)
      qsort(g->adj[u].e, g->adj[u].size, sizeof(entry_t), cmp_nearer);
}

/* random_init, graph.cpp:47-63: stream SplitMix64(mix_seed(seed, u)),
 * S distinct ids != u, dist = l2_sq(row(u), row(id)), fresh. */
int ro_random_init(ro_graph* g, const float* data, uint32_t d, uint32_t S,
                   uint64_t seed) {
  const uint64_t n = g->n;
  if (n < 2) return 1;
  if (S < 1 || S > n - 1) return 1;
  uint32_t* ids = (uint32_t*)malloc(sizeof(uint32_t) * S);
  for (uint64_t u = 0; u < n; ++u) {
    uint64_t st = ro_mix_seed(seed, u);
    ro_sample_distinct(&st, (uint32_t)n, S, (uint32_t)u, ids);
    list_t* l = &g->adj[u];
    l->size = 0;
    for (uint32_t j = 0; j < S; ++j) {
      entry_t x = {ids[j], ro_l2_sq(data + u * d, data + (uint64_t)ids[j] * d, d),
                   1};
      list_push(l, x);
    }
  }
  free(ids);
  return 0;
}

/* ------------------------------------------------------------- builder */

/* PendingEdge, builder.cpp:12-16 */
typedef struct {
  uint32_t src, dst;
  float dist;
} pending_t;

typedef struct {
  pending_t* p;
  uint64_t size, cap;
} pvec_t;

static void pvec_push(pvec_t* v, pending_t x) {
  if (v->size == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 1024;
    v->p = (pending_t*)realloc(v->p, sizeof(pending_t) * v->cap);
  }
  v->p[v->size++] = x;
}

/* pending_less, builder.cpp:18-20 */
static int cmp_pending(const void* x, const void* y) {
  const pending_t *a = (const pending_t*)x, *b = (const pending_t*)y;
  if (a->src != b->src) return a->src < b->src ? -1 : 1;
  if (a->dst != b->dst) return a->dst < b->dst ? -1 : 1;
  return 0;
}

/* has_target, builder.cpp:22-26 */
static int has_target(const list_t* l, uint32_t id) {
  for (uint32_t j = 0; j < l->size; ++j)
    if (l->e[j].id == id) return 1;
  return 0;
}

/* scan_vertex, builder.cpp:41-69.  Sorts cand by nearer, walks the kept list
 * in order for every candidate: old/old pairs are skipped (flag_skips),
 * otherwise a distance is computed (pair_checks) and the first kept w with
 * v.dist >= d(v,w) removes v and redirects it to (w, v, d(v,w)).  Survivors
 * are flagged old.  Result replaces cand (in place, kept prefix). */
static uint32_t scan_vertex(entry_t* cand, uint32_t U, const float* data,
                            uint32_t d, uint64_t counts[4], pvec_t* pend) {
  if (U > 1) qsort(cand, U, sizeof(entry_t), cmp_nearer);
  uint32_t nk = 0; /* kept = cand[0..nk) (in-place compaction is safe) */
  for (uint32_t i = 0; i < U; ++i) {
    entry_t v = cand[i];
    int keep = 1;
    for (uint32_t k = 0; k < nk; ++k) {
      const entry_t* w = &cand[k];
      if (!v.fresh && !w->fresh) {
        ++counts[2];
        continue;
      }
      ++counts[3];
      float dvw = ro_l2_sq(data + (uint64_t)v.id * d, data + (uint64_t)w->id * d, d);
      if (v.dist >= dvw) {
        keep = 0;
        ++counts[0];
        pending_t p = {w->id, v.id, dvw};
        pvec_push(pend, p);
        break;
      }
    }
    if (keep) cand[nk++] = v;
  }
  for (uint32_t k = 0; k < nk; ++k) cand[k].fresh = 0;
  return nk;
}

/* update_parallel, builder.cpp:88-139: scan every vertex against the pre-pass
 * state, then sort pending by (src, dst), drop duplicates, and append each
 * (dst, dist, fresh) to src's post-scan list unless already present. */
void ro_update_pass(ro_graph* g, const float* data, uint32_t d,
                    uint64_t counts[4]) {
  memset(counts, 0, sizeof(uint64_t) * 4);
  pvec_t pend = {0};
  for (uint64_t u = 0; u < g->n; ++u) {
    list_t* l = &g->adj[u];
    l->size = scan_vertex(l->e, l->size, data, d, counts, &pend);
  }
  if (pend.size) qsort(pend.p, pend.size, sizeof(pending_t), cmp_pending);
  uint64_t w = 0;
  for (uint64_t i = 0; i < pend.size; ++i)
    if (w == 0 || pend.p[i].src != pend.p[w - 1].src ||
        pend.p[i].dst != pend.p[w - 1].dst)
      pend.p[w++] = pend.p[i];
  for (uint64_t i = 0; i < w; ++i) {
    list_t* l = &g->adj[pend.p[i].src];
    if (!has_target(l, pend.p[i].dst)) {
      entry_t x = {pend.p[i].dst, pend.p[i].dist, 1};
      list_push(l, x);
      ++counts[1];
    }
  }
  free(pend.p);
}

/* update_serial, builder.cpp:71-86: redirects land mid-pass. */
void ro_update_pass_serial(ro_graph* g, const float* data, uint32_t d,
                           uint64_t counts[4]) {
  memset(counts, 0, sizeof(uint64_t) * 4);
  pvec_t pend = {0};
  for (uint64_t u = 0; u < g->n; ++u) {
    list_t* l = &g->adj[u];
    pend.size = 0;
    l->size = scan_vertex(l->e, l->size, data, d, counts, &pend);
    for (uint64_t i = 0; i < pend.size; ++i) {
      list_t* wl = &g->adj[pend.p[i].src];
      if (!has_target(wl, pend.p[i].dst)) {
        entry_t x = {pend.p[i].dst, pend.p[i].dist, 1};
        list_push(wl, x);
        ++counts[1];
      }
    }
  }
  free(pend.p);
}

/* out_prune, builder.cpp:141-150: lists longer than R keep their R nearest */
static void out_prune(ro_graph* g, uint32_t R) {
  for (uint64_t u = 0; u < g->n; ++u) {
    list_t* l = &g->adj[u];
    if (l->size > R) {
      qsort(l->e, l->size, sizeof(entry_t), cmp_nearer);
      l->size = R;
    }
  }
}

typedef struct {
  uint32_t target, source;
  float dist;
} inedge_t;

/* in_prune ordering, builder.cpp:162-166: (target, dist, source) */
static int cmp_inedge(const void* x, const void* y) {
  const inedge_t *a = (const inedge_t*)x, *b = (const inedge_t*)y;
  if (a->target != b->target) return a->target < b->target ? -1 : 1;
  if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
  if (a->source != b->source) return a->source < b->source ? -1 : 1;
  return 0;
}

static int cmp_u32(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return a < b ? -1 : (a > b);
}

/* in_prune, builder.cpp:152-192: every in-edge past a target's R nearest
 * (dist, then source) is deleted from its source list. */
static void in_prune(ro_graph* g, uint32_t R) {
  uint64_t m = ro_graph_edges(g);
  inedge_t* ins = (inedge_t*)malloc(sizeof(inedge_t) * (m ? m : 1));
  uint64_t k = 0;
  for (uint64_t u = 0; u < g->n; ++u)
    for (uint32_t j = 0; j < g->adj[u].size; ++j) {
      inedge_t x = {g->adj[u].e[j].id, (uint32_t)u, g->adj[u].e[j].dist};
      ins[k++] = x;
    }
  if (m) qsort(ins, m, sizeof(inedge_t), cmp_inedge);
  pvec_t del = {0};
  uint64_t i = 0;
  while (i < m) {
    uint64_t j = i + 1;
    while (j < m && ins[j].target == ins[i].target) ++j;
    for (uint64_t p = i + R; p < j; ++p) {
      pending_t x = {ins[p].source, ins[p].target, 0.0f};
      pvec_push(&del, x);
    }
    i = j;
  }
  free(ins);
  if (!del.size) return;
  qsort(del.p, del.size, sizeof(pending_t), cmp_pending);
  uint32_t* targets = (uint32_t*)malloc(sizeof(uint32_t) * del.size);
  i = 0;
  while (i < del.size) {
    uint64_t j = i + 1;
    while (j < del.size && del.p[j].src == del.p[i].src) ++j;
    uint64_t nt = 0;
    for (uint64_t p = i; p < j; ++p) targets[nt++] = del.p[p].dst;
    list_t* l = &g->adj[del.p[i].src];
    uint32_t w = 0;
    for (uint32_t q = 0; q < l->size; ++q)
      if (!bsearch(&l->e[q].id, targets, nt, sizeof(uint32_t), cmp_u32))
        l->e[w++] = l->e[q];
    l->size = w;
    i = j;
  }
  free(targets);
  free(del.p);
}

/* add_reverse_edges, builder.cpp:222-251 */
int ro_add_reverse_edges(ro_graph* g, uint32_t R, int order) {
  if (R < 1) return 1;
  uint64_t m = ro_graph_edges(g);
  pending_t* props = (pending_t*)malloc(sizeof(pending_t) * (m ? m : 1));
  uint64_t k = 0;
  for (uint64_t u = 0; u < g->n; ++u)
    for (uint32_t j = 0; j < g->adj[u].size; ++j) {
      pending_t x = {g->adj[u].e[j].id, (uint32_t)u, g->adj[u].e[j].dist};
      props[k++] = x;
    }
  if (m) qsort(props, m, sizeof(pending_t), cmp_pending);
  for (uint64_t i = 0; i < m; ++i) {
    list_t* l = &g->adj[props[i].src];
    if (!has_target(l, props[i].dst)) {
      entry_t x = {props[i].dst, props[i].dist, 1};
      list_push(l, x);
    }
  }
  free(props);
  if (order == 0) {
    out_prune(g, R);
    in_prune(g, R);
  } else {
    in_prune(g, R);
    out_prune(g, R);
  }
  return 0;
}

/* build, builder.cpp:253-289 */
int ro_build(ro_graph* g, const float* data, uint32_t d, uint32_t S, uint32_t R,
             uint32_t T1, uint32_t T2, uint64_t seed, int order, int serial,
             uint64_t* pass_counts) {
  const uint64_t n = g->n;
  if (n < 2) return 1;
  if (S < 1 || S > n - 1) return 1;
  if (R < 1) return 1;
  if (T1 < 1 || T2 < 1) return 1;
  int rc = ro_random_init(g, data, d, S, seed);
  if (rc) return rc;
  uint64_t c[4];
  for (uint32_t t1 = 1; t1 <= T1; ++t1) {
    for (uint32_t t2 = 0; t2 < T2; ++t2) {
      if (serial)
        ro_update_pass_serial(g, data, d, c);
      else
        ro_update_pass(g, data, d, c);
      if (pass_counts)
        memcpy(pass_counts + 4 * ((uint64_t)(t1 - 1) * T2 + t2), c, sizeof(c));
    }
    if (t1 != T1) ro_add_reverse_edges(g, R, order);
  }
  ro_graph_sort_lists(g);
  return 0;
}

/* rng_strategy, builder.cpp:196-212 (plain Alg. 3, no flags) */
int ro_rng_strategy(const float* data, uint32_t d, uint32_t u,
                    const uint32_t* cand_ids, const float* cand_dists,
                    uint32_t ncand, uint32_t* kept_ids, float* kept_dists) {
  entry_t* c = (entry_t*)malloc(sizeof(entry_t) * (ncand ? ncand : 1));
  for (uint32_t i = 0; i < ncand; ++i) {
    entry_t x = {cand_ids[i], cand_dists[i], 1};
    c[i] = x;
  }
  if (ncand > 1) qsort(c, ncand, sizeof(entry_t), cmp_nearer);
  uint32_t nk = 0;
  for (uint32_t i = 0; i < ncand; ++i) {
    if (c[i].id == u) {
      free(c);
      return -1;
    }
    int keep = 1;
    for (uint32_t k = 0; k < nk; ++k) {
      if (c[i].dist >= ro_l2_sq(data + (uint64_t)c[i].id * d,
                                data + (uint64_t)c[k].id * d, d)) {
        keep = 0;
        break;
      }
    }
    if (keep) c[nk++] = c[i];
  }
  for (uint32_t k = 0; k < nk; ++k) {
    kept_ids[k] = c[k].id;
    kept_dists[k] = c[k].dist;
  }
  free(c);
  return (int)nk;
}

/* ---------------------------------------------------------------- search */

typedef struct {
  float dist;
  uint32_t id;
  uint8_t expanded;
} pool_t;

/* pool_less, search.cpp:19-21 */
static int pool_less(const pool_t* a, const pool_t* b) {
  return a->dist != b->dist ? a->dist < b->dist : a->id < b->id;
}

/* select_nearest, graph.cpp:65-74: whole list if cap==0 or size<=cap, else
 * the cap nearest (dist, id) when the graph has distances, else the stored
 * prefix.  Writes into out, returns the count. */
static uint32_t select_nearest(const ro_graph* g, uint32_t u, uint32_t cap,
                               int has_distances, entry_t* out) {
  const list_t* l = &g->adj[u];
  memcpy(out, l->e, sizeof(entry_t) * l->size);
  if (cap == 0 || l->size <= cap) return l->size;
  if (has_distances) qsort(out, l->size, sizeof(entry_t), cmp_nearer);
  return cap;
}

/* search_impl, search.cpp:40-94 */
int ro_search(const ro_graph* g, const float* data, uint32_t d,
              const float* q, uint32_t L, uint32_t K, uint32_t k,
              int entry_mode, uint32_t entry_vertex, uint32_t entry_count,
              uint64_t seed, int has_distances, uint32_t* ids, float* dists,
              uint64_t* visited, uint64_t* dist_comps) {
  const uint64_t n = g->n;
  if (n == 0 || L < 1 || k < 1 || k > L) return -1;
  if (entry_mode == 1 && entry_vertex >= n) return -1;
  uint8_t* seen = (uint8_t*)calloc(n, 1);
  pool_t* pool = (pool_t*)malloc(sizeof(pool_t) * (L + 1));
  uint32_t psize = 0;
  uint32_t maxdeg = 0;
  for (uint64_t u = 0; u < n; ++u)
    if (g->adj[u].size > maxdeg) maxdeg = g->adj[u].size;
  entry_t* nbrs = (entry_t*)malloc(sizeof(entry_t) * (maxdeg ? maxdeg : 1));
  uint64_t vis = 0, comps = 0;

#define CONSIDER(ID)                                                         \
  do {                                                                       \
    uint32_t id_ = (ID);                                                     \
    if (!seen[id_]) {                                                        \
      seen[id_] = 1;                                                         \
      pool_t c_ = {ro_l2_sq(q, data + (uint64_t)id_ * d, d), id_, 0};        \
      ++comps;                                                               \
      if (!(psize == L && !pool_less(&c_, &pool[psize - 1]))) {              \
        uint32_t at_ = psize; /* upper_bound */                              \
        for (uint32_t z = 0; z < psize; ++z)                                 \
          if (pool_less(&c_, &pool[z])) { at_ = z; break; }                  \
        memmove(&pool[at_ + 1], &pool[at_], sizeof(pool_t) * (psize - at_)); \
        pool[at_] = c_;                                                      \
        ++psize;                                                             \
        if (psize > L) --psize;                                              \
      }                                                                      \
    }                                                                        \
  } while (0)

  if (entry_mode == 1) {
    CONSIDER(entry_vertex);
  } else {
    uint32_t count = entry_count ? (entry_count < n ? entry_count : (uint32_t)n)
                                 : (L < n ? L : (uint32_t)n);
    uint32_t* ent = (uint32_t*)malloc(sizeof(uint32_t) * count);
    uint64_t st = seed;
    ro_sample_distinct(&st, (uint32_t)n, count, UINT32_MAX, ent);
    for (uint32_t i = 0; i < count; ++i) CONSIDER(ent[i]);
    free(ent);
  }
  for (;;) {
    uint32_t at = psize;
    for (uint32_t i = 0; i < psize; ++i)
      if (!pool[i].expanded) { at = i; break; }
    if (at == psize) break;
    pool[at].expanded = 1;
    ++vis;
    uint32_t cnt = select_nearest(g, pool[at].id, K, has_distances, nbrs);
    for (uint32_t j = 0; j < cnt; ++j) CONSIDER(nbrs[j].id);
  }
#undef CONSIDER
  uint32_t take = k < psize ? k : psize;
  for (uint32_t i = 0; i < take; ++i) {
    ids[i] = pool[i].id;
    dists[i] = pool[i].dist;
  }
  if (visited) *visited = vis;
  if (dist_comps) *dist_comps = comps;
  free(nbrs);
  free(pool);
  free(seen);
  return (int)take;
}

/* brute_force_gt, dataset.cpp:175-205: k smallest (dist, id) per query */
void ro_brute_force(const float* base, uint64_t n, uint32_t d,
                    const float* queries, uint64_t nq, uint32_t k,
                    uint32_t* ids_out) {
  float* bd = (float*)malloc(sizeof(float) * (k + 1));
  uint32_t* bi = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
  for (uint64_t qi = 0; qi < nq; ++qi) {
    const float* qv = queries + qi * d;
    uint32_t m = 0; /* sorted ascending (dist, id) */
    for (uint64_t i = 0; i < n; ++i) {
      float dist = ro_l2_sq(qv, base + i * d, d);
      uint32_t id = (uint32_t)i;
      if (m == k && !(dist < bd[m - 1] || (dist == bd[m - 1] && id < bi[m - 1])))
        continue;
      uint32_t at = m;
      while (at > 0 && (dist < bd[at - 1] || (dist == bd[at - 1] && id < bi[at - 1]))) {
        if (at < k) {
          bd[at] = bd[at - 1];
          bi[at] = bi[at - 1];
        }
        --at;
      }
      bd[at] = dist;
      bi[at] = id;
      if (m < k) ++m;
    }
    for (uint32_t j = 0; j < k; ++j) ids_out[qi * k + j] = bi[j];
  }
  free(bd);
  free(bi);
}

/* degree_stats, graph.cpp:76-100 (summary fields only) */
void ro_degree_stats(const ro_graph* g, uint32_t cap, int has_distances,
                     uint64_t out[3]) {
  uint32_t* indeg = (uint32_t*)calloc(g->n ? g->n : 1, sizeof(uint32_t));
  uint32_t maxdeg = 0;
  for (uint64_t u = 0; u < g->n; ++u)
    if (g->adj[u].size > maxdeg) maxdeg = g->adj[u].size;
  entry_t* sel = (entry_t*)malloc(sizeof(entry_t) * (maxdeg ? maxdeg : 1));
  uint64_t edges = 0, max_out = 0, max_in = 0;
  for (uint64_t u = 0; u < g->n; ++u) {
    uint32_t c = select_nearest(g, (uint32_t)u, cap, has_distances, sel);
    edges += c;
    if (c > max_out) max_out = c;
    for (uint32_t j = 0; j < c; ++j) ++indeg[sel[j].id];
  }
  for (uint64_t u = 0; u < g->n; ++u)
    if (indeg[u] > max_in) max_in = indeg[u];
  out[0] = edges;
  out[1] = max_out;
  out[2] = max_in;
  free(sel);
  free(indeg);
}

static void put_u32(uint8_t* b, uint64_t* at, uint32_t v) {
  if (b) {
    b[*at] = (uint8_t)v;
    b[*at + 1] = (uint8_t)(v >> 8);
    b[*at + 2] = (uint8_t)(v >> 16);
    b[*at + 3] = (uint8_t)(v >> 24);
  }
  *at += 4;
}

static void put_u64(uint8_t* b, uint64_t* at, uint64_t v) {
  put_u32(b, at, (uint32_t)v);
  put_u32(b, at, (uint32_t)(v >> 32));
}

/* save_index byte layout, graph.cpp:102-126 / graph.hpp:67-71 */
uint64_t ro_index_bytes(const ro_graph* g, uint8_t* b) {
  uint64_t at = 0;
  if (b) memcpy(b, "RNND", 4);
  at = 4;
  put_u32(b, &at, 1);
  put_u64(b, &at, g->n);
  uint64_t off = 0;
  put_u64(b, &at, off);
  for (uint64_t u = 0; u < g->n; ++u) {
    off += g->adj[u].size;
    put_u64(b, &at, off);
  }
  for (uint64_t u = 0; u < g->n; ++u)
    for (uint32_t j = 0; j < g->adj[u].size; ++j) put_u32(b, &at, g->adj[u].e[j].id);
  uint32_t crc = b ? ro_crc32(b, at) : 0;
  put_u32(b, &at, crc);
  return at;
}

/* ---------------------------------------------------- NN-Descent baseline */

/* NnDescent::NnDescent + init, nndescent.cpp:11-37: pools start with
 * s = min(sample, n-1) distinct random ids (the random_init sampler,
 * stream mix_seed(seed, u)), fresh, sorted by nearer. */
int ro_nnd_init(ro_graph* P, const float* data, uint32_t d, uint32_t K,
                uint32_t sample, uint32_t iters, uint32_t pool, uint64_t seed) {
  const uint64_t n = P->n;
  if (n < 2) return 1;
  if (K < 1 || K > n - 1) return 1;
  if (sample < 1 || iters < 1) return 1;
  (void)pool;
  const uint32_t s = sample < n - 1 ? sample : (uint32_t)(n - 1);
  if (ro_random_init(P, data, d, s, seed)) return 1;
  ro_graph_sort_lists(P);
  return 0;
}

typedef struct {
  uint32_t dst, id;
  float dist;
} nnd_prop_t;

static int cmp_entry_flag(const void* x, const void* y) {
  /* nearer, then existing (old) entries before proposals of the same id */
  const entry_t *a = (const entry_t*)x, *b = (const entry_t*)y;
  if (nearer(a, b)) return -1;
  if (nearer(b, a)) return 1;
  return (int)a->fresh - (int)b->fresh;
}

static int cmp_prop_dst(const void* x, const void* y) {
  const nnd_prop_t *a = (const nnd_prop_t*)x, *b = (const nnd_prop_t*)y;
  return a->dst < b->dst ? -1 : a->dst > b->dst;
}

/* One join pass, canonical deferred form of NnDescent::join_pass
 * (nndescent.cpp:51-86).  Snapshot every vertex first (its nearest `sample`
 * fresh entries turn old and join; entries old before the pass join as old,
 * :60-70); then every pair (fresh x fresh, fresh x old, :77-80) proposes each
 * endpoint to the other's pool with d = l2_sq (:72-76); then each pool
 * becomes the max(cap, its size) nearest distinct entries of (pool +
 * proposals), new ones
 * fresh, existing ones keeping their flags (insert_candidate's cap, dedupe
 * and order, :39-49).  The reference applies proposals immediately under
 * per-vertex locks, which is order-dependent for threads > 1; this form is
 * order-free (l2_sq is bit-symmetric, so an id has one key per pool).
 * Returns the number of entries in the new pools that were not in the old. */
uint64_t ro_nnd_pass(ro_graph* P, const float* data, uint32_t d, uint32_t sample,
                     uint32_t cap) {
  const uint64_t n = P->n;
  uint32_t* F = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n * sample);
  uint32_t* fc = (uint32_t*)calloc(n, sizeof(uint32_t));
  list_t* O = (list_t*)calloc(n, sizeof(list_t));
  for (uint64_t u = 0; u < n; ++u) {
    list_t* l = &P->adj[u];
    for (uint32_t j = 0; j < l->size; ++j) {
      entry_t* e = &l->e[j];
      if (e->fresh && fc[u] < sample) {
        F[u * sample + fc[u]++] = e->id;
        e->fresh = 0;
      } else if (!e->fresh) {
        list_push(&O[u], *e);
      }
    }
  }
  nnd_prop_t* pr = NULL;
  size_t np = 0, pcap = 0;
#define NND_PUSH(a, b, dd)                                              \
  do {                                                                  \
    if (np + 2 > pcap) {                                                \
      pcap = pcap ? 2 * pcap : 1024;                                    \
      pr = (nnd_prop_t*)realloc(pr, sizeof(nnd_prop_t) * pcap);         \
    }                                                                   \
    pr[np].dst = (a); pr[np].id = (b); pr[np].dist = (dd); ++np;        \
    pr[np].dst = (b); pr[np].id = (a); pr[np].dist = (dd); ++np;        \
  } while (0)
  for (uint64_t u = 0; u < n; ++u) {
    const uint32_t* f = F + u * sample;
    for (uint32_t i = 0; i < fc[u]; ++i)
      for (uint32_t j = i + 1; j < fc[u]; ++j) {
        const float dd = ro_l2_sq(data + (uint64_t)f[i] * d, data + (uint64_t)f[j] * d, d);
        NND_PUSH(f[i], f[j], dd);
      }
    for (uint32_t i = 0; i < fc[u]; ++i)
      for (uint32_t j = 0; j < O[u].size; ++j) {
        const uint32_t o = O[u].e[j].id;
        const float dd = ro_l2_sq(data + (uint64_t)f[i] * d, data + (uint64_t)o * d, d);
        NND_PUSH(f[i], o, dd);
      }
  }
#undef NND_PUSH
  if (np) qsort(pr, np, sizeof(nnd_prop_t), cmp_prop_dst);
  uint64_t inserted = 0;
  size_t k = 0;
  list_t tmp = {NULL, 0, 0};
  for (uint64_t v = 0; v < n; ++v) {
    list_t* l = &P->adj[v];
    tmp.size = 0;
    for (uint32_t j = 0; j < l->size; ++j) list_push(&tmp, l->e[j]);
    const uint32_t old_n = l->size;
    /* a pool larger than cap (init fills min(sample, n-1) entries) keeps its
     * size: insert_candidate pops one entry per insertion (:46-47) */
    const uint32_t lim = old_n > cap ? old_n : cap;
    for (; k < np && pr[k].dst == v; ++k) {
      entry_t x = {pr[k].id, pr[k].dist, 1};
      list_push(&tmp, x);
    }
    if (tmp.size > 1) qsort(tmp.e, tmp.size, sizeof(entry_t), cmp_entry_flag);
    /* dedupe by id (equal ids are adjacent: same dist) and cap */
    entry_t* old = (entry_t*)malloc(sizeof(entry_t) * (old_n ? old_n : 1));
    memcpy(old, l->e, sizeof(entry_t) * old_n);
    l->size = 0;
    for (uint32_t j = 0; j < tmp.size && l->size < lim; ++j) {
      if (l->size && l->e[l->size - 1].id == tmp.e[j].id) continue;
      list_push(l, tmp.e[j]);
      int was = 0;
      for (uint32_t q = 0; q < old_n; ++q)
        if (old[q].id == tmp.e[j].id) { was = 1; break; }
      inserted += !was;
    }
    free(old);
  }
  free(tmp.e);
  free(pr);
  for (uint64_t u = 0; u < n; ++u) free(O[u].e);
  free(O);
  free(fc);
  free(F);
  return inserted;
}

/* NnDescent::finalize, nndescent.cpp:88-99: the K nearest pool entries,
 * flagged old. */
void ro_nnd_finalize(const ro_graph* P, uint32_t K, ro_graph* out) {
  for (uint64_t u = 0; u < P->n; ++u) {
    const list_t* l = &P->adj[u];
    list_t* o = &out->adj[u];
    o->size = 0;
    for (uint32_t j = 0; j < l->size && j < K; ++j) {
      entry_t x = l->e[j];
      x.fresh = 0;
      list_push(o, x);
    }
  }
}
