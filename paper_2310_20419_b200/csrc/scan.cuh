// scan.cuh -- launch interface of the distance stage (scan.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

struct rnndg_ctx;

namespace rnndg {

// capacity of the short-list kernel's shared-memory key / alive arrays (the
// hub threshold, build.cu hub_threshold(), is at most this); longer lists use
// global scratch at the list's CSR offset
constexpr uint32_t kScanUcap = 512;

// chain-blocked device copy of the store (see k_chain_layout in scan.cu)
struct ScanConfig {
  uint32_t nblk;    // 32-element blocks of the 4-aligned prefix
  uint32_t ntail;   // d % 4 tail elements
  uint32_t stride;  // row stride in floats (multiple of 8)
};

ScanConfig scan_config(rnndg_ctx* c);
void prepare_chain_layout(rnndg_ctx* c);
void launch_scan(rnndg_ctx* c, unsigned int* work);
// Gram-filtered walk for lists of at most gram_cap() entries (gram.cu;
// RNNDG_GRAM, 0 = off): k_mark_active queues them by size class
uint32_t gram_cap();
void launch_gram(rnndg_ctx* c, unsigned int* work);
void gram_trace(rnndg_ctx* c);
// round-synchronous walk of the short lists (bsp.cu; RNNDG_BSP = rounds per
// pass, 0 = off): lists of at most bsp_max_len() entries, queued in act_small
int bsp_rounds();
uint32_t bsp_max_len();
void launch_bsp(rnndg_ctx* c, unsigned int* work, cudaStream_t stream, int spec, int l2pf);
// shared-memory walk for short rows (rowwalk.cu): lists of at most
// rowwalk_cap() entries (0 = off), queued by size class like the Gram walk's;
// cursors at work[8 .. 12)
uint32_t rowwalk_cap(rnndg_ctx* c);
void rowwalk_classes(rnndg_ctx* c, uint32_t cls[8]);  // upper bounds of its 8 size classes (ctx.hpp kSizeClasses)
void launch_rowwalk(rnndg_ctx* c, unsigned int* work, cudaStream_t stream, int spec);
// provisional entries per push round (RNNDG_SPEC) and the hub-cluster size
// (0 = one CTA per hub list); build.cu queues big hubs only when clustered
int spec_mode();
int hub_cluster_size(rnndg_ctx* c);
// cached distances of the random initial lists (k_random_init left the raw
// samples in the keys' low 32 bits)
void launch_init_dists(rnndg_ctx* c, uint32_t S);
// NN-Descent join of vertices [u0, u1): every pair of their snapshot lists
// (fresh x fresh, fresh x old; pair p of vertex u at poff[u] + local index)
// proposes each endpoint to the other, written at 2 * (p - poff[u0])
void launch_nnd_join(rnndg_ctx* c, uint64_t u0, uint64_t u1, uint64_t npairs);

}  // namespace rnndg
