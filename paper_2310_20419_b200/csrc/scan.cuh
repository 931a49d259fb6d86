// scan.cuh -- launch interface of the distance stage (scan.cu).
#pragma once

#include <cstddef>
#include <cstdint>

struct rnndg_ctx;

namespace rnndg {

// lists up to this length keep their alive list in shared memory; longer ones
// use global scratch at the list's CSR offset (and are scheduled first)
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
// cached distances of the random initial lists (k_random_init left the raw
// samples in the keys' low 32 bits)
void launch_init_dists(rnndg_ctx* c, uint32_t S);

}  // namespace rnndg
