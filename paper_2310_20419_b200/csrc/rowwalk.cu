// rowwalk.cu -- the push walk (scan_vertex, builder.cpp:41-69; see scan.cu)
// for SHORT ROWS (d <= ~144: SIFT-like d = 128, Deep-like d = 96), one warp
// per list with the list's rows resident in shared memory.
//
// At d = 960 a pair costs 7.7 KB of row traffic and the walk is bound by the
// evaluation itself; at d = 96 a pair is 768 B and 288 flops, and the
// CTA-per-list kernels spend 55-75 SM-cycles per pair on round control and
// on the memory latency of every round's row loads, ten times the
// arithmetic.  Here a warp copies all rows of its list into shared memory
// once (cp.async, one memory round trip per list instead of one per round;
// a 64-entry list is 25 KB at d = 96) and then runs every round out of
// shared memory:
//
// * alive / touched sets are 32-bit masks (a lane owns positions lane + 32k),
//   the rounds are k_scan_spec's (an old-run window kept at once, or D
//   provisional entries whose fates are resolved in list order);
// * a round's pairs are enumerated kept-entry major into a small task list in
//   shared memory and evaluated 32 at a time, a lane per pair (every lane
//   busy: a first version with a lane per candidate, evaluating lazily,
//   left most lanes idle and was FP32-pipe bound on warp-level executions);
//   no block barriers anywhere;
// * rows are stored by list position with a stride of d + 4 floats ((d + 4) / 4
//   odd), so within a step the lanes' 128-bit reads of consecutive
//   candidates' rows are bank-conflict free and the kept entry's row is a
//   broadcast; the exact distance is the reference's four-chain sum read
//   straight from the row-major store (l2_step4).
//
// Lists are queued by size class (<= 16 / 32 / 64 / 128 entries, the queues
// the Gram walk uses) and each class is a launch with its own shared-memory
// budget per warp.  Results are the reference's bit for bit: the schedule of
// rounds never changes pair_checks, flag_skips, removed or a redirect
// (scan.cu header).
#include <array>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "ctx.hpp"
#include "quad.cuh"
#include "scan.cuh"

namespace rnndg {

namespace {

constexpr int kMaxD = 4;          // provisional entries per speculative round, at most
constexpr uint32_t kWin = 16;     // old-run window
constexpr uint32_t kSmemBudget = 216 * 1024;  // per SM, for the resident rows (200 KB: C4 1M 0.477 s, 216 KB: 0.459 s)

struct RowWalkArgs {
  const uint32_t* queue;      // this class's lists
  const unsigned long long* count;
  unsigned int* cursor;
  const float* x;             // row-major store, 16-byte aligned rows
  uint32_t d;                 // multiple of 4
  uint32_t rs;                // row stride in shared memory (floats): d + 4
  uint32_t max_rows;          // rows per warp region
  uint32_t warp_bytes;        // shared memory per warp
  const uint64_t* off;
  const uint32_t* cnt;
  uint64_t* keys;
  uint32_t* post_cnt;
  uint32_t* pend_src;
  uint64_t* pend_key;
  unsigned long long* bcnt;
  unsigned long long* ctr;
  int D;
  unsigned long long nz;      // (-0.0f, -0.0f), opaque to the compiler (dist_rows)
};

__device__ __forceinline__ uint32_t lt_mask(uint32_t lane) { return (1u << lane) - 1u; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   uint32_t(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// exact l2_sq of two shared-memory rows (metric.hpp:15-24 order; d % 4 == 0).
// A lane owns all four chains, so one 128-bit read holds one element of each
// and the three roundings of a step -- t = a - b, m = t * t, s = s + m -- run
// as packed f32x2 instructions on the chain pairs (0, 1) and (2, 3): the same
// IEEE round-to-nearest per element as the scalar FSUB / FMUL / FADD, at half
// the FP32-pipe issue.  The square is fma(t, t, nz) with nz = (-0, -0) read
// from the kernel arguments: adding -0 changes no value (a zero product
// stays +0), and because ptxas cannot see the constant it cannot turn the
// square and the following add into one fused multiply-add.
__device__ __forceinline__ float dist_rows(const float* a, const float* b, uint32_t q4,
                                           unsigned long long nz) {
  // (plain 128-bit loads, not inline asm: unrolled, they take immediate
  // offsets from one address register per row -- with asm loads a third of
  // the loop's instructions were address arithmetic)
  const ulonglong2* a2 = reinterpret_cast<const ulonglong2*>(a);
  const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(b);
  unsigned long long s01 = 0ull, s23 = 0ull;  // (+0, +0)
#pragma unroll 8
  for (uint32_t c = 0; c < q4; ++c) {
    const ulonglong2 av = a2[c], bv = b2[c];
    unsigned long long t01, t23, m01, m23;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t01) : "l"(av.x), "l"(bv.x));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t23) : "l"(av.y), "l"(bv.y));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m01) : "l"(t01), "l"(nz));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m23) : "l"(t23), "l"(nz));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s01) : "l"(s01), "l"(m01));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s23) : "l"(s23), "l"(m23));
  }
  float s0, s1, s2, s3;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(s0), "=f"(s1) : "l"(s01));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(s2), "=f"(s3) : "l"(s23));
  return l2_finish(s0, s1, s2, s3);
}

// One list per CTA.  Warp 0 walks it; with NW > 1 the other warps are helpers
// that share the two bulk steps -- the row copy and a round's evaluation --
// between two block barriers.  The rows a list keeps resident bound how many
// lists fit an SM, so for the larger size classes the helpers are lanes the
// shared memory has already paid for.
enum : uint32_t { kJobExit = 0, kJobCopy, kJobRun, kJobSpec };

__device__ __forceinline__ void copy_rows(const RowWalkArgs& g, float* rows, const uint32_t* ids,
                                          uint32_t U, uint32_t q4, uint32_t nt) {
  // chunk idx = r * q4 + c, stepped by nt without a division per chunk
  const uint32_t dr = nt / q4, dc = nt - dr * q4;
  uint32_t r = threadIdx.x / q4, c = threadIdx.x - r * q4;
  while (r < U) {
    cp_async16(rows + r * g.rs + 4 * c, g.x + uint64_t(ids[r]) * g.d + 4 * c);
    r += dr;
    c += dc;
    if (c >= q4) {
      c -= q4;
      ++r;
    }
  }
}
__device__ __forceinline__ void eval_run(const RowWalkArgs& g, const float* rows, const uint8_t* tpos,
                                         const uint32_t* wp, float* res, uint32_t ntask, uint32_t nf,
                                         uint32_t q4, uint32_t nt) {
  for (uint32_t t = threadIdx.x; t < ntask; t += nt) {
    const uint32_t i = t / nf, r = t - i * nf;
    res[t] = dist_rows(rows + uint32_t(tpos[r]) * g.rs, rows + wp[i] * g.rs, q4, g.nz);
  }
}
__device__ __forceinline__ void eval_spec(const RowWalkArgs& g, const float* rows,
                                          const uint8_t* tpos, const uint32_t* wp, float* res,
                                          uint32_t ntask, uint32_t b1, uint32_t b2, uint32_t b3,
                                          uint32_t q4, uint32_t nt) {
  for (uint32_t t = threadIdx.x; t < ntask; t += nt) {
    const uint32_t i = (t >= b1 ? 1u : 0u) + (t >= b2 ? 1u : 0u) + (t >= b3 ? 1u : 0u);
    res[t] = dist_rows(rows + uint32_t(tpos[t]) * g.rs, rows + wp[i] * g.rs, q4, g.nz);
  }
}

template <int NP, int NW, int MD>
__global__ void __launch_bounds__(32 * NW, NW == 1 ? (NP == 1 ? 24 : 12) : 1) k_walk_rows(RowWalkArgs g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr uint32_t NT = 32 * NW;
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  unsigned char* wbase = smem_raw;
  float* rows = reinterpret_cast<float*>(wbase);
  unsigned char* tail = wbase + size_t(g.max_rows) * g.rs * 4;
  uint64_t* wk = reinterpret_cast<uint64_t*>(tail);            // window / provisional keys
  uint32_t* wp = reinterpret_cast<uint32_t*>(tail + 8 * kWin);  // their positions
  float* fd = reinterpret_cast<float*>(tail + 12 * kWin);       // d(w_j, w_i), [j * kMaxD + i]
  const uint32_t tcap = kMaxD * g.max_rows;                     // tasks of a round, at most
  float* res = reinterpret_cast<float*>(tail + 12 * kWin + 4 * kMaxD * kMaxD);  // their distances
  uint8_t* tpos = reinterpret_cast<uint8_t*>(res + tcap);       // their candidates' positions
  uint32_t* job = reinterpret_cast<uint32_t*>(tpos + tcap);     // job, and its parameters
  uint32_t* ids = reinterpret_cast<uint32_t*>(res);             // row ids during the copy
  if (NW > 1 && wid > 0) {
    const uint32_t q4h = g.d >> 2;
    for (;;) {
      __syncthreads();  // a job is posted
      const uint32_t jb = job[0];
      if (jb == kJobExit) return;
      if (jb == kJobCopy) {
        copy_rows(g, rows, ids, job[1], q4h, NT);
        cp_async_wait_all();
      } else if (jb == kJobRun)
        eval_run(g, rows, tpos, wp, res, job[1], job[2], q4h, NT);
      else
        eval_spec(g, rows, tpos, wp, res, job[1], job[2], job[3], job[4], q4h, NT);
      __syncthreads();  // its results are visible
    }
  }
  const uint32_t q4 = g.d >> 2;
  const uint32_t count = uint32_t(*g.count);
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0, evals = 0;

  // The next list's vertex, offset, length and keys are fetched while the
  // current list's rows are still landing, so the chain of dependent global
  // loads (queue -> off / cnt -> keys) is off the walk's critical path.
  uint32_t u2 = 0, U2 = 0;
  uint64_t base2 = 0, kk2[NP];
  bool have2 = false;
  auto fetch_next = [&]() {
    uint32_t it = 0;
    if (lane == 0) it = atomicAdd(g.cursor, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    have2 = it < count;
    if (!have2) return;
    u2 = g.queue[it];
    base2 = g.off[u2];
    U2 = g.cnt[u2];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const uint32_t p = 32u * k + lane;
      kk2[k] = p < U2 ? g.keys[base2 + p] : 0ull;
    }
  };
  fetch_next();
  while (have2) {
    const uint32_t u = u2;
    const uint64_t base = base2;
    const uint32_t U = U2;
    uint64_t* L = g.keys + base;
    uint64_t kk[NP];
    uint32_t M[NP], T[NP], F[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const uint32_t p = 32u * k + lane;
      kk[k] = kk2[k];
      M[k] = __ballot_sync(0xffffffffu, p < U);
      F[k] = __ballot_sync(0xffffffffu, p < U && key_fresh(kk[k]));
      T[k] = 0;
    }
    // the list's rows -> shared memory, row r at rows + r * rs
    __syncwarp();  // the previous list's reads are done
#pragma unroll
    for (int k = 0; k < NP; ++k)
      if (32u * k + lane < U) ids[32u * k + lane] = key_id(kk[k]);
    if (lane == 0) {
      job[0] = kJobCopy;
      job[1] = U;
    }
    __syncthreads();
    copy_rows(g, rows, ids, U, q4, NT);
    fetch_next();  // in flight together with the row copies
    cp_async_wait_all();
    __syncthreads();
    bool pf_next = have2;
    uint32_t nk = 0;

    for (;;) {
      // ------------------------------------------------------------ plan
      uint32_t arank[NP];
      uint32_t na = 0, nf = 0;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        arank[k] = na + __popc(M[k] & lt_mask(lane));
        na += __popc(M[k]);
        nf += __popc(M[k] & F[k]);
      }
      if (na == 0) break;
      // alive entries ahead of the first fresh one
      uint32_t run = na;
      {
        uint32_t before = 0;
        bool found = false;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const uint32_t mf = M[k] & F[k];
          if (!found && mf) {
            const uint32_t b = uint32_t(__ffs(mf)) - 1u;
            run = before + __popc(M[k] & lt_mask(b));
            found = true;
          }
          before += __popc(M[k]);
        }
      }
      // a round's pairs are enumerated kept-entry major -- task base[i] + r is
      // the r-th candidate that needs w_i -- and evaluated 32 at a time, a lane
      // per pair: within one step the lanes share w_i's row (a broadcast) and
      // read consecutive candidates' rows (distinct banks)
      uint32_t frank[NP];
      {
        uint32_t f = 0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          frank[k] = f + __popc(M[k] & F[k] & lt_mask(lane));
          f += __popc(M[k] & F[k]);
        }
      }
      uint32_t wr = run < kWin ? run : kWin;
      if (wr * nf > tcap) wr = tcap / nf;  // window x fresh candidates must fit (rarely binds)
      const bool run_round = wr >= 2;
      const uint32_t De = run_round ? wr : (na < uint32_t(g.D) ? na : uint32_t(g.D));
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if ((M[k] >> lane & 1u) && arank[k] < De) {
          wk[arank[k]] = kk[k];
          wp[arank[k]] = 32u * k + lane;
        }
      uint32_t gone_m[NP], touch_m[NP];
      if (run_round) {
        // Old-run round: the window is kept whole (old / old pairs are
        // skipped, builder.cpp:53-56); every fresh candidate is tested against
        // it and walks the results in order up to its first occluder.
#pragma unroll
        for (int k = 0; k < NP; ++k)
          if (M[k] & F[k] & (1u << lane)) tpos[frank[k]] = uint8_t(32u * k + lane);
        __syncwarp();
        const uint32_t ntask = nf * wr;
        evals += lane == 0 ? ntask : 0u;
        if (lane == 0) {
          job[0] = kJobRun;
          job[1] = ntask;
          job[2] = nf;
        }
        __syncthreads();
        eval_run(g, rows, tpos, wp, res, ntask, nf, q4, NT);
        __syncthreads();
        uint32_t reach = 0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          bool gone = false;
          const bool al = M[k] >> lane & 1u;
          const bool mine = al && (F[k] >> lane & 1u);
          if (mine) {
            const uint64_t vk = kk[k];
            const uint32_t q = 32u * k + lane;
            for (uint32_t i = 0; i < wr; ++i) {
              const float d = res[i * nf + frank[k]];
              ++checks;
              reach = reach > i + 1 ? reach : i + 1;
              if (key_dist(vk) >= d) {
                gone = true;
                ++removed;
                const uint32_t w_id = key_id(wk[i]);
                g.pend_src[base + q] = w_id;
                g.pend_key[base + q] = make_key(d, key_id(vk), 1u);
                if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
                break;
              }
            }
          } else if (al && arank[k] >= wr) {
            skips += wr;  // an old candidate behind the window
          }
          gone_m[k] = __ballot_sync(0xffffffffu, gone);
          touch_m[k] = __ballot_sync(0xffffffffu, mine);
        }
        reach = __reduce_max_sync(0xffffffffu, reach);
        if (lane == 0) skips += uint64_t(wr) * (wr - 1) / 2;  // the window among itself
        __syncwarp();
        if (lane < wr) L[nk + lane] = wk[lane];  // old already
        nk += wr;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const bool al = M[k] >> lane & 1u;
          const uint32_t inwin = __ballot_sync(0xffffffffu, al && arank[k] < wr);
          const uint32_t tw = __ballot_sync(0xffffffffu, al && arank[k] < reach);
          T[k] |= touch_m[k] | tw;
          M[k] &= ~(inwin | gone_m[k]);
        }
      } else {
        // Speculative round: candidate ai >= 1 needs w_i for i < min(ai, De)
        // where a flag is fresh; the provisional entries w_2 .. w_De are
        // candidates too (their pairs decide the fates).
        __syncwarp();
        uint32_t nm[NP], lim[NP], idx[NP][MD];
        uint32_t bases[kMaxD + 1] = {};
        bases[0] = 0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const bool al = M[k] >> lane & 1u;
          const uint32_t ai = arank[k];
          const bool vf = key_fresh(kk[k]);
          lim[k] = al ? (ai < De ? ai : De) : 0u;
          uint32_t m = 0;
#pragma unroll
          for (int i = 0; i < MD; ++i)
            if (uint32_t(i) < lim[k] && (key_fresh(wk[i]) || vf)) m |= 1u << i;
          nm[k] = m;
        }
#pragma unroll
        for (int i = 0; i < MD; ++i) {
          uint32_t c = 0;
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const uint32_t bm = __ballot_sync(0xffffffffu, nm[k] >> i & 1u);
            idx[k][i] = bases[i] + c + __popc(bm & lt_mask(lane));
            c += __popc(bm);
          }
          bases[i + 1] = bases[i] + c;
        }
        const uint32_t ntask = bases[MD];
#pragma unroll
        for (int i = MD + 1; i <= kMaxD; ++i) bases[i] = ntask;
        evals += lane == 0 ? ntask : 0u;
#pragma unroll
        for (int k = 0; k < NP; ++k)
#pragma unroll
          for (int i = 0; i < MD; ++i)
            if (nm[k] >> i & 1u) tpos[idx[k][i]] = uint8_t(32u * k + lane);
        __syncwarp();
        // (two pairs per lane per step, for more loads and chains in flight,
        // measured no faster: the steps are not what the warps wait on)
        if (lane == 0) {
          job[0] = kJobSpec;
          job[1] = ntask;
          job[2] = bases[1];
          job[3] = bases[2];
          job[4] = bases[3];
        }
        __syncthreads();
        eval_spec(g, rows, tpos, wp, res, ntask, bases[1], bases[2], bases[3], q4, NT);
        __syncthreads();
        // the provisional entries publish their pairs; fates in list order,
        // the same on every lane
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const uint32_t j = arank[k];
          if ((M[k] >> lane & 1u) && j >= 1 && j < De)
#pragma unroll
            for (int i = 0; i < MD; ++i)
              if (nm[k] >> i & 1u) fd[j * kMaxD + i] = res[idx[k][i]];
        }
        __syncwarp();
        uint32_t kept = 1u;
        for (uint32_t j = 1; j < De; ++j) {
          const float dj = key_dist(wk[j]);
          bool occl = false;
          for (uint32_t i = 0; i < j && !occl; ++i) {
            if (!(key_fresh(wk[i]) || key_fresh(wk[j]))) continue;
            if ((kept >> i & 1u) && dj >= fd[j * kMaxD + i]) occl = true;
          }
          if (!occl) kept |= 1u << j;
        }
        uint32_t wtouch = 0;  // provisional entries with a counted check
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          bool gone = false, tch = false;
          const uint64_t vk = kk[k];
          const uint32_t q = 32u * k + lane;
#pragma unroll
          for (int i = 0; i < MD; ++i) {
            if (uint32_t(i) >= lim[k] || gone) continue;
            if (!(kept >> i & 1u)) continue;  // not in the reference's kept list
            if (!(nm[k] >> i & 1u)) {
              ++skips;
              continue;
            }
            const float d = res[idx[k][i]];
            ++checks;
            tch = true;
            wtouch |= 1u << i;
            if (key_dist(vk) >= d) {
              gone = true;
              ++removed;
              const uint32_t w_id = key_id(wk[i]);
              g.pend_src[base + q] = w_id;
              g.pend_key[base + q] = make_key(d, key_id(vk), 1u);
              if (g.bcnt) atomicAdd(&g.bcnt[w_id], 1ull);
            }
          }
          gone_m[k] = __ballot_sync(0xffffffffu, gone);
          touch_m[k] = __ballot_sync(0xffffffffu, tch);
        }
        wtouch = __reduce_or_sync(0xffffffffu, wtouch);
        __syncwarp();
        // kept entries, flagged old (builder.cpp:68), in list order
        {
          uint32_t n2 = nk;
#pragma unroll
          for (int i = 0; i < MD; ++i)
            if (uint32_t(i) < De && (kept >> i & 1u)) {
              if (lane == 0) L[n2] = wk[i] & ~1ull;
              ++n2;
            }
          nk = n2;
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          // a provisional entry leaves the alive set when kept, and is touched
          // when some candidate had a counted check with it
          const bool prov = (M[k] >> lane & 1u) && arank[k] < De;
          const uint32_t km = __ballot_sync(0xffffffffu, prov && (kept >> arank[k] & 1u));
          const uint32_t tm = __ballot_sync(0xffffffffu, prov && (wtouch >> arank[k] & 1u));
          T[k] |= touch_m[k] | tm;
          M[k] &= ~(km | gone_m[k]);
        }
      }
      if (pf_next) {
        // the next list's rows towards L2 (its keys have arrived by now)
        pf_next = false;
#pragma unroll
        for (int k = 0; k < NP; ++k)
          if (32u * k + lane < U2)
            prefetch_row_l2(g.x + uint64_t(key_id(kk2[k])) * g.d, g.d * 4u);
      }
    }
    if (lane == 0) {
      g.post_cnt[u] = nk;
      uint32_t tc = 0;
#pragma unroll
      for (int k = 0; k < NP; ++k) tc += __popc(T[k]);
      touched += tc;
    }
  }
  if (NW > 1) {
    if (lane == 0) job[0] = kJobExit;
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) {
    touched += __shfl_xor_sync(0xffffffffu, touched, o);
    removed += __shfl_xor_sync(0xffffffffu, removed, o);
    checks += __shfl_xor_sync(0xffffffffu, checks, o);
    skips += __shfl_xor_sync(0xffffffffu, skips, o);
    evals += __shfl_xor_sync(0xffffffffu, evals, o);
  }
  if (lane == 0) {
    if (touched) atomicAdd(&g.ctr[kTouched], touched);
    if (removed) atomicAdd(&g.ctr[kRemoved], removed);
    if (checks) atomicAdd(&g.ctr[kPairChecks], checks);
    if (skips) atomicAdd(&g.ctr[kFlagSkips], skips);
    if (evals) atomicAdd(&g.ctr[kEvalPairs], evals);
  }
}

}  // namespace

// Lists of at most this many entries take the shared-memory walk (0 = off):
// rows of at most 576 bytes with d % 4 == 0 and a 16-byte aligned store,
// Gram walk off.  RNNDG_ROWWALK = 0 | 16 | 32 | 64 | 128 overrides the cap.
uint32_t rowwalk_cap(rnndg_ctx* c) {
  static const int forced = [] {
    const char* e = std::getenv("RNNDG_ROWWALK");
    return e ? std::atoi(e) : -1;
  }();
  if (forced == 0 || gram_cap() || bsp_rounds()) return 0;
  if (c->d == 0 || c->d % 4 != 0 || c->d > 144) return 0;
  if (reinterpret_cast<uintptr_t>(c->x) % 16 != 0) return 0;
  // measured with one list per CTA and classes 20 / 32 / 44 / 64 (C4 1M d = 96:
  // 0.399 s; classes up to 80 / 96 / 128: 0.424 / 0.425 / 0.437 s; off 0.765 s.
  // C2 1M d = 128: 0.421 s; up to 48 / 96: 0.422 / 0.458 s; off 0.605 s)
  uint32_t cap = 64;
  if (const char* e = std::getenv("RNNDG_ROWWALK_CLS")) {  // explicit classes set the cap
    unsigned last = 0;
    for (const char* p = e; *p;) {
      last = unsigned(std::strtoul(p, nullptr, 10));
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
    if (last >= 4 && last <= 128) return last;
  }
  if (forced > 0) cap = forced <= 16 ? 16 : (forced <= 32 ? 32 : (forced <= 64 ? 64 : 128));
  return cap;
}

// Size classes: a warp's shared-memory region holds the class's longest list,
// so finer classes mean more resident warps for the shorter lists.
void rowwalk_classes(rnndg_ctx* c, uint32_t cls[kSizeClasses]) {
  const uint32_t cap = rowwalk_cap(c);
  // RNNDG_ROWWALK_CLS=a,b,...: explicit ascending class bounds (up to 8;
  // experiments); the last one is the cap
  static const std::array<uint32_t, kSizeClasses> forced = [] {
    std::array<uint32_t, kSizeClasses> v{};
    if (const char* e = std::getenv("RNNDG_ROWWALK_CLS")) {
      int n = 0;
      for (const char* p = e; *p && n < kSizeClasses;) {
        v[n++] = uint32_t(std::strtoul(p, nullptr, 10));
        while (*p && *p != ',') ++p;
        if (*p == ',') ++p;
      }
      for (int i = n; i < kSizeClasses; ++i) v[i] = n ? v[n - 1] : 0;
    }
    return v;
  }();
  bool ok = forced[0] > 0 && forced[kSizeClasses - 1] <= 128;
  for (int i = 1; i < kSizeClasses; ++i) ok = ok && forced[i] >= forced[i - 1];
  if (ok) {
    for (int i = 0; i < kSizeClasses; ++i) cls[i] = forced[i];
    return;
  }
  // a region holds its class's longest list, so finer classes mean more
  // resident lists; 20 = the initial list length S of the paper's builds
  // (most lists of an update phase's first passes)
  // (small stores are launch-bound: four classes -- duplicates are skipped --
  // keep C1 20k at 0.019 s where eight cost 0.022 s; at 1M / 10M rows eight
  // classes gain 1.5-3%: C4 1M 0.396 -> 0.389 s, C5 10M 7.15 -> 6.95 s)
  static const uint32_t k64s[kSizeClasses] = {20, 20, 32, 32, 44, 44, 64, 64};
  static const uint32_t k64[kSizeClasses] = {12, 16, 20, 26, 32, 40, 50, 64};
  static const uint32_t k128[kSizeClasses] = {16, 20, 32, 44, 64, 80, 100, 128};
  static const uint32_t k32[kSizeClasses] = {8, 12, 16, 20, 24, 28, 32, 32};
  static const uint32_t k16[kSizeClasses] = {4, 6, 8, 10, 12, 14, 16, 16};
  const uint32_t* t = cap >= 128 ? k128 : (cap >= 64 ? k64 : (cap >= 32 ? k32 : k16));
  if (cap == 64 && c->nv < (1u << 18)) t = k64s;
  for (int i = 0; i < kSizeClasses; ++i) cls[i] = t[i];
}

void launch_rowwalk(rnndg_ctx* c, unsigned int* work, cudaStream_t stream, int spec) {
  const uint32_t cap = rowwalk_cap(c);
  if (!cap) return;
  const uint64_t n = c->nv;
  RowWalkArgs a{};
  a.x = c->x;
  a.d = c->d;
  a.rs = c->d + 4;  // (rs / 4) odd for d % 32 == 0; any d % 4 == 0 keeps 16-byte alignment
  if ((a.rs / 4) % 2 == 0) a.rs += 4;
  a.off = c->off.p;
  a.cnt = c->cnt.p;
  a.keys = c->key.p;
  a.post_cnt = c->post_cnt.p;
  a.pend_src = c->pend_src.p;
  a.pend_key = c->pend_key.p;
  a.bcnt = c->partitioned ? nullptr : c->bcnt.p;
  a.ctr = c->counters.p;
  a.nz = 0x8000000080000000ull;
  // provisional entries per speculative round (RNNDG_ROWWALK_D, 2 .. 4): here a
  // step evaluates 32 pairs whether or not they are needed, so the depth is
  // chosen to fill the steps, not to save pairs (the first pass over the
  // random lists included, where the CTA kernels drop to 2)
  static const int forced_d = [] {
    const char* e = std::getenv("RNNDG_ROWWALK_D");
    const int v = e ? std::atoi(e) : 0;
    return v >= 2 && v <= kMaxD ? v : 0;
  }();
  (void)spec;
  a.D = forced_d ? forced_d : 3;
  uint32_t class_rows[kSizeClasses];
  rowwalk_classes(c, class_rows);
  for (int gc = kSizeClasses - 1; gc >= 0; --gc) {  // the longest walks first
    if (gc > 0 && class_rows[gc] == class_rows[gc - 1]) continue;  // an empty (duplicate) class
    a.queue = c->gram_q.p + uint64_t(gc) * n;
    a.count = c->counters.p + kGram0 + gc;
    a.cursor = work + 8 + gc;
    a.max_rows = class_rows[gc];
    a.warp_bytes = a.max_rows * a.rs * 4 + 12 * kWin + 4 * kMaxD * kMaxD +
                   5 * kMaxD * a.max_rows + 32;  // + task results, positions, the job words
    a.warp_bytes = (a.warp_bytes + 15u) & ~15u;
    static const uint32_t budget = [] {
      const char* e = std::getenv("RNNDG_ROWWALK_SMEM");  // KB per SM for the resident rows
      const int v = e ? std::atoi(e) : 0;
      return v >= 32 && v <= 224 ? uint32_t(v) * 1024u : kSmemBudget;
    }();
    uint32_t lists = budget / a.warp_bytes;  // resident lists (CTAs) per SM
    if (lists < 1) continue;
    if (lists > 32) lists = 32;
    // warps per list: helpers where the rows leave few lists per SM
    // (RNNDG_ROWWALK_NW forces 1 | 2 | 4)
    static const int forced_nw = [] {
      const char* e = std::getenv("RNNDG_ROWWALK_NW");
      const int v = e ? std::atoi(e) : 0;
      return v == 1 || v == 2 || v == 4 ? v : 0;
    }();
    // (helpers measured slower wherever tried -- C4 1M 0.407 s with one warp
    // per list, 0.461 s with two: they double a list's registers, which then
    // bound the resident lists instead of the rows -- so the default is 1)
    const int nw = forced_nw ? forced_nw : 1;
    (void)lists;
    const size_t smem = a.warp_bytes;
    const int np = class_rows[gc] <= 32 ? 1 : (class_rows[gc] <= 64 ? 2 : 4);
    void (*kern)(RowWalkArgs) = nullptr;
    if (a.D <= 3) {  // (the common depth: one iteration less in every unrolled loop over w)
      if (np == 1) kern = nw == 1 ? k_walk_rows<1, 1, 3> : (nw == 2 ? k_walk_rows<1, 2, 3> : k_walk_rows<1, 4, 3>);
      if (np == 2) kern = nw == 1 ? k_walk_rows<2, 1, 3> : (nw == 2 ? k_walk_rows<2, 2, 3> : k_walk_rows<2, 4, 3>);
      if (np == 4) kern = nw == 1 ? k_walk_rows<4, 1, 3> : (nw == 2 ? k_walk_rows<4, 2, 3> : k_walk_rows<4, 4, 3>);
    } else {
      if (np == 1) kern = nw == 1 ? k_walk_rows<1, 1, 4> : (nw == 2 ? k_walk_rows<1, 2, 4> : k_walk_rows<1, 4, 4>);
      if (np == 2) kern = nw == 1 ? k_walk_rows<2, 1, 4> : (nw == 2 ? k_walk_rows<2, 2, 4> : k_walk_rows<2, 4, 4>);
      if (np == 4) kern = nw == 1 ? k_walk_rows<4, 1, 4> : (nw == 2 ? k_walk_rows<4, 2, 4> : k_walk_rows<4, 4, 4>);
    }
    // the attribute is per function, not per launch: several host threads
    // (csrc/multi.cu drives one context each) launch the same instantiation
    // with different class sizes, so it is always set to the device maximum
    // -- a per-class value set by one thread could be lowered by another
    // between that thread's set and its launch
    static thread_local int optin_dev = -1, optin = 0;
    if (optin_dev != c->device) {
      RNNDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
      optin_dev = c->device;
    }
    if (smem > size_t(optin)) continue;
    RNNDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    kern<<<unsigned(sm_count(c)) * lists, 32 * nw, smem, stream>>>(a);
    ++c->launches;
  }
  RNNDG_CUDA(cudaGetLastError());
}

}  // namespace rnndg
