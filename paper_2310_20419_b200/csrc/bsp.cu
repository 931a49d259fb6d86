// bsp.cu -- the push walk (scan_vertex, builder.cpp:41-69; see scan.cu) of
// short lists, round-synchronous across lists instead of one resident CTA
// per list: RNNDG_BSP = R rounds (0 = off).
//
// k_scan_spec holds a CTA on a list for all of its rounds; every round is a
// barrier-delimited wave of at most 16 pair evaluations, so the SM runs the
// exact-L2 loop with 12 warps at ~127 SM-cycles per evaluation, while the same
// loop over a flat task array reaches ~86 (tools/ubench/flat_pairs.cu: no
// walk state in registers, no partial waves, no barriers).  Here a list's walk
// is cut at its round boundaries:
//
//   k_bsp_ctl   one warp per list (<= 128 entries: alive / touched sets are
//               4 x 32-bit masks, a lane owns positions lane + 32k).  It
//               resolves the list's previous round from the distances in
//               `res` (fates of the provisional entries, every candidate's
//               walk, redirect records, kept entries written in place), plans
//               the next round (old-run window or D provisional entries,
//               exactly the rounds of k_scan_spec) and appends its pairs to
//               the flat task array.  Rounds without pairs are resolved on
//               the spot.  The state between rounds is 40 bytes per list.
//   k_bsp_eval  evaluates the task array: a quad per pair, 64 registers,
//               dynamic 8-task claims; nothing else.
//
// Rounds alternate ctl / eval launches; in the last ctl launch every warp
// finishes its list by itself (its 8 quads evaluate the round's tasks from a
// per-warp scratch), which also takes lists whose tasks did not fit the task
// array.  The plan of a round is a pure function of the list's state, so the
// resolving launch recomputes it instead of storing it.  The schedule of
// rounds does not change any result (scan.cu header): pair_checks,
// flag_skips, removed and every redirect are the reference's.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "ctx.hpp"
#include "quad.cuh"
#include "scan.cuh"

namespace rnndg {

namespace {

constexpr int kP = 4;                      // mask words per list
constexpr uint32_t kBspMaxLen = 32 * kP;   // longest list walked here
constexpr int kMaxD = 4;                   // provisional entries per round, at most
constexpr uint32_t kRunMax = 16;           // old-run window
constexpr uint32_t kRunBudget = 256;       // tasks of an old-run round, at most
constexpr uint32_t kInlineSlots = 512;     // per-warp scratch >= kMaxD * 127, >= kRunBudget
constexpr uint32_t kStateWords = 2 * kP + 6;  // masks, kept, task base, vertex, length, offset
constexpr int kCtlWarps = 8;
constexpr int kMaxRounds = 64;

struct BspArgs {
  const uint64_t* act_small;  // round-0 worklist (low 32 bits = vertex), count *nsmall
  const int* nsmall;
  uint32_t* wl[2];            // worklists of later rounds (slots of act_small), by parity
  unsigned long long* claim;  // [round] lists parked for the next round << 40 | tasks allocated
  unsigned int* cursor;       // [round] ctl claims
  unsigned int* ecursor;      // [round] eval claims
  uint32_t* state;            // per slot: alive[kP], touched[kP], kept count, task base
  uint2* tasks;               // (candidate id, kept-entry id)
  float* res;
  uint32_t cap;               // task array capacity
  uint2* itasks;              // per-warp scratch of the finishing launch
  float* ires;
  const uint64_t* off;
  const uint32_t* cnt;
  uint64_t* keys;
  Row row;
  uint32_t* post_cnt;
  uint32_t* pend_src;
  uint64_t* pend_key;
  unsigned long long* bcnt;
  unsigned long long* ctr;
  int round;
  int last;   // finish every claimed list in this launch
  int D;      // provisional entries per speculative round
  int l2pf;
};

__device__ __forceinline__ uint32_t lt_mask(uint32_t lane) { return (1u << lane) - 1u; }

template <bool kNA, bool kLast>
__global__ void __launch_bounds__(32 * kCtlWarps, kLast ? 2 : 3) k_bsp_ctl(BspArgs g) {
  __shared__ uint64_t s_wk[kCtlWarps][kRunMax];   // window / provisional keys, in list order
  __shared__ uint32_t s_wp[kCtlWarps][kRunMax];   // their positions
  __shared__ uint32_t s_to[kCtlWarps][kMaxD];     // speculative rounds: task base and need
  __shared__ uint32_t s_nm[kCtlWarps][kMaxD];     //   mask of candidates 1 .. D-1
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const uint32_t quad = lane >> 2, chain = lane & 3u;
  const uint32_t gw = blockIdx.x * kCtlWarps + wid;
  const Row row = g.row;
  const uint32_t count =
      g.round == 0 ? uint32_t(*g.nsmall) : uint32_t(g.claim[g.round - 1] >> 40);
  unsigned long long removed = 0, checks = 0, skips = 0, touched = 0, evals = 0;
  uint64_t* wk = s_wk[wid];
  uint32_t* wp = s_wp[wid];

  for (uint32_t sub = 0, it0 = 0;; ++sub) {
    if ((sub & 3u) == 0) {  // four lists per claim
      if (lane == 0) it0 = atomicAdd(g.cursor + g.round, 4u);
      it0 = __shfl_sync(0xffffffffu, it0, 0);
    }
    const uint32_t it = it0 + (sub & 3u);
    if (it >= count) {
      if ((sub & 3u) == 0) break;
      sub |= 3u;  // this claim is past the end: take the next one, which ends the loop
      continue;
    }
    const uint32_t slot = g.round == 0 ? it : g.wl[g.round & 1][it];
    uint32_t* st = g.state + uint64_t(slot) * kStateWords;
    uint32_t u, U;
    uint64_t base;
    if (g.round == 0) {
      u = uint32_t(g.act_small[slot]);
      base = g.off[u];
      U = g.cnt[u];
    } else {
      // one coalesced read of the record
      const uint32_t w = lane < kStateWords ? st[lane] : 0u;
      u = __shfl_sync(0xffffffffu, w, 2 * kP + 2);
      U = __shfl_sync(0xffffffffu, w, 2 * kP + 3);
      base = uint64_t(__shfl_sync(0xffffffffu, w, 2 * kP + 4)) |
             uint64_t(__shfl_sync(0xffffffffu, w, 2 * kP + 5)) << 32;
    }
    uint64_t* L = g.keys + base;
    auto walk = [&](auto np_tag) {
    constexpr int NP = decltype(np_tag)::value;
    uint64_t kk[NP];
    uint32_t M[NP], T[NP], F[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const uint32_t p = 32u * k + lane;
      kk[k] = p < U ? L[p] : 0ull;
      F[k] = __ballot_sync(0xffffffffu, p < U && key_fresh(kk[k]));
    }
    uint32_t nk, tb;
    if (g.round == 0) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const uint32_t p = 32u * k + lane;
        M[k] = __ballot_sync(0xffffffffu, p < U);
        T[k] = 0;
        if (g.l2pf && p < U) prefetch_row_l2(row(kk[k]), row.stride * 4u);
      }
      nk = 0;
      tb = kNone;
    } else {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        M[k] = st[k];
        T[k] = st[kP + k];
      }
      nk = st[2 * kP];
      tb = st[2 * kP + 1];
    }
    bool have_res = tb != kNone;  // the planned round's distances are in g.res + tb
    const float* rs = g.res + (have_res ? tb : 0u);

    for (;;) {
      // ------------------------------------------------------------ plan
      uint32_t arank[NP], frank[NP];
      uint32_t na = 0, nf = 0;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        arank[k] = na + __popc(M[k] & lt_mask(lane));
        na += __popc(M[k]);
        const uint32_t mf = M[k] & F[k];
        frank[k] = nf + __popc(mf & lt_mask(lane));
        nf += __popc(mf);
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
      uint32_t wr = run < kRunMax ? run : kRunMax;
      {
        const uint32_t cap = kRunBudget / (nf ? nf : 1u);
        if (wr > cap) wr = cap;
      }
      const bool run_round = wr >= 2;
      const uint32_t De = run_round ? wr : (na < uint32_t(g.D) ? na : uint32_t(g.D));
      // the window / the provisional entries: the first De alive positions
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if ((M[k] >> lane & 1u) && arank[k] < De) {
          wk[arank[k]] = kk[k];
          wp[arank[k]] = 32u * k + lane;
        }
      __syncwarp();
      // tasks of my positions
      uint32_t to[NP], nm[NP], lim[NP];
      uint32_t ntask = 0;
      if (run_round) {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const bool mine = M[k] & F[k] & (1u << lane);
          nm[k] = mine ? 1u : 0u;  // a fresh candidate: wr tasks
          lim[k] = wr;
          to[k] = frank[k] * wr;
        }
        ntask = nf * wr;
      } else {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const bool al = M[k] >> lane & 1u;
          const uint32_t ai = arank[k];
          const bool vf = key_fresh(kk[k]);
          lim[k] = al ? (ai < De ? ai : De) : 0u;
          uint32_t m = 0;
#pragma unroll
          for (int i = 0; i < kMaxD; ++i)
            if (uint32_t(i) < lim[k] && (key_fresh(wk[i]) || vf)) m |= 1u << i;
          nm[k] = m;
          uint32_t x = __popc(m);
          const uint32_t c0 = x;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= uint32_t(o)) x += y;
          }
          to[k] = ntask + x - c0;
          ntask += __shfl_sync(0xffffffffu, x, 31);
          if (al && ai >= 1 && ai < De) {
            s_to[wid][ai] = to[k];
            s_nm[wid][ai] = m;
          }
        }
      }
      // ------------------------------------------------- emit / evaluate
      if (!have_res && ntask) {
        uint2* tdst;
        bool park = false;
        uint32_t wl_pos = 0;
        if (kLast) {
          tdst = g.itasks + uint64_t(gw) * kInlineSlots;
        } else {
          // one atomic claims the task range and the next worklist's slot
          unsigned long long cl = 0;
          if (lane == 0) cl = atomicAdd(g.claim + g.round, (1ull << 40) | ntask);
          cl = __shfl_sync(0xffffffffu, cl, 0);
          wl_pos = uint32_t(cl >> 40);
          const uint64_t b = cl & ((1ull << 40) - 1);
          tb = uint32_t(b);
          tdst = g.tasks + b;
          park = true;
          if (b + ntask > g.cap) {
            // no room: null tasks over the part inside the array, retry next launch
            for (uint64_t t = b + lane; t < g.cap; t += 32) g.tasks[t] = make_uint2(0u, 0u);
            tb = kNone;
            ntask = 0;
          }
        }
        if (ntask) {
          evals += lane == 0 ? ntask : 0u;
          if (run_round) {
#pragma unroll
            for (int k = 0; k < NP; ++k)
              if (nm[k])
                for (uint32_t i = 0; i < wr; ++i)
                  tdst[to[k] + i] = make_uint2(key_id(kk[k]), key_id(wk[i]));
          } else {
#pragma unroll
            for (int k = 0; k < NP; ++k) {
              uint32_t t = to[k];
#pragma unroll
              for (int i = 0; i < kMaxD; ++i)
                if (nm[k] >> i & 1u) tdst[t++] = make_uint2(key_id(kk[k]), key_id(wk[i]));
            }
          }
        }
        if (park) {
          if (lane == 0) {
#pragma unroll
            for (int k = 0; k < NP; ++k) {
              st[k] = M[k];
              st[kP + k] = T[k];
            }
            st[2 * kP] = nk;
            st[2 * kP + 1] = tb;
            if (g.round == 0) {
              st[2 * kP + 2] = u;
              st[2 * kP + 3] = U;
              st[2 * kP + 4] = uint32_t(base);
              st[2 * kP + 5] = uint32_t(base >> 32);
            }
            g.wl[(g.round + 1) & 1][wl_pos] = slot;
          }
          break;
        }
        // finishing launch: this warp's quads evaluate the round
        __syncwarp();
        float* rdst = g.ires + uint64_t(gw) * kInlineSlots;
        for (uint32_t t0 = 0; t0 < ntask; t0 += 8) {
          const uint32_t ti = t0 + quad;
          const bool has = ti < ntask;
          const uint2 pr = __ldcg(tdst + (has ? ti : t0));
          const float dist = quad_l2<kNA>(row.xp + uint64_t(pr.x) * row.stride,
                                          row.xp + uint64_t(pr.y) * row.stride, chain, row.nblk,
                                          row.ntail);
          if (has && chain == 0) __stcg(rdst + ti, dist);
        }
        __syncwarp();
        rs = rdst;
      }
      // --------------------------------------------------------- resolve
      __syncwarp();
      uint32_t gone_m[NP], touch_m[NP];
      if (run_round) {
        uint32_t reach = 0;  // window entries checked by my candidates
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          bool gone = false;
          if (nm[k]) {
            const uint64_t vk = kk[k];
            const uint32_t q = 32u * k + lane;
            for (uint32_t i = 0; i < wr; ++i) {
              const float d = __ldcg(rs + to[k] + i);
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
          } else if ((M[k] >> lane & 1u) && arank[k] >= wr) {
            skips += wr;  // an old candidate behind the window
          }
          gone_m[k] = __ballot_sync(0xffffffffu, gone);
          touch_m[k] = __ballot_sync(0xffffffffu, nm[k] != 0);
        }
        reach = __reduce_max_sync(0xffffffffu, reach);
        if (lane == 0) skips += uint64_t(wr) * (wr - 1) / 2;  // the window among itself
        __syncwarp();
        if (lane < wr) L[nk + lane] = wk[lane];  // old already
        nk += wr;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          // the window leaves the alive set; its checked entries are touched
          const uint32_t inwin = __ballot_sync(0xffffffffu, (M[k] >> lane & 1u) && arank[k] < wr);
          const uint32_t tw = __ballot_sync(0xffffffffu, (M[k] >> lane & 1u) && arank[k] < reach);
          T[k] |= touch_m[k] | tw;
          M[k] &= ~(inwin | gone_m[k]);
        }
      } else {
        // fates of w_2 .. w_De, in list order (every lane, same result)
        uint32_t kept = 1u;
        for (uint32_t j = 1; j < De; ++j) {
          const float dj = key_dist(wk[j]);
          uint32_t t = s_to[wid][j];
          const uint32_t m = s_nm[wid][j];
          bool occl = false;
          for (uint32_t i = 0; i < j; ++i) {
            if (!(m >> i & 1u)) continue;
            const float d = __ldcg(rs + t);
            ++t;
            if ((kept >> i & 1u) && dj >= d) {
              occl = true;
              break;
            }
          }
          if (!occl) kept |= 1u << j;
        }
        uint32_t wtouch = 0;  // provisional entries with a counted check
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          bool gone = false, tch = false;
          const uint64_t vk = kk[k];
          const uint32_t q = 32u * k + lane;
          uint32_t t = to[k];
#pragma unroll
          for (int i = 0; i < kMaxD; ++i) {
            if (uint32_t(i) >= lim[k] || gone) continue;
            const bool nd = nm[k] >> i & 1u;
            const float d = nd ? __ldcg(rs + t) : 0.f;
            if (nd) ++t;
            if (!(kept >> i & 1u)) continue;  // not in the reference's kept list
            if (!nd) {
              ++skips;
              continue;
            }
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
          for (int i = 0; i < kMaxD; ++i)
            if (uint32_t(i) < De && (kept >> i & 1u)) {
              if (lane == 0) L[n2] = wk[i] & ~1ull;
              ++n2;
            }
          nk = n2;
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          uint32_t km = 0, tm = 0;
#pragma unroll
          for (int i = 0; i < kMaxD; ++i)
            if (uint32_t(i) < De && (wp[i] >> 5) == uint32_t(k)) {
              if (kept >> i & 1u) km |= 1u << (wp[i] & 31u);
              if (wtouch >> i & 1u) tm |= 1u << (wp[i] & 31u);
            }
          T[k] |= touch_m[k] | tm;
          M[k] &= ~(km | gone_m[k]);
        }
      }
      have_res = false;
      tb = kNone;
    }
    // na == 0 here iff the walk is complete (parked lists leave with na = 1)
    {
      uint32_t left = 0;
#pragma unroll
      for (int k = 0; k < NP; ++k) left |= M[k];
      if (left == 0) {
        if (lane == 0) {
          g.post_cnt[u] = nk;
          uint32_t tc = 0;
#pragma unroll
          for (int k = 0; k < NP; ++k) tc += __popc(T[k]);
          touched += tc;
        }
      }
    }
    };
    if (U <= 32)
      walk(std::integral_constant<int, 1>{});
    else if (U <= 64)
      walk(std::integral_constant<int, 2>{});
    else
      walk(std::integral_constant<int, kP>{});
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

// The flat evaluation: a quad per task, 8 tasks per warp claim.
template <bool kNA>
__global__ void __launch_bounds__(256, 4)
k_bsp_eval(const uint2* __restrict__ tasks, float* __restrict__ res,
           const unsigned long long* __restrict__ claim_p, uint32_t cap, unsigned int* cursor,
           Row row) {
  const uint32_t lane = lane_id(), quad = lane >> 2, chain = lane & 3u;
  const uint64_t want = *claim_p & ((1ull << 40) - 1);
  const uint32_t nt = want < cap ? uint32_t(want) : cap;
  for (;;) {
    uint32_t t0 = 0;
    if (lane == 0) t0 = atomicAdd(cursor, 8u);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (t0 >= nt) break;
    const uint32_t ti = t0 + quad;
    const bool has = ti < nt;
    const uint2 pr = tasks[has ? ti : t0];
    const float dist = quad_l2<kNA>(row.xp + uint64_t(pr.x) * row.stride,
                                    row.xp + uint64_t(pr.y) * row.stride, chain, row.nblk,
                                    row.ntail);
    if (has && chain == 0) res[ti] = dist;
  }
}

}  // namespace

// RNNDG_BSP = rounds per pass of the round-synchronous walk (0 = off; the
// last round finishes every remaining list inside its warp)
int bsp_rounds() {
  static const int v = [] {
    const char* e = std::getenv("RNNDG_BSP");
    const int x = e ? std::atoi(e) : 0;
    return x < 0 ? 0 : (x > kMaxRounds ? kMaxRounds : x);
  }();
  return gram_cap() ? 0 : v;  // the Gram walk's pending distances are not handled here
}

// lists of at most this many entries take it (RNNDG_BSP_LEN, <= 128)
uint32_t bsp_max_len() {
  static const uint32_t v = [] {
    const char* e = std::getenv("RNNDG_BSP_LEN");
    const int x = e ? std::atoi(e) : int(kBspMaxLen);
    return uint32_t(x < 1 ? 1 : (x > int(kBspMaxLen) ? int(kBspMaxLen) : x));
  }();
  return v;
}

void launch_bsp(rnndg_ctx* c, unsigned int* work, cudaStream_t stream, int spec, int l2pf) {
  const int R = bsp_rounds();
  const ScanConfig cfg = scan_config(c);
  const uint64_t n = c->nv;
  const int sms = sm_count(c);
  const unsigned ctl_grid = unsigned(sms) * 4u;
  const uint64_t ctl_warps = uint64_t(ctl_grid) * kCtlWarps;
  uint64_t cap = c->span * 2 + (1u << 20);
  if (cap > (1ull << 28)) cap = 1ull << 28;
  c->bsp_wl.ensure(2 * n);
  c->bsp_state.ensure(n * kStateWords);
  c->bsp_ctl.ensure(4 * (kMaxRounds + 2));
  c->bsp_tasks.ensure(cap);
  c->bsp_res.ensure(cap);
  c->bsp_itasks.ensure(ctl_warps * kInlineSlots);
  c->bsp_ires.ensure(ctl_warps * kInlineSlots);
  RNNDG_CUDA(cudaMemsetAsync(c->bsp_ctl.p, 0, 4 * (kMaxRounds + 2) * sizeof(unsigned int), stream));
  BspArgs a{};
  a.act_small = c->act_small.p;
  a.nsmall = reinterpret_cast<const int*>(work + 2);
  a.wl[0] = c->bsp_wl.p;
  a.wl[1] = c->bsp_wl.p + n;
  a.claim = reinterpret_cast<unsigned long long*>(c->bsp_ctl.p);
  a.cursor = c->bsp_ctl.p + 2 * (kMaxRounds + 2);
  a.ecursor = c->bsp_ctl.p + 3 * (kMaxRounds + 2);
  a.state = c->bsp_state.p;
  a.tasks = c->bsp_tasks.p;
  a.res = c->bsp_res.p;
  a.cap = uint32_t(cap);
  a.itasks = c->bsp_itasks.p;
  a.ires = c->bsp_ires.p;
  a.off = c->off.p;
  a.cnt = c->cnt.p;
  a.keys = c->key.p;
  a.row = Row{c->xp.p, cfg.stride, cfg.nblk, cfg.ntail};
  a.post_cnt = c->post_cnt.p;
  a.pend_src = c->pend_src.p;
  a.pend_key = c->pend_key.p;
  a.bcnt = c->partitioned ? nullptr : c->bcnt.p;
  a.ctr = c->counters.p;
  a.D = spec;
  // a round-0 bulk prefetch of every list's rows would pass the whole store
  // through L2 long before the evaluation reads it (measured: +9 ms on the
  // first ctl launch of a 1M-list pass); RNNDG_BSP_L2PF=1 turns it on anyway
  static const int bsp_l2pf = [] {
    const char* e = std::getenv("RNNDG_BSP_L2PF");
    return e ? std::atoi(e) : 0;
  }();
  a.l2pf = l2pf && bsp_l2pf;
  const bool na = cfg.stride * sizeof(float) >= 2048;
  auto kctl = na ? k_bsp_ctl<true, false> : k_bsp_ctl<false, false>;
  auto kfin = na ? k_bsp_ctl<true, true> : k_bsp_ctl<false, true>;
  auto kev = na ? k_bsp_eval<true> : k_bsp_eval<false>;
  static thread_local int ev_per_sm = 0;
  if (!ev_per_sm) {
    RNNDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ev_per_sm, kev, 256, 0));
    if (ev_per_sm < 1) ev_per_sm = 1;
  }
  for (int r = 0; r < R; ++r) {
    a.round = r;
    a.last = r == R - 1;
    if (a.last)
      kfin<<<ctl_grid, 32 * kCtlWarps, 0, stream>>>(a);
    else
      kctl<<<ctl_grid, 32 * kCtlWarps, 0, stream>>>(a);
    ++c->launches;
    if (r == R - 1) break;
    kev<<<unsigned(sms * ev_per_sm), 256, 0, stream>>>(a.tasks, a.res, a.claim + r, a.cap,
                                                       a.ecursor + r, a.row);
    ++c->launches;
  }
  RNNDG_CUDA(cudaGetLastError());
}

}  // namespace rnndg
