// gp_exh.cuh -- shared pieces of the two exhaustive evaluators (GP_EXHAUSTIVE):
// launch arguments, the per-set input contract, per-lane accumulation of the
// per-set outputs {n_sched, pi*, first rank, verdict hash} and their flush.
#pragma once
#include "gp_common.cuh"
#include "gp_enum.cuh"

namespace gp {

constexpr int kWarps = 8;        // warps per CTA
constexpr int kGrab = 16;        // items per queue grab
constexpr int kMaxL = 64;        // candidates per lane per item

struct ExhArgs {
  const int32_t *T, *D, *B, *cn, *cc, *fn, *fc, *group;
  const uint8_t *type, *valid;
  int32_t n_sets, n, M, n_groups;
  RankLayout L;
  uint64_t lo, hi;
  int64_t *per_set;
  uint32_t *bits;
  int64_t words;
  int64_t *counts;
  int32_t slot0, n_slots, setting;
  unsigned long long *stats;
  unsigned long long *work_counter;
  uint32_t flags;  // gp_exhaustive_opts.flags
  int32_t force_ranges;  // bit-sliced evaluator: walk okb range by range (env GP_EXH_RANGES, tests)
  const uint64_t *R;      // bit-sliced evaluator: run-prefix hash table [a0][run + 1] (or null)
  uint64_t r_stride;      // entries per row of R (total runs + 1)
  const uint64_t *CT;     // bit-sliced evaluator: corner table [rank] (k >= 3; or null)
  const uint64_t *FCT;    // bit-sliced evaluator: full corner table [rank] (or null)
  unsigned long long *memo_counter;  // bit-sliced memo pass: next set (or null: static stride)
  uint64_t run_base[kEnumMaxTasks + 2];  // first global run index of the allocations with k blocks
  uint32_t rgs_base[kEnumMaxTasks + 2];  // bit-sliced evaluator: first RGS index with k blocks
  uint64_t items_per_set, total_items;
  uint64_t item_base[kEnumMaxTasks + 2];
  uint32_t chunks[kEnumMaxTasks + 2];
  int32_t lane_L[kEnumMaxTasks + 2];
  uint32_t adm[8];  // f4 admissible sizes: bit (m-1) % 32 of word (m-1) / 32 (all ones: every size)
};

// f4 on the exhaustive path (reading B-9): a partition of an inadmissible size is
// not deployable, so every candidate using one is unschedulable.  The W tables carry that
// verdict: W = INT32_MAX at an inadmissible size fails every block at its first deadline
// (C > D, gp_edf.cuh shortcut 1), so the evaluators themselves are unchanged.
GP_DEV bool size_admissible(const uint32_t (&adm)[8], int m) {
  return (adm[(m - 1) >> 5] >> ((m - 1) & 31)) & 1u;
}
GP_DEV int32_t wcet_adm(const uint32_t (&adm)[8], int32_t B, int32_t c, int32_t f, int32_t m) {
  return size_admissible(adm, m) ? wcet_sat(B, c, f, m) : INT32_MAX;
}


// Per-set input contract (gpart.h): returns H = lcm(T) or -1.
GP_DEV int64_t set_contract(const ExhArgs &a, int64_t set) {
  const int n = a.n;
  int64_t H = 1;
  const int64_t cap = ((int64_t)1 << 31) / (n + 1);
  for (int i = 0; i < n; ++i) {
    const int64_t o = set * n + i;
    const int32_t T = a.T[o], D = a.D[o];
    if (T < 1 || D < 1 || D > T || a.B[o] < 1 || a.cn[o] < 1 || a.cc[o] < a.cn[o] ||
        a.fn[o] < 0 || a.fc[o] < a.fn[o])
      return -1;
    H = lcm_capped(H, T, cap - 1);
    if (H < 0) return -1;
  }
  return H;
}

// ---- per-lane accumulation ---------------------------------------------------
struct LaneAcc {
  uint32_t n = 0;
  int32_t pi = INT32_MAX;
  uint64_t first = ~0ull, hash = 0;
  uint64_t st_cand = 0, st_blocks = 0, st_tasks = 0;
  uint32_t st_events = 0;
};

GP_DEV void record_ok(LaneAcc &acc, uint64_t rank, int32_t sum, uint32_t *bits, uint64_t lo) {
  ++acc.n;
  acc.pi = min(acc.pi, sum);
  acc.first = rank < acc.first ? rank : acc.first;
  acc.hash += splitmix64(rank);
  if (bits) {
    const uint64_t off = rank - lo;
    atomicOr(bits + (off >> 5), 1u << (off & 31));
  }
}

GP_DEV void exh_flush(const ExhArgs &a, LaneAcc &acc, int64_t cur, int lane) {
  if (cur < 0) return;
  const uint32_t tot = (uint32_t)warp_sum_i32((int32_t)acc.n);
  const int32_t pi = warp_min_i32(acc.pi);
  uint64_t first = acc.first;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t v = __shfl_xor_sync(GP_FULL, first, o);
    first = v < first ? v : first;
  }
  const uint64_t h = warp_sum_u64(acc.hash);
  if (lane == 0 && tot > 0) {
    long long *ps = reinterpret_cast<long long *>(a.per_set + cur * 4);
    atomicAdd(reinterpret_cast<unsigned long long *>(ps + 0), (unsigned long long)tot);
    atomicMin(ps + 1, (long long)pi);
    atomicMin(ps + 2, (long long)first);
    atomicAdd(reinterpret_cast<unsigned long long *>(ps + 3), h);
  }
  acc.n = 0;
  acc.pi = INT32_MAX;
  acc.first = ~0ull;
  acc.hash = 0;
}

GP_DEV void exh_stats_flush(const ExhArgs &a, LaneAcc &acc, int lane) {
  if (!a.stats) return;
  const uint64_t c0 = warp_sum_u64(acc.st_cand), c1 = warp_sum_u64(acc.st_blocks);
  const uint64_t c2 = warp_sum_u64(acc.st_events), c3 = warp_sum_u64(acc.st_tasks);
  if (lane == 0) {
    atomicAdd(a.stats + 0, c0);
    atomicAdd(a.stats + 1, c1);
    atomicAdd(a.stats + 2, c2);
    atomicAdd(a.stats + 3, c3);
  }
}

// Lexicographic successor of s, stored REVERSED (sr[0] = last part) so the
// common step -- grow the last part while sum < M -- touches a fixed register.
// Otherwise bump the part with the fewest followers jj >= 1 whose followers
// have slack (sum of sr[0..jj-1] > jj) and reset its followers to 1.
template <int NT>
GP_DEV void next_sizes_rev(int M, int k, int32_t (&sr)[NT], int32_t &sum) {
  if (sum < M) {  // common: grow the last part
    sr[0] += 1;
    sum += 1;
    return;
  }
  if (k >= 2 && sr[0] > 1) {  // next: bump the second-to-last part, last := 1
    sum -= sr[0] - 2;
    sr[0] = 1;
    sr[1] += 1;
    return;
  }
  int prefix = 0, pick = -1;
#pragma unroll
  for (int jj = 1; jj < NT; ++jj) {
    prefix += sr[jj - 1];
    if (pick < 0 && jj < k && prefix > jj) pick = jj;
  }
  if (pick < 0) return;  // last candidate of this allocation (never stepped past)
  int ns = 0;
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    sr[i] = i < pick ? 1 : (i == pick ? sr[i] + 1 : sr[i]);
    ns += i < k ? sr[i] : 0;
  }
  sum = ns;
}

}  // namespace gp
