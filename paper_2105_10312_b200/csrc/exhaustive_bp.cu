// exhaustive_bp.cu -- the default GP_EXHAUSTIVE evaluator for n <= 8 tasks and
// M <= 32 SMs: bit-sliced candidate verdicts over memoised block verdicts.
//
// C.1.8: a candidate (pi, s) is schedulable iff every block S_j of pi passes
// the EDF processor-demand test (C.1.7) at its size s_j.  That block verdict
// depends only on (S_j, s_j) within a set, so it is computed ONCE per
// (subset, size) instead of once per (candidate, block):
//   k_exh_memo: per set, V[S] = bitmask over sizes (bit m-1 = S schedulable on
//   m SMs) for all 2^n - 1 task subsets S -- C3: at most 63 x 20 = 1,260 EDF tests
//   per set where the per-candidate evaluator runs ~2.3 million.  A pair (S, m) is
//   skipped only when some S - {i} fails at m (then S fails: fewer tasks, no more
//   conflicts); no monotonicity in m is assumed (that is f3's GP_THRESHOLD).
//   The words are stored subset-major (V[S][set]; row 0 = the set's H).
//   k_exh_bp: items = (32 sets, up to 16 allocations pi), candidates in the rank
//   order of C.1.6.  FULL CORNER: when every block word of pi is one bit range from
//   its first passing size lo_j + 1 through M - k + 1 (checked per (set, pi)), the
//   schedulable candidates of pi are the corner s >= lo + 1 of pi's simplex: count,
//   pi*, first rank in closed form, the hash one read of the full corner table FCT.
//   Otherwise: candidates of pi that differ in the last part only form a RUN
//   (last part 1 .. len); its verdicts are one word V_last & len_mask when the
//   other blocks pass, i.e. up to 32 candidate verdicts per word operation.
//   The warp walks pi's runs in lockstep -- outer parts by a successor, the
//   third-to-last part with its block's word shifted per step, the
//   second-to-last likewise per run -- visiting only the runs some lane's set
//   can pass, and records the set bits: count by popcount (or range length),
//   pi* and the first rank from the lowest bit, the verdict hash from a prefix
//   table of splitmix64 over the rank space (whole sweeps and blocks in closed
//   form from the run-prefix table R and the corner table CT), verdict bits with
//   word-level atomics (tests).  The tables depend on (n, M) only and are built
//   once per caller workspace (gp_exhaustive_opts.tables_key).
// Outputs are byte-identical to the per-candidate evaluator (GP_EX_PER_CANDIDATE
// selects that one, for A/B runs and parity).
#include <stdlib.h>

#include <type_traits>

#include "gp_common.cuh"
#include "gp_edf.cuh"
#include "gp_enum.cuh"
#include "gp_exh.cuh"

namespace gp {

constexpr int kBpMaxN = 8;   // tasks per set (2^8 subset words per set)
constexpr int kBpMaxM = 32;  // sizes per verdict word
#ifndef GP_MEMO_MINB
#define GP_MEMO_MINB 4  // memo-pass CTAs per SM the register budget targets (A/B)
#endif
#ifndef GP_MEMO_DENSITY
#define GP_MEMO_DENSITY 1  // memo tests: density <= 1 passes without the demand walk (exact)
#endif
#ifndef GP_MEMO_DYNAMIC
#define GP_MEMO_DYNAMIC 1  // memo pass: persistent grid, sets from a counter (0: static stride)
#endif
#ifndef GP_MEMO_PAIRS_PER_ROUND
#define GP_MEMO_PAIRS_PER_ROUND 1  // rank-order lists: two sizes per subset and round (A/B: -0.4 %)
#endif
#ifndef GP_MEMO_RANK_ORDER
#define GP_MEMO_RANK_ORDER 1  // memo: compacted tests ordered by their rank within the subset
#endif
#ifndef GP_BP_MINB
#define GP_BP_MINB 4  // main-pass CTAs per SM the register budget targets (A/B: -DGP_BP_MINB=n)
#endif
#ifndef GP_BP_UNROLL
#define GP_BP_UNROLL 2
#endif
#ifndef GP_BP_LANE_V
#define GP_BP_LANE_V 1  // closed sweeps: per-lane v ranges instead of the warp union (A/B: 3.69 -> 3.54 ms)
#endif
#ifndef GP_BP_CLOSED2
#define GP_BP_CLOSED2 1  // closed items whose block k-3 words are top ranges too (A/B)
#endif
#ifndef GP_BP_EAGER_LOADS
#define GP_BP_EAGER_LOADS 1  // closed sweeps: R reads before the bit test (A/B: 3.53 -> 3.45 ms)
#endif
#ifndef GP_BP_CORNER
#define GP_BP_CORNER 1  // closed2 blocks: one corner-table read instead of the sweep loop (A/B)
#endif
#ifndef GP_BP_FULLCORNER
#define GP_BP_FULLCORNER 1  // (set, allocation) pairs whose every block word is a top range: closed form (A/B)
#endif
#ifndef GP_BP_SWEEP_UNROLL
#define GP_BP_SWEEP_UNROLL 2  // closed-sweep loop unroll (A/B: 1, 2, 4 -> 2 by 1.3 %)
#endif
#ifndef GP_BP_CHUNK
#define GP_BP_CHUNK 16  // allocations per main-pass work item (A/B: 1, 4, 8, 16 -> 16)
#endif
constexpr uint32_t kBpChunk = GP_BP_CHUNK;
constexpr int kBpUnroll = GP_BP_UNROLL;
constexpr int kBpSweepUnroll = GP_BP_SWEEP_UNROLL;  // run loop unroll (A/B builds: -DGP_BP_UNROLL=n)

// 64-bit table entry at byte address base + 8 * idx (one IMAD.WIDE + one load)
GP_DEV uint64_t ld_u64(uint64_t base, uint32_t idx) {
  return __ldg(reinterpret_cast<const unsigned long long *>(base + 8ull * idx));
}

// ---- pre-pass: V[S][set] for every subset S, one warp per set --------------------
// Subsets are taken level by level in order of increasing size c (a per-CTA table).
// At level c only the pairs (S, m) whose subsets S - {i} all pass at m are tested
// (the others fail exactly, see the kernel): they are compacted per chunk of 32
// subsets by a warp scan and spread over the lanes, so every warp step tests
// subsets of one size c on their c tasks only (templated on c; no divergence
// between task counts).  C3: 54 % of the 1,260 pairs per set are decided this way.
// The verdict bits meet in a shared-memory word per subset and are written out once.
// The set's WCETs W_i(m, x) (C.1.3) are tabulated once per set in shared memory
// (n x 2 x M entries), so a test reads its tasks' WCETs instead of recomputing
// ceil(B/m) per (pair, task).
struct MemoTask {  // one task of the set: one 16-byte shared-memory load per use
  int32_t D, T, q;  // deadline, period, H / T
  float invD;       // 1 / D (the density shortcut of memo_test)
};

struct MemoWarp {
  uint32_t vs[1 << kBpMaxN];          // verdict word per subset
  int32_t wt[kBpMaxN * 2 * kBpMaxM];  // W_i(m, x) at [(i*2 + x)*32 + m-1], x = 1: conflict
  MemoTask tk[kBpMaxN];
  uint32_t cs[32], cd[32];            // the chunk's subsets and their W-column descriptors
  uint16_t list[32 * kBpMaxM];        // compacted (chunk position, size) pairs of one chunk
};

// EDF-PDC of the c tasks of a subset at size m (gp_edf.cuh shortcuts), lane-serial.
// dsc: the subset's tasks as W columns (i*2 + x_i, 4 bits each; x_i = another task of i's
// type in the subset).
template <int c>
GP_DEV bool memo_test(const MemoWarp &w, uint32_t dsc, int m, int32_t H, uint32_t &events) {
  int32_t C[c], D[c], T[c], q[c];
  float iD[c];
  bool bad = false;
#pragma unroll
  for (int a = 0; a < c; ++a) {
    const uint32_t col = (dsc >> (4 * a)) & 15u;
    const MemoTask tk = w.tk[col >> 1];
    C[a] = w.wt[col * kBpMaxM + m - 1];
    D[a] = tk.D;
    T[a] = tk.T;
    q[a] = tk.q;
    iD[a] = tk.invD;
    bad |= C[a] > D[a];
  }
  if (bad) return false;
  int32_t UH = 0;
#pragma unroll
  for (int a = 0; a < c; ++a) UH += C[a] * q[a];
  if (UH > H) return false;
#if GP_MEMO_DENSITY
  // density test (exact sufficient condition): for t >= D_i, floor((t - D_i)/T_i) + 1 <=
  // t / D_i because D_i <= T_i, so dbf(t) <= t * sum_i C_i / D_i <= t when the density is
  // <= 1.  Evaluated in float against 1 - 1e-5 (the float sum's relative error is below
  // 2^-20 for <= 8 terms), so a pass here is always a pass of the definition.
  float dens = 0.f;
#pragma unroll
  for (int a = 0; a < c; ++a) dens = fmaf((float)C[a], iD[a], dens);
  if (dens <= 0.99999f) return true;
#endif
  const int32_t lcut = pdc_cutoff<c>(C, D, T, q, H, UH);
  return pdc_walk<c>(C, D, T, lcut, events);
}

template <int NT, bool kStats>
__global__ void __launch_bounds__(256, GP_MEMO_MINB) k_exh_memo(const ExhArgs a, uint32_t *memo) {
  __shared__ MemoWarp mw_all[8];
  __shared__ uint8_t sorder[1 << kBpMaxN];  // subsets 1 .. 2^n - 1 by (size, value)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  MemoWarp &w = mw_all[wid];
  const int n = a.n, M = a.M;
  const int nsub = 1 << n;
  for (int S = threadIdx.x + 1; S < nsub; S += blockDim.x) {  // rank of S in the order
    const int c = __popc((unsigned)S);
    int r = 0;
    for (int S2 = 1; S2 < nsub; ++S2) {
      const int c2 = __popc((unsigned)S2);
      r += c2 < c || (c2 == c && S2 < S);
    }
    sorder[r] = (uint8_t)S;
  }
  __syncthreads();
  uint64_t st_tests = 0, st_tasks = 0;
  uint32_t st_events = 0;
  const uint32_t Mmask = M >= 32 ? ~0u : (1u << M) - 1u;
  // sets: dynamic (a warp grabs its next set from a counter: sets differ widely in work)
  // or a static grid stride
  auto next_set = [&](int64_t cur) -> int64_t {
    if (GP_MEMO_DYNAMIC && a.memo_counter) {
      unsigned long long s0 = 0;
      if (lane == 0) s0 = atomicAdd(a.memo_counter, 1ull);
      return (int64_t)__shfl_sync(GP_FULL, s0, 0);
    }
    return cur < 0 ? ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5
                   : cur + (((int64_t)gridDim.x * blockDim.x) >> 5);
  };
  for (int64_t set = next_set(-1); set < a.n_sets; set = next_set(set)) {
    const int64_t H = set_contract(a, set);
    uint32_t *V = memo + set;  // subset-major: word S of this set at V[S * n_sets]
    const size_t vstride = (size_t)a.n_sets;
    if (H <= 0) {
      if (lane == 0) V[0] = 0u;  // word 0: the set's input contract
      continue;
    }
    const int32_t H32 = (int32_t)H;
    for (int S = lane; S < nsub; S += 32) w.vs[S] = 0u;
    for (int i = 0; i < n; ++i) {  // W_i(m, x) table: lane = size (M <= 32)
      const int64_t o = set * n + i;
      const int32_t Bi = a.B[o], cni = a.cn[o], cci = a.cc[o], fni = a.fn[o], fci = a.fc[o];
      if (lane < M) {
        w.wt[(i * 2) * kBpMaxM + lane] = wcet_adm(a.adm, Bi, cni, fni, lane + 1);
        w.wt[(i * 2 + 1) * kBpMaxM + lane] = wcet_adm(a.adm, Bi, cci, fci, lane + 1);
      }
    }
    if (lane < n) {
      const int64_t o = set * n + lane;
      const int32_t Dl = a.D[o], Tl = a.T[o];
      w.tk[lane] = MemoTask{Dl, Tl, (int32_t)(H / Tl), __frcp_rn((float)Dl)};
    }
    const uint32_t mem = __ballot_sync(GP_FULL, lane < n && a.type[set * n + min(lane, n - 1)] == 1);
    __syncwarp();
    // Levels of increasing subset size c.  Level 1: a single task passes iff C <= D (no
    // conflict).  Level c >= 2 tests (S, m) only if every S - {i} passes at m:
    // a block's subset S' fails whenever S fails -- S' has fewer tasks and no more
    // conflicts (x_i(S') <= x_i(S)) and W_i(m, 1) >= W_i(m, 0) (cc >= cn, fc >= fn:
    // the input contract), so dbf_{S'} <= dbf_S pointwise at the deadlines of S' -- hence
    // a failing S - {i} decides V[S] bit m = 0 exactly (no monotonicity in m is used).
    // The surviving pairs of a chunk of up to 32 subsets are compacted and tested 32 at a
    // time with c uniform across the warp.
    for (int e = lane; e < n * M; e += 32) {
      const int i = e / M, m = e - i * M + 1;
      ++st_tests;
      ++st_tasks;
      if (w.wt[(i * 2) * kBpMaxM + m - 1] <= w.tk[i].D) atomicOr(&w.vs[1u << i], 1u << (m - 1));
    }
    __syncwarp();
    int lv0 = 0, nlv = n;  // first sorder index of the level, subsets in it (C(n, c))
    for (int c = 2; c <= n; ++c) {
      lv0 += nlv;
      nlv = nlv * (n - c + 1) / c;
      for (int ch = 0; ch < nlv; ch += 32) {
        const bool hs = ch + lane < nlv;
        const uint32_t S = hs ? sorder[lv0 + ch + lane] : 0u;
        uint32_t A = hs ? Mmask : 0u;
        for (uint32_t b = S; b; b &= b - 1u) A &= w.vs[S & ~(b & (0u - b))];
        // the subset's tasks as W columns (conflict flags resolved once per subset)
        uint32_t dsc = 0u;
        {
          uint32_t bits = S;
          for (int q4 = 0; bits; q4 += 4) {
            const int i = __ffs(bits) - 1;
            bits &= bits - 1u;
            const uint32_t same = ((mem >> i) & 1u) ? mem : ~mem;
            dsc |= ((uint32_t)(i * 2) + (__popc(S & same) > 1 ? 1u : 0u)) << q4;
          }
        }
        w.cs[lane] = S;
        w.cd[lane] = dsc;
        int total = 0;
#if GP_MEMO_RANK_ORDER
        // list order: every subset's smallest surviving size first (the tests at a subset's
        // schedulability boundary, where U is near 1 and the demand walks are long), then
        // every subset's second, ...: a warp step's 32 walks are of similar length
        {
          uint32_t b = A;
          const uint32_t lt = (1u << lane) - 1u;
#if GP_MEMO_PAIRS_PER_ROUND
          // two sizes per subset and round (half the ballot rounds; a round's entries are
          // each subset's next two surviving sizes)
          for (;;) {
            const uint32_t has = __ballot_sync(GP_FULL, b != 0u);
            if (!has) break;
            const uint32_t has2 = __ballot_sync(GP_FULL, (b & (b - 1u)) != 0u);
            if (b) {
              const int pos = total + __popc(has & lt) + __popc(has2 & lt);
              w.list[pos] = (uint16_t)(lane | ((__ffs(b) - 1) << 5));
              b &= b - 1u;
              if (b) {
                w.list[pos + 1] = (uint16_t)(lane | ((__ffs(b) - 1) << 5));
                b &= b - 1u;
              }
            }
            total += __popc(has) + __popc(has2);
          }
#else
          for (;;) {
            const uint32_t has = __ballot_sync(GP_FULL, b != 0u);
            if (!has) break;
            if (b) {
              w.list[total + __popc(has & lt)] = (uint16_t)(lane | ((__ffs(b) - 1) << 5));
              b &= b - 1u;
            }
            total += __popc(has);
          }
#endif
        }
#else
        {
          const int cntA = __popc(A);
          int incl = cntA;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(GP_FULL, incl, o);
            if (lane >= o) incl += v;
          }
          total = __shfl_sync(GP_FULL, incl, 31);
          int p = incl - cntA;
          for (uint32_t b = A; b; b &= b - 1u) w.list[p++] = (uint16_t)(lane | ((__ffs(b) - 1) << 5));
        }
#endif
        __syncwarp();
        for (int e = lane; e < total; e += 32) {
          const uint32_t ent = w.list[e];
          const uint32_t pos = ent & 31u;
          const int m = (int)(ent >> 5) + 1;
          const uint32_t d2 = w.cd[pos];
          ++st_tests;
          st_tasks += c;
          bool ok;
          switch (c) {
            case 2: ok = memo_test<2>(w, d2, m, H32, st_events); break;
            case 3: ok = memo_test<3>(w, d2, m, H32, st_events); break;
            case 4: ok = memo_test<4>(w, d2, m, H32, st_events); break;
            case 5: ok = memo_test<(NT >= 5 ? 5 : 2)>(w, d2, m, H32, st_events); break;
            case 6: ok = memo_test<(NT >= 6 ? 6 : 2)>(w, d2, m, H32, st_events); break;
            case 7: ok = memo_test<(NT >= 7 ? 7 : 2)>(w, d2, m, H32, st_events); break;
            default: ok = memo_test<(NT >= 8 ? 8 : 2)>(w, d2, m, H32, st_events); break;
          }
          if (ok) atomicOr(&w.vs[w.cs[pos]], 1u << (m - 1));
        }
        __syncwarp();
      }
    }
    __syncwarp();
    // row 0: the set's H (lcm of the periods, > 0: contract kept; 0: violated), which the
    // heuristics reuse (gpart.h gp_alloc_opts.memo)
    for (int S2 = lane; S2 < nsub; S2 += 32) V[S2 * vstride] = S2 == 0 ? (uint32_t)H32 : w.vs[S2];
    __syncwarp();
  }
  if constexpr (kStats) {  // (the timed instantiation carries no counters)
    const uint64_t t0 = warp_sum_u64(st_tests), t1 = warp_sum_u64(st_tasks);
    const uint64_t t2 = warp_sum_u64((uint64_t)st_events);
    if (lane == 0) {
      atomicAdd(a.stats + 1, (unsigned long long)t0);
      atomicAdd(a.stats + 2, (unsigned long long)t2);
      atomicAdd(a.stats + 3, (unsigned long long)t1);
    }
  }
}

// ---- RGS table: labels of every allocation, in rank order (k, then lex) -------
__global__ void k_exh_rgs_table(const ExhArgs a, uint32_t *rgs) {
  extern __shared__ __align__(16) uint32_t smem[];
  const EnumTables tab = build_enum_tables(smem, a.M, a.n);
  uint32_t total = 0;
  for (int k = 1; k <= a.L.kmax; ++k) total += (uint32_t)a.L.n_pi[k];
  for (uint32_t g = threadIdx.x; g < total; g += blockDim.x) {
    int k = 1;
    uint32_t base = 0;
    while (g >= base + (uint32_t)a.L.n_pi[k]) base += (uint32_t)a.L.n_pi[k++];
    rgs[g] = (uint32_t)unrank_rgs(tab, k, g - base);  // 4 bits per task, n <= 8
  }
}

// ---- verdict-hash prefix table: P[r] = sum_{x < r} splitmix64(x) mod 2^64 -------
// The hash of a set is sum of splitmix64(rank) over its schedulable ranks; a run
// segment of consecutive ranks [r0, r1) then contributes P[r1] - P[r0] (exact in
// mod-2^64 arithmetic), so the main pass needs two table reads per contiguous
// range of schedulable candidates instead of one splitmix64 per candidate.
constexpr int kScanBlock = 1024;
constexpr int kPpad = 32;  // slack entries after the hash prefix table
constexpr uint32_t kMaxHashTable = 1u << 24;  // ranks per set covered by the table

GP_DEV uint64_t block_incl_scan_u64(uint64_t v, uint64_t *wsum) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t u = __shfl_up_sync(GP_FULL, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(GP_FULL, w, o);
      if (lane >= o) w += u;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  return v + (wid > 0 ? wsum[wid - 1] : 0ull);
}

// pass 1: P[r + 1] = inclusive sum within the block; block totals
__global__ void __launch_bounds__(kScanBlock) k_hash_scan_local(uint64_t *P, uint64_t n_ranks,
                                                                uint64_t *btot) {
  __shared__ uint64_t wsum[32];
  const uint64_t r = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const uint64_t v = r < n_ranks ? splitmix64(r) : 0ull;
  const uint64_t incl = block_incl_scan_u64(v, wsum);
  if (r < n_ranks) P[r + 1] = incl;
  if (threadIdx.x == kScanBlock - 1) btot[blockIdx.x] = incl;
  if (blockIdx.x == 0 && threadIdx.x == 0) P[0] = 0ull;
}

// pass 2 (one block): exclusive scan of the block totals, in place
__global__ void __launch_bounds__(kScanBlock) k_hash_scan_blocks(uint64_t *btot, uint32_t nb) {
  __shared__ uint64_t wsum[32];
  uint64_t carry = 0;
  for (uint32_t b0 = 0; b0 < nb; b0 += kScanBlock) {
    const uint32_t b = b0 + threadIdx.x;
    const uint64_t v = b < nb ? btot[b] : 0ull;
    const uint64_t incl = block_incl_scan_u64(v, wsum);
    if (b < nb) btot[b] = carry + incl - v;
    __syncthreads();
    carry += wsum[31];
    __syncthreads();
  }
}

// pass 3: add each block's offset
__global__ void __launch_bounds__(kScanBlock) k_hash_scan_add(uint64_t *P, uint64_t n_ranks,
                                                              const uint64_t *btot) {
  const uint64_t r = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  if (r < n_ranks) P[r + 1] += btot[blockIdx.x];
}

// ---- run-prefix hash table: R[a0][g] = sum over the runs g' < g (global rank order) of
// the verdict-hash contribution a run makes when its schedulable candidates are exactly
// last parts a0 + 1 .. len (the run's top range): c_a0(g') = P[end(g')] - P[start(g') + a0]
// if a0 < len(g'), else 0 (mod 2^64).  With it, a whole sweep's consecutive live runs
// [lo, hi) of one set -- when that set's words make them exactly top ranges from a0 --
// add R[a0][hi] - R[a0][lo]: two reads per (set, sweep) instead of two per (set, run).
// Runs of an allocation with k blocks <-> (k-1)-subsets {c_0 < ... < c_{k-2}} of
// {1..M-1} in lexicographic order (prefix sums of the first k-1 parts); the run's first
// candidate has the s-index of the k-subset {c_0, ..., c_{k-2}, c_{k-2} + 1} of {1..M}.
GP_DEV uint32_t subset_lex_rank(const int32_t *c, int k, int M) {
  // rank of the k-subset c (ascending) among k-subsets of {1..M} in lexicographic order
  uint32_t r = 0;
  int prev = 0;
  for (int j = 0; j < k; ++j) {
    for (int v = prev + 1; v < c[j]; ++v) {  // subsets with a smaller j-th element
      uint64_t b = 1;  // C(M - v, k - 1 - j)
      const int nn = M - v, kk = k - 1 - j;
      for (int i = 1; i <= kk; ++i) b = b * (uint64_t)(nn - kk + i) / (uint64_t)i;
      r += (uint32_t)b;
    }
    prev = c[j];
  }
  return r;
}

__global__ void __launch_bounds__(256) k_run_contrib(const ExhArgs a, const uint64_t *P,
                                                     uint64_t *R, uint64_t total_runs) {
  const int M = a.M;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total_runs;
       g += (uint64_t)gridDim.x * blockDim.x) {
    int k = 1;
    while (k < a.L.kmax && g >= a.run_base[k + 1]) ++k;
    const uint64_t loc = g - a.run_base[k];
    const uint32_t nr = a.L.n_runs[k];
    const uint64_t p = loc / nr;
    uint32_t rho = (uint32_t)(loc - p * nr);
    // unrank rho -> (k-1)-subset of {1..M-1}, lexicographic
    int32_t c[kBpMaxN + 1];
    int prev = 0;
    for (int j = 0; j < k - 1; ++j) {
      int v = prev + 1;
      for (;;) {
        uint64_t b = 1;  // subsets with c_j = v: C(M - 1 - v, k - 2 - j)
        const int nn = M - 1 - v, kk = k - 2 - j;
        for (int i = 1; i <= kk; ++i) b = b * (uint64_t)(nn - kk + i) / (uint64_t)i;
        if (rho < b) break;
        rho -= (uint32_t)b;
        ++v;
      }
      c[j] = v;
      prev = v;
    }
    const int last = k >= 2 ? c[k - 2] : 0;
    c[k - 1] = last + 1;
    const uint32_t len = (uint32_t)(M - last);
    const uint64_t start = a.L.k_base[k] + p * a.L.per_pi[k] + subset_lex_rank(c, k, M);
    const uint64_t pe = P[start + len];
    for (int a0 = 0; a0 < M; ++a0)
      R[(uint64_t)a0 * a.r_stride + g + 1] = (uint32_t)a0 < len ? pe - P[start + a0] : 0ull;
  }
}

// in-place inclusive scan of each row R[a0][1 .. total] (row a0 = blockIdx.y), R[a0][0] = 0
__global__ void __launch_bounds__(kScanBlock) k_rows_scan_local(uint64_t *R, uint64_t stride,
                                                                uint64_t total, uint64_t *btot,
                                                                uint32_t nb) {
  __shared__ uint64_t wsum[32];
  uint64_t *row = R + (uint64_t)blockIdx.y * stride;
  const uint64_t r = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const uint64_t v = r < total ? row[r + 1] : 0ull;
  const uint64_t incl = block_incl_scan_u64(v, wsum);
  if (r < total) row[r + 1] = incl;
  if (threadIdx.x == kScanBlock - 1) btot[(uint64_t)blockIdx.y * nb + blockIdx.x] = incl;
  if (blockIdx.x == 0 && threadIdx.x == 0) row[0] = 0ull;
}

__global__ void __launch_bounds__(kScanBlock) k_rows_scan_blocks(uint64_t *btot, uint32_t nb) {
  __shared__ uint64_t wsum[32];
  uint64_t *bt = btot + (uint64_t)blockIdx.x * nb;
  uint64_t carry = 0;
  for (uint32_t b0 = 0; b0 < nb; b0 += kScanBlock) {
    const uint32_t b = b0 + threadIdx.x;
    const uint64_t v = b < nb ? bt[b] : 0ull;
    const uint64_t incl = block_incl_scan_u64(v, wsum);
    if (b < nb) bt[b] = carry + incl - v;
    __syncthreads();
    carry += wsum[31];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanBlock) k_rows_scan_add(uint64_t *R, uint64_t stride,
                                                              uint64_t total, const uint64_t *btot,
                                                              uint32_t nb) {
  const uint64_t r = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  if (r < total) R[(uint64_t)blockIdx.y * stride + r + 1] += btot[(uint64_t)blockIdx.y * nb + blockIdx.x];
}

// ---- corner table: CT[r] for every candidate r of an allocation with k >= 3 blocks.  Fix
// the outer parts s_0 .. s_{k-4} of r's allocation pi (a BLOCK of candidates: the last
// three parts (v, s_{k-2}, s_{k-1}) range over v + s_{k-2} + s_{k-1} <= N = M - sum(outer)).
// CT[r] = the verdict-hash sum of the candidates of r's block that dominate r in all three
// last parts (v' >= v, s'_{k-2} >= s_{k-2}, s'_{k-1} >= s_{k-1}): a corner of the block.
// When a set's verdict words make its schedulable candidates of a block exactly such a
// corner (the main pass's closed2 items: blocks k-3, k-2, k-1 pass exactly from sizes
// lo2+1, lo1+1, a0+1 up), the block adds CT at the corner's apex -- one read per (set,
// block) instead of two per (set, sweep).  Each entry is built from R exactly as the
// closed2 sweep loop sums it (the sweeps v = x+1 .. of the corner, their live runs
// [y, len0 - z) as R[z] differences), so the two give the same sum mod 2^64.
__global__ void __launch_bounds__(256) k_corner_table(const ExhArgs a, const uint64_t *R,
                                                      uint64_t *CT) {
  const int M = a.M;
  if (a.L.kmax < 3) return;
  const uint64_t r0 = a.L.k_base[3], r1 = a.L.total;
  for (uint64_t r = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1;
       r += (uint64_t)gridDim.x * blockDim.x) {
    int k = 3;
    while (k < a.L.kmax && r >= a.L.k_base[k + 1]) ++k;
    const uint64_t loc = r - a.L.k_base[k];
    const uint64_t p = loc / a.L.per_pi[k];
    uint32_t rho = (uint32_t)(loc - p * a.L.per_pi[k]);
    // unrank rho -> the k-subset c of {1..M} (prefix sums of the parts), lexicographic
    int32_t c[kBpMaxN + 1];
    int prev = 0;
    for (int j = 0; j < k; ++j) {
      int v = prev + 1;
      for (;;) {
        uint64_t b = 1;  // subsets with c_j = v: C(M - v, k - 1 - j)
        const int nn = M - v, kk = k - 1 - j;
        for (int i = 1; i <= kk; ++i) b = b * (uint64_t)(nn - kk + i) / (uint64_t)i;
        if (rho < b) break;
        rho -= (uint32_t)b;
        ++v;
      }
      c[j] = v;
      prev = v;
    }
    const int qsum = k >= 4 ? c[k - 4] : 0;                      // outer parts
    const int x = c[k - 3] - qsum - 1, y = c[k - 2] - c[k - 3] - 1, z = c[k - 1] - c[k - 2] - 1;
    const int L1 = M - qsum - 2;
    // run offset (within pi) of sweep v = x + 1's first run: the (k-1)-subset
    // {c_0 .. c_{k-4}, qsum + v, qsum + v + 1} of {1..M-1}
    int32_t cc[kBpMaxN + 1];
    for (int j = 0; j < k - 3; ++j) cc[j] = c[j];
    cc[k - 3] = qsum + x + 1;
    cc[k - 2] = qsum + x + 2;
    uint32_t roff = subset_lex_rank(cc, k - 1, M - 1);
    const uint64_t *row = R + (uint64_t)z * a.r_stride + a.run_base[k] + p * a.L.n_runs[k];
    int len0 = L1 - x;
    uint64_t h = 0;
    for (int sp = len0 - z - y; sp >= 1; --sp) {
      h += row[roff + (uint32_t)(len0 - z)] - row[roff + (uint32_t)y];
      roff += (uint32_t)len0;
      --len0;
    }
    CT[r] = h;
  }
}

// ---- full corner table: FCT[r] = the verdict-hash sum of the candidates of r's allocation pi
// that dominate r in EVERY part (s' >= s componentwise, sum(s') <= M).  When a set's verdict
// word of every block of pi is one bit range from its first passing size lo_j up to the
// largest size a part can take (M - k + 1) -- checked per (set, allocation) in the main pass,
// never assumed -- the set's schedulable candidates of pi are exactly that corner with apex
// s_j = lo_j + 1: n_sched = C(M - sum lo, k), pi* = sum(lo) + k, the first rank is the apex's
// and the hash is FCT at the apex -- one read per (set, allocation).
// Built as k suffix scans over pi's simplex: level 0 = splitmix64(r); pass j (= 1 .. kmax)
// scans dimension i = k - j of every allocation with k >= j, one thread per CHAIN (the
// candidates that differ in part i only), walking part i downwards and summing in place.
// The candidate ranks come from the lex rank of the prefix-sum k-subset c of {1..M}:
// rank(c) = C(M, k) - 1 - sum_j C(M - c_j, k - j).
struct Binom {  // C(a, b), 0 <= a <= kBpMaxM, 0 <= b <= kBpMaxN (shared memory)
  uint32_t t[(kBpMaxM + 1) * (kBpMaxN + 1)];
  GP_DEV void build() {
    for (int e = threadIdx.x; e < (kBpMaxM + 1) * (kBpMaxN + 1); e += blockDim.x) {
      const int aa = e / (kBpMaxN + 1), bb = e - aa * (kBpMaxN + 1);
      uint64_t c = 1;
      for (int i = 1; i <= bb; ++i) c = c * (uint64_t)(aa - bb + i) / (uint64_t)i;
      t[e] = bb > aa ? 0u : (uint32_t)c;
    }
  }
  GP_DEV uint32_t operator()(int aa, int bb) const {
    return (aa < 0 || bb > aa) ? 0u : t[aa * (kBpMaxN + 1) + bb];
  }
  // 0 <= bb <= kBpMaxN, aa <= kBpMaxM: the table holds C(aa, bb) = 0 for bb > aa, and a
  // negative aa reads C(0, bb) (0 for bb >= 1; callers pass bb >= 1 there)
  GP_DEV uint32_t at(int aa, int bb) const { return t[max(aa, 0) * (kBpMaxN + 1) + bb]; }
};

__global__ void __launch_bounds__(256) k_fct_init(uint64_t *F, uint64_t n_ranks) {
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_ranks;
       r += (uint64_t)gridDim.x * blockDim.x)
    F[r] = splitmix64(r);
}

__global__ void __launch_bounds__(256) k_fct_pass(const ExhArgs a, uint64_t *F, int j) {
  __shared__ Binom C;
  C.build();
  __syncthreads();
  const int M = a.M;
  const uint64_t g0 = a.run_base[j], total = a.run_base[a.L.kmax + 1];
  for (uint64_t g = g0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    int k = j;
    while (k < a.L.kmax && g >= a.run_base[k + 1]) ++k;
    const uint64_t loc = g - a.run_base[k];
    const uint32_t nr = a.L.n_runs[k];
    const uint64_t p = loc / nr;
    uint32_t rho = (uint32_t)(loc - p * nr);
    // the chain's other parts: the (k-1)-subset d of {1..M-1} (their prefix sums), lex
    int32_t d[kBpMaxN + 1];
    int prev = 0;
    for (int m = 0; m < k - 1; ++m) {
      int v = prev + 1;
      while (rho >= C(M - 1 - v, k - 2 - m)) {
        rho -= C(M - 1 - v, k - 2 - m);
        ++v;
      }
      d[m] = v;
      prev = v;
    }
    const int i = k - j;                          // the scanned part
    const int dtot = k >= 2 ? d[k - 2] : 0;       // sum of the other parts
    const int dpre = i > 0 ? d[i - 1] : 0;        // sum of the parts before i
    // the part of the rank that does not depend on part i's value t
    uint32_t fixed = C(M, k) - 1u;
    for (int m = 0; m < i; ++m) fixed -= C(M - d[m], k - m);
    const uint64_t base = a.L.k_base[k] + p * (uint64_t)a.L.per_pi[k];
    uint64_t acc = 0;
    for (int t = M - dtot; t >= 1; --t) {
      uint32_t rk = fixed - C(M - (dpre + t), k - i);
      for (int m = i + 1; m < k; ++m) rk -= C(M - (d[m - 1] + t), k - m);
      acc += F[base + rk];
      F[base + rk] = acc;
    }
  }
}

// ---- main pass: bit-sliced verdicts over runs, lane = task set -------------------
// item = (group of 32 consecutive sets, allocation pi), items in k-DESCENDING
// groups (the largest allocations first, small ones fill the tail).  The run
// structure of pi -- prefixes in lexicographic order, run lengths, ranks --
// depends only on (k, M), so the whole warp walks it in lockstep (uniform
// control flow, no divergent successor) while each lane applies its own set's
// verdict words.
//
// Specialised on the call's shape: kWin (a rank window narrower than the whole
// space), kHash (0: no hash, 1: prefix table P, 2: splitmix64 per schedulable
// rank) and kBits (verdict bits wanted), so the common call carries none of
// the other modes' per-run checks.
//
// Per sweep (the last prefix part grows, runs i = 0 .. steps-1 of lengths
// len0 - i), run i can hold a schedulable candidate of a lane's set only if
// bit i of w1 (block k-2 at size pr[0] + i) is set and len0 - i exceeds the
// lowest set bit of the last block's word; the warp walks only the runs
// between the lowest such i and the highest over its lanes (warp min/max),
// skipping the others in closed form -- their verdict words are zero.
//
// Verdict hash: a run's schedulable candidates are the set bits of
// okb = V_last & len_mask (rank rk + b for bit b).  When the last block's word
// of every lane's set is one contiguous bit range (checked per item, never
// assumed), okb is one contiguous range [fb, e) and adds P[rk + e] - P[rk + fb];
// otherwise the contiguous ranges of okb are walked one by one.
template <bool kWin, int kHash, bool kBits, bool kStats>
__global__ void __launch_bounds__(kWarps * 32, GP_BP_MINB)
    k_exh_bp(const ExhArgs a, const uint32_t *memo, const uint32_t *rgs, const uint64_t *P) {
  const int n = a.n, M = a.M;
  const int lane = threadIdx.x & 31;
  const int nsub = 1 << n;
  // per-lane (= per-set) accumulators
  uint32_t acc_n = 0;
  int32_t acc_pi = INT32_MAX;
  uint64_t acc_first = ~0ull, acc_hash = 0, st_cand = 0, st_runs = 0, st_live = 0;
  uint64_t st_sweeps = 0, st_live_closed = 0, st_ct_blocks = 0, st_ct_sweeps = 0;
  uint64_t st_fc_items = 0, st_fc_blocks = 0;
  __shared__ Binom binom_s;  // C(a, b) for the full-corner closed forms
  binom_s.build();
  __syncthreads();
  auto bn = [&](int aa, int bb) -> uint32_t { return binom_s(aa, bb); };
  int64_t cur_g = -1, set = -1;
  const uint32_t *memo_set = memo;             // this lane's set's column of the memo words
  const size_t memo_stride = (size_t)a.n_sets;  // words between subsets' rows
  bool lane_ok = false;
  auto flush = [&]() {
    if (lane_ok && acc_n > 0) {
      long long *ps = reinterpret_cast<long long *>(a.per_set + set * 4);
      atomicAdd(reinterpret_cast<unsigned long long *>(ps + 0), (unsigned long long)acc_n);
      atomicMin(ps + 1, (long long)acc_pi);
      atomicMin(ps + 2, (long long)acc_first);
      if (kHash) atomicAdd(reinterpret_cast<unsigned long long *>(ps + 3), acc_hash);
    }
    acc_n = 0;
    acc_pi = INT32_MAX;
    acc_first = ~0ull;
    acc_hash = 0;
  };
  for (;;) {
    uint64_t base = 0;
    if (lane == 0) base = atomicAdd(a.work_counter, 1ull);  // items are large: one per grab
    base = __shfl_sync(GP_FULL, base, 0);
    if (base >= a.total_items) break;
    const uint64_t it = base;
    int k = a.L.kmax;  // groups k = kmax, ..., 1; item_base[k] = end of group k
    while (k > 1 && it >= a.item_base[k]) --k;
    const uint64_t local = it - (k == a.L.kmax ? 0 : a.item_base[k + 1]);
    const uint32_t npi = (uint32_t)a.L.n_pi[k];
    const uint32_t nch = (npi + kBpChunk - 1) / kBpChunk;  // chunks of allocations with k blocks
    const int64_t grp = (int64_t)(local / nch);
    const uint32_t p0 = (uint32_t)(local - (uint64_t)grp * nch) * kBpChunk;
    const uint32_t p1 = min(npi, p0 + kBpChunk);
    for (uint32_t p = p0; p < p1; ++p) {
    const uint32_t labels = rgs[a.rgs_base[k] + p];
    const int myb = lane < n ? (int)((labels >> (4 * lane)) & 15u) : -1;
    if (grp != cur_g) {
      flush();
      cur_g = grp;
      set = grp * 32 + lane;
      lane_ok = set < a.n_sets && memo[set] != 0;  // input contract (word 0)
      memo_set = memo + (lane_ok ? set : 0);
    }
    const uint32_t per_pi = (uint32_t)a.L.per_pi[k];
    const uint64_t rank_pi = a.L.k_base[k] + (uint64_t)p * per_pi;
    // the full corner table at pi's first rank
    const uint64_t fct_addr =
        (GP_BP_FULLCORNER && !kWin && kHash == 1 && !kBits && a.FCT) ? reinterpret_cast<uint64_t>(a.FCT) + 8ull * rank_pi
                                                                     : 0ull;
    bool full = true;
    if constexpr (kWin) {
      if (rank_pi >= a.hi || rank_pi + per_pi <= a.lo) continue;
      full = rank_pi >= a.lo && rank_pi + per_pi <= a.hi;
    }
    // block task masks of pi (warp-uniform ballots) -> this lane's set's
    // verdict words, reversed: Vr[jj] = V[set][S_{k-1-jj}]
    // (compile-time index jj, runtime block k-1-jj: no register-array indexing)
    uint32_t Vr[kBpMaxN];
    bool dead = true;
    // the verdict words, the dead check and the full corner, specialised on k (compile-time
    // loop bounds); returns true when no lane has anything left in this item
    auto front = [&](auto kc) -> bool {
      constexpr int K = decltype(kc)::value;
#pragma unroll
      for (int jj = 0; jj < kBpMaxN; ++jj) {
        Vr[jj] = 0u;
        if (jj < K) {
          const uint32_t bm = __ballot_sync(GP_FULL, myb == K - 1 - jj);
          if (lane_ok) Vr[jj] = memo_set[bm * memo_stride];  // coalesced: lane = set
        }
      }
      if (!__any_sync(GP_FULL, lane_ok)) return true;
      // candidates of pi inside the rank window (all evaluated, bit-sliced)
      if (lane_ok) {
        if constexpr (kWin) {
          const uint64_t w_lo = max(a.lo, rank_pi), w_hi = min(a.hi, rank_pi + per_pi);
          st_cand += w_hi > w_lo ? w_hi - w_lo : 0;
        } else {
          st_cand += per_pi;
        }
      }
      // a block never schedulable at any size: every candidate of pi fails
      dead = !lane_ok;
#pragma unroll
      for (int jj = 0; jj < K; ++jj) dead |= Vr[jj] == 0u;
      if (__all_sync(GP_FULL, dead)) return true;
#if GP_BP_FULLCORNER
      if constexpr (!kWin && !kBits && kHash != 2) {
        if ((kHash == 0 || a.FCT) && !a.force_ranges && !(a.flags & GP_EX_NO_FULL_CORNER)) {
          // full corner: when every block's word is one bit range from its first passing
          // size lo_j + 1 through the largest size a part can take (M - k + 1) -- checked
          // here per (set, allocation) -- the set's schedulable candidates of pi are the
          // corner with apex s_j = lo_j + 1 of pi's simplex: count, pi*, first rank in closed
          // form, the hash one read of the full corner table at the apex (lanes done here
          // skip the rest)
          bool corner = !dead;
          int csum = 0;      // prefix sums of the apex parts, block order j = 0 .. k-1
          uint32_t sub = 0;  // sum_j C(M - c_j, k - j): the apex's lex rank complement
#pragma unroll
          for (int jj = K - 1; jj >= 0; --jj) {  // block j = K - 1 - jj
            const uint32_t V = Vr[jj];
            const int lo = V ? __ffs(V) - 1 : 0;
            const int nb = M - K + 1 - lo;
            const uint32_t mk = nb >= 32 ? ~0u : (nb <= 0 ? 0u : (1u << nb) - 1u);
            corner &= ((V >> lo) & mk) == mk;
            csum += lo + 1;
            sub += binom_s.at(M - csum, jj + 1);  // (csum > M: unused, see below)
          }
          if (corner) {
            if (csum <= M) {  // the apex fits: C(M - sum lo, k) candidates
              acc_n += bn(M - csum + K, K);
              acc_pi = min(acc_pi, csum);
              const uint32_t off = bn(M, K) - 1u - sub;
              acc_first = min(acc_first, rank_pi + off);
              if constexpr (kHash == 1) acc_hash += ld_u64(fct_addr, off);
              if constexpr (kStats) {
                ++st_fc_items;
                st_fc_blocks += (uint64_t)K;
              }
            }
            dead = true;
          }
          if (__all_sync(GP_FULL, dead)) return true;
        }
      }
#endif
      return false;
    };
    bool skip;
    switch (k) {  // warp-uniform
      case 1: skip = front(std::integral_constant<int, 1>{}); break;
      case 2: skip = front(std::integral_constant<int, 2>{}); break;
      case 3: skip = front(std::integral_constant<int, 3>{}); break;
      case 4: skip = front(std::integral_constant<int, 4>{}); break;
      case 5: skip = front(std::integral_constant<int, 5>{}); break;
      case 6: skip = front(std::integral_constant<int, 6>{}); break;
      case 7: skip = front(std::integral_constant<int, 7>{}); break;
      default: skip = front(std::integral_constant<int, 8>{}); break;
    }
    if (skip) continue;
    const int kp = k - 1;
    const uint32_t V0 = dead ? 0u : Vr[0];
    // lowest size index of the last block that can pass; contiguity of its word
    const int a0 = V0 ? __ffs(V0) - 1 : 32;
    const uint32_t v0s = V0 >> (a0 & 31);
    const bool contig = !a.force_ranges && __all_sync(GP_FULL, (v0s & (v0s + 1u)) == 0u);
    const int b0 = a0 + __popc(V0);  // end of the last block's range when contiguous
    // the last block's word reaches size M in every live lane: a non-zero okb is then the
    // range [a0, len) -- its end is the next run's start, the same rank in every lane
    const bool top = contig && __all_sync(GP_FULL, V0 == 0u || b0 >= M);
    // hash-table byte addresses of pi's first rank (+ a0 in this lane; the table has
    // kPpad entries of slack for lanes whose a0 runs past a run's end)
    const uint64_t pu_addr = reinterpret_cast<uint64_t>(P) + 8ull * rank_pi;
    const uint64_t pl_addr = pu_addr + 8ull * (uint32_t)(a0 & 31);
    // this lane's row of the run-prefix table at pi's first run (closed-form sweeps)
    const uint64_t r_addr =
        (!kWin && kHash == 1 && !kBits && a.R)
            ? reinterpret_cast<uint64_t>(a.R) +
                  8ull * ((uint64_t)(a0 & 31) * a.r_stride + a.run_base[k] + (uint64_t)p * a.L.n_runs[k])
            : 0ull;
    // the corner table at pi's first rank (closed2 blocks)
    const uint64_t ct_addr =
        (GP_BP_CORNER && !kWin && kHash == 1 && !kBits && a.CT) ? reinterpret_cast<uint64_t>(a.CT) + 8ull * rank_pi
                                                                : 0ull;
    uint32_t *bits = nullptr;
    if constexpr (kBits) bits = lane_ok ? a.bits + set * a.words : nullptr;
    uint32_t first_off = UINT32_MAX;  // s-index of pi's first schedulable candidate
    // One sweep: every prefix part but s_{k-2} fixed (their blocks pass in the
    // lanes where w1 != 0), s_{k-2} = 1 + i for runs i = 0 .. steps-1, run i with
    // last part 1 .. len0 - i.  w1 bit i: block k-2 passes at size 1 + i.
    // `off` = s-index (within pi) of the sweep's first candidate.
    auto sweep = [&](int len0, int steps, uint32_t w1, uint32_t off, uint32_t roff) {
      // runs [i_lo, i_hi) can hold schedulable candidates of some lane's set
      const int lo_l = w1 ? __ffs(w1) - 1 : steps;
      const int hi_l = w1 ? min(steps, len0 - a0) : 0;
      if constexpr (!kWin && kHash != 2 && !kBits) {
        // the whole sweep at once: when in every lane the live runs are exactly
        // [lo_l, hi_l) (block k-2's word has every bit of that range) and each live run's
        // schedulable candidates are its top range a0+1 .. len (`top`), the lane's
        // count, pi*, first rank and hash follow in closed form, the hash from two reads
        // of the run-prefix table R (checked per sweep, never assumed; otherwise the runs
        // are walked one by one below)
        const int span = hi_l - lo_l;
        const bool fits = span <= 0 || ((w1 >> lo_l) & ((span >= 32 ? 0u : 1u << span) - 1u)) ==
                                           ((span >= 32 ? 0u : 1u << span) - 1u);
        if (top && (kHash == 0 || a.R) && __all_sync(GP_FULL, fits)) {
          if (span > 0) {
            if constexpr (kStats) {
              ++st_sweeps;
              st_live_closed += (uint64_t)span;
            }
            // run i holds len0 - i - a0 schedulable candidates (last part a0+1 .. len0-i)
            acc_n += (uint32_t)(span * (len0 - a0) - (((lo_l + hi_l - 1) * span) >> 1));
            acc_pi = min(acc_pi, M - len0 + 1 + lo_l + a0);
            // sweeps are visited in rank order: the lane's first live one holds its first rank
            if (first_off == UINT32_MAX)
              first_off = off + (uint32_t)(lo_l * len0 - ((lo_l * (lo_l - 1)) >> 1) + a0);
            if constexpr (kHash == 1)
              acc_hash += ld_u64(r_addr, roff + (uint32_t)hi_l) - ld_u64(r_addr, roff + (uint32_t)lo_l);
          }
          return;
        }
      }
      const int i_lo = (int)__reduce_min_sync(GP_FULL, (unsigned)lo_l);
      const int i_hi = (int)__reduce_max_sync(GP_FULL, (unsigned)max(hi_l, 0));
      if (i_lo >= i_hi) return;
      if constexpr (kStats) st_runs += lane_ok ? (uint64_t)(i_hi - i_lo) : 0;
      int len = len0 - i_lo;
      uint32_t o2 = off + (uint32_t)(i_lo * len0 - i_lo * (i_lo - 1) / 2);
      uint32_t lmask = len >= 32 ? ~0u : (1u << len) - 1u;
      w1 >>= i_lo;
      const int psb = M - len0 + 1;  // (sum of the prefix parts but s_{k-2}) + 1 + 1
      if constexpr (!kWin && kHash != 2) {
        if (top) {
          // per live run: n += len - a0, hash += P[next run start] - P[run start + a0]
#pragma unroll kBpUnroll
          for (int i = i_lo; i < i_hi; ++i) {
            const uint32_t o2n = o2 + (uint32_t)len;
            const uint32_t okb = V0 & lmask & (0u - (w1 & 1u));
            if (okb) {
              if constexpr (kStats) ++st_live;
              acc_n += (uint32_t)(len - a0);
              acc_pi = min(acc_pi, psb + i + a0);
              first_off = min(first_off, o2 + (uint32_t)a0);
              if constexpr (kHash == 1) acc_hash += ld_u64(pu_addr, o2n) - ld_u64(pl_addr, o2);
              if constexpr (kBits) {
                const uint64_t ob = rank_pi + o2 + (uint64_t)a0;
                const uint32_t w2 = okb >> a0;
                const uint32_t sh = (uint32_t)(ob & 31u);
                atomicOr(bits + (ob >> 5), w2 << sh);
                if (sh && (w2 >> (32u - sh))) atomicOr(bits + (ob >> 5) + 1, w2 >> (32u - sh));
              }
            }
            o2 = o2n;
            len -= 1;
            lmask >>= 1;
            w1 >>= 1;
          }
          return;
        }
      }
      for (int i = i_lo; i < i_hi; ++i) {
        uint32_t okb = V0 & lmask & (0u - (w1 & 1u));
        if constexpr (kWin) {
          if (!full) {  // rank window [lo, hi) (warp-uniform)
            const uint64_t rk = rank_pi + o2;
            if (rk < a.lo) okb &= a.lo - rk >= (uint64_t)len ? 0u : ~0u << (uint32_t)(a.lo - rk);
            if (rk + (uint64_t)len > a.hi) okb &= a.hi <= rk ? 0u : (1u << (uint32_t)(a.hi - rk)) - 1u;
          }
        }
        if (okb) {
          if constexpr (kStats) ++st_live;
          const int fb = __ffs(okb) - 1;
          acc_pi = min(acc_pi, psb + i + fb);
          first_off = min(first_off, o2 + (uint32_t)fb);
          if constexpr (kHash == 1) {
            const uint64_t *Pr = P + rank_pi + o2;
            if (contig) {  // one range [fb, e)
              const int e = 32 - __clz(okb);
              acc_n += (uint32_t)(e - fb);
              acc_hash += Pr[e] - Pr[fb];
            } else {  // contiguous ranges of schedulable ranks: P[r1] - P[r0]
              acc_n += __popc(okb);
              uint32_t w = okb;
              do {
                const int c0 = __ffs(w) - 1;
                const uint32_t t = ~(w >> c0);
                const int c1 = t ? c0 + __ffs(t) - 1 : 32;
                acc_hash += Pr[c1] - Pr[c0];
                w &= c1 >= 32 ? 0u : ~0u << c1;
              } while (w);
            }
          } else {
            acc_n += __popc(okb);
            if constexpr (kHash == 2) {
              const uint64_t rk = rank_pi + o2;
              uint32_t w = okb;
              do {
                const int b = __ffs(w) - 1;
                w &= w - 1u;
                acc_hash += splitmix64(rk + (uint64_t)b);
              } while (w);
            }
          }
          if constexpr (kBits) {  // verdict bits of the run, word-level
            const uint64_t ob = rank_pi + o2 - a.lo + (uint64_t)fb;
            const uint32_t w2 = okb >> fb;
            const uint32_t sh = (uint32_t)(ob & 31u);
            atomicOr(bits + (ob >> 5), w2 << sh);
            if (sh && (w2 >> (32u - sh))) atomicOr(bits + (ob >> 5) + 1, w2 >> (32u - sh));
          }
        }
        o2 += (uint32_t)len;
        len -= 1;
        lmask >>= 1;
        w1 >>= 1;
      }
    };
    if (kp == 0) {  // k = 1: one run, the single block at 1 .. M
      sweep(M, 1, dead ? 0u : 1u, 0u, 0u);
    } else if (kp == 1) {  // k = 2: one sweep over s_0
      sweep(M - 1, M - 1, dead ? 0u : Vr[1], 0u, 0u);
    } else {
      // k >= 3: the outer parts s_0 .. s_{k-4} (reversed: q[0] = s_{k-4}) in
      // lexicographic order (sum <= M - 3 leaves room for s_{k-3}, s_{k-2}, s_{k-1});
      // for each, s_{k-3} = v walks its sweeps with the verdict word of block k-3
      // shifted one bit per step, skipping v's no lane can pass at (the skipped
      // sweeps' candidates are counted in closed form: a sweep of len0 = L holds
      // L(L+1)/2 candidates, consecutive sweeps L, L-1, ... sum to tetrahedral numbers)
      const int k2 = kp - 2;
      // closed items: the closed-form sweep applies to every sweep of every lane -- block
      // k-2's word is one bit range from lo1 reaching the largest size a run can need
      // (bit M-2), and the last block's words are top ranges (checked per item)
      int lo1 = 0;
      bool c1 = true;
      if (!dead && Vr[1]) {
        lo1 = __ffs(Vr[1]) - 1;
        const int need = M - 1 - lo1;  // bits lo1 .. M-2
        const uint32_t mk = need >= 32 ? ~0u : (need <= 0 ? 0u : (1u << need) - 1u);
        c1 = ((Vr[1] >> lo1) & mk) == mk;
      }
      const bool closed = (!kWin && kHash != 2 && !kBits) && top && (kHash == 0 || a.R != nullptr) &&
                          !a.force_ranges && __all_sync(GP_FULL, c1);
      // closed2: block k-3's word is also one bit range from lo2 reaching the largest
      // size a sweep can need (bit M-3) in every lane, so a lane's live sweeps of an outer
      // prefix are exactly v = lo2+1 .. L1 - a0 - lo1 with spans span_hi .. 1: the count
      // is tetrahedral and only the hash reads remain per sweep (checked per item)
      int lo2 = 0;
      bool c2 = true;
      if (GP_BP_CLOSED2 && !dead && Vr[2]) {
        lo2 = __ffs(Vr[2]) - 1;
        const int need = M - 2 - lo2;  // bits lo2 .. M-3
        const uint32_t mk = need >= 32 ? ~0u : (need <= 0 ? 0u : (1u << need) - 1u);
        c2 = ((Vr[2] >> lo2) & mk) == mk;
      }
      const bool closed2 = GP_BP_CLOSED2 && closed && GP_BP_LANE_V &&
                           (!GP_BP_CORNER || kHash != 1 || a.CT != nullptr) && __all_sync(GP_FULL, c2);
      int32_t q[kBpMaxN];
#pragma unroll
      for (int t = 0; t < kBpMaxN; ++t) q[t] = 1;
      int qsum = k2;
      uint32_t off2 = 0, roff2 = 0;  // s-index / run index of the outer prefix's first candidate
      // the outer blocks' verdict bit at q: the blocks of q[1..] change only when the
      // odometer carries (rare), q[0]'s at every step
      auto outer_hi = [&]() {
        uint32_t r = dead ? 0u : 1u;
#pragma unroll
        for (int t = 1; t < kBpMaxN - 3; ++t)
          if (t < k2) r &= Vr[t + 3] >> (q[t] - 1);
        return r;
      };
      uint32_t rh_hi = outer_hi();
      int L1 = M - qsum - 2;  // len0 of the sweep with s_{k-3} = 1; s_{k-3} <= L1
      uint32_t tri1 = (uint32_t)(L1 * (L1 + 1) / 2);             // runs of the outer prefix
      uint32_t tet1 = (uint32_t)(L1 * (L1 + 1) * (L1 + 2) / 6);  // its candidates
      for (;;) {
        const uint32_t rh = k2 > 0 ? rh_hi & (Vr[3] >> (q[0] - 1)) : rh_hi;  // outer blocks pass
        if (closed2) {
          const int span_hi = L1 - lo2 - a0 - lo1;  // span of the lane's first sweep v = lo2+1
          if ((rh & 1u) && Vr[2] && span_hi >= 1) {
            const int len0f = L1 - lo2;
            if constexpr (kStats) {
              st_sweeps += (uint64_t)span_hi;
              st_live_closed += (uint64_t)((span_hi * (span_hi + 1)) >> 1);
            }
            acc_n += (uint32_t)(span_hi * (span_hi + 1) * (span_hi + 2) / 6);
            acc_pi = min(acc_pi, M - len0f + 1 + lo1 + a0);
            if (first_off == UINT32_MAX)
              first_off = off2 + tet1 - (uint32_t)(len0f * (len0f + 1) * (len0f + 2) / 6) +
                          (uint32_t)(lo1 * len0f - ((lo1 * (lo1 - 1)) >> 1) + a0);
            if constexpr (kHash == 1) {  // (without the hash the outer prefix is O(1))
#if GP_BP_CORNER
              // the lane's schedulable candidates of this block are the corner with apex
              // (lo2+1, lo1+1, a0+1): its hash is one corner-table read at the apex rank
              const uint32_t apex = off2 + tet1 - (uint32_t)(len0f * (len0f + 1) * (len0f + 2) / 6) +
                                    (uint32_t)(lo1 * len0f - ((lo1 * (lo1 - 1)) >> 1) + a0);
              acc_hash += ld_u64(ct_addr, apex);
              if constexpr (kStats) {
                ++st_ct_blocks;
                st_ct_sweeps += (uint64_t)span_hi;
              }
#else
              int len0 = len0f;
              uint32_t roffv = roff2 + tri1 - (uint32_t)((len0 * (len0 + 1)) >> 1);
              uint64_t hsum = 0;
#pragma unroll kBpSweepUnroll
              for (int sp = span_hi; sp >= 1; --sp) {
                hsum += ld_u64(r_addr, roffv + (uint32_t)(len0 - a0)) - ld_u64(r_addr, roffv + (uint32_t)lo1);
                roffv += (uint32_t)len0;
                --len0;
              }
              acc_hash += hsum;
#endif
            }
          }
        } else {
        const uint32_t w2 = (rh & 1u) ? Vr[2] : 0u;  // bit v-1: block k-3 passes at v
        const int vlo_l = w2 ? __ffs(w2) : 99;
        // sweep v's live runs need len0 - a0 > lo1 (closed items) / > 0 (run walk)
        const int vhi_l = w2 ? min(L1, L1 - a0 - (closed ? lo1 : 0)) : 0;
        // the warp's union of the lanes' sweep ranges (closed items walk per lane instead)
        int v_lo = 0, v_hi = -1;
        if (!(closed && GP_BP_LANE_V)) {
          v_lo = (int)__reduce_min_sync(GP_FULL, (unsigned)vlo_l);
          v_hi = (int)__reduce_max_sync(GP_FULL, (unsigned)max(vhi_l, 0));
        }
        if (closed) {
          // every lane's live runs of sweep v are exactly lo1 .. len0 - a0 - 1 (top ranges
          // from a0): span = len0 - a0 - lo1 live runs holding span (span + 1) / 2
          // candidates; the hash from two reads of R.  pi* and the first rank come from
          // the lane's first live sweep (the largest len0; sweeps are visited in rank
          // order), outside the loop.
          if (GP_BP_LANE_V ? vlo_l <= vhi_l : v_lo <= v_hi) {
            if (vlo_l <= vhi_l) {
              const int len0f = L1 - vlo_l + 1;
              acc_pi = min(acc_pi, M - len0f + 1 + lo1 + a0);
              if (first_off == UINT32_MAX)
                first_off = off2 + tet1 - (uint32_t)(len0f * (len0f + 1) * (len0f + 2) / 6) +
                            (uint32_t)(lo1 * len0f - ((lo1 * (lo1 - 1)) >> 1) + a0);
            }
#if GP_BP_LANE_V
            // each lane walks its own live range [vlo_l, vhi_l] (the warp runs the longest)
            const int v_first = vlo_l, v_last = vhi_l;
#else
            const int v_first = v_lo, v_last = v_hi;
#endif
            int len0 = L1 - v_first + 1;
            uint32_t roffv = roff2 + tri1 - (uint32_t)((len0 * (len0 + 1)) >> 1);
#pragma unroll kBpSweepUnroll
            for (int v = v_first; v <= v_last; ++v) {
              const int span = len0 - a0 - lo1;
#if GP_BP_LANE_V && GP_BP_EAGER_LOADS
              // inside the lane's own range span >= 1, so both indices lie in the
              // allocation's runs: read unconditionally (the unrolled iterations' loads
              // overlap), add when block k-3 passes at v
              uint64_t he = 0, hs = 0;
              if constexpr (kHash == 1) {
                he = ld_u64(r_addr, roffv + (uint32_t)(len0 - a0));
                hs = ld_u64(r_addr, roffv + (uint32_t)lo1);
              }
              if ((w2 >> (v - 1)) & 1u) {
                if constexpr (kStats) {
                  ++st_sweeps;
                  st_live_closed += (uint64_t)span;
                }
                acc_n += (uint32_t)((span * (span + 1)) >> 1);
                if constexpr (kHash == 1) acc_hash += he - hs;
              }
#else
              if (((w2 >> (v - 1)) & 1u) && span > 0) {
                if constexpr (kStats) {
                  ++st_sweeps;
                  st_live_closed += (uint64_t)span;
                }
                acc_n += (uint32_t)((span * (span + 1)) >> 1);
                if constexpr (kHash == 1)
                  acc_hash += ld_u64(r_addr, roffv + (uint32_t)(len0 - a0)) -
                              ld_u64(r_addr, roffv + (uint32_t)lo1);
              }
#endif
              roffv += (uint32_t)len0;
              --len0;
            }
          }
        } else {
          for (int v = v_lo; v <= v_hi; ++v) {
            const int len0 = L1 - v + 1;
            const uint32_t offv = off2 + tet1 - (uint32_t)(len0 * (len0 + 1) * (len0 + 2) / 6);
            const uint32_t roffv = roff2 + tri1 - (uint32_t)(len0 * (len0 + 1) / 2);
            sweep(len0, len0, ((w2 >> (v - 1)) & 1u) ? Vr[1] : 0u, offv, roffv);
          }
        }
        }  // !closed2
        off2 += tet1;
        roff2 += tri1;
        // lexicographic successor of the outer parts (sum <= M - 3)
        if (k2 == 0) break;
        if (qsum < M - 3) {
          q[0] += 1;
          qsum += 1;
          tet1 -= tri1;  // tet(L - 1) = tet(L) - tri(L), tri(L - 1) = tri(L) - L
          tri1 -= (uint32_t)L1;
          --L1;
        } else {
          int prefix = 0, pick = -1;
#pragma unroll
          for (int t = 1; t < kBpMaxN; ++t) {
            prefix += q[t - 1];
            if (pick < 0 && t < k2 && prefix > t) pick = t;
          }
          if (pick < 0) break;
          int ns = 0;
#pragma unroll
          for (int t = 0; t < kBpMaxN; ++t) {
            q[t] = t < pick ? 1 : (t == pick ? q[t] + 1 : q[t]);
            ns += t < k2 ? q[t] : 0;
          }
          qsum = ns;
          rh_hi = outer_hi();
          L1 = M - qsum - 2;
          tri1 = (uint32_t)(L1 * (L1 + 1) / 2);
          tet1 = (uint32_t)(L1 * (L1 + 1) * (L1 + 2) / 6);
        }
      }
    }
    if (first_off != UINT32_MAX) acc_first = min(acc_first, rank_pi + first_off);
    }  // allocations of the item
  }
  flush();
  if constexpr (kStats) {
    const uint64_t c0 = warp_sum_u64(st_cand);
    const uint64_t c4 = warp_sum_u64(st_runs), c5 = warp_sum_u64(st_live);
    const uint64_t c6 = warp_sum_u64(st_sweeps), c7 = warp_sum_u64(st_live_closed);
    const uint64_t c8 = warp_sum_u64(st_ct_blocks), c9 = warp_sum_u64(st_ct_sweeps);
    const uint64_t c10 = warp_sum_u64(st_fc_items), c11 = warp_sum_u64(st_fc_blocks);
    if (lane == 0) {
      atomicAdd(a.stats + 0, c0);
      if (a.flags & GP_EX_STATS_EXT) {
        atomicAdd(a.stats + 4, c4);
        atomicAdd(a.stats + 5, c5);
        atomicAdd(a.stats + 6, c6);
        atomicAdd(a.stats + 7, c7);
        atomicAdd(a.stats + 8, c8);
        atomicAdd(a.stats + 9, c9);
        atomicAdd(a.stats + 10, c10);
        atomicAdd(a.stats + 11, c11);
      }
    }
  }
}

template <bool kWin, int kHash, bool kBits>
static void launch_bp(unsigned grid, const ExhArgs &a, const uint32_t *memo, const uint32_t *rgs,
                      const uint64_t *P, cudaStream_t st) {
  if (a.stats) k_exh_bp<kWin, kHash, kBits, true><<<grid, kWarps * 32, 0, st>>>(a, memo, rgs, P);
  else k_exh_bp<kWin, kHash, kBits, false><<<grid, kWarps * 32, 0, st>>>(a, memo, rgs, P);
}

template <bool kWin, int kHash>
static void launch_bp_b(unsigned grid, const ExhArgs &a, const uint32_t *memo,
                        const uint32_t *rgs, const uint64_t *P, cudaStream_t st) {
  if (a.bits) launch_bp<kWin, kHash, true>(grid, a, memo, rgs, P, st);
  else launch_bp<kWin, kHash, false>(grid, a, memo, rgs, P, st);
}

template <bool kWin>
static void launch_bp_h(unsigned grid, const ExhArgs &a, const uint32_t *memo,
                        const uint32_t *rgs, const uint64_t *P, cudaStream_t st) {
  if (a.flags & GP_EX_NO_HASH) launch_bp_b<kWin, 0>(grid, a, memo, rgs, P, st);
  else if (P) launch_bp_b<kWin, 1>(grid, a, memo, rgs, P, st);
  else launch_bp_b<kWin, 2>(grid, a, memo, rgs, P, st);
}

}  // namespace gp

namespace gp {
// Workspace of one bit-sliced call, carved from one buffer (caller-provided or a
// stream-ordered temporary): memo words [2^n][n_sets], RGS labels, the hash prefix
// table P, the run-prefix table R, the corner tables CT / FCT and the memo pass's set
// counter.
struct BpLayout {
  size_t memo_words, words32, bytes, r_off, ct_off, fct_off;
  uint64_t n_rgs, n_ranks, total_runs, r_stride, mc_off;
  uint32_t nb, r_nb;
  bool use_P, use_R, use_CT, use_FCT;
};

static BpLayout bp_layout(const RankLayout &L, int n, int32_t n_sets, int32_t n_groups,
                          uint32_t flags) {
  BpLayout b{};
  b.n_rgs = 0;
  for (int k = 1; k <= L.kmax; ++k) b.n_rgs += L.n_pi[k];
  b.memo_words = (size_t)n_sets * ((size_t)1 << n);
  // hash prefix table over the rank space (when it is small enough and wanted)
  b.use_P = !(flags & GP_EX_NO_HASH) && L.total < kMaxHashTable;
  b.n_ranks = b.use_P ? L.total : 0;
  b.nb = (uint32_t)((b.n_ranks + kScanBlock - 1) / kScanBlock);
  b.words32 = (b.memo_words + b.n_rgs + 1) & ~(size_t)1;  // 8-byte alignment after
  // P: n_ranks + 1 prefix sums, then kPpad entries of slack (the main pass may read up to 31
  // entries past a run's end in lanes whose verdict word is zero there; never summed)
  b.bytes = b.words32 * 4 + (b.use_P ? (b.n_ranks + 1 + kPpad + b.nb) * 8 : 0);
  // run-prefix table R [M][total runs + 1] (+ block totals), with the hash table, while it
  // stays within 64 Mi entries (C3: 20 x 148,734)
  b.total_runs = 0;
  for (int k = 1; k <= L.kmax; ++k) {
    uint64_t c = 1;
    for (int i = 0; i < k - 1; ++i) c = c * (uint64_t)(L.M - 1 - i) / (uint64_t)(i + 1);
    b.total_runs += L.n_pi[k] * c;
  }
  b.r_stride = b.total_runs + 1;
  b.use_R = b.use_P && (uint64_t)L.M * b.r_stride <= ((uint64_t)1 << 26);
  b.r_nb = (uint32_t)((b.total_runs + kScanBlock - 1) / kScanBlock);
  b.r_off = b.bytes;
  if (b.use_R) b.bytes += ((uint64_t)L.M * b.r_stride + (uint64_t)L.M * b.r_nb) * 8;
  // corner table CT[rank] (allocations of k >= 3 blocks) next to R: 8 B per rank
  b.use_CT = GP_BP_CORNER && b.use_R && L.kmax >= 3;
  b.ct_off = b.bytes;
  if (b.use_CT) b.bytes += (uint64_t)L.total * 8;
  // full corner table FCT[rank]: 8 B per rank, with the hash prefix table
  b.use_FCT = GP_BP_FULLCORNER && b.use_P;
  b.fct_off = b.bytes;
  if (b.use_FCT) b.bytes += (uint64_t)L.total * 8;
  b.mc_off = b.bytes;  // the memo pass's set counter
  b.bytes += 8;
  return b;
}
}  // namespace gp

// Workspace bytes of the bit-sliced evaluator (0 when it would not run).
size_t gp_exhaustive_bp_workspace(const gp::RankLayout &L, int n, int M, int32_t n_sets,
                                  int32_t n_groups, uint32_t flags) {
  if (n > gp::kBpMaxN || M > gp::kBpMaxM) return 0;
  return gp::bp_layout(L, n, n_sets, n_groups, flags).bytes;
}

// Called by gp_exhaustive_launch (exhaustive.cu) when n <= 8, M <= 32 and the
// caller did not ask for the per-candidate evaluator.  `a` is fully set up
// (items, rank window, per_set initialised); finalize runs after.  `ws_user` /
// `ws_bytes`: the caller's workspace (gp_exhaustive_opts), or NULL for a
// stream-ordered temporary allocation released on `st`.
gp_status gp_exhaustive_bp_launch(const gp::ExhArgs &a0, void *ws_user, uint64_t ws_bytes,
                                  uint64_t *tables_key, cudaStream_t st) {
  using namespace gp;
  const int n = a0.n, M = a0.M;
  if (n > kBpMaxN || M > kBpMaxM) return gp_fail(GP_EINVAL, "EXHAUSTIVE(bp): n <= 8, M <= 32");
  // items = (set, allocation) in groups of k = kmax, ..., 1; item_base[k] =
  // the first item AFTER group k (group kmax starts at 0); rgs_base[k] = first
  // RGS index with k blocks (rank order)
  ExhArgs a = a0;
  // test hook: take the range-by-range hash path even for contiguous verdict words
  a.force_ranges = (a.flags & GP_EX_FORCE_RANGES) != 0;
  const BpLayout b = bp_layout(a.L, n, a.n_sets, a.n_groups, a.flags);
  uint64_t n_rgs = 0;
  for (int k = 1; k <= a.L.kmax; ++k) {
    a.rgs_base[k] = (uint32_t)n_rgs;
    n_rgs += a.L.n_pi[k];
  }
  uint64_t items = 0;
  const uint64_t groups32 = ((uint64_t)a.n_sets + 31) / 32;  // lane = set
  for (int k = a.L.kmax; k >= 1; --k) {  // item = (32 sets, <= kBpChunk allocations of k blocks)
    items += (a.L.n_pi[k] + kBpChunk - 1) / kBpChunk * groups32;
    a.item_base[k] = items;
  }
  a.items_per_set = n_rgs;
  a.total_items = items;
  const size_t memo_words = b.memo_words;
  const bool use_P = b.use_P;
  const uint64_t n_ranks = b.n_ranks;
  const uint32_t nb = b.nb;
  uint32_t *ws = nullptr;
  if (ws_user) {
    if (ws_bytes < b.bytes)
      return gp_fail(GP_EINVAL, "EXHAUSTIVE: workspace of %llu B < the %zu B needed",
                     (unsigned long long)ws_bytes, b.bytes);
    if (reinterpret_cast<uintptr_t>(ws_user) & 255)
      return gp_fail(GP_EINVAL, "EXHAUSTIVE: workspace must be 256-byte aligned");
    ws = static_cast<uint32_t *>(ws_user);
  } else if (cudaMallocAsync(reinterpret_cast<void **>(&ws), b.bytes, st) != cudaSuccess) {
    return gp_cuda_check("EXHAUSTIVE(bp): workspace allocation");
  }
  // input-independent tables (RGS labels, hash prefix P, run-prefix R, corner tables CT and
  // FCT: functions of (n, M) only) -- rebuilt unless the caller's key says this workspace
  // already holds them for this exact layout (gpart.h: gp_exhaustive_opts.tables_key)
  uint64_t key = 0xcbf29ce484222325ull;
  {
    const uint64_t parts[8] = {(uint64_t)n, (uint64_t)M, (uint64_t)a.n_sets, (uint64_t)a.n_groups,
                               (uint64_t)(a.flags & GP_EX_NO_HASH),
                               (uint64_t)reinterpret_cast<uintptr_t>(ws_user), ws_bytes,
                               (uint64_t)b.bytes};
    for (uint64_t v : parts) key = (key ^ v) * 0x100000001b3ull;
    key |= 1ull;  // never 0 (0 = no tables)
  }
  const bool build_tables = !(ws_user && tables_key && *tables_key == key);
  uint32_t *memo = ws, *rgs = ws + memo_words;
  uint64_t *P = use_P ? reinterpret_cast<uint64_t *>(ws + b.words32) : nullptr;
  if (use_P && build_tables) {
    uint64_t *btot = P + n_ranks + 1 + kPpad;
    k_hash_scan_local<<<nb, kScanBlock, 0, st>>>(P, n_ranks, btot);
    k_hash_scan_blocks<<<1, kScanBlock, 0, st>>>(btot, nb);
    k_hash_scan_add<<<nb, kScanBlock, 0, st>>>(P, n_ranks, btot);
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = ((enum_table_words(M, n) + 3) & ~(size_t)3) * 4;
  if (build_tables) k_exh_rgs_table<<<1, 256, smem, st>>>(a, rgs);
  // runs per allocation: C(M-1, k-1) prefixes; global run index of the first run of k
  uint64_t runs = 0;
  for (int k = 1; k <= a.L.kmax; ++k) {
    uint64_t c = 1;
    for (int i = 0; i < k - 1; ++i) c = c * (uint64_t)(M - 1 - i) / (uint64_t)(i + 1);
    a.L.n_runs[k] = (uint32_t)c;
    a.run_base[k] = runs;
    runs += a.L.n_pi[k] * c;
  }
  a.run_base[a.L.kmax + 1] = runs;
  a.R = nullptr;
  a.CT = nullptr;
  a.FCT = nullptr;
  if (b.use_FCT) {
    uint64_t *F = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(ws) + b.fct_off);
    int64_t gi = ((int64_t)a.L.total + 255) / 256;
    if (gi > (int64_t)sms * 16) gi = (int64_t)sms * 16;
    if (build_tables) {
      k_fct_init<<<(unsigned)(gi > 0 ? gi : 1), 256, 0, st>>>(F, a.L.total);
      for (int j = 1; j <= a.L.kmax; ++j) {
        int64_t gj = ((int64_t)(runs - a.run_base[j]) + 255) / 256;
        if (gj > (int64_t)sms * 16) gj = (int64_t)sms * 16;
        k_fct_pass<<<(unsigned)(gj > 0 ? gj : 1), 256, 0, st>>>(a, F, j);
      }
    }
    a.FCT = F;
  }
  if (b.use_R) {
    uint64_t *R = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(ws) + b.r_off);
    uint64_t *rbt = R + (uint64_t)M * b.r_stride;
    a.r_stride = b.r_stride;
    int64_t gk = ((int64_t)b.total_runs + 255) / 256;
    if (gk > (int64_t)sms * 16) gk = (int64_t)sms * 16;
    if (build_tables) {
      k_run_contrib<<<(unsigned)gk, 256, 0, st>>>(a, P, R, b.total_runs);
      k_rows_scan_local<<<dim3(b.r_nb, M), kScanBlock, 0, st>>>(R, b.r_stride, b.total_runs, rbt, b.r_nb);
      k_rows_scan_blocks<<<M, kScanBlock, 0, st>>>(rbt, b.r_nb);
      k_rows_scan_add<<<dim3(b.r_nb, M), kScanBlock, 0, st>>>(R, b.r_stride, b.total_runs, rbt, b.r_nb);
    }
    a.R = R;
    if (b.use_CT) {
      uint64_t *CT = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(ws) + b.ct_off);
      int64_t gc = ((int64_t)(a.L.total - a.L.k_base[3]) + 255) / 256;
      if (gc > (int64_t)sms * 16) gc = (int64_t)sms * 16;
      if (build_tables) k_corner_table<<<(unsigned)(gc > 0 ? gc : 1), 256, 0, st>>>(a, R, CT);
      a.CT = CT;
    }
  }
  {
    int64_t blocks = ((int64_t)a.n_sets + 7) / 8;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    a.memo_counter = nullptr;
    if (GP_MEMO_DYNAMIC) {  // one wave of resident CTAs, sets from the counter
      a.memo_counter = reinterpret_cast<unsigned long long *>(reinterpret_cast<unsigned char *>(ws) + b.mc_off);
      cudaMemsetAsync(a.memo_counter, 0, 8, st);
      if (blocks > (int64_t)sms * GP_MEMO_MINB) blocks = (int64_t)sms * GP_MEMO_MINB;
    }
    const unsigned g = (unsigned)(blocks > 0 ? blocks : 1);
    if (a.stats) {
      if (n <= 4) k_exh_memo<4, true><<<g, 256, 0, st>>>(a, memo);
      else if (n <= 6) k_exh_memo<6, true><<<g, 256, 0, st>>>(a, memo);
      else k_exh_memo<8, true><<<g, 256, 0, st>>>(a, memo);
    } else {
      if (n <= 4) k_exh_memo<4, false><<<g, 256, 0, st>>>(a, memo);
      else if (n <= 6) k_exh_memo<6, false><<<g, 256, 0, st>>>(a, memo);
      else k_exh_memo<8, false><<<g, 256, 0, st>>>(a, memo);
    }
  }
  gp_status r = gp_cuda_check("EXHAUSTIVE(bp) memo kernel");
  if (r == GP_OK) {
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_exh_bp<false, 1, false, false>, kWarps * 32, 0);
    if (occ < 1) occ = 1;
    uint64_t want = (a.total_items + kWarps - 1) / kWarps;
    uint64_t grid = (uint64_t)sms * occ;
    if (want < grid) grid = want > 0 ? want : 1;
    const bool win = !(a.lo == 0 && a.hi >= a.L.total);
    if (win) launch_bp_h<true>((unsigned)grid, a, memo, rgs, P, st);
    else launch_bp_h<false>((unsigned)grid, a, memo, rgs, P, st);
    r = gp_cuda_check("EXHAUSTIVE(bp) main kernel");
  }
  if (ws_user && tables_key) *tables_key = r == GP_OK ? key : 0ull;
  if (!ws_user) cudaFreeAsync(ws, st);
  return r;
}
