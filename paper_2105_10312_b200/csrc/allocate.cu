// allocate.cu -- A5: the paper's partition-and-allocate heuristics and the 1G
// baseline, one GROUP of G = 8, 16 or 32 lanes per task set (gp_allocate; the
// smallest power of two >= n, so small sets share a warp; every collective is
// group-masked), persistent warps grabbing sets from a counter, one kernel per
// variant.
//
// Lane roles: lane i holds task i (its parameters, its Lemma 2 size, its
// ACT forbidden row); lane s also holds partition SLOT s.  A live slot's index
// is always the lowest task id of its partition (a merge keeps the lower
// slot), so the par_list tie-break "lower min task id" (A-17) is the slot
// index and canonical output labels are popcounts.  The per-partition EDF
// test is group-cooperative (lane = task of the partition): conflict flags via
// popcount on the type mask, U*H via a shuffle sum, the demand walk with a
// shuffle-min over the next deadlines (gp_edf.cuh explains the exact L_a
// cut-off).  The ACT prefill runs the n(n-1)/2 pair merges lane-parallel with
// a per-lane two-task test; Algorithm 2's merge scans of one round run one
// partner per lane (G/E lanes per partner when E <= G/2, strided).
//
// Algorithm 1, Lemma 1, Lemma 2 (the minimal m is
// computed in closed form m = ceil(B / floor((D - f)/c)), exact for the W
// form), Lemma 3, Algorithm 2 (linear m scan, Def. 3
// strict bound), Algorithm 3, Def. 4 / Def. 5 orders
// (P:720-753), forbidden list; conventions C.1.9 / A-17..A-26.
// f4 variants (gp_alloc_opts): binary-search merge
// (P:704-706), increasing par_list order, admissible partition
// sizes -- compiled into a second instantiation (kGen) so that the
// paper's default path keeps its plain linear scan.
#include <stdlib.h>

#include "gp_common.cuh"
#include "gp_edf.cuh"
#include "gp_sizes.cuh"

gp_status gp_allocate_big_launch(const gp_tasksets *ts, int32_t v, const gp::AllocVariantOpts &vo,
                                 uint8_t *ok, int16_t *bot, int16_t *bs, int32_t *pi, int32_t *k,
                                 int64_t *n_tests, int64_t *eff, unsigned long long *stats,
                                 bool stats_ext, cudaStream_t st);

namespace gp {

struct AllocArgs {
  const int32_t *T, *D, *B, *cn, *cc, *fn, *fc;
  const uint8_t *type;
  int32_t n_sets, n, M, variant;
  uint8_t *ok;
  int16_t *bot;
  int16_t *bs;
  int32_t *pi, *k;
  int64_t *n_tests;
  int64_t *eff;               // optional [n_sets][4]: scheduled workload (f2)
  unsigned long long *stats;  // optional: += {EDF tests (paper's count), tasks tested, deadlines
                              // examined, sets} [+ {tests run, selections, partitions scanned,
                              // partner searches} with stats_ext]
  int32_t stats_ext;
  int32_t use_tab;            // per-warp table of ceil(B_i/m) in dynamic shared memory
  uint32_t pt_off;            // byte offset of the groups' pair tables in dynamic shared memory
  unsigned long long *next_set;  // work counter (zeroed per launch)
  AllocVariantOpts vo;        // f4
  const uint32_t *memo;       // optional [2^n][memo_stride] block verdict words of an EXHAUSTIVE call
  int64_t memo_stride;        // words between consecutive subsets' rows of memo
};

#ifndef GP_ALLOC_MINB8
#define GP_ALLOC_MINB8 5  // CTAs per SM the 8-lane-group kernels' register budget targets (A/B: 3, 4, 5, 6 -> 5)
#endif
#ifndef GP_ALLOC_MINB32
#define GP_ALLOC_MINB32 4  // the same for the 16- and 32-lane-group kernels (A/B: 3, 4 -> 4)
#endif
#ifndef GP_ALLOC_GATHER_PER_TEST
#define GP_ALLOC_GATHER_PER_TEST 1  // 16/32-lane groups: task records gathered per test (A/B: C4 -2 %, C5 -11 % with 4 CTAs)
#endif
#ifndef GP_ALLOC_N6
#define GP_ALLOC_N6 1  // 8-lane kernels specialised on n = 6 (A/B)
#endif
#ifndef GP_ALLOC_NS4
#define GP_ALLOC_NS4 8  // widest group that gets the <= 4-task lane-serial merge (0: none)
#endif
// lane-serial merge instantiation for <= 4 tasks besides <= 8: more code for the instruction
// cache, which the divergent groups of a warp already stress (no_instructions is the top stall
// of the heuristics kernels).  A/B-measured: it pays in 8-lane groups (C3: 4.72 vs 4.89 ms per
// step) and costs in 16- and 32-lane groups (C5 88 -> 85 ms, C4 124 -> 118 ms without it).
template <int G>
constexpr bool kAllocNs4 = G <= GP_ALLOC_NS4;

// A group of G lanes of one warp works on one task set (G = 8, 16 or 32: the
// smallest power of two >= n), so small sets share a warp.  Every collective is
// over the group's lanes (mask gmask, shuffles of width G); groups of a warp may
// diverge freely.
template <int G>
struct Grp {
  uint32_t gmask;
  int gl;  // lane within the group
  GP_DEV Grp() {
    const int lane = threadIdx.x & 31;
    gl = lane & (G - 1);
    gmask = G == 32 ? GP_FULL : (((1u << G) - 1u) << (lane & ~(G - 1)));
  }
  GP_DEV uint32_t ballot(bool p) const {
    const uint32_t b = __ballot_sync(gmask, p);
    return G == 32 ? b : (b >> ((threadIdx.x & 31) & ~(G - 1))) & ((1u << G) - 1u);
  }
  template <class T> GP_DEV T shfl(T v, int src) const { return __shfl_sync(gmask, v, src, G); }
  template <class T> GP_DEV T shfl_xor(T v, int o) const { return __shfl_xor_sync(gmask, v, o, G); }
  GP_DEV bool all(bool p) const { return __all_sync(gmask, p); }
  GP_DEV void sync() const { __syncwarp(gmask); }
  GP_DEV unsigned reduce_max(unsigned v) const { return __reduce_max_sync(gmask, v); }
  template <class T> GP_DEV T sum(T v) const {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += shfl_xor(v, o);
    return v;
  }
  GP_DEV int32_t sum_i32(int32_t v) const { return sum<int32_t>(v); }
  GP_DEV int64_t sum_i64(int64_t v) const { return sum<int64_t>(v); }
  GP_DEV uint64_t sum_u64(uint64_t v) const { return sum<uint64_t>(v); }
  // single-instruction group reductions (redux.sync)
  GP_DEV int32_t min_i32(int32_t v) const { return __reduce_min_sync(gmask, v); }
  GP_DEV uint32_t min_u32(uint32_t v) const { return __reduce_min_sync(gmask, v); }
  GP_DEV uint32_t or_u32(uint32_t v) const { return __reduce_or_sync(gmask, v); }
  GP_DEV uint32_t add_u32(uint32_t v) const { return __reduce_add_sync(gmask, v); }
};

// ceil(B_i / m) from the warp's per-set table (uint16, built once per set)
// or computed directly when the table is off or B does not fit 16 bits.
struct Waves {
  const uint16_t *tab;  // [n][M] or null
  int32_t M;
  GP_DEV int32_t operator()(int i, int32_t B, int32_t m) const {
    // merged sizes may exceed M (Alg. 2 scans up to |P1|+|P2|-1): compute those
    return (tab && m <= M) ? (int32_t)tab[i * M + m - 1] : ceil_div_pos(B, m);
  }
};

GP_DEV int32_t w_from_waves(int32_t waves, int32_t c, int32_t f) {
  const int64_t w = (int64_t)waves * (int64_t)c + (int64_t)f;
  return w > INT32_MAX ? INT32_MAX : (int32_t)w;
}

struct TaskLane {
  int32_t T, D, B, cn, cc, fn, fc, q;
  uint32_t same;  // mask of tasks with my type
  bool in;        // lane < n
  Waves wv;
};

GP_DEV int32_t task_w(const TaskLane &t, int lane, int32_t m, bool x) {
  const int32_t wv = t.wv(lane, t.B, m);
  return x ? w_from_waves(wv, t.cc, t.fc) : w_from_waves(wv, t.cn, t.fn);
}

// Group-cooperative EDF-PDC of partition S at size m (C.1.7).
template <int G>
GP_DEV bool warp_pdc(const Grp<G> &g, const TaskLane &t, uint32_t S, int32_t m, int32_t H,
                     uint64_t &st_tasks, uint64_t &st_events) {
  const int lane = g.gl;
  st_tasks += __popc(S);
  const bool in = (S >> lane) & 1u;
  const bool x = __popc(S & t.same) > 1;  // conflict
  const int32_t C = in ? task_w(t, lane, m, x) : 0;
  if (g.ballot(in && C > t.D)) return false;
  if (__popc(S) == 1) return true;
  const int32_t UH = g.sum_i32(in ? C * t.q : 0);
  if (UH > H) return false;
  int32_t lcut = H;
  if (UH < H) {
    float X = in ? (float)(t.T - t.D) * (float)(C * t.q) : 0.f;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) X += g.shfl_xor(X, o);
    const float L = X / (float)(H - UH) * 1.0001f + 2.0f;
    lcut = L >= (float)H ? H : (int32_t)L;
  }
  int32_t nx = in ? t.D : INT32_MAX, dem = 0;
  for (;;) {
    const int32_t tt = g.min_i32(nx);
    if (tt > lcut) return true;
    const bool hit = nx == tt;
    ++st_events;
    dem += g.sum_i32(hit ? C : 0);
    nx += hit ? t.T : 0;
    if (dem > tt) return false;
  }
}

// U(P)*H of partition S at size m (Def. 5 with /T_i, reading A-19).
template <int G>
GP_DEV int32_t warp_uh(const Grp<G> &g, const TaskLane &t, uint32_t S, int32_t m) {
  const int lane = g.gl;
  const bool in = (S >> lane) & 1u;
  const bool x = __popc(S & t.same) > 1;
  return g.sum_i32(in ? task_w(t, lane, m, x) * t.q : 0);
}

// Per-lane two-task EDF-PDC (ACT prefill), same exact shortcuts.
GP_DEV bool pair_pdc(const int32_t (&C)[2], const int32_t (&D)[2], const int32_t (&T)[2],
                     const int32_t (&q)[2], int32_t H, uint32_t &ev) {
  if (C[0] > D[0] || C[1] > D[1]) return false;
  const int32_t UH = C[0] * q[0] + C[1] * q[1];
  if (UH > H) return false;
  const int32_t lcut = pdc_cutoff<2>(C, D, T, q, H, UH);
  return pdc_walk<2>(C, D, T, lcut, ev);
}

template <int G>
struct WarpScratch {
  int32_t ord[G];    // ord[r] = slot with par_list rank r
  int32_t bord[G];   // bord[r] = slot with best-fit rank r (U*H desc, A-21)
  int32_t lab[G];    // output label of task i
  int32_t size[G];   // size of output label j
  uint32_t forb[G];  // ACT: forbidden task row
  int32_t plist[G];  // eligible partners of the selected partition, par_list order
  uint32_t pmask[G]; // task mask of output label j
  uint32_t pmS[G];   // task mask of partition slot s (for the pair evaluations)
  int32_t szS[G];    // size of partition slot s
  // the set's tasks, for the lane-serial merge tests
  int32_t T[G], D[G], B[G], cn[G], cc[G], fn[G], fc[G], q[G];
  uint32_t same[G];
};

// Algorithm 2 merge of partition S (<= NS tasks) by ONE lane: the first
// schedulable m in lo .. hi (Def. 3 bound hi = |P1| + |P2| - 1; 0 if none) and
// U*H there.  `counted` += the tests the paper's linear scan performs
// (alg2_search: one probe at hi + binary search instead of the scan, exact by
// monotonicity); `st_exec` += the tests actually run.
template <int NS, bool kGen, bool kMemo, class WS>
GP_DEV int32_t serial_merge(const WS &w, const Waves &wv, const SizeSpace &z, uint32_t S,
                            int32_t lo, int32_t hi, int32_t H, int32_t &uh_out, int64_t &counted,
                            uint64_t &st_tasks, uint32_t &st_events, uint32_t &st_exec,
                            const uint32_t *vm, size_t vst, int32_t M) {
  const int cnt = __popc(S);
  if constexpr (kMemo || GP_ALLOC_GATHER_PER_TEST) {
    // a test at m <= M with memo words is a lookup plus U*H, both from shared memory; the
    // task records are gathered into registers only for a full test (with memo words the
    // rare m > M), so they hold no registers across the search (more resident CTAs)
    auto test = [&](int32_t m) -> bool {
      ++st_exec;
      if (vm && m <= M) {
        if (!((vm[(size_t)S * vst] >> (m - 1)) & 1u)) return false;
        int32_t UH = 0;
        for (uint32_t b = S; b; b &= b - 1u) {
          const int i = __ffs(b) - 1;
          const bool x = __popc(S & w.same[i]) > 1;  // conflict
          UH += w_from_waves(wv(i, w.B[i], m), x ? w.cc[i] : w.cn[i], x ? w.fc[i] : w.fn[i]) * w.q[i];
        }
        uh_out = UH;
        return true;
      }
      st_tasks += cnt;
      int32_t C[NS], D[NS], T[NS], q[NS];
      uint32_t bits = S;
      bool bad = false;
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        const bool v = bits != 0;
        const int i = v ? __ffs(bits) - 1 : 0;
        bits &= bits - 1u;
        const bool x = __popc(S & w.same[i]) > 1;
        T[a] = v ? w.T[i] : INT32_MAX;
        D[a] = v ? w.D[i] : INT32_MAX;
        q[a] = v ? w.q[i] : 0;
        C[a] = v ? w_from_waves(wv(i, w.B[i], m), x ? w.cc[i] : w.cn[i], x ? w.fc[i] : w.fn[i]) : 0;
        bad |= C[a] > D[a];
      }
      if (bad) return false;
      int32_t UH = 0;
#pragma unroll
      for (int a = 0; a < NS; ++a) UH += C[a] * q[a];
      if (UH > H) return false;
      if (cnt > 1) {
        const int32_t lcut = pdc_cutoff<NS>(C, D, T, q, H, UH);
        if (!pdc_walk<NS>(C, D, T, lcut, st_events)) return false;
      }
      uh_out = UH;
      return true;
    };
    return alg2_search<kGen>(z, lo, hi, test, counted);
  }
  int32_t T[NS], D[NS], B[NS], c[NS], f[NS], q[NS], id[NS];
  uint32_t bits = S;
#pragma unroll
  for (int a = 0; a < NS; ++a) {
    const bool v = bits != 0;
    const int i = v ? __ffs(bits) - 1 : 0;
    bits &= bits - 1u;
    const bool x = __popc(S & w.same[i]) > 1;  // conflict
    T[a] = v ? w.T[i] : INT32_MAX;
    D[a] = v ? w.D[i] : INT32_MAX;
    B[a] = v ? w.B[i] : 1;
    id[a] = i;
    c[a] = v ? (x ? w.cc[i] : w.cn[i]) : 0;
    f[a] = v ? (x ? w.fc[i] : w.fn[i]) : 0;
    q[a] = v ? w.q[i] : 0;
  }
  // one EDF-PDC test at size m; on success U*H is recorded (the last success
  // of a search is its answer)
  auto test = [&](int32_t m) -> bool {
    ++st_exec;
    st_tasks += cnt;
    int32_t C[NS];
    bool bad = false;
#pragma unroll
    for (int a = 0; a < NS; ++a) {
      C[a] = c[a] ? w_from_waves(wv(id[a], B[a], m), c[a], f[a]) : 0;
      bad |= C[a] > D[a];
    }
    if (bad) return false;
    int32_t UH = 0;
#pragma unroll
    for (int a = 0; a < NS; ++a) UH += C[a] * q[a];
    if (UH > H) return false;
    if (cnt > 1) {
      const int32_t lcut = pdc_cutoff<NS>(C, D, T, q, H, UH);
      if (!pdc_walk<NS>(C, D, T, lcut, st_events)) return false;
    }
    uh_out = UH;
    return true;
  };
  return alg2_search<kGen>(z, lo, hi, test, counted);
}

// Pair-table entry: Algorithm 2's outcome for a pair of partition slots (i < j):
// the first schedulable size (0 if none), the tests the paper's scan counts and
// U*H of the merged partition at that size.
GP_DEV uint64_t pt_pack(int32_t got, int64_t cnt, int32_t uh) {
  return ((uint64_t)(uint32_t)got & 0xFFFu) | (((uint64_t)cnt & 0xFFFFFu) << 12) |
         ((uint64_t)(uint32_t)uh << 32);
}
GP_DEV void pt_unpack(uint64_t e, int32_t &got, int64_t &cnt, int32_t &uh) {
  got = (int32_t)(e & 0xFFFu);
  cnt = (int64_t)((e >> 12) & 0xFFFFFu);
  uh = (int32_t)(e >> 32);
}
GP_DEV int pt_index(int i, int j, int n) { return i * (2 * n - i - 1) / 2 + (j - i - 1); }
template <int G>
GP_DEV uint32_t pm_bcast(const Grp<G> &g, uint32_t pm, int src) { return g.shfl(pm, src); }

// kV >= 0: the variant is a compile-time constant (one kernel per variant: each carries only
// its own code, e.g. no ACT prefill in INA, which keeps the instruction working set small);
// kV = -1: runtime variant (the f4 kGen kernels)
// kN > 0: the task count as a compile-time constant (the paper-shaped n = 6 sets of C1-C3 scale:
// every loop over tasks, slots and pairs has a constant trip count); 0: runtime a.n
template <bool kGen, int G, int kV, bool kStats, int kN = 0>
// register budget: 5 CTAs per SM for 8-lane groups (48 registers), 4 otherwise (64): A/B
// measured, with the task records of a lane-serial merge gathered per test (no registers
// held across the size search)
__global__ void __launch_bounds__(256, G == 8 ? GP_ALLOC_MINB8 : GP_ALLOC_MINB32) k_allocate(const AllocArgs a) {
  const int variant = kV >= 0 ? kV : a.variant;
  // memoised verdicts exist for n <= 8 only, i.e. in 8-lane groups: the wider kernels keep
  // the plain tests (no extra code or registers)
  constexpr bool kMemo = G == 8;
  __shared__ WarpScratch<G> scr_all[256 / G];
  extern __shared__ __align__(16) uint16_t wtab_all[];
  const Grp<G> g;
  const int lane = g.gl, wid = threadIdx.x / G;  // lane within the group, group in the CTA
  WarpScratch<G> &scr = scr_all[wid];
  const int n = kN > 0 ? kN : a.n, M = a.M;
  uint16_t *wtab = a.use_tab ? wtab_all + (size_t)wid * n * M : nullptr;
  // this group's pair table (dynamic shared memory after the wave / size tables)
  uint64_t *pt_tab = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(wtab_all) +
                                                  a.pt_off) + (size_t)wid * (n * (n - 1) / 2);
  // f4: admissible-size tables after the ceil(B/m) tables
  SizeSpace z{nullptr, M, 0, false};
  bool incr = false;
  if constexpr (kGen) {
    z.binary = (a.vo.flags & GP_AL_BINARY_MERGE) != 0;
    incr = (a.vo.flags & GP_AL_INCREASING) != 0;
    if (a.vo.masked) {
      const size_t off = a.use_tab ? (size_t)(256 / G) * n * M : 0;
      SizeTables *tb = reinterpret_cast<SizeTables *>(wtab_all + ((off + 7) & ~(size_t)7));
      build_size_tables(*tb, a.vo.mask, M);
      z.tab = tb;
      z.A = tb->ge[M + 1];
    }
  }
  const uint32_t all = n == 32 ? GP_FULL : ((1u << n) - 1u);
  uint64_t st_tests = 0, st_tasks = 0, st_events = 0, st_sets = 0;  // group-uniform
  uint64_t st_exec = 0, st_rounds = 0, st_scan = 0, st_partners = 0; // group-uniform
  uint64_t st_pair_tasks = 0;                                        // per lane
  uint32_t st_pair_events = 0, st_pair_exec = 0;                     // per lane
  // persistent warps: each grabs its next set from a global counter (sets differ widely in
  // work -- utilisation bin, variant -- so a static stride leaves warps idle at the tail)
  for (;;) {
    int64_t set = 0;
    if (lane == 0) set = (int64_t)atomicAdd(a.next_set, 1ull);
    set = g.shfl(set, 0);
    if (set >= a.n_sets) break;
    const int64_t o = set * n + lane;
    TaskLane t;
    t.in = lane < n;
    const int64_t oo = t.in ? o : set * n;
    t.T = a.T[oo]; t.D = a.D[oo]; t.B = a.B[oo]; t.cn = a.cn[oo]; t.cc = a.cc[oo];
    t.fn = a.fn[oo]; t.fc = a.fc[oo];
    const bool mem = t.in && a.type[oo] == 1;
    const uint32_t memmask = g.ballot(mem);
    t.same = mem ? memmask : (all & ~memmask);
    // input contract and H = lcm of all periods (capped)
    const bool fields_ok = !t.in || (t.T >= 1 && t.D >= 1 && t.D <= t.T && t.B >= 1 && t.cn >= 1 &&
                                     t.cc >= t.cn && t.fn >= 0 && t.fc >= t.fn);
    int64_t h;
    bool contract;
    if (kMemo && a.memo) {
      // the exhaustive pass checked the same contract on the same sets and left H (the lcm of
      // the periods; 0 = violated) in its words' row 0
      const uint32_t hm = a.memo[set];
      h = hm ? (int64_t)hm : -1;
      contract = h > 0;
    } else {
      const int64_t cap = ((int64_t)1 << 31) / (n + 1) - 1;
      h = (t.in && fields_ok) ? t.T : (t.in ? -1 : 1);
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) {
        const int64_t other = g.shfl_xor(h, off);
        h = (h < 0 || other < 0) ? -1 : lcm_capped(h, other, cap);
      }
      contract = g.all(fields_ok) && h > 0;
    }
    const int32_t H = contract ? (int32_t)h : 1;
    t.q = (contract && t.in) ? H / t.T : 0;
    scr.T[lane] = t.T; scr.D[lane] = t.D; scr.B[lane] = t.B; scr.cn[lane] = t.cn;
    scr.cc[lane] = t.cc; scr.fn[lane] = t.fn; scr.fc[lane] = t.fc; scr.q[lane] = t.q;
    scr.same[lane] = t.same;
    // per-set table of ceil(B_i/m) (the wave counts of C.1.3), if B fits 16 bits
    // (1G tests one size only: no table)
    const bool tab_ok = wtab && variant != GP_1G && g.all(!t.in || t.B <= 65535);
    g.sync();
    if (tab_ok) {
      for (int i = 0; i < n; ++i) {
        const int32_t Bi = scr.B[i];
        for (int m = lane + 1; m <= M; m += G) wtab[i * M + m - 1] = (uint16_t)ceil_div_pos(Bi, m);
      }
    }
    t.wv.tab = tab_ok ? wtab : nullptr;
    t.wv.M = M;
    g.sync();

    // memoised block verdicts of this set (n <= 8: 2^n words), when the caller passes them
    // (subset-major: word S of this set at vm[S * vst])
    const uint32_t *vm = (kMemo && a.memo && contract) ? a.memo + set : nullptr;
    const size_t vst = (size_t)a.memo_stride;
    int64_t tests = 0;
    bool ok = false;
    int stage = 0;  // 0: rejected before partitions exist, 1: partitions to report
    // slot state (lane = slot)
    uint32_t pm = 0, pex = 0;
    int32_t psz = 0, puh = 0;

    if (!contract) {
      tests = -1;
    } else if (variant == GP_1G) {
      // 1G: the whole GPU as one partition
      tests = 1;
      ++st_exec;
      const int32_t m1 = z.largest();  // M, or the largest admissible size (f4)
      ok = (kMemo && vm && m1 <= M) ? ((vm[(size_t)all * vst] >> (m1 - 1)) & 1u) != 0
                           : warp_pdc(g, t, all, m1, H, st_tasks, st_events);
      pm = lane == 0 ? all : 0;
      psz = lane == 0 ? m1 : 0;
      stage = 1;
    } else {
      const bool act = variant == GP_SMS_ACT || variant == GP_BF_ACT;
      const bool sms = variant == GP_SMS_ACT || variant == GP_SMS_INA;
      // Lemma 1: sum_i W_i(1,n) * (H/T_i) > M*H  =>  reject
      const int64_t w1 = t.in ? ((int64_t)t.B * t.cn + t.fn) * (int64_t)t.q : 0;
      const bool lemma1 = g.sum_i64(w1) <= (int64_t)M * H;
      // Lemma 2: m_i = min{m : ceil(B/m) cn + fn <= D}
      int32_t mi = 0;
      if (t.in && t.D - t.fn >= t.cn) {
        const int32_t K = (t.D - t.fn) / t.cn;  // waves allowed: ceil(B/m) <= K
        const int64_t m0 = ((int64_t)t.B + K - 1) / K;  // 64-bit: B may reach INT32_MAX
        mi = m0 <= M ? (m0 < 1 ? 1 : (int32_t)m0) : 0;
        if (kGen && mi) mi = z.round_up(mi);  // f4: smallest admissible size >= m0
      }
      const bool lemma2 = !g.ballot(t.in && mi == 0);
      if (lemma1 && lemma2) {
        stage = 1;
        pm = t.in ? (1u << lane) : 0;
        psz = mi;
        puh = t.in ? task_w(t, lane, mi, false) * t.q : 0;
        int32_t Pi = g.sum_i32(psz);
        if (Pi <= M) {
          ok = true;  // Lemma 3: exit on success at any time (A-24)
        } else {
          // ---- the pair table.  Algorithm 2's outcome for a pair of partitions
          // depends only on the two partitions, and every pair the sequential
          // algorithm tries is tried at most once per partition state, so the
          // outcome of every pair of LIVE partitions is computed lane-parallel
          // (speculatively) and the rounds below read it: the Lemma-2 singletons
          // first (in ACT this is the prefill itself), then after each
          // commit the new partition against every live one.  Each entry keeps the
          // tests the paper's scan counts, so n_tests and every output are the
          // sequential algorithm's.
          scr.pmS[lane] = pm;
          scr.szS[lane] = psz;
          scr.forb[lane] = 0;
          g.sync();
          const int np = n * (n - 1) / 2;
          int64_t my_tests = 0;
          for (int base = 0; base < np; base += G) {
            const int idx = base + lane;
            int i = 0, rem = idx < np ? idx : 0;
            while (rem >= n - 1 - i) {
              rem -= n - 1 - i;
              ++i;
            }
            const int j = i + 1 + rem;
            if (idx < np) {
              int32_t uh = 0;
              int64_t cnt = 0;
              const int32_t got = serial_merge<2, kGen, kMemo>(
                  scr, t.wv, z, (1u << i) | (1u << j), max(scr.szS[i], scr.szS[j]),
                  scr.szS[i] + scr.szS[j] - 1, H, uh, cnt, st_pair_tasks, st_pair_events,
                  st_pair_exec, vm, vst, M);
              pt_tab[idx] = pt_pack(got, cnt, uh);
              my_tests += cnt;
              if (act && !got) {  // §5.3: the couple is forbidden
                atomicOr(&scr.forb[i], 1u << j);
                atomicOr(&scr.forb[j], 1u << i);
              }
            }
          }
          if (act) tests += g.add_u32((uint32_t)my_tests);  // the prefill's tests (INA: speculative)
          g.sync();
          const uint32_t forb_row = act ? scr.forb[lane] : 0u;
          // Algorithm 1 main loop.  par_list order (rank: position of my slot) and the
          // ACT exclusions depend only on the partitions: built once here, then updated
          // incrementally at each commit (two partitions leave, one enters).
          // par_list order: (U*H desc, slot asc), or U*H asc (f4 increasing); best-fit
          // partner order (brank): always U*H desc (A-21)
          bool live = pm != 0;
          uint32_t livemask = g.ballot(live);
          int rank = 0, brank = 0;
          for (int s2 = 0; s2 < n; ++s2) {
            const int32_t u2 = g.shfl(puh, s2);
            const bool lv = (livemask >> s2) & 1u;
            brank += lv && (u2 > puh || (u2 == puh && s2 < lane));
            if (kGen && incr) rank += lv && (u2 < puh || (u2 == puh && s2 < lane));
          }
          if (!(kGen && incr)) rank = brank;
          int len = __popc(livemask);
          // ACT: F = tasks forbidden with a task of my partition; forb_slots = the slots
          // holding such a task
          uint32_t F = forb_row, forb_slots = 0;
          if (act)
            for (int s2 = 0; s2 < n; ++s2)
              if (g.shfl(pm, s2) & F) forb_slots |= 1u << s2;
          bool rebuild = true;
          for (;;) {
            if (rebuild) {
              if (live) {
                scr.ord[rank] = lane;
                scr.bord[brank] = lane;
              }
              g.sync();
              rebuild = false;
            }
            if (Pi <= M) {
              ok = true;
              break;
            }
            // Algorithm 3: eligibility of every slot, pick the first in order
            const uint32_t elig_mine = live ? (livemask & ~(1u << lane) & ~pex & ~forb_slots) : 0;
            const int cand_rank = g.min_i32(elig_mine ? rank : 99);
            if (cand_rank == 99) break;  // no selectable partition: fail (Alg. 1 l.6-7)
            const int P = scr.ord[cand_rank];
            const uint32_t elig = g.shfl(elig_mine, P);
            const int32_t szP = g.shfl(psz, P);
            // eligible partners in best-fit order -> lane e holds partner plist[e]
            const int Qr = lane < len ? scr.bord[lane] : 0;
            const bool el = lane < len && ((elig >> Qr) & 1u);
            const uint32_t elb = g.ballot(el);
            if (el) scr.plist[__popc(elb & ((1u << lane) - 1u))] = Qr;
            g.sync();
            const int E = __popc(elb);
            ++st_rounds;       // one Algorithm 3 selection ...
            st_scan += len;    // ... over the len partitions of par_list (mask ops)
            st_partners += E;  // eligible partners tried with Algorithm 2
            const int Qe = lane < E ? scr.plist[lane] : 0;
            // Algorithm 2 for (P, Q_e): the pair table's entry
            int32_t got = 0, uh = 0;
            int64_t my_tests = 0;  // the paper's scan count for partner `lane`
            if (lane < E) pt_unpack(pt_tab[pt_index(min(P, Qe), max(P, Qe), n)], got, my_tests, uh);
            int best = -1;
            int32_t best_m = 0, best_uh = 0;
            const uint32_t succ = g.ballot(lane < E && got > 0);
            int cut = E;  // partners whose tests the sequential order performs
            if (sms) {  // Def. 4 order >>: smallest size, then U*H, then min id (A-20, A-22)
              const uint32_t k1 = (lane < E && got > 0) ? (uint32_t)got : ~0u;
              const uint32_t m1 = g.min_u32(k1);
              if (m1 != ~0u) {
                const uint32_t k2 = k1 == m1 ? (uint32_t)uh : ~0u;  // U*H >= 0
                const uint32_t m2 = g.min_u32(k2);
                best = (int)g.min_u32(k2 == m2 && k1 == m1 ? (uint32_t)Qe : ~0u);
                best_m = (int32_t)m1;
                best_uh = (int32_t)m2;
              }
            } else if (succ) {  // BF: the first success in par_list order commits (A-21)
              cut = __ffs(succ);  // partners 0 .. cut-1 were tried
              const int e0 = cut - 1;
              best = g.shfl(Qe, e0);
              best_m = g.shfl(got, e0);
              best_uh = g.shfl(uh, e0);
            }
            tests += g.add_u32(lane < cut ? (uint32_t)my_tests : 0u);
            const bool failed = lane < cut && lane < E && got == 0;
            const uint32_t failQ = g.or_u32(failed ? (1u << Qe) : 0u);
            if (lane == P) pex |= failQ;                 // add_to_forbidden_moves(P, Q)
            if ((failQ >> lane) & 1u) pex |= 1u << P;
            if (best >= 0) {  // commit: P u Q replaces P and Q in par_list
              const int Q = best;
              const int32_t szQ = g.shfl(psz, Q);
              const uint32_t pmP = g.shfl(pm, P), pmQ = g.shfl(pm, Q);
              const int32_t uP = g.shfl(puh, P), uQ = g.shfl(puh, Q);
              const uint32_t FP = g.shfl(F, P), FQ = g.shfl(F, Q);
              const int keep = min(P, Q), drop = max(P, Q);
              Pi -= szP + szQ - best_m;
              // incremental par_list / best-fit ranks: P and Q leave, (P u Q) enters at keep
              {
                auto before_d = [&](int32_t ux, int x) {  // slot x precedes me (U*H desc)
                  return ux > puh || (ux == puh && x < lane);
                };
                auto before_i = [&](int32_t ux, int x) {  // (U*H asc, f4 increasing)
                  return ux < puh || (ux == puh && x < lane);
                };
                if (lane != keep && lane != drop) {
                  brank += (int)before_d(best_uh, keep) - (int)before_d(uP, P) - (int)before_d(uQ, Q);
                  if (kGen && incr)
                    rank += (int)before_i(best_uh, keep) - (int)before_i(uP, P) - (int)before_i(uQ, Q);
                }
                // the new partition's ranks: live slots (other than P, Q) before it
                const bool other = live && lane != P && lane != Q;
                const uint32_t bd = g.ballot(other && (puh > best_uh || (puh == best_uh && lane < keep)));
                const uint32_t bi = (kGen && incr)
                                        ? g.ballot(other && (puh < best_uh || (puh == best_uh && lane < keep)))
                                        : 0u;
                if (lane == keep) {
                  brank = __popc(bd);
                  rank = (kGen && incr) ? __popc(bi) : brank;
                }
                if (!(kGen && incr)) rank = brank;
              }
              if (lane == keep) {
                pm = pmP | pmQ;
                psz = best_m;
                puh = best_uh;
                pex = 0;
                F = FP | FQ;
              } else if (lane == drop) {
                pm = 0;
                psz = 0;
                puh = 0;
                pex = 0;
                F = 0;
              }
              pex &= ~((1u << keep) | (1u << drop));
              live = pm != 0;
              livemask &= ~(1u << drop);
              len -= 1;
              if (act) {  // exclusions against the changed slots
                forb_slots &= ~((1u << keep) | (1u << drop));
                if (live && lane != keep && ((pmP | pmQ) & F)) forb_slots |= 1u << keep;
                const uint32_t fk = g.ballot(live && (pm & (FP | FQ)));
                if (lane == keep) forb_slots = fk;
              }
              rebuild = true;
              scr.pmS[lane] = pm;
              scr.szS[lane] = psz;
              g.sync();
              if (Pi > M) {
                // the new partition against every live one (lane = the other slot)
                const uint32_t pk = pm_bcast(g, pm, keep);
                // ACT never tries a partner holding a task forbidden with one of the new
                // partition's tasks: no entry needed for those pairs
                const uint32_t Fk = act ? g.shfl(F, keep) : 0u;
                const bool mine = pm != 0 && lane != keep && !(pm & Fk);
                const uint32_t S2 = pk | pm;
                const int c2 = mine ? __popc(S2) : 0;
                const int maxc = (int)g.reduce_max((unsigned)c2);
                int32_t got2 = 0, uh2 = 0;
                int64_t cnt2 = 0;
                const int32_t lo2 = max(best_m, psz), hi2 = best_m + psz - 1;
                if (mine && c2 <= 8) {
                  if (kAllocNs4<G> && maxc <= 4)
                    got2 = serial_merge<4, kGen, kMemo>(scr, t.wv, z, S2, lo2, hi2, H, uh2, cnt2, st_pair_tasks, st_pair_events, st_pair_exec, vm, vst, M);
                  else
                    got2 = serial_merge<8, kGen, kMemo>(scr, t.wv, z, S2, lo2, hi2, H, uh2, cnt2, st_pair_tasks, st_pair_events, st_pair_exec, vm, vst, M);
                  pt_tab[pt_index(min(keep, lane), max(keep, lane), n)] = pt_pack(got2, cnt2, uh2);
                }
                // (groups of 8 lanes hold <= 8 tasks: the group-cooperative path for merged
                // partitions of more than 8 tasks is compiled out -- smaller code)
                uint32_t big = G > 8 ? g.ballot(mine && c2 > 8) : 0u;
                while (G > 8 && big) {
                  const int s2 = __ffs(big) - 1;
                  big &= big - 1u;
                  const uint32_t S3 = pk | g.shfl(pm, s2);
                  const int32_t sz2 = g.shfl(psz, s2);
                  int64_t cnt3 = 0;
                  auto wtest = [&](int32_t m) -> bool {
                    ++st_exec;
                    return warp_pdc(g, t, S3, m, H, st_tasks, st_events);
                  };
                  const int32_t got3 =
                      alg2_search<kGen>(z, max(best_m, sz2), best_m + sz2 - 1, wtest, cnt3);
                  const int32_t uh3 = got3 ? warp_uh(g, t, S3, got3) : 0;
                  if (lane == 0) pt_tab[pt_index(min(keep, s2), max(keep, s2), n)] = pt_pack(got3, cnt3, uh3);
                }
                g.sync();
              }
            }
          }
        }
      }
    }
    // outputs: labels numbered by lowest task id (= slot index)
    const uint32_t livemask = g.ballot(pm != 0);
    const int kk = stage ? __popc(livemask) : 0;
    if (pm) {
      const int label = __popc(livemask & ((1u << lane) - 1u));
      scr.size[label] = psz;
      scr.pmask[label] = pm;
      uint32_t bits = pm;
      while (bits) {
        const int tsk = __ffs(bits) - 1;
        bits &= bits - 1;
        scr.lab[tsk] = label;
      }
    }
    g.sync();
    const int32_t Pi_out = stage ? g.sum_i32(psz) : 0;
    if (t.in) {
      a.bot[o] = (int16_t)(stage ? scr.lab[lane] : -1);
      a.bs[o] = (int16_t)((stage && lane < kk) ? scr.size[lane] : 0);
    }
    st_sets += 1;
    st_tests += tests > 0 ? (uint64_t)tests : 0;
    if (a.eff) {
      // f2: work c^x * B per period, x H
      const int64_t w = t.in ? (int64_t)t.B * t.q : 0;
      const int64_t lo = g.sum_i64(w * t.cn), up = g.sum_i64(w * t.cc);
      int64_t mine = 0;
      if (stage && t.in) {
        const bool x = __popc(scr.pmask[scr.lab[lane]] & t.same) > 1;  // conflict
        mine = w * (x ? t.cc : t.cn);
      }
      const int64_t ach = g.sum_i64(mine);
      if (lane == 0) {
        a.eff[set * 4 + 0] = lo;
        a.eff[set * 4 + 1] = up;
        a.eff[set * 4 + 2] = ach;
        a.eff[set * 4 + 3] = contract ? H : 0;
      }
    }
    if (lane == 0) {
      a.ok[set] = ok ? 1 : 0;
      a.pi[set] = Pi_out;
      a.k[set] = kk;
      a.n_tests[set] = tests;
    }
    g.sync();
  }
  if constexpr (kStats) {  // (the timed instantiation carries no counters: fewer registers)
    const uint64_t pt = g.sum_u64(st_pair_tasks), pe = g.sum_u64(st_pair_events);
    const uint64_t px = g.sum_u64(st_pair_exec);
    if (lane == 0) {
      atomicAdd(a.stats + 0, (unsigned long long)st_tests);
      atomicAdd(a.stats + 1, (unsigned long long)(st_tasks + pt));
      atomicAdd(a.stats + 2, (unsigned long long)(st_events + pe));
      atomicAdd(a.stats + 3, (unsigned long long)st_sets);
      if (a.stats_ext) {
        atomicAdd(a.stats + 4, (unsigned long long)(st_exec + px));
        atomicAdd(a.stats + 5, (unsigned long long)st_rounds);
        atomicAdd(a.stats + 6, (unsigned long long)st_scan);
        atomicAdd(a.stats + 7, (unsigned long long)st_partners);
      }
    }
  }
}

}  // namespace gp

// per-CTA wave-table budget (compile-time A/B switch -DGP_ALLOC_TAB_KB=n).  Default 0 (no
// table): since the pair tables, building the n x M table of ceil(B_i/m) per set costs more
// than the divisions it saves (A/B: C3 4.72 -> 4.68 ms per step, C5 99.9 -> 91.4 ms; C4's
// table never fit the 40 KB budget)
#ifndef GP_ALLOC_TAB_KB
#define GP_ALLOC_TAB_KB 0
#endif
// minimum group width (compile-time A/B switch -DGP_ALLOC_MIN_G=8|16|32, default 8)
#ifndef GP_ALLOC_MIN_G
#define GP_ALLOC_MIN_G 8
#endif

extern "C" gp_status gp_allocate(const gp_tasksets *ts, gp_variant v, const gp_alloc_opts *opts,
                                 uint8_t *ok, int16_t *block_of_task, int16_t *block_size,
                                 int32_t *pi, int32_t *k, int64_t *n_tests, int64_t *efficiency,
                                 unsigned long long *stats, void *stream) {
  using namespace gp;
  if (!ts || ts->n_tasks < 1 || ts->n_tasks > 256 || ts->M < 1 || ts->M > 1024 ||
      ts->n_sets < 0)
    return gp_fail(GP_EINVAL, "gp_allocate: bad task sets (n_tasks 1..256, M 1..1024)");
  if ((int)v < 0 || (int)v > 4) return gp_fail(GP_EINVAL, "gp_allocate: bad variant %d", (int)v);
  AllocVariantOpts vo{};
  bool stats_ext = false;
  if (opts) {
    if (opts->flags & ~(uint32_t)(GP_AL_BINARY_MERGE | GP_AL_INCREASING | GP_AL_STATS_EXT))
      return gp_fail(GP_EINVAL, "gp_allocate: unknown option flags 0x%x", opts->flags);
    vo.flags = opts->flags & ~(uint32_t)GP_AL_STATS_EXT;  // the f4 variant bits
    stats_ext = (opts->flags & GP_AL_STATS_EXT) != 0;
    if (opts->size_mask) {
      const int words = (ts->M + 31) / 32;
      int any = 0;
      for (int w = 0; w < words; ++w) {
        uint32_t m = opts->size_mask[w];
        if (w == words - 1 && (ts->M & 31)) m &= (1u << (ts->M & 31)) - 1u;  // sizes <= M only
        vo.mask[w] = m;
        any |= m != 0;
      }
      if (!any) return gp_fail(GP_EINVAL, "gp_allocate: size_mask admits no size in 1..M");
      vo.masked = 1;
    }
  }
  const uint32_t *memo = opts ? opts->memo : nullptr;
  const int64_t memo_stride = (opts && opts->memo_stride) ? opts->memo_stride : (int64_t)ts->n_sets;
  if (memo && memo_stride < ts->n_sets)
    return gp_fail(GP_EINVAL, "gp_allocate: memo_stride %lld < n_sets", (long long)memo_stride);
  if (memo && (ts->n_tasks > 8 || ts->M > 32))
    return gp_fail(GP_EINVAL, "gp_allocate: memo needs n_tasks <= 8 and M <= 32");
  if (ts->n_sets == 0) return gp_cuda_check("gp_allocate");
  if (!ok || !block_of_task || !block_size || !pi || !k || !n_tests || !ts->T || !ts->D ||
      !ts->B || !ts->cn || !ts->cc || !ts->fn || !ts->fc || !ts->type)
    return gp_fail(GP_EINVAL, "gp_allocate: null pointer");
  if (ts->n_tasks > kMaxTasks)  // 33..256 tasks: one CTA per set (allocate_big.cu)
    return gp_allocate_big_launch(ts, (int32_t)v, vo, ok, block_of_task, block_size, pi, k,
                                  n_tests, efficiency, stats, stats_ext,
                                  (cudaStream_t)stream);
  // group width: the smallest of 8, 16, 32 lanes that holds the set's tasks (and is at
  // least GP_ALLOC_MIN_G)
  int G = ts->n_tasks <= 8 ? 8 : (ts->n_tasks <= 16 ? 16 : 32);
  G = max(G, GP_ALLOC_MIN_G);
  // per-group ceil(B/m) table: 256/G groups x n x M x 2 bytes when it fits (C4: 76 KB)
  size_t tab = (size_t)(256 / G) * ts->n_tasks * ts->M * sizeof(uint16_t);
  // the table pays for itself only in the INA variants (most WCET evaluations per set), and
  // only while it does not cost resident CTAs (A/B-measured on C2-C5)
  const bool use_tab = (v == GP_SMS_INA || v == GP_BF_INA) && tab <= (size_t)GP_ALLOC_TAB_KB * 1024;
  if (!use_tab) tab = 0;
  const bool gen = vo.flags != 0 || vo.masked;
  size_t smem = tab;
  if (gen && vo.masked) smem = ((tab + 15) & ~(size_t)15) + sizeof(SizeTables);
  // the groups' pair tables (Algorithm 2 outcomes of partition pairs): n(n-1)/2 x 8 B each
  const size_t pt_off = (smem + 15) & ~(size_t)15;
  smem = pt_off + (size_t)(256 / G) * (ts->n_tasks * (ts->n_tasks - 1) / 2) * sizeof(uint64_t);
  AllocArgs a{ts->T, ts->D, ts->B, ts->cn, ts->cc, ts->fn, ts->fc, ts->type, ts->n_sets,
              ts->n_tasks, ts->M, (int32_t)v, ok, block_of_task, block_size, pi, k, n_tests,
              efficiency, stats, stats_ext ? 1 : 0, use_tab ? 1 : 0, (uint32_t)pt_off, nullptr,
              vo, memo, memo_stride};
  using KernFn = void (*)(AllocArgs);
  static const KernFn kdef[2][3][5] = {
      {{k_allocate<false, 8, 0, false>, k_allocate<false, 8, 1, false>, k_allocate<false, 8, 2, false>,
        k_allocate<false, 8, 3, false>, k_allocate<false, 8, 4, false>},
       {k_allocate<false, 16, 0, false>, k_allocate<false, 16, 1, false>, k_allocate<false, 16, 2, false>,
        k_allocate<false, 16, 3, false>, k_allocate<false, 16, 4, false>},
       {k_allocate<false, 32, 0, false>, k_allocate<false, 32, 1, false>, k_allocate<false, 32, 2, false>,
        k_allocate<false, 32, 3, false>, k_allocate<false, 32, 4, false>}},
      {{k_allocate<false, 8, 0, true>, k_allocate<false, 8, 1, true>, k_allocate<false, 8, 2, true>,
        k_allocate<false, 8, 3, true>, k_allocate<false, 8, 4, true>},
       {k_allocate<false, 16, 0, true>, k_allocate<false, 16, 1, true>, k_allocate<false, 16, 2, true>,
        k_allocate<false, 16, 3, true>, k_allocate<false, 16, 4, true>},
       {k_allocate<false, 32, 0, true>, k_allocate<false, 32, 1, true>, k_allocate<false, 32, 2, true>,
        k_allocate<false, 32, 3, true>, k_allocate<false, 32, 4, true>}}};
  static const KernFn kdef6[2][5] = {  // n = 6 (C2, C3 shapes), 8-lane groups
      {k_allocate<false, 8, 0, false, 6>, k_allocate<false, 8, 1, false, 6>, k_allocate<false, 8, 2, false, 6>,
       k_allocate<false, 8, 3, false, 6>, k_allocate<false, 8, 4, false, 6>},
      {k_allocate<false, 8, 0, true, 6>, k_allocate<false, 8, 1, true, 6>, k_allocate<false, 8, 2, true, 6>,
       k_allocate<false, 8, 3, true, 6>, k_allocate<false, 8, 4, true, 6>}};
  const int gi = G == 8 ? 0 : (G == 16 ? 1 : 2);
  const bool st_on = stats != nullptr;
  const KernFn kern =
      gen ? (st_on ? (G == 8 ? k_allocate<true, 8, -1, true>
                             : G == 16 ? k_allocate<true, 16, -1, true> : k_allocate<true, 32, -1, true>)
                   : (G == 8 ? k_allocate<true, 8, -1, false>
                             : G == 16 ? k_allocate<true, 16, -1, false> : k_allocate<true, 32, -1, false>))
          : (G == 8 && ts->n_tasks == 6 && GP_ALLOC_N6) ? kdef6[st_on ? 1 : 0][(int)v]
                                                          : kdef[st_on ? 1 : 0][gi][(int)v];
  // dynamic + static shared memory may pass 48 KB (e.g. 16-lane groups: 16 scratches + tables)
  // opt in to more than 48 KB (static + dynamic) only when needed: setting a function
  // attribute per call was measured to stall the stream (C3 step +1.4 ms)
  {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    if (fa.sharedSizeBytes + smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  // persistent grid: one wave of resident CTAs; the set counter lives in a stream-ordered
  // 8-byte allocation from the default pool
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  if (occ < 1) occ = 1;
  int64_t grid = ((int64_t)ts->n_sets + 256 / G - 1) / (256 / G);
  if (grid > (int64_t)sms * occ) grid = (int64_t)sms * occ;
  if (cudaMallocAsync(reinterpret_cast<void **>(&a.next_set), 8, (cudaStream_t)stream) != cudaSuccess)
    return gp_cuda_check("gp_allocate: work counter");
  cudaMemsetAsync(a.next_set, 0, 8, (cudaStream_t)stream);
  kern<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(a);
  cudaFreeAsync(a.next_set, (cudaStream_t)stream);
  return gp_cuda_check("gp_allocate");
}
