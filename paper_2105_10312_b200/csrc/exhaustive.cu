// exhaustive.cu -- A2-A4 fused: every (SM partitioning, task-to-partition
// allocation) candidate of every task set, evaluated directly (C.1.6-C.1.8).
//
// Work decomposition (B200: 148 SMs, persistent CTAs, warp-granular queue):
//   item = (set, k, RGS index p, chunk c): up to 32*L consecutive size vectors
//   s of ONE allocation pi.  A warp pulls 16 items at a time from a global
//   atomic queue, so load balances across SMs whatever the per-set cost.
//   Per item everything that does not depend on s is warp-uniform and built
//   once in the warp's shared memory: the block structure of pi, each task's
//   conflict flag x_i and its record {W-table offset, D, T, H/T}.
//   Per set the warp builds the W table W[i][x][s] = ceil(B_i/s) c_i^x + f_i^x
//   (C.1.3) in shared memory.
//   Lane = candidate: each lane unranks its first size vector once and then
//   steps lexicographic successors in registers (no per-candidate division).
//   Blocks are tested in order with a warp-uniform switch on the block's task
//   count (a template per count keeps every per-task array in registers);
//   a lane stops at its first unschedulable block; the warp skips the remaining
//   blocks as soon as no lane is alive (__any_sync).
//   Per set: n_sched / pi* / first rank / verdict hash are reduced in
//   registers and flushed with one set of atomics per item run.
#include <cstdio>
#include <cstdlib>

#include "gp_common.cuh"
#include "gp_edf.cuh"
#include "gp_enum.cuh"
#include "gp_exh.cuh"

namespace gp {

struct WarpSmem {
  int32_t set, H, okc, n_multi;
  int4 rec[kEnumMaxTasks];   // per task in block order: {W offset, D, T, H/T}
  int32_t T[kEnumMaxTasks], D[kEnumMaxTasks], q[kEnumMaxTasks];
  int32_t multi[kEnumMaxTasks];  // multi-task blocks: jj | len << 8 | start << 16
  uint32_t memmask, pad2[3];
};

// EDF-PDC of one block with SZ >= 2 tasks (records in shared memory, block
// order, starting at `start`), all lanes at their own size s.
template <int SZ>
GP_DEV bool eval_block(const WarpSmem &w, const int32_t *__restrict__ Wt, int start, int32_t s,
                       int32_t H, uint32_t &events) {
  int32_t C[SZ], D[SZ], T[SZ], q[SZ];
  bool bad = false;
#pragma unroll
  for (int a = 0; a < SZ; ++a) {
    const int4 r = w.rec[start + a];
    C[a] = Wt[r.x + s];
    D[a] = r.y;
    T[a] = r.z;
    q[a] = r.w;
    bad |= C[a] > D[a];
  }
  if (bad) return false;
  int32_t UH = 0;
#pragma unroll
  for (int a = 0; a < SZ; ++a) UH += C[a] * q[a];
  if (UH > H) return false;  // utilisation > 1
  if constexpr (SZ <= 8) {
    if (pdc_density_ok<SZ>(C, D)) return true;
  }
  const int32_t lcut = pdc_cutoff<SZ>(C, D, T, q, H, UH);
  return pdc_walk<SZ>(C, D, T, lcut, events);
}

template <int NT, int SZ>
struct BlockDispatch {
  GP_DEV static bool run(int sz, const WarpSmem &w, const int32_t *Wt, int start, int32_t s,
                         int32_t H, uint32_t &ev) {
    if (sz == SZ) return eval_block<SZ>(w, Wt, start, s, H, ev);
    return BlockDispatch<NT, SZ + 1>::run(sz, w, Wt, start, s, H, ev);
  }
};
template <int NT>
struct BlockDispatch<NT, NT + 1> {
  GP_DEV static bool run(int, const WarpSmem &, const int32_t *, int, int32_t, int32_t,
                         uint32_t &) {
    return false;
  }
};

// load one set into the warp's shared memory: contract, H, H/T_i, types and
// the W table W[i][x][s] = ceil(B_i/s) c_i^x + f_i^x (C.1.3)
GP_DEV void exh_load_set(const ExhArgs &a, WarpSmem &w, int32_t *Wt, int64_t set, int lane) {
  const int n = a.n, M = a.M;
  const int64_t H = set_contract(a, set);
  __syncwarp();
  if (lane < n) {
    const int64_t o = set * n + lane;
    w.T[lane] = a.T[o];
    w.D[lane] = a.D[o];
    w.q[lane] = H > 0 ? (int32_t)(H / a.T[o]) : 0;
  }
  const uint32_t mm = __ballot_sync(GP_FULL, lane < n && a.type[set * n + min(lane, n - 1)] == 1);
  if (lane == 0) {
    w.H = (int32_t)(H > 0 ? H : 0);
    w.okc = H > 0;
    w.memmask = mm;
  }
  if (H > 0) {
    for (int e = lane; e < 2 * n * M; e += 32) {
      const int i = e / (2 * M), x = (e / M) & 1, s = e % M + 1;
      const int64_t o = set * n + i;
      Wt[e] = x ? wcet_adm(a.adm, a.B[o], a.cc[o], a.fc[o], s)
                : wcet_adm(a.adm, a.B[o], a.cn[o], a.fn[o], s);
    }
  }
  __syncwarp();
}

template <int NT, bool kStats>
__global__ void __launch_bounds__(kWarps * 32, 3) k_exhaustive(const ExhArgs a) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int n = a.n, M = a.M;
  const EnumTables tab = build_enum_tables(smem, M, n);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  size_t off = (enum_table_words(M, n) + 3) & ~(size_t)3;
  const size_t wt_words = (size_t)2 * n * M;
  const size_t per_warp = ((sizeof(WarpSmem) / 4 + wt_words) + 3) & ~(size_t)3;
  WarpSmem &w = *reinterpret_cast<WarpSmem *>(smem + off + per_warp * warp);
  int32_t *Wt = reinterpret_cast<int32_t *>(&w + 1);
  const bool stats = kStats && a.stats != nullptr;

  LaneAcc acc;
  int64_t cur = -1;

  auto flush = [&]() {
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
  };

  for (;;) {
    uint64_t base = 0;
    if (lane == 0) base = atomicAdd(a.work_counter, (unsigned long long)kGrab);
    base = __shfl_sync(GP_FULL, base, 0);
    if (base >= a.total_items) break;
    const uint64_t end = min(base + (uint64_t)kGrab, a.total_items);
    for (uint64_t it = base; it < end; ++it) {
      const int64_t set = (int64_t)(it / a.items_per_set);
      uint64_t local = it - (uint64_t)set * a.items_per_set;
      if (set != cur) {
        flush();
        cur = set;
        // load the set: contract, H, H/T_i, types; then the W table
        int64_t H = set_contract(a, set);
        __syncwarp();
        if (lane < n) {
          const int64_t o = set * n + lane;
          w.T[lane] = a.T[o];
          w.D[lane] = a.D[o];
          w.q[lane] = H > 0 ? (int32_t)(H / a.T[o]) : 0;
        }
        const uint32_t mm = __ballot_sync(GP_FULL, lane < n && a.type[set * n + min(lane, n - 1)] == 1);
        if (lane == 0) {
          w.H = (int32_t)(H > 0 ? H : 0);
          w.okc = H > 0;
          w.memmask = mm;
        }
        if (H > 0) {
          for (int e = lane; e < 2 * n * M; e += 32) {
            const int i = e / (2 * M), x = (e / M) & 1, s = e % M + 1;
            const int64_t o = set * n + i;
            Wt[e] = x ? wcet_adm(a.adm, a.B[o], a.cc[o], a.fc[o], s)
                      : wcet_adm(a.adm, a.B[o], a.cn[o], a.fn[o], s);
          }
        }
        __syncwarp();
      }
      if (!w.okc) continue;  // contract violation: finalize reports it
      // decode item -> k, p, chunk
      int k = 1;
      while (k < a.L.kmax && local >= a.item_base[k + 1]) ++k;
      local -= a.item_base[k];
      const uint32_t chunks = a.chunks[k];
      const uint32_t p = (uint32_t)(local / chunks);
      const uint32_t c = (uint32_t)(local % chunks);
      const int Lk = a.lane_L[k];
      const uint32_t per_pi = (uint32_t)a.L.per_pi[k];
      const uint64_t rank_pi = a.L.k_base[k] + (uint64_t)p * per_pi;
      const uint32_t rho0 = c * 32u * (uint32_t)Lk;
      if (rank_pi + rho0 >= a.hi || rank_pi + min((uint64_t)per_pi, (uint64_t)rho0 + 32u * Lk) <= a.lo)
        continue;
      // ---- allocation pi (warp-uniform): blocks, conflict flags, records
      const uint64_t labels = unrank_rgs(tab, k, p);
      const int myb = lane < n ? (int)((labels >> (4 * lane)) & 15) : -1;
      // block j: mask, length, first position in block order; reversed copies
      // rlen[jj], rpos[jj] describe block k-1-jj (register-static indices)
      int rlen[NT], rpos[NT];
      uint32_t mine = 0;
      int mypos0 = 0, acc_pos = 0;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const uint32_t bm = __ballot_sync(GP_FULL, myb == j);
        const int len = __popc(bm);
        if (j == myb) {
          mine = bm;
          mypos0 = acc_pos;
        }
#pragma unroll
        for (int jj = 0; jj < NT; ++jj)
          if (jj == k - 1 - j) {
            rlen[jj] = len;
            rpos[jj] = acc_pos;
          }
        acc_pos += len;
      }
#pragma unroll
      for (int jj = 0; jj < NT; ++jj)
        if (jj >= k) rlen[jj] = 0, rpos[jj] = 0;
      if (lane < n) {
        const uint32_t same = ((w.memmask >> lane) & 1) ? w.memmask : ~w.memmask;
        const int x = __popc(mine & same) > 1 ? 1 : 0;  // conflict
        const int pos = mypos0 + __popc(mine & ((1u << lane) - 1u));
        w.rec[pos] = make_int4((lane * 2 + x) * M - 1, w.D[lane], w.T[lane], w.q[lane]);
      }
      if (lane == 0) {
        int nm = 0;
#pragma unroll
        for (int jj = 0; jj < NT; ++jj)
          if (rlen[jj] > 1) w.multi[nm++] = jj | (rlen[jj] << 8) | (rpos[jj] << 16);
        w.n_multi = nm;
      }
      __syncwarp();
      // singleton blocks: W-table offset and deadline in registers
      int32_t swoff[NT], sdl[NT];
      int n_single = 0;
#pragma unroll
      for (int jj = 0; jj < NT; ++jj) {
        const int4 r = w.rec[rpos[jj]];
        swoff[jj] = r.x;
        sdl[jj] = r.y;
        n_single += rlen[jj] == 1;
      }
      const int n_multi = w.n_multi;
      const int32_t H = w.H;
      uint32_t *bits = a.bits ? a.bits + cur * a.words : nullptr;
      // ---- this lane's run of candidates: s-index my0 .. my0 + Lk - 1
      const uint32_t my0 = rho0 + (uint32_t)lane * (uint32_t)Lk;
      const uint64_t r0 = rank_pi + my0;
      int t_hi = Lk;
      if (a.hi <= r0) t_hi = 0;
      else if (a.hi - r0 < (uint64_t)t_hi) t_hi = (int)(a.hi - r0);
      if ((int64_t)t_hi > (int64_t)per_pi - (int64_t)my0) t_hi = (int)max((int64_t)0, (int64_t)per_pi - (int64_t)my0);
      const int t_lo = a.lo > r0 ? (int)min(a.lo - r0, (uint64_t)Lk) : 0;
      if (t_lo >= t_hi) t_hi = 0;
      int32_t sr[NT];
      int32_t sum = 0;
      {
        int32_t s[NT];
        if (t_hi > 0) {
          unrank_sizes<NT>(tab, k, my0, s);
        } else {
#pragma unroll
          for (int j = 0; j < NT; ++j) s[j] = 1;
        }
#pragma unroll
        for (int jj = 0; jj < NT; ++jj) {
          sr[jj] = 1;
#pragma unroll
          for (int j = 0; j < NT; ++j)
            if (j == k - 1 - jj) sr[jj] = s[j];
          sum += jj < k ? sr[jj] : 0;
        }
      }
      if (stats && t_hi > 0) {
        acc.st_cand += (uint64_t)(t_hi - t_lo);
        acc.st_blocks += (uint64_t)(t_hi - t_lo) * n_single;
        acc.st_tasks += (uint64_t)(t_hi - t_lo) * n_single;
      }
      const int tmax = (int)__reduce_max_sync(GP_FULL, (unsigned)t_hi);
      for (int t = 0; t < tmax; ++t) {
        bool ok = t >= t_lo && t < t_hi;
        // blocks with one task: schedulable iff C <= D (C.1.7)
#pragma unroll
        for (int jj = 0; jj < NT; ++jj)
          if (rlen[jj] == 1) ok &= Wt[swoff[jj] + sr[jj]] <= sdl[jj];
        // blocks with >= 2 tasks: the EDF processor-demand test (gp_edf.cuh)
        for (int mb = 0; mb < n_multi; ++mb) {
          if (!__any_sync(GP_FULL, ok)) break;
          const int e = w.multi[mb];
          const int jj = e & 0xFF, len = (e >> 8) & 0xFF, start = e >> 16;
          int32_t s = 0;
#pragma unroll
          for (int q = 0; q < NT; ++q) s = q == jj ? sr[q] : s;
          if (ok) {
            if (stats) {
              ++acc.st_blocks;
              acc.st_tasks += len;
            }
            ok = BlockDispatch<NT, 2>::run(len, w, Wt, start, s, H, acc.st_events);
          }
        }
        if (ok) record_ok(acc, r0 + (uint32_t)t, sum, bits, a.lo);
        if (t + 1 < t_hi) next_sizes_rev<NT>(M, k, sr, sum);
      }
      __syncwarp();
    }
  }
  flush();
  if (kStats && stats) {
    const uint64_t c0 = warp_sum_u64(acc.st_cand), c1 = warp_sum_u64(acc.st_blocks);
    const uint64_t c2 = warp_sum_u64(acc.st_events), c3 = warp_sum_u64(acc.st_tasks);
    if (lane == 0) {
      atomicAdd(a.stats + 0, c0);
      atomicAdd(a.stats + 1, c1);
      atomicAdd(a.stats + 2, c2);
      atomicAdd(a.stats + 3, c3);
    }
  }
}

// ============================================================================
// Shape-specialised path (n <= 6), items in SHAPE-MAJOR order.
//
// The shape of an allocation pi is the sequence of its block sizes in label
// order (a composition of n; CUTS has bit p set when a block ends after task
// position p).  With the shape a template parameter, k, every block's task
// count and position are compile-time constants: the task records live in
// registers, the size vector is a fixed-length register array, the successor
// has no runtime bounds and the multi-task blocks need no dispatch.  Work
// items are ordered shape-major (all sets' items of shape 0, then shape 1,
// ...) so that, at any moment, the warps of the GPU execute the same shape's
// code: the instruction working set stays that of ONE instantiation.
// ============================================================================
constexpr int kMaxShapeN = 6;
constexpr int kMaxShapes = 1 << (kMaxShapeN - 1);  // compositions of n
constexpr int kMaxRgs = 203;                        // Bell(6)

struct ShapeTable {
  int32_t n_shapes;
  uint32_t cuts[kMaxShapes];
  int32_t k[kMaxShapes];
  int32_t first[kMaxShapes + 1];        // into entry[]
  uint32_t entry[kMaxRgs];              // labels (4 bits/task) | p << 24 (index among k-RGS)
  uint64_t item_base[kMaxShapes + 1];   // cumulative items over shapes
  uint32_t items_per_set[kMaxShapes];   // entries * chunks(k)
  int32_t n_single[kMaxShapes];         // blocks with one task
};

constexpr int cpopc(unsigned x) { return x ? (int)(x & 1u) + cpopc(x >> 1) : 0; }
constexpr int shape_start(int N, unsigned cuts, int j) {
  int b = 0;
  if (j == 0) return 0;
  for (int p = 0; p < N - 1; ++p)
    if ((cuts >> p) & 1u) {
      ++b;
      if (b == j) return p + 1;
    }
  return N;
}
constexpr int shape_len(int N, unsigned cuts, int j) {
  return shape_start(N, cuts, j + 1) - shape_start(N, cuts, j);
}

template <int N>
struct TaskRegs {
  int32_t woff[N], D[N], T[N], q[N];
};

template <int N, int S0, int L>
GP_DEV bool eval_multi(const int32_t *__restrict__ Wt, const TaskRegs<N> &r, int32_t s,
                       int32_t H, uint32_t &ev) {
  int32_t C[L], D[L], T[L], q[L];
  bool bad = false;
#pragma unroll
  for (int a = 0; a < L; ++a) {
    C[a] = Wt[r.woff[S0 + a] + s];
    D[a] = r.D[S0 + a];
    T[a] = r.T[S0 + a];
    q[a] = r.q[S0 + a];
    bad |= C[a] > D[a];
  }
  if (bad) return false;
  int32_t UH = 0;
#pragma unroll
  for (int a = 0; a < L; ++a) UH += C[a] * q[a];
  if (UH > H) return false;
  if constexpr (L <= 8) {
    if (pdc_density_ok<L>(C, D)) return true;
  }
  const int32_t lcut = pdc_cutoff<L>(C, D, T, q, H, UH);
  return pdc_walk<L>(C, D, T, lcut, ev);
}

// sizes are stored reversed: sr[jj] is the size of block K-1-jj
template <int N, unsigned CUTS, int JJ, int K>
GP_DEV void shape_singles(const int32_t *__restrict__ Wt, const TaskRegs<N> &r,
                          const int32_t (&sr)[K], bool &ok) {
  if constexpr (JJ < K) {
    constexpr int J = K - 1 - JJ;
    constexpr int S0 = shape_start(N, CUTS, J), L = shape_len(N, CUTS, J);
    if constexpr (L == 1) ok &= Wt[r.woff[S0] + sr[JJ]] <= r.D[S0];
    shape_singles<N, CUTS, JJ + 1, K>(Wt, r, sr, ok);
  }
}

template <int N, unsigned CUTS, int JJ, int K>
GP_DEV void shape_multis(const int32_t *__restrict__ Wt, const TaskRegs<N> &r,
                         const int32_t (&sr)[K], int32_t H, bool &ok, LaneAcc &acc, bool stats) {
  if constexpr (JJ < K) {
    constexpr int J = K - 1 - JJ;
    constexpr int S0 = shape_start(N, CUTS, J), L = shape_len(N, CUTS, J);
    if constexpr (L > 1) {
      if (__any_sync(GP_FULL, ok)) {
        if (ok) {
          if (stats) {
            ++acc.st_blocks;
            acc.st_tasks += L;
          }
          ok = eval_multi<N, S0, L>(Wt, r, sr[JJ], H, acc.st_events);
        }
      }
    }
    shape_multis<N, CUTS, JJ + 1, K>(Wt, r, sr, H, ok, acc, stats);
  }
}

template <int K>
GP_DEV void next_sizes_rev_static(int M, int32_t (&sr)[K], int32_t &sum) {
  if (sum < M) {  // common: grow the last part
    sr[0] += 1;
    sum += 1;
    return;
  }
  if constexpr (K >= 2) {
    if (sr[0] > 1) {  // bump the second-to-last part, last := 1
      sum -= sr[0] - 2;
      sr[0] = 1;
      sr[1] += 1;
      return;
    }
    int prefix = 0, pick = -1;
#pragma unroll
    for (int jj = 1; jj < K; ++jj) {
      prefix += sr[jj - 1];
      if (pick < 0 && prefix > jj) pick = jj;
    }
    if (pick < 0) return;
    int ns = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      sr[i] = i < pick ? 1 : (i == pick ? sr[i] + 1 : sr[i]);
      ns += sr[i];
    }
    sum = ns;
  }
}

struct ShapeItem {
  const int32_t *Wt;
  const WarpSmem *w;
  const EnumTables *tab;
  uint32_t *bits;
  uint64_t r0, lo;  // rank of this lane's first candidate; rank window start
  int32_t M, H, t_lo, t_hi;
  uint32_t my0;
  bool stats;
};

template <int N, unsigned CUTS>
GP_DEV void run_shape(const ShapeItem &c, LaneAcc &acc) {
  constexpr int K = cpopc(CUTS) + 1;
  TaskRegs<N> r;
#pragma unroll
  for (int p = 0; p < N; ++p) {
    const int4 v = c.w->rec[p];
    r.woff[p] = v.x;
    r.D[p] = v.y;
    r.T[p] = v.z;
    r.q[p] = v.w;
  }
  int32_t sr[K];
  int32_t sum = 0;
  {
    int32_t s[K];
    if (c.t_hi > 0) {
      unrank_sizes<K>(*c.tab, K, c.my0, s);
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j) s[j] = 1;
    }
#pragma unroll
    for (int jj = 0; jj < K; ++jj) {
      sr[jj] = s[K - 1 - jj];
      sum += sr[jj];
    }
  }
  const int tmax = (int)__reduce_max_sync(GP_FULL, (unsigned)c.t_hi);
  for (int t = 0; t < tmax; ++t) {
    bool ok = t >= c.t_lo && t < c.t_hi;
    shape_singles<N, CUTS, 0, K>(c.Wt, r, sr, ok);
    shape_multis<N, CUTS, 0, K>(c.Wt, r, sr, c.H, ok, acc, c.stats);
    if (ok) record_ok(acc, c.r0 + (uint32_t)t, sum, c.bits, c.lo);
    if (t + 1 < c.t_hi) next_sizes_rev_static<K>(c.M, sr, sum);
  }
}

template <int N, unsigned C>
GP_DEV void shape_dispatch(unsigned cuts, const ShapeItem &c, LaneAcc &acc) {
  if constexpr (C < (1u << (N - 1))) {
    if (cuts == C) run_shape<N, C>(c, acc);
    else shape_dispatch<N, C + 1>(cuts, c, acc);
  }
}

template <int N, bool kStats>
__global__ void __launch_bounds__(kWarps * 32, 3)
    k_exhaustive_shaped(const ExhArgs a, const ShapeTable sh) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int n = a.n, M = a.M;
  const EnumTables tab = build_enum_tables(smem, M, n);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t off = (enum_table_words(M, n) + 3) & ~(size_t)3;
  const size_t per_warp = ((sizeof(WarpSmem) / 4 + (size_t)2 * n * M) + 3) & ~(size_t)3;
  WarpSmem &w = *reinterpret_cast<WarpSmem *>(smem + off + per_warp * warp);
  int32_t *Wt = reinterpret_cast<int32_t *>(&w + 1);
  const bool stats = kStats && a.stats != nullptr;
  LaneAcc acc;
  int64_t cur = -1;
  int shape = 0;
  for (;;) {
    uint64_t base = 0;
    if (lane == 0) base = atomicAdd(a.work_counter, (unsigned long long)kGrab);
    base = __shfl_sync(GP_FULL, base, 0);
    if (base >= a.total_items) break;
    const uint64_t end = min(base + (uint64_t)kGrab, a.total_items);
    for (uint64_t it = base; it < end; ++it) {
      while (shape + 1 < sh.n_shapes && it >= sh.item_base[shape + 1]) ++shape;
      while (it < sh.item_base[shape]) --shape;
      const int k = sh.k[shape];
      const uint32_t chunks = a.chunks[k];
      const uint64_t local = it - sh.item_base[shape];
      const int64_t set = (int64_t)(local / sh.items_per_set[shape]);
      const uint32_t rem = (uint32_t)(local - (uint64_t)set * sh.items_per_set[shape]);
      const uint32_t e = rem / chunks, c = rem - e * chunks;
      if (set != cur) {
        exh_flush(a, acc, cur, lane);
        cur = set;
        exh_load_set(a, w, Wt, set, lane);
      }
      if (!w.okc) continue;
      const uint32_t ent = sh.entry[sh.first[shape] + e];
      const uint32_t p = ent >> 24;
      const int Lk = a.lane_L[k];
      const uint32_t per_pi = (uint32_t)a.L.per_pi[k];
      const uint64_t rank_pi = a.L.k_base[k] + (uint64_t)p * per_pi;
      const uint32_t rho0 = c * 32u * (uint32_t)Lk;
      if (rank_pi + rho0 >= a.hi || rank_pi + min((uint64_t)per_pi, (uint64_t)rho0 + 32u * Lk) <= a.lo)
        continue;
      // records in block order (block = label; labels ascend with first appearance)
      const int myb = lane < n ? (int)((ent >> (4 * lane)) & 15) : -1;
      uint32_t mine = 0;
      int mypos0 = 0, acc_pos = 0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const uint32_t bm = __ballot_sync(GP_FULL, myb == j);
        if (j == myb) {
          mine = bm;
          mypos0 = acc_pos;
        }
        acc_pos += __popc(bm);
      }
      if (lane < n) {
        const uint32_t same = ((w.memmask >> lane) & 1) ? w.memmask : ~w.memmask;
        const int x = __popc(mine & same) > 1 ? 1 : 0;  // conflict
        const int pos = mypos0 + __popc(mine & ((1u << lane) - 1u));
        w.rec[pos] = make_int4((lane * 2 + x) * M - 1, w.D[lane], w.T[lane], w.q[lane]);
      }
      __syncwarp();
      ShapeItem ctx;
      ctx.Wt = Wt;
      ctx.w = &w;
      ctx.tab = &tab;
      ctx.bits = a.bits ? a.bits + cur * a.words : nullptr;
      ctx.lo = a.lo;
      ctx.M = M;
      ctx.H = w.H;
      ctx.stats = stats;
      ctx.my0 = rho0 + (uint32_t)lane * (uint32_t)Lk;
      ctx.r0 = rank_pi + ctx.my0;
      {
        int t_hi = Lk;
        if (a.hi <= ctx.r0) t_hi = 0;
        else if (a.hi - ctx.r0 < (uint64_t)t_hi) t_hi = (int)(a.hi - ctx.r0);
        if ((int64_t)t_hi > (int64_t)per_pi - (int64_t)ctx.my0)
          t_hi = (int)max((int64_t)0, (int64_t)per_pi - (int64_t)ctx.my0);
        const int t_lo = a.lo > ctx.r0 ? (int)min(a.lo - ctx.r0, (uint64_t)Lk) : 0;
        ctx.t_lo = t_lo;
        ctx.t_hi = t_lo < t_hi ? t_hi : 0;
        if (stats && ctx.t_hi > 0) {
          // every candidate tests all of its single-task blocks (one task each)
          const int n_single = sh.n_single[shape];
          acc.st_cand += (uint64_t)(ctx.t_hi - ctx.t_lo);
          acc.st_blocks += (uint64_t)(ctx.t_hi - ctx.t_lo) * n_single;
          acc.st_tasks += (uint64_t)(ctx.t_hi - ctx.t_lo) * n_single;
        }
      }
      shape_dispatch<N, 0>(sh.cuts[shape], ctx, acc);
      __syncwarp();
    }
  }
  exh_flush(a, acc, cur, lane);
  if constexpr (kStats) exh_stats_flush(a, acc, lane);  // (the timed instantiation: no counters)
}

__global__ void k_exh_init(int64_t *per_set, int32_t n_sets) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_sets;
       g += (int64_t)gridDim.x * blockDim.x) {
    per_set[g * 4 + 0] = 0;
    per_set[g * 4 + 1] = INT64_MAX;
    per_set[g * 4 + 2] = INT64_MAX;
    per_set[g * 4 + 3] = 0;
  }
}

__global__ void k_exh_finalize(const ExhArgs a) {
  // whole warps iterate together (bound rounded up to 32) so the counts can be added once
  // per distinct group per warp (__match_any_sync): consecutive sets share their group
  const int lane = threadIdx.x & 31;
  const int64_t n32 = ((int64_t)a.n_sets + 31) & ~(int64_t)31;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n32;
       g += (int64_t)gridDim.x * blockDim.x) {
    const bool in = g < a.n_sets;
    bool okc = false;
    if (in) {
      int64_t *ps = a.per_set + g * 4;
      okc = set_contract(a, g) > 0;
      if (!okc) {
        ps[0] = -1; ps[1] = 0; ps[2] = -1; ps[3] = 0;
      } else {
        if (ps[1] == INT64_MAX) ps[1] = 0;
        if (ps[2] == INT64_MAX) ps[2] = -1;
      }
    }
    if (a.counts) {
      const int32_t grp = in ? a.group[g] : -1;
      const bool counted = grp >= 0 && grp < a.n_groups;
      const bool valid = counted && okc && a.valid[g];
      const bool exists = valid && a.per_set[g * 4] > 0;
      const uint32_t peers = __match_any_sync(GP_FULL, counted ? grp : -1);
      const uint32_t b_ok = __ballot_sync(GP_FULL, exists), b_inv = __ballot_sync(GP_FULL, counted && !valid);
      if (counted && lane == __ffs(peers) - 1) {
        unsigned long long *c = reinterpret_cast<unsigned long long *>(
            a.counts + (((int64_t)a.setting * a.n_groups + grp) * a.n_slots + a.slot0) * 3);
        if (b_ok & peers) atomicAdd(c + 0, (unsigned long long)__popc(b_ok & peers));
        atomicAdd(c + 1, (unsigned long long)__popc(peers));
        if (b_inv & peers) atomicAdd(c + 2, (unsigned long long)__popc(b_inv & peers));
      }
    }
  }
}

// No host-side caches: the attribute and the occupancy are queried per call (per device,
// thread-safe; microseconds against a launch of milliseconds).
template <int NT>
static gp_status launch_exh(ExhArgs &a, size_t smem, cudaStream_t st) {
  auto kern = a.stats ? k_exhaustive<NT, true> : k_exhaustive<NT, false>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarps * 32, smem);
  if (occ < 1) occ = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (a.total_items + kGrab * kWarps - 1) / (kGrab * kWarps);
  uint64_t grid = (uint64_t)sms * occ;
  if (want < grid) grid = want > 0 ? want : 1;
  kern<<<(unsigned)grid, kWarps * 32, smem, st>>>(a);
  return gp_cuda_check("gp_sched_ratio(EXHAUSTIVE) main kernel");
}

// Host: every RGS of length n in lexicographic order, grouped by shape.
static void build_shape_table(int n, const ExhArgs &a, ShapeTable &sh) {
  struct E {
    uint32_t cuts;
    int k;
    uint32_t entry;
    int n_single;
  };
  E list[kMaxRgs];
  int cnt = 0, lab[kMaxShapeN] = {0}, pcount[kMaxShapeN + 2] = {0};
  for (;;) {
    int k = 0, size[kMaxShapeN] = {0};
    uint32_t packed = 0;
    for (int i = 0; i < n; ++i) {
      k = lab[i] + 1 > k ? lab[i] + 1 : k;
      size[lab[i]] += 1;
      packed |= (uint32_t)lab[i] << (4 * i);
    }
    uint32_t cuts = 0;
    int acc = 0, singles = 0;
    for (int j = 0; j < k; ++j) {
      acc += size[j];
      singles += size[j] == 1;
      if (j < k - 1) cuts |= 1u << (acc - 1);
    }
    if (k <= a.L.kmax)  // k blocks need k <= M SMs
      list[cnt++] = E{cuts, k, packed | ((uint32_t)pcount[k]++ << 24), singles};
    int i = n - 1;  // lexicographic RGS successor
    for (; i >= 1; --i) {
      int mx = 0;
      for (int j = 0; j < i; ++j) mx = lab[j] > mx ? lab[j] : mx;
      if (lab[i] <= mx) break;
    }
    if (i < 1) break;
    lab[i] += 1;
    for (int j = i + 1; j < n; ++j) lab[j] = 0;
  }
  // stable grouping by shape (cuts ascending), lexicographic order kept inside
  sh.n_shapes = 0;
  int e = 0;
  uint64_t items = 0;
  for (uint32_t c = 0; c < (1u << (n - 1)); ++c) {
    const int first = e;
    int k = 0, singles = 0;
    for (int x = 0; x < cnt; ++x)
      if (list[x].cuts == c) {
        sh.entry[e++] = list[x].entry;
        k = list[x].k;
        singles = list[x].n_single;
      }
    if (e == first) continue;
    const int sidx = sh.n_shapes++;
    sh.cuts[sidx] = c;
    sh.k[sidx] = k;
    sh.first[sidx] = first;
    sh.n_single[sidx] = singles;
    sh.items_per_set[sidx] = (uint32_t)(e - first) * a.chunks[k];
    sh.item_base[sidx] = items;
    items += (uint64_t)sh.items_per_set[sidx] * (uint64_t)a.n_sets;
  }
  sh.first[sh.n_shapes] = e;
  sh.item_base[sh.n_shapes] = items;
}

template <int N>
static gp_status launch_shaped(ExhArgs &a, size_t smem, cudaStream_t st) {
  ShapeTable sh;  // host staging (per call), copied into the kernel parameters
  build_shape_table(N, a, sh);
  if (sh.item_base[sh.n_shapes] != a.total_items)
    return gp_fail(GP_EINVAL, "EXHAUSTIVE: shape table does not cover the candidate space");
  auto kern = a.stats ? k_exhaustive_shaped<N, true> : k_exhaustive_shaped<N, false>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarps * 32, smem);
  if (occ < 1) occ = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (a.total_items + kGrab * kWarps - 1) / (kGrab * kWarps);
  uint64_t grid = (uint64_t)sms * occ;
  if (want < grid) grid = want > 0 ? want : 1;
  kern<<<(unsigned)grid, kWarps * 32, smem, st>>>(a, sh);
  return gp_cuda_check("gp_sched_ratio(EXHAUSTIVE) shaped kernel");
}

}  // namespace gp

gp_status gp_exhaustive_bp_launch(const gp::ExhArgs &a, void *ws, uint64_t ws_bytes,
                                  uint64_t *tables_key, cudaStream_t st);
size_t gp_exhaustive_bp_workspace(const gp::RankLayout &L, int n, int M, int32_t n_sets,
                                  int32_t n_groups, uint32_t flags);

// Workspace of gp_sched_ratio for these shapes (gpart.h): the bit-sliced evaluator's
// memo / lane-order / hash tables; 0 for the per-candidate and threshold evaluators.
extern "C" gp_status gp_exhaustive_workspace_size(int32_t n_sets, int32_t n_tasks, int32_t M,
                                                  int32_t n_groups, gp_ratio_mode mode,
                                                  uint32_t flags, uint64_t *bytes) {
  using namespace gp;
  if (!bytes) return gp_fail(GP_EINVAL, "gp_exhaustive_workspace_size: null output");
  if (n_sets < 0 || n_tasks < 1 || n_tasks > kEnumMaxTasks || M < 1 || M > kEnumMaxM)
    return gp_fail(GP_EINVAL, "gp_exhaustive_workspace_size: need n_tasks <= 12, M <= 256");
  *bytes = 0;
  if (mode == GP_EXHAUSTIVE && !(flags & (GP_EX_PER_CANDIDATE | GP_EX_GENERIC))) {
    RankLayout L;
    gp_status s = rank_layout(M, n_tasks, &L, true);
    if (s != GP_OK) return s;
    *bytes = gp_exhaustive_bp_workspace(L, n_tasks, M, n_sets, n_groups, flags);
  }
  return gp_ok();
}

// Called by gp_sched_ratio (ratio.cu) for GP_EXHAUSTIVE.
gp_status gp_exhaustive_launch(const gp_tasksets *ts, int32_t slot0, int32_t n_slots,
                               int32_t setting, int64_t *counts, const gp_exhaustive_opts *ex,
                               cudaStream_t st) {
  using namespace gp;
  const int n = ts->n_tasks, M = ts->M;
  if (n < 1 || n > kEnumMaxTasks || M < 1 || M > kEnumMaxM)
    return gp_fail(GP_EINVAL, "EXHAUSTIVE: need n_tasks <= 12 and M <= 256 (n=%d M=%d)", n, M);
  if (!ex || !ex->per_set || !ex->work_counter)
    return gp_fail(GP_EINVAL, "EXHAUSTIVE: opts, per_set and work_counter are required");
  ExhArgs a;
  gp_status s = rank_layout(M, n, &a.L, true);
  if (s != GP_OK) return s;
  a.lo = ex->rank_lo;
  a.hi = ex->rank_hi > a.L.total ? a.L.total : ex->rank_hi;
  if (a.lo > a.hi) return gp_fail(GP_EINVAL, "EXHAUSTIVE: rank_lo > rank_hi");
  const bool full = a.lo == 0 && a.hi == a.L.total;
  if (counts && !full) return gp_fail(GP_EINVAL, "EXHAUSTIVE: counts need the full rank window");
  if (ex->verdict_bits && (uint64_t)ex->words_per_set * 32 < a.hi - a.lo)
    return gp_fail(GP_EINVAL, "EXHAUSTIVE: words_per_set too small for the window");
  a.T = ts->T; a.D = ts->D; a.B = ts->B; a.cn = ts->cn; a.cc = ts->cc; a.fn = ts->fn;
  a.fc = ts->fc; a.group = ts->group; a.type = ts->type; a.valid = ts->valid;
  a.n_sets = ts->n_sets; a.n = n; a.M = M; a.n_groups = ts->n_groups;
  a.per_set = ex->per_set; a.bits = ex->verdict_bits; a.words = ex->words_per_set;
  a.counts = counts; a.slot0 = slot0; a.n_slots = n_slots; a.setting = setting;
  a.stats = ex->stats; a.work_counter = ex->work_counter;
  if (ex->flags & ~(uint32_t)(GP_EX_NO_HASH | GP_EX_PER_CANDIDATE | GP_EX_STATS_EXT |
                              GP_EX_FORCE_RANGES | GP_EX_NATURAL_ORDER | GP_EX_GENERIC |
                              GP_EX_NO_FULL_CORNER))
    return gp_fail(GP_EINVAL, "EXHAUSTIVE: unknown flags 0x%x", ex->flags);
  a.flags = ex->flags;
  s = load_size_mask(ex->size_mask, M, a.adm, "EXHAUSTIVE");
  if (s != GP_OK) return s;
  uint64_t items = 0;
  for (int k = 1; k <= a.L.kmax; ++k) {
    // balanced chunks of at most 32 * kMaxL size vectors of one allocation
    const uint64_t per = a.L.per_pi[k];
    const uint64_t chunks = (per + 32ull * kMaxL - 1) / (32ull * kMaxL);
    const int Lk = (int)((per + 32ull * chunks - 1) / (32ull * chunks));
    a.lane_L[k] = Lk;
    a.chunks[k] = (uint32_t)chunks;
    a.item_base[k] = items;
    items += a.L.n_pi[k] * a.chunks[k];
  }
  a.items_per_set = items;
  a.total_items = items * (uint64_t)ts->n_sets;
  if (ts->n_sets == 0) return gp_cuda_check("EXHAUSTIVE");
  if (ex->verdict_bits)
    cudaMemsetAsync(ex->verdict_bits, 0, (size_t)ts->n_sets * ex->words_per_set * 4, st);
  cudaMemsetAsync(ex->work_counter, 0, 8, st);
  int64_t g1 = (ts->n_sets + 255) / 256;
  k_exh_init<<<(unsigned)(g1 > 4096 ? 4096 : g1), 256, 0, st>>>(ex->per_set, ts->n_sets);
  // default for n <= 8, M <= 32: bit-sliced verdicts over memoised block
  // verdicts (exhaustive_bp.cu); otherwise, or on request, per candidate
  if (n <= 8 && M <= 32 && !(ex->flags & (GP_EX_PER_CANDIDATE | GP_EX_GENERIC))) {
    gp_status r = gp_exhaustive_bp_launch(a, ex->workspace, ex->workspace_bytes, ex->tables_key, st);
    if (r != GP_OK) return r;
    k_exh_finalize<<<(unsigned)(g1 > 4096 ? 4096 : g1), 256, 0, st>>>(a);
    return gp_cuda_check("gp_sched_ratio(EXHAUSTIVE) finalize");
  }
  const size_t wt_words = (size_t)2 * n * M;
  const size_t per_warp = ((sizeof(WarpSmem) / 4 + wt_words) + 3) & ~(size_t)3;
  const size_t smem = (((enum_table_words(M, n) + 3) & ~(size_t)3) + per_warp * kWarps) * 4;
  if (smem > 227 * 1024) return gp_fail(GP_EINVAL, "EXHAUSTIVE: shared memory need %zu B too large", smem);
  gp_status r;
  if (n <= kMaxShapeN && !(ex->flags & GP_EX_GENERIC)) {
    switch (n) {
      case 1: r = launch_shaped<1>(a, smem, st); break;
      case 2: r = launch_shaped<2>(a, smem, st); break;
      case 3: r = launch_shaped<3>(a, smem, st); break;
      case 4: r = launch_shaped<4>(a, smem, st); break;
      case 5: r = launch_shaped<5>(a, smem, st); break;
      default: r = launch_shaped<6>(a, smem, st); break;
    }
    if (r != GP_OK) return r;
    k_exh_finalize<<<(unsigned)(g1 > 4096 ? 4096 : g1), 256, 0, st>>>(a);
    return gp_cuda_check("gp_sched_ratio(EXHAUSTIVE) finalize");
  }
  switch (n) {
    case 1: case 2: case 3: r = launch_exh<3>(a, smem, st); break;
    case 4: r = launch_exh<4>(a, smem, st); break;
    case 5: r = launch_exh<5>(a, smem, st); break;
    case 6: r = launch_exh<6>(a, smem, st); break;
    case 7: case 8: r = launch_exh<8>(a, smem, st); break;
    default: r = launch_exh<12>(a, smem, st); break;
  }
  if (r != GP_OK) return r;
  k_exh_finalize<<<(unsigned)(g1 > 4096 ? 4096 : g1), 256, 0, st>>>(a);
  return gp_cuda_check("gp_sched_ratio(EXHAUSTIVE) finalize");
}
