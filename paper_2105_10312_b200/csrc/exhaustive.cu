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

#include "gp_common.cuh"
#include "gp_edf.cuh"
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
  uint64_t items_per_set, total_items;
  uint64_t item_base[kEnumMaxTasks + 2];
  uint32_t chunks[kEnumMaxTasks + 2];
  int32_t lane_L[kEnumMaxTasks + 2];
};

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

template <int NT>
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
  const bool stats = a.stats != nullptr;

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
            Wt[e] = x ? wcet_sat(a.B[o], a.cc[o], a.fc[o], s) : wcet_sat(a.B[o], a.cn[o], a.fn[o], s);
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
  if (stats) {
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
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.n_sets;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t *ps = a.per_set + g * 4;
    const bool okc = set_contract(a, g) > 0;
    if (!okc) {
      ps[0] = -1; ps[1] = 0; ps[2] = -1; ps[3] = 0;
    } else {
      if (ps[1] == INT64_MAX) ps[1] = 0;
      if (ps[2] == INT64_MAX) ps[2] = -1;
    }
    if (a.counts) {
      const int32_t grp = a.group[g];
      if (grp < 0 || grp >= a.n_groups) continue;
      const bool valid = okc && a.valid[g];
      const bool exists = okc && ps[0] > 0;
      unsigned long long *c = reinterpret_cast<unsigned long long *>(
          a.counts + (((int64_t)a.setting * a.n_groups + grp) * a.n_slots + a.slot0) * 3);
      if (exists && valid) atomicAdd(c + 0, 1ull);
      atomicAdd(c + 1, 1ull);
      if (!valid) atomicAdd(c + 2, 1ull);
    }
  }
}

template <int NT>
static gp_status launch_exh(ExhArgs &a, size_t smem, cudaStream_t st) {
  static int occ = -1;
  static size_t occ_smem = 0;
  if (occ < 0 || occ_smem != smem) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_exhaustive<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_exhaustive<NT>, kWarps * 32, smem);
    occ_smem = smem;
    if (occ < 1) occ = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t want = (a.total_items + kGrab * kWarps - 1) / (kGrab * kWarps);
  uint64_t grid = (uint64_t)sms * occ;
  if (want < grid) grid = want > 0 ? want : 1;
  k_exhaustive<NT><<<(unsigned)grid, kWarps * 32, smem, st>>>(a);
  return gp_cuda_check("gp_sched_ratio(EXHAUSTIVE) main kernel");
}

}  // namespace gp

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
  const size_t wt_words = (size_t)2 * n * M;
  const size_t per_warp = ((sizeof(WarpSmem) / 4 + wt_words) + 3) & ~(size_t)3;
  const size_t smem = (((enum_table_words(M, n) + 3) & ~(size_t)3) + per_warp * kWarps) * 4;
  if (smem > 227 * 1024) return gp_fail(GP_EINVAL, "EXHAUSTIVE: shared memory need %zu B too large", smem);
  gp_status r;
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
