// exhaustive_bp.cu -- the default GP_EXHAUSTIVE evaluator for n <= 8 tasks and
// M <= 32 SMs: bit-sliced candidate verdicts over memoised block verdicts.
//
// C.1.8: a candidate (pi, s) is schedulable iff every block S_j of pi passes
// the EDF processor-demand test (C.1.7) at its size s_j.  That block verdict
// depends only on (S_j, s_j) within a set, so it is computed ONCE per
// (subset, size) instead of once per (candidate, block):
//   k_exh_memo: per set, V[S] = bitmask over sizes (bit m-1 = S schedulable on
//   m SMs) for all 2^n - 1 task subsets S -- C3: 63 x 20 = 1,260 EDF tests per
//   set where the per-candidate evaluator runs ~2.3 million.  Every (S, m) is
//   tested; no monotonicity in m is assumed (that is f3's GP_THRESHOLD).
//   k_exh_bp: the same work items, rank windows and lexicographic candidate
//   order as the per-candidate kernel (exhaustive.cu).  Candidates of one
//   allocation with a common prefix (s_0..s_{k-2}) form a RUN in which only
//   the last part moves (1 .. M - prefix sum); a lane evaluates a whole run
//   segment in one word:  prefix_ok ? (V_{k-1} >> (s_{k-1} - 1)) & seg_mask : 0,
//   i.e. up to 32 candidate verdicts per word operation, then records the set
//   bits (count by popcount; pi* and first rank from the lowest bit; the
//   verdict hash bit by bit; verdict bits with word-level atomics).
// Outputs are byte-identical to the per-candidate evaluator (GP_EX_PER_CANDIDATE
// selects that one, for A/B runs and parity).
#include "gp_common.cuh"
#include "gp_edf.cuh"
#include "gp_enum.cuh"
#include "gp_exh.cuh"

namespace gp {

constexpr int kBpMaxN = 8;   // tasks per set (2^8 subset words per set)
constexpr int kBpMaxM = 32;  // sizes per verdict word

// ---- pre-pass: V[set][S] for every subset S, one warp per set, lane = size --
__global__ void __launch_bounds__(256) k_exh_memo(const ExhArgs a, uint32_t *memo) {
  const int lane = threadIdx.x & 31;
  const int n = a.n, M = a.M;
  const int nsub = 1 << n;
  uint64_t st_tests = 0, st_tasks = 0;
  uint32_t st_events = 0;
  for (int64_t set = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; set < a.n_sets;
       set += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t H = set_contract(a, set);
    uint32_t *V = memo + set * nsub;
    if (lane == 0) V[0] = H > 0 ? 1u : 0u;  // word 0: the set's input contract
    if (H <= 0) continue;
    const int32_t H32 = (int32_t)H;
    // task i's fields in registers of every lane (n <= 8)
    int32_t T[kBpMaxN], D[kBpMaxN], B[kBpMaxN], cn[kBpMaxN], cc[kBpMaxN], fn[kBpMaxN],
        fc[kBpMaxN], q[kBpMaxN];
    uint32_t mem = 0;
#pragma unroll
    for (int i = 0; i < kBpMaxN; ++i) {
      const bool v = i < n;
      const int64_t o = set * n + (v ? i : 0);
      T[i] = v ? a.T[o] : INT32_MAX;
      D[i] = v ? a.D[o] : INT32_MAX;
      B[i] = v ? a.B[o] : 1;
      cn[i] = v ? a.cn[o] : 0;
      cc[i] = v ? a.cc[o] : 0;
      fn[i] = v ? a.fn[o] : 0;
      fc[i] = v ? a.fc[o] : 0;
      q[i] = v ? (int32_t)(H / T[i]) : 0;
      mem |= (v && a.type[o] == 1) ? 1u << i : 0u;
    }
    const int32_t m = lane + 1;  // this lane's size
    for (int S = 1; S < nsub; ++S) {
      bool ok = false;
      if (m <= M) {
        const int cnt = __popc((unsigned)S);
        int32_t C[kBpMaxN], Dv[kBpMaxN], Tv[kBpMaxN], qv[kBpMaxN];
        bool bad = false;
#pragma unroll
        for (int i = 0; i < kBpMaxN; ++i) {
          const bool in = (S >> i) & 1;
          const uint32_t same = ((mem >> i) & 1u) ? mem : ~mem;
          const bool x = __popc((unsigned)S & same) > 1;  // conflict
          C[i] = in ? (x ? wcet_sat(B[i], cc[i], fc[i], m) : wcet_sat(B[i], cn[i], fn[i], m)) : 0;
          Dv[i] = in ? D[i] : INT32_MAX;
          Tv[i] = in ? T[i] : INT32_MAX;
          qv[i] = in ? q[i] : 0;
          bad |= C[i] > Dv[i];
        }
        ++st_tests;
        st_tasks += cnt;
        if (!bad) {
          if (cnt == 1) {
            ok = true;  // a single task: C <= D decides (gp_edf.cuh shortcut 1)
          } else {
            int32_t UH = 0;
#pragma unroll
            for (int i = 0; i < kBpMaxN; ++i) UH += C[i] * qv[i];
            if (UH <= H32) {
              const int32_t lcut = pdc_cutoff<kBpMaxN>(C, Dv, Tv, qv, H32, UH);
              ok = pdc_walk<kBpMaxN>(C, Dv, Tv, lcut, st_events);
            }
          }
        }
      }
      const uint32_t word = __ballot_sync(GP_FULL, ok);
      if (lane == (S & 31)) V[S] = word;
    }
  }
  if (a.stats) {
    const uint64_t t0 = warp_sum_u64(st_tests), t1 = warp_sum_u64(st_tasks);
    const uint64_t t2 = warp_sum_u64((uint64_t)st_events);
    if (lane == 0) {
      atomicAdd(a.stats + 1, (unsigned long long)t0);
      atomicAdd(a.stats + 2, (unsigned long long)t2);
      atomicAdd(a.stats + 3, (unsigned long long)t1);
    }
  }
}

// ---- main pass: bit-sliced verdicts over runs ---------------------------------
__global__ void __launch_bounds__(kWarps * 32, 4) k_exh_bp(const ExhArgs a, const uint32_t *memo) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int n = a.n, M = a.M;
  const EnumTables tab = build_enum_tables(smem, M, n);
  const int lane = threadIdx.x & 31;
  const int nsub = 1 << n;
  const bool want_hash = !(a.flags & GP_EX_NO_HASH);
  LaneAcc acc;
  int64_t cur = -1;
  bool okc = false;
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
        exh_flush(a, acc, cur, lane);
        cur = set;
        okc = memo[set * nsub] != 0;
      }
      if (!okc) continue;  // contract violation: finalize reports it
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
      // allocation pi: block j's task mask -> its verdict word V[S_j]; reversed
      // into Vr[jj] = word of block k-1-jj to match the reversed sizes
      const uint64_t labels = unrank_rgs(tab, k, p);
      const int myb = lane < n ? (int)((labels >> (4 * lane)) & 15) : -1;
      uint32_t bmask = 0;
#pragma unroll
      for (int j = 0; j < kBpMaxN; ++j) {
        const uint32_t bm = __ballot_sync(GP_FULL, myb == j);
        if (lane == j) bmask = bm;
      }
      const uint32_t vw = lane < k ? memo[set * nsub + bmask] : 0u;
      uint32_t Vr[kBpMaxN];
#pragma unroll
      for (int jj = 0; jj < kBpMaxN; ++jj) Vr[jj] = __shfl_sync(GP_FULL, vw, max(k - 1 - jj, 0));
      // this lane's candidates: s-index my0 + t, t in [t_lo, t_hi)
      const uint32_t my0 = rho0 + (uint32_t)lane * (uint32_t)Lk;
      const uint64_t r0 = rank_pi + my0;
      int t_hi = Lk;
      if (a.hi <= r0) t_hi = 0;
      else if (a.hi - r0 < (uint64_t)t_hi) t_hi = (int)(a.hi - r0);
      if ((int64_t)t_hi > (int64_t)per_pi - (int64_t)my0)
        t_hi = (int)max((int64_t)0, (int64_t)per_pi - (int64_t)my0);
      const int t_lo = a.lo > r0 ? (int)min(a.lo - r0, (uint64_t)Lk) : 0;
      if (t_lo < t_hi) {  // no warp collective inside
        int32_t sr[kBpMaxN];
        int32_t sum = 0;
        {
          int32_t s[kBpMaxN];
          unrank_sizes<kBpMaxN>(tab, k, my0 + (uint32_t)t_lo, s);
#pragma unroll
          for (int jj = 0; jj < kBpMaxN; ++jj) {
            sr[jj] = 1;
#pragma unroll
            for (int j = 0; j < kBpMaxN; ++j)
              if (j == k - 1 - jj) sr[jj] = s[j];
            sum += jj < k ? sr[jj] : 0;
          }
        }
        acc.st_cand += (uint64_t)(t_hi - t_lo);
        uint32_t *bits = a.bits ? a.bits + cur * a.words : nullptr;
        int t = t_lo;
        for (;;) {
          // the run segment: last part sr[0] .. sr[0] + seg - 1
          const int seg = min(M - sum + 1, t_hi - t);
          uint32_t pre = 1u;
#pragma unroll
          for (int jj = 1; jj < kBpMaxN; ++jj)
            if (jj < k) pre &= Vr[jj] >> (sr[jj] - 1);
          uint32_t okb = 0;
          if (pre & 1u) {
            okb = Vr[0] >> (sr[0] - 1);
            if (seg < 32) okb &= (1u << seg) - 1u;
          }
          if (okb) {
            const int fb = __ffs(okb) - 1;
            const uint64_t rk = r0 + (uint32_t)t;
            acc.n += __popc(okb);
            acc.pi = min(acc.pi, sum + fb);
            acc.first = min(acc.first, rk + (uint64_t)fb);
            if (want_hash) {
              uint32_t w = okb;
              while (w) {
                const int b = __ffs(w) - 1;
                w &= w - 1u;
                acc.hash += splitmix64(rk + (uint64_t)b);
              }
            }
            if (bits) {  // verdict bits of the segment, word-level
              const uint64_t off = rk - a.lo;
              const uint32_t sh = (uint32_t)(off & 31u);
              atomicOr(bits + (off >> 5), okb << sh);
              if (sh && (okb >> (32u - sh))) atomicOr(bits + (off >> 5) + 1, okb >> (32u - sh));
            }
          }
          t += seg;
          if (t >= t_hi) break;
          sr[0] += seg - 1;  // end of this run (sum == M), then the lexicographic successor
          sum += seg - 1;
          next_sizes_rev<kBpMaxN>(M, k, sr, sum);
        }
      }
    }
  }
  exh_flush(a, acc, cur, lane);
  if (a.stats) {
    const uint64_t c0 = warp_sum_u64(acc.st_cand);
    if (lane == 0) atomicAdd(a.stats + 0, c0);
  }
}

}  // namespace gp

// Called by gp_exhaustive_launch (exhaustive.cu) when n <= 8, M <= 32 and the
// caller did not ask for the per-candidate evaluator.  `a` is fully set up
// (items, rank window, per_set initialised); finalize runs after.
gp_status gp_exhaustive_bp_launch(const gp::ExhArgs &a, cudaStream_t st) {
  using namespace gp;
  const int n = a.n, M = a.M;
  if (n > kBpMaxN || M > kBpMaxM) return gp_fail(GP_EINVAL, "EXHAUSTIVE(bp): n <= 8, M <= 32");
  uint32_t *memo = nullptr;
  const size_t bytes = (size_t)a.n_sets * ((size_t)1 << n) * sizeof(uint32_t);
  if (cudaMallocAsync(reinterpret_cast<void **>(&memo), bytes, st) != cudaSuccess)
    return gp_cuda_check("EXHAUSTIVE(bp): workspace allocation");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  {
    int64_t blocks = ((int64_t)a.n_sets + 7) / 8;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    k_exh_memo<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, st>>>(a, memo);
  }
  gp_status r = gp_cuda_check("EXHAUSTIVE(bp) memo kernel");
  if (r == GP_OK) {
    const size_t smem = ((enum_table_words(M, n) + 3) & ~(size_t)3) * 4;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_exh_bp, kWarps * 32, smem);
    if (occ < 1) occ = 1;
    uint64_t want = (a.total_items + kGrab * kWarps - 1) / (kGrab * kWarps);
    uint64_t grid = (uint64_t)sms * occ;
    if (want < grid) grid = want > 0 ? want : 1;
    k_exh_bp<<<(unsigned)grid, kWarps * 32, smem, st>>>(a, memo);
    r = gp_cuda_check("EXHAUSTIVE(bp) main kernel");
  }
  cudaFreeAsync(memo, st);
  return r;
}
