// threshold.cu -- §8(f) f3: the subset-threshold exhaustive evaluator
// (gp_sched_ratio mode GP_THRESHOLD).  Same per-set outputs as GP_EXHAUSTIVE,
// a different work unit: it does NOT test every candidate.
//
// Exactness (resource monotonicity, P:445 / S:175): W_i(m, x) is
// non-increasing in m and the conflict flags of a block do not depend on m,
// so EDF-PDC(S, s) is monotone in s.  With m*(S) = min{s in 1..M : EDF-PDC(S,s)}
// (M+1 if none), a candidate (pi, s) is schedulable iff s_j >= m*(S_j) for
// every block j.  Hence, per allocation pi with blocks S_0..S_{k-1}:
//   * its schedulable size vectors are s = m* + (s' - 1), s' >= 1,
//     sum(s') <= R = M - sum(m*_j - 1): there are C(R, k) of them;
//   * the lexicographically first one is s = m* itself;
//   * the minimum sum over them is sum(m*_j).
// So n_sched, pi_star and first_rank follow in closed form from the 2^n - 1
// thresholds; the verdict hash (sum of splitmix64 over schedulable ranks) is
// computed by enumerating the schedulable vectors only (skippable).
//
// Layout: one warp per set.  Phase 1: lanes = subsets; m*(S) by binary search
// over s (exact by monotonicity) with a lane-serial EDF-PDC (gp_edf.cuh).
// Phase 2: lanes = allocations (RGS); closed-form counts; optional hash walk.
#include "gp_common.cuh"
#include "gp_edf.cuh"
#include "gp_enum.cuh"

namespace gp {

constexpr int kThrWarps = 4;

struct ThrArgs {
  const int32_t *T, *D, *B, *cn, *cc, *fn, *fc, *group;
  const uint8_t *type, *valid;
  int32_t n_sets, n, M, n_groups;
  RankLayout L;
  int64_t *per_set;
  int64_t *counts;
  int32_t slot0, n_slots, setting, want_hash;
  unsigned long long *stats;  // += {sets, threshold tests, deadlines examined, schedulable enumerated}
  int32_t masked;             // f4 size mask given (reading B-9)
  uint32_t adm[8];            // admissible sizes, bit (m-1) % 32 of word (m-1) / 32
  unsigned long long *next;   // set counter (persistent warps take sets dynamically) or null
};

// f4 (reading B-9): first admissible size >= x, M + 1 if none.
GP_DEV int next_admissible(const ThrArgs &a, int x) {
  for (; x <= a.M; ++x)
    if ((a.adm[(x - 1) >> 5] >> ((x - 1) & 31)) & 1u) return x;
  return a.M + 1;
}

GP_DEV int64_t thr_contract(const ThrArgs &a, int64_t set) {
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

// EDF-PDC of subset S at size s, lane-serial over up to NT tasks.
template <int NT>
GP_DEV bool subset_pdc(uint32_t S, int32_t s, int n, int M, const int32_t *Wt, const int32_t *Dv,
                       const int32_t *Tv, const int32_t *qv, uint32_t memmask, int32_t H,
                       uint32_t &events) {
  int32_t C[NT], D[NT], T[NT], q[NT];
  bool bad = false;
  const int cnt = __popc(S);
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const bool in = i < n && ((S >> i) & 1u);
    const uint32_t same = ((memmask >> i) & 1u) ? memmask : ~memmask;
    const int x = __popc(S & same) > 1 ? 1 : 0;  // conflict
    C[i] = in ? Wt[(i * 2 + x) * M + s - 1] : 0;
    D[i] = in ? Dv[i] : INT32_MAX;
    T[i] = in ? Tv[i] : INT32_MAX;
    q[i] = in ? qv[i] : 0;
    bad |= C[i] > D[i];
  }
  if (bad) return false;
  if (cnt == 1) return true;
  int32_t UH = 0;
#pragma unroll
  for (int i = 0; i < NT; ++i) UH += C[i] * q[i];
  if (UH > H) return false;
  const int32_t lcut = pdc_cutoff<NT>(C, D, T, q, H, UH);
  return pdc_walk<NT>(C, D, T, lcut, events);
}

// lexicographic rank of the size vector s (k parts, sum <= M) among all such
// vectors: hockey-stick form of sum_j sum_{v=c_{j-1}+1}^{c_j-1} C(M-v, k-1-j)
template <int NT>
GP_DEV uint32_t lexrank_sizes(const EnumTables &t, int M, int k, const int32_t (&s)[NT]) {
  uint32_t r = 0;
  int prev = 0, c = 0;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < k) {
      c += s[j];
      r += t.C(M - prev, k - j) - t.C(M - c + 1, k - j);
      prev = c;
    }
  }
  return r;
}

// Phase 2 of one allocation under an admissible-size mask (f4, reading B-9).
// Block j is schedulable at s iff s >= m*_j (monotonicity, on the unmasked W) and
// s is admissible, so the schedulable vectors are prod_j A_j with A_j = {s in A :
// s >= m*_j}, sum <= M.  lo_j = min A_j: pi* = sum lo_j, the lexicographically first
// vector is lo.  The rest is walked run by run (a run: fixed s_0..s_{k-2}, last
// part v = lo_{k-1} .. M - prefix; candidate rank = rank(prefix, 1) + v - 1):
// the count adds the admissible v of each run, the hash their splitmix64.
template <int NT>
GP_DEV void thr_masked_alloc(const ThrArgs &a, const EnumTables &tab, int k, uint64_t rank_pi,
                             const int32_t (&m)[NT], uint64_t &n_sched, int32_t &pi_star,
                             uint64_t &first, uint64_t &hash, uint64_t &st_sched) {
  const int M = a.M;
  int32_t lo[NT], s[NT];
  int sum_lo = 0;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    lo[j] = j < k ? next_admissible(a, m[j]) : 0;
    if (j < k) sum_lo += lo[j];
    s[j] = lo[j];
  }
  if (sum_lo > M) return;  // also covers an empty A_j (lo_j = M + 1)
  pi_star = min(pi_star, sum_lo);
  const uint64_t r_first = rank_pi + lexrank_sizes(tab, M, k, lo);
  first = r_first < first ? r_first : first;
  int lo_last = 0;
#pragma unroll
  for (int j = 0; j < NT; ++j)
    if (j == k - 1) lo_last = lo[j];
  for (;;) {
    int prefix = 0;  // s_0 + ... + s_{k-2}
    int32_t s1[NT];  // (prefix, 1): rank base of the run
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j < k - 1) prefix += s[j];
      s1[j] = j == k - 1 ? 1 : s[j];
    }
    const uint64_t base = rank_pi + lexrank_sizes(tab, M, k, s1);
    uint64_t cnt = 0;
    for (int v = lo_last; v <= M - prefix; ++v) {
      if (!((a.adm[(v - 1) >> 5] >> ((v - 1) & 31)) & 1u)) continue;
      ++cnt;
      if (a.want_hash) hash += splitmix64(base + (uint64_t)(v - 1));
    }
    n_sched += cnt;
    if (a.want_hash) st_sched += cnt;
    // next prefix: the rightmost part j <= k-2 that can move to its next admissible
    // size with the parts after it reset to their minima
    int pick = -1, nxt = 0, before = 0;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j < k - 1) {
        int after = lo_last;  // minima of the parts after j
#pragma unroll
        for (int i = j + 1; i < NT; ++i)
          if (i < k - 1) after += lo[i];
        const int x = next_admissible(a, s[j] + 1);
        if (before + x + after <= M) {
          pick = j;
          nxt = x;
        }
        before += s[j];
      }
    }
    if (pick < 0) break;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j == pick) s[j] = nxt;
      else if (j > pick && j < k - 1) s[j] = lo[j];
    }
  }
}

__host__ __device__ inline size_t thr_warp_words(int n, int M) {
  return ((size_t)2 * n * M + 3 * 16 + ((size_t)1 << n) / 2 + 4 + 3) & ~(size_t)3;
}

template <int NT>
__global__ void __launch_bounds__(kThrWarps * 32) k_threshold(const ThrArgs a) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int n = a.n, M = a.M;
  const EnumTables tab = build_enum_tables(smem, M, n);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t off = (enum_table_words(M, n) + 3) & ~(size_t)3;
  const size_t per_warp = thr_warp_words(n, M);
  int32_t *Wt = reinterpret_cast<int32_t *>(smem + off + per_warp * warp);
  int32_t *Dv = Wt + 2 * n * M;
  int32_t *Tv = Dv + 16;
  int32_t *qv = Tv + 16;
  uint16_t *mstar = reinterpret_cast<uint16_t *>(qv + 16);  // [2^n], index = subset mask
  const int nsub = 1 << n;
  uint64_t st_tests = 0, st_sched = 0;
  uint32_t st_events = 0;
  uint64_t st_sets = 0;
  // sets from a counter (they differ widely in work) or, without one, a static stride
  auto next_set = [&](int64_t cur) -> int64_t {
    if (a.next) {
      unsigned long long s0 = 0;
      if (lane == 0) s0 = atomicAdd(a.next, 1ull);
      return (int64_t)__shfl_sync(GP_FULL, s0, 0);
    }
    return cur < 0 ? (int64_t)blockIdx.x * kThrWarps + warp : cur + (int64_t)gridDim.x * kThrWarps;
  };
  for (int64_t set = next_set(-1); set < a.n_sets; set = next_set(set)) {
    const int64_t H64 = thr_contract(a, set);
    int64_t *ps = a.per_set + set * 4;
    if (H64 <= 0) {
      if (lane == 0) {
        ps[0] = -1; ps[1] = 0; ps[2] = -1; ps[3] = 0;
      }
      continue;
    }
    const int32_t H = (int32_t)H64;
    st_sets += 1;
    __syncwarp();
    if (lane < n) {
      const int64_t o = set * n + lane;
      Dv[lane] = a.D[o];
      Tv[lane] = a.T[o];
      qv[lane] = (int32_t)(H / a.T[o]);
    }
    const uint32_t memmask =
        __ballot_sync(GP_FULL, lane < n && a.type[set * n + min(lane, n - 1)] == 1);
    for (int e = lane; e < 2 * n * M; e += 32) {
      const int i = e / (2 * M), x = (e / M) & 1, s = e % M + 1;
      const int64_t o = set * n + i;
      Wt[e] = x ? wcet_sat(a.B[o], a.cc[o], a.fc[o], s) : wcet_sat(a.B[o], a.cn[o], a.fn[o], s);
    }
    __syncwarp();
    // ---- phase 1: m*(S) for every non-empty subset, binary search over s
    for (uint32_t S = 1 + lane; S < (uint32_t)nsub; S += 32) {
      int lo = 1, hi = M + 1;  // answer in [lo, hi]; hi = M+1 means "none"
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        ++st_tests;
        if (subset_pdc<NT>(S, mid, n, M, Wt, Dv, Tv, qv, memmask, H, st_events)) hi = mid;
        else lo = mid + 1;
      }
      mstar[S] = (uint16_t)lo;
    }
    __syncwarp();
    // ---- phase 2: allocations pi (lanes), closed-form counts
    uint64_t n_sched = 0, hash = 0, first = ~0ull;
    int32_t pi_star = INT32_MAX;
    for (int k = 1; k <= a.L.kmax; ++k) {
      const uint32_t n_pi = (uint32_t)a.L.n_pi[k];
      const uint32_t per_pi = (uint32_t)a.L.per_pi[k];
      for (uint32_t p = lane; p < n_pi; p += 32) {
        const uint64_t labels = unrank_rgs(tab, k, p);
        int32_t m[NT];
        int sum_m = 0;
        bool feasible = true;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          uint32_t mask = 0;
#pragma unroll
          for (int i = 0; i < NT; ++i)
            if (i < n && (int)((labels >> (4 * i)) & 15) == j) mask |= 1u << i;
          m[j] = (j < k) ? (int32_t)mstar[mask] : 0;
          if (j < k) {
            feasible &= m[j] <= M;
            sum_m += m[j];
          }
        }
        if (!feasible || sum_m > M) continue;
        const uint64_t rank_pi = a.L.k_base[k] + (uint64_t)p * per_pi;
        if (a.masked) {
          thr_masked_alloc<NT>(a, tab, k, rank_pi, m, n_sched, pi_star, first, hash, st_sched);
          continue;
        }
        const int R = M - (sum_m - k);  // M - sum(m*_j - 1)
        const uint32_t cnt = tab.C(R, k);
        n_sched += cnt;
        pi_star = min(pi_star, sum_m);
        const uint64_t r_first = rank_pi + lexrank_sizes(tab, M, k, m);
        first = r_first < first ? r_first : first;
        if (a.want_hash) {
          // walk the schedulable vectors s = m* + (s' - 1) in lexicographic order
          int32_t s[NT];
          int32_t sum = sum_m;
#pragma unroll
          for (int j = 0; j < NT; ++j) s[j] = m[j];
          uint64_t r = r_first;
          for (uint32_t c = 0; c < cnt; ++c) {
            hash += splitmix64(r);
            if (c + 1 == cnt) break;
            if (sum < M) {  // grow the last part: the next rank
#pragma unroll
              for (int j = 0; j < NT; ++j)
                if (j == k - 1) s[j] += 1;
              sum += 1;
              r += 1;
            } else {  // bump the rightmost part with slack above its threshold
              int pick = -1, tail = 0;
#pragma unroll
              for (int j = NT - 1; j >= 0; --j) {
                if (j < k) {
                  if (pick < 0 && j < k - 1 && tail > 0) pick = j;
                  tail += s[j] - m[j];  // slack of the parts after j
                }
              }
              sum = 0;
#pragma unroll
              for (int j = 0; j < NT; ++j) {
                if (j < k) {
                  if (j == pick) s[j] += 1;
                  else if (j > pick) s[j] = m[j];
                  sum += s[j];
                }
              }
              r = rank_pi + lexrank_sizes(tab, M, k, s);
            }
          }
          st_sched += cnt;
        }
      }
    }
    // warp reduction of the per-set outputs
    const uint64_t tot = warp_sum_u64(n_sched);
    const int32_t pis = warp_min_i32(pi_star);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t v = __shfl_xor_sync(GP_FULL, first, o);
      first = v < first ? v : first;
    }
    const uint64_t h = warp_sum_u64(hash);
    if (lane == 0) {
      ps[0] = (int64_t)tot;
      ps[1] = tot ? pis : 0;
      ps[2] = tot ? (int64_t)first : -1;
      ps[3] = a.want_hash ? (int64_t)h : 0;
      if (a.counts) {
        const int32_t grp = a.group[set];
        if (grp >= 0 && grp < a.n_groups) {
          unsigned long long *c = reinterpret_cast<unsigned long long *>(
              a.counts + (((int64_t)a.setting * a.n_groups + grp) * a.n_slots + a.slot0) * 3);
          const bool valid = a.valid[set] != 0;
          if (tot > 0 && valid) atomicAdd(c + 0, 1ull);
          atomicAdd(c + 1, 1ull);
          if (!valid) atomicAdd(c + 2, 1ull);
        }
      }
    }
    __syncwarp();
  }
  // contract violations still count (as invalid) -- handled by the host-side
  // finalize below via per_set[0] == -1
  if (a.stats) {
    const uint64_t t1 = warp_sum_u64(st_tests), t2 = warp_sum_u64(st_events);
    const uint64_t t3 = warp_sum_u64(st_sched);
    if (lane == 0) {
      atomicAdd(a.stats + 0, (unsigned long long)st_sets);
      atomicAdd(a.stats + 1, (unsigned long long)t1);
      atomicAdd(a.stats + 2, (unsigned long long)t2);
      atomicAdd(a.stats + 3, (unsigned long long)t3);
    }
  }
}

// counts for sets that violated the contract (per_set[0] == -1): invalid
__global__ void k_thr_violations(const ThrArgs a) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.n_sets;
       g += (int64_t)gridDim.x * blockDim.x) {
    if (a.per_set[g * 4] != -1 || !a.counts) continue;
    const int32_t grp = a.group[g];
    if (grp < 0 || grp >= a.n_groups) continue;
    unsigned long long *c = reinterpret_cast<unsigned long long *>(
        a.counts + (((int64_t)a.setting * a.n_groups + grp) * a.n_slots + a.slot0) * 3);
    atomicAdd(c + 1, 1ull);
    atomicAdd(c + 2, 1ull);
  }
}

template <int NT>
static gp_status launch_thr(ThrArgs &a, size_t smem, cudaStream_t st) {
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_threshold<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_threshold<NT>, kThrWarps * 32, smem);
  if (occ < 1) occ = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = ((int64_t)a.n_sets + kThrWarps - 1) / kThrWarps;
  int64_t grid = (int64_t)sms * occ;
  if (want < grid) grid = want > 0 ? want : 1;
  k_threshold<NT><<<(unsigned)grid, kThrWarps * 32, smem, st>>>(a);
  return gp_cuda_check("gp_sched_ratio(THRESHOLD)");
}

}  // namespace gp

gp_status gp_threshold_launch(const gp_tasksets *ts, int32_t slot0, int32_t n_slots,
                              int32_t setting, int64_t *counts, const gp_exhaustive_opts *ex,
                              cudaStream_t st) {
  using namespace gp;
  const int n = ts->n_tasks, M = ts->M;
  if (n < 1 || n > kEnumMaxTasks || M < 1 || M > kEnumMaxM)
    return gp_fail(GP_EINVAL, "THRESHOLD: need n_tasks <= 12 and M <= 256 (n=%d M=%d)", n, M);
  if (!ex || !ex->per_set) return gp_fail(GP_EINVAL, "THRESHOLD: opts and per_set are required");
  if (ex->verdict_bits) return gp_fail(GP_EINVAL, "THRESHOLD: verdict bits are not produced");
  ThrArgs a;
  gp_status s = rank_layout(M, n, &a.L, true);
  if (s != GP_OK) return s;
  if (ex->rank_lo != 0 || (ex->rank_hi != UINT64_MAX && ex->rank_hi < a.L.total))
    return gp_fail(GP_EINVAL, "THRESHOLD: only the full rank window");
  a.T = ts->T; a.D = ts->D; a.B = ts->B; a.cn = ts->cn; a.cc = ts->cc; a.fn = ts->fn;
  a.fc = ts->fc; a.group = ts->group; a.type = ts->type; a.valid = ts->valid;
  a.n_sets = ts->n_sets; a.n = n; a.M = M; a.n_groups = ts->n_groups;
  a.per_set = ex->per_set; a.counts = counts; a.slot0 = slot0; a.n_slots = n_slots;
  a.setting = setting; a.want_hash = (ex->flags & GP_EX_NO_HASH) ? 0 : 1; a.stats = ex->stats;
  a.masked = ex->size_mask != nullptr;
  a.next = ex->work_counter;  // optional here: dynamic set scheduling when given
  {
    uint32_t adm[8];
    s = load_size_mask(ex->size_mask, M, adm, "THRESHOLD");
    if (s != GP_OK) return s;
    for (int w = 0; w < 8; ++w) a.adm[w] = adm[w];
  }
  if (ts->n_sets == 0) return gp_cuda_check("THRESHOLD");
  if (a.next) cudaMemsetAsync(a.next, 0, 8, st);
  const size_t per_warp = thr_warp_words(n, M);
  const size_t smem = (((enum_table_words(M, n) + 3) & ~(size_t)3) + per_warp * kThrWarps) * 4;
  if (smem > 227 * 1024) return gp_fail(GP_EINVAL, "THRESHOLD: shared memory need %zu B", smem);
  gp_status r;
  switch (n) {
    case 1: case 2: case 3: case 4: r = launch_thr<4>(a, smem, st); break;
    case 5: case 6: r = launch_thr<6>(a, smem, st); break;
    case 7: case 8: r = launch_thr<8>(a, smem, st); break;
    default: r = launch_thr<12>(a, smem, st); break;
  }
  if (r != GP_OK) return r;
  int64_t g1 = (ts->n_sets + 255) / 256;
  k_thr_violations<<<(unsigned)(g1 > 4096 ? 4096 : g1), 256, 0, st>>>(a);
  return gp_cuda_check("gp_sched_ratio(THRESHOLD) violations");
}
