// allocate_big.cu -- A5 for task sets of 33..256 tasks (the paper's own
// scenarios have 50 and 200 tasks): one CTA of 256 threads per set.
//
// Same algorithm and conventions as allocate.cu (Algorithm 1 P:507-533,
// Lemmas 1-3, Algorithm 2 with the linear m scan, Algorithm 3, Defs 4/5,
// ACT/INA forbidden lists, 1G; C.1.9, A-17..A-26), with partitions and
// forbidden rows as 256-bit sets in shared memory.  Thread t owns task t and
// partition slot t; a live slot's index is the lowest task id of its partition.
// Merge attempts of one selection round run one partner per thread (exact:
// the scans are independent, only failures feed later rounds) with a
// thread-serial EDF test for merged partitions of <= 16 tasks; larger merges
// and 1G use a CTA-cooperative EDF test (thread = task).
// f4 variants as in allocate.cu (kGen instantiation).
#include "gp_common.cuh"
#include "gp_edf.cuh"
#include "gp_sizes.cuh"

namespace gp {

constexpr int kBigN = 256;
constexpr int kBW = kBigN / 32;  // words per task bitset
constexpr int kSerialMax = 16;

struct BigArgs {
  const int32_t *T, *D, *B, *cn, *cc, *fn, *fc;
  const uint8_t *type;
  int32_t n_sets, n, M, variant;
  uint8_t *ok;
  int16_t *bot;
  int16_t *bs;
  int32_t *pi, *k;
  int64_t *n_tests;
  int64_t *eff;
  unsigned long long *stats;
  int32_t stats_ext;
  unsigned long long *next_set;  // work counter (zeroed per launch)
  AllocVariantOpts vo;  // f4
};

struct BigSmem {
  int32_t T[kBigN], D[kBigN], B[kBigN], cn[kBigN], cc[kBigN], fn[kBigN], fc[kBigN], q[kBigN];
  uint32_t mem[kBW], comp[kBW];   // task masks of each type
  uint32_t pm[kBigN][kBW];        // slot -> task set
  uint32_t pex[kBigN][kBW];       // slot -> slots whose merge failed (snapshots)
  uint32_t forb[kBigN][kBW];      // task -> forbidden tasks (ACT)
  uint32_t fslots[kBigN][kBW];    // slot -> slots excluded by ACT task pairs
  int32_t psz[kBigN], puh[kBigN], ord[kBigN], bord[kBigN], plist[kBigN], lab[kBigN], lsize[kBigN];
  uint32_t live[kBW];
  uint32_t scratch[kBW];          // broadcast of a merged task set
  int64_t red64[8];
  int32_t red32[8];
  int32_t bcast[4];
};

// ---- CTA reductions (256 threads) ---------------------------------------------
GP_DEV int64_t cta_sum64(BigSmem &s, int64_t v) {
  v = warp_sum_i64(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red64[threadIdx.x >> 5] = v;
  __syncthreads();
  int64_t t = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += s.red64[w];
  return t;
}
GP_DEV int32_t cta_min32(BigSmem &s, int32_t v) {
  v = warp_min_i32(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red32[threadIdx.x >> 5] = v;
  __syncthreads();
  int32_t t = INT32_MAX;
#pragma unroll
  for (int w = 0; w < 8; ++w) t = min(t, s.red32[w]);
  return t;
}
GP_DEV float cta_sumf(BigSmem &s, float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(GP_FULL, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red32[threadIdx.x >> 5] = __float_as_int(v);
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += __int_as_float(s.red32[w]);
  return t;
}

GP_DEV bool bs_has(const uint32_t *m, int i) { return (m[i >> 5] >> (i & 31)) & 1u; }
GP_DEV int bs_popc_and(const uint32_t *a, const uint32_t *b) {
  int c = 0;
#pragma unroll
  for (int w = 0; w < kBW; ++w) c += __popc(a[w] & b[w]);
  return c;
}

GP_DEV int32_t big_w(const BigSmem &s, int i, int32_t m, bool x) {
  return x ? wcet_sat(s.B[i], s.cc[i], s.fc[i], m) : wcet_sat(s.B[i], s.cn[i], s.fn[i], m);
}
GP_DEV bool big_conflict(const BigSmem &s, int i, const uint32_t *S) {
  const uint32_t *same = ((s.mem[i >> 5] >> (i & 31)) & 1u) ? s.mem : s.comp;
  return bs_popc_and(S, same) > 1;  // another task of my type in S
}

// CTA-cooperative EDF-PDC of the partition S (bitset in shared memory or a
// register copy broadcast through shared memory) at size m.
GP_DEV bool cta_pdc(BigSmem &s, const uint32_t *S, int32_t m, int32_t H, int n,
                    uint64_t &st_tasks, uint64_t &st_events) {
  const int i = threadIdx.x;
  const bool in = i < n && bs_has(S, i);
  const int32_t C = in ? big_w(s, i, m, big_conflict(s, i, S)) : 0;
  if (threadIdx.x == 0) st_tasks += (uint64_t)bs_popc_and(S, S);
  if (__syncthreads_or(in && C > s.D[i])) return false;
  const int64_t UH = cta_sum64(s, in ? (int64_t)C * s.q[i] : 0);
  if (UH > H) return false;
  int32_t lcut = H;
  if (UH < H) {
    const float X = cta_sumf(s, in ? (float)(s.T[i] - s.D[i]) * (float)((int64_t)C * s.q[i]) : 0.f);
    const float L = X / (float)(H - UH) * 1.0001f + 2.0f;
    lcut = L >= (float)H ? H : (int32_t)L;
  }
  int32_t nx = in ? s.D[i] : INT32_MAX, dem = 0;
  for (;;) {
    const int32_t t = cta_min32(s, nx);
    if (t > lcut) return true;
    const bool hit = nx == t;
    if (threadIdx.x == 0) ++st_events;
    dem += (int32_t)cta_sum64(s, hit ? C : 0);
    nx += hit ? s.T[i] : 0;
    if (dem > t) return false;
  }
}

// Algorithm 2 merge by ONE thread for a merged partition of <= kSerialMax tasks.
template <bool kGen>
GP_DEV int32_t big_serial_merge(const BigSmem &s, const SizeSpace &z, const uint32_t (&S)[kBW],
                                int32_t lo, int32_t hi, int32_t H, int32_t &uh_out, int64_t &counted,
                                uint64_t &st_tasks, uint32_t &st_events, uint32_t &st_exec) {
  int32_t T[kSerialMax], D[kSerialMax], Bv[kSerialMax], c[kSerialMax], f[kSerialMax],
      q[kSerialMax];
  int cnt = 0;
  int w = 0;
  uint32_t bits = S[0];
#pragma unroll
  for (int a = 0; a < kSerialMax; ++a) {
    while (bits == 0 && w < kBW - 1) bits = S[++w];
    const bool v = bits != 0;
    const int i = v ? (w << 5) + __ffs(bits) - 1 : 0;
    bits &= bits - 1u;
    const bool x = v && big_conflict(s, i, S);
    T[a] = v ? s.T[i] : INT32_MAX;
    D[a] = v ? s.D[i] : INT32_MAX;
    Bv[a] = v ? s.B[i] : 1;
    c[a] = v ? (x ? s.cc[i] : s.cn[i]) : 0;
    f[a] = v ? (x ? s.fc[i] : s.fn[i]) : 0;
    q[a] = v ? s.q[i] : 0;
    cnt += v;
  }
  auto test = [&](int32_t m) -> bool {
    ++st_exec;
    st_tasks += cnt;
    int32_t C[kSerialMax];
    bool bad = false;
#pragma unroll
    for (int a = 0; a < kSerialMax; ++a) {
      C[a] = c[a] ? wcet_sat(Bv[a], c[a], f[a], m) : 0;
      bad |= C[a] > D[a];
    }
    if (bad) return false;
    int32_t UH = 0;
#pragma unroll
    for (int a = 0; a < kSerialMax; ++a) UH += C[a] * q[a];
    if (UH > H) return false;
    if (cnt > 1) {
      const int32_t lcut = pdc_cutoff<kSerialMax>(C, D, T, q, H, UH);
      if (!pdc_walk<kSerialMax>(C, D, T, lcut, st_events)) return false;
    }
    uh_out = UH;
    return true;
  };
  return alg2_search<kGen>(z, lo, hi, test, counted);  // paper's count (gp_sizes.cuh)
}

template <bool kGen>
__global__ void __launch_bounds__(256) k_allocate_big(const BigArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BigSmem &s = *reinterpret_cast<BigSmem *>(smem_raw);
  const int t = threadIdx.x, n = a.n, M = a.M;
  SizeSpace z{nullptr, M, 0, false};
  bool incr = false;
  if constexpr (kGen) {
    z.binary = (a.vo.flags & GP_AL_BINARY_MERGE) != 0;
    incr = (a.vo.flags & GP_AL_INCREASING) != 0;
    if (a.vo.masked) {
      SizeTables *tb = reinterpret_cast<SizeTables *>(smem_raw + ((sizeof(BigSmem) + 15) & ~(size_t)15));
      build_size_tables(*tb, a.vo.mask, M);
      z.tab = tb;
      z.A = tb->ge[M + 1];
    }
  }
  const bool act = a.variant == GP_SMS_ACT || a.variant == GP_BF_ACT;
  const bool sms = a.variant == GP_SMS_ACT || a.variant == GP_SMS_INA;
  uint64_t st_tests = 0, st_tasks = 0, st_events = 0, st_sets = 0;  // thread 0's copies
  uint64_t st_exec = 0, st_rounds = 0, st_scan = 0, st_partners = 0;  // uniform
  uint64_t my_tasks = 0;
  uint32_t my_events = 0, my_exec = 0;
  // persistent CTAs grabbing their next set from a counter (work per set varies widely)
  for (;;) {
    if (threadIdx.x == 0) s.bcast[3] = (int32_t)atomicAdd(a.next_set, 1ull);
    __syncthreads();
    const int64_t set = s.bcast[3];
    __syncthreads();
    if (set >= a.n_sets) break;
    // ---- load, contract, hyperperiod
    const bool in = t < n;
    const int64_t o = set * n + t;
    if (in) {
      s.T[t] = a.T[o]; s.D[t] = a.D[o]; s.B[t] = a.B[o]; s.cn[t] = a.cn[o]; s.cc[t] = a.cc[o];
      s.fn[t] = a.fn[o]; s.fc[t] = a.fc[o];
    }
    if (t < kBW) s.mem[t] = s.comp[t] = 0;
    __syncthreads();
    if (in) {
      if (a.type[o] == 1) atomicOr(&s.mem[t >> 5], 1u << (t & 31));
      else atomicOr(&s.comp[t >> 5], 1u << (t & 31));
    }
    const bool fields_ok = !in || (s.T[t] >= 1 && s.D[t] >= 1 && s.D[t] <= s.T[t] && s.B[t] >= 1 &&
                                   s.cn[t] >= 1 && s.cc[t] >= s.cn[t] && s.fn[t] >= 0 &&
                                   s.fc[t] >= s.fn[t]);
    const bool all_ok = !__syncthreads_or(!fields_ok);
    int64_t H = 1;
    const int64_t cap = ((int64_t)1 << 31) / (n + 1) - 1;
    if (all_ok) {  // lcm reduction by thread 0 (once per set)
      if (t == 0) {
        int64_t h = 1;
        for (int i = 0; i < n && h > 0; ++i) h = lcm_capped(h, s.T[i], cap);
        s.red64[0] = h;
      }
      __syncthreads();
      H = s.red64[0];
      __syncthreads();
    }
    const bool contract = all_ok && H > 0;
    const int32_t H32 = contract ? (int32_t)H : 1;
    if (in) s.q[t] = contract ? H32 / s.T[t] : 0;
    s.pm[t][0] = 0;
    for (int w = 0; w < kBW; ++w) {
      s.pm[t][w] = 0;
      s.pex[t][w] = 0;
      s.forb[t][w] = 0;
      s.fslots[t][w] = 0;
    }
    s.psz[t] = 0;
    s.puh[t] = 0;
    if (t < kBW) s.live[t] = 0;
    __syncthreads();

    int64_t tests = 0;  // uniform
    bool ok = false;
    int stage = 0;
    if (!contract) {
      tests = -1;
    } else if (a.variant == GP_1G) {
      // 1G: all tasks, all M SMs
      if (in) atomicOr(&s.pm[0][t >> 5], 1u << (t & 31));
      __syncthreads();
      tests = 1;
      ++st_exec;
      const int32_t m1 = z.largest();  // M, or the largest admissible size (f4)
      ok = cta_pdc(s, s.pm[0], m1, H32, n, st_tasks, st_events);
      if (t == 0) {
        s.psz[0] = m1;
        s.live[0] = 1u;
      }
      stage = 1;
    } else {
      // Lemma 1
      const int64_t w1 = in ? ((int64_t)s.B[t] * s.cn[t] + s.fn[t]) * (int64_t)s.q[t] : 0;
      const bool lemma1 = cta_sum64(s, w1) <= (int64_t)M * H32;
      // Lemma 2, closed form (B-3)
      int32_t mi = 0;
      if (in && s.D[t] - s.fn[t] >= s.cn[t]) {
        const int32_t K = (s.D[t] - s.fn[t]) / s.cn[t];
        const int64_t m0 = ((int64_t)s.B[t] + K - 1) / K;  // 64-bit: B may reach INT32_MAX
        mi = m0 <= M ? max((int32_t)m0, 1) : 0;
        if (kGen && mi) mi = z.round_up(mi);  // f4: smallest admissible size >= m0
      }
      const bool lemma2 = !__syncthreads_or(in && mi == 0);
      if (lemma1 && lemma2) {
        stage = 1;
        if (in) {
          s.pm[t][t >> 5] = 1u << (t & 31);
          s.psz[t] = mi;
          s.puh[t] = big_w(s, t, mi, false) * s.q[t];
          atomicOr(&s.live[t >> 5], 1u << (t & 31));
        }
        int64_t Pi = cta_sum64(s, in ? mi : 0);
        if (Pi <= M) {
          ok = true;  // Lemma 3 (A-24)
        } else {
          if (act) {  // §5.3: every couple of tasks
            const int np = n * (n - 1) / 2;
            int64_t my_tests = 0;
            for (int idx = t; idx < np; idx += blockDim.x) {
              int i = 0, rem = idx;
              while (rem >= n - 1 - i) {
                rem -= n - 1 - i;
                ++i;
              }
              const int j = i + 1 + rem;
              uint32_t S[kBW];
#pragma unroll
              for (int w = 0; w < kBW; ++w) S[w] = 0;
              S[i >> 5] |= 1u << (i & 31);
              S[j >> 5] |= 1u << (j & 31);
              int32_t uh;
              const int32_t mi_ = s.psz[i], mj_ = s.psz[j];
              const int32_t got = big_serial_merge<kGen>(s, z, S, max(mi_, mj_), mi_ + mj_ - 1,
                                                         H32, uh, my_tests, my_tasks, my_events,
                                                         my_exec);
              if (!got) {
                atomicOr(&s.forb[i][j >> 5], 1u << (j & 31));
                atomicOr(&s.forb[j][i >> 5], 1u << (i & 31));
              }
            }
            tests += cta_sum64(s, my_tests);
          }
          bool dirty = true;
          int rank = 0, len = 0;
          for (;;) {
            if (dirty) {
              // par_list order (U*H desc, slot asc; f4: U*H asc), best-fit partner
              // order (U*H desc, A-21) and the ACT exclusions
              const bool live = bs_has(s.live, t);
              rank = 0;
              int brank = 0;
              if (live)
                for (int u = 0; u < n; ++u) {
                  const bool lv = bs_has(s.live, u);
                  brank += lv && (s.puh[u] > s.puh[t] || (s.puh[u] == s.puh[t] && u < t));
                  if (kGen && incr)
                    rank += lv && (s.puh[u] < s.puh[t] || (s.puh[u] == s.puh[t] && u < t));
                }
              if (!(kGen && incr)) rank = brank;
              if (live) {
                s.ord[rank] = t;
                s.bord[brank] = t;
              }
              len = 0;
#pragma unroll
              for (int w = 0; w < kBW; ++w) len += __popc(s.live[w]);
              if (act && live) {
                uint32_t F[kBW];
#pragma unroll
                for (int w = 0; w < kBW; ++w) F[w] = 0;
                for (int i = 0; i < n; ++i)
                  if (bs_has(s.pm[t], i))
#pragma unroll
                    for (int w = 0; w < kBW; ++w) F[w] |= s.forb[i][w];
                for (int u = 0; u < n; ++u) {
                  const bool hit = bs_has(s.live, u) && bs_popc_and(s.pm[u], F) > 0;
                  if (hit) s.fslots[t][u >> 5] |= 1u << (u & 31);
                  else s.fslots[t][u >> 5] &= ~(1u << (u & 31));
                }
              }
              __syncthreads();
              dirty = false;
            }
            if (Pi <= M) {
              ok = true;
              break;
            }
            // Algorithm 3: the first slot in order with an eligible partner
            bool nonempty = false;
            if (bs_has(s.live, t)) {
#pragma unroll
              for (int w = 0; w < kBW; ++w) {
                uint32_t e = s.live[w] & ~s.pex[t][w] & ~(act ? s.fslots[t][w] : 0u);
                if (w == (t >> 5)) e &= ~(1u << (t & 31));
                nonempty |= e != 0;
              }
            }
            const int cand = cta_min32(s, nonempty ? rank : INT32_MAX);
            if (cand == INT32_MAX) break;  // no selectable partition: fail
            const int P = s.ord[cand];
            // partners in best-fit order -> plist
            bool el = false;
            if (t < len) {
              const int Q = s.bord[t];
              el = Q != P && !bs_has(s.pex[P], Q) && !(act && bs_has(s.fslots[P], Q));
            }
            // block prefix of el over t (8 warps)
            const uint32_t bal = __ballot_sync(GP_FULL, el);
            __syncthreads();
            if ((t & 31) == 0) s.red32[t >> 5] = __popc(bal);
            __syncthreads();
            int before = 0, E = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
              before += w < (t >> 5) ? s.red32[w] : 0;
              E += s.red32[w];
            }
            if (el) s.plist[before + __popc(bal & ((1u << (t & 31)) - 1u))] = s.bord[t];
            ++st_rounds;       // one Algorithm 3 selection over len partitions,
            st_scan += len;
            st_partners += E;  // E partner searches (Algorithm 2)
            __syncthreads();
            // merged sizes
            const int Qe = t < E ? s.plist[t] : 0;
            uint32_t Se[kBW];
            int cnt = 0;
#pragma unroll
            for (int w = 0; w < kBW; ++w) {
              Se[w] = s.pm[P][w] | (t < E ? s.pm[Qe][w] : 0u);
              cnt += __popc(Se[w]);
            }
            const int maxcnt = cta_min32(s, t < E ? -cnt : 0) * -1;
            int best = -1;
            int32_t best_m = 0, best_uh = 0;
            uint32_t failQ[kBW];
#pragma unroll
            for (int w = 0; w < kBW; ++w) failQ[w] = 0;
            const int32_t szP = s.psz[P];
            if (maxcnt <= kSerialMax) {
              int64_t my_tests = 0;
              int32_t got = 0, uh = 0;
              if (t < E) {
                const int32_t szQ = s.psz[Qe];
                got = big_serial_merge<kGen>(s, z, Se, max(szP, szQ), szP + szQ - 1, H32, uh,
                                             my_tests, my_tasks, my_events, my_exec);
              }
              // first success (BF) / best (SMS), tests counted in sequential order
              const int first_ok = cta_min32(s, (t < E && got > 0) ? t : INT32_MAX);
              const int cut = sms ? E : (first_ok == INT32_MAX ? E : first_ok + 1);
              tests += cta_sum64(s, t < cut ? my_tests : 0);
              const bool failed = t < cut && t < E && got == 0;
              if (failed) {  // add_to_forbidden_moves(P, Q)
                atomicOr(&s.pex[P][Qe >> 5], 1u << (Qe & 31));
                atomicOr(&s.pex[Qe][P >> 5], 1u << (P & 31));
              }
              if (sms) {
                // smallest size, then U*H, then partner id (Def. 4, A-20)
                const int64_t key = (t < E && got > 0)
                                        ? (((int64_t)got << 40) | ((int64_t)uh << 8) | Qe)
                                        : INT64_MAX;
                int64_t kmin = key;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                  const int64_t k2 = __shfl_xor_sync(GP_FULL, kmin, off);
                  kmin = k2 < kmin ? k2 : kmin;
                }
                __syncthreads();
                if ((t & 31) == 0) s.red64[t >> 5] = kmin;
                __syncthreads();
                kmin = INT64_MAX;
#pragma unroll
                for (int w = 0; w < 8; ++w) kmin = s.red64[w] < kmin ? s.red64[w] : kmin;
                if (kmin != INT64_MAX) {
                  best = (int)(kmin & 0xFF);
                  best_m = (int32_t)(kmin >> 40);
                  best_uh = (int32_t)((kmin >> 8) & 0xFFFFFFFF);
                }
              } else if (first_ok != INT32_MAX) {
                __syncthreads();
                if (t == first_ok) {
                  s.bcast[0] = Qe;
                  s.bcast[1] = got;
                  s.bcast[2] = uh;
                }
                __syncthreads();
                best = s.bcast[0];
                best_m = s.bcast[1];
                best_uh = s.bcast[2];
              }
            } else {
              // large merges: partners in order, CTA-cooperative tests
              for (int e = 0; e < E; ++e) {
                const int Q = s.plist[e];
                const int32_t szQ = s.psz[Q];
                __syncthreads();
                if (t < kBW) s.scratch[t] = s.pm[P][t] | s.pm[Q][t];
                __syncthreads();
                uint32_t S2[kBW];
#pragma unroll
                for (int w = 0; w < kBW; ++w) S2[w] = s.scratch[w];
                auto ctest = [&](int32_t m) -> bool {
                  ++st_exec;
                  return cta_pdc(s, S2, m, H32, n, st_tasks, st_events);
                };
                const int32_t got =
                    alg2_search<kGen>(z, max(szP, szQ), szP + szQ - 1, ctest, tests);
                if (!got) {
                  if (t == 0) {
                    s.pex[P][Q >> 5] |= 1u << (Q & 31);
                    s.pex[Q][P >> 5] |= 1u << (P & 31);
                  }
                  continue;
                }
                const int i = t;
                const bool inS = i < n && bs_has(S2, i);
                const int32_t uh = (int32_t)cta_sum64(
                    s, inS ? (int64_t)big_w(s, i, got, big_conflict(s, i, S2)) * s.q[i] : 0);
                const bool better = best < 0 || got < best_m ||
                                    (got == best_m && (uh < best_uh || (uh == best_uh && Q < best)));
                if (!sms || better) {
                  best = Q;
                  best_m = got;
                  best_uh = uh;
                }
                if (!sms) break;
              }
            }
            __syncthreads();
            if (best >= 0) {  // commit: P u Q replaces P and Q
              const int Q = best;
              const int keep = min(P, Q), drop = max(P, Q);
              Pi -= szP + s.psz[Q] - best_m;
              __syncthreads();
              if (t < kBW) {
                const uint32_t u = s.pm[P][t] | s.pm[Q][t];
                s.pm[keep][t] = u;
                s.pm[drop][t] = 0;
                s.pex[keep][t] = 0;
                s.pex[drop][t] = 0;
              }
              if (t == 0) {
                s.psz[keep] = best_m;
                s.puh[keep] = best_uh;
                s.psz[drop] = 0;
                s.puh[drop] = 0;
                s.live[drop >> 5] &= ~(1u << (drop & 31));
              }
              __syncthreads();
              s.pex[t][keep >> 5] &= ~(1u << (keep & 31));
              s.pex[t][drop >> 5] &= ~(1u << (drop & 31));
              dirty = true;
            }
            __syncthreads();
          }
        }
      }
    }
    // ---- outputs: canonical labels (slots numbered by index among live slots)
    __syncthreads();
    const bool live = stage && bs_has(s.live, t);
    int label = 0;
    if (live) {
      for (int w = 0; w < (t >> 5); ++w) label += __popc(s.live[w]);
      label += __popc(s.live[t >> 5] & ((1u << (t & 31)) - 1u));
      s.lsize[label] = s.psz[t];
      for (int i = 0; i < n; ++i)
        if (bs_has(s.pm[t], i)) s.lab[i] = label;
    }
    __syncthreads();
    int kk = 0;
#pragma unroll
    for (int w = 0; w < kBW; ++w) kk += stage ? __popc(s.live[w]) : 0;
    const int64_t Pi_out = cta_sum64(s, live ? s.psz[t] : 0);
    if (in) {
      a.bot[o] = (int16_t)(stage ? s.lab[t] : -1);
      a.bs[o] = (int16_t)((stage && t < kk) ? s.lsize[t] : 0);
    }
    if (a.eff) {
      const int64_t w = (in && contract) ? (int64_t)s.B[t] * s.q[t] : 0;
      const int64_t lo = cta_sum64(s, w * (in ? s.cn[t] : 0));
      const int64_t up = cta_sum64(s, w * (in ? s.cc[t] : 0));
      int64_t mine = 0;
      if (stage && in) {
        const int L = s.lab[t];
        // the partition of task t: the live slot with label L
        int slot = -1;
        for (int u = 0, c = 0; u < n && slot < 0; ++u)
          if (bs_has(s.live, u)) {
            if (c == L) slot = u;
            ++c;
          }
        mine = w * (big_conflict(s, t, s.pm[slot]) ? s.cc[t] : s.cn[t]);
      }
      const int64_t ach = cta_sum64(s, mine);
      if (t == 0) {
        a.eff[set * 4 + 0] = lo;
        a.eff[set * 4 + 1] = up;
        a.eff[set * 4 + 2] = ach;
        a.eff[set * 4 + 3] = contract ? H32 : 0;
      }
    }
    if (t == 0) {
      a.ok[set] = ok ? 1 : 0;
      a.pi[set] = stage ? (int32_t)Pi_out : 0;
      a.k[set] = kk;
      a.n_tests[set] = tests;
      st_sets += 1;
      st_tests += tests > 0 ? (uint64_t)tests : 0;
    }
    __syncthreads();
  }
  if (a.stats) {
    const uint64_t pt = (uint64_t)cta_sum64(*reinterpret_cast<BigSmem *>(smem_raw), (int64_t)my_tasks);
    const uint64_t pe = (uint64_t)cta_sum64(*reinterpret_cast<BigSmem *>(smem_raw), (int64_t)my_events);
    const uint64_t px = (uint64_t)cta_sum64(*reinterpret_cast<BigSmem *>(smem_raw), (int64_t)my_exec);
    if (t == 0) {
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

gp_status gp_allocate_big_launch(const gp_tasksets *ts, int32_t v, const gp::AllocVariantOpts &vo,
                                 uint8_t *ok, int16_t *bot, int16_t *bs, int32_t *pi, int32_t *k,
                                 int64_t *n_tests, int64_t *eff, unsigned long long *stats,
                                 bool stats_ext, cudaStream_t st) {
  using namespace gp;
  BigArgs a{ts->T, ts->D, ts->B, ts->cn, ts->cc, ts->fn, ts->fc, ts->type, ts->n_sets,
            ts->n_tasks, ts->M, v, ok, bot, bs, pi, k, n_tests, eff, stats,
            stats_ext ? 1 : 0, nullptr, vo};
  const bool gen = vo.flags != 0 || vo.masked;
  size_t smem = sizeof(BigSmem);
  if (gen && vo.masked) smem = ((smem + 15) & ~(size_t)15) + sizeof(SizeTables);
  auto kern = gen ? k_allocate_big<true> : k_allocate_big<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)148 * occ;
  if (grid > ts->n_sets) grid = ts->n_sets;
  if (cudaMallocAsync(reinterpret_cast<void **>(&a.next_set), 8, st) != cudaSuccess)
    return gp_cuda_check("gp_allocate (n > 32): work counter");
  cudaMemsetAsync(a.next_set, 0, 8, st);
  kern<<<(unsigned)grid, 256, smem, st>>>(a);
  cudaFreeAsync(a.next_set, st);
  return gp_cuda_check("gp_allocate (n > 32)");
}
