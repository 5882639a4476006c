// gp_enum.cuh -- A2 candidate space (C.1.6): rank layout (host) and the
// unranking building blocks (device).  P:494-504 (§5 intro) states the space
// (SM partitioning x task-to-partition allocation) the heuristics avoid
// enumerating; on small GPUs this build enumerates it exactly.
//
// Candidate = (k, pi, s).  pi: restricted growth string (RGS) with exactly k
// labels; s in Z>=1^k, sum(s) <= M.  Rank order: k, then pi lexicographic,
// then s lexicographic.  s is handled through its prefix sums c_j = s_0+..+s_j,
// a strictly increasing k-subset of {1..M}; lexicographic order of s equals
// lexicographic order of c, so the s-index is the lex rank of a k-subset.
#pragma once
#include "gp_common.cuh"

namespace gp {

constexpr int kEnumMaxTasks = 12;  // exhaustive / enumerate limit (2^12 subsets)
constexpr int kEnumMaxM = 256;

struct RankLayout {
  int32_t M, n, kmax;
  uint64_t total;
  uint64_t k_base[kMaxTasks + 2];  // first rank with k blocks
  uint64_t n_pi[kMaxTasks + 2];    // S(n,k): number of RGS with k labels
  uint64_t per_pi[kMaxTasks + 2];  // C(M,k): size vectors per RGS
  uint32_t n_runs[kMaxTasks + 2];  // C(M-1,k-1): runs (prefixes) per RGS (bit-sliced evaluator)
};

// Host: exact layout with 128-bit arithmetic; GP_EOVERFLOW if N_c >= 2^63.
// need_u32: additionally require every C(a,b), a <= M, b <= min(n,M), < 2^32
// (the device binomial table is uint32).
static inline gp_status rank_layout(int32_t M, int32_t n, RankLayout *L, bool need_u32) {
  typedef unsigned __int128 u128;
  const u128 cap = (u128)1 << 100;
  u128 S[kMaxTasks + 2][kMaxTasks + 2] = {};
  S[0][0] = 1;
  for (int a = 1; a <= n; ++a)
    for (int b = 1; b <= a; ++b) {
      u128 v = (u128)b * S[a - 1][b] + S[a - 1][b - 1];
      S[a][b] = v > cap ? cap : v;
    }
  L->M = M;
  L->n = n;
  L->kmax = n < M ? n : M;
  u128 total = 0;
  for (int k = 1; k <= L->kmax; ++k) {
    u128 c = 1;  // C(M,k)
    for (int i = 1; i <= k; ++i) {
      c = c * (u128)(M - k + i) / (u128)i;
      if (c > cap) c = cap;
    }
    u128 cnt = S[n][k] * c;
    if (S[n][k] >= ((u128)1 << 64) || c >= ((u128)1 << 64) || cnt >= ((u128)1 << 63) ||
        total + cnt >= ((u128)1 << 63))
      return gp_fail(GP_EOVERFLOW, "candidate count N_c(M=%d,n=%d) >= 2^63", M, n);
    L->k_base[k] = (uint64_t)total;
    L->n_pi[k] = (uint64_t)S[n][k];
    L->per_pi[k] = (uint64_t)c;
    total += cnt;
  }
  L->total = (uint64_t)total;
  if (need_u32) {
    for (int a = 0; a <= M; ++a) {
      u128 c = 1;
      for (int b = 0; b <= L->kmax && b <= a; ++b) {
        if (b > 0) c = c * (u128)(a - b + 1) / (u128)b;
        if (c >= ((u128)1 << 32))
          return gp_fail(GP_EINVAL, "C(%d,%d) >= 2^32: exhaustive/enumerate limit", a, b);
      }
    }
  }
  return GP_OK;
}

// Device tables in shared memory:
//   binom[a*(n+1) + b] = C(a,b), a in 0..M, b in 0..n          (uint32)
//   rgs[((k*(n+1)) + i)*(n+2) + j] = completions of an RGS whose positions
//     0..i-1 are fixed and use j labels, ending with exactly k labels (uint32)
struct EnumTables {
  const uint32_t *binom;
  const uint32_t *rgs;
  int32_t n, M;
  GP_DEV uint32_t C(int a, int b) const {
    return (a < 0 || b < 0 || b > a) ? 0u : binom[a * (n + 1) + b];
  }
  GP_DEV uint32_t R(int k, int i, int j) const {
    return j > n + 1 ? 0u : rgs[(k * (n + 1) + i) * (n + 2) + j];
  }
};

__host__ __device__ inline size_t enum_table_words(int M, int n) {
  return (size_t)(M + 1) * (n + 1) + (size_t)(n + 1) * (n + 1) * (n + 2);
}

// Cooperative build by the whole CTA; ends with __syncthreads().
GP_DEV EnumTables build_enum_tables(uint32_t *smem, int M, int n) {
  uint32_t *binom = smem;
  uint32_t *rgs = smem + (size_t)(M + 1) * (n + 1);
  const int nb = (M + 1) * (n + 1);
  for (int e = threadIdx.x; e < nb; e += blockDim.x) {
    int a = e / (n + 1), b = e % (n + 1);
    uint64_t c = 0;
    if (b <= a) {
      c = 1;
      for (int i = 1; i <= b; ++i) c = c * (uint64_t)(a - b + i) / (uint64_t)i;
    }
    binom[e] = (uint32_t)c;
  }
  // one thread per k computes its (n+1) x (n+2) completion table
  for (int k = threadIdx.x; k <= n; k += blockDim.x) {
    uint32_t *Rk = rgs + (size_t)k * (n + 1) * (n + 2);
    for (int j = 0; j <= n + 1; ++j) Rk[n * (n + 2) + j] = (j == k) ? 1u : 0u;
    for (int i = n - 1; i >= 0; --i)
      for (int j = 0; j <= n + 1; ++j) {
        uint32_t stay = (j <= k) ? (uint32_t)j * Rk[(i + 1) * (n + 2) + j] : 0u;
        uint32_t grow = (j + 1 <= n + 1 && j + 1 <= k) ? Rk[(i + 1) * (n + 2) + j + 1] : 0u;
        Rk[i * (n + 2) + j] = stay + grow;
      }
  }
  __syncthreads();
  EnumTables t;
  t.binom = binom;
  t.rgs = rgs;
  t.n = n;
  t.M = M;
  return t;
}

// RGS index p (lexicographic among RGS with exactly k labels) -> labels.
// Returns the labels packed 4 bits per task (n <= 12 -> 48 bits).
GP_DEV uint64_t unrank_rgs(const EnumTables &t, int k, uint32_t p) {
  const int n = t.n;
  uint64_t packed = 0;
  int used = 0;
  for (int i = 0; i < n; ++i) {
    int lab = 0;
    for (; lab <= used; ++lab) {
      int used2 = (lab == used) ? used + 1 : used;
      uint32_t c = t.R(k, i + 1, used2);
      if (p < c) {
        used = used2;
        break;
      }
      p -= c;
    }
    packed |= (uint64_t)lab << (4 * i);
  }
  return packed;
}

// s-index rho (lexicographic among s >= 1, sum <= M, k parts) -> s[0..k-1].
template <int NT>
GP_DEV void unrank_sizes(const EnumTables &t, int k, uint32_t rho, int32_t (&s)[NT]) {
  int prev = 0;  // c_{j-1}
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < k) {
      int v = prev + 1;
      for (;;) {
        uint32_t cnt = t.binom[(t.M - v) * (t.n + 1) + (k - 1 - j)];  // valid ranks keep a >= b >= 0
        if (rho < cnt) break;
        rho -= cnt;
        ++v;
      }
      s[j] = v - prev;
      prev = v;
    } else {
      s[j] = 0;
    }
  }
}

// Lexicographic successor of s (sum <= M).  Returns false after the last one.
template <int NT>
GP_DEV bool next_sizes(int M, int k, int32_t (&s)[NT], int32_t &sum) {
  if (sum < M) {  // grow the last part
#pragma unroll
    for (int j = 0; j < NT; ++j)
      if (j == k - 1) s[j] += 1;
    sum += 1;
    return true;
  }
  // sum == M: bump the rightmost part j whose tail (parts after j) has slack,
  // reset the tail to ones.
  int tail = 0, pick = -1;
#pragma unroll
  for (int j = NT - 1; j >= 0; --j) {
    if (j < k) {
      if (pick < 0 && j < k - 1 && tail > (k - 1 - j)) pick = j;
      tail += s[j];
    }
  }
  if (pick < 0) return false;
  int newsum = 0;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < k) {
      if (j == pick) s[j] += 1;
      else if (j > pick) s[j] = 1;
      newsum += s[j];
    }
  }
  sum = newsum;
  return true;
}

}  // namespace gp
