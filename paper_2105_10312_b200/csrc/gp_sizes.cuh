// gp_sizes.cuh -- the partition sizes Algorithm 2 may try, and how it tries them
// (SURVEY §8(f) f4).
//
// Paper default (Def. 3): every m in max(|P1|,|P2|) ..
// |P1|+|P2|-1, in increasing order, first schedulable wins.  f4 variants:
//   * admissible sizes only (MIG-style slices): m in the caller's
//     mask, which lies in 1..M;
//   * binary search "between max{|P1|,|P2|} and |P1|+|P2|", as a
//     lower-bound search over the ascending candidate list: lo = 0, hi = |L|;
//     mid = (lo+hi)/2; schedulable(L[mid]) ? hi = mid : lo = mid + 1.
// Schedulability is monotone in m (W is non-increasing in m and the demand
// test is monotone in the C_i), so both searches return the same size.
#pragma once
#include "gp_common.cuh"

namespace gp {

constexpr int kMaxMaskWords = 32;  // M <= 1024

// gp_alloc_opts as the kernels receive it (by value: no device allocation)
struct AllocVariantOpts {
  uint32_t flags;
  int32_t masked;
  uint32_t mask[kMaxMaskWords];  // bits above M cleared by the launcher
};

// Shared-memory tables of an admissible-size mask (built once per CTA).
struct SizeTables {
  int16_t adm[1024];  // admissible sizes, ascending
  int16_t ge[1026];   // ge[m] = index in adm of the first admissible size >= m (m = 0..M+1)
};

struct SizeSpace {
  const SizeTables *tab;  // null: every size (the paper's default)
  int32_t M, A;           // A = number of admissible sizes
  bool binary;
  GP_DEV int32_t idx_ge(int32_t m) const { return tab ? tab->ge[min(max(m, 0), M + 1)] : m; }
  GP_DEV int32_t val(int32_t x) const { return tab ? tab->adm[x] : x; }
  // smallest admissible size >= m (0 if none); identity without a mask
  GP_DEV int32_t round_up(int32_t m) const {
    if (!tab) return m;
    const int32_t x = idx_ge(m);
    return x < A ? val(x) : 0;
  }
  GP_DEV int32_t largest() const { return tab ? tab->adm[A - 1] : M; }
};

// Build the tables from the mask (bit m-1 of word (m-1)/32 = size m admissible)
// with all threads of the CTA; ends with __syncthreads().
GP_DEV void build_size_tables(SizeTables &t, const uint32_t (&mask)[kMaxMaskWords], int32_t M) {
  for (int32_t m = threadIdx.x; m <= M + 1; m += blockDim.x) {
    // number of admissible sizes in 1..m-1
    int32_t below = 0;
    const int32_t bits = m - 1 < M ? max(m - 1, 0) : M;
    for (int w = 0; w < (bits >> 5); ++w) below += __popc(mask[w]);
    if (bits & 31) below += __popc(mask[bits >> 5] & ((1u << (bits & 31)) - 1u));
    t.ge[m] = (int16_t)below;
    if (m >= 1 && m <= M && ((mask[(m - 1) >> 5] >> ((m - 1) & 31)) & 1u)) t.adm[below] = (int16_t)m;
  }
  __syncthreads();
}

// Algorithm 2's size search: the smallest candidate m in [lo, hi] with test(m),
// 0 if none.  kGen = false compiles to the paper's plain linear scan.
template <bool kGen, class F>
GP_DEV int32_t search_sizes(const SizeSpace &z, int32_t lo, int32_t hi, F &&test) {
  if constexpr (!kGen) {
    for (int32_t m = lo; m <= hi; ++m)
      if (test(m)) return m;
    return 0;
  } else {
    if (hi < lo) return 0;
    int32_t l = z.idx_ge(lo), r = z.idx_ge(hi + 1);  // candidates [l, r)
    if (!z.binary) {
      for (int32_t x = l; x < r; ++x)
        if (test(z.val(x))) return z.val(x);
      return 0;
    }
    const int32_t R = r;
    while (l < r) {
      const int32_t mid = (l + r) >> 1;
      if (test(z.val(mid))) r = mid;
      else l = mid + 1;
    }
    return l < R ? z.val(l) : 0;
  }
}

// Algorithm 2's answer WITHOUT its linear scan (paper default, no f4 option): the
// first schedulable m in [lo, hi] (0 if none), found by one test at hi and then a
// binary search below it.  Exact: EDF-PDC(S, m) is monotone in m (W_i is
// non-increasing in m, C.1.3, and the demand test is monotone in the C_i; the
// conflict flags depend on S only), so the linear scan's first success is the
// binary search's -- the oracle's f4 binary merge proves the same equivalence and
// tests/test_oracle_f4.py pins it.  A failing scan, the common case (96-98 % of
// INA's merges at C4 load), costs one test instead of hi - lo + 1.  `counted` gets
// the tests the PAPER's linear scan performs -- the n_tests contract (C.1.9 step 7):
// first success - lo + 1, or hi - lo + 1 if none; the tests actually run are what the
// caller's test() counts (the roofline's executed work).
template <class F>
GP_DEV int32_t first_fit_size(int32_t lo, int32_t hi, F &&test, int64_t &counted) {
  if (hi < lo) return 0;
  // one call site of test() (it is inlined: a second site would double the code the
  // divergent groups of a warp must keep in the instruction cache)
  int32_t a = lo, b = hi, m = hi;
  bool probed = false, any = false;
  for (;;) {
    const bool ok = test(m);
    if (!probed) {  // the probe at hi: nothing below is schedulable if it fails
      probed = true;
      any = ok;
      if (!ok) break;
    } else if (ok) {
      b = m;  // test(b) holds; the answer lies in [a, b]
    } else {
      a = m + 1;
    }
    if (a >= b) break;
    m = (a + b) >> 1;
  }
  const int32_t got = any ? a : 0;  // the last success was at b == a (U*H recorded there)
  counted += got ? got - lo + 1 : hi - lo + 1;
  return got;
}

// The size search of one Algorithm 2 call: the paper's default through
// first_fit_size (counting the linear scan's tests), the f4 variants through
// search_sizes (counting the tests they run: binary search is the variant).
template <bool kGen, class F>
GP_DEV int32_t alg2_search(const SizeSpace &z, int32_t lo, int32_t hi, F &&test, int64_t &counted) {
  if constexpr (!kGen) {
    return first_fit_size(lo, hi, test, counted);
  } else {
    int64_t ran = 0;
    auto counted_test = [&](int32_t m) -> bool {
      ++ran;
      return test(m);
    };
    const int32_t r = search_sizes<true>(z, lo, hi, counted_test);
    counted += ran;
    return r;
  }
}

}  // namespace gp
