// gp_common.cuh -- device helpers shared by the sm_100a kernels of libgpart.
// Product code: independent of oracle/ (no shared code, header or table).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpart.h"

#define GP_DEV __device__ __forceinline__
#define GP_FULL 0xFFFFFFFFu

namespace gp {

constexpr int kMaxTasks = 32;
constexpr int kMaxMenu = 16;
constexpr int kMaxPrm = 16;

// ---- integer helpers -------------------------------------------------------
GP_DEV int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }
GP_DEV int32_t ceil_div32(int32_t a, int32_t b) { return (a + b - 1) / b; }

GP_DEV int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Binary (Stein) gcd of 32-bit values: shifts and subtractions only.
GP_DEV uint32_t gcd32(uint32_t u, uint32_t v) {
  if (u == 0) return v;
  if (v == 0) return u;
  const int sh = __ffs(u | v) - 1;
  u >>= __ffs(u) - 1;
  do {
    v >>= __ffs(v) - 1;
    const uint32_t lo = min(u, v), hi = max(u, v);
    u = lo;
    v = hi - lo;
  } while (v);
  return u << sh;
}

// lcm with saturation: returns -1 when it would exceed `cap` (q * b > cap
// <=> q > floor(cap / b) for positive integers).  32-bit path when every
// operand fits (every hyperperiod the contract admits: cap < 2^31).
GP_DEV int64_t lcm_capped(int64_t a, int64_t b, int64_t cap) {
  if (a < 0 || b < 0) return -1;
  if (((a | b | cap) >> 31) == 0) {
    const uint32_t g = gcd32((uint32_t)a, (uint32_t)b);
    if (g == 0) return 0;
    const uint64_t r = (uint64_t)((uint32_t)a / g) * (uint64_t)b;
    return r > (uint64_t)cap ? -1 : (int64_t)r;
  }
  int64_t g = gcd64(a, b);
  int64_t q = a / g;
  if (q > cap / b) return -1;
  return q * b;
}

// ceil(B/m) for 0 <= B <= INT32_MAX, 1 <= m <= 1024 without an integer division
// when B is small (< 2^22: every generated set, b_max <= 4096): a float
// reciprocal estimate is within 1 of the quotient and one correction each way
// makes it exact.  Larger B take a 64-bit division (B + m - 1 may exceed int32).
GP_DEV int32_t ceil_div_pos(int32_t B, int32_t m) {
  if (B < (1 << 22)) {
    const int32_t num = B + m - 1;
    int32_t q = (int32_t)((float)num * __frcp_rn((float)m));
    q += (q + 1) * m <= num;
    q -= q * m > num;
    return q;
  }
  return (int32_t)(((int64_t)B + m - 1) / m);
}

// W(m) = ceil(B/m)*c + f in 64-bit, saturated to INT32_MAX (C.1.3).
GP_DEV int32_t wcet_sat(int32_t B, int32_t c, int32_t f, int32_t m) {
  int64_t w = (int64_t)ceil_div_pos(B, m) * (int64_t)c + (int64_t)f;
  return w > INT32_MAX ? INT32_MAX : (int32_t)w;
}

// ---- warp reductions ---------------------------------------------------------
GP_DEV int32_t warp_sum_i32(int32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(GP_FULL, v, o);
  return v;
}
GP_DEV int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(GP_FULL, v, o);
  return v;
}
GP_DEV uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(GP_FULL, v, o);
  return v;
}
GP_DEV int32_t warp_min_i32(int32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(GP_FULL, v, o));
  return v;
}
GP_DEV int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t w = __shfl_xor_sync(GP_FULL, v, o);
    v = w < v ? w : v;
  }
  return v;
}
GP_DEV uint32_t warp_or_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(GP_FULL, v, o);
  return v;
}

// ---- SplitMix64 output for state x (order-independent verdict hash) ---------
GP_DEV uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace gp

// ---- host-side error plumbing (abi.cu) ---------------------------------------
gp_status gp_fail(gp_status st, const char *fmt, ...);
gp_status gp_cuda_check(const char *what);
gp_status gp_ok(void);  // clears gp_last_error() (host-only calls: no CUDA API touched)

namespace gp {
// Host: gp_exhaustive_opts.size_mask -> adm words (NULL -> every size).
inline gp_status load_size_mask(const uint32_t *mask, int M, uint32_t (&adm)[8], const char *who) {
  for (int w = 0; w < 8; ++w) adm[w] = ~0u;
  if (!mask) return GP_OK;
  bool any = false;
  for (int w = 0; w < 8; ++w) {
    const int lo = 32 * w + 1;  // sizes lo .. lo + 31
    uint32_t keep = 0u;
    if (lo <= M) {
      const uint32_t m = mask[w];
      keep = M - lo + 1 >= 32 ? m : m & ((1u << (M - lo + 1)) - 1u);
    }
    adm[w] = keep;
    any |= keep != 0u;
  }
  if (!any) return gp_fail(GP_EINVAL, "%s: size_mask admits no size in 1..M", who);
  return GP_OK;
}
}  // namespace gp
