// gp_edf.cuh -- A4: the per-partition EDF processor-demand test, device side.
//
// Policy: preemptive EDF inside a partition, tasks run one at a time on all
// its SMs (reading A-6).  A block S at size s is
// schedulable iff dbf_S(t) = sum_i [t >= D_i] (floor((t-D_i)/T_i)+1) C_i <= t
// at every absolute deadline t <= H (C.1.7).
//
// The kernels evaluate EXACTLY that verdict with three exact shortcuts (the
// oracle keeps the plain walk over every deadline up to the hyperperiod):
//   1. C_i > D_i fails at t = D_i already; a singleton passes iff C <= D.
//   2. U > 1 (in integers sum C_i*(H/T_i) > H) fails: dbf at the last
//      deadline <= H equals U*H.
//   3. For U < 1, dbf(t) <= t*U + sum_i (T_i-D_i) C_i/T_i, so no deadline
//      t >= L_a = sum_i (T_i-D_i) C_i/T_i / (1-U) can fail (George, Rivierre,
//      Spuri 1996).  The walk therefore stops at min(H, Lcut) with Lcut an
//      over-estimate of L_a (float with a relative margin, so never below it);
//      checking a few extra deadlines cannot change the verdict.
// H is the lcm of ALL periods of the set (a multiple of the block's own
// hyperperiod): for U <= 1, dbf(H_S p + t') = U H_S p + dbf(t') so the
// verdict over [0, H] equals the verdict over [0, H_S].
// Arithmetic is int32: C <= D < T (after shortcut 1), C * (H/T) < H, and the
// input contract H * (n+1) < 2^31 bounds every sum.
#pragma once
#include "gp_common.cuh"

namespace gp {

// Walk the deadlines of SZ tasks in increasing order up to `lcut`, adding
// C_a at each deadline of task a and checking the running demand against t.
// `events` counts the distinct deadlines examined.
template <int SZ>
GP_DEV bool pdc_walk(const int32_t (&C)[SZ], const int32_t (&D)[SZ], const int32_t (&T)[SZ],
                     int32_t lcut, uint32_t &events) {
  int32_t nx[SZ];
#pragma unroll
  for (int a = 0; a < SZ; ++a) nx[a] = D[a];
  int32_t dem = 0;
  for (;;) {
    int32_t t = nx[0];
#pragma unroll
    for (int a = 1; a < SZ; ++a) t = min(t, nx[a]);
    if (t > lcut) return true;
#pragma unroll
    for (int a = 0; a < SZ; ++a) {
      const bool hit = nx[a] == t;
      dem += hit ? C[a] : 0;
      nx[a] += hit ? T[a] : 0;
    }
    ++events;
    if (dem > t) return false;
  }
}

// Density test, an exact SUFFICIENT condition: for t >= D_i, floor((t - D_i)/T_i) + 1 <= t/D_i
// since D_i <= T_i, so dbf(t) <= t * sum_i C_i/D_i <= t whenever the density is <= 1.  Float
// with a 1e-5 margin (<= 8 terms of relative error < 2^-21 each), so true means the block
// passes the definition; false decides nothing (the walk follows).  Padded slots: C = 0.
#ifndef GP_DENSITY
#define GP_DENSITY 1
#endif
template <int SZ>
GP_DEV bool pdc_density_ok(const int32_t (&C)[SZ], const int32_t (&D)[SZ]) {
  static_assert(SZ <= 8, "the 1e-5 margin covers at most 8 terms");
  float d = 0.f;
#pragma unroll
  for (int a = 0; a < SZ; ++a) d += __fdividef((float)C[a], (float)D[a]);
  return GP_DENSITY && d <= 0.99999f;
}

// Upper bound on the walk: H when U == 1, else min(H, over-estimate of L_a).
template <int SZ>
GP_DEV int32_t pdc_cutoff(const int32_t (&C)[SZ], const int32_t (&D)[SZ], const int32_t (&T)[SZ],
                          const int32_t (&q)[SZ], int32_t H, int32_t UH) {
  if (UH >= H) return H;
  float X = 0.f;
#pragma unroll
  for (int a = 0; a < SZ; ++a) X += (float)(T[a] - D[a]) * (float)(C[a] * q[a]);
  const float L = __fdividef(X, (float)(H - UH)) * 1.0001f + 2.0f;
  return L >= (float)H ? H : (int32_t)L;
}

}  // namespace gp
