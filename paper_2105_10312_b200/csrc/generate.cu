// generate.cu -- A1: counter-based synthetic task sets (gp_generate).
// Paper: §7.1 task-set generation.  Definitions C.1.10, readings
// A-9..A-15 and A-31.
//
// Layout of the work: one GROUP of G lanes per task set, G = next power of two
// >= n_tasks (G = 8 for 6 tasks: 4 sets per warp; G = 32 for 32 tasks).  Lane
// j of the group owns task j: it draws its own Philox block (counter =
// (g, attempt, j)), the n-1 spacing points are sorted with a register bitonic
// network across the group (shuffles, no shared memory), each lane derives
// its utilisation as the gap to its left neighbour, computes its fields, and
// a group ballot implements the whole-vector discard.  Writes are coalesced
// because a set's tasks are contiguous ([set][task] layout).
#include <cstdarg>
#include <cstdio>

#include "gp_common.cuh"

namespace gp {

struct GenArgs {
  int32_t M, n, n_bins, n_prm, sets_per_group, Q, n_periods, b_max;
  int32_t beta_c, beta_m, beta_den, kc, km, k_den, max_attempts, G, curve_gran;
  int32_t rep_count, n_sets;
  uint32_t bden_mlo, bden_mhi;  // division by beta_den as a multiply: M = floor(2^64/d) + 1
  uint64_t rep_begin, seed;
  int32_t menu[kMaxMenu];
  uint64_t prm_q[kMaxPrm];
  int32_t *T, *D, *B, *cn, *cc, *fn, *fc, *group;
  uint8_t *type, *valid;
};

// Philox4x32-10 (Salmon et al., SC'11).
GP_DEV void philox4x32_10(uint32_t &x0, uint32_t &x1, uint32_t &x2, uint32_t &x3, uint32_t k0,
                          uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0 = 0xD2511F53u * x0, hi0 = __umulhi(0xD2511F53u, x0);
    uint32_t lo1 = 0xCD9E8D57u * x2, hi1 = __umulhi(0xCD9E8D57u, x2);
    uint32_t y0 = hi1 ^ x1 ^ k0, y2 = hi0 ^ x3 ^ k1;
    x0 = y0;
    x1 = lo1;
    x2 = y2;
    x3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// floor(n / d) for n < 2^32 and 2 <= d < 2^32 as floor(n * M / 2^64), M = floor(2^64/d) + 1
// (or 2^64/d when d is a power of two): n*M/2^64 lies in [n/d, n/d + n/2^64] and the
// fractional part of n/d is at most 1 - 1/d < 1 - 2^-32, so the floor is exact.
// M = mhi * 2^32 + mlo; d = 1 is passed as mhi = mlo = 0 and returns n.
GP_DEV uint32_t div_by_magic(uint32_t n, uint32_t mlo, uint32_t mhi) {
  if ((mlo | mhi) == 0u) return n;
  const uint64_t t = ((uint64_t)n * mlo) >> 32;
  return (uint32_t)(((uint64_t)n * mhi + t) >> 32);
}

// One task of §7.1 from its draws; the discard test of A-9.
struct TaskDraw {
  uint32_t T, D, cn, fn;
  int32_t B;
  bool feasible;
};

GP_DEV TaskDraw task_fields(const GenArgs &a, uint64_t u, int32_t pidx, int32_t Bv, uint8_t typ) {
  TaskDraw d;
  // period bump while the baseline execution time is "not reasonable" (A-10);
  // in curve mode B is derived from a, and the rule reduces to a < Q
  int64_t T = (int64_t)a.menu[pidx] * a.Q;
  int64_t ab = (int64_t)((u * (uint64_t)T) >> 20);
  const int64_t need = (a.curve_gran > 0 || Bv <= a.Q) ? a.Q : Bv;
  while (ab < need && pidx < a.n_periods - 1) {
    ++pidx;
    T = (int64_t)a.menu[pidx] * a.Q;
    ab = (int64_t)((u * (uint64_t)T) >> 20);
  }
  // host validation bounds a <= M * Tmax < 2^31, so 32-bit arithmetic is exact below
  const uint32_t a32 = (uint32_t)ab, T32 = (uint32_t)T;
  d.T = T32;
  d.D = 3u * (T32 / 4u);                                                          // P:944 (4 | T)
  if (a.curve_gran > 0) {  // C = k(a/m + b) as W form: B = ceil(a/g) granules, cn = g
    const uint32_t g = (uint32_t)a.curve_gran;
    d.B = (int32_t)max((a32 + g - 1u) / g, 1u);
    d.cn = g;
  } else {
    d.B = Bv;
    d.cn = max((a32 + (uint32_t)Bv - 1u) / (uint32_t)Bv, 1u);
  }
  // fn = ceil(a * beta_num / beta_den) without 64-bit division: a = qd*den + r
  const uint32_t bnum = typ ? (uint32_t)a.beta_m : (uint32_t)a.beta_c, bden = (uint32_t)a.beta_den;
  const uint32_t qd = div_by_magic(a32, a.bden_mlo, a.bden_mhi), rd = a32 - qd * bden;
  d.fn = qd * bnum + div_by_magic(rd * bnum + bden - 1u, a.bden_mlo, a.bden_mhi);
  const uint32_t waves = (uint32_t)ceil_div_pos(d.B, a.M);
  d.feasible = (uint64_t)waves * d.cn + d.fn <= (uint64_t)d.D;                   // A-9
  return d;
}

template <int G>
__global__ void __launch_bounds__(256) k_generate(const GenArgs a) {
  const int lane = threadIdx.x & 31;
  const int j = lane & (G - 1);  // task slot inside the group
  const int64_t l = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;  // local set
  const bool live = l < a.n_sets;
  const int n = a.n;
  const unsigned gbase = (unsigned)(lane & ~(G - 1));
  const unsigned gmask = (G == 32) ? GP_FULL : (((1u << G) - 1u) << gbase);

  int32_t grp = 0, prm_idx = 0, bin = 0;
  uint64_t g = 0;
  if (live) {
    grp = (int32_t)(l / a.rep_count);
    uint64_t rep = a.rep_begin + (uint64_t)(l % a.rep_count);
    g = (uint64_t)grp * (uint64_t)a.sets_per_group + rep;  // global set index
    prm_idx = grp / a.n_bins;
    bin = grp % a.n_bins;
  }
  // U_q = (bin+1) * M * 2^20 / n_bins: total utilisation in Q20 (A-31)
  const int64_t Uq = ((int64_t)(bin + 1) * a.M << 20) / a.n_bins;
  const uint64_t pq = a.prm_q[prm_idx];
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);

  int32_t oT = 0, oD = 0, oB = 0, ocn = 0, occ = 0, ofn = 0, ofc = 0;
  uint8_t otype = 0;
  bool done = !live, valid = false;
  for (int attempt = 0; attempt < a.max_attempts; ++attempt) {
    if (__ballot_sync(GP_FULL, !done) == 0) break;
    uint32_t x0 = (uint32_t)g, x1 = (uint32_t)(g >> 32), x2 = (uint32_t)attempt, x3 = (uint32_t)j;
    philox4x32_10(x0, x1, x2, x3, k0, k1);
    const uint8_t typ = ((uint64_t)x0 < pq) ? 1 : 0;
    const int32_t pidx = (int32_t)(((uint64_t)x1 * (uint64_t)a.n_periods) >> 32);    // A-11
    const int32_t Bv = 1 + (int32_t)(((uint64_t)x2 * (uint64_t)a.b_max) >> 32);     // A-13
    // spacing point; lanes >= n-1 carry the pad U_q so they sort last (U_q < 2^31)
    uint32_t pt = (j < n - 1) ? (uint32_t)(((uint64_t)x3 * (uint64_t)(Uq + 1)) >> 32) : (uint32_t)Uq;
    // bitonic sort ascending across the G lanes of the group
#pragma unroll
    for (int kk = 2; kk <= G; kk <<= 1) {
#pragma unroll
      for (int s = kk >> 1; s > 0; s >>= 1) {
        const uint32_t o = __shfl_xor_sync(GP_FULL, pt, s);
        const bool asc = (j & kk) == 0, lower = (j & s) == 0;
        pt = (lower == asc) ? min(o, pt) : max(o, pt);
      }
    }
    uint32_t left = __shfl_up_sync(GP_FULL, pt, 1, G);
    if (j == 0) left = 0;
    const uint64_t u = pt - left;  // UUniFast via sorted spacings (A-12)
    const TaskDraw d = task_fields(a, u, pidx, Bv, typ);
    const bool feasible = d.feasible;
    const unsigned bad = __ballot_sync(GP_FULL, (j < n) && !feasible) & gmask;
    if (!done) {
      oT = (int32_t)d.T; oD = (int32_t)d.D; oB = d.B;
      ocn = (int32_t)d.cn; ofn = (int32_t)d.fn;
      otype = typ;
      if (bad == 0) {
        done = true;
        valid = true;
      }
    }
  }
  // conflict costs of the committed draw (A-14): c^c = ceil(k cn), f^c = ceil(k fn)
  {
    const int64_t kf = otype ? a.km : a.kc;
    occ = (int32_t)ceil_div64((int64_t)ocn * kf, a.k_den);
    ofc = (int32_t)ceil_div64((int64_t)ofn * kf, a.k_den);
  }
  if (live && j < n) {
    const int64_t o = l * n + j;
    a.T[o] = oT; a.D[o] = oD; a.B[o] = oB; a.cn[o] = ocn; a.cc[o] = occ;
    a.fn[o] = ofn; a.fc[o] = ofc; a.type[o] = otype;
    if (j == 0) {
      a.valid[l] = valid ? 1 : 0;
      a.group[l] = grp;
    }
  }
}

// n > 32: one CTA of 256 threads per set; thread j owns task j; the spacing
// points are sorted by a shared-memory bitonic network; the whole-vector
// discard is a CTA vote.
__global__ void __launch_bounds__(256) k_generate_big(const GenArgs a) {
  __shared__ uint32_t pts[256];
  const int j = threadIdx.x, n = a.n;
  for (int64_t l = blockIdx.x; l < a.n_sets; l += gridDim.x) {
    const int32_t grp = (int32_t)(l / a.rep_count);
    const uint64_t rep = a.rep_begin + (uint64_t)(l % a.rep_count);
    const uint64_t g = (uint64_t)grp * (uint64_t)a.sets_per_group + rep;
    const int32_t prm_idx = grp / a.n_bins, bin = grp % a.n_bins;
    const int64_t Uq = ((int64_t)(bin + 1) * a.M << 20) / a.n_bins;
    const uint64_t pq = a.prm_q[prm_idx];
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    TaskDraw keep{};
    uint8_t ktype = 0;
    bool valid = false;
    for (int attempt = 0; attempt < a.max_attempts; ++attempt) {
      uint32_t x0 = (uint32_t)g, x1 = (uint32_t)(g >> 32), x2 = (uint32_t)attempt, x3 = (uint32_t)j;
      philox4x32_10(x0, x1, x2, x3, k0, k1);
      const uint8_t typ = ((uint64_t)x0 < pq) ? 1 : 0;
      const int32_t pidx = (int32_t)(((uint64_t)x1 * (uint64_t)a.n_periods) >> 32);  // A-11
      const int32_t Bv = 1 + (int32_t)(((uint64_t)x2 * (uint64_t)a.b_max) >> 32);   // A-13
      pts[j] = (j < n - 1) ? (uint32_t)(((uint64_t)x3 * (uint64_t)(Uq + 1)) >> 32) : (uint32_t)Uq;
      __syncthreads();
      for (int kk = 2; kk <= 256; kk <<= 1) {  // bitonic sort, ascending
        for (int s = kk >> 1; s > 0; s >>= 1) {
          const int p = j ^ s;
          if (p > j) {
            const uint32_t x = pts[j], y = pts[p];
            const bool asc = (j & kk) == 0;
            if ((x > y) == asc) {
              pts[j] = y;
              pts[p] = x;
            }
          }
          __syncthreads();
        }
      }
      const uint64_t u = pts[j] - (j == 0 ? 0u : pts[j - 1]);  // sorted spacings (A-12)
      const TaskDraw d = task_fields(a, u, pidx, Bv, typ);
      const int bad = __syncthreads_or(j < n && !d.feasible);
      keep = d;
      ktype = typ;
      if (!bad) {
        valid = true;
        break;
      }
    }
    if (j < n) {
      const int64_t kf = ktype ? a.km : a.kc;
      const int64_t o = l * n + j;
      a.T[o] = (int32_t)keep.T; a.D[o] = (int32_t)keep.D; a.B[o] = keep.B;
      a.cn[o] = (int32_t)keep.cn; a.fn[o] = (int32_t)keep.fn; a.type[o] = ktype;
      a.cc[o] = (int32_t)ceil_div64((int64_t)keep.cn * kf, a.k_den);  // P:951, A-14
      a.fc[o] = (int32_t)ceil_div64((int64_t)keep.fn * kf, a.k_den);
      if (j == 0) {
        a.valid[l] = valid ? 1 : 0;
        a.group[l] = grp;
      }
    }
    __syncthreads();
  }
}

}  // namespace gp

static int64_t host_gcd(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

extern "C" gp_status gp_generate(const gp_gen_params *p, uint64_t seed, uint64_t rep_begin,
                                 int32_t rep_count, gp_tasksets *out, void *stream) {
  using namespace gp;
  if (!p || !out) return gp_fail(GP_EINVAL, "gp_generate: null params or output");
  if (p->n_tasks < 1 || p->n_tasks > 256)
    return gp_fail(GP_EINVAL, "gp_generate: n_tasks %d not in 1..256", p->n_tasks);
  if (p->curve_gran < 0) return gp_fail(GP_EINVAL, "gp_generate: curve_gran < 0");
  if (p->M < 1 || p->M > 1024) return gp_fail(GP_EINVAL, "gp_generate: M %d not in 1..1024", p->M);
  if (p->n_bins < 1 || p->n_prm < 1 || p->n_prm > kMaxPrm || p->sets_per_group < 1)
    return gp_fail(GP_EINVAL, "gp_generate: bad n_bins/n_prm/sets_per_group");
  if (!p->prm_q || !p->period_menu) return gp_fail(GP_EINVAL, "gp_generate: null prm_q/menu");
  for (int i = 0; i < p->n_prm; ++i)
    if (p->prm_q[i] > (1ull << 32)) return gp_fail(GP_EINVAL, "gp_generate: prm_q > 2^32");
  if (p->ticks_per_unit < 1 || p->n_periods < 1 || p->n_periods > kMaxMenu)
    return gp_fail(GP_EINVAL, "gp_generate: bad Q or n_periods");
  int64_t Tmax = 0, H = 1;
  for (int i = 0; i < p->n_periods; ++i) {
    int64_t t = (int64_t)p->period_menu[i] * p->ticks_per_unit;
    if (p->period_menu[i] <= 0 || (i > 0 && p->period_menu[i] <= p->period_menu[i - 1]))
      return gp_fail(GP_EINVAL, "gp_generate: period menu must be positive and ascending");
    if (t % 4 != 0) return gp_fail(GP_EINVAL, "gp_generate: Q*T must be divisible by 4 (D=3T/4)");
    if (t > INT32_MAX) return gp_fail(GP_EOVERFLOW, "gp_generate: period overflows int32");
    Tmax = t > Tmax ? t : Tmax;
    H = H / host_gcd(H, t) * t;
    if (H > INT32_MAX) return gp_fail(GP_EOVERFLOW, "gp_generate: menu hyperperiod overflows");
  }
  if (p->b_max < 1 || p->beta_den < 1 || p->beta_c_num < 0 || p->beta_m_num < 0 || p->k_den < 1 ||
      p->kc_num < p->k_den || p->km_num < p->k_den || p->max_attempts < 1)
    return gp_fail(GP_EINVAL, "gp_generate: bad b_max/beta/k (k >= 1 required)/max_attempts");
  if ((int64_t)p->beta_den * (p->beta_c_num > p->beta_m_num ? p->beta_c_num : p->beta_m_num) >=
      (1ll << 31))
    return gp_fail(GP_EOVERFLOW, "gp_generate: beta_den * beta_num must stay below 2^31");
  if (rep_count < 0 || rep_begin + (uint64_t)rep_count > (uint64_t)p->sets_per_group)
    return gp_fail(GP_EINVAL, "gp_generate: rep range beyond sets_per_group");
  const int64_t n_groups = (int64_t)p->n_prm * p->n_bins;
  if (out->n_sets != n_groups * rep_count || out->n_tasks != p->n_tasks)
    return gp_fail(GP_EINVAL, "gp_generate: out->n_sets must be n_prm*n_bins*rep_count (%lld)",
                   (long long)(n_groups * rep_count));
  // field ranges: a <= M*Tmax, cn <= a, fn <= beta*a, cc <= k*cn, fc <= k*fn
  const int64_t amax = (int64_t)p->M * Tmax;
  const int64_t bmax = p->beta_c_num > p->beta_m_num ? p->beta_c_num : p->beta_m_num;
  const int64_t kmax = p->kc_num > p->km_num ? p->kc_num : p->km_num;
  const int64_t fnmax = (amax * bmax + p->beta_den - 1) / p->beta_den;
  const int64_t cnmax = p->curve_gran > 0 ? p->curve_gran : amax;
  const int64_t ccmax = (cnmax * kmax + p->k_den - 1) / p->k_den;
  const int64_t fcmax = (fnmax * kmax + p->k_den - 1) / p->k_den;
  if (ccmax > INT32_MAX || fcmax > INT32_MAX || amax > INT32_MAX)
    return gp_fail(GP_EOVERFLOW, "gp_generate: M*Tmax*k exceeds int32 (fields would overflow)");
  if (H * (p->n_tasks + 1) >= (1ll << 31))
    return gp_fail(GP_EOVERFLOW, "gp_generate: menu hyperperiod * (n+1) >= 2^31");
  if (!out->T || !out->D || !out->B || !out->cn || !out->cc || !out->fn || !out->fc ||
      !out->type || !out->valid || !out->group)
    return gp_fail(GP_EINVAL, "gp_generate: null output pointer");
  out->M = p->M;
  out->n_groups = (int32_t)n_groups;
  if (out->n_sets == 0) return GP_OK;

  GenArgs a;
  a.M = p->M; a.n = p->n_tasks; a.n_bins = p->n_bins; a.n_prm = p->n_prm;
  a.sets_per_group = p->sets_per_group; a.Q = p->ticks_per_unit; a.n_periods = p->n_periods;
  a.b_max = p->b_max; a.beta_c = p->beta_c_num; a.beta_m = p->beta_m_num; a.beta_den = p->beta_den;
  {
    const uint64_t d = (uint64_t)p->beta_den;
    const uint64_t mg = d >= 2 ? (~0ull) / d + 1ull : 0ull;  // exact: see div_by_magic
    a.bden_mlo = (uint32_t)mg;
    a.bden_mhi = (uint32_t)(mg >> 32);
  }
  a.kc = p->kc_num; a.km = p->km_num; a.k_den = p->k_den; a.max_attempts = p->max_attempts;
  a.curve_gran = p->curve_gran;
  int G = 1;
  while (G < p->n_tasks && G < 32) G <<= 1;
  a.G = G;
  a.rep_count = rep_count; a.n_sets = out->n_sets; a.rep_begin = rep_begin; a.seed = seed;
  for (int i = 0; i < kMaxMenu; ++i) a.menu[i] = i < p->n_periods ? p->period_menu[i] : 0;
  for (int i = 0; i < kMaxPrm; ++i) a.prm_q[i] = i < p->n_prm ? p->prm_q[i] : 0;
  a.T = out->T; a.D = out->D; a.B = out->B; a.cn = out->cn; a.cc = out->cc; a.fn = out->fn;
  a.fc = out->fc; a.group = out->group; a.type = out->type; a.valid = out->valid;
  if (p->n_tasks > 32) {
    int64_t grid = out->n_sets < 148 * 8 ? out->n_sets : 148 * 8;
    k_generate_big<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
    return gp_cuda_check("gp_generate");
  }
  const int64_t threads = (int64_t)out->n_sets * G;
  const int block = 256;
  const int64_t grid = (threads + block - 1) / block;
  switch (G) {  // group width: the sort network is unrolled for it
    case 1: k_generate<1><<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(a); break;
    case 2: k_generate<2><<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(a); break;
    case 4: k_generate<4><<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(a); break;
    case 8: k_generate<8><<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(a); break;
    case 16: k_generate<16><<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(a); break;
    default: k_generate<32><<<(unsigned)grid, block, 0, (cudaStream_t)stream>>>(a); break;
  }
  return gp_cuda_check("gp_generate");
}
