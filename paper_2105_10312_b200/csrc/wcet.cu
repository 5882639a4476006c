// wcet.cu -- A3 standalone: interference-aware WCET per task per candidate.
// Case equation P:479-486 (C_i = C^c if tau_i has conflict, else C^n), conflict
// definition, W form C.1.3 (ceil(B/m) waves, P:257-258 / P:762-763).
// The fused exhaustive evaluator computes the same values in registers.
#include "gp_common.cuh"

namespace gp {

struct WcetArgs {
  const int32_t *B, *cn, *cc, *fn, *fc;
  const uint8_t *type;
  int32_t n_sets, n;
  const int32_t *set_of_cand;
  const int8_t *bot;
  const int16_t *bs;
  int64_t n_cand;
  int32_t *wcet;
  uint8_t *conflict;
};

// Thread per (candidate, task).
__global__ void __launch_bounds__(256) k_wcet(const WcetArgs a) {
  const int n = a.n;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < a.n_cand * n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x / n;
    const int i = (int)(x % n);
    const int32_t set = a.set_of_cand[c];
    const int b = a.bot[c * n + i];
    const int m = (b >= 0 && b < n) ? a.bs[c * n + b] : 0;
    if (set < 0 || set >= a.n_sets || b < 0 || b >= n || m <= 0) {
      a.wcet[x] = -1;
      a.conflict[x] = 255;
      continue;
    }
    const int64_t base = (int64_t)set * n;
    const uint8_t ti = a.type[base + i];
    bool conf = false;  // another task of the same type in the same block
    for (int j = 0; j < n; ++j)
      conf |= (j != i) && (a.bot[c * n + j] == b) && (a.type[base + j] == ti);
    const int32_t Bi = a.B[base + i];
    a.wcet[x] = conf ? wcet_sat(Bi, a.cc[base + i], a.fc[base + i], m)
                     : wcet_sat(Bi, a.cn[base + i], a.fn[base + i], m);
    a.conflict[x] = conf ? 1 : 0;
  }
}

// Per-SM form of the worked example (C.1.4): thread j = SM j, then a block max.
__global__ void k_wcet_per_sm(int32_t B, int32_t m, const int32_t *cost, int32_t f,
                              int32_t *per_sm, int32_t *task_wcet) {
  __shared__ int32_t best;
  if (threadIdx.x == 0) best = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    int64_t blocks_on = B / m + (j < B % m ? 1 : 0);  // round robin from SM 0 (A-5)
    int64_t w = blocks_on * cost[j] + f;
    int32_t ws = w > INT32_MAX ? INT32_MAX : (int32_t)w;
    per_sm[j] = ws;
    atomicMax(&best, ws);
  }
  __syncthreads();
  if (threadIdx.x == 0) task_wcet[0] = best;
}

}  // namespace gp

extern "C" gp_status gp_wcet(const gp_tasksets *ts, const int32_t *set_of_cand,
                             const int8_t *block_of_task, const int16_t *block_size, int64_t n_cand,
                             int32_t *wcet, uint8_t *conflict, void *stream) {
  using namespace gp;
  if (!ts || ts->n_tasks < 1 || ts->n_tasks > kMaxTasks || ts->n_sets < 0)
    return gp_fail(GP_EINVAL, "gp_wcet: bad task sets");
  if (n_cand < 0) return gp_fail(GP_EINVAL, "gp_wcet: n_cand < 0");
  if (n_cand == 0) return gp_cuda_check("gp_wcet");
  if (!set_of_cand || !block_of_task || !block_size || !wcet || !conflict || !ts->B || !ts->cn ||
      !ts->cc || !ts->fn || !ts->fc || !ts->type)
    return gp_fail(GP_EINVAL, "gp_wcet: null pointer");
  WcetArgs a{ts->B, ts->cn, ts->cc, ts->fn, ts->fc, ts->type, ts->n_sets, ts->n_tasks,
             set_of_cand, block_of_task, block_size, n_cand, wcet, conflict};
  int64_t work = n_cand * ts->n_tasks;
  int64_t grid = (work + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  k_wcet<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(a);
  return gp_cuda_check("gp_wcet");
}

extern "C" gp_status gp_wcet_per_sm(int32_t B, int32_t m, const int32_t *cost_per_sm, int32_t f,
                                    int32_t *per_sm, int32_t *task_wcet, void *stream) {
  using namespace gp;
  if (m < 1 || m > 1024 || B < 0) return gp_fail(GP_EINVAL, "gp_wcet_per_sm: need 1<=m<=1024, B>=0");
  if (!cost_per_sm || !per_sm || !task_wcet) return gp_fail(GP_EINVAL, "gp_wcet_per_sm: null");
  k_wcet_per_sm<<<1, 256, 0, (cudaStream_t)stream>>>(B, m, cost_per_sm, f, per_sm, task_wcet);
  return gp_cuda_check("gp_wcet_per_sm");
}
