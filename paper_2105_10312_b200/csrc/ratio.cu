// ratio.cu -- A6: segmented reduction to schedulability-rate counts
// (gp_sched_ratio).  §7.2: "the classical schedulability rate,
// so that we count the number of schedulable tasksets"; C.1.11.
// Integer atomics are order-independent, so the counts are deterministic and
// identical under any sharding (sum over ranks = one all-reduce).
#include "gp_common.cuh"

gp_status gp_exhaustive_launch(const gp_tasksets *ts, int32_t slot0, int32_t n_slots,
                               int32_t setting, int64_t *counts, const gp_exhaustive_opts *ex,
                               cudaStream_t st);
gp_status gp_threshold_launch(const gp_tasksets *ts, int32_t slot0, int32_t n_slots,
                              int32_t setting, int64_t *counts, const gp_exhaustive_opts *ex,
                              cudaStream_t st);

namespace gp {

struct RatioArgs {
  const uint8_t *verdicts, *valid;
  const int32_t *group;
  int32_t n_sets, n_rows, n_groups, slot0, n_slots, setting;
  int64_t *counts;
};

// CTA-private histogram in shared memory, then one global atomic per bin.
__global__ void __launch_bounds__(256) k_ratio(const RatioArgs a) {
  extern __shared__ unsigned long long hist[];
  const int bins = a.n_groups * a.n_rows * 3;
  for (int e = threadIdx.x; e < bins; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  // whole warps iterate together; each warp adds once per distinct (group, row) bin
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)a.n_sets * a.n_rows;
  const int64_t total32 = (total + 31) & ~(int64_t)31;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total32;
       x += (int64_t)gridDim.x * blockDim.x) {
    int bin = -1;
    bool valid = false, ok = false;
    if (x < total) {
      const int row = (int)(x / a.n_sets);
      const int64_t set = x - (int64_t)row * a.n_sets;
      const int32_t g = a.group[set];
      if (g >= 0 && g < a.n_groups) {
        bin = g * a.n_rows + row;
        valid = a.valid[set] != 0;
        ok = a.verdicts[x] != 0;
      }
    }
    const uint32_t peers = __match_any_sync(GP_FULL, bin);
    const uint32_t b_ok = __ballot_sync(GP_FULL, bin >= 0 && ok && valid);
    const uint32_t b_inv = __ballot_sync(GP_FULL, bin >= 0 && !valid);
    if (bin >= 0 && lane == __ffs(peers) - 1) {
      unsigned long long *h = hist + (int64_t)bin * 3;
      if (b_ok & peers) atomicAdd(h + 0, (unsigned long long)__popc(b_ok & peers));
      atomicAdd(h + 1, (unsigned long long)__popc(peers));
      if (b_inv & peers) atomicAdd(h + 2, (unsigned long long)__popc(b_inv & peers));
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < bins; e += blockDim.x) {
    if (!hist[e]) continue;
    const int c = e % 3, gr = e / 3, row = gr % a.n_rows, g = gr / a.n_rows;
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(
        a.counts + (((int64_t)a.setting * a.n_groups + g) * a.n_slots + a.slot0 + row) * 3 + c);
    atomicAdd(dst, hist[e]);
  }
}

// GP_FROM_PER_SET: the EXHAUSTIVE finalize's counting from per-set outputs that were
// produced elsewhere (e.g. merged over candidate-rank shards, §8(e)): exists = n_sched > 0;
// n_sched < 0 (input contract violated) or valid = 0 counts as invalid.
struct PerSetArgs {
  const int64_t *per_set;
  const uint8_t *valid;
  const int32_t *group;
  int32_t n_sets, n_groups, slot0, n_slots, setting;
  int64_t *counts;
};

__global__ void __launch_bounds__(256) k_ratio_per_set(const PerSetArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t n32 = ((int64_t)a.n_sets + 31) & ~(int64_t)31;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n32;
       g += (int64_t)gridDim.x * blockDim.x) {
    const bool in = g < a.n_sets;
    const int32_t grp = in ? a.group[g] : -1;
    const bool counted = grp >= 0 && grp < a.n_groups;
    const int64_t ns = counted ? a.per_set[g * 4] : 0;
    const bool valid = counted && ns >= 0 && a.valid[g];
    const bool exists = valid && ns > 0;
    const uint32_t peers = __match_any_sync(GP_FULL, counted ? grp : -1);
    const uint32_t b_ok = __ballot_sync(GP_FULL, exists);
    const uint32_t b_inv = __ballot_sync(GP_FULL, counted && !valid);
    if (counted && lane == __ffs(peers) - 1) {
      unsigned long long *c = reinterpret_cast<unsigned long long *>(
          a.counts + (((int64_t)a.setting * a.n_groups + grp) * a.n_slots + a.slot0) * 3);
      if (b_ok & peers) atomicAdd(c + 0, (unsigned long long)__popc(b_ok & peers));
      atomicAdd(c + 1, (unsigned long long)__popc(peers));
      if (b_inv & peers) atomicAdd(c + 2, (unsigned long long)__popc(b_inv & peers));
    }
  }
}

}  // namespace gp

extern "C" gp_status gp_sched_ratio(const gp_tasksets *ts, gp_ratio_mode mode,
                                    const uint8_t *verdicts, int32_t n_rows, int32_t slot0,
                                    int32_t n_slots, int32_t setting, int64_t *counts,
                                    const gp_exhaustive_opts *ex, void *stream) {
  using namespace gp;
  if (!ts || ts->n_sets < 0 || ts->n_groups < 1 || ts->n_tasks < 1 || ts->n_tasks > 256)
    return gp_fail(GP_EINVAL, "gp_sched_ratio: bad task sets");
  if (n_rows < 1 || slot0 < 0 || slot0 + n_rows > n_slots || setting < 0)
    return gp_fail(GP_EINVAL, "gp_sched_ratio: need 0 <= slot0, slot0 + n_rows <= n_slots");
  if (ts->n_sets > 0 && (!ts->valid || !ts->group))
    return gp_fail(GP_EINVAL, "gp_sched_ratio: null valid/group");
  cudaStream_t st = (cudaStream_t)stream;
  if (mode == GP_EXHAUSTIVE || mode == GP_THRESHOLD) {
    if (verdicts || n_rows != 1) return gp_fail(GP_EINVAL, "EXHAUSTIVE: verdicts must be NULL, n_rows 1");
    if (mode == GP_THRESHOLD) return gp_threshold_launch(ts, slot0, n_slots, setting, counts, ex, st);
    return gp_exhaustive_launch(ts, slot0, n_slots, setting, counts, ex, st);
  }
  if (mode == GP_FROM_PER_SET) {
    if (verdicts || n_rows != 1) return gp_fail(GP_EINVAL, "FROM_PER_SET: verdicts must be NULL, n_rows 1");
    if (!ex || !ex->per_set || !counts)
      return gp_fail(GP_EINVAL, "FROM_PER_SET: opts->per_set and counts are required");
    if (ts->n_sets == 0) return gp_cuda_check("gp_sched_ratio");
    PerSetArgs a{ex->per_set, ts->valid, ts->group, ts->n_sets, ts->n_groups, slot0, n_slots,
                 setting, counts};
    int64_t g1 = (ts->n_sets + 255) / 256;
    k_ratio_per_set<<<(unsigned)(g1 > 4096 ? 4096 : g1), 256, 0, st>>>(a);
    return gp_cuda_check("gp_sched_ratio(FROM_PER_SET)");
  }
  if (mode != GP_FROM_VERDICTS) return gp_fail(GP_EINVAL, "gp_sched_ratio: bad mode");
  if (ex) return gp_fail(GP_EINVAL, "FROM_VERDICTS: exhaustive options must be NULL");
  if (!verdicts || !counts) return gp_fail(GP_EINVAL, "FROM_VERDICTS: null verdicts/counts");
  if (ts->n_sets == 0) return gp_cuda_check("gp_sched_ratio");
  const size_t smem = (size_t)ts->n_groups * n_rows * 3 * sizeof(unsigned long long);
  if (smem > 96 * 1024) return gp_fail(GP_EINVAL, "FROM_VERDICTS: n_groups*n_rows too large");
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_ratio, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  RatioArgs a{verdicts, ts->valid, ts->group, ts->n_sets, n_rows, ts->n_groups, slot0, n_slots,
              setting, counts};
  int64_t work = (int64_t)ts->n_sets * n_rows;
  int64_t grid = (work + 1023) / 1024;
  if (grid > 148 * 2) grid = 148 * 2;
  if (grid < 1) grid = 1;
  k_ratio<<<(unsigned)grid, 256, smem, st>>>(a);
  return gp_cuda_check("gp_sched_ratio(FROM_VERDICTS)");
}
