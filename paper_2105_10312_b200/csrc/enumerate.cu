// enumerate.cu -- A2 standalone: rank -> (block_of_task, block_size) (gp_enumerate).
// Thread per rank; the unranking tables live in shared memory.  The fused
// exhaustive evaluator (exhaustive.cu) uses the same building blocks but
// unranks once per lane and then steps successors in registers.
#include "gp_enum.cuh"

namespace gp {

struct EnumArgs {
  RankLayout L;
  uint64_t first;
  int64_t count;
  int8_t *bot;
  int16_t *bs;
};

__global__ void __launch_bounds__(256) k_enumerate(const EnumArgs a) {
  extern __shared__ uint32_t smem[];
  const EnumTables t = build_enum_tables(smem, a.L.M, a.L.n);
  const int n = a.L.n;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < a.count;
       x += (int64_t)gridDim.x * blockDim.x) {
    uint64_t r = a.first + (uint64_t)x;
    int k = 1;
    while (k < a.L.kmax && r >= a.L.k_base[k + 1]) ++k;
    uint64_t rr = r - a.L.k_base[k];
    uint32_t p = (uint32_t)(rr / a.L.per_pi[k]);
    uint32_t rho = (uint32_t)(rr % a.L.per_pi[k]);
    uint64_t labels = unrank_rgs(t, k, p);
    int32_t s[kEnumMaxTasks];
    unrank_sizes<kEnumMaxTasks>(t, k, rho, s);
    for (int i = 0; i < n; ++i) {
      a.bot[x * n + i] = (int8_t)((labels >> (4 * i)) & 15);
      a.bs[x * n + i] = (int16_t)(i < k ? s[i] : 0);
    }
  }
}

}  // namespace gp

extern "C" gp_status gp_enumerate(int32_t M, int32_t n, uint64_t first_rank, int64_t count,
                                  int8_t *block_of_task, int16_t *block_size, void *stream) {
  using namespace gp;
  if (n < 1 || n > kEnumMaxTasks || M < 1 || M > kEnumMaxM)
    return gp_fail(GP_EINVAL, "gp_enumerate: need 1 <= n <= 12 and 1 <= M <= 256 (n=%d M=%d)", n, M);
  if (count < 0) return gp_fail(GP_EINVAL, "gp_enumerate: count < 0");
  EnumArgs a;
  gp_status st = rank_layout(M, n, &a.L, true);
  if (st != GP_OK) return st;
  if (first_rank > a.L.total || (uint64_t)count > a.L.total - first_rank)
    return gp_fail(GP_EINVAL, "gp_enumerate: ranks beyond N_c = %llu", (unsigned long long)a.L.total);
  if (count == 0) return gp_cuda_check("gp_enumerate");
  if (!block_of_task || !block_size) return gp_fail(GP_EINVAL, "gp_enumerate: null output");
  a.first = first_rank;
  a.count = count;
  a.bot = block_of_task;
  a.bs = block_size;
  size_t smem = enum_table_words(M, n) * sizeof(uint32_t);
  int64_t grid = (count + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  k_enumerate<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(a);
  return gp_cuda_check("gp_enumerate");
}
