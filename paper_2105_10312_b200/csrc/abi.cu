// abi.cu -- host side of the C ABI: error plumbing and host-only calls.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "gp_common.cuh"
#include "gp_enum.cuh"

static thread_local char g_err[512] = "";

gp_status gp_fail(gp_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

gp_status gp_cuda_check(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return gp_fail(GP_ECUDA, "%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
  g_err[0] = '\0';
  return GP_OK;
}

gp_status gp_ok(void) {
  g_err[0] = '\0';
  return GP_OK;
}

extern "C" const char *gp_last_error(void) { return g_err; }

// N_c(M, n) = sum_k S(n,k) C(M,k) (C.1.6), host-only, exact with 128-bit checks.
extern "C" gp_status gp_count_candidates(int32_t M, int32_t n, uint64_t *count) {
  if (!count) return gp_fail(GP_EINVAL, "gp_count_candidates: null output");
  if (M < 1 || n < 1 || n > gp::kMaxTasks)
    return gp_fail(GP_EINVAL, "gp_count_candidates: M=%d n=%d out of range", M, n);
  gp::RankLayout L;
  gp_status st = gp::rank_layout(M, n, &L, /*need_u32_binom=*/false);
  if (st != GP_OK) return st;
  *count = L.total;
  g_err[0] = '\0';
  return GP_OK;
}
