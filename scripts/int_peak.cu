// int_peak.cu -- integer issue-rate microbenchmark ("the INT32 pipe
// rate per SMSP on sm_100 is not assumed; measure it with an IADD3/LOP3/IMAD
// dependent-chain microbenchmark").
//
// Every thread runs C independent dependency chains of one operation for N
// iterations (C chains hide the pipeline latency); the grid fills every SM.
// Throughput = threads * N * C ops / time, reported as lane-ops/s and as
// warp-instructions per clock per SMSP at the SM clock given on the command line
// (the bench records the clock under load with NVML).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak scripts/int_peak.cu
//   ./int_peak [sm_mhz]      -> one JSON line
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 1 << 14;

template <int OP>
__global__ void __launch_bounds__(256) k_chain(unsigned *out, unsigned seed) {
  unsigned a[kChains], b = seed ^ threadIdx.x, c = seed * 2654435761u + blockIdx.x;
#pragma unroll
  for (int j = 0; j < kChains; ++j) a[j] = threadIdx.x * (j + 1) + blockIdx.x;
  for (int it = 0; it < kIters; ++it) {
    unsigned o[kChains];  // operands from the previous iteration's neighbouring chain
#pragma unroll
    for (int j = 0; j < kChains; ++j) o[j] = a[(j + 1) % kChains];
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
      if (OP == 0) a[j] = a[j] + o[j] + b;            // IADD3
      else if (OP == 1) a[j] = (a[j] & o[j]) ^ b;     // LOP3
      else if (OP == 2) a[j] = a[j] * o[j] + b;       // IMAD
      else if (OP == 3) a[j] = (j & 1) ? (a[j] * o[j] + b) : ((a[j] & o[j]) ^ b);  // IMAD / LOP3
      else a[j] = (j & 1) ? (a[j] + o[j] + b) : ((a[j] & o[j]) ^ b);  // IADD3 / LOP3
    }
    b ^= c;
  }
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) r ^= a[j];
  if (r == 0x12345678u) out[blockIdx.x] = r;  // never true in practice; defeats dead-code removal
}

template <int OP>
static double run(int blocks, unsigned *out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_chain<OP><<<blocks, 256>>>(out, 1u);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_chain<OP><<<blocks, 256>>>(out, 7u + r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 5.0 * blocks * 256.0 * kIters * kChains;
  return ops / (ms * 1e-3);
}

int main(int argc, char **argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8;  // 2048 threads per SM
  unsigned *out = nullptr;
  cudaMalloc(&out, blocks * sizeof(unsigned));
  const char *names[5] = {"iadd3", "lop3", "imad", "imad_lop3_mix", "iadd3_lop3_mix"};
  double v[5];
  v[0] = run<0>(blocks, out);
  v[1] = run<1>(blocks, out);
  v[2] = run<2>(blocks, out);
  v[3] = run<3>(blocks, out);
  v[4] = run<4>(blocks, out);
  const double clk = mhz * 1e6, smsp = sms * 4.0;
  printf("{\"sms\": %d, \"sm_mhz_assumed\": %.0f, \"ops\": {", sms, mhz);
  for (int i = 0; i < 5; ++i)
    printf("%s\"%s\": {\"lane_ops_per_s\": %.4e, \"warp_inst_per_clk_per_smsp\": %.3f}",
           i ? ", " : "", names[i], v[i], v[i] / 32.0 / clk / smsp);
  printf("}, \"note\": \"%d chains per thread (each op reads its own and a neighbour chain's "
         "previous value), %d iterations, %d blocks x 256 threads; one extra LOP per iteration "
         "(b ^= c) per %d counted ops is not counted\"}\n",
         kChains, kIters, blocks, kChains);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
