// FP64 dependent-chain microbenchmark: DFMA throughput of C independent
// dependent chains per thread at W resident warps per SM (one CTA of 32 W
// threads per SM), as a fraction of 64 DFMA/clk/SM.  Answers: how many
// (warps x chains) per scheduler does the FP64 pipe need on B200?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dp_chain dp_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chain(double* out, long iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int i = 0; i < C; ++i) x[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 8; ++rep)
#pragma unroll
      for (int i = 0; i < C; ++i) x[i] = fma(x[i], a, b);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) r += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int C>
void run(double* buf, int sms, int warps, double clock_ghz) {
  const long iters = 1 << 13;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    chain<C><<<sms, 32 * warps>>>(buf, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double dfma = (double)sms * 32 * warps * iters * 8 * C;
  const double per_clk_sm = dfma / (best * 1e-3) / (clock_ghz * 1e9) / sms;
  printf("warps/SM %2d chains %d: %7.3f ms  %6.2f DFMA/clk/SM (%5.1f %% of 64)\n", warps, C, best,
         per_clk_sm, 100.0 * per_clk_sm / 64.0);
}

int main() {
  int sms, khz;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double ghz = khz * 1e-6;
  printf("SMs %d, clock %.3f GHz\n", sms, ghz);
  double* buf;
  cudaMalloc(&buf, sizeof(double) * sms * 1024);
  for (int w : {4, 8, 16, 24, 32}) {
    run<1>(buf, sms, w, ghz);
    run<2>(buf, sms, w, ghz);
    run<4>(buf, sms, w, ghz);
  }
  cudaFree(buf);
  return 0;
}
