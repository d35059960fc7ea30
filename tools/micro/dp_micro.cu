// FP64 issue-rate microbenchmark: how close to 64 DFMA/clk/SM do different
// operand patterns get on B200?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, long iters, double s) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = -1e-12 * s;
  double x[8], y[8], z[8];
  for (int i = 0; i < 8; ++i) { x[i] = i + 1.0; y[i] = a + i * 1e-10; z[i] = b * (i + 1); }
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = fma(x[i], a, b);                 // two shared operands
      else if (MODE == 1) x[i] = fma(x[i], y[i], z[i]);     // three distinct registers
      else if (MODE == 2) x[i] = fma(x[i], y[i], z[(i + 1) & 7]);
      else if (MODE == 3) x[i] = x[i] * y[i];
      else if (MODE == 4) { x[i] = fma(x[i], y[i], z[i]); z[i] = fma(z[i], y[i], x[i]); }
    }
  }
  double r = 0;
  for (int i = 0; i < 8; ++i) r += x[i] + z[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(double* buf, int sms, const char* name, int ops_per_it) {
  const int blocks = sms * 8, threads = 256;
  const long iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(buf, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double dfma = (double)blocks * threads * iters * ops_per_it;
  printf("%-28s %8.3f ms  %7.2f T DP-ops/s  (x2 = %6.2f TFLOP/s if FMA)\n", name, best,
         dfma / best / 1e9, 2 * dfma / best / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  cudaMalloc(&buf, sizeof(double) * sms * 8 * 256);
  run<0>(buf, sms, "fma(x, a, b) shared", 8);
  run<1>(buf, sms, "fma(x, y, z) distinct", 8);
  run<2>(buf, sms, "fma(x, y, z') distinct", 8);
  run<3>(buf, sms, "mul(x, y)", 8);
  run<4>(buf, sms, "2x fma chains distinct", 16);
  cudaFree(buf);
  return 0;
}
