// fp64_peak.cu -- measured FP64 roofline denominators for this B200:
// DFMA throughput (CUDA cores) and DMMA (mma.sync m8n8k4 f64) throughput.
// Prints one JSON line.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  const int iters = 20000;
  float best_f = 1e30f, best_m = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_f) best_f = ms;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_m) best_m = ms;
  }
  const double fl_f = 2.0 * 16 * (double)iters * blocks * threads;
  const double fl_m = 2.0 * 8 * 8 * 4 * 8 * (double)(iters / 4) * blocks * (threads / 32);
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"sms\": %d, "
         "\"clock_khz_attr\": %d, \"ms_dfma\": %.3f, \"ms_dmma\": %.3f}\n",
         fl_f / (best_f * 1e-3) / 1e12, fl_m / (best_m * 1e-3) / 1e12, sms, clk, best_f, best_m);
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) { printf("error %s\n", cudaGetErrorString(ce)); return 1; }
  return 0;
}
