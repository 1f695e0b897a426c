// fp64_mix.cu -- do DFMA (FP64 CUDA-core pipe) and DMMA (mma.sync f64) share
// one throughput budget on this B200?  Times DFMA-only, DMMA-only and mixed
// kernels (same warp interleaving both, and half the warps each); if the
// mixed time is ~max of the parts the units are separate, ~sum: shared.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NF, int NM>
__global__ void mix_kernel(double* out, int iters, double a, double b, int split) {
  double x[NF > 0 ? NF : 1];
  double c[NM > 0 ? NM : 1][2];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) c[i][0] = c[i][1] = 0.0;
  const int warp = threadIdx.x >> 5;
  const bool do_f = !split || (warp & 1) == 0;
  const bool do_m = !split || (warp & 1) == 1;
  const double ma = threadIdx.x * 1e-3, mb = 0.5;
  for (int it = 0; it < iters; ++it) {
    if (do_m) {
#pragma unroll
      for (int i = 0; i < NM; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(ma), "d"(mb));
    }
    if (do_f) {
#pragma unroll
      for (int i = 0; i < NF; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dadd_kernel(double* out, int iters, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = x[i] + b;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void rcp_kernel(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1.0 / x[i];
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
static float best_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256, iters = 4000;
  const double lanes = (double)blocks * threads;
  const double warps = lanes / 32;
  // per iteration: DFMA 16 per lane; DMMA 4 per warp (256 FMAs each)
  float tf = best_ms([&] { mix_kernel<16, 0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, 0); });
  float tm = best_ms([&] { mix_kernel<0, 4><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, 0); });
  float tfm = best_ms([&] { mix_kernel<16, 4><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, 0); });
  float tsplit = best_ms([&] { mix_kernel<16, 4><<<blocks, threads>>>(out, iters, 0.999999, 1e-7, 1); });
  float ta = best_ms([&] { dadd_kernel<<<blocks, threads>>>(out, iters, 1e-7); });
  float tr = best_ms([&] { rcp_kernel<<<blocks, threads>>>(out, iters); });
  const double fma_f = 16.0 * iters * lanes, fma_m = 4.0 * 256 * iters * warps;
  printf("{\"dfma_ms\": %.3f, \"dmma_ms\": %.3f, \"mixed_same_warp_ms\": %.3f, "
         "\"mixed_split_warps_ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, "
         "\"mixed_same_warp_tflops\": %.2f, \"mixed_split_tflops\": %.2f, "
         "\"dadd_gops\": %.1f, \"drcp_gops\": %.1f}\n",
         tf, tm, tfm, tsplit, 2 * fma_f / (tf * 1e9), 2 * fma_m / (tm * 1e9),
         2 * (fma_f + fma_m) / (tfm * 1e9), 2 * (fma_f + fma_m) / 2 / (tsplit * 1e9),
         16.0 * iters * lanes / (ta * 1e6), 8.0 * iters * lanes / (tr * 1e6));
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) { printf("error %s\n", cudaGetErrorString(ce)); return 1; }
  return 0;
}
