// probe.cu -- measurement probe (not part of the product): FP64 DFMA peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -cudart static \
//        tools/probe.cu -o tools/libfekprobe.so
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_peak(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

__global__ void __launch_bounds__(256) ffma_peak(float *out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-6f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 12345.678f) out[0] = s;
}

extern "C" int probe_fp32_peak(int blocks, int iters, float *ms_out, double *tflops_out) {
  float *d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return 1;
  ffma_peak<<<blocks, 256>>>(d, 1000, 0.999999f, 1e-7f);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  ffma_peak<<<blocks, 256>>>(d, iters, 0.999999f, 1e-7f);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0;
  cudaEventElapsedTime(&ms, s, e);
  *ms_out = ms;
  *tflops_out = 2.0 * 16.0 * 256.0 * blocks * (double)iters / (ms * 1e-3) / 1e12;
  cudaFree(d);
  cudaEventDestroy(s);
  cudaEventDestroy(e);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int probe_fp64_peak(int blocks, int iters, float *ms_out, double *tflops_out) {
  double *d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return 1;
  dfma_peak<<<blocks, 256>>>(d, 1000, 0.999999, 1e-7);  // warm
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  dfma_peak<<<blocks, 256>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0;
  cudaEventElapsedTime(&ms, s, e);
  *ms_out = ms;
  *tflops_out = 2.0 * 8.0 * 256.0 * blocks * (double)iters / (ms * 1e-3) / 1e12;
  cudaFree(d);
  cudaEventDestroy(s);
  cudaEventDestroy(e);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
