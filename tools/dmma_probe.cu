// dmma_probe.cu -- measurement probe (not part of the product): does FP64 MMA (DMMA) add
// throughput on top of the FP64 FMA pipe on this GPU?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_probe.cu -o build/dmma_probe
//   ./build/dmma_probe            (prints one line per mode)
//
// Modes, each on 148 x 8 CTAs of 256 threads:
//   dfma   -- 8 independent DFMA chains per thread
//   dmma   -- 4 independent mma.sync.m8n8k4.f64 accumulators per warp
//   mma16  -- 2 independent mma.sync.m16n8k16.f64 accumulators per warp
//   mixed  -- the dfma and dmma loop bodies interleaved in one loop
// If DMMA ran on a pipe of its own, `mixed` would take max(dfma, dmma) time, not the sum.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void dmma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int MODE>
__global__ void __launch_bounds__(256) probe(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  double acc[4][2] = {};
  double acc16[2][4] = {};
  double A16[8], B16[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) A16[k] = a * (k + 1) * 1e-3;
#pragma unroll
  for (int k = 0; k < 4; ++k) B16[k] = b * (k + 1);
  for (int i = 0; i < iters; ++i) {
    if constexpr (MODE == 0 || MODE == 3) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    if constexpr (MODE == 1 || MODE == 3) {
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma884(acc[k], a, b);
    }
    if constexpr (MODE == 2) {
#pragma unroll
      for (int k = 0; k < 2; ++k) dmma16816(acc16[k], A16, B16);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
#pragma unroll
  for (int k = 0; k < 2; ++k) s += acc16[k][0] + acc16[k][3];
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

template <int MODE>
float run(double *d, int blocks, int iters) {
  probe<MODE><<<blocks, 256>>>(d, 100, 0.999999, 1e-7);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  probe<MODE><<<blocks, 256>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0;
  cudaEventElapsedTime(&ms, s, e);
  cudaEventDestroy(s);
  cudaEventDestroy(e);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, iters = 20000;
  double *d = nullptr;
  cudaMalloc(&d, 8);
  const double threads = 256.0 * blocks, warps = threads / 32.0;
  const double fl_dfma = 2.0 * 8 * threads * iters;          // 8 DFMA per thread-iteration
  const double fl_dmma = 2.0 * 4 * 256 * warps * iters;      // 4 m8n8k4 per warp-iteration, 256 FMA each
  const double fl_16 = 2.0 * 2 * 2048 * warps * iters;       // 2 m16n8k16 per warp-iteration
  const float t0 = run<0>(d, blocks, iters), t1 = run<1>(d, blocks, iters), t2 = run<2>(d, blocks, iters),
              t3 = run<3>(d, blocks, iters);
  printf("dfma  %8.3f ms  %6.2f TFLOP/s\n", t0, fl_dfma / (t0 * 1e-3) / 1e12);
  printf("dmma  %8.3f ms  %6.2f TFLOP/s (m8n8k4)\n", t1, fl_dmma / (t1 * 1e-3) / 1e12);
  printf("mma16 %8.3f ms  %6.2f TFLOP/s (m16n8k16)\n", t2, fl_16 / (t2 * 1e-3) / 1e12);
  printf("mixed %8.3f ms  %6.2f TFLOP/s combined; dfma + dmma alone = %.3f ms, max = %.3f ms\n", t3,
         (fl_dfma + fl_dmma) / (t3 * 1e-3) / 1e12, t0 + t1, t0 > t1 ? t0 : t1);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
