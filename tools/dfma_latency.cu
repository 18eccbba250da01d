// dfma_latency.cu -- FP64 FMA latency and issue rate on one SM: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// launch <<<1, 32*W>>> with C independent dependent-chains per thread; prints cycles per DFMA per warp.
#include <cstdio>
template <int C>
__global__ void chains(double *out, int iters, long long *cyc) {
  double a[C];
#pragma unroll
  for (int c = 0; c < C; ++c) a[c] = threadIdx.x * 1e-3 + c;
  const double b = 0.9999999, d = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) a[c] = fma(a[c], b, d);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int C>
void run(int warps) {
  double *o;
  long long *c, h;
  cudaMalloc(&o, 1 << 20);
  cudaMalloc(&c, 8);
  const int iters = 4096;
  chains<C><<<1, 32 * warps>>>(o, iters, c);
  chains<C><<<1, 32 * warps>>>(o, iters, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("chains/thread %2d warps/CTA %2d (%d per SMSP): %.2f cycles per dependent DFMA step, %.3f DFMA warp-instr/clk/SM\n",
         C, warps, (warps + 3) / 4, double(h) / iters, double(C) * iters * warps / h);
  cudaFree(o);
  cudaFree(c);
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1);
  run<1>(4); run<2>(4); run<4>(4); run<8>(4);
  run<1>(8); run<2>(8); run<4>(8);
  run<1>(16); run<2>(16); run<4>(16);
  return 0;
}
