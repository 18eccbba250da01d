// fek_layout.cu -- on-device batch layout conversion.
//
// Device counterpart of layout.convert (pkg/src/feklab/layout.py:174-183,
// pack_rows/unpack_rows :72-94): a flat array of n rows of DS reals in one
// storage scheme (element-major = lane width 1, or lane-interleaved W) is
// rewritten in another, pad lanes of a partial interleaved block set to
// `pad`.  Interleaved index of (element e, datum d) = (e/W)*W*DS + d*W + e%W
// (layout.py:9), which is e*DS + d for W = 1.
//
// One CTA handles tiles of 128 elements: 128 is a multiple of every lane
// width, so a tile's input and output are each ONE contiguous range of the
// flat arrays.  The input range arrives by one TMA bulk copy (double-buffered
// on an mbarrier), the permutation runs shared -> shared, and the output range
// leaves by one bulk store (two output buffers): every byte crosses HBM once,
// in full lines, with the next tile's load in flight during the permutation.
// Arrays that are not 16-byte aligned take a plain-load kernel.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/fek.h"
#include "fek_device.cuh"
#include "fek_status.h"

namespace {

constexpr int kTile = 128;
constexpr int kThreads = 256;
constexpr int kMaxDs = 42;  // widest row the library handles: packed prism output rows (36 + 6)

long long padded(long long n, int w) { return (n + w - 1) / w * w; }

template <typename T>
__global__ void __launch_bounds__(kThreads) convert_kernel(const T *__restrict__ src, T *__restrict__ dst, long long n,
                                                           int ds, int w_in, int w_out, long long n_in,
                                                           long long n_out, long long tiles, T pad) {
  __shared__ T tile[kTile * kMaxDs];
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long long e0 = t * kTile;
    const int cnt_in = static_cast<int>(max(0ll, min(static_cast<long long>(kTile), n_in - e0)));
    const int cnt_out = static_cast<int>(max(0ll, min(static_cast<long long>(kTile), n_out - e0)));
    const T *s = src + e0 * ds;
    for (int i = threadIdx.x; i < cnt_in * ds; i += kThreads) tile[i] = s[i];
    __syncthreads();
    T *o = dst + e0 * ds;
    const int el = threadIdx.x % kTile;  // element within the tile
    if (el < cnt_out) {
      const bool real = e0 + el < n;
      const int bi = el / w_in, bo = el / w_out;
      const int src0 = bi * w_in * ds + (el - bi * w_in), dst0 = bo * w_out * ds + (el - bo * w_out);
      for (int d = threadIdx.x / kTile; d < ds; d += kThreads / kTile) o[dst0 + d * w_out] = real ? tile[src0 + d * w_in] : pad;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) convert_bulk_kernel(const T *__restrict__ src, T *__restrict__ dst,
                                                                long long n, int ds, int w_in, int w_out,
                                                                long long n_in, long long n_out, long long tiles,
                                                                T pad) {
  using namespace fek;
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned tile_bytes = kTile * ds * sizeof(T);  // a multiple of 512
  const uint32_t base = smem_u32(smem);
  auto in_addr = [&](int s) { return base + s * tile_bytes; };
  auto out_addr = [&](int k) { return base + (2 + k) * tile_bytes; };
  auto bar = [&](int s) { return base + 4 * tile_bytes + 8 * s; };
  const int tid = threadIdx.x;
  uint64_t policy = 0;
  if (tid == 0) {
    policy = policy_evict_first();
    mbar_init(bar(0), 1);
    mbar_init(bar(1), 1);
    fence_mbar_init();
  }
  __syncthreads();
  // thread 0: input range of tile t -> stage s (16-byte part by TMA, the
  // < 16-byte tail of a partial fp32 tile by plain loads before the arrive)
  auto issue = [&](long long t, int s) {
    if (t >= tiles) return;
    const long long e0 = t * kTile;
    const long long cnt = max(0ll, min(static_cast<long long>(kTile), n_in - e0));
    const unsigned bytes = static_cast<unsigned>(cnt * ds * sizeof(T)), b16 = bytes & ~15u;
    const char *g = reinterpret_cast<const char *>(src + e0 * ds);
    for (unsigned k = b16; k < bytes; k += 4) sts32(in_addr(s) + k, *reinterpret_cast<const uint32_t *>(g + k));
    mbar_arrive_expect_tx(bar(s), b16);
    if (b16) bulk_load(in_addr(s), g, b16, bar(s), policy);
  };
  if (tid == 0) {
    issue(blockIdx.x, 0);
    issue(blockIdx.x + static_cast<long long>(gridDim.x), 1);
  }
  for (int i = 0;; ++i) {
    const long long t = blockIdx.x + static_cast<long long>(i) * gridDim.x;
    if (t >= tiles) break;
    const int s = i & 1;
    const bool landed = mbar_wait(bar(s), (i >> 1) & 1);
    if (tid == 0) bulk_wait_read<1>();  // the store that last read output buffer s is done reading
    if (__syncthreads_or(!landed)) break;  // pipeline bug: leave rather than hang (output incomplete)
    const long long e0 = t * kTile;
    const int cnt_out = static_cast<int>(max(0ll, min(static_cast<long long>(kTile), n_out - e0)));
    const T *in = reinterpret_cast<const T *>(smem + s * tile_bytes);
    T *out = reinterpret_cast<T *>(smem + (2 + s) * tile_bytes);
    // thread -> one element of the tile (no per-datum index division); the
    // two halves of the CTA take alternate data
    const int el = tid % kTile;
    if (el < cnt_out) {
      const bool real = e0 + el < n;
      const int bi = el / w_in, bo = el / w_out;
      const int src0 = bi * w_in * ds + (el - bi * w_in), dst0 = bo * w_out * ds + (el - bo * w_out);
      for (int d = tid / kTile; d < ds; d += kThreads / kTile) out[dst0 + d * w_out] = real ? in[src0 + d * w_in] : pad;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const unsigned bytes = static_cast<unsigned>(cnt_out * ds * sizeof(T)), b16 = bytes & ~15u;
      char *g = reinterpret_cast<char *>(dst + e0 * ds);
      if (b16) bulk_store(g, out_addr(s), b16);
      bulk_commit();
      for (unsigned k = b16; k < bytes; k += 4) *reinterpret_cast<uint32_t *>(g + k) = lds32(out_addr(s) + k);
      issue(t + 2ll * gridDim.x, s);  // every thread is done reading stage s
    }
  }
  if (tid == 0) bulk_wait_all<0>();
}

template <typename T>
int launch_bulk(const T *src, T *dst, long long n, int ds, int w_in, int w_out, long long n_in, long long n_out,
                long long tiles, T pad, cudaStream_t st) {
  const int smem = 4 * kTile * ds * static_cast<int>(sizeof(T)) + 16;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute(convert_bulk_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, convert_bulk_kernel<T>, kThreads, smem);
  if (e != cudaSuccess) return fek::record_cuda_error(e, "fek_convert_layout setup");
  if (per_sm < 1) per_sm = 1;
  const long long cap = static_cast<long long>(sms) * per_sm;
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  convert_bulk_kernel<T><<<grid, kThreads, smem, st>>>(src, dst, n, ds, w_in, w_out, n_in, n_out, tiles, pad);
  e = cudaGetLastError();
  return e == cudaSuccess ? FEK_OK : fek::record_cuda_error(e, "fek_convert_layout launch");
}

bool valid_width(int w) { return w == 1 || w == 4 || w == 8 || w == 16 || w == 32 || w == 64; }

}  // namespace

extern "C" {

int fek_convert_layout(const void *src, int32_t in_lane_width, void *dst, int32_t out_lane_width, int64_t n_elements,
                       int32_t row_size, int32_t dtype, double pad_value, void *cuda_stream) {
  if (n_elements < 0 || row_size < 1 || row_size > kMaxDs || !valid_width(in_lane_width) ||
      !valid_width(out_lane_width) || (dtype != FEK_F64 && dtype != FEK_F32))
    return FEK_ERR_ARGUMENT;
  if (n_elements == 0) return FEK_OK;
  if (!src || !dst || src == dst) return FEK_ERR_ARGUMENT;
  const long long n_in = padded(n_elements, in_lane_width), n_out = padded(n_elements, out_lane_width);
  const long long tiles = (n_out + kTile - 1) / kTile;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0) {
    if (dtype == FEK_F64)
      return launch_bulk(static_cast<const double *>(src), static_cast<double *>(dst), n_elements, row_size,
                         in_lane_width, out_lane_width, n_in, n_out, tiles, pad_value, st);
    return launch_bulk(static_cast<const float *>(src), static_cast<float *>(dst), n_elements, row_size,
                       in_lane_width, out_lane_width, n_in, n_out, tiles, static_cast<float>(pad_value), st);
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(tiles < 8LL * sms ? tiles : 8LL * sms);
  if (dtype == FEK_F64) {
    convert_kernel<double><<<grid, kThreads, 0, st>>>(static_cast<const double *>(src), static_cast<double *>(dst),
                                                      n_elements, row_size, in_lane_width, out_lane_width, n_in,
                                                      n_out, tiles, pad_value);
  } else {
    convert_kernel<float><<<grid, kThreads, 0, st>>>(static_cast<const float *>(src), static_cast<float *>(dst),
                                                     n_elements, row_size, in_lane_width, out_lane_width, n_in, n_out,
                                                     tiles, static_cast<float>(pad_value));
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FEK_OK : fek::record_cuda_error(e, "fek_convert_layout launch");
}

}  // extern "C"
