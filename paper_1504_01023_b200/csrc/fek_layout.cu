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
// flat arrays.  The input range is read coalesced into shared memory, the
// output range written coalesced from it -- every byte crosses HBM once.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/fek.h"
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
    const int bw = w_out * ds;
    for (int i = threadIdx.x; i < cnt_out * ds; i += kThreads) {
      const int blk = i / bw, rem = i - blk * bw;
      const int d = rem / w_out, lane = rem - d * w_out;
      const int el = blk * w_out + lane;  // element within the tile
      T v = pad;
      if (e0 + el < n) {
        const int b_in = el / w_in;
        v = tile[b_in * w_in * ds + d * w_in + (el - b_in * w_in)];
      }
      o[i] = v;
    }
    __syncthreads();
  }
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
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(tiles < 8LL * sms ? tiles : 8LL * sms);
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
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
