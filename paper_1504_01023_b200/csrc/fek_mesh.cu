// fek_mesh.cu -- device-side synthetic inputs: the reference's
// unit-cube meshes (pkg/src/feklab/mesh.py:49-109) and numpy's
// Generator(PCG64).uniform stream, generated directly in HBM, bit-identical
// to the host generator for any element range [first, first + n).
//
// numpy PCG64 (numpy/random/src/pcg64): 128-bit LCG state' = a*state + inc,
// output XSL-RR 128/64 of the NEW state; Generator.uniform(low, high) =
// low + (high - low) * ((raw >> 11) * 2^-53).  Element ranges start anywhere
// thanks to the O(log k) LCG jump-ahead, so each GPU of a sharded run
// generates exactly its slice of the global mesh.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../include/fek.h"
#include "fek_status.h"

namespace {

using u128 = unsigned __int128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return (static_cast<u128>(2549297995355413924ull) << 64) | 4865540595714422341ull;
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ unsigned long long pcg_output(u128 s) {
  const unsigned long long x = static_cast<unsigned long long>(s >> 64) ^ static_cast<unsigned long long>(s);
  const unsigned r = static_cast<unsigned>(s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// next uniform draw of the stream; advances `s`
__device__ __forceinline__ double pcg_uniform(u128 &s, u128 inc, double low, double range) {
  s = s * pcg_mult() + inc;
  const double u = static_cast<double>(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
  return low + range * u;
}

struct Stream128 {
  u128 state, inc;
};

__host__ __forceinline__ Stream128 make_stream(const unsigned long long *s) {
  Stream128 r;
  r.state = (static_cast<u128>(s[0]) << 64) | s[1];
  r.inc = (static_cast<u128>(s[2]) << 64) | s[3];
  return r;
}

constexpr int kDrawChunk = 32;

__global__ void uniform_kernel(Stream128 st, long long first, long long count, double low, double range,
                               double *out) {
  const long long c0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * kDrawChunk;
  if (c0 >= count) return;
  u128 s = pcg_advance(st.state, st.inc, static_cast<unsigned long long>(first + c0));
  const long long c1 = c0 + kDrawChunk < count ? c0 + kDrawChunk : count;
  for (long long k = c0; k < c1; ++k) out[k] = pcg_uniform(s, st.inc, low, range);
}

// tet rows (mesh.py:49-68): cell (ix, iy, iz) C-order, then the six Kuhn path
// tets in itertools.permutations(range(3)) order; odd permutations swap
// vertices 1 and 2.  Every coordinate is i*h or i*h + h exactly as numpy
// forms it (int * float, then + h).
__constant__ int c_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__constant__ int c_odd[6] = {0, 1, 1, 0, 0, 1};

__global__ void tet_rows_kernel(long long nx, long long ny, long long nz, long long first, long long n,
                                double *out) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const long long e = first + k;
  const long long cell = e / 6;
  const int p = static_cast<int>(e % 6);
  const long long ix = cell / (ny * nz), rem = cell % (ny * nz);
  const long long iy = rem / nz, iz = rem % nz;
  const double h[3] = {1.0 / static_cast<double>(nx), 1.0 / static_cast<double>(ny), 1.0 / static_cast<double>(nz)};
  const double o[3] = {static_cast<double>(ix) * h[0], static_cast<double>(iy) * h[1], static_cast<double>(iz) * h[2]};
  const double up[3] = {o[0] + h[0], o[1] + h[1], o[2] + h[2]};
  double v[4][3];
  bool stepped[3] = {false, false, false};
  for (int i = 0; i < 3; ++i) v[0][i] = o[i];
  for (int m = 0; m < 3; ++m) {
    stepped[c_perm[p][m]] = true;
    for (int i = 0; i < 3; ++i) v[m + 1][i] = stepped[i] ? up[i] : o[i];
  }
  double *row = out + k * 12;
  const int order[4] = {0, c_odd[p] ? 2 : 1, c_odd[p] ? 1 : 2, 3};
  for (int a = 0; a < 4; ++a)
    for (int i = 0; i < 3; ++i) row[3 * a + i] = v[order[a]][i];
}

// prism rows (mesh.py:71-88) + optional top-face jitter (mesh.jitter_top_faces:
// draws 6e..6e+5 of the jitter stream, off = u * (amplitude * h))
constexpr int kPrismChunk = 8;

__global__ void prism_rows_kernel(long long nx, long long ny, long long first, long long n, int jitter,
                                  Stream128 js, double ax, double ay, double *out) {
  const long long k0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * kPrismChunk;
  if (k0 >= n) return;
  const double hx = 1.0 / static_cast<double>(nx), hy = 1.0 / static_cast<double>(ny);
  u128 s = 0;
  if (jitter) s = pcg_advance(js.state, js.inc, static_cast<unsigned long long>(6 * (first + k0)));
  const long long k1 = k0 + kPrismChunk < n ? k0 + kPrismChunk : n;
  for (long long k = k0; k < k1; ++k) {
    const long long e = first + k;
    const long long sq = e / 2;
    const int tri = static_cast<int>(e % 2);
    const long long ix = sq / ny, iy = sq % ny;
    const double x0 = static_cast<double>(ix) * hx, y0 = static_cast<double>(iy) * hy;
    const double x1 = x0 + hx, y1 = y0 + hy;
    double xy[3][2];
    if (tri == 0) {
      xy[0][0] = x0; xy[0][1] = y0; xy[1][0] = x1; xy[1][1] = y0; xy[2][0] = x0; xy[2][1] = y1;
    } else {
      xy[0][0] = x1; xy[0][1] = y0; xy[1][0] = x1; xy[1][1] = y1; xy[2][0] = x0; xy[2][1] = y1;
    }
    double *row = out + k * 18;
    for (int v = 0; v < 3; ++v) {
      row[3 * v + 0] = xy[v][0];
      row[3 * v + 1] = xy[v][1];
      row[3 * v + 2] = 0.0;
      double tx = xy[v][0], ty = xy[v][1];
      if (jitter) {
        tx = tx + pcg_uniform(s, js.inc, -1.0, 2.0) * ax;
        ty = ty + pcg_uniform(s, js.inc, -1.0, 2.0) * ay;
      }
      row[9 + 3 * v + 0] = tx;
      row[9 + 3 * v + 1] = ty;
      row[9 + 3 * v + 2] = 1.0;
    }
  }
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? FEK_OK : fek::record_cuda_error(e, "fek_mesh launch"); }

}  // namespace

extern "C" {

int fek_pcg64_uniform(const unsigned long long *stream, int64_t first, int64_t count, double low, double high,
                      double *out, void *cuda_stream) {
  if (!stream || first < 0 || count < 0 || (count > 0 && !out)) return FEK_ERR_ARGUMENT;
  if (count == 0) return FEK_OK;
  const long long threads = (count + kDrawChunk - 1) / kDrawChunk;
  const int block = 256;
  const long long grid = (threads + block - 1) / block;
  uniform_kernel<<<static_cast<unsigned>(grid), block, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
      make_stream(stream), first, count, low, high - low, out);
  return cuda_status(cudaGetLastError());
}

int fek_mesh_geometry(int32_t element, int64_t nx, int64_t ny, int64_t nz, int64_t first, int64_t n,
                      const unsigned long long *jitter_stream, double jitter_amplitude, double *out,
                      void *cuda_stream) {
  if (nx < 1 || ny < 1 || nz < 1 || first < 0 || n < 0 || (n > 0 && !out)) return FEK_ERR_ARGUMENT;
  if (n == 0) return FEK_OK;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  if (element == FEK_TETRAHEDRON) {
    if (jitter_stream) return FEK_ERR_ARGUMENT;
    if (first + n > 6 * nx * ny * nz) return FEK_ERR_ARGUMENT;
    tet_rows_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(nx, ny, nz, first, n, out);
  } else if (element == FEK_PRISM) {
    if (first + n > 2 * nx * ny) return FEK_ERR_ARGUMENT;
    const long long threads = (n + kPrismChunk - 1) / kPrismChunk;
    Stream128 js{0, 0};
    if (jitter_stream) js = make_stream(jitter_stream);
    // amplitude * h, formed exactly like jitter_top_faces (numpy: amplitude * h)
    const double ax = jitter_amplitude * (1.0 / static_cast<double>(nx));
    const double ay = jitter_amplitude * (1.0 / static_cast<double>(ny));
    prism_rows_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(nx, ny, first, n,
                                                                                   jitter_stream != nullptr, js, ax,
                                                                                   ay, out);
  } else {
    return FEK_ERR_ARGUMENT;
  }
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
