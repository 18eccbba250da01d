// fek_abi.cu -- C-ABI of libfek.so (include/fek.h): descriptor validation,
// kernel dispatch, the host-buffer pipeline, error decoding and checksums.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/fek.h"
#include "fek_dispatch.cuh"
#include "fek_status.h"

namespace {
thread_local char g_cuda_error[256] = "";
}  // namespace

int fek::record_cuda_error(cudaError_t e, const char *what) {
  std::snprintf(g_cuda_error, sizeof(g_cuda_error), "%s: %s", what, cudaGetErrorString(e));
  return FEK_ERR_CUDA;
}

namespace {

using fek::KernelEntry;
using fek::kIndexCount;
using fek::kernel_index;
using fek::LaunchParams;

int cuda_fail(cudaError_t e, const char *what) { return fek::record_cuda_error(e, what); }

#define FEK_CUDA(call)                              \
  do {                                              \
    cudaError_t _e = (call);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// kernels are instantiated per case in cases/*.cu (parallel compilation)
const KernelEntry *kernel_table() {
  static KernelEntry table[kIndexCount];
  static std::once_flag once;
  std::call_once(once, [] {
    fek::register_f64_tet_poisson(table);
    fek::register_f64_tet_convdiff(table);
    fek::register_f64_prism_poisson(table);
    fek::register_f64_prism_convdiff(table);
    fek::register_f32_tet_poisson(table);
    fek::register_f32_tet_convdiff(table);
    fek::register_f32_prism_poisson(table);
    fek::register_f32_prism_convdiff(table);
  });
  return table;
}

// per (device, kernel) launch geometry, computed once
struct LaunchGeometry {
  int ready = 0;
  int resident = 0;  // CTAs per SM
  int sms = 0;
};
constexpr int kMaxDevices = 16;
LaunchGeometry g_geometry[kMaxDevices][kIndexCount];
std::mutex g_geometry_mutex;

int launch_geometry(int idx, const KernelEntry &ke, LaunchGeometry *out) {
  int dev = 0;
  FEK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return FEK_ERR_ARGUMENT;
  std::lock_guard<std::mutex> lock(g_geometry_mutex);
  LaunchGeometry &lg = g_geometry[dev][idx];
  if (!lg.ready) {
    FEK_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void *>(ke.fn),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ke.smem)));
    FEK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lg.resident, ke.fn, ke.threads, ke.smem));
    FEK_CUDA(cudaDeviceGetAttribute(&lg.sms, cudaDevAttrMultiProcessorCount, dev));
    if (lg.resident < 1) lg.resident = 1;
    lg.ready = 1;
  }
  *out = lg;
  return FEK_OK;
}

int n_shape(int et) { return et == FEK_TETRAHEDRON ? 4 : 6; }
int n_quad(int et) { return et == FEK_TETRAHEDRON ? 4 : 6; }
int geometry_size(int et) { return 3 * n_shape(et); }
int coefficient_size(int et, int pb) { return pb == FEK_POISSON ? n_quad(et) : 20; }
int real_bytes(int dtype) { return dtype == FEK_F64 ? 8 : 4; }

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int validate(const fek_batch_desc *d, bool need_pointers) {
  if (!d) return FEK_ERR_ARGUMENT;
  if (d->element < 0 || d->element > 1 || d->problem < 0 || d->problem > 1) return FEK_ERR_ARGUMENT;
  if (d->variant < 0 || d->variant > 2 || d->geometry_path < 0 || d->geometry_path > 1) return FEK_ERR_ARGUMENT;
  if (d->dtype < 0 || d->dtype > 1) return FEK_ERR_ARGUMENT;
  if (d->geometry_path == FEK_GEO_LINEAR && d->element != FEK_TETRAHEDRON) return FEK_ERR_ARGUMENT;
  if (d->layout == FEK_ELEMENT_MAJOR) {
    if (d->lane_width != 1) return FEK_ERR_ARGUMENT;
  } else if (d->layout == FEK_LANE_INTERLEAVED) {
    const int w = d->lane_width;
    if (!(w == 1 || w == 4 || w == 8 || w == 16 || w == 32 || w == 64)) return FEK_ERR_ARGUMENT;
  } else {
    return FEK_ERR_ARGUMENT;
  }
  if (d->n_elements < 0 || d->base_index < 0 || d->ctas_per_sm < 0) return FEK_ERR_ARGUMENT;
  if (d->tile_elements != 0) {
    const int t = d->tile_elements;
    const bool natural = d->variant == FEK_QSS &&
                         d->geometry_path == (d->element == FEK_TETRAHEDRON ? FEK_GEO_LINEAR : FEK_GEO_GENERIC);
    if (!natural || !(t == 64 || t == 128 || t == 256)) return FEK_ERR_ARGUMENT;
  }
  const bool packed = d->out_format == FEK_OUT_PACKED;
  if (!packed && d->out_format != FEK_OUT_SPLIT) return FEK_ERR_ARGUMENT;
  if (packed) {
    const int w = d->out_lane_width;
    if (!(w == 1 || w == 4 || w == 8 || w == 16 || w == 32 || w == 64)) return FEK_ERR_ARGUMENT;
  }
  if (need_pointers && d->n_elements > 0) {
    if (!d->geometry || !d->coefficients || !d->stiffness || (!packed && !d->load)) return FEK_ERR_ARGUMENT;
    if (!aligned16(d->geometry) || !aligned16(d->coefficients) || !aligned16(d->stiffness) ||
        (!packed && !aligned16(d->load)))
      return FEK_ERR_ALIGNMENT;
    if (reinterpret_cast<uintptr_t>(d->scheduler) % 8) return FEK_ERR_ALIGNMENT;
  }
  return FEK_OK;
}

struct ApplyArgs {  // a consumer launch: fek_apply (mode 1) or fek_assemble (mode 2)
  int mode;
  const int32_t *element_nodes;
  const void *x;
  void *y;
  void *f;
  const int32_t *row_ptr;
  const int32_t *col;
};

int launch(const fek_batch_desc *d, cudaStream_t stream, int *grid_out, int *block_out, int *smem_out,
           int *tile_out, bool do_launch, const ApplyArgs *ap = nullptr) {
  const int idx = ap ? fek::consumer_index(d->dtype, d->element, d->problem, ap->mode) : d->tile_elements
                      ? fek::tiled_index(d->dtype, d->element, d->problem,
                                         d->tile_elements == 64 ? 0 : (d->tile_elements == 128 ? 1 : 2))
                      : kernel_index(d->dtype, d->element, d->problem, d->variant, d->geometry_path);
  const KernelEntry &ke = kernel_table()[idx];
  if (!ke.fn) return FEK_ERR_ARGUMENT;
  LaunchGeometry lg;
  if (int rc = launch_geometry(idx, ke, &lg)) return rc;
  const long long tiles = (d->n_elements + ke.tile - 1) / ke.tile;
  const int per_sm = (d->ctas_per_sm > 0 && d->ctas_per_sm < lg.resident) ? d->ctas_per_sm : lg.resident;
  const long long cap = static_cast<long long>(lg.sms) * per_sm;
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  if (grid_out) *grid_out = grid;
  if (block_out) *block_out = ke.threads;
  if (smem_out) *smem_out = static_cast<int>(ke.smem);
  if (tile_out) *tile_out = ke.tile;
  if (!do_launch || grid == 0) return FEK_OK;
  LaunchParams p;
  p.geometry = d->geometry;
  p.coefficients = d->coefficients;
  p.stiffness = d->stiffness;
  p.load = d->load;
  p.error_key = d->error_key;
  p.n = d->n_elements;
  p.base = d->base_index;
  p.lane_width = d->layout == FEK_ELEMENT_MAJOR ? 1 : d->lane_width;
  p.out_packed = d->out_format == FEK_OUT_PACKED;
  p.out_width = p.out_packed ? d->out_lane_width : 1;
  p.scheduler = d->scheduler;
  p.element_nodes = ap ? ap->element_nodes : nullptr;
  p.x = ap ? ap->x : nullptr;
  p.y = ap ? ap->y : nullptr;
  p.f = ap ? ap->f : nullptr;
  p.row_ptr = ap ? ap->row_ptr : nullptr;
  p.col = ap ? ap->col : nullptr;
  ke.fn<<<grid, ke.threads, ke.smem, stream>>>(p);
  FEK_CUDA(cudaGetLastError());
  return FEK_OK;
}

// --------------------------------------------------------------------------
// checksum kernels (deterministic fixed-order reduction)
// --------------------------------------------------------------------------

constexpr int kSumBlocks = 592;  // 148 SMs x 4
constexpr int kSumThreads = 256;

template <typename R>
__device__ __forceinline__ unsigned long long real_bits(R v) {
  if constexpr (sizeof(R) == 8) {
    return static_cast<unsigned long long>(__double_as_longlong(v));
  } else {
    return static_cast<unsigned long long>(__float_as_uint(v));
  }
}

template <typename R>
__global__ void __launch_bounds__(kSumThreads) checksum_partials(const R *A, const R *b, long long n, int na,
                                                                 int ns, long long base, double *part_f,
                                                                 unsigned long long *part_u) {
  __shared__ double sf[4][kSumThreads];
  __shared__ unsigned long long su[2][kSumThreads];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = per * blockIdx.x;
  const long long hi = lo + per < n ? lo + per : n;
  double f[4] = {0, 0, 0, 0};
  unsigned long long u[2] = {0, 0};
  for (long long i = lo * na + threadIdx.x; i < hi * na; i += blockDim.x) {
    const R v = A[i];
    f[0] += static_cast<double>(v);
    f[2] += fabs(static_cast<double>(v));
    u[0] += real_bits(v) * (2ull * static_cast<unsigned long long>(base * na + i) + 1ull);
  }
  for (long long i = lo * ns + threadIdx.x; i < hi * ns; i += blockDim.x) {
    const R v = b[i];
    f[1] += static_cast<double>(v);
    f[3] += fabs(static_cast<double>(v));
    u[1] += real_bits(v) * (2ull * static_cast<unsigned long long>(base * ns + i) + 1ull);
  }
  for (int k = 0; k < 4; ++k) sf[k][threadIdx.x] = f[k];
  su[0][threadIdx.x] = u[0];
  su[1][threadIdx.x] = u[1];
  __syncthreads();
  for (int stride = kSumThreads / 2; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride) {
      for (int k = 0; k < 4; ++k) sf[k][threadIdx.x] += sf[k][threadIdx.x + stride];
      su[0][threadIdx.x] += su[0][threadIdx.x + stride];
      su[1][threadIdx.x] += su[1][threadIdx.x + stride];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) part_f[4 * blockIdx.x + k] = sf[k][0];
    part_u[2 * blockIdx.x] = su[0][0];
    part_u[2 * blockIdx.x + 1] = su[1][0];
  }
}

__global__ void checksum_final(const double *part_f, const unsigned long long *part_u, int blocks, double *out_f,
                               unsigned long long *out_u) {
  if (threadIdx.x != 0) return;
  double f[4] = {0, 0, 0, 0};
  unsigned long long u[2] = {0, 0};
  for (int i = 0; i < blocks; ++i) {
    for (int k = 0; k < 4; ++k) f[k] += part_f[4 * i + k];
    u[0] += part_u[2 * i];
    u[1] += part_u[2 * i + 1];
  }
  for (int k = 0; k < 4; ++k) out_f[k] = f[k];
  out_u[0] = u[0];
  out_u[1] = u[1];
}

}  // namespace

extern "C" {

int fek_abi_version(void) { return FEK_ABI_VERSION; }

size_t fek_batch_desc_size(void) { return sizeof(fek_batch_desc); }

const char *fek_status_string(int status) {
  switch (status) {
    case FEK_OK: return "ok";
    case FEK_ERR_ARGUMENT: return "invalid argument";
    case FEK_ERR_ALIGNMENT: return "base pointer not 16-byte aligned";
    case FEK_ERR_CUDA: return "CUDA runtime error";
    case FEK_ERR_WORKSPACE: return "workspace too small";
    case FEK_ERR_GEOMETRY: return "degenerate or inverted element";
    default: return "unknown status";
  }
}

const char *fek_last_cuda_error(void) { return g_cuda_error; }

int fek_integrate(const fek_batch_desc *d, void *cuda_stream) {
  if (int rc = validate(d, true)) return rc;
  if (d->n_elements > 0 && !d->error_key) return FEK_ERR_ARGUMENT;
  return launch(d, static_cast<cudaStream_t>(cuda_stream), nullptr, nullptr, nullptr, nullptr, true);
}

static int consumer_launch(const fek_batch_desc *d, const ApplyArgs &ap, void *cuda_stream) {
  if (int rc = validate(d, false)) return rc;
  const bool natural = d->variant == FEK_QSS &&
                       d->geometry_path == (d->element == FEK_TETRAHEDRON ? FEK_GEO_LINEAR : FEK_GEO_GENERIC);
  if (!natural || d->layout != FEK_ELEMENT_MAJOR || d->tile_elements != 0) return FEK_ERR_ARGUMENT;
  if (d->n_elements == 0) return FEK_OK;
  if (!d->geometry || !d->coefficients || !d->error_key || !ap.element_nodes || !ap.y) return FEK_ERR_ARGUMENT;
  if (ap.mode == fek::MODE_APPLY && !ap.x) return FEK_ERR_ARGUMENT;
  if (ap.mode == fek::MODE_ASSEMBLE && (!ap.row_ptr || !ap.col)) return FEK_ERR_ARGUMENT;
  if (!aligned16(d->geometry) || !aligned16(d->coefficients) || reinterpret_cast<uintptr_t>(d->scheduler) % 8)
    return FEK_ERR_ALIGNMENT;
  return launch(d, static_cast<cudaStream_t>(cuda_stream), nullptr, nullptr, nullptr, nullptr, true, &ap);
}

int fek_apply(const fek_batch_desc *d, const int32_t *element_nodes, const void *x, void *y, void *f,
              void *cuda_stream) {
  return consumer_launch(d, ApplyArgs{fek::MODE_APPLY, element_nodes, x, y, f, nullptr, nullptr}, cuda_stream);
}

int fek_assemble(const fek_batch_desc *d, const int32_t *element_nodes, const int32_t *row_ptr, const int32_t *col,
                 void *values, void *f, void *cuda_stream) {
  return consumer_launch(d, ApplyArgs{fek::MODE_ASSEMBLE, element_nodes, nullptr, values, f, row_ptr, col},
                         cuda_stream);
}

int fek_launch_config(const fek_batch_desc *d, int *grid, int *block, int *smem_bytes, int *tile_elements) {
  if (int rc = validate(d, false)) return rc;
  return launch(d, nullptr, grid, block, smem_bytes, tile_elements, false);
}

int fek_decode_error(unsigned long long key, int64_t *element, int32_t *point, int32_t *kind) {
  if (key == FEK_NO_ERROR) return FEK_ERR_ARGUMENT;
  const unsigned long long blk = key >> 24;
  const int q = static_cast<int>((key >> 20) & 15ull);
  const unsigned long long within = (key >> 7) & 8191ull;
  if (element) *element = static_cast<int64_t>((blk << fek::ERROR_BLOCK_SHIFT) | within);
  if (point) *point = q == 15 ? -1 : q;
  if (kind) *kind = static_cast<int32_t>(key & 127ull);
  return FEK_OK;
}

}  // extern "C"

// one-thread element queries (templates: C++ linkage)
template <template <typename, int> class Kern>
static int element_query(const fek_batch_desc *d, int64_t element, int32_t point, double *out, void *cuda_stream) {
  if (int rc = validate(d, false)) return rc;
  if (!d->geometry || !out || element < 0 || element >= d->n_elements) return FEK_ERR_ARGUMENT;
  const int w = d->layout == FEK_ELEMENT_MAJOR ? 1 : d->lane_width;
  const int nq = n_quad(d->element);
  if (point >= nq || point < -1) return FEK_ERR_ARGUMENT;
  if (point < 0 && d->element != FEK_TETRAHEDRON) return FEK_ERR_ARGUMENT;  // affine path: tets only
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  if (d->dtype == FEK_F64) {
    if (d->element == FEK_TETRAHEDRON)
      Kern<double, fek::TET>::launch(d->geometry, element, w, point, out, s);
    else
      Kern<double, fek::PRISM>::launch(d->geometry, element, w, point, out, s);
  } else {
    if (d->element == FEK_TETRAHEDRON)
      Kern<float, fek::TET>::launch(d->geometry, element, w, point, out, s);
    else
      Kern<float, fek::PRISM>::launch(d->geometry, element, w, point, out, s);
  }
  FEK_CUDA(cudaGetLastError());
  return FEK_OK;
}

// exact classification pass (fek_classify)
template <typename R, int ET, int GEO>
static void launch_classify(const fek_batch_desc *d, int lane_width, int grid, cudaStream_t s) {
  fek::classify_kernel<R, ET, GEO><<<grid, 256, 0, s>>>(d->geometry, d->n_elements, d->base_index, lane_width,
                                                        d->error_key);
}

static int classify_batch(const fek_batch_desc *d, cudaStream_t s) {
  if (int rc = validate(d, false)) return rc;
  if (d->n_elements == 0) return FEK_OK;
  if (!d->geometry || !d->error_key) return FEK_ERR_ARGUMENT;
  int dev = 0, sms = 148;
  FEK_CUDA(cudaGetDevice(&dev));
  FEK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long blocks = (d->n_elements + 255) / 256, cap = 8ll * sms;
  const int grid = static_cast<int>(blocks < cap ? blocks : cap);
  const int w = d->layout == FEK_ELEMENT_MAJOR ? 1 : d->lane_width;
  const bool lin = d->geometry_path == FEK_GEO_LINEAR;
  if (d->dtype == FEK_F64) {
    if (d->element == FEK_PRISM) launch_classify<double, fek::PRISM, fek::GEO_GENERIC>(d, w, grid, s);
    else if (lin) launch_classify<double, fek::TET, fek::GEO_LINEAR>(d, w, grid, s);
    else launch_classify<double, fek::TET, fek::GEO_GENERIC>(d, w, grid, s);
  } else {
    if (d->element == FEK_PRISM) launch_classify<float, fek::PRISM, fek::GEO_GENERIC>(d, w, grid, s);
    else if (lin) launch_classify<float, fek::TET, fek::GEO_LINEAR>(d, w, grid, s);
    else launch_classify<float, fek::TET, fek::GEO_GENERIC>(d, w, grid, s);
  }
  FEK_CUDA(cudaGetLastError());
  return FEK_OK;
}

template <typename R, int ET>
struct ErrorDetail {
  static void launch(const void *g, int64_t e, int w, int q, double *out, cudaStream_t s) {
    fek::error_detail_kernel<R, ET><<<1, 1, 0, s>>>(g, e, w, q, out);
  }
};

template <typename R, int ET>
struct Jacobian {
  static void launch(const void *g, int64_t e, int w, int q, double *out, cudaStream_t s) {
    fek::jacobian_kernel<R, ET><<<1, 1, 0, s>>>(g, e, w, q, out);
  }
};

extern "C" {

int fek_classify(const fek_batch_desc *d, void *cuda_stream) {
  return classify_batch(d, static_cast<cudaStream_t>(cuda_stream));
}

int fek_error_detail(const fek_batch_desc *d, int64_t element, int32_t point, double *out_det_tol,
                     void *cuda_stream) {
  return element_query<ErrorDetail>(d, element, point, out_det_tol, cuda_stream);
}

int fek_jacobian(const fek_batch_desc *d, int64_t element, int32_t point, double *out20, void *cuda_stream) {
  return element_query<Jacobian>(d, element, point, out20, cuda_stream);
}

size_t fek_checksum_scratch_bytes(void) { return static_cast<size_t>(kSumBlocks) * (4 * 8 + 2 * 8); }

int fek_checksum(const fek_batch_desc *d, void *partials, double *out_f64, unsigned long long *out_u64,
                 void *cuda_stream) {
  if (int rc = validate(d, false)) return rc;
  if (!partials || !out_f64 || !out_u64 || d->out_format != FEK_OUT_SPLIT) return FEK_ERR_ARGUMENT;
  if (d->n_elements > 0 && (!d->stiffness || !d->load)) return FEK_ERR_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  double *pf = static_cast<double *>(partials);
  unsigned long long *pu = reinterpret_cast<unsigned long long *>(pf + 4 * kSumBlocks);
  const int ns = n_shape(d->element);
  if (d->dtype == FEK_F64) {
    checksum_partials<double><<<kSumBlocks, kSumThreads, 0, s>>>(
        static_cast<const double *>(d->stiffness), static_cast<const double *>(d->load), d->n_elements, ns * ns,
        ns, d->base_index, pf, pu);
  } else {
    checksum_partials<float><<<kSumBlocks, kSumThreads, 0, s>>>(
        static_cast<const float *>(d->stiffness), static_cast<const float *>(d->load), d->n_elements, ns * ns,
        ns, d->base_index, pf, pu);
  }
  checksum_final<<<1, 32, 0, s>>>(pf, pu, kSumBlocks, out_f64, out_u64);
  FEK_CUDA(cudaGetLastError());
  return FEK_OK;
}

// --------------------------------------------------------------------------
// host-buffer pipeline
// --------------------------------------------------------------------------

namespace {
struct SlotPlan {
  size_t geo, coef, A, b, slot;
};

size_t round256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }
// Chunk ci of the host pipeline, `rem` elements left, `chunk` the slot size.
// The first chunks ramp up (chunk/8, /4, /2) so the device-to-host engine
// starts early, and the last ones halve what is left down to chunk/8 so the
// final kernel + download (the only part nothing overlaps) is short.
// Multiples of `align` except the very last piece.
long long pipeline_chunk(long long ci, long long rem, long long chunk, long long align) {
  const long long floor_size = ((chunk / 8 + align - 1) / align) * align;
  long long size = ci < 3 ? (chunk >> (3 - ci)) : chunk;
  const long long half = (((rem + 1) / 2 + align - 1) / align) * align;
  if (half < size) size = half;
  if (size < floor_size) size = floor_size;
  size = ((size + align - 1) / align) * align;
  return size < rem ? size : rem;
}

// workspace header: the error word, then one [2]-word tile queue per stream slot
size_t host_header_bytes(int n_streams) { return round256(16 + 16 * static_cast<size_t>(n_streams)); }

SlotPlan slot_plan(const fek_batch_desc *d, long long chunk) {
  const size_t rb = real_bytes(d->dtype);
  const int ns = n_shape(d->element);
  SlotPlan p;
  p.geo = round256(chunk * geometry_size(d->element) * rb);
  p.coef = round256(chunk * coefficient_size(d->element, d->problem) * rb);
  p.A = round256(chunk * (ns * ns + ns) * rb);  // packed rows need ns*ns + ns per element
  p.b = round256(chunk * ns * rb);
  p.slot = p.geo + p.coef + p.A + p.b;
  return p;
}

long long flat_len(long long n, int ds, int w) { return n == 0 ? 0 : ((n + w - 1) / w) * w * ds; }
}  // namespace

// host pipeline chunks: multiples of 256 elements (every tile size, hence every lane width)
static constexpr long long kChunkAlign = 256;
static long long round_chunk(long long c) { return ((c + kChunkAlign - 1) / kChunkAlign) * kChunkAlign; }

size_t fek_host_workspace_bytes(const fek_batch_desc *d, int n_streams, int64_t chunk_elements) {
  if (!d || n_streams < 1 || chunk_elements < 1) return 0;
  return host_header_bytes(n_streams) + static_cast<size_t>(n_streams) * slot_plan(d, round_chunk(chunk_elements)).slot;
}

}  // extern "C"

namespace {
// Parallel host memcpy for the staged pipeline: `threads` workers created for one call, each
// copying a contiguous slice of every job (pageable <-> page-locked staging; one thread reaches
// ~15 GB/s, 8-16 threads 70-85 GB/s on the GPU box's host).
class CopyPool {
 public:
  explicit CopyPool(int threads) : n_(threads < 1 ? 1 : threads) {
    for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto &t : workers_) t.join();
  }
  // dst[0, bytes) = src[0, bytes), split across the pool; returns when done
  void copy(void *dst, const void *src, size_t bytes) {
    if (bytes < (4u << 20) || n_ == 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      dst_ = static_cast<char *>(dst);
      src_ = static_cast<const char *>(src);
      bytes_ = bytes;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    slice(0);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void slice(int i) {
    const size_t per = ((bytes_ + n_ - 1) / n_ + 63) & ~static_cast<size_t>(63);
    const size_t lo = per * i, hi = lo + per < bytes_ ? lo + per : bytes_;
    if (lo < hi) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void loop(int i) {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return quit_ || gen_ != seen; });
        if (quit_) return;
        seen = gen_;
      }
      slice(i);
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  bool quit_ = false;
  unsigned long long gen_ = 0;
  int pending_ = 0;
  char *dst_ = nullptr;
  const char *src_ = nullptr;
  size_t bytes_ = 0;
};

bool pageable(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // older drivers: unregistered host pointers report an error
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

struct StagePlan {
  size_t in, out, slot;
};
StagePlan stage_plan(const fek_batch_desc *d, long long chunk) {
  const size_t rb = real_bytes(d->dtype);
  const int ns = n_shape(d->element);
  StagePlan p;
  p.in = round256(chunk * (geometry_size(d->element) + coefficient_size(d->element, d->problem)) * rb);
  p.out = round256(chunk * (ns * ns + 2 * ns) * rb);  // split A + b, or packed rows (ns*ns + ns)
  p.slot = p.in + p.out;
  return p;
}

// Pageable inputs go through a ring of 3 pieces of up to 12 MiB at the start of the staging
// buffer (inside the host's last-level cache), each reused once the DMA after it completed.
// Sweep on the GPU box (C5, tools/e2e_pageable.py; 385 ms page-locked): chunk-sized slots
// 575 ms, rings of 4 MiB x 4 / 8 x 4 / 12 x 3 / 16 x 4 pieces 507 / 468 / 452 / 497 ms.
struct StageRing {
  int pieces = 0;
  size_t piece_bytes = 0;
};
StageRing stage_ring(const StagePlan &tp) {
  StageRing r;
  r.pieces = 3;
  r.piece_bytes = (tp.in / r.pieces) & ~static_cast<size_t>(255);
  if (r.piece_bytes > (12u << 20)) r.piece_bytes = 12u << 20;
  if (r.piece_bytes < (1u << 20)) r.pieces = 0;  // small batches: whole-slot staging
  return r;
}
// page-locked staging bytes the pipeline needs for d's pageable arrays: the input ring alone when
// only inputs are pageable, chunk-sized slots when outputs are (or the batch is too small for a
// ring), nothing when every array is page-locked
size_t staging_need(const fek_batch_desc *d, int n_streams, long long chunk, bool stage_in, bool stage_out) {
  const StagePlan tp = stage_plan(d, chunk);
  const StageRing ring = stage_ring(tp);
  if (stage_out || (stage_in && ring.pieces == 0)) return static_cast<size_t>(n_streams) * tp.slot;
  return stage_in ? ring.pieces * ring.piece_bytes : 0;
}

// The chunked H2D -> kernel -> D2H pipeline.  staging == nullptr: host buffers are DMA'd
// directly (page-locked buffers overlap; pageable ones serialise in the driver).  Otherwise
// every pageable array goes through the page-locked staging slots: the inputs of chunk i are
// copied in by the CopyPool while chunks i-1, i-2 are on the GPU, and staged outputs are copied
// out when their slot comes round again.
int host_pipeline(const fek_batch_desc *d, void *device_workspace, size_t workspace_bytes, int n_streams,
                  void *const *cuda_streams, int64_t chunk_elements, void *staging, size_t staging_bytes,
                  int copy_threads, unsigned long long *error_key_out) {
  if (int rc = validate(d, false)) return rc;
  if (n_streams < 1 || !cuda_streams || chunk_elements < 1 || !error_key_out) return FEK_ERR_ARGUMENT;
  const int w = d->layout == FEK_ELEMENT_MAJOR ? 1 : d->lane_width;
  // chunk boundaries on whole lane blocks and even element counts (fp32 rows)
  const long long align = kChunkAlign;
  long long chunk = round_chunk(chunk_elements);
  if (fek_host_workspace_bytes(d, n_streams, chunk) > workspace_bytes || !device_workspace)
    return FEK_ERR_WORKSPACE;
  if (!aligned16(device_workspace)) return FEK_ERR_ALIGNMENT;
  *error_key_out = FEK_NO_ERROR;
  const long long n = d->n_elements;
  if (n == 0) return FEK_OK;
  const bool packed = d->out_format == FEK_OUT_PACKED;
  if (!d->geometry || !d->coefficients || !d->stiffness || (!packed && !d->load)) return FEK_ERR_ARGUMENT;
  const StagePlan tp = stage_plan(d, chunk);
  const bool stage_in = staging && (pageable(d->geometry) || pageable(d->coefficients));
  const bool stage_out = staging && (pageable(d->stiffness) || (!packed && pageable(d->load)));
  if (staging && (staging_bytes < staging_need(d, n_streams, chunk, stage_in, stage_out) || !aligned16(staging)))
    return FEK_ERR_WORKSPACE;

  char *ws = static_cast<char *>(device_workspace);
  unsigned long long *dkey = reinterpret_cast<unsigned long long *>(ws);
  const SlotPlan sp = slot_plan(d, chunk);
  const size_t rb = real_bytes(d->dtype);
  const int dsg = geometry_size(d->element), dsc = coefficient_size(d->element, d->problem);
  const int ns = n_shape(d->element), dso = ns * ns + ns;
  cudaStream_t s0 = static_cast<cudaStream_t>(cuda_streams[0]);

  unsigned long long *queues = reinterpret_cast<unsigned long long *>(ws + 16);
  const size_t header = host_header_bytes(n_streams);

  // error word and tile queues initialised on stream 0; the other streams wait for it
  FEK_CUDA(cudaMemsetAsync(dkey, 0xFF, sizeof(unsigned long long), s0));
  FEK_CUDA(cudaMemsetAsync(queues, 0, 16 * static_cast<size_t>(n_streams), s0));
  cudaEvent_t ready;
  FEK_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  FEK_CUDA(cudaEventRecord(ready, s0));
  for (int i = 1; i < n_streams; ++i)
    FEK_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(cuda_streams[i]), ready, 0));
  std::vector<cudaEvent_t> slot_done(n_streams, nullptr);  // staged: the slot's last D2H finished
  std::vector<cudaEvent_t> in_free(n_streams, nullptr);    // staged: the slot's last H2D finished
  std::unique_ptr<CopyPool> pool;
  const StageRing ring = stage_ring(tp);
  const int ring_pieces = ring.pieces;
  const size_t piece_bytes = ring.piece_bytes;
  std::vector<cudaEvent_t> ring_ev(ring_pieces, nullptr);
  std::vector<char> ring_used(ring_pieces, 0);
  unsigned long long ring_next = 0;
  if (stage_in || stage_out) {
    for (auto &e : ring_ev) FEK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pool.reset(new CopyPool(copy_threads));
    for (auto &e : slot_done) FEK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : in_free) FEK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  struct Pending {
    long long lo = -1, cnt = 0;
  };
  std::vector<Pending> pending(n_streams);  // staged outputs waiting in each slot

  const char *hg = static_cast<const char *>(d->geometry);
  const char *hc = static_cast<const char *>(d->coefficients);
  char *hA = static_cast<char *>(d->stiffness);
  char *hb = static_cast<char *>(d->load);
  auto out_bytes = [&](long long cnt, size_t *a, size_t *b) {
    if (packed) {
      *a = flat_len(cnt, dso, d->out_lane_width) * rb;
      *b = 0;
    } else {
      *a = cnt * ns * ns * rb;
      *b = cnt * ns * rb;
    }
  };
  auto drain = [&](int slot) -> int {  // staged outputs of the slot's previous chunk -> caller arrays
    Pending &pd = pending[slot];
    if (pd.lo < 0) return FEK_OK;
    FEK_CUDA(cudaEventSynchronize(slot_done[slot]));
    const char *so = static_cast<const char *>(staging) + slot * tp.slot + tp.in;
    size_t ab, bb;
    out_bytes(pd.cnt, &ab, &bb);
    pool->copy(hA + pd.lo * (packed ? dso : ns * ns) * rb, so, ab);
    if (bb) pool->copy(hb + pd.lo * ns * rb, so + ab, bb);
    pd.lo = -1;
    return FEK_OK;
  };
  int rc = FEK_OK;
  long long ci = 0;
  long long cnt = 0;
  for (long long lo = 0; lo < n && rc == FEK_OK; lo += cnt, ++ci) {
    cnt = pipeline_chunk(ci, n - lo, chunk, align);
    const int slot = static_cast<int>(ci % n_streams);
    cudaStream_t st = static_cast<cudaStream_t>(cuda_streams[slot]);
    char *base = ws + header + slot * sp.slot;
    char *dg = base, *dc = base + sp.geo, *dA = dc + sp.coef, *db = dA + sp.A;
    // lo is a multiple of 256 (hence of W): the chunk's flat range starts at lo*DS
    const size_t gbytes = flat_len(cnt, dsg, w) * rb, cbytes = flat_len(cnt, dsc, w) * rb;
    const char *srcg = hg + lo * dsg * rb, *srcc = hc + lo * dsc * rb;
    if (pool && ci >= n_streams) {
      // the slot's previous chunk: staged outputs copied out, staged inputs consumed by its H2D
      if ((rc = drain(slot))) break;
      cudaError_t e = cudaEventSynchronize(in_free[slot]);
      if (e != cudaSuccess) {
        rc = cuda_fail(e, "cudaEventSynchronize");
        break;
      }
    }
    cudaError_t e = cudaSuccess;
    if (stage_in && ring_pieces) {
      // piecewise through a small ring that stays in the host's last-level cache: each piece
      // is copied (temporal stores) and DMA'd at once, so the copy engine reads it from cache
      auto put = [&](char *dst, const char *src, size_t bytes) {
        for (size_t off = 0; off < bytes && e == cudaSuccess; off += piece_bytes) {
          const size_t len = bytes - off < piece_bytes ? bytes - off : piece_bytes;
          const int r = static_cast<int>(ring_next++ % ring_pieces);
          if (ring_used[r]) e = cudaEventSynchronize(ring_ev[r]);
          if (e != cudaSuccess) break;
          char *piece = static_cast<char *>(staging) + r * piece_bytes;
          pool->copy(piece, src + off, len);
          e = cudaMemcpyAsync(dst + off, piece, len, cudaMemcpyHostToDevice, st);
          if (e == cudaSuccess) e = cudaEventRecord(ring_ev[r], st);
          ring_used[r] = 1;
        }
      };
      put(dg, srcg, gbytes);
      put(dc, srcc, cbytes);
    } else {
      if (pool && stage_in) {
        char *si = static_cast<char *>(staging) + slot * tp.slot;
        pool->copy(si, srcg, gbytes);
        pool->copy(si + gbytes, srcc, cbytes);
        srcg = si;
        srcc = si + gbytes;
      }
      e = cudaMemcpyAsync(dg, srcg, gbytes, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(dc, srcc, cbytes, cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess && pool) e = cudaEventRecord(in_free[slot], st);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "cudaMemcpyAsync H2D");
      break;
    }
    fek_batch_desc cd = *d;
    cd.n_elements = cnt;
    cd.base_index = d->base_index + lo;
    cd.geometry = dg;
    cd.coefficients = dc;
    cd.stiffness = dA;
    cd.load = db;
    cd.error_key = dkey;
    cd.scheduler = queues + 2 * slot;  // launches on one stream are ordered: one queue per slot
    rc = launch(&cd, st, nullptr, nullptr, nullptr, nullptr, true);
    if (rc) break;
    size_t ab, bb;
    out_bytes(cnt, &ab, &bb);
    char *dstA = hA + lo * (packed ? dso : ns * ns) * rb, *dstb = packed ? nullptr : hb + lo * ns * rb;
    if (stage_out) {
      dstA = static_cast<char *>(staging) + slot * tp.slot + tp.in;
      dstb = dstA + ab;
      pending[slot].lo = lo;
      pending[slot].cnt = cnt;
    }
    e = cudaMemcpyAsync(dstA, dA, ab, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && bb) e = cudaMemcpyAsync(dstb, db, bb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && pool) e = cudaEventRecord(slot_done[slot], st);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync D2H");
  }
  for (int i = 0; i < n_streams; ++i) {
    cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(cuda_streams[i]));
    if (e != cudaSuccess && rc == FEK_OK) rc = cuda_fail(e, "cudaStreamSynchronize");
  }
  if (rc == FEK_OK && stage_out)
    for (int i = 0; i < n_streams && rc == FEK_OK; ++i) rc = drain(i);
  pool.reset();
  for (auto &e : slot_done)
    if (e) cudaEventDestroy(e);
  for (auto &e : in_free)
    if (e) cudaEventDestroy(e);
  for (auto &e : ring_ev)
    if (e) cudaEventDestroy(e);
  cudaEventDestroy(ready);
  if (rc) return rc;
  FEK_CUDA(cudaMemcpy(error_key_out, dkey, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  if (*error_key_out != FEK_NO_ERROR && (*error_key_out & 127ull) == FEK_KIND_NEAR) {
    // an element within 16 tol of the degeneracy bound: re-classify the whole batch with
    // the reference's rounding, its geometry streamed once more through slot 0 (rare path)
    FEK_CUDA(cudaMemsetAsync(dkey, 0xFF, sizeof(unsigned long long), s0));
    char *dg = ws + header;
    for (long long lo = 0; lo < n; lo += chunk) {
      const long long cnt = n - lo < chunk ? n - lo : chunk;
      FEK_CUDA(cudaMemcpyAsync(dg, hg + lo * dsg * rb, flat_len(cnt, dsg, w) * rb, cudaMemcpyHostToDevice, s0));
      fek_batch_desc cd = *d;
      cd.n_elements = cnt;
      cd.base_index = d->base_index + lo;
      cd.geometry = dg;
      cd.error_key = dkey;
      if (int crc = classify_batch(&cd, s0)) return crc;
    }
    FEK_CUDA(cudaMemcpyAsync(error_key_out, dkey, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s0));
    FEK_CUDA(cudaStreamSynchronize(s0));
  }
  return *error_key_out == FEK_NO_ERROR ? FEK_OK : FEK_ERR_GEOMETRY;
}
}  // namespace

extern "C" {

int fek_integrate_host(const fek_batch_desc *d, void *device_workspace, size_t workspace_bytes, int n_streams,
                       void *const *cuda_streams, int64_t chunk_elements, unsigned long long *error_key_out) {
  return host_pipeline(d, device_workspace, workspace_bytes, n_streams, cuda_streams, chunk_elements, nullptr, 0, 0,
                       error_key_out);
}

size_t fek_host_staging_bytes(const fek_batch_desc *d, int n_streams, int64_t chunk_elements) {
  if (!d || n_streams < 1 || chunk_elements < 1) return 0;
  const bool packed = d->out_format == FEK_OUT_PACKED;
  const bool stage_in = (d->geometry && pageable(d->geometry)) || (d->coefficients && pageable(d->coefficients));
  const bool stage_out = (d->stiffness && pageable(d->stiffness)) || (!packed && d->load && pageable(d->load));
  return staging_need(d, n_streams, round_chunk(chunk_elements), stage_in, stage_out);
}

int fek_integrate_host_staged(const fek_batch_desc *d, void *device_workspace, size_t workspace_bytes, int n_streams,
                              void *const *cuda_streams, int64_t chunk_elements, void *host_staging,
                              size_t staging_bytes, int copy_threads, unsigned long long *error_key_out) {
  if (!host_staging) return FEK_ERR_ARGUMENT;
  return host_pipeline(d, device_workspace, workspace_bytes, n_streams, cuda_streams, chunk_elements, host_staging,
                       staging_bytes, copy_threads, error_key_out);
}

}  // extern "C"
