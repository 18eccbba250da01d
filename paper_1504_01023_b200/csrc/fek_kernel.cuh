// fek_kernel.cuh -- the persistent, TMA-pipelined integration kernel.
//
// One CTA = 128 threads = one tile of TILE = 128 elements at a time (one
// element per thread).  CTAs are persistent (grid = SMs x resident CTAs) and
// walk tiles t = blockIdx.x + k*gridDim.x.  Per tile:
//
//   1. the tile's geometry and coefficient byte ranges (contiguous in both
//      the element-major and the lane-interleaved layout, because TILE is a
//      multiple of every lane width) arrive by 1-D TMA bulk copies into stage
//      k % STAGES, completion counted on that stage's mbarrier;
//   2. each thread pulls its element's rows into registers (conflict-free
//      rotated 16-byte reads, fek_device.cuh) -- or, for the FP64-bound
//      prism path, only the coefficients, re-reading vertex coordinates from
//      the tile per quadrature point;
//   3. once the stage is consumed, thread 0 refills it with tile k+STAGES;
//   4. the element math runs in registers (fek_element.cuh);
//   5. A and b rows are written to one shared output tile (the exact global
//      byte image) and leave the SM as two TMA bulk stores, i.e. full-line
//      coalesced writes; the next tile waits for the store to have READ the
//      tile (bulk_wait_read) before overwriting it.
//
// Geometry failures are reduced to one 64-bit key per element and merged with
// a single atomicMin into the caller's error word.
#pragma once

#include "fek_element.cuh"

namespace fek {

struct LaunchParams {
  const void *geometry;
  const void *coefficients;
  void *stiffness;
  void *load;
  unsigned long long *error_key;
  long long n;
  long long base;
  int lane_width;
};

template <typename R_, int ET_, int PB_, int VAR_, int GEO_>
struct Traits {
  using R = R_;
  static constexpr int ET = ET_, PB = PB_, VAR = VAR_, GEO = GEO_;
  using S = Shape<ET>;
  static constexpr int NV = S::NV, NS = S::NS, NQ = S::NQ;
  static constexpr int DSG = 3 * NV;
  static constexpr int DSC = (PB == POISSON) ? NQ : 20;
  static constexpr int NA = NS * NS;
  static constexpr int THREADS = 128;
  static constexpr int TILE = 128;
  // prisms (and the re-computing generic variants) re-read coordinates from
  // the staged tile instead of pinning 18 reals in registers
  static constexpr bool LAZY_X = (GEO == GEO_GENERIC) && (ET == PRISM || VAR != QSS);
  // stages / resident CTAs: memory-bound tets keep >= 64 KB of loads in
  // flight per SM; prisms trade stages for resident warps (FP64 latency)
  static constexpr int STAGES = (ET == TET && PB == POISSON) ? 3 : (LAZY_X && PB == CONV_DIFF ? 1 : 2);
  static constexpr int MIN_BLOCKS = (ET == TET && PB == POISSON) ? 3 : 2;
  static constexpr unsigned GEO_TILE_BYTES = TILE * DSG * sizeof(R);
  static constexpr unsigned COEF_TILE_BYTES = TILE * DSC * sizeof(R);
  static constexpr unsigned STAGE_BYTES = GEO_TILE_BYTES + COEF_TILE_BYTES;
  static constexpr unsigned OUT_A_BYTES = TILE * NA * sizeof(R);
  static constexpr unsigned OUT_B_BYTES = TILE * NS * sizeof(R);
  static constexpr unsigned BAR_OFFSET = STAGES * STAGE_BYTES + OUT_A_BYTES + OUT_B_BYTES;
  static constexpr unsigned SMEM_BYTES = BAR_OFFSET + 8 * STAGES;
  static_assert(GEO_TILE_BYTES % 16 == 0 && COEF_TILE_BYTES % 16 == 0, "tile alignment");
  static_assert(OUT_A_BYTES % 16 == 0 && OUT_B_BYTES % 16 == 0, "tile alignment");
};

// bytes of `count` elements starting at tile origin, padded to the layout's
// lane block (interleaved tails are padded in the source array too)
__device__ __forceinline__ unsigned tile_bytes(int count, int w, int ds, int real_bytes) {
  const int padded = ((count + w - 1) / w) * w;
  return static_cast<unsigned>(padded * ds * real_bytes);
}

// At most 15 trailing bytes of a row range that bulk copies cannot move
// (fp32 rows of 72/24 bytes with an odd element count): plain loads/stores.
__device__ __forceinline__ void copy_tail(uint32_t dst, const char *src, unsigned bytes) {
  for (unsigned i = bytes & ~15u; i < bytes; i += 4) sts32(dst + i, *reinterpret_cast<const uint32_t *>(src + i));
}

template <class K>
__device__ __forceinline__ void issue_tile(const LaunchParams &p, long long t, uint32_t geo_dst, uint32_t coef_dst,
                                           uint32_t bar, uint64_t policy) {
  using R = typename K::R;
  const long long e0 = t * K::TILE;
  const int count = static_cast<int>(min(static_cast<long long>(K::TILE), p.n - e0));
  const unsigned gb = tile_bytes(count, p.lane_width, K::DSG, sizeof(R));
  const unsigned cb = tile_bytes(count, p.lane_width, K::DSC, sizeof(R));
  const char *gsrc = static_cast<const char *>(p.geometry) + e0 * K::DSG * sizeof(R);
  const char *csrc = static_cast<const char *>(p.coefficients) + e0 * K::DSC * sizeof(R);
  // sub-16-byte tails first (plain stores, ordered before the arrive's
  // release), then arm the barrier with the bulk byte count, then the bulk
  // copies: the phase completes when the arrival and all bytes are in
  copy_tail(geo_dst, gsrc, gb);
  copy_tail(coef_dst, csrc, cb);
  mbar_arrive_expect_tx(bar, (gb & ~15u) + (cb & ~15u));
  if (gb & ~15u) bulk_load(geo_dst, gsrc, gb & ~15u, bar, policy);
  if (cb & ~15u) bulk_load(coef_dst, csrc, cb & ~15u, bar, policy);
}

template <class K>
__global__ void __launch_bounds__(K::THREADS, K::MIN_BLOCKS) integrate_kernel(const LaunchParams p) {
  using R = typename K::R;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x;
  const long long tiles = (p.n + K::TILE - 1) / K::TILE;
  const uint32_t bars = sbase + K::BAR_OFFSET;
  const uint32_t out_a = sbase + K::STAGES * K::STAGE_BYTES;
  const uint32_t out_b = out_a + K::OUT_A_BYTES;
  auto geo_stage = [&](int s) { return sbase + s * K::STAGE_BYTES; };
  auto coef_stage = [&](int s) { return sbase + s * K::STAGE_BYTES + K::GEO_TILE_BYTES; };

  uint64_t policy = 0;
  if (tid == 0) {
    policy = policy_evict_first();
    for (int s = 0; s < K::STAGES; ++s) mbar_init(bars + 8 * s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < K::STAGES; ++s) {
      const long long t = blockIdx.x + static_cast<long long>(s) * gridDim.x;
      if (t < tiles) issue_tile<K>(p, t, geo_stage(s), coef_stage(s), bars + 8 * s, policy);
    }
  }

  int k = 0;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
    const int s = k % K::STAGES;
    const uint32_t parity = (k / K::STAGES) & 1;
    const bool landed = mbar_wait(bars + 8 * s, parity);
    if (__syncthreads_or(!landed)) {  // uniform bail-out instead of a hang
      if (tid == 0) atomicMin(p.error_key, static_cast<unsigned long long>(KIND_PIPELINE_TIMEOUT));
      return;
    }
    const long long e0 = t * K::TILE;
    const int count = static_cast<int>(min(static_cast<long long>(K::TILE), p.n - e0));
    const bool active = tid < count;
    const long long e_abs = p.base + e0 + tid;

    R C[K::DSC];
    R A[K::NA];
    R B[K::NS];
    int kind = 0, kind_point = -1;
    if constexpr (!K::LAZY_X) {
      R X[K::DSG];
      if (active) {
        RowIO<R, K::DSG>::load(geo_stage(s), tid, p.lane_width, X);
        RowIO<R, K::DSC>::load(coef_stage(s), tid, p.lane_width, C);
      }
      __syncthreads();  // stage s consumed by every thread
      if (tid == 0) {
        const long long tn = t + static_cast<long long>(K::STAGES) * gridDim.x;
        if (tn < tiles) issue_tile<K>(p, tn, geo_stage(s), coef_stage(s), bars + 8 * s, policy);
      }
      if (active) {
        if constexpr (K::GEO == GEO_LINEAR) {
          integrate_tet_linear<R, K::PB>(X, C, A, B, kind);
        } else {
          const R tol = degeneracy_tolerance<R, K::NV>(X);
          integrate_generic<R, K::ET, K::PB, K::VAR>(RegGeometry<R, K::DSG>{X}, C, tol, A, B, kind, kind_point);
        }
      }
    } else {
      if (active) {
        RowIO<R, K::DSC>::load(coef_stage(s), tid, p.lane_width, C);
        const SmemGeometry<R, K::DSG> geo{geo_stage(s), tid, p.lane_width};
        R X[K::DSG];
        geo.fetch(X);
        const R tol = degeneracy_tolerance<R, K::NV>(X);
        integrate_generic<R, K::ET, K::PB, K::VAR>(geo, C, tol, A, B, kind, kind_point);
      }
      __syncthreads();  // stage s consumed
      if (tid == 0) {
        const long long tn = t + static_cast<long long>(K::STAGES) * gridDim.x;
        if (tn < tiles) issue_tile<K>(p, tn, geo_stage(s), coef_stage(s), bars + 8 * s, policy);
      }
    }
    if (kind) atomicMin(p.error_key, make_error_key(e_abs, kind_point, kind));

    if (tid == 0) bulk_wait_read<0>();  // previous tile's stores have read the out tile
    __syncthreads();
    if (active) {
      RowIO<R, K::NA>::store_major(out_a, tid, A);
      RowIO<R, K::NS>::store_major(out_b, tid, B);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const unsigned ab = count * K::NA * sizeof(R);
      const unsigned bb = count * K::NS * sizeof(R);
      char *ga = static_cast<char *>(p.stiffness) + e0 * K::NA * sizeof(R);
      char *gb = static_cast<char *>(p.load) + e0 * K::NS * sizeof(R);
      const unsigned ab16 = ab & ~15u, bb16 = bb & ~15u;
      if (ab16) bulk_store(ga, out_a, ab16);
      if (bb16) bulk_store(gb, out_b, bb16);
      bulk_commit();
      // fp32 prism load rows (24 B) with an odd count leave an 8-byte tail
      for (unsigned i = ab16; i < ab; i += 4) *reinterpret_cast<uint32_t *>(ga + i) = lds32(out_a + i);
      for (unsigned i = bb16; i < bb; i += 4) *reinterpret_cast<uint32_t *>(gb + i) = lds32(out_b + i);
    }
  }
  if (tid == 0) bulk_wait_all<0>();
}

// ---------------------------------------------------------------------------
// error detail (message formatting only): det and tol of one element/point
// ---------------------------------------------------------------------------

template <typename R, int ET>
__global__ void error_detail_kernel(const void *geometry, long long element, int lane_width, int point,
                                    double *out) {
  constexpr int NV = Shape<ET>::NV, DS = 3 * NV;
  const R *g = static_cast<const R *>(geometry);
  R X[DS];
  const long long blk = element / lane_width, lane = element % lane_width;
  for (int d = 0; d < DS; ++d) X[d] = g[blk * lane_width * DS + d * lane_width + lane];
  const R tol = degeneracy_tolerance<R, NV>(X);
  R det = R(0);
  if (point < 0) {
    R J[3][3];
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) J[i][k] = X[3 * (k + 1) + i] - X[i];
    det = invert3(J).det;
  } else {
    static_for<Shape<ET>::NQ>([&](auto qc) {
      constexpr int Q = decltype(qc)::value;
      if (Q == point) {
        R J[3][3];
        point_jacobian<ET, Q>(X, J);
        det = invert3(J).det;
      }
    });
  }
  out[0] = static_cast<double>(det);
  out[1] = static_cast<double>(tol);
}

}  // namespace fek
