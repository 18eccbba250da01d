// fek_kernel.cuh -- the persistent, TMA-pipelined integration kernel.
//
// One CTA = 128 threads (4 warps) = one tile of TILE = 128 elements at a
// time, one element per thread -- except the fp64 prism ConvDiff kernel, which
// runs each element on a lane pair (one zeta level per lane, fek_element.cuh
// prism_pair) with 64-element tiles.  CTAs are persistent (grid = SMs x
// resident CTAs) and take tiles from a device queue (atomicAdd; static
// round-robin t = blockIdx.x + i*gridDim.x without one).  Per tile i:
//
//   1. the tile's geometry and coefficient byte ranges (contiguous in both
//      the element-major and the lane-interleaved layout, because TILE is a
//      multiple of every lane width) arrive by 1-D TMA bulk copies into stage
//      i % STAGES; completion is counted on full[stage] (arrival + bytes);
//   2. each thread pulls its element's rows into registers (conflict-free
//      16-byte reads, fek_device.cuh); the QSS prism kernels read the
//      coefficient row and form their distinct Jacobian entries from the
//      staged coordinates (their prologue);
//   3. once every thread is done with the stage -- the tile's ONLY CTA
//      barrier -- thread 0 refills it with tile i + STAGES (for the fp64 QSS
//      prism kernels right after the prologue, so the refill overlaps the
//      math).  Before that barrier every warp's lane 0 has waited until its
//      own bulk stores of tile i - 1 have read the output tile, so the
//      barrier frees the output tile as well;
//   4. the element math runs in registers (fek_element.cuh);
//   5. each warp writes its A and b rows into one shared output tile (the
//      exact global byte image); the LAST warp to finish (shared-memory
//      arrival counter) sends the tile out as two TMA bulk stores (full-line
//      coalesced writes) -- nobody waits for the slowest warp.
//
// A warp-decoupled variant (per-warp mbarrier release + per-warp output
// slices) was measured slower on every case -- up to 12% on the FP64-bound
// prism kernel, whose unrolled SASS thrashes the instruction cache once warps
// drift apart; per-warp output stores alone lost too, and direct global stores
// of the rows far more.  Geometry failures become one
// 64-bit key per element, merged with atomicMin into the caller's error word.
// With a consumer MODE (fek_apply / fek_assemble) step 5 is replaced by the matrix-free scatter
// or the CSR assembly scatter: A and b never leave the registers.
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
  int out_packed;  // FEK_OUT_PACKED: rows [A | b] into `stiffness` in the output layout
  int out_width;   // output lane width (1 = element-major rows)
  unsigned long long *scheduler;  // [next tile, CTAs done] or null (static round-robin)
  // consumers (Traits MODE): fek_apply  y[node] += A_e x_e,  fek_assemble  values[csr(i, j)] += A_e;
  // both  f[node] += b_e
  const int *element_nodes;  // (n, NS) int32, element-major
  const void *x;             // apply: the vector
  void *y;                   // apply: the result / assemble: the CSR values
  void *f;                   // may be null
  const int *row_ptr;        // assemble: CSR row pointers (n_nodes + 1)
  const int *col;            // assemble: CSR column indices, sorted within each row
};

enum : int { MODE_STORE = 0, MODE_APPLY = 1, MODE_ASSEMBLE = 2 };

// position of column j in CSR row i (the caller's pattern holds every element's node pairs)
__device__ __forceinline__ int csr_find(const LaunchParams &p, int i, int j) {
  int lo = __ldg(p.row_ptr + i), hi = __ldg(p.row_ptr + i + 1);
  if (hi <= lo) return -1;  // empty row
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(p.col + mid) <= j) {
      lo = mid;
    } else {
      hi = mid;
    }
  }
  return __ldg(p.col + lo) == j ? lo : -1;  // -1: (i, j) is not in the pattern
}

// values[csr(nodes[r], nodes[s])] += A[r][s] and f[nodes[r]] += b[r] for ROWS rows of one element
// starting at R0 (A_rows: those rows, NS columns each): fp atomicAdd
template <typename R, int NS, int ROWS>
__device__ __forceinline__ void assemble_rows(const LaunchParams &p, long long e_local, int r0, const R *A_rows,
                                              const R *B_rows) {
  const int *nd = p.element_nodes + e_local * NS;
  int node[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) node[s] = __ldg(nd + s);
  R *values = static_cast<R *>(p.y);
  R *f = static_cast<R *>(p.f);
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const int i = node[r0 + r];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int k = csr_find(p, i, node[s]);
      if (k >= 0) {
        atomicAdd(values + k, A_rows[NS * r + s]);
      } else {  // a pattern that misses this element's pair: reported, never written elsewhere
        atomicMin(p.error_key, make_error_key(p.base + e_local, -1, KIND_PATTERN));  // by element alone
      }
    }
    if (f) atomicAdd(f + i, B_rows[r]);
  }
}

// y[nodes[r]] += sum_s A[r][s] x[nodes[s]] for rows r of one element (RB rows starting at R0 of
// its A; A_rows holds those rows, NS columns each), f[nodes[r]] += B_rows[r]: fp atomicAdd
template <typename R, int NS, int ROWS>
__device__ __forceinline__ void apply_rows(const LaunchParams &p, long long e_local, int r0, const R *A_rows,
                                           const R *B_rows) {
  const int *nd = p.element_nodes + e_local * NS;
  int node[NS];
  R xs[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) node[s] = __ldg(nd + s);
#pragma unroll
  for (int s = 0; s < NS; ++s) xs[s] = __ldg(static_cast<const R *>(p.x) + node[s]);
  R *y = static_cast<R *>(p.y);
  R *f = static_cast<R *>(p.f);
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    R acc = A_rows[NS * r] * xs[0];
#pragma unroll
    for (int s = 1; s < NS; ++s) acc = fma(A_rows[NS * r + s], xs[s], acc);
    atomicAdd(y + node[r0 + r], acc);
    if (f) atomicAdd(f + node[r0 + r], B_rows[r]);
  }
}

// TILE_ = 0: the kernel's own tile; 64 / 128 / 256: the tuner's tile-size variants (fek_dispatch.cuh)
template <typename R_, int ET_, int PB_, int VAR_, int GEO_, int TILE_ = 0, int MODE_ = MODE_STORE>
struct Traits {
  using R = R_;
  static constexpr int ET = ET_, PB = PB_, VAR = VAR_, GEO = GEO_;
  using S = Shape<ET>;
  static constexpr int NV = S::NV, NS = S::NS, NQ = S::NQ;
  static constexpr int DSG = 3 * NV;
  static constexpr int DSC = (PB == POISSON) ? NQ : 20;
  static constexpr int NA = NS * NS;
  // fp64 prism ConvDiff (QSS, reference frame): each element on a lane pair, one zeta level per
  // lane (fek_element.cuh prism_pair; FEK_PRISM_PAIR=0 builds the one-thread kernel instead)
#ifndef FEK_PRISM_PAIR
#define FEK_PRISM_PAIR 1
#endif
#ifndef FEK_PAIR_TILE
#define FEK_PAIR_TILE 64
#endif
  static constexpr bool PAIR = FEK_PRISM_PAIR && ET == PRISM && PB == CONV_DIFF && GEO == GEO_GENERIC &&
                               VAR == QSS && sizeof(R) == 8;
  static constexpr int NATURAL_TILE = PAIR ? FEK_PAIR_TILE : 128;
  static constexpr int TILE = TILE_ ? TILE_ : NATURAL_TILE;  // elements per tile (a multiple of every lane width)
  // consumers (fused matrix-free apply, CSR assembly): A and b stay in registers, no output tile
  static constexpr int MODE = MODE_;
  static constexpr bool APPLY = MODE != MODE_STORE;
  static_assert(TILE % 64 == 0, "a tile must be a whole number of lane blocks for every lane width");
  static constexpr int LANES = PAIR ? 2 : 1;
  static constexpr int THREADS = TILE * LANES;
  // prisms (and the re-computing generic variants) re-read coordinates from
  // the staged tile instead of pinning 18 reals in registers
  static constexpr bool LAZY_X = (GEO == GEO_GENERIC) && (ET == PRISM || VAR != QSS);
  // reference-frame prism kernels (fek_element.cuh integrate_prism_qss): the
  // staged tile is only read by the prologue (C row, distinct Jacobian columns)
  static constexpr bool PRISM_REF = (ET == PRISM && GEO == GEO_GENERIC && VAR == QSS);
  // fp64: release the input stage after the prologue, so the refill's loads
  // overlap this tile's math (C4 2.175 -> 2.070 ms, C3 -1%; fp32 prism CDR,
  // with two stages, is 1% slower this way)
  static constexpr bool EARLY_RELEASE = PRISM_REF && sizeof(R) == 8;
  // fp32 prism Poisson (reference frame, 111 registers): 4 CTAs x 2 stages, C3 fp32 0.169 ms vs
  // 0.191 (3 x 1), 0.175 (early release, 3 or 4 CTAs); fp64 prism Poisson at 2 CTAs x 2 stages
  // (244 registers, no spill) is 4% slower than 3 x 1 with early release
  static constexpr bool P32 = (sizeof(R) == 4 && ET == PRISM && PB == POISSON && PRISM_REF);
  // stages / resident CTAs: memory-bound tets keep >= 64 KB of loads in
  // flight per SM; the prism kernels spend shared memory on resident warps
  // (latency hiding for the FP64 pipe) rather than on a second stage
  // prism Poisson: 3 resident CTAs (12 warps, <= 170 registers, one stage)
  // beat 2 CTAs with two stages by 4% (C3 0.428 vs 0.445 ms, same-session A/B)
  static constexpr bool PRISM_P = (ET == PRISM && PB == POISSON);
  // fp32 prism CDR (168 registers, half the smem) fits 3 CTAs with 2 stages
  static constexpr bool F32_PRISM_CD = (sizeof(R) == 4 && ET == PRISM && PB == CONV_DIFF);
  static constexpr int STAGES_ = F32_PRISM_CD ? 2 :
      ((PRISM_P || (LAZY_X && PB == CONV_DIFF)) ? 1 : ((ET == TET && PB == POISSON) ? 3 : 2));
  static constexpr int MIN_BLOCKS_ = (F32_PRISM_CD || PRISM_P || (ET == TET && PB == POISSON)) ? 3 : 2;
  // (PAIR: 2 CTAs x 256 threads = 16 warps/SM at <= 128 registers)
#ifndef FEK_PAIR_STAGES
#define FEK_PAIR_STAGES 1
#endif
#ifndef FEK_PAIR_CTAS
#define FEK_PAIR_CTAS 4
#endif
  static constexpr int STAGES = P32 ? 2 : (PAIR ? FEK_PAIR_STAGES : STAGES_);
  // resident CTAs scale with the tile so the register budget per thread stays the natural one
  static constexpr int MIN_BLOCKS_N = P32 ? 4 : (PAIR ? FEK_PAIR_CTAS * 64 / NATURAL_TILE : MIN_BLOCKS_);
  static constexpr int MIN_BLOCKS = (MIN_BLOCKS_N * NATURAL_TILE / TILE) > 0 ? (MIN_BLOCKS_N * NATURAL_TILE / TILE) : 1;
  static constexpr unsigned GEO_TILE_BYTES = TILE * DSG * sizeof(R);
  static constexpr unsigned COEF_TILE_BYTES = TILE * DSC * sizeof(R);
  static constexpr unsigned OUT_A_BYTES = APPLY ? 0u : TILE * NA * sizeof(R);
  static constexpr unsigned OUT_B_BYTES = APPLY ? 0u : TILE * NS * sizeof(R);
  static constexpr unsigned GEO_OFFSET = 0;
  static constexpr unsigned COEF_OFFSET = STAGES * GEO_TILE_BYTES;
  static constexpr unsigned OUT_A_OFFSET = COEF_OFFSET + STAGES * COEF_TILE_BYTES;
  static constexpr unsigned OUT_B_OFFSET = OUT_A_OFFSET + OUT_A_BYTES;
  static constexpr unsigned BAR_OFFSET = OUT_B_OFFSET + OUT_B_BYTES;
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
struct Pipe {
  using R = typename K::R;
  uint32_t sbase;
  long long tiles;
  uint64_t policy;

  __device__ __forceinline__ uint32_t geo(int s) const { return sbase + K::GEO_OFFSET + s * K::GEO_TILE_BYTES; }
  __device__ __forceinline__ uint32_t coef(int s) const { return sbase + K::COEF_OFFSET + s * K::COEF_TILE_BYTES; }
  __device__ __forceinline__ uint32_t full(int s) const { return sbase + K::BAR_OFFSET + 8 * s; }

  // thread 0: stage tile t into stage s.  Sub-16-byte tails first (plain
  // stores, ordered before the arrive's release), then arm the barrier with
  // the bulk byte count, then the bulk copies: the phase completes when the
  // arrival and all transaction bytes are in.
  __device__ __forceinline__ void issue(const LaunchParams &p, long long t, int s) const {
    if (t >= tiles) return;
    const long long e0 = t * K::TILE;
    const int count = static_cast<int>(min(static_cast<long long>(K::TILE), p.n - e0));
    const unsigned gb = tile_bytes(count, p.lane_width, K::DSG, sizeof(R));
    const unsigned cb = tile_bytes(count, p.lane_width, K::DSC, sizeof(R));
    const char *gsrc = static_cast<const char *>(p.geometry) + e0 * K::DSG * sizeof(R);
    const char *csrc = static_cast<const char *>(p.coefficients) + e0 * K::DSC * sizeof(R);
    copy_tail(geo(s), gsrc, gb);
    copy_tail(coef(s), csrc, cb);
    mbar_arrive_expect_tx(full(s), (gb & ~15u) + (cb & ~15u));
    if (gb & ~15u) bulk_load(geo(s), gsrc, gb & ~15u, full(s), policy);
    if (cb & ~15u) bulk_load(coef(s), csrc, cb & ~15u, full(s), policy);
  }

};

template <class K>
__global__ void __launch_bounds__(K::THREADS, K::MIN_BLOCKS) integrate_kernel(const LaunchParams p) {
  using R = typename K::R;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  Pipe<K> pipe;
  pipe.sbase = smem_u32(smem);
  pipe.tiles = (p.n + K::TILE - 1) / K::TILE;
  pipe.policy = 0;
  const uint32_t out_a = pipe.sbase + K::OUT_A_OFFSET;
  const uint32_t out_b = pipe.sbase + K::OUT_B_OFFSET;
  if (tid == 0) {
    pipe.policy = policy_evict_first();
    for (int s = 0; s < K::STAGES; ++s) mbar_init(pipe.full(s), 1);
    fence_mbar_init();
  }
  __syncthreads();
  // Tile sources: static round-robin (blockIdx.x + i*gridDim.x), or a dynamic
  // queue (atomicAdd on scheduler[0]) so CTAs that start late -- e.g. while
  // another launch holds part of the SM -- simply take fewer tiles.  Thread 0
  // records each stage's tile in smem before arriving on the stage barrier, so
  // consumers read it after the wait; tiles past the end arrive without bytes.
  __shared__ long long s_tile[K::STAGES];
  __shared__ unsigned s_out_done;  // warps done writing the output tile (the last one stores it)
  if (tid == 0) s_out_done = 0;
  long long static_next = blockIdx.x;
  auto issue_stage = [&](int s) {
    long long t;
    if (p.scheduler) {
      t = static_cast<long long>(atomicAdd(p.scheduler, 1ull));
    } else {
      t = static_next;
      static_next += gridDim.x;
    }
    s_tile[s] = t;
    if (t < pipe.tiles) {
      pipe.issue(p, t, s);
    } else {
      mbar_arrive(pipe.full(s));
    }
  };
  if (tid == 0)
    for (int s = 0; s < K::STAGES; ++s) issue_stage(s);

  for (int i = 0;; ++i) {
    const int s = i % K::STAGES;
    const bool landed = mbar_wait(pipe.full(s), (i / K::STAGES) & 1);
    // tiles are taken in increasing order per CTA, so the first stage past the
    // end means every later stage is past the end too (nothing in flight)
    const long long t = *static_cast<volatile long long *>(&s_tile[s]);
    // the end-of-work / timeout test rides on the stage-release barrier below
    // (one CTA barrier fewer per tile: C4 -1.3%, C4 fp32 -0.8%); a thread that
    // timed out may see a stale tile here, which only feeds discarded work
    // before that barrier.  A timeout is fatal: bulk loads of the other stages
    // may still be in flight into this CTA's shared memory, so leaving would let
    // them land in a co-resident CTA's; the key is recorded, then the kernel traps.
    const bool stop = !landed || t >= pipe.tiles;
    // The stage-release barrier is the tile's only CTA barrier.  Before it, every warp's lane 0
    // waits until its own bulk stores of the previous tile have read the output tile (the last
    // warp to finish a tile issues its store, below), so after it the output tile is free too.
    auto release = [&]() -> bool {
      if ((tid & 31) == 0) bulk_wait_read<0>();
      if (__syncthreads_or(stop)) {
        if (!landed) {
          atomicMin(p.error_key, static_cast<unsigned long long>(KIND_PIPELINE_TIMEOUT));
          __threadfence_system();
          __trap();
        }
        return false;
      }
      if (tid == 0) issue_stage(s);
      return true;
    };
    const long long e0 = t * K::TILE;
    const int count = static_cast<int>(min(static_cast<long long>(K::TILE), p.n - e0));
    if constexpr (K::PAIR) {
      // element el on lanes (2 el, 2 el + 1), lane z = zeta level (fek_element.cuh prism_pair).
      // Every thread runs the math, also past `count` (on stale stage data, results dropped), so
      // both lanes of a pair always meet at the shuffles.
      const int el = tid >> 1, z = tid & 1;
      const bool act = !stop && el < count;
      R Ah[18], Bh[3];
      int kind = 0, kind_point = -1;
      {
        R C[20], J2[3][3], J01[3][2], bound;
        RowIO<R, 20>::load_paired(pipe.coef(s), el, p.lane_width, C);
        {
          R X[18];
          RowIO<R, 18>::load_paired(pipe.geo(s), el, p.lane_width, X);
          prism_pair::level_geometry(X, z, bound, J2, J01);
        }
        // (release() also frees the output tile: C4 2.020 -> 2.004 ms for that merge; per-warp
        // output stores measured slower, 2.028 ms)
        if (!release()) break;
        prism_pair::integrate_cd_level(J2, J01, C, bound, z, Ah, Bh, kind, kind_point);
      }
      if (act && z == 0 && kind) atomicMin(p.error_key, make_error_key(p.base + e0 + el, kind_point, kind));
      if constexpr (K::MODE == MODE_APPLY) {
        if (act) apply_rows<R, 6, 3>(p, e0 + el, 3 * z, Ah, Bh);  // lane z: rows a + 3z
        continue;
      } else if constexpr (K::MODE == MODE_ASSEMBLE) {
        if (act) assemble_rows<R, 6, 3>(p, e0 + el, 3 * z, Ah, Bh);
        continue;
      }
      constexpr unsigned RB = sizeof(R);
      if (p.out_packed) {
        constexpr int DSO = 42;
        const int w = p.out_width;
        const int padded = ((count + w - 1) / w) * w;
        if (el < padded) {
          const R nan = R(__longlong_as_double(0x7ff8000000000000ll));
          if (w == 1) {
            const uint32_t row = out_a + static_cast<uint32_t>(el) * DSO * RB;
#pragma unroll
            for (int c = 0; c < 9; ++c)
              sts128(row + 144u * z + 16u * c, pack2(act ? Ah[2 * c] : nan, act ? Ah[2 * c + 1] : nan));
#pragma unroll
            for (int j = 0; j < 3; ++j) sts64(row + 288u + 24u * z + 8u * j, pack1(act ? Bh[j] : nan));
          } else {
            const uint32_t base = out_a + static_cast<uint32_t>((el / w) * w * DSO + (el % w)) * RB;
            const uint32_t stride = static_cast<uint32_t>(w) * RB;
#pragma unroll
            for (int j = 0; j < 18; ++j) sts64(base + (18u * z + j) * stride, pack1(act ? Ah[j] : nan));
#pragma unroll
            for (int j = 0; j < 3; ++j) sts64(base + (36u + 3u * z + j) * stride, pack1(act ? Bh[j] : nan));
          }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
          bulk_store(static_cast<char *>(p.stiffness) + e0 * DSO * RB, out_a, padded * DSO * RB);  // 336-B rows
          bulk_commit();
        }
        continue;
      }
      if (act) {
        // rows a + 3z of the element's 6x6 block (144 contiguous bytes): lanes 0..7 of a phase hit
        // 16-byte bank groups (18 el + 9 z + c) mod 8, all distinct
        const uint32_t row = out_a + static_cast<uint32_t>(el) * 36u * RB + 144u * z;
#pragma unroll
        for (int c = 0; c < 9; ++c) sts128(row + 16u * c, pack2(Ah[2 * c], Ah[2 * c + 1]));
#pragma unroll
        for (int j = 0; j < 3; ++j) sts64(out_b + static_cast<uint32_t>(el) * 6u * RB + 24u * z + 8u * j, pack1(Bh[j]));
      }
      // no CTA barrier: the last warp to finish its rows stores the whole tile (one bulk store
      // pair per tile, as before, without the others waiting for the slowest warp)
      fence_proxy_async_smem();
      __syncwarp();
      if ((tid & 31) == 0) {
        __threadfence_block();
        if (atomicAdd(&s_out_done, 1u) == K::THREADS / 32 - 1) {
          __threadfence_block();
          s_out_done = 0;  // next tile's arrivals come after the next release barrier
          // fp64 rows of 288 / 48 bytes: multiples of 16
          bulk_store(static_cast<char *>(p.stiffness) + e0 * K::NA * RB, out_a, count * K::NA * RB);
          bulk_store(static_cast<char *>(p.load) + e0 * K::NS * RB, out_b, count * K::NS * RB);
          bulk_commit();
        }
      }
      continue;
    }
    const bool active = !stop && tid < count;
    const long long e_abs = p.base + e0 + tid;
    R C[K::DSC];
    R A[K::NA];
    R B[K::NS];
    int kind = 0, kind_point = -1;
    if constexpr (K::EARLY_RELEASE) {
      // prologue from the staged tile, release the stage, then the math
      // overlaps the refill's loads
      prism_ref::Cols<R> cols;
      R bound;
      if (active) {
        RowIO<R, K::DSC>::load(pipe.coef(s), tid, p.lane_width, C);
        R X[K::DSG];
        RowIO<R, K::DSG>::load(pipe.geo(s), tid, p.lane_width, X);
        bound = near_bound<R, K::NV>(X);
        prism_ref::jacobian_columns(X, cols.J2, cols.J01);
      }
      if (!release()) break;
      if (active) integrate_prism_qss<R, K::PB>(cols, C, bound, A, B, kind, kind_point);
    } else if constexpr (!K::LAZY_X) {
      R X[K::DSG];
      if (active) {
        RowIO<R, K::DSG>::load(pipe.geo(s), tid, p.lane_width, X);
        RowIO<R, K::DSC>::load(pipe.coef(s), tid, p.lane_width, C);
      }
      if (!release()) break;
      if (active) {
        if constexpr (K::GEO == GEO_LINEAR) {
          integrate_tet_linear<R, K::PB>(X, C, A, B, kind);
        } else {
          const R bound = near_bound<R, K::NV>(X);
          integrate_generic<R, K::ET, K::PB, K::VAR>(RegGeometry<R, K::DSG>{X}, C, RegLoad<R>{C + (K::DSC >= 20 ? 16 : 0)},
                                                     bound, A, B, kind, kind_point);
        }
      }
    } else {
      if (active) {
        RowIO<R, K::DSC>::load(pipe.coef(s), tid, p.lane_width, C);
        const SmemGeometry<R, K::DSG> geo{pipe.geo(s), tid, p.lane_width};
        R X[K::DSG];
        geo.fetch(X);
        const R bound = near_bound<R, K::NV>(X);
        integrate_generic<R, K::ET, K::PB, K::VAR>(geo, C, RegLoad<R>{C + (K::DSC >= 20 ? 16 : 0)}, bound, A, B, kind,
                                                   kind_point);
      }
      if (!release()) break;
    }
    if (kind) atomicMin(p.error_key, make_error_key(e_abs, kind_point, kind));
    if constexpr (K::MODE == MODE_APPLY) {
      if (active) apply_rows<R, K::NS, K::NS>(p, e0 + tid, 0, A, B);
      continue;
    } else if constexpr (K::MODE == MODE_ASSEMBLE) {
      if (active) assemble_rows<R, K::NS, K::NS>(p, e0 + tid, 0, A, B);
      continue;
    }
    // outputs: each warp writes its rows into the output tile, and the LAST warp to finish issues
    // the tile's bulk store (shared-memory arrival counter) -- no CTA barrier, nobody waits for the
    // slowest warp (the output tile was freed by the release barrier)
    auto last_warp = [&]() -> bool {
      fence_proxy_async_smem();
      __syncwarp();
      if ((tid & 31) != 0) return false;
      __threadfence_block();
      if (atomicAdd(&s_out_done, 1u) != K::THREADS / 32 - 1) return false;
      __threadfence_block();
      s_out_done = 0;  // the next tile's arrivals come after the next release barrier
      return true;
    };
    if (p.out_packed) {
      // packed rows [A row-major | b] (BatchResult.output_rows) laid out in
      // the output layout; pad lanes of a partial interleaved block get NaN
      // (pack_rows' default pad, layout.py:72-82)
      constexpr int DSO = K::NA + K::NS;
      const int w = p.out_width;
      const int padded = ((count + w - 1) / w) * w;
      if (tid < padded) {
        R row[DSO];
#pragma unroll
        for (int k = 0; k < K::NA; ++k) row[k] = active ? A[k] : R(__longlong_as_double(0x7ff8000000000000ll));
#pragma unroll
        for (int k = 0; k < K::NS; ++k) row[K::NA + k] = active ? B[k] : R(__longlong_as_double(0x7ff8000000000000ll));
        if (w == 1) {
          RowIO<R, DSO>::store_major(out_a, tid, row);
        } else {
          RowIO<R, DSO>::store_interleaved(out_a, tid, w, row);
        }
      }
      if (last_warp()) {
        const unsigned ob = padded * DSO * sizeof(R);
        char *go = static_cast<char *>(p.stiffness) + e0 * DSO * sizeof(R);
        const unsigned ob16 = ob & ~15u;
        if (ob16) bulk_store(go, out_a, ob16);
        bulk_commit();
        for (unsigned k = ob16; k < ob; k += 4) *reinterpret_cast<uint32_t *>(go + k) = lds32(out_a + k);
      }
      continue;
    }
    if (active) {
      RowIO<R, K::NA>::store_major(out_a, tid, A);
      RowIO<R, K::NS>::store_major(out_b, tid, B);
    }
    if (last_warp()) {
      const unsigned ab = count * K::NA * sizeof(R), bb = count * K::NS * sizeof(R);
      char *ga = static_cast<char *>(p.stiffness) + e0 * K::NA * sizeof(R);
      char *gb = static_cast<char *>(p.load) + e0 * K::NS * sizeof(R);
      const unsigned ab16 = ab & ~15u, bb16 = bb & ~15u;
      if (ab16) bulk_store(ga, out_a, ab16);
      if (bb16) bulk_store(gb, out_b, bb16);
      bulk_commit();
      for (unsigned k = ab16; k < ab; k += 4) *reinterpret_cast<uint32_t *>(ga + k) = lds32(out_a + k);
      for (unsigned k = bb16; k < bb; k += 4) *reinterpret_cast<uint32_t *>(gb + k) = lds32(out_b + k);
    }
  }
  if ((tid & 31) == 0) bulk_wait_all<0>();  // the last-arriving warps' stores: done reading smem at exit
  if (tid == 0) {
    if (p.scheduler) {
      // the last CTA out resets the queue for the next launch on this buffer
      __threadfence();
      if (atomicAdd(p.scheduler + 1, 1ull) == gridDim.x - 1ull) {
        atomicExch(p.scheduler, 0ull);
        atomicExch(p.scheduler + 1, 0ull);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// error detail (message formatting only): det and tol of one element/point
// ---------------------------------------------------------------------------

// Jacobian of one element at one point (-1: the affine tet path), from its
// staged layout: out[0..8] = J[i][k] = dx_i/dxi_k (geometry.py:107-138),
// out[9..17] = dxi_dx[k][i] = adj[k][i] / det (the reference divides,
// geometry.py:86), out[18] = det, out[19] = the degeneracy tolerance.
template <typename R, int ET>
__device__ void element_jacobian(const void *geometry, long long element, int lane_width, int point, double *out,
                                 bool full) {
  constexpr int NV = Shape<ET>::NV, DS = 3 * NV;
  const R *g = static_cast<const R *>(geometry);
  R X[DS];
  const long long blk = element / lane_width, lane = element % lane_width;
  for (int d = 0; d < DS; ++d) X[d] = g[blk * lane_width * DS + d * lane_width + lane];
  const R tol = degeneracy_tolerance<R, NV>(X);
  R J[3][3] = {};
  if (point < 0) {
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) J[i][k] = X[3 * (k + 1) + i] - X[i];
  } else {
    static_for<Shape<ET>::NQ>([&](auto qc) {
      constexpr int Q = decltype(qc)::value;
      if (Q == point) point_jacobian<ET, Q>(X, J);
    });
  }
  // the reference's det and adjugate rounding (geometry.py:62-89; the classification of
  // classify_exact), not the kernels' FMA det
  const R det = det_ref(J);
  if (full) {
    R adj[3][3];
    adjugate_ref(J, adj);
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) {
        out[3 * i + k] = static_cast<double>(J[i][k]);
        out[9 + 3 * i + k] = static_cast<double>(adj[i][k] / det);
      }
    out[18] = static_cast<double>(det);
    out[19] = static_cast<double>(tol);
  } else {
    out[0] = static_cast<double>(det);
    out[1] = static_cast<double>(tol);
  }
}

// ---------------------------------------------------------------------------
// exact classification (fek_classify): the reference's geometry check alone
// ---------------------------------------------------------------------------

// First-error key of one element with the reference's rounding throughout: the
// reference-exact Jacobian (jac_entry), the unfused adjugate det (det_ref) and the
// correctly rounded tol, checked at the affine point (GEO_LINEAR, batched.py:343-349)
// or at q = 0, 1, ... (generic paths, batched.py:193-207) -- _check_dets, :166-177.
template <typename R, int ET, int GEO>
__device__ __forceinline__ unsigned long long classify_exact(const R *X, long long e_abs) {
  const R tol = degeneracy_tolerance<R, Shape<ET>::NV>(X);
  if constexpr (GEO == GEO_LINEAR) {
    R J[3][3];
    point_jacobian<ET, 0>(X, J);
    const int k = classify(det_ref(J), tol);
    return k ? make_error_key(e_abs, -1, k) : NO_ERROR;
  } else {
    unsigned long long key = NO_ERROR;
    static_for<Shape<ET>::NQ>([&](auto qc) {
      FEK_CI(Q, qc);
      if (key == NO_ERROR) {
        R J[3][3];
        point_jacobian<ET, Q>(X, J);
        const int k = classify(det_ref(J), tol);
        if (k) key = make_error_key(e_abs, Q, k);
      }
    });
    return key;
  }
}

template <typename R, int ET, int GEO>
__global__ void __launch_bounds__(256) classify_kernel(const void *geometry, long long n, long long base,
                                                       int lane_width, unsigned long long *error_key) {
  constexpr int DS = 3 * Shape<ET>::NV;
  const R *g = static_cast<const R *>(geometry);
  unsigned long long best = NO_ERROR;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    R X[DS];
    const long long blk = e / lane_width, lane = e % lane_width;
#pragma unroll
    for (int d = 0; d < DS; ++d) X[d] = g[blk * lane_width * DS + d * lane_width + lane];
    const unsigned long long key = classify_exact<R, ET, GEO>(X, base + e);
    best = key < best ? key : best;
  }
  if (best != NO_ERROR) atomicMin(error_key, best);
}

template <typename R, int ET>
__global__ void error_detail_kernel(const void *geometry, long long element, int lane_width, int point,
                                    double *out) {
  element_jacobian<R, ET>(geometry, element, lane_width, point, out, false);
}

template <typename R, int ET>
__global__ void jacobian_kernel(const void *geometry, long long element, int lane_width, int point, double *out) {
  element_jacobian<R, ET>(geometry, element, lane_width, point, out, true);
}

}  // namespace fek
