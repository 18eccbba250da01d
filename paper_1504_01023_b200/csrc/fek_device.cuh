// fek_device.cuh -- sm_100a building blocks for the element-integration kernels:
//   * 1-D TMA bulk copies (cp.async.bulk) global<->shared with mbarrier
//     completion (loads) and bulk-group completion (stores);
//   * bank-conflict-free staging of per-element rows between a shared-memory
//     tile (exact global byte image, so one bulk copy moves a whole tile) and
//     per-thread registers.
//
// Row staging.  Thread l owns element l of the tile; its
// row of DS reals starts at byte l*DS*sizeof(R).  A warp-wide 16-byte access
// (LDS.128/STS.128) is served in quarter-warp phases of 8 lanes; lanes whose
// 16-byte chunk maps to the same bank group (chunk index mod 8) serialize.
// With NCH = row bytes / 16 chunks per row, lane q of a phase touches bank
// group (NCH*q + c) mod 8.  Unless NCH is odd this repeats across lanes
// (NCH = 8, the 4x4 fp64 stiffness row, puts all 8 lanes on ONE bank group).
// We therefore let lane q visit its chunks in rotated order c = (j + rot(q))
// mod NCH at step j, with rot(q) = q >> (3 - min(ctz(NCH), 3)), which makes
// every step conflict-free (checked by static_assert), and undo the rotation
// in registers with a log2 barrel shifter of predicated selects (ALU pipe,
// cheaper than the 2-8x shared-memory replay it removes).
#pragma once

#include <cstdint>
#include <type_traits>
#include <utility>

namespace fek {

// ---------------------------------------------------------------------------
// compile-time loops
// ---------------------------------------------------------------------------

template <int N, class F>
__device__ __forceinline__ void static_for(F &&f) {
  [&]<int... I>(std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
  }(std::make_integer_sequence<int, N>{});
}

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(bar), "r"(parity)
      : "memory");
  return done != 0;
}

// Bounded wait: returns false if the phase never completed (a pipeline bug);
// the caller records FEK_KIND_PIPELINE_TIMEOUT instead of hanging the GPU.
__device__ __forceinline__ bool mbar_wait(uint32_t bar, uint32_t parity) {
#pragma unroll 1
  for (uint32_t spin = 0; spin < (1u << 24); ++spin) {
    if (mbar_try_wait(bar, parity)) return true;
  }
  return false;
}

// global -> shared, completion counted on an mbarrier (UBLKCP.S.G in SASS)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

// shared -> global, bulk-group completion
__device__ __forceinline__ void bulk_store(void *dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// generic-proxy smem writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint4 pack2(double a, double b) {
  return make_uint4(static_cast<uint32_t>(__double2loint(a)), static_cast<uint32_t>(__double2hiint(a)),
                    static_cast<uint32_t>(__double2loint(b)), static_cast<uint32_t>(__double2hiint(b)));
}
__device__ __forceinline__ uint2 pack1(double a) {
  return make_uint2(static_cast<uint32_t>(__double2loint(a)), static_cast<uint32_t>(__double2hiint(a)));
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ void sts64(uint32_t addr, uint2 v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(v.x), "r"(v.y) : "memory");
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// rotation schedule for conflict-free 16-byte row access
// ---------------------------------------------------------------------------

constexpr int ctz_capped3(int v) {
  int t = 0;
  while (t < 3 && (v & 1) == 0) {
    v >>= 1;
    ++t;
  }
  return t;
}

template <int NCH>
struct Rotation {
  static constexpr int BITS = ctz_capped3(NCH);  // number of barrel-shifter stages
  __host__ __device__ static constexpr int rot(int q) { return q >> (3 - BITS); }
  static constexpr bool conflict_free() {
    for (int j = 0; j < NCH; ++j) {
      bool used[8] = {false, false, false, false, false, false, false, false};
      for (int q = 0; q < 8; ++q) {
        int c = (j + rot(q) % NCH) % NCH;
        int g = (NCH * q + c) % 8;
        if (used[g]) return false;
        used[g] = true;
      }
    }
    return true;
  }
};

__device__ __forceinline__ uint4 sel4(bool p, uint4 a, uint4 b) {
  return make_uint4(p ? a.x : b.x, p ? a.y : b.y, p ? a.z : b.z, p ? a.w : b.w);
}

// v[j] holds chunk (j + rot) % NCH; afterwards v[c] holds chunk c.
template <int NCH>
__device__ __forceinline__ void unrotate(uint4 (&v)[NCH], int rot) {
  static_for<Rotation<NCH>::BITS>([&](auto k) {
    constexpr int step = 1 << decltype(k)::value;
    const bool on = (rot >> decltype(k)::value) & 1;
    uint4 old[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) old[j] = v[j];
#pragma unroll
    for (int j = 0; j < NCH; ++j) v[j] = sel4(on, old[(j - step % NCH + NCH) % NCH], old[j]);
  });
}

// v[c] holds chunk c; afterwards v[j] holds chunk (j + rot) % NCH.
template <int NCH>
__device__ __forceinline__ void rotate(uint4 (&v)[NCH], int rot) {
  static_for<Rotation<NCH>::BITS>([&](auto k) {
    constexpr int step = 1 << decltype(k)::value;
    const bool on = (rot >> decltype(k)::value) & 1;
    uint4 old[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) old[j] = v[j];
#pragma unroll
    for (int j = 0; j < NCH; ++j) v[j] = sel4(on, old[(j + step) % NCH], old[j]);
  });
}

// ---------------------------------------------------------------------------
// row <-> registers
// ---------------------------------------------------------------------------

template <typename R>
__device__ __forceinline__ R bits_to_real(uint32_t lo, uint32_t hi);
template <>
__device__ __forceinline__ double bits_to_real<double>(uint32_t lo, uint32_t hi) {
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

template <typename R, int DS>
struct RowIO {
  static constexpr int BYTES = DS * static_cast<int>(sizeof(R));
  static constexpr bool CHUNKED = (BYTES % 16) == 0;
  static constexpr int NCH = BYTES / 16;
  static constexpr int PER_CHUNK = 16 / static_cast<int>(sizeof(R));
  static_assert(!CHUNKED || Rotation<NCH>::conflict_free(), "rotation schedule not conflict-free");

  // element-major tile: row of element l at tile + l*BYTES
  __device__ __forceinline__ static void load_major(uint32_t tile, int l, R (&out)[DS]) {
    const uint32_t row = tile + static_cast<uint32_t>(l) * BYTES;
    if constexpr (CHUNKED) {
      const int rot = Rotation<NCH>::rot(l & 7);
      uint4 v[NCH];
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        int c = j + rot;
        c = c >= NCH ? c - NCH : c;
        v[j] = lds128(row + 16u * c);
      }
      unrotate<NCH>(v, rot);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
        for (int k = 0; k < PER_CHUNK; ++k) {
          if constexpr (sizeof(R) == 8) {
            out[c * PER_CHUNK + k] = bits_to_real<double>(w[2 * k], w[2 * k + 1]);
          } else {
            out[c * PER_CHUNK + k] = __uint_as_float(w[k]);
          }
        }
      }
    } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
      for (int j = 0; j < BYTES / 8; ++j) {
        const uint2 v = lds64(row + 8u * j);
        if constexpr (sizeof(R) == 8) {
          out[j] = bits_to_real<double>(v.x, v.y);
        } else {
          out[2 * j] = __uint_as_float(v.x);
          out[2 * j + 1] = __uint_as_float(v.y);
        }
      }
    } else {
      static_assert(sizeof(R) == 4, "odd byte rows only exist for fp32");
#pragma unroll
      for (int j = 0; j < DS; ++j) out[j] = __uint_as_float(lds32(row + 4u * j));
    }
  }

  // lane-interleaved tile (W lanes per block): datum d of element l at
  // ((l/W)*W*DS + d*W + l%W) reals
  __device__ __forceinline__ static void load_interleaved(uint32_t tile, int l, int w, R (&out)[DS]) {
    const uint32_t base = tile + static_cast<uint32_t>((l / w) * w * DS + (l % w)) * sizeof(R);
    const uint32_t stride = static_cast<uint32_t>(w) * sizeof(R);
#pragma unroll
    for (int d = 0; d < DS; ++d) {
      if constexpr (sizeof(R) == 8) {
        const uint2 v = lds64(base + d * stride);
        out[d] = bits_to_real<double>(v.x, v.y);
      } else {
        out[d] = __uint_as_float(lds32(base + d * stride));
      }
    }
  }

  __device__ __forceinline__ static void load(uint32_t tile, int l, int w, R (&out)[DS]) {
    if (w == 1) {
      load_major(tile, l, out);
    } else {
      load_interleaved(tile, l, w, out);
    }
  }

  // element-major row in natural chunk order, no rotation: for the lane-pair kernel, where a
  // quarter-warp phase touches 4 distinct rows (the two lanes of a pair read the same 16-byte
  // address: a broadcast) whose starts (NCH * e mod 8) fall in distinct bank groups for NCH = 9
  // (prism geometry) and 10 (ConvDiff coefficients) -- no barrel shifter needed
  __device__ __forceinline__ static void load_major_paired(uint32_t tile, int l, R (&out)[DS]) {
    static_assert(CHUNKED && sizeof(R) == 8, "paired row loads: fp64 rows of whole 16-byte chunks");
    static_assert((NCH * 1) % 8 != 0 && (NCH * 2) % 8 != 0 && (NCH * 3) % 8 != 0 && (NCH * 2) % 8 != NCH % 8 &&
                  (NCH * 3) % 8 != NCH % 8 && (NCH * 3) % 8 != (NCH * 2) % 8,
                  "4 rows per quarter-warp phase must start in distinct bank groups");
    const uint32_t row = tile + static_cast<uint32_t>(l) * BYTES;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const uint4 v = lds128(row + 16u * c);
      out[2 * c] = bits_to_real<double>(v.x, v.y);
      out[2 * c + 1] = bits_to_real<double>(v.z, v.w);
    }
  }
  __device__ __forceinline__ static void load_paired(uint32_t tile, int l, int w, R (&out)[DS]) {
    if (w == 1) {
      load_major_paired(tile, l, out);
    } else {
      load_interleaved(tile, l, w, out);
    }
  }

  // lane-interleaved output tile (datum d of element l at (l/W)*W*DS + d*W + l%W)
  __device__ __forceinline__ static void store_interleaved(uint32_t tile, int l, int w, const R (&in)[DS]) {
    const uint32_t base = tile + static_cast<uint32_t>((l / w) * w * DS + (l % w)) * sizeof(R);
    const uint32_t stride = static_cast<uint32_t>(w) * sizeof(R);
#pragma unroll
    for (int d = 0; d < DS; ++d) {
      if constexpr (sizeof(R) == 8) {
        sts64(base + d * stride, make_uint2(static_cast<uint32_t>(__double2loint(in[d])),
                                            static_cast<uint32_t>(__double2hiint(in[d]))));
      } else {
        sts32(base + d * stride, __float_as_uint(in[d]));
      }
    }
  }

  // element-major output tile
  __device__ __forceinline__ static void store_major(uint32_t tile, int l, const R (&in)[DS]) {
    const uint32_t row = tile + static_cast<uint32_t>(l) * BYTES;
    if constexpr (CHUNKED) {
      const int rot = Rotation<NCH>::rot(l & 7);
      uint4 v[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < PER_CHUNK; ++k) {
          if constexpr (sizeof(R) == 8) {
            const double x = in[c * PER_CHUNK + k];
            w[2 * k] = static_cast<uint32_t>(__double2loint(x));
            w[2 * k + 1] = static_cast<uint32_t>(__double2hiint(x));
          } else {
            w[k] = __float_as_uint(in[c * PER_CHUNK + k]);
          }
        }
        v[c] = make_uint4(w[0], w[1], w[2], w[3]);
      }
      rotate<NCH>(v, rot);
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        int c = j + rot;
        c = c >= NCH ? c - NCH : c;
        sts128(row + 16u * c, v[j]);
      }
    } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
      for (int j = 0; j < BYTES / 8; ++j) {
        if constexpr (sizeof(R) == 8) {
          sts64(row + 8u * j, make_uint2(static_cast<uint32_t>(__double2loint(in[j])),
                                         static_cast<uint32_t>(__double2hiint(in[j]))));
        } else {
          sts64(row + 8u * j, make_uint2(__float_as_uint(in[2 * j]), __float_as_uint(in[2 * j + 1])));
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < DS; ++j) sts32(row + 4u * j, __float_as_uint(in[j]));
    }
  }
};

}  // namespace fek
