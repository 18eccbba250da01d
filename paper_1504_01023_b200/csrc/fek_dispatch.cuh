// fek_dispatch.cuh -- kernel table shared by fek_abi.cu and the per-case
// translation units in cases/ (one TU per dtype x element x problem, so the
// 28 kernel instantiations compile in parallel).
#pragma once

#include "../../include/fek.h"
#include "fek_kernel.cuh"

namespace fek {

using KernelFn = void (*)(const LaunchParams);

struct KernelEntry {
  KernelFn fn = nullptr;
  unsigned smem = 0;
  int threads = 0;
  int tile = 0;
};

// index: dtype(2) x element(2) x problem(2) x variant(3) x path(2), then the tile-size variants of
// the QSS natural-path kernels (geo_linear tets, geo_generic prisms): dtype x element x problem x
// tile {64, 128, 256} (fek_batch_desc.tile_elements; the tuner's T dimension)
constexpr int kBaseCount = 2 * 2 * 2 * 3 * 2;
constexpr int kTiles[3] = {64, 128, 256};
constexpr int kTiledCount = 2 * 2 * 2 * 3;
constexpr int kIndexCount = kBaseCount + kTiledCount + 2 * 2 * 2 * 2;
inline int kernel_index(int dtype, int et, int pb, int var, int geo) {
  return (((dtype * 2 + et) * 2 + pb) * 3 + var) * 2 + geo;
}
inline int tiled_index(int dtype, int et, int pb, int tile_slot) {
  return kBaseCount + ((dtype * 2 + et) * 2 + pb) * 3 + tile_slot;
}
// the consumers of the QSS natural-path kernels: fused matrix-free apply (fek_apply, mode 1) and
// CSR assembly (fek_assemble, mode 2)
inline int consumer_index(int dtype, int et, int pb, int mode) {
  return kBaseCount + kTiledCount + (((mode - 1) * 2 + dtype) * 2 + et) * 2 + pb;
}

void register_f64_tet_poisson(KernelEntry *table);
void register_f64_tet_convdiff(KernelEntry *table);
void register_f64_prism_poisson(KernelEntry *table);
void register_f64_prism_convdiff(KernelEntry *table);
void register_f32_tet_poisson(KernelEntry *table);
void register_f32_tet_convdiff(KernelEntry *table);
void register_f32_prism_poisson(KernelEntry *table);
void register_f32_prism_convdiff(KernelEntry *table);

#ifdef FEK_CASE_TU
template <class K>
KernelEntry entry() {
  KernelEntry e;
  e.fn = integrate_kernel<K>;
  e.smem = K::SMEM_BYTES;
  e.threads = K::THREADS;
  e.tile = K::TILE;
  return e;
}

template <typename R, int ET, int PB>
void fill_case(KernelEntry *table, int dtype) {
  table[kernel_index(dtype, ET, PB, QSS, GEO_GENERIC)] = entry<Traits<R, ET, PB, QSS, GEO_GENERIC>>();
#ifndef FEK_QSS_ONLY  // (FEK_QSS_ONLY: fast single-kernel experiments only)
  table[kernel_index(dtype, ET, PB, SQS, GEO_GENERIC)] = entry<Traits<R, ET, PB, SQS, GEO_GENERIC>>();
  table[kernel_index(dtype, ET, PB, SSQ, GEO_GENERIC)] = entry<Traits<R, ET, PB, SSQ, GEO_GENERIC>>();
#endif
  if constexpr (ET == TET) {
    // the reference's three geo_linear loop nests are one hoisted arithmetic
    // (bitwise equal in the reference itself): one kernel serves all three
    const KernelEntry lin = entry<Traits<R, ET, PB, QSS, GEO_LINEAR>>();
    for (int v = 0; v < 3; ++v) table[kernel_index(dtype, ET, PB, v, GEO_LINEAR)] = lin;
  }
#ifndef FEK_NO_TILES  // (experiment builds skip the tuner's tile variants)
  constexpr int NAT = ET == TET ? GEO_LINEAR : GEO_GENERIC;
  table[tiled_index(dtype, ET, PB, 0)] = entry<Traits<R, ET, PB, QSS, NAT, kTiles[0]>>();
  table[tiled_index(dtype, ET, PB, 1)] = entry<Traits<R, ET, PB, QSS, NAT, kTiles[1]>>();
  table[tiled_index(dtype, ET, PB, 2)] = entry<Traits<R, ET, PB, QSS, NAT, kTiles[2]>>();
  table[consumer_index(dtype, ET, PB, MODE_APPLY)] = entry<Traits<R, ET, PB, QSS, NAT, 0, MODE_APPLY>>();
  table[consumer_index(dtype, ET, PB, MODE_ASSEMBLE)] = entry<Traits<R, ET, PB, QSS, NAT, 0, MODE_ASSEMBLE>>();
#endif
}
#endif

}  // namespace fek
