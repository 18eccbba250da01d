// fek_element.cuh -- per-element integration math, one thread per element.
//
// Reference semantics (paths under /root/reference/pkg/src/feklab):
//   geometry  : bbox scale batched.py:136-148; adjugate/det :151-163;
//               degeneracy/inversion check :166-177 (|det| <= 1e-14*diag^3
//               first, then det < 0); inverse = adj * (1/det) :180-182;
//               affine Jacobian columns v_{k+1}-v_0 :185-190; per-point
//               Jacobian X^T * ld_q :193-207; global derivatives :210-220.
//   Poisson   : A_rs = sum_q vol_q g_r.g_s, b_r = sum_q vol_q phi_r(q) d0[q]
//               (_PoissonBatch :238-251, symmetric mirror :373-380).
//   ConvDiff  : A_rs = sum_q vol_q sum_ij c_ij phi^i_r phi^j_s,
//               b_r = sum_q vol_q sum_i d_i phi^i_r (_ConvDiffBatch :254-275).
//   geo_linear: q-invariant parts hoisted out of the q loop (_linear_terms
//               :352-358, _ConvDiffLinear :298-335); the remaining q-sums of
//               tabulated basis values are the precomputed quadrature moments
//               WSUM/MV/MVV/WV of refconst.h.
//   variants  : QSS / SQS / SSQ loop nests of the generic path (:434-515);
//               SQS recomputes the point data per row, SSQ per entry, exactly
//               as the reference's loop skeletons do.
//
// Arithmetic is written with explicit fma() and the library is compiled with
// --fmad=false, so every element runs one fixed instruction sequence: results
// are bitwise independent of tile position, layout, chunking and GPU count.
// They differ from the reference's numpy evaluation order by rounding only
// (relative Frobenius ~1e-15, tolerance 1e-12 per SPEC).
#pragma once

#include <cstdint>
#include <type_traits>

#include "fek_device.cuh"
#include "refconst.h"

namespace fek {

enum : int { TET = 0, PRISM = 1 };
enum : int { POISSON = 0, CONV_DIFF = 1 };
enum : int { QSS = 0, SQS = 1, SSQ = 2 };
enum : int { GEO_LINEAR = 0, GEO_GENERIC = 1 };

constexpr unsigned long long NO_ERROR = 0xFFFFFFFFFFFFFFFFull;
constexpr int KIND_DEGENERATE = 1;
constexpr int KIND_INVERTED = 2;
constexpr int KIND_PIPELINE_TIMEOUT = 3;
// |det J| within NEAR_TOL_FACTOR * tol at the element's first flagged point: the kernels' FMA det
// cannot decide the class the reference's way there; fek_classify re-derives the key exactly
constexpr int KIND_NEAR = 4;
// fek_assemble: an element's node pair (row r, any column) is not in the caller's CSR pattern
constexpr int KIND_PATTERN = 5;
constexpr int ERROR_BLOCK_SHIFT = 13;  // batched.py:50 BLOCK_ELEMENTS = 8192

// Error key ordering = the reference's first-error rule (batched.py:528-533,
// :166-177): earliest 8192-element block, then smallest quadrature point
// inside the block (15 = affine / no point), then lowest element.
__host__ __device__ __forceinline__ unsigned long long make_error_key(long long element, int point,
                                                                      int kind) {
  const unsigned long long blk = static_cast<unsigned long long>(element) >> ERROR_BLOCK_SHIFT;
  const unsigned long long within = static_cast<unsigned long long>(element) & 8191ull;
  const unsigned long long q = point < 0 ? 15ull : static_cast<unsigned long long>(point);
  return (blk << 24) | (q << 20) | (within << 7) | static_cast<unsigned long long>(kind);
}

// ---------------------------------------------------------------------------
// element geometry helpers
// ---------------------------------------------------------------------------

template <int ET>
struct Shape;
template <>
struct Shape<TET> {
  static constexpr int NV = 4, NS = 4, NQ = 4;
  __host__ __device__ static constexpr double w(int q) { return refconst::TET_W[q]; }
  __host__ __device__ static constexpr double val(int q, int s) { return refconst::TET_VAL[q][s]; }
  __host__ __device__ static constexpr double ld(int q, int s, int k) { return refconst::TET_LD[q][s][k]; }
};
template <>
struct Shape<PRISM> {
  static constexpr int NV = 6, NS = 6, NQ = 6;
  __host__ __device__ static constexpr double w(int q) { return refconst::PRISM_W[q]; }
  __host__ __device__ static constexpr double val(int q, int s) { return refconst::PRISM_VAL[q][s]; }
  __host__ __device__ static constexpr double ld(int q, int s, int k) { return refconst::PRISM_LD[q][s][k]; }
};

template <typename R>
__device__ __forceinline__ R rmax(R a, R b) {
  return a > b ? a : b;
}
template <typename R>
__device__ __forceinline__ R rmin(R a, R b) {
  return a < b ? a : b;
}

// s**3 rounded ONCE, as the reference's `scale**3` is a single pow() (batched.py:167,
// geometry.py:89): s^2 = p + pe and p s = h + he exactly, so s^3 = h + (he + pe s) with only
// the final sum rounding (a double rounding needs the tail within ~2^-100 of a tie).  The
// naive (s*s)*s differs from the correctly rounded cube on ~26% of scales.  numpy's own
// scale**3 is host-ISA dependent: glibc pow is correctly rounded on all but
// ~0.1% of scales, the AVX-512 SVML pow numpy dispatches to is not on ~5%.
template <typename R>
__device__ __forceinline__ R cube_rn(R s) {
  const R p = s * s, pe = fma(s, s, -p);
  const R h = p * s, he = fma(p, s, -h);
  return h + fma(pe, s, he);
}

// 1e-14 * (bounding-box diagonal)^3   (geometry.py:22-24, batched.py:136-148)
template <typename R, int NV>
__device__ __forceinline__ R degeneracy_tolerance(const R *X) {
  R acc = R(0);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    R hi = X[i], lo = X[i];
#pragma unroll
    for (int v = 1; v < NV; ++v) {
      hi = fmax(hi, X[3 * v + i]);
      lo = fmin(lo, X[3 * v + i]);
    }
    const R span = hi - lo;
    acc = (i == 0) ? span * span : acc + span * span;  // batched.py:145-147 rounding
  }
  const R scale = sqrt(acc);
  return R(1e-14) * cube_rn(scale);
}

// The kernels classify on their own (FMA-contracted) det against this widened bound and leave
// the near elements to the exact classification (classify_exact / fek_classify).
// Both dets approximate the exact determinant within ~3 * 2^-53 * 6 M^3, M = max |J entry| <=
// the bounding-box diagonal (tet J columns are vertex differences; prism J entries are convex
// combinations of them, the zeta column half of one), i.e. within 0.2 tol each: beyond 16 tol
// the fast det's class (valid / inverted) is the reference's.  Valid meshes have det ~ diag^3,
// 1e13 tol, so the exact pass never runs on them.
constexpr int NEAR_TOL_FACTOR = 16;
template <typename R, int NV>
__device__ __forceinline__ R near_bound(const R *X) {
  return R(NEAR_TOL_FACTOR) * degeneracy_tolerance<R, NV>(X);  // exact: a power of two
}

// cofactor adjugate + determinant of J[i][k] (row i = physical x_i,
// column k = reference xi_k), batched.py:151-163
template <typename R>
struct Jac {
  R inv[3][3];  // inv[k][i] = d xi_k / d x_i
  R det;
};

// 1/x: hardware approximation + two Newton steps (~1 ulp; no slow-path
// branch).  x = 0 / denormal only happens for degenerate elements, which are
// reported and whose outputs are discarded.
__device__ __forceinline__ double recip(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ float recip(float x) { return 1.0f / x; }

template <typename R>
__device__ __forceinline__ R det3(const R (&J)[3][3]) {
  const R k00 = fma(J[1][1], J[2][2], -(J[1][2] * J[2][1]));
  const R k01 = fma(J[1][2], J[2][0], -(J[1][0] * J[2][2]));
  const R k02 = fma(J[1][0], J[2][1], -(J[1][1] * J[2][0]));
  return fma(J[0][0], k00, fma(J[0][1], k01, J[0][2] * k02));
}

// inverse from a precomputed determinant and its reciprocal
template <typename R>
__device__ __forceinline__ Jac<R> invert3_with(const R (&J)[3][3], R det, R r) {
  const R a = J[0][0], b = J[0][1], c = J[0][2];
  const R d = J[1][0], e = J[1][1], f = J[1][2];
  const R g = J[2][0], h = J[2][1], i = J[2][2];
  Jac<R> out;
  out.det = det;
  out.inv[0][0] = fma(e, i, -(f * h)) * r;
  out.inv[0][1] = fma(c, h, -(b * i)) * r;
  out.inv[0][2] = fma(b, f, -(c * e)) * r;
  out.inv[1][0] = fma(f, g, -(d * i)) * r;
  out.inv[1][1] = fma(a, i, -(c * g)) * r;
  out.inv[1][2] = fma(c, d, -(a * f)) * r;
  out.inv[2][0] = fma(d, h, -(e * g)) * r;
  out.inv[2][1] = fma(b, g, -(a * h)) * r;
  out.inv[2][2] = fma(a, e, -(b * d)) * r;
  return out;
}

template <typename R>
__device__ __forceinline__ Jac<R> invert3(const R (&J)[3][3]) {
  const R a = J[0][0], b = J[0][1], c = J[0][2];
  const R d = J[1][0], e = J[1][1], f = J[1][2];
  const R g = J[2][0], h = J[2][1], i = J[2][2];
  const R k00 = fma(e, i, -(f * h));
  const R k01 = fma(f, g, -(d * i));
  const R k02 = fma(d, h, -(e * g));
  Jac<R> out;
  out.det = fma(a, k00, fma(b, k01, c * k02));
  const R r = recip(out.det);
  out.inv[0][0] = k00 * r;
  out.inv[0][1] = fma(c, h, -(b * i)) * r;
  out.inv[0][2] = fma(b, f, -(c * e)) * r;
  out.inv[1][0] = k01 * r;
  out.inv[1][1] = fma(a, i, -(c * g)) * r;
  out.inv[1][2] = fma(c, d, -(a * f)) * r;
  out.inv[2][0] = k02 * r;
  out.inv[2][1] = fma(b, g, -(a * h)) * r;
  out.inv[2][2] = fma(a, e, -(b * d)) * r;
  return out;
}

// degenerate first, then inverted; NaN determinants pass (as in numpy)
template <typename R>
__device__ __forceinline__ int classify(R det, R tol) {
  if (fabs(det) <= tol) return KIND_DEGENERATE;
  if (det < R(0)) return KIND_INVERTED;
  return 0;
}

// the kernels' classification: near (|det| <= near_bound) first, then inverted
template <typename R>
__device__ __forceinline__ int classify_fast(R det, R bound) {
  if (fabs(det) <= bound) return KIND_NEAR;
  if (det < R(0)) return KIND_INVERTED;
  return 0;
}

__device__ __forceinline__ double mul_rn(double x, double y) { return __dmul_rn(x, y); }
__device__ __forceinline__ double add_rn(double x, double y) { return __dadd_rn(x, y); }
__device__ __forceinline__ double sub_rn(double x, double y) { return __dsub_rn(x, y); }
__device__ __forceinline__ float mul_rn(float x, float y) { return __fmul_rn(x, y); }
__device__ __forceinline__ float add_rn(float x, float y) { return __fadd_rn(x, y); }
__device__ __forceinline__ float sub_rn(float x, float y) { return __fsub_rn(x, y); }

// The reference's adjugate and determinant rounding (batched.py:151-163 = geometry.py:62-72):
// every product rounded, cofactors e*i - f*h, det = (a c00 + b c01) + c c02.  Never contracted.
template <typename R>
__device__ __forceinline__ R det_ref(const R (&J)[3][3]) {
  const R c00 = sub_rn(mul_rn(J[1][1], J[2][2]), mul_rn(J[1][2], J[2][1]));
  const R c01 = sub_rn(mul_rn(J[1][2], J[2][0]), mul_rn(J[1][0], J[2][2]));
  const R c02 = sub_rn(mul_rn(J[1][0], J[2][1]), mul_rn(J[1][1], J[2][0]));
  return add_rn(add_rn(mul_rn(J[0][0], c00), mul_rn(J[0][1], c01)), mul_rn(J[0][2], c02));
}
template <typename R>
__device__ __forceinline__ void adjugate_ref(const R (&J)[3][3], R (&adj)[3][3]) {
  auto cof = [](R x, R y, R u, R v) { return sub_rn(mul_rn(x, y), mul_rn(u, v)); };
  const R a = J[0][0], b = J[0][1], c = J[0][2];
  const R d = J[1][0], e = J[1][1], f = J[1][2];
  const R g = J[2][0], h = J[2][1], i = J[2][2];
  adj[0][0] = cof(e, i, f, h);
  adj[0][1] = cof(c, h, b, i);
  adj[0][2] = cof(b, f, c, e);
  adj[1][0] = cof(f, g, d, i);
  adj[1][1] = cof(a, i, c, g);
  adj[1][2] = cof(c, d, a, f);
  adj[2][0] = cof(d, h, e, g);
  adj[2][1] = cof(b, g, a, h);
  adj[2][2] = cof(a, e, b, d);
}

// (kind, point) of an element from per-point bitmasks: the SMALLEST flagged point, as the
// reference checks q = 0, 1, ... in order; a near point there leaves the verdict to fek_classify
__device__ __forceinline__ void first_failure(unsigned inverted, unsigned near, int &kind, int &point) {
  const unsigned m = inverted | near;
  kind = 0;
  point = -1;
  if (m) {
    point = __ffs(m) - 1;
    kind = ((near >> point) & 1u) ? KIND_NEAR : KIND_INVERTED;
  }
}

// sum_k c_k * x_k over compile-time coefficients, skipping zeros and using
// +-1 as add/sub (the reference's _axpy_fixed, batched.py:119-133).
// EXACT = the reference's rounding: every product rounded, then summed left
// to right (used for the Jacobian, whose entries are differences of absolute
// coordinates and therefore ill-conditioned on fine meshes: matching the
// reference's rounding there makes J bitwise equal to the reference's).
// Otherwise products are fused into the running sum.
template <typename R, bool EXACT = false>
struct Lin {
  R acc;
  bool any = false;
  __device__ __forceinline__ void add(double c, R x) {
    if (c == 0.0) return;
    const R term = (c == 1.0) ? x : (c == -1.0 ? -x : R(c) * x);
    if (!any) {
      acc = term;
      any = true;
    } else if (EXACT || c == 1.0 || c == -1.0) {
      acc = acc + term;
    } else {
      acc = fma(R(c), x, acc);
    }
  }
  __device__ __forceinline__ R get() const { return any ? acc : R(0); }
};

#define FEK_CI(name, ic) constexpr int name = decltype(ic)::value

// Jacobian entry J[i][K] at compile-time point Q: sum_v ld[Q][v][K] X[v][i]
// with the reference's rounding (batched.py:193-207 via _axpy_fixed)
template <int ET, int Q, int K, typename R>
__device__ __forceinline__ R jac_entry(const R *X, int i) {
  using S = Shape<ET>;
  Lin<R, true> acc;
  static_for<S::NV>([&](auto vc) {
    FEK_CI(v, vc);
    acc.add(S::ld(Q, v, K), X[3 * v + i]);
  });
  return acc.get();
}

template <int ET, int Q, typename R>
__device__ __forceinline__ void point_jacobian(const R *X, R (&J)[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    J[i][0] = jac_entry<ET, Q, 0>(X, i);
    J[i][1] = jac_entry<ET, Q, 1>(X, i);
    J[i][2] = jac_entry<ET, Q, 2>(X, i);
  }
}

// Global derivatives of shape function SF at point Q: g[i] = sum_k ld[Q][SF][k] inv[k][i]
template <int ET, int Q, int SF, typename R>
__device__ __forceinline__ void global_grad(const Jac<R> &jac, R (&g)[3]) {
  using S = Shape<ET>;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    Lin<R> t;
    static_for<3>([&](auto kc) {
      FEK_CI(k, kc);
      t.add(S::ld(Q, SF, k), jac.inv[k][i]);
    });
    g[i] = t.get();
  }
}

// Prism gradients from the factorisation of the reference derivatives
// (refelem.py:145-155): ld[a] = (dlam_a * lo, -lam_a/2), ld[a+3] = (dlam_a * hi,
// +lam_a/2) with dlam = (-1,-1), (1,0), (0,1).  With m_a = (lam_a/2) inv[2]:
// g_a = lo (dlam_a . inv[0:2]) - m_a and g_a+3 = hi (dlam_a . inv[0:2]) + m_a --
// 30 FP64 operations per point instead of 42.
template <int Q, typename R>
__device__ __forceinline__ void prism_grads(const Jac<R> &jac, R (&g)[6][3]) {
  using S = Shape<PRISM>;
  constexpr double lo = S::ld(Q, 1, 0), hi = S::ld(Q, 4, 0);
  static_assert(S::ld(Q, 0, 0) == -lo && S::ld(Q, 0, 1) == -lo && S::ld(Q, 1, 1) == 0.0 && S::ld(Q, 2, 0) == 0.0 &&
                S::ld(Q, 2, 1) == lo, "bottom-face derivative structure");
  static_assert(S::ld(Q, 3, 0) == -hi && S::ld(Q, 3, 1) == -hi && S::ld(Q, 4, 1) == 0.0 && S::ld(Q, 5, 0) == 0.0 &&
                S::ld(Q, 5, 1) == hi, "top-face derivative structure");
  static_assert(S::ld(Q, 0, 2) == -S::ld(Q, 3, 2) && S::ld(Q, 1, 2) == -S::ld(Q, 4, 2) &&
                S::ld(Q, 2, 2) == -S::ld(Q, 5, 2), "zeta derivative structure");
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const R x0 = jac.inv[0][i], x1 = jac.inv[1][i], x2 = jac.inv[2][i];
    const R s01 = x0 + x1;
    const R m0 = R(S::ld(Q, 3, 2)) * x2, m1 = R(S::ld(Q, 4, 2)) * x2, m2 = R(S::ld(Q, 5, 2)) * x2;
    g[0][i] = fma(R(-lo), s01, -m0);
    g[3][i] = fma(R(-hi), s01, m0);
    g[1][i] = fma(R(lo), x0, -m1);
    g[4][i] = fma(R(hi), x0, m1);
    g[2][i] = fma(R(lo), x1, -m2);
    g[5][i] = fma(R(hi), x1, m2);
  }
}

template <int ET, int Q, typename R>
__device__ __forceinline__ void all_grads(const Jac<R> &jac, R (&g)[Shape<ET>::NS][3]) {
  if constexpr (ET == PRISM && sizeof(R) == 8) {
    prism_grads<Q>(jac, g);
  } else {
    static_for<Shape<ET>::NS>([&](auto sc) {
      FEK_CI(s, sc);
      global_grad<ET, Q, s>(jac, g[s]);
    });
  }
}

// ---------------------------------------------------------------------------
// geo_linear: tetrahedra, Jacobian once per element (all three variants:
// the reference's _qss/_sqs/_ssq_linear are the same hoisted arithmetic)
// ---------------------------------------------------------------------------

template <typename R, int PB>
__device__ __forceinline__ void integrate_tet_linear(const R (&X)[12], const R *coef, R (&A)[16],
                                                     R (&B)[4], int &kind) {
  using namespace refconst;
  R J[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) J[i][k] = X[3 * (k + 1) + i] - X[i];
  const Jac<R> jac = invert3(J);
  kind = classify_fast(jac.det, near_bound<R, 4>(X));
  const R det = jac.det;
  // g[s][i]: shape 0 has local gradient (-1,-1,-1), shape k+1 the unit e_k
  R g[4][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    g[1][i] = jac.inv[0][i];
    g[2][i] = jac.inv[1][i];
    g[3][i] = jac.inv[2][i];
    g[0][i] = -((jac.inv[0][i] + jac.inv[1][i]) + jac.inv[2][i]);
  }
  constexpr R wsum = R(TET_WSUM);
  if constexpr (PB == POISSON) {
    const R vt = det * wsum;
    static_for<4>([&](auto rc) {
      FEK_CI(r, rc);
#pragma unroll
      for (int s = r; s < 4; ++s) {
        const R gg = fma(g[r][0], g[s][0], fma(g[r][1], g[s][1], g[r][2] * g[s][2]));
        A[4 * r + s] = vt * gg;
        A[4 * s + r] = A[4 * r + s];
      }
      constexpr R wv0 = R(TET_WV[0][r]);
      R acc = wv0 * coef[0];
      static_for<3>([&](auto qc) {
        FEK_CI(q, qc);
        constexpr R wv = R(TET_WV[q + 1][r]);
        acc = fma(wv, coef[q + 1], acc);
      });
      B[r] = det * acc;
    });
  } else {
    // coef row: c00 c01 c02 c03 c10 ... c33 d0 d1 d2 d3 (problems.py:136-140)
    const R *c = coef;
    const R *d = coef + 16;
    R Cg[4][3], row0[4], col0[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
        Cg[s][i] = fma(c[4 * (i + 1) + 1], g[s][0], fma(c[4 * (i + 1) + 2], g[s][1], c[4 * (i + 1) + 3] * g[s][2]));
      row0[s] = fma(c[1], g[s][0], fma(c[2], g[s][1], c[3] * g[s][2]));
      col0[s] = fma(c[4], g[s][0], fma(c[8], g[s][1], c[12] * g[s][2]));
    }
    const R c00 = c[0];
    static_for<4>([&](auto rc) {
      FEK_CI(r, rc);
      static_for<4>([&](auto sc) {
        FEK_CI(s, sc);
        const R dd = fma(g[r][0], Cg[s][0], fma(g[r][1], Cg[s][1], g[r][2] * Cg[s][2]));
        constexpr R mvv = R(TET_MVV[r][s]), mvs = R(TET_MV[s]), mvr = R(TET_MV[r]);
        R t = mvv * c00;
        t = fma(mvs, col0[r], t);
        t = fma(mvr, row0[s], t);
        t = fma(wsum, dd, t);
        A[4 * r + s] = det * t;
      });
      const R dg = fma(d[1], g[r][0], fma(d[2], g[r][1], d[3] * g[r][2]));
      constexpr R mvr = R(TET_MV[r]);
      B[r] = det * fma(wsum, dg, mvr * d[0]);
    });
  }
}

// ---------------------------------------------------------------------------
// geo_generic: Jacobian per quadrature point (prisms; tets on request)
// ---------------------------------------------------------------------------

// Point data at compile-time point Q from vertex coordinates X.
template <int ET, int Q, typename R>
struct PointData {
  Jac<R> jac;
  R vol;
  int kind;
  __device__ __forceinline__ PointData(const R *X, R bound) {
    R J[3][3];
    point_jacobian<ET, Q>(X, J);
    init(J, bound);
  }
  __device__ __forceinline__ PointData(const R (&J)[3][3], R bound) { init(J, bound); }
  __device__ __forceinline__ PointData(const R (&J)[3][3], R det, R r, R bound) {
    jac = invert3_with(J, det, r);
    kind = classify_fast(det, bound);
    constexpr R w = R(Shape<ET>::w(Q));
    vol = det * w;
  }
  __device__ __forceinline__ void init(const R (&J)[3][3], R bound) {
    jac = invert3(J);
    kind = classify_fast(jac.det, bound);
    constexpr R w = R(Shape<ET>::w(Q));
    vol = jac.det * w;
  }
};

// Geometry source for the generic path: each call returns the element's
// vertex coordinates, either from registers or re-read from the staged
// shared-memory tile (keeps registers free on the FP64-bound prism path and,
// for SQS/SSQ, makes the per-row / per-entry recomputation real work as in
// the reference's loop skeletons).
template <typename R, int DS>
struct RegGeometry {
  const R (&X)[DS];
  __device__ __forceinline__ void fetch(R (&out)[DS]) const {
#pragma unroll
    for (int i = 0; i < DS; ++i) out[i] = X[i];
  }
};

template <typename R, int DS>
struct SmemGeometry {
  uint32_t tile;
  int lane;
  int width;
  __device__ __forceinline__ void fetch(R (&out)[DS]) const { RowIO<R, DS>::load(tile, lane, width, out); }
};

// Visit every quadrature point with its point data, computing each DISTINCT
// Jacobian column once.  Tets: J is point-independent.  Prisms (q = 2t + z):
// columns 0/1 depend only on the zeta level z, column 2 only on the triangle
// point t (refelem.py:145-155).  The reference recomputes J per point; the
// values are bitwise the same (identical operations on identical operands).
// Points are visited z-major for prisms (accumulation order is free: A is
// not bitwise-matched, only J is).
template <typename R, int ET, class Geo, class F>
__device__ __forceinline__ void for_each_point(const Geo &geo, R bound, F &&f) {
  constexpr int DSG = 3 * Shape<ET>::NV;
  if constexpr (ET == TET) {
    R X[DSG];
    geo.fetch(X);
    R J[3][3];
    point_jacobian<TET, 0>(X, J);
    const PointData<TET, 0, R> pd(J, bound);  // w_q and J are the same at all 4 points
    static_for<4>([&](auto qc) {
      FEK_CI(Q, qc);
      f(std::integral_constant<int, Q>{}, pd);
    });
  } else {
    R J2[3][3];  // [t][i]
    R J01[2][3][2];  // [z][i][k]
    {
      R X[DSG];
      geo.fetch(X);
      static_for<3>([&](auto tc) {
        FEK_CI(t, tc);
#pragma unroll
        for (int i = 0; i < 3; ++i) J2[t][i] = jac_entry<PRISM, 2 * t, 2>(X, i);
      });
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        J01[0][i][0] = jac_entry<PRISM, 0, 0>(X, i);
        J01[0][i][1] = jac_entry<PRISM, 0, 1>(X, i);
        J01[1][i][0] = jac_entry<PRISM, 1, 0>(X, i);
        J01[1][i][1] = jac_entry<PRISM, 1, 1>(X, i);
      }
    }
    static_for<2>([&](auto zc) {
      FEK_CI(z, zc);
      static_for<3>([&](auto tc) {
        FEK_CI(t, tc);
        constexpr int Q = 2 * t + z;
        const R J[3][3] = {{J01[z][0][0], J01[z][0][1], J2[t][0]},
                           {J01[z][1][0], J01[z][1][1], J2[t][1]},
                           {J01[z][2][0], J01[z][2][1], J2[t][2]}};
        const PointData<PRISM, Q, R> pd(J, bound);
        f(std::integral_constant<int, Q>{}, pd);
      });
    });
  }
}

// ConvDiff t_s = vol * (C phi_s), phi_s = (val_s, g_s)
template <typename R>
__device__ __forceinline__ void cphi(const R *c, R val_s, const R (&g)[3], R vol, R (&t)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const R x = fma(c[4 * i + 1], g[0], fma(c[4 * i + 2], g[1], fma(c[4 * i + 3], g[2], c[4 * i] * val_s)));
    t[i] = vol * x;
  }
}

// acc + (val_r, g_r) . t, fused into the accumulator (4 FMA, no extra add)
template <typename R>
__device__ __forceinline__ R acc_dot4(R acc, R val_r, const R (&g)[3], const R (&t)[4]) {
  return fma(g[2], t[3], fma(g[1], t[2], fma(g[0], t[1], fma(val_r, t[0], acc))));
}

template <typename R>
__device__ __forceinline__ R load_term(const R *d, R val_r, const R (&g)[3]) {
  return fma(d[0], val_r, fma(d[1], g[0], fma(d[2], g[1], d[3] * g[2])));
}

// Source of the load coefficients d (ConvDiff).
template <typename R>
struct RegLoad {
  const R *d;
  __device__ __forceinline__ void fetch(R (&out)[4]) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = d[k];
  }
};

// ---------------------------------------------------------------------------
// prism ConvDiff (QSS, fp64 and fp32) in the reference frame, summed per zeta level.
//
// phi_s = (val_s, g_s) = P psi_s with psi_s = (val_s, ld_s) the reference
// 4-vector and P = diag(1, inv^T), so
//   A_rs = sum_q vol_q phi_r^T C phi_s = sum_q psi_r^T K_q psi_s,
//   K_q  = vol_q P^T C P = w [ det C00 , C0. adj^T ; adj C.0 , adj C.. adj^T / det ]
// (vol = w det and inv = adj / det: one reciprocal, no inverse).  The prism
// basis factors as psi_(a,b) = l_b(z) X_a(t) + l'_b Y_a(t) with
// X_a = (lam_a, dlam_a, 0), Y_a = (0, 0, 0, lam_a), l'_b = -+1/2
// (refelem.py:145-155), so per level z the four 3x3 sums over the triangle
// points
//   SXX = sum_t X^T K X,  SXY = sum_t lam_a' (X_a^T K_3),  SYX = sum_t lam_a (K^3 X_a'),
//   SYY = sum_q lam_a lam_a' K33 (same l'l' weight on both levels)
// carry everything, and A_(a,b)(a',b') = sum_z l_b l_b' SXX + l_b l'_b' SXY
// + l'_b l_b' SYX + l'_b l'_b' SYY is formed once at the end.  About 1500
// FP64 instructions per element instead of ~2300 for the physical-frame
// t_s = vol C phi_s, A_rs += phi_r . t_s loop; the load vector follows the
// same pattern with e = vol P^T d.  The Jacobian and its adjugate are the
// reference's (bitwise J, batched.py:193-207); only the contraction order
// differs, so results agree with the reference to rounding (~1e-15).
// ---------------------------------------------------------------------------

namespace prism_ref {
using S = Shape<PRISM>;
// lam_a at triangle point t (the +lam_a/2 zeta derivative of top shape a+3, doubled: exact)
__host__ __device__ constexpr double lam(int t, int a) { return 2.0 * S::ld(2 * t, a + 3, 2); }
// l_b at level z: the in-plane derivative of shape 1 (b = 0) / 4 (b = 1)
__host__ __device__ constexpr double ell(int z, int b) { return S::ld(z, b == 0 ? 1 : 4, 0); }
constexpr double dlx[3] = {-1.0, 1.0, 0.0}, dly[3] = {-1.0, 0.0, 1.0};
// packed upper triangle of a symmetric 3x3: (0,0) (0,1) (0,2) (1,1) (1,2) (2,2)
__host__ __device__ constexpr int sym_index(int a, int b) {
  return a <= b ? (a * (5 - a)) / 2 + b : (b * (5 - b)) / 2 + a;
}
static_assert(sym_index(0, 0) == 0 && sym_index(0, 2) == 2 && sym_index(1, 1) == 3 && sym_index(2, 1) == 4 &&
              sym_index(2, 2) == 5, "packed symmetric index");
__host__ __device__ constexpr double cabs(double x) { return x < 0 ? -x : x; }
__host__ __device__ constexpr bool structure_ok() {
  for (int t = 0; t < 3; ++t)
    for (int z = 0; z < 2; ++z) {
      const int q = 2 * t + z;
      if (S::w(q) != S::w(0)) return false;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 2; ++b) {
          const int s = a + 3 * b;
          const double l = ell(z, b), lp = b == 0 ? -0.5 : 0.5;
          if (S::ld(q, s, 0) != dlx[a] * l || S::ld(q, s, 1) != dly[a] * l) return false;
          if (S::ld(q, s, 2) != lp * lam(t, a)) return false;
          if (cabs(S::val(q, s) - lam(t, a) * l) > 1e-15) return false;
        }
    }
  return true;
}
static_assert(structure_ok(), "prism reference tables factor as lam_a(t) l_b(z)");

// acc (+)= X_a . (k0, k1, k2) with X_a = (lam, dlam_a): one FMA plus the +-1 terms
// s (+)= x * y; the first term of a sum is a plain product
template <bool FIRST, typename R>
__device__ __forceinline__ void mac(R &s, const R &x, const R &y) {
  if constexpr (FIRST) {
    s = x * y;
  } else {
    s = fma(x, y, s);
  }
}

template <int A_, bool FIRST, typename R>
__device__ __forceinline__ R xdot(const R &acc, const R &lam_a, const R &k0, const R &k1, const R &k2) {
  R r;
  if constexpr (FIRST) {
    r = lam_a * k0;
  } else {
    r = fma(lam_a, k0, acc);
  }
  if constexpr (A_ == 0) {
    r = r - k1;
    r = r - k2;
  } else if constexpr (A_ == 1) {
    r = r + k1;
  } else {
    r = r + k2;
  }
  return r;
}

// distinct Jacobian columns (for_each_point's reuse): J2[t][i] = J[i][2] at triangle point t,
// J01[z][i][k] = J[i][k] (k = 0, 1) on level z -- bitwise the reference's per-point J
template <typename R>
struct Cols {
  R J2[3][3];      // [t][i]
  R J01[2][3][2];  // [z][i][k]
};

template <typename R>
__device__ __forceinline__ void jacobian_columns(const R (&X)[18], R (&J2)[3][3], R (&J01)[2][3][2]) {
  static_for<3>([&](auto tc) {
    FEK_CI(t, tc);
#pragma unroll
    for (int i = 0; i < 3; ++i) J2[t][i] = jac_entry<PRISM, 2 * t, 2>(X, i);
  });
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    J01[0][i][0] = jac_entry<PRISM, 0, 0>(X, i);
    J01[0][i][1] = jac_entry<PRISM, 0, 1>(X, i);
    J01[1][i][0] = jac_entry<PRISM, 1, 0>(X, i);
    J01[1][i][1] = jac_entry<PRISM, 1, 1>(X, i);
  }
}

// adjugate (adj[k][i] = det * d xi_k / d x_i) and determinant of J = [J01 | J2], invert3's operations
template <typename R>
__device__ __forceinline__ R adjugate(const R (&J01)[3][2], const R (&J2)[3], R (&adj)[3][3]) {
  // (also instantiated for fp32 pairs, where -(x * y) is a packed negation)
  const R a_ = J01[0][0], b_ = J01[0][1], c_ = J2[0];
  const R d_ = J01[1][0], e_ = J01[1][1], f_ = J2[1];
  const R g_ = J01[2][0], h_ = J01[2][1], i_ = J2[2];
  adj[0][0] = fma(e_, i_, -(f_ * h_));
  adj[1][0] = fma(f_, g_, -(d_ * i_));
  adj[2][0] = fma(d_, h_, -(e_ * g_));
  const R det = fma(a_, adj[0][0], fma(b_, adj[1][0], c_ * adj[2][0]));
  adj[0][1] = fma(c_, h_, -(b_ * i_));
  adj[0][2] = fma(b_, f_, -(c_ * e_));
  adj[1][1] = fma(a_, i_, -(c_ * g_));
  adj[1][2] = fma(c_, d_, -(a_ * f_));
  adj[2][1] = fma(b_, g_, -(a_ * h_));
  adj[2][2] = fma(a_, e_, -(b_ * d_));
  return det;
}
}  // namespace prism_ref

// Two fp32 lanes on sm_100's packed FFMA2 / FMUL2 / FADD2: the fp32 prism
// kernel runs both zeta levels of a triangle point as one pair (the per-point
// work is identical on the two levels, with the same compile-time constants).
struct f2 {
  float2 v;
  __device__ __forceinline__ f2() {}
  __device__ __forceinline__ f2(float x) : v(make_float2(x, x)) {}
  __device__ __forceinline__ f2(float x, float y) : v(make_float2(x, y)) {}
  __device__ __forceinline__ explicit f2(float2 p) : v(p) {}
};
__device__ __forceinline__ f2 operator*(f2 a, f2 b) { return f2(__fmul2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 operator+(f2 a, f2 b) { return f2(__fadd2_rn(a.v, b.v)); }
__device__ __forceinline__ f2 operator-(f2 a) { return f2(make_float2(-a.v.x, -a.v.y)); }
__device__ __forceinline__ f2 operator-(f2 a, f2 b) { return f2(__ffma2_rn(b.v, make_float2(-1.f, -1.f), a.v)); }
__device__ __forceinline__ f2 fma(f2 a, f2 b, f2 c) { return f2(__ffma2_rn(a.v, b.v, c.v)); }
using ::fma;  // keep the scalar overloads visible next to the pair one

namespace prism_ref {
template <typename V>
struct Lanes;  // per-level view of a value: scalar (one level) or pair (both levels)
template <>
struct Lanes<double> {
  static constexpr int NZ = 2;  // levels looped
  __device__ static double get(double x, int) { return x; }
};
template <>
struct Lanes<float> {
  static constexpr int NZ = 2;
  __device__ static float get(float x, int) { return x; }
};
template <>
struct Lanes<f2> {
  static constexpr int NZ = 1;  // both levels in one pass
  __device__ static float get(f2 x, int lane) { return lane ? x.v.y : x.v.x; }
};

// classify_fast as bitmasks: returns the det < 0 bit, marks |det| <= bound as near
__device__ __forceinline__ unsigned kind_bits(double det, double bound, int q, unsigned &near) {
  near |= static_cast<unsigned>(fabs(det) <= bound) << q;
  return static_cast<unsigned>(det < 0.0) << q;
}
__device__ __forceinline__ unsigned kind_bits(float det, float bound, int q, unsigned &near) {
  near |= static_cast<unsigned>(fabsf(det) <= bound) << q;
  return static_cast<unsigned>(det < 0.0f) << q;
}
// pair: lane x is level 0 (point q), lane y level 1 (point q + 1)
__device__ __forceinline__ unsigned kind_bits(f2 det, float bound, int q, unsigned &near) {
  return kind_bits(det.v.x, bound, q, near) | kind_bits(det.v.y, bound, q + 1, near);
}
__device__ __forceinline__ double vrecip(double x) { return recip(x); }
__device__ __forceinline__ float vrecip(float x) { return recip(x); }
__device__ __forceinline__ f2 vrecip(f2 x) { return f2(recip(x.v.x), recip(x.v.y)); }
}  // namespace prism_ref

template <typename R, class Coef>
__device__ __forceinline__ void integrate_prism_cd_ref(const prism_ref::Cols<R> &cols, const Coef &c, R bound,
                                                       R (&A)[36], R (&B)[6], unsigned &fail_mask,
                                                       unsigned &near_mask) {
  using namespace prism_ref;
  // fp64: one level per pass (scalar); fp32: both levels per pass (FFMA2 pairs)
  using V = std::conditional_t<sizeof(R) == 8, R, f2>;
  constexpr int NZ = Lanes<V>::NZ;
  constexpr double w = S::w(0);
  // coefficient row: c00 .. c33, d0 .. d3 (problems.py:136-140)
  auto cv = [&](int k) { return V(c[k]); };
  auto d = [&](int k) { return V(c[16 + k]); };
  const auto &J2 = cols.J2;
  const auto &J01 = cols.J01;
  // per-pass sums [pass]; SYY / SbY carry the same weight on both levels
  V SXX[NZ][3][3], SXY[NZ][3][3], SYX[NZ][3][3], SbX[NZ][3];
  V SYY[6], SbY[3];
  static_for<NZ>([&](auto zc) {
    FEK_CI(z, zc);
    // J columns 0/1 of this pass (pairs: (level 0, level 1))
    V Jz[3][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if constexpr (NZ == 2) {
          Jz[i][k] = V(J01[z][i][k]);
        } else {
          Jz[i][k] = V(J01[0][i][k], J01[1][i][k]);
        }
      }
    static_for<3>([&](auto tc) {
      FEK_CI(t, tc);
      constexpr int Q = 2 * t + z;           // pairs: lane x = q, lane y = q + 1
      constexpr bool F = (t == 0);           // first point of the pass
      constexpr bool F2 = (t == 0 && z == 0);  // first point overall
      const V Jt[3] = {V(J2[t][0]), V(J2[t][1]), V(J2[t][2])};
      V adj[3][3];
      const V det = adjugate(Jz, Jt, adj);
      fail_mask |= kind_bits(det, bound, Q, near_mask);
      const V rdet = vrecip(det);
      // K (w folded into the final weights): K00 = det c00, K0l = c0. adj_l, Kk0 = adj_k c.0,
      // Kkl = adj_k C adj_l^T / det
      V K[4][4];
      K[0][0] = det * cv(0);
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        K[0][1 + l] = fma(cv(1), adj[l][0], fma(cv(2), adj[l][1], cv(3) * adj[l][2]));
        K[1 + l][0] = fma(adj[l][0], cv(4), fma(adj[l][1], cv(8), adj[l][2] * cv(12)));
      }
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        V M[3];  // M[i] = sum_j C[1+i][1+j] adj[l][j]
#pragma unroll
        for (int i = 0; i < 3; ++i)
          M[i] = fma(cv(4 * (1 + i) + 1), adj[l][0], fma(cv(4 * (1 + i) + 2), adj[l][1], cv(4 * (1 + i) + 3) * adj[l][2]));
#pragma unroll
        for (int k = 0; k < 3; ++k) K[1 + k][1 + l] = rdet * fma(adj[k][0], M[0], fma(adj[k][1], M[1], adj[k][2] * M[2]));
      }
      const V L[3] = {V(R(lam(t, 0))), V(R(lam(t, 1))), V(R(lam(t, 2)))};
      // XX: v_a' = K[0:3][0:3] X_a', then SXX[a][a'] (+)= X_a . v_a'
      static_for<3>([&](auto apc) {
        FEK_CI(ap, apc);
        V v[3];
#pragma unroll
        for (int al = 0; al < 3; ++al) v[al] = xdot<ap, true>(V(R(0)), L[ap], K[al][0], K[al][1], K[al][2]);
        static_for<3>([&](auto ac) {
          FEK_CI(a, ac);
          SXX[z][a][ap] = xdot<a, F>(SXX[z][a][ap], L[a], v[0], v[1], v[2]);
        });
      });
      // XY / YX / YY
      static_for<3>([&](auto ac) {
        FEK_CI(a, ac);
        const V p = xdot<a, true>(V(R(0)), L[a], K[0][3], K[1][3], K[2][3]);  // X_a . K[:,3]
        const V q = xdot<a, true>(V(R(0)), L[a], K[3][0], K[3][1], K[3][2]);  // K[3,:] . X_a
        static_for<3>([&](auto bc) {
          FEK_CI(ap, bc);
          mac<F>(SXY[z][a][ap], L[ap], p);
          mac<F>(SYX[z][ap][a], L[ap], q);
        });
      });
      static_for<3>([&](auto ac) {
        FEK_CI(a, ac);
        static_for<3>([&](auto bc) {
          FEK_CI(ap, bc);
          if constexpr (ap >= a) mac<F2>(SYY[sym_index(a, ap)], V(R(lam(t, a) * lam(t, ap))), K[3][3]);
        });
      });
      // load: e = vol P^T d / w = (det d0, adj d[1:4])
      const V e0 = det * d(0);
      V e[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) e[k] = fma(adj[k][0], d(1), fma(adj[k][1], d(2), adj[k][2] * d(3)));
      static_for<3>([&](auto ac) {
        FEK_CI(a, ac);
        SbX[z][a] = xdot<a, F>(SbX[z][a], L[a], e0, e[0], e[1]);
        mac<F2>(SbY[a], L[a], e[2]);
      });
    });
  });
  // per-level views of the sums (pairs: lane = level)
  auto lv = [&](const V &x, int z) -> R { return Lanes<V>::get(x, NZ == 2 ? 0 : z); };
  auto both = [&](const V &x) -> R {
    if constexpr (NZ == 2) {
      return x;
    } else {
      return x.v.x + x.v.y;
    }
  };
  // A_(a,b)(a',b') = w sum_z [l_b l_b' SXX + l_b l'_b' SXY + l'_b l_b' SYX] + w l'_b l'_b' SYY
  static_for<3>([&](auto ac) {
    FEK_CI(a, ac);
    static_for<3>([&](auto bc) {
      FEK_CI(ap, bc);
      constexpr int kyy = sym_index(a, ap);
      const R syy = both(SYY[kyy]);
      static_for<2>([&](auto b1c) {
        FEK_CI(b, b1c);
        static_for<2>([&](auto b2c) {
          FEK_CI(bp, b2c);
          constexpr double lpb = b == 0 ? -0.5 : 0.5, lpbp = bp == 0 ? -0.5 : 0.5;
          R acc = R(w * lpb * lpbp) * syy;
          static_for<2>([&](auto zc) {
            FEK_CI(z, zc);
            constexpr int zi = NZ == 2 ? z : 0;
            constexpr double lb = ell(z, b), lbp = ell(z, bp);
            acc = fma(R(w * lb * lbp), lv(SXX[zi][a][ap], z), acc);
            acc = fma(R(w * lb * lpbp), lv(SXY[zi][a][ap], z), acc);
            acc = fma(R(w * lpb * lbp), lv(SYX[zi][a][ap], z), acc);
          });
          A[6 * (a + 3 * b) + (ap + 3 * bp)] = acc;
        });
      });
    });
    const R sby = both(SbY[a]);
    static_for<2>([&](auto b1c) {
      FEK_CI(b, b1c);
      constexpr double lpb = b == 0 ? -0.5 : 0.5;
      R acc = R(w * lpb) * sby;
      static_for<2>([&](auto zc) {
        FEK_CI(z, zc);
        constexpr int zi = NZ == 2 ? z : 0;
        acc = fma(R(w * ell(z, b)), lv(SbX[zi][a], z), acc);
      });
      B[a + 3 * b] = acc;
    });
  });
}

// Prism Poisson (QSS) in the reference frame.  C = diag(0, I), so only the
// symmetric derivative block of K survives: K = (w / det) adj adj^T.  With
// psi_(a,b) = l_b (0, dlam_a, 0) + l'_b (0, 0, 0, lam_a):
//   XX = dlam^T K2 dlam with K2 the (xi, eta) block -- dlam is point
//   independent, so only sum_t K2 (3 numbers per level) is accumulated;
//   XY[a][a'] = lam_a' (dlam_a . K[xi eta][zeta]) (YX = XY^T, K symmetric);
//   YY[a][a'] = lam_a lam_a' K[zeta][zeta].
// Load: b_(a,b) = w sum_z l_b(z) sum_t lam_a(t) det_q d0[q].
// 706 FP64 instructions per element instead of 1120 (fp32: both levels as FFMA2 pairs).
template <typename R>
__device__ __forceinline__ void integrate_prism_poisson_ref(const prism_ref::Cols<R> &cols, const R *d0, R bound,
                                                            R (&A)[36], R (&B)[6], unsigned &fail_mask,
                                                            unsigned &near_mask) {
  using namespace prism_ref;
  // fp64: one level per pass; fp32: both levels per pass on FFMA2 pairs (as integrate_prism_cd_ref)
  using V = std::conditional_t<sizeof(R) == 8, R, f2>;
  constexpr int NZ = Lanes<V>::NZ;
  constexpr double w = S::w(0);
  const auto &J2 = cols.J2;
  const auto &J01 = cols.J01;
  V SK[NZ][3];      // sum_t (k00, k01, k11) of the (xi, eta) block, per pass
  V SXY[NZ][2][3];  // [z][a-1][a'] = sum_t lam_a'(t) p_a, p_1 = k02, p_2 = k12 (p_0 = -p_1 - p_2)
  V SYY[6];         // sum_q lam_a lam_a' k22 (packed symmetric)
  V SB[NZ][3];      // sum_t lam_a(t) det d0[q], per pass
  static_for<NZ>([&](auto zc) {
    FEK_CI(z, zc);
    V Jz[3][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if constexpr (NZ == 2) {
          Jz[i][k] = V(J01[z][i][k]);
        } else {
          Jz[i][k] = V(J01[0][i][k], J01[1][i][k]);
        }
      }
    static_for<3>([&](auto tc) {
      FEK_CI(t, tc);
      constexpr int Q = 2 * t + z;  // pairs: lane x = q, lane y = q + 1
      constexpr bool F = (t == 0);
      constexpr bool F2 = (t == 0 && z == 0);
      const V Jt[3] = {V(J2[t][0]), V(J2[t][1]), V(J2[t][2])};
      V adj[3][3];
      const V det = adjugate(Jz, Jt, adj);
      fail_mask |= kind_bits(det, bound, Q, near_mask);
      const V rdet = vrecip(det);
      auto kdot = [&](int k, int l) {
        return rdet * fma(adj[k][0], adj[l][0], fma(adj[k][1], adj[l][1], adj[k][2] * adj[l][2]));
      };
      const V k00 = kdot(0, 0), k01 = kdot(0, 1), k11 = kdot(1, 1);
      const V k02 = kdot(0, 2), k12 = kdot(1, 2), k22 = kdot(2, 2);
      if constexpr (F) {
        SK[z][0] = k00;
        SK[z][1] = k01;
        SK[z][2] = k11;
      } else {
        SK[z][0] = SK[z][0] + k00;
        SK[z][1] = SK[z][1] + k01;
        SK[z][2] = SK[z][2] + k11;
      }
      V dq;
      if constexpr (NZ == 2) {
        dq = det * V(d0[Q]);
      } else {
        dq = det * V(d0[Q], d0[Q + 1]);
      }
      static_for<3>([&](auto ac) {
        FEK_CI(a, ac);
        const V la = V(R(lam(t, a)));
        mac<F>(SXY[z][0][a], la, k02);
        mac<F>(SXY[z][1][a], la, k12);
        mac<F>(SB[z][a], la, dq);
        static_for<3>([&](auto bc) {
          FEK_CI(ap, bc);
          if constexpr (ap >= a) mac<F2>(SYY[sym_index(a, ap)], V(R(lam(t, a) * lam(t, ap))), k22);
        });
      });
    });
  });
  auto lv = [&](const V &x, int z) -> R { return Lanes<V>::get(x, NZ == 2 ? 0 : z); };
  // XX[a][a'] per level from the K2 sums (dlam = (-1,-1), (1,0), (0,1))
  R XX[2][6];
  R XY[2][3][3];
  static_for<2>([&](auto zc) {
    FEK_CI(z, zc);
    constexpr int zi = NZ == 2 ? z : 0;
    const R k00 = lv(SK[zi][0], z), k01 = lv(SK[zi][1], z), k11 = lv(SK[zi][2], z);
    const R s0 = k00 + k01, s1 = k01 + k11;
    XX[z][sym_index(1, 1)] = k00;
    XX[z][sym_index(1, 2)] = k01;
    XX[z][sym_index(2, 2)] = k11;
    XX[z][sym_index(0, 1)] = -s0;
    XX[z][sym_index(0, 2)] = -s1;
    XX[z][sym_index(0, 0)] = s0 + s1;
#pragma unroll
    for (int ap = 0; ap < 3; ++ap) {
      const R p1 = lv(SXY[zi][0][ap], z), p2 = lv(SXY[zi][1][ap], z);
      XY[z][1][ap] = p1;
      XY[z][2][ap] = p2;
      XY[z][0][ap] = -(p1 + p2);
    }
  });
  R syy[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if constexpr (NZ == 2) {
      syy[k] = SYY[k];
    } else {
      syy[k] = SYY[k].v.x + SYY[k].v.y;
    }
  }
  // A_(a,b)(a',b') = w sum_z [l_b l_b' XX + l_b l'_b' XY[a][a'] + l'_b l_b' XY[a'][a]] + w l'_b l'_b' SYY
  static_for<3>([&](auto ac) {
    FEK_CI(a, ac);
    static_for<3>([&](auto bc) {
      FEK_CI(ap, bc);
      static_for<2>([&](auto b1c) {
        FEK_CI(b, b1c);
        static_for<2>([&](auto b2c) {
          FEK_CI(bp, b2c);
          constexpr int r = a + 3 * b, s_ = ap + 3 * bp;
          if constexpr (s_ >= r) {
            constexpr double lpb = b == 0 ? -0.5 : 0.5, lpbp = bp == 0 ? -0.5 : 0.5;
            R acc = R(w * lpb * lpbp) * syy[sym_index(a, ap)];
            static_for<2>([&](auto zc) {
              FEK_CI(z, zc);
              constexpr double lb = ell(z, b), lbp = ell(z, bp);
              acc = fma(R(w * lb * lbp), XX[z][sym_index(a, ap)], acc);
              acc = fma(R(w * lb * lpbp), XY[z][a][ap], acc);
              acc = fma(R(w * lpb * lbp), XY[z][ap][a], acc);
            });
            A[6 * r + s_] = acc;
            A[6 * s_ + r] = acc;
          }
        });
      });
    });
    static_for<2>([&](auto b1c) {
      FEK_CI(b, b1c);
      R acc = R(w * ell(0, b)) * lv(SB[0][a], 0);
      B[a + 3 * b] = fma(R(w * ell(1, b)), lv(SB[NZ == 2 ? 1 : 0][a], 1), acc);
    });
  });
}

// ---------------------------------------------------------------------------
// prism ConvDiff fp64 (QSS) split over a LANE PAIR by zeta level.
//
// integrate_prism_cd_ref's per-level sums SXX/SXY/SYX/SbX depend only on that level's Jacobian
// columns 0/1 (6 entries) and the shared column-2 entries J2 (9), so lane z of a pair runs the
// three points of level z alone -- no point work is duplicated, only the 9 J2 entries and the
// degeneracy bound.  Each lane then forms, from its own sums, its level's contribution to all 36
// stiffness entries (and 6 load entries), sends the partner the half belonging to the partner's
// row block (rows b = 1 - z: 18 + 3 doubles over __shfl_xor) and adds the half it receives: lane z
// owns rows a + 3z.  Half the accumulators per thread (39 instead of 78 live sums) lets two CTAs
// of 256 threads (16 warps/SM) run at <= 128 registers where the one-thread kernel holds 8 warps
// at 255 registers + spill.  Both lanes execute one instruction stream: level-dependent constants
// are selected once per thread, and J01 is formed with the reference's rounding (the level's
// _axpy_fixed coefficients differ only in value, never in zero/+-1 pattern).
// ---------------------------------------------------------------------------

namespace prism_pair {
using prism_ref::S;
using prism_ref::lam;
using prism_ref::ell;
using prism_ref::sym_index;

// sum_v c_v x_v with the reference's _axpy_fixed rounding for coefficients c_v = C(v) (all nonzero,
// none +-1: products rounded, summed left to right); `x(v)` / `C(v)` may select at run time
template <typename R, int NV, class Cf, class Xf>
__device__ __forceinline__ R axpy_exact(Cf &&C, Xf &&x) {
  R acc = C(std::integral_constant<int, 0>{}) * x(0);
  static_for<NV - 1>([&](auto vc) {
    constexpr int v = decltype(vc)::value + 1;
    acc = acc + C(std::integral_constant<int, v>{}) * x(v);
  });
  return acc;
}

// The pair's shared geometry, split between the two lanes (both lanes end with all of it):
//  * bound2, the SQUARED near bound: (NEAR_TOL_FACTOR 1e-14)^2 D2^3 with D2 = 4 sum_v |X_v - X_0|^2.
//    The near test only needs a bound >= 1.4 tol (classify_fast: |det - det_ref| <= 0.4 tol), and
//    span_i <= 2 max_v |X_v,i - X_0,i| gives D2 >= diag^2, so this is >= (16 tol)^2 -- no min/max
//    (DSETP + 2 FSEL each), no sqrt, no cube: lane z sums coordinate dimension z over the five
//    vertices plus dimension 2 over vertices {1,2,3} (z = 0) or {4,5} (z = 1), one shuffle adds
//    the halves.  (Valid elements have det^2 ~ 1e26 bound2, so it never flags them.)
//  * J2[t][i] = sum_v ld[2t][v][2] X[v][i] (coefficients -+lam_a(t)/2, never 0 or +-1): lane z
//    forms triangle point t = z and J2[2][z], both form J2[2][2], the other four arrive by shuffle;
//  * this level's J01[i][k] = sum_v ld[z][v][k] X[v][i]: the level coefficients +-l_b(z) differ
//    from the other level's only in value (same zero / sign pattern), selected at run time.
// All entries are bitwise the reference's (jac_entry<PRISM, q, k> / degeneracy_tolerance).
template <typename R>
__device__ __forceinline__ void level_geometry(const R (&X)[18], int z, R &bound, R (&J2)[3][3], R (&J01)[3][2]) {
  // (`bound` receives the squared near bound, bound2)
  constexpr unsigned FULL = 0xffffffffu;
  // -- squared near bound
  R part = R(0);
  {
    const R x0 = z ? X[1] : X[0];
#pragma unroll
    for (int v = 1; v < 6; ++v) {
      const R d = (z ? X[3 * v + 1] : X[3 * v]) - x0;
      part = fma(d, d, part);
    }
    // dimension 2: vertices 1, 2, 3 on lane 0; 4, 5 (and vertex 0 itself, d = 0) on lane 1
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const R d = (z ? X[3 * (k == 2 ? 0 : 4 + k) + 2] : X[3 * (1 + k) + 2]) - X[2];
      part = fma(d, d, part);
    }
  }
  const R d2 = R(4) * (part + __shfl_xor_sync(FULL, part, 1));
  bound = R(NEAR_TOL_FACTOR * NEAR_TOL_FACTOR * 1e-28) * ((d2 * d2) * d2);
  // -- zeta column at the triangle points
  R own[3];  // J2[z][i]
#pragma unroll
  for (int i = 0; i < 3; ++i)
    own[i] = axpy_exact<R, 6>([&](auto vc) { FEK_CI(v, vc); return z ? R(S::ld(2, v, 2)) : R(S::ld(0, v, 2)); },
                              [&](int v) { return X[3 * v + i]; });
  const R j2z = axpy_exact<R, 6>([&](auto vc) { FEK_CI(v, vc); return R(S::ld(4, v, 2)); },
                                 [&](int v) { return z ? X[3 * v + 1] : X[3 * v]; });  // J2[2][z]
  J2[2][2] = axpy_exact<R, 6>([&](auto vc) { FEK_CI(v, vc); return R(S::ld(4, v, 2)); },
                              [&](int v) { return X[3 * v + 2]; });
  const R j2o = __shfl_xor_sync(FULL, j2z, 1);
  J2[2][0] = z ? j2o : j2z;
  J2[2][1] = z ? j2z : j2o;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const R other = __shfl_xor_sync(FULL, own[i], 1);
    J2[0][i] = z ? other : own[i];
    J2[1][i] = z ? own[i] : other;
  }
  // -- this level's columns 0/1
  const R lo = z ? R(ell(1, 0)) : R(ell(0, 0));  // bottom-face factor l_0(z)
  const R hi = z ? R(ell(1, 1)) : R(ell(0, 1));  // top-face factor l_1(z)
  static_for<2>([&](auto kc) {
    FEK_CI(k, kc);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      R acc = R(0);
      bool any = false;
      static_for<6>([&](auto vc) {
        FEK_CI(v, vc);
        constexpr double c0 = S::ld(0, v, k), c1 = S::ld(1, v, k);
        constexpr double sgn = (k == 0 ? prism_ref::dlx : prism_ref::dly)[v % 3];
        static_assert((c0 == 0.0) == (sgn == 0.0) && (c1 == 0.0) == (sgn == 0.0), "level zero pattern");
        static_assert(c0 == sgn * ell(0, v / 3) && c1 == sgn * ell(1, v / 3), "level coefficients");
        static_assert(c0 != 1.0 && c0 != -1.0 && c1 != 1.0 && c1 != -1.0, "no unit coefficients");
        if constexpr (sgn != 0.0) {
          const R m = (v < 3 ? lo : hi) * X[3 * v + i];  // (+-l) * x rounds like +-(l * x)
          if (!any) {
            acc = sgn > 0 ? m : -m;
            any = true;
          } else {
            acc = sgn > 0 ? acc + m : acc - m;
          }
        }
      });
      J01[i][k] = acc;
    }
  });
}
static_assert(S::ld(2, 0, 2) != 0.0 && S::ld(0, 0, 2) != 0.0 && S::ld(4, 0, 2) != 0.0, "zeta column coefficients");

template <typename R>
__device__ __forceinline__ void integrate_cd_level(const R (&J2)[3][3], const R (&J01)[3][2], const R (&c)[20],
                                                   R bound2, int z, R (&Ah)[18], R (&Bh)[3], int &kind,
                                                   int &kind_point) {
  using prism_ref::mac;
  using prism_ref::xdot;
  constexpr double w = S::w(0);
  // w folded into K and the load terms once per element (K' = w K, e' = w e); the zeta-derivative
  // factor l'_b = -+1/2 folded into the accumulation constants of SXY / SYX / SYY / SbY
  const R wc00 = R(w) * c[0];
  const R wc0[3] = {R(w) * c[1], R(w) * c[2], R(w) * c[3]};
  const R wcc[3] = {R(w) * c[4], R(w) * c[8], R(w) * c[12]};
  const R wd[4] = {R(w) * c[16], R(w) * c[17], R(w) * c[18], R(w) * c[19]};
  R SXX[3][3], SXY[3][3], SYX[3][3], SbX[3], SYY[6], SbY[3];
  unsigned fail_mask = 0, near_mask = 0;
  static_for<3>([&](auto tc) {
    FEK_CI(t, tc);
    constexpr bool F = (t == 0);
    const R Jt[3] = {J2[t][0], J2[t][1], J2[t][2]};
    R adj[3][3];
    const R det = prism_ref::adjugate(J01, Jt, adj);
    near_mask |= static_cast<unsigned>(det * det <= bound2) << (2 * t + z);  // squared near bound
    fail_mask |= static_cast<unsigned>(det < R(0)) << (2 * t + z);
    const R rdet = R(w) * recip(det);
    R K[4][4];
    K[0][0] = det * wc00;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      K[0][1 + l] = fma(wc0[0], adj[l][0], fma(wc0[1], adj[l][1], wc0[2] * adj[l][2]));
      K[1 + l][0] = fma(adj[l][0], wcc[0], fma(adj[l][1], wcc[1], adj[l][2] * wcc[2]));
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      R M[3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
        M[i] = fma(c[4 * (1 + i) + 1], adj[l][0], fma(c[4 * (1 + i) + 2], adj[l][1], c[4 * (1 + i) + 3] * adj[l][2]));
#pragma unroll
      for (int k = 0; k < 3; ++k) K[1 + k][1 + l] = rdet * fma(adj[k][0], M[0], fma(adj[k][1], M[1], adj[k][2] * M[2]));
    }
    const R L[3] = {R(lam(t, 0)), R(lam(t, 1)), R(lam(t, 2))};
    // X_0 = (lam_0, -1, -1): its products need k1 + k2, formed once and shared (fused: one
    // FMA instead of a product and two subtractions)
    auto x0dot = [&](const R &k0, const R &k1, const R &k2) { return fma(L[0], k0, -(k1 + k2)); };
    static_for<3>([&](auto apc) {
      FEK_CI(ap, apc);
      R v[3];
#pragma unroll
      for (int al = 0; al < 3; ++al)
        v[al] = ap == 0 ? x0dot(K[al][0], K[al][1], K[al][2]) : xdot<ap, true>(R(0), L[ap], K[al][0], K[al][1], K[al][2]);
      static_for<3>([&](auto ac) {
        FEK_CI(a, ac);
        if constexpr (F && a == 0) {
          SXX[a][ap] = x0dot(v[0], v[1], v[2]);
        } else {
          SXX[a][ap] = xdot<a, F>(SXX[a][ap], L[a], v[0], v[1], v[2]);
        }
      });
    });
    static_for<3>([&](auto ac) {
      FEK_CI(a, ac);
      const R p = a == 0 ? x0dot(K[0][3], K[1][3], K[2][3]) : xdot<a, true>(R(0), L[a], K[0][3], K[1][3], K[2][3]);
      const R q = a == 0 ? x0dot(K[3][0], K[3][1], K[3][2]) : xdot<a, true>(R(0), L[a], K[3][0], K[3][1], K[3][2]);
      static_for<3>([&](auto bc) {
        FEK_CI(ap, bc);
        mac<F>(SXY[a][ap], R(0.5 * lam(t, ap)), p);   // SXY / 2
        mac<F>(SYX[ap][a], R(0.5 * lam(t, ap)), q);   // SYX / 2
      });
    });
    static_for<3>([&](auto ac) {
      FEK_CI(a, ac);
      static_for<3>([&](auto bc) {
        FEK_CI(ap, bc);
        if constexpr (ap >= a) mac<F>(SYY[sym_index(a, ap)], R(0.25 * lam(t, a) * lam(t, ap)), K[3][3]);  // SYY / 4
      });
    });
    const R e0 = det * wd[0];
    R e[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) e[k] = fma(adj[k][0], wd[1], fma(adj[k][1], wd[2], adj[k][2] * wd[3]));
    static_for<3>([&](auto ac) {
      FEK_CI(a, ac);
      if constexpr (F && a == 0) {
        SbX[a] = x0dot(e0, e[0], e[1]);
      } else {
        SbX[a] = xdot<a, F>(SbX[a], L[a], e0, e[0], e[1]);
      }
      mac<F>(SbY[a], R(0.5 * lam(t, a)), e[2]);                        // SbY / 2
    });
  });
  // the element's classification: both levels' points (lane z holds q = 2t + z)
  fail_mask |= __shfl_xor_sync(0xffffffffu, fail_mask, 1);
  near_mask |= __shfl_xor_sync(0xffffffffu, near_mask, 1);
  first_failure(fail_mask, near_mask, kind, kind_point);

  // this level's share of A_(a,b)(a',b') = sum_z [l_b l_b' SXX + l_b l'_b' SXY + l'_b l_b' SYX]
  // + l'_b l'_b' SYY (w already in K) and of b_(a,b) = sum_z l_b SbX + l'_b SbY, for the own row
  // block b = z (l_b(z) = ell(z, z)) and the partner's b = 1 - z (ell(z, 1 - z)); with the
  // halves folded in, l'_b' terms are +-1 (compile-time signs) and l'_b = s (s = -1, +1 for b = 0, 1)
  static_assert(ell(0, 0) == ell(1, 1) && ell(0, 1) == ell(1, 0), "level factors swap between the levels");
  // l'_own / (1/2) = -1, +1 for z = 0, 1: applied as a sign-bit flip on the ALU, not a DMUL
  const unsigned long long sflip = z ? 0ull : 0x8000000000000000ull;
  auto sgn_times = [&](R v) { return __longlong_as_double(static_cast<long long>(__double_as_longlong(v) ^ sflip)); };
  const R lcol[2] = {z ? R(ell(1, 0)) : R(ell(0, 0)), z ? R(ell(1, 1)) : R(ell(0, 1))};  // l_b'(z)
  constexpr double l_own = ell(0, 0), l_oth = ell(0, 1);
  R Po[18], Bo[3];  // the partner's row block: sent
  static_for<3>([&](auto ac) {
    FEK_CI(a, ac);
    static_for<3>([&](auto bc) {
      FEK_CI(ap, bc);
      const R syy = SYY[sym_index(a, ap)];
      static_for<2>([&](auto b2c) {
        FEK_CI(bp, b2c);
        const R u = bp ? fma(lcol[bp], SXX[a][ap], SXY[a][ap]) : fma(lcol[bp], SXX[a][ap], -SXY[a][ap]);
        const R v = bp ? fma(lcol[bp], SYX[a][ap], syy) : fma(lcol[bp], SYX[a][ap], -syy);
        const R sv = sgn_times(v);
        Ah[6 * a + ap + 3 * bp] = fma(R(l_own), u, sv);
        Po[6 * a + ap + 3 * bp] = fma(R(l_oth), u, -sv);
      });
    });
    const R sb = sgn_times(SbY[a]);
    Bh[a] = fma(R(l_own), SbX[a], sb);
    Bo[a] = fma(R(l_oth), SbX[a], -sb);
  });
#pragma unroll
  for (int j = 0; j < 18; ++j) Ah[j] = Ah[j] + __shfl_xor_sync(0xffffffffu, Po[j], 1);
#pragma unroll
  for (int j = 0; j < 3; ++j) Bh[j] = Bh[j] + __shfl_xor_sync(0xffffffffu, Bo[j], 1);
}
}  // namespace prism_pair

// QSS prism kernels from the element's distinct Jacobian columns (computed by
// the caller, so the input stage can be released before the math starts)
template <typename R, int PB, class Coef>
__device__ __forceinline__ void integrate_prism_qss(const prism_ref::Cols<R> &cols, const Coef &coef, R bound,
                                                    R (&A)[36], R (&B)[6], int &kind, int &kind_point) {
  unsigned fail_mask = 0, near_mask = 0;
  if constexpr (PB == POISSON) {
    integrate_prism_poisson_ref<R>(cols, coef, bound, A, B, fail_mask, near_mask);
  } else {
    integrate_prism_cd_ref<R>(cols, coef, bound, A, B, fail_mask, near_mask);
  }
  first_failure(fail_mask, near_mask, kind, kind_point);
}

template <typename R, int ET, int PB, int VAR, class Geo, class Load>
__device__ __forceinline__ void integrate_generic(const Geo &geo, const R *coef, const Load &load, R bound,
                                                  R (&A)[Shape<ET>::NS * Shape<ET>::NS],
                                                  R (&B)[Shape<ET>::NS], int &kind, int &kind_point) {
  using S = Shape<ET>;
  constexpr int NS = S::NS, NQ = S::NQ, DSG = 3 * S::NV;
  constexpr bool SYM = (PB == POISSON);
  // failing points as bitmasks (branch-free); the reported point is the
  // SMALLEST failing q, as in the reference (q = 0, 1, ... checked in order;
  // prism points are visited zeta-major here)
  unsigned fail_mask = 0, near_mask = 0;
  auto note = [&](int k, int q) {
    fail_mask |= static_cast<unsigned>(k == KIND_INVERTED) << q;
    near_mask |= static_cast<unsigned>(k == KIND_NEAR) << q;
  };
#pragma unroll
  for (int i = 0; i < NS * NS; ++i) A[i] = R(0);
#pragma unroll
  for (int i = 0; i < NS; ++i) B[i] = R(0);

  if constexpr (VAR == QSS && ET == PRISM) {
    prism_ref::Cols<R> cols;
    {
      R X[DSG];
      geo.fetch(X);
      prism_ref::jacobian_columns(X, cols.J2, cols.J01);
    }
    if constexpr (SYM) {
      integrate_prism_poisson_ref<R>(cols, coef, bound, A, B, fail_mask, near_mask);
    } else {
      integrate_prism_cd_ref<R>(cols, coef, bound, A, B, fail_mask, near_mask);
    }
  } else if constexpr (VAR == QSS) {
    for_each_point<R, ET>(geo, bound, [&](auto qc, const auto &pd) {
      FEK_CI(Q, qc);
      note(pd.kind, Q);
      R g[NS][3];
      all_grads<ET, Q>(pd.jac, g);
      if constexpr (SYM) {
        static_for<NS>([&](auto rc) {
          FEK_CI(r, rc);
#pragma unroll
          for (int s = r; s < NS; ++s) {
            const R gg = fma(g[r][0], g[s][0], fma(g[r][1], g[s][1], g[r][2] * g[s][2]));
            A[NS * r + s] = fma(pd.vol, gg, A[NS * r + s]);
          }
          constexpr R vr = R(S::val(Q, r));
          B[r] = fma(pd.vol * vr, coef[Q], B[r]);
        });
      } else {
        static_for<NS>([&](auto sc) {
          FEK_CI(s, sc);
          R t[4];
          cphi(coef, R(S::val(Q, s)), g[s], pd.vol, t);
          static_for<NS>([&](auto rc) {
            FEK_CI(r, rc);
            A[NS * r + s] = acc_dot4(A[NS * r + s], R(S::val(Q, r)), g[r], t);
          });
        });
        // load vector as a 7th column: B_r += phi_r . (vol d)
        R tb[4];
        load.fetch(tb);
#pragma unroll
        for (int k = 0; k < 4; ++k) tb[k] = pd.vol * tb[k];
        static_for<NS>([&](auto rc) {
          FEK_CI(r, rc);
          B[r] = acc_dot4(B[r], R(S::val(Q, r)), g[r], tb);
        });
      }
    });
  } else if constexpr (VAR == SQS) {
    // row-at-a-time: point data recomputed for every (row, point)
    static_for<NS>([&](auto rc) {
      FEK_CI(r, rc);
      static_for<NQ>([&](auto qc) {
        FEK_CI(Q, qc);
        R X[DSG];
        geo.fetch(X);
        const PointData<ET, Q, R> pd(X, bound);
        note(pd.kind, Q);
        R g[NS][3];
        all_grads<ET, Q>(pd.jac, g);
        if constexpr (SYM) {
#pragma unroll
          for (int s = r; s < NS; ++s) {
            const R gg = fma(g[r][0], g[s][0], fma(g[r][1], g[s][1], g[r][2] * g[s][2]));
            A[NS * r + s] = fma(pd.vol, gg, A[NS * r + s]);
          }
          constexpr R vr = R(S::val(Q, r));
          B[r] = fma(pd.vol * vr, coef[Q], B[r]);
        } else {
          // row r: A_rs += vol * phi_r^T C phi_s = (vol C^T phi_r) . phi_s
          constexpr R vr = R(S::val(Q, r));
          R u[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            u[j] = pd.vol * fma(coef[4 + j], g[r][0], fma(coef[8 + j], g[r][1], fma(coef[12 + j], g[r][2], coef[j] * vr)));
          static_for<NS>([&](auto sc) {
            FEK_CI(s, sc);
            A[NS * r + s] = acc_dot4(A[NS * r + s], R(S::val(Q, s)), g[s], u);
          });
          B[r] = fma(pd.vol, load_term(coef + 16, vr, g[r]), B[r]);
        }
      });
    });
  } else {
    // entry-at-a-time: point data recomputed for every (row, column, point),
    // only the two shape functions involved are differentiated
    static_for<NS>([&](auto rc) {
      FEK_CI(r, rc);
      static_for<NS>([&](auto sc) {
        FEK_CI(s, sc);
        if constexpr (!SYM || s >= r) {
          static_for<NQ>([&](auto qc) {
            FEK_CI(Q, qc);
            R X[DSG];
            geo.fetch(X);
            const PointData<ET, Q, R> pd(X, bound);
            note(pd.kind, Q);
            R gr[3], gs[3];
            global_grad<ET, Q, r>(pd.jac, gr);
            global_grad<ET, Q, s>(pd.jac, gs);
            constexpr R vr = R(S::val(Q, r));
            constexpr R vs = R(S::val(Q, s));
            if constexpr (SYM) {
              const R gg = fma(gr[0], gs[0], fma(gr[1], gs[1], gr[2] * gs[2]));
              A[NS * r + s] = fma(pd.vol, gg, A[NS * r + s]);
              if constexpr (r == s) B[r] = fma(pd.vol * vr, coef[Q], B[r]);
            } else {
              R t[4];
              cphi(coef, vs, gs, pd.vol, t);
              A[NS * r + s] = acc_dot4(A[NS * r + s], vr, gr, t);
              if constexpr (r == s) B[r] = fma(pd.vol, load_term(coef + 16, vr, gr), B[r]);
            }
          });
        }
      });
    });
  }
  if constexpr (SYM) {
#pragma unroll
    for (int r = 0; r < NS; ++r)
#pragma unroll
      for (int s = 0; s < r; ++s) A[NS * r + s] = A[NS * s + r];
  }
  first_failure(fail_mask, near_mask, kind, kind_point);
}

}  // namespace fek
