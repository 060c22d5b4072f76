// Shared device helpers for the FE operator kernels (sm_100a, FP64).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/fe_b200.h"

#define FE_DEVICE __device__ __forceinline__

namespace fe {

constexpr int form_vs(int form, int dim) {
  return (form == FE_FORM_LAPLACIAN || form == FE_FORM_ELASTICITY ||
          form == FE_FORM_ELASTICITY_LAME || form == FE_FORM_NEOHOOKEAN ||
          form == FE_FORM_NEOHOOKEAN_TANGENT) ? dim : 1;
}
constexpr bool form_needs_values(int form) {
  return form == FE_FORM_MASS || form == FE_FORM_HELMHOLTZ;
}
constexpr bool form_needs_grads(int form) { return form != FE_FORM_MASS; }
// forms linearised at a state u0 (coef0): its reference gradient is interpolated too
constexpr bool form_has_state(int form) { return form == FE_FORM_NEOHOOKEAN_TANGENT; }

// Device-side view of a bound mesh, in the plan's internal layout.
struct MeshView {
  const int32_t* map;      // SoA [ndof][nc_stride] (dof ids; vertex ids in the first nv rows)
  const int32_t* vmap;     // SoA [nvert][nc_stride] when map0[:, :nv] is not the vertex map, else == map
  const double* coords;    // padded: [nverts][CSTRIDE] (CSTRIDE = 2 for 2D, 4 for 3D)
  int64_t nc_stride;
};

template <int DIM> struct CStride { static constexpr int value = DIM == 2 ? 2 : 4; };

template <int DIM>
FE_DEVICE void load_vertex(const double* __restrict__ coords, int v, double* x) {
  if constexpr (DIM == 2) {
    double2 c = __ldg(reinterpret_cast<const double2*>(coords) + v);
    x[0] = c.x; x[1] = c.y;
  } else {
    const double2* p = reinterpret_cast<const double2*>(coords) + 2 * (int64_t)v;
    double2 a = __ldg(p), b = __ldg(p + 1);
    x[0] = a.x; x[1] = a.y; x[2] = b.x;
  }
}

// 1/x without the IEEE division's slow-path subroutine: MUFU.RCP64H seed and
// two Newton steps (relative error ~1 ulp for the normal, non-tiny |det J|
// values it is used on).  The compiled 1.0/x is a BSSY/CALL region per use,
// which fences instruction scheduling across the unrolled quadrature points
// of a kernel.  Whether that helps is kernel-specific (it also frees ptxas to
// hoist more work and raise register pressure), so every caller picks per
// kernel variant from measurement (profiles/r01/sweep_rcp.txt).
#ifndef FE_RCP3
#define FE_RCP3 1   // C5 5.176 -> 5.127 ms, C4-quad-Q1/Q2, C4-hex-Q1 +1% (profiles/r02/ab_rcp3.txt); parity unchanged
#endif
FE_DEVICE double rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#if FE_RCP3
  // one cubically convergent step: r (1 + e + e^2), e = 1 - x r (seed error
  // 2^-23 -> 2^-69): three FMAs instead of two Newton steps' four
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
#else
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#endif
}
template <bool FAST>
FE_DEVICE double recip(double x) {
  if constexpr (FAST) return rcp(x);
  else return 1.0 / x;
}

// Natural logarithm without the library routine's slow-path branches (the
// hyperelastic kernels take ln det F at every point; measured, the library
// log() was 25% of C5's time).  x = 2^e m with m in [1/sqrt2, sqrt2),
// ln m = 2 atanh(s), s = (m - 1)/(m + 1), |s| <= 0.1716, as an odd series in s
// to s^23 (truncation < 2e-17 relative); e ln2 added with a two-part ln2.
// A few ulp for positive finite x (subnormals are rescaled by 2^54 first);
// +inf -> +inf, +-0 -> -inf, x < 0 or NaN -> NaN, as the library routine.
// Branch-free: the special cases are selects.
FE_DEVICE double fast_log(double x0) {
  const bool sub = x0 < 2.2250738585072014e-308;            // subnormal (or <= 0: NaN/-inf below)
  const double x = sub ? x0 * 18014398509481984.0 : x0;    // * 2^54
  const int hi = __double2hiint(x), lo = __double2loint(x);
  int e = ((hi >> 20) & 0x7ff) - 1023 - (sub ? 54 : 0);
  double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);  // [1, 2)
  const bool big = m > 1.4142135623730951;
  m = big ? 0.5 * m : m;
  e = big ? e + 1 : e;
  const double f = m - 1.0;  // exact (Sterbenz)
  const double s = f * rcp(m + 1.0);
  const double z = s * s;
  double p = 1.0 / 23.0;
  p = fma(p, z, 1.0 / 21.0);
  p = fma(p, z, 1.0 / 19.0);
  p = fma(p, z, 1.0 / 17.0);
  p = fma(p, z, 1.0 / 15.0);
  p = fma(p, z, 1.0 / 13.0);
  p = fma(p, z, 1.0 / 11.0);
  p = fma(p, z, 1.0 / 9.0);
  p = fma(p, z, 1.0 / 7.0);
  p = fma(p, z, 1.0 / 5.0);
  p = fma(p, z, 1.0 / 3.0);
  const double ts = 2.0 * s;
  const double r = fma(ts * z, p, ts);  // 2s (1 + z p)
  const double de = (double)e;
  const double res = fma(de, 6.93147180369123816490e-01, fma(de, 1.90821492927058770002e-10, r));
  const double special = x0 == 0.0 ? __longlong_as_double(0xfff0000000000000LL)     // -inf
                         : x0 == __longlong_as_double(0x7ff0000000000000LL) ? x0    // +inf
                                                                            : __longlong_as_double(0x7ff8000000000000LL);
  return (x0 > 0.0 && x0 < __longlong_as_double(0x7ff0000000000000LL)) ? res : special;
}

// determinant and inverse of a DIM x DIM matrix stored row-major J[a][b]
template <int DIM, bool FAST = false>
FE_DEVICE double det_inv(const double (&J)[DIM][DIM], double (&Ji)[DIM][DIM]) {
  if constexpr (DIM == 2) {
    double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    double r = recip<FAST>(det);
    Ji[0][0] = J[1][1] * r;  Ji[0][1] = -J[0][1] * r;
    Ji[1][0] = -J[1][0] * r; Ji[1][1] = J[0][0] * r;
    return det;
  } else {
    double a00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    double a01 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    double a02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    double a10 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    double a11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    double a12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    double a20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    double a21 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    double a22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    double det = J[0][0] * a00 + J[0][1] * a10 + J[0][2] * a20;
    double r = recip<FAST>(det);
    Ji[0][0] = a00 * r; Ji[0][1] = a01 * r; Ji[0][2] = a02 * r;
    Ji[1][0] = a10 * r; Ji[1][1] = a11 * r; Ji[1][2] = a12 * r;
    Ji[2][0] = a20 * r; Ji[2][1] = a21 * r; Ji[2][2] = a22 * r;
    return det;
  }
}

FE_DEVICE uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
FE_DEVICE void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
FE_DEVICE void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
FE_DEVICE void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
FE_DEVICE void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
FE_DEVICE void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// 8-byte copy that zero-fills the destination when !valid (src-size 0)
FE_DEVICE void cp_async8_zfill(void* s, const void* g, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(s)), "l"(g),
               "r"(valid ? 8 : 0) : "memory");
}
template <int N>
FE_DEVICE void cp_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// determinant and adjugate (J^-1 = adj / det) of a DIM x DIM matrix
template <int DIM>
FE_DEVICE double det_adj(const double (&J)[DIM][DIM], double (&A)[DIM][DIM]) {
  if constexpr (DIM == 2) {
    A[0][0] = J[1][1];  A[0][1] = -J[0][1];
    A[1][0] = -J[1][0]; A[1][1] = J[0][0];
    return J[0][0] * J[1][1] - J[0][1] * J[1][0];
  } else {
    A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    return J[0][0] * A[0][0] + J[0][1] * A[1][0] + J[0][2] * A[2][0];
  }
}

// Programmatic dependent launch: an overwrite apply zero-fills y with a
// kernel that lets the operator kernel start early (its prologue gathers and
// first cells overlap the fill); every operator kernel calls this before its
// first write to y.  A no-op when the kernel was not launched as a dependent.
FE_DEVICE void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// y[idx] += v.  The global scatter P_e^T: FP64 RED at L2 (REDG.E.ADD.F64).
FE_DEVICE void scatter_add(double* y, int64_t idx, double v) { atomicAdd(y + idx, v); }

}  // namespace fe
