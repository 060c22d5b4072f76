/*
 * CPU port of the reference's vectorised cell loop -- BASELINE INFRASTRUCTURE.
 *
 * Only bench.py's cpu_baseline / --impl reference legs and tests/ load this
 * library; the product never does.  It is the timed CPU baseline for the
 * configs the reference cannot emit (tets, hexes, vs = 3, mu/lambda,
 * neo-Hookean), built the way the paper builds its CPU code:
 *
 *  - the reference's quadrature-loop local kernel (kernels.py:67-269: J
 *    hoisted on affine cells, per point otherwise; det, inverse, |det|;
 *    values/gradients at the point; per-form pointwise algebra; accumulation
 *    over the test functions), specialised per (form, cell, degree, rule)
 *    with compile-time sizes, as the reference's emitted wrap_<form> has
 *    (codegen.py:409-442);
 *  - cross-element vectorisation: the cell loop split by the SIMD width
 *    W = 8 (AVX-512 doubles) and every scalar of the local kernel widened to
 *    a W-lane vector, one lane per cell (transforms.py:274-519: split_iname,
 *    tag_simd, lane-expanded temporaries; GNU vector extensions as the
 *    reference's "vector-ext" target, codegen.py:398-407); gather and the
 *    scatter-add stay per lane and sequential within a batch
 *    (transforms.py:428,483); peeled remainder cells run as a masked batch;
 *  - threads (SURVEY.md 8d CPU-baseline protocol): contiguous cell chunks,
 *    each scattering into two private windows of y (the dofs its cells'
 *    vertex columns touch, and the others'), windows then summed into y in
 *    parallel over dof ranges.
 *
 * Numerically it is the oracle's algorithm (oracle/fe_oracle.c) in a
 * different order; tests/test_cpu_port.py pins it to the oracle at 1e-13.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr int W = 8;
typedef double vd __attribute__((vector_size(8 * W)));

enum { MASS = 0, HELMHOLTZ = 1, LAPLACIAN_SCALAR = 4, ELASTICITY_LAME = 5, NEOHOOKEAN = 6,
       NEOHOOKEAN_TANGENT = 7 };

struct Tables {
  const double *qw, *phi, *dphi, *gphi, *gdphi;
  double p0, p1;
};

struct Mesh {
  const double* coords;
  const double* u;
  const int32_t* map0;
  const int32_t* map1;
  const double* c0;  // mu (vertex field) or the state u0 (dof field)
  const double* c1;  // lambda
};

inline vd splat(double x) { return vd{} + x; }
inline vd vabs(vd x) {
  vd r;
  for (int l = 0; l < W; ++l) r[l] = std::fabs(x[l]);
  return r;
}
inline vd vlog(vd x) {
  vd r;
  for (int l = 0; l < W; ++l) r[l] = std::log(x[l]);
  return r;
}

template <int D>
inline vd det_inv(const vd (&J)[D][D], vd (&Ji)[D][D]) {
  if constexpr (D == 2) {
    vd det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    vd r = 1.0 / det;
    Ji[0][0] = J[1][1] * r;
    Ji[0][1] = -J[0][1] * r;
    Ji[1][0] = -J[1][0] * r;
    Ji[1][1] = J[0][0] * r;
    return det;
  } else {
    vd a[3][3];
    a[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    a[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    a[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    a[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    a[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    a[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    a[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    a[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    a[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    vd det = J[0][0] * a[0][0] + J[0][1] * a[1][0] + J[0][2] * a[2][0];
    vd r = 1.0 / det;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Ji[i][j] = a[i][j] * r;
    return det;
  }
}

/* One batch of W cells [c, c + n), n <= W (lanes >= n replicate cell c and
 * are not scattered). */
template <int FORM, int D, int NV, int ND, int VS, int NQ, bool AFF>
void batch(const Tables& T, const Mesh& M, int64_t c, int n, double* ybv, int64_t lov, double* ybr,
           int64_t lor) {
  constexpr bool VALS = FORM == MASS || FORM == HELMHOLTZ;
  constexpr bool GRADS = FORM != MASS;
  constexpr bool STATE = FORM == NEOHOOKEAN_TANGENT;
  constexpr bool LAME = FORM == ELASTICITY_LAME;
  vd X[NV][D], w[ND][VS], A[ND][VS];
  vd muv[LAME ? NV : 1], lamv[LAME ? NV : 1];
  vd w0buf[(STATE ? ND : 1) * VS];
  int64_t cell[W];
  for (int l = 0; l < W; ++l) cell[l] = c + (l < n ? l : 0);
  // gather (per lane)
  for (int l = 0; l < W; ++l) {
    const int32_t* vm = M.map1 + cell[l] * NV;
    for (int v = 0; v < NV; ++v) {
      for (int a = 0; a < D; ++a) X[v][a][l] = M.coords[(int64_t)vm[v] * D + a];
      if constexpr (LAME) {
        muv[v][l] = M.c0[vm[v]];
        lamv[v][l] = M.c1[vm[v]];
      }
    }
    const int32_t* dm = M.map0 + cell[l] * ND;
    for (int i = 0; i < ND; ++i)
      for (int k = 0; k < VS; ++k) {
        w[i][k][l] = M.u[(int64_t)VS * dm[i] + k];
        if constexpr (STATE) w0buf[i * VS + k][l] = M.c0[(int64_t)VS * dm[i] + k];
      }
  }
  for (int i = 0; i < ND; ++i)
    for (int k = 0; k < VS; ++k) A[i][k] = splat(0.0);
  vd J[D][D], Ji[D][D], absdet;
  for (int q = 0; q < NQ; ++q) {
    if (q == 0 || !AFF) {
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
          vd s = splat(0.0);
          for (int v = 0; v < NV; ++v) s += X[v][a] * T.gdphi[(q * NV + v) * D + b];
          J[a][b] = s;
        }
      absdet = vabs(det_inv<D>(J, Ji));
    }
    const vd tw = T.qw[q] * absdet;
    const double* ph = T.phi + q * ND;
    const double* dp = T.dphi + q * ND * D;
    vd uq[VS], g[VS][D];
    for (int k = 0; k < VS; ++k) {
      uq[k] = splat(0.0);
      for (int b = 0; b < D; ++b) g[k][b] = splat(0.0);
    }
    for (int i = 0; i < ND; ++i)
      for (int k = 0; k < VS; ++k) {
        if constexpr (VALS) uq[k] += ph[i] * w[i][k];
        if constexpr (GRADS)
          for (int b = 0; b < D; ++b) g[k][b] += dp[i * D + b] * w[i][k];
      }
    vd cv[VS], cg[VS][D];
    if constexpr (VALS)
      for (int k = 0; k < VS; ++k) cv[k] = tw * uq[k];
    if constexpr (GRADS) {
      vd G[VS][D], Tm[VS][D];
      for (int k = 0; k < VS; ++k)
        for (int a = 0; a < D; ++a) {
          vd s = splat(0.0);
          for (int b = 0; b < D; ++b) s += Ji[b][a] * g[k][b];
          G[k][a] = s;
        }
      if constexpr (LAME) {
        vd mu = splat(0.0), lam = splat(0.0), tr = splat(0.0);
        for (int v = 0; v < NV; ++v) {
          mu += T.gphi[q * NV + v] * muv[v];
          lam += T.gphi[q * NV + v] * lamv[v];
        }
        for (int k = 0; k < D; ++k) tr += G[k][k];
        for (int k = 0; k < D; ++k)
          for (int a = 0; a < D; ++a) {
            vd e = 0.5 * (G[k][a] + G[a][k]);
            Tm[k][a] = 2.0 * mu * e + (k == a ? lam * tr : splat(0.0));
          }
      } else if constexpr (FORM == NEOHOOKEAN) {
        vd F[D][D], Fi[D][D];
        for (int k = 0; k < D; ++k)
          for (int a = 0; a < D; ++a) F[k][a] = G[k][a] + (k == a ? 1.0 : 0.0);
        vd Jf = det_inv<D>(F, Fi);
        vd ll = T.p1 * vlog(Jf);
        for (int k = 0; k < D; ++k)
          for (int a = 0; a < D; ++a) Tm[k][a] = T.p0 * (F[k][a] - Fi[a][k]) + ll * Fi[a][k];
      } else if constexpr (STATE) {
        vd g0[D][D], F[D][D], Fi[D][D], Mm[D][D];
        for (int k = 0; k < D; ++k)
          for (int b = 0; b < D; ++b) g0[k][b] = splat(0.0);
        for (int i = 0; i < ND; ++i)
          for (int k = 0; k < VS; ++k)
            for (int b = 0; b < D; ++b) g0[k][b] += dp[i * D + b] * w0buf[i * VS + k];
        for (int k = 0; k < D; ++k)
          for (int a = 0; a < D; ++a) {
            vd s = splat(0.0);
            for (int b = 0; b < D; ++b) s += Ji[b][a] * g0[k][b];
            F[k][a] = s + (k == a ? 1.0 : 0.0);
          }
        vd Jf = det_inv<D>(F, Fi);
        vd tr = splat(0.0);
        for (int a = 0; a < D; ++a)
          for (int k = 0; k < D; ++k) tr += Fi[a][k] * G[k][a];
        for (int a = 0; a < D; ++a)
          for (int e = 0; e < D; ++e) {
            vd s = splat(0.0);
            for (int k = 0; k < D; ++k) s += G[k][a] * Fi[e][k];
            Mm[a][e] = s;
          }
        vd cA = T.p0 - T.p1 * vlog(Jf);
        for (int k = 0; k < D; ++k)
          for (int a = 0; a < D; ++a) {
            vd s = splat(0.0);
            for (int b = 0; b < D; ++b) s += Fi[b][k] * Mm[b][a];
            Tm[k][a] = T.p0 * G[k][a] + cA * s + T.p1 * tr * Fi[a][k];
          }
      } else {
        for (int k = 0; k < VS; ++k)
          for (int a = 0; a < D; ++a) Tm[k][a] = G[k][a];
      }
      for (int k = 0; k < VS; ++k)
        for (int b = 0; b < D; ++b) {
          vd s = splat(0.0);
          for (int a = 0; a < D; ++a) s += Ji[b][a] * Tm[k][a];
          cg[k][b] = tw * s;
        }
    }
    for (int j = 0; j < ND; ++j)
      for (int k = 0; k < VS; ++k) {
        vd acc = splat(0.0);
        if constexpr (VALS) acc += ph[j] * cv[k];
        if constexpr (GRADS)
          for (int b = 0; b < D; ++b) acc += dp[j * D + b] * cg[k][b];
        A[j][k] += acc;
      }
  }
  // scatter-add P^T (sequential over lanes, as the reference) into the
  // thread's two windows: vertex columns (j < NV) and the others
  for (int l = 0; l < n; ++l) {
    const int32_t* dm = M.map0 + cell[l] * ND;
    for (int j = 0; j < ND; ++j) {
      double* yb = j < NV ? ybv - lov : ybr - lor;
      for (int k = 0; k < VS; ++k) yb[(int64_t)VS * dm[j] + k] += A[j][k][l];
    }
  }
}

typedef void (*BatchFn)(const Tables&, const Mesh&, int64_t, int, double*, int64_t, double*, int64_t);

struct Entry {
  int form, dim, nv, nd, vs, nq;
  bool affine;
  BatchFn fn;
};

#define E(FORM, D, NV, ND, VS, NQ, AFF) {FORM, D, NV, ND, VS, NQ, AFF, batch<FORM, D, NV, ND, VS, NQ, AFF>}

const Entry kEntries[] = {
    // C1 mass P2 triangles (degree-4 rule)
    E(MASS, 2, 3, 6, 1, 9, true),
    // C2 helmholtz P1..P4 tetrahedra, rules exact for 2k: (k+1)^3 points
    E(HELMHOLTZ, 3, 4, 4, 1, 8, true), E(HELMHOLTZ, 3, 4, 10, 1, 27, true),
    E(HELMHOLTZ, 3, 4, 20, 1, 64, true), E(HELMHOLTZ, 3, 4, 35, 1, 125, true),
    // C3 scalar Laplacian Q1..Q6 hexahedra, k+1 GL points per direction
    E(LAPLACIAN_SCALAR, 3, 8, 8, 1, 8, false), E(LAPLACIAN_SCALAR, 3, 8, 27, 1, 27, false),
    E(LAPLACIAN_SCALAR, 3, 8, 64, 1, 64, false), E(LAPLACIAN_SCALAR, 3, 8, 125, 1, 125, false),
    E(LAPLACIAN_SCALAR, 3, 8, 216, 1, 216, false), E(LAPLACIAN_SCALAR, 3, 8, 343, 1, 343, false),
    // C4 Lame elasticity Q1..Q4 quadrilaterals, Q1..Q3 hexahedra, k+2 GL points
    E(ELASTICITY_LAME, 2, 4, 4, 2, 9, false), E(ELASTICITY_LAME, 2, 4, 9, 2, 16, false),
    E(ELASTICITY_LAME, 2, 4, 16, 2, 25, false), E(ELASTICITY_LAME, 2, 4, 25, 2, 36, false),
    E(ELASTICITY_LAME, 3, 8, 8, 3, 27, false), E(ELASTICITY_LAME, 3, 8, 27, 3, 64, false),
    E(ELASTICITY_LAME, 3, 8, 64, 3, 125, false),
    // C5 neo-Hookean residual, C6 its tangent: P2 tetrahedra, degree-4 rule
    E(NEOHOOKEAN, 3, 4, 10, 3, 27, true), E(NEOHOOKEAN_TANGENT, 3, 4, 10, 3, 27, true),
};

const Entry* find(int form, int dim, int nv, int nd, int vs, int nq, int affine) {
  for (const Entry& e : kEntries)
    if (e.form == form && e.dim == dim && e.nv == nv && e.nd == nd && e.vs == vs && e.nq == nq &&
        e.affine == (affine != 0))
      return &e;
  return nullptr;
}

}  // namespace

extern "C" {

/* 1 if a specialisation exists for this (form, dim, nv, nd, vs, nq, affine). */
int fe_cpu_supported(int form, int dim, int nv, int nd, int vs, int nq, int affine) {
  return find(form, dim, nv, nd, vs, nq, affine) != nullptr;
}

/* y += sum over cells [start, end) of P_e^T A_e(P_e u) on nthreads threads.
 * Same argument meaning as oracle/fe_oracle.c fe_oracle_apply_mt; c0/c1 =
 * mu/lambda vertex fields, or c0 = the state u0 (neohookean_tangent).
 * Returns 0, or -1 when no specialisation exists. */
int fe_cpu_apply(int form, int dim, int nv, int nd, int vs, int nq, int affine, const double* qw,
                 const double* phi, const double* dphi, const double* gphi, const double* gdphi,
                 double p0, double p1, int64_t start, int64_t end, double* y, int64_t ny,
                 const double* coords, const double* u, const int32_t* map0, const int32_t* map1,
                 const double* c0, const double* c1, int nthreads) {
  const Entry* e = find(form, dim, nv, nd, vs, nq, affine);
  if (!e) return -1;
  if (end <= start) return 0;
  const Tables T{qw, phi, dphi, gphi, gdphi, p0, p1};
  std::vector<int32_t> m1;
  if (!map1) {  // vertex columns of map0
    m1.resize((size_t)(end) * nv);
    for (int64_t c = 0; c < end; ++c)
      for (int v = 0; v < nv; ++v) m1[c * nv + v] = map0[c * nd + v];
  }
  const Mesh Mv{coords, u, map0, map1 ? map1 : m1.data(), c0, c1};
  const int64_t ncell = end - start;
  int T_ = std::max(1, std::min<int>(nthreads, (int)((ncell + 4 * W - 1) / (4 * W))));
  // contiguous, W-aligned chunks
  std::vector<int64_t> cut(T_ + 1);
  for (int t = 0; t <= T_; ++t) cut[t] = start + (ncell * t / T_ + W - 1) / W * W;
  cut[0] = start;
  cut[T_] = end;
  for (int t = 1; t < T_; ++t) cut[t] = std::min(end, std::max(cut[t], cut[t - 1]));
  // per thread TWO windows of y: the dofs of its cells' vertex columns
  // (j < nv) and of the other columns -- with the vertex dofs numbered first
  // (the reference's convention, mesh.py:95) the two bands are far apart in
  // y and one window would span it all.  Window buffers are kept across
  // calls (their pages stay mapped); one caller at a time.
  std::vector<int64_t> lo(2 * T_), hi(2 * T_);
  static std::vector<std::vector<double>> buf;
  if ((int)buf.size() < 2 * T_) buf.resize(2 * T_);
#pragma omp parallel num_threads(T_)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    int64_t a = cut[t], b = cut[t + 1];
    int32_t mn[2] = {INT32_MAX, INT32_MAX}, mx[2] = {-1, -1};
    for (int64_t c = a; c < b; ++c)
      for (int j = 0; j < nd; ++j) {
        const int w = j < nv ? 0 : 1;
        const int32_t d = map0[c * nd + j];
        mn[w] = std::min(mn[w], d);
        mx[w] = std::max(mx[w], d);
      }
    for (int w = 0; w < 2; ++w) {
      const int i = 2 * t + w;
      if (mx[w] >= 0) {
        lo[i] = (int64_t)vs * mn[w];
        hi[i] = (int64_t)vs * mx[w] + vs;
      } else {
        lo[i] = hi[i] = 0;
      }
      if ((int64_t)buf[i].size() < std::max<int64_t>(1, hi[i] - lo[i])) buf[i].resize(std::max<int64_t>(1, hi[i] - lo[i]));
      std::fill(buf[i].begin(), buf[i].begin() + (hi[i] - lo[i]), 0.0);
    }
    for (int64_t c = a; c < b; c += W)
      e->fn(T, Mv, c, (int)std::min<int64_t>(W, b - c), buf[2 * t].data(), lo[2 * t], buf[2 * t + 1].data(),
            lo[2 * t + 1]);
  }
  // windows -> y, in parallel over dof ranges
  const int R = std::max(1, nthreads);
#pragma omp parallel for num_threads(R) schedule(static)
  for (int r = 0; r < R; ++r) {
    const int64_t r0 = ny * r / R, r1 = ny * (r + 1) / R;
    for (int i = 0; i < 2 * T_; ++i) {
      const int64_t a = std::max(r0, lo[i]), b = std::min(r1, hi[i]);
      const double* s = buf[i].data() - lo[i];
      for (int64_t k = a; k < b; ++k) y[k] += s[k];
    }
  }
  return 0;
}

}  // extern "C"
