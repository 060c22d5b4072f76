/*
 * CPU restatement of the reference hot loop -- TEST / BASELINE INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
 * --impl reference legs load this library; the product never does.
 *
 * It is the loop the reference generates for wrap_<form>
 * (/root/reference/pkg/src/fevec/transforms.py:112-266: gather P_e u and the
 * vertex coordinates, zero the local vector, run the inlined local kernel,
 * scatter-add P_e^T) with the local kernel of kernels.py:67-269 (Jacobian
 * hoisted on affine cells, per quadrature point otherwise; det, inverse,
 * |det|; values/gradients at the quadrature point; per-form pointwise
 * algebra; accumulation over test functions), extended to 3D cells, value
 * size 3 and the mu/lambda and neo-Hookean forms exactly as oracle/fe_oracle.py
 * does.  Tables (phi, dphi, gphi, gdphi, weights) are inputs, as the
 * reference bakes them into the emitted source (codegen.py:409-424).
 *
 * fe_oracle_apply_mt() runs the cell loop on T threads over contiguous cell
 * chunks (the SURVEY.md 8d CPU-baseline protocol): element vectors are
 * computed in parallel, then scattered in cell order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { MASS = 0, HELMHOLTZ = 1, LAPLACIAN = 2, ELASTICITY = 3, LAPLACIAN_SCALAR = 4,
       ELASTICITY_LAME = 5, NEOHOOKEAN = 6, NEOHOOKEAN_TANGENT = 7 };

#define MAXD 3

static double det_inv(int d, const double J[MAXD][MAXD], double Ji[MAXD][MAXD]) {
  if (d == 2) {
    double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    Ji[0][0] = J[1][1] / det; Ji[0][1] = -J[0][1] / det;
    Ji[1][0] = -J[1][0] / det; Ji[1][1] = J[0][0] / det;
    return det;
  }
  double a[3][3];
  a[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  a[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  a[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  a[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  a[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  a[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  a[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  a[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  a[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  double det = J[0][0] * a[0][0] + J[0][1] * a[1][0] + J[0][2] * a[2][0];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Ji[i][j] = a[i][j] / det;
  return det;
}

typedef struct {
  int form, dim, nv, nd, vs, nq, affine;
  const double *qw, *phi, *dphi, *gphi, *gdphi;
  double p0, p1;
} problem;

/* local kernel of one cell: A[nd*vs] from X[nv][dim], w[nd*vs] */
static void local_kernel(const problem* P, const double* X, const double* w, const double* muv,
                         const double* lamv, const double* w0, double* A) {
  const int d = P->dim, nd = P->nd, vs = P->vs, nv = P->nv;
  double J[MAXD][MAXD], Ji[MAXD][MAXD], absdet = 0.0;
  memset(A, 0, sizeof(double) * nd * vs);
  for (int q = 0; q < P->nq; ++q) {
    if (q == 0 || !P->affine) {
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          double s = 0.0;
          for (int v = 0; v < nv; ++v) s += X[v * d + a] * P->gdphi[(q * nv + v) * d + b];
          J[a][b] = s;
        }
      absdet = fabs(det_inv(d, J, Ji));
    }
    const double tw = P->qw[q] * absdet;
    const double* ph = P->phi + q * nd;
    const double* dp = P->dphi + q * nd * d;
    double uq[MAXD] = {0}, g[MAXD][MAXD] = {{0}}, G[MAXD][MAXD], T[MAXD][MAXD];
    for (int i = 0; i < nd; ++i)
      for (int c = 0; c < vs; ++c) {
        uq[c] += ph[i] * w[i * vs + c];
        for (int b = 0; b < d; ++b) g[c][b] += dp[i * d + b] * w[i * vs + c];
      }
    for (int c = 0; c < vs; ++c)
      for (int a = 0; a < d; ++a) {
        double s = 0.0;
        for (int b = 0; b < d; ++b) s += Ji[b][a] * g[c][b];
        G[c][a] = s;
      }
    double cv[MAXD] = {0}, cg[MAXD][MAXD] = {{0}};
    const int vals = P->form == MASS || P->form == HELMHOLTZ;
    const int grads = P->form != MASS;
    if (vals)
      for (int c = 0; c < vs; ++c) cv[c] = tw * uq[c];
    if (grads) {
      if (P->form == ELASTICITY || P->form == ELASTICITY_LAME) {
        double mu = 0.5, lam = 0.0, tr = 0.0;
        if (P->form == ELASTICITY_LAME) {
          mu = lam = 0.0;
          for (int v = 0; v < nv; ++v) {
            mu += P->gphi[q * nv + v] * muv[v];
            lam += P->gphi[q * nv + v] * lamv[v];
          }
        }
        for (int c = 0; c < d; ++c) tr += G[c][c];
        for (int c = 0; c < d; ++c)
          for (int a = 0; a < d; ++a) {
            double e = 0.5 * (G[c][a] + G[a][c]);
            T[c][a] = P->form == ELASTICITY ? e : 2.0 * mu * e + (c == a ? lam * tr : 0.0);
          }
      } else if (P->form == NEOHOOKEAN) {
        double F[MAXD][MAXD], Fi[MAXD][MAXD];
        for (int c = 0; c < d; ++c)
          for (int a = 0; a < d; ++a) F[c][a] = G[c][a] + (c == a ? 1.0 : 0.0);
        double Jf = det_inv(d, F, Fi);
        double ll = P->p1 * log(Jf);
        for (int c = 0; c < d; ++c)
          for (int a = 0; a < d; ++a) T[c][a] = P->p0 * (F[c][a] - Fi[a][c]) + ll * Fi[a][c];
      } else if (P->form == NEOHOOKEAN_TANGENT) {
        /* dP = mu dF + (mu - lam ln J) F^-T dF^T F^-T + lam tr(F^-1 dF) F^-T
         * at F = I + grad u0 (oracle/fe_oracle.py _local, neohookean_tangent) */
        double g0[MAXD][MAXD] = {{0}}, F[MAXD][MAXD], Fi[MAXD][MAXD];
        for (int i = 0; i < nd; ++i)
          for (int c = 0; c < vs; ++c)
            for (int b = 0; b < d; ++b) g0[c][b] += dp[i * d + b] * w0[i * vs + c];
        for (int c = 0; c < d; ++c)
          for (int a = 0; a < d; ++a) {
            double s = 0.0;
            for (int b = 0; b < d; ++b) s += Ji[b][a] * g0[c][b];
            F[c][a] = s + (c == a ? 1.0 : 0.0);
          }
        double Jf = det_inv(d, F, Fi);
        double tr = 0.0;                        /* tr(F^-1 dF) */
        for (int a = 0; a < d; ++a)
          for (int c = 0; c < d; ++c) tr += Fi[a][c] * G[c][a];
        double M[MAXD][MAXD];                   /* dF^T F^-T: M[a][e] = sum_c dF[c][a] Fi[e][c] */
        for (int a = 0; a < d; ++a)
          for (int e = 0; e < d; ++e) {
            double s = 0.0;
            for (int c = 0; c < d; ++c) s += G[c][a] * Fi[e][c];
            M[a][e] = s;
          }
        const double cA = P->p0 - P->p1 * log(Jf);
        for (int c = 0; c < d; ++c)
          for (int a = 0; a < d; ++a) {
            double s = 0.0;                     /* (F^-T M)[c][a] = sum_b Fi[b][c] M[b][a] */
            for (int b = 0; b < d; ++b) s += Fi[b][c] * M[b][a];
            T[c][a] = P->p0 * G[c][a] + cA * s + P->p1 * tr * Fi[a][c];
          }
      } else {
        for (int c = 0; c < vs; ++c)
          for (int a = 0; a < d; ++a) T[c][a] = G[c][a];
      }
      for (int c = 0; c < vs; ++c)
        for (int b = 0; b < d; ++b) {
          double s = 0.0;
          for (int a = 0; a < d; ++a) s += Ji[b][a] * T[c][a];
          cg[c][b] = tw * s;
        }
    }
    for (int j = 0; j < nd; ++j)
      for (int c = 0; c < vs; ++c) {
        double acc = 0.0;
        if (vals) acc += ph[j] * cv[c];
        if (grads)
          for (int b = 0; b < d; ++b) acc += dp[j * d + b] * cg[c][b];
        A[j * vs + c] += acc;
      }
  }
}

/* mu: the vertex field mu (elasticity_lame) or the state u0, a dof field
 * in the layout of u (neohookean_tangent, as the GPU ABI's coef0) */
static void gather(const problem* P, int64_t n, const double* coords, const double* u,
                   const int32_t* map0, const int32_t* map1, const double* mu, const double* lam,
                   double* X, double* w, double* muv, double* lamv, double* w0) {
  const int d = P->dim, nd = P->nd, vs = P->vs, nv = P->nv;
  const int state = P->form == NEOHOOKEAN_TANGENT;
  for (int v = 0; v < nv; ++v) {
    int vid = map1[n * nv + v];
    for (int a = 0; a < d; ++a) X[v * d + a] = coords[(int64_t)vid * d + a];
    if (mu && !state) { muv[v] = mu[vid]; lamv[v] = lam[vid]; }
  }
  for (int i = 0; i < nd; ++i)
    for (int c = 0; c < vs; ++c) {
      w[i * vs + c] = u[(int64_t)vs * map0[n * nd + i] + c];
      if (state) w0[i * vs + c] = mu[(int64_t)vs * map0[n * nd + i] + c];
    }
}

/* single-threaded wrap_<form> restatement: y += sum over [start,end) */
void fe_oracle_apply(int form, int dim, int nv, int nd, int vs, int nq, int affine,
                     const double* qw, const double* phi, const double* dphi, const double* gphi,
                     const double* gdphi, double p0, double p1, int start, int end, double* y,
                     const double* coords, const double* u, const int32_t* map0,
                     const int32_t* map1, const double* mu, const double* lam) {
  problem P = {form, dim, nv, nd, vs, nq, affine, qw, phi, dphi, gphi, gdphi, p0, p1};
  double X[8 * MAXD], muv[8], lamv[8];
  double* w = malloc(sizeof(double) * nd * vs);
  double* w0 = malloc(sizeof(double) * nd * vs);
  double* A = malloc(sizeof(double) * nd * vs);
  for (int64_t n = start; n < end; ++n) {
    gather(&P, n, coords, u, map0, map1, mu, lam, X, w, muv, lamv, w0);
    local_kernel(&P, X, w, muv, lamv, w0, A);
    for (int j = 0; j < nd; ++j)
      for (int c = 0; c < vs; ++c) y[(int64_t)vs * map0[n * nd + j] + c] += A[j * vs + c];
  }
  free(w);
  free(w0);
  free(A);
}

/* T threads over contiguous cell chunks; element vectors in a buffer, then
 * scattered in cell order (deterministic). */
void fe_oracle_apply_mt(int form, int dim, int nv, int nd, int vs, int nq, int affine,
                        const double* qw, const double* phi, const double* dphi, const double* gphi,
                        const double* gdphi, double p0, double p1, int start, int end, double* y,
                        const double* coords, const double* u, const int32_t* map0,
                        const int32_t* map1, const double* mu, const double* lam, int nthreads) {
  problem P = {form, dim, nv, nd, vs, nq, affine, qw, phi, dphi, gphi, gdphi, p0, p1};
  const int64_t n = end - start, L = (int64_t)nd * vs;
  double* buf = malloc(sizeof(double) * (n > 0 ? n : 1) * L);
#pragma omp parallel num_threads(nthreads)
  {
    double X[8 * MAXD], muv[8], lamv[8];
    double* w = malloc(sizeof(double) * L);
    double* w0 = malloc(sizeof(double) * L);
#pragma omp for schedule(static)
    for (int64_t c = start; c < end; ++c) {
      gather(&P, c, coords, u, map0, map1, mu, lam, X, w, muv, lamv, w0);
      local_kernel(&P, X, w, muv, lamv, w0, buf + (c - start) * L);
    }
    free(w);
    free(w0);
  }
  for (int64_t c = start; c < end; ++c) {
    const double* A = buf + (c - start) * L;
    for (int j = 0; j < nd; ++j)
      for (int k = 0; k < vs; ++k) y[(int64_t)vs * map0[c * nd + j] + k] += A[j * vs + k];
  }
  free(buf);
}
