// Generic thread-per-cell quadrature kernel: the reference algorithm
// (kernels.py:67-269 local kernel inlined into the transforms.py:112-266
// gather/compute/scatter cell loop) with one GPU thread per cell -- the GPU
// analogue of the paper's cross-element SIMD lanes (one lane per cell,
// transforms.py:409-491).  Tables (kernels.py:97-108) are staged in shared
// memory; every thread of a warp reads the same table entry (broadcast).
//
// Used for every (form, cell, degree) whose local vectors fit in registers;
// it is the production kernel for the neo-Hookean residual (C5) and the
// coverage kernel for the others.
#pragma once
#include "common.cuh"

namespace fe {

struct QuadParams {
  MeshView mesh;
  int32_t start, end;
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ mu;   // vertex fields (elasticity_lame)
  const double* __restrict__ lam;
  const double* __restrict__ tables;  // qw | phi | dphi | gphi | gdphi
  double p0, p1;                      // neohookean mu, lambda
};

#ifndef FE_LOG
#define FE_LOG fast_log
#endif
template <int NQ, int ND, int NV, int DIM>
struct QuadTables {
  static constexpr int qw = 0;
  static constexpr int phi = qw + NQ;
  static constexpr int dphi = phi + NQ * ND;
  static constexpr int gphi = dphi + NQ * ND * DIM;
  static constexpr int gdphi = gphi + NQ * NV;
  static constexpr int size = gdphi + NQ * NV * DIM;
};

// Pointwise flux at one quadrature point.  Inputs: inverse Jacobian Ji
// (Ji[b][a] = dxi_b/dx_a), weight tw = w_q |det J|, values uq[c] and
// reference gradients g[c][b] of u (and g0 of the state u0 for the
// linearised forms).  Outputs: cv[c] multiplies phi_j and cg[c][b] multiplies
// dphi_j/dxi_b in the accumulation A[j][c] += ... (kernels.py:202-252 for the
// reference forms).
template <int FORM, int DIM, int VS, bool FAST = false>
FE_DEVICE void pointwise(const double (&Ji)[DIM][DIM], double tw, const double (&uq)[VS],
                         const double (&g)[VS][DIM], double mu, double lam,
                         double (&cv)[VS], double (&cg)[VS][DIM],
                         const double (&g0)[VS][DIM] = {}) {
  if constexpr (form_needs_values(FORM)) {
#pragma unroll
    for (int c = 0; c < VS; ++c) cv[c] = tw * uq[c];
  }
  if constexpr (form_needs_grads(FORM)) {
    double G[VS][DIM];  // physical gradient du_c/dx_a
#pragma unroll
    for (int c = 0; c < VS; ++c)
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < DIM; ++b) s += Ji[b][a] * g[c][b];
        G[c][a] = s;
      }
    double T[VS][DIM];  // physical flux paired with dv_c/dx_a
    if constexpr (FORM == FE_FORM_HELMHOLTZ || FORM == FE_FORM_LAPLACIAN_SCALAR ||
                  FORM == FE_FORM_LAPLACIAN) {
#pragma unroll
      for (int c = 0; c < VS; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) T[c][a] = G[c][a];
    } else if constexpr (FORM == FE_FORM_ELASTICITY || FORM == FE_FORM_ELASTICITY_LAME) {
      // T = 2 mu eps + lam tr(eps) I = mu (G + G^T) + lam tr(G) I (reference
      // elasticity: eps = (G + G^T) / 2), with the weight folded into the two
      // scalars
      static_assert(VS == DIM, "vector form");
      double tr = 0.0;
#pragma unroll
      for (int c = 0; c < VS; ++c) tr += G[c][c];
      const double m = tw * (FORM == FE_FORM_ELASTICITY ? 0.5 : mu);
      const double lt = FORM == FE_FORM_ELASTICITY ? 0.0 : tw * lam * tr;
#pragma unroll
      for (int c = 0; c < VS; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) T[c][a] = fma(m, G[c][a] + G[a][c], c == a ? lt : 0.0);
    } else if constexpr (FORM == FE_FORM_NEOHOOKEAN) {
      // P = mu (F - F^-T) + lambda ln J F^-T = mu G + mu I + (lambda ln J - mu) F^-T
      // with F^-T[c][a] = adj(F)[a][c] / J; the weight tw is folded into the
      // two scalars (no inverse formed, no per-entry weight multiply)
      static_assert(VS == DIM, "vector form");
      double F[DIM][DIM], A[DIM][DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) F[c][a] = G[c][a] + (c == a ? 1.0 : 0.0);
      const double Jf = det_adj<DIM>(F, A);
      const double m = tw * mu;
      const double s = tw * (lam * FE_LOG(Jf) - mu) * recip<FAST>(Jf);
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) T[c][a] = fma(m, G[c][a], s * A[a][c]) + (c == a ? m : 0.0);
    } else if constexpr (FORM == FE_FORM_NEOHOOKEAN_TANGENT) {
      // dP = mu dF + (mu - lambda ln J) F^-T dF^T F^-T + lambda tr(F^-1 dF) F^-T
      // with F = I + grad u0 (state), dF = grad du = G.  With F^-1 = A / J
      // (A = adj F) and M = A dF: F^-T dF^T F^-T = (M A)^T / J^2 and
      // tr(F^-1 dF) = tr(M) / J; the weight tw is folded into the scalars.
      static_assert(VS == DIM, "vector form");
      double F[DIM][DIM], A[DIM][DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < DIM; ++b) s += Ji[b][a] * g0[c][b];
          F[c][a] = s + (c == a ? 1.0 : 0.0);
        }
      const double Jf = det_adj<DIM>(F, A);
      const double r = recip<FAST>(Jf);
      double M[DIM][DIM];
      double tr = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < DIM; ++c) s += A[a][c] * G[c][b];
          M[a][b] = s;
          if (a == b) tr += s;
        }
      const double m = tw * mu;
      const double r2 = tw * r * r;
      const double c2 = (mu - lam * FE_LOG(Jf)) * r2;
      const double l2 = lam * tr * r2;
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          double s = 0.0;  // (M A)[a][c]
#pragma unroll
          for (int b = 0; b < DIM; ++b) s += M[a][b] * A[b][c];
          T[c][a] = fma(m, G[c][a], fma(c2, s, l2 * A[a][c]));
        }
    }
    // hyperelastic fluxes already carry the weight
    constexpr bool WEIGHTED = FORM == FE_FORM_NEOHOOKEAN || FORM == FE_FORM_NEOHOOKEAN_TANGENT ||
                              FORM == FE_FORM_ELASTICITY || FORM == FE_FORM_ELASTICITY_LAME;
#pragma unroll
    for (int c = 0; c < VS; ++c)
#pragma unroll
      for (int b = 0; b < DIM; ++b) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) s += Ji[b][a] * T[c][a];
        cg[c][b] = WEIGHTED ? s : tw * s;
      }
  }
}

template <int FORM, int DIM, int NV, int ND, int NQ, bool AFFINE>
__global__ void __launch_bounds__(128) quad_kernel(QuadParams p) {
  constexpr int VS = form_vs(FORM, DIM);
  using TB = QuadTables<NQ, ND, NV, DIM>;
  extern __shared__ double smem[];
  for (int i = threadIdx.x; i < TB::size; i += blockDim.x) smem[i] = p.tables[i];
  __syncthreads();
  const double* s_qw = smem + TB::qw;
  const double* s_phi = smem + TB::phi;
  const double* s_dphi = smem + TB::dphi;
  const double* s_gphi = smem + TB::gphi;
  const double* s_gdphi = smem + TB::gdphi;

  const int cell = p.start + blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;

  int dof[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) dof[i] = __ldg(p.mesh.map + i * cs + cell);
  double X[NV][DIM];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    int vid = (p.mesh.vmap == p.mesh.map) ? dof[v] : __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<DIM>(p.mesh.coords, vid, X[v]);
  }
  double w[ND][VS];
#pragma unroll
  for (int i = 0; i < ND; ++i)
#pragma unroll
    for (int c = 0; c < VS; ++c) w[i][c] = __ldg(p.u + (int64_t)VS * dof[i] + c);
  double w0[form_has_state(FORM) ? ND : 1][VS];
  if constexpr (form_has_state(FORM)) {
#pragma unroll
    for (int i = 0; i < ND; ++i)
#pragma unroll
      for (int c = 0; c < VS; ++c) w0[i][c] = __ldg(p.mu + (int64_t)VS * dof[i] + c);
  }
  double muv[NV], lamv[NV];
  if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      int vid = (p.mesh.vmap == p.mesh.map) ? dof[v] : __ldg(p.mesh.vmap + v * cs + cell);
      muv[v] = __ldg(p.mu + vid);
      lamv[v] = __ldg(p.lam + vid);
    }
  }
  double A[ND][VS];
#pragma unroll
  for (int i = 0; i < ND; ++i)
#pragma unroll
    for (int c = 0; c < VS; ++c) A[i][c] = 0.0;

  double J[DIM][DIM], Ji[DIM][DIM], absdet = 0.0;
  auto jacobian = [&](int q) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) {
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) s += X[v][a] * s_gdphi[(q * NV + v) * DIM + b];
        J[a][b] = s;
      }
    absdet = fabs(det_inv<DIM>(J, Ji));
  };
  if constexpr (AFFINE) jacobian(0);

#pragma unroll 1
  for (int q = 0; q < NQ; ++q) {
    if constexpr (!AFFINE) jacobian(q);
    const double tw = s_qw[q] * absdet;
    double uq[VS], g[VS][DIM];
    if constexpr (form_needs_values(FORM)) {
#pragma unroll
      for (int c = 0; c < VS; ++c) uq[c] = 0.0;
#pragma unroll
      for (int i = 0; i < ND; ++i) {
        double ph = s_phi[q * ND + i];
#pragma unroll
        for (int c = 0; c < VS; ++c) uq[c] += ph * w[i][c];
      }
    }
    if constexpr (form_needs_grads(FORM)) {
#pragma unroll
      for (int c = 0; c < VS; ++c)
#pragma unroll
        for (int b = 0; b < DIM; ++b) g[c][b] = 0.0;
#pragma unroll
      for (int i = 0; i < ND; ++i)
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
          double d = s_dphi[(q * ND + i) * DIM + b];
#pragma unroll
          for (int c = 0; c < VS; ++c) g[c][b] += d * w[i][c];
        }
    }
    double mu = p.p0, lam = p.p1;
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
      mu = 0.0; lam = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double gv = s_gphi[q * NV + v];
        mu += gv * muv[v];
        lam += gv * lamv[v];
      }
    }
    double g0[VS][DIM];
    if constexpr (form_has_state(FORM)) {
#pragma unroll
      for (int c = 0; c < VS; ++c)
#pragma unroll
        for (int b = 0; b < DIM; ++b) g0[c][b] = 0.0;
#pragma unroll
      for (int i = 0; i < ND; ++i)
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
          double d = s_dphi[(q * ND + i) * DIM + b];
#pragma unroll
          for (int c = 0; c < VS; ++c) g0[c][b] += d * w0[i][c];
        }
    }
    double cv[VS], cg[VS][DIM];
    pointwise<FORM, DIM, VS>(Ji, tw, uq, g, mu, lam, cv, cg, g0);
#pragma unroll
    for (int j = 0; j < ND; ++j) {
#pragma unroll
      for (int c = 0; c < VS; ++c) {
        double acc = A[j][c];
        if constexpr (form_needs_values(FORM)) acc += s_phi[q * ND + j] * cv[c];
        if constexpr (form_needs_grads(FORM)) {
#pragma unroll
          for (int b = 0; b < DIM; ++b) acc += s_dphi[(q * ND + j) * DIM + b] * cg[c][b];
        }
        A[j][c] = acc;
      }
    }
  }
  griddep_wait();
#pragma unroll
  for (int j = 0; j < ND; ++j)
#pragma unroll
    for (int c = 0; c < VS; ++c) scatter_add(p.y, (int64_t)VS * dof[j] + c, A[j][c]);
}

// ---------------------------------------------------------------------------
// Operator diagonal (fe_diagonal, Jacobi preconditioner of a matrix-free
// solve): diag(A_e)[i][c] = the (i, c) entry of A_e applied to the unit
// vector e_(i,c), i.e. the reference quadrature loop with w = e_(i,c).  One
// thread per cell, loops over local dofs outermost (one RED per entry);
// geometry recomputed per (dof, point) on non-affine cells -- a one-time
// setup kernel, not a hot path.
// ---------------------------------------------------------------------------
template <int FORM, int DIM, int NV, int ND, int NQ, bool AFFINE>
__global__ void __launch_bounds__(128) quad_diag_kernel(QuadParams p) {
  constexpr int VS = form_vs(FORM, DIM);
  using TB = QuadTables<NQ, ND, NV, DIM>;
  extern __shared__ double smem[];
  for (int i = threadIdx.x; i < TB::size; i += blockDim.x) smem[i] = p.tables[i];
  __syncthreads();
  const double* s_qw = smem + TB::qw;
  const double* s_phi = smem + TB::phi;
  const double* s_dphi = smem + TB::dphi;
  const double* s_gphi = smem + TB::gphi;
  const double* s_gdphi = smem + TB::gdphi;
  const int cell = p.start + blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;
  double X[NV][DIM];
  int vid[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    vid[v] = __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<DIM>(p.mesh.coords, vid[v], X[v]);
  }
  double J[DIM][DIM], Ji[DIM][DIM], absdet = 0.0;
  auto jacobian = [&](int q) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) {
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) s += X[v][a] * s_gdphi[(q * NV + v) * DIM + b];
        J[a][b] = s;
      }
    absdet = fabs(det_inv<DIM>(J, Ji));
  };
  if constexpr (AFFINE) jacobian(0);
#pragma unroll 1
  for (int i = 0; i < ND; ++i) {
    const int dof = __ldg(p.mesh.map + i * cs + cell);
#pragma unroll 1
    for (int c = 0; c < VS; ++c) {
      double acc = 0.0;
#pragma unroll 1
      for (int q = 0; q < NQ; ++q) {
        if constexpr (!AFFINE) jacobian(q);
        const double tw = s_qw[q] * absdet;
        double uq[VS], g[VS][DIM], g0[VS][DIM];
#pragma unroll
        for (int cc = 0; cc < VS; ++cc) {
          uq[cc] = cc == c ? s_phi[q * ND + i] : 0.0;
#pragma unroll
          for (int b = 0; b < DIM; ++b) g[cc][b] = cc == c ? s_dphi[(q * ND + i) * DIM + b] : 0.0;
        }
        if constexpr (form_has_state(FORM)) {
#pragma unroll
          for (int cc = 0; cc < VS; ++cc)
#pragma unroll
            for (int b = 0; b < DIM; ++b) g0[cc][b] = 0.0;
          for (int j = 0; j < ND; ++j) {
            const int dj = __ldg(p.mesh.map + j * cs + cell);
#pragma unroll
            for (int cc = 0; cc < VS; ++cc) {
              const double w0 = __ldg(p.mu + (int64_t)VS * dj + cc);
#pragma unroll
              for (int b = 0; b < DIM; ++b) g0[cc][b] += s_dphi[(q * ND + j) * DIM + b] * w0;
            }
          }
        }
        double mu = p.p0, lam = p.p1;
        if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
          mu = 0.0;
          lam = 0.0;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const double gv = s_gphi[q * NV + v];
            mu += gv * __ldg(p.mu + vid[v]);
            lam += gv * __ldg(p.lam + vid[v]);
          }
        }
        double cv[VS], cg[VS][DIM];
        pointwise<FORM, DIM, VS>(Ji, tw, uq, g, mu, lam, cv, cg, g0);
        if constexpr (form_needs_values(FORM)) acc += s_phi[q * ND + i] * cv[c];
        if constexpr (form_needs_grads(FORM)) {
#pragma unroll
          for (int b = 0; b < DIM; ++b) acc += s_dphi[(q * ND + i) * DIM + b] * cg[c][b];
        }
      }
      griddep_wait();
      scatter_add(p.y, (int64_t)VS * dof + c, acc);
    }
  }
}

// ---------------------------------------------------------------------------
// Quadrature kernel with the tables in the kernel parameter block.
//  * affine simplices (C5: neo-Hookean P2 tetrahedra, 27 points): the
//    Jacobian and its inverse are computed once per cell from vertex
//    differences;
//  * low-order tensor cells (Q1 quads/hexes: C3-Q1, C4-quad-Q1, C4-hex-Q1):
//    the Jacobian is recomputed per point from the vertex basis gradients
//    (kernels.py:136-151), every cell fully in registers -- at p = 2 a
//    team-of-threads sum factorisation only adds synchronisation.
// Every table entry enters its DFMA as a uniform constant-bank operand (all
// threads of a warp read the same entry): no shared-memory traffic at all.
// ---------------------------------------------------------------------------

#ifndef QC_ADJ
#define QC_ADJ 1
#endif
constexpr bool linear_grad_form(int form) {
  return form == FE_FORM_LAPLACIAN_SCALAR || form == FE_FORM_LAPLACIAN || form == FE_FORM_ELASTICITY ||
         form == FE_FORM_ELASTICITY_LAME;
}

template <int NQ, int ND, int DIM, int NV, bool VALUES, bool AFFINE>
struct QuadConstParams {
  MeshView mesh;
  int32_t start, end;
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ mu;
  const double* __restrict__ lam;
  double p0, p1;
  double qw[NQ];
  double phi[VALUES ? NQ : 1][ND];
  double dphi[NQ][ND][DIM];
  double gphi[NQ][NV];
  double px[AFFINE ? 1 : NQ][DIM];  // reference coordinates of the points (tensor cells)
};

// MINB: CTAs of 128 threads per SM the register allocation must allow
// (chosen per variant from measurements)
// UNR: quadrature-loop unroll (table entries become immediate constant-bank
// operands instead of LDC loads; larger unrolls raise register pressure)
template <int FORM, int DIM, int NV, int ND, int NQ, bool AFFINE, int MINB = 1, int UNR = 1>
__global__ void __launch_bounds__(128, MINB)
quad_const_kernel(const __grid_constant__ QuadConstParams<NQ, ND, DIM, NV, form_needs_values(FORM), AFFINE> p) {
  constexpr int VS = form_vs(FORM, DIM);
  const int cell = p.start + blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;
  int dof[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) dof[i] = __ldg(p.mesh.map + i * cs + cell);
  double X[NV][DIM];
  int vid[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    vid[v] = __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<DIM>(p.mesh.coords, vid[v], X[v]);
  }
  double w[ND][VS];
#pragma unroll
  for (int i = 0; i < ND; ++i)
#pragma unroll
    for (int c = 0; c < VS; ++c) w[i][c] = __ldg(p.u + (int64_t)VS * dof[i] + c);
  double w0[form_has_state(FORM) ? ND : 1][VS];
  if constexpr (form_has_state(FORM)) {
#pragma unroll
    for (int i = 0; i < ND; ++i)
#pragma unroll
      for (int c = 0; c < VS; ++c) w0[i][c] = __ldg(p.mu + (int64_t)VS * dof[i] + c);
  }
  double muv[NV], lamv[NV];
  if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      muv[v] = __ldg(p.mu + vid[v]);
      lamv[v] = __ldg(p.lam + vid[v]);
    }
  }
  double J[DIM][DIM], Ji[DIM][DIM], absdet = 0.0;
  // multilinear map x = a0 + a1 xi + a2 eta (+ a3 zeta) + a4 xi eta (+ a5 xi zeta
  // + a6 eta zeta + a7 xi eta zeta): J at a point costs 3 FMAs per entry
  // (2D: 1) instead of a sum over all 2^d vertex-basis gradients
  double cf[DIM == 3 ? 7 : 3][DIM];
  if constexpr (AFFINE) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) J[a][b] = X[b + 1][a] - X[0][a];
    absdet = fabs(det_inv<DIM, true>(J, Ji));
  } else if constexpr (DIM == 3) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      cf[0][d] = X[1][d] - X[0][d];                                   // xi
      cf[1][d] = X[2][d] - X[0][d];                                   // eta
      cf[2][d] = X[4][d] - X[0][d];                                   // zeta
      cf[3][d] = (X[3][d] - X[2][d]) - cf[0][d];                      // xi eta
      cf[4][d] = (X[5][d] - X[4][d]) - cf[0][d];                      // xi zeta
      cf[5][d] = (X[6][d] - X[4][d]) - cf[1][d];                      // eta zeta
      cf[6][d] = ((X[7][d] - X[6][d]) - (X[5][d] - X[4][d])) - (X[3][d] - X[2][d]) + cf[0][d];
    }
  } else {
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      cf[0][d] = X[1][d] - X[0][d];
      cf[1][d] = X[2][d] - X[0][d];
      cf[2][d] = (X[3][d] - X[2][d]) - cf[0][d];
    }
  }
  double A[ND][VS];
#pragma unroll
  for (int i = 0; i < ND; ++i)
#pragma unroll
    for (int c = 0; c < VS; ++c) A[i][c] = 0.0;
#pragma unroll UNR
  for (int q = 0; q < NQ; ++q) {
    if constexpr (!AFFINE) {
      if constexpr (DIM == 3) {
        const double xi = p.px[q][0], eta = p.px[q][1], zeta = p.px[q][2];
        const double ez = eta * zeta, xz = xi * zeta, xe = xi * eta;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          J[d][0] = fma(cf[6][d], ez, fma(cf[4][d], zeta, fma(cf[3][d], eta, cf[0][d])));
          J[d][1] = fma(cf[6][d], xz, fma(cf[5][d], zeta, fma(cf[3][d], xi, cf[1][d])));
          J[d][2] = fma(cf[6][d], xe, fma(cf[5][d], eta, fma(cf[4][d], xi, cf[2][d])));
        }
      } else {
        const double xi = p.px[q][0], eta = p.px[q][1];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          J[d][0] = fma(cf[2][d], eta, cf[0][d]);
          J[d][1] = fma(cf[2][d], xi, cf[1][d]);
        }
      }
      if constexpr (QC_ADJ && linear_grad_form(FORM)) absdet = fabs(det_adj<DIM>(J, Ji));
      else absdet = fabs(det_inv<DIM, true>(J, Ji));
    }
    // linear gradient-only forms on non-affine cells: Ji holds adj(J) and the
    // weight w / |det J| absorbs both 1/det factors (no inverse formed)
    const double tw = (QC_ADJ && !AFFINE && linear_grad_form(FORM)) ? p.qw[q] * rcp(absdet) : p.qw[q] * absdet;
    double uq[VS], g[VS][DIM];
#pragma unroll
    for (int c = 0; c < VS; ++c) {
      uq[c] = 0.0;
#pragma unroll
      for (int b = 0; b < DIM; ++b) g[c][b] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < ND; ++i) {
#pragma unroll
      for (int c = 0; c < VS; ++c) {
        if constexpr (form_needs_values(FORM)) uq[c] = fma(p.phi[q][i], w[i][c], uq[c]);
        if constexpr (form_needs_grads(FORM)) {
#pragma unroll
          for (int b = 0; b < DIM; ++b) g[c][b] = fma(p.dphi[q][i][b], w[i][c], g[c][b]);
        }
      }
    }
    double mu = p.p0, lam = p.p1;
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
      mu = 0.0;
      lam = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        mu = fma(p.gphi[q][v], muv[v], mu);
        lam = fma(p.gphi[q][v], lamv[v], lam);
      }
    }
    double g0[VS][DIM];
    if constexpr (form_has_state(FORM)) {
#pragma unroll
      for (int c = 0; c < VS; ++c)
#pragma unroll
        for (int b = 0; b < DIM; ++b) g0[c][b] = 0.0;
#pragma unroll
      for (int i = 0; i < ND; ++i)
#pragma unroll
        for (int c = 0; c < VS; ++c)
#pragma unroll
          for (int b = 0; b < DIM; ++b) g0[c][b] = fma(p.dphi[q][i][b], w0[i][c], g0[c][b]);
    }
    double cv[VS], cg[VS][DIM];
    pointwise<FORM, DIM, VS, true>(Ji, tw, uq, g, mu, lam, cv, cg, g0);
#pragma unroll
    for (int j = 0; j < ND; ++j)
#pragma unroll
      for (int c = 0; c < VS; ++c) {
        double acc = A[j][c];
        if constexpr (form_needs_values(FORM)) acc = fma(p.phi[q][j], cv[c], acc);
        if constexpr (form_needs_grads(FORM)) {
#pragma unroll
          for (int b = 0; b < DIM; ++b) acc = fma(p.dphi[q][j][b], cg[c][b], acc);
        }
        A[j][c] = acc;
      }
  }
  griddep_wait();
#pragma unroll
  for (int j = 0; j < ND; ++j)
#pragma unroll
    for (int c = 0; c < VS; ++c) scatter_add(p.y, (int64_t)VS * dof[j] + c, A[j][c]);
}

// ---------------------------------------------------------------------------
// Vertex-gradient quadrature kernel for P2 simplices (C5 neo-Hookean, affine
// tetrahedra).  The reference gradient of a P2 field is P1, so it is fixed by
// its values at the 4 vertices: G_v = sum_i dphi_i(vertex v) u_i once per
// cell (360 FMAs), then at every point grad_ref u = sum_v lambda_v(x_q) G_v
// (36 FMAs instead of the 90 of the nodal sum, kernels.py:178-195).  The
// transposed integration likewise accumulates the 4 vertex moments
// S_v = sum_q lambda_v(x_q) flux_q (36 FMAs per point) and projects back to
// the 10 nodes once per cell.  Exact (not an approximation): lambda_v are the
// P1 barycentric functions, the same gphi table the geometry uses.
// ---------------------------------------------------------------------------
#ifndef FE_VTX_PHYS
#define FE_VTX_PHYS 1   // hyperelastic forms: physical vertex gradients / moments (0: reference-gradient loop)
#endif

template <int NQ, int ND, int DIM, int NV>
struct VtxParams {
  MeshView mesh;
  int32_t start, end;
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ mu;
  const double* __restrict__ lam;
  double p0, p1;
  double qw[NQ];
  double gphi[NQ][NV];          // barycentric (P1) values at the points
  double dphiv[NV][ND][DIM];    // reference gradients of the P2 basis at the vertices
};

template <int FORM, int DIM, int NV, int ND, int NQ, int MINB, int UNR>
__global__ void __launch_bounds__(128, MINB)
quad_vtx_kernel(const __grid_constant__ VtxParams<NQ, ND, DIM, NV> p) {
  constexpr int VS = form_vs(FORM, DIM);
  constexpr bool STATE = form_has_state(FORM);
  static_assert(!form_needs_values(FORM), "gradient-only forms");
  const int cell = p.start + blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;
  int dof[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) dof[i] = __ldg(p.mesh.map + i * cs + cell);
  double X[NV][DIM];
#pragma unroll
  for (int v = 0; v < NV; ++v) load_vertex<DIM>(p.mesh.coords, __ldg(p.mesh.vmap + v * cs + cell), X[v]);
  // vertex values of the reference gradient: increment u (and state u0)
  double Gv[NV][VS][DIM], G0v[STATE ? NV : 1][VS][DIM];
  auto vertex_grad = [&](const double* __restrict__ f, double (&out)[NV][VS][DIM]) {
    double w[ND][VS];
#pragma unroll
    for (int i = 0; i < ND; ++i)
#pragma unroll
      for (int c = 0; c < VS; ++c) w[i][c] = __ldg(f + (int64_t)VS * dof[i] + c);
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int c = 0; c < VS; ++c)
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < ND; ++i) s = fma(p.dphiv[v][i][b], w[i][c], s);
          out[v][c][b] = s;
        }
  };
  vertex_grad(p.u, Gv);
  if constexpr (STATE) vertex_grad(p.mu, G0v);
  double J[DIM][DIM], Ji[DIM][DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int b = 0; b < DIM; ++b) J[a][b] = X[b + 1][a] - X[0][a];
  const double absdet = fabs(det_inv<DIM, true>(J, Ji));
  double S[NV][VS][DIM];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int c = 0; c < VS; ++c)
#pragma unroll
      for (int b = 0; b < DIM; ++b) S[v][c][b] = 0.0;
#if FE_VTX_PHYS
  // physical vertex gradients H_v = G_v J^-1 once per cell (affine: J^-1 is
  // constant, so grad u(x_q) = sum_v lambda_v(x_q) H_v exactly); the flux is
  // accumulated as physical vertex moments sum_q lambda_v tw P_q and mapped
  // by J^-T once per cell.  Per point this drops the two 3x3x3 products
  // grad_ref -> grad_phys and P -> P J^-T of the reference quadrature loop.
  if constexpr (FORM == FE_FORM_NEOHOOKEAN || FORM == FE_FORM_NEOHOOKEAN_TANGENT) {
    static_assert(VS == DIM, "vector form");
    auto to_phys = [&](double (&Gr)[NV][VS][DIM]) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int c = 0; c < VS; ++c) {
          double h[DIM];
#pragma unroll
          for (int a = 0; a < DIM; ++a) {
            double t = 0.0;
#pragma unroll
            for (int b = 0; b < DIM; ++b) t = fma(Gr[v][c][b], Ji[b][a], t);
            h[a] = t;
          }
#pragma unroll
          for (int a = 0; a < DIM; ++a) Gr[v][c][a] = h[a];
        }
    };
    to_phys(Gv);
    if constexpr (STATE) to_phys(G0v);
    const double mu = p.p0, lam = p.p1;
#pragma unroll UNR
    for (int q = 0; q < NQ; ++q) {
      const double tw = p.qw[q] * absdet;
      double G[DIM][DIM], F[DIM][DIM], A[DIM][DIM], T[DIM][DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          double t = 0.0, t0 = 0.0;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            t = fma(p.gphi[q][v], Gv[v][c][a], t);
            if constexpr (STATE) t0 = fma(p.gphi[q][v], G0v[v][c][a], t0);
          }
          G[c][a] = t;
          F[c][a] = (STATE ? t0 : t) + (c == a ? 1.0 : 0.0);
        }
      const double Jf = det_adj<DIM>(F, A);
      const double m = tw * mu;
      if constexpr (FORM == FE_FORM_NEOHOOKEAN) {
        // P = mu G + mu I + (lambda ln J - mu) F^-T, F^-T[c][a] = A[a][c] / J
        const double sc = tw * (lam * FE_LOG(Jf) - mu) * recip<true>(Jf);
#pragma unroll
        for (int c = 0; c < DIM; ++c)
#pragma unroll
          for (int a = 0; a < DIM; ++a) T[c][a] = fma(m, G[c][a], sc * A[a][c]) + (c == a ? m : 0.0);
      } else {
        // dP = mu dF + (mu - lambda ln J) F^-T dF^T F^-T + lambda tr(F^-1 dF) F^-T
        // (pointwise<>, NEOHOOKEAN_TANGENT), dF = G, M = A dF
        const double r = recip<true>(Jf);
        double M[DIM][DIM], tr = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int b = 0; b < DIM; ++b) {
            double t = 0.0;
#pragma unroll
            for (int c = 0; c < DIM; ++c) t = fma(A[a][c], G[c][b], t);
            M[a][b] = t;
            if (a == b) tr += t;
          }
        const double r2 = tw * r * r;
        const double c2 = (mu - lam * FE_LOG(Jf)) * r2;
        const double l2 = lam * tr * r2;
#pragma unroll
        for (int c = 0; c < DIM; ++c)
#pragma unroll
          for (int a = 0; a < DIM; ++a) {
            double t = 0.0;
#pragma unroll
            for (int b = 0; b < DIM; ++b) t = fma(M[a][b], A[b][c], t);
            T[c][a] = fma(m, G[c][a], fma(c2, t, l2 * A[a][c]));
          }
      }
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int c = 0; c < DIM; ++c)
#pragma unroll
          for (int a = 0; a < DIM; ++a) S[v][c][a] = fma(p.gphi[q][v], T[c][a], S[v][c][a]);
    }
    // physical moments -> reference: S_v J^-T
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        double h[DIM];
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
          double t = 0.0;
#pragma unroll
          for (int a = 0; a < DIM; ++a) t = fma(Ji[b][a], S[v][c][a], t);
          h[b] = t;
        }
#pragma unroll
        for (int b = 0; b < DIM; ++b) S[v][c][b] = h[b];
      }
  } else
#endif
  {
#pragma unroll UNR
  for (int q = 0; q < NQ; ++q) {
    const double tw = p.qw[q] * absdet;
    double g[VS][DIM], g0[VS][DIM], uq[VS] = {};
#pragma unroll
    for (int c = 0; c < VS; ++c)
#pragma unroll
      for (int b = 0; b < DIM; ++b) {
        double s = 0.0, s0 = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          s = fma(p.gphi[q][v], Gv[v][c][b], s);
          if constexpr (STATE) s0 = fma(p.gphi[q][v], G0v[v][c][b], s0);
        }
        g[c][b] = s;
        g0[c][b] = s0;
      }
    double cv[VS], cg[VS][DIM];
    pointwise<FORM, DIM, VS, true>(Ji, tw, uq, g, p.p0, p.p1, cv, cg, g0);
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int c = 0; c < VS; ++c)
#pragma unroll
        for (int b = 0; b < DIM; ++b) S[v][c][b] = fma(p.gphi[q][v], cg[c][b], S[v][c][b]);
  }
  }
  griddep_wait();
#pragma unroll
  for (int j = 0; j < ND; ++j)
#pragma unroll
    for (int c = 0; c < VS; ++c) {
      double s = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int b = 0; b < DIM; ++b) s = fma(p.dphiv[v][j][b], S[v][c][b], s);
      scatter_add(p.y, (int64_t)VS * dof[j] + c, s);
    }
}

}  // namespace fe
