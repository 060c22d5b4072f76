// Thread-per-cell sum-factorised scalar Laplacian for trilinear Q1
// hexahedra on the 2x2x2 Gauss rule (C3-Q1).
//
// The quad_const_tensor kernel evaluates the reference gradient at each of
// the 8 points as a dense 8-term sum (and integrates back the same way): 384
// MACs per cell.  Here both directions are sum-factorised over the whole
// 2x2x2 tile held in registers (x, then y, then z contractions with the 1D
// value/derivative matrices B, D -- the reference's tabulate() factored per
// direction, elements.py:233-254): 128 MACs each way.  The pointwise flux
// uses the adjugate form of the reference's J^-1 J^-T (kernels.py:205-220):
//     f = (w_q / |det J|) adj(J) (adj(J)^T g_ref),
// with J from the multilinear-map coefficients (3 FMAs per entry), so no
// explicit inverse is formed.  Every table entry is a uniform constant-bank
// operand (kernel parameter block).
#pragma once
#include "common.cuh"
#include "kern_tensor.cuh"

namespace fe {

// The Q1 basis on [0,1] has B[a] = (1 - x_a, x_a) and D = (-1, 1) at every
// point (checked at plan time), so every contraction along a derivative
// direction is a difference and every value contraction one FMA on a
// difference: the reference gradient components depend on two of the three
// point indices only (d/dxi on (c, b), d/deta on (c, a), d/dzeta on (b, a)),
// and so do the Jacobian's columns.  ~650 FP64 instructions per cell
// instead of ~870.
template <int MINB>
__global__ void __launch_bounds__(128, MINB)
hexq1_lap_kernel(const __grid_constant__ TensorParams<2, 2> p) {
  const int cell = p.start + blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;
  int dof[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) dof[i] = __ldg(p.mesh.map + i * cs + cell);
  double X[8][3], u[2][2][2];  // u[k][j][i], i = x
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int vid = (p.mesh.vmap == p.mesh.map) ? dof[v] : __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<3>(p.mesh.coords, vid, X[v]);
    u[v >> 2][(v >> 1) & 1][v & 1] = __ldg(p.u + dof[v]);
  }
  const double x0 = p.x[0], x1 = p.x[1];
  const double xs[2] = {x0, x1};
  // multilinear map coefficients of the derivative terms
  double cf[7][3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    cf[0][d] = X[1][d] - X[0][d];
    cf[1][d] = X[2][d] - X[0][d];
    cf[2][d] = X[4][d] - X[0][d];
    cf[3][d] = (X[3][d] - X[2][d]) - cf[0][d];
    cf[4][d] = (X[5][d] - X[4][d]) - cf[0][d];
    cf[5][d] = (X[6][d] - X[4][d]) - cf[1][d];
    cf[6][d] = ((X[7][d] - X[6][d]) - (X[5][d] - X[4][d])) - (X[3][d] - X[2][d]) + cf[0][d];
  }
  // Jacobian columns: dx/dxi on (b, c), dx/deta on (a, c), dx/dzeta on (a, b)
  double Jx[2][2][3], Jy[2][2][3], Jz[2][2][3];
#pragma unroll
  for (int s1 = 0; s1 < 2; ++s1)
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const double e = xs[s1], z = xs[s2], ez = xs[s1] * xs[s2];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        Jx[s1][s2][d] = fma(cf[6][d], ez, fma(cf[4][d], z, fma(cf[3][d], e, cf[0][d])));  // (eta_b, zeta_c)
        Jy[s1][s2][d] = fma(cf[6][d], ez, fma(cf[5][d], z, fma(cf[3][d], e, cf[1][d])));  // (xi_a, zeta_c)
        Jz[s1][s2][d] = fma(cf[6][d], ez, fma(cf[5][d], z, fma(cf[4][d], e, cf[2][d])));  // (xi_a, eta_b)
      }
    }
  // forward contractions
  double xd[2][2], xb[2][2][2];  // [k][j], [k][j][a]
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      xd[k][j] = u[k][j][1] - u[k][j][0];
#pragma unroll
      for (int a = 0; a < 2; ++a) xb[k][j][a] = fma(xs[a], xd[k][j], u[k][j][0]);
    }
  double db[2][2], bb[2][2][2], bd[2][2];  // db[k][a], bb[k][b][a], bd[k][b]
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double dd = xd[k][1] - xd[k][0];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      db[k][a] = xb[k][1][a] - xb[k][0][a];
#pragma unroll
      for (int b = 0; b < 2; ++b) bb[k][b][a] = fma(xs[b], db[k][a], xb[k][0][a]);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) bd[k][b] = fma(xs[b], dd, xd[k][0]);
  }
  double gx[2][2], gy[2][2], gz[2][2];  // gx[c][b], gy[c][a], gz[b][a]
#pragma unroll
  for (int s1 = 0; s1 < 2; ++s1) {
    const double dx = bd[1][s1] - bd[0][s1], dy = db[1][s1] - db[0][s1];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      gx[c][s1] = fma(xs[c], dx, bd[0][s1]);
      gy[c][s1] = fma(xs[c], dy, db[0][s1]);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) gz[s1][a] = bb[1][s1][a] - bb[0][s1][a];
  }
  // pointwise adjugate-form flux at the 8 points
  double f[2][2][2][3];  // [c][b][a][dir]
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        double J[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          J[d][0] = Jx[b][c][d];
          J[d][1] = Jy[a][c][d];
          J[d][2] = Jz[a][b][d];
        }
        double A[3][3];
        const double det = det_adj<3>(J, A);
        const double s = p.w[a] * p.w[b] * p.w[c] * rcp(fabs(det));
        const double g[3] = {gx[c][b], gy[c][a], gz[b][a]};
        double t[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) t[e] = s * fma(A[2][e], g[2], fma(A[1][e], g[1], A[0][e] * g[0]));
#pragma unroll
        for (int r = 0; r < 3; ++r) f[c][b][a][r] = fma(A[r][2], t[2], fma(A[r][1], t[1], A[r][0] * t[0]));
      }
  // backward (transposed) contractions: sum_c B[c][k] v_c = (k ? T : S - T)
  // with S = v_0 + v_1, T = x_0 v_0 + x_1 v_1; sum_c D[c][k] v_c = (k ? S : -S)
  double tx[2][2][2], ty[2][2][2], sz[2][2];  // [k][b][a], sz[b][a]
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const double T0 = fma(x1, f[1][b][a][0], x0 * f[0][b][a][0]);
      const double T1 = fma(x1, f[1][b][a][1], x0 * f[0][b][a][1]);
      tx[1][b][a] = T0;
      tx[0][b][a] = (f[0][b][a][0] + f[1][b][a][0]) - T0;
      ty[1][b][a] = T1;
      ty[0][b][a] = (f[0][b][a][1] + f[1][b][a][1]) - T1;
      sz[b][a] = f[0][b][a][2] + f[1][b][a][2];  // tz[k] = (k ? sz : -sz)
    }
  double s1[2][2][2], s2[2][2][2];  // [k][j][a]
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const double Qs = sz[0][a] + sz[1][a];
    const double Q1 = fma(x1, sz[1][a], x0 * sz[0][a]);
    const double Q[2] = {Qs - Q1, Q1};  // sum_b B[b][j] sz[b][a]
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double T = fma(x1, tx[k][1][a], x0 * tx[k][0][a]);
      s1[k][1][a] = T;
      s1[k][0][a] = (tx[k][0][a] + tx[k][1][a]) - T;
      const double Dy = ty[k][0][a] + ty[k][1][a];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double dpart = j ? Dy : -Dy;
        s2[k][j][a] = k ? dpart + Q[j] : dpart - Q[j];
      }
    }
  }
  griddep_wait();
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double Sd = s1[k][j][0] + s1[k][j][1];
      const double R1 = fma(x1, s2[k][j][1], x0 * s2[k][j][0]);
      const double R0 = (s2[k][j][0] + s2[k][j][1]) - R1;
      scatter_add(p.y, dof[4 * k + 2 * j + 0], R0 - Sd);
      scatter_add(p.y, dof[4 * k + 2 * j + 1], R1 + Sd);
    }
}

}  // namespace fe
