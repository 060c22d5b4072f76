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
  // multilinear map x = a0 + a1 xi + a2 eta + a3 zeta + a4 xi eta + a5 xi zeta
  // + a6 eta zeta + a7 xi eta zeta (coefficients of the derivative terms)
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
  // forward: reference gradients g[c][b][a][dir] at point (x_a, x_b, x_c)
  double xb[2][2][2], xd[2][2][2];  // [k][j][a]
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        xb[k][j][a] = fma(p.B[a][1], u[k][j][1], p.B[a][0] * u[k][j][0]);
        xd[k][j][a] = fma(p.D[a][1], u[k][j][1], p.D[a][0] * u[k][j][0]);
      }
  double bb[2][2][2], db[2][2][2], bd[2][2][2];  // [k][b][a]: y-contractions
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        bb[k][b][a] = fma(p.B[b][1], xb[k][1][a], p.B[b][0] * xb[k][0][a]);
        db[k][b][a] = fma(p.D[b][1], xb[k][1][a], p.D[b][0] * xb[k][0][a]);
        bd[k][b][a] = fma(p.B[b][1], xd[k][1][a], p.B[b][0] * xd[k][0][a]);
      }
  double f[2][2][2][3];  // gradient, then flux, at point [c][b][a]
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        f[c][b][a][0] = fma(p.B[c][1], bd[1][b][a], p.B[c][0] * bd[0][b][a]);
        f[c][b][a][1] = fma(p.B[c][1], db[1][b][a], p.B[c][0] * db[0][b][a]);
        f[c][b][a][2] = fma(p.D[c][1], bb[1][b][a], p.D[c][0] * bb[0][b][a]);
      }
  // pointwise adjugate-form flux
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const double xi = p.x[a], eta = p.x[b], zeta = p.x[c];
        const double ez = eta * zeta, xz = xi * zeta, xe = xi * eta;
        double J[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          J[d][0] = fma(cf[6][d], ez, fma(cf[4][d], zeta, fma(cf[3][d], eta, cf[0][d])));
          J[d][1] = fma(cf[6][d], xz, fma(cf[5][d], zeta, fma(cf[3][d], xi, cf[1][d])));
          J[d][2] = fma(cf[6][d], xe, fma(cf[5][d], eta, fma(cf[4][d], xi, cf[2][d])));
        }
        // adj[r][s]: J^-1 = adj / det (J^-1[r][s] = dxi_r/dx_s)
        double A[3][3];
        A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
        A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
        A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
        A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
        A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
        A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double det = J[0][0] * A[0][0] + J[0][1] * A[1][0] + J[0][2] * A[2][0];
        const double s = (p.w[a] * p.w[b] * p.w[c]) * rcp(fabs(det));
        double* g = f[c][b][a];
        // t = adj^T g (physical gradient times det), scaled by w / |det|
        double t[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) t[e] = s * fma(A[2][e], g[2], fma(A[1][e], g[1], A[0][e] * g[0]));
#pragma unroll
        for (int r = 0; r < 3; ++r) g[r] = fma(A[r][2], t[2], fma(A[r][1], t[1], A[r][0] * t[0]));
      }
  // backward (transposed contractions): z, then y, then x
  double tx[2][2][2], ty[2][2][2], tz[2][2][2];  // [k][b][a]
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        tx[k][b][a] = fma(p.B[1][k], f[1][b][a][0], p.B[0][k] * f[0][b][a][0]);
        ty[k][b][a] = fma(p.B[1][k], f[1][b][a][1], p.B[0][k] * f[0][b][a][1]);
        tz[k][b][a] = fma(p.D[1][k], f[1][b][a][2], p.D[0][k] * f[0][b][a][2]);
      }
  double s1[2][2][2], s2[2][2][2];  // [k][j][a]
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        s1[k][j][a] = fma(p.B[1][j], tx[k][1][a], p.B[0][j] * tx[k][0][a]);
        s2[k][j][a] = fma(p.D[1][j], ty[k][1][a], fma(p.D[0][j], ty[k][0][a],
                      fma(p.B[1][j], tz[k][1][a], p.B[0][j] * tz[k][0][a])));
      }
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double yv = fma(p.D[1][i], s1[k][j][1], fma(p.D[0][i], s1[k][j][0],
                          fma(p.B[1][i], s2[k][j][1], p.B[0][i] * s2[k][j][0])));
        scatter_add(p.y, dof[4 * k + 2 * j + i], yv);
      }
}

}  // namespace fe
