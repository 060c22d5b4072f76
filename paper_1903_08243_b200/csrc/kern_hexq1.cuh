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


// ---------------------------------------------------------------------------
// Thread-per-cell sum-factorised scalar Laplacian for Q2 hexahedra on the
// 3x3x3 Gauss rule (C3-Q2), collocation form (12 q^4 MACs):
//   interpolate u to the Gauss points with three B contractions (in
//   registers), then per point differentiate with the collocation matrix Dc
//   along the three lines through it (9 MACs), apply the adjugate-form flux
//   and accumulate its Dc^T contributions into a point-space output (9 MACs);
//   three B^T contractions bring that back to the 27 dofs.
// The whole cell lives in one thread's registers (27 point values + 27
// outputs + the 21 monomial map coefficients): no shared memory, no barriers,
// no shuffles -- the team kernels spend ~45% of their issue slots on those
// (plane_t at Q = 3: FP64 pipe 53% active, profiles/r01/ncu13_summaries.txt).
// All 24 table entries (B, Dc, x, w) stay resident in uniform registers.
// ---------------------------------------------------------------------------
struct HexQ2Params {
  MeshView mesh;
  const double* __restrict__ u;
  double* __restrict__ y;
  int32_t start, end;
  int32_t lex[27];      // local dof of tensor node n = i + 3 j + 9 k
  double B[3][3], Dc[3][3], x[3], w[3];
};

template <int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
hexq2_lap_kernel(const __grid_constant__ HexQ2Params p) {
  constexpr int Q = 3;
  const int cell = p.start + blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;
  double uq[Q][Q][Q];  // [k][j][i] dof values, then [c][b][a] point values
#pragma unroll
  for (int n = 0; n < 27; ++n)
    uq[n / 9][(n / 3) % 3][n % 3] = __ldg(p.u + __ldg(p.mesh.map + p.lex[n] * cs + cell));
  double cf[7][3];
  {
    double X[8][3];
#pragma unroll
    for (int v = 0; v < 8; ++v) load_vertex<3>(p.mesh.coords, __ldg(p.mesh.vmap + v * cs + cell), X[v]);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      cf[0][d] = X[1][d] - X[0][d];                       // xi
      cf[1][d] = X[2][d] - X[0][d];                       // eta
      cf[2][d] = X[4][d] - X[0][d];                       // zeta
      cf[3][d] = (X[3][d] - X[2][d]) - cf[0][d];          // xi eta
      cf[4][d] = (X[5][d] - X[4][d]) - cf[0][d];          // xi zeta
      cf[5][d] = (X[6][d] - X[4][d]) - cf[1][d];          // eta zeta
      cf[6][d] = ((X[7][d] - X[6][d]) - (X[5][d] - X[4][d])) - (X[3][d] - X[2][d]) + cf[0][d];
    }
  }
  // ---- u at the Gauss points: B along x, y, z --------------------------------
#pragma unroll
  for (int k = 0; k < Q; ++k)
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const double v0 = uq[k][j][0], v1 = uq[k][j][1], v2 = uq[k][j][2];
#pragma unroll
      for (int a = 0; a < Q; ++a) uq[k][j][a] = fma(p.B[a][2], v2, fma(p.B[a][1], v1, p.B[a][0] * v0));
    }
#pragma unroll
  for (int k = 0; k < Q; ++k)
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const double v0 = uq[k][0][a], v1 = uq[k][1][a], v2 = uq[k][2][a];
#pragma unroll
      for (int b = 0; b < Q; ++b) uq[k][b][a] = fma(p.B[b][2], v2, fma(p.B[b][1], v1, p.B[b][0] * v0));
    }
#pragma unroll
  for (int b = 0; b < Q; ++b)
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const double v0 = uq[0][b][a], v1 = uq[1][b][a], v2 = uq[2][b][a];
#pragma unroll
      for (int c = 0; c < Q; ++c) uq[c][b][a] = fma(p.B[c][2], v2, fma(p.B[c][1], v1, p.B[c][0] * v0));
    }
  // ---- points: gradient, flux, transposed collocation derivative --------------
  double out[Q][Q][Q];
#pragma unroll
  for (int n = 0; n < 27; ++n) out[n / 9][(n / 3) % 3][n % 3] = 0.0;
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    const double zeta = p.x[c];
    double A0[3], A1[3], B0[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      A0[d] = fma(zeta, cf[4][d], cf[0][d]);   // dx/dxi   = A0 + eta A1
      A1[d] = fma(zeta, cf[6][d], cf[3][d]);   // dx/deta  = B0 + xi A1
      B0[d] = fma(zeta, cf[5][d], cf[1][d]);
    }
#pragma unroll
    for (int b = 0; b < Q; ++b) {
      const double eta = p.x[b], wbc = p.w[b] * p.w[c];
      double Jx[3], C0[3], C1[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        Jx[d] = fma(eta, A1[d], A0[d]);
        C0[d] = fma(eta, cf[5][d], cf[2][d]);  // dx/dzeta = C0 + xi C1
        C1[d] = fma(eta, cf[6][d], cf[4][d]);
      }
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        const double xi = p.x[a];
        double J[3][3], A[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          J[d][0] = Jx[d];
          J[d][1] = fma(xi, A1[d], B0[d]);
          J[d][2] = fma(xi, C1[d], C0[d]);
        }
        const double det = det_adj<3>(J, A);
        const double s = (p.w[a] * wbc) * rcp(fabs(det));
        double g[3];
        g[0] = fma(p.Dc[a][2], uq[c][b][2], fma(p.Dc[a][1], uq[c][b][1], p.Dc[a][0] * uq[c][b][0]));
        g[1] = fma(p.Dc[b][2], uq[c][2][a], fma(p.Dc[b][1], uq[c][1][a], p.Dc[b][0] * uq[c][0][a]));
        g[2] = fma(p.Dc[c][2], uq[2][b][a], fma(p.Dc[c][1], uq[1][b][a], p.Dc[c][0] * uq[0][b][a]));
        double t[3], f[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) t[e] = s * fma(A[2][e], g[2], fma(A[1][e], g[1], A[0][e] * g[0]));
#pragma unroll
        for (int r = 0; r < 3; ++r) f[r] = fma(A[r][2], t[2], fma(A[r][1], t[1], A[r][0] * t[0]));
#pragma unroll
        for (int e = 0; e < Q; ++e) {
          out[c][b][e] = fma(p.Dc[a][e], f[0], out[c][b][e]);
          out[c][e][a] = fma(p.Dc[b][e], f[1], out[c][e][a]);
          out[e][b][a] = fma(p.Dc[c][e], f[2], out[e][b][a]);
        }
      }
    }
  }
  // ---- back to the dofs: B^T along z, y, x ------------------------------------
#pragma unroll
  for (int b = 0; b < Q; ++b)
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const double v0 = out[0][b][a], v1 = out[1][b][a], v2 = out[2][b][a];
#pragma unroll
      for (int k = 0; k < Q; ++k) out[k][b][a] = fma(p.B[2][k], v2, fma(p.B[1][k], v1, p.B[0][k] * v0));
    }
#pragma unroll
  for (int k = 0; k < Q; ++k)
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const double v0 = out[k][0][a], v1 = out[k][1][a], v2 = out[k][2][a];
#pragma unroll
      for (int j = 0; j < Q; ++j) out[k][j][a] = fma(p.B[2][j], v2, fma(p.B[1][j], v1, p.B[0][j] * v0));
    }
  griddep_wait();
#pragma unroll
  for (int k = 0; k < Q; ++k)
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const double v0 = out[k][j][0], v1 = out[k][j][1], v2 = out[k][j][2];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const double r = fma(p.B[2][i], v2, fma(p.B[1][i], v1, p.B[0][i] * v0));
        scatter_add(p.y, __ldg(p.mesh.map + p.lex[i + 3 * j + 9 * k] * cs + cell), r);
      }
    }
}


// ---------------------------------------------------------------------------
// Lane-per-plane, shuffle-exchanged sum-factorised scalar Laplacian for Qk
// hexahedra on the (k+1)^3 Gauss rule, k = 3, 4 (C3-Q3, C3-Q4).
//
// The thread-per-cell kernel above stops at Q = 3 points per direction (the
// cell no longer fits one thread's registers).  Here a team of Q lanes owns a
// cell, lane c holding z-plane c: its dof plane, then the point plane
// uq[c][.][.] and the point-space output plane (2 Q^2 doubles).  The x and y
// contractions are local to a lane and use compile-time table entries
// (uniform-register operands); the four z contractions (B_z, Dc_z, Dc_z^T,
// B_z^T) exchange the Q values of a z line with Q warp shuffles per point and
// multiply by the lane's row / column of the table (4 Q doubles in vector
// registers).  Collocation form: 12 q^4 MACs.  No shared memory, no
// barriers, no loop over cells (straight-line code, one cell per team): the
// two things that hold the plane / team kernels near 55% FP64 pipe activity
// on sm_100a (table constants hoisted out of persistent loops, shared-memory
// round trips with barriers) are absent.
// ---------------------------------------------------------------------------
template <int Q>
struct HexLPParams {
  MeshView mesh;
  const int32_t* __restrict__ maplex;   // row-major [ncells][Q^3], tensor (x fastest) order
  const double* __restrict__ u;
  double* __restrict__ y;
  int32_t start, end;
  double B[Q][Q], Dc[Q][Q], x[Q], w[Q];
};

template <int Q, int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
hexlp_lap_kernel(const __grid_constant__ HexLPParams<Q> p) {
  constexpr int TPW = 32 / Q, QQ = Q * Q, ND = Q * Q * Q;
  const int lane = threadIdx.x & 31;
  const int T = lane / Q, c = lane % Q;
  const int gw = blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5);
  const int cell_raw = p.start + gw * TPW + T;
  const bool live = T < TPW && cell_raw < p.end;
  const int cell = live ? cell_raw : p.start;      // idle lanes compute on a valid cell, never scatter
  const int base = (T < TPW ? T : 0) * Q;          // first lane of the team
  const int cc = T < TPW ? c : 0;
  const int64_t cs = p.mesh.nc_stride;
  const unsigned FULL = 0xffffffffu;
  // the lane's rows / columns of the z tables and its zeta, weight
  double Bzr[Q], Bzc[Q], Dzr[Q], Dzc[Q];
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    Bzr[k] = p.B[cc][k];
    Bzc[k] = p.B[k][cc];
    Dzr[k] = p.Dc[cc][k];
    Dzc[k] = p.Dc[k][cc];
  }
  const double zeta = p.x[cc], wc = p.w[cc];
  // dof plane k = cc
  const int32_t* mrow = p.maplex + (int64_t)cell * ND + cc * QQ;
  double uq[Q][Q];   // [j][i] dof plane, then [b][a] point plane
#pragma unroll
  for (int e = 0; e < QQ; ++e) uq[e / Q][e % Q] = __ldg(p.u + __ldg(mrow + e));
  double cf[7][3];
  {
    double X[8][3];
#pragma unroll
    for (int v = 0; v < 8; ++v) load_vertex<3>(p.mesh.coords, __ldg(p.mesh.vmap + v * cs + cell), X[v]);
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
  }
  // ---- B along x, then y, on the lane's dof plane -----------------------------
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = uq[j][i];
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      double s = p.B[a][0] * v[0];
#pragma unroll
      for (int i = 1; i < Q; ++i) s = fma(p.B[a][i], v[i], s);
      uq[j][a] = s;
    }
  }
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    double v[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) v[j] = uq[j][a];
#pragma unroll
    for (int b = 0; b < Q; ++b) {
      double s = p.B[b][0] * v[0];
#pragma unroll
      for (int j = 1; j < Q; ++j) s = fma(p.B[b][j], v[j], s);
      uq[b][a] = s;
    }
  }
  // ---- B along z: the Q values of a z line live in the team's Q lanes ---------
#pragma unroll
  for (int e = 0; e < QQ; ++e) {
    const double v = uq[e / Q][e % Q];
    double s = Bzr[0] * __shfl_sync(FULL, v, base);
#pragma unroll
    for (int k = 1; k < Q; ++k) s = fma(Bzr[k], __shfl_sync(FULL, v, base + k), s);
    uq[e / Q][e % Q] = s;
  }
  // ---- points of plane cc: gradient, flux, transposed collocation derivative --
  double out[Q][Q];
#pragma unroll
  for (int e = 0; e < QQ; ++e) out[e / Q][e % Q] = 0.0;
  double A0[3], A1[3], B0[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    A0[d] = fma(zeta, cf[4][d], cf[0][d]);   // dx/dxi   = A0 + eta A1
    A1[d] = fma(zeta, cf[6][d], cf[3][d]);   // dx/deta  = B0 + xi A1
    B0[d] = fma(zeta, cf[5][d], cf[1][d]);
  }
#pragma unroll
  for (int b = 0; b < Q; ++b) {
    const double eta = p.x[b], wbc = p.w[b] * wc;
    double Jx[3], C0[3], C1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      Jx[d] = fma(eta, A1[d], A0[d]);
      C0[d] = fma(eta, cf[5][d], cf[2][d]);  // dx/dzeta = C0 + xi C1
      C1[d] = fma(eta, cf[6][d], cf[4][d]);
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const double xi = p.x[a];
      double J[3][3], A[3][3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        J[d][0] = Jx[d];
        J[d][1] = fma(xi, A1[d], B0[d]);
        J[d][2] = fma(xi, C1[d], C0[d]);
      }
      const double det = det_adj<3>(J, A);
      const double s = (p.w[a] * wbc) * rcp(fabs(det));
      double g[3];
      g[0] = p.Dc[a][0] * uq[b][0];
      g[1] = p.Dc[b][0] * uq[0][a];
#pragma unroll
      for (int e = 1; e < Q; ++e) {
        g[0] = fma(p.Dc[a][e], uq[b][e], g[0]);
        g[1] = fma(p.Dc[b][e], uq[e][a], g[1]);
      }
      {
        const double v = uq[b][a];
        g[2] = Dzr[0] * __shfl_sync(FULL, v, base);
#pragma unroll
        for (int e = 1; e < Q; ++e) g[2] = fma(Dzr[e], __shfl_sync(FULL, v, base + e), g[2]);
      }
      double t[3], f[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) t[e] = s * fma(A[2][e], g[2], fma(A[1][e], g[1], A[0][e] * g[0]));
#pragma unroll
      for (int r = 0; r < 3; ++r) f[r] = fma(A[r][2], t[2], fma(A[r][1], t[1], A[r][0] * t[0]));
#pragma unroll
      for (int e = 0; e < Q; ++e) {
        out[b][e] = fma(p.Dc[a][e], f[0], out[b][e]);
        out[e][a] = fma(p.Dc[b][e], f[1], out[e][a]);
      }
      // Dc_z^T: plane e collects sum_c Dc[c][e] f_zeta(c) of this point's z line
      double z = out[b][a];
#pragma unroll
      for (int k = 0; k < Q; ++k) z = fma(Dzc[k], __shfl_sync(FULL, f[2], base + k), z);
      out[b][a] = z;
    }
  }
  // ---- B^T along z (shuffles), then y, then x on the lane's plane -------------
#pragma unroll
  for (int e = 0; e < QQ; ++e) {
    const double v = out[e / Q][e % Q];
    double s = Bzc[0] * __shfl_sync(FULL, v, base);
#pragma unroll
    for (int k = 1; k < Q; ++k) s = fma(Bzc[k], __shfl_sync(FULL, v, base + k), s);
    out[e / Q][e % Q] = s;
  }
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    double v[Q];
#pragma unroll
    for (int b = 0; b < Q; ++b) v[b] = out[b][a];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      double s = p.B[0][j] * v[0];
#pragma unroll
      for (int b = 1; b < Q; ++b) s = fma(p.B[b][j], v[b], s);
      out[j][a] = s;
    }
  }
  griddep_wait();
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    double v[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) v[a] = out[j][a];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      double s = p.B[0][i] * v[0];
#pragma unroll
      for (int a = 1; a < Q; ++a) s = fma(p.B[a][i], v[a], s);
      if (live) scatter_add(p.y, __ldg(mrow + j * Q + i), s);
    }
  }
}

}  // namespace fe
