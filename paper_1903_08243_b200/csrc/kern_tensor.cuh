// Sum-factorised kernels for quadrilaterals and hexahedra (C3 scalar
// Laplacian Qk hex, C4 Lame elasticity Qk quad/hex; also the reference's
// vector Laplacian / elasticity and the neo-Hookean residual on tensor cells).
//
// The reference evaluates every basis function at every quadrature point
// (kernels.py:178-195, cost nd*nq per field).  On a tensor-product cell the
// same sums factor into 1D contractions with B[q][p] (1D basis values at
// the 1D Gauss points) and D[q][p] (1D derivatives).  Two algorithms
// (SURVEY.md Appendix B):
//  * "direct" (any p, q): du/dxi = (D x B x B) u, du/deta = (B x D x B) u,
//    du/dzeta = (B x B x D) u as z-, y-, x-contractions sharing partial
//    results (4qp^3 + 6q^2p^2 + 6q^3p per component);
//  * "collocation" (3D, p == q, the BASELINE C3 rule): interpolate u to the
//    Gauss points with three B contractions, then differentiate there with
//    the q x q collocation matrix Dc in each direction (12 q^4 instead of
//    16 q^4 per component).  Exact: along every line u is a degree-(q-1)
//    polynomial, which its q Gauss values determine.
// followed by the pointwise flux and the transposed chain back to the nodes.
//
// GPU mapping: a TEAM of Q^2 threads (3D) or Q threads (2D) per cell,
// 256-thread CTAs holding 256/team cells.  Every contraction stage assigns
// one thread per 1D pencil: the thread loads the inputs along the
// contraction direction from shared memory into registers once and emits a
// whole output pencil, so each shared-memory load feeds Q FMAs; B, D and Dc
// are passed by value in the kernel parameter block and enter the DFMAs as
// uniform constant-bank operands.  After the x-stage one thread holds all Q
// points of an x-pencil and evaluates the flux there: the trilinear Jacobian
// is recomputed per point (as kernels.py:136-151 does per qp on quads) from
// per-thread factors -- its d/dxi column is constant along the pencil and
// the other two are linear in xi (6 FMAs per point).
#pragma once
#include "common.cuh"
#include "kern_quad.cuh"

namespace fe {

template <int Q, int P>
struct TensorParams {
  MeshView mesh;
  const int32_t* __restrict__ maplex;  // row-major [ncells][P^DIM], tensor (x fastest) order
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ mu;
  const double* __restrict__ lam;
  int32_t start, end;
  double p0, p1;
  double B[Q][P], D[Q][P], Dc[Q][Q], x[Q], w[Q];
};

template <int DIM, int P, int Q, int VS>
struct TensorSmem {
  static constexpr int ND = DIM == 3 ? P * P * P : P * P;
  static constexpr int NV = DIM == 3 ? 8 : 4;
  static constexpr int U = 0;
  static constexpr int Z = U + VS * ND;                          // 3D: 2 x Q P^2
  static constexpr int Y = Z + (DIM == 3 ? 2 * Q * P * P : 0);    // 3D: 3 x Q^2 P; 2D: 2 x Q P
  static constexpr int X = Y + (DIM == 3 ? 3 * Q * Q * P : 2 * Q * P);
  static constexpr int MU = X + NV * DIM;
  static constexpr int LAM = MU + NV;
  static constexpr int size = LAM + NV;
};

template <int FORM, int DIM, int P, int Q>
__global__ void __launch_bounds__(256)
tensor_kernel(const __grid_constant__ TensorParams<Q, P> p) {
  static_assert(Q >= P, "team layout assumes Q >= P");
  constexpr int VS = form_vs(FORM, DIM);
  constexpr int TS = DIM == 3 ? Q * Q : Q;
  constexpr int CPB = 256 / TS;
  constexpr bool COLLOC = DIM == 3 && P == Q;
  using SM = TensorSmem<DIM, P, Q, VS>;
  constexpr int ND = SM::ND, NV = SM::NV;
  constexpr int QQQ = Q * Q * Q;
  extern __shared__ double smem_all[];

  const int team = threadIdx.x / TS;
  const int t = threadIdx.x % TS;
  const int cell = p.start + blockIdx.x * CPB + team;
  const bool active = team < CPB && cell < p.end;
  double* sm = smem_all + (team < CPB ? team : 0) * SM::size;
  double* sU = sm + SM::U;
  double* sZ = sm + SM::Z;
  double* sY = sm + SM::Y;
  double* sX = sm + SM::X;
  const int64_t cs = p.mesh.nc_stride;

  // ---- gather u, vertex coordinates, vertex fields --------------------------
  if (active) {
    const int32_t* mrow = p.maplex + (int64_t)cell * ND;
    for (int idx = t; idx < ND; idx += TS) {
      const int64_t dof = __ldg(mrow + idx);
#pragma unroll
      for (int c = 0; c < VS; ++c) sU[c * ND + idx] = __ldg(p.u + VS * dof + c);
    }
    for (int v = t; v < NV; v += TS) {
      const int vid = __ldg(p.mesh.vmap + v * cs + cell);
      double xv[DIM];
      load_vertex<DIM>(p.mesh.coords, vid, xv);
#pragma unroll
      for (int a = 0; a < DIM; ++a) sX[v * DIM + a] = xv[a];
      if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
        sm[SM::MU + v] = __ldg(p.mu + vid);
        sm[SM::LAM + v] = __ldg(p.lam + vid);
      }
    }
  }
  __syncthreads();

  // ---- forward: reference gradients at the points of this thread's x-pencil
  // thread (b, c) = (t % Q, t / Q) in 3D, b = t in 2D
  double g[VS][DIM][Q];
#pragma unroll
  for (int comp = 0; comp < VS; ++comp) {
    const double* uc = sU + comp * ND;
    if constexpr (DIM == 3) {
      // z: pencil (i, j) over k -> Z0 = B u (and Z1 = D u, direct only)
      if (active && t < P * P) {
        const int i = t % P, j = t / P;
        double pen[P];
#pragma unroll
        for (int k = 0; k < P; ++k) pen[k] = uc[(k * P + j) * P + i];
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double z0 = 0.0, z1 = 0.0;
#pragma unroll
          for (int k = 0; k < P; ++k) {
            z0 = fma(p.B[c][k], pen[k], z0);
            if constexpr (!COLLOC) z1 = fma(p.D[c][k], pen[k], z1);
          }
          sZ[(c * P + j) * P + i] = z0;
          if constexpr (!COLLOC) sZ[Q * P * P + (c * P + j) * P + i] = z1;
        }
      }
      __syncthreads();
      // y: pencil (i, c) over j -> Y0 = B Z0 (Y1 = D Z0, Y2 = B Z1: direct)
      if (active && t < Q * P) {
        const int i = t % P, c = t / P;
        double p0[P], p1[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
          p0[j] = sZ[(c * P + j) * P + i];
          if constexpr (!COLLOC) p1[j] = sZ[Q * P * P + (c * P + j) * P + i];
        }
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          double y0 = 0.0, y1 = 0.0, y2 = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) {
            y0 = fma(p.B[b][j], p0[j], y0);
            if constexpr (!COLLOC) {
              y1 = fma(p.D[b][j], p0[j], y1);
              y2 = fma(p.B[b][j], p1[j], y2);
            }
          }
          sY[(c * Q + b) * P + i] = y0;
          if constexpr (!COLLOC) {
            sY[Q * Q * P + (c * Q + b) * P + i] = y1;
            sY[2 * Q * Q * P + (c * Q + b) * P + i] = y2;
          }
        }
      }
      __syncthreads();
      if constexpr (COLLOC) {
        // x: pencil (b, c) over i -> u at the Gauss points; d/dxi locally
        if (active) {
          const int b = t % Q, c = t / Q;
          double q0[P], uq[Q];
#pragma unroll
          for (int i = 0; i < P; ++i) q0[i] = sY[(c * Q + b) * P + i];
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < P; ++i) s = fma(p.B[a][i], q0[i], s);
            uq[a] = s;
            sZ[(c * Q + b) * Q + a] = s;
          }
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < Q; ++e) s = fma(p.Dc[a][e], uq[e], s);
            g[comp][0][a] = s;
          }
        }
        __syncthreads();
        // d/deta, d/dzeta with Dc across the pencils of the team
        if (active) {
          const int b = t % Q, c = t / Q;
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            double s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int e = 0; e < Q; ++e) {
              s1 = fma(p.Dc[b][e], sZ[(c * Q + e) * Q + a], s1);
              s2 = fma(p.Dc[c][e], sZ[(e * Q + b) * Q + a], s2);
            }
            g[comp][1][a] = s1;
            g[comp][2][a] = s2;
          }
        }
        __syncthreads();
      } else {
        // x: pencil (b, c) over i -> d/dxi = D Y0, d/deta = B Y1, d/dzeta = B Y2
        if (active) {
          const int b = t % Q, c = t / Q;
          double q0[P], q1[P], q2[P];
#pragma unroll
          for (int i = 0; i < P; ++i) {
            q0[i] = sY[(c * Q + b) * P + i];
            q1[i] = sY[Q * Q * P + (c * Q + b) * P + i];
            q2[i] = sY[2 * Q * Q * P + (c * Q + b) * P + i];
          }
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            double g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
            for (int i = 0; i < P; ++i) {
              g0 = fma(p.D[a][i], q0[i], g0);
              g1 = fma(p.B[a][i], q1[i], g1);
              g2 = fma(p.B[a][i], q2[i], g2);
            }
            g[comp][0][a] = g0;
            g[comp][1][a] = g1;
            g[comp][2][a] = g2;
          }
        }
        __syncthreads();
      }
    } else {
      // y: pencil i over j -> Y0 = B u, Y1 = D u
      if (active && t < P) {
        const int i = t;
        double pen[P];
#pragma unroll
        for (int j = 0; j < P; ++j) pen[j] = uc[j * P + i];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          double y0 = 0.0, y1 = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) {
            y0 = fma(p.B[b][j], pen[j], y0);
            y1 = fma(p.D[b][j], pen[j], y1);
          }
          sY[b * P + i] = y0;
          sY[Q * P + b * P + i] = y1;
        }
      }
      __syncthreads();
      if (active) {
        const int b = t;
        double q0[P], q1[P];
#pragma unroll
        for (int i = 0; i < P; ++i) {
          q0[i] = sY[b * P + i];
          q1[i] = sY[Q * P + b * P + i];
        }
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double g0 = 0.0, g1 = 0.0;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            g0 = fma(p.D[a][i], q0[i], g0);
            g1 = fma(p.B[a][i], q1[i], g1);
          }
          g[comp][0][a] = g0;
          g[comp][1][a] = g1;
        }
      }
      __syncthreads();
    }
  }

  // ---- pointwise flux at the Q points of the x-pencil ----------------------
  if (active) {
    const int b = t % Q, c = DIM == 3 ? t / Q : 0;
    const double eta = p.x[b], zeta = DIM == 3 ? p.x[c] : 0.0;
    const double wbc = DIM == 3 ? p.w[b] * p.w[c] : p.w[b];
    const double Ly[2] = {1.0 - eta, eta}, Lz[2] = {1.0 - zeta, zeta};
    auto Xv = [&](int vx, int vy, int vz, int d) { return sX[(vx + 2 * vy + 4 * vz) * DIM + d]; };
    // J(:, 0) constant along the pencil; J(:, e>0) = J0e + xi * dJe
    double c0[DIM], j1[DIM], d1[DIM], j2[DIM], d2[DIM];
    double m0 = 0.0, dm = 0.0, l0 = 0.0, dl = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      if constexpr (DIM == 3) {
        double s = 0.0;
#pragma unroll
        for (int vy = 0; vy < 2; ++vy)
#pragma unroll
          for (int vz = 0; vz < 2; ++vz) s += (Xv(1, vy, vz, d) - Xv(0, vy, vz, d)) * (Ly[vy] * Lz[vz]);
        c0[d] = s;
        double e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          e0 += (Xv(0, 1, o, d) - Xv(0, 0, o, d)) * Lz[o];
          e1 += (Xv(1, 1, o, d) - Xv(1, 0, o, d)) * Lz[o];
          f0 += (Xv(0, o, 1, d) - Xv(0, o, 0, d)) * Ly[o];
          f1 += (Xv(1, o, 1, d) - Xv(1, o, 0, d)) * Ly[o];
        }
        j1[d] = e0; d1[d] = e1 - e0;
        j2[d] = f0; d2[d] = f1 - f0;
      } else {
        c0[d] = (Xv(1, 0, 0, d) - Xv(0, 0, 0, d)) * Ly[0] + (Xv(1, 1, 0, d) - Xv(0, 1, 0, d)) * Ly[1];
        const double e0 = Xv(0, 1, 0, d) - Xv(0, 0, 0, d), e1 = Xv(1, 1, 0, d) - Xv(1, 0, 0, d);
        j1[d] = e0; d1[d] = e1 - e0;
      }
    }
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
      double mx[2] = {0.0, 0.0}, lx[2] = {0.0, 0.0};
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int vx = v & 1, vy = (v >> 1) & 1, vz = v >> 2;
        const double wgt = DIM == 3 ? Ly[vy] * Lz[vz] : Ly[vy];
        mx[vx] += wgt * sm[SM::MU + v];
        lx[vx] += wgt * sm[SM::LAM + v];
      }
      m0 = mx[0]; dm = mx[1] - mx[0];
      l0 = lx[0]; dl = lx[1] - lx[0];
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const double xi = p.x[a];
      double J[DIM][DIM], Ji[DIM][DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        J[d][0] = c0[d];
        J[d][1] = fma(xi, d1[d], j1[d]);
        if constexpr (DIM == 3) J[d][2] = fma(xi, d2[d], j2[d]);
      }
      const double det = det_inv<DIM>(J, Ji);
      const double tw = (p.w[a] * wbc) * fabs(det);
      double mu = p.p0, lam = p.p1;
      if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
        mu = fma(xi, dm, m0);
        lam = fma(xi, dl, l0);
      }
      double gq[VS][DIM], uq[VS], cv[VS], cg[VS][DIM];
#pragma unroll
      for (int comp = 0; comp < VS; ++comp) {
        uq[comp] = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) gq[comp][d] = g[comp][d][a];
      }
      pointwise<FORM, DIM, VS>(Ji, tw, uq, gq, mu, lam, cv, cg);
#pragma unroll
      for (int comp = 0; comp < VS; ++comp)
#pragma unroll
        for (int d = 0; d < DIM; ++d) g[comp][d][a] = cg[comp][d];
    }
  }

  // ---- transposed chain and scatter, one component at a time --------------
#pragma unroll
  for (int comp = 0; comp < VS; ++comp) {
    if constexpr (DIM == 3) {
      if constexpr (COLLOC) {
        // Dc^T in eta/zeta needs the team's pencils: stage F1, F2
        if (active) {
          const int b = t % Q, c = t / Q;
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            sZ[(c * Q + b) * Q + a] = g[comp][1][a];
            sZ[QQQ + (c * Q + b) * Q + a] = g[comp][2][a];
          }
        }
        __syncthreads();
        // V = Dc^T F0 (local) + Dc^T F1 (eta) + Dc^T F2 (zeta); x^T: A = B^T V
        if (active) {
          const int b = t % Q, c = t / Q;
          double V[Q];
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < Q; ++e) {
              s = fma(p.Dc[e][a], g[comp][0][e], s);
              s = fma(p.Dc[e][b], sZ[(c * Q + e) * Q + a], s);
              s = fma(p.Dc[e][c], sZ[QQQ + (e * Q + b) * Q + a], s);
            }
            V[a] = s;
          }
#pragma unroll
          for (int i = 0; i < P; ++i) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < Q; ++a) s = fma(p.B[a][i], V[a], s);
            sY[(c * Q + b) * P + i] = s;
          }
        }
        __syncthreads();
        // y^T: pencil (i, c) over b: W = B^T A
        if (active && t < Q * P) {
          const int i = t % P, c = t / P;
          double a0[Q];
#pragma unroll
          for (int b = 0; b < Q; ++b) a0[b] = sY[(c * Q + b) * P + i];
#pragma unroll
          for (int j = 0; j < P; ++j) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < Q; ++b) s = fma(p.B[b][j], a0[b], s);
            sZ[(c * P + j) * P + i] = s;
          }
        }
        __syncthreads();
        // z^T: pencil (i, j) over c: y_k = B^T W; scatter
        if (active && t < P * P) {
          const int i = t % P, j = t / P;
          double w1[Q];
#pragma unroll
          for (int c = 0; c < Q; ++c) w1[c] = sZ[(c * P + j) * P + i];
          const int32_t* mrow = p.maplex + (int64_t)cell * ND;
#pragma unroll
          for (int k = 0; k < P; ++k) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < Q; ++c) s = fma(p.B[c][k], w1[c], s);
            scatter_add(p.y, (int64_t)VS * __ldg(mrow + (k * P + j) * P + i) + comp, s);
          }
        }
        __syncthreads();
      } else {
        // x^T: thread (b, c): A0 = D^T F0, A1 = B^T F1, A2 = B^T F2 over i
        if (active) {
          const int b = t % Q, c = t / Q;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              a0 = fma(p.D[a][i], g[comp][0][a], a0);
              a1 = fma(p.B[a][i], g[comp][1][a], a1);
              a2 = fma(p.B[a][i], g[comp][2][a], a2);
            }
            sY[(c * Q + b) * P + i] = a0;
            sY[Q * Q * P + (c * Q + b) * P + i] = a1;
            sY[2 * Q * Q * P + (c * Q + b) * P + i] = a2;
          }
        }
        __syncthreads();
        // y^T: pencil (i, c) over b: W1 = B^T A0 + D^T A1, W2 = B^T A2
        if (active && t < Q * P) {
          const int i = t % P, c = t / P;
          double a0[Q], a1[Q], a2[Q];
#pragma unroll
          for (int b = 0; b < Q; ++b) {
            a0[b] = sY[(c * Q + b) * P + i];
            a1[b] = sY[Q * Q * P + (c * Q + b) * P + i];
            a2[b] = sY[2 * Q * Q * P + (c * Q + b) * P + i];
          }
#pragma unroll
          for (int j = 0; j < P; ++j) {
            double w1 = 0.0, w2 = 0.0;
#pragma unroll
            for (int b = 0; b < Q; ++b) {
              w1 = fma(p.B[b][j], a0[b], w1);
              w1 = fma(p.D[b][j], a1[b], w1);
              w2 = fma(p.B[b][j], a2[b], w2);
            }
            sZ[(c * P + j) * P + i] = w1;
            sZ[Q * P * P + (c * P + j) * P + i] = w2;
          }
        }
        __syncthreads();
        // z^T: pencil (i, j) over c: y_k = B^T W1 + D^T W2; scatter
        if (active && t < P * P) {
          const int i = t % P, j = t / P;
          double w1[Q], w2[Q];
#pragma unroll
          for (int c = 0; c < Q; ++c) {
            w1[c] = sZ[(c * P + j) * P + i];
            w2[c] = sZ[Q * P * P + (c * P + j) * P + i];
          }
          const int32_t* mrow = p.maplex + (int64_t)cell * ND;
#pragma unroll
          for (int k = 0; k < P; ++k) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < Q; ++c) {
              s = fma(p.B[c][k], w1[c], s);
              s = fma(p.D[c][k], w2[c], s);
            }
            scatter_add(p.y, (int64_t)VS * __ldg(mrow + (k * P + j) * P + i) + comp, s);
          }
        }
        __syncthreads();
      }
    } else {
      if (active) {
        const int b = t;
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            a0 = fma(p.D[a][i], g[comp][0][a], a0);
            a1 = fma(p.B[a][i], g[comp][1][a], a1);
          }
          sY[b * P + i] = a0;
          sY[Q * P + b * P + i] = a1;
        }
      }
      __syncthreads();
      if (active && t < P) {
        const int i = t;
        double a0[Q], a1[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          a0[b] = sY[b * P + i];
          a1[b] = sY[Q * P + b * P + i];
        }
        const int32_t* mrow = p.maplex + (int64_t)cell * ND;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < Q; ++b) {
            s = fma(p.B[b][j], a0[b], s);
            s = fma(p.D[b][j], a1[b], s);
          }
          scatter_add(p.y, (int64_t)VS * __ldg(mrow + j * P + i) + comp, s);
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace fe

// registry hook (plan.cu): TV(form, cell, dim, degree, P, Q)
#define FE_TENSOR_VARIANTS                                                                   \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 1, 2, 2),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 2, 3, 3),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 3, 4, 4),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 4, 5, 5),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 5, 6, 6),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 6, 7, 7),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 1, 2, 3),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 2, 3, 4),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 3, 4, 5),                             \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 1, 2, 3),                              \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 2, 3, 4),                              \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 3, 4, 5),                              \
  TV(FE_FORM_NEOHOOKEAN, FE_CELL_HEXAHEDRON, 3, 1, 2, 3),                                   \
  TV(FE_FORM_NEOHOOKEAN, FE_CELL_HEXAHEDRON, 3, 2, 3, 4),                                   \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 1, 2, 3),                           \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 2, 3, 4),                           \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 3, 4, 5),                           \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 4, 5, 6),                           \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 1, 2, 3),                                \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 2, 3, 4),                                \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 3, 4, 5),                                \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 4, 5, 6),                                \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 1, 2, 3),                                 \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 2, 3, 4),                                 \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 3, 4, 5),                                 \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 4, 5, 6),                                 \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 1, 2, 3),                          \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 2, 3, 4),                          \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 3, 4, 5),                          \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 4, 5, 6),
