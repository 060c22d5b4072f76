// Whole-plane-transpose variant of the plane kernel (kern_plane.cuh): scalar
// Laplacian on hexahedra, used where its collocation flop count wins (C3-Q2).
//
// Same mathematics as tensor_kernel's collocation path (kern_tensor.cuh,
// SURVEY.md Appendix B), different GPU mapping.  tensor_kernel gives each
// thread one 1D pencil per stage, so every contraction stage passes its whole
// field through shared memory: P+Q shared accesses per P*Q FMAs, which with a
// 2-stage warp pipeline and 16 warps/SM left the FP64 pipe at ~53%
// (profiles/r01/prof5_C3-Q3.ncu-rep: short-scoreboard and wait stalls).
// Here a TEAM of Q threads owns a cell and each thread owns a whole 2D PLANE:
//
//   phase 1  thread j holds the dof plane u[i, j, k] (i = x, k = z):
//            z- and x-contractions stay in registers
//              Z  = B_z u          V0 = B_x Z          V1 = D_x Z
//   transpose V0, V1 through shared memory (plane j -> plane a)
//   phase 2  thread a holds V0[j, c], V1[j, c] for its x point a and walks the
//            y rows b: u, d/dxi, d/deta at (a, b, c) by y-contractions,
//            d/dzeta by the collocation derivative Dc along the row, the
//            Laplacian flux, and the transposed y-contractions accumulated
//            into W0, W1 (registers)
//   transpose W0, W1 back (plane a -> plane j)
//   phase 1' Zb = B_x^T W0 + D_x^T W1,  y = B_z^T Zb,  scatter (FP64 RED)
//
// Only the two transposes touch shared memory: 8 P Q^2 accesses per cell
// against ~14 Q^4 FMAs.  The flux uses the adjugate form
//   f = (w / |det J|) adj(J) adj(J)^T g_ref      (= |det J| w J^-1 J^-T g_ref)
// with the trilinear Jacobian built per point from per-thread / per-row
// factors (its columns are bilinear or linear in the point coordinates).
//
// Teams are packed into warps (32 / Q cells per warp) and every warp runs its
// own persistent loop over warp batches -- there are no CTA barriers.  The
// gather is asynchronous (cp.async, LDGSTS): the map row and vertex ids of
// batch n+2 and the u values and vertex coordinates of batch n+1 are copied
// into shared memory while batch n computes, so the indirect gather never
// occupies registers or stalls the arithmetic.
#pragma once
#include "common.cuh"
#include "kern_tensor.cuh"
#include "kern_plane.cuh"

namespace fe {

// ---- compile-time layout ------------------------------------------------------
// Lanes are team-major (lane = T * Q + t).  Worst count of 8-byte words on one
// bank (word mod 16) in a half-warp when lane (T, t < nt) touches T*cs + t*s.
constexpr int plane1_conflict(int cs, int s, int nt, int tpw, int q) {
  int worst = 0;
  for (int h = 0; h < 32; h += 16) {
    int cnt[16] = {0};
    for (int l = h; l < h + 16; ++l) {
      const int T = l / q, t = l % q;
      if (T >= tpw || t >= nt) continue;
      ++cnt[(T * cs + t * s) % 16];
    }
    for (int k = 0; k < 16; ++k) worst = cnt[k] > worst ? cnt[k] : worst;
  }
  return worst;
}
struct Plane1Pick { int su, sa, cs; };
// u plane  e = j*SU + k*P + i   (phase 1 reads: lanes vary j)
// transpose e = a*SA + j*Q + c  (phase 1 writes / reads: lanes vary j; phase 2: a)
// team stride CS.  Minimise the summed conflict degree, then the footprint.
template <int P, int Q>
constexpr Plane1Pick plane1_pick() {
  constexpr int tpw = 32 / Q;
  Plane1Pick best{P * P, P * Q, 0};
  int bc = 1 << 30, bsz = 1 << 30;
  for (int su = P * P; su < P * P + 8; ++su)
    for (int sa = P * Q; sa < P * Q + 8; ++sa) {
      const int nb = P * su > Q * sa ? P * su : Q * sa;
      for (int cs = nb; cs < nb + 16; ++cs) {
        const int c = plane1_conflict(cs, su, P, tpw, Q) + plane1_conflict(cs, Q, P, tpw, Q) +
                      plane1_conflict(cs, sa, Q, tpw, Q);
        if (c < bc || (c == bc && cs < bsz)) {
          bc = c;
          bsz = cs;
          best = Plane1Pick{su, sa, cs};
        }
      }
    }
  return best;
}

template <int P, int Q>
struct Plane1Layout {
  static constexpr int TPW = 32 / Q;  // cells (teams) per warp
  static constexpr int ND = P * P * P;
  static constexpr Plane1Pick pick = plane1_pick<P, Q>();
  static constexpr int SU = pick.su, SA = pick.sa, CS = pick.cs, SJ = Q;
  static constexpr int XS = 34;  // 8 vertices x (x, y, z, pad); cell stride 2 (mod 16) words
  static constexpr int MS = ((ND + 8) + 3) / 4 * 4;  // map row + 8 vertex ids (int32)
  // per warp: X[2][TPW][XS] doubles | U[2][TPW][CS] doubles | M[3][TPW][MS] int32
  static constexpr int X0 = 0;
  static constexpr int U0 = X0 + 2 * TPW * XS;
  static constexpr int M0 = U0 + 2 * TPW * CS;          // in doubles
  static constexpr int WARP_DOUBLES = M0 + (3 * TPW * MS + 3) / 4 * 2;  // keeps 16-byte alignment
};

template <int P, int Q, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
plane1_kernel(const __grid_constant__ TensorParams<Q, P> p) {
  using L = Plane1Layout<P, Q>;
  constexpr int TPW = L::TPW, ND = L::ND, CS = L::CS, SU = L::SU, SA = L::SA, SJ = L::SJ;
  constexpr int MS = L::MS, XS = L::XS;
  extern __shared__ double smem_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int T = lane / Q, t = lane % Q;
  const bool in_team = T < TPW;
  const int Tc = in_team ? T : 0;
  double* wbase = smem_all + warp * L::WARP_DOUBLES;
  double* sX0 = wbase + L::X0;
  double* sU0 = wbase + L::U0;
  int32_t* sM0 = reinterpret_cast<int32_t*>(wbase + L::M0);

  const int64_t ncs = p.mesh.nc_stride;
  const int nwb = (p.end - p.start + TPW - 1) / TPW;  // warp batches
  const int GW = gridDim.x * WARPS;
  auto cell_of = [&](int wb) { return p.start + wb * TPW + T; };
  auto valid = [&](int wb) { return in_team && wb < nwb && cell_of(wb) < p.end; };

  // map row (lexicographic) and vertex ids of warp batch wb -> map slot
  auto issue_map = [&](int wb, int slot) {
    if (!valid(wb)) return;
    const int c = cell_of(wb);
    int32_t* m = sM0 + (slot * TPW + T) * MS;
    const int32_t* src = p.maplex + (int64_t)c * ND;
    if constexpr (ND % 4 == 0) {
#pragma unroll
      for (int r = 0; r < (ND / 4 + Q - 1) / Q; ++r) {
        const int e = t + r * Q;
        if (e < ND / 4) cp_async16(m + 4 * e, src + 4 * e);
      }
    } else {
#pragma unroll
      for (int r = 0; r < (ND + Q - 1) / Q; ++r) {
        const int e = t + r * Q;
        if (e < ND) cp_async4(m + e, src + e);
      }
    }
#pragma unroll
    for (int r = 0; r < (8 + Q - 1) / Q; ++r) {
      const int v = t + r * Q;
      if (v < 8) cp_async4(m + ND + v, p.mesh.vmap + v * ncs + c);
    }
  };
  // u values and vertex coordinates of warp batch wb (its map in mslot) -> buffer buf
  auto issue_data = [&](int wb, int mslot, int buf) {
    if (!valid(wb)) return;
    const int32_t* m = sM0 + (mslot * TPW + T) * MS;
    double* su = sU0 + (buf * TPW + T) * CS;
#pragma unroll
    for (int r = 0; r < (ND + Q - 1) / Q; ++r) {
      const int e = t + r * Q;
      if (e < ND) {
        const int i = e % P, j = (e / P) % P, k = e / (P * P);
        cp_async8(su + j * SU + k * P + i, p.u + m[e]);
      }
    }
    double* sx = sX0 + (buf * TPW + T) * XS;
#pragma unroll
    for (int r = 0; r < (16 + Q - 1) / Q; ++r) {
      const int e = t + r * Q;
      if (e < 16) cp_async16(sx + 2 * e, p.mesh.coords + (int64_t)m[ND + (e >> 1)] * 4 + 2 * (e & 1));
    }
  };

  int wb = blockIdx.x * WARPS + warp;
  issue_map(wb, 0);
  cp_commit();
  cp_wait_all();
  __syncwarp();
  issue_data(wb, 0, 0);
  issue_map(wb + GW, 1);
  cp_commit();

  for (int it = 0; wb < nwb; wb += GW, ++it) {
    const int cur = it & 1;
    cp_wait_all();
    __syncwarp();
    // next batch's gather and the map of the one after, in flight while this batch computes
    issue_data(wb + GW, (it + 1) % 3, cur ^ 1);
    issue_map(wb + 2 * GW, (it + 2) % 3);
    cp_commit();

    const bool active = valid(wb);
    double* sU = sU0 + (cur * TPW + Tc) * CS;
    double* sX = sX0 + (cur * TPW + Tc) * XS;
    const int32_t* sM = sM0 + ((it % 3) * TPW + Tc) * MS;
#if FE_PLANE_MONO
    // trilinear map in monomial form, once per cell (kern_plane.cuh): thread
    // d < 3 converts coordinate d in place; consumed after the phase-1 barriers
    if (active && t < 3) {
      double xv[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) xv[v] = sX[v * 4 + t];
      sX[1 * 4 + t] = xv[1] - xv[0];
      sX[2 * 4 + t] = xv[2] - xv[0];
      sX[4 * 4 + t] = xv[4] - xv[0];
      sX[3 * 4 + t] = (xv[3] - xv[2]) - (xv[1] - xv[0]);
      sX[5 * 4 + t] = (xv[5] - xv[4]) - (xv[1] - xv[0]);
      sX[6 * 4 + t] = (xv[6] - xv[4]) - (xv[2] - xv[0]);
      sX[7 * 4 + t] = ((xv[7] - xv[6]) - (xv[5] - xv[4])) - ((xv[3] - xv[2]) - (xv[1] - xv[0]));
    }
#endif

    // ---- phase 1: thread j = t < P holds the dof plane u[i, j, k] --------
    double Z[P][Q];  // Z[i][c] = sum_k B[c][k] u[i][j][k]
    if (active && t < P) {
      double pu[P][P];
#pragma unroll
      for (int k = 0; k < P; ++k)
#pragma unroll
        for (int i = 0; i < P; ++i) pu[k][i] = sU[t * SU + k * P + i];
#pragma unroll
      for (int i = 0; i < P; ++i)
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < P; ++k) s = fma(p.B[c][k], pu[k][i], s);
          Z[i][c] = s;
        }
    }
    __syncwarp();
    // V0 = B_x Z  -> transpose
    if (active && t < P) {
#pragma unroll
      for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < P; ++i) s = fma(p.B[a][i], Z[i][c], s);
          sU[a * SA + t * SJ + c] = s;
        }
    }
    __syncwarp();
    double V0[P][Q], V1[P][Q];
    if (active) {
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int c = 0; c < Q; ++c) V0[j][c] = sU[t * SA + j * SJ + c];
    }
    __syncwarp();
    // V1 = D_x Z  -> transpose
    if (active && t < P) {
#pragma unroll
      for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < P; ++i) s = fma(p.D[a][i], Z[i][c], s);
          sU[a * SA + t * SJ + c] = s;
        }
    }
    __syncwarp();
    if (active) {
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int c = 0; c < Q; ++c) V1[j][c] = sU[t * SA + j * SJ + c];
    }

    // ---- phase 2: thread a = t, rows b, points c ---------------------------
    double W0[P][Q], W1[P][Q];
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int c = 0; c < Q; ++c) W0[j][c] = W1[j][c] = 0.0;
    if (active) {
      const double xi = p.x[t], wa = p.w[t];
      auto X = [&](int vx, int vy, int vz, int d) { return sX[(vx + 2 * vy + 4 * vz) * 4 + d]; };
      // d/deta column: linear in zeta; d/dzeta column: linear in eta (xi fixed)
      double e0[3], de[3], f0[3], df[3];
#if FE_PLANE_MONO
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        e0[d] = fma(xi, X(1, 1, 0, d), X(0, 1, 0, d));
        de[d] = fma(xi, X(1, 1, 1, d), X(0, 1, 1, d));
        f0[d] = fma(xi, X(1, 0, 1, d), X(0, 0, 1, d));
        df[d] = de[d];
      }
#else
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double s0 = (X(0, 1, 0, d) - X(0, 0, 0, d)) * (1.0 - xi) + (X(1, 1, 0, d) - X(1, 0, 0, d)) * xi;
        const double s1 = (X(0, 1, 1, d) - X(0, 0, 1, d)) * (1.0 - xi) + (X(1, 1, 1, d) - X(1, 0, 1, d)) * xi;
        const double g0 = (X(0, 0, 1, d) - X(0, 0, 0, d)) * (1.0 - xi) + (X(1, 0, 1, d) - X(1, 0, 0, d)) * xi;
        const double g1 = (X(0, 1, 1, d) - X(0, 1, 0, d)) * (1.0 - xi) + (X(1, 1, 1, d) - X(1, 1, 0, d)) * xi;
        e0[d] = s0; de[d] = s1 - s0;
        f0[d] = g0; df[d] = g1 - g0;
      }
#endif
#pragma unroll
      for (int b = 0; b < Q; ++b) {
        const double eta = p.x[b], wab = wa * p.w[b];
        // d/dxi column: bilinear in (eta, zeta) -> linear in zeta along the row
        double r0[3], dr[3], J2[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
#if FE_PLANE_MONO
          r0[d] = fma(eta, X(1, 1, 0, d), X(1, 0, 0, d));
          dr[d] = fma(eta, X(1, 1, 1, d), X(1, 0, 1, d));
#else
          const double q0 = (X(1, 0, 0, d) - X(0, 0, 0, d)) * (1.0 - eta) + (X(1, 1, 0, d) - X(0, 1, 0, d)) * eta;
          const double q1 = (X(1, 0, 1, d) - X(0, 0, 1, d)) * (1.0 - eta) + (X(1, 1, 1, d) - X(0, 1, 1, d)) * eta;
          r0[d] = q0; dr[d] = q1 - q0;
#endif
          J2[d] = fma(eta, df[d], f0[d]);
        }
        double uq[Q];
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) s = fma(p.B[b][j], V0[j][c], s);
          uq[c] = s;
        }
        double fz[Q];
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) {
            gx = fma(p.B[b][j], V1[j][c], gx);
            gy = fma(p.D[b][j], V0[j][c], gy);
          }
#pragma unroll
          for (int e = 0; e < Q; ++e) gz = fma(p.Dc[c][e], uq[e], gz);
          const double zeta = p.x[c];
          double J[3][3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            J[d][0] = fma(zeta, dr[d], r0[d]);
            J[d][1] = fma(zeta, de[d], e0[d]);
            J[d][2] = J2[d];
          }
          // adjugate (J^-1 = adj / det, rows = reference directions)
          const double a00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
          const double a01 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
          const double a02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
          const double a10 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
          const double a11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
          const double a12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
          const double a20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
          const double a21 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
          const double a22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
          const double det = J[0][0] * a00 + J[0][1] * a10 + J[0][2] * a20;
          const double s = (wab * p.w[c]) * recip<false>(fabs(det));
          // v = adj^T g (physical gradient * det), f = s adj v
          const double v0 = a00 * gx + a10 * gy + a20 * gz;
          const double v1 = a01 * gx + a11 * gy + a21 * gz;
          const double v2 = a02 * gx + a12 * gy + a22 * gz;
          const double fx = s * (a00 * v0 + a01 * v1 + a02 * v2);
          const double fy = s * (a10 * v0 + a11 * v1 + a12 * v2);
          fz[c] = s * (a20 * v0 + a21 * v1 + a22 * v2);
#pragma unroll
          for (int j = 0; j < P; ++j) {
            W1[j][c] = fma(p.B[b][j], fx, W1[j][c]);
            W0[j][c] = fma(p.D[b][j], fy, W0[j][c]);
          }
        }
        // Dc^T along the row for the zeta flux, then B_y^T
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double tz = 0.0;
#pragma unroll
          for (int e = 0; e < Q; ++e) tz = fma(p.Dc[e][c], fz[e], tz);
#pragma unroll
          for (int j = 0; j < P; ++j) W0[j][c] = fma(p.B[b][j], tz, W0[j][c]);
        }
      }
    }
    __syncwarp();  // V1 reads done: the buffer takes W0
    if (active) {
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int c = 0; c < Q; ++c) sU[t * SA + j * SJ + c] = W0[j][c];
    }
    __syncwarp();
    double Zb[P][Q];
    if (active && t < P) {
#pragma unroll
      for (int i = 0; i < P; ++i)
#pragma unroll
        for (int c = 0; c < Q; ++c) Zb[i][c] = 0.0;
#pragma unroll
      for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double w = sU[a * SA + t * SJ + c];
#pragma unroll
          for (int i = 0; i < P; ++i) Zb[i][c] = fma(p.B[a][i], w, Zb[i][c]);
        }
    }
    __syncwarp();
    if (active) {
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int c = 0; c < Q; ++c) sU[t * SA + j * SJ + c] = W1[j][c];
    }
    __syncwarp();
    if (active && t < P) {
#pragma unroll
      for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double w = sU[a * SA + t * SJ + c];
#pragma unroll
          for (int i = 0; i < P; ++i) Zb[i][c] = fma(p.D[a][i], w, Zb[i][c]);
        }
      // y[i, j, k] = sum_c B[c][k] Zb[i][c]; scatter
      griddep_wait();
#pragma unroll
      for (int k = 0; k < P; ++k)
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < Q; ++c) s = fma(p.B[c][k], Zb[i][c], s);
          scatter_add(p.y, sM[i + P * t + P * P * k], s);
        }
    }
    __syncwarp();  // buffers of this batch free for the batch after next
  }
  cp_wait_all();
}

}  // namespace fe

// registry hook (plan.cu): PL1V(degree, P, Q, WARPS, MINB)
#ifndef FE_PLANE1_MINB
#define FE_PLANE1_MINB 1
#endif
#define FE_PLANE1_VARIANTS PL1V(2, 3, 3, 4, FE_PLANE1_MINB),
