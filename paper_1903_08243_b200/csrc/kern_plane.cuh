// Plane-per-thread, column-streamed sum-factorised kernel: scalar Laplacian
// on hexahedra (C3).
//
// Same mathematics as tensor_kernel's direct path (kern_tensor.cuh, SURVEY.md
// Appendix B), different GPU mapping.  tensor_kernel gives each thread one 1D
// pencil per stage, so every contraction stage passes its whole field through
// shared memory (P+Q shared accesses per P*Q FMAs); with 16 warps/SM that left
// the FP64 pipe at ~53% (profiles/r01/prof5_C3-Q3.ncu-rep).  Here a TEAM of Q
// threads owns a cell and the work is streamed over the z points c:
//
//   phase 1  thread j < P holds the dof plane u[i, j, k] (i = x, k = z) in
//            registers; for point column c it forms the z-contractions
//            z0 = B_z u, z1 = D_z u (P values each) and the x-contractions
//            V0 = B_x z0, V1 = D_x z0, V2 = B_x z1 (Q values each), written to
//            a small shared column buffer T[field][a][j]
//   phase 2  thread a < Q reads V*[a][j] and walks the y points b:
//            d/dxi = B_y V1, d/deta = D_y V0, d/dzeta = B_y V2, the Laplacian
//            flux at (a, b, c), and the transposed y-contractions back into
//            W*[a][j] (written in place over its own V* slots)
//   phase 1' thread j reads W*[a][j]: zb0 = B_x^T W0 + D_x^T W1,
//            zb1 = B_x^T W2, and accumulates y[i][k] += B_z[c][k] zb0[i] +
//            D_z[c][k] zb1[i] in registers; after the last column: scatter.
//
// Nothing bigger than a column (3 P Q values per cell) ever sits in shared
// memory and no thread holds more than a dof plane and its output plane, so
// the kernel runs at low register pressure with many warps per SM.  The flux
// uses the adjugate form
//   f = (w / |det J|) adj(J) adj(J)^T g_ref      (= w |det J| J^-1 J^-T g_ref)
// with the trilinear Jacobian built per point from per-column factors (its
// columns are linear in eta along a y line).
//
// Teams are packed into warps (32 / Q cells per warp) and every warp runs its
// own persistent loop over warp batches -- there are no CTA barriers.  The
// gather is asynchronous (cp.async, LDGSTS): the map row and vertex ids of
// batch n+2 and the u values and vertex coordinates of batch n+1 are copied
// into shared memory while batch n computes.
#pragma once
#include "common.cuh"
#include "kern_tensor.cuh"

#ifndef FE_PLANE_MONO
#define FE_PLANE_MONO 1   // monomial trilinear geometry (round 2)
#endif
#ifndef FE_PLANE_SYM
#define FE_PLANE_SYM 1
#endif
#ifndef FE_PLANE_RCP
#define FE_PLANE_RCP 1    // MUFU-seeded reciprocal instead of the IEEE division at P = 4 (C3-Q3 224.2 -> 222.2 us;
#endif                    // slower at P = 5: 529 -> 565 us, profiles/r02/ab_plane_rcp.txt)

namespace fe {

// ---- compile-time layout ------------------------------------------------------
// Lanes are team-major (lane = T * Q + t).  Worst count of 8-byte words on one
// bank (word mod 16) in a half-warp when lane (T, t < nt) touches T*cs + t*s.
constexpr int plane_conflict(int cs, int s, int nt, int tpw, int q) {
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
struct PlanePick { int s, cs; };
// u plane e = j*SU + k*P + i, team stride CU (phase-1 reads: lanes vary j)
template <int P, int Q>
constexpr PlanePick plane_pick_u() {
  PlanePick best{P * P, P * P * P};
  int bc = 1 << 30;
  for (int su = P * P; su < P * P + 8; ++su)
    for (int cs = P * su; cs < P * su + 16; ++cs) {
      const int c = plane_conflict(cs, su, P, 32 / Q, Q);
      if (c < bc) { bc = c; best = PlanePick{su, cs}; }
    }
  return best;
}
// column buffer e = f*Q*SA + a*SA + j, team stride CT (writes: lanes vary j
// with stride 1; reads: lanes vary a with stride SA)
template <int P, int Q>
constexpr PlanePick plane_pick_t() {
  PlanePick best{P, 3 * Q * P};
  int bc = 1 << 30;
  for (int sa = P; sa < P + 8; ++sa)
    for (int cs = 3 * Q * sa; cs < 3 * Q * sa + 16; ++cs) {
      const int c = plane_conflict(cs, 1, P, 32 / Q, Q) + plane_conflict(cs, sa, Q, 32 / Q, Q);
      if (c < bc) { bc = c; best = PlanePick{sa, cs}; }
    }
  return best;
}

template <int P, int Q>
struct PlaneLayout {
  static constexpr int TPW = 32 / Q;  // cells (teams) per warp
  static constexpr int ND = P * P * P;
  static constexpr PlanePick pu = plane_pick_u<P, Q>(), pt = plane_pick_t<P, Q>();
  static constexpr int SU = pu.s, CU = pu.cs, SA = pt.s, CT = pt.cs;
  // 8 vertices x (x, y, z, pad); the cell stride is 2 (mod 16) words so the
  // teams of a warp reading the same vertex of their own cells hit distinct banks
  static constexpr int XS = 34;
  static constexpr int MS = ((ND + 8) + 3) / 4 * 4;  // map row + 8 vertex ids (int32)
  // per warp (doubles): X[2][TPW][XS] | U[TPW][CU] | T[2][TPW][CT] | M[3][TPW][MS] int32
  static constexpr int X0 = 0;
  static constexpr int U0 = X0 + 2 * TPW * XS;
  static constexpr int T0 = U0 + ((TPW * CU + 1) & ~1);
  static constexpr int M0 = T0 + ((2 * TPW * CT + 1) & ~1);
  static constexpr int WARP_DOUBLES = M0 + (3 * TPW * MS + 3) / 4 * 2;  // keeps 16-byte alignment
};

// COLU: point-column loop unroll (per measurement: 2 at P = 4, 1 at P = 5)
template <int P, int Q, int WARPS, int MINB, int COLU>
__global__ void __launch_bounds__(WARPS * 32, MINB)
plane_kernel(const __grid_constant__ TensorParams<Q, P> p) {
  using L = PlaneLayout<P, Q>;
  constexpr int TPW = L::TPW, ND = L::ND, SU = L::SU, CU = L::CU, SA = L::SA, CT = L::CT;
  constexpr int MS = L::MS, XS = L::XS, SF = Q * SA;
  extern __shared__ double smem_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int T = lane / Q, t = lane % Q;
  const bool in_team = T < TPW;
  const int Tc = in_team ? T : 0;
  double* wbase = smem_all + warp * L::WARP_DOUBLES;
  double* sX0 = wbase + L::X0;
  double* sU = wbase + L::U0 + Tc * CU;
  double* sT0 = wbase + L::T0 + Tc * CT;
  int32_t* sM0 = reinterpret_cast<int32_t*>(wbase + L::M0);

  const int64_t ncs = p.mesh.nc_stride;
  // mirror-symmetric table reads (verified at plan time) when the column loop
  // is fully unrolled (every index compile-time): half the distinct constants,
  // so all of them stay in uniform registers across the persistent loop
  constexpr bool SYM = FE_PLANE_SYM && COLU == Q;
  auto TB = [&](int q, int i) { return (!SYM || 2 * q < Q) ? p.B[q][i] : p.B[Q - 1 - q][P - 1 - i]; };
  auto TD = [&](int q, int i) { return (!SYM || 2 * q < Q) ? p.D[q][i] : -p.D[Q - 1 - q][P - 1 - i]; };
  auto TXc = [&](int q) { return (!SYM || 2 * q < Q) ? p.x[q] : 1.0 - p.x[Q - 1 - q]; };
  auto TWc = [&](int q) { return (!SYM || 2 * q < Q) ? p.w[q] : p.w[Q - 1 - q]; };
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
  // u values and vertex coordinates of warp batch wb (its map in mslot)
  auto issue_data = [&](int wb, int mslot, int xbuf) {
    if (!valid(wb)) return;
    const int32_t* m = sM0 + (mslot * TPW + T) * MS;
#pragma unroll
    for (int r = 0; r < (ND + Q - 1) / Q; ++r) {
      const int e = t + r * Q;
      if (e < ND) {
        const int i = e % P, j = (e / P) % P, k = e / (P * P);
        cp_async8(sU + j * SU + k * P + i, p.u + m[e]);
      }
    }
    double* sx = sX0 + (xbuf * TPW + T) * XS;
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
    const bool active = valid(wb);
    const bool jt = active && t < P;  // phase-1 role (dof plane j = t)

    // dof plane u[i, j = t, k] -> registers; then the buffer takes the next batch
    double pu[P][P];  // [k][i]
    if (jt) {
#pragma unroll
      for (int k = 0; k < P; ++k)
#pragma unroll
        for (int i = 0; i < P; ++i) pu[k][i] = sU[t * SU + k * P + i];
    }
    __syncwarp();
    issue_data(wb + GW, (it + 1) % 3, cur ^ 1);
    issue_map(wb + 2 * GW, (it + 2) % 3);
    cp_commit();

    double* sX = sX0 + (cur * TPW + Tc) * XS;
#if FE_PLANE_MONO
    // trilinear map in monomial form, once per cell: x = sum C_abc xi^a eta^b zeta^c.
    // Thread d < 3 converts coordinate d in place (slot v = a + 2b + 4c), so a
    // point line needs 6 FMAs per coordinate for its Jacobian factors instead
    // of 22 operations on vertex differences.
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
    __syncwarp();
#endif
    auto X = [&](int vx, int vy, int vz, int d) { return sX[(vx + 2 * vy + 4 * vz) * 4 + d]; };
    double yp[P][P];  // output plane y[i, j = t, k], [k][i]
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
      for (int i = 0; i < P; ++i) yp[k][i] = 0.0;

#pragma unroll COLU
    for (int c = 0; c < Q; ++c) {
      double* sT = sT0 + (c & 1) * TPW * CT;
      // ---- phase 1: column c of V0, V1, V2 from the dof plane ---------------
      if (jt) {
        double z0[P], z1[P];
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int k = 0; k < P; ++k) {
            s0 = fma(TB(c, k), pu[k][i], s0);
            s1 = fma(TD(c, k), pu[k][i], s1);
          }
          z0[i] = s0;
          z1[i] = s1;
        }
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          double v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            v0 = fma(TB(a, i), z0[i], v0);
            v1 = fma(TD(a, i), z0[i], v1);
            v2 = fma(TB(a, i), z1[i], v2);
          }
          sT[a * SA + t] = v0;
          sT[SF + a * SA + t] = v1;
          sT[2 * SF + a * SA + t] = v2;
        }
      }
      __syncwarp();
      // ---- phase 2: thread a = t, points (a, b, c) ----------------------------
      if (active) {
        double V0[P], V1[P], V2[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
          V0[j] = sT[t * SA + j];
          V1[j] = sT[SF + t * SA + j];
          V2[j] = sT[2 * SF + t * SA + j];
        }
        const double xi = p.x[t], zeta = TXc(c), wac = p.w[t] * TWc(c);
        const double lx0 = 1.0 - xi, lz0 = 1.0 - zeta;
        // d/dxi column: linear in eta; d/deta: constant on the line; d/dzeta: linear in eta
        double g0[3], dg[3], J1[3], h0[3], dh[3];
#if FE_PLANE_MONO
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          g0[d] = fma(zeta, X(1, 0, 1, d), X(1, 0, 0, d));
          dg[d] = fma(zeta, X(1, 1, 1, d), X(1, 1, 0, d));
          J1[d] = fma(xi, dg[d], fma(zeta, X(0, 1, 1, d), X(0, 1, 0, d)));
          h0[d] = fma(xi, X(1, 0, 1, d), X(0, 0, 1, d));
          dh[d] = fma(xi, X(1, 1, 1, d), X(0, 1, 1, d));
        }
        (void)lx0;
        (void)lz0;
#else
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double q0 = (X(1, 0, 0, d) - X(0, 0, 0, d)) * lz0 + (X(1, 0, 1, d) - X(0, 0, 1, d)) * zeta;
          const double q1 = (X(1, 1, 0, d) - X(0, 1, 0, d)) * lz0 + (X(1, 1, 1, d) - X(0, 1, 1, d)) * zeta;
          g0[d] = q0; dg[d] = q1 - q0;
          const double e0 = (X(0, 1, 0, d) - X(0, 0, 0, d)) * lx0 + (X(1, 1, 0, d) - X(1, 0, 0, d)) * xi;
          const double e1 = (X(0, 1, 1, d) - X(0, 0, 1, d)) * lx0 + (X(1, 1, 1, d) - X(1, 0, 1, d)) * xi;
          J1[d] = e0 * lz0 + e1 * zeta;
          const double f0 = (X(0, 0, 1, d) - X(0, 0, 0, d)) * lx0 + (X(1, 0, 1, d) - X(1, 0, 0, d)) * xi;
          const double f1 = (X(0, 1, 1, d) - X(0, 1, 0, d)) * lx0 + (X(1, 1, 1, d) - X(1, 1, 0, d)) * xi;
          h0[d] = f0; dh[d] = f1 - f0;
        }
#endif
        double W0[P], W1[P], W2[P];
#pragma unroll
        for (int j = 0; j < P; ++j) W0[j] = W1[j] = W2[j] = 0.0;
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          const double eta = TXc(b);
          double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) {
            gx = fma(TB(b, j), V1[j], gx);
            gy = fma(TD(b, j), V0[j], gy);
            gz = fma(TB(b, j), V2[j], gz);
          }
          double J[3][3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            J[d][0] = fma(eta, dg[d], g0[d]);
            J[d][1] = J1[d];
            J[d][2] = fma(eta, dh[d], h0[d]);
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
          const double s = (wac * TWc(b)) * recip<(FE_PLANE_RCP == 2) || ((FE_PLANE_RCP == 1) && P == 4)>(fabs(det));
          // v = adj^T g (= det * physical gradient), f = s adj v
          const double v0 = a00 * gx + a10 * gy + a20 * gz;
          const double v1 = a01 * gx + a11 * gy + a21 * gz;
          const double v2 = a02 * gx + a12 * gy + a22 * gz;
          const double fx = s * (a00 * v0 + a01 * v1 + a02 * v2);
          const double fy = s * (a10 * v0 + a11 * v1 + a12 * v2);
          const double fz = s * (a20 * v0 + a21 * v1 + a22 * v2);
#pragma unroll
          for (int j = 0; j < P; ++j) {
            W1[j] = fma(TB(b, j), fx, W1[j]);
            W0[j] = fma(TD(b, j), fy, W0[j]);
            W2[j] = fma(TB(b, j), fz, W2[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < P; ++j) {  // in place over this thread's V slots
          sT[t * SA + j] = W0[j];
          sT[SF + t * SA + j] = W1[j];
          sT[2 * SF + t * SA + j] = W2[j];
        }
      }
      __syncwarp();
      // ---- phase 1': x^T then z^T into the output plane -----------------------
      if (jt) {
        double zb0[P], zb1[P];
#pragma unroll
        for (int i = 0; i < P; ++i) zb0[i] = zb1[i] = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          const double w0 = sT[a * SA + t], w1 = sT[SF + a * SA + t], w2 = sT[2 * SF + a * SA + t];
#pragma unroll
          for (int i = 0; i < P; ++i) {
            zb0[i] = fma(TB(a, i), w0, zb0[i]);
            zb0[i] = fma(TD(a, i), w1, zb0[i]);
            zb1[i] = fma(TB(a, i), w2, zb1[i]);
          }
        }
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
          for (int i = 0; i < P; ++i) yp[k][i] = fma(TB(c, k), zb0[i], fma(TD(c, k), zb1[i], yp[k][i]));
      }
    }
    if (jt) {
      const int32_t* sM = sM0 + ((it % 3) * TPW + T) * MS;
      griddep_wait();
#pragma unroll
      for (int k = 0; k < P; ++k)
#pragma unroll
        for (int i = 0; i < P; ++i) scatter_add(p.y, sM[i + P * t + P * P * k], yp[k][i]);
    }
  }
  cp_wait_all();
}

}  // namespace fe

// registry hook (plan.cu): PLV(degree, P, Q, WARPS, MINB, CU)
// C3-Q3 (P = Q = 4) and C3-Q4 (P = Q = 5); Q2 uses the whole-plane-transpose
// variant (kern_plane1.cuh), Q1 the thread-per-cell quad_const_tensor kernel,
// Q5/Q6 the pencil team kernel (profiles/r01/sweep_plane.txt)
#ifndef FE_PLANE_MINB
#define FE_PLANE_MINB 1
#endif
#ifndef FE_PLANE_WARPS
#define FE_PLANE_WARPS 8   // C3-Q3 222 -> 212 us, C3-Q4 529 -> 521 us vs 4 warps (profiles/r02/ab_plane_warps.txt)
#endif
#ifndef FE_PLANE_CU4
#define FE_PLANE_CU4 2
#endif
#ifndef FE_PLANE_CU5
#define FE_PLANE_CU5 1
#endif
#define FE_PLANE_VARIANTS PLV(3, 4, 4, FE_PLANE_WARPS, FE_PLANE_MINB, FE_PLANE_CU4), PLV(4, 5, 5, FE_PLANE_WARPS, FE_PLANE_MINB, FE_PLANE_CU5),
