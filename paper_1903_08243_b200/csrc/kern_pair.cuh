// Component-pair kernel: 2D elasticity on quadrilaterals (C4-quad), sum
// factorised in registers.
//
// Two lanes per cell, lane c owning displacement component c.  Each lane
// holds its component's dof plane u_c[j][i] and output plane y_c[j][i] in
// registers and streams over the point rows b:
//   Y0 = B_y u_c, Y1 = D_y u_c                  (row b, P values each)
//   per point a:  du_c/dxi = D_x Y0, du_c/deta = B_x Y1
//                 gradient row (g_ref adj J)[c][:] (= det * physical); the
//                 partner lane's row arrives by one shuffle pair, giving the
//                 strain, the trace and the Lame stress row sigma[c][:]
//                 flux row (w/|det|) sigma[c][:] adj^T -> Z0 += D_x^T f0,
//                 Z1 += B_x^T f1
//   y_c += B_y^T Z0 + D_y^T Z1
// and finally scatters its P^2 values (FP64 RED).  No shared memory and no
// barriers: the team-of-threads kernel (kern_tensor.cuh) kept only 4-5 of
// every 6 lanes busy in its pencil stages and stalled on its shared-memory
// round trips (profiles/r01/prof9_C4-quad-Q3.ncu-rep: FP64 pipe 50%).
// The bilinear Jacobian's d/dxi column is constant along a point row, its
// d/deta column linear in xi; mu and lambda are bilinear vertex fields.
#pragma once
#include "common.cuh"
#include "kern_tensor.cuh"

namespace fe {

#ifndef FE_PAIR_RCP_MAXP
#define FE_PAIR_RCP_MAXP 5   // MUFU-seeded reciprocal up to this P: with the select-free kernel it wins at P = 5 too (0.5255 -> 0.4967 ms, profiles/r02/ab_pair_rcp.txt)
#endif
#ifndef FE_PAIR_T0ALT
#define FE_PAIR_T0ALT 1   // C4-quad-Q3 0.2733 -> 0.2652 ms (0.51 of its roof), Q4 0.4988 -> 0.4793 (profiles/r02/ab_pair_t0.txt)
#endif
#ifndef FE_PAIR_NOSEL
#define FE_PAIR_NOSEL 1
#endif
#ifndef FE_PAIR_SYM
#define FE_PAIR_SYM 1   // C4-quad-Q3 0.3205 -> 0.2960 ms, Q4 0.5808 -> 0.5746 (profiles/r02/ab_pair_sym.txt)
#endif
#ifndef FE_PAIR_RELOAD
#define FE_PAIR_RELOAD 1   // 1: re-read the dof ids for the scatter instead of holding them in registers
#endif
#ifndef FE_PAIR_BLOCK
#define FE_PAIR_BLOCK 32  // one warp per CTA: measured best (profiles/r01/sweep_warps.txt)
#endif
constexpr int kPairBlock = FE_PAIR_BLOCK;

template <int FORM, int P, int Q, int MINB>
__global__ void __launch_bounds__(kPairBlock, MINB)
pair_kernel(const __grid_constant__ TensorParams<Q, P> p) {
  static_assert(FORM == FE_FORM_ELASTICITY_LAME || FORM == FE_FORM_ELASTICITY, "2D elasticity forms");
  constexpr int NDS = P * P;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = gt & 1;
  const int cell = p.start + (gt >> 1);
  const unsigned live = __ballot_sync(0xffffffffu, cell < p.end);  // pairs live or die together
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;
#if FE_PAIR_SYM
  // mirror-symmetric table reads (verified at plan time): half the distinct
  // constants, so the uniform registers hold them across the unrolled rows
  auto TB = [&](int q, int i) { return 2 * q < Q ? p.B[q][i] : p.B[Q - 1 - q][P - 1 - i]; };
  auto TD = [&](int q, int i) { return 2 * q < Q ? p.D[q][i] : -p.D[Q - 1 - q][P - 1 - i]; };
  auto TX = [&](int q) { return 2 * q < Q ? p.x[q] : 1.0 - p.x[Q - 1 - q]; };
  auto TW = [&](int q) { return 2 * q < Q ? p.w[q] : p.w[Q - 1 - q]; };
#else
  auto TB = [&](int q, int i) { return p.B[q][i]; };
  auto TD = [&](int q, int i) { return p.D[q][i]; };
  auto TX = [&](int q) { return p.x[q]; };
  auto TW = [&](int q) { return p.w[q]; };
#endif

  const int32_t* mrow = p.maplex + (int64_t)cell * NDS;
  int dof[NDS];
#pragma unroll
  for (int e = 0; e < NDS; ++e) dof[e] = __ldg(mrow + e);
  double u[P][P];
#pragma unroll
  for (int j = 0; j < P; ++j)
#pragma unroll
    for (int i = 0; i < P; ++i) u[j][i] = __ldg(p.u + 2 * (int64_t)dof[j * P + i] + c);
  double X[4][2], mv[4], lv[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int vid = __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<2>(p.mesh.coords, vid, X[v]);
#if FE_PAIR_NOSEL
    // lane 1 works in the frame with the physical axes swapped (its own
    // component's axis first): both lanes then run the same formulas on
    // (own-axis, cross-axis) pairs and the per-point selects on c disappear.
    // The swap flips the sign of det J in lane 1, so the partner's values
    // arrive with the opposite sign convention and are SUBTRACTED below.
    {
      const double x0 = X[v][0], x1 = X[v][1];
      X[v][0] = c ? x1 : x0;
      X[v][1] = c ? x0 : x1;
    }
#endif
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
      mv[v] = __ldg(p.mu + vid);
      lv[v] = __ldg(p.lam + vid);
    } else {
      mv[v] = 0.5;
      lv[v] = 0.0;
    }
  }
  // d/deta column of J: linear in xi
  double j1[2], d1[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    j1[d] = X[2][d] - X[0][d];
    d1[d] = (X[3][d] - X[1][d]) - j1[d];
  }
  double y[P][P];
#pragma unroll
  for (int j = 0; j < P; ++j)
#pragma unroll
    for (int i = 0; i < P; ++i) y[j][i] = 0.0;

#pragma unroll
  for (int b = 0; b < Q; ++b) {
    const double eta = TX(b), le = 1.0 - eta, wb = TW(b);
    double Y0[P], Y1[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int j = 0; j < P; ++j) {
        s0 = fma(TB(b, j), u[j][i], s0);
        s1 = fma(TD(b, j), u[j][i], s1);
      }
      Y0[i] = s0;
      Y1[i] = s1;
    }
    // d/dxi column of J on this row; mu, lambda on the row: m0 + xi dm
    double J0[2];
#pragma unroll
    for (int d = 0; d < 2; ++d) J0[d] = (X[1][d] - X[0][d]) * le + (X[3][d] - X[2][d]) * eta;
    const double det0 = J0[0] * j1[1] - j1[0] * J0[1], ddet = J0[0] * d1[1] - d1[0] * J0[1];
    const double m0 = mv[0] * le + mv[2] * eta, dm = mv[1] * le + mv[3] * eta - m0;
    const double l0 = lv[0] * le + lv[2] * eta, dl = lv[1] * le + lv[3] * eta - l0;
    double Z0[P], Z1[P];
#pragma unroll
    for (int i = 0; i < P; ++i) Z0[i] = Z1[i] = 0.0;
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const double xi = TX(a);
      double gx = 0.0, gy = 0.0;  // du_c/dxi, du_c/deta
#pragma unroll
      for (int i = 0; i < P; ++i) {
        gx = fma(TD(a, i), Y0[i], gx);
        gy = fma(TB(a, i), Y1[i], gy);
      }
      // adjugate form: with adj = det J^-1 = [[J11, -J01], [-J10, J00]] the
      // flux tw sigma(G) J^-T equals (w / |det|) sigma(g adj) adj^T, so no
      // inverse is formed; det is linear in xi along the row
      const double J01 = fma(xi, d1[0], j1[0]), J11 = fma(xi, d1[1], j1[1]);
      const double det = fma(xi, ddet, det0);
      const double sc = (TW(a) * wb) * recip<(P <= FE_PAIR_RCP_MAXP)>(fabs(det));  // fast at Q3, IEEE at Q4 (measured)
      const double mu = sc * fma(xi, dm, m0), lam = sc * fma(xi, dl, l0);
      // own row of g adj, the partner's by shuffle
      const double g0 = gx * J11 - gy * J0[1], g1 = gy * J0[0] - gx * J01;
      const double o0 = __shfl_xor_sync(live, g0, 1), o1 = __shfl_xor_sync(live, g1, 1);
#if FE_PAIR_NOSEL
      // (own, cross) = (g0, g1): trace = own + partner's own, shear = cross + partner's cross
#if FE_PAIR_T0ALT
      // lam tr + 2 mu own = (lam + 2 mu) own - lam partner_own: one instruction fewer
      const double t0 = fma(fma(2.0, mu, lam), g0, -(lam * o0)), t1 = mu * (g1 - o1);
#else
      const double tr = g0 - o0;
      const double t0 = fma(mu, g0 + g0, lam * tr), t1 = mu * (g1 - o1);
#endif
#else
      const double tr = c ? (g1 + o0) : (g0 + o1);
      // (G + G^T)[c][:] and the Lame stress row (the scale folded into mu, lambda)
      const double s0 = g0 + (c ? o1 : g0), s1 = g1 + (c ? g1 : o0);
      const double t0 = fma(mu, s0, c ? 0.0 : lam * tr), t1 = fma(mu, s1, c ? lam * tr : 0.0);
#endif
      const double f0 = t0 * J11 - t1 * J01, f1 = t1 * J0[0] - t0 * J0[1];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        Z0[i] = fma(TD(a, i), f0, Z0[i]);
        Z1[i] = fma(TB(a, i), f1, Z1[i]);
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int i = 0; i < P; ++i) y[j][i] = fma(TB(b, j), Z0[i], fma(TD(b, j), Z1[i], y[j][i]));
  }
  griddep_wait();
#pragma unroll
  for (int j = 0; j < P; ++j)
#pragma unroll
    for (int i = 0; i < P; ++i)
      scatter_add(p.y, 2 * (int64_t)(FE_PAIR_RELOAD ? __ldg(mrow + j * P + i) : dof[j * P + i]) + c, y[j][i]);
}


// ---------------------------------------------------------------------------
// Even-odd variant (round 2): pair_kernel's arithmetic with EVERY 1D
// contraction in even-odd form, rows and points in mirror pairs (q, Q-1-q).
// Only the even / odd tables Be, Bo, De, Do (half the distinct constants) are
// read, so they stay in uniform registers; u is not held in registers but
// re-read (L1) column by column for each row pair.
// ---------------------------------------------------------------------------
template <int FORM, int P, int Q, int MINB>
__global__ void __launch_bounds__(kPairBlock, MINB)
pair_eo_kernel(const __grid_constant__ TensorParams<Q, P> p) {
  static_assert(FORM == FE_FORM_ELASTICITY_LAME || FORM == FE_FORM_ELASTICITY, "2D elasticity forms");
  constexpr int NDS = P * P, HP = P / 2, NE = (P + 1) / 2, HQ = Q / 2, NQ = (Q + 1) / 2;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = gt & 1;
  const int cell = p.start + (gt >> 1);
  const unsigned live = __ballot_sync(0xffffffffu, cell < p.end);
  if (cell >= p.end) return;
  const int64_t cs = p.mesh.nc_stride;
  const int32_t* mrow = p.maplex + (int64_t)cell * NDS;
  double X[4][2], mv[4], lv[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int vid = __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<2>(p.mesh.coords, vid, X[v]);
    {  // lane 1 works in the axis-swapped frame (see pair_kernel)
      const double x0 = X[v][0], x1 = X[v][1];
      X[v][0] = c ? x1 : x0;
      X[v][1] = c ? x0 : x1;
    }
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
      mv[v] = __ldg(p.mu + vid);
      lv[v] = __ldg(p.lam + vid);
    } else {
      mv[v] = 0.5;
      lv[v] = 0.0;
    }
  }
  double j1[2], d1[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    j1[d] = X[2][d] - X[0][d];
    d1[d] = (X[3][d] - X[1][d]) - j1[d];
  }
  // y in even / odd form along j: y[j] = YE[j] + YO[j], y[P-1-j] = YE[j] - YO[j]
  double YE[NE][P], YO[NE][P];
#pragma unroll
  for (int j = 0; j < NE; ++j)
#pragma unroll
    for (int i = 0; i < P; ++i) YE[j][i] = YO[j][i] = 0.0;

  // one point row: (Y0, Y1) -> (Z0, Z1), even-odd along the row
  auto row = [&](double eta, double wb, const double (&Y0)[P], const double (&Y1)[P], double (&Z0)[P],
                 double (&Z1)[P]) {
    const double le = 1.0 - eta;
    double J0[2];
#pragma unroll
    for (int d = 0; d < 2; ++d) J0[d] = (X[1][d] - X[0][d]) * le + (X[3][d] - X[2][d]) * eta;
    const double det0 = J0[0] * j1[1] - j1[0] * J0[1], ddet = J0[0] * d1[1] - d1[0] * J0[1];
    const double m0 = mv[0] * le + mv[2] * eta, dm = mv[1] * le + mv[3] * eta - m0;
    const double l0 = lv[0] * le + lv[2] * eta, dl = lv[1] * le + lv[3] * eta - l0;
    auto point = [&](double xi, double wa, double gx, double gy, double& f0, double& f1) {
      const double J01 = fma(xi, d1[0], j1[0]), J11 = fma(xi, d1[1], j1[1]);
      const double det = fma(xi, ddet, det0);
      const double sc = (wa * wb) * rcp(fabs(det));
      const double mu = sc * fma(xi, dm, m0), lam = sc * fma(xi, dl, l0);
      const double g0 = gx * J11 - gy * J0[1], g1 = gy * J0[0] - gx * J01;
      const double o0 = __shfl_xor_sync(live, g0, 1), o1 = __shfl_xor_sync(live, g1, 1);
      const double t0 = fma(fma(2.0, mu, lam), g0, -(lam * o0)), t1 = mu * (g1 - o1);
      f0 = t0 * J11 - t1 * J01;
      f1 = t1 * J0[0] - t0 * J0[1];
    };
    double Y0e[NE], Y0o[NE], Y1e[NE], Y1o[NE], ZE0[NE], ZO0[NE], ZE1[NE], ZO1[NE];
#pragma unroll
    for (int i = 0; i < HP; ++i) {
      Y0e[i] = Y0[i] + Y0[P - 1 - i];
      Y0o[i] = Y0[i] - Y0[P - 1 - i];
      Y1e[i] = Y1[i] + Y1[P - 1 - i];
      Y1o[i] = Y1[i] - Y1[P - 1 - i];
    }
    if constexpr (P % 2) {
      Y0e[HP] = Y0[HP];
      Y1e[HP] = Y1[HP];
      Y0o[HP] = Y1o[HP] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < NE; ++i) ZE0[i] = ZO0[i] = ZE1[i] = ZO1[i] = 0.0;
#pragma unroll
    for (int r = 0; r < HQ; ++r) {
      double ED = 0.0, OD = 0.0, EB = 0.0, OB = 0.0;
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        ED = fma(p.De[r][i], Y0e[i], ED);
        EB = fma(p.Be[r][i], Y1e[i], EB);
      }
#pragma unroll
      for (int i = 0; i < HP; ++i) {
        OD = fma(p.Do[r][i], Y0o[i], OD);
        OB = fma(p.Bo[r][i], Y1o[i], OB);
      }
      double f0a, f1a, f0b, f1b;
      point(p.x[r], p.w[r], OD + ED, EB + OB, f0a, f1a);
      point(1.0 - p.x[r], p.w[r], OD - ED, EB - OB, f0b, f1b);
      const double fm0 = f0a - f0b, fp0 = f0a + f0b, fp1 = f1a + f1b, fm1 = f1a - f1b;
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        ZE0[i] = fma(p.De[r][i], fm0, ZE0[i]);
        ZE1[i] = fma(p.Be[r][i], fp1, ZE1[i]);
      }
#pragma unroll
      for (int i = 0; i < HP; ++i) {
        ZO0[i] = fma(p.Do[r][i], fp0, ZO0[i]);
        ZO1[i] = fma(p.Bo[r][i], fm1, ZO1[i]);
      }
    }
    if constexpr (Q % 2) {
      double OD = 0.0, EB = 0.0;
#pragma unroll
      for (int i = 0; i < HP; ++i) OD = fma(p.Do[HQ][i], Y0o[i], OD);
#pragma unroll
      for (int i = 0; i < NE; ++i) EB = fma(p.Be[HQ][i], Y1e[i], EB);
      double f0, f1;
      point(p.x[HQ], p.w[HQ], OD, EB, f0, f1);
#pragma unroll
      for (int i = 0; i < HP; ++i) ZO0[i] = fma(p.Do[HQ][i], f0, ZO0[i]);
#pragma unroll
      for (int i = 0; i < NE; ++i) ZE1[i] = fma(p.Be[HQ][i], f1, ZE1[i]);
    }
#pragma unroll
    for (int i = 0; i < HP; ++i) {
      Z0[i] = ZE0[i] + ZO0[i];
      Z0[P - 1 - i] = ZE0[i] - ZO0[i];
      Z1[i] = ZE1[i] + ZO1[i];
      Z1[P - 1 - i] = ZE1[i] - ZO1[i];
    }
    if constexpr (P % 2) {
      Z0[HP] = ZE0[HP];
      Z1[HP] = ZE1[HP];
    }
  };

#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const bool pair = q < HQ;
    // forward along j for the row pair (q, Q-1-q): u re-read column by column
    double Y0a[P], Y1a[P], Y0b[P], Y1b[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      double uc[P];
#pragma unroll
      for (int j = 0; j < P; ++j) uc[j] = __ldg(p.u + 2 * (int64_t)__ldg(mrow + j * P + i) + c);
      double EB = 0.0, OB = 0.0, ED = 0.0, OD = 0.0;
#pragma unroll
      for (int j = 0; j < HP; ++j) {
        const double e = uc[j] + uc[P - 1 - j], o = uc[j] - uc[P - 1 - j];
        EB = fma(p.Be[q][j], e, EB);
        ED = fma(p.De[q][j], e, ED);
        OB = fma(p.Bo[q][j], o, OB);
        OD = fma(p.Do[q][j], o, OD);
      }
      if constexpr (P % 2) {
        EB = fma(p.Be[q][HP], uc[HP], EB);
        ED = fma(p.De[q][HP], uc[HP], ED);
      }
      Y0a[i] = EB + OB;
      Y1a[i] = OD + ED;
      Y0b[i] = EB - OB;
      Y1b[i] = OD - ED;
    }
    double Z0a[P], Z1a[P], Z0b[P], Z1b[P];
    row(p.x[q], p.w[q], Y0a, Y1a, Z0a, Z1a);
    if (pair) {
      row(1.0 - p.x[q], p.w[q], Y0b, Y1b, Z0b, Z1b);
      // y += B^T Z0 + D^T Z1 over the two rows, in even / odd form along j
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const double zp = Z0a[i] + Z0b[i], zm = Z0a[i] - Z0b[i];
        const double z1m = Z1a[i] - Z1b[i], z1p = Z1a[i] + Z1b[i];
#pragma unroll
        for (int j = 0; j < NE; ++j) YE[j][i] = fma(p.Be[q][j], zp, fma(p.De[q][j], z1m, YE[j][i]));
#pragma unroll
        for (int j = 0; j < HP; ++j) YO[j][i] = fma(p.Bo[q][j], zm, fma(p.Do[q][j], z1p, YO[j][i]));
      }
    } else {
      // middle row of an odd Q: B[mid] is even, D[mid] odd in j
#pragma unroll
      for (int i = 0; i < P; ++i) {
#pragma unroll
        for (int j = 0; j < NE; ++j) YE[j][i] = fma(p.Be[q][j], Z0a[i], YE[j][i]);
#pragma unroll
        for (int j = 0; j < HP; ++j) YO[j][i] = fma(p.Do[q][j], Z1a[i], YO[j][i]);
      }
    }
  }
  griddep_wait();
#pragma unroll
  for (int j = 0; j < HP; ++j)
#pragma unroll
    for (int i = 0; i < P; ++i) {
      scatter_add(p.y, 2 * (int64_t)__ldg(mrow + j * P + i) + c, YE[j][i] + YO[j][i]);
      scatter_add(p.y, 2 * (int64_t)__ldg(mrow + (P - 1 - j) * P + i) + c, YE[j][i] - YO[j][i]);
    }
  if constexpr (P % 2) {
#pragma unroll
    for (int i = 0; i < P; ++i) scatter_add(p.y, 2 * (int64_t)__ldg(mrow + HP * P + i) + c, YE[HP][i]);
  }
}

// ---------------------------------------------------------------------------
// Pipelined variant (round 2): the same arithmetic in PERSISTENT warps with
// the indirect gather P_e u taken off the critical path.  pair_kernel above
// issues map -> u loads and only then computes, with 8 warps per SM (255
// registers) to cover ~1.5 us of dependent DRAM latency per cell (ncu: FP64
// pipe 52% active).  Here every warp walks batches of 16 cells and keeps
// three stages in flight through cp.async (LDGSTS), all warp-local (no CTA
// barrier anywhere):
//   batch n+2: dof-id row + vertex ids          -> map ring (3 buffers)
//   batch n+1: u (own component), coordinates,
//              mu / lambda at the 4 vertices    -> data ring (2 buffers)
//   batch n  : compute from shared memory (u is re-read per point row: one
//              conflict-free LDS.64 per ~17 FP64 instructions) and scatter
//              with the ids still parked in the map ring.
// Neither the dof ids (P^2 registers) nor u (2 P^2 registers) live in
// registers any more.
// ---------------------------------------------------------------------------
template <int P>
struct PairPipeLayout {
  static constexpr int NDS = P * P;
  static constexpr int MR = NDS + 4;              // dof ids + vertex ids per cell
  static constexpr int MRS = MR | 1;              // odd stride: conflict-free id reads across cells
  static constexpr int MAP_INTS = 16 * MRS;       // one map buffer (16 cells)
  static constexpr int MAP_DOUBLES = (3 * MAP_INTS + 1) / 2;
  static constexpr int U = 0;                     // [NDS][32] own-component dof values
  static constexpr int X = U + NDS * 32;          // [4][16] double2 vertex coordinates
  static constexpr int MU = X + 4 * 16 * 2;       // [4][16]
  static constexpr int LAM = MU + 4 * 16;         // [4][16]
  static constexpr int DATA = LAM + 4 * 16;       // one data buffer
  static constexpr int WARP_DOUBLES = ((2 * DATA + MAP_DOUBLES) + 1) & ~1;
};

template <int FORM, int P, int Q, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
pair_pipe_kernel(const __grid_constant__ TensorParams<Q, P> p) {
  static_assert(FORM == FE_FORM_ELASTICITY_LAME || FORM == FE_FORM_ELASTICITY, "2D elasticity forms");
  using L = PairPipeLayout<P>;
  constexpr int NDS = L::NDS, MR = L::MR, MRS = L::MRS;
  constexpr bool LAME = FORM == FE_FORM_ELASTICITY_LAME;
  extern __shared__ double smem_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane & 1, slot = lane >> 1;
  double* const sw = smem_all + warp * L::WARP_DOUBLES;
  int32_t* const smap = reinterpret_cast<int32_t*>(sw + 2 * L::DATA);
  const int64_t cs = p.mesh.nc_stride;
  const int ncell = p.end - p.start;
  const int nbatch = (ncell + 15) / 16;
  const int wstride = gridDim.x * WARPS;
  // The 1D tables are mirror-symmetric (nodes and points symmetric about 1/2,
  // verified at plan time): B[q][i] = B[Q-1-q][P-1-i], D[q][i] = -D[Q-1-q][P-1-i].
  // Reading only the lower half keeps every table entry of the loop resident
  // in uniform registers (sm_100a feeds constant operands through ~80 URs; the
  // full tables do not fit and ptxas then parks them in vector registers and
  // moves them back with R2UR inside the loop).
  auto TB = [&](int q, int i) { return 2 * q < Q ? p.B[q][i] : p.B[Q - 1 - q][P - 1 - i]; };
  auto TD = [&](int q, int i) { return 2 * q < Q ? p.D[q][i] : -p.D[Q - 1 - q][P - 1 - i]; };
  auto TX = [&](int q) { return 2 * q < Q ? p.x[q] : 1.0 - p.x[Q - 1 - q]; };
  auto TW = [&](int q) { return 2 * q < Q ? p.w[q] : p.w[Q - 1 - q]; };

  auto issue_maps = [&](int batch, int mb) {
    const int cell = p.start + batch * 16 + slot;
    if (batch >= nbatch || cell >= p.end) return;
    int32_t* dst = smap + mb * L::MAP_INTS + slot * MRS;
    const int32_t* mrow = p.maplex + (int64_t)cell * NDS;
#pragma unroll
    for (int e = c; e < MR; e += 2) {
      if (e < NDS) cp_async4(dst + e, mrow + e);
      else cp_async4(dst + e, p.mesh.vmap + (e - NDS) * cs + cell);
    }
  };
  auto issue_data = [&](int batch, int mb, int db) {
    const int cell = p.start + batch * 16 + slot;
    if (batch >= nbatch || cell >= p.end) return;
    const int32_t* ids = smap + mb * L::MAP_INTS + slot * MRS;
    double* d = sw + db * L::DATA;
#pragma unroll
    for (int e = 0; e < NDS; ++e) cp_async8(d + L::U + e * 32 + lane, p.u + 2 * (int64_t)ids[e] + c);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int v = 2 * c + k;
      const int vid = ids[NDS + v];
      cp_async16(d + L::X + (v * 16 + slot) * 2, p.mesh.coords + 2 * (int64_t)vid);
      if constexpr (LAME) {
        cp_async8(d + L::MU + v * 16 + slot, p.mu + vid);
        cp_async8(d + L::LAM + v * 16 + slot, p.lam + vid);
      }
    }
  };

  int batch = blockIdx.x * WARPS + warp;
  issue_maps(batch, 0);
  cp_commit();
  issue_maps(batch + wstride, 1);
  cp_commit();
  cp_wait_group<1>();
  __syncwarp();
  issue_data(batch, 0, 0);
  cp_commit();
  int m0 = 0;  // map buffer of the current batch (ring of 3)
  int d0 = 0;  // data buffer of the current batch (ring of 2)
#pragma unroll 1
  for (; batch < nbatch; batch += wstride) {
    const int m1 = m0 == 2 ? 0 : m0 + 1, m2 = m1 == 2 ? 0 : m1 + 1;
    issue_maps(batch + 2 * wstride, m2);
    cp_commit();
    cp_wait_group<1>();        // data of this batch and ids of the next have landed
    __syncwarp();
    issue_data(batch + wstride, m1, d0 ^ 1);
    cp_commit();

    const int cell = p.start + batch * 16 + slot;
    const bool active = cell < p.end;
    const unsigned live = __ballot_sync(0xffffffffu, active);
    if (active) {
      const double* d = sw + d0 * L::DATA;
      const double* su = d + L::U + lane;
      double X[4][2], mv[4], lv[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const double2 xv = *reinterpret_cast<const double2*>(d + L::X + (v * 16 + slot) * 2);
        X[v][0] = xv.x;
        X[v][1] = xv.y;
        if constexpr (LAME) {
          mv[v] = d[L::MU + v * 16 + slot];
          lv[v] = d[L::LAM + v * 16 + slot];
        } else {
          mv[v] = 0.5;
          lv[v] = 0.0;
        }
      }
      double j1[2], d1[2];
#pragma unroll
      for (int dd = 0; dd < 2; ++dd) {
        j1[dd] = X[2][dd] - X[0][dd];
        d1[dd] = (X[3][dd] - X[1][dd]) - j1[dd];
      }
      double y[P][P];
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) y[j][i] = 0.0;

#pragma unroll
      for (int b = 0; b < Q; ++b) {
        const double eta = TX(b), le = 1.0 - eta, wb = TW(b);
        double Y0[P], Y1[P];
#pragma unroll
        for (int i = 0; i < P; ++i) Y0[i] = Y1[i] = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j)
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const double uv = su[(j * P + i) * 32];
            Y0[i] = fma(TB(b, j), uv, Y0[i]);
            Y1[i] = fma(TD(b, j), uv, Y1[i]);
          }
        double J0[2];
#pragma unroll
        for (int dd = 0; dd < 2; ++dd) J0[dd] = (X[1][dd] - X[0][dd]) * le + (X[3][dd] - X[2][dd]) * eta;
        const double det0 = J0[0] * j1[1] - j1[0] * J0[1], ddet = J0[0] * d1[1] - d1[0] * J0[1];
        const double mm0 = mv[0] * le + mv[2] * eta, dm = mv[1] * le + mv[3] * eta - mm0;
        const double l0 = lv[0] * le + lv[2] * eta, dl = lv[1] * le + lv[3] * eta - l0;
        double Z0[P], Z1[P];
#pragma unroll
        for (int i = 0; i < P; ++i) Z0[i] = Z1[i] = 0.0;
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          const double xi = TX(a);
          double gx = 0.0, gy = 0.0;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            gx = fma(TD(a, i), Y0[i], gx);
            gy = fma(TB(a, i), Y1[i], gy);
          }
          const double J01 = fma(xi, d1[0], j1[0]), J11 = fma(xi, d1[1], j1[1]);
          const double det = fma(xi, ddet, det0);
          const double sc = (TW(a) * wb) * recip<(P <= FE_PAIR_RCP_MAXP)>(fabs(det));
          const double mu = sc * fma(xi, dm, mm0), lam = sc * fma(xi, dl, l0);
          const double g0 = gx * J11 - gy * J0[1], g1 = gy * J0[0] - gx * J01;
          const double o0 = __shfl_xor_sync(live, g0, 1), o1 = __shfl_xor_sync(live, g1, 1);
          const double tr = c ? (g1 + o0) : (g0 + o1);
          const double s0 = g0 + (c ? o1 : g0), s1 = g1 + (c ? g1 : o0);
          const double t0 = fma(mu, s0, c ? 0.0 : lam * tr), t1 = fma(mu, s1, c ? lam * tr : 0.0);
          const double f0 = t0 * J11 - t1 * J01, f1 = t1 * J0[0] - t0 * J0[1];
#pragma unroll
          for (int i = 0; i < P; ++i) {
            Z0[i] = fma(TD(a, i), f0, Z0[i]);
            Z1[i] = fma(TB(a, i), f1, Z1[i]);
          }
        }
#pragma unroll
        for (int j = 0; j < P; ++j)
#pragma unroll
          for (int i = 0; i < P; ++i) y[j][i] = fma(TB(b, j), Z0[i], fma(TD(b, j), Z1[i], y[j][i]));
      }
      griddep_wait();
      const int32_t* ids = smap + m0 * L::MAP_INTS + slot * MRS;
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) scatter_add(p.y, 2 * (int64_t)ids[j * P + i] + c, y[j][i]);
    }
    __syncwarp();              // the rings are rewritten by the next iteration's copies
    m0 = m1;
    d0 ^= 1;
  }
  cp_wait_all();
}

}  // namespace fe

// registry hook (plan.cu): PRV(form, degree, P, Q, MINB); C4-quad-Q3/Q4 (Q1/Q2:
// the thread-per-cell quad_const_tensor kernel measured faster)
#ifndef FE_PAIR_MINB
#define FE_PAIR_MINB 1
#endif
#define FE_PAIR_VARIANTS                                                                     \
  PRV(FE_FORM_ELASTICITY_LAME, 3, 4, 5, FE_PAIR_MINB), PRV(FE_FORM_ELASTICITY_LAME, 4, 5, 6, FE_PAIR_MINB),
