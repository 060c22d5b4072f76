// Element-tensor kernels for affine simplices (C1 mass P2 triangles, C2
// Helmholtz P1..P3 tetrahedra).
//
// On an affine cell every term of mass/helmholtz/laplacian is a constant
// geometric coefficient times a reference matrix:
//   y_e = |det J| Mhat u_e + sum_{a<=b} K_ab (S_ab + S_ba [a!=b]) u_e,
//   K = |det J| J^-1 J^-T,  S_ab[i][j] = int dphi_i/dxi_a dphi_j/dxi_b,
// the "element-tensor" algorithm of SURVEY.md Appendix B (14 nd^2 + 13 nd +
// 80 flops on tets).  It is mathematically the reference's quadrature loop
// (kernels.py:136-252) with the quadrature sums hoisted out of the cell
// loop; results agree to round-off.
//
// One thread per cell, NM reference matrices passed BY VALUE in the kernel
// parameter block (constant bank 0): every DFMA of the unrolled S_m u_e
// products reads its matrix entry as a uniform constant operand, so the
// inner loop issues no shared-memory loads at all.
#pragma once
#include "common.cuh"

namespace fe {

template <int FORM, int DIM>
constexpr int et_nmats() {
  return ((FORM == FE_FORM_MASS || FORM == FE_FORM_HELMHOLTZ) ? 1 : 0) +
         (FORM != FE_FORM_MASS ? DIM * (DIM + 1) / 2 : 0);
}

template <int NM, int ND>
struct ETParams {
  MeshView mesh;
  const double* __restrict__ u;
  double* __restrict__ y;
  int32_t start, end;
  double S[NM][ND][ND];  // [mass?] then S_00, S_11, (S_22), S_01+S_10, ...
};

// Geometric coefficients of the NM matrices for one cell.
template <int FORM, int DIM, int NM>
FE_DEVICE void et_coeffs(const double (&X)[DIM + 1][DIM], double (&cm)[NM]) {
  double J[DIM][DIM], Ji[DIM][DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int b = 0; b < DIM; ++b) J[a][b] = X[b + 1][a] - X[0][a];
  double ad;
  if constexpr (FORM == FE_FORM_MASS) {
    double A[DIM][DIM];  // the mass form needs |det J| only: no inverse, no division
    ad = fabs(det_adj<DIM>(J, A));
    (void)Ji;
  } else {
    ad = fabs(det_inv<DIM>(J, Ji));
  }
  int m = 0;
  if constexpr (FORM == FE_FORM_MASS || FORM == FE_FORM_HELMHOLTZ) cm[m++] = ad;
  if constexpr (FORM != FE_FORM_MASS) {
    double K[DIM][DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = a; b < DIM; ++b) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < DIM; ++c) s += Ji[a][c] * Ji[b][c];
        K[a][b] = ad * s;
      }
#pragma unroll
    for (int a = 0; a < DIM; ++a) cm[m++] = K[a][a];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = a + 1; b < DIM; ++b) cm[m++] = K[a][b];
  }
}

// One thread's G consecutive cells are scattered together: contributions of
// the group to the same dof are summed in registers first and one RED is
// issued per distinct dof.  Consecutive cells of the structured meshes share
// vertices, edges and faces (the 6 Kuhn tets of a cube touch 8 vertices
// through 24 cell-vertex pairs), and at low degree the RED stream -- ~1.3
// LSU cycles per lane on the issuing SM -- rivals the arithmetic.  The
// duplicate search compares dof ids at run time (no mesh assumption); cells
// past `end` carry unique negative ids and are never scattered.
template <int G, int ND>
FE_DEVICE void group_scatter(double* __restrict__ y, const int (&dof)[G][ND], double (&yv)[G][ND]) {
  bool dup[G][ND];
#pragma unroll
  for (int r = 0; r < G; ++r)
#pragma unroll
    for (int i = 0; i < ND; ++i) dup[r][i] = false;
#pragma unroll
  for (int r = 1; r < G; ++r)
#pragma unroll
    for (int i = 0; i < ND; ++i)
#pragma unroll
      for (int r2 = 0; r2 < r; ++r2)
#pragma unroll
        for (int i2 = 0; i2 < ND; ++i2)
          if (!dup[r2][i2] && dof[r][i] == dof[r2][i2]) {  // at most one live match
            yv[r2][i2] += yv[r][i];
            dup[r][i] = true;
          }
  griddep_wait();
#pragma unroll
  for (int r = 0; r < G; ++r)
#pragma unroll
    for (int i = 0; i < ND; ++i)
      if (!dup[r][i] && dof[r][i] >= 0) scatter_add(y, dof[r][i], yv[r][i]);
}

// dof ids of a thread's G consecutive cells (lane l of a warp owns cells
// base + l*G + r); cells past `end` get unique negative ids.  (Staging the
// map columns through shared memory for coalescing measured slower.)
template <int G, int ND>
FE_DEVICE void group_dofs(const int32_t* __restrict__ map, int64_t cs, int base, int end, int lane,
                          int (&dof)[G][ND]) {
#pragma unroll
  for (int r = 0; r < G; ++r) {
    const int c = base + lane * G + r;
#pragma unroll
    for (int i = 0; i < ND; ++i) dof[r][i] = c < end ? __ldg(map + i * cs + c) : -1 - (r * ND + i);
  }
}

template <int FORM, int DIM, int ND>
FE_DEVICE void et_cell(const ETParams<et_nmats<FORM, DIM>(), ND>& p, int cell, const int (&dof)[ND],
                       double (&yv)[ND]) {
  constexpr int NM = et_nmats<FORM, DIM>();
  constexpr int NV = DIM + 1;
  const int64_t cs = p.mesh.nc_stride;
  double X[NV][DIM];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    int vid = (p.mesh.vmap == p.mesh.map) ? dof[v] : __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<DIM>(p.mesh.coords, vid, X[v]);
  }
  double w[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) w[i] = __ldg(p.u + dof[i]);
  double cm[NM];
  et_coeffs<FORM, DIM, NM>(X, cm);
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    double yi = 0.0;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < ND; ++j) t = fma(p.S[m][i][j], w[j], t);
      yi = fma(cm[m], t, yi);
    }
    yv[i] = yi;
  }
}

template <int FORM, int DIM, int ND, int G>
__global__ void __launch_bounds__(128)
affine_et_kernel(const __grid_constant__ ETParams<et_nmats<FORM, DIM>(), ND> p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = p.start + (blockIdx.x * blockDim.x + warp * 32) * G;
  if (base >= p.end) return;  // warp-uniform
  int dof[G][ND];
  group_dofs<G, ND>(p.mesh.map, p.mesh.nc_stride, base, p.end, lane, dof);
  double yv[G][ND];
#pragma unroll
  for (int r = 0; r < G; ++r) {
    if (dof[r][0] >= 0) {
      et_cell<FORM, DIM, ND>(p, base + lane * G + r, dof[r], yv[r]);
    } else {
#pragma unroll
      for (int i = 0; i < ND; ++i) yv[r][i] = 0.0;
    }
  }
  group_scatter<G, ND>(p.y, dof, yv);
}

// ---------------------------------------------------------------------------
// "Split" algorithm for Helmholtz / scalar Laplacian on affine simplices
// (the frozen-flop choice for C2-P1/P2): the stiffness
// term sum_ab K_ab int dphi_i/dxi_a dphi_j/dxi_b is integrated with the
// collapsed rule exact for degree 2k-2 (k^d points: 1 for P1, 8 for P2),
// i.e. interpolate the reference gradient at each point, multiply by K,
// integrate back (12 nd k^3 flops on tets), and the mass term uses the
// reference mass matrix (2 nd^2).  Exact on affine cells, so it equals the
// reference's quadrature result to round-off.
// ---------------------------------------------------------------------------

template <int NQS, int ND, int DIM>
struct SplitParams {
  MeshView mesh;
  const double* __restrict__ u;
  double* __restrict__ y;
  int32_t start, end;
  double qw[NQS];                 // weights of the low-order rule
  double dphi[NQS][ND][DIM];      // reference gradients at its points
  double M[ND][ND];               // reference mass matrix (unused for laplacian_scalar)
};

// reciprocal of |det J| per measurement (profiles/r01/sweep_split2.txt): the
// Newton rcp() for P1 (macro kernel 20.4 -> 19.2 us), the IEEE division for
// P2 (74.7 -> 66.5 us: rcp() lets ptxas hoist more and raise pressure)
constexpr bool split_fast_rcp(int nd) { return nd == 4; }

template <int FORM, int DIM, int ND, int NQS, bool MODAL = true>
FE_DEVICE void split_compute(const SplitParams<NQS, ND, DIM>& p, const double (&X)[DIM + 1][DIM],
                             const double (&w)[ND], double (&yv)[ND]) {
  // geometry: K = |det J| J^-1 J^-T = adj(J) adj(J)^T / |det J| (symmetric;
  // no explicit inverse)
  double J[DIM][DIM], A[DIM][DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int b = 0; b < DIM; ++b) J[a][b] = X[b + 1][a] - X[0][a];
  const double ad = fabs(det_adj<DIM>(J, A));
  const double rad = recip<split_fast_rcp(ND)>(ad);
  double K[DIM][DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int b = a; b < DIM; ++b) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < DIM; ++c) s = fma(A[a][c], A[b][c], s);
      K[a][b] = K[b][a] = rad * s;
    }
  // mass term
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    double s = 0.0;
    if constexpr (FORM == FE_FORM_HELMHOLTZ) {
#pragma unroll
      for (int j = 0; j < ND; ++j) s = fma(p.M[i][j], w[j], s);
      s *= ad;
    }
    yv[i] = s;
  }
  // stiffness term on the modes / low-order rule
#pragma unroll
  for (int q = 0; q < NQS; ++q) {
    double g[DIM];
#pragma unroll
    for (int b = 0; b < DIM; ++b) g[b] = 0.0;
#pragma unroll
    for (int i = 0; i < ND; ++i)
#pragma unroll
      for (int b = 0; b < DIM; ++b) g[b] = fma(p.dphi[q][i][b], w[i], g[b]);
    double f[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < DIM; ++b) s = fma(K[a][b], g[b], s);
      f[a] = MODAL ? s : p.qw[q] * s;  // stiffness modes carry unit weights
    }
#pragma unroll
    for (int j = 0; j < ND; ++j)
#pragma unroll
      for (int a = 0; a < DIM; ++a) yv[j] = fma(p.dphi[q][j][a], f[a], yv[j]);
  }
}

template <int FORM, int DIM, int ND, int NQS>
FE_DEVICE void split_cell(const SplitParams<NQS, ND, DIM>& p, int cell, const int (&dof)[ND],
                          double (&yv)[ND]) {
  constexpr int NV = DIM + 1;
  const int64_t cs = p.mesh.nc_stride;
  double X[NV][DIM];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    int vid = (p.mesh.vmap == p.mesh.map) ? dof[v] : __ldg(p.mesh.vmap + v * cs + cell);
    load_vertex<DIM>(p.mesh.coords, vid, X[v]);
  }
  double w[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) w[i] = __ldg(p.u + dof[i]);
  split_compute<FORM, DIM, ND, NQS>(p, X, w, yv);
}

template <int FORM, int DIM, int ND, int NQS, int G>
__global__ void __launch_bounds__(128)
affine_split_kernel(const __grid_constant__ SplitParams<NQS, ND, DIM> p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = p.start + (blockIdx.x * blockDim.x + warp * 32) * G;
  if (base >= p.end) return;  // warp-uniform
  int dof[G][ND];
  group_dofs<G, ND>(p.mesh.map, p.mesh.nc_stride, base, p.end, lane, dof);
  double yv[G][ND];
#pragma unroll
  for (int r = 0; r < G; ++r) {
    if (dof[r][0] >= 0) {
      split_cell<FORM, DIM, ND, NQS>(p, base + lane * G + r, dof[r], yv[r]);
    } else {
#pragma unroll
      for (int i = 0; i < ND; ++i) yv[r][i] = 0.0;
    }
  }
  group_scatter<G, ND>(p.y, dof, yv);
}

// ---------------------------------------------------------------------------
// Macro-cell variant (C2-P1).  At P1 the operator is bound by the global
// gathers and the FP64 RED stream (4 REDs per tet), not by arithmetic.  When
// the bound mesh consists of macro-cells -- MC consecutive cells whose dofs
// follow one fixed local pattern over NU distinct dofs, e.g. the 6 Kuhn
// tetrahedra of a cube over its 8 corners -- one thread takes a whole
// macro-cell: it gathers the NU dofs and coordinates once, runs the MC cells
// with compile-time local indices (all in registers, shared dofs summed in
// registers) and issues NU REDs instead of MC*ND (8 instead of 24 per cube).
// The pattern is verified for every macro-cell at bind time
// (fe_plan_bind_mesh); meshes that do not follow it, and the ragged ends of
// unaligned [start, end) ranges, run the per-cell kernel.
// ---------------------------------------------------------------------------

// the 6 Kuhn tetrahedra of a cube (mesh.kuhn_tets(): corner bit masks,
// positively oriented) as a local pattern over the cube's 8 corners
struct KuhnTetP1 {
  static constexpr int MC = 6, NU = 8, ND = 4;
  // rows {0,1,3,7} {0,1,7,5} {0,2,7,3} {0,2,6,7} {0,4,5,7} {0,4,7,6}, one nibble per entry
  __host__ __device__ static constexpr int at(int t, int i) {
    constexpr unsigned rows[6] = {0x7310u, 0x5710u, 0x3720u, 0x7620u, 0x7540u, 0x6740u};
    return (int)((rows[t] >> (4 * i)) & 15u);
  }
  __host__ __device__ static constexpr bool vertex(int) { return true; }
};

// P2 on the same 6 Kuhn tets: the 27 lattice points of the cube (8 corners,
// 12 edge + 6 face-diagonal + 1 body-diagonal midpoints); local node order
// vertices then edges (elements.lagrange_nodes), macro-dof ids in order of
// first appearance
struct KuhnTetP2 {
  static constexpr int MC = 6, NU = 27, ND = 10;
  __host__ __device__ static constexpr int at(int t, int i) {
    constexpr unsigned char tab[6][10] = {{0, 1, 2, 3, 4, 5, 6, 7, 8, 9},
                                          {0, 1, 3, 10, 4, 6, 11, 8, 12, 13},
                                          {0, 14, 3, 2, 15, 6, 5, 16, 17, 9},
                                          {0, 14, 18, 3, 15, 19, 6, 20, 16, 21},
                                          {0, 22, 10, 3, 23, 11, 6, 24, 25, 13},
                                          {0, 22, 3, 18, 23, 6, 19, 25, 26, 21}};
    return tab[t][i];
  }
  __host__ __device__ static constexpr bool vertex(int k) {
    return k == 0 || k == 1 || k == 2 || k == 3 || k == 10 || k == 14 || k == 18 || k == 22;
  }
};

// NCX consecutive Kuhn cubes along x (cells ordered x-fastest): they share
// their x-faces, so 4 + 4 NCX distinct corners; macro-dof id of corner bits
// (bx, by, bz) of cube c = (c + bx) + (NCX + 1) (by + 2 bz)
template <int NCX>
struct KuhnTetRowP1 {
  static constexpr int MC = 6 * NCX, NU = 4 * (NCX + 1), ND = 4;
  __host__ __device__ static constexpr int at(int t, int i) {
    const int c = t / 6, k = KuhnTetP1::at(t % 6, i);
    return (c + (k & 1)) + (NCX + 1) * (((k >> 1) & 1) + 2 * ((k >> 2) & 1));
  }
};

// P1 simplex with the element's tables as compile-time constants (what the
// reference's codegen bakes into the emitted source, codegen.py:409-424):
// reference gradients e_b - e_0, so grad_ref u = (w_b+1 - w_0); stiffness
// (1/(d! |det J|)) adj(J) adj(J)^T grad_ref u (adjugate form, no inverse);
// mass |det J| (1 + delta_ij) / ((d+1)(d+2) d!/2 ... ) = |det J|(1+delta_ij)/120
// in 3D, /24 in 2D -> |det J| c (w_i + sum w).  ~80 FP64 instructions per
// tet instead of ~110 for the table-driven split_compute; the plan only
// enables it after checking its tables against these constants.
template <int FORM, int DIM>
FE_DEVICE void p1_simplex_compute(const double (&X)[DIM + 1][DIM], const double (&w)[DIM + 1],
                                  double (&yv)[DIM + 1]) {
  constexpr double VREF = DIM == 3 ? 1.0 / 6.0 : 0.5;
  constexpr double CMASS = DIM == 3 ? 1.0 / 120.0 : 1.0 / 24.0;
  double J[DIM][DIM], A[DIM][DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int b = 0; b < DIM; ++b) J[a][b] = X[b + 1][a] - X[0][a];
  const double ad = fabs(det_adj<DIM>(J, A));
  const double rs = VREF * rcp(ad);
  double d[DIM], t[DIM], f[DIM];
#pragma unroll
  for (int b = 0; b < DIM; ++b) d[b] = w[b + 1] - w[0];
#pragma unroll
  for (int e = 0; e < DIM; ++e) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < DIM; ++r) s = fma(A[r][e], d[r], s);
    t[e] = rs * s;
  }
  double fs = 0.0;
#pragma unroll
  for (int r = 0; r < DIM; ++r) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < DIM; ++e) s = fma(A[r][e], t[e], s);
    f[r] = s;
    fs += s;
  }
  yv[0] = -fs;
#pragma unroll
  for (int b = 0; b < DIM; ++b) yv[b + 1] = f[b];
  if constexpr (FORM == FE_FORM_HELMHOLTZ) {
    double sw = w[0];
#pragma unroll
    for (int i = 1; i <= DIM; ++i) sw += w[i];
    const double cm = CMASS * ad;
#pragma unroll
    for (int i = 0; i <= DIM; ++i) yv[i] = fma(cm, w[i] + sw, yv[i]);
  }
}

#ifndef FE_MACRO_MINB
#define FE_MACRO_MINB 3   // 165 registers, no spill: C2-P1 21.5 -> 19.4 us (profiles/r02/ab_macro_minb.txt)
#endif
template <int FORM, int DIM, int ND, int NQS, class PAT, bool ANALYTIC = false>
__global__ void __launch_bounds__(128, FE_MACRO_MINB)
macro_split_kernel(const __grid_constant__ SplitParams<NQS, ND, DIM> p, const int32_t* __restrict__ corner,
                   int64_t mstride, int32_t m0, int32_t m1) {
  static_assert(PAT::ND == ND, "macro pattern of this element");
  constexpr int NU = PAT::NU, MC = PAT::MC;
  // persistent grid-stride loop; the macro-dof ids of the NEXT macro-cell are
  // loaded while this one computes, so only one dependent DRAM round trip
  // (ids -> coordinates/u) per macro-cell is exposed instead of two
  const int stride = gridDim.x * blockDim.x;
  int m = m0 + blockIdx.x * blockDim.x + threadIdx.x;
  int nxt[NU];
#pragma unroll
  for (int k = 0; k < NU; ++k) nxt[k] = m < m1 ? __ldg(corner + k * mstride + m) : 0;
  for (; m < m1; m += stride) {
  int dof[NU];
#pragma unroll
  for (int k = 0; k < NU; ++k) dof[k] = nxt[k];
#pragma unroll
  for (int k = 0; k < NU; ++k) nxt[k] = m + stride < m1 ? __ldg(corner + k * mstride + m + stride) : 0;
  double X[NU][DIM], w[NU], yl[NU];
#pragma unroll
  for (int k = 0; k < NU; ++k) {
    if (PAT::vertex(k)) load_vertex<DIM>(p.mesh.coords, dof[k], X[k]);  // vertex dof = vertex id
    w[k] = __ldg(p.u + dof[k]);
    yl[k] = 0.0;
  }
#pragma unroll
  for (int t = 0; t < MC; ++t) {
    double Xt[DIM + 1][DIM], wt[ND], yt[ND];
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      if (i <= DIM) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) Xt[i][a] = X[PAT::at(t, i)][a];
      }
      wt[i] = w[PAT::at(t, i)];
    }
    if constexpr (ANALYTIC) p1_simplex_compute<FORM, DIM>(Xt, wt, yt);
    else split_compute<FORM, DIM, ND, NQS>(p, Xt, wt, yt);
#pragma unroll
    for (int i = 0; i < ND; ++i) yl[PAT::at(t, i)] += yt[i];
  }
  griddep_wait();
#pragma unroll
  for (int k = 0; k < NU; ++k) scatter_add(p.y, dof[k], yl[k]);
  }
}

// Pipelined variant (round 2, P1 analytic case): macro_split_kernel above
// prefetches only the macro-dof ids; the coordinates and u values they point
// to are still a dependent DRAM round trip at the top of every macro-cell
// (ncu: long_scoreboard 4.1 of 7.4 stall cycles per instruction, FP64 pipe
// 40%).  Here that second hop is taken off the critical path too: while
// macro-cell n computes, cp.async (LDGSTS) copies the NU vertex coordinates
// and u values of macro-cell n+1 into a thread-private shared-memory column
// (double-buffered, layout [slot][thread]: conflict-free, no barriers) and the
// ids of macro-cell n+2 are loaded into registers.  The P1 case has no table
// constants, so the persistent loop costs no uniform registers.
template <int FORM, int DIM, int ND, class PAT>
__global__ void __launch_bounds__(128, FE_MACRO_MINB)
macro_pipe_kernel(const __grid_constant__ SplitParams<1, ND, DIM> p, const int32_t* __restrict__ corner,
                  int64_t mstride, int32_t m0, int32_t m1) {
  static_assert(PAT::ND == ND && ND == DIM + 1, "P1 macro pattern");
  constexpr int NU = PAT::NU, MC = PAT::MC, SL = NU * (DIM + 1);   // slots per thread and buffer
  extern __shared__ double smem_mp[];
  double* const sb = smem_mp + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  int m = m0 + blockIdx.x * blockDim.x + threadIdx.x;
  auto issue = [&](const int (&id)[NU], int buf) {
    double* d = sb + buf * SL * 128;
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      const double* x = p.mesh.coords + (int64_t)id[k] * CStride<DIM>::value;
#pragma unroll
      for (int a = 0; a < DIM; ++a) cp_async8(d + (k * (DIM + 1) + a) * 128, x + a);
      cp_async8(d + (k * (DIM + 1) + DIM) * 128, p.u + id[k]);
    }
  };
  int cur[NU], nxt[NU];
#pragma unroll
  for (int k = 0; k < NU; ++k) cur[k] = m < m1 ? __ldg(corner + k * mstride + m) : 0;
  if (m < m1) issue(cur, 0);
  cp_commit();
#pragma unroll
  for (int k = 0; k < NU; ++k) nxt[k] = m + stride < m1 ? __ldg(corner + k * mstride + m + stride) : 0;
  int buf = 0;
#pragma unroll 1
  for (; m < m1; m += stride) {
    if (m + stride < m1) issue(nxt, buf ^ 1);     // next macro-cell's data
    cp_commit();
    int nn[NU];                                   // ids two ahead
#pragma unroll
    for (int k = 0; k < NU; ++k) nn[k] = m + 2 * stride < m1 ? __ldg(corner + k * mstride + m + 2 * stride) : 0;
    cp_wait_group<1>();                           // this macro-cell's data has landed
    const double* d = sb + buf * SL * 128;
    double X[NU][DIM], w[NU], yl[NU];
#pragma unroll
    for (int k = 0; k < NU; ++k) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) X[k][a] = d[(k * (DIM + 1) + a) * 128];
      w[k] = d[(k * (DIM + 1) + DIM) * 128];
      yl[k] = 0.0;
    }
#pragma unroll
    for (int t = 0; t < MC; ++t) {
      double Xt[DIM + 1][DIM], wt[ND], yt[ND];
#pragma unroll
      for (int i = 0; i < ND; ++i) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) Xt[i][a] = X[PAT::at(t, i)][a];
        wt[i] = w[PAT::at(t, i)];
      }
      p1_simplex_compute<FORM, DIM>(Xt, wt, yt);
#pragma unroll
      for (int i = 0; i < ND; ++i) yl[PAT::at(t, i)] += yt[i];
    }
    griddep_wait();
#pragma unroll
    for (int k = 0; k < NU; ++k) scatter_add(p.y, cur[k], yl[k]);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      cur[k] = nxt[k];
      nxt[k] = nn[k];
    }
    buf ^= 1;
  }
  cp_wait_all();
}

// ---------------------------------------------------------------------------
// Patch-aggregated variant (low degree: C1, C2-P1/P2).  At these intensities
// the global FP64 RED stream (one per cell-dof pair: 6.3M for P1, 15.7M for
// P2) rivals the arithmetic.  The plan groups each CTA's 128 consecutive
// cells into a PATCH with a sorted list of its distinct dofs and a uint16
// patch-local index per cell-dof (built once at bind time): the CTA stages
// u of the patch in shared memory (one coalesced-ish read per distinct dof),
// accumulates the element vectors into a shared-memory patch vector, and
// flushes one global RED per distinct dof (3-6x fewer).
// ---------------------------------------------------------------------------

struct PatchView {
  const int32_t* __restrict__ off;    // [npatch + 1]
  const int32_t* __restrict__ dofs;   // [off[npatch]] sorted distinct dofs per patch
  const uint16_t* __restrict__ pidx;  // SoA [nd][nc_stride] patch-local index of each cell dof
};

constexpr int kPatchCells = 128;

template <int NM, int ND>
struct ETPatchParams {
  MeshView mesh;
  PatchView patch;
  const double* __restrict__ u;
  double* __restrict__ y;
  int32_t start, end;
  double S[NM][ND][ND];
};

template <int FORM, int DIM, int ND>
__global__ void __launch_bounds__(kPatchCells)
affine_et_patch_kernel(const __grid_constant__ ETPatchParams<et_nmats<FORM, DIM>(), ND> p) {
  constexpr int NM = et_nmats<FORM, DIM>();
  constexpr int NV = DIM + 1;
  extern __shared__ double sp[];
  const int blk = p.start / kPatchCells + blockIdx.x;
  const int off = __ldg(p.patch.off + blk);
  const int nu = __ldg(p.patch.off + blk + 1) - off;
  double* su = sp;
  double* sacc = sp + nu;
  for (int k = threadIdx.x; k < nu; k += kPatchCells) {
    su[k] = __ldg(p.u + __ldg(p.patch.dofs + off + k));
    sacc[k] = 0.0;
  }
  __syncthreads();
  const int cell = blk * kPatchCells + threadIdx.x;
  if (cell >= p.start && cell < p.end) {
    const int64_t cs = p.mesh.nc_stride;
    int li[ND];
#pragma unroll
    for (int i = 0; i < ND; ++i) li[i] = __ldg(p.patch.pidx + i * cs + cell);
    double X[NV][DIM];
#pragma unroll
    for (int v = 0; v < NV; ++v) load_vertex<DIM>(p.mesh.coords, __ldg(p.mesh.vmap + v * cs + cell), X[v]);
    double w[ND];
#pragma unroll
    for (int i = 0; i < ND; ++i) w[i] = su[li[i]];
    double cm[NM];
    et_coeffs<FORM, DIM, NM>(X, cm);
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      double yi = 0.0;
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < ND; ++j) t = fma(p.S[m][i][j], w[j], t);
        yi = fma(cm[m], t, yi);
      }
      atomicAdd(sacc + li[i], yi);
    }
  }
  __syncthreads();
  griddep_wait();
  for (int k = threadIdx.x; k < nu; k += kPatchCells) {
    const double v = sacc[k];
    if (v != 0.0) scatter_add(p.y, __ldg(p.patch.dofs + off + k), v);
  }
}

}  // namespace fe
