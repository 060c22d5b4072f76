// FP64 tensor-core (DMMA) element-tensor kernel for high-degree affine
// simplices (C2 Helmholtz P3/P4 tetrahedra).
//
// For a group of 8 cells the element-tensor action is one small GEMM
//   Y[i][e] = sum_m sum_j S_m[i][j] * (c_m(e) u_j(e)),
//   A = [S_1 | ... | S_NM]   (ND x NM*ND, the same for every cell)
//   B = [c_1 u; ...; c_NM u] (NM*ND x 8 cells, built on the fly),
// which maps onto mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; sm_100a has no FP64
// tcgen05 kind).  A lives in shared memory in fragment order (one
// conflict-free LDS.64 per fragment); B fragments never touch shared memory:
// lane l holds u_j of cell l/4 for j = l%4 (mod 4) in registers, so a B
// fragment is one DMUL c_m * u.  Each warp owns NT n-tiles (8 NT cells) per
// iteration; CTAs are persistent and load A once.
//
// The M (output dof) dimension is padded to a multiple of 8 and each S_m's
// K extent to a multiple of 4: 85% (P4) / 83% (P3) of the DMMA flops are
// useful.  The scatter P_e^T is FP64 RED from the accumulator registers.
#pragma once
#include "common.cuh"
#include "kern_affine.cuh"

namespace fe {

struct DmmaParams {
  MeshView mesh;
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ afrag;  // [NM][KT][MT][32] fragment-ordered A
  int32_t start, end;
};

FE_DEVICE void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int ND> struct DmmaShape {
  static constexpr int KT = (ND + 3) / 4;  // k-steps per reference matrix
  static constexpr int MT = (ND + 7) / 8;  // m-tiles of output dofs
};

template <int FORM, int DIM, int ND, int NT, int MINB>
__global__ void __launch_bounds__(256, MINB) dmma_et_kernel(DmmaParams p) {
  constexpr int NM = et_nmats<FORM, DIM>();
  constexpr int KT = DmmaShape<ND>::KT, MT = DmmaShape<ND>::MT, NV = DIM + 1;
  constexpr int ASIZE = NM * KT * MT * 32;
  extern __shared__ double sA[];
  {
    const double2* src = reinterpret_cast<const double2*>(p.afrag);
    double2* dst = reinterpret_cast<double2*>(sA);
    for (int i = threadIdx.x; i < ASIZE / 2; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, c4 = lane & 3;
  const int wpb = blockDim.x >> 5;
  const int64_t cs = p.mesh.nc_stride;
  const int ncell = p.end - p.start;
  const int ngroups = (ncell + 8 * NT - 1) / (8 * NT);
  const int gstride = gridDim.x * wpb;

  // The map entries of the NEXT group (gather positions, vertex ids and the
  // scatter rows) are loaded one group ahead, so at the top of a group the
  // u / coordinate loads issue at once: one memory round trip per group on
  // the critical path instead of two (map -> data).
  int pf_dof[NT][KT], pf_vid[NT][NV], pf_row[NT][2][MT];
  auto load_maps = [&](int g) {
    const int base = p.start + g * 8 * NT;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int cell = base + nt * 8 + r;
      const bool valid = g < ngroups && cell < p.end;
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        const int j = 4 * t + c4;
        pf_dof[nt][t] = (valid && j < ND) ? __ldg(p.mesh.map + j * cs + cell) : -1;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) pf_vid[nt][v] = valid ? __ldg(p.mesh.vmap + v * cs + cell) : -1;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int sc = base + nt * 8 + 2 * c4 + e;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int row = 8 * mt + r;
          pf_row[nt][e][mt] =
              (g < ngroups && sc < p.end && row < ND) ? __ldg(p.mesh.map + row * cs + sc) : -1;
        }
      }
    }
  };
  int g = blockIdx.x * wpb + (threadIdx.x >> 5);
  load_maps(g);
  for (; g < ngroups; g += gstride) {
    double ureg[NT][KT];
    double cm[NT][NM];
    double X[NT][NV][DIM];
    int row_dof[NT][2][MT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int t = 0; t < KT; ++t) ureg[nt][t] = pf_dof[nt][t] >= 0 ? __ldg(p.u + pf_dof[nt][t]) : 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) load_vertex<DIM>(p.mesh.coords, pf_vid[nt][v] >= 0 ? pf_vid[nt][v] : 0, X[nt][v]);
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) row_dof[nt][e][mt] = pf_row[nt][e][mt];
    }
    int vid0[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) vid0[nt] = pf_vid[nt][0];
    load_maps(g + gstride);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      et_coeffs<FORM, DIM, NM>(X[nt], cm[nt]);
      if (vid0[nt] < 0) {
#pragma unroll
        for (int m = 0; m < NM; ++m) cm[nt][m] = 0.0;
      }
    }
    double acc[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

#pragma unroll
    for (int m = 0; m < NM; ++m) {
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        double b[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = cm[nt][m] * ureg[nt][kk];
        const double* a_ptr = sA + ((m * KT + kk) * MT) * 32 + lane;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double a = a_ptr[mt * 32];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt], a, b[nt]);
        }
      }
    }
    // scatter: acc[mt][nt][e] = Y[row = 8 mt + r][cell = base + 8 nt + 2 c4 + e]
    griddep_wait();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          if (row_dof[nt][e][mt] >= 0) scatter_add(p.y, row_dof[nt][e][mt], acc[mt][nt][e]);
  }
}

// ---------------------------------------------------------------------------
// Modal two-stage DMMA kernel (Helmholtz / scalar Laplacian on affine
// simplices, C2-P3/P4).  The reference gradients of P_k lie in P_{k-1}
// (dimension m: 10 for P3, 20 for P4), so with G_a = the m x nd coefficients
// of d/dxi_a phi_i in an L2-orthonormal basis of P_{k-1} (elements.
// stiffness_modes) the stiffness tensor factors as S_ab = G_a^T G_b and
//   y = sum_a G_a^T ( sum_b K_ab G_b u ) + |det J| Mhat u,
// i.e. the reference's quadrature loop (kernels.py:178-220) on the smallest
// possible "rule": m modes instead of (k+1)^3 points, 12 m nd + 2 nd^2 flops
// instead of the 14 nd^2 of the seven-matrix element tensor.
//
// Per group of 8 cells, two DMMA GEMMs with the modal combine in registers:
//   stage 1 (transposed): Gt[cell][col] = sum_j u_j(cell) Gcat[col][j]
//     A = u fragments in registers (lane l: u_{4t+l%4} of cell l/4),
//     B = Gcat fragments from shared memory; the accumulator leaves lane l
//     holding columns 8J + 2(l%4) + e of cell l/4.
//   combine: columns are assigned so that the DIM directions of one mode
//     sit in the SAME lane (each lane owns 2 NJ columns = floor(2NJ/DIM)
//     mode tuples; 4 lanes x 5 tuples = 20 modes for P4 in 8 column tiles),
//     so h_a = sum_b K_ab(cell) g_b is a register-only 3x3 product.
//   stage 2: Y[dof][cell] = sum_col Gcat[col][dof] H[col][cell]
//     + sum_j Mhat[dof][j] |det J| u_j: the stage-1 accumulator element
//     (J, e) is directly the B fragment of k-step 2J+e (lane l: k = l%4,
//     cell = l/4), the mass steps reuse the u fragments times |det J|.
// DMMA per 8 cells: P4 72 + 120 = 192 (the element tensor takes 315), P3
// 25 + 42 = 67 (105).
// ---------------------------------------------------------------------------

#ifndef FE_MODAL_SPLIT
#define FE_MODAL_SPLIT 1
#endif
template <int DIM, int NMODE>
struct ModalShape {
  static constexpr int tuples(int nj) { return (2 * nj) / DIM; }
  static constexpr int pick() {
    int nj = 1;
    while (4 * tuples(nj) < NMODE) ++nj;
    return nj;
  }
  // SPLIT (P3: 10 modes x 3 directions = 30 columns): whole tuples need 5
  // column tiles (4 lanes x 3 tuples = 12 mode slots for 10 modes, 25 + 42
  // DMMA per 8 cells).  Four tiles suffice when the last two modes are split
  // over lane pairs -- each lane owns 8 slots: two whole tuples (modes
  // 2c, 2c+1) and two leftovers; mode 8 + c/2 puts directions 0, 1 in the
  // even lane and direction 2 in the odd lane's first leftover, and the
  // combine exchanges those three values with one shuffle pair: 20 + 39 DMMA.
  static constexpr bool SPLIT = FE_MODAL_SPLIT && DIM == 3 && NMODE == 10;
  static constexpr int NJ = SPLIT ? 4 : pick();        // stage-1 column tiles
  static constexpr int TPL = SPLIT ? 2 : tuples(NJ);   // whole mode tuples per lane
  static constexpr int NSTEP = SPLIT ? 2 * NJ : DIM * TPL;  // stage-2 modal k-steps (one per lane slot)
  // (mode, direction) held by slot li of lane group c (mode -1: empty slot)
  static constexpr int mode_of(int c, int li) {
    if (li < DIM * TPL) return c * TPL + li / DIM < NMODE ? c * TPL + li / DIM : -1;
    if (!SPLIT || li >= 2 * NJ) return -1;
    const int e = li - DIM * TPL;
    return ((c & 1) == 0 || e == 0) ? 4 * TPL + (c >> 1) : -1;
  }
  static constexpr int dir_of(int c, int li) {
    if (li < DIM * TPL) return li % DIM;
    return (c & 1) == 0 ? li - DIM * TPL : 2;
  }
};

template <int FORM, int DIM, int ND, int NMODE, int NT, int MINB, int BLK = 256>
__global__ void __launch_bounds__(BLK, MINB) dmma_modal_kernel(DmmaParams p) {
  constexpr bool MASS = FORM == FE_FORM_HELMHOLTZ;
  constexpr int NM = et_nmats<FORM, DIM>();
  constexpr int KT = DmmaShape<ND>::KT, MT = DmmaShape<ND>::MT, NV = DIM + 1;
  using MS = ModalShape<DIM, NMODE>;
  constexpr int NJ = MS::NJ, TPL = MS::TPL, NSTEP = MS::NSTEP;
  constexpr int S2 = NSTEP + (MASS ? KT : 0);
  constexpr int B1SIZE = NJ * KT * 32, A2SIZE = S2 * MT * 32;
  extern __shared__ double smem[];
  double* sB1 = smem;            // [NJ][KT][32]
  double* sA2 = smem + B1SIZE;   // [S2][MT][32]
  {
    const double2* src = reinterpret_cast<const double2*>(p.afrag);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < (B1SIZE + A2SIZE) / 2; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, c4 = lane & 3;
  const int wpb = blockDim.x >> 5;
  const int64_t cs = p.mesh.nc_stride;
  const int ncell = p.end - p.start;
  const int ngroups = (ncell + 8 * NT - 1) / (8 * NT);
  const int gstride = gridDim.x * wpb;

  int pf_dof[NT][KT], pf_vid[NT][NV], pf_row[NT][2][MT];
  auto load_maps = [&](int g) {
    const int base = p.start + g * 8 * NT;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int cell = base + nt * 8 + r;
      const bool valid = g < ngroups && cell < p.end;
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        const int j = 4 * t + c4;
        pf_dof[nt][t] = (valid && j < ND) ? __ldg(p.mesh.map + j * cs + cell) : -1;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) pf_vid[nt][v] = valid ? __ldg(p.mesh.vmap + v * cs + cell) : -1;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int sc = base + nt * 8 + 2 * c4 + e;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int row = 8 * mt + r;
          pf_row[nt][e][mt] =
              (g < ngroups && sc < p.end && row < ND) ? __ldg(p.mesh.map + row * cs + sc) : -1;
        }
      }
    }
  };
  int g = blockIdx.x * wpb + (threadIdx.x >> 5);
  load_maps(g);
  for (; g < ngroups; g += gstride) {
    double ureg[NT][KT];
    double X[NT][NV][DIM];
    int row_dof[NT][2][MT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int t = 0; t < KT; ++t) ureg[nt][t] = pf_dof[nt][t] >= 0 ? __ldg(p.u + pf_dof[nt][t]) : 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) load_vertex<DIM>(p.mesh.coords, pf_vid[nt][v] >= 0 ? pf_vid[nt][v] : 0, X[nt][v]);
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) row_dof[nt][e][mt] = pf_row[nt][e][mt];
    }
    int vid0[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) vid0[nt] = pf_vid[nt][0];
    load_maps(g + gstride);

    // stage 1: modal gradients of the lane's cell
    double acc1[NT][NJ][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc1[nt][j][0] = acc1[nt][j][1] = 0.0;
#pragma unroll
    for (int t = 0; t < KT; ++t)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const double b = sB1[(j * KT + t) * 32 + lane];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma884(acc1[nt][j], ureg[nt][t], b);
      }

    // geometry of the lane's cell and the register-only modal combine
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double cm[NM];
      et_coeffs<FORM, DIM, NM>(X[nt], cm);
      if (vid0[nt] < 0) {
#pragma unroll
        for (int m = 0; m < NM; ++m) cm[m] = 0.0;
      }
      constexpr int O = MASS ? 1 : 0;
      double K[DIM][DIM];
      int m = O;
#pragma unroll
      for (int a = 0; a < DIM; ++a) K[a][a] = cm[m++];
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int b = a + 1; b < DIM; ++b) K[a][b] = K[b][a] = cm[m++];
#pragma unroll
      for (int s = 0; s < TPL; ++s) {
        double gv[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) gv[a] = acc1[nt][(DIM * s + a) / 2][(DIM * s + a) % 2];
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          double h = 0.0;
#pragma unroll
          for (int b = 0; b < DIM; ++b) h = fma(K[a][b], gv[b], h);
          acc1[nt][(DIM * s + a) / 2][(DIM * s + a) % 2] = h;
        }
      }
      if constexpr (MS::SPLIT) {
        // modes 8, 9: directions (0, 1) in the even lane's leftover slots, 2 in the odd lane's
        double& a6 = acc1[nt][NJ - 1][0];
        double& a7 = acc1[nt][NJ - 1][1];
        const double o6 = __shfl_xor_sync(0xffffffffu, a6, 1), o7 = __shfl_xor_sync(0xffffffffu, a7, 1);
        const bool odd = c4 & 1;
        const double gv0 = odd ? o6 : a6, gv1 = odd ? o7 : a7, gv2 = odd ? a6 : o6;
        const double h0 = fma(K[0][2], gv2, fma(K[0][1], gv1, K[0][0] * gv0));
        const double h1 = fma(K[1][2], gv2, fma(K[1][1], gv1, K[1][0] * gv0));
        const double h2 = fma(K[2][2], gv2, fma(K[2][1], gv1, K[2][0] * gv0));
        a6 = odd ? h2 : h0;
        a7 = odd ? 0.0 : h1;
      }
      if constexpr (MASS) {
#pragma unroll
        for (int t = 0; t < KT; ++t) ureg[nt][t] *= cm[0];
      }
    }

    // stage 2: back to the element's dofs (+ mass term)
    double acc[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
    for (int s = 0; s < S2; ++s) {
      const double* a_ptr = sA2 + (s * MT) * 32 + lane;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double a = a_ptr[mt * 32];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          dmma884(acc[mt][nt], a, s < NSTEP ? acc1[nt][s / 2][s % 2] : ureg[nt][s - NSTEP]);
      }
    }
    griddep_wait();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          if (row_dof[nt][e][mt] >= 0) scatter_add(p.y, row_dof[nt][e][mt], acc[mt][nt][e]);
  }
}

}  // namespace fe

// registry hook (plan.cu)
#define FE_DMMA_VARIANTS                                                                     \
  DMV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 3, 20),                                    \
  DMV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 4, 35),                                    \
  DMV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 4, 35),                                         \
  DMV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 4, 35),                            \
  DMMV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 3, 20, 10),                               \
  DMMV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 4, 35, 20),                               \
  DMMV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 3, 20, 10),                        \
  DMMV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 4, 35, 20),
