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
// GPU mapping
//  * a TEAM of Q^2 threads (3D) or Q threads (2D) per cell.  Teams of <= 32
//    threads are packed whole into warps (32/team per warp), so every
//    team-level barrier is a __syncwarp and warps run independently; larger
//    teams (Q >= 6 in 3D) share CTA barriers.  256-thread CTAs are
//    PERSISTENT and walk batches of CPB cells.  While a batch is being computed, the dof indices of the
//    batch after next and the u values / vertex data of the next batch are
//    already in flight into registers, and are parked in shared memory at
//    the end of the iteration -- the indirect gather P_e u overlaps the
//    arithmetic instead of stalling every CTA at its start.
//  * every contraction stage gives one thread one 1D pencil: it loads the
//    inputs along the contraction direction into registers once and emits
//    a whole output pencil (each shared-memory load feeds Q FMAs); B, D and
//    Dc are passed by value in the kernel parameter block and enter the
//    DFMAs as uniform constant-bank operands.
//  * shared-memory layouts put the CONSUMER's pencil index innermost (reads
//    are contiguous), and each buffer's outer stride is chosen at compile
//    time (pick_stride) so the producer's transposed writes are spread over
//    the 16 eight-byte banks.
//  * after the x-stage one thread holds all Q points of an x-pencil and
//    evaluates the flux there: the trilinear Jacobian is recomputed per point
//    (as kernels.py:136-151 does per qp on quads) from per-thread factors --
//    its d/dxi column is constant along the pencil and the other two are
//    linear in xi (6 FMAs per point).
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
  // even / odd parts of the mirror-symmetric 1D tables, rows q < ceil(Q/2)
  // (fill_tensor_tables): Xe[q][j] = (X[q][j] + X[q][P-1-j]) / 2 for j < P/2 and
  // X[q][(P-1)/2] in the middle column of an odd P; Xo[q][j] = (X[q][j] - X[q][P-1-j]) / 2
  double Be[(Q + 1) / 2][(P + 1) / 2], Bo[(Q + 1) / 2][(P + 1) / 2];
  double De[(Q + 1) / 2][(P + 1) / 2], Do[(Q + 1) / 2][(P + 1) / 2];
};

// ---- compile-time bank-conflict-aware strides --------------------------------
// Worst number of distinct 8-byte addresses sharing a bank (addr mod 16) in a
// half-warp, for lanes enumerating (s fastest over ns values, then r over nr)
// and address = r * rstep + s * sstep.
constexpr int bank_degree(int rstep, int sstep, int nr, int ns) {
  int worst = 0;
  const int n = nr * ns;
  for (int h = 0; h < n; h += 16) {
    int cnt[16] = {0};
    for (int l = h; l < h + 16 && l < n; ++l) {
      const int a = (l / ns) * rstep + (l % ns) * sstep;
      ++cnt[((a % 16) + 16) % 16];
    }
    for (int k = 0; k < 16; ++k) worst = cnt[k] > worst ? cnt[k] : worst;
  }
  return worst;
}
// smallest stride >= lo minimising conflicts when it multiplies r (outer) ...
constexpr int pick_outer(int lo, int nr, int ns, int sstep) {
  int best = lo, bd = bank_degree(lo, sstep, nr, ns);
  for (int st = lo + 1; st < lo + 16; ++st) {
    const int d = bank_degree(st, sstep, nr, ns);
    if (d < bd) { bd = d; best = st; }
  }
  return best;
}
// ... or the lane-fastest index s (inner)
constexpr int pick_inner(int lo, int nr, int ns, int rstep) {
  int best = lo, bd = bank_degree(rstep, lo, nr, ns);
  for (int st = lo + 1; st < lo + 16; ++st) {
    const int d = bank_degree(rstep, st, nr, ns);
    if (d < bd) { bd = d; best = st; }
  }
  return best;
}
constexpr int cmax3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }

#ifndef FE_TK_MONO
#define FE_TK_MONO 1    // monomial trilinear geometry (round 2)
#endif
#ifndef FE_TK_SYM
#define FE_TK_SYM 1     // mirror-symmetric table reads (round 2)
#endif
#ifndef FE_TK_FLATZ
#define FE_TK_FLATZ 0   // 1: one z stage for all components of a vector form; measured neutral
#endif                  // (C4-hex-Q2 0.456 -> 0.460 ms, C4-hex-Q3 1.244 -> 1.239 ms, profiles/r02/ab_tensor_flatz.txt)
#ifndef FE_TK_EO
#define FE_TK_EO 1   // even-odd 1D contractions in the DIRECT variants: C3-Q5 0.967 -> 0.917 ms, C3-Q6 1.676 -> 1.532 ms (profiles/r02/ab_tensor_eo.txt)
#endif
#ifndef FE_TK_RCPALL
#define FE_TK_RCPALL 0
#endif
#ifndef FE_TK_CPENCIL
#define FE_TK_CPENCIL 1
#endif
#ifndef FE_TK_ASYNC
#define FE_TK_ASYNC 0   // 1: cp.async gather pipeline (no prefetch registers)
#endif

// DIRECT: use the direct algorithm even when p == q (measured faster at
// Q5/Q6, where the collocation stages' cross-pencil Dc reads, 2 q^4 shared
// loads per component, outweigh its 25% flop saving)
template <int DIM, int P, int Q, int VS, bool DIRECT = false, int BLOCK_ = 256, bool ASYNC = false>
struct TensorLayout {
  static constexpr int BLOCK = BLOCK_;                       // threads per CTA
  static constexpr int TS = DIM == 3 ? Q * Q : Q;          // threads per cell (team)
  // teams of <= 32 threads are packed whole into warps, so every team-level
  // barrier is a __syncwarp and warps never wait for each other
  static constexpr bool WARP_TEAMS = TS <= 32;
  static constexpr int TPW = WARP_TEAMS ? 32 / TS : 0;      // teams per warp
  static constexpr int CPB = WARP_TEAMS ? (BLOCK / 32) * TPW : BLOCK / TS;  // cells per CTA
  static constexpr int ND = DIM == 3 ? P * P * P : P * P;  // scalar dofs per cell
  static constexpr int NV = DIM == 3 ? 8 : 4;
  static constexpr int RU = (ND + TS - 1) / TS;            // dofs gathered per thread
  static constexpr int RX = (NV * DIM + TS - 1) / TS;      // vertex coordinates per thread
  static constexpr int RM = (NV + TS - 1) / TS;            // vertex field values per thread
  static constexpr bool COLLOC = !DIRECT && DIM == 3 && P == Q;
  // 3D buffers (producer pencil -> consumer pencil):
  //  Z[j][c][i]  stride SZ: written by (i,j) over c, read by (i,c) over j
  //  Y[i][c][b]  stride SY: written by (i,c) over b, read by (b,c) over i
  //  G[a][c][b]  stride Q^2 (collocation: u and flux at the points)
  //  A[b][c][i]  stride SA: written by (b,c) over i, read by (i,c) over b
  //  W[c][j][i]  stride SW: written by (i,c) over j, read by (i,j) over c
  // 2D: Y[b][i], A[b][i], stride S2 = 1 (mod 16)
  static constexpr int SZ = pick_outer(Q * P, P, P, 1);
  static constexpr int SY = pick_inner(Q * Q, Q, P, Q);
  static constexpr int SA = pick_inner(Q * P, Q, Q, P);
  static constexpr int SW = pick_outer(P * P, Q, P, 1);
  static constexpr int S2 = P + ((17 - P) % 16 + 16) % 16;
  static constexpr int NZ = COLLOC ? 1 : 2;
  static constexpr int NY = COLLOC ? 1 : 3;
  // FLATZ (vector forms, direct algorithm): the z stages of all VS components run
  // as one stage over VS P^2 pencils, so Z and W of every component are resident
  static constexpr bool FLATZ = FE_TK_FLATZ && DIM == 3 && VS > 1 && !COLLOC;
  static constexpr int ZS = NZ * P * SZ;                    // Z region of one component
  static constexpr int WS = 2 * Q * SW;                     // W region of one component
  static constexpr int R1 = DIM == 3 ? cmax3((FLATZ ? VS : 1) * ZS, 2 * Q * Q * Q, (FLATZ ? VS : 1) * WS) : 0;
  static constexpr int R2 = DIM == 3 ? cmax3(NY * P * SY, 3 * Q * SA, COLLOC ? Q * Q * Q : 0) : 2 * Q * S2;
  // per-cell region
  static constexpr int U = 0;
  static constexpr int O1 = U + VS * ND;
  static constexpr int O2 = O1 + R1;
  static constexpr int X = O2 + R2;
  static constexpr int MU = X + NV * DIM;
  static constexpr int LAM = MU + NV;
  // FE_TK_ASYNC: second data buffer (u, coordinates, mu/lambda) and two
  // map-row buffers (ND dof ids + NV vertex ids, int32) for the cp.async
  // gather pipeline
  static constexpr int MBW = (ND + NV + 1) / 2;            // map buffer width in doubles
  static constexpr int UA = LAM + NV;
  static constexpr int XA = UA + VS * ND;
  static constexpr int MUA = XA + NV * DIM;
  static constexpr int LAMA = MUA + NV;
  static constexpr int MB0 = LAMA + NV;
  static constexpr int MB1 = MB0 + MBW;
  static constexpr int raw = ASYNC ? MB1 + MBW : LAM + NV;
  static constexpr int size = raw + ((TS - raw) % 16 + 16) % 16;  // team stride == TS (mod 16)
};

// MINB: CTAs per SM the register allocation must allow, chosen per variant
// from measurements (profiles/r01/sweep_minb2.jsonl): 1 or 2 with 256-thread
// CTAs, 3 with 128-thread CTAs (<= 170 registers, 12 warps per SM)
// MINB >= 100 encodes a CTA size of MINB threads at 2 CTAs per SM (e.g.
// 192: 5 teams of 36 at Q = 6 with a 170-register budget instead of 7 teams
// and 128 registers + spills)
// MINB >= 1000: the same with the cp.async gather pipeline (FE_TK_ASYNC
// per variant: C3-Q5 0.38 -> 0.45 of its roof; slower where its extra
// shared memory costs occupancy, profiles/r02/ab_tensor_async.txt)
// mirror-symmetric table reads, where measured faster (profiles/r02/ab_tensor_sym.txt):
// (P, Q) = (4, 5), whose full tables overflow the uniform registers into vector
// registers + R2UR (C4-hex-Q3 1.269 -> 1.244 ms); neutral to slower elsewhere,
// and at Q = 7 halving the tables tips ptxas from in-loop LDCU loads to
// hoisting them into vector registers (459 R2UR, 1.68 -> 2.29 ms)
template <int P, int Q> constexpr bool tensor_sym() { return FE_TK_SYM != 0 && P == 4 && Q == 5; }
// even-odd 1D contractions: every 3D variant on the direct algorithm with P >= 4
// (measured: C3-Q5/Q6 -5% / -9%, C4-hex-Q3 -2.7%; slower at P = 3, profiles/r02/ab_tensor_eo.txt)
template <int DIM, int P, int Q, bool DIRECT> constexpr bool tensor_eo() {
  return FE_TK_EO != 0 && DIM == 3 && (DIRECT || P != Q) && P >= 4;
}
template <int MINB> constexpr bool tensor_async() { return MINB >= 1000 || FE_TK_ASYNC; }
template <int MINB> constexpr int tensor_block() {
  constexpr int m = MINB % 1000;
  return m >= 100 ? m : (m >= 3 ? 128 : 256);
}
template <int MINB> constexpr int tensor_minb() { return MINB % 1000 >= 100 ? 2 : MINB % 1000; }

template <int FORM, int DIM, int P, int Q, int MINB, bool DIRECT>
__global__ void __launch_bounds__(tensor_block<MINB>(), tensor_minb<MINB>())
tensor_kernel(const __grid_constant__ TensorParams<Q, P> p) {
  static_assert(Q >= P, "team layout assumes Q >= P");
  constexpr int VS = form_vs(FORM, DIM);
  constexpr bool ASYNC = tensor_async<MINB>();
  using L = TensorLayout<DIM, P, Q, VS, DIRECT, tensor_block<MINB>(), ASYNC>;
  constexpr int TS = L::TS, CPB = L::CPB, ND = L::ND, NV = L::NV, RU = L::RU;
  constexpr bool COLLOC = L::COLLOC;
  constexpr bool FASTR = FE_TK_RCPALL || !DIRECT;   // MUFU-seeded reciprocal (IEEE division in the DIRECT variants: measured)
  constexpr bool CPEN = COLLOC && FE_TK_CPENCIL && Q >= 6 && VS == 1;   // pencil-stage collocation derivatives
  constexpr int QQ = Q * Q;
  extern __shared__ double smem_all[];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int team = L::WARP_TEAMS ? warp * L::TPW + lane / TS : threadIdx.x / TS;
  const int t = L::WARP_TEAMS ? lane % TS : threadIdx.x % TS;
  const bool in_team = L::WARP_TEAMS ? lane < L::TPW * TS : team < CPB;
  auto team_sync = []() {
    if constexpr (L::WARP_TEAMS) __syncwarp();
    else __syncthreads();
  };
  double* sm = smem_all + (in_team ? team : 0) * L::size;
  double* sU = sm + L::U;              // the data buffers of the batch being computed
  double* s1 = sm + L::O1;
  double* s2 = sm + L::O2;
  double* sX = sm + L::X;
  double* sMU = sm + L::MU;
  double* sLAM = sm + L::LAM;
  const int64_t cs = p.mesh.nc_stride;
  const int ncell = p.end - p.start;
  const int nbatch = (ncell + CPB - 1) / CPB;
  // FE_TK_SYM: the 1D tables are mirror-symmetric about 1/2 (verified at plan
  // time): B[q][i] = B[Q-1-q][P-1-i], D[q][i] = -D[Q-1-q][P-1-i].  Reading
  // only the lower half halves the distinct constants of the persistent
  // loop: sm_100a feeds constant operands through ~80 uniform registers, and
  // when the tables do not fit ptxas parks them in vector registers and moves
  // them back with R2UR inside the loop (C4-hex-Q3: 303 R2UR + 139 MOV.SPILL
  // per 1598 FP64 instructions before this).
  constexpr bool SYM = tensor_sym<P, Q>();
  auto TB = [&](int q, int i) { return (!SYM || 2 * q < Q) ? p.B[q][i] : p.B[Q - 1 - q][P - 1 - i]; };
  auto TD = [&](int q, int i) { return (!SYM || 2 * q < Q) ? p.D[q][i] : -p.D[Q - 1 - q][P - 1 - i]; };
  auto TX = [&](int q) { return (!SYM || 2 * q < Q) ? p.x[q] : 1.0 - p.x[Q - 1 - q]; };
  auto TW = [&](int q) { return (!SYM || 2 * q < Q) ? p.w[q] : p.w[Q - 1 - q]; };
  // FE_TK_EO: even-odd decomposition of the 1D contractions (DIRECT 3D variants).
  // With mirror-symmetric tables the rows q and Q-1-q share their products:
  // out[q] = E + O, out[Q-1-q] = +-(E - O) with E = sum Xe[q][j] (x[j] + x[P-1-j]),
  // O = sum Xo[q][j] (x[j] - x[P-1-j]): P + 2 instead of 2P FP64 slots per output pair.
  constexpr bool EO = tensor_eo<DIM, P, Q, DIRECT>();
  constexpr int HP = P / 2, NE = (P + 1) / 2, HQ = Q / 2;
  auto eo_split = [&](const double (&x)[P], double (&xe)[NE], double (&xo)[NE]) {
#pragma unroll
    for (int j = 0; j < HP; ++j) {
      xe[j] = x[j] + x[P - 1 - j];
      xo[j] = x[j] - x[P - 1 - j];
    }
    if constexpr (P % 2) { xe[HP] = x[HP]; xo[HP] = 0.0; }
  };
  auto eo_fwdB = [&](const double (&xe)[NE], const double (&xo)[NE], double (&out)[Q]) {
#pragma unroll
    for (int q = 0; q < HQ; ++q) {
      double E = 0.0, O = 0.0;
#pragma unroll
      for (int j = 0; j < NE; ++j) E = fma(p.Be[q][j], xe[j], E);
#pragma unroll
      for (int j = 0; j < HP; ++j) O = fma(p.Bo[q][j], xo[j], O);
      out[q] = E + O;
      out[Q - 1 - q] = E - O;
    }
    if constexpr (Q % 2) {
      double E = 0.0;
#pragma unroll
      for (int j = 0; j < NE; ++j) E = fma(p.Be[HQ][j], xe[j], E);
      out[HQ] = E;
    }
  };
  auto eo_fwdD = [&](const double (&xe)[NE], const double (&xo)[NE], double (&out)[Q]) {
#pragma unroll
    for (int q = 0; q < HQ; ++q) {
      double E = 0.0, O = 0.0;
#pragma unroll
      for (int j = 0; j < NE; ++j) E = fma(p.De[q][j], xe[j], E);
#pragma unroll
      for (int j = 0; j < HP; ++j) O = fma(p.Do[q][j], xo[j], O);
      out[q] = O + E;
      out[Q - 1 - q] = O - E;
    }
    if constexpr (Q % 2) {
      double O = 0.0;
#pragma unroll
      for (int j = 0; j < HP; ++j) O = fma(p.Do[HQ][j], xo[j], O);
      out[HQ] = O;
    }
  };
  // adjoints: accumulate sum_q X[q][j] f[q] in even/odd form, then eo_merge
  auto eo_adjB = [&](const double (&f)[Q], double (&ae)[NE], double (&ao)[NE]) {
#pragma unroll
    for (int q = 0; q < HQ; ++q) {
      const double fp = f[q] + f[Q - 1 - q], fm = f[q] - f[Q - 1 - q];
#pragma unroll
      for (int j = 0; j < NE; ++j) ae[j] = fma(p.Be[q][j], fp, ae[j]);
#pragma unroll
      for (int j = 0; j < HP; ++j) ao[j] = fma(p.Bo[q][j], fm, ao[j]);
    }
    if constexpr (Q % 2) {
#pragma unroll
      for (int j = 0; j < NE; ++j) ae[j] = fma(p.Be[HQ][j], f[HQ], ae[j]);
    }
  };
  auto eo_adjD = [&](const double (&f)[Q], double (&ae)[NE], double (&ao)[NE]) {
#pragma unroll
    for (int q = 0; q < HQ; ++q) {
      const double fp = f[q] + f[Q - 1 - q], fm = f[q] - f[Q - 1 - q];
#pragma unroll
      for (int j = 0; j < NE; ++j) ae[j] = fma(p.De[q][j], fm, ae[j]);
#pragma unroll
      for (int j = 0; j < HP; ++j) ao[j] = fma(p.Do[q][j], fp, ao[j]);
    }
    if constexpr (Q % 2) {
#pragma unroll
      for (int j = 0; j < HP; ++j) ao[j] = fma(p.Do[HQ][j], f[HQ], ao[j]);
    }
  };
  auto eo_merge = [&](const double (&ae)[NE], const double (&ao)[NE], double (&out)[P]) {
#pragma unroll
    for (int j = 0; j < HP; ++j) {
      out[j] = ae[j] + ao[j];
      out[P - 1 - j] = ae[j] - ao[j];
    }
    if constexpr (P % 2) out[HP] = ae[HP];
  };
  auto eo_zero = [&](double (&ae)[NE], double (&ao)[NE]) {
#pragma unroll
    for (int j = 0; j < NE; ++j) ae[j] = ao[j] = 0.0;
  };

  // ---- prefetch pipeline: map indices two batches ahead, data one ahead ----
  constexpr int RX = L::RX, RM = L::RM;
  int pf_map[RU];
  double pf_u[RU][VS];
  double pf_x[RX], pf_m[RM], pf_l[RM];
  auto cell_of = [&](int batch) { return p.start + batch * CPB + team; };
  auto load_map = [&](int batch) {
    const int c = cell_of(batch);
    const bool ok = in_team && batch < nbatch && c < p.end;
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int idx = t + r * TS;
      pf_map[r] = (ok && idx < ND) ? __ldg(p.maplex + (int64_t)c * ND + idx) : -1;
    }
  };
  auto load_data = [&](int batch) {
    const int c = cell_of(batch);
    const bool ok = in_team && batch < nbatch && c < p.end;
#pragma unroll
    for (int r = 0; r < RU; ++r)
#pragma unroll
      for (int k = 0; k < VS; ++k)
        pf_u[r][k] = pf_map[r] >= 0 ? __ldg(p.u + (int64_t)VS * pf_map[r] + k) : 0.0;
#pragma unroll
    for (int r = 0; r < RX; ++r) {
      const int e = t + r * TS;
      pf_x[r] = 0.0;
      if (ok && e < NV * DIM) {
        const int vid = __ldg(p.mesh.vmap + (e / DIM) * cs + c);
        pf_x[r] = __ldg(p.mesh.coords + (int64_t)vid * CStride<DIM>::value + e % DIM);
      }
    }
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const int v = t + r * TS;
        pf_m[r] = pf_l[r] = 0.0;
        if (ok && v < NV) {
          const int vid = __ldg(p.mesh.vmap + v * cs + c);
          pf_m[r] = __ldg(p.mu + vid);
          pf_l[r] = __ldg(p.lam + vid);
        }
      }
    }
  };
  auto park = [&]() {  // prefetched registers -> this team's shared memory
    if (!in_team) return;
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int idx = t + r * TS;
      if (idx < ND)
#pragma unroll
        for (int k = 0; k < VS; ++k) sU[k * ND + idx] = pf_u[r][k];
    }
#pragma unroll
    for (int r = 0; r < RX; ++r)
      if (t + r * TS < NV * DIM) sX[t + r * TS] = pf_x[r];
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
#pragma unroll
      for (int r = 0; r < RM; ++r)
        if (t + r * TS < NV) {
          sMU[t + r * TS] = pf_m[r];
          sLAM[t + r * TS] = pf_l[r];
        }
    }
  };

  // ---- FE_TK_ASYNC: the same pipeline through cp.async (LDGSTS) straight
  // into shared memory -- map rows + vertex ids two batches ahead, u /
  // coordinates / mu, lambda one ahead, double-buffered -- so no prefetched
  // value occupies a register during the compute
  int32_t* const mbuf0 = reinterpret_cast<int32_t*>(sm + L::MB0);
  int32_t* const mbuf1 = reinterpret_cast<int32_t*>(sm + L::MB1);
  auto issue_maps = [&](int batch, int32_t* mb) {
    if (!in_team) return;
    const int c = cell_of(batch);
    const bool ok = batch < nbatch && c < p.end;
    for (int idx = t; idx < ND + NV; idx += TS) {
      if (!ok) mb[idx] = -1;
      else if (idx < ND) cp_async4(mb + idx, p.maplex + (int64_t)c * ND + idx);
      else cp_async4(mb + idx, p.mesh.vmap + (idx - ND) * cs + c);
    }
  };
  auto issue_data = [&](const int32_t* mb, int par) {
    if (!in_team) return;
    double* du = sm + (par ? L::UA : L::U);
    double* dx = sm + (par ? L::XA : L::X);
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int idx = t + r * TS;
      if (idx < ND) {
        const int m = mb[idx];
#pragma unroll
        for (int k = 0; k < VS; ++k) cp_async8_zfill(du + k * ND + idx, p.u + (m >= 0 ? (int64_t)VS * m + k : 0), m >= 0);
      }
    }
#pragma unroll
    for (int r = 0; r < RX; ++r) {
      const int e = t + r * TS;
      if (e < NV * DIM) {
        const int vid = mb[ND + e / DIM];
        cp_async8_zfill(dx + e, p.mesh.coords + (vid >= 0 ? (int64_t)vid * CStride<DIM>::value + e % DIM : 0), vid >= 0);
      }
    }
    if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
      double* dm = sm + (par ? L::MUA : L::MU);
      double* dl = sm + (par ? L::LAMA : L::LAM);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const int v = t + r * TS;
        if (v < NV) {
          const int vid = mb[ND + v];
          cp_async8_zfill(dm + v, p.mu + (vid >= 0 ? vid : 0), vid >= 0);
          cp_async8_zfill(dl + v, p.lam + (vid >= 0 ? vid : 0), vid >= 0);
        }
      }
    }
  };
  auto select_buffers = [&](int par) {
    sU = sm + (par ? L::UA : L::U);
    sX = sm + (par ? L::XA : L::X);
    sMU = sm + (par ? L::MUA : L::MU);
    sLAM = sm + (par ? L::LAMA : L::LAM);
  };

  int batch = blockIdx.x;
  if constexpr (ASYNC) {
    issue_maps(batch, mbuf0);
    cp_commit();
    cp_wait_group<0>();
    team_sync();
    issue_data(mbuf0, 0);
    cp_commit();
    issue_maps(batch + gridDim.x, mbuf1);
    cp_commit();
    cp_wait_group<1>();                  // data of the first batch
    team_sync();
  } else {
    load_map(batch);
    load_data(batch);
    park();
    load_map(batch + gridDim.x);
    team_sync();
  }

  for (int it = 0; batch < nbatch; batch += gridDim.x, ++it) {
    const int cell = cell_of(batch);
    const bool active = in_team && cell < p.end;
    if constexpr (ASYNC) {
      cp_wait_group<0>();                // map rows of the next batch
      team_sync();
      const int par = it & 1;
      select_buffers(par);
      issue_data(par ? mbuf0 : mbuf1, par ^ 1);   // next batch's data, other buffer
      cp_commit();
      issue_maps(batch + 2 * gridDim.x, par ? mbuf1 : mbuf0);
      cp_commit();
    } else {
      // issue the next batch's gathers now; they land while this batch computes
      load_data(batch + gridDim.x);
      load_map(batch + 2 * gridDim.x);
    }

#if FE_TK_MONO
    // trilinear map in monomial form, once per cell: x = sum C_abc xi^a eta^b
    // zeta^c, thread d < 3 converting coordinate d in place (slot a + 2b + 4c).
    // The per-pencil Jacobian factors below then cost 6 FMAs per coordinate
    // instead of ~40 operations on vertex differences.  Consumed after the
    // z-stage barrier.
    if constexpr (DIM == 3) {
      if (active && t < 3) {
        double xv[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) xv[v] = sX[v * 3 + t];
        sX[1 * 3 + t] = xv[1] - xv[0];
        sX[2 * 3 + t] = xv[2] - xv[0];
        sX[4 * 3 + t] = xv[4] - xv[0];
        sX[3 * 3 + t] = (xv[3] - xv[2]) - (xv[1] - xv[0]);
        sX[5 * 3 + t] = (xv[5] - xv[4]) - (xv[1] - xv[0]);
        sX[6 * 3 + t] = (xv[6] - xv[4]) - (xv[2] - xv[0]);
        sX[7 * 3 + t] = ((xv[7] - xv[6]) - (xv[5] - xv[4])) - ((xv[3] - xv[2]) - (xv[1] - xv[0]));
      }
      if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {   // mu, lambda likewise
        if (active && (t == 3 || t == 4)) {
          double* f = t == 3 ? sMU : sLAM;
          double xv[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) xv[v] = f[v];
          f[1] = xv[1] - xv[0];
          f[2] = xv[2] - xv[0];
          f[4] = xv[4] - xv[0];
          f[3] = (xv[3] - xv[2]) - (xv[1] - xv[0]);
          f[5] = (xv[5] - xv[4]) - (xv[1] - xv[0]);
          f[6] = (xv[6] - xv[4]) - (xv[2] - xv[0]);
          f[7] = ((xv[7] - xv[6]) - (xv[5] - xv[4])) - ((xv[3] - xv[2]) - (xv[1] - xv[0]));
        }
      }
    }
#endif
    // ---- forward: reference gradients at the points of this thread's x-pencil
    double g[VS][DIM][Q];
    constexpr bool FLATZ = L::FLATZ;
    // z: pencil (i, j) over k -> Z0 = B u (Z1 = D u: direct)      Z[j][c][i]
    auto z_stage = [&](const double* uc, double* zb, int e) {
      const int i = e % P, j = e / P;
      double pen[P];
#pragma unroll
      for (int k = 0; k < P; ++k) pen[k] = uc[k * P * P + e];
      if constexpr (EO) {
        double xe[NE], xo[NE], z0[Q], z1[Q];
        eo_split(pen, xe, xo);
        eo_fwdB(xe, xo, z0);
        eo_fwdD(xe, xo, z1);
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          zb[j * L::SZ + c * P + i] = z0[c];
          zb[P * L::SZ + j * L::SZ + c * P + i] = z1[c];
        }
        return;
      }
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double z0 = 0.0, z1 = 0.0;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          z0 = fma(TB(c, k), pen[k], z0);
          if constexpr (!COLLOC) z1 = fma(TD(c, k), pen[k], z1);
        }
        zb[j * L::SZ + c * P + i] = z0;
        if constexpr (!COLLOC) zb[P * L::SZ + j * L::SZ + c * P + i] = z1;
      }
    };
    if constexpr (FLATZ) {
      // all VS P^2 pencils of the cell as one stage: ceil(VS P^2 / TS) rounds of the
      // team instead of VS rounds with P^2 of its Q^2 threads busy
#pragma unroll
      for (int r = 0; r < (VS * P * P + TS - 1) / TS; ++r) {
        const int it = t + r * TS;
        if (active && it < VS * P * P) z_stage(sU + (it / (P * P)) * ND, s1 + (it / (P * P)) * L::ZS, it % (P * P));
      }
      team_sync();
    }
#pragma unroll
    for (int comp = 0; comp < VS; ++comp) {
      const double* uc = sU + comp * ND;
      if constexpr (DIM == 3) {
        double* const s1f = s1;   // this component's Z region
        double* s1 = s1f + (FLATZ ? comp * L::ZS : 0);
        if constexpr (!FLATZ) {
          if (active && t < P * P) z_stage(uc, s1, t);
          team_sync();
        }
        // y: pencil (i, c) over j -> Y0 = B Z0 (Y1 = D Z0, Y2 = B Z1)    Y[i][c][b]
        if (active && t < Q * P) {
          const int i = t % P, c = t / P;
          double p0[P], p1[P];
#pragma unroll
          for (int j = 0; j < P; ++j) {
            p0[j] = s1[j * L::SZ + t];
            if constexpr (!COLLOC) p1[j] = s1[P * L::SZ + j * L::SZ + t];
          }
          if constexpr (EO) {
            double xe[NE], xo[NE], y0[Q], y1[Q], y2[Q];
            eo_split(p0, xe, xo);
            eo_fwdB(xe, xo, y0);
            eo_fwdD(xe, xo, y1);
            eo_split(p1, xe, xo);
            eo_fwdB(xe, xo, y2);
#pragma unroll
            for (int b = 0; b < Q; ++b) {
              s2[i * L::SY + c * Q + b] = y0[b];
              s2[P * L::SY + i * L::SY + c * Q + b] = y1[b];
              s2[2 * P * L::SY + i * L::SY + c * Q + b] = y2[b];
            }
          } else
#pragma unroll
          for (int b = 0; b < Q; ++b) {
            double y0 = 0.0, y1 = 0.0, y2 = 0.0;
#pragma unroll
            for (int j = 0; j < P; ++j) {
              y0 = fma(TB(b, j), p0[j], y0);
              if constexpr (!COLLOC) {
                y1 = fma(TD(b, j), p0[j], y1);
                y2 = fma(TB(b, j), p1[j], y2);
              }
            }
            s2[i * L::SY + c * Q + b] = y0;
            if constexpr (!COLLOC) {
              s2[P * L::SY + i * L::SY + c * Q + b] = y1;
              s2[2 * P * L::SY + i * L::SY + c * Q + b] = y2;
            }
          }
        }
        team_sync();
        if constexpr (COLLOC) {
          // x: pencil (b, c) over i -> u at the points; d/dxi locally      G[a][c][b]
          if (active) {
            const int b = t % Q, c = t / Q;
            double q0[P], uq[Q];
#pragma unroll
            for (int i = 0; i < P; ++i) q0[i] = s2[i * L::SY + t];
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              double s = 0.0;
#pragma unroll
              for (int i = 0; i < P; ++i) s = fma(TB(a, i), q0[i], s);
              uq[a] = s;
              s1[a * QQ + t] = s;
            }
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              double s = 0.0;
#pragma unroll
              for (int e = 0; e < Q; ++e) s = fma(p.Dc[a][e], uq[e], s);
              g[comp][0][a] = s;
            }
            (void)b;
            (void)c;
          }
          team_sync();
          if constexpr (CPEN) {
            // d/deta, d/dzeta as pencil stages too: thread (a, c) differentiates the
            // eta line U[a][c][.] and thread (a, b) the zeta line U[a][.][b] -- every
            // table entry a compile-time (uniform) operand, Q loads + Q stores per Q^2
            // FMAs instead of one shared load per FMA and lane-indexed Dc rows
            if (active) {
              const int a = t % Q, o = t / Q;
              double pen[Q];
#pragma unroll
              for (int e = 0; e < Q; ++e) pen[e] = s1[a * QQ + o * Q + e];
#pragma unroll
              for (int b = 0; b < Q; ++b) {
                double s = 0.0;
#pragma unroll
                for (int e = 0; e < Q; ++e) s = fma(p.Dc[b][e], pen[e], s);
                s2[a * QQ + o * Q + b] = s;                       // d/deta   [a][c][b]
              }
#pragma unroll
              for (int e = 0; e < Q; ++e) pen[e] = s1[a * QQ + e * Q + o];
#pragma unroll
              for (int c = 0; c < Q; ++c) {
                double s = 0.0;
#pragma unroll
                for (int e = 0; e < Q; ++e) s = fma(p.Dc[c][e], pen[e], s);
                s1[Q * QQ + a * QQ + c * Q + o] = s;              // d/dzeta  [a][c][b]
              }
            }
            team_sync();
            if (active) {
#pragma unroll
              for (int a = 0; a < Q; ++a) {
                g[comp][1][a] = s2[a * QQ + t];
                g[comp][2][a] = s1[Q * QQ + a * QQ + t];
              }
            }
          } else {
          // d/deta, d/dzeta with Dc across the pencils of the team
          if (active) {
            const int b = t % Q, c = t / Q;
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              double sa = 0.0, sb = 0.0;
#pragma unroll
              for (int e = 0; e < Q; ++e) {
                sa = fma(p.Dc[b][e], s1[a * QQ + c * Q + e], sa);
                sb = fma(p.Dc[c][e], s1[a * QQ + e * Q + b], sb);
              }
              g[comp][1][a] = sa;
              g[comp][2][a] = sb;
            }
          }
          }
          team_sync();
        } else {
          // x: pencil (b, c) over i -> d/dxi = D Y0, d/deta = B Y1, d/dzeta = B Y2
          if (active) {
            double q0[P], q1[P], q2[P];
#pragma unroll
            for (int i = 0; i < P; ++i) {
              q0[i] = s2[i * L::SY + t];
              q1[i] = s2[P * L::SY + i * L::SY + t];
              q2[i] = s2[2 * P * L::SY + i * L::SY + t];
            }
            if constexpr (EO) {
              double xe[NE], xo[NE];
              eo_split(q0, xe, xo);
              eo_fwdD(xe, xo, g[comp][0]);
              eo_split(q1, xe, xo);
              eo_fwdB(xe, xo, g[comp][1]);
              eo_split(q2, xe, xo);
              eo_fwdB(xe, xo, g[comp][2]);
            } else
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              double g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
              for (int i = 0; i < P; ++i) {
                g0 = fma(TD(a, i), q0[i], g0);
                g1 = fma(TB(a, i), q1[i], g1);
                g2 = fma(TB(a, i), q2[i], g2);
              }
              g[comp][0][a] = g0;
              g[comp][1][a] = g1;
              g[comp][2][a] = g2;
            }
          }
          team_sync();
        }
      } else {
        // y: pencil i over j -> Y0 = B u, Y1 = D u                         Y[b][i]
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
              y0 = fma(TB(b, j), pen[j], y0);
              y1 = fma(TD(b, j), pen[j], y1);
            }
            s2[b * L::S2 + i] = y0;
            s2[Q * L::S2 + b * L::S2 + i] = y1;
          }
        }
        team_sync();
        if (active) {
          const int b = t;
          double q0[P], q1[P];
#pragma unroll
          for (int i = 0; i < P; ++i) {
            q0[i] = s2[b * L::S2 + i];
            q1[i] = s2[Q * L::S2 + b * L::S2 + i];
          }
#pragma unroll
          for (int a = 0; a < Q; ++a) {
            double g0 = 0.0, g1 = 0.0;
#pragma unroll
            for (int i = 0; i < P; ++i) {
              g0 = fma(TD(a, i), q0[i], g0);
              g1 = fma(TB(a, i), q1[i], g1);
            }
            g[comp][0][a] = g0;
            g[comp][1][a] = g1;
          }
        }
        team_sync();
      }
    }

    // ---- pointwise flux at the Q points of the x-pencil --------------------
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
        if constexpr (DIM == 3 && FE_TK_MONO) {
          d1[d] = fma(zeta, Xv(1, 1, 1, d), Xv(1, 1, 0, d));
          c0[d] = fma(eta, d1[d], fma(zeta, Xv(1, 0, 1, d), Xv(1, 0, 0, d)));
          j1[d] = fma(zeta, Xv(0, 1, 1, d), Xv(0, 1, 0, d));
          j2[d] = fma(eta, Xv(0, 1, 1, d), Xv(0, 0, 1, d));
          d2[d] = fma(eta, Xv(1, 1, 1, d), Xv(1, 0, 1, d));
        } else if constexpr (DIM == 3) {
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
      if constexpr (FORM == FE_FORM_ELASTICITY_LAME && DIM == 3 && FE_TK_MONO) {
        m0 = fma(eta, fma(zeta, sMU[6], sMU[2]), fma(zeta, sMU[4], sMU[0]));
        dm = fma(eta, fma(zeta, sMU[7], sMU[3]), fma(zeta, sMU[5], sMU[1]));
        l0 = fma(eta, fma(zeta, sLAM[6], sLAM[2]), fma(zeta, sLAM[4], sLAM[0]));
        dl = fma(eta, fma(zeta, sLAM[7], sLAM[3]), fma(zeta, sLAM[5], sLAM[1]));
      } else if constexpr (FORM == FE_FORM_ELASTICITY_LAME) {
        double mx[2] = {0.0, 0.0}, lx[2] = {0.0, 0.0};
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int vx = v & 1, vy = (v >> 1) & 1, vz = v >> 2;
          const double wgt = DIM == 3 ? Ly[vy] * Lz[vz] : Ly[vy];
          mx[vx] += wgt * sMU[v];
          lx[vx] += wgt * sLAM[v];
        }
        m0 = mx[0]; dm = mx[1] - mx[0];
        l0 = lx[0]; dl = lx[1] - lx[0];
      }
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        const double xi = TX(a);
        double J[DIM][DIM], Ji[DIM][DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          J[d][0] = c0[d];
          J[d][1] = fma(xi, d1[d], j1[d]);
          if constexpr (DIM == 3) J[d][2] = fma(xi, d2[d], j2[d]);
        }
        // fast reciprocal except in the DIRECT (Q5/Q6) variants: measured
        // (profiles/r01/sweep_rcp.txt)
#ifndef TK_ADJ
#define TK_ADJ 1
#endif
        // linear gradient forms: Ji holds adj(J), the weight w / |det J|
        // absorbs both 1/det factors (no inverse formed)
        constexpr bool ADJ = TK_ADJ && linear_grad_form(FORM);
        const double det = ADJ ? det_adj<DIM>(J, Ji) : det_inv<DIM, FASTR>(J, Ji);
        const double tw = ADJ ? (TW(a) * wbc) * recip<FASTR>(fabs(det)) : (TW(a) * wbc) * fabs(det);
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
        pointwise<FORM, DIM, VS, FASTR>(Ji, tw, uq, gq, mu, lam, cv, cg);
#pragma unroll
        for (int comp = 0; comp < VS; ++comp)
#pragma unroll
          for (int d = 0; d < DIM; ++d) g[comp][d][a] = cg[comp][d];
      }
    }

    // ---- transposed chain and scatter, one component at a time ------------
    griddep_wait();   // y zero-filled by the preceding kernel (PDL overwrite path)
    const int32_t* mrow = p.maplex + (int64_t)cell * ND;
    // z^T: pencil (i, j) = e over c: y_k = B^T W1 + D^T W2; scatter      W[c][j][i]
    auto zt_stage = [&](const double* wb, int e, int comp) {
      double w1[Q], w2[Q];
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        w1[c] = wb[c * L::SW + e];
        w2[c] = wb[Q * L::SW + c * L::SW + e];
      }
      if constexpr (EO) {
        double ae[NE], ao[NE], o[P];
        eo_zero(ae, ao);
        eo_adjB(w1, ae, ao);
        eo_adjD(w2, ae, ao);
        eo_merge(ae, ao, o);
#pragma unroll
        for (int k = 0; k < P; ++k) scatter_add(p.y, (int64_t)VS * __ldg(mrow + k * P * P + e) + comp, o[k]);
        return;
      }
#pragma unroll
      for (int k = 0; k < P; ++k) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          s = fma(TB(c, k), w1[c], s);
          s = fma(TD(c, k), w2[c], s);
        }
        scatter_add(p.y, (int64_t)VS * __ldg(mrow + k * P * P + e) + comp, s);
      }
    };
#pragma unroll
    for (int comp = 0; comp < VS; ++comp) {
      if constexpr (DIM == 3) {
        if constexpr (COLLOC) {
          // Dc^T in eta/zeta needs the team's pencils: stage F1, F2     G[a][c][b]
          if (active) {
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              s1[a * QQ + t] = g[comp][1][a];
              s1[Q * QQ + a * QQ + t] = g[comp][2][a];
            }
          }
          team_sync();
          if constexpr (CPEN) {
            // Dc^T along eta by thread (a, c), along zeta by thread (a, b), in place
            if (active) {
              const int a = t % Q, o = t / Q;
              double pen[Q];
#pragma unroll
              for (int e = 0; e < Q; ++e) pen[e] = s1[a * QQ + o * Q + e];
#pragma unroll
              for (int b = 0; b < Q; ++b) {
                double s = 0.0;
#pragma unroll
                for (int e = 0; e < Q; ++e) s = fma(p.Dc[e][b], pen[e], s);
                s1[a * QQ + o * Q + b] = s;
              }
#pragma unroll
              for (int e = 0; e < Q; ++e) pen[e] = s1[Q * QQ + a * QQ + e * Q + o];
#pragma unroll
              for (int c = 0; c < Q; ++c) {
                double s = 0.0;
#pragma unroll
                for (int e = 0; e < Q; ++e) s = fma(p.Dc[e][c], pen[e], s);
                s1[Q * QQ + a * QQ + c * Q + o] = s;
              }
            }
            team_sync();
          }
          // V = Dc^T F0 (local) + Dc^T F1 (eta) + Dc^T F2 (zeta); x^T: A = B^T V
          if (active) {
            const int b = t % Q, c = t / Q;
            double V[Q];
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              double s = 0.0;
#pragma unroll
              for (int e = 0; e < Q; ++e) s = fma(p.Dc[e][a], g[comp][0][e], s);
              if constexpr (CPEN) {
                s += s1[a * QQ + t] + s1[Q * QQ + a * QQ + t];
              } else {
#pragma unroll
                for (int e = 0; e < Q; ++e) {
                  s = fma(p.Dc[e][b], s1[a * QQ + c * Q + e], s);
                  s = fma(p.Dc[e][c], s1[Q * QQ + a * QQ + e * Q + b], s);
                }
              }
              V[a] = s;
            }
#pragma unroll
            for (int i = 0; i < P; ++i) {
              double s = 0.0;
#pragma unroll
              for (int a = 0; a < Q; ++a) s = fma(TB(a, i), V[a], s);
              s2[b * L::SA + c * P + i] = s;                            // A[b][c][i]
            }
          }
          team_sync();
          // y^T: pencil (i, c) over b: W = B^T A                           W[c][j][i]
          if (active && t < Q * P) {
            const int i = t % P, c = t / P;
            double a0[Q];
#pragma unroll
            for (int b = 0; b < Q; ++b) a0[b] = s2[b * L::SA + t];
#pragma unroll
            for (int j = 0; j < P; ++j) {
              double s = 0.0;
#pragma unroll
              for (int b = 0; b < Q; ++b) s = fma(TB(b, j), a0[b], s);
              s1[c * L::SW + j * P + i] = s;
            }
          }
          team_sync();
          // z^T: pencil (i, j) over c: y_k = B^T W; scatter
          if (active && t < P * P) {
            double w1[Q];
#pragma unroll
            for (int c = 0; c < Q; ++c) w1[c] = s1[c * L::SW + t];
#pragma unroll
            for (int k = 0; k < P; ++k) {
              double s = 0.0;
#pragma unroll
              for (int c = 0; c < Q; ++c) s = fma(TB(c, k), w1[c], s);
              scatter_add(p.y, (int64_t)VS * __ldg(mrow + k * P * P + t) + comp, s);
            }
          }
          team_sync();
        } else {
          double* const sw = s1 + (L::FLATZ ? comp * L::WS : 0);   // this component's W region
          // x^T: thread (b, c): A0 = D^T F0, A1 = B^T F1, A2 = B^T F2 over i  A[b][c][i]
          if (active) {
            const int b = t % Q, c = t / Q;
            if constexpr (EO) {
              double ae[NE], ao[NE], o0[P], o1[P], o2[P];
              eo_zero(ae, ao);
              eo_adjD(g[comp][0], ae, ao);
              eo_merge(ae, ao, o0);
              eo_zero(ae, ao);
              eo_adjB(g[comp][1], ae, ao);
              eo_merge(ae, ao, o1);
              eo_zero(ae, ao);
              eo_adjB(g[comp][2], ae, ao);
              eo_merge(ae, ao, o2);
#pragma unroll
              for (int i = 0; i < P; ++i) {
                s2[b * L::SA + c * P + i] = o0[i];
                s2[Q * L::SA + b * L::SA + c * P + i] = o1[i];
                s2[2 * Q * L::SA + b * L::SA + c * P + i] = o2[i];
              }
            } else
#pragma unroll
            for (int i = 0; i < P; ++i) {
              double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
              for (int a = 0; a < Q; ++a) {
                a0 = fma(TD(a, i), g[comp][0][a], a0);
                a1 = fma(TB(a, i), g[comp][1][a], a1);
                a2 = fma(TB(a, i), g[comp][2][a], a2);
              }
              s2[b * L::SA + c * P + i] = a0;
              s2[Q * L::SA + b * L::SA + c * P + i] = a1;
              s2[2 * Q * L::SA + b * L::SA + c * P + i] = a2;
            }
          }
          team_sync();
          // y^T: pencil (i, c) over b: W1 = B^T A0 + D^T A1, W2 = B^T A2    W[c][j][i]
          if (active && t < Q * P) {
            const int i = t % P, c = t / P;
            double a0[Q], a1[Q], a2[Q];
#pragma unroll
            for (int b = 0; b < Q; ++b) {
              a0[b] = s2[b * L::SA + t];
              a1[b] = s2[Q * L::SA + b * L::SA + t];
              a2[b] = s2[2 * Q * L::SA + b * L::SA + t];
            }
            if constexpr (EO) {
              double ae[NE], ao[NE], o1[P], o2[P];
              eo_zero(ae, ao);
              eo_adjB(a0, ae, ao);
              eo_adjD(a1, ae, ao);
              eo_merge(ae, ao, o1);
              eo_zero(ae, ao);
              eo_adjB(a2, ae, ao);
              eo_merge(ae, ao, o2);
#pragma unroll
              for (int j = 0; j < P; ++j) {
                sw[c * L::SW + j * P + i] = o1[j];
                sw[Q * L::SW + c * L::SW + j * P + i] = o2[j];
              }
            } else
#pragma unroll
            for (int j = 0; j < P; ++j) {
              double w1 = 0.0, w2 = 0.0;
#pragma unroll
              for (int b = 0; b < Q; ++b) {
                w1 = fma(TB(b, j), a0[b], w1);
                w1 = fma(TD(b, j), a1[b], w1);
                w2 = fma(TB(b, j), a2[b], w2);
              }
              sw[c * L::SW + j * P + i] = w1;
              sw[Q * L::SW + c * L::SW + j * P + i] = w2;
            }
          }
          team_sync();
          if constexpr (!L::FLATZ) {
            if (active && t < P * P) zt_stage(sw, t, comp);
            team_sync();
          }
        }
      } else {
        if (active) {
          const int b = t;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              a0 = fma(TD(a, i), g[comp][0][a], a0);
              a1 = fma(TB(a, i), g[comp][1][a], a1);
            }
            s2[b * L::S2 + i] = a0;
            s2[Q * L::S2 + b * L::S2 + i] = a1;
          }
        }
        team_sync();
        if (active && t < P) {
          const int i = t;
          double a0[Q], a1[Q];
#pragma unroll
          for (int b = 0; b < Q; ++b) {
            a0[b] = s2[b * L::S2 + i];
            a1[b] = s2[Q * L::S2 + b * L::S2 + i];
          }
#pragma unroll
          for (int j = 0; j < P; ++j) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < Q; ++b) {
              s = fma(TB(b, j), a0[b], s);
              s = fma(TD(b, j), a1[b], s);
            }
            scatter_add(p.y, (int64_t)VS * __ldg(mrow + j * P + i) + comp, s);
          }
        }
        team_sync();
      }
    }
    if constexpr (L::FLATZ) {
#pragma unroll
      for (int r = 0; r < (VS * P * P + TS - 1) / TS; ++r) {
        const int it = t + r * TS;
        if (active && it < VS * P * P) zt_stage(s1 + (it / (P * P)) * L::WS, it % (P * P), it / (P * P));
      }
      team_sync();
    }
    // the next batch's data (loads issued at the top of this iteration)
    if constexpr (ASYNC) {
      cp_wait_group<1>();
    } else {
      park();
    }
    team_sync();
  }
}

}  // namespace fe

#ifndef FE_TK_Q5_MINB
#define FE_TK_Q5_MINB 2      // 256-thread CTAs, 2 per SM, register prefetch: with the even-odd contractions it beats the cp.async gather (0.9165 -> 0.8653 ms, profiles/r02/ab_tensor_eo.txt)
#endif
#ifndef FE_TK_Q6_MINB
#define FE_TK_Q6_MINB 2
#endif
#ifndef FE_TK_Q5C_MINB
#define FE_TK_Q5C_MINB 1002
#endif
#ifndef FE_TK_Q6C_MINB
#define FE_TK_Q6C_MINB 2
#endif
#ifndef FE_TK_EQ2_MINB
#define FE_TK_EQ2_MINB 192   // 192-thread CTAs, 168 registers: C4-hex-Q2 0.504 -> 0.466 ms (profiles/r02/ab_tensor_blocks.txt)
#endif
// registry hook (plan.cu): TV(form, cell, dim, degree, P, Q, MINB[, DIRECT])
#define FE_TENSOR_VARIANTS                                                                   \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 1, 2, 2, 1),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 2, 3, 3, 2),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 3, 4, 4, 2),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 4, 5, 5, 2),                             \
  TVD(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 5, 6, 6, FE_TK_Q5_MINB),                \
  TVD(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 6, 7, 7, FE_TK_Q6_MINB),                \
  TVC(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 5, 6, 6, FE_TK_Q5C_MINB),               \
  TVC(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 6, 7, 7, FE_TK_Q6C_MINB),               \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 1, 2, 3, 1),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 2, 3, 4, 1),                             \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 3, 4, 5, 1),                             \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 1, 2, 3, 2),                              \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 2, 3, 4, FE_TK_EQ2_MINB),                 \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 3, 4, 5, 1),                              \
  TV(FE_FORM_NEOHOOKEAN, FE_CELL_HEXAHEDRON, 3, 1, 2, 3, 1),                                   \
  TV(FE_FORM_NEOHOOKEAN, FE_CELL_HEXAHEDRON, 3, 2, 3, 4, 1),                                   \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 1, 2, 3, 2),                           \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 2, 3, 4, 2),                           \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 3, 4, 5, 2),                           \
  TV(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 4, 5, 6, 2),                           \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 1, 2, 3, 2),                                \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 2, 3, 4, 2),                                \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 3, 4, 5, 2),                                \
  TV(FE_FORM_ELASTICITY, FE_CELL_QUADRILATERAL, 2, 4, 5, 6, 2),                                \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 1, 2, 3, 2),                                 \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 2, 3, 4, 2),                                 \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 3, 4, 5, 2),                                 \
  TV(FE_FORM_LAPLACIAN, FE_CELL_QUADRILATERAL, 2, 4, 5, 6, 2),                                 \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 1, 2, 3, 2),                          \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 2, 3, 4, 2),                          \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 3, 4, 5, 2),                          \
  TV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_QUADRILATERAL, 2, 4, 5, 6, 2),
