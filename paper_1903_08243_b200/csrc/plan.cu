// C ABI (include/fe_b200.h): plans, mesh binding and kernel dispatch.
//
// Plan = everything the reference bakes into one emitted wrap_<form>
// (codegen.py:345-447): the tables, the kernel specialisation for
// (form, cell, degree, rule) -- here chosen from a registry of sm_100a
// template instantiations instead of generated C -- plus the bound mesh in
// the GPU layout (element-batched SoA maps, padded coordinates).
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <omp.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>
#include <type_traits>
#include <utility>

#include "common.cuh"

#ifndef FE_HOST_UCHUNKS
#define FE_HOST_UCHUNKS 8  // u / cell chunks of the host entry
#endif
#include "kern_affine.cuh"
#include "kern_plane.cuh"
#include "kern_plane1.cuh"
#include "kern_pair.cuh"
#include "kern_quad.cuh"
#include "kern_tensor.cuh"
#include "kern_dmma.cuh"
#include "kern_hexq1.cuh"

using namespace fe;

namespace {
thread_local std::string g_err;
std::atomic<long long> g_launches{0};  // operator / diagonal kernel launches (fe_launch_count)
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Set by fe_apply right after it queued the PDL zero-fill of y (overwrite
// applies): the NEXT operator launch on this thread is a programmatic
// dependent of the fill -- its CTAs start while the fill runs, and every
// operator kernel waits (griddep_wait, common.cuh) before its first write
// to y.  Later launches of the same apply are ordinary stream launches.
thread_local bool g_pdl_next = false;

template <typename... KArgs, typename... Args>
void launch_op(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  if (g_pdl_next) {
    g_pdl_next = false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
  } else {
    k<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
  }
  note_launch();
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(FE_ECUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_),     \
                  __FILE__, __LINE__);                                                \
  } while (0)

int cell_dim(int cell) { return (cell == FE_CELL_TRIANGLE || cell == FE_CELL_QUADRILATERAL) ? 2 : 3; }
int cell_nv(int cell) {
  switch (cell) {
    case FE_CELL_TRIANGLE: return 3;
    case FE_CELL_QUADRILATERAL: return 4;
    case FE_CELL_TETRAHEDRON: return 4;
    default: return 8;
  }
}
}  // namespace

struct Variant;

struct fe_plan {
  // element description (scalars copied; tables copied into vectors)
  int form, cell, degree, vs, dim, nv, nd, nq, q1d;
  double params[4];
  std::vector<double> qw, phi, dphi, gphi, gdphi, B1d, D1d, w1d, x1d, qw_aux, dphi_aux;
  std::vector<int32_t> lex;
  const Variant* var = nullptr;
  uint32_t flags = 0;
  // device tables (kernel-family specific layout)
  double* d_tables = nullptr;
  size_t tables_bytes = 0;
  double* d_diag_tables = nullptr;  // generic quadrature tables of fe_diagonal (lazy)
  size_t diag_tables_bytes = 0;
  int persistent_ctas = 0;
  int dmma_cfg = 0;
  int cells_per_block = 0;
  void* host_params = nullptr;  // by-value kernel parameter block (element-tensor kernels)
  size_t host_params_bytes = 0;
  // bound mesh
  int32_t ncells = 0, nverts = 0;
  int64_t nglobal = 0;
  int64_t stride = 0;
  int32_t* d_map = nullptr;     // SoA [nd][stride]
  int32_t* d_vmap = nullptr;    // SoA [nv][stride] or == d_map
  int32_t* d_map_rm = nullptr;  // row-major [ncells][nd] copy
  int32_t* d_map_lex = nullptr; // row-major, tensor (lexicographic) local order (tensor kernels)
  int32_t* d_lex = nullptr;     // [nd] local node of tensor node
  // patches (CTA-level dof aggregation, kern_affine.cuh)
  bool wants_patch = false;
  int32_t* d_patch_off = nullptr;
  int32_t* d_patch_dofs = nullptr;
  uint16_t* d_pidx = nullptr;
  int patch_maxu = 0;
  // macro-cells (kern_affine.cuh macro_split_kernel): pattern requested by
  // the kernel family, SoA [NU][macro_stride] dofs of the verified mesh
  std::vector<int32_t> macro_pat;  // [MC][ND] local macro-dof of each cell dof
  int macro_mc = 0, macro_nu = 0;
  int32_t* d_macro = nullptr;
  int64_t macro_stride = 0;
  bool p1_analytic = false;  // tables verified equal to the compile-time P1 constants
  double* d_coords = nullptr;   // padded [nverts][cstride]
  const void* b_coords = nullptr;
  const void* b_map0 = nullptr;
  const void* b_map1 = nullptr;
  uint32_t b_flags = 0;
  bool auto_bound = false;      // bound implicitly by fe_wrap/fe_wrap_host (cells [0, end) of that call)
  // host-entry staging
  cudaStream_t hstream = nullptr;
  cudaStream_t hstream2 = nullptr;
  cudaEvent_t ev_u = nullptr, ev_y0 = nullptr;
  cudaEvent_t ev_uc[32] = {};   // per-chunk completion of the u upload (host entry)
  cudaStream_t hstream_u = nullptr;
  cudaStream_t hstream_d = nullptr;  // result downloads (host entry)
  cudaEvent_t ev_cell[32] = {};       // completion of each cell chunk (host entry)
  // host entry pipelining: cell chunks (FE_HOST_UCHUNKS, boundaries aligned
  // to 192 cells) and, per chunk, the mask of the 64 blocks (hblock entries
  // each) of the u / y vector its cells read and scatter into (computed at
  // bind): u is uploaded block by block in the order the cell chunks need it,
  // and a block of y is downloaded as soon as the last cell chunk touching it
  // is done -- for any dof numbering (vertex dofs first, lexicographic, ...)
  std::vector<int32_t> chunk_cell;
  std::vector<uint64_t> chunk_mask;
  int64_t hblock = 0;
  // two-phase overwrite apply (fe_apply): the zero-fill of the blocks of y the
  // first cell chunk scatters into runs first, the rest of the fill runs on a
  // side stream underneath that chunk's arithmetic
  cudaStream_t fill_stream = nullptr;
  cudaEvent_t ev_fill_a = nullptr, ev_fill_b = nullptr;
  std::mutex fill_mutex;
  double* d_u = nullptr;
  double* d_y = nullptr;
  double* d_y0 = nullptr;
  double* d_c0 = nullptr;
  double* d_c1 = nullptr;
  size_t cap_u = 0, cap_c = 0;
};

typedef int (*PrepareFn)(fe_plan*);
typedef int (*LaunchFn)(const fe_plan*, int32_t, int32_t, double*, const double*, const double*,
                        const double*, cudaStream_t);

typedef int (*DiagFn)(const fe_plan*, int32_t, int32_t, double*, const double*, const double*,
                      cudaStream_t);

struct Variant {
  int form, cell, degree, nq;  // nq = -1: any rule accepted by the prepare step
  int priority;                // higher wins
  const char* name;
  int block;
  PrepareFn prepare;
  LaunchFn launch;
  DiagFn diag = nullptr;       // operator diagonal (generic quadrature entries only)
};

// ---------------------------------------------------------------------------
// generic quadrature kernel
// ---------------------------------------------------------------------------

template <int FORM, int DIM, int NV, int ND, int NQ, bool AFFINE>
int quad_prepare(fe_plan* p) {
  using TB = QuadTables<NQ, ND, NV, DIM>;
  std::vector<double> t(TB::size);
  std::copy(p->qw.begin(), p->qw.end(), t.begin() + TB::qw);
  std::copy(p->phi.begin(), p->phi.end(), t.begin() + TB::phi);
  std::copy(p->dphi.begin(), p->dphi.end(), t.begin() + TB::dphi);
  std::copy(p->gphi.begin(), p->gphi.end(), t.begin() + TB::gphi);
  std::copy(p->gdphi.begin(), p->gdphi.end(), t.begin() + TB::gdphi);
  p->tables_bytes = t.size() * sizeof(double);
  CUDA_TRY(cudaMalloc(&p->d_tables, p->tables_bytes));
  CUDA_TRY(cudaMemcpy(p->d_tables, t.data(), p->tables_bytes, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaFuncSetAttribute(quad_kernel<FORM, DIM, NV, ND, NQ, AFFINE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)p->tables_bytes));
  return FE_OK;
}

MeshView mesh_view(const fe_plan* p) {
  MeshView m;
  m.map = p->d_map;
  m.vmap = p->d_vmap;
  m.coords = p->d_coords;
  m.nc_stride = p->stride;
  return m;
}

template <int FORM, int DIM, int NV, int ND, int NQ, bool AFFINE>
int quad_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                const double* c0, const double* c1, cudaStream_t s) {
  QuadParams k;
  k.mesh = mesh_view(p);
  k.start = start;
  k.end = end;
  k.u = u;
  k.y = y;
  k.mu = c0;
  k.lam = c1;
  k.tables = p->d_tables;
  k.p0 = p->params[0];
  k.p1 = p->params[1];
  int n = end - start;
  launch_op(quad_kernel<FORM, DIM, NV, ND, NQ, AFFINE>, (n + 127) / 128, 128, p->tables_bytes, s, k);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// operator diagonal: the generic tables, uploaded on first use
template <int FORM, int DIM, int NV, int ND, int NQ, bool AFFINE>
int quad_diag(const fe_plan* cp, int32_t start, int32_t end, double* y, const double* c0,
              const double* c1, cudaStream_t s) {
  if constexpr (FORM == FE_FORM_NEOHOOKEAN) {
    return fail(FE_EUNSUPPORTED, "the neohookean residual is nonlinear: no operator diagonal");
  } else {
    fe_plan* p = const_cast<fe_plan*>(cp);
    using TB = QuadTables<NQ, ND, NV, DIM>;
    if (!p->d_diag_tables) {
      std::vector<double> t(TB::size);
      std::copy(p->qw.begin(), p->qw.end(), t.begin() + TB::qw);
      std::copy(p->phi.begin(), p->phi.end(), t.begin() + TB::phi);
      std::copy(p->dphi.begin(), p->dphi.end(), t.begin() + TB::dphi);
      std::copy(p->gphi.begin(), p->gphi.end(), t.begin() + TB::gphi);
      std::copy(p->gdphi.begin(), p->gdphi.end(), t.begin() + TB::gdphi);
      p->diag_tables_bytes = t.size() * sizeof(double);
      CUDA_TRY(cudaMalloc(&p->d_diag_tables, p->diag_tables_bytes));
      CUDA_TRY(cudaMemcpy(p->d_diag_tables, t.data(), p->diag_tables_bytes, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaFuncSetAttribute(quad_diag_kernel<FORM, DIM, NV, ND, NQ, AFFINE>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)p->diag_tables_bytes));
    }
    QuadParams k;
    k.mesh = mesh_view(p);
    k.start = start;
    k.end = end;
    k.u = nullptr;
    k.y = y;
    k.mu = c0;
    k.lam = c1;
    k.tables = p->d_diag_tables;
    k.p0 = p->params[0];
    k.p1 = p->params[1];
    const int n = end - start;
    launch_op(quad_diag_kernel<FORM, DIM, NV, ND, NQ, AFFINE>, (n + 127) / 128, 128, p->diag_tables_bytes, s, k);
    CUDA_TRY(cudaGetLastError());
    return FE_OK;
  }
}

// ---------------------------------------------------------------------------
// quadrature kernel with tables in the parameter block (affine simplices)
// ---------------------------------------------------------------------------

template <int FORM, int DIM, int NV, int ND, int NQ, bool AFF, int MINB = 1, int UNR = 1>
int qc_prepare(fe_plan* p) {
  using P = QuadConstParams<NQ, ND, DIM, NV, form_needs_values(FORM), AFF>;
  static_assert(sizeof(P) <= 32000, "parameter block too large");
  if (p->nq != NQ || p->nd != ND || p->nv != NV) return fail(FE_EINVAL, "quad_const table size mismatch");
  P* hp = new P();
  for (int q = 0; q < NQ; ++q) {
    hp->qw[q] = p->qw[q];
    for (int i = 0; i < ND; ++i) {
      if constexpr (form_needs_values(FORM)) hp->phi[q][i] = p->phi[q * ND + i];
      for (int b = 0; b < DIM; ++b) hp->dphi[q][i][b] = p->dphi[((size_t)q * ND + i) * DIM + b];
    }
    for (int v = 0; v < NV; ++v) {
      hp->gphi[q][v] = p->gphi[q * NV + v];
    }
    if constexpr (!AFF) {
      // tensor rule, x slowest (elements.py:193-198): q = (ix * Q + iy) * Q + iz
      const int Q1 = p->q1d;
      if (Q1 <= 0) return fail(FE_EINVAL, "tensor quad_const plan needs the 1D rule");
      int rem = q;
      for (int b = DIM - 1; b >= 0; --b) {
        hp->px[q][b] = p->x1d[rem % Q1];
        rem /= Q1;
      }
    }
  }
  p->host_params = hp;
  p->host_params_bytes = sizeof(P);
  return FE_OK;
}

template <int FORM, int DIM, int NV, int ND, int NQ, bool AFF, int MINB = 1, int UNR = 1>
int qc_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
              const double* c0, const double* c1, cudaStream_t s) {
  using P = QuadConstParams<NQ, ND, DIM, NV, form_needs_values(FORM), AFF>;
  P hpv = *static_cast<const P*>(p->host_params);  // per-launch copy: concurrent launches on one plan stay independent
  P* hp = &hpv;
  hp->mesh = mesh_view(p);
  hp->start = start;
  hp->end = end;
  hp->u = u;
  hp->y = y;
  hp->mu = c0;
  hp->lam = c1;
  hp->p0 = p->params[0];
  hp->p1 = p->params[1];
  const int n = end - start;
  launch_op(quad_const_kernel<FORM, DIM, NV, ND, NQ, AFF, MINB, UNR>, (n + 127) / 128, 128, 0, s, *hp);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// vertex-gradient P2 kernel (kern_quad.cuh quad_vtx_kernel): the reference
// gradients of the P2 basis at the simplex vertices, recovered exactly from
// the point tables (they are P1: dphi[q] = sum_v gphi[q][v] dphiv[v]) by a
// least-squares solve of the NV x NV normal equations
template <int FORM, int DIM, int NV, int ND, int NQ, int MINB, int UNR>
int vtx_prepare(fe_plan* p) {
  using P = VtxParams<NQ, ND, DIM, NV>;
  static_assert(sizeof(P) <= 32000, "parameter block too large");
  if (p->nq != NQ || p->nd != ND || p->nv != NV) return fail(FE_EINVAL, "vertex-gradient table size mismatch");
  P* hp = new P();
  double Mn[NV][NV] = {};
  for (int q = 0; q < NQ; ++q) {
    hp->qw[q] = p->qw[q];
    for (int v = 0; v < NV; ++v) {
      hp->gphi[q][v] = p->gphi[q * NV + v];
      for (int v2 = 0; v2 < NV; ++v2) Mn[v][v2] += p->gphi[q * NV + v] * p->gphi[q * NV + v2];
    }
  }
  // Gauss-Jordan inverse of the (SPD, well-conditioned) normal matrix
  double inv[NV][NV] = {};
  for (int v = 0; v < NV; ++v) inv[v][v] = 1.0;
  for (int c = 0; c < NV; ++c) {
    const double piv = Mn[c][c];
    if (!(std::fabs(piv) > 1e-12)) { delete hp; return fail(FE_EINVAL, "singular vertex projection"); }
    for (int k = 0; k < NV; ++k) { Mn[c][k] /= piv; inv[c][k] /= piv; }
    for (int r = 0; r < NV; ++r)
      if (r != c) {
        const double f = Mn[r][c];
        for (int k = 0; k < NV; ++k) { Mn[r][k] -= f * Mn[c][k]; inv[r][k] -= f * inv[c][k]; }
      }
  }
  double worst = 0.0;
  for (int i = 0; i < ND; ++i)
    for (int b = 0; b < DIM; ++b) {
      double rhs[NV] = {};
      for (int q = 0; q < NQ; ++q)
        for (int v = 0; v < NV; ++v) rhs[v] += p->gphi[q * NV + v] * p->dphi[((size_t)q * ND + i) * DIM + b];
      for (int v = 0; v < NV; ++v) {
        double s = 0.0;
        for (int k = 0; k < NV; ++k) s += inv[v][k] * rhs[k];
        hp->dphiv[v][i][b] = s;
      }
      for (int q = 0; q < NQ; ++q) {  // the gradient must be exactly P1
        double s = 0.0;
        for (int v = 0; v < NV; ++v) s += p->gphi[q * NV + v] * hp->dphiv[v][i][b];
        worst = std::max(worst, std::fabs(s - p->dphi[((size_t)q * ND + i) * DIM + b]));
      }
    }
  if (worst > 1e-12) {
    delete hp;
    return fail(FE_EUNSUPPORTED, "basis gradients are not P1 (residual %.1e)", worst);
  }
  p->host_params = hp;
  p->host_params_bytes = sizeof(P);
  return FE_OK;
}

template <int FORM, int DIM, int NV, int ND, int NQ, int MINB, int UNR>
int vtx_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
               const double* c0, const double*, cudaStream_t s) {
  using P = VtxParams<NQ, ND, DIM, NV>;
  P hpv = *static_cast<const P*>(p->host_params);
  P* hp = &hpv;
  hp->mesh = mesh_view(p);
  hp->start = start;
  hp->end = end;
  hp->u = u;
  hp->y = y;
  hp->mu = c0;  // the state u0 of a linearised form
  hp->lam = nullptr;
  hp->p0 = p->params[0];
  hp->p1 = p->params[1];
  const int n = end - start;
  launch_op(quad_vtx_kernel<FORM, DIM, NV, ND, NQ, MINB, UNR>, (n + 127) / 128, 128, 0, s, *hp);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// ---------------------------------------------------------------------------
// element-tensor kernel (affine simplices)
// ---------------------------------------------------------------------------

// Reference matrices from the plan's quadrature tables (exact for the
// polynomial integrands of affine cells).
static void element_matrices(const fe_plan* p, bool mass, bool grads, std::vector<double>& S) {
  const int nd = p->nd, nq = p->nq, d = p->dim;
  S.clear();
  auto push = [&](auto f) {
    for (int i = 0; i < nd; ++i)
      for (int j = 0; j < nd; ++j) {
        double s = 0.0;
        for (int q = 0; q < nq; ++q) s += p->qw[q] * f(q, i, j);
        S.push_back(s);
      }
  };
  auto dp = [&](int q, int i, int a) { return p->dphi[((size_t)q * nd + i) * d + a]; };
  if (mass) push([&](int q, int i, int j) { return p->phi[q * nd + i] * p->phi[q * nd + j]; });
  if (grads) {
    for (int a = 0; a < d; ++a) push([&](int q, int i, int j) { return dp(q, i, a) * dp(q, j, a); });
    for (int a = 0; a < d; ++a)
      for (int b = a + 1; b < d; ++b)
        push([&](int q, int i, int j) { return dp(q, i, a) * dp(q, j, b) + dp(q, i, b) * dp(q, j, a); });
  }
}

// cells per thread of the affine kernels (group_scatter, kern_affine.cuh),
// per measurement (profiles/r01/sweep_group.txt: C2-P1 40 -> 34 us at G = 2;
// larger groups and every P2 grouping are slower -- registers and latency)
#ifndef FE_GROUP_TET_P1
#define FE_GROUP_TET_P1 2
#endif
#ifndef FE_GROUP_TET_P2
#define FE_GROUP_TET_P2 1
#endif
#ifndef FE_GROUP_TRI_P2
#define FE_GROUP_TRI_P2 1
#endif
// macro-cell of the P1 tet kernel: cubes per thread along x (measured,
// profiles/r01/sweep_p1const.txt)
#ifndef FE_MACRO_NCX
#define FE_MACRO_NCX 1
#endif
using MacroP1 = std::conditional_t<FE_MACRO_NCX == 1, KuhnTetP1, KuhnTetRowP1<FE_MACRO_NCX>>;
template <int ND>
using MacroFor = std::conditional_t<ND == 4, MacroP1, KuhnTetP2>;
#ifndef FE_MACRO_WAVES_DEFAULT
#define FE_MACRO_WAVES_DEFAULT 1
#endif

constexpr int affine_group(int dim, int nd) {
  return dim == 3 ? (nd == 4 ? FE_GROUP_TET_P1 : nd == 10 ? FE_GROUP_TET_P2 : 1)
                  : (nd == 6 ? FE_GROUP_TRI_P2 : 1);
}

template <int FORM, int DIM, int ND>
int et_prepare(fe_plan* p) {
  constexpr int NM = et_nmats<FORM, DIM>();
  using P = ETParams<NM, ND>;
  static_assert(sizeof(P) <= 32000, "parameter block too large");
  std::vector<double> S;
  element_matrices(p, FORM != FE_FORM_LAPLACIAN_SCALAR, FORM != FE_FORM_MASS, S);
  if ((int)S.size() != NM * ND * ND) return fail(FE_EINVAL, "element-tensor table size mismatch");
  P* hp = new P();
  std::memcpy(hp->S, S.data(), S.size() * sizeof(double));
  p->host_params = hp;
  p->host_params_bytes = sizeof(P);
  return FE_OK;
}

template <int FORM, int DIM, int ND>
int et_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
              const double*, const double*, cudaStream_t s) {
  constexpr int NM = et_nmats<FORM, DIM>();
  using P = ETParams<NM, ND>;
  P hpv = *static_cast<const P*>(p->host_params);
  P* hp = &hpv;
  hp->mesh = mesh_view(p);
  hp->u = u;
  hp->y = y;
  hp->start = start;
  hp->end = end;
  int n = end - start;
  constexpr int G = affine_group(DIM, ND);
  const int nt = (n + G - 1) / G;
  launch_op(affine_et_kernel<FORM, DIM, ND, G>, (nt + 127) / 128, 128, 0, s, *hp);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

template <int FORM, int DIM, int ND>
int etp_prepare(fe_plan* p) {
  constexpr int NM = et_nmats<FORM, DIM>();
  using P = ETPatchParams<NM, ND>;
  static_assert(sizeof(P) <= 32000, "parameter block too large");
  std::vector<double> S;
  element_matrices(p, FORM != FE_FORM_LAPLACIAN_SCALAR, FORM != FE_FORM_MASS, S);
  if ((int)S.size() != NM * ND * ND) return fail(FE_EINVAL, "element-tensor table size mismatch");
  P* hp = new P();
  std::memcpy(hp->S, S.data(), S.size() * sizeof(double));
  p->host_params = hp;
  p->host_params_bytes = sizeof(P);
  p->wants_patch = true;
  return FE_OK;
}

template <int FORM, int DIM, int ND>
int etp_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
               const double*, const double*, cudaStream_t s) {
  constexpr int NM = et_nmats<FORM, DIM>();
  using P = ETPatchParams<NM, ND>;
  if (!p->d_patch_off) return fail(FE_ENOMESH, "patch plan without patches");
  P hpv = *static_cast<const P*>(p->host_params);
  P* hp = &hpv;
  hp->mesh = mesh_view(p);
  hp->patch.off = p->d_patch_off;
  hp->patch.dofs = p->d_patch_dofs;
  hp->patch.pidx = p->d_pidx;
  hp->u = u;
  hp->y = y;
  hp->start = start;
  hp->end = end;
  const int b0 = start / kPatchCells, b1 = (end - 1) / kPatchCells;
  const size_t smem = 2 * (size_t)p->patch_maxu * sizeof(double);
  launch_op(affine_et_patch_kernel<FORM, DIM, ND>, b1 - b0 + 1, kPatchCells, smem, s, *hp);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

template <int FORM, int DIM, int ND, int NQS>
int split_prepare(fe_plan* p) {
  using P = SplitParams<NQS, ND, DIM>;
  static_assert(sizeof(P) <= 32000, "parameter block too large");
  if ((int)p->qw_aux.size() != NQS) return fail(FE_EUNSUPPORTED, "split kernel needs %d stiffness modes", NQS);
  for (double w : p->qw_aux)
    if (w != 1.0) return fail(FE_EUNSUPPORTED, "split kernel takes unit-weight stiffness modes");
  std::vector<double> S;
  element_matrices(p, true, false, S);  // reference mass matrix
  P* hp = new P();
  for (int q = 0; q < NQS; ++q) {
    hp->qw[q] = p->qw_aux[q];
    for (int i = 0; i < ND; ++i)
      for (int b = 0; b < DIM; ++b) hp->dphi[q][i][b] = p->dphi_aux[((size_t)q * ND + i) * DIM + b];
  }
  std::memcpy(hp->M, S.data(), sizeof(hp->M));
  p->host_params = hp;
  p->host_params_bytes = sizeof(P);
  if (DIM + 1 == ND && NQS == 1 && !getenv("FE_NO_P1CONST")) {
    // P1: the plan's tables must equal the constants p1_simplex_compute bakes in
    const double vref = DIM == 3 ? 1.0 / 6.0 : 0.5, cmass = DIM == 3 ? 1.0 / 120.0 : 1.0 / 24.0;
    auto gref = [](int i, int b) { return i == 0 ? -1.0 : (i == b + 1 ? 1.0 : 0.0); };
    bool ok = true;
    for (int i = 0; i < ND; ++i)
      for (int j = 0; j < ND; ++j) {
        if (std::fabs(hp->M[i][j] - cmass * (i == j ? 2.0 : 1.0)) > 1e-15) ok = false;
        for (int a = 0; a < DIM; ++a)
          for (int b = 0; b < DIM; ++b) {
            const double s = hp->qw[0] * hp->dphi[0][i][a] * hp->dphi[0][j][b];
            if (std::fabs(s - vref * gref(i, a) * gref(j, b)) > 1e-14) ok = false;
          }
      }
    p->p1_analytic = ok;
  }
  if constexpr (DIM == 3 && (ND == 4 || ND == 10)) {
    if (!getenv("FE_NO_MACRO") && (ND == 4 || getenv("FE_MACRO_P2"))) {
      using PAT = MacroFor<ND>;
      p->macro_mc = PAT::MC;
      p->macro_nu = PAT::NU;
      p->macro_pat.clear();
      for (int t = 0; t < PAT::MC; ++t)
        for (int i = 0; i < PAT::ND; ++i) p->macro_pat.push_back(PAT::at(t, i));
    }
  }
  return FE_OK;
}

template <int FORM, int DIM, int ND, int NQS>
int split_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                 const double*, const double*, cudaStream_t s) {
  using P = SplitParams<NQS, ND, DIM>;
  P hpv = *static_cast<const P*>(p->host_params);
  P* hp = &hpv;
  hp->mesh = mesh_view(p);
  hp->u = u;
  hp->y = y;
  hp->start = start;
  hp->end = end;
  constexpr int G = affine_group(DIM, ND);
  auto per_cell = [&](int32_t a, int32_t b) {
    if (a >= b) return;
    hp->start = a;
    hp->end = b;
    const int nt = (b - a + G - 1) / G;
    launch_op(affine_split_kernel<FORM, DIM, ND, NQS, G>, (nt + 127) / 128, 128, 0, s, *hp);
  };
  if constexpr (DIM == 3 && (ND == 4 || ND == 10)) {
    using PAT = MacroFor<ND>;
    if (p->d_macro) {
      // whole macro-cells inside [start, end) on the macro kernel, ragged ends per cell
      const int mc = PAT::MC;
      const int32_t m0 = (start + mc - 1) / mc, m1 = end / mc;
      if (m0 < m1) {
        // persistent grid: FE_MACRO_WAVES resident waves of CTAs (0 = one thread per macro-cell)
        static const int waves = getenv("FE_MACRO_WAVES") ? atoi(getenv("FE_MACRO_WAVES")) : FE_MACRO_WAVES_DEFAULT;
        int nb = (m1 - m0 + 127) / 128;
        auto launch = [&](auto kfn) {
          if (waves > 0) {
            int dev = 0, sms = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 128, 0);
            nb = std::min(nb, std::max(1, waves * sms * per_sm));
          }
          launch_op(kfn, nb, 128, 0, s, *hp, p->d_macro, p->macro_stride, m0, m1);
        };
        if constexpr (ND == 4) {
          // opt-in (FE_MACRO_PIPE=1): measured slower, 23.5 vs 19.5 us (profiles/r02/ab_macro_pipe.txt)
          static const bool pipe = getenv("FE_MACRO_PIPE") != nullptr;
          if (p->p1_analytic && pipe && waves > 0) {
            // cp.async-pipelined macro kernel: thread-private shared-memory columns, 2 buffers
            auto kfn = macro_pipe_kernel<FORM, DIM, ND, PAT>;
            constexpr size_t smem = 2 * (size_t)PAT::NU * (DIM + 1) * 128 * sizeof(double);
            static bool attr_done = false;
            if (!attr_done) {
              CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
              attr_done = true;
            }
            int dev = 0, sms = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 128, smem);
            nb = std::min(nb, std::max(1, waves * sms * per_sm));
            launch_op(kfn, nb, 128, smem, s, *hp, p->d_macro, p->macro_stride, m0, m1);
          } else if (p->p1_analytic)
            launch(macro_split_kernel<FORM, DIM, ND, NQS, PAT, true>);
          else
            launch(macro_split_kernel<FORM, DIM, ND, NQS, PAT>);
        } else {
          launch(macro_split_kernel<FORM, DIM, ND, NQS, PAT>);
        }
        per_cell(start, m0 * mc);
        per_cell(m1 * mc, end);
        CUDA_TRY(cudaGetLastError());
        return FE_OK;
      }
    }
  }
  per_cell(start, end);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// ---------------------------------------------------------------------------
// DMMA element-tensor kernel (high-degree affine simplices)
// ---------------------------------------------------------------------------

constexpr int kDmmaBlock = 256;

// (NT, MINB) configurations of the DMMA kernel: 0 = (2,1), 1 = (1,2),
// 2 = (2,2), 3 = (1,1); FE_DMMA_CFG selects one for experiments, the
// default is the measured best.

template <int FORM, int DIM, int ND, int NT, int MINB>
int dmma_setup(fe_plan* p) {
  CUDA_TRY(cudaFuncSetAttribute(dmma_et_kernel<FORM, DIM, ND, NT, MINB>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tables_bytes));
  int dev = 0, sms = 0, per_sm = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, dmma_et_kernel<FORM, DIM, ND, NT, MINB>, kDmmaBlock, p->tables_bytes));
  p->persistent_ctas = sms * (per_sm > 0 ? per_sm : 1);
  return FE_OK;
}

template <int FORM, int DIM, int ND>
int dmma_prepare(fe_plan* p) {
  constexpr int NM = et_nmats<FORM, DIM>();
  constexpr int KT = DmmaShape<ND>::KT, MT = DmmaShape<ND>::MT;
  std::vector<double> S;
  element_matrices(p, FORM != FE_FORM_LAPLACIAN_SCALAR, FORM != FE_FORM_MASS, S);
  if ((int)S.size() != NM * ND * ND) return fail(FE_EINVAL, "DMMA table size mismatch");
  std::vector<double> A((size_t)NM * KT * MT * 32, 0.0);
  for (int m = 0; m < NM; ++m)
    for (int kk = 0; kk < KT; ++kk)
      for (int mt = 0; mt < MT; ++mt)
        for (int lane = 0; lane < 32; ++lane) {
          int row = 8 * mt + (lane >> 2), col = 4 * kk + (lane & 3);
          if (row < ND && col < ND)
            A[(((size_t)m * KT + kk) * MT + mt) * 32 + lane] = S[((size_t)m * ND + row) * ND + col];
        }
  p->tables_bytes = A.size() * sizeof(double);
  CUDA_TRY(cudaMalloc(&p->d_tables, p->tables_bytes));
  CUDA_TRY(cudaMemcpy(p->d_tables, A.data(), p->tables_bytes, cudaMemcpyHostToDevice));
  const char* env = getenv("FE_DMMA_CFG");
  // measured with the map prefetch (profiles/r01/dmma_cfg_v3.txt): 1 n-tile
  // per warp x 2 CTAs/SM is best (P4 71.7%, P3 62.3% of the FP64 roof)
  p->dmma_cfg = env ? atoi(env) : 1;
  if (p->dmma_cfg < 0 || p->dmma_cfg > 3) p->dmma_cfg = 0;
  switch (p->dmma_cfg) {
    case 1: return dmma_setup<FORM, DIM, ND, 1, 2>(p);
    case 2: return dmma_setup<FORM, DIM, ND, 2, 2>(p);
    case 3: return dmma_setup<FORM, DIM, ND, 1, 1>(p);
    default: return dmma_setup<FORM, DIM, ND, 2, 1>(p);
  }
}

template <int FORM, int DIM, int ND, int NT, int MINB>
int dmma_run(const fe_plan* p, const DmmaParams& k, int32_t n, cudaStream_t s) {
  const int ngroups = (n + 8 * NT - 1) / (8 * NT);
  const int need = (ngroups + kDmmaBlock / 32 - 1) / (kDmmaBlock / 32);
  const int grid = need < p->persistent_ctas ? need : p->persistent_ctas;
  launch_op(dmma_et_kernel<FORM, DIM, ND, NT, MINB>, grid, kDmmaBlock, p->tables_bytes, s, k);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

template <int FORM, int DIM, int ND>
int dmma_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                const double*, const double*, cudaStream_t s) {
  DmmaParams k;
  k.mesh = mesh_view(p);
  k.u = u;
  k.y = y;
  k.afrag = p->d_tables;
  k.start = start;
  k.end = end;
  switch (p->dmma_cfg) {
    case 1: return dmma_run<FORM, DIM, ND, 1, 2>(p, k, end - start, s);
    case 2: return dmma_run<FORM, DIM, ND, 2, 2>(p, k, end - start, s);
    case 3: return dmma_run<FORM, DIM, ND, 1, 1>(p, k, end - start, s);
    default: return dmma_run<FORM, DIM, ND, 2, 1>(p, k, end - start, s);
  }
}

// modal two-stage DMMA kernel (kern_dmma.cuh): fragment-ordered G (stage 1,
// B operand) and [G^T | Mhat] (stage 2, A operand) from the plan's stiffness
// modes (qw_aux / dphi_aux, elements.stiffness_modes) and mass matrix.
// (NT, MINB, BLK) configurations of the modal kernel (FE_DMMA_CFG):
// 0 = (2,1,256) 1 = (1,2,256) 2 = (2,2,256) 3 = (1,1,256) 4 = (1,5,128)
// 5 = (1,6,128) 6 = (1,3,256)
#define FE_MODAL_CFGS(F)                                                          \
  switch (p->dmma_cfg) {                                                          \
    case 1: return F(1, 2, 256);                                                  \
    case 2: return F(2, 2, 256);                                                  \
    case 3: return F(1, 1, 256);                                                  \
    case 4: return F(1, 5, 128);                                                  \
    case 5: return F(1, 6, 128);                                                  \
    case 6: return F(1, 3, 256);                                                  \
    default: return F(2, 1, 256);                                                 \
  }

template <int FORM, int DIM, int ND, int NMODE, int NT, int MINB, int BLK>
int dmma_modal_setup(fe_plan* p) {
  auto kfn = dmma_modal_kernel<FORM, DIM, ND, NMODE, NT, MINB, BLK>;
  CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tables_bytes));
  int dev = 0, sms = 0, per_sm = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, BLK, p->tables_bytes));
  p->persistent_ctas = sms * (per_sm > 0 ? per_sm : 1);
  return FE_OK;
}

template <int FORM, int DIM, int ND, int NMODE>
int dmma_modal_prepare(fe_plan* p) {
  constexpr bool MASS = FORM == FE_FORM_HELMHOLTZ;
  constexpr int KT = DmmaShape<ND>::KT, MT = DmmaShape<ND>::MT;
  using MS = ModalShape<DIM, NMODE>;
  constexpr int NJ = MS::NJ, TPL = MS::TPL, NSTEP = MS::NSTEP;
  constexpr int S2 = NSTEP + (MASS ? KT : 0);
  if ((int)p->qw_aux.size() != NMODE) return fail(FE_EUNSUPPORTED, "modal kernel needs %d stiffness modes", NMODE);
  for (double w : p->qw_aux)
    if (!(w >= 0.0)) return fail(FE_EINVAL, "stiffness modes need non-negative weights");
  // G[r][i][a] = sqrt(w_r) dphi_aux[r][i][a]; column (lane-group c, slot li)
  // holds mode MS::mode_of(c, li), direction MS::dir_of(c, li)
  auto G = [&](int c, int li, int dof) -> double {
    const int r = MS::mode_of(c, li), a = MS::dir_of(c, li);
    if (r < 0 || r >= NMODE || dof >= ND) return 0.0;
    return std::sqrt(p->qw_aux[r]) * p->dphi_aux[((size_t)r * ND + dof) * DIM + a];
  };
  std::vector<double> S;
  if (MASS) element_matrices(p, true, false, S);
  std::vector<double> T((size_t)(NJ * KT + S2 * MT) * 32, 0.0);
  for (int j = 0; j < NJ; ++j)
    for (int t = 0; t < KT; ++t)
      for (int lane = 0; lane < 32; ++lane) {
        const int n = lane >> 2, k = 4 * t + (lane & 3);  // B[k][n], column 8j + n
        T[((size_t)j * KT + t) * 32 + lane] = G(n >> 1, 2 * j + (n & 1), k);
      }
  double* A2 = T.data() + (size_t)NJ * KT * 32;
  for (int s = 0; s < S2; ++s)
    for (int mt = 0; mt < MT; ++mt)
      for (int lane = 0; lane < 32; ++lane) {
        const int row = 8 * mt + (lane >> 2), c = lane & 3;  // A[row][k = c]
        double v = 0.0;
        if (s < NSTEP) {
          v = G(c, s, row);
        } else {
          const int col = 4 * (s - NSTEP) + c;
          if (row < ND && col < ND) v = S[(size_t)row * ND + col];
        }
        A2[((size_t)s * MT + mt) * 32 + lane] = v;
      }
  p->tables_bytes = T.size() * sizeof(double);
  CUDA_TRY(cudaMalloc(&p->d_tables, p->tables_bytes));
  CUDA_TRY(cudaMemcpy(p->d_tables, T.data(), p->tables_bytes, cudaMemcpyHostToDevice));
  const char* env = getenv("FE_DMMA_CFG");
  p->dmma_cfg = env ? atoi(env) : 1;
  if (p->dmma_cfg < 0 || p->dmma_cfg > 6) p->dmma_cfg = 0;
#define FE_SETUP(NT, MINB, BLK) dmma_modal_setup<FORM, DIM, ND, NMODE, NT, MINB, BLK>(p)
  FE_MODAL_CFGS(FE_SETUP)
#undef FE_SETUP
}

template <int FORM, int DIM, int ND, int NMODE, int NT, int MINB, int BLK>
int dmma_modal_run(const fe_plan* p, const DmmaParams& k, int32_t n, cudaStream_t s) {
  const int ngroups = (n + 8 * NT - 1) / (8 * NT);
  const int need = (ngroups + BLK / 32 - 1) / (BLK / 32);
  const int grid = need < p->persistent_ctas ? need : p->persistent_ctas;
  launch_op(dmma_modal_kernel<FORM, DIM, ND, NMODE, NT, MINB, BLK>, grid, BLK, p->tables_bytes, s, k);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

template <int FORM, int DIM, int ND, int NMODE>
int dmma_modal_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                      const double*, const double*, cudaStream_t s) {
  DmmaParams k;
  k.mesh = mesh_view(p);
  k.u = u;
  k.y = y;
  k.afrag = p->d_tables;
  k.start = start;
  k.end = end;
#define FE_RUN(NT, MINB, BLK) dmma_modal_run<FORM, DIM, ND, NMODE, NT, MINB, BLK>(p, k, end - start, s)
  FE_MODAL_CFGS(FE_RUN)
#undef FE_RUN
}

// ---------------------------------------------------------------------------
// sum-factorised tensor-cell kernel
// ---------------------------------------------------------------------------

// 1D factors of a tensor-cell plan -> the kernel parameter block
template <int Q, int P>
int fill_tensor_tables(const fe_plan* p, TensorParams<Q, P>* hp) {
  if (p->q1d != Q || p->degree + 1 != P) return fail(FE_EINVAL, "tensor factors do not match the kernel");
  for (int a = 0; a < Q; ++a) {
    for (int i = 0; i < P; ++i) {
      hp->B[a][i] = p->B1d[a * P + i];
      hp->D[a][i] = p->D1d[a * P + i];
    }
    hp->w[a] = p->w1d[a];
  }
  for (int a = 0; a < Q; ++a) hp->x[a] = p->x1d[a];
  // even / odd parts of the tables (used by the even-odd kernels, which also
  // verify the mirror symmetry they rely on)
  for (int q = 0; q < (Q + 1) / 2; ++q)
    for (int j = 0; j < (P + 1) / 2; ++j) {
      const bool mid = (P % 2) && j == P / 2;
      hp->Be[q][j] = mid ? hp->B[q][j] : 0.5 * (hp->B[q][j] + hp->B[q][P - 1 - j]);
      hp->Bo[q][j] = mid ? 0.0 : 0.5 * (hp->B[q][j] - hp->B[q][P - 1 - j]);
      hp->De[q][j] = mid ? hp->D[q][j] : 0.5 * (hp->D[q][j] + hp->D[q][P - 1 - j]);
      hp->Do[q][j] = mid ? 0.0 : 0.5 * (hp->D[q][j] - hp->D[q][P - 1 - j]);
    }
  // collocation derivative at the Gauss points: Dc[a][e] = l_e'(x_a) for the
  // Lagrange basis l_e on the Gauss points (barycentric formula)
  double bw[Q];
  for (int e = 0; e < Q; ++e) {
    double prod = 1.0;
    for (int m = 0; m < Q; ++m)
      if (m != e) prod *= hp->x[e] - hp->x[m];
    bw[e] = 1.0 / prod;
  }
  for (int a = 0; a < Q; ++a) {
    double diag = 0.0;
    for (int e = 0; e < Q; ++e) {
      if (e == a) continue;
      hp->Dc[a][e] = (bw[e] / bw[a]) / (hp->x[a] - hp->x[e]);
      diag -= hp->Dc[a][e];
    }
    hp->Dc[a][a] = diag;
  }
  return FE_OK;
}

template <int FORM, int DIM, int P, int Q, int MINB, bool DIRECT>
int tensor_prepare(fe_plan* p) {
  using TP = TensorParams<Q, P>;
  using SM = TensorLayout<DIM, P, Q, form_vs(FORM, DIM), DIRECT, tensor_block<MINB>(), tensor_async<MINB>()>;
  static_assert(sizeof(TP) <= 32000, "parameter block too large");
  TP* hp = new TP();
  if (int rc = fill_tensor_tables<Q, P>(p, hp)) {
    delete hp;
    return rc;
  }
  // the kernel reads the mirror-symmetric half of the 1D tables
  for (int q = 0; (tensor_sym<P, Q>() || tensor_eo<DIM, P, Q, DIRECT>()) && q < Q; ++q) {
    bool ok = std::fabs(hp->x[q] - (1.0 - hp->x[Q - 1 - q])) <= 1e-13 && std::fabs(hp->w[q] - hp->w[Q - 1 - q]) <= 1e-13;
    for (int i = 0; i < P; ++i)
      ok = ok && std::fabs(hp->B[q][i] - hp->B[Q - 1 - q][P - 1 - i]) <= 1e-12 &&
           std::fabs(hp->D[q][i] + hp->D[Q - 1 - q][P - 1 - i]) <= 1e-11;
    if (!ok) {
      delete hp;
      return fail(FE_EUNSUPPORTED, "sum-factorised kernel needs mirror-symmetric 1D tables");
    }
  }
  p->host_params = hp;
  p->host_params_bytes = sizeof(TP);
  constexpr int CPB = SM::CPB;
  p->tables_bytes = (size_t)CPB * SM::size * sizeof(double);
  CUDA_TRY(cudaFuncSetAttribute(tensor_kernel<FORM, DIM, P, Q, MINB, DIRECT>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tables_bytes));
  p->cells_per_block = CPB;
  int dev = 0, sms = 0, per_sm = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tensor_kernel<FORM, DIM, P, Q, MINB, DIRECT>, SM::BLOCK,
                                                         p->tables_bytes));
  p->persistent_ctas = sms * (per_sm > 0 ? per_sm : 1);
  return FE_OK;
}

template <int FORM, int DIM, int P, int Q, int MINB, bool DIRECT>
int tensor_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                  const double* c0, const double* c1, cudaStream_t s) {
  using TP = TensorParams<Q, P>;
  TP hpv = *static_cast<const TP*>(p->host_params);
  TP* hp = &hpv;
  if (!p->d_map_lex) return fail(FE_ENOMESH, "tensor plan without a lexicographic map");
  hp->mesh = mesh_view(p);
  hp->maplex = p->d_map_lex;
  hp->u = u;
  hp->y = y;
  hp->mu = c0;
  hp->lam = c1;
  hp->start = start;
  hp->end = end;
  hp->p0 = p->params[0];
  hp->p1 = p->params[1];
  const int n = end - start;
  const int cpb = p->cells_per_block;
  const int nbatch = (n + cpb - 1) / cpb;
  const int grid = nbatch < p->persistent_ctas ? nbatch : p->persistent_ctas;
  launch_op(tensor_kernel<FORM, DIM, P, Q, MINB, DIRECT>, grid, tensor_block<MINB>(), p->tables_bytes, s, *hp);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// plane-per-thread scalar Laplacian on hexahedra (kern_plane.cuh)
template <int P, int Q, int WARPS, int MINB, bool V1, int CU = 1>
int plane_prepare(fe_plan* p) {
  using TP = TensorParams<Q, P>;
  using L = std::conditional_t<V1, Plane1Layout<P, Q>, PlaneLayout<P, Q>>;
  const void* kfn;
  if constexpr (V1)
    kfn = (const void*)plane1_kernel<P, Q, WARPS, MINB>;
  else
    kfn = (const void*)plane_kernel<P, Q, WARPS, MINB, CU>;
  TP* hp = new TP();
  if (int rc = fill_tensor_tables<Q, P>(p, hp)) {
    delete hp;
    return rc;
  }
  if constexpr (!V1 && FE_PLANE_SYM && CU == Q) {
    // the fully unrolled plane kernel reads the mirror-symmetric half of the 1D tables
    for (int q = 0; q < Q; ++q) {
      bool ok = std::fabs(hp->x[q] - (1.0 - hp->x[Q - 1 - q])) <= 1e-13 && std::fabs(hp->w[q] - hp->w[Q - 1 - q]) <= 1e-13;
      for (int i = 0; i < P; ++i)
        ok = ok && std::fabs(hp->B[q][i] - hp->B[Q - 1 - q][P - 1 - i]) <= 1e-12 &&
             std::fabs(hp->D[q][i] + hp->D[Q - 1 - q][P - 1 - i]) <= 1e-11;
      if (!ok) {
        delete hp;
        return fail(FE_EUNSUPPORTED, "plane kernel needs mirror-symmetric 1D tables");
      }
    }
  }
  p->host_params = hp;
  p->host_params_bytes = sizeof(TP);
  p->tables_bytes = (size_t)WARPS * L::WARP_DOUBLES * sizeof(double);
  CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tables_bytes));
  p->cells_per_block = WARPS * L::TPW;
  int dev = 0, sms = 0, per_sm = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, WARPS * 32, p->tables_bytes));
  p->persistent_ctas = sms * (per_sm > 0 ? per_sm : 1);
  return FE_OK;
}

template <int P, int Q, int WARPS, int MINB, bool V1, int CU = 1>
int plane_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                 const double*, const double*, cudaStream_t s) {
  using TP = TensorParams<Q, P>;
  TP hpv = *static_cast<const TP*>(p->host_params);
  TP* hp = &hpv;
  if (!p->d_map_lex) return fail(FE_ENOMESH, "tensor plan without a lexicographic map");
  hp->mesh = mesh_view(p);
  hp->maplex = p->d_map_lex;
  hp->u = u;
  hp->y = y;
  hp->mu = hp->lam = nullptr;
  hp->start = start;
  hp->end = end;
  const int n = end - start;
  const int cpb = p->cells_per_block;
  const int nbatch = (n + cpb - 1) / cpb;
  const int grid = nbatch < p->persistent_ctas ? nbatch : p->persistent_ctas;
  if constexpr (V1)
    launch_op(plane1_kernel<P, Q, WARPS, MINB>, grid, WARPS * 32, p->tables_bytes, s, *hp);
  else
    launch_op(plane_kernel<P, Q, WARPS, MINB, CU>, grid, WARPS * 32, p->tables_bytes, s, *hp);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// thread-per-cell sum-factorised Q1 hex Laplacian (kern_hexq1.cuh)
int hexq1_prepare(fe_plan* p) {
  using TP = TensorParams<2, 2>;
  for (int i = 0; i < 8; ++i)
    if ((int)p->lex.size() != 8 || p->lex[i] != i)
      return fail(FE_EUNSUPPORTED, "hexq1 kernel needs the tensor-ordered Q1 element");
  TP* hp = new TP();
  if (int rc = fill_tensor_tables<2, 2>(p, hp)) {
    delete hp;
    return rc;
  }
  // the kernel uses the linear Lagrange structure on [0,1]: B[a] = (1-x_a, x_a), D = (-1, 1)
  for (int a = 0; a < 2; ++a)
    if (std::fabs(hp->B[a][0] - (1.0 - hp->x[a])) > 1e-14 || std::fabs(hp->B[a][1] - hp->x[a]) > 1e-14 ||
        std::fabs(hp->D[a][0] + 1.0) > 1e-14 || std::fabs(hp->D[a][1] - 1.0) > 1e-14) {
      delete hp;
      return fail(FE_EUNSUPPORTED, "hexq1 kernel needs the linear Lagrange basis on [0,1]");
    }
  p->host_params = hp;
  p->host_params_bytes = sizeof(TP);
  // CTAs of 128 threads per SM the register allocation must allow
  const char* env = getenv("FE_HEXQ1_MINB");
  p->dmma_cfg = env ? atoi(env) : 4;  // measured: 23.3 us at 4 (96 B spill), 23.6 at 3, 28.8 at 1
  return FE_OK;
}

int hexq1_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                 const double*, const double*, cudaStream_t s) {
  using TP = TensorParams<2, 2>;
  TP hpv = *static_cast<const TP*>(p->host_params);
  TP* hp = &hpv;
  hp->mesh = mesh_view(p);
  hp->maplex = p->d_map_lex;
  hp->u = u;
  hp->y = y;
  hp->mu = hp->lam = nullptr;
  hp->start = start;
  hp->end = end;
  const int n = end - start;
  static const int blk = getenv("FE_HEXQ1_BLOCK") ? atoi(getenv("FE_HEXQ1_BLOCK")) : 128;  // 32/64/128
  const unsigned g = (n + blk - 1) / blk;
  switch (p->dmma_cfg) {
    case 1: launch_op(hexq1_lap_kernel<1>, g, blk, 0, s, *hp); break;
    case 2: launch_op(hexq1_lap_kernel<2>, g, blk, 0, s, *hp); break;
    case 4: launch_op(hexq1_lap_kernel<4>, g, blk, 0, s, *hp); break;
    default: launch_op(hexq1_lap_kernel<3>, g, blk, 0, s, *hp); break;
  }
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// thread-per-cell sum-factorised Q2 hex Laplacian (kern_hexq1.cuh)
#ifndef FE_HEXQ2_BLOCK
#define FE_HEXQ2_BLOCK 64
#endif
int hexq2_prepare(fe_plan* p) {
  if ((int)p->lex.size() != 27) return fail(FE_EUNSUPPORTED, "hexq2 kernel needs the 27-node tensor map");
  TensorParams<3, 3> tp;
  if (int rc = fill_tensor_tables<3, 3>(p, &tp)) return rc;
  HexQ2Params* hp = new HexQ2Params();
  for (int n = 0; n < 27; ++n) hp->lex[n] = p->lex[n];
  for (int a = 0; a < 3; ++a) {
    for (int i = 0; i < 3; ++i) {
      hp->B[a][i] = tp.B[a][i];
      hp->Dc[a][i] = tp.Dc[a][i];
    }
    hp->x[a] = tp.x[a];
    hp->w[a] = tp.w[a];
  }
  p->host_params = hp;
  p->host_params_bytes = sizeof(HexQ2Params);
  return FE_OK;
}

int hexq2_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                 const double*, const double*, cudaStream_t s) {
  HexQ2Params hpv = *static_cast<const HexQ2Params*>(p->host_params);
  hpv.mesh = mesh_view(p);
  hpv.u = u;
  hpv.y = y;
  hpv.start = start;
  hpv.end = end;
  const int n = end - start;
  if (n > 0) launch_op(hexq2_lap_kernel<FE_HEXQ2_BLOCK, 1>, (unsigned)((n + FE_HEXQ2_BLOCK - 1) / FE_HEXQ2_BLOCK), FE_HEXQ2_BLOCK, 0, s, hpv);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// lane-per-plane shuffle-exchanged Qk hex Laplacian, k = 3, 4 (kern_hexq1.cuh)
#ifndef FE_HEXLP_BLOCK
#define FE_HEXLP_BLOCK 64
#endif
template <int Q>
int hexlp_prepare(fe_plan* p) {
  if ((int)p->lex.size() != Q * Q * Q) return fail(FE_EUNSUPPORTED, "hexlp kernel needs the tensor map");
  TensorParams<Q, Q> tp;
  if (int rc = fill_tensor_tables<Q, Q>(p, &tp)) return rc;
  HexLPParams<Q>* hp = new HexLPParams<Q>();
  for (int a = 0; a < Q; ++a) {
    for (int i = 0; i < Q; ++i) {
      hp->B[a][i] = tp.B[a][i];
      hp->Dc[a][i] = tp.Dc[a][i];
    }
    hp->x[a] = tp.x[a];
    hp->w[a] = tp.w[a];
  }
  p->host_params = hp;
  p->host_params_bytes = sizeof(HexLPParams<Q>);
  return FE_OK;
}

template <int Q>
int hexlp_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                 const double*, const double*, cudaStream_t s) {
  HexLPParams<Q> hpv = *static_cast<const HexLPParams<Q>*>(p->host_params);
  if (!p->d_map_lex) return fail(FE_ENOMESH, "tensor plan without a lexicographic map");
  hpv.mesh = mesh_view(p);
  hpv.maplex = p->d_map_lex;
  hpv.u = u;
  hpv.y = y;
  hpv.start = start;
  hpv.end = end;
  const int n = end - start;
  constexpr int CPB = (FE_HEXLP_BLOCK / 32) * (32 / Q);   // cells per CTA
  if (n > 0) launch_op(hexlp_lap_kernel<Q, FE_HEXLP_BLOCK, 1>, (unsigned)((n + CPB - 1) / CPB), FE_HEXLP_BLOCK, 0, s, hpv);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// component-pair 2D elasticity kernel (kern_pair.cuh).  FE_PAIR_CFG selects
// the kernel: 0 = round-1 kernel (one cell pair per thread pair, gather on
// the critical path), 1 = pipelined persistent kernel, 4-warp CTAs, 2 per SM,
// 2 = the round-1 structure with every 1D contraction in even-odd form
#ifndef FE_PAIR_CFG
#define FE_PAIR_CFG 2   // 0 = round-1 structure, 1 = pipelined persistent kernel (slower: ptxas hoists the table
#endif                  // constants out of the loop, profiles/r02/ab_pair_pipe.txt), 2 = even-odd kernel (kept:
                        // C4-quad-Q3 0.263 -> 0.257 ms, Q4 0.479 -> 0.444 ms, profiles/r02/ab_pair_eo.txt)
constexpr int kPairPipeWarps = 4;

template <int FORM, int P, int Q, int MINB>
int pair_pipe_setup(fe_plan* p, int dev_sms) {
  using L = PairPipeLayout<P>;
  auto kfn = pair_pipe_kernel<FORM, P, Q, kPairPipeWarps, MINB>;
  const size_t smem = (size_t)kPairPipeWarps * L::WARP_DOUBLES * sizeof(double);
  CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kPairPipeWarps * 32, smem));
  p->tables_bytes = smem;
  p->persistent_ctas = dev_sms * (per_sm > 0 ? per_sm : 1);
  return FE_OK;
}

template <int FORM, int P, int Q, int MINB>
int pair_prepare(fe_plan* p) {
  using TP = TensorParams<Q, P>;
  TP* hp = new TP();
  if (int rc = fill_tensor_tables<Q, P>(p, hp)) {
    delete hp;
    return rc;
  }
  p->host_params = hp;
  p->host_params_bytes = sizeof(TP);
  const char* env = getenv("FE_PAIR_CFG");
  p->dmma_cfg = env ? atoi(env) : FE_PAIR_CFG;
  if (p->dmma_cfg < 0 || p->dmma_cfg > 2) p->dmma_cfg = FE_PAIR_CFG;   // 2: even-odd kernel
  // the pipelined kernel (and the round-1 kernel under FE_PAIR_SYM) reads the
  // mirror-symmetric half of the 1D tables
  bool sym = true;
  for (int q = 0; q < Q; ++q) {
    if (std::fabs(hp->x[q] - (1.0 - hp->x[Q - 1 - q])) > 1e-13 || std::fabs(hp->w[q] - hp->w[Q - 1 - q]) > 1e-13)
      sym = false;
    for (int i = 0; i < P; ++i)
      if (std::fabs(hp->B[q][i] - hp->B[Q - 1 - q][P - 1 - i]) > 1e-12 ||
          std::fabs(hp->D[q][i] + hp->D[Q - 1 - q][P - 1 - i]) > 1e-11)
        sym = false;
  }
  if (!sym) {
    if (FE_PAIR_SYM) return fail(FE_EUNSUPPORTED, "pair kernel needs mirror-symmetric 1D tables");
    p->dmma_cfg = 0;
  }
  int dev = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (p->dmma_cfg == 1) return pair_pipe_setup<FORM, P, Q, 2>(p, sms);
  if (p->dmma_cfg == 2 && !sym) return fail(FE_EUNSUPPORTED, "even-odd pair kernel needs mirror-symmetric 1D tables");
  return FE_OK;
}

template <int FORM, int P, int Q, int MINB>
int pair_launch(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
                const double* c0, const double* c1, cudaStream_t s) {
  using TP = TensorParams<Q, P>;
  TP hpv = *static_cast<const TP*>(p->host_params);
  TP* hp = &hpv;
  if (!p->d_map_lex) return fail(FE_ENOMESH, "tensor plan without a lexicographic map");
  hp->mesh = mesh_view(p);
  hp->maplex = p->d_map_lex;
  hp->u = u;
  hp->y = y;
  hp->mu = c0;
  hp->lam = c1;
  hp->start = start;
  hp->end = end;
  if (p->dmma_cfg == 0 || p->dmma_cfg == 2) {
    const int64_t nt = 2 * (int64_t)(end - start);
    if (p->dmma_cfg == 2)
      launch_op(pair_eo_kernel<FORM, P, Q, MINB>, (unsigned)((nt + kPairBlock - 1) / kPairBlock), kPairBlock, 0, s, *hp);
    else
      launch_op(pair_kernel<FORM, P, Q, MINB>, (unsigned)((nt + kPairBlock - 1) / kPairBlock), kPairBlock, 0, s, *hp);
  } else {
    const int nbatch = (end - start + 15) / 16;
    const int need = (nbatch + kPairPipeWarps - 1) / kPairPipeWarps;
    const unsigned grid = (unsigned)(need < p->persistent_ctas ? need : p->persistent_ctas);
    if (grid > 0) {
      const unsigned blk = kPairPipeWarps * 32;
      launch_op(pair_pipe_kernel<FORM, P, Q, kPairPipeWarps, 2>, grid, blk, p->tables_bytes, s, *hp);
    }
  }
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

// ---------------------------------------------------------------------------
// registry
// ---------------------------------------------------------------------------

#define QV(FORM, CELL, DIM, NV, K, ND, NQ, AFF)                                              \
  {FORM, CELL, K, NQ, 0, "quad", 128, quad_prepare<FORM, DIM, NV, ND, NQ, AFF>,           \
   quad_launch<FORM, DIM, NV, ND, NQ, AFF>, quad_diag<FORM, DIM, NV, ND, NQ, AFF>}
#define DMV(FORM, CELL, DIM, K, ND)                                                          \
  {FORM, CELL, K, -1, 20, "dmma_element_tensor", kDmmaBlock, dmma_prepare<FORM, DIM, ND>,    \
   dmma_launch<FORM, DIM, ND>}
#define DMMV(FORM, CELL, DIM, K, ND, NMODE)                                                  \
  {FORM, CELL, K, -1, 21, "dmma_modal", kDmmaBlock, dmma_modal_prepare<FORM, DIM, ND, NMODE>,  \
   dmma_modal_launch<FORM, DIM, ND, NMODE>}
#define TV(FORM, CELL, DIM, K, P, Q, MINB)                                                   \
  {FORM, CELL, K, (DIM == 3 ? Q * Q * Q : Q * Q), 20, "sum_factorised", 256,                 \
   tensor_prepare<FORM, DIM, P, Q, MINB, false>, tensor_launch<FORM, DIM, P, Q, MINB, false>}
#define TVC(FORM, CELL, DIM, K, P, Q, MINB)                                                  \
  {FORM, CELL, K, (DIM == 3 ? Q * Q * Q : Q * Q), 19, "sum_factorised_colloc", 256,          \
   tensor_prepare<FORM, DIM, P, Q, MINB, false>, tensor_launch<FORM, DIM, P, Q, MINB, false>}
#define TVD(FORM, CELL, DIM, K, P, Q, MINB)                                                  \
  {FORM, CELL, K, (DIM == 3 ? Q * Q * Q : Q * Q), 20, "sum_factorised_direct", 256,          \
   tensor_prepare<FORM, DIM, P, Q, MINB, true>, tensor_launch<FORM, DIM, P, Q, MINB, true>}
#define PLV(K, P, Q, WARPS, MINB, CU)                                                        \
  {FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, K, Q * Q * Q, 22, "sum_factorised_plane",   \
   WARPS * 32, plane_prepare<P, Q, WARPS, MINB, false, CU>, plane_launch<P, Q, WARPS, MINB, false, CU>}
#define PL1V(K, P, Q, WARPS, MINB)                                                           \
  {FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, K, Q * Q * Q, 23, "sum_factorised_plane_t",  \
   WARPS * 32, plane_prepare<P, Q, WARPS, MINB, true>, plane_launch<P, Q, WARPS, MINB, true>}
#define PRV(FORM, K, P, Q, MINB)                                                             \
  {FORM, FE_CELL_QUADRILATERAL, K, Q * Q, 26, "component_pair", 128, pair_prepare<FORM, P, Q, MINB>, \
   pair_launch<FORM, P, Q, MINB>}
#define ETPV(FORM, CELL, DIM, K, ND)                                                         \
  {FORM, CELL, K, -1, 15, "element_tensor_patch", kPatchCells, etp_prepare<FORM, DIM, ND>,   \
   etp_launch<FORM, DIM, ND>}
#define QCV(FORM, CELL, DIM, K, ND, NQ)                                                      \
  {FORM, CELL, K, NQ, 5, "quad_const", 128, qc_prepare<FORM, DIM, DIM + 1, ND, NQ, true, 1, 3>, \
   qc_launch<FORM, DIM, DIM + 1, ND, NQ, true, 1, 3>}
#ifndef FE_VTX_MINB
#define FE_VTX_MINB 1
#endif
#ifndef FE_VTX_UNR
#define FE_VTX_UNR 3   // physical-gradient kernel: C5 5.29 ms at 1 and 2, 5.11 at 3 (profiles/r02/vtx_variants.log)
#endif
#ifndef FE_VTX_TUNR
#define FE_VTX_TUNR 1
#endif
#define VTXV(FORM, CELL, DIM, K, ND, NQ, MINB, UNR)                                          \
  {FORM, CELL, K, NQ, 6, "quad_vertex_grad", 128, vtx_prepare<FORM, DIM, DIM + 1, ND, NQ, MINB, UNR>, \
   vtx_launch<FORM, DIM, DIM + 1, ND, NQ, MINB, UNR>}
#define QCVU(FORM, CELL, DIM, K, ND, NQ, UNR)                                                \
  {FORM, CELL, K, NQ, 5, "quad_const", 128, qc_prepare<FORM, DIM, DIM + 1, ND, NQ, true, 1, UNR>, \
   qc_launch<FORM, DIM, DIM + 1, ND, NQ, true, 1, UNR>}
#define QCT(FORM, CELL, DIM, NV, K, ND, NQ, MINB, UNR)                                       \
  {FORM, CELL, K, NQ, 25, "quad_const_tensor", 128,                                          \
   qc_prepare<FORM, DIM, NV, ND, NQ, false, MINB, UNR>, qc_launch<FORM, DIM, NV, ND, NQ, false, MINB, UNR>}
#define HQ1V()                                                                               \
  {FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 1, 8, 27, "sum_factorised_q1", 128,           \
   hexq1_prepare, hexq1_launch}
#define HQ2V()                                                                               \
  {FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 2, 27, 28, "sum_factorised_q2", FE_HEXQ2_BLOCK, \
   hexq2_prepare, hexq2_launch}
#define HLPV(K, Q)                                                                           \
  {FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, K, Q * Q * Q, 29, "sum_factorised_lane_plane", FE_HEXLP_BLOCK, \
   hexlp_prepare<Q>, hexlp_launch<Q>}
#define SPV(FORM, CELL, DIM, K, ND, NQS)                                                     \
  {FORM, CELL, K, -1, 12, "element_split", 128, split_prepare<FORM, DIM, ND, NQS>,           \
   split_launch<FORM, DIM, ND, NQS>}
#define ETV(FORM, CELL, DIM, K, ND)                                                          \
  {FORM, CELL, K, -1, 10, "element_tensor", 128, et_prepare<FORM, DIM, ND>,                  \
   et_launch<FORM, DIM, ND>}

// 2D reference forms on triangles (nq = (k+1)^2) and quadrilaterals (nq = (k+2)^2)
#define TRI_FORM(F)                                                                           \
  QV(F, FE_CELL_TRIANGLE, 2, 3, 1, 3, 4, true), QV(F, FE_CELL_TRIANGLE, 2, 3, 2, 6, 9, true), \
  QV(F, FE_CELL_TRIANGLE, 2, 3, 3, 10, 16, true), QV(F, FE_CELL_TRIANGLE, 2, 3, 4, 15, 25, true)
#define QUAD_FORM(F)                                                                          \
  QV(F, FE_CELL_QUADRILATERAL, 2, 4, 1, 4, 9, false),                                         \
  QV(F, FE_CELL_QUADRILATERAL, 2, 4, 2, 9, 16, false),                                        \
  QV(F, FE_CELL_QUADRILATERAL, 2, 4, 3, 16, 25, false),                                       \
  QV(F, FE_CELL_QUADRILATERAL, 2, 4, 4, 25, 36, false)

static const Variant kVariants[] = {
    TRI_FORM(FE_FORM_MASS), TRI_FORM(FE_FORM_HELMHOLTZ), TRI_FORM(FE_FORM_LAPLACIAN),
    TRI_FORM(FE_FORM_ELASTICITY), TRI_FORM(FE_FORM_LAPLACIAN_SCALAR),
    TRI_FORM(FE_FORM_ELASTICITY_LAME), TRI_FORM(FE_FORM_NEOHOOKEAN),
    TRI_FORM(FE_FORM_NEOHOOKEAN_TANGENT),
    QUAD_FORM(FE_FORM_MASS), QUAD_FORM(FE_FORM_HELMHOLTZ), QUAD_FORM(FE_FORM_LAPLACIAN),
    QUAD_FORM(FE_FORM_ELASTICITY), QUAD_FORM(FE_FORM_LAPLACIAN_SCALAR),
    QUAD_FORM(FE_FORM_ELASTICITY_LAME),
    // tetrahedra: nq = (k+1)^3
    QV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 4, 1, 4, 8, true),
    QV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 4, 2, 10, 27, true),
    QV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 4, 1, 4, 8, true),
    QV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 4, 2, 10, 27, true),
    QV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 4, 3, 20, 64, true),
    QV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 4, 4, 35, 125, true),
    QV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 4, 1, 4, 8, true),
    QV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 4, 2, 10, 27, true),
    QV(FE_FORM_ELASTICITY_LAME, FE_CELL_TETRAHEDRON, 3, 4, 1, 4, 8, true),
    QV(FE_FORM_ELASTICITY_LAME, FE_CELL_TETRAHEDRON, 3, 4, 2, 10, 27, true),
    QV(FE_FORM_NEOHOOKEAN, FE_CELL_TETRAHEDRON, 3, 4, 1, 4, 8, true),
    QV(FE_FORM_NEOHOOKEAN, FE_CELL_TETRAHEDRON, 3, 4, 2, 10, 27, true),
    QV(FE_FORM_NEOHOOKEAN_TANGENT, FE_CELL_TETRAHEDRON, 3, 4, 1, 4, 8, true),
    QV(FE_FORM_NEOHOOKEAN_TANGENT, FE_CELL_TETRAHEDRON, 3, 4, 2, 10, 27, true),
    // hexahedra: default rule nq = (k+2)^3, BASELINE C3 rule nq = (k+1)^3
    QV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 8, false),
    QV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, false),
    QV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 8, 2, 27, 27, false),
    QV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 8, 2, 27, 64, false),
    QV(FE_FORM_HELMHOLTZ, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, false),
    QV(FE_FORM_MASS, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, false),
    QV(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, false),
    QV(FE_FORM_ELASTICITY, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, false),
    QV(FE_FORM_LAPLACIAN, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, false),
    QV(FE_FORM_NEOHOOKEAN, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, false),
    // element-tensor kernels (affine simplices)
    ETPV(FE_FORM_MASS, FE_CELL_TRIANGLE, 2, 1, 3), ETPV(FE_FORM_MASS, FE_CELL_TRIANGLE, 2, 2, 6),
    ETPV(FE_FORM_MASS, FE_CELL_TRIANGLE, 2, 3, 10), ETPV(FE_FORM_HELMHOLTZ, FE_CELL_TRIANGLE, 2, 1, 3),
    ETPV(FE_FORM_HELMHOLTZ, FE_CELL_TRIANGLE, 2, 2, 6), ETPV(FE_FORM_HELMHOLTZ, FE_CELL_TRIANGLE, 2, 3, 10),
    ETPV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 1, 4), ETPV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 2, 10),
    ETPV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 1, 4),
    ETPV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 2, 10),
    ETPV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 1, 4),
    ETPV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 2, 10),
    ETV(FE_FORM_MASS, FE_CELL_TRIANGLE, 2, 1, 3), ETV(FE_FORM_MASS, FE_CELL_TRIANGLE, 2, 2, 6),
    ETV(FE_FORM_MASS, FE_CELL_TRIANGLE, 2, 3, 10), ETV(FE_FORM_MASS, FE_CELL_TRIANGLE, 2, 4, 15),
    ETV(FE_FORM_HELMHOLTZ, FE_CELL_TRIANGLE, 2, 1, 3), ETV(FE_FORM_HELMHOLTZ, FE_CELL_TRIANGLE, 2, 2, 6),
    ETV(FE_FORM_HELMHOLTZ, FE_CELL_TRIANGLE, 2, 3, 10), ETV(FE_FORM_HELMHOLTZ, FE_CELL_TRIANGLE, 2, 4, 15),
    ETV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 1, 4), ETV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 2, 10),
    ETV(FE_FORM_MASS, FE_CELL_TETRAHEDRON, 3, 3, 20),
    ETV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 1, 4),
    ETV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 2, 10),
    ETV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 3, 20),
    ETV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 1, 4),
    ETV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 2, 10),
    ETV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 3, 20),
    QCV(FE_FORM_NEOHOOKEAN, FE_CELL_TETRAHEDRON, 3, 1, 4, 8),
    QCV(FE_FORM_NEOHOOKEAN, FE_CELL_TETRAHEDRON, 3, 2, 10, 27),
    VTXV(FE_FORM_NEOHOOKEAN, FE_CELL_TETRAHEDRON, 3, 2, 10, 27, FE_VTX_MINB, FE_VTX_UNR),
    VTXV(FE_FORM_NEOHOOKEAN_TANGENT, FE_CELL_TETRAHEDRON, 3, 2, 10, 27, FE_VTX_MINB, FE_VTX_TUNR),
    QCV(FE_FORM_NEOHOOKEAN_TANGENT, FE_CELL_TETRAHEDRON, 3, 1, 4, 8),
    // tangent P2: state + increment + output (90 doubles) in registers; the
    // point loop is not unrolled (UNR 3 spills)
    QCVU(FE_FORM_NEOHOOKEAN_TANGENT, FE_CELL_TETRAHEDRON, 3, 2, 10, 27, 1),
    QCV(FE_FORM_ELASTICITY_LAME, FE_CELL_TETRAHEDRON, 3, 1, 4, 8),
    QCV(FE_FORM_ELASTICITY_LAME, FE_CELL_TETRAHEDRON, 3, 2, 10, 27),
    QCV(FE_FORM_NEOHOOKEAN, FE_CELL_TRIANGLE, 2, 1, 3, 4),
    QCV(FE_FORM_NEOHOOKEAN, FE_CELL_TRIANGLE, 2, 2, 6, 9),
    SPV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 1, 4, 1),
    SPV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 2, 10, 4),
    SPV(FE_FORM_HELMHOLTZ, FE_CELL_TETRAHEDRON, 3, 3, 20, 10),
    SPV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 1, 4, 1),
    SPV(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_TETRAHEDRON, 3, 2, 10, 4),
    // (..., MINB, quadrature-loop unroll): per measurement, profiles/r01/sweep_unroll*.txt
    QCT(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 8, 1, 8),
    HQ1V(),
    HQ2V(),
    HLPV(3, 4),
    HLPV(4, 5),
    QCT(FE_FORM_LAPLACIAN_SCALAR, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, 1, 3),
    QCT(FE_FORM_ELASTICITY_LAME, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, 1, 3),
    QCT(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 4, 1, 4, 9, 1, 1),
    QCT(FE_FORM_ELASTICITY_LAME, FE_CELL_QUADRILATERAL, 2, 4, 2, 9, 16, 4, 4),
    QCT(FE_FORM_NEOHOOKEAN, FE_CELL_HEXAHEDRON, 3, 8, 1, 8, 27, 1, 3),
    FE_TENSOR_VARIANTS
    FE_PLANE_VARIANTS
    FE_PLANE1_VARIANTS
    FE_PAIR_VARIANTS
    FE_DMMA_VARIANTS
};

// ---------------------------------------------------------------------------
// mesh binding kernels
// ---------------------------------------------------------------------------

__global__ void k_transpose_map(const int32_t* __restrict__ rm, int32_t* __restrict__ soa, int nc,
                                int nd, int64_t stride) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * nd) return;
  int c = (int)(t / nd), i = (int)(t % nd);
  soa[i * stride + c] = rm[t];
}

__global__ void k_permute_rows(const int32_t* __restrict__ rm, const int32_t* __restrict__ perm,
                               int32_t* __restrict__ out, int nc, int nd) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * nd) return;
  int64_t c = t / nd;
  int l = (int)(t % nd);
  out[t] = rm[c * nd + perm[l]];
}

// Zero-fill of y for an overwrite apply; lets the operator kernel launch
// as soon as every fill CTA is resident (griddepcontrol.launch_dependents).
__global__ void __launch_bounds__(256) k_zero_pdl(double* __restrict__ y, int64_t n) {
  asm volatile("griddepcontrol.launch_dependents;");
  double2* y2 = reinterpret_cast<double2*>(y);
  const int64_t n2 = n / 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
    y2[i] = make_double2(0.0, 0.0);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) y[n - 1] = 0.0;
}

// Zero-fill of the blocks of y (bsz entries each, bsz % 2 == 0) selected by
// mask; lets a dependent kernel launch early like k_zero_pdl.
__global__ void __launch_bounds__(256) k_zero_blocks(double* __restrict__ y, int64_t n, int64_t bsz,
                                                     unsigned long long mask, int nblk) {
  asm volatile("griddepcontrol.launch_dependents;");
  for (int b = 0; b < nblk; ++b) {
    if (!((mask >> b) & 1)) continue;
    const int64_t a = (int64_t)b * bsz, e = a + bsz < n ? a + bsz : n;
    double2* y2 = reinterpret_cast<double2*>(y + a);
    const int64_t n2 = (e - a) / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
      y2[i] = make_double2(0.0, 0.0);
    if (blockIdx.x == 0 && threadIdx.x == 0 && ((e - a) & 1)) y[e - 1] = 0.0;
  }
}

__global__ void k_add(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}

__global__ void k_pad_coords(const double* __restrict__ x, double* __restrict__ out, int nv, int dim,
                             int cstride) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  for (int a = 0; a < cstride; ++a) out[(int64_t)v * cstride + a] = a < dim ? x[(int64_t)v * dim + a] : 0.0;
}

__global__ void k_check_vmap(const int32_t* __restrict__ map0, const int32_t* __restrict__ map1, int nc,
                             int nd, int nv, int* flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * nv) return;
  int c = (int)(t / nv), v = (int)(t % nv);
  if (map0[(int64_t)c * nd + v] != map1[t]) *flag = 1;
}

// host-entry pipelining: per chunk of cells, the 64-bit mask of the blocks
// (bsz entries each) of the vs-interleaved u / y vector its cells touch
// (row-major map; the gather and the scatter use the same map)
__global__ void k_chunk_blockmask(const int32_t* __restrict__ rm, int nc, int nd, const int32_t* __restrict__ bounds,
                                  int nchunk, int vs, int64_t bsz, unsigned long long* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * nd) return;
  const int c = (int)(t / nd);
  int k = 0;
  while (k + 1 < nchunk && c >= bounds[k + 1]) ++k;
  const int64_t e = (int64_t)vs * rm[t];
  const unsigned long long m = (1ull << (e / bsz)) | (1ull << ((e + vs - 1) / bsz));
  // one atomic per warp and chunk
  const unsigned grp = __match_any_sync(__activemask(), k);
  const unsigned lo = __reduce_or_sync(grp, (unsigned)m), hi = __reduce_or_sync(grp, (unsigned)(m >> 32));
  if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicOr(out + k, ((unsigned long long)hi << 32) | lo);
}

__global__ void k_check_range(const int32_t* __restrict__ m, int64_t n, int64_t hi, int* flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n && (m[t] < 0 || m[t] >= hi)) *flag = 1;
}

__global__ void k_check_vertex_cols(const int32_t* __restrict__ map0, int nc, int nd, int nv,
                                    int64_t nverts, int* flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * nv) return;
  int32_t v = map0[(t / nv) * nd + t % nv];
  if (v < 0 || v >= nverts) *flag = 1;
}

// macro-cell detection: corner dofs of macro-cell m from the first
// occurrence of each local macro-dof, then every cell dof of the macro-cell
// checked against the pattern (flag = 1 on any mismatch)
__global__ void k_macro_detect(const int32_t* __restrict__ rm, int nd, int64_t nmacro, int mc, int nu,
                               int npv, const int32_t* __restrict__ pat, const int32_t* __restrict__ first,
                               int32_t* __restrict__ corner, int64_t mstride, int* flag) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= nmacro) return;
  const int32_t* c = rm + m * mc * nd;
  for (int k = 0; k < nu; ++k) {
    const int f = first[k];
    corner[k * mstride + m] = c[(f / npv) * nd + f % npv];
  }
  for (int t = 0; t < mc; ++t)
    for (int i = 0; i < npv; ++i)
      if (c[t * nd + i] != corner[pat[t * npv + i] * mstride + m]) *flag = 1;
}

namespace {

void free_mesh(fe_plan* p) {
  if (p->d_vmap && p->d_vmap != p->d_map) cudaFree(p->d_vmap);
  cudaFree(p->d_map);
  cudaFree(p->d_map_rm);
  cudaFree(p->d_map_lex);
  cudaFree(p->d_coords);
  p->d_map = p->d_vmap = p->d_map_rm = p->d_map_lex = nullptr;
  cudaFree(p->d_patch_off);
  cudaFree(p->d_patch_dofs);
  cudaFree(p->d_pidx);
  cudaFree(p->d_macro);
  p->d_macro = nullptr;
  p->d_patch_off = p->d_patch_dofs = nullptr;
  p->d_pidx = nullptr;
  p->d_coords = nullptr;
  p->b_coords = p->b_map0 = p->b_map1 = nullptr;
}

const Variant* select_variant(const fe_plan* p, uint32_t flags) {
  const Variant* best = nullptr;
  for (const Variant& v : kVariants) {
    if (v.form != p->form || v.cell != p->cell || v.degree != p->degree) continue;
    if (v.nq >= 0 && v.nq != p->nq) continue;
    if (v.cell == FE_CELL_HEXAHEDRON || v.cell == FE_CELL_QUADRILATERAL)
      if (v.priority >= 20 && p->q1d == 0) continue;  // tensor kernels need 1D factors
    if ((flags & 1u) && v.priority > 0) continue;                // FE_PLAN_GENERIC: quad kernel only
    if (v.priority == 12 && (p->qw_aux.empty() || getenv("FE_NO_SPLIT"))) continue;  // split needs the modes
    // modal DMMA likewise; at P1/P2 it measured 2.7x / 1.8x slower than the
    // thread-per-cell split kernel (profiles/r01/sweep_modal2.txt), so only
    // P3/P4 are registered
    if (v.priority == 21 && (p->qw_aux.empty() || getenv("FE_NO_MODAL"))) continue;
    if (v.priority == 20 && getenv("FE_NO_DMMA") && v.cell == FE_CELL_TETRAHEDRON) continue;  // experiments
    if (v.priority == 25 && getenv("FE_NO_QCT")) continue;  // experiments: team kernel instead
    if (v.priority == 22 && getenv("FE_NO_PLANE")) continue;  // experiments: pencil team kernel
    if (v.priority == 23 && getenv("FE_NO_PLANE1")) continue;
    if (v.priority == 26 && getenv("FE_NO_PAIR")) continue;
    if (v.priority == 27 && getenv("FE_NO_HEXQ1")) continue;
    if (v.priority == 28 && getenv("FE_NO_HEXQ2")) continue;
    if (getenv("FE_TK_COLLOC56") && !strcmp(v.name, "sum_factorised_direct")) continue;   // experiments
    if (v.priority == 29 && !getenv("FE_HEXLP")) continue;   // opt-in until measured
    if (v.priority == 6 && getenv("FE_NO_VTX")) continue;
    // patch aggregation measured slower than plain REDs (profiles/r01/sweep_patch.jsonl):
    // opt-in only (FE_PATCH=1) for experiments
    if (v.priority == 15 && (!getenv("FE_PATCH") || (flags & 2u))) continue;
    if (!best || v.priority > best->priority) best = &v;
  }
  return best;
}

}  // namespace

// Verify the macro-cell pattern of the plan's kernel family on the bound
// mesh (every macro-cell) and keep the SoA corner dofs if it holds.
static int build_macro(fe_plan* p, cudaStream_t s) {
  const int mc = p->macro_mc, nu = p->macro_nu, npv = (int)p->macro_pat.size() / mc;
  const int64_t nmacro = p->ncells / mc;
  std::vector<int32_t> first(nu, -1);
  for (int f = 0; f < mc * npv; ++f)
    if (first[p->macro_pat[f]] < 0) first[p->macro_pat[f]] = f;
  std::vector<int32_t> tab(p->macro_pat);
  tab.insert(tab.end(), first.begin(), first.end());
  int32_t* d_tab = nullptr;
  int* d_flag = nullptr;
  p->macro_stride = (nmacro + 31) / 32 * 32;
  CUDA_TRY(cudaMalloc(&p->d_macro, (size_t)nu * p->macro_stride * sizeof(int32_t)));
  CUDA_TRY(cudaMalloc(&d_tab, tab.size() * sizeof(int32_t)));
  CUDA_TRY(cudaMalloc(&d_flag, sizeof(int)));
  CUDA_TRY(cudaMemcpyAsync(d_tab, tab.data(), tab.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
  k_macro_detect<<<(unsigned)((nmacro + 255) / 256), 256, 0, s>>>(
      p->d_map_rm, p->nd, nmacro, mc, nu, npv, d_tab, d_tab + mc * npv, p->d_macro, p->macro_stride, d_flag);
  int h_flag = 0;
  CUDA_TRY(cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(d_tab);
  cudaFree(d_flag);
  if (h_flag) {  // not a macro-cell mesh: the per-cell kernel runs
    cudaFree(p->d_macro);
    p->d_macro = nullptr;
  }
  return FE_OK;
}

// Patches of kPatchCells consecutive cells: sorted distinct dofs and the
// patch-local index of every cell dof (host side, once per bound mesh).
static int build_patches(fe_plan* p, const int32_t* map0, bool dev, cudaStream_t s) {
  const int nc = p->ncells, nd = p->nd;
  std::vector<int32_t> m((size_t)nc * nd);
  if (dev) {
    CUDA_TRY(cudaMemcpyAsync(m.data(), map0, m.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  } else {
    std::memcpy(m.data(), map0, m.size() * sizeof(int32_t));
  }
  const int np = (nc + kPatchCells - 1) / kPatchCells;
  std::vector<int32_t> off(np + 1, 0);
  std::vector<std::vector<int32_t>> uniq(np);
  std::vector<uint16_t> pidx((size_t)nd * p->stride, 0);
#pragma omp parallel for schedule(dynamic, 64)
  for (int b = 0; b < np; ++b) {
    const int c0 = b * kPatchCells, c1 = std::min(nc, c0 + kPatchCells);
    std::vector<int32_t>& u = uniq[b];
    u.assign(m.begin() + (size_t)c0 * nd, m.begin() + (size_t)c1 * nd);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    for (int c = c0; c < c1; ++c)
      for (int i = 0; i < nd; ++i)
        pidx[(size_t)i * p->stride + c] =
            (uint16_t)(std::lower_bound(u.begin(), u.end(), m[(size_t)c * nd + i]) - u.begin());
  }
  int maxu = 0;
  for (int b = 0; b < np; ++b) {
    off[b + 1] = off[b] + (int)uniq[b].size();
    maxu = std::max(maxu, (int)uniq[b].size());
  }
  std::vector<int32_t> dofs(off[np]);
  for (int b = 0; b < np; ++b) std::copy(uniq[b].begin(), uniq[b].end(), dofs.begin() + off[b]);
  CUDA_TRY(cudaMalloc(&p->d_patch_off, off.size() * sizeof(int32_t)));
  CUDA_TRY(cudaMalloc(&p->d_patch_dofs, std::max<size_t>(1, dofs.size()) * sizeof(int32_t)));
  CUDA_TRY(cudaMalloc(&p->d_pidx, pidx.size() * sizeof(uint16_t)));
  CUDA_TRY(cudaMemcpy(p->d_patch_off, off.data(), off.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_patch_dofs, dofs.data(), dofs.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_pidx, pidx.data(), pidx.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
  p->patch_maxu = maxu;
  return FE_OK;
}

__global__ void k_eval_log(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fast_log(x[i]);
}

__global__ void k_max_i32(const int32_t* __restrict__ m, int64_t nrows, int rowlen, int ncols,
                          int* __restrict__ out) {
  int best = -1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows * ncols;
       t += (int64_t)gridDim.x * blockDim.x)
    best = max(best, m[(t / ncols) * rowlen + t % ncols]);
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best >= 0) atomicMax(out, best);
}

extern "C" int fe_plan_bind_mesh(fe_plan*, int32_t, int32_t, int64_t, const double*, const int32_t*,
                                 const int32_t*, uint32_t, void*);

// Largest entry of columns [0, ncols) of a row-major [nrows][rowlen] map.
static int map_max(const int32_t* m, int64_t nrows, int rowlen, int ncols, bool dev, cudaStream_t s,
                   int* result) {
  *result = -1;
  if (nrows <= 0) return FE_OK;
  if (!dev) {
    int best = -1;
#pragma omp parallel for reduction(max : best) schedule(static)
    for (int64_t r = 0; r < nrows; ++r)
      for (int c = 0; c < ncols; ++c) best = std::max(best, m[r * rowlen + c]);
    *result = best;
    return FE_OK;
  }
  int* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(int)));
  CUDA_TRY(cudaMemsetAsync(d, 0xff, sizeof(int), s));
  k_max_i32<<<148 * 8, 256, 0, s>>>(m, nrows, rowlen, ncols, d);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(result, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(d);
  return FE_OK;
}

// fe_wrap / fe_wrap_host: the reference's wrap_<form> takes the mesh with
// every call and no sizes (codegen.py:375-394).  When dat1/map0/map1 (or the
// pointer kind) differ from the bound ones -- or an implicitly bound mesh is
// shorter than `end` -- the mesh is (re-)bound here: cells [0, end), nglobal
// = max(map0) + 1, nverts = max(vertex map) + 1, derived from the maps.  A
// mesh bound explicitly by fe_plan_bind_mesh with the same buffers is used
// as is (the GPU layout is built once per mesh, not per apply).
static int wrap_host_impl(fe_plan* p, int32_t start, int32_t end, double* dat0, const double* dat2,
                          const double* dat3, const double* dat4);

static int wrap_bind(fe_plan* p, int32_t end, const double* dat1, const int32_t* map0,
                     const int32_t* map1, bool dev, cudaStream_t s) {
  const bool same = p->d_map && p->b_coords == dat1 && p->b_map0 == map0 && p->b_map1 == map1 &&
                    (bool)(p->b_flags & FE_PTR_DEVICE) == dev;
  if (same && !(p->auto_bound && end > p->ncells)) return FE_OK;
  if (!dat1 || !map0) return fail(FE_EINVAL, "null dat1/map0");
  if (end < 0) return fail(FE_EINVAL, "bad end %d", end);
  int maxdof = -1, maxv = -1;
  int rc = map_max(map0, end, p->nd, p->nd, dev, s, &maxdof);
  if (!rc) rc = map1 ? map_max(map1, end, p->nv, p->nv, dev, s, &maxv) : map_max(map0, end, p->nd, p->nv, dev, s, &maxv);
  if (rc) return rc;
  if (end > 0 && (maxdof < 0 || maxv < 0)) return fail(FE_EINVAL, "map entry out of range");
  rc = fe_plan_bind_mesh(p, end, std::max(1, maxv + 1), std::max(1, maxdof + 1), dat1, map0, map1,
                         dev ? FE_PTR_DEVICE : FE_PTR_HOST, s);
  if (rc) return rc;
  p->auto_bound = true;
  return FE_OK;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

int fe_abi_version(void) { return FE_ABI_VERSION; }

const char* fe_last_error(void) { return g_err.c_str(); }

int fe_plan_create(fe_plan** out, const fe_element_desc* d, uint32_t flags) {
  if (!out || !d) return fail(FE_EINVAL, "null argument");
  *out = nullptr;
  if (d->cell < 0 || d->cell > 3) return fail(FE_EINVAL, "bad cell %d", d->cell);
  if (d->form < 0 || d->form > FE_FORM_NEOHOOKEAN_TANGENT) return fail(FE_EINVAL, "bad form %d", d->form);
  fe_plan* p = new fe_plan();
  p->form = d->form;
  p->cell = d->cell;
  p->degree = d->degree;
  p->dim = cell_dim(d->cell);
  p->nv = cell_nv(d->cell);
  p->vs = form_vs(d->form, p->dim);
  p->nd = d->ndof;
  p->nq = d->nq;
  p->q1d = d->q1d;
  p->flags = flags;
  std::memcpy(p->params, d->params, sizeof p->params);
  if (d->value_size != p->vs || d->nvert != p->nv) {
    delete p;
    return fail(FE_EINVAL, "value_size/nvert inconsistent with form/cell");
  }
  if (!d->qweights || !d->phi || !d->dphi || !d->gphi || !d->gdphi) {
    delete p;
    return fail(FE_EINVAL, "missing tables");
  }
  const int nq = p->nq, nd = p->nd, nv = p->nv, dim = p->dim;
  p->qw.assign(d->qweights, d->qweights + nq);
  p->phi.assign(d->phi, d->phi + (size_t)nq * nd);
  p->dphi.assign(d->dphi, d->dphi + (size_t)nq * nd * dim);
  p->gphi.assign(d->gphi, d->gphi + (size_t)nq * nv);
  p->gdphi.assign(d->gdphi, d->gdphi + (size_t)nq * nv * dim);
  if (p->q1d > 0) {
    const int pp = p->degree + 1;
    if (!d->B1d || !d->D1d || !d->w1d || !d->x1d || !d->lex) {
      delete p;
      return fail(FE_EINVAL, "missing tensor factors");
    }
    p->B1d.assign(d->B1d, d->B1d + (size_t)p->q1d * pp);
    p->D1d.assign(d->D1d, d->D1d + (size_t)p->q1d * pp);
    p->w1d.assign(d->w1d, d->w1d + p->q1d);
    p->x1d.assign(d->x1d, d->x1d + p->q1d);
    int n = 1;
    for (int a = 0; a < dim; ++a) n *= pp;
    p->lex.assign(d->lex, d->lex + n);
  }
  if (getenv("FE_NO_PATCH")) flags |= 2u;  // experiments: disable patch aggregation
  if (d->nq_aux > 0 && d->qw_aux && d->dphi_aux) {
    p->qw_aux.assign(d->qw_aux, d->qw_aux + d->nq_aux);
    p->dphi_aux.assign(d->dphi_aux, d->dphi_aux + (size_t)d->nq_aux * nd * dim);
  }
  p->var = select_variant(p, flags);
  if (!p->var) {
    int form = p->form, cell = p->cell, deg = p->degree;
    delete p;
    return fail(FE_EUNSUPPORTED, "no sm_100a kernel for form %d cell %d degree %d nq %d", form,
                cell, deg, nq);
  }
  int rc = p->var->prepare(p);
  if (rc) {
    std::string msg = g_err;
    fe_plan_destroy(p);
    g_err = msg;
    return rc;
  }
  *out = p;
  return FE_OK;
}

int fe_plan_bind_mesh(fe_plan* p, int32_t ncells, int32_t nverts, int64_t nglobal,
                      const double* coords, const int32_t* map0, const int32_t* map1,
                      uint32_t ptr_flags, void* stream) {
  if (!p || !coords || !map0) return fail(FE_EINVAL, "null argument");
  if (ncells < 0 || nverts <= 0 || nglobal <= 0) return fail(FE_EINVAL, "bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  free_mesh(p);
  const int nd = p->nd, nv = p->nv, dim = p->dim, cst = dim == 2 ? 2 : 4;
  p->ncells = ncells;
  p->nverts = nverts;
  p->nglobal = nglobal;
  p->stride = ((int64_t)ncells + 31) / 32 * 32;
  const bool dev = ptr_flags & FE_PTR_DEVICE;
  const size_t mbytes = (size_t)ncells * nd * sizeof(int32_t);
  // raw (row-major) map0 on the device
  CUDA_TRY(cudaMalloc(&p->d_map_rm, mbytes > 0 ? mbytes : 4));
  if (mbytes) CUDA_TRY(cudaMemcpyAsync(p->d_map_rm, map0, mbytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMalloc(&p->d_map, (size_t)nd * p->stride * sizeof(int32_t) + 4));
  int* d_flag = nullptr;
  CUDA_TRY(cudaMalloc(&d_flag, 2 * sizeof(int)));
  CUDA_TRY(cudaMemsetAsync(d_flag, 0, 2 * sizeof(int), s));
  const int T = 256;
  if (ncells > 0) {
    int64_t n = (int64_t)ncells * nd;
    k_transpose_map<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(p->d_map_rm, p->d_map, ncells, nd, p->stride);
    k_check_range<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(p->d_map_rm, n, nglobal, d_flag);
  }
  if (!p->lex.empty() && ncells > 0) {
    if (!p->d_lex) {
      CUDA_TRY(cudaMalloc(&p->d_lex, p->lex.size() * sizeof(int32_t)));
      CUDA_TRY(cudaMemcpy(p->d_lex, p->lex.data(), p->lex.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    CUDA_TRY(cudaMalloc(&p->d_map_lex, mbytes));
    int64_t n = (int64_t)ncells * nd;
    k_permute_rows<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(p->d_map_rm, p->d_lex, p->d_map_lex, ncells, nd);
  }
  p->d_vmap = p->d_map;
  int32_t* d_m1 = nullptr;
  if (map1 && ncells > 0) {
    size_t b1 = (size_t)ncells * nv * sizeof(int32_t);
    CUDA_TRY(cudaMalloc(&d_m1, b1));
    CUDA_TRY(cudaMemcpyAsync(d_m1, map1, b1, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    int64_t n = (int64_t)ncells * nv;
    k_check_vmap<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(p->d_map_rm, d_m1, ncells, nd, nv, d_flag + 1);
    k_check_range<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(d_m1, n, nverts, d_flag);
  } else if (ncells > 0) {
    // no vertex map given: map0[:, :nv] must be it -- at least every entry
    // must address a vertex (guards the coordinate gathers)
    int64_t n = (int64_t)ncells * nv;
    k_check_vertex_cols<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(p->d_map_rm, ncells, nd, nv,
                                                                  nverts, d_flag);
  }
  // coordinates, padded to 16/32 bytes per vertex
  double* d_x = nullptr;
  CUDA_TRY(cudaMalloc(&d_x, (size_t)nverts * dim * sizeof(double)));
  CUDA_TRY(cudaMemcpyAsync(d_x, coords, (size_t)nverts * dim * sizeof(double),
                           dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMalloc(&p->d_coords, (size_t)nverts * cst * sizeof(double)));
  k_pad_coords<<<(nverts + T - 1) / T, T, 0, s>>>(d_x, p->d_coords, nverts, dim, cst);
  int h_flag[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(h_flag, d_flag, sizeof h_flag, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(d_flag);
  cudaFree(d_x);
  if (h_flag[0]) {
    cudaFree(d_m1);
    free_mesh(p);
    return fail(FE_EINVAL, "map entry out of range");
  }
  {
    // host-entry pipelining: per cell chunk, the blocks of u / y it touches
    constexpr int NCH = FE_HOST_UCHUNKS;
    p->chunk_cell.assign(NCH + 1, 0);
    for (int c = 0; c <= NCH; ++c)
      p->chunk_cell[c] = (int32_t)std::min<int64_t>(ncells, ((int64_t)ncells * c / NCH + 191) / 192 * 192);
    p->chunk_cell[NCH] = ncells;
    p->chunk_mask.assign(NCH, 0);
    const int64_t ny = (int64_t)p->vs * p->nglobal;
    p->hblock = std::max<int64_t>(32, ((ny + 63) / 64 + 31) / 32 * 32);
    if (ncells > 0) {
      int32_t* d_b = nullptr;
      unsigned long long* d_o = nullptr;
      CUDA_TRY(cudaMalloc(&d_b, (NCH + 1) * sizeof(int32_t)));
      CUDA_TRY(cudaMalloc(&d_o, NCH * sizeof(unsigned long long)));
      CUDA_TRY(cudaMemcpyAsync(d_b, p->chunk_cell.data(), (NCH + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemsetAsync(d_o, 0, NCH * sizeof(unsigned long long), s));
      const int64_t n = (int64_t)ncells * nd;
      k_chunk_blockmask<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(p->d_map_rm, ncells, nd, d_b, NCH, p->vs,
                                                                 p->hblock, d_o);
      static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "mask type");
      CUDA_TRY(cudaMemcpyAsync(p->chunk_mask.data(), d_o, NCH * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      cudaFree(d_b);
      cudaFree(d_o);
    }
  }
  if (h_flag[1]) {
    // map0[:, :nv] is not the vertex map: keep a separate SoA vertex map
    CUDA_TRY(cudaMalloc(&p->d_vmap, (size_t)nv * p->stride * sizeof(int32_t) + 4));
    int64_t n = (int64_t)ncells * nv;
    k_transpose_map<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(d_m1, p->d_vmap, ncells, nv, p->stride);
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  cudaFree(d_m1);
  if (p->macro_mc > 0 && p->d_vmap == p->d_map && ncells >= p->macro_mc) {
    int rc = build_macro(p, s);
    if (rc) {
      free_mesh(p);
      return rc;
    }
  }
  if (p->wants_patch && ncells > 0) {
    int rc = build_patches(p, map0, dev, s);
    if (rc) {
      free_mesh(p);
      return rc;
    }
  }
  p->b_coords = coords;
  p->b_map0 = map0;
  p->b_map1 = map1;
  p->b_flags = ptr_flags;
  p->auto_bound = false;
  return FE_OK;
}

// the two-phase overwrite path pays when y is large and the range straddles
// the first cell chunk (FE_FILL_2PHASE_MB: threshold in MB, 0 disables)
static bool fill_two_phase(const fe_plan* p, int32_t start, int32_t end, int64_t ny) {
  // default off: measured SLOWER than the one-phase programmatic-dependent fill (C3-Q3 0.212 -> 0.238 ms,
  // C4-quad-Q3 0.271 -> 0.289 ms, profiles/r02/ab_fill_2phase.txt) -- the second operator launch and the
  // side-stream fill's CTAs cost more than the 2-10% of the apply the fill takes
  static const long mb = getenv("FE_FILL_2PHASE_MB") ? atol(getenv("FE_FILL_2PHASE_MB")) : 0;
  if (mb <= 0 || p->hblock <= 0 || p->chunk_mask.empty() || p->chunk_cell.size() < 3) return false;
  if (ny * (int64_t)sizeof(double) < (int64_t)mb << 20 || (p->hblock & 1)) return false;
  const int32_t ca = p->chunk_cell[1];
  return start < ca && ca < end && start >= p->chunk_cell[0];
}

int fe_apply(const fe_plan* p, int32_t start, int32_t end, double* y, const double* u,
             const double* c0, const double* c1, uint32_t apply_flags, void* stream) {
  if (!p) return fail(FE_EINVAL, "null plan");
  if (!p->d_map) return fail(FE_ENOMESH, "no mesh bound to the plan");
  if (start < 0 || end > p->ncells || start > end)
    return fail(FE_EINVAL, "cell range [%d, %d) outside [0, %d)", start, end, p->ncells);
  if (!y || !u) return fail(FE_EINVAL, "null dat0/dat2");
  if (p->form == FE_FORM_ELASTICITY_LAME && (!c0 || !c1))
    return fail(FE_EINVAL, "elasticity_lame needs the mu and lambda vertex fields");
  if (p->form == FE_FORM_NEOHOOKEAN_TANGENT && !c0)
    return fail(FE_EINVAL, "neohookean_tangent needs the state u (coef0)");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ny = (int64_t)p->vs * p->nglobal;
  if ((apply_flags & FE_APPLY_OVERWRITE) && (end == start || (reinterpret_cast<uintptr_t>(y) & 15) ||
                                              getenv("FE_NO_PDL"))) {
    CUDA_TRY(cudaMemsetAsync(y, 0, (size_t)ny * sizeof(double), s));
  } else if ((apply_flags & FE_APPLY_OVERWRITE) && fill_two_phase(p, start, end, ny)) {
    // Large y (the fill is 2-10% of the apply and the operator is FP64-bound):
    // hide the fill under the arithmetic.  Phase A: zero the blocks of y the
    // first cell chunk scatters into (chunk_mask[0], found at bind) and start
    // that chunk as a programmatic dependent of this short fill; the rest of y
    // is zeroed on a side stream while the chunk computes, and the remaining
    // cells are launched behind both.  Serialised per plan (try_lock): a
    // concurrent overwrite apply on the same plan takes the one-phase path.
    fe_plan* mp = const_cast<fe_plan*>(p);
    std::unique_lock<std::mutex> lk(mp->fill_mutex, std::try_to_lock);
    if (lk.owns_lock()) {
      if (!mp->fill_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&mp->fill_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&mp->ev_fill_a, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&mp->ev_fill_b, cudaEventDisableTiming));
      }
      const int nblk = (int)((ny + p->hblock - 1) / p->hblock);
      const uint64_t all = nblk >= 64 ? ~0ull : ((1ull << nblk) - 1);
      const uint64_t ma = p->chunk_mask[0] & all, mb = all & ~ma;
      const int32_t ca = p->chunk_cell[1];
      const unsigned grid = 148 * 4;
      // both fills are ordered after what is already queued on s (ev_fill_a);
      // no node sits between fill A and the first operator launch, so that
      // launch stays its programmatic dependent
      CUDA_TRY(cudaEventRecord(mp->ev_fill_a, s));
      CUDA_TRY(cudaStreamWaitEvent(mp->fill_stream, mp->ev_fill_a, 0));
      k_zero_blocks<<<grid, 256, 0, s>>>(y, ny, p->hblock, ma, nblk);
      k_zero_blocks<<<grid, 256, 0, mp->fill_stream>>>(y, ny, p->hblock, mb, nblk);
      CUDA_TRY(cudaEventRecord(mp->ev_fill_b, mp->fill_stream));
      CUDA_TRY(cudaGetLastError());
      g_pdl_next = true;
      int rc = p->var->launch(p, start, ca, y, u, c0, c1, s);
      g_pdl_next = false;
      CUDA_TRY(cudaStreamWaitEvent(s, mp->ev_fill_b, 0));
      if (!rc) rc = p->var->launch(p, ca, end, y, u, c0, c1, s);
      return rc;
    }
    CUDA_TRY(cudaMemsetAsync(y, 0, (size_t)ny * sizeof(double), s));
  } else if (apply_flags & FE_APPLY_OVERWRITE) {
    // zero-fill as a kernel the operator launch depends on programmatically:
    // the operator's prologue (map/u/coordinate gathers, first cells)
    // overlaps the fill instead of queueing behind it
    const int64_t blocks = std::min<int64_t>((ny / 2 + 255) / 256, 148 * 4);
    k_zero_pdl<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, s>>>(y, ny);
    CUDA_TRY(cudaGetLastError());
    g_pdl_next = true;
  }
  if (end == start) return FE_OK;
  const int rc = p->var->launch(p, start, end, y, u, c0, c1, s);
  g_pdl_next = false;
  return rc;
}

int fe_diagonal(const fe_plan* p, int32_t start, int32_t end, double* diag, const double* c0,
                const double* c1, uint32_t apply_flags, void* stream) {
  if (!p) return fail(FE_EINVAL, "null plan");
  if (!p->d_map) return fail(FE_ENOMESH, "no mesh bound to the plan");
  if (start < 0 || end > p->ncells || start > end)
    return fail(FE_EINVAL, "cell range [%d, %d) outside [0, %d)", start, end, p->ncells);
  if (!diag) return fail(FE_EINVAL, "null diag");
  if (p->form == FE_FORM_ELASTICITY_LAME && (!c0 || !c1))
    return fail(FE_EINVAL, "elasticity_lame needs the mu and lambda vertex fields");
  if (p->form == FE_FORM_NEOHOOKEAN_TANGENT && !c0)
    return fail(FE_EINVAL, "neohookean_tangent needs the state u (coef0)");
  // the generic quadrature entry of this (form, cell, degree, rule)
  const Variant* g = nullptr;
  for (const Variant& v : kVariants)
    if (v.diag && v.form == p->form && v.cell == p->cell && v.degree == p->degree && v.nq == p->nq) g = &v;
  if (!g) return fail(FE_EUNSUPPORTED, "no diagonal kernel for this (form, cell, degree, rule)");
  cudaStream_t s = (cudaStream_t)stream;
  if (apply_flags & FE_APPLY_OVERWRITE)
    CUDA_TRY(cudaMemsetAsync(diag, 0, (size_t)p->vs * p->nglobal * sizeof(double), s));
  if (end == start) return FE_OK;
  return g->diag(p, start, end, diag, c0, c1, s);
}

int fe_wrap(fe_plan* p, int32_t start, int32_t end, double* dat0, const double* dat1,
            const double* dat2, const double* dat3, const double* dat4, const int32_t* map0,
            const int32_t* map1, void* stream) {
  if (!p) return fail(FE_EINVAL, "null plan");
  int rc = wrap_bind(p, end, dat1, map0, map1, true, (cudaStream_t)stream);
  if (rc) return rc;
  return fe_apply(p, start, end, dat0, dat2, dat3, dat4, FE_APPLY_ACCUMULATE, stream);
}

int fe_wrap_host(fe_plan* p, int32_t start, int32_t end, double* dat0, const double* dat1,
                 const double* dat2, const double* dat3, const double* dat4,
                 const int32_t* map0, const int32_t* map1) {
  if (!p) return fail(FE_EINVAL, "null plan");
  if (!p->hstream) CUDA_TRY(cudaStreamCreateWithFlags(&p->hstream, cudaStreamNonBlocking));
  int rc = wrap_bind(p, end, dat1, map0, map1, false, p->hstream);
  if (rc) return rc;
  if (start < 0 || end > p->ncells || start > end)
    return fail(FE_EINVAL, "cell range [%d, %d) outside [0, %d)", start, end, p->ncells);
  if (!dat0 || !dat2) return fail(FE_EINVAL, "null dat0/dat2");
  rc = wrap_host_impl(p, start, end, dat0, dat2, dat3, dat4);
  if (rc) {
    // no copy may still read dat2 or write dat0 once the caller sees the error
    for (cudaStream_t q : {p->hstream_u, p->hstream2, p->hstream_d, p->hstream})
      if (q) cudaStreamSynchronize(q);
    cudaGetLastError();
  }
  return rc;
}

}  // extern "C"

static int wrap_host_impl(fe_plan* p, int32_t start, int32_t end, double* dat0, const double* dat2,
                          const double* dat3, const double* dat4) {
  cudaStream_t s = p->hstream;
  const size_t n = (size_t)p->vs * p->nglobal;
  if (p->cap_u < n) {
    cudaFree(p->d_u);
    cudaFree(p->d_y);
    cudaFree(p->d_y0);
    p->d_u = p->d_y = p->d_y0 = nullptr;
    CUDA_TRY(cudaMalloc(&p->d_u, n * sizeof(double)));
    CUDA_TRY(cudaMalloc(&p->d_y, n * sizeof(double)));
    CUDA_TRY(cudaMalloc(&p->d_y0, n * sizeof(double)));
    p->cap_u = n;
  }
  const double* c0 = nullptr;
  const double* c1 = nullptr;
  // the u upload (own stream) is ordered after what is already queued on s,
  // not after the coefficient copies below
  if (!p->ev_u) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_u, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(p->ev_u, s));
  // coefficient fields: mu/lambda vertex fields, or the state u of a
  // linearised form (a dof field with the layout of dat2)
  const bool state = p->form == FE_FORM_NEOHOOKEAN_TANGENT;
  if (state ? dat3 != nullptr : (dat3 && dat4)) {
    const size_t nc = state ? n : (size_t)p->nverts;
    if (p->cap_c < nc) {
      cudaFree(p->d_c0);
      cudaFree(p->d_c1);
      p->d_c0 = p->d_c1 = nullptr;
      CUDA_TRY(cudaMalloc(&p->d_c0, nc * sizeof(double)));
      CUDA_TRY(cudaMalloc(&p->d_c1, nc * sizeof(double)));
      p->cap_c = nc;
    }
    CUDA_TRY(cudaMemcpyAsync(p->d_c0, dat3, nc * sizeof(double), cudaMemcpyHostToDevice, s));
    c0 = p->d_c0;
    if (!state) {
      CUDA_TRY(cudaMemcpyAsync(p->d_c1, dat4, nc * sizeof(double), cudaMemcpyHostToDevice, s));
      c1 = p->d_c1;
    }
  }
  // Pipeline over the 64 blocks of the u / y vector (chunk_mask, found at
  // bind): u is uploaded on its own stream block by block in the order the
  // cell chunks need it; cell chunk r of the operator starts as soon as every
  // block it reads has landed; a block of the result is final once the last
  // cell chunk scattering into it is done and is then downloaded on a third
  // stream while later cell chunks run and the rest of u is still uploading
  // (PCIe is full duplex).  Blocks no cell of [start, end) touches are neither
  // uploaded nor downloaded (dat0 + 0 = dat0).  This holds for any dof
  // numbering: with vertex dofs numbered first, the vertex section and the
  // rest of the vector both stream in cell order.  Accumulate semantics:
  // result blocks whose dat0 is all zero (the common y = A u call, detected on
  // the host while u uploads) are downloaded straight into dat0; the others
  // upload dat0, add on the device, then download.
  constexpr int NCH = FE_HOST_UCHUNKS;  // cell chunks
  static_assert(NCH <= 32, "ev_uc size");
  if (!p->hstream2) {
    CUDA_TRY(cudaStreamCreateWithFlags(&p->hstream2, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->hstream_u, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->hstream_d, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_y0, cudaEventDisableTiming));
    for (int c = 0; c < NCH; ++c) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_uc[c], cudaEventDisableTiming));
    for (int c = 0; c < NCH; ++c) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_cell[c], cudaEventDisableTiming));
  }
  const int64_t bsz = p->hblock;
  const int nblk = bsz > 0 ? (int)((n + bsz - 1) / bsz) : 0;
  const int ncc = (int)p->chunk_cell.size() - 1;
  // cell chunks of this call and the blocks they touch
  uint64_t need[NCH] = {};
  int32_t ca[NCH] = {}, cb[NCH] = {};
  // short vectors (< 4 MB): one chunk -- the fixed cost of the per-chunk copies,
  // events and launches (~0.1 ms per call) outweighs what pipelining hides
  const bool single = n * sizeof(double) < (size_t)4 << 20;
  for (int r = 0; r < ncc && r < NCH; ++r) {
    const int32_t a = std::max(start, p->chunk_cell[r]), b = std::min(end, p->chunk_cell[r + 1]);
    if (a >= b) continue;
    const int k = single ? 0 : r;
    if (need[k] == 0) ca[k] = a;
    cb[k] = b;
    need[k] |= p->chunk_mask[r];
  }
  // maximal runs of set bits of a block mask -> [a, b) entry ranges
  auto for_runs = [&](uint64_t mask, auto&& fn) -> int {
    for (int b0 = 0; b0 < nblk;) {
      if (!((mask >> b0) & 1)) { ++b0; continue; }
      int b1 = b0;
      while (b1 + 1 < nblk && ((mask >> (b1 + 1)) & 1)) ++b1;
      const size_t a = (size_t)b0 * bsz, b = std::min(n, (size_t)(b1 + 1) * bsz);
      if (int rc = fn(a, b)) return rc;
      b0 = b1 + 1;
    }
    return FE_OK;
  };
  // u: the blocks each cell chunk needs that are not on the device yet
  CUDA_TRY(cudaStreamWaitEvent(p->hstream_u, p->ev_u, 0));
  uint64_t have = 0;
  for (int r = 0; r < ncc && r < NCH; ++r) {
    if (ca[r] >= cb[r]) continue;
    int rc = for_runs(need[r] & ~have, [&](size_t a, size_t b) -> int {
      CUDA_TRY(cudaMemcpyAsync(p->d_u + a, dat2 + a, (b - a) * sizeof(double), cudaMemcpyHostToDevice,
                               p->hstream_u));
      return FE_OK;
    });
    if (rc) return rc;
    have |= need[r];
    CUDA_TRY(cudaEventRecord(p->ev_uc[r], p->hstream_u));
  }
  // the operator (it does not read dat0): memset + one launch per cell chunk,
  // each gated on the upload of the blocks it reads
  CUDA_TRY(cudaMemsetAsync(p->d_y, 0, n * sizeof(double), s));
  int last_of[64];
  for (int b = 0; b < 64; ++b) last_of[b] = -1;
  for (int r = 0; r < ncc && r < NCH; ++r) {
    if (ca[r] >= cb[r]) continue;
    CUDA_TRY(cudaStreamWaitEvent(s, p->ev_uc[r], 0));
    static const bool noapply = getenv("FE_HOST_NOAPPLY") != nullptr;  // diagnosis: copy pipeline only
    int rc = noapply ? FE_OK : fe_apply(p, ca[r], cb[r], p->d_y, p->d_u, c0, c1, FE_APPLY_ACCUMULATE, s);
    if (rc) return rc;
    for (int b = 0; b < nblk; ++b)
      if ((need[r] >> b) & 1) last_of[b] = r;
    CUDA_TRY(cudaEventRecord(p->ev_cell[r], s));
  }
  // result blocks in the order they become final (one download stream: a
  // block waiting for the last cell chunk must not hold back the others);
  // runs of blocks finalised by the same cell chunk are one copy.  Scan dat0
  // on the host (all +0.0/-0.0 -> not uploaded), otherwise upload it and add
  // it on the device, then download
  const uint64_t* ybits = reinterpret_cast<const uint64_t*>(dat0);
  static const bool assume_zero = getenv("FE_HOST_ASSUME_ZERO") != nullptr;   // diagnosis (breaks accumulate)
  static const int scan_threads = getenv("FE_HOST_SCAN_THREADS") ? atoi(getenv("FE_HOST_SCAN_THREADS")) : 0;
  for (int r = 0; r < ncc && r < NCH; ++r) {
    uint64_t fin = 0;
    for (int b = 0; b < nblk; ++b)
      if (last_of[b] == r) fin |= 1ull << b;
    if (!fin) continue;
    CUDA_TRY(cudaStreamWaitEvent(p->hstream_d, p->ev_cell[r], 0));
    int rc = for_runs(fin, [&](size_t a, size_t b) -> int {
      int nonzero = 0;
      if (!assume_zero) {
        constexpr int NP = 64;
        const size_t w = (b - a + NP - 1) / NP;
        const int nthr = scan_threads > 0 ? scan_threads : omp_get_max_threads();
#pragma omp parallel for schedule(static) reduction(| : nonzero) num_threads(nthr)
        for (int part = 0; part < NP; ++part) {
          const size_t lo = std::min(b, a + part * w), hi = std::min(b, lo + w);
          uint64_t acc = 0;
          for (size_t k0 = lo; k0 < hi && !acc; k0 += 1024)  // stops at the first nonzero block
            for (size_t k = k0; k < std::min(hi, k0 + 1024); ++k) acc |= ybits[k] << 1;  // drop the sign bit
          nonzero |= acc != 0;
        }
      }
      if (nonzero) {
        CUDA_TRY(cudaMemcpyAsync(p->d_y0 + a, dat0 + a, (b - a) * sizeof(double), cudaMemcpyHostToDevice,
                                 p->hstream2));
        CUDA_TRY(cudaEventRecord(p->ev_y0, p->hstream2));
        CUDA_TRY(cudaStreamWaitEvent(p->hstream_d, p->ev_y0, 0));
        k_add<<<(unsigned)std::min<size_t>((b - a + 255) / 256, 148 * 16), 256, 0, p->hstream_d>>>(
            p->d_y + a, p->d_y0 + a, (int64_t)(b - a));
        CUDA_TRY(cudaGetLastError());
      }
      CUDA_TRY(cudaMemcpyAsync(dat0 + a, p->d_y + a, (b - a) * sizeof(double), cudaMemcpyDeviceToHost,
                               p->hstream_d));
      return FE_OK;
    });
    if (rc) return rc;
  }
  CUDA_TRY(cudaStreamSynchronize(p->hstream_d));
  CUDA_TRY(cudaStreamSynchronize(p->hstream2));
  CUDA_TRY(cudaStreamSynchronize(p->hstream_u));
  CUDA_TRY(cudaStreamSynchronize(s));
  return FE_OK;
}

extern "C" {

int64_t fe_launch_count(void) { return (int64_t)g_launches.load(); }

int fe_eval_log(const double* x, double* y, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return fail(FE_EINVAL, "bad arguments");
  if (n == 0) return FE_OK;
  k_eval_log<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(x, y, n);
  CUDA_TRY(cudaGetLastError());
  return FE_OK;
}

int fe_plan_get_info(const fe_plan* p, fe_plan_info* info) {
  if (!p || !info) return fail(FE_EINVAL, "null argument");
  std::memset(info, 0, sizeof *info);
  std::snprintf(info->kernel, sizeof info->kernel, "%s%s", p->var->name, p->d_macro ? "_macro" : "");
  info->threads_per_cell = 1;
  info->block = p->var->block;
  info->launches_per_apply = 1;
  info->ncells = p->ncells;
  info->nglobal = p->nglobal;
  return FE_OK;
}

void fe_plan_destroy(fe_plan* p) {
  if (!p) return;
  free_mesh(p);
  cudaFree(p->d_tables);
  cudaFree(p->d_diag_tables);
  cudaFree(p->d_lex);
  cudaFree(p->d_u);
  cudaFree(p->d_y);
  cudaFree(p->d_y0);
  cudaFree(p->d_c0);
  cudaFree(p->d_c1);
  if (p->fill_stream) cudaStreamDestroy(p->fill_stream);
  if (p->ev_fill_a) cudaEventDestroy(p->ev_fill_a);
  if (p->ev_fill_b) cudaEventDestroy(p->ev_fill_b);
  if (p->hstream) cudaStreamDestroy(p->hstream);
  if (p->hstream2) cudaStreamDestroy(p->hstream2);
  if (p->ev_u) cudaEventDestroy(p->ev_u);
  if (p->ev_y0) cudaEventDestroy(p->ev_y0);
  for (cudaEvent_t e : p->ev_uc)
    if (e) cudaEventDestroy(e);
  if (p->hstream_u) cudaStreamDestroy(p->hstream_u);
  if (p->hstream_d) cudaStreamDestroy(p->hstream_d);
  for (cudaEvent_t e : p->ev_cell)
    if (e) cudaEventDestroy(e);
  ::operator delete(p->host_params);
  delete p;
}

}  // extern "C"
