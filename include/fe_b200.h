/*
 * fe_b200.h -- C ABI of the B200-native matrix-free finite-element operator
 * action  y += sum_{e in [start,end)} P_e^T A_e(P_e u).
 *
 * This is the drop-in boundary for the reference's hot loop.  The reference
 * (fevec) emits one C function per form and calls it through ctypes:
 *
 *   void wrap_<form>(int const start, int const end,
 *                    double *__restrict__ dat0,          // output, accumulated
 *                    double const *__restrict__ dat1,    // vertex coordinates
 *                    double const *__restrict__ dat2,    // coefficient u
 *                    int const *__restrict__ map0,       // cell -> dof map
 *                    int const *__restrict__ map1);      // cell -> vertex map
 *
 *   (/root/reference/pkg/src/fevec/codegen.py:375-428, contract
 *    /root/reference/SPEC.md:318; called from jit.py:71-87 KernelHandle)
 *
 * Here the per-form tables that the reference bakes into the emitted source
 * as `static const` arrays (codegen.py:409-424) are handed to
 * fe_plan_create() instead, the mesh (dat1/map0/map1, which never change
 * between applies) is bound once with fe_plan_bind_mesh() and re-laid out
 * for the GPU (element-batched SoA maps, padded coordinates), and
 * fe_wrap()/fe_wrap_host() keep the reference's positional argument order.
 *
 * Semantics (reference bench.py:196-201, codegen.py:168-169): the output is
 * ACCUMULATED; the caller zeroes it.  Any [start, end) is honoured
 * (the reference's batched targets require width-aligned start,
 * transforms.py:304-308; this ABI does not).
 *
 * Buffers: dat0/dat2 are [value_size * ndofs] doubles, node-major,
 * component-fastest (reference SPEC.md:98); dat1 is [nverts][dim] doubles;
 * map0 is [ncells][ndof] int32, map1 is [ncells][nvert] int32, both
 * row-major as the reference builds them (bench.py:94-101).  For
 * elasticity_lame, dat3/dat4 are the vertex-valued mu/lambda fields
 * [nverts] read through map1.
 *
 * Errors: every entry point returns 0 on success, a positive FE_E* code on
 * failure; fe_last_error() returns a thread-local message.  No entry point
 * ever falls back to a CPU implementation.
 */
#ifndef FE_B200_H
#define FE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FE_ABI_VERSION 1

/* forms: reference forms first (elements.py:28), then the B200 extensions */
enum {
  FE_FORM_MASS = 0,
  FE_FORM_HELMHOLTZ = 1,
  FE_FORM_LAPLACIAN = 2,         /* vector Laplacian, value_size = dim (reference) */
  FE_FORM_ELASTICITY = 3,        /* eps(u):grad v, value_size = dim (reference) */
  FE_FORM_LAPLACIAN_SCALAR = 4,  /* grad u . grad v */
  FE_FORM_ELASTICITY_LAME = 5,   /* 2 mu eps(u):eps(v) + lambda div u div v */
  FE_FORM_NEOHOOKEAN = 6,        /* P(F) : grad v, P = mu(F - F^-T) + lambda ln J F^-T */
  FE_FORM_NEOHOOKEAN_TANGENT = 7 /* dP(F)[grad du] : grad v at the state u (coef0, same
                                    layout as u): mu dF + (mu - lambda ln J) F^-T dF^T F^-T
                                    + lambda tr(F^-1 dF) F^-T, the Newton-step operator of
                                    FE_FORM_NEOHOOKEAN */
};

enum {
  FE_CELL_TRIANGLE = 0,
  FE_CELL_QUADRILATERAL = 1,
  FE_CELL_TETRAHEDRON = 2,
  FE_CELL_HEXAHEDRON = 3
};

/* error codes */
enum {
  FE_OK = 0,
  FE_EINVAL = 1,        /* bad argument */
  FE_EUNSUPPORTED = 2,  /* no kernel for this (form, cell, degree, rule) */
  FE_ECUDA = 3,         /* CUDA runtime error */
  FE_ENOMESH = 4,       /* apply before fe_plan_bind_mesh */
  FE_ENOMEM = 5
};

/* fe_plan_bind_mesh flags */
#define FE_PTR_HOST 0u     /* coords/maps are host pointers */
#define FE_PTR_DEVICE 1u   /* coords/maps are device pointers */

/* fe_apply flags */
#define FE_APPLY_ACCUMULATE 0u  /* dat0 += A(u)  (reference semantics) */
#define FE_APPLY_OVERWRITE 1u   /* dat0 = A(u) restricted to [start,end) cells */

/* Everything the reference bakes into wrap_<form> as static tables
 * (kernels.py:97-108: qw, phi, dphi0/1, gphi0/1) plus the tensor-product
 * factors used by the sum-factorised kernels on quadrilaterals/hexahedra. */
typedef struct fe_element_desc {
  int32_t form, cell, degree, value_size;
  int32_t ndof;            /* scalar local dofs per cell */
  int32_t nvert;           /* vertices per cell (degree-1 geometry) */
  int32_t nq;              /* quadrature points */
  const double* qweights;  /* [nq] */
  const double* phi;       /* [nq][ndof]       basis values */
  const double* dphi;      /* [nq][ndof][dim]  reference gradients */
  const double* gphi;      /* [nq][nvert]      geometry basis values */
  const double* gdphi;     /* [nq][nvert][dim] geometry reference gradients */
  /* tensor cells only (else q1d = 0 and NULL pointers) */
  int32_t q1d;             /* 1D Gauss points per direction */
  const double* B1d;       /* [q1d][degree+1] 1D basis values at 1D points */
  const double* D1d;       /* [q1d][degree+1] 1D basis derivatives */
  const double* w1d;       /* [q1d] 1D weights on [0,1] */
  const double* x1d;       /* [q1d] 1D Gauss points on [0,1] */
  const int32_t* lex;      /* [(degree+1)^dim] local node index of tensor node (x fastest) */
  double params[4];        /* neohookean: mu, lambda */
  /* optional stiffness factorisation (else nq_aux = 0): weights w and
   * reference gradients G such that int dphi_i/dxi_a dphi_j/dxi_b =
   * sum_r w_r G[r][i][a] G[r][j][b] on the reference simplex -- a rule exact
   * for degree 2k-2, or its minimal-rank form (m = dim P_{k-1} modes,
   * elements.stiffness_modes).  Used by the split and modal DMMA
   * Helmholtz/Laplacian kernels of affine simplices. */
  int32_t nq_aux;
  const double* qw_aux;    /* [nq_aux] */
  const double* dphi_aux;  /* [nq_aux][ndof][dim] */
} fe_element_desc;

typedef struct fe_plan fe_plan;

typedef struct fe_plan_info {
  char kernel[64];         /* name of the kernel family selected */
  int32_t threads_per_cell;
  int32_t block;           /* threads per CTA */
  int32_t launches_per_apply;
  int64_t ncells;
  int64_t nglobal;         /* scalar dofs bound */
} fe_plan_info;

int fe_abi_version(void);

/* Create a plan for one (form, cell, degree, rule); uploads its tables. */
int fe_plan_create(fe_plan** plan, const fe_element_desc* desc, uint32_t flags);

/* Bind (and re-lay out on the device) the mesh: coordinates [nverts][dim],
 * map0 [ncells][ndof], map1 [ncells][nvert] (may be NULL when
 * map0[:, :nvert] is the vertex map, as in every reference numbering,
 * mesh.py:95).  nglobal = scalar dof count. */
int fe_plan_bind_mesh(fe_plan* plan, int32_t ncells, int32_t nverts, int64_t nglobal,
                      const double* coords, const int32_t* map0, const int32_t* map1,
                      uint32_t ptr_flags, void* stream);

/* Device apply on the bound mesh: dat0 (+)= sum over cells in [start,end).
 * coef0/coef1: device vertex fields mu/lambda for elasticity_lame; for
 * neohookean_tangent coef0 is the state u (vs*nglobal doubles, the layout of
 * dat2) and coef1 is NULL; else both NULL.
 * stream: a cudaStream_t (NULL = legacy default stream). */
int fe_apply(const fe_plan* plan, int32_t start, int32_t end, double* dat0,
             const double* dat2, const double* coef0, const double* coef1,
             uint32_t apply_flags, void* stream);

/* Reference-order entry on DEVICE pointers: (start, end, dat0, dat1, dat2,
 * dat3, dat4, map0, map1) -- the drop-in for wrap_<form>, which receives the
 * mesh with every call and no sizes (codegen.py:375-394).  When dat1/map0/
 * map1 differ from the bound buffers (or were bound as host pointers), the
 * mesh is (re-)bound first: cells [0, end), nglobal = max(map0) + 1, nverts =
 * max(vertex map) + 1, derived from the maps (a mesh bound implicitly this
 * way is re-bound again when a later call passes a larger end).  A mesh bound
 * explicitly by fe_plan_bind_mesh with the same buffers is used as is.
 * dat3/dat4 may be NULL. */
int fe_wrap(fe_plan* plan, int32_t start, int32_t end, double* dat0,
            const double* dat1, const double* dat2, const double* dat3,
            const double* dat4, const int32_t* map0, const int32_t* map1, void* stream);

/* Reference-order entry on HOST pointers (the drop-in for a ctypes caller
 * holding numpy buffers): uploads dat2 (+ dat3/dat4), applies, and
 * returns dat0 + A(u) in dat0; synchronous.  The u / dat0 vector is handled
 * in 64 blocks: u blocks are uploaded in the order the cell chunks of the
 * operator read them (a per-chunk block mask found at bind), each result
 * block is downloaded as soon as the last cell chunk scattering into it is
 * done, and blocks no cell of [start, end) touches move in neither direction.
 * dat0 is scanned per block run on the host: all-zero runs (+0.0 / -0.0) are
 * not uploaded, the others are uploaded and accumulated on the device.  The
 * mesh is
 * (re-)bound exactly as in fe_wrap when dat1/map0/map1 differ from the bound
 * HOST buffers.  [start, end) outside [0, ncells) -> FE_EINVAL before any
 * copy is queued; on any error every copy of the call has completed before
 * the function returns (nothing still reads dat2 or writes dat0). */
int fe_wrap_host(fe_plan* plan, int32_t start, int32_t end, double* dat0,
                 const double* dat1, const double* dat2, const double* dat3,
                 const double* dat4, const int32_t* map0, const int32_t* map1);

int fe_plan_get_info(const fe_plan* plan, fe_plan_info* info);

/* Operator diagonal on the bound mesh (Jacobi preconditioner
 * of a matrix-free solve): diag (+)= sum over cells in [start,end) of
 * P_e^T diag(A_e), vs*nglobal doubles in the layout of dat2.  Linear forms
 * only (and neohookean_tangent at the state coef0); FE_EUNSUPPORTED for the
 * nonlinear residual.  Same coef0/coef1/flags/stream meaning as fe_apply.
 * A one-time setup kernel: it recomputes the reference quadrature per local
 * dof (cost ~ ndof x apply). */
int fe_diagonal(const fe_plan* plan, int32_t start, int32_t end, double* diag,
                const double* coef0, const double* coef1, uint32_t apply_flags, void* stream);

/* Thread safety: fe_apply / fe_wrap / fe_diagonal build their kernel
 * parameter block per call, so concurrent calls on one plan from several
 * host threads (different streams, disjoint dat0) are safe; binding
 * (fe_plan_bind_mesh, or an implicit re-bind in fe_wrap*) and fe_wrap_host
 * (which owns the plan's staging buffers) must not run concurrently with
 * other calls on the same plan. */

/* Diagnostics: y[i] = ln x[i] with the branch-free logarithm the
 * hyperelastic kernels use (device pointers; exposes its special-value
 * behaviour to tests: +inf -> +inf, +-0 -> -inf, x < 0 / NaN -> NaN,
 * subnormals rescaled). */
int fe_eval_log(const double* x, double* y, int64_t n, void* stream);

/* Number of operator / diagonal kernels this library has launched in the
 * process (fe_apply, fe_wrap*, fe_diagonal; not the bind-time layout
 * kernels): bench.py's gpu_launches is the difference around its timed
 * region. */
int64_t fe_launch_count(void);

void fe_plan_destroy(fe_plan* plan);

const char* fe_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FE_B200_H */
