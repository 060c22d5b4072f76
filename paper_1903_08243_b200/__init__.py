"""B200-native matrix-free finite-element operator action
y = sum_e P_e^T A_e(P_e u), behind the reference ``fevec`` operator API
(``/root/reference/pkg/src/fevec/__init__.py:10-44``).

Host code (this package) builds meshes, dof maps, element tables and plans;
every apply runs hand-written sm_100a FP64 kernels in ``libfeb200.so``
through the C ABI of ``include/fe_b200.h``.  There is no CPU fallback.
"""

from .elements import (
    OPERATOR_FORMS,
    OperatorSpec,
    QuadratureRule,
    ReferenceElement,
    integrand_degree,
    lagrange_nodes,
    monomial_integral,
    operator_spec,
    quadrature_rule,
    reference_cell,
    reference_element,
    tabulate,
    tensor_factors,
)
from .harness import (
    BenchmarkRecord,
    CSV_COLUMNS,
    VerificationError,
    arithmetic_intensity,
    bytes_per_cell,
    flops_per_cell,
    make_bindings,
    random_coefficients,
    roofline_rows,
    run_configuration,
    verify_target,
    write_csv,
)
from .jit import (GpuKernelHandle, KernelError, PlanUnit, Target, ToolchainError, compile_and_load,
                  emit_for)
from . import solver
from .mesh import DofMap, Mesh, build_dof_map, build_mesh, jitter_mesh

__version__ = "0.1.0"
