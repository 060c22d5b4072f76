"""Parity of the sm_100a path with the reference (golden vectors) and the
CPU oracle, through the C ABI.  North-star tolerance: relative L2 <= 1e-12
in FP64 (BASELINE.json)."""

import numpy as np
import pytest

import paper_1903_08243_b200 as fe
from paper_1903_08243_b200 import configs as C
from oracle import fe_oracle as fo

pytestmark = pytest.mark.gpu
TOL = 1e-12


def oracle_fn(spec, mesh, dm, rule, u, mu=None, lam=None, start=0, end=None, state=None):
    P = fo.Problem(spec.form, spec.cell.kind, spec.element.degree, rule.exactness_degree, spec.params)
    return fo.assemble(P, mesh.coords, mesh.cell2vert, dm.cell2dof, u, mu, lam, start, end,
                       state=state)


def handle_for(spec, rule, generic=False):
    return fe.compile_and_load(fe.emit_for(spec, fe.Target(generic=generic), rule))


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("idx", range(32))
def test_gpu_matches_reference_golden(golden2d, idx, generic):
    name = str(golden2d["names"][idx])
    form, cell, deg = name.split("_")
    g = lambda k: golden2d[f"{name}/{k}"]
    spec = fe.operator_spec(form, cell, int(deg))
    rule = fe.quadrature_rule(cell, fe.integrand_degree(spec))
    h = handle_for(spec, rule, generic)
    out = np.zeros_like(g("y"))
    b = {"dat0": out, "dat1": g("coords").ravel(), "dat2": g("u"),
         "map0": g("cell2dof").ravel(), "map1": g("cell2vert").ravel()}
    h(0, len(g("cell2vert")), b)
    assert fe.harness.rel_l2(out, g("y")) <= TOL, (name, h.info)


def test_gpu_c1_full_size_matches_reference(golden_c1):
    prob = C.build_problem(C.get_config("C1"), 0)
    h = handle_for(prob.spec, prob.rule)
    out = np.zeros(prob.ndofs)
    h(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out))
    assert fe.harness.rel_l2(out, golden_c1["y"]) <= TOL


CONFIG_CASES = [
    ("C1", 16), ("C2-P1", 5), ("C2-P2", 5), ("C2-P3", 4), ("C2-P4", 3),
    ("C3-Q1", 5), ("C3-Q2", 4), ("C3-Q3", 3), ("C3-Q4", 3), ("C3-Q5", 2), ("C3-Q6", 2),
    ("C4-quad-Q1", 12), ("C4-quad-Q2", 10), ("C4-quad-Q3", 8), ("C4-quad-Q4", 6),
    ("C4-hex-Q1", 4), ("C4-hex-Q2", 3), ("C4-hex-Q3", 3), ("C5", 4), ("C6", 4),
]


def _supported(name):
    cfg = C.get_config(name)
    spec = fe.operator_spec(cfg.form, cfg.cell, cfg.degree)
    try:
        handle_for(spec, fe.quadrature_rule(cfg.cell, cfg.qdegree))
        return True
    except fe.ToolchainError:
        return False


@pytest.mark.parametrize("name,n", CONFIG_CASES)
def test_gpu_matches_oracle_on_config(name, n):
    prob = C.build_problem(C.get_config(name, n), seed=1)
    if not _supported(name):
        pytest.xfail(f"no sm_100a kernel for {name} yet")
    h = handle_for(prob.spec, prob.rule)
    ref = oracle_fn(prob.spec, prob.mesh, prob.dofmap, prob.rule, prob.u, prob.mu, prob.lam,
                    state=prob.state)
    out = np.zeros(prob.ndofs)
    h(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out, prob.mu, prob.lam,
                                            state=prob.state))
    assert fe.harness.rel_l2(out, ref) <= TOL, (name, h.info, fe.harness.rel_l2(out, ref))


@pytest.mark.parametrize("name", ["C1", "C2-P1", "C2-P2", "C2-P3", "C3-Q3", "C5", "C6"])
def test_arbitrary_cell_ranges(name):
    """Any [start, end) must be honoured (the reference's batched targets get
    unaligned start wrong)."""
    prob = C.build_problem(C.get_config(name, 3 if name != "C1" else 8), seed=2)
    h = handle_for(prob.spec, prob.rule)
    nc = prob.mesh.ncells
    for start, end in [(1, nc), (0, 1), (7, 7), (3, nc - 5), (nc - 1, nc), (6, 12), (5, 13),
                       (12, nc)]:
        ref = oracle_fn(prob.spec, prob.mesh, prob.dofmap, prob.rule, prob.u, prob.mu, prob.lam,
                        start, end, state=prob.state)
        out = np.zeros(prob.ndofs)
        h(start, end, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out, prob.mu, prob.lam,
                                       state=prob.state))
        if end == start:
            assert not out.any()
        else:
            assert fe.harness.rel_l2(out, ref) <= TOL, (start, end)


def _macro_problem(seed):
    prob = C.build_problem(C.get_config("C2-P1", 3), seed=seed)
    h = handle_for(prob.spec, prob.rule)
    return prob, h


def test_macro_cell_path_is_detected_and_matches_oracle():
    """The Kuhn-cube macro-cell kernel (C2-P1) is selected on the structured
    tet mesh and agrees with the oracle."""
    prob, h = _macro_problem(7)
    out = np.zeros(prob.ndofs)
    h(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out))
    assert h.info["kernel"] == "element_split_macro"
    ref = oracle_fn(prob.spec, prob.mesh, prob.dofmap, prob.rule, prob.u)
    assert fe.harness.rel_l2(out, ref) <= TOL


def test_macro_cell_path_falls_back_on_other_cell_orders():
    """Cells that do not follow the macro pattern (here: a cell permutation)
    must run the per-cell kernel, with the same result."""
    prob, h = _macro_problem(8)
    rng = np.random.default_rng(0)
    perm = rng.permutation(prob.mesh.ncells)
    mesh = fe.Mesh(prob.mesh.coords, np.ascontiguousarray(prob.mesh.cell2vert[perm]), prob.mesh.cell)
    dm = fe.DofMap(np.ascontiguousarray(prob.dofmap.cell2dof[perm]), prob.dofmap.ndofs_global,
                   prob.dofmap.element)
    out = np.zeros(prob.ndofs)
    h(0, mesh.ncells, fe.make_bindings(mesh, dm, prob.u, out))
    assert h.info["kernel"] == "element_split"
    ref = oracle_fn(prob.spec, mesh, dm, prob.rule, prob.u)
    assert fe.harness.rel_l2(out, ref) <= TOL


def test_accumulate_semantics():
    """dat0 is accumulated, not overwritten (reference codegen.py:168-169)."""
    prob = C.build_problem(C.get_config("C2-P2", 3), seed=3)
    h = handle_for(prob.spec, prob.rule)
    ref = oracle_fn(prob.spec, prob.mesh, prob.dofmap, prob.rule, prob.u)
    out = np.full(prob.ndofs, 0.5)
    h(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out))
    assert fe.harness.rel_l2(out - 0.5, ref) <= TOL


@pytest.mark.parametrize("name", ["C2-P3", "C5", "C6"])
def test_device_path_matches_host_path(name):
    import torch
    prob = C.build_problem(C.get_config(name, 3), seed=4)
    h = handle_for(prob.spec, prob.rule)
    host = np.zeros(prob.ndofs)
    h(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, host, state=prob.state))
    b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, np.zeros(prob.ndofs), state=prob.state)
    d = {k: torch.as_tensor(v, device="cuda") for k, v in b.items()}
    h(0, prob.mesh.ncells, d)
    torch.cuda.synchronize()
    assert fe.harness.rel_l2(d["dat0"].cpu().numpy(), host) <= 1e-14


def test_fault_injection_is_detected():
    """Perturb one map entry (cli.py --inject-fault analogue): parity must fail."""
    prob = C.build_problem(C.get_config("C2-P2", 3), seed=5)
    h = handle_for(prob.spec, prob.rule)
    ref = oracle_fn(prob.spec, prob.mesh, prob.dofmap, prob.rule, prob.u)
    b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, np.zeros(prob.ndofs))
    bad = b["map0"].copy()
    bad[5], bad[6] = bad[6], bad[5]
    b["map0"] = bad
    h(0, prob.mesh.ncells, b)
    assert fe.harness.rel_l2(b["dat0"], ref) > 1e-6
    with pytest.raises(fe.VerificationError):
        fe.verify_target(prob.spec, fe.Target(), prob.mesh,
                         type(prob.dofmap)(bad.reshape(prob.dofmap.cell2dof.shape), prob.nglobal,
                                           prob.spec.element),
                         prob.rule, h, prob.u, TOL,
                         lambda s, m, dm, r, u, mu, lam: ref)


def test_out_of_range_map_is_rejected():
    prob = C.build_problem(C.get_config("C2-P1", 2), seed=6)
    h = handle_for(prob.spec, prob.rule)
    b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, np.zeros(prob.ndofs))
    bad = b["map0"].copy()
    bad[3] = prob.nglobal + 10
    b["map0"] = bad
    with pytest.raises(fe.jit.KernelError, match="out of range"):
        h(0, prob.mesh.ncells, b)


def test_run_configuration_verifies_and_times():
    prob = C.build_problem(C.get_config("C2-P2", 6), seed=0)
    rec = fe.run_configuration(prob.spec, fe.Target(), prob.mesh, prob.dofmap, trials=5,
                               rule=prob.rule, oracle=oracle_fn, u=prob.u)
    assert rec.parity_rel_l2 <= TOL and rec.time_best_s > 0 and rec.gflops > 0


@pytest.mark.parametrize("name", ["C2-P2", "C2-P4", "C3-Q2", "C4-hex-Q1", "C5"])
def test_gpu_on_slab_numbering_with_separate_vertex_map(name):
    """Slab-local lattice numbering (distributed.py): dof ids are NOT vertex
    ids, so the plan must keep the separate vertex map (map1)."""
    import torch
    from paper_1903_08243_b200.distributed import build_slab
    cfg = C.get_config(name, (3, 2, 2))
    s = build_slab(cfg, 5, 0, 2, 4)
    h = handle_for(s.spec, s.rule)
    out = np.zeros(s.ndofs)
    h(0, s.mesh.ncells, fe.make_bindings(s.mesh, s.dofmap, s.u, out, s.mu, s.lam))
    ref = oracle_fn(s.spec, s.mesh, s.dofmap, s.rule, s.u, s.mu, s.lam)
    assert fe.harness.rel_l2(out, ref) <= TOL


def test_missing_vertex_map_with_non_vertex_numbering_is_rejected():
    """Without map1 the plan takes map0[:, :nv] as the vertex map; a dof
    numbering whose vertex columns are not vertex ids must be rejected
    (out-of-range coordinate index), not read out of bounds."""
    import torch
    prob = C.build_problem(C.get_config("C2-P2", (3, 2, 2)), 5)
    perm = np.random.default_rng(0).permutation(prob.dofmap.ndofs_global)   # vertex dofs not first
    c2d = perm[np.asarray(prob.dofmap.cell2dof)].astype(np.int32)
    assert c2d[:, :4].max() >= prob.mesh.nvertices
    h = handle_for(prob.spec, prob.rule)
    dev = torch.device("cuda")
    with pytest.raises(fe.jit.KernelError, match="out of range"):
        h.bind(torch.tensor(np.asarray(prob.mesh.coords).ravel(), device=dev),
               torch.tensor(c2d.ravel(), device=dev), None, nglobal=prob.dofmap.ndofs_global)


def test_tangent_needs_the_state():
    prob = C.build_problem(C.get_config("C6", 2), seed=9)
    h = handle_for(prob.spec, prob.rule)
    b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, np.zeros(prob.ndofs))
    with pytest.raises(KeyError):
        h(0, prob.mesh.ncells, b)


def test_tangent_matches_central_difference_of_gpu_residual():
    """GPU-only consistency: the tangent kernel (C6) against central
    differences of the GPU residual kernel (C5) at the same state."""
    prob = C.build_problem(C.get_config("C6", 3), seed=10)
    res_spec = fe.operator_spec("neohookean", "tetrahedron", 2)
    hr = handle_for(res_spec, prob.rule)
    ht = handle_for(prob.spec, prob.rule)
    eps = 1e-3 * 0.01 / 3

    def residual(u):
        out = np.zeros(prob.ndofs)
        hr(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, u, out))
        return out

    fd = (residual(prob.state + eps * prob.u) - residual(prob.state - eps * prob.u)) / (2 * eps)
    out = np.zeros(prob.ndofs)
    ht(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out, state=prob.state))
    assert fe.harness.rel_l2(out, fd) < 1e-6


@pytest.mark.parametrize("name,size", [("C2-P1", 32), ("C2-P4", 12), ("C4-quad-Q2", 160), ("C5", 16)])
def test_host_entry_mixed_zero_chunks(name, size):
    """Host entry (fe_wrap_host): result chunks whose dat0 is all zero are
    downloaded directly, the others are uploaded and accumulated, and each
    result chunk is downloaded as soon as its last cell chunk is done.  dat0
    here mixes zero, -0.0 and nonzero chunks; a cell sub-range is applied
    too (accumulate semantics, reference codegen.py:168-169)."""
    prob = C.build_problem(C.get_config(name, size), seed=6)
    h = handle_for(prob.spec, prob.rule)
    mu, lam = getattr(prob, "mu", None), getattr(prob, "lam", None)
    ref_full = oracle_fn(prob.spec, prob.mesh, prob.dofmap, prob.rule, prob.u, mu, lam,
                         state=prob.state)
    out = np.zeros_like(ref_full)
    flat = out.reshape(-1)
    m = flat.size
    rng = np.random.default_rng(1)
    y0 = np.zeros(m)
    y0[m // 8: m // 4] = rng.uniform(-1, 1, m // 4 - m // 8)   # one nonzero stripe
    y0[m // 2] = 3.0                                              # a single nonzero entry
    y0[-(m // 8):] = -0.0                                         # negative zeros
    flat[:] = y0
    h(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out, mu, lam, state=prob.state))
    assert fe.harness.rel_l2(out.reshape(-1) - y0, ref_full.reshape(-1)) <= TOL
    # sub-range [0, half): zero dat0, then the second half accumulated on top
    out2 = np.zeros_like(ref_full)
    half = prob.mesh.ncells // 2
    b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out2, mu, lam, state=prob.state)
    h(0, half, b)
    h(half, prob.mesh.ncells, b)
    assert fe.harness.rel_l2(out2, ref_full) <= TOL
