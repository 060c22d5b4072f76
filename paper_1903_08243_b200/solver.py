"""Matrix-free Krylov driver around the operator (the
caller side of the hot path -- the reference has no solver at all).

* :func:`cg` -- preconditioned conjugate gradients on device tensors; every
  iteration is ONE operator application (``apply(u, y)``: y = A u, e.g.
  ``GpuKernelHandle.apply(..., overwrite=True)`` or
  :meth:`DistributedOperator.apply`) plus five vector updates and two dot
  products.  No host synchronisation inside the loop other than the
  convergence check every ``check_every`` iterations.
* :class:`SlabDot` -- the dot product of the z-slab partition
  (``distributed.py``): both neighbouring ranks hold the shared interface
  plane (the operator sums it on both sides, so vectors stay consistent
  without a ghost update), so the upper rank's copy of its bottom plane is
  weighted 0 and the local sums are all-reduced over NCCL (gloo on CPU).
* :func:`jacobi` -- inverse operator diagonal (``GpuKernelHandle.diagonal``,
  fe_diagonal), interface entries summed across ranks like the action.

Symmetric positive definite forms: mass, Helmholtz, Lame elasticity (with
constraints), the neo-Hookean tangent near a stable state.
"""

from __future__ import annotations

from dataclasses import dataclass, field

__all__ = ["cg", "CGInfo", "SlabDot", "jacobi"]


@dataclass
class CGInfo:
    iterations: int = 0
    converged: bool = False
    residuals: list = field(default_factory=list)   # ||r|| / ||b|| at each check


def _local_dot(a, b):
    return (a * b).sum()


def cg(apply, b, x=None, rtol=1e-10, maxiter=1000, precond=None, dot=None, check_every=1):
    """Solve A x = b.  ``apply(u, y)`` overwrites y with A u; ``precond`` is a
    tensor (multiplied elementwise: Jacobi's inverse diagonal) or a callable
    z = M^-1 r, or None; ``dot(a, b)`` returns a 0-d tensor (default: local
    sum -- pass a :class:`SlabDot` on a partitioned mesh).  Returns (x, info)."""
    import torch
    dot = dot or _local_dot
    if x is None:
        x = torch.zeros_like(b)
    r = torch.empty_like(b)
    q = torch.empty_like(b)
    apply(x, q)
    torch.sub(b, q, out=r)

    def prec(v):
        if precond is None:
            return v.clone()
        if callable(precond):
            return precond(v)
        return precond * v

    z = prec(r)
    p = z.clone()
    rz = dot(r, z)
    bnorm = float(torch.sqrt(dot(b, b)))
    info = CGInfo()
    if bnorm == 0.0:
        x.zero_()
        info.converged = True
        return x, info
    for it in range(1, maxiter + 1):
        apply(p, q)
        alpha = rz / dot(p, q)
        x.add_(alpha * p)
        r.sub_(alpha * q)
        if it % check_every == 0 or it == maxiter:
            rel = float(torch.sqrt(dot(r, r))) / bnorm
            info.residuals.append(rel)
            if rel <= rtol:
                info.iterations = it
                info.converged = True
                return x, info
        z = prec(r)
        rz_new = dot(r, z)
        p.mul_(rz_new / rz).add_(z)
        rz = rz_new
    info.iterations = maxiter
    return x, info


class SlabDot:
    """Global dot product on the z-slab partition (distributed.py): local
    sums with each shared interface entry counted once (owned by the lower
    rank), all-reduced over ``torch.distributed``."""

    def __init__(self, slab, rank: int, world: int):
        vs = slab.spec.element.value_size
        self.skip = ([(vs * a, vs * b) for a, b in slab.interface_ranges("below")]
                     if (slab.has_below and world > 1) else [])
        self.world = world

    def __call__(self, a, b):
        import torch.distributed as dist
        s = (a * b).sum()
        for lo, hi in self.skip:                 # the lower rank owns the shared plane
            s = s - (a[lo:hi] * b[lo:hi]).sum()
        if self.world > 1:
            dist.all_reduce(s)
        return s


def jacobi(diag, op=None):
    """Inverse diagonal for :func:`cg` (``diag`` from
    ``GpuKernelHandle.diagonal``).  With a :class:`DistributedOperator` the
    interface entries are first summed with the neighbours, exactly like the
    operator's own output."""
    if op is not None and op.world > 1:
        op.exchange(diag)
    return 1.0 / diag
