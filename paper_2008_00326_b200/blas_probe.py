"""Start-up probe of the host BLAS rounding orders.

Three per-candidate steps of the reference go through numpy -> OpenBLAS, whose
small-matrix kernels FUSE multiply-adds in an order that depends on the operand
layout (geometry.py:131-145: `apply`, `compose`, `inverse`).  The device code
bakes those orders in (csrc/px_common.cuh: dot_f012 / dot_f102) and the host
planner relies on them when it builds candidate poses with batched matmuls
(proposals.compose_grid).  They are a property of the numpy / BLAS build
(DYNAMIC_ARCH kernels), so the first search of a process checks them on random
operands against correctly rounded fused chains and fails LOUDLY if this host
rounds differently -- candidate bits, and with them the z-buffer ownership,
would otherwise diverge silently from the device's.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from .errors import DeviceError


class BlasOrderError(DeviceError):
    """The host numpy/BLAS does not round 3x3 products the way libpx assumes."""


def _fma(a: float, b: float, c: float) -> float:
    """Correctly rounded a*b + c (exact rational arithmetic, one rounding)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def dot_f012(a, b) -> float:
    """fma(a2,b2, fma(a1,b1, a0*b0)): numpy mat@mat, (V,3)@R.T, transposed-view @ vec."""
    return _fma(a[2], b[2], _fma(a[1], b[1], a[0] * b[0]))


def dot_f102(a, b) -> float:
    """fma(a2,b2, fma(a0,b0, a1*b1)): numpy C-contiguous (3,3) @ (3,)."""
    return _fma(a[2], b[2], _fma(a[0], b[0], a[1] * b[1]))


def _mismatches(trials: int, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    bad = {"matmat_f012": 0, "matvec_contig_f102": 0, "matvec_view_f012": 0, "apply_f012": 0, "batched_equals_item": 0}
    for _ in range(trials):
        a = np.ascontiguousarray(rng.normal(size=(3, 3)))
        b = np.ascontiguousarray(rng.normal(size=(3, 3)))
        v = rng.normal(size=3)
        pts = rng.normal(size=(5, 3))
        mm = a @ b
        mv = a @ v
        view = np.ascontiguousarray(a.T).T  # non-contiguous rotation, as RigidTransform.inverse() produces
        mvv = view @ v
        ap = pts @ a.T
        for i in range(3):
            for j in range(3):
                bad["matmat_f012"] += mm[i, j] != dot_f012(a[i], b[:, j])
            bad["matvec_contig_f102"] += mv[i] != dot_f102(a[i], v)
            bad["matvec_view_f012"] += mvv[i] != dot_f012(view[i], v)
        for p in range(pts.shape[0]):
            for i in range(3):
                bad["apply_f012"] += ap[p, i] != dot_f012(pts[p], a[i])
        stack = rng.normal(size=(4, 3, 3))
        bad["batched_equals_item"] += not all(np.array_equal(np.matmul(a, stack)[k], a @ stack[k]) for k in range(4))
    return bad


_checked = None


def check_blas_orders(trials: int = 24, seed: int = 20080326, force: bool = False) -> dict:
    """Raise BlasOrderError unless this host's numpy reproduces the fused orders
    the device code assumes; the (cached) mismatch counts otherwise."""
    global _checked
    if _checked is not None and not force:
        return _checked
    bad = _mismatches(trials, seed)
    if any(bad.values()):
        import numpy.__config__ as cfg  # noqa: F401
        raise BlasOrderError(
            "host numpy/BLAS rounds small matrix products in an order libpx does not reproduce "
            f"(mismatches over {trials} random trials: {bad}); candidate poses built on this host would "
            "differ in their last bits from the device's compositions (SURVEY.md 7.3 H2). "
            "Use a numpy whose BLAS matches (OpenBLAS 0.3.x AVX2/AVX-512 kernels) or rebuild libpx with "
            "the observed orders in csrc/px_common.cuh.")
    _checked = bad
    return bad
