"""TU/TURBO Schur-update driver on one Morton-hybrid parent.

TURBO/TU decomposition spends its time in Schur-complement
updates  A22 <- A22 - A21 * A12  on views of ONE matrix whose origins follow the
recursion and are generally not tile-aligned.  The reference multiply forbids
views of the same container (multiply.hpp:59-60); this driver uses the GPU
engine's alias mode (snapshot semantics: operands are packed before the output
is written) and replays each update as a CUDA graph.

`schur_sweep` runs the update sequence of a right-looking block elimination
with panel width `block` (the panel factorisation / triangular solves of TU are
outside the hot path and outside this repo):

    for k0 = 0, block, 2*block, ...:   A[k1:, k1:] -= A[k1:, k0:k1] * A[k0:k1, k1:]

`SweepGraph` captures a whole sweep (every step's pack + GEMM) into ONE CUDA graph,
so a repeated sweep is a single launch: no host work between the steps (from Python
each plan launch costs tens of microseconds, more than the last steps' GPU time).
"""
from __future__ import annotations

from typing import List

from . import OP_SUB, Matrix, Plan, Problem, Sub, encode


def schur_views(M: Matrix, block: int):
    """(out, lhs, rhs) view triples of the sweep, in order."""
    lay = M.layout()
    n = lay.n
    if block <= 0:
        raise ValueError("block must be positive")
    out = []
    k0 = 0
    while k0 + block < n:
        k1 = k0 + block
        rest = n - k1
        out.append(Problem(Sub(M, encode(lay, k1, k1), rest, rest),
                           Sub(M, encode(lay, k1, k0), rest, block),
                           Sub(M, encode(lay, k0, k1), block, rest)))
        k0 = k1
    return out


def schur_plans(M: Matrix, block: int, op: int = OP_SUB) -> List[Plan]:
    """One planned (graph-replayed) aliased update per elimination step."""
    return [Plan(p, op, allow_alias=True) for p in schur_views(M, block)]


def sweep_macs(plans) -> int:
    """GF(p) multiply-adds of one sweep (the reference's scalar_macs counter, summed)."""
    return sum(pl.counters().scalar_macs for pl in plans)


def schur_sweep(M: Matrix, block: int, op: int = OP_SUB, stream=None, plans=None) -> int:
    """Run the sweep (asynchronously on `stream`); returns GF(p) MACs done."""
    plans = plans if plans is not None else schur_plans(M, block, op)
    for pl in plans:
        pl.run(stream)
    return sweep_macs(plans)


class SweepGraph:
    """A whole sweep captured into one CUDA graph (the C ABI's mhg_sweep): `replay(stream)`
    runs every step's pack and GEMM back to back with one launch and no host work in
    between.  The plans (and their workspaces) live as long as the graph; the parent's cells
    are read and written in place, so a replay is the same in-place update as schur_sweep."""

    def __init__(self, M: Matrix, block: int, op: int = OP_SUB, plans=None):
        from . import Sweep
        self.plans = plans if plans is not None else schur_plans(M, block, op)
        self._sweep = Sweep(self.plans) if self.plans else None  # block >= n: nothing to do
        self.macs = self._sweep.macs if self._sweep else 0

    def replay(self, stream=None) -> int:
        """Launch the captured sweep on `stream` (a torch stream or a raw handle; default: the
        default stream, like Plan.run); returns GF(p) MACs done."""
        return self._sweep.run(stream) if self._sweep else 0
