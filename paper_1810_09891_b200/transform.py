"""Module-level transform entry points (reference transform.py:92-176).

``trafo(plan, fhat)`` / ``adjoint(plan, f)`` delegate to the plan, which runs
D -> F -> B (resp. B^H -> F^H -> D^H) on the GPU.  The exact O(M |I_N|) sums
``ndft`` / ``ndft_adjoint`` of the reference are test oracles and live in
``oracle/`` (CPU), not in this package.
"""


def trafo(plan, fhat):
    return plan.trafo(fhat)


def adjoint(plan, f):
    return plan.adjoint(f)
