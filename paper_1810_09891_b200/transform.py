"""Module-level transform entry points (reference transform.py:92-234).

``trafo(plan, fhat)`` / ``adjoint(plan, f)`` delegate to the plan, which runs
D -> F -> B (resp. B^H -> F^H -> D^H) on the GPU.  ``ndft`` / ``ndft_adjoint``
are the exact O(M |I_N|) sums, also on the GPU (separable phases, one cuBLAS
ZGEMM over the last dimension per node chunk; csrc/ndft.cu).
"""


def trafo(plan, fhat):
    return plan.trafo(fhat)


def adjoint(plan, f):
    return plan.adjoint(f)


def ndft(plan, fhat):
    """Exact forward sums (transform.py:188-203)."""
    return plan.ndft(fhat)


def ndft_adjoint(plan, f):
    """Exact adjoint sums (transform.py:206-234)."""
    return plan.ndft_adjoint(f)
