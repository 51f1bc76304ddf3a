"""Multi-GPU NFFT: nodes sharded across ranks, one process per GPU.

Design:

* trafo   -- every rank holds the full coefficient vector, runs D and F on its
             own GPU (replicated, no communication) and interpolates only its
             node shard.  Samples stay sharded.
* adjoint -- every rank spreads its node shard into a private full n-grid,
             the grids are summed with one NCCL all-reduce over NVLink, then
             every rank runs F^H and D^H (replicated result).

The all-reduce is the only data-path collective; it is the real exchange
step of the adjoint (sum over all nodes).  ``torch.distributed`` supplies
the plumbing; the grid is a torch tensor bound into the plan
(``nfftk_bind_grid``) so the collective reduces the library's grid in place.
"""

import torch
import torch.distributed as dist

from .plan import Plan


class DistributedPlan:
    """A plan over this rank's node shard plus the grid reduction."""

    def __init__(self, N, M_local, n=None, m=None, f1=None, f2=None, window="kaiserbessel",
                 precision="double", group=None, device=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.plan = Plan(N, M_local, n=n, m=m, f1=f1, f2=f2, window=window, precision=precision)
        real = torch.float32 if self.plan.single else torch.float64
        # grid as interleaved reals: NCCL reduces it as a plain float buffer
        self.grid = torch.empty(2 * self.plan.grid_size, dtype=real, device=self.device)
        self.plan.bind_grid(self.grid)

    @property
    def M_local(self):
        return self.plan.M

    def set_nodes(self, coords_local):
        self.plan.set_nodes(coords_local)

    def precompute(self):
        self.plan.precompute()

    def trafo(self, fhat):
        """Sharded samples of this rank's nodes (no communication)."""
        return self.plan.trafo(fhat)

    def adjoint(self, f_local, out=None):
        """Full coefficient vector, identical on every rank."""
        self.plan.spread(f_local)
        if self.world > 1:
            dist.all_reduce(self.grid, op=dist.ReduceOp.SUM, group=self.group)
        if out is None:
            out = torch.empty(self.plan.num_freqs, dtype=f_local.dtype, device=f_local.device)
        return self.plan.adjoint_finish(out)

    def close(self):
        self.plan.close()


def shard_bounds(M_total, world, rank):
    """Contiguous node range of ``rank`` (balanced to within one node)."""
    lo = (M_total * rank) // world
    hi = (M_total * (rank + 1)) // world
    return lo, hi
