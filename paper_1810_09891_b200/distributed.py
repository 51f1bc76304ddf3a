"""Multi-GPU NFFT: nodes sharded across ranks, one process per GPU.

Design:

* trafo   -- every rank holds the full coefficient vector, runs D and F on its
             own GPU (replicated, no communication) and interpolates only its
             node shard.  Samples stay sharded.
* adjoint -- every rank spreads its node shard into a private full n-grid.
             The exchange step is one all-reduce (NCCL over NVLink on B200)
             of either
               - the coefficients (``reduce="fhat"``, default): every rank
                 runs F^H and D^H on its own grid and the |I_N|-sized
                 results are summed.  The adjoint is linear, so
                 sum_r D^H F^H g_r = D^H F^H sum_r g_r; on the B200 a
                 replicated FFT is cheaper than moving the oversampled grid
                 (|I_n| / |I_N| = sigma^d = 8x fewer bytes in 3-D, 4x in
                 2-D: C5 moves 256 MiB instead of 2 GiB per rank);
               - or the grid (``reduce="grid"``, the SURVEY 8(e) form):
                 the grids are summed, then every rank runs F^H and D^H.

The all-reduce is the only data-path collective; it is the real exchange step
of the adjoint (a sum over all nodes).  ``torch.distributed`` supplies the
plumbing.  The orchestration below is engine-agnostic: ``GpuEngine`` runs the
CUDA library (the grid is a torch tensor bound into the plan with
``nfftk_bind_grid`` so the collective reduces the library's grid in place);
tests drive the same ``DistributedNfft`` with a CPU engine over gloo.
"""

import torch
import torch.distributed as dist


def shard_bounds(M_total, world, rank):
    """Contiguous node range [lo, hi) of ``rank`` (balanced to within one node)."""
    lo = (M_total * rank) // world
    hi = (M_total * (rank + 1)) // world
    return lo, hi


class DistributedNfft:
    """Node-sharded trafo / adjoint over a process group.

    ``engine`` provides: ``trafo(fhat) -> f_local``, ``spread(f_local) -> grid``
    (a tensor the collective may reduce in place) and ``finish(grid) -> fhat``.
    """

    def __init__(self, engine, group=None, reduce="fhat"):
        if reduce not in ("fhat", "grid"):
            raise ValueError(f"reduce must be 'fhat' or 'grid', not {reduce!r}")
        self.engine = engine
        self.group = group
        self.reduce = reduce
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def trafo(self, fhat):
        """Samples at this rank's nodes (no communication)."""
        return self.engine.trafo(fhat)

    def adjoint(self, f_local, out=None, async_op=False):
        """Full coefficient vector, identical on every rank.

        ``async_op=True`` (coefficient reduction) returns ``(fhat, work)``:
        the all-reduce is in flight and ``work.wait()`` orders it before
        later work on the current stream, so independent work -- e.g. the
        trafo of a trafo + adjoint step -- overlaps the exchange (on NCCL the
        collective runs on its own stream)."""
        grid = self.engine.spread(f_local)
        if self.reduce == "grid" and self.world > 1:
            dist.all_reduce(grid, op=dist.ReduceOp.SUM, group=self.group)
        fhat = self.engine.finish(grid) if out is None else self.engine.finish(grid, out=out)
        work = None
        if self.reduce == "fhat" and self.world > 1:
            work = dist.all_reduce(torch.view_as_real(fhat), op=dist.ReduceOp.SUM, group=self.group,
                                   async_op=async_op)
        if async_op:
            return fhat, (work if work is not None else _Done())
        return fhat


class _Done:
    """Completed-work stand-in (one rank, or the grid reduction already done)."""

    def wait(self):
        return True


class GpuEngine:
    """The CUDA library as a DistributedNfft engine (one Plan per rank)."""

    def __init__(self, plan, device):
        self.plan = plan
        real = torch.float32 if plan.single else torch.float64
        # dense n-grid as interleaved reals: the collective reduces a plain buffer
        self.grid = torch.empty(2 * plan.grid_size, dtype=real, device=device)
        plan.bind_grid(self.grid)
        self._out = None

    def trafo(self, fhat, out=None):
        return self.plan.trafo(fhat, out=out)

    def spread(self, f_local):
        self.plan.spread(f_local)
        return self.grid

    def finish(self, grid, out=None):
        assert grid.data_ptr() == self.grid.data_ptr()
        if out is None:
            cdt = torch.complex64 if self.plan.single else torch.complex128
            out = torch.empty(self.plan.num_freqs, dtype=cdt, device=self.grid.device)
        return self.plan.adjoint_finish(out)


class DistributedPlan(DistributedNfft):
    """Convenience: a CUDA plan over this rank's node shard plus the reduction."""

    def __init__(self, N, M_local, n=None, m=None, f1=None, f2=None, window="kaiserbessel",
                 precision="double", group=None, device=None, reduce="fhat"):
        from .plan import Plan

        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.plan = Plan(N, M_local, n=n, m=m, f1=f1, f2=f2, window=window, precision=precision)
        self.device = device
        super().__init__(GpuEngine(self.plan, device), group, reduce)

    @property
    def M_local(self):
        return self.plan.M

    def set_nodes(self, coords_local):
        self.plan.set_nodes(coords_local)

    def precompute(self):
        self.plan.precompute()

    def close(self):
        self.plan.close()
