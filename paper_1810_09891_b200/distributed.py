"""Multi-GPU NFFT: one process per GPU, nodes sharded across ranks.

Node sharding: the global node set is ordered by
grid TILE (row-major over the tile grid, the library's own binning) and cut
into contiguous, count-balanced ranges -- so a rank's nodes occupy a compact
band of dim-0 rows (a slab, for uniform nodes) and clustered nodes (C4) stay
balanced by count.  Within its shard a rank keeps the nodes in their global
(natural) order; ``shard_index`` maps local sample i to global node
``shard_index[i]``.

Exchange modes (``reduce=``):

* ``"fhat"`` (default) -- trafo: every rank runs D and F on its own GPU
  (replicated, no communication) and interpolates its shard.  adjoint: every
  rank spreads into a private n-grid and runs F^H, D^H on it; the |I_N|
  coefficient vectors are all-reduced (the adjoint is linear:
  sum_r D^H F^H g_r = D^H F^H sum_r g_r; sigma^d = 8x fewer bytes than the
  grid in 3-D).
* ``"grid"`` -- the SURVEY 8(e) form: the spread n-grids are all-reduced,
  then every rank runs F^H and D^H.
* ``"slab"`` -- the spatially partitioned form (the GPU
  analogue of the reference's slab-owned adjoint, kernels.py:293-401 /
  transform.py:128-170): rank r OWNS grid rows S0_r = [n0 r/P, n0 (r+1)/P)
  of dim 0 and columns S1_r = [n1 r/P, n1 (r+1)/P) of dim 1.
    - adjoint: each rank spreads into a private grid; only the rows its
      nodes touch (its slab plus a (2m)-row halo for tile-sharded nodes) are
      sent, each to the rank owning them (one all-to-all of row blocks:
      |I_n|/P plus the halos per rank instead of a full-grid reduction);
      the owner sums them; F^H is a slab-decomposed FFT (local FFT over
      dims 1.., all-to-all transpose to dim-1 slabs, FFT over dim 0); D^H
      packs the owned frequencies and one all-reduce of the (disjoint)
      coefficient parts completes f_hat on every rank.
    - trafo: D builds only the owned dim-1 columns of the zero-padded grid,
      F is the same slab FFT in reverse (dims 0 and 2.. locally, transpose to
      dim-0 slabs, dim 1), and each rank receives from the row owners exactly
      the rows its nodes' stencils touch (owned slab + halos), then runs B.
  d = 2, 3 (d = 1 has no slab decomposition; use "fhat").

The collectives (``all_reduce``, ``all_to_all_single``) go through
``torch.distributed`` -- NCCL over NVLink on B200 ranks, gloo in the CPU
tests.  The local FFTs of the slab path are cuFFT through ``torch.fft``
(unnormalised: sign -1 forward = ``fftn``, sign +1 adjoint = ``ifftn`` with
``norm="forward"``, transform.py:98 / :174).  The orchestration is
engine-agnostic: ``GpuEngine`` runs the CUDA library (the plan's dense grid
is a torch tensor bound with ``nfftk_bind_grid``); the CPU tests drive the
same code with an oracle engine over gloo.
"""

import math

import torch
import torch.distributed as dist


def _staged(group, t):
    """gloo with CUDA tensors (the one-GPU functional test of the multi-rank
    path): collectives run on host copies.  NCCL takes device tensors as is."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


class _StagedWork:
    def __init__(self, work, dst, src):
        self.work, self.dst, self.src = work, dst, src

    def wait(self):
        if self.work is not None:
            self.work.wait()
        self.dst.copy_(self.src)
        return True


def all_reduce_sum(t, group=None, async_op=False):
    if not _staged(group, t):
        return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    h = t.cpu()
    w = dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    if async_op:
        return _StagedWork(w, t, h)
    t.copy_(h)
    return None


def all_to_all(recv, send, out_splits, in_splits, group=None):
    if not _staged(group, send):
        dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
        return
    h = torch.empty(recv.shape, dtype=recv.dtype)
    dist.all_to_all_single(h, send.cpu(), out_splits, in_splits, group=group)
    recv.copy_(h)


def all_gather(outs, t, group=None):
    if not _staged(group, t):
        dist.all_gather(outs, t, group=group)
        return
    hs = [torch.empty(o.shape, dtype=o.dtype) for o in outs]
    dist.all_gather(hs, t.cpu(), group=group)
    for o, h in zip(outs, hs):
        o.copy_(h)


def shard_bounds(M_total, world, rank):
    """Contiguous range [lo, hi) of ``rank`` (balanced to within one node)."""
    lo = (M_total * rank) // world
    hi = (M_total * (rank + 1)) // world
    return lo, hi


def tile_keys(x, n, tile):
    """Row-major tile index of every node: tile coordinate
    floor_mod(floor(n_i x_i), n_i) // T_i per dim (the library's k_bin_keys
    slot arithmetic, kernels.py:47 wrapping)."""
    key = torch.zeros(x.shape[0], dtype=torch.int64, device=x.device)
    for i, (ni, ti) in enumerate(zip(n, tile)):
        cell = torch.floor(x[:, i] * float(ni)).to(torch.int64).remainder(ni)
        key = key * ((ni + ti - 1) // ti) + cell // ti
    return key


def tile_shard_index(x, n, tile, world, rank):
    """Global indices (ascending) of this rank's nodes: the rank-th of
    ``world`` count-balanced contiguous ranges of the stable tile order."""
    x = torch.as_tensor(x)
    M = x.shape[0]
    lo, hi = shard_bounds(M, world, rank)
    if world == 1:
        return torch.arange(M, dtype=torch.int64, device=x.device)
    order = torch.sort(tile_keys(x, n, tile), stable=True).indices
    return torch.sort(order[lo:hi]).values


def row_slab(n0, world, rank):
    """Owned row range of dim 0 (and, with n1, of dim 1) in the slab mode."""
    return (n0 * rank) // world, (n0 * (rank + 1)) // world


def stencil_rows(x0, n0, m):
    """Bool mask over the n0 dim-0 rows touched by the stencils of nodes with
    dim-0 coordinates x0: rows ceil(n0 x - m) .. floor(n0 x + m) mod n0
    (indexing.py:114-124)."""
    mask = torch.zeros(n0, dtype=torch.bool, device=x0.device)
    if x0.numel() == 0:
        return mask
    y = x0 * float(n0)
    lo = torch.ceil(y - m).to(torch.int64)
    hi = torch.floor(y + m).to(torch.int64)
    for t in range(2 * m + 1):
        r = lo + t
        ok = r <= hi
        mask[r[ok].remainder(n0)] = True
    return mask


class DistributedNfft:
    """Node-sharded trafo / adjoint over a process group (see module doc).

    ``engine`` provides ``trafo(fhat)``, ``spread(f_local) -> grid`` (a tensor
    the collectives may reduce in place), ``finish(grid) -> fhat``; the slab
    mode also ``interp() -> f_local`` (B from the engine's grid),
    ``grid_view()`` (the dense grid as a complex tensor of shape n),
    ``deconv_cols()`` and ``node_rows()`` (rows its stencils touch), plus
    the attributes ``N``, ``n``, ``m``, ``cdtype``.
    """

    MODES = ("fhat", "grid", "slab")

    def __init__(self, engine, group=None, reduce="fhat"):
        if reduce not in self.MODES:
            raise ValueError(f"reduce must be one of {self.MODES}, not {reduce!r}")
        self.engine = engine
        self.group = group
        self.reduce = reduce
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if reduce == "slab":
            d = len(engine.n)
            if d < 2:
                raise ValueError("the slab decomposition needs d >= 2 (use reduce='fhat' for d = 1)")
            if self.world > min(engine.n[0], engine.n[1]):
                raise ValueError("slab mode needs world <= n_0 and n_1")
        self._rows_plan = None

    # ------------------------------------------------------------ trafo
    def trafo(self, fhat, out=None):
        """Samples at this rank's nodes."""
        if self.reduce != "slab" or self.world == 1:
            return self.engine.trafo(fhat) if out is None else self.engine.trafo(fhat, out=out)
        self._slab_forward(fhat)
        return self.engine.interp() if out is None else self.engine.interp(out=out)

    # ---------------------------------------------------------- adjoint
    def adjoint(self, f_local, out=None, async_op=False):
        """Full coefficient vector, identical on every rank.

        ``async_op=True`` (coefficient reduction) returns ``(fhat, work)``:
        the all-reduce is in flight and ``work.wait()`` orders it before
        later work on the current stream, so independent work -- e.g. the
        trafo of a trafo + adjoint step -- overlaps the exchange (on NCCL the
        collective runs on its own stream)."""
        grid = self.engine.spread(f_local)
        work = None
        if self.reduce == "slab" and self.world > 1:
            fhat = self._slab_adjoint(out)
            work = all_reduce_sum(torch.view_as_real(fhat), group=self.group, async_op=async_op)
        else:
            if self.reduce == "grid" and self.world > 1:
                all_reduce_sum(grid, group=self.group)
            fhat = self.engine.finish(grid) if out is None else self.engine.finish(grid, out=out)
            if self.reduce == "fhat" and self.world > 1:
                work = all_reduce_sum(torch.view_as_real(fhat), group=self.group, async_op=async_op)
        if async_op:
            return fhat, (work if work is not None else _Done())
        return fhat

    # ------------------------------------------------------ slab pieces
    def _rows(self):
        """Row exchange plan: need[r] = rows rank r's stencils touch (bool over
        n0), gathered from every rank; cached until the nodes change."""
        key = self.engine.nodes_version()
        if self._rows_plan is not None and self._rows_plan[0] == key:
            return self._rows_plan[1]
        n0 = self.engine.n[0]
        mine = self.engine.node_rows().to(torch.uint8)
        allm = [torch.empty_like(mine) for _ in range(self.world)]
        all_gather(allm, mine, group=self.group)
        need = [a.bool() for a in allm]
        dev = mine.device
        owned = [row_slab(n0, self.world, q) for q in range(self.world)]
        rowsel = torch.arange(n0, device=dev)
        # rows of rank r's need that q owns (increasing row order)
        send = {}
        for q in range(self.world):
            for r in range(self.world):
                lo, hi = owned[q]
                sel = rowsel[lo:hi][need[r][lo:hi]]
                send[(q, r)] = sel
        plan = {"need": need, "owned": owned, "send": send}
        self._rows_plan = (key, plan)
        return plan

    def _coef_tables(self, dev):
        e = self.engine
        d = len(e.n)
        slots, cols = [], []
        for i in range(d):
            p = torch.arange(e.N[i], dtype=torch.int64, device=dev)
            slots.append((p - e.N[i] // 2).remainder(e.n[i]))
            cols.append(torch.as_tensor(e.deconv_cols(i), dtype=torch.float64).to(dev))
        return slots, cols

    def _deconv_factor(self, cols, sel1, dev, real):
        """prod_i 1/(phi_hat_i wscale_i) / |I_n| over (N0, |sel1|, N2..)."""
        d = len(cols)
        fac = cols[0].view(-1, *([1] * (d - 1))) * cols[1][sel1].view(1, -1, *([1] * (d - 2)))
        if d == 3:
            fac = fac * cols[2].view(1, 1, -1)
        return (fac * (1.0 / math.prod(self.engine.n))).to(real)

    def _slab_forward(self, fhat):
        """D + slab-decomposed F into the rows this rank's nodes need."""
        e = self.engine
        P, r = self.world, self.rank
        n, N, d = e.n, e.N, len(e.n)
        grid = e.grid_view()  # complex, shape n
        dev, cdt = grid.device, grid.dtype
        real = torch.float32 if cdt == torch.complex64 else torch.float64
        slots, cols = self._coef_tables(dev)
        c_lo, c_hi = row_slab(n[1], P, r)
        # D: the owned dim-1 columns of the zero-padded, deconvolved grid
        sel1 = ((slots[1] >= c_lo) & (slots[1] < c_hi)).nonzero().flatten()
        g1 = torch.zeros((n[0], c_hi - c_lo) + tuple(n[2:]), dtype=cdt, device=dev)
        if sel1.numel():
            fh = torch.as_tensor(fhat).to(dev, cdt).reshape(N)
            vals = fh.index_select(1, sel1) * self._deconv_factor(cols, sel1, dev, real)
            idx = [slots[0].view(-1, *([1] * (d - 1))), (slots[1][sel1] - c_lo).view(1, -1, *([1] * (d - 2)))]
            if d == 3:
                idx.append(slots[2].view(1, 1, -1))
            g1.index_put_(tuple(idx), vals)
        # F: dims 0 (and 2) locally on the column slab
        g1 = torch.fft.fftn(g1, dim=(0,) + tuple(range(2, d)))
        # transpose: rows S0_q of my column slab go to q
        owned = [row_slab(n[0], P, q) for q in range(P)]
        cols_of = [row_slab(n[1], P, q) for q in range(P)]
        inner = math.prod(n[2:])
        send = torch.view_as_real(g1).reshape(-1)
        in_splits = [(hi - lo) * (c_hi - c_lo) * inner * 2 for lo, hi in owned]
        r_lo, r_hi = owned[r]
        out_splits = [(r_hi - r_lo) * (qh - ql) * inner * 2 for ql, qh in cols_of]
        recv = torch.empty(sum(out_splits), dtype=real, device=dev)
        all_to_all(recv, send, out_splits, in_splits, group=self.group)
        blocks = torch.split(recv, out_splits)
        slab = torch.cat([torch.view_as_complex(b.view((r_hi - r_lo), qh - ql, *n[2:], 2))
                          for b, (ql, qh) in zip(blocks, cols_of)], dim=1)
        slab = torch.fft.fft(slab, dim=1)  # my rows of F D f_hat
        # rows: send owned rows to every rank whose stencils touch them
        self._exchange_rows_out(slab, grid)

    def _exchange_rows_out(self, slab, grid):
        """Owner -> user: rows of my slab that rank q needs; received rows go
        into q's grid at their row index."""
        plan = self._rows()
        P, r = self.world, self.rank
        dev = slab.device
        real = torch.float32 if slab.dtype == torch.complex64 else torch.float64
        row = math.prod(self.engine.n[1:]) * 2
        lo = plan["owned"][r][0]
        parts = [slab.index_select(0, plan["send"][(r, q)] - lo) for q in range(P)]
        send = torch.cat([torch.view_as_real(p).reshape(-1) for p in parts])
        in_splits = [p.shape[0] * row for p in parts]
        rows_from = [plan["send"][(q, r)] for q in range(P)]
        out_splits = [rr.numel() * row for rr in rows_from]
        recv = torch.empty(sum(out_splits), dtype=real, device=dev)
        all_to_all(recv, send, out_splits, in_splits, group=self.group)
        allrows = torch.cat(rows_from)
        if allrows.numel():
            grid.index_copy_(0, allrows, torch.view_as_complex(recv.view(allrows.numel(), *self.engine.n[1:], 2)))

    def _slab_adjoint(self, out=None):
        """Row exchange of the spread grids, slab-decomposed F^H, D^H of the
        owned frequencies; returns this rank's (disjoint) part of f_hat."""
        e = self.engine
        P, r = self.world, self.rank
        n, N, d = e.n, e.N, len(e.n)
        grid = e.grid_view()
        dev, cdt = grid.device, grid.dtype
        real = torch.float32 if cdt == torch.complex64 else torch.float64
        plan = self._rows()
        row = math.prod(n[1:]) * 2
        # user -> owner: the rows I touched that q owns
        parts = [grid.index_select(0, plan["send"][(q, r)]) for q in range(P)]
        send = torch.cat([torch.view_as_real(p).reshape(-1) for p in parts])
        in_splits = [p.shape[0] * row for p in parts]
        rows_from = [plan["send"][(r, q)] for q in range(P)]
        out_splits = [rr.numel() * row for rr in rows_from]
        recv = torch.empty(sum(out_splits), dtype=real, device=dev)
        all_to_all(recv, send, out_splits, in_splits, group=self.group)
        r_lo, r_hi = plan["owned"][r]
        slab = torch.zeros((r_hi - r_lo,) + tuple(n[1:]), dtype=cdt, device=dev)
        for blk, rows in zip(torch.split(recv, out_splits), rows_from):  # rank order: deterministic
            if rows.numel():
                slab.index_add_(0, rows - r_lo, torch.view_as_complex(blk.view(rows.numel(), *n[1:], 2)))
        # F^H: dims 1.. on the row slab, transpose, dim 0 on the column slab
        slab = torch.fft.ifftn(slab, dim=tuple(range(1, d)), norm="forward")
        cols_of = [row_slab(n[1], P, q) for q in range(P)]
        owned = plan["owned"]
        inner = math.prod(n[2:])
        send = torch.cat([torch.view_as_real(slab[:, ql:qh].contiguous()).reshape(-1) for ql, qh in cols_of])
        in_splits = [(r_hi - r_lo) * (qh - ql) * inner * 2 for ql, qh in cols_of]
        c_lo, c_hi = cols_of[r]
        out_splits = [(hi - lo) * (c_hi - c_lo) * inner * 2 for lo, hi in owned]
        recv = torch.empty(sum(out_splits), dtype=real, device=dev)
        all_to_all(recv, send, out_splits, in_splits, group=self.group)
        g1 = torch.cat([torch.view_as_complex(b.view(hi - lo, c_hi - c_lo, *n[2:], 2))
                        for b, (lo, hi) in zip(torch.split(recv, out_splits), owned)], dim=0)
        g1 = torch.fft.ifft(g1, dim=0, norm="forward")
        # D^H: the owned frequency columns; the others stay zero
        slots, cols = self._coef_tables(dev)
        sel1 = ((slots[1] >= c_lo) & (slots[1] < c_hi)).nonzero().flatten()
        fh = out if out is not None else torch.empty(math.prod(N), dtype=cdt, device=dev)
        fh.zero_()
        if sel1.numel():
            idx = [slots[0].view(-1, *([1] * (d - 1))), (slots[1][sel1] - c_lo).view(1, -1, *([1] * (d - 2)))]
            if d == 3:
                idx.append(slots[2].view(1, 1, -1))
            vals = g1[tuple(idx)] * self._deconv_factor(cols, sel1, dev, real)
            fh.view(N)[:, sel1] = vals
        return fh


class _Done:
    """Completed-work stand-in (one rank, or the exchange already done)."""

    def wait(self):
        return True


class GpuEngine:
    """The CUDA library as a DistributedNfft engine (one Plan per rank)."""

    def __init__(self, plan, device):
        self.plan = plan
        self.N, self.n, self.m = tuple(plan.N), tuple(plan.n), plan.m
        real = torch.float32 if plan.single else torch.float64
        self.cdtype = torch.complex64 if plan.single else torch.complex128
        # dense n-grid as interleaved reals: the collective reduces a plain buffer
        self.grid = torch.empty(2 * plan.grid_size, dtype=real, device=device)
        plan.bind_grid(self.grid)
        self._version = 0

    def nodes_version(self):
        return self._version

    def nodes_changed(self):
        self._version += 1

    def trafo(self, fhat, out=None):
        return self.plan.trafo(fhat, out=out)

    def spread(self, f_local):
        self.plan.spread(f_local)
        return self.grid

    def interp(self, out=None):
        return self.plan.interp(out=out)

    def grid_view(self):
        return torch.view_as_complex(self.grid.view(*self.n, 2))

    def deconv_cols(self, i):
        return torch.from_numpy(self.plan.deconv_cols(i))

    def node_rows(self):
        x = self.plan.x
        x0 = (x if torch.is_tensor(x) else torch.from_numpy(x))[:, 0].to(self.grid.device)
        return stencil_rows(x0, self.n[0], self.m)

    def finish(self, grid, out=None):
        assert grid.data_ptr() == self.grid.data_ptr()
        if out is None:
            out = torch.empty(self.plan.num_freqs, dtype=self.cdtype, device=self.grid.device)
        return self.plan.adjoint_finish(out)


class DistributedPlan(DistributedNfft):
    """A CUDA plan over this rank's node shard plus the exchange.

    ``M`` is the GLOBAL node count; the rank's plan holds its shard (a
    count-balanced contiguous range of the tile order, ``tile_shard_index``).
    ``set_nodes(x)`` takes the global node set (every rank passes the same
    nodes) and keeps this rank's shard; ``scatter(v)`` / ``gather(v)`` move
    per-node vectors between global and shard order.
    """

    def __init__(self, N, M, n=None, m=None, f1=None, f2=None, window="kaiserbessel",
                 precision="double", group=None, device=None, reduce="fhat"):
        from .plan import Plan

        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.M_total = int(M)
        lo, hi = shard_bounds(self.M_total, world, rank)
        self.plan = Plan(N, hi - lo, n=n, m=m, f1=f1, f2=f2, window=window, precision=precision)
        self.device = device
        self.shard_index = None
        super().__init__(GpuEngine(self.plan, device), group, reduce)

    @property
    def M_local(self):
        return self.plan.M

    def set_nodes(self, coords):
        """Global nodes (M, d) -> this rank's tile-contiguous shard."""
        x = torch.as_tensor(coords).to(self.device, torch.float64)
        if x.shape[0] != self.M_total:
            raise ValueError(f"set_nodes takes the global node set ({self.M_total} nodes), got {x.shape[0]}")
        self.shard_index = tile_shard_index(x, self.plan.n, self.plan.tile, self.world, self.rank)
        # one rank owns every node in the given order: no gather of the coordinates
        self.plan.set_nodes(x if self.world == 1 else x.index_select(0, self.shard_index).contiguous())
        self.engine.nodes_changed()

    def scatter(self, v):
        """Global per-node vector -> this rank's shard (shard order)."""
        return torch.as_tensor(v).to(self.device).index_select(0, self.shard_index)

    def gather(self, v_local):
        """Shard vectors of every rank -> the global per-node vector."""
        if self.world == 1:
            return v_local
        sizes = [hi - lo for lo, hi in (shard_bounds(self.M_total, self.world, q) for q in range(self.world))]
        top = max(sizes)  # shards differ by at most one node: pad to equal size
        dev = v_local.device

        def padded(t):
            out = torch.zeros(top, dtype=t.dtype, device=dev)
            out[: t.numel()] = t
            return out

        vs = [torch.empty(top, dtype=v_local.dtype, device=dev) for _ in sizes]
        idx = [torch.empty(top, dtype=torch.int64, device=dev) for _ in sizes]
        all_gather(vs, padded(v_local.reshape(-1)), group=self.group)
        all_gather(idx, padded(self.shard_index), group=self.group)
        out = torch.empty(self.M_total, dtype=v_local.dtype, device=dev)
        out[torch.cat([i[:k] for i, k in zip(idx, sizes)])] = torch.cat([v[:k] for v, k in zip(vs, sizes)])
        return out

    def precompute(self):
        self.plan.precompute()

    def close(self):
        self.plan.close()
