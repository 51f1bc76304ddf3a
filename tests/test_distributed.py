"""Multi-rank (world_size 2, gloo on CPU) tests of the node-sharded NFFT
orchestration (paper_1810_09891_b200.distributed).  The same DistributedNfft
code drives the CUDA engine on B200 ranks; here a CPU engine built from the
oracle's spread / finish / trafo pieces stands in for the device, so the
sharding and the all-reduce exchange step are checked end to end against the
single-process reference adjoint."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_09891_b200.distributed import (DistributedNfft, shard_bounds, stencil_rows,
                                               tile_shard_index)


class OracleEngine:
    """CPU engine: oracle trafo / spread grid / gather / finish on this rank's
    shard, with a persistent dense grid (the slab mode reads and fills it)."""

    def __init__(self, N, n, m, x_local):
        from oracle import oracle as O

        self.O, self.N, self.n, self.m, self.x = O, tuple(N), tuple(n), m, x_local
        self.cdtype = torch.complex128
        self.g = torch.zeros(self.n, dtype=torch.complex128)

    def nodes_version(self):
        return 0

    def trafo(self, fhat):
        return torch.from_numpy(self.O.trafo(self.N, self.n, self.m, self.x, np.asarray(fhat)))

    def spread(self, f_local):
        g = self.O.spread_grid(self.N, self.n, self.m, self.x, f_local.numpy(), blockwise=False)
        self.g.copy_(torch.from_numpy(g).view(self.n))
        return torch.view_as_real(self.g)

    def interp(self, out=None):
        return torch.from_numpy(self.O.gather_grid(self.N, self.n, self.m, self.x, self.g.numpy()))

    def grid_view(self):
        return self.g

    def deconv_cols(self, i):
        O = self.O
        b = O.window_b(O.KAISER_BESSEL, self.N[i], self.n[i], self.m)
        k = range(-self.N[i] // 2, self.N[i] // 2)
        return torch.tensor([1.0 / O.phi_hat(O.KAISER_BESSEL, kk, self.n[i], self.m, b) for kk in k],
                            dtype=torch.float64)

    def node_rows(self):
        return stencil_rows(torch.from_numpy(np.ascontiguousarray(self.x[:, 0])), self.n[0], self.m)

    def finish(self, grid):
        g = torch.view_as_complex(grid).numpy()
        return torch.from_numpy(self.O.adjoint_finish(self.N, self.n, self.m, g))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, reduce, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, n, m, M = case
        rng = np.random.default_rng(42)
        x = rng.random((M, len(N))) - 0.5
        K = int(np.prod(N))
        fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
        f = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        lo, hi = shard_bounds(M, world, rank)
        eng = DistributedNfft(OracleEngine(N, n, m, x[lo:hi]), reduce=reduce)
        # adjoint first with the exchange in flight, the trafo overlapping it
        a, work = eng.adjoint(torch.from_numpy(f[lo:hi]), async_op=True)
        f_loc = eng.trafo(torch.from_numpy(fh))
        work.wait()
        q.put((rank, lo, f_loc.numpy(), a.numpy()))
    except Exception as exc:  # surface worker failures instead of a queue timeout
        q.put((rank, None, repr(exc), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [((16,), (32,), 4, 101), ((8, 8), (16, 20), 3, 333),
                                  ((8, 8, 8), (16, 16, 16), 3, 257)])
@pytest.mark.parametrize("reduce", ["fhat", "grid"])
def test_sharded_trafo_adjoint_world2(case, reduce):
    from oracle import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, reduce, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for r in results:
        assert r[1] is not None, r[2]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, n, m, M = case
    rng = np.random.default_rng(42)
    x = rng.random((M, len(N))) - 0.5
    K = int(np.prod(N))
    fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    f = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    ref_f = O.trafo(N, n, m, x, fh)
    ref_a = O.adjoint(N, n, m, x, f, blockwise=False)
    f_all = np.zeros(M, dtype=np.complex128)
    for rank, lo, f_loc, a in results:
        f_all[lo:lo + f_loc.size] = f_loc
        assert O.error_e2(ref_a, a) < 1e-13
    assert O.error_e2(ref_f, f_all) < 1e-15


def _slab_worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, n, m, M, tile, kind = case
        x, fh, f = _slab_inputs(case)
        idx = tile_shard_index(torch.from_numpy(x), n, tile, world, rank).numpy()
        eng = DistributedNfft(OracleEngine(N, n, m, x[idx]), reduce="slab")
        a, work = eng.adjoint(torch.from_numpy(f[idx]), async_op=True)
        f_loc = eng.trafo(torch.from_numpy(fh))
        work.wait()
        q.put((rank, idx, f_loc.numpy(), a.numpy()))
    except Exception as exc:
        q.put((rank, None, repr(exc), None))
        raise
    finally:
        dist.destroy_process_group()


def _slab_inputs(case):
    from paper_1810_09891_b200 import workloads as wl

    N, n, m, M, tile, kind = case
    rng = np.random.default_rng(43)
    if kind == "clustered":
        x = wl.clustered_nodes(M, len(N), seed=9)
    else:
        x = rng.random((M, len(N))) - 0.5
    K = int(np.prod(N))
    fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    f = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    return x, fh, f


def _spawn(target, world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for r in results:
        assert r[1] is not None, r[2]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [
    ((16, 16, 16), (32, 32, 32), 3, 900, (8, 8, 8), "uniform"),
    ((16, 12), (32, 24), 4, 700, (4, 4), "uniform"),
    ((32, 32), (64, 64), 5, 2000, (8, 8), "clustered"),
])
def test_slab_decomposed_trafo_adjoint(case, world):
    """tile-sharded nodes, row-owned grid slabs, row-block
    exchange of the spread grids (halos only), slab-decomposed F / F^H with an
    all-to-all transpose -- against the single-process reference path."""
    from oracle import oracle as O

    results = _spawn(_slab_worker, world, (case,))
    N, n, m, M, tile, kind = case
    x, fh, f = _slab_inputs(case)
    ref_f = O.trafo(N, n, m, x, fh)
    ref_a = O.adjoint(N, n, m, x, f, blockwise=False)
    f_all = np.full(M, np.nan, dtype=np.complex128)
    seen = np.zeros(M, dtype=int)
    for rank, idx, f_loc, a in results:
        f_all[idx] = f_loc
        seen[idx] += 1
        assert O.error_e2(ref_a, a) < 1e-13
    assert (seen == 1).all()  # the shards partition the nodes
    assert O.error_e2(ref_f, f_all) < 1e-13


def test_tile_shards_are_compact_and_balanced():
    """Contiguous ranges of the tile order: balanced counts, and for uniform
    nodes each rank's stencil rows are its slab plus a 2m halo."""
    rng = np.random.default_rng(0)
    n, tile, m, world = (64, 64, 64), (8, 8, 8), 4, 8
    x = torch.from_numpy(rng.random((40000, 3)) - 0.5)
    rows = []
    for r in range(world):
        idx = tile_shard_index(x, n, tile, world, r)
        lo, hi = shard_bounds(x.shape[0], world, r)
        assert idx.numel() == hi - lo and bool((idx[1:] > idx[:-1]).all())
        rows.append(int(stencil_rows(x[idx, 0], n[0], m).sum()))
    # count-balanced cuts fall inside tile rows: a shard spans at most its
    # slab plus parts of the two neighbouring tile rows, plus the 2m halo
    assert max(rows) <= n[0] // world + 2 * tile[0] + 2 * m
    assert sum(rows) < 2 * n[0] + world * 2 * m  # nowhere near every rank touching every row


def test_shard_bounds_partition():
    for M in (1, 7, 100, 2 ** 20 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(M, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_reduce_mode_validated():
    with pytest.raises(ValueError):
        DistributedNfft(object(), reduce="pencil")
