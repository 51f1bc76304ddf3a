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

from paper_1810_09891_b200.distributed import DistributedNfft, shard_bounds


class OracleEngine:
    """CPU engine: oracle trafo / spread grid / finish on this rank's shard."""

    def __init__(self, N, n, m, x_local):
        from oracle import oracle as O

        self.O, self.N, self.n, self.m, self.x = O, N, n, m, x_local

    def trafo(self, fhat):
        return torch.from_numpy(self.O.trafo(self.N, self.n, self.m, self.x, fhat.numpy()))

    def spread(self, f_local):
        g = self.O.spread_grid(self.N, self.n, self.m, self.x, f_local.numpy(), blockwise=False)
        return torch.view_as_real(torch.from_numpy(g)).contiguous()

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
        DistributedNfft(object(), reduce="slab")
