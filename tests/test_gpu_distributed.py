"""Multi-rank execution of the CUDA engine (GpuEngine / DistributedPlan) on one
B200: two processes share cuda:0 and talk over gloo (host-staged collectives;
on an 8-GPU box the same code runs one rank per GPU over NCCL).  Each rank
holds a tile-contiguous node shard, runs the library's kernels on it, and the
exchange modes -- coefficient all-reduce, grid all-reduce, and the
slab-decomposed F with row-block exchange -- are compared with the oracle
(the C port of the reference path) on the full node set.

Ranks on one GPU never wait on each other inside a kernel: every exchange is a
host-side gloo collective between complete device phases.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    ((32, 32, 32), (64, 64, 64), 4, 30000, "uniform"),
    ((64, 64), (128, 128), 6, 40000, "clustered"),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(case):
    from paper_1810_09891_b200 import workloads as wl

    N, n, m, M, kind = case
    x = wl.clustered_nodes(M, len(N), seed=5) if kind == "clustered" else wl.uniform_nodes(M, len(N), seed=5)
    fh = wl.complex_normal(int(np.prod(N)), 6)
    f = wl.complex_normal(M, 7)
    return x, fh, f


def _worker(rank, world, port, case, reduce, precision, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1810_09891_b200.distributed import DistributedPlan

        N, n, m, M, kind = case
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        x, fh, f = _inputs(case)
        cdt = torch.complex64 if precision == "single" else torch.complex128
        dp = DistributedPlan(N, M, n=n, m=m, precision=precision, device=dev, reduce=reduce)
        dp.set_nodes(torch.from_numpy(x).to(dev))
        dp.precompute()
        f_loc = dp.scatter(torch.from_numpy(f).to(dev, cdt))
        # the bench's step order: adjoint with its exchange in flight, trafo under it
        a, work = dp.adjoint(f_loc, async_op=True)
        t = dp.trafo(torch.from_numpy(fh).to(dev, cdt))
        work.wait()
        f_all = dp.gather(t)
        torch.cuda.synchronize()
        q.put((rank, "ok", f_all.cpu().numpy(), a.cpu().numpy(), dp.M_local))
        dp.close()
    except Exception as exc:  # surface worker failures instead of a queue timeout
        q.put((rank, repr(exc), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("reduce", ["fhat", "grid", "slab"])
@pytest.mark.parametrize("case", CASES, ids=["d3_uniform", "d2_clustered"])
def test_gpu_engine_world2(case, reduce, precision, oracle):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, reduce, precision, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for r in results:
        assert r[1] == "ok", r[1]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    N, n, m, M, kind = case
    x, fh, f = _inputs(case)
    ref_f = oracle.trafo(N, n, m, x, fh)
    ref_a = oracle.adjoint(N, n, m, x, f)
    tol = 1e-12 if precision == "double" else 1e-5
    assert sum(r[4] for r in results) == M
    for _, _, f_all, a, _ in results:
        assert oracle.error_e2(ref_f, f_all) < tol
        assert oracle.error_e2(ref_a, a) < tol
