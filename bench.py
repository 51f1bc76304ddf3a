#!/usr/bin/env python
"""Benchmark: NFFT trafo+adjoint nodes/sec on B200 (BASELINE.json metric).

One step = one forward transform (D -> F -> B) plus one adjoint
(B^H -> F^H -> D^H) over the configuration's M nodes on every rank.

* ``value``  : whole-job nodes/s with inputs resident in HBM, device-timed
               (CUDA events on the launching stream, max over ranks), L2 flushed
               (256 MiB write) before every timed step.
* ``e2e``    : same metric through the reference-facing C-ABI with HOST
               buffers (nfftk_set_fhat / nfftk_trafo / nfftk_set_f /
               nfftk_adjoint: H2D + compute + D2H inside the timed region).
* ``roofline``: dominant gridding kernel (interp / spread) against measured HBM.
* ``cpu_baseline``: the CPU oracle port of the reference (oracle/), all host
               threads, bounded sample, rank 0 at N=1.

``--impl reference`` times only that CPU port (rank 0; other ranks exit 0).
Multi-GPU (torchrun): strong scaling -- the configuration's M nodes are split
across the ranks in tile order; the exchange (default: slab-decomposed F with
NCCL all-to-all, paper_1810_09891_b200.distributed) runs inside the step.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1810_09891_b200 import workloads as wl  # noqa: E402

# The headline workload: the largest BASELINE configuration that fits one
# GPU (C5: d=3, 512^3 grid, M = 2^26, complex128); C1-C4 are parity cases
# with their own bench lines under profiles/.
DEFAULT_CONFIG = "C5"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(wl.CONFIGS))
    ap.add_argument("--precision", default="double", choices=["double", "single"])
    ap.add_argument("--psi", default="flags", choices=["flags", "direct", "tensor"])
    ap.add_argument("--reduce", default="slab", choices=["fhat", "grid", "slab"],
                    help="exchange at N>1 (distributed.py): slab-decomposed F with row-block "
                         "exchange (default; d >= 2), all-reduce of the coefficients, or of the n-grid")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of one CUDA-graph replay per step")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


EXCHANGE = {
    "fhat": "replicated D+F; NCCL all-reduce of the adjoint coefficients (|I_N|)",
    "grid": "replicated D+F; NCCL all-reduce of the spread n-grid (|I_n|)",
    "slab": "slab-decomposed F/F^H (NCCL all-to-all transpose), row-block exchange of "
            "owned slabs + halos, all-reduce of the disjoint coefficient parts",
}


def config_json(w, args, world):
    return {
        "workload": f"{w.name}: d={w.d} N={'x'.join(map(str, w.N))} n={'x'.join(map(str, w.n))} "
                    f"M={w.M} m={w.m} {w.dist} nodes, Kaiser-Bessel",
        "d": w.d, "N": list(w.N), "n": list(w.n), "M": w.M, "m": w.m,
        "nodes": w.dist, "window": "kaiserbessel", "flags": "default f1 (PRE_PHI_HUT|PRE_PSI|sort)"
        if args.psi == "flags" else f"psi={args.psi}",
        "step": "trafo + adjoint",
        "parallelism": "1 GPU" if world == 1 else
        f"{world} GPUs, nodes sharded by tile order (M/{world} per rank)",
        "exchange": "none (1 rank)" if world == 1 else EXCHANGE[args.reduce if w.d > 1 else "fhat"],
        "l2": "flushed (256 MiB write) before every timed step",
    }


def launch_mode(args, world):
    """How the step is issued (a property of the arm, not of the workload)."""
    if getattr(args, "impl", "ours") == "reference":
        return "host CPU (reference arm)"
    if getattr(args, "no_graph", False) or world > 1:
        return "eager"
    return "CUDA graph of the step (captured once, replayed per step)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = self.rows
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU legs
def host_cores():
    """Host threads the CPU legs may use (torchrun sets OMP_NUM_THREADS=1)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_oracle_rate(w):
    """Time the CPU oracle port (trafo + adjoint) on the FULL workload: one
    step at the configuration's full M and grid (no scaled sample, so the
    grid-sized work -- deconvolution, FFTs -- is not divided by a small M).
    As in the reference's own protocol (set_nodes / precompute timed apart
    from the transforms, metrics.py:59-67), the plan -- stencils,
    lexicographic order, PRE_PSI table -- is built before the timed step."""
    from oracle import oracle as O

    O.set_threads(host_cores())
    threads = O.max_threads()
    x = wl.nodes(w)
    fh = wl.fhat(w)
    fs = wl.samples(w)
    t0 = time.perf_counter()
    P = O.Plan(w.N, w.n, w.m, x)
    t_plan = time.perf_counter() - t0
    t0 = time.perf_counter()
    P.trafo(fh)
    P.adjoint(fs)
    elapsed = time.perf_counter() - t0
    P.close()
    rate = w.M / elapsed
    sample = (f"oracle/ C port (OpenMP) of the reference path, default flags (PRE_PSI, sorted "
              f"blockwise adjoint): one trafo+adjoint step of the full {w.name} workload "
              f"(M={w.M}, full grid) in {elapsed:.1f} s; plan build (sort + PRE_PSI) "
              f"{t_plan:.1f} s untimed; {threads} threads")
    return rate, threads, sample


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    w = wl.CONFIGS[args.config]
    from oracle import oracle as O

    O.set_threads(host_cores())
    threads = O.max_threads()
    x = wl.nodes(w)
    fh = wl.fhat(w)
    fs = wl.samples(w)
    # set_nodes + precompute (plan.py:202-299) once, outside the steps
    P = O.Plan(w.N, w.n, w.m, x)
    f_out = np.empty(w.M, dtype=np.complex128)
    a_out = np.empty(w.num_freqs, dtype=np.complex128)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        P.trafo(fh, out=f_out)
        P.adjoint(fs, out=a_out)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    P.close()
    ms = 1000.0 * sum(times) / len(times)
    value = w.M / (ms / 1000.0)
    line = {
        "metric": "NFFT trafo+adjoint nodes/sec", "value": value, "unit": "nodes/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded, SURVEY 8(d) generators)", "impl": "reference",
        "config": config_json(w, args, 1),
        "launch": launch_mode(args, 1),
        "cpu_baseline": {"value": value, "unit": "nodes/s", "cores": threads, "kind": "port",
                         "sample": f"full {w.name} workload (M={w.M}, full grid) per step, oracle/ "
                                   f"C port of the reference path with its default flags (plan "
                                   f"built once before the steps), {threads} OpenMP threads"},
        "e2e": {"value": value, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU legs
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_1810_09891_b200 as nf
    from paper_1810_09891_b200 import _lib
    from paper_1810_09891_b200.distributed import DistributedPlan

    rank, world, local = env_rank()
    # NFFTK_DIST_BACKEND=gloo: functional check of the N>1 orchestration on a
    # one-GPU box (ranks share the device; not a measurement)
    backend = os.environ.get("NFFTK_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    w = wl.CONFIGS[args.config]
    cdt = torch.complex64 if args.precision == "single" else torch.complex128
    s_elem = 8 if args.precision == "single" else 16

    # ---- plan over this rank's shard (strong scaling: the configuration's M
    # nodes split across the ranks in tile order)
    reduce = args.reduce if w.d > 1 else "fhat"
    dp = DistributedPlan(w.N, w.M, n=w.n, m=w.m, precision=args.precision, device=dev,
                         reduce=reduce)
    plan = dp.plan
    if args.psi != "flags":
        plan.set_psi_policy(nf.MODE_DIRECT if args.psi == "direct" else nf.MODE_TENSOR)
    x = torch.from_numpy(wl.nodes(w)).to(dev)
    # set_nodes + precompute (sort, stencil records, PRE_PSI): the first call
    # includes one-time costs (module loading, buffer allocation); the second,
    # on the same plan, is the steady-state cost the paper reports
    pre = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dp.set_nodes(x)
        dp.precompute()
        torch.cuda.synchronize()
        pre.append(1000 * (time.perf_counter() - t0))
    precompute_cold_ms, precompute_ms = pre
    del x
    fhat = torch.from_numpy(wl.fhat(w)).to(dev, cdt)
    fsamp = dp.scatter(torch.from_numpy(wl.samples(w)).to(dev, cdt))
    f_out = torch.empty(dp.M_local, dtype=cdt, device=dev)
    fhat_out = torch.empty(w.num_freqs, dtype=cdt, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        # adjoint first: at N > 1 its coefficient all-reduce is in flight
        # while the (independent) trafo runs
        _, work = dp.adjoint(fsamp, out=fhat_out, async_op=True)
        dp.trafo(fhat, out=f_out)
        work.wait()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # One rank: the step's launches (deconv, cuFFT, pad, gather, zero,
    # permute, spread, cuFFT, pack) are captured once into a CUDA graph and
    # replayed, so the device does not idle between launches.  The library
    # launches on the caller's (capturing) stream; its ticket counters reset
    # themselves, so a replay is the same work as an eager step.
    run, launches_per_step = step, None
    plan.set_timing(False)
    if world == 1 and not args.no_graph:
        l0 = nf.launch_count()
        step()
        torch.cuda.synchronize()
        launches_per_step = nf.launch_count() - l0
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
        run = graph.replay

    # ---- device-timed region (no per-phase instrumentation inside it)
    plan.set_timing(False)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = nf.launch_count()
    stream = torch.cuda.current_stream()
    total_ms = 0.0
    for _ in range(args.steps):
        flush.fill_(1)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        b.synchronize()
        total_ms += a.elapsed_time(b)
    torch.cuda.synchronize()
    launches = nf.launch_count() - launches0
    if launches_per_step is not None:  # graph replays: the host counter does not see them
        launches = launches_per_step * args.steps
    clk = clocks.stop()
    # ---- the same steps again with per-phase CUDA events (breakdown, roofline)
    plan.phase_times(reset=True)
    plan.set_timing(True)
    for _ in range(args.steps):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    plan.set_timing(False)
    phases = plan.phase_times(reset=True)
    if world > 1:
        dist.barrier()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    value = w.M / (ms_per_step / 1000.0)

    # ---- e2e through the reference-facing C-ABI with host buffers
    e2e = e2e_abi(w, args, rank, world, dp, dev, cdt)

    # ---- roofline of the dominant gridding kernel
    peaks = measured_peaks()
    fp64, fp32 = ctypes_fma_peaks(_lib)
    roof = roofline(w, phases, args.steps, s_elem, peaks, fp64 if s_elem == 16 else fp32,
                    tuple(plan.tile), args.psi, sm_mhz=clk.get("sm_mhz") or clk.get("sm_max_mhz"),
                    gridding=plan.gridding)
    if roof is not None and plan.fft == "pruned":
        roof["other"].update(fft_roofline(w, phases, s_elem, peaks, plan))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    line = {
        "metric": "NFFT trafo+adjoint nodes/sec", "value": value, "unit": "nodes/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c64" if args.precision == "single" else "c128",
        "data": "synthetic (seeded, SURVEY 8(d) generators)",
        "config": config_json(w, args, world),
        "launch": launch_mode(args, world),
        "e2e": e2e,
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clk,
        "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items() if v[1]},
        "precompute_ms": precompute_ms,
        "precompute_cold_ms": precompute_cold_ms,
        "fma_peaks_tflops": {"fp64": fp64, "fp32": fp32},
    }
    if world == 1 and not args.no_cpu_baseline:
        rate, cores, sample = cpu_oracle_rate(w)
        line["cpu_baseline"] = {"value": rate, "unit": "nodes/s", "cores": cores, "kind": "port",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_abi(w, args, rank, world, dp, dev, cdt):
    """Host-buffer end-to-end rate.  N=1: the reference C-ABI (set_fhat/trafo,
    set_f/adjoint) whose buffers are library-owned pinned memory.  N>1: the
    distributed API with pinned host tensors copied in and out every step."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_1810_09891_b200 import _lib

    fh = np.ascontiguousarray(wl.fhat(w)).view(np.float64)
    fs_all = wl.samples(w)
    s_el = 16 if args.precision == "double" else 8
    # whole-job bytes per step: every rank copies the coefficients in and out,
    # the samples are split across the ranks
    h2d = s_el * (world * w.num_freqs + w.M)
    d2h = h2d
    steps = max(3, min(args.steps, 10))
    if world == 1 and args.precision == "double":
        lib = _lib.load()
        N = _lib.i32_array(w.N)
        n = _lib.i32_array(w.n)
        flags = 0x1fd1 if w.d > 1 else 0xfd1
        h = lib.nfftk_create_advanced(N, w.d, w.M, n, w.m, flags, 0x41)
        assert h > 0, h
        x = np.ascontiguousarray(wl.nodes(w))
        assert lib.nfftk_set_x(h, x.ctypes.data, x.size) == 0, lib.nfftk_last_error_message(h)

        fs = np.ascontiguousarray(fs_all).view(np.float64)

        def one():
            rc = lib.nfftk_set_fhat(h, fh.ctypes.data, fh.size) or lib.nfftk_trafo(h)
            rc = rc or lib.nfftk_set_f(h, fs.ctypes.data, fs.size) or lib.nfftk_adjoint(h)
            assert rc == 0, lib.nfftk_last_error_message(h)
            return lib.nfftk_get_f(h), lib.nfftk_get_fhat(h)

        for _ in range(2):
            one()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        ms = 1000 * (time.perf_counter() - t0) / steps
        lib.nfftk_destroy(h)
        path = "C-ABI nfftk_set_fhat+nfftk_trafo+nfftk_set_f+nfftk_adjoint (host buffers)"
    else:
        fhh = torch.from_numpy(wl.fhat(w)).to(cdt).pin_memory()
        fsh = torch.from_numpy(fs_all[dp.shard_index.cpu().numpy()]).to(cdt).pin_memory()
        fo = torch.empty(dp.M_local, dtype=cdt).pin_memory()
        fho = torch.empty(w.num_freqs, dtype=cdt).pin_memory()

        def one():
            a = fhh.to(dev, non_blocking=True)
            b = fsh.to(dev, non_blocking=True)
            fo.copy_(dp.trafo(a), non_blocking=True)
            fho.copy_(dp.adjoint(b), non_blocking=True)
            torch.cuda.synchronize()

        for _ in range(2):
            one()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        ms = 1000 * (time.perf_counter() - t0) / steps
        path = "Plan/DistributedPlan API with pinned host tensors"
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": w.M / (ms / 1000.0), "unit": "nodes/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "path": path, "steps": steps}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "source": "MEASURED_PEAKS.json (measured)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "source": "B200_PROFILING.md fallback"}


def ctypes_fma_peaks(_lib):
    import ctypes

    a, b = ctypes.c_double(), ctypes.c_double()
    _lib.load().nfftk_measure_fma_peaks(ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def ncu_traffic(config, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel`` at
    ``config`` from the committed ncu --set full summary (profiles/*/ncu_traffic.json),
    or None when no capture exists."""
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_traffic.json"))):
        try:
            with open(path) as fh:
                best = json.load(fh).get(config, {}).get(kernel, best)
        except (OSError, ValueError):
            pass
    return best


def kernel_names(w, tile, psi, gridding=None):
    """Names of the interp / spread kernels the library launches for this
    workload (gridding.cu launchers): the pipelined register kernels in
    PRE_PSI mode on their tile geometries, the batch kernels otherwise."""
    tensor = psi in (None, "flags", "tensor")
    k = 2 * w.m + 1
    if gridding == "residue":  # residue.cu: d=3, m=4, 8^3 tiles, complex128
        return {"interp": "k_interp_pipe", "spread": "k_spread_res"}
    if tensor and w.d == 3 and w.m <= 6 and tuple(tile) == (8, 8, 8):
        return {"interp": "k_interp_pipe", "spread": "k_spread_pipe"}
    if tensor and w.d == 2 and w.m <= 8 and tuple(tile) == (32 - k, 8):
        return {"interp": "k_interp_pipe", "spread": "k_spread2_pipe"}
    rr = w.d == 3 and tuple(tile) == (8, 8, 8) and w.m <= 6
    return {"interp": "k_interp", "spread": "k_spread_rr" if rr else "k_spread"}


# What bounds each gridding kernel (ncu summaries in
# profiles/): neither is HBM-bound at these cutoffs; "hbm" is the contract's
# roofline, reported with the compulsory bytes.
BINDING = {
    "interp": "shared-memory wavefronts (one 16-byte halo cell per node-cell)",
    "spread": "instruction issue of the register-resident halo walk (FP64 FMAs plus the per-node "
              "factor loads and control)",
}


def smem_roof(w, s, per_ms, sm_mhz):
    """The gather's on-chip roof: it reads one s-byte halo cell per node-cell
    from shared memory ((2m)^d M cells per launch), against the SMs' shared-
    memory bandwidth of 128 B per clock each (one wavefront) at the SM clock
    sampled during the timed region."""
    import torch

    if not sm_mhz or not torch.cuda.is_available():
        return None
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    alg = (2 * w.m) ** w.d * w.M * s
    achieved = alg / (per_ms * 1e-3) / 1e12
    peak = sms * 128 * sm_mhz * 1e6 / 1e12
    return {"achieved": achieved, "peak": peak, "unit": "TB/s", "frac": achieved / peak,
            "algorithmic_bytes_per_launch": alg,
            "peak_source": f"{sms} SMs x 128 B/clk x {sm_mhz:.0f} MHz (sampled SM clock)"}


def fft_roofline(w, phases, s, peaks, plan):
    """The pruned F / F^H passes (csrc/fft.cu: k_fft_pass, with D, D^H and the
    ghost padding fused in) against measured HBM.  Algorithmic bytes: every
    pass reads its input and writes its output once -- f_hat, the band-compact
    intermediates (n0 N1 N2 and n0 n1 N2 cells for d = 3, n0 N1 for d = 2) and
    the ghost-padded grid (trafo) or the dense grid (adjoint)."""
    import numpy as np

    n, N = w.n, w.N
    inter = []
    for k in range(1, w.d):  # after pass k the first k dims are full, the rest band
        inter.append(int(np.prod(n[:k])) * int(np.prod(N[k:])))
    npad = 1
    for i in range(w.d):
        ntile = -(-n[i] // plan.tile[i])
        npad *= ntile * plan.tile[i] + 2 * w.m + 2
    cells = {"fft_fwd": w.num_freqs + 2 * sum(inter) + npad, "fft_inv": w.grid_size + 2 * sum(inter) + w.num_freqs}
    out = {}
    for ph, c in cells.items():
        ms, calls = phases.get(ph, (0.0, 0))
        if not calls:
            continue
        per = ms / calls
        achieved = c * s / (per * 1e-3) / 1e9
        out[ph] = {"kernel": "k_fft_pass (%d passes incl. %s)" % (w.d, "D + ghost padding" if ph == "fft_fwd" else "pack + D^H"),
                   "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                   "frac": achieved / peaks["hbm_gbs"], "algorithmic_bytes_per_launch": c * s,
                   "avg_launch_ms": per, "peak_source": peaks["source"]}
    return out


def roofline(w, phases, steps, s, peaks, fma_tflops, tile, psi=None, sm_mhz=None, gridding=None):
    """Dominant gridding kernel vs measured HBM (SURVEY 8(d) compulsory bytes:
    M (8d + s) + s |I_n| + 4 M for the permutation) and vs the FMA roof
    (4 w^d M flops with w = 2m).  Times are CUDA-event durations of the kernel
    launches inside the timed region (library phase events on the launch stream)."""
    kernels = kernel_names(w, tile, psi, gridding)
    out = {}
    for ph, kname in kernels.items():
        ms, calls = phases.get(ph, (0.0, 0))
        if not calls:
            continue
        per = ms / calls
        traffic_alg = w.M * (8 * w.d + s + 4) + s * w.grid_size
        achieved = traffic_alg / (per * 1e-3) / 1e9
        flops = 4 * (2 * w.m) ** w.d * w.M
        tflops = flops / (per * 1e-3) / 1e12
        out[ph] = {
            "kernel": kname, "bound": "hbm", "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "traffic": ncu_traffic(w.name, kname), "algorithmic_bytes_per_launch": traffic_alg,
            "avg_launch_ms": per, "peak_source": peaks["source"],
            "binding_resource": BINDING.get(ph, ""),
            "fma": {"achieved_tflops": tflops, "peak_tflops": fma_tflops,
                    "frac": tflops / fma_tflops if fma_tflops else None,
                    "flops_per_launch": flops,
                    "peak_source": "k_fma_peak microbenchmark (measured in run)"},
        }
        if psi in (None, "flags", "tensor"):
            # PRE_PSI mode (the reference's default f1) streams the factor table
            # M x d x (2m+1) doubles (kernels.py:56-72) every transform: with
            # it the compulsory bytes are what the DRAM traffic compares with
            alg_psi = traffic_alg + 8 * w.d * (2 * w.m + 1) * w.M
            out[ph]["hbm_with_pre_psi_table"] = {
                "algorithmic_bytes_per_launch": alg_psi,
                "achieved": alg_psi / (per * 1e-3) / 1e9, "unit": "GB/s",
                "frac": alg_psi / (per * 1e-3) / 1e9 / peaks["hbm_gbs"],
                "traffic_over_algorithmic": (out[ph]["traffic"] / alg_psi) if out[ph]["traffic"] else None}
        if ph == "interp":
            out[ph]["smem"] = smem_roof(w, s, per, sm_mhz)
    if not out:
        return None
    dom = max(out, key=lambda k: out[k]["avg_launch_ms"])
    line = dict(out[dom])
    line["other"] = {k: v for k, v in out.items() if k != dom}
    return line


if __name__ == "__main__":
    sys.exit(main())
