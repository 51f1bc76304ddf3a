"""Generate golden vectors by running the LIVE reference package ``nfftk``.

Run here (the reference exists only in this container, never on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (committed): ``tests/golden/*.npz``.  ``make_golden.py C3 C4 C5`` runs
the reference at those configurations' full sizes (C5: ~6 min, ~33 GB RSS on
8 cores) and writes ``<C>_full.npz``: 65,536 seeded entries of trafo and of
adjoint plus whole-vector norms, sums and 4,096 block sums.  Inputs are regenerated from the
seeds in ``paper_1810_09891_b200/workloads.py`` and stored alongside for the
small cases, so the fixtures are self-contained.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import nfftk  # noqa: E402  (the reference; PYTHONPATH must point at it)
from nfftk import indexing, transform, window  # noqa: E402

from paper_1810_09891_b200 import workloads as wl  # noqa: E402


def run_case(N, n, m, x, fhat, f, f1=None, win="kaiserbessel", threads=None):
    if threads is not None:
        nfftk.set_threads(threads)
    p = nfftk.Plan(N, x.shape[0], n=n, m=m, f1=f1, window=win)
    p.x = x
    p.precompute()
    out_f = p.trafo(fhat)
    out_fhat = p.adjoint(f)
    order = p.node_order
    return out_f, out_fhat, order, p


def small_cases():
    """Edge cases: d = 1..3, both windows, LUT mode, Bluestein n, grid-aligned
    nodes (width 2m+1, u == 0 window branch), nodes at -1/2, M = 1."""
    cases = {}
    rng = np.random.default_rng(7)

    def add(name, N, n, m, x, f1=None, win="kaiserbessel"):
        K = int(np.prod(N))
        fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
        fs = rng.standard_normal(x.shape[0]) + 1j * rng.standard_normal(x.shape[0])
        out_f, out_fhat, order, p = run_case(N, n, m, x, fh, fs, f1=f1, win=win)
        cases[name] = dict(N=np.array(N), n=np.array(n), m=m, x=x, fhat=fh, f=fs,
                           trafo=out_f, adjoint=out_fhat,
                           order=order if order is not None else np.array([], np.int64),
                           f1=p.f1, window=win,
                           ndft=transform.ndft(p, fh), ndft_adjoint=transform.ndft_adjoint(p, fs))

    add("d1_small", (16,), (32,), 4, rng.random((40, 1)) - 0.5)
    add("d1_m8", (512,), (1024,), 8, rng.random((1024, 1)) - 0.5)
    # grid-aligned and boundary nodes: x = j / n exactly, including -1/2
    xa = np.array([[-0.5], [0.0], [0.25], [-0.25], [31 / 64], [-31 / 64], [1 / 64]])
    add("d1_aligned", (32,), (64,), 5, xa)
    add("d1_bluestein", (16,), (20,), 3, rng.random((33, 1)) - 0.5)
    add("d1_gauss", (32,), (64,), 6, rng.random((50, 1)) - 0.5, win="gaussian")
    add("d1_lut", (32,), (64,), 6, rng.random((50, 1)) - 0.5, f1=nfftk.PRE_PHI_HUT | nfftk.PRE_LIN_PSI)
    add("d1_direct", (32,), (64,), 6, rng.random((50, 1)) - 0.5, f1=nfftk.PRE_PHI_HUT)
    add("d1_M1", (4,), (16,), 2, np.array([[0.0]]))
    add("d2_small", (16, 8), (32, 20), 3, rng.random((300, 2)) - 0.5)
    add("d2_m8", (32, 32), (64, 64), 8, rng.random((700, 2)) - 0.5)
    xb = rng.random((64, 2)) - 0.5
    xb[:8] = np.array([[-0.5, -0.5], [-0.5, 0.0], [0.0, -0.5], [0.0, 0.0],
                       [0.25, -0.125], [-0.5, 15 / 32], [15 / 32, 15 / 32], [-1 / 32, 3 / 32]])
    add("d2_aligned", (16, 16), (32, 32), 4, xb)
    add("d2_gauss", (16, 16), (32, 32), 5, rng.random((200, 2)) - 0.5, win="gaussian")
    add("d2_lut", (16, 16), (32, 32), 5, rng.random((200, 2)) - 0.5, f1=nfftk.PRE_PHI_HUT | nfftk.PRE_LIN_PSI)
    add("d2_clustered", (32, 32), (64, 64), 6, wl.clustered_nodes(2000, 2, seed=3))
    add("d3_small", (8, 8, 8), (16, 16, 16), 3, rng.random((200, 3)) - 0.5)
    add("d3_m6", (16, 16, 16), (32, 32, 32), 6, rng.random((500, 3)) - 0.5)
    add("d3_aniso", (8, 16, 12), (16, 24, 32), 4, rng.random((300, 3)) - 0.5)
    xc = rng.random((40, 3)) - 0.5
    xc[:4] = np.array([[-0.5, -0.5, -0.5], [0.0, 0.0, 0.0], [0.25, -0.5, 0.125], [-0.5, 7 / 16, 0.0]])
    add("d3_aligned", (8, 8, 8), (16, 16, 16), 4, xc)
    add("d3_lut", (8, 8, 8), (16, 16, 16), 4, rng.random((100, 3)) - 0.5, f1=nfftk.PRE_PHI_HUT | nfftk.PRE_LIN_PSI)
    add("d3_gauss", (8, 8, 8), (16, 16, 16), 4, rng.random((100, 3)) - 0.5, win="gaussian")
    return cases


def config_case(name, full, sub=4096):
    """One BASELINE configuration at its FULL size through the reference Plan
    (default flags, all reference threads).  ``full`` stores both output
    vectors; otherwise ``sub`` seeded entries of each plus whole-vector norms,
    sums and a checksum of per-block sums (so a GPU run at full size is
    compared entry-wise on the subsample and vector-wide through the sums)."""
    w = wl.CONFIGS[name]
    x = wl.nodes(w)
    fh = wl.fhat(w)
    fs = wl.samples(w)
    out_f, out_fhat, _, _ = run_case(w.N, w.n, w.m, x, fh, fs)
    rec = dict(norm_f=np.linalg.norm(out_f), norm_fhat=np.linalg.norm(out_fhat),
               sum_f=out_f.sum(), sum_fhat=out_fhat.sum(),
               blocksum_f=block_sums(out_f), blocksum_fhat=block_sums(out_fhat))
    if full:
        rec.update(trafo=out_f, adjoint=out_fhat)
    else:
        sel = np.random.default_rng(11)
        jf = np.sort(sel.choice(w.M, min(sub, w.M), replace=False))
        jk = np.sort(sel.choice(w.num_freqs, min(sub, w.num_freqs), replace=False))
        rec.update(trafo_idx=jf.astype(np.int64), trafo_sub=out_f[jf],
                   adjoint_idx=jk.astype(np.int64), adjoint_sub=out_fhat[jk])
    return rec


BLOCKS = 4096


def block_sums(v, blocks=BLOCKS):
    """Sums of ``blocks`` contiguous equal slices (the last absorbs the rest):
    a size-independent whole-vector check that localises a wrong region."""
    edges = (np.arange(blocks + 1, dtype=np.int64) * v.size) // blocks
    return np.add.reduceat(v, edges[:-1])


def pins():
    """Scalar pins from the reference's own tests and modules."""
    out = {}
    r = indexing.gather_range((0.1,), (16,), 2)
    out["gr_interior"] = np.array([r.lo[0], r.hi[0]])
    r = indexing.gather_range((-0.5,), (16,), 2)
    out["gr_left"] = np.array([r.lo[0], r.hi[0]])
    out["gr_left_cells"] = r.cells(0, 16)
    r = indexing.gather_range((0.0,), (8,), 1)
    out["gr_centered"] = np.array([r.lo[0], r.hi[0]])
    t = np.linspace(0, 120, 241)
    out["i0_x"] = t
    out["i0"] = np.array([window.bessel_i0(v) for v in t])
    for kind in ("kaiserbessel", "gaussian"):
        for (N, n, m) in [(16, 32, 4), (1024, 2048, 8), (64, 128, 6), (256, 512, 4), (16, 20, 3)]:
            w = window.WindowModel.make(kind, (N,), (n,), m)
            key = f"{kind}_{N}_{n}_{m}"
            out["phihat_" + key] = w.phi_hat_table(0, kmax=N // 2)
            ts = np.linspace(-m / n, m / n, 101)
            out["phi_t_" + key] = ts
            out["phi_" + key] = w.phi(ts)
            out["b_" + key] = np.array(w.b)
    rng = np.random.default_rng(5)
    for d, n, m in [(1, (32,), 4), (2, (16, 12), 3), (3, (16, 16, 16), 6)]:
        x = rng.random((100, d)) - 0.5
        lo, width = indexing.node_ranges(x, n, m)
        out[f"ranges_x_{d}"] = x
        out[f"ranges_lo_{d}"] = lo
        out[f"ranges_w_{d}"] = width
    out["default_f1_1"] = np.array(nfftk.default_f1(1))
    out["default_f1_3"] = np.array(nfftk.default_f1(3))
    out["default_n"] = np.array(nfftk.default_n((1000, 64, 6)))
    return out


def main():
    big = [a for a in sys.argv[1:] if a in ("C3", "C4", "C5")]
    if big:
        # full-size goldens for the large configs: 65,536 entries of each output
        for name in big:
            rec = config_case(name, False, sub=65536)
            np.savez_compressed(os.path.join(HERE, f"{name}_full.npz"), **rec)
            print(name, "full-size golden done", flush=True)
        return
    os.makedirs(HERE, exist_ok=True)
    threads = nfftk.get_threads()
    print("reference threads:", threads)
    cases = small_cases()
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"),
                        **{f"{k}__{f}": v for k, rec in cases.items() for f, v in rec.items()})
    np.savez_compressed(os.path.join(HERE, "pins.npz"), **pins())
    for name, full in (("C1", True), ("C2", True), ("C3", False)):
        rec = config_case(name, full)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
        print(name, "done")


if __name__ == "__main__":
    main()
