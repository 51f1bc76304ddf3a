"""torch.profiler view of one warm set_nodes + precompute (host API calls and kernels).
usage: python tools/precompute_profile.py C1"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1810_09891_b200 as nf
from paper_1810_09891_b200 import workloads as wl
name = sys.argv[1]
w = wl.CONFIGS[name]
p = nf.Plan(w.N, w.M, n=w.n, m=w.m)
x = torch.from_numpy(wl.nodes(w)).cuda()
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter(); p.set_nodes(x); torch.cuda.synchronize(); t1 = time.perf_counter(); p.precompute(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(name, it, f"set_nodes {1e3*(t1-t0):.2f} precompute {1e3*(t2-t1):.2f}")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    p.set_nodes(x); p.precompute(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
