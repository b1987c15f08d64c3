"""CUPTI timeline (torch.profiler) of host-buffer evaluations: kernels and copies per stream."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_1804_05061_b200 as S
cfg = synth.config("C5")
F, M = synth.make_pair("C5", 1, cfg["dims"])
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
p = synth.make_params(g.params_shape, "small", 1)
hp = torch.from_numpy(p.copy()).pin_memory(); hg = torch.empty_like(hp).pin_memory()
for _ in range(3): g.eval(hp, grad=hg)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for _ in range(3): g.eval(hp, grad=hg)
    torch.cuda.synchronize()
prof.export_chrome_trace(sys.argv[1])
