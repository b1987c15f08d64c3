"""One rank of a P-rank z-slab decomposition on one GPU (exchange skipped): for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1804_05061_b200 as S

name, P, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = synth.config(name)
F, M = synth.make_pair(name, 1, cfg["dims"])
Fd, Md = torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda()
g = S.Srwcr(Fd, Md, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=P, rank=r)
p = torch.from_numpy(synth.make_params(g.params_shape, "small", 1)).cuda()
gr = torch.empty_like(p)
for i in range(4):
    g.eval_begin(p)
    g.eval_end(grad=gr)
torch.cuda.synchronize()
print("ok", g.stats())
