"""Where the host-buffer evaluation's time goes: device-resident eval, host-buffer eval
(pipelined), plain H2D / D2H of the 18 MB params / gradient (pinned), C5."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1804_05061_b200 as S
cfg = synth.config("C5")
F, M = synth.make_pair("C5", 1, cfg["dims"])
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
p = synth.make_params(g.params_shape, "small", 1)
hp = torch.from_numpy(p.copy()).pin_memory(); hg = torch.empty_like(hp).pin_memory()
dp = hp.cuda(); dg = torch.empty_like(dp)
def t(fn, n=30):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
out = {"stats": {k: g.stats()[k] for k in ("pipe_items1", "pipe_items2", "items", "items2")},
       "device_eval_ms": t(lambda: g.eval(dp, grad=dg)),
       "host_eval_ms": t(lambda: g.eval(hp, grad=hg)),
       "h2d_18MB_ms": t(lambda: dp.copy_(hp, non_blocking=True)),
       "d2h_18MB_ms": t(lambda: hg.copy_(dg, non_blocking=True))}
print(json.dumps(out))
