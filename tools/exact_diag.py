"""Diagnose how many voxels take pass 2's fp64 exact-sample path at given params
(tools only: torch re-implementation of the FFD + trilinear for counting)."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = synth.config(name)
d = np.load(f"/tmp/srwcr_{name}.npz"); F, M = d["F"], d["M"]
phi = np.load(f"/tmp/srwcr_{name}_reg.npy") if len(sys.argv) < 3 else synth.make_params(None, "small")
nx, ny, nz = cfg["dims"]
L = cfg["bins"] - 1
delta = [c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])]
dev = "cuda"
def bmat(N, dl, G):
    B = torch.zeros(N, G, dtype=torch.float64)
    for i in range(N):
        s = i / dl; b = int(np.floor(s)); t = s - b
        w = [(1 - t) ** 3 / 6, (3 * t ** 3 - 6 * t * t + 4) / 6, (-3 * t ** 3 + 3 * t * t + 3 * t + 1) / 6, t ** 3 / 6]
        for k in range(4):
            B[i, b + k] = w[k]
    return B.to(dev)
nd, Gz, Gy, Gx = phi.shape
Bx, By, Bz = bmat(nx, delta[0], Gx), bmat(ny, delta[1], Gy), bmat(nz, delta[2], Gz)
P = torch.from_numpy(phi).to(dev)
Mt = torch.from_numpy(M).to(dev).double()
lo, hi = Mt.min(), Mt.max()
Mn = ((Mt - lo) * (L / (hi - lo))).float().clamp(0, L)
stats = {"voxels": nx * ny * nz}
cnt = {"nrx": 0, "nry": 0, "nrz": 0, "mnear": 0, "mnear_nonflat": 0, "any": 0, "clamped_any": 0}
for z0 in range(0, nz, 16):
    z1 = min(nz, z0 + 16)
    ffd = lambda Q: torch.einsum("zk,kyx->zyx", Bz[z0:z1], torch.einsum("yj,kjx->kyx", By, torch.einsum("xi,kji->kjx", Bx, Q))).float()
    u = [ffd(P[c]) for c in range(3)]
    Pf = P.float().abs()
    pad = torch.nn.functional.pad
    Wm = torch.nn.functional.max_pool3d(pad(Pf, (0, 3, 0, 3, 0, 3)).unsqueeze(0), 4, stride=1)[0]  # window max at base
    bx = (torch.arange(nx, device=dev) / delta[0]).floor().long(); by = (torch.arange(ny, device=dev) / delta[1]).floor().long()
    bz = (torch.arange(z0, z1, device=dev) / delta[2]).floor().long()
    A = [Wm[c][bz][:, by][:, :, bx] for c in range(3)]
    zz, yy, xx = torch.meshgrid(torch.arange(z0, z1, device=dev), torch.arange(ny, device=dev), torch.arange(nx, device=dev), indexing="ij")
    near, cl, cells, ts = [], [], [], []
    for ax, (base, N) in enumerate(((xx, nx), (yy, ny), (zz, nz))):
        uu = u[ax]
        fu = torch.floor(uu); c = base + fu.int(); t = uu - fu
        tol = 4e-6 * A[ax]
        nr = (uu - torch.round(uu)).abs() < tol
        out_lo = c < 0; out_hi = c > N - 2
        nr = torch.where(out_lo, (c == -1) & nr, nr)
        nr = torch.where(out_hi, (c == N - 1) & nr, nr)
        clm = out_lo | (out_hi & ~((c == N - 1) & (t == 0)))
        t = torch.where(out_lo, torch.zeros_like(t), torch.where(out_hi, torch.ones_like(t), t))
        c = c.clamp(0, N - 2)
        near.append(nr); cl.append(clm); cells.append(c.long()); ts.append(t)
    cx, cy, cz = cells
    def g(dx, dy, dz):
        return Mn[cz + dz, cy + dy, cx + dx]
    cs = [g(a, b, c) for c in (0, 1) for b in (0, 1) for a in (0, 1)]
    tx, ty, tz = ts
    e00 = cs[0] + tx * (cs[1] - cs[0]); e10 = cs[2] + tx * (cs[3] - cs[2])
    e01 = cs[4] + tx * (cs[5] - cs[4]); e11 = cs[6] + tx * (cs[7] - cs[6])
    f0 = e00 + ty * (e10 - e00); f1 = e01 + ty * (e11 - e01); m = f0 + tz * (f1 - f0)
    n = torch.floor(m).clamp(0, L - 1); fm = m - n
    mn = (fm < 5e-5) | (fm > 1 - 5e-5)
    flat = torch.ones_like(mn)
    for k in range(1, 8): flat &= cs[k] == cs[0]
    w = (near[0] | near[1] | near[2] | (mn & ~flat)).reshape(z1 - z0, ny, -1, 32).any(-1) if nx % 32 == 0 else None
    if w is not None: cnt["warps_any"] = cnt.get("warps_any", 0) + int(w.sum()); cnt["warps"] = cnt.get("warps", 0) + w.numel()
    cnt["nrx"] += int(near[0].sum()); cnt["nry"] += int(near[1].sum()); cnt["nrz"] += int(near[2].sum())
    cnt["mnear"] += int(mn.sum()); cnt["mnear_nonflat"] += int((mn & ~flat).sum())
    cnt["any"] += int((near[0] | near[1] | near[2] | (mn & ~flat)).sum())
    cnt["clamped_any"] += int((cl[0] | cl[1] | cl[2]).sum())
stats.update(cnt)
print(json.dumps(stats))
