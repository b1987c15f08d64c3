"""Multi-resolution SRWCR registration.

"The multi-resolution strategy and the concatenation of three isotropic control grids
are used", "the maximal iteration is set to 200, 200, 120 for low, medium
and high resolution".  Reading c21: level k of `levels` registers the
2^(levels-1-k)-times downsampled fixed image against the moving image already warped by
the composed field of the coarser levels, on a fresh control grid whose spacing is the
finest spacing in that level's voxels (so the three grids are isotropic with physical
spacings 4δ, 2δ, δ); each level's field is upsampled to full resolution and composed
with the running field (backward warps: U <- u_k + U(x + u_k)).  Every step runs in the
library's kernels (srwcr_register, srwcr_field, srwcr_resample, srwcr_compose,
srwcr_downsample2, srwcr_upsample2_field); torch only holds device memory.
"""
from __future__ import annotations

import numpy as np

from . import Srwcr, compose, downsample2, resample, upsample2_field


def register_multires(fixed, moving, spacing_mm, bins, spatial_bins, control_vox=5.0, levels=3,
                      iters=(200, 200, 120), w_p=0.1, verbose=False, orientation=0, **lbfgs):
    """Register moving onto fixed (fp32 CUDA tensors [Nz, Ny, Nx], raw intensities).

    control_vox: control spacing in voxels at every level (paper: 5 at the finest).
    spatial_bins: k cells per axis at every level, or "control": spatial bins = control
    cells at each level (k = round(N_level / control_vox) per axis; the paper's setting,
    P:91).  orientation: 0 = moving as the estimated image B, 1 = moving as the model A.
    Returns (U, reports): U = total displacement field [3, Nz, Ny, Nx] (full resolution,
    voxels) such that moving(x + U(x)) ~ fixed(x); reports = per-level L-BFGS reports."""
    import torch
    if len(iters) < levels:
        iters = tuple(iters) + (iters[-1],) * (levels - len(iters))
    shape = tuple(fixed.shape)
    shapes = [shape]   # pyramid shapes: ceil(N / 2) per level (a 1-slice z axis stays 1)
    for _ in range(levels - 1):
        nz, ny, nx = shapes[-1]
        shapes.append(((nz + 1) // 2 if nz > 1 else 1, (ny + 1) // 2, (nx + 1) // 2))
    U = torch.zeros((3, *shape), dtype=torch.float32, device=fixed.device)
    reports = []
    for k in range(levels):
        down = levels - 1 - k
        Mw = resample(moving, U)
        Fk, Mk = fixed, Mw
        for _ in range(down):
            Fk, Mk = downsample2(Fk), downsample2(Mk)
        scale = np.array([2.0 ** down, 2.0 ** down, 2.0 ** down if shape[0] > 1 else 1.0])
        sp = np.asarray(spacing_mm, dtype=np.float64) * scale
        if isinstance(spatial_bins, str):   # "control": one spatial cell per control cell
            sb = tuple(max(1, int(round(n / control_vox))) if n > 1 else 0 for n in tuple(Fk.shape)[::-1])
        else:
            sb = spatial_bins
        g = Srwcr(Fk, Mk, tuple(sp), bins, sb, tuple(control_vox * sp), orientation=orientation)
        try:
            x, rep = g.register(None, w_p=w_p, max_iter=int(iters[k]), verbose=int(verbose), **lbfgs)
            uk = torch.from_numpy(g.field(x)).to(fixed.device)
        finally:
            g.close()
        rep["level"], rep["dims"] = k, tuple(Fk.shape)
        reports.append(rep)
        for j in range(down, 0, -1):   # back up the pyramid to full resolution
            uk = upsample2_field(uk, shapes[j - 1])
        U = compose(U, uk)
    return U, reports
