"""Seeded synthetic inputs for the SRWCR hot path (shared by the oracle tests, the GPU
parity tests and bench.py).

This module holds NONE of the method's arithmetic: no B-spline FFD, no Parzen
window, no histogram, no normalization to [0, L].  Moving images are produced by
evaluating analytic phantoms at coordinates displaced by smooth analytic fields
(and numpy/scipy library primitives), never by the transform being tested.  It
returns RAW intensities; both the oracle and the library normalize them.

Workloads follow SURVEY.md s8(d) and BASELINE.json ``configs`` (the recipe is
restated in DESIGN.md s4):
  C1  2-D 64x64 pair, 4x4 spatial cells, 32 bins, 8x8 control cells
  C2  3-D 128^3 binary grid pair (paper s.III-A), 4^3 cells, 32 bins
  C3  4-D thoracic CT-shaped 256x256x128 (DIR-Lab-like), 64 bins
  C4  retinal OCT-shaped 512x128x1024 with multiplicative speckle
  C5  multi-modal CT/PET-shaped 512x512x320, 8^3 cells, 128 bins
Every generator is a pure function of (config, seed, dims).
"""
from __future__ import annotations

import numpy as np
from scipy import ndimage

# name -> workload geometry.  spacing / control spacing in mm; control spacing in
# voxels = control_mm / spacing_mm; spatial_cells = k cells per axis.
CONFIGS = {
    "C1": dict(dims=(64, 64, 1), spacing=(1.0, 1.0, 1.0), bins=32, cells=(4, 4, 0),
               control_mm=(8.0, 8.0, 8.0), desc="2-D synthetic pair 64x64"),
    "C2": dict(dims=(128, 128, 128), spacing=(1.0, 1.0, 1.0), bins=32, cells=(4, 4, 4),
               control_mm=(5.0, 5.0, 5.0), desc="3-D 128^3 binary grid + B-spline-like warp + bias"),
    "C3": dict(dims=(256, 256, 128), spacing=(1.0, 1.0, 2.5), bins=64, cells=(8, 8, 8),
               control_mm=(5.0, 5.0, 5.0), desc="4-D thoracic CT-shaped inhale/exhale pair"),
    "C4": dict(dims=(512, 128, 1024), spacing=(1.0, 1.0, 1.0), bins=32, cells=(8, 8, 8),
               control_mm=(5.0, 5.0, 5.0), desc="retinal OCT-shaped pair with speckle"),
    "C5": dict(dims=(512, 512, 320), spacing=(1.3, 1.3, 3.0), bins=128, cells=(8, 8, 8),
               control_mm=(6.5, 6.5, 15.0), desc="multi-modal CT/PET-shaped pair"),
}


def config(name: str, dims=None) -> dict:
    """Geometry of a config, optionally at reduced dims (same physical extent ratio)."""
    c = dict(CONFIGS[name])
    if dims is not None:
        c["dims"] = tuple(int(d) for d in dims)
    return c


def _grid(dims, z0, z1):
    """Normalized coordinates in [0,1] (x, y, z) for slices [z0, z1)."""
    nx, ny, nz = dims
    x = (np.arange(nx, dtype=np.float32) + 0.5) / nx
    y = (np.arange(ny, dtype=np.float32) + 0.5) / ny
    z = (np.arange(z0, z1, dtype=np.float32) + 0.5) / max(nz, 1)
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return X, Y, Z


def _smooth_field(rng, dims, coarse, amp):
    """Smooth random scalar field on `dims` ([Nz,Ny,Nx]): uniform(-amp, amp) values on a
    coarse lattice, upsampled by scipy cubic-spline zoom (a library primitive)."""
    nx, ny, nz = dims
    cshape = tuple(max(2, c) for c in coarse)[::-1]
    c = rng.uniform(-amp, amp, size=cshape).astype(np.float32)
    out_shape = (nz, ny, nx)
    zoom = [o / s for o, s in zip(out_shape, cshape)]
    f = ndimage.zoom(c, zoom, order=3, mode="nearest", grid_mode=True)
    f = f[: out_shape[0], : out_shape[1], : out_shape[2]]
    if f.shape != out_shape:
        pad = [(0, o - s) for o, s in zip(out_shape, f.shape)]
        f = np.pad(f, pad, mode="edge")
    return f.astype(np.float32)


def _chunks(nz, step):
    for z0 in range(0, nz, step):
        yield z0, min(nz, z0 + step)


# --------------------------------------------------------------------- C1 (2-D)

def _c1(rng, dims):
    nx, ny, _ = dims
    X, Y, _Z = _grid(dims, 0, 1)
    X, Y = X[0], Y[0]
    blobs = [(rng.uniform(0.1, 0.9), rng.uniform(0.1, 0.9), rng.uniform(4, 10) / nx, rng.uniform(0.5, 2.0))
             for _ in range(12)]
    period = 16.0 / nx

    def phantom(xx, yy):
        img = np.zeros_like(xx)
        for cx, cy, s, a in blobs:
            img += a * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))
        gx = (np.mod(xx, period) < 2.0 / nx) | (np.mod(yy, period) < 2.0 / nx)
        return img + 1.5 * gx.astype(np.float32)

    F = ndimage.gaussian_filter(phantom(X, Y), 0.6)
    dx = _smooth_field(rng, (nx, ny, 1), (9, 9, 1), 2.0)[0] / nx
    dy = _smooth_field(rng, (nx, ny, 1), (9, 9, 1), 2.0)[0] / ny
    bias = np.exp(0.2 * _smooth_field(rng, (nx, ny, 1), (5, 5, 1), 1.0)[0])
    M = ndimage.gaussian_filter(phantom(X + dx, Y + dy), 0.6) * bias
    M = M + rng.normal(0, 0.3 * M.std() / 3, size=M.shape).astype(np.float32)
    return F[None].astype(np.float32), M[None].astype(np.float32)


# -------------------------------------------------------------- C2 (s.III-A grid)

def _c2(rng, dims):
    nx, ny, nz = dims
    L = 31.0
    period, thick = 16.0, 2.0

    def grid_img(px, py, pz):
        on = ((np.mod(px, period) < thick).astype(np.int8) + (np.mod(py, period) < thick).astype(np.int8)
              + (np.mod(pz, period) < thick).astype(np.int8)) >= 2
        return np.where(on, L, 0.0).astype(np.float32)

    iz, iy, ix = np.meshgrid(np.arange(nz, dtype=np.float32), np.arange(ny, dtype=np.float32),
                             np.arange(nx, dtype=np.float32), indexing="ij")
    F = ndimage.gaussian_filter(grid_img(ix, iy, iz), 0.7)
    coarse = (nx // 32 + 2, ny // 32 + 2, nz // 32 + 2)
    d = [_smooth_field(rng, dims, coarse, 15.0) for _ in range(3)]
    bias = np.exp(0.3 * _smooth_field(rng, dims, (5, 5, 5), 1.0))
    M = ndimage.gaussian_filter(grid_img(ix + d[0], iy + d[1], iz + d[2]), 0.7) * bias
    M = M + rng.normal(0, 0.5, size=M.shape).astype(np.float32)
    return F.astype(np.float32), M.astype(np.float32)


# ------------------------------------------------------------- C3/C5 CT phantom

def _ct_geometry(rng, vessels: bool):
    g = dict(
        body=(0.5, 0.5, 0.42, 0.33),
        lungs=[(0.33, 0.47, 0.55, 0.12, 0.17, 0.42), (0.67, 0.47, 0.55, 0.12, 0.17, 0.42)],
        spine=(0.5, 0.74, 0.05),
        ribs=[(0.5, 0.5, 0.40, 0.31, zc) for zc in np.linspace(0.25, 0.85, 7)],
        diaphragm_z=0.2,
        heart=(0.55, 0.52, 0.45, 0.09),
        liver=(0.38, 0.55, 0.12, 0.14, 0.12, 0.10),
    )
    if vessels:
        pts = []
        for _ in range(200):
            lung = g["lungs"][rng.integers(2)]
            p = np.array([lung[0], lung[1], lung[2]]) + rng.uniform(-0.6, 0.6, 3) * np.array(lung[3:6])
            direc = rng.normal(size=3)
            direc /= np.linalg.norm(direc)
            r = rng.uniform(1.0, 3.0)
            n = 24
            for k in range(n):
                pts.append((*(p + direc * 0.006 * k), r))
        g["vessel_pts"] = np.array(pts, dtype=np.float32)
    return g


def _ct_hu(g, X, Y, Z, dims, spacing, exhale_shift=None, lung_hu=-850.0):
    """CT in HU on normalized coordinates; exhale_shift: callable giving the superior-
    inferior (z, normalized) displacement of the anatomy (diaphragm motion)."""
    if exhale_shift is not None:
        Z = Z + exhale_shift(X, Y, Z)
    bx, by, ax, ay = g["body"]
    body = ((X - bx) / ax) ** 2 + ((Y - by) / ay) ** 2 < 1.0
    img = np.where(body, 40.0, -1000.0).astype(np.float32)
    dz = g["diaphragm_z"]
    for (cx, cy, cz, rx, ry, rz) in g["lungs"]:
        inside = ((X - cx) / rx) ** 2 + ((Y - cy) / ry) ** 2 + ((Z - cz) / rz) ** 2 < 1.0
        inside &= Z > dz + 0.08 * ((X - cx) / rx) ** 2
        img = np.where(inside, lung_hu, img)
    sx, sy, sr = g["spine"]
    img = np.where(((X - sx) ** 2 + (Y - sy) ** 2) < sr * sr, 700.0, img)
    for (cx, cy, ax2, ay2, zc) in g["ribs"]:
        ring = np.abs(((X - cx) / ax2) ** 2 + ((Y - cy) / ay2) ** 2 - 1.0) < 0.035
        img = np.where(ring & (np.abs(Z - zc) < 0.012), 700.0, img)
    return img


def _vessel_volume(g, dims, spacing):
    nx, ny, nz = dims
    vol = np.zeros((nz, ny, nx), dtype=np.float32)
    p = g["vessel_pts"]
    ix = np.clip((p[:, 0] * nx).astype(np.int64), 0, nx - 1)
    iy = np.clip((p[:, 1] * ny).astype(np.int64), 0, ny - 1)
    iz = np.clip((p[:, 2] * nz).astype(np.int64), 0, nz - 1)
    np.add.at(vol, (iz, iy, ix), 1.0)
    sig = [max(0.5, 1.5 / s) for s in (spacing[2], spacing[1], spacing[0])]
    vol = ndimage.gaussian_filter(vol, sig)
    return (vol > 0.02).astype(np.float32)


def _diaphragm(amp_norm):
    def f(X, Y, Z):
        # largest at the lung base, decaying apically (P:291 inhale/exhale)
        return amp_norm * np.clip(1.0 - (Z - 0.2) / 0.7, 0.0, 1.0) ** 2 * (1.0 - 2.0 * (Y - 0.5) ** 2)
    return f


def _c3(rng, dims, spacing):
    nx, ny, nz = dims
    g = _ct_geometry(rng, vessels=True)
    ves = _vessel_volume(g, dims, spacing)
    amp = 15.0 / (nz * spacing[2])          # <= 15 mm superior-inferior
    F = np.empty((nz, ny, nx), np.float32)
    M = np.empty((nz, ny, nx), np.float32)
    for z0, z1 in _chunks(nz, 32):
        X, Y, Z = _grid(dims, z0, z1)
        f = _ct_hu(g, X, Y, Z, dims, spacing)
        f = np.where((f < -500) & (f > -900) & (ves[z0:z1] > 0), f + 890.0, f)
        F[z0:z1] = f
        m = _ct_hu(g, X, Y, Z, dims, spacing, exhale_shift=_diaphragm(amp), lung_hu=-700.0)
        M[z0:z1] = m
    F += rng.normal(0, 20.0, size=F.shape).astype(np.float32)
    M += rng.normal(0, 20.0, size=M.shape).astype(np.float32)
    return np.clip(F, -1000, 1000), np.clip(M, -1000, 1000)


def _pet_activity(g, X, Y, Z, spheres, exhale_shift=None):
    if exhale_shift is not None:
        Z = Z + exhale_shift(X, Y, Z)
    bx, by, ax, ay = g["body"]
    body = ((X - bx) / ax) ** 2 + ((Y - by) / ay) ** 2 < 1.0
    act = np.where(body, 1.0, 0.0).astype(np.float32)
    dz = g["diaphragm_z"]
    for (cx, cy, cz, rx, ry, rz) in g["lungs"]:
        inside = ((X - cx) / rx) ** 2 + ((Y - cy) / ry) ** 2 + ((Z - cz) / rz) ** 2 < 1.0
        inside &= Z > dz + 0.08 * ((X - cx) / rx) ** 2
        act = np.where(inside, 0.3, act)
    hx, hy, hz, hr = g["heart"]
    act = np.where(((X - hx) ** 2 + (Y - hy) ** 2 + (Z - hz) ** 2) < hr * hr, 3.0, act)
    lx, ly, lz, lrx, lry, lrz = g["liver"]
    act = np.where(((X - lx) / lrx) ** 2 + ((Y - ly) / lry) ** 2 + ((Z - lz) / lrz) ** 2 < 1.0, 3.0, act)
    sx, sy, sr = g["spine"]
    act = np.where(((X - sx) ** 2 + (Y - sy) ** 2) < sr * sr, 1.2, act)
    for (cx, cy, cz, r) in spheres:
        act = np.where(((X - cx) ** 2 + (Y - cy) ** 2 + (Z - cz) ** 2) < r * r, 8.0, act)
    return act


def _c5(rng, dims, spacing):
    nx, ny, nz = dims
    g = _ct_geometry(rng, vessels=False)
    spheres = [(rng.uniform(0.3, 0.7), rng.uniform(0.35, 0.6), rng.uniform(0.3, 0.8), rng.uniform(0.015, 0.03))
               for _ in range(int(rng.integers(5, 11)))]
    amp = 15.0 / (nz * spacing[2])
    F = np.empty((nz, ny, nx), np.float32)
    M = np.empty((nz, ny, nx), np.float32)
    for z0, z1 in _chunks(nz, 16):
        X, Y, Z = _grid(dims, z0, z1)
        F[z0:z1] = _ct_hu(g, X, Y, Z, dims, spacing)
        M[z0:z1] = _pet_activity(g, X, Y, Z, spheres, exhale_shift=_diaphragm(amp))
    F += rng.normal(0, 20.0, size=F.shape).astype(np.float32)
    np.clip(F, -1000, 1000, out=F)
    # PET: blur FWHM 6 mm, then noise with variance proportional to intensity
    sig = [6.0 / 2.355 / s for s in (spacing[2], spacing[1], spacing[0])]
    M = ndimage.gaussian_filter(M, sig)
    M += (np.sqrt(np.maximum(M, 0.0)) * 0.15 * rng.standard_normal(size=M.shape, dtype=np.float32))
    return F, M.astype(np.float32)


# ------------------------------------------------------------------- C4 OCT

def _c4(rng, dims):
    nx, ny, nz = dims
    # 11 smooth surfaces z = s_k(x, y) (depth, normalized), 10 layers between them
    base = np.sort(rng.uniform(0.25, 0.75, 11)).astype(np.float32)
    gaps = np.diff(base)
    refl = rng.uniform(0.2, 1.0, 10).astype(np.float32)
    undul = [(rng.uniform(0.005, 0.02), rng.uniform(1, 3), rng.uniform(0, 6.28), rng.uniform(0.5, 2))
             for _ in range(11)]
    X2, Y2 = np.meshgrid((np.arange(nx, dtype=np.float32) + 0.5) / nx,
                         (np.arange(ny, dtype=np.float32) + 0.5) / ny, indexing="xy")

    def surfaces(xx, yy):
        s = []
        for k in range(11):
            a, f, ph, fy = undul[k]
            sk = base[k] + a * np.sin(2 * np.pi * f * xx + ph) * np.cos(np.pi * fy * yy)
            s.append(sk)
        # keep order
        for k in range(1, 11):
            s[k] = np.maximum(s[k], s[k - 1] + 0.25 * gaps[k - 1])
        return s

    dz_ax = _smooth_field(rng, (nx, ny, 1), (6, 4, 1), 20.0)[0] / nz     # axial warp <= 20 vox
    dx_lat = _smooth_field(rng, (nx, ny, 1), (6, 4, 1), 5.0)[0] / nx     # lateral <= 5 vox
    sF = surfaces(X2, Y2)
    sM = surfaces(X2 + dx_lat, Y2)
    F = np.empty((nz, ny, nx), np.float32)
    M = np.empty((nz, ny, nx), np.float32)
    for z0, z1 in _chunks(nz, 64):
        zz = ((np.arange(z0, z1, dtype=np.float32) + 0.5) / nz)[:, None, None]
        for out, s, shift in ((F, sF, 0.0), (M, sM, dz_ax)):
            z_eff = zz + shift
            I = np.full((z1 - z0, ny, nx), 0.05, np.float32)
            for k in range(10):
                I = np.where((z_eff >= s[k]) & (z_eff < s[k + 1]), refl[k], I)
            out[z0:z1] = I
    # fully developed speckle, independent for F and M, then log compression
    F = np.log1p(F * rng.exponential(1.0, size=F.shape).astype(np.float32))
    M = np.log1p(M * rng.exponential(1.0, size=M.shape).astype(np.float32))
    return F.astype(np.float32), M.astype(np.float32)


def make_pair(name: str, seed: int = 1, dims=None):
    """Raw (unnormalized) fixed and moving volumes, float32 [Nz, Ny, Nx]."""
    c = config(name, dims)
    rng = np.random.default_rng([seed, list(CONFIGS).index(name) + 1])
    d = c["dims"]
    if name == "C1":
        return _c1(rng, d)
    if name == "C2":
        return _c2(rng, d)
    if name == "C3":
        return _c3(rng, d, c["spacing"])
    if name == "C4":
        return _c4(rng, d)
    if name == "C5":
        return _c5(rng, d, c["spacing"])
    raise KeyError(name)


def make_params(shape, kind: str = "small", seed: int = 1) -> np.ndarray:
    """Control-point displacements (voxels), float64 array of the given params shape
    [ndim, Gz, Gy, Gx].  kind: 'zero'; 'small' = U(-2, 2) per node; 'large' = smooth
    field of amplitude <= 15 voxels over the node index grid (paper s.III-A)."""
    rng = np.random.default_rng([seed, 7919])
    shape = tuple(int(s) for s in shape)
    if kind == "zero":
        return np.zeros(shape)
    if kind == "small":
        return rng.uniform(-2.0, 2.0, size=shape)
    if kind == "large":
        nd, gz, gy, gx = shape
        out = np.zeros(shape)
        kz, ky, kx = np.meshgrid(np.arange(gz) / max(gz, 1), np.arange(gy) / max(gy, 1), np.arange(gx) / max(gx, 1),
                                 indexing="ij")
        for c in range(nd):
            acc = np.zeros((gz, gy, gx))
            for _ in range(3):
                f = rng.uniform(0.5, 2.0, 3)
                ph = rng.uniform(0, 2 * np.pi, 3)
                acc += np.sin(2 * np.pi * f[0] * kx + ph[0]) * np.sin(2 * np.pi * f[1] * ky + ph[1]) * \
                    np.cos(2 * np.pi * f[2] * kz + ph[2])
            acc *= 15.0 / max(1e-9, np.abs(acc).max())
            out[c] = acc
        return out
    raise KeyError(kind)
