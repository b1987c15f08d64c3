"""CPU fp64 oracle for SRWCR (arXiv 1804.05061) -- ctypes binding of srwcr_oracle.c.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  It shares no code with ``paper_1804_05061_b200`` (the product) and never
imports it.  See the header of ``srwcr_oracle.c`` for the paper passages each
function follows; readings where the paper is silent are listed in DESIGN.md s3.

All array arguments are numpy arrays; volumes are float32 x-fastest ``[Nz,Ny,Nx]``;
params are float64 SoA ``[ndim, Gz, Gy, Gx]`` (displacements in voxels).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "srwcr_oracle.c")
_LIB = os.path.join(_HERE, "libsrwcr_oracle.so")

# -O2, no FMA contraction: every product/sum rounds as written.
CFLAGS = ["-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (gcc).  Returns its path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64 * 3),
        ("L", ctypes.c_int32),
        ("nthreads", ctypes.c_int32),
        ("delta", ctypes.c_double * 3),
        ("kcells", ctypes.c_int64 * 3),
        ("eps_mass", ctypes.c_double),
        ("eps_sigma", ctypes.c_double),
        ("orientation", ctypes.c_int32),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        c_cfg = P(_Cfg)
        vp = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.orc_derived.argtypes = [c_cfg, P(i64), P(i64)]
        lib.orc_beta.argtypes = [ctypes.c_double, vp]
        lib.orc_taps.argtypes = [i64, ctypes.c_double, ctypes.c_int, P(i64), vp]
        lib.orc_normalize.argtypes = [vp, i64, ctypes.c_int32, vp]
        lib.orc_parzen.argtypes = [ctypes.c_double]
        lib.orc_parzen.restype = ctypes.c_double
        lib.orc_parzen_deriv.argtypes = [ctypes.c_double]
        lib.orc_parzen_deriv.restype = ctypes.c_double
        lib.orc_displacement.argtypes = [c_cfg, vp, i64, i64, i64, vp]
        lib.orc_sample.argtypes = [c_cfg, vp, vp, vp, vp]
        lib.orc_warp.argtypes = [c_cfg, vp, vp, i64, i64, vp, vp]
        lib.orc_joint_hist.argtypes = [c_cfg, vp, vp, vp, i64, i64, vp]
        lib.orc_value_table1.argtypes = [c_cfg, vp, vp, vp]
        lib.orc_value_table1.restype = ctypes.c_double
        lib.orc_dDdm_eq27.argtypes = [c_cfg, vp, vp, vp, vp, vp, i64, i64, vp]
        lib.orc_grad_chain.argtypes = [c_cfg, vp, vp, vp, i64, i64, vp]
        lib.orc_eval_literal.argtypes = [c_cfg, vp, vp, vp, vp]
        lib.orc_eval_literal.restype = ctypes.c_double
        lib.orc_moments.argtypes = [c_cfg, vp, vp, vp, i64, i64, vp, vp, vp]
        lib.orc_combine.argtypes = [c_cfg, vp, vp, vp, vp, vp, vp, vp, P(ctypes.c_double)]
        lib.orc_combine.restype = ctypes.c_double
        lib.orc_grad_moments.argtypes = [c_cfg, vp, vp, vp, vp, vp, vp, ctypes.c_double, i64, i64, vp, vp]
        lib.orc_eval_moments.argtypes = [c_cfg, vp, vp, vp, vp]
        lib.orc_bending.argtypes = [c_cfg, vp, vp]
        lib.orc_grad_moments_A.argtypes = [c_cfg, vp, vp, vp, vp, vp, vp, ctypes.c_double, i64, i64, vp, vp]
        lib.orc_bending.restype = ctypes.c_double
        lib.orc_eval_moments.restype = ctypes.c_double
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Problem:
    """Geometry of one SRWCR problem (SURVEY 8 conventions, readings c14-c16).

    dims: (Nx, Ny, Nz), Nz == 1 means 2-D.  L: maximal bin (bins = L+1).
    delta: control spacing per axis in voxels.  kcells: spatial cells per axis
    (0 = degenerate axis: one real region).  eps_*: retention thresholds (c12).
    orientation: 0 = moving image as the estimated image B, 1 = moving image as
    the model image A (Eq 20-21, App. II).
    """

    dims: tuple
    L: int
    delta: tuple
    kcells: tuple
    eps_mass: float = 1e-12
    eps_sigma: float = 1e-6
    nthreads: int = 0
    orientation: int = 0   # 0: moving image = estimated image B; 1: moving = model image A (F2)

    def cfg(self) -> _Cfg:
        c = _Cfg()
        for i in range(3):
            c.n[i] = int(self.dims[i])
            c.delta[i] = float(self.delta[i])
            c.kcells[i] = int(self.kcells[i])
        c.L = int(self.L)
        c.nthreads = int(self.nthreads)
        c.eps_mass = float(self.eps_mass)
        c.eps_sigma = float(self.eps_sigma)
        c.orientation = int(self.orientation)
        return c

    @property
    def ndim(self) -> int:
        return 2 if self.dims[2] == 1 else 3

    @property
    def bins(self) -> int:
        return self.L + 1

    def derived(self):
        """(G, K): control nodes per axis and regions per axis (x, y, z)."""
        G = (ctypes.c_int64 * 3)()
        K = (ctypes.c_int64 * 3)()
        c = self.cfg()
        _load().orc_derived(ctypes.byref(c), G, K)
        return tuple(G), tuple(K)

    @property
    def params_shape(self):
        G, _ = self.derived()
        return (self.ndim, G[2], G[1], G[0])

    @property
    def nregions(self) -> int:
        _, K = self.derived()
        return K[0] * K[1] * K[2]


# ------------------------------------------------------------------ primitives

def beta(t: float) -> np.ndarray:
    """Eq 8: (beta_0..beta_3)(t)."""
    w = np.zeros(4)
    _load().orc_beta(float(t), _p(w))
    return w


def taps(i: int, spacing: float, degenerate: bool = False):
    """Tap base and weights of voxel index i on a lattice (Eq 17 indices)."""
    b = ctypes.c_int64()
    w = np.zeros(4)
    _load().orc_taps(int(i), float(spacing), int(degenerate), ctypes.byref(b), _p(w))
    return int(b.value), w


def normalize(v: np.ndarray, L: int) -> np.ndarray:
    """Intensity normalization to [0, L], reading c1."""
    v = _f32(v)
    out = np.empty_like(v)
    _load().orc_normalize(_p(v), v.size, int(L), _p(out))
    return out


def parzen(t: float) -> float:
    """h(t), Eq 5."""
    return _load().orc_parzen(float(t))


def parzen_deriv(t: float) -> float:
    """dh/dt with the two-sided average at the kinks (reading c4)."""
    return _load().orc_parzen_deriv(float(t))


def displacement(pb: Problem, params, x: int, y: int, z: int) -> np.ndarray:
    """u(x) of the cubic B-spline FFD (Eq 17)."""
    c = pb.cfg()
    params = _f64(params)
    u = np.zeros(3)
    _load().orc_displacement(ctypes.byref(c), _p(params), int(x), int(y), int(z), _p(u))
    return u


def sample(pb: Problem, M, pos):
    """Trilinear sample of M at continuous position pos=(x,y,z) and its gradient (c1-c3)."""
    c = pb.cfg()
    M = _f32(M)
    p = _f64(np.asarray(pos, dtype=np.float64).reshape(3))
    m = np.zeros(1)
    g = np.zeros(3)
    _load().orc_sample(ctypes.byref(c), _p(M), _p(p), _p(m), _p(g))
    return float(m[0]), g


def warp(pb: Problem, M, params, z0: int = 0, z1: int | None = None):
    """m(x) = M(T(x)) and its spatial gradient for every voxel of slab [z0, z1)."""
    z1 = pb.dims[2] if z1 is None else z1
    c = pb.cfg()
    M = _f32(M)
    params = _f64(params)
    nx, ny = pb.dims[0], pb.dims[1]
    m = np.zeros((z1 - z0, ny, nx))
    g = np.zeros((z1 - z0, ny, nx, 3))
    _load().orc_warp(ctypes.byref(c), _p(M), _p(params), int(z0), int(z1), _p(m), _p(g))
    return m, g


# -------------------------------------------------------------- literal route

def joint_hist(pb: Problem, F, M, params, z0: int = 0, z1: int | None = None) -> np.ndarray:
    """Unnormalized Eq 3 joint histogram P[r, a, b] over slab [z0, z1)."""
    z1 = pb.dims[2] if z1 is None else z1
    c = pb.cfg()
    F, M, params = _f32(F), _f32(M), _f64(params)
    B = pb.bins
    P = np.zeros((pb.nregions, B, B))
    _load().orc_joint_hist(ctypes.byref(c), _p(F), _p(M), _p(params), int(z0), int(z1), _p(P))
    return P


def value_table1(pb: Problem, P):
    """Table I on P.  Returns (D, reg[R,6], mu_ra[R,B]).

    reg columns: p(r), sigma_r^2, mu_r, 1-CR_r, retained, Z."""
    c = pb.cfg()
    P = _f64(P)
    R, B = pb.nregions, pb.bins
    reg = np.zeros((R, 6))
    mura = np.zeros((R, B))
    D = _load().orc_value_table1(ctypes.byref(c), _p(P), _p(reg), _p(mura))
    return D, reg, mura


def dDdm_eq27(pb: Problem, F, M, params, reg, mura, z0: int = 0, z1: int | None = None):
    """Per-voxel dD/dM(y) by Eq 27, readings c4, c7."""
    z1 = pb.dims[2] if z1 is None else z1
    c = pb.cfg()
    F, M, params = _f32(F), _f32(M), _f64(params)
    out = np.zeros((z1 - z0, pb.dims[1], pb.dims[0]))
    _load().orc_dDdm_eq27(ctypes.byref(c), _p(F), _p(M), _p(params), _p(_f64(reg)), _p(_f64(mura)),
                          int(z0), int(z1), _p(out))
    return out


def grad_chain(pb: Problem, M, params, dDdm, z0: int = 0, z1: int | None = None):
    """Eq 16-17 chain rule over slab [z0, z1): dD/dPhi, shape params_shape."""
    z1 = pb.dims[2] if z1 is None else z1
    c = pb.cfg()
    M, params = _f32(M), _f64(params)
    grad = np.zeros(pb.params_shape)
    _load().orc_grad_chain(ctypes.byref(c), _p(M), _p(params), _p(_f64(dDdm)), int(z0), int(z1), _p(grad))
    return grad


def eval_literal(pb: Problem, F, M, params, want_grad: bool = True):
    """(D, grad) by the literal route (Eq 3 + Table I + Eq 27 + Eq 16-17)."""
    c = pb.cfg()
    F, M, params = _f32(F), _f32(M), _f64(params)
    grad = np.zeros(pb.params_shape) if want_grad else None
    D = _load().orc_eval_literal(ctypes.byref(c), _p(F), _p(M), _p(params), _p(grad))
    return D, grad


# --------------------------------------------------------------- moment route

def moments(pb: Problem, F, M, params, z0: int = 0, z1: int | None = None):
    """(N, S, Q)[R, B] over slab [z0, z1)."""
    z1 = pb.dims[2] if z1 is None else z1
    c = pb.cfg()
    F, M, params = _f32(F), _f32(M), _f64(params)
    R, B = pb.nregions, pb.bins
    N, S, Q = (np.zeros((R, B)) for _ in range(3))
    _load().orc_moments(ctypes.byref(c), _p(F), _p(M), _p(params), int(z0), int(z1), _p(N), _p(S), _p(Q))
    return N, S, Q


def combine(pb: Problem, N, S, Q):
    """SURVEY a7 combine.  Returns (D, alpha[R], beta[R], gamma[R,B], reg[R,6], Z)."""
    c = pb.cfg()
    R, B = pb.nregions, pb.bins
    al, be, ga, reg = np.zeros(R), np.zeros(R), np.zeros((R, B)), np.zeros((R, 6))
    Z = ctypes.c_double()
    D = _load().orc_combine(ctypes.byref(c), _p(_f64(N)), _p(_f64(S)), _p(_f64(Q)), _p(al), _p(be), _p(ga),
                            _p(reg), ctypes.byref(Z))
    return D, al, be, ga, reg, Z.value


def grad_moments(pb: Problem, F, M, params, alpha, beta_, gamma, Z, z0: int = 0, z1: int | None = None,
                 want_dDdm: bool = False):
    """SURVEY a8 per-voxel dD/dm + Eq 16-17 over slab [z0, z1).  Returns grad (and dD/dm)."""
    z1 = pb.dims[2] if z1 is None else z1
    c = pb.cfg()
    F, M, params = _f32(F), _f32(M), _f64(params)
    grad = np.zeros(pb.params_shape)
    dd = np.zeros((z1 - z0, pb.dims[1], pb.dims[0])) if want_dDdm else None
    _load().orc_grad_moments(ctypes.byref(c), _p(F), _p(M), _p(params), _p(_f64(alpha)), _p(_f64(beta_)),
                             _p(_f64(gamma)), float(Z), int(z0), int(z1), _p(dd), _p(grad))
    return (grad, dd) if want_dDdm else grad


def grad_moments_A(pb: Problem, F, M, params, N, gamma, reg, Z, z0: int = 0, z1: int | None = None,
                   want_dDdm: bool = False):
    """Orientation 1 (moving = model image A): per-voxel dD/dm (App. II Eq 31 in moment
    form, readings c4/c23) + Eq 16-17 over slab [z0, z1).  N, gamma, reg from combine()."""
    z1 = pb.dims[2] if z1 is None else z1
    c = pb.cfg()
    F, M, params = _f32(F), _f32(M), _f64(params)
    grad = np.zeros(pb.params_shape)
    dd = np.zeros((z1 - z0, pb.dims[1], pb.dims[0])) if want_dDdm else None
    _load().orc_grad_moments_A(ctypes.byref(c), _p(F), _p(M), _p(params), _p(_f64(N)), _p(_f64(gamma)),
                               _p(_f64(reg)), float(Z), int(z0), int(z1), _p(dd), _p(grad))
    return (grad, dd) if want_dDdm else grad


def eval_moments(pb: Problem, F, M, params, want_grad: bool = True):
    """(D, grad) by the moment route."""
    c = pb.cfg()
    F, M, params = _f32(F), _f32(M), _f64(params)
    grad = np.zeros(pb.params_shape) if want_grad else None
    D = _load().orc_eval_moments(ctypes.byref(c), _p(F), _p(M), _p(params), _p(grad))
    return D, grad


# ------------------------------------------------------------ bending energy

def bending(pb: Problem, params, want_grad: bool = True):
    """(C_p, dC_p/dphi): bending energy of Eq 1 (reading c19)."""
    c = pb.cfg()
    params = _f64(params)
    grad = np.zeros(pb.params_shape) if want_grad else None
    E = _load().orc_bending(ctypes.byref(c), _p(params), _p(grad))
    return E, grad
